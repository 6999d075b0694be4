// GPTQ / SparseGPT weight quantisation on the device (reference
// gptq_quantize quantizer.cpp:292-297, sparsegpt_joint :299-337, prepare_state :101-146,
// quantize_column :171-191, finish_state :148-169, Hessian :193-240), FP64 throughout
// like the reference:
//
//   Hd = H[perm][perm] + lambda I,  lambda = damping * trace(H) / K     (host-summed trace)
//   C  = upper Cholesky factor of Hd^-1   (own blocked FP64 Cholesky / triangular inverse)
//   per-row scales from the base columns (optional clip search), fixed before the recursion
//   for each base column j (blocks of 64): q = round_away(w_j / s), err = (w_j - q s) / C_jj,
//   w_t -= err C_jt for t > j  (in-block: sequential per row; beyond the block: one GEMM)
//
// The panel kernel keeps the reference's per-element arithmetic (IEEE double mul / sub /
// div, floor(|t| + 0.5) rounding, stable 2:4 saliency order); the trailing update of a
// block and the Hessian X^T X run on a hand-written FP64 tensor-core GEMM
// (mma.sync.m8n8k4.f64, dgemm_kernel below), and so do the blocked Cholesky factorisations
// and the triangular inverse around their diagonal-block / panel kernels: the sums run in
// a different order than the reference's loops, so results agree with the reference to
// FP64 rounding (codes / scales / masks bit-identical on the test cases, outlier weights
// to float rounding). No cuBLAS / cuSOLVER.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "kernels.h"

namespace quikb200 {

namespace {

constexpr int kPanel = 64;     // columns per block
constexpr int kPanelRows = 128;  // rows (threads) per panel CTA

// quantize_to_grid (quantizer.cpp:17-22): nearest, ties away from zero, clamped
__device__ __forceinline__ int q_grid(double value, double inv_scale, int maxq) {
  const double t = __dmul_rn(value, inv_scale);
  double q = floor(__dadd_rn(fabs(t), 0.5));
  if (q > maxq) q = maxq;
  return static_cast<int>(t < 0.0 ? -q : q);
}

__global__ void permute_hessian_kernel(const double* __restrict__ h, const int* __restrict__ perm, double lam,
                                       int64_t K, double* __restrict__ hd) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < K * K;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e / K, j = e % K;
    double v = h[static_cast<int64_t>(perm[i]) * K + perm[j]];
    if (i == j) v = __dadd_rn(v, lam);
    hd[e] = v;
  }
}

__global__ void diag_kernel(const double* __restrict__ h, int64_t K, double* __restrict__ d) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < K;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    d[i] = h[i * K + i];
}

__global__ void permute_w_kernel(const float* __restrict__ w, const int* __restrict__ perm, int64_t N, int64_t K,
                                 double* __restrict__ wd) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < N * K;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = e / K, j = e % K;
    wd[e] = static_cast<double>(w[r * K + perm[j]]);
  }
}

// prepare_state's per-row scales (quantizer.cpp:131-143) incl. clip_search (:266-290):
// one thread per row, sequential sums in the reference's order
__global__ void scales_kernel(const double* __restrict__ wd, int64_t N, int64_t K, int64_t kb, int maxq,
                              int use_clipping, double* __restrict__ sd, float* __restrict__ sf) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= N) return;
  const double* row = wd + r * K;
  double amax = 0.0;
  for (int64_t j = 0; j < kb; ++j) amax = fmax(amax, static_cast<double>(fabsf(static_cast<float>(row[j]))));
  double s = 1.0;
  if (amax != 0.0) {
    float best_c = 1.0f;
    if (use_clipping && kb > 0) {
      double best_err = INFINITY;
      for (int step = 0; step <= 50; ++step) {
        const float c = static_cast<float>(__dadd_rn(0.50, __dmul_rn(0.01, static_cast<double>(step))));
        const double scale = __ddiv_rn(__dmul_rn(static_cast<double>(c), amax), static_cast<double>(maxq));
        const double inv = __ddiv_rn(1.0, scale);
        double err = 0.0;
        for (int64_t j = 0; j < kb; ++j) {
          const float v = static_cast<float>(row[j]);
          const double dq = __dmul_rn(static_cast<double>(q_grid(v, inv, maxq)), scale);
          const double d = __dsub_rn(static_cast<double>(v), dq);
          err = __dadd_rn(err, __dmul_rn(d, d));
        }
        if (err <= best_err) {  // ties resolve toward larger c
          best_err = err;
          best_c = c;
        }
      }
    }
    s = __ddiv_rn(__dmul_rn(static_cast<double>(best_c), amax), static_cast<double>(maxq));
  }
  sd[r] = s;
  sf[r] = static_cast<float>(s);
}

// One block of kPanel base columns [j0, j0 + jb) for kPanelRows rows: the reference's
// quantize_column loop restricted to the block (updates of columns inside the block,
// in column order), recording err for the trailing DGEMM. sparse: the 2:4 mask of each
// full group is decided at its first column from the current weights (w^2 / C_gg^2,
// stable order; quantizer.cpp:311-327).
__global__ void __launch_bounds__(kPanelRows) panel_kernel(double* __restrict__ wd, int64_t N, int64_t K, int64_t kb,
                                                            const double* __restrict__ c, int64_t j0, int jb,
                                                            const double* __restrict__ sd, int maxq,
                                                            int8_t* __restrict__ q, double* __restrict__ err,
                                                            int sparse, uint8_t* __restrict__ mask) {
  extern __shared__ double s_dyn[];
  double* s_c = s_dyn;                           // [jb][jb] block of C (upper part used)
  double* s_w = s_dyn + kPanel * kPanel;         // [kPanelRows][kPanel + 1]
  const int tid = threadIdx.x;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * kPanelRows;
  for (int e = tid; e < jb * jb; e += blockDim.x) {
    const int a = e / jb, b = e % jb;
    s_c[a * kPanel + b] = c[(j0 + a) * K + j0 + b];
  }
  for (int e = tid; e < kPanelRows * jb; e += blockDim.x) {
    const int rr = e / jb, b = e % jb;
    const int64_t r = r0 + rr;
    s_w[rr * (kPanel + 1) + b] = r < N ? wd[r * K + j0 + b] : 0.0;
  }
  __syncthreads();
  const int64_t r = r0 + tid;
  if (r >= N) return;
  double* w = s_w + tid * (kPanel + 1);
  const double scale = sd[r];
  const double inv = __ddiv_rn(1.0, scale);
  const int64_t full_groups = kb / 4;
  uint8_t keep4 = 0xF;
  for (int a = 0; a < jb; ++a) {
    const int64_t j = j0 + a;
    bool kept = true;
    if (sparse && j / 4 < full_groups) {
      if (j % 4 == 0) {
        double sal[4];
        for (int g = 0; g < 4; ++g) {
          const double cgg = s_c[(a + g) * kPanel + a + g];
          const double wv = w[a + g];
          sal[g] = __ddiv_rn(__dmul_rn(wv, wv), __dmul_rn(cgg, cgg));
        }
        keep4 = 0;
        for (int g = 0; g < 4; ++g) {
          int rank = 0;  // position in the stable ascending order
          for (int h = 0; h < 4; ++h) rank += (sal[h] < sal[g]) || (sal[h] == sal[g] && h < g);
          if (rank >= 2) keep4 |= 1u << g;
        }
      }
      kept = (keep4 >> (j % 4)) & 1u;
      mask[r * kb + j] = kept ? 1 : 0;
    } else if (sparse) {
      mask[r * kb + j] = 1;  // trailing remainder group stays dense (quantizer.cpp:308, :332-334)
    }
    double dq = 0.0;
    int qv = 0;
    if (kept) {
      qv = q_grid(w[a], inv, maxq);
      dq = __dmul_rn(static_cast<double>(qv), scale);
    }
    q[r * kb + j] = static_cast<int8_t>(qv);
    const double d = s_c[a * kPanel + a];
    const double e = __ddiv_rn(__dsub_rn(w[a], dq), d);
    err[r * kPanel + a] = e;
    for (int t = a + 1; t < jb; ++t) w[t] = __dsub_rn(w[t], __dmul_rn(e, s_c[a * kPanel + t]));
  }
  for (int a = jb; a < kPanel; ++a) err[r * kPanel + a] = 0.0;
}

// finish_state (quantizer.cpp:148-169): pack, wreduced, outlier weights
__global__ void finish_kernel(const double* __restrict__ wd, const int8_t* __restrict__ q, const float* __restrict__ sf,
                              int64_t N, int64_t K, int64_t kb, int bits, uint8_t* __restrict__ base,
                              float* __restrict__ wreduced, float* __restrict__ ow) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= N) return;
  const int8_t* qr = q + r * kb;
  long long qsum = 0;
  for (int64_t j = 0; j < kb; ++j) qsum += qr[j];
  wreduced[r] = static_cast<float>(__dmul_rn(static_cast<double>(sf[r]), static_cast<double>(qsum)));
  if (bits == 4) {
    const int64_t rb = (kb + 1) / 2;
    for (int64_t b = 0; b < rb; ++b) {
      const int lo = qr[2 * b] + 8;
      const int hi = 2 * b + 1 < kb ? qr[2 * b + 1] + 8 : 0;
      base[r * rb + b] = static_cast<uint8_t>(lo | (hi << 4));
    }
  } else {
    for (int64_t j = 0; j < kb; ++j) base[r * kb + j] = static_cast<uint8_t>(qr[j]);
  }
  for (int64_t j = 0; j < K - kb; ++j) ow[r * (K - kb) + j] = static_cast<float>(wd[r * K + kb + j]);
}

__global__ void to_double_kernel(const float* __restrict__ x, int64_t n, double* __restrict__ y) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    y[e] = static_cast<double>(x[e]);
}

unsigned blocks_for(int64_t n) { return static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 148 * 16)); }

// ---------------------------------------------------------------- FP64 tensor-core GEMM
// C(m, n) += alpha * sum_k A(m, k) * B(k, n) over strided operands
//   A(m, k) = A[m * a_m + k * a_k],  B(k, n) = B[k * b_k + n * b_n],  C(m, n) = C[m * ldc + n]
// (the strides express the transposes: the Hessian X^T X and the GPTQ trailing update
// W[:, j1:] -= E * C[j0:j1, j1:]). 64 x 64 tiles per CTA, 16-deep K slices staged in
// shared memory, four warps of 32 x 32 each as 4 x 4 tiles of
// mma.sync.m8n8k4.f64 (sm_80+ DMMA; FP64 accumulate, every product and sum IEEE
// double). Replaces cuBLAS DGEMM: a different summation order, FP64 either way.
constexpr int kDT = 64, kDK = 16;

__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(128) dgemm_kernel(int64_t M, int64_t N, int64_t K, double alpha,
                                                    const double* __restrict__ A, int64_t a_m, int64_t a_k,
                                                    const double* __restrict__ B, int64_t b_k, int64_t b_n,
                                                    double* __restrict__ C, int64_t ldc) {
  __shared__ double sa[kDT][kDK + 1];  // [m][k]
  __shared__ double sb[kDK][kDT + 1];  // [k][n]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;  // fragment row group / thread in group
  const int64_t m0 = static_cast<int64_t>(blockIdx.y) * kDT, n0 = static_cast<int64_t>(blockIdx.x) * kDT;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int64_t k0 = 0; k0 < K; k0 += kDK) {
    for (int e = tid; e < kDT * kDK; e += 128) {
      const int r = e / kDK, kk = e % kDK;  // A: consecutive threads walk k
      const int64_t m = m0 + r, k = k0 + kk;
      sa[r][kk] = (m < M && k < K) ? A[m * a_m + k * a_k] : 0.0;
      const int kk2 = e / kDT, c = e % kDT;  // B: consecutive threads walk n
      const int64_t k2 = k0 + kk2, n = n0 + c;
      sb[kk2][c] = (k2 < K && n < N) ? B[k2 * b_k + n * b_n] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < kDK; ks += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = sa[wm + 8 * i + g][ks + t4];  // A(8x4) row: [g][t4]
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = sb[ks + t4][wn + 8 * j + g];  // B(4x8) col: [t4][g]
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j], af[i], bf[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {  // D(8x8): [g][2 t4 + h]
        const int64_t m = m0 + wm + 8 * i + g, n = n0 + wn + 8 * j + 2 * t4 + h;
        if (m < M && n < N) C[m * ldc + n] = __dadd_rn(C[m * ldc + n], __dmul_rn(alpha, acc[i][j][h]));
      }
}

// ---------------------------------------------------------------- Cholesky and inverse (FP64)
// Row-major, blocks of kCb columns, right-looking: factor the diagonal block (one CTA,
// the reference's column recursion, quantizer.cpp:33-48), solve the panel below it (one
// thread per row), update the trailing matrix with the FP64 tensor-core GEMM.
constexpr int kCb = 32;

// Diagonal block A[j0:j0+jb, j0:j0+jb] -> its lower Cholesky factor (in place); *bad = 1
// when a pivot is not positive and finite (the reference's "not positive definite").
__global__ void chol_diag_kernel(double* __restrict__ a, int64_t K, int64_t j0, int jb, int* __restrict__ bad) {
  __shared__ double s[kCb][kCb + 1];
  const int t = threadIdx.x;  // row of the block
  for (int c = 0; c < jb; ++c) s[t][c] = t < jb ? a[(j0 + t) * K + j0 + c] : 0.0;
  __syncthreads();
  for (int j = 0; j < jb; ++j) {
    if (t == j) {
      double v = s[j][j];
      for (int k = 0; k < j; ++k) v = __dsub_rn(v, __dmul_rn(s[j][k], s[j][k]));
      if (!(v > 0.0) || !isfinite(v)) {
        *bad = 1;
        v = 1.0;
      }
      s[j][j] = __dsqrt_rn(v);
    }
    __syncthreads();
    if (t > j && t < jb) {
      double v = s[t][j];
      for (int k = 0; k < j; ++k) v = __dsub_rn(v, __dmul_rn(s[t][k], s[j][k]));
      s[t][j] = __ddiv_rn(v, s[j][j]);
    }
    __syncthreads();
  }
  if (t < jb)
    for (int c = 0; c < jb; ++c) a[(j0 + t) * K + j0 + c] = c <= t ? s[t][c] : 0.0;
}

// Panel below the diagonal block: row i: x = A[i, j0:j0+jb] L11^-T (forward substitution).
__global__ void chol_panel_kernel(double* __restrict__ a, int64_t K, int64_t j0, int jb) {
  __shared__ double l[kCb][kCb + 1];
  for (int e = threadIdx.x; e < jb * jb; e += blockDim.x) l[e / jb][e % jb] = a[(j0 + e / jb) * K + j0 + e % jb];
  __syncthreads();
  const int64_t i = j0 + jb + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= K) return;
  double x[kCb];
#pragma unroll
  for (int j = 0; j < kCb; ++j) {
    if (j >= jb) break;
    double v = a[i * K + j0 + j];
    for (int k = 0; k < j; ++k) v = __dsub_rn(v, __dmul_rn(x[k], l[j][k]));
    x[j] = __ddiv_rn(v, l[j][j]);
    a[i * K + j0 + j] = x[j];
  }
}

// One block row of Y = L^-1: Y[i0:i0+ib, :] = L_ii^-1 R, R = (rows of I) - L[i, :i0] Y[:i0, :]
// already formed in y; one thread per column, forward substitution over the ib rows.
__global__ void trinv_rows_kernel(const double* __restrict__ l, double* __restrict__ y, int64_t K, int64_t i0,
                                  int ib) {
  __shared__ double s[kCb][kCb + 1];
  for (int e = threadIdx.x; e < ib * ib; e += blockDim.x) s[e / ib][e % ib] = l[(i0 + e / ib) * K + i0 + e % ib];
  __syncthreads();
  const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= i0 + ib) return;  // Y is lower triangular: columns > the block's last row stay 0
  double x[kCb];
#pragma unroll
  for (int r = 0; r < kCb; ++r) {
    if (r >= ib) break;
    double v = y[(i0 + r) * K + c];
    for (int k = 0; k < r; ++k) v = __dsub_rn(v, __dmul_rn(s[r][k], x[k]));
    x[r] = __ddiv_rn(v, s[r][r]);
    y[(i0 + r) * K + c] = x[r];
  }
}

__global__ void zero_upper_kernel(double* __restrict__ a, int64_t K) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < K * K;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    if (e % K > e / K) a[e] = 0.0;
}

__global__ void identity_kernel(double* __restrict__ y, int64_t K) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < K * K;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    y[e] = (e / K == e % K) ? 1.0 : 0.0;
}

__global__ void transpose_kernel(const double* __restrict__ x, double* __restrict__ y, int64_t K) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < K * K;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    y[(e % K) * K + e / K] = x[e];
}

cudaError_t dgemm(int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t a_m, int64_t a_k,
                  const double* B, int64_t b_k, int64_t b_n, double* C, int64_t ldc, cudaStream_t st);

// Lower Cholesky factor of the symmetric positive definite A (row-major, in place; the
// upper triangle is left zero). Returns 1 if A is not numerically positive definite.
int potrf_lower(double* a, int64_t K, int* d_bad, std::string* msg) {
  if (cudaMemset(d_bad, 0, sizeof(int)) != cudaSuccess) { *msg = "cholesky: memset failed"; return 4; }
  for (int64_t j0 = 0; j0 < K; j0 += kCb) {
    const int jb = static_cast<int>(std::min<int64_t>(kCb, K - j0));
    chol_diag_kernel<<<1, kCb>>>(a, K, j0, jb, d_bad);
    const int64_t below = K - j0 - jb;
    if (below > 0) {
      chol_panel_kernel<<<static_cast<unsigned>((below + 127) / 128), 128>>>(a, K, j0, jb);
      // A22 -= L21 L21^T (the whole square; only its lower part is read later)
      const double* l21 = a + (j0 + jb) * K + j0;
      if (dgemm(below, below, jb, -1.0, l21, K, 1, l21, 1, K, a + (j0 + jb) * K + j0 + jb, K, nullptr) !=
          cudaSuccess) {
        *msg = "cholesky: trailing GEMM failed";
        return 4;
      }
    }
  }
  // zero the strict upper triangle (the trailing updates wrote both halves)
  zero_upper_kernel<<<blocks_for(K * K), 256>>>(a, K);
  int bad = 0;
  if (cudaMemcpy(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess) { *msg = "cholesky: failed"; return 4; }
  return bad ? 1 : 0;
}

cudaError_t dgemm(int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t a_m, int64_t a_k,
                  const double* B, int64_t b_k, int64_t b_n, double* C, int64_t ldc, cudaStream_t st) {
  if (M == 0 || N == 0 || K == 0) return cudaSuccess;
  const dim3 grid(static_cast<unsigned>((N + kDT - 1) / kDT), static_cast<unsigned>((M + kDT - 1) / kDT));
  dgemm_kernel<<<grid, 128, 0, st>>>(M, N, K, alpha, A, a_m, a_k, B, b_k, b_n, C, ldc);
  return cudaGetLastError();
}

struct DevMem {
  std::vector<void*> ptrs;
  ~DevMem() {
    for (void* p : ptrs) cudaFree(p);
  }
  template <typename T>
  T* alloc(int64_t n) {
    void* p = nullptr;
    if (cudaMalloc(&p, static_cast<size_t>(std::max<int64_t>(n, 1)) * sizeof(T)) != cudaSuccess) return nullptr;
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
};

}  // namespace

// status: 0 ok, 1 invalid argument, 3 numerical (not positive definite), 4 CUDA / library
int gptq_quantize_device(const GptqArgs& a, std::string* msg) {
  const int64_t N = a.N, K = a.K, O = a.n_out, kb = K - O;
  if (a.bits != 4 && a.bits != 8) { *msg = "weight bits must be 4 or 8"; return 1; }
  if (N < 0 || K <= 0 || O < 0 || O > K) { *msg = "gptq: bad shape"; return 1; }
  if (N == 0) return 0;
  const int maxq = (1 << (a.bits - 1)) - 1;
  // OutlierSet::permutation (calibration.cpp:69-91): base columns ascending, then outliers
  std::vector<int> perm;
  perm.reserve(static_cast<size_t>(K));
  {
    std::vector<uint8_t> is_out(static_cast<size_t>(K), 0);
    for (int64_t i = 0; i < O; ++i) {
      const int64_t c = a.outlier_idx[i];
      if (c < 0 || c >= K || is_out[c] || (i > 0 && a.outlier_idx[i - 1] >= c)) {
        *msg = "gptq: outlier indices must be sorted, unique and in range";
        return 1;
      }
      is_out[c] = 1;
    }
    for (int64_t j = 0; j < K; ++j)
      if (!is_out[j]) perm.push_back(static_cast<int>(j));
    for (int64_t i = 0; i < O; ++i) perm.push_back(static_cast<int>(a.outlier_idx[i]));
  }
  DevMem m;
  int* d_perm = m.alloc<int>(K);
  double* d_h = m.alloc<double>(K * K);
  double* d_c = m.alloc<double>(K * K);
  double* d_diag = m.alloc<double>(K);
  float* d_w = m.alloc<float>(N * K);
  double* d_wd = m.alloc<double>(N * K);
  double* d_sd = m.alloc<double>(N);
  float* d_sf = m.alloc<float>(N);
  int8_t* d_q = m.alloc<int8_t>(N * std::max<int64_t>(kb, 1));
  double* d_err = m.alloc<double>(N * kPanel);
  uint8_t* d_mask = a.sparse ? m.alloc<uint8_t>(N * std::max<int64_t>(kb, 1)) : nullptr;
  const int64_t rb = a.bits == 4 ? (kb + 1) / 2 : kb;
  uint8_t* d_base = m.alloc<uint8_t>(N * std::max<int64_t>(rb, 1));
  float* d_wr = m.alloc<float>(N);
  float* d_ow = m.alloc<float>(N * std::max<int64_t>(O, 1));
  if (!d_perm || !d_h || !d_c || !d_diag || !d_w || !d_wd || !d_sd || !d_sf || !d_q || !d_err || !d_base || !d_wr ||
      !d_ow || (a.sparse && !d_mask)) {
    *msg = "gptq: device allocation failed";
    return 4;
  }
#define GQ_CUDA(x)                                                              \
  do {                                                                          \
    cudaError_t _e = (x);                                                       \
    if (_e != cudaSuccess) { *msg = std::string("gptq: ") + cudaGetErrorString(_e); return 4; } \
  } while (0)
  GQ_CUDA(cudaMemcpy(d_perm, perm.data(), K * sizeof(int), cudaMemcpyHostToDevice));
  GQ_CUDA(cudaMemcpy(d_h, a.hessian_sum, K * K * sizeof(double), cudaMemcpyDefault));
  GQ_CUDA(cudaMemcpy(d_w, a.w, N * K * sizeof(float), cudaMemcpyDefault));
  // lambda = damping * trace / dim (quantizer.cpp:215-219), trace summed in index order
  diag_kernel<<<blocks_for(K), 256>>>(d_h, K, d_diag);
  std::vector<double> diag(static_cast<size_t>(K));
  GQ_CUDA(cudaMemcpy(diag.data(), d_diag, K * sizeof(double), cudaMemcpyDeviceToHost));
  double trace = 0.0;
  for (double v : diag) trace += v;
  const double lam = a.damping * trace / static_cast<double>(K);
  permute_hessian_kernel<<<blocks_for(K * K), 256>>>(d_h, d_perm, lam, K, d_c);
  GQ_CUDA(cudaGetLastError());

  // C = upper Cholesky factor of Hd^-1 (quantizer.cpp:50-99): L = chol(Hd), Y = L^-1,
  // Hd^-1 = Y^T Y, Lx = chol(Hd^-1), C = Lx^T -- every step hand-written FP64 (diagonal
  // block / panel kernels + the FP64 tensor-core GEMM)
  double* d_y = m.alloc<double>(K * K);
  int* d_bad = m.alloc<int>(1);
  if (!d_y || !d_bad) { *msg = "gptq: device allocation failed"; return 4; }
  {
    const int st = potrf_lower(d_c, K, d_bad, msg);
    if (st == 1) { *msg = "Hessian is not positive definite after damping; increase the damping fraction"; return 3; }
    if (st) return st;
  }
  identity_kernel<<<blocks_for(K * K), 256>>>(d_y, K);
  for (int64_t i0 = 0; i0 < K; i0 += kCb) {
    const int ib = static_cast<int>(std::min<int64_t>(kCb, K - i0));
    if (i0 > 0) {  // R = I[i rows] - L[i, :i0] Y[:i0, :(i0 + ib)]
      if (dgemm(ib, i0 + ib, i0, -1.0, d_c + i0 * K, K, 1, d_y, K, 1, d_y + i0 * K, K, nullptr) != cudaSuccess) {
        *msg = "gptq: triangular-inverse GEMM failed";
        return 4;
      }
    }
    trinv_rows_kernel<<<static_cast<unsigned>((i0 + ib + 127) / 128), 128>>>(d_c, d_y, K, i0, ib);
  }
  GQ_CUDA(cudaMemset(d_c, 0, K * K * sizeof(double)));
  if (dgemm(K, K, K, 1.0, d_y, 1, K, d_y, K, 1, d_c, K, nullptr) != cudaSuccess) {  // Y^T Y
    *msg = "gptq: inverse GEMM failed";
    return 4;
  }
  {
    const int st = potrf_lower(d_c, K, d_bad, msg);
    if (st == 1) { *msg = "inverse Hessian is not positive definite"; return 3; }
    if (st) return st;
  }
  transpose_kernel<<<blocks_for(K * K), 256>>>(d_c, d_y, K);  // C = Lx^T (row-major upper)
  GQ_CUDA(cudaGetLastError());
  GQ_CUDA(cudaMemcpy(d_c, d_y, K * K * sizeof(double), cudaMemcpyDeviceToDevice));

  permute_w_kernel<<<blocks_for(N * K), 256>>>(d_w, d_perm, N, K, d_wd);
  scales_kernel<<<static_cast<unsigned>((N + 127) / 128), 128>>>(d_wd, N, K, kb, maxq, a.use_clipping, d_sd, d_sf);
  GQ_CUDA(cudaGetLastError());

  const int smem = static_cast<int>((kPanel * kPanel + kPanelRows * (kPanel + 1)) * sizeof(double));
  GQ_CUDA(cudaFuncSetAttribute(panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  for (int64_t j0 = 0; j0 < kb; j0 += kPanel) {
    const int jb = static_cast<int>(std::min<int64_t>(kPanel, kb - j0));
    panel_kernel<<<static_cast<unsigned>((N + kPanelRows - 1) / kPanelRows), kPanelRows, smem>>>(
        d_wd, N, K, kb, d_c, j0, jb, d_sd, maxq, d_q, d_err, a.sparse, d_mask);
    GQ_CUDA(cudaGetLastError());
    const int64_t j1 = j0 + jb;
    if (j1 < K) {
      // W[:, j1:] -= E[N x jb] * C[j0:j1, j1:]   (row-major; the FP64 tensor-core GEMM)
      if (dgemm(N, K - j1, jb, -1.0, d_err, kPanel, 1, d_c + j0 * K + j1, K, 1, d_wd + j1, K, nullptr) != cudaSuccess) {
        *msg = "gptq: trailing-update GEMM failed";
        return 4;
      }
    }
  }
  finish_kernel<<<static_cast<unsigned>((N + 127) / 128), 128>>>(d_wd, d_q, d_sf, N, K, kb, a.bits, d_base, d_wr,
                                                                  d_ow);
  GQ_CUDA(cudaGetLastError());
  GQ_CUDA(cudaMemcpy(a.base, d_base, N * rb, cudaMemcpyDefault));
  GQ_CUDA(cudaMemcpy(a.scales, d_sf, N * sizeof(float), cudaMemcpyDefault));
  GQ_CUDA(cudaMemcpy(a.wreduced, d_wr, N * sizeof(float), cudaMemcpyDefault));
  if (O) GQ_CUDA(cudaMemcpy(a.outlier_weights, d_ow, N * O * sizeof(float), cudaMemcpyDefault));
  if (a.sparse && a.mask) GQ_CUDA(cudaMemcpy(a.mask, d_mask, N * kb, cudaMemcpyDefault));
  GQ_CUDA(cudaDeviceSynchronize());
#undef GQ_CUDA
  return 0;
}

// H += x^T x in FP64 (Hessian::accumulate, quantizer.cpp:193-213): x f32 [T][K]
int hessian_accumulate_device(const float* x, int64_t T, int64_t K, double* h, std::string* msg) {
  if (T == 0 || K == 0) return 0;
  DevMem m;
  float* d_x = m.alloc<float>(T * K);
  double* d_xd = m.alloc<double>(T * K);
  if (!d_x || !d_xd) { *msg = "hessian: device allocation failed"; return 4; }
  if (cudaMemcpy(d_x, x, T * K * sizeof(float), cudaMemcpyDefault) != cudaSuccess) { *msg = "hessian: copy failed"; return 4; }
  to_double_kernel<<<blocks_for(T * K), 256>>>(d_x, T * K, d_xd);
  // H[i][j] += sum_t X[t][i] X[t][j]: A(i, t) = X[t][i], B(t, j) = X[t][j] (FP64 tensor-core GEMM)
  if (dgemm(K, K, T, 1.0, d_xd, 1, K, d_xd, K, 1, h, K, nullptr) != cudaSuccess) {
    *msg = "hessian: GEMM failed";
    return 4;
  }
  if (cudaDeviceSynchronize() != cudaSuccess) { *msg = "hessian: kernel failed"; return 4; }
  return 0;
}

}  // namespace quikb200
