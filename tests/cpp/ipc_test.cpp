// C++ multi-process test of the fused all-gather through CUDA IPC (quik::b200::
// FusedShardedLayer): two processes (fork, before any CUDA call), both on GPU 0 — CUDA
// IPC maps allocations between processes on one device as well — each own half of the
// output rows; the IPC handles and a barrier go over pipes. Both ranks' [M][N] outputs
// must equal the unsharded layer's bit for bit over several steps (both buffers).
// Exit code = number of failed checks (both ranks).
#include <sys/wait.h>
#include <unistd.h>

#include <cstdio>
#include <random>
#include <vector>

#include <cuda_fp16.h>

#include "quik_b200.hpp"

namespace Q = quik::b200;

static void write_all(int fd, const void* p, size_t n) {
  const char* c = static_cast<const char*>(p);
  while (n) {
    const ssize_t w = write(fd, c, n);
    if (w <= 0) _exit(90);
    c += w;
    n -= static_cast<size_t>(w);
  }
}
static void read_all(int fd, void* p, size_t n) {
  char* c = static_cast<char*>(p);
  while (n) {
    const ssize_t r = read(fd, c, n);
    if (r <= 0) _exit(91);
    c += r;
    n -= static_cast<size_t>(r);
  }
}

static int run(int rank, int to_peer, int from_peer) {
  const int world = 2;
  auto exchange = [&](const std::vector<uint8_t>& mine) {
    const uint64_t n = mine.size();
    write_all(to_peer, &n, 8);
    write_all(to_peer, mine.data(), n);
    uint64_t m = 0;
    read_all(from_peer, &m, 8);
    std::vector<uint8_t> theirs(m);
    read_all(from_peer, theirs.data(), m);
    std::vector<std::vector<uint8_t>> all(2);
    all[rank] = mine;
    all[1 - rank] = theirs;
    return all;
  };
  auto barrier = [&]() {
    const char c = 1;
    char d = 0;
    write_all(to_peer, &c, 1);
    read_all(from_peer, &d, 1);
  };
  int fails = 0;
  for (auto [M, K, N, bits, O] : std::vector<std::tuple<int64_t, int64_t, int64_t, int, int64_t>>{
           {300, 1024, 768, 4, 32}, {16, 2048, 1024, 4, 64}, {200, 1024, 512, 8, 16}}) {
    std::mt19937 rng(static_cast<uint32_t>(7 + M));
    std::normal_distribution<float> nd(0.f, 1.f);
    Q::FpMatrix w(N, K), x(M, K);
    for (float& v : w.data) v = 0.5f * nd(rng);
    for (float& v : x.data) v = nd(rng);
    std::vector<int64_t> idx;
    for (int64_t i = 0; i < O; ++i) idx.push_back(i * (K / O) + 3);
    Q::QuikLinearLayer L;
    L.outliers = Q::OutlierSet::from_indices(K, idx);
    L.weights = Q::rtn_quantize_weights(w, L.outliers, bits);
    L.act_bits = bits;
    L.bias.resize(N);
    for (float& b : L.bias) b = 0.1f * nd(rng);
    std::vector<__half> xh(M * K);
    for (size_t i = 0; i < xh.size(); ++i) xh[i] = __float2half(x.data[i]);
    void *dx = nullptr, *dy = nullptr;
    cudaMalloc(&dx, xh.size() * 2);
    cudaMalloc(&dy, M * N * 2);
    cudaMemcpy(dx, xh.data(), xh.size() * 2, cudaMemcpyHostToDevice);
    Q::DeviceLayer full(L);
    full.forward_device(dx, QUIK_F16, M, dy, QUIK_F16);
    std::vector<uint16_t> want(M * N), got(M * N);
    cudaMemcpy(want.data(), dy, want.size() * 2, cudaMemcpyDeviceToHost);
    Q::FusedShardedLayer sh(L, rank, world, M, exchange);
    for (int step = 0; step < 4; ++step) {
      const void* y = sh.forward(dx, QUIK_F16, M);
      cudaDeviceSynchronize();
      barrier();  // every rank's peer stores of this step are complete
      cudaMemcpy(got.data(), y, got.size() * 2, cudaMemcpyDeviceToHost);
      if (got != want) {
        std::printf("rank %d: M=%lld K=%lld N=%lld step %d differs from the unsharded layer\n", rank,
                    static_cast<long long>(M), static_cast<long long>(K), static_cast<long long>(N), step);
        ++fails;
      }
      barrier();  // readers done before the buffer's next writes
    }
    cudaFree(dx);
    cudaFree(dy);
  }
  std::printf("ipc_test rank %d: %d failure(s)\n", rank, fails);
  return fails;
}

int main() {
  int a[2], b[2];  // a: rank 0 -> 1, b: rank 1 -> 0
  if (pipe(a) || pipe(b)) return 99;
  const pid_t pid = fork();
  if (pid == 0) {
    close(a[1]);
    close(b[0]);
    _exit(run(1, b[1], a[0]));
  }
  close(a[0]);
  close(b[1]);
  const int f0 = run(0, a[1], b[0]);
  int status = 0;
  waitpid(pid, &status, 0);
  const int f1 = WIFEXITED(status) ? WEXITSTATUS(status) : 100;
  return f0 + f1;
}
