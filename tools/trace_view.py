"""Summarises a QUIK_GEMM_TRACE timeline dump (gemm.cu: kTraceTiles x kTraceSlots
globaltimer stamps per leader CTA) into per-phase averages in microseconds."""
import sys

import numpy as np

T, S = 64, 16
a = np.fromfile(sys.argv[1], dtype=np.int64).reshape(-1, T, S)
import os

if os.path.exists(sys.argv[1] + ".w"):  # W4 clock64 stamps of cluster 0: MMA k-blocks, widening pairs
    w = np.fromfile(sys.argv[1] + ".w", dtype=np.int64).reshape(2, 128, 8)
    m = w[0][w[0][:, 0] > 0]
    if m.size:
        d = np.diff(m[:, :5], axis=1)
        print("mma k-block (clk): [0-1] %.0f  [1-2] %.0f  [2-3] %.0f  [3-4] %.0f  period %.0f (n=%d)"
              % (*np.median(d, axis=0), np.median(np.diff(m[:, 0])), len(m)))
    t = w[1][w[1][:, 0] > 0]
    if t.size:
        d = np.diff(t[:, :6], axis=1)
        print("widen k-block (clk): next-load %.0f  slot-wait %.0f  alu+sttm %.0f  st-wait %.0f  arrive %.0f  period %.0f (n=%d)"
              % (*np.median(d, axis=0), np.median(np.diff(t[:, 0])), len(t)))
valid = a[:, :, 0] > 0
t0 = a[:, :, 0][valid].min()
names = {"mma tempty wait": (0, 1), "mma int[0:h] issue": (1, 2), "mma tconv+outlier": (2, 3),
         "mma int[h:] issue": (3, 4), "epi tint wait": (6, 7), "epi pass1": (7, 8), "epi tfin wait": (8, 9),
         "epi pass2": (9, 10)}
for k, (i, j) in names.items():
    m = valid & (a[:, :, j] > 0) & (a[:, :, i] > 0)
    d = (a[:, :, j] - a[:, :, i])[m] / 1e3
    if d.size:
        print(f"{k:22s} mean {d.mean():7.2f} us  p50 {np.median(d):7.2f}  max {d.max():7.2f}  n={d.size}")
fw = a[:, :, 5][valid] / 1e3
print(f"{'mma full-wait / tile':22s} mean {fw.mean():7.2f} us")
rw = a[:, :, 11][valid] / 1e3
print(f"{'mma W4 ready-wait/tile':22s} mean {rw.mean():7.2f} us")
wv = valid & (a[:, :, 14] > 0)
if wv.any():
    print(f"{'widen tile span':22s} mean {((a[:, :, 15] - a[:, :, 14])[wv] / 1e3).mean():7.2f} us")
    print(f"{'widen full4-wait/tile':22s} mean {(a[:, :, 12][wv] / 1e3).mean():7.2f} us")
    print(f"{'widen aempty-wait/tile':22s} mean {(a[:, :, 13][wv] / 1e3).mean():7.2f} us")
c0 = np.nonzero(valid[0])[0]
print("cluster 0 tile starts (us):", ((a[0, c0, 0] - t0) / 1e3).round(1).tolist())
print("cluster 0 mma issue end (us):", ((a[0, c0, 4] - t0) / 1e3).round(1).tolist())
print("cluster 0 epi pass2 end (us):", ((a[0, c0, 10] - t0) / 1e3).round(1).tolist())
end = a[:, :, 10].max()
print("kernel span (first tile start -> last epilogue end): %.1f us" % ((end - t0) / 1e3))
