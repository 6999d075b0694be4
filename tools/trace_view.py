"""Summarises a QUIK_GEMM_TRACE timeline dump (gemm.cu: kTraceTiles x kTraceSlots
globaltimer stamps per leader CTA) into per-phase averages in microseconds."""
import sys

import numpy as np

T, S = 64, 12
a = np.fromfile(sys.argv[1], dtype=np.int64)
a = a.reshape(-1, T, S)
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
c0 = np.nonzero(valid[0])[0]
print("cluster 0 tile starts (us):", ((a[0, c0, 0] - t0) / 1e3).round(1).tolist())
print("cluster 0 mma issue end (us):", ((a[0, c0, 4] - t0) / 1e3).round(1).tolist())
print("cluster 0 epi pass2 end (us):", ((a[0, c0, 10] - t0) / 1e3).round(1).tolist())
end = a[:, :, 10].max()
print("kernel span (first tile start -> last epilogue end): %.1f us" % ((end - t0) / 1e3))
