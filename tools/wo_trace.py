"""Summarises a QUIK_WO_TRACE dump (wo.cu: CTA 0, per item [producer issue, widening
start (quadrant 0), widening end quadrants 0-3, MMA a_full seen, MMA committed]
globaltimer stamps) in microseconds."""
import sys

import numpy as np

a = np.fromfile(sys.argv[1], dtype=np.int64).reshape(256, 8)
n = int((a[:, 0] > 0).sum())
a = a[:n].astype(np.float64)
t0 = a[0, 0]
r = np.where(a > 0, (a - t0) / 1e3, np.nan)
for i in range(min(n, int(sys.argv[2]) if len(sys.argv) > 2 else 48)):
    print(f"item {i:3d}: issue {r[i,0]:7.2f} widen {r[i,1]:7.2f} -> q0 {r[i,2]:7.2f} q1 {r[i,3]:7.2f} "
          f"q2 {r[i,4]:7.2f} q3 {r[i,5]:7.2f}  mma seen {r[i,6]:7.2f} issued {r[i,7]:7.2f}")
w = a[:, 1] > 0
print("widen duration (q0) mean %.2f us" % ((a[w, 2] - a[w, 1]).mean() / 1e3))
print("last quadrant end -> mma seen mean %.2f us" % ((a[w, 6] - a[w, 2:6].max(axis=1)).mean() / 1e3))
print("mma seen -> issued mean %.2f us" % ((a[w, 7] - a[w, 6]).mean() / 1e3))
print("items/us over the CTA: %.2f" % (n / ((a[:, 7].max() - t0) / 1e3)))
