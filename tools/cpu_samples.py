"""SURVEY.md §8(d) CPU reference sample points: the reference's own quik_matmul
(oracle/_ref = proj/src compiled unchanged, OpenMP on every host core) on the cfg4
OPT-66B fc1 layer (9216 -> 36864, 256 outliers, W4A4) at M = 1, 16, 256, 2048 tokens,
median of 3 calls after one warm-up, with the per-stage split. Bench infrastructure
(the reference is the thing measured; nothing of the B200 path runs here).

  OMP_NUM_THREADS=$(nproc) python tools/cpu_samples.py > profiles/r2_cpu_samples.jsonl
"""
import json
import os
import statistics
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "tests"))
from oracle_lib import ref  # noqa: E402  (the reference's compiled sources)


def main(ms=(1, 16, 256, 2048), K=9216, N=36864, O=256, bits=4, seed=66):
    r = ref()
    rng = np.random.default_rng(seed)
    W = rng.standard_normal((N, K), dtype=np.float32)
    x_all = rng.standard_normal((max(ms), K), dtype=np.float32)
    heavy = np.unique(rng.integers(0, K, size=O))
    x_all[:, heavy] *= 50.0
    x_all = x_all.astype(np.float16).astype(np.float32)
    idx = r.select_outliers(x_all, O)
    q = r.rtn_quantize_weights(W, idx, bits)
    del W
    L = dict(in_features=K, out_features=N, bits=bits, act_bits=bits, base=q["base"], scales=q["scales"],
             wreduced=q["wreduced"], outlier_weights=q["outlier_weights"], idx=idx, bias=None)
    h, keep = r.layer_create(L)
    for M in ms:
        x = np.ascontiguousarray(x_all[:M])
        t = np.zeros(6)
        r.layer_forward(h, x, N, 2)
        per, stages = [], []
        for _ in range(3):
            t0 = time.perf_counter()
            st, _ = r.layer_forward(h, x, N, 2, t)
            per.append(time.perf_counter() - t0)
            stages.append(t.copy())
            assert st == 0
        med = statistics.median(per)
        print(json.dumps(dict(layer="OPT-66B fc1 9216->36864 O=256 W4A4", M=M, ms=1e3 * med,
                              tops=2.0 * M * N * K / med / 1e12, cores=int(os.environ.get("OMP_NUM_THREADS",
                                                                                          os.cpu_count())),
                              stage_ms=dict(zip(["split", "quantize", "int_matmul", "fp_matmul", "dequantize", "add"],
                                                np.median(stages, axis=0).round(3).tolist())),
                              impl="reference quik_matmul V3 (oracle/_ref)")), flush=True)
    r.layer_destroy(h)


if __name__ == "__main__":
    os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count() or 1))
    main()
