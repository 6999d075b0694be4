"""bench.py's reference arm on the CPU: one JSON line with the driver's contract keys
(the GPU arm is exercised on the B200 by the driver itself)."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

from oracle_lib import REF_SO

ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.skipif(not REF_SO.exists(), reason="oracle/_ref not built (needs /root/reference)")
def test_reference_arm_json_contract():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--workload", "cfg1",
                        "--steps", "3", "--warmup", "1", "--cpu-tokens", "4"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
    d = json.loads(line)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["steps"] == 3 and d["warmup"] == 1 and d["value"] > 0
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0


@pytest.mark.skipif(not REF_SO.exists(), reason="oracle/_ref not built (needs /root/reference)")
def test_cpu_leg_runs_reference_on_the_given_layer(tmp_path):
    """The GPU arm's cpu_baseline leg hands its own layer + sampled tokens to the
    reference (bench.py --layer-npz); the saved output is the reference's quik_matmul."""
    import numpy as np

    from oracle_lib import make_layer, ref

    rng = np.random.default_rng(5)
    L, x, _ = make_layer(rng, 6, 4096, 4096, 4, 128, heavy_cols=4, with_bias=False, checker=ref())
    lp, op = tmp_path / "layer.npz", tmp_path / "out.npy"
    np.savez(lp, x=x, base=L["base"], scales=L["scales"], wreduced=L["wreduced"],
             outlier_weights=L["outlier_weights"], idx=L["idx"], in_features=np.int64(4096),
             out_features=np.int64(4096), bits=np.int64(4))
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--workload", "cfg1",
                        "--steps", "2", "--warmup", "1", "--layer-npz", str(lp), "--ref-out", str(op)],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert d["config"]["sample_tokens"] == 6 and d["cpu_baseline"]["kind"] == "reference"
    st, want = ref().quik_matmul(L, x, 2)
    assert st == 0
    np.testing.assert_array_equal(np.load(op).view(np.uint32), want.view(np.uint32))


def test_bench_parity_bound_matches_tests():
    """bench.py's in-run parity bound is the tests' derived f16 bound."""
    import numpy as np

    import bench
    from oracle_lib import f16_output_bound

    rng = np.random.default_rng(3)
    want = rng.normal(size=(5, 40)).astype(np.float32)
    x = rng.normal(size=(5, 64)).astype(np.float32)
    idx = np.array([3, 9, 20])
    ow = rng.normal(size=(40, 3)).astype(np.float32)
    bias = rng.normal(size=40).astype(np.float32)
    L = dict(idx=idx, outlier_weights=ow, bias=bias)
    np.testing.assert_allclose(bench.f16_output_bound(want, x[:, idx], ow, bias), f16_output_bound(L, x, want),
                               rtol=1e-12)


def test_gpus_n_self_launches_ranks(monkeypatch):
    """python bench.py --gpus N (no torchrun env) launches N ranks through torchrun."""
    import bench

    seen = {}

    class R:
        returncode = 0

    def fake_run(cmd, *a, **k):
        seen["cmd"] = cmd
        return R()

    monkeypatch.setattr(bench.subprocess, "run", fake_run)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "5"])
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    with pytest.raises(SystemExit) as e:
        bench.main()
    assert e.value.code == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1" and cmd[-4:] == ["--gpus", "4", "--steps", "5"]
