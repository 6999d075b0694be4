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
