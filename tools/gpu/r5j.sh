# warp-per-row K1: parity, K1 timings (warp vs hot), GPU suite, bench, sweep of the cfg shapes
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "quantiz" 2>&1 | tail -15
for v in 1 2; do
echo "K1_VARIANT=$v"
QUIK_K1_VARIANT=$v timeout 300 python tools/k1_bench.py 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  try: r=json.loads(l)
  except Exception: print(l.strip()[:200]); continue
  print(r['name'], round(r['us'],1), round(r['frac'],3))"
done
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
timeout 600 python bench.py > gpurun_out/r5j_bench.json 2> gpurun_out/r5j_bench.err
python -c "
import json; r=json.loads(open('gpurun_out/r5j_bench.json').read().strip().splitlines()[-1]); print(r['value'], r['fp16_cublas']['speedup_step'], r['parity']['status'], r['quantizer']['ms_median'], r['quantizer']['frac'])"
tail -3 gpurun_out/r5j_bench.err
