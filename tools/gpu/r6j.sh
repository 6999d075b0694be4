mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "wide" 2>&1 | tail -1
QUIK_K1_WIDE_STAGES=2 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "wide" 2>&1 | tail -1
for i in 1 2; do
timeout 300 python tools/k1_bench.py 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  try: r=json.loads(l)
  except Exception: print(l.strip()[:200]); continue
  print(r['name'], round(r['us'],1), round(r['frac'],3))" | grep "fc2"
done
