# K1 L1M variant (masks re-read from L1 per row, no overwrite barrier) vs FILL
mkdir -p gpurun_out
QUIK_K1_FILL=3 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "quantiz" 2>&1 | tail -1
for f in 1 3 1 3; do
echo "FILL=$f"
QUIK_K1_FILL=$f timeout 300 python tools/k1_bench.py 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  try: r=json.loads(l)
  except Exception: print(l.strip()[:200]); continue
  print(r['name'], round(r['us'],1), round(r['frac'],3))" | grep "cfg3\|7B down\|Falcon-180B fc1"
done
