# K1 FILL variant (outlier columns overwritten in the ring row; no lane-mask registers): parity + 70B / 7B down timing
mkdir -p gpurun_out
QUIK_K1_FILL=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "quantiz" 2>&1 | tail -2
for cfg in "0 0" "1 0" "1 1" "0 1"; do
  set -- $cfg
  echo "FILL=$1 STAGES=$2"
  QUIK_K1_FILL=$1 QUIK_K1_STAGES=$2 timeout 300 python tools/k1_bench.py 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  try: r=json.loads(l)
  except Exception: print(l.strip()[:200]); continue
  print(r['name'], round(r['us'],1), round(r['frac'],3))" | grep -i "down\|fc1"
done
