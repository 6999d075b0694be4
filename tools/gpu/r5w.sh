mkdir -p gpurun_out
for cfg in "0 0" "1 0" "1 1"; do
  set -- $cfg
  echo "FILL=$1 STAGES=$2"
  QUIK_K1_FILL=$1 QUIK_K1_STAGES=$2 timeout 300 python tools/k1_bench.py 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  try: r=json.loads(l)
  except Exception: print(l.strip()[:200]); continue
  print(r['name'], round(r['us'],1), round(r['frac'],3))"
done
