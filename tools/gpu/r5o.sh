# K1: exact-fit 4-vector rows up to 512 threads, four hoisted outlier slots per thread at VPT <= 4
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "quantiz" 2>&1 | tail -2
for v in 0; do
  if [ $v = 0 ]; then unset QUIK_K1_VPT; else export QUIK_K1_VPT=$v; fi
  echo "QUIK_K1_VPT=$v"
  timeout 300 python tools/k1_bench.py 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  try: r=json.loads(l)
  except Exception: print(l.strip()[:200]); continue
  print(r['name'], round(r['us'],1), round(r['frac'],3))" | grep -i "down\|fc1\|qkvo\|up/gate"
  timeout 600 python tools/sweep.py --only "7B down" 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  try: r=json.loads(l)
  except Exception: continue
  print(r['name'], r['M'], round(r['step_ms']*1000,1), 'x', round(r['speedup_vs_f16'],2))"
done
