mkdir -p gpurun_out
: > gpurun_out/r3x.txt
summ() { python -c "
import sys,json
for l in sys.stdin:
  try: r=json.loads(l)
  except Exception: print(l.strip()); continue
  print(r['name'], round(r['step_ms']*1000,1), 'f16', round(r['cublas_f16_ms']*1000,1), round(r['speedup_vs_f16'],2))"; }
for sp in 0 1 2 3 -1; do
echo "splits=$sp" >> gpurun_out/r3x.txt
QUIK_S4_SPLITS=$sp timeout 600 python tools/sweep.py --only "decode 70B up/gate M=1" 2>&1 | summ >> gpurun_out/r3x.txt
QUIK_S4_SPLITS=$sp timeout 600 python tools/sweep.py --only "xx" --opt-m 1 2>&1 | summ >> gpurun_out/r3x.txt
done
cat gpurun_out/r3x.txt
