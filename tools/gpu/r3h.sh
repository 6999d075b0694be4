mkdir -p gpurun_out
: > gpurun_out/r3h.txt
summ() { python -c "
import sys,json
for l in sys.stdin:
  try: r=json.loads(l)
  except Exception: print(l.strip()); continue
  print(r['name'], round(r['step_ms']*1000,1), 'eager', round(r['step_eager_ms']*1000,1), 'f16', round(r['cublas_f16_ms']*1000,1), round(r['speedup_vs_f16'],2))"; }
echo "OLD" >> gpurun_out/r3h.txt
(cd ab_old && timeout 600 python tools/sweep.py --only "decode cfg1" 2>&1 | summ) >> gpurun_out/r3h.txt
(cd ab_old && timeout 600 python tools/sweep.py --only "decode 7B" 2>&1 | summ) >> gpurun_out/r3h.txt
for d in 0 4; do
echo "NEW dbg=$d" >> gpurun_out/r3h.txt
QUIK_S4_DBG=$d timeout 600 python tools/sweep.py --only "decode cfg1" 2>&1 | summ >> gpurun_out/r3h.txt
QUIK_S4_DBG=$d timeout 600 python tools/sweep.py --only "decode 7B" 2>&1 | summ >> gpurun_out/r3h.txt
done
cat gpurun_out/r3h.txt
