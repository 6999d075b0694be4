mkdir -p gpurun_out
: > gpurun_out/r3f.txt
for env in "QUIK_S4_PREFETCH=1" "QUIK_S4_PREFETCH=0" "QUIK_S4_PREFETCH=1"; do
echo "$env" >> gpurun_out/r3f.txt
env $env timeout 600 python tools/sweep.py --only "decode" 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  try: r=json.loads(l)
  except Exception: print(l.strip()); continue
  print(r['name'], round(r['step_ms']*1000,1), 'eager', round(r['step_eager_ms']*1000,1), 'f16', round(r['cublas_f16_ms']*1000,1), round(r['speedup_vs_f16'],2))" >> gpurun_out/r3f.txt
done
cat gpurun_out/r3f.txt
