mkdir -p gpurun_out
: > gpurun_out/r3d.txt
for s4 in 1 0; do
echo "stream4=$s4" >> gpurun_out/r3d.txt
QUIK_STREAM4=$s4 timeout 600 python tools/sweep.py --only "decode" 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  try: r=json.loads(l)
  except Exception: print(l.strip()); continue
  print(r['name'], round(r['step_ms']*1000,1), 'f16', round(r['cublas_f16_ms']*1000,1), round(r['speedup_vs_f16'],2))" >> gpurun_out/r3d.txt
done
cat gpurun_out/r3d.txt
