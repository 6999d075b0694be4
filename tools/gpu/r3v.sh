mkdir -p gpurun_out
: > gpurun_out/r3v.txt
summ() { python -c "
import sys,json
for l in sys.stdin:
  try: r=json.loads(l)
  except Exception: print(l.strip()); continue
  print(r['name'], round(r['step_ms']*1000,1), 'f16', round(r['cublas_f16_ms']*1000,1), round(r['speedup_vs_f16'],2))"; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "stream or decode" 2>&1 | tail -2 >> gpurun_out/r3v.txt
for s4 in 1 0; do
echo "stream4=$s4" >> gpurun_out/r3v.txt
QUIK_STREAM4=$s4 timeout 600 python tools/sweep.py --only "M=32" 2>&1 | summ >> gpurun_out/r3v.txt
done
cat gpurun_out/r3v.txt
