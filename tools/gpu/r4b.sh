mkdir -p gpurun_out
: > gpurun_out/r4b.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "quantizer or wide" 2>&1 | tail -3 >> gpurun_out/r4b.txt
timeout 300 python tools/k1_bench.py --only fc2 2>&1 | cut -c 1-200 >> gpurun_out/r4b.txt
timeout 600 python tools/sweep.py --only "fc2" 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  try: r=json.loads(l)
  except Exception: print(l.strip()); continue
  print(r['name'], round(r['step_ms']*1000,1), 'f16', round(r['cublas_f16_ms']*1000,1), round(r['speedup_vs_f16'],2))" >> gpurun_out/r4b.txt
cat gpurun_out/r4b.txt
