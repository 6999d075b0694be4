mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "stream or decode or int4_weight_mode or gated or sharded" 2>&1 | tail -3 > gpurun_out/r3e.txt
timeout 300 python -m pytest tests/test_gpu_fullshape.py -q -x -k "opt or cfg1" 2>&1 | tail -3 >> gpurun_out/r3e.txt
timeout 600 python tools/sweep.py --only "decode" --opt-m 1,16 --falcon 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  try: r=json.loads(l)
  except Exception: print(l.strip()); continue
  if r['M'] > 32: continue
  print(r['name'], round(r['step_ms']*1000,1), 'f16', round(r['cublas_f16_ms']*1000,1), round(r['speedup_vs_f16'],2))" >> gpurun_out/r3e.txt
timeout 300 python tools/cfg1_probe.py --m 1,16 | cut -c 1-200 >> gpurun_out/r3e.txt 2>&1
cat gpurun_out/r3e.txt
