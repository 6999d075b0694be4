mkdir -p gpurun_out
summ() { python -c "
import sys,json
for l in sys.stdin:
  try: r=json.loads(l)
  except Exception: print(l.strip()); continue
  if r['M'] > 32: continue
  print(r['name'], round(r['step_ms']*1000,1), 'eager', round(r['step_eager_ms']*1000,1), 'f16', round(r['cublas_f16_ms']*1000,1), round(r['speedup_vs_f16'],2))"; }
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "stream or decode or int4_weight_mode or gated or sharded" 2>&1 | tail -2 > gpurun_out/r3i.txt
echo NEW >> gpurun_out/r3i.txt
timeout 600 python tools/sweep.py --only "decode" --opt-m 1,16 --falcon 2>&1 | summ >> gpurun_out/r3i.txt


echo OLD >> gpurun_out/r3i.txt
(cd ab_old && timeout 600 python tools/sweep.py --only "decode 7B" 2>&1 | summ) >> gpurun_out/r3i.txt
cat gpurun_out/r3i.txt
