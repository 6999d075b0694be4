mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullshape.py -q -x 2>&1 | tail -3 > gpurun_out/r3s.txt
summ() { python -c "
import sys,json
for l in sys.stdin:
  try: r=json.loads(l)
  except Exception: print(l.strip()); continue
  print(r['name'], round(r['step_ms']*1000,1), 'f16', round(r['cublas_f16_ms']*1000,1), round(r['speedup_vs_f16'],2))"; }
for mm in 128 0 256; do
echo "W4_MID_M=$mm" >> gpurun_out/r3s.txt
QUIK_W4_MID_M=$mm timeout 600 python tools/sweep.py --only "xx" --opt-m 64,128,256 2>&1 | summ >> gpurun_out/r3s.txt
done
cat gpurun_out/r3s.txt
