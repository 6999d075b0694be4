mkdir -p gpurun_out
: > gpurun_out/r3o.txt
summ() { python -c "
import sys,json
for l in sys.stdin:
  try: r=json.loads(l)
  except Exception: print(l.strip()); continue
  print(r['name'], round(r['step_ms']*1000,1), 'k1', round(r['k1_ms']*1000,1), 'gemm', round(r['gemm_ms']*1000,1), 'f16', round(r['cublas_f16_ms']*1000,1), round(r['speedup_vs_f16'],2))"; }
for rep in 1 2; do
echo OLD >> gpurun_out/r3o.txt
(cd ab_old && timeout 600 python tools/sweep.py --only "fc2" 2>&1 | summ) >> gpurun_out/r3o.txt
echo NEW >> gpurun_out/r3o.txt
timeout 600 python tools/sweep.py --only "fc2" 2>&1 | summ >> gpurun_out/r3o.txt
done
cat gpurun_out/r3o.txt
