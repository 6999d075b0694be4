mkdir -p gpurun_out
: > gpurun_out/r3p.txt
summ() { python -c "
import sys,json
for l in sys.stdin:
  try: r=json.loads(l)
  except Exception: print(l.strip()); continue
  print(r['name'], round(r['step_ms']*1000,1), 'k1', round(r['k1_ms']*1000,1), 'gemm', round(r['gemm_ms']*1000,1), 'f16', round(r['cublas_f16_ms']*1000,1), round(r['speedup_vs_f16'],2))"; }
for rep in 1 2; do
for pdl in 1 0; do
echo "PDL=$pdl" >> gpurun_out/r3p.txt
QUIK_K1_WIDE_PDL=$pdl timeout 600 python tools/sweep.py --only "fc2" 2>&1 | summ >> gpurun_out/r3p.txt
done; done
cat gpurun_out/r3p.txt
