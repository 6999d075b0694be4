mkdir -p gpurun_out
: > gpurun_out/r4e.txt
QUIK_K1_WIDE_CTA=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "quantizer" 2>&1 | tail -2 >> gpurun_out/r4e.txt
for w in 0 1; do
echo "WIDE_CTA=$w" >> gpurun_out/r4e.txt
QUIK_K1_WIDE_CTA=$w timeout 300 python tools/k1_bench.py 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  try: r=json.loads(l)
  except Exception: print(l.strip()); continue
  print(r['name'], round(r['us'],1), round(r['frac'],3))" >> gpurun_out/r4e.txt
QUIK_K1_WIDE_CTA=$w timeout 300 python tools/sweep.py --only "cfg2 7B down" 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  try: r=json.loads(l)
  except Exception: print(l.strip()); continue
  print(r['name'], round(r['step_ms']*1000,1), 'f16', round(r['cublas_f16_ms']*1000,1), round(r['speedup_vs_f16'],2))" >> gpurun_out/r4e.txt
done
cat gpurun_out/r4e.txt
