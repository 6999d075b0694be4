mkdir -p gpurun_out
: > gpurun_out/r3z.txt
summ() { python -c "
import sys,json
for l in sys.stdin:
  try: r=json.loads(l)
  except Exception: print(l.strip()); continue
  print(r['name'], round(r['step_ms']*1000,1), 'f16', round(r['cublas_f16_ms']*1000,1), round(r['speedup_vs_f16'],2))"; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullshape.py -q -x 2>&1 | tail -4 >> gpurun_out/r3z.txt
for fq in 1 0; do
echo "FUSEQ=$fq" >> gpurun_out/r3z.txt
QUIK_S4_FUSEQ=$fq timeout 600 python tools/sweep.py --only "decode 70B up/gate M=1" --opt-m 1 --falcon 2>&1 | grep "M=1\"" | summ >> gpurun_out/r3z.txt
QUIK_S4_FUSEQ=$fq timeout 120 python tools/cfg1_probe.py --m 1 2>&1 | cut -c 1-200 >> gpurun_out/r3z.txt
done
cat gpurun_out/r3z.txt
