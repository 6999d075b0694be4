mkdir -p gpurun_out
: > gpurun_out/r3y.txt
summ() { python -c "
import sys,json
for l in sys.stdin:
  try: r=json.loads(l)
  except Exception: print(l.strip()); continue
  print(r['name'], round(r['step_ms']*1000,1), 'f16', round(r['cublas_f16_ms']*1000,1), round(r['speedup_vs_f16'],2))"; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "stream or decode or gated or int4_weight" 2>&1 | tail -2 >> gpurun_out/r3y.txt
for sp in 0; do
echo "splits=$sp" >> gpurun_out/r3y.txt
QUIK_S4_SPLITS=$sp timeout 600 python tools/sweep.py --only "decode 70B up/gate M=1" 2>&1 | summ >> gpurun_out/r3y.txt
QUIK_S4_SPLITS=$sp timeout 600 python tools/sweep.py --only "decode 7B up" --opt-m 1,16 --falcon 2>&1 | grep -v "M=128\|M=512\|M=2048\|M=8192" | summ >> gpurun_out/r3y.txt
done
cat gpurun_out/r3y.txt
