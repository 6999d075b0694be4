# FILL K1: next row's outlier overwrite before barrier B (barrier F merged into B)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mlp_fused.py -q -x -k "quantiz or eight_vector or fused_mlp or gated" 2>&1 | tail -2
QUIK_K1_STAGES=2 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "eight_vector or hot_quantizer" 2>&1 | tail -1
for i in 1 2; do
timeout 300 python tools/k1_bench.py 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  try: r=json.loads(l)
  except Exception: print(l.strip()[:200]); continue
  print(r['name'], round(r['us'],1), round(r['frac'],3))" | grep "cfg3\|7B down\|Falcon-180B fc1"
done
