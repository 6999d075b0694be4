mkdir -p gpurun_out
: > gpurun_out/r3j.txt
for s in 0 1 2 4 -1; do
echo "splits=$s" >> gpurun_out/r3j.txt
QUIK_S4_SPLITS=$s timeout 120 python tools/cfg1_probe.py --m 1,16 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  r=json.loads(l); print(r['M'], 'b2b', round(r['graph_back_to_back_us'],2), 'cublas b2b', round(r['cublas_f16_back_to_back_us'],2))" >> gpurun_out/r3j.txt
done
cat gpurun_out/r3j.txt
