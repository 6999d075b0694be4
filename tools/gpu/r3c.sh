mkdir -p gpurun_out
: > gpurun_out/r3c.txt
for rep in 1 2; do
for pf in 0 1; do
echo "prefetch=$pf" >> gpurun_out/r3c.txt
QUIK_S4_PREFETCH=$pf timeout 300 python tools/sweep.py --only "zzz" --falcon --opt-m 1,16 2>&1 | grep "M=1\"\|M=16\"" | python -c "
import sys,json
for l in sys.stdin:
  r=json.loads(l); print(r['name'], round(r['step_ms']*1000,1), round(r['speedup_vs_f16'],2))" >> gpurun_out/r3c.txt
QUIK_S4_PREFETCH=$pf timeout 300 python tools/cfg1_probe.py --m 1,16 >> gpurun_out/r3c.txt 2>&1
done
done
cat gpurun_out/r3c.txt | cut -c 1-200
