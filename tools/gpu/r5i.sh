mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_mlp_fused.py -q -x 2>&1 | tail -5
for sh in 7B 70B; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r5i_$sh.csv python tools/mlp_kernels.py $sh > /dev/null 2>&1
python - $sh <<'PY'
import csv,sys
rows=[r for r in csv.DictReader(l for l in open(f'gpurun_out/r5i_{sys.argv[1]}.csv') if not l.startswith('==')) if r.get('Metric Name')=='gpu__time_duration.sum']
print(sys.argv[1], [ (r['Kernel Name'][25:60], r['Metric Value']) for r in rows[-24:]][:8])
PY
done
timeout 300 python tools/mlp_bench.py 2>&1 | cut -c 1-330
