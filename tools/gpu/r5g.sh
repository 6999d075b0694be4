mkdir -p gpurun_out
for d in 0 256 512; do
QUIK_W4_DBG=$d timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r5g_$d.csv python tools/mlp_kernels.py 7B > /dev/null 2>&1
python - $d <<'PY'
import csv,sys
rows=[r for r in csv.DictReader(l for l in open(f'gpurun_out/r5g_{sys.argv[1]}.csv') if not l.startswith('==')) if r.get('Metric Name')=='gpu__time_duration.sum']
print('dbg', sys.argv[1], [ (r['Kernel Name'][25:60], r['Metric Value']) for r in rows[-24:-12]][:4])
PY
done
