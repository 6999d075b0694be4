mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r5f_launches_7b.csv python tools/mlp_kernels.py 7B > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.DictReader(l for l in open('gpurun_out/r5f_launches_7b.csv') if not l.startswith('==')) if r.get('Metric Name')=='gpu__time_duration.sum']
for r in rows[-24:]:
    print(r['ID'], r['Kernel Name'][:70], r['Metric Value'])
PY
for i in 1 2; do timeout 300 python tools/mlp_bench.py --only 7B 2>&1 | cut -c 1-330; done
