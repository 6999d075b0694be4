mkdir -p gpurun_out
for sh in 7B 70B; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r6m_launches_$sh.csv python tools/mlp_kernels.py $sh > /dev/null 2>&1
python - $sh <<'PY'
import csv,sys
rows=[r for r in csv.DictReader(l for l in open(f'gpurun_out/r6m_launches_{sys.argv[1]}.csv') if not l.startswith('==')) if r.get('Metric Name')=='gpu__time_duration.sum'][-24:]
f=[float(r['Metric Value'])/1000 for r in rows]
avg=lambda L:[round(sum(x[k] for x in L)/len(L),1) for k in range(4)]
fu=avg([f[i:i+4] for i in range(0,12,4)]); pl=avg([f[i:i+4] for i in range(12,24,4)])
print(sys.argv[1],'fused', fu, round(sum(fu),1), '| two forwards', pl, round(sum(pl),1))
PY
done
for i in 1 2; do timeout 300 python tools/mlp_bench.py --only 70B 2>&1 | cut -c 1-200; done
