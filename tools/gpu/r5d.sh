# prescaled sliced down K1: tests, MLP bench (sliced vs hot prescaled), launch lists
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_mlp_fused.py -q -x 2>&1 | tail -25 > gpurun_out/r5d_mlp_tests.txt
cat gpurun_out/r5d_mlp_tests.txt
timeout 300 python tools/mlp_bench.py > gpurun_out/r5d_mlp.jsonl 2>&1
QUIK_K1_PRE_SLICE_COLS=1000000 timeout 300 python tools/mlp_bench.py > gpurun_out/r5d_mlp_hotpre.jsonl 2>&1
cut -c 1-330 gpurun_out/r5d_mlp.jsonl gpurun_out/r5d_mlp_hotpre.jsonl
for v in sliced hot; do
  if [ $v = hot ]; then export QUIK_K1_PRE_SLICE_COLS=1000000; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r5d_launches_$v.csv python tools/mlp_kernels.py > /dev/null 2>&1
  python - $v <<'PY'
import csv, sys
rows=[r for r in csv.DictReader(l for l in open(f'gpurun_out/r5d_launches_{sys.argv[1]}.csv') if not l.startswith('==')) if r.get('Metric Name')=='gpu__time_duration.sum']
print(sys.argv[1])
for r in rows[-24:]:
    print(r['ID'], r['Kernel Name'][:70], r['Metric Value'])
PY
done
