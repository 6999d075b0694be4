# fused MLP block, stats in a separate GEMM mode: tests, MLP bench, launch list, GPU suite, bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_mlp_fused.py -q -x 2>&1 | tail -25 > gpurun_out/r5c_mlp_tests.txt
cat gpurun_out/r5c_mlp_tests.txt
timeout 300 python tools/mlp_bench.py > gpurun_out/r5c_mlp.jsonl 2>&1
timeout 300 python tools/mlp_bench.py --tokens 16 > gpurun_out/r5c_mlp16.jsonl 2>&1
cut -c 1-460 gpurun_out/r5c_mlp.jsonl gpurun_out/r5c_mlp16.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r5c_mlp_launches.csv python tools/mlp_kernels.py > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.DictReader(open('gpurun_out/r5c_mlp_launches.csv')) if r.get('Metric Name')=='gpu__time_duration.sum']
for r in rows[-20:]:
    print(r['ID'], r['Kernel Name'][:60], r['Metric Value'])
PY
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/r5c_pytest.txt
timeout 600 python bench.py > gpurun_out/r5c_bench.json 2> gpurun_out/r5c_bench.err
cat gpurun_out/r5c_pytest.txt; head -c 300 gpurun_out/r5c_bench.json; tail -3 gpurun_out/r5c_bench.err
