timeout 400 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --workload cfg5-up --no-cpu > gpurun_out/bench_cfg5.json 2>> gpurun_out/bench.err
timeout 300 python tools/sweep.py > gpurun_out/sweep.json 2> gpurun_out/sweep.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-cublas --no-clocks --soak-s 0 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:quik_gemm --launch-skip 3 -c 1 -o gpurun_out/gemm_cfg3 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-cublas --no-clocks --soak-s 0 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:quantize --launch-skip 3 -c 1 -o gpurun_out/k1_cfg3 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-cublas --no-clocks --soak-s 0 > /dev/null 2>&1
python -c "import __graft_entry__ as g; g.smoke()"
