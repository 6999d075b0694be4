# round-2 final validation: full GPU suite, smoke, default bench, launch list, sweeps, ncu of the wide K1 and decode kernels
mkdir -p gpurun_out
python -c "from paper_2310_09259_b200 import build as b; b.build_tests()" > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -8 > gpurun_out/r3u_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r3u_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/r3u_bench.json 2> gpurun_out/r3u_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r3u_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-cublas --soak-s 0 --no-clocks > /dev/null 2>&1
timeout 1500 python tools/sweep.py --falcon > gpurun_out/r3u_sweep.jsonl 2> gpurun_out/r3u_sweep.err
timeout 900 python tools/sweep.py --weights int4 --opt-m 1,16,64,128,256,2048 > gpurun_out/r3u_sweep_int4.jsonl 2>> gpurun_out/r3u_sweep.err
timeout 300 python tools/k1_bench.py > gpurun_out/r3u_k1.jsonl 2>&1
cat gpurun_out/r3u_pytest.txt gpurun_out/r3u_smoke.txt; tail -c 900 gpurun_out/r3u_bench.json; tail -3 gpurun_out/r3u_bench.err; wc -l gpurun_out/r3u_*.jsonl
