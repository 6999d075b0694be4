mkdir -p gpurun_out
python -c "from paper_2310_09259_b200 import build as b; b.build_tests()" > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/r2o_pytest.txt
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/r2o_bench.json 2> gpurun_out/r2o_bench.err
cat gpurun_out/r2o_pytest.txt; tail -c 600 gpurun_out/r2o_bench.json; tail -3 gpurun_out/r2o_bench.err
