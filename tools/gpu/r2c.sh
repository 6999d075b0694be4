# round-2 GPU session C: INT4-weight (TMEM-widened) GEMM: GPU suite + bench + shape sweep
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "every_tile or large_layer or stream_gemm or cfg1 or golden or variants or gated" 2>&1 | tail -30 > gpurun_out/r2c_quick.txt
cat gpurun_out/r2c_quick.txt
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/r2c_pytest.txt
timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err
cat gpurun_out/r2c_pytest.txt; tail -c 1500 gpurun_out/r2c_bench.json; tail -5 gpurun_out/r2c_bench.err
