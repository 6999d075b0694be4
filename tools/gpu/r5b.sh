# fused MLP block (down K1 reduction in the gated epilogue): new tests, GPU suite, MLP bench, bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_mlp_fused.py -q -x 2>&1 | tail -25 > gpurun_out/r5b_mlp_tests.txt
cat gpurun_out/r5b_mlp_tests.txt
timeout 300 python tools/mlp_bench.py > gpurun_out/r5b_mlp.jsonl 2>&1
timeout 300 python tools/mlp_bench.py --tokens 16 > gpurun_out/r5b_mlp16.jsonl 2>&1
cut -c 1-420 gpurun_out/r5b_mlp.jsonl gpurun_out/r5b_mlp16.jsonl
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/r5b_pytest.txt
timeout 600 python bench.py > gpurun_out/r5b_bench.json 2> gpurun_out/r5b_bench.err
cat gpurun_out/r5b_pytest.txt; head -c 400 gpurun_out/r5b_bench.json; tail -3 gpurun_out/r5b_bench.err
