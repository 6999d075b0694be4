mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_mlp_fused.py -q -x 2>&1 | tail -25 > gpurun_out/r5e_mlp_tests.txt
cat gpurun_out/r5e_mlp_tests.txt
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/r5e_pytest.txt
cat gpurun_out/r5e_pytest.txt
