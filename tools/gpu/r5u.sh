mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_mlp_fused.py -q 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "quantiz or gated" 2>&1 | tail -2
timeout 300 python tools/mlp_bench.py 2>&1 | cut -c 1-200
