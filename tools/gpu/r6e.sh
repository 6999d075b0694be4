mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "eight_vector or hot_quantizer or wide" 2>&1 | tail -3
QUIK_K1_FILL=0 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "eight_vector" 2>&1 | tail -2
