mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "every_tile or large_layer or stream_gemm or cfg1 or variants or sparse or gated" 2>&1 | tail -3 > gpurun_out/r2n.txt
timeout 600 python tools/sweep.py --only cfg > gpurun_out/r2n_sweep.jsonl 2>&1
cat gpurun_out/r2n.txt; cut -c 1-150 gpurun_out/r2n_sweep.jsonl
