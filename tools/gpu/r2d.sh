# round-2 GPU session D: INT4 GEMM x16 widening, IPC test, quick sweep, bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ipc.py -q -x -k "every_tile or large_layer or stream_gemm or cfg1 or golden or variants or gated or ipc" 2>&1 | tail -30 > gpurun_out/r2d_quick.txt
cat gpurun_out/r2d_quick.txt
timeout 900 python tools/sweep.py --only cfg > gpurun_out/r2d_sweep.jsonl 2> gpurun_out/r2d_sweep.err
timeout 600 python tools/sweep.py --opt-m 16,64,128,256,2048 > gpurun_out/r2d_sweep_opt.jsonl 2>> gpurun_out/r2d_sweep.err
timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err
cat gpurun_out/r2d_sweep.jsonl gpurun_out/r2d_sweep_opt.jsonl | cut -c 1-300; tail -3 gpurun_out/r2d_sweep.err; head -c 400 gpurun_out/r2d_bench.json
