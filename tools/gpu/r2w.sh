mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_acceptance.py -q -k "gptq or hessian or acceptance" 2>&1 | tail -5 > gpurun_out/r2w.txt
timeout 600 python tools/gptq_bench.py >> gpurun_out/r2w.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_ipc.py -q 2>&1 | tail -3 >> gpurun_out/r2w.txt
cat gpurun_out/r2w.txt | cut -c 1-300
