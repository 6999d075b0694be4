# round-2 GPU session A: the GPU suite, the new full-shape parity tests, bench, cuBLASLt INT8 peak
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt
timeout 900 python -m pytest tests/test_gpu_fullshape.py -q -x 2>&1 | tail -30 > gpurun_out/r2a_fullshape.txt
timeout 1500 python -m pytest tests -m gpu -q --deselect tests/test_gpu_fullshape.py 2>&1 | tail -30 > gpurun_out/r2a_pytest.txt
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
python tools/int8_peak.py > gpurun_out/r2a_int8.txt 2>&1
cat gpurun_out/r2a_fullshape.txt gpurun_out/r2a_pytest.txt gpurun_out/r2a_int8.txt; tail -c 1500 gpurun_out/r2a_bench.json
