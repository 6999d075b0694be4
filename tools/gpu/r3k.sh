mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "quantizer or wide" 2>&1 | tail -15 > gpurun_out/r3k.txt
timeout 300 python tools/k1_bench.py >> gpurun_out/r3k.txt 2>&1
QUIK_K1_VARIANT=2 timeout 300 python tools/k1_bench.py --only down >> gpurun_out/r3k.txt 2>&1
cat gpurun_out/r3k.txt | cut -c 1-250
