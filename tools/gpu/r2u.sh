mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "quantizer or hot or fused_quantizer" 2>&1 | tail -3 > gpurun_out/r2u.txt
for w in 0 1; do echo "== QUIK_K1_WAIT=$w" >> gpurun_out/r2u.txt; QUIK_K1_WAIT=$w timeout 300 python tools/k1_bench.py >> gpurun_out/r2u.txt 2>&1; done
cat gpurun_out/r2u.txt | cut -c 1-250
