mkdir -p gpurun_out
timeout 600 python tools/tile_sweep.py > gpurun_out/r3w.txt 2>&1
cat gpurun_out/r3w.txt
