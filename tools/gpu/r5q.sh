mkdir -p gpurun_out
timeout 600 python tools/sp_tile_sweep.py 2>&1 | tail -4
