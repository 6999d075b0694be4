mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2x.txt
timeout 300 tools/k1_probe > gpurun_out/r2x_probe.jsonl 2>&1
timeout 300 python tools/cfg1_probe.py >> gpurun_out/r2x.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2x_cfg1_launches.csv python tools/cfg1_probe.py --once > /dev/null 2>&1
timeout 300 python tools/k1_bench.py >> gpurun_out/r2x.txt 2>&1
tail -40 gpurun_out/r2x.txt | cut -c 1-300
