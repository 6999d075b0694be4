mkdir -p gpurun_out
timeout 300 tools/k1_probe > gpurun_out/r2y_probe.jsonl 2>&1
tail -3 gpurun_out/r2y_probe.jsonl
