mkdir -p gpurun_out
timeout 900 python tools/mlp_bench.py > gpurun_out/r3t_mlp.jsonl 2>&1
timeout 600 python tools/mlp_bench.py --tokens 1 > gpurun_out/r3t_mlp_m1.jsonl 2>&1
timeout 600 python tools/mlp_bench.py --tokens 16 > gpurun_out/r3t_mlp_m16.jsonl 2>&1
cat gpurun_out/r3t_mlp*.jsonl | cut -c 1-400
