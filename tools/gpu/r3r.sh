mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r3r_smi.txt
timeout 1500 python tools/sweep.py --falcon > gpurun_out/r3r_sweep.jsonl 2> gpurun_out/r3r_sweep.err
timeout 900 python tools/sweep.py --weights int4 --opt-m 1,16,64,128,256,2048 > gpurun_out/r3r_sweep_int4.jsonl 2> gpurun_out/r3r_sweep_int4.err
timeout 300 python tools/k1_bench.py > gpurun_out/r3r_k1.jsonl 2>&1
wc -l gpurun_out/r3r_*.jsonl
tail -3 gpurun_out/r3r_sweep.err gpurun_out/r3r_sweep_int4.err
