# round-2 GPU session P: sweeps (speed / int4 weights), N=2 gloo check mode, ncu launch list + full captures
mkdir -p gpurun_out
timeout 900 python tools/sweep.py --falcon > gpurun_out/r2p_sweep.jsonl 2> gpurun_out/r2p_sweep.err
timeout 600 python tools/sweep.py --weights int4 --opt-m 1,16,64,128,256,2048 > gpurun_out/r2p_sweep_int4.jsonl 2>> gpurun_out/r2p_sweep.err
QUIK_BENCH_DIST_BACKEND=gloo timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu --no-e2e --soak-s 0 > gpurun_out/r2p_gloo2.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r2p_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-cublas --soak-s 0 --no-clocks > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:quik_gemm_kernel -s 4 -c 1 -o gpurun_out/r2p_gemm python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-cublas --soak-s 0 --no-clocks > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:quantize_hot -s 4 -c 1 -o gpurun_out/r2p_k1 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-cublas --soak-s 0 --no-clocks > /dev/null 2>&1
ls -la gpurun_out/ | tail; tail -c 1500 gpurun_out/r2p_gloo2.txt
