# INT4-only weights (weights="int4") shape sweep with this session's K1
mkdir -p gpurun_out
timeout 1500 python tools/sweep.py --weights int4 > gpurun_out/r6h_sweep_int4.jsonl 2> gpurun_out/r6h_sweep_int4.err
wc -l gpurun_out/r6h_sweep_int4.jsonl; tail -2 gpurun_out/r6h_sweep_int4.err
