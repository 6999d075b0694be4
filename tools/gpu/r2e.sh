# W4 bottleneck experiment: GEMM time with W4 synchronisation steps skipped (garbage results)
mkdir -p gpurun_out
for d in 0 1 2 4 8 3 7 15; do
  echo "== QUIK_W4_DBG=$d" >> gpurun_out/r2e.txt
  QUIK_W4_DBG=$d timeout 300 python tools/sweep.py --only "cfg3 70B up/gate" --opt-m 128 2>&1 | grep -v "2:4" | cut -c 1-260 >> gpurun_out/r2e.txt
done
cat gpurun_out/r2e.txt
