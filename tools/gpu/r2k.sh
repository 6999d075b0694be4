mkdir -p gpurun_out
for d in 0 2 10 26; do
  echo "== dbg $d" >> gpurun_out/r2k.txt
  QUIK_W4_DBG=$d timeout 120 python tools/gemm_case.py --M 4096 --K 8192 --N 28672 --O 256 >> gpurun_out/r2k.txt 2>&1
  QUIK_W4_DBG=$d timeout 120 python tools/gemm_case.py --M 128 --K 9216 --N 36864 --O 256 >> gpurun_out/r2k.txt 2>&1
done
cat gpurun_out/r2k.txt
