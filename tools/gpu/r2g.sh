# W4 GEMM timeline: where the MMA and widening warps wait
mkdir -p gpurun_out
for c in "--M 4096 --K 8192 --N 28672 --O 256" "--M 128 --K 9216 --N 36864 --O 256" "--M 2048 --K 4096 --N 4096 --O 256"; do
  echo "== $c" >> gpurun_out/r2g.txt
  timeout 120 python tools/gemm_case.py $c >> gpurun_out/r2g.txt 2>&1
  timeout 120 python tools/gemm_case.py $c --probe >> gpurun_out/r2g.txt 2>&1
  QUIK_GEMM_TRACE=/tmp/tr.bin timeout 120 python tools/gemm_case.py $c --once >> gpurun_out/r2g.txt 2>&1
  python tools/trace_view.py /tmp/tr.bin >> gpurun_out/r2g.txt 2>&1
done
cat gpurun_out/r2g.txt
