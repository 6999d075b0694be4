mkdir -p gpurun_out
for c in "--M 4096 --K 8192 --N 28672 --O 256" "--M 128 --K 9216 --N 36864 --O 256"; do
  echo "== $c" >> gpurun_out/r2h.txt
  QUIK_GEMM_TRACE=/tmp/tr.bin timeout 120 python tools/gemm_case.py $c --once >> gpurun_out/r2h.txt 2>&1
  python tools/trace_view.py /tmp/tr.bin 2>&1 | grep -v "cluster 0 " >> gpurun_out/r2h.txt
done
cat gpurun_out/r2h.txt
