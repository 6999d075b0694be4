mkdir -p gpurun_out
for c in "--M 2048 --K 5120 --N 13824 --O 256 --sparse" "--M 2048 --K 5120 --N 13824 --O 256" "--M 4096 --K 8192 --N 28672 --O 256 --bits 8"; do
  echo "== $c" >> gpurun_out/r2q.txt
  timeout 120 python tools/gemm_case.py $c >> gpurun_out/r2q.txt 2>&1
  QUIK_GEMM_TRACE=/tmp/tr.bin timeout 120 python tools/gemm_case.py $c --once >> gpurun_out/r2q.txt 2>&1
  python tools/trace_view.py /tmp/tr.bin 2>&1 | grep "clk\|wait\|issue" >> gpurun_out/r2q.txt
done
cat gpurun_out/r2q.txt
