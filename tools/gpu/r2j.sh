mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "every_tile or large_layer or stream_gemm or cfg1 or variants" 2>&1 | tail -5 > gpurun_out/r2j.txt
for c in "--M 4096 --K 8192 --N 28672 --O 256" "--M 128 --K 9216 --N 36864 --O 256" "--M 2048 --K 4096 --N 4096 --O 256"; do
  echo "== $c" >> gpurun_out/r2j.txt
  timeout 120 python tools/gemm_case.py $c >> gpurun_out/r2j.txt 2>&1
  QUIK_GEMM_TRACE=/tmp/tr.bin timeout 120 python tools/gemm_case.py $c --once >> gpurun_out/r2j.txt 2>&1
  python tools/trace_view.py /tmp/tr.bin 2>&1 | grep -v "cluster 0 " >> gpurun_out/r2j.txt
done
cat gpurun_out/r2j.txt
