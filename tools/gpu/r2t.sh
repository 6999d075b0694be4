mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "every_tile or int4_weight or sparse or large_layer or variants" 2>&1 | tail -3 > gpurun_out/r2t.txt
timeout 900 python tools/sweep.py --only cfg >> gpurun_out/r2t.txt 2>&1
timeout 600 python tools/sweep.py --weights int4 --only "cfg3 70B up/gate" --opt-m 128,2048 2>&1 | grep -v "2:4" >> gpurun_out/r2t.txt
rm -f /tmp/tr.bin*
QUIK_GEMM_TRACE=/tmp/tr.bin timeout 120 python tools/gemm_case.py --M 2048 --K 5120 --N 13824 --O 256 --sparse --once >> gpurun_out/r2t.txt 2>&1
python tools/trace_view.py /tmp/tr.bin 2>&1 | grep "clk" >> gpurun_out/r2t.txt
cat gpurun_out/r2t.txt | cut -c 1-300
