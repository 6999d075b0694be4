mkdir -p gpurun_out
: > gpurun_out/r3m.txt
for sc in 4096 8192 16384; do
echo "slice_cols=$sc" >> gpurun_out/r3m.txt
QUIK_K1_DEBUG=1 QUIK_K1_SLICE_COLS=$sc timeout 300 python tools/k1_bench.py --only fc2 2>&1 | sort | uniq -c >> gpurun_out/r3m.txt
done
echo "general kernel" >> gpurun_out/r3m.txt
QUIK_K1_WIDE_MIN_K=999999 timeout 300 python tools/k1_bench.py --only fc2 >> gpurun_out/r3m.txt 2>&1
cat gpurun_out/r3m.txt | cut -c 1-200
