mkdir -p gpurun_out
: > gpurun_out/r3l.txt
for sc in 4096 8192 16384; do
echo "slice_cols=$sc" >> gpurun_out/r3l.txt
QUIK_K1_DEBUG=1 QUIK_K1_SLICE_COLS=$sc timeout 300 python tools/k1_bench.py --only down >> gpurun_out/r3l.txt 2>&1
done
cat gpurun_out/r3l.txt | sort | uniq -c | cut -c 1-250
