mkdir -p gpurun_out
: > gpurun_out/r4a.txt
echo "hot" >> gpurun_out/r4a.txt
timeout 300 python tools/k1_bench.py --only "7B down" 2>&1 | cut -c 1-160 >> gpurun_out/r4a.txt
for sc in 2752 3672 5504; do
echo "wide slice_cols=$sc" >> gpurun_out/r4a.txt
QUIK_K1_WIDE_MIN_K=8193 QUIK_K1_SLICE_COLS=$sc timeout 300 python tools/k1_bench.py --only "7B down" 2>&1 | cut -c 1-160 >> gpurun_out/r4a.txt
QUIK_K1_WIDE_MIN_K=8193 QUIK_K1_SLICE_COLS=$sc timeout 300 python tools/k1_bench.py --only "70B down" 2>&1 | cut -c 1-160 >> gpurun_out/r4a.txt
done
for v in 1 2 4; do
echo "hot vpt=$v" >> gpurun_out/r4a.txt
QUIK_K1_VPT=$v timeout 300 python tools/k1_bench.py --only "7B down" 2>&1 | cut -c 1-160 >> gpurun_out/r4a.txt
done
cat gpurun_out/r4a.txt
