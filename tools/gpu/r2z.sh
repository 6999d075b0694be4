mkdir -p gpurun_out
: > gpurun_out/r2z.txt
for s in 1 2 4 8; do echo "splits=$s" >> gpurun_out/r2z.txt; QUIK_S4_SPLITS=$s timeout 120 python tools/cfg1_probe.py --m 1,16,32 >> gpurun_out/r2z.txt 2>&1; done
echo "stream4=0" >> gpurun_out/r2z.txt; QUIK_STREAM4=0 timeout 120 python tools/cfg1_probe.py --m 1,16,32 >> gpurun_out/r2z.txt 2>&1
cat gpurun_out/r2z.txt | cut -c 1-250
