# ncu --set full of the 70B down K1: prescaled (quik_gated_mlp_forward) vs its own reduction (raw CSV only)
mkdir -p gpurun_out
for which in pre:3 plain:9; do
  n=${which%%:*}; sk=${which##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:quantize_hot_kernel -s $sk -c 1 -o /tmp/r5s_$n python tools/mlp_kernels.py 70B > /dev/null 2>&1
  ncu -i /tmp/r5s_$n.ncu-rep --page raw --csv > gpurun_out/r5s_ncu_${n}_k1_70b_raw.csv 2>/dev/null
  rm -f /tmp/r5s_$n.ncu-rep
done
ls -la gpurun_out/r5s*
