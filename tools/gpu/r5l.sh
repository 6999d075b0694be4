# the new graph test, bench line, MLP block, launch lists, ncu --set full of the 7B gated GEMM with / without statistics (raw CSV only)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_mlp_fused.py -q 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/r5l_bench.json 2> gpurun_out/r5l_bench.err
timeout 300 python tools/mlp_bench.py > gpurun_out/r5l_mlp.jsonl 2>&1
timeout 300 python tools/mlp_bench.py --tokens 16 >> gpurun_out/r5l_mlp.jsonl 2>&1
for sh in 7B 70B; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r5l_launches_$sh.csv python tools/mlp_kernels.py $sh > /dev/null 2>&1
done
for which in stats:8 plain:14; do
  n=${which%%:*}; sk=${which##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:quik_gemm_kernel -s $sk -c 1 -o /tmp/r5l_$n python tools/mlp_kernels.py 7B > /dev/null 2>&1
  ncu -i /tmp/r5l_$n.ncu-rep --page raw --csv > gpurun_out/r5l_ncu_${n}_gemm_7b_raw.csv 2>/dev/null
  rm -f /tmp/r5l_$n.ncu-rep
done
head -c 300 gpurun_out/r5l_bench.json; echo; cut -c 1-200 gpurun_out/r5l_mlp.jsonl; ls -la gpurun_out/r5l*
