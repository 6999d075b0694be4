# HEAD verification: GPU suite, smoke, bench, MLP block bench (prefill + decode), launch lists, ncu of the statistics GEMM
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/r5k_pytest.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r5k_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/r5k_bench.json 2> gpurun_out/r5k_bench.err
timeout 300 python tools/mlp_bench.py > gpurun_out/r5k_mlp.jsonl 2>&1
timeout 300 python tools/mlp_bench.py --tokens 16 >> gpurun_out/r5k_mlp.jsonl 2>&1
for sh in 7B 70B; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r5k_launches_$sh.csv python tools/mlp_kernels.py $sh > /dev/null 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:quik_gemm_kernel -s 8 -c 1 -o gpurun_out/r5k_stats_gemm_7b python tools/mlp_kernels.py 7B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:quik_gemm_kernel -s 14 -c 1 -o gpurun_out/r5k_plain_gemm_7b python tools/mlp_kernels.py 7B > /dev/null 2>&1
cat gpurun_out/r5k_pytest.txt gpurun_out/r5k_smoke.txt; head -c 300 gpurun_out/r5k_bench.json; cut -c 1-200 gpurun_out/r5k_mlp.jsonl; ls -la gpurun_out/r5k*
