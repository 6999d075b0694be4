# re-entry check: the GPU suite, smoke and the headline bench on the restored tree
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/r5a_pytest.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r5a_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/r5a_bench.json 2> gpurun_out/r5a_bench.err
timeout 300 python tools/mlp_bench.py > gpurun_out/r5a_mlp.jsonl 2>&1
cat gpurun_out/r5a_pytest.txt gpurun_out/r5a_smoke.txt; head -c 600 gpurun_out/r5a_bench.json; tail -3 gpurun_out/r5a_bench.err; cut -c 1-300 gpurun_out/r5a_mlp.jsonl
