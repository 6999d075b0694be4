# final numbers of the round: GPU suite, smoke, bench, K1 bench, MLP block, shape sweep
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/r6a_pytest.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r6a_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/r6a_bench.json 2> gpurun_out/r6a_bench.err
timeout 300 python tools/k1_bench.py > gpurun_out/r6a_k1_bench.jsonl 2>&1
timeout 300 python tools/mlp_bench.py > gpurun_out/r6a_mlp.jsonl 2>&1
timeout 300 python tools/mlp_bench.py --tokens 16 >> gpurun_out/r6a_mlp.jsonl 2>&1
timeout 1500 python tools/sweep.py > gpurun_out/r6a_sweep.jsonl 2> gpurun_out/r6a_sweep.err
cat gpurun_out/r6a_pytest.txt gpurun_out/r6a_smoke.txt; tail -2 gpurun_out/r6a_bench.err
python -c "
import json; r=json.loads(open('gpurun_out/r6a_bench.json').read().strip().splitlines()[-1]); print(r['value'], r['fp16_cublas']['speedup_step'], r['parity']['status'], r['quantizer']['ms_median'], r['quantizer']['frac'], r['int4_weights']['tops'])"
wc -l gpurun_out/r6a_sweep.jsonl; tail -2 gpurun_out/r6a_sweep.err
