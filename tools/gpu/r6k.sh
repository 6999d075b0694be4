# final: GPU suite, smoke, bench, K1 bench, MLP block, sweep
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/r6k_bench.json 2> gpurun_out/r6k_bench.err
python -c "
import json; r=json.loads(open('gpurun_out/r6k_bench.json').read().strip().splitlines()[-1]); print(r['value'], r['fp16_cublas']['speedup_step'], r['parity']['status'], r['quantizer']['ms_median'], r['quantizer']['frac'], r['int4_weights']['tops'])"
timeout 300 python tools/k1_bench.py > gpurun_out/r6k_k1_bench.jsonl 2>&1
timeout 300 python tools/mlp_bench.py > gpurun_out/r6k_mlp.jsonl 2>&1
timeout 300 python tools/mlp_bench.py --tokens 16 >> gpurun_out/r6k_mlp.jsonl 2>&1
timeout 1500 python tools/sweep.py > gpurun_out/r6k_sweep.jsonl 2> gpurun_out/r6k_sweep.err
cut -c 1-160 gpurun_out/r6k_mlp.jsonl; wc -l gpurun_out/r6k_sweep.jsonl
