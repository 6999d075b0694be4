# final verification: MLP tests (incl. the hidden row pitch), full GPU suite, smoke, bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_mlp_fused.py -q 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/r5r_bench.json 2> gpurun_out/r5r_bench.err
python -c "
import json; r=json.loads(open('gpurun_out/r5r_bench.json').read().strip().splitlines()[-1]); print(r['value'], r['fp16_cublas']['speedup_step'], r['parity']['status'], r['int4_weights']['tops'])"
