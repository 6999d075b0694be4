# HEAD check at the end of the session: GPU suite, smoke, bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/r6g_bench.json 2> gpurun_out/r6g_bench.err
python -c "
import json; r=json.loads(open('gpurun_out/r6g_bench.json').read().strip().splitlines()[-1]); print(r['value'], r['fp16_cublas']['speedup_step'], r['parity']['status'], r['quantizer']['ms_median'], r['quantizer']['frac'], r['roofline']['frac'], r['e2e']['value'], r['gpu_launches'])"
