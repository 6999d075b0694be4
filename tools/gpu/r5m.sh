# final verification of this session's build: GPU suite, smoke, bench (incl. the int4_weights key)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/r5m_pytest.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r5m_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/r5m_bench.json 2> gpurun_out/r5m_bench.err
cat gpurun_out/r5m_pytest.txt gpurun_out/r5m_smoke.txt; tail -3 gpurun_out/r5m_bench.err
python -c "
import json; r=json.loads(open('gpurun_out/r5m_bench.json').read().strip().splitlines()[-1]); print(r['value'], r['fp16_cublas']['speedup_step'], r['parity']['status']); print(json.dumps(r.get('int4_weights')))"
