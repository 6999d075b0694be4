mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/r4c_bench.json 2> gpurun_out/r4c_bench.err
python -c "
import json; r=json.loads(open('gpurun_out/r4c_bench.json').read().strip().splitlines()[-1]); print(r['value'], r['fp16_cublas']['speedup_step'], r['parity']['status']); print(json.dumps(r.get('decode')))"
tail -3 gpurun_out/r4c_bench.err
