# round-2 GPU session S: full GPU suite, bench, CPU reference sample points, ncu of the decode and weight-only kernels
mkdir -p gpurun_out
python -c "from paper_2310_09259_b200 import build as b; b.build_tests()" > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/r2s_pytest.txt
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/r2s_bench.json 2> gpurun_out/r2s_bench.err
OMP_NUM_THREADS=$(nproc) timeout 900 python tools/cpu_samples.py > gpurun_out/r2s_cpu_samples.jsonl 2> gpurun_out/r2s_cpu.err
cat > /tmp/dec.py <<'PY'
import sys; sys.path.insert(0, '.')
import torch, paper_2310_09259_b200 as q
dev = torch.device('cuda', 0); g = torch.Generator(device=dev).manual_seed(3)
K, N, O = 9216, 36864, 256
idx = torch.randperm(K, generator=g, device=dev)[:O].sort().values.cpu().numpy(); outl = q.OutlierSet.from_indices(K, idx)
W = torch.randn(N, K, device=dev, generator=g); base, sc, wr, ow = q.rtn_quantize_weights_device(W, outl, 4); del W
L = q.QuikLinear.from_device(outl, base, sc, wr, ow, 4)
for M in (16, 1):
    x = torch.randn(M, K, device=dev, dtype=torch.float16)
    for _ in range(3):
        L(x); L.weight_only(x)
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stream4 -s 2 -c 1 -o gpurun_out/r2s_decode python /tmp/dec.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:wo_gemm -s 4 -c 1 -o gpurun_out/r2s_wo python /tmp/dec.py > /dev/null 2>&1
cat gpurun_out/r2s_pytest.txt; tail -c 600 gpurun_out/r2s_bench.json; cat gpurun_out/r2s_cpu_samples.jsonl | cut -c 1-200; ls gpurun_out/r2s*
