# round-2 GPU session V: sanitizers over the new kernels, INT4-mode GEMM DRAM traffic, bench with the f32 drop-in e2e
mkdir -p gpurun_out
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "int4_weight or every_tile or stage_times or forward_model or streams or reserve or rtn_clipping or split_and_unpack" > gpurun_out/r2v_memcheck.txt 2>&1
timeout 1200 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "int4_weight or every_tile" > gpurun_out/r2v_synccheck.txt 2>&1
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_ipc.py -q > gpurun_out/r2v_memcheck_ipc.txt 2>&1
cat > /tmp/w4c.py <<'PY'
import sys; sys.path.insert(0, '.')
import torch, paper_2310_09259_b200 as q
dev = torch.device('cuda', 0); g = torch.Generator(device=dev).manual_seed(3)
K, N, O, M = 8192, 28672, 256, 4096
idx = torch.randperm(K, generator=g, device=dev)[:O].sort().values.cpu().numpy(); outl = q.OutlierSet.from_indices(K, idx)
W = torch.randn(N, K, device=dev, generator=g); base, sc, wr, ow = q.rtn_quantize_weights_device(W, outl, 4); del W
L = q.QuikLinear.from_device(outl, base, sc, wr, ow, 4, weights='int4'); x = torch.randn(M, K, device=dev, dtype=torch.float16)
for _ in range(3): L(x)
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:quik_gemm_kernel -s 2 -c 1 -o gpurun_out/r2v_gemm_int4 python /tmp/w4c.py > /dev/null 2>&1
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/r2v_bench.json 2> gpurun_out/r2v_bench.err
tail -3 gpurun_out/r2v_memcheck.txt gpurun_out/r2v_synccheck.txt gpurun_out/r2v_memcheck_ipc.txt; tail -c 400 gpurun_out/r2v_bench.json
