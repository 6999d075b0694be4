# ncu --set full of the round's new kernel paths: the wide-row K1 (OPT-66B fc2, cluster
# slices) and the decode kernel at 70B up / gate, one token (whole-block schedule)
mkdir -p gpurun_out
cat > /tmp/r4d.py <<'PY'
import sys; sys.path.insert(0, '.')
import torch, paper_2310_09259_b200 as q
dev = torch.device('cuda', 0); g = torch.Generator(device=dev).manual_seed(3)
def layer(K, N, O, bits):
    idx = torch.randperm(K, generator=g, device=dev)[:O].sort().values.cpu().numpy(); outl = q.OutlierSet.from_indices(K, idx)
    W = torch.randn(N, K, device=dev, generator=g); base, sc, wr, ow = q.rtn_quantize_weights_device(W, outl, bits); del W
    return q.QuikLinear.from_device(outl, base, sc, wr, ow, bits)
which = sys.argv[1]
if which == 'wide':
    L = layer(36864, 256, 256, 4); x = torch.randn(2048, 36864, device=dev, dtype=torch.float16)
else:
    L = layer(8192, 28672, 256, 4); x = torch.randn(1, 8192, device=dev, dtype=torch.float16)
for _ in range(4):
    L(x)
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:quantize_wide -s 2 -c 1 -o gpurun_out/r4d_wide python /tmp/r4d.py wide > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stream4 -s 2 -c 1 -o gpurun_out/r4d_decode python /tmp/r4d.py decode > /dev/null 2>&1
ls -la gpurun_out/r4d*
