# ncu --set full of the FILL K1 at the 70B down projection and at cfg3 (raw CSV), k1_bench --once shapes
mkdir -p gpurun_out
cat > /tmp/k1one.py <<'PY'
import sys; sys.path.insert(0, '.')
import torch, numpy as np, paper_2310_09259_b200 as q
dev = torch.device('cuda', 0); g = torch.Generator(device=dev).manual_seed(3)
M, K, O, bits = [int(v) for v in sys.argv[1:5]]
idx = torch.randperm(K, generator=g, device=dev)[:O].sort().values.cpu().numpy(); outl = q.OutlierSet.from_indices(K, idx)
W = torch.randn(256, K, device=dev, generator=g); base, sc, wr, ow = q.rtn_quantize_weights_device(W, outl, bits)
L = q.QuikLinear.from_device(outl, base, sc, wr, ow, bits)
x = torch.randn(M, K, device=dev, dtype=torch.float16, generator=g)
for _ in range(3): L.quantize_gemm_layout(x)
torch.cuda.synchronize()
PY
for c in "4096 28672 896 8 down70b" "4096 8192 256 4 cfg3"; do
  set -- $c
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:quantize_hot -s 2 -c 1 -o /tmp/k1_$5 python /tmp/k1one.py $1 $2 $3 $4 > /dev/null 2>&1
  ncu -i /tmp/k1_$5.ncu-rep --page raw --csv > gpurun_out/r6c_ncu_k1_$5_raw.csv 2>/dev/null
  rm -f /tmp/k1_$5.ncu-rep
done
ls -la gpurun_out/r6c*
