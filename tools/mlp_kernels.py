"""Per-kernel launch list of the gated MLP block (for ncu --metrics gpu__time_duration.sum):
LLaMA-2-70B (4096 tokens; argv[1] picks another SHAPES entry, e.g. 7B) through quik_gated_mlp_forward (statistics fused) and through
two plain forwards, 3 calls each after a warm-up."""
import sys

sys.path.insert(0, "."); sys.path.insert(0, "tools")
import torch  # noqa: E402

import paper_2310_09259_b200 as q  # noqa: E402
from mlp_bench import SHAPES, device_layer, host_layer  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "70B"
name, M, H, F, O, Od, b_ud, b_d = [s for s in SHAPES if which in s[0]][0]
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(5)
outl, tu = device_layer(dev, H, F, O, b_ud, g)
_, tg = device_layer(dev, H, F, O, b_ud, g, idx=outl.indices)
outl_d, td = device_layer(dev, F, H, Od, b_d, g)
mlp = q.QuikGatedMLP(host_layer(outl, tu, b_ud), host_layer(outl, tg, b_ud), host_layer(outl_d, td, b_d))
x = torch.randn(M, H, device=dev, dtype=torch.float16)
y = torch.empty(M, H, device=dev, dtype=torch.float16)
for fused in (True, False, True, False):
    mlp.forward(x, out=y, fused=fused)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("timed")
for fused in (True, True, True, False, False, False):
    mlp.forward(x, out=y, fused=fused)
torch.cuda.synchronize()
