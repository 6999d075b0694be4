mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "int4_weight_mode" 2>&1 | tail -3 > gpurun_out/r2r.txt
timeout 600 python tools/sweep.py --weights int4 --only "cfg3 70B up/gate" --opt-m 16,128,256,2048 2>&1 | grep -v "2:4" | cut -c 1-330 >> gpurun_out/r2r.txt
timeout 600 python tools/sweep.py --weights int4 --only "cfg2" 2>&1 | cut -c 1-330 >> gpurun_out/r2r.txt
rm -f /tmp/tr.bin*
QUIK_GEMM_TRACE=/tmp/tr.bin timeout 120 python -c "
import sys; sys.path.insert(0,'.')
import torch, paper_2310_09259_b200 as q
dev=torch.device('cuda',0); g=torch.Generator(device=dev).manual_seed(3)
K,N,O,M=8192,28672,256,4096
idx=torch.randperm(K,generator=g,device=dev)[:O].sort().values.cpu().numpy(); outl=q.OutlierSet.from_indices(K,idx)
W=torch.randn(N,K,device=dev,generator=g); base,sc,wr,ow=q.rtn_quantize_weights_device(W,outl,4); del W
L=q.QuikLinear.from_device(outl,base,sc,wr,ow,4,weights='int4'); x=torch.randn(M,K,device=dev,dtype=torch.float16)
L(x); torch.cuda.synchronize()" >> gpurun_out/r2r.txt 2>&1
python tools/trace_view.py /tmp/tr.bin 2>&1 | grep "clk" >> gpurun_out/r2r.txt
cat gpurun_out/r2r.txt
