mkdir -p gpurun_out
for c in "--M 2048 --K 5120 --N 13824 --O 256 --sparse" "--M 4096 --K 8192 --N 28672 --O 256"; do
  echo "== $c" >> gpurun_out/r2q.txt
  rm -f /tmp/tr.bin*
  QUIK_GEMM_TRACE=/tmp/tr.bin timeout 120 python tools/gemm_case.py $c --once >> gpurun_out/r2q.txt 2>&1
  python tools/trace_view.py /tmp/tr.bin 2>&1 | grep "clk" >> gpurun_out/r2q.txt
done
cat > /tmp/w4.py <<'PY'
import sys; sys.argv=['x','--M','4096','--K','8192','--N','28672','--O','256','--once']
PY
echo "== int4 cfg3" >> gpurun_out/r2q.txt
rm -f /tmp/tr.bin*
QUIK_GEMM_TRACE=/tmp/tr.bin timeout 120 python -c "
import sys; sys.path.insert(0,'.')
import torch, paper_2310_09259_b200 as q
dev=torch.device('cuda',0); g=torch.Generator(device=dev).manual_seed(3)
K,N,O,M=8192,28672,256,4096
idx=torch.randperm(K,generator=g,device=dev)[:O].sort().values.cpu().numpy(); outl=q.OutlierSet.from_indices(K,idx)
W=torch.randn(N,K,device=dev,generator=g); base,sc,wr,ow=q.rtn_quantize_weights_device(W,outl,4); del W
L=q.QuikLinear.from_device(outl,base,sc,wr,ow,4,weights='int4'); x=torch.randn(M,K,device=dev,dtype=torch.float16)
L(x); torch.cuda.synchronize()" >> gpurun_out/r2q.txt 2>&1
python tools/trace_view.py /tmp/tr.bin 2>&1 | grep "clk" >> gpurun_out/r2q.txt
cat gpurun_out/r2q.txt
