# decode-kernel hybrid schedule (whole-block waves + stream-K remainder) vs the existing schedules; MLP int4-mode test
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_mlp_fused.py -q -k int4 2>&1 | tail -3
for s in auto 1 -1 -2; do
  if [ $s = auto ]; then unset QUIK_S4_SPLITS; else export QUIK_S4_SPLITS=$s; fi
  timeout 600 python tools/s4_sched.py 2>&1 | tail -8
done
