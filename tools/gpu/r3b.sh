mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "stream or decode or int4_weight_mode or gated" 2>&1 | tail -3 > gpurun_out/r3b.txt
timeout 300 python -m pytest tests/test_gpu_fullshape.py -q -x -k "opt or cfg1" 2>&1 | tail -3 >> gpurun_out/r3b.txt
timeout 300 python tools/cfg1_probe.py --m 1,16 >> gpurun_out/r3b.txt 2>&1
timeout 600 python tools/sweep.py --only "OPT-66B fc1" --opt-m 1,16 >> gpurun_out/r3b.txt 2>&1
timeout 300 python tools/sweep.py --only "zzz" --falcon --opt-m 1 2>&1 | grep "M=1\"\|M=16\"" >> gpurun_out/r3b.txt
cat gpurun_out/r3b.txt | cut -c 1-300
