mkdir -p gpurun_out
timeout 900 python bench.py --impl reference > gpurun_out/r6f_ref.json 2> gpurun_out/r6f_ref.err
tail -c 600 gpurun_out/r6f_ref.json; tail -2 gpurun_out/r6f_ref.err
