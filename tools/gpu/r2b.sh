# round-2 GPU session B: full GPU suite (incl. full-shape parity and the new API surface) + bench
mkdir -p gpurun_out
python -c "from paper_2310_09259_b200 import build as b; b.build_tests()" > gpurun_out/r2b_build.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -40 > gpurun_out/r2b_pytest.txt
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
cat gpurun_out/r2b_pytest.txt; tail -c 800 gpurun_out/r2b_bench.json; tail -5 gpurun_out/r2b_bench.err
