mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab_pytest.log 2>&1
timeout 300 python bench.py --steps 2000 --warmup 50 > gpurun_out/bench_v2.json 2> gpurun_out/bench_v2.err
