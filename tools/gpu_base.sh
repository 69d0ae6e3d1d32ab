mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
timeout 400 python bench.py --steps 2000 --warmup 50 --sweep > gpurun_out/bench_base.json 2> gpurun_out/bench_base.err
timeout 500 ncu --set full --clock-control none --import-source on -k regex:k_dqgemv -s 6 -c 2 -o gpurun_out/base_full python tools/fwd_time.py --sim-tp 1 --ms 16 --reps 2 > gpurun_out/ncu_base.log 2>&1
ls gpurun_out
