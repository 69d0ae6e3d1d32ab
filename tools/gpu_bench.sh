# Round measurement: bench lines, reference arm, ncu launch list and full capture (gpurun_out/)
mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 300 python bench.py --steps 2000 --warmup 50 --m 1 --quick --no-cpu-baseline > gpurun_out/bench_m1.json 2> gpurun_out/bench_m1.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches.csv python bench.py --no-graph --steps 16 --warmup 3 --quick --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dqgemv -s 6 -c 2 -o gpurun_out/gemv_full python tools/fwd_time.py --sim-tp 1 --ms 16 --reps 2 > gpurun_out/ncu_full.log 2>&1
ls gpurun_out
