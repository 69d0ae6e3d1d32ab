set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python bench.py > gpurun_out/bench_m16.json 2> gpurun_out/bench_m16.err
timeout 300 python bench.py --m 1 --no-cpu-baseline > gpurun_out/bench_m1.json 2> gpurun_out/bench_m1.err
for tp in 1 2 4 8; do timeout 200 python tools/fwd_time.py --shape llama70b --sim-tp $tp; done > gpurun_out/sweep_llama.log 2>&1
for tp in 1 8; do timeout 200 python tools/fwd_time.py --shape granite20b --sim-tp $tp; done > gpurun_out/sweep_granite.log 2>&1
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --no-graph --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
