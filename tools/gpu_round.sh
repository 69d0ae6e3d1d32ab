# Round measurement: bench lines, launch list and full ncu captures (results in gpurun_out/).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 300 python bench.py > gpurun_out/bench_m16.json 2> gpurun_out/bench_m16.err
timeout 300 python bench.py --m 1 --no-cpu-baseline > gpurun_out/bench_m1.json 2> gpurun_out/bench_m1.err
timeout 300 python bench.py --m 4 --no-cpu-baseline > gpurun_out/bench_m4.json 2> gpurun_out/bench_m4.err
timeout 300 python bench.py --shape granite20b --m 16 --no-cpu-baseline > gpurun_out/bench_granite_m16.json 2> /dev/null
timeout 300 python bench.py --shape granite20b --m 1 --no-cpu-baseline > gpurun_out/bench_granite_m1.json 2> /dev/null
for tp in 2 4 8; do for m in 1 16; do
  timeout 300 python bench.py --sim-tp $tp --m $m --steps 2000 --warmup 50 --no-cpu-baseline > gpurun_out/bench_simtp${tp}_m$m.json 2>/dev/null
  TPQ_GEMV=r timeout 300 python bench.py --sim-tp $tp --m $m --steps 2000 --warmup 50 --no-cpu-baseline > gpurun_out/bench_reg_simtp${tp}_m$m.json 2>/dev/null
done; done
for m in 1 16; do TPQ_GEMV=r timeout 300 python bench.py --m $m --no-cpu-baseline > gpurun_out/bench_reg_m$m.json 2>/dev/null; done
timeout 300 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_reference.json 2>/dev/null
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches.csv python bench.py --no-graph --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_dqgemv -s 6 -c 2 -o gpurun_out/tc_m16_full python tools/fwd_time.py --sim-tp 1 --ms 16 --reps 2 > gpurun_out/ncu_tc.log 2>&1
ls gpurun_out
