mkdir -p gpurun_out
timeout 800 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for v in r tc; do for tp in 1 2 4 8; do
echo "$v tp=$tp $(TPQ_GEMV=$v timeout 200 python tools/fwd_time.py --sim-tp $tp --ms 1,4,16 2>&1 | tail -1)"
done; done
