timeout 800 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for e in "" 1; do for tp in 1 2 4 8; do
echo "nofused=$e tp=$tp $(env ${e:+TPQ_NO_FUSED_GATHER=1} timeout 200 python tools/fwd_time.py --sim-tp $tp --ms 1,4,16 2>&1 | tail -1)"
done; done
