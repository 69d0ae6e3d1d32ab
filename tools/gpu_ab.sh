for g in 148 120 96 74; do for tp in 4 8; do
echo "grid=$g tp=$tp $(TPQ_GRID=$g timeout 200 python tools/fwd_time.py --sim-tp $tp --ms 1,16 2>&1 | tail -1)"
done; done
