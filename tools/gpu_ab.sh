timeout 800 python -m pytest tests -q -m gpu 2>&1 | tail -1
timeout 250 python tools/stress_reg.py 1 tc | tail -1; timeout 250 python tools/stress_reg.py 4 tc | tail -1; timeout 250 python tools/stress_reg.py 16 tc | tail -1
for tp in 1 2 4 8; do echo "tp=$tp $(timeout 200 python tools/fwd_time.py --sim-tp $tp --ms 1,2,4,8,16 2>&1 | tail -1)"; done
for tp in 1 8; do echo "granite tp=$tp $(timeout 200 python tools/fwd_time.py --shape granite20b --sim-tp $tp --ms 1,4,16 2>&1 | tail -1)"; done
