timeout 800 python -m pytest tests -q -m gpu 2>&1 | tail -2
timeout 250 python tools/stress_reg.py 16 tc | tail -1; timeout 250 python tools/stress_reg.py 1 tc | tail -1; timeout 250 python tools/stress_reg.py 16 reg | tail -1
for tp in 1 2 4 8; do echo "tp=$tp $(timeout 200 python tools/fwd_time.py --sim-tp $tp --ms 1,4,16 2>&1 | tail -1)"; done
echo "granite $(timeout 200 python tools/fwd_time.py --shape granite20b --sim-tp 1 --ms 1,16 2>&1 | tail -1)"
echo "A7 $(timeout 300 python tools/fwd_time.py --sim-tp 8 --ms 32,64,128,256,512 2>&1 | tail -1)"
