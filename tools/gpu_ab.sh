timeout 800 python -m pytest tests -q -m gpu 2>&1 | tail -1
echo "A7 tp8 $(timeout 300 python tools/fwd_time.py --sim-tp 8 --ms 32,64,128,256,512 2>&1 | tail -1)"
for tp in 1 8; do echo "tp=$tp $(timeout 200 python tools/fwd_time.py --sim-tp $tp --ms 1,16 2>&1 | tail -1)"; done
