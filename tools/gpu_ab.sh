timeout 800 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
echo "M sweep $(timeout 200 python tools/fwd_time.py --sim-tp 1 --ms 1,4,8,16 2>&1 | tail -1)"
echo "M sweep tp8 $(timeout 200 python tools/fwd_time.py --sim-tp 8 --ms 1,4,8,16 2>&1 | tail -1)"
echo "M sweep tp2 $(timeout 200 python tools/fwd_time.py --sim-tp 2 --ms 1,16 2>&1 | tail -1)"
echo "tp4 $(timeout 200 python tools/fwd_time.py --sim-tp 4 --ms 1,16 2>&1 | tail -1)"
echo "granite $(timeout 200 python tools/fwd_time.py --shape granite20b --sim-tp 1 --ms 1,16 2>&1 | tail -1)"
