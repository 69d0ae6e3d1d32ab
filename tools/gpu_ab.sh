for rep in 1 2; do for v in "" _ns16 _ns12 _nx6; do for tp in 1 8; do
echo "$v tp=$tp $(TPQ_LIB_PATH=paper_2402_04925_b200/libtpq$v.so timeout 200 python tools/fwd_time.py --sim-tp $tp --ms 1,16 2>&1 | tail -1)"
done; done; done
