for e in "" 1; do for tp in 1 8; do
echo "inkernel=$e tp=$tp $(env ${e:+TPQ_INKERNEL_FIXUP=1} timeout 200 python tools/fwd_time.py --sim-tp $tp --ms 1,2,3,4,5,8,12,16 2>&1 | tail -1)"
done; done
