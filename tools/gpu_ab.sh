mkdir -p gpurun_out
export TPQ_LIB_PATH=paper_2402_04925_b200/libtpq_prof.so
timeout 120 python tools/trace_v2.py --m 16 > gpurun_out/trace_v2_m16.log 2>&1
timeout 120 python tools/trace_v2.py --m 1 > gpurun_out/trace_v2_m1.log 2>&1
for cfg in "1 1" "1 16" "8 1"; do set -- $cfg; echo "== tp=$1 M=$2"; timeout 120 python tools/cta_times.py --sim-tp $1 --m $2; done > gpurun_out/cta_times.log 2>&1
