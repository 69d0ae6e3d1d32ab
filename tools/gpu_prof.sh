mkdir -p gpurun_out
export TPQ_LIB_PATH=paper_2402_04925_b200/libtpq_prof.so
for cfg in "1 1" "8 1" "8 16" "1 16"; do set -- $cfg; echo "== tp=$1 M=$2"; timeout 120 python tools/cta_times.py --sim-tp $1 --m $2; done > gpurun_out/cta_times.log 2>&1
for cfg in "8 1" "8 16"; do set -- $cfg; echo "== tp=$1 M=$2"; timeout 120 python tools/prof_waits.py --sim-tp $1 --m $2; done > gpurun_out/prof_waits.log 2>&1
