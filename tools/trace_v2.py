"""Per-pair event timeline of CTA 0 of the layer-2 GEMV (profiling build, k_dqgemv2):
    TPQ_LIB_PATH=paper_2402_04925_b200/libtpq_prof.so python tools/trace_v2.py --m 16
Dequant warps 4/8/12 (sets 0-2): [pair start, weights landed, own buffer free, a_full arrive];
MMA warps 18/19: [before a_full wait, a_full acquired, -, commit issued]; producer 16: refill i
[before empty wait, after]."""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2402_04925_b200 as tpq  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="llama70b")
ap.add_argument("--m", type=int, default=16)
ap.add_argument("--sim-tp", type=int, default=1)
a = ap.parse_args()
p = synth.make_named(a.shape, 16, 0)
P1, _ = tpq.gptq_reorder(p.w1.g_idx, p.G)
P2, _ = tpq.gptq_reorder(p.w2.g_idx, p.G)
R = 2 if a.sim_tp == 1 else 8
hs = [tpq.TpMlp(p.w1, p.w2, P1, P2, tp=a.sim_tp, rank=0, M_max=16) for _ in range(R)]
X = torch.from_numpy(p.X).cuda()
Y = torch.empty(16, p.N2, dtype=torch.float16, device="cuda")
for i in range(10 * R + 1):
    hs[i % R].forward_local(X, a.m, Y)
torch.cuda.synchronize()
L = tpq.lib()
L.tpq_debug_trace.argtypes = [C.c_void_p]
tr = (C.c_longlong * (2 * 24 * 64 * 4))()
L.tpq_debug_trace(C.cast(tr, C.c_void_p))
t = np.array(tr, dtype=np.int64).reshape(2, 24, 64, 4)[0]
t0 = t[t > 0].min()
rel = np.where(t > 0, t - t0, -1)
print("pair | set0 w4: start landed free arrive | set1 w8 | set2 w12 | mma18: wait got - commit | mma19")
for pi in range(49):
    row = []
    w = [4, 8, 12][pi % 3]
    row.append(f"{pi:3d} s{pi % 3} " + " ".join(f"{v:7d}" for v in rel[w, pi]))
    m = 18 + pi % 2
    row.append(f"| m{m} " + " ".join(f"{v:7d}" for v in rel[m, pi]))
    print(" ".join(row))
print("producer refills (i: before, after empty wait):")
print(" ".join(f"{i}:{rel[16, i, 0]}/{rel[16, i, 1]}" for i in range(40)))
d = []
for pi in range(6, 45):
    w = [4, 8, 12][pi % 3]
    d.append(rel[w, pi, 3] - rel[w, pi - 3, 3])
print("set cycle (arrive-to-arrive, cycles) median", np.median(d), "-> per unit", np.median(d) / 6)
L.tpq_debug_cta.argtypes = [C.c_void_p]
buf = (C.c_ulonglong * (2 * 1024 * 10))()
L.tpq_debug_cta(C.cast(buf, C.c_void_p))
ct = np.array(buf, dtype=np.int64).reshape(2, 1024, 10)
cta = int(os.environ.get("TPQ_TRACE_CTA_ID", "0"))
for sl in (0, 1):
    r = ct[sl, cta]
    if r[0] > 0:
        print(f"slot {sl} cta {cta}: entry->work start {(r[1] - r[0]) / 1e3:.2f} us, entry->end {(r[2] - r[0]) / 1e3:.2f} us, "
              f"clock {(r[9] - r[8]) / max(1, r[2] - r[0]) * 1e3:.0f} MHz; entry clock64 {r[8]} (trace t0 {t0})")
