"""Wait-cycle accounting per warp role (profiling build):
    python -m paper_2402_04925_b200.build --prof
    TPQ_LIB_PATH=paper_2402_04925_b200/libtpq_prof.so python tools/prof_waits.py --m 1"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2402_04925_b200 as tpq  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="llama70b")
ap.add_argument("--m", type=int, default=1)
ap.add_argument("--sim-tp", type=int, default=1)
ap.add_argument("--iters", type=int, default=20)
a = ap.parse_args()
p = synth.make_named(a.shape, 16, 0)
P1, _ = tpq.gptq_reorder(p.w1.g_idx, p.G)
P2, _ = tpq.gptq_reorder(p.w2.g_idx, p.G)
h = tpq.TpMlp(p.w1, p.w2, P1, P2, tp=a.sim_tp, rank=0, M_max=16)
X = torch.from_numpy(p.X).cuda()
Y = torch.empty(16, p.N2, dtype=torch.float16, device="cuda")
L = tpq.lib()
L.tpq_debug_prof.argtypes = [C.c_void_p]
buf = (C.c_ulonglong * 32)()
h.forward_local(X, a.m, Y)
torch.cuda.synchronize()
L.tpq_debug_prof(C.cast(buf, C.c_void_p))  # reset
for _ in range(a.iters):
    h.forward_local(X, a.m, Y)
torch.cuda.synchronize()
L.tpq_debug_prof(C.cast(buf, C.c_void_p))
v = list(buf)
roles = [("dequant", 0, ["full", "A free", "st+wait", "-"]), ("epilogue", 5, ["done", "s_full", "-", "-"]),
         ("producer", 10, ["empty", "-", "-", "-"]), ("stager", 15, ["slot free", "tma issue", "-", "-"]),
         ("mma", 20, ["d_empty", "a_full", "xfull", "issue"])]
for name, base, keys in roles:
    T = v[base + 4] or 1
    print(f"{name:9s} total {T:14d}  " + "  ".join(f"{k} {100 * v[base + i] / T:5.1f}%" for i, k in enumerate(keys) if k != "-"))

# per-unit timeline of CTA 0 (layer-2 launch of the last forward), cycles relative to unit 16's MMA a_full
import numpy as np  # noqa: E402
L.tpq_debug_trace.argtypes = [C.c_void_p]
tr = (C.c_longlong * (24 * 64 * 4))()
L.tpq_debug_trace(C.cast(tr, C.c_void_p))
t = np.array(tr, dtype=np.int64).reshape(24, 64, 4)
nz = t[t > 0]
t0 = int(nz.min()) if nz.size else 1  # cycles relative to the first recorded event of CTA 0
def f(w, i, e):
    return f"{t[w, i, e] - t0:7d}" if t[w, i, e] else "      -"
print("pair | prod W(2p) | stage | deq(set p%2 w0, unit 2p): full computed Afree | arrive | mma: d_empty a_full xfull issued | epi: done s_full d_empty_arr")
for pp in range(0 if a.sim_tp > 1 else 5, 8 if a.sim_tp > 1 else 22):
    i = 2 * pp
    dw = 0 if pp % 2 == 0 else 8
    mw = 22 + pp % 2
    print(f"{pp:4d} | {f(20, i, 0)} | {f(21, i, 0)} | {f(dw, i, 0)} {f(dw, i, 1)} {f(dw, i, 2)} | {f(dw, i, 3)} | "
          f"{f(mw, i, 0)} {f(mw, i, 1)} {f(mw, i, 2)} {f(mw, i, 3)} | {f(16, i, 0)} {f(16, i, 1)} {f(16, i, 2)}")

print("epilogue (warp 16) per segment: d_full landed | partial+atomic done | segment done")
for sg in range(4):
    print(f"  seg {sg}: {f(16, sg, 0)} {f(16, sg, 1)} {f(16, sg, 2)}")
