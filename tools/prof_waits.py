"""Wait-cycle accounting per warp role (needs the profiling build):
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
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--sim-tp", type=int, default=1)
a = ap.parse_args()
p = synth.make_named(a.shape, 16, 0)
P1, _ = tpq.gptq_reorder(p.w1.g_idx, p.G)
P2, _ = tpq.gptq_reorder(p.w2.g_idx, p.G)
h = tpq.TpMlp(p.w1, p.w2, P1, P2, tp=a.sim_tp, M_max=16)
X = torch.from_numpy(p.X).cuda()
Y = torch.empty(16, p.N2, dtype=torch.float16, device="cuda")
L = tpq.lib()
L.tpq_debug_prof.argtypes = [C.c_void_p]
buf = (C.c_ulonglong * 16)()
h.forward_local(X, a.m, Y)
torch.cuda.synchronize()
L.tpq_debug_prof(C.cast(buf, C.c_void_p))  # reset
for _ in range(a.iters):
    h.forward_local(X, a.m, Y)
torch.cuda.synchronize()
L.tpq_debug_prof(C.cast(buf, C.c_void_p))
v = list(buf)
names = {0: "prod:xempty", 1: "prod:empty", 8: "prod:TOTAL", 2: "mma:xfull", 3: "mma:a_full", 4: "mma:d_empty",
         9: "mma:TOTAL", 5: "deq:full", 6: "deq:a_empty", 7: "deq:d_full", 10: "deq:TOTAL"}
names.update({11: "deq:alu", 12: "epi:s_full", 13: "deq:st(incl a_empty)", 14: "epi:TOTAL"})
for role, tot, keys in (("producer", 8, [0, 1]), ("mma", 9, [2, 3, 4]), ("dequant", 10, [5, 6, 11, 13]), ("epilogue", 14, [7, 12])):
    T = v[tot] or 1
    print(f"{role:9s} total {T:14d} cyc-warps  " + "  ".join(f"{names[k]} {100 * v[k] / T:5.1f}%" for k in keys))

# event timeline of CTA 0 (first units), cycles relative to the first event
L.tpq_debug_trace.argtypes = [C.c_void_p]
tr = (C.c_longlong * (16 * 32 * 8))()
L.tpq_debug_trace(C.cast(tr, C.c_void_p))
import numpy as np  # noqa: E402
t = np.array(tr, dtype=np.int64).reshape(16, 32, 8)
t0 = t[t > 0].min()
rel = np.where(t > 0, t - t0, -1)
print("unit | W_issue X_issue | deq0: full_ok alu_done a_full_arr | mma13: a_full_ok d_empty_ok issued | epi8: d_ok")
for i in range(32):
    print(f"{i:4d} | {rel[12, i, 0]:7d} {rel[12, i, 1]:7d} | " + " ".join(f"{rel[0, i, e]:7d}" for e in range(3)) +
          " | " + " ".join(f"{rel[13, i, e]:7d}" for e in range(3)) + f" | {rel[8, i, 0]:7d}")
