"""Per-pair globaltimer timeline of two CTAs of one GEMV launch (profiling build with
-DTPQ_TRACE_CTA=a -DTPQ_TRACE_CTA2=b -DTPQ_TRACE_N_GT_K=1 for layer 1):
    TPQ_LIB_PATH=paper_2402_04925_b200/libtpq_trp.so python tools/trace_pair.py --m 16
Prints, per pair, the a_full arrive time (A operands stored) of both CTAs in us from the earlier
CTA's first event, and the MMA commit times."""
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
a = ap.parse_args()
p = synth.make_named(a.shape, 16, 0)
P1, _ = tpq.gptq_reorder(p.w1.g_idx, p.G)
P2, _ = tpq.gptq_reorder(p.w2.g_idx, p.G)
hs = [tpq.TpMlp(p.w1, p.w2, P1, P2, tp=1, rank=0, M_max=16) for _ in range(2)]
X = torch.from_numpy(p.X).cuda()
Y = torch.empty(16, p.N2, dtype=torch.float16, device="cuda")
for i in range(21):
    hs[i % 2].forward_local(X, a.m, Y)
torch.cuda.synchronize()
L = tpq.lib()
L.tpq_debug_trace.argtypes = [C.c_void_p]
tr = (C.c_longlong * (2 * 24 * 64 * 4))()
L.tpq_debug_trace(C.cast(tr, C.c_void_p))
t = np.array(tr, dtype=np.int64).reshape(2, 24, 64, 4)
t0 = t[t > 0].min()
us = lambda x: (x - t0) / 1e3 if x > 0 else float("nan")  # noqa: E731
print("pair | A: set-warp arrive, landed, mma commit | B: same | B - A (arrive)")
for pi in range(49):
    w = [4, 8, 12][pi % 3]
    m = 18 + pi % 2
    ra = (us(t[0, w, pi, 3]), us(t[0, w, pi, 1]), us(t[0, m, pi, 3]))
    rb = (us(t[1, w, pi, 3]), us(t[1, w, pi, 1]), us(t[1, m, pi, 3]))
    print(f"{pi:3d} | {ra[0]:7.2f} {ra[1]:7.2f} {ra[2]:7.2f} | {rb[0]:7.2f} {rb[1]:7.2f} {rb[2]:7.2f} | {rb[0] - ra[0]:6.2f}")
pr = [(t[1, 16, i, 0] - t0) / 1e3 for i in range(40)]
print("producer A (before/after empty wait):", [(round(us(t[0, 16, i, 0]), 2), round(us(t[0, 16, i, 1]), 2)) for i in range(0, 40, 4)])
print("producer B (before/after empty wait):", [(round(us(t[1, 16, i, 0]), 2), round(us(t[1, 16, i, 1]), 2)) for i in range(0, 40, 4)])
print("MMA issuer events (before a_full wait, a_full acquired, commit issued) for A and B:")
for pi in range(10, 20):
    m = 18 + pi % 2
    print(pi, [round(us(t[0, m, pi, e]), 2) for e in (0, 1, 2, 3)], [round(us(t[1, m, pi, e]), 2) for e in (0, 1, 2, 3)])
for pi in range(44, 49):
    m = 18 + pi % 2
    print(pi, [round(us(t[0, m, pi, e]), 2) for e in (0, 1, 2, 3)], [round(us(t[1, m, pi, e]), 2) for e in (0, 1, 2, 3)])
