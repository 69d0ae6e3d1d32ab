"""k-step event timeline of pair 0 of the layer-1 CTA-pair SS GEMM (profiling build):
    TPQ_LIB_PATH=paper_2402_04925_b200/libtpq_prof.so python tools/trace_ss2.py --m 256
Rows (globaltimer ns, relative): dequant warp 0 of CTA 0 / 1 [before w_full, w_full, k_done(t-2), arrive];
A producer CTA 0 / 1 [before k_done(t-3), after]; W producer CTA 0 / 1 [before w_empty, after];
epilogue CTA 0 / 1 [d_full, done]; MMA [before a_full, a_full, b_full, committed]."""
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
ap.add_argument("--m", type=int, default=256)
ap.add_argument("--sim-tp", type=int, default=8)
a = ap.parse_args()
p = synth.make_named(a.shape, a.m, 0)
P1, _ = tpq.gptq_reorder(p.w1.g_idx, p.G)
P2, _ = tpq.gptq_reorder(p.w2.g_idx, p.G)
R = 4
hs = [tpq.TpMlp(p.w1, p.w2, P1, P2, tp=a.sim_tp, rank=0, M_max=a.m) for _ in range(R)]
X = torch.from_numpy(p.X).cuda()
Y = torch.empty(a.m, p.N2, dtype=torch.float16, device="cuda")
for i in range(4 * R + 1):
    hs[i % R].forward_local(X, a.m, Y)
torch.cuda.synchronize()
L = tpq.lib()
L.tpq_debug_trace.argtypes = [C.c_void_p]
tr = (C.c_longlong * (24 * 64 * 4))()
L.tpq_debug_trace(C.cast(tr, C.c_void_p))
T = np.array(tr, dtype=np.int64).reshape(24, 64, 4)
# clock64 per SM: rows of CTA 0 (deq0, apr0, wpr0, epi0, chunk rows 9) and the MMA row share one clock;
# CTA 1's rows (deq1, apr1, wpr1, epi1, 10) another.  Times in ns at 1.965 GHz, relative per CTA.
f = 1.0 / 1.965
for lay, off in (("layer 1", 0), ("layer 2", 12)):
    t = T[off:off + 11]
    if not (t > 0).any():
        continue
    c0rows, c1rows = [0, 2, 4, 6, 8, 9], [1, 3, 5, 7, 10]
    b0 = t[c0rows][t[c0rows] > 0].min()
    b1 = t[c1rows][t[c1rows] > 0].min() if (t[c1rows] > 0).any() else 0
    rel = np.full(t.shape, -1, np.int64)
    for r in range(11):
        b = b0 if r in c0rows else b1
        rel[r] = np.where(t[r] > 0, ((t[r] - b) * f).astype(np.int64), -1)
    n = int((rel[8, :, 0] >= 0).sum())
    print(lay, "k-steps traced:", n)
    names = ["deq0", "deq1", "apr0", "apr1", "wpr0", "wpr1", "epi0", "epi1", "mma"]
    for i in range(n):
        print(i, " | ".join(f"{names[r]} " + " ".join(f"{v:6d}" for v in rel[r, i]) for r in (0, 2, 4, 8, 1)))
    print("epilogue cta0", rel[6, :3].tolist(), "cta1", rel[7, :3].tolist())
    for c in range(8):
        print("  epi chunk", c, "cta0", rel[9, c].tolist(), "cta1", rel[10, c].tolist())
