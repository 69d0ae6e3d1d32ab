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
t = np.array(tr, dtype=np.int64).reshape(24, 64, 4)[:9]
t0 = t[t > 0].min()
rel = np.where(t > 0, t - t0, -1)
names = ["deq0", "deq1", "apr0", "apr1", "wpr0", "wpr1", "epi0", "epi1", "mma"]
n = int((rel[8, :, 0] >= 0).sum())
print("k-steps traced:", n)
for i in range(n):
    print(i, " | ".join(f"{names[r]} " + " ".join(f"{v:6d}" for v in rel[r, i]) for r in (0, 1, 2, 3, 4, 8)))
print("epilogue", rel[6, :2], rel[7, :2])
