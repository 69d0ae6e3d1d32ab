"""Minimal driver for ncu: a few TP-aware forwards of one config (no timing, no oracle).
    python tools/prof_forward.py --shape llama70b --m 16 --iters 6 [--sim-tp 8]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2402_04925_b200 as tpq  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="llama70b")
ap.add_argument("--m", type=int, default=16)
ap.add_argument("--iters", type=int, default=6)
ap.add_argument("--sim-tp", type=int, default=1)
ap.add_argument("--variant", default="tp_aware")
a = ap.parse_args()
p = synth.make_named(a.shape, a.m, 0)
P1, _ = tpq.gptq_reorder(p.w1.g_idx, p.G)
P2, _ = tpq.gptq_reorder(p.w2.g_idx, p.G)
v = tpq.TPQ_TP_AWARE if a.variant == "tp_aware" else tpq.TPQ_NAIVE
h = tpq.TpMlp(p.w1, p.w2, P1, P2, tp=a.sim_tp, rank=0, variant=v, M_max=16)
X = torch.from_numpy(p.X).cuda()
Y = torch.empty(a.m, p.N2, dtype=torch.float16, device="cuda")
for _ in range(a.iters):
    h.forward_local(X, a.m, Y)
torch.cuda.synchronize()
print("grid", h.info.grid1, h.info.grid2, "units", h.info.units1, h.info.units2)
