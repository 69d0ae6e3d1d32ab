"""Run a few TP=1 forwards (target for ncu captures):
    ncu --set full -k regex:k_tcgemv -s 4 -c 1 python tools/run_fwd.py --m 1"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2402_04925_b200 as tpq  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="llama70b")
ap.add_argument("--m", type=int, default=1)
ap.add_argument("--iters", type=int, default=6)
a = ap.parse_args()
p = synth.make_named(a.shape, 16, 0)
P1, _ = tpq.gptq_reorder(p.w1.g_idx, p.G)
P2, _ = tpq.gptq_reorder(p.w2.g_idx, p.G)
h = tpq.TpMlp(p.w1, p.w2, P1, P2, tp=1, M_max=16)
X = torch.from_numpy(p.X).cuda()
Y = torch.empty(16, p.N2, dtype=torch.float16, device="cuda")
for _ in range(a.iters):
    h.forward_local(X, a.m, Y)
torch.cuda.synchronize()
print("ok")
