"""Time TP-aware forwards (CUDA graph of 20, 2 replicas) for quick A/B experiments.
    python tools/fwd_time.py --shape llama70b --ms 1,4,16 [--sim-tp 1]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2402_04925_b200 as tpq  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="llama70b")
ap.add_argument("--ms", default="1,4,16")
ap.add_argument("--sim-tp", type=int, default=1)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
p = synth.make_named(a.shape, 16, 0)
P1, _ = tpq.gptq_reorder(p.w1.g_idx, p.G)
P2, _ = tpq.gptq_reorder(p.w2.g_idx, p.G)
R = 2 if a.sim_tp == 1 else 8
MM = max(16, max(int(m) for m in a.ms.split(",")))
hs = [tpq.TpMlp(p.w1, p.w2, P1, P2, tp=a.sim_tp, rank=0, M_max=MM) for _ in range(R)]
X = torch.from_numpy(synth.make_named(a.shape, MM, 0).X).cuda()
Y = torch.empty(MM, p.N2, dtype=torch.float16, device="cuda")
st = torch.cuda.Stream()
res = {}
for M in [int(m) for m in a.ms.split(",")]:
    with torch.cuda.stream(st):
        for i in range(10):
            hs[i % R].forward_local(X, M, Y, stream=st)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for i in range(20):
                hs[i % R].forward_local(X, M, Y, stream=st)
        for _ in range(3):
            g.replay()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(st)
        for _ in range(a.reps):
            g.replay()
        e.record(st)
    torch.cuda.synchronize()
    res[M] = s.elapsed_time(e) * 1e3 / (20 * a.reps)
print(a.shape, "tp", a.sim_tp, {k: round(v, 2) for k, v in res.items()})
