"""Graph-timed gated (gate_proj, f2) Llama forward at the given M values (cold weight replicas):
    python tools/gated_time.py --ms 1,16"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2402_04925_b200 as tpq  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ms", default="1,16")
a = ap.parse_args()
p = synth.make_named("llama70b", 16, 0)
q = synth.make_named("llama70b", 16, 1000)
ws = (p.w1, q.w1, p.w2)
Ps = [tpq.gptq_reorder(w.g_idx, p.G)[0] for w in ws]
hs = [tpq.TpMlp.gated(*ws, *Ps, M_max=16) for _ in range(2)]
X = torch.from_numpy(p.X).cuda()
Y = torch.empty(16, p.N2, dtype=torch.float16, device="cuda")
st = torch.cuda.Stream()
res = {}
for M in [int(m) for m in a.ms.split(",")]:
    with torch.cuda.stream(st):
        for i in range(6):
            hs[i % 2].forward_local(X, M, Y, stream=st)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for i in range(20):
                hs[i % 2].forward_local(X, M, Y, stream=st)
        g.replay()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(st)
        for _ in range(10):
            g.replay()
        e.record(st)
    torch.cuda.synchronize()
    res[M] = round(s.elapsed_time(e) * 1e3 / 200, 2)
print("gated", res)
