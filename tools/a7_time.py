"""Per-step device times of the A7 (M > 16) forward on one rank's Llama shard, for A/B experiments.
    python tools/a7_time.py --sim-tp 8 --ms 256,512        (graph-timed, cold weight replicas)
    python tools/a7_time.py --sim-tp 8 --ms 256 --once     (one eager forward: for ncu captures)"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2402_04925_b200 as tpq  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="llama70b")
ap.add_argument("--ms", default="256")
ap.add_argument("--sim-tp", type=int, default=8)
ap.add_argument("--once", action="store_true")
a = ap.parse_args()
Ms = [int(m) for m in a.ms.split(",")]
MM = max(Ms)
p = synth.make_named(a.shape, MM, 0)
P1, _ = tpq.gptq_reorder(p.w1.g_idx, p.G)
P2, _ = tpq.gptq_reorder(p.w2.g_idx, p.G)
R = 1 if a.once else (2 if a.sim_tp == 1 else 6)
hs = [tpq.TpMlp(p.w1, p.w2, P1, P2, tp=a.sim_tp, rank=0, M_max=MM) for _ in range(R)]
X = torch.from_numpy(p.X).cuda()
Y = torch.empty(MM, p.N2, dtype=torch.float16, device="cuda")
st = torch.cuda.Stream()
if a.once:
    with torch.cuda.stream(st):
        for M in Ms:
            hs[0].forward_local(X, M, Y, stream=st)
    torch.cuda.synchronize()
    sys.exit(0)
steps = [("gather", tpq.TPQ_STEP_GATHER), ("layer1", tpq.TPQ_STEP_LAYER1), ("layer2", tpq.TPQ_STEP_LAYER2)]
for M in Ms:
    with torch.cuda.stream(st):
        hs[0].forward_local(X, M, Y, stream=st)  # stages the step buffers
    res = {}
    for name, step in steps + [("forward", None)]:
        def call(i):
            if step is None:
                hs[i % R].forward_local(X, M, Y, stream=st)
            else:
                hs[i % R].run_step(step, M, stream=st)
        with torch.cuda.stream(st):
            for i in range(R):
                call(i)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                for i in range(12):
                    call(i)
            for _ in range(3):
                g.replay()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(st)
            for _ in range(10):
                g.replay()
            e.record(st)
        torch.cuda.synchronize()
        res[name] = round(s.elapsed_time(e) * 1e3 / 120, 2)
    fl = 2.0 * M * (p.K1 * p.N1 + p.N1 * p.N2) / a.sim_tp
    print(a.shape, "tp", a.sim_tp, "M", M, res, "TF/s", round(fl / (res["forward"] * 1e-6) / 1e12, 1), flush=True)
