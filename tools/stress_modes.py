"""Race stress for the split-tile reductions: many back-to-back forwards (graph replays, cold weight
replicas) of each partition mode must all be bit-identical to the first one.
    python tools/stress_modes.py [--reps 50]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2402_04925_b200 as tpq  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=50)
a = ap.parse_args()
fails = 0
for shape, tp, M, mmax in [("llama70b", 1, 16, 16), ("llama70b", 1, 1, 16), ("granite20b", 1, 16, 16),
                           ("llama70b", 2, 16, 16), ("llama70b", 4, 16, 16), ("llama70b", 8, 1, 16),
                           ("llama70b", 8, 16, 16), ("llama70b", 1, 32, 32), ("llama70b", 8, 32, 32)]:
    p = synth.make_named(shape, mmax, 0)
    P1, _ = tpq.gptq_reorder(p.w1.g_idx, p.G)
    P2, _ = tpq.gptq_reorder(p.w2.g_idx, p.G)
    hs = [tpq.TpMlp(p.w1, p.w2, P1, P2, tp=tp, rank=tp - 1, M_max=mmax) for _ in range(2)]
    X = torch.from_numpy(p.X[:M].copy()).cuda()
    Ys = [torch.empty(M, p.N2, dtype=torch.float16, device="cuda") for _ in range(2)]
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for i in range(4):
            hs[i % 2].forward_local(X, M, Ys[i % 2], stream=st)
    torch.cuda.synchronize()
    ref = [y.clone() for y in Ys]
    with torch.cuda.stream(st):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for i in range(16):
                hs[i % 2].forward_local(X, M, Ys[i % 2], stream=st)
    bad = 0
    for r in range(a.reps):
        g.replay()
        torch.cuda.synchronize()
        for k in range(2):
            if not torch.equal(Ys[k], ref[k]):
                bad += 1
    info = hs[0].info
    print(f"{shape} tp={tp} M={M}: split modes ({info.split1}, {info.split2}), {a.reps * 16} forwards, "
          f"{bad} replay(s) with a differing output", flush=True)
    fails += bad
    for h in hs:
        h.close()
print("FAILED" if fails else "all bit-identical")
sys.exit(1 if fails else 0)
