"""Stress: repeated layer-1 runs of the register-dequant GEMV must be bit-identical (deterministic
kernel); reports which tiles / columns / rows differ, and whether they are split (stream-K) tiles."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2402_04925_b200 as tpq  # noqa: E402
import synth  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 16
kind = tpq.TPQ_GEMV_REG if (len(sys.argv) < 3 or sys.argv[2] == "reg") else tpq.TPQ_GEMV_TC
p = synth.make_named("llama70b", M, 0)
P1, _ = tpq.gptq_reorder(p.w1.g_idx, p.G)
P2, _ = tpq.gptq_reorder(p.w2.g_idx, p.G)
h = tpq.TpMlp(p.w1, p.w2, P1, P2, M_max=16)
h.set_gemv_kernel(kind)
X = torch.from_numpy(p.X).cuda()
Y = torch.empty(M, p.N2, dtype=torch.float16, device="cuda")
ref = torch.empty(M, p.N1, dtype=torch.float16, device="cuda")
h.layer1(X, M, ref)
torch.cuda.synchronize()
bad = 0
for it in range(60):
    if it % 2 == 0:
        h.forward(X, M, Y)
    Y1 = torch.full((M, p.N1), float("nan"), dtype=torch.float16, device="cuda")
    h.layer1(X, M, Y1)
    torch.cuda.synchronize()
    d = (Y1 != ref).cpu().numpy()
    if d.any():
        bad += 1
        rows, cols = np.nonzero(d)
        tiles = sorted(set((cols // 128).tolist()))
        print(f"iter {it}: {d.sum()} mismatches, rows {sorted(set(rows.tolist()))[:16]}, tiles {tiles[:12]}, "
              f"cols%128 sample {sorted(set((cols % 128).tolist()))[:16]}, nan {torch.isnan(Y1).sum().item()}")
print("bad iterations", bad, "of 60")
