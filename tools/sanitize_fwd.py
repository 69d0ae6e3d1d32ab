"""Small forwards through every kernel path, for compute-sanitizer (memcheck / racecheck / synccheck):
    compute-sanitizer --tool racecheck python tools/sanitize_fwd.py
GEMV (M = 4, G = 32 / 128), A7 weights-as-TMEM (M = 40),
A7 SS GEMM (M = 160), naive staged path."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2402_04925_b200 as tpq  # noqa: E402
import synth  # noqa: E402

for (K1, N1, N2, G, M, variant) in [(256, 512, 256, 32, 4, tpq.TPQ_TP_AWARE), (1024, 1408, 640, 128, 4, tpq.TPQ_TP_AWARE),
                                     (1024, 1408, 640, 128, 40, tpq.TPQ_TP_AWARE), (1024, 2048, 768, 128, 160, tpq.TPQ_TP_AWARE),
                                     (512, 1024, 512, 64, 5, tpq.TPQ_NAIVE)]:
    p = synth.make_problem(K1, N1, N2, G, M, seed=1)
    P1, _ = tpq.gptq_reorder(p.w1.g_idx, p.w1.G)
    P2, _ = tpq.gptq_reorder(p.w2.g_idx, p.w2.G)
    h = tpq.TpMlp(p.w1, p.w2, P1, P2, M_max=256, variant=variant)
    X = torch.from_numpy(p.X).cuda()
    Y = torch.empty(M, p.N2, dtype=torch.float16, device="cuda")
    for _ in range(2):
        h.forward(X, M, Y)
    torch.cuda.synchronize()
    print("ok", K1, N1, N2, G, M, variant, float(Y.float().abs().mean()))
    h.close()
