"""Small forwards through every kernel path, for compute-sanitizer (memcheck / racecheck / synccheck):
    compute-sanitizer --tool memcheck python tools/sanitize_fwd.py
GEMV k_dqgemv (M = 1 / 4 / 5, G = 32 / 128; split tiles reduced in-kernel, and by k_split_fixup /
k_mm_fixup where a tile spans more than 4 CTA ranges: K1 = 4096, N1 = 1024), gated k_dqgemv<G,true>,
unordered k_dqgemv<0>, A7 weights-as-TMEM (M = 40), A7 SS GEMM (M = 160), naive staged path with the
P2 gather (k_gather_ag)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2402_04925_b200 as tpq  # noqa: E402
import synth  # noqa: E402


def run(h, p, M, label):
    X = torch.from_numpy(p.X[:M].copy()).cuda()
    Y = torch.empty(M, p.N2, dtype=torch.float16, device="cuda")
    for _ in range(2):
        h.forward(X, M, Y)
    torch.cuda.synchronize()
    print("ok", label, float(Y.float().abs().mean()), flush=True)
    h.close()


for (K1, N1, N2, G, M, variant) in [(256, 512, 256, 32, 4, tpq.TPQ_TP_AWARE), (1024, 1408, 640, 128, 1, tpq.TPQ_TP_AWARE),
                                     (1024, 1408, 640, 128, 5, tpq.TPQ_TP_AWARE), (1024, 1408, 640, 128, 40, tpq.TPQ_TP_AWARE),
                                     (1024, 2048, 768, 128, 160, tpq.TPQ_TP_AWARE), (512, 1024, 512, 64, 5, tpq.TPQ_NAIVE),
                                     (4096, 1024, 512, 128, 5, tpq.TPQ_TP_AWARE), (4096, 1024, 512, 128, 1, tpq.TPQ_TP_AWARE)]:
    p = synth.make_problem(K1, N1, N2, G, M, seed=1)
    P1, _ = tpq.gptq_reorder(p.w1.g_idx, p.w1.G)
    P2, _ = tpq.gptq_reorder(p.w2.g_idx, p.w2.G)
    run(tpq.TpMlp(p.w1, p.w2, P1, P2, M_max=256 if M > 16 else 16, variant=variant), p, M, f"{K1}x{N1}x{N2} G={G} M={M} v={variant}")
# gated (f2) at M = 2 (split fix-up) and M = 9 (k_mm_fixup)
for M in (2, 9):
    p = synth.make_problem(1024, 1408, 640, 128, M, seed=2)
    q = synth.make_problem(1024, 1408, 640, 128, M, seed=1002)
    Ps = [tpq.gptq_reorder(w.g_idx, 128)[0] for w in (p.w1, q.w1, p.w2)]
    run(tpq.TpMlp.gated(p.w1, q.w1, p.w2, *Ps, M_max=16), p, M, f"gated M={M}")
# unordered (f3)
p = synth.make_problem(1024, 1408, 640, 64, 3, seed=3)
run(tpq.TpMlp(p.w1, p.w2, None, None, variant=tpq.TPQ_UNORDERED, M_max=16), p, 3, "unordered M=3")
# naive staged with the P2 gather at tp = 2 (rank 0's shard)
p = synth.make_problem(512, 2048, 512, 128, 3, seed=4)
P1, _ = tpq.gptq_reorder(p.w1.g_idx, 128)
P2, _ = tpq.gptq_reorder(p.w2.g_idx, 128)
h = tpq.TpMlp(p.w1, p.w2, P1, P2, tp=2, rank=0, variant=tpq.TPQ_NAIVE, M_max=16)
X = torch.from_numpy(p.X).cuda()
buf = torch.zeros(2, 3, 1024, dtype=torch.float16, device="cuda")
h.layer1(X, 3, buf[0])
y1 = torch.empty(3, 1024, dtype=torch.float16, device="cuda")
h.naive_gather(buf, 3, y1)
Y = torch.empty(3, 512, dtype=torch.float16, device="cuda")
h.layer2(y1, 3, Y)
torch.cuda.synchronize()
print("ok naive staged", flush=True)
h.close()
