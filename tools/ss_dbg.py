import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2402_04925_b200 as tpq, synth
G = int(sys.argv[1]); M = int(sys.argv[2])
p = synth.make_problem(1024, 1408, 640, G, M, seed=1)
P1, _ = tpq.gptq_reorder(p.w1.g_idx, p.w1.G); P2, _ = tpq.gptq_reorder(p.w2.g_idx, p.w2.G)
h = tpq.TpMlp(p.w1, p.w2, P1, P2, M_max=512)
X = torch.from_numpy(p.X).cuda(); Y = torch.empty(M, p.N2, dtype=torch.float16, device="cuda")
h.forward(X, M, Y); torch.cuda.synchronize(); print("ok", float(Y.float().abs().mean()))
