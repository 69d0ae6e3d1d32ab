"""Per-CTA timeline of the GEMV kernels of the last forward (profiling build):
    TPQ_LIB_PATH=paper_2402_04925_b200/libtpq_prof.so python tools/cta_times.py --m 1
Per CTA (globaltimer): entry, work start (activations available), end, SM id, split-tile publish,
reducer wait start / end, reducer's own accumulator final."""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2402_04925_b200 as tpq  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="llama70b")
ap.add_argument("--m", type=int, default=1)
ap.add_argument("--sim-tp", type=int, default=1)
a = ap.parse_args()
p = synth.make_named(a.shape, 16, 0)
P1, _ = tpq.gptq_reorder(p.w1.g_idx, p.G)
P2, _ = tpq.gptq_reorder(p.w2.g_idx, p.G)
R = 2 if a.sim_tp == 1 else 8  # rotate replicas: cold L2 as in bench.py
hs = [tpq.TpMlp(p.w1, p.w2, P1, P2, tp=a.sim_tp, rank=0, M_max=16) for _ in range(R)]
X = torch.from_numpy(p.X).cuda()
Y = torch.empty(16, p.N2, dtype=torch.float16, device="cuda")
for i in range(10 * R + 1):
    hs[i % R].forward_local(X, a.m, Y)
torch.cuda.synchronize()
L = tpq.lib()
L.tpq_debug_cta.argtypes = [C.c_void_p]
buf = (C.c_ulonglong * (2 * 1024 * 16))()
L.tpq_debug_cta(C.cast(buf, C.c_void_p))
t = np.array(buf, dtype=np.int64).reshape(2, 1024, 16)
n1 = p.N1 // a.sim_tp
geo = {1: (p.K1 // 128, n1 // 128), 2: (n1 // 128, p.N2 // 128)}  # (NKB, NT)
slot = {1: int(n1 > p.K1), 2: int(p.N2 > n1)}  # the kernel files a launch under slot N > K
assert slot[1] != slot[2]
T0 = t[slot[1]][t[slot[1]][:, 0] > 0][:, 1].min()  # layer-1 work start: common origin
for layer in (1, 2):
    v = t[slot[layer]]
    grid = int((v[:, 0] > 0).sum())
    v = v[:grid]
    us = lambda x: (x - T0) / 1e3  # noqa: E731
    ent, ws, end = us(v[:, 0]), us(v[:, 1]), us(v[:, 3 - 1])
    print(f"layer {layer}: {grid} CTAs; entry [{ent.min():.2f}, {ent.max():.2f}]; work start [{ws.min():.2f}, {ws.max():.2f}];"
          f" end min {end.min():.2f} p10 {np.percentile(end, 10):.2f} med {np.median(end):.2f} p90 {np.percentile(end, 90):.2f}"
          f" max {end.max():.2f}  (us from layer-1 work start)")
    mhz = (v[:, 9] - v[:, 8]) / np.maximum(1, v[:, 2] - v[:, 0]) * 1e3
    print(f"   SM clock over the CTA's life: med {np.median(mhz):.0f} MHz (min {mhz.min():.0f})")
    NKB, NT = geo[layer]
    U = NKB * NT
    pub = v[:, 4] > 0
    red = v[:, 5] > 0
    if pub.any():
        print(f"   publish (after start): med {np.median(us(v[pub, 4]) - ws[pub]):.2f}")
    if red.any():
        wstart, wend, own = us(v[red, 5]), us(v[red, 6]), us(v[red, 7])
        print(f"   reducers {red.sum()}: wait {np.median(wend - wstart):.2f} med / {np.max(wend - wstart):.2f} max; "
              f"own final - wait end med {np.median(own - wend):.2f}; end - own final med {np.median(end[red] - own):.2f} max {np.max(end[red] - own):.2f}")
    fa, lc = us(v[:, 10]), us(v[:, 11])
    print(f"   first pair stored - work start: med {np.median(fa - ws):.2f} max {np.max(fa - ws):.2f}; "
          f"last commit - first pair: med {np.median(lc - fa):.2f} min {np.min(lc - fa):.2f} max {np.max(lc - fa):.2f}; "
          f"end - last commit: med {np.median(end - lc):.2f} max {np.max(end - lc):.2f}")
    wl, xl = us(v[:, 14]), us(v[:, 13])
    print(f"   unit 0 weights landed - work start: med {np.median(wl - ws):.2f} max {np.max(wl - ws):.2f}; "
          f"pair 0 activations seen - work start: med {np.median(xl - ws):.2f} max {np.max(xl - ws):.2f} "
          f"(after the pair's dequant)")
    order = np.argsort(end)
    for c in list(order[:3]) + list(order[-8:]):
        u0, u1 = c * U // grid, (c + 1) * U // grid
        c_last = lambda tile: ((((tile + 1) * NKB - 1) + 1) * grid + U - 1) // U - 1  # noqa: E731
        info = f"units {u1 - u0} first-kb {u0 % NKB} last-tile-units {(u1 - 1) % NKB + 1}"
        if v[c, 5] > 0:
            tile = (u1 - 1) // NKB
            others = range(c + 1, c_last(tile) + 1)
            pubs = [round(float(us(v[o, 4])), 2) if v[o, 4] > 0 else None for o in others]
            ends = [round(float(end[o]), 2) for o in others]
            info += (f" | reduce: wait {us(v[c, 5]):.2f}->{us(v[c, 6]):.2f} own {us(v[c, 7]):.2f} warps done "
                     f"{[round(float(us(v[c, 12 + q])), 2) for q in range(4)]}; others {list(others)}"
                     f" publish {pubs} end {ends}")
        print(f"   cta {c:3d} sm {int(v[c, 3]):3d} end {end[c]:.2f} (first pair {fa[c]:.2f}, last commit {lc[c]:.2f}) {info}")
