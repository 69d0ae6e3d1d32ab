"""Per-CTA entry / work-start / end times of the GEMV kernels of the last forward (profiling build):
    TPQ_LIB_PATH=paper_2402_04925_b200/libtpq_prof.so python tools/cta_times.py --m 1"""
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
buf = (C.c_ulonglong * (2 * 1024 * 4))()
L.tpq_debug_cta(C.cast(buf, C.c_void_p))
t = np.array(buf, dtype=np.int64).reshape(2, 1024, 4)
for layer in (0, 1):
    v = t[layer]
    v = v[v[:, 0] > 0]
    n = len(v)
    t0 = v[:, 1].min()
    ent, ws, end, sm = (v[:, 0] - t0) / 1e3, (v[:, 1] - t0) / 1e3, (v[:, 2] - t0) / 1e3, v[:, 3]
    print(f"layer {layer + 1}: {n} CTAs; entry [{ent.min():.2f}, {ent.max():.2f}] us; work start [{ws.min():.2f},"
          f" {ws.max():.2f}]; end min {end.min():.2f} p10 {np.percentile(end, 10):.2f} med {np.median(end):.2f}"
          f" p90 {np.percentile(end, 90):.2f} max {end.max():.2f}")
    dur = end - ws
    print(f"   busy (end - work start): min {dur.min():.2f} med {np.median(dur):.2f} max {dur.max():.2f}")
    for lo, hi in ((0, 74), (74, 148)):
        sel = (sm >= lo) & (sm < hi)
        if sel.any():
            print(f"   smid {lo}-{hi - 1}: {sel.sum()} CTAs, end med {np.median(end[sel]):.2f} max {end[sel].max():.2f}")
    order = np.argsort(end)
    print("   earliest:", [(int(i), int(sm[i]), round(float(end[i]), 2)) for i in order[:6]])
    print("   latest:  ", [(int(i), int(sm[i]), round(float(end[i]), 2)) for i in order[-6:]])
    # GPC-ish buckets of smid
    bk = {}
    for s_, e_ in zip(sm, end):
        bk.setdefault(int(s_) // 16, []).append(e_)
    print("   end med by smid//16:", {k: round(float(np.median(x)), 1) for k, x in sorted(bk.items())})
    # the CTAs sharing an SM
    by = {}
    for e_, s_ in zip(end, sm):
        by.setdefault(int(s_), []).append(e_)
    pairs = [sorted(x) for x in by.values() if len(x) == 2]
    if pairs:
        d = np.array([x[1] - x[0] for x in pairs])
        lo_ = np.array([x[0] for x in pairs])
        hi_ = np.array([x[1] for x in pairs])
        print(f"   SM pairs: {len(pairs)}; |dt| med {np.median(d):.2f} max {d.max():.2f}; first-finisher med "
              f"{np.median(lo_):.2f}, second med {np.median(hi_):.2f} max {hi_.max():.2f}")

# correlate layer-1 end times with the CTA's stream-K range: offset of its first unit in its tile,
# number of tile segments, whether it is the last arriver (fix-up) of its first / last tile
if os.environ.get("TPQ_CTA_CORR"):
    K1, N1 = p.K1, p.N1 // a.sim_tp
    NKB, NT = K1 // 128, N1 // 128
    U = NKB * NT
    v = t[0]
    grid = int((v[:, 0] > 0).sum())
    t0 = v[:grid, 1].min()
    ends = (v[:grid, 2] - t0) / 1e3
    rows = []
    for c in range(grid):
        u0, u1 = c * U // grid, (c + 1) * U // grid
        off = u0 % NKB
        nseg = (u1 - 1) // NKB - u0 // NKB + 1
        rows.append((ends[c], c, off, nseg, u1 - u0, (u1 - 1) % NKB))
    rows.sort()
    import collections
    by = collections.defaultdict(list)
    for e, c, off, nseg, n, last in rows:
        by[nseg].append(e)
    print("layer 1 end by #segments:", {k: (len(x), round(float(np.median(x)), 2)) for k, x in sorted(by.items())})
    for e, c, off, nseg, n, last in rows[:8] + rows[-12:]:
        print(f"  cta {c:3d} end {e:6.2f} first-kb {off:2d} last-kb {last:2d} segs {nseg} units {n}")
    offs = np.array([r[2] for r in rows]); es = np.array([r[0] for r in rows])
    print("corr(end, first-kb) =", round(float(np.corrcoef(offs, es)[0, 1]), 3),
          " corr(end, last-kb) =", round(float(np.corrcoef(np.array([r[5] for r in rows]), es)[0, 1]), 3))
