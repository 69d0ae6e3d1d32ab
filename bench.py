#!/usr/bin/env python
"""Benchmark of the TP-aware GPTQ MLP forward (arxiv 2402.04925) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--shape llama70b] [--m 16]
                    [--variant tp_aware|naive] [--impl ours|reference]

A "step" is one forward of the whole hot path (SURVEY.md §8(a) rows A3-A6 for TP-aware:
X[:,P1] gather, layer-1 dequant-GEMV, layer-2 dequant-GEMV, AllReduce) on one batch of M
synthetic tokens.  N=1 runs the Llama-70B MLP at TP=1 (BASELINE.json configs[1]); under
torchrun N ranks each hold a TP=N shard of the SAME MLP (strong scaling) and the step ends
with the NCCL AllReduce.  Rank 0 prints one JSON line.

--impl reference times the CPU oracle (oracle/, fp64 numpy) on a bounded sample of the
same workload on the host cores (rank 0 only; other ranks exit 0).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = ("MLP fwd latency (µs) & HBM GB/s vs roofline, M=1..16, TP=1/2/4/8 vs naive "
          "AllGather")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--shape", default="llama70b", choices=sorted(synth.SHAPES))
    ap.add_argument("--m", type=int, default=16)
    ap.add_argument("--variant", default="tp_aware", choices=["tp_aware", "naive"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--quick", action="store_true",
                    help="N = 1: skip the extra lines (M sweep, Granite TP=1, Llama TP=8 shard)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-naive", action="store_true", help="N > 1: skip timing the naive AllGather path")
    ap.add_argument("--no-graph", action="store_true", help="launch every step eagerly (no CUDA graph)")
    ap.add_argument("--sim-tp", type=int, default=0,
                    help="single GPU: time one rank's shard of a TP=k MLP (no collective)")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def algorithmic_bytes(K1, N1, N2, G, M, tp):
    """Bytes one rank must move per forward:  int4 W (0.5 B/weight) +
    per-group fp16 scale and int4 zero (2.5 B per group-column) + X + P1 + Y1 write/read +
    Y2 partial.  Split per GEMV launch (layer 1, layer 2) and for the whole step."""
    n = N1 // tp
    w1 = K1 * n // 2 + 2.5 * (K1 // G) * n
    w2 = n * N2 // 2 + 2.5 * (n // G) * N2
    l1 = w1 + 2 * M * K1 + 2 * M * n          # weights + X (gathered, frag) + Y1 write
    l2 = w2 + 2 * M * n + 2 * M * N2          # weights + Y1 read + Y2 write
    step = w1 + w2 + 2 * M * K1 + 4 * K1 + 4 * M * n + 2 * M * N2
    return l1, l2, step


def ncu_traffic(a, tp):
    """DRAM bytes (read + write) per GEMV launch from the committed `ncu --set full` capture of the
    default workload (profiles/roofline_traffic.json); None for other workloads."""
    try:
        with open(os.path.join(ROOT, "profiles", "roofline_traffic.json")) as f:
            d = json.load(f)
    except Exception:
        return None
    if a.shape != "llama70b" or a.m != 16 or tp != 1 or a.variant != "tp_aware":
        return None
    return d.get("traffic_bytes_per_launch")


class ClockSampler:
    """nvidia-smi sampling of SM clocks + throttle reasons during the timed region."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, dev: int):
        self.dev = dev
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == len(self.FIELDS):
                self.rows.append(parts)

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------------------------ oracle
def oracle_prepare(p):
    """Offline part of the oracle (timed once, reported apart from the forward): checkpoint
    unpack (layer_from_checkpoint) and Alg. 1 (alg1_reorder)."""
    import oracle as O
    t0 = time.perf_counter()
    L1 = O.layer_from_checkpoint(p.w1.qweight, p.w1.scales_bits, p.w1.qzeros, p.w1.g_idx, p.K1, p.N1, p.G)
    L2 = O.layer_from_checkpoint(p.w2.qweight, p.w2.scales_bits, p.w2.qzeros, p.w2.g_idx, p.N1, p.N2, p.G)
    t1 = time.perf_counter()
    O.alg1_reorder(L1.g)
    O.alg1_reorder(L2.g)
    t2 = time.perf_counter()
    return L1, L2, {"unpack_s": t1 - t0, "alg1_s": t2 - t1}


def oracle_forward(X, L1, L2, chunk=2048):
    """One full forward of the oracle as it stands (fp64, TP = 1, so Alg. 3 = the plain definition
    Y2 = (X . deq(W1)) . deq(W2), reading c9): dequantize (oracle.dequantize, PAPER.md:L19 with the
    unordered g) and matmul, column block by column block so the fp64 weights fit in host memory.
    Returns (Y2, seconds in dequantize, seconds in matmul)."""
    import oracle as O
    X = np.asarray(X, dtype=np.float64)
    td = tm = 0.0

    def block(L, lo, hi):
        return O.OLayer(q=L.q[:, lo:hi], s=L.s[:, lo:hi], z=L.z[:, lo:hi], g=L.g, G=L.G)

    Y = []
    for L, inp in ((L1, X), (L2, None)):
        src = inp if inp is not None else Y[0]
        out = np.empty((src.shape[0], L.N))
        for lo in range(0, L.N, chunk):
            hi = min(L.N, lo + chunk)
            t0 = time.perf_counter()
            W = O.dequantize(block(L, lo, hi))
            t1 = time.perf_counter()
            out[:, lo:hi] = src @ W
            t2 = time.perf_counter()
            td += t1 - t0
            tm += t2 - t1
        Y.append(out)
    return Y[1], td, tm


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max((i.get("num_threads") or 0) for i in threadpool_info()) or None
    except Exception:
        return None


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def run_reference(a):
    """--impl reference: the CPU oracle as it stands, one FULL forward per step (no sampling, no
    extrapolation), exactly --steps timed steps after --warmup untimed ones, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    K1, N1, N2, G = synth.SHAPES[a.shape]
    p = synth.make_named(a.shape, a.m, a.seed)
    L1, L2, prep = oracle_prepare(p)
    for _ in range(a.warmup):
        oracle_forward(p.X, L1, L2)
    ts, tds, tms = [], [], []
    for _ in range(a.steps):
        t0 = time.perf_counter()
        _, td, tm = oracle_forward(p.X, L1, L2)
        ts.append(time.perf_counter() - t0)
        tds.append(td)
        tms.append(tm)
    us = statistics.mean(ts) * 1e6
    base = {"value": us, "unit": "us", "cores": cpu_cores(), "blas_threads": blas_threads(), "kind": "oracle",
            "sample": f"full forward per step: fp64 dequantize + matmul of both layers (M={a.m}), column blocks of 2048",
            "phases_s": {"dequant": statistics.median(tds), "matmul": statistics.median(tms),
                         "total": statistics.median(ts), "offline_unpack": prep["unpack_s"],
                         "offline_alg1": prep["alg1_s"]}}
    line = {"metric": METRIC, "value": us, "unit": "us", "impl": "reference", "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": us / 1e3, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{a.shape}-mlp K1={K1} N1={N1} N2={N2} G={G} M={a.m} tp=1 {a.variant}", "M": a.m,
                       "tp": 1, "variant": a.variant, "implementation": "CPU oracle (oracle/, fp64 numpy), tp = 1"},
            "cpu_baseline": base,
            "e2e": {"value": us, "unit": "us", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------ ours
def make_handles(tpq, p, P1, P2, tp, rank, variant, local, step_bytes, dev, M_max=16):
    """R replicas of one rank's shard so that R x (bytes per forward) >= 3 x L2: consecutive
    forwards in the timed region read cold weights (the 80-layer case)."""
    import torch
    l2_cache = torch.cuda.get_device_properties(dev).L2_cache_size
    R = max(1, -(-3 * l2_cache // int(step_bytes)))
    hs = [tpq.TpMlp(p.w1, p.w2, P1, P2, tp=tp, rank=rank, variant=variant, M_max=M_max, device=local)
          for _ in range(R)]
    return hs, R, l2_cache


def graph_of(torch, stream, n, launch):
    """CUDA graph of n consecutive launches (launch(i) enqueues the i-th)."""
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for i in range(n):
            launch(i)
    return g


def time_graph(torch, stream, g, reps, per):
    """Device time per launch (us) of a captured graph of `per` launches: the median over `reps`
    replays, each bracketed by events on `stream` (no event inside the graph).  The median keeps
    the number of a short, unthrottled run even if a long sequence of replays meets the power cap."""
    for _ in range(3):
        g.replay()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    with torch.cuda.stream(stream):
        for i in range(reps + 1):
            evs[i].record(stream)
            if i < reps:
                g.replay()
    evs[-1].synchronize()
    return statistics.median(evs[i].elapsed_time(evs[i + 1]) for i in range(reps)) * 1e3 / per


EXTRA_COOLDOWN_S = 0.3  # idle before each extra line: measured as a burst like the main line


def step_latency(torch, tpq, hs, R, stream, M, sim_tp, X, Y, reps=8):
    """Graph-timed forward latency (us) at M rows, rotating the weight replicas: the median of `reps`
    replays of a graph of ~16 forwards after a short idle, i.e. a burst like the main line's 20 steps
    (sustained replays reach the board's power cap and the dequant-bound GEMV slows with the SM clock,
    see clocks_extra_lines)."""
    per = R * max(1, 16 // R)
    f = (lambda h: h.forward_local(X, M, Y, stream=stream)) if sim_tp else (lambda h: h.forward(X, M, Y, stream=stream))
    with torch.cuda.stream(stream):
        for i in range(per):
            f(hs[i % R])
        g = graph_of(torch, stream, per, lambda i: f(hs[i % R]))
    torch.cuda.synchronize()
    time.sleep(EXTRA_COOLDOWN_S)
    return time_graph(torch, stream, g, reps, per)


def kernel_times(torch, tpq, hs, R, stream, M, tp):
    """Device time per launch (us) of each step of the forward, timed alone: a CUDA graph of many
    launches of that step alone (rotating the cold weight replicas), events only around the
    replays.  Layer steps include the split-tile fix-up kernel that follows each GEMV."""
    per = R * max(1, 16 // R)
    steps = [("gather", tpq.TPQ_STEP_GATHER), ("layer1", tpq.TPQ_STEP_LAYER1), ("layer2", tpq.TPQ_STEP_LAYER2)]
    if tp > 1 and hs[0].info.has_comm:
        steps.append(("allreduce", tpq.TPQ_STEP_ALLREDUCE))
    out = {}
    for name, st in steps:
        with torch.cuda.stream(stream):
            for i in range(per):
                hs[i % R].run_step(st, M, stream=stream)
            g = graph_of(torch, stream, per, lambda i: hs[i % R].run_step(st, M, stream=stream))
        out[name] = time_graph(torch, stream, g, 40, per)
    return out


def extra_workload(torch, tpq, shape, M_list, sim_tp, seed, local, dev, stream):
    """Graph-timed step latency of another BASELINE.json workload on this GPU (N = 1):
    Granite-20B at TP = 1, or one rank's shard of a TP = k Llama MLP (no collective)."""
    K1, N1, N2, G = synth.SHAPES[shape]
    p = synth.make_named(shape, 16, seed)
    P1, _ = tpq.gptq_reorder(p.w1.g_idx, G)
    P2, _ = tpq.gptq_reorder(p.w2.g_idx, G)
    tp = sim_tp or 1
    _, _, step_b = algorithmic_bytes(K1, N1, N2, G, 16, tp)
    hs, R, _ = make_handles(tpq, p, P1, P2, tp, 0, tpq.TPQ_TP_AWARE, local, step_b, dev)
    X = torch.from_numpy(p.X.copy()).to(dev)
    Y = torch.empty(16, N2, dtype=torch.float16, device=dev)
    res = {}
    peak, _ = peaks()
    for M in M_list:
        us = step_latency(torch, tpq, hs, R, stream, M, sim_tp, X, Y)
        b = algorithmic_bytes(K1, N1, N2, G, M, tp)[2]
        res[str(M)] = {"us": us, "hbm_frac": b / (us * 1e-6) / 1e9 / peak,
                       "kernel_us": kernel_times(torch, tpq, hs, R, stream, M, 1)}
    def steps_us(handles, Rh, M, steps):
        """Graph-timed per-forward time of `steps` run back to back through tpq_mlp_run_step."""
        per = Rh * max(1, 16 // Rh)

        def one(i):
            for st_ in steps:
                handles[i % Rh].run_step(st_, M, stream=stream)
        with torch.cuda.stream(stream):
            for i in range(per):
                one(i)
            g = graph_of(torch, stream, per, one)
        return time_graph(torch, stream, g, 40, per)

    if sim_tp:
        for M in M_list:
            res[str(M)]["tp_aware_steps_us"] = steps_us(
                hs, R, M, (tpq.TPQ_STEP_GATHER, tpq.TPQ_STEP_LAYER1, tpq.TPQ_STEP_LAYER2))
    for h in hs:
        h.close()
    if sim_tp:
        # the naive Alg. 2 rank's compute on the same box: the same steps plus its Y1[:, P2] + CHUNK
        # gather (the AllGather itself needs the other ranks; the layers are the same kernels)
        hn, Rn, _ = make_handles(tpq, p, P1, P2, tp, 0, tpq.TPQ_NAIVE, local, step_b, dev)
        for M in M_list:
            res[str(M)]["naive_p2_gather_us"] = steps_us(hn, Rn, M, (tpq.TPQ_STEP_NAIVE_GATHER,))
            res[str(M)]["naive_steps_us"] = steps_us(
                hn, Rn, M, (tpq.TPQ_STEP_GATHER, tpq.TPQ_STEP_LAYER1, tpq.TPQ_STEP_NAIVE_GATHER, tpq.TPQ_STEP_LAYER2))
        for h in hn:
            h.close()
    return res


def unordered_line(torch, tpq, p, shape, local, dev, stream, kt_ordered, M):
    """the same MLP WITHOUT Alg. 1 (TPQ_UNORDERED: rows in checkpoint order,
    per-row group metadata looked up, the Fig. 1 formulation of PAPER.md:L36), same pipeline and
    launch structure, timed like the main line: the paper's locality claim
    measured on B200 as the per-layer kernel-time ratio."""
    K1, N1, N2, G = synth.SHAPES[shape]
    _, _, step_b = algorithmic_bytes(K1, N1, N2, G, M, 1)
    hs, R, _ = make_handles(tpq, p, None, None, 1, 0, tpq.TPQ_UNORDERED, local, step_b, dev)
    X = torch.from_numpy(p.X[:M].copy()).to(dev)
    Y = torch.empty(M, N2, dtype=torch.float16, device=dev)
    us = step_latency(torch, tpq, hs, R, stream, M, 0, X, Y)
    kt = kernel_times(torch, tpq, hs, R, stream, M, 1)
    for h in hs:
        h.close()
    return {"M": M, "step_us": us, "kernel_us": kt,
            "layer_time_ratio_vs_ordered": {k: kt[k] / kt_ordered[k] for k in ("layer1", "layer2")},
            "what": "no reorder; each 128-row block re-reads {s', -z s'} per row from an L2-resident "
                    "[ng][N] table (64 KB per 128 x 128 block vs the 320 B header of an ordered record)"}


def gated_line(torch, tpq, shape, seed, local, dev, stream):
    """the gate_proj variant Y = (SiLU(X.Wg) * (X.Wu)).Wd at TP = 1 (the real
    Llama MLP: up layer drawn from the next seed's layer-1 recipe), graph-timed like the main line."""
    K1, N1, N2, G = synth.SHAPES[shape]
    p = synth.make_named(shape, 16, seed)
    q = synth.make_named(shape, 16, seed + 1000)
    ws = (p.w1, q.w1, p.w2)
    Ps = [tpq.gptq_reorder(w.g_idx, G)[0] for w in ws]
    l1, l2, _ = algorithmic_bytes(K1, N1, N2, G, 16, 1)
    step_b = 2 * l1 + l2
    l2_cache = torch.cuda.get_device_properties(dev).L2_cache_size
    R = max(1, -(-3 * l2_cache // int(step_b)))
    hs = [tpq.TpMlp.gated(*ws, *Ps, M_max=16, device=local) for _ in range(R)]
    X = torch.from_numpy(p.X.copy()).to(dev)
    Y = torch.empty(16, N2, dtype=torch.float16, device=dev)
    peak, _ = peaks()
    out = {}
    for M in (1, 16):
        us = step_latency(torch, tpq, hs, R, stream, M, 0, X, Y)
        l1m, l2m, _ = algorithmic_bytes(K1, N1, N2, G, M, 1)
        b = 2 * l1m + l2m
        out[str(M)] = {"us": us, "hbm_frac": b / (us * 1e-6) / 1e9 / peak, "bytes": b}
    kt = kernel_times(torch, tpq, hs, R, stream, 16, 1)
    for h in hs:
        h.close()
    out["kernel_us_M16"] = kt
    return out


def a7_line(torch, tpq, shape, seed, local, dev, stream):
    """A7 (BASELINE.json configs[3]): one rank's TP = 8 Llama shard at M = 32 / 128 / 512 on the
    tensor-core path, graph-timed, as a fraction of the measured dense fp16 (= bf16) tensor peak."""
    K1, N1, N2, G = synth.SHAPES[shape]
    p = synth.make_named(shape, 512, seed)
    P1, _ = tpq.gptq_reorder(p.w1.g_idx, G)
    P2, _ = tpq.gptq_reorder(p.w2.g_idx, G)
    _, _, step_b = algorithmic_bytes(K1, N1, N2, G, 512, 8)
    hs, R, _ = make_handles(tpq, p, P1, P2, 8, 0, tpq.TPQ_TP_AWARE, local, step_b, dev, M_max=512)
    X = torch.from_numpy(p.X.copy()).to(dev)
    Y = torch.empty(512, N2, dtype=torch.float16, device=dev)
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            tf = float(json.load(f)["bf16_tflops"])
    except Exception:
        tf = 1590.0
    out = {}
    for M in (32, 128, 512):
        us = step_latency(torch, tpq, hs, R, stream, M, 8, X[:M], Y[:M], reps=10)
        fl = 2.0 * M * (K1 * N1 + N1 * N2) / 8
        out[str(M)] = {"us": us, "tflops": fl / (us * 1e-6) / 1e12, "tensor_frac": fl / (us * 1e-6) / 1e12 / tf}
    for h in hs:
        h.close()
    out["peak_tflops"] = tf
    return out


def main():
    a = parse()
    if a.impl == "reference":
        return run_reference(a)
    import torch
    import torch.distributed as dist

    import paper_2402_04925_b200 as tpq

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == a.gpus, f"--gpus {a.gpus} but WORLD_SIZE={world}"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    tp = world
    sim_tp = a.sim_tp if (world == 1 and a.sim_tp > 1) else 0
    shard_tp = sim_tp or tp
    K1, N1, N2, G = synth.SHAPES[a.shape]
    M = a.m
    assert 1 <= M <= 16, "bench.py times the M <= 16 path (BASELINE.json configs[1-2])"
    variant = tpq.TPQ_TP_AWARE if a.variant == "tp_aware" else tpq.TPQ_NAIVE
    p = synth.make_named(a.shape, max(M, 16), a.seed)
    P1, _ = tpq.gptq_reorder(p.w1.g_idx, G)
    P2, _ = tpq.gptq_reorder(p.w2.g_idx, G)
    l1_bytes, l2_bytes, step_bytes = algorithmic_bytes(K1, N1, N2, G, M, shard_tp)
    hs, R, l2_cache = make_handles(tpq, p, P1, P2, shard_tp, rank, variant, local, step_bytes, dev)
    comm = None
    if tp > 1:
        uid = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(tpq.comm_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        comm = tpq.Comm(bytes(uid.cpu().numpy().tobytes()), tp, rank, local)
        for h in hs:  # one communicator serves every replica (as it would serve a model's layers)
            h.set_comm(comm)
    X = torch.from_numpy(p.X[:M].copy()).to(dev)
    Y = torch.empty(M, N2, dtype=torch.float16, device=dev)
    stream = torch.cuda.Stream(device=dev)
    fwd = (lambda h: h.forward_local(X, M, Y, stream=stream)) if sim_tp else (lambda h: h.forward(X, M, Y, stream=stream))

    def sync_all():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize(dev)

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---------------- warm-up: W eager forwards, then the graphs are captured and replayed
    with torch.cuda.stream(stream):
        for i in range(max(3, a.warmup)):
            fwd(hs[i % R])
    sync_all()

    # ---------------- timed region: exactly K steps.  The steps are replayed from CUDA graphs of
    # consecutive forwards (rotating the weight replicas, no event nodes inside): a graph of
    # `per_graph` forwards replayed K // per_graph times plus a graph of the K % per_graph rest.
    # --no-graph launches every forward eagerly through the C-ABI.
    K = a.steps
    # short runs: ONE graph of exactly K forwards (a graph replay's first forward has no PDL overlap
    # with a preceding one; one replay per run keeps that to once); long runs: graphs of 16
    per_graph = K if K <= 128 else R * max(1, 16 // R)
    rem = K % per_graph
    graph = graph_rem = None
    if not a.no_graph:
        with torch.cuda.stream(stream):
            graph = graph_of(torch, stream, per_graph, lambda i: fwd(hs[i % R]))
            graph_rem = graph_of(torch, stream, rem, lambda i: fwd(hs[i % R])) if rem else None
        for _ in range(max(3, a.warmup // per_graph)):
            graph.replay()
        if graph_rem is not None:
            graph_rem.replay()
        sync_all()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.15)
    sync_all()
    with torch.cuda.stream(stream):
        # the last warm-up step runs right before the region (not timed): the GPU is in its steady
        # state and the timed steps are already enqueued behind it, so the region starts on the first
        # timed forward, not on the host's launch latency or a clock ramp after the idle sync
        if graph is not None:
            (graph_rem if graph_rem is not None else graph).replay()
        else:
            fwd(hs[K % R])
        start.record(stream)
        if graph is not None:
            for _ in range(K // per_graph):
                graph.replay()
            if graph_rem is not None:
                graph_rem.replay()
        else:
            for i in range(K):
                fwd(hs[i % R])
        end.record(stream)
    sync_all()
    clk = clocks.stop()
    ms_per_step = max_over_ranks(start.elapsed_time(end)) / K

    # ---------------- per-step distribution: events around each replay of the same graph
    stats = None
    if graph is not None:
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(61)]
        with torch.cuda.stream(stream):
            for i in range(61):
                evs[i].record(stream)
                if i < 60:
                    graph.replay()
        sync_all()
        per_step = sorted(evs[i].elapsed_time(evs[i + 1]) * 1e3 / per_graph for i in range(60))
        q = lambda f: per_step[min(59, int(f * 60))]  # noqa: E731
        stats = {"median_us": max_over_ranks(statistics.median(per_step)), "p10_us": max_over_ranks(q(0.1)),
                 "p90_us": max_over_ranks(q(0.9)), "samples": 60,
                 "what": f"60 replays of the {per_graph}-forward graph after the timed region, per-step mean "
                         "of each replay; max over ranks"}

    # ---------------- each step's kernels timed alone (roofline of the dominant kernel)
    kt = kernel_times(torch, tpq, hs, R, stream, M, tp)
    kt = {k: max_over_ranks(v) for k, v in kt.items()}
    peak, peak_kind = peaks()
    # the GEMV launches in their own sequence: a graph of layer-1, layer-2 launch pairs (no gather),
    # CUDA events around the replays only; a pair's time is <= the step's (the step adds the gather)
    per = R * max(1, 16 // R)

    def pair(i):
        hs[i % R].run_step(tpq.TPQ_STEP_LAYER1, M, stream=stream)
        hs[i % R].run_step(tpq.TPQ_STEP_LAYER2, M, stream=stream)
    with torch.cuda.stream(stream):
        for i in range(per):
            pair(i)
        gp = graph_of(torch, stream, per, pair)
    torch.cuda.synchronize()
    time.sleep(EXTRA_COOLDOWN_S)
    pair_us = max_over_ranks(time_graph(torch, stream, gp, 8, per))
    achieved = (l1_bytes + l2_bytes) / (pair_us * 1e-6) / 1e9

    # ---------------- e2e through the public host-buffer API (pinned host memory)
    # (--sim-tp has no host-buffer path: one rank's shard alone is not a complete forward)
    Xh = torch.from_numpy(p.X[:M].copy()).pin_memory()
    Yh = torch.empty(M, N2, dtype=torch.float16).pin_memory()
    Ke = max(20, min(K // 10, 2000))
    e2e = None
    if not sim_tp:
        for i in range(5):
            hs[i % R].forward_host(Xh.numpy(), Yh.numpy(), stream=stream)
        sync_all()
        es, ee = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        es.record(stream)
        for i in range(Ke):
            hs[i % R].forward_host(Xh.numpy(), Yh.numpy(), stream=stream)
        ee.record(stream)
        sync_all()
        e2e = {"value": max_over_ranks(es.elapsed_time(ee) / Ke) * 1e3, "unit": "us",
               "h2d_bytes_per_step": 2 * M * K1, "d2h_bytes_per_step": 2 * M * N2}

    line = {
        "metric": METRIC, "value": ms_per_step * 1e3, "unit": "us", "n_gpus": world, "steps": K,
        "warmup": max(3, a.warmup), "ms_per_step": ms_per_step, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f16", "data": "synthetic",
        "config": {
            "workload": f"{a.shape}-mlp K1={K1} N1={N1} N2={N2} G={G} M={M} tp={shard_tp} {a.variant}"
                        + (" (one rank's shard, no collective)" if sim_tp else ""),
            "M": M, "tp": shard_tp, "variant": a.variant, "int4_weights": True,
            "cold_l2": f"{R} rotating weight replicas x {step_bytes / 1e6:.1f} MB >= 3 x L2 ({l2_cache / 1e6:.0f} MB)",
            "launch": "eager C-ABI calls" if graph is None else
                      f"CUDA graphs: {per_graph} forwards x {K // per_graph} replays + {rem}",
            "parallelism": f"tp{shard_tp}",
        },
        "step_stats": stats,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": ncu_traffic(a, shard_tp), "peak_kind": peak_kind,
                     "kernel": "k_dqgemv, layer 1 and layer 2 (split tiles reduced in-kernel)",
                     "algorithmic_bytes_per_launch": (l1_bytes + l2_bytes) / 2,
                     "launch_us": {"mean_of_layer1_layer2": pair_us / 2, "pair": pair_us},
                     "how": "a CUDA graph of layer-1, layer-2 GEMV launch pairs over the cold replicas (the "
                            "forward without its gather), median of 8 replays, CUDA events around the replays "
                            "only; achieved = both layers' algorithmic bytes / the pair's time"},
        "kernel_us": kt,
        "kernel_sum_us": sum(kt.values()),
        "step_roofline": {"bytes": step_bytes, "GBps": step_bytes / (ms_per_step * 1e-3) / 1e9,
                          "frac": step_bytes / (ms_per_step * 1e-3) / 1e9 / peak},
        "e2e": e2e,
        "gpu_launches": K * launches_per_step(hs[0].info, variant == tpq.TPQ_NAIVE),
        "split_tile_modes": {"layer1": hs[0].info.split1, "layer2": hs[0].info.split2,
                             "legend": "0 in-kernel (stream-K), 1 fix-up kernel, c >= 2 cluster split-K of c CTAs"},
        "clocks": clk,
    }
    if world > 1 and variant == tpq.TPQ_TP_AWARE and not a.no_naive:
        # the paper's comparison on the same box, same kernels, same graph timing: Alg. 2 (naive
        # act_order TP, AllGather of Y1 + global P2 permute between the layers)
        try:
            line["naive_allgather"] = time_naive(a, p, P1, P2, shard_tp, rank, local, R, comm, X, Y, stream,
                                                 sync_all, world, dev, ms_per_step)
        except Exception as e:  # report, keep the TP-aware line
            line["naive_allgather"] = {"error": f"{type(e).__name__}: {e}"}
    clocks_x = ClockSampler(local)
    clocks_x.start()
    if world == 1 and not a.quick:
        # the rest of the metric's grid on this GPU (graph-timed, after the timed region)
        line["sweep_us_by_M"] = {str(m): step_latency(torch, tpq, hs, R, stream, m, sim_tp, X if m <= M else
                                                      torch.from_numpy(p.X[:m].copy()).to(dev), Y if m <= M else
                                                      torch.empty(m, N2, dtype=torch.float16, device=dev))
                                 for m in (1, 4, 8, 16)}
    for h in hs:
        h.close()
    if world == 1 and not a.quick and not sim_tp and a.shape == "llama70b":
        line["granite20b_tp1"] = extra_workload(torch, tpq, "granite20b", (1, 16), 0, a.seed, local, dev, stream)
        for k in (2, 4, 8):  # one rank's shard of the TP = k MLP (the metric's TP grid; no collective)
            line[f"llama70b_tp{k}_shard"] = extra_workload(torch, tpq, "llama70b", (1, 16), k, a.seed, local, dev, stream)
        line["granite20b_tp8_shard"] = extra_workload(torch, tpq, "granite20b", (1, 16), 8, a.seed, local, dev, stream)
        line["a7_llama70b_tp8_shard"] = a7_line(torch, tpq, "llama70b", a.seed, local, dev, stream)
    if world == 1 and not a.quick and not sim_tp and a.variant == "tp_aware":
        line["unordered_tp1"] = unordered_line(torch, tpq, p, a.shape, local, dev, stream, kt, M)
        line["gated_tp1"] = gated_line(torch, tpq, a.shape, a.seed, local, dev, stream)
    line["clocks_extra_lines"] = clocks_x.stop()
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        pc = synth.make_named(a.shape, M, a.seed)
        L1, L2, prep = oracle_prepare(pc)
        ts, tds, tms = [], [], []
        for _ in range(2):
            t0 = time.perf_counter()
            _, td, tm = oracle_forward(pc.X, L1, L2)
            ts.append(time.perf_counter() - t0)
            tds.append(td)
            tms.append(tm)
        line["cpu_baseline"] = {"value": min(ts) * 1e6, "unit": "us", "cores": cpu_cores(),
                                "blas_threads": blas_threads(), "kind": "oracle",
                                "sample": f"one full forward (fp64 dequantize + matmul, both layers, M={M}), "
                                          "best of 2, no extrapolation",
                                "phases_s": {"dequant": min(tds), "matmul": min(tms), "total": min(ts),
                                             "offline_unpack": prep["unpack_s"], "offline_alg1": prep["alg1_s"]}}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if tp > 1:
        comm.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def launches_per_step(info, naive):
    """Our kernels per forward (M <= 16): the X[:, P1] gather, per layer the GEMV plus a split-tile
    fix-up kernel where the layer uses one (tpq_mlp_info split mode 1), and the naive path's P2
    gather; NCCL kernels not counted."""
    return 1 + 2 + int(info.split1 == 1) + int(info.split2 == 1) + (1 if naive else 0)


def time_naive(a, p, P1, P2, tp, rank, local, R, comm, X, Y, stream, sync_all, world, dev, ours_ms):
    import torch
    import torch.distributed as dist

    import paper_2402_04925_b200 as tpq
    M = a.m
    hn = [tpq.TpMlp(p.w1, p.w2, P1, P2, tp=tp, rank=rank, variant=tpq.TPQ_NAIVE, M_max=16, device=local)
          for _ in range(R)]
    for h in hn:
        h.set_comm(comm)
    with torch.cuda.stream(stream):
        for i in range(max(3, a.warmup)):
            hn[i % R].forward(X, M, Y, stream=stream)
    sync_all()
    per = R * max(1, 16 // R)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for i in range(per):
            hn[i % R].forward(X, M, Y, stream=stream)
    for _ in range(3):
        g.replay()
    sync_all()
    reps = max(1, a.steps // per)
    s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        s_.record(stream)
        for _ in range(reps):
            g.replay()
        e_.record(stream)
    sync_all()
    ms = s_.elapsed_time(e_) / (reps * per)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    for h in hn:
        h.close()
    return {"value": ms * 1e3, "unit": "us", "steps": reps * per,
            "speedup_tp_aware": ms / ours_ms,
            "what": "Alg. 2: layer 1, ncclAllGather(Y1), P2 gather + CHUNK, layer 2, ncclAllReduce; "
                    "same kernels, CUDA-graph timed, max over ranks"}


if __name__ == "__main__":
    main()
