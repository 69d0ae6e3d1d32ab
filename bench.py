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
    ap.add_argument("--steps", type=int, default=5000)
    ap.add_argument("--warmup", type=int, default=200)
    ap.add_argument("--shape", default="llama70b", choices=sorted(synth.SHAPES))
    ap.add_argument("--m", type=int, default=16)
    ap.add_argument("--variant", default="tp_aware", choices=["tp_aware", "naive"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--sweep", action="store_true",
                    help="N = 1: add graph-timed step latencies at M = 1/4/8/16 (key sweep_us_by_M; runs after "
                         "the timed region, so power-capped boxes may report it slower)")
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
def oracle_sample_time(p, frac_den: int = 8, reps: int = 1):
    """Time the oracle (as it stands: checkpoint unpack, Alg. 1, Alg. 3 at tp=1, fp64) on the
    sub-MLP made of the first N1/frac_den intermediate columns (W1[:, :c], W2[:c, :]), which
    is 1/frac_den of the full forward's work; returns seconds per FULL forward."""
    import oracle as O
    c = p.N1 // frac_den
    w1, w2 = p.w1, p.w2
    qw1, sc1, qz1 = w1.qweight[:, :c], w1.scales_bits[:, :c], w1.qzeros[:, :c // 8]
    qw2, g2 = w2.qweight[:c // 8, :], w2.g_idx[:c]
    # the sub-MLP keeps W2's rows 0..c-1 whose act_order groups are re-indexed densely
    ug, g2d = np.unique(g2, return_inverse=True)
    sc2, qz2 = w2.scales_bits[ug], w2.qzeros[ug]
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        L1 = O.layer_from_checkpoint(qw1, sc1, qz1, w1.g_idx, p.K1, c, p.G)
        L2 = O.layer_from_checkpoint(qw2, sc2, qz2, g2d, c, p.N2, p.G)
        O.alg3_tp_aware(p.X, L1, L2, 1)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return best * frac_den


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    tp = a.gpus
    K1, N1, N2, G = synth.SHAPES[a.shape]
    p = synth.make_named(a.shape, a.m, a.seed)
    den = 4 if a.shape != "tiny" else 1
    for _ in range(min(a.warmup, 1)):
        oracle_sample_time(p, den)
    ts = [oracle_sample_time(p, den) for _ in range(max(1, min(a.steps, 3)))]
    us = statistics.median(ts) * 1e6
    sample = f"Alg.3 tp=1 oracle on W1[:, :N1/{den}], W2[:N1/{den}, :] (1/{den} of the work), x{den}"
    line = {"metric": METRIC, "value": us, "unit": "us", "impl": "reference", "n_gpus": a.gpus,
            "steps": len(ts), "warmup": min(a.warmup, 1), "ms_per_step": us / 1e3, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{a.shape}-mlp K1={K1} N1={N1} N2={N2} G={G} M={a.m} tp={tp} {a.variant}",
                       "M": a.m, "tp": tp},
            "cpu_baseline": {"value": us, "unit": "us", "cores": cpu_cores(), "kind": "oracle", "sample": sample},
            "e2e": {"value": us, "unit": "us", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------ ours
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
    variant = tpq.TPQ_TP_AWARE if a.variant == "tp_aware" else tpq.TPQ_NAIVE
    p = synth.make_named(a.shape, max(M, 16), a.seed)
    P1, _ = tpq.gptq_reorder(p.w1.g_idx, G)
    P2, _ = tpq.gptq_reorder(p.w2.g_idx, G)

    l1_bytes, l2_bytes, step_bytes = algorithmic_bytes(K1, N1, N2, G, M, shard_tp)
    # cold L2: rotate R weight replicas with R * bytes >= 3 x L2
    l2_cache = torch.cuda.get_device_properties(dev).L2_cache_size
    R = max(1, -(-3 * l2_cache // int(step_bytes)))
    hs = [tpq.TpMlp(p.w1, p.w2, P1, P2, tp=shard_tp, rank=rank, variant=variant, M_max=16, device=local)
          for _ in range(R)]
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

    # ---------------- warm-up
    with torch.cuda.stream(stream):
        for i in range(max(3, a.warmup)):
            fwd(hs[i % R])
    sync_all()

    # ---------------- timed region: exactly K steps.
    # Default: the steps are replayed from CUDA graphs of consecutive forwards (rotating the
    # weight replicas) so host launch overhead is not measured: a graph of `per_graph` forwards
    # replayed K // per_graph times plus a graph of the K % per_graph remaining forwards.  No
    # timing events sit inside these graphs (an event node between kernels would break the
    # programmatic-dependent-launch overlap); the per-kernel breakdown comes from a separate
    # graph with the library's event hook, replayed after the timed region.
    # --no-graph launches every forward eagerly through the C-ABI.
    K = a.steps
    per_graph = R * max(1, 16 // R)
    rem = K % per_graph

    def capture(n, timed_evs=None):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for i in range(n):
                h = hs[i % R]
                if timed_evs is not None:
                    h.set_timing(timed_evs[i])
                fwd(h)
                if timed_evs is not None:
                    h.set_timing(None)
        return g

    n_ev = per_graph
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(n_ev)]
    for es_ in evs:  # torch creates the cudaEvent_t lazily, on first record
        for e in es_:
            e.record(stream)
    sync_all()
    graph = graph_rem = None
    if not a.no_graph:
        graph = capture(per_graph)
        graph_rem = capture(rem) if rem else None
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
    total_ms = start.elapsed_time(end)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / K

    # ---------------- per-kernel breakdown (events around each launch; not the headline)
    with torch.cuda.stream(stream):
        if graph is not None:
            gev = capture(per_graph, evs)
            for _ in range(3):
                gev.replay()
        else:
            for i in range(n_ev):
                h = hs[i % R]
                h.set_timing(evs[i])
                fwd(h)
                h.set_timing(None)
    sync_all()
    t_l1 = statistics.mean(e[1].elapsed_time(e[2]) for e in evs) * 1e3  # us
    t_l2 = statistics.mean(e[3].elapsed_time(e[4]) for e in evs) * 1e3
    t_gather = statistics.mean(e[0].elapsed_time(e[1]) for e in evs) * 1e3
    t_coll = statistics.mean(e[4].elapsed_time(e[5]) for e in evs) * 1e3
    t_mid = statistics.mean(e[2].elapsed_time(e[3]) for e in evs) * 1e3

    # ---------------- e2e through the public host-buffer API (pinned host memory)
    # (--sim-tp has no host-buffer path: one rank's shard alone is not a complete forward)
    Xh = torch.from_numpy(p.X[:M].copy()).pin_memory()
    Yh = torch.empty(M, N2, dtype=torch.float16).pin_memory()
    Ke = max(20, min(K // 10, 2000))
    es, ee = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if not sim_tp:
        for i in range(5):
            hs[i % R].forward_host(Xh.numpy(), Yh.numpy(), stream=stream)
        sync_all()
        es.record(stream)
        for i in range(Ke):
            hs[i % R].forward_host(Xh.numpy(), Yh.numpy(), stream=stream)
        ee.record(stream)
    else:
        es.record(stream)
        ee.record(stream)
    sync_all()
    e2e_ms = es.elapsed_time(ee) / Ke if not sim_tp else float("nan")
    if world > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    # ---------------- roofline of the dominant kernel (the dequant GEMV, both launches)
    peak, peak_kind = peaks()
    gemv_us = t_l1 + t_l2
    achieved = (l1_bytes + l2_bytes) / (gemv_us * 1e-6) / 1e9
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
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": ncu_traffic(a, shard_tp), "peak_kind": peak_kind,
                     "kernel": "k_dqgemv (layer-1 + layer-2 launches)",
                     "algorithmic_bytes_per_launch": (l1_bytes + l2_bytes) / 2},
        "breakdown_us": {"gather": t_gather, "gemv_l1": t_l1, "between": t_mid, "gemv_l2": t_l2,
                         "allreduce": t_coll},
        "step_roofline": {"bytes": step_bytes, "GBps": step_bytes / (ms_per_step * 1e-3) / 1e9,
                          "frac": step_bytes / (ms_per_step * 1e-3) / 1e9 / peak},
        "e2e": None if sim_tp else {"value": e2e_ms * 1e3, "unit": "us", "h2d_bytes_per_step": 2 * M * K1,
                                    "d2h_bytes_per_step": 2 * M * N2},
        "gpu_launches": K * launches_per_step(M, variant == tpq.TPQ_NAIVE),
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
    if world == 1 and a.sweep:  # (collective forwards at N > 1 would need every rank)
        line["sweep_us_by_M"] = sweep_m(hs, p, R, stream, dev, sim_tp)
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        den = 4 if a.shape != "tiny" else 1
        t = oracle_sample_time(synth.make_named(a.shape, M, a.seed), den)
        line["cpu_baseline"] = {"value": t * 1e6, "unit": "us", "cores": cpu_cores(), "kind": "oracle",
                                "sample": f"Alg.3 tp=1 fp64 oracle on W1[:, :N1/{den}], W2[:N1/{den}, :] "
                                          f"(1/{den} of one forward), scaled x{den}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    for h in hs:
        h.close()
    if tp > 1:
        comm.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def launches_per_step(M, naive):
    """Our kernels per forward (M <= 16): the X[:, P1] gather, per layer the GEMV and its split-tile
    fix-up kernel, and the naive path's P2 gather; NCCL kernels not counted."""
    return 1 + 2 * 2 + (1 if naive else 0)


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


def sweep_m(hs, p, R, stream, dev, sim_tp):
    """Step latency (us) at M = 1, 4, 8, 16 on the same handles: CUDA graphs of R * k forwards
    (rotating the cold weight replicas) replayed after warm-up, as in the main timed region."""
    import torch
    out = {}
    per = R * max(1, 16 // R)
    for M in (1, 4, 8, 16):
        X = torch.from_numpy(p.X[:M].copy()).to(dev)
        Y = torch.empty(M, p.N2, dtype=torch.float16, device=dev)
        f = (lambda h: h.forward_local(X, M, Y, stream=stream)) if sim_tp else (lambda h: h.forward(X, M, Y, stream=stream))
        with torch.cuda.stream(stream):
            for i in range(per):
                f(hs[i % R])
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                for i in range(per):
                    f(hs[i % R])
            for _ in range(5):
                g.replay()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = max(1, 2000 // per)
            s.record(stream)
            for _ in range(reps):
                g.replay()
            e.record(stream)
        torch.cuda.synchronize(dev)
        out[str(M)] = s.elapsed_time(e) * 1e3 / (reps * per)
    return out


if __name__ == "__main__":
    main()
