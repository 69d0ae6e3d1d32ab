"""World-size-2 CPU tests (gloo) of the N>1 host logic: the NCCL unique-id exchange over the
process group, and per-rank sharding -- every rank builds its own host-only TP shard through
the C-ABI; gathered over gloo, the shards reassemble W1[P1,P2] / W2[P2] exactly, and the
rank-order AllReduce of per-rank partials (computed from the exported shards with oracle
arithmetic) equals the oracle's Alg. 3 and the dense product."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle as O
        import paper_2402_04925_b200 as tpq
        import synth
        from paper_2402_04925_b200.tp import exchange_unique_id

        uid = exchange_unique_id()
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        assert len(uid) == 128 and all(i == uid for i in ids) and any(uid)

        p = synth.make_problem(256, 512, 256, 32, 3, seed=17)
        P1, _ = tpq.gptq_reorder(p.w1.g_idx, 32)
        P2, _ = tpq.gptq_reorder(p.w2.g_idx, 32)
        h = tpq.TpMlp(p.w1, p.w2, P1, P2, tp=world, rank=rank, device=-1)
        q1, s1, z1 = h.export_canonical(1)
        q2, s2, z2 = h.export_canonical(2)
        cols, rows, lo, hi = h.index_maps()
        # rank-local Alg. 3 partial from this rank's exported shard (oracle arithmetic)
        W1l = O.dequantize(O.OLayer(q=q1.astype(np.int64), s=s1.view(np.float16).astype(np.float64),
                                    z=z1.astype(np.int64), g=np.arange(256) // 32, G=32))
        n = 512 // world
        W2l = O.dequantize(O.OLayer(q=q2.astype(np.int64), s=s2.view(np.float16).astype(np.float64),
                                    z=z2.astype(np.int64), g=np.arange(n) // 32, G=32))
        Xp = p.X.astype(np.float64)[:, P1]
        y2 = torch.from_numpy((Xp @ W1l) @ W2l)
        parts = [torch.zeros_like(y2) for _ in range(world)]
        dist.all_gather(parts, y2)
        Y2 = parts[0].clone()
        for t in parts[1:]:
            Y2 += t  # rank-order AllReduce
        allcols = [torch.zeros(n, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(allcols, torch.from_numpy(cols))
        if rank == 0:
            L1 = O.layer_from_checkpoint(p.w1.qweight, p.w1.scales_bits, p.w1.qzeros, p.w1.g_idx, 256, 512, 32)
            L2 = O.layer_from_checkpoint(p.w2.qweight, p.w2.scales_bits, p.w2.qzeros, p.w2.g_idx, 512, 256, 32)
            ref = O.alg3_tp_aware(p.X, L1, L2, world)["Y2"]
            _, dense = O.dense_mlp(p.X, O.dequantize(L1), O.dequantize(L2))
            assert torch.cat(allcols).numpy().tolist() == P2.tolist()
            assert np.max(np.abs(Y2.numpy() - ref)) <= 1e-12 * np.max(np.abs(ref))
            assert np.max(np.abs(Y2.numpy() - dense)) <= 1e-12 * np.max(np.abs(dense))
        h.close()
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))


def test_gloo_world2_sharding_and_uid():
    from paper_2402_04925_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
