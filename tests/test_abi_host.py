"""C-ABI host-side tests (no GPU): the library loads, exports every symbol include/tpq.h
declares, and its host functions (Alg. 1 reorder, TP-aware shard index maps, the packed
layout) match the oracle bit-exactly.  Device work is never requested here (device=-1)."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle as O
import synth
from conftest import ROOT, golden

tpq = pytest.importorskip("paper_2402_04925_b200")


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2402_04925_b200 import build
    build.build()


def _declared():
    src = open(os.path.join(ROOT, "include", "tpq.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\**(\w+)\s*\(", src, flags=re.M))


def test_exports_every_declared_symbol():
    declared = _declared()
    assert declared == set(tpq.EXPORTS), declared ^ set(tpq.EXPORTS)
    L = ctypes.CDLL(tpq.LIB_PATH)
    for name in declared:
        assert hasattr(L, name), name
    assert tpq.lib().tpq_version() >> 16 == 1


def test_reorder_spec_examples():
    for ex in golden("spec_examples.json")["alg1"]:
        G = 1 if ex["g"] == [2, 1, 0] else 2
        P, gs = tpq.gptq_reorder(ex["g"], G)
        assert P.tolist() == ex["P"], ex["cite"]
        assert gs.tolist() == ex["g_opt"]


def test_reorder_matches_oracle_bit_exact():
    rng = np.random.default_rng(0)
    for t in range(300):
        K = int(rng.integers(1, 3000))
        G = int(rng.integers(1, K + 1))
        g = O.eq3_g_idx_actorder(rng.permutation(K), G)
        P, gs = tpq.gptq_reorder(g, G)
        Po, go = O.alg1_reorder(g)
        assert P.tolist() == Po.tolist()
        assert gs.tolist() == go.tolist()
    g = O.eq3_g_idx_actorder(np.random.default_rng(1).permutation(28672), 128)
    P, gs = tpq.gptq_reorder(g, 128)
    assert P.tolist() == O.alg1_reorder(g)[0].tolist()


@pytest.mark.parametrize("g,G", [([0, 0, 2], 2), ([0, 0, 0, 1], 2), ([-1, 0], 1), ([0, 1, 1], 2)])
def test_reorder_rejects_non_eq3(g, G):
    with pytest.raises(tpq.TPQError) as e:
        tpq.gptq_reorder(g, G)
    assert e.value.code == 1  # EINVAL


def _prep(p):
    P1, _ = tpq.gptq_reorder(p.w1.g_idx, p.G)
    P2, _ = tpq.gptq_reorder(p.w2.g_idx, p.G)
    return P1, P2


def _olayers(p):
    return (O.layer_from_checkpoint(p.w1.qweight, p.w1.scales_bits, p.w1.qzeros, p.w1.g_idx, p.K1, p.N1, p.G),
            O.layer_from_checkpoint(p.w2.qweight, p.w2.scales_bits, p.w2.qzeros, p.w2.g_idx, p.N1, p.N2, p.G))


@pytest.mark.parametrize("variant", ["tp_aware", "naive"])
@pytest.mark.parametrize("tp", [1, 2, 4, 8])
def test_shard_maps_and_packed_layout_match_oracle(tp, variant):
    # tiny config widened to N1=1024 so every tp gives whole 128-column device tiles
    p = synth.make_problem(256, 1024, 256, 32, 1, seed=3)
    P1, P2 = _prep(p)
    L1, L2 = _olayers(p)
    v = tpq.TPQ_TP_AWARE if variant == "tp_aware" else tpq.TPQ_NAIVE
    for rank in range(tp):
        h = tpq.TpMlp(p.w1, p.w2, P1, P2, tp=tp, rank=rank, variant=v, M_max=4, device=-1)
        ref = O.canonical_shard(L1, L2, tp, rank, variant)
        cols, rows, lo, hi = h.index_maps()
        assert cols.tolist() == ref["w1_cols"].tolist()
        assert rows.tolist() == ref["w2_rows"].tolist()
        assert (lo, hi) == (ref["w2_group_lo"], ref["w2_group_hi"])
        q1, s1, z1 = h.export_canonical(1)
        assert (q1 == ref["w1_q"]).all() and (z1 == ref["w1_z"]).all()
        assert (s1.view(np.float16).astype(np.float64) == ref["w1_s"]).all()
        q2, s2, z2 = h.export_canonical(2)
        assert (q2 == ref["w2_q"]).all() and (z2 == ref["w2_z"]).all()
        assert (s2.view(np.float16).astype(np.float64) == ref["w2_s"]).all()
        # ordered groups: the row-k group is floor(k/G) (closed form of Alg. 1)
        assert (ref["w1_g"] == np.arange(p.K1) // p.G).all()
        assert (ref["w2_g"] == np.arange(p.N1 // tp) // p.G).all()
        i = h.info
        assert i.w1_bytes == (p.N1 // tp // 128) * (p.K1 // p.G) * (64 * p.G + 320)
        h.close()


def test_packed_bytes_are_algorithmic():
    """Packed bytes per weight = 0.5 + 2.5/G exactly (int4 + fp16 scale + int4 zero per
    group-column): the device layout adds no padding."""
    p = synth.make_problem(256, 512, 256, 128, 1, seed=1)
    P1, P2 = _prep(p)
    h = tpq.TpMlp(p.w1, p.w2, P1, P2, device=-1)
    assert h.info.w1_bytes == 256 * 512 // 2 + 2.5 * (256 // 128) * 512
    h.close()


def test_shard_errors():
    p = synth.make_named("tiny", 1, seed=0)
    P1, P2 = _prep(p)
    E = tpq.TPQError

    def code(**kw):
        args = dict(tp=1, rank=0, variant=1, M_max=16, device=-1)
        args.update(kw)
        w1 = kw.pop("w1", p.w1) if "w1" in kw else p.w1
        with pytest.raises(E) as e:
            tpq.TpMlp(w1, p.w2, args.pop("P1", P1), args.pop("P2", P2), **{k: args[k] for k in
                                                                           ("tp", "rank", "variant", "M_max", "device")})
        return e.value.code

    assert code(tp=3) == 1
    assert code(tp=2, rank=2) == 1
    assert code(variant=7) == 1
    assert code(M_max=0) == 1
    assert code(M_max=513) == 1
    bad = P1.copy()
    bad[[0, 1]] = bad[[1, 0]] if p.w1.g_idx[bad[0]] != p.w1.g_idx[bad[1]] else bad[[0, 1]]
    bad2 = P1[::-1].copy()
    assert code(P1=bad2) == 1  # not ordering g_idx
    dup = P1.copy()
    dup[0] = dup[1]
    assert code(P1=dup) == 1   # not a permutation
    # n % 64: tiny N1=512, tp=16 unsupported degree; N2 not multiple of 64
    q = synth.make_problem(256, 512, 96, 32, 1, seed=0)
    Q1, Q2 = _prep(q)
    with pytest.raises(E) as e:
        tpq.TpMlp(q.w1, q.w2, Q1, Q2, device=-1)
    assert e.value.code == 1
    # G = 16 is valid for the paper but not implemented -> EUNSUPPORTED
    r = synth.make_problem(256, 512, 256, 16, 1, seed=0)
    R1, R2 = _prep(r)
    with pytest.raises(E) as e:
        tpq.TpMlp(r.w1, r.w2, R1, R2, device=-1)
    assert e.value.code == 2


def test_forward_on_host_only_handle_is_estate():
    p = synth.make_named("tiny", 1, seed=0)
    P1, P2 = _prep(p)
    h = tpq.TpMlp(p.w1, p.w2, P1, P2, device=-1)
    X = np.zeros((1, 256), np.float16)
    Y = np.zeros((1, 256), np.float16)
    with pytest.raises(tpq.TPQError) as e:
        h.forward_host(X, Y, stream=0)
    assert e.value.code == 6
    h.close()


def test_export_exact_over_wide_and_extreme_scales():
    """The device records hold s' = s 2^E per column (reading c22); the canonical export must give
    back every scale bit-exactly, over 4.5 decades (synth wide_scales) plus hand-set extremes:
    subnormal scales, the largest finite fp16, an all-zero column and negative zeros."""
    p = synth.make_problem(256, 1024, 256, 32, 1, seed=9, wide_scales=True)
    s1 = p.w1.scales_f16
    s1[:, 0] = np.float16(2.0 ** -24)            # smallest subnormal everywhere in column 0
    s1[0, 1] = np.float16(65504.0)               # largest finite next to tiny ones
    s1[1:, 1] = np.float16(2.0 ** -20)
    s1[:, 2] = np.float16(0.0)                   # all-zero column
    s1[3, 3] = np.float16(-0.0)
    p.w2.scales_f16[:, 5] = np.float16(6.1e-5)   # just below the smallest normal
    P1, P2 = _prep(p)
    L1, L2 = _olayers(p)
    for tp, rank in ((1, 0), (4, 3)):
        h = tpq.TpMlp(p.w1, p.w2, P1, P2, tp=tp, rank=rank, M_max=4, device=-1)
        ref = O.canonical_shard(L1, L2, tp, rank, "tp_aware")
        _, s_1, _ = h.export_canonical(1)
        _, s_2, _ = h.export_canonical(2)
        want1 = np.asarray(p.w1.scales_bits)[:, ref["w1_cols"]]
        assert (s_1 == want1).all()
        assert (s_2 == np.asarray(p.w2.scales_bits)[ref["w2_group_lo"]:ref["w2_group_hi"]]).all()
        h.close()


def test_unordered_variant_host_export_and_checks():
    """TPQ_UNORDERED: rows stay in checkpoint order, so the exported shard is
    the checkpoint itself (codes, scales bit-exact through the per-column exponent, zeros); tp > 1
    and M_max > 16 are rejected."""
    p = synth.make_problem(256, 1024, 256, 32, 1, seed=12, wide_scales=True)
    L1, L2 = _olayers(p)
    h = tpq.TpMlp(p.w1, p.w2, None, None, tp=1, rank=0, variant=tpq.TPQ_UNORDERED, M_max=16, device=-1)
    q1, s1, z1 = h.export_canonical(1)
    q2, s2, z2 = h.export_canonical(2)
    assert (q1 == L1.q).all() and (z1 == L1.z).all() and (s1 == np.asarray(p.w1.scales_bits)).all()
    assert (q2 == L2.q).all() and (z2 == L2.z).all() and (s2 == np.asarray(p.w2.scales_bits)).all()
    h.close()
    with pytest.raises(tpq.TPQError) as e:
        tpq.TpMlp(p.w1, p.w2, None, None, tp=2, rank=0, variant=tpq.TPQ_UNORDERED, M_max=16, device=-1)
    assert e.value.code == 1
    with pytest.raises(tpq.TPQError) as e:
        tpq.TpMlp(p.w1, p.w2, None, None, tp=1, rank=0, variant=tpq.TPQ_UNORDERED, M_max=17, device=-1)
    assert e.value.code == 2


@pytest.mark.parametrize("tp", [1, 4])
def test_gated_shard_export(tp):
    """gate_proj variant (f2): the gate shard is Wg[P1g][:, P2 block] and the up shard Wu[P1u][:, P2
    block] -- the same columns for both (reading c24) -- with Wd[P2] rows, bit-exactly."""
    p = synth.make_problem(256, 1024, 256, 32, 1, seed=14)
    q = synth.make_problem(256, 1024, 256, 32, 1, seed=15)
    wg, wu, wd = p.w1, q.w1, p.w2
    Lg, Ld = _olayers(p)
    Lu = O.layer_from_checkpoint(wu.qweight, wu.scales_bits, wu.qzeros, wu.g_idx, 256, 1024, 32)
    Ps = [tpq.gptq_reorder(w.g_idx, 32)[0] for w in (wg, wu, wd)]
    for r in range(tp):
        h = tpq.TpMlp.gated(wg, wu, wd, *Ps, tp=tp, rank=r, M_max=16, device=-1)
        rg = O.canonical_shard(Lg, Ld, tp, r, "tp_aware")
        ru = O.canonical_shard(Lu, Ld, tp, r, "tp_aware")
        qg, sg, zg = h.export_canonical(1)
        qu, su, zu = h.export_canonical(3)
        qd, sd, zd = h.export_canonical(2)
        assert (qg == rg["w1_q"]).all() and (zg == rg["w1_z"]).all() and (sg.view(np.float16).astype(np.float64) == rg["w1_s"]).all()
        assert (qu == ru["w1_q"]).all() and (zu == ru["w1_z"]).all() and (su.view(np.float16).astype(np.float64) == ru["w1_s"]).all()
        assert (qd == rg["w2_q"]).all() and (zd == rg["w2_z"]).all()
        h.close()
    with pytest.raises(tpq.TPQError):
        tpq.TpMlp.gated(wg, wu, wd, *Ps, M_max=64, device=-1)
