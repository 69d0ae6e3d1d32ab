"""Pins for the CPU oracle (``-m "not gpu"``): each oracle function is tied to something
other than itself -- the SPEC/hand worked examples under tests/golden/, closed forms,
brute force on tiny inputs, and exact-arithmetic identities the paper fixes.

A plausible mistake (dropped term, wrong sign, wrong index, transposed operand,
unstable sort, wrong zero convention) fails at least one of these.
"""
import itertools
import math

import numpy as np
import pytest

import oracle as O
import synth
from conftest import golden

SPEC = golden("spec_examples.json")
HAND = golden("hand_mlp.json")
PACK = golden("gptq_packing.json")


# ----------------------------------------------------------------------------- worked examples
def test_eq1_spec_examples():
    for ex in SPEC["eq1"]:
        out = O.eq1_g_idx_naive(ex["K"], ex["G"])
        if "out" in ex:
            assert out.tolist() == ex["out"], ex["cite"]
        else:
            assert int(out[-1]) == ex["last"], ex["cite"]


def test_eq3_spec_examples():
    for ex in SPEC["eq3"]:
        assert O.eq3_g_idx_actorder(ex["phi"], ex["G"]).tolist() == ex["out"], ex["cite"]


def test_alg1_spec_examples():
    for ex in SPEC["alg1"]:
        P, g_opt = O.alg1_reorder(ex["g"])
        assert P.tolist() == ex["P"], ex["cite"]
        assert g_opt.tolist() == ex["g_opt"], ex["cite"]


def test_invert_spec_examples():
    for ex in SPEC["invert"]:
        assert O.invert_permutation(ex["P"]).tolist() == ex["Q"], ex["cite"]
    rng = np.random.default_rng(3)
    P = rng.permutation(50)
    assert O.invert_permutation(O.invert_permutation(P)).tolist() == P.tolist()


def test_metadata_loads_spec_examples():
    for ex in SPEC["metadata_loads"]:
        if "g" in ex:
            assert O.metadata_loads(ex["g"]) == ex["loads"], ex["cite"]
        else:
            K, G = ex["K"], ex["G"]
            assert O.metadata_loads(np.arange(K) // G) == ex["ordered_loads"], ex["cite"]


def test_all_reduce_spec_example():
    ex = SPEC["all_reduce_sum"][0]
    parts = [np.array([[float(v)]]) for v in ex["parts"]]
    assert O.tp_dequant._all_reduce_sum(parts)[0, 0] == ex["out"]


# ----------------------------------------------------------------------------- Alg. 1
def _bruteforce_stable_argsort(g):
    """O(K^2) rank construction: rank[j] = #{i : (g[i], i) < (g[j], j)}; P[rank[j]] = j."""
    K = len(g)
    P = [None] * K
    for j in range(K):
        r = 0
        for i in range(K):
            if g[i] < g[j] or (g[i] == g[j] and i < j):
                r += 1
        P[r] = j
    return P


def test_alg1_vs_bruteforce_1000_arrays():
    """SPEC.md:L460 acceptance: Alg. 1 vs an independent brute-force stable sort, K <= 512."""
    rng = np.random.default_rng(1234)
    for t in range(1000):
        K = int(rng.integers(1, 65)) if t < 950 else int(rng.integers(65, 513))
        G = int(rng.integers(1, K + 1))
        phi = rng.permutation(K)
        g = (phi // G).tolist() if t % 2 == 0 else rng.integers(0, max(1, K // G + 1), size=K).tolist()
        P, g_opt = O.alg1_reorder(g)
        assert P.tolist() == _bruteforce_stable_argsort(g)
        assert g_opt.tolist() == sorted(g)


@pytest.mark.parametrize("K,G", [(256, 32), (8192, 128), (1000, 128), (5, 2), (7, 3), (28672, 128)])
def test_alg1_closed_form(K, G):
    """g_idx_optimized[i] = floor(i/G): Eq. 3 is a permutation of Eq. 1's multiset
    (SPEC.md:L103), so sorting it gives Eq. 1 back ("consecutive")."""
    phi = np.random.default_rng(K + G).permutation(K)
    g = O.eq3_g_idx_actorder(phi, G)
    P, g_opt = O.alg1_reorder(g)
    assert g_opt.tolist() == [i // G for i in range(K)]
    assert sorted(P.tolist()) == list(range(K))
    # within a group the original indices stay ascending (stability, reading c6)
    for gg in range(-(-K // G)):
        members = P[g_opt == gg]
        assert np.all(np.diff(members) > 0)


def test_alg1_stable_differs_from_argsort_phi():
    """Reading c6: argsort(phi) also orders the groups but is a different P."""
    K, G = 64, 8
    phi = np.random.default_rng(0).permutation(K)
    g = O.eq3_g_idx_actorder(phi, G)
    P, _ = O.alg1_reorder(g)
    assert P.tolist() != np.argsort(phi).tolist()
    assert (g[np.argsort(phi)] == np.arange(K) // G).all()


def test_multiset_law_and_load_floor():
    """SPEC.md:L103/L105 and acceptance L459: ordered = ceil(K/G) loads; random phi
    with K >= 64, G <= K/8 needs >= 2x that, over 20 seeds."""
    for seed in range(20):
        rng = np.random.default_rng(seed)
        K = int(rng.integers(64, 2048))
        G = int(rng.integers(1, K // 8 + 1))
        phi = rng.permutation(K)
        g = O.eq3_g_idx_actorder(phi, G)
        assert sorted(g.tolist()) == O.eq1_g_idx_naive(K, G).tolist()
        ng = -(-K // G)
        _, g_opt = O.alg1_reorder(g)
        assert O.metadata_loads(g_opt) == ng
        assert O.metadata_loads(g) >= 2 * ng
    # Llama-70B K1 (SURVEY.md §8(c) locality pin: unordered 8058 vs ordered 64 at seed 0)
    g = O.eq3_g_idx_actorder(np.random.default_rng(0).permutation(8192), 128)
    assert O.metadata_loads(O.alg1_reorder(g)[1]) == 64
    assert O.metadata_loads(g) > 8000


def test_synth_gidx_is_eq3():
    p = synth.make_problem(256, 512, 256, 32, 1, seed=5)
    assert p.w1.g_idx.tolist() == O.eq3_g_idx_actorder(p.w1.phi, 32).tolist()
    assert p.w2.g_idx.tolist() == O.eq3_g_idx_actorder(p.w2.phi, 32).tolist()


# ----------------------------------------------------------------------------- packing / dequant
def test_unpack_golden_words():
    c = PACK["qweight_column"]
    q = O.unpack_qweight(np.array([[c["word"]]], dtype=np.uint32), 8)
    assert q[:, 0].tolist() == c["q_rows"]
    c = PACK["qweight_column2"]
    q = O.unpack_qweight(np.array([[c["word"]]], dtype=np.uint32), 8)
    assert q[:, 0].tolist() == c["q_rows"]
    c = PACK["qzeros_row"]
    z = O.unpack_qzeros(np.array([[c["word"]]], dtype=np.uint32), 8)
    assert z[0].tolist() == c["z_cols"]


def test_unpack_roundtrip_synth_packer():
    p = synth.make_problem(64, 128, 48, 16, 2, seed=9)
    assert (O.unpack_qweight(p.w1.qweight, 64) == p.w1.q).all()
    assert (O.unpack_qzeros(p.w1.qzeros, 128) == p.w1.z).all()


def _hand_layer(d):
    g = O.eq3_g_idx_actorder(d["phi"], d["G"])
    return O.OLayer(q=np.array(d["q"], dtype=np.int64), s=np.array(d["s"], dtype=np.float64),
                    z=np.array(d["z"], dtype=np.int64), g=g, G=d["G"])


def test_dequant_hand_example():
    L1, L2 = _hand_layer(HAND["layer1"]), _hand_layer(HAND["layer2"])
    assert L1.g.tolist() == HAND["g1"] and L2.g.tolist() == HAND["g2"]
    assert O.dequantize(L1).tolist() == HAND["W1"]
    assert O.dequantize(L2).tolist() == HAND["W2"]


def test_dequant_vs_scalar_loop():
    """Vectorised fancy-indexed dequant vs a scalar loop of the definition."""
    rng = np.random.default_rng(7)
    K, N, G = 24, 5, 8
    g = O.eq3_g_idx_actorder(rng.permutation(K), G)
    q = rng.integers(0, 16, (K, N))
    z = rng.integers(0, 16, (K // G, N))
    s = rng.uniform(0.1, 2, (K // G, N))
    W = O.dequantize(O.OLayer(q=q, s=s, z=z, g=g, G=G))
    for k in range(K):
        for n in range(N):
            assert W[k, n] == s[g[k]][n] * (float(q[k][n]) - float(z[g[k]][n]))


def test_dequant_G_equals_K_per_column():
    """G = K: one group, g == 0 and P = identity for any phi; dequant reduces to the
    per-column s[0,n]*(q-z[0,n]) (north_star pin)."""
    rng = np.random.default_rng(11)
    K, N = 32, 16
    phi = rng.permutation(K)
    g = O.eq3_g_idx_actorder(phi, K)
    assert (g == 0).all()
    P, _ = O.alg1_reorder(g)
    assert P.tolist() == list(range(K))
    q = rng.integers(0, 16, (K, N))
    z = rng.integers(0, 16, (1, N))
    s = rng.uniform(0.1, 2, (1, N))
    W = O.dequantize(O.OLayer(q=q, s=s, z=z, g=g, G=K))
    for n in range(N):
        col = [s[0][n] * (q[k][n] - z[0][n]) for k in range(K)]
        assert W[:, n].tolist() == col


# ----------------------------------------------------------------------------- MLP / Alg. 2 / Alg. 3
def test_hand_mlp_dense_and_tp():
    L1, L2 = _hand_layer(HAND["layer1"]), _hand_layer(HAND["layer2"])
    X = np.array(HAND["X"])
    Y1, Y2 = O.dense_mlp(X, O.dequantize(L1), O.dequantize(L2))
    assert Y1.tolist() == HAND["Y1"] and Y2.tolist() == HAND["Y2"]
    for tp in (1, 2):
        a3 = O.alg3_tp_aware(X, L1, L2, tp)
        a2 = O.alg2_naive(X, L1, L2, tp)
        assert a3["Y2"].tolist() == HAND["Y2"]
        assert a2["Y2"].tolist() == HAND["Y2"]
        assert a3["P1"].tolist() == HAND["P1"] and a3["P2"].tolist() == HAND["P2"]
    a3 = O.alg3_tp_aware(X, L1, L2, 2)
    assert [y.tolist() for y in a3["Y1_local"]] == HAND["tp2_tp_aware_Y1_local"]
    assert [y.tolist() for y in a3["Y2_local"]] == HAND["tp2_tp_aware_Y2_local"]
    a2 = O.alg2_naive(X, L1, L2, 2)
    assert [y.tolist() for y in a2["Y1_local"]] == HAND["tp2_naive_Y1_local"]
    assert [y.tolist() for y in a2["Y1_chunk"]] == HAND["tp2_naive_Y1_chunk"]


def _olayers(p):
    return (O.layer_from_checkpoint(p.w1.qweight, p.w1.scales_bits, p.w1.qzeros, p.w1.g_idx,
                                    p.K1, p.N1, p.G),
            O.layer_from_checkpoint(p.w2.qweight, p.w2.scales_bits, p.w2.qzeros, p.w2.g_idx,
                                    p.N1, p.N2, p.G))


def _bruteforce_mlp(X, L1, L2):
    """Triple loops of the definition in pure Python (tiny sizes only)."""
    M, K1 = X.shape
    N1, N2 = L1.N, L2.N
    W1 = [[L1.s[L1.g[k]][n] * (int(L1.q[k][n]) - int(L1.z[L1.g[k]][n])) for n in range(N1)] for k in range(K1)]
    W2 = [[L2.s[L2.g[k]][n] * (int(L2.q[k][n]) - int(L2.z[L2.g[k]][n])) for n in range(N2)] for k in range(N1)]
    Y1 = [[sum(float(X[m][k]) * W1[k][n] for k in range(K1)) for n in range(N1)] for m in range(M)]
    Y2 = [[sum(Y1[m][k] * W2[k][n] for k in range(N1)) for n in range(N2)] for m in range(M)]
    return np.array(Y1), np.array(Y2)


def test_integer_regime_bit_exact_all_tp():
    """Integer-exact regime (X in -2..2, q,z in 0..15, s = 2^-e): every product/partial sum
    is an exact dyadic rational in fp64, so naive (Alg. 2) = TP-aware (Alg. 3) = dense
    (unordered act_order dequant) = brute force, BIT-EXACTLY, at tp = 1/2/4/8
    (SPEC.md:L330 equivalence theorem; north_star 'reordered equals unreordered,
    TP=k equals TP=1').  Non-square K1 != N1 != N2 catches transposed operands."""
    p = synth.make_problem(64, 128, 48, 16, 3, seed=4, integer_regime=True)
    L1, L2 = _olayers(p)
    X = p.X.astype(np.float64)
    Y1d, Y2d = O.dense_mlp(X, O.dequantize(L1), O.dequantize(L2))
    Y1b, Y2b = _bruteforce_mlp(X, L1, L2)
    assert (Y1d == Y1b).all() and (Y2d == Y2b).all()
    for tp in (1, 2, 4, 8):
        a2 = O.alg2_naive(X, L1, L2, tp)
        a3 = O.alg3_tp_aware(X, L1, L2, tp)
        assert (a2["Y2"] == Y2d).all(), tp
        assert (a3["Y2"] == Y2d).all(), tp
        n = p.N1 // tp
        # Alg. 3 rank r's Y1 is Y1 restricted to the P2 columns of its shard
        for r in range(tp):
            assert (a3["Y1_local"][r] == Y1d[:, a3["P2"][r * n:(r + 1) * n]]).all()
            assert (a2["Y1_local"][r] == Y1d[:, r * n:(r + 1) * n]).all()
            assert (a2["Y1_chunk"][r] == a3["Y1_local"][r]).all()


def test_float_regime_tp_invariance():
    p = synth.make_problem(128, 256, 96, 32, 5, seed=2)
    L1, L2 = _olayers(p)
    X = p.X.astype(np.float64)
    _, Y2d = O.dense_mlp(X, O.dequantize(L1), O.dequantize(L2))
    for tp in (1, 2, 4, 8):
        for f in (O.alg2_naive, O.alg3_tp_aware):
            Y2 = f(X, L1, L2, tp)["Y2"]
            assert np.max(np.abs(Y2 - Y2d)) <= 1e-12 * np.max(np.abs(Y2d))


def test_tp_aware_w1_is_column_permuted_naive():
    """dequant(W1[P1,P2]) = permute_cols(dequant(W1[P1]), P2)."""
    p = synth.make_problem(64, 128, 48, 16, 1, seed=6)
    L1, L2 = _olayers(p)
    P1, _ = O.alg1_reorder(L1.g)
    P2, _ = O.alg1_reorder(L2.g)
    Wn = O.dequantize(O.permute_rows(L1, P1))
    Wa = O.dequantize(O.permute_cols(O.permute_rows(L1, P1), P2))
    assert (Wa == Wn[:, P2]).all()
    # and reordering rows is exact: W[P1] dequantized with the ordered g equals rows of W
    assert (Wn == O.dequantize(L1)[P1]).all()


def test_identity_phi_variants_identical():
    """identity phi => P1 = P2 = identity and both variants hold the same bytes."""
    p = synth.make_problem(64, 128, 64, 16, 1, seed=8, identity_phi=True)
    L1, L2 = _olayers(p)
    for tp in (1, 2, 4):
        for r in range(tp):
            a = O.canonical_shard(L1, L2, tp, r, "tp_aware")
            b = O.canonical_shard(L1, L2, tp, r, "naive")
            assert a["P1"].tolist() == list(range(64)) and a["P2"].tolist() == list(range(128))
            for key in ("w1_q", "w1_s", "w1_z", "w2_q"):
                assert (a[key] == b[key]).all()


def test_shard_maps_cover_and_groups():
    p = synth.make_problem(64, 256, 64, 16, 1, seed=10)
    L1, L2 = _olayers(p)
    P2, g2_opt = O.alg1_reorder(L2.g)
    for tp in (1, 2, 4, 8):
        n = 256 // tp
        cols = np.concatenate([O.shard_maps(P2, 256, tp, r, "tp_aware", 16)["w1_cols"] for r in range(tp)])
        assert cols.tolist() == P2.tolist()
        for r in range(tp):
            mp = O.shard_maps(P2, 256, tp, r, "tp_aware", 16)
            # W2 shard owns whole ordered groups [r n/G, (r+1) n/G)
            gs = g2_opt[r * n:(r + 1) * n]
            assert gs.min() == mp["w2_group_lo"] and gs.max() == mp["w2_group_hi"] - 1
            src = mp["gather_src"]
            assert (src[:, 0] * n + src[:, 1] == P2[r * n:(r + 1) * n]).all()


def test_naive_gather_map_matches_alg2():
    p = synth.make_problem(64, 128, 48, 16, 2, seed=12)
    L1, L2 = _olayers(p)
    X = p.X.astype(np.float64)
    for tp in (2, 4):
        a2 = O.alg2_naive(X, L1, L2, tp)
        buf = np.stack(a2["Y1_local"])  # [tp][M][n]  (NCCL AllGather layout, reading c17)
        for r in range(tp):
            src = O.shard_maps(a2["P2"], 128, tp, r, "naive", 16)["gather_src"]
            y1in = buf[src[:, 0], :, src[:, 1]].T
            assert (y1in == a2["Y1_chunk"][r]).all()


def test_check_rows_close():
    ref = np.array([[1.0, -2.0, 0.0], [0.0, 0.0, 0.0]])
    ok, w = O.check_rows_close(ref + [[0.019, 0, 0], [0, 0, 0]], ref)
    assert ok and abs(w - 0.0095) < 1e-12
    ok, _ = O.check_rows_close(ref + [[0.021, 0, 0], [0, 0, 0]], ref)
    assert not ok
    ok, _ = O.check_rows_close(ref + [[0, 0, 0], [0, 1e-30, 0]], ref)
    assert not ok


def test_dense_mlp_columns_equals_dense():
    """The column-blocked evaluation used at full size is the same definition: bit-equal to
    dense_mlp on the integer regime (and on sampled columns)."""
    p = synth.make_problem(64, 128, 48, 16, 3, seed=13, integer_regime=True)
    L1, L2 = _olayers(p)
    X = p.X.astype(np.float64)
    Y1, Y2 = O.dense_mlp(X, O.dequantize(L1), O.dequantize(L2))
    Y1c, Y2c = O.dense_mlp_columns(X, L1, L2, chunk=24)
    assert (Y1c == Y1).all() and (Y2c == Y2).all()
    cols = np.array([47, 0, 5])
    _, Y2s = O.dense_mlp_columns(X, L1, L2, cols2=cols, chunk=7)
    assert (Y2s == Y2[:, cols]).all()


# ----------------------------------------------------------------------------- fp16 decode
def test_fp16_bits_golden():
    """fp16_bits_to_f64 against binary16 values written out by hand (tests/golden/fp16_bits.json,
    IEEE 754 definition): normal, subnormal, extreme and signed patterns.  This is the decode every
    scale of the checkpoint goes through in layer_from_checkpoint."""
    g = golden("fp16_bits.json")
    for c in g["cases"]:
        v = O.fp16_bits_to_f64(np.array([int(c["bits"], 16)], dtype=np.uint16))[0]
        want = math.inf if c["value"] == "inf" else float(c["value"])
        assert v == want and math.copysign(1.0, v) == math.copysign(1.0, want), (c, v)


def test_layer_from_checkpoint_scales_decode():
    """The decoded scale of a checkpoint entry is its binary16 value (bits chosen by hand)."""
    bits = np.array([[0x3C00, 0x0001], [0x7BFF, 0x3555]], dtype=np.uint16)
    K, N, G = 16, 16, 8
    qw = np.zeros((K // 8, N), np.uint32)
    qz = np.zeros((K // G, N // 8), np.uint32)
    sb = np.tile(bits, (1, N // 2))
    L = O.layer_from_checkpoint(qw, sb, qz, np.arange(K) // G, K, N, G)
    assert L.s[0, 0] == 1.0 and L.s[0, 1] == 2.0 ** -24 and L.s[1, 0] == 65504.0 and L.s[1, 1] == 1365 / 4096


# ----------------------------------------------------------------------------- canonical shard
def _hand_shard_layers():
    """Hand example (non-identity phi): K1 = N1 = 4, N2 = 2, G = 2.
    phi1 = [2, 0, 1, 3] -> g1 = [1, 0, 0, 1] (Eq. 3); phi2 = [3, 1, 2, 0] -> g2 = [1, 0, 1, 0].
    q1[k][n] = 4k + n, s1[g][n] = 10 (g + 1) + n, z1[g][n] = g + n;
    q2[k][n] = 3k + n, s2 = [[1, 2], [3, 4]], z2 = [[5, 6], [7, 8]]."""
    q1 = np.arange(16, dtype=np.int64).reshape(4, 4)
    s1 = np.array([[10, 11, 12, 13], [20, 21, 22, 23]], dtype=np.float64)
    z1 = np.array([[0, 1, 2, 3], [1, 2, 3, 4]], dtype=np.int64)
    q2 = np.array([[0, 1], [3, 4], [6, 7], [9, 10]], dtype=np.int64)
    s2 = np.array([[1, 2], [3, 4]], dtype=np.float64)
    z2 = np.array([[5, 6], [7, 8]], dtype=np.int64)
    L1 = O.OLayer(q=q1, s=s1, z=z1, g=O.eq3_g_idx_actorder([2, 0, 1, 3], 2), G=2)
    L2 = O.OLayer(q=q2, s=s2, z=z2, g=O.eq3_g_idx_actorder([3, 1, 2, 0], 2), G=2)
    return L1, L2


def test_canonical_shard_hand_example():
    """canonical_shard at tp = 2 against values derived by hand:
    P1 = stable argsort([1,0,0,1]) = [1,2,0,3]; P2 = stable argsort([1,0,1,0]) = [1,3,0,2]; n = 2.
    TP-aware rank 0 keeps W1[P1, P2] columns P2[0:2] = [1, 3] and W2 rows [1, 3] (group 0);
    rank 1 columns [0, 2], rows [0, 2] (group 1).  Naive rank 0 keeps W1[P1] columns [0, 1]."""
    L1, L2 = _hand_shard_layers()
    a0 = O.canonical_shard(L1, L2, 2, 0, "tp_aware")
    assert a0["P1"].tolist() == [1, 2, 0, 3] and a0["P2"].tolist() == [1, 3, 0, 2]
    assert a0["w1_cols"].tolist() == [1, 3] and a0["w2_rows"].tolist() == [1, 3]
    assert a0["w1_q"].tolist() == [[5, 7], [9, 11], [1, 3], [13, 15]]
    assert a0["w1_s"].tolist() == [[11, 13], [21, 23]] and a0["w1_z"].tolist() == [[1, 3], [2, 4]]
    assert a0["w1_g"].tolist() == [0, 0, 1, 1]
    assert a0["w2_q"].tolist() == [[3, 4], [9, 10]] and a0["w2_g"].tolist() == [0, 0]
    assert a0["w2_s"].tolist() == [[1, 2]] and a0["w2_z"].tolist() == [[5, 6]]
    assert (a0["w2_group_lo"], a0["w2_group_hi"]) == (0, 1)
    assert a0["gather_src"].tolist() == [[0, 1], [1, 1]]
    a1 = O.canonical_shard(L1, L2, 2, 1, "tp_aware")
    assert a1["w1_cols"].tolist() == [0, 2] and a1["w2_rows"].tolist() == [0, 2]
    assert a1["w1_q"].tolist() == [[4, 6], [8, 10], [0, 2], [12, 14]]
    assert a1["w1_s"].tolist() == [[10, 12], [20, 22]] and a1["w1_z"].tolist() == [[0, 2], [1, 3]]
    assert a1["w2_q"].tolist() == [[0, 1], [6, 7]] and a1["w2_g"].tolist() == [0, 0]
    assert a1["w2_s"].tolist() == [[3, 4]] and a1["w2_z"].tolist() == [[7, 8]]
    assert (a1["w2_group_lo"], a1["w2_group_hi"]) == (1, 2)
    assert a1["gather_src"].tolist() == [[0, 0], [1, 0]]
    n0 = O.canonical_shard(L1, L2, 2, 0, "naive")
    assert n0["w1_cols"].tolist() == [0, 1] and n0["w1_q"].tolist() == [[4, 5], [8, 9], [0, 1], [12, 13]]
    assert n0["w2_q"].tolist() == a0["w2_q"].tolist()


# ----------------------------------------------------------------------------- gate_proj (f2)
def test_silu_closed_forms():
    """SiLU(x) = x sigmoid(x): sigmoid(ln 3) = 3/4 and sigmoid(-ln 3) = 1/4 exactly, SiLU(0) = 0,
    and SiLU(x) - SiLU(-x) = x (sigmoid(x) + sigmoid(-x) = 1) for any x."""
    ln3 = math.log(3.0)
    v = O.silu(np.array([0.0, ln3, -ln3, 2 * ln3]))
    assert v[0] == 0.0
    assert abs(v[1] - 0.75 * ln3) < 1e-15 and abs(v[2] + 0.25 * ln3) < 1e-15
    assert abs(v[3] - 2 * ln3 * 0.9) < 1e-15   # sigmoid(ln 9) = 9/10
    x = np.linspace(-20, 20, 81)
    assert np.max(np.abs(O.silu(x) - O.silu(-x) - x)) < 1e-12


def _gated_problem(K1, N1, N2, G, M, seed):
    p = synth.make_problem(K1, N1, N2, G, M, seed=seed)
    q = synth.make_problem(K1, N1, N2, G, M, seed=seed + 1000)  # an independent up_proj layer
    return p, p.w1, q.w1, p.w2


def _ol(w, K, N):
    return O.layer_from_checkpoint(w.qweight, w.scales_bits, w.qzeros, w.g_idx, K, N, w.G)


def test_gated_bruteforce_tiny():
    """gated_mlp against a pure-Python triple loop with the SiLU written out (math.exp)."""
    p, wg, wu, wd = _gated_problem(16, 16, 8, 4, 2, seed=3)
    Lg, Lu, Ld = _ol(wg, 16, 16), _ol(wu, 16, 16), _ol(wd, 16, 8)
    Wg, Wu, Wd = O.dequantize(Lg), O.dequantize(Lu), O.dequantize(Ld)
    X = p.X.astype(np.float64)
    _, Y2 = O.gated_mlp(X, Wg, Wu, Wd)
    for m in range(2):
        y1 = []
        for j in range(16):
            g = sum(X[m, k] * Lg.s[Lg.g[k], j] * (Lg.q[k, j] - Lg.z[Lg.g[k], j]) for k in range(16))
            u = sum(X[m, k] * Lu.s[Lu.g[k], j] * (Lu.q[k, j] - Lu.z[Lu.g[k], j]) for k in range(16))
            y1.append(g / (1.0 + math.exp(-g)) * u)
        for c in range(8):
            y2 = sum(y1[j] * Ld.s[Ld.g[j], c] * (Ld.q[j, c] - Ld.z[Ld.g[j], c]) for j in range(16))
            assert abs(y2 - Y2[m, c]) <= 1e-12 * max(1.0, abs(y2))


@pytest.mark.parametrize("tp", [1, 2, 4])
def test_gated_tp_variants_equal_dense(tp):
    """Both gated TP algorithms equal the dense definition (permutations and the AllReduce sum are
    exact up to fp64 rounding), and each rank's TP-aware Y1_local is the dense Y1 at columns
    P2[r n:(r+1) n] (the gate/up elementwise product commutes with the common column permutation)."""
    p, wg, wu, wd = _gated_problem(64, 128, 48, 16, 3, seed=7)
    Lg, Lu, Ld = _ol(wg, 64, 128), _ol(wu, 64, 128), _ol(wd, 128, 48)
    Y1d, Y2d = O.gated_mlp(p.X, O.dequantize(Lg), O.dequantize(Lu), O.dequantize(Ld))
    a = O.alg3_tp_aware_gated(p.X, Lg, Lu, Ld, tp)
    b = O.alg2_naive_gated(p.X, Lg, Lu, Ld, tp)
    scale = np.max(np.abs(Y2d))
    assert np.max(np.abs(a["Y2"] - Y2d)) <= 1e-12 * scale and np.max(np.abs(b["Y2"] - Y2d)) <= 1e-12 * scale
    n = 128 // tp
    for r in range(tp):
        assert np.max(np.abs(a["Y1_local"][r] - Y1d[:, a["P2"][r * n:(r + 1) * n]])) <= 1e-12 * np.max(np.abs(Y1d))
    assert not np.array_equal(a["P1g"], a["P1u"])  # the two layers carry their own act_order
