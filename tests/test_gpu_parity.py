"""GPU parity: the CUDA path (through the C-ABI) vs the fp64 oracle on the same seeded inputs.

Tolerance (reading c14, north_star): per output row m, max_n |err| <= 1e-2 * max_n |Y_oracle|.
Index plumbing is checked bit-exactly with one-hot probes in the integer regime.
"""
import numpy as np
import pytest

import oracle as O
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - GPU box only
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2402_04925_b200 as tpq  # noqa: E402

DEV = torch.device("cuda:0")
TOL = 1e-2


def _prep(p):
    P1, _ = tpq.gptq_reorder(p.w1.g_idx, p.w1.G)
    P2, _ = tpq.gptq_reorder(p.w2.g_idx, p.w2.G)
    return P1, P2


def _olayers(p):
    return (O.layer_from_checkpoint(p.w1.qweight, p.w1.scales_bits, p.w1.qzeros, p.w1.g_idx, p.K1, p.N1, p.w1.G),
            O.layer_from_checkpoint(p.w2.qweight, p.w2.scales_bits, p.w2.qzeros, p.w2.g_idx, p.N1, p.N2, p.w2.G))


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def _empty(*shape):
    return torch.full(shape, float("nan"), dtype=torch.float16, device=DEV)


def _np(t):
    torch.cuda.synchronize()
    return t.float().cpu().numpy().astype(np.float64)


def _mlp(*args, **kw):
    return tpq.TpMlp(*args, **kw)


def _assert_close(y, ref, what):
    ok, worst = O.check_rows_close(y, ref, TOL)
    assert ok, f"{what}: worst row error ratio {worst:.3e} > {TOL}"
    return worst


@pytest.mark.parametrize("M", [1, 3, 8, 9, 16])
def test_tiny_tp_aware_vs_oracle(M):
    p = synth.make_named("tiny", M, seed=0)
    P1, P2 = _prep(p)
    L1, L2 = _olayers(p)
    ref = O.alg3_tp_aware(p.X, L1, L2, 1)
    h = _mlp(p.w1, p.w2, P1, P2, M_max=16)
    X = _dev(p.X)
    Y = _empty(M, p.N2)
    h.forward(X, M, Y)
    _assert_close(_np(Y), ref["Y2"], "Y2")
    Y1 = _empty(M, p.N1)
    h.layer1(X, M, Y1)
    _assert_close(_np(Y1), ref["Y1_local"][0], "Y1")
    h.close()


@pytest.mark.parametrize("G", [32, 64, 128])
@pytest.mark.parametrize("M", [1, 5, 16])
def test_group_sizes_ragged_tail(G, M):
    """Several 64-col blocks x groups, N not a multiple of the CTA count (ragged stream-K)."""
    p = synth.make_problem(1024, 1408, 640, G, M, seed=G + M)
    P1, P2 = _prep(p)
    L1, L2 = _olayers(p)
    Y1r, Y2r = O.dense_mlp(p.X, O.dequantize(L1), O.dequantize(L2))
    h = _mlp(p.w1, p.w2, P1, P2, M_max=16)
    X = _dev(p.X)
    Y = _empty(M, p.N2)
    h.forward(X, M, Y)
    _assert_close(_np(Y), Y2r, "Y2")
    h.close()


def test_onehot_probes_exact_plumbing():
    """Integer regime + X = e_k: Y1_local[m, j] = W1[k, w1_cols[j]] exactly representable in
    fp16, so the device result must equal the oracle bit-for-bit: exposes P1 (row gather),
    P2 (column permutation) and the packed layout."""
    p = synth.make_problem(512, 1024, 256, 32, 16, seed=21, integer_regime=True)
    ks = np.random.default_rng(5).choice(512, size=16, replace=False)
    X = synth.onehot_x(16, 512, ks)
    P1, P2 = _prep(p)
    L1, L2 = _olayers(p)
    W1 = O.dequantize(L1)
    for tp in (1, 2, 4):
        for rank in range(tp):
            h = _mlp(p.w1, p.w2, P1, P2, tp=tp, rank=rank, M_max=16)
            cols, _, _, _ = h.index_maps()
            Y1 = _empty(16, 1024 // tp)
            h.layer1(_dev(X), 16, Y1)
            assert (_np(Y1) == W1[ks][:, cols]).all()
            h.close()


@pytest.mark.parametrize("tp", [2, 4, 8])
def test_tp_shards_on_one_gpu_tp_aware(tp):
    """Every rank's shard on cuda:0; partials summed in rank order (tpq_sum_partials): equals
    the oracle's Alg. 3 (and its per-rank Y1_local)."""
    M = 4
    p = synth.make_problem(512, 2048, 512, 128, M, seed=tp)
    P1, P2 = _prep(p)
    L1, L2 = _olayers(p)
    ref = O.alg3_tp_aware(p.X, L1, L2, tp)
    X = _dev(p.X)
    parts = []
    for r in range(tp):
        h = _mlp(p.w1, p.w2, P1, P2, tp=tp, rank=r, M_max=16)
        y2 = _empty(M, p.N2)
        h.forward_local(X, M, y2)
        y1 = _empty(M, p.N1 // tp)
        h.layer1(X, M, y1)
        _assert_close(_np(y1), ref["Y1_local"][r], f"Y1 rank {r}")
        _assert_close(_np(y2), ref["Y2_local"][r], f"Y2_local rank {r}")
        parts.append(y2)
        h.close()
    Y = _empty(M, p.N2)
    tpq.sum_partials(parts, Y)
    _assert_close(_np(Y), ref["Y2"], "Y2")


@pytest.mark.parametrize("tp", [1, 2, 4])
def test_naive_variant_staged(tp):
    """Alg. 2 step by step: layer1 per rank -> AllGather buffer [tp][M][n] -> P2 gather +
    CHUNK -> layer2 -> rank-order sum; and the fused forward at tp = 1."""
    M = 3
    p = synth.make_problem(512, 2048, 512, 128, M, seed=40 + tp)
    P1, P2 = _prep(p)
    L1, L2 = _olayers(p)
    ref = O.alg2_naive(p.X, L1, L2, tp)
    n = p.N1 // tp
    X = _dev(p.X)
    hs = [tpq.TpMlp(p.w1, p.w2, P1, P2, tp=tp, rank=r, variant=tpq.TPQ_NAIVE, M_max=16) for r in range(tp)]
    buf = torch.empty(tp, M, n, dtype=torch.float16, device=DEV)
    for r, h in enumerate(hs):
        h.layer1(X, M, buf[r])
        _assert_close(_np(buf[r]), ref["Y1_local"][r], f"Y1_local {r}")
    parts = []
    for r, h in enumerate(hs):
        y1in = _empty(M, n)
        h.naive_gather(buf, M, y1in)
        # the gather is pure data movement: bit-exact vs indexing the device buffer
        src = O.shard_maps(ref["P2"], p.N1, tp, r, "naive", 128)["gather_src"]
        b = buf.cpu().numpy()
        assert (y1in.cpu().numpy() == b[src[:, 0], :, src[:, 1]].T).all()
        y2 = _empty(M, p.N2)
        h.layer2(y1in, M, y2)
        parts.append(y2)
    Y = _empty(M, p.N2)
    tpq.sum_partials(parts, Y)
    _assert_close(_np(Y), ref["Y2"], "Y2 naive")
    if tp == 1:
        Yf = _empty(M, p.N2)
        hs[0].forward(X, M, Yf)
        _assert_close(_np(Yf), ref["Y2"], "Y2 naive fused")
    for h in hs:
        h.close()


def test_deterministic_and_graph_capturable():
    M = 16
    p = synth.make_problem(2048, 4096, 2048, 128, M, seed=77)
    P1, P2 = _prep(p)
    h = _mlp(p.w1, p.w2, P1, P2, M_max=16)
    X = _dev(p.X)
    Ya, Yb = _empty(M, p.N2), _empty(M, p.N2)
    h.forward(X, M, Ya)
    for _ in range(3):
        h.forward(X, M, Yb)
        torch.cuda.synchronize()
        assert torch.equal(Ya, Yb)
    s = torch.cuda.Stream()
    Yg = _empty(M, p.N2)
    with torch.cuda.stream(s):
        h.forward(X, M, Yg, stream=s)  # warm
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            h.forward(X, M, Yg, stream=s)
    Yg.fill_(0)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(Ya, Yg)
    h.close()


def test_m_above_16_chunks_and_host_e2e():
    M = 37
    p = synth.make_problem(1024, 2048, 1024, 128, M, seed=3)
    P1, P2 = _prep(p)
    L1, L2 = _olayers(p)
    _, Y2r = O.dense_mlp(p.X, O.dequantize(L1), O.dequantize(L2))
    h = tpq.TpMlp(p.w1, p.w2, P1, P2, M_max=64)
    Yh = np.zeros((M, p.N2), np.float16)
    h.forward_host(p.X, Yh, stream=torch.cuda.current_stream().cuda_stream)
    _assert_close(Yh.astype(np.float64), Y2r, "Y2 host e2e")
    Y = _empty(M, p.N2)
    h.forward(_dev(p.X), M, Y)
    assert (Y.cpu().numpy() == Yh).all()
    with pytest.raises(tpq.TPQError):
        h.forward(_dev(p.X), 65, Y)
    h.close()


@pytest.mark.parametrize("shape,M", [("llama70b", 1), ("llama70b", 16), ("granite20b", 4)])
def test_full_size_sampled(shape, M):
    """BASELINE.json configs at full size in the launch configuration bench.py times:
    all of Y1 and 512 sampled columns of Y2 against the oracle."""
    p = synth.make_named(shape, M, seed=0)
    P1, P2 = _prep(p)
    L1, L2 = _olayers(p)
    cols = np.sort(np.random.default_rng(0).choice(p.N2, 512, replace=False))
    h = _mlp(p.w1, p.w2, P1, P2, M_max=16)
    X = _dev(p.X)
    Y = _empty(M, p.N2)
    h.forward(X, M, Y)
    Y1 = _empty(M, p.N1)
    h.layer1(X, M, Y1)
    P1o, _ = O.alg1_reorder(L1.g)
    P2o, _ = O.alg1_reorder(L2.g)
    Y1r, Y2r = O.dense_mlp_columns(p.X, L1, L2, cols2=cols)
    _assert_close(_np(Y1), Y1r[:, P2o], "Y1 (P2 order)")
    _assert_close(_np(Y)[:, cols], Y2r, "Y2 sampled")
    h.close()


def test_full_size_repeat_bit_identical():
    """Llama-70B layer 1 at M = 16, interleaved with full forwards: every repeat must be
    bit-identical (fixed split-K order, reading c20).  Catches ring races: a stage released
    before its loads returned made 24 of 60 repeats differ in the register GEMV."""
    M = 16
    p = synth.make_named("llama70b", M, seed=0)
    P1, P2 = _prep(p)
    h = _mlp(p.w1, p.w2, P1, P2, M_max=16)
    X = _dev(p.X)
    Y = _empty(M, p.N2)
    ref = _empty(M, p.N1)
    h.layer1(X, M, ref)
    for it in range(24):
        if it % 2 == 0:
            h.forward(X, M, Y)
        Y1 = _empty(M, p.N1)
        h.layer1(X, M, Y1)
        torch.cuda.synchronize()
        assert torch.equal(Y1, ref), f"repeat {it}: {(Y1 != ref).sum().item()} elements differ"
    h.close()


# ----------------------------------------------------------------------------- A7 (M > 16)
@pytest.mark.parametrize("G", [32, 64, 128])
@pytest.mark.parametrize("M", [17, 64, 100, 256, 300])
def test_a7_tensor_core_path(G, M):
    """M > 16 runs the A7 tensor-core GEMM (N = 64 / 128 / 256 rows per pass, several passes
    above 256) on ragged stream-K shapes: Y2 and the staged Y1 against the fp64 oracle."""
    p = synth.make_problem(1024, 1408, 640, G, M, seed=100 + G + M)
    P1, P2 = _prep(p)
    L1, L2 = _olayers(p)
    Y1r, Y2r = O.dense_mlp(p.X, O.dequantize(L1), O.dequantize(L2))
    h = tpq.TpMlp(p.w1, p.w2, P1, P2, M_max=512)
    X = _dev(p.X)
    Y = _empty(M, p.N2)
    h.forward(X, M, Y)
    _assert_close(_np(Y), Y2r, "Y2")
    Y1 = _empty(M, p.N1)
    h.layer1(X, M, Y1)
    P2o, _ = O.alg1_reorder(L2.g)
    _assert_close(_np(Y1), Y1r[:, P2o], "Y1 (P2 order)")
    h.close()


def test_a7_naive_and_tp_shards():
    """A7 on the naive variant's staged path and on TP=4 shards summed in rank order."""
    M, tp = 72, 4
    p = synth.make_problem(512, 2048, 512, 128, M, seed=7)
    P1, P2 = _prep(p)
    L1, L2 = _olayers(p)
    ref = O.alg3_tp_aware(p.X, L1, L2, tp)
    X = _dev(p.X)
    parts = []
    for r in range(tp):
        h = tpq.TpMlp(p.w1, p.w2, P1, P2, tp=tp, rank=r, M_max=256)
        y2 = _empty(M, p.N2)
        h.forward_local(X, M, y2)
        _assert_close(_np(y2), ref["Y2_local"][r], f"Y2_local rank {r}")
        parts.append(y2)
        h.close()
    Y = _empty(M, p.N2)
    tpq.sum_partials(parts, Y)
    _assert_close(_np(Y), ref["Y2"], "Y2")
    hn = tpq.TpMlp(p.w1, p.w2, P1, P2, tp=1, variant=tpq.TPQ_NAIVE, M_max=256)
    Yn = _empty(M, p.N2)
    hn.forward(X, M, Yn)
    _assert_close(_np(Yn), ref["Y2"], "Y2 naive tp=1")
    hn.close()


@pytest.mark.parametrize("M", [200, 512])
def test_a7_full_size_llama_tp8_shard(M):
    """BASELINE.json configs[3]: Llama-70B MLP at TP=8 (rank 0's shard), M = 200 / 512, in the
    launch configuration bench.py times; Y1_local in full and 256 sampled columns of Y2_local."""
    p = synth.make_named("llama70b", M, seed=1)
    P1, P2 = _prep(p)
    L1, L2 = _olayers(p)
    tp, n = 8, p.N1 // 8
    h = tpq.TpMlp(p.w1, p.w2, P1, P2, tp=tp, rank=0, M_max=512)
    X = _dev(p.X)
    Y2 = _empty(M, p.N2)
    h.forward_local(X, M, Y2)
    Y1 = _empty(M, n)
    h.layer1(X, M, Y1)
    P2o, _ = O.alg1_reorder(L2.g)
    cols = np.sort(np.random.default_rng(1).choice(p.N2, 256, replace=False))
    # rank 0: X[:, P1] . W1[P1, P2][:, :n] = X . W1[:, P2[:n]];  Y2_local = Y1_local . W2[P2[:n]]
    y1r = np.asarray(p.X, np.float64) @ O.dequantize(O.permute_cols(L1, P2o[:n]))
    L2r = O.permute_rows(L2, P2o[:n])
    y2r = y1r @ O.dequantize(O.OLayer(q=L2r.q[:, cols], s=L2r.s[:, cols], z=L2r.z[:, cols], g=L2r.g, G=L2r.G))
    _assert_close(_np(Y1), y1r, "Y1_local")
    _assert_close(_np(Y2)[:, cols], y2r, "Y2_local sampled")
    h.close()


@pytest.mark.parametrize("G", [64, 128])
@pytest.mark.parametrize("M", [128, 200])
def test_a7_ss_wide_tiles(G, M):
    """M >= 128 runs the SS GEMM (k-splits, fix-up); deterministic across runs."""
    p = synth.make_problem(1024, 2048, 768, G, M, seed=300 + G + M)
    P1, P2 = _prep(p)
    L1, L2 = _olayers(p)
    Y1r, Y2r = O.dense_mlp(p.X, O.dequantize(L1), O.dequantize(L2))
    h = tpq.TpMlp(p.w1, p.w2, P1, P2, M_max=256)
    X = _dev(p.X)
    Y = _empty(M, p.N2)
    h.forward(X, M, Y)
    _assert_close(_np(Y), Y2r, "Y2")
    Y1 = _empty(M, p.N1)
    h.layer1(X, M, Y1)
    P2o, _ = O.alg1_reorder(L2.g)
    _assert_close(_np(Y1), Y1r[:, P2o], "Y1 (P2 order)")
    Y2 = _empty(M, p.N2)
    h.forward(X, M, Y2)
    assert torch.equal(Y, Y2), "SS GEMM not deterministic"
    h.close()


@pytest.mark.parametrize("G", [32, 64, 128])
@pytest.mark.parametrize("M", [129, 256, 384])
def test_a7_cta_pair(G, M):
    """Passes of more than 128 rows over an even tile count run the CTA-pair SS GEMM (cta_group::2,
    256 x 256 per pair): the 129-row pass leaves the second CTA's rows padding, 384 = a full pair
    pass + a 128-row pass on the 1-CTA kernel; NKB = 9 gives ragged k-splits."""
    p = synth.make_problem(1152, 2304, 512, G, M, seed=500 + G + M)
    P1, P2 = _prep(p)
    L1, L2 = _olayers(p)
    Y1r, Y2r = O.dense_mlp(p.X, O.dequantize(L1), O.dequantize(L2))
    h = tpq.TpMlp(p.w1, p.w2, P1, P2, M_max=512)
    X = _dev(p.X)
    Y = _empty(M, p.N2)
    h.forward(X, M, Y)
    _assert_close(_np(Y), Y2r, "Y2")
    Y1 = _empty(M, p.N1)
    h.layer1(X, M, Y1)
    P2o, _ = O.alg1_reorder(L2.g)
    _assert_close(_np(Y1), Y1r[:, P2o], "Y1 (P2 order)")
    Yb = _empty(M, p.N2)
    h.forward(X, M, Yb)
    assert torch.equal(Y, Yb), "pair GEMM not deterministic"
    h.close()


def _check_elementwise(y, ref, absref, tol, what):
    """|y - ref| <= tol * absref element by element, absref = |inputs| . |W| (the worst-case
    rounding bound of a dot product: each term carries its own relative error, so a column made of
    small scales is held to its own magnitude, and cancellation in the output does not matter)."""
    ratio = np.abs(y - ref) / np.where(absref > 0, absref, 1.0)
    worst = np.unravel_index(int(np.argmax(ratio)), ratio.shape)
    assert np.all(ratio <= tol), f"{what}: element {worst} error {ratio[worst]:.3e} x |inputs|.|W| > {tol}"
    return float(ratio.max())


@pytest.mark.parametrize("M", [1, 8, 40, 160])
def test_wide_scale_range_per_column(M):
    """Scales log-uniform over 5.5 decades (whole columns up to 4 decades below the largest, 1.5
    within a column; synth wide_scales): every output element within 2e-3 (layer 1) / 4e-3
    (layer 2, fp16 Y1 input) of |inputs| . |W|.  A single operand shift per layer (round 1) leaves
    the fp16 A operand of the small-scale columns subnormal: emulated in numpy it reaches 1.0e-2 on
    this recipe, against 1.8e-4 for the per-column exponent of the records (reading c22).  M covers
    the GEMV and both A7 kernels."""
    p = synth.make_problem(1024, 2048, 1024, 128, M, seed=5, wide_scales=True)
    P1, P2 = _prep(p)
    L1, L2 = _olayers(p)
    h = tpq.TpMlp(p.w1, p.w2, P1, P2, M_max=256)
    X = _dev(p.X)
    Y1 = _empty(M, p.N1)
    h.layer1(X, M, Y1)
    Y = _empty(M, p.N2)
    h.forward(X, M, Y)
    P2o, _ = O.alg1_reorder(L2.g)
    W1, W2 = O.dequantize(L1), O.dequantize(L2)
    Xf = p.X.astype(np.float64)
    Y1r, Y2r = O.dense_mlp(Xf, W1, W2)
    b1 = np.abs(Xf) @ np.abs(W1)
    b2 = np.abs(Y1r) @ np.abs(W2)
    _check_elementwise(_np(Y1), Y1r[:, P2o], b1[:, P2o], 2e-3, "Y1 (P2 order)")
    _check_elementwise(_np(Y), Y2r, b2, 4e-3, "Y2")
    h.close()


@pytest.mark.parametrize("tp", [2, 4, 8])
@pytest.mark.parametrize("M", [1, 16, 32])
def test_full_size_tp_shards(tp, M):
    """Llama-70B shards at TP = 2/4/8 in the launch configuration of a TP-rank (the small-shard
    grid, 5-6 stream-K contributors per layer-1 tile), first and last rank: Y1_local in full and
    512 sampled columns of Y2_local against the oracle's Alg. 3 L1-L2 for that rank."""
    p = synth.make_named("llama70b", M, seed=1)
    P1, P2 = _prep(p)
    L1, L2 = _olayers(p)
    n = p.N1 // tp
    X = _dev(p.X)
    cols = np.sort(np.random.default_rng(tp).choice(p.N2, 512, replace=False))
    for r in (0, tp - 1):
        mp = O.shard_maps(O.alg1_reorder(L2.g)[0], p.N1, tp, r, "tp_aware", p.G)
        # Alg. 3 L1 for rank r: X[:, P1] W1[P1, P2][:, r n:(r+1) n] = X W1[:, w1_cols]
        Xf = p.X.astype(np.float64)
        c1 = mp["w1_cols"]
        Y1r = np.concatenate([Xf @ O.dequantize(O.permute_cols(L1, c1[lo:lo + 2048])) for lo in range(0, n, 2048)], axis=1)
        # Alg. 3 L2 for rank r: Y1_local W2[P2][r n:(r+1) n]
        W2r = O.permute_rows(L2, mp["w2_rows"])
        W2rc = O.OLayer(q=W2r.q[:, cols], s=W2r.s[:, cols], z=W2r.z[:, cols], g=W2r.g, G=W2r.G)
        Y2r = Y1r @ O.dequantize(W2rc)
        h = tpq.TpMlp(p.w1, p.w2, P1, P2, tp=tp, rank=r, M_max=max(16, M))  # M = 32: the N = 32 GEMV
        Y1 = _empty(M, n)
        h.layer1(X, M, Y1)
        Y2 = _empty(M, p.N2)
        h.forward_local(X, M, Y2)
        _assert_close(_np(Y1), Y1r, f"tp={tp} rank {r} Y1_local")
        _assert_close(_np(Y2)[:, cols], Y2r, f"tp={tp} rank {r} Y2_local sampled")
        h.close()


@pytest.mark.parametrize("G,M", [(32, 1), (64, 5), (128, 16)])
def test_unordered_locality_baseline(G, M):
    """TPQ_UNORDERED (f3, the Fig. 1 formulation): no reordering, per-row group metadata looked up
    from the table; Y1 (checkpoint column order) and Y2 against the oracle's plain definition with
    the unordered g_idx (exactly what oracle.dequantize computes)."""
    p = synth.make_problem(1024, 1408, 640, G, M, seed=31)
    L1, L2 = _olayers(p)
    h = tpq.TpMlp(p.w1, p.w2, None, None, variant=tpq.TPQ_UNORDERED, M_max=16)
    X = _dev(p.X)
    Y1 = _empty(M, p.N1)
    h.layer1(X, M, Y1)
    Y = _empty(M, p.N2)
    h.forward(X, M, Y)
    Y1r, Y2r = O.dense_mlp(p.X, O.dequantize(L1), O.dequantize(L2))
    _assert_close(_np(Y1), Y1r, "Y1 unordered")
    _assert_close(_np(Y), Y2r, "Y2 unordered")
    h.close()


@pytest.mark.parametrize("M", [1, 16])
def test_unordered_full_size_llama(M):
    p = synth.make_named("llama70b", M, seed=0)
    L1, L2 = _olayers(p)
    cols = np.sort(np.random.default_rng(3).choice(p.N2, 256, replace=False))
    h = tpq.TpMlp(p.w1, p.w2, None, None, variant=tpq.TPQ_UNORDERED, M_max=16)
    Y = _empty(M, p.N2)
    h.forward(_dev(p.X), M, Y)
    _, Y2r = O.dense_mlp_columns(p.X, L1, L2, cols2=cols)
    _assert_close(_np(Y)[:, cols], Y2r, "Y2 unordered, full size")
    h.close()


def _gated(K1, N1, N2, G, M, seed):
    """gate (p.w1), up (an independent layer from another seed's w1), down (p.w2)."""
    p = synth.make_problem(K1, N1, N2, G, M, seed=seed)
    q = synth.make_problem(K1, N1, N2, G, M, seed=seed + 1000)
    wg, wu, wd = p.w1, q.w1, p.w2
    Lg = O.layer_from_checkpoint(wg.qweight, wg.scales_bits, wg.qzeros, wg.g_idx, K1, N1, G)
    Lu = O.layer_from_checkpoint(wu.qweight, wu.scales_bits, wu.qzeros, wu.g_idx, K1, N1, G)
    Ld = O.layer_from_checkpoint(wd.qweight, wd.scales_bits, wd.qzeros, wd.g_idx, N1, N2, G)
    Ps = [tpq.gptq_reorder(w.g_idx, G)[0] for w in (wg, wu, wd)]
    return p, (wg, wu, wd), (Lg, Lu, Ld), Ps


@pytest.mark.parametrize("G,M", [(32, 1), (64, 5), (128, 16)])
def test_gated_tp_aware_vs_oracle(G, M):
    """f2: Y = (SiLU(X.Wg) * (X.Wu)).Wd, one GEMV over interleaved gate/up records with the SiLU
    product in its epilogue (and in the split-tile fix-up), vs the oracle's Alg. 3 generalization."""
    p, ws, Ls, Ps = _gated(1024, 1408, 640, G, M, seed=50 + G)
    ref = O.alg3_tp_aware_gated(p.X, *Ls, 1)
    h = tpq.TpMlp.gated(*ws, *Ps, M_max=16)
    X = _dev(p.X)
    Y1 = _empty(M, p.N1)
    h.layer1(X, M, Y1)
    Y = _empty(M, p.N2)
    h.forward(X, M, Y)
    _assert_close(_np(Y1), ref["Y1_local"][0], "gated Y1 (P2 order)")
    _assert_close(_np(Y), ref["Y2"], "gated Y2")
    h.close()


@pytest.mark.parametrize("tp", [2, 4, 8])
def test_gated_tp_shards_and_naive(tp):
    """Every rank's gated shard on cuda:0 (partials summed in rank order) vs the gated Alg. 3, and
    the gated Alg. 2 step by step (layer 1 -> AllGather buffer -> P2 gather + CHUNK -> layer 2)."""
    M = 4
    p, ws, Ls, Ps = _gated(512, 2048, 512, 128, M, seed=60 + tp)
    X = _dev(p.X)
    ref = O.alg3_tp_aware_gated(p.X, *Ls, tp)
    parts = []
    for r in range(tp):
        h = tpq.TpMlp.gated(*ws, *Ps, tp=tp, rank=r, M_max=16)
        y1 = _empty(M, p.N1 // tp)
        h.layer1(X, M, y1)
        _assert_close(_np(y1), ref["Y1_local"][r], f"gated Y1 rank {r}")
        y2 = _empty(M, p.N2)
        h.forward_local(X, M, y2)
        parts.append(y2)
        h.close()
    Y = _empty(M, p.N2)
    tpq.sum_partials(parts, Y)
    _assert_close(_np(Y), ref["Y2"], "gated Y2 TP-aware")
    refn = O.alg2_naive_gated(p.X, *Ls, tp)
    n = p.N1 // tp
    hs = [tpq.TpMlp.gated(*ws, *Ps, tp=tp, rank=r, variant=tpq.TPQ_NAIVE, M_max=16) for r in range(tp)]
    buf = torch.empty(tp, M, n, dtype=torch.float16, device=DEV)
    for r, h in enumerate(hs):
        h.layer1(X, M, buf[r])
        _assert_close(_np(buf[r]), refn["Y1_local"][r], f"gated naive Y1 rank {r}")
    parts = []
    for h in hs:
        y1in = _empty(M, n)
        h.naive_gather(buf, M, y1in)
        y2 = _empty(M, p.N2)
        h.layer2(y1in, M, y2)
        parts.append(y2)
        h.close()
    tpq.sum_partials(parts, Y)
    _assert_close(_np(Y), refn["Y2"], "gated Y2 naive")


@pytest.mark.parametrize("M", [1, 16])
def test_gated_full_size_llama(M):
    """Llama-70B with a gate_proj layer (K1=8192, N1=28672 for gate and up): all of Y1 and 256
    sampled columns of Y2 against the oracle's definition."""
    p, ws, Ls, Ps = _gated(8192, 28672, 8192, 128, M, seed=70)
    Lg, Lu, Ld = Ls
    h = tpq.TpMlp.gated(*ws, *Ps, M_max=16)
    X = _dev(p.X)
    Y1 = _empty(M, p.N1)
    h.layer1(X, M, Y1)
    Y = _empty(M, p.N2)
    h.forward(X, M, Y)
    Xf = p.X.astype(np.float64)
    g = np.concatenate([Xf @ O.dequantize(O.permute_cols(Lg, np.arange(lo, lo + 2048))) for lo in range(0, p.N1, 2048)], 1)
    u = np.concatenate([Xf @ O.dequantize(O.permute_cols(Lu, np.arange(lo, lo + 2048))) for lo in range(0, p.N1, 2048)], 1)
    Y1r = O.silu(g) * u
    cols = np.sort(np.random.default_rng(4).choice(p.N2, 256, replace=False))
    Y2r = Y1r @ O.dequantize(O.permute_cols(Ld, cols))
    _assert_close(_np(Y1), Y1r[:, Ps[2]], "gated Y1 full size (P2 order)")
    _assert_close(_np(Y)[:, cols], Y2r, "gated Y2 full size, sampled")
    h.close()


# Split-tile reduction modes of the M <= 16 GEMV (tpq.h tpq_mlp_info_t.split1/2): stream-K with the
# in-kernel reduction (0), stream-K with the fix-up kernel (1), cluster split-K of 2 or 4 CTAs
# reduced through distributed shared memory.  TPQ_CLUSTER / TPQ_FIXUP_KERNEL / TPQ_INRED_MAX are
# read when the handle is built.
_MODES = {"inkernel": {"TPQ_CLUSTER": "1", "TPQ_INRED_MAX": "64"}, "fixup": {"TPQ_CLUSTER": "1", "TPQ_FIXUP_KERNEL": "1"},
          "cluster2": {"TPQ_CLUSTER": "2"}, "cluster4": {"TPQ_CLUSTER": "4"}}


def _mode_handle(monkeypatch, mode, *args, **kw):
    for k in ("TPQ_CLUSTER", "TPQ_FIXUP_KERNEL", "TPQ_INRED_MAX"):
        monkeypatch.delenv(k, raising=False)
    for k, v in _MODES[mode].items():
        monkeypatch.setenv(k, v)
    h = _mlp(*args, **kw)
    for k in _MODES[mode]:
        monkeypatch.delenv(k, raising=False)
    return h


@pytest.mark.parametrize("mode", ["inkernel", "fixup", "cluster2", "cluster4"])
@pytest.mark.parametrize("G", [32, 64, 128])
@pytest.mark.parametrize("M", [1, 7, 16])
def test_split_tile_reduction_modes(monkeypatch, mode, G, M):
    """Every split-tile reduction mode against the oracle's Alg. 3 (tp = 2 shards of a small MLP whose
    tiles span several CTAs), bit-identical across repeats; the mode is the one requested."""
    tp = 2
    p = synth.make_problem(2048, 2048, 2048, G, M, seed=G + M)
    P1, P2 = _prep(p)
    L1, L2 = _olayers(p)
    ref = O.alg3_tp_aware(p.X, L1, L2, tp)
    X = _dev(p.X)
    want = {"inkernel": 0, "fixup": 1, "cluster2": 2, "cluster4": 4}[mode]
    for r in range(tp):
        h = _mode_handle(monkeypatch, mode, p.w1, p.w2, P1, P2, tp=tp, rank=r, M_max=16)
        info = h.info
        if want == 4 and G != 128:  # the landing zone holds one partial only below G = 128
            assert info.split1 in (1, 0, 2) and info.split2 in (0, 1, 2)
        else:
            assert info.split1 == want and info.split2 == want, (info.split1, info.split2)
        y2, y2b = _empty(M, p.N2), _empty(M, p.N2)
        h.forward_local(X, M, y2)
        y1 = _empty(M, p.N1 // tp)
        h.layer1(X, M, y1)
        _assert_close(_np(y1), ref["Y1_local"][r], f"{mode} Y1 rank {r}")
        _assert_close(_np(y2), ref["Y2_local"][r], f"{mode} Y2_local rank {r}")
        for _ in range(2):
            h.forward_local(X, M, y2b)
            torch.cuda.synchronize()
            assert torch.equal(y2, y2b), f"{mode}: repeated forward differs"
        h.close()


@pytest.mark.parametrize("G", [32, 64, 128])
@pytest.mark.parametrize("M", [17, 24, 32])
def test_gemv_n32_passes(G, M):
    """Passes of 17..32 rows run the GEMV pipeline with N = 32 (tpq_host.cpp gemv32): tiny / ragged
    shapes at tp = 1 and a tp = 2 shard pair against the oracle, bit-identical repeats."""
    p = synth.make_problem(1024, 2560, 768, G, M, seed=3 * G + M)
    P1, P2 = _prep(p)
    L1, L2 = _olayers(p)
    X = _dev(p.X)
    ref = O.alg3_tp_aware(p.X, L1, L2, 1)
    h = _mlp(p.w1, p.w2, P1, P2, M_max=32)
    Y, Yb = _empty(M, p.N2), _empty(M, p.N2)
    h.forward(X, M, Y)
    _assert_close(_np(Y), ref["Y2"], f"N=32 GEMV M={M} G={G}")
    h.forward(X, M, Yb)
    torch.cuda.synchronize()
    assert torch.equal(Y, Yb)
    h.close()
    ref2 = O.alg3_tp_aware(p.X, L1, L2, 2)
    parts = []
    for r in range(2):
        hr = _mlp(p.w1, p.w2, P1, P2, tp=2, rank=r, M_max=32)
        y2 = _empty(M, p.N2)
        hr.forward_local(X, M, y2)
        _assert_close(_np(y2), ref2["Y2_local"][r], f"N=32 GEMV tp=2 rank {r}")
        parts.append(y2)
        hr.close()


@pytest.mark.parametrize("tp", [1, 8])
def test_partition_modes_repeat_under_graph_replay(tp):
    """Race check of the split-tile reductions in their production launch configuration: 160
    graph-replayed forwards (two cold weight replicas, back to back with programmatic dependent
    launch) of one Llama rank's shard -- stream-K with the in-kernel reduction at TP=1, clusters of
    4 and 2 at TP=8 -- all bit-identical to the first (tools/stress_modes.py runs more)."""
    M = 16
    p = synth.make_named("llama70b", M, 0)
    P1, P2 = _prep(p)
    hs = [_mlp(p.w1, p.w2, P1, P2, tp=tp, rank=tp - 1, M_max=16) for _ in range(2)]
    X = _dev(p.X)
    Ys = [_empty(M, p.N2) for _ in range(2)]
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for i in range(4):
            hs[i % 2].forward_local(X, M, Ys[i % 2], stream=st)
    torch.cuda.synchronize()
    ref = [y.clone() for y in Ys]
    with torch.cuda.stream(st):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for i in range(16):
                hs[i % 2].forward_local(X, M, Ys[i % 2], stream=st)
    for _ in range(10):
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(Ys[0], ref[0]) and torch.equal(Ys[1], ref[1])
    for h in hs:
        h.close()
