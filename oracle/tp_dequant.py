"""Plain fp64 oracle of the TP-aware GPTQ MLP forward.  TEST INFRASTRUCTURE ONLY.

(See ``oracle/__init__.py``: only tests/, smoke() and bench.py's cpu-baseline legs
may use this module.)

Citations are ``PAPER.md:L<a>-<b>`` into /root/reference/PAPER.md (the paper's
LaTeX), and ``SPEC.md:L<n>`` into /root/reference/SPEC.md where the paper is
silent.  Readings of silent / ambiguous points are the DESIGN.md ledger entries
``c1``..``c21`` (same numbering as SURVEY.md §8(c)).

Nothing here is blocked, fused or reordered beyond what the cited definition
states.  Library primitives used as steps: numpy fancy indexing (gather),
``@`` (fp64 matmul), Python's stable ``sorted`` (Alg. 1's ARGSORT, reading c6).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = [
    "eq1_g_idx_naive", "eq3_g_idx_actorder", "alg1_reorder", "invert_permutation",
    "unpack_qweight", "unpack_qzeros", "fp16_bits_to_f64", "OLayer", "layer_from_checkpoint",
    "dequantize", "metadata_loads", "dense_mlp", "permute_rows", "permute_cols",
    "alg2_naive", "alg3_tp_aware", "shard_maps", "canonical_shard", "check_rows_close",
    "dense_mlp_columns", "silu", "gated_mlp", "alg3_tp_aware_gated", "alg2_naive_gated",
]


# ----------------------------------------------------------------------------- Eq. 1 / Eq. 3
def eq1_g_idx_naive(K: int, G: int) -> np.ndarray:
    """Eq. 1: g_idx_naive[i] = floor(i / G), i = 0..K-1."""
    if K < 1 or G < 1:
        raise ValueError("K and G must be >= 1 (SPEC.md:L56)")
    return np.array([i // G for i in range(K)], dtype=np.int64)


def eq3_g_idx_actorder(phi, G: int) -> np.ndarray:
    """Eq. 3: g_idx_actorder[i] = floor(phi(i) / G)."""
    phi = np.asarray(phi, dtype=np.int64)
    if G < 1:
        raise ValueError("G must be >= 1")
    return np.array([int(p) // G for p in phi], dtype=np.int64)


# ----------------------------------------------------------------------------- Alg. 1
def alg1_reorder(g_idx):
    """Alg. 1 "Reorder Function".

    Line 2: P <- ARGSORT(g_idx_actorder).  ARGSORT is read as the *stable* argsort
    (ties by ascending original index), reading c6 / SPEC.md:L140.
    Line 3: g_idx_optimized <- g_idx_actorder[P].
    Line 4: return P, g_idx_optimized.
    """
    g = [int(v) for v in np.asarray(g_idx).ravel()]
    P = sorted(range(len(g)), key=g.__getitem__)  # Python's sort is stable
    P = np.array(P, dtype=np.int64)
    g_opt = np.asarray(g, dtype=np.int64)[P]
    return P, g_opt


def invert_permutation(P) -> np.ndarray:
    """Q with Q[P[i]] = i."""
    P = np.asarray(P, dtype=np.int64)
    Q = np.empty_like(P)
    for i, p in enumerate(P):
        Q[p] = i
    return Q


# ----------------------------------------------------------------------------- checkpoint
def unpack_qweight(qweight: np.ndarray, K: int) -> np.ndarray:
    """GPTQ qweight [K/8][N] uint32 -> q [K][N]; row k is nibble k%8 of word k//8 (reading c4)."""
    qw = np.asarray(qweight, dtype=np.uint64)
    rows = []
    for k in range(K):
        rows.append((qw[k // 8] >> np.uint64(4 * (k % 8))) & np.uint64(0xF))
    return np.stack(rows).astype(np.int64)


def unpack_qzeros(qzeros: np.ndarray, N: int) -> np.ndarray:
    """GPTQ qzeros [ng][N/8] uint32 -> z [ng][N]; column n is nibble n%8 of word n//8 (c4)."""
    qz = np.asarray(qzeros, dtype=np.uint64)
    cols = []
    for n in range(N):
        cols.append((qz[:, n // 8] >> np.uint64(4 * (n % 8))) & np.uint64(0xF))
    return np.stack(cols, axis=1).astype(np.int64)


def fp16_bits_to_f64(bits: np.ndarray) -> np.ndarray:
    return np.asarray(bits, dtype=np.uint16).view(np.float16).astype(np.float64)


@dataclass
class OLayer:
    """A quantized K x N matrix: codes q, per-group scales s and zeros z, group index g.

    PAPER.md:L19 ("every group size number of input channels ... share the same
    quantization metadata (scales and zeros)"); field layout SPEC.md:L38-44.
    """

    q: np.ndarray   # int64 [K][N] in 0..15
    s: np.ndarray   # float64 [ng][N]
    z: np.ndarray   # int64 [ng][N]
    g: np.ndarray   # int64 [K]    group of each row
    G: int

    @property
    def K(self):
        return self.q.shape[0]

    @property
    def N(self):
        return self.q.shape[1]


def layer_from_checkpoint(qweight, scales_bits, qzeros, g_idx, K: int, N: int, G: int) -> OLayer:
    return OLayer(q=unpack_qweight(qweight, K), s=fp16_bits_to_f64(scales_bits),
                  z=unpack_qzeros(qzeros, N), g=np.asarray(g_idx, dtype=np.int64).copy(), G=G)


def dequantize(L: OLayer) -> np.ndarray:
    """W[k, n] = s[g[k], n] * (q[k, n] - z[g[k], n]) in fp64.

    PAPER.md:L19 (scales and zeros per group, "used during deployment when
    performing dequantization"), formula SPEC.md:L43, zero convention reading c3.
    Uses the layer's own group index row by row -- with the *unordered* Eq.-3 g
    this is the naive act_order formulation of PAPER.md:L36 / Fig. 1.
    """
    s_rows = L.s[L.g, :]
    z_rows = L.z[L.g, :].astype(np.float64)
    return s_rows * (L.q.astype(np.float64) - z_rows)


def metadata_loads(g_idx) -> int:
    """Metadata (re)loads when rows are visited in order: 1 + #{i : g[i] != g[i-1]}.

    PAPER.md:L36 ("frequently reload quantization metadata"), L57 ordered groups
    are consecutive; counting convention SPEC.md:L92-100.
    """
    g = [int(v) for v in np.asarray(g_idx).ravel()]
    if not g:
        return 0
    return 1 + sum(1 for i in range(1, len(g)) if g[i] != g[i - 1])


def dense_mlp(X, W1, W2):
    """Y1 = X . W1 ; Y2 = Y1 . W2 in fp64 (north_star Y=(X.W1).W2; PAPER.md:L151 single
    up_proj followed by down_proj, no activation -- reading c9)."""
    X = np.asarray(X, dtype=np.float64)
    Y1 = X @ W1
    Y2 = Y1 @ W2
    return Y1, Y2


def dense_mlp_columns(X, L1: OLayer, L2: OLayer, cols2=None, chunk: int = 2048):
    """The same definition as ``dense_mlp(X, dequantize(L1), dequantize(L2))`` evaluated one
    block of output columns at a time so full-size shapes fit in host memory: column j of
    Y1 is X . W1[:, j] (column blocks of W1 dequantized independently), and only the
    requested columns ``cols2`` of Y2 = Y1 . W2[:, cols2] are produced (sampled outputs).
    Returns (Y1 [M][N1], Y2 [M][len(cols2)])."""
    X = np.asarray(X, dtype=np.float64)
    Y1 = np.empty((X.shape[0], L1.N))
    for lo in range(0, L1.N, chunk):
        hi = min(L1.N, lo + chunk)
        Y1[:, lo:hi] = X @ dequantize(_col_block(L1, lo, hi))
    cols2 = np.arange(L2.N) if cols2 is None else np.asarray(cols2, dtype=np.int64)
    L2c = OLayer(q=L2.q[:, cols2], s=L2.s[:, cols2], z=L2.z[:, cols2], g=L2.g, G=L2.G)
    return Y1, Y1 @ dequantize(L2c)


# ----------------------------------------------------------------------------- M[P1, P2]
def permute_rows(L: OLayer, P) -> OLayer:
    """W[P]: rows gathered by P (notation PAPER.md:L104, gather reading c7).  The group
    index travels with its row, so W[P] dequantizes to dequantize(W)[P]."""
    P = np.asarray(P, dtype=np.int64)
    return OLayer(q=L.q[P, :], s=L.s, z=L.z, g=L.g[P], G=L.G)


def permute_cols(L: OLayer, P) -> OLayer:
    """W[:, P]: columns of codes AND of per-column metadata gathered by P (reading c8,
    PAPER.md:L127 "re-ordering the columns of W1 with the permutation array P2")."""
    P = np.asarray(P, dtype=np.int64)
    return OLayer(q=L.q[:, P], s=L.s[:, P], z=L.z[:, P], g=L.g, G=L.G)


def _col_block(L: OLayer, lo: int, hi: int) -> OLayer:
    return OLayer(q=L.q[:, lo:hi], s=L.s[:, lo:hi], z=L.z[:, lo:hi], g=L.g, G=L.G)


def _row_block(L: OLayer, lo: int, hi: int) -> OLayer:
    return OLayer(q=L.q[lo:hi, :], s=L.s, z=L.z, g=L.g[lo:hi], G=L.G)


def _all_reduce_sum(parts):
    """AllReduce(op=SUM); summed in rank order 0,1,..,tp-1."""
    acc = parts[0].copy()
    for p in parts[1:]:
        acc = acc + p
    return acc


def _check_tp(N1: int, tp: int):
    if tp < 1 or N1 % tp:
        raise ValueError("N1 must be divisible by tp (CHUNK, PAPER.md:L119; reading c12)")


# ----------------------------------------------------------------------------- Alg. 2
def alg2_naive(X, L1: OLayer, L2: OLayer, tp: int):
    """Alg. 2 "Naive Algorithm", simulated over ranks r = 0..tp-1.

    Offline: P1, g1_opt = Reorder(g1); P2, g2_opt = Reorder(g2);
    weights are stored as W1[P1] and W2[P2] (Require), then W1 is
    split column-wise and W2 row-wise.
      L1: Y1_local = X1_global[:, P1] @ W1_local
      L2: Y1_global = AllGather(Y1_local)          (concatenate along dim 1, rank order; c17)
      L3: Y1_global = Y1_global[:, P2]
      L4: Y1_local = CHUNK(Y1_global, rank, size, dim=1)
      L5: Y2_local = Y1_local @ W2_local
      L6: Y2_global = AllReduce(Y2_local, op=SUM)
    Returns a dict with every intermediate, per rank.
    """
    X = np.asarray(X, dtype=np.float64)
    N1 = L1.N
    _check_tp(N1, tp)
    n = N1 // tp
    P1, _ = alg1_reorder(L1.g)
    P2, _ = alg1_reorder(L2.g)
    W1r = permute_rows(L1, P1)           # W1[P1]
    W2r = permute_rows(L2, P2)           # W2[P2]
    y1_local = []
    for r in range(tp):
        W1_local = _col_block(W1r, r * n, (r + 1) * n)
        y1_local.append(X[:, P1] @ dequantize(W1_local))                      # L1
    y1_global = np.concatenate(y1_local, axis=1)                               # L2
    y1_perm = y1_global[:, P2]                                                 # L3
    y2_local, y1_chunk = [], []
    for r in range(tp):
        y1c = y1_perm[:, r * n:(r + 1) * n]                                    # L4
        W2_local = _row_block(W2r, r * n, (r + 1) * n)
        y1_chunk.append(y1c)
        y2_local.append(y1c @ dequantize(W2_local))                            # L5
    Y2 = _all_reduce_sum(y2_local)                                             # L6
    return {"Y2": Y2, "Y1_local": y1_local, "Y1_global": y1_global, "Y1_chunk": y1_chunk,
            "Y2_local": y2_local, "P1": P1, "P2": P2}


# ----------------------------------------------------------------------------- Alg. 3
def alg3_tp_aware(X, L1: OLayer, L2: OLayer, tp: int):
    """Alg. 3 "TP-Aware Algorithm", simulated over ranks.

    Offline: W1 stored as W1[P1, P2] -- rows by P1 and, the paper's insight, columns
    by P2 (Require L137) -- and W2 as W2[P2]; W1 split column-wise,
    W2 row-wise.
      L1: Y1_local = X1_global[:, P1] @ W1_local
      L2: Y2_local = Y1_local @ W2_local           (no AllGather, no permute)
      L3: Y2_global = AllReduce(Y2_local, op=SUM)
    """
    X = np.asarray(X, dtype=np.float64)
    N1 = L1.N
    _check_tp(N1, tp)
    n = N1 // tp
    P1, _ = alg1_reorder(L1.g)
    P2, _ = alg1_reorder(L2.g)
    W1ra = permute_cols(permute_rows(L1, P1), P2)   # W1[P1, P2]
    W2r = permute_rows(L2, P2)                      # W2[P2]
    y1_local, y2_local = [], []
    for r in range(tp):
        W1_local = _col_block(W1ra, r * n, (r + 1) * n)
        W2_local = _row_block(W2r, r * n, (r + 1) * n)
        y1 = X[:, P1] @ dequantize(W1_local)                                   # L1
        y1_local.append(y1)
        y2_local.append(y1 @ dequantize(W2_local))                             # L2
    Y2 = _all_reduce_sum(y2_local)                                             # L3
    return {"Y2": Y2, "Y1_local": y1_local, "Y2_local": y2_local, "P1": P1, "P2": P2}


# ----------------------------------------------------------------------------- gate_proj (f2)
def silu(x):
    """SiLU(x) = x * sigmoid(x) = x / (1 + exp(-x)), the gate activation of the Llama MLP (reading
    c23: PAPER.md:L151 only says the method "can be generalized to the implementation in practice
    where a gate_proj layer is also present")."""
    x = np.asarray(x, dtype=np.float64)
    return x / (1.0 + np.exp(-x))


def gated_mlp(X, Wg, Wu, Wd):
    """Y1 = SiLU(X . Wg) * (X . Wu) (elementwise), Y2 = Y1 . Wd in fp64 (reading c23)."""
    X = np.asarray(X, dtype=np.float64)
    Y1 = silu(X @ Wg) * (X @ Wu)
    return Y1, Y1 @ Wd


def alg3_tp_aware_gated(X, Lg: OLayer, Lu: OLayer, Ld: OLayer, tp: int):
    """Alg. 3 generalized to a gate_proj layer (reading c24): P1g, P1u, P2 from
    Alg. 1 on each layer's own g_idx; Wg and Wu stored as Wg[P1g, P2] and Wu[P1u, P2] -- the SAME
    column permutation P2 on both, so their elementwise product lands in Wd[P2]'s row order
    (an elementwise op commutes with a common column permutation); Wd stored as Wd[P2].
      L1: Y1_local = SiLU(X[:, P1g] @ Wg_local) * (X[:, P1u] @ Wu_local)
      L2: Y2_local = Y1_local @ Wd_local
      L3: Y2_global = AllReduce(Y2_local, op=SUM)"""
    X = np.asarray(X, dtype=np.float64)
    N1 = Lg.N
    _check_tp(N1, tp)
    n = N1 // tp
    P1g, _ = alg1_reorder(Lg.g)
    P1u, _ = alg1_reorder(Lu.g)
    P2, _ = alg1_reorder(Ld.g)
    Wga = permute_cols(permute_rows(Lg, P1g), P2)
    Wua = permute_cols(permute_rows(Lu, P1u), P2)
    Wdr = permute_rows(Ld, P2)
    y1_local, y2_local = [], []
    for r in range(tp):
        g = X[:, P1g] @ dequantize(_col_block(Wga, r * n, (r + 1) * n))
        u = X[:, P1u] @ dequantize(_col_block(Wua, r * n, (r + 1) * n))
        y1 = silu(g) * u                                                       # L1
        y1_local.append(y1)
        y2_local.append(y1 @ dequantize(_row_block(Wdr, r * n, (r + 1) * n)))  # L2
    return {"Y2": _all_reduce_sum(y2_local), "Y1_local": y1_local, "Y2_local": y2_local,
            "P1g": P1g, "P1u": P1u, "P2": P2}


def alg2_naive_gated(X, Lg: OLayer, Lu: OLayer, Ld: OLayer, tp: int):
    """Alg. 2 with a gate_proj layer: Wg[P1g], Wu[P1u] column blocks (original
    column order), Y1_local = SiLU(gate) * up, then AllGather, Y1[:, P2], CHUNK, Wd[P2] rows."""
    X = np.asarray(X, dtype=np.float64)
    N1 = Lg.N
    _check_tp(N1, tp)
    n = N1 // tp
    P1g, _ = alg1_reorder(Lg.g)
    P1u, _ = alg1_reorder(Lu.g)
    P2, _ = alg1_reorder(Ld.g)
    Wgr, Wur, Wdr = permute_rows(Lg, P1g), permute_rows(Lu, P1u), permute_rows(Ld, P2)
    y1_local = []
    for r in range(tp):
        g = X[:, P1g] @ dequantize(_col_block(Wgr, r * n, (r + 1) * n))
        u = X[:, P1u] @ dequantize(_col_block(Wur, r * n, (r + 1) * n))
        y1_local.append(silu(g) * u)                                           # L1
    y1_perm = np.concatenate(y1_local, axis=1)[:, P2]                         # L2-L3
    y2_local = [y1_perm[:, r * n:(r + 1) * n] @ dequantize(_row_block(Wdr, r * n, (r + 1) * n))
                for r in range(tp)]                                            # L4-L5
    return {"Y2": _all_reduce_sum(y2_local), "Y1_local": y1_local, "Y2_local": y2_local}


# ----------------------------------------------------------------------------- shard maps
def shard_maps(P2, N1: int, tp: int, rank: int, variant: str, G2: int):
    """Index maps of rank `rank`'s shard.

    TP-aware (Alg. 3): W1 columns P2[r n:(r+1) n] (W1[P1,P2] column block r);
    naive (Alg. 2): W1 columns r n..(r+1) n (W1[P1] column block r).
    Both: W2 rows P2[r n:(r+1) n] (W2[P2] row block r), i.e. ordered groups
    [r n / G2, (r+1) n / G2) when n % G2 == 0 (reading c12).
    Naive AllGather source map: Y1in[:, i] = buf[c // n][:, c % n] with
    c = P2[r n + i] into the rank-ordered buffer buf[tp][M][n] (reading c17).
    """
    P2 = np.asarray(P2, dtype=np.int64)
    _check_tp(N1, tp)
    n = N1 // tp
    if variant == "tp_aware":
        w1_cols = P2[rank * n:(rank + 1) * n].copy()
    elif variant == "naive":
        w1_cols = np.arange(rank * n, (rank + 1) * n, dtype=np.int64)
    else:
        raise ValueError(variant)
    w2_rows = P2[rank * n:(rank + 1) * n].copy()
    c = P2[rank * n:(rank + 1) * n]
    src = np.stack([c // n, c % n], axis=1)
    return {"w1_cols": w1_cols, "w2_rows": w2_rows,
            "w2_group_lo": (rank * n) // G2, "w2_group_hi": -(-((rank + 1) * n) // G2),
            "gather_src": src}


def canonical_shard(L1: OLayer, L2: OLayer, tp: int, rank: int, variant: str):
    """Unpacked shard in canonical (reordered) row/column order, by plain indexing.

    W1 shard: rows P1, columns w1_cols (q, s, z) with ordered group index g1[P1];
    W2 shard: rows w2_rows with ordered group index g2[P2] restricted to the block.
    """
    P1, g1_opt = alg1_reorder(L1.g)
    P2, g2_opt = alg1_reorder(L2.g)
    mp = shard_maps(P2, L1.N, tp, rank, variant, L2.G)
    c = mp["w1_cols"]
    n = L1.N // tp
    lo, hi = mp["w2_group_lo"], mp["w2_group_hi"]
    return {
        "w1_q": L1.q[P1][:, c], "w1_s": L1.s[:, c], "w1_z": L1.z[:, c], "w1_g": g1_opt,
        "w2_q": L2.q[mp["w2_rows"], :], "w2_g": g2_opt[rank * n:(rank + 1) * n] - lo,
        "w2_s": L2.s[lo:hi], "w2_z": L2.z[lo:hi], "P1": P1, "P2": P2, **mp,
    }


# ----------------------------------------------------------------------------- tolerance
def check_rows_close(y_test, y_ref, rel: float = 1e-2):
    """Reading c14: per row m, max_n |y_test - y_ref| <= rel * max_n |y_ref|; a row whose
    reference is all-zero must be reproduced exactly.  Returns (ok, worst_ratio)."""
    y_test = np.asarray(y_test, dtype=np.float64)
    y_ref = np.asarray(y_ref, dtype=np.float64)
    assert y_test.shape == y_ref.shape, (y_test.shape, y_ref.shape)
    worst = 0.0
    ok = True
    for m in range(y_ref.shape[0]):
        err = np.max(np.abs(y_test[m] - y_ref[m])) if y_ref.shape[1] else 0.0
        norm = np.max(np.abs(y_ref[m])) if y_ref.shape[1] else 0.0
        if norm == 0.0:
            if err != 0.0:
                ok = False
                worst = max(worst, np.inf)
            continue
        ratio = err / norm
        worst = max(worst, ratio)
        if not (ratio <= rel):
            ok = False
    return ok, worst
