"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no reorder, no permutation of
weights, no dequantisation, no GEMM).  It only draws random numbers and writes
them in the GPTQ checkpoint format the C-ABI consumes, so that the oracle
(`oracle/`) and the CUDA path (`paper_2402_04925_b200/`) see byte-identical
inputs.  Recipe:

* ``SeedSequence(seed).spawn(9)`` in the fixed order
  [phi1, phi2, q1, q2, z1, z2, s1, s2, X].
* phi_l: uniform random permutation of range(K_l)   -- PAPER.md:L25-29 (Eq. 2,
  "we use a random permutation function phi to emulate an arbitrary reordering").
* g_idx_l[i] = phi_l[i] // G                         -- the act_order checkpoint
  field the paper consumes, PAPER.md:L32-34 (Eq. 3).  Computed here only to
  *synthesise* the checkpoint; the oracle re-derives it independently (eq3) and a
  test asserts the two agree.
* q ~ U{0..15} i.i.d. per (row, col); z ~ U{0..15} per (group, col).
* s = fp16(U[0.5, 1.5] / (6.52 * sqrt(K_l))) per (group, col): 6.52 ~ sqrt(42.5)
  is the rms of (q - z), so std(Y1) ~ std(Y2) ~ 1 and fp16 never overflows.
* X = fp16(N(0, 1)), shape [M][K1].
* wide_scales=True (precision tests only): s = fp16(2^-2 * 10^-(1.5 u + 4 v)), u ~ U[0, 1) per
  (group, col) and v ~ U[0, 1) per column: 5.5 decades across the layer (whole columns up to 4
  decades below the largest), 1.5 within a column.

GPTQ packing (reading c4): ``qweight[K/8][N]`` uint32 with row k's
nibble at bits 4*(k%8) of word k//8; ``qzeros[ceil(K/G)][N/8]`` uint32 with
column n's nibble at bits 4*(n%8); ``scales`` are fp16 bit patterns
``[ceil(K/G)][N]`` (uint16).  Zeros are stored as-is (no GPTQ-v1 "-1").
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

SHAPES = {
    # name: (K1, N1, N2, G)  -- BASELINE.json configs; N2 = K1 (reading c18)
    "tiny": (256, 512, 256, 32),
    "llama70b": (8192, 28672, 8192, 128),
    "granite20b": (6144, 24576, 6144, 128),
}


@dataclass
class Layer:
    """One GPTQ act_order layer in checkpoint (on-disk) form, row order untouched."""

    K: int
    N: int
    G: int
    phi: np.ndarray          # int64 [K]    the random permutation (Eq. 2)
    g_idx: np.ndarray        # int32 [K]    Eq. 3 group index (unordered)
    q: np.ndarray            # uint8 [K][N] unpacked int4 codes
    z: np.ndarray            # uint8 [ceil(K/G)][N]
    scales_f16: np.ndarray   # float16 [ceil(K/G)][N]
    qweight: np.ndarray = field(default=None)  # uint32 [K/8][N]
    qzeros: np.ndarray = field(default=None)   # uint32 [ceil(K/G)][N/8]

    @property
    def scales_bits(self) -> np.ndarray:
        return self.scales_f16.view(np.uint16)

    @property
    def n_groups(self) -> int:
        return -(-self.K // self.G)


def pack_rows_u4(q: np.ndarray) -> np.ndarray:
    """[K][N] uint8 codes -> [K/8][N] uint32, row k in bits 4*(k%8) (GPTQ qweight)."""
    K, N = q.shape
    assert K % 8 == 0
    q = q.astype(np.uint32).reshape(K // 8, 8, N)
    out = np.zeros((K // 8, N), dtype=np.uint32)
    for j in range(8):
        out |= q[:, j, :] << np.uint32(4 * j)
    return out


def pack_cols_u4(z: np.ndarray) -> np.ndarray:
    """[R][N] uint8 codes -> [R][N/8] uint32, column n in bits 4*(n%8) (GPTQ qzeros)."""
    R, N = z.shape
    assert N % 8 == 0
    z = z.astype(np.uint32).reshape(R, N // 8, 8)
    out = np.zeros((R, N // 8), dtype=np.uint32)
    for j in range(8):
        out |= z[:, :, j] << np.uint32(4 * j)
    return out


def make_layer(K: int, N: int, G: int, ss_phi, ss_q, ss_z, ss_s, *, identity_phi=False,
               integer_regime=False, wide_scales=False) -> Layer:
    rng_phi = np.random.Generator(np.random.PCG64(ss_phi))
    phi = np.arange(K, dtype=np.int64) if identity_phi else rng_phi.permutation(K).astype(np.int64)
    g_idx = (phi // G).astype(np.int32)
    ng = -(-K // G)
    q = np.random.Generator(np.random.PCG64(ss_q)).integers(0, 16, size=(K, N), dtype=np.uint8)
    z = np.random.Generator(np.random.PCG64(ss_z)).integers(0, 16, size=(ng, N), dtype=np.uint8)
    rng_s = np.random.Generator(np.random.PCG64(ss_s))
    if integer_regime:
        # power-of-two scales 2^-e, e in {0..3}: every product and partial sum is
        # an exactly representable dyadic rational.
        e = rng_s.integers(0, 4, size=(ng, N))
        s = np.ldexp(1.0, -e).astype(np.float16)
    elif wide_scales:
        u = rng_s.uniform(0.0, 1.0, size=(ng, N))
        v = rng_s.uniform(0.0, 1.0, size=(1, N))
        s = (0.25 * 10.0 ** -(1.5 * u + 4.0 * v)).astype(np.float16)
    else:
        s = (rng_s.uniform(0.5, 1.5, size=(ng, N)) / (6.52 * np.sqrt(K))).astype(np.float16)
    lay = Layer(K=K, N=N, G=G, phi=phi, g_idx=g_idx, q=q, z=z, scales_f16=s)
    if K % 8 == 0:
        lay.qweight = pack_rows_u4(q)
    if N % 8 == 0:
        lay.qzeros = pack_cols_u4(z)
    return lay


@dataclass
class Problem:
    K1: int
    N1: int
    N2: int
    G: int
    M: int
    seed: int
    w1: Layer
    w2: Layer
    X: np.ndarray  # float16 [M][K1]


def make_problem(K1: int, N1: int, N2: int, G: int, M: int, seed: int = 0, *,
                 G2: int | None = None, identity_phi=False, integer_regime=False, wide_scales=False) -> Problem:
    """Build the seeded synthetic MLP problem Y = (X.W1).W2 (PAPER.md:L151 shapes)."""
    G2 = G if G2 is None else G2
    ss = np.random.SeedSequence(seed).spawn(9)
    w1 = make_layer(K1, N1, G, ss[0], ss[2], ss[4], ss[6], identity_phi=identity_phi,
                    integer_regime=integer_regime, wide_scales=wide_scales)
    w2 = make_layer(N1, N2, G2, ss[1], ss[3], ss[5], ss[7], identity_phi=identity_phi,
                    integer_regime=integer_regime, wide_scales=wide_scales)
    rng_x = np.random.Generator(np.random.PCG64(ss[8]))
    if integer_regime:
        X = rng_x.integers(-2, 3, size=(M, K1)).astype(np.float16)
    else:
        X = rng_x.standard_normal(size=(M, K1)).astype(np.float16)
    return Problem(K1=K1, N1=N1, N2=N2, G=G, M=M, seed=seed, w1=w1, w2=w2, X=X)


def make_named(name: str, M: int, seed: int = 0) -> Problem:
    K1, N1, N2, G = SHAPES[name]
    return make_problem(K1, N1, N2, G, M, seed)


def onehot_x(M: int, K1: int, ks) -> np.ndarray:
    """X = rows of the identity (one-hot probes, SURVEY.md §4 tier 3)."""
    X = np.zeros((M, K1), dtype=np.float16)
    for m, k in enumerate(ks):
        X[m, k] = 1.0
    return X
