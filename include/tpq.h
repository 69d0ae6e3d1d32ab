/*
 * tpq.h -- C-ABI of the B200-native TP-aware GPTQ MLP hot path
 *          (arxiv 2402.04925, "TP-Aware Dequantization").
 *
 * Library: paper_2402_04925_b200/libtpq.so (sm_100a CUDA + C++ host code, NCCL 2.28).
 * Citations: PAPER.md:L<a>-<b> = /root/reference/PAPER.md lines (LaTeX of the paper);
 *            reading cN = the DESIGN.md ambiguity ledger entry N (same numbering as
 *            SURVEY.md section 8(c)).
 *
 * Conventions (all entry points):
 *  - Every function returns an int status: TPQ_OK (0) or one of the TPQ_E* codes.
 *    No C++ exception and no abort crosses this boundary.  tpq_last_error() returns a
 *    thread-local, NUL-terminated message describing the last failure on the calling
 *    thread (valid until that thread's next call into the library).
 *  - Sizes are int64_t element counts unless stated otherwise.
 *  - "host" pointers are ordinary CPU memory; "dev" pointers are CUDA device pointers on
 *    the handle's device.  The caller owns every pointer it passes; the library copies
 *    what it keeps and never frees caller memory.
 *  - Streams are passed as `void*` holding a cudaStream_t (NULL = legacy default stream).
 *  - fp16 values are IEEE binary16 bit patterns (uint16_t on the host).
 */
#ifndef TPQ_H_
#define TPQ_H_

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TPQ_OK 0
#define TPQ_EINVAL 1        /* bad shape / divisibility / permutation / g_idx / variant / rank */
#define TPQ_EUNSUPPORTED 2  /* valid for the paper but not implemented here (bits != 4, G not in
                               {32,64,128}, ragged last group, M > M_max, ...) */
#define TPQ_ECUDA 3         /* a CUDA runtime call failed (message carries cudaGetErrorString) */
#define TPQ_ENCCL 4         /* an NCCL call failed */
#define TPQ_ENOMEM 5        /* host or device allocation failed */
#define TPQ_ESTATE 6        /* call not valid in the handle's state (e.g. forward on a host-only
                               handle, tp > 1 forward without tpq_comm_init) */

#define TPQ_NAIVE 0         /* Alg. 2: W1[P1] + AllGather + Y1[:,P2] + CHUNK */
#define TPQ_TP_AWARE 1      /* Alg. 3: W1[P1,P2], no AllGather               */
#define TPQ_UNORDERED 2     /* locality baseline (Fig. 1): no reorder, per-row g_idx */

const char* tpq_last_error(void);
int tpq_version(void); /* returns (major << 16) | minor; never fails */

/* ---------------------------------------------------------------------------------------
 * gptq_reorder -- Alg. 1 "Reorder Function", PAPER.md:L44-54 (offline).
 *   P <- ARGSORT(g_idx); g_idx_optimized <- g_idx[P].
 * ARGSORT is the STABLE argsort: ties are broken by ascending original index (reading c6).
 *   g_idx            host int32[K], the act_order group index of Eq. 3.
 *   K, G             rows and group size; K >= 1, G >= 1.
 *   perm_out         host int32[K], receives P.
 *   g_idx_sorted_out host int32[K] or NULL, receives g_idx[P] (always floor(i/G): the
 *                    multiset of Eq. 3 equals that of Eq. 1).
 * Errors: TPQ_EINVAL if K < 1, G < 1, a pointer is NULL, any g outside [0, ceil(K/G)), or a
 * group's multiplicity differs from min(G, K - g*G) (g_idx is not an Eq.-3 array).
 * Pure host function: thread-safe, deterministic, no device access.
 * ------------------------------------------------------------------------------------- */
int gptq_reorder(const int32_t* g_idx, int64_t K, int32_t G, int32_t* perm_out,
                 int32_t* g_idx_sorted_out);

/* One GPTQ act_order layer as stored on disk (stored "without ... the
 * ordering"), K x N, rows in original (unordered) order.  Host arrays, read-only; the
 * library copies what it needs during tp_shard_mlp.  Packing = reading c4:
 *   qweight  uint32[K/8][N]            row k's code in bits 4*(k%8) of word k/8
 *   scales   uint16[ceil(K/G)][N]      fp16 bit patterns
 *   qzeros   uint32[ceil(K/G)][N/8]    column n's zero in bits 4*(n%8), stored as-is (c3:
 *                                      dequant = s * (q - z), no GPTQ-v1 "-1")
 *   g_idx    int32[K]                  Eq. 3 group index                              */
typedef struct gptq_layer {
  int64_t K, N;
  int32_t G, bits; /* bits must be 4 */
  const uint32_t* qweight;
  const uint16_t* scales;
  const uint32_t* qzeros;
  const int32_t* g_idx;
} gptq_layer;

typedef struct tpq_mlp tpq_mlp; /* opaque: one rank's shard of the two-layer MLP */

/* ---------------------------------------------------------------------------------------
 * tp_shard_mlp -- offline TP-aware transform + shard + pack (PAPER.md:L75 offline,
 * L102 column-/row-TP split, L127-129 + Alg. 3 Require L137 "W1[P1, P2], W2[P2]").
 *   w1, w2    layers of Y = (X.W1).W2 (PAPER.md:L151 up_proj then down_proj); w1->N == w2->K.
 *   P1, P2    host int32[K1], int32[N1]: Alg. 1 permutations of w1->g_idx, w2->g_idx
 *             (from gptq_reorder).  Validated: permutation AND g_idx[P[i]] == i / G.
 *   tp, rank  tensor-parallel degree in {1,2,4,8}, this rank in [0, tp).
 *   variant   TPQ_TP_AWARE: rank keeps W1[P1,P2] columns [r*n, (r+1)*n) (= original
 *             columns P2[r*n..]) and W2[P2] rows [r*n, (r+1)*n);  TPQ_NAIVE: rank keeps W1[P1]
 *             columns [r*n, (r+1)*n) and the same W2 rows.  n = N1 / tp.
 *             TPQ_UNORDERED: the locality baseline of SURVEY.md §8(f) f3 -- NO reordering: rows
 *             stay in checkpoint order with their Eq.-3 g_idx and the kernel looks each row's
 *             group metadata up (the Fig. 1 formulation).  tp must be 1
 *             (TPQ_EINVAL), M_max <= 16 and K/G <= 256 per layer (TPQ_EUNSUPPORTED); P1 and P2
 *             are ignored (may be NULL); g_idx values must lie in [0, K/G).
 *   M_max     largest batch (rows of X) later passed to the forward; 1 <= M_max <= 512.
 *   device    CUDA device ordinal that will own the shard, or -1 for a HOST-ONLY handle
 *             (packing + index maps + export only; no CUDA call is made; forward = ESTATE).
 *   out       receives the handle (NULL on failure).
 * Requirements (TPQ_EINVAL): bits == 4; K1 % 8 == 0, N1 % 8 == 0, N2 % 8 == 0 (GPTQ packing);
 *   N1 % tp == 0; n % 128 == 0 and N2 % 128 == 0 (128-column device tiles); n % G2 == 0 so each
 *   W2 shard owns whole groups (reading c12); K1 % G1 == 0 and K1 % 128 == 0 (else
 *   TPQ_EUNSUPPORTED, c13; 128-row device k-blocks); G1, G2 in {32, 64, 128} (else
 *   TPQ_EUNSUPPORTED).
 * The library owns the device shard (packed int4 + metadata in its private tile x k-block
 * layout), P1 and the workspace for M_max.  Not thread-safe per
 * handle; distinct handles are independent.
 * ------------------------------------------------------------------------------------- */
int tp_shard_mlp(const gptq_layer* w1, const gptq_layer* w2, const int32_t* P1,
                 const int32_t* P2, int tp, int rank, int variant, int64_t M_max, int device,
                 tpq_mlp** out);

/* tp_shard_gated_mlp -- the gate_proj variant ("can be
 * generalized to the implementation in practice where a gate_proj layer is also present"):
 * Y = (SiLU(X.Wg) * (X.Wu)).Wd, the Llama MLP (readings c23-c25).
 *   wg, wu    gate and up layers, K1 x N1 each with their own act_order g_idx and equal G;
 *   wd        down layer, N1 x N2;  P1g, P1u, P2 = Alg. 1 permutations of wg, wu, wd g_idx.
 * TPQ_TP_AWARE: the rank keeps Wg[P1g, P2] and Wu[P1u, P2] columns [r n, (r+1) n) -- the SAME
 * column permutation P2 on both, so SiLU(gate) * up lands in Wd[P2]'s row order with no exchange
 * (the elementwise product commutes with a common column permutation) -- and Wd[P2] rows
 * [r n, (r+1) n); TPQ_NAIVE: Wg[P1g], Wu[P1u] column blocks, AllGather + P2 gather before Wd.
 * The forward entry points are those of tp_shard_mlp; layer 1 is one GEMV over interleaved gate/up
 * records whose epilogue writes fp16(SiLU(gate) * up) from fp32 accumulators.  Same requirements
 * and errors as tp_shard_mlp, plus: wu matching wg in K, N and G (TPQ_EINVAL); M_max <= 16
 * (TPQ_EUNSUPPORTED: no tensor-core A7 path for the gated layer); TPQ_UNORDERED is rejected.
 * tpq_mlp_export_canonical: layer 1 = gate, 3 = up, 2 = down. */
int tp_shard_gated_mlp(const gptq_layer* wg, const gptq_layer* wu, const gptq_layer* wd, const int32_t* P1g,
                       const int32_t* P1u, const int32_t* P2, int tp, int rank, int variant, int64_t M_max,
                       int device, tpq_mlp** out);
int tpq_mlp_destroy(tpq_mlp* h); /* NULL is a no-op; frees device memory and the NCCL comm */

/* ---------------------------------------------------------------------------------------
 * NCCL communicator for tp > 1 (the collectives of PAPER.md:L117 AllGather / L121, L142
 * AllReduce run over NVLink 5 / NVSwitch).  Rank 0 calls tpq_comm_unique_id, the caller ships
 * the 128 bytes to every rank (e.g. a torch.distributed broadcast), then every rank calls
 * tpq_comm_create (collective, blocking) for its device.  One communicator serves any number
 * of MLP handles (a model's layers): tpq_mlp_set_comm attaches it WITHOUT taking ownership;
 * the comm must outlive every forward enqueued with it and be destroyed by its creator.
 * Errors: TPQ_EINVAL (NULL, tp/rank mismatch with the handle), TPQ_ENCCL, TPQ_ECUDA.
 * ------------------------------------------------------------------------------------- */
typedef struct tpq_comm tpq_comm;
int tpq_comm_unique_id(uint8_t out[128]);
int tpq_comm_create(const uint8_t id[128], int tp, int rank, int device, tpq_comm** out);
int tpq_comm_destroy(tpq_comm* c); /* NULL is a no-op */
int tpq_mlp_set_comm(tpq_mlp* h, tpq_comm* c); /* c may be NULL to detach */

/* ---------------------------------------------------------------------------------------
 * tp_mlp_forward -- the hot path, one rank.  TPQ_TP_AWARE = Alg. 3:
 *   Y1_local = X[:, P1] @ W1_local; Y2_local = Y1_local @ W2_local; Y = AllReduce(Y2_local).
 * TPQ_NAIVE = Alg. 2: adds AllGather(Y1_local), Y1[:, P2] and CHUNK
 * (fused into one gather kernel feeding layer 2, reading c16).
 *   X  dev fp16 [M][K1] row-major, identical on every rank (reading c19).
 *   M  1 <= M <= M_max.
 *   Y  dev fp16 [M][N2] row-major, caller-owned; identical on every rank on completion.
 * Arithmetic (reading c22): the shard stores each column n's scales as
 * s' = s * 2^E_n (E_n >= 0, exact, the column's largest scale in [2^14, 2^16)); the tensor-core
 * A operand is the fp16 dequantized weight -- passes of M <= 16 rows, and of 17..32 rows on the
 * plain TP-aware / naive MLP (the same GEMV with N = 32): fp16(q s' 2^-24 + fp16(-z s' 2^-24)), one
 * HFMA2 per pair, i.e. s (q - z) with at most two fp16 roundings, normal while the group's scale
 * is >= ~2^-5 of the column's largest; other passes (the A7 tensor-core GEMMs): fp16((q - z) s' 2^-12),
 * one rounding of the exact (q - z) -- times fp16 activations, accumulated in fp32 over whole tile segments (the ordered
 * groups make the records self-contained), times 2^(24 - E_n) resp. 2^(12 - E_n)
 * in the epilogue (exact); Y1 rounded to fp16 (RN) between the layers (reading c10), fp16
 * AllReduce (c11).  Tiles split between CTAs are summed in a fixed order (bit-identical repeats).
 * Collective when tp > 1: every rank must call it with the same M (NCCL semantics; a
 * mismatch is a documented precondition violation -> hang, not a status).  Asynchronous on
 * `stream`, no allocation, no host synchronisation, CUDA-graph capturable.
 * Errors: TPQ_ESTATE (host-only handle, tp > 1 without comm), TPQ_EINVAL (NULL, M out of
 * range), TPQ_ECUDA / TPQ_ENCCL (launch / collective enqueue failure).
 * ------------------------------------------------------------------------------------- */
int tp_mlp_forward(tpq_mlp* h, const void* X, int64_t M, void* Y, void* stream);

/* End-to-end variant with HOST buffers (the call a CPU-side user makes): copies X
 * (host fp16 [M][K1], pinned or pageable) to the handle's device staging buffer, runs
 * tp_mlp_forward, copies Y back to host fp16 [M][N2] and synchronises `stream`. */
int tp_mlp_forward_host(tpq_mlp* h, const uint16_t* X_host, int64_t M, uint16_t* Y_host,
                        void* stream);

/* Rank-local forward without any collective: Y2_local (dev fp16 [M][N2]) of this rank.
 * For tp == 1 it equals tp_mlp_forward.  Used for independent replicas and to run every
 * rank's shard on one GPU (tests / per-rank kernel timing). */
int tp_mlp_forward_local(tpq_mlp* h, const void* X, int64_t M, void* Y2_local, void* stream);

/* The algorithm's lines as separate steps (row-major fp16 interfaces, for step parity):
 *   tpq_layer1:       Y1_local (dev fp16 [M][n]) = X[:, P1] @ W1_local      (Alg. 2/3 L1)
 *   tpq_naive_gather: Y1in (dev fp16 [M][n]) = CHUNK(AllGather-buffer[:, P2], rank) where
 *                     buf is dev fp16 [tp][M][n] (NCCL AllGather layout, reading c17)
 *                     (Alg. 2 L3-4; EINVAL for a TP_AWARE handle)
 *   tpq_layer2:       Y2_local (dev fp16 [M][N2]) = Y1in @ W2_local          (Alg. 2 L5 / Alg. 3 L2) */
int tpq_layer1(tpq_mlp* h, const void* X, int64_t M, void* Y1_local, void* stream);
int tpq_naive_gather(tpq_mlp* h, const void* buf, int64_t M, void* Y1in, void* stream);
int tpq_layer2(tpq_mlp* h, const void* Y1in, int64_t M, void* Y2_local, void* stream);

/* Deterministic elementwise sum of nparts dev fp16 arrays of `count` elements, in part order,
 * accumulated in fp32 and rounded once (rank-order sum for single-GPU shard simulation).
 * `parts` is a HOST array of nparts dev pointers. */
int tpq_sum_partials(const void* const* parts, int nparts, int64_t count, void* out,
                     void* stream);

/* Benchmarking export: enqueue ONE step of the M <= 16 TP-aware forward on the handle's own
 * device buffers (contents are whatever the buffers hold; no result is defined), so that each
 * step's kernels can be timed alone, e.g. as a CUDA graph of many launches (bench.py):
 *   TPQ_STEP_GATHER    (0)  X[:, P1] gather (Alg. 3 L1 operand) from the host-forward staging buffer
 *   TPQ_STEP_LAYER1    (1)  layer-1 dequant-GEMV + its split-tile fix-up      (Alg. 3 L1)
 *   TPQ_STEP_LAYER2    (2)  layer-2 dequant-GEMV + its split-tile fix-up      (Alg. 3 L2)
 *   TPQ_STEP_ALLREDUCE (3)  ncclAllReduce of the [M][N2] output (tp > 1 with a comm; Alg. 3 L3)
 *   TPQ_STEP_NAIVE_GATHER (4)  TPQ_NAIVE handles: Y1[:, P2] + CHUNK from the AllGather buffer
 *                              (Alg. 2 L3-4) into layer 2's input
 *   TPQ_STEP_ALLGATHER (5)  TPQ_NAIVE handles with a comm: ncclAllGather of Y1_local (Alg. 2 L2)
 * TPQ_EINVAL for an unknown step, a naive step on another variant or M outside one pass, [1, min(P, M_max)]
 * with P = 16 for handles with M_max <= 16, else 256 (the A7 pass);
 * TPQ_ESTATE for a host-only handle or a collective step without a comm. */
#define TPQ_STEP_GATHER 0
#define TPQ_STEP_LAYER1 1
#define TPQ_STEP_LAYER2 2
#define TPQ_STEP_ALLREDUCE 3
#define TPQ_STEP_NAIVE_GATHER 4
#define TPQ_STEP_ALLGATHER 5
int tpq_mlp_run_step(tpq_mlp* h, int step, int64_t M, void* stream);


/* ------------------------------- introspection / test-only exports ------------------- */
typedef struct tpq_mlp_info_t {
  int64_t K1, N1, N2, n, M_max;
  int32_t G1, G2, tp, rank, variant, device;
  int64_t w1_bytes, w2_bytes;       /* packed device bytes of each layer shard (int4 + meta) */
  int64_t units1, units2;           /* (128-column tile x 128-row k-block) units per layer */
  int32_t grid1, grid2;             /* CTAs launched per layer by the M <= 16 GEMV        */
  int32_t has_comm;
  /* how the M <= 16 GEMV finishes tiles split between CTAs, per layer: 0 = stream-K with the
   * split tiles summed inside the kernel (per-tile release counters), 1 = stream-K with the
   * fix-up kernel after it, c >= 2 = cluster split-K, one tile per cluster of c CTAs reduced
   * through distributed shared memory.  All sum the partials in a fixed order (bit-identical
   * repeats). */
  int32_t split1, split2;
} tpq_mlp_info_t;
int tpq_mlp_info(const tpq_mlp* h, tpq_mlp_info_t* out);

/* Index maps of the shard (bit-exact targets of the oracle's shard_maps):
 *   w1_cols host int32[n]: original W1 column held at local column j;
 *   w2_rows host int32[n]: original W2 row held at local row i (= P2[r*n + i]);
 *   w2_group_lo/hi: this shard's ordered W2 groups [lo, hi). */
int tpq_mlp_index_maps(const tpq_mlp* h, int32_t* w1_cols, int32_t* w2_rows,
                       int32_t* w2_group_lo, int32_t* w2_group_hi);

/* Decode the packed shard of `layer` (1 or 2) back to canonical (reordered) order, from the
 * library's own packed bytes: q uint8[K][N], s uint16[K/G][N], z uint8[K/G][N] (host),
 * where (K, N) = (K1, n) for layer 1 and (n, N2) for layer 2. */
int tpq_mlp_export_canonical(const tpq_mlp* h, int layer, uint8_t* q, uint16_t* s, uint8_t* z);

#ifdef __cplusplus
}
#endif
#endif /* TPQ_H_ */
