"""B200-native TP-aware GPTQ MLP hot path (arxiv 2402.04925).

The product is libtpq.so (C-ABI in include/tpq.h); this package is its thin binding.
"""
from ._lib import (  # noqa: F401
    Comm, EXPORTS, LIB_PATH, TPQ_NAIVE, TPQ_STEP_ALLREDUCE, TPQ_STEP_GATHER, TPQ_STEP_LAYER1, TPQ_STEP_LAYER2, TPQ_STEP_NAIVE_GATHER, TPQ_STEP_ALLGATHER, TPQ_TP_AWARE, TPQ_UNORDERED, TPQError, TpMlp, comm_unique_id, gptq_reorder, lib,
    sum_partials,
)
