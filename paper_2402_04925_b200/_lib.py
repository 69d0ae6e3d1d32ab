"""Thin ctypes binding of include/tpq.h (argument marshalling only).

Every step of the hot path runs inside libtpq.so (sm_100a kernels + NCCL); this module only
converts numpy arrays / torch tensors into pointers.  There is no fallback: if the library
is missing, importing the binding raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# TPQ_LIB_PATH may point at the profiling build (libtpq_prof.so) for wait-cycle accounting.
LIB_PATH = os.environ.get("TPQ_LIB_PATH") or os.path.join(_PKG, "libtpq.so")

TPQ_OK, TPQ_EINVAL, TPQ_EUNSUPPORTED, TPQ_ECUDA, TPQ_ENCCL, TPQ_ENOMEM, TPQ_ESTATE = range(7)
TPQ_NAIVE, TPQ_TP_AWARE, TPQ_UNORDERED = 0, 1, 2
TPQ_STEP_GATHER, TPQ_STEP_LAYER1, TPQ_STEP_LAYER2, TPQ_STEP_ALLREDUCE = 0, 1, 2, 3
TPQ_STEP_NAIVE_GATHER, TPQ_STEP_ALLGATHER = 4, 5
_CODES = {1: "EINVAL", 2: "EUNSUPPORTED", 3: "ECUDA", 4: "ENCCL", 5: "ENOMEM", 6: "ESTATE"}

# Every symbol include/tpq.h declares (tests check the .so exports all of them).
EXPORTS = [
    "tpq_last_error", "tpq_version", "gptq_reorder", "tp_shard_mlp", "tp_shard_gated_mlp", "tpq_mlp_destroy",
    "tpq_comm_unique_id", "tpq_comm_create", "tpq_comm_destroy", "tpq_mlp_set_comm",
    "tp_mlp_forward", "tp_mlp_forward_host",
    "tp_mlp_forward_local", "tpq_layer1", "tpq_naive_gather", "tpq_layer2", "tpq_sum_partials",
    "tpq_mlp_info", "tpq_mlp_index_maps", "tpq_mlp_export_canonical", "tpq_mlp_run_step",
]


class TPQError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_CODES.get(code, code)}: {msg}")
        self.code = code


class GptqLayer(C.Structure):
    _fields_ = [("K", C.c_int64), ("N", C.c_int64), ("G", C.c_int32), ("bits", C.c_int32),
                ("qweight", C.c_void_p), ("scales", C.c_void_p), ("qzeros", C.c_void_p),
                ("g_idx", C.c_void_p)]


class MlpInfo(C.Structure):
    _fields_ = [("K1", C.c_int64), ("N1", C.c_int64), ("N2", C.c_int64), ("n", C.c_int64),
                ("M_max", C.c_int64), ("G1", C.c_int32), ("G2", C.c_int32), ("tp", C.c_int32),
                ("rank", C.c_int32), ("variant", C.c_int32), ("device", C.c_int32),
                ("w1_bytes", C.c_int64), ("w2_bytes", C.c_int64), ("units1", C.c_int64),
                ("units2", C.c_int64), ("grid1", C.c_int32), ("grid2", C.c_int32),
                ("has_comm", C.c_int32), ("split1", C.c_int32), ("split2", C.c_int32)]


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp, i64, i32 = C.c_void_p, C.c_int64, C.c_int32
        L.tpq_last_error.restype = C.c_char_p
        L.tpq_version.restype = C.c_int
        sig = {
            "gptq_reorder": [vp, i64, i32, vp, vp],
            "tp_shard_mlp": [C.POINTER(GptqLayer), C.POINTER(GptqLayer), vp, vp, C.c_int, C.c_int,
                             C.c_int, i64, C.c_int, C.POINTER(vp)],
            "tp_shard_gated_mlp": [C.POINTER(GptqLayer), C.POINTER(GptqLayer), C.POINTER(GptqLayer), vp, vp, vp,
                                   C.c_int, C.c_int, C.c_int, C.c_int64, C.c_int, C.POINTER(vp)],
            "tpq_mlp_destroy": [vp],
            "tpq_comm_unique_id": [vp],
            "tpq_comm_create": [vp, C.c_int, C.c_int, C.c_int, C.POINTER(vp)],
            "tpq_comm_destroy": [vp],
            "tpq_mlp_set_comm": [vp, vp],
            "tp_mlp_forward": [vp, vp, i64, vp, vp],
            "tp_mlp_forward_host": [vp, vp, i64, vp, vp],
            "tp_mlp_forward_local": [vp, vp, i64, vp, vp],
            "tpq_layer1": [vp, vp, i64, vp, vp],
            "tpq_naive_gather": [vp, vp, i64, vp, vp],
            "tpq_layer2": [vp, vp, i64, vp, vp],
            "tpq_sum_partials": [vp, C.c_int, i64, vp, vp],
            "tpq_mlp_info": [vp, C.POINTER(MlpInfo)],
            "tpq_mlp_index_maps": [vp, vp, vp, C.POINTER(i32), C.POINTER(i32)],
            "tpq_mlp_export_canonical": [vp, C.c_int, vp, vp, vp],
            "tpq_mlp_run_step": [vp, C.c_int, C.c_int64, vp],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        _lib = L
    return _lib


def _check(rc: int):
    if rc != TPQ_OK:
        raise TPQError(rc, lib().tpq_last_error().decode(errors="replace"))


def _ptr(a) -> int:
    """Pointer of a numpy array (host) or anything with data_ptr() (torch tensor, device)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    if isinstance(a, np.ndarray):
        assert a.flags["C_CONTIGUOUS"], "arrays must be C-contiguous"
        return a.ctypes.data
    return int(a)


def _stream(stream) -> int:
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except ImportError:
            pass
        return None
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


# ------------------------------------------------------------------------------ entry points
def gptq_reorder(g_idx, G: int):
    """Alg. 1 through the C-ABI: returns (P, g_idx_sorted) as int32 arrays."""
    g = np.ascontiguousarray(np.asarray(g_idx, dtype=np.int32))
    P = np.empty(g.shape[0], dtype=np.int32)
    gs = np.empty(g.shape[0], dtype=np.int32)
    _check(lib().gptq_reorder(_ptr(g), g.shape[0], int(G), _ptr(P), _ptr(gs)))
    return P, gs


def comm_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(lib().tpq_comm_unique_id(C.cast(buf, C.c_void_p)))
    return bytes(buf)


def sum_partials(parts, out, stream=None):
    arr = (C.c_void_p * len(parts))(*[_ptr(p) for p in parts])
    count = out.numel() if hasattr(out, "numel") else out.size
    _check(lib().tpq_sum_partials(C.cast(arr, C.c_void_p), len(parts), count, _ptr(out), _stream(stream)))


def _layer_struct(layer) -> tuple[GptqLayer, list]:
    """layer: object with K, N, G, qweight (u32 [K/8][N]), scales_bits (u16), qzeros (u32), g_idx."""
    keep = [np.ascontiguousarray(layer.qweight, dtype=np.uint32),
            np.ascontiguousarray(layer.scales_bits, dtype=np.uint16),
            np.ascontiguousarray(layer.qzeros, dtype=np.uint32),
            np.ascontiguousarray(layer.g_idx, dtype=np.int32)]
    s = GptqLayer(layer.K, layer.N, layer.G, 4, *[_ptr(k) for k in keep])
    return s, keep


class Comm:
    """NCCL communicator (tpq_comm_create); every rank constructs it with the same uid."""

    def __init__(self, uid: bytes, tp: int, rank: int, device: int):
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        c = C.c_void_p()
        _check(lib().tpq_comm_create(C.cast(buf, C.c_void_p), tp, rank, device, C.byref(c)))
        self._c = c

    def close(self):
        if getattr(self, "_c", None):
            _check(lib().tpq_comm_destroy(self._c))
            self._c = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class TpMlp:
    """One rank's shard (tp_shard_mlp handle)."""

    def __init__(self, w1, w2, P1, P2, tp: int = 1, rank: int = 0, variant: int = TPQ_TP_AWARE,
                 M_max: int = 16, device: int = 0):
        s1, k1 = _layer_struct(w1)
        s2, k2 = _layer_struct(w2)
        # TPQ_UNORDERED ignores the permutations (NULL pointers)
        P1 = None if P1 is None else np.ascontiguousarray(P1, dtype=np.int32)
        P2 = None if P2 is None else np.ascontiguousarray(P2, dtype=np.int32)
        h = C.c_void_p()
        _check(lib().tp_shard_mlp(C.byref(s1), C.byref(s2), _ptr(P1), _ptr(P2), tp, rank, variant,
                                  M_max, device, C.byref(h)))
        self._h = h
        self.info = MlpInfo()
        _check(lib().tpq_mlp_info(self._h, C.byref(self.info)))

    @classmethod
    def gated(cls, wg, wu, wd, P1g, P1u, P2, tp: int = 1, rank: int = 0, variant: int = TPQ_TP_AWARE,
              M_max: int = 16, device: int = 0) -> "TpMlp":
        """gate_proj variant (tp_shard_gated_mlp): Y = (SiLU(X.Wg) * (X.Wu)).Wd."""
        self = cls.__new__(cls)
        sg, kg = _layer_struct(wg)
        su, ku = _layer_struct(wu)
        sd, kd = _layer_struct(wd)
        Ps = [np.ascontiguousarray(P, dtype=np.int32) for P in (P1g, P1u, P2)]
        h = C.c_void_p()
        _check(lib().tp_shard_gated_mlp(C.byref(sg), C.byref(su), C.byref(sd), *[_ptr(P) for P in Ps], tp, rank,
                                        variant, M_max, device, C.byref(h)))
        self._h = h
        self.info = MlpInfo()
        _check(lib().tpq_mlp_info(self._h, C.byref(self.info)))
        return self

    def close(self):
        if getattr(self, "_h", None):
            lib().tpq_mlp_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # --- collectives
    def set_comm(self, comm: "Comm | None"):
        """Attach (not own) a communicator; keep `comm` alive while forwards are in flight."""
        self._comm = comm
        _check(lib().tpq_mlp_set_comm(self._h, comm._c if comm is not None else None))

    # --- forward (device pointers / torch tensors)
    def forward(self, X, M: int, Y, stream=None):
        _check(lib().tp_mlp_forward(self._h, _ptr(X), M, _ptr(Y), _stream(stream)))

    def forward_local(self, X, M: int, Y2, stream=None):
        _check(lib().tp_mlp_forward_local(self._h, _ptr(X), M, _ptr(Y2), _stream(stream)))

    def forward_host(self, X_host: np.ndarray, Y_host: np.ndarray, stream=None):
        assert X_host.dtype == np.float16 and Y_host.dtype == np.float16
        _check(lib().tp_mlp_forward_host(self._h, _ptr(X_host), X_host.shape[0], _ptr(Y_host),
                                         _stream(stream)))

    def layer1(self, X, M: int, Y1, stream=None):
        _check(lib().tpq_layer1(self._h, _ptr(X), M, _ptr(Y1), _stream(stream)))

    def naive_gather(self, buf, M: int, Y1in, stream=None):
        _check(lib().tpq_naive_gather(self._h, _ptr(buf), M, _ptr(Y1in), _stream(stream)))

    def layer2(self, Y1in, M: int, Y2, stream=None):
        _check(lib().tpq_layer2(self._h, _ptr(Y1in), M, _ptr(Y2), _stream(stream)))

    def run_step(self, step: int, M: int, stream=None):
        """Benchmarking: enqueue one step (TPQ_STEP_*) on the handle's own buffers."""
        _check(lib().tpq_mlp_run_step(self._h, int(step), M, _stream(stream)))

    # --- test exports
    def index_maps(self):
        n = self.info.n
        c = np.empty(n, np.int32)
        r = np.empty(n, np.int32)
        lo, hi = C.c_int32(), C.c_int32()
        _check(lib().tpq_mlp_index_maps(self._h, _ptr(c), _ptr(r), C.byref(lo), C.byref(hi)))
        return c, r, lo.value, hi.value

    def export_canonical(self, layer: int):
        i = self.info
        K, N, G = (i.K1, i.n, i.G1) if layer in (1, 3) else (i.n, i.N2, i.G2)  # 3: up layer of a gated shard
        q = np.empty((K, N), np.uint8)
        s = np.empty((K // G, N), np.uint16)
        z = np.empty((K // G, N), np.uint8)
        _check(lib().tpq_mlp_export_canonical(self._h, layer, _ptr(q), _ptr(s), _ptr(z)))
        return q, s, z
