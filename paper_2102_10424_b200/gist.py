"""Thin ctypes binding of include/gist.h (argument marshalling only).

Every computation happens inside libgist.so (hand-written sm_100a kernels).
There is no CPU fallback: if the library or a B200 is missing, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgist.so")

GIST_ARCH_GCN, GIST_ARCH_SAGE, GIST_ARCH_GAT = 0, 1, 2
ARCHS = {"gcn": GIST_ARCH_GCN, "sage": GIST_ARCH_SAGE, "gat": GIST_ARCH_GAT}
GIST_OPT_SGD, GIST_OPT_ADAM = 0, 1
GIST_PREC_FP32, GIST_PREC_BF16, GIST_PREC_TF32 = 0, 1, 2
GIST_GRAPH_DEVICE = 0
TRACE_NODES, TRACE_ACT, TRACE_LOGITS, TRACE_GRAD, TRACE_LOSS = range(5)
(STAT_ROUND, STAT_STEP, STAT_SELF_LOOPS_DROPPED, STAT_LAST_NNZ_B, STAT_LAST_NB, STAT_KERNELS,
 STAT_H2D_BYTES, STAT_D2H_BYTES, STAT_MAX_NB, STAT_BLOCK_AGG, STAT_BLOCK_DENSITY_PPM, STAT_THETA_BYTES) = range(12)

# every symbol include/gist.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "gist_config_default", "gist_create", "gist_load_graph", "gist_init_params", "gist_partition",
    "gist_subtrain", "gist_aggregate", "gist_eval", "gist_eval_parts", "gist_get_params", "gist_set_params",
    "gist_get_partition", "gist_sub_shape", "gist_get_sub_params", "gist_get_trace", "gist_stat",
    "gist_stream", "gist_last_error", "gist_status_str", "gist_destroy", "gist_spmm", "gist_gemm",
    "gist_profile", "gist_profile_get", "gist_nccl_unique_id", "gist_slot_owner", "gist_slots_per_rank",
    "gist_eval_logits", "gist_loopback_create", "gist_loopback_destroy", "gist_gemm_reps",
    "gist_save_checkpoint", "gist_load_checkpoint",
]
PROF_CLASSES = ["batch", "spmm", "gemm", "loss", "optim", "partition", "aggregate", "agg_tc", "comm"]


GIST_OPT_STATE_RESET, GIST_OPT_STATE_PERSISTENT = 0, 1
GIST_AGG_ALLGATHER, GIST_AGG_P2P, GIST_AGG_SYMM = 0, 1, 2


class GistConfig(C.Structure):
    _fields_ = [
        ("arch", C.c_int32), ("num_layers", C.c_int32), ("dims", C.POINTER(C.c_int32)),
        ("optimizer", C.c_int32), ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float),
        ("precision", C.c_int32), ("clusters_per_batch", C.c_int32), ("batch_seed", C.c_uint64),
        ("graph_residency", C.c_int32), ("rank", C.c_int32), ("world_size", C.c_int32),
        ("device", C.c_int32), ("nccl_unique_id", C.c_void_p), ("stream", C.c_void_p),
        ("opt_state", C.c_int32), ("agg_mode", C.c_int32), ("loopback", C.c_void_p), ("eval_scale", C.c_int32),
        ("theta_mode", C.c_int32),
    ]


_lib = None


def lib() -> C.CDLL:
    """Loads libgist.so; raises if it was not built (no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build() (no CPU fallback exists)")
    L = C.CDLL(LIB_PATH)
    i32, i64, u64, vp, f32 = C.c_int32, C.c_int64, C.c_uint64, C.c_void_p, C.c_float
    P = C.POINTER
    sig = {
        "gist_config_default": (None, [P(GistConfig)]),
        "gist_create": (i32, [P(GistConfig), P(vp)]),
        "gist_load_graph": (i32, [vp, i64, vp, vp, i64, vp, vp, i32, vp, vp, i32]),
        "gist_init_params": (i32, [vp, u64]),
        "gist_partition": (i32, [vp, u64, i32]),
        "gist_subtrain": (i32, [vp, i32, f32, vp]),
        "gist_aggregate": (i32, [vp]),
        "gist_eval": (i32, [vp, i32, P(f32), P(f32)]),
        "gist_eval_parts": (i32, [vp, i32, vp, i32, i64, P(f32), P(f32), vp, vp]),
        "gist_get_params": (i32, [vp, i32, vp]),
        "gist_set_params": (i32, [vp, i32, vp]),
        "gist_get_partition": (i32, [vp, i32, vp, vp]),
        "gist_sub_shape": (i32, [vp, i32, i32, P(i64), P(i64)]),
        "gist_get_sub_params": (i32, [vp, i32, i32, vp]),
        "gist_get_trace": (i32, [vp, i32, i32, i32, vp, P(i64)]),
        "gist_stat": (i64, [vp, i32]),
        "gist_stream": (vp, [vp]),
        "gist_last_error": (C.c_char_p, [vp]),
        "gist_status_str": (C.c_char_p, [i32]),
        "gist_destroy": (None, [vp]),
        "gist_spmm": (i32, [vp, vp, i64, vp, vp, i32, vp, vp, i64, i64, i32, vp]),
        "gist_gemm": (i32, [i32, i32, i64, i64, i64, vp, i64, vp, i64, vp, i64, i32, i32, i32, vp]),
        "gist_gemm_reps": (i32, [i32, i32, i64, i64, i64, vp, i64, vp, i64, vp, i64, i32, i32, i32, vp, i32]),
        "gist_profile": (i32, [vp, i32]),
        "gist_nccl_unique_id": (i32, [vp]),
        "gist_slot_owner": (i32, [i32, i32]),
        "gist_slots_per_rank": (i32, [i32, i32]),
        "gist_profile_get": (i32, [vp, i32, P(C.c_double), P(i64), P(C.c_double)]),
        "gist_eval_logits": (i32, [vp, i32, vp, i32, i64, vp]),
        "gist_loopback_create": (i32, [i32, P(vp)]),
        "gist_loopback_destroy": (None, [vp]),
        "gist_save_checkpoint": (i32, [vp, C.c_char_p]),
        "gist_load_checkpoint": (i32, [vp, C.c_char_p]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


class GistError(RuntimeError):
    pass


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class Gist:
    """One GIST context (one GPU).  Method names mirror the C ABI."""

    def __init__(self, arch: str, dims, optimizer: str = "adam", precision: str = "fp32",
                 clusters_per_batch: int = 1, batch_seed: int = 0, rank: int = 0, world_size: int = 1,
                 device: int = 0, nccl_unique_id: bytes | None = None, stream: int | None = None,
                 beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8, opt_state: str = "reset",
                 agg_mode: str = "allgather", loopback: "Loopback | None" = None, eval_scale: str = "none",
                 theta: str = "replicated"):
        L = lib()
        self.arch = arch
        self.dims = [int(d) for d in dims]
        self._dims = (C.c_int32 * len(self.dims))(*self.dims)
        cfg = GistConfig()
        L.gist_config_default(C.byref(cfg))
        cfg.arch = ARCHS[arch]
        cfg.num_layers = len(self.dims) - 1
        cfg.dims = self._dims
        cfg.optimizer = GIST_OPT_ADAM if optimizer == "adam" else GIST_OPT_SGD
        cfg.beta1, cfg.beta2, cfg.eps = beta1, beta2, eps
        cfg.precision = {"fp32": GIST_PREC_FP32, "bf16": GIST_PREC_BF16, "tf32": GIST_PREC_TF32}[precision]
        cfg.clusters_per_batch = clusters_per_batch
        cfg.batch_seed = batch_seed
        cfg.rank, cfg.world_size, cfg.device = rank, world_size, device
        self._uid = None
        if nccl_unique_id is not None:
            self._uid = C.create_string_buffer(bytes(nccl_unique_id), 128)
            cfg.nccl_unique_id = C.cast(self._uid, C.c_void_p)
        cfg.stream = stream
        cfg.opt_state = {"reset": GIST_OPT_STATE_RESET, "persistent": GIST_OPT_STATE_PERSISTENT}[opt_state]
        cfg.agg_mode = {"allgather": GIST_AGG_ALLGATHER, "p2p": GIST_AGG_P2P, "symm": GIST_AGG_SYMM}[agg_mode]
        cfg.eval_scale = {"none": 0, "mean": 1}[eval_scale]
        cfg.theta_mode = {"replicated": 0, "sharded": 1}[theta]
        self._lb = loopback  # keeps the group alive while this context exists
        cfg.loopback = loopback.h if loopback is not None else None
        self._cfg = cfg
        h = C.c_void_p()
        self._check(L.gist_create(C.byref(cfg), C.byref(h)), None)
        self.h = h
        self.L = cfg.num_layers

    def _check(self, st: int, h=...):
        if st != 0:
            L = lib()
            msg = L.gist_last_error(self.h if h is ... else h).decode() if (h is ... and self.h) else ""
            raise GistError(f"{L.gist_status_str(st).decode()} ({st}): {msg}")

    def close(self):
        if getattr(self, "h", None):
            lib().gist_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- ABI calls ----
    def load_graph(self, g: dict):
        rp = np.ascontiguousarray(g["row_ptr"], dtype=np.int64)
        ci = np.ascontiguousarray(g["col_idx"], dtype=np.int32)
        X = np.ascontiguousarray(g["X"], dtype=np.float32)
        lab = np.ascontiguousarray(g["labels"], dtype=np.int32)
        sp = np.ascontiguousarray(g["split"], dtype=np.uint8)
        cl = np.ascontiguousarray(g["cluster_ids"], dtype=np.int32)
        n = len(rp) - 1
        self._check(lib().gist_load_graph(self.h, n, _ptr(rp), _ptr(ci), int(rp[-1]), _ptr(X), _ptr(lab),
                                          int(g["num_classes"]), _ptr(sp), _ptr(cl), int(g["num_clusters"])))
        self.num_clusters = int(g["num_clusters"])
        self.num_nodes = n

    def init_params(self, seed: int):
        self._check(lib().gist_init_params(self.h, seed))

    def partition(self, seed: int, m: int):
        self._check(lib().gist_partition(self.h, seed, m))
        self.m = m

    def subtrain(self, local_iters: int, lr: float, want_loss: bool = True):
        out = np.zeros(self.m, dtype=np.float32) if want_loss else None
        self._check(lib().gist_subtrain(self.h, local_iters, lr, _ptr(out) if out is not None else None))
        return out

    def aggregate(self):
        self._check(lib().gist_aggregate(self.h))

    def eval(self, split_code: int):
        loss, acc = C.c_float(), C.c_float()
        self._check(lib().gist_eval(self.h, split_code, C.byref(loss), C.byref(acc)))
        return loss.value, acc.value

    def eval_parts(self, split_code: int, part_ids=None, num_parts: int = 0, max_rows: int = 0):
        """Partition-wise evaluation (gist_eval_parts); part_ids indexed by original node id,
        None = the training clusters.  Returns (loss, acc, per-partition loss, per-partition acc)."""
        if part_ids is not None:
            part_ids = np.ascontiguousarray(part_ids, dtype=np.int32)
            npart = int(num_parts)
        else:
            npart = int(self.num_clusters)
        loss, acc = C.c_float(), C.c_float()
        lp = np.zeros(npart, dtype=np.float32)
        ap = np.zeros(npart, dtype=np.float32)
        self._check(lib().gist_eval_parts(self.h, split_code, _ptr(part_ids) if part_ids is not None else None,
                                          num_parts if part_ids is not None else 0, max_rows,
                                          C.byref(loss), C.byref(acc), _ptr(lp), _ptr(ap)))
        return loss.value, acc.value, lp, ap

    def eval_logits(self, mode: int = 0, part_ids=None, num_parts: int = 0, max_rows: int = 0) -> np.ndarray:
        """Per-node logits [n x d_L] (original node ids) of the forward gist_eval (mode 0) or
        gist_eval_parts (mode 1) runs."""
        n = self.num_nodes
        out = np.zeros((n, self.dims[-1]), dtype=np.float32)
        if part_ids is not None:
            part_ids = np.ascontiguousarray(part_ids, dtype=np.int32)
        self._check(lib().gist_eval_logits(self.h, mode, _ptr(part_ids) if part_ids is not None else None,
                                           int(num_parts) if part_ids is not None else 0, max_rows, _ptr(out)))
        return out

    def save_checkpoint(self, path: str):
        self._check(lib().gist_save_checkpoint(self.h, os.fsencode(path)))

    def load_checkpoint(self, path: str):
        self._check(lib().gist_load_checkpoint(self.h, os.fsencode(path)))

    def param_shape(self, layer: int):
        d = self.dims[layer]
        rows = 2 * d if self.arch == "sage" else (d + 2 if self.arch == "gat" else d)
        return rows, self.dims[layer + 1]

    def get_params(self, layer: int) -> np.ndarray:
        out = np.zeros(self.param_shape(layer), dtype=np.float32)
        self._check(lib().gist_get_params(self.h, layer, _ptr(out)))
        return out

    def set_params(self, layer: int, w: np.ndarray):
        w = np.ascontiguousarray(w, dtype=np.float32)
        assert w.shape == self.param_shape(layer)
        self._check(lib().gist_set_params(self.h, layer, _ptr(w)))

    def get_partition(self, dim: int):
        units = np.zeros(self.dims[dim], dtype=np.int32)
        offs = np.zeros(self.m + 1, dtype=np.int32)
        self._check(lib().gist_get_partition(self.h, dim, _ptr(units), _ptr(offs)))
        return [units[offs[i]:offs[i + 1]] for i in range(self.m)] if 0 < dim < self.L else \
            [units.copy() for _ in range(self.m)]

    def sub_shape(self, slot: int, layer: int):
        r, c = C.c_int64(), C.c_int64()
        self._check(lib().gist_sub_shape(self.h, slot, layer, C.byref(r), C.byref(c)))
        return r.value, c.value

    def get_sub_params(self, slot: int, layer: int) -> np.ndarray:
        out = np.zeros(self.sub_shape(slot, layer), dtype=np.float32)
        self._check(lib().gist_get_sub_params(self.h, slot, layer, _ptr(out)))
        return out

    def trace(self, slot: int, what: int, layer: int = 0):
        cnt = C.c_int64()
        self._check(lib().gist_get_trace(self.h, slot, what, layer, None, C.byref(cnt)))
        dt = np.int32 if what == TRACE_NODES else np.float32
        out = np.zeros(cnt.value, dtype=dt)
        self._check(lib().gist_get_trace(self.h, slot, what, layer, _ptr(out), C.byref(cnt)))
        return out

    def stat(self, which: int) -> int:
        return int(lib().gist_stat(self.h, which))

    def stream(self) -> int:
        return lib().gist_stream(self.h)

    def profile(self, stride: int):
        self._check(lib().gist_profile(self.h, stride))

    def profile_get(self) -> dict:
        out = {}
        for k, name in enumerate(PROF_CLASSES):
            ms, n, w = C.c_double(), C.c_int64(), C.c_double()
            self._check(lib().gist_profile_get(self.h, k, C.byref(ms), C.byref(n), C.byref(w)))
            out[name] = {"ms": ms.value, "launches": n.value, "work": w.value}
        return out


class Loopback:
    """Loopback transport group (gist_loopback_create): `world` contexts of this process, each
    driven by its own thread, stand in for `world` ranks on one GPU (tests of the W > 1 paths)."""

    def __init__(self, world: int):
        h = C.c_void_p()
        st = lib().gist_loopback_create(world, C.byref(h))
        if st != 0:
            raise GistError(f"gist_loopback_create: {lib().gist_status_str(st).decode()}")
        self.h = h
        self.world = world

    def close(self):
        if getattr(self, "h", None):
            lib().gist_loopback_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def slot_owner(slot: int, world: int) -> int:
    """Rank owning sub-GCN slot `slot` (host-only, from the library)."""
    return int(lib().gist_slot_owner(slot, world))


def slots_per_rank(m: int, world: int) -> int:
    return int(lib().gist_slots_per_rank(m, world))


def local_slots(m: int, world: int, rank: int) -> list:
    return [i for i in range(m) if slot_owner(i, world) == rank]


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    st = lib().gist_nccl_unique_id(buf)
    if st != 0:
        raise GistError(f"gist_nccl_unique_id: {lib().gist_status_str(st).decode()}")
    return buf.raw


def spmm(row_ptr_dev: int, col_dev: int, rows: int, rowscale_dev: int | None, colscale_dev: int | None,
         self_loop: bool, H_dev: int, out_dev: int, w: int, ld: int, dtype: int, stream: int | None = None):
    st = lib().gist_spmm(row_ptr_dev, col_dev, rows, rowscale_dev, colscale_dev, int(self_loop), H_dev, out_dev,
                         w, ld, dtype, stream)
    if st != 0:
        raise GistError(f"gist_spmm: {lib().gist_status_str(st).decode()}")


def gemm(transA: bool, transB: bool, M: int, N: int, K: int, A_dev: int, lda: int, B_dev: int, ldb: int,
         C_dev: int, ldc: int, dtype: int, out_f32: bool = True, relu: bool = False, stream: int | None = None,
         reps: int = 1):
    st = lib().gist_gemm_reps(int(transA), int(transB), M, N, K, A_dev, lda, B_dev, ldb, C_dev, ldc, dtype,
                              int(out_f32), int(relu), stream, reps)
    if st != 0:
        raise GistError(f"gist_gemm: {lib().gist_status_str(st).decode()}")
