"""ctypes binding of libgraphblast_sm100a.so (the C ABI in include/graphblast.h).

This module is the only place the product talks to native code.  There is no
CPU fallback: if the library or a CUDA device is missing, every compute entry
point raises ``RuntimeError`` immediately.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .errors import FormatError, ShapeError

_HERE = os.path.dirname(os.path.abspath(__file__))
# GB_LIB: load another build of the library (A/B of compile-time variants)
LIB_PATH = os.environ.get("GB_LIB") or os.path.join(_HERE, "libgraphblast_sm100a.so")

# gb_status codes (graphblast.h)
GB_OK = 0
GB_ERR_SHAPE = -1
GB_ERR_FORMAT = -2
GB_ERR_INDEX = -3
GB_ERR_VALUE = -4
GB_ERR_UNSUPPORTED = -5
GB_ERR_CUDA = -6
GB_ERR_OOM = -7
GB_ERR_ARG = -8

GB_I64 = 0
GB_F64 = 1
GB_I32 = 2

# operator ids
OP_PLUS, OP_PLUS_WRAP, OP_MINUS, OP_TIMES, OP_MIN, OP_MAX, OP_LOR, OP_LAND, OP_LESS, OP_NE, \
    OP_SECOND, OP_FIRST = range(12)
# folds whose result does not depend on the order (gb_mv.cu fold_is_commutative)
COMMUTATIVE_FOLD_IDS = (OP_PLUS, OP_PLUS_WRAP, OP_TIMES, OP_MIN, OP_MAX, OP_LOR, OP_LAND)

DIR_AUTO, DIR_PUSH, DIR_PULL = 0, 1, 2
PART_NONZERO, PART_ROW = 0, 1

vp = C.c_void_p
i32 = C.c_int32
i64 = C.c_int64
u64 = C.c_uint64
f64 = C.c_double
pi64 = C.POINTER(C.c_int64)
pi32 = C.POINTER(C.c_int32)
pf64 = C.POINTER(C.c_double)


# gb_abi_version() of the library these bindings describe (include/graphblast.h)
ABI_VERSION = 2


class gb_csr(C.Structure):
    _fields_ = [
        ("nrows", i64), ("ncols", i64), ("nnz", i64),
        ("offsets", vp), ("indices", vp), ("values", vp),
        ("dtype", i32), ("pad_", i32), ("iso_i64", i64), ("iso_f64", f64), ("gen", C.c_uint64),
    ]


class gb_row_plan(C.Structure):
    _fields_ = [("nrows_nz", i64), ("nz_rows", vp), ("nz_off", vp), ("tile_first", vp)]


class gb_bin_plan(C.Structure):
    _fields_ = [("n_short", i64), ("n_mid", i64), ("n_long_tiles", i64), ("short_rows", vp),
                ("mid_rows", vp), ("tile_row", vp), ("tile_beg", vp), ("tile_end", vp)]


# name -> (restype, argtypes)
SIGNATURES = {
    "gb_abi_version": (i32, []),
    "gb_ctx_create": (i32, [C.c_int, C.POINTER(vp)]),
    "gb_ctx_destroy": (i32, [vp]),
    "gb_ctx_set_stream": (i32, [vp, vp]),
    "gb_ctx_sync": (i32, [vp]),
    "gb_last_error": (C.c_char_p, [vp]),
    "gb_scratch_bytes": (i64, [vp]),
    "gb_ctx_trim": (i32, [vp]),
    "gb_event_create": (i32, [C.POINTER(vp)]),
    "gb_event_record": (i32, [vp, vp]),
    "gb_event_sync": (i32, [vp]),
    "gb_event_destroy": (i32, [vp]),
    "gb_iota": (i32, [vp, i32, i64, vp]),
    "gb_cast": (i32, [vp, i64, i32, vp, i32, vp]),
    "gb_select_flags": (i32, [vp, i64, vp, vp, vp, i32, vp, vp, pi64]),
    "gb_gather_i32": (i32, [vp, i32, i64, vp, vp, vp]),
    "gb_edges_clean": (i32, [vp, i64, vp, vp, vp, i32, vp, vp, vp, pi64]),
    "gb_scale_rows": (i32, [vp, i64, vp, f64, vp]),
    "gb_lower_by_rank": (i32, [vp, C.POINTER(gb_csr), vp, vp, vp, pi64]),
    "gb_launch_count": (i64, [vp]),
    "gb_ctx_set_profiling": (i32, [vp, i32]),
    "gb_prof_read": (i32, [vp, i32, vp, vp, vp]),
    "gb_build_csr": (i32, [vp, i64, i64, i64, vp, vp, vp, i32, i32, vp, vp, vp, pi64]),
    "gb_transpose_csr": (i32, [vp, C.POINTER(gb_csr), vp, vp, vp]),
    "gb_csr_equal": (i32, [vp, C.POINTER(gb_csr), C.POINTER(gb_csr), pi32]),
    "gb_values_iso": (i32, [vp, i64, vp, i32, pi32]),
    "gb_values_minmax": (i32, [vp, i64, vp, i32, pf64, pf64]),
    "gb_rmat_generate": (i32, [vp, i32, i64, u64, f64, f64, f64, vp, vp]),
    "gb_edges_to_csr": (i32, [vp, i64, i64, vp, vp, i32, vp, vp, pi64]),
    "gb_assign_weights": (i32, [vp, i64, i64, vp, vp, u64, i64, i64, vp]),
    "gb_csr_row_ids": (i32, [vp, i64, i64, vp, vp]),
    "gb_count_ne": (i32, [vp, i64, vp, i32, vp, pi64]),
    "gb_compact": (i32, [vp, i64, i64, vp, vp, i32, vp, vp, vp, pi64]),
    "gb_scatter_dense": (i32, [vp, i64, i64, vp, vp, i32, vp, vp]),
    "gb_mask_bitmap": (i32, [vp, i64, i64, vp, vp, i32, i32, vp]),
    "gb_nonempty_rows": (i32, [vp, i64, vp, vp]),
    "gb_decide_direction": (i32, [i64, i64, i64, f64, i32, pi64]),
    "gb_bfs": (i32, [vp, C.POINTER(gb_csr), C.POINTER(gb_csr), vp, i64, i64, f64, i32, vp,
                     vp, vp, vp, pi64]),
    "gb_bfs_ordered": (i32, [vp, C.POINTER(gb_csr), C.POINTER(gb_csr), vp, vp, i64, i64, f64, i32,
                             vp, vp, vp, vp, pi64]),
    "gb_bfs_ordered_async": (i32, [vp, C.POINTER(gb_csr), C.POINTER(gb_csr), vp, vp, i64, i64,
                                   f64, i32, vp, vp, vp, vp]),
    "gb_count_launches": (None, [vp, i64]),
    "gb_bfs_parents": (i32, [vp, C.POINTER(gb_csr), vp, i64, vp]),
    "gb_bfs_counters": (i32, [vp, C.POINTER(gb_csr), C.POINTER(gb_csr), vp, i64, vp, i32, vp]),
    "gb_sssp_certify": (i32, [vp, C.POINTER(gb_csr), i64, vp, vp]),
    "gb_cc_certify": (i32, [vp, C.POINTER(gb_csr), vp, vp]),
    "gb_bfs_validate": (i32, [vp, C.POINTER(gb_csr), C.POINTER(gb_csr), i64, vp, vp, vp]),
    "gb_bfs_engine": (i32, [i32]),
    "gb_loop_engine": (i32, [i32]),
    "gb_bfs_coop_max_n": (i64, [i64]),
    "gb_degree_order": (i32, [vp, i64, vp, vp, vp]),
    "gb_csr_relabel_t": (i32, [vp, C.POINTER(gb_csr), vp, vp, vp, vp, vp]),
    "gb_mxv_pull": (i32, [vp, i32, i32, C.POINTER(gb_csr), C.POINTER(gb_row_plan), vp, vp, i32,
                          i32, vp, vp]),
    "gb_row_plan_build": (i32, [vp, C.POINTER(gb_csr), vp, vp, vp, pi64]),
    "gb_mxv_pull_ordered": (i32, [vp, i32, i32, C.POINTER(gb_csr), C.POINTER(gb_row_plan), vp,
                                  i64, vp, vp, vp, vp]),
    "gb_row_plan_remap": (i32, [vp, i64, vp, vp, vp]),
    "gb_bin_plan_counts": (i32, [vp, C.POINTER(gb_csr), vp]),
    "gb_bin_plan_fill": (i32, [vp, C.POINTER(gb_csr), C.POINTER(gb_bin_plan)]),
    "gb_mxv_pull_binned": (i32, [vp, i32, i32, C.POINTER(gb_csr), C.POINTER(gb_bin_plan), vp, vp,
                                 vp, vp]),
    "gb_mxv_pull_striped": (i32, [vp, i32, i32, i32, vp, vp, vp, vp, vp, vp]),
    "gb_index_max": (i32, [vp, i64, vp, pi64]),
    "gb_probe_rate": (i32, [vp, i64, i64, C.POINTER(f64)]),
    "gb_gather_replay_rate": (i32, [vp, C.POINTER(gb_csr), vp, C.POINTER(f64)]),
    "gb_mxv_push": (i32, [vp, i32, i32, C.POINTER(gb_csr), i64, i64, vp, vp, vp, vp, vp, pi64,
                          vp]),
    "gb_mxm_masked": (i32, [vp, i32, i32, C.POINTER(gb_csr), C.POINTER(gb_csr),
                            C.POINTER(gb_csr), vp, vp, vp, pi64, vp]),
    "gb_has_diagonal": (i32, [vp, C.POINTER(gb_csr), pi32]),
    "gb_ewise_dense": (i32, [vp, i32, i32, i64, vp, vp, vp, i32, vp, vp, vp]),
    "gb_union_sparse": (i32, [vp, i32, i32, i64, vp, vp, i64, vp, vp, vp, vp, pi64]),
    "gb_intersect_sparse": (i32, [vp, i32, i32, i64, vp, vp, i64, vp, vp, vp, vp, vp, pi64]),
    "gb_gather_pair": (i32, [vp, i32, i32, i64, vp, vp, vp, i32, vp]),
    "gb_filter_mask": (i32, [vp, i32, i64, vp, vp, vp, vp, vp, pi64]),
    "gb_assign_scalar": (i32, [vp, i32, i64, vp, vp, vp]),
    "gb_check_bounds": (i32, [vp, i64, vp, i64, pi32]),
    "gb_scatter_min": (i32, [vp, i32, i64, vp, i64, vp, vp, vp]),
    "gb_gather": (i32, [vp, i32, i64, vp, i64, vp, vp]),
    "gb_gather_sparse": (i32, [vp, i32, i64, vp, i64, i64, vp, vp, vp, vp]),
    "gb_apply_affine": (i32, [vp, i32, i64, vp, vp, vp, vp]),
    "gb_reduce": (i32, [vp, i32, i32, i64, vp, vp, vp, pi64]),
    "gb_reduce_rows": (i32, [vp, i32, C.POINTER(gb_csr), vp]),
    "gb_sssp": (i32, [vp, C.POINTER(gb_csr), C.POINTER(gb_csr), i64, i64, f64, i32, f64, vp, vp,
                      vp, vp, pi64, "ITER_CB", vp]),
    "gb_pagerank": (i32, [vp, C.POINTER(gb_csr), vp, f64, f64, i64, f64, i32, vp, vp, vp, vp,
                          vp, pi64]),
    "gb_cc": (i32, [vp, C.POINTER(gb_csr), C.POINTER(gb_csr), i64, f64, i32, i32, vp, vp, vp,
                    vp, pi64]),
    "gb_tc": (i32, [vp, C.POINTER(gb_csr), pi64]),
    "gb_bitmap_count": (i32, [vp, i64, vp, pi64]),
    "gb_bfs_dist_init": (i32, [vp, i64, i64, vp, vp, vp, vp, vp]),
    "gb_bfs_dist_push": (i32, [vp, C.POINTER(gb_csr), i64, vp, vp]),
    "gb_bfs_dist_collect": (i32, [vp, i64, i64, i64, vp, vp, vp]),
    "gb_bfs_dist_pull": (i32, [vp, C.POINTER(gb_csr), i64, i64, vp, i64, i64, vp, vp, vp, vp, vp]),
    "gb_bfs_dist_apply": (i32, [vp, i64, i64, vp, vp, vp, vp, vp, vp, pi64]),
    "gb_bfs_dist_unstamp": (i32, [vp, i64, vp, vp]),
    "gb_bfs_dist_owned": (i32, [vp, i64, i64, vp, vp, vp]),
    "gb_bfs_dist_pack_words": (i32, [vp, i64, i64, i64, vp, vp]),
    "gb_bfs_dist_unpack_words": (i32, [vp, i32, i64, vp, vp, vp]),
    "gb_bfs_dist_set_ids": (i32, [vp, i64, i32, i64, vp, vp, vp]),
    "gb_bfs_dist_dev_init": (i32, [vp, vp, vp, i64, i64, i64, i64, f64, i32, vp, vp, vp, vp, vp]),
    "gb_bfs_dist_dev_level": (i32, [vp, vp, vp, C.POINTER(gb_csr), C.POINTER(gb_csr), i64, i64, vp,
                                    i64, vp, vp, vp, vp, vp, vp, i32]),
    "gb_bfs_dist_dev_apply": (i32, [vp, vp, i64, vp, vp, vp, vp, vp, vp]),
    "gb_csr_column_block": (i32, [vp, C.POINTER(gb_csr), i64, i64, vp, vp, pi64]),
    "gb_cc_dist_init": (i32, [vp, i64, vp, vp, vp, vp]),
    "gb_cc_dist_hook": (i32, [vp, i32, C.POINTER(gb_csr), C.POINTER(gb_csr), i64, i64, i64, vp,
                              vp, vp, vp]),
    "gb_cc_dist_propose": (i32, [vp, i64, i64, i64, vp, vp, vp, vp]),
    "gb_cc_dist_shortcut": (i32, [vp, i64, vp, vp, vp, vp, vp, i32, pi64, pi64]),
    "gb_widen_i32": (i32, [vp, i64, vp, vp]),
}

ITER_CB = C.CFUNCTYPE(None, C.c_int64, C.c_void_p)

_lib = None
_lib_err = None
_lock = threading.Lock()


def load(path: str = LIB_PATH):
    """Load the shared library and bind every declared symbol (no GPU needed)."""
    global _lib, _lib_err
    with _lock:
        if _lib is not None:
            return _lib
        try:
            lib = C.CDLL(path)
        except OSError as exc:
            _lib_err = f"cannot load {path}: {exc}"
            raise RuntimeError(_lib_err + " (run __graft_entry__.build())") from None
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = [ITER_CB if a == "ITER_CB" else a for a in args]
        got = lib.gb_abi_version()
        if got != ABI_VERSION:
            _lib_err = f"{path} has ABI {got}, this package binds ABI {ABI_VERSION}"
            raise RuntimeError(_lib_err + " (rebuild with __graft_entry__.build())")
        _lib = lib
        return lib


class GraphBlastError(RuntimeError):
    pass


def _raise(status, ctx_ptr, what):
    msg = ""
    if _lib is not None and ctx_ptr:
        raw = _lib.gb_last_error(ctx_ptr)
        msg = raw.decode(errors="replace") if raw else ""
    text = f"{what}: {msg}" if msg else what
    if status == GB_ERR_SHAPE:
        raise ShapeError(text)
    if status == GB_ERR_FORMAT:
        raise FormatError(text)
    if status == GB_ERR_INDEX:
        raise IndexError(text)
    if status == GB_ERR_VALUE:
        raise ValueError(text)
    if status == GB_ERR_UNSUPPORTED:
        raise NotImplementedError(text)
    raise GraphBlastError(f"{text} (status {status})")


class Context:
    """A gb_ctx bound to one CUDA device; follows torch's current stream."""

    def __init__(self, device_index: int):
        lib = load()
        self.device_index = device_index
        ptr = vp()
        st = lib.gb_ctx_create(device_index, C.byref(ptr))
        if st != GB_OK:
            raise GraphBlastError(f"gb_ctx_create({device_index}) failed with status {st}")
        self.ptr = ptr
        self.lib = lib
        self._stream = None
        self._trim_hooks = []

    def launches(self) -> int:
        return int(self.lib.gb_launch_count(self.ptr))

    def profiling(self, on: bool):
        self.lib.gb_ctx_set_profiling(self.ptr, 1 if on else 0)

    def prof_read(self, cap=4096):
        kind = np.zeros(cap, np.int32)
        arg = np.zeros(cap, np.int64)
        ms = np.zeros(cap, np.float32)
        k = self.lib.gb_prof_read(self.ptr, cap, kind.ctypes.data_as(vp), arg.ctypes.data_as(vp),
                                  ms.ctypes.data_as(vp))
        return [(int(kind[i]), int(arg[i]), float(ms[i])) for i in range(k)]

    def on_trim(self, fn):
        """Run fn() before the scratch pool is released (Python-side caches)."""
        self._trim_hooks.append(fn)

    def trim(self):
        for fn in self._trim_hooks:
            fn()
        self.lib.gb_ctx_trim(self.ptr)

    def call(self, name, *args):
        s = _raw_stream(self.device_index)
        if s != self._stream:
            self.lib.gb_ctx_set_stream(self.ptr, vp(s))
            self._stream = s
        st = getattr(self.lib, name)(self.ptr, *args)
        if st != GB_OK:
            _raise(st, self.ptr, name)
        return st


def _raw_stream(device_index):
    """cudaStream_t of torch's current stream on the device (the raw getter
    skips building a Stream object: ~10 us per call on the host)."""
    import torch
    get = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if get is not None:
        return get(device_index)
    return torch.cuda.current_stream(device_index).cuda_stream


class DeviceEvent:
    """A cudaEvent recorded on the context's stream through the library (no
    torch Stream object per record); sync() waits for it."""

    __slots__ = ("lib", "ev")

    def __init__(self, ctx):
        self.lib = ctx.lib
        self.ev = vp()
        st = self.lib.gb_event_create(C.byref(self.ev))
        if st != GB_OK:
            raise RuntimeError("gb_event_create failed")

    def record(self, ctx):
        ctx.call("gb_event_record", self.ev)

    def sync(self):
        self.lib.gb_event_sync(self.ev)

    def __del__(self):
        try:
            if self.ev:
                self.lib.gb_event_destroy(self.ev)
        except Exception:
            pass


_contexts = {}


_CUDA_OK = False


def require_cuda():
    global _CUDA_OK
    if _CUDA_OK:
        return
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_1908_01407_b200 needs a CUDA device (B200, sm_100a); there is no CPU fallback")
    _CUDA_OK = True


def context(device=None) -> Context:
    import torch
    require_cuda()
    idx = torch.cuda.current_device() if device is None else torch.device(device).index
    if idx is None:
        idx = torch.cuda.current_device()
    ctx = _contexts.get(idx)
    if ctx is None:
        with torch.cuda.device(idx):
            ctx = Context(idx)
        _contexts[idx] = ctx
    return ctx


def ptr(t):
    """Device address of a tensor (or None)."""
    return None if t is None else vp(t.data_ptr())


def dtype_code(np_dtype) -> int:
    k = np.dtype(np_dtype)
    if k == np.int64:
        return GB_I64
    if k == np.float64:
        return GB_F64
    raise NotImplementedError(f"device kernels compute in int64 or float64, not {k}")


def scalar_buf(value, np_dtype):
    """8-byte host buffer holding `value` in the given dtype (for zero_host args)."""
    arr = np.asarray([value], dtype=np_dtype)
    buf = C.create_string_buffer(arr.tobytes(), 8)
    return buf
