"""ctypes binding of libsparsekit_b200.so (the C ABI in include/sparsekit_b200.h).

There is no CPU fallback: importing a compute entry point without the built
library or without a CUDA device raises immediately.
"""

from __future__ import annotations

import ctypes
import os
import sys
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SKB_LIB_PATH: another build of the same library (same-box A/B of kernel variants)
LIB_PATH = os.environ.get("SKB_LIB_PATH") or os.path.join(_HERE, "libsparsekit_b200.so")

SKB_OK, SKB_E_VALUE, SKB_E_INDEX, SKB_E_KEY, SKB_E_CUDA, SKB_E_NOMEM, SKB_E_ARG, SKB_E_UNSUPPORTED = range(8)
SKB_E_IO = 8

_i64, _u64, _i32, _p = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int32, ctypes.c_void_p


class AdamScalars(ctypes.Structure):
    """skb_adam_t (host-computed float32 scalars, optim.py:69-75)."""
    _fields_ = [("lr", ctypes.c_float), ("beta1", ctypes.c_float), ("beta2", ctypes.c_float),
                ("eps", ctypes.c_float), ("one_minus_beta1", ctypes.c_float),
                ("one_minus_beta2", ctypes.c_float), ("bc1", ctypes.c_float), ("bc2", ctypes.c_float),
                ("lr_wd", ctypes.c_float), ("decoupled_decay", ctypes.c_int32)]


# name -> argtypes (restype int unless noted)
_SIGS = {
    "skb_version": ([], ctypes.c_char_p),
    "skb_last_error": ([], ctypes.c_char_p),
    "skb_last_error_arg": ([], _i64),
    "skb_device_sm_count": ([ctypes.c_int, ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "skb_launch_count": ([], _i64),
    "skb_memcpy_async": ([_p, _p, _i64, _p], ctypes.c_int),
    "skb_mix64": ([_p, _i64, _p, _p], ctypes.c_int),
    "skb_shard_of": ([_p, _i64, _i64, _p, _p], ctypes.c_int),
    "skb_keys_for": ([_p, _i64, _u64, _p, _p], ctypes.c_int),
    "skb_fnv1a64_host": ([ctypes.c_char_p, _i64], _u64),
    "skb_fnv1a64_strings": ([_p, _p, _i64, _p, _p], ctypes.c_int),
    "skb_fnv1a64_pairs": ([_p, _p, _i64, _p, _p], ctypes.c_int),
    "skb_unique_partition": ([_p, _i64, _i64, _p, _p, _p, _p, _p], ctypes.c_int),
    "skb_shard_unique_counts": ([_p, _i64, _i64, _p, _p], ctypes.c_int),
    "skb_partition_restore": ([_p, _i64, _p, _p, _p, _i64, _p, _p], ctypes.c_int),
    "skb_table_create": ([_i64, _i64, _i64, _i64, _i64, ctypes.POINTER(_p)], ctypes.c_int),
    "skb_table_destroy": ([_p], ctypes.c_int),
    "skb_initial_rows": ([_i64, _p, _i64, _i64, _p, _p], ctypes.c_int),
    "skb_table_stats": ([_p, ctypes.POINTER(_i64), _p], ctypes.c_int),
    "skb_table_lookup_or_insert": ([_p, _p, _i64, _i64, _p, _p], ctypes.c_int),
    "skb_table_admit_unique": ([_p, _p, _i64, _i64, _p, _p], ctypes.c_int),
    "skb_table_gather": ([_p, _p, _i64, _p, _p], ctypes.c_int),
    "skb_table_gather_unchecked": ([_p, _p, _i64, _p, _p], ctypes.c_int),
    "skb_sparse_adam_step_unchecked": ([_p, _p, _i64, _p, ctypes.POINTER(AdamScalars), _p], ctypes.c_int),
    "skb_table_scatter_update": ([_p, _p, _i64, _p, _p], ctypes.c_int),
    "skb_table_gather_deferred": ([_p, _p, _i64, _p, _p, _p], ctypes.c_int),
    "skb_table_scatter_update_deferred": ([_p, _p, _i64, _p, _p, _p], ctypes.c_int),
    "skb_table_evict": ([_p, _i64, ctypes.POINTER(_i64), _p], ctypes.c_int),
    "skb_table_export": ([_p, _p, _p, _p, _p, _p, _i64, ctypes.POINTER(_i64), _p], ctypes.c_int),
    "skb_table_restore": ([_p, _p, _i64, _p, _p, _p, _p, _p], ctypes.c_int),
    "skb_table_read_rows": ([_p, _p, _i64, _i32, _p, _p], ctypes.c_int),
    "skb_table_write_rows": ([_p, _p, _i64, _i32, _p, _p], ctypes.c_int),
    "skb_table_read_last_step": ([_p, _p, _i64, _p, _p], ctypes.c_int),
    "skb_table_write_last_step": ([_p, _p, _i64, _p, _i64, _p], ctypes.c_int),
    "skb_table_clear_aux": ([_p, _p, _i64, _p], ctypes.c_int),
    "skb_table_ensure_capacity": ([_p, _i64, _p], ctypes.c_int),
    "skb_table_idmap_get": ([_p, _p, _i64, _p, _p], ctypes.c_int),
    "skb_table_idmap_put": ([_p, _i64, _i64, _p], ctypes.c_int),
    "skb_table_idmap_remove": ([_p, _i64, ctypes.POINTER(_i64), _p], ctypes.c_int),
    "skb_table_free_list": ([_p, _p, _i64, ctypes.POINTER(_i64), _p], ctypes.c_int),
    "skb_table_set_free_list": ([_p, _p, _i64, _p], ctypes.c_int),
    "skb_table_items": ([_p, _p, _p, _i64, ctypes.POINTER(_i64), _p], ctypes.c_int),
    "skb_sparse_adam_step": ([_p, _p, _i64, _p, ctypes.POINTER(AdamScalars), _p], ctypes.c_int),
    "skb_segment_reduce": ([_p, _i64, _i64, _p, _i64, _i32, _i32, _p, _p], ctypes.c_int),
    "skb_segment_tile": ([_p, _i64, _i64, _p, _i64, _i64, ctypes.c_float, _p, _p], ctypes.c_int),
    "skb_segment_reduce_f64": ([_p, _i64, _i64, _p, _i64, _i32, _i32, _p, _p], ctypes.c_int),
    "skb_segment_sum_i64": ([_p, _i64, _i64, _p, _i64, _p, _p], ctypes.c_int),
    "skb_segment_tile_x64": ([_p, _i64, _i64, _p, _i64, _i64, _u64, _p, _p], ctypes.c_int),
    "skb_validate_offsets": ([_p, _i64, _i64, _p], ctypes.c_int),
    "skb_grad_fold": ([_p, _i64, _i64, _p, _i64, _p, _p], ctypes.c_int),
    "skb_fused_forward": ([_p, _p, _i64, ctypes.POINTER(_i64), ctypes.POINTER(_u64), _i32, _i32, _p, _i64,
                           ctypes.POINTER(_i64), ctypes.POINTER(_i32), _i32, _i64, _p, _p], ctypes.c_int),
    "skb_fused_prepare": ([_p, _p, _i64, ctypes.POINTER(_i64), ctypes.POINTER(_u64), _i32, _i32, _p, _i64,
                           ctypes.POINTER(_i64), ctypes.POINTER(_i32), _i32, _i64, _p], ctypes.c_int),
    "skb_fused_prepare_tile": ([_p, _p, _i64, ctypes.POINTER(_i64), ctypes.POINTER(_u64), _i32, _i32, _p, _i64,
                                ctypes.POINTER(_i64), _i64, ctypes.c_float, _i64, _p], ctypes.c_int),
    "skb_fused_forward_tile": ([_p, _p, _i64, ctypes.POINTER(_i64), ctypes.POINTER(_u64), _i32, _i32, _p, _i64,
                                ctypes.POINTER(_i64), _i64, ctypes.c_float, _i64, _p, _p], ctypes.c_int),
    "skb_fused_backward": ([_p, _p, ctypes.POINTER(AdamScalars), _p], ctypes.c_int),
    "skb_fused_backward_ex": ([_p, _p, ctypes.POINTER(AdamScalars), _i32, _p], ctypes.c_int),
    "skb_fused_shard_counts": ([_p, _i64, _p, _p], ctypes.c_int),
    "skb_ipc_alloc": ([_i64, ctypes.POINTER(_p), _p], ctypes.c_int),
    "skb_ipc_open": ([_p, ctypes.POINTER(_p)], ctypes.c_int),
    "skb_ipc_close": ([_p], ctypes.c_int),
    "skb_ipc_free": ([_p], ctypes.c_int),
    "skb_p2p_send_rows": ([_p, _p, _p, _i64, _p, _i32, _p, _p, _p], ctypes.c_int),
    "skb_p2p_send_grads": ([_p, _i64, _i64, _p, _i32, _p, _p, _p], ctypes.c_int),
    "skb_p2p_memops_supported": ([ctypes.POINTER(_i32)], ctypes.c_int),
    "skb_p2p_barrier": ([_p, _i32, _i32, _i64, _p], ctypes.c_int),
    "skb_p2p_put_counts": ([_p, _i32, _i32, _p, _p], ctypes.c_int),
    "skb_fused_last_unique": ([_p, ctypes.POINTER(_i64), ctypes.POINTER(_i64), _p], ctypes.c_int),
    "skb_fused_stats_async": ([_p, _p, _p], ctypes.c_int),
    "skb_fused_profile": ([_p, _i64, _p], ctypes.c_int),
    "skb_fused_profile_read": ([_p, _i32, ctypes.POINTER(ctypes.c_float), _i64, ctypes.POINTER(_i64)], ctypes.c_int),
    "skb_dist_create": ([_i64, _i32, ctypes.POINTER(_p)], ctypes.c_int),
    "skb_dist_destroy": ([_p], ctypes.c_int),
    "skb_dist_prepare": ([_p, _p, _i64, _p, _p, _i32, _i32, _p, _i64, _p, _p, _p, _p], ctypes.c_int),
    "skb_dist_send_ids": ([_p, _i64, _p, _p, _p, _p], ctypes.c_int),
    "skb_dist_pool": ([_p, _p, _i32, _p, _p], ctypes.c_int),
    "skb_dist_fold_send": ([_p, _p, _i32, _i64, _p, _p, _p, _p], ctypes.c_int),
    "skb_dist_buffers": ([_p, ctypes.POINTER(_p), ctypes.POINTER(_p), ctypes.POINTER(_p)], ctypes.c_int),
    "skb_fused_forward_send": ([_p, _p, _i64, _i64, _p, _i32, _p, _p, _p], ctypes.c_int),
    "skb_keys_members": ([_p, _i64, _p, _i32, _p, _p], ctypes.c_int),
    "skb_pool_indexed": ([_p, _i64, _p, _p, _i64, _p, _i32, _i32, _i32, _i64, _p, _p], ctypes.c_int),
    "skb_fold_bags": ([_p, _i64, _p, _i64, _i64, _p, _i64, _i32, _i64, _p, _p], ctypes.c_int),
    "skb_bucketize_multi": ([_p, _p, _i64, _p, _p, _p, _i64, _p], ctypes.c_int),
    "skb_bucketize_multi_async": ([_p, _p, _i64, _p, _p, _p, _i64, _p, _p], ctypes.c_int),
    "skb_mod_multi": ([_p, _p, _i64, _p, _p, _i64, _p], ctypes.c_int),
    "skb_cross_offsets": ([_p, _p, _i64, _p, _p], ctypes.c_int),
    "skb_bucketize_cols": ([_p, _p, _i64, _p, _p, _p, _i64, _p, _p], ctypes.c_int),
    "skb_mod_cols": ([_p, _p, _i64, _p, _p, _i64, _p], ctypes.c_int),
    "skb_pack_members": ([_p, _p, _p, _p, _i64, _i64, _i64, _p, _p, _p], ctypes.c_int),
    "skb_cross": ([_p, _p, _p, _p, _i64, _p, _i64, _p, _p, _p], ctypes.c_int),
    "skb_cross_offsets_many": ([_p, _i64, _p], ctypes.c_int),
    "skb_cross_many": ([_p, _i64, _i64, _p, _p], ctypes.c_int),
    "skb_ragged_truncate": ([_p, _i64, _i64, _i32, _p, _p, _p], ctypes.c_int),
    "skb_gather_elems": ([_p, _i64, _p, _i64, _p, _p], ctypes.c_int),
    "skb_ragged_pad_dense": ([_p, _i64, _i64, _p, _i64, _i64, _p, _p, _p, _p], ctypes.c_int),
    "skb_fused_set_fold_mode": ([_p, _i32], ctypes.c_int),
    "skb_fused_set_variants": ([_p, _i32, _i32], ctypes.c_int),
    "skb_fused_last_variants": ([_p, ctypes.POINTER(_i32), ctypes.POINTER(_i32)], ctypes.c_int),
    "skb_fused_set_graphs": ([_p, ctypes.c_int32], ctypes.c_int),
    # checkpoint boundary (checkpoint.py:192-313)
    "skb_argsort_i64": ([_p, _i64, _p, _p, _p], ctypes.c_int),
    "skb_gather_rows": ([_p, _i64, _p, _i64, _p, _p], ctypes.c_int),
    "skb_scatter_rows": ([_p, _i64, _p, _i64, _p, _p], ctypes.c_int),
    "skb_partition_dest": ([_p, _p, _p, _i64, _p, _p], ctypes.c_int),
    # input side (columnio.py:328-409): host-side native reader
    "skb_reader_open": ([_p, _i64, _p, _i64, _p, _p, _p, _p, _i64, _i64, _i64, ctypes.c_int32, ctypes.c_int32,
                         ctypes.c_int32, _p], ctypes.c_int),
    "skb_reader_next": ([_p, _p], ctypes.c_int),
    "skb_reader_column": ([_p, _i64, _p, _p, _p, _p, _p], ctypes.c_int),
    "skb_reader_close": ([_p], ctypes.c_int),
}

EXPORTED = tuple(_SIGS)

_lock = threading.Lock()
_lib = None


def load_library(path: str = LIB_PATH):
    """dlopen the library and bind every declared symbol (no CUDA calls)."""
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


_host_lib = None


def host_lib():
    """The bound library for HOST-ONLY entry points (the columnar reader's
    file decode); needs no CUDA device because that work is host IO by
    nature — no device computation is ever routed through here."""
    global _host_lib
    if _lib is not None:
        return _lib
    if _host_lib is None:
        with _lock:
            if _host_lib is None:
                _host_lib = load_library()
    return _host_lib


def lib():
    """The bound library; requires a CUDA device (fails loudly otherwise)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                import torch
                if not torch.cuda.is_available():
                    raise RuntimeError("paper_2509_20883_b200 needs a CUDA device (sm_100a); no CPU fallback")
                _lib = load_library()
    return _lib


_EXC = {SKB_E_VALUE: ValueError, SKB_E_INDEX: IndexError, SKB_E_KEY: KeyError,
        SKB_E_ARG: ValueError, SKB_E_UNSUPPORTED: NotImplementedError, SKB_E_NOMEM: MemoryError}


def check(status: int) -> None:
    if status == SKB_OK:
        return
    msg = _lib.skb_last_error().decode("utf-8", "replace")
    if status == SKB_E_KEY:
        raise KeyError(int(_lib.skb_last_error_arg()))
    raise _EXC.get(status, RuntimeError)(msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))


if os.environ.get("SKB_PROFILE_CALLS"):
    # host time spent inside each C-ABI entry point (diagnostics only)
    import atexit
    import collections
    import time as _time

    _CALL_T = collections.defaultdict(lambda: [0, 0.0, 0.0])
    _plain_call = call

    def call(name: str, *args) -> None:  # noqa: F811
        t0 = _time.perf_counter()
        try:
            _plain_call(name, *args)
        finally:
            rec = _CALL_T[name]
            dt = _time.perf_counter() - t0
            rec[0] += 1
            rec[1] += dt
            rec[2] = max(rec[2], dt)

    @atexit.register
    def _report_calls():
        for k, (n, t, mx) in sorted(_CALL_T.items(), key=lambda kv: -kv[1][1])[:20]:
            print(f"[skb calls] {k:36s} {n:7d} calls {t * 1e3:10.2f} ms  {t / n * 1e6:8.1f} us/call  max {mx * 1e3:8.2f} ms",
                  file=sys.stderr)


# ---------------------------------------------------------------------------
# tensor plumbing (torch is the device-memory / stream provider)
# ---------------------------------------------------------------------------

def torch():
    import torch as _t
    return _t


def ctypes_byref(x):
    return ctypes.byref(x)


_RAW_STREAM = None


def stream_ptr(device=None):
    """The current CUDA stream as a cudaStream_t (the raw-pointer query of
    torch's C API when available: ~0.3 us instead of building a Stream object
    per call — the launch-bound C1 step makes a dozen of these)."""
    global _RAW_STREAM
    t = torch()
    if device is None:
        if _RAW_STREAM is None:
            raw, getdev = getattr(t._C, "_cuda_getCurrentRawStream", None), getattr(t._C, "_cuda_getDevice", None)
            _RAW_STREAM = (lambda: raw(getdev())) if raw and getdev else False
        if _RAW_STREAM:
            return ctypes.c_void_p(_RAW_STREAM())
    return ctypes.c_void_p(t.cuda.current_stream(device).cuda_stream)


def ptr(x):
    return ctypes.c_void_p(x.data_ptr()) if x is not None and x.numel() else ctypes.c_void_p(
        x.data_ptr() if x is not None else 0)


_NP2T = {np.dtype(np.int64): "int64", np.dtype(np.float32): "float32", np.dtype(np.uint8): "uint8",
         np.dtype(np.int32): "int32", np.dtype(np.float64): "float64"}


def is_torch(x) -> bool:
    t = torch()
    return isinstance(x, t.Tensor)


def to_dev(x, dtype: str, device=None):
    """numpy/list/torch -> contiguous CUDA tensor of `dtype` (a copy only if needed)."""
    t = torch()
    tdt = getattr(t, dtype)
    if device is None and isinstance(x, t.Tensor) and x.is_cuda and x.dtype == tdt and x.is_contiguous() \
            and x.get_device() == t._C._cuda_getDevice():
        return x  # the common case, without building device objects
    dev = t.device("cuda", t.cuda.current_device()) if device is None else t.device(device)
    if isinstance(x, t.Tensor):
        if x.dtype != tdt:
            x = x.to(tdt)
        if x.device != dev:
            x = x.to(dev)
        return x.contiguous()
    a = np.ascontiguousarray(np.asarray(x, dtype=np.dtype(dtype)))
    if a.nbytes <= _H2DStaging.SLOT and dev.type == "cuda":
        return _staging().put(a, tdt, dev)
    if not a.flags.writeable:
        a = a.copy()
    return t.from_numpy(a).to(dev)


class _H2DStaging:
    """Pinned ring for small host->device copies (offsets, counts, member
    tables): a pageable copy synchronizes the stream, so every such upload
    inside a step would stall the host behind the GPU.  Each slot is refilled
    only after the event of its previous copy has completed."""

    SLOT = 64 << 10
    NSLOT = 64

    def __init__(self):
        t = torch()
        self.buf = t.empty(self.SLOT * self.NSLOT, dtype=t.uint8, pin_memory=True)
        self.host = self.buf.numpy()
        self.events = [None] * self.NSLOT
        self.next = 0
        self.lock = threading.Lock()

    def put(self, a: np.ndarray, tdt, dev):
        t = torch()
        with self.lock:
            k = self.next
            self.next = (k + 1) % self.NSLOT
            if self.events[k] is not None:
                self.events[k].synchronize()
            lo = k * self.SLOT
            self.host[lo:lo + a.nbytes] = a.reshape(-1).view(np.uint8)
            src = self.buf[lo:lo + a.nbytes].view(tdt).reshape(a.shape)
            out = t.empty(a.shape, dtype=tdt, device=dev)
            out.copy_(src, non_blocking=True)
            ev = t.cuda.Event()
            ev.record()
            self.events[k] = ev
        return out


_STAGING = None
_STAGING_LOCK = threading.Lock()


def _staging() -> _H2DStaging:
    global _STAGING
    if _STAGING is None:
        with _STAGING_LOCK:
            if _STAGING is None:
                _STAGING = _H2DStaging()
    return _STAGING


def neg_ones(n: int, device=None):
    """int64[n] of -1 on the device (deferred-check flag arrays): uploaded
    through the pinned staging ring — a host-to-device copy, not a fill
    kernel launched into the step."""
    return to_dev(np.full(n, -1, np.int64), "int64", device)


def empty(shape, dtype: str, device=None):
    t = torch()
    dev = t.device("cuda", t.cuda.current_device()) if device is None else t.device(device)
    return t.empty(shape, dtype=getattr(t, dtype), device=dev)


def out_like(result, as_numpy: bool):
    """Return numpy when the caller passed numpy (drop-in), else the CUDA tensor."""
    if as_numpy:
        return result.cpu().numpy()
    return result
