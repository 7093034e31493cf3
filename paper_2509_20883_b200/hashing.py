"""64-bit hashing primitives on the GPU (reference hashing.py:1-86).

`mix64`, `fnv1a64_batch` and `fnv1a64_pairs` run as sm_100a kernels
(csrc/hashing.cu).  numpy inputs return numpy uint64 like the reference;
torch inputs return int64 CUDA tensors carrying the same bit patterns.
`fnv1a64` of a single host byte string (member-name salts) is host math.
"""

from __future__ import annotations

import numpy as np

from . import _native as N

FNV_OFFSET_BASIS = 0xCBF29CE484222325
FNV_PRIME = 0x100000001B3
GOLDEN_GAMMA = 0x9E3779B97F4A7C15
_M64 = 0xFFFFFFFFFFFFFFFF


def to_u64(ids) -> np.ndarray:
    """Reinterpret int64 values as uint64 bit patterns (hashing.py:27-32)."""
    arr = np.asarray(ids)
    if arr.dtype == np.uint64:
        return arr
    return arr.astype(np.int64).astype(np.uint64)


def _as_i64_bits(x):
    if N.is_torch(x):
        return x, False
    a = np.asarray(x)
    if a.dtype == np.uint64:
        a = a.view(np.int64)
    return np.ascontiguousarray(a.astype(np.int64, copy=False)), True


def mix64(x):
    """SplitMix64 finalizer (hashing.py:35-40) on the GPU."""
    scalar = np.ndim(x) == 0 and not N.is_torch(x)
    a, as_np = _as_i64_bits(np.atleast_1d(x) if scalar else x)
    d = N.to_dev(a, "int64")
    out = N.empty(d.shape, "int64")
    N.call("skb_mix64", N.ptr(d), d.numel(), N.ptr(out), N.stream_ptr())
    if as_np:
        r = out.cpu().numpy().view(np.uint64)
        return r[0] if scalar else r
    return out


def fnv1a64(data: bytes) -> int:
    """FNV-1a 64 of one host byte string (hashing.py:43-48)."""
    h = FNV_OFFSET_BASIS
    for b in bytes(data):
        h = ((h ^ b) * FNV_PRIME) & _M64
    return h


def pack_strings(strings):
    """Host packing of byte strings into (blob uint8, offsets int64) — the
    columnar (lengths, blob) layout (columnio.py:96-102)."""
    strings = [bytes(s) if not isinstance(s, str) else s.encode("utf-8") for s in strings]
    lens = np.fromiter((len(s) for s in strings), count=len(strings), dtype=np.int64)
    offs = np.zeros(len(strings) + 1, np.int64)
    np.cumsum(lens, out=offs[1:])
    blob = np.frombuffer(b"".join(strings), np.uint8) if strings else np.zeros(0, np.uint8)
    return blob, offs


def fnv1a64_packed(blob, offsets):
    """FNV-1a 64 of each blob[offsets[i]:offsets[i+1]] on the GPU -> int64 bits."""
    as_np = not N.is_torch(offsets)
    b = N.to_dev(blob if len(blob) else np.zeros(1, np.uint8), "uint8")
    o = N.to_dev(offsets, "int64")
    n = o.numel() - 1
    out = N.empty((max(n, 0),), "int64")
    if n > 0:
        N.call("skb_fnv1a64_strings", N.ptr(b), N.ptr(o), n, N.ptr(out), N.stream_ptr())
    return N.out_like(out, as_np)


def fnv1a64_batch(strings) -> np.ndarray:
    """FNV-1a 64 over a sequence of byte strings (hashing.py:51-71), uint64."""
    blob, offs = pack_strings(strings)
    return fnv1a64_packed(blob, offs).view(np.uint64)


def fnv1a64_pairs(x, y):
    """FNV-1a 64 over LE8(x) || LE8(y) (hashing.py:74-86)."""
    a, as_np = _as_i64_bits(x)
    b, _ = _as_i64_bits(y)
    da, db = N.to_dev(a, "int64"), N.to_dev(b, "int64")
    out = N.empty(da.shape, "int64")
    if da.numel():
        N.call("skb_fnv1a64_pairs", N.ptr(da), N.ptr(db), da.numel(), N.ptr(out), N.stream_ptr())
    return out.cpu().numpy().view(np.uint64) if as_np else out
