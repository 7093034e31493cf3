"""Ragged combiner pooling on the GPU (reference segments.py:1-116).

`segment_reduce` keeps the reference's two strategies and its `auto` switch
(mean segment length >= 16 -> sequential); both are bit-exact kernels
(csrc/segments.cu): `scatter` is the np.add.at left fold, `sequential` the
np.add.reduceat first + numpy-pairwise order.
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from . import telemetry

AUTO_SEQUENTIAL_MIN_MEAN_LEN = 16

_MODES = {"sum": 0, "mean": 1}
_STRATEGIES = {"sequential": 0, "scatter": 1}


def _check_segments(segments, n: int):
    """segments.py:25-33 (host check for host offsets, device check otherwise)."""
    if N.is_torch(segments):
        offs = segments.to(N.torch().int64).contiguous()
        if offs.ndim != 1 or offs.numel() < 1:
            raise ValueError("segment offsets must be 1-D and start at 0")
        d = N.to_dev(offs, "int64")
        try:
            N.call("skb_validate_offsets", N.ptr(d), d.numel(), n, N.stream_ptr())
        except ValueError as e:
            code = str(e)
            if "start" in code:
                raise ValueError("segment offsets must be 1-D and start at 0") from None
            if "nondecreasing" in code:
                raise ValueError("segment offsets must be nondecreasing") from None
            raise ValueError(f"segment offsets end {int(d[-1].item())} != num rows {n}") from None
        return d
    offs = np.asarray(segments, dtype=np.int64)
    if offs.ndim != 1 or len(offs) < 1 or offs[0] != 0:
        raise ValueError("segment offsets must be 1-D and start at 0")
    if np.any(np.diff(offs) < 0):
        raise ValueError("segment offsets must be nondecreasing")
    if offs[-1] != n:
        raise ValueError(f"segment offsets end {int(offs[-1])} != num rows {n}")
    return offs


def resolve_strategy(strategy: str, n: int, num_segments: int) -> str:
    if strategy == "auto":
        mean_len = n / num_segments if num_segments else 0.0
        return "sequential" if mean_len >= AUTO_SEQUENTIAL_MIN_MEAN_LEN else "scatter"
    if strategy not in _STRATEGIES:
        raise ValueError(f"unknown strategy {strategy!r}")
    return strategy


def _rows2d(rows):
    if N.is_torch(rows):
        return rows if rows.ndim == 2 else rows.reshape(-1, 1), False
    r = np.asarray(rows)
    return (r if r.ndim == 2 else r[:, None]), True


def segment_reduce(rows, segments, mode: str = "sum", strategy: str = "auto"):
    """Pool contiguous row segments (segments.py:61-91)."""
    telemetry.bump("segments.segment_reduce")
    rows, as_np = _rows2d(rows)
    n, dim = int(rows.shape[0]), int(rows.shape[1])
    offs = _check_segments(segments, n)
    if mode not in _MODES:
        raise ValueError(f"unknown mode {mode!r}")
    G = (offs.numel() if N.is_torch(offs) else len(offs)) - 1
    strategy = resolve_strategy(strategy, n, G)
    r = N.to_dev(rows, "float32")
    o = N.to_dev(offs, "int64")
    out = N.empty((G, dim), "float32")
    if G and dim:
        if n == 0:
            out.zero_()
        else:
            N.call("skb_segment_reduce", N.ptr(r), n, dim, N.ptr(o), G, _MODES[mode], _STRATEGIES[strategy],
                   N.ptr(out), N.stream_ptr())
    return N.out_like(out, as_np)


def segment_tile(rows, segments, k: int, pad: float = 0.0):
    """First min(k, len) rows of each segment, padded to k*dim (segments.py:94-116)."""
    telemetry.bump("segments.segment_tile")
    if k < 0:
        raise ValueError("k must be >= 0")
    rows, as_np = _rows2d(rows)
    n, dim = int(rows.shape[0]), int(rows.shape[1])
    offs = _check_segments(segments, n)
    G = (offs.numel() if N.is_torch(offs) else len(offs)) - 1
    out = N.empty((G, k * dim), "float32")
    if G and k and dim:
        r = N.to_dev(rows, "float32")
        o = N.to_dev(offs, "int64")
        N.call("skb_segment_tile", N.ptr(r), n, dim, N.ptr(o), G, int(k), float(pad), N.ptr(out), N.stream_ptr())
    return N.out_like(out, as_np)
