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


def _row_kind(rows):
    """(kind, device dtype, output dtype name).  The output dtype follows the
    rows (segments.py:51-58, 103-116): float32 and float64 have bit-exact
    kernels, integer rows are widened to int64 (wrapping sums, cast back)."""
    name = str(rows.dtype).replace("torch.", "")
    if name in ("float32", "float64"):
        return name, name, name
    if name in ("int8", "int16", "int32", "int64", "uint8", "uint16", "uint32", "uint64"):
        return "int", "int64", name
    raise TypeError(f"segment ops take float or integer rows, got {name}")


def _cast_out(out, name):
    t = N.torch()
    if str(out.dtype).replace("torch.", "") == name:
        return out
    if name.startswith("uint") and not hasattr(t, name):
        return out  # reinterpreted below on the numpy side
    return out.to(getattr(t, name))


def _finish(out, name, as_np):
    if as_np:
        a = out.cpu().numpy()
        return a if a.dtype == np.dtype(name) else a.astype(np.dtype(name))
    return _cast_out(out, name)


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
    kind, dt, oname = _row_kind(rows)
    if kind == "int" and strategy == "sequential":
        # np.add.reduceat promotes integers narrower than int64 (numpy's reduce dtype rule)
        oname = "uint64" if oname.startswith("uint") else "int64"
    if kind == "int" and mode == "mean":
        # segments.py:88-90 divides in place into the integer output
        raise TypeError(f"Cannot cast ufunc 'divide' output from dtype('float64') to dtype('{oname}') "
                        "with casting rule 'same_kind'")
    r = N.to_dev(rows.astype(np.int64) if (kind == "int" and not N.is_torch(rows)) else rows, dt)
    o = N.to_dev(offs, "int64")
    out = N.empty((G, dim), dt)
    if G and dim:
        if n == 0:
            out.zero_()
        elif kind == "int":
            N.call("skb_segment_sum_i64", N.ptr(r), n, dim, N.ptr(o), G, N.ptr(out), N.stream_ptr())
        else:
            fn = "skb_segment_reduce" if dt == "float32" else "skb_segment_reduce_f64"
            N.call(fn, N.ptr(r), n, dim, N.ptr(o), G, _MODES[mode], _STRATEGIES[strategy], N.ptr(out),
                   N.stream_ptr())
    return _finish(out, oname, as_np)


def segment_tile(rows, segments, k: int, pad: float = 0.0):
    """First min(k, len) rows of each segment, padded to k*dim (segments.py:94-116)."""
    telemetry.bump("segments.segment_tile")
    if k < 0:
        raise ValueError("k must be >= 0")
    rows, as_np = _rows2d(rows)
    n, dim = int(rows.shape[0]), int(rows.shape[1])
    offs = _check_segments(segments, n)
    G = (offs.numel() if N.is_torch(offs) else len(offs)) - 1
    kind, dt, oname = _row_kind(rows)
    out = N.empty((G, k * dim), dt)
    if G and k and dim:
        r = N.to_dev(rows.astype(np.int64) if (kind == "int" and not N.is_torch(rows)) else rows, dt)
        o = N.to_dev(offs, "int64")
        if dt == "float32":
            N.call("skb_segment_tile", N.ptr(r), n, dim, N.ptr(o), G, int(k), float(pad), N.ptr(out), N.stream_ptr())
        else:
            # np.full(..., pad, dtype=rows.dtype): the pad cast to the row dtype, as raw 8-byte bits
            bits = np.array([pad], dtype=np.dtype(oname)).astype(np.dtype(dt)).view(np.uint64)[0]
            N.call("skb_segment_tile_x64", N.ptr(r), n, dim, N.ptr(o), G, int(k), int(bits), N.ptr(out),
                   N.stream_ptr())
    return _finish(out, oname, as_np)
