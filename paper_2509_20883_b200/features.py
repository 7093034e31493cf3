"""Feature engine on the GPU (reference features.py:1-189).

Every transform is one multi-column descriptor kernel (csrc/features.cu,
csrc/hashing.cu); a FusedPlan runs all its columns in one launch and counts
that launch as its single dispatch (features.py:139-146).
"""

from __future__ import annotations

import ctypes

import threading

import numpy as np

from . import _native as N
from . import telemetry
from .hashing import fnv1a64_packed, pack_strings
from .ragged import RaggedTensor


def _check_boundaries(boundaries) -> np.ndarray:
    """features.py:21-27."""
    b = np.asarray(boundaries.cpu().numpy() if N.is_torch(boundaries) else boundaries, dtype=np.float32)
    if b.ndim != 1:
        raise ValueError("boundaries must be a 1-D array")
    if len(b) > 1 and np.any(np.diff(b) <= 0):
        raise ValueError("boundaries must be strictly increasing")
    return b


def hash_feature(strings: RaggedTensor) -> RaggedTensor:
    """Byte strings -> int64 ids via FNV-1a 64 (features.py:30-38).

    Object arrays of bytes are packed on the host into the columnar
    (offsets, blob) layout (columnio.py:96-102) and hashed on the GPU.
    """
    telemetry.bump("features.hash_feature")
    vals = strings.values
    if hasattr(vals, "blob") and hasattr(vals, "offsets"):  # columnio.PackedStrings (reader output)
        return RaggedTensor._trusted(fnv1a64_packed(vals.blob, vals.offsets), strings.row_offsets)
    blob, offs = pack_strings(list(vals))
    hashed = fnv1a64_packed(blob, offs)
    return strings.with_values(hashed)


def hash_feature_packed(blob, str_offsets, row_offsets) -> RaggedTensor:
    """Columnar variant: strings already packed as (blob uint8, str_offsets int64)."""
    telemetry.bump("features.hash_feature")
    return RaggedTensor(fnv1a64_packed(blob, str_offsets), row_offsets)


_DEFERRED = threading.local()


class deferred_checks:
    """Context for input pipelines: data-dependent checks of the feature
    engine (bucketize's NaN -> ValueError, features.py:50-51) are recorded on
    the device instead of being read back per call — no host synchronisation
    inside the step — and raised (same exception and message) when the
    context exits or at `check_deferred()`.  Outside the context every call
    raises synchronously, exactly like the reference."""

    def __enter__(self):
        stack = getattr(_DEFERRED, "stack", None)
        if stack is None:
            stack = _DEFERRED.stack = []
        stack.append([])
        return self

    def __exit__(self, exc_type, exc, tb):
        flags = _DEFERRED.stack.pop()
        if exc_type is None:
            _raise_pending(flags)
        return False


def check_deferred() -> None:
    """Read the checks recorded so far in the innermost deferred_checks()
    context (one synchronisation) and raise the first failure."""
    stack = getattr(_DEFERRED, "stack", None)
    if stack:
        flags, stack[-1] = stack[-1], []
        _raise_pending(flags)


def _raise_pending(flags):
    """Read every recorded flag array in one copy and raise the first
    failure.  An entry is (int64 device flags, message): ValueError(message)
    when flags[0] != -1 (~0: nothing flagged); or (flags, fn): fn(list of the
    flag values) returns the exception to raise, or None."""
    if not flags:
        return
    t = N.torch()
    vals = t.cat([f.reshape(-1) for f, _ in flags]).cpu().tolist()
    k = 0
    for f, msg in flags:
        v = vals[k:k + f.numel()]
        k += f.numel()
        if callable(msg):
            exc = msg(v)
            if exc is not None:
                raise exc
        elif v[0] != -1:
            raise ValueError(msg)


def _deferred_stack():
    """The innermost deferred_checks() record list, or None outside one."""
    stack = getattr(_DEFERRED, "stack", None)
    return stack[-1] if stack else None


def _bucketize_flat(vals_d, col_offs_d, C, edges_d, edge_offs_d):
    n = vals_d.numel()
    out = N.empty((n,), "int64")
    if n:
        stack = getattr(_DEFERRED, "stack", None)
        if stack:
            flag = N.neg_ones(1, vals_d.device)
            N.call("skb_bucketize_multi_async", N.ptr(vals_d), N.ptr(col_offs_d), C, N.ptr(edges_d),
                   N.ptr(edge_offs_d), N.ptr(out), n, N.ptr(flag), N.stream_ptr())
            stack[-1].append((flag, "bucketize input contains NaN"))
        else:
            N.call("skb_bucketize_multi", N.ptr(vals_d), N.ptr(col_offs_d), C, N.ptr(edges_d), N.ptr(edge_offs_d),
                   N.ptr(out), n, N.stream_ptr())
    return out


def bucketize(values: RaggedTensor, boundaries) -> RaggedTensor:
    """bin(v) = #{edges e : v >= e} (features.py:41-53); NaN -> ValueError."""
    telemetry.bump("features.bucketize")
    b = _check_boundaries(boundaries)
    as_np = not N.is_torch(values.values)
    v = N.to_dev(values.values, "float32").reshape(-1)
    edges = N.to_dev(b if len(b) else np.zeros(1, np.float32), "float32")
    eo = N.to_dev(np.array([0, len(b)], np.int64), "int64")
    co = N.to_dev(np.array([0, v.numel()], np.int64), "int64")
    out = _bucketize_flat(v, co, 1, edges, eo)
    return values.with_values(N.out_like(out, as_np))


def mod_transform(ids: RaggedTensor, modulus: int) -> RaggedTensor:
    """Non-negative remainder modulo `modulus` (features.py:56-62)."""
    telemetry.bump("features.mod_transform")
    if modulus <= 0:
        raise ValueError("modulus must be > 0")
    as_np = not N.is_torch(ids.values)
    v = N.to_dev(ids.values, "int64").reshape(-1)
    n = v.numel()
    out = N.empty((n,), "int64")
    if n:
        co = N.to_dev(np.array([0, n], np.int64), "int64")
        m = N.to_dev(np.array([modulus], np.int64), "int64")
        N.call("skb_mod_multi", N.ptr(v), N.ptr(co), 1, N.ptr(m), N.ptr(out), n, N.stream_ptr())
    return ids.with_values(N.out_like(out, as_np))


def cross(a: RaggedTensor, b: RaggedTensor) -> RaggedTensor:
    """Per-row x-major Cartesian product hashed pairwise (features.py:65-89)."""
    telemetry.bump("features.cross")
    return _cross_pairs([(a, b)])[0]


def cross_many(pairs, sizes=None) -> list:
    """`cross` over many column pairs with ONE host read of the output sizes
    (a step's crossed features: offsets for every pair, one readback of all
    totals, then one hashing launch per pair).  `sizes`: the output lengths
    (sum over rows of len_a * len_b) when the caller already knows them from
    host-side offsets (e.g. the input pipeline) — then nothing synchronizes."""
    telemetry.bump("features.cross", len(pairs))
    return _cross_pairs(list(pairs), sizes)


_CROSS_MAX_PAIRS = 1024  # pairs per skb_cross_many launch
_CROSS_BATCH_MAX_ROWS = 1 << 16  # rows one scanning CTA of k_cross_offsets_many takes in stride


def _cross_pairs_each(pairs, sizes=None):
    """Per-pair launches (multi-CTA scan of each pair's row products): for a
    single pair or pairs too long for one scanning CTA."""
    t = N.torch()
    prep = []
    for a, b in pairs:
        if a.num_rows != b.num_rows:
            raise ValueError(f"row-count mismatch: {a.num_rows} vs {b.num_rows}")
        as_np = not N.is_torch(a.values)
        av, bv = N.to_dev(a.values, "int64").reshape(-1), N.to_dev(b.values, "int64").reshape(-1)
        ao, bo = N.to_dev(a.row_offsets, "int64"), N.to_dev(b.row_offsets, "int64")
        rows = a.num_rows
        oo = N.empty((rows + 1,), "int64")
        N.call("skb_cross_offsets", N.ptr(ao), N.ptr(bo), rows, N.ptr(oo), N.stream_ptr())
        prep.append((as_np, av, ao, bv, bo, rows, oo))
    if not prep:
        return []
    flags = None
    if sizes is not None:
        if len(sizes) != len(prep):
            raise ValueError(f"{len(sizes)} sizes for {len(prep)} column pairs")
        totals = [int(x) for x in sizes]
        if any(x < 0 for x in totals):
            raise ValueError("cross sizes must be >= 0")
        # caller-supplied sizes are checked against the device totals: inside
        # deferred_checks() at its exit, otherwise right here (one sync)
        flags = N.neg_ones(len(prep), prep[0][1].device)
    else:
        totals = t.stack([p[6][-1] for p in prep]).cpu().tolist()  # the single synchronisation
    res = []
    for i, ((as_np, av, ao, bv, bo, rows, oo), total) in enumerate(zip(prep, totals)):
        out = N.empty((int(total),), "int64")
        if total or flags is not None:
            N.call("skb_cross", N.ptr(av), N.ptr(ao), N.ptr(bv), N.ptr(bo), rows, N.ptr(oo), int(total), N.ptr(out),
                   N.ptr(flags[i:i + 1]) if flags is not None else None, N.stream_ptr())
        # offsets come from the validated inputs by construction: carried as trusted
        res.append((as_np, out, oo))
    if flags is not None:
        stack = getattr(_DEFERRED, "stack", None)
        pending = [(flags[i:i + 1], f"cross_many: sizes[{i}] = {totals[i]} does not match the rows' product count")
                   for i in range(len(prep))]
        # host (numpy) results are read back here anyway: check them now
        if stack and not any(r[0] for r in res):
            stack[-1].extend(pending)
        else:
            _raise_pending(pending)
    return [RaggedTensor(out.cpu().numpy(), oo.cpu().numpy()) if as_np else RaggedTensor._trusted(out, oo)
            for as_np, out, oo in res]




def _cross_pairs(pairs, sizes=None):
    """All pairs in two launches (csrc/hashing.cu k_cross_offsets_many +
    k_cross_many): one 80-byte descriptor per pair, every pair's offsets in
    one buffer and every pair's products in another (the results are views)."""
    if len(pairs) > _CROSS_MAX_PAIRS:
        k = _CROSS_MAX_PAIRS
        if sizes is not None and len(sizes) != len(pairs):
            raise ValueError(f"{len(sizes)} sizes for {len(pairs)} column pairs")
        return _cross_pairs(pairs[:k], None if sizes is None else sizes[:k]) + \
            _cross_pairs(pairs[k:], None if sizes is None else sizes[k:])
    if len(pairs) <= 1 or max(a.num_rows for a, _ in pairs) > _CROSS_BATCH_MAX_ROWS:
        return _cross_pairs_each(pairs, sizes)
    t = N.torch()
    prep = []
    for a, b in pairs:
        if a.num_rows != b.num_rows:
            raise ValueError(f"row-count mismatch: {a.num_rows} vs {b.num_rows}")
        as_np = not N.is_torch(a.values)
        av, bv = N.to_dev(a.values, "int64").reshape(-1), N.to_dev(b.values, "int64").reshape(-1)
        ao, bo = N.to_dev(a.row_offsets, "int64"), N.to_dev(b.row_offsets, "int64")
        prep.append((as_np, av, ao, bv, bo, a.num_rows))
    if not prep:
        return []
    P = len(prep)
    totals = None
    if sizes is not None:
        if len(sizes) != P:
            raise ValueError(f"{len(sizes)} sizes for {P} column pairs")
        totals = [int(x) for x in sizes]
        if any(x < 0 for x in totals):
            raise ValueError("cross sizes must be >= 0")
    dev = prep[0][1].device
    oo_start = np.zeros(P + 1, np.int64)
    np.cumsum([r + 1 for *_, r in prep], out=oo_start[1:])
    oo_all = N.empty((int(oo_start[-1]),), "int64", dev)
    # caller-supplied sizes are checked against the device totals: inside
    # deferred_checks() at its exit, otherwise right here (one sync)
    flags = N.neg_ones(P, dev) if totals is not None else None
    desc = np.zeros((P, 10), np.int64)
    oo_ptr, fl_ptr = oo_all.data_ptr(), flags.data_ptr() if flags is not None else 0
    for i, (_, av, ao, bv, bo, rows) in enumerate(prep):
        desc[i, :6] = (av.data_ptr(), ao.data_ptr(), bv.data_ptr(), bo.data_ptr(), rows, oo_ptr + 8 * oo_start[i])
        desc[i, 8] = fl_ptr + 8 * i if fl_ptr else 0
    if totals is not None:
        desc[:, 6] = totals
    desc_d = N.to_dev(desc, "int64", dev)
    N.call("skb_cross_offsets_many", N.ptr(desc_d), P, N.stream_ptr())
    if totals is None:  # the single synchronisation: every pair's total in one read
        ends = t.from_numpy(oo_start[1:] - 1).to(dev)
        totals = [int(x) for x in oo_all[ends].cpu().tolist()]
        desc[:, 6] = totals
    base = np.zeros(P + 1, np.int64)
    np.cumsum(totals, out=base[1:])
    desc[:, 7] = base[:-1]
    T = int(base[-1])
    out_all = N.empty((T,), "int64", dev)
    if T:
        desc_d = N.to_dev(desc, "int64", dev)
        N.call("skb_cross_many", N.ptr(desc_d), P, T, N.ptr(out_all), N.stream_ptr())
    # offsets come from the validated inputs by construction: carried as trusted
    res = [(p[0], out_all[base[i]:base[i + 1]], oo_all[oo_start[i]:oo_start[i + 1]]) for i, p in enumerate(prep)]
    if flags is not None:
        stack = getattr(_DEFERRED, "stack", None)
        pending = [(flags[i:i + 1], f"cross_many: sizes[{i}] = {totals[i]} does not match the rows' product count")
                   for i in range(P)]
        # host (numpy) results are read back here anyway: check them now
        if stack and not any(r[0] for r in res):
            stack[-1].extend(pending)
        else:
            _raise_pending(pending)
    return [RaggedTensor(out.cpu().numpy(), oo.cpu().numpy()) if as_np else RaggedTensor._trusted(out, oo)
            for as_np, out, oo in res]


class FusedPlan:
    """Same-kind column transforms executed as one dispatch (features.py:92-162)."""

    def __init__(self, kind: str, params: list):
        if kind not in ("bucketize", "mod"):
            raise ValueError(f"unknown fused kind {kind!r}")
        self.kind = kind
        self._lock = threading.Lock()
        self._dispatches = 0
        self._dev = None
        if kind == "bucketize":
            self.boundaries = [_check_boundaries(b) for b in params]
        else:
            self.moduli = np.asarray(params, dtype=np.int64)
            if self.moduli.ndim != 1 or np.any(self.moduli <= 0):
                raise ValueError("moduli must be positive")

    @classmethod
    def for_bucketize(cls, boundaries_per_column) -> "FusedPlan":
        return cls("bucketize", list(boundaries_per_column))

    @classmethod
    def for_mod(cls, moduli) -> "FusedPlan":
        return cls("mod", list(moduli))

    @property
    def num_columns(self) -> int:
        return len(self.boundaries) if self.kind == "bucketize" else len(self.moduli)

    @property
    def dispatch_count(self) -> int:
        with self._lock:
            return self._dispatches

    def _record_dispatch(self) -> None:
        with self._lock:
            self._dispatches += 1

    def _params_dev(self):
        """Per-column edges / moduli, uploaded once per plan."""
        if self._dev is None:
            if self.kind == "bucketize":
                e = np.concatenate(self.boundaries) if self.boundaries else np.zeros(0, np.float32)
                eo = np.zeros(len(self.boundaries) + 1, np.int64)
                np.cumsum([len(b) for b in self.boundaries], out=eo[1:])
                self._dev = (N.to_dev(e if len(e) else np.zeros(1, np.float32), "float32"), N.to_dev(eo, "int64"))
            else:
                self._dev = (N.to_dev(self.moduli, "int64"),)
        return self._dev

    def _columns(self, columns, dtype: str):
        """Per-column device inputs + a device pointer table (no concatenation)."""
        if len(columns) != self.num_columns:
            raise ValueError(f"plan has {self.num_columns} columns, got {len(columns)}")
        parts = [N.to_dev(c.values, dtype).reshape(-1) for c in columns]
        co = np.zeros(len(parts) + 1, np.int64)
        np.cumsum([p.numel() for p in parts], out=co[1:])
        # empty columns still need a valid address (never dereferenced)
        ptrs = np.array([p.data_ptr() for p in parts], np.int64) if parts else np.zeros(1, np.int64)
        tab = N.to_dev(np.concatenate([ptrs, co]), "int64")
        return parts, tab, co


def _split(out, co, columns, as_np):
    res = []
    for i, c in enumerate(columns):
        piece = out[co[i]:co[i + 1]]
        res.append(c.with_values(piece.cpu().numpy() if as_np else piece))
    return res


def fused_bucketize(plan: FusedPlan, columns: list) -> list:
    """Bucketize many columns in one kernel launch (features.py:165-177),
    reading every column in place through a device pointer table."""
    telemetry.bump("features.fused_bucketize")
    if plan.kind != "bucketize":
        raise ValueError("plan is not a bucketize plan")
    parts, tab, co = plan._columns(columns, "float32")
    edges, eo = plan._params_dev()
    C, n = plan.num_columns, int(co[-1])
    out = N.empty((n,), "int64")
    if n:
        ptrs, offs = ctypes.c_void_p(tab.data_ptr()), ctypes.c_void_p(tab.data_ptr() + 8 * max(C, 1))
        stack = getattr(_DEFERRED, "stack", None)
        if stack:
            flag = N.neg_ones(1, out.device)
            N.call("skb_bucketize_cols", ptrs, offs, C, N.ptr(edges), N.ptr(eo), N.ptr(out), n, N.ptr(flag),
                   N.stream_ptr())
            stack[-1].append((flag, "bucketize input contains NaN"))
        else:
            N.call("skb_bucketize_cols", ptrs, offs, C, N.ptr(edges), N.ptr(eo), N.ptr(out), n, None,
                   N.stream_ptr())
    plan._record_dispatch()
    as_np = bool(columns) and not N.is_torch(columns[0].values)
    return _split(out, co, columns, as_np)


def fused_mod(plan: FusedPlan, columns: list) -> list:
    """Modulus-reduce many columns in one kernel launch (features.py:180-189),
    reading every column in place through a device pointer table."""
    telemetry.bump("features.fused_mod")
    if plan.kind != "mod":
        raise ValueError("plan is not a mod plan")
    parts, tab, co = plan._columns(columns, "int64")
    (mods,) = plan._params_dev()
    C, n = plan.num_columns, int(co[-1])
    out = N.empty((n,), "int64")
    if n:
        N.call("skb_mod_cols", ctypes.c_void_p(tab.data_ptr()), ctypes.c_void_p(tab.data_ptr() + 8 * max(C, 1)), C,
               N.ptr(mods), N.ptr(out), n, N.stream_ptr())
    plan._record_dispatch()
    as_np = bool(columns) and not N.is_torch(columns[0].values)
    return _split(out, co, columns, as_np)
