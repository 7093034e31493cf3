"""Fused sparse step for a request-merged logical table (SURVEY §8b additions).

`lookup_pool` = keys_for + dedup/admission + gather + per-bag pooling in one
native call; `pool_grad_adam` = the pooled-gradient backward: per unique row
an in-order fold of dpooled[bag] (/len for mean) followed by Adam/AdamW on
the row.  On a single shard the results are bit-identical to the reference
pipeline train.py:130-195 (all_to_all_lookup -> segment_reduce ->
per-row grad expansion -> all_to_all_grad_update), with per-position grads
defined in float32 as dpooled[bag] / float32(len) for mean bags.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N
from . import telemetry
from .optim import AdamConfig, adam_scalars
from .segments import resolve_strategy
from .sharding import LogicalTable

_MODES = {"sum": 0, "mean": 1, "tile": 2}


class PackedBatch:
    """One logical table's batch: member ids concatenated + bag offsets.

    ids       int64 CUDA [N]      members' raw ids, members in `members` order
    bag_offs  int64 CUDA [G+1]    bag offsets over positions (members' bags concatenated)
    member_pos / member_bag       host int64 [F+1] ranges per member
    """

    def __init__(self, lt: LogicalTable, members, ids_list, offsets_list, strategy="auto"):
        t = N.torch()
        self.members = list(members)
        ids_d = [N.to_dev(x, "int64").reshape(-1) for x in ids_list]
        offs_d = [N.to_dev(o, "int64").reshape(-1) for o in offsets_list]
        F = len(ids_d)
        self.member_pos = np.zeros(F + 1, np.int64)
        self.member_bag = np.zeros(F + 1, np.int64)
        for f in range(F):
            self.member_pos[f + 1] = self.member_pos[f] + ids_d[f].numel()
            self.member_bag[f + 1] = self.member_bag[f] + offs_d[f].numel() - 1
        G = int(self.member_bag[F])
        if F == 1:
            self.ids, self.bag_offs = ids_d[0], offs_d[0]
        else:
            # one launch through per-member pointer tables (no cat / repeat_interleave)
            dev = ids_d[0].device
            tab = np.concatenate([[x.data_ptr() for x in ids_d], [o.data_ptr() for o in offs_d],
                                  self.member_pos, self.member_bag]).astype(np.int64)
            tab_d = N.to_dev(tab, "int64", dev)
            self.ids = N.empty((self.num_ids,), "int64", dev)
            self.bag_offs = N.empty((G + 1,), "int64", dev)
            b = tab_d.data_ptr()
            vp = ctypes.c_void_p
            N.call("skb_pack_members", vp(b), vp(b + 8 * F), vp(b + 16 * F), vp(b + 16 * F + 8 * (F + 1)), F,
                   self.num_ids, G, N.ptr(self.ids), N.ptr(self.bag_offs), N.stream_ptr())
        self.salts = np.array([lt.salt(m) if lt.namespaced else 0 for m in self.members], np.uint64)
        self.strategy = np.array(
            [0 if resolve_strategy(strategy, int(self.member_pos[f + 1] - self.member_pos[f]),
                                   int(self.member_bag[f + 1] - self.member_bag[f])) == "sequential" else 1
             for f in range(F)], np.int32)
        self.namespaced = lt.namespaced
        self._c_args = None

    @property
    def num_ids(self) -> int:
        return int(self.member_pos[-1])

    @property
    def num_bags(self) -> int:
        return int(self.member_bag[-1])


def _batch_args(lt: LogicalTable, batch: PackedBatch, step: int, mode: str):
    if mode not in _MODES:
        raise ValueError(f"unknown mode {mode!r}")
    if lt.num_shards != 1 or lt.dist:
        raise NotImplementedError("the fused step runs on one shard; use all_to_all_lookup for S > 1")
    F = len(batch.members)
    if batch._c_args is None:
        batch._c_args = ((ctypes.c_int64 * (F + 1))(*batch.member_pos.tolist()),
                         (ctypes.c_uint64 * max(F, 1))(*[int(s) for s in batch.salts]),
                         (ctypes.c_int64 * (F + 1))(*batch.member_bag.tolist()),
                         (ctypes.c_int32 * max(F, 1))(*batch.strategy.tolist()))
    mp, sl, mb, st = batch._c_args
    return (lt.local_table.handle, N.ptr(batch.ids), batch.num_ids, mp, sl, F, 1 if batch.namespaced else 0,
            N.ptr(batch.bag_offs), batch.num_bags, mb, st, _MODES[mode], int(step))


def _tile_args(args, k, pad):
    """Entry-point arguments of the tile combiner (segment_tile: k rows per bag, `pad` after)."""
    if k is None:
        raise ValueError("mode 'tile' needs k (rows kept per bag)")
    if k < 0:
        raise ValueError("k must be >= 0")
    h, ids, n, mp, sl, F, ns, bo, G, mb, _st, _mode, step = args
    return (h, ids, n, mp, sl, F, ns, bo, G, mb, int(k), float(pad), step)


def prefetch(lt: LogicalTable, batch: PackedBatch, step: int, mode: str = "mean", k=None, pad: float = 0.0) -> None:
    """Enqueue the index phase (probe, admission, sort) of a future step.

    Issue it for step k+1 before `lookup_pool` of step k (or between that
    and `pool_grad_adam` of step k): the index work of step k+1 then runs on
    the table's index stream underneath step k's pool and fold+Adam.  At
    most two batches are in flight.  Admission happens at prefetch time, so
    table edits that would move slots the prefetched batch already holds
    (evict, restore_rows, IDMap put / remove / free_list, scatter_update)
    raise ValueError until that batch has been pooled and backwarded.
    """
    telemetry.bump("fused.prefetch")
    args = _batch_args(lt, batch, step, mode)
    if mode == "tile":
        N.call("skb_fused_prepare_tile", *_tile_args(args, k, pad), N.stream_ptr())
    else:
        N.call("skb_fused_prepare", *args, N.stream_ptr())


def lookup_pool(lt: LogicalTable, batch: PackedBatch, step: int, mode: str = "mean", out=None, k=None,
                pad: float = 0.0):
    """Pooled embeddings [G, D] of every bag of the batch (single shard);
    mode "tile": the bags' first k rows concatenated, [G, k*D], rows past a
    bag's length filled with `pad` (segment_tile, segments.py:94-116)."""
    telemetry.bump("fused.lookup_pool")
    args = _batch_args(lt, batch, step, mode)
    if mode == "tile":
        targs = _tile_args(args, k, pad)
        if out is None:
            out = N.empty((batch.num_bags, int(k) * lt.dim), "float32")
        N.call("skb_fused_forward_tile", *targs, N.ptr(out), N.stream_ptr())
        return out
    if out is None:
        out = N.empty((batch.num_bags, lt.dim), "float32")
    N.call("skb_fused_forward", *args, N.ptr(out), N.stream_ptr())
    return out


def pool_grad_adam(lt: LogicalTable, dpooled, cfg: AdamConfig, step: int, prescaled: bool = False) -> None:
    """Backward of the last lookup_pool on `lt`: grad fold + Adam/AdamW on touched rows.
    `dpooled` has the forward output's shape ([G, D], or [G, k*D] for tile).

    prescaled=True: `dpooled` already is each bag's per-position gradient —
    train.py:181-186 builds float32(dpooled64 / len) in float64 — and is
    folded as given, so the step is bit-exact with the reference's float64
    expansion (the default divides a float32 dpooled by float32(len))."""
    telemetry.bump("fused.pool_grad_adam")
    if step < 1:
        raise ValueError("global step t must be >= 1")
    g = N.to_dev(dpooled, "float32")
    sc = adam_scalars(cfg, step)
    N.call("skb_fused_backward_ex", lt.local_table.handle, N.ptr(g), ctypes.byref(sc), 1 if prescaled else 0,
           N.stream_ptr())


def step_load_stats(lt: LogicalTable, plan, out=None, sync: bool = True):
    """load_stats (sharding.py:103-119) of the keys of the last prepared fused
    batch for `plan` — train.py:223-228's per-step probe — from the step's
    own sorted slots (one pass over the run heads on the device).
    sync=False returns the device counts tensor (no host round trip)."""
    from .sharding import LoadStats
    S = plan.num_shards
    counts = out if out is not None else N.empty((S,), "int64")
    N.call("skb_fused_shard_counts", lt.local_table.handle, S, N.ptr(counts), N.stream_ptr())
    if not sync:
        return counts
    c = counts.cpu().numpy()
    total = int(c.sum())
    return LoadStats(c, float(c.max()) / (total / S) if total else 1.0)


def last_step_stats(lt: LogicalTable):
    """(unique rows touched, new rows admitted) of the last fused step (synchronizes)."""
    u, k = ctypes.c_int64(), ctypes.c_int64()
    N.call("skb_fused_last_unique", lt.local_table.handle, ctypes.byref(u), ctypes.byref(k), N.stream_ptr())
    return int(u.value), int(k.value)


def use_graphs(lt: LogicalTable, enable: bool = True) -> None:
    """CUDA-graph mode for the fused step on `lt`: each
    phase's device work — index phase, pool, fold+Adam — is captured on its
    second call with an unchanged signature (same batch / output / grad
    buffers and sizes, no table growth) and replayed with one graph launch,
    the step and Adam scalars patched in.  Results are identical to eager
    mode; it removes the per-kernel launch cost that dominates small batches."""
    for t in lt.shards:
        N.call("skb_fused_set_graphs", t.handle, int(bool(enable)))


def set_fold_mode(lt: LogicalTable, mode: str = "exact") -> None:
    """How the fused backward folds the gradients of hot ids (runs of > 32
    positions in one batch).  "exact" (default): np.add.at's serial left fold
    (sharding.py:283-290), bit-exact with the reference.  "tree": opt-in
    tolerance mode — chunks of 256 positions folded in parallel, then the
    chunk sums in order; per column |error| <= (256 + len/256) * 2^-24 *
    sum|g|, below the serial fold's own len * 2^-24 * sum|g| bound.  Hot
    ids then cost memory bandwidth instead of one FADD latency per position."""
    if mode not in ("exact", "tree"):
        raise ValueError(f"unknown fold mode {mode!r}")
    for t in lt.shards:
        N.call("skb_fused_set_fold_mode", t.handle, 1 if mode == "tree" else 0)


def set_variants(lt: LogicalTable, adam: int = -1, pool: int = -1) -> None:
    """Force the fused step's fold+Adam / pool kernel variant on `lt`
    (-1 = environment default, 0 = auto).  Every variant is
    bit-exact; this exists for sweeps and for the parity tests."""
    for t in lt.shards:
        N.call("skb_fused_set_variants", t.handle, int(adam), int(pool))


def last_variants(lt: LogicalTable):
    """(fold+Adam variant, pool variant) the last fused step ran on shard 0."""
    a, p = ctypes.c_int32(), ctypes.c_int32()
    N.call("skb_fused_last_variants", lt.shards[0].handle, ctypes.byref(a), ctypes.byref(p))
    return int(a.value), int(p.value)
