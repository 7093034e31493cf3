"""Row-wise hash sharding, fused dedup + partition and the sharded exchange
(reference sharding.py:1-297).

In one process a `LogicalTable` holds S native tables on the current GPU
("S virtual shards"), and the two-phase exchange of the reference becomes
device-side routing with no host loops: `unique_partition` (one dedup kernel
pipeline), per-shard admission + gather, and one restore kernel.  With
`torch.distributed` initialised and a table built with `dist=True` each rank
owns shard `rank` and the exchange runs over NCCL (see distributed.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from . import telemetry
from .embedding import DEFAULT_BLOCK_SIZE, EmbeddingTable
from .hashing import fnv1a64
from .optim import AdamConfig, adam_scalars


@dataclass(frozen=True)
class ShardPlan:
    """Stateless id -> shard assignment: mix64(id) mod num_shards (sharding.py:27-43)."""

    num_shards: int

    def __post_init__(self):
        if self.num_shards < 1:
            raise ValueError("num_shards must be >= 1")

    def shard_of(self, ids):
        as_np = not N.is_torch(ids)
        d = N.to_dev(ids, "int64").reshape(-1)
        out = N.empty(d.shape, "int64")
        if d.numel():
            N.call("skb_shard_of", N.ptr(d), d.numel(), self.num_shards, N.ptr(out), N.stream_ptr())
        return N.out_like(out, as_np)


@dataclass
class PartitionResult:
    """Per-shard unique ids (first-occurrence order) + inverse routing (sharding.py:46-71)."""

    shard_ids: list
    inverse_shard: object
    inverse_pos: object
    _uniq_cat: object = None      # device int64[U], shards concatenated
    _counts: tuple = ()           # host per-shard counts
    _as_numpy: bool = True

    @property
    def num_unique(self) -> int:
        return int(sum(self._counts)) if self._counts else sum(len(s) for s in self.shard_ids)

    def _bases(self):
        b = np.zeros(len(self._counts) + 1, np.int64)
        np.cumsum(self._counts, out=b[1:])
        return b

    def restore(self, per_shard_rows):
        """Scatter per-shard response rows back to input order (sharding.py:58-66)."""
        t = N.torch()
        as_np = not N.is_torch(per_shard_rows[0])
        parts = [N.to_dev(r, "float32") for r in per_shard_rows]
        parts = [p.reshape(p.shape[0], -1) for p in parts]
        dim = parts[0].shape[1]
        cat = t.cat(parts).contiguous() if len(parts) > 1 else parts[0]
        bases = N.to_dev(self._bases()[:-1] if self._counts else
                         np.concatenate([[0], np.cumsum([len(s) for s in self.shard_ids])[:-1]]), "int64")
        ish, ipos = N.to_dev(self.inverse_shard, "int64"), N.to_dev(self.inverse_pos, "int64")
        n = ish.numel()
        out = N.empty((n, dim), "float32")
        if n and dim:
            N.call("skb_partition_restore", N.ptr(cat), dim, N.ptr(bases), N.ptr(ish), N.ptr(ipos), n, N.ptr(out),
                   N.stream_ptr())
        shape = tuple(per_shard_rows[0].shape[1:])
        out = out.reshape((n,) + shape)
        return N.out_like(out, as_np)

    def reconstruct_ids(self):
        """Inverse of the partition: the original id array (sharding.py:68-71)."""
        t = N.torch()
        parts = [N.to_dev(s, "int64").reshape(-1) for s in self.shard_ids]
        cat = t.cat(parts) if len(parts) > 1 else parts[0]
        counts = [p.numel() for p in parts]
        bases = N.to_dev(np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int64), "int64")
        ish, ipos = N.to_dev(self.inverse_shard, "int64"), N.to_dev(self.inverse_pos, "int64")
        n = ish.numel()
        out = N.empty((n,), "int64")
        if n:
            ginv = (bases[ish] + ipos).contiguous()
            N.call("skb_gather_elems", N.ptr(cat), 8, N.ptr(ginv), n, N.ptr(out), N.stream_ptr())
        return N.out_like(out, self._as_numpy)


def _partition_dev(ids_d, S: int):
    """Device dedup + partition; returns (uniq_cat, counts_host, inv_shard, inv_pos)."""
    n = ids_d.numel()
    uniq = N.empty((max(n, 1),), "int64")
    counts = N.empty((S,), "int64")
    inv_s = N.empty((n,), "int64")
    inv_p = N.empty((n,), "int64")
    N.call("skb_unique_partition", N.ptr(ids_d), n, S, N.ptr(uniq), N.ptr(counts), N.ptr(inv_s), N.ptr(inv_p),
           N.stream_ptr())
    counts_h = tuple(int(c) for c in counts.cpu().tolist())
    return uniq[: sum(counts_h)], counts_h, inv_s, inv_p


def unique_partition(ids, plan: ShardPlan) -> PartitionResult:
    """Deduplicate ids and split them by owning shard in one pass (sharding.py:74-100)."""
    telemetry.bump("sharding.unique_partition")
    as_np = not N.is_torch(ids)
    d = N.to_dev(ids, "int64").reshape(-1)
    S = plan.num_shards
    uniq, counts, inv_s, inv_p = _partition_dev(d, S)
    bases = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    shard_ids = [uniq[bases[s]:bases[s + 1]] for s in range(S)]
    if as_np:
        u = uniq.cpu().numpy()
        shard_ids = [u[bases[s]:bases[s + 1]].copy() for s in range(S)]
        return PartitionResult(shard_ids, inv_s.cpu().numpy(), inv_p.cpu().numpy(), uniq, counts, True)
    return PartitionResult(shard_ids, inv_s, inv_p, uniq, counts, False)


@dataclass
class LoadStats:
    counts: np.ndarray
    imbalance: float


def load_stats(ids, plan: ShardPlan) -> LoadStats:
    """Per-shard unique-id counts and max/mean imbalance (sharding.py:103-119)."""
    telemetry.bump("sharding.load_stats")
    d = N.to_dev(ids, "int64").reshape(-1)
    counts = N.empty((plan.num_shards,), "int64")
    N.call("skb_shard_unique_counts", N.ptr(d), d.numel(), plan.num_shards, N.ptr(counts), N.stream_ptr())
    c = counts.cpu().numpy()
    total = int(c.sum())
    if total == 0:
        return LoadStats(c, 1.0)
    return LoadStats(c, float(c.max()) / (total / plan.num_shards))


class LogicalTable:
    """Same-dimension tables merged into one sharded table (sharding.py:122-181).

    dist=True: this process owns only shard `rank` of a torch.distributed
    world of size num_shards (one process per GPU).
    """

    def __init__(self, name: str, dim: int, num_shards: int, seed: int = 0, members: list | None = None,
                 namespaced: bool = False, block_size: int = DEFAULT_BLOCK_SIZE, evict_threshold: int | None = None,
                 dtype=np.float32, *, dist: bool = False, capacity_hint: int = 0, group=None):
        if num_shards < 1:
            raise ValueError("num_shards must be >= 1")
        self.name = name
        self.dim = dim
        self.seed = seed
        self.members = list(members) if members is not None else [name]
        self.namespaced = namespaced
        self.dist = dist
        self.group = group
        self._num_shards = num_shards
        if dist:
            from .distributed import ThreadRankGroup
            if isinstance(group, ThreadRankGroup):
                ws, self.rank = group.size, group.rank
            else:
                import torch.distributed as tdist
                ws, self.rank = tdist.get_world_size(group), tdist.get_rank(group)
            if ws != num_shards:
                raise ValueError(f"dist table needs num_shards == world size ({ws}), got {num_shards}")
            self.shards = [EmbeddingTable(f"{name}/shard{self.rank}", dim, seed=seed, block_size=block_size,
                                          evict_threshold=evict_threshold, dtype=dtype, capacity_hint=capacity_hint)]
        else:
            self.rank = 0
            self.shards = [EmbeddingTable(f"{name}/shard{s}", dim, seed=seed, block_size=block_size,
                                          evict_threshold=evict_threshold, dtype=dtype, capacity_hint=capacity_hint)
                           for s in range(num_shards)]
        self._member_salt = {m: fnv1a64(m.encode("utf-8")) for m in self.members}

    @property
    def num_shards(self) -> int:
        return self._num_shards

    @property
    def local_table(self) -> EmbeddingTable:
        return self.shards[0]

    @property
    def num_rows(self) -> int:
        n = sum(t.num_rows for t in self.shards)
        if self.dist and hasattr(self.group, "all_reduce_int"):
            return self.group.all_reduce_int(n)
        if self.dist:
            import torch.distributed as tdist
            x = N.torch().tensor([n], dtype=N.torch().int64, device="cuda")
            tdist.all_reduce(x, group=self.group)
            n = int(x.item())
        return n

    def salt(self, member: str) -> int:
        s = self._member_salt.get(member)
        if s is None:
            raise KeyError(f"{member!r} is not a member of logical table {self.name!r}")
        return s

    def keys_for(self, member: str, ids):
        """Storage keys for a member column's raw ids (sharding.py:170-178)."""
        if not self.namespaced:
            return ids if N.is_torch(ids) else np.asarray(ids, dtype=np.int64)
        salt = self.salt(member)
        as_np = not N.is_torch(ids)
        d = N.to_dev(ids, "int64").reshape(-1)
        out = N.empty(d.shape, "int64")
        if d.numel():
            N.call("skb_keys_for", N.ptr(d), d.numel(), salt, N.ptr(out), N.stream_ptr())
        return N.out_like(out, as_np)

    def evict(self, current_step: int) -> int:
        n = sum(t.evict(current_step) for t in self.shards)
        if self.dist and hasattr(self.group, "all_reduce_int"):
            return self.group.all_reduce_int(n)
        if self.dist:
            import torch.distributed as tdist
            x = N.torch().tensor([n], dtype=N.torch().int64, device="cuda")
            tdist.all_reduce(x, group=self.group)
            n = int(x.item())
        return n


def merge_tables_by_dim(tables, num_shards: int = 1, seed: int = 0, block_size: int = DEFAULT_BLOCK_SIZE,
                        evict_threshold: int | None = None, dtype=np.float32, **kw) -> list:
    """One namespaced LogicalTable per distinct dim, sorted by dim (sharding.py:184-219)."""
    telemetry.bump("sharding.merge_tables_by_dim")
    names = [n for n, _ in tables]
    if len(set(names)) != len(names):
        raise ValueError("duplicate table name")
    by_dim: dict = {}
    for n, d in tables:
        by_dim.setdefault(int(d), []).append(n)
    return [LogicalTable(f"dim{d}", d, num_shards, seed=seed, members=by_dim[d], namespaced=True,
                         block_size=block_size, evict_threshold=evict_threshold, dtype=dtype, **kw)
            for d in sorted(by_dim)]


def _check_plan(lt: LogicalTable, plan: ShardPlan):
    if plan.num_shards != lt.num_shards:
        raise ValueError(f"plan has {plan.num_shards} shards, table has {lt.num_shards}")


def all_to_all_lookup(lt: LogicalTable, ids, plan: ShardPlan, step: int, parallel: bool = True):
    """Rows for ids served by their owning shards (sharding.py:230-254).

    Bit-identical to a single-shard lookup of the same ids.
    `parallel` is accepted for API compatibility: shards are device work on
    one stream (or one rank each when lt.dist).
    """
    telemetry.bump("sharding.all_to_all_lookup")
    _check_plan(lt, plan)
    if lt.dist:
        from .distributed import dist_lookup
        return dist_lookup(lt, ids, step)
    as_np = not N.is_torch(ids)
    d = N.to_dev(ids, "int64").reshape(-1)
    uniq, counts, inv_s, inv_p = _partition_dev(d, lt.num_shards)
    U = sum(counts)
    rows = N.empty((U, lt.dim), "float32")
    base = 0
    for s, c in enumerate(counts):
        if c:
            seg = uniq[base:base + c]
            offs = lt.shards[s]._admit_unique(seg, step)
            N.call("skb_table_gather_unchecked", lt.shards[s].handle, N.ptr(offs), c, N.ptr(rows[base:base + c]),
                   N.stream_ptr())
        base += c
    n = d.numel()
    out = N.empty((n, lt.dim), "float32")
    if n:
        bases = N.to_dev(np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int64), "int64")
        N.call("skb_partition_restore", N.ptr(rows), lt.dim, N.ptr(bases), N.ptr(inv_s), N.ptr(inv_p), n,
               N.ptr(out), N.stream_ptr())
    return N.out_like(out, as_np)


def all_to_all_grad_update(lt: LogicalTable, ids, grads, plan: ShardPlan, cfg: AdamConfig, step: int,
                           parallel: bool = True) -> None:
    """Pre-sum duplicate grads in input order, route to owners, sparse Adam (sharding.py:257-297)."""
    telemetry.bump("sharding.all_to_all_grad_update")
    _check_plan(lt, plan)
    d = N.to_dev(ids, "int64").reshape(-1)
    gshape = tuple(grads.shape) if hasattr(grads, "shape") else np.asarray(grads).shape
    if gshape != (d.numel(), lt.dim):
        raise ValueError(f"grads shape {gshape} != ({d.numel()}, {lt.dim})")
    if lt.dist:
        from .distributed import dist_grad_update
        return dist_grad_update(lt, d, grads, cfg, step)
    g = N.to_dev(grads, "float32")
    uniq, counts, inv_s, inv_p = _partition_dev(d, lt.num_shards)
    U = sum(counts)
    n = d.numel()
    bases_h = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    ginv = N.to_dev(bases_h[:-1], "int64")[inv_s] + inv_p if n else inv_p
    agg = N.empty((max(U, 1), lt.dim), "float32")
    if n:
        N.call("skb_grad_fold", N.ptr(g), n, lt.dim, N.ptr(ginv), U, N.ptr(agg), N.stream_ptr())
    sc = adam_scalars(cfg, step)
    if step < 1:
        raise ValueError("global step t must be >= 1")
    for s, c in enumerate(counts):
        if c:
            b = int(bases_h[s])
            offs = lt.shards[s]._admit_unique(uniq[b:b + c], step)
            N.call("skb_sparse_adam_step_unchecked", lt.shards[s].handle, N.ptr(offs), c, N.ptr(agg[b:b + c]),
                   N.ctypes_byref(sc), N.stream_ptr())
    telemetry.bump("optim.sparse_adam_step", sum(1 for c in counts if c))
