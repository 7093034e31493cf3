"""CPU oracle for the sparse hot path — TEST INFRASTRUCTURE ONLY.

This module is a from-scratch numpy restatement of the reference package
`sparsekit` (RecIS desk-scale re-statement, /root/reference/pkg/src/sparsekit)
for the functions on the dynamic-embedding hot path.  It is the *checker*:
only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import it.  The product package
`paper_2509_20883_b200` never imports it and has no CPU fallback.

Parity pinning: every function here is checked against golden vectors that
were produced by importing the reference itself in the build container
(`tests/golden/make_golden.py` -> `tests/golden/*.npz`) and against the
known-answer examples of SPEC.md (see tests/test_oracle_golden.py).  The
reference's float semantics rest on numpy (pinned by running numpy 2.3.5);
the exact recipes are restated below and in DESIGN.md §Oracle.

Citations are `module.py:line` relative to /root/reference/pkg/src/sparsekit/.
"""

from __future__ import annotations

import numpy as np

M64 = 0xFFFFFFFFFFFFFFFF
_U = np.uint64

# ---------------------------------------------------------------------------
# L0 hashing (hashing.py:14-86)
# ---------------------------------------------------------------------------
FNV_BASIS = 0xCBF29CE484222325          # hashing.py:14
FNV_PRIME = 0x100000001B3               # hashing.py:15
MIX_C1 = 0xBF58476D1CE4E5B9             # hashing.py:22
MIX_C2 = 0x94D049BB133111EB             # hashing.py:23
GAMMA = 0x9E3779B97F4A7C15              # hashing.py:24


def as_u64(x) -> np.ndarray:
    """Two's-complement reinterpretation int64 -> uint64 (hashing.py:27-32)."""
    a = np.asarray(x)
    if a.dtype == np.uint64:
        return a
    return a.astype(np.int64).view(np.uint64) if a.ndim else np.int64(a).view(np.uint64)


def splitmix_finalize(x) -> np.ndarray:
    """SplitMix64 finalizer, wrapping uint64 (hashing.py:35-40)."""
    z = as_u64(x).copy() if np.ndim(x) else as_u64(x)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> _U(30))) * _U(MIX_C1)
        z = (z ^ (z >> _U(27))) * _U(MIX_C2)
        z = z ^ (z >> _U(31))
    return z


def fnv1a_bytes(data: bytes) -> int:
    """FNV-1a 64 of a byte string as unsigned int (hashing.py:43-48)."""
    h = FNV_BASIS
    for byte in data:
        h = ((h ^ byte) * FNV_PRIME) & M64
    return h


def fnv1a_many(strings) -> np.ndarray:
    """FNV-1a 64 per byte string, uint64 result (hashing.py:51-71)."""
    return np.array([fnv1a_bytes(bytes(s)) for s in strings], dtype=np.uint64)


def fnv1a_pair(x, y) -> np.ndarray:
    """FNV-1a over LE8(x) || LE8(y), elementwise (hashing.py:74-86)."""
    xs, ys = as_u64(x), as_u64(y)
    h = np.full(xs.shape, FNV_BASIS, dtype=np.uint64)
    with np.errstate(over="ignore"):
        for word in (xs, ys):
            for k in range(8):
                h = (h ^ ((word >> _U(8 * k)) & _U(0xFF))) * _U(FNV_PRIME)
    return h


# ---------------------------------------------------------------------------
# L2 embedding storage (embedding.py)
# ---------------------------------------------------------------------------

def init_rows(seed: int, ids, dim: int) -> np.ndarray:
    """Deterministic per-(seed, id, column) rows (embedding.py:24-36).

    base = mix(u64(id) ^ mix(u64(seed))); u_c = mix(base + (c+1)*GAMMA);
    row_c = f32( (2 * (u_c >> 11) * 2^-53 - 1) * (1/sqrt(dim)) ), math in f64.
    """
    keys = as_u64(np.atleast_1d(np.asarray(ids, dtype=np.int64)))
    seed_mix = splitmix_finalize(np.uint64(seed & M64))
    base = splitmix_finalize(keys ^ seed_mix)
    with np.errstate(over="ignore"):
        ctr = np.arange(1, dim + 1, dtype=np.uint64) * _U(GAMMA)
        u = splitmix_finalize(base[:, None] + ctr[None, :])
    unit = (u >> _U(11)).astype(np.float64) * (2.0 ** -53)
    return ((2.0 * unit - 1.0) * (1.0 / np.sqrt(float(dim)))).astype(np.float32)


class OracleTable:
    """Single-shard dynamic table: dict IDMap + LIFO free list + flat arrays.

    Mirrors EmbeddingTable (embedding.py:151-308) and BlockStore
    (embedding.py:64-148); rows are kept in one flat array instead of blocks
    (results never depend on block size) but `capacity` reports
    the reference's block-granular value.
    """

    def __init__(self, dim: int, seed: int = 0, block_size: int = 65536,
                 evict_threshold=None):
        self.dim, self.seed, self.block_size = dim, seed, block_size
        self.evict_threshold = evict_threshold
        self.map: dict[int, int] = {}
        self.free: list[int] = []
        self.allocated = 0
        self.w = np.zeros((0, dim), np.float32)
        self.m = np.zeros((0, dim), np.float32)
        self.v = np.zeros((0, dim), np.float32)
        self.last = np.zeros(0, np.int64)
        self.live = np.zeros(0, bool)

    # capacity in block_size units (embedding.py:83-92)
    @property
    def capacity(self) -> int:
        nb = -(-self.allocated // self.block_size)
        return nb * self.block_size

    @property
    def num_rows(self) -> int:
        return len(self.map)

    def _grow(self):
        cap = max(self.capacity, self.allocated)
        if len(self.w) < cap:
            extra = cap - len(self.w)
            self.w = np.concatenate([self.w, np.zeros((extra, self.dim), np.float32)])
            self.m = np.concatenate([self.m, np.zeros((extra, self.dim), np.float32)])
            self.v = np.concatenate([self.v, np.zeros((extra, self.dim), np.float32)])
            self.last = np.concatenate([self.last, np.zeros(extra, np.int64)])
            self.live = np.concatenate([self.live, np.zeros(extra, bool)])

    def _take_slot(self) -> int:
        # free list LIFO first, then the sequential counter (embedding.py:203-207)
        if self.free:
            return self.free.pop()
        s = self.allocated
        self.allocated += 1
        return s

    def lookup_or_insert(self, uniq, step: int) -> np.ndarray:
        """embedding.py:185-223."""
        ids = np.asarray(uniq, dtype=np.int64)
        if len(np.unique(ids)) != len(ids):
            raise ValueError("lookup_or_insert requires duplicate-free ids")
        out = np.empty(len(ids), np.int64)
        fresh = []
        for i, key in enumerate(ids.tolist()):
            s = self.map.get(key)
            if s is None:
                s = self._take_slot()
                self.map[key] = s
                fresh.append(i)
            out[i] = s
        if fresh:
            self._grow()
            fi = np.asarray(fresh, np.int64)
            so = out[fi]
            self.w[so] = init_rows(self.seed, ids[fi], self.dim)
            self.m[so] = 0.0
            self.v[so] = 0.0
            self.live[so] = True
        if len(out):
            self.last[out] = step
        return out

    def _check_live(self, offs, op):
        bad = (offs < 0) | (offs >= len(self.live))
        if not bad.any():
            bad = ~self.live[offs]
        if bad.any():
            raise IndexError(f"{op}: offset {int(offs[np.argmax(bad)])} is not a live slot")

    def gather(self, offsets) -> np.ndarray:
        """embedding.py:233-238."""
        offs = np.asarray(offsets, np.int64)
        self._check_live(offs, "gather")
        return self.w[offs].copy()

    def scatter_update(self, offsets, rows) -> None:
        """embedding.py:240-250."""
        offs = np.asarray(offsets, np.int64)
        rows = np.asarray(rows, np.float32)
        if rows.shape != (len(offs), self.dim):
            raise ValueError(f"rows shape {rows.shape} != ({len(offs)}, {self.dim})")
        if len(np.unique(offs)) != len(offs):
            raise ValueError("scatter_update requires distinct offsets")
        self._check_live(offs, "scatter_update")
        self.w[offs] = rows

    def evict(self, step: int) -> int:
        """embedding.py:252-274: stale slots join the free list in dict order."""
        if self.evict_threshold is None or not self.map:
            return 0
        keys = list(self.map.keys())
        slots = np.fromiter(self.map.values(), np.int64, len(keys))
        stale = (step - self.last[slots]) > self.evict_threshold
        if not stale.any():
            return 0
        for k, st in zip(keys, stale.tolist()):
            if st:
                del self.map[k]
        gone = slots[stale]
        self.free.extend(gone.tolist())
        self.live[gone] = False
        self.m[gone] = 0.0
        self.v[gone] = 0.0
        self.last[gone] = 0
        return int(stale.sum())

    def export_rows(self):
        """embedding.py:276-284: live rows sorted by id."""
        keys = np.fromiter(self.map.keys(), np.int64, len(self.map))
        slots = np.fromiter(self.map.values(), np.int64, len(self.map))
        o = np.argsort(keys, kind="stable")
        keys, slots = keys[o], slots[o]
        return keys, self.w[slots].copy(), self.m[slots].copy(), self.v[slots].copy(), self.last[slots].copy()

    def restore_rows(self, ids, weight, m, v, last_step) -> None:
        """embedding.py:286-308 (raises before any mutation on a present id)."""
        ids = np.asarray(ids, np.int64)
        if len(ids) == 0:
            return
        seen = set()
        for key in ids.tolist():
            if key in self.map or key in seen:
                raise ValueError(f"restore_rows: id {key} already present")
            seen.add(key)
        out = np.empty(len(ids), np.int64)
        for i, key in enumerate(ids.tolist()):
            s = self._take_slot()
            self.map[key] = s
            out[i] = s
        self._grow()
        self.w[out] = np.asarray(weight, np.float32)
        self.m[out] = np.asarray(m, np.float32)
        self.v[out] = np.asarray(v, np.float32)
        self.last[out] = np.asarray(last_step, np.int64)
        self.live[out] = True


# ---------------------------------------------------------------------------
# L3 sharding (sharding.py)
# ---------------------------------------------------------------------------

def owner_of(ids, num_shards: int) -> np.ndarray:
    """mix64(key) % S, unsigned (sharding.py:41-43)."""
    return (splitmix_finalize(np.asarray(ids, np.int64)) % _U(num_shards)).astype(np.int64)


def namespaced_keys(ids, member: str) -> np.ndarray:
    """int64(mix64(u64(id) ^ fnv1a64(member))) (sharding.py:160, 170-178)."""
    salt = _U(fnv1a_bytes(member.encode("utf-8")))
    return splitmix_finalize(as_u64(np.asarray(ids, np.int64)) ^ salt).view(np.int64)


def dedup_partition(ids, num_shards: int):
    """First-occurrence dedup + stable owner split (sharding.py:74-100).

    Returns (shard_ids list, inverse_shard, inverse_pos).
    """
    ids = np.asarray(ids, np.int64)
    S = num_shards
    if len(ids) == 0:
        e = np.empty(0, np.int64)
        return [e.copy() for _ in range(S)], e.copy(), e.copy()
    # first-occurrence order via a dict walk (equivalent to np.unique +
    # argsort(first_index) at sharding.py:87-91)
    rank_of: dict[int, int] = {}
    order = []
    inv_rank = np.empty(len(ids), np.int64)
    for i, key in enumerate(ids.tolist()):
        r = rank_of.get(key)
        if r is None:
            r = len(order)
            rank_of[key] = r
            order.append(key)
        inv_rank[i] = r
    uniq = np.asarray(order, np.int64)
    own = owner_of(uniq, S)
    pos = np.empty(len(uniq), np.int64)
    shards = []
    for s in range(S):
        sel = np.nonzero(own == s)[0]
        shards.append(uniq[sel])
        pos[sel] = np.arange(len(sel))
    return shards, own[inv_rank], pos[inv_rank]


def restore_rows_to_positions(per_shard_rows, inverse_shard, inverse_pos):
    """PartitionResult.restore (sharding.py:58-66)."""
    n = len(inverse_shard)
    first = per_shard_rows[0]
    out = np.empty((n,) + first.shape[1:], first.dtype)
    for s, rows in enumerate(per_shard_rows):
        sel = inverse_shard == s
        out[sel] = rows[inverse_pos[sel]]
    return out


def shard_load(ids, num_shards: int):
    """load_stats (sharding.py:103-119): per-owner unique counts + max/mean."""
    uniq = np.unique(np.asarray(ids, np.int64))
    counts = np.bincount(owner_of(uniq, num_shards), minlength=num_shards).astype(np.int64)
    tot = int(counts.sum())
    return counts, (1.0 if tot == 0 else float(counts.max()) / (tot / num_shards))


def group_by_dim(tables):
    """merge_tables_by_dim grouping (sharding.py:184-219): [(name, dim, members)]."""
    names = [n for n, _ in tables]
    if len(set(names)) != len(names):
        raise ValueError("duplicate table name")
    by = {}
    for n, d in tables:
        by.setdefault(int(d), []).append(n)
    return [(f"dim{d}", d, by[d]) for d in sorted(by)]


# ---------------------------------------------------------------------------
# L2 pooling (segments.py)
# ---------------------------------------------------------------------------
AUTO_SEQ_MIN_MEAN = 16  # segments.py:22


def _valid_offsets(offs, n):
    o = np.asarray(offs, np.int64)
    if o.ndim != 1 or len(o) < 1 or o[0] != 0:
        raise ValueError("segment offsets must be 1-D and start at 0")
    if np.any(np.diff(o) < 0):
        raise ValueError("segment offsets must be nondecreasing")
    if o[-1] != n:
        raise ValueError(f"segment offsets end {int(o[-1])} != num rows {n}")
    return o


def numpy_pairwise(x: np.ndarray) -> np.float32:
    """numpy's float32 pairwise summation for a 1-D run (pinned to numpy 2.3.5).

    n<8: left fold starting at -0.0; n<=128: 8 strided partial sums seeded
    with x[0..7], combined ((0+1)+(2+3))+((4+5)+(6+7)), then the tail in
    order; n>128: split at n/2 rounded down to a multiple of 8, recurse.
    """
    f = np.float32
    n = len(x)
    if n < 8:
        acc = f(-0.0)
        for t in x:
            acc = f(acc + t)
        return acc
    if n <= 128:
        r = [f(x[j]) for j in range(8)]
        i = 8
        lim = n - (n % 8)
        while i < lim:
            for j in range(8):
                r[j] = f(r[j] + x[i + j])
            i += 8
        acc = f(f(f(r[0] + r[1]) + f(r[2] + r[3])) + f(f(r[4] + r[5]) + f(r[6] + r[7])))
        while i < n:
            acc = f(acc + x[i])
            i += 1
        return acc
    half = n // 2
    half -= half % 8
    return f(numpy_pairwise(x[:half]) + numpy_pairwise(x[half:]))


def pool_sequential(rows, offs):
    """np.add.reduceat semantics: rows[s] + pairwise(rows[s+1:e]) (segments.py:36-48)."""
    G = len(offs) - 1
    n = len(rows)
    if G == 0 or n == 0:
        return np.zeros((G, rows.shape[1]), rows.dtype)
    idx = np.minimum(offs[:-1], n - 1)
    out = np.add.reduceat(rows, idx, axis=0)
    out[offs[1:] == offs[:-1]] = 0
    return out


def pool_scatter(rows, offs):
    """np.add.at: left fold from +0 in row order (segments.py:51-58)."""
    G = len(offs) - 1
    out = np.zeros((G, rows.shape[1]), rows.dtype)
    if G and len(rows):
        np.add.at(out, np.repeat(np.arange(G), np.diff(offs)), rows)
    return out


def pool(rows, offsets, mode="sum", strategy="auto"):
    """segment_reduce (segments.py:61-91)."""
    rows = np.asarray(rows)
    if rows.ndim == 1:
        rows = rows[:, None]
    offs = _valid_offsets(offsets, len(rows))
    if mode not in ("sum", "mean"):
        raise ValueError(f"unknown mode {mode!r}")
    if strategy == "auto":
        G = len(offs) - 1
        strategy = "sequential" if (len(rows) / G if G else 0.0) >= AUTO_SEQ_MIN_MEAN else "scatter"
    if strategy == "sequential":
        out = pool_sequential(rows, offs)
    elif strategy == "scatter":
        out = pool_scatter(rows, offs)
    else:
        raise ValueError(f"unknown strategy {strategy!r}")
    if mode == "mean":
        ln = np.diff(offs).astype(out.dtype)
        np.divide(out, ln[:, None], out=out, where=ln[:, None] > 0)
    return out


def tile(rows, offsets, k, pad=0.0):
    """segment_tile (segments.py:94-116): first min(k,len) rows, padded."""
    if k < 0:
        raise ValueError("k must be >= 0")
    rows = np.asarray(rows)
    if rows.ndim == 1:
        rows = rows[:, None]
    offs = _valid_offsets(offsets, len(rows))
    G, D = len(offs) - 1, rows.shape[1]
    out = np.full((G, k, D), pad, rows.dtype)
    for g in range(G):
        take = min(k, int(offs[g + 1] - offs[g]))
        out[g, :take] = rows[offs[g]:offs[g] + take]
    return out.reshape(G, k * D)


# ---------------------------------------------------------------------------
# L2 optimizer (optim.py:42-83)
# ---------------------------------------------------------------------------

def adam_scalars(lr, beta1, beta2, eps, weight_decay, variant, t):
    """Host-side float32 scalars exactly as optim.py:69-75 builds them."""
    f = np.float32
    return dict(lr=f(lr), b1=f(beta1), b2=f(beta2), eps=f(eps), one=f(1.0),
                bc1=f(1.0 - beta1 ** t), bc2=f(1.0 - beta2 ** t),
                lrwd=f(f(lr) * f(weight_decay)),
                decay=(variant == "adamw" and weight_decay != 0.0))


def adam_rows(p, m, v, g, sc):
    """One lazy Adam/AdamW update on row blocks, float32 throughout (optim.py:77-83)."""
    p = np.asarray(p, np.float32)
    if sc["decay"]:
        p = p - sc["lrwd"] * p
    m = sc["b1"] * m + (sc["one"] - sc["b1"]) * g
    v = sc["b2"] * v + (sc["one"] - sc["b2"]) * (g * g)
    p = p - sc["lr"] * (m / sc["bc1"]) / (np.sqrt(v / sc["bc2"]) + sc["eps"])
    return p.astype(np.float32), m.astype(np.float32), v.astype(np.float32)


def sparse_adam(table: OracleTable, offsets, grads, lr=1e-3, beta1=0.9, beta2=0.999,
                eps=1e-8, weight_decay=0.0, variant="adam", t=1):
    """sparse_adam_step on an OracleTable (optim.py:42-83)."""
    if t < 1:
        raise ValueError("global step t must be >= 1")
    offs = np.asarray(offsets, np.int64)
    if len(np.unique(offs)) != len(offs):
        raise ValueError("sparse_adam_step requires distinct offsets")
    g = np.asarray(grads, np.float32)
    if g.shape != (len(offs), table.dim):
        raise ValueError(f"grads shape {g.shape} != ({len(offs)}, {table.dim})")
    if not len(offs):
        return
    sc = adam_scalars(lr, beta1, beta2, eps, weight_decay, variant, t)
    p, m, v = adam_rows(table.w[offs], table.m[offs], table.v[offs], g, sc)
    table.w[offs], table.m[offs], table.v[offs] = p, m, v


def fold_grads(inverse_pos, grads, num_unique):
    """Pre-aggregation np.add.at left fold in input order (sharding.py:283-290)."""
    g = np.zeros((num_unique, grads.shape[1]), grads.dtype)
    np.add.at(g, inverse_pos, grads)
    return g


# ---------------------------------------------------------------------------
# L3 orchestration (sharding.py:230-297)
# ---------------------------------------------------------------------------

class OracleLogical:
    """LogicalTable (sharding.py:122-181): S OracleTables + member salts."""

    def __init__(self, name, dim, num_shards, seed=0, members=None, namespaced=False,
                 block_size=65536, evict_threshold=None):
        self.name, self.dim, self.namespaced = name, dim, namespaced
        self.members = list(members) if members is not None else [name]
        self.shards = [OracleTable(dim, seed, block_size, evict_threshold) for _ in range(num_shards)]

    def keys_for(self, member, ids):
        ids = np.asarray(ids, np.int64)
        if not self.namespaced:
            return ids
        if member not in self.members:
            raise KeyError(f"{member!r} is not a member of logical table {self.name!r}")
        return namespaced_keys(ids, member)

    @property
    def num_rows(self):
        return sum(t.num_rows for t in self.shards)

    def evict(self, step):
        return sum(t.evict(step) for t in self.shards)


def lookup(lt: OracleLogical, ids, step):
    """all_to_all_lookup (sharding.py:230-254)."""
    S = len(lt.shards)
    shard_ids, inv_s, inv_p = dedup_partition(ids, S)
    rows = []
    for s in range(S):
        offs = lt.shards[s].lookup_or_insert(shard_ids[s], step)
        rows.append(lt.shards[s].gather(offs))
    return restore_rows_to_positions(rows, inv_s, inv_p)


def grad_update(lt: OracleLogical, ids, grads, step, **adam):
    """all_to_all_grad_update (sharding.py:257-297)."""
    ids = np.asarray(ids, np.int64)
    grads = np.asarray(grads)
    if grads.shape != (len(ids), lt.dim):
        raise ValueError(f"grads shape {grads.shape} != ({len(ids)}, {lt.dim})")
    S = len(lt.shards)
    shard_ids, inv_s, inv_p = dedup_partition(ids, S)
    for s in range(S):
        sel = inv_s == s
        g = fold_grads(inv_p[sel], grads[sel], len(shard_ids[s]))
        offs = lt.shards[s].lookup_or_insert(shard_ids[s], step)
        sparse_adam(lt.shards[s], offs, g, t=step, **adam)


# ---------------------------------------------------------------------------
# Feature engine (features.py)
# ---------------------------------------------------------------------------

def _edges(b):
    e = np.asarray(b, np.float32)
    if e.ndim != 1:
        raise ValueError("boundaries must be a 1-D array")
    if len(e) > 1 and np.any(np.diff(e) <= 0):
        raise ValueError("boundaries must be strictly increasing")
    return e


def bucketize_values(values, boundaries) -> np.ndarray:
    """bin = #{e <= f32(v)} (features.py:41-53)."""
    e = _edges(boundaries)
    x = np.asarray(values, np.float32)
    if np.isnan(x).any():
        raise ValueError("bucketize input contains NaN")
    return np.searchsorted(e, x, side="right").astype(np.int64)


def floor_mod(values, modulus: int) -> np.ndarray:
    """Non-negative remainder (features.py:56-62)."""
    if modulus <= 0:
        raise ValueError("modulus must be > 0")
    return np.remainder(np.asarray(values, np.int64), np.int64(modulus))


def hash_strings(strings) -> np.ndarray:
    """hash_feature values (features.py:30-38)."""
    return fnv1a_many(list(strings)).view(np.int64)


def cross_rows(a_vals, a_offs, b_vals, b_offs):
    """cross (features.py:65-89): x-major per-row products, FNV of pairs."""
    a_offs = np.asarray(a_offs, np.int64)
    b_offs = np.asarray(b_offs, np.int64)
    if len(a_offs) != len(b_offs):
        raise ValueError(f"row-count mismatch: {len(a_offs) - 1} vs {len(b_offs) - 1}")
    la, lb = np.diff(a_offs), np.diff(b_offs)
    offs = np.zeros(len(la) + 1, np.int64)
    np.cumsum(la * lb, out=offs[1:])
    xs, ys = [], []
    for r in range(len(la)):
        for i in range(int(la[r])):
            for j in range(int(lb[r])):
                xs.append(a_vals[a_offs[r] + i])
                ys.append(b_vals[b_offs[r] + j])
    vals = fnv1a_pair(np.asarray(xs, np.int64), np.asarray(ys, np.int64)).view(np.int64)
    return vals, offs


# ---------------------------------------------------------------------------
# Checkpoint container (checkpoint.py:1-17, 47-72, 123-252)
# ---------------------------------------------------------------------------

def safetensors_bytes(tensors: dict) -> bytes:
    """One SafeTensors container, assembled by hand: u64-LE header length,
    compact JSON header with entries in name order, packed LE payloads
    (checkpoint.py:47-72, no __metadata__)."""
    import json
    import struct
    entries, raws, off = [], [], 0
    for name in sorted(tensors):
        a = np.asarray(tensors[name])
        if a.dtype == np.float32:
            tag, raw = "F32", a.astype("<f4").tobytes()
        elif a.dtype == np.int64:
            tag, raw = "I64", a.astype("<i8").tobytes()
        else:
            raise TypeError(a.dtype)
        shape = ",".join(str(d) for d in a.shape)
        entries.append(f'{json.dumps(name)}:{{"dtype":"{tag}","shape":[{shape}],'
                       f'"data_offsets":[{off},{off + len(raw)}]}}')
        raws.append(raw)
        off += len(raw)
    head = ("{" + ",".join(entries) + "}").encode("utf-8")
    return struct.pack("<Q", len(head)) + head + b"".join(raws)


def checkpoint_files(groups, num_files: int, global_step: int) -> dict:
    """save_sharded (checkpoint.py:192-252) as {file name: bytes}.

    groups: [(name, [OracleTable shards], members, namespaced)], members = []
    for a plain table.  Rows of all shards are merged in key order and split
    contiguously, the first n % num_files files taking one extra row."""
    import json
    names = [f"ckpt-{i:05d}-of-{num_files:05d}.safetensors" for i in range(num_files)]
    files = [dict() for _ in range(num_files)]
    metas = []
    for name, shards, members, namespaced in groups:
        ex = [t.export_rows() for t in shards]
        cols = [np.concatenate([e[i] for e in ex]) for i in range(5)]
        order = np.argsort(cols[0], kind="stable")
        cols = [c[order] for c in cols]
        n = len(order)
        counts = [n // num_files + (1 if i < n % num_files else 0) for i in range(num_files)]
        t0 = shards[0]
        metas.append({"name": name, "dim": t0.dim, "rows_per_file": counts, "global_step": global_step,
                      "seed": t0.seed, "block_size": t0.block_size, "evict_threshold": t0.evict_threshold,
                      "members": list(members), "namespaced": bool(namespaced)})
        lo = 0
        for i, c in enumerate(counts):
            for part, col in zip(("ids", "weight", "m", "v", "last_step"), cols):
                files[i][f"{name}.{part}"] = col[lo:lo + c]
            lo += c
    out = {fn: safetensors_bytes(t) for fn, t in zip(names, files)}
    out["manifest.json"] = json.dumps({"version": 1, "files": names, "tables": metas}, indent=2).encode("utf-8")
    return out
