"""Sharded checkpoints of GPU tables in the SafeTensors container (reference checkpoint.py).

Same on-disk contract as the reference (checkpoint.py:1-17), so either side
reads the other's checkpoints byte for byte:

* one container per file: u64-LE header length, compact JSON header
  (optional ``__metadata__`` first, then tensor entries in name order, each
  ``{"dtype","shape","data_offsets"}``), then the packed LE payloads;
* per table the parallel tensors ``<t>.ids / .last_step / .m / .v / .weight``,
  rows globally sorted by stored key and split contiguously over the files
  (``_split_counts``, checkpoint.py:185-187);
* ``manifest.json`` (indent 2) written last as the completion marker.

The B200 path: each shard exports its live rows on the device already sorted
by key (``skb_table_export``); several shards (or ranks) are merged by one
stable device argsort (``skb_argsort_i64``) and row gathers
(``skb_gather_rows``); each column crosses PCIe once into pinned host memory
and the files are written from views of those buffers by a thread pool.
Loading reads the files, copies each column to the device once, routes rows
to the target shard count with ``skb_unique_partition`` +
``skb_partition_dest`` + ``skb_scatter_rows`` and bulk-admits them with
``skb_table_restore`` (checkpoint.py:255-313).

Multi-process (``LogicalTable(dist=True)``, one shard per rank): ``save_sharded``
gathers every rank's export to rank 0 (the only writer) and all ranks return
the same manifest; ``load_sharded(..., dist=True)`` gives each rank its own
shard of the target plan (target_num_shards == world size).
"""

from __future__ import annotations

import json
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import asdict, dataclass, field

import numpy as np

from . import _native as N
from . import telemetry
from .embedding import DEFAULT_BLOCK_SIZE, EmbeddingTable
from .sharding import LogicalTable, _partition_dev

MANIFEST_NAME = "manifest.json"
FORMAT_VERSION = 1
_PARTS = ("ids", "weight", "m", "v", "last_step")

# SafeTensors dtype tags this format uses (checkpoint.py:36-37)
_TAGS = {"F32": np.dtype("<f4"), "I64": np.dtype("<i8")}


def _tag(dt: np.dtype):
    if dt.kind == "f" and dt.itemsize == 4:
        return "F32"
    if dt.kind == "i" and dt.itemsize == 8:
        return "I64"
    return None


class CheckpointError(RuntimeError):
    """Malformed or incomplete checkpoint (reference checkpoint.py:40-41)."""


# ---------------------------------------------------------------------------
# SafeTensors container
# ---------------------------------------------------------------------------

def _le(arr) -> np.ndarray:
    """C-contiguous little-endian array (payloads are LE, row-major)."""
    a = np.ascontiguousarray(arr)
    return a.astype(a.dtype.newbyteorder("<")) if a.dtype.byteorder == ">" else a


def _header(tensors: dict, metadata: dict | None):
    """(header bytes, payload arrays in file order) — checkpoint.py:47-67 layout."""
    head: dict = {}
    if metadata:
        head["__metadata__"] = {str(k): str(metadata[k]) for k in sorted(metadata)}
    arrays, pos = [], 0
    for name in sorted(tensors):
        a = _le(tensors[name])
        tag = _tag(a.dtype)
        if tag is None:
            raise CheckpointError(f"unsupported tensor dtype {a.dtype} for {name!r}")
        head[name] = {"dtype": tag, "shape": list(a.shape), "data_offsets": [pos, pos + a.nbytes]}
        arrays.append(a)
        pos += a.nbytes
    return json.dumps(head, separators=(",", ":")).encode("utf-8"), arrays


def write_safetensors(path, tensors: dict, metadata: dict | None = None) -> None:
    """One container from named arrays; payloads are written straight from
    the arrays' buffers (pinned host staging on the save path)."""
    hb, arrays = _header(tensors, metadata)
    with open(path, "wb") as f:
        f.write(len(hb).to_bytes(8, "little"))
        f.write(hb)
        for a in arrays:
            if a.nbytes:
                f.write(memoryview(a).cast("B"))


def read_safetensors_header(path):
    """(header dict, payload start) with framing validation (checkpoint.py:75-90)."""
    with open(path, "rb") as f:
        raw = f.read(8)
        if len(raw) != 8:
            raise CheckpointError(f"{path}: truncated header length field")
        hlen = int.from_bytes(raw, "little")
        hj = f.read(hlen)
    if len(hj) != hlen:
        raise CheckpointError(f"{path}: truncated header JSON")
    try:
        return json.loads(hj.decode("utf-8")), 8 + hlen
    except (UnicodeDecodeError, json.JSONDecodeError) as e:
        raise CheckpointError(f"{path}: invalid header JSON: {e}") from e


def read_safetensors(path) -> dict:
    """All tensors of a container as numpy arrays (checkpoint.py:93-113): one
    read of the payload into a writable buffer, arrays are views of it."""
    header, start = read_safetensors_header(path)
    size = os.path.getsize(path)
    payload = bytearray(size - start)
    with open(path, "rb") as f:
        f.seek(start)
        f.readinto(payload)
    out = {}
    for name, meta in header.items():
        if name == "__metadata__":
            continue
        dt = _TAGS.get(meta.get("dtype"))
        if dt is None:
            raise CheckpointError(f"{path}: unknown dtype tag {meta.get('dtype')!r} for {name!r}")
        b, e = meta["data_offsets"]
        shape = tuple(meta["shape"])
        want = int(np.prod(shape, dtype=np.int64)) * dt.itemsize
        if e - b != want or e > len(payload) or b < 0:
            raise CheckpointError(f"{path}: bad data_offsets for {name!r}")
        out[name] = np.frombuffer(payload, dtype=dt, count=want // dt.itemsize, offset=b).reshape(shape) \
            .astype(dt.newbyteorder("="), copy=False)
    return out


def read_safetensors_metadata(path) -> dict:
    return read_safetensors_header(path)[0].get("__metadata__", {})


# ---------------------------------------------------------------------------
# manifest (checkpoint.py:123-168) — field order is part of the file format
# ---------------------------------------------------------------------------

@dataclass
class TableMeta:
    name: str
    dim: int
    rows_per_file: list
    global_step: int
    seed: int = 0
    block_size: int = DEFAULT_BLOCK_SIZE
    evict_threshold: int | None = None
    members: list = field(default_factory=list)
    namespaced: bool = False


@dataclass
class CheckpointManifest:
    version: int
    files: list
    tables: list

    def to_json(self) -> str:
        doc = {"version": self.version, "files": self.files, "tables": [asdict(t) for t in self.tables]}
        return json.dumps(doc, indent=2, sort_keys=False)

    @classmethod
    def from_json(cls, text: str) -> "CheckpointManifest":
        d = json.loads(text)
        return cls(d["version"], list(d["files"]), [TableMeta(**t) for t in d["tables"]])


def read_manifest(ckpt_dir) -> CheckpointManifest:
    path = os.path.join(ckpt_dir, MANIFEST_NAME)
    if not os.path.exists(path):
        raise CheckpointError(f"{ckpt_dir}: missing {MANIFEST_NAME}")
    with open(path, "r", encoding="utf-8") as f:
        man = CheckpointManifest.from_json(f.read())
    if man.version != FORMAT_VERSION:
        raise CheckpointError(f"unknown checkpoint format version {man.version}")
    return man


def _split_counts(n: int, parts: int) -> list:
    q, r = divmod(n, parts)
    return [q + (i < r) for i in range(parts)]


def _file_names(num_files: int) -> list:
    return [f"ckpt-{i:05d}-of-{num_files:05d}.safetensors" for i in range(num_files)]


# ---------------------------------------------------------------------------
# device side: export, merge by key, stage to pinned host
# ---------------------------------------------------------------------------

def _group_of(table):
    """(name, local shard tables, logical table or None) — checkpoint.py:176-182."""
    if isinstance(table, LogicalTable):
        return table.name, table.shards, table
    if isinstance(table, EmbeddingTable):
        return table.name, [table], None
    raise TypeError(f"cannot checkpoint {type(table).__name__}")


def _cat(parts):
    torch = N.torch()
    return parts[0] if len(parts) == 1 else torch.cat(parts)


def _gather_to_rank0(cols, logical):
    """Every rank's export columns -> rank 0 (others get None); NCCL on GPUs,
    staged through host memory on gloo."""
    import torch.distributed as dist
    torch = N.torch()
    group = logical.group
    world = dist.get_world_size(group)
    on_gpu = dist.get_backend(group) == "nccl"
    dev = cols[0].device if on_gpu else torch.device("cpu")
    n = torch.tensor([cols[0].shape[0]], dtype=torch.int64, device=dev)
    ns = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(ns, n, group=group)
    counts = [int(x.item()) for x in ns]
    cap = max(max(counts), 1)
    out = []
    for c in cols:
        pad = torch.zeros((cap,) + tuple(c.shape[1:]), dtype=c.dtype, device=dev)
        pad[: c.shape[0]] = c.to(dev)
        bufs = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(bufs, pad, group=group)
        out.append(torch.cat([b[:k] for b, k in zip(bufs, counts)]).to(cols[0].device)
                   if logical.rank == 0 else None)
    return out if logical.rank == 0 else None, sum(counts)


def _export_sorted(shards, logical):
    """(ids, weight, m, v, last_step) device columns of all live rows sorted
    by key (rank 0 only when dist), and the global row count."""
    parts = [t.export_rows(as_numpy=False) for t in shards]
    cols = [_cat([p[i] for p in parts]) for i in range(5)]
    multi = len(shards) > 1
    if logical is not None and logical.dist and logical.num_shards > 1:
        cols, total = _gather_to_rank0(cols, logical)
        if cols is None:
            return None, total
        multi = True
    total = cols[0].shape[0]
    if multi and total:
        keys, perm = N.empty((total,), "int64"), N.empty((total,), "int64")
        N.call("skb_argsort_i64", N.ptr(cols[0]), total, N.ptr(keys), N.ptr(perm), N.stream_ptr())
        out = [keys]
        for c in cols[1:]:
            o = N.torch().empty_like(c)
            row_bytes = c.element_size() * (c.shape[1] if c.dim() == 2 else 1)
            N.call("skb_gather_rows", N.ptr(c), row_bytes, N.ptr(perm), total, N.ptr(o), N.stream_ptr())
            out.append(o)
        cols = out
    return cols, total


def _to_pinned(cols):
    """One D2H per column into pinned host memory; numpy views of it."""
    torch = N.torch()
    host = []
    for c in cols:
        h = torch.empty(c.shape, dtype=c.dtype, pin_memory=True)
        h.copy_(c, non_blocking=True)
        host.append(h)
    torch.cuda.current_stream().synchronize()
    return [h.numpy() for h in host]


# ---------------------------------------------------------------------------
# save / load
# ---------------------------------------------------------------------------

def save_sharded(tables, ckpt_dir, num_files: int, global_step: int = 0) -> CheckpointManifest:
    """Write tables to ``num_files`` SafeTensors files plus the manifest
    (checkpoint.py:192-252); identical logical state -> identical bytes."""
    telemetry.bump("checkpoint.save_sharded")
    if num_files < 1:
        raise ValueError("num_files must be >= 1")
    names = _file_names(num_files)
    per_file = [dict() for _ in range(num_files)]
    metas, seen = [], set()
    writer = True
    for table in tables:
        name, shards, logical = _group_of(table)
        if name in seen:
            raise ValueError(f"duplicate table name {name!r} in checkpoint")
        seen.add(name)
        cols, total = _export_sorted(shards, logical)
        counts = _split_counts(total, num_files)
        first = shards[0]
        metas.append(TableMeta(name=name, dim=first.dim, rows_per_file=counts, global_step=global_step,
                               seed=first.seed, block_size=first.store.block_size,
                               evict_threshold=first.evict_threshold,
                               members=list(logical.members) if logical else [],
                               namespaced=bool(logical.namespaced) if logical else False))
        if cols is None:  # a non-writing rank of a dist table
            writer = False
            continue
        host = _to_pinned(cols)
        lo = 0
        for i, c in enumerate(counts):
            for part, arr in zip(_PARTS, host):
                per_file[i][f"{name}.{part}"] = arr[lo:lo + c]
            lo += c
    manifest = CheckpointManifest(FORMAT_VERSION, names, metas)
    if writer:
        os.makedirs(ckpt_dir, exist_ok=True)
        with ThreadPoolExecutor(max_workers=min(8, num_files)) as ex:
            list(ex.map(lambda i: write_safetensors(os.path.join(ckpt_dir, names[i]), per_file[i]),
                        range(num_files)))
        with open(os.path.join(ckpt_dir, MANIFEST_NAME), "w", encoding="utf-8") as f:
            f.write(manifest.to_json())
    _barrier_if_dist(tables)
    return manifest


def _barrier_if_dist(tables):
    for t in tables:
        if isinstance(t, LogicalTable) and t.dist and t.num_shards > 1:
            import torch.distributed as dist
            dist.barrier(group=t.group)
            return


def _read_columns(ckpt_dir, manifest):
    def one(fname):
        path = os.path.join(ckpt_dir, fname)
        if not os.path.exists(path):
            raise CheckpointError(f"missing shard file {fname}")
        return read_safetensors(path)

    with ThreadPoolExecutor(max_workers=max(1, min(8, len(manifest.files)))) as ex:
        contents = list(ex.map(one, manifest.files))
    tables = []
    for meta in manifest.tables:
        cols = {}
        for part in _PARTS:
            key = f"{meta.name}.{part}"
            chunks = []
            for fname, tensors in zip(manifest.files, contents):
                if key not in tensors:
                    raise CheckpointError(f"{fname}: missing tensor {key!r}")
                chunks.append(tensors[key])
            cols[part] = np.concatenate(chunks) if chunks else np.empty(0)
        n = len(cols["ids"])
        for part in ("weight", "m", "v"):
            if cols[part].shape != (n, meta.dim):
                raise CheckpointError(f"table {meta.name!r}: {part} shape {cols[part].shape} "
                                      f"does not match {n} ids of dim {meta.dim}")
        tables.append((meta, cols))
    return tables


def load_sharded(ckpt_dir, target_num_shards: int, *, dist: bool = False, group=None) -> list:
    """LogicalTables rebuilt under a new shard plan (checkpoint.py:255-313);
    lookups after load bit-match the saved state.  dist=True: this rank
    builds and fills only its own shard (target_num_shards == world size)."""
    telemetry.bump("checkpoint.load_sharded")
    if target_num_shards < 1:
        raise ValueError("target_num_shards must be >= 1")
    manifest = read_manifest(ckpt_dir)
    out = []
    for meta, cols in _read_columns(ckpt_dir, manifest):
        lt = LogicalTable(meta.name, meta.dim, target_num_shards, seed=meta.seed, members=meta.members or None,
                          namespaced=meta.namespaced, block_size=meta.block_size,
                          evict_threshold=meta.evict_threshold, dist=dist, group=group)
        n = len(cols["ids"])
        if n:
            _route_and_restore(lt, cols, n, target_num_shards)
        out.append(lt)
    return out


def _route_and_restore(lt, cols, n, S):
    torch = N.torch()
    dev = {p: N.to_dev(np.ascontiguousarray(cols[p]), "int64" if p in ("ids", "last_step") else "float32")
           for p in _PARTS}
    ids = dev["ids"].reshape(-1)
    _, counts, inv_s, inv_p = _partition_dev(ids, S)
    if sum(counts) != n:
        raise CheckpointError(f"table {lt.name!r}: duplicate ids in checkpoint")
    bases = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    grouped = dev
    if S > 1:
        dest = N.empty((n,), "int64")
        N.call("skb_partition_dest", N.ptr(N.to_dev(bases[:-1].copy(), "int64")), N.ptr(inv_s), N.ptr(inv_p), n,
               N.ptr(dest), N.stream_ptr())
        grouped = {}
        for p, c in dev.items():
            o = torch.empty_like(c)
            row_bytes = c.element_size() * (c.shape[1] if c.dim() == 2 else 1)
            N.call("skb_scatter_rows", N.ptr(c), row_bytes, N.ptr(dest), n, N.ptr(o), N.stream_ptr())
            grouped[p] = o
    owned = [lt.rank] if lt.dist else range(S)
    for k, s in enumerate(owned):
        b, e = int(bases[s]), int(bases[s + 1])
        if e > b:
            lt.shards[k].restore_rows(*(grouped[p][b:e] for p in _PARTS))


def inspect_checkpoint(ckpt_dir) -> str:
    """Readable summary: tables, then per-file tensors (checkpoint.py:319-346)."""
    telemetry.bump("checkpoint.inspect")
    man = read_manifest(ckpt_dir)
    lines = [f"checkpoint: version {man.version}, {len(man.files)} file(s)"]
    lines += [f"table {t.name}: dim {t.dim}, rows {sum(t.rows_per_file)}, global_step {t.global_step}"
              for t in man.tables]
    for fname in man.files:
        path = os.path.join(ckpt_dir, fname)
        if not os.path.exists(path):
            raise CheckpointError(f"missing shard file {fname}")
        header, start = read_safetensors_header(path)
        end = max((m["data_offsets"][1] for k, m in header.items() if k != "__metadata__"), default=0)
        if start + end > os.path.getsize(path):
            raise CheckpointError(f"{fname}: truncated payload")
        lines.append(f"file {fname}:")
        for name in sorted(k for k in header if k != "__metadata__"):
            shape = "x".join(str(d) for d in header[name]["shape"]) or "scalar"
            lines.append(f"  {name} {header[name]['dtype']} [{shape}]")
    return "\n".join(lines) + "\n"
