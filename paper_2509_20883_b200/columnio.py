"""Columnar sample files and the sharded batch reader (reference columnio.py).

Same file format as the reference (columnio.py:1-20): ``RCOL`` magic, u32
version, u64 header length, compact JSON header ``{"schema", "chunk_index"}``,
then chunk payloads; per chunk and column ``u8 compressed | u64 raw length |
u64 stored length | payload`` with the payload = chunk-local int64 row
offsets (ragged columns) + values, byte strings as int64 lengths + blob, raw
DEFLATE when compressed.  ``write_dataset`` here produces the reference's
bytes; files written by either side read identically.

Reading is split by plane.  This module parses headers and plans the shard
(global chunk index mod num_shards, columnio.py:306-325).  The data plane is
native (csrc/columnio.cpp through ``skb_reader_*``): decoder threads pread and
inflate chunks out of order, an assembler thread slices fixed-row batches
across chunk boundaries in chunk order into reusable — for GPU delivery,
page-locked — buffers.  ``open_reader(..., device="cuda")`` then moves each
column to the GPU with one async copy per column and yields RaggedTensors of
device tensors; byte-string columns arrive as :class:`PackedStrings`
(string offsets + blob, no Python objects) which ``hash_feature`` hashes on
the GPU directly.  ``device=None`` is the drop-in: fresh numpy arrays, byte
strings as object arrays, exactly the reference's batches.
"""

from __future__ import annotations

import ctypes
import json
import os
import zlib
from dataclasses import dataclass

import numpy as np

from . import _native as N
from . import telemetry
from .ragged import RaggedTensor

MAGIC = b"RCOL"
FORMAT_VERSION = 1
_DTYPES = ("float32", "int64", "bytes")
_CODE = {"float32": 0, "int64": 1, "bytes": 2}
_NP = {"float32": np.dtype("<f4"), "int64": np.dtype("<i8")}


class ColumnIOError(RuntimeError):
    """Malformed / truncated dataset file (reference columnio.py:40-41)."""


@dataclass(frozen=True)
class ColumnSpec:
    name: str
    dtype: str
    ragged: bool

    def __post_init__(self):
        if self.dtype not in _DTYPES:
            raise ValueError(f"unsupported column dtype {self.dtype!r}")


@dataclass(frozen=True)
class ColumnSchema:
    columns: tuple

    def __post_init__(self):
        names = [c.name for c in self.columns]
        if len(names) != len(set(names)):
            raise ValueError("duplicate column name in schema")

    def to_obj(self) -> dict:
        return {"columns": [{"name": c.name, "dtype": c.dtype, "ragged": c.ragged} for c in self.columns]}

    @classmethod
    def from_obj(cls, obj) -> "ColumnSchema":
        return cls(tuple(ColumnSpec(c["name"], c["dtype"], bool(c["ragged"])) for c in obj["columns"]))


class PackedStrings:
    """Byte strings packed columnar: ``offsets`` int64 [n+1] into ``blob``
    uint8 (numpy or CUDA tensors) — the layout ``skb_fnv1a64_strings`` hashes."""

    __slots__ = ("blob", "offsets")

    def __init__(self, blob, offsets):
        self.blob = blob
        self.offsets = offsets

    def __len__(self) -> int:
        return (int(self.offsets.numel()) if N.is_torch(self.offsets) else len(self.offsets)) - 1

    def to_objects(self) -> np.ndarray:
        """numpy object array of bytes (the reference's representation)."""
        blob = self.blob.cpu().numpy() if N.is_torch(self.blob) else np.asarray(self.blob)
        offs = (self.offsets.cpu().numpy() if N.is_torch(self.offsets) else np.asarray(self.offsets)).tolist()
        raw = blob.tobytes()
        out = np.empty(len(offs) - 1, dtype=object)
        for i in range(len(offs) - 1):
            out[i] = raw[offs[i]:offs[i + 1]]
        return out

    @classmethod
    def from_objects(cls, values) -> "PackedStrings":
        lens = np.fromiter((len(s) for s in values), count=len(values), dtype=np.int64)
        offs = np.zeros(len(values) + 1, np.int64)
        np.cumsum(lens, out=offs[1:])
        return cls(np.frombuffer(b"".join(values), np.uint8).copy(), offs)


# ---------------------------------------------------------------------------
# writer (columnio.py:127-199)
# ---------------------------------------------------------------------------

def _schema_for(data: dict) -> ColumnSchema:
    specs = []
    for name, rt in data.items():
        v = rt.values
        if isinstance(v, PackedStrings) or (isinstance(v, np.ndarray) and v.dtype == object):
            dt = "bytes"
        elif np.asarray(v).dtype == np.int64:
            dt = "int64"
        else:
            dt = "float32"
        specs.append(ColumnSpec(name, dt, True))
    return ColumnSchema(tuple(specs))


def _host(x):
    return x.cpu().numpy() if N.is_torch(x) else x


def _column_payload(spec: ColumnSpec, rt: RaggedTensor, lo: int, hi: int) -> bytes:
    offs = np.asarray(_host(rt.row_offsets), np.int64)
    e0, e1 = int(offs[lo]), int(offs[hi])
    parts = [(offs[lo:hi + 1] - e0).astype("<i8").tobytes()] if spec.ragged else []
    v = rt.values
    if spec.dtype == "bytes":
        ps = v if isinstance(v, PackedStrings) else PackedStrings.from_objects(list(v[e0:e1]))
        so = np.asarray(_host(ps.offsets), np.int64)
        if isinstance(v, PackedStrings):
            so, b0 = so[e0:e1 + 1], int(so[e0])
            blob = np.asarray(_host(ps.blob), np.uint8)[b0:int(so[-1])]
        else:
            blob = np.asarray(ps.blob, np.uint8)
        parts.append(np.diff(so).astype("<i8").tobytes())
        parts.append(blob.tobytes())
    else:
        parts.append(np.asarray(_host(v)[e0:e1], _NP[spec.dtype]).tobytes())
    return b"".join(parts)


def write_dataset(path, data: dict, chunk_rows: int, compress: bool = False,
                  schema: ColumnSchema | None = None) -> None:
    """Named ragged columns -> one dataset file in chunks of ``chunk_rows``
    rows (byte-identical to the reference writer)."""
    telemetry.bump("columnio.write_dataset")
    if chunk_rows < 1:
        raise ValueError("chunk_rows must be >= 1")
    data = {k: v if isinstance(v, RaggedTensor) else RaggedTensor.from_rows(v) for k, v in data.items()}
    schema = schema or _schema_for(data)
    names = [c.name for c in schema.columns]
    if set(names) != set(data):
        raise ValueError("schema columns do not match data columns")
    counts = {n: data[n].num_rows for n in names}
    if len(set(counts.values())) > 1:
        raise ValueError(f"row-count mismatch across columns: {counts}")
    total = counts[names[0]] if names else 0
    for spec in schema.columns:
        if not spec.ragged and np.any(np.diff(np.asarray(_host(data[spec.name].row_offsets))) != 1):
            raise ValueError(f"column {spec.name!r} declared flat but has ragged rows")
    index, payloads, pos = [], [], 0
    for lo in range(0, total, chunk_rows):
        hi = min(lo + chunk_rows, total)
        out = bytearray()
        for spec in schema.columns:
            raw = _column_payload(spec, data[spec.name], lo, hi)
            stored = raw
            if compress:
                z = zlib.compressobj(6, zlib.DEFLATED, -15)
                stored = z.compress(raw) + z.flush()
            out += bytes([1 if compress else 0]) + len(raw).to_bytes(8, "little") + len(stored).to_bytes(8, "little")
            out += stored
        payloads.append(bytes(out))
        index.append({"byte_offset": pos, "byte_len": len(out), "rows": hi - lo})
        pos += len(out)
    head = json.dumps({"schema": schema.to_obj(), "chunk_index": index}, separators=(",", ":")).encode("utf-8")
    with open(path, "wb") as f:
        f.write(MAGIC + FORMAT_VERSION.to_bytes(4, "little") + len(head).to_bytes(8, "little") + head)
        for p in payloads:
            f.write(p)


# ---------------------------------------------------------------------------
# header + shard plan (columnio.py:202-221, 306-325)
# ---------------------------------------------------------------------------

def read_header(path):
    """(schema, chunk_index, payload_start) of one dataset file."""
    with open(path, "rb") as f:
        magic = f.read(4)
        if magic != MAGIC:
            raise ColumnIOError(f"{path}: bad magic {magic!r}")
        version = int.from_bytes(f.read(4), "little")
        if version != FORMAT_VERSION:
            raise ColumnIOError(f"{path}: unsupported version {version}")
        hlen = int.from_bytes(f.read(8), "little")
        raw = f.read(hlen)
    if len(raw) != hlen:
        raise ColumnIOError(f"{path}: truncated header")
    try:
        head = json.loads(raw.decode("utf-8"))
    except (UnicodeDecodeError, json.JSONDecodeError) as e:
        raise ColumnIOError(f"{path}: invalid header JSON: {e}") from e
    return ColumnSchema.from_obj(head["schema"]), head["chunk_index"], 16 + hlen


def _plan(paths, shard_index: int, num_shards: int):
    """Schema + this shard's chunks [path_idx, abs offset, len, rows, chunk idx]."""
    if num_shards < 1 or not 0 <= shard_index < num_shards:
        raise ValueError(f"invalid shard {shard_index}/{num_shards}")
    schema, owned, g = None, [], 0
    for pi, path in enumerate(paths):
        s, index, start = read_header(path)
        if schema is None:
            schema = s
        elif s != schema:
            raise ColumnIOError(f"{path}: schema differs from first file")
        for j, meta in enumerate(index):
            if g % num_shards == shard_index:
                owned.append((pi, start + meta["byte_offset"], meta["byte_len"], meta["rows"], j))
            g += 1
    if schema is None:
        raise ColumnIOError("no input files")
    return schema, np.asarray(owned, np.int64).reshape(-1, 5)


# ---------------------------------------------------------------------------
# reader (columnio.py:328-409)
# ---------------------------------------------------------------------------

def _view(ptr: int, dtype, n: int) -> np.ndarray:
    if n == 0:
        return np.empty(0, dtype)
    buf = (ctypes.c_uint8 * (n * np.dtype(dtype).itemsize)).from_address(ptr)
    return np.frombuffer(buf, dtype=dtype, count=n)


class _NativeReader:
    def __init__(self, paths, chunks, schema, selected, batch_rows, depth, threads, pinned, device):
        self.lib = N.host_lib()
        self.paths = [os.fsencode(p) for p in paths]
        cols = schema.columns
        self.names_b = [c.name.encode("utf-8") for c in cols]
        arr = lambda t, xs: (t * max(len(xs), 1))(*xs)  # noqa: E731
        self._keep = (arr(ctypes.c_char_p, self.paths), np.ascontiguousarray(chunks, np.int64),
                      arr(ctypes.c_char_p, self.names_b), arr(ctypes.c_int32, [_CODE[c.dtype] for c in cols]),
                      arr(ctypes.c_int32, [int(c.ragged) for c in cols]),
                      arr(ctypes.c_int32, [int(c.name in selected) for c in cols]))
        h = ctypes.c_void_p()
        st = self.lib.skb_reader_open(ctypes.cast(self._keep[0], ctypes.c_void_p), len(self.paths),
                                      self._keep[1].ctypes.data, len(chunks),
                                      ctypes.cast(self._keep[2], ctypes.c_void_p),
                                      ctypes.cast(self._keep[3], ctypes.c_void_p),
                                      ctypes.cast(self._keep[4], ctypes.c_void_p),
                                      ctypes.cast(self._keep[5], ctypes.c_void_p), len(cols), batch_rows, depth,
                                      threads, int(pinned), int(device), ctypes.byref(h))
        self._check(st)
        self.h = h

    def _check(self, st):
        if st == N.SKB_OK:
            return
        msg = self.lib.skb_last_error().decode("utf-8", "replace")
        raise ColumnIOError(msg) if st == N.SKB_E_IO else ValueError(msg)

    def next(self) -> int:
        rows = ctypes.c_int64()
        self._check(self.lib.skb_reader_next(self.h, ctypes.byref(rows)))
        return rows.value

    def column(self, j: int, rows: int, dtype: str):
        """numpy VIEWS of the current batch's buffers (valid until next())."""
        ro, vals, strs = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        nv, nb = ctypes.c_int64(), ctypes.c_int64()
        self._check(self.lib.skb_reader_column(self.h, j, ctypes.byref(ro), ctypes.byref(vals), ctypes.byref(nv),
                                               ctypes.byref(strs), ctypes.byref(nb)))
        offs = _view(ro.value, np.int64, rows + 1)
        if dtype == "bytes":
            return offs, PackedStrings(_view(vals.value, np.uint8, nb.value), _view(strs.value, np.int64, nv.value + 1))
        return offs, _view(vals.value, _NP[dtype], nv.value)

    def close(self):
        if getattr(self, "h", None):
            self.lib.skb_reader_close(self.h)
            self.h = None

    __del__ = close


def open_reader(paths, shard_index: int = 0, num_shards: int = 1, batch_rows: int = 256, prefetch_depth: int = 0,
                columns=None, *, device=None, threads: int | None = None, packed_strings: bool = False):
    """Iterate name -> RaggedTensor batches over this shard's chunks
    (columnio.py:328-376).  Output never depends on prefetch_depth / threads.

    device=None: numpy batches as the reference yields them (byte strings as
    object arrays; ``packed_strings=True`` keeps them packed).
    device="cuda" (or a torch device): every column lands in device memory
    through one async H2D copy from page-locked buffers; byte strings as
    :class:`PackedStrings` of device tensors.
    """
    if isinstance(paths, (str, bytes, os.PathLike)):
        paths = [paths]
    paths = [os.fspath(p) for p in paths]
    if batch_rows < 1:
        raise ValueError("batch_rows must be >= 1")
    schema, chunks = _plan(paths, shard_index, num_shards)
    select = set(columns) if columns is not None else None
    if select is not None:
        missing = select - {c.name for c in schema.columns}
        if missing:
            raise ColumnIOError(f"unknown columns requested: {sorted(missing)}")
    specs = [c for c in schema.columns if select is None or c.name in select]
    nthreads = threads or max(1, min(8, os.cpu_count() or 1))
    dev = None
    if device is not None:
        import torch
        dev = torch.device(device)
        if dev.type != "cuda":
            raise ValueError("device must be a CUDA device (or None for numpy batches)")
        N.lib()  # fails loudly without a GPU / the built library
    reader = _NativeReader(paths, chunks, schema, {c.name for c in specs}, batch_rows, max(1, prefetch_depth),
                           nthreads, dev is not None, dev.index if dev is not None and dev.index is not None else
                           (N.torch().cuda.current_device() if dev is not None else 0))
    return _batches(reader, specs, dev, packed_strings)


def _batches(reader, specs, dev, packed_strings):
    torch = N.torch() if dev is not None else None
    stream = torch.cuda.Stream(device=dev) if dev is not None else None
    done = None
    try:
        while True:
            if done is not None:
                done.synchronize()  # the previous batch's copies left the recycled buffers
            rows = reader.next()
            if rows == 0:
                return
            batch = {}
            if dev is None:
                for j, spec in enumerate(specs):
                    offs, vals = reader.column(j, rows, spec.dtype)
                    if spec.dtype == "bytes":
                        copy = PackedStrings(vals.blob.copy(), vals.offsets.copy())
                        vals = copy if packed_strings else copy.to_objects()
                    else:
                        vals = vals.copy()
                    batch[spec.name] = RaggedTensor._trusted(vals, offs.copy())
            else:
                with torch.cuda.stream(stream):
                    for j, spec in enumerate(specs):
                        offs, vals = reader.column(j, rows, spec.dtype)
                        o = torch.from_numpy(offs).to(dev, non_blocking=True)
                        if spec.dtype == "bytes":
                            v = PackedStrings(torch.from_numpy(vals.blob).to(dev, non_blocking=True),
                                              torch.from_numpy(vals.offsets).to(dev, non_blocking=True))
                        else:
                            v = torch.from_numpy(vals).to(dev, non_blocking=True)
                        batch[spec.name] = RaggedTensor._trusted(v, o)
                    done = torch.cuda.Event()
                    done.record(stream)
                # consumers on the current stream see the copies
                torch.cuda.current_stream(dev).wait_stream(stream)
            telemetry.bump("columnio.batch")
            yield batch
    finally:
        reader.close()
