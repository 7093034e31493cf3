"""Golden columnar datasets + reader batches from the REFERENCE (build container only).

Usage:  python tests/golden/make_golden_columnio.py
Writes, through the reference's own `write_dataset` / `open_reader`
(columnio.py:146-199, 328-376; alias `sparsekit_ref` of the read-only tree):
  tests/golden/cio/data{0,1}.rcol      two files (plain, compressed), 3 columns
  tests/golden/cio_batches.npz         the batches of several reader configs,
                                       byte strings packed as (blob, offsets)
Nothing on the GPU box reads /root/reference.
"""

from __future__ import annotations

import os
import shutil
import sys

import numpy as np

sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import load_ref  # noqa: E402

OUT = os.path.join(HERE, "cio")
NPZ = os.path.join(HERE, "cio_batches.npz")
# (shard_index, num_shards, batch_rows, columns) configurations of open_reader
CONFIGS = [(0, 1, 7, None), (1, 3, 5, None), (0, 2, 64, ("tags", "price")), (2, 3, 1, ("uid",)),
           (0, 1, 1000, None)]


def make_columns(rng, rows):
    """price: ragged float32, uid: flat int64, tags: ragged byte strings
    (empty rows, empty strings, non-ASCII bytes)."""
    plen = rng.integers(0, 4, rows)
    price = [rng.random(int(k), dtype=np.float32).tolist() for k in plen]
    uid = [[int(x)] for x in rng.integers(-(2**62), 2**62, rows)]
    tags = []
    for _ in range(rows):
        k = int(rng.integers(0, 3))
        tags.append([bytes(rng.integers(0, 256, int(rng.integers(0, 6)), dtype=np.uint8)) for _ in range(k)])
    return price, uid, tags


def pack(values):
    lens = np.fromiter((len(s) for s in values), count=len(values), dtype=np.int64)
    offs = np.zeros(len(values) + 1, np.int64)
    np.cumsum(lens, out=offs[1:])
    return np.frombuffer(b"".join(values), np.uint8).copy(), offs


def main():
    ref = load_ref()
    from sparsekit_ref import columnio as CIO
    from sparsekit_ref.ragged import RaggedTensor
    rng = np.random.Generator(np.random.PCG64(99))
    if os.path.exists(OUT):
        shutil.rmtree(OUT)
    os.makedirs(OUT)
    schema = CIO.ColumnSchema((CIO.ColumnSpec("price", "float32", True), CIO.ColumnSpec("uid", "int64", False),
                               CIO.ColumnSpec("tags", "bytes", True)))
    g = {}
    paths = []
    for i, (rows, chunk, comp) in enumerate(((53, 8, False), (37, 5, True))):
        price, uid, tags = make_columns(rng, rows)
        data = {"price": RaggedTensor.from_rows(price, dtype=np.float32),
                "uid": RaggedTensor.from_rows(uid, dtype=np.int64),
                "tags": RaggedTensor.from_rows(tags)}
        p = os.path.join(OUT, f"data{i}.rcol")
        CIO.write_dataset(p, data, chunk, compress=comp, schema=schema)
        paths.append(p)
        # the writer's inputs, so this repo's writer can be checked byte for byte
        for name in ("price", "uid"):
            g[f"in{i}.{name}.values"] = data[name].values
            g[f"in{i}.{name}.offsets"] = data[name].row_offsets
        blob, so = pack(list(data["tags"].values))
        g[f"in{i}.tags.blob"], g[f"in{i}.tags.str_offsets"] = blob, so
        g[f"in{i}.tags.offsets"] = data["tags"].row_offsets
    for c, (si, ns, br, cols) in enumerate(CONFIGS):
        for b, batch in enumerate(CIO.open_reader(paths, si, ns, br, prefetch_depth=2, columns=cols)):
            for name, rt in batch.items():
                key = f"cfg{c}.b{b}.{name}"
                g[key + ".offsets"] = rt.row_offsets
                if rt.values.dtype == object:
                    g[key + ".blob"], g[key + ".str_offsets"] = pack(list(rt.values))
                else:
                    g[key + ".values"] = rt.values
            g[f"cfg{c}.nbatches"] = np.array(b + 1)
    np.savez_compressed(NPZ, **g)
    print("wrote", sorted(os.listdir(OUT)), NPZ, len(g))


if __name__ == "__main__":
    main()
