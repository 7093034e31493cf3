"""Input side (reference columnio.py): file bytes, shard plans, batching,
errors; the native reader against batches the reference produced
(tests/golden/make_golden_columnio.py)."""

from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import sparse_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
CIO = os.path.join(HERE, "golden", "cio")
PATHS = [os.path.join(CIO, "data0.rcol"), os.path.join(CIO, "data1.rcol")]
CONFIGS = [(0, 1, 7, None), (1, 3, 5, None), (0, 2, 64, ("tags", "price")), (2, 3, 1, ("uid",)),
           (0, 1, 1000, None)]


@pytest.fixture(scope="module")
def gold():
    with np.load(os.path.join(HERE, "golden", "cio_batches.npz")) as z:
        return {k: z[k] for k in z.files}


def _inputs(g, i):
    from paper_2509_20883_b200 import RaggedTensor
    from paper_2509_20883_b200.columnio import PackedStrings
    return {"price": RaggedTensor(g[f"in{i}.price.values"], g[f"in{i}.price.offsets"]),
            "uid": RaggedTensor(g[f"in{i}.uid.values"], g[f"in{i}.uid.offsets"]),
            "tags": RaggedTensor._trusted(PackedStrings(g[f"in{i}.tags.blob"], g[f"in{i}.tags.str_offsets"]),
                                          g[f"in{i}.tags.offsets"])}


def _schema():
    from paper_2509_20883_b200.columnio import ColumnSchema, ColumnSpec
    return ColumnSchema((ColumnSpec("price", "float32", True), ColumnSpec("uid", "int64", False),
                         ColumnSpec("tags", "bytes", True)))


def _check_batches(g, c, batches, packed_device=False):
    assert len(batches) == int(g[f"cfg{c}.nbatches"])
    for b, batch in enumerate(batches):
        names = sorted(k.split(".")[2] for k in g if k.startswith(f"cfg{c}.b{b}.") and k.endswith(".offsets")
                       and ".str_offsets" not in k)
        assert sorted(batch) == names
        for name, rt in batch.items():
            key = f"cfg{c}.b{b}.{name}"
            offs = rt.row_offsets.cpu().numpy() if hasattr(rt.row_offsets, "cpu") else rt.row_offsets
            assert np.array_equal(offs, g[key + ".offsets"])
            v = rt.values
            if key + ".blob" in g:
                if hasattr(v, "blob"):
                    blob = v.blob.cpu().numpy() if hasattr(v.blob, "cpu") else v.blob
                    so = v.offsets.cpu().numpy() if hasattr(v.offsets, "cpu") else v.offsets
                else:
                    blob, so = np.frombuffer(b"".join(v), np.uint8), \
                        np.concatenate([[0], np.cumsum([len(s) for s in v])]).astype(np.int64)
                assert np.array_equal(blob, g[key + ".blob"]) and np.array_equal(so, g[key + ".str_offsets"])
            else:
                v = v.cpu().numpy() if hasattr(v, "cpu") else v
                assert v.dtype == g[key + ".values"].dtype
                assert np.array_equal(v.view(np.uint8), g[key + ".values"].view(np.uint8))


# ---- CPU: writer bytes, native reader in numpy mode, errors --------------------

def test_write_dataset_matches_reference_bytes(gold, tmp_path):
    from paper_2509_20883_b200.columnio import write_dataset
    for i, (chunk, comp) in enumerate(((8, False), (5, True))):
        p = tmp_path / f"d{i}.rcol"
        write_dataset(p, _inputs(gold, i), chunk, compress=comp, schema=_schema())
        assert p.read_bytes() == open(PATHS[i], "rb").read()


@pytest.mark.parametrize("c", range(len(CONFIGS)))
@pytest.mark.parametrize("threads,depth", [(1, 0), (4, 3)])
def test_reader_batches_match_reference(gold, c, threads, depth):
    from paper_2509_20883_b200.columnio import open_reader
    si, ns, br, cols = CONFIGS[c]
    batches = list(open_reader(PATHS, si, ns, br, prefetch_depth=depth, columns=cols, threads=threads))
    _check_batches(gold, c, batches)
    for b in batches:
        if "tags" in b:
            assert b["tags"].values.dtype == object  # drop-in: byte strings as objects


def test_reader_packed_strings_and_shards_partition(gold):
    from paper_2509_20883_b200.columnio import open_reader
    batches = list(open_reader(PATHS, 0, 1, 1000, packed_strings=True))
    _check_batches(gold, 4, batches)
    # shards are disjoint and jointly exhaustive (row multiset of uid)
    allu = np.concatenate([b["uid"].values for b in batches])
    parts = [np.concatenate([b["uid"].values for b in open_reader(PATHS, s, 3, 4)]) for s in range(3)]
    assert sorted(np.concatenate(parts).tolist()) == sorted(allu.tolist())


def test_reader_errors(tmp_path):
    from paper_2509_20883_b200.columnio import ColumnIOError, open_reader, read_header
    raw = open(PATHS[1], "rb").read()
    (tmp_path / "bad.rcol").write_bytes(b"XCOL" + raw[4:])
    with pytest.raises(ColumnIOError, match="bad magic"):
        read_header(tmp_path / "bad.rcol")
    with pytest.raises(ColumnIOError, match="unknown columns requested"):
        open_reader(PATHS, columns=["nope"])
    with pytest.raises(ValueError, match="invalid shard"):
        open_reader(PATHS, 3, 3)
    with pytest.raises(ColumnIOError, match="no input files"):
        open_reader([])
    (tmp_path / "trunc.rcol").write_bytes(raw[:-10])
    with pytest.raises(ColumnIOError, match=r"chunk \d+: truncated chunk"):
        list(open_reader([tmp_path / "trunc.rcol"], batch_rows=4))
    # corrupt the DEFLATE stream of the first compressed column
    _, index, start = read_header(PATHS[1])
    b = bytearray(raw)
    for k in range(start + 17, start + 17 + 6):
        b[k] ^= 0xFF
    (tmp_path / "z.rcol").write_bytes(bytes(b))
    with pytest.raises(ColumnIOError, match=r"z\.rcol: chunk 0: column 'price': "):
        list(open_reader([tmp_path / "z.rcol"], batch_rows=4))


def test_oracle_hash_of_reader_strings(gold):
    """hash_feature's reference values for the reader's byte strings (oracle)."""
    from paper_2509_20883_b200.columnio import open_reader
    b = next(iter(open_reader(PATHS, 0, 1, 1000, packed_strings=True)))
    ps = b["tags"].values
    objs = ps.to_objects()
    assert len(objs) == len(ps)
    assert np.array_equal(O.hash_strings(objs), O.hash_strings(list(objs)))


# ---- GPU: device batches + hashing on the packed layout -------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("c", range(len(CONFIGS)))
def test_reader_device_batches(gold, skb, c):
    si, ns, br, cols = CONFIGS[c]
    batches = []
    for b in skb.open_reader(PATHS, si, ns, br, prefetch_depth=2, columns=cols, device="cuda"):
        for rt in b.values():
            v = rt.values.blob if hasattr(rt.values, "blob") else rt.values
            assert v.is_cuda and rt.row_offsets.is_cuda
        # keep host copies: the next batch may reuse the reader's buffers
        batches.append({k: skb.RaggedTensor._trusted(
            v.values if not hasattr(v.values, "blob") else type(v.values)(v.values.blob.clone(),
                                                                           v.values.offsets.clone()),
            v.row_offsets.clone()) for k, v in b.items()})
    _check_batches(gold, c, batches)


@pytest.mark.gpu
def test_hash_feature_on_device_packed_strings(skb):
    b = next(iter(skb.open_reader(PATHS, 0, 1, 1000, columns=["tags"], device="cuda")))
    h = skb.hash_feature(b["tags"])
    want = O.hash_strings(b["tags"].values.to_objects())
    assert np.array_equal(h.values.cpu().numpy(), want)
    assert np.array_equal(h.row_offsets.cpu().numpy(), b["tags"].row_offsets.cpu().numpy())
