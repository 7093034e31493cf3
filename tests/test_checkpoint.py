"""Checkpoint boundary (reference checkpoint.py): SafeTensors bytes, manifest,
resharding on load.  Pinned by the reference's own checkpoint written by
tests/golden/make_golden_ckpt.py (tests/golden/ckpt*)."""

from __future__ import annotations

import os
import shutil

import numpy as np
import pytest

from oracle import sparse_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden", "ckpt")
RESAVED = os.path.join(HERE, "golden", "ckpt_resaved")
STEPS, EVICT_AT, NUM_FILES, GLOBAL_STEP = 6, 4, 3, 6
ADAM = dict(lr=1e-2, weight_decay=0.01, variant="adamw")


def trace():
    return np.load(os.path.join(HERE, "golden", "ckpt_trace.npz"))


def golden_bytes(d=GOLD):
    return {f: open(os.path.join(d, f), "rb").read() for f in sorted(os.listdir(d))}


def dir_bytes(d):
    return {f: open(os.path.join(d, f), "rb").read() for f in sorted(os.listdir(d))}


def replay_oracle():
    tr = trace()
    lt = O.OracleLogical("dim8", 8, 4, seed=5, members=["u", "i"], namespaced=True, evict_threshold=2)
    plain = O.OracleTable(4, seed=9, block_size=16, evict_threshold=2)
    for step in range(1, STEPS + 1):
        keys = np.concatenate([lt.keys_for("u", tr[f"{step}.u"]), lt.keys_for("i", tr[f"{step}.i"])])
        O.lookup(lt, keys, step)
        O.grad_update(lt, keys, tr[f"{step}.dim8.grads"], step, **ADAM)
        offs = plain.lookup_or_insert(tr[f"{step}.plain4.ids"], step)
        O.sparse_adam(plain, offs, tr[f"{step}.plain4.grads"], t=step, **ADAM)
        if step == EVICT_AT:
            lt.evict(step)
            plain.evict(step)
    return lt, plain


# ---- CPU: oracle + host container logic --------------------------------------

def test_oracle_checkpoint_bytes_match_reference():
    lt, plain = replay_oracle()
    files = O.checkpoint_files([("dim8", lt.shards, lt.members, True), ("plain4", [plain], [], False)],
                               NUM_FILES, GLOBAL_STEP)
    assert files == golden_bytes()


def test_container_round_trip_bytes(tmp_path):
    from paper_2509_20883_b200 import checkpoint as C
    for f, raw in golden_bytes().items():
        if not f.endswith(".safetensors"):
            continue
        t = C.read_safetensors(os.path.join(GOLD, f))
        C.write_safetensors(tmp_path / f, t)
        assert (tmp_path / f).read_bytes() == raw
        assert O.safetensors_bytes(t) == raw
    man = C.read_manifest(GOLD)
    assert man.to_json() == open(os.path.join(GOLD, "manifest.json")).read()
    assert C.inspect_checkpoint(GOLD) == open(os.path.join(HERE, "golden", "ckpt_inspect.txt")).read()


def test_container_metadata_and_errors(tmp_path):
    from paper_2509_20883_b200 import checkpoint as C
    p = tmp_path / "a.safetensors"
    C.write_safetensors(p, {"z": np.arange(3, dtype=np.int64), "a": np.ones((2, 2), np.float32)},
                        metadata={"step": 3, "b": "x"})
    assert C.read_safetensors_metadata(p) == {"b": "x", "step": "3"}
    t = C.read_safetensors(p)
    assert t["z"].tolist() == [0, 1, 2] and t["a"].shape == (2, 2)
    t["a"][0, 0] = 5.0  # arrays are writable
    with pytest.raises(C.CheckpointError, match="unsupported tensor dtype"):
        C.write_safetensors(tmp_path / "b.safetensors", {"x": np.zeros(2, np.int32)})
    raw = p.read_bytes()
    (tmp_path / "t1.safetensors").write_bytes(raw[:5])
    with pytest.raises(C.CheckpointError, match="truncated header length"):
        C.read_safetensors(tmp_path / "t1.safetensors")
    (tmp_path / "t2.safetensors").write_bytes(raw[:20])
    with pytest.raises(C.CheckpointError, match="truncated header JSON"):
        C.read_safetensors(tmp_path / "t2.safetensors")
    (tmp_path / "t3.safetensors").write_bytes(raw[:-4])
    with pytest.raises(C.CheckpointError, match="bad data_offsets"):
        C.read_safetensors(tmp_path / "t3.safetensors")
    with pytest.raises(C.CheckpointError, match="missing manifest.json"):
        C.read_manifest(tmp_path)
    d = tmp_path / "ck"
    shutil.copytree(GOLD, d)
    txt = (d / "manifest.json").read_text().replace('"version": 1', '"version": 2')
    (d / "manifest.json").write_text(txt)
    with pytest.raises(C.CheckpointError, match="unknown checkpoint format version 2"):
        C.read_manifest(d)


def test_split_counts_and_names():
    from paper_2509_20883_b200 import checkpoint as C
    assert C._split_counts(10, 3) == [4, 3, 3] and C._split_counts(0, 2) == [0, 0]
    assert C._file_names(2) == ["ckpt-00000-of-00002.safetensors", "ckpt-00001-of-00002.safetensors"]


# ---- GPU: the device export / merge / reshard path ----------------------------

def replay_gpu(skb):
    tr = trace()
    cfg = skb.AdamConfig(**ADAM)
    lt = skb.LogicalTable("dim8", 8, 4, seed=5, members=["u", "i"], namespaced=True, evict_threshold=2)
    plain = skb.EmbeddingTable("plain4", 4, seed=9, block_size=16, evict_threshold=2)
    plan = skb.ShardPlan(4)
    for step in range(1, STEPS + 1):
        keys = np.concatenate([lt.keys_for("u", tr[f"{step}.u"]), lt.keys_for("i", tr[f"{step}.i"])])
        skb.all_to_all_lookup(lt, keys, plan, step)
        skb.all_to_all_grad_update(lt, keys, tr[f"{step}.dim8.grads"], plan, cfg, step)
        offs = plain.lookup_or_insert(tr[f"{step}.plain4.ids"], step)
        skb.sparse_adam_step(plain.store, offs, tr[f"{step}.plain4.grads"], cfg, step)
        if step == EVICT_AT:
            lt.evict(step)
            plain.evict(step)
    return lt, plain


@pytest.mark.gpu
def test_save_sharded_bytes_match_reference(skb, tmp_path):
    lt, plain = replay_gpu(skb)
    man = skb.save_sharded([lt, plain], tmp_path / "ck", NUM_FILES, global_step=GLOBAL_STEP)
    assert dir_bytes(tmp_path / "ck") == golden_bytes()
    assert [t.rows_per_file for t in man.tables] == [[70, 70, 70], [25, 25, 24]]
    with pytest.raises(ValueError, match="duplicate table name"):
        skb.save_sharded([lt, lt], tmp_path / "x", 1)
    with pytest.raises(ValueError):
        skb.save_sharded([lt], tmp_path / "x", 0)


@pytest.mark.gpu
@pytest.mark.parametrize("S", [1, 2, 3, 4, 8])
def test_load_sharded_reshards_bit_exact(skb, tmp_path, S):
    from paper_2509_20883_b200 import checkpoint as C
    tabs = skb.load_sharded(GOLD, S)
    gold = {}
    for f in sorted(os.listdir(GOLD)):
        if f.endswith(".safetensors"):
            for k, a in C.read_safetensors(os.path.join(GOLD, f)).items():
                gold.setdefault(k, []).append(a)
    for lt in tabs:
        assert lt.num_shards == S
        ex = [sh.export_rows() for sh in lt.shards]
        ids = np.concatenate([e[0] for e in ex])
        o = np.argsort(ids)
        for j, part in enumerate(("ids", "weight", "m", "v", "last_step")):
            got = np.concatenate([e[j] for e in ex])[o]
            want = np.concatenate(gold[f"{lt.name}.{part}"])
            assert np.array_equal(got.view(np.uint8), want.view(np.uint8)), (lt.name, part)
        # every row lives on its owner shard of the target plan
        for s, e in enumerate(ex):
            assert (O.owner_of(e[0], S) == s).all()
    # the reference's own round trip (load under 2, save to 2 files) bit-matches
    if S == 2:
        skb.save_sharded(tabs, tmp_path / "re", 2, global_step=GLOBAL_STEP + 1)
        assert dir_bytes(tmp_path / "re") == golden_bytes(RESAVED)


@pytest.mark.gpu
def test_load_then_train_matches_oracle(skb):
    """After a 3-shard load, the next lookups / updates equal the oracle's
    tables restored from the same checkpoint (free lists start empty)."""
    tabs = skb.load_sharded(GOLD, 3)
    lt = tabs[0]
    olt = O.OracleLogical("dim8", 8, 3, seed=5, members=["u", "i"], namespaced=True, evict_threshold=2)
    from paper_2509_20883_b200 import checkpoint as C
    cols = {}
    for f in sorted(os.listdir(GOLD)):
        if f.endswith(".safetensors"):
            for k, a in C.read_safetensors(os.path.join(GOLD, f)).items():
                cols.setdefault(k, []).append(a)
    ids = np.concatenate(cols["dim8.ids"])
    own = O.owner_of(ids, 3)
    for s in range(3):
        sel = own == s
        olt.shards[s].restore_rows(*(np.concatenate(cols[f"dim8.{p}"])[sel]
                                     for p in ("ids", "weight", "m", "v", "last_step")))
    rng = np.random.default_rng(3)
    cfg = skb.AdamConfig(**ADAM)
    plan = skb.ShardPlan(3)
    for step in (7, 8):
        keys = np.concatenate([lt.keys_for("u", rng.zipf(1.3, 50).astype(np.int64)),
                               lt.keys_for("i", rng.integers(0, 40, 20))])
        rows = skb.all_to_all_lookup(lt, keys, plan, step)
        want = O.lookup(olt, keys, step)
        assert np.array_equal(np.asarray(rows).view(np.int32), want.view(np.int32))
        g = (rng.standard_normal((len(keys), 8)) * 0.05).astype(np.float32)
        skb.all_to_all_grad_update(lt, keys, g, plan, cfg, step)
        O.grad_update(olt, keys, g, step, **ADAM)
    for s in range(3):
        a, b = lt.shards[s].export_rows(), olt.shards[s].export_rows()
        for x, y in zip(a, b):
            assert np.array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8))


@pytest.mark.gpu
def test_save_empty_and_single_file(skb, tmp_path):
    t = skb.EmbeddingTable("e", 4)
    man = skb.save_sharded([t], tmp_path / "e", 2)
    assert man.tables[0].rows_per_file == [0, 0]
    back = skb.load_sharded(tmp_path / "e", 3)
    assert back[0].num_rows == 0
    lt = skb.LogicalTable("dim4", 4, 2, seed=1)
    lt.shards[0].lookup_or_insert(np.array([5, -3], np.int64), 1)
    lt.shards[1].lookup_or_insert(np.array([2**62, -(2**63)], np.int64), 2)
    skb.save_sharded([lt], tmp_path / "one", 1, global_step=2)
    t1 = O.OracleTable(4, seed=1)
    t1.lookup_or_insert(np.array([5, -3], np.int64), 1)
    t2 = O.OracleTable(4, seed=1)
    t2.lookup_or_insert(np.array([2**62, -(2**63)], np.int64), 2)
    assert dir_bytes(tmp_path / "one") == O.checkpoint_files([("dim4", [t1, t2], ["dim4"], False)], 1, 2)


def _free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _dist_ckpt_worker(rank, port, out_dir):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    torch.cuda.set_device(0)
    import paper_2509_20883_b200 as skb
    tabs = skb.load_sharded(GOLD, 2, dist=True)
    for lt in tabs:
        ids = lt.local_table.export_rows()[0]
        assert (O.owner_of(ids, 2) == rank).all()
    man = skb.save_sharded(tabs, os.path.join(out_dir, "re"), 2, global_step=GLOBAL_STEP + 1)
    with open(os.path.join(out_dir, f"man{rank}.json"), "w") as f:
        f.write(man.to_json())
    dist.destroy_process_group()


@pytest.mark.gpu
def test_dist_load_save_round_trip(cuda, tmp_path):
    """One shard per rank (2 ranks on one GPU, gloo): load_sharded(dist=True)
    keeps each rank's own rows; save_sharded gathers to rank 0 and writes the
    reference's round-trip bytes; every rank returns the same manifest."""
    import torch.multiprocessing as mp
    mp.spawn(_dist_ckpt_worker, args=(_free_port(), str(tmp_path)), nprocs=2, join=True)
    assert dir_bytes(tmp_path / "re") == golden_bytes(RESAVED)
    assert (tmp_path / "man0.json").read_text() == (tmp_path / "man1.json").read_text() == \
        open(os.path.join(RESAVED, "manifest.json")).read()
