"""Generate golden fixtures by running the REFERENCE itself (build container only).

Usage:  python tests/golden/make_golden.py
Imports /root/reference/pkg/src/sparsekit under the alias `sparsekit_ref`
(read-only tree; bytecode writing disabled), runs seeded cases through the
reference's own public API, and writes tests/golden/golden.npz.  The fixture
travels with the repo; nothing on the GPU box reads /root/reference.
"""

from __future__ import annotations

import importlib.util
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src/sparsekit"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
OUT2 = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_edges.npz")


def load_ref():
    spec = importlib.util.spec_from_file_location(
        "sparsekit_ref", os.path.join(REF, "__init__.py"), submodule_search_locations=[REF])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["sparsekit_ref"] = mod
    spec.loader.exec_module(mod)
    return mod


EDGE_IDS = np.array([0, 1, -1, 2, 42, 7, 2**62, -(2**62), 2**63 - 1, -(2**63), 123456789,
                     -987654321, 1 << 40, (1 << 40) + 1], dtype=np.int64)


def main():
    ref = load_ref()
    from sparsekit_ref import hashing as H, sharding as SH, segments as SG, features as FE
    from sparsekit_ref import embedding as EM, optim as OP, ragged as RG
    rng = np.random.Generator(np.random.PCG64(2024))
    g = {}

    # --- hashing -------------------------------------------------------------
    ids = np.concatenate([EDGE_IDS, rng.integers(-(2**63), 2**63 - 1, 500, dtype=np.int64, endpoint=True)])
    g["hash.ids"] = ids
    g["hash.mix64"] = H.mix64(ids).view(np.int64)
    for S in (1, 2, 3, 8, 13):
        g[f"hash.shard_of.S{S}"] = SH.ShardPlan(S).shard_of(ids)
    lt = SH.LogicalTable("dimx", 8, 1, members=["C0", "user_id", "ünï"], namespaced=True)
    for m in lt.members:
        g[f"hash.keys_for.{m}"] = lt.keys_for(m, ids)
    strs = [b"", b"a", b"b", b"abc", b"hello world", bytes(range(256)), "ünïcode".encode()] + \
        [bytes(rng.integers(0, 256, rng.integers(0, 40), dtype=np.uint8)) for _ in range(200)]
    g["fnv.blob"] = np.frombuffer(b"".join(strs), np.uint8)
    g["fnv.offs"] = np.concatenate([[0], np.cumsum([len(s) for s in strs])]).astype(np.int64)
    g["fnv.hash"] = H.fnv1a64_batch(strs).view(np.int64)
    px, py = ids[:200], ids[200:400]
    g["fnv.pairs.x"], g["fnv.pairs.y"] = px, py
    g["fnv.pairs.h"] = H.fnv1a64_pairs(px, py).view(np.int64)

    # --- initial rows ----------------------------------------------------------
    for seed, dim in ((0, 16), (7, 64), (-3, 8), (2**40 + 5, 3), (123, 128)):
        g[f"init.{seed}.{dim}"] = EM.initial_rows(seed, ids, dim)

    # --- unique_partition --------------------------------------------------------
    cases = {
        "rand": rng.integers(0, 50, 300),
        "wide": rng.integers(-(2**63), 2**63 - 1, 300, dtype=np.int64, endpoint=True),
        "dups": np.full(40, 9, np.int64),
        "edge": np.concatenate([EDGE_IDS, EDGE_IDS[::-1], EDGE_IDS]),
        "spec": np.array([8, 3, 8, 16], np.int64),
        "empty": np.empty(0, np.int64),
        "zipf": rng.zipf(1.1, 2000).astype(np.int64),
    }
    for name, x in cases.items():
        for S in (1, 2, 8):
            pr = SH.unique_partition(x, SH.ShardPlan(S))
            g[f"part.{name}.ids"] = np.asarray(x, np.int64)
            g[f"part.{name}.S{S}.uniq"] = np.concatenate(pr.shard_ids) if S else pr.shard_ids
            g[f"part.{name}.S{S}.counts"] = np.array([len(s) for s in pr.shard_ids], np.int64)
            g[f"part.{name}.S{S}.inv_shard"] = pr.inverse_shard
            g[f"part.{name}.S{S}.inv_pos"] = pr.inverse_pos
            st = SH.load_stats(x, SH.ShardPlan(S))
            g[f"part.{name}.S{S}.load_counts"] = st.counts
            g[f"part.{name}.S{S}.imbalance"] = np.float64(st.imbalance)

    # --- table trace (SURVEY A.6 trace + random ops) ----------------------------------
    t = EM.EmbeddingTable("t", 4, seed=11, block_size=4, evict_threshold=5)
    trace = []

    def rec(tag, arr):
        trace.append(tag)
        g[f"table.trace.{len(trace) - 1}"] = np.asarray(arr)

    rec("lookup", t.lookup_or_insert([10, 20, 30], 1))
    rec("evict", [t.evict(10)])
    rec("lookup", t.lookup_or_insert([40, 50], 11))
    rec("lookup", t.lookup_or_insert([10], 12))
    rec("evict", [t.evict(30)])
    rec("lookup", t.lookup_or_insert([60, 70, 80, 90], 31))
    rec("lookup", t.lookup_or_insert([60], 36))
    rec("evict", [t.evict(40)])
    rec("lookup", t.lookup_or_insert([-5, 2**63 - 1, -(2**63), 70], 41))
    rec("gather", t.gather(t.lookup_or_insert([-5, 60], 41)))
    t.scatter_update(t.lookup_or_insert([60], 41), np.arange(4, dtype=np.float32)[None, :])
    rec("gather", t.gather(t.lookup_or_insert([60, -5], 42)))
    ex = t.export_rows()
    for k, a in zip(("ids", "w", "m", "v", "last"), ex):
        g[f"table.export.{k}"] = a
    g["table.capacity"] = np.int64(t.store.capacity)
    g["table.num_rows"] = np.int64(t.num_rows)
    g["table.free_list"] = np.asarray(t.idmap.free_list, np.int64)
    g["table.trace_kinds"] = np.array(trace)
    # restore into a fresh table with a pre-existing free list
    t2 = EM.EmbeddingTable("t2", 4, seed=11, block_size=4, evict_threshold=1)
    t2.lookup_or_insert([1, 2, 3, 4, 5], 1)
    t2.lookup_or_insert([3], 5)
    t2.evict(5)
    t2.restore_rows(*ex)
    g["table.restore.offsets"] = t2.lookup_or_insert(ex[0], 50)
    g["table.restore.free_list"] = np.asarray(t2.idmap.free_list, np.int64)

    # random model-based sequence (ids from small space, periodic evictions)
    t3 = EM.EmbeddingTable("t3", 8, seed=5, block_size=16, evict_threshold=3)
    rs = np.random.Generator(np.random.PCG64(77))
    seq_ids, seq_offs, seq_ev = [], [], []
    for step in range(1, 41):
        u = np.unique(rs.integers(0, 60, rs.integers(0, 25)))
        u = rs.permutation(u)
        seq_ids.append(u)
        seq_offs.append(t3.lookup_or_insert(u, step))
        seq_ev.append(t3.evict(step) if step % 4 == 0 else -1)
    g["table.seq.lens"] = np.array([len(u) for u in seq_ids], np.int64)
    g["table.seq.ids"] = np.concatenate(seq_ids).astype(np.int64)
    g["table.seq.offs"] = np.concatenate(seq_offs).astype(np.int64)
    g["table.seq.evicted"] = np.array(seq_ev, np.int64)
    ex3 = t3.export_rows()
    for k, a in zip(("ids", "w", "m", "v", "last"), ex3):
        g[f"table.seq.export.{k}"] = a

    # --- segment_reduce / tile ---------------------------------------------------------
    def segs(lens):
        return np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)

    seg_cases = {
        "short": rng.integers(0, 6, 200),
        "long": np.array([1000, 0, 1, 7, 8, 9, 15, 16, 17, 127, 128, 129, 130, 255, 256, 257, 513, 2049]),
        "len1": np.ones(300, np.int64),
        "empty_all": np.zeros(5, np.int64),
        "spec": np.array([2, 1]),
    }
    for name, lens in seg_cases.items():
        offs = segs(lens)
        n = int(offs[-1])
        for D in (1, 3, 16):
            rows = (rng.standard_normal((n, D)) * rng.choice([1.0, 1e4, 1e-4], size=(n, D))).astype(np.float32)
            if name == "spec" and D == 1:
                continue
            key = f"seg.{name}.D{D}"
            g[key + ".rows"] = rows
            g[key + ".offs"] = offs
            for mode in ("sum", "mean"):
                for strat in ("auto", "sequential", "scatter"):
                    g[f"{key}.{mode}.{strat}"] = SG.segment_reduce(rows, offs, mode, strat)
            for k in (0, 1, 3, 8):
                g[f"{key}.tile{k}"] = SG.segment_tile(rows, offs, k, pad=-1.5)
    spec_rows = np.array([[1, 2], [3, 4], [5, 6]], np.float32)
    g["seg.spec2.rows"] = spec_rows
    g["seg.spec2.sum"] = SG.segment_reduce(spec_rows, [0, 2, 3], "sum")
    g["seg.spec2.mean"] = SG.segment_reduce(spec_rows, [0, 2, 3], "mean")
    g["seg.spec2.tile2"] = SG.segment_tile(spec_rows, [0, 2, 3], 2)

    # --- sparse adam ------------------------------------------------------------------------
    for variant, wd in (("adam", 0.0), ("adamw", 0.01), ("adamw", 0.0), ("adam", 0.3)):
        cfg = OP.AdamConfig(lr=0.01, weight_decay=wd, variant=variant)
        tb = EM.EmbeddingTable("o", 8, seed=3)
        offs = tb.lookup_or_insert(np.arange(50), 1)
        ra = np.random.Generator(np.random.PCG64(9))
        for t_ in range(1, 8):
            sel = ra.permutation(50)[: ra.integers(1, 50)]
            gr = (ra.standard_normal((len(sel), 8)) * 0.1).astype(np.float32)
            g[f"adam.{variant}.{wd}.sel{t_}"] = sel
            g[f"adam.{variant}.{wd}.g{t_}"] = gr
            OP.sparse_adam_step(tb.store, offs[sel], gr, cfg, t_)
        p = tb.store.read(offs)
        m, v = tb.store.read_state(offs)
        g[f"adam.{variant}.{wd}.p"], g[f"adam.{variant}.{wd}.m"], g[f"adam.{variant}.{wd}.v"] = p, m, v
    tb = EM.EmbeddingTable("spec", 1, seed=0)
    o = tb.lookup_or_insert([0], 1)
    tb.store.write(o, np.zeros((1, 1), np.float32))
    OP.sparse_adam_step(tb.store, o, np.ones((1, 1), np.float32), OP.AdamConfig(lr=0.1), 1)
    g["adam.spec.p"] = tb.store.read(o)
    g["adam.spec.mv"] = np.concatenate(tb.store.read_state(o), axis=1)

    # --- sharded lookup/update invariance (S = 1, 4) ------------------------------------------
    cfg = OP.AdamConfig(lr=1e-2, weight_decay=0.01, variant="adamw")
    for S in (1, 4):
        lts = SH.merge_tables_by_dim([("A", 8), ("B", 8), ("C", 4)], num_shards=S, seed=17)
        plan = SH.ShardPlan(S)
        rg = np.random.Generator(np.random.PCG64(31))
        outs = []
        for step in range(1, 6):
            for lt_ in lts:
                keys = np.concatenate([lt_.keys_for(m, rg.zipf(1.3, 64).astype(np.int64)) for m in lt_.members])
                rows = SH.all_to_all_lookup(lt_, keys, plan, step)
                grads = (rg.standard_normal(rows.shape) * 0.05).astype(np.float32)
                SH.all_to_all_grad_update(lt_, keys, grads, plan, cfg, step)
                g[f"a2a.S{S}.{lt_.name}.{step}.keys"] = keys
                g[f"a2a.S{S}.{lt_.name}.{step}.rows"] = rows
                g[f"a2a.S{S}.{lt_.name}.{step}.grads"] = grads
        for lt_ in lts:
            allx = [sh.export_rows() for sh in lt_.shards]
            ids_ = np.concatenate([a[0] for a in allx])
            o = np.argsort(ids_)
            g[f"a2a.S{S}.{lt_.name}.final.ids"] = ids_[o]
            g[f"a2a.S{S}.{lt_.name}.final.w"] = np.concatenate([a[1] for a in allx])[o]
            g[f"a2a.S{S}.{lt_.name}.final.m"] = np.concatenate([a[2] for a in allx])[o]
            g[f"a2a.S{S}.{lt_.name}.final.v"] = np.concatenate([a[3] for a in allx])[o]

    # --- feature engine ---------------------------------------------------------------------
    vals = np.concatenate([rng.random(300, dtype=np.float32) * 1.2 - 0.1,
                           np.linspace(0.05, 0.95, 10, dtype=np.float32), [-np.inf, np.inf]]).astype(np.float32)
    rt = RG.RaggedTensor(vals, np.array([0, len(vals)], np.int64))
    edges_list = [np.linspace(0.05, 0.95, 10, dtype=np.float32), np.array([0.5], np.float32),
                  np.empty(0, np.float32), np.array([-0.05, 0.2, 0.21, 0.9], np.float32)]
    g["fe.bucket.vals"] = vals
    for i, e in enumerate(edges_list):
        g[f"fe.bucket.edges{i}"] = e
        g[f"fe.bucket.out{i}"] = FE.bucketize(rt, e).values
    plan = FE.FusedPlan.for_bucketize(edges_list)
    cols = [RG.RaggedTensor(vals[i * 50:(i + 1) * 50 + i], np.array([0, 50 + i], np.int64)) for i in range(4)]
    fo = FE.fused_bucketize(plan, cols)
    for i in range(4):
        g[f"fe.fbucket.out{i}"] = fo[i].values
    mvals = np.concatenate([EDGE_IDS, rng.integers(-(2**63), 2**63 - 1, 300, dtype=np.int64, endpoint=True)])
    g["fe.mod.vals"] = mvals
    for mval in (1, 2, 10, 1_000_003, 2**40 + 7, 2**63 - 1):
        g[f"fe.mod.{mval}"] = FE.mod_transform(RG.RaggedTensor(mvals, np.array([0, len(mvals)])), mval).values
    a_lens = rng.integers(0, 4, 50)
    b_lens = rng.integers(0, 4, 50)
    a = RG.RaggedTensor(rng.integers(-1000, 1000, a_lens.sum()), np.concatenate([[0], np.cumsum(a_lens)]))
    b = RG.RaggedTensor(rng.integers(-(2**63), 2**63 - 1, b_lens.sum(), dtype=np.int64, endpoint=True),
                        np.concatenate([[0], np.cumsum(b_lens)]))
    c = FE.cross(a, b)
    g["fe.cross.a"], g["fe.cross.aoffs"] = a.values, a.row_offsets
    g["fe.cross.b"], g["fe.cross.boffs"] = b.values, b.row_offsets
    g["fe.cross.out"], g["fe.cross.offs"] = c.values, c.row_offsets
    rr = RG.RaggedTensor(np.arange(20, dtype=np.int64), np.array([0, 5, 5, 12, 20]))
    g["ragged.trunc.tail3"] = rr.truncate(3, "tail").values
    g["ragged.trunc.tail3.offs"] = rr.truncate(3, "tail").row_offsets
    g["ragged.trunc.head3"] = rr.truncate(3, "head").values

    np.savez_compressed(OUT, **g)
    print(f"wrote {len(g)} arrays to {OUT}")


def table_edge_trace(tb, log):
    """IDMap edits (remove / put / free_list mutation) interleaved with
    admission, eviction and export (embedding.py:39-61, 185-308).  The same
    driver runs the reference, the oracle and the GPU table; `log` records
    every observable result.  `tb` exposes the reference's table API."""
    log("o1", tb.lookup_or_insert(np.arange(10, dtype=np.int64), 1))
    log("rm3", np.array([tb.idmap.remove(3)], np.int64))       # slot stays live, leaves the dict
    log("len1", np.array([len(tb.idmap)], np.int64))
    log("ex1", *tb.export_rows())
    log("o2", tb.lookup_or_insert(np.arange(5, 15, dtype=np.int64), 4))
    log("ev1", np.array([tb.evict(4)], np.int64))             # ids 0..4 minus 3 are stale
    log("fl1", np.array(tb.idmap.free_list, np.int64))
    fl = tb.idmap.free_list
    fl.reverse()                                              # in-place mutation of the reference's list
    fl.append(3)                                              # the removed id's slot, reused next
    log("fl2", np.array(tb.idmap.free_list, np.int64))
    log("o3", tb.lookup_or_insert(np.array([100, 101, 102], np.int64), 5))
    tb.idmap.put(200, 15)                                     # an entry on a never-allocated slot
    log("len2", np.array([len(tb.idmap)], np.int64))
    log("ex2", *tb.export_rows())
    log("ev2", np.array([tb.evict(9)], np.int64))
    log("fl3", np.array(tb.idmap.free_list, np.int64))
    log("ex3", *tb.export_rows())


def negative_threshold_trace(tb, log):
    """evict_threshold < 0: `step - last > thr` holds for every row."""
    log("o1", tb.lookup_or_insert(np.arange(6, dtype=np.int64), 3))
    log("ev", np.array([tb.evict(3)], np.int64))
    log("fl", np.array(tb.idmap.free_list, np.int64))
    log("o2", tb.lookup_or_insert(np.array([50, 51], np.int64), 4))


def edges():
    """golden_edges.npz: drop-in edge cases added in round 2."""
    load_ref()
    from sparsekit_ref import segments as SG, embedding as EM
    rng = np.random.Generator(np.random.PCG64(77))
    g = {}

    def logger(prefix):
        def log(name, *arrs):
            for i, a in enumerate(arrs):
                g[f"{prefix}.{name}.{i}"] = np.asarray(a)
        return log

    table_edge_trace(EM.EmbeddingTable("e", 4, seed=2, block_size=4, evict_threshold=2), logger("idmap"))
    negative_threshold_trace(EM.EmbeddingTable("n", 4, seed=2, block_size=4, evict_threshold=-1), logger("negthr"))
    # float64 / integer rows keep their dtype (segments.py:51-58, 103-116)
    lens = np.array([0, 1, 2, 7, 8, 9, 17, 130, 300, 0, 3])
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    n = int(offs[-1])
    r64 = rng.standard_normal((n, 3)) * rng.choice([1.0, 1e8, 1e-8], size=(n, 3))
    ri = rng.integers(-(2**40), 2**40, (n, 3))
    g["seg64.offs"], g["seg64.rows"], g["segi.rows"] = offs, r64, ri
    for mode in ("sum", "mean"):
        for strat in ("sequential", "scatter", "auto"):
            g[f"seg64.{mode}.{strat}"] = SG.segment_reduce(r64, offs, mode, strat)
    for strat in ("sequential", "scatter"):
        g[f"segi.sum.{strat}"] = SG.segment_reduce(ri, offs, "sum", strat)
        g[f"segi32.sum.{strat}"] = SG.segment_reduce(ri.astype(np.int32), offs, "sum", strat)
    g["seg64.tile4"] = SG.segment_tile(r64, offs, 4, pad=-2.5)
    g["segi.tile4"] = SG.segment_tile(ri, offs, 4, pad=-7)
    np.savez_compressed(OUT2, **g)
    print(f"wrote {len(g)} arrays to {OUT2}")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "edges":
        edges()
    else:
        main()
        edges()
