"""GPU parity: the CUDA path (through the C ABI) vs the reference's golden
vectors and the CPU oracle.  Bit-exact for integer/index work and for every
float result the reference defines by a fixed operation order."""

import numpy as np
import pytest

from oracle import sparse_oracle as O

pytestmark = pytest.mark.gpu


def bits(a):
    a = np.asarray(a)
    if a.dtype == np.float32:
        return a.view(np.int32)
    if a.dtype == np.float64:
        return a.view(np.int64)
    return a


def eq(a, b):
    a = a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)
    b = np.asarray(b)
    assert a.shape == b.shape, (a.shape, b.shape)
    if a.dtype.kind == "f":
        b = b.astype(a.dtype)
    assert np.array_equal(bits(a), bits(b)), (a, b)


@pytest.fixture(scope="module")
def skb(cuda):
    import paper_2509_20883_b200 as m
    return m


def test_native_library_is_loaded(skb):
    from paper_2509_20883_b200 import _native
    lib = _native.lib()
    assert lib.skb_version().decode().startswith("sparsekit_b200")
    import ctypes
    n = ctypes.c_int()
    _native.check(lib.skb_device_sm_count(0, ctypes.byref(n)))
    assert n.value >= 132


def test_hashing(skb, golden):
    ids = golden["hash.ids"]
    eq(skb.hashing.mix64(ids).view(np.int64), golden["hash.mix64"])
    for S in (1, 2, 3, 8, 13):
        eq(skb.ShardPlan(S).shard_of(ids), golden[f"hash.shard_of.S{S}"])
    lt = skb.LogicalTable("dimx", 8, 1, members=["C0", "user_id", "ünï"], namespaced=True)
    for m in lt.members:
        eq(lt.keys_for(m, ids), golden[f"hash.keys_for.{m}"])
    with pytest.raises(KeyError):
        lt.keys_for("nope", ids)
    blob, offs = golden["fnv.blob"], golden["fnv.offs"]
    eq(skb.hashing.fnv1a64_packed(blob, offs), golden["fnv.hash"])
    eq(skb.hashing.fnv1a64_pairs(golden["fnv.pairs.x"], golden["fnv.pairs.y"]).view(np.int64),
       golden["fnv.pairs.h"])


def test_initial_rows(skb, golden):
    ids = golden["hash.ids"]
    for seed, dim in ((0, 16), (7, 64), (-3, 8), (2**40 + 5, 3), (123, 128)):
        eq(skb.initial_rows(seed, ids, dim), golden[f"init.{seed}.{dim}"])


@pytest.mark.parametrize("name", ["rand", "wide", "dups", "edge", "spec", "empty", "zipf"])
@pytest.mark.parametrize("S", [1, 2, 8])
def test_unique_partition(skb, golden, name, S):
    ids = golden[f"part.{name}.ids"]
    pr = skb.unique_partition(ids, skb.ShardPlan(S))
    eq(np.concatenate(pr.shard_ids), golden[f"part.{name}.S{S}.uniq"])
    eq([len(s) for s in pr.shard_ids], golden[f"part.{name}.S{S}.counts"])
    eq(pr.inverse_shard, golden[f"part.{name}.S{S}.inv_shard"])
    eq(pr.inverse_pos, golden[f"part.{name}.S{S}.inv_pos"])
    eq(pr.reconstruct_ids(), ids)
    st = skb.load_stats(ids, skb.ShardPlan(S))
    eq(st.counts, golden[f"part.{name}.S{S}.load_counts"])
    assert st.imbalance == float(golden[f"part.{name}.S{S}.imbalance"])


def test_unique_partition_torch_and_large(skb, cuda):
    import torch
    rng = np.random.default_rng(5)
    ids = rng.integers(0, 300_000, 1_000_000)
    for S in (1, 8):
        pr = skb.unique_partition(torch.from_numpy(ids).to(cuda), skb.ShardPlan(S))
        shards, inv_s, inv_p = O.dedup_partition(ids, S)
        eq(torch.cat(pr.shard_ids), np.concatenate(shards))
        eq(pr.inverse_shard, inv_s)
        eq(pr.inverse_pos, inv_p)


def test_table_trace(skb, golden):
    t = skb.EmbeddingTable("t", 4, seed=11, block_size=4, evict_threshold=5)
    out = [t.lookup_or_insert([10, 20, 30], 1), [t.evict(10)], t.lookup_or_insert([40, 50], 11),
           t.lookup_or_insert([10], 12), [t.evict(30)], t.lookup_or_insert([60, 70, 80, 90], 31),
           t.lookup_or_insert([60], 36), [t.evict(40)],
           t.lookup_or_insert(np.array([-5, 2**63 - 1, -(2**63), 70], np.int64), 41)]
    out.append(t.gather(t.lookup_or_insert([-5, 60], 41)))
    t.scatter_update(t.lookup_or_insert([60], 41), np.arange(4, dtype=np.float32)[None, :])
    out.append(t.gather(t.lookup_or_insert([60, -5], 42)))
    for i, o in enumerate(out):
        eq(o, golden[f"table.trace.{i}"])
    ex = t.export_rows()
    for k, a in zip(("ids", "w", "m", "v", "last"), ex):
        eq(a, golden[f"table.export.{k}"])
    assert t.store.capacity == golden["table.capacity"]
    assert t.num_rows == golden["table.num_rows"]
    eq(t.idmap.free_list, golden["table.free_list"])
    assert t.idmap.get(-(2**63)) is not None and t.idmap.get(123456) is None
    t2 = skb.EmbeddingTable("t2", 4, seed=11, block_size=4, evict_threshold=1)
    t2.lookup_or_insert([1, 2, 3, 4, 5], 1)
    t2.lookup_or_insert([3], 5)
    t2.evict(5)
    t2.restore_rows(*ex)
    eq(t2.lookup_or_insert(ex[0], 50), golden["table.restore.offsets"])
    eq(t2.idmap.free_list, golden["table.restore.free_list"])
    with pytest.raises(ValueError, match="already present"):
        t2.restore_rows(ex[0][:1], ex[1][:1], ex[2][:1], ex[3][:1], ex[4][:1])


def test_table_random_sequence(skb, golden):
    t = skb.EmbeddingTable("t3", 8, seed=5, block_size=16, evict_threshold=3)
    lens = golden["table.seq.lens"]
    ids = np.split(golden["table.seq.ids"], np.cumsum(lens)[:-1])
    offs, ev = [], []
    for step in range(1, 41):
        offs.append(t.lookup_or_insert(ids[step - 1], step))
        ev.append(t.evict(step) if step % 4 == 0 else -1)
    eq(np.concatenate(offs), golden["table.seq.offs"])
    eq(ev, golden["table.seq.evicted"])
    for k, a in zip(("ids", "w", "m", "v", "last"), t.export_rows()):
        eq(a, golden[f"table.seq.export.{k}"])


def test_table_model_based_random(skb):
    """Random op sequences (admit / evict / scatter / gather) vs the oracle table."""
    rng = np.random.default_rng(11)
    for trial in range(3):
        g = skb.EmbeddingTable("m", 4, seed=trial, block_size=8, evict_threshold=2)
        o = O.OracleTable(4, seed=trial, block_size=8, evict_threshold=2)
        for step in range(1, 30):
            op = rng.integers(0, 4)
            if op <= 1:
                u = rng.permutation(np.unique(rng.integers(-20, 40, rng.integers(0, 30))))
                eq(g.lookup_or_insert(u, step), o.lookup_or_insert(u, step))
            elif op == 2:
                assert g.evict(step) == o.evict(step)
            elif o.num_rows:
                keys = np.fromiter(o.map.keys(), np.int64)
                sel = rng.permutation(keys)[: rng.integers(1, len(keys) + 1)]
                offs = np.array([o.map[k] for k in sel], np.int64)
                rows = rng.standard_normal((len(offs), 4)).astype(np.float32)
                g.scatter_update(offs, rows)
                o.scatter_update(offs, rows)
                eq(g.gather(offs), o.gather(offs))
            assert g.num_rows == o.num_rows
            assert g.store.capacity == o.capacity
        for a, b in zip(g.export_rows(), o.export_rows()):
            eq(a, b)
        eq(g.idmap.free_list, o.free)


def test_table_errors(skb):
    t = skb.EmbeddingTable("e", 2)
    with pytest.raises(ValueError, match="duplicate-free"):
        t.lookup_or_insert([1, 2, 1], 1)
    o = t.lookup_or_insert([1, 2], 1)
    with pytest.raises(IndexError, match="gather: offset 5 is not a live slot"):
        t.gather([0, 5, 7])
    with pytest.raises(IndexError, match="offset -1"):
        t.gather([-1])
    with pytest.raises(ValueError, match="distinct"):
        t.scatter_update([o[0], o[0]], np.zeros((2, 2), np.float32))
    with pytest.raises(ValueError, match="shape"):
        t.scatter_update(o, np.zeros((3, 2), np.float32))
    with pytest.raises(IndexError, match="scatter_update: offset 9"):
        t.scatter_update([9], np.zeros((1, 2), np.float32))
    eq(t.gather(np.zeros(0, np.int64)), np.zeros((0, 2), np.float32))
    eq(t.gather([o[1], o[1]]), np.repeat(t.gather([o[1]]), 2, axis=0))
    items = t.idmap.items()
    assert [k for k, _ in items] == [1, 2]
    assert t.idmap.remove(1) == o[0]
    with pytest.raises(KeyError):
        t.idmap.remove(1)
    assert len(t.idmap) == 1


@pytest.mark.parametrize("D", [3, 16])
def test_checked_row_ops_leave_table_untouched_and_rearm(skb, D):
    """scatter_update / BlockStore.write check before writing (one cooperative
    launch): on error nothing is written, the persistent device flags and the
    distinctness bitmap are re-armed, and repeated calls with the same
    offsets do not see stale duplicate bits."""
    rng = np.random.default_rng(D)
    n = 200_000
    t = skb.EmbeddingTable("c", D, seed=1, block_size=4096)
    o = t.lookup_or_insert(np.arange(n, dtype=np.int64) * 7 + 3, 1)
    before = t.gather(o)
    perm = rng.permutation(n)
    rows = rng.standard_normal((n, D)).astype(np.float32)
    bad = o[perm].copy()
    bad[n - 1] = bad[17]  # one duplicate at the end
    with pytest.raises(ValueError, match="distinct"):
        t.scatter_update(bad, rows)
    eq(t.gather(o), before)
    bad = o[perm].copy()
    bad[5] = n + 10  # in the arena, not live
    with pytest.raises(IndexError, match=f"scatter_update: offset {n + 10} is not a live slot"):
        t.scatter_update(bad, rows)
    eq(t.gather(o), before)
    for _ in range(2):  # same offsets twice: the bitmap was cleared by the first call
        t.scatter_update(o[perm], rows)
        eq(t.gather(o[perm]), rows)
    cap = t.store.capacity
    with pytest.raises(IndexError, match="outside the store capacity"):
        t.store.write(np.array([0, cap + 5], np.int64), np.zeros((2, D), np.float32))
    eq(t.gather(o[perm]), rows)
    t.store.write(o[:3], np.ones((3, D), np.float32))
    eq(t.gather(o[:3]), np.ones((3, D), np.float32))
    with pytest.raises(IndexError, match="gather: offset -4"):
        t.gather(np.array([o[0], -4], np.int64))
    eq(t.gather(o[:3]), np.ones((3, D), np.float32))


@pytest.mark.parametrize("D", [3, 16])
def test_deferred_gather_scatter(skb, D):
    """gather / scatter_update inside deferred_checks(): same results as the
    eager calls, nothing read back per call, and the eager path's exception
    (type, message, duplicate-before-liveness order) raised at the context's
    exit — with the table untouched by a failing scatter."""
    import torch
    rng = np.random.default_rng(D + 1)
    n = 50_000
    t = skb.EmbeddingTable("d", D, seed=2)
    o = torch.from_numpy(t.lookup_or_insert(np.arange(n, dtype=np.int64) * 5 + 1, 1)).cuda()
    perm = torch.from_numpy(rng.permutation(n)).cuda()
    rows = torch.from_numpy(rng.standard_normal((n, D)).astype(np.float32)).cuda()
    before = t.gather(o).clone()
    with skb.deferred_checks():
        g = t.gather(o[perm])
        t.scatter_update(o[perm], rows)
        g2 = t.gather(o[perm])
    eq(g.cpu().numpy(), before[perm].cpu().numpy())
    eq(g2.cpu().numpy(), rows.cpu().numpy())
    snap = t.gather(o).clone()
    cases = [
        (lambda x: x.__setitem__(n - 1, x[17]), ValueError, "requires distinct"),
        (lambda x: x.__setitem__(5, n + 10), IndexError, f"scatter_update: offset {n + 10} is not a live slot"),
        # a duplicate AND a dead slot: the duplicate wins, as in the eager path
        (lambda x: (x.__setitem__(3, n + 20), x.__setitem__(9, x[2])), ValueError, "requires distinct"),
        # two equal out-of-range offsets: distinctness decided on the host
        (lambda x: (x.__setitem__(4, -7), x.__setitem__(8, -7)), ValueError, "requires distinct"),
        (lambda x: x.__setitem__(6, -7), IndexError, "scatter_update: offset -7 is not a live slot"),
    ]
    for mutate, exc, msg in cases:
        bad = o[perm].clone()
        mutate(bad)
        with pytest.raises(exc, match=msg):
            with skb.deferred_checks():
                t.scatter_update(bad, rows * 2)
        eq(t.gather(o).cpu().numpy(), snap.cpu().numpy())
    with pytest.raises(IndexError, match=f"gather: offset {n + 3} is not a live slot"):
        with skb.deferred_checks():
            x = o.clone()
            x[11] = n + 3
            t.gather(x)
    # the same failures eagerly: identical messages
    bad = o[perm].clone()
    bad[5] = n + 10
    with pytest.raises(IndexError, match=f"scatter_update: offset {n + 10} is not a live slot"):
        t.scatter_update(bad, rows)


@pytest.mark.parametrize("name", ["short", "long", "len1", "empty_all"])
@pytest.mark.parametrize("D", [1, 3, 16])
def test_segments(skb, golden, name, D):
    key = f"seg.{name}.D{D}"
    rows, offs = golden[key + ".rows"], golden[key + ".offs"]
    for mode in ("sum", "mean"):
        for strat in ("auto", "sequential", "scatter"):
            eq(skb.segment_reduce(rows, offs, mode, strat), golden[f"{key}.{mode}.{strat}"])
    for k in (0, 1, 3, 8):
        eq(skb.segment_tile(rows, offs, k, pad=-1.5), golden[f"{key}.tile{k}"])


def test_segments_torch_and_errors(skb, golden, cuda):
    import torch
    rows, offs = golden["seg.long.D16.rows"], golden["seg.long.D16.offs"]
    out = skb.segment_reduce(torch.from_numpy(rows).to(cuda), torch.from_numpy(offs).to(cuda), "sum", "sequential")
    eq(out, golden["seg.long.D16.sum.sequential"])
    with pytest.raises(ValueError, match="start at 0"):
        skb.segment_reduce(rows, offs + 1)
    with pytest.raises(ValueError, match="nondecreasing"):
        skb.segment_reduce(rows[:2], [0, 2, 1, 2])
    with pytest.raises(ValueError, match="unknown mode"):
        skb.segment_reduce(rows, offs, "max")
    with pytest.raises(ValueError, match="unknown strategy"):
        skb.segment_reduce(rows, offs, "sum", "atomic")
    with pytest.raises(ValueError, match="!= num rows"):
        skb.segment_reduce(torch.from_numpy(rows).to(cuda), torch.from_numpy(offs[:-1]).to(cuda))


def test_segments_large_random(skb):
    rng = np.random.default_rng(3)
    for lens in (rng.integers(0, 3000, 40), rng.integers(0, 5, 20000)):
        offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        rows = rng.standard_normal((int(offs[-1]), 16)).astype(np.float32)
        for strat in ("sequential", "scatter"):
            eq(skb.segment_reduce(rows, offs, "mean", strat), O.pool(rows, offs, "mean", strat))


@pytest.mark.parametrize("D", [16, 3])
def test_segments_long_sequential_tree(skb, D):
    """Long sequential segments take the warp-parallel pairwise kernel (leaves
    on lanes, tree combined in numpy order): lengths 129-6000 (1 to > 32
    leaves), empty segments, and trailing empties (the reduceat clip)."""
    rng = np.random.default_rng(D)
    lens = np.concatenate([[129, 130, 137, 256, 1000, 1001, 4095, 4097, 6000, 0, 1, 2],
                           rng.integers(100, 3000, 20), [0, 0]])
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    rows = (rng.standard_normal((int(offs[-1]), D)) * 100).astype(np.float32)
    for mode in ("sum", "mean"):
        eq(skb.segment_reduce(rows, offs, mode, "sequential"), O.pool(rows, offs, mode, "sequential"))


@pytest.mark.parametrize("variant,wd", [("adam", 0.0), ("adamw", 0.01), ("adamw", 0.0), ("adam", 0.3)])
def test_adam(skb, golden, variant, wd):
    cfg = skb.AdamConfig(lr=0.01, weight_decay=wd, variant=variant)
    t = skb.EmbeddingTable("o", 8, seed=3)
    offs = t.lookup_or_insert(np.arange(50), 1)
    for s in range(1, 8):
        sel = golden[f"adam.{variant}.{wd}.sel{s}"]
        skb.sparse_adam_step(t.store, offs[sel], golden[f"adam.{variant}.{wd}.g{s}"], cfg, s)
    eq(t.store.read(offs), golden[f"adam.{variant}.{wd}.p"])
    m, v = t.store.read_state(offs)
    eq(m, golden[f"adam.{variant}.{wd}.m"])
    eq(v, golden[f"adam.{variant}.{wd}.v"])


def test_adam_spec_and_errors(skb, golden):
    t = skb.EmbeddingTable("spec", 1, seed=0)
    o = t.lookup_or_insert([0], 1)
    t.store.write(o, np.zeros((1, 1), np.float32))
    skb.sparse_adam_step(t.store, o, np.ones((1, 1), np.float32), skb.AdamConfig(lr=0.1), 1)
    eq(t.store.read(o), golden["adam.spec.p"])
    with pytest.raises(ValueError, match="distinct"):
        skb.sparse_adam_step(t.store, [0, 0], np.ones((2, 1), np.float32), skb.AdamConfig(), 1)
    with pytest.raises(ValueError, match="t must be"):
        skb.sparse_adam_step(t.store, [0], np.ones((1, 1), np.float32), skb.AdamConfig(), 0)


def test_distinctness_checks_large(skb):
    """lookup_or_insert's duplicate test (key-claim table) and
    sparse_adam_step's offset checks (slot bitmap): a single repeated pair in
    1M positions is caught, INT64_MIN is a key like any other, duplicates are
    reported before out-of-range offsets, and a rejected call leaves the
    table untouched and the bitmap clear for the next call."""
    rng = np.random.default_rng(11)
    n = 1_000_000
    ids = rng.permutation(np.arange(-n, n, 2, dtype=np.int64))
    bad = ids.copy()
    bad[n - 1] = bad[12345]
    t = skb.EmbeddingTable("dup", 4, seed=2, capacity_hint=n)
    with pytest.raises(ValueError, match="duplicate-free"):
        t.lookup_or_insert(bad, 1)
    assert t.num_rows == 0
    mn = np.iinfo(np.int64).min
    with pytest.raises(ValueError, match="duplicate-free"):
        t.lookup_or_insert([mn, 5, mn], 1)
    t.lookup_or_insert([mn, 5], 1)
    offs = t.lookup_or_insert(ids, 1)
    assert t.num_rows == n + 2
    g = np.ones((n, 4), np.float32)
    cfg = skb.AdamConfig(lr=0.1)
    before = t.store.read(offs[:8])
    dup = offs.copy()
    dup[-1] = dup[0]
    with pytest.raises(ValueError, match="distinct"):
        skb.sparse_adam_step(t.store, dup, g, cfg, 1)
    far = offs.copy()
    far[7] = 1 << 40
    far[9] = 1 << 40  # duplicated out-of-range offset: still a ValueError first
    with pytest.raises(ValueError, match="distinct"):
        skb.sparse_adam_step(t.store, far, g, cfg, 1)
    far[9] = -3
    with pytest.raises(IndexError, match="offset 1099511627776"):
        skb.sparse_adam_step(t.store, far, g, cfg, 1)
    eq(t.store.read(offs[:8]), before)
    skb.sparse_adam_step(t.store, offs, g, cfg, 1)  # bitmap left clear by the rejected calls
    assert not np.array_equal(t.store.read(offs[:8]), before)


@pytest.mark.parametrize("S", [3, 8, 5000])
def test_load_stats_large(skb, cuda, S):
    import torch
    rng = np.random.default_rng(S)
    ids = rng.integers(-(1 << 62), 1 << 62, 300_000)
    ids = np.concatenate([ids, ids[:50_000], [np.iinfo(np.int64).min] * 3])
    st = skb.load_stats(torch.from_numpy(ids).to(cuda), skb.ShardPlan(S))
    c, imb = O.shard_load(ids, S)
    eq(st.counts, c)
    assert st.imbalance == imb


@pytest.mark.parametrize("S", [1, 4])
def test_sharded_lookup_update(skb, golden, S):
    lts = skb.merge_tables_by_dim([("A", 8), ("B", 8), ("C", 4)], num_shards=S, seed=17)
    plan = skb.ShardPlan(S)
    cfg = skb.AdamConfig(lr=1e-2, weight_decay=0.01, variant="adamw")
    for step in range(1, 6):
        for lt in lts:
            keys = golden[f"a2a.S{S}.{lt.name}.{step}.keys"]
            eq(skb.all_to_all_lookup(lt, keys, plan, step), golden[f"a2a.S{S}.{lt.name}.{step}.rows"])
            skb.all_to_all_grad_update(lt, keys, golden[f"a2a.S{S}.{lt.name}.{step}.grads"], plan, cfg, step)
    for lt in lts:
        allx = [sh.export_rows() for sh in lt.shards]
        ids = np.concatenate([a[0] for a in allx])
        o = np.argsort(ids)
        eq(ids[o], golden[f"a2a.S{S}.{lt.name}.final.ids"])
        for j, k in ((1, "w"), (2, "m"), (3, "v")):
            eq(np.concatenate([a[j] for a in allx])[o], golden[f"a2a.S{S}.{lt.name}.final.{k}"])


def test_features(skb, golden):
    vals = golden["fe.bucket.vals"]
    rt = skb.RaggedTensor(vals, np.array([0, len(vals)], np.int64))
    edges = [golden[f"fe.bucket.edges{i}"] for i in range(4)]
    for i in range(4):
        eq(skb.bucketize(rt, edges[i]).values, golden[f"fe.bucket.out{i}"])
    plan = skb.FusedPlan.for_bucketize(edges)
    cols = [skb.RaggedTensor(vals[i * 50:(i + 1) * 50 + i], np.array([0, 50 + i], np.int64)) for i in range(4)]
    fo = skb.fused_bucketize(plan, cols)
    assert plan.dispatch_count == 1
    for i in range(4):
        eq(fo[i].values, golden[f"fe.fbucket.out{i}"])
    with pytest.raises(ValueError, match="NaN"):
        skb.bucketize(skb.RaggedTensor(np.array([1.0, np.nan], np.float32), [0, 2]), [0.5])
    mv = golden["fe.mod.vals"]
    rtm = skb.RaggedTensor(mv, np.array([0, len(mv)]))
    for m in (1, 2, 10, 1_000_003, 2**40 + 7, 2**63 - 1):
        eq(skb.mod_transform(rtm, m).values, golden[f"fe.mod.{m}"])
    mplan = skb.FusedPlan.for_mod([10, 1_000_003])
    half = len(mv) // 2
    fm = skb.fused_mod(mplan, [skb.RaggedTensor(mv[:half], [0, half]), skb.RaggedTensor(mv[half:], [0, len(mv) - half])])
    eq(np.concatenate([fm[0].values, fm[1].values]), np.concatenate([golden["fe.mod.10"][:half],
                                                                     golden["fe.mod.1000003"][half:]]))
    with pytest.raises(ValueError):
        skb.mod_transform(rtm, 0)
    a = skb.RaggedTensor(golden["fe.cross.a"], golden["fe.cross.aoffs"])
    b = skb.RaggedTensor(golden["fe.cross.b"], golden["fe.cross.boffs"])
    c = skb.cross(a, b)
    eq(c.values, golden["fe.cross.out"])
    eq(c.row_offsets, golden["fe.cross.offs"])
    blob, offs = golden["fnv.blob"].tobytes(), golden["fnv.offs"]
    strs = np.array([blob[offs[i]:offs[i + 1]] for i in range(len(offs) - 1)], dtype=object)
    h = skb.hash_feature(skb.RaggedTensor(strs, [0, 3, len(strs)]))
    eq(h.values, golden["fnv.hash"])


def test_deferred_feature_checks(skb, cuda):
    """deferred_checks(): bucketize's NaN ValueError is raised at the context
    exit / check_deferred() instead of per call; results are unchanged."""
    import torch
    edges = np.linspace(0.05, 0.95, 10, dtype=np.float32)
    vals = np.random.default_rng(3).random(1000, dtype=np.float32)
    rt = skb.RaggedTensor(torch.from_numpy(vals).to(cuda), torch.tensor([0, 1000]).to(cuda))
    with skb.deferred_checks():
        got = skb.bucketize(rt, edges)
    eq(got.values, O.bucketize_values(vals, edges))
    bad = vals.copy()
    bad[517] = np.nan
    rb = skb.RaggedTensor(torch.from_numpy(bad).to(cuda), torch.tensor([0, 1000]).to(cuda))
    with pytest.raises(ValueError, match="NaN"):
        with skb.deferred_checks():
            skb.bucketize(rb, edges)  # no exception here
            skb.bucketize(rt, edges)
    with skb.deferred_checks():
        skb.bucketize(rb, edges)
        with pytest.raises(ValueError, match="NaN"):
            skb.check_deferred()
    with pytest.raises(ValueError, match="NaN"):
        skb.bucketize(rb, edges)  # outside: synchronous, as the reference


def test_cross_many(skb, golden, cuda):
    """cross_many == cross per pair, with the sizes read back or given."""
    import torch
    rng = np.random.default_rng(11)
    pairs, sizes = [], []
    for _ in range(5):
        la, lb = rng.integers(0, 6, 300), rng.integers(0, 6, 300)
        oa = np.concatenate([[0], np.cumsum(la)]).astype(np.int64)
        ob = np.concatenate([[0], np.cumsum(lb)]).astype(np.int64)
        a = skb.RaggedTensor(torch.from_numpy(rng.integers(-50, 50, oa[-1])).to(cuda), torch.from_numpy(oa).to(cuda))
        b = skb.RaggedTensor(torch.from_numpy(rng.integers(0, 10**12, ob[-1])).to(cuda), torch.from_numpy(ob).to(cuda))
        pairs.append((a, b))
        sizes.append(int((la * lb).sum()))
    for res in (skb.cross_many(pairs), skb.cross_many(pairs, sizes=sizes)):
        for (a, b), c in zip(pairs, res):
            ov, oo = O.cross_rows(a.values.cpu().numpy(), a.row_offsets.cpu().numpy(), b.values.cpu().numpy(),
                                  b.row_offsets.cpu().numpy())
            eq(c.values, ov)
            eq(c.row_offsets, oo)
    with pytest.raises(ValueError, match="sizes"):
        skb.cross_many(pairs, sizes=sizes[:2])


def test_ragged(skb, golden):
    rr = skb.RaggedTensor(np.arange(20, dtype=np.int64), np.array([0, 5, 5, 12, 20]))
    t3 = rr.truncate(3, "tail")
    eq(t3.values, golden["ragged.trunc.tail3"])
    eq(t3.row_offsets, golden["ragged.trunc.tail3.offs"])
    eq(rr.truncate(3, "head").values, golden["ragged.trunc.head3"])
    d, m = skb.RaggedTensor(np.array([1, 2, 7], np.int64), [0, 2, 2, 3]).pad_to_dense(4, 0)
    eq(d, [[1, 2, 0, 0], [0, 0, 0, 0], [7, 0, 0, 0]])
    eq(m, [[1, 1, 0, 0], [0, 0, 0, 0], [1, 0, 0, 0]])
    with pytest.raises(ValueError):
        rr.pad_to_dense(3)
    rows = skb.RaggedTensor(np.arange(12, dtype=np.float32), [0, 2, 6], dim=2)
    eq(rows.truncate(1, "tail").values, np.array([2, 3, 10, 11], np.float32))


def _fused_vs_oracle(skb, D, member_specs, steps, mode, seed=0, evict_every=0, thr=None, cfg=None, k=None, pad=0.0,
                     variants=None, check=None, id_hi=500, mid_export_every=0):
    """Drive the fused step and the oracle pipeline side by side (mode "tile":
    oracle = segment_tile + per-position tile gradients, zero past k).
    variants=(adam, pool) forces the fused kernels; check(step, lt) runs
    after every backward (e.g. to assert which kernel ran); mid_export_every:
    every that many steps the rows are exported and compared between a
    backward and the next forward (a deferred long fold must be joined);
    mode may be a function of the step."""
    import torch
    rng = np.random.default_rng(seed)
    members = [m for m, _, _ in member_specs]
    lt = skb.LogicalTable(f"dim{D}", D, 1, seed=seed, members=members, namespaced=True, evict_threshold=thr)
    if variants is not None:
        skb.set_variants(lt, *variants)
    olt = O.OracleLogical(f"dim{D}", D, 1, seed=seed, members=members, namespaced=True, evict_threshold=thr)
    cfg = cfg or skb.AdamConfig(lr=1e-2, weight_decay=0.01, variant="adamw")
    mode_of = mode if callable(mode) else (lambda _step: mode)  # mode per step (a table may switch)
    for step in range(1, steps + 1):
        mode = mode_of(step)
        ids, offs = [], []
        for m, B, gen in member_specs:
            lens = gen(rng, B)
            offs.append(np.concatenate([[0], np.cumsum(lens)]).astype(np.int64))
            ids.append(rng.zipf(1.2, int(lens.sum())).astype(np.int64) if m.startswith("z")
                       else rng.integers(0, id_hi, int(lens.sum())))
        batch = skb.PackedBatch(lt, members, ids, offs)
        pooled = skb.lookup_pool(lt, batch, step, mode, k=k, pad=pad)
        G = batch.num_bags
        W = D * k if mode == "tile" else D
        dp = rng.standard_normal((G, W)).astype(np.float32)
        skb.pool_grad_adam(lt, torch.from_numpy(dp).cuda(), cfg, step)
        if check is not None:
            check(step, lt)
        # oracle: train.py-style pipeline on the concatenated keys
        keys = np.concatenate([olt.keys_for(m, x) for m, x in zip(members, ids)])
        rows = O.lookup(olt, keys, step)
        ref, grads, pos, bag = [], [], 0, 0
        for f, (m, B, _) in enumerate(member_specs):
            n_f = len(ids[f])
            lens = np.diff(offs[f])
            g = dp[bag:bag + B]
            if mode == "tile":
                ref.append(O.tile(rows[pos:pos + n_f], offs[f], k, pad))
                gt = np.zeros((n_f, D), np.float32)
                for b in range(B):
                    take = min(k, int(lens[b]))
                    gt[offs[f][b]:offs[f][b] + take] = g[b].reshape(k, D)[:take]
                grads.append(gt)
            else:
                ref.append(O.pool(rows[pos:pos + n_f], offs[f], mode))
                if mode == "mean":
                    g = g / np.maximum(lens, 1).astype(np.float32)[:, None]
                grads.append(np.repeat(g, lens, axis=0).astype(np.float32))
            pos += n_f
            bag += B
        eq(pooled, np.concatenate(ref))
        O.grad_update(olt, keys, np.concatenate(grads), step, lr=cfg.lr, beta1=cfg.beta1, beta2=cfg.beta2,
                      eps=cfg.eps, weight_decay=cfg.weight_decay, variant=cfg.variant)
        if evict_every and step % evict_every == 0:
            assert lt.evict(step) == olt.evict(step)
        if mid_export_every and step % mid_export_every == 0 and step < steps:
            for a, b in zip(lt.local_table.export_rows(), olt.shards[0].export_rows()):
                eq(a, b)
    for a, b in zip(lt.local_table.export_rows(), olt.shards[0].export_rows()):
        eq(a, b)
    eq(lt.local_table.idmap.free_list, olt.shards[0].free)


def _expect_adam(want):
    def check(step, lt):
        got = skb_last(lt)[0]
        # auto mode starts every table on the register kernel until a backward
        # has shown no long runs (one sampled readback), then takes the TMA ring
        if want != 0 or step >= 3:
            assert got == want, (step, got, want)
    return check


def skb_last(lt):
    import paper_2509_20883_b200 as m
    return m.last_variants(lt)


@pytest.mark.parametrize("variant", list(range(9)))
@pytest.mark.parametrize("D", [64, 128])
def test_fused_adam_variants_onehot_sum(skb, variant, D):
    """The headline fold+Adam kernels against the oracle on the C2 regime:
    sum, bag length 1, uniform ids with repeats (multi-position runs), 5
    steps.  variant 0 = auto, which must settle on the TMA ring
    k_fused_adam_tma<16,192,4>; 1-3 register shapes; 4-8 TMA ring shapes."""
    specs = [("a", 3000, lambda r, B: np.ones(B, np.int64)), ("b", 2000, lambda r, B: np.ones(B, np.int64))]
    _fused_vs_oracle(skb, D, specs, steps=5, mode="sum", seed=30 + variant, variants=(variant, -1),
                     check=_expect_adam(variant), id_hi=2500)


@pytest.mark.parametrize("variant", [0, 2, 3, 4, 5, 6, 7, 8])
def test_fused_adam_variants_mean_hot(skb, variant):
    """Forced fold+Adam variants with mean bags, empty bags and zipf hot ids
    (runs > 32 positions leave the ring for the long fold)."""
    specs = [("a", 700, lambda r, B: r.integers(0, 5, B)), ("zb", 400, lambda r, B: r.integers(1, 9, B))]
    _fused_vs_oracle(skb, 64, specs, steps=4, mode="mean", seed=50 + variant, variants=(variant, -1),
                     check=_expect_adam(variant if variant else 3))


@pytest.mark.parametrize("D,mode", [(8, "mean"), (12, "sum"), (16, "mean"), (32, "sum"), (64, "sum"), (64, "mean"),
                                    (96, "mean"), (128, "sum"), (128, "mean")])
def test_fused_pool_stream(skb, D, mode):
    """Default pool for rows of 8 <= D <= 128 (D % 4 == 0, bags not all one-hot):
    k_fused_pool_stream, sub-groups streaming their bags' positions in
    batches — empty bags, long bags and chunk tails against the oracle."""
    specs = [("a", 1000, lambda r, B: np.where(r.random(B) < 0.1, 0, r.geometric(0.25, B))),
             ("b", 333, lambda r, B: r.integers(0, 13, B))]  # mean length < 16: every member pools with scatter
    _fused_vs_oracle(skb, D, specs, steps=3, mode=mode, seed=90 + D,
                     check=lambda step, lt: skb_last(lt)[1] == 6 or pytest.fail("stream pool"))


@pytest.mark.parametrize("pool", [1, 2, 3, 4, 5])
def test_fused_pool_variants(skb, pool):
    """Forced pool kernels (1-3 and 5 register shapes, 4 staged one-hot
    gather with its register fallback for mixed chunks) against the oracle."""
    specs = [("a", 900, lambda r, B: np.where(r.random(B) < 0.8, 1, r.integers(0, 4, B)))]
    _fused_vs_oracle(skb, 64, specs, steps=3, mode="sum", seed=70 + pool, variants=(-1, pool),
                     check=lambda step, lt: skb_last(lt)[1] == pool or pytest.fail("pool variant"))


@pytest.mark.parametrize("D,mode", [(64, "sum"), (64, "mean"), (128, "sum"), (8, "sum")])
def test_fused_onehot_negative_zero(skb, D, mode):
    """One-hot chunks take the staged row-gather pool: it must still fold from
    +0 like np.add.at (-0.0 -> +0.0), and chunks mixing bag lengths 0/1/2
    take the general path in the same launch."""
    import torch
    lt = skb.LogicalTable(f"nz{D}", D, 1, seed=4, members=["f"], namespaced=False)
    keys = np.arange(200, dtype=np.int64)
    t = lt.local_table
    offs = t.lookup_or_insert(keys, 1)
    rows = np.random.default_rng(D).standard_normal((200, D)).astype(np.float32)
    rows[::3, ::2] = -0.0
    t.scatter_update(offs, rows)
    lens = np.ones(160, np.int64)
    lens[100:] = np.tile([0, 2, 1], 20)  # n == G: the batch takes the staged kernel, chunks 3-4 its general path
    ids = np.concatenate([np.arange(100), np.random.default_rng(2).integers(0, 200, int(lens[100:].sum()))])
    bo = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    batch = skb.PackedBatch(lt, ["f"], [ids], [bo])
    pooled = skb.lookup_pool(lt, batch, 2, mode)
    eq(pooled, O.pool(rows[ids], bo, mode))
    assert rows[0, 0] == 0 and np.signbit(rows[0, 0]) and not np.signbit(pooled.cpu().numpy()[0, 0])
    dp = np.random.default_rng(D + 1).standard_normal((160, D)).astype(np.float32)
    dp[::5] = -0.0
    skb.pool_grad_adam(lt, torch.from_numpy(dp).cuda(), skb.AdamConfig(), 2)
    # the backward against the oracle (same rows, the same per-position grads)
    olt = O.OracleLogical(f"nz{D}", D, 1, seed=4, members=["f"], namespaced=False)
    o = olt.shards[0]
    o.scatter_update(o.lookup_or_insert(keys, 1), rows)
    O.lookup(olt, ids, 2)
    g = dp / np.maximum(np.diff(bo), 1).astype(np.float32)[:, None] if mode == "mean" else dp
    O.grad_update(olt, ids, np.repeat(g, np.diff(bo), axis=0).astype(np.float32), 2)
    for a, b in zip(t.export_rows(), o.export_rows()):
        eq(a, b)


def test_fused_c1_shape(skb):
    # C1: dim16, B4096, 1 feature, bag length 1, sum, AdamW
    _fused_vs_oracle(skb, 16, [("f0", 4096, lambda r, B: np.ones(B, np.int64))], steps=4, mode="sum")


def test_fused_multi_member_mean(skb):
    specs = [("a", 300, lambda r, B: np.minimum(r.geometric(0.25, B) - 1, 64)),
             ("zb", 200, lambda r, B: r.integers(0, 6, B)),
             ("long", 20, lambda r, B: r.integers(0, 400, B)),   # mean len >= 16 -> sequential
             # sequential member ending in empty bags: the reduceat n-1 clip quirk
             ("tail", 12, lambda r, B: np.concatenate([r.integers(20, 300, B - 3), [0, 0, 0]]))]
    _fused_vs_oracle(skb, 8, specs, steps=5, mode="mean", seed=4)


def test_fused_with_eviction(skb):
    specs = [("a", 128, lambda r, B: r.integers(1, 4, B))]
    _fused_vs_oracle(skb, 4, specs, steps=12, mode="sum", seed=9, evict_every=3, thr=2,
                     cfg=skb.AdamConfig(lr=0.05))


@pytest.mark.parametrize("D", [16, 3])
def test_fused_tile_combiner(skb, D):
    """Fused tile combiner == segment_tile + tile-gradient expansion + grad
    update: bags shorter than k (pad rows), longer than k (positions past k
    fold a zero gradient but their rows are still updated), empty bags, and a
    zipf member whose hot ids take the long-run fold."""
    specs = [("a", 150, lambda r, B: r.integers(0, 12, B)),
             ("zb", 60, lambda r, B: r.integers(20, 90, B))]
    _fused_vs_oracle(skb, D, specs, steps=3, mode="tile", seed=5, k=7, pad=-1.5)


def test_fused_tile_c4_like(skb):
    """C4 shape in miniature: truncated length-k sequences of zipf ids, k = len
    (the head id's run exceeds 8192 positions: packed stage images)."""
    specs = [("zseq", 320, lambda r, B: np.full(B, 200, np.int64))]
    _fused_vs_oracle(skb, 16, specs, steps=3, mode="tile", seed=6, k=200, pad=0.0)


def test_fused_tile_mega_runs_past_k(skb):
    """Tile combiner with bags far longer than k: most positions of the hot
    ids' mega runs fold the zero row (packed images included)."""
    specs = [("zlong", 160, lambda r, B: r.integers(100, 300, B))]
    _fused_vs_oracle(skb, 32, specs, steps=2, mode="tile", seed=7, k=40, pad=0.5)


def test_fused_tile_hot_rows_mid_export_and_mode_switch(skb):
    """C4 in miniature over 7 steps with the rows exported between a backward
    and the next forward every 3rd step (the long-run fold of the hot ids
    runs on its own stream: every reader must see it joined), then a table
    switching from tile to mean bags and back."""
    _fused_vs_oracle(skb, 64, [("zseq", 120, lambda r, B: np.full(B, 400, np.int64))], steps=7, mode="tile", k=400,
                     seed=11, mid_export_every=3)
    _fused_vs_oracle(skb, 16, [("zt", 90, lambda r, B: r.integers(100, 300, B))], steps=6,
                     mode=lambda st: "mean" if st == 4 else "tile", k=40, seed=13, mid_export_every=2)


def test_fused_generic_dim(skb):
    specs = [("a", 64, lambda r, B: r.integers(0, 5, B))]
    _fused_vs_oracle(skb, 3, specs, steps=3, mode="mean", seed=2)


@pytest.mark.parametrize("early", [False, True])
def test_fused_pipelined_prefetch(skb, early):
    """Prefetching step k+1's index phase under step k's fold+Adam (issued
    before or after step k's pool) gives the same table state and pooled
    rows as the unpipelined oracle pipeline."""
    import torch
    rng = np.random.default_rng(21)
    D, members, B, steps = 8, ["a", "b"], 96, 6
    lt = skb.LogicalTable("dim8", D, 1, seed=2, members=members, namespaced=True)
    olt = O.OracleLogical("dim8", D, 1, seed=2, members=members, namespaced=True)
    cfg = skb.AdamConfig(lr=1e-2, weight_decay=0.01, variant="adamw")
    batches, raw = [], []
    for k in range(steps):
        ids = [rng.integers(0, 300 + 100 * k, B * 2) for _ in members]  # new ids keep arriving
        offs = [np.arange(0, 2 * B + 1, 2, dtype=np.int64) for _ in members]
        batches.append(skb.PackedBatch(lt, members, ids, offs))
        raw.append((ids, offs, rng.standard_normal((2 * B, D)).astype(np.float32)))
    skb.prefetch(lt, batches[0], 1, "mean")
    pooled_all = []
    for k in range(steps):
        if early and k + 1 < steps:
            skb.prefetch(lt, batches[k + 1], k + 2, "mean")
        pooled_all.append(skb.lookup_pool(lt, batches[k], k + 1, "mean").clone())
        if not early and k + 1 < steps:
            skb.prefetch(lt, batches[k + 1], k + 2, "mean")
        skb.pool_grad_adam(lt, torch.from_numpy(raw[k][2]).cuda(), cfg, k + 1)
    with pytest.raises(ValueError):
        skb.pool_grad_adam(lt, torch.from_numpy(raw[0][2]).cuda(), cfg, 9)
    for k in range(steps):
        ids, offs, dp = raw[k]
        keys = np.concatenate([olt.keys_for(m, x) for m, x in zip(members, ids)])
        rows = O.lookup(olt, keys, k + 1)
        ref = np.concatenate([O.pool(rows[f * 2 * B:(f + 1) * 2 * B], offs[f], "mean") for f in range(2)])
        eq(pooled_all[k], ref)
        grads = np.repeat(dp / np.float32(2.0), 2, axis=0).astype(np.float32)
        O.grad_update(olt, keys, grads, k + 1, lr=1e-2, weight_decay=0.01, variant="adamw")
    for a, b in zip(lt.local_table.export_rows(), olt.shards[0].export_rows()):
        eq(a, b)


def test_fused_hot_ids_long_runs(skb):
    """Hot ids (runs of thousands of positions) take the CTA-per-run long
    fold; still the exact np.add.at order (mean and sum, D = 8 and 64)."""
    import torch
    # 3000 bags: long runs (cp.async path); 24000 bags: mega runs >= 8192
    # positions (grid-packed stage images + TMA streaming)
    for D, mode, nb in ((64, "mean", 3000), (8, "sum", 3000), (16, "mean", 3000), (64, "mean", 24000),
                        (16, "sum", 24000), (128, "sum", 24000)):
        rng = np.random.default_rng(D + nb)
        members = ["h"]
        lt = skb.LogicalTable(f"dim{D}", D, 1, seed=1, members=members, namespaced=True)
        olt = O.OracleLogical(f"dim{D}", D, 1, seed=1, members=members, namespaced=True)
        cfg = skb.AdamConfig(lr=1e-2, weight_decay=0.01, variant="adamw")
        for step in range(1, 4):
            lens = rng.integers(1, 9, nb)
            offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
            ids = rng.integers(0, 5000, int(offs[-1]))
            hot = rng.random(len(ids)) < 0.6          # 60% of positions on 3 hot ids
            ids[hot] = rng.integers(0, 3, int(hot.sum()))
            batch = skb.PackedBatch(lt, members, [ids], [offs])
            pooled = skb.lookup_pool(lt, batch, step, mode)
            dp = rng.standard_normal((nb, D)).astype(np.float32)
            skb.pool_grad_adam(lt, torch.from_numpy(dp).cuda(), cfg, step)
            keys = olt.keys_for("h", ids)
            rows = O.lookup(olt, keys, step)
            eq(pooled, O.pool(rows, offs, mode))
            g = dp / lens.astype(np.float32)[:, None] if mode == "mean" else dp
            O.grad_update(olt, keys, np.repeat(g, lens, axis=0).astype(np.float32), step, lr=1e-2,
                          weight_decay=0.01, variant="adamw")
        for a, b in zip(lt.local_table.export_rows(), olt.shards[0].export_rows()):
            eq(a, b)


def test_grad_update_hot_ids_long_runs(skb):
    """Drop-in all_to_all_grad_update with 40k-position runs == oracle."""
    rng = np.random.default_rng(12)
    D = 16
    ids = rng.integers(0, 50, 60000)
    ids[rng.random(60000) < 0.7] = 7
    grads = (rng.standard_normal((60000, D)) * rng.choice([1.0, 1e3, 1e-3], (60000, D))).astype(np.float32)
    cfg = skb.AdamConfig(lr=1e-2)
    for S in (1, 3):
        lt = skb.LogicalTable("t", D, S, seed=4)
        olt = O.OracleLogical("t", D, S, seed=4)
        plan = skb.ShardPlan(S)
        eq(skb.all_to_all_lookup(lt, ids, plan, 1), O.lookup(olt, ids, 1))
        skb.all_to_all_grad_update(lt, ids, grads, plan, cfg, 1)
        O.grad_update(olt, ids, grads, 1, lr=1e-2)
        for s in range(S):
            for a, b in zip(lt.shards[s].export_rows(), olt.shards[s].export_rows()):
                eq(a, b)


def test_fused_growth_under_async_snapshots(skb):
    """Every step admits only new ids into a table that starts empty and is
    enqueued without host syncs, so the host's row bound must stay an upper
    bound while its counter snapshots are still in flight (regression: a
    stale snapshot under-reserved the arena and admission wrote past it)."""
    import torch
    D, members, B, steps = 16, ["a"], 60_000, 8
    lt = skb.LogicalTable("dim16", D, 1, seed=3, members=members, namespaced=True)
    olt = O.OracleLogical("dim16", D, 1, seed=3, members=members, namespaced=True)
    cfg = skb.AdamConfig(lr=1e-2)
    offs = [np.arange(B + 1, dtype=np.int64)]
    batches = [skb.PackedBatch(lt, members, [np.arange(k * B, (k + 1) * B, dtype=np.int64)], offs)
               for k in range(steps)]
    dp = torch.zeros((B, D), device="cuda")
    pooled = []
    skb.prefetch(lt, batches[0], 1, "sum")
    for k in range(steps):
        pooled.append(skb.lookup_pool(lt, batches[k], k + 1, "sum").clone())
        if k + 1 < steps:
            skb.prefetch(lt, batches[k + 1], k + 2, "sum")
        skb.pool_grad_adam(lt, dp, cfg, k + 1)
    torch.cuda.synchronize()
    assert lt.num_rows == steps * B
    for k in (0, steps - 1):
        keys = olt.keys_for("a", np.arange(k * B, (k + 1) * B, dtype=np.int64))
        eq(pooled[k], O.pool(O.lookup(olt, keys, k + 1), offs[0], "sum"))


@pytest.mark.parametrize("D", [16, 64])
@pytest.mark.parametrize("mode", ["sum", "mean"])
def test_fused_graph_mode_equals_eager(skb, mode, D):
    """Graph-mode steps (capture on the 2nd call, replay with patched step /
    Adam scalars) leave bit-identical pooled rows and table state; table
    growth and eviction between steps re-prime the graphs.  D=64 bags of 3
    run the streaming pool kernel."""
    import torch
    members, B = ["a", "b"], 64
    cfg = skb.AdamConfig(lr=1e-2, weight_decay=0.01, variant="adamw")
    rng = np.random.default_rng(8)
    specs = []
    for k in range(9):
        hi = 200 if k < 4 else 2000   # new ids keep arriving after step 4: growth
        ids = [rng.integers(0, hi, 3 * B) for _ in members]
        ids[0][: B] = 7                 # a hot id: long runs through the long fold
        offs = [np.arange(0, 3 * B + 1, 3, dtype=np.int64) for _ in members]
        specs.append((ids, offs, rng.standard_normal((2 * B, D)).astype(np.float32)))
    outs = []
    for graphs in (False, True):
        lt = skb.LogicalTable(f"dim{D}", D, 1, seed=4, members=members, namespaced=True, evict_threshold=3)
        skb.use_graphs(lt, graphs)
        # fixed device buffers refilled every step: the graph-replay contract
        bufs = [skb.PackedBatch(lt, members, specs[0][0], specs[0][1]) for _ in range(2)]
        pooled = torch.empty((2 * B, D), device="cuda")
        dp = torch.empty((2 * B, D), device="cuda")
        got = []

        def load(k):
            b = bufs[k % 2]
            b.ids.copy_(torch.from_numpy(np.concatenate(specs[k][0])).cuda())
            return b

        skb.prefetch(lt, load(0), 1, mode)
        for k in range(9):
            if k == 6:  # eviction: drains, rebuilds the IDMap (graphs re-prime)
                skb.lookup_pool(lt, bufs[k % 2], k + 1, mode, out=pooled)
                dp.copy_(torch.from_numpy(specs[k][2]).cuda())
                skb.pool_grad_adam(lt, dp, cfg, k + 1)
                got.append(pooled.cpu().numpy().copy())
                lt.evict(k + 1)
                if k + 1 < 9:
                    skb.prefetch(lt, load(k + 1), k + 2, mode)
                continue
            skb.lookup_pool(lt, bufs[k % 2], k + 1, mode, out=pooled)
            if k + 1 < 9 and k != 5:
                skb.prefetch(lt, load(k + 1), k + 2, mode)
            dp.copy_(torch.from_numpy(specs[k][2]).cuda())
            skb.pool_grad_adam(lt, dp, cfg, k + 1)
            got.append(pooled.cpu().numpy().copy())
        ex = lt.local_table.export_rows()
        outs.append((got, ex))
    for a, b in zip(outs[0][0], outs[1][0]):
        assert np.array_equal(a.view(np.int32), b.view(np.int32))
    for x, y in zip(outs[0][1], outs[1][1]):
        assert np.array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8))


def test_fused_prescaled_backward_matches_train_py(skb):
    """train.py:181-186 builds each position's gradient in float64 as
    float32(dpooled64 / len); pool_grad_adam(prescaled=True) folds exactly
    those rows for mean bags -> bit-exact with the reference's expansion."""
    import torch
    rng = np.random.default_rng(17)
    D, members = 16, ["u", "v"]
    lt = skb.LogicalTable("dim16", D, 1, seed=2, members=members, namespaced=True)
    olt = O.OracleLogical("dim16", D, 1, seed=2, members=members, namespaced=True)
    cfg = skb.AdamConfig(lr=1e-2, weight_decay=0.01, variant="adamw")
    for step in range(1, 4):
        lens = [rng.integers(0, 7, 300) for _ in members]
        offs = [np.concatenate([[0], np.cumsum(l)]).astype(np.int64) for l in lens]
        ids = [rng.integers(0, 400, int(o[-1])) for o in offs]
        batch = skb.PackedBatch(lt, members, ids, offs)
        skb.lookup_pool(lt, batch, step, "mean")
        dp64 = rng.standard_normal((600, D))  # float64, like train.py's dlogits * w
        L = np.concatenate(lens).astype(np.float64)
        g = (dp64 / np.maximum(L, 1.0)[:, None]).astype(np.float32)
        skb.pool_grad_adam(lt, torch.from_numpy(g).cuda(), cfg, step, prescaled=True)
        keys = np.concatenate([olt.keys_for(m, x) for m, x in zip(members, ids)])
        O.lookup(olt, keys, step)
        per_row = np.repeat(dp64 / np.maximum(L, 1.0)[:, None], L.astype(np.int64), axis=0).astype(np.float32)
        O.grad_update(olt, keys, per_row, step, lr=1e-2, weight_decay=0.01, variant="adamw")
    for a, b in zip(lt.local_table.export_rows(), olt.shards[0].export_rows()):
        eq(a, b)


@pytest.mark.parametrize("P", [1, 3, 8])
def test_fused_step_load_stats(skb, P):
    """load_stats of the step's keys (train.py:223-228) from the fused
    step's sorted slots == the reference's load_stats on the same keys."""
    rng = np.random.default_rng(P)
    members = ["a", "b", "c"]
    lt = skb.LogicalTable("dim8", 8, 1, seed=1, members=members, namespaced=True)
    olt = O.OracleLogical("dim8", 8, 1, seed=1, members=members, namespaced=True)
    for step in (1, 2):
        ids = [rng.integers(0, 5000, 4000) for _ in members]
        offs = [np.arange(4001, dtype=np.int64)] * 3
        batch = skb.PackedBatch(lt, members, ids, offs)
        skb.lookup_pool(lt, batch, step, "sum")
        got = skb.step_load_stats(lt, skb.ShardPlan(P))
        keys = np.concatenate([olt.keys_for(m, x) for m, x in zip(members, ids)])
        counts, imbalance = O.shard_load(keys, P)
        eq(got.counts, counts)
        assert got.imbalance == imbalance
        import torch
        skb.pool_grad_adam(lt, torch.zeros((12000, 8), device="cuda"), skb.AdamConfig(), step)


@pytest.mark.parametrize("mode,D", [("sum", 64), ("mean", 16), ("sum", 8)])
def test_fused_tree_fold_within_normwise_bound(skb, mode, D):
    """Opt-in tree fold for hot ids: ids / slots / pooled rows exact; the
    folded gradient of every run within (256 + len/256) * 2^-24 * sum|g|
    per column, carried into Adam's moments; w within a stated relative
    tolerance.  The oracle is re-synced to the GPU rows after every step so
    each step's pooled rows are checked bit-exact from identical weights."""
    import torch
    rng = np.random.default_rng(77 + D)
    members = ["h"]
    lt = skb.LogicalTable(f"dim{D}", D, 1, seed=1, members=members, namespaced=True)
    skb.set_fold_mode(lt, "tree")
    olt = O.OracleLogical(f"dim{D}", D, 1, seed=1, members=members, namespaced=True)
    cfg = skb.AdamConfig(lr=1e-2, weight_decay=0.01, variant="adamw")
    nb = 24000
    for step in (1, 2):
        lens = rng.integers(1, 9, nb)
        offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        ids = rng.integers(0, 5000, int(offs[-1]))
        hot = rng.random(len(ids)) < 0.6
        ids[hot] = rng.integers(0, 3, int(hot.sum()))
        batch = skb.PackedBatch(lt, members, [ids], [offs])
        pooled = skb.lookup_pool(lt, batch, step, mode)
        dp = rng.standard_normal((nb, D)).astype(np.float32)
        skb.pool_grad_adam(lt, torch.from_numpy(dp).cuda(), cfg, step)
        keys = olt.keys_for("h", ids)
        rows = O.lookup(olt, keys, step)
        eq(pooled, O.pool(rows, offs, mode))
        g = dp / lens.astype(np.float32)[:, None] if mode == "mean" else dp
        per = np.repeat(g, lens, axis=0).astype(np.float32)
        O.grad_update(olt, keys, per, step, lr=1e-2, weight_decay=0.01, variant="adamw")
        got, want = lt.local_table.export_rows(), olt.shards[0].export_rows()
        eq(got[0], want[0])
        eq(got[4], want[4])
        # per-run fold bound delta = (256 + len/256) 2^-24 sum|g|
        # through the moments from identical state (the oracle is re-synced to
        # the GPU rows after every step): dm = (1-b1) delta,
        # dv = (1-b2)(2|g| delta + delta^2), plus a few ulps of rounding
        u, inv = np.unique(keys, return_inverse=True)
        absum = np.zeros((len(u), D), np.float64)
        np.add.at(absum, inv, np.abs(per).astype(np.float64))
        gsum = np.zeros((len(u), D), np.float64)
        np.add.at(gsum, inv, per.astype(np.float64))
        cnt = np.bincount(inv, minlength=len(u))[:, None]
        delta = (256 + cnt / 256.0) * 2.0 ** -24 * absum + 1e-30
        j = np.searchsorted(u, want[0])
        hit = (j < len(u)) & (u[np.minimum(j, len(u) - 1)] == want[0])
        j = np.minimum(j, len(u) - 1)
        bm = np.where(hit[:, None], 0.1 * delta[j], 0.0)
        bv = np.where(hit[:, None], 0.001 * (2 * np.abs(gsum[j]) * delta[j] + delta[j] ** 2), 0.0)
        dm_ = np.abs(got[2].astype(np.float64) - want[2])
        dv_ = np.abs(got[3].astype(np.float64) - want[3])
        assert np.all(dm_ <= bm + 4e-7 * np.abs(want[2]) + 1e-30), float((dm_ - bm).max())
        assert np.all(dv_ <= bv + 4e-7 * np.abs(want[3]) + 1e-30), float((dv_ - bv).max())
        np.testing.assert_allclose(got[1], want[1], rtol=1e-5, atol=1e-6)
        tab = olt.shards[0]
        slots = np.array([tab.map[k] for k in got[0].tolist()], np.int64)
        tab.w[slots], tab.m[slots], tab.v[slots] = got[1], got[2], got[3]
