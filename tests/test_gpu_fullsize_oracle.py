"""BASELINE.json's configs at FULL size against the CPU oracle, bit for bit.

One (or two) fused steps of C2, C4 and C5 at the benchmark's exact shapes,
checked directly against the oracle's train.py call sequence (keys_for ->
all_to_all_lookup -> segment_reduce / segment_tile -> per-position grads ->
all_to_all_grad_update): pooled / tiled outputs and the whole table state
(ids, weights, Adam moments, last_step) after the steps.  The oracle runs
the reference algorithm on the host at ~3e5 ids/s, so these take minutes;
they are marked slow.  Every kernel variant the benchmark runs is pinned
here at the benchmark's own sizes: the TMA fold+Adam ring (C2 step 2), the
staged one-hot pool (C2), the tile combiner with packed mega runs and the
long-run fold (C4), the general mean pool, the feature engine and the
five-table merged step (C5).
"""

import numpy as np
import pytest

from oracle import sparse_oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def same_bits(a, b, what):
    a = a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)
    b = np.asarray(b)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    assert a.dtype == b.dtype, (what, a.dtype, b.dtype)
    if not np.array_equal(a.view(np.uint8), b.view(np.uint8)):
        bad = np.flatnonzero((a != b).reshape(len(a), -1).any(axis=1)) if a.ndim else []
        raise AssertionError(f"{what}: {len(bad)} rows differ, first {bad[:5]}")


def same_tables(gpu_table, oracle_table, what):
    names = ("ids", "weight", "m", "v", "last_step")
    for name, a, b in zip(names, gpu_table.export_rows(), oracle_table.export_rows()):
        same_bits(a, b, f"{what} {name}")


@pytest.fixture(scope="module")
def skb(cuda):
    import paper_2509_20883_b200 as m
    return m


def test_c2_full_size_vs_oracle(skb):
    """C2: 26 x dim64 merged namespaced table, B=65536 one-hot bags, sum,
    SparseAdamW; a cold step (1.65M admissions) then a warm-ish step on which
    the auto kernel choice is the TMA fold+Adam ring."""
    import torch
    F, B, D = 26, 65536, 64
    members = [f"C{f}" for f in range(F)]
    cfg = skb.AdamConfig(lr=1e-3, weight_decay=0.01, variant="adamw")
    lt = skb.merge_tables_by_dim([(m, D) for m in members])[0]
    olt = O.OracleLogical("dim64", D, 1, seed=0, members=members, namespaced=True)
    offs = [np.arange(B + 1, dtype=np.int64)] * F
    for step in (1, 2):
        ids = [np.random.Generator(np.random.PCG64([100 + f, 0, step])).integers(0, 1_000_000, B) for f in range(F)]
        dp = np.random.Generator(np.random.PCG64([7, step])).normal(0, 1e-2, (F * B, D)).astype(np.float32)
        batch = skb.PackedBatch(lt, members, ids, offs)
        pooled = skb.lookup_pool(lt, batch, step, "sum")
        skb.pool_grad_adam(lt, torch.from_numpy(dp).cuda(), cfg, step)
        adam_kernel, pool_kernel = skb.last_variants(lt)
        assert pool_kernel == 4, pool_kernel          # staged one-hot gather
        if step == 2:
            assert adam_kernel == 0, adam_kernel      # k_fused_adam_tma<16,192,4>
        keys = np.concatenate([olt.keys_for(m, x) for m, x in zip(members, ids)])
        rows = O.lookup(olt, keys, step)
        same_bits(pooled, O.pool(rows, np.arange(F * B + 1, dtype=np.int64), "sum"), f"C2 step {step} pooled")
        O.grad_update(olt, keys, dp, step, lr=1e-3, weight_decay=0.01, variant="adamw")
    same_tables(lt.local_table, olt.shards[0], "C2")


def test_c4_full_size_vs_oracle(skb):
    """C4: 8192 zipf(1.1) sequences of length 1000, dim64, truncate(1000,
    'tail') + tile combiner k=1000 -> [8192, 64000]; tile-gradient backward
    (the head id's run is ~780K positions: packed mega runs + long fold)."""
    import torch
    G, L, D = 8192, 1000, 64
    n = G * L
    ids = np.random.Generator(np.random.PCG64(4)).zipf(1.1, n).astype(np.int64)
    offs = np.arange(0, n + 1, L, dtype=np.int64)
    lt = skb.LogicalTable("seq", D, 1, seed=4, members=["seq"], namespaced=False)
    x = skb.RaggedTensor(torch.from_numpy(ids).cuda(), torch.from_numpy(offs).cuda()).truncate(L, "tail")
    batch = skb.PackedBatch(lt, ["seq"], [x.values], [x.row_offsets])
    cfg = skb.AdamConfig(lr=1e-3, weight_decay=0.01, variant="adamw")
    tiles = skb.lookup_pool(lt, batch, 1, "tile", k=L, pad=0.0)
    dtile = np.random.Generator(np.random.PCG64(44)).normal(0, 1e-2, (G, L * D)).astype(np.float32)
    skb.pool_grad_adam(lt, torch.from_numpy(dtile).cuda(), cfg, 1)
    tiles_h = tiles.cpu().numpy()
    del tiles
    olt = O.OracleLogical("seq", D, 1, seed=4, members=["seq"], namespaced=False)
    rows = O.lookup(olt, ids, 1)
    same_bits(tiles_h, O.tile(rows, offs, L, 0.0), "C4 tiles")
    del rows, tiles_h
    # k = L: every position owns exactly one tile row, its gradient
    O.grad_update(olt, ids, dtile.reshape(n, D), 1, lr=1e-3, weight_decay=0.01, variant="adamw")
    same_tables(lt.local_table, olt.shards[0], "C4")


def test_c5_full_size_vs_oracle(skb):
    """C5: 200 features (dims 8..128 -> 5 merged namespaced tables), B=16384,
    mean, ragged bags (10% empty, 1% at 64), with the feature engine in the
    step (hash_feature, fused bucketize, cross + fused mod); cold tables."""
    import torch
    import bench_configs as BC
    from paper_2509_20883_b200.hashing import fnv1a64_packed
    Bn, dims = 16384, BC.DIMS5
    members = {d: [f"f{i}" for i in range(200) if dims[i % 5] == d] for d in dims}
    lts = {d: skb.LogicalTable(f"dim{d}", d, 1, seed=0, members=members[d], namespaced=True) for d in dims}
    olts = {d: O.OracleLogical(f"dim{d}", d, 1, seed=0, members=members[d], namespaced=True) for d in dims}
    cfg = skb.AdamConfig(lr=1e-3, weight_decay=0.01, variant="adamw")
    edges = np.linspace(0.05, 0.95, 10, dtype=np.float32)
    hb = BC._c5_batch(0, Bn)
    # feature engine: GPU vs oracle, column by column
    cols_g, cols_o = [None] * 200, [None] * 200
    blob = np.concatenate([x[0] for x in hb["str"]])
    so, base = [], 0
    for x in hb["str"]:
        so.append(x[1][:-1] + base)
        base += int(x[1][-1])
    so.append(np.array([base], np.int64))
    h = fnv1a64_packed(torch.from_numpy(blob).cuda(), torch.from_numpy(np.concatenate(so)).cuda())
    base = 0
    for j, (b_, s_, o) in enumerate(hb["str"]):
        m = len(s_) - 1
        cols_g[j] = (h[base:base + m], torch.from_numpy(o).cuda())
        cols_o[j] = (O.hash_strings([bytes(b_[s_[q]:s_[q + 1]]) for q in range(m)]), o)
        base += m
    bplan = skb.FusedPlan.for_bucketize([edges] * 20)
    flt = [skb.RaggedTensor(torch.from_numpy(v).cuda(), torch.from_numpy(o).cuda()) for v, o in hb["flt"]]
    for j, r in enumerate(skb.fused_bucketize(bplan, flt)):
        cols_g[20 + j] = (r.values, r.row_offsets)
        cols_o[20 + j] = (O.bucketize_values(hb["flt"][j][0], edges), hb["flt"][j][1])
    crosses = [(skb.RaggedTensor(torch.from_numpy(a).cuda(), torch.from_numpy(oa).cuda()),
                skb.RaggedTensor(torch.from_numpy(c).cuda(), torch.from_numpy(ob).cuda()))
               for a, oa, c, ob in hb["cross"]]
    sizes = [int((np.diff(oa) * np.diff(ob)).sum()) for _, oa, _, ob in hb["cross"]]
    mplan = skb.FusedPlan.for_mod([1_000_003] * 20)
    with skb.deferred_checks():
        crossed = skb.cross_many(crosses, sizes=sizes)
        for j, r in enumerate(skb.fused_mod(mplan, crossed)):
            cols_g[40 + j] = (r.values, r.row_offsets)
    for j, (a, oa, c, ob) in enumerate(hb["cross"]):
        cv, co = O.cross_rows(a, oa, c, ob)
        cols_o[40 + j] = (O.floor_mod(cv, 1_000_003), co)
    for j, (v, o) in enumerate(hb["raw"]):
        cols_g[60 + j] = (torch.from_numpy(v).cuda(), torch.from_numpy(o).cuda())
        cols_o[60 + j] = (v, o)
    for i in range(200):
        same_bits(cols_g[i][0], cols_o[i][0].astype(np.int64), f"C5 feature {i} values")
        same_bits(cols_g[i][1], cols_o[i][1].astype(np.int64), f"C5 feature {i} offsets")
    # the fused step per merged table, against the oracle's train.py sequence
    for di, d in enumerate(dims):
        idx = [i for i in range(200) if i % 5 == di]
        batch = skb.PackedBatch(lts[d], members[d], [cols_g[i][0] for i in idx], [cols_g[i][1] for i in idx])
        pooled = skb.lookup_pool(lts[d], batch, 1, "mean")
        dp = np.random.Generator(np.random.PCG64([55, d])).normal(0, 1e-2, (batch.num_bags, d)).astype(np.float32)
        skb.pool_grad_adam(lts[d], torch.from_numpy(dp).cuda(), cfg, 1)
        keys = np.concatenate([olts[d].keys_for(f"f{i}", cols_o[i][0]) for i in idx])
        rows = O.lookup(olts[d], keys, 1)
        ref, grads, pos, bag = [], [], 0, 0
        for i in idx:
            o = cols_o[i][1]
            m, nb = int(o[-1]), len(o) - 1
            lens = np.diff(o)
            ref.append(O.pool(rows[pos:pos + m], o, "mean"))
            g = dp[bag:bag + nb] / np.maximum(lens, 1).astype(np.float32)[:, None]
            grads.append(np.repeat(g, lens, axis=0).astype(np.float32))
            pos += m
            bag += nb
        same_bits(pooled, np.concatenate(ref), f"C5 dim{d} pooled")
        del rows, ref
        O.grad_update(olts[d], keys, np.concatenate(grads), 1, lr=1e-3, weight_decay=0.01, variant="adamw")
        same_tables(lts[d].local_table, olts[d].shards[0], f"C5 dim{d}")
