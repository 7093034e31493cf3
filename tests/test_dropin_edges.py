"""Drop-in edge cases of the reference API (round 2): IDMap edits outside
admission (remove / put / free_list mutation) with eviction and export
following dict membership, negative eviction thresholds, float64 / integer
segment rows, the fused pipeline's prefetch contract, counter reads after a
prefetch, and caller-supplied cross sizes.

Golden values: tests/golden/golden_edges.npz, written by
`python tests/golden/make_golden.py edges` from the reference itself; the
trace drivers live in make_golden.py so the reference, the oracle and the
GPU table run the very same call sequence.
"""

import importlib.util
import os

import numpy as np
import pytest

from oracle import sparse_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))


def _drivers():
    spec = importlib.util.spec_from_file_location("make_golden", os.path.join(HERE, "golden", "make_golden.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


@pytest.fixture(scope="module")
def gold():
    with np.load(os.path.join(HERE, "golden", "golden_edges.npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def _check_trace(drive, table, prefix, gold):
    seen = set()

    def log(name, *arrs):
        for i, a in enumerate(arrs):
            key = f"{prefix}.{name}.{i}"
            want = gold[key]
            got = np.asarray(a.cpu().numpy() if hasattr(a, "cpu") else a)
            assert got.shape == want.shape, (key, got.shape, want.shape)
            if got.size:
                assert np.array_equal(got.view(np.uint8), want.astype(got.dtype).view(np.uint8)), key
            seen.add(key)
    drive(table, log)
    assert seen == {k for k in gold if k.startswith(prefix + ".")}


class _OracleIDMap:
    """The reference's IDMap attributes over an OracleTable's dict + list."""

    def __init__(self, t):
        self.t = t

    def __len__(self):
        return len(self.t.map)

    def remove(self, fid):
        return self.t.map.pop(int(fid))

    def put(self, fid, slot):
        self.t.map[int(fid)] = int(slot)

    @property
    def free_list(self):
        return self.t.free


class _OracleTable:
    def __init__(self, *a, **k):
        self.t = O.OracleTable(*a, **k)
        self.idmap = _OracleIDMap(self.t)

    def __getattr__(self, name):
        return getattr(self.t, name)


def test_oracle_edge_traces_match_reference(gold):
    """CPU: the oracle reproduces the reference's IDMap-edit / negative
    threshold traces (pins the oracle for the GPU tests below)."""
    d = _drivers()
    _check_trace(d.table_edge_trace, _OracleTable(4, seed=2, block_size=4, evict_threshold=2), "idmap", gold)
    _check_trace(d.negative_threshold_trace, _OracleTable(4, seed=2, block_size=4, evict_threshold=-1), "negthr",
                 gold)


def test_free_list_proxy_is_a_list():
    """CPU: FreeList keeps list semantics and writes back after every
    in-place mutation (no device needed: the write-back is stubbed)."""
    from paper_2509_20883_b200.embedding import FreeList
    pushed = []

    class P(FreeList):
        def _push(self):
            pushed.append(list(self))

    fl = P(None, [1, 2, 3])
    fl.append(4)
    fl.reverse()
    assert fl.pop() == 1
    fl += [9]
    fl[0] = 7
    del fl[1]
    assert fl == [7, 2, 9] and isinstance(fl, list)
    assert pushed == [[1, 2, 3, 4], [4, 3, 2, 1], [4, 3, 2], [4, 3, 2, 9], [7, 3, 2, 9], [7, 2, 9]]


@pytest.mark.gpu
def test_gpu_idmap_edits_evict_export(skb, gold):
    """IDMap.remove / put and free_list mutation: export and eviction follow
    dict membership (a removed id's live slot is neither exported nor
    evicted; a put entry is), bit-exact with the reference trace."""
    d = _drivers()
    _check_trace(d.table_edge_trace, skb.EmbeddingTable("e", 4, seed=2, block_size=4, evict_threshold=2), "idmap",
                 gold)


@pytest.mark.gpu
def test_gpu_negative_evict_threshold(skb, gold):
    d = _drivers()
    _check_trace(d.negative_threshold_trace, skb.EmbeddingTable("n", 4, seed=2, block_size=4, evict_threshold=-1),
                 "negthr", gold)


@pytest.mark.gpu
def test_gpu_free_list_rejects_bad_slots(skb):
    t = skb.EmbeddingTable("f", 4, block_size=4)
    t.lookup_or_insert(np.arange(3), 1)
    with pytest.raises(ValueError, match="outside the store"):
        t.idmap.free_list = [1, 10**9]
    t.idmap.free_list = [2]
    assert t.idmap.free_list == [2]


@pytest.mark.gpu
def test_gpu_segments_keep_dtype(skb, gold):
    """float64 rows fold in double in the reference's orders; integer rows
    sum in their own dtype; mean of integer rows raises TypeError."""
    import torch
    offs, r64, ri = gold["seg64.offs"], gold["seg64.rows"], gold["segi.rows"]

    def same(a, b):
        a = np.asarray(a)
        assert a.dtype == b.dtype and a.shape == b.shape
        assert np.array_equal(a.view(np.uint8), b.view(np.uint8))

    for mode in ("sum", "mean"):
        for strat in ("sequential", "scatter", "auto"):
            same(skb.segment_reduce(r64, offs, mode, strat), gold[f"seg64.{mode}.{strat}"])
    for strat in ("sequential", "scatter"):
        same(skb.segment_reduce(ri, offs, "sum", strat), gold[f"segi.sum.{strat}"])
        same(skb.segment_reduce(ri.astype(np.int32), offs, "sum", strat), gold[f"segi32.sum.{strat}"])
    same(skb.segment_tile(r64, offs, 4, pad=-2.5), gold["seg64.tile4"])
    same(skb.segment_tile(ri, offs, 4, pad=-7), gold["segi.tile4"])
    # CUDA tensors in -> CUDA tensors out, dtype kept
    out = skb.segment_reduce(torch.from_numpy(r64).cuda(), torch.from_numpy(offs).cuda(), "sum", "sequential")
    assert out.dtype == torch.float64
    same(out.cpu().numpy(), gold["seg64.sum.sequential"])
    with pytest.raises(TypeError):
        skb.segment_reduce(ri, offs, "mean")
    with pytest.raises(TypeError):
        skb.segment_reduce(r64.astype(np.float16), offs)


@pytest.mark.gpu
def test_gpu_prefetch_contract(skb):
    """Table edits that would change slots a prefetched (admitted, not yet
    pooled) batch already holds raise ValueError and leave the table as it
    was; after the step completes they run normally."""
    import torch
    D = 8
    lt = skb.LogicalTable("dim8", D, 1, seed=1, members=["a"], namespaced=False, evict_threshold=0)
    t = lt.local_table
    cfg = skb.AdamConfig(lr=1e-2)
    b1 = skb.PackedBatch(lt, ["a"], [np.arange(64)], [np.arange(65)])
    b2 = skb.PackedBatch(lt, ["a"], [np.arange(32, 96)], [np.arange(65)])
    skb.lookup_pool(lt, b1, 1, "sum")
    skb.pool_grad_adam(lt, torch.zeros((64, D), device="cuda"), cfg, 1)
    skb.prefetch(lt, b2, 2, "sum")
    before = t.export_rows()
    for op in (lambda: t.evict(5), lambda: t.idmap.remove(3), lambda: t.idmap.put(999, 1),
               lambda: t.restore_rows([5000], np.zeros((1, D), np.float32), np.zeros((1, D), np.float32),
                                      np.zeros((1, D), np.float32), [1]),
               lambda: t.scatter_update(np.array([0]), np.zeros((1, D), np.float32))):
        with pytest.raises(ValueError, match="prefetched"):
            op()
    skb.lookup_pool(lt, b2, 2, "sum")
    with pytest.raises(ValueError, match="between a fused lookup_pool"):
        t.evict(5)
    skb.pool_grad_adam(lt, torch.zeros((64, D), device="cuda"), cfg, 2)
    after = t.export_rows()
    assert len(after[0]) == 96 and set(before[0].tolist()) <= set(after[0].tolist())
    assert t.evict(5) == 96


@pytest.mark.gpu
def test_gpu_counters_after_prefetch(skb):
    """num_rows / export_rows right after a prefetch see that batch's
    admission (the counter read waits for the index stream), and the next
    step still reserves enough rows."""
    import torch
    D = 16
    lt = skb.LogicalTable("dim16", D, 1, seed=3, members=["a"], namespaced=False)
    cfg = skb.AdamConfig(lr=1e-2)
    B = 50_000
    batches = [skb.PackedBatch(lt, ["a"], [np.arange(k * B, (k + 1) * B)], [np.arange(B + 1)]) for k in range(4)]
    skb.prefetch(lt, batches[0], 1, "sum")
    for k in range(4):
        skb.lookup_pool(lt, batches[k], k + 1, "sum")
        if k + 1 < 4:
            skb.prefetch(lt, batches[k + 1], k + 2, "sum")
            assert lt.num_rows == (k + 2) * B
        skb.pool_grad_adam(lt, torch.zeros((B, D), device="cuda"), cfg, k + 1)
    assert len(lt.local_table.export_rows()[0]) == 4 * B


def test_deferred_verdicts_in_record_order():
    """CPU: deferred_checks' read-back raises the first recorded failure —
    plain flags (ValueError with the message) and verdict callables (their
    exception, or None) in one read, in recording order."""
    import torch
    from paper_2509_20883_b200 import features as F
    ok = torch.full((4,), -1, dtype=torch.int64)
    seen = []
    recs = [(torch.tensor([-1]), "never"),
            (ok, lambda v: seen.append(v) or None),
            (torch.tensor([-1, 7, -1, -1]), lambda v: IndexError(f"bad {v[1]}")),
            (torch.tensor([3]), "later")]
    with pytest.raises(IndexError, match="bad 7"):
        F._raise_pending(recs)
    assert seen == [[-1, -1, -1, -1]]
    with pytest.raises(ValueError, match="later"):
        F._raise_pending(recs[:2] + recs[3:])
    F._raise_pending([])


@pytest.mark.gpu
def test_gpu_cross_many_batched(skb):
    """cross_many's two-launch path (per-pair descriptors) against the
    oracle pair by pair: empty rows, empty pairs, zero-row pairs, mixed
    sizes, and more pairs than one launch takes (chunked)."""
    import torch
    from oracle import sparse_oracle as O
    rng = np.random.default_rng(9)
    pairs, host = [], []
    for p in range(1100):
        rows = 0 if p % 97 == 5 else int(rng.integers(1, 40))
        la = rng.integers(0, 4, rows) * (p % 13 != 3)
        lb = rng.integers(0, 5, rows)
        oa, ob = np.concatenate([[0], np.cumsum(la)]), np.concatenate([[0], np.cumsum(lb)])
        a = rng.integers(-2**62, 2**62, int(oa[-1]))
        b = rng.integers(-2**62, 2**62, int(ob[-1]))
        host.append((a, oa, b, ob))
        dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
        pairs.append((skb.RaggedTensor(dev(a), dev(oa)), skb.RaggedTensor(dev(b), dev(ob))))
    sizes = [int((np.diff(oa) * np.diff(ob)).sum()) for _, oa, _, ob in host]
    for kw in ({}, {"sizes": sizes}):
        with skb.deferred_checks():
            got = skb.cross_many(pairs, **kw)
        assert len(got) == len(pairs)
        for r, (a, oa, b, ob) in zip(got, host):
            v, o = O.cross_rows(a, oa, b, ob)
            assert np.array_equal(r.values.cpu().numpy(), v) and np.array_equal(r.row_offsets.cpu().numpy(), o)


@pytest.mark.gpu
def test_gpu_cross_many_sizes_checked(skb):
    """cross_many(sizes=...) trusts nothing: a wrong size raises ValueError
    (synchronously, or at deferred_checks exit) and never reads past the
    inputs."""
    rng = np.random.default_rng(3)
    lens_a, lens_b = rng.integers(0, 4, 50), rng.integers(0, 4, 50)
    a = skb.RaggedTensor(rng.integers(0, 100, int(lens_a.sum())), np.concatenate([[0], np.cumsum(lens_a)]))
    b = skb.RaggedTensor(rng.integers(0, 100, int(lens_b.sum())), np.concatenate([[0], np.cumsum(lens_b)]))
    true = int((lens_a * lens_b).sum())
    ref = skb.cross(a, b)
    (ok,) = skb.cross_many([(a, b)], sizes=[true])
    assert np.array_equal(ok.values, ref.values)
    import torch
    ad = skb.RaggedTensor(torch.from_numpy(a.values).cuda(), torch.from_numpy(a.row_offsets).cuda())
    bd = skb.RaggedTensor(torch.from_numpy(b.values).cuda(), torch.from_numpy(b.row_offsets).cuda())
    for bad in (true - 1, true + 5):
        with pytest.raises(ValueError, match="sizes"):
            skb.cross_many([(a, b)], sizes=[bad])
        with pytest.raises(ValueError, match="sizes"):
            with skb.deferred_checks():
                skb.cross_many([(a, b)], sizes=[bad])
        with pytest.raises(ValueError, match="sizes"):  # device results: raised at the context exit
            with skb.deferred_checks():
                (r,) = skb.cross_many([(ad, bd)], sizes=[bad])
                assert r.values.numel() == bad
