"""N > 1 exchange protocol (paper_2509_20883_b200/distributed.py) on world_size-2
process groups.

CPU (gloo): the protocol driven by oracle-backed local ops; checks rows and
slots bit-exactly against the single-process oracle fed the rank-ordered
concatenated batch, and grads/optimizer state within tolerance (cross-rank
partial sums change the association).
GPU (gloo staging, both ranks on cuda:0): the same protocol over our kernels.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle import sparse_oracle as O

S = 2
DIM = 4
STEPS = 4
LR = 0.05


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def batches(rank):
    rng = np.random.default_rng(100 + rank)
    return [rng.integers(-30, 60, 40 + 7 * rank).astype(np.int64) for _ in range(STEPS)]


def grads_for(rank, step, n):
    return np.random.default_rng(1000 * rank + step).standard_normal((n, DIM)).astype(np.float32)


class OracleOps:
    """Local steps restated with the CPU oracle (test-only)."""

    def partition(self, keys, S):
        shards, inv_s, inv_p = O.dedup_partition(keys.numpy(), S)
        return (torch.from_numpy(np.concatenate(shards)), [len(s) for s in shards],
                torch.from_numpy(inv_s), torch.from_numpy(inv_p))

    def dedup(self, ids):
        shards, _, inv = O.dedup_partition(ids.numpy(), 1)
        return torch.from_numpy(shards[0]), torch.from_numpy(inv)

    def admit(self, table, uniq, step):
        return torch.from_numpy(table.lookup_or_insert(uniq.numpy(), step))

    def gather(self, table, offs):
        return torch.from_numpy(table.gather(offs.numpy()))

    def take_rows(self, rows, idx):
        return rows[idx]

    def global_index(self, counts, inv_s, inv_p):
        bases = torch.from_numpy(np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int64))
        return bases[inv_s] + inv_p

    def restore(self, rows_cat, counts, inv_s, inv_p):
        return rows_cat[self.global_index(counts, inv_s, inv_p)]

    def fold(self, grads, inverse, U):
        return torch.from_numpy(O.fold_grads(inverse.numpy(), grads.numpy(), U))

    def adam(self, table, offs, g, cfg, step):
        O.sparse_adam(table, offs.numpy(), g.numpy(), lr=LR, weight_decay=0.01, variant="adamw", t=step)


def _worker(rank, port, out_dir, use_gpu):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=S)
    from paper_2509_20883_b200 import distributed as D
    comm = D.Comm()
    rows_out = []
    if use_gpu:
        import paper_2509_20883_b200 as skb
        torch.cuda.set_device(0)
        ops = D.GpuOps()
        table = skb.EmbeddingTable(f"shard{rank}", DIM, seed=7)
        cfg = skb.AdamConfig(lr=LR, weight_decay=0.01, variant="adamw")
        for step, ids in enumerate(batches(rank), start=1):
            keys = torch.from_numpy(ids).cuda()
            rows_out.append(D.exchange_lookup(comm, ops, table, keys, step, DIM).cpu().numpy())
            g = torch.from_numpy(grads_for(rank, step, len(ids))).cuda()
            D.exchange_grad_update(comm, ops, table, keys, g, cfg, step, DIM)
        ex = table.export_rows()
        slots = table.idmap.get_many(ex[0])
    else:
        ops = OracleOps()
        table = O.OracleTable(DIM, seed=7)
        for step, ids in enumerate(batches(rank), start=1):
            keys = torch.from_numpy(ids)
            rows_out.append(D.exchange_lookup(comm, ops, table, keys, step, DIM).numpy())
            D.exchange_grad_update(comm, ops, table, keys, torch.from_numpy(grads_for(rank, step, len(ids))),
                                   None, step, DIM)
        ex = table.export_rows()
        slots = np.array([table.map[int(i)] for i in ex[0]], np.int64)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), *rows_out, ids=ex[0], w=ex[1], m=ex[2], v=ex[3],
             last=ex[4], slots=slots)
    dist.barrier()
    dist.destroy_process_group()


def _reference():
    """Single-process oracle with S shards fed the rank-ordered concatenation."""
    lt = O.OracleLogical("t", DIM, S, seed=7)
    rows = {r: [] for r in range(S)}
    per_rank = [batches(r) for r in range(S)]
    for k in range(STEPS):
        ids = np.concatenate([per_rank[r][k] for r in range(S)])
        out = O.lookup(lt, ids, k + 1)
        pos = 0
        for r in range(S):
            n = len(per_rank[r][k])
            rows[r].append(out[pos:pos + n])
            pos += n
        g = np.concatenate([grads_for(r, k + 1, len(per_rank[r][k])) for r in range(S)])
        O.grad_update(lt, ids, g, k + 1, lr=LR, weight_decay=0.01, variant="adamw")
    return lt, rows


def _run(tmp_path, use_gpu):
    port = _free_port()
    mp.spawn(_worker, args=(port, str(tmp_path), use_gpu), nprocs=S, join=True)
    lt, ref_rows = _reference()
    for r in range(S):
        z = np.load(os.path.join(tmp_path, f"rank{r}.npz"))
        for k in range(STEPS):
            got = z[f"arr_{k}"]
            if k == 0:  # fresh rows: initializer only -> exact
                assert np.array_equal(got.view(np.int32), ref_rows[r][k].view(np.int32))
            else:       # rows after cross-rank-summed updates -> tolerance
                np.testing.assert_allclose(got, ref_rows[r][k], rtol=1e-5, atol=1e-6)
        ex = lt.shards[r].export_rows()
        assert np.array_equal(z["ids"], ex[0])          # ownership + admission exact
        assert np.array_equal(z["last"], ex[4])
        assert np.array_equal(z["slots"], [lt.shards[r].map[int(i)] for i in ex[0]])  # slots exact
        for key, j in (("w", 1), ("m", 2), ("v", 3)):
            np.testing.assert_allclose(z[key], ex[j], rtol=1e-5, atol=1e-6)
    # slot assignment is exact: the owner's offsets for every id equal the oracle's
    return lt


def test_exchange_protocol_gloo_cpu(tmp_path):
    _run(tmp_path, use_gpu=False)


# ---- the fused multi-GPU step (DistSparseStep) ------------------------------
MEMBERS = ["a", "b"]
FB = 48  # bags per member per rank


def fused_inputs(rank, k):
    rng = np.random.default_rng(500 + 10 * rank + k)
    ids, offs = [], []
    for _ in MEMBERS:
        # step 2 carries ~30x the positions: the P2P windows must grow collectively
        lens = rng.integers(0, 4, FB) if k != 2 else rng.integers(20, 100, FB)
        offs.append(np.concatenate([[0], np.cumsum(lens)]).astype(np.int64))
        ids.append(rng.integers(0, 80 if k != 2 else 4000, int(lens.sum())).astype(np.int64))
    dp = rng.standard_normal((len(MEMBERS) * FB, DIM)).astype(np.float32)
    return ids, offs, dp


def _fused_worker(rank, port, out_dir, transport="nccl"):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=S)
    import paper_2509_20883_b200 as skb
    from paper_2509_20883_b200.distributed import DistSparseStep
    torch.cuda.set_device(0)
    lt = skb.LogicalTable("dim4", DIM, S, seed=3, members=MEMBERS, namespaced=True, dist=True)
    stepper = DistSparseStep(lt, transport=transport)
    cfg = skb.AdamConfig(lr=LR, weight_decay=0.01, variant="adamw")
    pooled = []
    for k in range(STEPS):
        ids, offs, dp = fused_inputs(rank, k)
        batch = skb.PackedBatch(lt, MEMBERS, ids, offs)
        pooled.append(stepper.forward(batch, k + 1, "mean").cpu().numpy())
        stepper.backward(torch.from_numpy(dp).cuda(), cfg, k + 1)
    ex = lt.local_table.export_rows()
    np.savez(os.path.join(out_dir, f"fused{rank}.npz"), *pooled, ids=ex[0], w=ex[1], m=ex[2], v=ex[3])
    if stepper.win is not None:
        stepper.win.close_all()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_dist_sparse_step_gpu(tmp_path, cuda):
    """Fused multi-GPU step (2 ranks on one GPU, gloo staging) vs the oracle
    train.py pipeline fed the rank-ordered concatenated batch with S = 2."""
    mp.spawn(_fused_worker, args=(_free_port(), str(tmp_path)), nprocs=S, join=True)
    olt = O.OracleLogical("dim4", DIM, S, seed=3, members=MEMBERS, namespaced=True)
    for k in range(STEPS):
        ins = [fused_inputs(r, k) for r in range(S)]
        # concatenation: rank 0's member-a ids, member-b ids, then rank 1's ...
        keys = np.concatenate([olt.keys_for(m, ins[r][0][f]) for r in range(S) for f, m in enumerate(MEMBERS)])
        rows = O.lookup(olt, keys, k + 1)
        pos, grads = 0, []
        for r in range(S):
            ref = []
            for f in range(len(MEMBERS)):
                o = ins[r][1][f]
                n_f = int(o[-1])
                ref.append(O.pool(rows[pos:pos + n_f], o, "mean"))
                lens = np.diff(o)
                g = ins[r][2][f * FB:(f + 1) * FB] / np.maximum(lens, 1).astype(np.float32)[:, None]
                grads.append(np.repeat(g, lens, axis=0).astype(np.float32))
                pos += n_f
            got = np.load(os.path.join(tmp_path, f"fused{r}.npz"))[f"arr_{k}"]
            if k == 0:
                assert np.array_equal(got.view(np.int32), np.concatenate(ref).view(np.int32))
            else:
                np.testing.assert_allclose(got, np.concatenate(ref), rtol=1e-5, atol=1e-6)
        O.grad_update(olt, keys, np.concatenate(grads), k + 1, lr=LR, weight_decay=0.01, variant="adamw")
    for r in range(S):
        z = np.load(os.path.join(tmp_path, f"fused{r}.npz"))
        ex = olt.shards[r].export_rows()
        assert np.array_equal(z["ids"], ex[0])
        for key, j in (("w", 1), ("m", 2), ("v", 3)):
            np.testing.assert_allclose(z[key], ex[j], rtol=1e-5, atol=1e-6)


@pytest.mark.gpu
def test_dist_sparse_step_p2p_transport(tmp_path, cuda):
    """Peer-memory transport (rows gathered straight into the requester's IPC
    window, folded grads stored straight into the owner's window) is
    bit-identical to the all_to_all transport (2 ranks sharing one GPU)."""
    a, b = tmp_path / "a2a", tmp_path / "p2p"
    a.mkdir()
    b.mkdir()
    mp.spawn(_fused_worker, args=(_free_port(), str(a), "nccl"), nprocs=S, join=True)
    mp.spawn(_fused_worker, args=(_free_port(), str(b), "p2p"), nprocs=S, join=True)
    for r in range(S):
        za, zb = np.load(a / f"fused{r}.npz"), np.load(b / f"fused{r}.npz")
        assert sorted(za.files) == sorted(zb.files)
        for k in za.files:
            assert np.array_equal(za[k].view(np.uint8), zb[k].view(np.uint8)), k


@pytest.mark.gpu
def test_exchange_protocol_gpu_kernels(tmp_path, cuda):
    _run(tmp_path, use_gpu=True)
