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

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

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


def _fused_steps(skb, stepper, lt, rank, cfg, prefetch, sink):
    """STEPS fused steps; prefetch: step k+1's prepare + count exchange issued
    between forward(k) and backward(k) (the cross-step pipeline)."""
    batches = [skb.PackedBatch(lt, MEMBERS, *fused_inputs(rank, k)[:2]) for k in range(STEPS)]
    if prefetch:
        stepper.prefetch(batches[0], 1)
    for k in range(STEPS):
        dp = fused_inputs(rank, k)[2]
        sink(k, stepper.forward(batches[k], k + 1, "mean").cpu().numpy())
        if prefetch and k + 1 < STEPS:
            stepper.prefetch(batches[k + 1], k + 2)
        stepper.backward(torch.from_numpy(dp).cuda(), cfg, k + 1)


def _fused_worker(rank, port, out_dir, barrier="p2p", prefetch=False):
    import torch.distributed as dist
    os.environ["SKB_DIST_BARRIER"] = barrier
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=S)
    import paper_2509_20883_b200 as skb
    from paper_2509_20883_b200.distributed import DistSparseStep
    torch.cuda.set_device(0)
    lt = skb.LogicalTable("dim4", DIM, S, seed=3, members=MEMBERS, namespaced=True, dist=True)
    stepper = DistSparseStep(lt)
    cfg = skb.AdamConfig(lr=LR, weight_decay=0.01, variant="adamw")
    pooled = []
    _fused_steps(skb, stepper, lt, rank, cfg, prefetch, lambda k, x: pooled.append(x))
    ex = lt.local_table.export_rows()
    np.savez(os.path.join(out_dir, f"fused{rank}.npz"), *pooled, ids=ex[0], w=ex[1], m=ex[2], v=ex[3])
    np.save(os.path.join(out_dir, f"grows{rank}.npy"), np.array([stepper.win.grows, stepper.syncs, stepper.p2p_sync]))
    stepper.win.close_all()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("prefetch", [False, True])
@pytest.mark.parametrize("barrier", ["p2p", "comm"])
def test_dist_sparse_step_gpu(tmp_path, cuda, barrier, prefetch):
    """Fused multi-GPU step (2 ranks on one GPU) vs the oracle train.py
    pipeline fed the rank-ordered concatenated batch with S = 2; ordering by
    stream-ordered peer-memory barriers (default) or process-group barriers;
    with and without the cross-step prefetch."""
    mp.spawn(_fused_worker, args=(_free_port(), str(tmp_path), barrier, prefetch), nprocs=S, join=True)
    for r in range(S):
        grows, syncs, p2p = np.load(os.path.join(tmp_path, f"grows{r}.npy")).tolist()
        assert syncs == STEPS                      # one host sync per step: the count matrix
        assert bool(p2p) == (barrier == "p2p")
    _check_fused_vs_oracle(S, lambda r: np.load(os.path.join(tmp_path, f"fused{r}.npz")))


def _check_fused_vs_oracle(W, load):
    """Every rank's pooled rows and table shard vs the oracle fed the
    rank-ordered concatenation with W shards (first step exact)."""
    olt = O.OracleLogical("dim4", DIM, W, seed=3, members=MEMBERS, namespaced=True)
    for k in range(STEPS):
        ins = [fused_inputs(r, k) for r in range(W)]
        keys = np.concatenate([olt.keys_for(m, ins[r][0][f]) for r in range(W) for f, m in enumerate(MEMBERS)])
        rows = O.lookup(olt, keys, k + 1)
        pos, grads = 0, []
        for r in range(W):
            ref = []
            for f in range(len(MEMBERS)):
                o = ins[r][1][f]
                n_f = int(o[-1])
                ref.append(O.pool(rows[pos:pos + n_f], o, "mean"))
                lens = np.diff(o)
                g = ins[r][2][f * FB:(f + 1) * FB] / np.maximum(lens, 1).astype(np.float32)[:, None]
                grads.append(np.repeat(g, lens, axis=0).astype(np.float32))
                pos += n_f
            got = load(r)[f"arr_{k}"]
            if k == 0:
                assert np.array_equal(got.view(np.int32), np.concatenate(ref).view(np.int32))
            else:
                np.testing.assert_allclose(got, np.concatenate(ref), rtol=1e-5, atol=1e-6)
        O.grad_update(olt, keys, np.concatenate(grads), k + 1, lr=LR, weight_decay=0.01, variant="adamw")
    for r in range(W):
        z = load(r)
        ex = olt.shards[r].export_rows()
        assert np.array_equal(z["ids"], ex[0])
        for key, j in (("w", 1), ("m", 2), ("v", 3)):
            np.testing.assert_allclose(z[key], ex[j], rtol=1e-5, atol=1e-6)


@pytest.mark.gpu
@pytest.mark.parametrize("prefetch", [False, True])
@pytest.mark.parametrize("W", [2, 3])
def test_dist_sparse_step_thread_ranks(cuda, W, prefetch):
    """The multi-GPU protocol with W ranks as threads of one process on one
    GPU (ThreadRanks: plain-pointer windows, stream-ordered peer barriers,
    every rank on its own stream) vs the oracle."""
    import threading
    import paper_2509_20883_b200 as skb
    from paper_2509_20883_b200.distributed import DistSparseStep, ThreadRanks
    world = ThreadRanks(W)
    out, errs = [None] * W, []

    def body(rank):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                lt = skb.LogicalTable("dim4", DIM, W, seed=3, members=MEMBERS, namespaced=True, dist=True,
                                      group=world.group(rank))
                stepper = DistSparseStep(lt)
                assert stepper.p2p_sync
                cfg = skb.AdamConfig(lr=LR, weight_decay=0.01, variant="adamw")
                res = {}
                _fused_steps(skb, stepper, lt, rank, cfg, prefetch, lambda k, x: res.__setitem__(f"arr_{k}", x))
                ex = lt.local_table.export_rows()
                res.update(ids=ex[0], w=ex[1], m=ex[2], v=ex[3])
                assert stepper.syncs == STEPS
                stepper.win.close_all()
                out[rank] = res
        except BaseException as e:
            errs.append(repr(e))
            world._barrier.abort()

    ths = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(W)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout=300)
    assert not any(t.is_alive() for t in ths), "thread ranks did not finish (deadlock?)"
    assert not errs, errs
    _check_fused_vs_oracle(W, lambda r: out[r])


@pytest.mark.parametrize("S", [1, 2, 3, 5, 8])
def test_exchange_plan_places_every_row(S):
    """CPU: the ExchangePlan offsets move every id, row and gradient to the
    place the reference's per-shard lists define.  Simulated windows: each
    rank's unique list split by owner, ids stored into owner windows, rows
    stored back into requester windows, grads into owner windows."""
    from paper_2509_20883_b200.distributed import ExchangePlan
    rng = np.random.default_rng(S)
    cmat = rng.integers(0, 7, (S, S)).tolist()
    # rank q's unique list: owner-concatenated, each id tagged (q, owner, k)
    uniq = {q: [(q, j, k) for j in range(S) for k in range(cmat[q][j])] for q in range(S)}
    plans = [ExchangePlan(cmat, r) for r in range(S)]
    id_win = {j: [None] * plans[0].recv_need[j] for j in range(S)}
    for q in range(S):
        p = plans[q]
        for i, x in enumerate(uniq[q]):
            j = next(j for j in range(S) if p.send_pre[j] <= i < p.send_pre[j + 1])
            id_win[j][p.to_owner_base[j] + i - p.send_pre[j]] = x
    for j in range(S):  # owner windows: rank-ordered segments, each in the requester's order
        assert id_win[j] == [x for q in range(S) for x in uniq[q] if x[1] == j]
        assert len(id_win[j]) == plans[j].n_recv
    row_win = {q: [None] * plans[0].rows_need[q] for q in range(S)}
    for j in range(S):  # owner j sends received position i's "row" (the id itself) back
        p = plans[j]
        for i, x in enumerate(id_win[j]):
            q = next(q for q in range(S) if p.recv_pre[q] <= i < p.recv_pre[q + 1])
            row_win[q][p.to_req_base[q] + i - p.recv_pre[q]] = x
    for q in range(S):  # every requester gets its rows in its own unique order
        assert row_win[q] == uniq[q]


@pytest.mark.gpu
def test_dist_sparse_step_one_host_sync(tmp_path, cuda):
    """The fused multi-GPU step (2 ranks on one GPU): window growth happens
    only when the batch outgrows the windows, and the step's host
    synchronisation is the count matrix (table counter refreshes stay off
    the steady-state path)."""
    mp.spawn(_fused_worker, args=(_free_port(), str(tmp_path)), nprocs=S, join=True)
    for r in range(S):
        grows = int(np.load(os.path.join(tmp_path, f"grows{r}.npy"))[0])
        assert grows <= 9, grows  # 2 flag windows + counts once; 3 data windows created once, grown once for the 30x step


@pytest.mark.gpu
def test_exchange_protocol_gpu_kernels(tmp_path, cuda):
    _run(tmp_path, use_gpu=True)


def test_bench_self_launch_command():
    """`bench.py --gpus N` started without torchrun re-executes itself under
    torch.distributed.run with N ranks on 127.0.0.1."""
    import bench
    cmd = bench.launch_cmd(["--gpus", "4", "--steps", "3"], 4, 29555)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd and "--master-port=29555" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "3"] and cmd[-5].endswith("bench.py")


def test_bench_gpus_n_fails_loudly_without_gpus():
    """No silent single-GPU run for --gpus 2: with fewer visible GPUs the
    launcher prints an error line and exits non-zero."""
    import json
    import subprocess
    import sys
    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("enough GPUs: the launcher would really run")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "BENCH_SHARED_GPU")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "1"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 2, (r.returncode, r.stderr[-2000:])
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and "needs 2 visible GPUs" in line["error"]
