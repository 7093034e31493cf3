"""Row-sharded exchange over torch.distributed (reference sharding.py:230-297).

One process per GPU; rank r owns shard r of every logical table
(`LogicalTable(..., dist=True)`), rows owned by `mix64(key) % S`
(sharding.py:41-43).  Per logical table and step:

forward  (all_to_all_lookup)
  1. local dedup + owner partition                  unique_partition kernel
  2. all-to-all of per-owner counts                 NCCL
  3. all-to-all-v of the unique ids                 NCCL
  4. owner: dedup of the rank-ordered concatenation (= global first-occurrence
     order of the rank-ordered batch, so slots match the oracle fed that
     concatenation bit-exactly), admission + gather
  5. all-to-all-v of the rows back                  NCCL
  6. requester: restore rows to positions           restore kernel
backward (all_to_all_grad_update)
  1. requester pre-aggregates per local unique id in input order
  2. all-to-all-v of the folded grads               NCCL
  3. owner folds across ranks in rank order, admission (last_step), Adam

Grads/optimizer state differ from the single-process reference only by the
association of the cross-rank partial sums (tolerance); ids,
slots and rows are exact.

The protocol is written against a small `ops` interface so it runs with
our CUDA kernels (`GpuOps`, production) or with any other local
implementation (the gloo CPU tests inject an oracle-backed one).  With a
gloo group and CUDA tensors the collectives are staged through host memory.
"""

from __future__ import annotations

import numpy as np

from . import _native as N


class Comm:
    """all-to-all helpers on a process group (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.size = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.backend = dist.get_backend(group)

    def _stage(self, t):
        return t.cpu() if (self.backend == "gloo" and t.is_cuda) else t

    def counts(self, send_counts):
        """Exchange per-peer counts: send_counts[j] goes to rank j."""
        import torch
        dev = "cuda" if self.backend == "nccl" else "cpu"
        s = torch.as_tensor(list(send_counts), dtype=torch.int64, device=dev)
        r = torch.empty_like(s)
        self.dist.all_to_all_single(r, s, group=self.group)
        return [int(x) for x in r.cpu().tolist()]

    def count_matrix(self, send_counts):
        """All ranks' per-owner counts, C[r][s] (one all_gather + one readback)."""
        import torch
        dev = "cuda" if self.backend == "nccl" else "cpu"
        s = torch.as_tensor(list(send_counts), dtype=torch.int64, device=dev)
        out = [torch.empty_like(s) for _ in range(self.size)]
        self.dist.all_gather(out, s, group=self.group)
        return [[int(x) for x in t.cpu().tolist()] for t in out]

    def barrier_after_device_writes(self):
        """Order every rank's peer-memory stores before any rank reads them:
        a one-element all-reduce on the stream (NCCL: no host sync), or a
        device sync + host barrier (gloo)."""
        import torch
        if self.backend == "nccl":
            if getattr(self, "_one", None) is None:
                self._one = torch.zeros(1, device="cuda")
            self.dist.all_reduce(self._one, group=self.group)
        else:
            torch.cuda.synchronize()
            self.dist.barrier(group=self.group)

    def a2av(self, send, send_counts, recv_counts):
        """all_to_all_v along dim 0 with per-peer splits."""
        import torch
        like = send
        src = self._stage(send.contiguous())
        out = torch.empty((sum(recv_counts),) + tuple(send.shape[1:]), dtype=send.dtype, device=src.device)
        self.dist.all_to_all_single(out, src, list(recv_counts), list(send_counts), group=self.group)
        return out.to(like.device) if out.device != like.device else out


class GpuOps:
    """Local steps on this rank's GPU shard, all through libsparsekit_b200."""

    def partition(self, ids, S):
        from .sharding import _partition_dev
        d = N.to_dev(ids, "int64").reshape(-1)
        uniq, counts, inv_s, inv_p = _partition_dev(d, S)
        return uniq, list(counts), inv_s, inv_p

    def dedup(self, ids):
        from .sharding import _partition_dev
        uniq, counts, _, inv = _partition_dev(N.to_dev(ids, "int64").reshape(-1), 1)
        return uniq, inv

    def admit(self, table, uniq, step):
        return table._admit_unique(uniq, step)

    def gather(self, table, offsets):
        rows = N.empty((offsets.numel(), table.dim), "float32")
        if offsets.numel():
            N.call("skb_table_gather_unchecked", table.handle, N.ptr(offsets), offsets.numel(), N.ptr(rows),
                   N.stream_ptr())
        return rows

    def take_rows(self, rows, idx):
        """rows[idx] through the restore kernel (one segment)."""
        n, dim = idx.numel(), rows.shape[1]
        out = N.empty((n, dim), "float32")
        if n:
            zero = N.to_dev(np.zeros(1, np.int64), "int64")
            sh = N.torch().zeros(n, dtype=N.torch().int64, device=idx.device)
            N.call("skb_partition_restore", N.ptr(rows), dim, N.ptr(zero), N.ptr(sh), N.ptr(idx), n, N.ptr(out),
                   N.stream_ptr())
        return out

    def restore(self, rows_cat, counts, inv_s, inv_p):
        n, dim = inv_s.numel(), rows_cat.shape[1]
        out = N.empty((n, dim), "float32")
        if n:
            bases = N.to_dev(np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int64), "int64")
            N.call("skb_partition_restore", N.ptr(rows_cat), dim, N.ptr(bases), N.ptr(inv_s), N.ptr(inv_p), n,
                   N.ptr(out), N.stream_ptr())
        return out

    def global_index(self, counts, inv_s, inv_p):
        bases = N.to_dev(np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int64), "int64")
        return (bases[inv_s] + inv_p).contiguous() if inv_s.numel() else inv_p

    def fold(self, grads, inverse, U):
        dim = grads.shape[1]
        out = N.empty((max(U, 1), dim), "float32")
        n = inverse.numel()
        if n or U:
            N.call("skb_grad_fold", N.ptr(grads), n, dim, N.ptr(inverse), U, N.ptr(out), N.stream_ptr())
        return out[:U]

    def adam(self, table, offsets, grads, cfg, step):
        from .optim import adam_scalars
        if offsets.numel():
            sc = adam_scalars(cfg, step)
            N.call("skb_sparse_adam_step_unchecked", table.handle, N.ptr(offsets), offsets.numel(),
                   N.ptr(grads.contiguous()), N.ctypes_byref(sc), N.stream_ptr())

    def to_device(self, x, dtype):
        return N.to_dev(x, dtype)


def exchange_lookup(comm: Comm, ops, table, keys, step: int, dim: int):
    """Rows for this rank's keys, served by their owner ranks."""
    S = comm.size
    uniq, counts, inv_s, inv_p = ops.partition(keys, S)
    recv_counts = comm.counts(counts)
    recv_ids = comm.a2av(uniq, counts, recv_counts)
    u2, inv2 = ops.dedup(recv_ids)
    offs = ops.admit(table, u2, step)
    rows2 = ops.gather(table, offs)
    send_rows = ops.take_rows(rows2, inv2)
    recv_rows = comm.a2av(send_rows.reshape(-1, dim), recv_counts, counts)
    return ops.restore(recv_rows.reshape(-1, dim), counts, inv_s, inv_p)


def exchange_grad_update(comm: Comm, ops, table, keys, grads, cfg, step: int, dim: int):
    """Pre-aggregate locally, route to owners, fold across ranks, Adam."""
    S = comm.size
    uniq, counts, inv_s, inv_p = ops.partition(keys, S)
    U = int(sum(counts))
    agg = ops.fold(grads, ops.global_index(counts, inv_s, inv_p), U)
    recv_counts = comm.counts(counts)
    recv_ids = comm.a2av(uniq, counts, recv_counts)
    recv_grads = comm.a2av(agg.reshape(-1, dim), counts, recv_counts)
    u2, inv2 = ops.dedup(recv_ids)
    g2 = ops.fold(recv_grads.reshape(-1, dim), inv2, len(u2))
    offs = ops.admit(table, u2, step)
    ops.adam(table, offs, g2, cfg, step)


def _keys_and_comm(lt, ids):
    comm = getattr(lt, "_comm", None)
    if comm is None:
        comm = Comm(lt.group)
        lt._comm = comm
    return comm


def dist_lookup(lt, ids, step: int):
    """all_to_all_lookup for a dist=True LogicalTable (this rank's batch)."""
    as_np = not N.is_torch(ids)
    comm = _keys_and_comm(lt, ids)
    keys = N.to_dev(ids, "int64").reshape(-1)
    out = exchange_lookup(comm, GpuOps(), lt.local_table, keys, step, lt.dim)
    return N.out_like(out, as_np)


def dist_grad_update(lt, ids_d, grads, cfg, step: int):
    """all_to_all_grad_update for a dist=True LogicalTable."""
    if step < 1:
        raise ValueError("global step t must be >= 1")
    comm = _keys_and_comm(lt, ids_d)
    g = N.to_dev(grads, "float32")
    exchange_grad_update(comm, GpuOps(), lt.local_table, ids_d, g, cfg, step, lt.dim)


class P2PWindows:
    """Receive windows in CUDA IPC memory that every peer maps: the producing
    kernel stores rows straight into the consuming rank's window (NVLink P2P
    stores between GPUs; ranks sharing one GPU in the tests).  Grown
    collectively: every rank takes the same decision from the all-gathered
    count matrix, then handles are re-exchanged."""

    def __init__(self, comm: "Comm", dim: int):
        self.comm, self.dim = comm, dim
        self.cap, self.local, self.opened, self.peers_dev = {}, {}, {}, {}

    def ensure(self, name: str, rows_per_rank) -> None:
        need = max(rows_per_rank) if rows_per_rank else 0
        if need <= self.cap.get(name, 0) and name in self.local:
            return
        import ctypes as C
        import torch
        cap = max(need, int(self.cap.get(name, 0) * 1.5), 1024)
        self.close(name)
        ptr, handle = C.c_void_p(), (C.c_char * 64)()
        N.call("skb_ipc_alloc", cap * self.dim * 4, C.byref(ptr), handle)
        handles = [None] * self.comm.size
        self.comm.dist.all_gather_object(handles, bytes(handle), group=self.comm.group)
        peers = []
        for j, h in enumerate(handles):
            if j == self.comm.rank:
                peers.append(ptr.value)
            else:
                q = C.c_void_p()
                N.call("skb_ipc_open", (C.c_char * 64).from_buffer_copy(h), C.byref(q))
                peers.append(q.value)
                self.opened.setdefault(name, []).append(q.value)
        self.local[name], self.cap[name] = ptr.value, cap
        self.peers_dev[name] = torch.tensor(peers, dtype=torch.int64, device="cuda")

    def ptr(self, name: str):
        import ctypes as C
        return C.c_void_p(self.local[name])

    def close(self, name: str) -> None:
        if name not in self.local:
            return
        import ctypes as C
        import torch
        torch.cuda.synchronize()
        self.comm.dist.barrier(group=self.comm.group)  # nobody touches the old windows any more
        for q in self.opened.pop(name, []):
            N.call("skb_ipc_close", C.c_void_p(q))
        N.call("skb_ipc_free", C.c_void_p(self.local.pop(name)))

    def close_all(self) -> None:
        for name in list(self.local):
            self.close(name)


def _prefix(xs):
    out = [0]
    for x in xs:
        out.append(out[-1] + int(x))
    return out


class DistSparseStep:
    """Fused multi-GPU sparse step for one row-sharded logical table.

    forward : member keys (one launch) -> local dedup/partition -> counts +
              ids all-to-all -> owner dedup (rank order) + admission + gather
              -> rows all-to-all back -> pooling straight from the received
              unique rows through the per-position index (no N x D restore).
    backward: per-local-unique ordered fold of dpooled[bag] (/len) -> grads
              all-to-all -> owner cross-rank fold in rank order -> AdamW.
    """

    def __init__(self, lt, comm: Comm | None = None, transport: str = "nccl"):
        if not lt.dist:
            raise ValueError("DistSparseStep needs a LogicalTable built with dist=True")
        if transport not in ("nccl", "p2p"):
            raise ValueError(f"unknown transport {transport!r}")
        self.lt = lt
        self.comm = comm or Comm(lt.group)
        self.ops = GpuOps()
        self.transport = transport
        self.win = P2PWindows(self.comm, lt.dim) if transport == "p2p" else None
        self._ctx = None
        self.last_counts = None

    @staticmethod
    def members_dev(batch):
        """int64[F+1][4] {first position, first bag, salt, strategy} (C-ABI members_dev)."""
        t = N.torch()
        F = len(batch.members)
        if getattr(batch, "_members_dev", None) is None:
            m = np.zeros((F + 1, 4), np.int64)
            m[:, 0] = batch.member_pos
            m[:, 1] = batch.member_bag
            m[:F, 2] = batch.salts.view(np.int64)
            m[:F, 3] = batch.strategy
            batch._members_dev = t.from_numpy(m).cuda()
        return batch._members_dev

    def forward(self, batch, step: int, mode: str = "mean", out=None):
        t = N.torch()
        lt, comm, ops = self.lt, self.comm, self.ops
        D, S, n, G = lt.dim, comm.size, batch.num_ids, batch.num_bags
        F = len(batch.members)
        mdev = self.members_dev(batch)
        if batch.namespaced:
            keys = N.empty((n,), "int64")
            if n:
                N.call("skb_keys_members", N.ptr(batch.ids), n, N.ptr(mdev), F, N.ptr(keys), N.stream_ptr())
        else:
            keys = batch.ids
        uniq, counts, inv_s, inv_p = ops.partition(keys, S)
        gidx = ops.global_index(counts, inv_s, inv_p).to(t.int32)
        cmat = None
        if self.win is None:
            recv_counts = comm.counts(counts)
        else:
            cmat = comm.count_matrix(counts)
            recv_counts = [cmat[r][comm.rank] for r in range(S)]
        recv_ids = comm.a2av(uniq, counts, recv_counts)
        u2, inv2 = ops.dedup(recv_ids)
        offs = ops.admit(lt.local_table, u2, step)
        if self.win is None:
            rows2 = ops.gather(lt.local_table, offs)
            send_rows = ops.take_rows(rows2, inv2)
            recv_rows = comm.a2av(send_rows, recv_counts, counts)
            rows_ptr = N.ptr(recv_rows)
        else:
            # owner gathers each requested row straight into the requester's window
            me = comm.rank
            self.win.ensure("rows", [sum(cmat[j]) for j in range(S)])
            nrecv = int(sum(recv_counts))
            pre = N.to_dev(np.array(_prefix(recv_counts), np.int64), "int64")
            base = N.to_dev(np.array([sum(cmat[j][:me]) for j in range(S)], np.int64), "int64")
            if nrecv:
                N.call("skb_p2p_send_rows", lt.local_table.handle, N.ptr(offs), N.ptr(inv2), nrecv, N.ptr(pre), S,
                       N.ptr(self.win.peers_dev["rows"]), N.ptr(base), N.stream_ptr())
            comm.barrier_after_device_writes()
            rows_ptr = self.win.ptr("rows")
        pooled = out if out is not None else N.empty((G, D), "float32")
        mcode = {"sum": 0, "mean": 1}[mode]
        any_seq = int(bool((batch.strategy == 0).any()))
        if G:
            N.call("skb_pool_indexed", rows_ptr, D, N.ptr(gidx), N.ptr(batch.bag_offs), G, N.ptr(mdev), F,
                   any_seq, mcode, D, N.ptr(pooled), N.stream_ptr())
        self._ctx = dict(batch=batch, counts=counts, recv_counts=recv_counts, gidx=gidx, U=int(sum(counts)),
                         inv2=inv2, u2=u2, offs=offs, mode=mcode, cmat=cmat)
        self.last_counts = {"send": list(counts), "recv": list(recv_counts), "owner_unique": int(u2.numel())}
        return pooled

    def backward(self, dpooled, cfg, step: int):
        c = self._ctx
        if c is None:
            raise ValueError("backward without a preceding forward")
        lt, comm, ops = self.lt, self.comm, self.ops
        D, b = lt.dim, c["batch"]
        g = N.to_dev(dpooled, "float32")
        agg = N.empty((max(c["U"], 1), D), "float32")
        n = b.num_ids
        if n:
            N.call("skb_fold_bags", N.ptr(g), D, N.ptr(c["gidx"]), n, c["U"], N.ptr(b.bag_offs), b.num_bags,
                   c["mode"], max(c["U"] - 1, 0), N.ptr(agg), N.stream_ptr())
        if self.win is None:
            recv_g = comm.a2av(agg[: c["U"]], c["counts"], c["recv_counts"])
            g2 = ops.fold(recv_g, c["inv2"], c["u2"].numel())
        else:
            # requester stores its folded gradients straight into each owner's
            # window, at the owner's rank-ordered receive offset
            cmat, S, me = c["cmat"], comm.size, comm.rank
            self.win.ensure("grads", [sum(cmat[r][s] for r in range(S)) for s in range(S)])
            seg = N.to_dev(np.array(_prefix(c["counts"]), np.int64), "int64")
            base = N.to_dev(np.array([sum(cmat[r][s] for r in range(me)) for s in range(S)], np.int64), "int64")
            if c["U"]:
                N.call("skb_p2p_send_grads", N.ptr(agg), D, c["U"], N.ptr(seg), S, N.ptr(self.win.peers_dev["grads"]),
                       N.ptr(base), N.stream_ptr())
            comm.barrier_after_device_writes()
            nrecv = int(sum(c["recv_counts"]))
            U2 = c["u2"].numel()
            g2 = N.empty((max(U2, 1), D), "float32")
            if nrecv or U2:
                N.call("skb_grad_fold", self.win.ptr("grads"), nrecv, D, N.ptr(c["inv2"]), U2, N.ptr(g2),
                       N.stream_ptr())
            g2 = g2[:U2]
        ops.adam(lt.local_table, c["offs"], g2, cfg, step)
        self._ctx = None
