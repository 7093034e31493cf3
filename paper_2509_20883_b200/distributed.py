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

import os

import numpy as np

from . import _native as N


class ThreadRanks:
    """S ranks of one process, one thread each, sharing one GPU context —
    the multi-GPU step's protocol run with every rank's kernels on its own
    stream of one device (bench.py BENCH_SHARED_GPU=1 and tests).  Windows are
    plain device memory exchanged by pointer; ordering uses the same
    stream-ordered peer-memory barriers as separate processes on separate
    GPUs.  `group(rank)` is the per-thread handle passed as `group=`."""

    def __init__(self, size: int):
        import threading
        self.size = size
        self._barrier = threading.Barrier(size)
        self._slots = [None] * size

    def group(self, rank: int) -> "ThreadRankGroup":
        return ThreadRankGroup(self, rank)


class ThreadRankGroup:
    """One thread's view of a ThreadRanks world (the torch.distributed subset
    the step uses: rank, size, barrier, all_gather_object, all_reduce of a
    host integer)."""

    def __init__(self, world: ThreadRanks, rank: int):
        self.world, self.rank, self.size = world, rank, world.size

    def barrier(self, group=None):
        self.world._barrier.wait()

    def all_gather_object(self, out, obj, group=None):
        self.world._slots[self.rank] = obj
        self.world._barrier.wait()
        out[:] = list(self.world._slots)
        self.world._barrier.wait()

    def all_reduce_int(self, x: int) -> int:
        vals = [None] * self.size
        self.all_gather_object(vals, int(x))
        return sum(vals)


class Comm:
    """all-to-all helpers on a process group (NCCL on GPUs, gloo on CPU), or
    on a ThreadRankGroup (backend "local": ranks are threads of one process)."""

    def __init__(self, group=None):
        if isinstance(group, ThreadRankGroup):
            self.dist, self.group = group, None
            self.size, self.rank, self.backend = group.size, group.rank, "local"
            return
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
    kernel stores straight into the consuming rank's window (NVLink P2P
    stores between GPUs; ranks sharing one GPU in the tests).  Grown
    collectively: every rank takes the same decision from the all-gathered
    count matrix (`ensure` gets every rank's need), then the IPC handles are
    re-exchanged — the only host round trip besides the count matrix, and
    only when a window grows."""

    def __init__(self, comm: "Comm"):
        self.comm = comm
        self.cap, self.local, self.opened, self.peers_dev = {}, {}, {}, {}
        self.grows = 0

    def ensure(self, name: str, units_per_rank, unit_bytes: int) -> None:
        need = max(units_per_rank) if units_per_rank else 0
        if need <= self.cap.get(name, 0) and name in self.local:
            return
        import ctypes as C
        import torch
        cap = max(need + need // 4, int(self.cap.get(name, 0) * 1.5), 1024)
        self.close(name)
        ptr, handle = C.c_void_p(), (C.c_char * 64)()
        N.call("skb_ipc_alloc", cap * unit_bytes, C.byref(ptr), handle)
        local = self.comm.backend == "local"  # ranks share this process: plain pointers
        handles = [None] * self.comm.size
        self.comm.dist.all_gather_object(handles, ptr.value if local else bytes(handle), group=self.comm.group)
        peers = []
        for j, h in enumerate(handles):
            if j == self.comm.rank or local:
                peers.append(ptr.value if j == self.comm.rank else h)
            else:
                q = C.c_void_p()
                N.call("skb_ipc_open", (C.c_char * 64).from_buffer_copy(h), C.byref(q))
                peers.append(q.value)
                self.opened.setdefault(name, []).append(q.value)
        self.local[name], self.cap[name] = ptr.value, cap
        self.peers_dev[name] = torch.tensor(peers, dtype=torch.int64, device="cuda")
        self.grows += 1

    def ptr(self, name: str):
        import ctypes as C
        return C.c_void_p(self.local[name])

    def peers(self, name: str):
        return N.ptr(self.peers_dev[name])

    def close(self, name: str) -> None:
        if name not in self.local:
            return
        import ctypes as C
        import torch
        torch.cuda.synchronize()
        self.comm.dist.barrier(group=self.comm.group)  # nobody touches the old windows any more
        if self.comm.backend == "local":
            self.opened.pop(name, None)
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


class ExchangePlan:
    """Every offset of one step's exchange, from the all-gathered count
    matrix C[q][j] = unique ids rank q requests from owner j (sharding.py's
    per-shard unique lists, rank q's batch).  Pure host arithmetic; every
    rank derives the same windows from the same matrix.

    requester `me`:  uniq list = owner segments send_pre[j]..send_pre[j+1];
                     segment j goes to owner j's id / grad window at
                     to_owner_base[j] (the ranks before me, rank order).
    owner `me`:      received list = requester segments recv_pre[q]..; the
                     row of received position i goes to requester q's row
                     window at to_req_base[q] + i - recv_pre[q] (q's uniq
                     index of that id: q's owners before me come first).
    """

    def __init__(self, cmat, me: int):
        S = len(cmat)
        self.S, self.me, self.cmat = S, me, [list(map(int, r)) for r in cmat]
        c = self.cmat
        self.send = c[me]
        self.U = sum(self.send)
        self.send_pre = _prefix(self.send)
        self.recv = [c[q][me] for q in range(S)]
        self.n_recv = sum(self.recv)
        self.recv_pre = _prefix(self.recv)
        self.to_owner_base = [sum(c[q][j] for q in range(me)) for j in range(S)]
        self.to_req_base = [sum(c[q][:me]) for q in range(S)]
        self.rows_need = [sum(c[q]) for q in range(S)]                       # requester q's row window
        self.recv_need = [sum(c[q][j] for q in range(S)) for j in range(S)]  # owner j's id / grad window

    def meta(self):
        """int64 [4, S+1]: send_pre, to_owner_base, recv_pre, to_req_base."""
        m = np.zeros((4, self.S + 1), np.int64)
        m[0] = self.send_pre
        m[1, :self.S] = self.to_owner_base
        m[2] = self.recv_pre
        m[3, :self.S] = self.to_req_base
        return m


class DistSparseStep:
    """Fused multi-GPU sparse step for one row-sharded logical table
    (reference sharding.py:222-297 driven by train.py:120-195).

    forward : requester prepare (keys, dedup + owner split, sort; csrc/dist.cu)
              -> count matrix (all-gather; the step's ONE host sync) -> ids
              stored into the owners' id windows -> owner: the single-GPU
              fused index phase on the received ids (admission in the
              rank-ordered first-occurrence order = the oracle's slots) and a
              row gather stored straight into each requester's row window ->
              requester pools from its window.
    backward: requester folds dpooled per local unique id (np.add.at order)
              and stores the sums into the owners' grad windows -> owner:
              the single-GPU fused fold+Adam (TMA ring / register kernels,
              long-run fold) over the window, ranks' partial sums folded in
              rank order.

    Ordering between ranks is stream-ordered: a one-element NCCL all-reduce
    after each round of peer stores (gloo: device sync + host barrier).
    Results: slots and first-step rows exact vs the oracle fed the
    rank-ordered concatenation; updates within tolerance (cross-rank partial
    sums re-associate the fold).
    """

    def __init__(self, lt, comm: Comm | None = None):
        if not lt.dist:
            raise ValueError("DistSparseStep needs a LogicalTable built with dist=True")
        import ctypes as C
        import torch
        self.lt = lt
        self.comm = comm or Comm(lt.group)
        self.S, self.me, self.D = self.comm.size, self.comm.rank, lt.dim
        # two requester contexts (dedup / split / sort buffers), used by
        # alternate steps, so step k+1's prepare can run (prefetch) while
        # step k's backward still reads step k's
        self.hs = []
        for _ in range(2):
            h = C.c_void_p()
            N.call("skb_dist_create", self.D, self.S, C.byref(h))
            self.hs.append(h)
        self.h = self.hs[0]
        self._next = 0  # context of the next prepare
        self._free = [None, None]  # event after the backward that last read each context
        self._pre = None  # prefetched (batch, step, context, plan)
        self._side = None  # stream of prefetched prepares
        self.win = P2PWindows(self.comm)
        self.counts_h = [torch.zeros(self.S, dtype=torch.int64, device="cuda") for _ in range(2)]
        self.counts = self.counts_h[0]
        # stream-ordered peer-memory barriers when the driver has stream memory
        # operations (every B200 driver): then the step needs no collective at
        # all — counts all-gathered by P2P stores, one readback of the matrix
        ok = C.c_int32()
        N.call("skb_p2p_memops_supported", C.byref(ok))
        self.p2p_sync = bool(ok.value) and os.environ.get("SKB_DIST_BARRIER", "p2p") == "p2p"
        self.epoch = 0
        self.epoch2 = 0  # barrier channel of prefetched count exchanges (own flag words)
        if self.p2p_sync:
            S = self.S
            self.win.ensure("flags", [S] * S, 8)
            self.win.ensure("flags2", [S] * S, 8)
            self.win.ensure("cmat", [S * S] * S, 8)
            self._flag_ptrs = (C.c_int64 * S)(*self.win.peers_dev["flags"].cpu().tolist())
            self._flag_ptrs2 = (C.c_int64 * S)(*self.win.peers_dev["flags2"].cpu().tolist())
        self.cmat_host = torch.zeros(self.S * self.S, dtype=torch.int64).pin_memory()
        self.cmat_dev = torch.zeros(self.S * self.S, dtype=torch.int64, device="cuda")
        self.syncs = 0  # host synchronisations of the step path (the count matrix readback)
        self.plan = None
        self._meta = None
        self._mode = None
        self.last_counts = None

    def __del__(self):
        try:
            for h in getattr(self, "hs", []):
                N.lib().skb_dist_destroy(h)
            self.hs = []
        except Exception:
            pass

    def _barrier(self, channel: int = 1):
        """Order every rank's prior peer stores before any rank's later reads
        (channel 2: the prefetched count exchange, own flag words and epoch,
        so it can run on a side stream while channel-1 barriers are pending)."""
        if self.comm.backend == "local":
            # ranks are threads of one process: every stream waits on events the
            # others have ALREADY recorded — a wait on a not-yet-enqueued peer
            # write (the memop barrier) could deadlock against any implicit
            # device-wide synchronisation (cudaMalloc) of another rank's thread
            import torch
            ev = torch.cuda.Event()
            ev.record()
            evs = [None] * self.S
            self.comm.dist.all_gather_object(evs, ev)
            cur = torch.cuda.current_stream()
            for j, e in enumerate(evs):
                if j != self.me:
                    cur.wait_event(e)
        elif self.p2p_sync:
            if channel == 2:
                self.epoch2 += 1
                N.call("skb_p2p_barrier", self._flag_ptrs2, self.S, self.me, self.epoch2, N.stream_ptr())
            else:
                self.epoch += 1
                N.call("skb_p2p_barrier", self._flag_ptrs, self.S, self.me, self.epoch, N.stream_ptr())
        else:
            self.comm.barrier_after_device_writes()

    def _count_matrix(self, channel: int = 1, defer: bool = False, counts=None):
        """C[q][j] for all ranks: every rank stores its counts into row `rank`
        of each peer's count window, barrier, one readback (the step's host
        synchronisation).  Without stream memory operations: an all-gather.
        defer (peer-memory path): enqueue the readback and return an event;
        `_matrix()` reads it once the event has completed."""
        self.syncs += 1
        counts = self.counts if counts is None else counts
        if self.p2p_sync:
            import torch
            sp = N.stream_ptr()
            N.call("skb_p2p_put_counts", N.ptr(counts), self.S, self.me, self.win.peers("cmat"), sp)
            self._barrier(channel)
            N.call("skb_memcpy_async", self.cmat_host.data_ptr(), self.win.ptr("cmat"), 8 * self.S * self.S, sp)
            if defer:
                ev = torch.cuda.Event()
                ev.record()
                return ev
            torch.cuda.current_stream().synchronize()
            return self._matrix()
        if self.comm.backend == "nccl":
            self.comm.dist.all_gather_into_tensor(self.cmat_dev, counts, group=self.comm.group)
            flat = self.cmat_dev.cpu().tolist()
        else:
            import torch
            out = [torch.empty(self.S, dtype=torch.int64) for _ in range(self.S)]
            self.comm.dist.all_gather(out, counts.cpu(), group=self.comm.group)
            flat = [int(x) for t in out for x in t.tolist()]
        return [flat[q * self.S:(q + 1) * self.S] for q in range(self.S)]

    def _matrix(self):
        flat = self.cmat_host.tolist()
        return [flat[q * self.S:(q + 1) * self.S] for q in range(self.S)]

    def _prepare(self, batch, channel: int, defer: bool = False):
        """Requester prepare of `batch` into the next context + the count
        exchange (the step's one host synchronisation) on the current stream;
        returns (context index, count matrix, or the readback's event when
        deferred)."""
        import ctypes as C
        F = len(batch.members)
        if batch._c_args is None:
            batch._c_args = ((C.c_int64 * (F + 1))(*batch.member_pos.tolist()),
                             (C.c_uint64 * max(F, 1))(*[int(x) for x in batch.salts]),
                             (C.c_int64 * (F + 1))(*batch.member_bag.tolist()),
                             (C.c_int32 * max(F, 1))(*batch.strategy.tolist()))
        mp, sl, mb, st = batch._c_args
        ci = self._next
        self._next ^= 1
        counts = self.counts_h[ci]
        N.call("skb_dist_prepare", self.hs[ci], N.ptr(batch.ids), batch.num_ids, mp, sl, F,
               1 if batch.namespaced else 0, N.ptr(batch.bag_offs), batch.num_bags, mb, st, N.ptr(counts),
               N.stream_ptr())
        return ci, self._count_matrix(channel, defer, counts)

    def prefetch(self, batch, step: int) -> None:
        """Prepare step `step`'s batch now (cross-step pipeline, like the
        single-GPU `prefetch`): issue it between forward(k) and backward(k) for
        step k+1.  The dedup / split / sort and the count exchange are only
        enqueued (on a side stream, after the work already queued on the
        caller's stream — forward(k) — and after the backward that last used
        the context); the host reads the count matrix in forward(k+1), by when
        backward(k) keeps the GPU busy.  Every rank must call it at the same
        point of its step sequence."""
        import torch
        if self._pre is not None:
            raise ValueError("a prefetched batch is already pending")
        if self._side is None:
            lo, hi = torch.cuda.Stream.priority_range()
            self._side = torch.cuda.Stream(priority=hi)
        cur = torch.cuda.current_stream()
        side = self._side
        side.wait_stream(cur)  # the batch's ids / offsets are ready
        ev = self._free[self._next]
        if ev is not None:
            side.wait_event(ev)  # the backward that last read this context
        with torch.cuda.stream(side):
            ci, cm = self._prepare(batch, 2, defer=True)
            done = torch.cuda.Event()
            done.record(side)
        self._pre = (batch, int(step), ci, cm, done)

    def forward(self, batch, step: int, mode: str = "mean", out=None):
        from .fused import _MODES
        import torch
        if mode not in ("sum", "mean"):
            raise ValueError(f"unknown mode {mode!r} (the multi-GPU step pools with sum or mean)")
        lt, S, D = self.lt, self.S, self.D
        if self._pre is not None:
            pb, pstep, ci, cm, done = self._pre
            if pb is not batch or pstep != int(step):
                raise ValueError("forward of a different batch / step than the pending prefetch")
            self._pre = None
            if isinstance(cm, torch.cuda.Event):
                cm.synchronize()  # the step's one host synchronisation
                cm = self._matrix()
            torch.cuda.current_stream().wait_event(done)
        else:
            ev = self._free[self._next]
            if ev is not None:
                torch.cuda.current_stream().wait_event(ev)
            ci, cm = self._prepare(batch, 1)
        plan = ExchangePlan(cm, self.me)
        self._ci = ci  # the context this step's pool and backward read
        self.h, self.counts = self.hs[ci], self.counts_h[ci]
        sp = N.stream_ptr()
        self.win.ensure("ids", plan.recv_need, 8)
        self.win.ensure("grads", plan.recv_need, 4 * D)
        self.win.ensure("rows", plan.rows_need, 4 * D)
        meta = N.to_dev(plan.meta(), "int64")
        N.call("skb_dist_send_ids", self.h, plan.U, N.ptr(meta[0]), self.win.peers("ids"), N.ptr(meta[1]), sp)
        self._barrier()
        N.call("skb_fused_forward_send", lt.local_table.handle, self.win.ptr("ids"), plan.n_recv, int(step),
               N.ptr(meta[2]), S, self.win.peers("rows"), N.ptr(meta[3]), sp)
        self._barrier()
        G = batch.num_bags
        pooled = out if out is not None else N.empty((G, D), "float32")
        N.call("skb_dist_pool", self.h, self.win.ptr("rows"), _MODES[mode], N.ptr(pooled), sp)
        self.plan, self._meta, self._mode = plan, meta, _MODES[mode]
        self.last_counts = {"send": list(plan.send), "recv": list(plan.recv), "n_recv": plan.n_recv}
        return pooled

    def backward(self, dpooled, cfg, step: int):
        from .optim import adam_scalars
        import ctypes as C
        if self.plan is None:
            raise ValueError("backward without a preceding forward")
        if step < 1:
            raise ValueError("global step t must be >= 1")
        plan, meta = self.plan, self._meta
        g = N.to_dev(dpooled, "float32")
        sp = N.stream_ptr()
        N.call("skb_dist_fold_send", self.hs[self._ci], N.ptr(g), self._mode, plan.U, N.ptr(meta[0]),
               self.win.peers("grads"), N.ptr(meta[1]), sp)
        import torch
        ev = torch.cuda.Event()
        ev.record()
        self._free[self._ci] = ev  # this context may be prepared again after here
        self._barrier()
        sc = adam_scalars(cfg, step)
        N.call("skb_fused_backward", self.lt.local_table.handle, self.win.ptr("grads"), C.byref(sc), sp)
        self.plan = None

    def owner_unique(self) -> int:
        """Rows this rank's shard touched in the last step (synchronizes)."""
        from .fused import last_step_stats
        return last_step_stats(self.lt)[0]
