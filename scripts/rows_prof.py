#!/usr/bin/env python
"""Run the slower §8(a) row ops of `ops_bench.py --rows` twice each, with an
NVTX-free marker (a 1-element torch fill) between ops, so an ncu launch list
shows each op's kernels and their share of the op's time.

  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/rows_launches.csv python scripts/rows_prof.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_2509_20883_b200 as skb
    torch.cuda.set_device(0)
    rng = np.random.Generator(np.random.PCG64(0))
    n = 1_000_000
    ids1 = torch.from_numpy(rng.integers(-(1 << 62), 1 << 62, n, dtype=np.int64)).cuda()
    plan8 = skb.ShardPlan(8)
    t2 = skb.EmbeddingTable("a5", 16, seed=0, capacity_hint=2 * n)
    uniq = torch.arange(n, dtype=torch.int64, device="cuda") * 7919
    t2.lookup_or_insert(uniq, 1)
    offs_u = t2.lookup_or_insert(uniq, 2)
    seq_o = torch.arange(0, n + 1, 250, dtype=torch.int64, device="cuda")
    RT = skb.RaggedTensor(ids1, seq_o)
    marker = torch.zeros(1, device="cuda")
    from paper_2509_20883_b200 import _native as N
    pos = torch.from_numpy(rng.integers(0, n // 4, n, dtype=np.int64)).cuda()
    pr = skb.unique_partition(pos, skb.ShardPlan(4))
    grads = torch.randn((n, 16), device="cuda")
    inv = (pr.inverse_pos + torch.tensor(pr._bases(), device="cuda")[pr.inverse_shard]).contiguous()
    fout = torch.empty((pr.num_unique, 16), device="cuda")
    t3 = skb.EmbeddingTable("a14", 16, seed=0, evict_threshold=1, capacity_hint=2 * n)

    def evict_cycle():
        t3.lookup_or_insert(uniq, 10)
        t3.evict(20)

    ops = [("a4", lambda: skb.initial_rows(3, ids1, 16)),
           ("a5", lambda: t2.lookup_or_insert(uniq, 2)),
           ("a19", lambda: skb.load_stats(ids1, plan8)),
           ("a20", lambda: RT.truncate(100, "tail")),
           ("a12", lambda: N.call("skb_grad_fold", N.ptr(grads), n, 16, N.ptr(inv), pr.num_unique, N.ptr(fout),
                                  N.stream_ptr())),
           ("a14", evict_cycle)]
    for _, fn in ops:
        fn()
    torch.cuda.synchronize()
    for name, fn in ops:
        for _ in range(2):
            marker.fill_(float(len(name)))
            fn()
    torch.cuda.synchronize()
    del offs_u


if __name__ == "__main__":
    main()
