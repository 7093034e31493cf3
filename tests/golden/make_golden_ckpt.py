"""Golden checkpoint fixtures from the REFERENCE itself (build container only).

Usage:  python tests/golden/make_golden_ckpt.py
Replays a seeded op trace (lookups, grad updates, evictions) on two tables
through the reference's public API (`sparsekit_ref`, read-only alias of
/root/reference/pkg/src/sparsekit), saves them with the reference's
`save_sharded` (checkpoint.py:192-252) and commits:
  tests/golden/ckpt/           the reference's checkpoint directory (bytes)
  tests/golden/ckpt_trace.npz  the op trace, to replay through this repo
  tests/golden/ckpt_resaved/   load_sharded(ckpt, 2) saved again to 2 files
  tests/golden/ckpt_inspect.txt  inspect_checkpoint(ckpt)
Nothing on the GPU box reads /root/reference.
"""

from __future__ import annotations

import os
import shutil
import sys

import numpy as np

sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import load_ref  # noqa: E402

OUT_DIR = os.path.join(HERE, "ckpt")
TRACE = os.path.join(HERE, "ckpt_trace.npz")
RESAVED = os.path.join(HERE, "ckpt_resaved")
INSPECT = os.path.join(HERE, "ckpt_inspect.txt")

# the trace: logical table "dim8" (members u, i; namespaced; 4 shards) and a
# plain EmbeddingTable "plain4"; 6 steps, eviction at step 4 (threshold 2)
STEPS, EVICT_AT, NUM_FILES, GLOBAL_STEP = 6, 4, 3, 6
CFG = dict(lr=1e-2, weight_decay=0.01, variant="adamw")


def make_trace():
    rng = np.random.Generator(np.random.PCG64(77))
    t = {}
    for step in range(1, STEPS + 1):
        t[f"{step}.u"] = rng.zipf(1.3, 40).astype(np.int64)
        t[f"{step}.i"] = rng.integers(-(2**40), 2**40, 25, dtype=np.int64)
        t[f"{step}.dim8.grads"] = (rng.standard_normal((65, 8)) * 0.05).astype(np.float32)
        t[f"{step}.plain4.ids"] = np.unique(rng.integers(0, 90, 30, dtype=np.int64))
        t[f"{step}.plain4.grads"] = (rng.standard_normal((len(t[f"{step}.plain4.ids"]), 4)) * 0.05).astype(np.float32)
    return t


def main():
    ref = load_ref()
    from sparsekit_ref import checkpoint as CK, optim as OP, sharding as SH
    trace = make_trace()
    cfg = OP.AdamConfig(**CFG)
    lt = SH.LogicalTable("dim8", 8, 4, seed=5, members=["u", "i"], namespaced=True, evict_threshold=2)
    plain = ref.EmbeddingTable("plain4", 4, seed=9, block_size=16, evict_threshold=2)
    plan = SH.ShardPlan(4)
    for step in range(1, STEPS + 1):
        keys = np.concatenate([lt.keys_for("u", trace[f"{step}.u"]), lt.keys_for("i", trace[f"{step}.i"])])
        SH.all_to_all_lookup(lt, keys, plan, step)
        SH.all_to_all_grad_update(lt, keys, trace[f"{step}.dim8.grads"], plan, cfg, step)
        ids = trace[f"{step}.plain4.ids"]
        offs = plain.lookup_or_insert(ids, step)
        OP.sparse_adam_step(plain.store, offs, trace[f"{step}.plain4.grads"], cfg, step)
        if step == EVICT_AT:
            lt.evict(step)
            plain.evict(step)
    if os.path.exists(OUT_DIR):
        shutil.rmtree(OUT_DIR)
    CK.save_sharded([lt, plain], OUT_DIR, NUM_FILES, global_step=GLOBAL_STEP)
    # the reference's own round trip: reload under 2 shards, save to 2 files
    if os.path.exists(RESAVED):
        shutil.rmtree(RESAVED)
    CK.save_sharded(CK.load_sharded(OUT_DIR, 2), RESAVED, 2, global_step=GLOBAL_STEP + 1)
    with open(INSPECT, "w") as f:
        f.write(CK.inspect_checkpoint(OUT_DIR))
    np.savez_compressed(TRACE, **trace)
    print("wrote", OUT_DIR, sorted(os.listdir(OUT_DIR)), RESAVED, INSPECT, TRACE)


if __name__ == "__main__":
    main()
