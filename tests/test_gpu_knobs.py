"""Kernel paths selected by environment knobs read once per process
(DESIGN §11), each run in its own subprocess and checked bit-exactly against
the oracle with the same driver as test_gpu_parity._fused_vs_oracle:

- SKB_LF_PACK=0: mega runs folded by column-group units whose producers
  gather the group's columns straight from the gradient rows (no pack pass);
- SKB_LF_EXCLUSIVE=2 / SKB_LF_CARVEOUT=100: the long fold claiming whole
  SMs, or the maximum shared-memory carveout, on every launch;
- SKB_POOL_VARIANT=5: the register pool shape that is not the default any more;
- SKB_LF_STREAM_PACK=1 (+ SKB_LF_MIX_TEST=1): the pack on its own stream
  beside the long fold, whose producers stream the images already flagged
  ready and gather the others — with the mix test every odd stage of a run
  is gathered, so TMA-image and gathered stages alternate in one chain.
"""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, {root!r})
sys.path.insert(0, {tests!r})
import paper_2509_20883_b200 as skb
import test_gpu_parity as T

hot = lambda r, B: r.integers(1, 9, B)
# zipf(1.2) ids over ~60K positions: the head id holds >8192 positions (a
# mega run for sum bags), several more >2048 (mega for mean bags)
for D, mode in ((64, "sum"), (64, "mean"), (16, "mean"), (8, "sum")):
    T._fused_vs_oracle(skb, D, [("zh", 12000, hot), ("a", 500, lambda r, B: r.integers(0, 4, B))], steps=3,
                       mode=mode, seed=7 + D)
T._fused_vs_oracle(skb, 64, [("zt", 60, lambda r, B: r.integers(500, 900, B))], steps=2, mode="tile", k=700, seed=3)
print("ok")
"""


@pytest.mark.gpu
@pytest.mark.parametrize("env", [{"SKB_LF_PACK": "0"}, {"SKB_LF_EXCLUSIVE": "2"}, {"SKB_LF_CARVEOUT": "100"},
                                 {"SKB_POOL_VARIANT": "5"},
                                 {"SKB_LF_STREAM_PACK": "1", "SKB_LF_MIX_TEST": "1"},
                                 {"SKB_LF_STREAM_PACK": "1", "SKB_LF_EXCLUSIVE": "2"}])
def test_knob_paths_vs_oracle(cuda, env):
    e = dict(os.environ)
    e.update(env)
    code = _SCRIPT.format(root=ROOT, tests=os.path.join(ROOT, "tests"))
    r = subprocess.run([sys.executable, "-c", code], env=e, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), (env, r.stdout[-2000:], r.stderr[-4000:])
