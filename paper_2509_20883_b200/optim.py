"""Sparse Adam / AdamW over the device-resident row arena (reference optim.py:1-83).

Lazy semantics and global-step bias correction as in the reference; the
float32 scalars are formed on the host exactly as optim.py:69-75 does and
every device op is separately rounded (no FMA), so updates are bit-identical
to the numpy float32 reference given identical gradients.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from . import telemetry


@dataclass(frozen=True)
class AdamConfig:
    lr: float = 0.001
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.0
    variant: str = "adam"

    def __post_init__(self):
        if not (0.0 <= self.beta1 < 1.0 and 0.0 <= self.beta2 < 1.0):
            raise ValueError("betas must be in [0, 1)")
        if self.eps <= 0.0:
            raise ValueError("eps must be > 0")
        if self.weight_decay < 0.0:
            raise ValueError("weight_decay must be >= 0")
        if self.variant not in ("adam", "adamw"):
            raise ValueError(f"unknown variant {self.variant!r}")

    @classmethod
    def from_dict(cls, d: dict) -> "AdamConfig":
        return cls(**d)


_SCALARS = {}


def adam_scalars(cfg: AdamConfig, t: int) -> N.AdamScalars:
    """float32 scalars of optim.py:69-75 (bias corrections via Python double pow).

    The step-independent ones are computed once per configuration with numpy
    float32 arithmetic; per call only bc1 / bc2 = float32(1 - beta**t) are
    set — the double result rounded to float32 by the c_float field, the same
    single rounding as np.float32(...) (the launch-bound C1 step calls this
    every step; a dozen numpy scalar ops cost ~15 us)."""
    key = (cfg.lr, cfg.beta1, cfg.beta2, cfg.eps, cfg.weight_decay, cfg.variant)
    base = _SCALARS.get(key)
    if base is None:
        f = np.float32
        lr, b1, b2 = f(cfg.lr), f(cfg.beta1), f(cfg.beta2)
        base = N.AdamScalars(
            lr=lr, beta1=b1, beta2=b2, eps=f(cfg.eps),
            one_minus_beta1=f(f(1.0) - b1), one_minus_beta2=f(f(1.0) - b2), bc1=0.0, bc2=0.0,
            lr_wd=f(lr * f(cfg.weight_decay)),
            decoupled_decay=1 if (cfg.variant == "adamw" and cfg.weight_decay != 0.0) else 0)
        if len(_SCALARS) < 64:
            _SCALARS[key] = base
    sc = N.AdamScalars.from_buffer_copy(base)
    sc.bc1 = 1.0 - cfg.beta1 ** t
    sc.bc2 = 1.0 - cfg.beta2 ** t
    return sc


def sparse_adam_step(store, offsets, grads, cfg: AdamConfig, t: int) -> None:
    """One bias-corrected Adam/AdamW update of the rows at distinct offsets (optim.py:42-83)."""
    telemetry.bump("optim.sparse_adam_step")
    if t < 1:
        raise ValueError("global step t must be >= 1")
    o = N.to_dev(offsets, "int64").reshape(-1)
    gshape = tuple(grads.shape) if hasattr(grads, "shape") else np.asarray(grads).shape
    if gshape != (o.numel(), store.dim):
        raise ValueError(f"grads shape {gshape} != ({o.numel()}, {store.dim})")
    if o.numel() == 0:
        return
    g = N.to_dev(grads, "float32")
    sc = adam_scalars(cfg, t)
    N.call("skb_sparse_adam_step", store._h.h, N.ptr(o), o.numel(), N.ptr(g), N.ctypes_byref(sc), N.stream_ptr())
