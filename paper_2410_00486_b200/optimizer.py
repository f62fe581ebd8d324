"""Adam with per-attribute learning rates on B200 (drop-in for
``splatstream.optimizer``, optimizer.py:19-146).

Moments are float32 device planes keyed like the reference
(position, rotation, log_scale, opacity_logit, sh_dc, sh_rest); the update
runs in one fused kernel (K9) that also renormalises the quaternions.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import check, lib, traced
from .core import GaussianMap
from . import errors
from .rasterizer import P, ParamGrads, finite_flags, finite_flags_device, stream_handle

PARAM_SHAPES = {
    "position": (3,),
    "rotation": (4,),
    "log_scale": (3,),
    "opacity_logit": (),
    "sh_dc": (1, 3),
    "sh_rest": (15, 3),
}
_FLAT = {"position": 3, "rotation": 4, "log_scale": 3, "opacity_logit": 1, "sh_dc": 3,
         "sh_rest": 45}


@dataclass
class LearningRates:
    """optimizer.py:29-37."""

    position: float = 1.6e-4
    position_final: float = 1.6e-6
    sh_dc: float = 2.5e-3
    sh_rest: float = 1.25e-4
    opacity_logit: float = 5e-2
    log_scale: float = 5e-3
    rotation: float = 1e-3


@dataclass
class AdamState:
    """optimizer.py:40-76 with float32 device moments."""

    lrs: LearningRates = field(default_factory=LearningRates)
    horizon: int = 30000
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-15
    step_count: int = 0
    m: dict = field(default_factory=dict)
    v: dict = field(default_factory=dict)
    sh_rest_active: bool = False  # set once sh_rest ever receives a gradient

    @classmethod
    def for_map(cls, gmap: GaussianMap, lrs: LearningRates | None = None,
                horizon: int = 30000) -> "AdamState":
        st = cls(lrs=lrs or LearningRates(), horizon=horizon)
        n = len(gmap)
        for name, k in _FLAT.items():
            shape = (n,) if k == 1 else (n, k)
            st.m[name] = torch.zeros(shape, dtype=torch.float32, device=gmap.device)
            st.v[name] = torch.zeros(shape, dtype=torch.float32, device=gmap.device)
        return st

    def position_lr(self) -> float:
        """optimizer.py:63-67."""
        t = min(self.step_count / max(self.horizon, 1), 1.0)
        lr0, lr1 = self.lrs.position, self.lrs.position_final
        return float(lr0 * (lr1 / lr0) ** t)

    def rate_for(self, name: str) -> float:
        if name == "position":
            return self.position_lr()
        return getattr(self.lrs, name)

    def hparams(self, update_sh_rest: bool) -> _lib.SSAdamHP:
        """Resolved for the current (post-increment) step count."""
        h = _lib.SSAdamHP()
        h.lr_position = self.position_lr()
        h.lr_rotation = self.lrs.rotation
        h.lr_log_scale = self.lrs.log_scale
        h.lr_opacity = self.lrs.opacity_logit
        h.lr_sh_dc = self.lrs.sh_dc
        h.lr_sh_rest = self.lrs.sh_rest
        h.beta1, h.beta2, h.eps = self.beta1, self.beta2, self.eps
        t = self.step_count
        h.bias1 = 1.0 - self.beta1 ** t
        h.bias2 = 1.0 - self.beta2 ** t
        h.update_sh_rest = 1 if update_sh_rest else 0
        return h

    def planes(self, which: str) -> _lib.SSParamGrads:
        d = self.m if which == "m" else self.v
        g = _lib.SSParamGrads()
        g.d_position, g.d_rotation = P(d["position"]), P(d["rotation"])
        g.d_log_scale, g.d_opacity = P(d["log_scale"]), P(d["opacity_logit"])
        g.d_sh_dc, g.d_sh_rest = P(d["sh_dc"]), P(d["sh_rest"])
        g.d_pos2d_norm = None
        return g


@traced("ss.adam_step")
def adam_step(gmap: GaussianMap, grads: ParamGrads, state: AdamState, sh_degree: int | None = None):
    """optimizer.py:101-133.  Returns (gmap, state)."""
    if len(grads) != len(gmap):
        raise ValueError(
            f"gradient length {len(grads)} does not match map length {len(gmap)}")
    named = (("position", grads.position), ("rotation", grads.rotation),
             ("log_scale", grads.log_scale), ("opacity_logit", grads.opacity_logit),
             ("sh_dc", grads.sh_dc), ("sh_rest", grads.sh_rest))

    def raise_nonfinite(bad):
        for (name, _), b in zip(named, [int(v) for v in bad[:len(named)]]):
            if b:
                raise FloatingPointError(f"non-finite gradient for parameter '{name}'")
    deferred = errors.deferred()
    if deferred:
        # the check stays on the device (errors.py); the Adam kernel leaves
        # Gaussians with non-finite gradients untouched.  sh_rest is updated
        # unless the gradients are known to come from an SH-0 render (then they
        # are exactly 0 and so are the moments: the skip is bit-exact)
        errors.defer(finite_flags_device([t for _, t in named])[:len(named)], raise_nonfinite)
        upd_rest = state.sh_rest_active or grads.sh_degree is None or grads.sh_degree > 0
    else:
        # the finite checks and the "sh_rest in use" test: one kernel, one host
        # read -- for the tensors backward_splatwise's eager check has not
        # already passed unmodified (ParamGrads.known_finite)
        known = [grads.known_finite(k, t) if hasattr(grads, "known_finite") else (False, None)
                 for k, t in named]
        todo = [i for i, (ok, _) in enumerate(known) if not ok]
        bad = [0] * len(named)
        nonzero = [nz for _, nz in known]
        if todo:
            host = finite_flags([named[i][1] for i in todo], extra_nonzero=True)
            for j, i in enumerate(todo):
                bad[i] = 0 if host[j] else 1
                nonzero[i] = host[len(todo) + j]
        raise_nonfinite(bad)
        upd_rest = state.sh_rest_active or bool(nonzero[len(named) - 1])
    state.sh_rest_active = upd_rest
    state.step_count += 1
    st = torch.empty(_lib.STATUS_WORDS, dtype=torch.int64, device=gmap.device)
    s = stream_handle()
    check(lib().ss_status_reset(P(st), s), "ss_status_reset")
    mp, gr = gmap.ss(), grads.ss()
    hp = state.hparams(upd_rest)
    check(lib().ss_adam_step(ctypes.byref(mp), ctypes.byref(gr), ctypes.byref(state.planes("m")),
                             ctypes.byref(state.planes("v")), ctypes.byref(hp), P(st), s),
          "ss_adam_step")
    def raise_zero_quat(h):
        if int(h[0]) != _lib.INT64_MAX:
            raise ValueError("zero-norm quaternion in map")
    if deferred:
        errors.defer(st[_lib.ST_ZERO_QUAT:_lib.ST_ZERO_QUAT + 1], raise_zero_quat)
    else:
        raise_zero_quat(st[_lib.ST_ZERO_QUAT:_lib.ST_ZERO_QUAT + 1].cpu())
    return gmap, state


@traced("ss.resize_for_densify")
def resize_for_densify(state: AdamState, survivors, n_new: int) -> AdamState:
    """optimizer.py:136-146: moments of the survivors gathered in order, zero
    rows appended for the n_new fresh primitives (one ss_resize_moments
    launch for every m / v plane)."""
    dev = next(iter(state.m.values())).device
    surv = torch.as_tensor(survivors, dtype=torch.int64).to(dev).reshape(-1)
    n_old = next(iter(state.m.values())).shape[0]
    if surv.numel() and (int(surv.min()) < 0 or int(surv.max()) >= n_old):
        raise ValueError("survivor index out of range")
    n_out = int(surv.numel()) + int(n_new)
    pin, pout, pk, names = [], [], [], []
    for d in (state.m, state.v):
        for name, t in d.items():
            out = torch.empty((n_out,) + tuple(t.shape[1:]), dtype=t.dtype, device=dev)
            k = int(t[0].numel()) if t.shape[0] else int(np.prod(t.shape[1:], dtype=np.int64))
            pin.append(t.contiguous())
            pout.append(out)
            pk.append(max(k, 1))
            names.append((d, name))
    n_pl = len(pin)
    arr_in = (ctypes.c_void_p * n_pl)(*[p.data_ptr() for p in pin])
    arr_out = (ctypes.c_void_p * n_pl)(*[p.data_ptr() for p in pout])
    arr_k = (ctypes.c_int32 * n_pl)(*pk)
    check(lib().ss_resize_moments(n_out, P(surv), int(surv.numel()), n_pl, arr_in, arr_out,
                                  arr_k, stream_handle()), "ss_resize_moments")
    for (d, name), out in zip(names, pout):
        d[name] = out
    return state
