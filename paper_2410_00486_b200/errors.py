"""When the drop-in API reports the reference's data-dependent errors.

The reference raises from the call that detects a problem
(``ValueError`` for a non-finite parameter, api.py:127-129;
``FloatingPointError`` for a non-finite gradient, api.py:74-79 and
optimizer.py:111-113; ``ValueError`` for a zero-norm quaternion,
core.py:225-229).  On the GPU every such check is a device reduction, and
raising from the detecting call costs one host read (a stream sync) per
check: five per ``train_one``-shaped iteration (rasterize_forward's status,
the loss scalars, validate_finite, adam_step's finite check and its
zero-quaternion word).

``set_error_mode("eager")`` (default) keeps the reference's behaviour.
``set_error_mode("deferred")`` keeps the checks on the device and raises
their errors, in call order, at the next host read the API needs anyway
(the pair count rasterize_forward reads to size its buffers) or at an
explicit :func:`check_errors`; ``LossBreakdown`` scalars are read when
first used.  An iteration then synchronises once for the binning and once
where the caller reads its loss.  In deferred mode a non-finite gradient
still never reaches the map: the Adam kernel leaves every Gaussian whose
gradient is non-finite untouched (parameters and moments), but -- unlike the
reference, which raises before any update -- the other Gaussians of that
step are updated.
"""

from __future__ import annotations

import torch

_MODE = "eager"
_PENDING: list = []  # (device tensor, raiser(host values) -> None)


def set_error_mode(mode: str) -> None:
    global _MODE
    if mode not in ("eager", "deferred"):
        raise ValueError("error mode must be 'eager' or 'deferred'")
    if mode == "eager":
        check_errors()
    _MODE = mode


def error_mode() -> str:
    return _MODE


def deferred() -> bool:
    return _MODE == "deferred"


def defer(flags: torch.Tensor, raiser) -> None:
    """Register a device check; raiser(host copy of flags) raises if it failed."""
    _PENDING.append((flags, raiser))


def take_pending():
    """The registered checks, cleared (for a caller that reads them together
    with its own device words)."""
    out = list(_PENDING)
    _PENDING.clear()
    return out


def raise_pending(pending, host_values) -> None:
    for (_, raiser), h in zip(pending, host_values):
        raiser(h)


def read_with_pending(own: torch.Tensor | None):
    """One host read of `own` (an int64 device tensor, may be None) plus every
    pending check; raises the pending errors in call order, then returns the
    host copy of `own`."""
    pending = take_pending()
    parts = [p[0].reshape(-1).to(torch.int64) for p in pending]
    if own is not None:
        parts.append(own.reshape(-1).to(torch.int64))
    if not parts:
        return None
    host = torch.cat(parts).cpu() if len(parts) > 1 else parts[0].cpu()
    off = 0
    vals = []
    for p in pending:
        k = p[0].numel()
        vals.append(host[off:off + k])
        off += k
    raise_pending(pending, vals)
    return host[off:] if own is not None else None


def check_errors() -> None:
    """Raise any error the deferred checks recorded (one host read)."""
    if _PENDING:
        read_with_pending(None)
