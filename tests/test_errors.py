"""Deferred error mode bookkeeping (errors.py) on host tensors (no GPU)."""

import pytest
import torch

from paper_2410_00486_b200 import errors


def test_deferred_checks_raise_in_call_order_at_the_next_read():
    errors.set_error_mode("deferred")
    try:
        seen = []

        def first(h):
            seen.append(("first", h.tolist()))
            if not all(h.tolist()):
                raise FloatingPointError("first")

        def second(h):
            seen.append(("second", h.tolist()))
            raise ValueError("second")

        errors.defer(torch.tensor([True, False]), first)
        errors.defer(torch.tensor([7]), second)
        with pytest.raises(FloatingPointError, match="first"):
            errors.read_with_pending(torch.tensor([1, 2, 3]))
        assert seen == [("first", [1, 0])]
        assert errors.take_pending() == []  # consumed
        errors.defer(torch.tensor([1, 1]), first)
        own = errors.read_with_pending(torch.tensor([4, 5]))
        assert own.tolist() == [4, 5]
        errors.check_errors()  # nothing pending
    finally:
        errors.take_pending()
        errors.set_error_mode("eager")
    assert errors.error_mode() == "eager"
    with pytest.raises(ValueError):
        errors.set_error_mode("lazy")
