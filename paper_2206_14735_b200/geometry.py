"""Geometric initialisation (sphere pre-fit, gs/decoders.py:102-177).

SURVEY.md 8f #1: not yet on the device; build_model(skip_init=True) is the
supported path in this round."""

from __future__ import annotations


class InitError(RuntimeError):
    """Geometric initialization failed to reach tolerance in budget."""


def geometric_init(model, center, radius, seed=0, max_steps=2000, tol=0.01, batch=4096,
                   lr_grid=1e-2, lr_net=1e-3):
    raise NotImplementedError("geometric_init is not implemented on the B200 path yet; "
                              "use build_model(..., skip_init=True)")
