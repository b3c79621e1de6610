"""Ray-sharded data parallelism.

One process per GPU.  Every rank draws the same global batch from the host
RNG (gs/optimizer.py:363-366) and keeps a contiguous block of rows; its
device PCG streams start at the block's global row (``ray_base``), so the
shards together are exactly the 1-GPU batch.  The step has two exchange
points:

1. after sampling (phase 1): all-reduce of the partition counts, because the
   depth and eikonal normalisers (n_valid, n_eik; gs/renderer.py:372-414)
   are global and n_eik depends on the sampled depths;
2. after the backward (phase 2): all-reduce of the gradient arena (and of the
   additive loss parts), then every rank runs the same Adam.

Rank 0 owns the smoothness points; every loss keeps its global normaliser
(``m_global``, ``smooth_global``)."""

from __future__ import annotations

import dataclasses

from . import _lib

S_SLOT = _lib.PART_NAMES.index("s")  # sharpness: reported, not additive


def shard_rows(m_global, rank, world):
    """Contiguous row block [lo, hi) of ``rank``; the first m % world ranks
    take one extra row."""
    base, extra = divmod(int(m_global), int(world))
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_draws(draws, rank, world):
    """This rank's slice of one global iteration's host draws, plus the
    step keyword arguments (ray_base, m_global, smooth_global)."""
    m = len(draws.ray_ids)
    lo, hi = shard_rows(m, rank, world)
    n_smooth = draws.n_smooth
    d = dataclasses.replace(draws, ray_ids=draws.ray_ids[lo:hi].copy(),
                            smooth=draws.smooth if rank == 0 else None,
                            smooth_raw=draws.smooth_raw if rank == 0 else None)
    return d, dict(ray_base=lo, m_global=m, smooth_global=max(n_smooth, 1))


class DataParallelStep:
    """Objective + backward of one iteration across ranks.

    ``engine`` is a StepEngine (or anything with the same ``launch`` and a
    ``model.arena.grads`` tensor); ``dist`` is ``torch.distributed`` with an
    initialised process group (NCCL on GPUs, gloo in the CPU tests)."""

    def __init__(self, engine, dist, group=None):
        self.engine = engine
        self.dist = dist
        self.group = group

    def __call__(self, cfg, draws, ids, sm, **kw):
        eng = self.engine
        ws = eng.launch(cfg, draws, ids, sm, phases=1, **kw)
        self.dist.all_reduce(ws["counts"], group=self.group)            # exchange 1
        ws = eng.launch(cfg, draws, ids, sm, phases=2, fresh=False, **kw)
        self.dist.all_reduce(eng.model.arena.grads, group=self.group)   # exchange 2
        parts = ws["parts"]
        s = parts[S_SLOT].clone()
        self.dist.all_reduce(parts, group=self.group)
        parts[S_SLOT] = s
        return ws
