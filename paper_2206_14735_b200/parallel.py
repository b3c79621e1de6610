"""Ray-sharded data parallelism.

One process per GPU.  Every rank draws the same global batch from the host
RNG (gs/optimizer.py:363-366) and keeps a contiguous block of rows; its
device PCG streams start at the block's global row (``ray_base``), so the
shards together are exactly the 1-GPU batch.  The step has two exchange
points:

1. after sampling (phase 1): all-reduce of the partition counts, because the
   depth and eikonal normalisers (n_valid, n_eik; gs/renderer.py:372-414)
   are global and n_eik depends on the sampled depths;
2. after the backward (phase 2): the gradient arena is reduce-scattered
   (each rank receives the global sum of its 1/N shard), every rank runs Adam
   on its shard only, and the updated parameters are all-gathered -- the
   wire bytes of one all-reduce, with Adam's HBM bytes divided by N (ZeRO-1;
   Adam m / v are valid on the owning rank, ``gather_adam_state`` assembles
   them for a checkpoint).  ``shard_adam=False`` keeps the all-reduce +
   replicated Adam form.

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

    def __init__(self, engine, dist, group=None, shard_adam=True):
        self.engine = engine
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.nccl = dist.get_backend(group) == "nccl"
        self.shard_adam = bool(shard_adam) and self.world > 1
        self._inplace_ok = True  # NCCL in-place reduce-scatter / all-gather accepted

    def shard(self, n):
        """This rank's arena range [lo, hi) (n is a multiple of 4 x world)."""
        chunk = n // self.world
        if chunk * self.world != n or chunk % 4:
            raise ValueError("arena length must split into equal 16-byte-aligned shards")
        return self.rank * chunk, (self.rank + 1) * chunk

    def __call__(self, cfg, draws, ids, sm, **kw):
        eng = self.engine
        ws = eng.launch(cfg, draws, ids, sm, phases=1, **kw)
        self.dist.all_reduce(ws["counts"], group=self.group)            # exchange 1
        ws = eng.launch(cfg, draws, ids, sm, phases=2, fresh=False, **kw)
        g = eng.model.arena.grads                                       # exchange 2
        done = False
        if self.shard_adam and self.nccl and self._inplace_ok:
            lo, hi = self.shard(g.numel())
            try:
                self.dist.reduce_scatter_tensor(g[lo:hi], g, group=self.group)  # in place
                done = True
            except (RuntimeError, ValueError):  # argument check refused the aliasing
                self._inplace_ok = False
        if not done:  # gloo has no reduce-scatter: the sum everywhere, the shard is a slice
            self.dist.all_reduce(g, group=self.group)
        parts = ws["parts"]
        s = parts[S_SLOT].clone()
        self.dist.all_reduce(parts, group=self.group)
        parts[S_SLOT] = s
        return ws

    def adam(self, opt, **kw):
        """The optimizer step after ``__call__``: sharded update + all-gather."""
        if not self.shard_adam:
            opt._launch(**kw)
            return
        a = opt.arena
        lo, hi = self.shard(a.n)
        opt._launch(lo=lo, hi=hi, **kw)       # zeroes grads[lo:hi]
        a.grads[:lo].zero_()                  # partial sums of the other shards
        a.grads[hi:].zero_()
        self._all_gather(a.params, lo, hi)

    def _all_gather(self, t, lo, hi):
        if self.nccl and self._inplace_ok:
            try:
                self.dist.all_gather_into_tensor(t, t[lo:hi], group=self.group)  # in place
                return
            except (RuntimeError, ValueError):
                self._inplace_ok = False
        n = hi - lo
        parts = [t[r * n:(r + 1) * n] for r in range(self.world)]
        self.dist.all_gather(parts, t[lo:hi].clone(), group=self.group)

    def gather_adam_state(self, opt):
        """Assemble the full Adam m / v on every rank (e.g. before save_model)."""
        if not self.shard_adam:
            return
        lo, hi = self.shard(opt.arena.n)
        self._all_gather(opt.m_arena, lo, hi)
        self._all_gather(opt.v_arena, lo, hi)
