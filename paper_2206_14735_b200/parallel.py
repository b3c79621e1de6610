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
   replicated Adam form.  ``overlap=True`` (NCCL, opt-in) runs the backward in
   two launches and issues the geometry grids' reduce-scatter (their
   gradients are final after the geometry backward) under the colour
   backward; off by default: the colour backward fills the register file, so
   concurrent kernels cannot share its SMs (a single-GPU overlap of Adam with
   it measured slower), and this run has no multi-GPU box to measure on.

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

    def __init__(self, engine, dist, group=None, shard_adam=True, overlap=False):
        self.engine = engine
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.nccl = dist.get_backend(group) == "nccl"
        self.shard_adam = bool(shard_adam) and self.world > 1
        self.overlap = overlap

    def chunks(self, n):
        """Arena chunks exchanged separately: [(0, a), (a, n)] with a the end of
        the geometry grids rounded down to 4 x world (overlap form), else [(0, n)]."""
        eng = self.engine
        q = 4 * self.world
        a = 0
        # overlap="always": the two-chunk form on any backend (tests run it on gloo)
        if (self.overlap and (self.nccl or self.overlap == "always") and self.shard_adam
                and not getattr(eng, "deterministic", False)):
            try:
                a = int(eng.model.arena["colorgrid"].offset) // q * q
            except (KeyError, AttributeError, TypeError):
                a = 0
        if 0 < a < n and (n - a) % q == 0:
            return [(0, a), (a, n)]
        return [(0, n)]

    def shards(self, n):
        """This rank's [lo, hi) in every chunk."""
        out = []
        for c0, c1 in self.chunks(n):
            chunk = (c1 - c0) // self.world
            if chunk * self.world != c1 - c0 or chunk % 4:
                raise ValueError("arena chunks must split into equal 16-byte-aligned shards")
            out.append((c0 + self.rank * chunk, c0 + (self.rank + 1) * chunk))
        return out

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
        g = eng.model.arena.grads                                       # exchange 2
        chunks = self.chunks(g.numel()) if self.shard_adam else [(0, g.numel())]
        if len(chunks) == 2:  # geometry-grid reduce-scatter under the colour backward
            eng.launch(cfg, draws, ids, sm, phases=2 | 4, fresh=False, **kw)
            works = [self._reduce_scatter(g, *chunks[0], async_op=True)]
            ws = eng.launch(cfg, draws, ids, sm, phases=2 | 8, fresh=False, **kw)
            works.append(self._reduce_scatter(g, *chunks[1], async_op=True))
            for wk in works:
                if wk is not None:
                    wk.wait()
        else:
            ws = eng.launch(cfg, draws, ids, sm, phases=2, fresh=False, **kw)
            if self.shard_adam:
                self._reduce_scatter(g, *chunks[0])
            else:
                self.dist.all_reduce(g, group=self.group)
        parts = ws["parts"]
        s = parts[S_SLOT].clone()
        self.dist.all_reduce(parts, group=self.group)
        parts[S_SLOT] = s
        # every rank raises (and skips Adam) if any rank's step flagged an error
        self.dist.all_reduce(ws["status"], op=self.dist.ReduceOp.MAX, group=self.group)
        return ws

    def _reduce_scatter(self, g, c0, c1, async_op=False):
        """Sum of chunk [c0, c1) into this rank's shard of it (NCCL, in place:
        the output is the rank's slice of the input).  gloo has no
        reduce-scatter, so the CPU tests take the chunk's sum everywhere (a
        superset of the shard).  NCCL errors propagate."""
        t = g[c0:c1]
        if self.nccl:
            chunk = (c1 - c0) // self.world
            lo = self.rank * chunk
            return self.dist.reduce_scatter_tensor(t[lo:lo + chunk], t, group=self.group,
                                                   async_op=async_op)
        return self.dist.all_reduce(t, group=self.group, async_op=async_op)

    def adam(self, opt, **kw):
        """The optimizer step after ``__call__``: sharded update + all-gather."""
        if not self.shard_adam:
            opt._launch(**kw)
            return
        a = opt.arena
        mine = self.shards(a.n)
        # one launch: Adam on this rank's shards, and the partial sums left in
        # the other ranks' shards zeroed (the guard gates all of it)
        opt._launch(owned=mine, **kw)
        for (c0, c1), (lo, hi) in zip(self.chunks(a.n), mine):
            self._all_gather(a.params[c0:c1], lo - c0, hi - c0)

    def _all_gather(self, t, lo, hi):
        if self.nccl:
            self.dist.all_gather_into_tensor(t, t[lo:hi], group=self.group)  # in place
            return
        n = hi - lo
        parts = [t[r * n:(r + 1) * n] for r in range(self.world)]
        self.dist.all_gather(parts, t[lo:hi].clone(), group=self.group)

    def gather_adam_state(self, opt):
        """Assemble the full Adam m / v on every rank (e.g. before save_model)."""
        if not self.shard_adam:
            return
        for (c0, c1), (lo, hi) in zip(self.chunks(opt.arena.n), self.shards(opt.arena.n)):
            self._all_gather(opt.m_arena[c0:c1], lo - c0, hi - c0)
            self._all_gather(opt.v_arena[c0:c1], lo - c0, hi - c0)
