"""Ray-sharded data parallelism: the package's
DataParallelStep / shard_draws over a world of 2 must reproduce the
unsharded step (all-reduced gradients, loss parts, partition counts).

* CPU (gloo): the oracle stands in for each rank's device step.
* GPU: the real device step on both ranks (this environment has one GPU, so
  both ranks share it and the collectives are gloo on the host; the NCCL
  path of bench.py runs the same DataParallelStep)."""

import os
import socket
import sys
from types import SimpleNamespace

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)


def test_shard_rows_partition():
    from paper_2206_14735_b200.parallel import shard_rows
    for m in (1, 7, 64, 6144, 6145):
        for world in (1, 2, 3, 8):
            blocks = [shard_rows(m, r, world) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == m
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1


def test_shard_draws_slices_rays_and_keeps_smoothness_on_rank0():
    from paper_2206_14735_b200.engine import HostDraws
    from paper_2206_14735_b200.parallel import shard_draws
    d = HostDraws(3, np.arange(10, dtype=np.int64) * 7, np.ones((8, 3), np.float32), None, [])
    d0, kw0 = shard_draws(d, 0, 3)
    d2, kw2 = shard_draws(d, 2, 3)
    assert list(d0.ray_ids) == [0, 7, 14, 21] and d0.smooth is not None
    assert list(d2.ray_ids) == [49, 56, 63] and d2.smooth is None
    assert kw0 == dict(ray_base=0, m_global=10, smooth_global=4)
    assert kw2 == dict(ray_base=7, m_global=10, smooth_global=4)
    assert d2.iteration == 3


def _sub_batch(b, lo, hi):
    from oracle import gridsurf_oracle as O
    m = len(b)

    def cut(x):
        return x[lo:hi] if isinstance(x, np.ndarray) and x.shape[:1] == (m,) else x
    return O.Batch(*(cut(getattr(b, k)) for k in
                     ("frame_ids", "pixels", "color", "depth_ray", "valid", "dir_cam", "near", "far")))


class OracleEngine:
    """Stand-in for StepEngine on CPU: phase 1 = sampling + local partition
    counts, phase 2 = objective + backward with the global normalisers read
    back from the (all-reduced) counts; gradients land in a flat arena."""

    def __init__(self, torch, G, P, cfg, batch, it):
        self.torch, self.G, self.P, self.cfg, self.batch, self.it = torch, G, P, cfg, batch, it
        n = sum(a.size for a in P.arrays())
        self.model = SimpleNamespace(arena=SimpleNamespace(grads=torch.zeros(n, dtype=torch.float64)))
        self.ws = dict(counts=torch.zeros(4, dtype=torch.int64),
                       parts=torch.zeros(8, dtype=torch.float64),
                       status=torch.zeros(8, dtype=torch.int32))

    def launch(self, cfg, draws, ids, sm, phases=3, fresh=True, ray_base=0, m_global=None,
               smooth_global=None):
        from oracle import gridsurf_oracle as O
        lo, hi = ray_base, ray_base + len(ids)
        sub = _sub_batch(self.batch, lo, hi)
        shard = dict(row_base=lo, m_global=m_global, smooth=sm is not None)
        if phases == 1:
            R = O.train_objective(self.P, self.G.ds, sub, self.it, self.cfg, want_grads=False,
                                  shard=shard)
            e = R["extras"]
            self.ws["counts"][:] = self.torch.tensor(
                [e["n_valid_rays"], e["n_tr"], e["n_fs"], e["n_eik"]], dtype=self.torch.int64)
            return self.ws
        c = self.ws["counts"].tolist()
        shard.update(n_valid=c[0], n_eik=c[3], n_smooth=smooth_global)
        R = O.train_objective(self.P, self.G.ds, sub, self.it, self.cfg, shard=shard)
        flat = np.concatenate([R["grads"][n].reshape(-1) for n in self.P.names()])
        self.model.arena.grads.copy_(self.torch.from_numpy(flat))
        names = ("total", "rgb", "depth", "sdf", "fs", "eik", "smooth", "s")
        self.ws["parts"][:] = self.torch.tensor([R["parts"][k] for k in names], dtype=self.torch.float64)
        return self.ws


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    from _golden import load, oracle_params
    from oracle import gridsurf_oracle as O
    from paper_2206_14735_b200.engine import HostDraws
    from paper_2206_14735_b200.parallel import DataParallelStep, shard_draws

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        G = load("tiny", "double")
        P = oracle_params(G)
        cfg = G.cfg
        it = G.meta["iteration"]
        rng = O.substream(cfg.seed, O.RAYS, it)
        intr = G.ds.intrinsics
        flat = rng.integers(0, G.ds.colors.shape[0] * intr.height * intr.width, size=cfg.batch_rays)
        batch = O.batch_from_flat(G.ds, flat)
        draws = HostDraws(it, flat, np.zeros((2, 3)), None, [])  # smoothness drawn by the oracle
        d, kw = shard_draws(draws, rank, world)
        kw["smooth_global"] = cfg.weights.smooth_count
        eng = OracleEngine(torch, G, P, cfg, batch, it)
        ws = DataParallelStep(eng, dist)(cfg, d, d.ray_ids, d.smooth, **kw)
        if rank == 0:
            R = O.train_objective(P, G.ds, batch, it, cfg)
            ref = np.concatenate([R["grads"][n].reshape(-1) for n in P.names()])
            got = eng.model.arena.grads.numpy()
            names = ("total", "rgb", "depth", "sdf", "fs", "eik", "smooth", "s")
            np.savez(out, got=got, ref=ref, parts=ws["parts"].numpy(),
                     ref_parts=np.array([R["parts"][k] for k in names]),
                     counts=ws["counts"].numpy(),
                     ref_counts=np.array([R["extras"]["n_valid_rays"], R["extras"]["n_tr"],
                                          R["extras"]["n_fs"], R["extras"]["n_eik"]]))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.timeout(600)
def test_data_parallel_gloo_world2_equals_unsharded(tmp_path):
    import torch.multiprocessing as mp
    out = str(tmp_path / "dp.npz")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    z = np.load(out)
    # counts are integers: exact; parts / gradients: float64 summation order only
    assert (z["counts"] == z["ref_counts"]).all()
    np.testing.assert_allclose(z["parts"], z["ref_parts"], rtol=1e-12, atol=1e-15)
    scale = np.abs(z["ref"]).max()
    assert np.abs(z["got"] - z["ref"]).max() <= 1e-12 * scale


def _gpu_worker(rank, world, port, out, precision="double", refine=False):
    """Real device step under DataParallelStep; gloo collectives (both ranks
    share the one GPU of this environment; collectives run on the host).
    ``refine``: pose refinement on (per-rank partial pose gradients)."""
    import torch
    import torch.distributed as dist
    from _golden import load
    from paper_2206_14735_b200 import data, engine, optimizer, seeds
    from paper_2206_14735_b200.parallel import DataParallelStep, shard_draws
    from paper_2206_14735_b200.renderer import engine_for

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        G = load("small", precision)
        cfg = optimizer.TrainConfig(precision=precision, **{
            k: v for k, v in G.meta["cfg"].items() if k not in ("bounds", "voxel_sizes")},
            voxel_sizes=G.cfg.voxel_sizes, bounds=G.cfg.bounds, refine_poses=refine)
        cfg.weights.smooth_count = G.meta["smooth_count"]
        ds = data.Dataset(G.a["colors_u8"], G.a["depths_u16"], G.a["poses"], G.ds.intrinsics)
        model = optimizer.build_model(ds, cfg, skip_init=True, device=torch.device("cuda", 0))
        eng = engine_for(model, ds)
        it = G.meta["iteration"]
        full = engine.host_draws(model, ds, cfg, it)
        d, kw = shard_draws(full, rank, world)
        ids, sm = eng.upload(d)
        ws = DataParallelStep(eng, dist)(cfg, d, ids, sm, **kw)
        got = model.arena.grads.cpu().numpy().copy()
        parts = ws["parts"].cpu().numpy().copy()
        counts = ws["counts"].cpu().numpy().copy()
        if rank == 0:  # the unsharded step on the same process/GPU
            ids1, sm1 = eng.upload(full)
            ws1 = eng.launch(cfg, full, ids1, sm1)
            ref = model.arena.grads.cpu().numpy()
            np.savez(out, got=got, ref=ref, parts=parts, ref_parts=ws1["parts"].cpu().numpy(),
                     counts=counts, ref_counts=ws1["counts"].cpu().numpy())
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.timeout(900)
@pytest.mark.parametrize("refine", [False, True])
def test_data_parallel_device_step_world2_equals_unsharded(tmp_path, refine):
    import torch.multiprocessing as mp
    out = str(tmp_path / "dpgpu.npz")
    mp.spawn(_gpu_worker, args=(2, _free_port(), out, "double", refine), nprocs=2, join=True)
    z = np.load(out)
    assert (z["counts"] == z["ref_counts"]).all()
    np.testing.assert_allclose(z["parts"], z["ref_parts"], rtol=1e-12, atol=1e-15)
    assert np.abs(z["got"] - z["ref"]).max() <= 1e-11 * np.abs(z["ref"]).max()


class _FakeArena:
    def __init__(self, torch, n):
        self.n = n
        self.params = torch.linspace(-1.0, 1.0, n, dtype=torch.float64)
        self.grads = torch.zeros(n, dtype=torch.float64)

    def __getitem__(self, name):  # the "colorgrid" parameter starts at element 300
        from types import SimpleNamespace
        return SimpleNamespace(offset=300)


class _TorchAdam:
    """Adam restated in torch (gs/optimizer.py:38-55) over an arena range,
    standing in for gsb_adam_step in the CPU choreography test."""

    def __init__(self, torch, arena, lr=1e-2):
        self.arena, self.lr, self.t = arena, lr, [0]
        self.m_arena = torch.zeros_like(arena.params)
        self.v_arena = torch.zeros_like(arena.params)

    def _launch(self, lo=0, hi=None, owned=None, **kw):
        a = self.arena
        if owned is not None:  # the rank's shards; the rest is only zeroed
            for x, y in owned:
                self._launch(x, y)
            a.grads.zero_()
            return
        hi = a.n if hi is None else hi
        t = float(self.t[0])
        g = a.grads[lo:hi]
        m = self.m_arena[lo:hi]
        v = self.v_arena[lo:hi]
        m.mul_(0.9).add_(0.1 * g)
        v.mul_(0.999).add_(0.001 * g * g)
        a.params[lo:hi] -= self.lr * (m / (1 - 0.9 ** t)) / ((v / (1 - 0.999 ** t)).sqrt() + 1e-8)
        g.zero_()


class _FakeStepEngine:
    def __init__(self, torch, arena, rank):
        import types
        self.torch, self.rank = torch, rank
        self.model = types.SimpleNamespace(arena=arena)
        self.split = 300  # "colorgrid" offset of the fake arena
        self.ws = dict(counts=torch.zeros(4, dtype=torch.int64), parts=torch.zeros(8, dtype=torch.float64),
                       status=torch.zeros(8, dtype=torch.int32))

    def launch(self, cfg, draws, ids, sm, phases=3, fresh=True, it=0, **kw):
        if phases == 1:
            self.ws["counts"][:] = self.torch.tensor([1, 2, 3, 4]) * (self.rank + 1)
            return self.ws
        a = self.model.arena
        gen = self.torch.Generator().manual_seed(1000 * kw.get("step", 0) + self.rank)
        full = self.torch.randn(a.n, generator=gen, dtype=self.torch.float64)
        cut = self.split  # split backward: part A writes [0, cut), part B the rest
        if phases & 12 == 4:
            a.grads[:cut] += full[:cut]
        elif phases & 12 == 8:
            a.grads[cut:] += full[cut:]
        else:
            a.grads += full
        self.ws["parts"][:] = float(self.rank + 1)
        return self.ws


def _shard_worker(rank, world, port, out, steps, n, overlap):
    import torch
    import torch.distributed as dist
    from paper_2206_14735_b200.parallel import DataParallelStep
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        arena = _FakeArena(torch, n)
        opt = _TorchAdam(torch, arena)
        dp = DataParallelStep(_FakeStepEngine(torch, arena, rank), dist, overlap=overlap)
        assert dp.shard_adam
        assert len(dp.chunks(n)) == (2 if overlap == "always" else 1)
        for k in range(steps):
            ws = dp(None, None, None, None, step=k)
            opt.t = [k + 1]
            dp.adam(opt)
            assert float(arena.grads.abs().max()) == 0.0
        dp.gather_adam_state(opt)
        if rank == 0:
            np.savez(out, params=arena.params.numpy(), m=opt.m_arena.numpy(), v=opt.v_arena.numpy(),
                     counts=ws["counts"].numpy(), parts=ws["parts"].numpy())
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("overlap", [True, "always"])
def test_sharded_adam_gloo_world2_equals_replicated(tmp_path, overlap):
    """reduce-scatter -> Adam on the rank's shard -> all-gather (parallel.py)
    gives the replicated all-reduce + full Adam result, parameters and the
    gathered moments alike (gloo: the reduce-scatter falls back to all-reduce)."""
    import torch
    import torch.multiprocessing as mp
    out, steps, n, world = str(tmp_path / "shard.npz"), 3, 1024, 2
    mp.spawn(_shard_worker, args=(world, _free_port(), out, steps, n, overlap), nprocs=world, join=True)
    z = np.load(out)
    arena = _FakeArena(torch, n)
    opt = _TorchAdam(torch, arena)
    for k in range(steps):
        for r in range(world):
            gen = torch.Generator().manual_seed(1000 * k + r)
            arena.grads += torch.randn(n, generator=gen, dtype=torch.float64)
        opt.t = [k + 1]
        opt._launch()
    np.testing.assert_allclose(z["params"], arena.params.numpy(), rtol=0, atol=1e-15)
    np.testing.assert_allclose(z["m"], opt.m_arena.numpy(), rtol=0, atol=1e-15)
    np.testing.assert_allclose(z["v"], opt.v_arena.numpy(), rtol=0, atol=1e-15)
    assert list(z["counts"]) == [3, 6, 9, 12]
    assert z["parts"][0] == 3.0 and z["parts"][7] == 1.0  # s slot is not summed


def test_adam_segments_owned():
    """ZeRO-1 segments over the whole arena: the owned ranges keep their
    learning-rate runs, everything else is marked not-owned (lr -1)."""
    from types import SimpleNamespace
    from paper_2206_14735_b200.optimizer import Adam
    a = Adam.__new__(Adam)
    a.arena = SimpleNamespace(n=256)
    a._segments = lambda: ([0, 64, 128, 200], [0.01, 0.001, 0.0005, 0.0])
    assert a._segments_owned([(0, 256)]) == ([0, 64, 128, 200], [0.01, 0.001, 0.0005, 0.0])
    assert a._segments_owned([(32, 160)]) == ([0, 32, 64, 128, 160], [-1.0, 0.01, 0.001, 0.0005, -1.0])
    assert a._segments_owned([(0, 64), (128, 192)]) == ([0, 64, 128, 192], [0.01, -1.0, 0.0005, -1.0])


def test_adam_segments_in_range():
    """Learning-rate runs of a shard, relative to its start."""
    from paper_2206_14735_b200.optimizer import Adam
    a = Adam.__new__(Adam)
    a._segments = lambda: ([0, 64, 128, 200], [0.01, 0.001, 0.0005, 0.0])
    assert a._segments_in(0, 64) == ([0], [0.01])
    assert a._segments_in(32, 160) == ([0, 32, 96], [0.01, 0.001, 0.0005])
    assert a._segments_in(128, 256) == ([0, 72], [0.0005, 0.0])
    assert a._segments_in(200, 256) == ([0], [0.0])


def _gpu_adam_worker(rank, world, port, out):
    """Two device steps + sharded gsb_adam_step on each rank (gloo collectives,
    both ranks on the one GPU), against the 1-process step + full Adam."""
    import torch
    import torch.distributed as dist
    from _golden import load
    from paper_2206_14735_b200 import data, engine, optimizer
    from paper_2206_14735_b200.parallel import DataParallelStep, shard_draws
    from paper_2206_14735_b200.renderer import engine_for

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        G = load("small", "double")
        cfg = optimizer.TrainConfig(precision="double", **{
            k: v for k, v in G.meta["cfg"].items() if k not in ("bounds", "voxel_sizes")},
            voxel_sizes=G.cfg.voxel_sizes, bounds=G.cfg.bounds)
        cfg.weights.smooth_count = G.meta["smooth_count"]
        ds = data.Dataset(G.a["colors_u8"], G.a["depths_u16"], G.a["poses"], G.ds.intrinsics)
        res = []
        for sharded in (True, False):
            model = optimizer.build_model(ds, cfg, skip_init=True, device=torch.device("cuda", 0))
            opt = optimizer.make_optimizer(model, cfg)
            eng = engine_for(model, ds)
            dp = DataParallelStep(eng, dist, overlap="always") if sharded else None
            for it in range(2):
                full = engine.host_draws(model, ds, cfg, it)
                if sharded:
                    d, kw = shard_draws(full, rank, world)
                    ids, sm = eng.upload(d)
                    dp(cfg, d, ids, sm, **kw)
                    opt.t = [t + 1 for t in opt.t]
                    dp.adam(opt)
                else:
                    ids, sm = eng.upload(full)
                    eng.launch(cfg, full, ids, sm)
                    opt.t = [t + 1 for t in opt.t]
                    opt._launch()
            if sharded:
                dp.gather_adam_state(opt)
            torch.cuda.synchronize()
            res.append((model.arena.params.cpu().numpy().copy(), opt.m_arena.cpu().numpy().copy()))
        if rank == 0:
            np.savez(out, p_sh=res[0][0], m_sh=res[0][1], p_1=res[1][0], m_1=res[1][1])
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.timeout(900)
def test_sharded_adam_device_world2_equals_single(tmp_path):
    import torch.multiprocessing as mp
    out = str(tmp_path / "shadam.npz")
    mp.spawn(_gpu_adam_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    z = np.load(out)
    # sharded gradients are a float64 sum in another order: Adam amplifies
    # last-bit differences of near-zero gradients only up to lr
    assert np.abs(z["p_sh"] - z["p_1"]).max() <= 1e-9
    assert np.abs(z["m_sh"] - z["m_1"]).max() <= 1e-9 * max(np.abs(z["m_1"]).max(), 1e-300)


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["single", "double"])
def test_adam_owned_ranges_on_device(precision):
    """One Adam launch over the whole arena with owned ranges (a data-parallel
    rank's shards): the owned parameters, moments and cleared gradients are
    bit-identical to a plain update, the foreign ones keep their parameters
    and moments and get their gradients zeroed -- including ranges that start
    and end half-way into an 8-float vector (the float32 kernel moves 32-byte
    vectors, the ranges are 16-byte aligned)."""
    import torch
    from paper_2206_14735_b200 import optimizer
    from test_train import small_setup
    ds, cfg = small_setup(precision=precision)
    model = optimizer.build_model(ds, cfg, skip_init=True, device=torch.device("cuda", 0))
    a = model.arena
    n = a.n
    tdt = a.params.dtype

    def init(opt):
        a.params.copy_(torch.randn(n, generator=g0, dtype=torch.float64).to(tdt))
        a.grads.copy_(torch.randn(n, generator=g0, dtype=torch.float64).to(tdt))
        a.grads[: n // 3].zero_()  # untouched gradients too
        opt.m_arena.copy_(torch.randn(n, generator=g0, dtype=torch.float64).to(tdt) * 0.1)
        opt.v_arena.copy_(torch.rand(n, generator=g0, dtype=torch.float64).to(tdt) * 0.01)
        opt.t = [4] * len(opt.t)

    lo, hi = (n // 16) * 8 + 4, (n // 2) // 8 * 8 - 4  # both 4 floats off the 8-float grid
    owned = [(lo, hi), (hi + 8, n)]
    out = []
    for ranges in (None, owned):
        g0 = torch.Generator().manual_seed(11)
        opt = optimizer.make_optimizer(model, cfg)
        init(opt)
        before = (a.params.cpu().numpy().copy(), opt.m_arena.cpu().numpy().copy(),
                  opt.v_arena.cpu().numpy().copy())
        opt.t = [5] * len(opt.t)
        if ranges is None:
            opt._launch()
        else:
            opt._launch(owned=ranges)
        torch.cuda.synchronize()
        out.append((before, a.params.cpu().numpy().copy(), opt.m_arena.cpu().numpy().copy(),
                    opt.v_arena.cpu().numpy().copy(), a.grads.cpu().numpy().copy()))
    (b0, p_full, m_full, v_full, _), (b1, p_own, m_own, v_own, g_own) = out
    for x, y in zip(b0, b1):
        np.testing.assert_array_equal(x, y)  # same starting state
    mine = np.zeros(n, dtype=bool)
    for x, y in owned:
        mine[x:y] = True
    np.testing.assert_array_equal(p_own[mine], p_full[mine])
    np.testing.assert_array_equal(m_own[mine], m_full[mine])
    np.testing.assert_array_equal(v_own[mine], v_full[mine])
    np.testing.assert_array_equal(p_own[~mine], b1[0][~mine])
    np.testing.assert_array_equal(m_own[~mine], b1[1][~mine])
    np.testing.assert_array_equal(v_own[~mine], b1[2][~mine])
    assert not np.any(g_own)


def test_strong_split_rows_cover_the_global_batch():
    """bench.py --strong: the global batch (BASELINE c3(i), M = 6144) split by
    rows over N ranks covers every row once, in order, sizes within one, and
    each rank's ray_base is its first global row (so its device PCG streams
    start where the 1-GPU batch's rows do)."""
    import numpy as np
    from paper_2206_14735_b200.engine import HostDraws
    from paper_2206_14735_b200.parallel import shard_draws, shard_rows
    for m, world in [(6144, 1), (6144, 2), (6144, 3), (6145, 4), (6144, 8), (7, 8)]:
        spans = [shard_rows(m, r, world) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == m
        assert all(a[1] == b[0] for a, b in zip(spans[:-1], spans[1:]))
        sizes = [hi - lo for lo, hi in spans]
        assert max(sizes) - min(sizes) <= 1
        ids = np.arange(m, dtype=np.int64) * 3
        d = HostDraws(0, ids, np.zeros((2, 3)), None, [])
        got = []
        for r in range(world):
            dr, kw = shard_draws(d, r, world)
            assert kw["ray_base"] == spans[r][0] and kw["m_global"] == m
            got.append(dr.ray_ids)
        np.testing.assert_array_equal(np.concatenate(got), ids)
