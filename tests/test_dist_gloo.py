"""Multi-rank host logic of the sharded mapping (config 4) on CPU with gloo, world size 2.

The kernels need a GPU; what is tested here is everything around them: keyframe sharding, the
gradient all-reduce (the per-rank gradients are the oracle's, so the reduced sum is compared
with the single-process sum over all keyframes), and the rank-ordered gather of densify
candidates that makes every rank append identical Gaussians."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _mapping_module():
    """paper_2311_11700_b200.mapping imports the ctypes binding, which needs libgs.so; the helpers
    under test are pure torch.distributed, so load the module source with a stub package."""
    import importlib.util
    import sys
    import types
    if "paper_2311_11700_b200" not in sys.modules:
        try:
            import paper_2311_11700_b200  # noqa: F401
        except ImportError:
            stub = types.ModuleType("paper_2311_11700_b200")
            stub.__path__ = [os.path.join(ROOT, "paper_2311_11700_b200")]
            for name in ("GS_DENSIFY_ADD", "GS_DENSIFY_PRUNE", "GS_FLAG_NO_HOST_SYNC", "GS_DENSIFY_DEGENERATE_APPLY",
                         "GS_DENSIFY_DEGENERATE_FLAG", "GS_FLAG_POSE_COV_PATH", "GS_FLAG_BWD_SCREEN_ONLY",
                         "GS_FLAG_BWD_CHAIN_ONLY"):
                setattr(stub, name, 0)
            for name in ("densify_cfg", "gs_adam_step", "gs_adam_step_rows", "gs_densify_append", "gs_densify_prune",
                         "make_camera", "gs_densify_accum_grad", "gs_densify_split_clone", "gs_pose_step",
                         "gs_render_bwd_l1"):
                setattr(stub, name, None)
            sys.modules["paper_2311_11700_b200"] = stub
            pl = types.ModuleType("paper_2311_11700_b200.pipeline")
            pl.RenderPipeline = None
            sys.modules["paper_2311_11700_b200.pipeline"] = pl
    spec = importlib.util.spec_from_file_location("paper_2311_11700_b200.mapping",
                                                  os.path.join(ROOT, "paper_2311_11700_b200", "mapping.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules[spec.name] = mod   # dataclasses resolve their module through sys.modules
    spec.loader.exec_module(mod)
    return mod


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_covers_keyframes_contiguously():
    m = _mapping_module()
    for world in (1, 2, 4, 8):
        got = [m.shard(8, world, r) for r in range(world)]
        assert sum(got, []) == list(range(8))
        assert all(len(g) == 8 // world for g in got)


def test_learning_rate_schedule_endpoints():
    m = _mapping_module()
    assert math.isclose(m.learning_rates(0)[0], 1.6e-5)
    assert math.isclose(m.learning_rates(100)[0], 1.7e-7, rel_tol=1e-9)
    assert m.learning_rates(50)[10] == 1e-2 and m.learning_rates(7)[11] == 5e-4
    # first-order SH coefficients (rows 14-22) only in bundle adjustment
    lr = m.learning_rates(3, rows=23, sh_linear=False)
    assert lr[11:14] == [5e-4] * 3 and lr[14:] == [0.0] * 9
    assert m.learning_rates(3, rows=23, sh_linear=True)[14:] == [5e-4] * 9


def test_uneven_shards_pad_to_equal_exchange_sizes():
    m = _mapping_module()
    for nk, world in ((8, 3), (1, 2), (5, 4), (3, 8)):
        per = m.shard_size(nk, world)
        got = [m.shard(nk, world, r) for r in range(world)]
        assert sum(got, []) == list(range(nk))
        assert all(len(g) <= per for g in got)


def _tiny_world(seed=0):
    import gs_inputs as gi
    rng = np.random.default_rng(seed)
    cam = gi.Camera(30.0, 30.0, 15.5, 11.5, 32, 24)
    n = 10
    z = rng.uniform(1.5, 3, n)
    p = np.zeros((14, n))
    p[0] = rng.uniform(-0.3, 0.3, n) * z
    p[1] = rng.uniform(-0.3, 0.3, n) * z
    p[2] = z
    p[3:6] = 0.1
    q = rng.normal(size=(4, n))
    p[6:10] = q / np.linalg.norm(q, axis=0)
    p[10] = rng.uniform(0.3, 0.8, n)
    p[11:14] = rng.uniform(0, 1, (3, n))
    views = []
    for k in range(4):
        import oracle
        d = np.concatenate([rng.normal(size=3) * 0.05, rng.normal(size=3) * 0.03])
        views.append(oracle.apply_twist(d, gi.identity_view().astype(np.float64)))
    return p, cam, views


def _degen_flags(p, cam, views, k):
    import gs_inputs as gi
    import oracle
    pr = oracle.project(p, views[k], cam, "f32")
    _, td = gi.random_images(cam.width, cam.height, 200 + k, 0.5, 3.0)
    return oracle.degenerate_mask(pr["mean2d"], pr["depth"], pr["tiles"], td, gamma=0.10)


def _gather_worker(rank, world, port, nk, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = _mapping_module()
        local = m.shard(nk, world, rank)
        S = m.shard_size(nk, world)
        cand = torch.zeros(S, 14, 4)
        counts = torch.zeros(S, dtype=torch.int64)
        for j, k in enumerate(local):
            counts[j] = 1 + k % 4
            cand[j, :, :1 + k % 4] = float(k)
        allc, allk = m.gather_candidates(cand, counts)
        g = torch.arange(5, dtype=torch.float32).repeat(3, 1) * (rank + 1)
        m.allreduce_grads(g, 3)   # only the first 3 columns are summed
        out[rank] = (allc.numpy().copy(), allk.numpy().copy(), g.numpy().copy())
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gloo_world3_uneven_candidate_gather_and_partial_allreduce():
    """8 keyframes over 3 ranks (3/3/2) and 1 keyframe over 2 ranks (1/0): equal-sized exchanges, the
    sets arrive in global keyframe order with the padding sets empty; allreduce_grads(g, n) sums only
    the n live columns of every row."""
    ctx = mp.get_context("spawn")
    for nk, world in ((8, 3), (1, 2)):
        mgr = ctx.Manager()
        out = mgr.dict()
        port = _free_port()
        procs = [ctx.Process(target=_gather_worker, args=(r, world, port, nk, out)) for r in range(world)]
        for pr in procs:
            pr.start()
        for pr in procs:
            pr.join(240)
            assert pr.exitcode == 0
        allc, allk, g = out[0]
        for r in range(1, world):
            np.testing.assert_array_equal(out[r][0], allc)
            np.testing.assert_array_equal(out[r][1], allk)
        got = [int(c) for c in allk if c > 0]
        assert got == [1 + k % 4 for k in range(nk)]
        live = [i for i, c in enumerate(allk) if c > 0]
        for k, i in enumerate(live):
            assert (allc[i, :, :1 + k % 4] == k).all()
        tot = sum(range(1, world + 1))
        np.testing.assert_array_equal(g[:, :3], np.arange(3, dtype=np.float32)[None].repeat(3, 0) * tot)
        np.testing.assert_array_equal(g[:, 3:], np.arange(3, 5, dtype=np.float32)[None].repeat(3, 0))


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import gs_inputs as gi
        import oracle
        m = _mapping_module()
        p, cam, views = _tiny_world()
        local = m.shard(len(views), world, rank)
        grad = torch.zeros(14, p.shape[1], dtype=torch.float64)
        for k in local:
            dc, dd = gi.upstream(cam.width, cam.height, 100 + k)
            grad += torch.from_numpy(oracle.backward(p, views[k], cam, dc, dd, "f64")["grad_params"])
        m.allreduce_grads(grad, grad.shape[1])
        # densify candidates: one padded set per local keyframe, count = k + 1, payload tagged by k
        max_add = 6
        cand = torch.zeros(len(local), 14, max_add)
        counts = torch.zeros(len(local), dtype=torch.int64)
        for j, k in enumerate(local):
            counts[j] = k + 1
            cand[j, :, : k + 1] = float(k)
        allc, allk = m.gather_candidates(cand, counts)
        # Eq. 9 flags: OR over the local keyframes, then the max all-reduce (ShardedMapper.step)
        mask = torch.zeros(p.shape[1], dtype=torch.uint8)
        for k in local:
            mask |= torch.from_numpy(_degen_flags(p, cam, views, k).astype(np.uint8))
        m.allreduce_mask(mask)
        out[rank] = (grad.numpy().copy(), allc.numpy().copy(), allk.numpy().copy(), mask.numpy().copy())
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gloo_world2_allreduce_and_candidate_gather():
    import gs_inputs as gi
    import oracle
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(240)
        assert pr.exitcode == 0
    p, cam, views = _tiny_world()
    want = np.zeros((14, p.shape[1]))
    for k in range(len(views)):
        dc, dd = gi.upstream(cam.width, cam.height, 100 + k)
        want += oracle.backward(p, views[k], cam, dc, dd, "f64")["grad_params"]
    g0, c0, k0, m0 = out[0]
    g1, c1, k1, m1 = out[1]
    want_m = np.zeros(p.shape[1], bool)
    per = [_degen_flags(p, cam, views, k) for k in range(len(views))]
    for f in per:
        want_m |= f
    np.testing.assert_array_equal(m0, m1)
    np.testing.assert_array_equal(m0.astype(bool), want_m)
    assert want_m.sum() > max(f.sum() for f in per)   # the union is larger than any one keyframe's set
    np.testing.assert_array_equal(g0, g1)                 # identical reduced bytes on every rank
    np.testing.assert_allclose(g0, want, rtol=1e-12, atol=1e-12)
    np.testing.assert_array_equal(c0, c1)
    np.testing.assert_array_equal(k0, k1)
    assert k0.tolist() == [1, 2, 3, 4]                     # global keyframe order: rank 0's, then rank 1's
    for k in range(4):
        assert (c0[k, :, : k + 1] == k).all()


def test_column_chunks_partition_and_alignment():
    m = _mapping_module()
    for n, c in ((0, 4), (1, 4), (31, 4), (32, 4), (1000, 4), (2_000_000, 4), (100, 1), (100, 7)):
        ch = m.column_chunks(n, c)
        assert len(ch) <= max(c, 1)
        assert [a for a, _ in ch] == sorted(a for a, _ in ch)
        covered = [i for a, b in ch for i in range(a, b)] if n <= 2000 else None
        if covered is not None:
            assert covered == list(range(n))
        else:
            assert ch[0][0] == 0 and ch[-1][1] == n and all(b == a2 for (_, b), (a2, _) in zip(ch, ch[1:]))
        assert all(a % 32 == 0 for a, _ in ch)


def _adam_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = _mapping_module()
        rows, cap, n = 14, 300, 261
        g = torch.arange(rows * cap, dtype=torch.float32).view(rows, cap) * (rank + 1)
        res = torch.full((rows, cap), -1.0)
        calls = []

        def adam(c0, c1):   # a per-column stand-in for the optimiser: reads the reduced gradient
            calls.append((c0, c1))
            res[:, c0:c1] = 2.0 * g[:, c0:c1]
        m.allreduce_adam(g, n, adam, packed=torch.empty(rows * cap), chunks=4)
        out[rank] = (g.numpy().copy(), res.numpy().copy(), calls)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gloo_bucketed_allreduce_overlapped_with_adam():
    """allreduce_adam at world sizes 2 and 3: the live columns [0, n) reduced in 32-aligned buckets,
    each bucket's optimiser call made on its reduced values in column order; columns >= n untouched."""
    ctx = mp.get_context("spawn")
    for world in (2, 3):
        mgr = ctx.Manager()
        out = mgr.dict()
        port = _free_port()
        procs = [ctx.Process(target=_adam_worker, args=(r, world, port, out)) for r in range(world)]
        for pr in procs:
            pr.start()
        for pr in procs:
            pr.join(240)
            assert pr.exitcode == 0
        rows, cap, n = 14, 300, 261
        base = np.arange(rows * cap, dtype=np.float32).reshape(rows, cap)
        tot = sum(range(1, world + 1))
        for r in range(world):
            g, res, calls = out[r]
            np.testing.assert_array_equal(g[:, :n], base[:, :n] * tot)
            np.testing.assert_array_equal(g[:, n:], base[:, n:] * (r + 1))
            np.testing.assert_array_equal(res[:, :n], 2.0 * base[:, :n] * tot)
            assert (res[:, n:] == -1.0).all()
            assert calls == [(0, 96), (96, 192), (192, 261)]
