"""ShardedMapper.step end to end with 2 ranks (-m gpu): both ranks on cuda:0, gloo over CUDA tensors
(this pool's boxes have one GPU; NCCL needs one GPU per rank). SURVEY.md §4 tests/dist, §8(e):

- after every step the parameters (all rows, the live columns), the map size and the Adam state are
  bitwise equal on the two ranks (NCCL and gloo deliver identical reduced bytes to every rank);
- the first step's all-reduced gradient equals the 1-rank run's (all 4 keyframes on one rank)
  within the summation-bound criterion of DESIGN.md §4.3 (bound from the oracle);
- with densification on the Eq. 8 expansion and the split/clone schedule (reading C30; every 2
  iterations in this test) change the map identically on both ranks, and each split/clone
  decision equals oracle.split_clone on the same (all-reduced) statistics.
"""
import os
import socket

import numpy as np
import pytest
import torch

import gs_inputs as gi
import oracle
from gpu_helpers import bound_factor, check_grads, key_cap_for, to_dev

pytestmark = pytest.mark.gpu

CAM = gi.Camera(300.0, 300.0, 159.5, 119.5, 320, 240)
N = 20_000
VIEWS = (221, 222, 223, 224)


def _world():
    p = gi.gaussians(N, 21)
    tgt = gi.gaussians(N, 22)
    views = [gi.room_view(s) for s in VIEWS]
    kc = max(key_cap_for(p, vv, CAM, slack=2.0)[0] for vv in views) + (1 << 20)
    return p, tgt, views, kc


def _run(rank, world, port, out, densify, steps):
    import torch.distributed as dist
    import paper_2311_11700_b200 as g
    from paper_2311_11700_b200.mapping import Keyframe, ShardedMapper, SplitClone
    torch.cuda.set_device(0)
    if world > 1:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p, tgt, views, kc = _world()
        cap = N + 60_000
        P = torch.zeros(14, cap, device="cuda")
        P[:, :N] = to_dev(p)
        probe = g.RenderPipeline(N, kc, CAM.width, CAM.height)
        kfs = []
        for vv in views:
            fr = probe.forward(to_dev(tgt), N, to_dev(vv), CAM)
            kfs.append(Keyframe(to_dev(vv), fr.color.clone(), fr.depth.clone()))
        mp = ShardedMapper(P, N, kfs, CAM, kc, max_add_per_kf=2048, densify=densify,
                           split_clone=SplitClone(every=2, until=10, grad_thresh=2e-4) if densify else None)
        mp.split_log = []
        rec = {"n": [], "grad1": None, "digest": []}
        for it in range(steps):
            mp.step()
            if it == 0:
                rec["grad1"] = mp.grad[:, :N].cpu().numpy().copy()
            n = mp.sync()
            rec["n"].append(n)
            state = torch.cat([mp.P[:, :n].reshape(-1), mp.raw[:, :n].reshape(-1), mp.m[:, :n].reshape(-1),
                               mp.v[:, :n].reshape(-1)]).cpu().numpy()
            if world > 1:   # bitwise equality across ranks, checked in-process
                lst = [None] * world
                dist.all_gather_object(lst, state.tobytes())
                assert all(x == lst[0] for x in lst), f"ranks diverged at step {it}"
            rec["digest"].append(state.view(np.uint32).astype(np.uint64).sum())
        rec["splits"] = [[t.cpu().numpy() for t in e] for e in mp.split_log]
        rec["local"] = mp.local
        out[rank] = rec
    finally:
        if world > 1:
            dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _spawn(world, densify, steps):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_run, args=(r, world, port, out, densify, steps)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(600)
        assert pr.exitcode == 0, f"rank exited with {pr.exitcode}"
    return [out[r] for r in range(world)]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.timeout(900)
def test_two_ranks_bitwise_equal_and_match_one_rank():
    two = _spawn(2, densify=False, steps=3)
    one = _spawn(1, densify=False, steps=1)
    assert two[0]["local"] == [0, 1] and two[1]["local"] == [2, 3]
    assert two[0]["digest"] == two[1]["digest"]
    # the first step's reduced gradient against the 1-rank sum over the same 4 keyframes
    p, tgt, views, kc = _world()
    bound = np.zeros((14, N))
    chain = np.zeros((14, N))
    nl_max = 0
    for vv in views:   # the L1 upstream's magnitudes are the oracle's as well (sign(0) aside)
        t = oracle.forward(tgt, vv, CAM, "f32")
        f = oracle.forward(p, vv, CAM, "f32")
        L = oracle.loss_l1(f["color"], f["depth"], t["color"], t["depth"], 0.9, 0.1)
        nl_max = max(nl_max, int(f["n_last"].max()))
        ob = oracle.backward(p, vv, CAM, L["dL_dcolor"], L["dL_ddepth"], "f32", bound=True)
        bound += ob["grad_bound"]
        chain += ob["chain_scale"]
    check_grads(two[0]["grad1"], one[0]["grad1"], bound, "2-rank vs 1-rank reduced gradient", k=bound_factor(nl_max),
                chain=chain)


@pytest.mark.timeout(900)
def test_two_ranks_densify_and_split_clone_identically():
    two = _spawn(2, densify=True, steps=4)
    assert two[0]["n"] == two[1]["n"] and two[0]["digest"] == two[1]["digest"]
    assert len(set(two[0]["n"])) > 1, two[0]["n"]   # the map changed size
    splits = two[0]["splits"]
    assert len(splits) == 2   # iterations 2 and 4
    for P0, acc, cnt, noise, P1, n1 in splits:
        want, clone, split = oracle.split_clone(P0, acc, cnt, noise, 2e-4, 0.02, capacity=P1.shape[1])
        assert clone.size + split.size > 0
        assert int(n1[0]) == want.shape[1]
        n_keep = P0.shape[1] - split.size
        np.testing.assert_array_equal(P1[:, :n_keep + clone.size], want[:, :n_keep + clone.size].astype(np.float32))
        np.testing.assert_allclose(P1[:, n_keep + clone.size:want.shape[1]], want[:, n_keep + clone.size:],
                                   rtol=1e-5, atol=1e-6)
    for (a0, c0, *_), (a1, c1, *_) in zip(two[0]["splits"], two[1]["splits"]):
        np.testing.assert_array_equal(a0, a1)
        np.testing.assert_array_equal(c0, c1)
