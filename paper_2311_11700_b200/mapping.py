"""Keyframe-sharded multi-GPU mapping (BASELINE config 4).

One process per GPU; each rank holds a full replica of the map and renders ITS keyframes:
  per local keyframe:  gs_project -> gs_bin_sort -> gs_render_fwd -> gs_loss_l1 -> gs_render_bwd (+=)
  exchange:            all_reduce(sum) of grad[14][cap] over NCCL (NVLink 5 / NVSwitch)
  optimiser:           gs_adam_step (identical on every rank -> parameters stay bitwise equal)
  adaptive expansion:  gs_densify_prune(ADD, gather mode) per local keyframe (Eq. 8)
                       -> all_gather of candidate counts and padded candidates (rank order)
                       -> gs_densify_append in global keyframe order (identical on every rank)
                       -> gs_densify_prune(PRUNE, opacity < 0.005)
  bundle adjustment:   Eq. 13 with `ba_iters`: map only for
                       the first half of the iterations, then map and keyframe poses (gs_render_bwd
                       with grad_pose per local keyframe -> gs_pose_step on that keyframe's view). A
                       keyframe's pose gradient comes only from its own render, so it stays on the rank
                       that owns the keyframe: no exchange.
Learning rates follow PAPER.md:931-933 (position 1.6e-5 -> 1.7e-7 exponentially over 100 steps,
colour 5e-4, opacity 1e-2, scale 2e-4, rotation 4e-5). The collective helpers are plain
torch.distributed calls and work with gloo on CPU tensors as well (tests/test_dist_gloo.py).
"""
from __future__ import annotations

import dataclasses

import torch
import torch.distributed as dist

from . import (GS_DENSIFY_ADD, GS_DENSIFY_DEGENERATE_APPLY, GS_DENSIFY_DEGENERATE_FLAG, GS_DENSIFY_PRUNE,
               GS_FLAG_NO_HOST_SYNC, densify_cfg, gs_adam_step, gs_adam_step_rows,
               gs_densify_append, gs_densify_prune, gs_pose_step, make_camera)
from .pipeline import RenderPipeline


def shard(n_items: int, world: int, rank: int) -> list[int]:
    """Contiguous keyframe shard of `rank` (8 keyframes over 1/2/4/8 ranks -> 8/4/2/1 each)."""
    per = (n_items + world - 1) // world
    return list(range(min(n_items, rank * per), min(n_items, (rank + 1) * per)))


def learning_rates(it: int, iters: int = 100, rows: int = 14) -> list[float]:
    """Per-row Adam learning rates at iteration `it`; with 23 rows (degree-1 SH)
    every SH coefficient takes the colour rate (the paper prints one colour rate)."""
    t = min(max(it, 0) / max(iters, 1), 1.0)
    lr_x = 1.6e-5 * (1.7e-7 / 1.6e-5) ** t
    return [lr_x] * 3 + [2e-4] * 3 + [4e-5] * 4 + [1e-2] + [5e-4] * (rows - 11)


def allreduce_grads(grad: torch.Tensor, group=None) -> None:
    """Sum the gradient buffer over ranks in place (NCCL on GPU, gloo on CPU)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(grad, op=dist.ReduceOp.SUM, group=group)


def allreduce_mask(mask: torch.Tensor, group=None) -> None:
    """OR of per-rank u8 flag masks (max all-reduce), so every rank applies the same Eq. 9 set."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(mask, op=dist.ReduceOp.MAX, group=group)


def gather_candidates(cand: torch.Tensor, counts: torch.Tensor, group=None):
    """all_gather of per-rank candidate sets cand[L][14][max_add] and counts[L] -> rank-ordered
    [R*L][14][max_add], [R*L] (the global keyframe order, since shards are contiguous)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return cand, counts
    world = dist.get_world_size(group)
    cs = [torch.empty_like(counts) for _ in range(world)]
    dist.all_gather(cs, counts, group=group)
    xs = [torch.empty_like(cand) for _ in range(world)]
    dist.all_gather(xs, cand, group=group)
    return torch.cat(xs, 0), torch.cat(cs, 0)


def raw_from_activated(p: torch.Tensor) -> torch.Tensor:
    """Inverse activations (log-scale, logit-opacity; reading C18) for the optimiser state (setup)."""
    r = p.clone()
    r[3:6] = torch.log(p[3:6])
    o = p[10].clamp(1e-6, 1 - 1e-6)
    r[10] = torch.log(o / (1 - o))
    return r


@dataclasses.dataclass
class Keyframe:
    view: torch.Tensor      # [3][4] world->camera (device)
    color: torch.Tensor     # [3][H][W] target colour
    depth: torch.Tensor     # [H][W] target depth


class ShardedMapper:
    def __init__(self, params: torch.Tensor, n: int, keyframes: list[Keyframe], cam, key_cap: int,
                 max_add_per_kf: int = 8192, w_color: float = 0.9, w_depth: float = 0.1, group=None,
                 densify: bool = True, ba_iters: int | None = None, lr_rho: float = 1e-3, lr_phi: float = 1e-3,
                 degenerate: tuple[float, float] | None = None):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if self.world > 1 else 0
        self.P = params                                   # activated [14][cap] or [23][cap] (degree-1 SH)
        self.rows = params.shape[0]
        self.cap = params.shape[1]
        self.raw = raw_from_activated(params)
        self.m = torch.zeros_like(params)
        self.v = torch.zeros_like(params)
        self.grad = torch.zeros_like(params)
        self.n = n
        self.n_dev = torch.tensor([n], dtype=torch.int64, device=params.device)
        self.cam = cam
        self.cm = make_camera(cam)
        self.pipe = RenderPipeline(self.cap, key_cap, cam.width, cam.height, params.device)
        self.w_color, self.w_depth = w_color, w_depth
        self.max_add = max_add_per_kf
        self.densify = densify
        self.it = 0
        self.ba_iters = ba_iters
        self.lr_rho, self.lr_phi = lr_rho, lr_phi
        self.pose_step = 0
        # Eq. 9 opacity degeneration (NEXT-2, reading C27) in expansion steps: (eta, gamma)
        self.degenerate = degenerate
        self.dmask = torch.zeros(self.cap, dtype=torch.uint8, device=params.device) if degenerate else None
        self.set_keyframes(keyframes)

    def set_keyframes(self, keyframes: list[Keyframe]):
        """(Re)assign the keyframe set (the SLAM driver's window, slam.py); per-keyframe buffers
        follow the local count."""
        dev = self.P.device
        self.keyframes = keyframes
        self.local = shard(len(keyframes), self.world, self.rank)
        L = len(self.local)
        if getattr(self, "cand", None) is None or self.cand.shape[0] != L:
            self.cand = torch.zeros(L, self.rows, self.max_add, device=dev)
            self.counts = torch.zeros(L, dtype=torch.int64, device=dev)
            # bundle adjustment state (Eq. 13): per local keyframe pose gradient and Adam moments
            self.gpose = torch.zeros(L, 6, dtype=torch.float64, device=dev)
            self.pm = torch.zeros(L, 6, device=dev)
            self.pv = torch.zeros(L, 6, device=dev)

    def poses_active(self) -> bool:
        """Eq. 13: poses are optimised only in the second half of the BA iterations."""
        return self.ba_iters is not None and self.it >= self.ba_iters // 2

    def render_backward(self):
        """fwd + L1 + bwd for every local keyframe, accumulating into grad."""
        self.grad[:, :self.n].zero_()
        degen = self.degenerate is not None and self.densify
        if degen:
            self.dmask.zero_()
        for j, k in enumerate(self.local):
            kf = self.keyframes[k]
            self.pipe.forward(self.P, self.n, kf.view, self.cam, bin_flags=GS_FLAG_NO_HOST_SYNC, fwd_flags=0)
            if degen:   # Eq. 9 flags from this keyframe's projection, ORed over the local keyframes
                gs_densify_prune(None, None, self.n_dev, self.n, self.cap, None, None, None, None, None, kf.depth,
                                 None, kf.view, self.cm, densify_cfg(GS_DENSIFY_DEGENERATE_FLAG,
                                                                     gamma=self.degenerate[1]),
                                 self.dmask, None, self.pipe.ws)
            dc, dd = self.pipe.loss_l1(self.cam, kf.color, kf.depth, self.w_color, self.w_depth)
            gp = None
            if self.poses_active():
                gp = self.gpose[j]
                gp.zero_()
            self.pipe.backward(self.P, self.n, kf.view, self.cam, dc, dd, self.grad, gp)
            if self.densify:   # Eq. 8 candidates from this keyframe's render (gather mode)
                cnt = self.counts[j:j + 1]
                gs_densify_prune(self.P, None, cnt, self.cap, self.cap, None, None, self.pipe.alpha, self.pipe.depth,
                                 kf.color, kf.depth, None, kf.view, self.cm,
                                 densify_cfg(GS_DENSIFY_ADD, max_add=self.max_add, rows=self.rows), None, self.cand[j],
                                 self.pipe.ws)

    def step(self):
        poses = self.poses_active()
        self.render_backward()
        allreduce_grads(self.grad, self.group)
        if self.degenerate is not None and self.densify:   # one Eq. 9 application per expansion step
            allreduce_mask(self.dmask, self.group)
            gs_densify_prune(self.P, self.raw, self.n_dev, self.n, self.cap, None, None, None, None, None, None,
                             None, None, None, densify_cfg(GS_DENSIFY_DEGENERATE_APPLY, eta=self.degenerate[0]),
                             self.dmask, None, self.pipe.ws)
        if poses:   # each rank updates the poses of its own keyframes (device-only pose step)
            self.pose_step += 1
            for j, k in enumerate(self.local):
                gs_pose_step(self.keyframes[k].view, self.gpose[j], self.pm[j], self.pv[j], self.pose_step,
                             self.lr_rho, self.lr_phi)
        self.it += 1
        lr = learning_rates(self.it - 1, rows=self.rows)
        if self.rows == 14:
            gs_adam_step(self.raw, self.P, self.grad, self.m, self.v, self.n, self.cap, lr, self.it)
        else:
            gs_adam_step_rows(self.raw, self.P, self.grad, self.m, self.v, self.n, self.cap, self.rows, lr, self.it)
        if self.densify:
            cand, counts = gather_candidates(self.cand, self.counts, self.group)
            gs_densify_append(self.P, self.raw, self.m, self.v, self.n_dev, self.cap, self.cap, cand, counts,
                              cand.shape[0], self.max_add, rows=self.rows)
            gs_densify_prune(self.P, self.raw, self.n_dev, self.cap, self.cap, self.m, self.v, None, None, None, None,
                             None, None, None, densify_cfg(GS_DENSIFY_PRUNE, rows=self.rows), None, None, self.pipe.ws)
            self.n = int(self.n_dev.item())   # one host read per mapping iteration (map size)
        return self.n
