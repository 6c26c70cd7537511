"""Keyframe-sharded multi-GPU mapping (BASELINE config 4).

One process per GPU; each rank holds a full replica of the map and renders ITS keyframes:
  per local keyframe:  gs_project -> gs_bin_sort -> gs_render_fwd -> gs_render_bwd_l1 (+=; the L1 loss fused)
  exchange:            all_reduce(sum) of the live columns grad[rows][:n] over NCCL (NVLink 5 /
                       NVSwitch) in 4 column buckets, each packed contiguously; each bucket's Adam step
                       overlaps the next buckets' reductions (allreduce_adam)
  optimiser:           gs_adam_step (identical on every rank -> parameters stay bitwise equal)
  adaptive expansion:  gs_densify_prune(ADD, gather mode) per local keyframe (Eq. 8)
                       -> all_gather of candidate counts and padded candidates (rank order)
                       -> gs_densify_append in global keyframe order (identical on every rank)
                       -> gs_densify_prune(PRUNE, opacity < 0.005)
  split / clone:       PAPER.md:935 (reading C30) with `split_clone`: gs_densify_accum_grad after every
                       local backward; every 10 iterations before 70 the statistics are all-reduced and
                       gs_densify_split_clone runs with the same seeded noise on every rank
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
               GS_FLAG_BWD_CHAIN_ONLY, GS_FLAG_BWD_SCREEN_ONLY, GS_FLAG_NO_HOST_SYNC, GS_FLAG_POSE_COV_PATH,
               densify_cfg, gs_adam_step, gs_adam_step_rows,
               gs_densify_accum_grad, gs_densify_append, gs_densify_prune, gs_densify_split_clone, gs_pose_step,
               gs_render_bwd_l1, make_camera)
from .pipeline import RenderPipeline


def shard(n_items: int, world: int, rank: int) -> list[int]:
    """Contiguous keyframe shard of `rank` (8 keyframes over 1/2/4/8 ranks -> 8/4/2/1 each; uneven
    counts give ceil-sized leading shards, e.g. 3/3/2 over 3 ranks)."""
    per = shard_size(n_items, world)
    return list(range(min(n_items, rank * per), min(n_items, (rank + 1) * per)))


def shard_size(n_items: int, world: int) -> int:
    """Sets per rank in the candidate exchange: every rank sends ceil(n / world) (padding count 0)."""
    return max(1, (n_items + world - 1) // world)


def learning_rates(it: int, iters: int = 100, rows: int = 14, sh_linear: bool = True) -> list[float]:
    """Per-row Adam learning rates at iteration `it`. With 23 rows (degree-1 SH)
    the DC coefficients take the colour rate; the first-order coefficients (rows 14-22) take it only
    when `sh_linear` ("first-order coefficients of spherical harmonics coefficients are only
    optimized in bundle adjustment"), else 0."""
    t = min(max(it, 0) / max(iters, 1), 1.0)
    lr_x = 1.6e-5 * (1.7e-7 / 1.6e-5) ** t
    lr = [lr_x] * 3 + [2e-4] * 3 + [4e-5] * 4 + [1e-2] + [5e-4] * 3
    if rows > 14:
        lr += [5e-4 if sh_linear else 0.0] * (rows - 14)
    return lr


def _dist_on(group=None) -> bool:
    return dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1


def allreduce_grads(grad: torch.Tensor, n: int | None = None, group=None, packed: torch.Tensor | None = None) -> None:
    """Sum the gradient buffer [rows][ld] over ranks in place, only its first n columns (the live
    Gaussians). The live block is packed into one contiguous buffer (rows x n, `packed` if given, of at
    least that size) and reduced with ONE all_reduce (NCCL on GPU, gloo on CPU or CUDA tensors), then
    copied back: 2 x 56 n bytes of HBM copies instead of 14 collective launches or reducing the unused
    capacity columns."""
    if not _dist_on(group):
        return
    n = grad.shape[1] if n is None else n
    if n == grad.shape[1] or grad.dim() == 1:
        dist.all_reduce(grad, op=dist.ReduceOp.SUM, group=group)
        return
    rows = grad.shape[0]
    if packed is None or packed.numel() < rows * n:
        packed = torch.empty(rows * n, dtype=grad.dtype, device=grad.device)
    buf = packed[:rows * n].view(rows, n)
    buf.copy_(grad[:, :n])
    dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    grad[:, :n].copy_(buf)


def column_chunks(n: int, chunks: int, align: int = 32) -> list[tuple[int, int]]:
    """[0, n) split into <= chunks column ranges whose starts are multiples of `align` (16-byte aligned
    rows for the Adam kernel's vector path)."""
    if n <= 0:
        return []
    w = max(align, -(-((n + chunks - 1) // chunks) // align) * align)
    return [(c0, min(n, c0 + w)) for c0 in range(0, n, w)]


def allreduce_adam(grad: torch.Tensor, n: int, adam, group=None, packed: torch.Tensor | None = None,
                   chunks: int = 4) -> None:
    """The gradient exchange overlapped with the optimiser (bucketed overlap): the
    live columns [0, n) in `chunks` column ranges; each range is packed into its own slice of `packed`
    and its sum all_reduce issued asynchronously (the collectives run in issue order on the
    communicator's stream), then, range by range, the step waits for that range's reduction, copies
    it back and runs adam(c0, c1) on those columns while the next ranges are still being reduced.
    Adam is per column, so the result is the reduction followed by one Adam step over [0, n). One
    rank: adam(0, n)."""
    if not _dist_on(group):
        if n > 0:
            adam(0, n)
        return
    rows = grad.shape[0]
    if packed is None or packed.numel() < rows * n:
        packed = torch.empty(rows * n, dtype=grad.dtype, device=grad.device)
    pending, off = [], 0
    for c0, c1 in column_chunks(n, chunks):
        buf = packed[off:off + rows * (c1 - c0)].view(rows, c1 - c0)
        off += rows * (c1 - c0)
        buf.copy_(grad[:, c0:c1])
        pending.append((c0, c1, buf, dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group, async_op=True)))
    for c0, c1, buf, work in pending:
        work.wait()
        grad[:, c0:c1].copy_(buf)
        adam(c0, c1)


def allreduce_sum(t: torch.Tensor, group=None) -> None:
    """Plain sum all-reduce (densification statistics, reading C30: summed over ranks before the
    split/clone decision so every rank decides on the same values)."""
    if _dist_on(group):
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)


def allreduce_mask(mask: torch.Tensor, group=None) -> None:
    """OR of per-rank u8 flag masks (max all-reduce), so every rank applies the same Eq. 9 set."""
    if _dist_on(group):
        dist.all_reduce(mask, op=dist.ReduceOp.MAX, group=group)


def gather_candidates(cand: torch.Tensor, counts: torch.Tensor, group=None):
    """all_gather of per-rank candidate sets cand[S][rows][max_add] and counts[S] -> rank-ordered
    [R*S][rows][max_add], [R*S]. Every rank sends the same S = shard_size(keyframes, R) sets (the
    unused ones with count 0), so uneven shards exchange equal-sized buffers; with contiguous shards
    the rank order is the global keyframe order."""
    if not _dist_on(group):
        return cand, counts
    world = dist.get_world_size(group)
    dev = cand.device
    if cand.is_cuda and dist.get_backend(group) != "nccl":   # gloo gathers host tensors
        cand, counts = cand.cpu(), counts.cpu()
    cs = [torch.empty_like(counts) for _ in range(world)]
    dist.all_gather(cs, counts, group=group)
    xs = [torch.empty_like(cand) for _ in range(world)]
    dist.all_gather(xs, cand, group=group)
    return torch.cat(xs, 0).to(dev), torch.cat(cs, 0).to(dev)


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
    fixed: bool = False     # pose held fixed in bundle adjustment (the SLAM's first keyframe)


@dataclasses.dataclass(frozen=True)
class SplitClone:
    """Split/clone densification schedule and thresholds (reading C30): every `every`
    iterations before `until`, Gaussians whose mean NDC mean-gradient norm since the last decision
    is >= grad_thresh are cloned (max scale <= scale_thresh) or split."""
    every: int = 10
    until: int = 70
    grad_thresh: float = 0.002
    scale_thresh: float = 0.02
    seed: int = 0           # the split noise: same generator and seed on every rank


class ShardedMapper:
    """Mapping over a keyframe set, sharded by keyframe across the ranks of `group` (one per GPU).

    step() = one mapping iteration: render + L1 + backward of the local keyframes into grad, the
    exchange (all-reduce of grad[:, :n]), the Adam step (identical on every rank), then, when
    `densify`, the Eq. 8 expansion (candidates all-gathered in keyframe order, appended) and the
    opacity prune; on the split/clone schedule the densification statistics are summed over ranks
    and the split/clone decision taken identically everywhere. The map size n lives on the device
    (n_dev); the host reads it (with the key-capacity flag) only after a step that changed it, so a
    step without densification has no host synchronisation."""

    def __init__(self, params: torch.Tensor, n: int, keyframes: list[Keyframe], cam, key_cap: int,
                 max_add_per_kf: int = 8192, w_color: float = 0.9, w_depth: float = 0.1, group=None,
                 densify: bool = True, ba_iters: int | None = None, lr_rho: float = 1e-3, lr_phi: float = 1e-3,
                 degenerate: tuple[float, float] | None = None, split_clone: SplitClone | None = None,
                 iters: int = 100, pipelines: int = 2):
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
        self.packed = torch.empty(params.numel(), device=params.device) if self.world > 1 else None
        self.exchange_chunks = 4   # gradient buckets overlapped with Adam (allreduce_adam)
        self.n = n
        self.n_dev = torch.tensor([n], dtype=torch.int64, device=params.device)
        self.cam = cam
        self.cm = make_camera(cam)
        # `pipelines` render workspaces on as many streams: keyframe j renders on pipeline j % count,
        # so one keyframe's projection, binning and forward overlap the previous keyframe's backward
        # (the backward chains stay in keyframe order: render_backward)
        self.pipes = [RenderPipeline(self.cap, key_cap, cam.width, cam.height, params.device)
                      for _ in range(max(1, pipelines))]
        self.pipe = self.pipes[0]
        self.side = [torch.cuda.Stream(device=params.device) for _ in self.pipes[1:]]
        self.w_color, self.w_depth = w_color, w_depth
        self.max_add = max_add_per_kf
        self.densify = densify
        self.iters = iters          # length of the learning-rate schedule (100)
        self.it = 0                 # schedule position (reset per keyframe window by the SLAM driver)
        self.adam_t = 0             # Adam's step count: monotone, never reset with the schedule
        self.ba_iters = ba_iters
        self.lr_rho, self.lr_phi = lr_rho, lr_phi
        self.pose_step = 0
        # Eq. 9 opacity degeneration (NEXT-2, reading C27) in expansion steps: (eta, gamma)
        self.degenerate = degenerate
        self.dmask = torch.zeros(self.cap, dtype=torch.uint8, device=params.device) if degenerate else None
        self.split = split_clone
        if split_clone is not None:
            self.acc = torch.zeros(self.cap, device=params.device)
            self.cnt = torch.zeros(self.cap, device=params.device)
            self.noise = torch.zeros(6, self.cap, device=params.device)
            self.gen = torch.Generator(device=params.device)
        self.splits_done = 0
        self.split_log: list | None = None   # set to [] to record each split/clone decision's inputs
        self.key_cap = key_cap
        # the workspaces' key-capacity flags are reset by every gs_bin_sort: OR them over the renders
        # here (one accumulator per pipeline: each is written from its own stream)
        self.err_flags = [pp.arrays(0)["error_flag"] for pp in self.pipes]
        self.err_acc = torch.zeros(len(self.pipes), dtype=torch.int32, device=params.device)
        self.cand = None
        self.set_keyframes(keyframes)

    def set_keyframes(self, keyframes: list[Keyframe]):
        """(Re)assign the keyframe set (the SLAM driver's window, slam.py). Candidate buffers hold
        shard_size sets on every rank; the keyframe poses' Adam state starts afresh (it belongs to a
        keyframe, and the window's keyframes change)."""
        dev = self.P.device
        self.keyframes = keyframes
        self.local = shard(len(keyframes), self.world, self.rank)
        S = shard_size(len(keyframes), self.world)
        if self.cand is None or self.cand.shape[0] != S:
            self.cand = torch.zeros(S, self.rows, self.max_add, device=dev)
            self.counts = torch.zeros(S, dtype=torch.int64, device=dev)
            self.gpose = torch.zeros(S, 6, dtype=torch.float64, device=dev)
            self.pm = torch.zeros(S, 6, device=dev)
            self.pv = torch.zeros(S, 6, device=dev)
        self.counts.zero_()
        self.pm.zero_()
        self.pv.zero_()
        self.pose_step = 0

    def poses_active(self) -> bool:
        """Eq. 13: poses are optimised only in the second half of the BA iterations."""
        return self.ba_iters is not None and self.it >= self.ba_iters // 2

    def split_due(self) -> bool:
        """Split/clone after iteration `it` (1-based count) every `every` iterations before `until`."""
        s = self.split
        return s is not None and self.it % s.every == 0 and self.it < s.until

    def render_backward(self):
        """fwd + L1 + bwd for every local keyframe, accumulating into grad.
        Keyframe j runs on pipeline / stream j % len(pipes); its backward is split in two
        (GS_FLAG_BWD_SCREEN_ONLY / _CHAIN_ONLY): the tile pass runs at once, the per-Gaussian chain
        (and the split/clone statistics) waits for keyframe j-1's chain, so the chains accumulate into
        grad in keyframe order as with one pipeline (no two touch grad at once), while the next
        keyframe's projection, binning, forward and tile pass overlap. (The tile pass's screen-gradient atomics already make two
        runs differ in the last bits, with one pipeline or two.)"""
        self.grad[:, :self.n].zero_()
        degen = self.degenerate is not None and self.densify
        if degen:
            self.dmask.zero_()
        cur = torch.cuda.current_stream(self.P.device)
        streams = [cur] + self.side
        for st in self.side:
            st.wait_stream(cur)
        prev = None   # event: the previous keyframe's backward chain is done
        for j, k in enumerate(self.local):
            q = j % len(streams)
            pipe, st = self.pipes[q], streams[q]
            kf = self.keyframes[k]
            with torch.cuda.stream(st):
                pipe.forward(self.P, self.n, kf.view, self.cam, bin_flags=GS_FLAG_NO_HOST_SYNC, fwd_flags=0)
                torch.bitwise_or(self.err_acc[q:q + 1], self.err_flags[q], out=self.err_acc[q:q + 1])
                if degen:   # Eq. 9 flags from this keyframe's projection, ORed over the local keyframes
                    gs_densify_prune(None, None, self.n_dev, self.n, self.cap, None, None, None, None, None, kf.depth,
                                     None, kf.view, self.cm, densify_cfg(GS_DENSIFY_DEGENERATE_FLAG,
                                                                         gamma=self.degenerate[1]),
                                     self.dmask, None, pipe.ws)
                gp = None
                if self.poses_active():
                    gp = self.gpose[j]
                    gp.zero_()
                # L1 (Eq. 6) formed inside the backward's pixel loads (gs_render_bwd_l1): no dL/dC, dL/dD
                # images. The tile pass (screen gradients, in this pipeline's workspace) runs at once; the
                # per-Gaussian chain, which accumulates into grad, waits for the previous keyframe's
                color, depth, _ = pipe._imgs(self.cam)
                args = (self.P, self.n, self.P.shape[1], kf.view, pipe.ws, self.cm, color, depth, kf.color, kf.depth,
                        self.w_color, self.w_depth, self.grad, gp, pipe.loss)
                gs_render_bwd_l1(*args, GS_FLAG_POSE_COV_PATH | GS_FLAG_BWD_SCREEN_ONLY)
                if prev is not None:
                    st.wait_event(prev)
                gs_render_bwd_l1(*args, GS_FLAG_POSE_COV_PATH | GS_FLAG_BWD_CHAIN_ONLY)
                if self.split is not None:   # reading C30 statistics of this view (NDC mean-gradient norm)
                    gs_densify_accum_grad(pipe.ws, self.acc, self.cnt)
                prev = torch.cuda.Event()
                prev.record(st)
                if self.densify:   # Eq. 8 candidates from this keyframe's render (gather mode)
                    cnt = self.counts[j:j + 1]
                    gs_densify_prune(self.P, None, cnt, self.cap, self.cap, None, None, pipe.alpha, pipe.depth,
                                     kf.color, kf.depth, None, kf.view, self.cm,
                                     densify_cfg(GS_DENSIFY_ADD, max_add=self.max_add, rows=self.rows), None,
                                     self.cand[j], pipe.ws)
        for st in self.side:
            cur.wait_stream(st)

    def step(self):
        poses = self.poses_active()
        self.render_backward()
        if self.degenerate is not None and self.densify:   # one Eq. 9 application per expansion step
            allreduce_mask(self.dmask, self.group)
            gs_densify_prune(self.P, self.raw, self.n_dev, self.n, self.cap, None, None, None, None, None, None,
                             None, None, None, densify_cfg(GS_DENSIFY_DEGENERATE_APPLY, eta=self.degenerate[0]),
                             self.dmask, None, self.pipe.ws)
        if poses:   # each rank updates the poses of its own keyframes (device-only pose step)
            self.pose_step += 1
            for j, k in enumerate(self.local):
                if self.keyframes[k].fixed:
                    continue
                gs_pose_step(self.keyframes[k].view, self.gpose[j], self.pm[j], self.pv[j], self.pose_step,
                             self.lr_rho, self.lr_phi)
        self.it += 1
        self.adam_t += 1
        lr = learning_rates(self.it - 1, self.iters, rows=self.rows, sh_linear=self.ba_iters is not None)

        def adam(c0: int, c1: int):   # columns [c0, c1): pointers offset by c0, the same row stride
            a = (self.raw[:, c0:], self.P[:, c0:], self.grad[:, c0:], self.m[:, c0:], self.v[:, c0:], c1 - c0,
                 self.cap)
            if self.rows == 14:
                gs_adam_step(*a, lr, self.adam_t)
            else:
                gs_adam_step_rows(*a, self.rows, lr, self.adam_t)
        # all-reduce of grad[:, :n] in column buckets, each bucket's Adam step overlapping the next
        # buckets' reductions (the Eq. 9 degeneration and the pose steps above read no map gradient)
        allreduce_adam(self.grad, self.n, adam, self.group, self.packed, self.exchange_chunks)
        changed = False
        if self.split_due():
            # statistics summed over ranks before the decision: identical splits and clones everywhere
            allreduce_sum(self.acc[:self.n], self.group)
            allreduce_sum(self.cnt[:self.n], self.group)
            self.gen.manual_seed(self.split.seed * 1000003 + self.adam_t)
            torch.randn(6, self.cap, generator=self.gen, device=self.P.device, out=self.noise)
            if self.split_log is not None:   # inspection (tests): the decision's inputs
                n0 = self.n
                self.split_log.append([self.P[:, :n0].clone(), self.acc[:n0].clone(), self.cnt[:n0].clone(),
                                       self.noise[:, :n0].clone()])
            gs_densify_split_clone(self.P, self.raw, self.m, self.v, self.n_dev, self.cap, self.cap, self.acc,
                                   self.cnt, self.noise, self.split.grad_thresh, self.split.scale_thresh,
                                   self.pipe.ws, rows=self.rows)
            if self.split_log is not None:
                self.split_log[-1].append(self.P[:, :self.cap].clone())
                self.split_log[-1].append(self.n_dev.clone())
            self.splits_done += 1
            changed = True
        if self.densify:
            cand, counts = gather_candidates(self.cand, self.counts, self.group)
            gs_densify_append(self.P, self.raw, self.m, self.v, self.n_dev, self.cap, self.cap, cand, counts,
                              cand.shape[0], self.max_add, rows=self.rows)
            gs_densify_prune(self.P, self.raw, self.n_dev, self.cap, self.cap, self.m, self.v, None, None, None, None,
                             None, None, None, densify_cfg(GS_DENSIFY_PRUNE, rows=self.rows), None, None, self.pipe.ws)
            if self.split is not None:   # the prune compacts columns: statistics restart with it
                self.acc.zero_()
                self.cnt.zero_()
            changed = True
        if changed:
            self.sync()
        return self.n

    def sync(self) -> int:
        """One host read: the map size after densification and the workspace's key-capacity flag
        (a NO_HOST_SYNC render that overflowed its key capacity produced no lists; raise)."""
        both = torch.stack([self.n_dev[0], self.err_acc.max().to(torch.int64)]).cpu()
        self.n = int(both[0])
        if int(both[1]) != 0:
            raise RuntimeError(f"key capacity overflow in a mapping render (key_cap {self.key_cap}); raise key_cap")
        return self.n
