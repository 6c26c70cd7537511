"""Coarse-to-fine camera tracking (Alg. 1; Eq. 10-12).

Every step runs in libgs kernels; this module only sequences the calls:
  coarse stage  T_c x [ gs_project (H/2 x W/2) -> gs_bin_sort -> gs_render_fwd
                        -> gs_pose_grad_l1 (Eq. 6 fused into the pose-only pass) -> gs_pose_step ]
  selection     gs_render_fwd (full res, GS_FLAG_ACCUM_WEIGHT) -> gs_densify_prune(SELECT)  (Eq. 12)
  fine stage    T_f x [ same at full resolution, gs_project with the selection mask ]
The pose lives on the device (world->camera 3x4) and is updated in place; no host sync inside
the loops (bin_sort runs in GS_FLAG_NO_HOST_SYNC mode). Readings: C12 (half-resolution camera),
C23 (loss and twist learning rate), C24 (selection rule) of DESIGN.md §3.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np
import torch

from . import (GS_DENSIFY_SELECT, GS_FLAG_ACCUM_WEIGHT, GS_FLAG_GRAD_ASSIGN, GS_FLAG_NO_HOST_SYNC,
               GS_FLAG_POSE_COV_PATH, densify_cfg,
               gs_densify_prune, gs_frame_stats, gs_loss_l1_masked, gs_pose_extrapolate, gs_pose_step, make_camera)
from .pipeline import RenderPipeline


@dataclasses.dataclass
class TrackConfig:
    iters_coarse: int = 50
    iters_fine: int = 50
    lr_rho: float = 1e-3
    lr_phi: float = 1e-3
    w_color: float = 0.9
    w_depth: float = 0.1
    sel_weight: float = 0.5
    sel_depth: float = 0.05
    pose_flags: int = GS_FLAG_POSE_COV_PATH
    observed_alpha: float | None = None   # NEXT-4 / reading C31: loss only where the render's alpha >= this
    outlier_k: float = 0.0                # reading C32: drop pixels whose loss > k x median; 0 = off


class Tracker:
    def __init__(self, n_cap: int, key_cap_full: int, key_cap_half: int, cam_full, device="cuda"):
        self.cam_full = cam_full
        self.cam_half = cam_full.half()
        self.full = RenderPipeline(n_cap, key_cap_full, cam_full.width, cam_full.height, device)
        self.half = RenderPipeline(n_cap, key_cap_half, self.cam_half.width, self.cam_half.height, device)
        dev = torch.device(device)
        self.grad_pose = torch.zeros(6, dtype=torch.float64, device=dev)
        self.m6 = torch.zeros(6, dtype=torch.float32, device=dev)
        self.v6 = torch.zeros(6, dtype=torch.float32, device=dev)
        self.mask = torch.zeros(n_cap, dtype=torch.uint8, device=dev)
        self.accum = torch.zeros(n_cap, dtype=torch.float32, device=dev)
        self.n_dev = torch.zeros(1, dtype=torch.int64, device=dev)
        self.step = 0
        self.graphs: dict = {}   # track(graph=True): captured stages per (buffers, n, cfg)

    def reset(self):
        self.m6.zero_()
        self.v6.zero_()
        self.step = 0

    def _iter(self, pipe, cam, P, n, V, tc, td, cfg: TrackConfig, mask=None):
        pipe.forward(P, n, V, cam, mask=mask, bin_flags=GS_FLAG_NO_HOST_SYNC, fwd_flags=0)
        if cfg.observed_alpha is None and cfg.outlier_k == 0:
            # Eq. 6 L1 fused into the pose-only pass (gs_pose_grad_l1): the gradient is assigned
            pipe.pose_grad_l1(P, n, V, cam, tc, td, self.grad_pose, cfg.w_color, cfg.w_depth,
                              flags=cfg.pose_flags | GS_FLAG_GRAD_ASSIGN)
        else:   # "only rendered at previously observed areas"
            color, depth, alpha = pipe._imgs(cam)
            npx = cam.width * cam.height
            dc = pipe.dL_dcolor.view(-1)[:3 * npx].view(3, cam.height, cam.width)
            dd = pipe.dL_ddepth.view(-1)[:npx].view(cam.height, cam.width)
            amin = cfg.observed_alpha if cfg.observed_alpha is not None else float("-inf")
            gs_loss_l1_masked(color, depth, tc, td, alpha, amin, cfg.outlier_k, cam.width, cam.height, cfg.w_color,
                              cfg.w_depth, dc, dd, pipe.loss, pipe.ws)
            pipe.pose_grad(P, n, V, cam, dc, dd, self.grad_pose, flags=cfg.pose_flags | GS_FLAG_GRAD_ASSIGN)
        self.step += 1
        gs_pose_step(V, self.grad_pose, self.m6, self.v6, self.step, cfg.lr_rho, cfg.lr_phi)

    def coarse_iter(self, P, n, V, tc_half, td_half, cfg: TrackConfig):
        self._iter(self.half, self.cam_half, P, n, V, tc_half, td_half, cfg)

    def select(self, P, n, V, td_full, cfg: TrackConfig):
        """Eq. 12 with reading C24: accumulated alpha*T > sel_weight and |D* - d| < sel_depth."""
        self.accum[:n].zero_()
        self.full.forward(P, n, V, self.cam_full, bin_flags=GS_FLAG_NO_HOST_SYNC, fwd_flags=GS_FLAG_ACCUM_WEIGHT,
                          accum_weight=self.accum)
        self.n_dev.fill_(n)
        gs_densify_prune(P, None, self.n_dev, n, P.shape[1], None, None, None, None, None, td_full, self.accum, V,
                         make_camera(self.cam_full),
                         densify_cfg(GS_DENSIFY_SELECT, sel_weight=cfg.sel_weight, sel_depth=cfg.sel_depth),
                         self.mask, None, self.full.ws)
        return self.mask[:n]

    def fine_iter(self, P, n, V, tc_full, td_full, cfg: TrackConfig):
        self._iter(self.full, self.cam_full, P, n, V, tc_full, td_full, cfg, mask=self.mask)

    def coarse_stage(self, P, n, V, tc_half, td_half, cfg: TrackConfig):
        self.reset()
        for _ in range(cfg.iters_coarse):
            self.coarse_iter(P, n, V, tc_half, td_half, cfg)

    def fine_stage(self, P, n, V, td_full, tc_full, cfg: TrackConfig):
        self.select(P, n, V, td_full, cfg)
        for _ in range(cfg.iters_fine):
            self.fine_iter(P, n, V, tc_full, td_full, cfg)

    def stage_graphs(self, P, n, V, tc_half, td_half, tc_full, td_full, cfg: TrackConfig):
        """The two stages of Alg. 1 captured as CUDA graphs (every call is device-only in
        GS_FLAG_NO_HOST_SYNC mode; the Adam step counts are baked in, and reset() is part of the coarse
        graph, so a replay repeats the same schedule). Cached per (buffer addresses, n, cfg): replaying
        reads the CURRENT contents of P, V and the targets, so a caller refills those buffers and
        replays. The first call runs both stages once eagerly (warm-up) and restores V."""
        key = (P.data_ptr(), n, V.data_ptr(), tc_half.data_ptr(), td_half.data_ptr(), tc_full.data_ptr(),
               td_full.data_ptr(), dataclasses.astuple(cfg))
        gr = self.graphs.get(key)
        if gr is None:
            V0 = V.clone()
            self.coarse_stage(P, n, V, tc_half, td_half, cfg)
            self.fine_stage(P, n, V, td_full, tc_full, cfg)
            V.copy_(V0)
            torch.cuda.synchronize()
            gr = (torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph())
            with torch.cuda.graph(gr[0]):
                self.coarse_stage(P, n, V, tc_half, td_half, cfg)
            with torch.cuda.graph(gr[1]):
                self.fine_stage(P, n, V, td_full, tc_full, cfg)
            self.graphs[key] = gr
        return gr

    def track(self, P, n, V, tc_half, td_half, tc_full, td_full, cfg: TrackConfig = TrackConfig(), graph=False):
        """Alg. 1: T_c coarse iterations, selection, T_f fine iterations. Updates V in place. graph:
        replay the captured stages (stage_graphs) instead of issuing ~10 library calls per iteration
        from Python."""
        if graph:
            g_coarse, g_fine = self.stage_graphs(P, n, V, tc_half, td_half, tc_full, td_full, cfg)
            g_coarse.replay()
            g_fine.replay()
            return V
        self.coarse_stage(P, n, V, tc_half, td_half, cfg)
        self.fine_stage(P, n, V, td_full, tc_full, cfg)
        return V


@dataclasses.dataclass
class FrontendConfig:
    track: TrackConfig = dataclasses.field(default_factory=lambda: TrackConfig(observed_alpha=0.5, outlier_k=10.0))
    kf_reliable: float = 0.7     # keyframe when the reliable share of valid pixels drops below this
    kf_max_gap: int = 30         # ... or this many frames after the last keyframe (mu_k)
    tau_alpha: float = 0.5       # Eq. 8 thresholds for "reliable"
    tau_depth: float = 0.10


class Frontend:
    """Tracking front end: constant-velocity pose
    initialisation (gs_pose_extrapolate), coarse-to-fine tracking on previously observed areas
    with the 10x-median pixel rejection (gs_loss_l1_masked, readings C31-C32), and the keyframe rule (gs_frame_stats: reliable share of the observed
    image, or a maximum frame gap). One host read per frame (the keyframe decision)."""

    def __init__(self, tracker: Tracker, cfg: FrontendConfig = FrontendConfig()):
        self.tr = tracker
        self.cfg = cfg
        self.poses: list[torch.Tensor] = []
        self.since_kf = 0
        self.counts = torch.zeros(3, dtype=torch.int32, device=tracker.grad_pose.device)

    def initial_pose(self) -> torch.Tensor:
        """Constant velocity from the last two poses (or the last one)."""
        V = torch.empty(3, 4, dtype=torch.float32, device=self.counts.device)
        if len(self.poses) >= 2:
            gs_pose_extrapolate(self.poses[-2], self.poses[-1], V)
        else:
            V.copy_(self.poses[-1])
        return V

    def add_pose(self, V: torch.Tensor, keyframe: bool = True):
        self.poses.append(V.clone())
        self.since_kf = 0 if keyframe else self.since_kf + 1

    def track_frame(self, P, n, tc_half, td_half, tc_full, td_full) -> tuple[torch.Tensor, bool, float]:
        """Track one frame from the constant-velocity guess; returns (pose, keyframe?, reliable share)."""
        V = self.initial_pose()
        self.tr.track(P, n, V, tc_half, td_half, tc_full, td_full, self.cfg.track)
        cam = self.tr.cam_full
        fr = self.tr.full.forward(P, n, V, cam, bin_flags=GS_FLAG_NO_HOST_SYNC, fwd_flags=0)
        gs_frame_stats(fr.alpha, fr.depth, td_full, cam.width, cam.height, self.cfg.tau_alpha, self.cfg.tau_depth,
                       self.counts)
        rel, valid, _ = (int(x) for x in self.counts.cpu().tolist())
        share = rel / max(valid, 1)
        keyframe = share < self.cfg.kf_reliable or self.since_kf + 1 >= self.cfg.kf_max_gap
        self.add_pose(V, keyframe)
        return V, keyframe, share


def pose_error(view, view_gt) -> tuple[float, float]:
    """(camera-centre distance in metres, rotation angle in degrees) between two world->camera poses."""
    a = np.asarray(view, np.float64)
    b = np.asarray(view_gt, np.float64)
    ca = -a[:, :3].T @ a[:, 3]
    cb = -b[:, :3].T @ b[:, 3]
    dr = a[:, :3] @ b[:, :3].T
    s = 0.5 * np.linalg.norm([dr[2, 1] - dr[1, 2], dr[0, 2] - dr[2, 0], dr[1, 0] - dr[0, 1]])
    c = 0.5 * (np.trace(dr) - 1.0)
    ang = math.degrees(math.atan2(s, c))   # accurate for small angles, unlike acos
    return float(np.linalg.norm(ca - cb)), ang
