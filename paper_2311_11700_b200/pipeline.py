"""Convenience layer: one render iteration (gs_project + gs_bin_sort +
gs_render_fwd + gs_loss_l1 + gs_render_bwd) over caller-owned torch CUDA tensors.
Argument marshalling only; every step is a libgs call."""
from __future__ import annotations

import dataclasses

import torch

from . import (GS_FLAG_EXAMINED, GS_FLAG_GRAD_ASSIGN, GS_FLAG_POSE_COV_PATH, Workspace, gs_bin_sort, gs_loss_l1, gs_pose_grad,
               gs_pose_grad_l1, gs_project_ex, gs_render_bwd, gs_render_bwd_l1, gs_render_fwd, make_camera)


@dataclasses.dataclass
class Frame:
    color: torch.Tensor     # [3][H][W]
    depth: torch.Tensor     # [H][W]
    alpha: torch.Tensor     # [H][W]
    n_keys: int


class RenderPipeline:
    """Owns a workspace and the image / upstream-gradient buffers for one camera size."""

    def __init__(self, n_cap: int, key_cap: int, width: int, height: int, device="cuda"):
        self.ws = Workspace(n_cap, key_cap, width, height, device)
        self.device = torch.device(device)
        self.width, self.height = width, height
        f32 = dict(dtype=torch.float32, device=self.device)
        self.color = torch.zeros(3, height, width, **f32)
        self.depth = torch.zeros(height, width, **f32)
        self.alpha = torch.zeros(height, width, **f32)
        self.dL_dcolor = torch.zeros(3, height, width, **f32)
        self.dL_ddepth = torch.zeros(height, width, **f32)
        self.loss = torch.zeros(1, dtype=torch.float64, device=self.device)
        self.n_keys = -1

    def _imgs(self, cam):
        h, w = cam.height, cam.width
        if (h, w) == (self.height, self.width):
            return self.color, self.depth, self.alpha
        npx = h * w
        return (self.color.view(-1)[:3 * npx].view(3, h, w), self.depth.view(-1)[:npx].view(h, w),
                self.alpha.view(-1)[:npx].view(h, w))

    def forward(self, params, n, viewmat, cam, mask=None, bin_flags=0, fwd_flags=GS_FLAG_EXAMINED,
                accum_weight=None, stream=None, proj_flags=0) -> Frame:
        """params [14][ld] (RGB) or [23][ld] (degree-1 SH, gs_project_sh); proj_flags: gs_project_ex
        flags (GS_FLAG_OPACITY_RADIUS)."""
        c = make_camera(cam)
        ld = params.shape[1]
        sh = {14: 0, 23: 1}[params.shape[0]]
        gs_project_ex(params, n, ld, sh, proj_flags, mask, viewmat, c, self.ws, stream)
        self.n_keys = gs_bin_sort(self.ws, bin_flags, stream)
        color, depth, alpha = self._imgs(cam)
        gs_render_fwd(self.ws, c, color, depth, alpha, accum_weight, fwd_flags, stream)
        return Frame(color, depth, alpha, self.n_keys)

    def loss_l1(self, cam, tgt_color, tgt_depth, w_color=0.9, w_depth=0.1, stream=None):
        color, depth, _ = self._imgs(cam)
        npx = cam.width * cam.height
        dc = self.dL_dcolor.view(-1)[:3 * npx].view(3, cam.height, cam.width)
        dd = self.dL_ddepth.view(-1)[:npx].view(cam.height, cam.width)
        gs_loss_l1(color, depth, tgt_color, tgt_depth, cam.width, cam.height, w_color, w_depth, dc, dd, self.loss,
                   self.ws, stream)
        return dc, dd

    def backward(self, params, n, viewmat, cam, dL_dcolor, dL_ddepth, grad_params, grad_pose=None,
                 flags=GS_FLAG_POSE_COV_PATH, stream=None):
        gs_render_bwd(params, n, params.shape[1], viewmat, self.ws, make_camera(cam), dL_dcolor, dL_ddepth, grad_params,
                      grad_pose, flags, stream)

    def pose_grad(self, params, n, viewmat, cam, dL_dcolor, dL_ddepth, grad_pose, flags=GS_FLAG_POSE_COV_PATH,
                  stream=None):
        gs_pose_grad(params, n, params.shape[1], viewmat, self.ws, make_camera(cam), dL_dcolor, dL_ddepth, grad_pose,
                     flags, stream)

    def pose_grad_l1(self, params, n, viewmat, cam, tgt_color, tgt_depth, grad_pose, w_color=0.9, w_depth=0.1,
                     flags=GS_FLAG_POSE_COV_PATH, stream=None):
        """gs_pose_grad_l1: the L1 loss of the last forward's images fused into the pose pass; self.loss
        receives L."""
        color, depth, _ = self._imgs(cam)
        gs_pose_grad_l1(params, n, params.shape[1], viewmat, self.ws, make_camera(cam), color, depth, tgt_color,
                        tgt_depth, w_color, w_depth, grad_pose, self.loss, flags, stream)

    def iteration(self, params, n, viewmat, cam, tgt_color, tgt_depth, grad_params, grad_pose=None, bin_flags=0,
                  fwd_flags=0, w_color=0.9, w_depth=0.1, stream=None, assign_grads=False, fused_loss=False,
                  proj_flags=0):
        """The headline fwd+bwd iteration. assign_grads: the gradients overwrite
        grad_params[:, :n] / grad_pose (GS_FLAG_GRAD_ASSIGN) instead of accumulating into them.
        fused_loss: gs_render_bwd_l1 (the L1 loss formed in the backward's pixel loads; dL/dC and
        dL/dD are not materialised) instead of gs_loss_l1 + gs_render_bwd. self.loss receives L."""
        self.forward(params, n, viewmat, cam, bin_flags=bin_flags, fwd_flags=fwd_flags, stream=stream,
                     proj_flags=proj_flags)
        flags = GS_FLAG_POSE_COV_PATH | (GS_FLAG_GRAD_ASSIGN if assign_grads else 0)
        if fused_loss:
            color, depth, _ = self._imgs(cam)
            gs_render_bwd_l1(params, n, params.shape[1], viewmat, self.ws, make_camera(cam), color, depth, tgt_color,
                             tgt_depth, w_color, w_depth, grad_params, grad_pose, self.loss, flags, stream)
            return
        dc, dd = self.loss_l1(cam, tgt_color, tgt_depth, w_color, w_depth, stream)
        self.backward(params, n, viewmat, cam, dc, dd, grad_params, grad_pose, flags=flags, stream=stream)

    # ------------------------------------------------------------------ introspection (tests, bench)
    def arrays(self, n: int | None = None, n_keys: int | None = None) -> dict:
        v = self.ws.view()
        n = v.n if n is None else n
        K = self.n_keys if n_keys is None else n_keys
        npx = v.width * v.height
        ntiles = v.grid_x * v.grid_y
        t = self.ws.tensor
        out = dict(records=t(v.records, n * 12, torch.float32).view(n, 12),
                   depth_key=t(v.depth_key, n, torch.int32), rect=t(v.rect, n * 4, torch.int16).view(n, 4),
                   radius=t(v.radius, n, torch.int32), tiles=t(v.tiles, n, torch.int32),
                   offsets=t(v.offsets, n, torch.int32),
                   ranges=t(v.ranges, ntiles * 2, torch.int32).view(ntiles, 2),
                   t_final=t(v.t_final, npx, torch.float32).view(v.height, v.width),
                   n_last=t(v.n_last, npx, torch.int32).view(v.height, v.width),
                   examined=t(v.examined, npx, torch.int32).view(v.height, v.width),
                   n_keys_dev=t(v.n_keys_dev, 1, torch.int64), error_flag=t(v.error_flag, 1, torch.int32),
                   live_cnt=t(v.live_cnt, ntiles, torch.int32))
        if K is not None and K >= 0:
            if v.keys:   # path A only (path B never materialises the 64-bit keys)
                out["keys"] = t(v.keys, K, torch.int64)
            out["vals"] = t(v.vals, K, torch.int32)
            out["live_g"] = t(v.live_g, K, torch.int32)
            out["live_j"] = t(v.live_j, K, torch.int32)
        return out
