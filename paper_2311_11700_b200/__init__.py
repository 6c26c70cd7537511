"""B200-native differentiable RGB-D Gaussian-splatting renderer (GS-SLAM hot path, arXiv 2311.11700).

Thin ctypes binding over the C ABI of `libgs.so` (include/gs.h): argument marshalling only —
every step of the path runs in the library's sm_100a kernels. PyTorch supplies device memory,
streams and process groups. There is no CPU fallback: importing this package fails loudly if the
library is missing.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# GS_DEBUG=1 loads the debug build (output invariant checks after every stage, csrc/debug.cu)
DEBUG = os.environ.get("GS_DEBUG", "0") == "1"
LIB_PATH = os.path.join(_HERE, "libgs_debug.so" if DEBUG else "libgs.so")
# GS_LIB: an explicit library path (A/B experiments, tools/variant_build.py)
LIB_PATH = os.environ.get("GS_LIB") or LIB_PATH

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{os.path.basename(LIB_PATH)} not built at {LIB_PATH}: run `python -m paper_2311_11700_b200.build` "
                      "(or __graft_entry__.build()); there is no fallback path")

_lib = ctypes.CDLL(LIB_PATH)

# ----------------------------------------------------------------------------------- types
GS_OK, GS_ERR_INVALID_ARG, GS_ERR_CAPACITY, GS_ERR_STALE, GS_ERR_CUDA, GS_ERR_UNSUPPORTED = range(6)
GS_FLAG_POSE_COV_PATH = 1
GS_FLAG_NO_HOST_SYNC = 2
GS_FLAG_ACCUM_WEIGHT = 4
GS_FLAG_EXAMINED = 8
GS_FLAG_BINSORT_KEYS = 16
GS_FLAG_GRAD_ASSIGN = 32
GS_FLAG_OPACITY_RADIUS = 64
GS_FLAG_BINSORT_EMIT_ONLY = 256
GS_FLAG_BWD_SCREEN_ONLY = 512
GS_FLAG_BWD_CHAIN_ONLY = 1024
GS_DENSIFY_ADD, GS_DENSIFY_PRUNE, GS_DENSIFY_SELECT, GS_DENSIFY_DEGENERATE = 1, 2, 3, 4
GS_DENSIFY_DEGENERATE_FLAG, GS_DENSIFY_DEGENERATE_APPLY = 5, 6


class gs_camera(ctypes.Structure):
    _fields_ = [("fx", ctypes.c_float), ("fy", ctypes.c_float), ("cx", ctypes.c_float), ("cy", ctypes.c_float),
                ("width", ctypes.c_int32), ("height", ctypes.c_int32), ("znear", ctypes.c_float),
                ("bg", ctypes.c_float * 3), ("cov2d_dilation", ctypes.c_float)]


class gs_ws(ctypes.Structure):
    _fields_ = [("opaque", ctypes.c_uint64 * 128)]


class gs_ws_view(ctypes.Structure):
    _fields_ = [("records", ctypes.c_void_p), ("depth_key", ctypes.c_void_p), ("rect", ctypes.c_void_p),
                ("radius", ctypes.c_void_p), ("tiles", ctypes.c_void_p), ("offsets", ctypes.c_void_p),
                ("keys", ctypes.c_void_p),
                ("vals", ctypes.c_void_p), ("ranges", ctypes.c_void_p), ("t_final", ctypes.c_void_p),
                ("n_last", ctypes.c_void_p), ("examined", ctypes.c_void_p), ("n_keys_dev", ctypes.c_void_p),
                ("error_flag", ctypes.c_void_p), ("live_g", ctypes.c_void_p), ("live_j", ctypes.c_void_p),
                ("live_cnt", ctypes.c_void_p), ("n", ctypes.c_int64), ("key_cap", ctypes.c_int64),
                ("n_cap", ctypes.c_int64), ("grid_x", ctypes.c_int32), ("grid_y", ctypes.c_int32),
                ("width", ctypes.c_int32), ("height", ctypes.c_int32)]


class gs_densify_cfg(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("tau_alpha", ctypes.c_float), ("tau_depth", ctypes.c_float),
                ("min_opacity", ctypes.c_float), ("sel_weight", ctypes.c_float), ("sel_depth", ctypes.c_float),
                ("init_opacity", ctypes.c_float), ("stride", ctypes.c_int32), ("max_add", ctypes.c_int64),
                ("eta", ctypes.c_float), ("gamma", ctypes.c_float), ("rows", ctypes.c_int32)]


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_U32 = ctypes.c_uint32
_F = ctypes.c_float

_SIGS = {
    "gs_workspace_bytes": (ctypes.c_size_t, [_I64, _I64, _I32, _I32]),
    "gs_ws_init": (ctypes.c_int, [ctypes.POINTER(gs_ws), _P, ctypes.c_size_t, _I64, _I64, _I32, _I32]),
    "gs_project": (ctypes.c_int, [_P, _I64, _I64, _P, _P, ctypes.POINTER(gs_camera), ctypes.POINTER(gs_ws), _P]),
    "gs_densify_accum_grad": (ctypes.c_int, [ctypes.POINTER(gs_ws), _P, _P, _P]),
    "gs_densify_split_clone": (ctypes.c_int, [_P, _P, _P, _P, _P, _I64, _I64, _P, _P, _P, _F, _F, _I32, ctypes.POINTER(gs_ws),
                                              _P]),
    "gs_render_bwd_l1": (ctypes.c_int, [_P, _I64, _I64, _P, ctypes.POINTER(gs_ws), ctypes.POINTER(gs_camera), _P, _P,
                                        _P, _P, _F, _F, _P, _P, _P, _U32, _P]),
    "gs_pose_grad_l1": (ctypes.c_int, [_P, _I64, _I64, _P, ctypes.POINTER(gs_ws), ctypes.POINTER(gs_camera), _P, _P,
                                       _P, _P, _F, _F, _P, _P, _U32, _P]),
    "gs_pose_extrapolate": (ctypes.c_int, [_P, _P, _P, _P]),
    "gs_adam_step_rows": (ctypes.c_int, [_P, _P, _P, _P, _P, _I64, _I64, _I32, _P, _I32, _F, _F, _F, _P]),
    "gs_image_half": (ctypes.c_int, [_P, _P, _I32, _I32, _P, _P, _P]),
    "gs_frame_stats": (ctypes.c_int, [_P, _P, _P, _I32, _I32, _F, _F, _P, _P]),
    "gs_loss_l1_masked": (ctypes.c_int, [_P, _P, _P, _P, _P, _F, _F, _I32, _I32, _F, _F, _P, _P, _P, ctypes.POINTER(gs_ws),
                                         _P]),
    "gs_project_ex": (ctypes.c_int, [_P, _I64, _I64, _I32, _U32, _P, _P, ctypes.POINTER(gs_camera),
                                     ctypes.POINTER(gs_ws), _P]),
    "gs_project_sh": (ctypes.c_int, [_P, _I64, _I64, _I32, _P, _P, ctypes.POINTER(gs_camera), ctypes.POINTER(gs_ws),
                                     _P]),
    "gs_bin_sort": (ctypes.c_int, [ctypes.POINTER(gs_ws), ctypes.POINTER(_I64), _U32, _P]),
    "gs_render_fwd": (ctypes.c_int, [ctypes.POINTER(gs_ws), ctypes.POINTER(gs_camera), _P, _P, _P, _P, _U32, _P]),
    "gs_render_bwd": (ctypes.c_int, [_P, _I64, _I64, _P, ctypes.POINTER(gs_ws), ctypes.POINTER(gs_camera), _P, _P,
                                     _P, _P, _U32, _P]),
    "gs_pose_grad": (ctypes.c_int, [_P, _I64, _I64, _P, ctypes.POINTER(gs_ws), ctypes.POINTER(gs_camera), _P, _P,
                                    _P, _U32, _P]),
    "gs_loss_l1": (ctypes.c_int, [_P, _P, _P, _P, _I32, _I32, _F, _F, _P, _P, _P, ctypes.POINTER(gs_ws), _P]),
    "gs_adam_step": (ctypes.c_int, [_P, _P, _P, _P, _P, _I64, _I64, ctypes.POINTER(_F), _I32, _F, _F, _F, _P]),
    "gs_pose_step": (ctypes.c_int, [_P, _P, _P, _P, _I32, _F, _F, _P]),
    "gs_densify_prune": (ctypes.c_int, [_P, _P, _P, _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P,
                                        ctypes.POINTER(gs_camera), ctypes.POINTER(gs_densify_cfg), _P, _P,
                                        ctypes.POINTER(gs_ws), _P]),
    "gs_densify_append": (ctypes.c_int, [_P, _P, _P, _P, _P, _I64, _I64, _P, _P, _I32, _I64, _I32, _P]),
    "gs_ws_get_view": (ctypes.c_int, [ctypes.POINTER(gs_ws), ctypes.POINTER(gs_ws_view)]),
    "gs_ws_launch_count": (_I64, [ctypes.POINTER(gs_ws)]),
    "gs_ws_set_event_log": (ctypes.c_int, [ctypes.POINTER(gs_ws), _P, _P, _I32]),
    "gs_ws_event_log_count": (_I32, [ctypes.POINTER(gs_ws)]),
    "gs_events_create": (ctypes.c_int, [_P, _I32]),
    "gs_events_destroy": (ctypes.c_int, [_P, _I32]),
    "gs_events_elapsed": (ctypes.c_int, [_P, _I32, _P]),
    "gs_kernel_name": (ctypes.c_char_p, [_I32]),
    "gs_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "gs_last_cuda_error": (ctypes.c_char_p, []),
}
for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(_lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args

EXPORTED = tuple(_SIGS)


class GSError(RuntimeError):
    def __init__(self, status: int, what: str):
        msg = _lib.gs_status_string(status).decode()
        if status == GS_ERR_CUDA:
            msg += " (" + _lib.gs_last_cuda_error().decode() + ")"
        super().__init__(f"{what}: {msg}")
        self.status = status


def _check(status: int, what: str) -> None:
    if status != GS_OK:
        raise GSError(status, what)


def _ptr(t) -> ctypes.c_void_p | None:
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def make_camera(cam) -> gs_camera:
    """gs_camera from any object with fx, fy, cx, cy, width, height, znear, bg, cov2d_dilation."""
    c = gs_camera()
    c.fx, c.fy, c.cx, c.cy = cam.fx, cam.fy, cam.cx, cam.cy
    c.width, c.height = cam.width, cam.height
    c.znear = cam.znear
    for k in range(3):
        c.bg[k] = cam.bg[k]
    c.cov2d_dilation = cam.cov2d_dilation
    return c


# ----------------------------------------------------------------------------------- workspace
class Workspace:
    """Device workspace (a torch uint8 CUDA tensor) + the host state gs_ws."""

    def __init__(self, n_cap: int, key_cap: int, width: int, height: int, device="cuda"):
        import torch
        nbytes = int(_lib.gs_workspace_bytes(n_cap, key_cap, width, height))
        if nbytes == 0:
            raise GSError(GS_ERR_INVALID_ARG, "gs_workspace_bytes")
        self.dev = torch.empty(nbytes + 256, dtype=torch.uint8, device=device)
        base = self.dev.data_ptr()
        self._aligned = (base + 255) & ~255
        self.state = gs_ws()
        self.n_cap, self.key_cap, self.width, self.height = n_cap, key_cap, width, height
        self.nbytes = nbytes
        with torch.cuda.device(self.dev.device):
            _check(_lib.gs_ws_init(ctypes.byref(self.state), ctypes.c_void_p(self._aligned), nbytes, n_cap, key_cap,
                                   width, height), "gs_ws_init")

    def view(self) -> gs_ws_view:
        v = gs_ws_view()
        _check(_lib.gs_ws_get_view(ctypes.byref(self.state), ctypes.byref(v)), "gs_ws_get_view")
        return v

    def launches(self) -> int:
        return int(_lib.gs_ws_launch_count(ctypes.byref(self.state)))

    def tensor(self, addr: int, count: int, dtype):
        """A torch view of `count` elements of workspace memory at device address `addr` (tests/bench)."""
        import torch
        esz = torch.empty((), dtype=dtype).element_size()
        off = addr - self.dev.data_ptr()
        assert 0 <= off and off + count * esz <= self.dev.numel()
        return self.dev[off: off + count * esz].view(dtype)


class EventLog:
    """Per-kernel CUDA-event log attached to a workspace (gs_ws_set_event_log)."""

    def __init__(self, ws: Workspace, capacity: int):
        self.ws, self.capacity = ws, capacity
        self.events = (ctypes.c_void_p * (2 * capacity))()
        self.ids = (ctypes.c_int32 * capacity)()
        _check(_lib.gs_events_create(self.events, 2 * capacity), "gs_events_create")

    def __enter__(self):
        _check(_lib.gs_ws_set_event_log(ctypes.byref(self.ws.state), self.events, self.ids, self.capacity),
               "gs_ws_set_event_log")
        return self

    def __exit__(self, *exc):
        self.count = int(_lib.gs_ws_event_log_count(ctypes.byref(self.ws.state)))
        _check(_lib.gs_ws_set_event_log(ctypes.byref(self.ws.state), None, None, 0), "gs_ws_set_event_log")
        return False

    def read(self) -> list[tuple[str, float]]:
        """[(kernel name, ms)] for every logged launch (call after synchronising)."""
        ms = (ctypes.c_float * max(self.count, 1))()
        _check(_lib.gs_events_elapsed(self.events, self.count, ms), "gs_events_elapsed")
        return [(_lib.gs_kernel_name(self.ids[i]).decode(), float(ms[i])) for i in range(self.count)]

    def close(self):
        _lib.gs_events_destroy(self.events, 2 * self.capacity)


# ----------------------------------------------------------------------------------- ABI calls
def gs_project(params, n, ld, mask, viewmat, cam: gs_camera, ws: Workspace, stream=None):
    _check(_lib.gs_project(_ptr(params), n, ld, _ptr(mask), _ptr(viewmat), ctypes.byref(cam), ctypes.byref(ws.state),
                           _stream(stream)), "gs_project")


def gs_project_sh(params, n, ld, sh_degree, mask, viewmat, cam: gs_camera, ws: Workspace, stream=None):
    _check(_lib.gs_project_sh(_ptr(params), n, ld, sh_degree, _ptr(mask), _ptr(viewmat), ctypes.byref(cam),
                              ctypes.byref(ws.state), _stream(stream)), "gs_project_sh")


def gs_project_ex(params, n, ld, sh_degree, flags, mask, viewmat, cam: gs_camera, ws: Workspace, stream=None):
    _check(_lib.gs_project_ex(_ptr(params), n, ld, sh_degree, flags, _ptr(mask), _ptr(viewmat), ctypes.byref(cam),
                              ctypes.byref(ws.state), _stream(stream)), "gs_project_ex")


def gs_bin_sort(ws: Workspace, flags: int = 0, stream=None) -> int:
    k = _I64(-1)
    st = _lib.gs_bin_sort(ctypes.byref(ws.state), ctypes.byref(k), flags, _stream(stream))
    if st == GS_ERR_CAPACITY:
        raise GSError(st, f"gs_bin_sort (K={k.value} > key_cap={ws.key_cap})")
    _check(st, "gs_bin_sort")
    return int(k.value)


def gs_render_fwd(ws: Workspace, cam: gs_camera, color, depth, alpha, accum_weight=None, flags: int = 0, stream=None):
    _check(_lib.gs_render_fwd(ctypes.byref(ws.state), ctypes.byref(cam), _ptr(color), _ptr(depth), _ptr(alpha),
                              _ptr(accum_weight), flags, _stream(stream)), "gs_render_fwd")


def gs_render_bwd(params, n, ld, viewmat, ws: Workspace, cam: gs_camera, dL_dcolor, dL_ddepth, grad_params,
                  grad_pose=None, flags: int = GS_FLAG_POSE_COV_PATH, stream=None):
    _check(_lib.gs_render_bwd(_ptr(params), n, ld, _ptr(viewmat), ctypes.byref(ws.state), ctypes.byref(cam),
                              _ptr(dL_dcolor), _ptr(dL_ddepth), _ptr(grad_params), _ptr(grad_pose), flags,
                              _stream(stream)), "gs_render_bwd")


def gs_render_bwd_l1(params, n, ld, viewmat, ws: Workspace, cam: gs_camera, color, depth, tgt_color, tgt_depth,
                     w_color, w_depth, grad_params, grad_pose=None, loss=None, flags: int = GS_FLAG_POSE_COV_PATH,
                     stream=None):
    _check(_lib.gs_render_bwd_l1(_ptr(params), n, ld, _ptr(viewmat), ctypes.byref(ws.state), ctypes.byref(cam),
                                 _ptr(color), _ptr(depth), _ptr(tgt_color), _ptr(tgt_depth), w_color, w_depth,
                                 _ptr(grad_params), _ptr(grad_pose), _ptr(loss), flags, _stream(stream)),
           "gs_render_bwd_l1")


def gs_pose_grad(params, n, ld, viewmat, ws: Workspace, cam: gs_camera, dL_dcolor, dL_ddepth, grad_pose,
                 flags: int = GS_FLAG_POSE_COV_PATH, stream=None):
    _check(_lib.gs_pose_grad(_ptr(params), n, ld, _ptr(viewmat), ctypes.byref(ws.state), ctypes.byref(cam),
                             _ptr(dL_dcolor), _ptr(dL_ddepth), _ptr(grad_pose), flags, _stream(stream)),
           "gs_pose_grad")


def gs_pose_grad_l1(params, n, ld, viewmat, ws: Workspace, cam: gs_camera, color, depth, tgt_color, tgt_depth,
                    w_color, w_depth, grad_pose, loss=None, flags: int = GS_FLAG_POSE_COV_PATH, stream=None):
    _check(_lib.gs_pose_grad_l1(_ptr(params), n, ld, _ptr(viewmat), ctypes.byref(ws.state), ctypes.byref(cam),
                                _ptr(color), _ptr(depth), _ptr(tgt_color), _ptr(tgt_depth), w_color, w_depth,
                                _ptr(grad_pose), _ptr(loss), flags, _stream(stream)), "gs_pose_grad_l1")


def gs_loss_l1(color, depth, tgt_color, tgt_depth, width, height, w_color, w_depth, dL_dcolor, dL_ddepth, loss,
               ws: Workspace, stream=None):
    _check(_lib.gs_loss_l1(_ptr(color), _ptr(depth), _ptr(tgt_color), _ptr(tgt_depth), width, height, w_color,
                           w_depth, _ptr(dL_dcolor), _ptr(dL_ddepth), _ptr(loss), ctypes.byref(ws.state),
                           _stream(stream)), "gs_loss_l1")


def gs_pose_extrapolate(view_prev2, view_prev, view_out, stream=None):
    _check(_lib.gs_pose_extrapolate(_ptr(view_prev2), _ptr(view_prev), _ptr(view_out), _stream(stream)),
           "gs_pose_extrapolate")


def gs_image_half(color, depth, width, height, color_half, depth_half, stream=None):
    _check(_lib.gs_image_half(_ptr(color), _ptr(depth), width, height, _ptr(color_half), _ptr(depth_half),
                              _stream(stream)), "gs_image_half")


def gs_frame_stats(alpha, depth, target_depth, width, height, tau_alpha, tau_depth, counts, stream=None):
    _check(_lib.gs_frame_stats(_ptr(alpha), _ptr(depth), _ptr(target_depth), width, height, tau_alpha, tau_depth,
                               _ptr(counts), _stream(stream)), "gs_frame_stats")


def gs_loss_l1_masked(color, depth, tgt_color, tgt_depth, alpha, alpha_min, outlier_k, width, height, w_color,
                      w_depth, dL_dcolor, dL_ddepth, loss, ws: Workspace, stream=None):
    _check(_lib.gs_loss_l1_masked(_ptr(color), _ptr(depth), _ptr(tgt_color), _ptr(tgt_depth), _ptr(alpha), alpha_min,
                                  outlier_k, width, height, w_color, w_depth, _ptr(dL_dcolor), _ptr(dL_ddepth), _ptr(loss),
                                  ctypes.byref(ws.state), _stream(stream)), "gs_loss_l1_masked")


def gs_adam_step_rows(params_raw, params_act, grad_act, m, v, n, ld, rows, lr, step, b1=0.9, b2=0.999, eps=1e-8,
                      stream=None):
    lr_arr = (ctypes.c_float * rows)(*[float(x) for x in lr])
    _check(_lib.gs_adam_step_rows(_ptr(params_raw), _ptr(params_act), _ptr(grad_act), _ptr(m), _ptr(v), n, ld, rows,
                                  ctypes.cast(lr_arr, ctypes.c_void_p), step, b1, b2, eps, _stream(stream)),
           "gs_adam_step_rows")


def gs_adam_step(params_raw, params_act, grad_act, m, v, n, ld, lr, step, b1=0.9, b2=0.999, eps=1e-8, stream=None):
    lr_arr = (_F * 14)(*[float(x) for x in lr])
    _check(_lib.gs_adam_step(_ptr(params_raw), _ptr(params_act), _ptr(grad_act), _ptr(m), _ptr(v), n, ld, lr_arr,
                             step, b1, b2, eps, _stream(stream)), "gs_adam_step")


def gs_pose_step(viewmat, grad_pose, m6, v6, step, lr_rho, lr_phi, stream=None):
    _check(_lib.gs_pose_step(_ptr(viewmat), _ptr(grad_pose), _ptr(m6), _ptr(v6), step, lr_rho, lr_phi,
                             _stream(stream)), "gs_pose_step")


def densify_cfg(mode, tau_alpha=0.5, tau_depth=0.10, min_opacity=0.005, sel_weight=0.5, sel_depth=0.05,
                init_opacity=0.5, stride=2, max_add=0, eta=0.1, gamma=0.10, rows=14) -> gs_densify_cfg:
    c = gs_densify_cfg()
    c.mode, c.tau_alpha, c.tau_depth, c.min_opacity = mode, tau_alpha, tau_depth, min_opacity
    c.sel_weight, c.sel_depth, c.init_opacity, c.stride, c.max_add = sel_weight, sel_depth, init_opacity, stride, max_add
    c.eta, c.gamma, c.rows = eta, gamma, rows
    return c


def gs_densify_prune(params, params_raw, n_dev, capacity, ld, adam_m, adam_v, alpha, depth, target_rgb, target_depth,
                     accum_weight, viewmat, cam, cfg: gs_densify_cfg, select_mask, add_out, ws: Workspace,
                     stream=None):
    _check(_lib.gs_densify_prune(_ptr(params), _ptr(params_raw), _ptr(n_dev), capacity, ld, _ptr(adam_m),
                                 _ptr(adam_v), _ptr(alpha), _ptr(depth), _ptr(target_rgb), _ptr(target_depth),
                                 _ptr(accum_weight), _ptr(viewmat), ctypes.byref(cam) if cam is not None else None,
                                 ctypes.byref(cfg), _ptr(select_mask), _ptr(add_out), ctypes.byref(ws.state),
                                 _stream(stream)), "gs_densify_prune")


def gs_densify_accum_grad(ws: Workspace, grad_accum, count, stream=None):
    _check(_lib.gs_densify_accum_grad(ctypes.byref(ws.state), _ptr(grad_accum), _ptr(count), _stream(stream)),
           "gs_densify_accum_grad")


def gs_densify_split_clone(params, params_raw, adam_m, adam_v, n_dev, capacity, ld, grad_accum, count, noise,
                           grad_thresh, scale_thresh, ws: Workspace, stream=None, rows=14):
    _check(_lib.gs_densify_split_clone(_ptr(params), _ptr(params_raw), _ptr(adam_m), _ptr(adam_v), _ptr(n_dev), capacity,
                                       ld, _ptr(grad_accum), _ptr(count), _ptr(noise), grad_thresh, scale_thresh,
                                       rows, ctypes.byref(ws.state), _stream(stream)), "gs_densify_split_clone")


def gs_densify_append(params, params_raw, adam_m, adam_v, n_dev, capacity, ld, cand, counts, n_sets, max_add,
                      stream=None, rows=14):
    _check(_lib.gs_densify_append(_ptr(params), _ptr(params_raw), _ptr(adam_m), _ptr(adam_v), _ptr(n_dev), capacity,
                                  ld, _ptr(cand), _ptr(counts), n_sets, max_add, rows, _stream(stream)),
           "gs_densify_append")


from .pipeline import Frame, RenderPipeline  # noqa: E402  (convenience layer over the calls above)

__all__ = [*EXPORTED, "Workspace", "RenderPipeline", "Frame", "make_camera", "densify_cfg", "GSError"]
