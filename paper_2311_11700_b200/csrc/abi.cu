// C ABI entry points of libgs (include/gs.h): argument checks on the host, workspace carving,
// generation tracking, and dispatch to the kernels. No allocation, no global device state.
#include <algorithm>
#include <cstring>
#include <string>

#include "gs_internal.cuh"
#include "onesweep.cuh"

namespace gs {

static thread_local std::string g_last_cuda_error;

void set_cuda_error(cudaError_t e, const char* what) {
    g_last_cuda_error = std::string(what) + ": " + cudaGetErrorString(e);
}

void set_error_text(const char* msg) { g_last_cuda_error = msg; }

gs_status check_launch(WsState*, const char* what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_cuda_error(e, what);
        return GS_ERR_CUDA;
    }
    return GS_OK;
}

struct Carver {
    uint64_t off = 0;
    Region take(uint64_t bytes) {
        Region r{off, bytes};
        off += (bytes + 255) & ~uint64_t(255);
        return r;
    }
};

static int64_t sort_parts(int64_t key_cap) { return (std::max<int64_t>(key_cap, 1) + kSortTile - 1) / kSortTile; }

static void carve(WsState* s, Carver& c) {
    const int64_t n = std::max<int64_t>(s->n_cap, 1), K = std::max<int64_t>(s->key_cap, 1);
    const int64_t px = int64_t(s->W) * s->H;
    const int64_t tiles = int64_t(s->GX) * s->GY;
    const int64_t scan_items = std::max(n, px);
    s->rec = c.take(uint64_t(n) * 48);
    s->depth_key = c.take(uint64_t(n) * 4);
    s->rect = c.take(uint64_t(n) * 8);
    s->radius = c.take(uint64_t(n) * 4);
    s->tiles = c.take(uint64_t(n) * 4);
    s->offsets = c.take(uint64_t(n) * 4);
    s->sgrad = c.take(uint64_t(n) * 4 * 10);
    s->scan_state = c.take(uint64_t((scan_items + 2047) / 2048 + 1) * 8);
    s->keys0 = c.take(uint64_t(K) * 8);
    s->keys1 = c.take(uint64_t(K) * 8);
    s->vals0 = c.take(uint64_t(K) * 4);
    s->vals1 = c.take(uint64_t(K) * 4);
    s->ranges = c.take(uint64_t(tiles) * 8);
    s->t_final = c.take(uint64_t(px) * 4);
    s->n_last = c.take(uint64_t(px) * 4);
    s->examined = c.take(uint64_t(px) * 4);
    s->sort_hist = c.take(8 * 256 * 4);
    // look-back rows: path A sorts key_cap keys in kSortTile-key (2048) partitions, path B n_cap keys in 1024-key ones
    s->max_parts = std::max(sort_parts(s->key_cap), (std::max<int64_t>(s->n_cap, 1) + 1023) / 1024);
    s->sort_look = c.take(uint64_t(s->max_parts) * 256 * 8);
    s->misc = c.take(sizeof(Misc));
    s->scratch = c.take(uint64_t(px) * 4 * 4);
    // in-place compaction (prune, split/clone): per-256-column counts / offsets, ticket + read flags
    s->cmp = c.take(uint64_t(2 * ((n + 255) / 256 + 2)) * 4);
    s->dkey_sorted = c.take(uint64_t(n) * 4 * 2);
    s->dval_sorted = c.take(uint64_t(n) * 4 * 2);
    // densify block counts; also the backward prologue's per-block valid counts (148 * 4 blocks)
    s->chunk_hist = c.take(uint64_t(std::max<int64_t>({(n + 2047) / 2048, (px + 2047) / 2048, 1024}) + 1) * 4);
    s->chunk_mat = c.take(uint64_t((n + 255) / 256 + 1) * tiles * 4);   // path B count/base matrix
    s->srect = c.take(uint64_t(n) * 8);
    s->tile_tot = c.take(uint64_t(tiles) * 4 * 10);   // totals, starts, 8 segment sums
    s->pose_part = c.take(uint64_t(2 * ((n + 255) / 256) + 1) * 16 * 8);   // per-block pose partials (gaussian_bwd grid)
    s->onlist = c.take(uint64_t(n) * 4);                              // on-screen Gaussians, index order
    s->live_cnt = c.take(uint64_t(tiles) * 4);                        // per-tile live-list lengths
    s->svals = c.take(uint64_t(n) * 4);                               // path B: depth-sorted on-screen Gaussians
    // path B cooperative kernel: per-pass per-CTA digit histograms, pass totals, per-CTA counts,
    // tile totals and per-(segment, tile) sums
    s->coop = c.take((uint64_t(kCoopPasses) * kCoopGridMax * kCoopBins + kCoopPasses * kCoopBins + kCoopGridMax +
                      uint64_t(tiles) * (1 + kCoopSegs)) * 4);
    s->tile_order = c.take(uint64_t(tiles) * 4);                     // backward LPT tile order
    s->tile_pose = c.take(uint64_t(tiles) * 6 * 8);                  // pose-only pass: per-tile twist partials
}

static bool ws_ok(const gs_ws* ws) { return ws && state(ws)->magic == kMagic; }

}  // namespace gs

using namespace gs;

extern "C" {

size_t gs_workspace_bytes(int64_t n_cap, int64_t key_cap, int32_t W, int32_t H) {
    if (n_cap < 0 || key_cap < 0 || W <= 0 || H <= 0) return 0;
    WsState s{};
    s.n_cap = n_cap;
    s.key_cap = key_cap;
    s.W = W;
    s.H = H;
    s.GX = (W + kTile - 1) / kTile;
    s.GY = (H + kTile - 1) / kTile;
    Carver c;
    carve(&s, c);
    return size_t(c.off);
}

gs_status gs_ws_init(gs_ws* ws, void* dev, size_t dev_bytes, int64_t n_cap, int64_t key_cap, int32_t W, int32_t H) {
    if (!ws || !dev || n_cap < 0 || key_cap < 0 || key_cap >= (int64_t(1) << 30) || n_cap >= (int64_t(1) << 31) ||
        W <= 0 || H <= 0 || (reinterpret_cast<uintptr_t>(dev) & 255))
        return GS_ERR_INVALID_ARG;
    if (dev_bytes < gs_workspace_bytes(n_cap, key_cap, W, H)) return GS_ERR_INVALID_ARG;
    std::memset(ws, 0, sizeof(gs_ws));
    WsState* s = state(ws);
    s->magic = kMagic;
    s->dev = static_cast<char*>(dev);
    s->dev_bytes = dev_bytes;
    s->n_cap = n_cap;
    s->key_cap = key_cap;
    s->W = W;
    s->H = H;
    s->GX = (W + kTile - 1) / kTile;
    s->GY = (H + kTile - 1) / kTile;
    Carver c;
    carve(s, c);
    s->n_keys_host = -1;
    s->epoch = 1;
    // look-back words must not carry a live epoch: clear them once (legacy stream, synchronous)
    if (cudaMemset(s->dev + s->scan_state.off, 0, s->scan_state.bytes) != cudaSuccess ||
        cudaMemset(s->dev + s->sort_look.off, 0, s->sort_look.bytes) != cudaSuccess ||
        cudaMemset(s->dev + s->misc.off, 0, s->misc.bytes) != cudaSuccess) {
        set_cuda_error(cudaGetLastError(), "gs_ws_init memset");
        return GS_ERR_CUDA;
    }
    return GS_OK;
}

static bool cam_ok(const WsState* s, const gs_camera* cam) {
    return cam && cam->width > 0 && cam->height > 0 && cam->width <= s->W * 1 && cam->height <= s->H &&
           int64_t(cam->width) * cam->height <= int64_t(s->W) * s->H && cam->fx > 0 && cam->fy > 0 &&
           ((cam->width + kTile - 1) / kTile) * ((cam->height + kTile - 1) / kTile) <= s->GX * s->GY;
}

gs_status gs_project(const float* params, int64_t n, int64_t ld, const uint8_t* mask, const float* viewmat,
                     const gs_camera* cam, gs_ws* ws, void* stream) {
    GS_NVTX("gs_project");
    return gs_project_sh(params, n, ld, 0, mask, viewmat, cam, ws, stream);
}

gs_status gs_project_sh(const float* params, int64_t n, int64_t ld, int32_t sh_degree, const uint8_t* mask,
                        const float* viewmat, const gs_camera* cam, gs_ws* ws, void* stream) {
    GS_NVTX("gs_project_sh");
    return gs_project_ex(params, n, ld, sh_degree, 0u, mask, viewmat, cam, ws, stream);
}

gs_status gs_project_ex(const float* params, int64_t n, int64_t ld, int32_t sh_degree, uint32_t flags,
                        const uint8_t* mask, const float* viewmat, const gs_camera* cam, gs_ws* ws, void* stream) {
    GS_NVTX("gs_project_ex");
    if (!ws_ok(ws)) return GS_ERR_INVALID_ARG;
    WsState* s = state(ws);
    if (n < 0 || n > s->n_cap || ld < n || (n > 0 && !params) || !viewmat || !cam_ok(s, cam) ||
        (sh_degree != 0 && sh_degree != 1) || (flags & ~uint32_t(GS_FLAG_OPACITY_RADIUS)))
        return GS_ERR_INVALID_ARG;
    s->n = n;
    s->sh_degree = sh_degree;
    s->opacity_radius = (flags & GS_FLAG_OPACITY_RADIUS) ? 1 : 0;
    s->cam_w = cam->width;
    s->cam_h = cam->height;
    s->cam_gx = (cam->width + kTile - 1) / kTile;
    s->cam_gy = (cam->height + kTile - 1) / kTile;
    s->gen_project += 1;
    launch_project(s, params, n, ld, mask, viewmat, *cam, static_cast<cudaStream_t>(stream));
    const gs_status rc = check_launch(s, "gs_project");
    if (GS_DEBUG && rc == GS_OK) return dbg_after_project(s, static_cast<cudaStream_t>(stream));
    return rc;
}

gs_status gs_bin_sort(gs_ws* ws, int64_t* n_keys, uint32_t flags, void* stream) {
    GS_NVTX("gs_bin_sort");
    if (!ws_ok(ws)) return GS_ERR_INVALID_ARG;
    WsState* s = state(ws);
    if (s->gen_project == 0) return GS_ERR_STALE;
    const gs_status rc = (flags & GS_FLAG_BINSORT_KEYS)
                             ? run_bin_sort_keys(s, n_keys, flags, static_cast<cudaStream_t>(stream))
                             : run_bin_sort_bucket(s, n_keys, flags, static_cast<cudaStream_t>(stream));
    if (GS_DEBUG && rc == GS_OK && !(flags & GS_FLAG_BINSORT_EMIT_ONLY))
        return dbg_after_bin_sort(s, static_cast<cudaStream_t>(stream));
    return rc;
}

gs_status gs_render_fwd(gs_ws* ws, const gs_camera* cam, float* color, float* depth, float* alpha, float* accum_weight,
                        uint32_t flags, void* stream) {
    GS_NVTX("gs_render_fwd");
    if (!ws_ok(ws)) return GS_ERR_INVALID_ARG;
    WsState* s = state(ws);
    if (!cam_ok(s, cam) || !color || !depth || !alpha) return GS_ERR_INVALID_ARG;
    if (cam->width != s->cam_w || cam->height != s->cam_h) return GS_ERR_INVALID_ARG;
    if (s->gen_project == 0) return GS_ERR_STALE;
    launch_render_fwd(s, *cam, color, depth, alpha, accum_weight, flags, static_cast<cudaStream_t>(stream));
    s->gen_fwd = s->gen_project;
    const gs_status rc = check_launch(s, "gs_render_fwd");
    if (GS_DEBUG && rc == GS_OK) return dbg_after_fwd(s, static_cast<cudaStream_t>(stream), color, depth, alpha);
    return rc;
}

// mode: BWD_FULL (gs_render_bwd[_l1]); gs_pose_grad[_l1] picks a pose-only tile pass (render.cu BwdMode):
// the paper's gradient (no POSE_COV_PATH) needs only that pass; with the covariance path the pass keeps
// the 6 quantities the per-Gaussian chain reads (degree-1 SH: all 10, the colour reaches the pose).
static gs_status backward_common(const float* params, int64_t n, int64_t ld, const float* viewmat, gs_ws* ws,
                                 const gs_camera* cam, const float* dLdC, const float* dLdD, float* grad,
                                 double* grad_pose, uint32_t flags, void* stream, const L1Fuse* fuse = nullptr,
                                 bool pose_only = false) {
    if (!ws_ok(ws)) return GS_ERR_INVALID_ARG;
    WsState* s = state(ws);
    if (!cam_ok(s, cam) || (!fuse && (!dLdC || !dLdD)) || !viewmat || (n > 0 && !params) || ld < n)
        return GS_ERR_INVALID_ARG;
    if (s->gen_fwd == 0 || s->gen_fwd != s->gen_project || n != s->n || cam->width != s->cam_w ||
        cam->height != s->cam_h)
        return GS_ERR_STALE;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int mode = !pose_only ? 0 : !(flags & GS_FLAG_POSE_COV_PATH) ? 2 : (s->sh_degree == 1 ? 0 : 1);
    const int assign = (flags & GS_FLAG_GRAD_ASSIGN) ? 1 : 0;
    const bool screen_only = (flags & GS_FLAG_BWD_SCREEN_ONLY) != 0, chain_only = (flags & GS_FLAG_BWD_CHAIN_ONLY) != 0;
    if ((screen_only || chain_only) && (pose_only || (screen_only && chain_only))) return GS_ERR_INVALID_ARG;
    if (chain_only) {   // the per-Gaussian chain from the screen gradients of this forward's tile pass
        if (s->gen_screen != s->gen_fwd) return GS_ERR_STALE;
        launch_zero(&at<Misc>(s, s->misc)->gbwd_zero_chunk, sizeof(unsigned int), st, s);
        launch_gaussian_bwd(s, params, n, ld, viewmat, *cam, grad, grad_pose, flags, st,
                            LossFin{nullptr, nullptr, 0.f, 0.f, 0});
        s->gen_bwd = s->gen_fwd;
        const gs_status rc = check_launch(s, "gs_render_bwd (chain)");
        if (GS_DEBUG && rc == GS_OK) return dbg_after_bwd(s, st, grad, n, ld, grad_pose);
        return rc;
    }
    // prologue: screen accumulators [10][V_s] (rank-indexed; not needed by the paper-mode pose pass),
    // LPT tile order, fused-L1 valid count
    if (n > 0 || fuse)
        launch_zero_sgrad(s, st, fuse ? fuse->td : nullptr, fuse ? int64_t(cam->width) * cam->height : 0, mode != 2);
    if (mode == 2) {   // the pose-only pass is the whole backward (its last block writes twist and loss)
        launch_render_bwd_tiles(s, *cam, nullptr, dLdC, dLdD, st, fuse, true, mode, grad_pose, assign);
        s->gen_bwd = s->gen_fwd;
        const gs_status rc = check_launch(s, "gs_pose_grad");
        if (GS_DEBUG && rc == GS_OK) return dbg_after_bwd(s, st, nullptr, n, ld, grad_pose);
        return rc;
    }
    // fused L1 with a pose gradient: gaussian_bwd's last block (which exists then) writes the loss
    const bool fin_in_gbwd = fuse && fuse->loss && grad_pose && n > 0 && !screen_only;
    launch_render_bwd_tiles(s, *cam, nullptr, dLdC, dLdD, st, fuse, !fin_in_gbwd, mode);
    s->gen_screen = s->gen_fwd;
    if (screen_only) {
        s->gen_bwd = s->gen_fwd;   // the screen gradients are there (gs_densify_accum_grad reads them)
        return check_launch(s, "gs_render_bwd (screen)");
    }
    LossFin lf{nullptr, nullptr, 0.f, 0.f, 0};
    if (fin_in_gbwd)
        lf = LossFin{at<Misc>(s, s->misc)->loss_acc, fuse->loss, fuse->wc, fuse->wd, int64_t(cam->width) * cam->height};
    launch_gaussian_bwd(s, params, n, ld, viewmat, *cam, grad, grad_pose, flags, st, lf);
    s->gen_bwd = s->gen_fwd;
    const gs_status rc = check_launch(s, "gs_render_bwd");
    if (GS_DEBUG && rc == GS_OK) return dbg_after_bwd(s, st, grad, n, ld, grad_pose);
    return rc;
}

gs_status gs_render_bwd(const float* params, int64_t n, int64_t ld, const float* viewmat, gs_ws* ws,
                        const gs_camera* cam, const float* dL_dcolor, const float* dL_ddepth, float* grad_params,
                        double* grad_pose, uint32_t flags, void* stream) {
    GS_NVTX("gs_render_bwd");
    if (!grad_params) return GS_ERR_INVALID_ARG;
    return backward_common(params, n, ld, viewmat, ws, cam, dL_dcolor, dL_ddepth, grad_params, grad_pose, flags,
                           stream);
}

gs_status gs_render_bwd_l1(const float* params, int64_t n, int64_t ld, const float* viewmat, gs_ws* ws,
                           const gs_camera* cam, const float* color, const float* depth, const float* tgt_color,
                           const float* tgt_depth, float w_color, float w_depth, float* grad_params,
                           double* grad_pose, double* loss, uint32_t flags, void* stream) {
    GS_NVTX("gs_render_bwd_l1");
    if (!grad_params || !color || !depth || !tgt_color || !tgt_depth) return GS_ERR_INVALID_ARG;
    const L1Fuse fuse{color, depth, tgt_color, tgt_depth, w_color, w_depth, loss};
    return backward_common(params, n, ld, viewmat, ws, cam, nullptr, nullptr, grad_params, grad_pose, flags, stream,
                           &fuse);
}

gs_status gs_pose_grad(const float* params, int64_t n, int64_t ld, const float* viewmat, gs_ws* ws,
                       const gs_camera* cam, const float* dL_dcolor, const float* dL_ddepth, double* grad_pose,
                       uint32_t flags, void* stream) {
    GS_NVTX("gs_pose_grad");
    if (!grad_pose) return GS_ERR_INVALID_ARG;
    return backward_common(params, n, ld, viewmat, ws, cam, dL_dcolor, dL_ddepth, nullptr, grad_pose, flags, stream,
                           nullptr, true);
}

gs_status gs_pose_grad_l1(const float* params, int64_t n, int64_t ld, const float* viewmat, gs_ws* ws,
                          const gs_camera* cam, const float* color, const float* depth, const float* tgt_color,
                          const float* tgt_depth, float w_color, float w_depth, double* grad_pose, double* loss,
                          uint32_t flags, void* stream) {
    GS_NVTX("gs_pose_grad_l1");
    if (!grad_pose || !color || !depth || !tgt_color || !tgt_depth) return GS_ERR_INVALID_ARG;
    const L1Fuse fuse{color, depth, tgt_color, tgt_depth, w_color, w_depth, loss};
    return backward_common(params, n, ld, viewmat, ws, cam, nullptr, nullptr, nullptr, grad_pose, flags, stream, &fuse,
                           true);
}

gs_status gs_loss_l1(const float* color, const float* depth, const float* tgt_color, const float* tgt_depth, int32_t W,
                     int32_t H, float w_color, float w_depth, float* dL_dcolor, float* dL_ddepth, double* loss,
                     gs_ws* ws, void* stream) {
    GS_NVTX("gs_loss_l1");
    if (!ws_ok(ws) || !color || !depth || !tgt_color || !tgt_depth || !dL_dcolor || !dL_ddepth || W <= 0 || H <= 0)
        return GS_ERR_INVALID_ARG;
    WsState* s = state(ws);
    launch_loss_l1(s, color, depth, tgt_color, tgt_depth, W, H, w_color, w_depth, dL_dcolor, dL_ddepth, loss,
                   static_cast<cudaStream_t>(stream));
    return check_launch(s, "gs_loss_l1");
}

gs_status gs_loss_l1_masked(const float* color, const float* depth, const float* tgt_color, const float* tgt_depth,
                            const float* alpha, float alpha_min, float outlier_k, int32_t W, int32_t H, float w_color,
                            float w_depth, float* dL_dcolor, float* dL_ddepth, double* loss, gs_ws* ws, void* stream) {
    GS_NVTX("gs_loss_l1_masked");
    if (!ws_ok(ws) || !color || !depth || !tgt_color || !tgt_depth || !alpha || !dL_dcolor || !dL_ddepth || W <= 0 ||
        H <= 0 || !(outlier_k >= 0.f))
        return GS_ERR_INVALID_ARG;
    WsState* s = state(ws);
    launch_loss_l1_masked(s, color, depth, tgt_color, tgt_depth, alpha, alpha_min, outlier_k, W, H, w_color, w_depth, dL_dcolor,
                          dL_ddepth, loss, static_cast<cudaStream_t>(stream));
    return check_launch(s, "gs_loss_l1_masked");
}

gs_status gs_frame_stats(const float* alpha, const float* depth, const float* target_depth, int32_t W, int32_t H,
                         float tau_alpha, float tau_depth, uint32_t* counts, void* stream) {
    GS_NVTX("gs_frame_stats");
    if (!alpha || !depth || !target_depth || !counts || W <= 0 || H <= 0) return GS_ERR_INVALID_ARG;
    launch_frame_stats(alpha, depth, target_depth, W, H, tau_alpha, tau_depth, counts, static_cast<cudaStream_t>(stream));
    return check_launch(nullptr, "gs_frame_stats");
}

gs_status gs_pose_extrapolate(const float* view_prev2, const float* view_prev, float* view_out, void* stream) {
    GS_NVTX("gs_pose_extrapolate");
    if (!view_prev2 || !view_prev || !view_out || view_out == view_prev || view_out == view_prev2)
        return GS_ERR_INVALID_ARG;
    launch_pose_extrapolate(view_prev2, view_prev, view_out, static_cast<cudaStream_t>(stream));
    return check_launch(nullptr, "gs_pose_extrapolate");
}

gs_status gs_image_half(const float* color, const float* depth, int32_t W, int32_t H, float* color_half,
                        float* depth_half, void* stream) {
    GS_NVTX("gs_image_half");
    if (!color || !depth || !color_half || !depth_half || W < 2 || H < 2) return GS_ERR_INVALID_ARG;
    launch_image_half(color, depth, W, H, color_half, depth_half, static_cast<cudaStream_t>(stream));
    return check_launch(nullptr, "gs_image_half");
}

gs_status gs_adam_step(float* params_raw, float* params_act, const float* grad_act, float* m, float* v, int64_t n,
                       int64_t ld, const float lr[14], int32_t step, float b1, float b2, float eps, void* stream) {
    GS_NVTX("gs_adam_step");
    if ((n > 0 && (!params_raw || !params_act || !grad_act || !m || !v)) || !lr || n < 0 || ld < n || step < 1)
        return GS_ERR_INVALID_ARG;
    launch_adam(params_raw, params_act, grad_act, m, v, n, ld, lr, 14, step, b1, b2, eps,
                static_cast<cudaStream_t>(stream));
    return check_launch(nullptr, "gs_adam_step");
}

gs_status gs_adam_step_rows(float* params_raw, float* params_act, const float* grad_act, float* m, float* v,
                            int64_t n, int64_t ld, int32_t rows, const float* lr, int32_t step, float b1, float b2,
                            float eps, void* stream) {
    GS_NVTX("gs_adam_step_rows");
    if ((n > 0 && (!params_raw || !params_act || !grad_act || !m || !v)) || !lr || n < 0 || ld < n || step < 1 ||
        (rows != 14 && rows != 23))
        return GS_ERR_INVALID_ARG;
    launch_adam(params_raw, params_act, grad_act, m, v, n, ld, lr, rows, step, b1, b2, eps,
                static_cast<cudaStream_t>(stream));
    return check_launch(nullptr, "gs_adam_step_rows");
}

gs_status gs_pose_step(float* viewmat, const double* grad_pose, float* m6, float* v6, int32_t step, float lr_rho,
                       float lr_phi, void* stream) {
    GS_NVTX("gs_pose_step");
    if (!viewmat || !grad_pose || !m6 || !v6 || step < 1) return GS_ERR_INVALID_ARG;
    launch_pose_step(viewmat, grad_pose, m6, v6, step, lr_rho, lr_phi, static_cast<cudaStream_t>(stream));
    return check_launch(nullptr, "gs_pose_step");
}

gs_status gs_densify_prune(float* params, float* params_raw, int64_t* n_dev, int64_t capacity, int64_t ld,
                           float* adam_m, float* adam_v, const float* alpha, const float* depth,
                           const float* target_rgb, const float* target_depth, const float* accum_weight,
                           const float* viewmat, const gs_camera* cam, const gs_densify_cfg* cfg,
                           uint8_t* select_mask, float* add_out, gs_ws* ws, void* stream) {
    GS_NVTX("gs_densify_prune");
    if (!ws_ok(ws) || !cfg || !n_dev || capacity < 0 || ld < capacity) return GS_ERR_INVALID_ARG;
    WsState* s = state(ws);
    if (cfg->rows != 0 && cfg->rows != 14 && cfg->rows != 23) return GS_ERR_INVALID_ARG;
    switch (cfg->mode) {
        case GS_DENSIFY_ADD:
            if (!params || !alpha || !depth || !target_rgb || !target_depth || !viewmat || !cam_ok(s, cam) ||
                cfg->stride < 1 || cfg->max_add < 0)
                return GS_ERR_INVALID_ARG;
            break;
        case GS_DENSIFY_PRUNE:
            if (!params || capacity > s->n_cap) return GS_ERR_INVALID_ARG;
            break;
        case GS_DENSIFY_SELECT:
            if (!select_mask || !accum_weight || !target_depth || !cam_ok(s, cam) || capacity > s->n_cap)
                return GS_ERR_INVALID_ARG;
            if (s->gen_project == 0) return GS_ERR_STALE;
            break;
        case GS_DENSIFY_DEGENERATE:
            if (!params || !target_depth || !cam_ok(s, cam) || capacity > s->n_cap || !(cfg->eta >= 0.f) ||
                !(cfg->eta <= 1.f))
                return GS_ERR_INVALID_ARG;
            if (s->gen_project == 0) return GS_ERR_STALE;
            break;
        case GS_DENSIFY_DEGENERATE_FLAG:
            if (!select_mask || !target_depth || !cam_ok(s, cam) || capacity > s->n_cap) return GS_ERR_INVALID_ARG;
            if (s->gen_project == 0) return GS_ERR_STALE;
            break;
        case GS_DENSIFY_DEGENERATE_APPLY:
            if (!params || !select_mask || !(cfg->eta >= 0.f) || !(cfg->eta <= 1.f)) return GS_ERR_INVALID_ARG;
            break;
        default:
            return GS_ERR_INVALID_ARG;
    }
    const gs_camera dummy{};
    return run_densify(s, params, params_raw, n_dev, capacity, ld, adam_m, adam_v, alpha, depth, target_rgb,
                       target_depth, accum_weight, viewmat, cam ? *cam : dummy, *cfg, select_mask, add_out,
                       static_cast<cudaStream_t>(stream));
}

gs_status gs_densify_append(float* params, float* params_raw, float* adam_m, float* adam_v, int64_t* n_dev,
                            int64_t capacity, int64_t ld, const float* cand, const int64_t* counts, int32_t n_sets,
                            int64_t max_add, int32_t rows, void* stream) {
    GS_NVTX("gs_densify_append");
    if (!params || !n_dev || capacity < 0 || ld < capacity || n_sets < 0 || max_add < 0 ||
        (n_sets > 0 && (!cand || !counts)) || (rows != 14 && rows != 23))
        return GS_ERR_INVALID_ARG;
    launch_append(params, params_raw, adam_m, adam_v, n_dev, capacity, ld, cand, counts, n_sets, max_add, rows,
                  static_cast<cudaStream_t>(stream));
    return check_launch(nullptr, "gs_densify_append");
}

gs_status gs_densify_accum_grad(gs_ws* ws, float* grad_accum, float* count, void* stream) {
    GS_NVTX("gs_densify_accum_grad");
    if (!ws_ok(ws) || !grad_accum || !count) return GS_ERR_INVALID_ARG;
    WsState* s = state(ws);
    if (s->gen_fwd == 0 || s->gen_bwd != s->gen_fwd || s->gen_fwd != s->gen_project) return GS_ERR_STALE;
    launch_accum_grad(s, grad_accum, count, static_cast<cudaStream_t>(stream));
    return check_launch(s, "gs_densify_accum_grad");
}

gs_status gs_densify_split_clone(float* params, float* params_raw, float* adam_m, float* adam_v, int64_t* n_dev,
                                 int64_t capacity, int64_t ld, float* grad_accum, float* count, const float* noise,
                                 float grad_thresh, float scale_thresh, int32_t rows, gs_ws* ws, void* stream) {
    GS_NVTX("gs_densify_split_clone");
    if (!ws_ok(ws) || !params || !n_dev || !grad_accum || !count || !noise || capacity < 0 || ld < capacity ||
        !(grad_thresh >= 0.f) || !(scale_thresh >= 0.f) || (rows != 14 && rows != 23))
        return GS_ERR_INVALID_ARG;
    WsState* s = state(ws);
    if (capacity > s->n_cap) return GS_ERR_INVALID_ARG;
    return run_split_clone(s, params, params_raw, adam_m, adam_v, n_dev, capacity, ld, grad_accum, count, noise,
                           grad_thresh, scale_thresh, rows, static_cast<cudaStream_t>(stream));
}

gs_status gs_ws_get_view(const gs_ws* ws, gs_ws_view* out) {
    if (!ws_ok(ws) || !out) return GS_ERR_INVALID_ARG;
    const WsState* s = state(ws);
    Misc* misc = at<Misc>(s, s->misc);
    out->records = at<float>(s, s->rec);
    out->depth_key = at<uint32_t>(s, s->depth_key);
    out->rect = at<int16_t>(s, s->rect);
    out->radius = at<int32_t>(s, s->radius);
    out->tiles = at<uint32_t>(s, s->tiles);
    out->offsets = at<uint32_t>(s, s->offsets);
    out->keys = !s->keys_valid ? nullptr : s->sorted_in_1 ? at<uint64_t>(s, s->keys1) : at<uint64_t>(s, s->keys0);
    out->vals = s->sorted_in_1 ? at<uint32_t>(s, s->vals1) : at<uint32_t>(s, s->vals0);
    out->ranges = at<uint32_t>(s, s->ranges);
    out->t_final = at<float>(s, s->t_final);
    out->n_last = at<uint32_t>(s, s->n_last);
    out->examined = at<uint32_t>(s, s->examined);
    out->n_keys_dev = reinterpret_cast<const uint64_t*>(&misc->n_keys);
    out->error_flag = &misc->error_flag;
    // live lists: the value / key buffers that do not hold the sorted list (render.cu live_bufs)
    out->live_g = s->sorted_in_1 ? at<uint32_t>(s, s->vals0) : at<uint32_t>(s, s->vals1);
    out->live_j = reinterpret_cast<const uint32_t*>(s->sorted_in_1 ? at<uint64_t>(s, s->keys0)
                                                                   : at<uint64_t>(s, s->keys1));
    out->live_cnt = at<uint32_t>(s, s->live_cnt);
    out->n = s->n;
    out->key_cap = s->key_cap;
    out->n_cap = s->n_cap;
    out->grid_x = s->cam_gx;
    out->grid_y = s->cam_gy;
    out->width = s->cam_w;
    out->height = s->cam_h;
    return GS_OK;
}

int64_t gs_ws_launch_count(const gs_ws* ws) { return ws_ok(ws) ? state(ws)->launches : -1; }

gs_status gs_ws_set_event_log(gs_ws* ws, void** events, int32_t* ids, int32_t capacity) {
    if (!ws_ok(ws) || capacity < 0 || (capacity > 0 && (!events || !ids))) return GS_ERR_INVALID_ARG;
    WsState* s = state(ws);
    s->ev = capacity > 0 ? events : nullptr;
    s->ev_ids = capacity > 0 ? ids : nullptr;
    s->ev_cap = capacity;
    s->ev_n = 0;
    return GS_OK;
}

int32_t gs_ws_event_log_count(const gs_ws* ws) { return ws_ok(ws) ? state(ws)->ev_n : -1; }

gs_status gs_events_create(void** events, int32_t count) {
    if (!events || count < 0) return GS_ERR_INVALID_ARG;
    for (int32_t i = 0; i < count; ++i) {
        cudaEvent_t e;
        const cudaError_t err = cudaEventCreate(&e);
        if (err != cudaSuccess) {
            set_cuda_error(err, "cudaEventCreate");
            return GS_ERR_CUDA;
        }
        events[i] = e;
    }
    return GS_OK;
}

gs_status gs_events_destroy(void** events, int32_t count) {
    if (!events || count < 0) return GS_ERR_INVALID_ARG;
    for (int32_t i = 0; i < count; ++i)
        if (events[i]) cudaEventDestroy(static_cast<cudaEvent_t>(events[i]));
    return GS_OK;
}

gs_status gs_events_elapsed(void* const* events, int32_t pairs, float* ms) {
    if (!events || !ms || pairs < 0) return GS_ERR_INVALID_ARG;
    for (int32_t i = 0; i < pairs; ++i) {
        const cudaError_t err = cudaEventElapsedTime(ms + i, static_cast<cudaEvent_t>(events[2 * i]),
                                                     static_cast<cudaEvent_t>(events[2 * i + 1]));
        if (err != cudaSuccess) {
            set_cuda_error(err, "cudaEventElapsedTime");
            return GS_ERR_CUDA;
        }
    }
    return GS_OK;
}

const char* gs_kernel_name(int32_t id) {
    static const char* names[KID_COUNT] = {"project", "chained_scan", "emit_keys", "sort_hist", "sort_digit_scan",
                                           "sort_pass", "tile_ranges", "render_fwd", "render_bwd_tiles",
                                           "gaussian_bwd", "pose_finalize", "loss_l1", "densify", "depth_sort",
                                           "chunk_hist", "chunk_scan", "bucket_emit", "bin_coop", "sgrad_clear",
                                           "loss_count", "loss_finalize", "render_pose_tiles"};
    return (id >= 0 && id < KID_COUNT) ? names[id] : "unknown";
}

const char* gs_status_string(gs_status st) {
    switch (st) {
        case GS_OK: return "GS_OK";
        case GS_ERR_INVALID_ARG: return "GS_ERR_INVALID_ARG";
        case GS_ERR_CAPACITY: return "GS_ERR_CAPACITY";
        case GS_ERR_STALE: return "GS_ERR_STALE";
        case GS_ERR_CUDA: return "GS_ERR_CUDA";
        case GS_ERR_UNSUPPORTED: return "GS_ERR_UNSUPPORTED";
    }
    return "GS_ERR_UNKNOWN";
}

const char* gs_last_cuda_error(void) { return g_last_cuda_error.c_str(); }

}  // extern "C"
