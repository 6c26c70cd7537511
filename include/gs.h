/* gs.h — C ABI of the B200 differentiable RGB-D Gaussian-splatting renderer (GS-SLAM hot path,
 * arXiv 2311.11700). Library: paper_2311_11700_b200/libgs.so (sm_100a).
 *
 * Conventions (all entry points)
 *  - Pointers are CUDA DEVICE pointers unless marked (host).
 *  - Every call is asynchronous on `stream` (a cudaStream_t passed as void*; NULL = legacy default
 *    stream) and never allocates device memory. The caller owns every buffer, including the
 *    device workspace and the host workspace state `gs_ws` (see gs_ws_init).
 *  - The library holds no global device state; calls on distinct workspaces are independent. Its only
 *    process-wide state is a per-device host cache of kernel attributes and SM counts (thread-safe).
 *  - Argument errors are detected on the host before any launch (GS_ERR_INVALID_ARG);
 *    a failed launch returns GS_ERR_CUDA (gs_last_cuda_error() gives the CUDA error string).
 *  - Gaussian parameters are ACTIVATED values in a structure-of-arrays float32 buffer
 *    params[14][ld] (row k at params + k*ld), columns 0..n-1:
 *      rows 0-2  mean X (world, metres)                    Eq. 1 "position X_i"
 *      rows 3-5  scale s (linear, > 0)                      Eq. 2 "S"
 *      rows 6-9  rotation quaternion (r,i,j,k), raw; normalised inside gs_project
 *      row  10   opacity Lambda in (0,1)                    Eq. 1
 *      rows 11-13 RGB colour (SH degree 0, "light" model)
 *    Gradients are returned with respect to these 14 activated values.
 *  - viewmat: float[12] row-major 3x4 WORLD->CAMERA [W | t] (reading C1: X^c = W X + t,
 *    PAPER.md:626). It is a device pointer so CUDA graphs can update the pose in place.
 *  - Images are planar float32: colour [3][H][W], depth / alpha [H][W]; pixel (u,v) has its
 *    centre at integer coordinates (reading C12).
 *  - Pose gradients are a left-perturbation twist (rho, phi): T <- exp(delta^) T (reading C1/C7).
 */
#ifndef GS_H_
#define GS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    GS_OK = 0,
    GS_ERR_INVALID_ARG = 1,
    GS_ERR_CAPACITY = 2,     /* key or Gaussian capacity exceeded; required size reported */
    GS_ERR_STALE = 3,        /* backward on a workspace whose last forward does not match */
    GS_ERR_CUDA = 4,
    GS_ERR_UNSUPPORTED = 5
} gs_status;

/* Pinhole camera + render settings (host struct). */
typedef struct {
    float fx, fy, cx, cy;    /* intrinsics K */
    int32_t width, height;   /* image size; width*height <= the workspace's W*H */
    float znear;             /* near-plane cull, metres (reading C13: 0.2) */
    float bg[3];             /* background colour (reading C15: black) */
    float cov2d_dilation;    /* added to the diagonal of Sigma' (reading C11: 0.3 px^2) */
} gs_camera;

/* Host-side workspace state: opaque, caller-allocated, initialised by gs_ws_init. */
typedef struct { uint64_t opaque[128]; } gs_ws;

enum {
    GS_FLAG_POSE_COV_PATH = 1u,   /* include dSigma'/dpose in pose gradients (reading C7; exact, FD-parity
                                     default). Off = the paper's approximation */
    GS_FLAG_NO_HOST_SYNC = 2u,    /* gs_bin_sort: do not read K back; grids sized from key_cap, K stays on
                                     the device; overflow sets the device error flag (CUDA-graph mode) */
    GS_FLAG_ACCUM_WEIGHT = 4u,    /* gs_render_fwd: accumulate per-Gaussian sum_px alpha*T (Eq. 12 select) */
    GS_FLAG_EXAMINED = 8u,        /* gs_render_fwd: write the per-pixel examined count (for E_f) */
    GS_FLAG_BINSORT_KEYS = 16u,   /* gs_bin_sort: emit 64-bit (tile|depth) keys and onesweep-sort them
                                     (north_star literal path); default = depth-presort + tile bucketing
                                     (bit-identical lists, fewer HBM bytes) */
    GS_FLAG_GRAD_ASSIGN = 32u,    /* gs_render_bwd / gs_pose_grad: ASSIGN instead of accumulate: every column
                                     [0, n) of grad_params is written (zero for off-screen Gaussians) and
                                     grad_pose = the pose gradient; no zeroing pass needed by the caller */
    GS_FLAG_OPACITY_RADIUS = 64u, /* gs_project_ex: opacity-aware radius (reading C33) */
    GS_FLAG_BINSORT_EMIT_ONLY = 256u, /* testing: with GS_FLAG_BINSORT_KEYS, stop after key emission (the
                                     view's keys/vals then hold the unsorted index-order emission) */
    GS_FLAG_BWD_SCREEN_ONLY = 512u,   /* gs_render_bwd[_l1]: the tile pass only: screen-space gradients into
                                     the workspace (and the fused L1 loss); grad_params / grad_pose untouched */
    GS_FLAG_BWD_CHAIN_ONLY = 1024u    /* gs_render_bwd[_l1]: the per-Gaussian chain only, from the screen
                                     gradients a SCREEN_ONLY call left for the same forward (else
                                     GS_ERR_STALE): grad_params / grad_pose as a full call. The two halves
                                     let a caller order the accumulating halves of several workspaces'
                                     backward passes while their tile passes overlap */
};

/* ---------------------------------------------------------------------------------------------
 * Workspace. Device bytes needed for up to n_cap Gaussians, key_cap (tile, Gaussian) keys and
 * images up to W x H pixels. gs_ws_init carves `dev` (>= gs_workspace_bytes, 256-B aligned) and
 * fills the host state. Ownership stays with the caller; the library never frees.
 * Errors: GS_ERR_INVALID_ARG on non-positive sizes, misalignment or too few bytes.
 * ------------------------------------------------------------------------------------------- */
size_t gs_workspace_bytes(int64_t n_cap, int64_t key_cap, int32_t W, int32_t H);
gs_status gs_ws_init(gs_ws* ws /*(host)*/, void* dev, size_t dev_bytes, int64_t n_cap, int64_t key_cap,
                     int32_t W, int32_t H);

/* gs_project — Eq. 2-3, O1: per Gaussian i < n
 *   X^c = W X + t; cull unless z^c > znear; q_hat = q/|q|; R(q_hat) by Eq. S1;
 *   Sigma = R diag(s)^2 R^T; Sigma' = (J W) Sigma (J W)^T + dil I with the affine-projection
 *   Jacobian J; conic = Sigma'^-1; radius r = ceil(3 sqrt(lambda_max)); mean m = (fx x/z + cx,
 *   fy y/z + cy); 16x16-tile rect of the 3-sigma box; depth d = z^c (Eq. 5 text).
 * mask: optional u8[n]; mask[i] == 0 culls Gaussian i (coarse-to-fine selection, Eq. 12).
 * Writes the projected records into the workspace (consumed by gs_bin_sort / gs_render_*).
 * Culling is a value, not an error (radius 0, no tiles). Bit-exact with the oracle on depth key,
 * radius, rect and tile count (fixed fp32 operation order, no FMA contraction). */
gs_status gs_project(const float* params, int64_t n, int64_t ld, const uint8_t* mask /*nullable*/,
                     const float* viewmat, const gs_camera* cam /*(host)*/, gs_ws* ws, void* stream);

/* gs_project_sh — gs_project with the colour model selected by sh_degree:
 *   0: params [14][ld], rows 11-13 = RGB (reading C17; identical to gs_project);
 *   1: params [23][ld], rows 11 + 3k + c = degree-1 SH coefficient k of channel c ("1-degree
 *      spherical harmonics per colour channel, a total of 12 coefficients"). The
 *      colour is evaluated per Gaussian at the view direction u = (X - c)/|X - c|, c = -W^T t:
 *      rgb_c = max(0, 1/2 + C0 Y_0c + C1 (-u_y Y_1c + u_z Y_2c - u_x Y_3c)) (reading C29).
 * The degree is kept in the workspace: the following gs_render_bwd / gs_pose_grad use it, and
 * grad_params then has the same row count (14 or 23). Errors: GS_ERR_INVALID_ARG if sh_degree is
 * not 0 or 1, else as gs_project. */
gs_status gs_project_sh(const float* params, int64_t n, int64_t ld, int32_t sh_degree,
                        const uint8_t* mask /*nullable*/, const float* viewmat, const gs_camera* cam /*(host)*/,
                        gs_ws* ws, void* stream);

/* gs_project_ex — gs_project_sh with flags. GS_FLAG_OPACITY_RADIUS replaces the 3-sigma radius by
 * the reach of the alpha >= 1/255 test (PAPER.md:27 skip rule applied to Eq. 4's
 * alpha = o exp(-q/2); reading C33): q_o = fp32(2 ln(255 o)) evaluated in fp64 and rounded once;
 * o <= 1/255 (q_o <= 0) culls the Gaussian (radius 0, no tiles), else r = ceil(sqrt(q_o lambda_max))
 * (fp32, that order), and the rect, tile count and lists follow from r as before. Every pixel where
 * alpha >= 1/255 lies inside the rect, so the tile lists hold exactly the contributing Gaussians
 * and no more; the image differs from the 3-sigma one where the 3-sigma box cuts a Gaussian with
 * o > e^4.5/255 ~ 0.35 short. Other flags: GS_ERR_INVALID_ARG. */
gs_status gs_project_ex(const float* params, int64_t n, int64_t ld, int32_t sh_degree, uint32_t flags,
                        const uint8_t* mask /*nullable*/, const float* viewmat, const gs_camera* cam /*(host)*/,
                        gs_ws* ws, void* stream);

/* gs_bin_sort — tile binning + depth sort ("sorting the Gaussians in depth order", PAPER.md:83;
 * north_star: 64-bit (tile << 32 | depth-bits) keys, 16x16 tiles). Produces, per tile t, the list
 * of Gaussian indices whose rect contains t, ordered by (depth bits, index) — the stable ascending
 * sort of keys emitted in index order (O2) — and ranges[t] = [start, end).
 * n_keys (host, nullable): receives K. If K > key_cap: returns GS_ERR_CAPACITY with the required K
 * in *n_keys (host-sync mode) or sets the device error flag (GS_FLAG_NO_HOST_SYNC). */
gs_status gs_bin_sort(gs_ws* ws, int64_t* n_keys /*(host) out, nullable*/, uint32_t flags, void* stream);

/* gs_render_fwd — Eq. 4-5 and the cumulative opacity of Eq. 8:
 * per pixel, front to back over its tile's list: alpha = min(0.99, o exp(-1/2 d^T Sigma'^-1 d)),
 * skip alpha < 1/255, stop before the Gaussian that would take T below 1e-4 (reading C9);
 * colour = sum c_i alpha_i T_i + T_final bg, depth = sum d_i alpha_i T_i, alpha = 1 - T_final.
 * accum_weight: float[n] (+=) per-Gaussian sum of alpha_i T_i, written iff GS_FLAG_ACCUM_WEIGHT.
 * Keeps T_final and the last-contributor position per pixel in the workspace for the backward. */
gs_status gs_render_fwd(gs_ws* ws, const gs_camera* cam /*(host)*/, float* color, float* depth, float* alpha,
                        float* accum_weight /*nullable*/, uint32_t flags, void* stream);

/* gs_render_bwd — analytic backward of the last gs_render_fwd on this workspace (Eq. 11,
 * PAPER.md:155-168; Supplement A, PAPER.md:608-749 incl. Eq. S6): given dL/dcolor [3][H][W] and
 * dL/ddepth [H][W], ACCUMULATES (+=) dL/dparams into grad_params[14][ld] and, if grad_pose is
 * non-NULL, dL/d(rho, phi) into grad_pose[6] (fp64); with GS_FLAG_GRAD_ASSIGN both are assigned
 * instead (off-screen columns set to 0). params/viewmat must be those of the forward.
 * Returns GS_ERR_STALE if gs_project ran after the last gs_render_fwd or n changed. */
gs_status gs_render_bwd(const float* params, int64_t n, int64_t ld, const float* viewmat, gs_ws* ws,
                        const gs_camera* cam /*(host)*/, const float* dL_dcolor, const float* dL_ddepth,
                        float* grad_params /*[14][ld], +=*/, double* grad_pose /*nullable [6], +=*/,
                        uint32_t flags, void* stream);

/* gs_render_bwd_l1 — gs_loss_l1 followed by gs_render_bwd in one pass over the pixels: the L1 loss
 * of Eq. 6 (reading C20: L = w_c/(3HW) sum|C - C*| + w_d/#valid sum_valid|D - D*|)
 * is formed inside the backward's pixel loads (dL/dC = w_c/(3HW) sign(C - C*), dL/dD = w_d/#valid
 * sign(D - D*) on valid pixels: the same fp32 values gs_loss_l1 writes), so dL/dC, dL/dD are never
 * written to memory. color [3][H][W], depth [H][W] are the last gs_render_fwd's outputs; loss
 * (nullable, device fp64 [1]) receives L. Other arguments, flags and errors as gs_render_bwd. */
gs_status gs_render_bwd_l1(const float* params, int64_t n, int64_t ld, const float* viewmat, gs_ws* ws,
                           const gs_camera* cam /*(host)*/, const float* color, const float* depth,
                           const float* tgt_color, const float* tgt_depth, float w_color, float w_depth,
                           float* grad_params, double* grad_pose /*nullable*/, double* loss /*nullable*/,
                           uint32_t flags, void* stream);

/* gs_pose_grad — pose-only backward (Eq. 11; supplement P:626-729; tracking, Alg. 1
 * PAPER.md:774-800): same inputs as gs_render_bwd, ACCUMULATES dL/d(rho, phi)
 * into grad_pose[6] (GS_FLAG_GRAD_ASSIGN: overwrites); no per-Gaussian outputs.
 *   Paper mode (no GS_FLAG_POSE_COV_PATH; P:168 drops Sigma' through the pose): ONE tile pass. Per
 *   (tile, Gaussian) only the mean and depth sums (3 pixel moments + the depth sum) are formed and
 *   turned into dL/dX^c = J^T dL/dm + e_z dL/dd with J and X^c rebuilt from the projected record;
 *   rho += dL/dX^c, phi += X^c x dL/dX^c in fp64; per-tile partials are reduced in a fixed order by the
 *   last tile block. No screen-space atomics, no per-Gaussian pass.
 *   Covariance path (exact gradient, reading C7): a tile pass keeping the 6 quantities the chain
 *   reads (mean, conic, depth; all 10 for degree-1 SH, whose colour reaches the pose through the
 *   camera centre), then the per-Gaussian chain writing only the pose partials.
 * Errors as gs_render_bwd. */
gs_status gs_pose_grad(const float* params, int64_t n, int64_t ld, const float* viewmat, gs_ws* ws,
                       const gs_camera* cam /*(host)*/, const float* dL_dcolor, const float* dL_ddepth,
                       double* grad_pose /*[6] (rho_xyz, phi_xyz), +=*/, uint32_t flags, void* stream);

/* gs_pose_grad_l1 — gs_loss_l1 fused into gs_pose_grad (as gs_render_bwd_l1 fuses it into the full
 * backward): dL/dC, dL/dD of Eq. 6 (reading C20) are formed in the pose pass' pixel loads and never
 * written; loss (nullable, device fp64 [1]) receives L. color, depth: the last gs_render_fwd's
 * outputs. Other arguments, flags and errors as gs_pose_grad. */
gs_status gs_pose_grad_l1(const float* params, int64_t n, int64_t ld, const float* viewmat, gs_ws* ws,
                          const gs_camera* cam /*(host)*/, const float* color, const float* depth,
                          const float* tgt_color, const float* tgt_depth, float w_color, float w_depth,
                          double* grad_pose /*[6], +=*/, double* loss /*nullable*/, uint32_t flags, void* stream);

/* gs_loss_l1 — Eq. 6 as means (reading C20):
 *   L = w_c/(3HW) sum|C - C*| + w_d/#valid sum_{D*>0}|D - D*|
 * writes dL/dC = w_c/(3HW) sign(C - C*) (sign(0) = 0), dL/dD likewise on valid pixels, and
 * loss[0] = L (fp64, device). */
gs_status gs_loss_l1(const float* color, const float* depth, const float* tgt_color, const float* tgt_depth,
                     int32_t W, int32_t H, float w_color, float w_depth, float* dL_dcolor, float* dL_ddepth,
                     double* loss /*[1]*/, gs_ws* ws, void* stream);

/* gs_adam_step — Adam (betas/eps = b1,b2,eps) over params_raw[14][ld] (raw space:
 * rows 3-5 log-scale, row 10 logit-opacity, others identity) with per-row learning rates lr[14]
 * (host), using gradients w.r.t. the ACTIVATED values (chain rule fused) and bias correction at
 * `step` (1-based). Also writes the activated copy params_act[14][ld]. m, v: [14][ld]. */
gs_status gs_adam_step(float* params_raw, float* params_act, const float* grad_act, float* m, float* v,
                       int64_t n, int64_t ld, const float lr[14] /*(host)*/, int32_t step, float b1, float b2,
                       float eps, void* stream);

/* gs_adam_step_rows — gs_adam_step over `rows` parameter rows: 14 (RGB, identical to gs_adam_step)
 * or 23 (degree-1 SH, gs_project_sh's layout): rows 3-5 log-scale, row 10
 * logit-opacity, every other row (mean, quaternion, colour / SH coefficients) identity. lr: host
 * float[rows]. Other row counts: GS_ERR_INVALID_ARG. */
gs_status gs_adam_step_rows(float* params_raw, float* params_act, const float* grad_act, float* m, float* v,
                            int64_t n, int64_t ld, int32_t rows, const float* lr /*(host) [rows]*/, int32_t step,
                            float b1, float b2, float eps, void* stream);

/* gs_pose_step — Adam on the pose twist (reading C23; "FusedAdam" PAPER.md:954) then
 * T <- exp(delta^) T applied to viewmat in place (device-only, no host sync). m6, v6: float[6]. */
gs_status gs_pose_step(float* viewmat, const double* grad_pose, float* m6, float* v6, int32_t step,
                       float lr_rho, float lr_phi, void* stream);

/* gs_pose_extrapolate — constant-velocity initialisation of a new frame's pose ("transforms the last
 * known pose based on the relative transformation between the second-to-last pose and the last pose",
 * PAPER.md:147): with world->camera poses T1 (second-to-last) and T2 (last),
 * out = (T2 T1^-1) T2, computed in fp64 on the device. All three are device float[12] (3x4 row-major);
 * out may alias neither input. */
gs_status gs_pose_extrapolate(const float* view_prev2, const float* view_prev, float* view_out, void* stream);

/* gs_image_half — the coarse stage's H/2 x W/2 target ("a coarse image with resolution
 * H/2 x W/2"; reading C12's camera: half pixel (u, v) covers full pixels 2u..2u+1 x 2v..2v+1):
 * colour_half = ((c00 + c01) + (c10 + c11)) * 0.25 per channel (fp32, that order), depth_half = the
 * mean of the valid (> 0) depths among the four in the order 00, 01, 10, 11, or 0 if none. color
 * [3][H][W], depth [H][W] in; color_half [3][H/2][W/2], depth_half [H/2][W/2] out (floor sizes;
 * an odd last row / column is dropped). W, H >= 2, else GS_ERR_INVALID_ARG. */
gs_status gs_image_half(const float* color, const float* depth, int32_t W, int32_t H, float* color_half,
                        float* depth_half, void* stream);

/* gs_frame_stats — the keyframe rule's measurement ("the proportion of the currently
 * observed image's reliable region"): counts[0] = pixels with valid target
 * depth that are reliable by Eq. 8 (alpha >= tau_alpha and |D* - D| <= tau_depth), counts[1] = pixels
 * with valid target depth, counts[2] = pixels with alpha >= tau_alpha (observed). counts: device u32[3],
 * overwritten. */
gs_status gs_frame_stats(const float* alpha, const float* depth, const float* target_depth, int32_t W, int32_t H,
                         float tau_alpha, float tau_depth, uint32_t* counts, void* stream);

/* gs_loss_l1_masked — the tracking loss restricted to previously observed areas ("only rendered at
 * previously observed areas"; reading C31): as gs_loss_l1 over the kept pixels only,
 * the colour mean over those pixels (3 N_kept) and the depth mean over those with valid D*; other
 * pixels get zero gradient. Kept = alpha >= alpha_min (alpha: the render's [H][W] alpha) and, when
 * outlier_k > 0, the outlier rule of PAPER.md:954 ("if the loss on the pixel is more than ten times
 * the median loss, the pixel will be ignored"; reading C32): l_p = (|dC_0| + |dC_1|) + |dC_2| in fp32,
 * m = the lower median of l_p over the alpha-kept pixels, kept iff l_p <= outlier_k * m (fp32).
 * outlier_k = 0 turns the rule off; negative or NaN -> GS_ERR_INVALID_ARG. The outlier path is one
 * cooperative launch (one CTA per SM) that uses the workspace's binning scratch: do not run it
 * concurrently with gs_bin_sort on the same workspace. */
gs_status gs_loss_l1_masked(const float* color, const float* depth, const float* tgt_color, const float* tgt_depth,
                            const float* alpha, float alpha_min, float outlier_k, int32_t W, int32_t H, float w_color,
                            float w_depth, float* dL_dcolor, float* dL_ddepth, double* loss /*[1]*/, gs_ws* ws,
                            void* stream);

/* gs_densify_prune — adaptive expansion (Sec. 3.2) and selection (Eq. 12):
 *  GS_DENSIFY_ADD    Eq. 8: pixel unreliable iff alpha < tau_alpha or |D* - D| > tau_depth, with
 *                    D* > 0 and (u+v) % stride == 0, in pixel order; back-projected at D* through
 *                    the inverse pose; init rgb = C*, opacity = init_opacity, quat (1,0,0,0),
 *                    scale = D* stride/(fx+fy) (reading C22). Appended at columns [n, n+added) of
 *                    params (and logit/log in params_raw, zero moments); n_dev updated; at most
 *                    max_add and capacity - n. If add_out != NULL the candidates are instead written
 *                    to add_out[14][max_add] (activated) and *n_dev RECEIVES their count (<= max_add)
 *                    (multi-GPU gather mode; see gs_densify_append).
 *  GS_DENSIFY_PRUNE  drop Gaussians with opacity < min_opacity by stable compaction of params,
 *                    params_raw, adam_m, adam_v (any of the last three may be NULL); n_dev updated.
 *  GS_DENSIFY_SELECT Eq. 12 (reading C24): select_mask[i] = accum_weight[i] > sel_weight and
 *                    |D*(round m_i) - d_i| < sel_depth, using the last gs_project on this ws.
 *  GS_DENSIFY_DEGENERATE  Eq. 9 (reading C27): every
 *                    Gaussian visible in the last gs_project on this ws (tiles > 0) whose centre
 *                    pixel round(m_i) is inside the image with valid D* > 0 and lies in front of
 *                    the observed surface by more than gamma (D* - d_i > gamma, fp32) has its
 *                    opacity scaled: o_i <- eta o_i (params row 10; params_raw row 10 <- logit of
 *                    the new opacity if params_raw != NULL; Adam moments unchanged). select_mask
 *                    (nullable) receives the per-Gaussian flag. The map size is unchanged.
 *  GS_DENSIFY_DEGENERATE_FLAG  the same test, but only ORed into select_mask (select_mask[i] = 1 for
 *                    every flagged Gaussian, others untouched; params may be NULL and are not
 *                    changed): the per-keyframe half of a multi-keyframe / multi-GPU degeneration
 *                    (mapping.py: flags of all keyframes, max-all-reduced over ranks, then APPLY).
 *  GS_DENSIFY_DEGENERATE_APPLY  o_i <- eta o_i for every i < n with select_mask[i] != 0 (params
 *                    row 10; params_raw row 10 <- logit if non-NULL). No projection needed.
 * n_dev: device int64 [1] (in/out). All compaction is deterministic. */
enum { GS_DENSIFY_ADD = 1, GS_DENSIFY_PRUNE = 2, GS_DENSIFY_SELECT = 3, GS_DENSIFY_DEGENERATE = 4,
       GS_DENSIFY_DEGENERATE_FLAG = 5, GS_DENSIFY_DEGENERATE_APPLY = 6 };
typedef struct {
    int32_t mode;
    float tau_alpha, tau_depth, min_opacity, sel_weight, sel_depth, init_opacity;
    int32_t stride;
    int64_t max_add;
    float eta, gamma;        /* DEGENERATE: opacity factor (0.1) and floater margin in metres (0.10) */
    int32_t rows;            /* parameter rows: 0 or 14 = RGB, 23 = degree-1 SH (ADD writes the colour as
                                the DC coefficient (c - 1/2)/C0 and zero linear terms, reading C34; PRUNE
                                compacts all rows; other values: GS_ERR_INVALID_ARG) */
} gs_densify_cfg;
gs_status gs_densify_prune(float* params, float* params_raw /*nullable*/, int64_t* n_dev, int64_t capacity,
                           int64_t ld, float* adam_m /*nullable*/, float* adam_v /*nullable*/, const float* alpha,
                           const float* depth, const float* target_rgb, const float* target_depth,
                           const float* accum_weight, const float* viewmat, const gs_camera* cam /*(host)*/,
                           const gs_densify_cfg* cfg /*(host)*/, uint8_t* select_mask, float* add_out,
                           gs_ws* ws, void* stream);

/* gs_densify_accum_grad — densification statistics (3DGS adaptive density control, which the paper
 * uses for "splits large points into smaller ones and clones them"; reading C30):
 * for every on-screen Gaussian i of the last gs_render_bwd on ws,
 *   grad_accum[i] += |(dL/dm_x W/2, dL/dm_y H/2)|  (the screen-space mean gradient in NDC units),
 *   count[i] += 1.
 * grad_accum, count: device float[>= n]. Errors: GS_ERR_STALE without a backward since the last
 * forward. */
gs_status gs_densify_accum_grad(gs_ws* ws, float* grad_accum, float* count, void* stream);

/* gs_densify_split_clone — one densification step (every 10 mapping iterations before the 70th,
 * thresholds 0.002 and 0.02 m; reading C30) over params[rows][ld] columns [0, n)
 * (rows 14, or 23 for degree-1 SH: children copy the SH rows):
 * avg_i = grad_accum_i / count_i (0 if count_i == 0); i is a candidate iff avg_i >= grad_thresh;
 * a candidate with max scale <= scale_thresh is CLONED (a copy appended), otherwise SPLIT: two
 * children X + R(q) diag(s) eps_k, k = 0, 1 (eps_k = noise rows 3k..3k+2 at column i, N(0,1) drawn by
 * the caller), scale s / 1.6, the other parameters copied, are appended and the original removed.
 * Result order: the kept originals (index order), then the clones (index order), then the children
 * (index order, child 0 then child 1). Appends beyond capacity are dropped (clones first; a split
 * is applied only if both children fit). Appended Gaussians get raw copies (log scale, logit
 * opacity) and zero Adam moments; grad_accum and count are reset to 0 over [0, capacity); n_dev
 * updated. Deterministic. noise: device float[6][ld]. */
gs_status gs_densify_split_clone(float* params, float* params_raw /*nullable*/, float* adam_m /*nullable*/,
                                 float* adam_v /*nullable*/, int64_t* n_dev, int64_t capacity, int64_t ld,
                                 float* grad_accum, float* count, const float* noise, float grad_thresh,
                                 float scale_thresh, int32_t rows /*14 or 23*/, gs_ws* ws, void* stream);

/* gs_densify_append — append gathered ADD candidates (multi-GPU mapping):
 * cand[k][rows][max_add] (activated, k < n_sets, in global keyframe order; rows 14 or 23) with
 * counts[k] (device int64) are appended in order k = 0, 1, ... at columns [n, n + sum counts) of params[rows][ld]
 * (raw copies: log-scale / logit-opacity; zero Adam moments), truncated at capacity; n_dev updated.
 * Deterministic: every rank appending the same gathered sets produces identical parameters. */
gs_status gs_densify_append(float* params, float* params_raw /*nullable*/, float* adam_m /*nullable*/,
                            float* adam_v /*nullable*/, int64_t* n_dev, int64_t capacity, int64_t ld,
                            const float* cand, const int64_t* counts, int32_t n_sets, int64_t max_add,
                            int32_t rows /*14 or 23*/, void* stream);

/* Introspection for tests and benchmarks (host struct of device pointers into the workspace). */
typedef struct {
    const float* records;        /* [n][12]: mx, my, -a/2, -b | -c/2, opacity, depth, q_max | r, g, b, pad
                                    (conic [[a, b], [b, c]] = Sigma'^-1, exactly scaled; q_max ~ 2 ln(255 o)
                                    is the tile-reach bound of the forward's live lists) */
    const uint32_t* depth_key;   /* [n] float bits of z^c */
    const int16_t* rect;         /* [n][4] xlo, xhi, ylo, yhi */
    const int32_t* radius;       /* [n] */
    const uint32_t* tiles;       /* [n] tiles touched */
    const uint32_t* offsets;     /* [n] exclusive prefix of tiles (key-emission offsets, GS_FLAG_BINSORT_KEYS) */
    const uint64_t* keys;        /* [K] sorted (tile << 32 | depth key); valid after gs_bin_sort */
    const uint32_t* vals;        /* [K] sorted Gaussian indices */
    const uint32_t* ranges;      /* [GX*GY][2] */
    const float* t_final;        /* [H*W] */
    const uint32_t* n_last;      /* [H*W] 1-based position of the last blended Gaussian (0: none) */
    const uint32_t* examined;    /* [H*W] (GS_FLAG_EXAMINED) */
    const uint64_t* n_keys_dev;  /* [1] K on the device */
    const uint32_t* error_flag;  /* [1] nonzero after a device-side capacity overflow */
    /* live lists written by gs_render_fwd, walked by gs_render_bwd: for tile t, entries
     * [ranges[t][0], ranges[t][0] + live_cnt[t]) hold (Gaussian, 1-based list position) of the
     * list entries that can reach alpha >= 1/255 somewhere in the tile (ascending positions) */
    const uint32_t* live_g;      /* [K] */
    const uint32_t* live_j;      /* [K] */
    const uint32_t* live_cnt;    /* [GX*GY] */
    int64_t n, key_cap, n_cap;
    int32_t grid_x, grid_y, width, height;
} gs_ws_view;
gs_status gs_ws_get_view(const gs_ws* ws, gs_ws_view* out /*(host)*/);

/* Per-launch accounting: number of kernels this library launched on the workspace since init
 * (host counter; bench.py reports it as gpu_launches). */
int64_t gs_ws_launch_count(const gs_ws* ws);

/* Optional per-kernel timing (bench.py roofline). While attached, every kernel launch issued on
 * `ws` is bracketed by cudaEventRecord(events[2k]) / (events[2k+1]) on its stream and its kernel id
 * is stored in ids[k], for k < capacity (later launches are not logged). events: 2*capacity
 * cudaEvent_t (host array, e.g. from gs_events_create); capacity 0 detaches. The caller owns both
 * arrays; read the times with gs_events_elapsed after synchronising. */
gs_status gs_ws_set_event_log(gs_ws* ws, void** events /*(host)*/, int32_t* ids /*(host)*/, int32_t capacity);
int32_t gs_ws_event_log_count(const gs_ws* ws);
gs_status gs_events_create(void** events /*(host) out*/, int32_t count);
gs_status gs_events_destroy(void** events /*(host)*/, int32_t count);
gs_status gs_events_elapsed(void* const* events /*(host)*/, int32_t pairs, float* ms /*(host) out [pairs]*/);
const char* gs_kernel_name(int32_t id);

const char* gs_status_string(gs_status s);
const char* gs_last_cuda_error(void);

#ifdef __cplusplus
}
#endif
#endif /* GS_H_ */
