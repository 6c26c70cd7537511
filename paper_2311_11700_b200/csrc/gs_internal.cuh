// Internal declarations of libgs (B200 / sm_100a). Not part of the ABI; see include/gs.h.
#pragma once
#include <atomic>

#include <cuda_runtime.h>
#include <utility>
#include <stdint.h>

#include "../../include/gs.h"
#include <nvtx3/nvToolsExt.h>   // header-only NVTX 3: ranges cost a few ns unless a profiler attaches

namespace gs {
// NVTX range per ABI call (nsys / ncu --nvtx timelines name the library's stages)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace gs
#define GS_NVTX(name) ::gs::NvtxRange gs_nvtx_range_(name)

namespace gs {

constexpr int kTile = 16;                 // 16x16 pixel tiles (north_star)
constexpr int kTilePx = kTile * kTile;    // 256 pixels = 256 threads per tile CTA
constexpr int kRecFloats = 12;            // projected record: 3 x float4 (48 B)
constexpr int kChunk = 256;               // path B: depth-ordered Gaussians per emission chunk
constexpr int kCoopGridMax = 256;         // path B: CTAs of bin_coop_kernel (one per SM)
constexpr int kCoopBins = 512;            // path B: depth-sort digit bins (<= 9-bit digits)
constexpr int kCoopPasses = 4;            // path B: depth-sort passes at most (ceil(32 / 9))
constexpr int kCoopSegs = 32;             // path B: chunk segments per tile in the tile scans

// ------------------------------------------------------------------ workspace (host state)
struct Region { uint64_t off, bytes; };

struct WsState {
    uint64_t magic;
    char* dev;
    uint64_t dev_bytes;
    int64_t n_cap, key_cap;
    int32_t W, H, GX, GY;          // capacity image size and tile grid
    // carve
    Region rec, depth_key, rect, radius, tiles, offsets, sgrad, scan_state,
        keys0, keys1, vals0, vals1, ranges, t_final, n_last, examined, sort_hist, sort_look,
        misc, scratch, cmp, dkey_sorted, dval_sorted, chunk_hist, chunk_mat, srect, tile_tot, pose_part,
        onlist, live_cnt, svals, coop, tile_order, tile_pose;
    // run state
    int64_t n;                     // Gaussians of the last gs_project
    int32_t sh_degree;             // colour model of the last gs_project_sh (0 = RGB, 1 = degree-1 SH)
    int32_t opacity_radius;        // last gs_project_ex used GS_FLAG_OPACITY_RADIUS (reading C33)
    int32_t pad_sh;
    int32_t cam_w, cam_h, cam_gx, cam_gy;   // image of the last gs_project
    uint64_t gen_project, gen_fwd; // generation counters (GS_ERR_STALE)
    uint64_t gen_bwd;              // gen_fwd of the last gs_render_bwd / gs_pose_grad
    uint64_t gen_screen;           // gen_fwd whose screen gradients the workspace holds (tile pass done)
    int32_t sorted_in_1;           // final sorted keys/vals live in buffer 1
    int32_t keys_valid;            // path A materialised the 64-bit keys (view.keys valid)
    int64_t n_keys_host;           // K of the last host-synced gs_bin_sort (-1 unknown)
    int64_t launches;              // kernels launched (gs_ws_launch_count)
    int64_t max_parts;             // sort lookback partitions per pass
    uint64_t epoch;                // look-back epoch (scan and sort status words)
    // optional per-kernel event log (gs_ws_set_event_log)
    void** ev;                     // 2*ev_cap caller-created cudaEvent_t
    int32_t* ev_ids;               // kernel id per logged launch
    int32_t ev_cap, ev_n;
};
static_assert(sizeof(WsState) <= sizeof(gs_ws), "WsState must fit in gs_ws");
constexpr uint64_t kMagic = 0x67735F62323030ull;   // "gs_b200"

inline WsState* state(gs_ws* ws) { return reinterpret_cast<WsState*>(ws); }
inline const WsState* state(const gs_ws* ws) { return reinterpret_cast<const WsState*>(ws); }
template <class T> inline T* at(const WsState* s, const Region& r) { return reinterpret_cast<T*>(s->dev + r.off); }

// misc region layout (device scalars)
struct Misc {
    unsigned long long n_keys;     // K
    unsigned long long n_keys_eff; // K if K <= key_cap else 0 (what sort / ranges / render consume)
    unsigned int error_flag;
    unsigned int scan_counter;
    unsigned int sort_counter[8];  // per-pass partition counters
    unsigned int n_onscreen;       // path B: Gaussians with tiles > 0
    unsigned int coop_bar;         // path B: grid-barrier arrivals of bin_coop_kernel (zeroed per call)
    unsigned long long n_items;    // path B: items of the depth sort (= V_s)
    unsigned int kmin_inv;         // path B: ~min and max of the on-screen depth keys (atomicMax, zeroed)
    unsigned int kmax;
    unsigned int coop_pad[2];
    double loss_acc[4];            // |C-C*| sum, |D-D*| valid sum, valid count, spare
    double pose_acc[16];
    unsigned long long add_count;  // densify
    unsigned long long keep_count;
    unsigned int chunk_counter;
    unsigned int pose_done;        // gaussian_bwd last-block ticket (self-resetting)
    unsigned int prep_done;        // bwd_prep_kernel last-block ticket (self-resetting)
    unsigned int tile_pose_done;   // pose-only tile pass last-block ticket (self-resetting)
    unsigned int debug_flag;       // debug builds: violated checks (debug.cu), cleared when reported
    unsigned int gbwd_zero_chunk;  // gaussian_bwd: off-screen zeroing chunks claimed (reset by the bwd prologue)
};

// Programmatic dependent launch (PDL): kernels of the iteration are launched with programmatic
// stream serialisation, so a kernel's CTAs can be scheduled while its predecessor's last wave drains;
// each such kernel waits (griddepcontrol.wait) before touching anything, so data dependencies are
// exactly those of plain stream order. Without the attribute the wait is a no-op.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Grid barrier for cooperative launches (all CTAs co-resident): block barrier, one thread fences and
// arrives on a monotone counter (zeroed before the launch), spins on an acquire load.
__device__ __forceinline__ void grid_sync(unsigned int* bar, unsigned int& goal) {
    __syncthreads();
    if (threadIdx.x == 0) {
        goal += gridDim.x;
        __threadfence();
        atomicAdd(bar, 1u);
        unsigned int v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
        } while (v < goal);
    }
    __syncthreads();
}
__device__ __forceinline__ void st_release_u32(unsigned int* p, unsigned int v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// Zero `bytes` (a multiple of 4, 4-byte aligned) on stream st with a small kernel rather than
// cudaMemsetAsync: inside the iteration's CUDA graph a memset node measured ~3 us slower per
// iteration than a kernel node (optim.cu)
void launch_zero(void* p, size_t bytes, cudaStream_t st, WsState* s = nullptr);   // s: counts the launch
// debug library (-DGS_DEBUG=1): output invariant checks after each stage (debug.cu)
void set_error_text(const char* msg);
gs_status dbg_after_project(WsState* s, cudaStream_t st);
gs_status dbg_after_bin_sort(WsState* s, cudaStream_t st);
gs_status dbg_after_fwd(WsState* s, cudaStream_t st, const float* color, const float* depth, const float* alpha);
gs_status dbg_after_bwd(WsState* s, cudaStream_t st, const float* grad, int64_t n, int64_t ld, const double* pose);
#ifndef GS_DEBUG
#define GS_DEBUG 0
#endif

int coop_sm_count();   // SMs of the current device (cached per device; multiProcessorCount)
inline int sm_count() { const int v = coop_sm_count(); return v > 0 ? v : 148; }

// Per-device one-time initialisation: kernel attributes (max dynamic shared memory, carveout) are
// per device, so a process using several GPUs sets them once on each. A bitmask of done devices,
// updated atomically (the tracking and mapping threads of slam.py launch concurrently; setting an
// attribute twice is harmless).
struct PerDeviceOnce {
    std::atomic<unsigned long long> done{0ull};
    template <class F> bool run(F&& f) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return false;
        const unsigned long long bit = 1ull << dev;
        if (done.load(std::memory_order_acquire) & bit) return true;
        if (!f()) return false;
        done.fetch_or(bit, std::memory_order_acq_rel);
        return true;
    }
};

// ------------------------------------------------------------------ launch helpers
// Kernel ids for the event log; names in gs_kernel_name (abi.cu). Keep in sync.
enum KernelId {
    KID_PROJECT = 0, KID_SCAN, KID_EMIT, KID_SORT_HIST, KID_SORT_DSCAN, KID_SORT_PASS, KID_RANGES,
    KID_FWD, KID_BWD_TILE, KID_BWD_GAUSS, KID_POSE_FIN, KID_LOSS, KID_DENSIFY,
    KID_DEPTH_SORT, KID_CHUNK_HIST, KID_CHUNK_SCAN, KID_BUCKET_EMIT, KID_BIN_COOP, KID_SGRAD_CLEAR,
    KID_LOSS_COUNT, KID_LOSS_FINALIZE, KID_POSE_TILE, KID_COUNT
};

// RAII bracket around one kernel launch: counts it and, when an event log is attached, records
// an event before and after it on the launching stream.
struct KTimer {
    WsState* s;
    cudaStream_t st;
    bool on;
    KTimer(WsState* s_, int kid, cudaStream_t st_) : s(s_), st(st_), on(false) {
        if (s && s->ev && s->ev_n < s->ev_cap) {
            on = true;
            s->ev_ids[s->ev_n] = kid;
            cudaEventRecord(static_cast<cudaEvent_t>(s->ev[2 * s->ev_n]), st);
        }
    }
    ~KTimer() {
        if (!s) return;
        s->launches += 1;
        if (on) {
            cudaEventRecord(static_cast<cudaEvent_t>(s->ev[2 * s->ev_n + 1]), st);
            s->ev_n += 1;
        }
    }
};

gs_status check_launch(WsState* s, const char* what);
void set_cuda_error(cudaError_t e, const char* what);

// kernels-side entry points (defined in the .cu files; host wrappers)
void launch_project(WsState* s, const float* params, int64_t n, int64_t ld, const uint8_t* mask,
                    const float* viewmat, const gs_camera& cam, cudaStream_t st);   // colour: s->sh_degree
gs_status run_bin_sort_keys(WsState* s, int64_t* n_keys, uint32_t flags, cudaStream_t st);
gs_status run_compact_onscreen(WsState* s, cudaStream_t st);   // path A
gs_status run_bin_sort_bucket(WsState* s, int64_t* n_keys, uint32_t flags, cudaStream_t st);
void launch_render_fwd(WsState* s, const gs_camera& cam, float* color, float* depth, float* alpha,
                       float* accum_weight, uint32_t flags, cudaStream_t st);
void launch_zero_sgrad(WsState* s, cudaStream_t st, const float* td_l1 = nullptr, int64_t npx = 0, bool clear = true);
struct L1Fuse {   // gs_render_bwd_l1: the L1 loss formed inside the backward's pixel loads
    const float *color, *depth, *tc, *td;
    float wc, wd;
    double* loss;    // nullable
};
void launch_render_bwd_tiles(WsState* s, const gs_camera& cam, const float* color_unused,
                             const float* dL_dcolor, const float* dL_ddepth, cudaStream_t st,
                             const L1Fuse* fuse = nullptr, bool finalize_loss = true, int mode = 0,
                             double* grad_pose = nullptr, int assign = 0);
struct LossFin {   // the fused L1 loss scalar, written by gaussian_bwd's last block (loss == nullptr: none)
    const double* acc;
    double* loss;
    float wc, wd;
    int64_t npx;
};
void launch_gaussian_bwd(WsState* s, const float* params, int64_t n, int64_t ld, const float* viewmat,
                         const gs_camera& cam, float* grad_params, double* grad_pose, uint32_t flags,
                         cudaStream_t st, LossFin lf = LossFin{nullptr, nullptr, 0.f, 0.f, 0});
void launch_loss_l1(WsState* s, const float* color, const float* depth, const float* tc, const float* td,
                    int32_t W, int32_t H, float wc, float wd, float* dc, float* dd, double* loss, cudaStream_t st);
void launch_loss_l1_masked(WsState* s, const float* color, const float* depth, const float* tc, const float* td,
                           const float* alpha, float amin, float outlier_k, int32_t W, int32_t H, float wc, float wd,
                           float* dc, float* dd, double* loss, cudaStream_t st);
void launch_frame_stats(const float* alpha, const float* depth, const float* td, int32_t W, int32_t H, float ta,
                        float tdep, uint32_t* counts, cudaStream_t st);
void launch_pose_extrapolate(const float* t1, const float* t2, float* out, cudaStream_t st);
void launch_image_half(const float* c, const float* d, int32_t W, int32_t H, float* ch, float* dh, cudaStream_t st);
void launch_adam(float* raw, float* act, const float* g, float* m, float* v, int64_t n, int64_t ld, const float* lr,
                 int32_t rows, int32_t step, float b1, float b2, float eps, cudaStream_t st);
void launch_pose_step(float* viewmat, const double* gp, float* m6, float* v6, int32_t step, float lr_rho,
                      float lr_phi, cudaStream_t st);
void launch_append(float* params, float* raw, float* m, float* v, int64_t* n_dev, int64_t capacity, int64_t ld,
                   const float* cand, const int64_t* counts, int32_t n_sets, int64_t max_add, int32_t rows,
                   cudaStream_t st);
void launch_accum_grad(WsState* s, float* grad_accum, float* count, cudaStream_t st);
gs_status run_split_clone(WsState* s, float* params, float* raw, float* m, float* v, int64_t* n_dev, int64_t capacity,
                          int64_t ld, float* grad_accum, float* count, const float* noise, float grad_thresh,
                          float scale_thresh, int32_t rows, cudaStream_t st);
gs_status run_densify(WsState* s, float* params, float* raw, int64_t* n_dev, int64_t capacity, int64_t ld,
                      float* m, float* v, const float* alpha, const float* depth, const float* trgb,
                      const float* tdepth, const float* accum, const float* viewmat, const gs_camera& cam,
                      const gs_densify_cfg& cfg, uint8_t* select_mask, float* add_out, cudaStream_t st);

// ------------------------------------------------------------------ device helpers
__device__ __forceinline__ float4 ldg4(const float4* p) { return __ldg(p); }

// Packed fp32 pairs (sm_100 FADD2 / FMUL2 / FFMA2): one issue slot for two IEEE round-to-nearest
// operations, each bit-identical to its scalar __fadd_rn / __fmul_rn / __fmaf_rn. The render kernels
// keep two pixels per thread, so every per-pixel operation comes in pairs; a per-Gaussian scalar
// operand is a broadcast pair, which ptxas encodes as a plain register (no extra move).
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pk2(float lo, float hi) {
    f32x2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ f32x2 bc2(float v) { return pk2(v, v); }
__device__ __forceinline__ float lo2(f32x2 v) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
    return lo;
}
__device__ __forceinline__ float hi2(f32x2 v) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
    return hi;
}
__device__ __forceinline__ f32x2 add2(f32x2 a, f32x2 b) {
    f32x2 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f32x2 sub2(f32x2 a, f32x2 b) {
    f32x2 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) {
    f32x2 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
    f32x2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

// Projected record (48 B): r0 = {mx, my, A, B}, r1 = {C, o, depth, q_max}, r2 = {r, g, b, rank} (rank:
// the on-screen rank as uint bits, written by gs_bin_sort's compaction; indexes the backward's screen
// accumulators) with the
// exactly scaled conic A = -a/2, B = -b, C = -c/2 (conic = Sigma'^-1 = [[a, b], [b, c]]).
// alpha at pixel (px, py). Shared by the forward and both backward kernels so every decision is
// bit-identical between them, and written with explicit round-to-nearest intrinsics in the
// oracle's fp32 order (reading R1): power = fma(A dx, dx, fma(C dy, dy, (B dx) dy)).
// For elongated conics the terms cancel, so any other order would move power by many ulps and
// flip alpha-vs-1/255 decisions. Returns alpha (0 when skipped), G and the 0.99-clamp flag.
struct AlphaEval { float alpha, G, dx, dy; bool clamped; };

__device__ __forceinline__ AlphaEval eval_alpha(float4 r0, float4 r1, float px, float py) {
    AlphaEval e;
    e.dx = __fsub_rn(r0.x, px);
    e.dy = __fsub_rn(r0.y, py);
    const float inner = __fmaf_rn(__fmul_rn(r1.x, e.dy), e.dy, __fmul_rn(__fmul_rn(r0.w, e.dx), e.dy));
    const float power = __fmaf_rn(__fmul_rn(r0.z, e.dx), e.dx, inner);
    // G = exp(power) via ex2.approx (MUFU): power * log2(e)
    float G;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(G) : "f"(__fmul_rn(power, 1.4426950408889634f)));
    const float og = __fmul_rn(r1.y, G);
    e.G = G;
    e.clamped = og > 0.99f;
    float a = fminf(0.99f, og);
    if (power > 0.f || a < (1.0f / 255.0f)) a = 0.f;   // skipped: contributes nothing
    e.alpha = a;
    return e;
}

}  // namespace gs
