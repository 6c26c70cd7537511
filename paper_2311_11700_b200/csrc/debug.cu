// Debug-build checks (libgs_debug.so, compiled with -DGS_DEBUG=1). compute-sanitizer
// is not available on this pool's boxes, so the debug library verifies the invariants of every
// stage's outputs after the call, on the caller's stream, and turns a violation into GS_ERR_CUDA
// with a message naming the check:
//   gs_project     records finite for every Gaussian with radius > 0; rect inside the tile grid and
//                  tiles == its area
//   gs_bin_sort    ranges[t] = [start, end) with start <= end <= K; every listed value < n; list
//                  starts consistent (each non-empty range begins where the previous non-empty ended)
//   gs_render_fwd  colour / depth / alpha finite, alpha in [0, 1]; per-tile live counts <= the tile's
//                  list length
//   backward       gradients finite over [rows][n]; the pose twist finite
// The release library compiles none of this (the entry points call it only #if GS_DEBUG).
#include "gs_internal.cuh"

#include <cstdio>

namespace gs {

enum : unsigned { DBG_REC = 1u, DBG_RECT = 2u, DBG_RANGE = 4u, DBG_VAL = 8u, DBG_IMG = 16u, DBG_LIVE = 32u,
                  DBG_GRAD = 64u, DBG_POSE = 128u };

__device__ __forceinline__ bool finite(float v) { return isfinite(v); }

__device__ void flag(unsigned* f, unsigned bit, const char* what, long long i) {
    const unsigned old = atomicOr(f, bit);
    if (!(old & bit)) printf("[gs debug] %s violated at %lld\n", what, i);
}

__global__ void dbg_project_kernel(const float4* rec, const short4* rect, const int32_t* radius, const uint32_t* tiles,
                                   int64_t n, int GX, int GY, unsigned* f) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        if (radius[i] <= 0) continue;
        const float4 a = rec[3 * i], b = rec[3 * i + 1], c = rec[3 * i + 2];
        if (!(finite(a.x) && finite(a.y) && finite(a.z) && finite(a.w) && finite(b.x) && finite(b.y) && finite(b.z) &&
              finite(c.x) && finite(c.y) && finite(c.z)))
            flag(f, DBG_REC, "record finite", i);
        const short4 r = rect[i];
        if (r.x < 0 || r.y > GX || r.z < 0 || r.w > GY || r.x > r.y || r.z > r.w ||
            tiles[i] != uint32_t(r.y - r.x) * uint32_t(r.w - r.z))
            flag(f, DBG_RECT, "rect in grid, tiles == area", i);
    }
}

__global__ void dbg_bins_kernel(const uint2* ranges, int T, const uint32_t* vals, const unsigned long long* K_eff,
                                int64_t n, unsigned* f) {
    const unsigned long long K = *K_eff;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < T; t += gridDim.x * blockDim.x) {
        const uint2 r = ranges[t];
        if (r.x > r.y || r.y > K) flag(f, DBG_RANGE, "range start <= end <= K", t);
    }
    for (unsigned long long j = blockIdx.x * blockDim.x + threadIdx.x; j < K; j += gridDim.x * blockDim.x)
        if (vals[j] >= uint64_t(n)) flag(f, DBG_VAL, "listed value < n", (long long)j);
}

__global__ void dbg_fwd_kernel(const float* color, const float* depth, const float* alpha, int64_t npx,
                               const uint2* ranges, const uint32_t* live_cnt, int T, unsigned* f) {
    for (int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < npx; p += int64_t(gridDim.x) * blockDim.x) {
        const float a = alpha[p];
        if (!(finite(color[p]) && finite(color[npx + p]) && finite(color[2 * npx + p]) && finite(depth[p]) &&
              a >= 0.f && a <= 1.f))
            flag(f, DBG_IMG, "image finite, alpha in [0,1]", p);
    }
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < T; t += gridDim.x * blockDim.x)
        if (live_cnt[t] > ranges[t].y - ranges[t].x) flag(f, DBG_LIVE, "live count <= list length", t);
}

__global__ void dbg_grad_kernel(const float* grad, int rows, int64_t n, int64_t ld, const double* pose, unsigned* f) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        for (int k = 0; k < rows; ++k)
            if (!finite(grad[k * ld + i])) flag(f, DBG_GRAD, "gradient finite", k * n + i);
    if (pose && blockIdx.x == 0 && threadIdx.x < 6 && !isfinite(pose[threadIdx.x]))
        flag(f, DBG_POSE, "pose twist finite", threadIdx.x);
}

static gs_status dbg_collect(WsState* s, cudaStream_t st, const char* stage) {
    unsigned* f = &at<Misc>(s, s->misc)->debug_flag;
    unsigned h = 0;
    cudaError_t e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = cudaMemcpy(&h, f, sizeof(h), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) {
        set_cuda_error(e, stage);
        return GS_ERR_CUDA;
    }
    if (h) {
        char msg[160];
        snprintf(msg, sizeof(msg), "%s: debug check failed (flags 0x%x)", stage, h);
        set_error_text(msg);
        cudaMemset(f, 0, sizeof(unsigned));
        return GS_ERR_CUDA;
    }
    return GS_OK;
}

static int dbg_blocks(int64_t items) { return int(std::max<int64_t>(1, std::min<int64_t>((items + 255) / 256, 1024))); }

gs_status dbg_after_project(WsState* s, cudaStream_t st) {
    unsigned* f = &at<Misc>(s, s->misc)->debug_flag;
    if (s->n > 0)
        dbg_project_kernel<<<dbg_blocks(s->n), 256, 0, st>>>(at<float4>(s, s->rec), at<short4>(s, s->rect),
                                                             at<int32_t>(s, s->radius), at<uint32_t>(s, s->tiles), s->n,
                                                             s->cam_gx, s->cam_gy, f);
    return dbg_collect(s, st, "gs_project");
}

gs_status dbg_after_bin_sort(WsState* s, cudaStream_t st) {
    Misc* m = at<Misc>(s, s->misc);
    const int T = s->cam_gx * s->cam_gy;
    const uint32_t* vals = s->sorted_in_1 ? at<uint32_t>(s, s->vals1) : at<uint32_t>(s, s->vals0);
    dbg_bins_kernel<<<dbg_blocks(std::max<int64_t>(T, s->key_cap)), 256, 0, st>>>(at<uint2>(s, s->ranges), T, vals,
                                                                                  &m->n_keys_eff, s->n, &m->debug_flag);
    return dbg_collect(s, st, "gs_bin_sort");
}

gs_status dbg_after_fwd(WsState* s, cudaStream_t st, const float* color, const float* depth, const float* alpha) {
    const int64_t npx = int64_t(s->cam_w) * s->cam_h;
    const int T = s->cam_gx * s->cam_gy;
    dbg_fwd_kernel<<<dbg_blocks(npx), 256, 0, st>>>(color, depth, alpha, npx, at<uint2>(s, s->ranges),
                                                    at<uint32_t>(s, s->live_cnt), T, &at<Misc>(s, s->misc)->debug_flag);
    return dbg_collect(s, st, "gs_render_fwd");
}

gs_status dbg_after_bwd(WsState* s, cudaStream_t st, const float* grad, int64_t n, int64_t ld, const double* pose) {
    if (grad || pose)
        dbg_grad_kernel<<<dbg_blocks(n), 256, 0, st>>>(grad, grad ? (s->sh_degree == 1 ? 23 : 14) : 0, grad ? n : 0, ld,
                                                       pose, &at<Misc>(s, s->misc)->debug_flag);
    return dbg_collect(s, st, "backward");
}

}  // namespace gs
