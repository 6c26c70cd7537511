// gs_render_fwd / gs_render_bwd / gs_pose_grad kernels (sm_100a).
//
// Forward (Eq. 4-5): one 256-thread CTA per 16x16 tile, one pixel per thread.
// The tile's sorted Gaussian indices are gathered 256 records (48 B each) at a time into shared
// memory with cp.async (LDGSTS; the records are an index gather, so a TMA tensor copy does not
// apply), double-buffered against the blend of the previous batch.
//
// Backward, front to back: with e_i = c_i.dL/dC + d_i dL/dD, Q = colour.dL/dC +
// depth.dL/dD (forward outputs incl. T_f bg) and the running prefix P_i = sum_{k<=i} alpha_k T_k e_k,
//     dL/dalpha_i = T_i e_i - (Q - P_i) / (1 - alpha_i)
// which equals Eq. S6 plus its colour/background analogue. T_i is recomputed
// front to back with the forward's exact fp32 operations, so no transmittance is recovered by
// division. Per 32-Gaussian batch: phase 1 (thread = pixel) writes (alpha T, G dL/dalpha) to shared
// memory; phase 2 (warp = 32 pixels, lane = Gaussian) accumulates the 10 per-Gaussian sums as
// pixel moments; the 8 warps' partials are combined in shared memory and each (tile, Gaussian)
// issues one atomic per component (warp/block reduction before global atomics, north_star).
#include <cub/block/block_reduce.cuh>

#include "gs_internal.cuh"

namespace gs {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N> __device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ------------------------------------------------------------------ forward
constexpr int kFwdBatch = 256;

template <bool kAccum>
__global__ void __launch_bounds__(kTilePx) render_fwd_kernel(
    const float4* __restrict__ rec, const uint32_t* __restrict__ vals, const uint2* __restrict__ ranges, int W, int H,
    int GX, float bgr, float bgg, float bgb, float* __restrict__ color, float* __restrict__ depth,
    float* __restrict__ alpha, float* __restrict__ t_final, uint32_t* __restrict__ n_last, uint32_t* __restrict__ examined,
    float* __restrict__ accum_weight) {
    __shared__ float4 s_rec[2][kFwdBatch][3];
    const int tile = blockIdx.x;
    const int tx = tile % GX, ty = tile / GX;
    const int lx = threadIdx.x & 15, ly = threadIdx.x >> 4;
    const int px = tx * kTile + lx, py = ty * kTile + ly;
    const bool inside = px < W && py < H;
    const float fpx = float(px), fpy = float(py);
    const uint2 rg = ranges[tile];
    const uint32_t start = rg.x, len = rg.y - rg.x;
    const int nbatch = int((len + kFwdBatch - 1) / kFwdBatch);

    float T = 1.f, Cr = 0.f, Cg = 0.f, Cb = 0.f, D = 0.f;
    uint32_t nl = 0, exam = len;
    bool done = !inside;

    auto stage = [&](int b) {
        const uint32_t j = uint32_t(b) * kFwdBatch + threadIdx.x;
        if (j < len) {
            const uint32_t g = vals[start + j];
            float4* dst = s_rec[b & 1][threadIdx.x];
            const float4* src = rec + 3 * size_t(g);
            cp_async16(dst + 0, src + 0);
            cp_async16(dst + 1, src + 1);
            cp_async16(dst + 2, src + 2);
        }
        cp_async_commit();
    };
    if (nbatch > 0) stage(0);
    for (int b = 0; b < nbatch; ++b) {
        if (b + 1 < nbatch) {
            stage(b + 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const int cnt = min(kFwdBatch, int(len) - b * kFwdBatch);
        const float4(*buf)[3] = s_rec[b & 1];
        if (!kAccum) {
            if (!done) {
                for (int k = 0; k < cnt; ++k) {
                    const float4 r0 = buf[k][0], r1 = buf[k][1];
                    const AlphaEval e = eval_alpha(r0, r1, fpx, fpy);
                    if (e.alpha == 0.f) continue;
                    const float Tn = __fmul_rn(T, __fsub_rn(1.f, e.alpha));
                    if (Tn < 1e-4f) {
                        done = true;
                        exam = uint32_t(b * kFwdBatch + k + 1);
                        break;
                    }
                    const float4 r2 = buf[k][2];
                    const float w = __fmul_rn(e.alpha, T);
                    Cr = fmaf(w, r2.x, Cr);
                    Cg = fmaf(w, r2.y, Cg);
                    Cb = fmaf(w, r2.z, Cb);
                    D = fmaf(w, r1.z, D);
                    T = Tn;
                    nl = uint32_t(b * kFwdBatch + k + 1);
                }
            }
        } else {
            for (int k = 0; k < cnt; ++k) {   // warp-uniform trip count: shuffles below are safe
                float w = 0.f;
                if (!done) {
                    const float4 r0 = buf[k][0], r1 = buf[k][1];
                    const AlphaEval e = eval_alpha(r0, r1, fpx, fpy);
                    if (e.alpha != 0.f) {
                        const float Tn = __fmul_rn(T, __fsub_rn(1.f, e.alpha));
                        if (Tn < 1e-4f) {
                            done = true;
                            exam = uint32_t(b * kFwdBatch + k + 1);
                        } else {
                            const float4 r2 = buf[k][2];
                            w = __fmul_rn(e.alpha, T);
                            Cr = fmaf(w, r2.x, Cr);
                            Cg = fmaf(w, r2.y, Cg);
                            Cb = fmaf(w, r2.z, Cb);
                            D = fmaf(w, r1.z, D);
                            T = Tn;
                            nl = uint32_t(b * kFwdBatch + k + 1);
                        }
                    }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
                if ((threadIdx.x & 31) == 0 && w != 0.f) atomicAdd(accum_weight + vals[start + b * kFwdBatch + k], w);
            }
        }
        if (__syncthreads_and(done)) break;   // also orders buffer reuse
    }
    if (inside) {
        const size_t pix = size_t(py) * W + px, plane = size_t(W) * H;
        const float cr = fmaf(T, bgr, Cr), cg = fmaf(T, bgg, Cg), cb = fmaf(T, bgb, Cb);
        color[pix] = cr;
        color[plane + pix] = cg;
        color[2 * plane + pix] = cb;
        depth[pix] = D;
        alpha[pix] = 1.f - T;
        t_final[pix] = T;
        n_last[pix] = nl;
        if (examined) examined[pix] = exam;
    }
}

void launch_render_fwd(WsState* s, const gs_camera& cam, float* color, float* depth, float* alpha,
                       float* accum_weight, uint32_t flags, cudaStream_t st) {
    const int ntiles = s->cam_gx * s->cam_gy;
    const uint32_t* sorted_vals = s->sorted_in_1 ? at<uint32_t>(s, s->vals1) : at<uint32_t>(s, s->vals0);
    uint32_t* exam = (flags & GS_FLAG_EXAMINED) ? at<uint32_t>(s, s->examined) : nullptr;
    if (ntiles == 0) return;
    KTimer kt(s, KID_FWD, st);
    if ((flags & GS_FLAG_ACCUM_WEIGHT) && accum_weight) {
        render_fwd_kernel<true><<<ntiles, kTilePx, 0, st>>>(
            at<float4>(s, s->rec), sorted_vals, at<uint2>(s, s->ranges), cam.width, cam.height, s->cam_gx, cam.bg[0],
            cam.bg[1], cam.bg[2], color, depth, alpha, at<float>(s, s->t_final), at<uint32_t>(s, s->n_last), exam,
            accum_weight);
    } else {
        render_fwd_kernel<false><<<ntiles, kTilePx, 0, st>>>(
            at<float4>(s, s->rec), sorted_vals, at<uint2>(s, s->ranges), cam.width, cam.height, s->cam_gx, cam.bg[0],
            cam.bg[1], cam.bg[2], color, depth, alpha, at<float>(s, s->t_final), at<uint32_t>(s, s->n_last), exam,
            nullptr);
    }
}

// ------------------------------------------------------------------ backward, tile pass
constexpr int kBwdBatch = 32;
constexpr int kWarps = kTilePx / 32;

struct BwdSmem {
    float4 rec[2][kBwdBatch][3];
    float w[kTilePx][kBwdBatch + 1];    // alpha_i T_i     (padded: conflict-free row writes)
    float go[kTilePx][kBwdBatch + 1];   // G dL/dalpha_i    (0 when clamped or skipped)
    float4 dl[kTilePx];                 // dL/dC (r,g,b), dL/dD per pixel
    float part[kWarps][10][kBwdBatch];  // per-warp partial sums
    uint32_t idx[2][kBwdBatch];
    uint32_t max_nl;
};

__global__ void __launch_bounds__(kTilePx, 2) render_bwd_kernel(
    const float4* __restrict__ rec, const uint32_t* __restrict__ vals, const uint2* __restrict__ ranges, int W, int H,
    int GX, const float* __restrict__ t_final, float bgr, float bgg, float bgb, const uint32_t* __restrict__ n_last,
    const float* __restrict__ dLdC, const float* __restrict__ dLdD, float* __restrict__ sgrad, int64_t sld) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    BwdSmem& sm = *reinterpret_cast<BwdSmem*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int tile = blockIdx.x;
    const int tx = tile % GX, ty = tile / GX;
    const int lx = tid & 15, ly = tid >> 4;
    const int px = tx * kTile + lx, py = ty * kTile + ly;
    const bool inside = px < W && py < H;
    const float fpx = float(px), fpy = float(py);
    const uint2 rg = ranges[tile];
    const uint32_t start = rg.x;
    const size_t pix = size_t(py) * W + px, plane = size_t(W) * H;

    uint32_t nl = 0;
    float4 dl = make_float4(0.f, 0.f, 0.f, 0.f);
    float T = 1.f;   // T_{i+1} while walking back; starts at T_final
    if (inside) {
        nl = n_last[pix];
        dl = make_float4(dLdC[pix], dLdC[plane + pix], dLdC[2 * plane + pix], dLdD[pix]);
        T = t_final[pix];
    }
    const float tfb = T * (bgr * dl.x + bgg * dl.y + bgb * dl.z);   // T_f bg . dL/dC
    if (tid == 0) sm.max_nl = 0;
    sm.dl[tid] = dl;
    __syncthreads();
    if (nl) atomicMax(&sm.max_nl, nl);
    __syncthreads();
    const uint32_t len = sm.max_nl;
    const int nbatch = int((len + kBwdBatch - 1) / kBwdBatch);

    // batch bb holds list positions [bb*32, bb*32+32); batches are visited back to front
    auto stage = [&](int bb, int slot) {
        if (tid < kBwdBatch) {
            const uint32_t j = uint32_t(bb) * kBwdBatch + tid;
            if (j < len) {
                const uint32_t g = vals[start + j];
                sm.idx[slot][tid] = g;
                float4* dst = sm.rec[slot][tid];
                const float4* src = rec + 3 * size_t(g);
                cp_async16(dst + 0, src + 0);
                cp_async16(dst + 1, src + 1);
                cp_async16(dst + 2, src + 2);
            }
        }
        cp_async_commit();
    };

    float S = 0.f;   // sum_{k>i} alpha_k T_k e_k  (suffix sum, accumulated from the back)
    if (nbatch > 0) stage(nbatch - 1, 0);
    for (int it = 0; it < nbatch; ++it) {
        const int bb = nbatch - 1 - it;
        if (it + 1 < nbatch) {
            stage(bb - 1, (it + 1) & 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const int buf = it & 1;
        const int cnt = min(kBwdBatch, int(len) - bb * kBwdBatch);
        // ---- phase 1: thread = pixel, back to front over the batch (3DGS-style recurrence):
        //      T_i = T_{i+1} / (1 - alpha_i);  dL/dalpha_i = T_i e_i - (S_i + T_f bg.dL/dC) / (1 - alpha_i)
#pragma unroll 4
        for (int k = kBwdBatch - 1; k >= 0; --k) {
            float w = 0.f, go = 0.f;
            const uint32_t jpos = uint32_t(bb * kBwdBatch + k + 1);
            if (k < cnt && jpos <= nl) {
                const float4 r0 = sm.rec[buf][k][0], r1 = sm.rec[buf][k][1];
                const AlphaEval e = eval_alpha(r0, r1, fpx, fpy);
                if (e.alpha != 0.f) {
                    const float4 r2 = sm.rec[buf][k][2];
                    const float ev = fmaf(r2.x, dl.x, fmaf(r2.y, dl.y, fmaf(r2.z, dl.z, r1.z * dl.w)));
                    const float ro = __frcp_rn(__fsub_rn(1.f, e.alpha));
                    T = T * ro;
                    w = e.alpha * T;
                    const float ga = fmaf(T, ev, -(S + tfb) * ro);
                    go = e.clamped ? 0.f : e.G * ga;
                    S = fmaf(w, ev, S);
                }
            }
            sm.w[tid][k] = w;
            sm.go[tid][k] = go;
        }
        __syncthreads();
        // ---- phase 2: warp = 32 pixels, lane = Gaussian; pixel moments
        {
            float S0 = 0.f, Sx = 0.f, Sy = 0.f, Sxx = 0.f, Sxy = 0.f, Syy = 0.f, Sr = 0.f, Sg = 0.f, Sb = 0.f, Sd = 0.f;
#pragma unroll 8
            for (int p = 0; p < 32; ++p) {
                const int q = warp * 32 + p;
                const float fx = float(q & 15), fy = float(q >> 4);
                const float g = sm.go[q][lane], w = sm.w[q][lane];
                const float4 d = sm.dl[q];
                S0 += g;
                Sx = fmaf(g, fx, Sx);
                Sy = fmaf(g, fy, Sy);
                Sxx = fmaf(g, fx * fx, Sxx);
                Sxy = fmaf(g, fx * fy, Sxy);
                Syy = fmaf(g, fy * fy, Syy);
                Sr = fmaf(w, d.x, Sr);
                Sg = fmaf(w, d.y, Sg);
                Sb = fmaf(w, d.z, Sb);
                Sd = fmaf(w, d.w, Sd);
            }
            float* pp = &sm.part[warp][0][lane];
            pp[0 * kBwdBatch] = S0; pp[1 * kBwdBatch] = Sx; pp[2 * kBwdBatch] = Sy; pp[3 * kBwdBatch] = Sxx;
            pp[4 * kBwdBatch] = Sxy; pp[5 * kBwdBatch] = Syy; pp[6 * kBwdBatch] = Sr; pp[7 * kBwdBatch] = Sg;
            pp[8 * kBwdBatch] = Sb; pp[9 * kBwdBatch] = Sd;
        }
        __syncthreads();
        // ---- combine the 8 warps; convert moments to screen-space gradients; one atomic each
        if (tid < cnt) {
            float Mo[10];   // pixel moments of this Gaussian over the tile
#pragma unroll
            for (int c = 0; c < 10; ++c) {
                float a = 0.f;
#pragma unroll
                for (int w2 = 0; w2 < kWarps; ++w2) a += sm.part[w2][c][tid];
                Mo[c] = a;
            }
            const float4 r0 = sm.rec[buf][tid][0], r1 = sm.rec[buf][tid][1];
            const float o = r1.y;
            const float X = r0.x - float(tx * kTile), Y = r0.y - float(ty * kTile);
            // sum g dx, sum g dy, sum g dx^2, sum g dx dy, sum g dy^2 with dx = X - lx, dy = Y - ly
            const float gdx = X * Mo[0] - Mo[1];
            const float gdy = Y * Mo[0] - Mo[2];
            const float gdxx = X * X * Mo[0] - 2.f * X * Mo[1] + Mo[3];
            const float gdxy = X * Y * Mo[0] - X * Mo[2] - Y * Mo[1] + Mo[4];
            const float gdyy = Y * Y * Mo[0] - 2.f * Y * Mo[2] + Mo[5];
            const float ca = r0.z, cb = r0.w, cc = r1.x;
            float out[10];
            out[0] = -o * (ca * gdx + cb * gdy);   // mean2d x
            out[1] = -o * (cb * gdx + cc * gdy);   // mean2d y
            out[2] = -0.5f * o * gdxx;             // conic a
            out[3] = -o * gdxy;                    // conic b
            out[4] = -0.5f * o * gdyy;             // conic c
            out[5] = Mo[0];                        // opacity
            out[6] = Mo[6];
            out[7] = Mo[7];
            out[8] = Mo[8];                        // rgb
            out[9] = Mo[9];                        // depth
            const uint32_t g = sm.idx[buf][tid];
#pragma unroll
            for (int c = 0; c < 10; ++c)
                if (out[c] != 0.f) atomicAdd(sgrad + c * sld + g, out[c]);
        }
        __syncthreads();   // protect sm.part / w / go / rec[buf] before the next batch
    }
}

void launch_render_bwd_tiles(WsState* s, const gs_camera& cam, const float*, const float* dL_dcolor,
                             const float* dL_ddepth, cudaStream_t st) {
    const int ntiles = s->cam_gx * s->cam_gy;
    if (ntiles == 0) return;
    const uint32_t* sorted_vals = s->sorted_in_1 ? at<uint32_t>(s, s->vals1) : at<uint32_t>(s, s->vals0);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(render_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(BwdSmem)));
        attr = true;
    }
    KTimer kt(s, KID_BWD_TILE, st);
    render_bwd_kernel<<<ntiles, kTilePx, sizeof(BwdSmem), st>>>(
        at<float4>(s, s->rec), sorted_vals, at<uint2>(s, s->ranges), cam.width, cam.height, s->cam_gx,
        at<float>(s, s->t_final), cam.bg[0], cam.bg[1], cam.bg[2], at<uint32_t>(s, s->n_last), dL_dcolor, dL_ddepth,
        at<float>(s, s->sgrad), s->n_cap);
}

// ------------------------------------------------------------------ backward, per-Gaussian chain
// Screen-space gradients -> the 14 parameters (Eq. 11 / Supplement A) and the pose twist.
// pose partial sums: rho(3), phi(3), dW_cov(9)  (reading C7: A = W (sum dW_cov)^T).
constexpr int kPoseSums = 15;

__global__ void __launch_bounds__(256) gaussian_bwd_kernel(
    const float* __restrict__ params, int64_t n, int64_t ld, const float* __restrict__ viewmat, gs_camera cam,
    const uint32_t* __restrict__ tiles, const float4* __restrict__ rec, const float* __restrict__ sgrad, int64_t sld,
    float* __restrict__ grad, int cov_path, double* __restrict__ pose_acc) {
    __shared__ float V[12];
    if (threadIdx.x < 12) V[threadIdx.x] = viewmat[threadIdx.x];
    __syncthreads();
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    float pose[kPoseSums];
#pragma unroll
    for (int k = 0; k < kPoseSums; ++k) pose[k] = 0.f;
    if (i < n && tiles[i] > 0) {
        float s[10];
#pragma unroll
        for (int c = 0; c < 10; ++c) s[c] = sgrad[c * sld + i];
        float p[14];
#pragma unroll
        for (int k = 0; k < 14; ++k) p[k] = params[k * ld + i];
        const float W[3][3] = {{V[0], V[1], V[2]}, {V[4], V[5], V[6]}, {V[8], V[9], V[10]}};
        float Xc[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) Xc[a] = W[a][0] * p[0] + W[a][1] * p[1] + W[a][2] * p[2] + V[4 * a + 3];
        const float x = Xc[0], y = Xc[1], z = Xc[2];
        const float iz = 1.f / z, iz2 = iz * iz;
        const float nq = sqrtf(p[6] * p[6] + p[7] * p[7] + p[8] * p[8] + p[9] * p[9]);
        const float qr = p[6] / nq, qi = p[7] / nq, qj = p[8] / nq, qk = p[9] / nq;
        const float R[3][3] = {{1.f - 2.f * (qj * qj + qk * qk), 2.f * (qi * qj - qr * qk), 2.f * (qi * qk + qr * qj)},
                               {2.f * (qi * qj + qr * qk), 1.f - 2.f * (qi * qi + qk * qk), 2.f * (qj * qk - qr * qi)},
                               {2.f * (qi * qk - qr * qj), 2.f * (qj * qk + qr * qi), 1.f - 2.f * (qi * qi + qj * qj)}};
        float M[3][3], S[3][3];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int k = 0; k < 3; ++k) M[a][k] = R[a][k] * p[3 + k];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) S[a][b] = M[a][0] * M[b][0] + M[a][1] * M[b][1] + M[a][2] * M[b][2];
        const float J[2][3] = {{cam.fx * iz, 0.f, -cam.fx * x * iz2}, {0.f, cam.fy * iz, -cam.fy * y * iz2}};
        float E[2][3];
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int k = 0; k < 3; ++k) E[a][k] = J[a][0] * W[0][k] + J[a][1] * W[1][k] + J[a][2] * W[2][k];
        // conic -> Sigma':  dSp = -Q Gbar Q
        const float4 r0 = rec[3 * i], r1 = rec[3 * i + 1];
        const float Q[2][2] = {{r0.z, r0.w}, {r0.w, r1.x}};
        const float Gb[2][2] = {{s[2], 0.5f * s[3]}, {0.5f * s[3], s[4]}};
        float QG[2][2], dSp[2][2];
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int b = 0; b < 2; ++b) QG[a][b] = Q[a][0] * Gb[0][b] + Q[a][1] * Gb[1][b];
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int b = 0; b < 2; ++b) dSp[a][b] = -(QG[a][0] * Q[0][b] + QG[a][1] * Q[1][b]);
        // dSigma = E^T dSp E ; dE = 2 dSp E Sigma
        float dSE[2][3];   // dSp E
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int k = 0; k < 3; ++k) dSE[a][k] = dSp[a][0] * E[0][k] + dSp[a][1] * E[1][k];
        float dS[3][3];
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
            for (int l = 0; l < 3; ++l) dS[k][l] = E[0][k] * dSE[0][l] + E[1][k] * dSE[1][l];
        float dE[2][3];
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int l = 0; l < 3; ++l) dE[a][l] = 2.f * (dSE[a][0] * S[0][l] + dSE[a][1] * S[1][l] + dSE[a][2] * S[2][l]);
        // E = J W: dJ = dE W^T ; dW_cov = J^T dE
        float dJ[2][3];
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) dJ[a][b] = dE[a][0] * W[b][0] + dE[a][1] * W[b][1] + dE[a][2] * W[b][2];
        const float iz3 = iz2 * iz;
        const float dXJ[3] = {dJ[0][2] * (-cam.fx * iz2), dJ[1][2] * (-cam.fy * iz2),
                              dJ[0][0] * (-cam.fx * iz2) + dJ[0][2] * (2.f * cam.fx * x * iz3) +
                                  dJ[1][1] * (-cam.fy * iz2) + dJ[1][2] * (2.f * cam.fy * y * iz3)};
        const float dXm[3] = {J[0][0] * s[0], J[1][1] * s[1], J[0][2] * s[0] + J[1][2] * s[1] + s[9]};
        const float dX[3] = {dXm[0] + dXJ[0], dXm[1] + dXJ[1], dXm[2] + dXJ[2]};
        if (grad) {
            // mean: W^T dX
#pragma unroll
            for (int k = 0; k < 3; ++k) grad[k * ld + i] += W[0][k] * dX[0] + W[1][k] * dX[1] + W[2][k] * dX[2];
            // Sigma = M M^T
            float dM[3][3];
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int k = 0; k < 3; ++k) dM[a][k] = 2.f * (dS[a][0] * M[0][k] + dS[a][1] * M[1][k] + dS[a][2] * M[2][k]);
#pragma unroll
            for (int k = 0; k < 3; ++k) grad[(3 + k) * ld + i] += dM[0][k] * R[0][k] + dM[1][k] * R[1][k] + dM[2][k] * R[2][k];
            float dR[3][3];
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int k = 0; k < 3; ++k) dR[a][k] = dM[a][k] * p[3 + k];
            // Eq. S1 derivatives
            float dq[4];
            dq[0] = 2.f * (-qk * dR[0][1] + qj * dR[0][2] + qk * dR[1][0] - qi * dR[1][2] - qj * dR[2][0] + qi * dR[2][1]);
            dq[1] = 2.f * (qj * dR[0][1] + qk * dR[0][2] + qj * dR[1][0] - 2.f * qi * dR[1][1] - qr * dR[1][2] +
                           qk * dR[2][0] + qr * dR[2][1] - 2.f * qi * dR[2][2]);
            dq[2] = 2.f * (-2.f * qj * dR[0][0] + qi * dR[0][1] + qr * dR[0][2] + qi * dR[1][0] + qk * dR[1][2] -
                           qr * dR[2][0] + qk * dR[2][1] - 2.f * qj * dR[2][2]);
            dq[3] = 2.f * (-2.f * qk * dR[0][0] - qr * dR[0][1] + qi * dR[0][2] + qr * dR[1][0] - 2.f * qk * dR[1][1] +
                           qj * dR[1][2] + qi * dR[2][0] + qj * dR[2][1]);
            const float qd = dq[0] * qr + dq[1] * qi + dq[2] * qj + dq[3] * qk;
            grad[6 * ld + i] += (dq[0] - qr * qd) / nq;
            grad[7 * ld + i] += (dq[1] - qi * qd) / nq;
            grad[8 * ld + i] += (dq[2] - qj * qd) / nq;
            grad[9 * ld + i] += (dq[3] - qk * qd) / nq;
            grad[10 * ld + i] += s[5];
            grad[11 * ld + i] += s[6];
            grad[12 * ld + i] += s[7];
            grad[13 * ld + i] += s[8];
        }
        if (pose_acc) {
            const float* g = cov_path ? dX : dXm;
            pose[0] = g[0];
            pose[1] = g[1];
            pose[2] = g[2];
            pose[3] = y * g[2] - z * g[1];
            pose[4] = z * g[0] - x * g[2];
            pose[5] = x * g[1] - y * g[0];
            if (cov_path) {
#pragma unroll
                for (int a = 0; a < 3; ++a)
#pragma unroll
                    for (int b = 0; b < 3; ++b) pose[6 + 3 * a + b] = J[0][a] * dE[0][b] + J[1][a] * dE[1][b];
            }
        }
    }
    if (pose_acc) {
        using BR = cub::BlockReduce<double, 256>;
        __shared__ typename BR::TempStorage tmp;
#pragma unroll 1
        for (int k = 0; k < kPoseSums; ++k) {
            const double v = BR(tmp).Sum(double(pose[k]));
            if (threadIdx.x == 0 && v != 0.0) atomicAdd(pose_acc + k, v);
            __syncthreads();
        }
    }
}

// twist = (rho, phi + (A12 - A21, A20 - A02, A01 - A10)),  A = W (sum dW_cov)^T
__global__ void pose_finalize_kernel(const double* __restrict__ acc, const float* __restrict__ viewmat,
                                     double* __restrict__ grad_pose) {
    if (threadIdx.x != 0) return;
    double W[3][3], A[3][3];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) W[a][b] = viewmat[4 * a + b];
    const double* dW = acc + 6;
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) A[a][b] = W[a][0] * dW[3 * b + 0] + W[a][1] * dW[3 * b + 1] + W[a][2] * dW[3 * b + 2];
    grad_pose[0] += acc[0];
    grad_pose[1] += acc[1];
    grad_pose[2] += acc[2];
    grad_pose[3] += acc[3] + (A[1][2] - A[2][1]);
    grad_pose[4] += acc[4] + (A[2][0] - A[0][2]);
    grad_pose[5] += acc[5] + (A[0][1] - A[1][0]);
}

void launch_gaussian_bwd(WsState* s, const float* params, int64_t n, int64_t ld, const float* viewmat,
                         const gs_camera& cam, float* grad_params, double* grad_pose, uint32_t flags, cudaStream_t st) {
    if (n == 0) return;
    Misc* misc = at<Misc>(s, s->misc);
    double* acc = grad_pose ? misc->pose_acc : nullptr;
    if (acc) cudaMemsetAsync(misc->pose_acc, 0, sizeof(misc->pose_acc), st);
    const int blocks = int((n + 255) / 256);
    {
    KTimer kt(s, KID_BWD_GAUSS, st);
    gaussian_bwd_kernel<<<blocks, 256, 0, st>>>(params, n, ld, viewmat, cam, at<uint32_t>(s, s->tiles),
                                                at<float4>(s, s->rec), at<float>(s, s->sgrad), s->n_cap, grad_params,
                                                (flags & GS_FLAG_POSE_COV_PATH) ? 1 : 0, acc);
    }
    if (grad_pose) {
        KTimer kt(s, KID_POSE_FIN, st);
        pose_finalize_kernel<<<1, 32, 0, st>>>(acc, viewmat, grad_pose);
    }
}

}  // namespace gs
