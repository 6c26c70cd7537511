// gs_render_fwd / gs_render_bwd / gs_pose_grad kernels (sm_100a).
//
// Forward (Eq. 4-5): one CTA per 16x16 tile (render_fwd2_kernel: 128 threads, two
// pixels each). The tile's sorted Gaussian indices are gathered into shared memory with cp.async
// (LDGSTS; the records are an index gather, so a TMA tensor copy does not apply), double-buffered
// against the blend of the previous batch. render_fwd_kernel<true> (one pixel per thread) is the
// GS_FLAG_ACCUM_WEIGHT variant used by the Eq. 12 selection.
//
// Backward, back to front: T_i = T_{i+1} / (1 - alpha_i) from T_final, suffix
// sum S_i = sum_{k>i} alpha_k T_k e_k with e_k = c_k.dL/dC + d_k dL/dD, and
//     dL/dalpha_i = T_i e_i - (S_i + T_f bg.dL/dC) / (1 - alpha_i)
// which is Eq. S6 plus its colour/background analogue. Per 16-Gaussian batch:
// phase 1 (thread = pixel) writes (alpha T, G dL/dalpha) to shared memory; phase 2 (lane =
// (Gaussian, pixel row)) accumulates the 10 per-Gaussian sums as pixel moments; the partial sets
// are combined in shared memory and each (tile, Gaussian) issues one atomic per component
// (block reduction before global atomics, north_star).
#include <algorithm>

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "gs_internal.cuh"

namespace gs {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N> __device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ------------------------------------------------------------------ tile order
// Longest-processing-time-first tile order for the backward tile pass (4.4 waves of tiles at
// config 2): tiles sorted by descending cost bucket (live-list length >> 5, 1024 buckets; order
// inside a bucket is arbitrary). CTAs are dispatched in blockIdx order, so the heaviest tiles start
// first and the tail of the launch holds the lightest ones. One CTA of NT threads. (Measured: the
// backward gains 6 us at config 2; for the forward a separate ordering launch cost more than the
// 3.6-wave tail it removed.)
constexpr int kOrderBuckets = 1024;
template <int NT, class Cost>
__device__ __forceinline__ void lpt_tile_order(Cost cost, int T, uint32_t* __restrict__ order) {
    using BS = cub::BlockScan<uint32_t, NT>;
    __shared__ typename BS::TempStorage tmp;
    __shared__ uint32_t hist[kOrderBuckets];
    constexpr int PER = kOrderBuckets / NT;
    for (int b = threadIdx.x; b < kOrderBuckets; b += NT) hist[b] = 0;
    __syncthreads();
    auto bucket = [&](int t) { return kOrderBuckets - 1 - int(min(cost(t), uint32_t(kOrderBuckets - 1))); };
    for (int t = threadIdx.x; t < T; t += NT) atomicAdd(hist + bucket(t), 1u);
    __syncthreads();
    uint32_t v[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) v[j] = hist[threadIdx.x * PER + j];
    BS(tmp).ExclusiveSum(v, v);
#pragma unroll
    for (int j = 0; j < PER; ++j) hist[threadIdx.x * PER + j] = v[j];
    __syncthreads();
    for (int t = threadIdx.x; t < T; t += NT) order[atomicAdd(hist + bucket(t), 1u)] = uint32_t(t);
}

// ------------------------------------------------------------------ forward
constexpr int kFwdBatch = 256;

template <bool kAccum>
__global__ void __launch_bounds__(kTilePx) render_fwd_kernel(
    const float4* __restrict__ rec, const uint32_t* __restrict__ vals, const uint2* __restrict__ ranges, int W, int H,
    int GX, float bgr, float bgg, float bgb, float* __restrict__ color, float* __restrict__ depth,
    float* __restrict__ alpha, float* __restrict__ t_final, uint32_t* __restrict__ n_last, uint32_t* __restrict__ examined,
    float* __restrict__ accum_weight, uint32_t* __restrict__ live_g, uint32_t* __restrict__ live_j,
    uint32_t* __restrict__ live_cnt) {
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

    uint32_t staged = 0;   // this variant publishes every staged entry as live (no reach test)
    auto stage = [&](int b) {
        const uint32_t j = uint32_t(b) * kFwdBatch + threadIdx.x;
        staged = min(len, uint32_t(b + 1) * kFwdBatch);
        if (j < len) {
            const uint32_t g = vals[start + j];
            live_g[start + j] = g;
            live_j[start + j] = j + 1;
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
    if (threadIdx.x == 0) live_cnt[tile] = staged;
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

// Fast forward: 128 threads per tile, two pixels per thread (rows ly and ly + 8) so the record
// loads, the x-terms of power and the loop overhead are shared. Bit-identical decisions and
// results to render_fwd_kernel (same per-pixel operation sequence as eval_alpha).
struct PixState {
    float T, Cr, Cg, Cb, D;
    uint32_t nl, exam;
    bool done;
};

// Branch-free blend step (predicated selects): a skipped, terminated or already-done pixel gets
// w = 0, and fma(0, c, C) == C bitwise, so the result equals the branchy definition exactly.
__device__ __forceinline__ void blend_step(PixState& p, float power, float4 r1, float4 r2, uint32_t j) {
    float G;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(G) : "f"(__fmul_rn(power, 1.4426950408889634f)));
    const float a = fminf(0.99f, __fmul_rn(r1.y, G));
    const bool live = !p.done && !(power > 0.f) && a >= (1.0f / 255.0f);
    const float Tn = __fmul_rn(p.T, __fsub_rn(1.f, a));
    const bool term = live && Tn < 1e-4f;
    const bool blend = live && !(Tn < 1e-4f);
    const float w = blend ? __fmul_rn(a, p.T) : 0.f;
    p.Cr = fmaf(w, r2.x, p.Cr);
    p.Cg = fmaf(w, r2.y, p.Cg);
    p.Cb = fmaf(w, r2.z, p.Cb);
    p.D = fmaf(w, r1.z, p.D);
    p.T = blend ? Tn : p.T;
    p.nl = blend ? j : p.nl;
    p.exam = term ? j : p.exam;
    p.done = p.done || term;
}

// Blend step without the termination test (the fast path of render_fwd2_kernel): identical
// arithmetic to blend_step for every entry that does not terminate the pixel. A skipped entry gets
// alpha 0, so w = 0 and T (1 - 0) == T bitwise.
__device__ __forceinline__ void blend_fast(PixState& p, float power, float4 r1, float4 r2, uint32_t j) {
    float G;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(G) : "f"(__fmul_rn(power, 1.4426950408889634f)));
    const float a0 = fminf(0.99f, __fmul_rn(r1.y, G));
    const bool live = !p.done && !(power > 0.f) && a0 >= (1.0f / 255.0f);
    const float a = live ? a0 : 0.f;
    const float w = __fmul_rn(a, p.T);
    p.Cr = fmaf(w, r2.x, p.Cr);
    p.Cg = fmaf(w, r2.y, p.Cg);
    p.Cb = fmaf(w, r2.z, p.Cb);
    p.D = fmaf(w, r1.z, p.D);
    p.T = __fmul_rn(p.T, __fsub_rn(1.f, a));
    p.nl = live ? j : p.nl;
}

// The same two steps for a PAIR of pixels (rows ly and ly + 8 of the thread), with the per-pixel
// arithmetic in packed fp32 pairs (gs_internal.cuh): every operation is the scalar one above, per
// pixel, in the same order and rounding, so results are bit-identical to blend_step / blend_fast.
struct PixPair {
    f32x2 T, Cr, Cg, Cb, D;   // lo = pixel A, hi = pixel B
    uint32_t nlA, nlB, exA, exB;
    bool dA, dB;
};

__device__ __forceinline__ f32x2 alpha_pair(f32x2 power, float o, f32x2& G) {
    const f32x2 l = mul2(power, bc2(1.4426950408889634f));
    float gA, gB;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(gA) : "f"(lo2(l)));
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(gB) : "f"(hi2(l)));
    G = pk2(gA, gB);
    return mul2(bc2(o), G);   // o G
}

__device__ __forceinline__ void blend_fast_pair(PixPair& p, f32x2 power, float4 r1, float4 r2, uint32_t j) {
    f32x2 G;
    const f32x2 og = alpha_pair(power, r1.y, G);
    const float a0A = fminf(0.99f, lo2(og)), a0B = fminf(0.99f, hi2(og));
    const bool liveA = !p.dA && !(lo2(power) > 0.f) && a0A >= (1.0f / 255.0f);
    const bool liveB = !p.dB && !(hi2(power) > 0.f) && a0B >= (1.0f / 255.0f);
    const f32x2 a = pk2(liveA ? a0A : 0.f, liveB ? a0B : 0.f);
    const f32x2 w = mul2(a, p.T);
    p.Cr = fma2(w, bc2(r2.x), p.Cr);
    p.Cg = fma2(w, bc2(r2.y), p.Cg);
    p.Cb = fma2(w, bc2(r2.z), p.Cb);
    p.D = fma2(w, bc2(r1.z), p.D);
    p.T = mul2(p.T, sub2(bc2(1.f), a));
    p.nlA = liveA ? j : p.nlA;
    p.nlB = liveB ? j : p.nlB;
}

__device__ __forceinline__ void blend_step_pair(PixPair& p, f32x2 power, float4 r1, float4 r2, uint32_t j) {
    f32x2 G;
    const f32x2 og = alpha_pair(power, r1.y, G);
    const float aA = fminf(0.99f, lo2(og)), aB = fminf(0.99f, hi2(og));
    const bool liveA = !p.dA && !(lo2(power) > 0.f) && aA >= (1.0f / 255.0f);
    const bool liveB = !p.dB && !(hi2(power) > 0.f) && aB >= (1.0f / 255.0f);
    const f32x2 a = pk2(aA, aB);
    const f32x2 Tn = mul2(p.T, sub2(bc2(1.f), a));
    const bool termA = liveA && lo2(Tn) < 1e-4f, termB = liveB && hi2(Tn) < 1e-4f;
    const bool blA = liveA && !(lo2(Tn) < 1e-4f), blB = liveB && !(hi2(Tn) < 1e-4f);
    const f32x2 Ta = mul2(a, p.T);
    const f32x2 w = pk2(blA ? lo2(Ta) : 0.f, blB ? hi2(Ta) : 0.f);
    p.Cr = fma2(w, bc2(r2.x), p.Cr);
    p.Cg = fma2(w, bc2(r2.y), p.Cg);
    p.Cb = fma2(w, bc2(r2.z), p.Cb);
    p.D = fma2(w, bc2(r1.z), p.D);
    p.T = pk2(blA ? lo2(Tn) : lo2(p.T), blB ? hi2(Tn) : hi2(p.T));
    p.nlA = blA ? j : p.nlA;
    p.nlB = blB ? j : p.nlB;
    p.exA = termA ? j : p.exA;
    p.exB = termB ? j : p.exB;
    p.dA = p.dA || termA;
    p.dB = p.dB || termB;
}

constexpr int kFwd2Batch = kTilePx / 2;   // one staged record per thread

// Can Gaussian (r0, r1) reach alpha >= 1/255 at any pixel of the box [x0, x1] x [y0, y1]? Conservative:
// alpha >= 1/255 needs q = (conic quadratic form) <= q_max = 2 ln(255 o) (r1.w, from gs_project, with
// a margin), so the test compares the minimum of q over the (continuous) box with q_max, loosened by
// 3e-5 of the terms' magnitude (covers the fp32 evaluation error of both this minimum and the
// kernel's per-pixel power) and 1e-5 absolute. A "false" therefore guarantees that every per-pixel
// fp32 decision skips this Gaussian in this tile, so dropping it changes no output.
__device__ __forceinline__ bool can_reach(float4 r0, float4 r1, float x0, float y0, float x1, float y1) {
    const float qmax = r1.w;
    const float mx = r0.x, my = r0.y, a = -2.f * r0.z, b = -r0.w, c = -2.f * r1.x;
    if (mx >= x0 && mx <= x1 && my >= y0 && my <= y1) return qmax >= -1e-5f;
    auto q = [&](float dx, float dy) { return fmaf(a * dx, dx, fmaf(2.f * b * dx, dy, c * dy * dy)); };
    // The edge minimisers use approximate reciprocals: a minimiser off by d changes q by c d^2
    // (second order; with rcp.approx's 2^-22 relative error at most a dx^2 2^-44 <= qmag 2^-44),
    // far inside the 3e-5 qmag slack below, so the test stays conservative.
    float rc, ra;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rc) : "f"(c));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(ra) : "f"(a));
    const float bc = b * rc, ba = b * ra;
    float qmin = 3.0e38f;
#pragma unroll
    for (int e = 0; e < 2; ++e) {   // vertical edges x = x0, x1: minimise over y in [y0, y1]
        const float dx = mx - (e ? x1 : x0);
        const float y = fminf(fmaxf(fmaf(bc, dx, my), y0), y1);
        qmin = fminf(qmin, q(dx, my - y));
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {   // horizontal edges y = y0, y1: minimise over x in [x0, x1]
        const float dy = my - (e ? y1 : y0);
        const float x = fminf(fmaxf(fmaf(ba, dy, mx), x0), x1);
        qmin = fminf(qmin, q(mx - x, dy));
    }
    const float dxm = fmaxf(fabsf(mx - x0), fabsf(mx - x1)), dym = fmaxf(fabsf(my - y0), fabsf(my - y1));
    const float qmag = fabsf(a) * dxm * dxm + 2.f * fabsf(b) * dxm * dym + fabsf(c) * dym * dym;
    return qmin - 3e-5f * qmag - 1e-5f <= qmax;
}

__global__ void __launch_bounds__(kTilePx / 2, 6) render_fwd2_kernel(
    const float4* __restrict__ rec, const uint32_t* __restrict__ vals, const uint2* __restrict__ ranges, int W, int H,
    int GX, float bgr, float bgg, float bgb, float* __restrict__ color, float* __restrict__ depth,
    float* __restrict__ alpha, float* __restrict__ t_final, uint32_t* __restrict__ n_last,
    uint32_t* __restrict__ examined, uint32_t* __restrict__ live_g, uint32_t* __restrict__ live_j,
    uint32_t* __restrict__ live_cnt) {
    griddep_wait();   // PDL (gs_internal.cuh)
    using BS = cub::BlockScan<int, kFwd2Batch>;
    __shared__ typename BS::TempStorage scan_tmp;
    constexpr int kU = 4;   // Gaussians per fast-path group (below)
    __shared__ float4 s_rec[2][kFwd2Batch][3];       // staged records (double-buffered)
    __shared__ uint32_t s_g[2][kFwd2Batch];
    __shared__ float4 s_lrec[kFwd2Batch + kU][3];    // the batch's live records, in order, padded to a
                                                     // multiple of kU with zero records; .w of the third
                                                     // float4 holds the 1-based list position
    __shared__ int s_nlive;
    const int tile = blockIdx.x;
    const int tx = tile % GX, ty = tile / GX;
    const int lx = threadIdx.x & 15, ly = threadIdx.x >> 4;   // ly in [0, 8)
    const int px = tx * kTile + lx, pyA = ty * kTile + ly, pyB = pyA + 8;
    const bool inA = px < W && pyA < H, inB = px < W && pyB < H;
    const float fpx = float(px), fyA = float(pyA), fyB = float(pyB);
    const float bx0 = float(tx * kTile), by0 = float(ty * kTile);
    const uint2 rg = ranges[tile];
    const uint32_t start = rg.x, len = rg.y - rg.x;
    const int nbatch = int((len + kFwd2Batch - 1) / kFwd2Batch);
    PixPair P{bc2(1.f), bc2(0.f), bc2(0.f), bc2(0.f), bc2(0.f), 0u, 0u, len, len, !inA, !inB};
    const f32x2 fy2 = pk2(fyA, fyB);
    uint32_t acc = 0;   // live entries written so far (this tile)

    auto stage = [&](int b) {
        const int slot = threadIdx.x;
        const uint32_t j = uint32_t(b) * kFwd2Batch + slot;
        float4* dst = s_rec[b & 1][slot];
        if (j < len) {
            const uint32_t g = vals[start + j];
            s_g[b & 1][slot] = g;
            const float4* src = rec + 3 * size_t(g);
            cp_async16(dst + 0, src + 0);
            cp_async16(dst + 1, src + 1);
            cp_async16(dst + 2, src + 2);
        } else {   // pad: opacity 0 -> alpha 0 -> skipped exactly (no blend, no termination)
            const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
            dst[0] = z;
            dst[1] = z;
            dst[2] = z;
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
        const int cnt = min(kFwd2Batch, int(len) - b * kFwd2Batch);
        const float4(*buf)[3] = s_rec[b & 1];
        // ordered compaction of the batch's Gaussians that can reach alpha >= 1/255 in this tile;
        // the live list (Gaussian, 1-based list position) is also what the backward walks
        {
            const int k = threadIdx.x;
            const int lv = (k < cnt && can_reach(buf[k][0], buf[k][1], bx0, by0, bx0 + 15.f, by0 + 15.f)) ? 1 : 0;
            int off, tot;
            BS(scan_tmp).ExclusiveSum(lv, off, tot);
            if (lv) {
                const uint32_t j = uint32_t(b * kFwd2Batch + k + 1);
                live_g[start + acc + off] = s_g[b & 1][k];
                live_j[start + acc + off] = j;
                float4 r2 = buf[k][2];
                r2.w = __uint_as_float(j);
                s_lrec[off][0] = buf[k][0];
                s_lrec[off][1] = buf[k][1];
                s_lrec[off][2] = r2;
            }
            if (k >= tot && k < ((tot + kU - 1) & ~(kU - 1))) {   // zero record: opacity 0 -> alpha 0
                const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
                s_lrec[k][0] = z;
                s_lrec[k][1] = z;
                s_lrec[k][2] = z;
            }
            if (k == 0) s_nlive = tot;
            __syncthreads();
        }
        const int nlive = s_nlive;
        acc += uint32_t(nlive);
        // Groups of kU Gaussians run a fast path without the termination test, which is exact
        // whenever no pixel of the warp terminates inside the group: T only decreases, so if T
        // after the group is >= 1e-4, every T (1 - alpha) tested inside it was too. Otherwise the
        // warp restores the group's entry state and replays it with the exact step (rare: once
        // per pixel at most).
        auto entry = [&](int k0, int u, float4& r1, float4& r2, uint32_t& j, f32x2& pw) {
            // past nlive the list is padded with zero records: opacity 0 -> alpha 0 -> skipped exactly
            const float4 r0 = s_lrec[k0 + u][0];
            r1 = s_lrec[k0 + u][1];
            r2 = s_lrec[k0 + u][2];
            j = __float_as_uint(r2.w);
            // eval_alpha's operation sequence per pixel; the x-terms are shared by the pair
            const float dx = __fsub_rn(r0.x, fpx);
            const float Adx = __fmul_rn(r0.z, dx), Bdx = __fmul_rn(r0.w, dx);
            const f32x2 dy = sub2(bc2(r0.y), fy2);
            pw = fma2(bc2(Adx), bc2(dx), fma2(mul2(bc2(r1.x), dy), dy, mul2(bc2(Bdx), dy)));
        };
        auto group = [&](int k0) {
            const PixPair P0 = P;
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                float4 r1, r2;
                uint32_t j;
                f32x2 pw;
                entry(k0, u, r1, r2, j, pw);
                blend_fast_pair(P, pw, r1, r2, j);
            }
            if (__any_sync(0xffffffffu, lo2(P.T) < 1e-4f || hi2(P.T) < 1e-4f)) {
                P = P0;
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    float4 r1, r2;
                    uint32_t j;
                    f32x2 pw;
                    entry(k0, u, r1, r2, j, pw);
                    blend_step_pair(P, pw, r1, r2, j);
                }
            }
        };
        // two groups per trip: the second group's state can take the registers the first group's
        // entry state (kept for its replay) held, so the loop carries no register copies
        for (int k0 = 0; k0 < nlive; k0 += 2 * kU) {
            if (__all_sync(0xffffffffu, P.dA && P.dB)) break;
            group(k0);
            if (k0 + kU >= nlive || __all_sync(0xffffffffu, P.dA && P.dB)) break;
            group(k0 + kU);
        }
        if (__syncthreads_and(P.dA && P.dB)) break;   // also orders buffer reuse
    }
    if (threadIdx.x == 0) live_cnt[tile] = acc;
    const size_t plane = size_t(W) * H;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        if (!(h ? inB : inA)) continue;
        const float T = h ? hi2(P.T) : lo2(P.T);
        const size_t pix = size_t(h ? pyB : pyA) * W + px;
        color[pix] = fmaf(T, bgr, h ? hi2(P.Cr) : lo2(P.Cr));
        color[plane + pix] = fmaf(T, bgg, h ? hi2(P.Cg) : lo2(P.Cg));
        color[2 * plane + pix] = fmaf(T, bgb, h ? hi2(P.Cb) : lo2(P.Cb));
        depth[pix] = h ? hi2(P.D) : lo2(P.D);
        alpha[pix] = 1.f - T;
        t_final[pix] = T;
        n_last[pix] = h ? P.nlB : P.nlA;
        if (examined) examined[pix] = h ? P.exB : P.exA;
    }
}

// Per-tile live lists written by the forward and walked by the backward: (Gaussian, 1-based list
// position) of every entry that can reach alpha >= 1/255 in the tile, at [ranges[t].x, + live_cnt[t]).
// They live in the value / key buffers that do not hold the sorted lists.
struct LiveBufs {
    uint32_t *g, *j, *cnt;
};
static LiveBufs live_bufs(WsState* s) {
    uint32_t* g = s->sorted_in_1 ? at<uint32_t>(s, s->vals0) : at<uint32_t>(s, s->vals1);
    uint32_t* j = reinterpret_cast<uint32_t*>(s->sorted_in_1 ? at<uint64_t>(s, s->keys0) : at<uint64_t>(s, s->keys1));
    return {g, j, at<uint32_t>(s, s->live_cnt)};
}

void launch_render_fwd(WsState* s, const gs_camera& cam, float* color, float* depth, float* alpha,
                       float* accum_weight, uint32_t flags, cudaStream_t st) {
    const int ntiles = s->cam_gx * s->cam_gy;
    const uint32_t* sorted_vals = s->sorted_in_1 ? at<uint32_t>(s, s->vals1) : at<uint32_t>(s, s->vals0);
    uint32_t* exam = (flags & GS_FLAG_EXAMINED) ? at<uint32_t>(s, s->examined) : nullptr;
    const LiveBufs lb = live_bufs(s);
    if (ntiles == 0) return;
    KTimer kt(s, KID_FWD, st);
    if ((flags & GS_FLAG_ACCUM_WEIGHT) && accum_weight) {
        render_fwd_kernel<true><<<ntiles, kTilePx, 0, st>>>(
            at<float4>(s, s->rec), sorted_vals, at<uint2>(s, s->ranges), cam.width, cam.height, s->cam_gx, cam.bg[0],
            cam.bg[1], cam.bg[2], color, depth, alpha, at<float>(s, s->t_final), at<uint32_t>(s, s->n_last), exam,
            accum_weight, lb.g, lb.j, lb.cnt);
    } else {
        launch_pdl(render_fwd2_kernel, dim3(ntiles), dim3(kTilePx / 2), 0, st,
            at<float4>(s, s->rec), sorted_vals, at<uint2>(s, s->ranges), cam.width, cam.height, s->cam_gx, cam.bg[0],
            cam.bg[1], cam.bg[2], color, depth, alpha, at<float>(s, s->t_final), at<uint32_t>(s, s->n_last), exam,
            lb.g, lb.j, lb.cnt);
    }
}

// ------------------------------------------------------------------ backward, tile pass
// One CTA of 128 threads per tile; each thread owns two pixels (rows ly and ly + 8), so the record
// loads and the x-terms of power are shared between them (same operation order as eval_alpha, so
// every decision is bit-identical to the forward's). Live-list entries (§5.3) are processed in
// batches of kBB, back to front:
//   phase 1  thread = 2 pixels: T_i = T_{i+1} / (1 - alpha_i), suffix sum S, and
//            (alpha_i T_i, G dL/dalpha_i) per (pixel, Gaussian) into shared memory (branch-free:
//            after the live-list skip ~97 % of the walked evaluations blend at config 2)
//   phase 2  lane = (Gaussian, row group): pixel moments with compile-time x
//   combine  one thread per (component, Gaussian) sums the per-warp partial moments it needs, turns
//            them into the screen-space gradient and issues its atomic.
// The staged batches rotate through 4 slots (gathered two ahead), so a batch needs 2 block barriers and none at its end.
constexpr int kBB = 16;                          // Gaussians per backward batch
constexpr int kBwdThreads = kTilePx / 2;         // 128
constexpr int kBwdWarps = kBwdThreads / 32;
constexpr int kGroups = kBwdWarps * (32 / kBB);  // phase-2 row groups (= partial sets)
constexpr int kRowsPerGroup = kTile / kGroups;
constexpr int kSlots = 4;
static_assert(kTile % kGroups == 0, "row groups must tile the 16 rows");

static_assert(kRowsPerGroup == 2 && kGroups == 8, "phase 2 pairs rows ly and ly + 8 like phase 1");

// Per-(pixel pair, Gaussian) values are stored as packed pairs: lo = pixel A (row ly), hi = pixel B
// (row ly + 8) of thread ly * 16 + lx, so phase 2's lane (Gaussian, row group gi), whose two rows are
// gi and gi + 8, reads exactly those pairs and accumulates them with packed fp32 operations.
struct BwdSmem {
    float4 rec[kSlots][kBB][3];
    float4 wg[kBB][kBwdThreads + 1];  // (-(alpha_i T_i) pair, G dL/dalpha_i pair); 0 when skipped, the
                                      // second also when clamped (rows padded: conflict-free)
    f32x2 dl[kBwdThreads][4];         // dL/dC (r, g, b), dL/dD
    float part[kBwdWarps][10][kBB];   // per-warp pixel moments (its two row groups combined)
    uint32_t pos[kSlots][kBB];        // 1-based list positions of the staged live entries (~0u: padding)
    uint32_t max_nl, len;
};

struct BwdPair {
    f32x2 T, Qn;              // T_{i+1} while walking back (starts at T_final); Qn = -(S + T_f bg.dL/dC)
                              // with the suffix sum S_i = sum_{k>i} alpha_k T_k e_k
    f32x2 dr, dg, db, dd;     // dL/dC, dL/dD
    uint32_t nlA, nlB;
};

// One back-to-front step for the pixel pair; power in eval_alpha's order (the decisions match the
// forward bit for bit). A skipped entry (past n_last, power > 0, alpha < 1/255, or padding) leaves T
// and Q unchanged and yields (0, 0). Gradient arithmetic (no decisions) in packed pairs:
//   T_i = T_{i+1} / (1 - alpha_i) (MUFU rcp.approx, <= 1 ulp), w = alpha_i T_i,
//   e_i = c_i.dL/dC + d_i dL/dD, dL/dalpha_i = T_i e_i - Q / (1 - alpha_i), go = G dL/dalpha_i.
__device__ __forceinline__ void bwd_step_pair(BwdPair& p, f32x2 power, float4 r1, float4 r2, uint32_t pk, f32x2& wn,
                                              f32x2& go) {
    f32x2 G;
    const f32x2 og = alpha_pair(power, r1.y, G);
    const float a0A = fminf(0.99f, lo2(og)), a0B = fminf(0.99f, hi2(og));
    const bool liveA = pk <= p.nlA && !(lo2(power) > 0.f) && a0A >= (1.0f / 255.0f);
    const bool liveB = pk <= p.nlB && !(hi2(power) > 0.f) && a0B >= (1.0f / 255.0f);
    const f32x2 an = pk2(liveA ? -a0A : 0.f, liveB ? -a0B : 0.f);   // -alpha
    const f32x2 om = add2(bc2(1.f), an);                              // 1 - alpha
    float roA, roB;   // skipped: rcp.approx(1) == 1, T unchanged
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(roA) : "f"(lo2(om)));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(roB) : "f"(hi2(om)));
    const f32x2 ro = pk2(roA, roB);
    p.T = mul2(p.T, ro);
    wn = mul2(an, p.T);
    const f32x2 ev = fma2(bc2(r2.x), p.dr, fma2(bc2(r2.y), p.dg, fma2(bc2(r2.z), p.db, mul2(bc2(r1.z), p.dd))));
    // gradient to o and power only when live and not clamped: G masked in place (no select after)
    const f32x2 Gm = pk2((liveA && !(lo2(og) > 0.99f)) ? lo2(G) : 0.f, (liveB && !(hi2(og) > 0.99f)) ? hi2(G) : 0.f);
    go = mul2(Gm, fma2(p.T, ev, mul2(p.Qn, ro)));
    p.Qn = fma2(wn, ev, p.Qn);   // wn == 0 when skipped: Q unchanged (ev finite; padding is zero-filled)
}

// Fused L1 loss (gs_render_bwd_l1): the pixel loads form dL/dC, dL/dD of Eq. 6 (reading C20) from
// the rendered and target images with exactly gs_loss_l1's arithmetic, and each block adds its
// |C - C*| and valid |D - D*| sums to acc[0], acc[1] (acc[2] = valid-pixel count, counted before).
struct FusedL1 {
    const float *color, *depth, *tc, *td;
    float wc, wd;
    double* acc;
};

__device__ __forceinline__ float sgn1(float x) { return float((x > 0.f) - (x < 0.f)); }

// Tile-pass modes: the full backward (10 screen quantities per Gaussian), and the two pose-only
// passes of gs_pose_grad (§8(a) a10): POSE_COV accumulates only the 6 quantities the pose chain reads
// (mean, conic, depth) for the per-Gaussian pass; POSE_PAPER (the paper's gradient) needs only
// the mean and depth paths, so each (tile, Gaussian) turns its sums directly into its share of the
// twist (rho += dL/dX^c, phi += X^c x dL/dX^c, with J and X^c rebuilt from the record) in fp64, and
// the last tile block reduces the per-tile partials in a fixed order: no screen atomics and no
// per-Gaussian pass.
enum BwdMode { BWD_FULL = 0, BWD_POSE_COV = 1, BWD_POSE_PAPER = 2 };

struct PoseTile {              // BWD_POSE_PAPER only
    float fx, fy, cx, cy;
    double* part;              // [6][gridDim.x] per-tile twist partials
    unsigned int* ticket;      // last-block ticket (self-resetting)
    double* grad_pose;         // [6], += (or = with assign)
    int assign;
    LossFin lf;                // fused L1: the loss scalar, written by the last block
};

template <bool L1, int MODE>
__global__ void __launch_bounds__(kBwdThreads, 5) render_bwd_kernel(
    const float4* __restrict__ rec, const uint32_t* __restrict__ live_g, const uint32_t* __restrict__ live_j,
    const uint32_t* __restrict__ live_cnt, const uint2* __restrict__ ranges, int W, int H,
    int GX, const float* __restrict__ t_final, float bgr, float bgg, float bgb, const uint32_t* __restrict__ n_last,
    const float* __restrict__ dLdC, const float* __restrict__ dLdD, float* __restrict__ sgrad, int64_t sld,
    FusedL1 l1, const uint32_t* __restrict__ order, PoseTile pt) {
    griddep_wait();   // PDL (gs_internal.cuh)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    BwdSmem& sm = *reinterpret_cast<BwdSmem*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int tile = order ? int(order[blockIdx.x]) : int(blockIdx.x);   // LPT order (zero_sgrad_kernel)
    const int tx = tile % GX, ty = tile / GX;
    const int lx = tid & 15, ly = tid >> 4;   // ly in [0, 8)
    const int px = tx * kTile + lx, pyA = ty * kTile + ly, pyB = pyA + 8;
    const float fpx = float(px), fyA = float(pyA), fyB = float(pyB);
    const uint32_t start = ranges[tile].x;
    const size_t plane = size_t(W) * H;

    BwdPair P;
    {
        float t[2] = {1.f, 1.f}, d[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
        uint32_t nl[2] = {0u, 0u};
        float sum_c = 0.f, sum_d = 0.f;   // L1: this thread's |C - C*| and valid |D - D*|
        float sc = 0.f, sd = 0.f;
        if (L1) {
            const double nvalid = __ldcg(l1.acc + 2);
            sc = float(double(l1.wc) / (3.0 * double(plane)));
            sd = nvalid > 0 ? float(double(l1.wd) / nvalid) : 0.f;
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int py = h ? pyB : pyA;
            if (px < W && py < H) {
                const size_t pix = size_t(py) * W + px;
                nl[h] = n_last[pix];
                if (L1) {
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const float e = l1.color[c * plane + pix] - l1.tc[c * plane + pix];
                        sum_c += fabsf(e);
                        d[h][c] = sc * sgn1(e);
                    }
                    const float tdv = l1.td[pix], e = l1.depth[pix] - tdv;
                    if (tdv > 0.f) sum_d += fabsf(e);
                    d[h][3] = tdv > 0.f ? sd * sgn1(e) : 0.f;
                } else {
                    d[h][0] = dLdC[pix];
                    d[h][1] = dLdC[plane + pix];
                    d[h][2] = dLdC[2 * plane + pix];
                    d[h][3] = dLdD[pix];
                }
                t[h] = t_final[pix];
            }
        }
        if (L1) {   // block sums -> one fp64 atomic per quantity
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                sum_c += __shfl_xor_sync(0xffffffffu, sum_c, o);
                sum_d += __shfl_xor_sync(0xffffffffu, sum_d, o);
            }
            if (lane == 0) {
                atomicAdd(l1.acc + 0, double(sum_c));
                atomicAdd(l1.acc + 1, double(sum_d));
            }
        }
        P.T = pk2(t[0], t[1]);
        P.dr = pk2(d[0][0], d[1][0]);
        P.dg = pk2(d[0][1], d[1][1]);
        P.db = pk2(d[0][2], d[1][2]);
        P.dd = pk2(d[0][3], d[1][3]);
        P.nlA = nl[0];
        P.nlB = nl[1];
        // S = 0 at the back: Q = T_f bg.dL/dC
        P.Qn = pk2(-(t[0] * (bgr * d[0][0] + bgg * d[0][1] + bgb * d[0][2])),
                   -(t[1] * (bgr * d[1][0] + bgg * d[1][1] + bgb * d[1][2])));
        sm.dl[tid][0] = P.dr;
        sm.dl[tid][1] = P.dg;
        sm.dl[tid][2] = P.db;
        sm.dl[tid][3] = P.dd;
    }
    const f32x2 fy2 = pk2(fyA, fyB);
    if (tid == 0) sm.max_nl = 0;
    __syncthreads();
    uint32_t mnl = max(P.nlA, P.nlB);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mnl = max(mnl, __shfl_xor_sync(0xffffffffu, mnl, o));
    if (lane == 0 && mnl) atomicMax(&sm.max_nl, mnl);
    __syncthreads();
    // the live entries to walk: those with list position <= max n_last (positions ascend), found by
    // one warp with a 32-ary search over the forward's live list
    if (warp == 0) {
        const uint32_t mx = sm.max_nl;
        uint32_t lo = 0, hi = live_cnt[tile];   // answer in [lo, hi]
        while (hi > lo) {
            const uint32_t step = (hi - lo + 31) / 32;
            const uint32_t probe = lo + uint32_t(lane) * step;   // is entry `probe` within max n_last?
            const bool in = probe < hi && live_j[start + probe] <= mx;
            const unsigned m = __ballot_sync(0xffffffffu, in);
            if (m == 0u) { hi = lo; break; }
            const uint32_t last = lo + uint32_t(31 - __clz(m)) * step;   // last probe within
            lo = last + 1;
            hi = min(hi, last + step);
        }
        if (lane == 0) sm.len = lo;
    }
    __syncthreads();
    const uint32_t len = sm.len;
    const int nbatch = int((len + kBB - 1) / kBB);

    // batch bb holds live entries [bb*kBB, bb*kBB+kBB); batches are visited back to front
    auto stage = [&](int bb, int slot) {
        if (tid < kBB) {
            const uint32_t j = uint32_t(bb) * kBB + tid;
            float4* dst = sm.rec[slot][tid];
            if (j < len) {
                const uint32_t g = live_g[start + j];
                sm.pos[slot][tid] = live_j[start + j];
                const float4* src = rec + 3 * size_t(g);
                cp_async16(dst + 0, src + 0);
                cp_async16(dst + 1, src + 1);
                cp_async16(dst + 2, src + 2);
            } else {   // padding: never live, zero record keeps every product finite
                const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
                sm.pos[slot][tid] = 0xffffffffu;
                dst[0] = z;
                dst[1] = z;
                dst[2] = z;
            }
        }
        cp_async_commit();
    };

    // phase-2 lane roles: Gaussian k2 of the batch, row group gi (rows gi + kGroups r)
    const int k2 = lane & (kBB - 1), gi = warp * (32 / kBB) + lane / kBB;
    // records are gathered two batches ahead (4 slots: staging it + 2, phase 1 on it, gradients of
    // it - 1; the slot staged at iteration it was last read by batch it - 2's gradients, which every
    // warp finished before the previous iteration's barrier [B])
    if (nbatch > 0) stage(nbatch - 1, 0);
    if (nbatch > 1) stage(nbatch - 2, 1);
    // ---- moments -> screen-space gradients of batch bb (staged in slot gbuf); one thread and one
    // atomic per (component, Gaussian). Each thread sums the per-warp partial sets it needs. Batch
    // bb's gradients run right after the NEXT batch's barrier [A] (or after the loop): part and the
    // slot are rewritten only after that batch's barrier [B] and two stagings later, so no barrier of
    // their own is needed (two barriers per batch).
    double tw[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};   // BWD_POSE_PAPER: this thread's twist sums
    auto gradients = [&](int gbuf, int gbb) {
        const int cnt = min(kBB, int(len) - gbb * kBB);
        auto moment = [&](int c, int k) {
            float a = 0.f;
#pragma unroll
            for (int p = 0; p < kBwdWarps; ++p) a += sm.part[p][c][k];
            return a;
        };
        if (MODE == BWD_POSE_PAPER) {
            const int k = tid;
            if (k >= cnt) return;
            const float M0 = moment(0, k), Mx = moment(1, k), My = moment(2, k);
            const float4 r0 = sm.rec[gbuf][k][0], r1 = sm.rec[gbuf][k][1];
            const float o = r1.y;
            const float X = r0.x - (float(tx * kTile) + 7.5f), Y = r0.y - (float(ty * kTile) + 7.5f);
            const float gdx = X * M0 - Mx, gdy = Y * M0 - My;
            const float dmx = o * (2.f * r0.z * gdx + r0.w * gdy);   // as the full pass' mean gradients
            const float dmy = o * (r0.w * gdx + 2.f * r1.x * gdy);
            const float dd = moment(9, k);
            // X^c and J from the record: z = d, x = (m_x - c_x) z / f_x (C3 typo fixed)
            const double z = double(r1.z), ux = double(r0.x - pt.cx), uy = double(r0.y - pt.cy);
            const double x = ux * z / double(pt.fx), y = uy * z / double(pt.fy);
            const double g0 = double(pt.fx) / z * double(dmx), g1 = double(pt.fy) / z * double(dmy);
            const double g2 = -(ux / z) * double(dmx) - (uy / z) * double(dmy) + double(dd);
            tw[0] += g0;
            tw[1] += g1;
            tw[2] += g2;
            tw[3] += y * g2 - z * g1;
            tw[4] += z * g0 - x * g2;
            tw[5] += x * g1 - y * g0;
            return;
        }
        constexpr int kComps = MODE == BWD_FULL ? 10 : 6;
        for (int t = tid; t < kComps * kBB; t += kBwdThreads) {
            const int ci = t / kBB, k = t % kBB;
            const int c = (MODE == BWD_FULL || ci < 5) ? ci : 9;   // POSE_COV: mean, conic, depth
            if (k >= cnt) continue;
            float v;
            if (c >= 5) {
                v = moment(c == 5 ? 0 : c, k);   // opacity (sum g), rgb, depth
            } else {
                const float M0 = moment(0, k), Mx = moment(1, k), My = moment(2, k);
                const float4 r0 = sm.rec[gbuf][k][0];
                const float o = sm.rec[gbuf][k][1].y;
                // moments are about the tile centre (lx, ly in -7.5 .. 7.5: no cancellation between
                // X^2 M0, 2 X Mx and Mxx beyond the sum's own when the mean is near the tile)
                const float X = r0.x - (float(tx * kTile) + 7.5f), Y = r0.y - (float(ty * kTile) + 7.5f);
                // sums of g dx, g dy, g dx^2, g dx dy, g dy^2 with dx = X - lx, dy = Y - ly
                const float gdx = X * M0 - Mx, gdy = Y * M0 - My;
                if (c == 0) {
                    v = o * (2.f * r0.z * gdx + r0.w * gdy);            // mean2d x: -o (a gdx + b gdy)
                } else if (c == 1) {
                    v = o * (r0.w * gdx + 2.f * sm.rec[gbuf][k][1].x * gdy);   // mean2d y: -o (b gdx + c gdy)
                } else if (c == 2) {
                    v = -0.5f * o * (X * X * M0 - 2.f * X * Mx + moment(3, k));            // conic a
                } else if (c == 3) {
                    v = -o * (X * Y * M0 - X * My - Y * Mx + moment(4, k));                 // conic b
                } else {
                    v = -0.5f * o * (Y * Y * M0 - 2.f * Y * My + moment(5, k));            // conic c
                }
            }
            // screen accumulators are indexed by on-screen rank (record r2.w, written by gs_bin_sort)
            if (v != 0.f) atomicAdd(sgrad + c * sld + __float_as_uint(sm.rec[gbuf][k][2].w), v);
        }
    };
    for (int it = 0; it < nbatch; ++it) {
        const int bb = nbatch - 1 - it;
        const int buf = it % kSlots;
        if (it + 2 < nbatch) {
            stage(bb - 2, (it + 2) % kSlots);
            cp_async_wait<2>();
        } else if (it + 1 < nbatch) {
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();   // [A] batch staged (and the previous batch's partial sets complete)
        if (it > 0) gradients((it - 1) % kSlots, bb + 1);
        // ---- phase 1
        // records are read one step ahead (shared-memory latency off the dependent chain)
        uint32_t pk_n = sm.pos[buf][kBB - 1];
        float4 r0_n = sm.rec[buf][kBB - 1][0], r1_n = sm.rec[buf][kBB - 1][1], r2_n = sm.rec[buf][kBB - 1][2];
#pragma unroll 4
        for (int k = kBB - 1; k >= 0; --k) {
            const uint32_t pk = pk_n;
            const float4 r0 = r0_n, r1 = r1_n, r2 = r2_n;
            const int kn = k > 0 ? k - 1 : 0;
            pk_n = sm.pos[buf][kn];
            r0_n = sm.rec[buf][kn][0];
            r1_n = sm.rec[buf][kn][1];
            r2_n = sm.rec[buf][kn][2];
            const float dx = __fsub_rn(r0.x, fpx);
            const float Adx = __fmul_rn(r0.z, dx), Bdx = __fmul_rn(r0.w, dx);
            const f32x2 dy = sub2(bc2(r0.y), fy2);
            const f32x2 pw = fma2(bc2(Adx), bc2(dx), fma2(mul2(bc2(r1.x), dy), dy, mul2(bc2(Bdx), dy)));
            f32x2 wn, go;
            bwd_step_pair(P, pw, r1, r2, pk, wn, go);
            sm.wg[k][tid] = make_float4(lo2(wn), hi2(wn), lo2(go), hi2(go));
        }
        __syncthreads();   // [B] wg complete
        // ---- phase 2: moments over the group's two rows (gi, gi + 8) as packed pairs, compile-time x
        {
            f32x2 R0 = bc2(0.f), Rx = bc2(0.f), Rxx = bc2(0.f);
            f32x2 Sr = bc2(0.f), Sg = bc2(0.f), Sb = bc2(0.f), Sd = bc2(0.f);
#pragma unroll
            for (int x = 0; x < 16; ++x) {
                const int q = gi * 16 + x;
                const float4 v = sm.wg[k2][q];
                const f32x2 w = pk2(v.x, v.y), g = pk2(v.z, v.w);
                R0 = add2(R0, g);
                Rx = fma2(g, bc2(float(x) - 7.5f), Rx);                               // exact constants
                if (MODE != BWD_POSE_PAPER) Rxx = fma2(g, bc2((float(x) - 7.5f) * (float(x) - 7.5f)), Rxx);
                if (MODE == BWD_FULL) {
                    Sr = fma2(w, sm.dl[q][0], Sr);
                    Sg = fma2(w, sm.dl[q][1], Sg);
                    Sb = fma2(w, sm.dl[q][2], Sb);
                }
                Sd = fma2(w, sm.dl[q][3], Sd);
            }
            const float fyA_ = float(gi) - 7.5f, fyB_ = float(gi + kGroups) - 7.5f;   // about the centre
            float m[10];
            m[0] = lo2(R0) + hi2(R0);                                 // sum g
            m[1] = lo2(Rx) + hi2(Rx);                                 // sum g lx
            m[2] = fyA_ * lo2(R0) + fyB_ * hi2(R0);                   // sum g ly
            m[3] = lo2(Rxx) + hi2(Rxx);                               // sum g lx^2
            m[4] = fyA_ * lo2(Rx) + fyB_ * hi2(Rx);                   // sum g lx ly
            m[5] = fyA_ * fyA_ * lo2(R0) + fyB_ * fyB_ * hi2(R0);     // sum g ly^2
            m[6] = -(lo2(Sr) + hi2(Sr));                              // (wg holds -alpha T)
            m[7] = -(lo2(Sg) + hi2(Sg));
            m[8] = -(lo2(Sb) + hi2(Sb));
            m[9] = -(lo2(Sd) + hi2(Sd));
            // lanes l and l + 16 hold the same Gaussian for the warp's two row groups
#pragma unroll
            for (int c = 0; c < 10; ++c) {
                if (MODE == BWD_POSE_PAPER && c >= 3 && c < 9) continue;
                if (MODE == BWD_POSE_COV && c >= 6 && c < 9) continue;
                m[c] += __shfl_xor_sync(0xffffffffu, m[c], 16);
                if (lane < kBB) sm.part[warp][c][k2] = m[c];
            }
        }
    }
    if (nbatch > 0) {
        __syncthreads();   // the last batch's partial sets are complete
        gradients((nbatch - 1) % kSlots, 0);
    }
    if (MODE == BWD_POSE_PAPER) {
        // this tile's twist partial: the kBB gradient threads (warp 0) reduce in a fixed order
        __shared__ bool s_last;
        if (warp == 0) {
#pragma unroll
            for (int c = 0; c < 6; ++c) {
                double v = tw[c];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (lane == 0) pt.part[size_t(c) * gridDim.x + blockIdx.x] = v;
            }
            if (lane == 0) __threadfence();   // the writer publishes the partials before the ticket
        }
        __syncthreads();
        if (tid == 0) s_last = atomicAdd(pt.ticket, 1u) == gridDim.x - 1;
        __syncthreads();
        if (!s_last) return;
        __threadfence();
        // last block: fixed-order sums over the tiles, warp w sums component w (and w + 4)
        __shared__ double acc6[6];
        for (int c = warp; c < 6; c += kBwdWarps) {
            double v = 0.0;
            for (unsigned b = lane; b < gridDim.x; b += 32) v += __ldcg(pt.part + size_t(c) * gridDim.x + b);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) acc6[c] = v;
        }
        __syncthreads();
        if (tid == 0) {
            for (int c = 0; c < 6; ++c) pt.grad_pose[c] = (pt.assign ? 0.0 : pt.grad_pose[c]) + acc6[c];
            if (pt.lf.loss) {   // fused L1: every block's loss sums are in (atomics before the ticket)
                const double nvalid = __ldcg(pt.lf.acc + 2);
                const float sc = float(double(pt.lf.wc) / (3.0 * double(pt.lf.npx)));
                const float sd = nvalid > 0 ? float(double(pt.lf.wd) / nvalid) : 0.f;
                *pt.lf.loss = double(sc) * __ldcg(pt.lf.acc) + (nvalid > 0 ? double(sd) * __ldcg(pt.lf.acc + 1) : 0.0);
            }
            *pt.ticket = 0u;
        }
    }
}

// Backward prologue (one launch): the screen accumulators [10][V_s] (rank-indexed) cleared; block 0
// builds the LPT tile order; with the fused L1 loss, the valid-pixel count of the target depth
// (reading C20's depth mean): per-block counts, and the last block to finish (atomic ticket,
// self-resetting) sums them in a fixed order into acc[2] and zeroes the loss sums acc[0..1] that
// the tile pass accumulates. No memset and no second kernel.
inline int prep_blocks() { return std::min(sm_count() * 4, 1024); }   // <= chunk_hist rows
__global__ void __launch_bounds__(256) zero_sgrad_kernel(float* __restrict__ sgrad, int64_t sld,
                                                         const unsigned int* __restrict__ n_on,
                                                         const uint32_t* __restrict__ live_cnt, int T,
                                                         uint32_t* __restrict__ order, const float* __restrict__ td,
                                                         int64_t npx, uint32_t* __restrict__ part, double* acc,
                                                         unsigned int* ticket, unsigned int* zero_chunk) {
    griddep_wait();   // PDL (gs_internal.cuh)
    if (blockIdx.x == 0 && threadIdx.x == 0) *zero_chunk = 0u;   // gaussian_bwd's zeroing chunk counter
    // block 0 also builds the backward's LPT tile order from the forward's live-list lengths
    if (blockIdx.x == 0) lpt_tile_order<256>([&](int t) { return live_cnt[t]; }, T, order);
    const int64_t V = n_on ? int64_t(*n_on) : 0;   // nullptr: no clear (the pose-only paper-mode pass)
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < V; t += int64_t(gridDim.x) * blockDim.x)
#pragma unroll
        for (int c = 0; c < 10; ++c) sgrad[c * sld + t] = 0.f;
    if (!td) return;
    __shared__ uint32_t s_c[8];
    __shared__ bool s_last;
    uint32_t c = 0;
    const bool v4 = (reinterpret_cast<uintptr_t>(td) & 15) == 0;
    const int64_t n4 = v4 ? npx / 4 : 0;
    const float4* td4 = reinterpret_cast<const float4*>(td);
    for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < n4; q += int64_t(gridDim.x) * blockDim.x) {
        const float4 v = td4[q];
        c += (v.x > 0.f) + (v.y > 0.f) + (v.z > 0.f) + (v.w > 0.f);
    }
    for (int64_t p = 4 * n4 + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < npx;
         p += int64_t(gridDim.x) * blockDim.x)
        c += td[p] > 0.f ? 1u : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) s_c[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int w = 0; w < 8; ++w) t += s_c[w];
        part[blockIdx.x] = t;
        __threadfence();
        s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    uint32_t t = 0;   // fixed-order sum of the block counts (integers: exact in any order anyway)
    for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) t += __ldcg(part + b);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) s_c[threadIdx.x >> 5] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t tot = 0;
        for (int w = 0; w < 8; ++w) tot += s_c[w];
        acc[0] = 0.0;
        acc[1] = 0.0;
        acc[2] = double(tot);
        *ticket = 0u;
    }
}

void launch_zero_sgrad(WsState* s, cudaStream_t st, const float* td_l1, int64_t npx, bool clear) {
    KTimer kt(s, KID_SGRAD_CLEAR, st);
    Misc* misc = at<Misc>(s, s->misc);
    launch_pdl(zero_sgrad_kernel, dim3(prep_blocks()), dim3(256), 0, st, at<float>(s, s->sgrad), s->n_cap,
                                                   clear ? &misc->n_onscreen : nullptr,
                                                   at<uint32_t>(s, s->live_cnt), s->cam_gx * s->cam_gy,
                                                   at<uint32_t>(s, s->tile_order), td_l1, npx,
                                                   at<uint32_t>(s, s->chunk_hist), misc->loss_acc, &misc->prep_done,
                                                   &misc->gbwd_zero_chunk);
}

__global__ void loss_finalize_kernel(const double* acc, int64_t npx, float wc, float wd, double* loss) {
    const double nvalid = acc[2];
    const float sc = float(double(wc) / (3.0 * double(npx)));
    const float sd = nvalid > 0 ? float(double(wd) / nvalid) : 0.f;
    *loss = double(sc) * acc[0] + (nvalid > 0 ? double(sd) * acc[1] : 0.0);
}

void launch_render_bwd_tiles(WsState* s, const gs_camera& cam, const float*, const float* dL_dcolor,
                             const float* dL_ddepth, cudaStream_t st, const L1Fuse* fuse, bool finalize_loss,
                             int mode, double* grad_pose, int assign) {
    const int ntiles = s->cam_gx * s->cam_gy;
    if (ntiles == 0) return;
    const LiveBufs lb = live_bufs(s);
    static PerDeviceOnce attr;
    attr.run([] {
        for (auto k : {render_bwd_kernel<false, BWD_FULL>, render_bwd_kernel<true, BWD_FULL>,
                       render_bwd_kernel<false, BWD_POSE_COV>, render_bwd_kernel<true, BWD_POSE_COV>,
                       render_bwd_kernel<false, BWD_POSE_PAPER>, render_bwd_kernel<true, BWD_POSE_PAPER>}) {
            if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(BwdSmem))) != cudaSuccess)
                return false;
            cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, int(cudaSharedmemCarveoutMaxShared));
        }
        return true;
    });
    FusedL1 l1{};
    double* acc = at<Misc>(s, s->misc)->loss_acc;
    const int64_t npx = int64_t(cam.width) * cam.height;
    if (fuse) l1 = FusedL1{fuse->color, fuse->depth, fuse->tc, fuse->td, fuse->wc, fuse->wd, acc};   // acc: zero_sgrad_kernel
    PoseTile pt{cam.fx, cam.fy, cam.cx, cam.cy, at<double>(s, s->tile_pose), &at<Misc>(s, s->misc)->tile_pose_done,
                grad_pose, assign, LossFin{nullptr, nullptr, 0.f, 0.f, 0}};
    const bool paper = mode == BWD_POSE_PAPER;
    if (paper && fuse && fuse->loss && finalize_loss) {   // the pose pass' last block writes the loss
        pt.lf = LossFin{acc, fuse->loss, fuse->wc, fuse->wd, npx};
        finalize_loss = false;
    }
    {
        KTimer kt(s, paper ? KID_POSE_TILE : KID_BWD_TILE, st);
        auto k = fuse ? (mode == BWD_FULL ? render_bwd_kernel<true, BWD_FULL>
                         : mode == BWD_POSE_COV ? render_bwd_kernel<true, BWD_POSE_COV>
                                                : render_bwd_kernel<true, BWD_POSE_PAPER>)
                      : (mode == BWD_FULL ? render_bwd_kernel<false, BWD_FULL>
                         : mode == BWD_POSE_COV ? render_bwd_kernel<false, BWD_POSE_COV>
                                                : render_bwd_kernel<false, BWD_POSE_PAPER>);
        launch_pdl(k, dim3(ntiles), dim3(kBwdThreads), sizeof(BwdSmem), st,
            at<float4>(s, s->rec), lb.g, lb.j, lb.cnt, at<uint2>(s, s->ranges), cam.width, cam.height, s->cam_gx,
            at<float>(s, s->t_final), cam.bg[0], cam.bg[1], cam.bg[2], at<uint32_t>(s, s->n_last), dL_dcolor,
            dL_ddepth, at<float>(s, s->sgrad), s->n_cap, l1,
            s->n > 0 ? at<uint32_t>(s, s->tile_order) : nullptr, pt);
    }
    if (fuse && fuse->loss && finalize_loss) {
        KTimer kt(s, KID_LOSS_FINALIZE, st);
        loss_finalize_kernel<<<1, 1, 0, st>>>(acc, npx, fuse->wc, fuse->wd, fuse->loss);
    }
}

// ------------------------------------------------------------------ backward, per-Gaussian chain
// Screen-space gradients -> the 14 parameters (Eq. 11 / Supplement A) and the pose twist.
// pose partial sums: rho(3), phi(3), dW_cov(9)  (reading C7: A = W (sum dW_cov)^T).
constexpr int kPoseSums = 15;
constexpr int kGbwdBlocksPerSM = 2;   // resident blocks per SM (register budget 128: no spills)

// Persistent grid (a few blocks per SM) striding over the on-screen list; each thread keeps its pose
// partial sums across its Gaussians. The last block to finish (atomic ticket) reduces the per-block
// pose partials in a fixed order and applies the twist map, so the pose gradient is deterministic
// and needs no second launch. (Clearing the screen-space accumulators here as they are consumed,
// instead of the per-call memset, was measured 2x slower: scattered 4-B zero stores.)
__device__ void pose_finalize_block(const double* __restrict__ part, int nblocks, const float* __restrict__ viewmat,
                                    double* __restrict__ grad_pose, int assign);

__device__ __forceinline__ void gacc(float* p, float v, bool assign) {   // GS_FLAG_GRAD_ASSIGN: = instead of +=
    if (assign) *p = v;
    else *p += v;
}

template <int SH, bool ASSIGN>
__global__ void __launch_bounds__(256, kGbwdBlocksPerSM) gaussian_bwd_kernel(
    const float* __restrict__ params, int64_t n, int64_t ld, const float* __restrict__ viewmat, gs_camera cam,
    const uint32_t* __restrict__ onlist, const unsigned int* __restrict__ n_on, const float4* __restrict__ rec,
    const float* __restrict__ sgrad, int64_t sld, float* __restrict__ grad, int cov_path,
    double* __restrict__ pose_part, unsigned int* done_ctr, double* __restrict__ grad_pose, LossFin lf,
    const uint32_t* __restrict__ tiles, unsigned int* zero_chunk) {
    griddep_wait();   // PDL (gs_internal.cuh)
    constexpr bool assign = ASSIGN;
    __shared__ float V[12];
    __shared__ bool s_last;
    if (threadIdx.x < 12) V[threadIdx.x] = viewmat[threadIdx.x];
    __syncthreads();
    float pose[kPoseSums];   // a thread sums a few Gaussians (fp32); blocks reduce in fp64
#pragma unroll
    for (int k = 0; k < kPoseSums; ++k) pose[k] = 0.f;
    const int64_t Von = int64_t(*n_on);
    // thread t handles the t-th on-screen Gaussians (index order); off-screen ones have zero gradient
    // (GS_FLAG_GRAD_ASSIGN: written after the items, below)
    const int compute_blocks = int(gridDim.x);
    // the next item's Gaussian index is loaded one item ahead, so an item's parameter loads do not
    // wait for its index load first (one DRAM round trip per item instead of two)
    const int64_t tstride = int64_t(compute_blocks) * blockDim.x;
    int64_t t0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    uint32_t i_next = (t0 < Von && int(blockIdx.x) < compute_blocks) ? onlist[t0] : 0u;
    for (int64_t t = t0; t < Von && int(blockIdx.x) < compute_blocks; t += tstride) {
        const int64_t i = int64_t(i_next);
        i_next = t + tstride < Von ? onlist[t + tstride] : 0u;
        if (i >= n) continue;
        float s[10];
#pragma unroll
        for (int c = 0; c < 10; ++c) s[c] = sgrad[c * sld + t];   // rank-indexed (coalesced)
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
        const float4 r0 = rec[3 * i], r1 = rec[3 * i + 1];   // scaled conic: A = -a/2, B = -b, C = -c/2
        const float Q[2][2] = {{-2.f * r0.z, -r0.w}, {-r0.w, -2.f * r1.x}};
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
        // degree-1 SH colour (gs_project_sh, reading C29): per channel c, rgb = max(0, 1/2 + C0 Y0 +
        // C1 (-u_y Y1 + u_z Y2 - u_x Y3)), u = (X - c)/|X - c|, c = -W^T t. The clamp decision is
        // recomputed in the projection's fp32 order (same bits). gdir = dL/dX through u.
        float gdir[3] = {0.f, 0.f, 0.f};
        if (SH == 1) {
            const float cwx = -((V[0] * V[3] + V[4] * V[7]) + V[8] * V[11]);
            const float cwy = -((V[1] * V[3] + V[5] * V[7]) + V[9] * V[11]);
            const float cwz = -((V[2] * V[3] + V[6] * V[7]) + V[10] * V[11]);
            const float ddx = __fsub_rn(p[0], cwx), ddy = __fsub_rn(p[1], cwy), ddz = __fsub_rn(p[2], cwz);
            const float len = __fsqrt_rn(__fadd_rn(__fadd_rn(__fmul_rn(ddx, ddx), __fmul_rn(ddy, ddy)), __fmul_rn(ddz, ddz)));
            const float ux = __fdiv_rn(ddx, len), uy = __fdiv_rn(ddy, len), uz = __fdiv_rn(ddz, len);
            constexpr float C0 = 0.28209479177387814f, C1 = 0.4886025119029199f;
            float du[3] = {0.f, 0.f, 0.f};
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const float y1 = params[(14 + c) * ld + i], y2 = params[(17 + c) * ld + i], y3 = params[(20 + c) * ld + i];
                const float lin = __fsub_rn(__fadd_rn(-__fmul_rn(uy, y1), __fmul_rn(uz, y2)), __fmul_rn(ux, y3));
                const float v = __fadd_rn(__fadd_rn(__fmul_rn(C0, p[11 + c]), __fmul_rn(C1, lin)), 0.5f);
                const float gc = v > 0.f ? s[6 + c] : 0.f;   // clamped channel: no gradient
                if (grad) {
                    gacc(grad + ((11 + c) * ld + i), gc * C0, assign);
                    gacc(grad + ((14 + c) * ld + i), gc * (-C1 * uy), assign);
                    gacc(grad + ((17 + c) * ld + i), gc * (C1 * uz), assign);
                    gacc(grad + ((20 + c) * ld + i), gc * (-C1 * ux), assign);
                }
                du[0] -= gc * C1 * y3;
                du[1] -= gc * C1 * y1;
                du[2] += gc * C1 * y2;
            }
            const float ud = ux * du[0] + uy * du[1] + uz * du[2];
            const float il = 1.f / len;
            gdir[0] = (du[0] - ux * ud) * il;
            gdir[1] = (du[1] - uy * ud) * il;
            gdir[2] = (du[2] - uz * ud) * il;
        }
        if (grad) {
            // mean: W^T dX (+ the SH view-direction path)
#pragma unroll
            for (int k = 0; k < 3; ++k)
                gacc(grad + (k * ld + i), W[0][k] * dX[0] + W[1][k] * dX[1] + W[2][k] * dX[2] + gdir[k], assign);
            // Sigma = M M^T
            float dM[3][3];
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int k = 0; k < 3; ++k) dM[a][k] = 2.f * (dS[a][0] * M[0][k] + dS[a][1] * M[1][k] + dS[a][2] * M[2][k]);
#pragma unroll
            for (int k = 0; k < 3; ++k) gacc(grad + ((3 + k) * ld + i), dM[0][k] * R[0][k] + dM[1][k] * R[1][k] + dM[2][k] * R[2][k], assign);
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
            gacc(grad + (6 * ld + i), (dq[0] - qr * qd) / nq, assign);
            gacc(grad + (7 * ld + i), (dq[1] - qi * qd) / nq, assign);
            gacc(grad + (8 * ld + i), (dq[2] - qj * qd) / nq, assign);
            gacc(grad + (9 * ld + i), (dq[3] - qk * qd) / nq, assign);
            gacc(grad + (10 * ld + i), s[5], assign);
            if (SH == 0) {
                gacc(grad + (11 * ld + i), s[6], assign);
                gacc(grad + (12 * ld + i), s[7], assign);
                gacc(grad + (13 * ld + i), s[8], assign);
            }
        }
        if (pose_part) {
            const float g0 = cov_path ? dX[0] : dXm[0], g1 = cov_path ? dX[1] : dXm[1],
                        g2 = cov_path ? dX[2] : dXm[2];
            pose[0] += g0;
            pose[1] += g1;
            pose[2] += g2;
            if (cov_path && SH == 1) {   // colour through the camera centre: rho += W gdir (phi: none)
#pragma unroll
                for (int a = 0; a < 3; ++a) pose[a] += W[a][0] * gdir[0] + W[a][1] * gdir[1] + W[a][2] * gdir[2];
            }
            pose[3] += y * g2 - z * g1;
            pose[4] += z * g0 - x * g2;
            pose[5] += x * g1 - y * g0;
            if (cov_path) {
#pragma unroll
                for (int a = 0; a < 3; ++a)
#pragma unroll
                    for (int b = 0; b < 3; ++b) pose[6 + 3 * a + b] += J[0][a] * dE[0][b] + J[1][a] * dE[1][b];
            }
        }
    }
    if (ASSIGN && grad) {
        // off-screen columns get zero gradients: 2048-column chunks claimed from a counter, so blocks
        // with fewer items above take more chunks (a second wave of zeroing-only blocks would run
        // after the items: the grid is one wave at 2 blocks per SM)
        constexpr int kZeroChunk = 2048;
        const int rows = SH == 1 ? 23 : 14;
        __shared__ unsigned int s_chunk;
        for (;;) {
            if (threadIdx.x == 0) s_chunk = atomicAdd(zero_chunk, 1u);
            __syncthreads();
            const int64_t c0 = int64_t(s_chunk) * kZeroChunk;
            __syncthreads();   // s_chunk read by every thread before the next claim
            if (c0 >= n) break;
            const int64_t c1 = c0 + kZeroChunk < n ? c0 + kZeroChunk : n;
            for (int64_t i = c0 + threadIdx.x; i < c1; i += blockDim.x)
                if (tiles[i] == 0u)
                    for (int k = 0; k < rows; ++k) grad[k * ld + i] = 0.f;
        }
    }
    if (pose_part) {   // per-block partial sums (fp64), reduced in a fixed order by the last block
        __shared__ double red[8][kPoseSums];
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
        for (int k = 0; k < kPoseSums; ++k) {
            double v = double(pose[k]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) red[warp][k] = v;
        }
        __syncthreads();
        if (threadIdx.x < kPoseSums) {   // component-major: pose_part[k][block]
            double v = 0.0;
#pragma unroll
            for (int w = 0; w < 8; ++w) v += red[w][threadIdx.x];
            pose_part[size_t(threadIdx.x) * gridDim.x + blockIdx.x] = v;
            __threadfence();   // the writers publish their partials before the ticket (membar: writers only)
        }
        __syncthreads();
        if (threadIdx.x == 0) s_last = atomicAdd(done_ctr, 1u) == gridDim.x - 1;
        __syncthreads();
        if (s_last) {
            __threadfence();
            pose_finalize_block(pose_part, gridDim.x, viewmat, grad_pose, ASSIGN ? 1 : 0);
            if (lf.loss && threadIdx.x == 0) {   // fused L1: the loss scalar (as loss_finalize_kernel)
                const double nvalid = __ldcg(lf.acc + 2);
                const float sc = float(double(lf.wc) / (3.0 * double(lf.npx)));
                const float sd = nvalid > 0 ? float(double(lf.wd) / nvalid) : 0.f;
                *lf.loss = double(sc) * __ldcg(lf.acc) + (nvalid > 0 ? double(sd) * __ldcg(lf.acc + 1) : 0.0);
            }
            if (threadIdx.x == 0) *done_ctr = 0u;   // ready for the next call
        }
    }
}

// Fixed-order reduction of the per-block pose partials (by the last block of gaussian_bwd_kernel), then
// twist = (rho, phi + (A12 - A21, A20 - A02, A01 - A10)),  A = W (sum dW_cov)^T
__device__ void pose_finalize_block(const double* __restrict__ part, int nblocks, const float* __restrict__ viewmat,
                                    double* __restrict__ grad_pose, int assign) {
    __shared__ double acc[16];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;   // warp w sums components w, w + 8
    for (int k = w; k < kPoseSums; k += 8) {
        double v = 0.0;
        for (int b = lane; b < nblocks; b += 32) v += __ldcg(part + size_t(k) * nblocks + b);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) acc[k] = v;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    double W[3][3], A[3][3];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) W[a][b] = viewmat[4 * a + b];
    const double* dW = acc + 6;
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) A[a][b] = W[a][0] * dW[3 * b + 0] + W[a][1] * dW[3 * b + 1] + W[a][2] * dW[3 * b + 2];
    const double tw[6] = {acc[0], acc[1], acc[2], acc[3] + (A[1][2] - A[2][1]), acc[4] + (A[2][0] - A[0][2]),
                          acc[5] + (A[0][1] - A[1][0])};
    for (int k = 0; k < 6; ++k) grad_pose[k] = (assign ? 0.0 : grad_pose[k]) + tw[k];
}

void launch_gaussian_bwd(WsState* s, const float* params, int64_t n, int64_t ld, const float* viewmat,
                         const gs_camera& cam, float* grad_params, double* grad_pose, uint32_t flags, cudaStream_t st,
                         LossFin lf) {
    if (n == 0) return;
    double* part = grad_pose ? at<double>(s, s->pose_part) : nullptr;
    const int sms = sm_count();
    // grid sized without a host sync: at most 4 blocks per SM, at most ceil(n / 256)
    const int blocks = int(std::min<int64_t>((n + 255) / 256, int64_t(sms) * kGbwdBlocksPerSM));
    KTimer kt(s, KID_BWD_GAUSS, st);
    const int assign = (flags & GS_FLAG_GRAD_ASSIGN) ? 1 : 0;
    auto kern = s->sh_degree == 1 ? (assign ? gaussian_bwd_kernel<1, true> : gaussian_bwd_kernel<1, false>)
                                  : (assign ? gaussian_bwd_kernel<0, true> : gaussian_bwd_kernel<0, false>);
    launch_pdl(kern, dim3(blocks), dim3(256), 0, st,
        params, n, ld, viewmat, cam, at<uint32_t>(s, s->onlist), &at<Misc>(s, s->misc)->n_onscreen,
        at<float4>(s, s->rec), at<float>(s, s->sgrad), s->n_cap, grad_params, (flags & GS_FLAG_POSE_COV_PATH) ? 1 : 0,
        part, &at<Misc>(s, s->misc)->pose_done, grad_pose, part ? lf : LossFin{}, at<uint32_t>(s, s->tiles),
        &at<Misc>(s, s->misc)->gbwd_zero_chunk);
}

}  // namespace gs
