// gs_loss_l1, gs_adam_step, gs_pose_step, gs_densify_prune kernels (sm_100a).
// All elementwise / compaction work is HBM-bound; no host synchronisation (device counts).
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "gs_internal.cuh"

namespace gs {

// ------------------------------------------------------------------ L1 loss, Eq. 6 (reading C20)
// Two passes (the depth term's scale needs the valid-pixel count first). Both read four pixels per
// thread per step with 16-B loads when the planes are 16-B aligned (npx % 4 == 0), else one.
// Per-thread sums are fp32 over a few pixels; blocks reduce in fp64.
template <int V>
struct LossVec;
template <>
struct LossVec<4> {
    using T = float4;
    __device__ static float4 ld(const float* p, int64_t i) { return reinterpret_cast<const float4*>(p)[i]; }
    __device__ static void st(float* p, int64_t i, float4 v) { reinterpret_cast<float4*>(p)[i] = v; }
    __device__ static float get(const float4& v, int e) { return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w; }
    __device__ static void set(float4& v, int e, float x) {
        if (e == 0) v.x = x; else if (e == 1) v.y = x; else if (e == 2) v.z = x; else v.w = x;
    }
};
template <>
struct LossVec<1> {
    using T = float;
    __device__ static float ld(const float* p, int64_t i) { return p[i]; }
    __device__ static void st(float* p, int64_t i, float v) { p[i] = v; }
    __device__ static float get(const float& v, int) { return v; }
    __device__ static void set(float& v, int, float x) { v = x; }
};

template <int V>
__global__ void __launch_bounds__(256) loss_reduce_kernel(const float* __restrict__ c, const float* __restrict__ d,
                                                          const float* __restrict__ tc, const float* __restrict__ td,
                                                          int64_t npx, double* __restrict__ acc) {
    using L = LossVec<V>;
    const int64_t nv = npx / V;   // vectors per plane
    float sc = 0.f, sd = 0.f, cn = 0.f;
    for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < nv; q += int64_t(gridDim.x) * blockDim.x) {
        const auto c0 = L::ld(c, q), c1 = L::ld(c + npx, q), c2 = L::ld(c + 2 * npx, q);
        const auto t0 = L::ld(tc, q), t1 = L::ld(tc + npx, q), t2 = L::ld(tc + 2 * npx, q);
        const auto dv = L::ld(d, q), tv = L::ld(td, q);
#pragma unroll
        for (int e = 0; e < V; ++e) {
            sc += fabsf(L::get(c0, e) - L::get(t0, e)) + fabsf(L::get(c1, e) - L::get(t1, e)) +
                  fabsf(L::get(c2, e) - L::get(t2, e));
            const float t = L::get(tv, e);
            if (t > 0.f) {
                sd += fabsf(L::get(dv, e) - t);
                cn += 1.f;
            }
        }
    }
    using BR = cub::BlockReduce<double, 256>;
    __shared__ typename BR::TempStorage tmp;
    const double a = BR(tmp).Sum(double(sc));
    __syncthreads();
    const double b = BR(tmp).Sum(double(sd));
    __syncthreads();
    const double e = BR(tmp).Sum(double(cn));
    if (threadIdx.x == 0) {
        atomicAdd(acc + 0, a);
        atomicAdd(acc + 1, b);
        atomicAdd(acc + 2, e);
    }
}

__device__ __forceinline__ float sgnf(float x) { return float((x > 0.f) - (x < 0.f)); }

template <int V>
__global__ void __launch_bounds__(256) loss_grad_kernel(const float* __restrict__ c, const float* __restrict__ d,
                                                        const float* __restrict__ tc, const float* __restrict__ td,
                                                        int64_t npx, float wc, float wd, const double* __restrict__ acc,
                                                        float* __restrict__ dc, float* __restrict__ dd,
                                                        double* __restrict__ loss) {
    using L = LossVec<V>;
    const double nvalid = acc[2];
    const float sc = float(double(wc) / (3.0 * double(npx)));
    const float sd = nvalid > 0 ? float(double(wd) / nvalid) : 0.f;
    if (blockIdx.x == 0 && threadIdx.x == 0 && loss)
        *loss = double(sc) * acc[0] + (nvalid > 0 ? double(sd) * acc[1] : 0.0);
    const int64_t nv = npx / V;
    for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < nv; q += int64_t(gridDim.x) * blockDim.x) {
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            const auto cv = L::ld(c + ch * npx, q), tv = L::ld(tc + ch * npx, q);
            typename L::T o;
#pragma unroll
            for (int e = 0; e < V; ++e) L::set(o, e, sc * sgnf(L::get(cv, e) - L::get(tv, e)));
            L::st(dc + ch * npx, q, o);
        }
        const auto dv = L::ld(d, q), tv = L::ld(td, q);
        typename L::T o;
#pragma unroll
        for (int e = 0; e < V; ++e) {
            const float t = L::get(tv, e);
            L::set(o, e, t > 0.f ? sd * sgnf(L::get(dv, e) - t) : 0.f);
        }
        L::st(dd, q, o);
    }
}

void launch_loss_l1(WsState* s, const float* color, const float* depth, const float* tc, const float* td, int32_t W,
                    int32_t H, float wc, float wd, float* dc, float* dd, double* loss, cudaStream_t st) {
    Misc* misc = at<Misc>(s, s->misc);
    const int64_t npx = int64_t(W) * H;
    launch_zero(misc->loss_acc, sizeof(misc->loss_acc), st, s);
    auto aligned = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    const bool v4 = npx % 4 == 0 && aligned(color) && aligned(depth) && aligned(tc) && aligned(td) && aligned(dc) &&
                    aligned(dd);
    const int64_t nv = v4 ? npx / 4 : npx;
    const int blocks = int(std::min<int64_t>((nv + 255) / 256, sm_count() * 4));
    {
        KTimer kt(s, KID_LOSS, st);
        if (v4) loss_reduce_kernel<4><<<blocks, 256, 0, st>>>(color, depth, tc, td, npx, misc->loss_acc);
        else loss_reduce_kernel<1><<<blocks, 256, 0, st>>>(color, depth, tc, td, npx, misc->loss_acc);
    }
    KTimer kt(s, KID_LOSS, st);
    if (v4) loss_grad_kernel<4><<<blocks, 256, 0, st>>>(color, depth, tc, td, npx, wc, wd, misc->loss_acc, dc, dd, loss);
    else loss_grad_kernel<1><<<blocks, 256, 0, st>>>(color, depth, tc, td, npx, wc, wd, misc->loss_acc, dc, dd, loss);
}

int coop_sm_count() {
    static std::atomic<int> cached[64];   // zero-initialised (static storage); per device
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 0;
    int v = cached[dev].load(std::memory_order_relaxed);
    if (!v) {
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
        cached[dev].store(v, std::memory_order_relaxed);
    }
    return v;
}

// ------------------------------------------------------------------ tracking front end (NEXT-4)
// masked L1 (reading C31): pass 1 counts / sums over the observed pixels, pass 2 writes the gradients
__global__ void __launch_bounds__(256) loss_masked_reduce_kernel(const float* __restrict__ c,
                                                                 const float* __restrict__ d,
                                                                 const float* __restrict__ tc,
                                                                 const float* __restrict__ td,
                                                                 const float* __restrict__ alpha, float amin,
                                                                 int64_t npx, double* __restrict__ acc) {
    float sc = 0.f, sd = 0.f, nobs = 0.f, nv = 0.f;
    for (int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < npx; p += int64_t(gridDim.x) * blockDim.x) {
        if (!(alpha[p] >= amin)) continue;
        nobs += 1.f;
        sc += fabsf(c[p] - tc[p]) + fabsf(c[npx + p] - tc[npx + p]) + fabsf(c[2 * npx + p] - tc[2 * npx + p]);
        const float t = td[p];
        if (t > 0.f) {
            sd += fabsf(d[p] - t);
            nv += 1.f;
        }
    }
    using BR = cub::BlockReduce<double, 256>;
    __shared__ typename BR::TempStorage tmp;
    const double v[4] = {double(sc), double(sd), double(nv), double(nobs)};
    for (int k = 0; k < 4; ++k) {
        const double r = BR(tmp).Sum(v[k]);
        if (threadIdx.x == 0) atomicAdd(acc + k, r);
        __syncthreads();
    }
}

__global__ void __launch_bounds__(256) loss_masked_grad_kernel(const float* __restrict__ c, const float* __restrict__ d,
                                                               const float* __restrict__ tc,
                                                               const float* __restrict__ td,
                                                               const float* __restrict__ alpha, float amin,
                                                               int64_t npx, float wc, float wd,
                                                               const double* __restrict__ acc, float* __restrict__ dc,
                                                               float* __restrict__ dd, double* __restrict__ loss) {
    const double nvalid = acc[2], nobs = acc[3];
    const float sc = nobs > 0 ? float(double(wc) / (3.0 * nobs)) : 0.f;
    const float sd = nvalid > 0 ? float(double(wd) / nvalid) : 0.f;
    if (blockIdx.x == 0 && threadIdx.x == 0 && loss)
        *loss = (nobs > 0 ? double(sc) * acc[0] : 0.0) + (nvalid > 0 ? double(sd) * acc[1] : 0.0);
    for (int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < npx; p += int64_t(gridDim.x) * blockDim.x) {
        const bool obs = alpha[p] >= amin;
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) dc[ch * npx + p] = obs ? sc * sgnf(c[ch * npx + p] - tc[ch * npx + p]) : 0.f;
        const float t = td[p];
        dd[p] = (obs && t > 0.f) ? sd * sgnf(d[p] - t) : 0.f;
    }
}

// 10x-median pixel rejection (reading C32), one cooperative kernel: the per-pixel
// colour loss l_p = (|dC_0| + |dC_1|) + |dC_2| (fp32) of the observed pixels is non-negative, so its
// bit pattern orders like the value; a three-pass radix select (11 + 11 + 9 bits, block histograms
// -> global histogram -> every CTA scans it) finds the lower median m (rank floor((N_obs - 1) / 2)).
// Pixels with l_p > k m (fp32) are dropped from both loss terms; then the masked reduction and the
// gradient pass run as above. l_p is recomputed each pass from the images (28 B/px, L2-resident
// after the first pass) rather than stored.
struct RobustScratch {   // in the workspace's coop region, zeroed before the launch
    uint32_t h0[2048], h1[2048], h2[512];
    uint32_t bar, nobs, pad[2];
};

__device__ __forceinline__ uint32_t pixel_loss_bits(const float* __restrict__ c, const float* __restrict__ tc,
                                                    int64_t npx, int64_t p) {
    const float l = __fadd_rn(__fadd_rn(fabsf(c[p] - tc[p]), fabsf(c[npx + p] - tc[npx + p])),
                              fabsf(c[2 * npx + p] - tc[2 * npx + p]));
    return __float_as_uint(l);
}

// every CTA: find the bin of rank k in hist[nb] (ld.cg: written by other CTAs before the barrier);
// returns the bin and leaves the rank within it in k
template <int NB>
__device__ __forceinline__ uint32_t select_bin(const uint32_t* hist, uint32_t& k, uint32_t* sh) {
    using BS = cub::BlockScan<uint32_t, 1024>;
    __shared__ typename BS::TempStorage tmp;
    constexpr int PER = (NB + 1023) / 1024;
    uint32_t v[PER], tot = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const int b = threadIdx.x * PER + j;
        v[j] = b < NB ? __ldcg(hist + b) : 0u;
        tot += v[j];
    }
    uint32_t ex;
    BS(tmp).ExclusiveSum(tot, ex);
    if (ex <= k && k < ex + tot) {   // exactly one thread holds rank k
        uint32_t run = ex;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            if (run <= k && k < run + v[j]) {
                sh[0] = threadIdx.x * PER + j;
                sh[1] = k - run;
            }
            run += v[j];
        }
    }
    __syncthreads();
    const uint32_t b = sh[0];
    k = sh[1];
    __syncthreads();
    return b;
}

__global__ void __launch_bounds__(1024, 1) loss_robust_kernel(const float* __restrict__ c, const float* __restrict__ d,
                                                              const float* __restrict__ tc,
                                                              const float* __restrict__ td,
                                                              const float* __restrict__ alpha, float amin, float kout,
                                                              int64_t npx, float wc, float wd, RobustScratch* rs,
                                                              double* __restrict__ acc, float* __restrict__ dc,
                                                              float* __restrict__ dd, double* __restrict__ loss) {
    __shared__ uint32_t sh_h[2048];
    __shared__ uint32_t sh[4];
    unsigned int goal = 0;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    const int64_t p0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    // pass 1: top 11 bits (bit 31 is the sign: 0)
    for (int b = threadIdx.x; b < 2048; b += blockDim.x) sh_h[b] = 0;
    __syncthreads();
    uint32_t nobs = 0;
    for (int64_t p = p0; p < npx; p += stride) {
        if (!(alpha[p] >= amin)) continue;
        ++nobs;
        atomicAdd(sh_h + (pixel_loss_bits(c, tc, npx, p) >> 20), 1u);
    }
    nobs = __reduce_add_sync(0xffffffffu, nobs);
    if ((threadIdx.x & 31) == 0 && nobs) atomicAdd(&rs->nobs, nobs);
    __syncthreads();
    for (int b = threadIdx.x; b < 2048; b += blockDim.x)
        if (sh_h[b]) atomicAdd(rs->h0 + b, sh_h[b]);
    grid_sync(&rs->bar, goal);
    const uint32_t n_obs = __ldcg(&rs->nobs);
    float thr = -1.f;   // no observed pixel: nothing kept
    if (n_obs > 0) {
        uint32_t k = (n_obs - 1) / 2;
        const uint32_t b0 = select_bin<2048>(rs->h0, k, sh);
        // pass 2: bits 20..9 of the pixels in bin b0
        for (int b = threadIdx.x; b < 2048; b += blockDim.x) sh_h[b] = 0;
        __syncthreads();
        for (int64_t p = p0; p < npx; p += stride) {
            if (!(alpha[p] >= amin)) continue;
            const uint32_t key = pixel_loss_bits(c, tc, npx, p);
            if ((key >> 20) == b0) atomicAdd(sh_h + ((key >> 9) & 2047u), 1u);
        }
        __syncthreads();
        for (int b = threadIdx.x; b < 2048; b += blockDim.x)
            if (sh_h[b]) atomicAdd(rs->h1 + b, sh_h[b]);
        grid_sync(&rs->bar, goal);
        const uint32_t b1 = select_bin<2048>(rs->h1, k, sh);
        const uint32_t hi = (b0 << 11) | b1;
        // pass 3: bits 8..0
        for (int b = threadIdx.x; b < 512; b += blockDim.x) sh_h[b] = 0;
        __syncthreads();
        for (int64_t p = p0; p < npx; p += stride) {
            if (!(alpha[p] >= amin)) continue;
            const uint32_t key = pixel_loss_bits(c, tc, npx, p);
            if ((key >> 9) == hi) atomicAdd(sh_h + (key & 511u), 1u);
        }
        __syncthreads();
        for (int b = threadIdx.x; b < 512; b += blockDim.x)
            if (sh_h[b]) atomicAdd(rs->h2 + b, sh_h[b]);
        grid_sync(&rs->bar, goal);
        const uint32_t b2 = select_bin<512>(rs->h2, k, sh);
        thr = __fmul_rn(kout, __uint_as_float((hi << 9) | b2));
    }
    // pass 4: sums over the kept pixels
    float sc = 0.f, sd = 0.f, nk = 0.f, nv = 0.f;
    for (int64_t p = p0; p < npx; p += stride) {
        if (!(alpha[p] >= amin) || !(__uint_as_float(pixel_loss_bits(c, tc, npx, p)) <= thr)) continue;
        nk += 1.f;
        sc += fabsf(c[p] - tc[p]) + fabsf(c[npx + p] - tc[npx + p]) + fabsf(c[2 * npx + p] - tc[2 * npx + p]);
        const float t = td[p];
        if (t > 0.f) {
            sd += fabsf(d[p] - t);
            nv += 1.f;
        }
    }
    {
        using BR = cub::BlockReduce<double, 1024>;
        __shared__ typename BR::TempStorage tmp;
        const double v[4] = {double(sc), double(sd), double(nv), double(nk)};
        for (int q = 0; q < 4; ++q) {
            const double r = BR(tmp).Sum(v[q]);
            if (threadIdx.x == 0) atomicAdd(acc + q, r);
            __syncthreads();
        }
    }
    grid_sync(&rs->bar, goal);
    // pass 5: gradients
    const double nvalid = __ldcg(acc + 2), nkept = __ldcg(acc + 3);
    const float scl = nkept > 0 ? float(double(wc) / (3.0 * nkept)) : 0.f;
    const float sdl = nvalid > 0 ? float(double(wd) / nvalid) : 0.f;
    if (blockIdx.x == 0 && threadIdx.x == 0 && loss)
        *loss = (nkept > 0 ? double(scl) * __ldcg(acc) : 0.0) + (nvalid > 0 ? double(sdl) * __ldcg(acc + 1) : 0.0);
    for (int64_t p = p0; p < npx; p += stride) {
        const bool kept = alpha[p] >= amin && __uint_as_float(pixel_loss_bits(c, tc, npx, p)) <= thr;
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) dc[ch * npx + p] = kept ? scl * sgnf(c[ch * npx + p] - tc[ch * npx + p]) : 0.f;
        const float t = td[p];
        dd[p] = (kept && t > 0.f) ? sdl * sgnf(d[p] - t) : 0.f;
    }
}

void launch_loss_l1_masked(WsState* s, const float* color, const float* depth, const float* tc, const float* td,
                           const float* alpha, float amin, float outlier_k, int32_t W, int32_t H, float wc, float wd,
                           float* dc, float* dd, double* loss, cudaStream_t st) {
    Misc* misc = at<Misc>(s, s->misc);
    const int64_t npx = int64_t(W) * H;
    launch_zero(misc->loss_acc, sizeof(misc->loss_acc), st, s);
    if (outlier_k > 0.f) {
        RobustScratch* rs = at<RobustScratch>(s, s->coop);
        launch_zero(rs, sizeof(RobustScratch), st, s);
        const int grid = coop_sm_count();
        if (grid <= 0) return;   // check_launch reports the device error
        int64_t n = npx;
        double* acc = misc->loss_acc;
        void* args[] = {&color, &depth, &tc, &td, &alpha, &amin, &outlier_k, &n, &wc, &wd, &rs, &acc, &dc, &dd, &loss};
        KTimer kt(s, KID_LOSS, st);
        cudaLaunchCooperativeKernel(reinterpret_cast<void*>(loss_robust_kernel), dim3(grid), dim3(1024), args, 0, st);
        return;
    }
    const int blocks = int(std::min<int64_t>((npx + 255) / 256, sm_count() * 4));
    {
        KTimer kt(s, KID_LOSS, st);
        loss_masked_reduce_kernel<<<blocks, 256, 0, st>>>(color, depth, tc, td, alpha, amin, npx, misc->loss_acc);
    }
    KTimer kt(s, KID_LOSS, st);
    loss_masked_grad_kernel<<<blocks, 256, 0, st>>>(color, depth, tc, td, alpha, amin, npx, wc, wd, misc->loss_acc,
                                                    dc, dd, loss);
}

__global__ void frame_stats_kernel(const float* __restrict__ alpha, const float* __restrict__ depth,
                                   const float* __restrict__ td, int64_t npx, float ta, float tdep,
                                   uint32_t* __restrict__ counts) {
    uint32_t rel = 0, val = 0, obs = 0;
    for (int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < npx; p += int64_t(gridDim.x) * blockDim.x) {
        const float t = td[p];
        const bool o = alpha[p] >= ta;
        obs += o;
        if (t > 0.f) {
            ++val;
            rel += (o && fabsf(t - depth[p]) <= tdep) ? 1u : 0u;
        }
    }
#pragma unroll
    for (int k = 16; k > 0; k >>= 1) {
        rel += __shfl_xor_sync(0xffffffffu, rel, k);
        val += __shfl_xor_sync(0xffffffffu, val, k);
        obs += __shfl_xor_sync(0xffffffffu, obs, k);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(counts + 0, rel);
        atomicAdd(counts + 1, val);
        atomicAdd(counts + 2, obs);
    }
}

void launch_frame_stats(const float* alpha, const float* depth, const float* td, int32_t W, int32_t H, float ta,
                        float tdep, uint32_t* counts, cudaStream_t st) {
    launch_zero(counts, 3 * sizeof(uint32_t), st);
    const int64_t npx = int64_t(W) * H;
    frame_stats_kernel<<<int(std::min<int64_t>((npx + 255) / 256, sm_count() * 2)), 256, 0, st>>>(alpha, depth, td, npx, ta,
                                                                                           tdep, counts);
}

// constant velocity: out = (T2 T1^-1) T2 for world->camera [R | t] poses, fp64
__global__ void pose_extrapolate_kernel(const float* __restrict__ t1, const float* __restrict__ t2,
                                        float* __restrict__ out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double R1[3][3], R2[3][3], a[3], b[3];
    for (int i = 0; i < 3; ++i) {
        for (int j = 0; j < 3; ++j) {
            R1[i][j] = t1[4 * i + j];
            R2[i][j] = t2[4 * i + j];
        }
        a[i] = t1[4 * i + 3];
        b[i] = t2[4 * i + 3];
    }
    // D = T2 T1^-1: R_D = R2 R1^T, t_D = b - R_D a;  out = D T2: R = R_D R2, t = R_D b + t_D
    double RD[3][3], tD[3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) RD[i][j] = R2[i][0] * R1[j][0] + R2[i][1] * R1[j][1] + R2[i][2] * R1[j][2];
    for (int i = 0; i < 3; ++i) tD[i] = b[i] - (RD[i][0] * a[0] + RD[i][1] * a[1] + RD[i][2] * a[2]);
    for (int i = 0; i < 3; ++i) {
        for (int j = 0; j < 3; ++j)
            out[4 * i + j] = float(RD[i][0] * R2[0][j] + RD[i][1] * R2[1][j] + RD[i][2] * R2[2][j]);
        out[4 * i + 3] = float(RD[i][0] * b[0] + RD[i][1] * b[1] + RD[i][2] * b[2] + tD[i]);
    }
}

// 2x2 mean of the RGB-D frame for the coarse stage (reading C12's half-resolution camera: half
// pixel (u, v) covers full pixels 2u..2u+1 x 2v..2v+1): colour ((c00 + c01) + (c10 + c11)) * 0.25,
// depth the mean of the valid (> 0) samples in the order 00, 01, 10, 11, else 0.
__global__ void image_half_kernel(const float* __restrict__ c, const float* __restrict__ d, int W, int H,
                                  float* __restrict__ ch, float* __restrict__ dh) {
    const int Wh = W / 2, Hh = H / 2;
    const int64_t nh = int64_t(Wh) * Hh, n = int64_t(W) * H;
    for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < nh; q += int64_t(gridDim.x) * blockDim.x) {
        const int v = int(q / Wh), u = int(q - int64_t(v) * Wh);
        const int64_t p00 = int64_t(2 * v) * W + 2 * u, p10 = p00 + W;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const float* ck = c + k * n;
            ch[k * nh + q] = __fmul_rn(__fadd_rn(__fadd_rn(ck[p00], ck[p00 + 1]), __fadd_rn(ck[p10], ck[p10 + 1])), 0.25f);
        }
        const float ds[4] = {d[p00], d[p00 + 1], d[p10], d[p10 + 1]};
        float s = 0.f;
        int cnt = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (ds[k] > 0.f) {
                s = __fadd_rn(s, ds[k]);
                ++cnt;
            }
        dh[q] = cnt ? __fdiv_rn(s, float(cnt)) : 0.f;
    }
}

void launch_image_half(const float* c, const float* d, int32_t W, int32_t H, float* ch, float* dh, cudaStream_t st) {
    const int64_t nh = int64_t(W / 2) * (H / 2);
    if (nh == 0) return;
    const int blocks = int(std::min<int64_t>((nh + 255) / 256, sm_count() * 8));
    image_half_kernel<<<blocks, 256, 0, st>>>(c, d, W, H, ch, dh);
}

void launch_pose_extrapolate(const float* t1, const float* t2, float* out, cudaStream_t st) {
    pose_extrapolate_kernel<<<1, 32, 0, st>>>(t1, t2, out);
}

__global__ void zero_u32_kernel(uint32_t* __restrict__ p, size_t nw) {
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nw; i += size_t(gridDim.x) * blockDim.x) p[i] = 0u;
}

void launch_zero(void* p, size_t bytes, cudaStream_t st, WsState* s) {
    const size_t nw = bytes / 4;
    if (nw == 0) return;
    if (s) s->launches += 1;
    const int blocks = int(std::min<size_t>((nw + 255) / 256, 64));
    zero_u32_kernel<<<blocks, 256, 0, st>>>(static_cast<uint32_t*>(p), nw);
}

// ------------------------------------------------------------------ Adam
struct Lr14 { float v[23]; };   // per-row rates: 14 (RGB) or 23 (degree-1 SH) rows

__device__ __forceinline__ float adam_one(float r, float gr, float& m, float& v, int k, float lrk, float b1, float b2,
                                         float eps, float bc1, float bc2, float& act) {
    if (k >= 3 && k < 6) gr *= expf(r);                       // d/dlog s = s d/ds
    else if (k == 10) { const float s = 1.f / (1.f + expf(-r)); gr *= s * (1.f - s); }   // d/dlogit o
    m = b1 * m + (1.f - b1) * gr;
    v = b2 * v + (1.f - b2) * gr * gr;
    const float nr = r - lrk * (m / bc1) / (sqrtf(v / bc2) + eps);
    act = (k >= 3 && k < 6) ? expf(nr) : (k == 10 ? 1.f / (1.f + expf(-nr)) : nr);
    return nr;
}

// One row per blockIdx.y. With 16-byte aligned arrays the row body moves float4s (the row's
// unaligned head and tail go element by element): 4x the bytes in flight per load instruction, which
// the elementwise update needs to approach HBM bandwidth (~0.9 GB per step at 2M x 14).
__global__ void __launch_bounds__(256) adam_kernel(float* __restrict__ raw, float* __restrict__ act,
                                                   const float* __restrict__ g, float* __restrict__ m,
                                                   float* __restrict__ v, int64_t n, int64_t ld, Lr14 lr, float b1,
                                                   float b2, float eps, float bc1, float bc2, bool vec) {
    const int k = blockIdx.y;
    const float lrk = lr.v[k];
    const int64_t row = k * ld;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x, t0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    int64_t head = n, body_end = n;
    if (vec) {
        head = std::min<int64_t>(n, (4 - (row & 3)) & 3);
        body_end = head + ((n - head) & ~int64_t(3));
    }
    auto one = [&](int64_t i) {
        const int64_t o = row + i;
        float mm = m[o], vv = v[o], a;
        raw[o] = adam_one(raw[o], g[o], mm, vv, k, lrk, b1, b2, eps, bc1, bc2, a);
        m[o] = mm;
        v[o] = vv;
        act[o] = a;
    };
    for (int64_t i = t0; i < head; i += stride) one(i);
    if (!vec) return;
    for (int64_t q = t0; head + 4 * q < body_end; q += stride) {
        const int64_t o = row + head + 4 * q;
        const float4 r4 = *reinterpret_cast<const float4*>(raw + o), g4 = *reinterpret_cast<const float4*>(g + o);
        float4 m4 = *reinterpret_cast<const float4*>(m + o), v4 = *reinterpret_cast<const float4*>(v + o);
        float4 nr, a4;
        nr.x = adam_one(r4.x, g4.x, m4.x, v4.x, k, lrk, b1, b2, eps, bc1, bc2, a4.x);
        nr.y = adam_one(r4.y, g4.y, m4.y, v4.y, k, lrk, b1, b2, eps, bc1, bc2, a4.y);
        nr.z = adam_one(r4.z, g4.z, m4.z, v4.z, k, lrk, b1, b2, eps, bc1, bc2, a4.z);
        nr.w = adam_one(r4.w, g4.w, m4.w, v4.w, k, lrk, b1, b2, eps, bc1, bc2, a4.w);
        *reinterpret_cast<float4*>(raw + o) = nr;
        *reinterpret_cast<float4*>(m + o) = m4;
        *reinterpret_cast<float4*>(v + o) = v4;
        *reinterpret_cast<float4*>(act + o) = a4;
    }
    for (int64_t i = body_end + t0; i < n; i += stride) one(i);
}

void launch_adam(float* raw, float* act, const float* g, float* m, float* v, int64_t n, int64_t ld, const float* lr,
                 int32_t rows, int32_t step, float b1, float b2, float eps, cudaStream_t st) {
    if (n == 0) return;
    Lr14 l{};
    for (int k = 0; k < rows; ++k) l.v[k] = lr[k];
    const float bc1 = float(1.0 - std::pow(double(b1), step)), bc2 = float(1.0 - std::pow(double(b2), step));
    const bool vec = ((reinterpret_cast<uintptr_t>(raw) | reinterpret_cast<uintptr_t>(act) |
                       reinterpret_cast<uintptr_t>(g) | reinterpret_cast<uintptr_t>(m) |
                       reinterpret_cast<uintptr_t>(v)) & 15) == 0;
    const int64_t work = vec ? (n + 3) / 4 : n;
    dim3 grid(unsigned(std::min<int64_t>((work + 255) / 256, sm_count() * 8)), unsigned(rows));
    adam_kernel<<<grid, 256, 0, st>>>(raw, act, g, m, v, n, ld, l, b1, b2, eps, bc1, bc2, vec);
}

// ------------------------------------------------------------------ pose step (reading C23)
__global__ void pose_step_kernel(float* viewmat, const double* gp, float* m6, float* v6, int32_t step, float lr_rho,
                                 float lr_phi) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const double b1 = 0.9, b2 = 0.999, eps = 1e-8;
    const double bc1 = 1.0 - pow(b1, step), bc2 = 1.0 - pow(b2, step);
    double d[6];
    for (int k = 0; k < 6; ++k) {
        const double g = gp[k];
        const double mm = b1 * m6[k] + (1 - b1) * g, vv = b2 * v6[k] + (1 - b2) * g * g;
        m6[k] = float(mm);
        v6[k] = float(vv);
        d[k] = -double(k < 3 ? lr_rho : lr_phi) * (mm / bc1) / (sqrt(vv / bc2) + eps);
    }
    // exp(delta^): Rodrigues + V(phi) rho
    const double px = d[3], py = d[4], pz = d[5];
    const double th2 = px * px + py * py + pz * pz, th = sqrt(th2);
    const double K[3][3] = {{0, -pz, py}, {pz, 0, -px}, {-py, px, 0}};
    double K2[3][3];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) K2[a][b] = K[a][0] * K[0][b] + K[a][1] * K[1][b] + K[a][2] * K[2][b];
    double A, B, C;
    if (th < 1e-8) { A = 1.0; B = 0.5; C = 1.0 / 6.0; }
    else { A = sin(th) / th; B = (1 - cos(th)) / th2; C = (th - sin(th)) / (th2 * th); }
    double R[3][3], Vm[3][3];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
            const double I = a == b ? 1.0 : 0.0;
            R[a][b] = I + A * K[a][b] + B * K2[a][b];
            Vm[a][b] = I + B * K[a][b] + C * K2[a][b];
        }
    double W[3][3], t[3];
    for (int a = 0; a < 3; ++a) {
        for (int b = 0; b < 3; ++b) W[a][b] = viewmat[4 * a + b];
        t[a] = viewmat[4 * a + 3];
    }
    for (int a = 0; a < 3; ++a) {
        for (int b = 0; b < 3; ++b) viewmat[4 * a + b] = float(R[a][0] * W[0][b] + R[a][1] * W[1][b] + R[a][2] * W[2][b]);
        viewmat[4 * a + 3] = float(R[a][0] * t[0] + R[a][1] * t[1] + R[a][2] * t[2] + Vm[a][0] * d[0] +
                                   Vm[a][1] * d[1] + Vm[a][2] * d[2]);
    }
}

void launch_pose_step(float* viewmat, const double* gp, float* m6, float* v6, int32_t step, float lr_rho, float lr_phi,
                      cudaStream_t st) {
    pose_step_kernel<<<1, 32, 0, st>>>(viewmat, gp, m6, v6, step, lr_rho, lr_phi);
}

// ------------------------------------------------------------------ densify / prune / select
// Ordered compaction: a block-local scan + one look-back per block would do; counts here are
// small (pixels / Gaussians), so a two-level scan is used: per-block counts -> exclusive scan
// of the block counts in one block -> scatter. Deterministic (order-preserving).
constexpr int kCmpThreads = 256, kCmpItems = 8, kCmpTile = kCmpThreads * kCmpItems;

template <class Pred>
__global__ void __launch_bounds__(kCmpThreads) count_kernel(int64_t n, const int64_t* n_dev, Pred pred,
                                                            uint32_t* __restrict__ block_counts) {
    using BR = cub::BlockReduce<uint32_t, kCmpThreads>;
    __shared__ typename BR::TempStorage tmp;
    const int64_t nn = n_dev ? *n_dev : n;
    const int64_t base = int64_t(blockIdx.x) * kCmpTile;
    uint32_t c = 0;
    for (int k = 0; k < kCmpItems; ++k) {
        const int64_t i = base + int64_t(threadIdx.x) * kCmpItems + k;
        if (i < nn && pred(i)) ++c;
    }
    const uint32_t tot = BR(tmp).Sum(c);
    if (threadIdx.x == 0) block_counts[blockIdx.x] = tot;
}

// exclusive scan of nb block counts (single block, sequential chunks of 1024)
__global__ void scan_blocks_kernel(uint32_t* __restrict__ counts, int nb, unsigned long long* __restrict__ total) {
    using BS = cub::BlockScan<uint32_t, 1024>;
    __shared__ typename BS::TempStorage tmp;
    __shared__ uint32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < nb; base += 1024) {
        const int i = base + threadIdx.x;
        const uint32_t v = i < nb ? counts[i] : 0u;
        uint32_t ex, agg;
        BS(tmp).ExclusiveSum(v, ex, agg);
        if (i < nb) counts[i] = carry + ex;
        __syncthreads();
        if (threadIdx.x == 0) carry += agg;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = carry;
}

template <class Pred, class Emit>
__global__ void __launch_bounds__(kCmpThreads) scatter_kernel(int64_t n, const int64_t* n_dev, Pred pred, Emit emit,
                                                              const uint32_t* __restrict__ block_offsets) {
    using BS = cub::BlockScan<uint32_t, kCmpThreads>;
    __shared__ typename BS::TempStorage tmp;
    const int64_t nn = n_dev ? *n_dev : n;
    const int64_t base = int64_t(blockIdx.x) * kCmpTile + int64_t(threadIdx.x) * kCmpItems;
    bool f[kCmpItems];
    uint32_t c = 0;
    for (int k = 0; k < kCmpItems; ++k) {
        f[k] = (base + k < nn) && pred(base + k);
        c += f[k];
    }
    uint32_t ex;
    BS(tmp).ExclusiveSum(c, ex);
    uint32_t o = block_offsets[blockIdx.x] + ex;
    for (int k = 0; k < kCmpItems; ++k)
        if (f[k]) emit(base + k, o++);
}

constexpr int kMaxRows = 23;   // parameter rows: 14 (RGB) or 23 (degree-1 SH)

struct AddPred {
    const float *alpha, *depth, *td;
    int W;
    float tau_a, tau_d;
    int stride;
    __device__ bool operator()(int64_t p) const {
        const int u = int(p % W), v = int(p / W);
        const float t = td[p];
        return t > 0.f && (alpha[p] < tau_a || fabsf(t - depth[p]) > tau_d) && ((u + v) % stride) == 0;
    }
};

struct AddEmit {
    const float *td, *trgb;
    const float* viewmat;
    int W;
    int64_t npx;
    float fx, fy, cx, cy, init_o;
    int stride;
    float* params;   // [14][ld] (activated), columns n + o
    float* raw;      // nullable
    float *m, *v;    // nullable
    float* out;      // nullable: [14][max_add] candidate records
    int64_t ld, capacity, max_add;
    const int64_t* n_dev;
    int rows;        // 14 (RGB) or 23 (degree-1 SH: colour as the DC coefficient, reading C34)
    __device__ void operator()(int64_t p, uint32_t o) const {
        if (int64_t(o) >= max_add) return;
        const int64_t n = *n_dev;
        const float z = td[p];
        const float u = float(p % W), v_ = float(p / W);
        const float xc = (u - cx) / fx * z, yc = (v_ - cy) / fy * z, zc = z;
        const float* V = viewmat;
        // X = W^T (X^c - t)
        const float a0 = xc - V[3], a1 = yc - V[7], a2 = zc - V[11];
        float rec[kMaxRows];
        rec[0] = V[0] * a0 + V[4] * a1 + V[8] * a2;
        rec[1] = V[1] * a0 + V[5] * a1 + V[9] * a2;
        rec[2] = V[2] * a0 + V[6] * a1 + V[10] * a2;
        const float s = z * float(stride) / (fx + fy);
        rec[3] = rec[4] = rec[5] = s;
        rec[6] = 1.f;
        rec[7] = rec[8] = rec[9] = 0.f;
        rec[10] = init_o;
        for (int c = 0; c < 3; ++c) {
            const float col = trgb[c * npx + p];
            // SH: the DC coefficient whose view-independent colour 1/2 + C0 Y0 is the target colour
            rec[11 + c] = rows == 23 ? (col - 0.5f) / 0.28209479177387814f : col;
        }
        for (int k = 14; k < rows; ++k) rec[k] = 0.f;
        if (out) {
            for (int k = 0; k < rows; ++k) out[k * max_add + o] = rec[k];
            return;
        }
        const int64_t col = n + o;
        if (col >= capacity) return;
        for (int k = 0; k < rows; ++k) params[k * ld + col] = rec[k];
        if (raw) {
            for (int k = 0; k < rows; ++k) raw[k * ld + col] = rec[k];
            for (int k = 3; k < 6; ++k) raw[k * ld + col] = logf(s);
            raw[10 * ld + col] = logf(init_o / (1.f - init_o));
        }
        if (m) for (int k = 0; k < rows; ++k) m[k * ld + col] = 0.f;
        if (v) for (int k = 0; k < rows; ++k) v[k * ld + col] = 0.f;
    }
};

__global__ void add_count_out_kernel(int64_t* n_dev, const unsigned long long* count, int64_t max_add) {
    const int64_t a = int64_t(*count);
    *n_dev = a < max_add ? a : max_add;
}

// Append gathered candidate sets in order (gs_densify_append). One thread per (set, candidate).
__global__ void __launch_bounds__(256) append_kernel(float* __restrict__ params, float* __restrict__ raw,
                                                     float* __restrict__ m, float* __restrict__ v, int64_t* n_dev,
                                                     int64_t capacity, int64_t ld, const float* __restrict__ cand,
                                                     const int64_t* __restrict__ counts, int n_sets, int64_t max_add,
                                                     int rows) {
    const int64_t n = *n_dev;
    const int set = blockIdx.y;
    int64_t off = 0;
    for (int k = 0; k < set; ++k) off += counts[k];
    const int64_t cnt = counts[set];
    const float* src = cand + size_t(set) * rows * max_add;
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < cnt; j += int64_t(gridDim.x) * blockDim.x) {
        const int64_t col = n + off + j;
        if (col >= capacity) break;
        for (int k = 0; k < rows; ++k) params[k * ld + col] = src[k * max_add + j];
        if (raw) {
            for (int k = 0; k < rows; ++k) raw[k * ld + col] = src[k * max_add + j];
            for (int k = 3; k < 6; ++k) raw[k * ld + col] = logf(src[k * max_add + j]);
            const float o = src[10 * max_add + j];
            raw[10 * ld + col] = logf(o / (1.f - o));
        }
        if (m) for (int k = 0; k < rows; ++k) m[k * ld + col] = 0.f;
        if (v) for (int k = 0; k < rows; ++k) v[k * ld + col] = 0.f;
    }
}

__global__ void append_commit_kernel(int64_t* n_dev, const int64_t* counts, int n_sets, int64_t capacity) {
    int64_t n = *n_dev;
    for (int k = 0; k < n_sets; ++k) n += counts[k];
    *n_dev = n < capacity ? n : capacity;
}

void launch_append(float* params, float* raw, float* m, float* v, int64_t* n_dev, int64_t capacity, int64_t ld,
                   const float* cand, const int64_t* counts, int32_t n_sets, int64_t max_add, int32_t rows,
                   cudaStream_t st) {
    if (n_sets <= 0 || max_add <= 0) return;
    dim3 grid(unsigned(std::min<int64_t>((max_add + 255) / 256, 64)), unsigned(n_sets));
    append_kernel<<<grid, 256, 0, st>>>(params, raw, m, v, n_dev, capacity, ld, cand, counts, n_sets, max_add, rows);
    append_commit_kernel<<<1, 1, 0, st>>>(n_dev, counts, n_sets, capacity);
}

__global__ void add_commit_kernel(int64_t* n_dev, const unsigned long long* count, int64_t max_add, int64_t capacity) {
    const int64_t n = *n_dev;
    int64_t a = int64_t(*count);
    if (a > max_add) a = max_add;
    if (n + a > capacity) a = capacity - n;
    *n_dev = n + a;
}

struct KeepPred {
    const float* opacity;   // row 10 of params
    float min_o;
    __device__ bool operator()(int64_t i) const { return opacity[i] >= min_o; }
};

__global__ void set_n_kernel(int64_t* n_dev, const unsigned long long* count) { *n_dev = int64_t(*count); }

// ------------------------------------------------------------------ in-place stable compaction
// PRUNE and the split/clone removal keep the columns a predicate accepts, in index order, in up to
// four [rows][ld] arrays at once. One CTA per 256-column tile: count -> exclusive scan of the tile
// counts -> compact. The compaction is in place: tile t's destination [off_t, off_t + cnt_t) lies at
// or below its own columns and spans at most two source tiles, so the CTA reads its tile (all rows
// of all arrays) into registers, publishes "read" for t, waits for the "read" flag of the earlier
// tiles its destination overlaps, then writes. Tiles are claimed through a ticket counter, so every
// tile waited on belongs to a CTA that is already running and whose read phase waits on nothing.
// A tile with no removal at or before it moves nothing and only publishes its flag; a map with
// nothing to remove costs one read of the predicate's row. Traffic: the moved columns once read and
// once written (the two-pass scratch scheme it replaces moved every column four times).
constexpr int kCmp = 256;

template <class Pred>
__global__ void __launch_bounds__(kCmp) count256_kernel(const int64_t* n_dev, Pred pred, uint32_t* __restrict__ counts) {
    using BR = cub::BlockReduce<uint32_t, kCmp>;
    __shared__ typename BR::TempStorage tmp;
    const int64_t nn = *n_dev;
    const int64_t i = int64_t(blockIdx.x) * kCmp + threadIdx.x;
    const uint32_t c = BR(tmp).Sum((i < nn && pred(i)) ? 1u : 0u);
    if (threadIdx.x == 0) counts[blockIdx.x] = c;
}

template <int ROWS, class Pred>
__global__ void __launch_bounds__(kCmp) compact_inplace_kernel(float* a0, float* a1, float* a2, float* a3, int64_t ld,
                                                               const int64_t* n_dev, Pred pred, int nt,
                                                               const uint32_t* __restrict__ offs,
                                                               const unsigned long long* __restrict__ total,
                                                               uint32_t* ctl) {
    using BS = cub::BlockScan<uint32_t, kCmp>;
    __shared__ typename BS::TempStorage tmp;
    __shared__ uint32_t s_t;
    if (threadIdx.x == 0) s_t = atomicAdd(&ctl[0], 1u);
    __syncthreads();
    const int t = int(s_t);
    const int64_t nn = *n_dev;
    const int64_t base = int64_t(t) * kCmp, i = base + threadIdx.x;
    const int64_t off = offs[t];
    const int64_t end = t + 1 < nt ? int64_t(offs[t + 1]) : int64_t(*total);
    const int64_t valid = base < nn ? (nn - base < kCmp ? nn - base : kCmp) : 0;
    uint32_t* flag = ctl + 1;
    if (off == base && end - off == valid) {   // nothing at or before this tile moves
        if (threadIdx.x == 0) st_release_u32(&flag[t], 1u);
        return;
    }
    const bool keep = i < nn && pred(i);
    float* arr[4] = {a0, a1, a2, a3};
    float v[4][ROWS];
    if (keep) {
#pragma unroll
        for (int a = 0; a < 4; ++a)
            if (arr[a])
#pragma unroll
                for (int k = 0; k < ROWS; ++k) v[a][k] = arr[a][k * ld + i];
    }
    uint32_t rank;
    BS(tmp).ExclusiveSum(keep ? 1u : 0u, rank);
    __syncthreads();   // every thread's reads of the tile precede the release below
    if (threadIdx.x == 0) {
        __threadfence();
        st_release_u32(&flag[t], 1u);
        // destination [off, end) overlaps source tiles off/256 .. (end-1)/256 (all <= t)
        if (end > off) {
            for (int64_t u = off / kCmp; u <= (end - 1) / kCmp && u < t; ++u)
                while (ld_acquire_u32(&flag[u]) == 0u) __nanosleep(64);
        }
        __threadfence();
    }
    __syncthreads();
    if (keep) {
        const int64_t o = off + rank;
#pragma unroll
        for (int a = 0; a < 4; ++a)
            if (arr[a])
#pragma unroll
                for (int k = 0; k < ROWS; ++k) arr[a][k * ld + o] = v[a][k];
    }
}

// count + scan + in-place compaction of arrays[4] (nullable) over columns [0, *n_dev) of [rows][ld];
// the kept count lands in *kept (the caller sets n from it)
template <class Pred>
void compact_inplace(WsState* s, float* const arrays[4], int rows, int64_t ld, int64_t capacity, const int64_t* n_dev,
                     Pred pred, unsigned long long* kept, cudaStream_t st) {
    const int nt = int((std::max<int64_t>(capacity, 1) + kCmp - 1) / kCmp);
    uint32_t* counts = at<uint32_t>(s, s->cmp);
    uint32_t* ctl = counts + (nt + 2);
    launch_zero(ctl, size_t(nt + 1) * 4, st, s);
    count256_kernel<<<nt, kCmp, 0, st>>>(n_dev, pred, counts);
    scan_blocks_kernel<<<1, 1024, 0, st>>>(counts, nt, kept);
    if (rows == 23)
        compact_inplace_kernel<23><<<nt, kCmp, 0, st>>>(arrays[0], arrays[1], arrays[2], arrays[3], ld, n_dev, pred,
                                                        nt, counts, kept, ctl);
    else
        compact_inplace_kernel<14><<<nt, kCmp, 0, st>>>(arrays[0], arrays[1], arrays[2], arrays[3], ld, n_dev, pred,
                                                        nt, counts, kept, ctl);
}

// ------------------------------------------------------------------ split / clone (reading C30)
__global__ void accum_grad_kernel(const uint32_t* __restrict__ onlist, const unsigned int* __restrict__ n_on,
                                  const float* __restrict__ sgrad, int64_t sld, float hw, float hh,
                                  float* __restrict__ accum, float* __restrict__ count) {
    const int64_t V = int64_t(*n_on);
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < V; t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = onlist[t];
        const float gx = sgrad[t] * hw, gy = sgrad[sld + t] * hh;   // dL/dm in NDC units (rank-indexed)
        accum[i] += sqrtf(gx * gx + gy * gy);
        count[i] += 1.f;
    }
}

void launch_accum_grad(WsState* s, float* grad_accum, float* count, cudaStream_t st) {
    KTimer kt(s, KID_DENSIFY, st);
    accum_grad_kernel<<<sm_count() * 4, 256, 0, st>>>(at<uint32_t>(s, s->onlist), &at<Misc>(s, s->misc)->n_onscreen,
                                               at<float>(s, s->sgrad), s->n_cap, 0.5f * float(s->cam_w),
                                               0.5f * float(s->cam_h), grad_accum, count);
}

// candidate type of Gaussian i: 1 clone, 2 split, 0 none
__device__ __forceinline__ int dens_type(const float* params, int64_t ld, const float* accum, const float* count,
                                         int64_t i, float gthr, float sthr) {
    const float c = count[i];
    const float avg = c > 0.f ? accum[i] / c : 0.f;
    if (!(avg >= gthr)) return 0;
    const float smax = fmaxf(fmaxf(params[3 * ld + i], params[4 * ld + i]), params[5 * ld + i]);
    return smax <= sthr ? 1 : 2;
}

struct TypePred {
    const float *params, *accum, *count;
    int64_t ld;
    float gthr, sthr;
    int type;
    __device__ bool operator()(int64_t i) const { return dens_type(params, ld, accum, count, i, gthr, sthr) == type; }
};

struct SplitCloneEmit {   // appends clones (type 1) or split children (type 2)
    float *params, *raw, *m, *v, *accum;
    const float* noise;
    int64_t ld, capacity;
    const int64_t* n_dev;
    const unsigned long long* n_clone;   // clones found (type 2 pass: the clones applied come first)
    int type;
    int rows;                            // 14 or 23: children copy every row but mean and scale
    __device__ void put(int64_t col, const float* rec) const {
        for (int k = 0; k < rows; ++k) params[k * ld + col] = rec[k];
        if (raw) {
            for (int k = 0; k < rows; ++k) raw[k * ld + col] = rec[k];
            for (int k = 3; k < 6; ++k) raw[k * ld + col] = logf(rec[k]);
            raw[10 * ld + col] = logf(rec[10] / (1.f - rec[10]));
        }
        if (m) for (int k = 0; k < rows; ++k) m[k * ld + col] = 0.f;
        if (v) for (int k = 0; k < rows; ++k) v[k * ld + col] = 0.f;
    }
    __device__ void operator()(int64_t i, uint32_t o) const {
        const int64_t n = *n_dev, avail = capacity - n;
        float rec[kMaxRows];
        for (int k = 0; k < rows; ++k) rec[k] = params[k * ld + i];
        if (type == 1) {
            if (int64_t(o) < avail) put(n + o, rec);
            return;
        }
        const int64_t nc = min(int64_t(*n_clone), avail);
        const int64_t col = n + nc + 2 * int64_t(o);
        if (col + 2 > capacity) return;   // does not fit: the split is not applied
        // children: X + R(q) diag(s) eps_k, scale s / 1.6 (3DGS, reading C30)
        const float qn = sqrtf(rec[6] * rec[6] + rec[7] * rec[7] + rec[8] * rec[8] + rec[9] * rec[9]);
        const float r = rec[6] / qn, x = rec[7] / qn, y = rec[8] / qn, z = rec[9] / qn;
        const float R[3][3] = {{1.f - 2.f * (y * y + z * z), 2.f * (x * y - r * z), 2.f * (x * z + r * y)},
                               {2.f * (x * y + r * z), 1.f - 2.f * (x * x + z * z), 2.f * (y * z - r * x)},
                               {2.f * (x * z - r * y), 2.f * (y * z + r * x), 1.f - 2.f * (x * x + y * y)}};
        float child[kMaxRows];
        for (int c = 0; c < 2; ++c) {
            for (int k = 0; k < rows; ++k) child[k] = rec[k];
            float e[3];
            for (int a = 0; a < 3; ++a) e[a] = rec[3 + a] * noise[(3 * c + a) * ld + i];
            for (int a = 0; a < 3; ++a) child[a] = rec[a] + (R[a][0] * e[0] + R[a][1] * e[1] + R[a][2] * e[2]);
            for (int a = 0; a < 3; ++a) child[3 + a] = rec[3 + a] / 1.6f;
            put(col + c, child);
        }
        accum[i] = -1.f;   // applied: the original is removed by the compaction below
    }
};

struct KeepSplitPred {
    const float* accum;
    const int64_t* n_dev;
    __device__ bool operator()(int64_t i) const { return i >= *n_dev || accum[i] >= 0.f; }
};

__global__ void split_clone_total_kernel(int64_t* total, const int64_t* n_dev, const unsigned long long* nc,
                                         const unsigned long long* ns, int64_t capacity) {
    const int64_t n = *n_dev, avail = capacity - n;
    const int64_t c = min(int64_t(*nc), avail);
    const int64_t sp = min(int64_t(*ns), (avail - c) / 2);
    *total = n + c + 2 * sp;   // columns holding originals and appended Gaussians before the compaction
}

__global__ void zero2_kernel(float* a, float* b, int64_t n) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        a[i] = 0.f;
        b[i] = 0.f;
    }
}

gs_status run_split_clone(WsState* s, float* params, float* raw, float* m, float* v, int64_t* n_dev, int64_t capacity,
                          int64_t ld, float* accum, float* count, const float* noise, float gthr, float sthr,
                          int32_t rows, cudaStream_t st) {
    Misc* misc = at<Misc>(s, s->misc);
    uint32_t* bcounts = at<uint32_t>(s, s->chunk_hist);
    const int nb = int((capacity + kCmpTile - 1) / kCmpTile);
    unsigned long long* nclone = &misc->add_count;
    unsigned long long* nsplit = &misc->keep_count;
    // clones (index order)
    TypePred pc{params, accum, count, ld, gthr, sthr, 1};
    KTimer kt(s, KID_DENSIFY, st);
    count_kernel<<<nb, kCmpThreads, 0, st>>>(capacity, n_dev, pc, bcounts);
    scan_blocks_kernel<<<1, 1024, 0, st>>>(bcounts, nb, nclone);
    scatter_kernel<<<nb, kCmpThreads, 0, st>>>(capacity, n_dev, pc,
                                               SplitCloneEmit{params, raw, m, v, accum, noise, ld, capacity, n_dev,
                                                              nclone, 1, rows},
                                               bcounts);
    // splits (index order), after the clones
    TypePred ps{params, accum, count, ld, gthr, sthr, 2};
    count_kernel<<<nb, kCmpThreads, 0, st>>>(capacity, n_dev, ps, bcounts);
    scan_blocks_kernel<<<1, 1024, 0, st>>>(bcounts, nb, nsplit);
    scatter_kernel<<<nb, kCmpThreads, 0, st>>>(capacity, n_dev, ps,
                                               SplitCloneEmit{params, raw, m, v, accum, noise, ld, capacity, n_dev,
                                                              nclone, 2, rows},
                                               bcounts);
    // n_dev <- columns in use; then drop the applied split originals by stable compaction
    int64_t* ncols = reinterpret_cast<int64_t*>(at<char>(s, s->scratch));
    split_clone_total_kernel<<<1, 1, 0, st>>>(ncols, n_dev, nclone, nsplit, capacity);
    const KeepSplitPred keep{accum, n_dev};
    // compaction over [0, ncols): n_dev stays the original n inside the predicate (appended columns kept)
    float* const arrays[4] = {raw, m, v, params};
    compact_inplace(s, arrays, rows, ld, capacity, ncols, keep, &misc->keep_count, st);
    set_n_kernel<<<1, 1, 0, st>>>(n_dev, &misc->keep_count);
    zero2_kernel<<<sm_count() * 4, 256, 0, st>>>(accum, count, capacity);
    return check_launch(s, "densify_split_clone");
}

__global__ void select_kernel(int64_t n, const int64_t* n_dev, const float4* __restrict__ rec,
                              const uint32_t* __restrict__ tiles, const float* __restrict__ accum,
                              const float* __restrict__ td, int W, int H, float sel_w, float sel_d,
                              uint8_t* __restrict__ mask) {
    const int64_t nn = n_dev ? *n_dev : n;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nn; i += int64_t(gridDim.x) * blockDim.x) {
        uint8_t keep = 0;
        if (tiles[i] > 0) {
            const float4 r0 = rec[3 * i], r1 = rec[3 * i + 1];
            const float u = floorf(r0.x + 0.5f), v = floorf(r0.y + 0.5f);
            if (u >= 0.f && u < float(W) && v >= 0.f && v < float(H)) {
                const float t = td[int64_t(v) * W + int64_t(u)];
                keep = (t > 0.f && accum[i] > sel_w && fabsf(t - r1.z) < sel_d) ? 1 : 0;
            }
        }
        mask[i] = keep;
    }
}

// Eq. 9 (reading C27): opacity degeneration of floaters in front of the observed surface
__global__ void degenerate_kernel(int64_t n, const int64_t* n_dev, const float4* __restrict__ rec,
                                  const uint32_t* __restrict__ tiles, const float* __restrict__ td, int W, int H,
                                  float gamma, float eta, float* __restrict__ opacity, float* __restrict__ raw_opacity,
                                  uint8_t* __restrict__ mask, bool flag_only) {
    const int64_t nn = n_dev ? *n_dev : n;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nn; i += int64_t(gridDim.x) * blockDim.x) {
        bool hit = false;
        if (tiles[i] > 0) {
            const float4 r0 = rec[3 * i], r1 = rec[3 * i + 1];
            const float u = floorf(r0.x + 0.5f), v = floorf(r0.y + 0.5f);
            if (u >= 0.f && u < float(W) && v >= 0.f && v < float(H)) {
                const float t = td[int64_t(v) * W + int64_t(u)];
                hit = t > 0.f && __fsub_rn(t, r1.z) > gamma;
            }
        }
        if (flag_only) {   // GS_DENSIFY_DEGENERATE_FLAG: OR into the mask, opacities untouched
            if (hit) mask[i] = 1;
            continue;
        }
        if (hit) {
            const float o = __fmul_rn(eta, opacity[i]);
            opacity[i] = o;
            if (raw_opacity) raw_opacity[i] = logf(o / (1.f - o));
        }
        if (mask) mask[i] = hit ? 1 : 0;
    }
}

// GS_DENSIFY_DEGENERATE_APPLY: the Eq. 9 scaling for the Gaussians a (reduced) flag mask names
__global__ void degenerate_apply_kernel(int64_t n, const int64_t* n_dev, const uint8_t* __restrict__ mask, float eta,
                                        float* __restrict__ opacity, float* __restrict__ raw_opacity) {
    const int64_t nn = n_dev ? *n_dev : n;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nn; i += int64_t(gridDim.x) * blockDim.x) {
        if (!mask[i]) continue;
        const float o = __fmul_rn(eta, opacity[i]);
        opacity[i] = o;
        if (raw_opacity) raw_opacity[i] = logf(o / (1.f - o));
    }
}

#define GS_K(call)                              \
    do {                                        \
        KTimer kt_(s, KID_DENSIFY, st);         \
        call;                                   \
    } while (0)

gs_status run_densify(WsState* s, float* params, float* raw, int64_t* n_dev, int64_t capacity, int64_t ld, float* m,
                      float* v, const float* alpha, const float* depth, const float* trgb, const float* tdepth,
                      const float* accum, const float* viewmat, const gs_camera& cam, const gs_densify_cfg& cfg,
                      uint8_t* select_mask, float* add_out, cudaStream_t st) {
    Misc* misc = at<Misc>(s, s->misc);
    uint32_t* bcounts = at<uint32_t>(s, s->chunk_hist);
    const int rows = cfg.rows == 23 ? 23 : 14;   // 0 -> 14 (RGB)
    if (cfg.mode == GS_DENSIFY_SELECT) {
        const int blocks = int(std::min<int64_t>((capacity + 255) / 256, sm_count() * 8));
        GS_K((select_kernel<<<blocks, 256, 0, st>>>(capacity, n_dev, at<float4>(s, s->rec), at<uint32_t>(s, s->tiles),
                                                    accum, tdepth, cam.width, cam.height, cfg.sel_weight,
                                                    cfg.sel_depth, select_mask)));
        return check_launch(s, "densify_select");
    }
    if (cfg.mode == GS_DENSIFY_DEGENERATE || cfg.mode == GS_DENSIFY_DEGENERATE_FLAG) {
        const int blocks = int(std::min<int64_t>((capacity + 255) / 256, sm_count() * 8));
        GS_K((degenerate_kernel<<<blocks, 256, 0, st>>>(capacity, n_dev, at<float4>(s, s->rec), at<uint32_t>(s, s->tiles),
                                                        tdepth, cam.width, cam.height, cfg.gamma, cfg.eta,
                                                        params ? params + 10 * ld : nullptr,
                                                        raw ? raw + 10 * ld : nullptr, select_mask,
                                                        cfg.mode == GS_DENSIFY_DEGENERATE_FLAG)));
        return check_launch(s, "densify_degenerate");
    }
    if (cfg.mode == GS_DENSIFY_DEGENERATE_APPLY) {
        const int blocks = int(std::min<int64_t>((capacity + 255) / 256, sm_count() * 8));
        GS_K((degenerate_apply_kernel<<<blocks, 256, 0, st>>>(capacity, n_dev, select_mask, cfg.eta, params + 10 * ld,
                                                              raw ? raw + 10 * ld : nullptr)));
        return check_launch(s, "densify_degenerate_apply");
    }
    if (cfg.mode == GS_DENSIFY_ADD) {
        const int64_t npx = int64_t(cam.width) * cam.height;
        const int nb = int((npx + kCmpTile - 1) / kCmpTile);
        AddPred pred{alpha, depth, tdepth, cam.width, cfg.tau_alpha, cfg.tau_depth, cfg.stride};
        AddEmit emit{tdepth, trgb, viewmat, cam.width, npx, cam.fx, cam.fy, cam.cx, cam.cy, cfg.init_opacity,
                     cfg.stride, params, raw, m, v, add_out, ld, capacity, cfg.max_add, n_dev, rows};
        GS_K((count_kernel<<<nb, kCmpThreads, 0, st>>>(npx, nullptr, pred, bcounts)));
        GS_K((scan_blocks_kernel<<<1, 1024, 0, st>>>(bcounts, nb, &misc->add_count)));
        GS_K((scatter_kernel<<<nb, kCmpThreads, 0, st>>>(npx, nullptr, pred, emit, bcounts)));
        if (!add_out) GS_K((add_commit_kernel<<<1, 1, 0, st>>>(n_dev, &misc->add_count, cfg.max_add, capacity)));
        else GS_K((add_count_out_kernel<<<1, 1, 0, st>>>(n_dev, &misc->add_count, cfg.max_add)));
        return check_launch(s, "densify_add");
    }
    if (cfg.mode == GS_DENSIFY_PRUNE) {
        KeepPred pred{params + 10 * ld, cfg.min_opacity};
        float* const arrays[4] = {raw, m, v, params};   // each column's predicate is read before it moves
        GS_K((compact_inplace(s, arrays, rows, ld, capacity, n_dev, pred, &misc->keep_count, st)));
        GS_K((set_n_kernel<<<1, 1, 0, st>>>(n_dev, &misc->keep_count)));
        return check_launch(s, "densify_prune");
    }
    return GS_ERR_INVALID_ARG;
}
#undef GS_K

}  // namespace gs
