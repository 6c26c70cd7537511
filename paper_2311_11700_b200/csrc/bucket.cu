// gs_bin_sort, path B (default): depth presort + ordered tile bucketing.
//
// Output-identical to path A (the stable sort of the index-order (tile|depth) keys, O2)
// without materialising or sorting the K keys:
//   B1  compaction: the V_s on-screen Gaussians in index order (decoupled look-back, binsort.cu)
//   B2  depth sort: onesweep LSD radix sort of their (depth bits, index) pairs (stable: ties by index)
//   B3  chunk count: the depth-ordered Gaussians are cut into chunks of 256; per chunk, a 2-D
//                   difference array over the tile grid in shared memory gives count[c][t]
//   B4  tile scan:  per-tile totals (8 chunk segments per tile in flight), one exclusive scan over
//                   tiles (ranges, K), then per-tile exclusive scans over chunks -> base[c][t]
//   B5  emission:   warp work item = (chunk, 32-tile segment): the warp compacts (in depth order)
//                   the chunk's Gaussians meeting its segment, then per tile its lanes test 32 of
//                   them at a time and a ballot/popc prefix places the hits at base[c][t] + rank
//                   (coalesced 4-B stores, depth order preserved)
// Per tile, entries come out in chunk order and in depth order within a chunk, i.e. ordered by
// (depth bits, index): exactly the per-tile lists of path A (checked bit-exact in the tests).
// HBM traffic is ~4 B per key (+ per-Gaussian and per-chunk terms) instead of ~150 B per key.
#include <cub/block/block_scan.cuh>

#include <algorithm>

#include "gs_internal.cuh"
#include "onesweep.cuh"

namespace gs {

constexpr int kChunk = 256;      // Gaussians per chunk (depth order)
constexpr int kSeg = 32;         // consecutive tiles per emission work item (one warp)

gs_status chained_scan(WsState* s, const uint32_t* in, uint32_t* out, int64_t n, unsigned long long* total,
                       cudaStream_t st, int64_t cap, unsigned long long* total_eff);
gs_status resolve_keys(WsState* s, int64_t* n_keys, uint32_t flags, cudaStream_t st, int64_t* Kgrid);

// B3 ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kChunk) chunk_count_kernel(const uint32_t* __restrict__ svals,
                                                             const short4* __restrict__ rect,
                                                             const unsigned int* __restrict__ n_on, int GX, int GY,
                                                             uint32_t* __restrict__ cmat, short4* __restrict__ srect) {
    extern __shared__ int diff[];   // (GY + 1) x (GX + 1)
    const int c = blockIdx.x;
    const uint32_t Von = *n_on;
    const uint32_t base = uint32_t(c) * kChunk;
    if (base >= Von) return;
    const int W1 = GX + 1, cells = (GY + 1) * W1, T = GX * GY;
    for (int i = threadIdx.x; i < cells; i += blockDim.x) diff[i] = 0;
    __syncthreads();
    const uint32_t s = base + threadIdx.x;
    if (s < Von) {
        const short4 r = rect[svals[s]];
        srect[s] = r;
        atomicAdd(&diff[r.z * W1 + r.x], 1);
        atomicAdd(&diff[r.z * W1 + r.y], -1);
        atomicAdd(&diff[r.w * W1 + r.x], -1);
        atomicAdd(&diff[r.w * W1 + r.y], 1);
    }
    __syncthreads();
    for (int y = threadIdx.x; y < GY; y += blockDim.x) {   // prefix along x
        int run = 0;
        for (int x = 0; x < GX; ++x) {
            run += diff[y * W1 + x];
            diff[y * W1 + x] = run;
        }
    }
    __syncthreads();
    uint32_t* row = cmat + size_t(c) * T;
    for (int x = threadIdx.x; x < GX; x += blockDim.x) {   // prefix along y, write counts
        int run = 0;
        for (int y = 0; y < GY; ++y) {
            run += diff[y * W1 + x];
            row[y * GX + x] = uint32_t(run);
        }
    }
}

// B4 ---------------------------------------------------------------------------------------
// Per-tile column sums over the chunks: block = 32 tiles (lanes) x 8 chunk segments (warps), so
// 8 independent loads per thread are in flight and every warp load is one coalesced 128-B row.
constexpr int kSegs = 8;

__device__ __forceinline__ void seg_range(int nch, int seg, int& c0, int& c1) {
    const int per = (nch + kSegs - 1) / kSegs;
    c0 = min(nch, seg * per);
    c1 = min(nch, c0 + per);
}

__global__ void __launch_bounds__(256) tile_total_kernel(const uint32_t* __restrict__ cmat,
                                                         const unsigned int* __restrict__ n_on, int T,
                                                         uint32_t* __restrict__ segsum, uint32_t* __restrict__ tot) {
    __shared__ uint32_t sh[kSegs][32];
    const int lane = threadIdx.x & 31, seg = threadIdx.x >> 5;
    const int t = blockIdx.x * 32 + lane;
    const int nch = int((*n_on + kChunk - 1) / kChunk);
    int c0, c1;
    seg_range(nch, seg, c0, c1);
    uint32_t sum = 0;
    if (t < T) {
#pragma unroll 8
        for (int c = c0; c < c1; ++c) sum += __ldg(cmat + size_t(c) * T + t);
        segsum[size_t(seg) * T + t] = sum;
    }
    sh[seg][lane] = sum;
    __syncthreads();
    if (seg == 0 && t < T) {
        uint32_t s = 0;
#pragma unroll
        for (int q = 0; q < kSegs; ++q) s += sh[q][lane];
        tot[t] = s;
    }
}

__global__ void __launch_bounds__(1024) tile_scan_kernel(const uint32_t* __restrict__ tot, int T,
                                                         uint32_t* __restrict__ tstart, uint2* __restrict__ ranges,
                                                         unsigned long long* n_keys, unsigned long long* n_keys_eff,
                                                         int64_t key_cap, unsigned int* error_flag) {
    using BS = cub::BlockScan<unsigned long long, 1024>;
    __shared__ typename BS::TempStorage tmp;
    __shared__ unsigned long long carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int b = 0; b < T; b += 1024) {
        const int t = b + threadIdx.x;
        const unsigned long long v = t < T ? tot[t] : 0ull;
        unsigned long long ex, agg;
        BS(tmp).ExclusiveSum(v, ex, agg);
        const unsigned long long st = carry + ex;
        if (t < T) {
            tstart[t] = uint32_t(st);
            ranges[t] = v ? make_uint2(uint32_t(st), uint32_t(st + v)) : make_uint2(0u, 0u);
        }
        __syncthreads();
        if (threadIdx.x == 0) carry += agg;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        *n_keys = carry;
        const bool over = carry > (unsigned long long)key_cap;
        *n_keys_eff = over ? 0ull : carry;
        if (over) atomicOr(error_flag, 1u);
    }
}

__global__ void __launch_bounds__(256) chunk_base_kernel(uint32_t* __restrict__ cmat,
                                                         const uint32_t* __restrict__ tstart,
                                                         const uint32_t* __restrict__ segsum,
                                                         const unsigned int* __restrict__ n_on, int T) {
    const int lane = threadIdx.x & 31, seg = threadIdx.x >> 5;
    const int t = blockIdx.x * 32 + lane;
    if (t >= T) return;
    const int nch = int((*n_on + kChunk - 1) / kChunk);
    int c0, c1;
    seg_range(nch, seg, c0, c1);
    uint32_t run = tstart[t];
    for (int q = 0; q < seg; ++q) run += segsum[size_t(q) * T + t];
    for (int cb = c0; cb < c1; cb += 8) {   // 8 independent loads in flight, then 8 stores
        uint32_t v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = (cb + u < c1) ? cmat[size_t(cb + u) * T + t] : 0u;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (cb + u < c1) cmat[size_t(cb + u) * T + t] = run;
            run += v[u];
        }
    }
}

// B5 ---------------------------------------------------------------------------------------
// Block = (chunk, 8 segments of kSeg consecutive tiles); blocks of chunks beyond ceil(V_s / kChunk),
// read on the device, exit at once. The block first pre-filters (ordered BlockScan compaction) the
// chunk's Gaussians meeting its tile range; then each warp, independently, compacts those meeting its
// segment with a per-Gaussian 32-bit tile mask, and per tile a ballot + popc ranks the hits of 32
// Gaussians at a time and places them at base[chunk][tile] + rank (coalesced 4-B stores).
__device__ __forceinline__ uint32_t bits_below(int n) { return n >= 32 ? 0xffffffffu : ((1u << n) - 1u); }

// bits [lo, hi) of the segment mask for rect r on tile row `row`, whose segment tiles are columns
// [x0, x0 + cnt) at mask bits [bit0, bit0 + cnt)
__device__ __forceinline__ uint32_t run_mask(short4 r, int row, int x0, int cnt, int bit0) {
    if (row < r.z || row >= r.w) return 0u;
    const int lo = max(int(r.x), x0) - x0, hi = min(int(r.y), x0 + cnt) - x0;
    return hi > lo ? (bits_below(hi) & ~bits_below(lo)) << bit0 : 0u;
}

__global__ void __launch_bounds__(256) bucket_emit_kernel(
    const uint32_t* __restrict__ svals, const short4* __restrict__ srect, const uint32_t* __restrict__ cmat,
    const unsigned int* __restrict__ n_on, const unsigned long long* __restrict__ n_keys_eff,
    const unsigned long long* __restrict__ n_keys, int GX, int T, uint32_t* __restrict__ vals_out) {
    using BS = cub::BlockScan<int, 256>;
    __shared__ typename BS::TempStorage scan;
    __shared__ short4 b_rect[kChunk];
    __shared__ uint32_t b_g[kChunk];
    __shared__ uint32_t l_mask[8][kChunk];
    __shared__ uint32_t l_g[8][kChunk];
    if (*n_keys_eff != *n_keys) return;   // capacity overflow: emit nothing (error flag is set)
    const uint32_t Von = *n_on;
    const int c = blockIdx.x;
    const uint32_t base = uint32_t(c) * kChunk;
    if (base >= Von) return;   // chunk beyond the on-screen count (grid sized by n)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    // 1. block pre-filter: the chunk's Gaussians (depth order kept) whose rect meets the block's
    //    tile range [g0, g1] (8 segments)
    const int g0 = blockIdx.y * (8 * kSeg), g1 = min(T, g0 + 8 * kSeg) - 1;
    {
        const int gy0 = g0 / GX, gy1 = g1 / GX;
        const int cx0 = g0 - gy0 * GX, cx1 = g1 - gy1 * GX;   // first / last row columns
        const uint32_t s = base + tid;
        short4 r = make_short4(0, 0, 0, 0);
        bool meet = false;
        if (s < Von) {
            r = srect[s];
            const int ylo = max(int(r.z), gy0), yhi = min(int(r.w) - 1, gy1);
            if (ylo <= yhi && r.x < r.y) {
                auto row_meets = [&](int y) {
                    const int c0 = y == gy0 ? cx0 : 0, c1 = y == gy1 ? cx1 + 1 : GX;
                    return max(int(r.x), c0) < min(int(r.y), c1);
                };
                meet = (yhi - ylo >= 2) || row_meets(ylo) || row_meets(yhi);
            }
        }
        int off, tot;
        BS(scan).ExclusiveSum(meet ? 1 : 0, off, tot);
        if (meet) {
            b_rect[off] = r;
            b_g[off] = svals[s];
        }
        if (tid == 0) l_g[0][0] = uint32_t(tot);   // broadcast (l_g is rewritten below, after the barrier)
        __syncthreads();
    }
    const int tot = int(l_g[0][0]);
    __syncthreads();
    // 2. warp = one segment of kSeg consecutive tiles (row-major) starting at (tx0, ty0); it spans
    //    n0 tiles of row ty0 and then whole or partial following rows. Warps are independent.
    const int t0 = g0 + warp * kSeg;
    if (t0 >= T || tot == 0) return;   // warp-uniform
    const int nseg = min(kSeg, T - t0);
    const int ty0 = t0 / GX, tx0 = t0 - ty0 * GX;
    const int n0 = min(nseg, GX - tx0);
    int L = 0;
    for (int k0 = 0; k0 < tot; k0 += 32) {
        const int k = k0 + lane;
        uint32_t mask = 0;
        if (k < tot) {
            const short4 r = b_rect[k];
            mask = run_mask(r, ty0, tx0, n0, 0);
            for (int bit = n0, row = ty0 + 1; bit < nseg; bit += GX, ++row)   // narrow grids: more rows
                mask |= run_mask(r, row, 0, min(GX, nseg - bit), bit);
        }
        const uint32_t m = __ballot_sync(0xffffffffu, mask != 0u);
        if (mask) {
            const int o = L + __popc(m & lt);
            l_mask[warp][o] = mask;
            l_g[warp][o] = b_g[k];
        }
        L += __popc(m);
    }
    __syncwarp();
    // lane j < nseg keeps tile j's running output position
    uint32_t mypos = lane < nseg ? cmat[size_t(c) * T + t0 + lane] : 0u;
    for (int k0 = 0; k0 < L; k0 += 32) {
        const int k = k0 + lane;
        const uint32_t mask = k < L ? l_mask[warp][k] : 0u;
        const uint32_t g = k < L ? l_g[warp][k] : 0u;
#pragma unroll
        for (int j = 0; j < kSeg; ++j) {
            const bool hit = (mask >> j) & 1u;
            const uint32_t m = __ballot_sync(0xffffffffu, hit);
            if (m == 0u) continue;   // warp-uniform
            const uint32_t pj = __shfl_sync(0xffffffffu, mypos, j);
            if (hit) vals_out[pj + __popc(m & lt)] = g;
            if (lane == j) mypos += __popc(m);
        }
    }
}

// ------------------------------------------------------------------ host driver
gs_status run_bin_sort_bucket(WsState* s, int64_t* n_keys, uint32_t flags, cudaStream_t st) {
    Misc* misc = at<Misc>(s, s->misc);
    const int GX = s->cam_gx, GY = s->cam_gy, T = GX * GY;
    const int64_t n = s->n;
    cudaMemsetAsync(misc, 0, offsetof(Misc, loss_acc), st);   // K, flags, tickets, counters
    uint32_t* k0 = at<uint32_t>(s, s->dkey_sorted);
    uint32_t* k1 = k0 + s->n_cap;
    uint32_t* v0 = at<uint32_t>(s, s->dval_sorted);
    uint32_t* v1 = v0 + s->n_cap;
    // B1: ordered compaction of the on-screen Gaussians -> (depth key, index) pairs in k0/v0
    gs_status rc = run_compact_onscreen(s, st, true);   // also the depth keys' digit histograms
    if (rc != GS_OK) return rc;
    // B2: stable depth sort of the V_s on-screen pairs (grid sized by n, V_s read on the device)
    int which = 0;
    rc = onesweep_sort_pairs<uint32_t, kSortItemsSmall>(s, k0, v0, k1, v1, &misc->n_items, n, 32, st, &which, true);
    if (rc != GS_OK) return rc;
    const uint32_t* svals = which ? v1 : v0;
    uint32_t* cmat = at<uint32_t>(s, s->chunk_mat);
    short4* srect = at<short4>(s, s->srect);
    uint32_t* tot = at<uint32_t>(s, s->tile_tot);
    uint32_t* tstart = tot + s->GX * s->GY;
    uint32_t* segsum = tstart + s->GX * s->GY;   // [kSegs][T]
    const int nch = int((n + kChunk - 1) / kChunk);
    if (nch > 0) {
        const size_t smem = size_t(GX + 1) * (GY + 1) * sizeof(int);
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(chunk_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
            attr = true;
        }
        KTimer kt(s, KID_CHUNK_HIST, st);
        chunk_count_kernel<<<nch, kChunk, smem, st>>>(svals, at<short4>(s, s->rect), &misc->n_onscreen, GX, GY, cmat,
                                                      srect);
    }
    {
        KTimer kt(s, KID_CHUNK_SCAN, st);
        tile_total_kernel<<<(T + 31) / 32, 256, 0, st>>>(cmat, &misc->n_onscreen, T, segsum, tot);
    }
    {
        KTimer kt(s, KID_CHUNK_SCAN, st);
        tile_scan_kernel<<<1, 1024, 0, st>>>(tot, T, tstart, at<uint2>(s, s->ranges), &misc->n_keys, &misc->n_keys_eff,
                                             s->key_cap, &misc->error_flag);
    }
    {
        KTimer kt(s, KID_CHUNK_SCAN, st);
        chunk_base_kernel<<<(T + 31) / 32, 256, 0, st>>>(cmat, tstart, segsum, &misc->n_onscreen, T);
    }
    if (nch > 0) {
        KTimer kt(s, KID_BUCKET_EMIT, st);
        const dim3 grid(unsigned(nch), unsigned(((T + kSeg - 1) / kSeg + 7) / 8));
        bucket_emit_kernel<<<grid, 256, 0, st>>>(svals, srect, cmat, &misc->n_onscreen, &misc->n_keys_eff,
                                                    &misc->n_keys, GX, T, at<uint32_t>(s, s->vals0));
    }
    s->sorted_in_1 = 0;
    s->keys_valid = 0;
    int64_t Kgrid = 0;
    rc = resolve_keys(s, n_keys, flags, st, &Kgrid);   // host-sync mode: K readback + capacity status
    if (rc != GS_OK) return rc;
    return check_launch(s, "bin_sort_bucket");
}

}  // namespace gs
