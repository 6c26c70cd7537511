// gs_bin_sort, path A (north_star literal; GS_FLAG_BINSORT_KEYS):
//   ordered decoupled-look-back scan of tiles_touched  ->  warp-cooperative key emission
//   ->  onesweep LSD radix sort of (tile << 32 | depth-bits, index) pairs  ->  per-tile ranges.
// DESIGN.md O2 / SURVEY.md §8(a) rows a2-a5. Output: the stable ascending sort of the keys emitted
// in Gaussian-index order (ties by index), i.e. "sorting the Gaussians in depth order" per tile
// (PAPER.md:83).
#include <cub/block/block_scan.cuh>

#include <algorithm>

#include "gs_internal.cuh"
#include "onesweep.cuh"

namespace gs {

// ------------------------------------------------------------------ chained scan (look-back)
// status word: [epoch:30 | flag:2 | value:32]; flag 1 = aggregate, 2 = inclusive prefix.
constexpr int kScanThreads = 256, kScanItems = 8, kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ unsigned long long scan_word(uint32_t epoch, uint32_t flag, uint32_t v) {
    return (uint64_t(epoch & 0x3fffffffu) << 34) | (uint64_t(flag) << 32) | v;
}

// Decoupled look-back by one warp: publish this partition's aggregate, sum predecessors' words
// (32 per round) until the nearest inclusive prefix, publish the inclusive prefix, and return the
// exclusive prefix of the partition. Partition order comes from an atomic ticket, so every
// predecessor of a running partition has started: the spin always makes progress.
__device__ uint32_t lookback_prefix(unsigned long long* status, uint32_t part, uint32_t epoch, uint32_t agg) {
    const unsigned lane = threadIdx.x & 31;
    uint32_t prefix = 0;
    if (part == 0) {
        if (lane == 0) atomicExch(status + part, scan_word(epoch, 2, agg));
        return 0;
    }
    if (lane == 0) atomicExch(status + part, scan_word(epoch, 1, agg));
    int64_t j = int64_t(part) - 1 - lane;   // each lane inspects one predecessor
    while (true) {
        uint64_t w = 0;
        uint32_t flag = 0;
        if (j >= 0) {
            do {
                w = *reinterpret_cast<volatile unsigned long long*>(status + j);
                flag = (uint32_t(w >> 34) == (epoch & 0x3fffffffu)) ? uint32_t((w >> 32) & 3u) : 0u;
            } while (flag == 0);
        } else {
            flag = 2;   // virtual prefix 0 before partition 0
            w = 0;
        }
        const uint32_t val = j >= 0 ? uint32_t(w) : 0u;
        const unsigned pre_mask = __ballot_sync(0xffffffffu, flag == 2);
        // lanes up to and including the nearest (lowest lane = highest index) prefix
        const int stop = pre_mask ? __ffs(pre_mask) - 1 : 31;
        uint32_t contrib = (int(lane) <= stop) ? val : 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) contrib += __shfl_xor_sync(0xffffffffu, contrib, o);
        prefix += contrib;
        if (pre_mask) break;
        j -= 32;
    }
    if (lane == 0) atomicExch(status + part, scan_word(epoch, 2, prefix + agg));
    return prefix;
}

// Ordered compaction of the on-screen Gaussians (tiles > 0), in index order: list[r] = i and the
// (depth key, i) pairs; *count = V_s. Path A's on-screen list for the per-Gaussian backward (path B
// compacts inside bincoop.cu).
__global__ void __launch_bounds__(kScanThreads) compact_onscreen_kernel(
    const uint32_t* __restrict__ tiles, const uint32_t* __restrict__ dkey, int64_t n,
    unsigned long long* status, unsigned int* ticket, uint32_t epoch, uint32_t* __restrict__ list,
    uint32_t* __restrict__ key_out, uint32_t* __restrict__ val_out, unsigned int* count,
    unsigned long long* count64, float* __restrict__ rec_f) {
    using BlockScan = cub::BlockScan<uint32_t, kScanThreads>;
    __shared__ typename BlockScan::TempStorage tmp;
    __shared__ uint32_t s_part, s_excl;
    if (threadIdx.x == 0) s_part = atomicAdd(ticket, 1u);
    __syncthreads();
    const uint32_t part = s_part;
    const int64_t base = int64_t(part) * kScanTile + int64_t(threadIdx.x) * kScanItems;
    bool f[kScanItems];
    uint32_t sum = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        f[k] = (base + k < n) && tiles[base + k] > 0;
        sum += f[k];
    }
    uint32_t excl_thread, agg;
    BlockScan(tmp).ExclusiveSum(sum, excl_thread, agg);
    if (threadIdx.x < 32) {
        const uint32_t prefix = lookback_prefix(status, part, epoch, agg);
        if (threadIdx.x == 0) s_excl = prefix;
    }
    __syncthreads();
    uint32_t r = s_excl + excl_thread;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        if (f[k]) {
            const uint32_t i = uint32_t(base + k);
            list[r] = i;
            rec_f[kRecFloats * size_t(i) + 11] = __uint_as_float(r);   // on-screen rank -> record r2.w
            key_out[r] = dkey[i];
            val_out[r] = i;
            ++r;
        }
    }
    if (base < n && base + kScanItems >= n) {   // the partition holding element n-1 publishes V_s
        *count = r;
        *count64 = r;
    }
}

// Exclusive prefix of in[0..n) (u32) -> out (u32); total written to *total (u64).
__global__ void __launch_bounds__(kScanThreads) chained_scan_kernel(
    const uint32_t* __restrict__ in, uint32_t* __restrict__ out, int64_t n, unsigned long long* status,
    unsigned int* ticket, uint32_t epoch, unsigned long long* total, int64_t cap, unsigned long long* total_eff,
    unsigned int* error_flag) {
    using BlockScan = cub::BlockScan<uint32_t, kScanThreads>;
    __shared__ typename BlockScan::TempStorage tmp;
    __shared__ uint32_t s_part, s_excl;
    if (threadIdx.x == 0) s_part = atomicAdd(ticket, 1u);
    __syncthreads();
    const uint32_t part = s_part;
    const int64_t base = int64_t(part) * kScanTile + int64_t(threadIdx.x) * kScanItems;
    uint32_t v[kScanItems];
    uint32_t sum = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        v[k] = (base + k < n) ? in[base + k] : 0u;
        sum += v[k];
    }
    uint32_t excl_thread, agg;
    BlockScan(tmp).ExclusiveSum(sum, excl_thread, agg);
    if (threadIdx.x < 32) {
        const uint32_t prefix = lookback_prefix(status, part, epoch, agg);
        if (threadIdx.x == 0) s_excl = prefix;
    }
    __syncthreads();
    uint32_t run = s_excl + excl_thread;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        if (base + k < n) out[base + k] = run;
        run += v[k];
    }
    if (base < n && base + kScanItems >= n) {
        const unsigned long long t = (unsigned long long)(s_excl + excl_thread) + sum;
        *total = t;
        if (total_eff) {   // consumers size their work by the clamped count: never past the capacity
            const bool over = t > (unsigned long long)cap;
            *total_eff = over ? 0ull : t;
            if (over) atomicOr(error_flag, 1u);
        }
    }
}

// ------------------------------------------------------------------ key emission
// One warp per 32 consecutive Gaussians; their outputs are contiguous, so lanes write
// consecutive slots (coalesced). Slot -> Gaussian by a 5-step shuffle binary search.
__global__ void __launch_bounds__(256) emit_keys_kernel(
    int64_t n, const uint32_t* __restrict__ tiles, const uint32_t* __restrict__ offsets,
    const short4* __restrict__ rect, const uint32_t* __restrict__ dkey, int GX,
    const unsigned long long* __restrict__ n_keys, int64_t key_cap, unsigned int* error_flag,
    uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    if (*n_keys > (unsigned long long)key_cap) {
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(error_flag, 1u);
        return;
    }
    const int lane = threadIdx.x & 31;
    const int64_t g0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) - lane;
    if (g0 >= n) return;
    const int64_t g = g0 + lane;
    const bool in = g < n;
    const uint32_t cnt = in ? tiles[g] : 0u;
    const uint32_t start = in ? offsets[g] : 0u;
    const uint32_t base = __shfl_sync(0xffffffffu, start, 0);
    uint32_t rel = in ? start - base : 0xffffffffu;        // monotone in lane (OOB lanes at the end)
    const uint32_t total = __reduce_add_sync(0xffffffffu, cnt);
    short4 rc = in ? rect[g] : make_short4(0, 0, 0, 0);
    const uint32_t dk = in ? dkey[g] : 0u;
    for (uint32_t j0 = 0; j0 < total; j0 += 32) {   // warp-uniform trip count (full-mask shuffles)
        const uint32_t j = j0 + lane;
        int lo = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
            const uint32_t r = __shfl_sync(0xffffffffu, rel, lo + step < 32 ? lo + step : 31);
            if (lo + step < 32 && r <= j) lo += step;
        }
        const uint32_t my_rel = __shfl_sync(0xffffffffu, rel, lo);
        const int xlo = __shfl_sync(0xffffffffu, int(rc.x), lo);
        const int xhi = __shfl_sync(0xffffffffu, int(rc.y), lo);
        const int ylo = __shfl_sync(0xffffffffu, int(rc.z), lo);
        const uint32_t d = __shfl_sync(0xffffffffu, dk, lo);
        if (j < total) {
            const uint32_t l = j - my_rel;
            const uint32_t w = uint32_t(xhi - xlo);
            const uint32_t row = l / w;
            const uint32_t tx = uint32_t(xlo) + (l - row * w), ty = uint32_t(ylo) + row;
            const uint64_t o = uint64_t(base) + j;
            keys[o] = (uint64_t(ty * uint32_t(GX) + tx) << 32) | d;
            vals[o] = uint32_t(g0 + lo);
        }
    }
}

// ------------------------------------------------------------------ per-tile ranges
__global__ void tile_ranges_kernel(const uint64_t* __restrict__ keys, const unsigned long long* __restrict__ n_keys,
                                   uint2* __restrict__ ranges) {
    const uint64_t K = *n_keys;
    for (uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < K; j += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t t = uint32_t(keys[j] >> 32);
        if (j == 0 || uint32_t(keys[j - 1] >> 32) != t) ranges[t].x = uint32_t(j);
        if (j + 1 == K || uint32_t(keys[j + 1] >> 32) != t) ranges[t].y = uint32_t(j + 1);
    }
}

// ------------------------------------------------------------------ host driver
static int ceil_log2(uint32_t v) { int b = 0; while ((1u << b) < v) ++b; return b; }

gs_status chained_scan(WsState* s, const uint32_t* in, uint32_t* out, int64_t n, unsigned long long* total,
                       cudaStream_t st, int64_t cap, unsigned long long* total_eff) {
    Misc* misc = at<Misc>(s, s->misc);
    launch_zero(total, sizeof(*total), st, s);
    if (total_eff) launch_zero(total_eff, sizeof(*total_eff), st, s);
    if (n == 0) return GS_OK;
    launch_zero(&misc->scan_counter, sizeof(misc->scan_counter), st, s);
    const uint32_t epoch = uint32_t(++s->epoch) & 0x3fffffffu;
    const int parts = int((n + kScanTile - 1) / kScanTile);
    KTimer kt(s, KID_SCAN, st);
    chained_scan_kernel<<<parts, kScanThreads, 0, st>>>(in, out, n, at<unsigned long long>(s, s->scan_state),
                                                        &misc->scan_counter, epoch, total, cap, total_eff,
                                                        &misc->error_flag);
    return GS_OK;
}

// On-screen compaction (both paths): list in index order + path B's depth-sort input in
// dkey_sorted / dval_sorted (first half); V_s in misc->n_onscreen and misc->n_items.
gs_status run_compact_onscreen(WsState* s, cudaStream_t st) {
    Misc* misc = at<Misc>(s, s->misc);
    launch_zero(&misc->n_onscreen, sizeof(misc->n_onscreen), st, s);
    launch_zero(&misc->n_items, sizeof(misc->n_items), st, s);
    if (s->n == 0) return GS_OK;
    launch_zero(&misc->scan_counter, sizeof(misc->scan_counter), st, s);
    const uint32_t epoch = uint32_t(++s->epoch) & 0x3fffffffu;
    const int parts = int((s->n + kScanTile - 1) / kScanTile);
    KTimer kt(s, KID_DEPTH_SORT, st);
    compact_onscreen_kernel<<<parts, kScanThreads, 0, st>>>(
        at<uint32_t>(s, s->tiles), at<uint32_t>(s, s->depth_key), s->n, at<unsigned long long>(s, s->scan_state),
        &misc->scan_counter, epoch, at<uint32_t>(s, s->onlist), at<uint32_t>(s, s->dkey_sorted),
        at<uint32_t>(s, s->dval_sorted), &misc->n_onscreen, &misc->n_items, at<float>(s, s->rec));
    return GS_OK;
}

// K readback (host-sync mode) or device-only K (graph mode); returns the grid size to use.
gs_status resolve_keys(WsState* s, int64_t* n_keys, uint32_t flags, cudaStream_t st, int64_t* Kgrid) {
    Misc* misc = at<Misc>(s, s->misc);
    if (!(flags & GS_FLAG_NO_HOST_SYNC)) {
        unsigned long long k = 0;
        if (cudaMemcpyAsync(&k, &misc->n_keys, sizeof(k), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            return check_launch(s, "n_keys readback");
        s->n_keys_host = int64_t(k);
        if (n_keys) *n_keys = int64_t(k);
        if (int64_t(k) > s->key_cap) return GS_ERR_CAPACITY;
        *Kgrid = int64_t(k);
    } else {
        s->n_keys_host = -1;
        if (n_keys) *n_keys = -1;
        *Kgrid = s->key_cap;
    }
    return GS_OK;
}

int ceil_log2_tiles(int64_t ntiles) { return ceil_log2(uint32_t(ntiles)); }

gs_status run_bin_sort_keys(WsState* s, int64_t* n_keys, uint32_t flags, cudaStream_t st) {
    Misc* misc = at<Misc>(s, s->misc);
    const int64_t ntiles = int64_t(s->cam_gx) * s->cam_gy;
    launch_zero(misc, offsetof(Misc, loss_acc), st, s);                 // K, flags, tickets
    launch_zero(at<char>(s, s->ranges), size_t(ntiles) * sizeof(uint2), st, s);
    gs_status rc = chained_scan(s, at<uint32_t>(s, s->tiles), at<uint32_t>(s, s->offsets), s->n, &misc->n_keys, st,
                                s->key_cap, &misc->n_keys_eff);
    if (rc != GS_OK) return rc;
    rc = run_compact_onscreen(s, st);   // on-screen list for the per-Gaussian backward
    if (rc != GS_OK) return rc;
    int64_t Kgrid = 0;
    rc = resolve_keys(s, n_keys, flags, st, &Kgrid);
    if (rc != GS_OK) return rc;
    // emission
    const int blocks = int((s->n + 255) / 256);
    if (blocks > 0) {
        KTimer kt(s, KID_EMIT, st);
        emit_keys_kernel<<<blocks, 256, 0, st>>>(s->n, at<uint32_t>(s, s->tiles), at<uint32_t>(s, s->offsets),
                                                 at<short4>(s, s->rect), at<uint32_t>(s, s->depth_key), s->cam_gx,
                                                 &misc->n_keys, s->key_cap, &misc->error_flag,
                                                 at<uint64_t>(s, s->keys0), at<uint32_t>(s, s->vals0));
    }
    s->keys_valid = 1;
    if (flags & GS_FLAG_BINSORT_EMIT_ONLY) {
        s->sorted_in_1 = 0;
        return check_launch(s, "bin_sort_keys(emit only)");
    }
    // onesweep LSD radix sort over bits [0, 32 + TB)
    const int bits = 32 + ceil_log2(uint32_t(ntiles));
    int which = 0;
    rc = onesweep_sort_pairs(s, at<uint64_t>(s, s->keys0), at<uint32_t>(s, s->vals0), at<uint64_t>(s, s->keys1),
                             at<uint32_t>(s, s->vals1), &misc->n_keys_eff, Kgrid, bits, st, &which);
    if (rc != GS_OK) return rc;
    s->sorted_in_1 = which;
    const uint64_t* sk = which ? at<uint64_t>(s, s->keys1) : at<uint64_t>(s, s->keys0);
    if (Kgrid > 0) {
        const int rblocks = int(std::min<int64_t>((Kgrid + 255) / 256, sm_count() * 16));
        KTimer kt(s, KID_RANGES, st);
        tile_ranges_kernel<<<rblocks, 256, 0, st>>>(sk, &misc->n_keys_eff, at<uint2>(s, s->ranges));
    }
    return check_launch(s, "bin_sort_keys");
}

}  // namespace gs
