// Onesweep-style LSD radix sort of (key, u32 value) pairs, 8-bit digits (sm_100a).
//  1. one upfront pass builds the digit histograms of every pass (reads the keys once), or the
//     producer of the keys accumulates them; each pass kernel scans its histogram in-CTA;
//  2. each digit pass is ONE kernel: a CTA takes the next partition from an atomic ticket
//     (forward progress for the look-back), ranks its kSortTile (2048) keys stably with warp match_any,
//     publishes its per-digit counts, resolves its global digit offsets by decoupled look-back
//     over its predecessors, and scatters through shared memory so stores are coalesced per digit.
// Look-back words are [epoch:30 | flag:2 | count:32]; a fresh epoch per pass makes stale words
// from earlier passes read as "not ready", so no memset is needed between passes.
// Stability: within a partition, keys are ranked in (warp, item, lane) order, which is their
// input order; across partitions by ticket order. So ties keep their input order (LSD-correct).
#pragma once
#include <cub/block/block_scan.cuh>

#include "gs_internal.cuh"

namespace gs {

constexpr int kSortThreads = 256, kSortItems = 8, kSortTile = kSortThreads * kSortItems;
constexpr int kSortItemsSmall = 4;   // 1024-key partitions for small sorts (more CTAs, shorter latency)

template <class KT>
__global__ void __launch_bounds__(256) onesweep_hist_kernel(const KT* __restrict__ keys,
                                                            const unsigned long long* __restrict__ n_keys,
                                                            int npass, uint32_t* __restrict__ hist) {
    __shared__ uint32_t sh[8][256];
    for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) (&sh[0][0])[i] = 0;
    __syncthreads();
    const uint64_t K = *n_keys;
    for (uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < K; j += uint64_t(gridDim.x) * blockDim.x) {
        const KT k = keys[j];
        for (int p = 0; p < npass; ++p) atomicAdd(&sh[p][uint32_t(k >> (8 * p)) & 255u], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < npass * 256; i += blockDim.x) {
        const uint32_t c = (&sh[0][0])[i];
        if (c) atomicAdd(hist + i, c);
    }
}

__device__ __forceinline__ unsigned long long look_word(uint32_t epoch, uint32_t flag, uint32_t v) {
    return (uint64_t(epoch & 0x3fffffffu) << 34) | (uint64_t(flag) << 32) | v;
}

template <class KT, int IPT>
struct OnesweepSmem {
    KT keys[kSortThreads * IPT];
    uint32_t vals[kSortThreads * IPT];
    uint32_t wh[kSortThreads / 32][256];
    uint32_t local_start[256];
    uint32_t gbase[256];
    typename cub::BlockScan<uint32_t, 256>::TempStorage scan;
    uint32_t part;
};

template <class KT, int IPT>
__global__ void __launch_bounds__(kSortThreads) onesweep_pass_kernel(
    const KT* __restrict__ kin, const uint32_t* __restrict__ vin, KT* __restrict__ kout, uint32_t* __restrict__ vout,
    const unsigned long long* __restrict__ n_keys, int shift, const uint32_t* __restrict__ digit_hist,
    unsigned long long* look, unsigned int* ticket, uint32_t epoch) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    OnesweepSmem<KT, IPT>& sm = *reinterpret_cast<OnesweepSmem<KT, IPT>*>(smem_raw);
    constexpr int kTileKeys = kSortThreads * IPT;
    const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
    if (tid == 0) sm.part = atomicAdd(ticket, 1u);
    for (int i = tid; i < (kSortThreads / 32) * 256; i += kSortThreads) (&sm.wh[0][0])[i] = 0;
    // this pass' global digit offsets: exclusive scan of its histogram (thread t = digit t)
    uint32_t dbase;
    cub::BlockScan<uint32_t, 256>(sm.scan).ExclusiveSum(digit_hist[tid], dbase);
    __syncthreads();
    const uint32_t part = sm.part;
    const uint64_t K = *n_keys;
    const uint64_t tile_base = uint64_t(part) * kTileKeys;
    if (tile_base >= K) return;   // block-uniform

    KT key[IPT];
    uint32_t val[IPT], dig[IPT], rnk[IPT];
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
        const uint64_t idx = tile_base + uint64_t(w) * (32 * IPT) + uint64_t(i) * 32 + lane;
        const bool ok = idx < K;
        key[i] = ok ? kin[idx] : KT(0);
        val[i] = ok ? vin[idx] : 0u;
        dig[i] = ok ? (uint32_t(key[i] >> shift) & 255u) : 256u;
    }
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
        const uint32_t d = dig[i];
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const int leader = __ffs(peers) - 1;
        uint32_t pre = 0;
        if (d < 256) pre = sm.wh[w][d];
        __syncwarp();
        if (d < 256 && lane == leader) sm.wh[w][d] = pre + __popc(peers);
        __syncwarp();
        rnk[i] = pre + __popc(peers & lt);
    }
    __syncthreads();
    // digit t: per-warp exclusive offsets and the partition's count
    const int t = tid;
    uint32_t cnt = 0;
#pragma unroll
    for (int w2 = 0; w2 < kSortThreads / 32; ++w2) {
        const uint32_t c = sm.wh[w2][t];
        sm.wh[w2][t] = cnt;
        cnt += c;
    }
    // decoupled look-back for digit t
    unsigned long long* my = look + uint64_t(part) * 256 + t;
    uint32_t excl = 0;
    if (part == 0) {
        atomicExch(my, look_word(epoch, 2, cnt));
    } else {
        atomicExch(my, look_word(epoch, 1, cnt));
        // walk back 8 predecessors per round: 8 independent loads in flight, then consume in order
        const uint32_t ep = epoch & 0x3fffffffu;
        auto flag_of = [ep](uint64_t wd) { return (uint32_t(wd >> 34) == ep) ? uint32_t((wd >> 32) & 3u) : 0u; };
        int64_t j = int64_t(part) - 1;
        bool done = false;
        while (!done && j >= 0) {
            uint64_t wd[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                wd[u] = (j - u >= 0) ? *reinterpret_cast<volatile unsigned long long*>(look + uint64_t(j - u) * 256 + t)
                                     : 0ull;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                if (done || j - u < 0) break;
                uint32_t flag = flag_of(wd[u]);
                while (flag == 0) {   // not published yet: spin on this predecessor
                    wd[u] = *reinterpret_cast<volatile unsigned long long*>(look + uint64_t(j - u) * 256 + t);
                    flag = flag_of(wd[u]);
                }
                excl += uint32_t(wd[u]);
                if (flag == 2) done = true;
            }
            j -= 8;
        }
        atomicExch(my, look_word(epoch, 2, excl + cnt));
    }
    uint32_t lstart;
    cub::BlockScan<uint32_t, 256>(sm.scan).ExclusiveSum(cnt, lstart);
    sm.local_start[t] = lstart;
    sm.gbase[t] = dbase + excl;
    __syncthreads();
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
        const uint32_t d = dig[i];
        if (d < 256) {
            const uint32_t pos = sm.local_start[d] + sm.wh[w][d] + rnk[i];
            sm.keys[pos] = key[i];
            sm.vals[pos] = val[i];
        }
    }
    __syncthreads();
    const uint64_t rem = K - tile_base;
    const uint32_t nvalid = rem < uint64_t(kTileKeys) ? uint32_t(rem) : uint32_t(kTileKeys);
    for (uint32_t j = tid; j < nvalid; j += kSortThreads) {
        const KT k = sm.keys[j];
        const uint32_t d = uint32_t(k >> shift) & 255u;
        const uint32_t o = sm.gbase[d] + (j - sm.local_start[d]);
        kout[o] = k;
        vout[o] = sm.vals[j];
    }
}

// Sort (k0, v0) by bits [0, bits). Ping-pongs with (k1, v1); *which = buffer holding the result.
// K lives on the device (n_keys); Kgrid >= K sizes the grids (exact in host-sync mode).
// hist_ready: the producer of (k0, v0) already accumulated the per-pass digit histograms into the
// workspace's sort_hist (zeroed beforehand), so the histogram kernel is skipped.
template <class KT, int IPT = kSortItems>
gs_status onesweep_sort_pairs(WsState* s, KT* k0, uint32_t* v0, KT* k1, uint32_t* v1, const unsigned long long* n_keys,
                              int64_t Kgrid, int bits, cudaStream_t st, int* which, bool hist_ready = false) {
    Misc* misc = at<Misc>(s, s->misc);
    const int npass = (bits + 7) / 8;
    uint32_t* hist = at<uint32_t>(s, s->sort_hist);
    *which = 0;
    if (Kgrid <= 0) return GS_OK;
    cudaMemsetAsync(misc->sort_counter, 0, sizeof(misc->sort_counter), st);
    if (!hist_ready) {
        cudaMemsetAsync(hist, 0, sizeof(uint32_t) * 256 * npass, st);
        const int blocks = int(std::min<int64_t>((Kgrid + 255) / 256, sm_count() * 8));
        KTimer kt(s, KID_SORT_HIST, st);
        onesweep_hist_kernel<KT><<<blocks, 256, 0, st>>>(k0, n_keys, npass, hist);
    }
    const size_t smem = sizeof(OnesweepSmem<KT, IPT>);
    static PerDeviceOnce attr;   // the attribute is per device
    attr.run([smem] {
        return cudaFuncSetAttribute(onesweep_pass_kernel<KT, IPT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(smem)) == cudaSuccess;
    });
    const int64_t parts = (Kgrid + kSortThreads * IPT - 1) / (kSortThreads * IPT);
    if (parts > s->max_parts) return GS_ERR_CAPACITY;
    KT* kin = k0; uint32_t* vin = v0; KT* ko = k1; uint32_t* vo = v1;
    for (int p = 0; p < npass; ++p) {
        const uint32_t epoch = uint32_t(++s->epoch) & 0x3fffffffu;
        KTimer kt(s, KID_SORT_PASS, st);
        onesweep_pass_kernel<KT, IPT><<<int(parts), kSortThreads, smem, st>>>(
            kin, vin, ko, vo, n_keys, 8 * p, hist + 256 * p, at<unsigned long long>(s, s->sort_look),
            misc->sort_counter + p, epoch);
        std::swap(kin, ko);
        std::swap(vin, vo);
        *which ^= 1;
    }
    return GS_OK;
}

}  // namespace gs
