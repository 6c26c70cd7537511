// gs_bin_sort, path B (default): depth presort + ordered tile bucketing.
//
// Output-identical to path A (the stable sort of the index-order (tile|depth) keys, O2)
// without materialising or sorting the K keys:
//   B1-B4 (one cooperative kernel, bincoop.cu): compaction of the V_s on-screen Gaussians; stable
//         LSD radix sort of their (depth bits, index) pairs; chunks of 256 depth-ordered Gaussians
//         with per-chunk tile counts count[c][t] (2-D difference arrays); per-tile exclusive scans
//         -> ranges, K and base[c][t]
//   B5  emission:   warp work item = (chunk, 8x4-tile area): the warp lists (in depth order) the
//                   chunk's Gaussians meeting its area with 32-bit tile masks, then per tile a
//                   ballot/popc prefix ranks the hits of 32 Gaussians at a time and places them at
//                   base[c][t] + rank (coalesced 4-B stores, depth order preserved)
// Per tile, entries come out in chunk order and in depth order within a chunk, i.e. ordered by
// (depth bits, index): exactly the per-tile lists of path A (checked bit-exact in the tests).
// HBM traffic is ~4 B per key (+ per-Gaussian and per-chunk terms) instead of ~150 B per key.
#include <cub/block/block_scan.cuh>

#include <algorithm>

#include "gs_internal.cuh"

namespace gs {

gs_status resolve_keys(WsState* s, int64_t* n_keys, uint32_t flags, cudaStream_t st, int64_t* Kgrid);

// B5 ---------------------------------------------------------------------------------------
// Block = (16x16-tile area, chunks c = blockIdx.x + i * gridDim.x below ceil(V_s / 256), read on the
// device). Warp-specialised, with no block barriers in the loop:
//   producer warps (8, 9; alternating chunks): per chunk, test its 256 Gaussians (8 per lane, depth order)
//      against the block area and compacts the hits in order (ballot + popc) into a slot of a
//      4-deep shared-memory ring, then arrives on the slot's "full" mbarrier;
//   consumer warps 0-7, each an 8x4-tile sub-area (lane j = tile (j & 7, j >> 3)): wait on "full",
//      list the slot's Gaussians meeting the sub-area with 32-bit tile masks (the rect's x-run
//      replicated over its rows: one multiply), arrive on the slot's "empty" mbarrier, then per group
//      of 32 listed Gaussians and per tile present in the group, a ballot of the mask bit ranks the
//      hits (popc below the lane), which go to base[c][t_j] + running count: coalesced 4-B stores
//      straight from registers. Lane j keeps tile j's running position.
// Square sub-areas keep the masks dense (the rects are roughly square); the ring lets a consumer run
// up to 4 chunks ahead of the slowest one instead of meeting it at a barrier every chunk.
constexpr int kWX = 8, kWY = 4;        // consumer tile area (lane j = tile (j & 7, j >> 3))
constexpr int kBX = 16, kBY = 16;      // block tile area: 2 x 4 consumer areas
// grid.x (chunk stride): 256 up to ~1M Gaussians, 512 beyond (measured, round 2: config 2 with 128 /
// 256 / 512 / 1024 -> 0.080 / 0.073 / 0.077 / 0.083 ms; config-4 size 0.384 / 0.349 / 0.333 / 0.340 ms)
constexpr int kEmitChunkBlocksMin = 256, kEmitChunkBlocksMax = 512;
constexpr int kRing = 4;               // chunk slots in flight
constexpr int kConsumers = 8;
constexpr int kProducers = 2;          // producer warps, alternating chunks (ring order kept)

struct EmitSmem {
    short4 rect[kRing][kChunk];
    uint32_t g[kRing][kChunk];
    int cnt[kRing];
    unsigned long long full[kRing], empty[kRing];   // mbarriers
    uint2 l_mg[kConsumers][kChunk];                 // (tile mask, Gaussian) of each consumer's list
};

__device__ __forceinline__ uint32_t span_bits(int lo, int hi) {   // bits [lo, hi), 0 <= lo < hi <= 8
    return ((1u << hi) - 1u) & ~((1u << lo) - 1u);
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(unsigned(__cvta_generic_to_shared(b))), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(
                     unsigned(__cvta_generic_to_shared(b)))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
    const unsigned a = unsigned(__cvta_generic_to_shared(b));
    unsigned done = 0;
    do {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done)
                     : "r"(a), "r"(parity)
                     : "memory");
    } while (!done);
}

__global__ void __launch_bounds__((kConsumers + kProducers) * 32) bucket_emit_kernel(
    const uint32_t* __restrict__ svals, const short4* __restrict__ srect, const uint32_t* __restrict__ cmat,
    const unsigned int* __restrict__ n_on, const unsigned long long* __restrict__ n_keys_eff,
    const unsigned long long* __restrict__ n_keys, int GX, int GY, uint32_t* __restrict__ vals_out,
    uint2* __restrict__ ranges) {
    __shared__ EmitSmem sm;
    griddep_wait();   // PDL (gs_internal.cuh)
    if (*n_keys_eff != *n_keys) {
        // capacity overflow (the error flag is set): emit nothing and empty every tile's range, so the
        // render kernels that follow in NO_HOST_SYNC mode read no list entry beyond key_cap
        const int nb = gridDim.x * gridDim.y * gridDim.z;
        const int b = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
        for (int t = b * blockDim.x + threadIdx.x; t < GX * GY; t += nb * blockDim.x) ranges[t] = make_uint2(0u, 0u);
        return;
    }
    const uint32_t Von = *n_on;
    const int nch = int((Von + kChunk - 1) / kChunk);
    const int T = GX * GY;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    const int bx0 = blockIdx.y * kBX, by0 = blockIdx.z * kBY;
    if (threadIdx.x == 0) {
        for (int r = 0; r < kRing; ++r) {
            mbar_init(&sm.full[r], 1);
            mbar_init(&sm.empty[r], kConsumers);
        }
    }
    __syncthreads();
    if (warp >= kConsumers) {
        // ---------------------------------------------------------------- producers
        const int pw = warp - kConsumers;
        int it = pw;
        for (int c = blockIdx.x + pw * gridDim.x; c < nch; c += kProducers * gridDim.x, it += kProducers) {
            const int slot = it % kRing;
            const uint32_t s0 = uint32_t(c) * kChunk;
            short4 r[kChunk / 32];
            uint32_t gq[kChunk / 32];
#pragma unroll
            for (int q = 0; q < kChunk / 32; ++q) {   // loads first (independent of the ring)
                const uint32_t s = s0 + q * 32 + lane;
                r[q] = s < Von ? srect[s] : make_short4(0, 0, 0, 0);
                gq[q] = s < Von ? svals[s] : 0u;
            }
            if (it >= kRing) mbar_wait(&sm.empty[slot], ((it / kRing) - 1) & 1);
            int L = 0;
#pragma unroll
            for (int q = 0; q < kChunk / 32; ++q) {
                const bool meet = max(int(r[q].x), bx0) < min(int(r[q].y), bx0 + kBX) &&
                                  max(int(r[q].z), by0) < min(int(r[q].w), by0 + kBY);
                const uint32_t m = __ballot_sync(0xffffffffu, meet);
                if (meet) {
                    const int o = L + __popc(m & lt);
                    sm.rect[slot][o] = r[q];
                    sm.g[slot][o] = gq[q];
                }
                L += __popc(m);
            }
            if (lane == 0) sm.cnt[slot] = L;
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.full[slot]);   // release: the slot's writes are visible
        }
        return;
    }
    // -------------------------------------------------------------------- consumers
    const int x0 = bx0 + (warp & 1) * kWX, y0 = by0 + (warp >> 1) * kWY;
    const int tx = x0 + (lane & 7), ty = y0 + (lane >> 3);
    const bool valid = tx < GX && ty < GY;
    const bool warp_in = x0 < GX && y0 < GY;
    uint2* list = sm.l_mg[warp];
    int it = 0;
    uint32_t pos_nx = (valid && blockIdx.x < nch) ? cmat[size_t(blockIdx.x) * T + ty * GX + tx] : 0u;
    for (int c = blockIdx.x; c < nch; c += gridDim.x, ++it) {
        const int slot = it % kRing;
        // this chunk's base position of my tile, and the next chunk's (loaded a chunk ahead)
        uint32_t mypos = pos_nx;
        const int cn = c + gridDim.x;
        pos_nx = (valid && cn < nch) ? cmat[size_t(cn) * T + ty * GX + tx] : 0u;
        mbar_wait(&sm.full[slot], (it / kRing) & 1);
        const int tot = sm.cnt[slot];
        int L = 0;
        if (warp_in) {
            for (int k0 = 0; k0 < tot; k0 += 32) {
                const int k = k0 + lane;
                uint32_t mask = 0;
                if (k < tot) {
                    const short4 r = sm.rect[slot][k];
                    const int xlo = max(int(r.x) - x0, 0), xhi = min(int(r.y) - x0, kWX);
                    const int ylo = max(int(r.z) - y0, 0), yhi = min(int(r.w) - y0, kWY);
                    if (xlo < xhi && ylo < yhi)
                        mask = span_bits(xlo, xhi) * ((span_bits(ylo, yhi) * 0x00204081u) & 0x01010101u);
                }
                const uint32_t m = __ballot_sync(0xffffffffu, mask != 0u);
                if (mask) list[L + __popc(m & lt)] = make_uint2(mask, sm.g[slot][k]);
                L += __popc(m);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[slot]);   // the slot is no longer read by this warp
        if (L == 0) continue;                          // warp-uniform
        for (int k0 = 0; k0 < L; k0 += 32) {
            const int k = k0 + lane;
            const uint2 mg = k < L ? list[k] : make_uint2(0u, 0u);
            // the 32x32 bit matrix (row = lane's tile mask) transposed with five butterfly exchanges:
            // lane j then holds column j, i.e. which of the 32 Gaussians hit tile j (its ballot)
            uint32_t x = mg.x;
#pragma unroll
            for (int sh = 16; sh >= 1; sh >>= 1) {
                const uint32_t lo = sh == 16 ? 0x0000FFFFu : sh == 8 ? 0x00FF00FFu : sh == 4 ? 0x0F0F0F0Fu
                                  : sh == 2 ? 0x33333333u : 0x55555555u;
                const uint32_t y = __shfl_xor_sync(0xffffffffu, x, sh);
                x = (lane & sh) ? ((x & ~lo) | ((y & ~lo) >> sh)) : ((x & lo) | ((y & lo) << sh));
            }
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const uint32_t m = __shfl_sync(0xffffffffu, x, j);
                const uint32_t pj = __shfl_sync(0xffffffffu, mypos, j);
                if (mg.x & (1u << j)) vals_out[pj + __popc(m & lt)] = mg.y;
            }
            mypos += __popc(x);
        }
        __syncwarp();   // list reuse
    }
}

gs_status run_bin_coop(WsState* s, cudaStream_t st);   // bincoop.cu (B1-B4)

gs_status run_bin_sort_bucket(WsState* s, int64_t* n_keys, uint32_t flags, cudaStream_t st) {
    Misc* misc = at<Misc>(s, s->misc);
    const int T = s->cam_gx * s->cam_gy;
    const int64_t n = s->n;
    launch_zero(misc, offsetof(Misc, loss_acc), st, s);   // K, flags, barrier, key range
    gs_status rc = GS_OK;
    if (n > 0) {
        rc = run_bin_coop(s, st);   // B1-B4: compaction, depth sort, chunk counts, tile scans
        if (rc != GS_OK) return rc;
        const int nch = int((n + kChunk - 1) / kChunk);
        KTimer kt(s, KID_BUCKET_EMIT, st);
        const int gx = std::min(kEmitChunkBlocksMax, std::max(kEmitChunkBlocksMin, nch / 8));
        const dim3 grid(unsigned(std::min(nch, gx)), unsigned((s->cam_gx + kBX - 1) / kBX),
                        unsigned((s->cam_gy + kBY - 1) / kBY));
        launch_pdl(bucket_emit_kernel, grid, dim3((kConsumers + kProducers) * 32), 0, st, at<uint32_t>(s, s->svals), at<short4>(s, s->srect),
                                                 at<uint32_t>(s, s->chunk_mat), &misc->n_onscreen, &misc->n_keys_eff,
                                                 &misc->n_keys, s->cam_gx, s->cam_gy, at<uint32_t>(s, s->vals0),
                                                 at<uint2>(s, s->ranges));
    } else {
        launch_zero(at<char>(s, s->ranges), size_t(T) * sizeof(uint2), st, s);
    }
    s->sorted_in_1 = 0;
    s->keys_valid = 0;
    int64_t Kgrid = 0;
    rc = resolve_keys(s, n_keys, flags, st, &Kgrid);   // host-sync mode: K readback + capacity status
    if (rc != GS_OK) return rc;
    return check_launch(s, "bin_sort_bucket");
}

}  // namespace gs
