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
// device); warp = 8x4-tile sub-area (square, like the rects, so a Gaussian meeting the area covers
// more of it than of a 32-tile row segment: fewer empty (Gaussian, tile) slots). Per chunk:
//   1. block pre-filter: the chunk's Gaussians whose rect meets the block area, in depth order
//      (BlockScan compaction; the next chunk's rects and indices are loaded meanwhile);
//   2. warp list: those meeting the warp area with their 32-bit masks over its 8x4 tiles (the rect's
//      x-run replicated over its rows: one multiply), compacted in order with ballot + popc;
//   3. per group of 32 listed Gaussians and per tile j present in the group: a ballot of the mask
//      bit ranks the group's hits (popc below the lane), which go to base[c][t_j] + running count:
//      coalesced 4-B stores straight from registers. Lane j keeps tile j's running position.
constexpr int kWX = 8, kWY = 4;        // warp tile area (lane j = tile (j & 7, j >> 3))
constexpr int kBX = 16, kBY = 16;      // block tile area: 2 x 4 warp areas
constexpr int kEmitChunkBlocks = 96;   // grid.x: chunk stride

struct EmitSmem {
    short4 b_rect[kChunk];
    uint32_t b_g[kChunk];
    uint2 l_mg[8][kChunk];             // (tile mask, Gaussian) of each warp's list
};

__device__ __forceinline__ uint32_t span_bits(int lo, int hi) {   // bits [lo, hi), 0 <= lo < hi <= 8
    return ((1u << hi) - 1u) & ~((1u << lo) - 1u);
}

__global__ void __launch_bounds__(256) bucket_emit_kernel(
    const uint32_t* __restrict__ svals, const short4* __restrict__ srect, const uint32_t* __restrict__ cmat,
    const unsigned int* __restrict__ n_on, const unsigned long long* __restrict__ n_keys_eff,
    const unsigned long long* __restrict__ n_keys, int GX, int GY, uint32_t* __restrict__ vals_out) {
    __shared__ EmitSmem sm;
    using BS = cub::BlockScan<int, 256>;
    __shared__ typename BS::TempStorage scan;
    __shared__ int s_tot;
    if (*n_keys_eff != *n_keys) return;   // capacity overflow: emit nothing (error flag is set)
    const uint32_t Von = *n_on;
    const int nch = int((Von + kChunk - 1) / kChunk);
    const int T = GX * GY;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    const int bx0 = blockIdx.y * kBX, by0 = blockIdx.z * kBY;
    const int x0 = bx0 + (warp & 1) * kWX, y0 = by0 + (warp >> 1) * kWY;
    const int tx = x0 + (lane & 7), ty = y0 + (lane >> 3);
    const bool valid = tx < GX && ty < GY;
    const bool warp_in = x0 < GX && y0 < GY;
    auto fetch = [&](int c, short4& r, uint32_t& g) {
        const uint32_t s = uint32_t(c) * kChunk + tid;
        const bool ok = c < nch && s < Von;
        r = ok ? srect[s] : make_short4(0, 0, 0, 0);
        g = ok ? svals[s] : 0u;
    };
    short4 r_nx;
    uint32_t g_nx;
    fetch(blockIdx.x, r_nx, g_nx);
    for (int c = blockIdx.x; c < nch; c += gridDim.x) {
        // 1. block pre-filter (an empty rect, r.x == r.y, meets nothing)
        {
            const short4 r = r_nx;
            const uint32_t g = g_nx;
            fetch(c + gridDim.x, r_nx, g_nx);
            const bool meet =
                max(int(r.x), bx0) < min(int(r.y), bx0 + kBX) && max(int(r.z), by0) < min(int(r.w), by0 + kBY);
            int off, tot;
            BS(scan).ExclusiveSum(meet ? 1 : 0, off, tot);
            if (meet) {
                sm.b_rect[off] = r;
                sm.b_g[off] = g;
            }
            if (tid == 0) s_tot = tot;
            __syncthreads();
        }
        const int tot = s_tot;
        if (tot > 0 && warp_in) {   // warp-uniform: no block barriers inside
            // 2. warp list
            int L = 0;
            for (int k0 = 0; k0 < tot; k0 += 32) {
                const int k = k0 + lane;
                uint32_t mask = 0;
                if (k < tot) {
                    const short4 r = sm.b_rect[k];
                    const int xlo = max(int(r.x) - x0, 0), xhi = min(int(r.y) - x0, kWX);
                    const int ylo = max(int(r.z) - y0, 0), yhi = min(int(r.w) - y0, kWY);
                    if (xlo < xhi && ylo < yhi)
                        mask = span_bits(xlo, xhi) * ((span_bits(ylo, yhi) * 0x00204081u) & 0x01010101u);
                }
                const uint32_t m = __ballot_sync(0xffffffffu, mask != 0u);
                if (mask) sm.l_mg[warp][L + __popc(m & lt)] = make_uint2(mask, sm.b_g[k]);
                L += __popc(m);
            }
            __syncwarp();
            // 3. ranked stores, 32 Gaussians x 32 tiles per group
            uint32_t mypos = valid && L > 0 ? cmat[size_t(c) * T + ty * GX + tx] : 0u;
            for (int k0 = 0; k0 < L; k0 += 32) {
                const int k = k0 + lane;
                const uint2 mg = k < L ? sm.l_mg[warp][k] : make_uint2(0u, 0u);
                const uint32_t any = __reduce_or_sync(0xffffffffu, mg.x);
                uint32_t mine = 0;   // lane j: ballot of tile j
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    if (!(any & (1u << j))) continue;   // warp-uniform
                    const bool hit = mg.x & (1u << j);
                    const uint32_t m = __ballot_sync(0xffffffffu, hit);
                    const uint32_t pj = __shfl_sync(0xffffffffu, mypos, j);
                    if (hit) vals_out[pj + __popc(m & lt)] = mg.y;
                    mine = lane == j ? m : mine;
                }
                mypos += __popc(mine);
            }
        }
        __syncthreads();   // b_rect / b_g reuse by the next chunk
    }
}

gs_status run_bin_coop(WsState* s, cudaStream_t st);   // bincoop.cu (B1-B4)

gs_status run_bin_sort_bucket(WsState* s, int64_t* n_keys, uint32_t flags, cudaStream_t st) {
    Misc* misc = at<Misc>(s, s->misc);
    const int T = s->cam_gx * s->cam_gy;
    const int64_t n = s->n;
    cudaMemsetAsync(misc, 0, offsetof(Misc, loss_acc), st);   // K, flags, barrier, key range
    gs_status rc = GS_OK;
    if (n > 0) {
        rc = run_bin_coop(s, st);   // B1-B4: compaction, depth sort, chunk counts, tile scans
        if (rc != GS_OK) return rc;
        const int nch = int((n + kChunk - 1) / kChunk);
        KTimer kt(s, KID_BUCKET_EMIT, st);
        const dim3 grid(unsigned(std::min(nch, kEmitChunkBlocks)), unsigned((s->cam_gx + kBX - 1) / kBX),
                        unsigned((s->cam_gy + kBY - 1) / kBY));
        bucket_emit_kernel<<<grid, 256, 0, st>>>(at<uint32_t>(s, s->svals), at<short4>(s, s->srect),
                                                 at<uint32_t>(s, s->chunk_mat), &misc->n_onscreen, &misc->n_keys_eff,
                                                 &misc->n_keys, s->cam_gx, s->cam_gy, at<uint32_t>(s, s->vals0));
    } else {
        cudaMemsetAsync(at<char>(s, s->ranges), 0, size_t(T) * sizeof(uint2), st);
    }
    s->sorted_in_1 = 0;
    s->keys_valid = 0;
    int64_t Kgrid = 0;
    rc = resolve_keys(s, n_keys, flags, st, &Kgrid);   // host-sync mode: K readback + capacity status
    if (rc != GS_OK) return rc;
    return check_launch(s, "bin_sort_bucket");
}

}  // namespace gs
