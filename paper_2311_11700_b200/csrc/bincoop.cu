// gs_bin_sort, path B, front half: ONE cooperative (grid-synchronised) kernel, one CTA per SM.
//
// Everything before the bucket emission (bucket.cu B5) is latency-bound at the paper's sizes
// (V_s ~ 1e5 on-screen Gaussians): as separate launches, compaction + a 4-pass onesweep depth sort +
// chunk counts + three tile-scan kernels cost ~0.13 ms at config 2, mostly launch and look-back
// latency. Here the same work runs as phases of one persistent kernel separated by grid barriers:
//   C0  compaction: per CTA a contiguous slice of the n Gaussians; counts and
//       the on-screen depth-key range -> barrier -> ordered writes of onlist[V_s] (index order) and
//       the depth-sort pairs (key - kmin, i), with every pass' digit histogram
//   C1  stable LSD radix sort (a4) of the V_s pairs over the bits that vary (kmax - kmin), in
//       P = ceil(bits / 9) passes of <= 9-bit digits (3 passes at config 2). A pass: global digit
//       base + the sum of the preceding CTAs' histograms of this digit -> stable in-CTA ranking
//       (warp match_any, per-warp digit counts) -> scatter; the scatter also counts the next pass'
//       digits per destination slice (global atomics), so each pass costs one barrier. Ties keep
//       their order (slices are contiguous and ranked in order), so equal depths stay by index.
//       The last pass writes svals[s] (the s-th on-screen Gaussian in (depth, index) order) and its
//       rect srect[s] instead of keys.
//   C2  chunk counts: per 256-Gaussian chunk of svals, a 2-D difference array over the tile grid in
//       shared memory -> count[c][t] (4 chunks per CTA in flight)
//   C3  per tile group (CTA) and chunk segment (warp): segment sums, their exclusive prefix over the
//       tile's segments and the tile totals, in shared memory -> barrier ->
//   C4  per tile group: its start (sum of all earlier totals), the tiles' starts (ranges = a5, K,
//       capacity flag) and the exclusive scans over chunks: count[c][t] is replaced by
//       base[c][t] = start of chunk c's entries in tile t's list.
// The grid barrier is the cooperative-groups pattern (block barrier, one thread fences and arrives
// on a monotone counter, spins on an acquire load); cudaLaunchCooperativeKernel guarantees that all
// CTAs are co-resident. Data produced inside the kernel is read with ld.global.cg (L2), never
// through the non-coherent L1.
#include <cub/block/block_scan.cuh>

#include <algorithm>

#include "gs_internal.cuh"

namespace gs {

constexpr int kCT = 1024;                // threads per CTA
constexpr int kCW = kCT / 32;            // warps per CTA
constexpr int kDigitBits = 9;            // <= 9-bit digits (kCoopBins = 512)
constexpr int kCGroups = 4;              // chunk-count groups of 256 threads
constexpr int kRounds = 4;               // compaction: 1024-element rounds loaded at once
static_assert(kRounds * kCW <= kCT, "one scan over the (round, warp) counts");
static_assert(kCoopSegs == kCW, "C3/C4: one warp per chunk segment");

struct CoopArgs {
    const uint32_t* tiles;   // [n] tiles touched (gs_project)
    const uint32_t* dkey;    // [n] depth key bits
    const short4* rect;      // [n] tile rect {x_lo, x_hi, y_lo, y_hi}
    int64_t n;
    int GX, GY;
    int64_t key_cap;
    uint32_t* onlist;        // [n] on-screen Gaussians, index order
    float* rec_f;            // projected records, 12 floats each (r2.w <- on-screen rank)
    uint32_t* k0; uint32_t* v0; uint32_t* k1; uint32_t* v1;   // [n] ping-pong sort buffers
    uint32_t* svals;         // [n] depth-sorted on-screen Gaussians
    short4* srect;           // [n] their rects
    uint32_t* cmat;          // [nch][T] counts -> bases
    uint32_t* H;             // [kCoopPasses][kCoopGridMax][kCoopBins] per-pass per-CTA digit counts
    uint32_t* hist_all;      // [kCoopPasses][kCoopBins] per-pass digit totals
    uint32_t* cta_cnt;       // [kCoopGridMax] on-screen count per compaction slice
    uint32_t* tot;           // [T] tile totals
    uint32_t* segsum;        // [kCoopSegs][T] exclusive prefix of a tile's chunk-segment sums
    uint2* ranges;           // [T]
    Misc* misc;
    int groups;              // chunk-count groups per CTA (shared-memory bound)
};

__device__ __forceinline__ uint32_t ldcg(const uint32_t* p) { return __ldcg(p); }

__device__ __forceinline__ void group_sync(int g) {   // named barrier of one 256-thread group
    asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "r"(256) : "memory");
}

__device__ __forceinline__ void seg_range(int nch, int seg, int& c0, int& c1) {
    const int per = (nch + kCoopSegs - 1) / kCoopSegs;
    c0 = min(nch, seg * per);
    c1 = min(nch, c0 + per);
}

__global__ void __launch_bounds__(kCT, 1) bin_coop_kernel(CoopArgs a) {
    extern __shared__ __align__(16) uint32_t dyn[];
    using BScan = cub::BlockScan<uint32_t, kCT>;
    __shared__ typename BScan::TempStorage bscan;
    __shared__ uint32_t s_hist[kCoopPasses][kCoopBins];
    __shared__ uint32_t s_run[kCoopBins], s_gpos[kCoopBins];
    __shared__ uint32_t s_u[8];
    __shared__ uint32_t s_wc[kCW];
    __shared__ uint32_t s_rw[kRounds * kCW];   // per-(round, warp) on-screen counts -> offsets
    const int G = gridDim.x, k = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int T = a.GX * a.GY;
    Misc* misc = a.misc;
    unsigned int goal = 0;

    // zero the accumulators of later phases (ordered before their use by the first barrier)
    {
        const int64_t nz1 = int64_t(kCoopPasses) * kCoopGridMax * kCoopBins;   // H (rows of passes >= 1 used)
        for (int64_t i = int64_t(k) * kCT + tid; i < nz1; i += int64_t(G) * kCT)
            if (i >= int64_t(kCoopGridMax) * kCoopBins) a.H[i] = 0u;
        for (int i = k * kCT + tid; i < kCoopPasses * kCoopBins; i += G * kCT) a.hist_all[i] = 0u;
    }
    // ---------------------------------------------------------------- C0 compaction: count
    // Slices are read kRounds x 1024 elements at a time, all loads in flight before any use.
    const int64_t S1 = (a.n + G - 1) / G;
    const int64_t b0 = min(a.n, int64_t(k) * S1), b1 = min(a.n, b0 + S1);
    uint32_t kmin = 0xffffffffu, kmax = 0u, cnt = 0;
    if (tid == 0) { s_u[0] = 0xffffffffu; s_u[1] = 0u; }
    for (int64_t r0 = b0; r0 < b1; r0 += int64_t(kRounds) * kCT) {
        uint32_t tl[kRounds], dk[kRounds];
#pragma unroll
        for (int r = 0; r < kRounds; ++r) {
            const int64_t i = r0 + int64_t(r) * kCT + tid;
            tl[r] = i < b1 ? a.tiles[i] : 0u;
            dk[r] = i < b1 ? a.dkey[i] : 0u;
        }
#pragma unroll
        for (int r = 0; r < kRounds; ++r) {
            if (tl[r] > 0u) {
                kmin = min(kmin, dk[r]);
                kmax = max(kmax, dk[r]);
                ++cnt;
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
        kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    }
    __syncthreads();
    if (lane == 0) {
        if (kmax >= kmin) {
            atomicMin(&s_u[0], kmin);
            atomicMax(&s_u[1], kmax);
        }
        s_wc[warp] = cnt;
    }
    __syncthreads();
    if (tid == 0) {
        uint32_t c = 0;
        for (int w = 0; w < kCW; ++w) c += s_wc[w];
        a.cta_cnt[k] = c;
        if (c) {
            atomicMax(&misc->kmin_inv, ~s_u[0]);
            atomicMax(&misc->kmax, s_u[1]);
        }
    }
    grid_sync(&misc->coop_bar, goal);

    // every CTA: its compaction base, V_s and the sort geometry
    if (warp == 0) {
        uint32_t pre = 0, all = 0;
        for (int j = lane; j < G; j += 32) {
            const uint32_t c = ldcg(a.cta_cnt + j);
            all += c;
            pre += j < k ? c : 0u;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            pre += __shfl_xor_sync(0xffffffffu, pre, o);
            all += __shfl_xor_sync(0xffffffffu, all, o);
        }
        if (lane == 0) {
            s_u[2] = pre;
            s_u[3] = all;
            s_u[4] = ~ldcg(&misc->kmin_inv);
            s_u[5] = ldcg(&misc->kmax);
        }
    }
    __syncthreads();
    const uint32_t base_k = s_u[2], Vs = s_u[3], key_lo = s_u[4], key_hi = s_u[5];
    const uint32_t range = Vs ? key_hi - key_lo : 0u;
    const int bits = range ? 32 - __clz(range) : 0;
    const int P = Vs == 0 ? 0 : (bits == 0 ? 1 : (bits + kDigitBits - 1) / kDigitBits);
    const int dbits = P ? (bits + P - 1) / P : 0;
    const uint32_t nbins = 1u << dbits, dmask = nbins - 1u;
    const uint32_t S2 = (Vs + G - 1) / G;

    // ---------------------------------------------------------------- C0 compaction: ordered writes
    // Per batch of kRounds x 1024 elements: ballots give each (round, warp) its count; one scan over
    // the kRounds x 32 counts, in element order, places every on-screen element.
    for (int i = tid; i < kCoopPasses * kCoopBins; i += kCT) (&s_hist[0][0])[i] = 0u;
    {
        uint32_t r_base = base_k;
        for (int64_t r0 = b0; r0 < b1; r0 += int64_t(kRounds) * kCT) {
            uint32_t tl[kRounds], dk[kRounds], bal[kRounds];
#pragma unroll
            for (int r = 0; r < kRounds; ++r) {
                const int64_t i = r0 + int64_t(r) * kCT + tid;
                tl[r] = i < b1 ? a.tiles[i] : 0u;
                dk[r] = i < b1 ? a.dkey[i] : 0u;
            }
#pragma unroll
            for (int r = 0; r < kRounds; ++r) {
                bal[r] = __ballot_sync(0xffffffffu, tl[r] > 0u);
                if (lane == 0) s_rw[r * kCW + warp] = __popc(bal[r]);
            }
            __syncthreads();
            const uint32_t v = tid < kRounds * kCW ? s_rw[tid] : 0u;
            uint32_t ex, agg;
            BScan(bscan).ExclusiveSum(v, ex, agg);
            if (tid < kRounds * kCW) s_rw[tid] = ex;
            __syncthreads();
#pragma unroll
            for (int r = 0; r < kRounds; ++r) {
                if (tl[r] > 0u) {
                    const uint32_t o = r_base + s_rw[r * kCW + warp] + __popc(bal[r] & ((1u << lane) - 1u));
                    const uint32_t i = uint32_t(r0 + int64_t(r) * kCT + tid);
                    const uint32_t key = dk[r] - key_lo;
                    a.onlist[o] = i;
                    a.rec_f[kRecFloats * size_t(i) + 11] = __uint_as_float(o);   // on-screen rank -> record r2.w
                    a.k0[o] = key;
                    a.v0[o] = i;
                    for (int p = 0; p < P; ++p) atomicAdd(&s_hist[p][(key >> (p * dbits)) & dmask], 1u);
                }
            }
            r_base += agg;
            __syncthreads();   // s_rw / bscan reuse
        }
    }
    __syncthreads();
    for (int d = tid; d < kCoopBins; d += kCT) a.H[size_t(k) * kCoopBins + d] = s_hist[0][d];   // pass-0 row
    for (int i = tid; i < P * kCoopBins; i += kCT) {
        const uint32_t c = (&s_hist[0][0])[i];
        if (c) atomicAdd(a.hist_all + i, c);
    }
    if (k == 0 && tid == 0) {
        misc->n_onscreen = Vs;
        misc->n_items = Vs;
    }
    grid_sync(&misc->coop_bar, goal);

    // ---------------------------------------------------------------- C1 depth sort passes
    uint32_t* wh = dyn;   // [kCW][kCoopBins] per-warp digit counts -> offsets (also prefix partials)
    for (int p = 0; p < P; ++p) {
        const uint32_t* kin = (p & 1) ? a.k1 : a.k0;
        const uint32_t* vin = (p & 1) ? a.v1 : a.v0;
        uint32_t* kout = (p & 1) ? a.k0 : a.k1;
        uint32_t* vout = (p & 1) ? a.v0 : a.v1;
        const bool last = p == P - 1;
        const int shift = p * dbits;
        const uint32_t s0 = p == 0 ? base_k : min(Vs, uint32_t(k) * S2);
        const uint32_t s1 = p == 0 ? base_k + ldcg(a.cta_cnt + k) : min(Vs, s0 + S2);
        // global start of each digit for this CTA: digit base (scan of the pass totals) + the
        // preceding CTAs' counts. Thread (4-bin column c4, row set rs) sums rows k' = rs, rs + 8, ...
        // < k with 16-B loads (rows are zero beyond nbins); CTAs in the second half sum the rows
        // k' >= k instead (preceding = total - following). (Keeping per-group row sums to shorten
        // this walk was measured slower: the extra scatter atomics contend.)
        const uint32_t* Hp = a.H + size_t(p) * kCoopGridMax * kCoopBins;
        {
            const int c4 = tid & (kCoopBins / 4 - 1), rs = tid / (kCoopBins / 4);   // 128 x 8
            uint4 acc = make_uint4(0u, 0u, 0u, 0u);
            // the second half of the CTAs sums the rows AFTER theirs and subtracts from the digit
            // total, so no CTA walks more than half of the rows (the walk is the pass' critical path)
            const bool suffix = 2 * k >= G;
            const int klo = suffix ? k : 0, khi = suffix ? G : k;
#pragma unroll 4
            for (int kk = klo + rs; kk < khi; kk += kCT / (kCoopBins / 4)) {
                const uint4 v = __ldcg(reinterpret_cast<const uint4*>(Hp + size_t(kk) * kCoopBins) + c4);
                acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
            }
            reinterpret_cast<uint4*>(wh + rs * kCoopBins)[c4] = acc;
            __syncthreads();
            uint32_t tot = 0, pre = 0;
            if (uint32_t(tid) < nbins) {
#pragma unroll
                for (int q = 0; q < kCT / (kCoopBins / 4); ++q) pre += wh[q * kCoopBins + tid];
                tot = ldcg(a.hist_all + p * kCoopBins + tid);
                if (suffix) pre = tot - pre;
            }
            uint32_t dbase;
            BScan(bscan).ExclusiveSum(tot, dbase);
            if (uint32_t(tid) < nbins) {
                s_gpos[tid] = dbase + pre;
                s_run[tid] = 0u;
            }
            __syncthreads();
        }
        // per-warp digit counts wh[warp][digit] are zero between rounds: the scan below rewrites only
        // the non-zero entries and each warp's leader lanes clear their own entries after the
        // scatter, so a round needs no clearing pass and two block barriers
        for (int i = tid; i < (kCW << dbits); i += kCT) wh[(i >> dbits) * kCoopBins + (i & int(dmask))] = 0u;
        __syncthreads();
        for (uint32_t r0 = s0; r0 < s1; r0 += kCT) {
            const uint32_t idx = r0 + tid;
            const bool ok = idx < s1;
            const uint32_t key = ok ? ldcg(kin + idx) : 0u;
            const uint32_t val = ok ? ldcg(vin + idx) : 0u;
            const uint32_t dg = ok ? (key >> shift) & dmask : nbins;   // nbins: sentinel digit
            const uint32_t peers = __match_any_sync(0xffffffffu, dg);
            const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
            const bool leader = ok && lane == __ffs(peers) - 1;
            if (leader) wh[warp * kCoopBins + dg] = __popc(peers);
            __syncthreads();   // [R] counts complete (and the previous round's scatter done)
            for (uint32_t d = tid; d < nbins; d += kCT) {   // per digit: exclusive over warps + running
                uint32_t c[kCW];
#pragma unroll
                for (int w = 0; w < kCW; ++w) c[w] = wh[w * kCoopBins + d];
                uint32_t run = s_run[d];
#pragma unroll
                for (int w = 0; w < kCW; ++w) {
                    if (c[w]) wh[w * kCoopBins + d] = run;
                    run += c[w];
                }
                s_run[d] = run;
            }
            __syncthreads();   // [S] offsets complete
            if (ok) {
                const uint32_t pos = s_gpos[dg] + wh[warp * kCoopBins + dg] + rank;
                if (last) {
                    a.svals[pos] = val;
                    a.srect[pos] = a.rect[val];
                } else {
                    kout[pos] = key;
                    vout[pos] = val;
                    const uint32_t dn = (key >> (shift + dbits)) & dmask;
                    atomicAdd(a.H + (size_t(p + 1) * kCoopGridMax + pos / S2) * kCoopBins + dn, 1u);
                }
            }
            __syncwarp();   // every lane of the warp has read its entry
            if (leader) wh[warp * kCoopBins + dg] = 0u;
            // the next round's [R] orders these clears and this round's reads before the next scan
        }
        grid_sync(&misc->coop_bar, goal);
    }

    // ---------------------------------------------------------------- C2 chunk counts
    const int nch = int((Vs + kChunk - 1) / kChunk);
    {
        const int GXp = a.GX + 1, cells = (a.GY + 1) * GXp;
        const int g = tid >> 8, lt = tid & 255, gw = lt >> 5;
        if (g < a.groups) {
            int* diff = reinterpret_cast<int*>(dyn) + g * cells;
            for (int c = k * a.groups + g; c < nch; c += G * a.groups) {
                for (int i = lt; i < cells; i += 256) diff[i] = 0;
                group_sync(g);
                const uint32_t s = uint32_t(c) * kChunk + lt;
                if (s < Vs) {
                    const short4 r = __ldcg(a.srect + s);
                    atomicAdd(&diff[r.z * GXp + r.x], 1);
                    atomicAdd(&diff[r.z * GXp + r.y], -1);
                    atomicAdd(&diff[r.w * GXp + r.x], -1);
                    atomicAdd(&diff[r.w * GXp + r.y], 1);
                }
                group_sync(g);
                for (int y = gw; y < a.GY; y += 8) {   // prefix along x: one warp per row
                    int carry = 0;
                    for (int x0 = 0; x0 < a.GX; x0 += 32) {
                        const int x = x0 + lane;
                        int v = x < a.GX ? diff[y * GXp + x] : 0;
#pragma unroll
                        for (int o = 1; o < 32; o <<= 1) {
                            const int u = __shfl_up_sync(0xffffffffu, v, o);
                            if (lane >= o) v += u;
                        }
                        v += carry;
                        if (x < a.GX) diff[y * GXp + x] = v;
                        carry = __shfl_sync(0xffffffffu, v, 31);
                    }
                }
                group_sync(g);
                uint32_t* row = a.cmat + size_t(c) * T;
                for (int x = lt; x < a.GX; x += 256) {   // prefix along y, write counts
                    int run = 0;
                    for (int y = 0; y < a.GY; ++y) {
                        run += diff[y * GXp + x];
                        row[y * a.GX + x] = uint32_t(run);
                    }
                }
                group_sync(g);
            }
        }
    }
    grid_sync(&misc->coop_bar, goal);

    // ---------------------------------------------------------------- C3 segment sums, tile totals
    // CTA = group of 32 tiles (lanes), warp = chunk segment: the segment prefix over the 32 segments
    // and the tile totals are formed in shared memory (no atomics, no deep load chains later)
    const int ntg = (T + 31) / 32;
    uint32_t* ssum = dyn;   // [kCW][32]
    for (int tg = k; tg < ntg; tg += G) {
        const int t = tg * 32 + lane;
        int c0, c1;
        seg_range(nch, warp, c0, c1);
        uint32_t sum = 0;
        if (t < T) {
#pragma unroll 8
            for (int c = c0; c < c1; ++c) sum += ldcg(a.cmat + size_t(c) * T + t);
        }
        ssum[warp * 32 + lane] = sum;
        __syncthreads();
        uint32_t pre = 0;
        for (int q = 0; q < warp; ++q) pre += ssum[q * 32 + lane];
        if (t < T) {
            a.segsum[size_t(warp) * T + t] = pre;   // exclusive prefix over the tile's segments
            if (warp == kCW - 1) a.tot[t] = pre + sum;
        }
        __syncthreads();
    }
    grid_sync(&misc->coop_bar, goal);

    // ---------------------------------------------------------------- C4 tile starts and chunk bases
    for (int tg = k; tg < ntg; tg += G) {
        // start of the group: sum of the totals of all earlier tiles
        uint32_t part = 0;
        for (int t = tid; t < tg * 32; t += kCT) part += ldcg(a.tot + t);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        if (lane == 0) dyn[warp] = part;
        __syncthreads();
        if (warp == 0) {
            uint32_t base = 0;
            for (int q = 0; q < kCW; ++q) base += dyn[q];
            const int t = tg * 32 + lane;
            const uint32_t v = t < T ? ldcg(a.tot + t) : 0u;
            uint32_t incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += u;
            }
            const uint32_t st = base + incl - v;
            dyn[kCW + lane] = st;
            if (t < T) a.ranges[t] = v ? make_uint2(st, st + v) : make_uint2(0u, 0u);
            if (tg == ntg - 1 && lane == 31) {   // the last group knows K
                const unsigned long long K = (unsigned long long)(base + incl);
                misc->n_keys = K;
                const bool over = K > (unsigned long long)a.key_cap;
                misc->n_keys_eff = over ? 0ull : K;
                if (over) atomicOr(&misc->error_flag, 1u);
            }
        }
        __syncthreads();
        const int t = tg * 32 + lane;
        int c0, c1;
        seg_range(nch, warp, c0, c1);
        if (t < T && c1 > c0) {
            uint32_t run = dyn[kCW + lane] + ldcg(a.segsum + size_t(warp) * T + t);
            for (int cb = c0; cb < c1; cb += 8) {   // 8 loads in flight, then 8 stores
                uint32_t v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = (cb + u < c1) ? ldcg(a.cmat + size_t(cb + u) * T + t) : 0u;
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    if (cb + u < c1) a.cmat[size_t(cb + u) * T + t] = run;
                    run += v[u];
                }
            }
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ host driver
struct CoopGeom {
    int grid = 0;
    size_t smem = 0;
    int groups = 0;
};

gs_status run_bin_coop(WsState* s, cudaStream_t st) {
    Misc* misc = at<Misc>(s, s->misc);
    const int GX = s->cam_gx, GY = s->cam_gy, T = GX * GY;
    const size_t cells = size_t(GX + 1) * (GY + 1) * sizeof(int);
    constexpr size_t kSmemMax = 200 * 1024;
    CoopGeom g;
    g.groups = int(std::min<size_t>(kCGroups, kSmemMax / std::max<size_t>(cells, 1)));
    if (g.groups < 1 || size_t(T) * 4 > kSmemMax) return GS_ERR_UNSUPPORTED;   // tile grid too large
    g.smem = std::max({size_t(kCW) * kCoopBins * 4, size_t(g.groups) * cells, size_t(T) * 4});
    static PerDeviceOnce attr;
    if (!attr.run([] {
            return cudaFuncSetAttribute(bin_coop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemMax)) ==
                   cudaSuccess;
        }))
        return check_launch(s, "bin_coop attribute");
    const int sms = coop_sm_count();
    if (sms <= 0) return check_launch(s, "bin_coop sm count");
    g.grid = std::min(sms, kCoopGridMax);
    CoopArgs a;
    a.tiles = at<uint32_t>(s, s->tiles);
    a.dkey = at<uint32_t>(s, s->depth_key);
    a.rect = at<short4>(s, s->rect);
    a.n = s->n;
    a.GX = GX;
    a.GY = GY;
    a.key_cap = s->key_cap;
    a.onlist = at<uint32_t>(s, s->onlist);
    a.rec_f = at<float>(s, s->rec);
    a.k0 = at<uint32_t>(s, s->dkey_sorted);
    a.k1 = a.k0 + s->n_cap;
    a.v0 = at<uint32_t>(s, s->dval_sorted);
    a.v1 = a.v0 + s->n_cap;
    a.svals = at<uint32_t>(s, s->svals);
    a.srect = at<short4>(s, s->srect);
    a.cmat = at<uint32_t>(s, s->chunk_mat);
    uint32_t* c = at<uint32_t>(s, s->coop);
    a.H = c;
    a.hist_all = a.H + size_t(kCoopPasses) * kCoopGridMax * kCoopBins;
    a.cta_cnt = a.hist_all + kCoopPasses * kCoopBins;
    a.tot = a.cta_cnt + kCoopGridMax;
    a.segsum = a.tot + size_t(s->GX) * s->GY;   // capacity tile grid (region layout)


    a.ranges = at<uint2>(s, s->ranges);
    a.misc = misc;
    a.groups = g.groups;
    void* args[] = {&a};
    KTimer kt(s, KID_BIN_COOP, st);
    const cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(bin_coop_kernel), dim3(g.grid),
                                                      dim3(kCT), args, g.smem, st);
    if (e != cudaSuccess) {
        set_cuda_error(e, "bin_coop_kernel");
        return GS_ERR_CUDA;
    }
    return GS_OK;
}

}  // namespace gs
