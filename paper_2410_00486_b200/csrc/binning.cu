// binning.cu -- K2-K4b: duplicate-with-keys, radix sort, tile ranges.
//
// Replaces build_tile_index (rasterizer/tiles.py:29-65), whose order is
// np.lexsort((splat, depth, tile)) (tiles.py:58): pairs sorted by tile,
// then camera depth, then splat index.  That order equals a STABLE sort of
// 64-bit keys tile<<32 | float_bits(depth) over pairs emitted in splat
// order (depth > near > 0, so the float bits are monotone).  An LSD radix
// sort of those keys processes the 32 depth bits first; because the depth
// half of a pair's key is a function of its splat alone, those passes are
// run here over the N splats instead of the P ~ 12 N pairs:
//
//   1. LSD sort of the N depth keys (8-bit passes), stable, values = splat
//      index                                    -> splats in (depth, index) order
//   2. default (bin_front_kernel + fe_direct): every pair is written
//      straight to its final slot, start[tile] + (pairs of that tile earlier
//      in depth order), counted per (CTA, placer warp) and prefixed across
//      them; tile ranges come out of the same scan.
//      fallback (SS_BIN_DIRECT=0, > 8192 tiles, or the per-pass path):
//      exclusive scan of touched-tile counts, coalesced emission of
//      (tile, splat) pairs in depth order, LSD sort of the pair tile ids
//      (ceil(log2 T / 8) passes), tile ranges by boundary detection;
//   3. checkpoint slot bases by scan.
//
// The result is bit-identical to the reference order (tests/test_gpu_parity.py
// compares it with the oracle's build_tile_index fed this projection, and
// the default path with both fallbacks).
//
// Each radix pass is reduce-then-scan (upsweep counts, per-digit scan,
// downsweep with warp ballot ranking and a shared-memory reorder so the
// scatter writes coalesced runs).  A one-sweep pass with decoupled look-back
// was measured first and was latency-bound here: with hundreds of CTAs
// co-resident, each CTA walks back over all its predecessors' aggregates.
#include <cooperative_groups.h>
#include <cstdlib>

#include "common.cuh"

namespace ss {

__device__ __forceinline__ unsigned long long ld_volatile64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_volatile64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Decoupled look-back (used by the scans), executed by one full warp: lane
// l reads the status word of predecessor j - l, so each round covers 32
// predecessors with independent loads.  The nearest-first run of published
// words is consumed up to (and including) the first inclusive prefix; when
// an unpublished word interrupts the run, the published part is added and
// the walk resumes from there.  Returns the exclusive prefix (all lanes).
__device__ __forceinline__ unsigned long long lookback_warp(const unsigned long long* status,
                                                            int64_t j,
                                                            unsigned long long flag_inc,
                                                            unsigned long long mask) {
    const int l = threadIdx.x & 31;
    unsigned long long excl = 0;
    while (j >= 0) {
        const unsigned long long v = (j - l >= 0) ? ld_volatile64(status + (j - l)) : flag_inc;
        const unsigned long long f = v & ~mask;
        const unsigned not_ready = __ballot_sync(0xffffffffu, f == 0);
        const unsigned inc = __ballot_sync(0xffffffffu, f == flag_inc);
        const int limit = not_ready ? __ffs(not_ready) - 1 : 32;  // lanes [0, limit) published
        const int first_inc = inc ? __ffs(inc) - 1 : 32;
        const bool done = first_inc < limit;
        const int take = done ? first_inc + 1 : limit;
        unsigned long long part = l < take ? (v & mask) : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        excl += part;
        if (done) break;
        j -= take;
        if (take < 32) __nanosleep(32);
    }
    return excl;
}

// Lanes holding the same 8-bit digit (warp multi-split by 8 ballots; the
// ballots are independent, unlike the serialised MATCH.ANY).  Invalid lanes
// (valid == false) get an empty mask and are excluded from everyone's mask.
template <int BITS = 8>
__device__ __forceinline__ unsigned peers8(uint32_t d, bool valid) {
    unsigned peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
    for (int b = 0; b < BITS; ++b) {
        const bool bit = (d >> b) & 1u;
        const unsigned bal = __ballot_sync(0xffffffffu, bit);
        peers &= bit ? bal : ~bal;
    }
    return valid ? peers : 0u;
}

// Block-wide exclusive scan of one value per thread (256 threads).
__device__ __forceinline__ uint32_t block_excl_scan256(uint32_t v, uint32_t* s_warp) {
    const int t = threadIdx.x, w = t >> 5, l = t & 31;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (l >= o) incl += y;
    }
    if (l == 31) s_warp[w] = incl;
    __syncthreads();
    uint32_t pre = 0;
    for (int k = 0; k < w; ++k) pre += s_warp[k];
    __syncthreads();
    return pre + incl - v;
}

// ------------------------------------------------------- reduce-then-scan
// Chain-free LSD pass in three launches (the one-sweep look-back above is
// latency-bound when hundreds of CTAs are co-resident: every CTA walks back
// over all its predecessors' aggregates):
//   rs_upsweep   : per-block digit counts -> counts[digit][block]
//   rs_scan      : one CTA per digit, exclusive scan over blocks (in place)
//                  and the digit total
//   rs_downsweep : digit starts from the 256 totals, stable warp ranking,
//                  block-local reorder, coalesced scatter
template <int ITEMS>
__global__ void __launch_bounds__(256) rs_upsweep_kernel(const uint32_t* __restrict__ keys,
                                                         const uint32_t* d_count,
                                                         uint32_t n_static, uint32_t cap,
                                                         int shift, uint32_t nblk,
                                                         uint32_t* __restrict__ counts) {
    constexpr int TILE = 256 * ITEMS;
    __shared__ uint32_t h[8][256];
    const int t = threadIdx.x, w = t >> 5;
#pragma unroll
    for (int k = 0; k < 8; ++k) h[k][t] = 0;
    __syncthreads();
    const uint32_t n = d_count ? min(*d_count, cap) : n_static;
    const uint32_t base = blockIdx.x * TILE;
    uint32_t k[ITEMS];  // all loads in flight before the shared-memory atomics
#pragma unroll
    for (int r = 0; r < ITEMS; ++r) {
        const uint32_t i = base + r * 256 + t;
        k[r] = i < n ? keys[i] : 0xffffffffu;
    }
#pragma unroll
    for (int r = 0; r < ITEMS; ++r)
        if (base + r * 256 + t < n) atomicAdd(&h[w][(k[r] >> shift) & 255u], 1u);
    __syncthreads();
    uint32_t c = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) c += h[k][t];
    counts[(size_t)t * nblk + blockIdx.x] = c;
}

__global__ void __launch_bounds__(256) rs_scan_kernel(uint32_t nblk, uint32_t* __restrict__ counts,
                                                      uint32_t* __restrict__ totals) {
    __shared__ uint32_t s_warp[8];
    uint32_t* row = counts + (size_t)blockIdx.x * nblk;
    const int t = threadIdx.x;
    uint32_t carry = 0;
    for (uint32_t b0 = 0; b0 < nblk; b0 += 256 * 4) {
        uint32_t v[4], sum = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t i = b0 + t * 4 + k;
            v[k] = i < nblk ? row[i] : 0u;
            sum += v[k];
        }
        const uint32_t ex = block_excl_scan256(sum, s_warp);
        __shared__ uint32_t s_tot;
        if (t == 255) s_tot = ex + sum;
        uint32_t run = carry + ex;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t i = b0 + t * 4 + k;
            if (i < nblk) row[i] = run;
            run += v[k];
        }
        __syncthreads();
        carry += s_tot;
        __syncthreads();
    }
    if (t == 0) totals[blockIdx.x] = carry;
}

template <int ITEMS, bool KEYS_ONLY, int BITS>
__global__ void __launch_bounds__(256) rs_downsweep_kernel(
    const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
    uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out, const uint32_t* d_count,
    uint32_t n_static, uint32_t cap, int shift, uint32_t nblk,
    const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ totals) {
    constexpr int WARP_ITEMS = 32 * ITEMS;
    constexpr int TILE = 256 * ITEMS;
    __shared__ uint32_t s_cnt[8][256];
    __shared__ uint32_t s_base[256];
    __shared__ uint32_t s_local[256];
    __shared__ uint32_t s_warp[8];
    __shared__ uint32_t s_keys[TILE];
    __shared__ uint32_t s_vals[KEYS_ONLY ? 1 : TILE];
    const int t = threadIdx.x, w = t >> 5, l = t & 31;
#pragma unroll
    for (int k = 0; k < 8; ++k) s_cnt[k][t] = 0;
    const uint32_t n = d_count ? min(*d_count, cap) : n_static;
    const uint32_t base = blockIdx.x * TILE;
    if (base >= n) return;  // uniform per block
    const uint32_t nloc = min((uint32_t)TILE, n - base);
    const uint32_t gstart = block_excl_scan256(totals[t], s_warp);  // also syncs s_cnt
    s_base[t] = gstart + offsets[(size_t)t * nblk + blockIdx.x];
    uint32_t key[ITEMS], val[ITEMS], rank[ITEMS];
    const uint32_t wbase = w * WARP_ITEMS;
#pragma unroll
    for (int r = 0; r < ITEMS; ++r) {
        const uint32_t li = wbase + r * 32 + l;
        key[r] = li < nloc ? keys_in[base + li] : 0u;
        if (!KEYS_ONLY) val[r] = li < nloc ? (vals_in ? vals_in[base + li] : base + li) : 0u;
    }
#pragma unroll
    for (int r = 0; r < ITEMS; ++r) {
        const uint32_t li = wbase + r * 32 + l;
        const bool valid = li < nloc;
        const uint32_t d = (key[r] >> shift) & 255u;
        const unsigned peers = peers8<BITS>(d, valid);
        const uint32_t before = valid ? s_cnt[w][d] : 0u;
        rank[r] = before + __popc(peers & lanemask_lt());
        __syncwarp();
        if (valid && (peers & lanemask_lt()) == 0) s_cnt[w][d] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    uint32_t run = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint32_t c = s_cnt[k][t];
        s_cnt[k][t] = run;
        run += c;
    }
    s_local[t] = block_excl_scan256(run, s_warp);
    __syncthreads();
#pragma unroll
    for (int r = 0; r < ITEMS; ++r) {
        const uint32_t li = wbase + r * 32 + l;
        if (li < nloc) {
            const uint32_t d = (key[r] >> shift) & 255u;
            const uint32_t lp = s_local[d] + s_cnt[w][d] + rank[r];
            s_keys[lp] = key[r];
            if (!KEYS_ONLY) s_vals[lp] = val[r];
        }
    }
    __syncthreads();
    for (uint32_t i = t; i < nloc; i += 256) {
        const uint32_t k = s_keys[i];
        const uint32_t d = (k >> shift) & 255u;
        const uint32_t gp = s_base[d] + (i - s_local[d]);
        if (!KEYS_ONLY) vals_out[gp] = s_vals[i];
        if (keys_out) keys_out[gp] = k;
    }
}

// One reduce-then-scan pass (3 launches).
template <int ITEMS>
static void rs_pass(const uint32_t* kin, const uint32_t* vin, uint32_t* kout, uint32_t* vout,
                    const uint32_t* d_count, uint32_t n_static, uint32_t cap, int shift,
                    uint32_t* counts, uint32_t* totals, cudaStream_t s, int bits = 8) {
    const uint32_t nblk = (uint32_t)div_up(cap > 0 ? cap : 1, 256 * ITEMS);
    rs_upsweep_kernel<ITEMS><<<nblk, 256, 0, s>>>(kin, d_count, n_static, cap, shift, nblk, counts);
    rs_scan_kernel<<<256, 256, 0, s>>>(nblk, counts, totals);
    // digits narrower than 8 bits (a last partial pass) rank with fewer ballots
    if (vout)
        rs_downsweep_kernel<ITEMS, false, 8><<<nblk, 256, 0, s>>>(kin, vin, kout, vout, d_count,
                                                                  n_static, cap, shift, nblk,
                                                                  counts, totals);
    else if (bits <= 4)
        rs_downsweep_kernel<ITEMS, true, 4><<<nblk, 256, 0, s>>>(kin, nullptr, kout, nullptr,
                                                                 d_count, n_static, cap, shift,
                                                                 nblk, counts, totals);
    else
        rs_downsweep_kernel<ITEMS, true, 8><<<nblk, 256, 0, s>>>(kin, nullptr, kout, nullptr,
                                                                 d_count, n_static, cap, shift,
                                                                 nblk, counts, totals);
}

// ------------------------------------------------------------------ scan
// Exclusive scan of in[gather ? gather[i] : i] (u32), 64-bit look-back
// words (2 flag bits + 62-bit sum).  total_out (u64, optional) and
// optional capacity check writing the overflow flag.
constexpr int kScanItems = 16;
constexpr int kScanItemsTiles = 4;  // checkpoint-base scan (few thousand tiles)
constexpr unsigned long long kSFlagAgg = 1ull << 62;
constexpr unsigned long long kSFlagInc = 2ull << 62;
constexpr unsigned long long kSValMask = (1ull << 62) - 1;

template <bool CEIL_DIV32>
__global__ void __launch_bounds__(256) scan_kernel(const uint32_t* __restrict__ in,
                                                   const uint32_t* __restrict__ gather,
                                                   const uint32_t* __restrict__ in_end, uint32_t n,
                                                   uint32_t* __restrict__ out,
                                                   unsigned long long* status, uint32_t* counter,
                                                   int64_t* total_out, int64_t* overflow_out,
                                                   int64_t capacity) {
    constexpr int ITEMS = CEIL_DIV32 ? kScanItemsTiles : kScanItems;
    constexpr int TILE = 256 * ITEMS;
    __shared__ uint32_t s_bid;
    __shared__ unsigned long long s_warp[8], s_wpre[8];
    __shared__ unsigned long long s_excl;
    const int t = threadIdx.x, w = t >> 5, l = t & 31;
    if (t == 0) s_bid = atomicAdd(counter, 1u);
    __syncthreads();
    const uint32_t bid = s_bid;
    const uint32_t base = bid * TILE + t * ITEMS;
    uint32_t v[ITEMS];
    unsigned long long sum = 0;
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        uint32_t i = base + k;
        uint32_t x = 0;
        if (i < n) {
            uint32_t src = gather ? gather[i] : i;
            if (CEIL_DIV32)
                x = (i + 1 < n) ? (in_end[src] - in[src] + 31u) >> 5 : 0u;
            else
                x = in[src];
        }
        v[k] = x;
        sum += x;
    }
    unsigned long long incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
        if (l >= o) incl += y;
    }
    if (l == 31) s_warp[w] = incl;
    __syncthreads();
    if (w == 0) {
        unsigned long long tot = 0;
        for (int k = 0; k < 8; ++k) tot += s_warp[k];
        unsigned long long* my = status + bid;
        unsigned long long excl = 0;
        if (bid == 0) {
            if (l == 0) st_volatile64(my, kSFlagInc | tot);
        } else {
            if (l == 0) st_volatile64(my, kSFlagAgg | tot);
            excl = lookback_warp(status, (int64_t)bid - 1, kSFlagInc, kSValMask);
            if (l == 0) st_volatile64(my, kSFlagInc | (excl + tot));
        }
        if (l == 0) {
            s_excl = excl;
            if ((bid + 1) * (uint32_t)TILE >= n) {  // last block writes the total
                if (total_out) *total_out = (int64_t)(excl + tot);
                if (overflow_out && (int64_t)(excl + tot) > capacity) *overflow_out = 1;  // sticky
            }
        }
        __syncwarp();
        if (l < 8) {  // warp offsets within the block
            unsigned long long pre = 0;
            for (int k = 0; k < l; ++k) pre += s_warp[k];
            s_wpre[l] = pre;
        }
    }
    __syncthreads();
    unsigned long long run = s_excl + s_wpre[w] + incl - sum;
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        uint32_t i = base + k;
        if (i < n) out[i] = (uint32_t)run;
        run += v[k];
    }
}

// 1-CTA tile metadata (n_tiles <= SS_ORDER_MAX_TILES): the checkpoint slot
// bases -- exclusive scan of ceil(len/32) over n_tiles + 1 entries, as
// scan_kernel<true> -- and the forward's tile order for this call, costliest
// first by the previous forward's per-tile cost (64 linear buckets of
// cost / max cost; order within a bucket is arbitrary).  The forward's
// per-tile durations vary 70x and follow the previous iteration's closely;
// a raster-order grid leaves the longest tiles to start last.
constexpr int kOrderBuckets = 64;

__global__ void __launch_bounds__(1024) tile_meta_kernel(const uint32_t* __restrict__ tstart,
                                                         const uint32_t* __restrict__ tend,
                                                         int n_tiles,
                                                         uint32_t* __restrict__ ckpt_base,  // null: order only
                                                         const uint32_t* __restrict__ cost,
                                                         uint32_t* __restrict__ order) {
    __shared__ uint32_t s_warp[32];
    __shared__ uint32_t s_max;
    __shared__ uint32_t s_h[kOrderBuckets];
    const int t = threadIdx.x, w = t >> 5, l = t & 31;
    const int n = n_tiles + 1;
    const int per = (n + 1023) / 1024;  // <= 17
    const int i0 = t * per;
    uint32_t sum = 0, cmax = 0;
    for (int k = 0; k < per; ++k) {
        const int i = i0 + k;
        if (i < n_tiles) {
            if (ckpt_base) sum += (tend[i] - tstart[i] + 31u) >> 5;
            cmax = max(cmax, cost[i]);
        }
    }
    if (t < kOrderBuckets) s_h[t] = 0u;
    if (t == 0) s_max = 0u;
    // block exclusive scan of the per-thread sums
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (l >= o) incl += y;
    }
    if (l == 31) s_warp[w] = incl;
    cmax = __reduce_max_sync(0xffffffffu, cmax);
    __syncthreads();
    if (l == 0) atomicMax(&s_max, cmax);
    if (w == 0) {
        uint32_t v = s_warp[l], vi = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, vi, o);
            if (l >= o) vi += y;
        }
        s_warp[l] = vi - v;
    }
    __syncthreads();
    uint32_t run = s_warp[w] + incl - sum;
    if (ckpt_base)
        for (int k = 0; k < per; ++k) {
            const int i = i0 + k;
            if (i < n) ckpt_base[i] = run;
            if (i < n_tiles) run += (tend[i] - tstart[i] + 31u) >> 5;
        }
    // counting sort by cost bucket, descending
    const unsigned long long mx = (unsigned long long)s_max + 1ull;
    for (int i = t; i < n_tiles; i += 1024) {
        const uint32_t b = (uint32_t)(((unsigned long long)cost[i] * kOrderBuckets) / mx);
        atomicAdd(&s_h[kOrderBuckets - 1 - b], 1u);
    }
    __syncthreads();
    if (w == 0) {
        uint32_t a = s_h[l], b = s_h[l + 32], ai = a, bi = b;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t ya = __shfl_up_sync(0xffffffffu, ai, o);
            const uint32_t yb = __shfl_up_sync(0xffffffffu, bi, o);
            if (l >= o) ai += ya, bi += yb;
        }
        const uint32_t atot = __shfl_sync(0xffffffffu, ai, 31);
        s_h[l] = ai - a;
        s_h[l + 32] = atot + bi - b;
    }
    __syncthreads();
    for (int i = t; i < n_tiles; i += 1024) {
        const uint32_t b = (uint32_t)(((unsigned long long)cost[i] * kOrderBuckets) / mx);
        order[atomicAdd(&s_h[kOrderBuckets - 1 - b], 1u)] = (uint32_t)i;
    }
}

// ------------------------------------------------------------------- emit
// One warp per 32 consecutive splats in (depth, index) order: the warp's
// pairs form one contiguous output range, written lane-strided (coalesced);
// each output element finds its splat by a 5-step shuffle binary search
// over the 32 exclusive offsets.
__global__ void __launch_bounds__(256) emit_pairs_kernel(
    uint32_t n, const uint32_t* __restrict__ order, const uint32_t* __restrict__ tiles,
    const uint2* __restrict__ rect, const uint32_t* __restrict__ offsets, int tiles_x,
    const int64_t* total, int64_t cap, uint32_t* __restrict__ keys,
    uint32_t* __restrict__ vals, int sb) {
    const bool ok = *total <= cap;
    const int lane = threadIdx.x & 31;
    const uint32_t j = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32 + lane;
    uint32_t s = 0, c = 0, o = 0, x0 = 0, y0 = 0, wx = 1;
    if (ok && j < n) {
        s = order[j];
        c = tiles[s];
        o = offsets[j];
        if (c) {
            uint2 rc = rect[s];
            x0 = rc.x & 0xffffu;
            y0 = rc.x >> 16;
            wx = (rc.y & 0xffffu) - x0 + 1;
        }
    }
    const uint32_t base = __shfl_sync(0xffffffffu, o, 0);
    const uint32_t rel = (ok && j < n) ? o - base : 0x7fffffffu;
    uint32_t endw = (ok && j < n) ? rel + c : 0u;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) endw = max(endw, __shfl_xor_sync(0xffffffffu, endw, d));
    // warp-uniform trip count: every lane reaches every __shfl_sync
    for (uint32_t e0 = 0; e0 < endw; e0 += 32) {
        const uint32_t e = e0 + lane;
        // owner = largest lane with rel <= e (never an empty lane for e < endw)
        int lo = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
            uint32_t r = __shfl_sync(0xffffffffu, rel, lo + step);
            if (r <= e) lo += step;
        }
        const uint32_t li = e - __shfl_sync(0xffffffffu, rel, lo);
        const uint32_t ox = __shfl_sync(0xffffffffu, x0, lo), oy = __shfl_sync(0xffffffffu, y0, lo);
        const uint32_t ow = __shfl_sync(0xffffffffu, wx, lo), sid = __shfl_sync(0xffffffffu, s, lo);
        if (e < endw) {
            const uint32_t ry = li / ow;
            const uint32_t tid = (oy + ry) * tiles_x + ox + (li - ry * ow);
            if (vals) {
                keys[base + e] = tid;
                vals[base + e] = sid;
            } else {
                keys[base + e] = (tid << sb) | sid;  // packed (tile, splat)
            }
        }
    }
}

// ----------------------------------------------------------------- ranges
// Tile ranges by boundary detection on the sorted keys, 4 keys per thread
// (16-byte loads).  Packed keys (sb > 0) hold tile << sb | splat: the splat
// ids are unpacked into the pair list in the same pass.
__global__ void __launch_bounds__(256) tile_ranges_kernel(const uint32_t* __restrict__ keys,
                                                          const int64_t* total, int64_t cap,
                                                          int sb, uint32_t* __restrict__ start,
                                                          uint32_t* __restrict__ end,
                                                          uint32_t* __restrict__ splat_out) {
    int64_t P = *total;
    if (P > cap) P = 0;
    const uint32_t smask = sb ? (1u << sb) - 1u : 0u;
    for (int64_t i0 = 4 * (blockIdx.x * (int64_t)blockDim.x + threadIdx.x); i0 < P;
         i0 += 4 * (int64_t)gridDim.x * blockDim.x) {
        uint32_t k[6];
        if (i0 + 4 <= P) {
            const uint4 v = *reinterpret_cast<const uint4*>(keys + i0);
            k[1] = v.x, k[2] = v.y, k[3] = v.z, k[4] = v.w;
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) k[1 + j] = (i0 + j < P) ? keys[i0 + j] : 0u;
        }
        k[0] = i0 > 0 ? keys[i0 - 1] : 0u;
        k[5] = i0 + 4 < P ? keys[i0 + 4] : 0u;
        uint32_t tl[6];
#pragma unroll
        for (int j = 0; j < 6; ++j) tl[j] = sb ? k[j] >> sb : k[j];
#pragma unroll
        for (int j = 1; j <= 4; ++j) {
            const int64_t i = i0 + j - 1;
            if (i >= P) break;
            if (i == 0 || tl[j - 1] != tl[j]) start[tl[j]] = (uint32_t)i;
            if (i == P - 1 || tl[j + 1] != tl[j]) end[tl[j]] = (uint32_t)(i + 1);
        }
        if (sb) {
            if (i0 + 4 <= P) {
                *reinterpret_cast<uint4*>(splat_out + i0) =
                    make_uint4(k[1] & smask, k[2] & smask, k[3] & smask, k[4] & smask);
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (i0 + j < P) splat_out[i0 + j] = k[1 + j] & smask;
            }
        }
    }
}

__global__ void bin_clear_kernel(uint32_t* ctrl, uint32_t ctrl_words, uint32_t* start,
                                 uint32_t* end, uint32_t n_tiles) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    for (uint32_t k = i; k < ctrl_words; k += gridDim.x * blockDim.x) ctrl[k] = 0u;
    for (uint32_t k = i; k < n_tiles; k += gridDim.x * blockDim.x) {
        start[k] = 0u;
        end[k] = 0u;
    }
}

// Copy a device int64 (clamped) into a u32 count for the pair passes.
__global__ void clamp_count_kernel(const int64_t* total, int64_t cap, uint32_t* out) {
    int64_t P = *total;
    *out = (P > cap) ? 0u : (uint32_t)P;
}

// ------------------------------------------------- persistent front end
// Depth sort + pair offsets + pair emission in ONE cooperative launch (the
// per-pass kernels above are latency-bound at N = 300k: 12 launches of
// 147 CTAs, then a look-back scan and the emission).  One sort tile of
// kFeTile keys per CTA; no atomics (deterministic); nine grid barriers:
//   pass p, phase A  load the tile (from the previous pass's output),
//                    stable warp multi-split ranking, publish the tile's
//                    digit histogram                                 -> sync
//   pass p, phase B  digit totals and the column prefix over preceding
//                    tiles from the published histograms (4 thread groups
//                    x 256 digits), local reorder, coalesced scatter -> sync
//   chunk sums       each CTA sums the touched-tile counts of its tile of
//                    the final order                                 -> sync
//   emission         tile prefix, block scan -> pair offsets, P, capacity
//                    check, warp-cooperative emission (as emit_pairs).
constexpr int kFeThreads = 1024;
constexpr int kFeWarps = kFeThreads / 32;
constexpr int kFeColChunks = 5;  // column walk covers n_tiles <= 160 (one CTA per SM)
// keys per thread: 2, 4 or 8 (2048 / 4096 / 8192-key tiles), the smallest
// that gives every co-resident CTA at most one tile
template <int ITEMS>
constexpr size_t fe_smem_bytes() {
    return sizeof(uint32_t) * (kFeWarps * 256 + 2 * kFeThreads * ITEMS + 4 * 512);
}
inline size_t fe_smem_bytes_rt(int items) {
    return sizeof(uint32_t) * (kFeWarps * 256 + 2 * kFeThreads * items + 4 * 512);
}

struct FeArgs {
    uint32_t n;
    uint32_t n_tiles;
    const uint32_t* key_in;
    uint32_t *kA, *vA, *kB, *vB;
    uint32_t* counts;      // [2][n_tiles][256] (pass parity)
    uint32_t* chunk_sum;   // [n_tiles]
    const uint32_t* tiles;
    const uint2* rect;
    int tiles_x;
    uint32_t* pair_k;
    uint32_t* pair_v;      // null: packed words
    int sb;
    int64_t* total;
    int64_t* overflow;
    int64_t cap;
    uint32_t* pcount;
    // direct tile emission (fe_direct); direct == 0 -> depth-order emission
    int direct;
    uint32_t n_img_tiles;
    uint32_t* col;         // [n_img_tiles][gridDim.x] per-CTA tile counts -> column prefixes
    uint32_t* col_tot;     // [n_img_tiles] tile totals
    uint32_t* out_splat;   // pair list (Gaussian ids) in (tile, depth, id) order
    uint32_t* tile_start;
    uint32_t* tile_end;
    uint4* drec;           // [n] depth-order splat records (fe_direct)
    uint32_t* keyred;      // [2 n_tiles] per-CTA AND / OR of the keys with pairs
    uint32_t* ckpt_base;   // [n_img_tiles + 1] checkpoint slot bases (written by CTA 0)
};

template <int NT>
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* s_warp) {
    const int t = threadIdx.x, w = t >> 5, l = t & 31;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (l >= o) incl += y;
    }
    if (l == 31) s_warp[w] = incl;
    __syncthreads();
    if (w == 0) {
        const uint32_t x = l < NT / 32 ? s_warp[l] : 0u;
        uint32_t xi = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, xi, o);
            if (l >= o) xi += y;
        }
        if (l < NT / 32) s_warp[l] = xi - x;
    }
    __syncthreads();
    const uint32_t r = s_warp[w] + incl - v;
    __syncthreads();
    return r;
}


#ifdef SS_FE_TRACE
// diagnostics build only (tools/trace_front.py): per CTA, globaltimer stamps
// at the phase boundaries of bin_front_kernel
constexpr int kFeTraceSlots = 40;
__device__ unsigned long long g_fe_trace[160 * kFeTraceSlots];
__device__ __forceinline__ void fe_stamp(int slot) {
    if (threadIdx.x == 0 && slot < kFeTraceSlots) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_fe_trace[blockIdx.x * kFeTraceSlots + slot] = t;
    }
}
#define FE_STAMP(k) fe_stamp(k)
#else
#define FE_STAMP(k)
#endif

// ------------------------------------------------- direct tile emission
// After the depth sort every pair goes straight to its final slot in
// (tile, depth, id) order -- no emission in depth order followed by radix
// passes over all P pairs:
//   slot = start[tile] + (pairs of that tile earlier in depth order).
// The P pairs, in depth order, are split evenly over the CTAs (pair-balanced:
// near splats cover many more tiles than far ones), and each CTA's range over
// G "placer" warps.  A placer warp walks its contiguous range 32 pairs per
// step and ranks each pair among the step's pairs of the same tile with a
// ballot multi-split; a per-(warp, tile) counter in shared memory carries the
// running count, so the order inside the warp's range is exactly the depth
// order.  Pass 1 counts; per-tile totals per CTA -> grid barrier -> prefix
// over the CTAs per tile -> grid barrier -> tile starts (every CTA scans the
// totals) -> pass 2 repeats the walk with the counters preset to each warp's
// first slot per tile and writes the Gaussian ids.  Deterministic, atomic-
// free.
constexpr int kDirMaxTiles = 8192;  // image tiles handled by the direct path
constexpr int kDirSmemBytes = 200 * 1024;
constexpr uint32_t kDirPiece = 65535;  // pairs per piece (16-bit counters)
// placer warps: 16-bit counters per (warp, tile) + a 32-bit base per tile
__host__ __device__ inline int fe_direct_warps(int n_img_tiles) {
    const int nt = n_img_tiles > 0 ? n_img_tiles : 1;
    const int g = (kDirSmemBytes - 4 * nt) / (2 * (nt + 1));
    return g > 32 ? 32 : g;
}
inline size_t fe_direct_smem_bytes(int n_img_tiles) {
    const size_t g = (size_t)fe_direct_warps(n_img_tiles);
    return 2 * g * (size_t)((n_img_tiles + 1) & ~1) + 4 * (size_t)n_img_tiles;
}

// Block-wide exclusive scan of s[0..n) in place (n <= 8 * kFeThreads);
// returns the total.
__device__ __forceinline__ uint32_t fe_scan_smem(uint32_t* s, uint32_t n, uint32_t* s_warp) {
    const int t = threadIdx.x;
    const uint32_t per = (n + kFeThreads - 1) / kFeThreads;
    const uint32_t q0 = t * per;
    uint32_t v[8], sum = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        v[k] = (k < (int)per && q0 + k < n) ? s[q0 + k] : 0u;
        sum += v[k];
    }
    __shared__ uint32_t s_total;
    const uint32_t ex = block_excl_scan<kFeThreads>(sum, s_warp);
    if (t == kFeThreads - 1) s_total = ex + sum;
    uint32_t run = ex;
#pragma unroll
    for (int k = 0; k < 8; ++k)
        if (k < (int)per && q0 + k < n) {
            s[q0 + k] = run;
            run += v[k];
        }
    __syncthreads();
    return s_total;
}

// One warp's walk over the depth-order pairs [q0, q1), 32 consecutive pairs
// per step (lane = pair; its splat = owner lane of the current row of 32
// splats, found by a shuffle binary search).  drec[j] = depth-order record of
// splat j: (first pair, Gaussian id, x0 | y0 << 16, wx | wy << 16).  Counters
// are 16-bit, packed two per word: c16w = the word array, index = tile.
// MODE 1: count (red.add, order-free).  MODE 0: rank = counter value before
// the step + number of earlier lanes of the step with the same tile, then
// fn(tile, rank, Gaussian id); the earlier same-tile lanes can only belong
// to earlier splats of the step (a splat's tiles are distinct), so each lane
// tests, for every earlier splat of the step, whether its rect holds the
// lane's tile at a pair index inside this step -- no MATCH.ANY.
template <int MODE, typename F>
__device__ __forceinline__ void fe_walk(const uint4* __restrict__ drec,
                                        const uint32_t* __restrict__ cb, int cshift, uint32_t n,
                                        uint32_t q0, uint32_t q1, int tiles_x,
                                        uint32_t* __restrict__ c16w, F&& fn) {
    const int l = threadIdx.x & 31;
    if (q0 >= q1) return;
    // owner of pair q0 = largest j with first[j] <= q0 (zero-count splats
    // share their successor's first pair, so the owner has pairs); the warp
    // narrows [lo, hi) 32-fold per round
    uint32_t lo = 0, hi = n;
    while (hi - lo > 1) {
        const uint32_t step = (hi - lo + 31) / 32;
        const uint32_t j = lo + l * step;
        const bool le = j < hi && drec[j].x + cb[j >> cshift] <= q0;
        const unsigned m = __ballot_sync(0xffffffffu, le);  // lanes 0..k set (monotone)
        const int k = 31 - __clz(m);                           // m has bit 0: drec[lo].x <= q0
        lo = lo + k * step;
        hi = min(hi, lo + step);
    }
    const uint4 kEnd = make_uint4(0xffffffffu, 0u, 0u, 0u);
    uint32_t js = lo;
    uint4 cur = js + l < n ? drec[js + l] : kEnd;
    uint32_t q = q0;
    while (q < q1) {
        const uint4 nxt = js + 32 + l < n ? drec[js + 32 + l] : kEnd;  // prefetch
        if (cur.x != 0xffffffffu) cur.x += cb[(js + l) >> cshift];
        const bool valid = cur.x != 0xffffffffu;
        const uint32_t wx = max(cur.w & 0xffffu, 1u), wy = cur.w >> 16;
        const uint32_t c = valid ? wx * wy : 0u;
        const uint32_t rlo = __shfl_sync(0xffffffffu, cur.x, 0);
        const uint32_t rel = valid ? cur.x - rlo : 0x7fffffffu;
        uint32_t endw = valid ? rel + c : 0u;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) endw = max(endw, __shfl_xor_sync(0xffffffffu, endw, d));
        const uint32_t a1 = min(rlo + endw, q1);
#pragma unroll 2
        for (uint32_t e0 = q - rlo; e0 < a1 - rlo; e0 += 32) {
            const uint32_t e = e0 + l;
            const bool in = e < a1 - rlo;
            int o = 0;  // owner lane = largest lane with rel <= e
#pragma unroll
            for (int st = 16; st > 0; st >>= 1) {
                const uint32_t r = __shfl_sync(0xffffffffu, rel, o + st);
                if (r <= e) o += st;
            }
            const uint32_t li = e - __shfl_sync(0xffffffffu, rel, o);
            const uint32_t oxy = __shfl_sync(0xffffffffu, cur.z, o);
            const uint32_t ow = __shfl_sync(0xffffffffu, wx, o);
            uint32_t tx = 0, ty = 0;
            if (in) {
                // li / ow through a float quotient, corrected to the exact one
                uint32_t ry = __float2uint_rz(__fdividef((float)li, (float)ow));
                if (ry * ow > li) --ry;
                if ((ry + 1) * ow <= li) ++ry;
                tx = (oxy & 0xffffu) + (li - ry * ow);
                ty = (oxy >> 16) + ry;
            }
            const uint32_t tile = ty * (uint32_t)tiles_x + tx;
            uint32_t* word = c16w + (tile >> 1);
            const uint32_t sh = 16 * (tile & 1);
            if (MODE == 2) {  // 32-bit counters
                if (in) atomicAdd(c16w + tile, 1u);
            } else if (MODE == 1) {
                if (in) atomicAdd(word, 1u << sh);
            } else {
                const uint32_t gid = __shfl_sync(0xffffffffu, cur.y, o);
                // rank = the tile's counter before this pair.  The step's
                // pairs take their counters splat by splat (one predicated
                // atomic per splat of the step, in depth order); a splat's
                // tiles are distinct, so within one atomic every lane owns
                // its own 16-bit half and the returned half is exact
                const int o_first = __shfl_sync(0xffffffffu, o, 0);
                const int o_last =
                    __shfl_sync(0xffffffffu, in ? o : 0, 31 - __clz(__ballot_sync(0xffffffffu, in)));
                uint32_t old = 0;
#pragma unroll 1
                for (int k = o_first; k <= o_last; ++k)
                    if (in && o == k) old = atomicAdd(word, 1u << sh);
                if (in) fn(tile, (old >> sh) & 0xffffu, gid);
            }
            __syncwarp();
        }
        q = a1;
        js += 32;
        cur = nxt;
    }
}


template <int ITEMS>
__device__ void fe_direct(const FeArgs& a, cooperative_groups::grid_group& grid, uint32_t* sm,
                          uint32_t* s_warp, const uint32_t* order) {
    constexpr int kFeTile = kFeThreads * ITEMS;
    const int t = threadIdx.x, w = t >> 5, l = t & 31;
    const uint32_t cta = blockIdx.x, nc = gridDim.x;
    const uint32_t base = cta * kFeTile;
    const uint32_t wbase = w * 32 * ITEMS;
    const uint32_t NT = a.n_img_tiles;
    const uint32_t G = (uint32_t)fe_direct_warps((int)NT);
    const uint32_t NT2 = (NT + 1) & ~1u;  // counter row stride (whole words)
    uint16_t* s_c16 = reinterpret_cast<uint16_t*>(sm);  // [G][NT2] placer-warp counters
    uint32_t* s_base = sm + (size_t)G * NT2 / 2;       // [NT] 32-bit per tile

    // ---- this CTA's depth-sort chunk: pair counts, chunk total
    uint32_t sid[ITEMS], cnt[ITEMS], off[ITEMS];
    uint2 rct[ITEMS];
    uint32_t wtot = 0;
#pragma unroll
    for (int r = 0; r < ITEMS; ++r) {
        const uint32_t j = base + wbase + r * 32 + l;
        sid[r] = j < a.n ? order[j] : 0u;
    }
#pragma unroll
    for (int r = 0; r < ITEMS; ++r) {
        const uint32_t j = base + wbase + r * 32 + l;
        cnt[r] = j < a.n ? a.tiles[sid[r]] : 0u;
        rct[r] = j < a.n ? a.rect[sid[r]] : make_uint2(0u, 0u);  // loaded with the count
    }
#pragma unroll
    for (int r = 0; r < ITEMS; ++r) {
        uint32_t x = cnt[r];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (l >= o) x += y;
        }
        off[r] = wtot + x - cnt[r];
        wtot += __shfl_sync(0xffffffffu, x, 31);
    }
    const uint32_t wex = block_excl_scan<kFeThreads>(l == 0 ? wtot : 0u, s_warp);
    const uint32_t wpre = __shfl_sync(0xffffffffu, wex, 0);
    if (t == kFeThreads - 1) a.chunk_sum[cta] = wpre + wtot;
    // depth-order records with chunk-local first pairs (the walks add the
    // chunk's base from s_cb)
#pragma unroll
    for (int r = 0; r < ITEMS; ++r) {
        const uint32_t j = base + wbase + r * 32 + l;
        if (j < a.n) {
            uint4 d = make_uint4(wpre + off[r], sid[r], 0u, 0u);
            if (cnt[r]) {
                const uint2 rc = rct[r];
                d.z = rc.x;
                d.w = ((rc.y & 0xffffu) - (rc.x & 0xffffu) + 1) |
                      (((rc.y >> 16) - (rc.x >> 16) + 1) << 16);
            }
            a.drec[j] = d;
        }
    }
    for (uint32_t q = t; q < (uint32_t)G * NT2 / 2; q += kFeThreads) sm[q] = 0u;
    for (uint32_t q = t; q < NT; q += kFeThreads) s_base[q] = 0u;
    FE_STAMP(10);
    grid.sync();
    FE_STAMP(11);
    // ---- chunk bases (exclusive prefix of the chunk sums), P, capacity
    __shared__ uint32_t s_cb[32 * kFeColChunks + 1];
    if (w == 0) {
        uint32_t c[kFeColChunks], sum = 0;
#pragma unroll
        for (int k = 0; k < kFeColChunks; ++k) {
            const uint32_t i = l * kFeColChunks + k;
            c[k] = i < nc ? a.chunk_sum[i] : 0u;
            sum += c[k];
        }
        uint32_t x = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (l >= o) x += y;
        }
        uint32_t run = x - sum;
#pragma unroll
        for (int k = 0; k < kFeColChunks; ++k) {
            const uint32_t i = l * kFeColChunks + k;
            if (i < nc) s_cb[i] = run;
            run += c[k];
        }
        if (l == 31) s_cb[nc] = x;
    }
    __syncthreads();
    const uint32_t P = s_cb[nc];
    if ((int64_t)P > a.cap) {
        if (cta == 0 && t == 0) {
            *a.total = (int64_t)P;
            *a.overflow = 1;  // sticky; the step is replayed with larger buffers
            *a.pcount = 0u;
        }
        return;
    }
    if (cta == 0 && t == 0) {
        *a.total = (int64_t)P;
        *a.pcount = P;
    }
    const int cshift = 31 - __clz(kFeTile);
    // the CTA's pair range (pair-balanced), processed in pieces of at most
    // kDirPiece pairs so the per-(warp, tile) counters fit 16 bits
    const uint32_t p0 = (uint32_t)(((uint64_t)P * cta) / nc);
    const uint32_t p1 = (uint32_t)(((uint64_t)P * (cta + 1)) / nc);
    const uint32_t npieces = (p1 - p0 + kDirPiece - 1) / kDirPiece;
    // count walk over [c0, c1): placer warp g counts its own share into its
    // private row (the same split as the rank walk)
    auto count_piece = [&](uint32_t c0, uint32_t c1) {
        if (w < (int)G) {
            const uint32_t span = c1 - c0;
            const uint32_t g0 = c0 + (uint32_t)(((uint64_t)span * w) / G);
            const uint32_t g1 = c0 + (uint32_t)(((uint64_t)span * (w + 1)) / G);
            fe_walk<1>(a.drec, s_cb, cshift, a.n, g0, g1, a.tiles_x, sm + (size_t)w * (NT2 / 2),
                       [](uint32_t, uint32_t, uint32_t) {});
        }
    };
    // placer-warp counters -> exclusive prefix over the warps (per tile);
    // returns nothing, totals land in tot (may alias nothing)
    // (two tiles per 32-bit word: the 16-bit halves never carry, a tile's
    // count in one piece is < 2^16; the G words of a column are loaded
    // before the running sum walks them)
    auto prefix_warps = [&](uint32_t* tot) {
        const uint32_t NW = NT2 / 2;
        for (uint32_t k = t; k < NW; k += kFeThreads) {
            uint32_t v[32];
#pragma unroll
            for (int g = 0; g < 32; ++g) v[g] = g < (int)G ? sm[(size_t)g * NW + k] : 0u;
            uint32_t run = 0;
#pragma unroll
            for (int g = 0; g < 32; ++g)
                if (g < (int)G) {
                    sm[(size_t)g * NW + k] = run;
                    run += v[g];
                }
            if (tot) {
                if (2 * k < NT) tot[2 * k] = run & 0xffffu;
                if (2 * k + 1 < NT) tot[2 * k + 1] = run >> 16;
            }
        }
    };
    auto zero_c16 = [&]() {
        for (uint32_t q = t; q < (uint32_t)G * NT2 / 2; q += kFeThreads) sm[q] = 0u;
    };
    // ---- count: per-tile totals of the CTA's range -> col[cta][tile]
    if (npieces <= 1) {
        count_piece(p0, p1);
        __syncthreads();
        FE_STAMP(12);
        prefix_warps(s_base);
        FE_STAMP(13);
    } else {
        for (uint32_t q0 = p0 + w * 32 * 64; q0 < p1; q0 += kFeWarps * 32 * 64)
            fe_walk<2>(a.drec, s_cb, cshift, a.n, q0, min(p1, q0 + 32 * 64), a.tiles_x, s_base,
                       [](uint32_t, uint32_t, uint32_t) {});
    }
    __syncthreads();
    for (uint32_t q = t; q < NT; q += kFeThreads) a.col[(size_t)cta * NT + q] = s_base[q];
    FE_STAMP(14);
    grid.sync();
    FE_STAMP(15);
    // ---- per tile: exclusive prefix over the CTAs (in place), tile total;
    //      a warp per tile (tiles spread over the CTAs), lane l holds CTAs
    //      5 l .. 5 l + 4
    for (uint32_t q = w * nc + cta; q < NT; q += nc * kFeWarps) {
        uint32_t c[kFeColChunks], sum = 0;
#pragma unroll
        for (int k = 0; k < kFeColChunks; ++k) {
            const uint32_t i = l * kFeColChunks + k;
            c[k] = i < nc ? a.col[(size_t)i * NT + q] : 0u;
            sum += c[k];
        }
        uint32_t x = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (l >= o) x += y;
        }
        uint32_t run = x - sum;
#pragma unroll
        for (int k = 0; k < kFeColChunks; ++k) {
            const uint32_t i = l * kFeColChunks + k;
            if (i < nc) a.col[(size_t)i * NT + q] = run;
            run += c[k];
        }
        if (l == 31) a.col_tot[q] = x;
    }
    FE_STAMP(16);
    grid.sync();
    FE_STAMP(17);
    // ---- tile starts (every CTA scans the totals); the CTA's first slot per
    //      tile -> s_base
    for (uint32_t q = t; q < NT; q += kFeThreads) s_base[q] = a.col_tot[q];
    __syncthreads();
    fe_scan_smem(s_base, NT, s_warp);
    for (uint32_t q = t; q < NT; q += kFeThreads) {
        const uint32_t st = s_base[q];
        if (cta == 0) {
            a.tile_start[q] = st;
            a.tile_end[q] = st + a.col_tot[q];
        }
        s_base[q] = st + a.col[(size_t)cta * NT + q];
    }
    if (cta == 0) {
        // checkpoint slot bases: exclusive scan of ceil(len / 32) over the
        // tiles, n_tiles + 1 entries (thread t: tiles t per .. t per + per - 1)
        const uint32_t per = (NT + kFeThreads - 1) / kFeThreads;
        const uint32_t q0 = t * per;
        uint32_t sum = 0;
        for (uint32_t k = 0; k < per; ++k)
            if (q0 + k < NT) sum += (a.col_tot[q0 + k] + 31u) >> 5;
        uint32_t run = block_excl_scan<kFeThreads>(sum, s_warp);
        for (uint32_t k = 0; k < per; ++k)
            if (q0 + k < NT) {
                a.ckpt_base[q0 + k] = run;
                run += (a.col_tot[q0 + k] + 31u) >> 5;
            }
        if (q0 < NT && q0 + per >= NT) a.ckpt_base[NT] = run;  // the thread holding the last tile
    }
    __syncthreads();
    FE_STAMP(18);
    // ---- rank + write, piece by piece: placer warp g walks its share of the
    //      piece in depth order; slot = CTA base + earlier pieces + earlier
    //      placer warps + rank in the warp's walk
    uint32_t* out = a.out_splat;
#pragma unroll 1
    for (uint32_t pc = 0; pc < max(npieces, 1u); ++pc) {
        const uint32_t c0 = p0 + pc * kDirPiece, c1 = min(p1, c0 + kDirPiece);
        if (npieces > 1) {
            zero_c16();
            __syncthreads();
            count_piece(c0, c1);
            __syncthreads();
            prefix_warps(nullptr);
            __syncthreads();
        }
        if (w < (int)G) {
            const uint32_t span = c1 - c0;
            const uint32_t g0 = c0 + (uint32_t)(((uint64_t)span * w) / G);
            const uint32_t g1 = c0 + (uint32_t)(((uint64_t)span * (w + 1)) / G);
            const uint32_t* sb = s_base;
            fe_walk<0>(a.drec, s_cb, cshift, a.n, g0, g1, a.tiles_x, sm + (size_t)w * (NT2 / 2),
                       [out, sb](uint32_t tile, uint32_t r, uint32_t gid) {
                           out[sb[tile] + r] = gid;
                       });
        }
        __syncthreads();
        if (pc + 1 < npieces) {
            // the last placer warp's counters ended at the piece totals
            for (uint32_t q = t; q < NT; q += kFeThreads)
                s_base[q] += s_c16[(size_t)(G - 1) * NT2 + q];
            __syncthreads();
        }
    }
    FE_STAMP(19);
}

template <int ITEMS>
__global__ void __launch_bounds__(kFeThreads, 1) bin_front_kernel(FeArgs a) {
    constexpr int kFeTile = kFeThreads * ITEMS;
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ uint32_t fe_smem[];
    uint32_t(*s_cnt)[256] = reinterpret_cast<uint32_t(*)[256]>(fe_smem);  // [kFeWarps]
    uint32_t* s_keys = fe_smem + kFeWarps * 256;
    uint32_t* s_vals = s_keys + kFeTile;
    uint32_t(*s_part)[512] = reinterpret_cast<uint32_t(*)[512]>(s_vals + kFeTile);  // [4]
    __shared__ uint32_t s_base[256], s_local[256], s_warp[32];
    const int t = threadIdx.x, w = t >> 5, l = t & 31;
    const uint32_t tile = blockIdx.x;    // gridDim.x == n_tiles
    const uint32_t base = tile * kFeTile;
    const uint32_t nloc = min((uint32_t)kFeTile, a.n - base);
    const uint32_t wbase = w * 32 * ITEMS;

    FE_STAMP(0);
    // Direct mode skips the passes whose digit is the same for every splat
    // that has pairs (e.g. the exponent byte when all depths lie in one
    // binade pair): splats without pairs never reach the pair list, so their
    // relative order is irrelevant, and a stable pass over a constant digit
    // is the identity on the others.  The AND / OR of those keys is reduced
    // in pass 0; the mask is known after its first barrier.
    __shared__ uint32_t s_red[2][kFeWarps], s_skip;
    const uint32_t* ksrc = a.key_in;
    const uint32_t* vsrc = nullptr;
    int par = 0, lastp = 3;
    uint32_t skipmask = 0;
#pragma unroll 1
    for (int p = 0; p < 4; ++p) {
        if ((skipmask >> p) & 1u) continue;  // block- and grid-uniform
        const uint32_t* kin = ksrc;
        const uint32_t* vin = vsrc;
        uint32_t* kout = par ? a.kB : a.kA;
        uint32_t* vout = par ? a.vB : a.vA;
        uint32_t* cnt = a.counts + (size_t)par * a.n_tiles * 256;
        const int shift = 8 * p;
        // ---- phase A: rank within the tile, publish the digit histogram
        for (int k = t; k < kFeWarps * 256; k += kFeThreads) (&s_cnt[0][0])[k] = 0u;
        __syncthreads();
        uint32_t key[ITEMS], val[ITEMS], rank[ITEMS];
#pragma unroll
        for (int r = 0; r < ITEMS; ++r) {
            const uint32_t li = wbase + r * 32 + l;
            key[r] = li < nloc ? kin[base + li] : 0u;
            val[r] = li < nloc ? (vin ? vin[base + li] : base + li) : 0u;
        }
#pragma unroll
        for (int r = 0; r < ITEMS; ++r) {
            const uint32_t li = wbase + r * 32 + l;
            const bool valid = li < nloc;
            const uint32_t d = (key[r] >> shift) & 255u;
            const unsigned peers = peers8(d, valid);
            const uint32_t before = valid ? s_cnt[w][d] : 0u;
            rank[r] = before + __popc(peers & lanemask_lt());
            __syncwarp();
            if (valid && (peers & lanemask_lt()) == 0) s_cnt[w][d] = before + __popc(peers);
            __syncwarp();
        }
        __syncthreads();
        uint32_t run = 0;
        if (t < 256) {
#pragma unroll 8
            for (int k = 0; k < kFeWarps; ++k) {
                const uint32_t c = s_cnt[k][t];
                s_cnt[k][t] = run;
                run += c;
            }
            cnt[(size_t)t * a.n_tiles + tile] = run;  // this tile's digit histogram ([d][tile])
        }
        const uint32_t loc = block_excl_scan<kFeThreads>(t < 256 ? run : 0u, s_warp);
        if (t < 256) s_local[t] = loc;
        if (p == 0 && a.direct) {
            uint32_t kand = 0xffffffffu, kor = 0u;
#pragma unroll
            for (int r = 0; r < ITEMS; ++r) {
                const uint32_t li = wbase + r * 32 + l;
                if (li < nloc && a.tiles[base + li] != 0u) {
                    kand &= key[r];
                    kor |= key[r];
                }
            }
            kand = __reduce_and_sync(0xffffffffu, kand);
            kor = __reduce_or_sync(0xffffffffu, kor);
            if (l == 0) {
                s_red[0][w] = kand;
                s_red[1][w] = kor;
            }
            __syncthreads();
            if (t == 0) {
                for (int k = 1; k < kFeWarps; ++k) {
                    kand &= s_red[0][k];
                    kor |= s_red[1][k];
                }
                a.keyred[2 * tile] = s_red[0][0] & kand;
                a.keyred[2 * tile + 1] = s_red[1][0] | kor;
            }
        }
        FE_STAMP(1 + 2 * p);
        grid.sync();
        FE_STAMP(20 + p);
        if (p == 0 && a.direct) {
            if (w == 0) {
                uint32_t kand = 0xffffffffu, kor = 0u;
                for (uint32_t q = l; q < a.n_tiles; q += 32) {
                    kand &= a.keyred[2 * q];
                    kor |= a.keyred[2 * q + 1];
                }
                kand = __reduce_and_sync(0xffffffffu, kand);
                kor = __reduce_or_sync(0xffffffffu, kor);
                const uint32_t diff = kand ^ kor;
                uint32_t m = 0;
                for (int q = 1; q < 4; ++q)
                    if (((diff >> (8 * q)) & 255u) == 0u) m |= 1u << q;
                if (l == 0) s_skip = m;
            }
            __syncthreads();
            skipmask = s_skip;
            lastp = 3;
            while (lastp > 0 && ((skipmask >> lastp) & 1u)) --lastp;
        }
        // ---- phase B: digit starts = exclusive digit total + column prefix;
        //      warp w reduces the columns of digits w + 32 k (coalesced rows of
        //      the [digit][tile] histograms), all loads of a batch in flight
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            uint32_t c[4][kFeColChunks];
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
                for (int j = 0; j < kFeColChunks; ++j) {
                    const uint32_t q = l + 32 * j;
                    const int d = w + kFeWarps * (4 * half + k);
                    c[k][j] = q < a.n_tiles ? cnt[(size_t)d * a.n_tiles + q] : 0u;
                }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                uint32_t before = 0, all = 0;
#pragma unroll
                for (int j = 0; j < kFeColChunks; ++j) {
                    all += c[k][j];
                    before += (l + 32 * j) < tile ? c[k][j] : 0u;
                }
                all = warp_sum(all);
                before = warp_sum(before);
                if (l == 0) {
                    const int d = w + kFeWarps * (4 * half + k);
                    s_part[0][d] = before;
                    s_part[0][256 + d] = all;
                }
            }
        }
        __syncthreads();
        FE_STAMP(24 + 4 * p);
        const uint32_t col = t < 256 ? s_part[0][t] : 0u;
        const uint32_t tot = t < 256 ? s_part[0][256 + t] : 0u;
        const uint32_t excl = block_excl_scan<kFeThreads>(t < 256 ? tot : 0u, s_warp);
        if (t < 256) s_base[t] = excl + col;
#pragma unroll
        for (int r = 0; r < ITEMS; ++r) {
            const uint32_t li = wbase + r * 32 + l;
            if (li < nloc) {
                const uint32_t d = (key[r] >> shift) & 255u;
                const uint32_t lp = s_local[d] + s_cnt[w][d] + rank[r];
                s_keys[lp] = key[r];
                s_vals[lp] = val[r];
            }
        }
        __syncthreads();
        FE_STAMP(25 + 4 * p);
        for (uint32_t i = t; i < nloc; i += kFeThreads) {
            const uint32_t k = s_keys[i];
            const uint32_t d = (k >> shift) & 255u;
            const uint32_t gp = s_base[d] + (i - s_local[d]);
            vout[gp] = s_vals[i];
            if (p < lastp) kout[gp] = k;
        }
        FE_STAMP(26 + 4 * p);
        grid.sync();
        FE_STAMP(2 + 2 * p);
        ksrc = kout;
        vsrc = vout;
        par ^= 1;
    }

    if (a.direct) {
        fe_direct<ITEMS>(a, grid, fe_smem, s_warp, vsrc);
        return;
    }
    // ---- chunk sums of the final order (vB: pass 3 wrote the B buffers);
    //      warp w holds rows of 32 consecutive splats, wbase + 32 r + lane
    const uint32_t* order = a.vB;
    uint32_t sidr[ITEMS], cr[ITEMS], ir[ITEMS], rpre[ITEMS];
    uint32_t wtot = 0;
#pragma unroll
    for (int r = 0; r < ITEMS; ++r) {
        const uint32_t j = base + wbase + r * 32 + l;
        sidr[r] = j < a.n ? order[j] : 0u;
        cr[r] = j < a.n ? a.tiles[sidr[r]] : 0u;
        uint32_t x = cr[r];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (l >= o) x += y;
        }
        ir[r] = x;
        rpre[r] = wtot;
        wtot += __shfl_sync(0xffffffffu, x, 31);
    }
    const uint32_t wex = block_excl_scan<kFeThreads>(l == 0 ? wtot : 0u, s_warp);
    const uint32_t wpre = __shfl_sync(0xffffffffu, wex, 0);
    if (t == kFeThreads - 1) a.chunk_sum[tile] = wpre + wtot;  // last warp: tile total
    grid.sync();
    // ---- P, capacity check, tile prefix
    uint32_t P = 0, pre = 0;
    for (uint32_t q = l; q < a.n_tiles; q += 32) {
        const uint32_t c = a.chunk_sum[q];
        P += c;
        pre += q < tile ? c : 0u;
    }
    P = warp_sum(P);
    pre = warp_sum(pre);
    if ((int64_t)P > a.cap) {
        if (tile == 0 && t == 0) {
            *a.total = (int64_t)P;
            *a.overflow = 1;  // sticky; the step is replayed with larger buffers
            *a.pcount = 0u;
        }
        return;
    }
    if (tile == 0 && t == 0) {
        *a.total = (int64_t)P;
        *a.pcount = P;
    }
    // ---- emission, warp-cooperative per row of 32 splats
#pragma unroll
    for (int r = 0; r < ITEMS; ++r) {
        const uint32_t j = base + wbase + r * 32 + l;
        const uint32_t cc = cr[r];
        const uint32_t o = pre + wpre + rpre[r] + ir[r] - cc;
        uint32_t x0 = 0, y0 = 0, wx = 1;
        if (j < a.n && cc) {
            const uint2 rc = a.rect[sidr[r]];
            x0 = rc.x & 0xffffu;
            y0 = rc.x >> 16;
            wx = (rc.y & 0xffffu) - x0 + 1;
        }
        const uint32_t b0 = __shfl_sync(0xffffffffu, o, 0);
        const uint32_t rel = j < a.n ? o - b0 : 0x7fffffffu;
        uint32_t endw = j < a.n ? rel + cc : 0u;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) endw = max(endw, __shfl_xor_sync(0xffffffffu, endw, d));
        for (uint32_t e0 = 0; e0 < endw; e0 += 32) {
            const uint32_t e = e0 + l;
            int lo = 0;
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const uint32_t rr = __shfl_sync(0xffffffffu, rel, lo + step);
                if (rr <= e) lo += step;
            }
            const uint32_t li = e - __shfl_sync(0xffffffffu, rel, lo);
            const uint32_t ox = __shfl_sync(0xffffffffu, x0, lo);
            const uint32_t oy = __shfl_sync(0xffffffffu, y0, lo);
            const uint32_t ow = __shfl_sync(0xffffffffu, wx, lo);
            const uint32_t sid = __shfl_sync(0xffffffffu, sidr[r], lo);
            if (e < endw) {
                const uint32_t ry = li / ow;
                const uint32_t tid = (oy + ry) * a.tiles_x + ox + (li - ry * ow);
                if (a.pair_v) {
                    a.pair_k[b0 + e] = tid;
                    a.pair_v[b0 + e] = sid;
                } else {
                    a.pair_k[b0 + e] = (tid << a.sb) | sid;
                }
            }
        }
    }
}

// ------------------------------------------------------------ workspace
struct BinWorkspace {
    size_t off = 0;
    char* base = nullptr;
    template <typename T>
    T* take(size_t count) {
        off = (off + 255) & ~size_t(255);
        T* p = reinterpret_cast<T*>(base ? base + off : nullptr);
        off += count * sizeof(T);
        return p;
    }
};

constexpr int kDepthItems = 8;  // 2048 splats per radix CTA
constexpr int kPairItems = 8;   // 2048 pairs per radix CTA

struct BinLayout {
    // zero-initialised control region first
    uint32_t* ctrl;            // counters
    unsigned long long* st_scan1;
    unsigned long long* st_scan2;
    size_t ctrl_bytes;
    // data
    uint32_t *kA, *vA, *kB, *vB;      // N
    uint32_t* offsets;                // N
    uint32_t *pk0, *pk1, *pv0, *pv1;  // pair capacity
    uint32_t* pcount;                 // 1
    uint32_t* rs_counts;              // 256 * max blocks
    uint32_t* rs_totals;              // 256
    // persistent front end (in the zeroed control region)
    uint32_t* fe_counts;              // 2 * n_fe_tiles * 256
    uint32_t* fe_chunk;               // n_fe_tiles
    uint32_t* fe_col;                 // 32 * kFeColChunks * n_tiles (direct emission)
    uint32_t* fe_col_tot;             // n_tiles
    uint4* fe_drec;                   // n (direct emission)
    uint32_t* fe_keyred;              // 2 * n_fe_tiles
};

inline int tile_passes(int n_tiles) {
    int bits = 1;
    while ((1ll << bits) < n_tiles) ++bits;
    return (bits + 7) / 8;
}

BinLayout bin_layout(int64_t n, int64_t cap, int n_tiles, void* ws, size_t* bytes) {
    BinWorkspace w;
    w.base = reinterpret_cast<char*>(ws);
    BinLayout L;
    L.ctrl = w.take<uint32_t>(16);
    L.st_scan1 = w.take<unsigned long long>(div_up(n > 0 ? n : 1, 256 * kScanItems) + 1);
    L.st_scan2 = w.take<unsigned long long>(div_up(n_tiles + 1, 256 * kScanItemsTiles) + 1);
    w.off = (w.off + 255) & ~size_t(255);
    L.ctrl_bytes = w.off;
    L.kA = w.take<uint32_t>(n);
    L.vA = w.take<uint32_t>(n);
    L.kB = w.take<uint32_t>(n);
    L.vB = w.take<uint32_t>(n);
    L.offsets = w.take<uint32_t>(n);
    L.pk0 = w.take<uint32_t>(cap);
    L.pk1 = w.take<uint32_t>(cap);
    L.pv0 = w.take<uint32_t>(cap);
    L.pv1 = w.take<uint32_t>(cap);
    L.pcount = w.take<uint32_t>(4);
    {
        const int64_t nft = div_up(n > 0 ? n : 1, 2 * kFeThreads);  // smallest tiles
        L.fe_counts = w.take<uint32_t>(2 * nft * 256);
        L.fe_chunk = w.take<uint32_t>(nft);
        L.fe_col = w.take<uint32_t>((size_t)32 * kFeColChunks * (n_tiles > 0 ? n_tiles : 1));
        L.fe_col_tot = w.take<uint32_t>(n_tiles > 0 ? n_tiles : 1);
        L.fe_drec = w.take<uint4>(n > 0 ? n : 1);
        L.fe_keyred = w.take<uint32_t>(2 * nft);
    }
    {
        int64_t mx = cap > n ? cap : n;
        L.rs_counts = w.take<uint32_t>(
            (size_t)256 * (div_up(mx > 0 ? mx : 1, 256 * (kDepthItems < kPairItems ? kDepthItems
                                                                               : kPairItems)) +
                           1));
        L.rs_totals = w.take<uint32_t>(256);
    }
    if (bytes) *bytes = w.off + 256;
    return L;
}

size_t bin_workspace_bytes(int64_t n, int64_t cap, int n_tiles) {
    size_t b = 0;
    bin_layout(n, cap, n_tiles, nullptr, &b);
    return b;
}

template <int ITEMS>
static int fe_capacity(size_t bytes) {  // co-resident CTAs of bin_front_kernel<ITEMS>, 0 = unusable
    int dev = 0, coop = 0, sms = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (!coop ||
        cudaFuncSetAttribute(bin_front_kernel<ITEMS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)bytes) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, bin_front_kernel<ITEMS>, kFeThreads,
                                                      bytes) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return sms * occ;
}

// Cooperative launch of bin_front_kernel (one sort tile per co-resident
// CTA); false -> use the per-pass kernels (N too large, cooperative launch
// unavailable, or SS_BIN_FRONT=0 in the environment).  *direct: the kernel
// also wrote the final pair list and the tile ranges (fe_direct; off with
// SS_BIN_DIRECT=0 or more than kDirMaxTiles image tiles).
static bool front_end_launch(int64_t n, const ss_splats* sp, const ss_bins* bins, int tiles_x,
                             int n_tiles, const BinLayout& L, bool packed, int sbits, int64_t cap,
                             ss_status* st, cudaStream_t s, bool* direct) {
    static int enabled = -1, direct_ok = -1;
    if (enabled < 0) {
        const char* env = getenv("SS_BIN_FRONT");
        enabled = !(env && env[0] == '0');
        const char* env2 = getenv("SS_BIN_DIRECT");
        direct_ok = !(env2 && env2[0] == '0');
    }
    *direct = false;
    if (!enabled) return false;
    const bool dir = direct_ok && n_tiles <= kDirMaxTiles && n_tiles > 0;
    FeArgs a;
    a.n = (uint32_t)n;
    a.key_in = sp->d_depth_key;
    a.kA = L.kA;
    a.vA = L.vA;
    a.kB = L.kB;
    a.vB = L.vB;
    a.counts = L.fe_counts;
    a.chunk_sum = L.fe_chunk;
    a.tiles = sp->d_tiles;
    a.rect = reinterpret_cast<const uint2*>(sp->d_rect);
    a.tiles_x = tiles_x;
    a.pair_k = L.pk0;
    a.pair_v = packed ? nullptr : L.pv0;
    a.sb = sbits;
    a.total = &st->pair_count;
    a.overflow = &st->pair_overflow;
    a.cap = cap;
    a.pcount = L.pcount;
    a.direct = dir ? 1 : 0;
    a.n_img_tiles = (uint32_t)n_tiles;
    a.col = L.fe_col;
    a.col_tot = L.fe_col_tot;
    a.out_splat = bins->d_pair_splat;
    a.tile_start = bins->d_tile_start;
    a.tile_end = bins->d_tile_end;
    a.drec = L.fe_drec;
    a.keyred = L.fe_keyred;
    a.ckpt_base = bins->d_ckpt_base;
    void* args[] = {&a};
    auto go = [&](auto kern, int items, int capacity) -> bool {
        const int64_t nft = div_up(n, (int64_t)kFeThreads * items);
        if (nft > capacity || nft > 32 * kFeColChunks) return false;
        a.n_tiles = (uint32_t)nft;
        size_t bytes = fe_smem_bytes_rt(items);
        if (dir && fe_direct_smem_bytes(n_tiles) > bytes) bytes = fe_direct_smem_bytes(n_tiles);
        if (cudaLaunchCooperativeKernel((const void*)kern, (int)nft, kFeThreads, args, bytes,
                                        s) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        return true;
    };
    // capacities for the largest shared-memory footprint this launch may use
    static int cap2 = -1, cap4 = -1, cap8 = -1;
    static size_t cap_bytes = 0;
    const size_t want = (size_t)kDirSmemBytes + 16 > fe_smem_bytes<8>() ? (size_t)kDirSmemBytes + 16
                                                                        : fe_smem_bytes<8>();
    if (cap_bytes != want) {
        cap_bytes = want;
        cap2 = fe_capacity<2>(want);
        cap4 = fe_capacity<4>(want);
        cap8 = fe_capacity<8>(want);
    }
    const bool ok = go(bin_front_kernel<2>, 2, cap2) || go(bin_front_kernel<4>, 4, cap4) ||
                    go(bin_front_kernel<8>, 8, cap8);
    *direct = ok && dir;
    return ok;
}

// The forward's tile order alone (costliest first by d_tile_cost), e.g. on
// a side stream while the next step's projection runs.
cudaError_t launch_tile_order(const ss_camera* cam, const ss_bins* bins, cudaStream_t s) {
    const int n_tiles = div_up(cam->width, kTile) * div_up(cam->height, kTile);
    if (!bins->d_tile_order || !bins->d_tile_cost || n_tiles > SS_ORDER_MAX_TILES)
        return cudaErrorInvalidValue;
    tile_meta_kernel<<<1, 1024, 0, s>>>(bins->d_tile_start, bins->d_tile_end, n_tiles, nullptr,
                                        bins->d_tile_cost, bins->d_tile_order);
    return cudaGetLastError();
}

cudaError_t launch_bin_sort(int64_t n, const ss_splats* sp, const ss_camera* cam,
                            const ss_bins* bins, void* ws, size_t ws_bytes, ss_status* st,
                            cudaStream_t s) {
    int tiles_x = div_up(cam->width, kTile), tiles_y = div_up(cam->height, kTile);
    int n_tiles = tiles_x * tiles_y;
    int64_t cap = bins->pair_capacity;
    size_t need = 0;
    BinLayout L = bin_layout(n, cap, n_tiles, ws, &need);
    if (need > ws_bytes) return cudaErrorInvalidValue;
    // one launch clears the look-back control words and the tile ranges
    bin_clear_kernel<<<div_up(n_tiles > 1024 ? n_tiles : 1024, 256), 256, 0, s>>>(
        reinterpret_cast<uint32_t*>(L.ctrl), (uint32_t)(L.ctrl_bytes / 4), bins->d_tile_start,
        bins->d_tile_end, (uint32_t)n_tiles);
    cudaError_t e = cudaSuccess;
    int64_t* P = &st->pair_count;
    bool direct_done = false;  // the direct front end also wrote the checkpoint bases
    if (n > 0) {
        uint32_t nn = (uint32_t)n;
        int sbits = 1, tbits = 1;
        while ((1ll << sbits) < n) ++sbits;
        while ((1ll << tbits) < n_tiles) ++tbits;
        const bool packed = sbits + tbits <= 32;
        bool direct = false;
        const bool fe = front_end_launch(n, sp, bins, tiles_x, n_tiles, L, packed, sbits, cap,
                                         st, s, &direct);
        direct_done = direct;
        if (fe) {
            // depth sort + offsets + emission done by the persistent kernel
        } else {
        // 1. depth sort of splats (4 stable 8-bit reduce-then-scan passes)
        const uint32_t* kin = sp->d_depth_key;
        const uint32_t* vin = nullptr;
        uint32_t *ko[2] = {L.kA, L.kB}, *vo[2] = {L.vA, L.vB};
        for (int p = 0; p < 4; ++p) {
            rs_pass<kDepthItems>(kin, vin, p < 3 ? ko[p & 1] : nullptr, vo[p & 1], nullptr, nn, nn,
                                 8 * p, L.rs_counts, L.rs_totals, s);
            kin = ko[p & 1];
            vin = vo[p & 1];
        }
        const uint32_t* order = vo[1];  // pass 3 wrote vB
        // 2. offsets of each splat's pairs in depth order, total P
        scan_kernel<false><<<div_up(n, 256 * kScanItems), 256, 0, s>>>(
            sp->d_tiles, order, nullptr, nn, L.offsets, L.st_scan1, L.ctrl + 8, P,
            &st->pair_overflow, cap);
        // 3. emission of (tile, splat) pairs in depth order; one packed
        //    32-bit word per pair when tile and splat ids fit
        emit_pairs_kernel<<<div_up(n, 256), 256, 0, s>>>(
            nn, order, sp->d_tiles, reinterpret_cast<const uint2*>(sp->d_rect), L.offsets, tiles_x,
            P, cap, L.pk0, packed ? nullptr : L.pv0, sbits);
        clamp_count_kernel<<<1, 1, 0, s>>>(P, cap, L.pcount);
        }
        // 4. stable sort of pairs by tile id (the direct front end already
        //    wrote the final list and the ranges)
        const int np = direct ? 0 : tile_passes(n_tiles);
        const uint32_t* pk = L.pk0;
        const uint32_t* pv = L.pv0;
        for (int p = 0; p < np; ++p) {
            bool last = p == np - 1;
            uint32_t* kdst = (pk == L.pk0) ? L.pk1 : L.pk0;
            if (packed) {
                rs_pass<kPairItems>(pk, nullptr, kdst, nullptr, L.pcount, 0u, (uint32_t)cap,
                                    sbits + 8 * p, L.rs_counts, L.rs_totals, s,
                                    tbits - 8 * p < 8 ? tbits - 8 * p : 8);
            } else {
                // the last pass lands in d_pair_splat
                uint32_t* vdst = last ? bins->d_pair_splat : ((pv == L.pv0) ? L.pv1 : L.pv0);
                rs_pass<kPairItems>(pk, pv, kdst, vdst, L.pcount, 0u, (uint32_t)cap, 8 * p,
                                    L.rs_counts, L.rs_totals, s);
                pv = vdst;
            }
            pk = kdst;
        }
        // 5. ranges by boundary detection on the sorted tile ids (+ unpack)
        if (!direct)
            tile_ranges_kernel<<<div_up(cap > 0 ? cap : 1, 4 * 256), 256, 0, s>>>(
                pk, P, cap, packed ? sbits : 0, bins->d_tile_start, bins->d_tile_end,
                bins->d_pair_splat);
    } else {
        e = cudaMemsetAsync(P, 0, sizeof(int64_t) * 2, s);
        if (e != cudaSuccess) return e;
    }
    // checkpoint slot bases: exclusive scan of ceil(len/32), n_tiles+1 entries
    // (+ the forward's tile order when the caller keeps one)
    const bool order = bins->d_tile_order && bins->d_tile_cost && n_tiles <= SS_ORDER_MAX_TILES;
    if (direct_done) {
        // the front end wrote the checkpoint bases; the order alone remains
        if (order)
            tile_meta_kernel<<<1, 1024, 0, s>>>(bins->d_tile_start, bins->d_tile_end, n_tiles,
                                                nullptr, bins->d_tile_cost, bins->d_tile_order);
    } else if (order) {
        tile_meta_kernel<<<1, 1024, 0, s>>>(bins->d_tile_start, bins->d_tile_end, n_tiles,
                                            bins->d_ckpt_base, bins->d_tile_cost,
                                            bins->d_tile_order);
    } else {
        scan_kernel<true><<<div_up(n_tiles + 1, 256 * kScanItemsTiles), 256, 0, s>>>(
            bins->d_tile_start, nullptr, bins->d_tile_end, (uint32_t)n_tiles + 1,
            bins->d_ckpt_base, L.st_scan2, L.ctrl + 9, nullptr, nullptr, 0);
    }
    return cudaGetLastError();
}

}  // namespace ss

namespace ss {
// Generic exclusive scan of u32 (used by densification's compaction).
size_t scan_ws_bytes(int64_t n) {
    return sizeof(unsigned long long) * (size_t)(div_up(n > 0 ? n : 1, 256 * kScanItems) + 1) + 256;
}

cudaError_t launch_scan_u32(const uint32_t* in, int64_t n, uint32_t* out, int64_t* total,
                            void* ws, cudaStream_t s) {
    if (n <= 0) return cudaMemsetAsync(total, 0, sizeof(int64_t), s);
    int nb = div_up(n, 256 * kScanItems);
    unsigned long long* st = reinterpret_cast<unsigned long long*>(ws);
    uint32_t* counter = reinterpret_cast<uint32_t*>(st + nb);
    cudaError_t e = cudaMemsetAsync(ws, 0, sizeof(unsigned long long) * (nb + 1), s);
    if (e != cudaSuccess) return e;
    scan_kernel<false><<<nb, 256, 0, s>>>(in, nullptr, nullptr, (uint32_t)n, out, st, counter,
                                          total, nullptr, 0);
    return cudaGetLastError();
}
}  // namespace ss

#ifdef SS_FE_TRACE
extern "C" int ss_debug_fe_trace_clear() {
    static const unsigned long long zeros[160 * ss::kFeTraceSlots] = {};
    return (int)cudaMemcpyToSymbol(ss::g_fe_trace, zeros, sizeof(zeros));
}
extern "C" int ss_debug_fe_trace(void* host, size_t bytes) {
    if (bytes > sizeof(ss::g_fe_trace)) bytes = sizeof(ss::g_fe_trace);
    return (int)cudaMemcpyFromSymbol(host, ss::g_fe_trace, bytes);
}
#endif
