// blend_forward.cu -- K5: per-tile front-to-back alpha blending.
//
// Restates rasterize_forward's tile loop (rasterizer/api.py:153-196) and
// forward_tile (rasterizer/kernels.py:34-109) with checkpoint_tile
// (kernels.py:112-152) folded in: one 128-thread CTA per 16x16 tile, a warp
// per 8x8 quadrant, two pixels per thread (rows r and r+4 of one column: two
// independent blend chains for ILP, sharing the dx terms, as the (lo, hi)
// lanes of packed f32x2 state).  The tile's depth-sorted list is walked in batches of
// 256 splat records staged in shared memory (each thread gathers two
// records; every thread then reads the batch with broadcast LDS.128).
// The default kernel (blend_forward_warp_kernel) has no CTA barriers: each
// quadrant warp walks the list alone, one 32-position bucket per step, the
// next bucket's records prefetched into registers, and leaves the list once
// its 64 pixels stopped (85 -> 82 us, 224 -> 219 us after 250 iterations;
// bit-identical outputs); the batched kernel serves the variant that sets
// the blend loop's contributed flags.
// Reference semantics kept:
//  - a splat is skipped when m > m_cut or alpha < alpha_min, alpha clamped
//    at alpha_max (kernels.py:14-31);
//  - the splat that drives T below t_min is blended, then the pixel stops
//    (kernels.py:78-92); n_contrib = last blended position + 1;
//  - the CTA stops when every pixel has stopped (kernels.py:96-97);
//  - (T, r, g, b) is archived before every 32nd list position
//    (kernels.py:61-67) -- only for pixels still blending, because a
//    stopped pixel has n_contrib <= that position and the backward never
//    reads its later checkpoints;
//  - image = acc + background * T (kernels.py:98-108).
// B200 addition: per (pixel, bucket) a 32-bit mask of the bucket positions
// that were blended into the pixel.  The backward replays exactly these
// pairs (identical arithmetic, so identical decisions) and skips the rest.
// Extension A15 (builder-defined): D = sum z a T in a 4th accumulator.
// The CTA also emits k_eff (kernels.py:86-87,109) and appends its
// ceil(k_eff/64) (tile, unit) entries to the splat-wise backward work list
// (a unit = two checkpoint buckets, one warp, two list positions per lane).
#include <cuda_fp16.h>

#include "common.cuh"

namespace ss {

#ifdef SS_FWD_TRACE
// diagnostics build only (tools/trace_forward.py): per-CTA (tile, smid,
// start, end) from the global timer
__device__ unsigned long long g_fwd_trace[4 * 65536];
#endif

struct PixState {
    float T, c0, c1, c2, D;
    int last;
    uint32_t bm;
    bool done, live;
};

template <bool DEPTH, bool CONTRIB>
__global__ void __launch_bounds__(128) blend_forward_kernel(
    int W, int H, int tiles_x, const uint32_t* __restrict__ tile_start,
    const uint32_t* __restrict__ tile_end, const uint32_t* __restrict__ ckpt_base,
    const uint32_t* __restrict__ pairs, const SplatRec* __restrict__ rec, float t_min, float amin,
    float amax, float bg0, float bg1, float bg2, float* __restrict__ image,
    float* __restrict__ final_t, int32_t* __restrict__ n_contrib, float* __restrict__ depth_img,
    int32_t* __restrict__ k_eff, uint8_t* __restrict__ contributed, float4* __restrict__ ckpt,
    float* __restrict__ ckpt_depth, uint32_t* __restrict__ ckpt_mask, uint2* __restrict__ work,
    int64_t work_cap, int64_t* bucket_count, const uint32_t* __restrict__ tile_order,
    uint32_t* __restrict__ tile_cost) {
    __shared__ SplatRec s_rec[256];
    __shared__ uint32_t s_id[256];
    __shared__ uint8_t s_band[256];  // bit w: the splat's blend region reaches warp w's quadrant
    __shared__ int s_hit[CONTRIB ? 256 : 1];
    __shared__ int s_kmax[4];
    __shared__ unsigned long long s_wbase;
    // CTA -> tile through the costliest-first order of ss_bin_sort (the
    // tiles' results do not depend on it); the CTA's cycles feed the next one
    PDL_WAIT();
    const int tile = tile_order ? (int)tile_order[blockIdx.x] : (int)blockIdx.x;
    const long long clk0 = clock64();
    const int t = threadIdx.x;
#ifdef SS_FWD_TRACE
    unsigned long long tr0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr0));
    uint32_t tr_iters = 0;
#endif
    const int x0 = (tile % tiles_x) * kTile, y0 = (tile / tiles_x) * kTile;
    // warp w owns the 8x8 quadrant (w & 1, w >> 1) of the tile; a thread owns
    // rows r and r + 4 of one of its columns (the two pixels share the dx terms)
    const int w = t >> 5, lane = t & 31;
    const int col = 8 * (w & 1) + (lane & 7);
    const int row0 = 8 * (w >> 1) + (lane >> 3), row1 = row0 + 4;
    const int ix = x0 + col, iy0 = y0 + row0, iy1 = y0 + row1;
    const int p0 = row0 * kTile + col, p1 = row1 * kTile + col;  // tile-local ids
    const float px = (float)ix, py0 = (float)iy0, py1 = (float)iy1;
    const uint32_t start = tile_start[tile];
    const uint32_t len = tile_end[tile] - start;
    const uint32_t cbase = ckpt_base[tile];

    // the thread's two pixels as the (lo, hi) lanes of packed f32x2 state:
    // transmittance, colour (and depth); FADD2/FMUL2/FFMA2 give per lane the
    // scalar IEEE results, so everything the backward replays is unchanged
    f32x2 T2 = pk2(1.f, 1.f), R2 = pk2(0.f, 0.f), G2 = R2, B2 = R2, D2 = R2;
    const f32x2 PY2 = pk2(py0, py1), KE2 = pk2(-0.5f * kLog2e, -0.5f * kLog2e),
                ONE2 = pk2(1.f, 1.f);
    PixState s0 = {1.f, 0.f, 0.f, 0.f, 0.f, 0, 0u, !(ix < W && iy0 < H), false};
    PixState s1 = {1.f, 0.f, 0.f, 0.f, 0.f, 0, 0u, !(ix < W && iy1 < H), false};
    auto sync_state = [&]() {  // packed -> scalar (checkpoints, outputs)
        upk2(T2, s0.T, s1.T);
        upk2(R2, s0.c0, s1.c0);
        upk2(G2, s0.c1, s1.c1);
        upk2(B2, s0.c2, s1.c2);
        if (DEPTH) upk2(D2, s0.D, s1.D);
    };
    int open_bucket = -1;
    for (uint32_t b0 = 0; b0 < len; b0 += 256) {
        if (__syncthreads_count(!(s0.done && s1.done)) == 0) break;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const uint32_t k = b0 + t + 128 * r;
            if (k < len) {
                uint32_t s = pairs[start + k];
                s_id[t + 128 * r] = s;
                const SplatRec sr = rec[s];
                s_rec[t + 128 * r] = sr;
                // 8x8 quadrants (one per warp) the splat's blend region can
                // reach: |x - mx| <= ext_x and |y - my| <= ext_y within the
                // quadrant (a square block culls small splats better than a
                // 16 x 4 band: 91 -> 86 us, 244 -> 225 us after 250 iterations)
                const float2 ext = __half22float2(*reinterpret_cast<const __half2*>(&sr.c.w));
                const bool xin0 = fabsf(sr.a.x - ((float)x0 + 3.5f)) <= ext.x + 3.5f;
                const bool xin1 = fabsf(sr.a.x - ((float)x0 + 11.5f)) <= ext.x + 3.5f;
                const bool yin0 = fabsf(sr.a.y - ((float)y0 + 3.5f)) <= ext.y + 3.5f;
                const bool yin1 = fabsf(sr.a.y - ((float)y0 + 11.5f)) <= ext.y + 3.5f;
                const uint32_t bm = (uint32_t)(xin0 && yin0) | ((uint32_t)(xin1 && yin0) << 1) |
                                    ((uint32_t)(xin0 && yin1) << 2) | ((uint32_t)(xin1 && yin1) << 3);
                s_band[t + 128 * r] = (uint8_t)bm;
                if (CONTRIB) s_hit[t + 128 * r] = 0;
            }
        }
        __syncthreads();
        const int nb = (int)min(256u, len - b0);
        for (int j0 = 0; j0 < nb; j0 += 32) {
            const int bucket = (int)((b0 + j0) >> 5);
            // close the previous bucket's blend masks, open this bucket
            if (open_bucket >= 0) {
                const size_t prev = (size_t)(cbase + open_bucket) * kTilePx;
                if (s0.live) ckpt_mask[prev + p0] = s0.bm;
                if (s1.live) ckpt_mask[prev + p1] = s1.bm;
                // n_contrib = last blended position + 1, from the closed mask
                if (s0.bm) s0.last = 32 * open_bucket + 32 - __clz(s0.bm);
                if (s1.bm) s1.last = 32 * open_bucket + 32 - __clz(s1.bm);
            }
            open_bucket = bucket;
            s0.live = !s0.done;
            s1.live = !s1.done;
            s0.bm = s1.bm = 0u;
            sync_state();
            const size_t slot = (size_t)(cbase + bucket) * kTilePx;
            if (s0.live) {
                ckpt[slot + p0] = make_float4(s0.T, s0.c0, s0.c1, s0.c2);
                if (DEPTH) ckpt_depth[slot + p0] = s0.D;
            }
            if (s1.live) {
                ckpt[slot + p1] = make_float4(s1.T, s1.c0, s1.c1, s1.c2);
                if (DEPTH) ckpt_depth[slot + p1] = s1.D;
            }
            if (__all_sync(0xffffffffu, s0.done && s1.done)) continue;  // whole warp stopped
            // the bucket's splats whose blend region reaches this warp's quadrant
            unsigned todo = __ballot_sync(0xffffffffu, j0 + lane < nb && ((s_band[j0 + lane] >> w) & 1u));
            while (todo) {
                const int j = j0 + __ffs(todo) - 1;
                const uint32_t qb = todo & (0u - todo);  // bit (b0 + j) & 31 of the masks
                todo &= todo - 1;
#ifdef SS_FWD_TRACE
                ++tr_iters;
#endif
                const float4 A = s_rec[j].a, B = s_rec[j].b, C = s_rec[j].c;
                // the two pixels share a column: dx-only terms once; then the
                // quad_finish / splat_falloff operations of both pixels packed
                const float dx = __fsub_rn(px, A.x);
                const float q0 = quad_dx0(A, dx), q1 = quad_dx1(A, dx);
                const f32x2 dy2 = sub2(PY2, pk2(A.y, A.y));
                const f32x2 m2 = fma2(mul2(pk2(B.x, B.x), dy2), dy2,
                                      fma2(pk2(q1, q1), dy2, pk2(q0, q0)));
                float m0, m1;
                upk2(m2, m0, m1);
                const bool in0 = !s0.done && !(m0 > B.z);
                const bool in1 = !s1.done && !(m1 > B.z);
                if (in0 || in1) {
                    float e0, e1, a0, a1;
                    upk2(mul2(m2, KE2), e0, e1);
                    upk2(mul2(pk2(B.y, B.y), pk2(ex2_approx(e0), ex2_approx(e1))), a0, a1);
                    const bool ok0 = in0 && !(a0 < amin), ok1 = in1 && !(a1 < amin);
                    // a pixel that does not blend gets a = 0: its state is unchanged
                    const f32x2 a2 = pk2(ok0 ? fminf(a0, amax) : 0.f, ok1 ? fminf(a1, amax) : 0.f);
                    const f32x2 w2 = mul2(a2, T2);
                    R2 = fma2(pk2(C.x, C.x), w2, R2);
                    G2 = fma2(pk2(C.y, C.y), w2, G2);
                    B2 = fma2(pk2(C.z, C.z), w2, B2);
                    if (DEPTH) D2 = fma2(pk2(B.w, B.w), w2, D2);
                    T2 = mul2(T2, sub2(ONE2, a2));
                    float T0, T1;
                    upk2(T2, T0, T1);
                    if (ok0) {
                        s0.bm |= qb;
                        if (T0 < t_min) s0.done = true;
                    }
                    if (ok1) {
                        s1.bm |= qb;
                        if (T1 < t_min) s1.done = true;
                    }
                    if (CONTRIB && (ok0 || ok1)) s_hit[j] = 1;
                }
            }
        }
        if (CONTRIB) {
            __syncthreads();
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const uint32_t k = b0 + t + 128 * r;
                if (k < len && s_hit[t + 128 * r]) contributed[s_id[t + 128 * r]] = 1;
            }
        }
    }
    if (open_bucket >= 0) {
        const size_t prev = (size_t)(cbase + open_bucket) * kTilePx;
        if (s0.live) ckpt_mask[prev + p0] = s0.bm;
        if (s1.live) ckpt_mask[prev + p1] = s1.bm;
        if (s0.bm) s0.last = 32 * open_bucket + 32 - __clz(s0.bm);
        if (s1.bm) s1.last = 32 * open_bucket + 32 - __clz(s1.bm);
    }
    sync_state();
    if (ix < W) {
        if (iy0 < H) {
            const size_t o = (size_t)iy0 * W + ix;
            final_t[o] = s0.T;
            image[3 * o] = s0.c0 + bg0 * s0.T;
            image[3 * o + 1] = s0.c1 + bg1 * s0.T;
            image[3 * o + 2] = s0.c2 + bg2 * s0.T;
            n_contrib[o] = s0.last;
            if (DEPTH) depth_img[o] = s0.D;
        }
        if (iy1 < H) {
            const size_t o = (size_t)iy1 * W + ix;
            final_t[o] = s1.T;
            image[3 * o] = s1.c0 + bg0 * s1.T;
            image[3 * o + 1] = s1.c1 + bg1 * s1.T;
            image[3 * o + 2] = s1.c2 + bg2 * s1.T;
            n_contrib[o] = s1.last;
            if (DEPTH) depth_img[o] = s1.D;
        }
    }
    int km = warp_max(max(s0.last, s1.last));
    if ((t & 31) == 0) s_kmax[t >> 5] = km;
    __syncthreads();
    const int kmax = max(max(s_kmax[0], s_kmax[1]), max(s_kmax[2], s_kmax[3]));
    if (t == 0) {
        k_eff[tile] = kmax;
        if (tile_cost) tile_cost[tile] = (uint32_t)min(clock64() - clk0, 0xffffffffll);
    }
#ifdef SS_FWD_TRACE
    __shared__ uint32_t s_iters;
    if (t == 0) s_iters = 0;
    __syncthreads();
    if ((t & 31) == 0) atomicAdd(&s_iters, tr_iters);
    __syncthreads();
    if (t == 0 && tile < 65536) {
        unsigned long long tr1;
        uint32_t smid;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr1));
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_fwd_trace[4 * tile] = s_iters;
        g_fwd_trace[4 * tile + 1] = smid;
        g_fwd_trace[4 * tile + 2] = tr0;
        g_fwd_trace[4 * tile + 3] = tr1;
    }
#endif
    const int nbk = (kmax + kUnit - 1) / kUnit;  // backward units of 64 list positions
    if (nbk > 0 && work) {
        if (t == 0)
            s_wbase = atomicAdd(reinterpret_cast<unsigned long long*>(bucket_count),
                                (unsigned long long)nbk);
        __syncthreads();
        for (int b = t; b < nbk; b += blockDim.x) {
            long long idx = (long long)s_wbase + b;
            if (idx < work_cap) work[idx] = make_uint2((uint32_t)tile, (uint32_t)b);
        }
    }
}

// Variant without CTA barriers: each quadrant warp walks the tile's list on
// its own, one 32-position bucket per step (a lane gathers one record, the
// warp's reach test and blend loop as above, records staged in the warp's
// own shared slots), the next bucket's records prefetched into registers;
// a warp whose 64 pixels all stopped leaves the list at once.  Same
// arithmetic, same per-pixel splat order: results identical to
// blend_forward_kernel.  No contributed flags (CONTRIB = false only).
template <bool DEPTH>
__global__ void __launch_bounds__(128) blend_forward_warp_kernel(
    int W, int H, int tiles_x, const uint32_t* __restrict__ tile_start,
    const uint32_t* __restrict__ tile_end, const uint32_t* __restrict__ ckpt_base,
    const uint32_t* __restrict__ pairs, const SplatRec* __restrict__ rec, float t_min, float amin,
    float amax, float bg0, float bg1, float bg2, float* __restrict__ image,
    float* __restrict__ final_t, int32_t* __restrict__ n_contrib, float* __restrict__ depth_img,
    int32_t* __restrict__ k_eff, uint8_t* __restrict__ contributed, float4* __restrict__ ckpt,
    float* __restrict__ ckpt_depth, uint32_t* __restrict__ ckpt_mask, uint2* __restrict__ work,
    int64_t work_cap, int64_t* bucket_count, const uint32_t* __restrict__ tile_order,
    uint32_t* __restrict__ tile_cost) {
    __shared__ SplatRec s_rec[4][32];
    __shared__ int s_kmax[4];
    __shared__ unsigned long long s_wbase;
    PDL_WAIT();
    const int tile = tile_order ? (int)tile_order[blockIdx.x] : (int)blockIdx.x;
    const long long clk0 = clock64();
    const int t = threadIdx.x;
    const int x0 = (tile % tiles_x) * kTile, y0 = (tile / tiles_x) * kTile;
    const int w = t >> 5, lane = t & 31;
    const int col = 8 * (w & 1) + (lane & 7);
    const int row0 = 8 * (w >> 1) + (lane >> 3), row1 = row0 + 4;
    const int ix = x0 + col, iy0 = y0 + row0, iy1 = y0 + row1;
    const int p0 = row0 * kTile + col, p1 = row1 * kTile + col;
    const float px = (float)ix, py0 = (float)iy0, py1 = (float)iy1;
    const uint32_t start = tile_start[tile];
    const uint32_t len = tile_end[tile] - start;
    const uint32_t cbase = ckpt_base[tile];
    // this warp's quadrant centre for the reach test
    const float qx = (float)(x0 + 8 * (w & 1)) + 3.5f, qy = (float)(y0 + 8 * (w >> 1)) + 3.5f;

    f32x2 T2 = pk2(1.f, 1.f), R2 = pk2(0.f, 0.f), G2 = R2, B2 = R2, D2 = R2;
    const f32x2 PY2 = pk2(py0, py1), KE2 = pk2(-0.5f * kLog2e, -0.5f * kLog2e),
                ONE2 = pk2(1.f, 1.f);
    PixState s0 = {1.f, 0.f, 0.f, 0.f, 0.f, 0, 0u, !(ix < W && iy0 < H), false};
    PixState s1 = {1.f, 0.f, 0.f, 0.f, 0.f, 0, 0u, !(ix < W && iy1 < H), false};
    auto sync_state = [&]() {
        upk2(T2, s0.T, s1.T);
        upk2(R2, s0.c0, s1.c0);
        upk2(G2, s0.c1, s1.c1);
        upk2(B2, s0.c2, s1.c2);
        if (DEPTH) upk2(D2, s0.D, s1.D);
    };
    int open_bucket = -1;
    // software pipeline: pair id two buckets ahead, record one bucket ahead
    uint32_t id_n = lane < (int)len ? pairs[start + lane] : 0u;
    uint32_t id_nn = 32 + lane < (int)len ? pairs[start + 32 + lane] : 0u;
    SplatRec r_n;
    if (lane < (int)len) r_n = rec[id_n];
    for (uint32_t b0 = 0; b0 < len; b0 += 32) {
        if (__all_sync(0xffffffffu, s0.done && s1.done)) break;  // the warp's pixels all stopped
        const SplatRec sr = r_n;
        const bool valid = b0 + lane < len;
        // next bucket's record (its id is already here), the id after that
        if (b0 + 32 + lane < len) r_n = rec[id_nn];
        id_nn = b0 + 64 + lane < len ? pairs[start + b0 + 64 + lane] : 0u;
        const int bucket = (int)(b0 >> 5);
        if (open_bucket >= 0) {
            const size_t prev = (size_t)(cbase + open_bucket) * kTilePx;
            if (s0.live) ckpt_mask[prev + p0] = s0.bm;
            if (s1.live) ckpt_mask[prev + p1] = s1.bm;
            if (s0.bm) s0.last = 32 * open_bucket + 32 - __clz(s0.bm);
            if (s1.bm) s1.last = 32 * open_bucket + 32 - __clz(s1.bm);
        }
        open_bucket = bucket;
        s0.live = !s0.done;
        s1.live = !s1.done;
        s0.bm = s1.bm = 0u;
        sync_state();
        const size_t slot = (size_t)(cbase + bucket) * kTilePx;
        if (s0.live) {
            ckpt[slot + p0] = make_float4(s0.T, s0.c0, s0.c1, s0.c2);
            if (DEPTH) ckpt_depth[slot + p0] = s0.D;
        }
        if (s1.live) {
            ckpt[slot + p1] = make_float4(s1.T, s1.c0, s1.c1, s1.c2);
            if (DEPTH) ckpt_depth[slot + p1] = s1.D;
        }
        bool reach = false;
        if (valid) {
            const float2 ext = __half22float2(*reinterpret_cast<const __half2*>(&sr.c.w));
            reach = fabsf(sr.a.x - qx) <= ext.x + 3.5f && fabsf(sr.a.y - qy) <= ext.y + 3.5f;
        }
        unsigned todo = __ballot_sync(0xffffffffu, reach);
        __syncwarp();  // the previous bucket's readers are done with the slots
        s_rec[w][lane] = sr;
        __syncwarp();
        while (todo) {
            const int j = __ffs(todo) - 1;
            const uint32_t qb = todo & (0u - todo);
            todo &= todo - 1;
            const float4 A = s_rec[w][j].a, B = s_rec[w][j].b, C = s_rec[w][j].c;
            const float dx = __fsub_rn(px, A.x);
            const float q0 = quad_dx0(A, dx), q1 = quad_dx1(A, dx);
            const f32x2 dy2 = sub2(PY2, pk2(A.y, A.y));
            const f32x2 m2 = fma2(mul2(pk2(B.x, B.x), dy2), dy2,
                                  fma2(pk2(q1, q1), dy2, pk2(q0, q0)));
            float m0, m1;
            upk2(m2, m0, m1);
            const bool in0 = !s0.done && !(m0 > B.z);
            const bool in1 = !s1.done && !(m1 > B.z);
            if (in0 || in1) {
                float e0, e1, a0, a1;
                upk2(mul2(m2, KE2), e0, e1);
                upk2(mul2(pk2(B.y, B.y), pk2(ex2_approx(e0), ex2_approx(e1))), a0, a1);
                const bool ok0 = in0 && !(a0 < amin), ok1 = in1 && !(a1 < amin);
                const f32x2 a2 = pk2(ok0 ? fminf(a0, amax) : 0.f, ok1 ? fminf(a1, amax) : 0.f);
                const f32x2 w2 = mul2(a2, T2);
                R2 = fma2(pk2(C.x, C.x), w2, R2);
                G2 = fma2(pk2(C.y, C.y), w2, G2);
                B2 = fma2(pk2(C.z, C.z), w2, B2);
                if (DEPTH) D2 = fma2(pk2(B.w, B.w), w2, D2);
                T2 = mul2(T2, sub2(ONE2, a2));
                float T0, T1;
                upk2(T2, T0, T1);
                if (ok0) {
                    s0.bm |= qb;
                    if (T0 < t_min) s0.done = true;
                }
                if (ok1) {
                    s1.bm |= qb;
                    if (T1 < t_min) s1.done = true;
                }
            }
        }
    }
    if (open_bucket >= 0) {
        const size_t prev = (size_t)(cbase + open_bucket) * kTilePx;
        if (s0.live) ckpt_mask[prev + p0] = s0.bm;
        if (s1.live) ckpt_mask[prev + p1] = s1.bm;
        if (s0.bm) s0.last = 32 * open_bucket + 32 - __clz(s0.bm);
        if (s1.bm) s1.last = 32 * open_bucket + 32 - __clz(s1.bm);
    }
    sync_state();
    if (ix < W) {
        if (iy0 < H) {
            const size_t o = (size_t)iy0 * W + ix;
            final_t[o] = s0.T;
            image[3 * o] = s0.c0 + bg0 * s0.T;
            image[3 * o + 1] = s0.c1 + bg1 * s0.T;
            image[3 * o + 2] = s0.c2 + bg2 * s0.T;
            n_contrib[o] = s0.last;
            if (DEPTH) depth_img[o] = s0.D;
        }
        if (iy1 < H) {
            const size_t o = (size_t)iy1 * W + ix;
            final_t[o] = s1.T;
            image[3 * o] = s1.c0 + bg0 * s1.T;
            image[3 * o + 1] = s1.c1 + bg1 * s1.T;
            image[3 * o + 2] = s1.c2 + bg2 * s1.T;
            n_contrib[o] = s1.last;
            if (DEPTH) depth_img[o] = s1.D;
        }
    }
    int km = warp_max(max(s0.last, s1.last));
    if (lane == 0) s_kmax[w] = km;
    __syncthreads();
    const int kmax = max(max(s_kmax[0], s_kmax[1]), max(s_kmax[2], s_kmax[3]));
    if (t == 0) {
        k_eff[tile] = kmax;
        if (tile_cost) tile_cost[tile] = (uint32_t)min(clock64() - clk0, 0xffffffffll);
    }
    const int nbk = (kmax + kUnit - 1) / kUnit;
    if (nbk > 0 && work) {
        if (t == 0)
            s_wbase = atomicAdd(reinterpret_cast<unsigned long long*>(bucket_count),
                                (unsigned long long)nbk);
        __syncthreads();
        for (int b = t; b < nbk; b += blockDim.x) {
            long long idx = (long long)s_wbase + b;
            if (idx < work_cap) work[idx] = make_uint2((uint32_t)tile, (uint32_t)b);
        }
    }
}

// replay_pixel_states (api.py:340-368) over replay_tile (kernels.py:155-178):
// advance one tile's archived pixel states from checkpoint bucket
// `from_bucket` to list position pos_to, with the forward's exact
// arithmetic (quad_finish / splat_falloff, the same skip tests), so a replay
// to k_eff reproduces the forward's final state bit for bit.  A pixel that
// stopped (T < t_min) before the bucket has no archived state there (the
// forward archives live pixels only): its state is the final one.
__global__ void __launch_bounds__(256) replay_kernel(
    int W, int H, int tiles_x, int tile, int from_bucket, int pos_to,
    const uint32_t* __restrict__ tile_start, const uint32_t* __restrict__ ckpt_base,
    const uint32_t* __restrict__ pairs, const SplatRec* __restrict__ rec,
    const float4* __restrict__ ckpt, const float* __restrict__ image,
    const float* __restrict__ final_t, const int32_t* __restrict__ n_contrib, float t_min,
    float amin, float amax, float bg0, float bg1, float bg2, float* __restrict__ out) {
    const int p = threadIdx.x, row = p >> 4, col = p & 15;
    const int x0 = (tile % tiles_x) * kTile, y0 = (tile / tiles_x) * kTile;
    const int ix = x0 + col, iy = y0 + row;
    if (ix >= W || iy >= H) return;
    const int tw = min(kTile, W - x0);
    const size_t o = (size_t)iy * W + ix;
    const int pos_from = kBucket * from_bucket;
    float T, c0, c1, c2;
    if (n_contrib[o] <= pos_from && final_t[o] < t_min) {
        T = final_t[o];
        c0 = image[3 * o] - bg0 * T;
        c1 = image[3 * o + 1] - bg1 * T;
        c2 = image[3 * o + 2] - bg2 * T;
    } else {
        const float4 s = ckpt[(size_t)(ckpt_base[tile] + from_bucket) * kTilePx + p];
        T = s.x, c0 = s.y, c1 = s.z, c2 = s.w;
    }
    const float px = (float)ix, py = (float)iy;
    const uint32_t start = tile_start[tile];
    for (int k = pos_from; k < pos_to; ++k) {
        if (T < t_min) continue;
        const SplatRec r = rec[pairs[start + k]];
        float dx, dy;
        const float m = splat_power(px, py, r.a, r.b, dx, dy);
        if (m > r.b.z) continue;
        float a = splat_falloff(m, r.b);
        if (a < amin) continue;
        a = fminf(a, amax);
        const float w = __fmul_rn(a, T);
        c0 = __fmaf_rn(r.c.x, w, c0);
        c1 = __fmaf_rn(r.c.y, w, c1);
        c2 = __fmaf_rn(r.c.z, w, c2);
        T = __fmul_rn(T, __fsub_rn(1.f, a));
    }
    float4* dst = reinterpret_cast<float4*>(out) + (row * tw + col);
    *dst = make_float4(T, c0, c1, c2);
}

cudaError_t launch_replay(const ss_camera* cam, const ss_raster_opts* o, const ss_splats* sp,
                          const ss_bins* bins, const float* image, const float* final_t,
                          const int32_t* n_contrib, const void* ckpt, int tile, int from_bucket,
                          int pos_to, float* out, cudaStream_t s) {
    const int tx = div_up(cam->width, kTile);
    replay_kernel<<<1, kTilePx, 0, s>>>(
        cam->width, cam->height, tx, tile, from_bucket, pos_to, bins->d_tile_start,
        bins->d_ckpt_base, bins->d_pair_splat, reinterpret_cast<const SplatRec*>(sp->d_rec),
        reinterpret_cast<const float4*>(ckpt), image, final_t, n_contrib, o->t_min,
        o->alpha_min, o->alpha_max, o->background[0], o->background[1], o->background[2], out);
    return cudaGetLastError();
}

cudaError_t launch_blend_forward(const ss_camera* cam, const ss_raster_opts* o,
                                 const ss_splats* sp, const ss_bins* bins, float* image,
                                 float* final_t, int32_t* n_contrib, float* depth,
                                 int32_t* k_eff, uint8_t* contributed, void* ckpt,
                                 float* ckpt_depth, uint32_t* ckpt_mask, uint32_t* work,
                                 int64_t work_cap, ss_status* st, cudaStream_t s) {
    int tx = div_up(cam->width, kTile), ty = div_up(cam->height, kTile);
    int n_tiles = tx * ty;
    const bool depthf = o->with_depth != 0;
    const bool contribf = contributed != nullptr;
    const bool ordered = bins->d_tile_order && bins->d_tile_cost && n_tiles <= SS_ORDER_MAX_TILES;
    auto args = [&](auto kern) {
        launch_pdl(kern, dim3(n_tiles), dim3(128), 0, s,
            cam->width, cam->height, tx, bins->d_tile_start, bins->d_tile_end, bins->d_ckpt_base,
            bins->d_pair_splat, reinterpret_cast<const SplatRec*>(sp->d_rec), o->t_min,
            o->alpha_min, o->alpha_max, o->background[0], o->background[1], o->background[2],
            image, final_t, n_contrib, depth, k_eff, contributed, reinterpret_cast<float4*>(ckpt),
            ckpt_depth, ckpt_mask, reinterpret_cast<uint2*>(work), work_cap, &st->bucket_count,
            ordered ? bins->d_tile_order : nullptr, ordered ? bins->d_tile_cost : nullptr);
    };
    // the per-warp kernel unless the blend loop's contributed flag is asked
    // for (or SS_FWD_CTA=1: the CTA-batched kernel, same results)
    static const bool cta = [] {
        const char* e = getenv("SS_FWD_CTA");
        return e && e[0] == '1';
    }();
    if (depthf && contribf)
        args(blend_forward_kernel<true, true>);
    else if (depthf)
        cta ? args(blend_forward_kernel<true, false>) : args(blend_forward_warp_kernel<true>);
    else if (contribf)
        args(blend_forward_kernel<false, true>);
    else
        cta ? args(blend_forward_kernel<false, false>) : args(blend_forward_warp_kernel<false>);
    return cudaGetLastError();
}

// The splats that blended at least one pixel (kernels.py:94-95), from the
// forward's per-(pixel, bucket) blend masks instead of a per-pair flag in
// the blend loop: a warp per backward work unit (tile, two buckets) of the
// forward's list; the OR of the masks of the pixels still blending at a
// bucket's start names its contributing list positions.  (The engine never
// needs this: the backward derives the same set.)
__global__ void __launch_bounds__(256) contributed_kernel(
    int W, int H, int tiles_x, const uint32_t* __restrict__ tile_start,
    const uint32_t* __restrict__ ckpt_base, const uint32_t* __restrict__ pairs,
    const int32_t* __restrict__ n_contrib, const int32_t* __restrict__ k_eff,
    const uint32_t* __restrict__ ckpt_mask, const uint2* __restrict__ work,
    const int64_t* __restrict__ work_count, int64_t work_cap, uint8_t* __restrict__ contributed) {
    const int lane = threadIdx.x & 31;
    const int64_t count = min(*work_count, work_cap);
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t it = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); it < count;
         it += nw) {
        const uint2 wk = work[it];
        const int tile = (int)wk.x, u = (int)wk.y;
        const int x0 = (tile % tiles_x) * kTile, y0 = (tile / tiles_x) * kTile;
        const int ke = k_eff[tile];
        const int kbase = u * kUnit;
        const bool two = kbase + kBucket < ke;
        const size_t slot0 = (size_t)(ckpt_base[tile] + 2 * u) * kTilePx;
        uint32_t o0 = 0u, o1 = 0u;
        int nct[kTilePx / 32];
        uint32_t m0[kTilePx / 32], m1[kTilePx / 32];
#pragma unroll
        for (int c = 0; c < kTilePx / 32; ++c) {  // every load of the unit in flight
            const int p = c * 32 + lane;
            const int ix = x0 + (p & 15), iy = y0 + (p >> 4);
            nct[c] = (ix < W && iy < H) ? n_contrib[(size_t)iy * W + ix] : 0;
            m0[c] = ckpt_mask[slot0 + p];
            m1[c] = two ? ckpt_mask[slot0 + kTilePx + p] : 0u;
        }
#pragma unroll
        for (int c = 0; c < kTilePx / 32; ++c) {
            o0 |= nct[c] > kbase ? m0[c] : 0u;
            o1 |= nct[c] > kbase + kBucket ? m1[c] : 0u;
        }
        o0 = __reduce_or_sync(0xffffffffu, o0);
        o1 = __reduce_or_sync(0xffffffffu, o1);
        const uint32_t start = tile_start[tile] + kbase;
        if ((o0 >> lane) & 1u) contributed[pairs[start + lane]] = 1;
        if ((o1 >> lane) & 1u) contributed[pairs[start + kBucket + lane]] = 1;
    }
}

cudaError_t launch_contributed(const ss_camera* cam, const ss_bins* bins, const int32_t* n_contrib,
                               const int32_t* k_eff, const uint32_t* ckpt_mask,
                               const uint32_t* work, int64_t work_cap, const ss_status* st,
                               uint8_t* contributed, int64_t n, cudaStream_t s) {
    const int tx = div_up(cam->width, kTile);
    cudaError_t e = cudaMemsetAsync(contributed, 0, (size_t)n, s);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    contributed_kernel<<<sms * 8, 256, 0, s>>>(cam->width, cam->height, tx, bins->d_tile_start,
                                                bins->d_ckpt_base, bins->d_pair_splat, n_contrib,
                                                k_eff, ckpt_mask,
                                                reinterpret_cast<const uint2*>(work),
                                                &st->bucket_count, work_cap, contributed);
    return cudaGetLastError();
}
}  // namespace ss

#ifdef SS_FWD_TRACE
extern "C" int ss_debug_fwd_trace(void* host, size_t bytes) {
    if (bytes > sizeof(ss::g_fwd_trace)) bytes = sizeof(ss::g_fwd_trace);
    return (int)cudaMemcpyFromSymbol(host, ss::g_fwd_trace, bytes);
}
#endif
