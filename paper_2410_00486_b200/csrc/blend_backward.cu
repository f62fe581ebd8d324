// blend_backward.cu -- K7: CaRtGS splat-wise backward on B200.
//
// Restates backward_splatwise (rasterizer/api.py:275-337) over
// backward_splat_tile / _splat_bucket_inner (rasterizer/kernels.py:271-373).
// The reference's work unit is a (tile, bucket of 32 list positions) pair
// that restores pixel states from the bucket's checkpoint and lets each
// splat accumulate its gradient privately over the tile's pixels.  On B200
// that unit is one WARP, lane i owning list position 32 b + i:
//
//   - the pixels still blending at the bucket start (n_contrib > 32 b) are
//     compacted into a per-warp shared-memory list with their gradient,
//     g . image and checkpoint state;
//   - the pixel states then flow down the warp as a diagonal wavefront:
//     at step t lane i handles list pixel t - i, receiving that pixel's
//     state after splats 32b..32b+i-1 from lane i-1 by __shfl_up_sync, so
//     every (pixel, splat) term sees exactly the state the reference's
//     sequential replay produces (kernels.py:322-333);
//   - each lane keeps its splat's 9 screen-space gradients in registers
//     (no per-pixel atomics) and adds them to g2d with one red.add row per
//     (tile, splat) at the end -- the float32 counterpart of the
//     reference's ordered per-tile merge (api.py:331-336).
//
// Pixel state carried between lanes: (T, G) with G = g . c_acc, the
// gradient-weighted accumulated colour.  The reference's dL/dalpha
//   sum_c (rgb_c T - (image_c - c_acc_c)/(1 - a)) g_c     (kernels.py:344-352)
// equals T (g . rgb) - (g . image - G_after) / (1 - a), so two floats move
// per shuffle instead of four.  Warps are persistent and pull work units
// from the list the forward appended.
#include "common.cuh"

namespace ss {

constexpr int kBwdWarps = 2;

// The wavefront carries TWO pixels per lane and step, as the (lo, hi) lanes
// of packed f32x2 values (FADD2/FMUL2/FFMA2: per lane the scalar IEEE
// result, so alpha is recomputed with exactly the forward's operations).
// The two pixel chains are independent, which doubles the work between the
// shuffles and halves the number of wavefront steps.
struct SplatAcc2 {  // one splat's partial sums, (pixel a, pixel b) lanes
    f32x2 r0, r1, r2, rz, s_da, s_dx, s_dy, s_xx, s_xy, s_yy;
};
struct SplatP2 {  // one splat's record fields, duplicated into both lanes
    f32x2 mx, my, c0, c1x2, c2, sig, cr, cg, cb, z;
};

__device__ __forceinline__ SplatP2 splat_p2(const float4& A, const float4& B, const float4& C) {
    SplatP2 p;
    p.mx = pk2(A.x, A.x);
    p.my = pk2(A.y, A.y);
    p.c0 = pk2(A.z, A.z);
    p.c1x2 = pk2(A.w, A.w);
    p.c2 = pk2(B.x, B.x);
    p.sig = pk2(B.y, B.y);
    p.cr = pk2(C.x, C.x);
    p.cg = pk2(C.y, C.y);
    p.cb = pk2(C.z, C.z);
    p.z = pk2(B.w, B.w);
    return p;
}

// One splat applied to a pixel pair.  `ba` / `bb` are the forward's blend
// mask bits of the two pixels; a pair that was not blended gets a = 0, which
// leaves T and G bit-exactly unchanged and contributes nothing, so the term
// runs branch-free.
template <bool DEPTH, bool CLAMP>
__device__ __forceinline__ void bwd_term2(uint32_t ba, uint32_t bb, f32x2 px, f32x2 py, f32x2 gx,
                                          f32x2 gy, f32x2 gz, f32x2 gw, f32x2 gd,
                                          const SplatP2& S, float amax, f32x2& T, f32x2& G,
                                          SplatAcc2& q) {
    // splat_power / splat_falloff (common.cuh) per lane: same operations,
    // same rounding as the forward's blend decision
    const f32x2 dx = sub2(px, S.mx), dy = sub2(py, S.my);
    const f32x2 m = fma2(mul2(S.c2, dy), dy, fma2(mul2(S.c1x2, dx), dy, mul2(mul2(S.c0, dx), dx)));
    float e0, e1;
    upk2(mul2(m, pk2(-0.5f * kLog2e, -0.5f * kLog2e)), e0, e1);
    float a0, a1;
    upk2(mul2(S.sig, pk2(ex2_approx(e0), ex2_approx(e1))), a0, a1);
    // CLAMP == false: no splat of the unit has sigma >= alpha_max, so the
    // clamp is the identity
    if (CLAMP) {
        a0 = fminf(a0, amax);
        a1 = fminf(a1, amax);
    }
    a0 = ba ? a0 : 0.f;
    a1 = bb ? a1 : 0.f;
    const f32x2 a = pk2(a0, a1);
    const f32x2 w = mul2(a, T);
    f32x2 grgb = fma2(gz, S.cb, fma2(gy, S.cg, mul2(gx, S.cr)));
    if (DEPTH) {
        grgb = fma2(gd, S.z, grgb);
        q.rz = fma2(w, gd, q.rz);
    }
    const f32x2 Gafter = fma2(grgb, w, G);
    q.r0 = fma2(w, gx, q.r0);
    q.r1 = fma2(w, gy, q.r1);
    q.r2 = fma2(w, gz, q.r2);
    // alpha-path gradient (kernels.py:342-364):
    //   dL/da = T (g . rgb) - (g . image - G_after) / (1 - a)
    // zero when clamped (and when not blended: a = 0)
    const f32x2 om = sub2(pk2(1.f, 1.f), a);
    float o0, o1;
    upk2(om, o0, o1);
    const f32x2 dal = fma2(T, grgb, mul2(sub2(Gafter, gw), pk2(rcp_approx(o0), rcp_approx(o1))));
    const f32x2 da =
        mul2(dal, CLAMP ? pk2(a0 != amax ? a0 : 0.f, a1 != amax ? a1 : 0.f) : a);
    const f32x2 tx = mul2(da, dx), ty = mul2(da, dy);
    q.s_da = add2(q.s_da, da);
    q.s_dx = add2(q.s_dx, tx);
    q.s_dy = add2(q.s_dy, ty);
    q.s_xx = fma2(tx, dx, q.s_xx);
    q.s_xy = fma2(tx, dy, q.s_xy);
    q.s_yy = fma2(ty, dy, q.s_yy);
    T = mul2(T, om);
    G = Gafter;
}

__device__ __forceinline__ float hsum(f32x2 v) {
    float lo, hi;
    upk2(v, lo, hi);
    return lo + hi;
}

// Commit one splat's sums as its 9 (10) screen-space gradients.
template <int NC>
__device__ __forceinline__ void bwd_commit(const SplatAcc2& q, const float4& A, const float4& B,
                                           float* __restrict__ row) {
    const float c1 = 0.5f * A.w;
    const float s_dx = hsum(q.s_dx), s_dy = hsum(q.s_dy);
    float acc[NC];
    acc[0] = hsum(q.r0);
    acc[1] = hsum(q.r1);
    acc[2] = hsum(q.r2);
    acc[3] = A.z * s_dx + c1 * s_dy;
    acc[4] = c1 * s_dx + B.x * s_dy;
    acc[5] = -0.5f * hsum(q.s_xx);
    acc[6] = -hsum(q.s_xy);
    acc[7] = -0.5f * hsum(q.s_yy);
    acc[8] = hsum(q.s_da) / B.y;
    if (NC == 10) acc[NC - 1] = hsum(q.rz);
#pragma unroll
    for (int c = 0; c < NC; ++c)
        if (acc[c] != 0.f) atomicAdd(row + c, acc[c]);
}

// shfl.up by one lane inside each half-warp (the two buckets' chains)
__device__ __forceinline__ f32x2 shfl_up2(f32x2 v) {
    float lo, hi;
    upk2(v, lo, hi);
    return pk2(__shfl_up_sync(0xffffffffu, lo, 1, 16), __shfl_up_sync(0xffffffffu, hi, 1, 16));
}

// Per-warp compacted pixel list, pair-interleaved so that one pair's values
// load as ready-made f32x2 operands: pixel j of pair jp = j >> 1 sits in lane
// (j & 1) of each packed field.
struct BwdList {
    float xy[2 * kTilePx];         // per pair: x, x', y, y'
    float ga[2 * kTilePx];         // per pair: gx, gx', gy, gy'  (16 B per pair: the
    float gb[2 * kTilePx];         // per pair: gz, gz', gw, gw'   step's loads are contiguous)
    float s[kTilePx * 2];          // per pair: T0, T0', G0, G0' (state at the unit start)
    float s2[kTilePx * 2];         // the same at the second bucket's start
    uint32_t ma[kTilePx];          // first bucket's blend masks (pair = uint2)
    uint32_t mb[kTilePx];          // second bucket's (each half-warp loads only its own)
};

// Diagonal wavefronts over the warp's compacted pixel pairs, one per half-
// warp: lanes 0-15 carry the unit's first bucket, lanes 16-31 the second,
// each chain starting from its own bucket's checkpoint, so the ramp is 15
// steps instead of 31.  Lane i applies list positions 2i and 2i+1 to each
// pixel pair in turn.  Returns the lane's blended-bit summary (bit 0: first
// splat blended somewhere, bit 1: second).
template <bool DEPTH, bool CLAMP>
__device__ __forceinline__ uint32_t bwd_wavefront(int npair, int lane, bool hi, int sh,
                                                  const BwdList& L, const float* __restrict__ sD,
                                                  const SplatP2& S0, const SplatP2& S1,
                                                  float amax, SplatAcc2& q0, SplatAcc2& q1) {
    f32x2 T = pk2(0.f, 0.f), G = T;
    uint32_t seen = 0u;
    const int steps = npair + 15;
    const int hl = lane & 15;
    const uint2* M2 = reinterpret_cast<const uint2*>(hi ? L.mb : L.ma);
    const float4* S4 = reinterpret_cast<const float4*>(hi ? L.s2 : L.s);
    const float4* GA = reinterpret_cast<const float4*>(L.ga);
    const float4* GB = reinterpret_cast<const float4*>(L.gb);
    const float4* XY = reinterpret_cast<const float4*>(L.xy);
#pragma unroll 2
    for (int st = 0; st < steps; ++st) {
        T = shfl_up2(T);
        G = shfl_up2(G);
        // lanes outside the diagonal run with bits = 0 on pair 0 (a = 0:
        // nothing changes, T and G stay finite), so the only branch is
        // warp-uniform -- no divergence bookkeeping per step
        const int j = st - hl;
        const bool inr = (unsigned)j < (unsigned)npair;
        const int jj = inr ? j : 0;
        const uint2 m = M2[jj];
        if (hl == 0 && inr) {
            const float4 s = S4[jj];
            T = pk2(s.x, s.y);
            G = pk2(s.z, s.w);
        }
        const uint32_t ba = inr ? (m.x >> sh) & 3u : 0u;
        const uint32_t bb = inr ? (m.y >> sh) & 3u : 0u;
        // (no warp-uniform skip: a branch here would split the unrolled steps)
        seen |= ba | bb;
        const float4 xy = XY[jj];
        const float4 g0 = GA[jj], g1 = GB[jj];
        const f32x2 px = pk2(xy.x, xy.y), py = pk2(xy.z, xy.w);
        const f32x2 gx = pk2(g0.x, g0.y), gy = pk2(g0.z, g0.w), gz = pk2(g1.x, g1.y),
                    gw = pk2(g1.z, g1.w);
        f32x2 gd = pk2(0.f, 0.f);
        if (DEPTH) {
            const float2 d = reinterpret_cast<const float2*>(sD)[jj];
            gd = pk2(d.x, d.y);
        }
        bwd_term2<DEPTH, CLAMP>(ba & 1u, bb & 1u, px, py, gx, gy, gz, gw, gd, S0, amax, T, G, q0);
        bwd_term2<DEPTH, CLAMP>(ba & 2u, bb & 2u, px, py, gx, gy, gz, gw, gd, S1, amax, T, G, q1);
    }
    return seen;
}

template <bool DEPTH>
__global__ void __launch_bounds__(32 * kBwdWarps) backward_splat_kernel(
    int W, int H, int tiles_x, const uint32_t* __restrict__ tile_start,
    const uint32_t* __restrict__ ckpt_base, const int32_t* __restrict__ k_eff,
    const uint32_t* __restrict__ pairs, const SplatRec* __restrict__ rec, float amax,
    const float* __restrict__ image, const float* __restrict__ grad_image,
    const float4* __restrict__ pixgrad, const float* __restrict__ depth_img,
    const float* __restrict__ grad_depth, const int32_t* __restrict__ n_contrib,
    const float4* __restrict__ ckpt, const float* __restrict__ ckpt_depth,
    const uint32_t* __restrict__ ckpt_mask, const uint2* __restrict__ work,
    const int64_t* __restrict__ work_count, int64_t work_cap, uint32_t* work_counter,
    float* __restrict__ g2d, uint8_t* __restrict__ contributed, int n_tiles) {
    constexpr int NC = DEPTH ? 10 : 9;
    // per-warp compacted pixel list: gradient side (g, g . image), state at
    // the unit start (T0, G0), coordinates, the two buckets' blend masks,
    // depth gradient
    __shared__ BwdList sL[kBwdWarps];
    __shared__ float sD[DEPTH ? kBwdWarps : 1][DEPTH ? kTilePx : 1];
    PDL_WAIT();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const bool hi = lane >= 16;            // lane's splats live in the second bucket
    const int sh = (2 * lane) & 31;        // their bit pair in that bucket's mask
    const int64_t count = min(*work_count, work_cap);
    // schedule built by bwd_schedule_kernel (mode 0: the forward's list)
    const uint32_t mode = work_counter[1];
    const uint32_t mu = mode >> 1;
    const uint32_t* sched_start =
        reinterpret_cast<const uint32_t*>(work) + (2 * work_cap - (n_tiles + (int64_t)mu + 2));
    const uint32_t* sched_tiles = sched_start + mu + 1;

    for (;;) {
        uint32_t item = 0;
        if (lane == 0) item = atomicAdd(work_counter, 1u);
        item = __shfl_sync(0xffffffffu, item, 0);
        if ((int64_t)item >= count) break;
        int tile, u;
        if (mode & 1u) {
            uint32_t lo = 0, hi_ = mu;  // largest u with start[u] <= item
            while (hi_ - lo > 1) {
                const uint32_t mid = (lo + hi_) >> 1;
                if (sched_start[mid] <= item) lo = mid;
                else hi_ = mid;
            }
            u = (int)lo;
            tile = (int)sched_tiles[item - sched_start[lo]];
        } else {
            const uint2 wk = work[item];
            tile = (int)wk.x;
            u = (int)wk.y;
        }
        const int x0 = (tile % tiles_x) * kTile, y0 = (tile / tiles_x) * kTile;
        const uint32_t start = tile_start[tile];
        const int ke = k_eff[tile];
        const int kbase = u * kUnit;
        const int k0 = kbase + 2 * lane, k1 = k0 + 1;
        uint32_t s0 = 0, s1 = 0;
        float4 A0 = make_float4(0.f, 0.f, 0.f, 0.f), B0 = make_float4(0.f, 1.f, -1.f, 0.f),
               C0 = make_float4(0.f, 0.f, 0.f, 0.f);
        float4 A1 = A0, B1 = B0, C1 = C0;
        if (k0 < ke) {
            s0 = pairs[start + k0];
            const SplatRec r = rec[s0];
            A0 = r.a;
            B0 = r.b;
            C0 = r.c;
        }
        if (k1 < ke) {
            s1 = pairs[start + k1];
            const SplatRec r = rec[s1];
            A1 = r.a;
            B1 = r.b;
            C1 = r.c;
        }
        // ---- compact the pixels that blended any splat of this unit
        const size_t slot0 = (size_t)(ckpt_base[tile] + 2 * u) * kTilePx;
        // the lane's 8 pixels' n_contrib and masks, all loads in flight
        // together (the records of the active ones follow per pixel)
        uint32_t mk0[kTilePx / 32], mk1[kTilePx / 32];
        {
            int nct[kTilePx / 32];
#pragma unroll
            for (int c = 0; c < kTilePx / 32; ++c) {
                const int p = c * 32 + lane;
                const int ix = x0 + (p & 15), iy = y0 + (p >> 4);
                nct[c] = (ix < W && iy < H) ? n_contrib[(size_t)iy * W + ix] : 0;
            }
#pragma unroll
            for (int c = 0; c < kTilePx / 32; ++c) {
                const int p = c * 32 + lane;
                // a bucket's mask exists for pixels still blending at its start
                mk0[c] = nct[c] > kbase ? ckpt_mask[slot0 + p] : 0u;
                mk1[c] = nct[c] > kbase + kBucket ? ckpt_mask[slot0 + kTilePx + p] : 0u;
            }
        }
        int nact = 0;
#pragma unroll
        for (int c = 0; c < kTilePx / 32; ++c) {
            const int p = c * 32 + lane;
            const int ix = x0 + (p & 15), iy = y0 + (p >> 4);
            const size_t o = (size_t)iy * W + ix;
            const uint32_t m0 = mk0[c], m1 = mk1[c];
            const bool act = (m0 | m1) != 0u;
            const unsigned bal = __ballot_sync(0xffffffffu, act);
            if (act) {
                const int pos = nact + __popc(bal & lanemask_lt());
                float4 pg;
                if (pixgrad) {
                    pg = pixgrad[o];
                } else {
                    pg.x = grad_image[3 * o];
                    pg.y = grad_image[3 * o + 1];
                    pg.z = grad_image[3 * o + 2];
                    pg.w = pg.x * image[3 * o] + pg.y * image[3 * o + 1] + pg.z * image[3 * o + 2];
                }
                const float4 ck = ckpt[slot0 + p];
                float G0 = pg.x * ck.y + pg.y * ck.z + pg.z * ck.w;
                if (DEPTH) {
                    const float gd = grad_depth ? grad_depth[o] : 0.f;
                    if (!pixgrad) pg.w += gd * depth_img[o];
                    G0 += gd * ckpt_depth[slot0 + p];
                    sD[wid][pos] = gd;
                }
                // state at the second bucket's start (only pixels still
                // blending there have that checkpoint; the others get an
                // inert finite state: their second-bucket bits are 0)
                float T1 = 0.f, G1 = 0.f;
                if (m1 != 0u) {
                    const float4 c2 = ckpt[slot0 + kTilePx + p];
                    T1 = c2.x;
                    G1 = pg.x * c2.y + pg.y * c2.z + pg.z * c2.w;
                    if (DEPTH)
                        G1 += (grad_depth ? grad_depth[o] : 0.f) * ckpt_depth[slot0 + kTilePx + p];
                }
                BwdList& L = sL[wid];
                const int ps = (pos >> 1) * 4 + (pos & 1);  // pair-interleaved slots
                L.ga[ps] = pg.x;
                L.ga[ps + 2] = pg.y;
                L.gb[ps] = pg.z;
                L.gb[ps + 2] = pg.w;
                L.s[ps] = ck.x;
                L.s[ps + 2] = G0;
                L.s2[ps] = T1;
                L.s2[ps + 2] = G1;
                L.ma[pos] = m0;
                L.mb[pos] = m1;
                L.xy[ps] = (float)ix;
                L.xy[ps + 2] = (float)iy;
            }
            nact += __popc(bal);
        }
        // odd count: pad the last pair with an inert pixel (no blend bits,
        // zero gradient, finite state)
        if ((nact & 1) && lane == 0) {
            BwdList& L = sL[wid];
            const int ps = (nact >> 1) * 4 + 1;
            L.ga[ps] = L.ga[ps + 2] = L.gb[ps] = L.gb[ps + 2] = 0.f;
            L.s[ps] = 1.f;
            L.s[ps + 2] = 0.f;
            L.s2[ps] = 1.f;
            L.s2[ps + 2] = 0.f;
            L.ma[nact] = L.mb[nact] = 0u;
            L.xy[ps] = L.xy[ps + 2] = 0.f;
            if (DEPTH) sD[wid][nact] = 0.f;
        }
        __syncwarp();
        // ---- diagonal wavefront over the active pixel pairs; lane i applies
        // list positions 2i and 2i+1 to each pair in turn.
        // Per-splat sums; the splat-constant factors (conic, 1/sigma, -1/2)
        // are applied once at the end:
        //   d mean  = (c0 S_dx + c1 S_dy, c1 S_dx + c2 S_dy),  S_d. = sum da d.
        //   d conic = -1/2 (S_dxdx, 2 S_dxdy, S_dydy),        d sigma = S_da / sigma
        const f32x2 z2 = pk2(0.f, 0.f);
        SplatAcc2 q0 = {z2, z2, z2, z2, z2, z2, z2, z2, z2, z2}, q1 = q0;
        const SplatP2 S0 = splat_p2(A0, B0, C0), S1 = splat_p2(A1, B1, C1);
        const int npair = (nact + 1) >> 1;
        uint32_t seen;
        // the clamp at alpha_max can only bind for splats with sigma >= alpha_max
        const bool clamp = __any_sync(0xffffffffu, (k0 < ke && B0.y >= amax * 0.999999f) ||
                                                       (k1 < ke && B1.y >= amax * 0.999999f));
        if (clamp)
            seen = bwd_wavefront<DEPTH, true>(npair, lane, hi, sh, sL[wid],
                                              DEPTH ? sD[wid] : nullptr, S0, S1, amax, q0, q1);
        else
            seen = bwd_wavefront<DEPTH, false>(npair, lane, hi, sh, sL[wid],
                                               DEPTH ? sD[wid] : nullptr, S0, S1, amax, q0, q1);
        if (k0 < ke) {
            bwd_commit<NC>(q0, A0, B0, g2d + (size_t)s0 * NC);
            if (contributed && (seen & 1u)) contributed[s0] = 1;
        }
        if (k1 < ke) {
            bwd_commit<NC>(q1, A1, B1, g2d + (size_t)s1 * NC);
            if (contributed && (seen & 2u)) contributed[s1] = 1;
        }
        __syncwarp();
    }
}

// Longest-units-first schedule.  A unit's size is roughly the number of
// pixels still blending at its first bucket, so earlier units of a tile are
// larger, and tiles with more units are the deeper ones.  Handing units out
// unit-index-major with the tiles of each index in descending unit count
// approximates longest-processing-time-first and shortens the tail of the
// persistent backward.  One CTA builds it from k_eff: tiles counting-sorted
// by unit count, descending (S), and start[u] = sum over u' < u of #tiles
// with more than u' units; item c is unit u (largest u with start[u] <= c)
// of tile S[c - start[u]].  Written at the end of the work buffer (past the
// forward's list); the mode word (high half of the status block's counter
// word) = 1 | max_units << 1, or 0 to keep the forward's list (more than
// kMaxUnits units in a tile, too many tiles, or no room).
constexpr int kMaxUnits = 1024;
constexpr int kSchedTiles = 16384;  // 4K frames at 16 px tiles fit

__global__ void __launch_bounds__(1024) bwd_schedule_kernel(uint32_t* counter,
                                                            const int32_t* __restrict__ k_eff,
                                                            int n_tiles, uint32_t* __restrict__ wl,
                                                            int64_t wl_cap,
                                                            const int64_t* __restrict__ total) {
    __shared__ uint32_t h[kMaxUnits + 1];
    __shared__ uint16_t s_nb[kSchedTiles];
    __shared__ uint32_t s_max;
    const int t = threadIdx.x;
    if (n_tiles > kSchedTiles) {
        if (t == 0) counter[1] = 0u;
        return;
    }
    for (int v = t; v <= kMaxUnits; v += blockDim.x) h[v] = 0u;
    if (t == 0) s_max = 0u;
#pragma unroll 8
    for (int q = t; q < n_tiles; q += blockDim.x)  // independent loads, all in flight
        s_nb[q] = (uint16_t)min((k_eff[q] + kUnit - 1) / kUnit, 65535);
    __syncthreads();
    uint32_t m = 0;
    for (int q = t; q < n_tiles; q += blockDim.x) {
        const uint32_t nb = s_nb[q];
        m = max(m, nb);
        if (nb <= kMaxUnits) atomicAdd(&h[nb], 1u);
    }
    atomicMax(&s_max, m);
    __syncthreads();
    const uint32_t mu = s_max;
    const int64_t off = wl_cap - ((int64_t)n_tiles + mu + 2);
    if (mu > (uint32_t)kMaxUnits || off < 2 * min(*total, wl_cap / 2)) {
        if (t == 0) counter[1] = 0u;  // keep the forward's list
        return;
    }
    uint32_t* start = wl + off;    // [mu + 1]
    uint32_t* S = start + mu + 1;  // [n_tiles]
    if (t == 0) {
        uint32_t above = 0;
        for (int v = (int)mu; v >= 0; --v) {  // h[v] -> #tiles with more than v units
            const uint32_t c = h[v];           //         = first position of bucket v in S
            h[v] = above;
            above += c;
        }
        uint32_t pre = 0;
        for (uint32_t u = 0; u < mu; ++u) {
            start[u] = pre;
            pre += h[u];
        }
        start[mu] = pre;
    }
    __syncthreads();
    for (int q = t; q < n_tiles; q += blockDim.x) {
        const uint32_t nb = s_nb[q];
        if (nb != 0) S[atomicAdd(&h[nb], 1u)] = (uint32_t)q;
    }
    __syncthreads();
    if (t == 0) {
        __threadfence();
        counter[1] = 1u | (mu << 1);
    }
}

__global__ void bwd_clear_kernel(float* __restrict__ g2d, int64_t nf, uint8_t* contributed,
                                 int64_t n, uint32_t* counter) {
    PDL_WAIT();
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    if (i == 0) *counter = 0u;
    const int64_t nf4 = (reinterpret_cast<uintptr_t>(g2d) & 15) ? 0 : nf / 4;
    float4* g4 = reinterpret_cast<float4*>(g2d);
    for (int64_t k = i; k < nf4; k += stride) g4[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t k = nf4 * 4 + i; k < nf; k += stride) g2d[k] = 0.f;
    if (contributed)
        for (int64_t k = i; k < n; k += stride) contributed[k] = 0;
}

cudaError_t launch_backward_schedule(const ss_camera* cam, const int32_t* k_eff, uint32_t* work,
                                     int64_t work_cap, ss_status* st, cudaStream_t s) {
    const int tx = div_up(cam->width, kTile), ty = div_up(cam->height, kTile);
    uint32_t* counter = reinterpret_cast<uint32_t*>(&st->reserved);
    bwd_schedule_kernel<<<1, 1024, 0, s>>>(counter, k_eff, tx * ty, work, 2 * work_cap,
                                          &st->bucket_count);
    return cudaGetLastError();
}

cudaError_t launch_backward_splat(const ss_camera* cam, const ss_raster_opts* o,
                                  const ss_splats* sp, const ss_bins* bins, const float* image,
                                  const float* grad_image, const float4* pixgrad,
                                  const float* depth, const float* grad_depth,
                                  const int32_t* n_contrib, const int32_t* k_eff, const void* ckpt,
                                  const float* ckpt_depth, const uint32_t* ckpt_mask,
                                  const uint32_t* work, int64_t work_cap, int64_t n, float* g2d,
                                  uint8_t* contributed, const ss_status* st, uint32_t* counter,
                                  cudaStream_t s) {
    const bool depthf = o->with_depth != 0;
    const int ncol = depthf ? 10 : 9;
    // one launch clears the gradient rows, the contributed marks and the
    // work-unit counter
    int tx = div_up(cam->width, kTile), ty = div_up(cam->height, kTile);
    launch_pdl(bwd_clear_kernel, dim3(div_up(n * ncol > 4 ? n * ncol / 4 : 1, 256)), dim3(256),
               0, s, g2d, (int64_t)n * ncol, contributed, n, counter);
    const int threads = 32 * kBwdWarps;
    const size_t smem = 0;
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    auto go = [&](auto kern) -> cudaError_t {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
        if (per_sm < 1) per_sm = 1;
        launch_pdl(kern, dim3(sms * per_sm), dim3(threads), smem, s,
            cam->width, cam->height, tx, bins->d_tile_start, bins->d_ckpt_base, k_eff,
            bins->d_pair_splat, reinterpret_cast<const SplatRec*>(sp->d_rec), o->alpha_max, image,
            grad_image, pixgrad, depth, grad_depth, n_contrib,
            reinterpret_cast<const float4*>(ckpt), ckpt_depth, ckpt_mask,
            reinterpret_cast<const uint2*>(work), &st->bucket_count, work_cap, counter, g2d,
            contributed, tx * ty);
        return cudaGetLastError();
    };
    return depthf ? go(backward_splat_kernel<true>) : go(backward_splat_kernel<false>);
}

}  // namespace ss
