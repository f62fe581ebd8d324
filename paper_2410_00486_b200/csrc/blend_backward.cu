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
//
// Three kernels share this structure: backward_quad_kernel (default) runs
// one chain per 8x8 quadrant of the tile over only the positions that
// quadrant blended; backward_splat_kernel (SS_BWD_UNIT=1) one chain per
// bucket over the whole tile; backward_sparse_kernel (SS_BWD_SPARSE=1)
// evaluates only the blended pairs in two phases.
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
    float mxs, c0s, c1x2s;  // the dx-only terms are shared by a pair (one column)
};

__device__ __forceinline__ SplatP2 splat_p2(const float4& A, const float4& B, const float4& C) {
    SplatP2 p;
    p.mxs = A.x;
    p.c0s = A.z;
    p.c1x2s = A.w;
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

// One splat applied to a pixel pair -- two pixels of one column, rows y and
// y + 1 (the forward also shares a column's dx-only terms between its two
// pixels).  `ba` / `bb` are the forward's blend mask bits of the two pixels;
// a pair that was not blended gets a = 0, which leaves T and G bit-exactly
// unchanged and contributes nothing, so the term runs branch-free.
template <bool DEPTH, bool CLAMP>
__device__ __forceinline__ void bwd_term2(uint32_t ba, uint32_t bb, float pxs, f32x2 py, f32x2 gx,
                                          f32x2 gy, f32x2 gz, f32x2 gw, f32x2 gd,
                                          const SplatP2& S, float amax, f32x2& T, f32x2& G,
                                          SplatAcc2& q) {
    // splat_power / splat_falloff (common.cuh) per lane: the forward's
    // operations and rounding (quad_dx0 / quad_dx1 once for the column)
    const float dxs = __fsub_rn(pxs, S.mxs);
    const float q0s = __fmul_rn(__fmul_rn(S.c0s, dxs), dxs), q1s = __fmul_rn(S.c1x2s, dxs);
    const f32x2 dx = pk2(dxs, dxs), dy = sub2(py, S.my);
    const f32x2 m = fma2(mul2(S.c2, dy), dy, fma2(pk2(q1s, q1s), dy, pk2(q0s, q0s)));
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

// shfl.up by one lane across the warp (chains as lane segments)
__device__ __forceinline__ f32x2 shfl_up2w(f32x2 v) {
    float lo, hi;
    upk2(v, lo, hi);
    return pk2(__shfl_up_sync(0xffffffffu, lo, 1), __shfl_up_sync(0xffffffffu, hi, 1));
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
        const float4 xy = XY[jj];  // (x, x, y, y + 1): one column
        const float4 g0 = GA[jj], g1 = GB[jj];
        const float px = xy.x;
        const f32x2 py = pk2(xy.z, xy.w);
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
    for (;;) {
        uint32_t item = 0;
        if (lane == 0) item = atomicAdd(work_counter, 1u);
        item = __shfl_sync(0xffffffffu, item, 0);
        if ((int64_t)item >= count) break;
        // (tile, unit) in bwd_schedule_kernel's longest-first order
        const uint2 wk = work[item];
        const int tile = (int)wk.x, u = (int)wk.y;
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
        // pairs = the two pixels of one column in rows 2c and 2c + 1 (lanes l and
        // l + 16 of group c); a pair is kept when either pixel blended a splat of
        // the unit, its other pixel then rides along inert (no blend bits, zero
        // gradient, finite state)
        int npair = 0;
#pragma unroll
        for (int c = 0; c < kTilePx / 32; ++c) {
            const int p = c * 32 + lane;
            const int ix = x0 + (p & 15), iy = y0 + (p >> 4);
            const size_t o = (size_t)iy * W + ix;
            const uint32_t m0 = mk0[c], m1 = mk1[c];
            const bool act = (m0 | m1) != 0u;
            const int partner = __shfl_xor_sync(0xffffffffu, (int)act, 16);  // every lane
            const bool pact = act || partner;
            const unsigned bal = __ballot_sync(0xffffffffu, pact) & 0xffffu;
            if (pact) {
                const int pr = npair + __popc(bal & ((1u << (lane & 15)) - 1u));
                const int hi = lane >> 4;  // the pair's lane: row 2c (lo) or 2c + 1 (hi)
                float4 pg = make_float4(0.f, 0.f, 0.f, 0.f);
                float4 ck = make_float4(1.f, 0.f, 0.f, 0.f);
                float G0 = 0.f, T1 = 1.f, G1 = 0.f, gd = 0.f;
                if (act) {
                    if (pixgrad) {
                        pg = pixgrad[o];
                    } else {
                        pg.x = grad_image[3 * o];
                        pg.y = grad_image[3 * o + 1];
                        pg.z = grad_image[3 * o + 2];
                        pg.w = pg.x * image[3 * o] + pg.y * image[3 * o + 1] +
                               pg.z * image[3 * o + 2];
                    }
                    ck = ckpt[slot0 + p];
                    G0 = pg.x * ck.y + pg.y * ck.z + pg.z * ck.w;
                    if (DEPTH) {
                        gd = grad_depth ? grad_depth[o] : 0.f;
                        if (!pixgrad) pg.w += gd * depth_img[o];
                        G0 += gd * ckpt_depth[slot0 + p];
                    }
                    // state at the second bucket's start (only pixels still
                    // blending there have that checkpoint; the others get an
                    // inert finite state: their second-bucket bits are 0)
                    if (m1 != 0u) {
                        const float4 c2 = ckpt[slot0 + kTilePx + p];
                        T1 = c2.x;
                        G1 = pg.x * c2.y + pg.y * c2.z + pg.z * c2.w;
                        if (DEPTH) G1 += gd * ckpt_depth[slot0 + kTilePx + p];
                    }
                }
                if (DEPTH) sD[wid][2 * pr + hi] = gd;
                BwdList& L = sL[wid];
                const int ps = pr * 4 + hi;  // pair-interleaved slots
                L.ga[ps] = pg.x;
                L.ga[ps + 2] = pg.y;
                L.gb[ps] = pg.z;
                L.gb[ps + 2] = pg.w;
                L.s[ps] = ck.x;
                L.s[ps + 2] = G0;
                L.s2[ps] = T1;
                L.s2[ps + 2] = G1;
                L.ma[2 * pr + hi] = m0;
                L.mb[2 * pr + hi] = m1;
                L.xy[ps] = (float)ix;
                L.xy[ps + 2] = (float)iy;
            }
            npair += __popc(bal);
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

// --------------------------------------------------------------------------
// Quadrant chains (default).  A pixel of the tile only blends the splats
// whose blend region reaches its 8x8 quadrant, and at the bench workload a
// quadrant's pixels together blend ~22 of a unit's 64 list positions (the
// forward iterates per quadrant too).  The unit is therefore split into one
// chain per quadrant: the quadrant's active column pairs (<= 32) flow
// through only the positions some pixel of that quadrant blended (the OR
// of its pixels' blend masks, compacted in list order), starting from the
// state at the unit start -- the positions left out did not touch these
// pixels, so every blended term still sees exactly the reference's state.
// A chain of <= 32 positions runs on a half-warp (2 positions per lane,
// np + ceil(n/2) - 1 steps); a quadrant with more is split at the bucket
// boundary (the second part starts from the second bucket's checkpoint).
// The two half-warps take two chains at a time, longest first.  A position
// appears in several chains: each chain folds its per-splat sums into a
// per-warp shared row, and the position's owner lane commits the row with
// one red.add per (tile, splat) column as before.
//
// The chain carries (T, G - g . image) instead of (T, G): dL/dalpha needs
// only G_after - g . image, so g . image leaves the per-step loads.
constexpr int kQWarps = 2;
constexpr int kQPairs = kTilePx / 2;  // pair slots: quadrant q at [32 q, 32 q + 32); + 1 inert slot

template <bool DEPTH>
struct QuadList {
    static constexpr int NC = DEPTH ? 10 : 9;
    float4 ga[kQPairs + 1];        // per pair: (gx, gx', gy, gy')
    float4 gb[kQPairs + 1];        // (gz, gz', y, y + 1)
    float4 s[kQPairs + 1];         // (T, T', G - gw, G' - gw') at the unit start
    float4 s2[kQPairs + 1];        // the same at the second bucket's start
    uint4 m[kQPairs + 1];          // blend masks (bucket 0 lo, hi; bucket 1 lo, hi)
    float px[kQPairs + 1];         // the pair's column x
    float2 gd[DEPTH ? kQPairs + 1 : 1];  // depth gradient (lo, hi)
    float acc[kUnit][NC];          // raw per-splat sums of the unit, over its chains
    uint32_t sid[kUnit];           // the unit's splats (records are re-read through L1/L2)
    uint8_t qpos[4][kUnit];        // per quadrant: its positions, compacted in list order
    uint8_t lanejob[8][32];        // per round and lane: chain id << 5 | lane in its segment, 255 idle
    int32_t rsteps[8];             // per round: the longest chain's step count
};

template <typename T>
__device__ __forceinline__ T sel4(int q, T a, T b, T c, T d) {
    return q == 0 ? a : q == 1 ? b : q == 2 ? c : d;
}

// One splat applied to a pixel pair of a chain (bwd_term2 with the state
// (T, G - g . image)).
template <bool DEPTH, bool CLAMP>
__device__ __forceinline__ void chain_term2(uint32_t ba, uint32_t bb, float pxs, f32x2 py,
                                            f32x2 gx, f32x2 gy, f32x2 gz, f32x2 gd,
                                            const SplatP2& S, float amax, f32x2& T, f32x2& G,
                                            SplatAcc2& q) {
    const float dxs = __fsub_rn(pxs, S.mxs);
    const float q0s = __fmul_rn(__fmul_rn(S.c0s, dxs), dxs), q1s = __fmul_rn(S.c1x2s, dxs);
    const f32x2 dx = pk2(dxs, dxs), dy = sub2(py, S.my);
    const f32x2 m = fma2(mul2(S.c2, dy), dy, fma2(pk2(q1s, q1s), dy, pk2(q0s, q0s)));
    float e0, e1;
    upk2(mul2(m, pk2(-0.5f * kLog2e, -0.5f * kLog2e)), e0, e1);
    float a0, a1;
    upk2(mul2(S.sig, pk2(ex2_approx(e0), ex2_approx(e1))), a0, a1);
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
    // dL/da = T (g . rgb) - (g . image - G_after) / (1 - a)   (kernels.py:342-364)
    const f32x2 om = sub2(pk2(1.f, 1.f), a);
    float o0, o1;
    upk2(om, o0, o1);
    const f32x2 dal = fma2(T, grgb, mul2(Gafter, pk2(rcp_approx(o0), rcp_approx(o1))));
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

// The half-warp wavefront of one chain: lane hl applies its positions pa,
// pb (-1: none) to pair j = step - hl of the chain's pairs [lb, lb + np);
// lanes off the diagonal read the inert slot (no blend bits).
template <bool DEPTH, bool CLAMP>
__device__ __forceinline__ void quad_wavefront(int steps, int np, int hl, int lb, int pa, int pb,
                                               const QuadList<DEPTH>& L,
                                               const float4* __restrict__ S4, const SplatP2& S0,
                                               const SplatP2& S1, float amax, SplatAcc2& q0,
                                               SplatAcc2& q1) {
    f32x2 T = pk2(0.f, 0.f), G = T;
    const bool wa = pa >= 32, wb = pb >= 32;
    const uint32_t bitA = pa >= 0 ? 1u << (pa & 31) : 0u;
    const uint32_t bitB = pb >= 0 ? 1u << (pb & 31) : 0u;
#pragma unroll 1
    for (int st = 0; st < steps; ++st) {
        T = shfl_up2w(T);
        G = shfl_up2w(G);
        const int j = st - hl;
        const bool inr = (unsigned)j < (unsigned)np;
        const int jj = inr ? lb + j : kQPairs;
        const uint4 m = L.m[jj];
        if (hl == 0 && inr) {
            const float4 s = S4[jj];
            T = pk2(s.x, s.y);
            G = pk2(s.z, s.w);
        }
        const uint32_t xa0 = (wa ? m.z : m.x) & bitA, xa1 = (wa ? m.w : m.y) & bitA;
        const uint32_t xb0 = (wb ? m.z : m.x) & bitB, xb1 = (wb ? m.w : m.y) & bitB;
        const float pxs = L.px[jj];
        const float4 g0 = L.ga[jj], g1 = L.gb[jj];
        const f32x2 py = pk2(g1.z, g1.w);
        const f32x2 gx = pk2(g0.x, g0.y), gy = pk2(g0.z, g0.w), gz = pk2(g1.x, g1.y);
        f32x2 gd = pk2(0.f, 0.f);
        if (DEPTH) {
            const float2 d = L.gd[jj];
            gd = pk2(d.x, d.y);
        }
        chain_term2<DEPTH, CLAMP>(xa0, xa1, pxs, py, gx, gy, gz, gd, S0, amax, T, G, q0);
        chain_term2<DEPTH, CLAMP>(xb0, xb1, pxs, py, gx, gy, gz, gd, S1, amax, T, G, q1);
    }
}

template <bool DEPTH>
__device__ __forceinline__ void quad_fold(QuadList<DEPTH>& L, int p, const SplatAcc2& q) {
    if (p < 0) return;
    float* row = L.acc[p];
    row[0] += hsum(q.r0);
    row[1] += hsum(q.r1);
    row[2] += hsum(q.r2);
    row[3] += hsum(q.s_da);
    row[4] += hsum(q.s_dx);
    row[5] += hsum(q.s_dy);
    row[6] += hsum(q.s_xx);
    row[7] += hsum(q.s_xy);
    row[8] += hsum(q.s_yy);
    if (DEPTH) row[9] += hsum(q.rz);
}

// One round: the lane runs chain `id` (-1: idle) as lane hl of its segment;
// `steps` = the longest chain of the round.  Chain id = 2 q + part: a
// quadrant with <= 32 positions is one chain (part 0: both buckets from the
// unit start), one with more is split at the bucket boundary (part 0:
// bucket 0; part 1: bucket 1 from its checkpoint).
template <bool DEPTH>
__device__ __forceinline__ void quad_round(QuadList<DEPTH>& L, const SplatRec* __restrict__ rec,
                                           int id, int hl, int steps, uint32_t chains,
                                           const int (&qn0)[4],
                                           const int (&qn1)[4], const int (&qnp)[4],
                                           float amax) {
    int np = 0, off = 0, n = 0, q = 0;
    bool second = false;
    if (id >= 0) {
        q = id >> 1;
        const int n0 = sel4(q, qn0[0], qn0[1], qn0[2], qn0[3]);
        const int n1 = sel4(q, qn1[0], qn1[1], qn1[2], qn1[3]);
        const bool split = n0 + n1 > 32;
        second = (id & 1) != 0;
        off = second ? n0 : 0;
        n = split ? (second ? n1 : n0) : n0 + n1;
        np = sel4(q, qnp[0], qnp[1], qnp[2], qnp[3]);
    }
    const int pa = 2 * hl < n ? L.qpos[q][off + 2 * hl] : -1;
    const int pb = 2 * hl + 1 < n ? L.qpos[q][off + 2 * hl + 1] : -1;
    float4 A0 = make_float4(0.f, 0.f, 0.f, 0.f), B0 = make_float4(0.f, 1.f, -1.f, 0.f), C0 = A0;
    float4 A1 = A0, B1 = B0, C1 = C0;
    if (pa >= 0) {
        const SplatRec r = rec[L.sid[pa]];
        A0 = r.a;
        B0 = r.b;
        C0 = r.c;
    }
    if (pb >= 0) {
        const SplatRec r = rec[L.sid[pb]];
        A1 = r.a;
        B1 = r.b;
        C1 = r.c;
    }
    const f32x2 z2 = pk2(0.f, 0.f);
    SplatAcc2 q0 = {z2, z2, z2, z2, z2, z2, z2, z2, z2, z2}, q1 = q0;
    const SplatP2 S0 = splat_p2(A0, B0, C0), S1 = splat_p2(A1, B1, C1);
    const float4* S4 = second ? L.s2 : L.s;
    const bool clamp = __any_sync(0xffffffffu, (pa >= 0 && B0.y >= amax * 0.999999f) ||
                                                   (pb >= 0 && B1.y >= amax * 0.999999f));
    if (clamp)
        quad_wavefront<DEPTH, true>(steps, np, hl, q * 32, pa, pb, L, S4, S0, S1, amax, q0, q1);
    else
        quad_wavefront<DEPTH, false>(steps, np, hl, q * 32, pa, pb, L, S4, S0, S1, amax, q0, q1);
    // fold into the unit's rows: chains of different quadrants may share
    // positions, so the round's chains take turns (a chain's own positions
    // are distinct: plain read-modify-writes, no atomics)
    while (chains) {
        const int c = __ffs(chains) - 1;
        chains &= chains - 1u;
        if (id == c) {
            quad_fold(L, pa, q0);
            quad_fold(L, pb, q1);
        }
        __syncwarp();
    }
}

template <bool DEPTH>
__global__ void __launch_bounds__(32 * kQWarps, 8) backward_quad_kernel(
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
    __shared__ QuadList<DEPTH> sQ[kQWarps];
    PDL_WAIT();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    QuadList<DEPTH>& L = sQ[wid];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        L.acc[2 * lane][c] = 0.f;
        L.acc[2 * lane + 1][c] = 0.f;
    }
    if (lane == 0) {  // the inert slot read by lanes off the diagonal
        L.ga[kQPairs] = make_float4(0.f, 0.f, 0.f, 0.f);
        L.gb[kQPairs] = make_float4(0.f, 0.f, 0.f, 0.f);
        L.s[kQPairs] = make_float4(1.f, 1.f, 0.f, 0.f);
        L.s2[kQPairs] = make_float4(1.f, 1.f, 0.f, 0.f);
        L.m[kQPairs] = make_uint4(0u, 0u, 0u, 0u);
        L.px[kQPairs] = 0.f;
        if (DEPTH) L.gd[kQPairs] = make_float2(0.f, 0.f);
    }
    const int64_t count = min(*work_count, work_cap);
    for (;;) {
        uint32_t item = 0;
        if (lane == 0) item = atomicAdd(work_counter, 1u);
        item = __shfl_sync(0xffffffffu, item, 0);
        if ((int64_t)item >= count) break;
        const uint2 wk = work[item];
        const int tile = (int)wk.x, u = (int)wk.y;
        const int x0 = (tile % tiles_x) * kTile, y0 = (tile / tiles_x) * kTile;
        const uint32_t start = tile_start[tile];
        const int ke = k_eff[tile];
        const int kbase = u * kUnit;
        const int k0 = kbase + 2 * lane, k1 = k0 + 1;
        // ---- the unit's splats (the lane's two positions)
        const uint32_t s0 = k0 < ke ? pairs[start + k0] : 0u;
        const uint32_t s1 = k1 < ke ? pairs[start + k1] : 0u;
        L.sid[2 * lane] = s0;
        L.sid[2 * lane + 1] = s1;
        // ---- the lane's 8 pixels (rows 2c + (lane >> 4), column lane & 15)
        const size_t slot0 = (size_t)(ckpt_base[tile] + 2 * u) * kTilePx;
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
                mk0[c] = nct[c] > kbase ? ckpt_mask[slot0 + p] : 0u;
                mk1[c] = nct[c] > kbase + kBucket ? ckpt_mask[slot0 + kTilePx + p] : 0u;
            }
        }
        // ---- per quadrant: the positions its pixels blended (both buckets),
        //      compacted in list order; their union = the splats that
        //      contributed in this unit
        int qn0[4], qn1[4];
        uint32_t u0 = 0u, u1 = 0u;
        {
            uint32_t t0 = 0, t1 = 0, b0 = 0, b1 = 0;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                t0 |= mk0[c];
                t1 |= mk1[c];
                b0 |= mk0[c + 4];
                b1 |= mk1[c + 4];
            }
            const bool right = (lane & 8) != 0;
            const unsigned lt = lanemask_lt();
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t v0 = q < 2 ? t0 : b0, v1 = q < 2 ? t1 : b1;
                const bool mine = (q & 1) ? right : !right;
                const uint32_t m0 = __reduce_or_sync(0xffffffffu, mine ? v0 : 0u);
                const uint32_t m1 = __reduce_or_sync(0xffffffffu, mine ? v1 : 0u);
                qn0[q] = __popc(m0);
                qn1[q] = __popc(m1);
                if ((m0 >> lane) & 1u) L.qpos[q][__popc(m0 & lt)] = (uint8_t)lane;
                if ((m1 >> lane) & 1u) L.qpos[q][qn0[q] + __popc(m1 & lt)] = (uint8_t)(32 + lane);
                u0 |= m0;
                u1 |= m1;
            }
        }
        // ---- the compaction's per-pixel rows (gradient, both checkpoints) are
        //      requested into L1 now, so its eight column-pair rounds do not each
        //      wait a DRAM round trip
#pragma unroll
        for (int c = 0; c < kTilePx / 32; ++c) {
            const int p = c * 32 + lane;
            const int ix = x0 + (p & 15), iy = y0 + (p >> 4);
            if ((mk0[c] | mk1[c]) != 0u) {
                const size_t o = (size_t)iy * W + ix;
                if (pixgrad) asm volatile("prefetch.global.L1 [%0];" ::"l"(pixgrad + o));
                asm volatile("prefetch.global.L1 [%0];" ::"l"(ckpt + slot0 + p));
                const int q = (c < 4 ? 0 : 2) + ((lane & 8) ? 1 : 0);
                if (mk1[c] != 0u && sel4(q, qn0[0] + qn1[0], qn0[1] + qn1[1], qn0[2] + qn1[2],
                                         qn0[3] + qn1[3]) > 32)
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(ckpt + slot0 + kTilePx + p));
            }
        }
        // ---- compact each quadrant's active column pairs (rows 2c, 2c + 1)
        //      into its 32-slot region of the list
        int qnp[4] = {0, 0, 0, 0};
#pragma unroll
        for (int c = 0; c < kTilePx / 32; ++c) {
            const int p = c * 32 + lane;
            const int ix = x0 + (p & 15), iy = y0 + (p >> 4);
            const size_t o = (size_t)iy * W + ix;
            const uint32_t m0 = mk0[c], m1 = mk1[c];
            const bool act = (m0 | m1) != 0u;
            const int partner = __shfl_xor_sync(0xffffffffu, (int)act, 16);  // every lane
            const bool pact = act || partner;
            const unsigned bal = __ballot_sync(0xffffffffu, pact) & 0xffffu;
            const int qbase = c < 4 ? 0 : 2;
            if (pact) {
                const bool right = (lane & 8) != 0;
                const int q = qbase + (right ? 1 : 0);
                const unsigned grp = right ? 0xff00u : 0x00ffu;
                const int pr = q * 32 + (right ? qnp[qbase + 1] : qnp[qbase]) +
                               __popc(bal & grp & ((1u << (lane & 15)) - 1u));
                const int hi = lane >> 4;  // the pair's lane: row 2c (lo) or 2c + 1 (hi)
                float4 pg = make_float4(0.f, 0.f, 0.f, 0.f);
                float T0 = 1.f, G0 = 0.f, T1 = 1.f, G1 = 0.f, gd = 0.f;
                if (act) {
                    if (pixgrad) {
                        pg = pixgrad[o];
                    } else {
                        pg.x = grad_image[3 * o];
                        pg.y = grad_image[3 * o + 1];
                        pg.z = grad_image[3 * o + 2];
                        pg.w = pg.x * image[3 * o] + pg.y * image[3 * o + 1] +
                               pg.z * image[3 * o + 2];
                    }
                    const float4 ck = ckpt[slot0 + p];
                    T0 = ck.x;
                    G0 = pg.x * ck.y + pg.y * ck.z + pg.z * ck.w;
                    if (DEPTH) {
                        gd = grad_depth ? grad_depth[o] : 0.f;
                        if (!pixgrad) pg.w += gd * depth_img[o];
                        G0 += gd * ckpt_depth[slot0 + p];
                    }
                    G0 -= pg.w;
                    // state at the second bucket's start: only split chains (a
                    // quadrant with > 32 positions) start there; pixels not
                    // blending there, or in unsplit quadrants, get an inert
                    // finite state (never read)
                    if (m1 != 0u && sel4(q, qn0[0] + qn1[0], qn0[1] + qn1[1],
                                         qn0[2] + qn1[2], qn0[3] + qn1[3]) > 32) {
                        const float4 c2 = ckpt[slot0 + kTilePx + p];
                        T1 = c2.x;
                        G1 = pg.x * c2.y + pg.y * c2.z + pg.z * c2.w;
                        if (DEPTH) G1 += gd * ckpt_depth[slot0 + kTilePx + p];
                        G1 -= pg.w;
                    }
                }
                float* fga = reinterpret_cast<float*>(&L.ga[pr]);
                float* fgb = reinterpret_cast<float*>(&L.gb[pr]);
                float* fs = reinterpret_cast<float*>(&L.s[pr]);
                float* fs2 = reinterpret_cast<float*>(&L.s2[pr]);
                uint32_t* fm = reinterpret_cast<uint32_t*>(&L.m[pr]);
                fga[hi] = pg.x;
                fga[2 + hi] = pg.y;
                fgb[hi] = pg.z;
                fgb[2 + hi] = (float)iy;
                fs[hi] = T0;
                fs[2 + hi] = G0;
                fs2[hi] = T1;
                fs2[2 + hi] = G1;
                fm[hi] = m0;
                fm[2 + hi] = m1;
                if (DEPTH) reinterpret_cast<float*>(&L.gd[pr])[hi] = gd;
                if (!hi) L.px[pr] = (float)ix;
            }
            qnp[qbase] += __popc(bal & 0x00ffu);
            qnp[qbase + 1] += __popc(bal & 0xff00u);
        }
        __syncwarp();
        // ---- chains sorted by length (steps), longest first, two per round
        int key[8], cid[8];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int n0 = qn0[q], n1 = qn1[q];
            const bool split = n0 + n1 > 32;
            cid[2 * q] = 2 * q;
            cid[2 * q + 1] = 2 * q + 1;
            const int na = split ? n0 : n0 + n1;
            key[2 * q] = na > 0 ? qnp[q] + (na + 1) / 2 - 1 : -1;
            key[2 * q + 1] = (split && n1 > 0) ? qnp[q] + (n1 + 1) / 2 - 1 : -1;
        }
#define SS_CX(a, b)                         \
    if (key[a] < key[b]) {                  \
        const int tk = key[a], tq = cid[a]; \
        key[a] = key[b];                    \
        cid[a] = cid[b];                    \
        key[b] = tk;                        \
        cid[b] = tq;                        \
    }
        // Batcher's odd-even merge sort network for 8 (19 compare-exchanges)
        SS_CX(0, 1) SS_CX(2, 3) SS_CX(4, 5) SS_CX(6, 7)
        SS_CX(0, 2) SS_CX(1, 3) SS_CX(4, 6) SS_CX(5, 7)
        SS_CX(1, 2) SS_CX(5, 6)
        SS_CX(0, 4) SS_CX(1, 5) SS_CX(2, 6) SS_CX(3, 7)
        SS_CX(2, 4) SS_CX(3, 5)
        SS_CX(1, 2) SS_CX(3, 4) SS_CX(5, 6)
#undef SS_CX
        // first-fit decreasing: chain i (2 positions per lane, L_i lanes)
        // goes to the first round with L_i free lanes; each lane records its
        // (chain, segment lane) per round in shared memory
        int nr = 0;
        {
            int used[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                used[r] = 0;
                L.lanejob[r][lane] = 255;
            }
            if (lane < 8) L.rsteps[lane] = 0;
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (key[i] >= 0) {
                    const int q = cid[i] >> 1;
                    const int n0 = sel4(q, qn0[0], qn0[1], qn0[2], qn0[3]);
                    const int n1 = sel4(q, qn1[0], qn1[1], qn1[2], qn1[3]);
                    const int n = n0 + n1 > 32 ? ((cid[i] & 1) ? n1 : n0) : n0 + n1;
                    const int Lc = (n + 1) >> 1;
                    int rs = -1, o = 0;
#pragma unroll
                    for (int r = 0; r < 8; ++r)
                        if (rs < 0 && r <= nr && used[r] + Lc <= 32) {
                            rs = r;
                            o = used[r];
                        }
#pragma unroll
                    for (int r = 0; r < 8; ++r)
                        if (r == rs) used[r] += Lc;
                    nr = max(nr, rs + 1);
                    if (lane >= o && lane < o + Lc) L.lanejob[rs][lane] = (uint8_t)(cid[i] << 5 | (lane - o));
                    if (lane == 0) {  // steps | chain ids of the round << 16
                        const int cur = L.rsteps[rs];
                        L.rsteps[rs] = max(cur & 0xffff, key[i]) | (cur & ~0xffff) |
                                       (1 << (16 + cid[i]));
                    }
                }
            }
            __syncwarp();
        }
#pragma unroll 1
        for (int r = 0; r < nr; ++r) {
            const int code = L.lanejob[r][lane];
            const int rs = L.rsteps[r];
            quad_round<DEPTH>(L, rec, code != 255 ? code >> 5 : -1, code & 31, rs & 0xffff,
                              (uint32_t)rs >> 16, qn0, qn1, qnp, amax);
        }
        __syncwarp();
        // ---- commit: lane l owns positions 2l, 2l + 1
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int p = 2 * lane + h;
            if (kbase + p < ke) {
                const uint32_t sg = h ? s1 : s0;
                const float4 A = rec[sg].a, B = rec[sg].b;
                float* r = L.acc[p];
                const float c1 = 0.5f * A.w;
                float acc[NC];
                acc[0] = r[0];
                acc[1] = r[1];
                acc[2] = r[2];
                acc[3] = A.z * r[4] + c1 * r[5];
                acc[4] = c1 * r[4] + B.x * r[5];
                acc[5] = -0.5f * r[6];
                acc[6] = -r[7];
                acc[7] = -0.5f * r[8];
                acc[8] = r[3] / B.y;
                if (DEPTH) acc[NC - 1] = r[9];
                float* row = g2d + (size_t)sg * NC;
#pragma unroll
                for (int c = 0; c < NC; ++c)
                    if (acc[c] != 0.f) atomicAdd(row + c, acc[c]);
                const uint32_t um = p < 32 ? u0 : u1;
                if (contributed && ((um >> (p & 31)) & 1u)) contributed[sg] = 1;
            }
#pragma unroll
            for (int c = 0; c < NC; ++c) L.acc[p][c] = 0.f;
        }
        __syncwarp();
    }
}

// --------------------------------------------------------------------------
// Sparse variant (opt-in: SS_BWD_SPARSE=1).  The wavefront above evaluates
// every (pixel, list position) slot of a unit and zeroes the ones the pixel
// did not blend; at the bench workload only 25 % of those slots are blended
// (15 % after 250 training iterations: low opacities, long lists).  Here
// only blended pairs are evaluated.  A CTA of 256 threads (one per tile
// pixel) takes a unit (tile, 2 checkpoint buckets); per bucket each WARP
// works on its own 32 pixels without CTA barriers:
//
//   phase 1 (lane = pixel): walk the set bits of the pixel's blend mask in
//     list order from the bucket's checkpoint -- exactly the pairs the
//     forward blended, with its arithmetic (splat_power / splat_falloff) --
//     and store per pair w = alpha T and da = alpha dL/dalpha
//     (kernels.py:342-364) position-major in the warp's shared-memory
//     region; the slot of (pixel, position) comes from the warp's 32 x 32
//     mask matrix transposed in registers (rank among the warp's pixels that
//     blended the position);
//   phase 2 (lane = list position): sum the position's pairs (<= 32) into
//     its 9 (10) screen-space gradients -- no shuffles -- and park them in
//     shared memory;
//
// then one CTA barrier, the 8 warps' rows are summed per position and
// committed with one red.add row per (tile, splat), as in the wavefront.
constexpr int kSpThreads = kTilePx;  // one thread per tile pixel
constexpr int kSpWarps = kSpThreads / 32;
constexpr int kSpWarpPairs = 32 * kBucket;  // a warp's pixels x a bucket's positions
constexpr int kSpPart = 10;                // parked row: 9 (10) gradients + pair count

struct SpShared {
    float2 wd[kSpWarps][kSpWarpPairs];     // (alpha T, alpha dL/dalpha), position-major
    uint8_t pid[kSpWarps][kSpWarpPairs];   // lane (pixel) of the pair
    float part[2][kSpWarps][kBucket][kSpPart + 1];  // per warp, per position (double-buffered)
    uint32_t bal[kSpWarps][kBucket];       // lanes that blended each position
    uint32_t base[kSpWarps][kBucket + 1];  // position slot ranges in the warp's region
    float4 g[kTilePx];                     // per pixel (g_r, g_g, g_b, g_depth)
    float2 xy[kTilePx];                    // per pixel (x, y)
    SplatRec rec[kUnit];                   // the unit's 64 list positions
    uint32_t sid[kUnit];
    int next;
};

// 32 x 32 bit-matrix transpose across a warp: lane l holds row l (bit k =
// M[l][k]); returns column `lane` (bit l = M[l][lane]).
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, int lane) {
    const uint32_t masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
    for (int s = 0; s < 5; ++s) {
        const int j = 16 >> s;
        const uint32_t m = masks[s];
        const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
        x = (lane & j) ? ((x & ~m) | ((y & ~m) >> j)) : ((x & m) | ((y & m) << j));
    }
    return x;
}

template <bool DEPTH>
__global__ void __launch_bounds__(kSpThreads, 2) backward_sparse_kernel(
    int W, int H, int tiles_x, const uint32_t* __restrict__ tile_start,
    const uint32_t* __restrict__ ckpt_base, const int32_t* __restrict__ k_eff,
    const uint32_t* __restrict__ pairs, const SplatRec* __restrict__ rec, float amax,
    const float* __restrict__ image, const float* __restrict__ grad_image,
    const float4* __restrict__ pixgrad, const float* __restrict__ depth_img,
    const float* __restrict__ grad_depth, const int32_t* __restrict__ n_contrib,
    const float4* __restrict__ ckpt, const float* __restrict__ ckpt_depth,
    const uint32_t* __restrict__ ckpt_mask, const uint2* __restrict__ work,
    const int64_t* __restrict__ work_count, int64_t work_cap, uint32_t* work_counter,
    float* __restrict__ g2d, uint8_t* __restrict__ contributed) {
    constexpr int NC = DEPTH ? 10 : 9;
    extern __shared__ __align__(16) unsigned char sp_smem[];
    SpShared& S = *reinterpret_cast<SpShared*>(sp_smem);
    PDL_WAIT();
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    const int64_t count = min(*work_count, work_cap);
    if (t == 0) S.next = (int)atomicAdd(work_counter, 1u);
    __syncthreads();
    int par = 0;  // parked-row buffer of the current bucket

    for (;;) {
        const uint32_t item = (uint32_t)S.next;
        if ((int64_t)item >= count) break;
        __syncthreads();  // everyone has read S.next and finished the last commit
        // the next item's index is fetched now; its latency hides under this one
        if (t == 0) S.next = (int)atomicAdd(work_counter, 1u);
        const uint2 wk = work[item];  // (tile, unit), longest-first order
        const int tile = (int)wk.x, u = (int)wk.y;
        const int x0 = (tile % tiles_x) * kTile, y0 = (tile / tiles_x) * kTile;
        const uint32_t start = tile_start[tile];
        const int ke = k_eff[tile];
        const uint32_t cb = ckpt_base[tile];
        const int kb0 = u * kUnit;
        const int nbk = min(2, (ke - kb0 + kBucket - 1) / kBucket);  // buckets of the unit
        // ---- every global load of the unit issued up front: the pixel's
        //      n_contrib, both buckets' masks and states, its gradient; the
        //      64 positions' records (validity is applied after the loads)
        const int ix = x0 + (t & 15), iy = y0 + (t >> 4);
        const bool inimg = ix < W && iy < H;
        const size_t o = inimg ? (size_t)iy * W + ix : 0;
        const size_t slot0 = (size_t)(cb + 2 * u) * kTilePx + t;
        const int nct = inimg ? n_contrib[o] : 0;
        uint32_t m0 = ckpt_mask[slot0];
        uint32_t m1 = nbk > 1 ? ckpt_mask[slot0 + kTilePx] : 0u;
        const float4 ck0 = ckpt[slot0];
        const float4 ck1 = nbk > 1 ? ckpt[slot0 + kTilePx] : make_float4(1.f, 0.f, 0.f, 0.f);
        float cd0 = 0.f, cd1 = 0.f;
        if (DEPTH) {
            cd0 = ckpt_depth[slot0];
            cd1 = nbk > 1 ? ckpt_depth[slot0 + kTilePx] : 0.f;
        }
        float4 pg = make_float4(0.f, 0.f, 0.f, 0.f);
        float gd = 0.f;
        if (inimg) {
            if (pixgrad) {
                pg = pixgrad[o];
            } else {
                pg.x = grad_image[3 * o];
                pg.y = grad_image[3 * o + 1];
                pg.z = grad_image[3 * o + 2];
                pg.w = pg.x * image[3 * o] + pg.y * image[3 * o + 1] + pg.z * image[3 * o + 2];
            }
            if (DEPTH) {
                gd = grad_depth ? grad_depth[o] : 0.f;
                if (!pixgrad) pg.w += gd * depth_img[o];
            }
        }
        if (t < kUnit) {
            const int k = kb0 + t;
            uint32_t sg = 0xffffffffu;
            if (k < ke) {
                sg = pairs[start + k];
                S.rec[t] = rec[sg];
            }
            S.sid[t] = sg;
        }
        const float px = (float)ix, py = (float)iy;
        S.g[t] = make_float4(pg.x, pg.y, pg.z, gd);
        S.xy[t] = make_float2(px, py);
        __syncthreads();  // records and pixel data visible to every warp
        // a bucket's mask and state exist for pixels still blending at its start
        m0 = nct > kb0 ? m0 : 0u;
        m1 = nct > kb0 + kBucket ? m1 : 0u;
        float2* WD = S.wd[wid];
        uint8_t* PID = S.pid[wid];
        for (int half = 0; half < nbk; ++half) {
            const uint32_t mask = half ? m1 : m0;
            const float4 ck = half ? ck1 : ck0;
            float T = ck.x;
            float G = pg.x * ck.y + pg.y * ck.z + pg.z * ck.w;
            if (DEPTH) G += gd * (half ? cd1 : cd0);
            const SplatRec* R32 = S.rec + kBucket * half;
            // lane k: which of the warp's pixels blended position k, and the
            // slot range of position k in the warp's region
            const uint32_t balk = warp_transpose32(mask, lane);
            const uint32_t cnt = __popc(balk);
            uint32_t inc = cnt;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t v = __shfl_up_sync(0xffffffffu, inc, d);
                if (lane >= d) inc += v;
            }
            S.bal[wid][lane] = balk;
            S.base[wid][lane] = inc - cnt;
            if (lane == 31) S.base[wid][kBucket] = inc;
            __syncwarp();
            // ---- phase 1: the pixel's blended pairs in list order; the next
            //      pair's record is loaded while this one computes (two record
            //      registers used in turn)
            if (mask) {
                const uint32_t lt = lanemask_lt();
                auto term = [&](int k, const SplatRec& R) {
                    float dx, dy;
                    const float a0 = splat_falloff(splat_power(px, py, R.a, R.b, dx, dy), R.b);
                    const float a = fminf(a0, amax);
                    const float w = __fmul_rn(a, T);
                    float grgb = fmaf(pg.z, R.c.z, fmaf(pg.y, R.c.y, pg.x * R.c.x));
                    if (DEPTH) grgb = fmaf(gd, R.b.w, grgb);
                    const float Gafter = fmaf(grgb, w, G);
                    const float om = __fsub_rn(1.f, a);
                    // dL/da = T (g . rgb) - (g . image - G_after) / (1 - a); 0 when clamped
                    const float dal = fmaf(T, grgb, (Gafter - pg.w) * rcp_approx(om));
                    const float da = dal * (a != amax ? a : 0.f);
                    T = __fmul_rn(T, om);
                    G = Gafter;
                    const uint32_t r = S.base[wid][k] + __popc(S.bal[wid][k] & lt);
                    WD[r] = make_float2(w, da);
                    PID[r] = (uint8_t)lane;
                };
                uint32_t m = mask;
                int k = __ffs(m) - 1;
                m &= m - 1;
                SplatRec R = R32[k];
                for (;;) {
                    if (!m) {
                        term(k, R);
                        break;
                    }
                    const int k2 = __ffs(m) - 1;
                    m &= m - 1;
                    const SplatRec R2 = R32[k2];
                    term(k, R);
                    if (!m) {
                        term(k2, R2);
                        break;
                    }
                    k = __ffs(m) - 1;
                    m &= m - 1;
                    R = R32[k];
                    term(k2, R2);
                }
            }
            __syncwarp();
            // ---- phase 2: lane k sums position k's pairs of this warp
            {
                const float4 A = R32[lane].a, B = R32[lane].b;
                const f32x2 mxy = pk2(A.x, A.y);
                f32x2 acc_rg = pk2(0.f, 0.f), s_d = acc_rg, s_xxy = acc_rg;
                float acc_b = 0.f, acc_z = 0.f, s_da = 0.f, s_yy = 0.f;
                const uint32_t r1 = inc;
                const float4* Gw = S.g + 32 * wid;
                const float2* XYw = S.xy + 32 * wid;
                for (uint32_t r = inc - cnt; r < r1; ++r) {
                    const float2 wd = WD[r];
                    const int p = PID[r];
                    const float4 g = Gw[p];
                    const float2 xy = XYw[p];
                    acc_rg = fma2(pk2(wd.x, wd.x), pk2(g.x, g.y), acc_rg);
                    acc_b = fmaf(wd.x, g.z, acc_b);
                    if (DEPTH) acc_z = fmaf(wd.x, g.w, acc_z);
                    const f32x2 dxy = sub2(pk2(xy.x, xy.y), mxy);
                    const f32x2 txy = mul2(pk2(wd.y, wd.y), dxy);
                    s_da += wd.y;
                    s_d = add2(s_d, txy);
                    float tx, ty, dx, dy;
                    upk2(txy, tx, ty);
                    upk2(dxy, dx, dy);
                    s_xxy = fma2(pk2(tx, tx), dxy, s_xxy);
                    s_yy = fmaf(ty, dy, s_yy);
                }
                // the splat-constant factors (linear: summing the warps' rows
                // afterwards gives the same result)
                float s_dx, s_dy, s_xx, s_xy;
                upk2(s_d, s_dx, s_dy);
                upk2(s_xxy, s_xx, s_xy);
                float* row = S.part[par][wid][lane];
                upk2(acc_rg, row[0], row[1]);
                row[2] = acc_b;
                const float c1 = 0.5f * A.w;
                row[3] = A.z * s_dx + c1 * s_dy;
                row[4] = c1 * s_dx + B.x * s_dy;
                row[5] = -0.5f * s_xx;
                row[6] = -s_xy;
                row[7] = -0.5f * s_yy;
                row[8] = cnt ? s_da / B.y : 0.f;
                if (DEPTH) row[9] = acc_z;
                row[kSpPart] = (float)cnt;
            }
            __syncthreads();  // every warp's rows are parked
            // ---- commit: sum the 8 warps' rows per (position, column)
            {
                const int k = t >> 3, c0 = t & 7;
                const uint32_t sg = S.sid[kBucket * half + k];
                float n = 0.f;
#pragma unroll
                for (int w = 0; w < kSpWarps; ++w) n += S.part[par][w][k][kSpPart];
                if (n > 0.f) {
                    float* grow = g2d + (size_t)sg * NC;
                    for (int c = c0; c < NC; c += 8) {
                        float v = 0.f;
#pragma unroll
                        for (int w = 0; w < kSpWarps; ++w) v += S.part[par][w][k][c];
                        if (v != 0.f) atomicAdd(grow + c, v);
                    }
                    if (contributed && c0 == 0) contributed[sg] = 1;
                }
            }
            par ^= 1;
        }
    }
}

// Longest-units-first schedule.  A unit's size is roughly the number of
// pixels still blending at its first bucket, so earlier units of a tile are
// larger, and tiles with more units are the deeper ones.  Handing units out
// unit-index-major with the tiles of each index in descending unit count
// approximates longest-processing-time-first and shortens the tail of the
// persistent backward.  One CTA builds it from k_eff: tiles counting-sorted
// by unit count, descending (S; the tiles with more than u units are a
// prefix of S), start[u] = sum over u' < u of #tiles with more than u'
// units; item start[u] + i is unit u of tile S[i].  The list is written IN
// PLACE over the forward's (same items, any order), so the backward reads
// its items with one load.  Tiles with more than kMaxUnits units, or more
// than kSchedTiles tiles: the forward's list is kept.
constexpr int kMaxUnits = 1024;
constexpr int kSchedTiles = 16384;  // 4K frames at 16 px tiles fit

__global__ void __launch_bounds__(1024) bwd_schedule_kernel(uint32_t* counter,
                                                            const int32_t* __restrict__ k_eff,
                                                            int n_tiles, uint32_t* __restrict__ wl,
                                                            int64_t wl_cap,
                                                            const int64_t* __restrict__ total) {
    __shared__ uint32_t h[kMaxUnits + 1];
    __shared__ uint32_t s_start[kMaxUnits + 1];
    __shared__ uint16_t s_nb[kSchedTiles];
    __shared__ uint32_t s_max;
    const int t = threadIdx.x;
    if (t == 0) counter[1] = 0u;  // items are read as work[item] (kept for the ABI word)
    if (n_tiles > kSchedTiles) return;
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
    if (mu > (uint32_t)kMaxUnits || *total > wl_cap / 2) return;  // keep the forward's list
    if (t == 0) {
        uint32_t above = 0;
        for (int v = (int)mu; v >= 0; --v) {  // h[v] -> #tiles with more than v units
            const uint32_t c = h[v];           //         = first position of bucket v in S
            h[v] = above;
            above += c;
        }
        uint32_t pre = 0;
        for (uint32_t u = 0; u < mu; ++u) {
            s_start[u] = pre;
            pre += h[u];
        }
        s_start[mu] = pre;
    }
    __syncthreads();
    for (int q = t; q < n_tiles; q += blockDim.x) {
        const uint32_t nb = s_nb[q];
        if (nb == 0) continue;
        const uint32_t pos = atomicAdd(&h[nb], 1u);  // this tile's index in S
        for (uint32_t u = 0; u < nb; ++u) {
            const uint32_t c = s_start[u] + pos;
            wl[2 * c] = (uint32_t)q;
            wl[2 * c + 1] = u;
        }
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

// one launch clears the gradient rows, the contributed marks and the
// work-unit counter (also usable ahead of time on another stream: the
// engine runs it beside the loss kernels, ss_backward_clear)
cudaError_t launch_backward_clear(int64_t n, int ncol, float* g2d, uint8_t* contributed,
                                  uint32_t* counter, cudaStream_t s) {
    launch_pdl(bwd_clear_kernel, dim3(div_up(n * ncol > 4 ? n * ncol / 4 : 1, 256)), dim3(256),
               0, s, g2d, (int64_t)n * ncol, contributed, n, counter);
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
                                  bool clear, cudaStream_t s) {
    const bool depthf = o->with_depth != 0;
    const int ncol = depthf ? 10 : 9;
    int tx = div_up(cam->width, kTile), ty = div_up(cam->height, kTile);
    if (clear) launch_backward_clear(n, ncol, g2d, contributed, counter, s);
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    static const bool wavefront = [] {
        const char* e = getenv("SS_BWD_SPARSE");  // 1: the sparse two-phase kernel
        return !(e && e[0] == '1');
    }();
    static const bool unit_chains = [] {
        const char* e = getenv("SS_BWD_UNIT");  // 1: one chain per bucket over the whole tile
        return e && e[0] == '1';
    }();
    if (!wavefront) {
        const size_t sm_bytes = sizeof(SpShared);
        auto go = [&](auto kern) -> cudaError_t {
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)sm_bytes);
            if (e != cudaSuccess) return e;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSpThreads, sm_bytes);
            if (per_sm < 1) per_sm = 1;
            launch_pdl(kern, dim3(sms * per_sm), dim3(kSpThreads), sm_bytes, s,
                cam->width, cam->height, tx, bins->d_tile_start, bins->d_ckpt_base, k_eff,
                bins->d_pair_splat, reinterpret_cast<const SplatRec*>(sp->d_rec), o->alpha_max,
                image, grad_image, pixgrad, depth, grad_depth, n_contrib,
                reinterpret_cast<const float4*>(ckpt), ckpt_depth, ckpt_mask,
                reinterpret_cast<const uint2*>(work), &st->bucket_count, work_cap, counter, g2d,
                contributed);
            return cudaGetLastError();
        };
        return depthf ? go(backward_sparse_kernel<true>) : go(backward_sparse_kernel<false>);
    }
    const int threads = 32 * kBwdWarps;
    const size_t smem = 0;
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
    if (unit_chains)
        return depthf ? go(backward_splat_kernel<true>) : go(backward_splat_kernel<false>);
    const int qthreads = 32 * kQWarps;
    auto goq = [&](auto kern) -> cudaError_t {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, qthreads, 0);
        if (per_sm < 1) per_sm = 1;
        launch_pdl(kern, dim3(sms * per_sm), dim3(qthreads), 0, s,
            cam->width, cam->height, tx, bins->d_tile_start, bins->d_ckpt_base, k_eff,
            bins->d_pair_splat, reinterpret_cast<const SplatRec*>(sp->d_rec), o->alpha_max, image,
            grad_image, pixgrad, depth, grad_depth, n_contrib,
            reinterpret_cast<const float4*>(ckpt), ckpt_depth, ckpt_mask,
            reinterpret_cast<const uint2*>(work), &st->bucket_count, work_cap, counter, g2d,
            contributed, tx * ty);
        return cudaGetLastError();
    };
    return depthf ? goq(backward_quad_kernel<true>) : goq(backward_quad_kernel<false>);
}

}  // namespace ss
