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

// Per-warp pixel list capacity: a tile's 256 pixels as 128 (even, odd) pairs.
constexpr int kBwdWarps = 4;
constexpr int kPairs = kTilePx / 2;

// One (pixel, splat) term of the wavefront.  `bit` is the forward's blend
// mask bit; a pair that was not blended gets a = 0, which leaves T and G
// bit-exactly unchanged and contributes nothing, so both pixels of a step
// run branch-free as two independent dependency chains.
template <bool DEPTH>
__device__ __forceinline__ void bwd_term(bool bit, float px, float py, const float4& pg, float gd,
                                         const float4& A, const float4& B, const float4& C,
                                         float amax, float& T, float& G, float& r0, float& r1,
                                         float& r2, float& rz, float& s_da, float& s_dx,
                                         float& s_dy, float& s_xx, float& s_xy, float& s_yy) {
    float dx, dy;
    float a = splat_alpha_blended(px, py, A, B, amax, dx, dy);
    a = bit ? a : 0.f;
    const float w = __fmul_rn(a, T);
    float grgb = pg.x * C.x + pg.y * C.y + pg.z * C.z;
    if (DEPTH) {
        grgb += gd * B.w;
        rz += w * gd;
    }
    const float Gafter = G + grgb * w;
    r0 += w * pg.x;
    r1 += w * pg.y;
    r2 += w * pg.z;
    // alpha-path gradient (kernels.py:342-364); zero when clamped or not blended
    const float dal = T * grgb - (pg.w - Gafter) * rcp_approx(1.0f - a);
    const float da = (bit && a != amax) ? dal * a : 0.f;
    const float tx = da * dx, ty = da * dy;
    s_da += da;
    s_dx += tx;
    s_dy += ty;
    s_xx += tx * dx;
    s_xy += tx * dy;
    s_yy += ty * dy;
    T = __fmul_rn(T, __fsub_rn(1.0f, a));
    G = Gafter;
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
    float* __restrict__ g2d, uint8_t* __restrict__ contributed) {
    constexpr int NC = DEPTH ? 10 : 9;
    // per-warp compacted pixel list, list position q -> pair q/2, half q&1:
    // gradient side (g, g . image), state at the bucket start (T0, G0),
    // coordinates, blend mask, depth gradient
    __shared__ float4 sGe[kBwdWarps][kPairs], sGo[kBwdWarps][kPairs];
    __shared__ float4 sS[kBwdWarps][kPairs];   // (T0, G0) even, (T0, G0) odd
    __shared__ float4 sXY[kBwdWarps][kPairs];  // (x, y) even, (x, y) odd
    __shared__ uint2 sM[kBwdWarps][kPairs];
    __shared__ float2 sD[DEPTH ? kBwdWarps : 1][DEPTH ? kPairs : 1];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t count = min(*work_count, work_cap);

    for (;;) {
        uint32_t item = 0;
        if (lane == 0) item = atomicAdd(work_counter, 1u);
        item = __shfl_sync(0xffffffffu, item, 0);
        if ((int64_t)item >= count) break;
        const uint2 wk = work[item];
        const int tile = (int)wk.x, b = (int)wk.y;
        const int x0 = (tile % tiles_x) * kTile, y0 = (tile / tiles_x) * kTile;
        const uint32_t start = tile_start[tile];
        const int ke = k_eff[tile];
        const int kbase = b * kBucket;
        const int k = kbase + lane;
        uint32_t s = 0;
        float4 A = make_float4(0.f, 0.f, 0.f, 0.f), B = make_float4(0.f, 1.f, -1.f, 0.f),
               C = make_float4(0.f, 0.f, 0.f, 0.f);
        if (k < ke) {
            s = pairs[start + k];
            const SplatRec r = rec[s];
            A = r.a;
            B = r.b;
            C = r.c;
        }
        // ---- compact the pixels that blended any splat of this bucket
        const size_t slot0 = (size_t)(ckpt_base[tile] + b) * kTilePx;
        int nact = 0;
#pragma unroll 1
        for (int c = 0; c < kTilePx / 32; ++c) {
            const int p = c * 32 + lane;
            const int ix = x0 + (p & 15), iy = y0 + (p >> 4);
            const bool inside = ix < W && iy < H;
            const size_t o = (size_t)iy * W + ix;
            const int nc = inside ? n_contrib[o] : 0;
            const uint32_t mask = nc > kbase ? ckpt_mask[slot0 + p] : 0u;
            const unsigned bal = __ballot_sync(0xffffffffu, mask != 0u);
            if (mask) {
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
                const int h = pos & 1, q = pos >> 1;
                if (DEPTH) {
                    const float gd = grad_depth ? grad_depth[o] : 0.f;
                    if (!pixgrad) pg.w += gd * depth_img[o];
                    G0 += gd * ckpt_depth[slot0 + p];
                    reinterpret_cast<float*>(&sD[wid][q])[h] = gd;
                }
                (h ? sGo : sGe)[wid][q] = pg;
                reinterpret_cast<float2*>(&sS[wid][q])[h] = make_float2(ck.x, G0);
                reinterpret_cast<uint32_t*>(&sM[wid][q])[h] = mask;
                reinterpret_cast<float2*>(&sXY[wid][q])[h] = make_float2((float)ix, (float)iy);
            }
            nact += __popc(bal);
        }
        if ((nact & 1) && lane == 0) {  // pad the last pair with an empty pixel
            const int q = nact >> 1;
            sGo[wid][q] = make_float4(0.f, 0.f, 0.f, 0.f);
            sS[wid][q].z = sS[wid][q].w = 0.f;
            sXY[wid][q].z = sXY[wid][q].w = 0.f;
            sM[wid][q].y = 0u;
            if (DEPTH) sD[wid][q].y = 0.f;
        }
        __syncwarp();
        // ---- diagonal wavefront over the active pixel pairs
        // per-lane sums; the splat-constant factors (conic, 1/sigma, -1/2)
        // are applied once at the end:
        //   d mean  = (c0 S_dx + c1 S_dy, c1 S_dx + c2 S_dy),  S_d. = sum da d.
        //   d conic = -1/2 (S_dxdx, 2 S_dxdy, S_dydy),        d sigma = S_da / sigma
        float acc_rgb0 = 0.f, acc_rgb1 = 0.f, acc_rgb2 = 0.f, acc_z = 0.f;
        float s_da = 0.f, s_dx = 0.f, s_dy = 0.f, s_xx = 0.f, s_xy = 0.f, s_yy = 0.f;
        float T0 = 0.f, G0 = 0.f, T1 = 0.f, G1 = 0.f;
        uint32_t any = 0u;
        const int npair = (nact + 1) >> 1;
        const int steps = npair + 31;
#pragma unroll 1
        for (int st = 0; st < steps; ++st) {
            float Ta = __shfl_up_sync(0xffffffffu, T0, 1);
            float Ga = __shfl_up_sync(0xffffffffu, G0, 1);
            float Tb = __shfl_up_sync(0xffffffffu, T1, 1);
            float Gb = __shfl_up_sync(0xffffffffu, G1, 1);
            const int q = st - lane;
            if ((unsigned)q >= (unsigned)npair) continue;
            const uint2 m = sM[wid][q];
            if (lane == 0) {
                const float4 s0 = sS[wid][q];
                Ta = s0.x;
                Ga = s0.y;
                Tb = s0.z;
                Gb = s0.w;
            }
            T0 = Ta;
            G0 = Ga;
            T1 = Tb;
            G1 = Gb;
            const bool b0 = (m.x >> lane) & 1u, b1 = (m.y >> lane) & 1u;
            if (!(b0 || b1)) continue;
            any = 1u;
            const float4 xy = sXY[wid][q];
            const float4 pe = sGe[wid][q], po = sGo[wid][q];
            float2 gd = make_float2(0.f, 0.f);
            if (DEPTH) gd = sD[wid][q];
            bwd_term<DEPTH>(b0, xy.x, xy.y, pe, gd.x, A, B, C, amax, T0, G0, acc_rgb0, acc_rgb1,
                            acc_rgb2, acc_z, s_da, s_dx, s_dy, s_xx, s_xy, s_yy);
            bwd_term<DEPTH>(b1, xy.z, xy.w, po, gd.y, A, B, C, amax, T1, G1, acc_rgb0, acc_rgb1,
                            acc_rgb2, acc_z, s_da, s_dx, s_dy, s_xx, s_xy, s_yy);
        }
        const float c1 = 0.5f * A.w;
        float acc[NC];
        acc[0] = acc_rgb0;
        acc[1] = acc_rgb1;
        acc[2] = acc_rgb2;
        acc[3] = A.z * s_dx + c1 * s_dy;
        acc[4] = c1 * s_dx + B.x * s_dy;
        acc[5] = -0.5f * s_xx;
        acc[6] = -s_xy;
        acc[7] = -0.5f * s_yy;
        acc[8] = s_da / B.y;
        if (DEPTH) acc[NC - 1] = acc_z;
        if (k < ke) {
            float* row = g2d + (size_t)s * NC;
#pragma unroll
            for (int q = 0; q < NC; ++q)
                if (acc[q] != 0.f) atomicAdd(row + q, acc[q]);
            if (contributed && any) contributed[s] = 1;
        }
        __syncwarp();
    }
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
    cudaError_t e = cudaMemsetAsync(g2d, 0, sizeof(float) * (size_t)n * ncol, s);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(counter, 0, sizeof(uint32_t), s);
    if (e != cudaSuccess) return e;
    int tx = div_up(cam->width, kTile);
    const int threads = 32 * kBwdWarps;
    const size_t smem = 0;
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    auto go = [&](auto kern) -> cudaError_t {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
        if (per_sm < 1) per_sm = 1;
        kern<<<sms * per_sm, threads, smem, s>>>(
            cam->width, cam->height, tx, bins->d_tile_start, bins->d_ckpt_base, k_eff,
            bins->d_pair_splat, reinterpret_cast<const SplatRec*>(sp->d_rec), o->alpha_max, image,
            grad_image, pixgrad, depth, grad_depth, n_contrib,
            reinterpret_cast<const float4*>(ckpt), ckpt_depth, ckpt_mask,
            reinterpret_cast<const uint2*>(work), &st->bucket_count, work_cap, counter, g2d,
            contributed);
        return cudaGetLastError();
    };
    return depthf ? go(backward_splat_kernel<true>) : go(backward_splat_kernel<false>);
}

}  // namespace ss
