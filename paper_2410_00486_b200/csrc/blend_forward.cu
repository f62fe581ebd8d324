// blend_forward.cu -- K5: per-tile front-to-back alpha blending.
//
// Restates rasterize_forward's tile loop (rasterizer/api.py:153-196) and
// forward_tile (rasterizer/kernels.py:34-109) with checkpoint_tile
// (kernels.py:112-152) folded in: one 256-thread CTA per 16x16 tile, one
// thread per pixel.  The tile's depth-sorted list is walked in batches of
// 256 splat records staged in shared memory (one coalesced gather per
// batch, each thread loading one record); every thread walks the batch
// from shared memory with broadcast reads.  Reference semantics kept:
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
// Extension A15 (builder-defined): D = sum z a T in a 4th accumulator.
// The CTA also emits k_eff (kernels.py:86-87,109) and appends its
// ceil(k_eff/32) (tile, bucket) units to the splat-wise backward work list.
#include "common.cuh"

namespace ss {

template <bool DEPTH, bool CONTRIB>
__global__ void __launch_bounds__(256) blend_forward_kernel(
    int W, int H, int tiles_x, const uint32_t* __restrict__ tile_start,
    const uint32_t* __restrict__ tile_end, const uint32_t* __restrict__ ckpt_base,
    const uint32_t* __restrict__ pairs, const SplatRec* __restrict__ rec, float t_min, float amin,
    float amax, float bg0, float bg1, float bg2, float* __restrict__ image,
    float* __restrict__ final_t, int32_t* __restrict__ n_contrib, float* __restrict__ depth_img,
    int32_t* __restrict__ k_eff, uint8_t* __restrict__ contributed, float4* __restrict__ ckpt,
    float* __restrict__ ckpt_depth, uint2* __restrict__ work, int64_t work_cap,
    int64_t* bucket_count) {
    __shared__ SplatRec s_rec[256];
    __shared__ uint32_t s_id[256];
    __shared__ int s_hit[CONTRIB ? 256 : 1];
    __shared__ int s_kmax[8];
    const int tile = blockIdx.x;
    const int t = threadIdx.x;
    const int x0 = (tile % tiles_x) * kTile, y0 = (tile / tiles_x) * kTile;
    const int ix = x0 + (t & 15), iy = y0 + (t >> 4);
    const bool inside = ix < W && iy < H;
    const float px = (float)ix, py = (float)iy;
    const uint32_t start = tile_start[tile];
    const uint32_t len = tile_end[tile] - start;
    const uint32_t cbase = ckpt_base[tile];

    float T = 1.0f, c0 = 0.f, c1 = 0.f, c2 = 0.f, D = 0.f;
    bool done = !inside;
    int last = 0;
    for (uint32_t b0 = 0; b0 < len; b0 += 256) {
        if (__syncthreads_count(!done) == 0) break;
        if (b0 + t < len) {
            uint32_t s = pairs[start + b0 + t];
            s_id[t] = s;
            s_rec[t] = rec[s];
            if (CONTRIB) s_hit[t] = 0;
        }
        __syncthreads();
        const int nb = (int)min(256u, len - b0);
        for (int j0 = 0; j0 < nb; j0 += 32) {
            if (__all_sync(0xffffffffu, done)) break;  // whole warp stopped
            const uint32_t q0 = b0 + j0;                 // multiple of 32
            if (!done) {
                size_t slot = (size_t)(cbase + (q0 >> 5)) * kTilePx + t;
                ckpt[slot] = make_float4(T, c0, c1, c2);
                if (DEPTH) ckpt_depth[slot] = D;
            }
            const int jn = min(nb, j0 + 32);
            for (int j = j0; j < jn; ++j) {
                if (done) continue;
                const float4 A = s_rec[j].a, B = s_rec[j].b;
                float dx, dy;
                float a = splat_alpha(px, py, A, B, amin, amax, dx, dy);
                if (a < 0.f) continue;
                const float4 C = s_rec[j].c;
                float w = __fmul_rn(a, T);
                c0 = __fmaf_rn(C.x, w, c0);
                c1 = __fmaf_rn(C.y, w, c1);
                c2 = __fmaf_rn(C.z, w, c2);
                if (DEPTH) D = __fmaf_rn(B.w, w, D);
                T = __fmul_rn(T, __fsub_rn(1.0f, a));
                last = (int)(b0 + j) + 1;
                if (CONTRIB) s_hit[j] = 1;
                if (T < t_min) done = true;
            }
        }
        if (CONTRIB) {
            __syncthreads();
            if (b0 + t < len && s_hit[t]) contributed[s_id[t]] = 1;
        }
    }
    if (inside) {
        const size_t o = (size_t)iy * W + ix;
        final_t[o] = T;
        image[3 * o] = c0 + bg0 * T;
        image[3 * o + 1] = c1 + bg1 * T;
        image[3 * o + 2] = c2 + bg2 * T;
        n_contrib[o] = last;
        if (DEPTH) depth_img[o] = D;
    }
    int km = warp_max(last);
    if ((t & 31) == 0) s_kmax[t >> 5] = km;
    __syncthreads();
    if (t < 32) {
        int v = t < 8 ? s_kmax[t] : 0;
        v = warp_max(v);
        if (t == 0) s_kmax[0] = v;
    }
    __syncthreads();
    const int kmax = s_kmax[0];
    if (t == 0) k_eff[tile] = kmax;
    const int nbk = (kmax + kBucket - 1) / kBucket;
    if (nbk > 0 && work) {
        __shared__ unsigned long long s_wbase;
        if (t == 0) s_wbase = atomicAdd(reinterpret_cast<unsigned long long*>(bucket_count),
                                        (unsigned long long)nbk);
        __syncthreads();
        for (int b = t; b < nbk; b += blockDim.x) {
            long long idx = (long long)s_wbase + b;
            if (idx < work_cap) work[idx] = make_uint2((uint32_t)tile, (uint32_t)b);
        }
    }
}

cudaError_t launch_blend_forward(const ss_camera* cam, const ss_raster_opts* o,
                                 const ss_splats* sp, const ss_bins* bins, float* image,
                                 float* final_t, int32_t* n_contrib, float* depth,
                                 int32_t* k_eff, uint8_t* contributed, void* ckpt,
                                 float* ckpt_depth, uint32_t* work, int64_t work_cap,
                                 ss_status* st, cudaStream_t s) {
    int tx = div_up(cam->width, kTile), ty = div_up(cam->height, kTile);
    int n_tiles = tx * ty;
    const bool depthf = o->with_depth != 0;
    const bool contribf = contributed != nullptr;
    auto args = [&](auto kern) {
        kern<<<n_tiles, 256, 0, s>>>(
            cam->width, cam->height, tx, bins->d_tile_start, bins->d_tile_end, bins->d_ckpt_base,
            bins->d_pair_splat, reinterpret_cast<const SplatRec*>(sp->d_rec), o->t_min,
            o->alpha_min, o->alpha_max, o->background[0], o->background[1], o->background[2],
            image, final_t, n_contrib, depth, k_eff, contributed, reinterpret_cast<float4*>(ckpt),
            ckpt_depth, reinterpret_cast<uint2*>(work), work_cap, &st->bucket_count);
    };
    if (depthf && contribf)
        args(blend_forward_kernel<true, true>);
    else if (depthf)
        args(blend_forward_kernel<true, false>);
    else if (contribf)
        args(blend_forward_kernel<false, true>);
    else
        args(blend_forward_kernel<false, false>);
    return cudaGetLastError();
}

}  // namespace ss
