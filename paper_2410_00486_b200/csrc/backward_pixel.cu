// backward_pixel.cu -- F2: pixel-wise backward, the paper's ablation baseline.
//
// Restates backward_pixelwise (rasterizer/api.py:227-272) over
// backward_pixel_tile (rasterizer/kernels.py:181-268): every pixel re-runs
// its forward prefix and produces, for each splat it blended, the same
// per-(pixel, splat) terms as the splat-wise backward; the per-splat sums
// over a tile's pixels become one accumulator row per (tile, list position)
// merged into g2d.  The reference walks the prefix forward (stashing alpha,
// T and the accumulated colour) and the splats in reverse; the suffix
// colour it needs behind splat k is image - c_after(k), so on the GPU a
// single front-to-back pass yields every term without a stash.
//
// B200 shape: one 128-thread CTA per tile, two pixels per thread (one
// column, rows r and r + 2 of the warp's 4-row band, as the forward), the
// tile's list walked in batches of 256 records staged in shared memory.
// Per splat, each warp reduces its 32 lanes' sums with shuffles (skipped
// when no lane blended it) and adds them to a shared per-position row;
// one red.add row per (tile, splat) at the end of the batch.  This is the
// pixel-parallel accumulation pattern the splat-wise kernel replaces:
// 9 butterfly reductions per (warp, splat) instead of per-lane registers.
#include "common.cuh"

namespace ss {

constexpr int kPxThreads = 128;

__global__ void __launch_bounds__(kPxThreads) backward_pixel_kernel(
    int W, int H, int tiles_x, const uint32_t* __restrict__ tile_start,
    const int32_t* __restrict__ k_eff, const uint32_t* __restrict__ pairs,
    const SplatRec* __restrict__ rec, float amin, float amax, const float* __restrict__ image,
    const float* __restrict__ grad_image, const int32_t* __restrict__ n_contrib,
    float* __restrict__ g2d) {
    __shared__ SplatRec s_rec[256];
    __shared__ uint32_t s_id[256];
    __shared__ float s_acc[9][256];  // per list position of the batch: colour 3, S_da, S_dx,
                                     // S_dy, S_xx, S_xy, S_yy
    const int tile = blockIdx.x;
    const int t = threadIdx.x, w = t >> 5, lane = t & 31;
    const int x0 = (tile % tiles_x) * kTile, y0 = (tile / tiles_x) * kTile;
    const int row0 = 4 * w + (lane >> 4), row1 = row0 + 2;
    const int ix = x0 + (lane & 15);
    const int iy[2] = {y0 + row0, y0 + row1};
    const float px = (float)ix;
    float py[2], T[2], cacc[2][3], g[2][3], img[2][3];
    int nc[2];
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        py[p] = (float)iy[p];
        T[p] = 1.f;
        const bool in = ix < W && iy[p] < H;
        const size_t o = in ? (size_t)iy[p] * W + ix : 0;
        nc[p] = in ? n_contrib[o] : 0;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            cacc[p][c] = 0.f;
            g[p][c] = in ? grad_image[3 * o + c] : 0.f;
            img[p][c] = in ? image[3 * o + c] : 0.f;
        }
        // backward_pixel_tile skips pixels with zero gradient (kernels.py:198-200)
        if (g[p][0] == 0.f && g[p][1] == 0.f && g[p][2] == 0.f) nc[p] = 0;
    }
    const uint32_t start = tile_start[tile];
    const int ke = k_eff[tile];
    for (int b0 = 0; b0 < ke; b0 += 256) {
        const int nb = min(256, ke - b0);
        for (int k = t; k < nb; k += kPxThreads) {
            const uint32_t s = pairs[start + b0 + k];
            s_id[k] = s;
            s_rec[k] = rec[s];
        }
        for (int k = t; k < 9 * 256; k += kPxThreads) (&s_acc[0][0])[k] = 0.f;
        __syncthreads();
        const int wmax = warp_max(max(nc[0], nc[1])) - b0;  // this warp's live positions
        const int jn = min(nb, wmax);
        for (int j = 0; j < jn; ++j) {
            const float4 A = s_rec[j].a, B = s_rec[j].b, C = s_rec[j].c;
            const float dx = __fsub_rn(px, A.x);
            const float q0 = quad_dx0(A, dx), q1 = quad_dx1(A, dx);
            float v[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            bool any = false;
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                if (b0 + j >= nc[p]) continue;
                const float dy = __fsub_rn(py[p], A.y);
                const float m = quad_finish(q0, q1, B, dy);
                if (m > B.z) continue;  // _alpha's m_cut test (kernels.py:24-25)
                float a = splat_falloff(m, B);
                if (a < amin) continue;  // kernels.py:27-28
                a = fminf(a, amax);
                any = true;
                const float Tk = T[p];
                const float wgt = __fmul_rn(a, Tk);
                const float rgb[3] = {C.x, C.y, C.z};
                float after[3];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    after[c] = __fmaf_rn(rgb[c], wgt, cacc[p][c]);
                    v[c] += wgt * g[p][c];
                }
                const float am1 = __fsub_rn(1.0f, a);
                if (am1 > 0.f && a != amax) {  // kernels.py:248
                    const float r = rcp_approx(am1);
                    float dal = 0.f;
#pragma unroll
                    for (int c = 0; c < 3; ++c)
                        dal += (rgb[c] * Tk - (img[p][c] - after[c]) * r) * g[p][c];
                    const float da = dal * a;
                    const float tx = da * dx, ty = da * dy;
                    v[3] += da;
                    v[4] += tx;
                    v[5] += ty;
                    v[6] += tx * dx;
                    v[7] += tx * dy;
                    v[8] += ty * dy;
                }
#pragma unroll
                for (int c = 0; c < 3; ++c) cacc[p][c] = after[c];
                T[p] = __fmul_rn(Tk, am1);
            }
            if (__ballot_sync(0xffffffffu, any) == 0u) continue;
#pragma unroll
            for (int c = 0; c < 9; ++c) v[c] = warp_sum(v[c]);
            if (lane == 0) {
#pragma unroll
                for (int c = 0; c < 9; ++c)
                    if (v[c] != 0.f) atomicAdd(&s_acc[c][j], v[c]);
            }
        }
        __syncthreads();
        // one row per (tile, list position), conic/sigma factors applied here
        for (int k = t; k < nb; k += kPxThreads) {
            const float4 A = s_rec[k].a, B = s_rec[k].b;
            const float sdx = s_acc[4][k], sdy = s_acc[5][k];
            const float c1 = 0.5f * A.w;
            float r[9];
            r[0] = s_acc[0][k];
            r[1] = s_acc[1][k];
            r[2] = s_acc[2][k];
            r[3] = A.z * sdx + c1 * sdy;
            r[4] = c1 * sdx + B.x * sdy;
            r[5] = -0.5f * s_acc[6][k];
            r[6] = -s_acc[7][k];
            r[7] = -0.5f * s_acc[8][k];
            r[8] = s_acc[3][k] / B.y;
            float* row = g2d + (size_t)s_id[k] * 9;
#pragma unroll
            for (int c = 0; c < 9; ++c)
                if (r[c] != 0.f) atomicAdd(row + c, r[c]);
        }
        __syncthreads();
    }
}

__global__ void px_clear_kernel(float* __restrict__ g2d, int64_t nf) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nf;
         k += (int64_t)gridDim.x * blockDim.x)
        g2d[k] = 0.f;
}

cudaError_t launch_backward_pixel(const ss_camera* cam, const ss_raster_opts* o,
                                  const ss_splats* sp, const ss_bins* bins, const float* image,
                                  const float* grad_image, const int32_t* n_contrib,
                                  const int32_t* k_eff, int64_t n, float* g2d, cudaStream_t s) {
    const int tx = div_up(cam->width, kTile), ty = div_up(cam->height, kTile);
    px_clear_kernel<<<div_up(n * 9 > 0 ? n * 9 : 1, 1024), 256, 0, s>>>(g2d, n * 9);
    backward_pixel_kernel<<<tx * ty, kPxThreads, 0, s>>>(
        cam->width, cam->height, tx, bins->d_tile_start, k_eff, bins->d_pair_splat,
        reinterpret_cast<const SplatRec*>(sp->d_rec), o->alpha_min, o->alpha_max, image,
        grad_image, n_contrib, g2d);
    return cudaGetLastError();
}

}  // namespace ss
