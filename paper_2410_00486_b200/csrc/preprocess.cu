// preprocess.cu -- K1: per-Gaussian EWA projection, SH colour, footprint
// radius and inclusive tile rectangle, over the SoA map.
//
// Restates project_map (rasterizer/projection.py:73-163) in float32, one
// thread per Gaussian (no compaction: culled Gaussians get tiles = 0 and a
// max depth key, so every later stage indexes by Gaussian id), and the
// tile-rectangle half of build_tile_index (rasterizer/tiles.py:40-48).
// Also folds rasterize_forward's finite-parameter check (api.py:127-129,
// core.py:231-241) and the zero-quaternion check (projection.py:99-102)
// into device error words.
#include <cuda_fp16.h>

#include "common.cuh"
#include "sh.cuh"

namespace ss {

struct CamF {
    float fx, fy, cx, cy;
    int W, H;
    float R[9], t[3], c[3];
};

__device__ __forceinline__ void load_camf(const ss_camera* __restrict__ c, CamF& f) {
    f.fx = c->fx;
    f.fy = c->fy;
    f.cx = c->cx;
    f.cy = c->cy;
    f.W = c->width;
    f.H = c->height;
#pragma unroll
    for (int k = 0; k < 9; ++k) f.R[k] = c->R[k];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        f.t[k] = c->t[k];
        f.c[k] = c->center[k];
    }
}

__device__ __forceinline__ float sigmoid_stable(float x) {
    // projection.py:68-70
    float e = expf(-fabsf(x));
    return x >= 0.f ? 1.0f / (1.0f + e) : e / (1.0f + e);
}

// Camera-frame covariance and the dilated 2D covariance (projection.py:98-121).
struct Proj2D {
    float t[3];
    float a, b, c;
};

__device__ __forceinline__ void project_cov(const float p[3], const float4 q, const float ls[3],
                                            const CamF& cam, float dilation, Proj2D& o,
                                            float qhat[4], float rot[9], float s2[3],
                                            float covc[9], float& qn) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
        o.t[i] = p[0] * cam.R[3 * i] + p[1] * cam.R[3 * i + 1] + p[2] * cam.R[3 * i + 2] + cam.t[i];
    qn = sqrtf(q.x * q.x + q.y * q.y + q.z * q.z + q.w * q.w);
    float inv = 1.0f / qn;
    qhat[0] = q.x * inv;
    qhat[1] = q.y * inv;
    qhat[2] = q.z * inv;
    qhat[3] = q.w * inv;
    quat_to_rot(qhat, rot);
#pragma unroll
    for (int k = 0; k < 3; ++k) s2[k] = expf(2.0f * ls[k]);
    // cov3 = R diag(s2) R^T ; covc = Rcw cov3 Rcw^T
    float M[9];  // M = Rcw * R  -> covc = M diag(s2) M^T
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            M[3 * i + j] = cam.R[3 * i] * rot[j] + cam.R[3 * i + 1] * rot[3 + j] +
                           cam.R[3 * i + 2] * rot[6 + j];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int l = 0; l < 3; ++l)
            covc[3 * i + l] = M[3 * i] * s2[0] * M[3 * l] + M[3 * i + 1] * s2[1] * M[3 * l + 1] +
                              M[3 * i + 2] * s2[2] * M[3 * l + 2];
    float iz = 1.0f / o.t[2], iz2 = iz * iz;
    float j00 = cam.fx * iz, j02 = -cam.fx * o.t[0] * iz2;
    float j11 = cam.fy * iz, j12 = -cam.fy * o.t[1] * iz2;
    // c2 = J covc J^T with J = [[j00,0,j02],[0,j11,j12]]
    float r0[3] = {j00 * covc[0] + j02 * covc[6], j00 * covc[1] + j02 * covc[7],
                   j00 * covc[2] + j02 * covc[8]};
    float r1[3] = {j11 * covc[3] + j12 * covc[6], j11 * covc[4] + j12 * covc[7],
                   j11 * covc[5] + j12 * covc[8]};
    o.a = r0[0] * j00 + r0[2] * j02 + dilation;
    o.b = r0[1] * j11 + r0[2] * j12;
    o.c = r1[1] * j11 + r1[2] * j12 + dilation;
}

__global__ void __launch_bounds__(256) preprocess_kernel(
    int64_t n, const float* __restrict__ pos, const float4* __restrict__ rot,
    const float* __restrict__ ls, const float* __restrict__ opl, const float* __restrict__ sh_dc,
    const float* __restrict__ sh_rest, CamF cam_v, const ss_camera* __restrict__ d_cam,
    int sh_degree, float near_plane, float dilation, float log_amin, int tiles_x, int tiles_y,
    SplatRec* __restrict__ rec,
    uint32_t* __restrict__ depth_key, uint32_t* __restrict__ tiles, uint2* __restrict__ rect,
    uint8_t* __restrict__ flags, float* __restrict__ aux, ss_status* status) {
    PDL_WAIT();
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    CamF cam = cam_v;
    if (d_cam) load_camf(d_cam, cam);  // graph replay: camera from device memory
    // SH bands 1-3 (sh_degree > 0): a thread's 45-float row is strided 180 B
    // from its neighbour's, so the CTA's 256 rows (one contiguous span) are
    // staged through shared memory with coalesced loads first
    extern __shared__ __align__(16) float s_rest[];
    const float* my_rest = sh_rest + 45 * i;
    if (sh_degree > 0) {
        const int64_t r0 = blockIdx.x * (int64_t)blockDim.x;
        const int64_t nr = min((int64_t)blockDim.x, n - r0);
        const float* src = sh_rest + 45 * r0;
        if (nr == blockDim.x && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
            // every 16-byte piece of the span in flight at once (cp.async, no registers)
            const int n4 = 45 * (int)nr / 4;
            const uint32_t dst = (uint32_t)__cvta_generic_to_shared(s_rest);
            for (int k = threadIdx.x; k < n4; k += blockDim.x)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16 * k),
                             "l"(src + 4 * k)
                             : "memory");
            asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
        } else {
            for (int k = threadIdx.x; k < 45 * nr; k += blockDim.x) s_rest[k] = src[k];
        }
        __syncthreads();
        my_rest = s_rest + 45 * threadIdx.x;
    }
    bool vis = false;
    if (i < n) {
        float p[3] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
        float4 q = rot[i];
        float l[3] = {ls[3 * i], ls[3 * i + 1], ls[3 * i + 2]};
        float o = opl[i];
        float dc[3] = {sh_dc[3 * i], sh_dc[3 * i + 1], sh_dc[3 * i + 2]};
        bool fin = finitef(p[0]) && finitef(p[1]) && finitef(p[2]) && finitef(q.x) &&
                   finitef(q.y) && finitef(q.z) && finitef(q.w) && finitef(l[0]) &&
                   finitef(l[1]) && finitef(l[2]) && finitef(o) && finitef(dc[0]) &&
                   finitef(dc[1]) && finitef(dc[2]);
        if (sh_degree > 0) {
            // sh_rest only changes when it is optimised (sh_degree > 0); at
            // degree 0 the host validates it once on upload.
            // non-short-circuit: all 45 loads in flight (a && chain waits on each)
            bool rf = true;
#pragma unroll 15
            for (int k = 0; k < 45; ++k) rf &= finitef(my_rest[k]);
            fin = fin && rf;
        }
        if (!fin) report_first(&status->first_nonfinite_param, i);

        float z = p[0] * cam.R[6] + p[1] * cam.R[7] + p[2] * cam.R[8] + cam.t[2];
        uint32_t ntiles = 0;
        uint2 rc = make_uint2(0u, 0u);
        uint8_t fl = 0;
        SplatRec r;
        r.a = make_float4(0.f, 0.f, 0.f, 0.f);
        r.b = make_float4(0.f, 0.f, -1.f, 0.f);
        r.c = make_float4(0.f, 0.f, 0.f, 0.f);
        float auxv[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (z > near_plane) {
            float qn2 = q.x * q.x + q.y * q.y + q.z * q.z + q.w * q.w;
            if (qn2 == 0.0f) report_first(&status->first_zero_quat, i);
            Proj2D P;
            float qhat[4], R9[9], s2[3], covc[9], qn;
            project_cov(p, q, l, cam, dilation, P, qhat, R9, s2, covc, qn);
            float mx = cam.fx * P.t[0] / P.t[2] + cam.cx;
            float my = cam.fy * P.t[1] / P.t[2] + cam.cy;
            float det = P.a * P.c - P.b * P.b;
            float mid = (P.a + P.c) / 2.0f;
            float disc = mid * mid - det;
            float lmax = mid + sqrtf(fmaxf(disc, 0.0f));
            float sg = sigmoid_stable(o);
            float mcut = 2.0f * (logf(sg) - log_amin);
            float rad = ceilf(sqrtf(fmaxf(mcut, 0.0f) * lmax));
            vis = (det > 0.f) && (mcut > 0.f) && (mx + rad >= 0.f) &&
                  (mx - rad <= (float)(cam.W - 1)) && (my + rad >= 0.f) &&
                  (my - rad <= (float)(cam.H - 1)) && (qn2 != 0.0f);
            if (vis) {
                // tiles.py:42-47: inclusive rect, float32 arithmetic as numpy
                // (x / 16 and x * (1/16) round identically: a power of two)
                float fx0 = floorf(__fmul_rn(__fsub_rn(mx, rad), 1.0f / kTile));
                float fx1 = floorf(__fmul_rn(__fadd_rn(mx, rad), 1.0f / kTile));
                float fy0 = floorf(__fmul_rn(__fsub_rn(my, rad), 1.0f / kTile));
                float fy1 = floorf(__fmul_rn(__fadd_rn(my, rad), 1.0f / kTile));
                int x0 = (int)fminf(fmaxf(fx0, 0.f), (float)(tiles_x - 1));
                int x1 = (int)fminf(fmaxf(fx1, 0.f), (float)(tiles_x - 1));
                int y0 = (int)fminf(fmaxf(fy0, 0.f), (float)(tiles_y - 1));
                int y1 = (int)fminf(fmaxf(fy1, 0.f), (float)(tiles_y - 1));
                ntiles = (uint32_t)((x1 - x0 + 1) * (y1 - y0 + 1));
                rc = make_uint2((uint32_t)x0 | ((uint32_t)y0 << 16),
                                (uint32_t)x1 | ((uint32_t)y1 << 16));
                // colour (projection.py:147-155)
                float rgb[3];
                bool act[3];
                if (sh_degree == 0) {  // view-independent: no direction needed
#pragma unroll
                    for (int ch = 0; ch < 3; ++ch) {
                        const float raw = kSH_C0 * dc[ch] + 0.5f;
                        act[ch] = raw > 0.f;
                        rgb[ch] = fmaxf(raw, 0.f);
                    }
                } else {
                    float u[3] = {p[0] - cam.c[0], p[1] - cam.c[1], p[2] - cam.c[2]};
                    float vl = fmaxf(sqrtf(u[0] * u[0] + u[1] * u[1] + u[2] * u[2]), 1e-12f);
                    float d[3] = {u[0] / vl, u[1] / vl, u[2] / vl};
                    sh_color(d, sh_degree, dc, my_rest, rgb, act);
                }
                fl = 1u | (act[0] ? 2u : 0u) | (act[1] ? 4u : 0u) | (act[2] ? 8u : 0u);
                r.a = make_float4(mx, my, P.c / det, 2.0f * (-P.b / det));
                r.b = make_float4(P.a / det, sg, mcut, P.t[2]);
                // half-extents of the blend region m <= m_cut
                // (sqrt(m_cut * cov_xx), sqrt(m_cut * cov_yy)) + 1 px margin,
                // as a half2 rounded up: lets a warp of the forward skip
                // splats that cannot reach its rows (blend_forward.cu)
                const float ext_x = sqrtf(fmaxf(mcut, 0.0f) * P.a) * 1.0001f + 1.0f;
                const float ext_y = sqrtf(fmaxf(mcut, 0.0f) * P.c) * 1.0001f + 1.0f;
                const __half2 ext = __halves2half2(__float2half_ru(fminf(ext_x, 60000.f)),
                                                   __float2half_ru(fminf(ext_y, 60000.f)));
                r.c = make_float4(rgb[0], rgb[1], rgb[2], *reinterpret_cast<const float*>(&ext));
                auxv[0] = P.t[0];
                auxv[1] = P.t[1];
                auxv[2] = P.t[2];
                auxv[3] = P.a;
                auxv[4] = P.b;
                auxv[5] = P.c;
                auxv[6] = rad;
            }
        }
        rec[i] = r;
        depth_key[i] = vis ? __float_as_uint(z) : 0xFFFFFFFFu;
        tiles[i] = ntiles;
        rect[i] = rc;
        flags[i] = fl;
        if (aux) {
            float4* a4 = reinterpret_cast<float4*>(aux + 8 * i);
            a4[0] = make_float4(auxv[0], auxv[1], auxv[2], auxv[3]);
            a4[1] = make_float4(auxv[4], auxv[5], auxv[6], auxv[7]);
        }
    }
    unsigned bal = __ballot_sync(0xffffffffu, vis);
    if (lane_id() == 0 && bal)
        atomicAdd(reinterpret_cast<unsigned long long*>(&status->visible_count),
                  (unsigned long long)__popc(bal));
    // opacity regulariser value, sum of sigmoid(logit) over ALL Gaussians
    // with the pre-update logits (losses.py:157-168)
    __shared__ double s_os[8];
    double os = warp_sum(i < n ? (double)sigmoid_stable(opl[i]) : 0.0);
    if (lane_id() == 0) s_os[threadIdx.x >> 5] = os;
    __syncthreads();
    if (threadIdx.x == 0) {
        double b = 0.0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) b += s_os[k];
        atomicAdd(&status->opacity_sum, b);
    }
}

// build_tile_index (tiles.py:29-65) fed an external projection: the K1
// outputs the binning reads (inclusive tile rect in float32 arithmetic as
// numpy does, tile count, depth key) for m projection rows; the pair list
// then holds row indices, as the reference's pair_splat does.
__global__ void splats_from_projection_kernel(int64_t m, const float* __restrict__ mean2d,
                                              const float* __restrict__ radius,
                                              const float* __restrict__ depth, int tiles_x,
                                              int tiles_y, SplatRec* __restrict__ rec,
                                              uint32_t* __restrict__ depth_key,
                                              uint32_t* __restrict__ tiles,
                                              uint2* __restrict__ rect, uint8_t* __restrict__ flags) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    const float mx = mean2d[2 * i], my = mean2d[2 * i + 1], rad = radius[i], z = depth[i];
    const float fx0 = floorf(__fmul_rn(__fsub_rn(mx, rad), 1.0f / kTile));
    const float fx1 = floorf(__fmul_rn(__fadd_rn(mx, rad), 1.0f / kTile));
    const float fy0 = floorf(__fmul_rn(__fsub_rn(my, rad), 1.0f / kTile));
    const float fy1 = floorf(__fmul_rn(__fadd_rn(my, rad), 1.0f / kTile));
    const int x0 = (int)fminf(fmaxf(fx0, 0.f), (float)(tiles_x - 1));
    const int x1 = (int)fminf(fmaxf(fx1, 0.f), (float)(tiles_x - 1));
    const int y0 = (int)fminf(fmaxf(fy0, 0.f), (float)(tiles_y - 1));
    const int y1 = (int)fminf(fmaxf(fy1, 0.f), (float)(tiles_y - 1));
    SplatRec r;
    r.a = make_float4(mx, my, 0.f, 0.f);
    r.b = make_float4(0.f, 0.f, 0.f, z);
    r.c = make_float4(0.f, 0.f, 0.f, 0.f);
    rec[i] = r;
    depth_key[i] = __float_as_uint(z);
    tiles[i] = (uint32_t)((x1 - x0 + 1) * (y1 - y0 + 1));
    rect[i] = make_uint2((uint32_t)x0 | ((uint32_t)y0 << 16), (uint32_t)x1 | ((uint32_t)y1 << 16));
    flags[i] = 1;
}

cudaError_t launch_splats_from_projection(int64_t m, const float* mean2d, const float* radius,
                                          const float* depth, const ss_camera* cam,
                                          const ss_splats* out, cudaStream_t s) {
    if (m == 0) return cudaSuccess;
    splats_from_projection_kernel<<<div_up(m, 256), 256, 0, s>>>(
        m, mean2d, radius, depth, div_up(cam->width, kTile), div_up(cam->height, kTile),
        reinterpret_cast<SplatRec*>(out->d_rec), out->d_depth_key, out->d_tiles,
        reinterpret_cast<uint2*>(out->d_rect), out->d_flags);
    return cudaGetLastError();
}

void fill_camf(const ss_camera* c, CamF& f) {
    f.fx = c->fx;
    f.fy = c->fy;
    f.cx = c->cx;
    f.cy = c->cy;
    f.W = c->width;
    f.H = c->height;
    for (int k = 0; k < 9; ++k) f.R[k] = c->R[k];
    for (int k = 0; k < 3; ++k) {
        f.t[k] = c->t[k];
        f.c[k] = c->center[k];
    }
}

cudaError_t launch_preprocess(const ss_map* map, const ss_camera* cam, const ss_camera* d_cam,
                              const ss_raster_opts* o, const ss_splats* out, ss_status* st,
                              cudaStream_t s) {
    if (map->n == 0) return cudaSuccess;
    CamF cf;
    fill_camf(cam, cf);
    int tx = div_up(cam->width, kTile), ty = div_up(cam->height, kTile);
    int threads = 256;
    int blocks = div_up(map->n, threads);
    const size_t smem = o->sh_degree > 0 ? sizeof(float) * 45 * threads : 0;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(preprocess_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    launch_pdl(preprocess_kernel, dim3(blocks), dim3(threads), smem, s,
        map->n, map->d_positions, reinterpret_cast<const float4*>(map->d_rotations),
        map->d_log_scales, map->d_opacity_logits, map->d_sh_dc, map->d_sh_rest, cf, d_cam,
        o->sh_degree, o->near_plane, o->dilation, logf(o->alpha_min), tx, ty,
        reinterpret_cast<SplatRec*>(out->d_rec), out->d_depth_key, out->d_tiles,
        reinterpret_cast<uint2*>(out->d_rect), out->d_flags, out->d_aux, st);
    return cudaGetLastError();
}

}  // namespace ss
