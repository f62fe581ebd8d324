// loss.cu -- K6: fused L1 + SSIM loss and its analytic image gradient,
// plus the opacity regulariser and the builder-defined depth term.
//
// Restates compute_losses (losses.py:198-228) with _ssim_terms (:99-109),
// _ssim_with_grad (:119-134), the separable 11-tap Gaussian window
// (sigma 1.5, losses.py:23-28) with mirror padding (losses.py:31-55) and
// its exact adjoint (losses.py:69-88): the adjoint of "reflect-pad then
// correlate" spreads each value over the padded domain and folds the
// padded positions back through the reflection; for an axis of length
// n >= 6 that fold is
//     out[i] = gp(i) + [1<=i<=5] gp(-i) + [n-6<=i<=n-2] gp(2n-2-i),
//     gp(u)  = sum_m w[m] g[u-5+m]   (g zero outside [0, n)).
// Two tiled kernels, 32x32 output pixels per CTA, 5-pixel halo in shared
// memory, channels processed in turn:
//   ssim_fwd : moments (x, y, x^2, y^2, xy), SSIM map and the three
//              gradient maps dS/d(mu_x), dS/d(F x^2), dS/d(F xy), per-CTA
//              partial sums of |x - y| and SSIM;
//   ssim_bwd : the folded adjoint of the three maps, combined into
//              (1-l) sign(x-y)/n - l (F*g_mu + 2x F*g_xx + y F*g_xy).
#include "common.cuh"

namespace ss {

constexpr int LR = 5;                 // half window
constexpr int LT = 32;                // output tile side
constexpr int LH = LT + 2 * LR;       // 42: halo side
constexpr int LP = 44;                // padded row pitch (float4 rows)

#ifdef SS_FWD_TRACE
// diagnostics build only: per-CTA (smid, start, end) of ssim_fwd [0] and ssim_bwd [1]
__device__ unsigned long long g_ssim_trace[2][4 * 4096];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    return v;
}
#define SSIM_TRACE_BEGIN const unsigned long long tr0 = gtimer();
#define SSIM_TRACE_END(K)                                                          \
    if (threadIdx.x == 0) {                                                        \
        uint32_t smid;                                                             \
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));                          \
        const int b = blockIdx.y * gridDim.x + blockIdx.x;                         \
        if (b < 4096) {                                                            \
            g_ssim_trace[K][4 * b] = b;                                            \
            g_ssim_trace[K][4 * b + 1] = smid;                                     \
            g_ssim_trace[K][4 * b + 2] = tr0;                                      \
            g_ssim_trace[K][4 * b + 3] = gtimer();                                 \
        }                                                                          \
    }
#else
#define SSIM_TRACE_BEGIN
#define SSIM_TRACE_END(K)
#endif

struct SsimWindow {
    float w[11];
    double wd[11];  // the same weights widened (exact), for the float64 vertical taps
};

__device__ __forceinline__ int reflect1(int i, int n) {
    // symmetric reflection without edge repeat (losses.py:31-41), n >= 6
    if (i < 0) i = -i;
    if (i >= n) i = 2 * n - 2 - i;
    return i;
}

// 4-byte global -> shared copy that bypasses registers (zero-fills when
// !valid); the halo of the next channel streams in under the current
// channel's compute.
__device__ __forceinline__ void cp_async4(float* dst, const float* src, bool valid) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(src),
                 "r"(valid ? 4 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// 11-tap correlation of 4 consecutive outputs from 14 register values.
__device__ __forceinline__ void taps4(const float* v, const SsimWindow& win, float out[4]) {
#pragma unroll
    for (int o = 0; o < 4; ++o) {
        float a = 0.f;
#pragma unroll
        for (int m = 0; m < 11; ++m) a += win.w[m] * v[o + m];
        out[o] = a;
    }
}

// 11-tap correlation of 4 consecutive outputs of a packed (lo, hi) pair of
// quantities: FFMA2 with the tap weight broadcast to both lanes.
__device__ __forceinline__ void taps4x2(const f32x2* v, const SsimWindow& win, f32x2 out[4]) {
#pragma unroll
    for (int o = 0; o < 4; ++o) {
        f32x2 a = pk2(0.f, 0.f);
#pragma unroll
        for (int m = 0; m < 11; ++m) a = fma2(pk2(win.w[m], win.w[m]), v[o + m], a);
        out[o] = a;
    }
}

// Tiles of 32x32 output pixels, one channel at a time; both separable
// passes give every thread 4 consecutive outputs from one register window
// (14 loads per 4 outputs instead of 11 per output).  The five moments run
// as two packed pairs, (x, y) and (x^2, y^2), plus xy: FFMA2 halves the
// issue slots of four of them.
__global__ void __launch_bounds__(256, 3) ssim_fwd_kernel(int H, int W, const float* __restrict__ x,
                                                       const float* __restrict__ y,
                                                       SsimWindow win, float* __restrict__ gmu,
                                                       float* __restrict__ gxx,
                                                       float* __restrict__ gxy,
                                                       double* __restrict__ partials) {
    __shared__ __align__(16) float2 s_xy[LH][LP];   // (x, y) halo
    __shared__ __align__(16) float2 shp[LH][LT];   // horizontal pass: (x, y)
    __shared__ __align__(16) float2 shq[LH][LT];   //                  (x^2, y^2)
    __shared__ __align__(16) float shm[LH][LT];    //                  xy
    __shared__ double red[2][8];
    __shared__ float s_shift[2][8];
    PDL_WAIT();
    SSIM_TRACE_BEGIN
    const int t = threadIdx.x;
    const int x0 = blockIdx.x * LT, y0 = blockIdx.y * LT;
    const double C1d = 0.01 * 0.01, C2d = 0.03 * 0.03;
    const double gsd = 1.0 / ((double)H * W * 3);
    double l1 = 0.0, ssum = 0.0;
    // vertical-pass task of this thread: column q, rows 4 rg .. 4 rg + 3
    const int q = t & 31, rg = t >> 5;
    for (int c = 0; c < 3; ++c) {
        {
            // halo: all 7 loads per thread in flight before the stores
            constexpr int NL = (LH * LH + 255) / 256;
            float vx[NL], vy[NL];
#pragma unroll
            for (int i = 0; i < NL; ++i) {
                const int k = t + 256 * i;
                const int r = k / LH, cc = k - r * LH;
                const int gy = reflect1(y0 - LR + r, H), gx = reflect1(x0 - LR + cc, W);
                const size_t o = ((size_t)gy * W + gx) * 3 + c;
                vx[i] = k < LH * LH ? x[o] : 0.f;
                vy[i] = k < LH * LH ? y[o] : 0.f;
            }
            float hx = INFINITY, hy = INFINITY;
#pragma unroll
            for (int i = 0; i < NL; ++i) {
                const int k = t + 256 * i;
                if (k < LH * LH) {
                    const int r = k / LH, cc = k - r * LH;
                    s_xy[r][cc] = make_float2(vx[i], vy[i]);
                    hx = fminf(hx, vx[i]);
                    hy = fminf(hy, vy[i]);
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                hx = fminf(hx, __shfl_xor_sync(0xffffffffu, hx, o));
                hy = fminf(hy, __shfl_xor_sync(0xffffffffu, hy, o));
            }
            if ((t & 31) == 0) {
                s_shift[0][t >> 5] = hx;
                s_shift[1][t >> 5] = hy;
            }
        }
        __syncthreads();
        // The CTA's moments are taken about its halo minima (cx, cy): every
        // output's window lies inside this halo, so sxx = F((x-cx)^2) -
        // (F(x)-cx)^2 holds exactly, and the shift trims the float32
        // cancellation of F(x^2) - F(x)^2 where a tile has no black pixels
        // (exact zeros keep the unshifted, exact arithmetic).  With the
        // epilogue below in float64, grad_image is within ~5e-6 norm-wise and
        // ~8e-6 max-abs of the float64 oracle at configs[1] (float32
        // emulation: 1.2e-5 / 1.4e-5 without both).
        float cx = INFINITY, cy = INFINITY;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            cx = fminf(cx, s_shift[0][k]);
            cy = fminf(cy, s_shift[1][k]);
        }
        // horizontal (axis 1): 42 rows x 8 groups of 4 columns
        for (int task = t; task < LH * 8; task += 256) {
            const int r = task >> 3, c0 = (task & 7) * 4;
            f32x2 pv[14], qv[14];
            float mv[14];
#pragma unroll
            for (int k = 0; k < 7; ++k) {
                const float4 a = *reinterpret_cast<const float4*>(&s_xy[r][c0 + 2 * k]);
                const float ax = a.x - cx, ay = a.y - cy, az = a.z - cx, aw = a.w - cy;
                pv[2 * k] = pk2(ax, ay);
                pv[2 * k + 1] = pk2(az, aw);
                mv[2 * k] = ax * ay;
                mv[2 * k + 1] = az * aw;
            }
#pragma unroll
            for (int k = 0; k < 14; ++k) qv[k] = mul2(pv[k], pv[k]);
            f32x2 o2[4];
            float o4[4];
            taps4x2(pv, win, o2);
            *reinterpret_cast<float4*>(&shp[r][c0]) = *reinterpret_cast<const float4*>(&o2[0]);
            *reinterpret_cast<float4*>(&shp[r][c0 + 2]) = *reinterpret_cast<const float4*>(&o2[2]);
            taps4x2(qv, win, o2);
            *reinterpret_cast<float4*>(&shq[r][c0]) = *reinterpret_cast<const float4*>(&o2[0]);
            *reinterpret_cast<float4*>(&shq[r][c0 + 2]) = *reinterpret_cast<const float4*>(&o2[2]);
            taps4(mv, win, o4);
            *reinterpret_cast<float4*>(&shm[r][c0]) = make_float4(o4[0], o4[1], o4[2], o4[3]);
        }
        __syncthreads();
        // vertical (axis 0): column q, 4 consecutive rows
        float mom[2][4];
        double mom2[3][4];  // second moments: the vertical taps accumulate in float64
        {
            f32x2 v2[14], o2[4];
#pragma unroll
            for (int i = 0; i < 14; ++i) {
                const float2 e = shp[4 * rg + i][q];
                v2[i] = pk2(e.x, e.y);
            }
            taps4x2(v2, win, o2);
#pragma unroll
            for (int o = 0; o < 4; ++o) upk2(o2[o], mom[0][o], mom[1][o]);
            float vx[14], vy[14], vm[14];
#pragma unroll
            for (int i = 0; i < 14; ++i) {
                const float2 e = shq[4 * rg + i][q];
                vx[i] = e.x;
                vy[i] = e.y;
                vm[i] = shm[4 * rg + i][q];
            }
#pragma unroll
            for (int o = 0; o < 4; ++o) {
                double axx = 0.0, ayy = 0.0, axy = 0.0;
#pragma unroll
                for (int m = 0; m < 11; ++m) {
                    const double wd = win.wd[m];
                    axx = fma(wd, (double)vx[o + m], axx);
                    ayy = fma(wd, (double)vy[o + m], ayy);
                    axy = fma(wd, (double)vm[o + m], axy);
                }
                mom2[0][o] = axx;
                mom2[1][o] = ayy;
                mom2[2][o] = axy;
            }
        }
        const int ox = x0 + q;
#pragma unroll
        for (int o = 0; o < 4; ++o) {
            const int oy = y0 + 4 * rg + o;
            if (ox < W && oy < H) {
                // epilogue in float64 (losses.py:99-109,119-134): ~30 flops per
                // output, small next to the 110 float32 moment taps
                const double mxs = mom[0][o], mys = mom[1][o];  // means about (cx, cy)
                const double sxx = mom2[0][o] - mxs * mxs, syy = mom2[1][o] - mys * mys;
                const double sxy = mom2[2][o] - mxs * mys;
                const double mx = mxs + cx, my = mys + cy;
                const double a1 = 2.0 * mx * my + C1d, a2 = 2.0 * sxy + C2d;
                const double b1 = mx * mx + my * my + C1d, b2 = sxx + syy + C2d;
                // 1/(b1 b2) (then 1/b1 = b2/bb, 1/b2 = b1/bb): a float seed and two
                // Newton steps in float64 instead of the slow IEEE double divide
                const double bb = b1 * b2;
                double ibb = (double)rcp_approx((float)bb);
                ibb = ibb * fma(-bb, ibb, 2.0);
                ibb = ibb * fma(-bb, ibb, 2.0);
                const double ss = a1 * a2 * ibb;
                const double ga1 = gsd * a2 * ibb, ga2 = gsd * a1 * ibb;
                const double gb1 = -gsd * ss * (b2 * ibb), gb2 = -gsd * ss * (b1 * ibb);
                // gradient maps are workspace: planar per channel, so the
                // adjoint kernel's halo loads are coalesced
                const size_t go = ((size_t)c * H + oy) * W + ox;
                gmu[go] = (float)(2.0 * my * ga1 + 2.0 * mx * gb1 - 2.0 * mx * gb2 - my * 2.0 * ga2);
                gxx[go] = (float)gb2;
                gxy[go] = (float)(2.0 * ga2);
                ssum += ss;
                const float2 e = s_xy[LR + 4 * rg + o][LR + q];
                l1 += (double)fabsf(e.x - e.y);
            }
        }
        __syncthreads();
    }
    l1 = warp_sum(l1);
    ssum = warp_sum(ssum);
    if ((t & 31) == 0) {
        red[0][t >> 5] = l1;
        red[1][t >> 5] = ssum;
    }
    __syncthreads();
    if (t == 0) {
        double a = 0.0, b = 0.0;
        for (int k = 0; k < 8; ++k) {
            a += red[0][k];
            b += red[1][k];
        }
        const size_t bid = (size_t)blockIdx.y * gridDim.x + blockIdx.x;
        partials[2 * bid] = a;
        partials[2 * bid + 1] = b;
    }
    SSIM_TRACE_END(0)
}

// gp(u) = sum_m w[m] g[u - 5 + m] over a zero-extended shared line; lc is
// the local index of u - 5, `at(k)` reads local element k (0 <= k < LH).
template <typename AT>
__device__ __forceinline__ float gp_line(int lc, const SsimWindow& win, AT at) {
    float a = 0.f;
#pragma unroll
    for (int m = 0; m < 11; ++m) {
        const int k = lc + m;
        a += (k >= 0 && k < LH) ? win.w[m] * at(k) : 0.f;
    }
    return a;
}

// Mirror-fold extras of the adjoint for global index i on an axis of
// length n whose local index 0 is global org - 5.
template <typename AT>
__device__ __forceinline__ float fold_extra(int i, int n, int org, const SsimWindow& win, AT at) {
    float r = 0.f;
    if (i >= 1 && i <= LR) r += gp_line(-i - org, win, at);
    if (i >= n - 6 && i <= n - 2) r += gp_line(2 * n - 2 - i - org, win, at);
    return r;
}

__global__ void __launch_bounds__(256, 3) ssim_bwd_kernel(int H, int W, const float* __restrict__ x,
                                                       const float* __restrict__ y,
                                                       SsimWindow win,
                                                       const float* __restrict__ gmu,
                                                       const float* __restrict__ gxx,
                                                       const float* __restrict__ gxy, float lam,
                                                       float* __restrict__ grad,
                                                       float4* __restrict__ pixgrad,
                                                       const double* __restrict__ partials,
                                                       int n_partials,
                                                       double* __restrict__ sums) {
    extern __shared__ __align__(16) float smem_b[];
    PDL_WAIT();
    SSIM_TRACE_BEGIN
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x < 32) {
        // fixed-order reduction of ssim_fwd's per-CTA (|x-y|, SSIM) sums
        double a = 0.0, b = 0.0;
        for (int i = threadIdx.x; i < n_partials; i += 32) {
            a += partials[2 * i];
            b += partials[2 * i + 1];
        }
        a = warp_sum(a);
        b = warp_sum(b);
        if (threadIdx.x == 0) {
            sums[0] = a;
            sums[1] = b;
        }
    }
    float(*sgb)[3][LH][LP] = reinterpret_cast<float(*)[3][LH][LP]>(smem_b);          // [2]
    float(*sh)[LH][LT] = reinterpret_cast<float(*)[LH][LT]>(smem_b + 6 * LH * LP);  // [3]
    const int t = threadIdx.x;
    const int x0 = blockIdx.x * LT, y0 = blockIdx.y * LT;
    const double inv_nd = 1.0 / ((double)H * W * 3);
    const int q = t & 31, rg = t >> 5;
    const int ox = x0 + q;
    float gdot[4] = {0.f, 0.f, 0.f, 0.f};
    float* pg = reinterpret_cast<float*>(pixgrad);
    const bool xborder = x0 <= LR || x0 + LT - 1 >= W - 6;
    const bool yborder = y0 <= LR || y0 + LT - 1 >= H - 6;
    // halo of channel c (zero outside the image) into buffer b
    auto issue = [&](int c, int b) {
        for (int k = t; k < LH * LH; k += 256) {
            const int r = k / LH, cc = k - r * LH;
            const int gy = y0 - LR + r, gx = x0 - LR + cc;
            const bool in = gy >= 0 && gy < H && gx >= 0 && gx < W;
            const size_t o = ((size_t)c * H + (in ? gy : 0)) * W + (in ? gx : 0);
            cp_async4(&sgb[b][0][r][cc], gmu + o, in);
            cp_async4(&sgb[b][1][r][cc], gxx + o, in);
            cp_async4(&sgb[b][2][r][cc], gxy + o, in);
        }
        cp_async_commit();
    };
    issue(0, 0);
    for (int c = 0; c < 3; ++c) {
        if (c < 2) {
            issue(c + 1, (c + 1) & 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        float(*sg)[LH][LP] = sgb[c & 1];
        // axis 1 (columns) first, as losses.py:87-88
        for (int task = t; task < LH * 8; task += 256) {
            const int r = task >> 3, c0 = (task & 7) * 4;
#pragma unroll
            for (int f = 0; f < 3; ++f) {
                float v[16];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const float4 a = *reinterpret_cast<const float4*>(&sg[f][r][c0 + 4 * k]);
                    v[4 * k] = a.x, v[4 * k + 1] = a.y, v[4 * k + 2] = a.z, v[4 * k + 3] = a.w;
                }
                float o4[4];
                taps4(v, win, o4);
                *reinterpret_cast<float4*>(&sh[f][r][c0]) = make_float4(o4[0], o4[1], o4[2], o4[3]);
            }
        }
        __syncthreads();
        if (xborder) {
            // mirror folds of the <= 10 columns next to the image borders as
            // their own (column, row, map) tasks: inside the row pass every
            // warp held a folding lane and ran the fold for all of them
            for (int task = t; task < 2 * LR * LH * 3; task += 256) {
                const int idx = task % (2 * LR), rest = task / (2 * LR);
                const int r = rest % LH, f = rest / LH;
                const int j = idx < LR ? 1 + idx : W - 6 + (idx - LR);
                if (j < x0 || j >= x0 + LT || (idx >= LR && j <= LR)) continue;
                sh[f][r][j - x0] += fold_extra(j, W, x0, win, [&](int k) { return sg[f][r][k]; });
            }
            __syncthreads();
        }
        // axis 0 (rows): column q, 4 consecutive rows; combine
        float adj[3][4];
#pragma unroll
        for (int f = 0; f < 3; ++f) {
            float v[14];
#pragma unroll
            for (int i = 0; i < 14; ++i) v[i] = sh[f][4 * rg + i][q];
            taps4(v, win, adj[f]);
            if (yborder) {
#pragma unroll
                for (int o = 0; o < 4; ++o) {
                    const int i = y0 + 4 * rg + o;  // warp-uniform
                    if ((i >= 1 && i <= LR) || (i >= H - 6 && i <= H - 2))
                        adj[f][o] += fold_extra(i, H, y0, win, [&](int k) { return sh[f][k][q]; });
                }
            }
        }
#pragma unroll
        for (int o = 0; o < 4; ++o) {
            const int oy = y0 + 4 * rg + o;
            if (ox < W && oy < H) {
                const size_t go = ((size_t)oy * W + ox) * 3 + c;
                const float xv = x[go], yv = y[go];
                const float d = xv - yv;
                const float sgn = d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f);  // np.sign(0) = 0
                // the three adjoint terms cancel to a few digits: combine in float64
                const double gx = (double)adj[0][o] + (double)adj[1][o] * (2.0 * xv) +
                                  (double)adj[2][o] * yv;
                const float gv = (float)((1.0 - lam) * sgn * inv_nd - lam * gx);
                if (grad) grad[go] = gv;  // the engine only needs pixgrad
                if (pg) pg[4 * ((size_t)oy * W + ox) + c] = gv;
                gdot[o] += gv * xv;
            }
        }
        __syncthreads();
    }
    if (pg && ox < W) {
#pragma unroll
        for (int o = 0; o < 4; ++o) {
            const int oy = y0 + 4 * rg + o;
            if (oy < H) pg[4 * ((size_t)oy * W + ox) + 3] = gdot[o];
        }
    }
    SSIM_TRACE_END(1)
}

// L1-only variant (lambda_ssim == 0): losses.py:147-153
__global__ void l1_only_kernel(size_t n, const float* __restrict__ x, const float* __restrict__ y,
                               float* __restrict__ grad, double* __restrict__ partials) {
    double acc = 0.0;
    const float inv_n = 1.0f / (float)n;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        float d = x[i] - y[i];
        acc += fabs((double)d);
        grad[i] = (d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f)) * inv_n;
    }
    acc = warp_sum(acc);
    __shared__ double red[32];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) a += red[k];
        partials[2 * blockIdx.x] = a;
        partials[2 * blockIdx.x + 1] = 0.0;
    }
}

// Fixed-order reduction of per-CTA partial pairs into sums[0..1].
__global__ void reduce_pairs_kernel(int nb, const double* __restrict__ partials,
                                    double* __restrict__ sums) {
    double a = 0.0, b = 0.0;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) {
        a += partials[2 * i];
        b += partials[2 * i + 1];
    }
    __shared__ double ra[256], rb[256];
    ra[threadIdx.x] = a;
    rb[threadIdx.x] = b;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) {
            ra[threadIdx.x] += ra[threadIdx.x + s];
            rb[threadIdx.x] += rb[threadIdx.x + s];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        sums[0] = ra[0];
        sums[1] = rb[0];
    }
}

static SsimWindow make_window() {
    SsimWindow w;
    double v[11], s = 0.0;
    for (int m = 0; m < 11; ++m) {
        double xx = m - 5.0;
        v[m] = exp(-(xx * xx) / (2 * 1.5 * 1.5));
        s += v[m];
    }
    for (int m = 0; m < 11; ++m) {
        w.w[m] = (float)(v[m] / s);
        w.wd[m] = (double)w.w[m];
    }
    return w;
}

size_t loss_workspace_bytes(int H, int W) {
    size_t maps = (size_t)H * W * 3 * sizeof(float) * 3;
    size_t nb = (size_t)div_up(W, LT) * div_up(H, LT);
    size_t nb2 = 1184;
    return maps + 2 * sizeof(double) * (nb > nb2 ? nb : nb2) + 512;
}

cudaError_t launch_loss(int H, int W, const float* x, const float* y, float lam, float* grad,
                        float* pixgrad, double* sums, void* ws, size_t ws_bytes, cudaStream_t s) {
    if (ws_bytes < loss_workspace_bytes(H, W)) return cudaErrorInvalidValue;
    size_t plane = (size_t)H * W * 3;
    float* gmu = reinterpret_cast<float*>(ws);
    float* gxx = gmu + plane;
    float* gxy = gxx + plane;
    double* partials = reinterpret_cast<double*>(
        (reinterpret_cast<uintptr_t>(gxy + plane) + 255) & ~uintptr_t(255));
    if (lam == 0.0f) {
        int nb = 1184;
        l1_only_kernel<<<nb, 256, 0, s>>>(plane, x, y, grad, partials);
        reduce_pairs_kernel<<<1, 256, 0, s>>>(nb, partials, sums);
        return cudaGetLastError();
    }
    if (H < 6 || W < 6) return cudaErrorInvalidValue;
    SsimWindow win = make_window();
    dim3 grid(div_up(W, LT), div_up(H, LT));
    const int smem_b = (6 * LH * LP + 3 * LH * LT) * (int)sizeof(float);
    cudaError_t e =
        cudaFuncSetAttribute(ssim_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_b);
    if (e != cudaSuccess) return e;
    launch_pdl(ssim_fwd_kernel, grid, dim3(256), 0, s, H, W, x, y, win, gmu, gxx, gxy, partials);
    launch_pdl(ssim_bwd_kernel, grid, dim3(256), (size_t)smem_b, s, H, W, x, y, win, gmu, gxx, gxy, lam, grad,
                                              reinterpret_cast<float4*>(pixgrad), partials,
                                              (int)(grid.x * grid.y), sums);
    return cudaGetLastError();
}

// ------------------------------------------------------------- opacity reg
// losses.py:157-168,220-223: sum sigma and lambda_o sigma (1 - sigma) / n.
__global__ void opacity_reg_kernel(int64_t n, const float* __restrict__ logits, float lo_over_n,
                                   float* __restrict__ grad, int accumulate,
                                   double* __restrict__ partials) {
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        float l = logits[i];
        float e = expf(-fabsf(l));
        float sg = l >= 0.f ? 1.f / (1.f + e) : e / (1.f + e);
        acc += (double)sg;
        float g = lo_over_n * sg * (1.f - sg);
        if (grad) grad[i] = accumulate ? grad[i] + g : g;
    }
    acc = warp_sum(acc);
    __shared__ double red[32];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) a += red[k];
        partials[2 * blockIdx.x] = a;
        partials[2 * blockIdx.x + 1] = 0.0;
    }
}

cudaError_t launch_opacity_reg(int64_t n, const float* logits, float lambda_o, float* grad,
                               int accumulate, double* sum, double* partials, cudaStream_t s) {
    const int nb = 592;
    float lon = n > 0 ? (float)((double)lambda_o / (double)n) : 0.f;
    opacity_reg_kernel<<<nb, 256, 0, s>>>(n, logits, lon, grad, accumulate, partials);
    reduce_pairs_kernel<<<1, 256, 0, s>>>(nb, partials, sum);
    return cudaGetLastError();
}

// --------------------------------------------------------------- depth L1
__global__ void depth_l1_kernel(size_t n, const float* __restrict__ d,
                                const float* __restrict__ tgt, float* __restrict__ sgn,
                                double* __restrict__ partials) {
    double acc = 0.0, cnt = 0.0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        float tv = tgt[i];
        bool valid = tv > 0.f;
        float e = d[i] - tv;
        if (valid) {
            acc += fabs((double)e);
            cnt += 1.0;
        }
        sgn[i] = valid ? (e > 0.f ? 1.f : (e < 0.f ? -1.f : 0.f)) : 0.f;
    }
    acc = warp_sum(acc);
    cnt = warp_sum(cnt);
    __shared__ double ra[32], rb[32];
    if ((threadIdx.x & 31) == 0) {
        ra[threadIdx.x >> 5] = acc;
        rb[threadIdx.x >> 5] = cnt;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
            a += ra[k];
            b += rb[k];
        }
        partials[2 * blockIdx.x] = a;
        partials[2 * blockIdx.x + 1] = b;
    }
}

__global__ void depth_scale_kernel(size_t n, float* __restrict__ g, const double* sums,
                                   float weight) {
    float inv = (float)(weight / fmax(sums[1], 1.0));
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x)
        g[i] *= inv;
}

cudaError_t launch_depth_l1(int H, int W, const float* d, const float* tgt, float weight,
                            float* grad, double* sums, double* partials, cudaStream_t s) {
    size_t n = (size_t)H * W;
    const int nb = 592;
    depth_l1_kernel<<<nb, 256, 0, s>>>(n, d, tgt, grad, partials);
    reduce_pairs_kernel<<<1, 256, 0, s>>>(nb, partials, sums);
    depth_scale_kernel<<<nb, 256, 0, s>>>(n, grad, sums, weight);
    return cudaGetLastError();
}

}  // namespace ss

#ifdef SS_FWD_TRACE
extern "C" int ss_debug_ssim_trace(int kind, void* host, size_t bytes) {
    if (bytes > sizeof(ss::g_ssim_trace[0])) bytes = sizeof(ss::g_ssim_trace[0]);
    return (int)cudaMemcpyFromSymbol(host, ss::g_ssim_trace, bytes,
                                     (size_t)kind * sizeof(ss::g_ssim_trace[0]));
}
#endif
