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
// Two tiled kernels, 32x8 output pixels per CTA, 5-pixel halo in shared
// memory, channels processed in turn:
//   ssim_fwd : moments (x, y, x^2, y^2, xy), SSIM map and the three
//              gradient maps dS/d(mu_x), dS/d(F x^2), dS/d(F xy), per-CTA
//              partial sums of |x - y| and SSIM;
//   ssim_bwd : the folded adjoint of the three maps, combined into
//              (1-l) sign(x-y)/n - l (F*g_mu + 2x F*g_xx + y F*g_xy).
#include "common.cuh"

namespace ss {

constexpr int LTW = 32, LTH = 8, LR = 5;
constexpr int LHW = LTW + 2 * LR, LHH = LTH + 2 * LR;  // 42 x 18

struct SsimWindow {
    float w[11];
};

__device__ __forceinline__ int reflect1(int i, int n) {
    // symmetric reflection without edge repeat (losses.py:31-41), n >= 6
    if (i < 0) i = -i;
    if (i >= n) i = 2 * n - 2 - i;
    return i;
}

__global__ void __launch_bounds__(256) ssim_fwd_kernel(int H, int W, const float* __restrict__ x,
                                                       const float* __restrict__ y,
                                                       SsimWindow win, float* __restrict__ gmu,
                                                       float* __restrict__ gxx,
                                                       float* __restrict__ gxy,
                                                       double* __restrict__ partials) {
    __shared__ float sx[LHH][LHW + 1], sy[LHH][LHW + 1];
    __shared__ float sh[5][LHH][LTW];
    __shared__ double red[2][8];
    const int t = threadIdx.x;
    const int tx = t & 31, ty = t >> 5;
    const int x0 = blockIdx.x * LTW, y0 = blockIdx.y * LTH;
    const int ox = x0 + tx, oy = y0 + ty;
    const bool inside = ox < W && oy < H;
    const float C1 = 0.01f * 0.01f, C2 = 0.03f * 0.03f;
    const float gs = 1.0f / (float)((double)H * W * 3);
    double l1 = 0.0, ssum = 0.0;
    for (int c = 0; c < 3; ++c) {
        for (int k = t; k < LHH * LHW; k += 256) {
            int r = k / LHW, q = k % LHW;
            int gy = reflect1(y0 - LR + r, H), gx = reflect1(x0 - LR + q, W);
            size_t o = ((size_t)gy * W + gx) * 3 + c;
            sx[r][q] = x[o];
            sy[r][q] = y[o];
        }
        __syncthreads();
        for (int k = t; k < LHH * LTW; k += 256) {
            int r = k / LTW, q = k % LTW;
            float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f, a4 = 0.f;
#pragma unroll
            for (int m = 0; m < 11; ++m) {
                float xv = sx[r][q + m], yv = sy[r][q + m], wm = win.w[m];
                a0 += wm * xv;
                a1 += wm * yv;
                a2 += wm * (xv * xv);
                a3 += wm * (yv * yv);
                a4 += wm * (xv * yv);
            }
            sh[0][r][q] = a0;
            sh[1][r][q] = a1;
            sh[2][r][q] = a2;
            sh[3][r][q] = a3;
            sh[4][r][q] = a4;
        }
        __syncthreads();
        if (inside) {
            float mx = 0.f, my = 0.f, fxx = 0.f, fyy = 0.f, fxy = 0.f;
#pragma unroll
            for (int m = 0; m < 11; ++m) {
                float wm = win.w[m];
                mx += wm * sh[0][ty + m][tx];
                my += wm * sh[1][ty + m][tx];
                fxx += wm * sh[2][ty + m][tx];
                fyy += wm * sh[3][ty + m][tx];
                fxy += wm * sh[4][ty + m][tx];
            }
            float sxx = fxx - mx * mx, syy = fyy - my * my, sxy = fxy - mx * my;
            float a1 = 2.f * mx * my + C1, a2 = 2.f * sxy + C2;
            float b1 = mx * mx + my * my + C1, b2 = sxx + syy + C2;
            float bb = b1 * b2;
            float s = a1 * a2 / bb;
            float ga1 = gs * a2 / bb, ga2 = gs * a1 / bb;
            float gb1 = -gs * s / b1, gb2 = -gs * s / b2;
            size_t o = ((size_t)oy * W + ox) * 3 + c;
            gmu[o] = 2.f * my * ga1 + 2.f * mx * gb1 - 2.f * mx * gb2 - my * 2.f * ga2;
            gxx[o] = gb2;
            gxy[o] = 2.f * ga2;
            ssum += (double)s;
            l1 += (double)fabsf(sx[ty + LR][tx + LR] - sy[ty + LR][tx + LR]);
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
        size_t bid = (size_t)blockIdx.y * gridDim.x + blockIdx.x;
        partials[2 * bid] = a;
        partials[2 * bid + 1] = b;
    }
}

// gp(u) over a zero-extended shared row/column: v(k) returns g at local k.
template <typename V>
__device__ __forceinline__ float fold_gather(int i, int n, int org, const SsimWindow& win, V v) {
    // i: global index on this axis; org: global index of local 0
    auto gp = [&](int u) {
        float acc = 0.f;
#pragma unroll
        for (int m = 0; m < 11; ++m) acc += win.w[m] * v(u - LR + m - org);
        return acc;
    };
    float r = gp(i);
    if (i >= 1 && i <= LR) r += gp(-i);
    if (i >= n - 6 && i <= n - 2) r += gp(2 * n - 2 - i);
    return r;
}

__global__ void __launch_bounds__(256) ssim_bwd_kernel(int H, int W, const float* __restrict__ x,
                                                       const float* __restrict__ y,
                                                       SsimWindow win,
                                                       const float* __restrict__ gmu,
                                                       const float* __restrict__ gxx,
                                                       const float* __restrict__ gxy, float lam,
                                                       float* __restrict__ grad,
                                                       float4* __restrict__ pixgrad) {
    __shared__ float sg[3][LHH][LHW + 1];
    __shared__ float sh[3][LHH][LTW];
    const int t = threadIdx.x;
    const int tx = t & 31, ty = t >> 5;
    const int x0 = blockIdx.x * LTW, y0 = blockIdx.y * LTH;
    const int ox = x0 + tx, oy = y0 + ty;
    const float inv_n = 1.0f / (float)((double)H * W * 3);
    float gsave[3] = {0.f, 0.f, 0.f}, gdot = 0.f;
    for (int c = 0; c < 3; ++c) {
        for (int k = t; k < LHH * LHW; k += 256) {
            int r = k / LHW, q = k % LHW;
            int gy = y0 - LR + r, gx = x0 - LR + q;
            bool in = gy >= 0 && gy < H && gx >= 0 && gx < W;
            size_t o = ((size_t)(in ? gy : 0) * W + (in ? gx : 0)) * 3 + c;
            sg[0][r][q] = in ? gmu[o] : 0.f;
            sg[1][r][q] = in ? gxx[o] : 0.f;
            sg[2][r][q] = in ? gxy[o] : 0.f;
        }
        __syncthreads();
        // axis 1 (columns) first, as losses.py:87-88
        for (int k = t; k < LHH * LTW; k += 256) {
            int r = k / LTW, q = k % LTW;
            int j = x0 + q;
            if (j >= W) continue;
#pragma unroll
            for (int f = 0; f < 3; ++f) {
                sh[f][r][q] = fold_gather(j, W, x0 - LR, win, [&](int loc) {
                    return (loc >= 0 && loc < LHW) ? sg[f][r][loc] : 0.f;
                });
            }
        }
        __syncthreads();
        if (ox < W && oy < H) {
            float adj[3];
#pragma unroll
            for (int f = 0; f < 3; ++f) {
                adj[f] = fold_gather(oy, H, y0 - LR, win, [&](int loc) {
                    return (loc >= 0 && loc < LHH) ? sh[f][loc][tx] : 0.f;
                });
            }
            size_t o = ((size_t)oy * W + ox) * 3 + c;
            float xv = x[o], yv = y[o];
            float d = xv - yv;
            float sg0 = d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f);  // np.sign: sign(0) = 0
            float gx = adj[0] + adj[1] * 2.f * xv + adj[2] * yv;
            float gv = (1.0f - lam) * sg0 * inv_n - lam * gx;
            grad[o] = gv;
            gsave[c] = gv;
            gdot += gv * xv;
        }
        __syncthreads();
    }
    if (pixgrad && ox < W && oy < H)
        pixgrad[(size_t)oy * W + ox] = make_float4(gsave[0], gsave[1], gsave[2], gdot);
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
    for (int m = 0; m < 11; ++m) w.w[m] = (float)(v[m] / s);
    return w;
}

size_t loss_workspace_bytes(int H, int W) {
    size_t maps = (size_t)H * W * 3 * sizeof(float) * 3;
    size_t nb = (size_t)div_up(W, LTW) * div_up(H, LTH);
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
    dim3 grid(div_up(W, LTW), div_up(H, LTH));
    ssim_fwd_kernel<<<grid, 256, 0, s>>>(H, W, x, y, win, gmu, gxx, gxy, partials);
    ssim_bwd_kernel<<<grid, 256, 0, s>>>(H, W, x, y, win, gmu, gxx, gxy, lam, grad,
                                         reinterpret_cast<float4*>(pixgrad));
    reduce_pairs_kernel<<<1, 256, 0, s>>>(grid.x * grid.y, partials, sums);
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
