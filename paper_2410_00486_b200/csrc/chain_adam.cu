// chain_adam.cu -- K8 chain backward, K9 Adam, and their single-view fusion.
//
// K8 restates chain_backward (rasterizer/projection.py:200-299, _quat_grad
// :302-325) one thread per Gaussian: the projection context is recomputed
// from the parameters (cheaper than storing the reference's per-splat
// rot / cov_cam / viewdir arrays), then screen-space rows
// [rgb(3), mean2d(2), conic(3), opacity(, z)] are chained to position,
// rotation, log-scale, opacity logit and SH.  Folded in: the opacity
// regulariser's gradient for every Gaussian (losses.py:220-223 added at
// trainer.py:206), accumulate_grad_stats (densify.py:86-100) and the
// finite-gradient check (api.py:74-79) as a device error word.
// K9 restates adam_step (optimizer.py:101-133): bias-corrected moments,
// per-element step clipped to +-lr, position lr decayed on the host,
// quaternion renormalisation (core.py:225-229) in the same pass.
// ss_chain_adam fuses both for a single-view iteration so the per-Gaussian
// gradients never touch HBM.
#include "common.cuh"
#include "sh.cuh"

namespace ss {

struct CamC {
    float fx, fy, cx, cy;
    int W, H;
    float R[9], t[3], c[3];
};

void fill_camc(const ss_camera* c, CamC& f) {
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

__device__ __forceinline__ void load_camc(const ss_camera* __restrict__ c, CamC& f) {
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

struct GaussGrad {
    float pos[3], rot[4], ls[3], op, dc[3];
    float n2d;
};

__device__ __forceinline__ void prefetch_l1(const void* p) {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

__device__ __forceinline__ float rsqrt_approx(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float sqrt_approx(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// The chain and Adam math runs on MUFU reciprocals / square roots (relative
// error ~1e-7, far inside the 1e-3 parity tolerance on gradients and
// post-Adam parameters): the IEEE divide/sqrt sequences dominated the
// fused kernel's instruction count.
__device__ __forceinline__ float sigm(float x) {
    float e = expf(-fabsf(x));
    float r = rcp_approx(1.f + e);
    return x >= 0.f ? r : e * r;
}

// Chain one visible Gaussian.  g: screen-space row (9 or 10 values).
// rest_grad (45 floats, may be null) receives the SH bands 1..15.
template <int NC>
__device__ __forceinline__ void chain_one(const float p[3], float4 q4, const float l[3], float opl,
                                          const float dc[3], const float* __restrict__ rest,
                                          const CamC& cam, int deg, float dilation,
                                          const float* g, uint8_t flags, GaussGrad& o,
                                          float* rest_grad, float* basis_out = nullptr) {
    // ---- projection context (projection.py:86-121)
    float t[3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
        t[i] = p[0] * cam.R[3 * i] + p[1] * cam.R[3 * i + 1] + p[2] * cam.R[3 * i + 2] + cam.t[i];
    const float rqn = rsqrt_approx(q4.x * q4.x + q4.y * q4.y + q4.z * q4.z + q4.w * q4.w);
    float qh[4] = {q4.x * rqn, q4.y * rqn, q4.z * rqn, q4.w * rqn};
    float R[9];
    quat_to_rot(qh, R);
    float s2[3] = {expf(2.f * l[0]), expf(2.f * l[1]), expf(2.f * l[2])};
    float M[9];  // Rcw * R
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            M[3 * i + j] = cam.R[3 * i] * R[j] + cam.R[3 * i + 1] * R[3 + j] + cam.R[3 * i + 2] * R[6 + j];
    float covc[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k)
            covc[3 * i + k] = M[3 * i] * s2[0] * M[3 * k] + M[3 * i + 1] * s2[1] * M[3 * k + 1] +
                              M[3 * i + 2] * s2[2] * M[3 * k + 2];
    const float fx = cam.fx, fy = cam.fy;
    float iz = rcp_approx(t[2]), iz2 = iz * iz;
    float J[6] = {fx * iz, 0.f, -fx * t[0] * iz2, 0.f, fy * iz, -fy * t[1] * iz2};
    float JC[6];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k)
            JC[3 * i + k] = J[3 * i] * covc[k] + J[3 * i + 1] * covc[3 + k] + J[3 * i + 2] * covc[6 + k];
    float a = JC[0] * J[0] + JC[1] * J[1] + JC[2] * J[2] + dilation;
    float b = JC[0] * J[3] + JC[1] * J[4] + JC[2] * J[5];
    float c = JC[3] * J[3] + JC[4] * J[4] + JC[5] * J[5] + dilation;
    float det = a * c - b * b;
    const float idet = rcp_approx(det);
    float Q00 = c * idet, Q01 = -b * idet, Q11 = a * idet;

    // ---- opacity (projection.py:217-218)
    float sg = sigm(opl);
    o.op = g[8] * sg * (1.f - sg);
    // ---- conic -> cov2d: GC = -Q GQ Q (projection.py:220-229)
    float G00 = g[5], G01 = g[6] * 0.5f, G11 = g[7];
    float QG00 = Q00 * G00 + Q01 * G01, QG01 = Q00 * G01 + Q01 * G11;
    float QG10 = Q01 * G00 + Q11 * G01, QG11 = Q01 * G01 + Q11 * G11;
    float GC00 = -(QG00 * Q00 + QG01 * Q01), GC01 = -(QG00 * Q01 + QG01 * Q11);
    float GC10 = -(QG10 * Q00 + QG11 * Q01), GC11 = -(QG10 * Q01 + QG11 * Q11);
    // ---- dSc = J^T GC J ; dJ = 2 GC J covc (projection.py:231-241)
    float GJ[6];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        GJ[k] = GC00 * J[k] + GC01 * J[3 + k];
        GJ[3 + k] = GC10 * J[k] + GC11 * J[3 + k];
    }
    float dSc[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k) dSc[3 * i + k] = J[i] * GJ[k] + J[3 + i] * GJ[3 + k];
    float dJ[6];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k)
            dJ[3 * i + k] = 2.f * (GJ[3 * i] * covc[k] + GJ[3 * i + 1] * covc[3 + k] +
                                   GJ[3 * i + 2] * covc[6 + k]);
    // ---- dS3 = Rcw^T dSc Rcw (projection.py:244)
    float t1[9], dS3[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k)
            t1[3 * i + k] = cam.R[i] * dSc[k] + cam.R[3 + i] * dSc[3 + k] + cam.R[6 + i] * dSc[6 + k];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k)
            dS3[3 * i + k] = t1[3 * i] * cam.R[k] + t1[3 * i + 1] * cam.R[3 + k] + t1[3 * i + 2] * cam.R[6 + k];
    // ---- log-scale: 2 s2 diag(R^T dS3 R) (projection.py:245-247)
#pragma unroll
    for (int aa = 0; aa < 3; ++aa) {
        float acc = 0.f;
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int k = 0; k < 3; ++k) acc += R[3 * j + aa] * dS3[3 * j + k] * R[3 * k + aa];
        o.ls[aa] = 2.f * s2[aa] * acc;
    }
    // ---- rotation (projection.py:248-251, _quat_grad :302-325)
    float dR[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k)
            dR[3 * i + k] = 2.f * (dS3[3 * i] * R[k] * s2[k] + dS3[3 * i + 1] * R[3 + k] * s2[k] +
                                   dS3[3 * i + 2] * R[6 + k] * s2[k]);
    float w = qh[0], x = qh[1], y = qh[2], z = qh[3];
    float gq[4];
    gq[0] = 2.f * (-dR[1] * z + dR[2] * y + dR[3] * z - dR[5] * x - dR[6] * y + dR[7] * x);
    gq[1] = 2.f * (dR[1] * y + dR[2] * z + dR[3] * y - 2.f * dR[4] * x - dR[5] * w + dR[6] * z +
                   dR[7] * w - 2.f * dR[8] * x);
    gq[2] = 2.f * (-2.f * dR[0] * y + dR[1] * x + dR[2] * w + dR[3] * x + dR[5] * z - dR[6] * w +
                   dR[7] * z - 2.f * dR[8] * y);
    gq[3] = 2.f * (-2.f * dR[0] * z - dR[1] * w + dR[2] * x + dR[3] * w - 2.f * dR[4] * z +
                   dR[5] * y + dR[6] * x + dR[7] * y);
    float dot = qh[0] * gq[0] + qh[1] * gq[1] + qh[2] * gq[2] + qh[3] * gq[3];
#pragma unroll
    for (int k = 0; k < 4; ++k) o.rot[k] = (gq[k] - qh[k] * dot) * rqn;
    // ---- position through mean2d and J (projection.py:253-265)
    float gm0 = g[3], gm1 = g[4];
    float gt0 = (fx * iz) * gm0 - dJ[2] * fx * iz2;
    float gt1 = (fy * iz) * gm1 - dJ[5] * fy * iz2;
    float gt2 = -fx * t[0] * iz2 * gm0 - fy * t[1] * iz2 * gm1 - dJ[0] * fx * iz2 -
                dJ[4] * fy * iz2 + dJ[2] * 2.f * fx * t[0] * iz2 * iz +
                dJ[5] * 2.f * fy * t[1] * iz2 * iz;
    if (NC == 10) gt2 += g[9];  // depth extension: z = t_cam.z
#pragma unroll
    for (int k = 0; k < 3; ++k) o.pos[k] = gt0 * cam.R[k] + gt1 * cam.R[3 + k] + gt2 * cam.R[6 + k];
    // ---- colour (projection.py:267-277)
    float u[3] = {p[0] - cam.c[0], p[1] - cam.c[1], p[2] - cam.c[2]};
    // 1 / max(|u|, 1e-12)
    const float ivl = rsqrt_approx(fmaxf(u[0] * u[0] + u[1] * u[1] + u[2] * u[2], 1e-24f));
    float d[3] = {u[0] * ivl, u[1] * ivl, u[2] * ivl};
    float grgb[3] = {(flags & 2) ? g[0] : 0.f, (flags & 4) ? g[1] : 0.f, (flags & 8) ? g[2] : 0.f};
    float bs[16];
    sh_basis16(d, deg, bs);
    if (basis_out) {  // rest gradient factors: g_rest[k][ch] = bs[k] * grgb[ch]
#pragma unroll
        for (int k = 0; k < 16; ++k) basis_out[k] = bs[k];
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) basis_out[16 + ch] = grgb[ch];
    }
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) o.dc[ch] = bs[0] * grgb[ch];
    if (deg > 0) {
        float coef[16];
        coef[0] = dc[0] * grgb[0] + dc[1] * grgb[1] + dc[2] * grgb[2];
        int nb = (deg + 1) * (deg + 1);
#pragma unroll
        for (int k = 1; k < 16; ++k) {
            if (k < nb) {
                const float* r = rest + 3 * (k - 1);
                coef[k] = r[0] * grgb[0] + r[1] * grgb[1] + r[2] * grgb[2];
                if (rest_grad) {
#pragma unroll
                    for (int ch = 0; ch < 3; ++ch) rest_grad[3 * (k - 1) + ch] = bs[k] * grgb[ch];
                }
            } else {
                coef[k] = 0.f;
                if (rest_grad) {
#pragma unroll
                    for (int ch = 0; ch < 3; ++ch) rest_grad[3 * (k - 1) + ch] = 0.f;
                }
            }
        }
        float gdir[3];
        sh_dir_grad(d, deg, coef, gdir);
        float vd = d[0] * gdir[0] + d[1] * gdir[1] + d[2] * gdir[2];
#pragma unroll
        for (int k = 0; k < 3; ++k) o.pos[k] += (gdir[k] - d[k] * vd) * ivl;
    } else if (rest_grad) {
        for (int k = 0; k < 45; ++k) rest_grad[k] = 0.f;
    }
    float n0 = gm0 * (cam.W / 2.f), n1 = gm1 * (cam.H / 2.f);
    o.n2d = sqrtf(n0 * n0 + n1 * n1);
}

__device__ __forceinline__ bool grad_finite(const GaussGrad& o) {
    bool f = finitef(o.op) && finitef(o.n2d);
#pragma unroll
    for (int k = 0; k < 3; ++k) f = f && finitef(o.pos[k]) && finitef(o.ls[k]) && finitef(o.dc[k]);
#pragma unroll
    for (int k = 0; k < 4; ++k) f = f && finitef(o.rot[k]);
    return f;
}

// ---------------------------------------------------------------- chain
template <int NC>
__global__ void __launch_bounds__(256) chain_kernel(
    int64_t n, const float* __restrict__ pos, const float4* __restrict__ rot,
    const float* __restrict__ ls, const float* __restrict__ opl, const float* __restrict__ shdc,
    const float* __restrict__ shrest, CamC cam, int deg, float dilation,
    const float* __restrict__ g2d, const uint8_t* __restrict__ flags,
    const uint8_t* __restrict__ contributed, float lo_over_n, int mode, ss_param_grads G,
    float* __restrict__ grad2d_accum, float* __restrict__ grad3d_accum,
    int32_t* __restrict__ obs_count, ss_status* st) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    GaussGrad o = {};
    uint8_t fl = flags[i];
    float rtmp[45];
    float* rgo = (deg > 0 && G.d_sh_rest) ? G.d_sh_rest + 45 * i : nullptr;
    float* rg = (rgo && (mode & SS_CHAIN_ACCUMULATE)) ? rtmp : rgo;
    if (fl & 1) {
        float p[3] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
        float l[3] = {ls[3 * i], ls[3 * i + 1], ls[3 * i + 2]};
        float dc[3] = {shdc[3 * i], shdc[3 * i + 1], shdc[3 * i + 2]};
        float g[NC];
#pragma unroll
        for (int k = 0; k < NC; ++k) g[k] = g2d[NC * i + k];
        chain_one<NC>(p, rot[i], l, opl[i], dc, shrest + 45 * i, cam, deg, dilation, g, fl, o, rg);
        if (rg == rtmp)
            for (int k = 0; k < 45; ++k) rgo[k] += rtmp[k];
    } else if (rg && rg != rtmp) {
        for (int k = 0; k < 45; ++k) rg[k] = 0.f;
    }
    if (lo_over_n != 0.f) {
        float sg = sigm(opl[i]);
        o.op += lo_over_n * sg * (1.f - sg);
    }
    if (!grad_finite(o)) report_first(&st->first_nonfinite_grad, i);
    const bool accum = (mode & SS_CHAIN_ACCUMULATE) != 0;
    const bool seen = contributed && contributed[i];
    if (accum) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            G.d_position[3 * i + k] += o.pos[k];
            G.d_log_scale[3 * i + k] += o.ls[k];
            G.d_sh_dc[3 * i + k] += o.dc[k];
        }
        float4 r = reinterpret_cast<float4*>(G.d_rotation)[i];
        r.x += o.rot[0];
        r.y += o.rot[1];
        r.z += o.rot[2];
        r.w += o.rot[3];
        reinterpret_cast<float4*>(G.d_rotation)[i] = r;
        G.d_opacity[i] += o.op;
        if (G.d_pos2d_norm) G.d_pos2d_norm[i] += o.n2d;
    } else {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            G.d_position[3 * i + k] = o.pos[k];
            G.d_log_scale[3 * i + k] = o.ls[k];
            G.d_sh_dc[3 * i + k] = o.dc[k];
        }
        reinterpret_cast<float4*>(G.d_rotation)[i] =
            make_float4(o.rot[0], o.rot[1], o.rot[2], o.rot[3]);
        G.d_opacity[i] = o.op;
        if (G.d_pos2d_norm) G.d_pos2d_norm[i] = o.n2d;
    }
    if ((mode & SS_CHAIN_STAT_PLANES) && seen && G.d_stat_cnt) {
        G.d_stat_g2d[i] += o.n2d;
        G.d_stat_g3d[3 * i] += o.pos[0];
        G.d_stat_g3d[3 * i + 1] += o.pos[1];
        G.d_stat_g3d[3 * i + 2] += o.pos[2];
        G.d_stat_cnt[i] += 1.0f;
    }
    if ((mode & SS_CHAIN_STATS) && seen) {
        grad2d_accum[i] += o.n2d;
        grad3d_accum[3 * i] += o.pos[0];
        grad3d_accum[3 * i + 1] += o.pos[1];
        grad3d_accum[3 * i + 2] += o.pos[2];
        obs_count[i] += 1;
    }
}

__global__ void apply_stat_planes_kernel(int64_t n, ss_param_grads G, float* grad2d_accum,
                                         float* grad3d_accum, int32_t* obs_count) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    float c = G.d_stat_cnt[i];
    if (c == 0.f) return;
    grad2d_accum[i] += G.d_stat_g2d[i];
    grad3d_accum[3 * i] += G.d_stat_g3d[3 * i];
    grad3d_accum[3 * i + 1] += G.d_stat_g3d[3 * i + 1];
    grad3d_accum[3 * i + 2] += G.d_stat_g3d[3 * i + 2];
    obs_count[i] += (int32_t)lrintf(c);
}

// ----------------------------------------------------------------- adam
struct AdamHP {
    float lr[6];  // position, rotation, log_scale, opacity, sh_dc, sh_rest
    float b1, b2, eps, bc1, bc2;
    float ibc1, ibc2;  // 1 / bias corrections
};

__device__ __forceinline__ void load_hp(const ss_adam_hparams* __restrict__ h, AdamHP& hp) {
    hp.lr[0] = h->lr_position;
    hp.lr[1] = h->lr_rotation;
    hp.lr[2] = h->lr_log_scale;
    hp.lr[3] = h->lr_opacity;
    hp.lr[4] = h->lr_sh_dc;
    hp.lr[5] = h->lr_sh_rest;
    hp.b1 = h->beta1;
    hp.b2 = h->beta2;
    hp.eps = h->eps;
    hp.bc1 = h->bias1;
    hp.bc2 = h->bias2;
    hp.ibc1 = 1.f / hp.bc1;
    hp.ibc2 = 1.f / hp.bc2;
}

__device__ __forceinline__ float adam_elem(float& p, float g, float& m, float& v, float lr,
                                           const AdamHP& hp) {
    m = m * hp.b1 + (1.f - hp.b1) * g;
    v = v * hp.b2 + (1.f - hp.b2) * g * g;
    float step = lr * (m * hp.ibc1) * rcp_approx(sqrt_approx(v * hp.ibc2) + hp.eps);
    step = fminf(fmaxf(step, -lr), lr);
    p -= step;
    return step;
}

// Adam over one Gaussian given its gradients (o) and plane pointers.
__device__ __forceinline__ void adam_gaussian(int64_t i, const GaussGrad& o, const float* rest_g,
                                              float* pos, float4* rot, float* ls, float* opl,
                                              float* shdc, float* shrest, const ss_param_grads& M,
                                              const ss_param_grads& V, const AdamHP& hp,
                                              bool upd_rest, ss_status* st) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        adam_elem(pos[3 * i + k], o.pos[k], M.d_position[3 * i + k], V.d_position[3 * i + k],
                  hp.lr[0], hp);
        adam_elem(ls[3 * i + k], o.ls[k], M.d_log_scale[3 * i + k], V.d_log_scale[3 * i + k],
                  hp.lr[2], hp);
        adam_elem(shdc[3 * i + k], o.dc[k], M.d_sh_dc[3 * i + k], V.d_sh_dc[3 * i + k], hp.lr[4],
                  hp);
    }
    adam_elem(opl[i], o.op, M.d_opacity[i], V.d_opacity[i], hp.lr[3], hp);
    float4 q = rot[i];
    float4 mq = reinterpret_cast<float4*>(M.d_rotation)[i];
    float4 vq = reinterpret_cast<float4*>(V.d_rotation)[i];
    adam_elem(q.x, o.rot[0], mq.x, vq.x, hp.lr[1], hp);
    adam_elem(q.y, o.rot[1], mq.y, vq.y, hp.lr[1], hp);
    adam_elem(q.z, o.rot[2], mq.z, vq.z, hp.lr[1], hp);
    adam_elem(q.w, o.rot[3], mq.w, vq.w, hp.lr[1], hp);
    // normalize_rotations (core.py:225-229)
    const float nn2 = q.x * q.x + q.y * q.y + q.z * q.z + q.w * q.w;
    if (nn2 == 0.f) report_first(&st->first_zero_quat, i);
    const float rn = rsqrt_approx(nn2);
    q.x *= rn;
    q.y *= rn;
    q.z *= rn;
    q.w *= rn;
    rot[i] = q;
    reinterpret_cast<float4*>(M.d_rotation)[i] = mq;
    reinterpret_cast<float4*>(V.d_rotation)[i] = vq;
    if (upd_rest) {
        for (int k = 0; k < 45; ++k)
            adam_elem(shrest[45 * i + k], rest_g ? rest_g[k] : 0.f, M.d_sh_rest[45 * i + k],
                      V.d_sh_rest[45 * i + k], hp.lr[5], hp);
    }
}

__global__ void __launch_bounds__(256) adam_kernel(int64_t n, float* pos, float4* rot, float* ls,
                                                   float* opl, float* shdc, float* shrest,
                                                   ss_param_grads Gr, ss_param_grads M,
                                                   ss_param_grads V, AdamHP hp, int upd_rest,
                                                   ss_status* st) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    GaussGrad o;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        o.pos[k] = Gr.d_position[3 * i + k];
        o.ls[k] = Gr.d_log_scale[3 * i + k];
        o.dc[k] = Gr.d_sh_dc[3 * i + k];
    }
    float4 gq = reinterpret_cast<const float4*>(Gr.d_rotation)[i];
    o.rot[0] = gq.x;
    o.rot[1] = gq.y;
    o.rot[2] = gq.z;
    o.rot[3] = gq.w;
    o.op = Gr.d_opacity[i];
    o.n2d = 0.f;
    bool fin = grad_finite(o);
    const float* rg = (upd_rest && Gr.d_sh_rest) ? Gr.d_sh_rest + 45 * i : nullptr;
    if (rg)
        for (int k = 0; k < 45; ++k) fin &= finitef(rg[k]);  // loads in flight together
    if (!fin) {  // optimizer.py:111-113 raises before touching the map: leave this one as is
        report_first(&st->first_nonfinite_grad, i);
        return;
    }
    adam_gaussian(i, o, rg, pos, rot, ls, opl, shdc, shrest, M, V, hp, upd_rest != 0, st);
}

// ----------------------------------------------------------- chain+adam
template <int NC, bool REST>
__global__ void __launch_bounds__(256, REST ? 2 : 4) chain_adam_kernel(
    int64_t n, float* __restrict__ pos, float4* __restrict__ rot, float* __restrict__ ls,
    float* __restrict__ opl, float* __restrict__ shdc, float* __restrict__ shrest, CamC cam_v,
    const ss_camera* __restrict__ d_cam, int deg, float dilation, const float* __restrict__ g2d,
    const uint8_t* __restrict__ flags, const uint8_t* __restrict__ contributed, float lo_over_n,
    ss_param_grads M, ss_param_grads V, AdamHP hp_v, const ss_adam_hparams* __restrict__ d_hp,
    float* __restrict__ grad2d_accum, float* __restrict__ grad3d_accum,
    int32_t* __restrict__ obs_count, ss_status* st) {
    PDL_WAIT();
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    // every independent load first (the parameters are needed by Adam
    // whether or not the Gaussian is visible; a culled Gaussian's g2d row is
    // zero), then the overflow word and the flag test
    const uint8_t fl = flags[i];
    const float opi = opl[i];
    float p[3] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
    const float4 q4 = rot[i];
    float l[3] = {ls[3 * i], ls[3 * i + 1], ls[3 * i + 2]};
    float dc[3] = {shdc[3 * i], shdc[3 * i + 1], shdc[3 * i + 2]};
    float g[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) g[k] = g2d[NC * i + k];
    // the Adam moments this thread updates after the chain: their lines are
    // requested now (no registers held), so those loads hit L1
    prefetch_l1(M.d_position + 3 * i);
    prefetch_l1(V.d_position + 3 * i);
    prefetch_l1(M.d_log_scale + 3 * i);
    prefetch_l1(V.d_log_scale + 3 * i);
    prefetch_l1(M.d_sh_dc + 3 * i);
    prefetch_l1(V.d_sh_dc + 3 * i);
    prefetch_l1(M.d_rotation + 4 * i);
    prefetch_l1(V.d_rotation + 4 * i);
    prefetch_l1(M.d_opacity + i);
    prefetch_l1(V.d_opacity + i);
    if (contributed) {
        prefetch_l1(contributed + i);
        prefetch_l1(grad2d_accum + i);
        prefetch_l1(grad3d_accum + 3 * i);
        prefetch_l1(obs_count + i);
    }
    CamC cam = cam_v;
    AdamHP hp = hp_v;
    if (d_cam) load_camc(d_cam, cam);  // graph replay: per-step values from device memory
    if (d_hp) load_hp(d_hp, hp);
    if (st->pair_overflow) return;
    GaussGrad o = {};
    float rest_g[REST ? 45 : 1];
    if (fl & 1) {
        chain_one<NC>(p, q4, l, opi, dc, shrest + 45 * i, cam, deg, dilation, g, fl, o,
                      REST ? rest_g : nullptr);
    } else if (REST) {
#pragma unroll
        for (int k = 0; k < (REST ? 45 : 1); ++k) rest_g[k] = 0.f;
    }
    if (lo_over_n != 0.f) {
        float sg = sigm(opi);
        o.op += lo_over_n * sg * (1.f - sg);
    }
    if (!grad_finite(o)) {
        // the reference raises before any update (api.py:74-79, optimizer.py:111-113): this
        // Gaussian's parameters, moments and statistics stay as they were
        report_first(&st->first_nonfinite_grad, i);
        return;
    }
    if (contributed && contributed[i]) {
        grad2d_accum[i] += o.n2d;
        grad3d_accum[3 * i] += o.pos[0];
        grad3d_accum[3 * i + 1] += o.pos[1];
        grad3d_accum[3 * i + 2] += o.pos[2];
        obs_count[i] += 1;
    }
    adam_gaussian(i, o, REST ? rest_g : nullptr, pos, rot, ls, opl, shdc, shrest, M, V, hp, REST,
                  st);
}

// ------------------------------------------------ chain+adam, SH rest on
// sh_rest is (N, 45) per Gaussian: a thread walking its own row strides
// 180 B between lanes.  Here the CTA's 256 rows (one contiguous span) are
// staged through shared memory for the chain's direction gradient, each
// thread exports its 16 basis values and 3 colour gradients, and the CTA
// then runs Adam over the span's 256 x 45 parameters and moments with
// consecutive threads on consecutive elements.
constexpr int kRestCTA = 256;
constexpr int kRestRow = 45;

template <int NC>
__global__ void __launch_bounds__(kRestCTA, 3) chain_adam_rest_kernel(
    int64_t n, float* __restrict__ pos, float4* __restrict__ rot, float* __restrict__ ls,
    float* __restrict__ opl, float* __restrict__ shdc, float* __restrict__ shrest, CamC cam_v,
    const ss_camera* __restrict__ d_cam, int deg, float dilation, const float* __restrict__ g2d,
    const uint8_t* __restrict__ flags, const uint8_t* __restrict__ contributed, float lo_over_n,
    ss_param_grads M, ss_param_grads V, AdamHP hp_v, const ss_adam_hparams* __restrict__ d_hp,
    float* __restrict__ grad2d_accum, float* __restrict__ grad3d_accum,
    int32_t* __restrict__ obs_count, ss_status* st) {
    extern __shared__ float rs_smem[];
    __shared__ uint8_t s_ok[kRestCTA];               // gradient finite: update this row
    float* s_rest = rs_smem;                         // [kRestCTA * 45] parameters
    float* s_fac = rs_smem + kRestCTA * kRestRow;    // [kRestCTA * 19] basis, colour grad
    if (st->pair_overflow) return;  // uniform: the step is replayed
    const int t = threadIdx.x;
    const int64_t base = (int64_t)blockIdx.x * kRestCTA;
    const int cnt = (int)min((int64_t)kRestCTA, n - base);
    const int span = cnt * kRestRow;
    const float* rest_g = shrest + base * kRestRow;
    for (int e = t; e < span; e += kRestCTA) s_rest[e] = rest_g[e];
    __syncthreads();
    if (t < cnt) {
        const int64_t i = base + t;
        CamC cam = cam_v;
        AdamHP hp = hp_v;
        if (d_cam) load_camc(d_cam, cam);
        if (d_hp) load_hp(d_hp, hp);
        GaussGrad o = {};
        const uint8_t fl = flags[i];
        const float opi = opl[i];
        float* fac = s_fac + 19 * t;
        if (fl & 1) {
            float p[3] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
            float l[3] = {ls[3 * i], ls[3 * i + 1], ls[3 * i + 2]};
            float dc[3] = {shdc[3 * i], shdc[3 * i + 1], shdc[3 * i + 2]};
            float g[NC];
#pragma unroll
            for (int k = 0; k < NC; ++k) g[k] = g2d[NC * i + k];
            chain_one<NC>(p, rot[i], l, opi, dc, s_rest + kRestRow * t, cam, deg, dilation, g,
                          fl, o, nullptr, fac);
        } else {
#pragma unroll
            for (int k = 0; k < 19; ++k) fac[k] = 0.f;
        }
        if (lo_over_n != 0.f) {
            float sg = sigm(opi);
            o.op += lo_over_n * sg * (1.f - sg);
        }
        const bool fin = grad_finite(o);
        s_ok[t] = fin;
        if (!fin) {
            report_first(&st->first_nonfinite_grad, i);  // row left unchanged (see above)
        } else {
            if (contributed && contributed[i]) {
                grad2d_accum[i] += o.n2d;
                grad3d_accum[3 * i] += o.pos[0];
                grad3d_accum[3 * i + 1] += o.pos[1];
                grad3d_accum[3 * i + 2] += o.pos[2];
                obs_count[i] += 1;
            }
            adam_gaussian(i, o, nullptr, pos, rot, ls, opl, shdc, shrest, M, V, hp, false, st);
        }
    }
    __syncthreads();
    // Adam over the CTA's contiguous sh_rest span (bands >= deg + 1 get g = 0)
    AdamHP hp = hp_v;
    if (d_hp) load_hp(d_hp, hp);
    const int nb = (deg + 1) * (deg + 1);
    float* __restrict__ pm = M.d_sh_rest + base * kRestRow;
    float* __restrict__ pv = V.d_sh_rest + base * kRestRow;
    float* __restrict__ pp = shrest + base * kRestRow;
    // 9 elements per thread and round, all 18 moment loads in flight before
    // the updates (the span is 45 rows of kRestCTA: latency, not bandwidth,
    // bounded this loop with one element per round)
    constexpr int U = 9;
#pragma unroll 1
    for (int e0 = t; e0 < span; e0 += kRestCTA * U) {
        float m[U], v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int e = e0 + u * kRestCTA;
            m[u] = e < span ? pm[e] : 0.f;
            v[u] = e < span ? pv[e] : 0.f;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int e = e0 + u * kRestCTA;
            const int gi = e / kRestRow;
            if (e < span && s_ok[gi]) {
                const int j = e - gi * kRestRow;
                const int k = j / 3 + 1, ch = j - 3 * (k - 1);
                const float* fac = s_fac + 19 * gi;
                const float gr = k < nb ? fac[k] * fac[16 + ch] : 0.f;
                float p = s_rest[e];
                adam_elem(p, gr, m[u], v[u], hp.lr[5], hp);
                pp[e] = p;
                pm[e] = m[u];
                pv[e] = v[u];
            }
        }
    }
}

// ---------------------------------------------------------------- stats
__global__ void stats_kernel(int64_t n, const float* __restrict__ gpos,
                             const float* __restrict__ n2d, const uint8_t* __restrict__ contributed,
                             float* grad2d_accum, float* grad3d_accum, int32_t* obs_count) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n || !contributed[i]) return;
    grad2d_accum[i] += n2d[i];
    grad3d_accum[3 * i] += gpos[3 * i];
    grad3d_accum[3 * i + 1] += gpos[3 * i + 1];
    grad3d_accum[3 * i + 2] += gpos[3 * i + 2];
    obs_count[i] += 1;
}

// -------------------------------------------------------- opacity reset
__global__ void opacity_reset_kernel(int64_t n, float* opl, float ceiling, float* m, float* v) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double l = opl[i];
    double e = exp(-fabs(l));
    double sg = l >= 0 ? 1.0 / (1.0 + e) : e / (1.0 + e);
    double s = fmin(sg, (double)ceiling);
    opl[i] = (float)(log(s) - log1p(-s));
    if (m) m[i] = 0.f;
    if (v) v[i] = 0.f;
}

// ------------------------------------------------------------ launchers
static AdamHP make_hp(const ss_adam_hparams* h) {
    AdamHP hp;
    hp.lr[0] = h->lr_position;
    hp.lr[1] = h->lr_rotation;
    hp.lr[2] = h->lr_log_scale;
    hp.lr[3] = h->lr_opacity;
    hp.lr[4] = h->lr_sh_dc;
    hp.lr[5] = h->lr_sh_rest;
    hp.b1 = h->beta1;
    hp.b2 = h->beta2;
    hp.eps = h->eps;
    hp.bc1 = h->bias1;
    hp.bc2 = h->bias2;
    hp.ibc1 = 1.f / hp.bc1;
    hp.ibc2 = 1.f / hp.bc2;
    return hp;
}

cudaError_t launch_chain(const ss_map* mp, const ss_camera* cam, const ss_raster_opts* o,
                         const float* g2d, const uint8_t* flags, const uint8_t* contributed,
                         float lo_over_n, int acc_stats, const ss_param_grads* G, ss_status* st,
                         cudaStream_t s) {
    if (mp->n == 0) return cudaSuccess;
    CamC cc;
    fill_camc(cam, cc);
    int blocks = div_up(mp->n, 256);
    auto go = [&](auto kern) {
        kern<<<blocks, 256, 0, s>>>(mp->n, mp->d_positions,
                                    reinterpret_cast<const float4*>(mp->d_rotations),
                                    mp->d_log_scales, mp->d_opacity_logits, mp->d_sh_dc,
                                    mp->d_sh_rest, cc, o->sh_degree, o->dilation, g2d, flags,
                                    contributed, lo_over_n, acc_stats, *G, mp->d_grad2d_accum,
                                    mp->d_grad3d_accum, mp->d_obs_count, st);
    };
    if (o->with_depth)
        go(chain_kernel<10>);
    else
        go(chain_kernel<9>);
    return cudaGetLastError();
}

cudaError_t launch_apply_stat_planes(const ss_map* mp, const ss_param_grads* G, cudaStream_t s) {
    if (mp->n == 0) return cudaSuccess;
    apply_stat_planes_kernel<<<div_up(mp->n, 256), 256, 0, s>>>(mp->n, *G, mp->d_grad2d_accum,
                                                                 mp->d_grad3d_accum,
                                                                 mp->d_obs_count);
    return cudaGetLastError();
}

cudaError_t launch_adam(const ss_map* mp, const ss_param_grads* G, const ss_param_grads* M,
                        const ss_param_grads* V, const ss_adam_hparams* h, ss_status* st,
                        cudaStream_t s) {
    if (mp->n == 0) return cudaSuccess;
    adam_kernel<<<div_up(mp->n, 256), 256, 0, s>>>(
        mp->n, mp->d_positions, reinterpret_cast<float4*>(mp->d_rotations), mp->d_log_scales,
        mp->d_opacity_logits, mp->d_sh_dc, mp->d_sh_rest, *G, *M, *V, make_hp(h),
        h->update_sh_rest, st);
    return cudaGetLastError();
}

cudaError_t launch_chain_adam(const ss_map* mp, const ss_camera* cam, const ss_camera* d_cam,
                              const ss_raster_opts* o, const float* g2d, const uint8_t* flags,
                              const uint8_t* contributed, float lo_over_n,
                              const ss_param_grads* M, const ss_param_grads* V,
                              const ss_adam_hparams* h, const ss_adam_hparams* d_hp,
                              ss_status* st, cudaStream_t s) {
    if (mp->n == 0) return cudaSuccess;
    CamC cc;
    fill_camc(cam, cc);
    auto go = [&](auto kern) {
        launch_pdl(kern, dim3(div_up(mp->n, 256)), dim3(256), 0, s,
            mp->n, mp->d_positions, reinterpret_cast<float4*>(mp->d_rotations), mp->d_log_scales,
            mp->d_opacity_logits, mp->d_sh_dc, mp->d_sh_rest, cc, d_cam, o->sh_degree, o->dilation,
            g2d, flags, contributed, lo_over_n, *M, *V, make_hp(h), d_hp, mp->d_grad2d_accum,
            mp->d_grad3d_accum, mp->d_obs_count, st);
    };
    const bool rest = h->update_sh_rest != 0;
    if (rest) {
        const int smem = (int)(sizeof(float) * kRestCTA * (kRestRow + 19));
        auto gor = [&](auto kern) -> cudaError_t {
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 smem);
            if (e != cudaSuccess) return e;
            kern<<<div_up(mp->n, kRestCTA), kRestCTA, smem, s>>>(
                mp->n, mp->d_positions, reinterpret_cast<float4*>(mp->d_rotations),
                mp->d_log_scales, mp->d_opacity_logits, mp->d_sh_dc, mp->d_sh_rest, cc, d_cam,
                o->sh_degree, o->dilation, g2d, flags, contributed, lo_over_n, *M, *V, make_hp(h),
                d_hp, mp->d_grad2d_accum, mp->d_grad3d_accum, mp->d_obs_count, st);
            return cudaGetLastError();
        };
        return o->with_depth ? gor(chain_adam_rest_kernel<10>) : gor(chain_adam_rest_kernel<9>);
    }
    if (o->with_depth)
        go(chain_adam_kernel<10, false>);
    else
        go(chain_adam_kernel<9, false>);
    return cudaGetLastError();
}

cudaError_t launch_stats(const ss_map* mp, const ss_param_grads* G, const uint8_t* contributed,
                         cudaStream_t s) {
    if (mp->n == 0) return cudaSuccess;
    stats_kernel<<<div_up(mp->n, 256), 256, 0, s>>>(mp->n, G->d_position, G->d_pos2d_norm,
                                                     contributed, mp->d_grad2d_accum,
                                                     mp->d_grad3d_accum, mp->d_obs_count);
    return cudaGetLastError();
}

cudaError_t launch_opacity_reset(const ss_map* mp, float ceiling, float* m, float* v,
                                 cudaStream_t s) {
    if (mp->n == 0) return cudaSuccess;
    opacity_reset_kernel<<<div_up(mp->n, 256), 256, 0, s>>>(mp->n, mp->d_opacity_logits, ceiling,
                                                            m, v);
    return cudaGetLastError();
}

// ---------------------------------------------------------- finite check
// api.py:74-79 / optimizer.py:111-113 for up to 8 float tensors in one
// launch: flags[t] |= 1 when tensor t holds a non-finite value, flags[n + t]
// |= 1 when it holds a non-zero value (adam_step's "sh_rest in use" test).
// The caller zeroes flags (2n int32) first.
struct FiniteSet {
    const float* p[8];
    int64_t n[8];
};

// validate_finite (api.py:74-79) and the non-zero tests over up to 8
// tensors in one launch: 16-byte loads where the tensor is aligned, four in
// flight per thread, and one flag update per CTA and tensor (block OR), so
// the flag words see ~a thousand atomics instead of one per warp.
__global__ void __launch_bounds__(256) check_finite_kernel(int nt, FiniteSet S,
                                                           int32_t* __restrict__ flags) {
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int t = 0; t < nt; ++t) {
        const float* p = S.p[t];
        const int64_t n = S.n[t];
        bool bad = false, nz = false;
        auto test = [&](float v) {
            bad |= !isfinite(v);
            nz |= v != 0.f;
        };
        const int64_t n4 = (reinterpret_cast<uintptr_t>(p) & 15) ? 0 : n / 4;
        const float4* p4 = reinterpret_cast<const float4*>(p);
        int64_t e = tid;
        for (; e + 3 * stride < n4; e += 4 * stride) {
            const float4 a = p4[e], b = p4[e + stride], c = p4[e + 2 * stride],
                         d = p4[e + 3 * stride];
            test(a.x), test(a.y), test(a.z), test(a.w), test(b.x), test(b.y), test(b.z), test(b.w);
            test(c.x), test(c.y), test(c.z), test(c.w), test(d.x), test(d.y), test(d.z), test(d.w);
        }
        for (; e < n4; e += stride) {
            const float4 a = p4[e];
            test(a.x), test(a.y), test(a.z), test(a.w);
        }
        for (int64_t k = 4 * n4 + tid; k < n; k += stride) test(p[k]);
        const bool bb = __syncthreads_or(bad), bn = __syncthreads_or(nz);
        if (threadIdx.x == 0) {
            if (bb) atomicOr(flags + t, 1);
            // the non-zero word is usually set by the first CTAs: skip the atomic then
            if (bn && *reinterpret_cast<volatile int32_t*>(flags + nt + t) == 0)
                atomicOr(flags + nt + t, 1);
        }
    }
}

cudaError_t launch_check_finite(int nt, const float* const* ptrs, const int64_t* counts,
                                int32_t* flags, cudaStream_t s) {
    FiniteSet S = {};
    int64_t mx = 1;
    for (int t = 0; t < nt; ++t) {
        S.p[t] = ptrs[t];
        S.n[t] = counts[t];
        mx = counts[t] > mx ? counts[t] : mx;
    }
    cudaError_t e = cudaMemsetAsync(flags, 0, sizeof(int32_t) * 2 * nt, s);
    if (e != cudaSuccess) return e;
    // enough CTAs for every SM (about 16 floats per thread and round)
    const int64_t want = (mx / 16 + 255) / 256;
    const int blocks = (int)(want < 1 ? 1 : (want < 1184 ? want : 1184));
    check_finite_kernel<<<blocks, 256, 0, s>>>(nt, S, flags);
    return cudaGetLastError();
}

}  // namespace ss
