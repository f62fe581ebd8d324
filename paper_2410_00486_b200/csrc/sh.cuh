// sh.cuh -- real spherical harmonics (degree <= 3) and quaternion helpers.
// Constants and basis: sh.py:11-70; direction gradient: sh.py:73-119;
// rotation from a unit quaternion: projection.py:166-178.
#pragma once

namespace ss {

constexpr float kSH_C0 = 0.28209479177387814f;
constexpr float kSH_C1 = 0.4886025119029199f;
constexpr float kSH_C2_0 = 1.0925484305920792f;
constexpr float kSH_C2_1 = -1.0925484305920792f;
constexpr float kSH_C2_2 = 0.31539156525252005f;
constexpr float kSH_C2_3 = -1.0925484305920792f;
constexpr float kSH_C2_4 = 0.5462742152960396f;
constexpr float kSH_C3_0 = -0.5900435899266435f;
constexpr float kSH_C3_1 = 2.890611442640554f;
constexpr float kSH_C3_2 = -0.4570457994644658f;
constexpr float kSH_C3_3 = 0.3731763325901154f;
constexpr float kSH_C3_4 = -0.4570457994644658f;
constexpr float kSH_C3_5 = 1.445305721320277f;
constexpr float kSH_C3_6 = -0.5900435899266435f;

__device__ __forceinline__ void quat_to_rot(const float q[4], float R[9]) {
    float w = q[0], x = q[1], y = q[2], z = q[3];
    R[0] = 1.f - 2.f * (y * y + z * z);
    R[1] = 2.f * (x * y - w * z);
    R[2] = 2.f * (x * z + w * y);
    R[3] = 2.f * (x * y + w * z);
    R[4] = 1.f - 2.f * (x * x + z * z);
    R[5] = 2.f * (y * z - w * x);
    R[6] = 2.f * (x * z - w * y);
    R[7] = 2.f * (y * z + w * x);
    R[8] = 1.f - 2.f * (x * x + y * y);
}

// 16 basis values at a unit direction (entries above the degree are 0).
__device__ __forceinline__ void sh_basis16(const float d[3], int degree, float b[16]) {
#pragma unroll
    for (int k = 0; k < 16; ++k) b[k] = 0.f;
    b[0] = kSH_C0;
    if (degree < 1) return;
    float x = d[0], y = d[1], z = d[2];
    b[1] = -kSH_C1 * y;
    b[2] = kSH_C1 * z;
    b[3] = -kSH_C1 * x;
    if (degree < 2) return;
    float xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
    b[4] = kSH_C2_0 * xy;
    b[5] = kSH_C2_1 * yz;
    b[6] = kSH_C2_2 * (2.f * zz - xx - yy);
    b[7] = kSH_C2_3 * xz;
    b[8] = kSH_C2_4 * (xx - yy);
    if (degree < 3) return;
    b[9] = kSH_C3_0 * y * (3.f * xx - yy);
    b[10] = kSH_C3_1 * xy * z;
    b[11] = kSH_C3_2 * y * (4.f * zz - xx - yy);
    b[12] = kSH_C3_3 * z * (2.f * zz - 3.f * xx - 3.f * yy);
    b[13] = kSH_C3_4 * x * (4.f * zz - xx - yy);
    b[14] = kSH_C3_5 * z * (xx - yy);
    b[15] = kSH_C3_6 * x * (xx - 3.f * yy);
}

// d basis_k / d dir, accumulated against per-coefficient weights coef[k]:
// gdir = sum_k coef[k] * grad basis_k (sh.py:73-119 contracted as in
// projection.py:272-274).
__device__ __forceinline__ void sh_dir_grad(const float d[3], int degree, const float coef[16],
                                            float gdir[3]) {
    gdir[0] = gdir[1] = gdir[2] = 0.f;
    if (degree < 1) return;
    float x = d[0], y = d[1], z = d[2];
    gdir[1] += coef[1] * -kSH_C1;
    gdir[2] += coef[2] * kSH_C1;
    gdir[0] += coef[3] * -kSH_C1;
    if (degree < 2) return;
    gdir[0] += coef[4] * kSH_C2_0 * y;
    gdir[1] += coef[4] * kSH_C2_0 * x;
    gdir[1] += coef[5] * kSH_C2_1 * z;
    gdir[2] += coef[5] * kSH_C2_1 * y;
    gdir[0] += coef[6] * kSH_C2_2 * -2.f * x;
    gdir[1] += coef[6] * kSH_C2_2 * -2.f * y;
    gdir[2] += coef[6] * kSH_C2_2 * 4.f * z;
    gdir[0] += coef[7] * kSH_C2_3 * z;
    gdir[2] += coef[7] * kSH_C2_3 * x;
    gdir[0] += coef[8] * kSH_C2_4 * 2.f * x;
    gdir[1] += coef[8] * kSH_C2_4 * -2.f * y;
    if (degree < 3) return;
    float xx = x * x, yy = y * y, zz = z * z;
    gdir[0] += coef[9] * kSH_C3_0 * 6.f * x * y;
    gdir[1] += coef[9] * kSH_C3_0 * (3.f * xx - 3.f * yy);
    gdir[0] += coef[10] * kSH_C3_1 * y * z;
    gdir[1] += coef[10] * kSH_C3_1 * x * z;
    gdir[2] += coef[10] * kSH_C3_1 * x * y;
    gdir[0] += coef[11] * kSH_C3_2 * -2.f * x * y;
    gdir[1] += coef[11] * kSH_C3_2 * (4.f * zz - xx - 3.f * yy);
    gdir[2] += coef[11] * kSH_C3_2 * 8.f * y * z;
    gdir[0] += coef[12] * kSH_C3_3 * -6.f * x * z;
    gdir[1] += coef[12] * kSH_C3_3 * -6.f * y * z;
    gdir[2] += coef[12] * kSH_C3_3 * (6.f * zz - 3.f * xx - 3.f * yy);
    gdir[0] += coef[13] * kSH_C3_4 * (4.f * zz - 3.f * xx - yy);
    gdir[1] += coef[13] * kSH_C3_4 * -2.f * x * y;
    gdir[2] += coef[13] * kSH_C3_4 * 8.f * x * z;
    gdir[0] += coef[14] * kSH_C3_5 * 2.f * x * z;
    gdir[1] += coef[14] * kSH_C3_5 * -2.f * y * z;
    gdir[2] += coef[14] * kSH_C3_5 * (xx - yy);
    gdir[0] += coef[15] * kSH_C3_6 * (3.f * xx - 3.f * yy);
    gdir[1] += coef[15] * kSH_C3_6 * -6.f * x * y;
}

// rgb = max(0, sum_k b_k sh_k + 0.5), active = pre-clamp > 0
// (sh.py:122-132, projection.py:151-155).  rest = coefficients 1..15.
__device__ __forceinline__ void sh_color(const float d[3], int degree, const float dc[3],
                                         const float* __restrict__ rest, float rgb[3],
                                         bool act[3]) {
    float b[16];
    sh_basis16(d, degree, b);
    int nb = (degree + 1) * (degree + 1);
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        float raw = b[0] * dc[ch];
        // static indices (b stays in registers), same summation order
#pragma unroll
        for (int k = 1; k < 16; ++k)
            if (k < nb) raw += b[k] * rest[3 * (k - 1) + ch];
        raw += 0.5f;
        act[ch] = raw > 0.f;
        rgb[ch] = fmaxf(raw, 0.f);
    }
}

}  // namespace ss
