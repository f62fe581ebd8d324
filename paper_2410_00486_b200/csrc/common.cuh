// common.cuh -- shared device definitions for the B200 mapping hot path.
//
// Semantics follow the reference `splatstream` package (paths relative to
// /root/reference/pkg/src/splatstream); every threshold decision that the
// forward blend, the checkpoint replay and the splat-wise backward must agree
// on is made by ONE inline function (`splat_alpha`) built from explicit
// round-to-nearest intrinsics, so the compiler cannot contract it differently
// in the two kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/splatstream_b200.h"

namespace ss {

constexpr int kTile = 16;                 // RasterOpts.tile_size (api.py:41)
constexpr int kTilePx = kTile * kTile;    // 256 pixels = 256 threads per tile CTA
constexpr int kBucket = 32;               // RasterOpts.bucket_size (api.py:42) = warp width
constexpr int kUnit = 2 * kBucket;        // list positions per backward work unit (2 per lane)
constexpr float kLog2e = 1.4426950408889634f;

// Per-Gaussian screen-space record written by the preprocess kernel and
// gathered by the blend kernels through the sorted pair list (48 B, one
// 16-B-aligned struct so a gather is three LDG.128 from one 64-B window).
struct __align__(16) SplatRec {
    float4 a;  // mean2d.x, mean2d.y, conic[0], 2 * conic[1]
    float4 b;  // conic[2], sigma, m_cut, depth (camera-frame z)
    float4 c;  // r, g, b, half2 (x, y) half-extents of the blend region (+1 px, rounded up)
};

// Pixel-state checkpoint (T, r, g, b) archived before every 32nd list
// position (kernels.py:61-67); the depth channel adds a second plane.
// Layout: ckpt[(ckpt_base[tile] + bucket) * 256 + pixel].

// ------------------------------------------------------------------ alpha
// _alpha (kernels.py:14-31): m = c0 dx^2 + 2 c1 dx dy + c2 dy^2; skip when
// m > m_cut; a = sigma exp(-m/2); skip when a < alpha_min; clamp alpha_max.
// The forward applies the two skip tests around quad_* / splat_falloff; the
// backward recomputes alpha of recorded-blended pairs with the same
// operations.  Pixel coordinates are integers (api.py:108-115).
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Quadratic form m = c0 dx^2 + 2 c1 dx dy + c2 dy^2 with pinned rounding,
// as fma(c2 dy, dy, fma(2c1 dx, dy, (c0 dx) dx)); the record stores 2 c1
// (exact) in A.w.  The forward evaluates two pixels of one column with the
// dx-only terms shared; every evaluation uses exactly these operations.
__device__ __forceinline__ float quad_dx0(const float4& A, float dx) {
    return __fmul_rn(__fmul_rn(A.z, dx), dx);
}
__device__ __forceinline__ float quad_dx1(const float4& A, float dx) {
    return __fmul_rn(A.w, dx);
}
__device__ __forceinline__ float quad_finish(float q0, float q1, const float4& B, float dy) {
    return __fmaf_rn(__fmul_rn(B.x, dy), dy, __fmaf_rn(q1, dy, q0));
}
__device__ __forceinline__ float splat_power(float px, float py, const float4& A, const float4& B,
                                             float& dx, float& dy) {
    dx = __fsub_rn(px, A.x);
    dy = __fsub_rn(py, A.y);
    return quad_finish(quad_dx0(A, dx), quad_dx1(A, dx), B, dy);
}

// sigma * exp(-m/2) with pinned rounding (MUFU.EX2, flush-to-zero: values
// that small are far below alpha_min anyway).
__device__ __forceinline__ float splat_falloff(float m, const float4& B) {
    return __fmul_rn(B.y, ex2_approx(__fmul_rn(m, -0.5f * kLog2e)));
}

// Alpha of a pair the forward already recorded as blended (same
// arithmetic, no skip tests: they passed in the forward).
__device__ __forceinline__ float splat_alpha_blended(float px, float py, const float4& A,
                                                     const float4& B, float amax, float& dx,
                                                     float& dy) {
    return fminf(splat_falloff(splat_power(px, py, A, B, dx, dy), B), amax);
}

// ------------------------------------------------------- packed f32 x 2
// sm_100 FADD2 / FMUL2 / FFMA2: two IEEE float ops (round-to-nearest, per
// lane identical to the scalar op) in one issue slot.  Lane lo / hi.
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pk2(float lo, float hi) {
    f32x2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void upk2(f32x2 v, float& lo, float& hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f32x2 add2(f32x2 a, f32x2 b) {
    f32x2 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f32x2 sub2(f32x2 a, f32x2 b) {
    f32x2 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) {
    f32x2 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
    f32x2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

// ----------------------------------------------------------- error words
// Device error word layout (ss_error): first failing index via atomicMin.
__device__ __forceinline__ void report_first(int64_t* word, int64_t idx) {
    atomicMin(reinterpret_cast<unsigned long long*>(word), static_cast<unsigned long long>(idx));
}

__device__ __forceinline__ bool finitef(float x) { return isfinite(x); }

// ------------------------------------------------------------ warp utils
__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ int warp_max(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

inline int div_up(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

// Programmatic dependent launch: the kernel may be launched while its
// stream predecessor drains; every kernel launched this way begins with
// PDL_WAIT() (griddepcontrol.wait: the predecessor grid has completed and
// its memory is visible), so the stream semantics are unchanged and only
// the launch latency overlaps the predecessor's tail.
#define PDL_WAIT() asm volatile("griddepcontrol.wait;" ::: "memory")
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

}  // namespace ss
