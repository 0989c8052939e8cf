// stage1_lean.cuh — per-triangle pieces of the f32 / u32 stage-1 cull
// filter: the decision under a bound (lean_decide), the per-triangle bound
// (lean_bits), used by the generic (non-strip) lanes of the kernels in
// stage1_v2.cuh.  Decisions are a
// subset of filter_tri's (filter.cuh error model), so the result is
// bit-identical to the all-fp64 path.
#pragma once
#include "exact.cuh"
#include "filter.cuh"
#include "qxres.cuh"

namespace curast {

// bit 0: needs fp64, bit 1: frustum-culled (else tiny-culled), from the fp32
// bbox [mn, mx] of the projected vertices and its error bound eps
__device__ __forceinline__ unsigned lean_decide(float mnx, float mxx, float mny, float mxy,
                                                float eps, bool near_ok, float W, float H,
                                                bool tiny) {
    const float lox = mnx - eps, loy = mny - eps, hix = mxx + eps, hiy = mxy + eps;
    // interior: neither frustum test can hold; offscreen then needs a
    // zero-extent bbox: hi - lo > 4 eps  <=>  max - min > 2 eps
    const bool interior = lox > 0.0f && loy > 0.0f && hix < W && hiy < H;
    const float e4 = 4.0f * eps;
    const bool ext = (hix - lox > e4) && (hiy - loy > e4);
    // tiny: ceil(min - eps - 0.5) + 0.5 > max + eps, per axis
    const bool tx = ceilf(lox - 0.5f) > hix - 0.5f;
    const bool ty = ceilf(loy - 0.5f) > hiy - 0.5f;
    const bool is_tiny = near_ok && interior && tiny && ext && (tx || ty);
    // border / outside: only the frustum cull is decided here
    const bool is_fr = near_ok && !interior && (hix < 0.0f || hiy < 0.0f || lox > W || loy > H);
    unsigned bits = 0;
    if (!(is_tiny || is_fr)) bits |= 1u;
    if (is_fr) bits |= 2u;
    return bits;
}

// One projected vertex: P = (X', Y') / d', D = d' (the per-vertex half of
// lean_bits; a strip vertex shared by several triangles is projected once).
struct LeanV {
    float2 P;
    float D;
};

__device__ __forceinline__ LeanV lean_vertex(const LeanConsts &F, float x, float y, float z) {
    LeanV v;
    v.D = __fmaf_rn(F.dz, z, __fmaf_rn(F.dy, y, __fmaf_rn(F.dx, x, F.d3)));
    float2 t = __ffma2_rn(F.cx, make_float2(x, x), F.c3);
    t = __ffma2_rn(F.cy, make_float2(y, y), t);
    t = __ffma2_rn(F.cz, make_float2(z, z), t);
    const float r = rcp_approx(v.D);
    v.P = __fmul2_rn(t, make_float2(r, r));
    return v;
}

// The per-triangle half: symmetric in the three vertices (min / max only).
__device__ __forceinline__ unsigned lean_bits_v(const LeanConsts &F, const LeanV &a,
                                                const LeanV &b, const LeanV &c, float W, float H,
                                                float slack, bool tiny) {
    const float dmin = fminf(a.D, fminf(b.D, c.D));
    const float mnx = fminf(a.P.x, fminf(b.P.x, c.P.x));
    const float mxx = fmaxf(a.P.x, fmaxf(b.P.x, c.P.x));
    const float mny = fminf(a.P.y, fminf(b.P.y, c.P.y));
    const float mxy = fmaxf(a.P.y, fmaxf(b.P.y, c.P.y));
    const float M = fmaxf(fmaxf(fabsf(mnx), fabsf(mxx)), fmaxf(fabsf(mny), fabsf(mxy)));
    float eps = __fmaf_rn(M, F.ed, F.exy) * rcp_approx(dmin);
    eps = __fmaf_rn(eps, 1.5f, __fmaf_rn(M, kRelSlack, slack));
    return lean_decide(mnx, mxx, mny, mxy, eps, dmin > F.near_hi, W, H, tiny);
}

__device__ __forceinline__ unsigned lean_bits(const LeanConsts &F, const float *x, const float *y,
                                              const float *z, float W, float H, float slack,
                                              bool tiny) {
    return lean_bits_v(F, lean_vertex(F, x[0], y[0], z[0]), lean_vertex(F, x[1], y[1], z[1]),
                       lean_vertex(F, x[2], y[2], z[2]), W, H, slack, tiny);
}

}  // namespace curast
