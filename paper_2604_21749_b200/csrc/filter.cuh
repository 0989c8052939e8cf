// filter.cuh — conservative fp32 cull filter for stage 1.
//
// The reference decides every triangle in fp64 (kernels.py:49-128).  On the
// B200 the fp64 pipe runs at half the fp32 rate and the exact setup costs
// ~250 DP instructions per triangle, so stage 1 first evaluates the
// projection in fp32 with a rigorous per-triangle error bound `eps` on the
// pixel coordinates and only takes a decision the fp64 path provably makes
// too:
//   * CULL_FRUSTUM (kernels.py:85-89)   all px64 < 0 / > W or py64 < 0 / > H
//   * CULL_TINY    (kernels.py:110-115) no sample centre in the bbox on an
//                                        axis, after frustum/offscreen are
//                                        provably false
// Everything else (near-plane cases, survivors, ambiguous margins) returns
// EXACT and is re-done bit-exactly in fp64 after block-local compaction.
//
// Error model (host computes E_xy, E_d per item, see device.py):
//   X = px*d and Y = py*d are affine in the object position, d likewise.
//   |X' - X| <= E_xy, |d' - d| <= E_d over the item's vertex box, with
//   E = k u * sum|coeff|*|pos| (u = 2^-24; k = 6 / 7 / 10 for f32 / f64 /
//   u16 positions) covering coefficient rounding, the 3-FMA chain, and fp32
//   rounding/decode of the positions.
//   |px' - px| <= 4/3 (E_xy + |px'| E_d) / d' + |px'| 1.5 * 2^-23 (rcp + mul)
//   when d' > 4 E_d; fp64 rounding of the reference (<= 2^-50 relative) and
//   the fp32 comparison arithmetic are covered by the 1.5x / 2^-21 / 2^-36
//   slack terms.
#pragma once
#include "exact.cuh"

namespace curast {

enum { FILT_EXACT = 0 };

// relative slack on |px'|: rcp.approx (1 ulp = 2^-23), the fp32 multiply
// (2^-24) and the comparison additions (2^-24 each) need < 1.5 * 2^-22;
// 2^-21 keeps a 1.3x margin
constexpr float kRelSlack = 4.76837158203125e-07f;

__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

struct FilterConsts {
    float c[12];
    float exy, ed, near_hi;
};

// The block's (X, Y) rows are stored interleaved (curast.h
// CURAST_FILTER_FLOATS): X0 Y0 X1 Y1 | X2 Y2 X3 Y3 | d0 d1 d2 d3 | E_xy E_d
// near_hi -, so a lane's 128-bit loads give FFMA2-ready register pairs.
__device__ __forceinline__ void load_filter(FilterConsts &F, const float *__restrict__ p) {
    const float4 *q = (const float4 *)p;
    float4 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2), d = __ldg(q + 3);
    F.c[0] = a.x; F.c[1] = a.z; F.c[2] = b.x; F.c[3] = b.z;
    F.c[4] = a.y; F.c[5] = a.w; F.c[6] = b.y; F.c[7] = b.w;
    F.c[8] = c.x; F.c[9] = c.y; F.c[10] = c.z; F.c[11] = c.w;
    F.exy = d.x; F.ed = d.y; F.near_hi = d.z;
}

__device__ __forceinline__ float frow(const float *c, float x, float y, float z) {
    return __fmaf_rn(c[2], z, __fmaf_rn(c[1], y, __fmaf_rn(c[0], x, c[3])));
}

// Returns CULL_FRUSTUM, CULL_TINY or FILT_EXACT.
__device__ __forceinline__ int filter_tri(const FilterConsts &F, float ax, float ay, float az,
                                          float bx, float by, float bz, float cx, float cy,
                                          float cz, float W, float H, float WH_slack,
                                          bool tiny_cull) {
    float X0 = frow(F.c, ax, ay, az), Y0 = frow(F.c + 4, ax, ay, az), D0 = frow(F.c + 8, ax, ay, az);
    float X1 = frow(F.c, bx, by, bz), Y1 = frow(F.c + 4, bx, by, bz), D1 = frow(F.c + 8, bx, by, bz);
    float X2 = frow(F.c, cx, cy, cz), Y2 = frow(F.c + 4, cx, cy, cz), D2 = frow(F.c + 8, cx, cy, cz);
    float dmin = fminf(D0, fminf(D1, D2));
    if (!(dmin > F.near_hi)) return FILT_EXACT;   // near-plane outcomes: exact
    float r0 = rcp_approx(D0), r1 = rcp_approx(D1), r2 = rcp_approx(D2);
    float px0 = X0 * r0, py0 = Y0 * r0;
    float px1 = X1 * r1, py1 = Y1 * r1;
    float px2 = X2 * r2, py2 = Y2 * r2;
    float minx = fminf(px0, fminf(px1, px2)), maxx = fmaxf(px0, fmaxf(px1, px2));
    float miny = fminf(py0, fminf(py1, py2)), maxy = fmaxf(py0, fmaxf(py1, py2));
    float Mx = fmaxf(fmaxf(fabsf(minx), fabsf(maxx)), fmaxf(fabsf(miny), fabsf(maxy)));
    float eps = __fmaf_rn(Mx, F.ed, F.exy) * rcp_approx(dmin) * 1.5f;
    eps = __fmaf_rn(Mx, kRelSlack, eps) + WH_slack;
    // NDC frustum test (kernels.py:85-89) in pixel space: nx < -1 <=> px < 0
    if (maxx + eps < 0.0f || minx - eps > W || miny - eps > H || maxy + eps < 0.0f)
        return CULL_FRUSTUM;
    bool not_frustum = (maxx - eps > 0.0f) && (minx + eps < W) && (miny + eps < H) &&
                       (maxy - eps > 0.0f);
    if (!not_frustum || !tiny_cull) return FILT_EXACT;
    // offscreen (kernels.py:98-108) is then only possible for a zero-extent bbox
    float e2 = eps + eps;
    if (!(maxx - minx > e2 && maxy - miny > e2)) return FILT_EXACT;
    // tiny (kernels.py:110-115): smallest sample centre >= minx lies > maxx
    float hx = ceilf((minx - eps) - 0.5f) + 0.5f;
    float hy = ceilf((miny - eps) - 0.5f) + 0.5f;
    if (hx > maxx + eps || hy > maxy + eps) return CULL_TINY;
    return FILT_EXACT;
}

// ---------------------------------------------------------------- lean form
// The same filter block as packed (X, Y) rows for FFMA2/FMUL2.
struct LeanConsts {
    float2 cx, cy, cz, c3;   // (X, Y) rows
    float dx, dy, dz, d3;    // d row
    float exy, ed, near_hi;
};

__device__ __forceinline__ void lean_from(LeanConsts &F, const float4 &a, const float4 &b,
                                          const float4 &c, const float4 &d) {
    F.cx = make_float2(a.x, a.y);
    F.cy = make_float2(a.z, a.w);
    F.cz = make_float2(b.x, b.y);
    F.c3 = make_float2(b.z, b.w);
    F.dx = c.x; F.dy = c.y; F.dz = c.z; F.d3 = c.w;
    F.exy = d.x; F.ed = d.y; F.near_hi = d.z;
}

__device__ __forceinline__ void lean_load(LeanConsts &F, const float *__restrict__ p) {
    const float4 *q = (const float4 *)p;
    lean_from(F, __ldg(q), __ldg(q + 1), __ldg(q + 2), __ldg(q + 3));
}

}  // namespace curast
