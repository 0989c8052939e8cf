// prove.cuh — fp32 proof that a queued stage-1 triangle writes no fragment.
//
// Most triangles the cull filter cannot decide on a dense mesh are
// ST_RASTERIZED (kernels.py:116-157): their bbox holds a sample centre on
// both axes, yet about half of them cover no sample (the neighbouring
// triangle of the quad does).  The reference still counts them as rasterized
// with zero fragments.  This prover re-derives that outcome from the fp32
// projection (|px' - px64| <= eps, filter.cuh) and only answers when every
// test of _process_tri that precedes rasterization is decided, and every
// candidate sample is provably outside:
//
//   near plane  d' > near_hi                           (no clip, no forward)
//   frustum     bbox provably inside the viewport      (kernels.py:85-89)
//   offscreen   max - min > 4 eps on both axes         (kernels.py:103-108)
//   tiny        a sample centre provably in the bbox   (kernels.py:110-115)
//   degenerate  |denom' | > err_d; denom < 0 proves CULL_BACKFACE
//   small       widened pixel box area < small_max     (kernels.py:121-123)
//   coverage    for every pixel of the widened box one of s < 0, t < 0,
//               s + t > 1 holds beyond its error bound
//
// Edge functions at a sample S, with e1 = P1 - P0, e2 = P2 - P0,
// a = Sx - P0x, c = Sy - P0y:
//   Es = a e2y - c e2x  (= s * denom),  Et = c e1x - a e1y  (= t * denom),
//   E3 = denom - Es - Et  (= (1 - s - t) * denom).
// With every vertex coordinate off by <= eps and fp32 rounding u = 2^-24:
//   |dEs| <= eps (2|a| + |e2y| + 2|c| + |e2x|) + 4 eps^2 + 4u (|a e2y| + |c e2x|)
//   |dD|  <= 2 eps (|e1x| + |e1y| + |e2x| + |e2y|) + 8 eps^2 + 4u (|e1x e2y| + |e1y e2x|)
//   |dE3| <= |dD| + |dEs| + |dEt| + 2u (|D| + |Es| + |Et|)
// (second-order u*eps terms and the fp32 evaluation of the bounds are
// covered by a 2^-10 relative margin).  The reference evaluates s and t in
// fp64 from the fp64 vertices (incremental stepping, kernels.py:140-157);
// its rounding is < 2^-45 (W + H) sum|e| in edge units, covered by the
// 2^-30 (W + H) (1 + sum|e|) term.  Any NaN fails a test and answers NONE.
#pragma once
#include "filter.cuh"

namespace curast {

enum { PROVE_NONE = 0, PROVE_EMPTY = 1, PROVE_BACKFACE = 2 };

constexpr float kU24 = 5.9604644775390625e-08f;   // 2^-24
constexpr float kSafety = 1.0009765625f;            // 1 + 2^-10
constexpr float k2m30 = 9.313225746154785e-10f;     // 2^-30

// largest widened pixel box (per axis) the prover enumerates
constexpr int kProveMaxSpan = 4;

__device__ __forceinline__ int prove_no_fragments(const LeanConsts &F, const float *x,
                                                  const float *y, const float *z, float W,
                                                  float H, float slack, bool tiny,
                                                  float small_max) {
    LeanTri T;
    lean_project(T, F, x, y, z, slack);
    if (!(T.dmin > F.near_hi)) return PROVE_NONE;
    const float eps = T.eps;
    const float e2 = eps + eps;          // covers the rounding of the box arithmetic
    const float lox = T.mnx - e2, loy = T.mny - e2, hix = T.mxx + e2, hiy = T.mxy + e2;
    if (!(lox > 0.0f && loy > 0.0f && hix < W && hiy < H)) return PROVE_NONE;
    if (!(T.mxx - T.mnx > 2.0f * e2 && T.mxy - T.mny > 2.0f * e2)) return PROVE_NONE;
    if (tiny) {
        // smallest sample >= min lies <= max on both axes
        const float kx = ceilf((T.mnx + e2) - 0.5f), ky = ceilf((T.mny + e2) - 0.5f);
        if (!(kx + 0.5f <= T.mxx - e2 && ky + 0.5f <= T.mxy - e2)) return PROVE_NONE;
    }
    const float2 P0 = T.P[0];
    const float e1x = T.P[1].x - P0.x, e1y = T.P[1].y - P0.y;
    const float e2x = T.P[2].x - P0.x, e2y = T.P[2].y - P0.y;
    const float t1 = e1x * e2y, t2 = e1y * e2x;
    const float den = t1 - t2;
    const float esum = fabsf(e1x) + fabsf(e1y) + fabsf(e2x) + fabsf(e2y);
    const float ee = eps * eps;
    const float s64 = k2m30 * (W + H) * (1.0f + esum);
    const float errD = kSafety * (2.0f * eps * esum + 8.0f * ee + 4.0f * kU24 * (fabsf(t1) + fabsf(t2))) + s64;
    if (den < -errD) return PROVE_BACKFACE;
    if (!(den > errD)) return PROVE_NONE;
    const float fx0 = floorf(lox), fy0 = floorf(loy);
    const float bx = ceilf(hix) - fx0, by = ceilf(hiy) - fy0;
    if (!(bx * by < small_max)) return PROVE_NONE;            // would be forwarded
    if (bx > (float)kProveMaxSpan || by > (float)kProveMaxSpan) return PROVE_NONE;
    const int nx = (int)bx, ny = (int)by;
    for (int j = 0; j < ny; ++j) {
        const float c = (fy0 + (float)j + 0.5f) - P0.y;
        for (int i = 0; i < nx; ++i) {
            const float a = (fx0 + (float)i + 0.5f) - P0.x;
            const float u1 = a * e2y, u2 = c * e2x;
            const float Es = u1 - u2;
            const float v1 = c * e1x, v2 = a * e1y;
            const float Et = v1 - v2;
            const float E3 = (den - Es) - Et;
            const float errS = kSafety * (eps * (2.0f * fabsf(a) + fabsf(e2y) + 2.0f * fabsf(c) + fabsf(e2x)) +
                                          4.0f * ee + 4.0f * kU24 * (fabsf(u1) + fabsf(u2))) + s64;
            const float errT = kSafety * (eps * (2.0f * fabsf(c) + fabsf(e1x) + 2.0f * fabsf(a) + fabsf(e1y)) +
                                          4.0f * ee + 4.0f * kU24 * (fabsf(v1) + fabsf(v2))) + s64;
            const float err3 = kSafety * (errD + errS + errT +
                                          2.0f * kU24 * (fabsf(den) + fabsf(Es) + fabsf(Et))) + s64;
            if (!(Es < -errS || Et < -errT || E3 < -err3)) return PROVE_NONE;
        }
    }
    return PROVE_EMPTY;
}

}  // namespace curast
