// stage1_lean.cuh — lean stage-1 cull filter for u32 index buffers (the
// roofline layout): the per-triangle instruction count is the budget.
//
//   * warp-granular chunk claims (2048 triangles), no block barriers;
//   * each lane owns 4 consecutive triangles per step: 3 x 128-bit index
//     loads, 36 independent position loads issued before the math;
//   * projection on packed f32x2 FFMA2/FMUL2 ((X, Y) per vertex);
//   * branch-free decision: near-plane cases and triangles touching the
//     viewport border (not provably interior, not provably outside) go to
//     fp64 — rare, and it removes the border logic from the hot path;
//   * 32-bit offsets inside a chunk, one atomic per 128 triangles for the
//     fp64 queue, stats from popcounts.
// Decisions are a subset of filter_tri's (filter.cuh error model), so the
// result is bit-identical to the all-fp64 path.
#pragma once
#include "exact.cuh"
#include "filter.cuh"

namespace curast {

struct LeanConsts {
    float2 cx, cy, cz, c3;   // (X, Y) rows
    float dx, dy, dz, d3;    // d row
    float exy, ed, near_hi;
};

__device__ __forceinline__ void lean_load(LeanConsts &F, const float *__restrict__ p) {
    const float4 *q = (const float4 *)p;
    const float4 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2), d = __ldg(q + 3);
    F.cx = make_float2(a.x, b.x);
    F.cy = make_float2(a.y, b.y);
    F.cz = make_float2(a.z, b.z);
    F.c3 = make_float2(a.w, b.w);
    F.dx = c.x; F.dy = c.y; F.dz = c.z; F.d3 = c.w;
    F.exy = d.x; F.ed = d.y; F.near_hi = d.z;
}

// 0 = fp64 needed, CULL_FRUSTUM, CULL_TINY
__device__ __forceinline__ int lean_filter(const LeanConsts &F, const float *x, const float *y,
                                           const float *z, float W, float H, float slack,
                                           bool tiny) {
    float2 P[3];
    float D[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        D[k] = __fmaf_rn(F.dz, z[k], __fmaf_rn(F.dy, y[k], __fmaf_rn(F.dx, x[k], F.d3)));
        float2 t = __ffma2_rn(F.cx, make_float2(x[k], x[k]), F.c3);
        t = __ffma2_rn(F.cy, make_float2(y[k], y[k]), t);
        t = __ffma2_rn(F.cz, make_float2(z[k], z[k]), t);
        const float r = rcp_approx(D[k]);
        P[k] = __fmul2_rn(t, make_float2(r, r));
    }
    const float dmin = fminf(D[0], fminf(D[1], D[2]));
    const float mnx = fminf(P[0].x, fminf(P[1].x, P[2].x));
    const float mxx = fmaxf(P[0].x, fmaxf(P[1].x, P[2].x));
    const float mny = fminf(P[0].y, fminf(P[1].y, P[2].y));
    const float mxy = fmaxf(P[0].y, fmaxf(P[1].y, P[2].y));
    const float M = fmaxf(fmaxf(fabsf(mnx), fabsf(mxx)), fmaxf(fabsf(mny), fabsf(mxy)));
    float eps = __fmaf_rn(M, F.ed, F.exy) * rcp_approx(dmin);
    eps = __fmaf_rn(eps, 1.5f, __fmaf_rn(M, kRelSlack, slack));
    const float lox = mnx - eps, loy = mny - eps, hix = mxx + eps, hiy = mxy + eps;
    const bool near_ok = dmin > F.near_hi;
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
    return is_tiny ? CULL_TINY : (is_fr ? CULL_FRUSTUM : FILT_EXACT);
}

// bit 0: needs fp64, bit 1: frustum-culled (else tiny-culled)
__device__ __forceinline__ unsigned lean_bits(const LeanConsts &F, const float *x, const float *y,
                                              const float *z, float W, float H, float slack,
                                              bool tiny) {
    float2 P[3];
    float D[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        D[k] = __fmaf_rn(F.dz, z[k], __fmaf_rn(F.dy, y[k], __fmaf_rn(F.dx, x[k], F.d3)));
        float2 t = __ffma2_rn(F.cx, make_float2(x[k], x[k]), F.c3);
        t = __ffma2_rn(F.cy, make_float2(y[k], y[k]), t);
        t = __ffma2_rn(F.cz, make_float2(z[k], z[k]), t);
        const float r = rcp_approx(D[k]);
        P[k] = __fmul2_rn(t, make_float2(r, r));
    }
    const float dmin = fminf(D[0], fminf(D[1], D[2]));
    const float mnx = fminf(P[0].x, fminf(P[1].x, P[2].x));
    const float mxx = fmaxf(P[0].x, fmaxf(P[1].x, P[2].x));
    const float mny = fminf(P[0].y, fminf(P[1].y, P[2].y));
    const float mxy = fmaxf(P[0].y, fmaxf(P[1].y, P[2].y));
    const float M = fmaxf(fmaxf(fabsf(mnx), fabsf(mxx)), fmaxf(fabsf(mny), fabsf(mxy)));
    float eps = __fmaf_rn(M, F.ed, F.exy) * rcp_approx(dmin);
    eps = __fmaf_rn(eps, 1.5f, __fmaf_rn(M, kRelSlack, slack));
    const float lox = mnx - eps, loy = mny - eps, hix = mxx + eps, hiy = mxy + eps;
    const bool near_ok = dmin > F.near_hi;
    const bool interior = lox > 0.0f && loy > 0.0f && hix < W && hiy < H;
    const float e4 = 4.0f * eps;
    const bool ext = (hix - lox > e4) && (hiy - loy > e4);
    const bool tx = ceilf(lox - 0.5f) > hix - 0.5f;
    const bool ty = ceilf(loy - 0.5f) > hiy - 0.5f;
    const bool is_tiny = near_ok && interior && tiny && ext && (tx || ty);
    const bool is_fr = near_ok && !interior && (hix < 0.0f || hiy < 0.0f || lox > W || loy > H);
    unsigned bits = 0;
    if (!(is_tiny || is_fr)) bits |= 1u;
    if (is_fr) bits |= 2u;
    return bits;
}

template <int PF, int MINB, int TPL>
__global__ void __launch_bounds__(256, MINB) k_s1_lean(const curast_frame_t f, int64_t cbeg,
                                                        int64_t cend, int claim_slot) {
    // processes chunks [cbeg, min(cend, total)) of the flat table, claimed
    // through counters[claim_slot] (slices of one frame use distinct slots)
    constexpr int CHUNK = 2048, STEP = 32 * TPL;
    const int lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    unsigned n_frustum = 0, n_tiny = 0;
    const float W = (float)f.width, H = (float)f.height;
    const float slack = (float)(f.width > f.height ? f.width : f.height) * 1.4551915e-11f;
    const bool tiny = f.tiny_cull != 0;
    const int64_t total = min(cend, __ldg(f.unit_chunk_prefix + f.n_units));
    unsigned long long *qcount = (unsigned long long *)(f.counters + CURAST_C_QX);

    for (;;) {
        long long c = 0, item = 0, lo = 0, hi = 0;
        if (lane == 0) {
            c = cbeg + (long long)atomicAdd((unsigned long long *)(f.counters + claim_slot), 1ull);
            if (c < total) {
                const int64_t u = upper_index(f.unit_chunk_prefix, f.n_units + 1, c);
                item = __ldg(f.unit_index + u);
                lo = __ldg(f.unit_lo + u) + (c - __ldg(f.unit_chunk_prefix + u)) * CHUNK;
                hi = __ldg(f.unit_hi + u);
                hi = lo + CHUNK < hi ? lo + CHUNK : hi;
            }
        }
        c = __shfl_sync(0xffffffffu, c, 0);
        if (c >= total) break;
        item = __shfl_sync(0xffffffffu, item, 0);
        lo = __shfl_sync(0xffffffffu, lo, 0);
        hi = __shfl_sync(0xffffffffu, hi, 0);

        LeanConsts F;
        lean_load(F, f.item_filter + CURAST_FILTER_FLOATS * item);
        const int64_t vo = __ldg(f.item_vtx_off + item);
        const int64_t io = __ldg(f.item_idx_off + item);
        // float4 positions: one 128-bit gather per vertex (the [V][3]
        // layout cost 3 loads and ~3x the L1 wavefronts per warp gather)
        const float4 *pb = (const float4 *)f.positions + vo;
        const uint32_t *ib = (const uint32_t *)f.indices + io + 3 * lo;
        const int n = (int)(hi - lo);
        const bool vec = (((uintptr_t)ib) & 15) == 0;
        const long long tag = (item << 40) | lo;

        for (int s0 = 0; s0 < n; s0 += STEP) {
            const int o = s0 + TPL * lane;
            const int nv = max(0, min(TPL, n - o));
            uint32_t ix[3 * TPL];
            if (TPL == 4 && vec && nv == TPL) {
                const uint4 *v = (const uint4 *)(ib + 3 * o);
                const uint4 a = __ldg(v), b = __ldg(v + 1), d = __ldg(v + 2);
                ix[0] = a.x; ix[1] = a.y; ix[2] = a.z; ix[3] = a.w;
                ix[4] = b.x; ix[5] = b.y; ix[6] = b.z; ix[7] = b.w;
                ix[8] = d.x; ix[9] = d.y; ix[10] = d.z; ix[11] = d.w;
            } else if (TPL == 2 && vec && nv == TPL) {
                const uint2 *v = (const uint2 *)(ib + 3 * o);
                const uint2 a = __ldg(v), b = __ldg(v + 1), d = __ldg(v + 2);
                ix[0] = a.x; ix[1] = a.y; ix[2] = b.x; ix[3] = b.y; ix[4] = d.x; ix[5] = d.y;
            } else {
#pragma unroll
                for (int k = 0; k < 3 * TPL; ++k) ix[k] = (k < 3 * nv) ? __ldg(ib + 3 * o + k) : 0u;
            }
            float px[3 * TPL], py[3 * TPL], pz[3 * TPL];
#pragma unroll
            for (int k = 0; k < 3 * TPL; ++k) {
                const float4 q = __ldg(pb + ix[k]);
                px[k] = q.x;
                py[k] = q.y;
                pz[k] = q.z;
            }
            unsigned need = 0, fr = 0;
#pragma unroll
            for (int t = 0; t < TPL; ++t) {
                const unsigned bits = lean_bits(F, px + 3 * t, py + 3 * t, pz + 3 * t, W, H, slack, tiny);
                if (t < nv) {
                    need |= (bits & 1u) << t;
                    fr |= (bits >> 1) << t;
                }
            }
            n_frustum += __popc(fr);
            n_tiny += nv - __popc(need) - __popc(fr);
            unsigned b[TPL];
            int tot = 0;
#pragma unroll
            for (int t = 0; t < TPL; ++t) {
                b[t] = __ballot_sync(0xffffffffu, (need >> t) & 1u);
                tot += __popc(b[t]);
            }
            if (tot) {
                unsigned long long base = 0;
                if (lane == 0) base = atomicAdd(qcount, (unsigned long long)tot);
                base = __shfl_sync(0xffffffffu, base, 0);
#pragma unroll
                for (int t = 0; t < TPL; ++t) {
                    if ((need >> t) & 1u) {
                        const long long slot = (long long)base + __popc(b[t] & lt_mask);
                        if (slot < f.qx_cap) {
                            // positions travel with the entry: the fp64 kernel
                            // does not re-gather them from HBM
                            int64_t *e = f.qx + CURAST_QX_WORDS * slot;
                            *(float4 *)e = make_float4(px[3 * t], py[3 * t], pz[3 * t], px[3 * t + 1]);
                            *(float4 *)(e + 2) = make_float4(py[3 * t + 1], pz[3 * t + 1],
                                                             px[3 * t + 2], py[3 * t + 2]);
                            *(float2 *)(e + 4) = make_float2(pz[3 * t + 2], 0.0f);
                            e[CURAST_QX_TAG] = tag + o + t;
                        }
                    }
                    base += __popc(b[t]);
                }
            }
        }
    }
    unsigned long long cnt[2] = {n_frustum, n_tiny};
    flush_stats(f.counters + CURAST_C_S1 + CULL_FRUSTUM, cnt, 1);
    flush_stats(f.counters + CURAST_C_S1 + CULL_TINY, cnt + 1, 1);
}

// Instanced stage-1 filter (kernels.py:205-254): a lane owns one unique
// triangle of a node group, fetches its indices and positions once and tests
// it under every surviving instance transform of the group (the group is
// uniform across the warp, so each instance's filter block is one broadcast
// load).  Undecided (instance, triangle) pairs go to the fp64 queue with their
// object-space positions; the exact kernel applies the instance's matrix.
template <int PF, int MINB>
__global__ void __launch_bounds__(256, MINB) k_s1i_lean(const curast_frame_t f) {
    const int64_t CHUNK = f.inst_chunk_tris;             // unique triangles per warp claim
    const int lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    unsigned n_frustum = 0, n_tiny = 0;
    const float W = (float)f.width, H = (float)f.height;
    const float slack = (float)(f.width > f.height ? f.width : f.height) * 1.4551915e-11f;
    const bool tiny = f.tiny_cull != 0;
    const int64_t total = __ldg(f.inst_unit_chunk_prefix + f.n_inst_units);
    unsigned long long *qcount = (unsigned long long *)(f.counters + CURAST_C_QX);

    for (;;) {
        long long c = 0, g = 0, lo = 0, hi = 0;
        if (lane == 0) {
            c = (long long)atomicAdd((unsigned long long *)(f.counters + CURAST_C_CLAIM1I), 1ull);
            if (c < total) {
                const int64_t u = upper_index(f.inst_unit_chunk_prefix, f.n_inst_units + 1, c);
                g = __ldg(f.inst_unit_index + u);
                lo = __ldg(f.inst_unit_lo + u) + (c - __ldg(f.inst_unit_chunk_prefix + u)) * CHUNK;
                hi = __ldg(f.inst_unit_hi + u);
                hi = lo + CHUNK < hi ? lo + CHUNK : hi;
            }
        }
        c = __shfl_sync(0xffffffffu, c, 0);
        if (c >= total) break;
        g = __shfl_sync(0xffffffffu, g, 0);
        lo = __shfl_sync(0xffffffffu, lo, 0);
        hi = __shfl_sync(0xffffffffu, hi, 0);
        // unit = group | first instance << 32 (CURAST_INST_BLOCK instances)
        const int64_t k0 = g >> 32;
        g &= 0xFFFFFFFFll;
        const int64_t ioff = __ldg(f.group_item_off + g);
        const int64_t icount = min(__ldg(f.group_item_count + g), k0 + CURAST_INST_BLOCK);
        const int64_t first = __ldg(f.group_items + ioff);
        const float4 *pb = (const float4 *)f.positions + __ldg(f.item_vtx_off + first);
        const uint32_t *ib = (const uint32_t *)f.indices + __ldg(f.item_idx_off + first);
      for (long long sub = lo; sub < hi; sub += 32) {
        const int64_t local = sub + lane;
        const bool valid = local < hi;
        float x[3], y[3], z[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const uint32_t v = valid ? __ldg(ib + 3 * local + k) : 0u;
            const float4 q = __ldg(pb + v);
            x[k] = q.x;
            y[k] = q.y;
            z[k] = q.z;
        }
        for (int64_t k = k0; k < icount; ++k) {
            const int64_t item = __ldg(f.group_items + ioff + k);
            LeanConsts F;
            lean_load(F, f.item_filter + CURAST_FILTER_FLOATS * item);
            const unsigned bits = lean_bits(F, x, y, z, W, H, slack, tiny);
            const bool need = valid && (bits & 1u);
            if (valid && (bits & 2u)) ++n_frustum;
            if (valid && bits == 0u) ++n_tiny;
            const unsigned b = __ballot_sync(0xffffffffu, need);
            if (b) {
                unsigned long long base = 0;
                if (lane == 0) base = atomicAdd(qcount, (unsigned long long)__popc(b));
                base = __shfl_sync(0xffffffffu, base, 0);
                if (need) {
                    const long long slot = (long long)base + __popc(b & lt_mask);
                    if (slot < f.qx_cap) {
                        int64_t *e = f.qx + CURAST_QX_WORDS * slot;
                        *(float4 *)e = make_float4(x[0], y[0], z[0], x[1]);
                        *(float4 *)(e + 2) = make_float4(y[1], z[1], x[2], y[2]);
                        *(float2 *)(e + 4) = make_float2(z[2], 0.0f);
                        e[CURAST_QX_TAG] = (item << 40) | local;
                    }
                }
            }
        }
      }
    }
    unsigned long long cnt[2] = {n_frustum, n_tiny};
    flush_stats(f.counters + CURAST_C_S1 + CULL_FRUSTUM, cnt, 1);
    flush_stats(f.counters + CURAST_C_S1 + CULL_TINY, cnt + 1, 1);
}

}  // namespace curast
