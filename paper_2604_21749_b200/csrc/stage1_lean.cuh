// stage1_lean.cuh — per-triangle pieces of the f32 / u32 stage-1 cull
// filter (the decision and the per-triangle bound) and the two kernels that
// use them directly:
//   * k_s1_lean_ilv: the flat table over lane-major index steps
//     (indices_ilv), used for instanced frames drawn through the flat table
//     (their unique geometry is L2-resident, so the loads are L1-latency
//     bound and fewer L1 lines per gather win);
//   * k_s1i_lean: the instanced work space (a unique triangle's vertices
//     fetched once, tested under CURAST_INST_BLOCK instance transforms).
// The streamed flat path (k_s1_v2) is in stage1_v2.cuh.  Decisions are a
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

// fp64 queue entry: the 9 object-space positions + tag (CURAST_QX_WORDS)
__device__ __forceinline__ void qx_write(const curast_frame_t &f, long long slot, const float *x,
                                         const float *y, const float *z, long long tag) {
    if (slot >= f.qx_cap) return;
    int64_t *e = f.qx + CURAST_QX_WORDS * slot;
    *(float4 *)e = make_float4(x[0], y[0], z[0], x[1]);
    *(float4 *)(e + 2) = make_float4(y[1], z[1], x[2], y[2]);
    *(float2 *)(e + 4) = make_float2(z[2], 0.0f);
    e[CURAST_QX_TAG] = tag;
}

// Per-triangle lean kernel over the lane-major index steps (indices_ilv):
// the same per-triangle decisions as k_s1_v2's generic lanes, but lane l
// owns triangles l, l+32, l+64, l+96 of a 128-triangle step, so each of the 12 vertex
// gathers of a warp reads the vertices of 32 consecutive triangles — about
// half the L1 lines (the filter is bound by L1 data-pipe wavefronts).
template <int MINB>
__global__ void __launch_bounds__(256, MINB) k_s1_lean_ilv(const curast_frame_t f, int64_t cbeg,
                                                           int64_t cend, int claim_slot) {
    constexpr int CHUNK = kS1Chunk, MT = CURAST_STEP_TRIS, SW = 384;
    const int lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    unsigned n_frustum = 0, n_tiny = 0;
    const float W = (float)f.width, H = (float)f.height;
    const float slack = (float)(f.width > f.height ? f.width : f.height) * 1.4551915e-11f;
    const bool tiny = f.tiny_cull != 0;
    const int64_t total = min(cend, __ldg(f.unit_chunk_prefix + f.n_units));
    unsigned long long *qcount = (unsigned long long *)(f.counters + CURAST_C_QX);
    __shared__ QxReserve sres[8];
    QxReserve &R = sres[threadIdx.x >> 5];
    if (lane == 0) R = QxReserve{0u, 0};
    __syncwarp();
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
        const float4 *pb = (const float4 *)f.positions + __ldg(f.item_vtx_off + item);
        // chunk-relative 32-bit triangle numbers from the first step it touches
        const long long s0 = lo / MT, base = s0 * MT;
        const int rlo = (int)(lo - base), rhi = (int)(hi - base);
        const uint4 *sp = (const uint4 *)(f.indices_ilv + __ldg(f.item_ilv_off + item) + s0 * SW);
        const long long tag = (item << 40) | base;
        const int nst = (rhi + MT - 1) / MT;
        for (int st = 0; st < nst; ++st) {
            const uint4 *v = sp + st * (SW / 4) + 3 * lane;
            const uint4 a = __ldg(v), b4 = __ldg(v + 1), d = __ldg(v + 2);
            const uint32_t ix[12] = {a.x, a.y, a.z, a.w, b4.x, b4.y, b4.z, b4.w, d.x, d.y, d.z, d.w};
            const int tb = st * MT + lane;            // slot t: tb + 32 t
            const int lim = min(rhi, st * MT + MT);
            unsigned valid = 0;
#pragma unroll
            for (int t = 0; t < 4; ++t) valid |= (unsigned)(tb + 32 * t >= rlo && tb + 32 * t < lim) << t;
            float px[12], py[12], pz[12];
#pragma unroll
            for (int k = 0; k < 12; ++k) {
                const float4 q = __ldg(pb + ix[k]);
                px[k] = q.x;
                py[k] = q.y;
                pz[k] = q.z;
            }
            unsigned need = 0, fr = 0;
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const unsigned bits = lean_bits(F, px + 3 * t, py + 3 * t, pz + 3 * t, W, H, slack, tiny);
                need |= (bits & 1u) << t;
                fr |= (bits >> 1) << t;
            }
            need &= valid;
            fr &= valid;
            n_frustum += __popc(fr);
            n_tiny += __popc(valid) - __popc(need) - __popc(fr);
            unsigned b[4];
            int tot = 0;
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                b[t] = __ballot_sync(0xffffffffu, (need >> t) & 1u);
                tot += __popc(b[t]);
            }
            if (tot) {
                const QxSlots qs = qx_reserve(R, qcount, tot, lane);
                int qb = 0;
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    if ((need >> t) & 1u)
                        qx_write(f, qs.at(qb + __popc(b[t] & lt_mask)), px + 3 * t, py + 3 * t,
                                 pz + 3 * t, tag + tb + 32 * t);
                    qb += __popc(b[t]);
                }
            }
        }
    }
    qx_reserve_close(f, R, lane);
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
    __shared__ QxReserve sres[8];
    QxReserve &R = sres[threadIdx.x >> 5];
    if (lane == 0) R = QxReserve{0u, 0};
    __syncwarp();

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
                const QxSlots qs = qx_reserve(R, qcount, __popc(b), lane);
                if (need) {
                    const long long slot = qs.at(__popc(b & lt_mask));
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
    qx_reserve_close(f, R, lane);
    unsigned long long cnt[2] = {n_frustum, n_tiny};
    flush_stats(f.counters + CURAST_C_S1 + CULL_FRUSTUM, cnt, 1);
    flush_stats(f.counters + CURAST_C_S1 + CULL_TINY, cnt + 1, 1);
}

}  // namespace curast
