// stage1_v2.cuh — the streamed stage-1 cull filter (f32 positions, u32
// indices): per-vertex projection sharing and a per-lane error bound.
//
// A lane owns 4 consecutive triangles of a 128-triangle warp step (3 x
// 128-bit index loads).  When the whole warp's index runs are quad-strip
// runs — (a,c,b),(b,c,d) (make_tessellated_quad) or (a,b,c),(b,d,c)
// (make_sphere) — the lane's 12 vertex refs name 6 distinct vertices: each
// is gathered and projected ONCE (6 LDG.128 + 6 projections instead of 12).
// The filter bound eps (filter.cuh) grows with max|p'| and 1/min d', so one
// eps over the lane's vertices bounds all four triangles; when every lane's
// vertex box lies provably inside the viewport and in front of the near
// margin (the warp-uniform common case) only the tiny cull is left to decide
// per triangle, else the full decision (lean_decide) runs.  Decisions are a
// subset of the fp64 path's (CULL_FRUSTUM / CULL_TINY proven with the
// rigorous bound), so the output is bit-identical to the all-fp64 path.
//
// Undecided triangles go to the global fp64 queue (48-byte entries with
// their positions, one reservation per 128 slots, qxres.cuh) for k_s1_exact.
#pragma once
#include "exact.cuh"
#include "filter.cuh"
#include "qxres.cuh"



namespace curast {

// lean_load through volatile non-coherent loads (kept inside the step loop).
__device__ __forceinline__ float4 ldg_step(const float *p) {
    float4 v;
    asm volatile("ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ void lean_load_step(LeanConsts &F, const float *p) {
    lean_from(F, ldg_step(p), ldg_step(p + 4), ldg_step(p + 8), ldg_step(p + 12));
}

// lean_load from a shared-memory copy of the filter block.
__device__ __forceinline__ void lean_load_smem(LeanConsts &F, const float4 *q) {
    lean_from(F, q[0], q[1], q[2], q[3]);
}

// One projected vertex (filter units): P = (X', Y') / d', D = d'.
struct PV {
    float2 P;
    float D;
};

__device__ __forceinline__ PV pv_project(const LeanConsts &F, const float4 &q) {
    PV v;
    v.D = __fmaf_rn(F.dz, q.z, __fmaf_rn(F.dy, q.y, __fmaf_rn(F.dx, q.x, F.d3)));
    float2 t = __ffma2_rn(F.cx, make_float2(q.x, q.x), F.c3);
    t = __ffma2_rn(F.cy, make_float2(q.y, q.y), t);
    t = __ffma2_rn(F.cz, make_float2(q.z, q.z), t);
    const float r = rcp_approx(v.D);
    v.P = __fmul2_rn(t, make_float2(r, r));
    return v;
}

// Lane bound over NV projected vertices: eps as filter.cuh / lean_bits_v
// with M = max |p'| and dmin = min d' over all of them (eps is monotone in
// both, so it bounds each of the lane's triangles), the lane's vertex box,
// and whether that box is provably interior (no frustum / near decision).
struct LaneB {
    float eps, e2, lo5, hi5;
    bool near_ok, interior;
};

template <int NV>
__device__ __forceinline__ LaneB lane_bound(const LeanConsts &F, const PV *v, float W, float H,
                                            float slack) {
    float dmin = v[0].D, mnx = v[0].P.x, mxx = v[0].P.x, mny = v[0].P.y, mxy = v[0].P.y;
#pragma unroll
    for (int k = 1; k < NV; ++k) {
        dmin = fminf(dmin, v[k].D);
        mnx = fminf(mnx, v[k].P.x);
        mxx = fmaxf(mxx, v[k].P.x);
        mny = fminf(mny, v[k].P.y);
        mxy = fmaxf(mxy, v[k].P.y);
    }
    LaneB b;
    const float M = fmaxf(fmaxf(fabsf(mnx), fabsf(mxx)), fmaxf(fabsf(mny), fabsf(mxy)));
    float eps = __fmaf_rn(M, F.ed, F.exy) * rcp_approx(dmin);
    eps = __fmaf_rn(eps, 1.5f, __fmaf_rn(M, kRelSlack, slack));
    b.eps = eps;
    b.e2 = eps + eps;
    b.lo5 = eps + 0.5f;
    b.hi5 = eps - 0.5f;
    b.near_ok = dmin > F.near_hi;
    b.interior = b.near_ok && (mnx - eps > 0.0f) && (mny - eps > 0.0f) && (mxx + eps < W) &&
                 (mxy + eps < H);
    return b;
}

// Tiny-cull decision of an interior triangle (every frustum / near /
// offscreen outcome provably false except a zero extent): 1 = fp64 needed.
template <bool FLAT_LOGIC = false>
__device__ __forceinline__ unsigned tri_fast(const PV &a, const PV &b, const PV &c, const LaneB &L,
                                             bool tiny) {
    const float mnx = fminf(a.P.x, fminf(b.P.x, c.P.x)), mxx = fmaxf(a.P.x, fmaxf(b.P.x, c.P.x));
    const float mny = fminf(a.P.y, fminf(b.P.y, c.P.y)), mxy = fmaxf(a.P.y, fmaxf(b.P.y, c.P.y));
    const float2 ext = __fadd2_rn(make_float2(mxx, mxy), make_float2(-mnx, -mny));
    const float2 lo = __fadd2_rn(make_float2(mnx, mny), make_float2(-L.lo5, -L.lo5));
    const float2 hi = __fadd2_rn(make_float2(mxx, mxy), make_float2(L.hi5, L.hi5));
    if constexpr (FLAT_LOGIC) {
        // non-short-circuit predicate logic: fewer selects (instanced kernel,
        // issue-bound: D 3.11 -> 3.05 ms); the streamed kernel keeps the
        // short-circuit form, whose predicated ceil is off its load chain
        const bool e = (ext.x > L.e2) & (ext.y > L.e2);
        const bool t = (ceilf(lo.x) > hi.x) | (ceilf(lo.y) > hi.y);
        return (tiny & e & t) ? 0u : 1u;
    } else {
        const bool e = (ext.x > L.e2) && (ext.y > L.e2);
        const bool t = (ceilf(lo.x) > hi.x) || (ceilf(lo.y) > hi.y);
        return (tiny && e && t) ? 0u : 1u;
    }
}

// Full decision (lean_decide) under the lane bound: bit 0 fp64, bit 1 frustum.
__device__ __forceinline__ unsigned tri_full(const PV &a, const PV &b, const PV &c, const LaneB &L,
                                             float W, float H, bool tiny) {
    const float mnx = fminf(a.P.x, fminf(b.P.x, c.P.x)), mxx = fmaxf(a.P.x, fmaxf(b.P.x, c.P.x));
    const float mny = fminf(a.P.y, fminf(b.P.y, c.P.y)), mxy = fmaxf(a.P.y, fmaxf(b.P.y, c.P.y));
    const float lox = mnx - L.eps, loy = mny - L.eps, hix = mxx + L.eps, hiy = mxy + L.eps;
    const bool interior = lox > 0.0f && loy > 0.0f && hix < W && hiy < H;
    const float e4 = 4.0f * L.eps;
    const bool ext = (hix - lox > e4) && (hiy - loy > e4);
    const bool tx = ceilf(lox - 0.5f) > hix - 0.5f;
    const bool ty = ceilf(loy - 0.5f) > hiy - 0.5f;
    const bool is_tiny = L.near_ok && interior && tiny && ext && (tx || ty);
    const bool is_fr = L.near_ok && !interior && (hix < 0.0f || hiy < 0.0f || lox > W || loy > H);
    return (is_tiny || is_fr) ? (is_fr ? 2u : 0u) : 1u;
}

// Vertex-ref patterns of a lane's 4 triangles (refs 3t..3t+2), two quads of
// a strip in the two triangulations of the benchmark generators:
//   0 generic: 12 gathered vertices, triangle t = (3t, 3t+1, 3t+2)
//   1 grid quads (a,c,b),(b,c,d) (make_tessellated_quad, scenedesc.py:207-214):
//     distinct refs 0,1,2,5,8,11 = U0..U5,
//     triangles (U0,U1,U2) (U2,U1,U3) (U2,U3,U4) (U4,U3,U5)
//   2 sphere quads (a,d,c),(a,b,d) (make_sphere, scenedesc.py:218-245):
//     distinct refs 0,1,2,4,7,10 = U0..U5,
//     triangles (U0,U1,U2) (U0,U3,U1) (U3,U4,U1) (U3,U5,U4)
// (each triangle's vertex order is irrelevant: the bbox tests are symmetric)
__device__ __forceinline__ int strip_kind(const uint32_t *ix, bool full) {
    const bool gq = full && ix[3] == ix[2] && ix[4] == ix[1] && ix[6] == ix[2] &&
                    ix[7] == ix[5] && ix[9] == ix[8] && ix[10] == ix[5];
    const bool sq = full && ix[3] == ix[0] && ix[5] == ix[1] && ix[6] == ix[4] &&
                    ix[8] == ix[1] && ix[9] == ix[4];
    return __all_sync(0xffffffffu, gq) ? 1 : (__all_sync(0xffffffffu, sq) ? 2 : 0);
}

// Distinct vertex refs of a strip lane (strip_r) and its triangles' vertex
// slots (strip_g: reference k = 3t + e -> slot among the 6 distinct ones).
__host__ __device__ constexpr int strip_r(int kind, int k) {
    return k < 3 ? k : (kind == 1 ? 3 * k - 4 : 3 * k - 5);
}
__host__ __device__ constexpr int strip_g(int kind, int k) {
    // kind 1: 0 1 2 | 2 1 3 | 2 3 4 | 4 3 5    kind 2: 0 1 2 | 0 3 1 | 3 4 1 | 3 5 4
    return kind == 1 ? (k == 0 ? 0 : k == 1 ? 1 : k == 2 ? 2 : k == 3 ? 2 : k == 4 ? 1 :
                        k == 5 ? 3 : k == 6 ? 2 : k == 7 ? 3 : k == 8 ? 4 : k == 9 ? 4 :
                        k == 10 ? 3 : 5)
                     : (k == 0 ? 0 : k == 1 ? 1 : k == 2 ? 2 : k == 3 ? 0 : k == 4 ? 3 :
                        k == 5 ? 1 : k == 6 ? 3 : k == 7 ? 4 : k == 8 ? 1 : k == 9 ? 3 :
                        k == 10 ? 5 : 4);
}
static_assert(strip_r(1, 3) == 5 && strip_r(1, 5) == 11 && strip_r(2, 3) == 4 &&
              strip_r(2, 5) == 10, "strip refs");

// Decisions of a strip lane's 4 triangles from its 6 distinct projected
// vertices under one lane bound: need bits in bits 0-3, frustum bits in bits
// 4-7, bit 8 = the lane's vertices are provably in front of the near plane
// and inside the viewport (CURAST_QX_INTERIOR for its queue entries).
template <int KIND, bool FLAT_LOGIC = false>
__device__ __forceinline__ unsigned strip_bits(const LeanConsts &F, const PV *v, float W, float H,
                                               float slack, bool tiny) {
    const LaneB L = lane_bound<6>(F, v, W, H, slack);
    unsigned bits = L.interior ? 0x100u : 0u;
    if (__all_sync(0xffffffffu, L.interior)) {
#pragma unroll
        for (int t = 0; t < 4; ++t)
            bits |= tri_fast<FLAT_LOGIC>(v[strip_g(KIND, 3 * t)], v[strip_g(KIND, 3 * t + 1)],
                                         v[strip_g(KIND, 3 * t + 2)], L, tiny) << t;
    } else {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const unsigned b = tri_full(v[strip_g(KIND, 3 * t)], v[strip_g(KIND, 3 * t + 1)],
                                        v[strip_g(KIND, 3 * t + 2)], L, W, H, tiny);
            bits |= ((b & 1u) << t) | ((b >> 1) << (4 + t));
        }
    }
    return bits;
}

// Generic lane (no strip pattern): triangle by triangle, 3 gathers and a
// per-triangle bound each (lean_bits), so only one triangle's vertices are
// live at a time.
template <int PF, int IF>
__device__ __forceinline__ unsigned generic_bits(const LeanConsts &F, const ItemGeo<PF, IF> &G,
                                                 const uint32_t *ix, float W, float H,
                                                 float slack, bool tiny) {
    unsigned bits = 0;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        float x[3], y[3], z[3];
#pragma unroll
        for (int e = 0; e < 3; ++e) G.pos32(ix[3 * t + e], x[e], y[e], z[e]);
        const unsigned r = lean_bits(F, x, y, z, W, H, slack, tiny);
        bits |= ((r & 1u) << t) | ((r >> 1) << (4 + t));
    }
    return bits;
}

// A stored vertex: its fp32 position for the filter and, for POS_U16, the raw
// grid coordinates the queue entry carries (k_s1_exact decodes them in fp64).
template <int PF>
struct SV {
    float3 p;
};
template <>
struct SV<CURAST_POS_U16> {
    uint2 q;
};

// KEEP: L2 evict-last hint for the vertex gathers — a grid row's vertices
// are read again by the next row's chunk, while the index and queue streams
// around them are evict-first (B 0.659 -> 0.653 ms stage 1, E200 3.61 ->
// 3.54 ms; D unchanged)
template <int PF, int IF, bool KEEP = true>
__device__ __forceinline__ SV<PF> sv_load(const ItemGeo<PF, IF> &G, uint32_t v) {
    SV<PF> s;
    if constexpr (PF == CURAST_POS_U16) {
        s.q = __ldg((const uint2 *)G.pos + v);
    } else if constexpr (KEEP) {
        uint64_t pol;
        asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
        float4 q;
        asm("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
            : "=f"(q.x), "=f"(q.y), "=f"(q.z), "=f"(q.w)
            : "l"((const float4 *)G.pos + v), "l"(pol));
        s.p = make_float3(q.x, q.y, q.z);
    } else {
        const float4 q = __ldg((const float4 *)G.pos + v);
        s.p = make_float3(q.x, q.y, q.z);
    }
    return s;
}

// fp32 position of a stored vertex (POS_U16: ItemGeo::pos32's decode)
template <int PF, int IF>
__device__ __forceinline__ float4 sv_pos(const ItemGeo<PF, IF> &G, const SV<PF> &s) {
    if constexpr (PF == CURAST_POS_U16) {
        return make_float4(__fmaf_rn(q16_half(s.q.x & 0xFFFFu), G.gs32[0], G.gm32[0]),
                           __fmaf_rn(q16_half(s.q.x >> 16), G.gs32[1], G.gm32[1]),
                           __fmaf_rn(q16_half(s.q.y & 0xFFFFu), G.gs32[2], G.gm32[2]), 0.f);
    } else {
        return make_float4(s.p.x, s.p.y, s.p.z, 0.f);
    }
}

// queue entry payload (words 0-4) of a triangle's three stored vertices
template <int PF>
__device__ __forceinline__ void qx_put_sv(const curast_frame_t &f, long long slot,
                                          const SV<PF> &a, const SV<PF> &b, const SV<PF> &c,
                                          long long tag) {
    if (slot >= f.qx_cap) return;
    int64_t *e = f.qx + CURAST_QX_WORDS * slot;
    if constexpr (PF == CURAST_POS_U16) {
        // the 9 raw u16 coordinates in words 0-2 (k_s1_exact qx_load_q16)
        const uint64_t q[9] = {a.q.x & 0xFFFFu, a.q.x >> 16, a.q.y & 0xFFFFu,
                               b.q.x & 0xFFFFu, b.q.x >> 16, b.q.y & 0xFFFFu,
                               c.q.x & 0xFFFFu, c.q.x >> 16, c.q.y & 0xFFFFu};
        __stcs((int4 *)e, make_int4((int)(q[0] | q[1] << 16), (int)(q[2] | q[3] << 16),
                                    (int)(q[4] | q[5] << 16), (int)(q[6] | q[7] << 16)));
        __stcs((long long *)(e + 2), (long long)q[8]);
        __stcs((long long *)(e + CURAST_QX_TAG), tag);
        return;
    } else {
        // streaming stores (evict-first): the queue is read once, by the
        // fp64 pass, and should not displace the vertex rows L2 holds for
        // the next grid row's chunk (with the index stream's streaming loads:
        // B 0.668 -> 0.661 ms stage 1, E200 3.97 -> 3.68 ms)
        __stcs((float4 *)e, make_float4(a.p.x, a.p.y, a.p.z, b.p.x));
        __stcs((float4 *)(e + 2), make_float4(b.p.y, b.p.z, c.p.x, c.p.y));
        __stcs((float2 *)(e + 4), make_float2(c.p.z, 0.0f));
        __stcs((long long *)(e + CURAST_QX_TAG), tag);
        return;
    }
    e[CURAST_QX_TAG] = tag;
}

// The warp's 128-triangle step at chunk offset s0: indices of triangles
// o .. o+3 (o = s0 + 4 lane) into ix[12]; nv valid triangles.
// STREAM: the flat table reads each index once per frame — streaming
// (evict-first) loads; the instanced kernel re-reads a group's run for every
// instance block and keeps the default policy.
template <bool STREAM = false>
__device__ __forceinline__ void load_step_indices(const uint32_t *__restrict__ ib, int o, int nv,
                                                  bool vec, uint32_t *ix) {
    if (vec && nv == 4) {
        const uint4 *v = (const uint4 *)(ib + 3 * o);
        uint4 a, b, d;
        if constexpr (STREAM) {
            a = __ldcs(v); b = __ldcs(v + 1); d = __ldcs(v + 2);
        } else {
            a = __ldg(v); b = __ldg(v + 1); d = __ldg(v + 2);
        }
        ix[0] = a.x; ix[1] = a.y; ix[2] = a.z; ix[3] = a.w;
        ix[4] = b.x; ix[5] = b.y; ix[6] = b.z; ix[7] = b.w;
        ix[8] = d.x; ix[9] = d.y; ix[10] = d.z; ix[11] = d.w;
    } else {
#pragma unroll
        for (int k = 0; k < 12; ++k) ix[k] = (k < 3 * nv) ? __ldg(ib + 3 * o + k) : 0u;
    }
}

// warp claim of the next flat-table chunk (lane 0), broadcast
__device__ __forceinline__ bool claim_flat(const curast_frame_t &f, int lane, int64_t total,
                                           long long &item, long long &lo, long long &hi) {
    long long c = 0;
    if (lane == 0) {
        c = (long long)atomicAdd((unsigned long long *)(f.counters + CURAST_C_CLAIM1), 1ull);
        if (c < total) {
            const int64_t u = upper_index(f.unit_chunk_prefix, f.n_units + 1, c);
            item = __ldg(f.unit_index + u);
            lo = __ldg(f.unit_lo + u) + (c - __ldg(f.unit_chunk_prefix + u)) * f.chunk_tris;
            hi = __ldg(f.unit_hi + u);
            hi = lo + f.chunk_tris < hi ? lo + f.chunk_tris : hi;
        }
    }
    c = __shfl_sync(0xffffffffu, c, 0);
    if (c >= total) return false;
    item = __shfl_sync(0xffffffffu, item, 0);
    lo = __shfl_sync(0xffffffffu, lo, 0);
    hi = __shfl_sync(0xffffffffu, hi, 0);
    return true;
}

// One warp step of k_s1_v2 for a lane pattern KIND (warp-uniform): gather,
// decide, count, queue the undecided triangles with their stored positions.
// The strip kinds keep their 6 stored vertices for the queue entries.
template <int KIND, int PF, int IF>
__device__ __forceinline__ void v2_step(const curast_frame_t &f, const LeanConsts &F,
                                        const ItemGeo<PF, IF> &G, const uint32_t *ix, int nv,
                                        long long tag, float W, float H, float slack, bool tiny,
                                        unsigned &cnt16, QxReserve &R,
                                        unsigned long long *qcount, int lane, unsigned lt_mask) {
    SV<PF> sv[KIND == 0 ? 1 : 6];
    unsigned bits;
    if constexpr (KIND == 0) {
        bits = generic_bits(F, G, ix, W, H, slack, tiny);
    } else {
        PV v[6];
#pragma unroll
        for (int k = 0; k < 6; ++k) sv[k] = sv_load(G, ix[strip_r(KIND, k)]);
#pragma unroll
        for (int k = 0; k < 6; ++k) v[k] = pv_project(F, sv_pos(G, sv[k]));
        bits = strip_bits<KIND>(F, v, W, H, slack, tiny);
    }
    const unsigned vmask = (1u << nv) - 1u;
    const unsigned need = bits & vmask, fr = (bits >> 4) & vmask;
    cnt16 += (unsigned)__popc(fr) + ((unsigned)(nv - __popc(need) - __popc(fr)) << 16);
    unsigned b[4];
    int tot = 0;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        b[t] = __ballot_sync(0xffffffffu, (need >> t) & 1u);
        tot += __popc(b[t]);
    }
    if (!tot) return;
    const QxSlots qs = qx_reserve(R, qcount, tot, lane);
    const long long flag = (bits & 0x100u) ? CURAST_QX_INTERIOR : 0ll;
    int base = 0;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        if ((need >> t) & 1u) {
            const long long slot = qs.at(base + __popc(b[t] & lt_mask));
            if constexpr (KIND == 0) {
                // generic lanes re-read the stored vertices (L1 hits) instead
                // of keeping 12 of them live
                qx_put_sv<PF>(f, slot, sv_load(G, ix[3 * t]), sv_load(G, ix[3 * t + 1]),
                              sv_load(G, ix[3 * t + 2]), (tag + t) | flag);
            } else {
                qx_put_sv<PF>(f, slot, sv[strip_g(KIND, 3 * t)], sv[strip_g(KIND, 3 * t + 1)],
                              sv[strip_g(KIND, 3 * t + 2)], (tag + t) | flag);
            }
        }
        base += __popc(b[t]);
    }
}

template <int MINB, int PF = CURAST_POS_F32, int IF = CURAST_IDX_U32>
__global__ void __launch_bounds__(256, MINB) k_s1_v2(const curast_frame_t f) {
    constexpr int STEP = 128;
    const int lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    unsigned cnt16 = 0;   // frustum | tiny << 16
    const float W = (float)f.width, H = (float)f.height;
    const float slack = (float)(f.width > f.height ? f.width : f.height) * 1.4551915e-11f;
    const bool tiny = f.tiny_cull != 0;
    const int64_t total = __ldg(f.unit_chunk_prefix + f.n_units);
    unsigned long long *qcount = (unsigned long long *)(f.counters + CURAST_C_QX);
    __shared__ QxReserve sres[8];
    QxReserve &R = sres[threadIdx.x >> 5];
    if (lane == 0) R = QxReserve{0u, 0};
    __syncwarp();
    for (;;) {
        long long item = 0, lo = 0, hi = 0;
        if (!claim_flat(f, lane, total, item, lo, hi)) break;
        if (__any_sync(0xffffffffu, cnt16 & 0x80008000u)) {
            unsigned long long cnt[2] = {cnt16 & 0xffffu, cnt16 >> 16};
            flush_stats(f.counters + CURAST_C_S1 + CULL_FRUSTUM, cnt, 1);
            flush_stats(f.counters + CURAST_C_S1 + CULL_TINY, cnt + 1, 1);
            cnt16 = 0;
        }
        const float *frow = f.item_filter + CURAST_FILTER_FLOATS * item;
        ItemGeo<PF, IF> G;
        G.load(f, item);
        const uint32_t *ib = G.idx + 3 * lo;
        const int n = (int)(hi - lo);
        const bool vec = (((uintptr_t)ib) & 15) == 0;
        const long long tag = (item << 40) | lo;
        for (int s0 = 0; s0 < n; s0 += STEP) {
            // the filter block is re-read per step (L1 hits, not hoisted):
            // its 15 registers are then not live across the whole loop
            LeanConsts F;
            lean_load_step(F, frow);
            const int o = s0 + 4 * lane;
            const int nv = max(0, min(4, n - o));
            uint32_t ix[12];
            if constexpr (IF == CURAST_IDX_U32) load_step_indices<true>(ib, o, nv, vec, ix);
            else G.template index_run<12>(3 * (lo + o), 3 * nv, ix);   // bit reader
            if constexpr (IF == CURAST_IDX_U32) {
                // L2 prefetch of the next step's index lines (12 x 128 B,
                // lanes 0-11): the index run is read once, in order, and its
                // load starts each step's dependency chain (index -> vertex
                // gathers -> decisions), so starting it one step early takes
                // an HBM latency off the chain (B: 0.714 -> 0.674 ms stage 1;
                // two steps ahead 0.682, four 0.732; a bulk prefetch of the
                // whole 24 KB chunk run at claim time thrashed L2: 0.784)
                const int sp = s0 + STEP;
                if (lane < 12 && sp < n) {
                    const uintptr_t a = ((uintptr_t)(ib + 3 * sp) & ~(uintptr_t)127) + 128 * lane;
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
                }
            }
            const int kind = strip_kind(ix, nv == 4);
            if (kind == 1)
                v2_step<1>(f, F, G, ix, nv, tag + o, W, H, slack, tiny, cnt16, R, qcount, lane,
                           lt_mask);
            else if (kind == 2)
                v2_step<2>(f, F, G, ix, nv, tag + o, W, H, slack, tiny, cnt16, R, qcount, lane,
                           lt_mask);
            else
                v2_step<0>(f, F, G, ix, nv, tag + o, W, H, slack, tiny, cnt16, R, qcount, lane,
                           lt_mask);
        }
    }
    qx_reserve_close(f, R, lane);
    unsigned long long cnt[2] = {cnt16 & 0xffffu, cnt16 >> 16};
    flush_stats(f.counters + CURAST_C_S1 + CULL_FRUSTUM, cnt, 1);
    flush_stats(f.counters + CURAST_C_S1 + CULL_TINY, cnt + 1, 1);
}

// ------------------------------------------------ instanced (node groups)
// Instanced stage 1 (kernels.py:205-254, pipeline.py:244: the work space is
// the unique triangles of the node groups).  A work unit is a 2048-triangle
// chunk of a group's mesh under a block of CURAST_INST_BLOCK instances: the
// warp copies the block's filter rows to shared memory once, then per
// 128-triangle step loads the indices and gathers the (strip-shared)
// vertices ONCE and runs the projection / lane bound / decisions for every
// instance from registers + shared memory — no global load in the instance
// loop.  Undecided (instance, triangle) pairs go to the fp64 queue with their
// object-space positions and the instance's item in the tag.
template <int KIND, int PF, int IF>
__device__ __forceinline__ void v2i_step(const curast_frame_t &f, const float4 (*sF)[4],
                                         const long long *sItem, int ninst,
                                         const ItemGeo<PF, IF> &G, const uint32_t *ix, int nv,
                                         long long local0, float W, float H, float slack,
                                         bool tiny, unsigned &cnt16, QxReserve &R,
                                         unsigned long long *qcount, int lane,
                                         unsigned lt_mask) {
    const unsigned vmask = (1u << nv) - 1u;
    if constexpr (KIND == 0) {
        // generic lanes: triangle by triangle, every instance per triangle
#pragma unroll 1
        for (int t = 0; t < 4; ++t) {
            const SV<PF> sa = sv_load(G, ix[3 * t]), sb = sv_load(G, ix[3 * t + 1]),
                         sc = sv_load(G, ix[3 * t + 2]);
            const float4 a = sv_pos(G, sa), b = sv_pos(G, sb), c = sv_pos(G, sc);
            const float x[3] = {a.x, b.x, c.x}, y[3] = {a.y, b.y, c.y}, z[3] = {a.z, b.z, c.z};
            const bool valid = (vmask >> t) & 1u;
#pragma unroll 1
            for (int k = 0; k < ninst; ++k) {
                LeanConsts F;
                lean_load_smem(F, sF[k]);
                const unsigned r = lean_bits(F, x, y, z, W, H, slack, tiny);
                const bool need = valid && (r & 1u);
                const bool fr = valid && (r & 2u);
                cnt16 += (unsigned)fr + ((unsigned)(valid && r == 0u) << 16);
                const unsigned bb = __ballot_sync(0xffffffffu, need);
                if (bb) {
                    const QxSlots qs = qx_reserve(R, qcount, __popc(bb), lane);
                    if (need)
                        qx_put_sv<PF>(f, qs.at(__popc(bb & lt_mask)), sa, sb, sc,
                                      (sItem[k] << 40) | (local0 + t));
                }
            }
        }
    } else {
    SV<PF> sv[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) sv[k] = sv_load(G, ix[strip_r(KIND, k)]);
    // the decisions of all instances first (need / frustum bits of
    // instance k in bits 4k..4k+3, interior flag in bit k), then one
    // reservation and the queue writes of the whole step
    // need bits of instances 0-7 / 8-15 in two words (the instance index is
    // warp-uniform, so the half is a uniform branch, not a 64-bit shift);
    // frustum outcomes are only counted
    unsigned need_lo = 0, need_hi = 0, intm = 0;
    int nfr = 0;
#pragma unroll 1
    for (int k = 0; k < ninst; ++k) {
        LeanConsts F;
        lean_load_smem(F, sF[k]);
        PV v[6];
#pragma unroll
        for (int j = 0; j < 6; ++j) v[j] = pv_project(F, sv_pos(G, sv[j]));
        const unsigned bits = strip_bits<KIND, true>(F, v, W, H, slack, tiny);
        if (k < 8) need_lo |= (bits & vmask) << (4 * k);
        else need_hi |= (bits & vmask) << (4 * (k - 8));
        nfr += __popc((bits >> 4) & vmask);
        intm |= ((bits >> 8) & 1u) << k;
    }
    unsigned long long needm = ((unsigned long long)need_hi << 32) | need_lo;
    const int nneed = __popcll(needm);
    cnt16 += (unsigned)nfr + ((unsigned)(nv * ninst - nneed - nfr) << 16);
    // warp prefix sum of the per-lane entry counts
    int incl = nneed;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += u;
    }
    const int tot = __shfl_sync(0xffffffffu, incl, 31);
    if (!tot) return;
    const QxSlots qs = reserve_slots(R, qcount, tot, lane);
    int i = incl - nneed;
    while (needm) {
        const int bit = __ffsll((long long)needm) - 1;
        needm &= needm - 1;
        const int k = bit >> 2, t = bit & 3;
        const long long tag = ((sItem[k] << 40) | (local0 + t)) |
                              (((intm >> k) & 1u) ? CURAST_QX_INTERIOR : 0ll);
        const long long slot = qs.at(i++);
        switch (t) {
        case 0: qx_put_sv<PF>(f, slot, sv[strip_g(KIND, 0)], sv[strip_g(KIND, 1)],
                              sv[strip_g(KIND, 2)], tag); break;
        case 1: qx_put_sv<PF>(f, slot, sv[strip_g(KIND, 3)], sv[strip_g(KIND, 4)],
                              sv[strip_g(KIND, 5)], tag); break;
        case 2: qx_put_sv<PF>(f, slot, sv[strip_g(KIND, 6)], sv[strip_g(KIND, 7)],
                              sv[strip_g(KIND, 8)], tag); break;
        default: qx_put_sv<PF>(f, slot, sv[strip_g(KIND, 9)], sv[strip_g(KIND, 10)],
                               sv[strip_g(KIND, 11)], tag); break;
        }
    }
    }
}

template <int MINB, int PF = CURAST_POS_F32, int IF = CURAST_IDX_U32>
__global__ void __launch_bounds__(256, MINB) k_s1i_v2(const curast_frame_t f) {
    constexpr int STEP = 128;
    __shared__ float4 sF[8][CURAST_INST_BLOCK][4];
    __shared__ long long sItem[8][CURAST_INST_BLOCK];
    __shared__ QxReserve sres[8];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned lt_mask = (1u << lane) - 1u;
    unsigned cnt16 = 0;
    const float W = (float)f.width, H = (float)f.height;
    const float slack = (float)(f.width > f.height ? f.width : f.height) * 1.4551915e-11f;
    const bool tiny = f.tiny_cull != 0;
    const int64_t CHUNK = f.inst_chunk_tris;
    const int64_t total = __ldg(f.inst_unit_chunk_prefix + f.n_inst_units);
    unsigned long long *qcount = (unsigned long long *)(f.counters + CURAST_C_QX);
    QxReserve &R = sres[w];
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
        if (__any_sync(0xffffffffu, cnt16 & 0x80008000u)) {
            unsigned long long cnt[2] = {cnt16 & 0xffffu, cnt16 >> 16};
            flush_stats(f.counters + CURAST_C_S1 + CULL_FRUSTUM, cnt, 1);
            flush_stats(f.counters + CURAST_C_S1 + CULL_TINY, cnt + 1, 1);
            cnt16 = 0;
        }
        // unit = group | first instance << 32 (CURAST_INST_BLOCK instances)
        const int64_t k0 = g >> 32;
        g &= 0xFFFFFFFFll;
        const int64_t ioff = __ldg(f.group_item_off + g);
        const int ninst = (int)(min(__ldg(f.group_item_count + g), k0 + CURAST_INST_BLOCK) - k0);
        // the block's instances: items and filter rows into shared memory
        __syncwarp();
        if (lane < ninst) sItem[w][lane] = __ldg(f.group_items + ioff + k0 + lane);
        __syncwarp();
        for (int j = lane; j < 4 * ninst; j += 32)
            sF[w][j >> 2][j & 3] =
                __ldg((const float4 *)(f.item_filter + CURAST_FILTER_FLOATS * sItem[w][j >> 2]) +
                      (j & 3));
        __syncwarp();
        ItemGeo<PF, IF> G;
        G.load(f, sItem[w][0]);
        const uint32_t *ib = G.idx + 3 * lo;
        const int n = (int)(hi - lo);
        const bool vec = (((uintptr_t)ib) & 15) == 0;
        for (int s0 = 0; s0 < n; s0 += STEP) {
            const int o = s0 + 4 * lane;
            const int nv = max(0, min(4, n - o));
            uint32_t ix[12];
            if constexpr (IF == CURAST_IDX_U32) load_step_indices(ib, o, nv, vec, ix);
            else G.template index_run<12>(3 * (lo + o), 3 * nv, ix);   // bit reader
            const int kind = strip_kind(ix, nv == 4);
            if (kind == 1)
                v2i_step<1>(f, sF[w], sItem[w], ninst, G, ix, nv, lo + o, W, H, slack, tiny,
                            cnt16, R, qcount, lane, lt_mask);
            else if (kind == 2)
                v2i_step<2>(f, sF[w], sItem[w], ninst, G, ix, nv, lo + o, W, H, slack, tiny,
                            cnt16, R, qcount, lane, lt_mask);
            else
                v2i_step<0>(f, sF[w], sItem[w], ninst, G, ix, nv, lo + o, W, H, slack, tiny,
                            cnt16, R, qcount, lane, lt_mask);
        }
    }
    qx_reserve_close(f, R, lane);
    unsigned long long cnt[2] = {cnt16 & 0xffffu, cnt16 >> 16};
    flush_stats(f.counters + CURAST_C_S1 + CULL_FRUSTUM, cnt, 1);
    flush_stats(f.counters + CURAST_C_S1 + CULL_TINY, cnt + 1, 1);
}

}  // namespace curast
