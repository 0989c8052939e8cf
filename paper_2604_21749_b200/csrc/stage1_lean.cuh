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

// Fast-path decision for a triangle of a chunk proven (chunk_class) to lie
// entirely in front of the near margin and inside the viewport: only the
// tiny cull (with its nonzero-extent precondition) is left to decide, with
// eps = M K1 + K0 the filter bound under the chunk's lower depth bound.
// Returns 1 when the fp64 pass is needed.
__device__ __forceinline__ unsigned lean_fast_bits(const LeanConsts &F, const float *x,
                                                   const float *y, const float *z, float K0,
                                                   float K1) {
    float2 P[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const float D = __fmaf_rn(F.dz, z[k], __fmaf_rn(F.dy, y[k], __fmaf_rn(F.dx, x[k], F.d3)));
        float2 t = __ffma2_rn(F.cx, make_float2(x[k], x[k]), F.c3);
        t = __ffma2_rn(F.cy, make_float2(y[k], y[k]), t);
        t = __ffma2_rn(F.cz, make_float2(z[k], z[k]), t);
        const float r = rcp_approx(D);
        P[k] = __fmul2_rn(t, make_float2(r, r));
    }
    const float mnx = fminf(P[0].x, fminf(P[1].x, P[2].x));
    const float mxx = fmaxf(P[0].x, fmaxf(P[1].x, P[2].x));
    const float mny = fminf(P[0].y, fminf(P[1].y, P[2].y));
    const float mxy = fmaxf(P[0].y, fmaxf(P[1].y, P[2].y));
    // every coordinate is positive inside the viewport: M = max(mxx, mxy)
    const float eps = __fmaf_rn(fmaxf(mxx, mxy), K1, K0);
    const float e2 = eps + eps, lo5 = eps + 0.5f, hi5 = eps - 0.5f;
    const bool ext = (mxx - mnx > e2) && (mxy - mny > e2);
    const bool tx = ceilf(mnx - lo5) > mxx + hi5;
    const bool ty = ceilf(mny - lo5) > mxy + hi5;
    return (ext && (tx || ty)) ? 0u : 1u;
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

struct LeanCtx {
    float W, H, slack;
    bool tiny;
    int lane;
    unsigned lt_mask;
    unsigned long long *qcount;
};

__device__ __forceinline__ LeanCtx lean_ctx(const curast_frame_t &f) {
    LeanCtx C;
    C.W = (float)f.width;
    C.H = (float)f.height;
    C.slack = (float)(f.width > f.height ? f.width : f.height) * 1.4551915e-11f;
    C.tiny = f.tiny_cull != 0;
    C.lane = threadIdx.x & 31;
    C.lt_mask = (1u << C.lane) - 1u;
    C.qcount = (unsigned long long *)(f.counters + CURAST_C_QX);
    return C;
}

// Chunk class for the fast path: the 8 corners of the chunk's object box
// (two boxes when a sharded chunk straddles a box boundary; lanes 0-15)
// projected with their own filter bounds.  fast = every corner d' exceeds
// near_hi by 2 E_d (so every vertex d' does) and every corner's pixel
// interval lies inside (0, W) x (0, H) (px is linear-fractional in the
// object position, so the box's image lies within its corners' hull).
// Then dl = min d'_corner - 2 E_d bounds every vertex d' from below and the
// triangle bound is eps = 1.5 (E_xy + M E_d) / dl + 2^-21 M + slack.
__device__ __forceinline__ bool chunk_class(const curast_frame_t &f, const LeanConsts &F,
                                            const LeanCtx &C, long long item, long long lo,
                                            long long hi, float &K0, float &K1) {
    if (!f.chunk_box || !C.tiny) return false;
    const int64_t cb = __ldg(f.item_cb_off + item);
    const long long b = (C.lane < 8 ? lo : hi - 1) / kS1Chunk;
    const float4 *box = (const float4 *)(f.chunk_box + 8 * (cb + b));
    const float4 mn = __ldg(box), mx = __ldg(box + 1);
    const int c = C.lane & 7;
    const float x = (c & 1) ? mx.x : mn.x, y = (c & 2) ? mx.y : mn.y, z = (c & 4) ? mx.z : mn.z;
    const float D = __fmaf_rn(F.dz, z, __fmaf_rn(F.dy, y, __fmaf_rn(F.dx, x, F.d3)));
    float2 t = __ffma2_rn(F.cx, make_float2(x, x), F.c3);
    t = __ffma2_rn(F.cy, make_float2(y, y), t);
    t = __ffma2_rn(F.cz, make_float2(z, z), t);
    const float r = rcp_approx(D);
    const float2 P = __fmul2_rn(t, make_float2(r, r));
    const float M = fmaxf(fabsf(P.x), fabsf(P.y));
    float eps = __fmaf_rn(M, F.ed, F.exy) * r;
    eps = __fmaf_rn(eps, 1.5f, __fmaf_rn(M, kRelSlack, C.slack));
    const bool ok = C.lane >= 16 ||
                    (D - 2.0f * F.ed > F.near_hi && P.x - eps > 0.0f && P.y - eps > 0.0f &&
                     P.x + eps < C.W && P.y + eps < C.H);
    if (!__all_sync(0xffffffffu, ok)) return false;
    float dl = C.lane < 16 ? D : __int_as_float(0x7f800000);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dl = fminf(dl, __shfl_xor_sync(0xffffffffu, dl, o));
    dl -= 2.0f * F.ed;
    const float rd = rcp_approx(dl) * 1.0000010f;     // covers the folding roundings
    K1 = __fmaf_rn(1.5f * F.ed, rd, kRelSlack);
    K0 = __fmaf_rn(1.5f * F.exy, rd, C.slack);
    return true;
}

// Triangles [0, n) of an index range (ib = first triangle's indices, tag =
// item << 40 | its local index): lane l owns TPL consecutive triangles per
// 32*TPL step, 128-bit index loads when aligned, 3*TPL independent vertex
// gathers issued before the math.  Warp-uniform n.
// ILV: lane -> triangle map of a step.  0: lane l owns TPL consecutive
// triangles (3 x 128-bit index loads); 1: lane l owns l, l+32, ... (scalar
// index loads; each vertex gather of the warp then reads consecutive
// triangles' vertices: fewer L1 lines per gather); 2: as 1, the indices
// loaded as in 0 and transposed through shared memory (sidx: 32*3*TPL words
// per warp).
// PROBE (timing experiments only, wrong output): 1 = loads only.
template <int TPL, int PROBE = 0, int ILV = 0, bool FAST = false>
__device__ __forceinline__ void lean_range(const curast_frame_t &f, const LeanConsts &F,
                                           const LeanCtx &C, const float4 *__restrict__ pb,
                                           const uint32_t *__restrict__ ib, int n, long long tag,
                                           unsigned &n_frustum, unsigned &n_tiny,
                                           uint32_t *sidx = nullptr, float K0 = 0.0f,
                                           float K1 = 0.0f) {
    constexpr int STEP = 32 * TPL;
    constexpr int DT = ILV ? 32 : 1;
    const bool vec = (((uintptr_t)ib) & 15) == 0;
    for (int s0 = 0; s0 < n; s0 += STEP) {
        const int o = ILV ? s0 + C.lane : s0 + TPL * C.lane;
        unsigned valid;
        if (ILV) {
            valid = 0;
#pragma unroll
            for (int t = 0; t < TPL; ++t) valid |= (unsigned)(o + DT * t < n) << t;
        } else {
            const int nv = max(0, min(TPL, n - o));
            valid = (1u << nv) - 1u;
        }
        uint32_t ix[3 * TPL];
        if (ILV == 2 && TPL == 4 && vec && s0 + STEP <= n) {
            const uint4 *v = (const uint4 *)(ib + 3 * s0) + 3 * C.lane;
            uint4 *w = (uint4 *)sidx + 3 * C.lane;
            w[0] = __ldg(v);
            w[1] = __ldg(v + 1);
            w[2] = __ldg(v + 2);
            __syncwarp();
#pragma unroll
            for (int t = 0; t < TPL; ++t)
#pragma unroll
                for (int k = 0; k < 3; ++k) ix[3 * t + k] = sidx[3 * (C.lane + 32 * t) + k];
            __syncwarp();
        } else if (ILV == 0 && TPL == 4 && vec && valid == 15u) {
            const uint4 *v = (const uint4 *)(ib + 3 * o);
            const uint4 a = __ldg(v), b = __ldg(v + 1), d = __ldg(v + 2);
            ix[0] = a.x; ix[1] = a.y; ix[2] = a.z; ix[3] = a.w;
            ix[4] = b.x; ix[5] = b.y; ix[6] = b.z; ix[7] = b.w;
            ix[8] = d.x; ix[9] = d.y; ix[10] = d.z; ix[11] = d.w;
        } else if (ILV == 0) {
            const int lim = 3 * __popc(valid);
#pragma unroll
            for (int k = 0; k < 3 * TPL; ++k) ix[k] = k < lim ? __ldg(ib + 3 * o + k) : 0u;
        } else {
#pragma unroll
            for (int t = 0; t < TPL; ++t)
#pragma unroll
                for (int k = 0; k < 3; ++k)
                    ix[3 * t + k] = ((valid >> t) & 1u) ? __ldg(ib + 3 * (o + DT * t) + k) : 0u;
        }
        float px[3 * TPL], py[3 * TPL], pz[3 * TPL];
#pragma unroll
        for (int k = 0; k < 3 * TPL; ++k) {
            const float4 q = __ldg(pb + ix[k]);
            px[k] = q.x;
            py[k] = q.y;
            pz[k] = q.z;
        }
        if (PROBE == 1) {
            float acc = 0.0f;
#pragma unroll
            for (int k = 0; k < 3 * TPL; ++k) acc += px[k] + py[k] + pz[k];
            n_tiny += acc == 12345.0f;
            continue;
        }
        unsigned need = 0, fr = 0;
#pragma unroll
        for (int t = 0; t < TPL; ++t) {
            const unsigned bits =
                FAST ? lean_fast_bits(F, px + 3 * t, py + 3 * t, pz + 3 * t, K0, K1)
                     : lean_bits(F, px + 3 * t, py + 3 * t, pz + 3 * t, C.W, C.H, C.slack, C.tiny);
            if ((valid >> t) & 1u) {
                need |= (bits & 1u) << t;
                fr |= (bits >> 1) << t;
            }
        }
        n_frustum += __popc(fr);
        n_tiny += __popc(valid) - __popc(need) - __popc(fr);
        unsigned b[TPL];
        int tot = 0;
#pragma unroll
        for (int t = 0; t < TPL; ++t) {
            b[t] = __ballot_sync(0xffffffffu, (need >> t) & 1u);
            tot += __popc(b[t]);
        }
        if (tot) {
            unsigned long long base = 0;
            if (C.lane == 0) base = atomicAdd(C.qcount, (unsigned long long)tot);
            base = __shfl_sync(0xffffffffu, base, 0);
#pragma unroll
            for (int t = 0; t < TPL; ++t) {
                // positions travel with the entry: the fp64 kernel does not
                // re-gather them from HBM
                if ((need >> t) & 1u)
                    qx_write(f, (long long)base + __popc(b[t] & C.lt_mask), px + 3 * t, py + 3 * t,
                             pz + 3 * t, tag + o + DT * t);
                base += __popc(b[t]);
            }
        }
    }
}

// claims chunk c of the flat table through counters[claim_slot]; -1 when done
__device__ __forceinline__ bool lean_claim(const curast_frame_t &f, int lane, int64_t cbeg,
                                           int64_t total, int claim_slot, long long &item,
                                           long long &lo, long long &hi) {
    constexpr int CHUNK = kS1Chunk;
    long long c = 0;
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
    if (c >= total) return false;
    item = __shfl_sync(0xffffffffu, item, 0);
    lo = __shfl_sync(0xffffffffu, lo, 0);
    hi = __shfl_sync(0xffffffffu, hi, 0);
    return true;
}

// Per-triangle lean kernel over the flat table: chunks [cbeg, min(cend,
// total)) claimed through counters[claim_slot] (slices of one frame use
// distinct slots).
template <int PF, int MINB, int TPL, int PROBE = 0, int ILV = 0>
__global__ void __launch_bounds__(256, MINB) k_s1_lean(const curast_frame_t f, int64_t cbeg,
                                                        int64_t cend, int claim_slot) {
    __shared__ uint32_t sidx[ILV == 2 ? 8 : 1][ILV == 2 ? 3 * 32 * TPL : 1];
    const LeanCtx C = lean_ctx(f);
    unsigned n_frustum = 0, n_tiny = 0;
    const int64_t total = min(cend, __ldg(f.unit_chunk_prefix + f.n_units));
    for (;;) {
        long long item = 0, lo = 0, hi = 0;
        if (!lean_claim(f, C.lane, cbeg, total, claim_slot, item, lo, hi)) break;
        LeanConsts F;
        lean_load(F, f.item_filter + CURAST_FILTER_FLOATS * item);
        // float4 positions: one 128-bit gather per vertex
        const float4 *pb = (const float4 *)f.positions + __ldg(f.item_vtx_off + item);
        const uint32_t *ib = (const uint32_t *)f.indices + __ldg(f.item_idx_off + item) + 3 * lo;
        // (the chunk-class fast path, chunk_class + FAST, measured slower
        // here: this kernel is bound by L1 wavefronts, not instructions, and
        // the second inlined copy spills)
        lean_range<TPL, PROBE, ILV>(f, F, C, pb, ib, (int)(hi - lo), (item << 40) | lo, n_frustum,
                                    n_tiny, sidx[ILV == 2 ? (threadIdx.x >> 5) : 0]);
    }
    unsigned long long cnt[2] = {n_frustum, n_tiny};
    flush_stats(f.counters + CURAST_C_S1 + CULL_FRUSTUM, cnt, 1);
    flush_stats(f.counters + CURAST_C_S1 + CULL_TINY, cnt + 1, 1);
}

// Per-triangle lean kernel, written out flat (the default): the
// lean_range-based k_s1_lean below carries the experiment switches and
// costs 5% more instructions and some spills (measured r01: 418 M vs 398 M
// warp instructions on config B).
// adds the packed (frustum | tiny << 16) lane counts to the frame counters
__device__ __forceinline__ void lean_flush16(const curast_frame_t &f, unsigned c) {
    unsigned long long cnt[2] = {c & 0xffffu, c >> 16};
    flush_stats(f.counters + CURAST_C_S1 + CULL_FRUSTUM, cnt, 1);
    flush_stats(f.counters + CURAST_C_S1 + CULL_TINY, cnt + 1, 1);
}

// PFI: L1 prefetch of the next step's index lines (switch only).  STRIP:
// the quad-strip vertex-reuse gathers below (the default instantiation:
// config B stage-1 filter 526 vs 544 us without).  Before the per-warp queue
// reservation both were bimodal across processes (0.77 / 1.10 ms stage 1):
// the same-address queue atomics were the floor, see qx_reserve.
// DIE: two claim sequences, one per half of the SM ids (the two dies of a
// B200): SMs of the lower half walk the chunks of the first half of the
// table, the upper half the second, and a half that runs out continues in
// the other's sequence.  Neighbouring chunks (which share vertex rows) then
// stay on one die's L2.
template <int PF, int MINB, int TPL, bool PFI = false, bool STRIP = false, bool DIE = false>
__global__ void __launch_bounds__(256, MINB) k_s1_lean_flat(const curast_frame_t f, int64_t cbeg,
                                                        int64_t cend, int claim_slot) {
    // processes chunks [cbeg, min(cend, total)) of the flat table, claimed
    // through counters[claim_slot] (slices of one frame use distinct slots)
    constexpr int CHUNK = kS1Chunk, STEP = 32 * TPL;
    const int lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    // frustum / tiny counts as two 16-bit fields of one register (one
    // register less than two counters: the loop runs at the 64-register cap);
    // flushed before a field can pass 2^15 (<= 64 per lane per chunk)
    unsigned cnt16 = 0;
    const float W = (float)f.width, H = (float)f.height;
    const float slack = (float)(f.width > f.height ? f.width : f.height) * 1.4551915e-11f;
    const bool tiny = f.tiny_cull != 0;
    const int64_t total = min(cend, __ldg(f.unit_chunk_prefix + f.n_units));
    unsigned long long *qcount = (unsigned long long *)(f.counters + CURAST_C_QX);
    // lane 0's reservation state lives in shared memory: the filter loop is
    // at the 64-register cap (two more live registers spill)
    __shared__ QxReserve sres[8];
    QxReserve &R = sres[threadIdx.x >> 5];
    if (lane == 0) R = QxReserve{0u, 0};
    __syncwarp();

    for (;;) {
        long long c = 0, item = 0, lo = 0, hi = 0;
        if (lane == 0) {
            if (DIE) {
                unsigned smid, nsmid;
                asm("mov.u32 %0, %%smid;" : "=r"(smid));
                asm("mov.u32 %0, %%nsmid;" : "=r"(nsmid));
                int h = smid >= nsmid / 2 ? 1 : 0;
                const long long mid = cbeg + (total - cbeg) / 2;
                c = total;
                for (int tries = 0; tries < 2; ++tries, h ^= 1) {
                    const long long b0 = h ? mid : cbeg, e0 = h ? total : mid;
                    const long long cc = b0 + (long long)atomicAdd(
                        (unsigned long long *)(f.counters + (h ? CURAST_C_CLAIM1B : claim_slot)), 1ull);
                    if (cc < e0) { c = cc; break; }
                }
            } else {
                c = cbeg + (long long)atomicAdd((unsigned long long *)(f.counters + claim_slot), 1ull);
            }
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

        if (__any_sync(0xffffffffu, cnt16 & 0x80008000u)) {
            lean_flush16(f, cnt16);
            cnt16 = 0;
        }
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
            if (PFI && s0 + STEP < n) {
                // the next step's index lines into L1 (12 x 128 B per warp)
                const uintptr_t b1 = ((uintptr_t)(ib + 3 * (s0 + STEP))) & ~(uintptr_t)127;
                const uintptr_t e1 = (uintptr_t)(ib + 3 * min(n, s0 + 2 * STEP));
                if (b1 + 128 * lane < e1)
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(b1 + 128 * lane));
            }
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
            // Quad-strip vertex reuse: a lane's 4 consecutive triangles are 2
            // quads of a strip in the two standard triangulations — (a,c,b),
            // (b,c,d) (make_tessellated_quad) and (a,b,c),(b,d,c)
            // (make_sphere) — so 6 of its 12 vertex refs repeat earlier ones.
            // Every lane checks the pattern on its own indices; only when the
            // whole warp matches are the 6 repeated gathers skipped (their
            // values are the repeated registers), else all 12 are loaded.
            int strip = 0;
            if (STRIP && TPL == 4) {
                const bool full = nv == TPL;
                const bool gq = full && ix[3] == ix[2] && ix[4] == ix[1] && ix[6] == ix[2] &&
                                ix[7] == ix[5] && ix[9] == ix[8] && ix[10] == ix[5];
                const bool sq = full && ix[3] == ix[1] && ix[5] == ix[2] && ix[6] == ix[1] &&
                                ix[8] == ix[4] && ix[9] == ix[7] && ix[11] == ix[4];
                strip = __all_sync(0xffffffffu, gq) ? 1 : (__all_sync(0xffffffffu, sq) ? 2 : 0);
            }
            auto gather = [&](int k) {
                const float4 q = __ldg(pb + ix[k]);
                px[k] = q.x;
                py[k] = q.y;
                pz[k] = q.z;
            };
            auto copy = [&](int k, int from) {
                px[k] = px[from];
                py[k] = py[from];
                pz[k] = pz[from];
            };
            if (TPL == 4 && strip == 1) {
                gather(0); gather(1); gather(2); gather(5); gather(8); gather(11);
                copy(3, 2); copy(4, 1); copy(6, 2); copy(7, 5); copy(9, 8); copy(10, 5);
            } else if (TPL == 4 && strip == 2) {
                gather(0); gather(1); gather(2); gather(4); gather(7); gather(10);
                copy(3, 1); copy(5, 2); copy(6, 1); copy(8, 4); copy(9, 7); copy(11, 4);
            } else {
#pragma unroll
                for (int k = 0; k < 3 * TPL; ++k) gather(k);
            }
            unsigned need = 0, fr = 0;
            unsigned bt[TPL];
#pragma unroll
            for (int t = 0; t < TPL; ++t)
                bt[t] = lean_bits(F, px + 3 * t, py + 3 * t, pz + 3 * t, W, H, slack, tiny);
#pragma unroll
            for (int t = 0; t < TPL; ++t) {
                if (t < nv) {
                    need |= (bt[t] & 1u) << t;
                    fr |= (bt[t] >> 1) << t;
                }
            }
            cnt16 += (unsigned)__popc(fr) + ((unsigned)(nv - __popc(need) - __popc(fr)) << 16);
            unsigned b[TPL];
            int tot = 0;
#pragma unroll
            for (int t = 0; t < TPL; ++t) {
                b[t] = __ballot_sync(0xffffffffu, (need >> t) & 1u);
                tot += __popc(b[t]);
            }
            if (tot) {
                const QxSlots qs = qx_reserve(R, qcount, tot, lane);
                int base = 0;
#pragma unroll
                for (int t = 0; t < TPL; ++t) {
                    if ((need >> t) & 1u) {
                        const long long slot = qs.at(base + __popc(b[t] & lt_mask));
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
    qx_reserve_close(f, R, lane);
    lean_flush16(f, cnt16);
}

// Per-triangle lean kernel over the lane-major index steps (indices_ilv):
// the same per-triangle work as k_s1_lean_flat, but lane l owns triangles
// l, l+32, l+64, l+96 of a 126-triangle step, so each of the 12 vertex
// gathers of a warp reads the vertices of 32 consecutive triangles — about
// half the L1 lines (the filter is bound by L1 data-pipe wavefronts).
template <int MINB>
__global__ void __launch_bounds__(256, MINB) k_s1_lean_ilv(const curast_frame_t f, int64_t cbeg,
                                                           int64_t cend, int claim_slot) {
    constexpr int CHUNK = kS1Chunk, MT = CURAST_MESHLET_TRIS, SW = 384;
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

// Meshlet lean kernel (flat table, meshes with meshlets; CURAST_MESHLETS=1).
// Per batch of triangles a warp
//   1. gathers and projects each listed vertex once (lanes j, j+32, ...; the
//      ids are ascending, so the gathers are nearly contiguous) and keeps
//      p' = (px', py') in shared memory (8 B per vertex, one pad slot per 16
//      so that the strip pattern of lookups is bank-conflict free);
//   2. decides its triangles from 3 local indices each.  In a chunk of
//      class "fast" (chunk_class: in front of the near margin, inside the
//      viewport) only tiny + extent are tested, with the chunk bound
//      eps = M K1 + K0.  Otherwise the batch reduces d'_min and max |p'|
//      into one bound for all its triangles (the filter bound grows with
//      |p'| and 1/d') and runs the full lean_decide.
// A regular batch is one meshlet (126 triangles, <= 240 unique vertices, u8
// slot numbers, 4 triangles per lane).  A meshlet with more vertices runs
// as two RAW batches of 63 triangles whose vertex list is the index stream
// itself (189 entries, local index 3t + e).  Undecided triangles re-gather
// their 3 object positions (L1-hot) into the fp64 queue.
constexpr int MESH_WARPS = 8;
constexpr int MESH_SLOTS = 256;   // >= CURAST_MESHLET_MAX_VERTS + its pad slots
static_assert(CURAST_MESHLET_MAX_VERTS + CURAST_MESHLET_MAX_VERTS / 16 <= MESH_SLOTS, "slots");

__device__ __forceinline__ int mesh_slot(int j) { return j + (j >> 4); }

__device__ __forceinline__ int byte_of(const uint32_t *w, int b) {
    return (int)__byte_perm(w[b >> 2], 0u, 0x4440u | (unsigned)(b & 3));
}

template <bool RAW>
__device__ __forceinline__ void mesh_batch(const curast_frame_t &f, const LeanConsts &F,
                                           const LeanCtx &C, float2 (*sP)[MESH_SLOTS], int warp,
                                           const float4 *__restrict__ pb,
                                           const uint32_t *__restrict__ vsrc, int nu,
                                           const uint32_t *__restrict__ ltri, int rb,
                                           int rlo, int rhi, long long tagb, bool fast,
                                           float K0, float K1, unsigned &n_frustum,
                                           unsigned &n_tiny) {
    // triangles of this batch: chunk-relative [rb, rb + 32*TPL) ∩ [rlo, rhi)
    constexpr int TPL = RAW ? 2 : 4;
    const int lane = C.lane;
    // 1. listed vertices: id loads, then gathers, then math
    float dmin = __int_as_float(0x7f800000), M = 0.0f;
    for (int g = 0; g < nu; g += 128) {
        uint32_t vid[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int j = g + lane + 32 * r;
            vid[r] = j < nu ? __ldg(vsrc + j) : 0u;
        }
        float4 q[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) q[r] = __ldg(pb + vid[r]);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int j = g + lane + 32 * r;
            const float D = __fmaf_rn(F.dz, q[r].z, __fmaf_rn(F.dy, q[r].y, __fmaf_rn(F.dx, q[r].x, F.d3)));
            float2 t = __ffma2_rn(F.cx, make_float2(q[r].x, q[r].x), F.c3);
            t = __ffma2_rn(F.cy, make_float2(q[r].y, q[r].y), t);
            t = __ffma2_rn(F.cz, make_float2(q[r].z, q[r].z), t);
            const float rr = rcp_approx(D);
            const float2 P = __fmul2_rn(t, make_float2(rr, rr));
            if (j < nu) {
                sP[warp][mesh_slot(j)] = P;
                dmin = fminf(dmin, D);
                M = fmaxf(M, fmaxf(fabsf(P.x), fabsf(P.y)));
            }
        }
    }
    float eps = 0.0f;
    bool near_ok = true;
    if (!fast) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            dmin = fminf(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
            M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
        }
        near_ok = dmin > F.near_hi;
        eps = __fmaf_rn(M, F.ed, F.exy) * rcp_approx(dmin);
        eps = __fmaf_rn(eps, 1.5f, __fmaf_rn(M, kRelSlack, C.slack));
    }
    __syncwarp();
    // 2. triangles rb + TPL*lane + k; slot numbers from the u8 record (RAW:
    //    list entry 3t + e, slot computed)
    uint32_t w[3] = {0u, 0u, 0u};
    if (!RAW) {
        const uint32_t *tw = ltri + 3 * lane;
        w[0] = __ldg(tw);
        w[1] = __ldg(tw + 1);
        w[2] = __ldg(tw + 2);
    }
    auto slot = [&](int k, int e) -> int {
        return RAW ? mesh_slot(3 * (TPL * lane + k) + e) : byte_of(w, 3 * k + e);
    };
    const int tb = rb + TPL * lane;
    // valid triangles of this lane: k in [rlo - tb, rhi - tb)
    const int vlo = max(0, min(TPL, rlo - tb)), vhi = max(0, min(TPL, rhi - tb));
    const unsigned valid = ((1u << vhi) - 1u) & ~((1u << vlo) - 1u);
    unsigned keep = 0, fr = 0;          // keep: decided (tiny or frustum)
#pragma unroll
    for (int k = 0; k < TPL; ++k) {
        const float2 A = sP[warp][slot(k, 0)], B = sP[warp][slot(k, 1)], Q = sP[warp][slot(k, 2)];
        const float mnx = fminf(A.x, fminf(B.x, Q.x)), mxx = fmaxf(A.x, fmaxf(B.x, Q.x));
        const float mny = fminf(A.y, fminf(B.y, Q.y)), mxy = fmaxf(A.y, fmaxf(B.y, Q.y));
        if (fast) {
            const float e = __fmaf_rn(fmaxf(mxx, mxy), K1, K0);
            const float e2 = e + e, lo5 = e + 0.5f, hi5 = e - 0.5f;
            const bool ext = (mxx - mnx > e2) && (mxy - mny > e2);
            const bool tx = ceilf(mnx - lo5) > mxx + hi5;
            const bool ty = ceilf(mny - lo5) > mxy + hi5;
            keep |= (unsigned)(ext && (tx || ty)) << k;
        } else {
            const unsigned bits = lean_decide(mnx, mxx, mny, mxy, eps, near_ok, C.W, C.H, C.tiny);
            keep |= (~bits & 1u) << k;
            fr |= (bits >> 1) << k;
        }
    }
    fr &= valid;
    const unsigned need = valid & ~keep;
    n_frustum += __popc(fr);
    n_tiny += __popc(valid) - __popc(need) - __popc(fr);
    unsigned bq[TPL];
    int tot = 0;
#pragma unroll
    for (int k = 0; k < TPL; ++k) {
        bq[k] = __ballot_sync(0xffffffffu, (need >> k) & 1u);
        tot += __popc(bq[k]);
    }
    if (tot) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(C.qcount, (unsigned long long)tot);
        base = __shfl_sync(0xffffffffu, base, 0);
#pragma unroll
        for (int k = 0; k < TPL; ++k) {
            if ((need >> k) & 1u) {
                float x[3], y[3], z[3];
#pragma unroll
                for (int e = 0; e < 3; ++e) {
                    const int sl = slot(k, e);
                    const float4 q = __ldg(pb + __ldg(vsrc + (sl - sl / 17)));   // slot -> entry
                    x[e] = q.x;
                    y[e] = q.y;
                    z[e] = q.z;
                }
                qx_write(f, (long long)base + __popc(bq[k] & C.lt_mask), x, y, z, tagb + tb + k);
            }
            base += __popc(bq[k]);
        }
    }
    __syncwarp();
}

template <int MINB>
__global__ void __launch_bounds__(32 * MESH_WARPS, MINB) k_s1_mesh(const curast_frame_t f,
                                                                    int64_t cbeg, int64_t cend,
                                                                    int claim_slot) {
    constexpr int MT = CURAST_MESHLET_TRIS, MV = CURAST_MESHLET_MAX_VERTS;
    constexpr int MB = CURAST_MESHLET_BYTES;
    static_assert(MV >= 3 * ((MT + 1) / 2), "RAW half-meshlet batches need their vertex slots");
    static_assert(MB >= 12 * 32, "4 triangles x 3 bytes per lane");
    __shared__ float2 sP[MESH_WARPS][MESH_SLOTS];
    const int warp = threadIdx.x >> 5;
    const LeanCtx C = lean_ctx(f);
    unsigned n_frustum = 0, n_tiny = 0;
    const int64_t total = min(cend, __ldg(f.unit_chunk_prefix + f.n_units));
    for (;;) {
        long long item = 0, lo = 0, hi = 0;
        if (!lean_claim(f, C.lane, cbeg, total, claim_slot, item, lo, hi)) break;
        LeanConsts F;
        lean_load(F, f.item_filter + CURAST_FILTER_FLOATS * item);
        float K0 = 0.0f, K1 = 0.0f;
        const bool fast = chunk_class(f, F, C, item, lo, hi, K0, K1);
        const float4 *pb = (const float4 *)f.positions + __ldg(f.item_vtx_off + item);
        // chunk-relative 32-bit indexing from the first meshlet it touches
        const long long m0 = lo / MT, base = m0 * MT;
        const int rlo = (int)(lo - base), rhi = (int)(hi - base);
        const int64_t gm0 = __ldg(f.item_ml_off + item) + m0;
        const int64_t *voff = f.ml_voff + gm0;
        const uint32_t *trib = (const uint32_t *)(f.ml_tris + gm0 * MB);
        const uint32_t *ib = (const uint32_t *)f.indices + __ldg(f.item_idx_off + item) + 3 * base;
        const long long tagb = (item << 40) | base;
        const int nml = (rhi + MT - 1) / MT;
        for (int m = 0; m < nml; ++m) {
            const int64_t vb = __ldg(voff + m);
            const int nu = (int)(__ldg(voff + m + 1) - vb);
            if (nu <= MV) {
                mesh_batch<false>(f, F, C, sP, warp, pb, f.ml_verts + vb, nu, trib + m * (MB / 4),
                                  m * MT, rlo, min(rhi, m * MT + MT), tagb, fast, K0, K1,
                                  n_frustum, n_tiny);
            } else {
                constexpr int H1 = (MT + 1) / 2;
                mesh_batch<true>(f, F, C, sP, warp, pb, ib + 3 * m * MT, 3 * H1, nullptr, m * MT,
                                 rlo, min(rhi, m * MT + H1), tagb, fast, K0, K1, n_frustum,
                                 n_tiny);
                mesh_batch<true>(f, F, C, sP, warp, pb, ib + 3 * (m * MT + H1), 3 * (MT - H1),
                                 nullptr, m * MT + H1, max(rlo, m * MT + H1), min(rhi, m * MT + MT),
                                 tagb, fast, K0, K1, n_frustum, n_tiny);
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
