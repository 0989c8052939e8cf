// stage1.cuh — generic-format stage-1 cull filter (k_s1_cull): f64 / f32 /
// u16 positions and u32 / bit-packed indices through ItemGeo, 4 consecutive
// triangles per lane, warp-granular chunk claims, undecided triangles to the
// fp64 queue with one atomic per 128 triangles.  The f32 + u32 layout uses
// the leaner k_s1_lean (stage1_lean.cuh).
#pragma once
#include "exact.cuh"
#include "filter.cuh"
#include "qxres.cuh"

namespace curast {

constexpr int W_THREADS = 256;
constexpr int W_WARPS = W_THREADS / 32;
constexpr int W_TPL = 4;                       // consecutive triangles per lane per step
constexpr int W_STEP = 32 * W_TPL;             // triangles per warp step
constexpr int W_QCAP = 32 + W_STEP;            // per-warp fp64 queue

struct FilterPairs {
    float2 cx, cy, cz, c3;   // (X, Y) rows, per input coordinate
    float dx, dy, dz, d3;    // d row
    float exy, ed, near_hi;
};

__device__ __forceinline__ void load_filter_pairs(FilterPairs &F, const float *__restrict__ p) {
    const float4 *q = (const float4 *)p;
    float4 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2), d = __ldg(q + 3);
    F.cx = make_float2(a.x, a.y);   // interleaved (X, Y) rows (filter.cuh)
    F.cy = make_float2(a.z, a.w);
    F.cz = make_float2(b.x, b.y);
    F.c3 = make_float2(b.z, b.w);
    F.dx = c.x; F.dy = c.y; F.dz = c.z; F.d3 = c.w;
    F.exy = d.x; F.ed = d.y; F.near_hi = d.z;
}


// Scalar fp32 cull filter, same decisions and bound as filter_tri, with a
// short path for triangles whose eps-expanded bbox lies strictly inside the
// viewport (then neither frustum cull can apply).
__device__ __forceinline__ int filter_fast(const FilterConsts &F, const float *vx, const float *vy,
                                           const float *vz, float W, float H, float slack,
                                           bool tiny_cull) {
    float px[3], py[3], D[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        D[k] = frow(F.c + 8, vx[k], vy[k], vz[k]);
        const float X = frow(F.c, vx[k], vy[k], vz[k]);
        const float Y = frow(F.c + 4, vx[k], vy[k], vz[k]);
        const float r = rcp_approx(D[k]);
        px[k] = X * r;
        py[k] = Y * r;
    }
    const float dmin = fminf(D[0], fminf(D[1], D[2]));
    if (!(dmin > F.near_hi)) return FILT_EXACT;
    const float minx = fminf(px[0], fminf(px[1], px[2])), maxx = fmaxf(px[0], fmaxf(px[1], px[2]));
    const float miny = fminf(py[0], fminf(py[1], py[2])), maxy = fmaxf(py[0], fmaxf(py[1], py[2]));
    const float M = fmaxf(fmaxf(fabsf(minx), fabsf(maxx)), fmaxf(fabsf(miny), fabsf(maxy)));
    float eps = __fmaf_rn(M, F.ed, F.exy) * rcp_approx(dmin);
    eps = __fmaf_rn(eps, 1.5f, __fmaf_rn(M, kRelSlack, slack));
    const float lox = minx - eps, loy = miny - eps, hix = maxx + eps, hiy = maxy + eps;
    if (lox > 0.0f && loy > 0.0f && hix < W && hiy < H) {
        if (!tiny_cull) return FILT_EXACT;
        const float e2 = eps + eps;
        const bool ext = (maxx - minx > e2) && (maxy - miny > e2);
        const bool tx = ceilf(lox - 0.5f) + 0.5f > hix;
        const bool ty = ceilf(loy - 0.5f) + 0.5f > hiy;
        return (ext && (tx || ty)) ? CULL_TINY : FILT_EXACT;
    }
    if (hix < 0.0f || lox > W || loy > H || hiy < 0.0f) return CULL_FRUSTUM;
    const bool not_frustum = (maxx - eps > 0.0f) && (minx + eps < W) && (miny + eps < H) &&
                             (maxy - eps > 0.0f);
    if (!not_frustum || !tiny_cull) return FILT_EXACT;
    const float e2 = eps + eps;
    if (!(maxx - minx > e2 && maxy - miny > e2)) return FILT_EXACT;
    if (ceilf(lox - 0.5f) + 0.5f > hix || ceilf(loy - 0.5f) + 0.5f > hiy) return CULL_TINY;
    return FILT_EXACT;
}

// filter_fast with the (X, Y) rows and (px, py) on packed f32x2 FFMA2/FMUL2.
__device__ __forceinline__ int filter_fast2(const FilterPairs &F, const float *vx, const float *vy,
                                            const float *vz, float W, float H, float slack,
                                            bool tiny_cull) {
    float px[3], py[3], D[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        D[k] = __fmaf_rn(F.dz, vz[k], __fmaf_rn(F.dy, vy[k], __fmaf_rn(F.dx, vx[k], F.d3)));
        float2 t = __ffma2_rn(F.cx, make_float2(vx[k], vx[k]), F.c3);
        t = __ffma2_rn(F.cy, make_float2(vy[k], vy[k]), t);
        t = __ffma2_rn(F.cz, make_float2(vz[k], vz[k]), t);
        const float r = rcp_approx(D[k]);
        const float2 p = __fmul2_rn(t, make_float2(r, r));
        px[k] = p.x;
        py[k] = p.y;
    }
    const float dmin = fminf(D[0], fminf(D[1], D[2]));
    if (!(dmin > F.near_hi)) return FILT_EXACT;
    const float minx = fminf(px[0], fminf(px[1], px[2])), maxx = fmaxf(px[0], fmaxf(px[1], px[2]));
    const float miny = fminf(py[0], fminf(py[1], py[2])), maxy = fmaxf(py[0], fmaxf(py[1], py[2]));
    const float M = fmaxf(fmaxf(fabsf(minx), fabsf(maxx)), fmaxf(fabsf(miny), fabsf(maxy)));
    float eps = __fmaf_rn(M, F.ed, F.exy) * rcp_approx(dmin);
    eps = __fmaf_rn(eps, 1.5f, __fmaf_rn(M, kRelSlack, slack));
    const float lox = minx - eps, loy = miny - eps, hix = maxx + eps, hiy = maxy + eps;
    if (lox > 0.0f && loy > 0.0f && hix < W && hiy < H) {
        if (!tiny_cull) return FILT_EXACT;
        const float e2 = eps + eps;
        const bool ext = (maxx - minx > e2) && (maxy - miny > e2);
        const bool tx = ceilf(lox - 0.5f) + 0.5f > hix;
        const bool ty = ceilf(loy - 0.5f) + 0.5f > hiy;
        return (ext && (tx || ty)) ? CULL_TINY : FILT_EXACT;
    }
    if (hix < 0.0f || lox > W || loy > H || hiy < 0.0f) return CULL_FRUSTUM;
    const bool not_frustum = (maxx - eps > 0.0f) && (minx + eps < W) && (miny + eps < H) &&
                             (maxy - eps > 0.0f);
    if (!not_frustum || !tiny_cull) return FILT_EXACT;
    const float e2 = eps + eps;
    if (!(maxx - minx > e2 && maxy - miny > e2)) return FILT_EXACT;
    if (ceilf(lox - 0.5f) + 0.5f > hix || ceilf(loy - 0.5f) + 0.5f > hiy) return CULL_TINY;
    return FILT_EXACT;
}

// Stage-1 cull filter (split mode producer): every warp claims chunks and
// appends the triangles it cannot decide to the global fp64 queue with one
// atomic per 128 triangles (warp prefix sum).
// WP: the queue entry carries the triangle's positions (POS_U16: the 9 raw
// u16 grid coordinates in words 0-2; POS_F32: the 9 floats) for
// k_s1_exact<.., WITHPOS>.
template <int PF, int IF, int MINB, bool PAIR, bool WP = false>
__global__ void __launch_bounds__(W_THREADS, MINB) k_s1_cull(const curast_frame_t f) {
    const int lane = threadIdx.x & 31;
    unsigned long long *qcount = (unsigned long long *)(f.counters + CURAST_C_QX);
    __shared__ QxReserve sres[W_THREADS / 32];
    QxReserve &R = sres[threadIdx.x >> 5];
    if (lane == 0) R = QxReserve{0u, 0};
    __syncwarp();
    unsigned int n_frustum = 0, n_tiny = 0;
    const float W = (float)f.width, H = (float)f.height;
    const float slack = (float)(f.width > f.height ? f.width : f.height) * 1.4551915e-11f;
    const bool tiny = f.tiny_cull != 0;
    const int64_t total = __ldg(f.unit_chunk_prefix + f.n_units);

    for (;;) {
        long long c = 0, item = 0, lo = 0, hi = 0;
        if (lane == 0) {
            c = (long long)atomicAdd((unsigned long long *)(f.counters + CURAST_C_CLAIM1), 1ull);
            if (c < total) {
                int64_t u = upper_index(f.unit_chunk_prefix, f.n_units + 1, c);
                item = __ldg(f.unit_index + u);
                lo = __ldg(f.unit_lo + u) + (c - __ldg(f.unit_chunk_prefix + u)) * f.chunk_tris;
                hi = __ldg(f.unit_hi + u);
                hi = lo + f.chunk_tris < hi ? lo + f.chunk_tris : hi;
            }
        }
        c = __shfl_sync(0xffffffffu, c, 0);
        if (c >= total) break;
        item = __shfl_sync(0xffffffffu, item, 0);
        lo = __shfl_sync(0xffffffffu, lo, 0);
        hi = __shfl_sync(0xffffffffu, hi, 0);

        FilterConsts F;
        FilterPairs FP;
        if (PAIR) load_filter_pairs(FP, f.item_filter + CURAST_FILTER_FLOATS * item);
        else load_filter(F, f.item_filter + CURAST_FILTER_FLOATS * item);
        ItemGeo<PF, IF> G;
        G.load(f, item);
        const int n_chunk = (int)(hi - lo);
        const uint32_t *ibase = G.idx + 3 * lo;
        const int64_t tag = (item << 40) | lo;
        for (int s0 = 0; s0 < n_chunk; s0 += W_STEP) {
            const int o = s0 + W_TPL * lane;
            const int nv = max(0, min(W_TPL, n_chunk - o));
            uint32_t ix[3 * W_TPL];
            const uint32_t *ip = ibase + 3 * o;
            if (IF == CURAST_IDX_U32 && nv == W_TPL && ((uintptr_t)ip & 15) == 0) {
                const uint4 *v = (const uint4 *)ip;
                uint4 a = __ldg(v), b = __ldg(v + 1), d = __ldg(v + 2);
                ix[0] = a.x; ix[1] = a.y; ix[2] = a.z; ix[3] = a.w;
                ix[4] = b.x; ix[5] = b.y; ix[6] = b.z; ix[7] = b.w;
                ix[8] = d.x; ix[9] = d.y; ix[10] = d.z; ix[11] = d.w;
            } else {
                G.template index_run<3 * W_TPL>(3 * (lo + o), 3 * nv, ix);
            }
            float px[3 * W_TPL], py[3 * W_TPL], pz[3 * W_TPL];
#pragma unroll
            for (int k = 0; k < 3 * W_TPL; ++k) G.pos32(ix[k], px[k], py[k], pz[k]);
            unsigned need = 0;
#pragma unroll
            for (int t = 0; t < W_TPL; ++t) {
                if (t < nv) {
                    const int code =
                        PAIR ? filter_fast2(FP, px + 3 * t, py + 3 * t, pz + 3 * t, W, H, slack, tiny)
                             : filter_fast(F, px + 3 * t, py + 3 * t, pz + 3 * t, W, H, slack, tiny);
                    n_frustum += (code == CULL_FRUSTUM);
                    n_tiny += (code == CULL_TINY);
                    need |= (code == FILT_EXACT) ? (1u << t) : 0u;
                }
            }
            // warp prefix sum of the per-lane counts -> one atomic per step
            const int mine = __popc(need);
            int incl = mine;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, d);
                if (lane >= d) incl += v;
            }
            const int wtotal = __shfl_sync(0xffffffffu, incl, 31);
            if (wtotal) {
                const QxSlots qs = qx_reserve(R, qcount, wtotal, lane);
                int si = incl - mine;
                while (need) {
                    const int t = __ffs(need) - 1;
                    need &= need - 1;
                    const long long slot = qs.at(si);
                    if (slot < f.qx_cap) {
                        int64_t *e = f.qx + CURAST_QX_WORDS * slot;
                        if (WP && PF == CURAST_POS_U16) {
                            uint64_t q[9];
#pragma unroll
                            for (int v = 0; v < 3; ++v) {
                                uint32_t a, b, c;
                                q16_load(G.pos, ix[3 * t + v], a, b, c);
                                q[3 * v] = a; q[3 * v + 1] = b; q[3 * v + 2] = c;
                            }
                            e[0] = (int64_t)(q[0] | q[1] << 16 | q[2] << 32 | q[3] << 48);
                            e[1] = (int64_t)(q[4] | q[5] << 16 | q[6] << 32 | q[7] << 48);
                            e[2] = (int64_t)q[8];
                        } else if (WP && PF == CURAST_POS_F32) {
                            *(float4 *)e = make_float4(px[3 * t], py[3 * t], pz[3 * t], px[3 * t + 1]);
                            *(float4 *)(e + 2) = make_float4(py[3 * t + 1], pz[3 * t + 1],
                                                             px[3 * t + 2], py[3 * t + 2]);
                            *(float2 *)(e + 4) = make_float2(pz[3 * t + 2], 0.0f);
                        }
                        e[CURAST_QX_TAG] = tag + o + t;
                    }
                    ++si;
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
