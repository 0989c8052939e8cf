// stage1_ws.cuh — warp-specialised stage 1: fp32 filter warps and fp64 exact
// warps in the same CTA, connected by a shared-memory ring.
//
// The filter (FFMA2/MUFU, issue-bound) and the exact path (DMUL/DFMA, FP64
// pipe) use different pipes, so running them on the same SM at the same time
// overlaps their issue; the queued triangles never leave the SM (no 48 B/entry
// HBM round trip as in the split lean/exact pair).
//
//   producers (warps 0..7): k_s1_lean's per-step body; undecided triangles get
//     a ticket from the ring tail, wait for their slot to be free, write the 9
//     fp32 positions + tag and publish the slot (pub[slot] = ticket + 1).
//   consumers (warps 8..11): claim 32 tickets at a time, wait for publication,
//     run the bit-exact fp64 _process_tri (kernels.py:49-157) on all lanes,
//     release the slot (free[slot] = ticket + RING).
// Termination: the last producer warp of the CTA records the final tail; a
// consumer lane whose ticket is >= final has no work.
#pragma once
#include "exact.cuh"
#include "filter.cuh"
#include "stage1_lean.cuh"

namespace curast {

constexpr int WS_PRODUCERS = 8;
constexpr int WS_CONSUMERS = 4;
constexpr int WS_THREADS = 32 * (WS_PRODUCERS + WS_CONSUMERS);
constexpr int WS_RING = 512;
// register budgets: launched at 80/thread (2 CTAs of 384 per SM); producers
// give 24 back, consumers take 48: 256*56 + 128*128 = 384*80
#ifndef WS_SETMAXNREG
#define WS_SETMAXNREG 1
#endif
constexpr int WS_PROD_REGS = 56;
constexpr int WS_CONS_REGS = 128;

struct WsEntry {
    float4 a, b;
    float c, pad;
    long long tag;
};

struct WsShared {
    WsEntry ring[WS_RING];
    unsigned pub[WS_RING];
    unsigned freeq[WS_RING];
    unsigned tail, claim, prod_done, final_tail;
};

__device__ __forceinline__ unsigned vld(const unsigned *p) {
    return *(const volatile unsigned *)p;
}

template <int PF>
__global__ void __launch_bounds__(WS_THREADS, 2) k_s1_ws(const curast_frame_t f) {
    __shared__ WsShared s;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < WS_RING; i += WS_THREADS) {
        s.pub[i] = 0u;
        s.freeq[i] = (unsigned)i;
    }
    if (threadIdx.x == 0) {
        s.tail = 0u;
        s.claim = 0u;
        s.prod_done = 0u;
        s.final_tail = 0xFFFFFFFFu;
    }
    __syncthreads();

    if (warp < WS_PRODUCERS) {
        // ------------------------------------------------------ producers
#if WS_SETMAXNREG
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(WS_PROD_REGS));
#endif
        constexpr int CHUNK = 2048, TPL = 4, STEP = 32 * TPL;
        const unsigned lt_mask = (1u << lane) - 1u;
        unsigned n_frustum = 0, n_tiny = 0;
        const float W = (float)f.width, H = (float)f.height;
        const float slack = (float)(f.width > f.height ? f.width : f.height) * 1.4551915e-11f;
        const bool tiny = f.tiny_cull != 0;
        const int64_t total = __ldg(f.unit_chunk_prefix + f.n_units);
        for (;;) {
            long long c = 0, item = 0, lo = 0, hi = 0;
            if (lane == 0) {
                c = (long long)atomicAdd((unsigned long long *)(f.counters + CURAST_C_CLAIM1), 1ull);
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
            const float *pb = (const float *)f.positions + 3 * vo;
            const uint32_t *ib = (const uint32_t *)f.indices + io + 3 * lo;
            const int n = (int)(hi - lo);
            const bool vec = (((uintptr_t)ib) & 15) == 0;
            const long long tag = (item << 40) | lo;
            for (int s0 = 0; s0 < n; s0 += STEP) {
                const int o = s0 + TPL * lane;
                const int nv = max(0, min(TPL, n - o));
                uint32_t ix[3 * TPL];
                if (vec && nv == TPL) {
                    const uint4 *v = (const uint4 *)(ib + 3 * o);
                    const uint4 a = __ldg(v), b = __ldg(v + 1), d = __ldg(v + 2);
                    ix[0] = a.x; ix[1] = a.y; ix[2] = a.z; ix[3] = a.w;
                    ix[4] = b.x; ix[5] = b.y; ix[6] = b.z; ix[7] = b.w;
                    ix[8] = d.x; ix[9] = d.y; ix[10] = d.z; ix[11] = d.w;
                } else {
#pragma unroll
                    for (int k = 0; k < 3 * TPL; ++k) ix[k] = (k < 3 * nv) ? __ldg(ib + 3 * o + k) : 0u;
                }
                float px[3 * TPL], py[3 * TPL], pz[3 * TPL];
#pragma unroll
                for (int k = 0; k < 3 * TPL; ++k) {
                    const float *p = pb + 3 * ix[k];
                    px[k] = __ldg(p);
                    py[k] = __ldg(p + 1);
                    pz[k] = __ldg(p + 2);
                }
                unsigned need = 0, fr = 0;
#pragma unroll
                for (int t = 0; t < TPL; ++t) {
                    const unsigned bits = lean_bits(F, px + 3 * t, py + 3 * t, pz + 3 * t, W, H,
                                                    slack, tiny);
                    if (t < nv) {
                        need |= (bits & 1u) << t;
                        fr |= (bits >> 1) << t;
                    }
                }
                n_frustum += __popc(fr);
                n_tiny += nv - __popc(need) - __popc(fr);
                unsigned b[TPL];
                unsigned tot = 0;
#pragma unroll
                for (int t = 0; t < TPL; ++t) {
                    b[t] = __ballot_sync(0xffffffffu, (need >> t) & 1u);
                    tot += __popc(b[t]);
                }
                if (tot) {
                    unsigned base = 0;
                    if (lane == 0) base = atomicAdd(&s.tail, tot);
                    base = __shfl_sync(0xffffffffu, base, 0);
#pragma unroll
                    for (int t = 0; t < TPL; ++t) {
                        if ((need >> t) & 1u) {
                            const unsigned T = base + __popc(b[t] & lt_mask);
                            const unsigned slot = T & (WS_RING - 1);
                            while (vld(&s.freeq[slot]) != T) __nanosleep(64);
                            WsEntry &e = s.ring[slot];
                            e.a = make_float4(px[3 * t], py[3 * t], pz[3 * t], px[3 * t + 1]);
                            e.b = make_float4(py[3 * t + 1], pz[3 * t + 1], px[3 * t + 2], py[3 * t + 2]);
                            e.c = pz[3 * t + 2];
                            e.tag = tag + o + t;
                            __threadfence_block();
                            *(volatile unsigned *)&s.pub[slot] = T + 1u;
                        }
                        base += __popc(b[t]);
                    }
                }
            }
        }
        __syncwarp();
        __threadfence_block();
        if (lane == 0) {
            const unsigned done = atomicAdd(&s.prod_done, 1u) + 1u;
            if (done == WS_PRODUCERS) {
                __threadfence_block();
                *(volatile unsigned *)&s.final_tail = vld(&s.tail);
            }
        }
        unsigned long long cnt[2] = {n_frustum, n_tiny};
        flush_stats(f.counters + CURAST_C_S1 + CULL_FRUSTUM, cnt, 1);
        flush_stats(f.counters + CURAST_C_S1 + CULL_TINY, cnt + 1, 1);
    } else {
        // ------------------------------------------------------ consumers
#if WS_SETMAXNREG
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(WS_CONS_REGS));
#endif
        unsigned long long cnt[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
        for (;;) {
            unsigned tb = 0;
            if (lane == 0) tb = atomicAdd(&s.claim, 32u);
            tb = __shfl_sync(0xffffffffu, tb, 0);
            const unsigned T = tb + lane;
            const unsigned slot = T & (WS_RING - 1);
            bool have = false;
            for (;;) {
                if (vld(&s.pub[slot]) == T + 1u) { have = true; break; }
                const unsigned fin = vld(&s.final_tail);
                if (fin != 0xFFFFFFFFu && T >= fin) break;
                __nanosleep(256);     // idle consumers must not steal issue slots
            }
            if (have) {
                __threadfence_block();
                const WsEntry &e = s.ring[slot];
                const float4 a = e.a, b = e.b;
                const float cc = e.c;
                const long long ent = e.tag;
                __threadfence_block();
                *(volatile unsigned *)&s.freeq[slot] = T + (unsigned)WS_RING;
                const int64_t item = ent >> 40, local = ent & ((1ll << 40) - 1);
                const uint64_t gid = (uint64_t)(__ldg(f.prefix + item) + local);
                int64_t frags;
                const int code = process_tri_exact(a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, cc,
                                                   f.item_mv + 12 * item, gid, f.p0, f.p1, f.width,
                                                   f.height, f.near, f.tiny_cull, f.force_stage,
                                                   f.small_max, f.fb, frags);
#pragma unroll
                for (int k = 0; k < 7; ++k) cnt[k] += (code == k);
                cnt[7] += (unsigned long long)frags;
                cnt[8] += 1;
                const int64_t qslot = warp_reserve(f.counters + CURAST_C_Q2, code == ST_FORWARD);
                if (qslot >= 0 && qslot < f.q2_cap) {
                    f.q2[2 * qslot] = item;
                    f.q2[2 * qslot + 1] = local;
                }
            }
            __syncwarp();
            if (__ballot_sync(0xffffffffu, have) == 0u) {
                // no lane had work: all tickets of this batch are past the end
                break;
            }
        }
        flush_stats(f.counters + CURAST_C_S1, cnt, 8);
        flush_stats(f.counters + CURAST_C_EXACT, cnt + 8, 1);
    }
}

}  // namespace curast
