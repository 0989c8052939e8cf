// qxres.cuh — per-warp slot reservation in the stage-1 fp64 queue.
#pragma once
#include "../../include/curast.h"

namespace curast {

// Per-warp slot reservation in the fp64 queue.  One u64 atomicAdd per warp
// step on the single queue counter serialises at the L2: ~1.5 G same-address
// atomics/s measured on the B200 (tools/atomic_probe.cu: 0.52 ms for the 780 K
// steps of a config-B frame, the filter's own length), and the filter ran at
// that floor, bimodally slower in some processes.  A warp instead takes
// CURAST_QX_RES slots at a time and hands them to its steps; a step that
// overruns the block continues in the next one.  The warp's final rest is left
// as holes (tag -1), skipped by the fp64 pass (which counts them in
// CURAST_C_QXHOLES).  The queue counter therefore counts reserved slots, which
// is what the host sizes the queue by.  Slots are 32-bit (< 2^32 entries).
struct QxReserve {
    unsigned next;   // next free reserved slot
    int left;        // reserved slots left
};

// The slots of one step: step-relative index i < split goes to base + i, the
// rest to base2 + i (the next block, base2 = block - split).
struct QxSlots {
    unsigned base, base2;
    int split;
    __device__ __forceinline__ long long at(int i) const {
        return (long long)(i < split ? base + (unsigned)i : base2 + (unsigned)i);
    }
};

// tot consecutive slots for this step (whole warp, 0 < tot <= 128)
__device__ __forceinline__ QxSlots qx_reserve(QxReserve &R, unsigned long long *qcount, int tot,
                                              int lane) {
    QxSlots q;
    unsigned base = 0, base2 = 0;
    int split = 0;
    if (lane == 0) {
        const unsigned next = R.next;
        const int left = R.left;
        base = next;
        if (left < tot) {
            const unsigned blk = (unsigned)atomicAdd(qcount, (unsigned long long)CURAST_QX_RES);
            split = left;
            base2 = blk - (unsigned)left;
            R.next = blk + (unsigned)(tot - left);
            R.left = CURAST_QX_RES - (tot - left);
        } else {
            split = tot;
            R.next = next + (unsigned)tot;
            R.left = left - tot;
        }
    }
    q.base = __shfl_sync(0xffffffffu, base, 0);
    q.split = __shfl_sync(0xffffffffu, split, 0);
    q.base2 = q.split < tot ? __shfl_sync(0xffffffffu, base2, 0) : 0u;   // uniform branch
    return q;
}

// tot slots for a step of any size: the reservation blocks for up to
// CURAST_QX_RES slots, one direct allocation beyond (no holes either way)
__device__ __forceinline__ QxSlots reserve_slots(QxReserve &R, unsigned long long *qcount,
                                                 int tot, int lane) {
    if (tot <= CURAST_QX_RES) return qx_reserve(R, qcount, tot, lane);
    unsigned base = 0;
    if (lane == 0) base = (unsigned)atomicAdd(qcount, (unsigned long long)tot);
    QxSlots q;
    q.base = __shfl_sync(0xffffffffu, base, 0);
    q.base2 = 0;
    q.split = tot;
    return q;
}

// the warp's final rest becomes holes
__device__ __forceinline__ void qx_reserve_close(const curast_frame_t &f, const QxReserve &R, int lane) {
    __syncwarp();
    const unsigned b = R.next;
    const int n = R.left;
#pragma unroll 1
    for (int j = lane; j < n; j += 32)
        if ((long long)b + j < f.qx_cap) f.qx[CURAST_QX_WORDS * ((long long)b + j) + CURAST_QX_TAG] = -1;
}

}  // namespace curast
