// tma_probe.cu — does TMA gather4 beat per-lane LDG.128 gathers for the
// stage-1 vertex fetch pattern?  (experiment for DESIGN.md §7; not shipped)
//
// Config-B-shaped data generated on the device: an n x n quad grid
// (make_tessellated_quad index order), float4 vertices.  Both kernels walk
// 128-triangle steps (lane = 4 consecutive triangles), fetch the 12 vertex
// refs of each lane and sum them (no filter math):
//   ldg : 12 x LDG.128 per lane from HBM/L2 through L1
//   tma : 3 x cp.async.bulk.tensor.2d.tile::gather4 per lane into shared
//         memory (one mbarrier per warp, double buffered), then 12 x LDS.128
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_probe tma_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_grid(float4 *pos, uint32_t *idx, int n) {
    const int64_t V = (int64_t)(n + 1) * (n + 1), Q = (int64_t)n * n;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / (n + 1), c = i % (n + 1);
        pos[i] = make_float4(c * 1e-3f, r * 1e-3f, 0.0f, 0.0f);
    }
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < Q; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = q / n, i = q % n;
        const uint32_t a = (uint32_t)(j * (n + 1) + i), b = a + 1, c = a + n + 1, d = c + 1;
        uint32_t *t = idx + 6 * q;
        t[0] = a; t[1] = c; t[2] = b; t[3] = b; t[4] = c; t[5] = d;
    }
}

__global__ void __launch_bounds__(256, 4) k_ldg(const float4 *pos, const uint32_t *idx, int64_t steps, float *out) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    float acc = 0.0f;
    for (int64_t s = warp; s < steps; s += nw) {
        const uint4 *v = (const uint4 *)(idx + 384 * s) + 3 * lane;
        const uint4 a = __ldg(v), b = __ldg(v + 1), d = __ldg(v + 2);
        const uint32_t ix[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, d.x, d.y, d.z, d.w};
#pragma unroll
        for (int k = 0; k < 12; ++k) {
            const float4 q = __ldg(pos + ix[k]);
            acc += q.x + q.y + q.z;
        }
    }
    if (acc == 123.456f) out[0] = acc;
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__global__ void __launch_bounds__(128, 8) k_tma(const __grid_constant__ CUtensorMap map, const uint32_t *idx,
                                                int64_t steps, float *out) {
    // per warp: 2 buffers x 32 lanes x 12 rows x 16 B = 12 KB
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar[4][2];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    float4 *buf = (float4 *)(smem + wid * 12288);
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    if (lane == 0) {
        for (int b = 0; b < 2; ++b)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar[wid][b])), "r"(1));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    float acc = 0.0f;
    uint32_t phase[2] = {0, 0};
    auto issue = [&](int64_t s, int b) {
        const uint4 *v = (const uint4 *)(idx + 384 * s) + 3 * lane;
        const uint4 a = __ldg(v), c = __ldg(v + 1), d = __ldg(v + 2);
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[wid][b])),
                         "r"(32 * 12 * 16));
        __syncwarp();
        float4 *dst = buf + b * 384 + 12 * lane;
        const uint32_t bs = smem_u32(&bar[wid][b]);
        asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
                     " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)), "l"(&map), "r"(0),
                     "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(bs) : "memory");
        asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
                     " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst + 4)), "l"(&map), "r"(0),
                     "r"(c.x), "r"(c.y), "r"(c.z), "r"(c.w), "r"(bs) : "memory");
        asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
                     " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst + 8)), "l"(&map), "r"(0),
                     "r"(d.x), "r"(d.y), "r"(d.z), "r"(d.w), "r"(bs) : "memory");
    };
    int64_t s = warp;
    if (s < steps) issue(s, 0);
    int b = 0;
    for (; s < steps; s += nw) {
        if (s + nw < steps) issue(s + nw, b ^ 1);
        // wait for buffer b
        const uint32_t bs = smem_u32(&bar[wid][b]);
        uint32_t done = 0;
        while (!done) {
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(bs), "r"(phase[b]) : "memory");
        }
        phase[b] ^= 1;
        const float4 *src = buf + b * 384 + 12 * lane;
#pragma unroll
        for (int k = 0; k < 12; ++k) {
            const float4 q = src[k];
            acc += q.x + q.y + q.z;
        }
        __syncwarp();
        b ^= 1;
    }
    if (acc == 123.456f) out[0] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const int n = 7071;
    const int64_t V = (int64_t)(n + 1) * (n + 1), T = 2LL * n * n;
    const int64_t steps = T / 128;
    float4 *pos;
    uint32_t *idx;
    float *out;
    CK(cudaMalloc(&pos, V * 16));
    CK(cudaMalloc(&idx, 3 * T * 4 + 4096));
    CK(cudaMalloc(&out, 16));
    k_grid<<<148 * 8, 256>>>(pos, idx, n);
    CK(cudaDeviceSynchronize());
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    CUtensorMap map;
    cuuint64_t dims[2] = {4, (cuuint64_t)V};
    cuuint64_t strides[1] = {16};
    cuuint32_t box[2] = {4, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = ((EncodeFn)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, pos, dims, strides, box, es,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode rc=%d\n", (int)r);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int nsm = 148;
    CK(cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 12288));
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        k_ldg<<<nsm * 4, 256>>>(pos, idx, steps, out);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("ldg  %.3f ms\n", ms);
        cudaEventRecord(e0);
        k_tma<<<nsm * 4, 128, 4 * 12288>>>(map, idx, steps, out);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        CK(cudaGetLastError());
        cudaEventElapsedTime(&ms, e0, e1);
        printf("tma  %.3f ms\n", ms);
    }
    // correctness of the gather: compare sums on one step via a tiny check
    return 0;
}
