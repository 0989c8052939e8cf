// resolve.cu — resolve/shading pass over the visibility buffer
// (resolvepass.py:297-395) and the supersampling box filter
// (resolvepass.py:398-407).
//
// K4: one thread per pixel.  Background words (CLEAR) get the background
// colour; otherwise the owning draw item is found by binary search over the
// global-ID prefix sums (resolvepass.py:316), the triangle is
// transformed to world space, the pixel ray intersects its plane
// (ray/plane barycentrics, resolvepass.py:184-205), barycentrics are clamped
// into the simplex and the pixel is shaded (flat / vertex colour / textured
// with mip selection from neighbouring pixel rays, resolvepass.py:138-294),
// optionally with a headlight term, rounded half-to-even and clipped.
//
// Parity is tolerance based: the reference evaluates the
// 3-term dot products with BLAS/einsum whose summation order is not
// specified, so channels may differ by 1 where a value lands on a rounding
// boundary; background pixels and the per-pixel item/triangle choice are
// exact.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/curast.h"
#include "exact.cuh"

using namespace curast;

namespace {

struct V3 { double x, y, z; };
__device__ __forceinline__ V3 v3(double x, double y, double z) { return {x, y, z}; }
__device__ __forceinline__ V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ V3 cross(V3 a, V3 b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}

// the resolve pass reads the frame's geometry through a curast_frame_t-like
// view so the fetch templates of the rasterizer can be reused
__device__ __forceinline__ curast_frame_t geo_view(const curast_resolve_t &r) {
    curast_frame_t f;
    f.pos_format = r.pos_format;
    f.idx_format = r.idx_format;
    f.positions = r.positions;
    f.indices = r.indices;
    f.item_vtx_off = r.item_vtx_off;
    f.item_idx_off = r.item_idx_off;
    f.item_qgrid = r.item_qgrid;
    f.item_pack = r.item_pack;
    return f;
}

// numpy float mod: result takes the sign of the divisor (1.0)
__device__ __forceinline__ double np_mod1(double a) {
    double m = fmod(a, 1.0);
    if (m != 0.0) {
        if (m < 0.0) m += 1.0;
    } else {
        m = 0.0;
    }
    return m;
}

__device__ __forceinline__ void bilinear(const curast_resolve_t &r, int64_t level, double u,
                                         double v, double out[4]) {
    const int64_t *ld = r.level_desc + 3 * level;
    const int64_t w = ld[0], h = ld[1];
    const uint8_t *img = r.texels + ld[2];
    double x = u * (double)w - 0.5;
    double y = (1.0 - v) * (double)h - 0.5;
    double fx0 = floor(x), fy0 = floor(y);
    double fx = x - fx0, fy = y - fy0;
    int64_t x0 = (int64_t)fx0, y0 = (int64_t)fy0;
    int64_t x0m = ((x0 % w) + w) % w, x1m = (((x0 + 1) % w) + w) % w;
    int64_t y0m = ((y0 % h) + h) % h, y1m = (((y0 + 1) % h) + h) % h;
    for (int c = 0; c < 4; ++c) {
        double c00 = img[(y0m * w + x0m) * 4 + c], c10 = img[(y0m * w + x1m) * 4 + c];
        double c01 = img[(y1m * w + x0m) * 4 + c], c11 = img[(y1m * w + x1m) * 4 + c];
        double top = c00 * (1 - fx) + c10 * fx;
        double bot = c01 * (1 - fx) + c11 * fx;
        out[c] = top * (1 - fy) + bot * fy;
    }
}

__device__ __forceinline__ V3 pixel_dir(const curast_resolve_t &r, double xs, double ys) {
    // _pixel_dirs (resolvepass.py:208-214): d_view @ rot
    double ndx = 2.0 * (xs + 0.5) / (double)r.width - 1.0;
    double ndy = 1.0 - 2.0 * (ys + 0.5) / (double)r.height;
    double a = ndx / r.p0, b = ndy / r.p1, c = -1.0;
    const double *R = r.rot;
    return v3(a * R[0] + b * R[3] + c * R[6], a * R[1] + b * R[4] + c * R[7],
              a * R[2] + b * R[5] + c * R[8]);
}

__device__ __forceinline__ uint32_t rgba(uint32_t r, uint32_t g, uint32_t b, uint32_t a) {
    return r | (g << 8) | (b << 16) | (a << 24);
}

// 4 resident blocks per SM (64 registers; 128 without the bound held
// the kernel at 16 warps per SM, latency-bound on its gathers)
#ifndef CURAST_RESOLVE_MINB
#define CURAST_RESOLVE_MINB 4
#endif
template <int PF, int IF>
__global__ void __launch_bounds__(256, CURAST_RESOLVE_MINB) k_resolve(const curast_resolve_t r) {
    __shared__ unsigned long long s_cnt[3];
    if (threadIdx.x < 3) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    const curast_frame_t f = geo_view(r);
    unsigned long long shaded = 0, bg = 0, degen = 0;
    const int64_t npix = r.width * (r.rows > 0 ? r.rows : r.height);
    for (int64_t pix = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; pix < npix;
         pix += (int64_t)gridDim.x * blockDim.x) {
        uint64_t word = r.fb[pix];
        // one 32-bit store per pixel (RGBA8)
        uint32_t *o = (uint32_t *)r.out_rgba + pix;
        if (word == ~0ull) {
            *o = rgba(r.background[0], r.background[1], r.background[2], r.background[3]);
            bg++;
            continue;
        }
        const int64_t gid = (int64_t)(word & ((1ull << 36) - 1));
        int64_t lo = 0, hi = r.n_items + 1;
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if (r.prefix[mid] <= gid) lo = mid + 1; else hi = mid;
        }
        const int64_t item = lo - 1;
        const int64_t local = gid - r.prefix[item];
        const double *m = r.item_mw + 12 * item;
        uint32_t vi[3];
        V3 w[3];
        for (int k = 0; k < 3; ++k) {
            vi[k] = fetch_index<IF>(f, item, 3 * local + k);
            double x, y, z;
            fetch_pos64<PF>(f, item, vi[k], x, y, z);
            // obj @ m[:3,:3].T + m[:3,3]
            w[k] = v3(x * m[0] + y * m[1] + z * m[2] + m[3], x * m[4] + y * m[5] + z * m[6] + m[7],
                      x * m[8] + y * m[9] + z * m[10] + m[11]);
        }
        // width * rows < 2^31: 32-bit index arithmetic
        const int p32 = (int)pix, w32 = (int)r.width;
        const double xs = (double)(p32 % w32), ys = (double)(r.row0 + p32 / w32);
        const V3 dir = pixel_dir(r, xs, ys);
        const V3 org = v3(r.cam[0], r.cam[1], r.cam[2]);
        // _moller_trumbore_bulk (resolvepass.py:184-205)
        V3 e1 = sub(w[1], w[0]), e2 = sub(w[2], w[0]);
        V3 nrm = cross(e1, e2);
        double denom = dot(dir, nrm);
        bool ok = denom != 0.0;
        double safe = ok ? denom : 1.0;
        double t_ray = dot(sub(w[0], org), nrm) / safe;
        V3 hit = v3(org.x + t_ray * dir.x, org.y + t_ray * dir.y, org.z + t_ray * dir.z);
        V3 wv = sub(hit, w[0]);
        double d00 = dot(e1, e1), d01 = dot(e1, e2), d11 = dot(e2, e2);
        double den = d00 * d11 - d01 * d01;
        ok = ok && den != 0.0;
        if (!ok) den = 1.0;
        double we1 = dot(wv, e1), we2 = dot(wv, e2);
        double s = (d11 * we1 - d01 * we2) / den;
        double t = (d00 * we2 - d01 * we1) / den;
        if (!ok) {
            degen++;
            *o = rgba(255, 0, 255, 255);
            shaded++;
            continue;
        }
        s = fmax(s, 0.0);
        t = fmax(t, 0.0);
        double tot = s + t;
        if (tot > 1.0) { s = s / tot; t = t / tot; }
        double v = 1.0 - s - t;
        int mode = r.item_mode[item];
        double col[4];
        if (mode == 1) {
            const uint8_t *c0 = r.colors + 4 * (r.item_color_off[item] + vi[0]);
            const uint8_t *c1 = r.colors + 4 * (r.item_color_off[item] + vi[1]);
            const uint8_t *c2 = r.colors + 4 * (r.item_color_off[item] + vi[2]);
            for (int c = 0; c < 4; ++c)
                col[c] = v * (double)c0[c] + s * (double)c1[c] + t * (double)c2[c];
        } else if (mode == 2) {
            const double *uv0 = r.uvs + 2 * (r.item_color_off[item] + vi[0]);
            const double *uv1 = r.uvs + 2 * (r.item_color_off[item] + vi[1]);
            const double *uv2 = r.uvs + 2 * (r.item_color_off[item] + vi[2]);
            const int64_t tex = r.item_tex[item];
            const int64_t nlev = r.tex_desc[2 * tex], lev0 = r.tex_desc[2 * tex + 1];
            const double tw = (double)r.level_desc[3 * lev0], th = (double)r.level_desc[3 * lev0 + 1];
            // _estimate_levels_bulk (resolvepass.py:262-294)
            double level = 0.0;
            {
                bool lok = (d00 * d11 - d01 * d01) != 0.0;
                double dd = d00 * d11 - d01 * d01;
                if (!lok) dd = 1.0;
                double us[3], vs[3];
                const int ox[3] = {0, 1, 0}, oy[3] = {0, 0, -1};
                for (int q = 0; q < 3; ++q) {
                    V3 dq = pixel_dir(r, xs + ox[q], ys + oy[q]);
                    double dn = dot(dq, nrm);
                    if (dn == 0.0) { lok = false; dn = 1.0; }
                    double tr = dot(sub(w[0], org), nrm) / dn;
                    V3 wq = sub(v3(org.x + tr * dq.x, org.y + tr * dq.y, org.z + tr * dq.z), w[0]);
                    double a1 = dot(wq, e1), a2 = dot(wq, e2);
                    double sq = (d11 * a1 - d01 * a2) / dd;
                    double tq = (d00 * a2 - d01 * a1) / dd;
                    double vq = 1.0 - sq - tq;
                    us[q] = vq * uv0[0] + sq * uv1[0] + tq * uv2[0];
                    vs[q] = vq * uv0[1] + sq * uv1[1] + tq * uv2[1];
                }
                double dr = fmax(fabs(us[1] - us[0]) * tw, fabs(vs[1] - vs[0]) * th);
                double dt = fmax(fabs(us[2] - us[0]) * tw, fabs(vs[2] - vs[0]) * th);
                double ext = fmax(dr, dt);
                level = ext > 0.0 ? log2(fmax(ext, 1e-300)) : 0.0;
                level = fmin(fmax(level, 0.0), (double)(nlev - 1));
                if (!lok) level = 0.0;
            }
            double uu = np_mod1(v * uv0[0] + s * uv1[0] + t * uv2[0]);
            double vv = np_mod1(v * uv0[1] + s * uv1[1] + t * uv2[1]);
            if (r.trilinear) {
                double flo = floor(level);
                int64_t l0 = (int64_t)flo;
                int64_t l1 = l0 + 1 < nlev - 1 ? l0 + 1 : nlev - 1;
                double fr = level - flo;
                double a[4], b[4];
                bilinear(r, lev0 + l0, uu, vv, a);
                bilinear(r, lev0 + l1, uu, vv, b);
                for (int c = 0; c < 4; ++c) col[c] = a[c] * (1 - fr) + b[c] * fr;
            } else {
                int64_t ln = (int64_t)rint(level);
                bilinear(r, lev0 + ln, uu, vv, col);
            }
        } else {
            for (int c = 0; c < 4; ++c) col[c] = (double)r.base_color[c];
        }
        if (r.headlight) {
            double nlen = sqrt(dot(nrm, nrm)), dlen = sqrt(dot(dir, dir));
            double ndl = fabs(dot(nrm, dir)) / fmax(nlen * dlen, 1e-300);
            double sh = 0.2 + 0.8 * ndl;
            col[0] *= sh; col[1] *= sh; col[2] *= sh;
        }
        uint32_t q8[4];
        for (int c = 0; c < 4; ++c) {
            double q = rint(col[c]);
            q = fmin(fmax(q, 0.0), 255.0);
            q8[c] = (uint32_t)q;
        }
        *o = rgba(q8[0], q8[1], q8[2], q8[3]);
        shaded++;
    }
    atomicAdd(&s_cnt[0], shaded);
    atomicAdd(&s_cnt[1], bg);
    atomicAdd(&s_cnt[2], degen);
    __syncthreads();
    if (threadIdx.x < 3 && s_cnt[threadIdx.x])
        atomicAdd((unsigned long long *)(r.counters + threadIdx.x), s_cnt[threadIdx.x]);
}

// box filter with floor rounding (resolvepass.py:398-407): one thread per
// output pixel, a source row of `factor` RGBA8 pixels as one 4/8/16-byte
// load, the four channels summed in registers, one 32-bit store
template <int FACTOR>
__global__ void k_downsample(const uint8_t *__restrict__ src, int64_t w, int64_t h,
                             uint8_t *__restrict__ dst) {
    const int64_t ow = w / FACTOR, oh = h / FACTOR;
    const int64_t n = ow * oh;
    const uint32_t *s32 = (const uint32_t *)src;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int ox = (int)p % (int)ow, oy = (int)p / (int)ow;
        uint32_t sum[4] = {0, 0, 0, 0};
#pragma unroll
        for (int dy = 0; dy < FACTOR; ++dy) {
            const uint32_t *row = s32 + (oy * FACTOR + dy) * w + ox * FACTOR;
            uint32_t px[FACTOR];
            if (FACTOR == 4) {
                const uint4 v = __ldg((const uint4 *)row);
                px[0] = v.x; px[1] = v.y; px[2 % FACTOR] = v.z; px[3 % FACTOR] = v.w;
            } else if (FACTOR == 2) {
                const uint2 v = __ldg((const uint2 *)row);
                px[0] = v.x; px[1 % FACTOR] = v.y;
            } else {
#pragma unroll
                for (int dx = 0; dx < FACTOR; ++dx) px[dx] = __ldg(row + dx);
            }
#pragma unroll
            for (int dx = 0; dx < FACTOR; ++dx)
#pragma unroll
                for (int c = 0; c < 4; ++c) sum[c] += (px[dx] >> (8 * c)) & 0xffu;
        }
        constexpr uint32_t d = FACTOR * FACTOR;
        ((uint32_t *)dst)[p] = (sum[0] / d) | ((sum[1] / d) << 8) | ((sum[2] / d) << 16) |
                               ((sum[3] / d) << 24);
    }
}

__global__ void k_downsample_any(const uint8_t *__restrict__ src, int64_t w, int64_t h, int factor,
                                 uint8_t *__restrict__ dst) {
    const int64_t ow = w / factor, oh = h / factor;
    const int64_t n = ow * oh * 4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t c = i & 3, p = i >> 2;
        int64_t ox = p % ow, oy = p / ow;
        uint32_t sum = 0;
        for (int dy = 0; dy < factor; ++dy)
            for (int dx = 0; dx < factor; ++dx)
                sum += src[((oy * factor + dy) * w + ox * factor + dx) * 4 + c];
        dst[i] = (uint8_t)(sum / (uint32_t)(factor * factor));
    }
}

int sms() {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
}


// ------------------------------------------------------------ debug views
// resolvepass.py:417-490.  depth: grey = rint(255 (1 - log(d/lo)/log(hi/lo)))
// over the covered pixels' depth range; meshID: palette of the owning item;
// stageID / bboxSize: the winning triangle re-transformed as the reference
// does ((obj @ T^T) @ view^T, left-to-right 4-term sums) and routed by
// classify_route (pipeline.py, kernels.clip_near for near crossers).
__constant__ uint8_t kStageColor[4][4] = {
    {80, 190, 90, 255}, {235, 205, 60, 255}, {225, 70, 70, 255}, {255, 0, 255, 255}};

__global__ void k_debug_range(const uint64_t *fb, int64_t npix, uint32_t *scratch) {
    uint32_t lo = 0xFFFFFFFFu, hi = 0u;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npix;
         p += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t w = fb[p];
        if (w == ~0ull) continue;
        const uint32_t bits = (uint32_t)(w >> 36) << 3;     // positive f32: uint order
        lo = min(lo, bits);
        hi = max(hi, bits);
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(scratch, lo);
        atomicMax(scratch + 1, hi);
    }
}

// 0 STAGE1, 1 STAGE2_DIRECT, 2 STAGE3_TILED, 3 None; area out
__device__ __forceinline__ int debug_route(const double *vx, const double *vy, const double *vz,
                                           double p0, double p1, double near, int64_t W,
                                           int64_t H, int64_t small_max, int64_t medium_max,
                                           int64_t &area) {
    area = 0;
    const double d0 = -vz[0], d1 = -vz[1], d2 = -vz[2];
    if (d0 < near && d1 < near && d2 < near) return 3;
    const bool cross = d0 < near || d1 < near || d2 < near;
    double px[4], py[4], pz[4];
    int n = 3;
    if (cross) {
        n = clip_near(vx, vy, vz, near, px, py, pz);
    } else {
        for (int k = 0; k < 3; ++k) { px[k] = vx[k]; py[k] = vy[k]; pz[k] = vz[k]; }
    }
    if (n == 0) return 3;
    double mnx = 0, mxx = 0, mny = 0, mxy = 0;
    for (int k = 0; k < n; ++k) {
        double d = -pz[k];
        d = d < near ? near : d;                                   // np.maximum
        const double sx = M(M(A(D(M(px[k], p0), d), 1.0), 0.5), (double)W);
        const double sy = M(M(S(1.0, D(M(py[k], p1), d)), 0.5), (double)H);
        if (k == 0) { mnx = mxx = sx; mny = mxy = sy; }
        mnx = fmin(mnx, sx); mxx = fmax(mxx, sx);
        mny = fmin(mny, sy); mxy = fmax(mxy, sy);
    }
    const int64_t ix0 = max((int64_t)floor(mnx), (int64_t)0), ix1 = min((int64_t)ceil(mxx), W);
    const int64_t iy0 = max((int64_t)floor(mny), (int64_t)0), iy1 = min((int64_t)ceil(mxy), H);
    if (ix0 >= ix1 || iy0 >= iy1) return 3;
    area = (ix1 - ix0) * (iy1 - iy0);
    if (cross || area >= medium_max) return 2;
    if (area >= small_max) return 1;
    return 0;
}

template <int PF, int IF>
__global__ void k_debug_view(const curast_debug_t d) {
    curast_frame_t f;
    f.pos_format = d.pos_format;
    f.idx_format = d.idx_format;
    f.positions = d.positions;
    f.indices = d.indices;
    f.item_vtx_off = d.item_vtx_off;
    f.item_idx_off = d.item_idx_off;
    f.item_qgrid = d.item_qgrid;
    f.item_pack = d.item_pack;
    const int64_t npix = d.width * d.height;
    double lo = 0.0, hi = 0.0, span = 1.0;
    if (d.mode == 0) {
        lo = (double)__uint_as_float(d.scratch[0]);
        hi = (double)__uint_as_float(d.scratch[1]);
        span = hi > lo ? log(D(hi, lo)) : 1.0;
    }
    for (int64_t pix = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; pix < npix;
         pix += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t w = d.fb[pix];
        uint8_t *o = d.out_rgba + 4 * pix;
        uint8_t c[4] = {d.background[0], d.background[1], d.background[2], d.background[3]};
        if (w != ~0ull) {
            if (d.mode == 0) {
                const double dep = (double)__uint_as_float((uint32_t)(w >> 36) << 3);
                const double shade = hi > lo ? D(log(D(dep, lo)), span) : 0.0;
                double g = rint(M(255.0, S(1.0, shade)));
                g = g < 0.0 ? 0.0 : (g > 255.0 ? 255.0 : g);
                c[0] = c[1] = c[2] = (uint8_t)g;
                c[3] = 255;
            } else {
                const int64_t gid = (int64_t)(w & ((1ull << 36) - 1));
                int64_t a = 0, b = d.n_items + 1;
                while (a < b) {
                    const int64_t mid = (a + b) >> 1;
                    if (d.prefix[mid] <= gid) a = mid + 1; else b = mid;
                }
                const int64_t item = a - 1;
                if (d.mode == 3) {
                    const int k = (int)(item & 255);
                    c[0] = (uint8_t)((53 + 97 * k) & 255);
                    c[1] = (uint8_t)((131 + 61 * k) & 255);
                    c[2] = (uint8_t)((197 + 151 * k) & 255);
                    c[3] = 255;
                } else {
                    const int64_t local = gid - d.prefix[item];
                    const double *T = d.item_xform + 16 * item;
                    double vx[3], vy[3], vz[3];
                    for (int k = 0; k < 3; ++k) {
                        const uint32_t vi = fetch_index<IF>(f, item, 3 * local + k);
                        double x, y, z;
                        fetch_pos64<PF>(f, item, vi, x, y, z);
                        double wv[4];
                        for (int r = 0; r < 4; ++r)
                            wv[r] = A(A(A(M(x, T[4 * r]), M(y, T[4 * r + 1])), M(z, T[4 * r + 2])),
                                      M(1.0, T[4 * r + 3]));
                        double vv[3];
                        for (int r = 0; r < 3; ++r)
                            vv[r] = A(A(A(M(wv[0], d.view[4 * r]), M(wv[1], d.view[4 * r + 1])),
                                        M(wv[2], d.view[4 * r + 2])), M(wv[3], d.view[4 * r + 3]));
                        vx[k] = vv[0]; vy[k] = vv[1]; vz[k] = vv[2];
                    }
                    int64_t area;
                    const int route = debug_route(vx, vy, vz, d.p0, d.p1, d.near, d.width,
                                                  d.height, d.small_max, d.medium_max, area);
                    int ci = route;
                    if (route != 3 && d.mode == 2)
                        ci = area < d.small_max ? 0 : (area < d.medium_max ? 1 : 2);
                    for (int q = 0; q < 4; ++q) c[q] = kStageColor[ci][q];
                }
            }
        }
        o[0] = c[0]; o[1] = c[1]; o[2] = c[2]; o[3] = c[3];
    }
}
}  // namespace

extern "C" {

int curast_resolve(const curast_resolve_t *r, void *stream) {
    if (!r || !r->fb || !r->out_rgba || !r->counters || r->width <= 0 || r->height <= 0 ||
        r->row0 < 0 || r->rows < 0 || r->row0 + r->rows > r->height ||
        r->width * r->height >= (1ll << 31))
        return CURAST_E_INVALID;
    cudaStream_t st = (cudaStream_t)stream;
    int grid = sms() * 8;
    int pf = r->pos_format, ix = r->idx_format;
    if (pf == CURAST_POS_F32 && ix == CURAST_IDX_U32) k_resolve<1, 0><<<grid, 256, 0, st>>>(*r);
    else if (pf == CURAST_POS_F64 && ix == CURAST_IDX_U32) k_resolve<0, 0><<<grid, 256, 0, st>>>(*r);
    else if (pf == CURAST_POS_U16 && ix == CURAST_IDX_U32) k_resolve<2, 0><<<grid, 256, 0, st>>>(*r);
    else if (pf == CURAST_POS_F32 && ix == CURAST_IDX_PACKED) k_resolve<1, 1><<<grid, 256, 0, st>>>(*r);
    else if (pf == CURAST_POS_F64 && ix == CURAST_IDX_PACKED) k_resolve<0, 1><<<grid, 256, 0, st>>>(*r);
    else if (pf == CURAST_POS_U16 && ix == CURAST_IDX_PACKED) k_resolve<2, 1><<<grid, 256, 0, st>>>(*r);
    else return CURAST_E_INVALID;
    return cudaGetLastError() == cudaSuccess ? 0 : CURAST_E_CUDA;
}

int curast_debug_view(const curast_debug_t *d, void *stream) {
    if (!d || !d->fb || !d->out_rgba || d->width <= 0 || d->height <= 0 || d->mode < 0 ||
        d->mode > 3 || (d->mode == 0 && !d->scratch))
        return CURAST_E_INVALID;
    cudaStream_t st = (cudaStream_t)stream;
    const int grid = sms() * 8;
    if (d->mode == 0) {
        const uint32_t init[2] = {0xFFFFFFFFu, 0u};
        cudaMemcpyAsync(d->scratch, init, sizeof(init), cudaMemcpyHostToDevice, st);
        k_debug_range<<<grid, 256, 0, st>>>(d->fb, d->width * d->height, d->scratch);
    }
    int pf = d->pos_format, ix = d->idx_format;
    if (pf == CURAST_POS_F32 && ix == CURAST_IDX_U32) k_debug_view<1, 0><<<grid, 256, 0, st>>>(*d);
    else if (pf == CURAST_POS_F64 && ix == CURAST_IDX_U32) k_debug_view<0, 0><<<grid, 256, 0, st>>>(*d);
    else if (pf == CURAST_POS_U16 && ix == CURAST_IDX_U32) k_debug_view<2, 0><<<grid, 256, 0, st>>>(*d);
    else if (pf == CURAST_POS_F32 && ix == CURAST_IDX_PACKED) k_debug_view<1, 1><<<grid, 256, 0, st>>>(*d);
    else if (pf == CURAST_POS_F64 && ix == CURAST_IDX_PACKED) k_debug_view<0, 1><<<grid, 256, 0, st>>>(*d);
    else if (pf == CURAST_POS_U16 && ix == CURAST_IDX_PACKED) k_debug_view<2, 1><<<grid, 256, 0, st>>>(*d);
    else return CURAST_E_INVALID;
    return cudaGetLastError() == cudaSuccess ? 0 : CURAST_E_CUDA;
}

int curast_downsample(const uint8_t *src, int64_t w, int64_t h, int32_t factor, uint8_t *dst,
                      void *stream) {
    if (!src || !dst || factor < 1 || w % factor || h % factor) return CURAST_E_INVALID;
    cudaStream_t st = (cudaStream_t)stream;
    if (factor == 2 && ((uintptr_t)src & 7) == 0) k_downsample<2><<<sms() * 8, 256, 0, st>>>(src, w, h, dst);
    else if (factor == 4 && ((uintptr_t)src & 15) == 0) k_downsample<4><<<sms() * 8, 256, 0, st>>>(src, w, h, dst);
    else k_downsample_any<<<sms() * 4, 256, 0, st>>>(src, w, h, factor, dst);
    return cudaGetLastError() == cudaSuccess ? 0 : CURAST_E_CUDA;
}

}  // extern "C"
