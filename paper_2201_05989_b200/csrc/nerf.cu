// nerf.cu — NeRF training on the hash-grid fields (the
// paper's §5.4 and Appendix E; BASELINE config 4). The reference declares
// NeRF out of scope, so the oracle is a restatement of the
// paper's appendix (oracle/oracle.py, "parity unpinned").
//
// Per training step (all on the device, one host sync for the sample count):
//   1. R rays: (view, pixel) from the device Pcg32 stream
//   2. occupancy-grid ray marching, pass 1: samples per ray (fixed step
//      dt = sqrt(3)/1024 in the unit cube, empty 128^3 cells skipped by a
//      DDA step to the next cell boundary, <= max samples per ray)
//   3. exclusive scan -> sample offsets; the rays that fit the fixed sample
//      budget are kept ("as many rays as possible in batches of fixed size",
//      PAPER.md:954), R adapts to the measured samples per ray
//   4. pass 2 writes the COMPACTED samples (position, direction) into dense
//      buffers
//   5. density network (hash encoding -> 1x64 -> 16, fused inference),
//      color network input [16 density outputs | SH degree-4 of the
//      direction] -> 2x64 -> RGB (sigmoid)
//   6. compositing per ray (alpha = 1 - exp(-sigma dt), transmittance early
//      stop at 1e-4, background), L2 loss, and its backward (dRGB per
//      sample, dsigma through the suffix sums)
//   7. backward through the color MLP, then the density network (encode
//      backward scatter), Adam on both
//   8. every 16 steps: occupancy update (decay 0.95, max with the density at
//      a random point of sampled cells, threshold 0.01 * 1024 / sqrt(3)
//      capped by the mean cell density, as instant-ngp does in practice)
// Ray arithmetic is fp32 without contraction (-fmad=false) in the order of the
// numpy restatement, so sample positions compare bit-exactly.
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/nfg.h"
#include "host_common.h"


namespace {

using nfg::hc::Buf;
using nfg::hc::Fail;
using nfg::hc::grid_for;
using nfg::hc::ok;
using nfg::hc::run;

constexpr int OCC_RES = 128;
constexpr int OCC_CELLS = OCC_RES * OCC_RES * OCC_RES;
constexpr float SQRT3 = 1.7320508075688772f;







// ---- occupancy grid: 128^3 bits in Morton order ---------
__host__ __device__ inline uint32_t spread3(uint32_t v)   // 7 bits -> every third bit
{
    v &= 0x7fu;
    v = (v | (v << 8)) & 0x0000f00fu;
    v = (v | (v << 4)) & 0x000c30c3u;
    v = (v | (v << 2)) & 0x00249249u;
    return v;
}

__host__ __device__ inline uint32_t morton3(uint32_t x, uint32_t y, uint32_t z)
{
    return spread3(x) | (spread3(y) << 1) | (spread3(z) << 2);
}

__host__ __device__ inline uint32_t compact3(uint32_t v)
{
    v &= 0x00249249u;
    v = (v | (v >> 2)) & 0x000c30c3u;
    v = (v | (v >> 4)) & 0x0000f00fu;
    v = (v | (v >> 8)) & 0x0000007fu;
    return v;
}

__device__ __forceinline__ int cell_coord(float p)
{
    const int c = int(p * float(OCC_RES));
    return c < 0 ? 0 : (c > OCC_RES - 1 ? OCC_RES - 1 : c);
}

__device__ __forceinline__ bool occupied(const uint8_t* bits, float px, float py, float pz)
{
    const uint32_t m = morton3(uint32_t(cell_coord(px)), uint32_t(cell_coord(py)), uint32_t(cell_coord(pz)));
    return (bits[m >> 3] >> (m & 7u)) & 1u;
}

// Ray / unit-cube slab test in fp32 (NaN-ignoring min/max).
__device__ __forceinline__ bool ray_cube(const float* o, const float* d, float& t0, float& t1)
{
    t0 = -INFINITY;
    t1 = INFINITY;
    for (int k = 0; k < 3; ++k) {
        const float inv = 1.0f / d[k];
        const float a = (0.0f - o[k]) * inv, b = (1.0f - o[k]) * inv;
        t0 = fmaxf(t0, fminf(a, b));
        t1 = fminf(t1, fmaxf(a, b));
    }
    t0 = fmaxf(t0, 0.0f);
    return t1 > t0;
}

// Marching defines the samples of a ray as the grid points
//   t_k = t_base + k dt,  t_base = t0 + dt/2,  t_k < t1,
// whose 128^3 occupancy cell is set, in k order, capped at max_steps. A lane
// walks its own contiguous k-range: at an occupied point it emits and steps
// by one; at an empty point it jumps by a DDA step to the cell boundary,
// floor(tn / dt) - 1 points (>= 1) so no point past the boundary is ever
// skipped — every lane, and the serial restatement, therefore produce exactly
// the same set whatever their starting k. One WARP marches one ray (32
// k-ranges), so a batch of a few thousand rays still fills the GPU.
struct RayGrid {
    float tb, t1;
    int kmax;   // upper bound on the points (exclusive)
};

__device__ __forceinline__ bool ray_grid(const float* o, const float* d, RayGrid& g)
{
    float t0, t1;
    if (!ray_cube(o, d, t0, t1))
        return false;
    const float dt = SQRT3 / 1024.0f;
    g.tb = t0 + 0.5f * dt;
    g.t1 = t1;
    g.kmax = int(ceilf((t1 - g.tb) / dt)) + 1;
    return g.kmax > 0;
}

template <class Emit>
__device__ int march_range(const float* o, const float* d, const uint8_t* bits, const RayGrid& g, int k0, int k1,
                           Emit&& emit)
{
    const float dt = SQRT3 / 1024.0f;
    int n = 0;
    for (int k = k0; k < k1;) {
        const float t = g.tb + float(k) * dt;
        if (!(t < g.t1))
            break;
        const float px = o[0] + t * d[0], py = o[1] + t * d[1], pz = o[2] + t * d[2];
        if (occupied(bits, px, py, pz)) {
            emit(n, px, py, pz);
            ++n;
            ++k;
            continue;
        }
        const float p[3] = { px, py, pz };
        float tn = INFINITY;
        for (int a = 0; a < 3; ++a) {
            const float c = float(cell_coord(p[a]) + (d[a] > 0.0f ? 1 : 0));
            const float ta = (c / float(OCC_RES) - p[a]) / d[a];
            tn = fminf(tn, ta);
        }
        const float steps = floorf(tn / dt) - 1.0f;
        k += steps > 1.0f ? (steps < 1e6f ? int(steps) : 1000000) : 1;
    }
    return n;
}

__device__ __forceinline__ uint32_t warp_excl_scan(uint32_t v, int lane, uint32_t& total)
{
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o)
            x += y;
    }
    total = __shfl_sync(0xffffffffu, x, 31);
    return x - v;
}

__global__ void k_march_count(const float* __restrict__ rays, int64_t n, const uint8_t* __restrict__ bits,
                              int max_steps, uint32_t* __restrict__ counts)
{
    const int lane = threadIdx.x & 31;
    const int64_t wid = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t r = wid; r < n; r += nw) {
        const float* o = rays + 6 * r;
        RayGrid g;
        uint32_t c = 0;
        if (ray_grid(o, o + 3, g)) {
            const int chunk = (g.kmax + 31) / 32;
            c = uint32_t(march_range(o, o + 3, bits, g, lane * chunk, min(g.kmax, (lane + 1) * chunk),
                                     [](int, float, float, float) {}));
        }
        uint32_t total;
        warp_excl_scan(c, lane, total);
        if (lane == 0)
            counts[r] = min(total, uint32_t(max_steps));
    }
}

__global__ void k_march_write(const float* __restrict__ rays, int64_t n, const uint8_t* __restrict__ bits,
                              int max_steps, const uint32_t* __restrict__ offsets, float* __restrict__ pos,
                              float* __restrict__ dirs)
{
    const int lane = threadIdx.x & 31;
    const int64_t wid = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t r = wid; r < n; r += nw) {
        const float* o = rays + 6 * r;
        const float* d = o + 3;
        RayGrid g;
        if (!ray_grid(o, d, g))
            continue;   // warp-uniform
        const int chunk = (g.kmax + 31) / 32;
        const int k0 = lane * chunk, k1 = min(g.kmax, (lane + 1) * chunk);
        const uint32_t c = uint32_t(march_range(o, d, bits, g, k0, k1, [](int, float, float, float) {}));
        uint32_t total;
        const uint32_t first = warp_excl_scan(c, lane, total);
        const uint32_t base = offsets[r];
        const uint32_t cap = uint32_t(max_steps);
        if (first < cap)
            march_range(o, d, bits, g, k0, k1, [&](int i, float px, float py, float pz) {
                const uint32_t j = first + uint32_t(i);
                if (j >= cap)
                    return;
                const size_t sidx = size_t(base) + j;
                pos[3 * sidx] = px;
                pos[3 * sidx + 1] = py;
                pos[3 * sidx + 2] = pz;
                dirs[3 * sidx] = d[0];
                dirs[3 * sidx + 1] = d[1];
                dirs[3 * sidx + 2] = d[2];
            });
    }
}

// Largest prefix of rays whose samples fit the budget.
__global__ void k_fit_budget(const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ counts, int64_t n,
                             int64_t budget, int64_t* out /* [rays, samples] */)
{
    // offsets are non-decreasing: binary search the last ray with offset + count <= budget
    if (blockIdx.x != 0 || threadIdx.x != 0)
        return;
    int64_t lo = 0, hi = n;   // answer in [0, n]
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) / 2;   // candidate ray count
        if (int64_t(offsets[mid - 1]) + int64_t(counts[mid - 1]) <= budget)
            lo = mid;
        else
            hi = mid - 1;
    }
    out[0] = lo;
    out[1] = lo > 0 ? int64_t(offsets[lo - 1]) + int64_t(counts[lo - 1]) : 0;
}

// ---- SH degree 4 (16 coefficients) of a unit direction ----------------------
__host__ __device__ inline void sh4(float x, float y, float z, float* o)
{
    const float xy = x * y, xz = x * z, yz = y * z, x2 = x * x, y2 = y * y, z2 = z * z;
    o[0] = 0.28209479177387814f;
    o[1] = -0.48860251190291987f * y;
    o[2] = 0.48860251190291987f * z;
    o[3] = -0.48860251190291987f * x;
    o[4] = 1.0925484305920792f * xy;
    o[5] = -1.0925484305920792f * yz;
    o[6] = 0.94617469575755997f * z2 - 0.31539156525251999f;
    o[7] = -1.0925484305920792f * xz;
    o[8] = 0.54627421529603959f * x2 - 0.54627421529603959f * y2;
    o[9] = 0.59004358992664352f * y * (-3.0f * x2 + y2);
    o[10] = 2.8906114426405538f * xy * z;
    o[11] = 0.45704579946446572f * y * (1.0f - 5.0f * z2);
    o[12] = 0.3731763325901154f * z * (5.0f * z2 - 3.0f);
    o[13] = 0.45704579946446572f * x * (1.0f - 5.0f * z2);
    o[14] = 1.4453057213202769f * z * (x2 - y2);
    o[15] = 0.59004358992664352f * x * (-x2 + 3.0f * y2);
}

// color input = [16 density outputs | SH4(direction)] (128 B rows, float4 stores)
__global__ void k_color_input(const float* __restrict__ dens, const float* __restrict__ dirs, int64_t n,
                              float* __restrict__ Y)
{
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        float sh[16];
        sh4(dirs[3 * i], dirs[3 * i + 1], dirs[3 * i + 2], sh);
        const float4* src = reinterpret_cast<const float4*>(dens + 16 * i);
        float4* dst = reinterpret_cast<float4*>(Y + 32 * i);
#pragma unroll
        for (int k = 0; k < 4; ++k)
            dst[k] = src[k];
#pragma unroll
        for (int k = 0; k < 4; ++k)
            dst[4 + k] = make_float4(sh[4 * k], sh[4 * k + 1], sh[4 * k + 2], sh[4 * k + 3]);
    }
}

// ---- volume compositing (forward + backward), one warp per ray -------------
// sigma = exp(raw) (the density output is log-density); the
// gradient uses exp(min(raw, 15)) (truncated exponential). Transmittance is
// carried in log space across 32-sample chunks: T_i = exp(-sum_{j<i} sigma_j dt)
// by a warp prefix sum; samples from the first T_i < 1e-4 on are dropped
// (transmittance stop); dC/dc_i = w_i, dC/dsigma_i = dt (T_{i+1} c_i -
// sum_{j>i} w_j c_j - T_end bg).
__device__ __forceinline__ float warp_incl_scan_f(float v, int lane)
{
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const float y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o)
            v += y;
    }
    return v;
}

__device__ __forceinline__ float warp_sum_f(float v)
{
#pragma unroll
    for (int m = 16; m > 0; m >>= 1)
        v += __shfl_xor_sync(0xffffffffu, v, m);
    return v;
}

__global__ void k_composite(const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ counts, int64_t n_rays,
                            const float* __restrict__ raw, int raw_stride, const float* __restrict__ rgb,
                            const float* __restrict__ target, float3 bg, float dt, float inv_count,
                            float* __restrict__ out_color, float* __restrict__ d_rgb, float* __restrict__ d_raw,
                            double* loss_sum, uint32_t* __restrict__ used_counts = nullptr)
{
    const int lane = threadIdx.x & 31;
    const int64_t wid = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    double lsum = 0.0;
    for (int64_t r = wid; r < n_rays; r += nw) {
        const uint32_t base = offsets[r], n = counts[r];
        // forward
        float logT = 0.0f, cr = 0.0f, cg = 0.0f, cb = 0.0f;
        uint32_t n_used = 0;
        for (uint32_t c0 = 0; c0 < n && __expf(logT) >= 1e-4f; c0 += 32) {
            const uint32_t i = c0 + lane;
            float x = 0.0f, r0 = 0.0f, r1 = 0.0f, r2 = 0.0f;
            if (i < n) {
                const size_t s = size_t(base) + i;
                x = expf(raw[s * raw_stride]) * dt;
                r0 = rgb[3 * s];
                r1 = rgb[3 * s + 1];
                r2 = rgb[3 * s + 2];
            }
            const float incl = warp_incl_scan_f(x, lane);
            const float Ti = expf(logT - (incl - x));
            const float w = (i < n && Ti >= 1e-4f) ? Ti * (1.0f - expf(-x)) : 0.0f;
            cr += warp_sum_f(w * r0);
            cg += warp_sum_f(w * r1);
            cb += warp_sum_f(w * r2);
            // transmittance after the last used sample of this chunk
            const bool used = i < n && Ti >= 1e-4f;
            const unsigned um = __ballot_sync(0xffffffffu, used);
            const int last = um ? 31 - __clz(um) : -1;
            n_used += uint32_t(__popc(um));
            const float incl_last = last >= 0 ? __shfl_sync(0xffffffffu, incl, last) : 0.0f;
            logT -= incl_last;
            if (um != 0xffffffffu)
                break;   // a sample of this chunk crossed the stop (or the ray ended)
        }
        const float Tend = expf(logT);
        if (used_counts && lane == 0)
            used_counts[r] = n_used;   // the used samples are the first n_used of the ray
        const float Cr = cr + Tend * bg.x, Cg = cg + Tend * bg.y, Cb = cb + Tend * bg.z;
        if (out_color && lane == 0) {
            out_color[3 * r] = Cr;
            out_color[3 * r + 1] = Cg;
            out_color[3 * r + 2] = Cb;
        }
        if (!target)
            continue;
        const float er = Cr - target[3 * r], eg = Cg - target[3 * r + 1], eb = Cb - target[3 * r + 2];
        if (lane == 0)
            lsum += double(er * er + eg * eg + eb * eb);
        const float gr = 2.0f * er * inv_count, gg = 2.0f * eg * inv_count, gb = 2.0f * eb * inv_count;
        // backward (second sweep, same chunking)
        float logT2 = 0.0f, pr = 0.0f, pg = 0.0f, pb = 0.0f;
        for (uint32_t c0 = 0; c0 < n; c0 += 32) {
            const uint32_t i = c0 + lane;
            const size_t s = size_t(base) + i;
            float x = 0.0f, rw = 0.0f, r0 = 0.0f, r1 = 0.0f, r2 = 0.0f;
            if (i < n) {
                rw = raw[s * raw_stride];
                x = expf(rw) * dt;
                r0 = rgb[3 * s];
                r1 = rgb[3 * s + 1];
                r2 = rgb[3 * s + 2];
            }
            const float incl = warp_incl_scan_f(x, lane);
            const float Ti = expf(logT2 - (incl - x));
            const bool used = i < n && Ti >= 1e-4f;
            const float w = used ? Ti * (1.0f - expf(-x)) : 0.0f;
            const float qr = warp_incl_scan_f(w * r0, lane) + pr;
            const float qg = warp_incl_scan_f(w * r1, lane) + pg;
            const float qb = warp_incl_scan_f(w * r2, lane) + pb;
            if (i < n) {
                if (used) {
                    const float T1 = expf(logT2 - incl);   // T_{i+1}
                    d_rgb[3 * s] = w * gr;
                    d_rgb[3 * s + 1] = w * gg;
                    d_rgb[3 * s + 2] = w * gb;
                    const float sr = T1 * r0 - (cr - qr) - Tend * bg.x;
                    const float sg = T1 * r1 - (cg - qg) - Tend * bg.y;
                    const float sb = T1 * r2 - (cb - qb) - Tend * bg.z;
                    d_raw[s] = dt * (sr * gr + sg * gg + sb * gb) * expf(fminf(rw, 15.0f));
                } else {
                    d_rgb[3 * s] = d_rgb[3 * s + 1] = d_rgb[3 * s + 2] = 0.0f;
                    d_raw[s] = 0.0f;
                }
            }
            pr = __shfl_sync(0xffffffffu, qr, 31);
            pg = __shfl_sync(0xffffffffu, qg, 31);
            pb = __shfl_sync(0xffffffffu, qb, 31);
            logT2 -= __shfl_sync(0xffffffffu, incl, 31);
        }
    }
    if (loss_sum) {
        for (int m = 16; m > 0; m >>= 1)
            lsum += __shfl_xor_sync(0xffffffffu, lsum, m);
        if (lane == 0)
            atomicAdd(loss_sum, lsum);
    }
}

// Second compaction ("compaction of samples into dense buffers"):
// only the samples before a ray's transmittance stop reach the backward
// networks. One warp per ray copies its used prefix (position, color input
// row, dL/dRGB, dL/draw) to the compacted buffers.
__global__ void k_compact_used(const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ used,
                               const uint32_t* __restrict__ used_off, int64_t n_rays, const float* __restrict__ pos,
                               const float* __restrict__ Yc, const float* __restrict__ d_rgb,
                               const float* __restrict__ d_raw, float* __restrict__ pos_c, float* __restrict__ Yc_c,
                               float* __restrict__ d_rgb_c, float* __restrict__ d_raw_c)
{
    const int lane = threadIdx.x & 31;
    const int64_t wid = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t r = wid; r < n_rays; r += nw) {
        const uint32_t src0 = offsets[r], dst0 = used_off[r], n = used[r];
        for (uint32_t i = lane; i < n; i += 32) {
            const size_t a = size_t(src0) + i, b = size_t(dst0) + i;
            for (int k = 0; k < 3; ++k) {
                pos_c[3 * b + k] = pos[3 * a + k];
                d_rgb_c[3 * b + k] = d_rgb[3 * a + k];
            }
            d_raw_c[b] = d_raw[a];
            const float4* ys = reinterpret_cast<const float4*>(Yc + 32 * a);
            float4* yd = reinterpret_cast<float4*>(Yc_c + 32 * b);
#pragma unroll
            for (int k = 0; k < 8; ++k)
                yd[k] = ys[k];
        }
    }
}

// d(density outputs) = [dY_color[0:16]] + d_raw on output 0
__global__ void k_density_grad(const float* __restrict__ dYc, const float* __restrict__ d_raw, int64_t n,
                               float* __restrict__ d_dens)
{
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const float4* src = reinterpret_cast<const float4*>(dYc + 32 * i);
        float4* dst = reinterpret_cast<float4*>(d_dens + 16 * i);
        float4 v = src[0];
        v.x += d_raw[i];
        dst[0] = v;
#pragma unroll
        for (int k = 1; k < 4; ++k)
            dst[k] = src[k];
    }
}

// ---- rays from views: cams are (position, forward, right, up) x 3 floats ----
__device__ __forceinline__ void pixel_ray(const float* cam, uint32_t px, int w, int h, float focal, float* ray)
{
    const int x = int(px % uint32_t(w)), y = int(px / uint32_t(w));
    const float u = (float(x) + 0.5f - 0.5f * float(w)) / focal;
    const float v = (0.5f * float(h) - float(y) - 0.5f) / focal;
    float d[3];
    for (int k = 0; k < 3; ++k)
        d[k] = cam[3 + k] + u * cam[6 + k] + v * cam[9 + k];
    const float nn = sqrtf(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    for (int k = 0; k < 3; ++k) {
        ray[k] = cam[k];
        ray[3 + k] = d[k] / nn;
    }
}

__global__ void k_train_rays(const uint32_t* __restrict__ views, const uint32_t* __restrict__ pixels, int64_t n,
                             const float* __restrict__ cams, const float* __restrict__ images, int w, int h, float focal,
                             float* __restrict__ rays, float* __restrict__ target)
{
    for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n; r += int64_t(gridDim.x) * blockDim.x) {
        const uint32_t v = views[r], p = pixels[r];
        pixel_ray(cams + 12 * v, p, w, h, focal, rays + 6 * r);
        const float* src = images + (size_t(v) * w * h + p) * 3;
        target[3 * r] = src[0];
        target[3 * r + 1] = src[1];
        target[3 * r + 2] = src[2];
    }
}

__global__ void k_view_rays(const float* __restrict__ cam, int w, int h, float focal, float* __restrict__ rays)
{
    const int64_t n = int64_t(w) * h;
    for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n; r += int64_t(gridDim.x) * blockDim.x)
        pixel_ray(cam, uint32_t(r), w, h, focal, rays + 6 * r);
}

// ---- the synthetic procedural scene (ground truth; BASELINE config 4) --------
// Three soft spheres with textured colours; view-independent emission.
struct SceneSphere {
    float cx, cy, cz, r, R, G, B;
};
__constant__ SceneSphere c_scene[3] = {
    { 0.40f, 0.45f, 0.50f, 0.18f, 0.90f, 0.30f, 0.20f },
    { 0.62f, 0.55f, 0.45f, 0.14f, 0.20f, 0.70f, 0.90f },
    { 0.50f, 0.30f, 0.62f, 0.10f, 0.85f, 0.85f, 0.25f },
};

__device__ void scene_eval(float x, float y, float z, float& sigma, float* rgb)
{
    sigma = 0.0f;
    float best = 1e9f;
    int bi = 0;
    for (int k = 0; k < 3; ++k) {
        const SceneSphere s = c_scene[k];
        const float dx = x - s.cx, dy = y - s.cy, dz = z - s.cz;
        const float dist = sqrtf(dx * dx + dy * dy + dz * dz) - s.r;
        sigma += 80.0f / (1.0f + expf(dist * 150.0f));
        if (dist < best) {
            best = dist;
            bi = k;
        }
    }
    const float tex = 0.65f + 0.35f * sinf(18.0f * (x + 0.7f * y - 0.4f * z));
    rgb[0] = c_scene[bi].R * tex;
    rgb[1] = c_scene[bi].G * tex;
    rgb[2] = c_scene[bi].B * tex;
}

__global__ void k_scene_render(const float* __restrict__ cams, int n_views, int w, int h, float focal, float3 bg,
                               float* __restrict__ out)
{
    const int64_t n = int64_t(n_views) * w * h;
    const float dt = SQRT3 / 1024.0f;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int v = int(i / (int64_t(w) * h));
        const uint32_t p = uint32_t(i % (int64_t(w) * h));
        float ray[6];
        pixel_ray(cams + 12 * v, p, w, h, focal, ray);
        float t0, t1, T = 1.0f, c[3] = { 0.0f, 0.0f, 0.0f };
        if (ray_cube(ray, ray + 3, t0, t1)) {
            for (float t = t0 + 0.5f * dt; t < t1 && T >= 1e-4f; t = t + dt) {
                float sigma, rgb[3];
                scene_eval(ray[0] + t * ray[3], ray[1] + t * ray[4], ray[2] + t * ray[5], sigma, rgb);
                const float alpha = 1.0f - expf(-sigma * dt);
                for (int k = 0; k < 3; ++k)
                    c[k] += T * alpha * rgb[k];
                T *= 1.0f - alpha;
            }
        }
        out[3 * i] = c[0] + T * bg.x;
        out[3 * i + 1] = c[1] + T * bg.y;
        out[3 * i + 2] = c[2] + T * bg.z;
    }
}

// ---- occupancy update ------------------------------------
// (the 0.95 decay, max with the density at a random point of M sampled cells:
// all cells in the first 256 steps, then a quarter of them uniformly)
__global__ void k_occ_points(const uint32_t* __restrict__ cells, const float* __restrict__ jitter, int64_t m,
                             int64_t all_from, float* __restrict__ pos, uint32_t* __restrict__ cell_out)
{
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x) {
        const uint32_t c = cells ? cells[i] : uint32_t(all_from + i);
        const float x = float(compact3(c)), y = float(compact3(c >> 1)), z = float(compact3(c >> 2));
        pos[3 * i] = (x + jitter[3 * i]) / float(OCC_RES);
        pos[3 * i + 1] = (y + jitter[3 * i + 1]) / float(OCC_RES);
        pos[3 * i + 2] = (z + jitter[3 * i + 2]) / float(OCC_RES);
        cell_out[i] = c;
    }
}

__global__ void k_occ_decay(float* grid, int64_t n, float f)
{
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        grid[i] *= f;
}

__global__ void k_occ_max(float* grid, const uint32_t* __restrict__ cells, const float* __restrict__ dens, int64_t m)
{
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x) {
        const float sigma = expf(fminf(dens[16 * i], 30.0f));
        atomicMax(reinterpret_cast<int*>(grid + cells[i]), __float_as_int(sigma));   // non-negative floats
    }
}

// Mean cell density: per-block partial sums, then one ordered sum.
__global__ void __launch_bounds__(256) k_occ_sum(const float* __restrict__ grid, double* __restrict__ partial)
{
    __shared__ double sh[256];
    double s = 0.0;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < OCC_CELLS; i += int64_t(gridDim.x) * blockDim.x)
        s += grid[i];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int k = 128; k > 0; k >>= 1) {
        if (int(threadIdx.x) < k)
            sh[threadIdx.x] += sh[threadIdx.x + k];
        __syncthreads();
    }
    if (threadIdx.x == 0)
        partial[blockIdx.x] = sh[0];
}

// Occupancy threshold: 0.01 * 1024 / sqrt(3), capped by the
// mean cell density so an untrained field (density ~ 1 everywhere) keeps the
// cells it is denser in rather than culling everything.
__global__ void k_occ_thresh(const double* __restrict__ partial, int n, float cap, float* thresh)
{
    double s = 0.0;
    for (int i = 0; i < n; ++i)
        s += partial[i];
    *thresh = fminf(cap, float(s / double(OCC_CELLS)));
}

__global__ void k_occ_bits(const float* __restrict__ grid, uint8_t* __restrict__ bits, const float* __restrict__ th)
{
    const float thresh = *th;
    for (int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; b < OCC_CELLS / 8;
         b += int64_t(gridDim.x) * blockDim.x) {
        uint8_t v = 0;
        for (int k = 0; k < 8; ++k)
            v |= uint8_t(grid[8 * b + k] > thresh ? 1u : 0u) << k;
        bits[b] = v;
    }
}

}   // namespace

struct nfg_nerf {
    nfg_ctx* ctx = nullptr;
    cudaStream_t st = nullptr;
    nfg_nerf_config cfg{};
    nfg_field* density = nullptr;
    nfg_field* color = nullptr;
    nfg_rng* rng = nullptr;
    int n_views = 0, w = 0, h = 0;
    float focal = 1.0f;
    int64_t n_rays = 1 << 13;   // adapted to the sample budget
    double last_used_frac = 1.0;   // samples before the transmittance stop / marched (previous step)
    // The networks' Adam step of a training step is deferred to the next call:
    // the next step enqueues it behind its ray marching (which only reads the
    // occupancy grid) and ahead of the host sync for the sample count, so the
    // GPU runs Adam while the host waits; every other entry point that uses
    // the networks flushes it first.
    bool adam_pending = false;
    void flush_adam()
    {
        if (!adam_pending)
            return;
        adam_pending = false;
        ok(nfg_adam_step_device(color, float(cfg.lr)));
        ok(nfg_adam_step_device(density, float(cfg.lr)));
    }
    uint32_t* h_used = nullptr;    // pinned
    Buf occ_grid, occ_bits, cams, images;
    Buf rays, target, views, pixels, counts, offsets, fit, scan_tmp, pos, dirs, dens, Yc, rgb, color_out, d_rgb, d_raw,
        dYc, d_dens, loss, used, used_off, pos_c, Yc_c, d_rgb_c, d_raw_c;
    Buf occ_cells, occ_jit, occ_pos, occ_cell, occ_dens, occ_sum, occ_th;

    ~nfg_nerf()
    {
        if (h_used)
            cudaFreeHost(h_used);
        if (rng)
            nfg_rng_destroy(rng);
        if (density)
            nfg_field_destroy(density);
        if (color)
            nfg_field_destroy(color);
    }

    // march + compact a ray set; returns (rays kept, samples)
    std::pair<int64_t, int64_t> march_compact(const float* ray_buf, int64_t R, int64_t budget,
                                              bool flush_before_sync = false)
    {
        uint32_t* cnt = counts.as<uint32_t>(size_t(R));
        uint32_t* off = offsets.as<uint32_t>(size_t(R));
        k_march_count<<<grid_for(R * 32), 256, 0, st>>>(ray_buf, R, static_cast<const uint8_t*>(occ_bits.p),
                                                   cfg.max_samples_per_ray, cnt);
        NFG_HC_CUDA(cudaGetLastError());
        size_t tb = 0;
        NFG_HC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, off, R, st));
        NFG_HC_CUDA(cub::DeviceScan::ExclusiveSum(scan_tmp.get(tb), tb, cnt, off, R, st));
        int64_t* f = fit.as<int64_t>(2);
        k_fit_budget<<<1, 1, 0, st>>>(off, cnt, R, budget, f);
        int64_t h_fit[2] = { 0, 0 };
        NFG_HC_CUDA(cudaMemcpyAsync(h_fit, f, sizeof(h_fit), cudaMemcpyDeviceToHost, st));
        if (flush_before_sync)
            flush_adam();   // runs on the GPU while the host waits for the counts
        NFG_HC_CUDA(cudaStreamSynchronize(st));
        const int64_t ns = h_fit[1];
        float* P = pos.as<float>(size_t(std::max<int64_t>(ns, 1)) * 3);
        float* D = dirs.as<float>(size_t(std::max<int64_t>(ns, 1)) * 3);
        if (h_fit[0] > 0) {
            k_march_write<<<grid_for(h_fit[0] * 32), 256, 0, st>>>(ray_buf, h_fit[0], static_cast<const uint8_t*>(occ_bits.p),
                                                              cfg.max_samples_per_ray, off, P, D);
            NFG_HC_CUDA(cudaGetLastError());
        }
        return { h_fit[0], ns };
    }

    // density + color forward on the compacted samples
    void forward(int64_t ns)
    {
        float* dn = dens.as<float>(size_t(ns) * 16);
        float* y = Yc.as<float>(size_t(ns) * 32);
        float* c = rgb.as<float>(size_t(ns) * 3);
        ok(nfg_field_evaluate_device(density, static_cast<const float*>(pos.p), ns, dn));
        k_color_input<<<grid_for(ns), 256, 0, st>>>(dn, static_cast<const float*>(dirs.p), ns, y);
        NFG_HC_CUDA(cudaGetLastError());
        ok(nfg_mlp_forward_device(color, y, ns, c));
    }

    void update_occupancy(int64_t step)
    {
        float* grid = static_cast<float*>(occ_grid.p);
        k_occ_decay<<<grid_for(OCC_CELLS), 256, 0, st>>>(grid, OCC_CELLS, 0.95f);
        const bool warm = step < 256;
        const int64_t m = warm ? OCC_CELLS : OCC_CELLS / 4;
        const int64_t chunk = int64_t(1) << 19;
        for (int64_t done = 0; done < m; done += chunk) {
            const int64_t k = std::min(chunk, m - done);
            uint32_t* cells = nullptr;
            if (!warm) {
                cells = occ_cells.as<uint32_t>(size_t(k));
                ok(nfg_rng_below_device(rng, uint32_t(OCC_CELLS), k, cells));
            }
            float* jit = occ_jit.as<float>(size_t(k) * 3);
            ok(nfg_rng_floats_device(rng, k * 3, jit));
            float* p = occ_pos.as<float>(size_t(k) * 3);
            uint32_t* cl = occ_cell.as<uint32_t>(size_t(k));
            k_occ_points<<<grid_for(k), 256, 0, st>>>(cells, jit, k, done, p, cl);
            float* dn = occ_dens.as<float>(size_t(k) * 16);
            ok(nfg_field_evaluate_device(density, p, k, dn));
            k_occ_max<<<grid_for(k), 256, 0, st>>>(grid, cl, dn, k);
            NFG_HC_CUDA(cudaGetLastError());
        }
        constexpr int SUM_BLOCKS = 296;
        double* part = occ_sum.as<double>(SUM_BLOCKS);
        float* th = occ_th.as<float>(1);
        k_occ_sum<<<SUM_BLOCKS, 256, 0, st>>>(grid, part);
        k_occ_thresh<<<1, 1, 0, st>>>(part, SUM_BLOCKS, 0.01f * 1024.0f / SQRT3, th);
        k_occ_bits<<<grid_for(OCC_CELLS / 8), 256, 0, st>>>(grid, static_cast<uint8_t*>(occ_bits.p), th);
        NFG_HC_CUDA(cudaGetLastError());
    }
};

extern "C" {

nfg_status nfg_nerf_create(nfg_ctx* ctx, const nfg_nerf_config* cfg, uint64_t seed, nfg_nerf** out)
{
    return run([&] {
        *out = nullptr;
        auto n = std::make_unique<nfg_nerf>();
        n->ctx = ctx;
        n->st = static_cast<cudaStream_t>(nfg_ctx_stream(ctx));
        n->cfg = *cfg;
        if (n->cfg.target_samples <= 0 || n->cfg.max_samples_per_ray <= 0)
            throw std::invalid_argument("nerf: target_samples and max_samples_per_ray must be positive");
        nfg_grid_config g = cfg->grid;
        g.dims = 3;
        if (g.levels * g.features != 32)
            throw Fail{ NFG_EUNSUPPORTED, "nerf: the density encoding must have levels * features == 32" };
        nfg_adam_hyper hy{ cfg->lr, 0.9, 0.99, 1e-15, 1e-6 };
        nfg_options o{ 0, 1, 0, 0 };
        // density MLP: 1 hidden layer of 64 -> 16 outputs, the first is log-density
        nfg_mlp_config md{ 0, 1, 64, 16, NFG_ACT_LINEAR };
        ok(nfg_field_create(ctx, &g, &md, &hy, &o, &n->density));
        ok(nfg_field_init(n->density, seed));
        // color MLP: [16 density outputs | SH4] -> 2 x 64 -> RGB sigmoid. It is an MLP-only field: its
        // (tiny) grid is never encoded, so its table gradients stay zero and Adam skips them.
        nfg_grid_config gc{ 16, 16u, 2, 1, 1, 3, 0 };
        nfg_mlp_config mc{ 0, 2, 64, 3, NFG_ACT_SIGMOID };
        ok(nfg_field_create(ctx, &gc, &mc, &hy, &o, &n->color));
        ok(nfg_field_init(n->color, seed + 7));
        ok(nfg_rng_create(ctx, seed, 0xe7f, &n->rng));
        NFG_HC_CUDA(cudaMallocHost(&n->h_used, sizeof(uint32_t)));
        *n->h_used = 0;
        // per-sample buffers sized for the budget once (no reallocation, which
        // would synchronise, as the ray count adapts)
        const size_t S = size_t(n->cfg.target_samples);
        n->pos.get(S * 12);
        n->dirs.get(S * 12);
        n->dens.get(S * 64);
        n->Yc.get(S * 128);
        n->rgb.get(S * 12);
        n->d_rgb.get(S * 12);
        n->d_raw.get(S * 4);
        n->dYc.get(S * 128);
        n->d_dens.get(S * 64);
        n->pos_c.get(S * 12);
        n->Yc_c.get(S * 128);
        n->d_rgb_c.get(S * 12);
        n->d_raw_c.get(S * 4);
        // occupancy: all cells occupied until the first update
        n->occ_grid.get(size_t(OCC_CELLS) * 4);
        n->occ_bits.get(OCC_CELLS / 8);
        NFG_HC_CUDA(cudaMemsetAsync(n->occ_grid.p, 0, size_t(OCC_CELLS) * 4, n->st));
        NFG_HC_CUDA(cudaMemsetAsync(n->occ_bits.p, 0xff, OCC_CELLS / 8, n->st));
        NFG_HC_CUDA(cudaStreamSynchronize(n->st));
        *out = n.release();
    });
}

nfg_status nfg_nerf_destroy(nfg_nerf* n)
{
    return run([&] { delete n; });
}

nfg_status nfg_nerf_fields(nfg_nerf* n, nfg_field** density, nfg_field** color)
{
    return run([&] {
        n->flush_adam();   // the caller sees the trained parameters
        if (density)
            *density = n->density;
        if (color)
            *color = n->color;
    });
}

nfg_status nfg_nerf_set_dataset(nfg_nerf* n, int32_t n_views, int32_t width, int32_t height, float focal,
                                const float* cams, const float* rgb)
{
    return run([&] {
        if (n_views < 1 || width < 1 || height < 1 || !(focal > 0))
            throw std::invalid_argument("nerf: empty dataset");
        n->n_views = n_views;
        n->w = width;
        n->h = height;
        n->focal = focal;
        const size_t npx = size_t(n_views) * width * height;
        NFG_HC_CUDA(cudaMemcpyAsync(n->cams.get(size_t(n_views) * 12 * 4), cams, size_t(n_views) * 12 * 4,
                                cudaMemcpyHostToDevice, n->st));
        NFG_HC_CUDA(cudaMemcpyAsync(n->images.get(npx * 12), rgb, npx * 12, cudaMemcpyHostToDevice, n->st));
        NFG_HC_CUDA(cudaStreamSynchronize(n->st));
    });
}

nfg_status nfg_nerf_train_step(nfg_nerf* n, int64_t step, float* loss, int64_t* rays_used, int64_t* samples_used)
{
    return nfg_nerf_train_step2(n, step, loss, rays_used, samples_used, nullptr);
}

nfg_status nfg_nerf_train_step2(nfg_nerf* n, int64_t step, float* loss, int64_t* rays_used, int64_t* samples_used,
                                int64_t* samples_backward)
{
    return run([&] {
        if (n->n_views == 0)
            throw std::invalid_argument("nerf: no dataset");
        cudaStream_t st = n->st;
        if (step % 16 == 0) {
            n->flush_adam();   // the occupancy update evaluates the density network
            n->update_occupancy(step);
        }
        const int64_t R = n->n_rays;
        uint32_t* vw = n->views.as<uint32_t>(size_t(R));
        uint32_t* px = n->pixels.as<uint32_t>(size_t(R));
        ok(nfg_rng_below_device(n->rng, uint32_t(n->n_views), R, vw));
        ok(nfg_rng_below_device(n->rng, uint32_t(n->w) * uint32_t(n->h), R, px));
        float* rays = n->rays.as<float>(size_t(R) * 6);
        float* tgt = n->target.as<float>(size_t(R) * 3);
        k_train_rays<<<grid_for(R), 256, 0, st>>>(vw, px, R, static_cast<const float*>(n->cams.p),
                                                  static_cast<const float*>(n->images.p), n->w, n->h, n->focal, rays,
                                                  tgt);
        NFG_HC_CUDA(cudaGetLastError());
        const auto fit = n->march_compact(rays, R, n->cfg.target_samples, /*flush_before_sync=*/true);
        const int64_t nr = fit.first, ns = fit.second;
        // adapt the ray count to the sample budget (measured samples per ray)
        const double spr = nr > 0 ? std::max(1.0, double(ns) / double(nr)) : 1.0;
        n->n_rays = std::max<int64_t>(1024, std::min<int64_t>(int64_t(1) << 22,
                                                              int64_t(double(n->cfg.target_samples) / spr * 1.05)));
        if (rays_used)
            *rays_used = nr;
        if (samples_used)
            *samples_used = ns;
        double* ls = n->loss.as<double>(1);
        NFG_HC_CUDA(cudaMemsetAsync(ls, 0, 8, st));
        if (ns > 0) {
            n->forward(ns);
            float* drgb = n->d_rgb.as<float>(size_t(ns) * 3);
            float* draw = n->d_raw.as<float>(size_t(ns));
            const float3 bg = make_float3(n->cfg.background[0], n->cfg.background[1], n->cfg.background[2]);
            uint32_t* used = n->used.as<uint32_t>(size_t(nr) + 1);
            NFG_HC_CUDA(cudaMemsetAsync(used + nr, 0, 4, st));   // scan sentinel: uoff[nr] = total
            k_composite<<<grid_for(nr * 32), 256, 0, st>>>(static_cast<const uint32_t*>(n->offsets.p),
                                                      static_cast<const uint32_t*>(n->counts.p), nr,
                                                      static_cast<const float*>(n->dens.p), 16,
                                                      static_cast<const float*>(n->rgb.p), tgt, bg, SQRT3 / 1024.0f,
                                                      float(1.0 / (3.0 * double(nr))), nullptr, drgb, draw, ls,
                                                      used);
            NFG_HC_CUDA(cudaGetLastError());
            // second compaction: the backward networks see only contributing samples
            uint32_t* uoff = n->used_off.as<uint32_t>(size_t(nr) + 1);
            size_t tb = 0;
            NFG_HC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, used, uoff, nr + 1, st));
            NFG_HC_CUDA(cub::DeviceScan::ExclusiveSum(n->scan_tmp.get(tb), tb, used, uoff, nr + 1, st));
            // Compacting costs a mid-step sync (the launch sizes need the count):
            // it is done when the previous step found >= 20% of the samples past
            // their ray's transmittance stop (opaque scenes), else the backward
            // runs on all samples (their gradients are zero).
            const char* force = getenv("NFG_NERF_COMPACT");   // "1": always, "0": never (tests, A/B)
            const bool compact = force ? force[0] == '1' : n->last_used_frac < 0.8;
            int64_t nu = ns;
            if (compact) {
                uint32_t h_nu = 0;
                NFG_HC_CUDA(cudaMemcpyAsync(&h_nu, uoff + nr, 4, cudaMemcpyDeviceToHost, st));
                NFG_HC_CUDA(cudaStreamSynchronize(st));
                nu = h_nu;
            }
            NFG_HC_CUDA(cudaMemcpyAsync(n->h_used, uoff + nr, 4, cudaMemcpyDeviceToHost, st));   // read at the end
            const float* bpos = static_cast<const float*>(n->pos.p);
            const float* bY = static_cast<const float*>(n->Yc.p);
            const float* bdrgb = drgb;
            const float* bdraw = draw;
            if (compact && nu < ns) {
                float* pc = n->pos_c.as<float>(size_t(std::max<int64_t>(nu, 1)) * 3);
                float* yc = n->Yc_c.as<float>(size_t(std::max<int64_t>(nu, 1)) * 32);
                float* dc = n->d_rgb_c.as<float>(size_t(std::max<int64_t>(nu, 1)) * 3);
                float* wc = n->d_raw_c.as<float>(size_t(std::max<int64_t>(nu, 1)));
                k_compact_used<<<grid_for(nr * 32), 256, 0, st>>>(static_cast<const uint32_t*>(n->offsets.p), used,
                                                                  uoff, nr, bpos, bY, drgb, draw, pc, yc, dc, wc);
                NFG_HC_CUDA(cudaGetLastError());
                bpos = pc;
                bY = yc;
                bdrgb = dc;
                bdraw = wc;
            }

            if (nu > 0) {
                float* dyc = n->dYc.as<float>(size_t(nu) * 32);
                ok(nfg_mlp_backward_device(n->color, bY, nu, bdrgb, dyc));
                float* dd = n->d_dens.as<float>(size_t(nu) * 16);
                k_density_grad<<<grid_for(nu), 256, 0, st>>>(dyc, bdraw, nu, dd);
                NFG_HC_CUDA(cudaGetLastError());
                ok(nfg_field_backward_device(n->density, bpos, nu, dd));
            }
            n->adam_pending = true;   // enqueued by the next call (flush_adam)
        }
        double h = 0.0;
        NFG_HC_CUDA(cudaMemcpyAsync(&h, ls, 8, cudaMemcpyDeviceToHost, st));
        NFG_HC_CUDA(cudaStreamSynchronize(st));
        if (ns > 0) {
            n->last_used_frac = double(*n->h_used) / double(ns);
            if (samples_backward)
                *samples_backward = int64_t(*n->h_used);
        } else if (samples_backward) {
            *samples_backward = 0;
        }
        ok(nfg_field_check(n->color));
        ok(nfg_field_check(n->density));
        if (loss)
            *loss = nr > 0 ? float(h / (3.0 * double(nr))) : 0.0f;
    });
}

nfg_status nfg_nerf_sync(nfg_nerf* n)
{
    return run([&] {
        n->flush_adam();
        NFG_HC_CUDA(cudaStreamSynchronize(n->st));
        ok(nfg_field_check(n->color));
        ok(nfg_field_check(n->density));
    });
}

nfg_status nfg_nerf_update_occupancy(nfg_nerf* n, int64_t step)
{
    return run([&] {
        n->flush_adam();
        n->update_occupancy(step);
        NFG_HC_CUDA(cudaStreamSynchronize(n->st));
    });
}

nfg_status nfg_nerf_render(nfg_nerf* n, const float* cam12, int32_t width, int32_t height, float focal,
                           float* rgb_host)
{
    return run([&] {
        n->flush_adam();
        cudaStream_t st = n->st;
        const int64_t R = int64_t(width) * height;
        Buf cam, rays, color;
        NFG_HC_CUDA(cudaMemcpyAsync(cam.get(48), cam12, 48, cudaMemcpyHostToDevice, st));
        float* rb = rays.as<float>(size_t(R) * 6);
        k_view_rays<<<grid_for(R), 256, 0, st>>>(static_cast<const float*>(cam.p), width, height, focal, rb);
        NFG_HC_CUDA(cudaGetLastError());
        const int64_t budget = int64_t(1) << 31;
        const auto fit = n->march_compact(rb, R, std::min<int64_t>(budget, R * int64_t(n->cfg.max_samples_per_ray)));
        float* out = color.as<float>(size_t(R) * 3);
        if (fit.second > 0)
            n->forward(fit.second);
        const float3 bg = make_float3(n->cfg.background[0], n->cfg.background[1], n->cfg.background[2]);
        k_composite<<<grid_for(fit.first * 32), 256, 0, st>>>(static_cast<const uint32_t*>(n->offsets.p),
                                                         static_cast<const uint32_t*>(n->counts.p), fit.first,
                                                         static_cast<const float*>(n->dens.p), 16,
                                                         static_cast<const float*>(n->rgb.p), nullptr, bg,
                                                         SQRT3 / 1024.0f, 0.0f, out, nullptr, nullptr, nullptr);
        NFG_HC_CUDA(cudaGetLastError());
        NFG_HC_CUDA(cudaMemcpyAsync(rgb_host, out, size_t(R) * 12, cudaMemcpyDeviceToHost, st));
        NFG_HC_CUDA(cudaStreamSynchronize(st));
        ok(nfg_field_check(n->density));
    });
}

nfg_status nfg_nerf_occupancy(nfg_nerf* n, uint8_t* bits_host, float* density_host)
{
    return run([&] {
        if (bits_host)
            NFG_HC_CUDA(cudaMemcpyAsync(bits_host, n->occ_bits.p, OCC_CELLS / 8, cudaMemcpyDeviceToHost, n->st));
        if (density_host)
            NFG_HC_CUDA(cudaMemcpyAsync(density_host, n->occ_grid.p, size_t(OCC_CELLS) * 4, cudaMemcpyDeviceToHost, n->st));
        NFG_HC_CUDA(cudaStreamSynchronize(n->st));
    });
}

nfg_status nfg_nerf_set_occupancy(nfg_nerf* n, const uint8_t* bits_host)
{
    return run([&] {
        NFG_HC_CUDA(cudaMemcpyAsync(n->occ_bits.p, bits_host, OCC_CELLS / 8, cudaMemcpyHostToDevice, n->st));
        NFG_HC_CUDA(cudaStreamSynchronize(n->st));
    });
}

// ---- components on host buffers (tests) -------------------------------------
nfg_status nfg_nerf_march(nfg_ctx* ctx, const float* rays, int64_t n, const uint8_t* bits, int32_t max_steps,
                          uint32_t* counts, float* samples, int64_t cap, int64_t* total)
{
    return run([&] {
        cudaStream_t st = static_cast<cudaStream_t>(nfg_ctx_stream(ctx));
        Buf r, b, c, o, t, P, D;
        NFG_HC_CUDA(cudaMemcpyAsync(r.get(size_t(n) * 24), rays, size_t(n) * 24, cudaMemcpyHostToDevice, st));
        NFG_HC_CUDA(cudaMemcpyAsync(b.get(OCC_CELLS / 8), bits, OCC_CELLS / 8, cudaMemcpyHostToDevice, st));
        uint32_t* cnt = c.as<uint32_t>(size_t(n));
        uint32_t* off = o.as<uint32_t>(size_t(n));
        k_march_count<<<grid_for(n * 32), 256, 0, st>>>(static_cast<const float*>(r.p), n,
                                                   static_cast<const uint8_t*>(b.p), max_steps, cnt);
        size_t tb = 0;
        NFG_HC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, off, n, st));
        NFG_HC_CUDA(cub::DeviceScan::ExclusiveSum(t.get(tb), tb, cnt, off, n, st));
        std::vector<uint32_t> hc(static_cast<size_t>(n)), ho(static_cast<size_t>(n));
        NFG_HC_CUDA(cudaMemcpyAsync(hc.data(), cnt, size_t(n) * 4, cudaMemcpyDeviceToHost, st));
        NFG_HC_CUDA(cudaMemcpyAsync(ho.data(), off, size_t(n) * 4, cudaMemcpyDeviceToHost, st));
        NFG_HC_CUDA(cudaStreamSynchronize(st));
        const int64_t tot = n > 0 ? int64_t(ho[size_t(n) - 1]) + hc[size_t(n) - 1] : 0;
        *total = tot;
        std::copy(hc.begin(), hc.end(), counts);
        if (tot > cap)
            throw std::invalid_argument("nerf_march: sample buffer too small");
        float* pp = P.as<float>(size_t(std::max<int64_t>(tot, 1)) * 3);
        float* dd = D.as<float>(size_t(std::max<int64_t>(tot, 1)) * 3);
        k_march_write<<<grid_for(n * 32), 256, 0, st>>>(static_cast<const float*>(r.p), n, static_cast<const uint8_t*>(b.p),
                                                   max_steps, off, pp, dd);
        NFG_HC_CUDA(cudaGetLastError());
        NFG_HC_CUDA(cudaMemcpyAsync(samples, pp, size_t(tot) * 12, cudaMemcpyDeviceToHost, st));
        NFG_HC_CUDA(cudaStreamSynchronize(st));
    });
}

nfg_status nfg_nerf_composite(nfg_ctx* ctx, int64_t n_rays, const uint32_t* counts, const float* raw,
                              const float* rgb, const float* target, const float* bg, float dt, float* color,
                              float* d_rgb, float* d_raw, double* loss_sum)
{
    return run([&] {
        cudaStream_t st = static_cast<cudaStream_t>(nfg_ctx_stream(ctx));
        std::vector<uint32_t> off(static_cast<size_t>(std::max<int64_t>(n_rays, 1)));
        int64_t ns = 0;
        for (int64_t r = 0; r < n_rays; ++r) {
            off[size_t(r)] = uint32_t(ns);
            ns += counts[r];
        }
        Buf c, o, rw, rg, tg, co, dr, dw, ls;
        NFG_HC_CUDA(cudaMemcpyAsync(c.get(size_t(n_rays) * 4), counts, size_t(n_rays) * 4, cudaMemcpyHostToDevice, st));
        NFG_HC_CUDA(cudaMemcpyAsync(o.get(size_t(n_rays) * 4), off.data(), size_t(n_rays) * 4, cudaMemcpyHostToDevice, st));
        NFG_HC_CUDA(cudaMemcpyAsync(rw.get(size_t(ns) * 4), raw, size_t(ns) * 4, cudaMemcpyHostToDevice, st));
        NFG_HC_CUDA(cudaMemcpyAsync(rg.get(size_t(ns) * 12), rgb, size_t(ns) * 12, cudaMemcpyHostToDevice, st));
        NFG_HC_CUDA(cudaMemcpyAsync(tg.get(size_t(n_rays) * 12), target, size_t(n_rays) * 12, cudaMemcpyHostToDevice, st));
        double* L = ls.as<double>(1);
        NFG_HC_CUDA(cudaMemsetAsync(L, 0, 8, st));
        k_composite<<<grid_for(n_rays * 32), 256, 0, st>>>(
            static_cast<const uint32_t*>(o.p), static_cast<const uint32_t*>(c.p), n_rays, static_cast<const float*>(rw.p),
            1, static_cast<const float*>(rg.p), static_cast<const float*>(tg.p), make_float3(bg[0], bg[1], bg[2]), dt,
            float(1.0 / (3.0 * double(n_rays))), co.as<float>(size_t(n_rays) * 3), dr.as<float>(size_t(ns) * 3),
            dw.as<float>(size_t(ns)), L);
        NFG_HC_CUDA(cudaGetLastError());
        NFG_HC_CUDA(cudaMemcpyAsync(color, co.p, size_t(n_rays) * 12, cudaMemcpyDeviceToHost, st));
        NFG_HC_CUDA(cudaMemcpyAsync(d_rgb, dr.p, size_t(ns) * 12, cudaMemcpyDeviceToHost, st));
        NFG_HC_CUDA(cudaMemcpyAsync(d_raw, dw.p, size_t(ns) * 4, cudaMemcpyDeviceToHost, st));
        NFG_HC_CUDA(cudaMemcpyAsync(loss_sum, L, 8, cudaMemcpyDeviceToHost, st));
        NFG_HC_CUDA(cudaStreamSynchronize(st));
    });
}

nfg_status nfg_nerf_sh4(nfg_ctx* ctx, const float* dirs, int64_t n, float* out)
{
    return run([&] {
        cudaStream_t st = static_cast<cudaStream_t>(nfg_ctx_stream(ctx));
        Buf d, z, y;
        NFG_HC_CUDA(cudaMemcpyAsync(d.get(size_t(n) * 12), dirs, size_t(n) * 12, cudaMemcpyHostToDevice, st));
        NFG_HC_CUDA(cudaMemsetAsync(z.get(size_t(n) * 64), 0, size_t(n) * 64, st));
        float* Y = y.as<float>(size_t(n) * 32);
        k_color_input<<<grid_for(n), 256, 0, st>>>(static_cast<const float*>(z.p), static_cast<const float*>(d.p), n, Y);
        NFG_HC_CUDA(cudaGetLastError());
        std::vector<float> h(static_cast<size_t>(n) * 32);
        NFG_HC_CUDA(cudaMemcpyAsync(h.data(), Y, h.size() * 4, cudaMemcpyDeviceToHost, st));
        NFG_HC_CUDA(cudaStreamSynchronize(st));
        for (int64_t i = 0; i < n; ++i)
            for (int k = 0; k < 16; ++k)
                out[16 * i + k] = h[size_t(32 * i + 16 + k)];
    });
}

nfg_status nfg_nerf_scene_render(nfg_ctx* ctx, const float* cams, int32_t n_views, int32_t width, int32_t height,
                                 float focal, const float* bg, float* rgb)
{
    return run([&] {
        cudaStream_t st = static_cast<cudaStream_t>(nfg_ctx_stream(ctx));
        Buf c, o;
        NFG_HC_CUDA(cudaMemcpyAsync(c.get(size_t(n_views) * 48), cams, size_t(n_views) * 48, cudaMemcpyHostToDevice, st));
        const int64_t n = int64_t(n_views) * width * height;
        float* out = o.as<float>(size_t(n) * 3);
        k_scene_render<<<grid_for(n), 256, 0, st>>>(static_cast<const float*>(c.p), n_views, width, height, focal,
                                                    make_float3(bg[0], bg[1], bg[2]), out);
        NFG_HC_CUDA(cudaGetLastError());
        NFG_HC_CUDA(cudaMemcpyAsync(rgb, out, size_t(n) * 12, cudaMemcpyDeviceToHost, st));
        NFG_HC_CUDA(cudaStreamSynchronize(st));
    });
}

}   // extern "C"
