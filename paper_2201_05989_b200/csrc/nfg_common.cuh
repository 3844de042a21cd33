// nfg_common.cuh — shared device-side definitions for the sm_100a kernels.
//
// The grid-encoding arithmetic here restates grid.hpp:88-133,199-212 of the
// reference with explicit IEEE round-to-nearest intrinsics (__fmul_rn,
// __fadd_rn, __fsub_rn) so nvcc cannot contract it into FMAs: vertex selection
// (corner + row index) and the interpolation weights are bit-identical to the
// reference's fp32 path.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define NFG_MAX_LEVELS 32

namespace nfg {

// One level of the multiresolution grid as the kernels see it. Built on the
// host from level_resolutions (grid.hpp:66-84) and passed by value.
struct LevelDev {
    uint32_t res;       // N_l
    float res_f;        // float(N_l), the reference's Scalar(resolution)
    uint32_t stride;    // N_l + 1 (dense levels)
    uint32_t dense;     // (N_l+1)^d <= T
    uint32_t row_off;   // first row of this level in the flat table
    uint32_t len;       // rows at this level
};

struct GridDev {
    int32_t L;
    int32_t F;
    int32_t d;
    int32_t smooth;     // Interpolation::Smoothstep
    uint32_t mask;      // T - 1
    LevelDev lv[NFG_MAX_LEVELS];
};

// The clamp of grid.hpp:199-201 (NaN -> 0, as fmaxf returns the number).
__device__ __forceinline__ float clamp_unit(float x) { return fminf(fmaxf(x, 0.0f), 1.0f - 0x1p-20f); }

// Clamp, scale, optional half-voxel offset, floor (grid.hpp:199-212). PC: x was
// already clamped once per sample (clamp_x), so the per-level clamp is skipped
// (clamping is idempotent: bit-identical corners and fractions).
template <bool PC = false>
__device__ __forceinline__ void voxel_of(float x, float n, bool half, uint32_t& corner, float& frac)
{
    float p = __fmul_rn(PC ? x : clamp_unit(x), n);
    if (half)
        p = fminf(__fadd_rn(p, 0.5f), __fmul_rn(n, 1.0f - 0x1p-20f));
    const float f = floorf(p);
    corner = static_cast<uint32_t>(f);
    frac = __fsub_rn(p, f);
}

// smoothstep1 (grid.hpp:112-116): (x*x) * (3 - 2x), no contraction.
__device__ __forceinline__ float smoothstep1(float x)
{
    return __fmul_rn(__fmul_rn(x, x), __fsub_rn(3.0f, __fmul_rn(2.0f, x)));
}

// Per-dimension partial indices of the two candidate corners along each
// axis; corner c's row is a combination selected by the bits of c. For hashed
// levels the combination is XOR of prime products (grid.hpp:88-95, pi_1 = 1),
// for dense levels the row-major sum (grid.hpp:100-110) — both identical to
// the reference's per-corner evaluation.
template <int D>
struct CornerSet {
    uint32_t lo[D], hi[D];
    float t[D];   // interpolation parameter per axis (frac or smoothstep(frac))
    uint32_t dense, mask;

    __device__ __forceinline__ uint32_t row(int c) const
    {
        uint32_t r = (c & 1) ? hi[0] : lo[0];
#pragma unroll
        for (int i = 1; i < D; ++i) {
            const uint32_t v = ((c >> i) & 1) ? hi[i] : lo[i];
            r = dense ? r + v : (r ^ v);
        }
        return dense ? r : (r & mask);
    }

    // interpolation_weights (grid.hpp:120-133): w = ((1*a0)*a1)*a2.
    __device__ __forceinline__ float weight(int c) const
    {
        float w = (c & 1) ? t[0] : __fsub_rn(1.0f, t[0]);
#pragma unroll
        for (int i = 1; i < D; ++i)
            w = __fmul_rn(w, ((c >> i) & 1) ? t[i] : __fsub_rn(1.0f, t[i]));
        return w;
    }
};

template <int D>
__device__ __forceinline__ void clamp_x(float* x)
{
#pragma unroll
    for (int i = 0; i < D; ++i)
        x[i] = clamp_unit(x[i]);
}

// IP: interpolation known at compile time (IP_LINEAR / IP_SMOOTH), or read from
// the grid at run time (IP_RUNTIME; both variants are then computed and one is
// selected per axis).
enum { IP_RUNTIME = 0, IP_LINEAR = 1, IP_SMOOTH = 2 };

template <int D, bool PC = false, int IP = IP_RUNTIME>
__device__ __forceinline__ CornerSet<D> corners_of(const GridDev& g, const LevelDev& lv, const float* x)
{
    CornerSet<D> cs;
    cs.dense = lv.dense;
    cs.mask = g.mask;
    const uint32_t primes[3] = { 1u, 2654435761u, 805459861u };
    uint32_t mul = 1u;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        uint32_t c;
        float fr;
        const bool smooth = IP == IP_RUNTIME ? g.smooth != 0 : IP == IP_SMOOTH;
        voxel_of<PC>(x[i], lv.res_f, smooth, c, fr);
        cs.t[i] = smooth ? smoothstep1(fr) : fr;
        if (lv.dense) {
            cs.lo[i] = c * mul;
            cs.hi[i] = (c + 1u) * mul;
            mul *= lv.stride;
        } else {
            cs.lo[i] = c * primes[i];
            cs.hi[i] = (c + 1u) * primes[i];
        }
    }
    return cs;
}

// ---- small helpers ------------------------------------------------------
__device__ __forceinline__ uint32_t pack_half2(float a, float b)
{
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ float2 unpack_half2(uint32_t v)
{
    __half2 h = *reinterpret_cast<__half2*>(&v);
    return __half22float2(h);
}

__device__ __forceinline__ bool finite_f(float x) { return (__float_as_uint(x) & 0x7f800000u) != 0x7f800000u; }

}   // namespace nfg
