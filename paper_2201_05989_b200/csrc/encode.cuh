// encode.cuh — per-(sample, level) gather / scatter of the hash-grid encoding.
//
// encode_pair restates the forward blend of grid.hpp:245-271 for one sample
// and one pair of output columns; scatter_pair restates the backward scatter of
// grid.hpp:286-294. The "pair" granularity matches the mma.sync fragment
// ownership (a lane owns columns 2t, 2t+1 of a k16 block), so the fused kernels
// encode straight into A fragments and scatter straight out of C fragments.
#pragma once

#include "nfg_common.cuh"

namespace nfg {

template <typename TT>
struct Gather;

template <>
struct Gather<__half> {
    __device__ __forceinline__ static float one(const __half* p) { return __half2float(__ldg(p)); }
    __device__ __forceinline__ static float2 two(const __half* p)
    {
        const uint32_t u = __ldg(reinterpret_cast<const unsigned int*>(p));
        return unpack_half2(u);
    }
};

template <>
struct Gather<float> {
    __device__ __forceinline__ static float one(const float* p) { return __ldg(p); }
    __device__ __forceinline__ static float2 two(const float* p) { return __ldg(reinterpret_cast<const float2*>(p)); }
};

// Feature `fo` (F == 1) of level l at x: one scalar.
template <int D, int F, typename TT>
__device__ __forceinline__ float encode_one(const GridDev& g, const LevelDev* lvs, const float* x, int l,
                                            const TT* __restrict__ table)
{
    if (l >= g.L)
        return 0.0f;
    const LevelDev lv = lvs[l];
    const CornerSet<D> cs = corners_of<D>(g, lv, x);
    const TT* base = table + size_t(lv.row_off) * F;
    float acc = 0.0f;
#pragma unroll
    for (int c = 0; c < (1 << D); ++c)
        acc = fmaf(cs.weight(c), Gather<TT>::one(base + size_t(cs.row(c)) * F), acc);
    return acc;
}

// Output columns (col, col+1) of the (L*F)-wide encoding of one sample.
template <int D, int F, typename TT>
__device__ __forceinline__ float2 encode_pair(const GridDev& g, const LevelDev* lvs, const float* x, int col,
                                              const TT* __restrict__ table)
{
    if (F == 1)
        return make_float2(encode_one<D, F, TT>(g, lvs, x, col, table),
                           encode_one<D, F, TT>(g, lvs, x, col + 1, table));
    const int l = col / F;
    float2 acc = make_float2(0.0f, 0.0f);
    if (l >= g.L)
        return acc;
    const LevelDev lv = lvs[l];
    const CornerSet<D> cs = corners_of<D>(g, lv, x);
    const TT* base = table + size_t(lv.row_off) * F + (col % F);
    float2 v[1 << D];
#pragma unroll
    for (int c = 0; c < (1 << D); ++c)
        v[c] = Gather<TT>::two(base + size_t(cs.row(c)) * F);
#pragma unroll
    for (int c = 0; c < (1 << D); ++c) {
        const float w = cs.weight(c);
        acc.x = fmaf(w, v[c].x, acc.x);
        acc.y = fmaf(w, v[c].y, acc.y);
    }
    return acc;
}

__device__ __forceinline__ void red_add2(float* p, float a, float b)
{
    // vector reduction to global memory (sm_90+): one L2 atomic for both features
    atomicAdd(reinterpret_cast<float2*>(p), make_float2(a, b));
}

// Backward of encode_pair: grads[row] += w_c * dy for each corner.
template <int D, int F>
__device__ __forceinline__ void scatter_pair(const GridDev& g, const LevelDev* lvs, const float* x, int col,
                                             float2 dy, float* __restrict__ grads)
{
    if (F == 1) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int l = col + h;
            if (l >= g.L)
                continue;
            const LevelDev lv = lvs[l];
            const CornerSet<D> cs = corners_of<D>(g, lv, x);
            float* base = grads + size_t(lv.row_off);
            const float v = h ? dy.y : dy.x;
#pragma unroll
            for (int c = 0; c < (1 << D); ++c)
                atomicAdd(base + cs.row(c), cs.weight(c) * v);
        }
        return;
    }
    const int l = col / F;
    if (l >= g.L)
        return;
    const LevelDev lv = lvs[l];
    const CornerSet<D> cs = corners_of<D>(g, lv, x);
    float* base = grads + size_t(lv.row_off) * F + (col % F);
#pragma unroll
    for (int c = 0; c < (1 << D); ++c) {
        const float w = cs.weight(c);
        red_add2(base + size_t(cs.row(c)) * F, w * dy.x, w * dy.y);
    }
}

}   // namespace nfg
