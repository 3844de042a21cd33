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
#if !defined(NFG_NO_PAIR_LOADS)   // +7% k_infer (3.15e9 -> 3.37e9 queries/s): 25% fewer L1 requests on an L1-bound kernel
    if (F == 2 && sizeof(TT) == 2) {
        // x-adjacent corners whose rows share an aligned 2-row block (levels
        // start on even rows): one 8-byte load instead of two 4-byte loads
#pragma unroll
        for (int c = 0; c < (1 << D); c += 2) {
            const uint32_t r0 = cs.row(c), r1 = cs.row(c + 1);
            if (r1 == (r0 ^ 1u)) {
                const uint2 u = __ldg(reinterpret_cast<const uint2*>(base + size_t(r0 & ~1u) * 2));
                const float2 lo = unpack_half2(u.x), hi = unpack_half2(u.y);
                v[c] = (r0 & 1u) ? hi : lo;
                v[c + 1] = (r0 & 1u) ? lo : hi;
            } else {
                v[c] = Gather<TT>::two(base + size_t(r0) * F);
                v[c + 1] = Gather<TT>::two(base + size_t(r1) * F);
            }
        }
    } else
#endif
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

// ---- asynchronous (cp.async) staged gathers --------------------------------
// The fused training kernel runs one CTA per SM, so it cannot hide the L2
// latency of its corner gathers with warps. Instead each thread issues ALL of
// its corner loads for a tile as cp.async copies into private shared-memory
// slots (no registers held while in flight), waits once, then blends.
template <int F, typename TT>
struct Stage {
    // bytes per staged element: the (col, col+1) feature pair of one corner
    // (F >= 2), or the aligned 4-byte word holding one feature (F == 1)
    static constexpr int SB = (F == 1) ? 4 : 2 * int(sizeof(TT));
};

template <int BYTES>
__device__ __forceinline__ void cp_async(void* smem, const void* gmem)
{
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(s), "l"(gmem), "n"(BYTES));
}

__device__ __forceinline__ void cp_async_wait_all()
{
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// Elements staged per (sample, col-pair): 2^D corners, times 2 levels for F == 1.
template <int D, int F>
struct PairElems {
    static constexpr int NE = (F == 1 ? 2 : 1) << D;
};

// Where a thread's k-th staged element lives. Linear: a private column of a
// CTA-wide staging area (k-th element of every thread in one row). Chunked:
// the same per-warp rows mapped onto shared-memory chunks the warp owns
// exclusively until the end-of-tile barrier (see k_train).
struct SlotsLinear {
    unsigned char* base;   // stage + tid * SB
    int stride;            // bytes between a thread's consecutive elements
    __device__ __forceinline__ unsigned char* ptr(int k) const { return base + k * stride; }
};

template <int ROWS, int ROW_STRIDE, int NCHUNK>
struct SlotsChunked {
    unsigned char* chunk[NCHUNK];   // each holds ROWS element rows, ROW_STRIDE bytes apart
    int lane_off;                   // lane * SB
    __device__ __forceinline__ unsigned char* ptr(int k) const
    {
        return chunk[k / ROWS] + (k % ROWS) * ROW_STRIDE + lane_off;
    }
};

template <int D, int F, typename TT, class Slots>
__device__ __forceinline__ void gather_issue(const GridDev& g, const LevelDev* lvs, const float* x, int col,
                                             const TT* __restrict__ table, const Slots& slots, int k0)
{
    constexpr int SB = Stage<F, TT>::SB;
#pragma unroll
    for (int h = 0; h < (F == 1 ? 2 : 1); ++h) {
        const int l = F == 1 ? col + h : col / F;
        if (l >= g.L)
            continue;
        const LevelDev lv = lvs[l];
        const CornerSet<D> cs = corners_of<D>(g, lv, x);
#pragma unroll
        for (int c = 0; c < (1 << D); ++c) {
            const size_t e = (size_t(lv.row_off) + cs.row(c)) * F + (F == 1 ? 0 : (col % F));
            const TT* src = table + e;
            if (F == 1 && sizeof(TT) == 2)   // aligned 4-byte word holding the half
                src = table + (e & ~size_t(1));
            cp_async<SB>(slots.ptr(k0 + h * (1 << D) + c), src);
        }
    }
}

template <int D, int F, typename TT, class Slots>
__device__ __forceinline__ float2 gather_blend(const GridDev& g, const LevelDev* lvs, const float* x, int col,
                                               const Slots& slots, int k0)
{
    float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
    for (int h = 0; h < (F == 1 ? 2 : 1); ++h) {
        const int l = F == 1 ? col + h : col / F;
        if (l >= g.L)
            continue;
        const LevelDev lv = lvs[l];
        const CornerSet<D> cs = corners_of<D>(g, lv, x);
        float a = 0.0f, b = 0.0f;
#pragma unroll
        for (int c = 0; c < (1 << D); ++c) {
            const unsigned char* s = slots.ptr(k0 + h * (1 << D) + c);
            const float w = cs.weight(c);
            if (F == 1) {
                float v;
                if (sizeof(TT) == 2) {
                    const float2 two = unpack_half2(*reinterpret_cast<const uint32_t*>(s));
                    v = (cs.row(c) + lv.row_off) & 1u ? two.y : two.x;
                } else {
                    v = *reinterpret_cast<const float*>(s);
                }
                a = fmaf(w, v, a);
            } else {
                const float2 v = sizeof(TT) == 2 ? unpack_half2(*reinterpret_cast<const uint32_t*>(s))
                                                 : *reinterpret_cast<const float2*>(s);
                a = fmaf(w, v.x, a);
                b = fmaf(w, v.y, b);
            }
        }
        if (F == 1) {
            if (h == 0)
                acc.x = a;
            else
                acc.y = a;
        } else {
            acc = make_float2(a, b);
        }
    }
    return acc;
}

// ---- lane-pair gathers and reductions (F == 2) -----------------------------
// In the mma fragment layout lanes 2i and 2i+1 own levels l and l+1 (l even)
// of the same two samples. Per (sample, level) of such a pair, the even lane
// handles the corners with x-offset 0 and the odd lane those with x-offset 1,
// so both corners of every x-adjacent pair sit in the SAME warp instruction
// and the L1 merges them when they share a 32-byte sector: 7/8 of pairs for
// fp16 rows, 3/4 for fp32 gradient rows (pi_1 = 1: hashed rows of x and x+1
// differ in the low bits only; dense rows are consecutive). A divergent L1
// access costs per distinct sector (profiles/lsu_r1.md), so this cuts the
// gather sectors per sample from 128 to ~72 and the reductions from ~98 to ~80.
template <int D>
struct LanePair {
    static constexpr int HC = (1 << D) / 2;   // corners per lane and (sample, level)
};

// Register-path lane-pair encode (k_infer): this lane gathers its x-parity
// corners of both levels of the pair, blends them into two partial sums and
// swaps the partner's partial with one shuffle. Every lane of the warp must
// call it (invalid samples with x = 0 and the result discarded).
template <int D, int F, typename TT, bool PC = false, int IP = IP_RUNTIME>
__device__ __forceinline__ float2 encode_pair_lp(const GridDev& g, const LevelDev* lvs, const float* x, int col,
                                                 const TT* __restrict__ table)
{
    static_assert(F == 2, "lane pairs map one level per lane");
    constexpr int HC = LanePair<D>::HC;
    const int par = (col / F) & 1, lb = (col / F) & ~1;
    float2 part[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        part[q] = make_float2(0.0f, 0.0f);
        if (lb + q >= g.L)
            continue;
        const LevelDev lv = lvs[lb + q];
        const CornerSet<D> cs = corners_of<D, PC, IP>(g, lv, x);
        const TT* base = table + size_t(lv.row_off) * F;
        float2 v[HC];
#pragma unroll
        for (int m = 0; m < HC; ++m)
            v[m] = Gather<TT>::two(base + size_t(cs.row(2 * m + par)) * F);
#pragma unroll
        for (int m = 0; m < HC; ++m) {
            const float w = cs.weight(2 * m + par);
            part[q].x = fmaf(w, v[m].x, part[q].x);
            part[q].y = fmaf(w, v[m].y, part[q].y);
        }
    }
    const float2 give = par ? part[0] : part[1];   // the partner level's partial
    const float2 got = make_float2(__shfl_xor_sync(0xffffffffu, give.x, 1), __shfl_xor_sync(0xffffffffu, give.y, 1));
    const float2 own = par ? part[1] : part[0];
    return make_float2(own.x + got.x, own.y + got.y);
}

// Issue this lane's half of the corner loads of levels (l & ~1) and (l | 1):
// slot k0 + q*HC + m holds corner 2m + par of level (l & ~1) + q.
template <int D, int F, typename TT, bool PC = false, int IP = IP_RUNTIME, class Slots>
__device__ __forceinline__ void gather_issue_lp(const GridDev& g, const LevelDev* lvs, const float* x, int col,
                                                const TT* __restrict__ table, const Slots& slots, int k0)
{
    static_assert(F == 2, "lane pairs map one level per lane");
    constexpr int SB = Stage<F, TT>::SB, HC = LanePair<D>::HC;
    const int par = (col / F) & 1, lb = (col / F) & ~1;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        if (lb + q >= g.L)
            continue;
        const LevelDev lv = lvs[lb + q];
        const CornerSet<D> cs = corners_of<D, PC, IP>(g, lv, x);
#pragma unroll
        for (int m = 0; m < HC; ++m)
            cp_async<SB>(slots.ptr(k0 + q * HC + m), table + (size_t(lv.row_off) + cs.row(2 * m + par)) * F);
    }
}

// Blend of this lane's own level: corners of its parity from its own slots,
// the others from the partner lane's (same warp; call after the copies have
// completed on both lanes and a __syncwarp). Same summation order as
// gather_blend.
template <int D, int F, typename TT, bool PC = false, int IP = IP_RUNTIME, class Slots>
__device__ __forceinline__ float2 gather_blend_lp(const GridDev& g, const LevelDev* lvs, const float* x, int col,
                                                  const Slots& slots, int k0)
{
    constexpr int SB = Stage<F, TT>::SB, HC = LanePair<D>::HC;
    const int l = col / F, par = l & 1;
    if (l >= g.L)
        return make_float2(0.0f, 0.0f);
    const LevelDev lv = lvs[l];
    const CornerSet<D> cs = corners_of<D, PC, IP>(g, lv, x);
    const int pdelta = par ? -SB : SB;
    float a = 0.0f, b = 0.0f;
#pragma unroll
    for (int c = 0; c < (1 << D); ++c) {
        const unsigned char* s = slots.ptr(k0 + par * HC + c / 2) + ((c & 1) == par ? 0 : pdelta);
        const float w = cs.weight(c);
        const float2 v = sizeof(TT) == 2 ? unpack_half2(*reinterpret_cast<const uint32_t*>(s))
                                         : *reinterpret_cast<const float2*>(s);
        a = fmaf(w, v.x, a);
        b = fmaf(w, v.y, b);
    }
    return make_float2(a, b);
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
#ifndef NFG_NO_PAIR_RED
    if constexpr (F == 2) {
        // x-adjacent corners (c, c+1) whose rows form an aligned pair {2k, 2k+1}
        // (always at hashed levels with even x since pi_1 = 1, and at dense
        // levels with an even row) share one 16-byte vector reduction.
        const bool odd_base = (lv.row_off & 1u) != 0;
#pragma unroll
        for (int c = 0; c < (1 << D); c += 2) {
            const uint32_t r0 = cs.row(c), r1 = cs.row(c + 1);
            const float w0 = cs.weight(c), w1 = cs.weight(c + 1);
            if (!odd_base && r1 == (r0 ^ 1u)) {
                const bool lo0 = r0 < r1;
                const uint32_t rl = lo0 ? r0 : r1;
                const float wl = lo0 ? w0 : w1, wh = lo0 ? w1 : w0;
                atomicAdd(reinterpret_cast<float4*>(base + size_t(rl) * 2),
                          make_float4(wl * dy.x, wl * dy.y, wh * dy.x, wh * dy.y));
            } else {
                red_add2(base + size_t(r0) * 2, w0 * dy.x, w0 * dy.y);
                red_add2(base + size_t(r1) * 2, w1 * dy.x, w1 * dy.y);
            }
        }
    } else
#endif
    {
#pragma unroll
        for (int c = 0; c < (1 << D); ++c) {
            const float w = cs.weight(c);
            red_add2(base + size_t(cs.row(c)) * F, w * dy.x, w * dy.y);
        }
    }
}

// Lane-pair backward (F == 2): this lane's corner half of levels (l & ~1) and
// (l | 1) of one sample; dy_own is this lane's level gradient, dy_partner the
// partner lane's (exchanged by the caller with __shfl_xor_sync(.., 1)).
template <int D, bool PC = false, int IP = IP_RUNTIME>
__device__ __forceinline__ void scatter_pair_lp(const GridDev& g, const LevelDev* lvs, const float* x, int col,
                                                float2 dy_own, float2 dy_partner, float* __restrict__ grads)
{
    constexpr int F = 2, HC = LanePair<D>::HC;
    const int par = (col / F) & 1, lb = (col / F) & ~1;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        if (lb + q >= g.L)
            continue;
        const LevelDev lv = lvs[lb + q];
        const CornerSet<D> cs = corners_of<D, PC, IP>(g, lv, x);
        const float2 dy = q == par ? dy_own : dy_partner;
        float* base = grads + size_t(lv.row_off) * F;
#pragma unroll
        for (int m = 0; m < HC; ++m) {
            const int c = 2 * m + par;
            const float w = cs.weight(c);
            red_add2(base + size_t(cs.row(c)) * F, w * dy.x, w * dy.y);
        }
    }
}

}   // namespace nfg
