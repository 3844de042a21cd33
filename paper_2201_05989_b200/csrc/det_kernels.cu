// det_kernels.cu — the deterministic-backward option (nfg_options.deterministic).
//
// The reference's encode_backward is single-threaded "so accumulation order is
// fixed" (grid.hpp:274-295: for each level, points ascending, corners
// ascending, grad.col(row) += w * dY), and SPEC.md:139 requires a strictly
// deterministic mode for tests. On the GPU that order is reproduced per row
// instead of serially:
//
//   per level l:  key = row(l, p, c), value = p * 2^d + c      (k_det_keys)
//                 stable radix sort of (key, value)             (CUB)
//                 one thread per run of equal keys adds w*dy in
//                 value order = (p, c) ascending                 (k_det_segsum)
//
// Each row therefore receives exactly the reference's sequence of fp32
// additions (round-to-nearest, no FMA), so for identical dY the table
// gradients are bit-identical to the reference loop — and run-to-run
// reproducible. The MLP gradients and the loss sum of the deterministic path
// are reduced from per-CTA partials in CTA order (k_reduce_partials) instead of
// by float atomics.
#include <algorithm>

#include <cub/device/device_radix_sort.cuh>

#include "encode.cuh"
#include "kernels.h"

namespace nfg {

template <int D>
__global__ void __launch_bounds__(256)
k_det_keys(const GridDev g, LevelDev lv, const float* __restrict__ X, int64_t B, uint32_t* __restrict__ keys,
           uint32_t* __restrict__ vals, const unsigned int* flags)
{
    if (flags && flags[3] != 0u)
        return;
    const int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= B)
        return;
    float x[D];
#pragma unroll
    for (int i = 0; i < D; ++i)
        x[i] = X[p * D + i];
    const CornerSet<D> cs = corners_of<D>(g, lv, x);
    constexpr int NC = 1 << D;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        keys[p * NC + c] = cs.row(c);
        vals[p * NC + c] = uint32_t(p * NC + c);
    }
}

// F == 2: the payload is the contribution itself, w * dy for both features
// (the reference's product, rounded once, no FMA), packed in 64 bits; the
// stable sort keeps equal rows in (p, c) order and the run sum then reads its
// contributions contiguously instead of recomputing corners per element.
template <int D>
__global__ void __launch_bounds__(256)
k_det_keys_contrib(const GridDev g, LevelDev lv, int l, const float* __restrict__ X, int64_t B,
                   const float* __restrict__ dY, uint32_t* __restrict__ keys, unsigned long long* __restrict__ vals,
                   const unsigned int* flags)
{
    if (flags && flags[3] != 0u)
        return;
    const int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= B)
        return;
    float x[D];
#pragma unroll
    for (int i = 0; i < D; ++i)
        x[i] = X[p * D + i];
    const CornerSet<D> cs = corners_of<D>(g, lv, x);
    const int LF = g.L * 2;
    const float dy0 = dY[p * LF + l * 2], dy1 = dY[p * LF + l * 2 + 1];
    constexpr int NC = 1 << D;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        const float w = cs.weight(c);
        keys[p * NC + c] = cs.row(c);
        vals[p * NC + c] = (static_cast<unsigned long long>(__float_as_uint(__fmul_rn(w, dy1))) << 32) |
                           __float_as_uint(__fmul_rn(w, dy0));
    }
}

// All levels in one pass (F == 2): entry (l, p, c) at (l * B + p) * 2^d + c,
// key = (l << lb) | row — one stable sort then orders every level's rows and
// keeps each row's contributions in (p, c) order.
template <int D>
__global__ void __launch_bounds__(256)
k_det_keys_all(const GridDev g, int lb, const float* __restrict__ X, int64_t B, const float* __restrict__ dY,
               uint32_t* __restrict__ keys, unsigned long long* __restrict__ vals, const unsigned int* flags)
{
    if (flags && flags[3] != 0u)
        return;
    const int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= B)
        return;
    float x[D];
#pragma unroll
    for (int i = 0; i < D; ++i)
        x[i] = X[p * D + i];
    const int LF = g.L * 2;
    constexpr int NC = 1 << D;
    for (int l = 0; l < g.L; ++l) {
        const CornerSet<D> cs = corners_of<D>(g, g.lv[l], x);
        const float dy0 = dY[p * LF + l * 2], dy1 = dY[p * LF + l * 2 + 1];
        const int64_t e0 = (int64_t(l) * B + p) * NC;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            const float w = cs.weight(c);
            keys[e0 + c] = (uint32_t(l) << lb) | cs.row(c);
            vals[e0 + c] = (static_cast<unsigned long long>(__float_as_uint(__fmul_rn(w, dy1))) << 32) |
                           __float_as_uint(__fmul_rn(w, dy0));
        }
    }
}

// Run sums over the all-level sort: the level comes from the key's top bits.
__global__ void __launch_bounds__(256)
k_det_segsum_all(const GridDev g, int lb, int64_t n, const uint32_t* __restrict__ keys,
                 const unsigned long long* __restrict__ vals, float* __restrict__ grads, const unsigned int* flags)
{
    if (flags && flags[3] != 0u)
        return;
    const int64_t i0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i0 >= n)
        return;
    const uint32_t key = keys[i0];
    if (i0 > 0 && keys[i0 - 1] == key)
        return;   // not the head of its run
    int64_t end = i0 + 1;
    while (end < n && keys[end] == key)
        ++end;
    const uint32_t l = key >> lb, row = key & ((1u << lb) - 1u);
    float2* dst = reinterpret_cast<float2*>(grads + (size_t(g.lv[l].row_off) + row) * 2);
    float2 acc = *dst;
    int64_t i = i0;
    for (; i + 8 <= end; i += 8) {
        unsigned long long v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k)
            v[k] = vals[i + k];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            acc.x = __fadd_rn(acc.x, __uint_as_float(uint32_t(v[k])));
            acc.y = __fadd_rn(acc.y, __uint_as_float(uint32_t(v[k] >> 32)));
        }
    }
    for (; i < end; ++i) {
        const unsigned long long v = vals[i];
        acc.x = __fadd_rn(acc.x, __uint_as_float(uint32_t(v)));
        acc.y = __fadd_rn(acc.y, __uint_as_float(uint32_t(v >> 32)));
    }
    *dst = acc;
}

// One thread per run of equal rows adds the run's contributions in order
// (round-to-nearest, the reference's sequence); loads are issued 8 ahead.
__global__ void __launch_bounds__(256)
k_det_segsum_contrib(LevelDev lv, int64_t n, const uint32_t* __restrict__ keys,
                     const unsigned long long* __restrict__ vals, float* __restrict__ grads, const unsigned int* flags)
{
    if (flags && flags[3] != 0u)
        return;
    const int64_t i0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i0 >= n)
        return;
    const uint32_t row = keys[i0];
    if (i0 > 0 && keys[i0 - 1] == row)
        return;   // not the head of its run
    int64_t end = i0 + 1;
    while (end < n && keys[end] == row)
        ++end;
    float2* dst = reinterpret_cast<float2*>(grads + (size_t(lv.row_off) + row) * 2);
    float2 acc = *dst;
    int64_t i = i0;
    for (; i + 8 <= end; i += 8) {
        unsigned long long v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k)
            v[k] = vals[i + k];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            acc.x = __fadd_rn(acc.x, __uint_as_float(uint32_t(v[k])));
            acc.y = __fadd_rn(acc.y, __uint_as_float(uint32_t(v[k] >> 32)));
        }
    }
    for (; i < end; ++i) {
        const unsigned long long v = vals[i];
        acc.x = __fadd_rn(acc.x, __uint_as_float(uint32_t(v)));
        acc.y = __fadd_rn(acc.y, __uint_as_float(uint32_t(v >> 32)));
    }
    *dst = acc;
}

template <int D, int F>
__global__ void __launch_bounds__(256)
k_det_segsum(const GridDev g, LevelDev lv, int l, const float* __restrict__ X, int64_t B,
             const float* __restrict__ dY, const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals,
             float* __restrict__ grads, const unsigned int* flags)
{
    if (flags && flags[3] != 0u)
        return;
    constexpr int NC = 1 << D;
    const int64_t n = B * NC;
    const int64_t i0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i0 >= n)
        return;
    const uint32_t row = keys[i0];
    if (i0 > 0 && keys[i0 - 1] == row)
        return;   // not the head of its run
    float* dst = grads + (size_t(lv.row_off) + row) * F;
    float acc[F];
#pragma unroll
    for (int f = 0; f < F; ++f)
        acc[f] = dst[f];
    const int LF = g.L * F;
    for (int64_t i = i0; i < n && keys[i] == row; ++i) {
        const uint32_t v = vals[i];
        const int64_t p = v / NC;
        const int c = int(v % NC);
        float x[D];
#pragma unroll
        for (int k = 0; k < D; ++k)
            x[k] = X[p * D + k];
        const float w = corners_of<D>(g, lv, x).weight(c);
#pragma unroll
        for (int f = 0; f < F; ++f)
            acc[f] = __fadd_rn(acc[f], __fmul_rn(w, dY[p * LF + l * F + f]));
    }
#pragma unroll
    for (int f = 0; f < F; ++f)
        dst[f] = acc[f];
}

// Sums per-CTA partials in CTA order: out[i] += sum_c part[c * n + i]; the
// loss partials likewise into *loss_sum.
__global__ void __launch_bounds__(256)
k_reduce_partials(const float* __restrict__ part, int nparts, int64_t n, float* __restrict__ out,
                  const double* __restrict__ part_loss, int nloss, double* loss_sum, const unsigned int* flags)
{
    if (flags && flags[3] != 0u)
        return;
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) {
        float s = 0.0f;
        for (int c = 0; c < nparts; ++c)
            s = __fadd_rn(s, part[int64_t(c) * n + i]);
        out[i] = __fadd_rn(out[i], s);
    }
    if (part_loss && i == 0) {
        double s = 0.0;
        for (int k = 0; k < nloss; ++k)
            s += part_loss[k];
        *loss_sum += s;
    }
}

static int bits_for(uint64_t n)
{
    int b = 1;
    while (b < 32 && (uint64_t(1) << b) < n)
        ++b;
    return b;
}

size_t encode_bwd_det_scratch(int64_t B, int d, int L)
{
    const size_t n = (size_t(B) << d) * size_t(L);   // all levels (F == 2); a per-level sort needs less
    size_t cub32 = 0, cub64 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, cub32, static_cast<const uint32_t*>(nullptr),
                                    static_cast<uint32_t*>(nullptr), static_cast<const uint32_t*>(nullptr),
                                    static_cast<uint32_t*>(nullptr), n, 0, 32);
    cub::DeviceRadixSort::SortPairs(nullptr, cub64, static_cast<const uint32_t*>(nullptr),
                                    static_cast<uint32_t*>(nullptr), static_cast<const unsigned long long*>(nullptr),
                                    static_cast<unsigned long long*>(nullptr), n, 0, 32);
    // keys x 2 + 64-bit payloads x 2 (the F != 2 path uses 32-bit payloads in the same space)
    return 6 * n * sizeof(uint32_t) + ((std::max(cub32, cub64) + 255) & ~size_t(255));
}

template <int D, int F>
static cudaError_t enc_bwd_det(const FieldShape& s, const LevelDev* lv, const float* X, int64_t B, const float* dY,
                               float* grads, const unsigned int* flags, void* scratch, size_t bytes, cudaStream_t st)
{
    (void)lv;
    const size_t n = size_t(B) << D;
    const unsigned blocks_p = unsigned((B + 255) / 256), blocks_n = unsigned((n + 255) / 256);
    if constexpr (F == 2) {
        // one sort over every level: key = (level << lb) | row
        int lb = 1;
        for (int l = 0; l < s.grid.L; ++l)
            lb = std::max(lb, bits_for(s.grid.lv[l].len));
        const int kb = lb + bits_for(uint64_t(s.grid.L));
        const size_t na = n * size_t(s.grid.L);
        if (kb <= 32 && na < (size_t(1) << 31)) {
            uint32_t* k0 = static_cast<uint32_t*>(scratch);
            uint32_t* k1 = k0 + na;
            unsigned long long* v0 = reinterpret_cast<unsigned long long*>(k1 + na);   // 8-byte aligned: na even
            unsigned long long* v1 = v0 + na;
            void* tmp = v1 + na;
            size_t tmp_bytes = bytes - 6 * na * sizeof(uint32_t);
            k_det_keys_all<D><<<blocks_p, 256, 0, st>>>(s.grid, lb, X, B, dY, k0, v0, flags);
            cudaError_t e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k0, k1, v0, v1, na, 0, kb, st);
            if (e != cudaSuccess)
                return e;
            k_det_segsum_all<<<unsigned((na + 255) / 256), 256, 0, st>>>(s.grid, lb, int64_t(na), k1, v1, grads,
                                                                          flags);
            return cudaGetLastError();
        }
        uint32_t* k0 = static_cast<uint32_t*>(scratch);
        uint32_t* k1 = k0 + n;
        unsigned long long* v0 = reinterpret_cast<unsigned long long*>(k1 + n);   // 8-byte aligned: n even
        unsigned long long* v1 = v0 + n;
        void* tmp = v1 + n;
        size_t tmp_bytes = bytes - 6 * n * sizeof(uint32_t);
        for (int l = 0; l < s.grid.L; ++l) {
            const LevelDev L = s.grid.lv[l];
            k_det_keys_contrib<D><<<blocks_p, 256, 0, st>>>(s.grid, L, l, X, B, dY, k0, v0, flags);
            cudaError_t e =
                cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k0, k1, v0, v1, n, 0, bits_for(L.len), st);
            if (e != cudaSuccess)
                return e;
            k_det_segsum_contrib<<<blocks_n, 256, 0, st>>>(L, int64_t(n), k1, v1, grads, flags);
        }
        return cudaGetLastError();
    }
    uint32_t* k0 = static_cast<uint32_t*>(scratch);
    uint32_t* v0 = k0 + n;
    uint32_t* k1 = v0 + n;
    uint32_t* v1 = k1 + n;
    void* tmp = v1 + n;
    size_t tmp_bytes = bytes - 4 * n * sizeof(uint32_t);
    for (int l = 0; l < s.grid.L; ++l) {
        const LevelDev L = s.grid.lv[l];
        k_det_keys<D><<<blocks_p, 256, 0, st>>>(s.grid, L, X, B, k0, v0, flags);
        cudaError_t e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k0, k1, v0, v1, n, 0, bits_for(L.len), st);
        if (e != cudaSuccess)
            return e;
        k_det_segsum<D, F><<<blocks_n, 256, 0, st>>>(s.grid, L, l, X, B, dY, k1, v1, grads, flags);
    }
    return cudaGetLastError();
}

cudaError_t launch_encode_bwd_det(const FieldShape& s, const LevelDev* lv, const float* X, int64_t B,
                                  const float* dY, float* grads, const unsigned int* flags, void* scratch,
                                  size_t bytes, cudaStream_t st)
{
    if (B <= 0)
        return cudaSuccess;
    if ((uint64_t(B) << s.grid.d) > (uint64_t(1) << 31))
        return cudaErrorInvalidValue;
    if (bytes < encode_bwd_det_scratch(B, s.grid.d, s.grid.L))
        return cudaErrorInvalidValue;
#define NFG_DET_B(D_, F_)                                                                                   \
    if (s.grid.d == D_ && s.grid.F == F_)                                                                    \
        return enc_bwd_det<D_, F_>(s, lv, X, B, dY, grads, flags, scratch, bytes, st);
    NFG_DET_B(2, 1) NFG_DET_B(2, 2) NFG_DET_B(2, 4) NFG_DET_B(2, 8)
    NFG_DET_B(3, 1) NFG_DET_B(3, 2) NFG_DET_B(3, 4) NFG_DET_B(3, 8)
#undef NFG_DET_B
    return cudaErrorNotSupported;
}

cudaError_t launch_reduce_partials(const float* part, int nparts, int64_t n, float* out, const double* part_loss,
                                   int nloss, double* loss_sum, const unsigned int* flags, cudaStream_t st)
{
    const int64_t blocks = std::max<int64_t>(1, (n + 255) / 256);
    k_reduce_partials<<<unsigned(blocks), 256, 0, st>>>(part, nparts, n, out, part_loss, nloss, loss_sum, flags);
    return cudaGetLastError();
}

}   // namespace nfg
