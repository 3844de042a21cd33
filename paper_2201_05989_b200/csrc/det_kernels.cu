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

size_t encode_bwd_det_scratch(int64_t B, int d)
{
    const size_t n = size_t(B) << d;
    size_t cub_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, static_cast<const uint32_t*>(nullptr),
                                    static_cast<uint32_t*>(nullptr), static_cast<const uint32_t*>(nullptr),
                                    static_cast<uint32_t*>(nullptr), n, 0, 32);
    return 4 * n * sizeof(uint32_t) + ((cub_bytes + 255) & ~size_t(255));
}

template <int D, int F>
static cudaError_t enc_bwd_det(const FieldShape& s, const LevelDev* lv, const float* X, int64_t B, const float* dY,
                               float* grads, const unsigned int* flags, void* scratch, size_t bytes, cudaStream_t st)
{
    (void)lv;
    const size_t n = size_t(B) << D;
    uint32_t* k0 = static_cast<uint32_t*>(scratch);
    uint32_t* v0 = k0 + n;
    uint32_t* k1 = v0 + n;
    uint32_t* v1 = k1 + n;
    void* tmp = v1 + n;
    size_t tmp_bytes = bytes - 4 * n * sizeof(uint32_t);
    const unsigned blocks_p = unsigned((B + 255) / 256), blocks_n = unsigned((n + 255) / 256);
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
    if (bytes < encode_bwd_det_scratch(B, s.grid.d))
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
