// diag.cu — live L2-level throughput peaks for the roofline (nfg_diag_l2_peak).
//
// The hash-grid hot path is neither HBM- nor tensor-bound at T <= 2^19: its
// tables (fp16, 24 MB at config 2) and fp32 gradients (49 MB) stay in the
// 126 MB L2, and every corner gather / gradient reduction is a divergent
// 4-8 byte access to its own 32-byte sector (grid.hpp:245-271, 286-294). The
// honest denominator is therefore the chip's throughput for exactly that
// access, measured on this GPU at full occupancy with an L2-resident footprint:
//   op 0: random 4 B loads, L1 bypassed (ld.global.cg): L2 sector reads
//   op 1: random 4 B cp.async.ca (k_train's gather instruction)
//   op 2: random red.global.add.v2.f32 on 8-byte aligned pairs (k_train's scatter)
//   op 3: coalesced 16 B/lane loads, L1 bypassed: streaming L2 read bandwidth
//   op 4: random 4 B ld.global.nc (k_infer's gather instruction)
// Result: sectors per second (ops 0-2, 4: one 32-byte sector per lane-op),
// bytes per second for op 3. bench.py divides k_train's and k_infer's
// algorithmic sector bytes by these rates.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/nfg.h"

namespace nfg {
namespace {

constexpr int TPB = 256;
constexpr int UNROLL = 8;

__device__ __forceinline__ uint32_t mix32(uint32_t x)
{
    x ^= x >> 16;
    x *= 0x7feb352dU;
    x ^= x >> 15;
    x *= 0x846ca68bU;
    x ^= x >> 16;
    return x;
}

template <int OP>
__global__ void __launch_bounds__(TPB) k_l2_peak(const uint32_t* __restrict__ table, float* grads, uint32_t mask_words,
                                                 int iters, uint32_t* sink)
{
    __shared__ __align__(16) uint32_t stage[UNROLL * TPB];
    const uint32_t tid = blockIdx.x * TPB + threadIdx.x;
    uint32_t acc = 0;
    uint32_t s = mix32(tid * 0x9E3779B9u + 1u);
    if constexpr (OP == 3) {
        const uint32_t nthreads = gridDim.x * TPB;
        const uint32_t n4 = (mask_words + 1u) / 4u;
        const uint4* t4 = reinterpret_cast<const uint4*>(table);
        for (int it = 0; it < iters; ++it)
            for (uint32_t i = tid; i < n4; i += nthreads) {
                uint4 v;
                asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                             : "l"(t4 + i));
                acc ^= v.x ^ v.y ^ v.z ^ v.w;
            }
    } else {
        for (int it = 0; it < iters; ++it) {
            uint32_t a[UNROLL];
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {
                s = mix32(s + u);
                a[u] = s & mask_words;
            }
            if constexpr (OP == 0 || OP == 4) {
#pragma unroll
                for (int u = 0; u < UNROLL; ++u) {
                    uint32_t v;
                    if (OP == 0)
                        asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(table + a[u]));
                    else
                        asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(table + a[u]));
                    acc += v;
                }
            } else if constexpr (OP == 1) {
#pragma unroll
                for (int u = 0; u < UNROLL; ++u) {
                    const uint32_t dst = uint32_t(__cvta_generic_to_shared(&stage[u * TPB + threadIdx.x]));
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(table + a[u]) : "memory");
                }
                asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
#pragma unroll
                for (int u = 0; u < UNROLL; ++u)
                    acc += stage[u * TPB + threadIdx.x];
            } else {
#pragma unroll
                for (int u = 0; u < UNROLL; ++u) {
                    float* p = grads + ((a[u] << 1) & (2u * mask_words + 1u) & ~1u);
                    asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(1.0f), "f"(2.0f) : "memory");
                }
            }
        }
    }
    if (acc == 0x12345678u)
        sink[0] = acc;
}

template <int OP>
cudaError_t run_peak(const uint32_t* table, float* grads, uint32_t words, int sms, cudaStream_t st, double* rate)
{
    int occ = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_l2_peak<OP>, TPB, 0);
    if (e != cudaSuccess)
        return e;
    const int grid = sms * (occ > 0 ? occ : 1);
    const int iters = OP == 3 ? 4 : 64;
    k_l2_peak<OP><<<grid, TPB, 0, st>>>(table, grads, words - 1u, OP == 3 ? 1 : 4,
                                        reinterpret_cast<uint32_t*>(grads));   // warm L2
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0, st);
        k_l2_peak<OP><<<grid, TPB, 0, st>>>(table, grads, words - 1u, iters, reinterpret_cast<uint32_t*>(grads));
        cudaEventRecord(e1, st);
        if ((e = cudaEventSynchronize(e1)) != cudaSuccess)
            break;
        float ms = 0.0f;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (e != cudaSuccess)
        return e;
    const double work = OP == 3 ? double(words) * 4.0 * iters : double(grid) * TPB * iters * UNROLL;
    *rate = work / (double(best) * 1e-3);
    return cudaGetLastError();
}

}   // namespace
}   // namespace nfg

extern "C" nfg_status nfg_diag_l2_peak(nfg_ctx* ctx, int32_t op, double* rate)
{
    if (!ctx || !rate || op < 0 || op > 4)
        return NFG_EINVAL;
    cudaStream_t st = static_cast<cudaStream_t>(nfg_ctx_stream(ctx));
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint32_t words = 1u << 23;   // 32 MB of 4-byte rows + 64 MB of fp32 pairs: config 2's footprint
    uint32_t* table = nullptr;
    float* grads = nullptr;
    if (cudaMalloc(&table, size_t(words) * 4) != cudaSuccess)
        return NFG_ECUDA;
    if (cudaMalloc(&grads, size_t(words) * 8) != cudaSuccess) {
        cudaFree(table);
        return NFG_ECUDA;
    }
    cudaMemsetAsync(table, 1, size_t(words) * 4, st);
    cudaMemsetAsync(grads, 0, size_t(words) * 8, st);
    cudaError_t e = cudaErrorInvalidValue;
    switch (op) {
    case 0: e = nfg::run_peak<0>(table, grads, words, sms, st, rate); break;
    case 1: e = nfg::run_peak<1>(table, grads, words, sms, st, rate); break;
    case 2: e = nfg::run_peak<2>(table, grads, words, sms, st, rate); break;
    case 3: e = nfg::run_peak<3>(table, grads, words, sms, st, rate); break;
    case 4: e = nfg::run_peak<4>(table, grads, words, sms, st, rate); break;
    }
    cudaStreamSynchronize(st);
    cudaFree(table);
    cudaFree(grads);
    return e == cudaSuccess ? NFG_OK : NFG_ECUDA;
}
