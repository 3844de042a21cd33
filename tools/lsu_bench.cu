// lsu_bench.cu — the throughput ceiling of k_train's memory instructions.
// k_train's table traffic is L2-resident (tables 32 MB fp16 + grads 64 MB fp32
// at config 2), so HBM does not bound it. What bounds it is the per-SM rate of
// DIVERGENT lane operations: every 4-byte corner gather and every v2/v4
// gradient reduction goes to its own 32-byte sector. This tool measures that
// rate at full occupancy on uniformly random L2-resident addresses:
//   cp.async 4 B (k_train's gather), ld.global 4 B / 8 B (k_infer's),
//   red.global.add.v2.f32 / .v4.f32 (k_train's scatter).
// It reports ns per lane-op per SM, which tools/ncu counts turn into a bound.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/lsu_bench.cu -o tools/lsu_bench
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                                        \
    do {                                                                                             \
        cudaError_t e = (x);                                                                         \
        if (e != cudaSuccess) {                                                                      \
            std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);      \
            std::exit(1);                                                                            \
        }                                                                                            \
    } while (0)

constexpr int TPB = 256;
constexpr int UNROLL = 8;

__device__ __forceinline__ uint32_t mix(uint32_t x)
{
    x ^= x >> 16;
    x *= 0x7feb352dU;
    x ^= x >> 15;
    x *= 0x846ca68bU;
    x ^= x >> 16;
    return x;
}

template <int OP>   // 0: cp.async 4 B, 1: ld 4 B, 2: ld 8 B, 3: red v2.f32, 4: red v4.f32,
                    // 5: ld 4 B on even lanes only, 6: ld 4 B with lane pairs sharing a sector,
                    // 7: red v2 on even lanes only, 8: red v2 with lane pairs sharing a sector,
                    // 9: cp.async 8 B, 10: cp.async 16 B, 11: cp.async 4 B on even lanes only,
                    // 12: ld 16 B, 13: ld 32 B (LDG.256),
                    // 14: cp.async 4 B, lane pairs in one sector (adjacent words),
                    // 15: red v2, lane pairs in one sector but different 16-byte halves,
                    // 16: cp.async 4 B, lane pairs at the two ends of one sector
__global__ void __launch_bounds__(TPB) k_lsu(uint32_t* table, float* grads, uint32_t mask_words, int iters,
                                             uint32_t* sink)
{
    extern __shared__ __align__(16) uint32_t stage_raw[];   // cp.async variants: UNROLL x TPB x (SZ/4) words
    const uint32_t tid = blockIdx.x * TPB + threadIdx.x;
    uint32_t acc = 0;
    uint32_t s = mix(tid * 0x9E3779B9u + 1u);
    for (int it = 0; it < iters; ++it) {
        uint32_t a[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            s = mix(s + u);
            a[u] = s & mask_words;
        }
        if constexpr (OP == 0) {
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {
                const uint32_t dst = uint32_t(__cvta_generic_to_shared(&stage_raw[u * TPB + threadIdx.x]));
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(table + a[u]) : "memory");
            }
            asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
#pragma unroll
            for (int u = 0; u < UNROLL; ++u)
                acc += stage_raw[u * TPB + threadIdx.x];
        } else if constexpr (OP == 9 || OP == 10 || OP == 11) {
            constexpr int SZ = OP == 9 ? 8 : OP == 10 ? 16 : 4;
            if (OP != 11 || (threadIdx.x & 1) == 0) {
#pragma unroll
                for (int u = 0; u < UNROLL; ++u) {
                    const uint32_t dst = uint32_t(__cvta_generic_to_shared(&stage_raw[(u * TPB + threadIdx.x) * (SZ / 4)]));
                    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(dst),
                                 "l"(table + (a[u] & ~uint32_t(SZ / 4 - 1))), "n"(SZ)
                                 : "memory");
                }
            }
            asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
#pragma unroll
            for (int u = 0; u < UNROLL; ++u)
                acc += stage_raw[(u * TPB + threadIdx.x) * (SZ / 4)];
        } else if constexpr (OP == 14 || OP == 16) {
            const uint32_t other = threadIdx.x & 1;
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {
                const uint32_t b = __shfl_sync(0xffffffffu, a[u], (threadIdx.x & 31) & ~1u);
                const uint32_t wi = OP == 14 ? ((b & ~1u) | other) : ((b & ~7u) | (other * 7u));
                const uint32_t dst = uint32_t(__cvta_generic_to_shared(&stage_raw[u * TPB + threadIdx.x]));
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(table + wi) : "memory");
            }
            asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
#pragma unroll
            for (int u = 0; u < UNROLL; ++u)
                acc += stage_raw[u * TPB + threadIdx.x];
        } else if constexpr (OP == 15) {
            const uint32_t other = threadIdx.x & 1;
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {
                const uint32_t b = __shfl_sync(0xffffffffu, a[u], (threadIdx.x & 31) & ~1u);
                float* p = grads + ((((b << 1) & (2 * mask_words + 1)) & ~7u) | (other << 2));
                asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(1.0f), "f"(2.0f) : "memory");
            }
        } else if constexpr (OP == 12) {
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(table + (a[u] & ~3u)));
                acc += v.x ^ v.y ^ v.z ^ v.w;
            }
        } else if constexpr (OP == 13) {
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {
                uint32_t r[8];
                asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                             : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                               "=r"(r[7])
                             : "l"(table + (a[u] & ~7u)));
                acc += r[0] ^ r[1] ^ r[2] ^ r[3] ^ r[4] ^ r[5] ^ r[6] ^ r[7];
            }
        } else if constexpr (OP == 1) {
#pragma unroll
            for (int u = 0; u < UNROLL; ++u)
                acc += __ldg(table + a[u]);
        } else if constexpr (OP == 2) {
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {
                const uint2 v = __ldg(reinterpret_cast<const uint2*>(table + (a[u] & ~1u)));
                acc += v.x ^ v.y;
            }
        } else if constexpr (OP == 3) {
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {
                float* p = grads + ((a[u] << 1) & (2 * mask_words + 1) & ~1u);
                asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(1.0f), "f"(2.0f) : "memory");
            }
        } else if constexpr (OP == 5) {
            if ((threadIdx.x & 1) == 0) {
#pragma unroll
                for (int u = 0; u < UNROLL; ++u)
                    acc += __ldg(table + a[u]);
            }
        } else if constexpr (OP == 6) {
            const uint32_t other = threadIdx.x & 1;
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {
                const uint32_t b = __shfl_sync(0xffffffffu, a[u], (threadIdx.x & 31) & ~1u);
                acc += __ldg(table + ((b & ~1u) | other));
            }
        } else if constexpr (OP == 7) {
            if ((threadIdx.x & 1) == 0) {
#pragma unroll
                for (int u = 0; u < UNROLL; ++u) {
                    float* p = grads + ((a[u] << 1) & (2 * mask_words + 1) & ~1u);
                    asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(1.0f), "f"(2.0f) : "memory");
                }
            }
        } else if constexpr (OP == 8) {
            const uint32_t other = threadIdx.x & 1;
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {
                const uint32_t b = __shfl_sync(0xffffffffu, a[u], (threadIdx.x & 31) & ~1u);
                float* p = grads + ((((b << 1) & (2 * mask_words + 1)) & ~3u) | (other << 1));
                asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(1.0f), "f"(2.0f) : "memory");
            }
        } else {
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {
                float* p = grads + ((a[u] << 1) & (2 * mask_words + 1) & ~3u);
                asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(1.0f), "f"(2.0f),
                             "f"(3.0f), "f"(4.0f)
                             : "memory");
            }
        }
    }
    if (acc == 0x12345678u)
        sink[0] = acc;
}

int main(int argc, char** argv)
{
    const int iters = argc > 1 ? std::atoi(argv[1]) : 64;
    int sms = 0, clk_khz = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
    const uint32_t words = 1u << 23;   // 32 MB table of 4-byte entries (config 2: 2^19 x 16 levels x fp16x2)
    uint32_t *table, *sink;
    float* grads;                      // 64 MB fp32 grads (2 floats per entry)
    CK(cudaMalloc(&table, size_t(words) * 4));
    CK(cudaMalloc(&grads, size_t(words) * 8));
    CK(cudaMalloc(&sink, 4));
    CK(cudaMemset(table, 1, size_t(words) * 4));
    CK(cudaMemset(grads, 0, size_t(words) * 8));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char* names[17] = { "cp.async 4B gather", "ld.global 4B gather", "ld.global 8B gather", "red.v2.f32 scatter",
                             "red.v4.f32 scatter", "ld 4B, even lanes", "ld 4B, lane pairs/sector",
                             "red.v2, even lanes", "red.v2, lane pairs/16B", "cp.async 8B", "cp.async 16B",
                             "cp.async 4B, even lanes", "ld.global 16B gather", "ld.global 32B gather",
                             "cp.async 4B, lane pairs/sector", "red.v2, lane pairs/sector", "cp.async 4B, pairs 28B apart" };
    auto run = [&](int op, auto kern) {
        const int sz = op == 0 || op == 11 || op == 14 || op == 16 ? 4 : op == 9 ? 8 : op == 10 ? 16 : 0;
        const int smem = UNROLL * TPB * sz;
        int occ = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, TPB, smem));
        const int grid = sms * occ;
        kern<<<grid, TPB, smem>>>(table, grads, words - 1, 4, sink);   // warm L2
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        kern<<<grid, TPB, smem>>>(table, grads, words - 1, iters, sink);
        cudaEventRecord(e1);
        CK(cudaDeviceSynchronize());
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double ops = double(grid) * TPB * iters * UNROLL;
        const double ns_per_op_sm = ms * 1e6 / (ops / sms);
        std::printf("%-22s %2d CTAs/SM: %7.3f ms, %.3g lane-ops/s, %.3f ns per lane-op per SM (%.2f cycles at %d MHz "
                    "nominal)\n",
                    names[op], occ, ms, ops / (ms * 1e-3), ns_per_op_sm, ns_per_op_sm * clk_khz * 1e-6, clk_khz / 1000);
    };
    run(0, k_lsu<0>);
    run(1, k_lsu<1>);
    run(2, k_lsu<2>);
    run(3, k_lsu<3>);
    run(4, k_lsu<4>);
    run(5, k_lsu<5>);
    run(6, k_lsu<6>);
    run(7, k_lsu<7>);
    run(8, k_lsu<8>);
    run(9, k_lsu<9>);
    run(10, k_lsu<10>);
    run(11, k_lsu<11>);
    run(12, k_lsu<12>);
    run(13, k_lsu<13>);
    run(14, k_lsu<14>);
    run(15, k_lsu<15>);
    run(16, k_lsu<16>);
    return 0;
}
