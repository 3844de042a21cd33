// adam_bw.cu — the DRAM ceiling of Adam's access pattern on this B200.
// k_adam streams p, m, v in and out (3 reads + 3 writes of 4 B per parameter;
// g and the fp16 shadow stay in L2). This measures, on the same sizes
// (config 2: 15.2 M table + MLP parameters), a kernel that does only that traffic
// (a trivial update) so the optimizer's achieved DRAM rate can be compared with
// what the memory system gives for this 3-in / 3-out pattern, plus a plain
// 1-in / 1-out copy of the same bytes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/adam_bw.cu -o tools/adam_bw
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

__global__ void __launch_bounds__(256) k_pmv(float4* p, float4* m, float4* v, uint64_t n4)
{
    for (uint64_t q = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < n4; q += uint64_t(gridDim.x) * blockDim.x) {
        float4 P = __ldcs(p + q), M = __ldcs(m + q), V = __ldcs(v + q);
        P.x += 1.0f;
        M.y += 1.0f;
        V.z += 1.0f;
        __stcs(p + q, P);
        __stcs(m + q, M);
        __stcs(v + q, V);
    }
}

__global__ void __launch_bounds__(256) k_copy(const float4* a, float4* b, uint64_t n4)
{
    for (uint64_t q = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < n4; q += uint64_t(gridDim.x) * blockDim.x)
        __stcs(b + q, __ldcs(a + q));
}

int main(int argc, char** argv)
{
    const uint64_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 15200000ull;   // parameters
    const uint64_t n4 = n / 4;
    int sms = 148;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    float4 *p, *m, *v, *a, *b, *flush;
    CK(cudaMalloc(&p, n4 * 16));
    CK(cudaMalloc(&m, n4 * 16));
    CK(cudaMalloc(&v, n4 * 16));
    CK(cudaMalloc(&a, n4 * 16 * 3));
    CK(cudaMalloc(&b, n4 * 16 * 3));
    const size_t flush_bytes = size_t(512) << 20;   // > L2: every timed launch starts cold
    CK(cudaMalloc(&flush, flush_bytes));
    for (auto* x : { p, m, v })
        CK(cudaMemset(x, 0, n4 * 16));
    CK(cudaMemset(a, 0, n4 * 48));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int grid_per_sm : { 4, 8, 16 }) {
        const int grid = sms * grid_per_sm;
        float best_pmv = 1e9f, best_copy = 1e9f;
        for (int r = 0; r < 10; ++r) {
            CK(cudaMemsetAsync(flush, r, flush_bytes));
            cudaEventRecord(e0);
            k_pmv<<<grid, 256>>>(p, m, v, n4);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best_pmv = ms < best_pmv ? ms : best_pmv;
            CK(cudaMemsetAsync(flush, r, flush_bytes));
            cudaEventRecord(e0);
            k_copy<<<grid, 256>>>(a, b, n4 * 3);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            cudaEventElapsedTime(&ms, e0, e1);
            best_copy = ms < best_copy ? ms : best_copy;
        }
        const double bytes = double(n4) * 16 * 6;   // 3 streams in, 3 out
        std::printf("grid %d/SM: p/m/v 3-in/3-out %.1f us = %.0f GB/s | 1-in/1-out copy of the same bytes %.1f us = %.0f GB/s\n",
                    grid_per_sm, best_pmv * 1e3, bytes / (best_pmv * 1e-3) / 1e9, best_copy * 1e3,
                    bytes / (best_copy * 1e-3) / 1e9);
    }
    return 0;
}
