// tma_gather_bench.cu — research probe for the next k_train step:
// can the TMA unit's gather4 mode (UTMALDG.2D.GATHER4: four 16-byte rows of a
// 2-D tensor per instruction) serve the hash-grid corner gathers faster than the
// LSU's per-lane cp.async (the path k_train uses, which ncu shows L1/LSU-limited)?
// Same random-row pattern for both: an fp16 F=2 table (4-byte rows) of
// `rows` entries, `per_lane` random rows per lane per iteration.
//   (a) cp.async.ca 4 B per row (the product path);
//   (b) TMA gather4 of the 16-byte chunk holding each row (4 rows = 4 chunks per
//       instruction, issued by one lane per warp from shuffled indices).
// Reports rows/s and the equivalent 32-byte sector rate.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/tma_gather_bench.cu -o tools/tma_gather_bench
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>

#define CK(x)                                                                                        \
    do {                                                                                             \
        cudaError_t e_ = (x);                                                                        \
        if (e_ != cudaSuccess) {                                                                     \
            std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);     \
            std::exit(1);                                                                            \
        }                                                                                            \
    } while (0)

constexpr int PER_LANE = 64;   // rows per lane per iteration (k_train: 64 staged corners per lane and tile)

__device__ __forceinline__ uint32_t hash_row(uint32_t seed, uint32_t i, uint32_t mask)
{
    uint32_t x = seed * 0x9E3779B9u ^ (i * 0x85EBCA6Bu);
    x ^= x >> 16;
    x *= 0x7FEB352Du;
    x ^= x >> 15;
    x *= 0x846CA68Bu;
    x ^= x >> 16;
    return x & mask;
}

__global__ void __launch_bounds__(128) k_cpasync(const uint32_t* __restrict__ table, uint32_t mask, int iters,
                                                 float* out)
{
    __shared__ uint32_t slots[PER_LANE][128];
    const int tid = threadIdx.x;
    float acc = 0.0f;
    for (int it = 0; it < iters; ++it) {
        const uint32_t seed = blockIdx.x * 7919u + it * 104729u + tid;
#pragma unroll 8
        for (int k = 0; k < PER_LANE; ++k) {
            const uint32_t r = hash_row(seed, k, mask);
            const uint32_t s = uint32_t(__cvta_generic_to_shared(&slots[k][tid]));
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(table + r));
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
#pragma unroll 8
        for (int k = 0; k < PER_LANE; ++k)
            acc += __half2float(reinterpret_cast<const __half2*>(&slots[k][tid])->x);
        __syncwarp();
    }
    if (acc == 12345.0f)
        out[0] = acc;
}

// one warp per block: 32 lanes x PER_LANE chunks of 16 B; each gather4 lands on a
// 128-byte aligned slot (the bulk-tensor destination alignment), 64 KB of dynamic smem
__global__ void __launch_bounds__(32) k_tma_gather4(const __grid_constant__ CUtensorMap tmap, uint32_t mask,
                                                    int iters, float* out)
{
    extern __shared__ __align__(128) uint4 dst[];
    __shared__ __align__(8) uint64_t mbar;
    const int lane = threadIdx.x;
    const uint32_t mb = uint32_t(__cvta_generic_to_shared(&mbar));
    if (lane == 0)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    float acc = 0.0f;
    uint32_t phase = 0;
    for (int it = 0; it < iters; ++it) {
        const uint32_t seed = blockIdx.x * 7919u + it * 104729u + lane;
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(PER_LANE * 32 * 16));
        __syncwarp();
        for (int k = 0; k < PER_LANE; k += 4) {
            uint32_t c[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
                c[q] = hash_row(seed, k + q, mask) >> 2;   // the 16-byte chunk of the row
            // every lane's 4 chunks, issued by lane 0 (TMA coordinates are uniform operands)
            for (int j = 0; j < 32; ++j) {
                const uint32_t c0 = __shfl_sync(0xffffffffu, c[0], j), c1 = __shfl_sync(0xffffffffu, c[1], j);
                const uint32_t c2 = __shfl_sync(0xffffffffu, c[2], j), c3 = __shfl_sync(0xffffffffu, c[3], j);
                if (lane == 0) {
                    const uint32_t s = uint32_t(__cvta_generic_to_shared(&dst[(k / 4) * 256 + j * 8]));
                    asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
                                 " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(s),
                                 "l"(&tmap), "r"(0), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(mb)
                                 : "memory");
                }
            }
        }
        asm volatile("{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
                     "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
                     "@P1 bra DONE_%=;\n\tbra WAIT_%=;\n\tDONE_%=:\n\t}\n" ::"r"(mb), "r"(phase)
                     : "memory");
        phase ^= 1u;
#pragma unroll 8
        for (int k = 0; k < PER_LANE; ++k)
            acc += __half2float(reinterpret_cast<const __half2*>(&dst[(k / 4) * 256 + lane * 8 + (k & 3)])->x);
        __syncwarp();
    }
    if (acc == 12345.0f)
        out[0] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv)
{
    const int log_rows = argc > 1 ? std::atoi(argv[1]) : 23;   // 2^23 rows x 4 B = 32 MB (L2-resident, like config 2)
    const int iters = argc > 2 ? std::atoi(argv[2]) : 200;
    const uint64_t rows = uint64_t(1) << log_rows;
    int sms = 148;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    uint32_t* table;
    float* out;
    CK(cudaMalloc(&table, rows * 4));
    CK(cudaMalloc(&out, 16));
    CK(cudaMemset(table, 0x3c, rows * 4));
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    CUtensorMap tm;
    const cuuint64_t dims[2] = { 4, rows / 4 };          // 4 u32 (16 B) per chunk, rows/4 chunks
    const cuuint64_t strides[1] = { 16 };
    const cuuint32_t box[2] = { 4, 1 };
    const cuuint32_t estr[2] = { 1, 1 };
    CUresult r = reinterpret_cast<EncodeFn>(fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, table, dims, strides, box, estr,
                                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                                CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    std::printf("cuTensorMapEncodeTiled: %d\n", int(r));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const uint32_t mask = uint32_t(rows - 1);
    auto run = [&](const char* name, auto launch, int blocks) {
        launch(blocks, 2);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        launch(blocks, iters);
        cudaEventRecord(e1);
        CK(cudaDeviceSynchronize());
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double n = double(blocks) * (name[0] == 't' ? 32 : 128) * PER_LANE * iters;
        std::printf("%-16s blocks %5d: %8.3f ms, %.3g rows/s\n", name, blocks, ms, n / (ms / 1e3));
    };
    CK(cudaFuncSetAttribute(k_tma_gather4, cudaFuncAttributeMaxDynamicSharedMemorySize, PER_LANE * 32 * 32));
    for (int per_sm : { 1, 2, 3 }) {
        run("cp.async 4B", [&](int b, int it) { k_cpasync<<<b, 128>>>(table, mask, it, out); }, sms * per_sm);
        if (r == CUDA_SUCCESS)
            run("tma gather4", [&](int b, int it) { k_tma_gather4<<<b, 32, PER_LANE * 32 * 32>>>(tm, mask, it, out); },
                sms * per_sm);
    }
    return 0;
}
