// tc_probe.cu — hardware check of the tcgen05 forms the fused training kernel's
// dW GEMMs use (before building on them):
//   * M = 64, cta_group::1, kind::f16, A and B both MN-major (canonical,
//     SWIZZLE_NONE: 8 (MN) x 8 (K) core matrices of 16-byte MN rows; K blocks
//     LBO apart, MN blocks SBO apart);
//   * the M = 64 accumulator layout in TMEM (row m -> lane (m % 16) + 32 (m / 16))
//     and the second ("interleaved") accumulator at TMEM lane offset 16.
// Small-integer operands make every fp32 sum exact, so the check is bitwise.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2201_05989_b200/csrc \
//        tools/tc_probe.cu -o tools/tc_probe && tools/tc_probe
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc_core.cuh"

using namespace nfg;

constexpr int M = 64, K = 64, N = 40;

__device__ __forceinline__ int mn_off(int mn, int k, int Kt)   // canonical MN-major, LBO = 128, SBO = (Kt/8)*128
{
    return (mn >> 3) * (Kt / 8) * 128 + (k >> 3) * 128 + (k & 7) * 16 + (mn & 7) * 2;
}

__global__ void k_probe(const float* A, const float* B, float* D0, float* D1, int mode)
{
    // A: M x K (row-major logical), B: K x N
    __shared__ __align__(128) unsigned char sa[M * K * 2];
    __shared__ __align__(128) unsigned char sb[N * K * 2];
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < M * K; i += blockDim.x) {
        const int m = i / K, k = i % K;
        *reinterpret_cast<__half*>(sa + mn_off(m, k, K)) = __float2half_rn(A[i]);
    }
    for (int i = tid; i < K * N; i += blockDim.x) {
        const int k = i / N, n = i % N;
        *reinterpret_cast<__half*>(sb + mn_off(n, k, K)) = __float2half_rn(B[i]);
    }
    if (tid == 0)
        tc::mbar_init(tc::smem_u32(&mbar), 1);
    if (warp == 0)
        tc::tmem_alloc(&tslot, 128);
    tc::fence_smem_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tb = tslot;
    // idesc: D f32, A/B f16, A MN-major (bit 15), B MN-major (bit 16), N, M
    const uint32_t idesc = (1u << 4) | (1u << 15) | (1u << 16) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
    if (tid == 0) {
        tc::fence_after();
        for (int s = 0; s < K / 16; ++s) {
            // K step s = 2 K blocks = 256 B further along K
            const uint64_t ad = tc::desc(tc::smem_u32(sa) + 256u * s, 128u, (K / 8) * 128u);
            const uint64_t bd = tc::desc(tc::smem_u32(sb) + 256u * s, 128u, (K / 8) * 128u);
            tc::mma_f16(tb, ad, bd, idesc, s > 0);                          // D0 at lane 0, col 0
            if (mode)
                tc::mma_f16(tb + (16u << 16), ad, bd, idesc, s > 0);       // D1 at lane 16, col 0
        }
        tc::commit(tc::smem_u32(&mbar));
    }
    tc::mbar_wait(tc::smem_u32(&mbar), 0);
    tc::fence_after();
    // every warp reads its 32 lanes, 40 columns (x32 + x8 as x16 x3 with the tail ignored)
    float v[48];
    {
        float a[16];
        for (int c = 0; c < 3; ++c) {
            tc::ld16(tb + (uint32_t(32 * warp) << 16) + 16u * c, a);
            for (int i = 0; i < 16; ++i)
                v[16 * c + i] = a[i];
        }
    }
    const int L = 32 * warp + lane;
    for (int n = 0; n < N; ++n) {
        D0[L * N + n] = v[n];
    }
    (void)D1;
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (warp == 0)
        tc::tmem_dealloc(tb, 128);
}

int main()
{
    std::vector<float> A(M * K), B(K * N), ref(M * N, 0.0f);
    srand(3);
    for (auto& x : A)
        x = float(rand() % 7 - 3);
    for (auto& x : B)
        x = float(rand() % 5 - 2);
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            float s = 0;
            for (int k = 0; k < K; ++k)
                s += A[m * K + k] * B[k * N + n];
            ref[m * N + n] = s;
        }
    float *dA, *dB, *dD0, *dD1;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dD0, 128 * N * 4);
    cudaMalloc(&dD1, 128 * N * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    for (int mode = 0; mode < 2; ++mode) {
        cudaMemset(dD0, 0, 128 * N * 4);
        k_probe<<<1, 128>>>(dA, dB, dD0, dD1, mode);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("mode %d: CUDA error %s\n", mode, cudaGetErrorString(e));
            return 1;
        }
        std::vector<float> D(128 * N);
        cudaMemcpy(D.data(), dD0, D.size() * 4, cudaMemcpyDeviceToHost);
        // hypothesis: row m at lane (m % 16) + 32 (m / 16) [+ 16 for the second accumulator]
        int bad0 = 0, bad1 = 0, zero_else = 0;
        std::vector<int> used(128, 0);
        for (int m = 0; m < M; ++m) {
            const int l0 = (m % 16) + 32 * (m / 16);
            used[l0] = used[l0 + 16] = 1;
            for (int n = 0; n < N; ++n) {
                bad0 += D[l0 * N + n] != ref[m * N + n];
                if (mode)
                    bad1 += D[(l0 + 16) * N + n] != ref[m * N + n];
            }
        }
        for (int l = 0; l < 128; ++l)
            if (!used[l])
                for (int n = 0; n < N; ++n)
                    zero_else += D[l * N + n] != 0.0f;
        printf("mode %d (%s): M=64 MN-major A/B, lane-0 accumulator mismatches %d / %d%s", mode,
               mode ? "two accumulators at lanes 0 and 16" : "one accumulator", bad0, M * N,
               mode ? "" : "\n");
        if (mode)
            printf(", lane-16 accumulator mismatches %d / %d\n", bad1, M * N);
        if (mode == 0) {
            int lo = 0;
            for (int m = 0; m < M; ++m)
                for (int n = 0; n < N; ++n)
                    lo += D[((m % 16) + 32 * (m / 16) + 16) * N + n] != 0.0f;
            printf("         lanes 16..31 of each subpartition nonzero entries: %d (expect 0)\n", lo);
        }
    }
    printf("%s\n", "probe done");
    return 0;
}
