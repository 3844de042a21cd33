// tc_mlp_bench.cu — the north star's "mma.sync or tcgen05, whichever ncu shows
// is faster at width 64": the config-2 MLP forward (32 -> 64 -> 64 -> 1, padded
// to 16 outputs) on 128-sample tiles resident in shared memory, repeated R
// times per CTA, as
//   (a) mma.sync.m16n8k16 with activations kept in registers across layers
//       (the formulation of the product kernels, mlp_core.cuh), and
//   (b) tcgen05.mma (M=128) with the accumulator in TMEM; each layer's
//       epilogue is tcgen05.ld -> bias/ReLU/fp16 -> st.shared into the next
//       layer's canonical K-major operand -> fence.proxy.async -> barrier.
// Checks (b) against (a) on one tile, then times both.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2201_05989_b200/csrc \
//        tools/tc_mlp_bench.cu -o tools/tc_mlp_bench
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "mlp_core.cuh"

using namespace nfg;
using namespace nfg::mlp;

#define CK(x)                                                                                        \
    do {                                                                                             \
        cudaError_t e = (x);                                                                         \
        if (e != cudaSuccess) {                                                                      \
            std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);      \
            std::exit(1);                                                                            \
        }                                                                                            \
    } while (0)

constexpr int TM = 128;   // samples per tile
constexpr int KIN = 32;   // encoded width

// ---------------------------------------------------------------- (a) mma.sync
__global__ void __launch_bounds__(128) k_mma_sync(const float* W, const float* b, const __half* Yg, int reps,
                                                  float* out, float* checksum)
{
    using Lay = WLayout<2, 2>;
    extern __shared__ __align__(16) unsigned char sm[];
    __half* ws = reinterpret_cast<__half*>(sm);
    float* bs = reinterpret_cast<float*>(sm + Lay::HALVES * 2);
    __half* ybuf = reinterpret_cast<__half*>(sm + ((Lay::BYTES + 15) & ~15));
    const MlpShape sh{ KIN, 1, 0 };
    load_weights<2, 2>(ws, bs, W, b, sh);
    for (int i = threadIdx.x; i < TM * KIN; i += blockDim.x)
        ybuf[(i / KIN) * Lay::INS + i % KIN] = Yg[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, t = lane & 3, g = lane >> 2;
    const __half* W0s = ws;
    const __half* W1s = ws + Lay::W0_HALVES;
    const __half* Wos = ws + Lay::W0_HALVES + Lay::WH_HALVES;
    float sum = 0.0f;
    for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int half = 0; half < 2; ++half) {   // warp w: rows 32w .. 32w+31 (two m16 tiles)
            const int row0 = 32 * warp + 16 * half;
            uint32_t a[2][4];
            load_a<2>(a, ybuf, Lay::INS, row0, lane);
            float acc[HT][4];
            uint32_t ah[4][4];
            layer_fwd<2, HT>(a, W0s, Lay::INS, acc, lane);
            bias_relu<HT>(acc, bs, lane);
            c_to_a<4, false>(acc, ah);
            layer_fwd<4, HT>(ah, W1s, HS, acc, lane);
            bias_relu<HT>(acc, bs + H, lane);
            c_to_a<4, false>(acc, ah);
            float ao[2][4];
            layer_fwd<4, 2>(ah, Wos, HS, ao, lane);
            if (t == 0) {
                const float o0 = ao[0][0] + bs[2 * H], o8 = ao[0][2] + bs[2 * H];
                sum += o0 + o8;
                if (r == 0 && blockIdx.x == 0) {
                    out[row0 + g] = o0;
                    out[row0 + g + 8] = o8;
                }
            }
        }
    }
    atomicAdd(checksum, sum);
}

// ---------------------------------------------------------------- (b) tcgen05
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

// canonical K-major, no swizzle: 8-row x 16-byte core matrices, contiguous
// along K (LBO = 128 B), rows of core matrices SBO = (K/8)*128 B apart
__device__ __forceinline__ int cm_off(int r, int k, int K) { return (r >> 3) * (K / 8) * 128 + (k >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2; }

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo)
{
    uint64_t d = 0;
    d |= uint64_t((saddr >> 4) & 0x3FFFu);
    d |= uint64_t((lbo >> 4) & 0x3FFFu) << 16;
    d |= uint64_t((sbo >> 4) & 0x3FFFu) << 32;
    d |= uint64_t(1) << 46;   // sm_100 descriptor version; base offset 0; layout SWIZZLE_NONE (0)
    return d;
}

__host__ __device__ constexpr uint32_t make_idesc(int M, int N)
{
    return (1u << 4)                     // D: f32
           | (0u << 7) | (0u << 10)      // A, B: f16
           | (0u << 15) | (0u << 16)     // A, B K-major
           | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t accum)
{
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
                 "l"(ad), "l"(bd), "r"(idesc), "r"(accum));
}

__device__ __forceinline__ void mma_commit(uint32_t mbar)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t phase)
{
    asm volatile("{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
                 "@P1 bra DONE_%=;\n\tbra WAIT_%=;\n\tDONE_%=:\n\t}\n" ::"r"(mbar),
                 "r"(phase)
                 : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16])
{
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                   "=r"(r[15])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i)
        v[i] = __uint_as_float(r[i]);
}

struct TcSmem {   // byte offsets
    static constexpr int A0 = 0;                       // 128 x 32 fp16
    static constexpr int A1 = A0 + TM * KIN * 2;       // 128 x 64
    static constexpr int A2 = A1;                      // 128 x 64: written after layer 1's MMA completed
    static constexpr int W0 = A1 + TM * H * 2;         // 64 x 32
    static constexpr int W1 = W0 + H * KIN * 2;        // 64 x 64
    static constexpr int W2 = W1 + H * H * 2;          // 16 x 64
    static constexpr int BIAS = W2 + 16 * H * 2;       // 64 + 64 + 16 floats
    static constexpr int MBAR = BIAS + (2 * H + 16) * 4;
    static constexpr int TSLOT = MBAR + 8;
    static constexpr int BYTES = TSLOT + 8;
};

__global__ void __launch_bounds__(128) k_tcgen05(const float* W, const float* b, const __half* Yg, int reps,
                                                 float* out, float* checksum)
{
    extern __shared__ __align__(16) unsigned char sm[];
    const int tid = threadIdx.x, warp = tid >> 5;
    // operands into the canonical layouts
    for (int i = tid; i < TM * KIN; i += 128)
        *reinterpret_cast<__half*>(sm + TcSmem::A0 + cm_off(i / KIN, i % KIN, KIN)) = Yg[i];
    for (int i = tid; i < H * KIN; i += 128) {   // W0: out n x in k (reference col-major W[n + k*64])
        const int n = i / KIN, k = i % KIN;
        *reinterpret_cast<__half*>(sm + TcSmem::W0 + cm_off(n, k, KIN)) = __float2half_rn(W[n + k * H]);
    }
    for (int i = tid; i < H * H; i += 128) {
        const int n = i / H, k = i % H;
        *reinterpret_cast<__half*>(sm + TcSmem::W1 + cm_off(n, k, H)) = __float2half_rn(W[H * KIN + n + k * H]);
    }
    for (int i = tid; i < 16 * H; i += 128) {
        const int n = i / H, k = i % H;
        *reinterpret_cast<__half*>(sm + TcSmem::W2 + cm_off(n, k, H)) =
            __float2half_rn(n < 1 ? W[H * KIN + H * H + k] : 0.0f);
    }
    float* bias = reinterpret_cast<float*>(sm + TcSmem::BIAS);
    for (int i = tid; i < 2 * H + 16; i += 128)
        bias[i] = i < 2 * H + 1 ? b[i] : 0.0f;
    const uint32_t mbar = smem_u32(sm + TcSmem::MBAR);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(sm + TcSmem::TSLOT);
    if (tid == 0)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar));
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // operand writes -> tensor core
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tbase = *tslot;
    const uint32_t tlane = uint32_t(32 * warp) << 16;   // this warp's TMEM lanes
    const uint32_t a0 = smem_u32(sm + TcSmem::A0), a1 = smem_u32(sm + TcSmem::A1), a2 = smem_u32(sm + TcSmem::A2);
    const uint32_t w0 = smem_u32(sm + TcSmem::W0), w1 = smem_u32(sm + TcSmem::W1), w2 = smem_u32(sm + TcSmem::W2);
    constexpr uint32_t ID64 = make_idesc(128, 64), ID16 = make_idesc(128, 16);
    uint32_t phase = 0;
    float sum = 0.0f;
    const int m = tid;   // this thread's sample row (TMEM lane)

    auto relu_store = [&](uint32_t col0, const float* bsub, uint32_t abuf) {
        // D[m][0..63] -> +bias, ReLU, fp16 -> next layer's A (K = 64)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            float v[16];
            tmem_ld16(tbase + tlane + col0 + 16 * c, v);
            uint32_t h[8];
#pragma unroll
            for (int j = 0; j < 8; ++j)
                h[j] = pack_half2(fmaxf(v[2 * j] + bsub[16 * c + 2 * j], 0.0f),
                                  fmaxf(v[2 * j + 1] + bsub[16 * c + 2 * j + 1], 0.0f));
            unsigned char* dst = sm + (abuf - smem_u32(sm));
            *reinterpret_cast<uint4*>(dst + cm_off(m, 16 * c, H)) = make_uint4(h[0], h[1], h[2], h[3]);
            *reinterpret_cast<uint4*>(dst + cm_off(m, 16 * c + 8, H)) = make_uint4(h[4], h[5], h[6], h[7]);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;");
    };

    for (int r = 0; r < reps; ++r) {
        // layer 0: D[0..63] = A0 (128x32) * W0^T
        if (tid == 0) {
#pragma unroll
            for (int k = 0; k < KIN / 16; ++k)
                mma_f16(tbase + 0, make_desc(a0 + 256 * k, 128, (KIN / 8) * 128), make_desc(w0 + 256 * k, 128, (KIN / 8) * 128),
                        ID64, k > 0);
            mma_commit(mbar);
        }
        mbar_wait(mbar, phase);
        phase ^= 1u;
        asm volatile("tcgen05.fence::after_thread_sync;");
        relu_store(0, bias, a1);
        // layer 1: D[0..63] = A1 (layer 0's D was read into registers before the barrier)
        // (128x64) * W1^T
        if (tid == 0) {
#pragma unroll
            for (int k = 0; k < H / 16; ++k)
                mma_f16(tbase + 0, make_desc(a1 + 256 * k, 128, (H / 8) * 128), make_desc(w1 + 256 * k, 128, (H / 8) * 128),
                        ID64, k > 0);
            mma_commit(mbar);
        }
        mbar_wait(mbar, phase);
        phase ^= 1u;
        asm volatile("tcgen05.fence::after_thread_sync;");
        relu_store(0, bias + H, a2);
        // output layer: D[0..15] = A2 (128x64) * W2^T
        if (tid == 0) {
#pragma unroll
            for (int k = 0; k < H / 16; ++k)
                mma_f16(tbase + 0, make_desc(a2 + 256 * k, 128, (H / 8) * 128), make_desc(w2 + 256 * k, 128, (H / 8) * 128),
                        ID16, k > 0);
            mma_commit(mbar);
        }
        mbar_wait(mbar, phase);
        phase ^= 1u;
        asm volatile("tcgen05.fence::after_thread_sync;");
        float v[16];
        tmem_ld16(tbase + tlane + 0, v);
        const float o = v[0] + bias[2 * H];
        sum += o;
        if (r == 0 && blockIdx.x == 0)
            out[m] = o;
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();   // D columns 0..15 are reused by the next repetition's layer 0
        asm volatile("tcgen05.fence::after_thread_sync;");
    }
    atomicAdd(checksum, sum);
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tbase));
}

int main(int argc, char** argv)
{
    const int reps = argc > 1 ? std::atoi(argv[1]) : 200;
    int sms = 148;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    std::mt19937 rng(3);
    std::uniform_real_distribution<float> U(-1.f, 1.f);
    const int nW = H * KIN + H * H + H, nb = 2 * H + 1;
    std::vector<float> W(nW), b(nb);
    for (int i = 0; i < H * KIN; ++i)
        W[i] = U(rng) * std::sqrt(6.0f / (KIN + H));
    for (int i = H * KIN; i < H * KIN + H * H; ++i)
        W[i] = U(rng) * std::sqrt(6.0f / (2 * H));
    for (int i = H * KIN + H * H; i < nW; ++i)
        W[i] = U(rng) * std::sqrt(6.0f / (H + 1));
    for (auto& v : b)
        v = 0.1f * U(rng);
    std::vector<__half> Y(TM * KIN);
    for (auto& v : Y)
        v = __float2half(U(rng));
    float *dW, *db, *dout_a, *dout_b, *dsum;
    __half* dY;
    CK(cudaMalloc(&dW, nW * 4));
    CK(cudaMalloc(&db, nb * 4));
    CK(cudaMalloc(&dY, TM * KIN * 2));
    CK(cudaMalloc(&dout_a, TM * 4));
    CK(cudaMalloc(&dout_b, TM * 4));
    CK(cudaMalloc(&dsum, 8));
    CK(cudaMemcpy(dW, W.data(), nW * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(db, b.data(), nb * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dY, Y.data(), TM * KIN * 2, cudaMemcpyHostToDevice));
    const int smem_a = ((WLayout<2, 2>::BYTES + 15) & ~15) + TM * WLayout<2, 2>::INS * 2;
    const int smem_b = TcSmem::BYTES;
    CK(cudaFuncSetAttribute(k_mma_sync, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_a));
    CK(cudaFuncSetAttribute(k_tcgen05, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_b));
    CK(cudaFuncSetAttribute(k_mma_sync, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    CK(cudaFuncSetAttribute(k_tcgen05, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    int occ_a = 0, occ_b = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_a, k_mma_sync, 128, smem_a));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_b, k_tcgen05, 128, smem_b));
    std::printf("occupancy query: mma.sync %d, tcgen05 %d CTAs/SM\n", occ_a, occ_b);
    occ_b = argc > 2 ? std::atoi(argv[2]) : std::min(std::max(occ_b, 1), 8);   // TMEM: 8 x 64 columns per SM
    // correctness on one tile
    CK(cudaMemset(dsum, 0, 8));
    k_mma_sync<<<1, 128, smem_a>>>(dW, db, dY, 1, dout_a, dsum);
    k_tcgen05<<<1, 128, smem_b>>>(dW, db, dY, 1, dout_b, dsum);
    CK(cudaDeviceSynchronize());
    std::vector<float> oa(TM), ob(TM);
    CK(cudaMemcpy(oa.data(), dout_a, TM * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ob.data(), dout_b, TM * 4, cudaMemcpyDeviceToHost));
    float maxd = 0, maxa = 0;
    for (int i = 0; i < TM; ++i) {
        maxd = std::max(maxd, std::fabs(oa[i] - ob[i]));
        maxa = std::max(maxa, std::fabs(oa[i]));
    }
    std::printf("tile check: max|mma.sync - tcgen05| = %.3g (max|out| %.3g)\n", maxd, maxa);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](const char* name, auto kern, int smem, int occ) {
        const int grid = sms * occ;
        kern<<<grid, 128, smem>>>(dW, db, dY, 5, dout_a, dsum);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        kern<<<grid, 128, smem>>>(dW, db, dY, reps, dout_a, dsum);
        cudaEventRecord(e1);
        CK(cudaDeviceSynchronize());
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double samples = double(grid) * TM * reps;
        const double flop = samples * 2.0 * (KIN * H + H * H + H * 16);
        std::printf("%-10s CTAs/SM %d: %8.3f ms, %.3g samples/s, %.1f TFLOP/s (padded output)\n", name, occ, ms,
                    samples / (ms / 1e3), flop / (ms / 1e3) / 1e12);
    };
    timeit("mma.sync", k_mma_sync, smem_a, occ_a);
    if (argc > 3)
        timeit("mma.sync", k_mma_sync, smem_a, std::atoi(argv[3]));
    timeit("tcgen05", k_tcgen05, smem_b, occ_b);
    return 0;
}
