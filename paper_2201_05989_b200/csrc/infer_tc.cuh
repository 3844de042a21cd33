// infer_tc.cuh — fused encode + MLP inference with the MLP on tcgen05.
//
// Same contract as k_infer (model.cpp:102-109: encode_forward grid.hpp:219-272
// -> mlp_forward mlp.hpp:104-124 -> output activation), different MLP engine:
// the CTA is NQ independent "quads" of 4 warps; a quad owns a 128-sample tile.
//   1. each warp encodes its 32 rows (lane-pair gathers, encode.cuh) and stores
//      them as fp16 into the quad's canonical K-major A tile in shared memory;
//   2. one elected thread issues the layer's tcgen05.mma (M = 128, N = 64 or 16,
//      K = 16 per instruction) with the fp32 accumulator in the quad's 64 TMEM
//      columns and commits to the quad's mbarrier;
//   3. every thread reads its own sample's accumulator row (tcgen05.ld: warp
//      w % 4 owns TMEM lanes 32 (w % 4) ..), adds the bias, applies ReLU and
//      writes the fp16 row back as the next layer's A operand; the output
//      layer's row is the sample's result.
// Quads synchronise with a named barrier of 128 threads, so one quad's MMAs and
// epilogues overlap the other quads' gathers. Weights stay in shared memory as
// the B operands (one copy per SM).
#pragma once

#include "field_kernels.cuh"
#include "tc_core.cuh"

namespace nfg {

#ifndef NFG_IQ
#define NFG_IQ 6
#endif
constexpr int IQ = NFG_IQ;   // quads (4 warps, one 128-sample tile) per tcgen05 inference CTA

template <int IN_STEPS, int NH>
struct InferTcSmem {
    static constexpr int K0 = 16 * IN_STEPS;
    static constexpr int W0_OFF = 0;                                  // 64 x K0 fp16
    static constexpr int WH_OFF = W0_OFF + H * K0 * 2;                // (NH-1) x 64 x 64
    static constexpr int WO_OFF = WH_OFF + (NH - 1) * H * H * 2;      // 16 x 64
    static constexpr int BIAS_OFF = WO_OFF + OUTP * H * 2;            // fp32 [H*NH + OUTP]
    static constexpr int LV_OFF = align16(BIAS_OFF + (H * NH + OUTP) * 4);
    static constexpr int MBAR_OFF = align16(LV_OFF + int(sizeof(LevelDev)) * NFG_MAX_LEVELS);
    static constexpr int TSLOT_OFF = MBAR_OFF + 8 * IQ;
    static constexpr int ACT_OFF = (TSLOT_OFF + 16 + 127) & ~127;
    static constexpr int ACT_BYTES = 128 * H * 2;                     // 128 x 64 fp16 per quad
    static constexpr int BYTES = ACT_OFF + IQ * ACT_BYTES;
};

constexpr uint32_t tmem_cols_for(int q)
{
    return q * 64 <= 32 ? 32u : q * 64 <= 64 ? 64u : q * 64 <= 128 ? 128u : q * 64 <= 256 ? 256u : 512u;
}

template <int SRC, int D, int F, typename TT, int IN_STEPS, int NH>
__global__ void __launch_bounds__(IQ * 128, 1)
k_infer_tc(const InferArgs a, const FieldShape s, const LevelDev* __restrict__ levels)
{
    static_assert(SRC == SRC_ENCODE, "the tcgen05 inference kernel encodes its own inputs");
    using SM = InferTcSmem<IN_STEPS, NH>;
    constexpr int K0 = SM::K0;
    extern __shared__ __align__(16) unsigned char sm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, q = warp >> 2, wq = warp & 3;
    float* bs = reinterpret_cast<float*>(sm + SM::BIAS_OFF);
    LevelDev* lvs = reinterpret_cast<LevelDev*>(sm + SM::LV_OFF);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(sm + SM::TSLOT_OFF);

    // ---- weights -> canonical K-major B operands (reference W_k: out x in,
    // col-major, hidden width hw; zero rows / columns pad the layers to 64)
    const int hw = s.hidden_width;
    for (int i = tid; i < H * K0; i += blockDim.x) {
        const int n = i / K0, k = i % K0;
        *reinterpret_cast<__half*>(sm + SM::W0_OFF + tc::cm_off(n, k, K0)) =
            __float2half_rn(k < s.in_real && n < hw ? a.W[n + k * hw] : 0.0f);
    }
    const size_t wh0 = size_t(hw) * s.in_real;
    for (int i = tid; i < (NH - 1) * H * H; i += blockDim.x) {
        const int l = i / (H * H), n = (i / H) % H, k = i % H;
        *reinterpret_cast<__half*>(sm + SM::WH_OFF + l * H * H * 2 + tc::cm_off(n, k, H)) =
            __float2half_rn(n < hw && k < hw ? a.W[wh0 + size_t(l) * hw * hw + n + k * hw] : 0.0f);
    }
    const size_t wo0 = wh0 + size_t(NH - 1) * hw * hw;
    for (int i = tid; i < OUTP * H; i += blockDim.x) {
        const int n = i / H, k = i % H;
        *reinterpret_cast<__half*>(sm + SM::WO_OFF + tc::cm_off(n, k, H)) =
            __float2half_rn(n < s.n_out && k < hw ? a.W[wo0 + n + k * s.n_out] : 0.0f);
    }
    for (int i = tid; i < H * NH; i += blockDim.x)
        bs[i] = (i % H) < hw ? a.b[(i / H) * hw + (i % H)] : 0.0f;
    for (int i = tid; i < OUTP; i += blockDim.x)
        bs[H * NH + i] = i < s.n_out ? a.b[hw * NH + i] : 0.0f;
    for (int i = tid; i < s.grid.L; i += blockDim.x)
        lvs[i] = levels[i];
    const uint32_t mbar = tc::smem_u32(sm + SM::MBAR_OFF) + 8u * q;
    if (tid < IQ)
        tc::mbar_init(tc::smem_u32(sm + SM::MBAR_OFF) + 8u * tid, 1);
    if (warp == 0)
        tc::tmem_alloc(tslot, tmem_cols_for(IQ));
    tc::fence_smem_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();

    const uint32_t tcol = *tslot + 64u * q;                 // this quad's accumulator columns
    const uint32_t trow = uint32_t(32 * wq) << 16;          // this warp's TMEM lanes
    unsigned char* act = sm + SM::ACT_OFF + q * SM::ACT_BYTES;
    const uint32_t act_s = tc::smem_u32(act);
    const uint32_t w0_s = tc::smem_u32(sm + SM::W0_OFF), wh_s = tc::smem_u32(sm + SM::WH_OFF),
                   wo_s = tc::smem_u32(sm + SM::WO_OFF);
    constexpr uint32_t ID64 = tc::idesc_f16(128, 64), ID16 = tc::idesc_f16(128, OUTP);
    const bool issuer = wq == 0 && lane == 0;
    const int g = lane >> 2, t = lane & 3;
    const int m = 32 * wq + lane;                           // this thread's sample row in the tile
    uint32_t phase = 0;

    // one layer: act (K-wide canonical) x B^T -> TMEM, then wait
    auto run_layer = [&](uint32_t b_s, int K, int ksteps, uint32_t idesc) {
        tc::fence_smem_async();
        tc::fence_before();
        tc::bar_sync(1 + q, 128);
        if (issuer) {
            tc::fence_after();
            for (int k = 0; k < ksteps; ++k)
                tc::mma_f16(tcol, tc::kstep_desc(act_s, K, k), tc::kstep_desc(b_s, K, k), idesc, k > 0);
            tc::commit(mbar);
        }
        tc::mbar_wait(mbar, phase);
        phase ^= 1u;
        tc::fence_after();
    };

    const int64_t ntiles = (a.B + 127) / 128;
    for (int64_t tile = int64_t(q) * gridDim.x + blockIdx.x; tile < ntiles; tile += int64_t(gridDim.x) * IQ) {
        // ---- encode this warp's 32 rows (two 16-sample fragment blocks)
#pragma unroll
        for (int hb = 0; hb < 2; ++hb) {
            const int r0 = 32 * wq + 16 * hb;
            const int64_t sg = tile * 128 + r0 + g, sg8 = sg + 8;
            const bool vg = sg < a.B, vg8 = sg8 < a.B;
            float xg[D], xg8[D];
            load_x<D>(xg, a.X, sg, vg);
            load_x<D>(xg8, a.X, sg8, vg8);
            clamp_x<D>(xg);
            clamp_x<D>(xg8);
            uint32_t afr[IN_STEPS][4];
            input_frags<SRC, D, F, TT, IN_STEPS, true>(afr, s, lvs, xg, xg8, vg, vg8, sg, a.Y, a.table, lane);
#pragma unroll
            for (int st = 0; st < IN_STEPS; ++st) {
                const int k = 16 * st + 2 * t;
                *reinterpret_cast<uint32_t*>(act + tc::cm_off(r0 + g, k, K0)) = afr[st][0];
                *reinterpret_cast<uint32_t*>(act + tc::cm_off(r0 + g + 8, k, K0)) = afr[st][1];
                *reinterpret_cast<uint32_t*>(act + tc::cm_off(r0 + g, k + 8, K0)) = afr[st][2];
                *reinterpret_cast<uint32_t*>(act + tc::cm_off(r0 + g + 8, k + 8, K0)) = afr[st][3];
            }
        }
        run_layer(w0_s, K0, IN_STEPS, ID64);
        // ---- hidden layers: epilogue of layer k-1 feeds layer k
#pragma unroll
        for (int k = 1; k <= NH; ++k) {
            const float* bias = bs + H * (k - 1);
#pragma unroll
            for (int hv = 0; hv < 2; ++hv) {
                float v[32];
                tc::ld32(tcol + trow + 32u * hv, v);
                uint32_t hp[16];
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    hp[j] = pack_half2(fmaxf(v[2 * j] + bias[32 * hv + 2 * j], 0.0f),
                                       fmaxf(v[2 * j + 1] + bias[32 * hv + 2 * j + 1], 0.0f));
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    *reinterpret_cast<uint4*>(act + tc::cm_off(m, 32 * hv + 8 * c, H)) =
                        make_uint4(hp[4 * c], hp[4 * c + 1], hp[4 * c + 2], hp[4 * c + 3]);
            }
            if (k < NH)
                run_layer(wh_s + uint32_t(k - 1) * H * H * 2, H, H / 16, ID64);
            else
                run_layer(wo_s, H, H / 16, ID16);
        }
        // ---- output epilogue: this thread's sample
        float v[16];
        tc::ld16(tcol + trow, v);
        const int64_t smp = tile * 128 + m;
        if (smp < a.B) {
            const float* bout = bs + H * NH;
            for (int c = 0; c < s.n_out; ++c) {
                const float z = v[c] + bout[c];
                a.out[smp * s.n_out + c] = s.sigmoid ? 1.0f / (1.0f + expf(-z)) : z;
            }
        }
        tc::fence_before();   // the next tile's first MMA overwrites these columns after the quad barrier
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (warp == 0)
        tc::tmem_dealloc(*tslot, tmem_cols_for(IQ));
}

}   // namespace nfg
