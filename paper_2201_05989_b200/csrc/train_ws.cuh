// train_ws.cuh — warp-specialised fused training kernel (experiment / option).
//
// Same step as k_train<SRC_ENCODE, GRAD_LOSS, SINK_SCATTER, ..., TCW = true>
// (model.cpp:111-138: encode grid.hpp:245-271 -> MLP mlp.hpp:113-123 ->
// loss losses.hpp -> MLP backward mlp.hpp:146-157 -> encode backward
// grid.hpp:286-294 -> dW / db), split over two warpgroups per CTA:
//   * producers (warps 0-3): load the tile's inputs, issue the lane-pair
//     cp.async corner gathers into their own staging slots, blend them into the
//     mma A fragments and hand the fragments + coordinates over through a
//     double-buffered shared-memory slot (mbarrier full / empty per warp);
//   * consumers (warps 4-7): the mma.sync forward / backward chains, loss,
//     encode-backward reductions and the tcgen05 dW / db into TMEM (as k_train).
// Consumer warp c takes the rows producer warp c encoded, so the hand-off is
// pairwise (no CTA barrier); consumers synchronise among themselves with a
// named barrier for the tile's dz scale and the dW MMA. setmaxnreg moves
// registers from the producers (gather state) to the consumers (MLP chains).
// The gathers of tile t+1 overlap the MLP and the reductions of tile t.
#pragma once

#include "field_kernels.cuh"

namespace nfg {

#ifndef NFG_WS_PRODUCER_REGS
#define NFG_WS_PRODUCER_REGS 88
#endif
#ifndef NFG_WS_CONSUMER_REGS
#define NFG_WS_CONSUMER_REGS 168
#endif

template <int D, typename TT, int IN_STEPS, int NH>
struct TrainWsSmem {
    using Lay = WLayout<IN_STEPS, NH>;
    using SG = StageGeo<SRC_ENCODE, D, 2, TT, IN_STEPS>;
    static constexpr int K0 = 16 * IN_STEPS;
    static constexpr int NFR = 4 * IN_STEPS;                             // A-fragment words per lane
    static constexpr int LV_OFF = align16(Lay::BYTES);
    static constexpr int ACT0_OFF = (LV_OFF + int(sizeof(LevelDev)) * NFG_MAX_LEVELS + 127) & ~127;
    static constexpr int ACT0_BYTES = (K0 / 8 + 1) * KC_SBO;
    static constexpr int ACTH_OFF = ACT0_OFF + ACT0_BYTES;
    static constexpr int ACTH_BYTES = (H / 8 + 1) * KC_SBO;
    static constexpr int DZH_OFF = ACTH_OFF + NH * ACTH_BYTES;
    static constexpr int DZH_BYTES = H / 8 * KC_SBO;
    static constexpr int DZO_OFF = DZH_OFF + NH * DZH_BYTES;
    static constexpr int DZO_BYTES = OUTP / 8 * KC_SBO;
    static constexpr int HAND_OFF = DZO_OFF + DZO_BYTES;                // hand-off slots [2]
    static constexpr int HAND_FR = NFR * 128 * 4;                        // fragments [word][thread]
    static constexpr int HAND_X = 2 * D * 128 * 4;                       // coordinates [i][thread]
    static constexpr int HAND_BYTES = HAND_FR + HAND_X;
    static constexpr int STAGE_OFF = HAND_OFF + 2 * HAND_BYTES;          // producer staging (linear)
    static constexpr int STAGE_BYTES = 128 * SG::STS * 4 * SG::NE * SG::SB;
    static constexpr int RED_OFF = STAGE_OFF + STAGE_BYTES;
    static constexpr int DBO_OFF = RED_OFF + 4 * TW * 4;
    static constexpr int MBAR_OFF = align16(DBO_OFF + TW * OUTP * 4);    // full[2][4], empty[2][4], dw
    static constexpr int TSLOT_OFF = MBAR_OFF + 17 * 8;
    static constexpr int BYTES = align16(TSLOT_OFF + 8);
    static constexpr int NCOLS = TcSlots<NH>::ncols(K0);
    static constexpr uint32_t TMEM_COLS = tc::alloc_cols(NCOLS);
};

__device__ __forceinline__ void mbar_arrive(uint32_t mbar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(mbar) : "memory");
}

template <int D, typename TT, int IN_STEPS, int NH>
__global__ void __launch_bounds__(256, 2)
k_train_ws(const TrainArgs a, const FieldShape s, const LevelDev* __restrict__ levels)
{
    constexpr int F = 2;
    using Lay = WLayout<IN_STEPS, NH>;
    using SG = StageGeo<SRC_ENCODE, D, F, TT, IN_STEPS>;
    using SM = TrainWsSmem<D, TT, IN_STEPS, NH>;
    extern __shared__ __align__(16) unsigned char sm[];
    __half* ws = reinterpret_cast<__half*>(sm);
    float* bs = reinterpret_cast<float*>(sm + Lay::HALVES * 2);
    LevelDev* lvs = reinterpret_cast<LevelDev*>(sm + SM::LV_OFF);
    float* red = reinterpret_cast<float*>(sm + SM::RED_OFF);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const bool producer = warp < 4;
    const int w4 = warp & 3, rtid = tid & 127;   // role-local warp / thread
    const uint32_t mb0 = tc::smem_u32(sm + SM::MBAR_OFF);
    auto full_bar = [&](int b, int w) { return mb0 + 8u * uint32_t(b * 4 + w); };
    auto empty_bar = [&](int b, int w) { return mb0 + 8u * uint32_t(8 + b * 4 + w); };
    const uint32_t dw_bar = mb0 + 8u * 16u;

    if (a.scratch.flags[3] != 0u)
        return;   // invalid input (k_validate): the reference throws before any update
    const MlpShape msh{ s.in_real, s.n_out, s.sigmoid, s.hidden_width };
    load_weights<IN_STEPS, NH>(ws, bs, a.W, a.b, msh);
    for (int i = tid; i < s.grid.L; i += blockDim.x)
        lvs[i] = levels[i];
    for (int i = tid; i < TS * 8; i += blockDim.x) {   // ones blocks (db = dz^T 1)
        const int smp = i >> 3, c = i & 7;
        const __half v = __float2half_rn(c == 0 ? 1.0f : 0.0f);
        *reinterpret_cast<__half*>(sm + SM::ACT0_OFF + kc_off(16 * IN_STEPS + c, smp)) = v;
#pragma unroll
        for (int k = 0; k < NH; ++k)
            *reinterpret_cast<__half*>(sm + SM::ACTH_OFF + k * SM::ACTH_BYTES + kc_off(H + c, smp)) = v;
    }
    if (tid < 16)
        tc::mbar_init(mb0 + 8u * tid, 32);   // full / empty: every lane of the warp arrives
    if (tid == 16)
        tc::mbar_init(dw_bar, 1);            // the dW MMA commit
    if (warp == 4)
        tc::tmem_alloc(reinterpret_cast<uint32_t*>(sm + SM::TSLOT_OFF), SM::TMEM_COLS);
    tc::fence_smem_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tbase = *reinterpret_cast<const uint32_t*>(sm + SM::TSLOT_OFF);
    const int64_t ntiles = (a.B + TS - 1) / TS;
    const int r0 = 16 * w4;
    const TT* tab = static_cast<const TT*>(a.table);
    bool bad = false;
    unsigned int invalid = 0u;

    if (producer) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(NFG_WS_PRODUCER_REGS));
        const SlotsLinear slots{ sm + SM::STAGE_OFF + rtid * SG::SB, 128 * SG::SB };
        int k = 0;
        for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++k) {
            const int b = k & 1;
            const uint32_t use = uint32_t(k >> 1);
            tc::mbar_wait(empty_bar(b, w4), (use & 1u) ^ 1u);   // the consumer took this slot's last tile
            if (a.ready) {   // streamed inputs: this warp's rows landed
                if (lane == 0) {
                    const int64_t last = min(a.B, tile * TS + r0 + 16) - 1;
                    const unsigned int* f = a.ready + (last < a.chunk0 ? 0 : 1 + (last - a.chunk0) / a.chunk);
                    unsigned int v;
                    for (;;) {
                        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
                        if (int(v - a.epoch) >= 0)
                            break;
                        __nanosleep(100);
                    }
                }
                __syncwarp();
            }
            const int64_t sg = tile * TS + r0 + g, sg8 = sg + 8;
            const bool vg = sg < a.B, vg8 = sg8 < a.B;
            float xg[D], xg8[D];
            load_x<D>(xg, a.X, sg, vg);
            load_x<D>(xg8, a.X, sg8, vg8);
            if (a.validate) {   // encode_forward's checks (grid.hpp:226-229)
                const float lo = -1e-6f, hi = 1.0f + 1e-6f;
#pragma unroll
                for (int i = 0; i < D; ++i) {
                    invalid |= (finite_f(xg[i]) ? 0u : 1u) | ((xg[i] < lo || xg[i] > hi) ? 2u : 0u);
                    invalid |= (finite_f(xg8[i]) ? 0u : 1u) | ((xg8[i] < lo || xg8[i] > hi) ? 2u : 0u);
                }
            }
            clamp_x<D>(xg);   // once per sample (the consumers' scatter reads the clamped copy)
            clamp_x<D>(xg8);
            uint32_t afr[IN_STEPS][4];
#pragma unroll
            for (int s0 = 0; s0 < IN_STEPS; s0 += SG::STS) {
#pragma unroll
                for (int sl = 0; sl < SG::STS; ++sl)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int col = 16 * (s0 + sl) + 8 * h + 2 * t;
                        const int p = (sl * 2 + h) * 2;
                        if (s0 + sl < IN_STEPS && vg)
                            gather_issue_lp<D, F, TT, true>(s.grid, lvs, xg, col, tab, slots, p * SG::NE);
                        if (s0 + sl < IN_STEPS && vg8)
                            gather_issue_lp<D, F, TT, true>(s.grid, lvs, xg8, col, tab, slots, (p + 1) * SG::NE);
                    }
                cp_async_wait_all();
                __syncwarp();   // the partner lane's copies landed too
#pragma unroll
                for (int sl = 0; sl < SG::STS; ++sl)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        if (s0 + sl >= IN_STEPS)
                            continue;
                        const int col = 16 * (s0 + sl) + 8 * h + 2 * t;
                        const int p = (sl * 2 + h) * 2;
                        float2 e0 = make_float2(0.f, 0.f), e8 = make_float2(0.f, 0.f);
                        if (vg)
                            e0 = gather_blend_lp<D, F, TT, true>(s.grid, lvs, xg, col, slots, p * SG::NE);
                        if (vg8)
                            e8 = gather_blend_lp<D, F, TT, true>(s.grid, lvs, xg8, col, slots, (p + 1) * SG::NE);
                        afr[s0 + sl][2 * h] = pack_half2(e0.x, e0.y);
                        afr[s0 + sl][2 * h + 1] = pack_half2(e8.x, e8.y);
                    }
                __syncwarp();   // every lane's (and partner's) slots consumed before the next issue
            }
            // hand the fragments and coordinates to consumer warp w4
            unsigned char* hb = sm + SM::HAND_OFF + b * SM::HAND_BYTES;
            uint32_t* hfr = reinterpret_cast<uint32_t*>(hb);
            float* hx = reinterpret_cast<float*>(hb + SM::HAND_FR);
#pragma unroll
            for (int st = 0; st < IN_STEPS; ++st)
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    hfr[(4 * st + e) * 128 + rtid] = afr[st][e];
#pragma unroll
            for (int i = 0; i < D; ++i) {
                hx[i * 128 + rtid] = xg[i];
                hx[(D + i) * 128 + rtid] = xg8[i];
            }
            mbar_arrive(full_bar(b, w4));
        }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(NFG_WS_CONSUMER_REGS));
        const __half* W0s = ws;
        const __half* Whs = ws + Lay::W0_HALVES;
        const __half* Wos = ws + Lay::W0_HALVES + (NH - 1) * Lay::WH_HALVES;
        const float* bout = bs + H * NH;
        auto csync = [] { tc::bar_sync(1, 128); };
        float kscale = 0.0f;
        bool pending = false, first_mma = true;
        uint32_t mphase = 0;
        float dbo4[2][2] = { { 0.0f, 0.0f }, { 0.0f, 0.0f } };
        double loss_acc = 0.0;
        int k = 0;
        for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++k) {
            const int b = k & 1;
            const uint32_t use = uint32_t(k >> 1);
            const int64_t sg = tile * TS + r0 + g, sg8 = sg + 8;
            const bool vg = sg < a.B, vg8 = sg8 < a.B;
            tc::mbar_wait(full_bar(b, w4), use & 1u);
            uint32_t afr[IN_STEPS][4];
            float xg[D], xg8[D];
            {
                const unsigned char* hb = sm + SM::HAND_OFF + b * SM::HAND_BYTES;
                const uint32_t* hfr = reinterpret_cast<const uint32_t*>(hb);
                const float* hx = reinterpret_cast<const float*>(hb + SM::HAND_FR);
#pragma unroll
                for (int st = 0; st < IN_STEPS; ++st)
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        afr[st][e] = hfr[(4 * st + e) * 128 + rtid];
#pragma unroll
                for (int i = 0; i < D; ++i) {
                    xg[i] = hx[i * 128 + rtid];
                    xg8[i] = hx[(D + i) * 128 + rtid];
                }
            }
            mbar_arrive(empty_bar(b, w4));   // the producer may refill this slot
            if (pending) {   // the previous tile's dW MMAs read the operand buffers
                tc::mbar_wait(dw_bar, mphase);
                mphase ^= 1u;
                pending = false;
                tc::fence_after();
            }
            store_a_kc<IN_STEPS>(afr, sm + SM::ACT0_OFF, r0, lane);

            // ---- MLP forward ----------------------------------------------
            float acc[HT][4];
            uint32_t mask[NH];
            uint32_t ah[4][4];
            layer_fwd<IN_STEPS, HT>(afr, W0s, Lay::INS, acc, lane);
            mask[0] = bias_relu<HT>(acc, bs, lane);
            c_to_a<4, false>(acc, ah);
            store_a_kc<4>(ah, sm + SM::ACTH_OFF, r0, lane);
#pragma unroll
            for (int kk = 1; kk < NH; ++kk) {
                layer_fwd<4, HT>(ah, Whs + (kk - 1) * Lay::WH_HALVES, HS, acc, lane);
                mask[kk] = bias_relu<HT>(acc, bs + H * kk, lane);
                c_to_a<4, false>(acc, ah);
                store_a_kc<4>(ah, sm + SM::ACTH_OFF + kk * SM::ACTH_BYTES, r0, lane);
            }
            float ao[2][4];
            layer_fwd<4, 2>(ah, Wos, HS, ao, lane);

            // ---- output activation, loss, dLoss/dpred ----------------------
            float term = 0.0f, mx = 0.0f;
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int col = 8 * j + 2 * t + (e & 1);
                    const bool valid = (e < 2 ? vg : vg8) && col < s.n_out;
                    const int64_t smp = e < 2 ? sg : sg8;
                    const float z = ao[j][e] + bout[col];
                    const float p = s.sigmoid ? 1.0f / (1.0f + expf(-z)) : z;
                    float d = 0.0f;
                    if (valid) {
                        if (a.pred)
                            a.pred[smp * s.n_out + col] = p;
                        d = loss_grad(a.loss_kind, p, a.target[smp * s.n_out + col], term);
                        if (s.sigmoid)
                            d = d * (p * (1.0f - p));
                    }
                    bad |= !sane(d);
                    ao[j][e] = d;
                    mx = fmaxf(mx, fabsf(d));
                }
#pragma unroll
            for (int m = 16; m > 0; m >>= 1) {
                mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, m));
                term += __shfl_xor_sync(0xffffffffu, term, m);
            }
            if (lane == 0) {
                red[w4] = mx;
                loss_acc += double(term);
            }
            csync();
            float tmax = 0.0f;
#pragma unroll
            for (int w = 0; w < TW; ++w)
                tmax = fmaxf(tmax, red[w]);
            float sc = 1.0f;
            if (tmax > 0.0f && tmax <= 1e30f) {
                int ex;
                frexpf(tmax, &ex);
                sc = ldexpf(1.0f, max(-100, min(100, 4 - ex)));
            }
            if (kscale == 0.0f) {
                kscale = sc;
            } else if (sc != kscale) {   // rescale the TMEM accumulators to this tile's scale (exact power of two)
                if (pending) {
                    tc::mbar_wait(dw_bar, mphase);
                    mphase ^= 1u;
                    pending = false;
                    tc::fence_after();
                }
                const float ratio = sc / kscale;
#pragma unroll
                for (int c8 = 0; c8 < (SM::NCOLS + 7) / 8; ++c8) {
                    float v[8];
                    const uint32_t ta = tbase + (uint32_t(32 * w4) << 16) + 8u * c8;
                    tc::ld8(ta, v);
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                        v[i] *= ratio;
                    tc::st8(ta, v);
                }
                tc::wait_st();
                kscale = sc;
            }
            const float isc = 1.0f / sc;

            // ---- MLP backward -----------------------------------------------
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    ao[j][e] *= sc;
            uint32_t azo[1][4];
            c_to_a<1, true>(ao, azo);
            store_a_kc<1>(azo, sm + SM::DZO_OFF, r0, lane);
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const float2 top = unpack_half2(azo[0][2 * j]), bot = unpack_half2(azo[0][2 * j + 1]);
                float sx = top.x + bot.x, sy = top.y + bot.y;
#pragma unroll
                for (int m = 4; m < 32; m <<= 1) {
                    sx += __shfl_xor_sync(0xffffffffu, sx, m);
                    sy += __shfl_xor_sync(0xffffffffu, sy, m);
                }
                dbo4[j][0] = fmaf(sx, isc, dbo4[j][0]);
                dbo4[j][1] = fmaf(sy, isc, dbo4[j][1]);
            }
            layer_bwd<1, HT>(azo, Wos, HS, acc, lane);
            apply_mask<HT>(acc, mask[NH - 1]);
#pragma unroll
            for (int kk = NH - 1; kk >= 1; --kk) {
                c_to_a<4, true>(acc, ah);
                store_a_kc<4>(ah, sm + SM::DZH_OFF + kk * SM::DZH_BYTES, r0, lane);
                layer_bwd<4, HT>(ah, Whs + (kk - 1) * Lay::WH_HALVES, HS, acc, lane);
                apply_mask<HT>(acc, mask[kk - 1]);
            }
            c_to_a<4, true>(acc, ah);
            store_a_kc<4>(ah, sm + SM::DZH_OFF, r0, lane);
            float ay[2 * IN_STEPS][4];
            layer_bwd<4, 2 * IN_STEPS>(ah, W0s, Lay::INS, ay, lane);

            // ---- dY -> encode backward (lane-pair reductions) ----------------
            const float dysc = isc * a.inv_count;
#pragma unroll
            for (int j = 0; j < 2 * IN_STEPS; ++j) {
                const int col = 8 * j + 2 * t;
                const float2 d0 = make_float2(ay[j][0] * dysc, ay[j][1] * dysc);
                const float2 d8 = make_float2(ay[j][2] * dysc, ay[j][3] * dysc);
                bad |= !(sane(d0.x) && sane(d0.y) && sane(d8.x) && sane(d8.y));
                const float2 p0 = make_float2(__shfl_xor_sync(0xffffffffu, d0.x, 1),
                                              __shfl_xor_sync(0xffffffffu, d0.y, 1));
                const float2 p8 = make_float2(__shfl_xor_sync(0xffffffffu, d8.x, 1),
                                              __shfl_xor_sync(0xffffffffu, d8.y, 1));
                if (vg)
                    scatter_pair_lp<D, true>(s.grid, lvs, xg, col, d0, p0, a.table_grad);
                if (vg8)
                    scatter_pair_lp<D, true>(s.grid, lvs, xg8, col, d8, p8, a.table_grad);
            }

            // ---- dW / db += dz^T [act | 1] on tcgen05 (TMEM) -------------------
            tc::fence_smem_async();
            tc::fence_before();
            csync();
            if (rtid == 0) {
                tc::fence_after();
                constexpr int K0 = 16 * IN_STEPS;
                constexpr uint32_t ID0 = tc::idesc_f16_mn(64, K0 + 8), IDH = tc::idesc_f16_mn(64, H + 8),
                                   IDO = tc::idesc_f16_mn(64, OUTP);
                const uint32_t s0a = tc::smem_u32(sm);
                auto slot = [&](int kk) {
                    return tbase + ((kk & 1) ? (16u << 16) : 0u) + uint32_t((kk >> 1) * TcSlots<NH>::COLS);
                };
#pragma unroll
                for (int ks = 0; ks < TS / 16; ++ks) {
                    const uint32_t acc_on = (ks > 0 || !first_mma) ? 1u : 0u;
                    auto dsc = [&](int off) { return tc::desc(s0a + off + 256u * ks, 128u, uint32_t(KC_SBO)); };
                    tc::mma_f16(slot(0), dsc(SM::DZH_OFF), dsc(SM::ACT0_OFF), ID0, acc_on);
#pragma unroll
                    for (int kk = 1; kk < NH; ++kk)
                        tc::mma_f16(slot(kk), dsc(SM::DZH_OFF + kk * SM::DZH_BYTES),
                                    dsc(SM::ACTH_OFF + (kk - 1) * SM::ACTH_BYTES), IDH, acc_on);
                    tc::mma_f16(slot(NH), dsc(SM::ACTH_OFF + (NH - 1) * SM::ACTH_BYTES), dsc(SM::DZO_OFF), IDO,
                                acc_on);
                }
                tc::commit(dw_bar);
            }
            first_mma = false;
            pending = true;
        }
        if (lane == 0 && loss_acc != 0.0)
            atomicAdd(a.scratch.loss_sum, loss_acc);
        // ---- flush the TMEM accumulators (x 1/count) -------------------------
        if (pending) {
            tc::mbar_wait(dw_bar, mphase);
            tc::fence_after();
        }
        const float ic = a.inv_count;
        const int hw = s.hidden_width;
        if (!first_mma) {
            const float fs = ic / kscale;
            const int half = lane >> 4, m = 16 * w4 + (lane & 15);
            const size_t wo_off = size_t(hw) * s.in_real + size_t(NH - 1) * hw * hw;
#pragma unroll
            for (int c8 = 0; c8 < (SM::NCOLS + 7) / 8; ++c8) {
                float v[8];
                tc::ld8(tbase + (uint32_t(32 * w4) << 16) + 8u * c8, v);
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int col = 8 * c8 + i, region = col / TcSlots<NH>::COLS;
                    const int lc = col - region * TcSlots<NH>::COLS, kk = 2 * region + half;
                    if (m >= hw || kk > NH)
                        continue;
                    size_t idx;
                    bool is_b = false;
                    if (kk < NH) {
                        const int nin = kk == 0 ? 16 * IN_STEPS : H, in_k = kk == 0 ? s.in_real : hw;
                        if (lc < in_k)
                            idx = (kk == 0 ? 0 : size_t(hw) * s.in_real + size_t(kk - 1) * hw * hw) + m +
                                  size_t(lc) * hw;
                        else if (lc == nin) {
                            idx = size_t(kk) * hw + m;
                            is_b = true;
                        } else
                            continue;
                    } else {
                        if (lc >= s.n_out)
                            continue;
                        idx = wo_off + lc + size_t(m) * s.n_out;
                    }
                    const float val = v[i] * fs;
                    bad |= !sane(val);
                    atomicAdd((is_b ? a.gb : a.gW) + idx, val);
                }
            }
        }
        float* dbo_s = reinterpret_cast<float*>(sm + SM::DBO_OFF);
        if (g == 0)
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int bb = 0; bb < 2; ++bb)
                    dbo_s[w4 * OUTP + 8 * j + 2 * t + bb] = dbo4[j][bb];
        tc::fence_before();
        csync();
        tc::fence_after();
        if (rtid < s.n_out) {
            float v = 0.0f;
#pragma unroll
            for (int w = 0; w < TW; ++w)
                v += dbo_s[w * OUTP + rtid];
            v *= ic;
            bad |= !sane(v);
            atomicAdd(a.gb + NH * hw + rtid, v);
        }
    }
    tc::fence_before();
    __syncthreads();   // every consumer has read its TMEM columns
    tc::fence_after();
    if (warp == 4)
        tc::tmem_dealloc(tbase, SM::TMEM_COLS);
    if (__any_sync(0xffffffffu, bad) && lane == 0)
        atomicOr(a.scratch.flags, 1u);
    invalid = __reduce_or_sync(0xffffffffu, invalid);
    if (invalid && lane == 0) {
        atomicOr(&a.scratch.flags[3], invalid);
        atomicOr(&a.scratch.flags[1], 1u);
    }
}

}   // namespace nfg
