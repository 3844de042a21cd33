// field_kernels.cuh — the fused training and inference kernels (templates).
//
// k_train: persistent, two CTAs of 4 warps per SM loop over 64-sample tiles.
// Per tile:
//   encode fwd (grid.hpp:245-271)   cp.async corner gathers split over lane
//                                   pairs (encode.cuh), blended straight into
//                                   mma A fragments (+ smem copy)
//   MLP fwd (mlp.hpp:113-123)       activations in registers, smem copy for dW
//   loss + dPred (losses.hpp)       fused in the output epilogue
//   MLP bwd (mlp.hpp:146-157)       dz chain in registers, dz copies in smem
//   encode bwd (grid.hpp:286-294)   straight out of the dY C fragments as
//                                   float2 vector reductions into fp32 grads
//   dW/db                           K = 64-sample MMA from smem, accumulated in
//                                   registers across all tiles of the CTA and
//                                   flushed once per CTA.
// Backward operands are fp16 with a per-tile power-of-two scale (chosen from
// the tile's max |dLoss/dpred|) so gradients of order 1e-6 stay normal; all
// accumulation is fp32 and the scale is removed exactly (powers of two).
//
// k_infer: per-warp 16-sample tiles, no block barriers in the loop; encode ->
// MLP -> output activation (model.cpp:102-109).
#pragma once

#include <type_traits>

#include "encode.cuh"
#include "kernels.h"
#include "mlp_core.cuh"
#include "tc_core.cuh"

namespace nfg {

using namespace mlp;

#ifndef NFG_TW
#define NFG_TW 4
#endif
constexpr int TW = NFG_TW;          // warps per training CTA
constexpr int TS = 16 * NFG_TW;     // samples per training tile (16 per warp)
#ifndef NFG_IW
// One CTA of 24 warps per SM: one copy of the weights leaves the L1 to the
// gathers (+6% over 8 CTAs x 4 warps), and with lane-pair gathers 24 warps at
// 76 registers beat 32 warps at the 64-register cap (+2%, tools/exp_iw.sh).
#define NFG_IW 24
#endif
constexpr int IW = NFG_IW;   // warps per inference CTA

__host__ __device__ constexpr int align16(int x) { return (x + 15) & ~15; }

// Staged-gather geometry of the fused kernel: per pass, STS k16 steps of
// input columns (4 (sample, col-pair) items per step per thread) with NE
// corner elements of SB bytes each, at most 256 B of slots per thread.
template <int SRC, int D, int F, typename TT, int IN_STEPS>
struct StageGeo {
    static constexpr int NE = PairElems<D, F>::NE;
    static constexpr int SB = Stage<F, TT>::SB;
    static constexpr int PER_STEP = 4 * NE * SB;
    static constexpr int STS_RAW = 256 / PER_STEP;
    static constexpr int STS = STS_RAW < 1 ? 1 : (STS_RAW > IN_STEPS ? IN_STEPS : STS_RAW);
    static constexpr int BYTES = SRC == SRC_ENCODE ? TW * 32 * STS * PER_STEP : 0;
};

template <int IN_STEPS, int NH, int STAGE_BYTES = 0, bool ALIAS = false>
struct TrainSmem {
    using Lay = WLayout<IN_STEPS, NH>;
    static constexpr int INS = Lay::INS;
    static constexpr int OS = OUTP + 8;
    static constexpr int LV_OFF = align16(Lay::BYTES);
    static constexpr int ACT0_OFF = LV_OFF + align16(int(sizeof(LevelDev)) * NFG_MAX_LEVELS);
    static constexpr int ACTH_OFF = ACT0_OFF + TS * INS * 2;
    static constexpr int DZH_OFF = ACTH_OFF + NH * TS * HS * 2;
    static constexpr int DZO_OFF = DZH_OFF + NH * TS * HS * 2;
    static constexpr int DB_OFF = DZO_OFF + TS * OS * 2;
    static constexpr int RED_OFF = DB_OFF + (NH + 1) * H * 4;
    static constexpr int STAGE_OFF = align16(RED_OFF + 4 * TW * 4);
    static constexpr int BYTES = STAGE_OFF + (ALIAS ? 0 : STAGE_BYTES);
    static constexpr int GROUP_BYTES = 0;   // one group per CTA
};

// Per-warp aliasing of the gather staging (fp16 tables, F = 2, >= 2 hidden
// layers): a warp's staged corner rows live in the first 64 columns of ITS OWN
// 16 rows of the two hidden-activation and two dz buffers. The warp writes
// those rows only after its own blend (forward / backward of the same tile),
// other warps read them only after the pre-dW barrier, and the end-of-tile
// barrier precedes the next tile's gathers; the padding columns (the ones
// column of the bias gradient) are never touched. Saves the 32 KB staging area
// per CTA, which the SM gives to L1 for the gathers.
template <int SRC, int D, int F, typename TT, int IN_STEPS, int NH>
struct StageAlias {
    using SG = StageGeo<SRC, D, F, TT, IN_STEPS>;
    static constexpr int ROWS = 16;                               // sample rows per warp
    static constexpr int ELEMS = SG::STS * 4 * SG::NE;            // staged elements per thread and pass
#ifdef NFG_PREFETCH
    // gather-ahead (opt-in experiment): the next tile's corner loads are issued
    // right after the loss barrier and land while this tile runs its backward,
    // scatter and dW. Measured 2% SLOWER than the aliased single-tile staging
    // (287 vs 281 us, tools/exp_pf.sh): the two CTAs per SM already overlap one
    // CTA's gathers with the other's compute, and the separate staging area
    // costs L1 capacity.
    static constexpr bool PREFETCH = SRC == SRC_ENCODE && SG::STS >= IN_STEPS;
#else
    static constexpr bool PREFETCH = false;
#endif
#ifdef NFG_NO_ALIAS_STAGE
    static constexpr bool ON = false;
#else
    static constexpr bool ON = !PREFETCH && SRC == SRC_ENCODE && NH >= 2 && SG::SB == 4 && 32 * SG::SB <= 2 * H &&
                               ELEMS <= 4 * ROWS;
#endif
};

// ---- tcgen05 dW (k_train<..., TCW = true>) -----------------------------------
// The per-warp forward / backward chains stay on mma.sync with activations in
// registers (they feed straight from the encode and into the scatter); the
// CTA-wide dW / db reductions over the tile's TS samples run on tcgen05 with the
// accumulators in TMEM across all tiles of the CTA (instead of 62 registers per
// thread). The tile's activations and dz are kept in shared memory in the
// canonical MN-major operand layout with the samples as K:
//   element (feature f, sample s) at (f / 8) * KC_SBO + (s / 8) * 128 + (s % 8) * 16 + (f % 8) * 2
// (core matrices of 8 samples x 8 features; LBO = 128 B between sample blocks,
// SBO = KC_SBO between feature blocks). Layer k's dW^T | db accumulates as
// D_k[unit][in | 1] += dz_k^T act_k (M = 64; the activation buffers carry a
// block whose first feature is 1, so the bias gradient is column `in`); the
// output layer accumulates transposed, D[hidden][out] += act^T dz_out (M = 64,
// N = 16). M = 64 accumulators occupy TMEM lanes 0-15 (or 16-31, "interleaved")
// of each 32-lane subpartition: slot k uses lane half k & 1, columns 72 (k >> 1).
// Validated on the hardware by tools/tc_probe.cu.
constexpr int KC_SBO = TS / 8 * 128;

__device__ __forceinline__ int kc_off(int f, int smp)
{
    return (f >> 3) * KC_SBO + (smp >> 3) * 128 + (smp & 7) * 16 + (f & 7) * 2;
}

// Stores an A-fragment block (samples row0 .. row0+15, 16*KS features) into a
// canonical MN-major buffer (conflict-free: 32 lanes -> 32 banks).
template <int KS>
__device__ __forceinline__ void store_a_kc(const uint32_t (&a)[KS][4], unsigned char* buf, int row0, int lane)
{
    const int g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int s = 0; s < KS; ++s) {
        const int f = 16 * s + 2 * t;
        *reinterpret_cast<uint32_t*>(buf + kc_off(f, row0 + g)) = a[s][0];
        *reinterpret_cast<uint32_t*>(buf + kc_off(f, row0 + g + 8)) = a[s][1];
        *reinterpret_cast<uint32_t*>(buf + kc_off(f + 8, row0 + g)) = a[s][2];
        *reinterpret_cast<uint32_t*>(buf + kc_off(f + 8, row0 + g + 8)) = a[s][3];
    }
}

template <int NH>
struct TcSlots {
    static constexpr int COLS = H + 8;   // columns per TMEM region (a hidden layer's 64 inputs + the db column block)
    __host__ __device__ static constexpr int ncols(int k0)
    {
        int n = 0;
        for (int k = 0; k <= NH; ++k) {
            const int w = k < NH ? (k == 0 ? k0 : H) + 8 : OUTP;
            const int e = (k >> 1) * COLS + w;
            n = e > n ? e : n;
        }
        return n;
    }
};

// NG groups of TW warps per CTA (TCW): the weights, biases and level table
// are shared (one copy per SM), everything from ACT0_OFF on is per group
// (GROUP_BYTES apart); each group runs its own tiles like a CTA of its own,
// synchronising with a named barrier.
template <int IN_STEPS, int NH, int STAGE_BYTES = 0, bool ALIAS = false, int NG = 1>
struct TrainSmemTc {
    using Lay = WLayout<IN_STEPS, NH>;
    static constexpr int K0 = 16 * IN_STEPS;
    static constexpr int LV_OFF = align16(Lay::BYTES);
    static constexpr int ACT0_OFF = (LV_OFF + int(sizeof(LevelDev)) * NFG_MAX_LEVELS + 127) & ~127;
    static constexpr int ACT0_BYTES = (K0 / 8 + 1) * KC_SBO;   // + the ones block
    static constexpr int ACTH_OFF = ACT0_OFF + ACT0_BYTES;
    static constexpr int ACTH_BYTES = (H / 8 + 1) * KC_SBO;    // + the ones block
    static constexpr int DZH_OFF = ACTH_OFF + NH * ACTH_BYTES;
    static constexpr int DZH_BYTES = H / 8 * KC_SBO;
    static constexpr int DZO_OFF = DZH_OFF + NH * DZH_BYTES;
    static constexpr int DZO_BYTES = OUTP / 8 * KC_SBO;
    static constexpr int RED_OFF = DZO_OFF + DZO_BYTES;
    static constexpr int DBO_OFF = RED_OFF + 4 * TW * 4;                 // per-warp output-bias partials
    static constexpr int MBAR_OFF = align16(DBO_OFF + TW * OUTP * 4);
    static constexpr int TSLOT_OFF = MBAR_OFF + 8;
    static constexpr int STAGE_OFF = align16(TSLOT_OFF + 8);
    static constexpr int GROUP_BYTES = ((STAGE_OFF + (ALIAS ? 0 : STAGE_BYTES) - ACT0_OFF) + 127) & ~127;
    static constexpr int BYTES = ACT0_OFF + NG * GROUP_BYTES;
    static constexpr int INS = Lay::INS, OS = OUTP + 8, DB_OFF = RED_OFF;   // (mma.sync-path names; unused)
    static constexpr int NCOLS = TcSlots<NH>::ncols(K0);
    static constexpr uint32_t GROUP_COLS = tc::alloc_cols(NCOLS);       // TMEM columns per group
    static constexpr uint32_t TMEM_COLS = tc::alloc_cols(int(GROUP_COLS) * NG);
};

#ifndef NFG_TRAIN_GROUPS
#define NFG_TRAIN_GROUPS 1   // TCW: groups of TW warps per CTA; 3 (one weight copy per SM) measured slower: 290 vs 271 us
#endif

// Aliased gather staging in the canonical buffers: slot k of this lane lives in
// buffer k / 16 (acth[0], acth[1], dz[0], dz[1]), feature block (k % 16) / 2,
// sample block 2 warp + (k % 2) — the warp's own samples, below the ones block.
template <class SMT>
struct SlotsKC {
    unsigned char* base;   // sm + warp * 256 + lane * SB
    __device__ __forceinline__ unsigned char* ptr(int k) const
    {
        const int b = k >> 4, r = k & 15;
        const int off = b < 2 ? SMT::ACTH_OFF + b * SMT::ACTH_BYTES : SMT::DZH_OFF + (b - 2) * SMT::DZH_BYTES;
        return base + off + (r >> 1) * KC_SBO + (r & 1) * 128;
    }
};

template <int IN_STEPS, int NH>
struct InferSmem {
    using Lay = WLayout<IN_STEPS, NH>;
    static constexpr int LV_OFF = align16(Lay::BYTES);
    static constexpr int BYTES = LV_OFF + align16(int(sizeof(LevelDev)) * NFG_MAX_LEVELS);
};

// Phase timing of k_train (build with -DNFG_PHASE_TIMING; a.phase_clk != null):
// per-warp clock64 deltas of encode / fwd / loss+barrier / bwd / scatter /
// barrier / dW / barrier, summed into a.phase_clk[8].
#ifdef NFG_PHASE_TIMING
#define NFG_PT_DECL unsigned long long pt_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0}, pt_t = 0;
#define NFG_PT_START() pt_t = clock64();
#define NFG_PT(i)                                  \
    {                                              \
        const unsigned long long n_ = clock64();   \
        pt_acc[i] += n_ - pt_t;                    \
        pt_t = n_;                                 \
    }
#define NFG_PT_FLUSH()                                                 \
    if (a.phase_clk && lane == 0)                                      \
        for (int i_ = 0; i_ < 8; ++i_)                                 \
            atomicAdd(a.phase_clk + i_, pt_acc[i_]);
#else
#define NFG_PT_DECL
#define NFG_PT_START()
#define NFG_PT(i)
#define NFG_PT_FLUSH()
#endif

__device__ __forceinline__ bool sane(float v) { return fabsf(v) <= 1e30f; }   // false for NaN/inf/huge

// Input fragments of the warp's 16 rows: encoded from X, or loaded from Y.
// PC: xg / xg8 were clamped once (clamp_x).
template <int SRC, int D, int F, typename TT, int IN_STEPS, bool PC = false, int IP = IP_RUNTIME>
__device__ __forceinline__ void input_frags(uint32_t (&afr)[IN_STEPS][4], const FieldShape& s, const LevelDev* lvs,
                                            const float* xg, const float* xg8, bool vg, bool vg8, int64_t sg,
                                            const float* __restrict__ Y, const void* table, int lane)
{
    const int t = lane & 3;
#pragma unroll
    for (int st = 0; st < IN_STEPS; ++st) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int col = 16 * st + 8 * h + 2 * t;
            float2 e0 = make_float2(0.f, 0.f), e8 = make_float2(0.f, 0.f);
            if (SRC == SRC_ENCODE) {
                const TT* tab = static_cast<const TT*>(table);
#ifndef NFG_NO_LANE_PAIRS
                if constexpr (F == 2) {   // warp-uniform: invalid samples encode x = 0, discarded
                    e0 = encode_pair_lp<D, F, TT, PC, IP>(s.grid, lvs, xg, col, tab);
                    e8 = encode_pair_lp<D, F, TT, PC, IP>(s.grid, lvs, xg8, col, tab);
                    if (!vg)
                        e0 = make_float2(0.f, 0.f);
                    if (!vg8)
                        e8 = make_float2(0.f, 0.f);
                } else
#endif
                {
                    if (vg)
                        e0 = encode_pair<D, F, TT>(s.grid, lvs, xg, col, tab);
                    if (vg8)
                        e8 = encode_pair<D, F, TT>(s.grid, lvs, xg8, col, tab);
                }
            } else {
                const int w = s.in_real;
                if (vg) {
                    if (col < w) e0.x = Y[sg * w + col];
                    if (col + 1 < w) e0.y = Y[sg * w + col + 1];
                }
                if (vg8) {
                    if (col < w) e8.x = Y[(sg + 8) * w + col];
                    if (col + 1 < w) e8.y = Y[(sg + 8) * w + col + 1];
                }
            }
            afr[st][2 * h] = pack_half2(e0.x, e0.y);
            afr[st][2 * h + 1] = pack_half2(e8.x, e8.y);
        }
    }
}

template <int D>
__device__ __forceinline__ void load_x(float* x, const float* __restrict__ X, int64_t sidx, bool valid)
{
#pragma unroll
    for (int i = 0; i < D; ++i)
        x[i] = valid ? X[sidx * D + i] : 0.0f;
}

// 2 CTAs of 4 warps per SM (measured 5% faster than 1 CTA of 8 warps: the two
// CTAs drift out of phase, overlapping one's gathers/reductions with the
// other's tensor-core MLP).
#ifndef NFG_TRAIN_MIN_BLOCKS
#define NFG_TRAIN_MIN_BLOCKS 2
#endif
// With the dW accumulators in TMEM (TCW) the kernel fits 3 CTAs per SM.
#ifndef NFG_TRAIN_MIN_BLOCKS_TC
#define NFG_TRAIN_MIN_BLOCKS_TC 3
#endif
template <bool TCW>
struct TrainGroups {
    static constexpr int NG = TCW ? NFG_TRAIN_GROUPS : 1;   // groups of TW warps per CTA
    static constexpr int MIN_BLOCKS = TCW ? (NFG_TRAIN_MIN_BLOCKS_TC + NG - 1) / NG : NFG_TRAIN_MIN_BLOCKS;
};

// IP: interpolation mode (nfg_common.cuh), fixed per instantiation for the
// encoding kernels so the linear path carries no smoothstep work.
template <int SRC, int GRAD, int SINK, int D, int F, typename TT, int IN_STEPS, int NH, bool TCW = false,
          int IP = IP_RUNTIME>
__global__ void __launch_bounds__(TW * 32 * TrainGroups<TCW>::NG, TrainGroups<TCW>::MIN_BLOCKS)
k_train(const TrainArgs a, const FieldShape s, const LevelDev* __restrict__ levels)
{
    using Lay = WLayout<IN_STEPS, NH>;
    using SG = StageGeo<SRC, D, F, TT, IN_STEPS>;
    using SA = StageAlias<SRC, D, F, TT, IN_STEPS, NH>;
    static_assert(!(TCW && SA::PREFETCH), "gather-ahead is an mma.sync-path experiment");
    constexpr int NG = TrainGroups<TCW>::NG;
    using SM = std::conditional_t<TCW, TrainSmemTc<IN_STEPS, NH, SG::BYTES, SA::ON, NG>,
                                  TrainSmem<IN_STEPS, NH, SG::BYTES, SA::ON>>;
    extern __shared__ __align__(16) unsigned char sm[];
    // TCW: NG groups of TW warps; a group works like a CTA of its own (its
    // tiles, buffers, barrier, TMEM columns); tid / warp are group-local
    const int ctid = threadIdx.x, gi = (ctid >> 5) / TW;
    const int64_t vblk = int64_t(blockIdx.x) * NG + gi, vgrid = int64_t(gridDim.x) * NG;
    unsigned char* const smg = sm + (TCW ? gi * SM::GROUP_BYTES : 0);   // this group's buffers
    auto gsync = [&] {
        if constexpr (NG == 1)
            __syncthreads();
        else
            tc::bar_sync(1 + gi, TW * 32);
    };
    __half* ws = reinterpret_cast<__half*>(sm);
    float* bs = reinterpret_cast<float*>(sm + Lay::HALVES * 2);
    LevelDev* lvs = reinterpret_cast<LevelDev*>(sm + SM::LV_OFF);
    __half* act0 = reinterpret_cast<__half*>(smg + SM::ACT0_OFF);
    __half* acth = reinterpret_cast<__half*>(smg + SM::ACTH_OFF);
    __half* dzh = reinterpret_cast<__half*>(smg + SM::DZH_OFF);
    __half* dzo = reinterpret_cast<__half*>(smg + SM::DZO_OFF);
    float* db = reinterpret_cast<float*>(smg + SM::DB_OFF);
    float* red = reinterpret_cast<float*>(smg + SM::RED_OFF);

    const int tid = ctid % (TW * 32), lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
    // lane-pair gathers / reductions (encode.cuh): one level per lane (F == 2)
#ifdef NFG_NO_LANE_PAIRS
    constexpr bool LPG = false, LPS = false;
#else
    constexpr bool LPG = SRC == SRC_ENCODE && F == 2, LPS = SINK == SINK_SCATTER && F == 2;
#endif
    // programmatic dependent launch: this grid may have been scheduled while
    // the previous kernel (the step's scratch reset, behind Adam) drained;
    // wait for it before reading the scratch, weights and tables. The
    // optimizer launched behind this kernel may in turn get scheduled as CTAs
    // retire; it waits for this grid's completion.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    if (a.scratch.flags[3] != 0u)
        return;   // invalid input (k_validate): the reference throws before any update
    const MlpShape msh{ s.in_real, s.n_out, s.sigmoid, s.hidden_width };
    load_weights<IN_STEPS, NH>(ws, bs, a.W, a.b, msh);
    if (SRC == SRC_ENCODE)
        for (int i = ctid; i < s.grid.L; i += blockDim.x)
            lvs[i] = levels[i];
    uint32_t tbase = 0, mbar = 0;
    if constexpr (TCW) {
        // ones blocks of the activation buffers (db = dz^T 1), TMEM, mbarrier
        for (int i = tid; i < TS * 8; i += TW * 32) {
            const int smp = i >> 3, c = i & 7;
            const __half v = __float2half_rn(c == 0 ? 1.0f : 0.0f);
            *reinterpret_cast<__half*>(smg + SM::ACT0_OFF + kc_off(16 * IN_STEPS + c, smp)) = v;
#pragma unroll
            for (int k = 0; k < NH; ++k)
                *reinterpret_cast<__half*>(smg + SM::ACTH_OFF + k * SM::ACTH_BYTES + kc_off(H + c, smp)) = v;
        }
        mbar = tc::smem_u32(smg + SM::MBAR_OFF);
        if (tid == 0)
            tc::mbar_init(mbar, 1);
        if (ctid < 32)   // one allocation for the CTA; group gi uses columns [gi, gi + 1) * GROUP_COLS
            tc::tmem_alloc(reinterpret_cast<uint32_t*>(sm + SM::TSLOT_OFF), SM::TMEM_COLS);
        tc::fence_smem_async();
        tc::fence_before();
        __syncthreads();
        tc::fence_after();
        tbase = *reinterpret_cast<const uint32_t*>(sm + SM::TSLOT_OFF) + uint32_t(gi) * SM::GROUP_COLS;
    }
    // padding columns of the activation buffers: a 1 then zeros (db_tile)
    for (int r = tid; !TCW && r < TS; r += blockDim.x) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            act0[r * SM::INS + 16 * IN_STEPS + c] = __float2half_rn(c == 0 ? 1.0f : 0.0f);
#pragma unroll
            for (int k = 0; k < NH; ++k)
                acth[k * TS * HS + r * HS + H + c] = __float2half_rn(c == 0 ? 1.0f : 0.0f);
        }
    }
    __syncthreads();

    const __half* W0s = ws;
    const __half* Whs = ws + Lay::W0_HALVES;
    const __half* Wos = ws + Lay::W0_HALVES + (NH - 1) * Lay::WH_HALVES;
    const float* bout = bs + H * NH;

    constexpr int P0 = 4 * IN_STEPS, PH = 16, PO = 4;
    constexpr int C0 = (P0 + TW - 1) / TW, CH = PH / TW, NHM = NH > 1 ? NH - 1 : 1;
    float dw0[C0][2][4], dwh[NHM][CH][2][4], dwo[2][4];
    float dbh[NH][2], dbo[2] = { 0.0f, 0.0f };
#pragma unroll
    for (int k = 0; k < NH; ++k)
        dbh[k][0] = dbh[k][1] = 0.0f;
#pragma unroll
    for (int c = 0; c < C0; ++c)
#pragma unroll
        for (int e = 0; e < 8; ++e)
            dw0[c][e >> 2][e & 3] = 0.0f;
#pragma unroll
    for (int k = 0; k < NHM; ++k)
#pragma unroll
        for (int c = 0; c < CH; ++c)
#pragma unroll
            for (int e = 0; e < 8; ++e)
                dwh[k][c][e >> 2][e & 3] = 0.0f;
#pragma unroll
    for (int e = 0; e < 8; ++e)
        dwo[e >> 2][e & 3] = 0.0f;

    bool bad = false;
    unsigned int invalid = 0u;
    double loss_acc = 0.0;   // this warp's loss sum over its tiles (lane 0)
    // TCW: dz scale of the TMEM accumulators (power of two: the scale of the
    // tile last added; a tile with another scale rescales them first), the
    // pending dW commit, the output bias gradient (lanes g == 0)
    float kscale = 0.0f;
    bool pending = false, first_mma = true;
    uint32_t mphase = 0;
    float dbo4[2][2] = { { 0.0f, 0.0f }, { 0.0f, 0.0f } };
    NFG_PT_DECL
    const int64_t ntiles = (a.B + TS - 1) / TS;
    const int r0 = 16 * warp;
    const TT* tab = static_cast<const TT*>(a.table);
    // streamed inputs: thread 0 waits for the chunk holding tile tl's last sample
    auto wait_ready = [&](int64_t tl) {
        if (a.ready && tid == 0) {
            const int64_t last = min(a.B, (tl + 1) * TS) - 1;
            const unsigned int* f = a.ready + (last < a.chunk0 ? 0 : 1 + (last - a.chunk0) / a.chunk);
            unsigned int v;
            for (;;) {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
                if (int(v - a.epoch) >= 0)
                    break;
                __nanosleep(100);
            }
        }
    };
    auto load_inputs = [&](int64_t tl, float* x, float* x8) {
        const int64_t s0_ = tl * TS + r0 + g, s8_ = s0_ + 8;
        load_x<D>(x, a.X, s0_, s0_ < a.B);
        load_x<D>(x8, a.X, s8_, s8_ < a.B);
        if (a.validate) {   // encode_forward's checks (grid.hpp:226-229)
            const float lo = -1e-6f, hi = 1.0f + 1e-6f;
#pragma unroll
            for (int i = 0; i < D; ++i) {
                invalid |= (finite_f(x[i]) ? 0u : 1u) | ((x[i] < lo || x[i] > hi) ? 2u : 0u);
                invalid |= (finite_f(x8[i]) ? 0u : 1u) | ((x8[i] < lo || x8[i] > hi) ? 2u : 0u);
            }
        }
        // clamp once per sample; every level's corners skip their own clamp
        clamp_x<D>(x);
        clamp_x<D>(x8);
    };
    // corner loads of one pass (SG::STS k16 steps) as cp.async copies
    auto issue_pass = [&](int s0, const auto& slots, const float* x, const float* x8, bool v, bool v8) {
#pragma unroll
        for (int sl = 0; sl < SG::STS; ++sl)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int col = 16 * (s0 + sl) + 8 * h + 2 * t;
                const int p = (sl * 2 + h) * 2;
                if constexpr (LPG) {
                    if (s0 + sl < IN_STEPS && v)
                        gather_issue_lp<D, F, TT, true, IP>(s.grid, lvs, x, col, tab, slots, p * SG::NE);
                    if (s0 + sl < IN_STEPS && v8)
                        gather_issue_lp<D, F, TT, true, IP>(s.grid, lvs, x8, col, tab, slots, (p + 1) * SG::NE);
                } else {
                    if (s0 + sl < IN_STEPS && v)
                        gather_issue<D, F, TT>(s.grid, lvs, x, col, tab, slots, p * SG::NE);
                    if (s0 + sl < IN_STEPS && v8)
                        gather_issue<D, F, TT>(s.grid, lvs, x8, col, tab, slots, (p + 1) * SG::NE);
                }
            }
    };
    auto blend_pass = [&](int s0, const auto& slots, const float* x, const float* x8, bool v, bool v8,
                          uint32_t (&fr)[IN_STEPS][4]) {
#pragma unroll
        for (int sl = 0; sl < SG::STS; ++sl)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (s0 + sl >= IN_STEPS)
                    continue;
                const int col = 16 * (s0 + sl) + 8 * h + 2 * t;
                const int p = (sl * 2 + h) * 2;
                float2 e0 = make_float2(0.f, 0.f), e8 = make_float2(0.f, 0.f);
                if constexpr (LPG) {
                    if (v)
                        e0 = gather_blend_lp<D, F, TT, true, IP>(s.grid, lvs, x, col, slots, p * SG::NE);
                    if (v8)
                        e8 = gather_blend_lp<D, F, TT, true, IP>(s.grid, lvs, x8, col, slots, (p + 1) * SG::NE);
                } else {
                    if (v)
                        e0 = gather_blend<D, F, TT>(s.grid, lvs, x, col, slots, p * SG::NE);
                    if (v8)
                        e8 = gather_blend<D, F, TT>(s.grid, lvs, x8, col, slots, (p + 1) * SG::NE);
                }
                fr[s0 + sl][2 * h] = pack_half2(e0.x, e0.y);
                fr[s0 + sl][2 * h + 1] = pack_half2(e8.x, e8.y);
            }
    };
    const SlotsLinear lin_slots{ smg + SM::STAGE_OFF + tid * SG::SB, TW * 32 * SG::SB };
    float xn[D], xn8[D];   // gather-ahead: inputs of the next tile
    if (SA::PREFETCH && vblk < ntiles) {
        wait_ready(vblk);
        if (a.ready)
            gsync();
        load_inputs(vblk, xn, xn8);
        const int64_t s0_ = vblk * TS + r0 + g;
        issue_pass(0, lin_slots, xn, xn8, s0_ < a.B, s0_ + 8 < a.B);
    }
    for (int64_t tile = vblk; tile < ntiles; tile += vgrid) {
        NFG_PT_START();
        if (TCW && pending) {   // the previous tile's dW MMAs read the activation / dz / staging buffers
            tc::mbar_wait(mbar, mphase);
            mphase ^= 1u;
            pending = false;
            tc::fence_after();
        }
        const int64_t sg = tile * TS + r0 + g, sg8 = sg + 8;
        const bool vg = sg < a.B, vg8 = sg8 < a.B;
        if (!SA::PREFETCH && a.ready) {   // streamed inputs: wait for this tile's chunk to land
            wait_ready(tile);
            gsync();
        }
        float xg[D], xg8[D];
        if (SA::PREFETCH) {
#pragma unroll
            for (int i = 0; i < D; ++i) {
                xg[i] = xn[i];
                xg8[i] = xn8[i];
            }
        } else if (SRC == SRC_ENCODE) {
            load_inputs(tile, xg, xg8);
        }
        // ---- encode / load inputs -------------------------------------
        uint32_t afr[IN_STEPS][4];
        if (SRC == SRC_ENCODE) {
            // all corner loads of SG::STS k16 steps in flight at once (cp.async)
            auto encode_all = [&](const auto& slots) {
#pragma unroll
                for (int s0 = 0; s0 < IN_STEPS; s0 += SG::STS) {
                    issue_pass(s0, slots, xg, xg8, vg, vg8);
                    cp_async_wait_all();
                    if (LPG)
                        __syncwarp();   // the partner lane's copies landed too
                    blend_pass(s0, slots, xg, xg8, vg, vg8, afr);
                    if (SA::ON && s0 + SG::STS < IN_STEPS)
                        __syncwarp();   // next pass reuses the warp's rows
                }
            };
            if constexpr (SA::PREFETCH) {
                cp_async_wait_all();   // this tile's loads, issued during the previous tile
                if (LPG)
                    __syncwarp();
                blend_pass(0, lin_slots, xg, xg8, vg, vg8, afr);
            } else if constexpr (SA::ON && TCW) {
                const SlotsKC<SM> slots{ smg + warp * 256 + lane * SG::SB };
                encode_all(slots);
                __syncwarp();   // every lane's staged rows consumed before the warp writes them
            } else if constexpr (SA::ON) {
                SlotsChunked<SA::ROWS, HS * 2, 4> slots;
                slots.chunk[0] = reinterpret_cast<unsigned char*>(acth + r0 * HS);
                slots.chunk[1] = reinterpret_cast<unsigned char*>(acth + TS * HS + r0 * HS);
                slots.chunk[2] = reinterpret_cast<unsigned char*>(dzh + r0 * HS);
                slots.chunk[3] = reinterpret_cast<unsigned char*>(dzh + TS * HS + r0 * HS);
                slots.lane_off = lane * SG::SB;
                encode_all(slots);
                __syncwarp();   // every lane's staged rows consumed before the warp writes them
            } else {
                encode_all(lin_slots);
            }
        } else {
            input_frags<SRC, D, F, TT, IN_STEPS>(afr, s, lvs, xg, xg8, vg, vg8, sg, a.Y, a.table, lane);
        }
        if constexpr (TCW)
            store_a_kc<IN_STEPS>(afr, smg + SM::ACT0_OFF, r0, lane);
        else
            store_a<IN_STEPS>(afr, act0, SM::INS, r0, lane);
        NFG_PT(0);

        // ---- MLP forward --------------------------------------------------
        float acc[HT][4];
        uint32_t mask[NH];
        uint32_t ah[4][4];
        layer_fwd<IN_STEPS, HT>(afr, W0s, SM::INS, acc, lane);
        mask[0] = bias_relu<HT>(acc, bs, lane);
        c_to_a<4, false>(acc, ah);
        if constexpr (TCW)
            store_a_kc<4>(ah, smg + SM::ACTH_OFF, r0, lane);
        else
            store_a<4>(ah, acth, HS, r0, lane);
#pragma unroll
        for (int k = 1; k < NH; ++k) {
            layer_fwd<4, HT>(ah, Whs + (k - 1) * Lay::WH_HALVES, HS, acc, lane);
            mask[k] = bias_relu<HT>(acc, bs + H * k, lane);
            c_to_a<4, false>(acc, ah);
            if constexpr (TCW)
                store_a_kc<4>(ah, smg + SM::ACTH_OFF + k * SM::ACTH_BYTES, r0, lane);
            else
                store_a<4>(ah, acth + k * TS * HS, HS, r0, lane);
        }
        float ao[2][4];
        layer_fwd<4, 2>(ah, Wos, HS, ao, lane);
        NFG_PT(1);

        // ---- output activation, loss, dLoss/dpred --------------------------
        float term = 0.0f, mx = 0.0f;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
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
                    if (GRAD == GRAD_LOSS)
                        d = loss_grad(a.loss_kind, p, a.target[smp * s.n_out + col], term);
                    else
                        d = a.dout[smp * s.n_out + col];
                    if (s.sigmoid)
                        d = d * (p * (1.0f - p));
                }
                bad |= !sane(d);
                ao[j][e] = d;
                mx = fmaxf(mx, fabsf(d));
            }
        }
#pragma unroll
        for (int m = 16; m > 0; m >>= 1) {
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, m));
            term += __shfl_xor_sync(0xffffffffu, term, m);
        }
        if (lane == 0) {
            red[warp] = mx;
            if (GRAD == GRAD_LOSS)
                loss_acc += double(term);   // one atomic per warp at the end, not per tile
        }
        const int64_t next_tile = tile + vgrid;
        if (SA::PREFETCH && next_tile < ntiles)
            wait_ready(next_tile);   // published to the CTA by the barrier below
        gsync();
        NFG_PT(2);
        if (SA::PREFETCH && next_tile < ntiles) {
            // every warp has blended this tile (barrier above): its slots are free
            load_inputs(next_tile, xn, xn8);
            const int64_t s0_ = next_tile * TS + r0 + g;
            issue_pass(0, lin_slots, xn, xn8, s0_ < a.B, s0_ + 8 < a.B);
        }
        float tmax = 0.0f;
#pragma unroll
        for (int w = 0; w < TW; ++w)
            tmax = fmaxf(tmax, red[w]);
        float sc = 1.0f, isc = 1.0f;
        if (tmax > 0.0f && tmax <= 1e30f) {
            int ex;
            frexpf(tmax, &ex);                 // tmax < 2^ex
            const int k = max(-100, min(100, 4 - ex));   // scaled max < 16
            sc = ldexpf(1.0f, k);
            isc = ldexpf(1.0f, -k);
        }
        if constexpr (TCW) {
            // the TMEM accumulators hold dz^T act at the scale of the tile last
            // added; a tile with another power-of-two scale first rescales them
            // by the exact ratio (fp32, in place), so every tile's fp16 dz
            // operands use the tile's own scale (as the mma.sync reduction)
            if (kscale == 0.0f) {
                kscale = sc;
            } else if (sc != kscale) {
                if (pending) {
                    tc::mbar_wait(mbar, mphase);
                    mphase ^= 1u;
                    pending = false;
                    tc::fence_after();
                }
                const float ratio = sc / kscale;
#pragma unroll
                for (int c8 = 0; c8 < (SM::NCOLS + 7) / 8; ++c8) {
                    float v[8];
                    const uint32_t ta = tbase + (uint32_t(32 * warp) << 16) + 8u * c8;
                    tc::ld8(ta, v);
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                        v[i] *= ratio;
                    tc::st8(ta, v);
                }
                tc::wait_st();
                kscale = sc;
            }
        }

        // ---- MLP backward ---------------------------------------------------
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int e = 0; e < 4; ++e)
                ao[j][e] *= sc;
        uint32_t azo[1][4];
        c_to_a<1, true>(ao, azo);
        if constexpr (TCW) {
            store_a_kc<1>(azo, smg + SM::DZO_OFF, r0, lane);
            // output bias gradient from the same fp16 dz the MMAs see
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
        } else {
            store_a<1>(azo, dzo, SM::OS, r0, lane);
        }
        layer_bwd<1, HT>(azo, Wos, HS, acc, lane);
        apply_mask<HT>(acc, mask[NH - 1]);
#pragma unroll
        for (int k = NH - 1; k >= 1; --k) {
            c_to_a<4, true>(acc, ah);
            if constexpr (TCW)
                store_a_kc<4>(ah, smg + SM::DZH_OFF + k * SM::DZH_BYTES, r0, lane);
            else
                store_a<4>(ah, dzh + k * TS * HS, HS, r0, lane);
            layer_bwd<4, HT>(ah, Whs + (k - 1) * Lay::WH_HALVES, HS, acc, lane);
            apply_mask<HT>(acc, mask[k - 1]);
        }
        c_to_a<4, true>(acc, ah);
        if constexpr (TCW)
            store_a_kc<4>(ah, smg + SM::DZH_OFF, r0, lane);
        else
            store_a<4>(ah, dzh, HS, r0, lane);
        float ay[2 * IN_STEPS][4];
        layer_bwd<4, 2 * IN_STEPS>(ah, W0s, SM::INS, ay, lane);

        NFG_PT(3);
        // ---- dY -> encode backward / store -------------------------------------
        const float dysc = isc * a.inv_count;
#pragma unroll
        for (int j = 0; j < 2 * IN_STEPS; ++j) {
            const int col = 8 * j + 2 * t;
            const float2 d0 = make_float2(ay[j][0] * dysc, ay[j][1] * dysc);
            const float2 d8 = make_float2(ay[j][2] * dysc, ay[j][3] * dysc);
            bad |= !(sane(d0.x) && sane(d0.y) && sane(d8.x) && sane(d8.y));
            if constexpr (LPS) {   // levels >= L (cols >= in_real) are skipped per level inside
                const float2 p0 = make_float2(__shfl_xor_sync(0xffffffffu, d0.x, 1),
                                              __shfl_xor_sync(0xffffffffu, d0.y, 1));
                const float2 p8 = make_float2(__shfl_xor_sync(0xffffffffu, d8.x, 1),
                                              __shfl_xor_sync(0xffffffffu, d8.y, 1));
                if (vg)
                    scatter_pair_lp<D, true, IP>(s.grid, lvs, xg, col, d0, p0, a.table_grad);
                if (vg8)
                    scatter_pair_lp<D, true, IP>(s.grid, lvs, xg8, col, d8, p8, a.table_grad);
                continue;
            }
            if (col >= s.in_real)
                continue;
#ifdef NFG_EXP_SKIP_LEVELS   // experiment builds only (tools/kbench.cu): drop coarse-level reductions
            if (col / F < NFG_EXP_SKIP_LEVELS)
                continue;
#endif
            if (SINK == SINK_SCATTER) {
                if (vg)
                    scatter_pair<D, F>(s.grid, lvs, xg, col, d0, a.table_grad);
                if (vg8)
                    scatter_pair<D, F>(s.grid, lvs, xg8, col, d8, a.table_grad);
            } else {
                const int w = s.in_real;
                if (vg) {
                    a.dY[sg * w + col] = d0.x;
                    if (col + 1 < w) a.dY[sg * w + col + 1] = d0.y;
                }
                if (vg8) {
                    a.dY[sg8 * w + col] = d8.x;
                    if (col + 1 < w) a.dY[sg8 * w + col + 1] = d8.y;
                }
            }
        }
        NFG_PT(4);
        if constexpr (TCW) {
            // ---- dW / db += dz^T [act | 1] on tcgen05, accumulated in TMEM ----------
            tc::fence_smem_async();   // this tile's activation / dz stores -> tensor core
            tc::fence_before();
            gsync();
            NFG_PT(5);
            if (tid == 0) {
                tc::fence_after();
                constexpr int K0 = 16 * IN_STEPS;
                constexpr uint32_t ID0 = tc::idesc_f16_mn(64, K0 + 8), IDH = tc::idesc_f16_mn(64, H + 8),
                                   IDO = tc::idesc_f16_mn(64, OUTP);
                const uint32_t s0 = tc::smem_u32(smg);
                auto slot = [&](int k) {
                    return tbase + ((k & 1) ? (16u << 16) : 0u) + uint32_t((k >> 1) * TcSlots<NH>::COLS);
                };
#pragma unroll
                for (int ks = 0; ks < TS / 16; ++ks) {
                    const uint32_t acc_on = (ks > 0 || !first_mma) ? 1u : 0u;
                    auto dsc = [&](int off) { return tc::desc(s0 + off + 256u * ks, 128u, uint32_t(KC_SBO)); };
                    tc::mma_f16(slot(0), dsc(SM::DZH_OFF), dsc(SM::ACT0_OFF), ID0, acc_on);
#pragma unroll
                    for (int k = 1; k < NH; ++k)
                        tc::mma_f16(slot(k), dsc(SM::DZH_OFF + k * SM::DZH_BYTES),
                                    dsc(SM::ACTH_OFF + (k - 1) * SM::ACTH_BYTES), IDH, acc_on);
                    tc::mma_f16(slot(NH), dsc(SM::ACTH_OFF + (NH - 1) * SM::ACTH_BYTES), dsc(SM::DZO_OFF), IDO,
                                acc_on);
                }
                tc::commit(mbar);
            }
            first_mma = false;
            pending = true;
            NFG_PT(6);
            NFG_PT(7);
            continue;
        }
        __syncthreads();
        NFG_PT(5);

        // ---- dW = dz^T act over the tile's 128 samples ------------------------
#pragma unroll
        for (int c = 0; c < C0; ++c) {
            const int p = warp + c * TW;
            if (p < P0) {
                float c0[4], c1[4];
                dw_pair<TS>(c0, c1, dzh, HS, act0, SM::INS, p / IN_STEPS, p % IN_STEPS, lane);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    dw0[c][0][e] = fmaf(c0[e], isc, dw0[c][0][e]);
                    dw0[c][1][e] = fmaf(c1[e], isc, dw0[c][1][e]);
                }
            }
        }
#pragma unroll
        for (int k = 1; k < NH; ++k)
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                const int p = warp + c * TW;
                float c0[4], c1[4];
                dw_pair<TS>(c0, c1, dzh + k * TS * HS, HS, acth + (k - 1) * TS * HS, HS, p / 4, p % 4, lane);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    dwh[k - 1][c][0][e] = fmaf(c0[e], isc, dwh[k - 1][c][0][e]);
                    dwh[k - 1][c][1][e] = fmaf(c1[e], isc, dwh[k - 1][c][1][e]);
                }
            }
        if (warp < PO) {
            float c0[4], c1[4];
            dw_pair<TS>(c0, c1, dzo, SM::OS, acth + (NH - 1) * TS * HS, HS, 0, warp, lane);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                dwo[0][e] = fmaf(c0[e], isc, dwo[0][e]);
                dwo[1][e] = fmaf(c1[e], isc, dwo[1][e]);
            }
        }
        // db = dz^T * 1 through the ones column of each activation buffer
        if (warp < 4) {
#pragma unroll
            for (int k = 0; k < NH; ++k) {
                float c[4];
                if (k == 0)
                    db_tile<TS>(c, dzh, HS, act0, SM::INS, warp, 16 * IN_STEPS, lane);
                else
                    db_tile<TS>(c, dzh + k * TS * HS, HS, acth + (k - 1) * TS * HS, HS, warp, H, lane);
                dbh[k][0] = fmaf(c[0], isc, dbh[k][0]);
                dbh[k][1] = fmaf(c[2], isc, dbh[k][1]);
            }
        }
        if (warp == TW - 1) {
            float c[4];
            db_tile<TS>(c, dzo, SM::OS, acth + (NH - 1) * TS * HS, HS, 0, H, lane);
            dbo[0] = fmaf(c[0], isc, dbo[0]);
            dbo[1] = fmaf(c[2], isc, dbo[1]);
        }
        NFG_PT(6);
        __syncthreads();
        NFG_PT(7);
    }

    NFG_PT_FLUSH();
    // ---- flush per-CTA dW / db (x 1/count) ----------------------------------
    const float ic = a.inv_count;
    const int hw = s.hidden_width;
    if constexpr (TCW) {
        if (pending) {
            tc::mbar_wait(mbar, mphase);
            tc::fence_after();
        }
        if (!first_mma) {
            // warp w, lane L < 16 (L >= 16): TMEM lane 32 w + L = row 16 w + (L % 16) of
            // the lane-half-0 (half-1) accumulator slots
            const float fs = ic / kscale;
            const int half = lane >> 4, m = 16 * warp + (lane & 15);
            const size_t wo_off = size_t(hw) * s.in_real + size_t(NH - 1) * hw * hw;
#pragma unroll
            for (int c8 = 0; c8 < (SM::NCOLS + 7) / 8; ++c8) {
                float v[8];
                tc::ld8(tbase + (uint32_t(32 * warp) << 16) + 8u * c8, v);
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int col = 8 * c8 + i, region = col / TcSlots<NH>::COLS;
                    const int lc = col - region * TcSlots<NH>::COLS, k = 2 * region + half;
                    if (m >= hw || k > NH)
                        continue;
                    size_t idx;
                    bool is_b = false;
                    if (k < NH) {
                        const int nin = k == 0 ? 16 * IN_STEPS : H, in_k = k == 0 ? s.in_real : hw;
                        if (lc < in_k)
                            idx = (k == 0 ? 0 : size_t(hw) * s.in_real + size_t(k - 1) * hw * hw) + m + size_t(lc) * hw;
                        else if (lc == nin) {
                            idx = size_t(k) * hw + m;
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
                    if (a.part_wb)
                        a.part_wb[vblk * a.n_wb + (is_b ? a.n_w : 0) + idx] = val;
                    else
                        atomicAdd((is_b ? a.gb : a.gW) + idx, val);
                }
            }
        }
        // output bias: per-warp partials (lanes g == 0), summed over the warps in order
        float* dbo_s = reinterpret_cast<float*>(smg + SM::DBO_OFF);
        if (g == 0)
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int b = 0; b < 2; ++b)
                    dbo_s[warp * OUTP + 8 * j + 2 * t + b] = dbo4[j][b];
        tc::fence_before();
        gsync();
        tc::fence_after();
        if (tid < s.n_out) {
            float v = 0.0f;
#pragma unroll
            for (int w = 0; w < TW; ++w)
                v += dbo_s[w * OUTP + tid];
            v *= ic;
            bad |= !sane(v);
            if (a.part_wb)
                a.part_wb[vblk * a.n_wb + a.n_w + NH * hw + tid] = v;
            else
                atomicAdd(a.gb + NH * hw + tid, v);
        }
        if constexpr (NG > 1)
            __syncthreads();   // every group has read its TMEM columns (before the dbo barrier)
        if (ctid < 32)
            tc::tmem_dealloc(*reinterpret_cast<const uint32_t*>(sm + SM::TSLOT_OFF), SM::TMEM_COLS);
    } else {
    auto flush = [&](const float (&cq)[2][4], int mt, int np, int out_k, int in_k, size_t woff) {
#ifdef NFG_EXP_NO_FLUSH   // experiment builds only (tools/kbench.cu): upper bound of the dW flush cost
        return;
#endif
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int m = 16 * mt + g + (e >= 2 ? 8 : 0);
                const int n = 8 * (2 * np + q) + 2 * t + (e & 1);
                if (m < out_k && n < in_k) {
                    const float v = cq[q][e] * ic;
                    bad |= !sane(v);
                    if (a.part_wb)
                        a.part_wb[blockIdx.x * a.n_wb + woff + m + size_t(n) * out_k] = v;
                    else
                        atomicAdd(a.gW + woff + m + size_t(n) * out_k, v);
                }
            }
    };
    {
#pragma unroll
        for (int c = 0; c < C0; ++c) {
            const int p = warp + c * TW;
            if (p < P0)
                flush(dw0[c], p / IN_STEPS, p % IN_STEPS, hw, s.in_real, 0);
        }
#pragma unroll
        for (int k = 1; k < NH; ++k)
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                const int p = warp + c * TW;
                flush(dwh[k - 1][c], p / 4, p % 4, hw, hw, size_t(hw) * s.in_real + size_t(k - 1) * hw * hw);
            }
        if (warp < PO)
            flush(dwo, 0, warp, s.n_out, hw, size_t(hw) * s.in_real + size_t(NH - 1) * hw * hw);
    }
    if (t == 0) {
        if (warp < 4)
#pragma unroll
            for (int k = 0; k < NH; ++k)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int j = 16 * warp + g + 8 * h;
                    if (j >= hw)
                        continue;
                    const float v = dbh[k][h] * ic;
                    bad |= !sane(v);
                    if (a.part_wb)
                        a.part_wb[blockIdx.x * a.n_wb + a.n_w + k * hw + j] = v;
                    else
                        atomicAdd(a.gb + k * hw + j, v);
                }
        if (warp == TW - 1)
#pragma unroll
            for (int h = 0; h < 2; ++h)
                if (g + 8 * h < s.n_out) {
                    const float v = dbo[h] * ic;
                    bad |= !sane(v);
                    if (a.part_wb)
                        a.part_wb[blockIdx.x * a.n_wb + a.n_w + NH * hw + g + 8 * h] = v;
                    else
                        atomicAdd(a.gb + NH * hw + g + 8 * h, v);
                }
    }
    }   // mma.sync dW path
    if (GRAD == GRAD_LOSS && lane == 0) {
        if (a.part_loss)
            a.part_loss[vblk * TW + warp] = loss_acc;
        else if (loss_acc != 0.0)
            atomicAdd(a.scratch.loss_sum, loss_acc);
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0)
        atomicOr(a.scratch.flags, 1u);
    invalid = __reduce_or_sync(0xffffffffu, invalid);
    if (invalid && lane == 0) {
        atomicOr(&a.scratch.flags[3], invalid);
        atomicOr(&a.scratch.flags[1], 1u);
    }
}

template <int SRC, int D, int F, typename TT, int IN_STEPS, int NH, int IP = IP_RUNTIME>
__global__ void __launch_bounds__(IW * 32)
k_infer(const InferArgs a, const FieldShape s, const LevelDev* __restrict__ levels)
{
    using Lay = WLayout<IN_STEPS, NH>;
    using SM = InferSmem<IN_STEPS, NH>;
    extern __shared__ __align__(16) unsigned char sm[];
    __half* ws = reinterpret_cast<__half*>(sm);
    float* bs = reinterpret_cast<float*>(sm + Lay::HALVES * 2);
    LevelDev* lvs = reinterpret_cast<LevelDev*>(sm + SM::LV_OFF);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
    const MlpShape msh{ s.in_real, s.n_out, s.sigmoid, s.hidden_width };
    load_weights<IN_STEPS, NH>(ws, bs, a.W, a.b, msh);
    if (SRC == SRC_ENCODE)
        for (int i = tid; i < s.grid.L; i += blockDim.x)
            lvs[i] = levels[i];
    __syncthreads();
    const __half* W0s = ws;
    const __half* Whs = ws + Lay::W0_HALVES;
    const __half* Wos = ws + Lay::W0_HALVES + (NH - 1) * Lay::WH_HALVES;
    const float* bout = bs + H * NH;

    const int64_t ntiles = (a.B + 15) / 16;
    for (int64_t tile = int64_t(blockIdx.x) * IW + warp; tile < ntiles; tile += int64_t(gridDim.x) * IW) {
        const int64_t sg = tile * 16 + g, sg8 = sg + 8;
        const bool vg = sg < a.B, vg8 = sg8 < a.B;
        float xg[D], xg8[D];
        if (SRC == SRC_ENCODE) {
            load_x<D>(xg, a.X, sg, vg);
            load_x<D>(xg8, a.X, sg8, vg8);
            clamp_x<D>(xg);
            clamp_x<D>(xg8);
        }
        uint32_t afr[IN_STEPS][4];
        input_frags<SRC, D, F, TT, IN_STEPS, SRC == SRC_ENCODE, IP>(afr, s, lvs, xg, xg8, vg, vg8, sg, a.Y, a.table, lane);
        float acc[HT][4];
        uint32_t ah[4][4];
        layer_fwd<IN_STEPS, HT>(afr, W0s, Lay::INS, acc, lane);
        bias_relu<HT>(acc, bs, lane);
        c_to_a<4, false>(acc, ah);
#pragma unroll
        for (int k = 1; k < NH; ++k) {
            layer_fwd<4, HT>(ah, Whs + (k - 1) * Lay::WH_HALVES, HS, acc, lane);
            bias_relu<HT>(acc, bs + H * k, lane);
            c_to_a<4, false>(acc, ah);
        }
        float ao[2][4];
        layer_fwd<4, 2>(ah, Wos, HS, ao, lane);
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int col = 8 * j + 2 * t + (e & 1);
                const bool valid = (e < 2 ? vg : vg8) && col < s.n_out;
                if (valid) {
                    const float z = ao[j][e] + bout[col];
                    a.out[(e < 2 ? sg : sg8) * s.n_out + col] = s.sigmoid ? 1.0f / (1.0f + expf(-z)) : z;
                }
            }
    }
}

}   // namespace nfg
