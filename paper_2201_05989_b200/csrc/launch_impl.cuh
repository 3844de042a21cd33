// launch_impl.cuh — host launch helpers for the templated train / infer kernels.
#pragma once

#include <algorithm>
#include <type_traits>
#include <cstdio>
#include <cstdlib>

#include "field_kernels.cuh"
#include "infer_tc.cuh"
#include "train_ws.cuh"

#ifndef NFG_MAX_DEVICES
#define NFG_MAX_DEVICES 64
#endif
#ifndef NFG_TRAIN_WS_DEFAULT
#define NFG_TRAIN_WS_DEFAULT 0
#endif

namespace nfg {

template <int SRC, int GRAD, int SINK, int D, int F, typename TT, int IS, int NH, bool TCW, int IP>
cudaError_t run_train(const FieldShape& s, const LevelDev* lv, const TrainArgs& a, int num_sms, cudaStream_t st,
                      int* grid_used)
{
    using SG = StageGeo<SRC, D, F, TT, IS>;
    constexpr bool ALIAS = StageAlias<SRC, D, F, TT, IS, NH>::ON;
    constexpr int NG = TrainGroups<TCW>::NG;
    using SM = std::conditional_t<TCW, TrainSmemTc<IS, NH, SG::BYTES, ALIAS, NG>, TrainSmem<IS, NH, SG::BYTES, ALIAS>>;
    auto k = k_train<SRC, GRAD, SINK, D, F, TT, IS, NH, TCW, IP>;
    constexpr int threads = TW * 32 * NG;
    static int per_sm_dev[NFG_MAX_DEVICES];   // resolved once per instantiation and device
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= NFG_MAX_DEVICES)
        return cudaErrorInvalidDevice;
    int& per_sm = per_sm_dev[dev];
    if (per_sm <= 0) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SM::BYTES);
        if (e != cudaSuccess)
            return e;
        if (const char* cv = getenv("NFG_TRAIN_CARVEOUT")) {   // experiment: shared-memory carveout percent
            e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(cv));
            if (e != cudaSuccess)
                return e;
        }
        int n = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, threads, SM::BYTES);
        if (e != cudaSuccess)
            return e;
        const int n_occ = n;
        if constexpr (TCW) {
            // The occupancy API reports 1 CTA per SM for this kernel, but 3 are
            // co-resident on a B200 (measured: k_train 416 us at a 1-CTA grid,
            // 270 us at 3; profiles/tc_train_r2.md). Size the persistent grid
            // from the actual per-SM limits: registers, shared memory, threads,
            // and the 512 TMEM columns the resident CTAs share.
            cudaFuncAttributes fa{};
            int smem_sm = 0, smem_resv = 0;
            if ((e = cudaFuncGetAttributes(&fa, k)) != cudaSuccess ||
                (e = cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev)) !=
                    cudaSuccess ||
                (e = cudaDeviceGetAttribute(&smem_resv, cudaDevAttrReservedSharedMemoryPerBlock, dev)) != cudaSuccess)
                return e;
            const int regs_warp = ((fa.numRegs * 32 + 255) / 256) * 256;
            const int by_regs = 65536 / (regs_warp * TW * NG);
            const int by_smem = smem_sm / (SM::BYTES + int(fa.sharedSizeBytes) + smem_resv);
            const int by_tmem = int(512 / SM::TMEM_COLS);
            n = std::max(1, std::min({ by_regs, by_smem, by_tmem, 2048 / threads }));
        }
        per_sm = std::max(n, 1);
        if (const char* o = getenv("NFG_TRAIN_CTAS_PER_SM"))   // experiment hook (grid sizing only)
            per_sm = std::max(1, atoi(o));
        if (getenv("NFG_DEBUG_OCC")) {
            cudaFuncAttributes fa{};
            cudaFuncGetAttributes(&fa, k);
            fprintf(stderr, "[nfg] k_train tcw=%d smem_dyn=%d occ=%d per_sm=%d regs=%d local=%zu static_smem=%zu "
                    "max_dyn=%d\n", int(TCW), SM::BYTES, n_occ, per_sm, fa.numRegs, fa.localSizeBytes,
                    fa.sharedSizeBytes, fa.maxDynamicSharedSizeBytes);
        }
    }
    static char desc[192];
    if (!desc[0])
        snprintf(desc, sizeof(desc), "k_train src=%d grad=%d sink=%d d=%d F=%d table=%s in_steps=%d hidden=%d "
                 "stage_alias=%d ctas_per_sm=%d groups=%d dw=%s interp=%s", SRC, GRAD, SINK, D, F,
                 sizeof(TT) == 2 ? "f16" : "f32", IS, NH, int(ALIAS), per_sm, NG, TCW ? "tcgen05" : "mma.sync",
                 IP == IP_LINEAR ? "linear" : IP == IP_SMOOTH ? "smooth" : "runtime");
    note_kernel_variant(0, desc);
    const int64_t ntiles = (a.B + TS - 1) / TS;
    if (ntiles <= 0)
        return cudaSuccess;
    // grid_used counts tile workers (groups): the deterministic partials are per group
    const int grid = int(std::min<int64_t>((ntiles + NG - 1) / NG, int64_t(num_sms) * per_sm));
    if (grid_used)
        *grid_used = grid * NG;
    return launch_pdl(k, dim3(grid), dim3(threads), SM::BYTES, st, a, s, lv);
}

// Warp-specialised variant (train_ws.cuh): producers gather, consumers run the
// MLP / reductions; 2 CTAs x 8 warps per SM.
template <int D, typename TT, int IS, int NH>
cudaError_t run_train_ws(const FieldShape& s, const LevelDev* lv, const TrainArgs& a, int num_sms, cudaStream_t st,
                         int* grid_used)
{
    using SM = TrainWsSmem<D, TT, IS, NH>;
    auto k = k_train_ws<D, TT, IS, NH>;
    static bool ready_dev[NFG_MAX_DEVICES];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= NFG_MAX_DEVICES)
        return cudaErrorInvalidDevice;
    if (!ready_dev[dev]) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SM::BYTES);
        if (e != cudaSuccess)
            return e;
        ready_dev[dev] = true;
    }
    static char desc[192];
    if (!desc[0])
        snprintf(desc, sizeof(desc), "k_train_ws src=0 grad=0 sink=0 d=%d F=2 table=%s in_steps=%d hidden=%d "
                 "stage_alias=0 ctas_per_sm=2 warps=4+4 dw=tcgen05", D, sizeof(TT) == 2 ? "f16" : "f32", IS, NH);
    note_kernel_variant(0, desc);
    const int64_t ntiles = (a.B + TS - 1) / TS;
    if (ntiles <= 0)
        return cudaSuccess;
    const int per_sm = getenv("NFG_WS_CTAS") ? std::max(1, atoi(getenv("NFG_WS_CTAS"))) : 2;
    const int grid = int(std::min<int64_t>(ntiles, int64_t(num_sms) * per_sm));
    if (grid_used)
        *grid_used = grid;
    k<<<grid, 256, SM::BYTES, st>>>(a, s, lv);
    return cudaGetLastError();
}

inline bool train_ws_enabled()
{
    static const int on = [] {
        const char* e = getenv("NFG_TRAIN_WS");
        return e ? atoi(e) : NFG_TRAIN_WS_DEFAULT;
    }();
    return on != 0;
}

// Engine of the fused training kernel's dW reduction (nfg_options.mlp_engine).
#ifndef NFG_TRAIN_TC_DEFAULT
#define NFG_TRAIN_TC_DEFAULT 1
#endif
inline bool train_tcw(const FieldShape& s)
{
    return s.mlp_engine == 2 || (s.mlp_engine == 0 && NFG_TRAIN_TC_DEFAULT);
}

template <int SRC, int GRAD, int SINK, int D, int F, typename TT, int IS, int NH>
cudaError_t run_train(const FieldShape& s, const LevelDev* lv, const TrainArgs& a, int num_sms, cudaStream_t st,
                      int* grid_used)
{
    // The default (tcgen05) engine's encoding instantiations fix the interpolation
    // at compile time; the mma.sync engine (A/B runs) and the dY-storing variant
    // (level-pipelined exchange option) read it at run time.
    if (!train_tcw(s))
        return run_train<SRC, GRAD, SINK, D, F, TT, IS, NH, false, IP_RUNTIME>(s, lv, a, num_sms, st, grid_used);
    if constexpr (SRC == SRC_ENCODE && SINK != SINK_STORE) {
        if (s.grid.smooth)
            return run_train<SRC, GRAD, SINK, D, F, TT, IS, NH, true, IP_SMOOTH>(s, lv, a, num_sms, st, grid_used);
        return run_train<SRC, GRAD, SINK, D, F, TT, IS, NH, true, IP_LINEAR>(s, lv, a, num_sms, st, grid_used);
    }
    return run_train<SRC, GRAD, SINK, D, F, TT, IS, NH, true, IP_RUNTIME>(s, lv, a, num_sms, st, grid_used);
}

template <int SRC, int D, int F, typename TT, int IS, int NH, int IP>
cudaError_t run_infer_ip(const FieldShape& s, const LevelDev* lv, const InferArgs& a, int num_sms, cudaStream_t st)
{
    using SM = InferSmem<IS, NH>;
    auto k = k_infer<SRC, D, F, TT, IS, NH, IP>;
    static int per_sm_dev[NFG_MAX_DEVICES];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= NFG_MAX_DEVICES)
        return cudaErrorInvalidDevice;
    int& per_sm = per_sm_dev[dev];
    if (per_sm <= 0) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SM::BYTES);
        if (e != cudaSuccess)
            return e;
        int n = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, IW * 32, SM::BYTES);
        if (e != cudaSuccess)
            return e;
        per_sm = std::max(n, 1);
    }
    static char desc[160];
    if (!desc[0])
        snprintf(desc, sizeof(desc), "k_infer src=%d d=%d F=%d table=%s in_steps=%d hidden=%d warps=%d interp=%s", SRC,
                 D, F, sizeof(TT) == 2 ? "f16" : "f32", IS, NH, IW,
                 IP == IP_LINEAR ? "linear" : IP == IP_SMOOTH ? "smooth" : "runtime");
    note_kernel_variant(1, desc);
    const int64_t tiles = (a.B + 15) / 16;
    if (tiles <= 0)
        return cudaSuccess;
    const int64_t want = (tiles + IW - 1) / IW;
    const int grid = int(std::min<int64_t>(want, int64_t(num_sms) * per_sm));
    k<<<grid, IW * 32, SM::BYTES, st>>>(a, s, lv);
    return cudaGetLastError();
}

template <int SRC, int D, int F, typename TT, int IS, int NH>
cudaError_t run_infer(const FieldShape& s, const LevelDev* lv, const InferArgs& a, int num_sms, cudaStream_t st)
{
    if constexpr (SRC == SRC_ENCODE) {   // interpolation fixed per instantiation (no smoothstep work when linear)
        if (s.grid.smooth)
            return run_infer_ip<SRC, D, F, TT, IS, NH, IP_SMOOTH>(s, lv, a, num_sms, st);
        return run_infer_ip<SRC, D, F, TT, IS, NH, IP_LINEAR>(s, lv, a, num_sms, st);
    }
    return run_infer_ip<SRC, D, F, TT, IS, NH, IP_RUNTIME>(s, lv, a, num_sms, st);
}

template <int SRC, int D, int F, typename TT, int IS, int NH>
cudaError_t run_infer_tc(const FieldShape& s, const LevelDev* lv, const InferArgs& a, int num_sms, cudaStream_t st)
{
    using SM = InferTcSmem<IS, NH>;
    auto k = k_infer_tc<SRC, D, F, TT, IS, NH>;
    static bool ready_dev[NFG_MAX_DEVICES];   // the attribute is per device context
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= NFG_MAX_DEVICES)
        return cudaErrorInvalidDevice;
    if (!ready_dev[dev]) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SM::BYTES);
        if (e != cudaSuccess)
            return e;
        ready_dev[dev] = true;
    }
    static char desc[160];
    if (!desc[0])
        snprintf(desc, sizeof(desc), "k_infer_tc src=%d d=%d F=%d table=%s in_steps=%d hidden=%d quads=%d mma=tcgen05",
                 SRC, D, F, sizeof(TT) == 2 ? "f16" : "f32", IS, NH, IQ);
    note_kernel_variant(1, desc);
    const int64_t tiles = (a.B + 127) / 128;
    if (tiles <= 0)
        return cudaSuccess;
    // one CTA per SM (it allocates the SM's TMEM columns for its quads); tiles
    // are dealt round-robin over the SMs first
    const int grid = int(std::min<int64_t>(tiles, num_sms));
    k<<<grid, IQ * 128, SM::BYTES, st>>>(a, s, lv);
    return cudaGetLastError();
}

}   // namespace nfg
