// launch_impl.cuh — host launch helpers for the templated train / infer kernels.
#pragma once

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "field_kernels.cuh"
#include "infer_tc.cuh"

namespace nfg {

template <int SRC, int GRAD, int SINK, int D, int F, typename TT, int IS, int NH>
cudaError_t run_train(const FieldShape& s, const LevelDev* lv, const TrainArgs& a, int num_sms, cudaStream_t st,
                      int* grid_used)
{
    using SM = TrainSmem<IS, NH, StageGeo<SRC, D, F, TT, IS>::BYTES, StageAlias<SRC, D, F, TT, IS, NH>::ON>;
    auto k = k_train<SRC, GRAD, SINK, D, F, TT, IS, NH>;
    static int per_sm = -1;   // resolved once per instantiation
    if (per_sm < 0) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SM::BYTES);
        if (e != cudaSuccess)
            return e;
        if (const char* cv = getenv("NFG_TRAIN_CARVEOUT")) {   // experiment: shared-memory carveout percent
            e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(cv));
            if (e != cudaSuccess)
                return e;
        }
        int n = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, TW * 32, SM::BYTES);
        if (e != cudaSuccess)
            return e;
        per_sm = std::max(n, 1);
    }
    static char desc[160];
    if (!desc[0])
        snprintf(desc, sizeof(desc), "k_train src=%d grad=%d sink=%d d=%d F=%d table=%s in_steps=%d hidden=%d "
                 "stage_alias=%d ctas_per_sm=%d", SRC, GRAD, SINK, D, F, sizeof(TT) == 2 ? "f16" : "f32", IS, NH,
                 int(StageAlias<SRC, D, F, TT, IS, NH>::ON), per_sm);
    note_kernel_variant(0, desc);
    const int64_t ntiles = (a.B + TS - 1) / TS;
    if (ntiles <= 0)
        return cudaSuccess;
    const int grid = int(std::min<int64_t>(ntiles, int64_t(num_sms) * per_sm));
    if (grid_used)
        *grid_used = grid;
    k<<<grid, TW * 32, SM::BYTES, st>>>(a, s, lv);
    return cudaGetLastError();
}

template <int SRC, int D, int F, typename TT, int IS, int NH>
cudaError_t run_infer(const FieldShape& s, const LevelDev* lv, const InferArgs& a, int num_sms, cudaStream_t st)
{
    using SM = InferSmem<IS, NH>;
    auto k = k_infer<SRC, D, F, TT, IS, NH>;
    static int per_sm = -1;
    if (per_sm < 0) {
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
        snprintf(desc, sizeof(desc), "k_infer src=%d d=%d F=%d table=%s in_steps=%d hidden=%d warps=%d", SRC, D, F,
                 sizeof(TT) == 2 ? "f16" : "f32", IS, NH, IW);
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
cudaError_t run_infer_tc(const FieldShape& s, const LevelDev* lv, const InferArgs& a, int num_sms, cudaStream_t st)
{
    using SM = InferTcSmem<IS, NH>;
    auto k = k_infer_tc<SRC, D, F, TT, IS, NH>;
    static bool ready = false;
    if (!ready) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SM::BYTES);
        if (e != cudaSuccess)
            return e;
        ready = true;
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
