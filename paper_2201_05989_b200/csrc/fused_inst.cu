// fused_inst.cu — sm_100a instantiations of the fused encode+MLP kernels for
// one input dimensionality (compiled twice: -DNFG_D=2 and -DNFG_D=3).
#include "launch_impl.cuh"
#include "../../include/nfg.h"

#ifndef NFG_D
#error "compile with -DNFG_D=2 or -DNFG_D=3"
#endif
#ifndef NFG_PART
#error "compile with -DNFG_PART=0..5"
#endif
#define NFG_CAT2(a, b) a##b
#define NFG_CAT(a, b) NFG_CAT2(a, b)

// Default engine of the fused inference kernel (nfg_options.mlp_engine ==
// NFG_MMA_DEFAULT): the measured-faster one per batch size.
#ifndef NFG_INFER_TC_BELOW
#define NFG_INFER_TC_BELOW (int64_t(1) << 18)
#endif

namespace nfg {

// Built combinations (anything else is NFG_EUNSUPPORTED):
//   F = 2: fp16 or fp32 tables, in_steps 1..2 (L*F <= 32), hidden_layers 1..3
//   F = 1, 4, 8: fp16 or fp32 tables, in_steps 2, hidden_layers 2
// the training lists are split in two (F = 2, in_steps 2 | the rest) so each
// half compiles in its own translation unit
#define NFG_FUSED_LIST_A(X)                                                   \
    X(2, __half, 2, 1) X(2, __half, 2, 2) X(2, __half, 2, 3)                  \
    X(2, float, 2, 1) X(2, float, 2, 2) X(2, float, 2, 3)
#define NFG_FUSED_LIST_B(X)                                                   \
    X(2, __half, 1, 1) X(2, __half, 1, 2) X(2, __half, 1, 3)                  \
    X(2, float, 1, 1) X(2, float, 1, 2) X(2, float, 1, 3)                     \
    X(1, __half, 2, 2) X(4, __half, 2, 2) X(8, __half, 2, 2)                  \
    X(1, float, 2, 2) X(4, float, 2, 2) X(8, float, 2, 2)
#define NFG_FUSED_LIST(X) NFG_FUSED_LIST_A(X) NFG_FUSED_LIST_B(X)

// The instantiations are split over six translation units per dimension
// (NFG_PART 0..5, Makefile) so a parallel build compiles them side by side.
cudaError_t NFG_CAT(launch_fused_train_f32_d, NFG_D)(const FieldShape& s, const LevelDev* lv, const TrainArgs& a,
                                                     int num_sms, cudaStream_t st, int* grid_used);
cudaError_t NFG_CAT(launch_fused_train_b_d, NFG_D)(const FieldShape& s, const LevelDev* lv, const TrainArgs& a,
                                                   int num_sms, cudaStream_t st, int* grid_used);
cudaError_t NFG_CAT(launch_fused_train_f32_b_d, NFG_D)(const FieldShape& s, const LevelDev* lv, const TrainArgs& a,
                                                       int num_sms, cudaStream_t st, int* grid_used);

#if NFG_PART == 0
cudaError_t NFG_CAT(launch_fused_train_d, NFG_D)(const FieldShape& s, const LevelDev* lv, const TrainArgs& a,
                                                 int num_sms, cudaStream_t st, int* grid_used)
{
    if (s.table_fp32 != 0)
        return NFG_CAT(launch_fused_train_f32_d, NFG_D)(s, lv, a, num_sms, st, grid_used);
    if (train_ws_enabled() && train_tcw(s) && s.grid.F == 2 && s.in_steps == 2 && s.hidden_layers == 2 &&
        a.part_wb == nullptr)   // warp-specialised variant (train_ws.cuh)
        return run_train_ws<NFG_D, __half, 2, 2>(s, lv, a, num_sms, st, grid_used);
#define X(F_, TT_, IS_, NH_)                                                                               \
    if (sizeof(TT_) == 2 && s.grid.F == F_ && s.in_steps == IS_ && s.hidden_layers == NH_)                 \
        return run_train<SRC_ENCODE, GRAD_LOSS, SINK_SCATTER, NFG_D, F_, __half, IS_, NH_>(s, lv, a, num_sms,  \
                                                                                            st, grid_used);
    NFG_FUSED_LIST_A(X)
#undef X
    return NFG_CAT(launch_fused_train_b_d, NFG_D)(s, lv, a, num_sms, st, grid_used);
}
#endif

#if NFG_PART == 4
cudaError_t NFG_CAT(launch_fused_train_b_d, NFG_D)(const FieldShape& s, const LevelDev* lv, const TrainArgs& a,
                                                   int num_sms, cudaStream_t st, int* grid_used)
{
#define X(F_, TT_, IS_, NH_)                                                                               \
    if (sizeof(TT_) == 2 && s.grid.F == F_ && s.in_steps == IS_ && s.hidden_layers == NH_)                 \
        return run_train<SRC_ENCODE, GRAD_LOSS, SINK_SCATTER, NFG_D, F_, __half, IS_, NH_>(s, lv, a, num_sms,  \
                                                                                            st, grid_used);
    NFG_FUSED_LIST_B(X)
#undef X
    return cudaErrorNotSupported;
}
#endif

#if NFG_PART == 1
cudaError_t NFG_CAT(launch_fused_train_f32_d, NFG_D)(const FieldShape& s, const LevelDev* lv, const TrainArgs& a,
                                                     int num_sms, cudaStream_t st, int* grid_used)
{
#define X(F_, TT_, IS_, NH_)                                                                               \
    if (sizeof(TT_) == 4 && s.grid.F == F_ && s.in_steps == IS_ && s.hidden_layers == NH_)                 \
        return run_train<SRC_ENCODE, GRAD_LOSS, SINK_SCATTER, NFG_D, F_, float, IS_, NH_>(s, lv, a, num_sms,   \
                                                                                           st, grid_used);
    NFG_FUSED_LIST_A(X)
#undef X
    return NFG_CAT(launch_fused_train_f32_b_d, NFG_D)(s, lv, a, num_sms, st, grid_used);
}
#endif

#if NFG_PART == 5
cudaError_t NFG_CAT(launch_fused_train_f32_b_d, NFG_D)(const FieldShape& s, const LevelDev* lv, const TrainArgs& a,
                                                       int num_sms, cudaStream_t st, int* grid_used)
{
#define X(F_, TT_, IS_, NH_)                                                                               \
    if (sizeof(TT_) == 4 && s.grid.F == F_ && s.in_steps == IS_ && s.hidden_layers == NH_)                 \
        return run_train<SRC_ENCODE, GRAD_LOSS, SINK_SCATTER, NFG_D, F_, float, IS_, NH_>(s, lv, a, num_sms,   \
                                                                                           st, grid_used);
    NFG_FUSED_LIST_B(X)
#undef X
    return cudaErrorNotSupported;
}
#endif

#if NFG_PART == 3
// Whether a fused instantiation exists for this shape (the field falls back to
// the staged kernels otherwise).
bool NFG_CAT(fused_supported_d, NFG_D)(const FieldShape& s)
{
    const bool f32 = s.table_fp32 != 0;
#define X(F_, TT_, IS_, NH_)                                                                               \
    if (s.grid.F == F_ && f32 == (sizeof(TT_) == 4) && s.in_steps == IS_ && s.hidden_layers == NH_)         \
        return true;
    NFG_FUSED_LIST(X)
#undef X
    return false;
}

#endif

#if NFG_PART == 2
// Fused backward with an external dLoss/dOutput (nfg_field_backward_device:
// the NeRF density network, 3D, L*F = 32, 1 or 2 hidden layers).
cudaError_t NFG_CAT(launch_fused_dout_d, NFG_D)(const FieldShape& s, const LevelDev* lv, const TrainArgs& a,
                                                int num_sms, cudaStream_t st, int* grid_used)
{
#if NFG_D == 3
    const bool f32 = s.table_fp32 != 0;
#define X(F_, TT_, IS_, NH_)                                                                               \
    if (s.grid.F == F_ && f32 == (sizeof(TT_) == 4) && s.in_steps == IS_ && s.hidden_layers == NH_)         \
        return run_train<SRC_ENCODE, GRAD_DOUT, SINK_SCATTER, NFG_D, F_, TT_, IS_, NH_>(s, lv, a, num_sms, st, \
                                                                                         grid_used);
    X(2, __half, 2, 1) X(2, __half, 2, 2) X(2, float, 2, 1) X(2, float, 2, 2)
#undef X
#else
    (void)s, (void)lv, (void)a, (void)num_sms, (void)st, (void)grid_used;
#endif
    return cudaErrorNotSupported;
}

// Fused encode + MLP forward / loss / MLP backward with dY stored instead of
// scattered (the data-parallel level-pipelined exchange: the table-gradient
// scatter then runs per level group so each group's all-reduce starts early).
cudaError_t NFG_CAT(launch_fused_store_d, NFG_D)(const FieldShape& s, const LevelDev* lv, const TrainArgs& a,
                                                 int num_sms, cudaStream_t st, int* grid_used)
{
    const bool f32 = s.table_fp32 != 0;
#define X(F_, TT_, IS_, NH_)                                                                               \
    if (s.grid.F == F_ && f32 == (sizeof(TT_) == 4) && s.in_steps == IS_ && s.hidden_layers == NH_)         \
        return run_train<SRC_ENCODE, GRAD_LOSS, SINK_STORE, NFG_D, F_, TT_, IS_, NH_>(s, lv, a, num_sms, st,   \
                                                                                       grid_used);
    X(2, __half, 1, 1) X(2, __half, 1, 2) X(2, __half, 1, 3) X(2, __half, 2, 1) X(2, __half, 2, 2)
    X(2, __half, 2, 3) X(2, float, 1, 1) X(2, float, 1, 2) X(2, float, 1, 3) X(2, float, 2, 1)
    X(2, float, 2, 2) X(2, float, 2, 3)
#undef X
    return cudaErrorNotSupported;
}

#endif

#if NFG_PART == 3
cudaError_t NFG_CAT(launch_fused_infer_d, NFG_D)(const FieldShape& s, const LevelDev* lv, const InferArgs& a,
                                                 int num_sms, cudaStream_t st)
{
    const bool f32 = s.table_fp32 != 0;
    // default engine: tcgen05 below 2^18 queries (its 128-sample tiles dealt over all SMs beat the
    // mma.sync kernel's 1.15 waves of 16-sample warp tiles at 2^16 by 1.27x), mma.sync above (1.10x faster
    // from 2^22: the L1 is the binding unit and the tcgen05 epilogues' shared-memory round trips compete
    // with the gathers for it); profiles/tc_infer_r2.md
    const bool tc = s.mlp_engine == NFG_MMA_TCGEN05 ||
                    (s.mlp_engine == NFG_MMA_DEFAULT && a.B < NFG_INFER_TC_BELOW);
#define X(F_, TT_, IS_, NH_)                                                                               \
    if (s.grid.F == F_ && f32 == (sizeof(TT_) == 4) && s.in_steps == IS_ && s.hidden_layers == NH_)         \
        return tc ? run_infer_tc<SRC_ENCODE, NFG_D, F_, TT_, IS_, NH_>(s, lv, a, num_sms, st)                 \
                  : run_infer<SRC_ENCODE, NFG_D, F_, TT_, IS_, NH_>(s, lv, a, num_sms, st);
    NFG_FUSED_LIST(X)
#undef X
    return cudaErrorNotSupported;
}

#endif

}   // namespace nfg
