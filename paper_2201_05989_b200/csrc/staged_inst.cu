// staged_inst.cu — MLP-only instantiations (input Y from global memory): the
// component mlp_forward / mlp_backward entry points and the staged train path.
#include "launch_impl.cuh"

namespace nfg {

#define NFG_STAGED_LIST(X) \
    X(1, 1) X(1, 2) X(1, 3) X(2, 1) X(2, 2) X(2, 3) X(3, 2) X(4, 1) X(4, 2) X(4, 3)

cudaError_t launch_staged_train(const FieldShape& s, int grad, const TrainArgs& a, int num_sms, cudaStream_t st,
                                int* grid_used)
{
#define X(IS_, NH_)                                                                                         \
    if (s.in_steps == IS_ && s.hidden_layers == NH_)                                                         \
        return grad == GRAD_LOSS                                                                             \
                   ? run_train<SRC_LOAD_Y, GRAD_LOSS, SINK_STORE, 2, 2, __half, IS_, NH_>(s, nullptr, a, num_sms, \
                                                                                          st, grid_used)     \
                   : run_train<SRC_LOAD_Y, GRAD_DOUT, SINK_STORE, 2, 2, __half, IS_, NH_>(s, nullptr, a, num_sms, \
                                                                                          st, grid_used);
    NFG_STAGED_LIST(X)
#undef X
    return cudaErrorNotSupported;
}

cudaError_t launch_staged_infer(const FieldShape& s, const InferArgs& a, int num_sms, cudaStream_t st)
{
#define X(IS_, NH_)                                                                                         \
    if (s.in_steps == IS_ && s.hidden_layers == NH_)                                                         \
        return run_infer<SRC_LOAD_Y, 2, 2, __half, IS_, NH_>(s, nullptr, a, num_sms, st);
    NFG_STAGED_LIST(X)
#undef X
    return cudaErrorNotSupported;
}

cudaError_t launch_fused_train_d2(const FieldShape&, const LevelDev*, const TrainArgs&, int, cudaStream_t, int*);
cudaError_t launch_fused_train_d3(const FieldShape&, const LevelDev*, const TrainArgs&, int, cudaStream_t, int*);
cudaError_t launch_fused_dout_d2(const FieldShape&, const LevelDev*, const TrainArgs&, int, cudaStream_t, int*);
cudaError_t launch_fused_dout_d3(const FieldShape&, const LevelDev*, const TrainArgs&, int, cudaStream_t, int*);
cudaError_t launch_fused_store_d2(const FieldShape&, const LevelDev*, const TrainArgs&, int, cudaStream_t, int*);
cudaError_t launch_fused_store_d3(const FieldShape&, const LevelDev*, const TrainArgs&, int, cudaStream_t, int*);
cudaError_t launch_fused_infer_d2(const FieldShape&, const LevelDev*, const InferArgs&, int, cudaStream_t);
cudaError_t launch_fused_infer_d3(const FieldShape&, const LevelDev*, const InferArgs&, int, cudaStream_t);

cudaError_t launch_train(const FieldShape& s, const LevelDev* lv, int src, int grad, int sink, const TrainArgs& a,
                         int num_sms, cudaStream_t st, int* grid_used)
{
    if (src == SRC_ENCODE) {
        if (sink == SINK_STORE)
            return grad != GRAD_LOSS ? cudaErrorNotSupported
                   : s.grid.d == 2   ? launch_fused_store_d2(s, lv, a, num_sms, st, grid_used)
                                     : launch_fused_store_d3(s, lv, a, num_sms, st, grid_used);
        if (grad == GRAD_DOUT)
            return s.grid.d == 2 ? launch_fused_dout_d2(s, lv, a, num_sms, st, grid_used)
                                 : launch_fused_dout_d3(s, lv, a, num_sms, st, grid_used);
        return s.grid.d == 2 ? launch_fused_train_d2(s, lv, a, num_sms, st, grid_used)
                             : launch_fused_train_d3(s, lv, a, num_sms, st, grid_used);
    }
    if (sink != SINK_STORE)
        return cudaErrorNotSupported;
    return launch_staged_train(s, grad, a, num_sms, st, grid_used);
}

int train_warps_per_cta() { return TW; }

bool fused_supported_d2(const FieldShape&);
bool fused_supported_d3(const FieldShape&);

bool fused_supported(const FieldShape& s)
{
    return s.grid.d == 2 ? fused_supported_d2(s) : fused_supported_d3(s);
}

bool staged_supported(const FieldShape& s)
{
#define X(IS_, NH_)                                                                                         \
    if (s.in_steps == IS_ && s.hidden_layers == NH_)                                                         \
        return true;
    NFG_STAGED_LIST(X)
#undef X
    return false;
}

cudaError_t launch_infer(const FieldShape& s, const LevelDev* lv, int src, const InferArgs& a, int num_sms,
                         cudaStream_t st)
{
    if (src == SRC_ENCODE)
        return s.grid.d == 2 ? launch_fused_infer_d2(s, lv, a, num_sms, st)
                             : launch_fused_infer_d3(s, lv, a, num_sms, st);
    return launch_staged_infer(s, a, num_sms, st);
}

}   // namespace nfg
