// kernels.h — host-side launch interface of the sm_100a kernels (internal to libnfg).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "nfg_common.cuh"

namespace nfg {

// Static shape of one field model, resolved on the host.
struct FieldShape {
    GridDev grid;
    int in_real;       // L*F
    int in_steps;      // ceil(in_real / 16)
    int hidden_layers;
    int hidden_width;  // reference hidden_width (<= 64; the kernels pad to 64 with exact zeros)
    int n_out;
    int sigmoid;
    int table_fp32;
    int mlp_engine;    // nfg_options.mlp_engine (NFG_MMA_*)
};

// Gradient-side device scratch of one training step.
struct StepScratch {
    double* loss_sum;        // [1]
    unsigned int* flags;     // [0]: maybe non-finite; [1]: abort; [2]: first bad group (+1);
                             // [3]: invalid input (1 non-finite, 2 outside [0,1]^d), 4 = stood down behind an
                             // earlier asynchronous abort (k_step_begin)
    float* dy_max;           // [1] max |dY| (as float bits, non-negative)
};

enum TrainSource { SRC_ENCODE = 0, SRC_LOAD_Y = 1 };
enum TrainGrad { GRAD_LOSS = 0, GRAD_DOUT = 1 };
enum TrainSink { SINK_SCATTER = 0, SINK_STORE = 1 };

struct TrainArgs {
    // inputs
    const float* X;          // d x B            (SRC_ENCODE)
    const float* Y;          // in_real x B      (SRC_LOAD_Y)
    const float* target;     // n_out x B        (GRAD_LOSS)
    const float* dout;       // n_out x B        (GRAD_DOUT)
    int64_t B;
    int loss_kind;
    float inv_count;         // 1 / (global batch * n_out); 1 for GRAD_DOUT
    // parameters (fp32 master, reference layout) and tables
    const void* table;       // fp16 shadow or fp32 master tables
    const float* W;
    const float* b;
    // outputs
    float* table_grad;       // SINK_SCATTER
    float* dY;               // SINK_STORE: in_real x B
    float* gW;
    float* gb;
    float* pred;             // optional n_out x B
    StepScratch scratch;
    unsigned long long* phase_clk;   // NFG_PHASE_TIMING builds only
    // Streamed inputs (host-pointer train_step): tile t may start once the
    // flag of the chunk holding its last sample s is >= epoch (written by the
    // copy stream after the chunk's H2D); chunk of s = s < chunk0 ? 0 :
    // 1 + (s - chunk0) / chunk. ready == nullptr: inputs already resident.
    const unsigned int* ready;
    unsigned int epoch;
    int64_t chunk0;   // samples in the first (small) chunk
    int64_t chunk;    // samples in each later chunk
    // 1: check the inputs inside the kernel (grid.hpp:226-229) and flag an
    // invalid batch (flags[3], abort flags[1]); Adam's check kernel then
    // restores the (clean) gradient slab, so no state changes.
    int validate;
    // Deterministic mode (nfg_options.deterministic): per-CTA partials instead
    // of float atomics. part_wb[cta * n_wb + i] (i over [W | b], pre-zeroed),
    // part_loss[cta * TW + warp]; reduced in CTA order by launch_reduce_partials.
    float* part_wb;
    double* part_loss;
    int64_t n_w, n_wb;
};

struct InferArgs {
    const float* X;
    const float* Y;
    int64_t B;
    const void* table;
    const float* W;
    const float* b;
    float* out;
};

// Returns cudaErrorNotSupported when the (dims, F, in_steps, hidden_layers)
// combination has no sm_100a instantiation.
// `lv` is the device copy of the level table (LevelDev[L]).
cudaError_t launch_train(const FieldShape& s, const LevelDev* lv, int src, int grad, int sink, const TrainArgs& a,
                         int num_sms, cudaStream_t st, int* grid_used);
cudaError_t launch_infer(const FieldShape& s, const LevelDev* lv, int src, const InferArgs& a, int num_sms,
                         cudaStream_t st);
cudaError_t launch_encode_fwd_lv(const FieldShape& s, const LevelDev* lv, const float* X, int64_t B,
                                 const void* table, float* Y, uint32_t* rows, float* weights, cudaStream_t st);
// Levels [l0, l1) only (l1 < 0: all): the data-parallel exchange scatters level groups separately.
cudaError_t launch_encode_bwd_lv(const FieldShape& s, const LevelDev* lv, const float* X, int64_t B,
                                 const float* dY, float* grads, cudaStream_t st, const unsigned int* flags = nullptr,
                                 int l0 = 0, int l1 = -1);

struct AdamArgs {
    float* p;
    float* g;
    float* m;
    float* v;
    __half* shadow;          // fp16 table shadow (may be null)
    uint64_t n_tab, n_w, n_b;
    float b1, b2, omb1, omb2, bc1, bc2, eps, l2, lr;
    unsigned int* flags;
    int restore_on_invalid;   // zero the gradient slab if flags[3] (speculative step)
    int eager;                // 1: load p/m/v with g (dense steps), 0: only for non-zero gradient quads
    // Pipelined data-parallel Adam (field.cu): mode 0 updates [0, n) after
    // k_adam_check; mode 1 updates [lo, hi) (lo a multiple of 4) as soon as that
    // chunk is all-reduced, unless a producer flagged a possibly non-finite
    // gradient (flags[0]); mode 2 is the fallback full pass that runs only then.
    int mode;
    uint64_t lo, hi;
    unsigned int* sticky;     // sticky abort word (k_step_begin); counts stood-down steps in [3]
};
cudaError_t launch_adam_range(const AdamArgs& a, int num_sms, cudaStream_t st);
cudaError_t launch_adam_fallback(const AdamArgs& a, int num_sms, cudaStream_t st);
cudaError_t launch_adam(const AdamArgs& a, bool force_check, int num_sms, cudaStream_t st);
cudaError_t launch_validate(const float* X, int64_t n, unsigned int* flags, cudaStream_t st);
cudaError_t launch_step_begin(double* loss_sum, unsigned int* flags, float* dy_max, unsigned int* sticky, int inherit,
                              cudaStream_t st);
cudaError_t launch_shadow(const float* p, __half* shadow, uint64_t n, cudaStream_t st);
size_t encode_bwd_det_scratch(int64_t B, int d, int L);
cudaError_t launch_encode_bwd_det(const FieldShape& s, const LevelDev* lv, const float* X, int64_t B,
                                  const float* dY, float* grads, const unsigned int* flags, void* scratch,
                                  size_t bytes, cudaStream_t st);
cudaError_t launch_reduce_partials(const float* part, int nparts, int64_t n, float* out, const double* part_loss,
                                   int nloss, double* loss_sum, const unsigned int* flags, cudaStream_t st);
int train_warps_per_cta();
// Programmatic dependent launch (NFG_NO_PDL=1 disables it): the step's kernels
// are launched so the next grid is scheduled while its predecessor drains and
// waits in griddepcontrol.wait for the predecessor's completion.
bool pdl_enabled();
template <class K, class... Args>
cudaError_t launch_pdl(K kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args)
{
    if (!pdl_enabled()) {
        kernel<<<grid, block, smem, st>>>(args...);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}
// Records the template instantiation a launch helper just launched (which: 0 =
// train, 1 = infer), so tests can assert that the benchmarked variant is the
// one they checked (nfg_last_kernel_variant).
void note_kernel_variant(int which, const char* desc);
bool fused_supported(const FieldShape& s);    // fused encode+MLP kernels built for this shape
bool staged_supported(const FieldShape& s);   // staged MLP kernels built for this shape
cudaError_t launch_loss_out(const double* loss_sum, const unsigned int* flags, double count, float* out,
                            cudaStream_t st);
cudaError_t launch_loss(int kind, const float* pred, const float* target, int64_t n, float count, float* dpred,
                        double* loss_sum, cudaStream_t st);

}   // namespace nfg
