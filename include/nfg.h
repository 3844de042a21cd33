/* nfg.h — C ABI of the B200 (sm_100a) hash-grid encoding + fused MLP + Adam path.
 *
 * This is the drop-in boundary for the reference's C++ hot-path API
 * (/root/reference/proj/include/nf/{grid,mlp,adam,losses,model}.hpp). Every
 * entry point names the reference interface it replaces. Plain C types only:
 * no torch, no Eigen, no C++ in the signatures. The C++ shim in include/nf/
 * and the Python package paper_2201_05989_b200 sit on top of this.
 *
 * Layouts are the reference's Eigen column-major layouts:
 *   X       d x B            X[s*d + i]
 *   Y, dY   (L*F) x B        Y[s*L*F + l*F + f]
 *   out     n_out x B        out[s*n_out + o]
 *   params  one flat fp32 vector in param-group order (model.cpp:117-143):
 *           [tables: level 0 rows .. level L-1 rows, F floats per row]
 *           [MLP weights: W_0 .. W_n, each out x in column-major]
 *           [MLP biases: b_0 .. b_n]
 *   grads, Adam m and v use the same flat layout.
 *
 * Errors: every call returns an nfg_status; nfg_last_error() (thread-local)
 * holds the message. The reference's std::invalid_argument maps to
 * NFG_EINVAL, std::runtime_error (non-finite gradient, adam.hpp:86-90) to
 * NFG_ENONFINITE, std::logic_error to NFG_ELOGIC.
 *
 * Host-pointer calls are synchronous (reference semantics). *_device calls take
 * device pointers and are asynchronous on the context's stream.
 */
#ifndef NFG_H
#define NFG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NFG_ABI_VERSION 4

typedef enum {
    NFG_OK = 0,
    NFG_EINVAL = 1,        /* std::invalid_argument */
    NFG_ENONFINITE = 2,    /* std::runtime_error from adam_step / non-finite loss */
    NFG_EUNSUPPORTED = 3,  /* valid for the reference, not built for sm_100a (e.g. hidden_width != 64) */
    NFG_ECUDA = 4,
    NFG_ENCCL = 5,
    NFG_ELOGIC = 6,
    NFG_EIO = 7            /* std::runtime_error from checkpoint / report IO (io.cpp) */
} nfg_status;

typedef enum { NFG_INTERP_LINEAR = 0, NFG_INTERP_SMOOTHSTEP = 1 } nfg_interpolation; /* grid.hpp:20 */
typedef enum { NFG_ACT_LINEAR = 0, NFG_ACT_SIGMOID = 1 } nfg_output_activation;     /* mlp.hpp:13 */
typedef enum { NFG_LOSS_L2 = 0, NFG_LOSS_MAPE = 1, NFG_LOSS_RELATIVE_L2 = 2 } nfg_loss_kind; /* model.hpp:17 */
typedef enum { NFG_BUF_PARAMS = 0, NFG_BUF_GRADS = 1, NFG_BUF_ADAM_M = 2, NFG_BUF_ADAM_V = 3 } nfg_buffer;

/* HashEncodingConfig, grid.hpp:25-57. */
typedef struct {
    int32_t levels;
    uint32_t table_size;
    int32_t features;
    int32_t n_min;
    int32_t n_max;
    int32_t dims;
    int32_t interpolation; /* nfg_interpolation */
} nfg_grid_config;

/* GridLevelSpec, grid.hpp:59-64, plus the level's first row in the flat table. */
typedef struct {
    int32_t level;
    uint32_t resolution;
    uint32_t table_len;
    int32_t dense;
    uint64_t row_offset;
} nfg_level_spec;

/* MlpConfig, mlp.hpp:15-40. input_width is overwritten with levels*features
 * by nfg_field_create (model.cpp:101). */
typedef struct {
    int32_t input_width;
    int32_t hidden_layers;
    int32_t hidden_width;
    int32_t output_width;
    int32_t output_activation; /* nfg_output_activation */
} nfg_mlp_config;

/* AdamHyper, adam.hpp:13-25. */
typedef struct {
    double lr;
    double beta1;
    double beta2;
    double eps;
    double l2;
} nfg_adam_hyper;

/* Build options of the sm_100a path (no reference equivalent). */
typedef struct {
    int32_t table_fp32;    /* 1: gather fp32 master tables (exact-parity mode); 0: fp16 shadow (default) */
    int32_t fused_train;   /* 1: one fused encode+MLP+loss+backward kernel per step (default); 0: staged kernels */
    int32_t deterministic; /* 1: run-to-run bit-reproducible backward: table gradients accumulate per
                              row in the reference's order (grid.hpp:286-294; bit-identical to it for equal dY),
                              MLP gradients and the loss sum reduce per-CTA partials in a fixed order. Slower. */
    int32_t mlp_engine;    /* tensor-core engine of the fused kernels' MLP (north star: "mma.sync or tcgen05,
                              whichever is faster at width 64"): NFG_MMA_DEFAULT picks the measured-faster one per
                              kernel, NFG_MMA_SYNC / NFG_MMA_TCGEN05 force one. Kernels or shapes
                              without a tcgen05 build use mma.sync. */
    int32_t dp_exchange;   /* data-parallel gradient exchange (an NCCL communicator attached).
                              NFG_DP_ALLREDUCE (= NFG_DP_DEFAULT): one fused kernel, then the gradient slab all-reduced
                              in chunks on a comm stream, Adam updating each chunk as soon as it is reduced.
                              NFG_DP_LEVELS: the fused kernel stores dY instead of scattering; the table gradients are
                              then scattered level group by level group (finest first) and each group's all-reduce and
                              Adam start while later groups scatter. Hides the exchange behind the scatter but the
                              unfused scatter costs more than it hides (measured). */
} nfg_options;

enum { NFG_MMA_DEFAULT = 0, NFG_MMA_SYNC = 1, NFG_MMA_TCGEN05 = 2 };
enum { NFG_DP_DEFAULT = 0, NFG_DP_ALLREDUCE = 1, NFG_DP_LEVELS = 2 };

typedef struct nfg_ctx nfg_ctx;
typedef struct nfg_field nfg_field;

/* ---- context ---------------------------------------------------------- */
const char* nfg_last_error(void);
/* Diagnostics (no reference equivalent): the template instantiation of the
 * last fused train (which = 0) or inference (which = 1) kernel this thread
 * launched, e.g. "k_train ... table=f16 ... stage_alias=1". Lets parity tests
 * assert they exercised the exact variant bench.py measures. Thread-local. */
const char* nfg_last_kernel_variant(int32_t which);
/* Diagnostics (no reference equivalent): live L2-level throughput of this GPU
 * for the hot path's access patterns, measured at full occupancy on a 32 MB +
 * 64 MB L2-resident footprint (csrc/diag.cu). op 0: random 4 B L2 reads
 * (sectors/s); 1: random 4 B cp.async (sectors/s); 2: random
 * red.global.add.v2.f32 (sectors/s); 3: coalesced L2 streaming reads (bytes/s);
 * 4: random 4 B ld.global.nc (sectors/s). The roofline denominators of
 * bench.py. Synchronises the context stream. */
nfg_status nfg_diag_l2_peak(nfg_ctx* ctx, int32_t op, double* rate);
int nfg_abi_version(void);
nfg_status nfg_ctx_create(int device, nfg_ctx** out);
nfg_status nfg_ctx_destroy(nfg_ctx* ctx);
nfg_status nfg_ctx_synchronize(nfg_ctx* ctx);
void* nfg_ctx_stream(nfg_ctx* ctx); /* cudaStream_t */
/* Number of kernels this library has launched on ctx (for the bench's gpu_launches). */
uint64_t nfg_ctx_launch_count(nfg_ctx* ctx);

/* Device-side phase timing with CUDA events on the context stream (off by
 * default). read_profile returns the summed milliseconds since the last read:
 * ms[0] fused train kernel (or staged encode+MLP+encode-bwd), ms[1] Adam,
 * ms[2] gradient all-reduce, ms[3] inference kernel; *steps = train steps. */
nfg_status nfg_ctx_set_profiling(nfg_ctx* ctx, int on);
nfg_status nfg_ctx_read_profile(nfg_ctx* ctx, double ms[4], int64_t* steps);

/* Multi-GPU data parallelism (one process per GPU). id is an opaque 128-byte
 * ncclUniqueId produced on rank 0 and broadcast by the caller. With a comm
 * attached, train steps all-reduce the gradient slab before Adam. */
nfg_status nfg_comm_unique_id(uint8_t id[128]);
nfg_status nfg_ctx_attach_comm(nfg_ctx* ctx, const uint8_t id[128], int rank, int nranks);
/* Rank and size as the attached NCCL communicator reports them (0 and 1
 * without one): the bench asserts the job really runs on N ranks. */
nfg_status nfg_ctx_comm_info(nfg_ctx* ctx, int* rank, int* nranks);

/* ---- level table (grid.hpp:66-84), host only ---------------------------- */
/* Writes min(cap, levels) specs; returns the level count or -1 on error. */
int32_t nfg_level_resolutions(const nfg_grid_config* cfg, nfg_level_spec* out, int32_t cap);
double nfg_growth_factor(const nfg_grid_config* cfg);            /* grid.hpp:49-54 */
uint32_t nfg_spatial_hash(const uint32_t* coords, int32_t dims, uint32_t table_size); /* grid.hpp:88-95 */

/* ---- FieldModel (model.hpp:21-63) -------------------------------------- */
/* hyper and opts may be NULL (reference defaults / library defaults). */
nfg_status nfg_field_create(nfg_ctx* ctx, const nfg_grid_config* grid, const nfg_mlp_config* mlp,
                            const nfg_adam_hyper* hyper, const nfg_options* opts, nfg_field** out);
nfg_status nfg_field_destroy(nfg_field* f);
/* FieldModel::init (model.cpp:23-37): PCG32 table init, Glorot MLP, zero grads/moments. */
nfg_status nfg_field_init(nfg_field* f, uint64_t seed);
nfg_status nfg_field_set_hyper(nfg_field* f, const nfg_adam_hyper* hyper);
/* LrSchedule (adam.hpp:124-137). */
nfg_status nfg_field_set_schedule(nfg_field* f, const int64_t* milestones, int32_t n, double factor);
/* {table params, MLP weights, MLP biases} counts. */
nfg_status nfg_field_sizes(const nfg_field* f, uint64_t out[3]);
nfg_status nfg_field_levels(const nfg_field* f, nfg_level_spec* out, int32_t cap);
/* Host mirrors of the public members (tables.values, mlp, adam state). */
nfg_status nfg_field_read(nfg_field* f, int32_t which, uint64_t offset, uint64_t count, float* host);
nfg_status nfg_field_write(nfg_field* f, int32_t which, uint64_t offset, uint64_t count, const float* host);
nfg_status nfg_field_device_buffer(nfg_field* f, int32_t which, float** dev, uint64_t* count);
/* AdamState::step (adam.hpp:56-73). */
nfg_status nfg_field_get_config(const nfg_field* f, nfg_grid_config* grid, nfg_mlp_config* mlp);
nfg_status nfg_field_context(const nfg_field* f, nfg_ctx** ctx);
nfg_status nfg_field_get_step(const nfg_field* f, uint64_t* step);
nfg_status nfg_field_set_step(nfg_field* f, uint64_t step);
/* Data parallelism: every rank takes root's parameters, Adam m/v and step
 * (ncclBroadcast on the attached communicator; a no-op without one). The
 * replicated Adam step of the ranks stays in lock-step only from identical
 * state (no reference equivalent: the reference is single-process). */
nfg_status nfg_field_broadcast(nfg_field* f, int root);

/* FieldModel::train_step (model.cpp:111-138): encode -> MLP -> loss ->
 * backward -> Adam at lr_at(schedule, lr, step). Host pointers; returns the
 * batch loss. X is dims x B, target n_out x B. */
nfg_status nfg_field_train_step(nfg_field* f, const float* X, const float* target, int64_t B,
                                int32_t loss_kind, int64_t step, float* loss);
/* The same with an explicit global batch (SURVEY §8b's nfg_field_train_step
 * signature): with data-parallel ranks holding ragged shards, every rank passes
 * its own B_local and the common B_global; the loss gradient is normalised by
 * B_global * n_out (losses.hpp:16) and the returned loss is this shard's share.
 * nfg_field_train_step is this call with B_global = B * nranks. Pinned and
 * pageable host buffers are both streamed under the fused kernel (pageable ones
 * through pinned bounce buffers filled by host copy threads). */
nfg_status nfg_field_train_step_global(nfg_field* f, const float* X, const float* target, int64_t B_local,
                                       int64_t B_global, int32_t loss_kind, int64_t step, float* loss);
/* Same on device pointers, asynchronous. B_global is the global batch across
 * data-parallel ranks (loss normalisation, losses.hpp:16). loss_dev (device
 * float, may be NULL) receives the global-batch loss of this rank's shard. */
nfg_status nfg_field_train_step_device(nfg_field* f, const float* X, const float* target,
                                       int64_t B_local, int64_t B_global, int32_t loss_kind,
                                       int64_t step, float* loss_dev);
/* Per-step status of asynchronous device steps, for loops that check lazily
 * (nfg_fit_image): nfg_field_step_record copies the step's 32-byte device
 * scratch (loss sum + abort flags) into rec_dev, stream-ordered after the last
 * enqueued step; nfg_step_record_check turns a host copy of it into exactly
 * what the synchronous train_step would have done: the same error (EINVAL for
 * invalid input, ENONFINITE naming the group) or the step's loss. */
typedef struct {
    double loss_sum;
    uint32_t flags[4];
    float dy_max;
    float pad;
} nfg_step_record;
nfg_status nfg_field_step_record(nfg_field* f, nfg_step_record* rec_dev);
nfg_status nfg_step_record_check(nfg_field* f, const nfg_step_record* rec, int64_t B_global, float* loss);
/* Forward + loss + backward of train_step WITHOUT the Adam update: gradients
 * accumulate into the field's grad slab (mlp_backward / encode_backward
 * semantics, mlp.hpp:147-148, grid.hpp:292); pair with nfg_adam_step. */
nfg_status nfg_field_gradients(nfg_field* f, const float* X, const float* target, int64_t B,
                               int32_t loss_kind, float* loss);
/* Non-finite check of the last device step (synchronises). */
nfg_status nfg_field_check(nfg_field* f);

/* FieldModel::evaluate (model.cpp:102-109): fused encode + MLP inference. */
nfg_status nfg_field_evaluate(nfg_field* f, const float* X, int64_t B, float* out);
nfg_status nfg_field_evaluate_device(nfg_field* f, const float* X, int64_t B, float* out);

/* ---- components on the field's tables / MLP (host pointers) ------------- */
/* encode_forward (grid.hpp:219-272). rows (u32) and weights (f32), shaped
 * (L, B, 2^d) like EncodeCache (grid.hpp:183-195), are exported when non-NULL. */
nfg_status nfg_encode_forward(nfg_field* f, const float* X, int64_t B, float* Y, uint32_t* rows,
                              float* weights);
/* encode_backward (grid.hpp:277-295): accumulates dLoss/dTables into the
 * field's table grads. The GPU cache is the input X itself (rows and weights
 * are recomputed, never materialised). */
nfg_status nfg_encode_backward(nfg_field* f, const float* X, int64_t B, const float* dY);
/* mlp_forward (mlp.hpp:104-124) with the field's MLP. Y is input_width x B. */
nfg_status nfg_mlp_forward(nfg_field* f, const float* Y, int64_t B, float* out);
/* mlp_backward (mlp.hpp:129-158): recomputes the forward for Y, accumulates
 * into the field's MLP grads and writes dY. */
nfg_status nfg_mlp_backward(nfg_field* f, const float* Y, int64_t B, const float* dOut, float* dY);
/* l2_loss / mape_loss / relative_l2_loss (losses.hpp:10-59): n values,
 * gradient normalised by count (= n for the reference). */
nfg_status nfg_loss(nfg_ctx* ctx, int32_t loss_kind, const float* pred, const float* target,
                    int64_t n, int64_t count, float* dpred, float* loss);
/* adam_step over the field's three groups (model.cpp:49-77 + adam.hpp:78-122). */
nfg_status nfg_adam_step(nfg_field* f, float lr_now);
/* lr_at (adam.hpp:139-146). */
double nfg_lr_at(const int64_t* milestones, int32_t n, double factor, double base_lr, int64_t step);

/* ---- pinned host memory for zero-copy-staged inputs -------------------- */
/* ---- device-pointer components (asynchronous; errors via nfg_field_check) --
 * For pipelines that chain fields on the device (the NeRF density -> color
 * networks). Gradients accumulate into the field's slab (mlp.hpp:147-148,
 * grid.hpp:292); nfg_adam_step_device applies adam_step (adam.hpp:78-122)
 * and zeroes them (the exact non-finite scan runs when a producer kernel
 * flagged a possibly non-finite gradient). dOut is dLoss/d(output after
 * the output activation), as mlp_backward's dOut. */
nfg_status nfg_field_backward_device(nfg_field* f, const float* X, int64_t B, const float* dOut);
nfg_status nfg_mlp_forward_device(nfg_field* f, const float* Y, int64_t B, float* out);
nfg_status nfg_mlp_backward_device(nfg_field* f, const float* Y, int64_t B, const float* dOut, float* dY);
nfg_status nfg_adam_step_device(nfg_field* f, float lr_now);

/* ---- checkpoint (io.cpp:222-351, NFC1/HGE1/MLP1/ADM1) --------------------
 * Byte-compatible with the reference's save_checkpoint / load_checkpoint for
 * hash-encoder models. load creates a new field from the file's configs (the
 * reference's load_checkpoint also replaces hash_cfg / mlp_cfg), with hyper
 * and options supplied by the caller as a resume does (test_tasks.cpp:313-315).
 * Errors: NFG_EIO with the reference's messages ("checkpoint: missing ...
 * section", "checkpoint: truncated ...", "checkpoint: level length mismatch",
 * "cannot read/write checkpoint: <path>"); NFG_EUNSUPPORTED for OCT1 /
 * frequency-encoder files. */
nfg_status nfg_field_save(nfg_field* f, const char* path);
nfg_status nfg_field_load(nfg_ctx* ctx, const char* path, const nfg_adam_hyper* hyper, const nfg_options* opts,
                          nfg_field** out);

/* ---- training-loop data path on the device (tasks.cpp) ---
 * nfg_rng: the reference's Pcg32 (pcg32.hpp) as a device stream. Draws are
 * generated in parallel by jump-ahead, bit-identical to the sequential host
 * generator INCLUDING next_below's rejection sampling: n draws advance the
 * stream exactly as n host calls would. Asynchronous on the context stream;
 * nfg_rng_get_state synchronises. */
typedef struct nfg_rng nfg_rng;
nfg_status nfg_rng_create(nfg_ctx* ctx, uint64_t seed, uint64_t seq, nfg_rng** out);   /* Pcg32(seed, seq) */
nfg_status nfg_rng_destroy(nfg_rng* r);
nfg_status nfg_rng_below_device(nfg_rng* r, uint32_t bound, int64_t n, uint32_t* out_dev);   /* next_below x n */
nfg_status nfg_rng_floats_device(nfg_rng* r, int64_t n, float* out_dev);                     /* next_float x n */
nfg_status nfg_rng_u32_device(nfg_rng* r, int64_t n, uint32_t* out_dev);                      /* next_u32 x n */
nfg_status nfg_rng_get_state(nfg_rng* r, uint64_t* state, uint64_t* inc);

/* fit_image's batch assembly (tasks.cpp:114-120): pixel p -> X = (((p % w) +
 * 0.5) / w, ((p / w) + 0.5) / h) in fp32, T = rgb column p (rgb: 3 x w*h,
 * the reference's Image::rgb). idx_dev == NULL means p = i. */
nfg_status nfg_image_batch_device(nfg_ctx* ctx, const uint32_t* idx_dev, int64_t n, const float* rgb_dev,
                                  int32_t width, int32_t height, float* X_dev, float* T_dev);

/* ImageTask (tasks.hpp:16-31) for the hash encoder; cfg.dims is forced to 2,
 * cfg.n_max <= 0 means width / 2, cfg.interpolation is task.interpolation. */
typedef struct {
    int32_t width, height;
    nfg_grid_config cfg;
    int32_t hidden_layers;
    int32_t hidden_width;
    int32_t batch_size;
    int64_t total_steps;
    int64_t log_interval;
    double lr;
    double lr_decay;
} nfg_image_task;

/* TrainReportRow (io.hpp:25-31). */
typedef struct {
    int64_t step;
    double time_s;
    double loss;
    double metric;
    double lr;
} nfg_report_row;

/* fit_image (tasks.cpp:49-131) with every step on the device: batches drawn
 * from Pcg32(seed, 1) on the GPU (identical pixel sequence), PSNR rows on the
 * full image (<= 2^20 pixels) or 2^16 pixels from Pcg32(seed, 7). The model is
 * returned in *model_out (destroy with nfg_field_destroy); up to rows_cap
 * report rows are written, *n_rows = rows produced. Errors as the reference:
 * EINVAL ("fit_image: image must be at least 2x2"), ENONFINITE ("fit_image:
 * non-finite loss at step N" / adam_step's non-finite gradient). */
nfg_status nfg_fit_image(nfg_ctx* ctx, const nfg_image_task* task, const float* rgb, uint64_t seed,
                         const nfg_options* opts, nfg_field** model_out, nfg_report_row* rows, int64_t rows_cap,
                         int64_t* n_rows);

/* ---- inference consumers (tasks.cpp:195-356) -------------
 * A field is an nfg_field model, evaluated by the fused sm_100a inference, or, when field == NULL, a
 * host FieldFn callback (tasks.hpp:70): X is d x n column-major on the host,
 * out receives 1 x n (any function, e.g. an analytic SDF). */
typedef void (*nfg_field_fn)(const float* X, int64_t n, float* out, void* user);
/* oracle sign for iou (tasks.hpp:90-92): the point is 3 doubles. */
typedef int (*nfg_sign_fn)(const double* p, void* user);
/* Camera (tasks.hpp:72-77). */
typedef struct {
    double position[3];
    double target[3];
    double up[3];
    double fov_deg;
} nfg_camera;

/* render_image (tasks.cpp:195-209): the 2D model at every pixel centre;
 * rgb_host receives output_width x (width*height), pixel i = y*width + x. */
nfg_status nfg_render_image(nfg_field* f, int32_t width, int32_t height, float* rgb_host);
/* render_sdf_shaded (tasks.cpp:233-329): sphere tracing (step = field value,
 * hit at < 1e-4, <= 256 steps) with active-ray compaction on the device,
 * central-difference normals (h = 1e-3), Lambert headlight; background 1.
 * rgb_host: 3 x (width*height). */
nfg_status nfg_render_sdf_shaded(nfg_ctx* ctx, nfg_field* field, nfg_field_fn fn, void* user, const nfg_camera* cam,
                                 int32_t width, int32_t height, float* rgb_host);
/* iou (tasks.cpp:331-356): interior IoU of the field (< 0) and oracle_sign
 * (< 0) at n_points uniform points in [lo, hi] drawn from rng exactly as
 * Pcg32::uniform<double> (x, y, z per point); 1 when neither interior shows. */
nfg_status nfg_iou(nfg_ctx* ctx, nfg_field* field, nfg_field_fn fn, void* user, nfg_sign_fn oracle_sign,
                   void* sign_user, int64_t n_points, nfg_rng* rng, const double lo[3], const double hi[3],
                   double* out);

/* ---- NeRF (§5.4 + Appendix E) -------------------
 * Density network: hash encoding (levels * features == 32) -> 1 x 64 -> 16
 * outputs, the first is log-density; color network: [16 density outputs |
 * SH degree-4 of the view direction] -> 2 x 64 -> RGB (sigmoid). Training
 * steps march rays through a 128^3 occupancy bitfield (Morton order) at
 * dt = sqrt(3)/1024 in [0,1]^3, compact the samples into dense buffers,
 * composite (transmittance stop at 1e-4), and update the occupancy grid
 * every 16 steps. The reference has no NeRF: parity is against
 * a restatement of the paper's appendix (oracle/oracle.py). */
typedef struct {
    nfg_grid_config grid;        /* density encoding; dims forced to 3 */
    double lr;                   /* Adam learning rate (eps 1e-15, beta 0.9 / 0.99) */
    int32_t target_samples;      /* samples per training step (2^18) */
    int32_t max_samples_per_ray; /* 1024 */
    float background[3];
} nfg_nerf_config;
typedef struct nfg_nerf nfg_nerf;
nfg_status nfg_nerf_create(nfg_ctx* ctx, const nfg_nerf_config* cfg, uint64_t seed, nfg_nerf** out);
nfg_status nfg_nerf_destroy(nfg_nerf* n);
nfg_status nfg_nerf_fields(nfg_nerf* n, nfg_field** density, nfg_field** color);
/* cams: n_views x 12 floats (position, forward, right, up); a pixel (x, y)
 * looks along normalize(forward + u right + v up), u = (x + 0.5 - w/2) / focal,
 * v = (h/2 - y - 0.5) / focal. rgb: n_views x height x width x 3. */
nfg_status nfg_nerf_set_dataset(nfg_nerf* n, int32_t n_views, int32_t width, int32_t height, float focal,
                                const float* cams, const float* rgb);
nfg_status nfg_nerf_train_step(nfg_nerf* n, int64_t step, float* loss, int64_t* rays_used, int64_t* samples_used);
/* ... also reporting how many samples reached the backward networks (those
 * before their ray's transmittance stop, compacted into dense buffers). */
nfg_status nfg_nerf_train_step2(nfg_nerf* n, int64_t step, float* loss, int64_t* rays_used, int64_t* samples_used,
                                int64_t* samples_backward);
nfg_status nfg_nerf_update_occupancy(nfg_nerf* n, int64_t step);
/* Completes the work a training step defers (its networks' Adam step runs at the
 * start of the next call; every entry point that uses the networks applies it
 * first) and synchronises the NeRF's stream. */
nfg_status nfg_nerf_sync(nfg_nerf* n);
nfg_status nfg_nerf_render(nfg_nerf* n, const float* cam12, int32_t width, int32_t height, float focal, float* rgb);
nfg_status nfg_nerf_occupancy(nfg_nerf* n, uint8_t* bits, float* density);   /* 128^3/8 bytes, 128^3 floats */
nfg_status nfg_nerf_set_occupancy(nfg_nerf* n, const uint8_t* bits);
/* components on host buffers (tests): marching + compaction (rays n x 6:
 * origin, unit direction; samples: total x 3 positions), compositing forward
 * and backward (raw = log-density per sample), SH4, and the synthetic scene
 * (three textured soft spheres) rendered by fine marching. */
nfg_status nfg_nerf_march(nfg_ctx* ctx, const float* rays, int64_t n, const uint8_t* bits, int32_t max_steps,
                          uint32_t* counts, float* samples, int64_t cap, int64_t* total);
nfg_status nfg_nerf_composite(nfg_ctx* ctx, int64_t n_rays, const uint32_t* counts, const float* raw,
                              const float* rgb, const float* target, const float* bg, float dt, float* color,
                              float* d_rgb, float* d_raw, double* loss_sum);
nfg_status nfg_nerf_sh4(nfg_ctx* ctx, const float* dirs, int64_t n, float* out);
nfg_status nfg_nerf_scene_render(nfg_ctx* ctx, const float* cams, int32_t n_views, int32_t width, int32_t height,
                                 float focal, const float* bg, float* rgb);

/* fit_sdf (tasks.cpp:133-193) on the ANALYTIC CSG target of BASELINE config 2
 * (sphere r=0.3 at the centre union a torus R=0.25, r=0.08 in the xz-plane):
 * uniform points from Pcg32(seed, 2) replace the reference's mesh sampling
 * (geometry is out of scope), the metric column is the interior IoU against
 * the analytic sign on iou_eval_points from Pcg32(seed, 11) (tasks.cpp:163-171),
 * row 0 has loss 0 (tasks.cpp:173). */
typedef struct {
    nfg_grid_config cfg;     /* dims forced to 3 */
    int32_t hidden_layers;
    int32_t hidden_width;
    int32_t batch_size;
    int32_t loss;            /* nfg_loss_kind; the reference's SdfTask default is MAPE */
    int64_t total_steps;
    int64_t log_interval;
    int64_t iou_eval_points;
    double lr;
    double lr_decay;
} nfg_sdf_task;
nfg_status nfg_fit_sdf_analytic(nfg_ctx* ctx, const nfg_sdf_task* task, uint64_t seed, const nfg_options* opts,
                                nfg_field** model_out, nfg_report_row* rows, int64_t rows_cap, int64_t* n_rows);
/* The config-2 CSG SDF at n points (X: n x 3 device), in the oracle's fp32 order. */
nfg_status nfg_csg_sdf_device(nfg_ctx* ctx, const float* X_dev, int64_t n, float* out_dev);

nfg_status nfg_host_alloc(size_t bytes, void** out);
nfg_status nfg_host_free(void* p);

#ifdef __cplusplus
}
#endif

#endif /* NFG_H */
