// field.cu — the C ABI (include/nfg.h): contexts, the device-resident
// FieldModel and the component entry points. Host orchestration only; the
// math lives in the kernels.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/nfg.h"
#include "host_init.h"
#include "kernels.h"

namespace nfg {
namespace {
thread_local std::string g_variant[2];
}
void note_kernel_variant(int which, const char* desc) { g_variant[which & 1] = desc; }
}   // namespace nfg

namespace {

thread_local std::string g_err;

struct Fail {
    nfg_status st;
    std::string msg;
};

#define NFG_CUDA(call)                                                                                  \
    do {                                                                                                \
        const cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess)                                                                          \
            throw Fail{ e_ == cudaErrorNotSupported ? NFG_EUNSUPPORTED : NFG_ECUDA,                     \
                        std::string(#call) + ": " + cudaGetErrorString(e_) };                           \
    } while (0)

// NCCL is resolved at run time (dlopen) and only when a communicator is
// attached: a process that imported torch first reuses torch's libnccl.so.2,
// and single-GPU users never load NCCL at all.
struct NcclApi {
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) comm_init_rank = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclAllReduce) all_reduce = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
    decltype(&ncclCommCount) comm_count = nullptr;
    decltype(&ncclCommUserRank) comm_user_rank = nullptr;
    decltype(&ncclBroadcast) broadcast = nullptr;
};

const NcclApi& nccl()
{
    static NcclApi api;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (h) {
            api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
            api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
            api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
            api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
            api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
            api.comm_count = reinterpret_cast<decltype(api.comm_count)>(dlsym(h, "ncclCommCount"));
            api.comm_user_rank = reinterpret_cast<decltype(api.comm_user_rank)>(dlsym(h, "ncclCommUserRank"));
            api.broadcast = reinterpret_cast<decltype(api.broadcast)>(dlsym(h, "ncclBroadcast"));
        }
    }
    if (!api.get_unique_id || !api.comm_init_rank || !api.all_reduce)
        throw Fail{ NFG_ENCCL, "libnccl.so.2 could not be loaded" };
    return api;
}

#define NFG_NCCL(call)                                                                                  \
    do {                                                                                                \
        const ncclResult_t r_ = (call);                                                                 \
        if (r_ != ncclSuccess)                                                                          \
            throw Fail{ NFG_ENCCL, std::string(#call) + ": " + nccl().error_string(r_) };               \
    } while (0)

template <class Fn>
nfg_status guard(Fn&& fn)
{
    try {
        fn();
        return NFG_OK;
    } catch (const Fail& f) {
        g_err = f.msg;
        return f.st;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return NFG_EINVAL;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return NFG_ELOGIC;
    } catch (const std::exception& e) {
        g_err = e.what();
        return NFG_ECUDA;
    }
}

void require(bool ok, const char* msg)
{
    if (!ok)
        throw std::invalid_argument(msg);
}

// Page-locked host staging (bounce) buffer for pageable callers.
struct HostBuf {
    void* p = nullptr;
    size_t bytes = 0;
    void* get(size_t n)
    {
        if (n > bytes) {
            if (p)
                cudaFreeHost(p);
            p = nullptr;
            bytes = 0;
            if (cudaHostAlloc(&p, n, cudaHostAllocDefault) != cudaSuccess)
                throw Fail{ NFG_ECUDA, "cudaHostAlloc bounce buffer failed" };
            bytes = n;
        }
        return p;
    }
    ~HostBuf()
    {
        if (p)
            cudaFreeHost(p);
    }
};

// Pageable -> pinned copies of a streamed batch on the calling thread plus a
// few persistent host threads. A job is a list of chunks; every participant
// copies its 1/n slice of chunk 0, then of chunk 1, ... and bumps the chunk's
// counter, so the caller puts chunk k on the copy engine as soon as all slices
// of chunk k landed, while the others already copy chunk k+1 (and the fused
// kernel runs). Workers spin for a while after a job (back-to-back steps
// arrive well within that window) before they block, so a step does not pay
// thread wake-ups.
struct CopyPool {
    struct Part {
        const char* src;
        char* dst;
        size_t bytes;
    };
    std::vector<std::thread> threads;
    std::mutex mu;
    std::condition_variable cv;
    std::atomic<uint64_t> gen{ 0 };
    std::atomic<bool> stop{ false };
    std::atomic<int> sleepers{ 0 };
    const std::vector<std::vector<Part>>* job = nullptr;   // job[k] = copies of chunk k
    std::atomic<int> done[64];                              // >= NFG_MAX_CHUNKS
    int n = 0;                                              // participants: workers + the caller

    explicit CopyPool(int workers) : n(workers + 1)
    {
        for (auto& d : done)
            d.store(0);
        for (int i = 0; i < workers; ++i)
            threads.emplace_back([this, i] { run(i + 1); });
    }
    ~CopyPool()
    {
        {
            std::lock_guard<std::mutex> l(mu);
            stop.store(true);
        }
        cv.notify_all();
        for (auto& t : threads)
            t.join();
    }
    void copy_slice(size_t k, int me)
    {
        for (const Part& p : (*job)[k]) {
            const size_t lo = p.bytes * size_t(me) / size_t(n), hi = p.bytes * size_t(me + 1) / size_t(n);
            std::memcpy(p.dst + lo, p.src + lo, hi - lo);
        }
        done[k].fetch_add(1, std::memory_order_acq_rel);
    }
    void run(int me)
    {
        uint64_t seen = 0;
        for (;;) {
            int spins = 0;
            while (gen.load(std::memory_order_acquire) == seen && !stop.load(std::memory_order_relaxed)) {
                if (++spins < 200000) {
                    std::this_thread::yield();
                    continue;
                }
                std::unique_lock<std::mutex> l(mu);
                sleepers.fetch_add(1);
                cv.wait(l, [&] { return stop.load() || gen.load() != seen; });
                sleepers.fetch_sub(1);
            }
            if (stop.load())
                return;
            seen = gen.load(std::memory_order_acquire);
            for (size_t k = 0; k < job->size(); ++k)
                copy_slice(k, me);
        }
    }
    void start(const std::vector<std::vector<Part>>& j)
    {
        for (size_t k = 0; k < j.size(); ++k)
            done[k].store(0, std::memory_order_relaxed);
        job = &j;
        {
            std::lock_guard<std::mutex> l(mu);
            gen.fetch_add(1, std::memory_order_acq_rel);
        }
        if (sleepers.load() > 0)
            cv.notify_all();
    }
    // the caller's share of chunk k, then wait for the workers' shares
    void finish_chunk(size_t k)
    {
        copy_slice(k, 0);
        while (done[k].load(std::memory_order_acquire) < n)
            std::this_thread::yield();
    }
    void drain(size_t nchunks)
    {
        for (size_t k = 0; k < nchunks; ++k)
            while (done[k].load(std::memory_order_acquire) < n)
                std::this_thread::yield();
    }
};

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    void* get(size_t n)
    {
        if (n > bytes) {
            if (p)
                cudaFree(p);
            p = nullptr;
            bytes = 0;
            if (cudaMalloc(&p, n) != cudaSuccess)
                throw Fail{ NFG_ECUDA, "cudaMalloc staging buffer failed" };
            bytes = n;
        }
        return p;
    }
    ~DevBuf()
    {
        if (p)
            cudaFree(p);
    }
};

}   // namespace

namespace nfg {
void set_last_error(const std::string& msg) { g_err = msg; }
}   // namespace nfg

struct nfg_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    int num_sms = 148;
    uint64_t launches = 0;
    ncclComm_t comm = nullptr;
    int rank = 0, nranks = 1;
    DevBuf s0, s1, s2, s3;   // staging for host-pointer calls
    HostBuf h0, h1;          // pinned bounce buffers for pageable streamed steps
    CopyPool* copy_pool = nullptr;
    double* d_red = nullptr;
    // streamed inputs: H2D chunks on a copy stream, each followed by a
    // stream memory write of its ready flag (copy engine + front end only)
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev_order = nullptr;
    // early step result (host-pointer steps): the loss / flags are read back on
    // res_stream as soon as the backward is final, while Adam still runs
    cudaStream_t res_stream = nullptr;
    cudaEvent_t ev_res = nullptr, ev_res_done = nullptr;
    // the last host call was a train step that returned once its fused kernel
    // had finished: nothing queued on the main stream reads the staging buffers
    bool staging_idle = false;
    // data parallelism: NCCL runs the gradient all-reduce in chunks on its own
    // stream while Adam updates the chunks already reduced
    cudaStream_t comm_stream = nullptr;
    cudaEvent_t ev_grads = nullptr;
    cudaEvent_t ev_chunk[8] = {};
    // level-pipelined exchange: per level group, scatter done (main) / reduced (comm)
    cudaEvent_t ev_scat[8] = {}, ev_red[8] = {}, ev_scr = nullptr;
    CUresult (*write_value32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int) = nullptr;
    // phase timing (nfg_ctx_set_profiling)
    bool profile = false;
    std::vector<cudaEvent_t> ev_pool;
    struct Rec {
        int kind;
        cudaEvent_t a, b;
    };
    std::vector<Rec> recs;
    int64_t prof_steps = 0;

    cudaEvent_t ev()
    {
        if (ev_pool.empty()) {
            cudaEvent_t e;
            if (cudaEventCreate(&e) != cudaSuccess)
                throw std::runtime_error("cudaEventCreate failed");
            return e;
        }
        cudaEvent_t e = ev_pool.back();
        ev_pool.pop_back();
        return e;
    }
};

namespace {
// RAII span: records a start/end event pair on the ctx stream when profiling.
struct Span {
    nfg_ctx* c;
    int kind;
    cudaEvent_t a = nullptr;
    Span(nfg_ctx* c_, int k) : c(c_), kind(k)
    {
        if (c->profile) {
            a = c->ev();
            cudaEventRecord(a, c->stream);
        }
    }
    ~Span()
    {
        if (a) {
            cudaEvent_t b = c->ev();
            cudaEventRecord(b, c->stream);
            c->recs.push_back({ kind, a, b });
        }
    }
};
}   // namespace

// Scratch block written by kernels and read back in one 32-byte copy.
struct StepResult {
    double loss_sum;
    unsigned int flags[4];
    float dy_max;
    float pad;
};

struct nfg_field {
    nfg_ctx* ctx = nullptr;
    nfg_grid_config gcfg{};
    nfg_mlp_config mcfg{};
    nfg_adam_hyper hyper{ 1e-2, 0.9, 0.99, 1e-15, 1e-6 };
    nfg_options opts{ 0, 1, 0, 0 };
    int train_grid = 0;   // CTAs of the last fused train launch (the persistent kernel's first wave)
    bool early_result = false;   // host_train_step: read the step result before Adam finishes
    std::vector<int64_t> milestones;
    double factor = 0.33;
    std::vector<nfg_level_spec> levels;
    nfg::FieldShape shape{};
    nfg::LevelDev* d_levels = nullptr;
    uint64_t n_tab = 0, n_w = 0, n_b = 0, n_total = 0, n_alloc = 0;   // reference (API) layout counts
    uint64_t n_tab_dev = 0, n_total_dev = 0;   // device layout: each level starts on an 8-row multiple
    std::vector<uint64_t> dev_row_off;        // per-level first row in the device layout
    float* d_p = nullptr;
    float* d_g = nullptr;
    float* d_m = nullptr;
    float* d_v = nullptr;
    __half* d_shadow = nullptr;
    StepResult* d_res = nullptr;   // followed in the same allocation by the 4-word sticky abort state
    StepResult* h_res = nullptr;   // pinned, same layout
    unsigned int* d_sticky = nullptr;   // [0] latched abort, [1] its group + 1, [2] its input flags, [3] Adam stand-downs
    uint64_t step = 0;
    uint64_t pending_steps = 0;    // device steps not yet checked (async API)
    // The gradient slab is all-zero (after init / a completed Adam step). Then a
    // step may validate its inputs speculatively inside the fused kernel and
    // undo by re-zeroing; otherwise k_validate runs first.
    bool grads_clean = true;
    int64_t last_batch = 0;            // global batch of the last backward (Adam's dense/sparse choice)
    // the step scratch was already reset at the end of the previous synchronous
    // train_step (after its status was read), so the next step skips it
    bool scratch_ready = false;
    // Streamed host-pointer steps start only after one plain step of this field
    // has run: with CUDA's lazy module loading, the first launch of a kernel
    // (Adam's) can block the host until the device idles, while the already
    // running fused kernel waits for copies the host has not enqueued yet.
    bool stream_warm = false;
    bool fused_ok = true;   // fused encode+MLP kernels exist for this shape
    unsigned int* d_ready = nullptr;   // NFG_MAX_CHUNKS chunk-ready flags
    unsigned int epoch = 0;
    DevBuf det_part, det_loss, det_sort;   // deterministic mode scratch
    DevBuf comp_y, comp_dy;                // nfg_field_backward_device scratch
};

#define NFG_MAX_CHUNKS 64
#define NFG_STREAM_CHUNKS 8   // H2D chunks per streamed step (<= NFG_MAX_CHUNKS)

namespace {

nfg::StepScratch scratch_of(nfg_field* f)
{
    nfg::StepScratch s;
    s.loss_sum = &f->d_res->loss_sum;
    s.flags = f->d_res->flags;
    s.dy_max = &f->d_res->dy_max;
    return s;
}

// Starts a step's scratch (k_step_begin). With unchecked asynchronous steps
// pending, a previous abort is latched into the sticky word and this step
// stands down; otherwise (the host has read every result) the sticky word is
// cleared too.
void reset_scratch(nfg_field* f)
{
    f->scratch_ready = false;   // any other user dirties it after this reset
    const int inherit = f->pending_steps > 0 ? 1 : 0;
    NFG_CUDA(nfg::launch_step_begin(&f->d_res->loss_sum, f->d_res->flags, &f->d_res->dy_max, f->d_sticky, inherit,
                                    f->ctx->stream));
    f->ctx->launches++;
}

const unsigned int* sticky_host(const nfg_field* f) { return reinterpret_cast<const unsigned int*>(f->h_res + 1); }

const char* group_name(unsigned g)
{
    switch (g) {
    case 0: return "tables";
    case 1: return "mlp_weights";
    default: return "mlp_biases";
    }
}

void fetch_result(nfg_field* f)
{
    NFG_CUDA(cudaMemcpyAsync(f->h_res, f->d_res, sizeof(StepResult) + 4 * sizeof(unsigned int), cudaMemcpyDeviceToHost,
                             f->ctx->stream));
    NFG_CUDA(cudaStreamSynchronize(f->ctx->stream));
}

void raise_if_aborted(nfg_field* f)
{
    if (f->h_res->flags[3] == 4u)
        throw std::logic_error("train_step: skipped because an earlier asynchronous step aborted "
                               "(nfg_field_check reports it)");
    if (f->h_res->flags[3] & 1u)
        throw std::invalid_argument("encode_forward: non-finite input");
    if (f->h_res->flags[3] & 2u)
        throw std::invalid_argument("encode_forward: input outside [0,1]^d");
    if (f->h_res->flags[1]) {
        const unsigned g = f->h_res->flags[2] == 0xffffffffu ? 0u : f->h_res->flags[2] - 1u;
        throw Fail{ NFG_ENONFINITE, std::string("adam_step: non-finite gradient in group '") + group_name(g) + "'" };
    }
}

// Reads back the asynchronous steps issued since the last check. The first
// abort among them (latched in the sticky word, or the last step's own) is
// reported like the reference's throw; every step that stood down behind it
// left the state untouched, and the host step counter drops by the number of
// Adam launches that did not apply (sticky[3]).
void settle_pending(nfg_field* f)
{
    fetch_result(f);
    f->pending_steps = 0;
    const unsigned int* sk = sticky_host(f);
    if (sk[0] == 0u && f->h_res->flags[1] == 0u)
        return;
    f->step -= sk[3];
    if (sk[0]) {
        f->h_res->flags[1] = 1u;
        f->h_res->flags[2] = sk[1];
        f->h_res->flags[3] = sk[2];
    }
    // invalid input on a clean slab was undone by re-zeroing; a non-finite
    // gradient stays in the slab (the reference throws before zeroing)
    f->grads_clean = (f->h_res->flags[3] & 3u) != 0;
    reset_scratch(f);   // pending == 0: clears the sticky word as well
    f->scratch_ready = true;
    raise_if_aborted(f);
}

const void* table_ptr(nfg_field* f) { return f->opts.table_fp32 ? static_cast<const void*>(f->d_p) : f->d_shadow; }

void refresh_shadow(nfg_field* f)
{
    NFG_CUDA(nfg::launch_shadow(f->d_p, f->d_shadow, f->n_tab_dev, f->ctx->stream));
    f->ctx->launches++;
}

// Kernel launches may block until completion (profilers and sanitizers inject
// through CUDA_INJECTION64_PATH; CUDA_LAUNCH_BLOCKING=1): a kernel that waits
// on copies enqueued after its launch would then never start them.
bool launches_serialized()
{
    static const bool v = [] {
        const char* lb = getenv("CUDA_LAUNCH_BLOCKING");
        const char* inj = getenv("CUDA_INJECTION64_PATH");
        const char* force = getenv("NFG_NO_STREAMING");
        return (lb && lb[0] == '1') || (inj && inj[0]) || (force && force[0] == '1');
    }();
    return v;
}

// True for page-locked (cudaHostAlloc / cudaHostRegister) host memory.
// The answer only steers the streamed-copy heuristic (a pageable source is
// still copied correctly), so the last few answers are cached per thread to
// keep cudaPointerGetAttributes off the per-step path.
bool is_pinned(const void* p)
{
    thread_local const void* cache_p[4] = { nullptr, nullptr, nullptr, nullptr };
    thread_local bool cache_v[4] = { false, false, false, false };
    thread_local int next = 0;
    for (int i = 0; i < 4; ++i)
        if (cache_p[i] == p)
            return cache_v[i];
    cudaPointerAttributes at{};
    bool v = false;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess)
        cudaGetLastError();
    else
        v = at.type == cudaMemoryTypeHost;
    cache_p[next] = p;
    cache_v[next] = v;
    next = (next + 1) & 3;
    return v;
}

template <class T>
T* stage(DevBuf& b, const T* host, size_t count, cudaStream_t st)
{
    T* d = static_cast<T*>(b.get(std::max<size_t>(count * sizeof(T), 16)));
    if (count)
        NFG_CUDA(cudaMemcpyAsync(d, host, count * sizeof(T), cudaMemcpyHostToDevice, st));
    return d;
}

nfg::AdamArgs adam_args(nfg_field* f, float lr_now)
{
    const uint64_t next = f->step + 1;
    const nfg::host::AdamScalars s = nfg::host::adam_scalars(f->hyper, next, lr_now);
    nfg::AdamArgs a{};
    a.p = f->d_p;
    a.g = f->d_g;
    a.m = f->d_m;
    a.v = f->d_v;
    a.shadow = f->d_shadow;
    a.n_tab = f->n_tab_dev;
    a.n_w = f->n_w;
    a.n_b = f->n_b;
    a.b1 = s.b1;
    a.b2 = s.b2;
    a.omb1 = s.omb1;
    a.omb2 = s.omb2;
    a.bc1 = s.bc1;
    a.bc2 = s.bc2;
    a.eps = s.eps;
    a.l2 = s.l2;
    a.lr = s.lr;
    a.flags = f->d_res->flags;
    a.restore_on_invalid = f->grads_clean ? 1 : 0;
    // Dense steps (the batch's corners cover at least every table row once:
    // B * 2^d >= T) load p/m/v together with g (one round trip, -9% Adam time
    // at config 2); sparse steps keep the g-first skip of untouched quads.
    // NFG_ADAM_EAGER=0/1 overrides (A/B runs).
    {
        static const int forced = [] {
            const char* e = getenv("NFG_ADAM_EAGER");
            return e ? atoi(e) : -1;
        }();
        const bool dense = (double(f->last_batch) * double(1u << f->gcfg.dims)) >= double(f->gcfg.table_size);
        a.eager = forced >= 0 ? forced : (dense ? 1 : 0);
    }
    a.mode = 0;
    a.sticky = f->d_sticky;
    return a;
}

void run_adam(nfg_field* f, float lr_now, bool force_check)
{
    const nfg::AdamArgs a = adam_args(f, lr_now);
    const uint64_t next = f->step + 1;
    NFG_CUDA(nfg::launch_adam(a, force_check, f->ctx->num_sms, f->ctx->stream));
    f->ctx->launches += 2;
    f->step = next;
}

// Deterministic-mode helpers (nfg_options.deterministic; det_kernels.cu).
// The staged MLP kernel writes per-CTA partials of dW/db (and the loss sum),
// reduced in CTA order; the table gradients go through the sorted per-row
// reduction that reproduces the reference's accumulation order.
void det_prepare(nfg_field* f, nfg::TrainArgs& a, int64_t B, bool with_loss)
{
    nfg_ctx* c = f->ctx;
    const int64_t ntiles = (B + 15) / 16;   // >= tiles of any train instantiation
    // tile workers: CTAs, or groups of CTAs (k_train TCW), plus a group's rounding slack
    const int64_t max_grid = std::min<int64_t>(ntiles, int64_t(c->num_sms) * 16) + 8;
    a.n_w = int64_t(f->n_w);
    a.n_wb = int64_t(f->n_w + f->n_b);
    a.part_wb = static_cast<float*>(f->det_part.get(size_t(std::max<int64_t>(max_grid, 1)) * size_t(a.n_wb) * 4));
    // idle workers (no tile) write no dW partials: start from zeros
    NFG_CUDA(cudaMemsetAsync(a.part_wb, 0, size_t(max_grid) * size_t(a.n_wb) * 4, c->stream));
    a.part_loss = with_loss ? static_cast<double*>(f->det_loss.get(
                                  size_t(std::max<int64_t>(max_grid, 1)) * nfg::train_warps_per_cta() * 8))
                            : nullptr;
}

void det_finish(nfg_field* f, const nfg::TrainArgs& a, int grid)
{
    nfg_ctx* c = f->ctx;
    if (grid <= 0)
        return;
    NFG_CUDA(nfg::launch_reduce_partials(a.part_wb, grid, a.n_wb, f->d_g + f->n_tab_dev, a.part_loss,
                                         grid * nfg::train_warps_per_cta(), &f->d_res->loss_sum, f->d_res->flags,
                                         c->stream));
    c->launches++;
}

void det_encode_bwd(nfg_field* f, const float* X, int64_t B, const float* dY)
{
    nfg_ctx* c = f->ctx;
    const size_t bytes = nfg::encode_bwd_det_scratch(B, f->gcfg.dims, f->gcfg.levels);
    void* scratch = f->det_sort.get(std::max<size_t>(bytes, 16));
    NFG_CUDA(nfg::launch_encode_bwd_det(f->shape, f->d_levels, X, B, dY, f->d_g, f->d_res->flags, scratch, bytes,
                                        c->stream));
    c->launches += 3 * size_t(f->gcfg.levels);
}

// Forward + loss + backward: gradients ACCUMULATE into the grad slab (the
// reference's mlp_backward / encode_backward semantics); no optimizer step.
struct Streamed {
    const unsigned int* ready = nullptr;
    unsigned int epoch = 0;
    int64_t chunk0 = 0, chunk = 0;
};

// Cross-rank reduction of the step scratch: loss sums (sum), the
// maybe-non-finite and abort flags (max), the first bad group + 1 (min) and the
// invalid-input flag (max), so every rank takes the same decision.
void reduce_scratch(nfg_field* f, cudaStream_t st)
{
    nfg_ctx* c = f->ctx;
    const NcclApi& n = nccl();
    NFG_NCCL(n.all_reduce(&f->d_res->loss_sum, &f->d_res->loss_sum, 1, ncclFloat64, ncclSum, c->comm, st));
    NFG_NCCL(n.all_reduce(f->d_res->flags, f->d_res->flags, 2, ncclUint32, ncclMax, c->comm, st));
    NFG_NCCL(n.all_reduce(f->d_res->flags + 2, f->d_res->flags + 2, 1, ncclUint32, ncclMin, c->comm, st));
    NFG_NCCL(n.all_reduce(f->d_res->flags + 3, f->d_res->flags + 3, 1, ncclUint32, ncclMax, c->comm, st));
}

void device_backward(nfg_field* f, const float* X, const float* target, int64_t B_local, int64_t B_global,
                     int loss_kind, const Streamed& sm = Streamed(), bool allow_speculative = true,
                     bool reduce_grads = true, float* store_dy = nullptr)
{
    require(loss_kind >= 0 && loss_kind <= 2, "train_step: unknown loss");
    require(B_local >= 0 && B_global >= B_local, "train_step: invalid batch size");
    nfg_ctx* c = f->ctx;
    if (!f->scratch_ready)
        reset_scratch(f);
    f->scratch_ready = false;
    // encode_forward's input checks (grid.hpp:226-229). With a clean gradient
    // slab the fused kernel checks its own inputs and Adam's check kernel
    // undoes the step on failure (re-zeroing); otherwise a separate k_validate
    // aborts every later kernel before any update.
    const bool fused = f->opts.fused_train && !f->opts.deterministic;
    const bool speculative = allow_speculative && f->grads_clean && fused;
    require(speculative || sm.ready == nullptr, "streamed inputs need the speculative fused path");
    if (!speculative) {
        NFG_CUDA(nfg::launch_validate(X, B_local * f->gcfg.dims, f->d_res->flags, c->stream));
        c->launches++;
    }
    const double count = double(B_global) * double(f->mcfg.output_width);
    f->last_batch = B_global;
    nfg::TrainArgs a{};
    a.X = X;
    a.target = target;
    a.B = B_local;
    a.loss_kind = loss_kind;
    a.inv_count = count > 0 ? float(1.0 / count) : 0.0f;
    a.table = table_ptr(f);
    a.W = f->d_p + f->n_tab_dev;
    a.b = f->d_p + f->n_tab_dev + f->n_w;
    a.table_grad = f->d_g;
    a.gW = f->d_g + f->n_tab_dev;
    a.gb = f->d_g + f->n_tab_dev + f->n_w;
    a.scratch = scratch_of(f);
    a.validate = speculative ? 1 : 0;
    a.ready = sm.ready;
    a.epoch = sm.epoch;
    a.chunk0 = sm.chunk0;
    a.chunk = sm.chunk;
    if (c->profile)
        c->prof_steps++;
    if (B_local > 0) {
        Span span(c, 0);
        if (fused && store_dy) {   // level-pipelined data parallelism: dY out, scattered per level group
            a.dY = store_dy;
            NFG_CUDA(nfg::launch_train(f->shape, f->d_levels, nfg::SRC_ENCODE, nfg::GRAD_LOSS, nfg::SINK_STORE, a,
                                       c->num_sms, c->stream, &f->train_grid));
            c->launches++;
        } else if (fused) {
            NFG_CUDA(nfg::launch_train(f->shape, f->d_levels, nfg::SRC_ENCODE, nfg::GRAD_LOSS, nfg::SINK_SCATTER, a,
                                       c->num_sms, c->stream, &f->train_grid));
            c->launches++;
        } else if (f->opts.deterministic) {
            const size_t LF = size_t(f->shape.in_real);
            float* Y = static_cast<float*>(c->s2.get(size_t(B_local) * LF * 4));
            float* dY = static_cast<float*>(c->s3.get(size_t(B_local) * LF * 4));
            NFG_CUDA(nfg::launch_encode_fwd_lv(f->shape, f->d_levels, X, B_local, table_ptr(f), Y, nullptr, nullptr,
                                               c->stream));
            a.Y = Y;
            a.dY = dY;
            det_prepare(f, a, B_local, true);
            int grid = 0;
            NFG_CUDA(nfg::launch_train(f->shape, nullptr, nfg::SRC_LOAD_Y, nfg::GRAD_LOSS, nfg::SINK_STORE, a,
                                       c->num_sms, c->stream, &grid));
            c->launches += 2;
            det_finish(f, a, grid);
            det_encode_bwd(f, X, B_local, dY);
        } else {
            const size_t LF = size_t(f->shape.in_real);
            float* Y = static_cast<float*>(c->s2.get(size_t(B_local) * LF * 4));
            float* dY = static_cast<float*>(c->s3.get(size_t(B_local) * LF * 4));
            NFG_CUDA(nfg::launch_encode_fwd_lv(f->shape, f->d_levels, X, B_local, table_ptr(f), Y, nullptr, nullptr,
                                               c->stream));
            a.Y = Y;
            a.dY = dY;
            NFG_CUDA(nfg::launch_train(f->shape, nullptr, nfg::SRC_LOAD_Y, nfg::GRAD_LOSS, nfg::SINK_STORE, a,
                                       c->num_sms, c->stream, nullptr));
            NFG_CUDA(nfg::launch_encode_bwd_lv(f->shape, f->d_levels, X, B_local, dY, f->d_g, c->stream,
                                               f->d_res->flags));
            c->launches += 3;
        }
    }
    if (c->comm && reduce_grads) {
        Span span(c, 2);
        // Data-parallel exchange: sum of the shards' (globally normalised)
        // gradients == the single-GPU gradient of the global batch; loss sums
        // and the flags travel with it.
        NFG_NCCL(nccl().all_reduce(f->d_g, f->d_g, f->n_total_dev, ncclFloat32, ncclSum, c->comm, c->stream));
        reduce_scratch(f, c->stream);
    }
}

// Early step result: once the loss sum and the flags are final on `st`, copy
// them to the host on the side stream (host_train_step may return before Adam).
void enqueue_early_result(nfg_field* f, cudaStream_t st)
{
    nfg_ctx* c = f->ctx;
    NFG_CUDA(cudaEventRecord(c->ev_res, st));
    NFG_CUDA(cudaStreamWaitEvent(c->res_stream, c->ev_res, 0));
    NFG_CUDA(cudaMemcpyAsync(f->h_res, f->d_res, sizeof(StepResult) + 4 * sizeof(unsigned int), cudaMemcpyDeviceToHost,
                             c->res_stream));
    NFG_CUDA(cudaEventRecord(c->ev_res_done, c->res_stream));
}

// Whether a data-parallel step takes the level-pipelined exchange (NFG_DP_LEVELS).
bool dp_levels(const nfg_field* f)
{
    return f->ctx->comm && f->opts.dp_exchange == NFG_DP_LEVELS && f->opts.fused_train &&
           !f->opts.deterministic && f->gcfg.features == 2 && f->shape.in_steps <= 2 && nfg::fused_supported(f->shape);
}

// Level groups of the level-pipelined exchange, finest first: contiguous level
// ranges [l0, l1) whose gradient slices reach ~4 MB (one NCCL call each,
// enough to run near bus bandwidth); the coarsest group also carries the MLP
// parameters. At config 2 (11 hashed levels of 4 MB) this is 8 groups.
struct LevelGroup {
    int l0, l1;
    uint64_t lo, hi;   // slab range
};
std::vector<LevelGroup> level_groups(const nfg_field* f, int max_groups)
{
    const int L = f->gcfg.levels, F = f->gcfg.features;
    auto start = [&](int l) { return l >= L ? f->n_tab_dev : f->dev_row_off[size_t(l)] * uint64_t(F); };
    std::vector<LevelGroup> g;
    int l1 = L;
    while (l1 > 0) {
        int l0 = l1 - 1;
        while (l0 > 0 && (start(l1) - start(l0)) * 4 < (uint64_t(4) << 20))
            --l0;
        g.push_back({ l0, l1, start(l0), start(l1) });
        l1 = l0;
    }
    // merge the coarsest groups until the count fits the event slots
    while (int(g.size()) > max_groups) {
        LevelGroup& a = g[g.size() - 2];
        const LevelGroup b = g.back();
        a.l0 = b.l0;
        a.lo = b.lo;
        g.pop_back();
    }
    return g;   // g.back() is the coarsest group, l0 = 0, lo = 0
}

template <class AfterBackward>
void device_train_step(nfg_field* f, const float* X, const float* target, int64_t B_local, int64_t B_global,
                       int loss_kind, int64_t step, const Streamed& sm, AfterBackward&& after_backward)
{
    nfg_ctx* c = f->ctx;
    const bool dp = c->comm != nullptr;
    if (dp && dp_levels(f)) {
        // Level-pipelined exchange: the fused kernel stores dY (no table
        // scatter); the loss / flags scratch is reduced at once; then each level
        // group, finest first, is scattered on the main stream and all-reduced
        // on the comm stream as soon as its scatter is done, and Adam updates
        // each reduced group while later groups are still scattering / reducing.
        // Only the coarsest (smallest) group's reduction follows the last scatter.
        const size_t LF = size_t(f->shape.in_real);
        float* dY = static_cast<float*>(c->s3.get(size_t(std::max<int64_t>(B_local, 1)) * LF * 4));
        device_backward(f, X, target, B_local, B_global, loss_kind, sm, true, /*reduce_grads=*/false, dY);
        after_backward();
        const float lr_now = float(nfg::host::lr_at(f->milestones, f->factor, f->hyper.lr, step));
        Span span(c, 2);
        NFG_CUDA(cudaEventRecord(c->ev_grads, c->stream));
        NFG_CUDA(cudaStreamWaitEvent(c->comm_stream, c->ev_grads, 0));
        reduce_scratch(f, c->comm_stream);
        NFG_CUDA(cudaEventRecord(c->ev_scr, c->comm_stream));
        const int ng_max = int(sizeof(c->ev_scat) / sizeof(c->ev_scat[0]));
        const std::vector<LevelGroup> groups = level_groups(f, ng_max);
        for (size_t k = 0; k < groups.size(); ++k) {
            const LevelGroup& gk = groups[k];
            const bool last = k + 1 == groups.size();
            NFG_CUDA(nfg::launch_encode_bwd_lv(f->shape, f->d_levels, X, B_local, dY, f->d_g, c->stream,
                                               f->d_res->flags, gk.l0, gk.l1));
            c->launches++;
            NFG_CUDA(cudaEventRecord(c->ev_scat[k], c->stream));
            NFG_CUDA(cudaStreamWaitEvent(c->comm_stream, c->ev_scat[k], 0));
            NFG_NCCL(nccl().all_reduce(f->d_g + gk.lo, f->d_g + gk.lo, gk.hi - gk.lo, ncclFloat32, ncclSum, c->comm,
                                       c->comm_stream));
            if (last)   // the MLP W, b (final since the fused kernel) travel with the coarsest group
                NFG_NCCL(nccl().all_reduce(f->d_g + f->n_tab_dev, f->d_g + f->n_tab_dev, f->n_total_dev - f->n_tab_dev,
                                           ncclFloat32, ncclSum, c->comm, c->comm_stream));
            NFG_CUDA(cudaEventRecord(c->ev_red[k], c->comm_stream));
        }
        nfg::AdamArgs a = adam_args(f, lr_now);
        NFG_CUDA(cudaStreamWaitEvent(c->stream, c->ev_scr, 0));
        if (f->early_result)   // after the reduced scratch AND the last scatter (it reads the staged inputs)
            enqueue_early_result(f, c->stream);
        for (size_t k = 0; k < groups.size(); ++k) {
            const bool last = k + 1 == groups.size();
            NFG_CUDA(cudaStreamWaitEvent(c->stream, c->ev_red[k], 0));
            a.lo = groups[k].lo;
            a.hi = groups[k].hi;
            NFG_CUDA(nfg::launch_adam_range(a, c->num_sms, c->stream));
            if (last) {   // the MLP parameters
                a.lo = f->n_tab_dev;
                a.hi = f->n_total_dev;
                NFG_CUDA(nfg::launch_adam_range(a, c->num_sms, c->stream));
                c->launches++;
            }
            c->launches++;
        }
        NFG_CUDA(nfg::launch_adam_fallback(a, c->num_sms, c->stream));
        c->launches += 2;
        f->step += 1;
        return;
    }
    device_backward(f, X, target, B_local, B_global, loss_kind, sm, true, /*reduce_grads=*/!dp);
    after_backward();   // streamed steps: enqueue the batch copies before the optimizer launches
    const float lr_now = float(nfg::host::lr_at(f->milestones, f->factor, f->hyper.lr, step));
    // the loss sum and the producers' flags are final here (after the
    // cross-rank scratch reduction with a communicator): read them back on a
    // side stream while Adam runs (host_train_step returns without waiting for
    // Adam when no flag is set: Adam then cannot abort)
    if (!dp && f->early_result)
        enqueue_early_result(f, c->stream);
    if (!dp) {
        Span span(c, 1);
        run_adam(f, lr_now, false);
        return;
    }
    // Data parallel: the gradient slab is all-reduced in chunks on the comm
    // stream while Adam updates every chunk as soon as it is reduced (comm and
    // the HBM-bound Adam overlap). The scratch (loss, flags) is reduced first,
    // so a possibly non-finite gradient anywhere (flags[0]) makes every chunk
    // kernel stand down and the checked full pass run instead: the reference's
    // "throw before any update" (adam.hpp:86-90) holds across ranks.
    Span span(c, 2);
    reduce_scratch(f, c->stream);
    if (f->early_result)
        enqueue_early_result(f, c->stream);
    nfg::AdamArgs a = adam_args(f, lr_now);
    NFG_CUDA(cudaEventRecord(c->ev_grads, c->stream));
    NFG_CUDA(cudaStreamWaitEvent(c->comm_stream, c->ev_grads, 0));
    const uint64_t n = f->n_total_dev;
    const uint64_t kmax = sizeof(c->ev_chunk) / sizeof(c->ev_chunk[0]);
    const uint64_t nk = std::max<uint64_t>(1, std::min<uint64_t>(kmax, (n + (uint64_t(1) << 20) - 1) >> 20));
    const uint64_t chunk = ((n + nk - 1) / nk + 63) & ~uint64_t(63);   // 4 MB+ pieces, 256-byte aligned
    for (uint64_t k = 0; k < nk; ++k) {
        const uint64_t lo = k * chunk, hi = std::min(n, lo + chunk);
        if (lo >= hi)
            break;
        NFG_NCCL(nccl().all_reduce(f->d_g + lo, f->d_g + lo, hi - lo, ncclFloat32, ncclSum, c->comm, c->comm_stream));
        NFG_CUDA(cudaEventRecord(c->ev_chunk[k], c->comm_stream));
        NFG_CUDA(cudaStreamWaitEvent(c->stream, c->ev_chunk[k], 0));
        a.lo = lo;
        a.hi = hi;
        NFG_CUDA(nfg::launch_adam_range(a, c->num_sms, c->stream));
        c->launches++;
    }
    NFG_CUDA(nfg::launch_adam_fallback(a, c->num_sms, c->stream));
    c->launches += 2;
    f->step += 1;
}

void device_train_step(nfg_field* f, const float* X, const float* target, int64_t B_local, int64_t B_global,
                       int loss_kind, int64_t step, const Streamed& sm = Streamed())
{
    device_train_step(f, X, target, B_local, B_global, loss_kind, step, sm, [] {});
}

nfg::FieldShape make_shape(const nfg_grid_config& g, const nfg_mlp_config& m, const std::vector<nfg_level_spec>& lv, const std::vector<uint64_t>& dev_off,
                           const nfg_options& o)
{
    nfg::FieldShape s{};
    s.grid.L = g.levels;
    s.grid.F = g.features;
    s.grid.d = g.dims;
    s.grid.smooth = g.interpolation == NFG_INTERP_SMOOTHSTEP;
    s.grid.mask = g.table_size - 1u;
    s.in_real = g.levels * g.features;
    s.in_steps = (s.in_real + 15) / 16;
    s.hidden_layers = m.hidden_layers;
    s.hidden_width = m.hidden_width;
    s.n_out = m.output_width;
    s.sigmoid = m.output_activation == NFG_ACT_SIGMOID;
    s.table_fp32 = o.table_fp32;
    s.mlp_engine = o.mlp_engine;
    for (size_t l = 0; l < lv.size() && l < NFG_MAX_LEVELS; ++l) {
        nfg::LevelDev& d = s.grid.lv[l];
        d.res = lv[l].resolution;
        d.res_f = float(lv[l].resolution);
        d.stride = lv[l].resolution + 1u;
        d.dense = uint32_t(lv[l].dense);
        d.row_off = uint32_t(dev_off[l]);
        d.len = lv[l].table_len;
    }
    return s;
}

// Copies a reference-layout range [off, off + n) of one flat buffer between the
// host and the device layout (levels padded to 8-row multiples; see nfg_field_create).
void copy_ref(nfg_field* f, float* dev, uint64_t off, uint64_t n, float* host, cudaMemcpyKind kind)
{
    const uint64_t F = uint64_t(f->gcfg.features), end = off + n;
    auto seg = [&](uint64_t ref_lo, uint64_t ref_hi, uint64_t dev_lo) {
        const uint64_t a = std::max(ref_lo, off), b = std::min(ref_hi, end);
        if (a >= b)
            return;
        float* d = dev + dev_lo + (a - ref_lo);
        float* h = host + (a - off);
        if (kind == cudaMemcpyHostToDevice)
            NFG_CUDA(cudaMemcpyAsync(d, h, (b - a) * 4, kind, f->ctx->stream));
        else
            NFG_CUDA(cudaMemcpyAsync(h, d, (b - a) * 4, kind, f->ctx->stream));
    };
    for (size_t l = 0; l < f->levels.size(); ++l) {
        const uint64_t lo = f->levels[l].row_offset * F;
        seg(lo, lo + uint64_t(f->levels[l].table_len) * F, f->dev_row_off[l] * F);
    }
    seg(f->n_tab, f->n_total, f->n_tab_dev);
}

// encode_forward's input validation (grid.hpp:226-229) for host-pointer calls;
// runs before anything touches device state, as in the reference.
void validate_inputs(const float* X, int64_t B, int d)
{
    const int64_t n = B * d;
    bool nonfinite = false, outside = false;
    const float lo = -1e-6f, hi = 1.0f + 1e-6f;
    for (int64_t i = 0; i < n; ++i) {
        const float v = X[i];
        nonfinite |= !std::isfinite(v);
        outside |= (v < lo) || (v > hi);
    }
    if (nonfinite)
        throw std::invalid_argument("encode_forward: non-finite input");
    if (outside)
        throw std::invalid_argument("encode_forward: input outside [0,1]^d");
}

float* buffer_of(nfg_field* f, int which)
{
    switch (which) {
    case NFG_BUF_PARAMS: return f->d_p;
    case NFG_BUF_GRADS: return f->d_g;
    case NFG_BUF_ADAM_M: return f->d_m;
    case NFG_BUF_ADAM_V: return f->d_v;
    }
    throw std::invalid_argument("unknown buffer");
}

}   // namespace

extern "C" {

const char* nfg_last_error(void) { return g_err.c_str(); }
const char* nfg_last_kernel_variant(int32_t which) { return nfg::g_variant[which & 1].c_str(); }
int nfg_abi_version(void) { return NFG_ABI_VERSION; }

nfg_status nfg_ctx_create(int device, nfg_ctx** out)
{
    return guard([&] {
        require(out != nullptr, "nfg_ctx_create: null out");
        auto* c = new nfg_ctx;
        try {
            c->device = device;
            NFG_CUDA(cudaSetDevice(device));
            NFG_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
            NFG_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
            NFG_CUDA(cudaEventCreateWithFlags(&c->ev_order, cudaEventDisableTiming));
            NFG_CUDA(cudaStreamCreateWithFlags(&c->res_stream, cudaStreamNonBlocking));
            NFG_CUDA(cudaEventCreateWithFlags(&c->ev_res, cudaEventDisableTiming));
            NFG_CUDA(cudaEventCreateWithFlags(&c->ev_res_done, cudaEventDisableTiming));
            void* fn = nullptr;
            cudaDriverEntryPointQueryResult q;
            if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &fn, cudaEnableDefault, &q) == cudaSuccess &&
                q == cudaDriverEntryPointSuccess && fn) {
                c->write_value32 = reinterpret_cast<decltype(c->write_value32)>(fn);
                unsigned int* probe = nullptr;   // stream memory ops usable on this device?
                NFG_CUDA(cudaMalloc(&probe, 4));
                if (c->write_value32(c->copy_stream, CUdeviceptr(probe), 1u, 0) != CUDA_SUCCESS ||
                    cudaStreamSynchronize(c->copy_stream) != cudaSuccess)
                    c->write_value32 = nullptr;
                cudaFree(probe);
            }
            NFG_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
}

nfg_status nfg_ctx_destroy(nfg_ctx* c)
{
    return guard([&] {
        if (!c)
            return;
        if (c->stream)
            cudaStreamSynchronize(c->stream);   // an early-returned step's Adam may still run
        if (c->comm)
            nccl().comm_destroy(c->comm);
        for (auto& r : c->recs) {
            cudaEventDestroy(r.a);
            cudaEventDestroy(r.b);
        }
        for (auto e : c->ev_pool)
            cudaEventDestroy(e);
        if (c->stream)
            cudaStreamDestroy(c->stream);
        if (c->copy_stream)
            cudaStreamDestroy(c->copy_stream);
        delete c->copy_pool;
        if (c->ev_order)
            cudaEventDestroy(c->ev_order);
        if (c->comm_stream)
            cudaStreamDestroy(c->comm_stream);
        if (c->ev_grads)
            cudaEventDestroy(c->ev_grads);
        for (auto e : c->ev_chunk)
            if (e)
                cudaEventDestroy(e);
        for (auto e : c->ev_scat)
            if (e)
                cudaEventDestroy(e);
        for (auto e : c->ev_red)
            if (e)
                cudaEventDestroy(e);
        for (cudaEvent_t e : { c->ev_scr, c->ev_res, c->ev_res_done })
            if (e)
                cudaEventDestroy(e);
        if (c->res_stream)
            cudaStreamDestroy(c->res_stream);
        delete c;
    });
}

nfg_status nfg_ctx_synchronize(nfg_ctx* c)
{
    return guard([&] { NFG_CUDA(cudaStreamSynchronize(c->stream)); });
}

void* nfg_ctx_stream(nfg_ctx* c) { return c ? c->stream : nullptr; }
uint64_t nfg_ctx_launch_count(nfg_ctx* c) { return c ? c->launches : 0; }

nfg_status nfg_ctx_set_profiling(nfg_ctx* c, int on)
{
    return guard([&] { c->profile = on != 0; });
}

nfg_status nfg_ctx_read_profile(nfg_ctx* c, double ms[4], int64_t* steps)
{
    return guard([&] {
        NFG_CUDA(cudaStreamSynchronize(c->stream));
        for (int i = 0; i < 4; ++i)
            ms[i] = 0.0;
        for (const auto& r : c->recs) {
            float t = 0.0f;
            NFG_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
            ms[r.kind] += t;
            c->ev_pool.push_back(r.a);
            c->ev_pool.push_back(r.b);
        }
        c->recs.clear();
        *steps = c->prof_steps;
        c->prof_steps = 0;
    });
}

nfg_status nfg_comm_unique_id(uint8_t id[128])
{
    return guard([&] {
        ncclUniqueId u;
        NFG_NCCL(nccl().get_unique_id(&u));
        static_assert(sizeof(u) == 128, "ncclUniqueId size");
        std::memcpy(id, &u, 128);
    });
}

nfg_status nfg_ctx_attach_comm(nfg_ctx* c, const uint8_t id[128], int rank, int nranks)
{
    return guard([&] {
        require(nranks >= 1 && rank >= 0 && rank < nranks, "attach_comm: bad rank");
        ncclUniqueId u;
        std::memcpy(&u, id, 128);
        NFG_CUDA(cudaSetDevice(c->device));
        NFG_NCCL(nccl().comm_init_rank(&c->comm, nranks, u, rank));
        c->rank = rank;
        c->nranks = nranks;
        if (!c->comm_stream) {
            NFG_CUDA(cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
            NFG_CUDA(cudaEventCreateWithFlags(&c->ev_grads, cudaEventDisableTiming));
            for (auto& e : c->ev_chunk)
                NFG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            for (auto& e : c->ev_scat)
                NFG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            for (auto& e : c->ev_red)
                NFG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            NFG_CUDA(cudaEventCreateWithFlags(&c->ev_scr, cudaEventDisableTiming));
        }
    });
}

nfg_status nfg_ctx_comm_info(nfg_ctx* c, int* rank, int* nranks)
{
    return guard([&] {
        int r = 0, n = 1;
        if (c->comm) {   // ask NCCL itself, not the values attach_comm was given
            const NcclApi& api = nccl();
            require(api.comm_count && api.comm_user_rank, "comm_info: NCCL lacks ncclCommCount/ncclCommUserRank");
            NFG_NCCL(api.comm_count(c->comm, &n));
            NFG_NCCL(api.comm_user_rank(c->comm, &r));
        }
        if (rank)
            *rank = r;
        if (nranks)
            *nranks = n;
    });
}

int32_t nfg_level_resolutions(const nfg_grid_config* cfg, nfg_level_spec* out, int32_t cap)
{
    int32_t n = -1;
    const nfg_status st = guard([&] {
        const auto lv = nfg::host::level_resolutions(*cfg);
        for (size_t i = 0; i < lv.size() && int32_t(i) < cap; ++i)
            out[i] = lv[i];
        n = int32_t(lv.size());
    });
    return st == NFG_OK ? n : -1;
}

double nfg_growth_factor(const nfg_grid_config* cfg) { return nfg::host::growth_factor(*cfg); }

uint32_t nfg_spatial_hash(const uint32_t* coords, int32_t dims, uint32_t table_size)
{
    return nfg::host::spatial_hash(coords, dims, table_size);
}

double nfg_lr_at(const int64_t* ms, int32_t n, double factor, double base, int64_t step)
{
    return nfg::host::lr_at(std::vector<int64_t>(ms, ms + n), factor, base, step);
}

nfg_status nfg_field_create(nfg_ctx* ctx, const nfg_grid_config* grid, const nfg_mlp_config* mlp,
                            const nfg_adam_hyper* hyper, const nfg_options* opts, nfg_field** out)
{
    return guard([&] {
        require(ctx && grid && mlp && out, "nfg_field_create: null argument");
        auto* f = new nfg_field;
        try {
            f->ctx = ctx;
            f->gcfg = *grid;
            f->mcfg = *mlp;
            f->mcfg.input_width = grid->levels * grid->features;   // model.cpp:101
            if (hyper)
                f->hyper = *hyper;
            if (opts)
                f->opts = *opts;
            nfg::host::validate(f->gcfg);
            nfg::host::validate(f->mcfg);
            nfg::host::validate(f->hyper);
            require(f->opts.mlp_engine >= NFG_MMA_DEFAULT && f->opts.mlp_engine <= NFG_MMA_TCGEN05,
                    "nfg_options.mlp_engine must be NFG_MMA_DEFAULT, NFG_MMA_SYNC or NFG_MMA_TCGEN05");
            require(f->opts.dp_exchange >= NFG_DP_DEFAULT && f->opts.dp_exchange <= NFG_DP_LEVELS,
                    "nfg_options.dp_exchange must be NFG_DP_DEFAULT, NFG_DP_ALLREDUCE or NFG_DP_LEVELS");
            if (f->mcfg.hidden_width > 64)
                throw Fail{ NFG_EUNSUPPORTED, "sm_100a MLP is built for hidden_width <= 64" };
            if (f->mcfg.hidden_layers < 1 || f->mcfg.hidden_layers > 3)
                throw Fail{ NFG_EUNSUPPORTED, "sm_100a MLP is built for 1..3 hidden layers" };
            if (f->mcfg.output_width > 16)
                throw Fail{ NFG_EUNSUPPORTED, "sm_100a MLP is built for output_width <= 16" };
            if (f->gcfg.levels > NFG_MAX_LEVELS || f->mcfg.input_width > 64)
                throw Fail{ NFG_EUNSUPPORTED, "sm_100a encoding is built for levels <= 32 and levels*features <= 64" };
            if (f->gcfg.features != 1 && f->gcfg.features != 2 && f->gcfg.features != 4 && f->gcfg.features != 8)
                throw Fail{ NFG_EUNSUPPORTED, "sm_100a encoding is built for features in {1, 2, 4, 8}" };
            f->levels = nfg::host::level_resolutions(f->gcfg);
            const uint64_t rows = f->levels.back().row_offset + f->levels.back().table_len;
            if (rows >= (uint64_t(1) << 32))
                throw Fail{ NFG_EUNSUPPORTED, "table rows exceed 2^32" };
            f->n_tab = rows * uint64_t(f->gcfg.features);
            uint64_t nw = 0, nb = 0;
            int in = f->mcfg.input_width;
            for (int k = 0; k <= f->mcfg.hidden_layers; ++k) {
                const int o = k < f->mcfg.hidden_layers ? f->mcfg.hidden_width : f->mcfg.output_width;
                nw += uint64_t(in) * uint64_t(o);
                nb += uint64_t(o);
                in = o;
            }
            f->n_w = nw;
            f->n_b = nb;
            f->n_total = f->n_tab + nw + nb;
            // Device layout: every level starts on a multiple of 8 rows, so
            // the relative row blocks of a level are the absolute 32-byte
            // sectors of the fp16 tables (8 rows) and of the fp32 gradients (4
            // rows): the lane-pair gathers / reductions merge x-adjacent
            // corners per sector, and aligned pairs {2k, 2k+1} take one
            // 16-byte vector reduction. Padding rows carry zero gradients,
            // which the skip-zero Adam group never touches.
            uint64_t drow = 0;
            f->dev_row_off.clear();
            for (const auto& s : f->levels) {
                f->dev_row_off.push_back(drow);
                drow += (uint64_t(s.table_len) + 7u) & ~uint64_t(7);
            }
            f->n_tab_dev = drow * uint64_t(f->gcfg.features);
            f->n_total_dev = f->n_tab_dev + nw + nb;
            f->n_alloc = (f->n_total_dev + 63) & ~uint64_t(63);
            f->shape = make_shape(f->gcfg, f->mcfg, f->levels, f->dev_row_off, f->opts);
            // shapes without a fused instantiation run the staged kernels
            // (encode -> MLP -> encode backward as separate launches)
            if (!nfg::staged_supported(f->shape))
                throw Fail{ NFG_EUNSUPPORTED, "sm_100a MLP kernels are not built for this input width / depth" };
            f->fused_ok = nfg::fused_supported(f->shape);
            if (!f->fused_ok)
                f->opts.fused_train = 0;
            NFG_CUDA(cudaSetDevice(ctx->device));
            const size_t bytes = f->n_alloc * sizeof(float);
            NFG_CUDA(cudaMalloc(&f->d_p, bytes));
            NFG_CUDA(cudaMalloc(&f->d_g, bytes));
            NFG_CUDA(cudaMalloc(&f->d_m, bytes));
            NFG_CUDA(cudaMalloc(&f->d_v, bytes));
            NFG_CUDA(cudaMalloc(&f->d_shadow, std::max<uint64_t>(f->n_tab_dev, 1) * sizeof(__half)));
            NFG_CUDA(cudaMalloc(&f->d_levels, sizeof(nfg::LevelDev) * NFG_MAX_LEVELS));
            NFG_CUDA(cudaMalloc(&f->d_res, sizeof(StepResult) + 4 * sizeof(unsigned int)));
            f->d_sticky = reinterpret_cast<unsigned int*>(f->d_res + 1);
            NFG_CUDA(cudaMemset(f->d_sticky, 0, 4 * sizeof(unsigned int)));
            NFG_CUDA(cudaMalloc(&f->d_ready, NFG_MAX_CHUNKS * sizeof(unsigned int)));
            NFG_CUDA(cudaMemset(f->d_ready, 0, NFG_MAX_CHUNKS * sizeof(unsigned int)));
            NFG_CUDA(cudaMallocHost(&f->h_res, sizeof(StepResult) + 4 * sizeof(unsigned int)));
            NFG_CUDA(cudaMemcpy(f->d_levels, f->shape.grid.lv, sizeof(nfg::LevelDev) * NFG_MAX_LEVELS,
                                cudaMemcpyHostToDevice));
            for (float* p : { f->d_p, f->d_g, f->d_m, f->d_v })
                NFG_CUDA(cudaMemsetAsync(p, 0, bytes, ctx->stream));
            NFG_CUDA(cudaMemsetAsync(f->d_shadow, 0, std::max<uint64_t>(f->n_tab_dev, 1) * sizeof(__half), ctx->stream));
            reset_scratch(f);   // a check before the first step must read a clean status
            std::memset(f->h_res, 0, sizeof(StepResult) + 4 * sizeof(unsigned int));
            NFG_CUDA(cudaStreamSynchronize(ctx->stream));
        } catch (...) {
            nfg_field_destroy(f);
            throw;
        }
        *out = f;
    });
}

nfg_status nfg_field_destroy(nfg_field* f)
{
    return guard([&] {
        if (!f)
            return;
        // a host-pointer train_step may return while its Adam still runs
        if (f->ctx && f->ctx->stream)
            cudaStreamSynchronize(f->ctx->stream);
        for (void* p : { (void*)f->d_p, (void*)f->d_g, (void*)f->d_m, (void*)f->d_v, (void*)f->d_shadow,
                         (void*)f->d_levels, (void*)f->d_res, (void*)f->d_ready })
            if (p)
                cudaFree(p);
        if (f->h_res)
            cudaFreeHost(f->h_res);
        delete f;
    });
}

nfg_status nfg_field_init(nfg_field* f, uint64_t seed)
{
    return guard([&] {
        std::vector<float> host(f->n_total);
        nfg::host::init_tables(seed, host.data(), f->n_tab);                         // grid.hpp:158-164
        nfg::host::glorot(f->mcfg, seed + 1, host.data() + f->n_tab, host.data() + f->n_tab + f->n_w);   // model.cpp:34
        cudaStream_t st = f->ctx->stream;
        for (float* p : { f->d_p, f->d_g, f->d_m, f->d_v })
            NFG_CUDA(cudaMemsetAsync(p, 0, f->n_alloc * 4, st));
        copy_ref(f, f->d_p, 0, f->n_total, host.data(), cudaMemcpyHostToDevice);
        refresh_shadow(f);
        NFG_CUDA(cudaStreamSynchronize(st));
        f->step = 0;
        f->grads_clean = true;
    });
}

nfg_status nfg_field_set_hyper(nfg_field* f, const nfg_adam_hyper* h)
{
    return guard([&] {
        nfg::host::validate(*h);
        f->hyper = *h;
    });
}

nfg_status nfg_field_set_schedule(nfg_field* f, const int64_t* ms, int32_t n, double factor)
{
    return guard([&] {
        // LrSchedule::validate (adam.hpp:129-136)
        require(factor > 0 && factor <= 1, "LrSchedule: factor must be in (0, 1]");
        for (int32_t i = 1; i < n; ++i)
            require(ms[i] > ms[i - 1], "LrSchedule: milestones must be strictly increasing");
        f->milestones.assign(ms, ms + n);
        f->factor = factor;
    });
}

nfg_status nfg_field_sizes(const nfg_field* f, uint64_t out[3])
{
    return guard([&] {
        out[0] = f->n_tab;
        out[1] = f->n_w;
        out[2] = f->n_b;
    });
}

nfg_status nfg_field_levels(const nfg_field* f, nfg_level_spec* out, int32_t cap)
{
    return guard([&] {
        for (size_t i = 0; i < f->levels.size() && int32_t(i) < cap; ++i)
            out[i] = f->levels[i];
    });
}

nfg_status nfg_field_read(nfg_field* f, int32_t which, uint64_t off, uint64_t n, float* host)
{
    return guard([&] {
        require(off + n <= f->n_total, "nfg_field_read: range out of bounds");
        copy_ref(f, buffer_of(f, which), off, n, host, cudaMemcpyDeviceToHost);
        NFG_CUDA(cudaStreamSynchronize(f->ctx->stream));
    });
}

nfg_status nfg_field_write(nfg_field* f, int32_t which, uint64_t off, uint64_t n, const float* host)
{
    return guard([&] {
        require(off + n <= f->n_total, "nfg_field_write: range out of bounds");
        copy_ref(f, buffer_of(f, which), off, n, const_cast<float*>(host), cudaMemcpyHostToDevice);
        if (which == NFG_BUF_GRADS)
            f->grads_clean = false;
        if (which == NFG_BUF_PARAMS && off < f->n_tab)
            refresh_shadow(f);
        NFG_CUDA(cudaStreamSynchronize(f->ctx->stream));
    });
}

nfg_status nfg_field_device_buffer(nfg_field* f, int32_t which, float** dev, uint64_t* count)
{
    return guard([&] {
        *dev = buffer_of(f, which);
        *count = f->n_total_dev;   // device layout (levels start on 8-row multiples)
    });
}

nfg_status nfg_field_context(const nfg_field* f, nfg_ctx** ctx)
{
    return guard([&] { *ctx = f->ctx; });
}

nfg_status nfg_field_get_config(const nfg_field* f, nfg_grid_config* grid, nfg_mlp_config* mlp)
{
    return guard([&] {
        if (grid)
            *grid = f->gcfg;
        if (mlp)
            *mlp = f->mcfg;
    });
}

nfg_status nfg_field_get_step(const nfg_field* f, uint64_t* step)
{
    return guard([&] { *step = f->step; });
}

nfg_status nfg_field_set_step(nfg_field* f, uint64_t step)
{
    return guard([&] { f->step = step; });
}

nfg_status nfg_field_broadcast(nfg_field* f, int root)
{
    return guard([&] {
        nfg_ctx* c = f->ctx;
        if (!c->comm)
            return;   // one rank: nothing to agree on
        require(root >= 0 && root < c->nranks, "nfg_field_broadcast: bad root");
        if (f->pending_steps)
            settle_pending(f);
        const NcclApi& n = nccl();
        require(n.broadcast != nullptr, "nfg_field_broadcast: NCCL lacks ncclBroadcast");
        // params, Adam m and v in the device layout, then the step counter:
        // data-parallel ranks apply the same replicated Adam step, so they must
        // start from bit-identical state
        for (float* b : { f->d_p, f->d_m, f->d_v })
            NFG_NCCL(n.broadcast(b, b, f->n_total_dev, ncclFloat32, root, c->comm, c->stream));
        uint64_t* d_step = static_cast<uint64_t*>(c->s3.get(sizeof(uint64_t)));
        NFG_CUDA(cudaMemcpyAsync(d_step, &f->step, sizeof(uint64_t), cudaMemcpyHostToDevice, c->stream));
        NFG_NCCL(n.broadcast(d_step, d_step, 1, ncclUint64, root, c->comm, c->stream));
        uint64_t s = 0;
        NFG_CUDA(cudaMemcpyAsync(&s, d_step, sizeof(uint64_t), cudaMemcpyDeviceToHost, c->stream));
        refresh_shadow(f);
        NFG_CUDA(cudaStreamSynchronize(c->stream));
        f->step = s;
    });
}

// The reference's synchronous train_step on host pointers (model.cpp:111-138).
static void host_train_step(nfg_field* f, const float* X, const float* target, int64_t B, int64_t B_global,
                     int32_t loss_kind, int64_t step, float* loss)
{
    nfg_ctx* c = f->ctx;
    if (f->pending_steps)
        settle_pending(f);   // a deferred abort of earlier asynchronous steps surfaces here
    require(B >= 0 && B_global >= B, "train_step: B_global must cover the local batch");
    const int d = f->gcfg.dims, no = f->mcfg.output_width;
    const uint64_t before = f->step;
    const bool was_clean = f->grads_clean;
    const bool staging_idle = c->staging_idle;
    c->staging_idle = false;
    f->early_result = true;   // read the result while Adam (and a data-parallel exchange) runs
    struct EarlyReset {       // no other entry point may see it set (an exception leaves through here)
        nfg_field* f;
        ~EarlyReset() { f->early_result = false; }
    } early_reset{ f };
    const bool can_stream = f->stream_warm && f->grads_clean && f->opts.fused_train && !f->opts.deterministic &&
                            c->write_value32 && B >= (int64_t(1) << 15) && !launches_serialized();
    const bool pinned = can_stream && is_pinned(X) && is_pinned(target);
    if (can_stream) {
        // Overlap the H2D of the batch with the step: the fused kernel is
        // launched first and waits per tile for its chunk's ready flag,
        // which the copy stream writes (cuStreamWriteValue32) after each
        // chunk lands, while the host enqueues the copies. Not used when
        // launches may be serialised (a profiler or sanitizer injected,
        // CUDA_LAUNCH_BLOCKING=1): a kernel waiting on another stream can
        // then never finish, so those runs take the plain staged path.
        // Pageable sources (a caller's Eigen::MatrixXf or numpy array) are
        // first copied chunk by chunk into pinned bounce buffers by a few
        // host threads, so the copy engine and the kernel start on chunk 0
        // while the host still copies the rest.
        float* dX = static_cast<float*>(c->s0.get(size_t(B) * d * 4));
        float* dT = static_cast<float*>(c->s1.get(size_t(B) * no * 4));
        // a first chunk covering the persistent kernel's first wave of tiles
        // (its CTAs x 64 samples, known from the plain step that precedes
        // streaming; NFG_STREAM_CHUNK0 overrides), then NFG_STREAM_CHUNKS - 1
        // equal chunks
        static const int64_t chunk0_env = [] {
            const char* e = getenv("NFG_STREAM_CHUNK0");
            return e ? int64_t(atoll(e)) : int64_t(0);
        }();
        const int64_t wave = f->train_grid > 0 ? int64_t(f->train_grid) * nfg::train_warps_per_cta() * 16
                                               : int64_t(c->num_sms) * 128;
        const int64_t chunk0 = std::min<int64_t>(B, chunk0_env > 0 ? chunk0_env : wave);
        const int64_t chunk = std::max<int64_t>(4096, (B - chunk0 + NFG_STREAM_CHUNKS - 2) / (NFG_STREAM_CHUNKS - 1));
        const int64_t nchunks = 1 + (B - chunk0 + chunk - 1) / chunk;
        const float* srcX = X;
        const float* srcT = target;
        std::vector<std::vector<CopyPool::Part>> job;
        if (!pinned) {
            float* hX = static_cast<float*>(c->h0.get(size_t(B) * d * 4));
            float* hT = static_cast<float*>(c->h1.get(size_t(B) * no * 4));
            // helper threads next to the caller (NFG_COPY_THREADS; 0 = the caller
            // copies alone). Measured at config 2 on a 16-core host: pageable e2e
            // 5.5e8 (caller alone), 6.6 / 6.8 / 6.9 / 7.0e8 samples/s with 1 / 2 /
            // 3 / 5 helpers, pinned 7.15e8; the driver's own pageable staging 4.35e8.
            static const int workers = [] {
                const char* e = getenv("NFG_COPY_THREADS");
                const int hw = int(std::thread::hardware_concurrency());
                return e ? std::max(0, atoi(e)) : std::max(1, std::min(4, hw / 4));
            }();
            if (!c->copy_pool && workers > 0)
                c->copy_pool = new CopyPool(workers);
            job.resize(size_t(nchunks));
            for (int64_t k = 0; k < nchunks; ++k) {
                const int64_t s0 = k == 0 ? 0 : chunk0 + (k - 1) * chunk;
                const int64_t n = std::min(k == 0 ? chunk0 : chunk, B - s0);
                job[size_t(k)] = { { reinterpret_cast<const char*>(X + s0 * d), reinterpret_cast<char*>(hX + s0 * d),
                                     size_t(n) * d * 4 },
                                   { reinterpret_cast<const char*>(target + s0 * no),
                                     reinterpret_cast<char*>(hT + s0 * no), size_t(n) * no * 4 } };
            }
            // the previous step's DMA out of the bounce buffers finished:
            // host-pointer steps are synchronous
            if (c->copy_pool)
                c->copy_pool->start(job);
            srcX = hX;
            srcT = hT;
        }
        const unsigned int epoch = ++f->epoch;
        if (!staging_idle) {   // else the previous step's Adam may still run: the copies start under it
            NFG_CUDA(cudaEventRecord(c->ev_order, c->stream));   // staging buffers free
            NFG_CUDA(cudaStreamWaitEvent(c->copy_stream, c->ev_order, 0));
        }
        int64_t k = 0, caller_chunks = 0;
        auto enqueue_copies = [&] {
            for (; k < nchunks; ++k) {
                const int64_t s0 = k == 0 ? 0 : chunk0 + (k - 1) * chunk;
                const int64_t n = std::min(k == 0 ? chunk0 : chunk, B - s0);
                if (!pinned && c->copy_pool) {
                    c->copy_pool->finish_chunk(size_t(k));
                    caller_chunks = k + 1;
                } else if (!pinned)
                    for (const CopyPool::Part& p : job[size_t(k)])
                        std::memcpy(p.dst, p.src, p.bytes);
                NFG_CUDA(cudaMemcpyAsync(dX + s0 * d, srcX + s0 * d, size_t(n) * d * 4, cudaMemcpyHostToDevice,
                                         c->copy_stream));
                NFG_CUDA(cudaMemcpyAsync(dT + s0 * no, srcT + s0 * no, size_t(n) * no * 4,
                                         cudaMemcpyHostToDevice, c->copy_stream));
                if (c->write_value32(c->copy_stream, CUdeviceptr(f->d_ready + k), epoch, 0) != CUDA_SUCCESS)
                    throw Fail{ NFG_ECUDA, "cuStreamWriteValue32 failed" };
            }
        };
        const Streamed streamed{ f->d_ready, epoch, chunk0, chunk };
        // the copies are enqueued right after the fused kernel's launch,
        // ahead of the optimizer launches, so its first tiles wait less
        auto copies = [&] {
            try {
                enqueue_copies();
            } catch (...) {
                for (; k < nchunks; ++k)   // never leave the kernel waiting
                    c->write_value32(c->copy_stream, CUdeviceptr(f->d_ready + k), epoch, 0);
                throw;
            }
        };
        auto drain_pool = [&] {   // never return while workers still read the caller's arrays
            if (!pinned && c->copy_pool) {
                for (int64_t j = caller_chunks; j < nchunks; ++j)   // the caller's shares it never reached
                    c->copy_pool->copy_slice(size_t(j), 0);
                c->copy_pool->drain(size_t(nchunks));
            }
        };
        try {
            device_train_step(f, dX, dT, B, B_global, loss_kind, step, streamed, copies);
        } catch (...) {
            for (; k < nchunks; ++k)   // a failure before or after the copies: release every chunk
                c->write_value32(c->copy_stream, CUdeviceptr(f->d_ready + k), epoch, 0);
            drain_pool();
            throw;
        }
        drain_pool();
    } else {
        const float* dX = stage(c->s0, X, size_t(B) * d, c->stream);
        const float* dT = stage(c->s1, target, size_t(B) * no, c->stream);
        device_train_step(f, dX, dT, B, B_global, loss_kind, step);
    }
    bool settled = false;
    if (f->early_result) {
        f->early_result = false;
        NFG_CUDA(cudaEventSynchronize(c->ev_res_done));
        const unsigned int* fl = f->h_res->flags;
        // no producer flag and no abort: Adam cannot abort (its exact scan only
        // runs when a producer flagged a possibly non-finite gradient), so the
        // step's outcome is known and the host returns while Adam runs; every
        // later use of the field is stream-ordered after it
        settled = fl[0] == 0u && fl[1] == 0u && fl[3] == 0u && sticky_host(f)[0] == 0u;
    }
    if (!settled)
        fetch_result(f);
    // host-pointer calls are synchronous: every kernel that read this step's
    // staged inputs has finished (the fused kernel, or the whole step)
    c->staging_idle = true;
    reset_scratch(f);   // for the next step, off its critical path (h_res holds this one)
    f->scratch_ready = true;
    if (f->h_res->flags[1]) {
        f->step = before;   // the reference throws before incrementing (adam.hpp:86-92)
        // invalid input on a clean slab was undone by re-zeroing; a
        // non-finite gradient leaves the accumulated gradients in place
        f->grads_clean = was_clean && (f->h_res->flags[3] & 3u) != 0;
        raise_if_aborted(f);
    }
    f->grads_clean = true;   // Adam zeroed every gradient (adam.hpp:118-120)
    f->stream_warm = true;   // every kernel of the step is loaded now
    const double count = double(B_global) * no;
    if (loss)
        *loss = count > 0 ? float(f->h_res->loss_sum / count) : 0.0f;
}

nfg_status nfg_field_train_step(nfg_field* f, const float* X, const float* target, int64_t B, int32_t loss_kind,
                                int64_t step, float* loss)
{
    return guard([&] { host_train_step(f, X, target, B, B * f->ctx->nranks, loss_kind, step, loss); });
}

nfg_status nfg_field_train_step_global(nfg_field* f, const float* X, const float* target, int64_t B_local,
                                       int64_t B_global, int32_t loss_kind, int64_t step, float* loss)
{
    return guard([&] { host_train_step(f, X, target, B_local, B_global, loss_kind, step, loss); });
}

nfg_status nfg_field_gradients(nfg_field* f, const float* X, const float* target, int64_t B, int32_t loss_kind,
                               float* loss)
{
    return guard([&] {
        nfg_ctx* c = f->ctx;
        if (f->pending_steps)
            settle_pending(f);
        const float* dX = stage(c->s0, X, size_t(B) * f->gcfg.dims, c->stream);
        const float* dT = stage(c->s1, target, size_t(B) * f->mcfg.output_width, c->stream);
        device_backward(f, dX, dT, B, B * c->nranks, loss_kind, Streamed(), false);
        f->grads_clean = false;
        fetch_result(f);
        if (f->h_res->flags[3])
            raise_if_aborted(f);
        const double count = double(B) * c->nranks * f->mcfg.output_width;
        if (loss)
            *loss = count > 0 ? float(f->h_res->loss_sum / count) : 0.0f;
    });
}

nfg_status nfg_field_train_step_device(nfg_field* f, const float* X, const float* target, int64_t B_local,
                                       int64_t B_global, int32_t loss_kind, int64_t step, float* loss_dev)
{
    return guard([&] {
        device_train_step(f, X, target, B_local, B_global, loss_kind, step);
        f->pending_steps++;
        f->grads_clean = true;   // optimistic; nfg_field_check corrects it
        if (loss_dev) {
            NFG_CUDA(nfg::launch_loss_out(&f->d_res->loss_sum, f->d_res->flags,
                                          double(B_global) * f->mcfg.output_width, loss_dev, f->ctx->stream));
            f->ctx->launches++;
        }
    });
}

static_assert(sizeof(StepResult) == sizeof(nfg_step_record), "nfg_step_record mirrors the device scratch");

nfg_status nfg_field_step_record(nfg_field* f, nfg_step_record* rec_dev)
{
    return guard([&] {
        NFG_CUDA(cudaMemcpyAsync(rec_dev, f->d_res, sizeof(StepResult), cudaMemcpyDeviceToDevice, f->ctx->stream));
    });
}

nfg_status nfg_step_record_check(nfg_field* f, const nfg_step_record* rec, int64_t B_global, float* loss)
{
    return guard([&] {
        StepResult saved = *f->h_res;
        std::memcpy(f->h_res, rec, sizeof(StepResult));
        try {
            if (f->h_res->flags[1])
                raise_if_aborted(f);
        } catch (...) {
            *f->h_res = saved;
            throw;
        }
        *f->h_res = saved;
        const double count = double(B_global) * f->mcfg.output_width;
        if (loss)
            *loss = count > 0 ? float(rec->loss_sum / count) : 0.0f;
    });
}

nfg_status nfg_field_check(nfg_field* f)
{
    return guard([&] { settle_pending(f); });
}

nfg_status nfg_field_evaluate_device(nfg_field* f, const float* X, int64_t B, float* out)
{
    return guard([&] {
        nfg::InferArgs a{};
        a.X = X;
        a.B = B;
        a.table = table_ptr(f);
        a.W = f->d_p + f->n_tab_dev;
        a.b = f->d_p + f->n_tab_dev + f->n_w;
        a.out = out;
        Span span(f->ctx, 3);
        if (f->fused_ok) {
            NFG_CUDA(nfg::launch_infer(f->shape, f->d_levels, nfg::SRC_ENCODE, a, f->ctx->num_sms, f->ctx->stream));
            f->ctx->launches++;
        } else if (B > 0) {   // staged: encode into scratch, then the MLP
            float* Y = static_cast<float*>(f->comp_y.get(size_t(B) * size_t(f->shape.in_real) * 4));
            NFG_CUDA(nfg::launch_encode_fwd_lv(f->shape, f->d_levels, X, B, table_ptr(f), Y, nullptr, nullptr,
                                               f->ctx->stream));
            a.X = nullptr;
            a.Y = Y;
            NFG_CUDA(nfg::launch_infer(f->shape, nullptr, nfg::SRC_LOAD_Y, a, f->ctx->num_sms, f->ctx->stream));
            f->ctx->launches += 2;
        }
    });
}

nfg_status nfg_field_evaluate(nfg_field* f, const float* X, int64_t B, float* out)
{
    return guard([&] {
        nfg_ctx* c = f->ctx;
        validate_inputs(X, B, f->gcfg.dims);
        const float* dX = stage(c->s0, X, size_t(B) * f->gcfg.dims, c->stream);
        float* dO = static_cast<float*>(c->s1.get(std::max<size_t>(size_t(B) * f->mcfg.output_width * 4, 16)));
        const nfg_status st = nfg_field_evaluate_device(f, dX, B, dO);
        if (st != NFG_OK)
            throw Fail{ st, g_err };
        if (B > 0)
            NFG_CUDA(cudaMemcpyAsync(out, dO, size_t(B) * f->mcfg.output_width * 4, cudaMemcpyDeviceToHost, c->stream));
        NFG_CUDA(cudaStreamSynchronize(c->stream));
    });
}

nfg_status nfg_encode_forward(nfg_field* f, const float* X, int64_t B, float* Y, uint32_t* rows, float* weights)
{
    return guard([&] {
        nfg_ctx* c = f->ctx;
        const size_t LF = size_t(f->shape.in_real), nc = size_t(1) << f->gcfg.dims, L = size_t(f->gcfg.levels);
        validate_inputs(X, B, f->gcfg.dims);
        const float* dX = stage(c->s0, X, size_t(B) * f->gcfg.dims, c->stream);
        float* dY = static_cast<float*>(c->s1.get(std::max<size_t>(size_t(B) * LF * 4, 16)));
        uint32_t* dR = nullptr;
        float* dW = nullptr;
        if (rows && weights) {
            dR = static_cast<uint32_t*>(c->s2.get(std::max<size_t>(L * B * nc * 4, 16)));
            dW = static_cast<float*>(c->s3.get(std::max<size_t>(L * B * nc * 4, 16)));
        }
        NFG_CUDA(nfg::launch_encode_fwd_lv(f->shape, f->d_levels, dX, B, table_ptr(f), dY, dR, dW, c->stream));
        c->launches++;
        if (B > 0) {
            NFG_CUDA(cudaMemcpyAsync(Y, dY, size_t(B) * LF * 4, cudaMemcpyDeviceToHost, c->stream));
            if (dR) {
                NFG_CUDA(cudaMemcpyAsync(rows, dR, L * B * nc * 4, cudaMemcpyDeviceToHost, c->stream));
                NFG_CUDA(cudaMemcpyAsync(weights, dW, L * B * nc * 4, cudaMemcpyDeviceToHost, c->stream));
            }
        }
        NFG_CUDA(cudaStreamSynchronize(c->stream));
    });
}

nfg_status nfg_encode_backward(nfg_field* f, const float* X, int64_t B, const float* dY)
{
    return guard([&] {
        nfg_ctx* c = f->ctx;
        validate_inputs(X, B, f->gcfg.dims);
        const float* dX = stage(c->s0, X, size_t(B) * f->gcfg.dims, c->stream);
        const float* ddY = stage(c->s1, dY, size_t(B) * f->shape.in_real, c->stream);
        if (f->opts.deterministic) {
            reset_scratch(f);
            det_encode_bwd(f, dX, B, ddY);
        } else {
            NFG_CUDA(nfg::launch_encode_bwd_lv(f->shape, f->d_levels, dX, B, ddY, f->d_g, c->stream));
            c->launches++;
        }
        f->grads_clean = false;
        NFG_CUDA(cudaStreamSynchronize(c->stream));
    });
}

nfg_status nfg_mlp_forward(nfg_field* f, const float* Y, int64_t B, float* out)
{
    return guard([&] {
        nfg_ctx* c = f->ctx;
        const float* dY = stage(c->s0, Y, size_t(B) * f->shape.in_real, c->stream);
        float* dO = static_cast<float*>(c->s1.get(std::max<size_t>(size_t(B) * f->mcfg.output_width * 4, 16)));
        nfg::InferArgs a{};
        a.Y = dY;
        a.B = B;
        a.W = f->d_p + f->n_tab_dev;
        a.b = f->d_p + f->n_tab_dev + f->n_w;
        a.out = dO;
        NFG_CUDA(nfg::launch_infer(f->shape, nullptr, nfg::SRC_LOAD_Y, a, c->num_sms, c->stream));
        c->launches++;
        if (B > 0)
            NFG_CUDA(cudaMemcpyAsync(out, dO, size_t(B) * f->mcfg.output_width * 4, cudaMemcpyDeviceToHost, c->stream));
        NFG_CUDA(cudaStreamSynchronize(c->stream));
    });
}

nfg_status nfg_mlp_backward(nfg_field* f, const float* Y, int64_t B, const float* dOut, float* dY)
{
    return guard([&] {
        nfg_ctx* c = f->ctx;
        const float* dYin = stage(c->s0, Y, size_t(B) * f->shape.in_real, c->stream);
        const float* dO = stage(c->s1, dOut, size_t(B) * f->mcfg.output_width, c->stream);
        float* ddY = static_cast<float*>(c->s2.get(std::max<size_t>(size_t(B) * f->shape.in_real * 4, 16)));
        reset_scratch(f);
        nfg::TrainArgs a{};
        a.Y = dYin;
        a.dout = dO;
        a.B = B;
        a.inv_count = 1.0f;
        a.W = f->d_p + f->n_tab_dev;
        a.b = f->d_p + f->n_tab_dev + f->n_w;
        a.dY = ddY;
        a.gW = f->d_g + f->n_tab_dev;
        a.gb = f->d_g + f->n_tab_dev + f->n_w;
        a.scratch = scratch_of(f);
        if (f->opts.deterministic)
            det_prepare(f, a, B, false);
        int grid = 0;
        NFG_CUDA(nfg::launch_train(f->shape, nullptr, nfg::SRC_LOAD_Y, nfg::GRAD_DOUT, nfg::SINK_STORE, a, c->num_sms,
                                   c->stream, &grid));
        c->launches++;
        if (f->opts.deterministic)
            det_finish(f, a, grid);
        f->grads_clean = false;
        if (B > 0)
            NFG_CUDA(cudaMemcpyAsync(dY, ddY, size_t(B) * f->shape.in_real * 4, cudaMemcpyDeviceToHost, c->stream));
        NFG_CUDA(cudaStreamSynchronize(c->stream));
    });
}

nfg_status nfg_loss(nfg_ctx* c, int32_t kind, const float* pred, const float* target, int64_t n, int64_t count,
                    float* dpred, float* loss)
{
    return guard([&] {
        require(kind >= 0 && kind <= 2, "loss_with_grad: unknown loss");
        const float* dP = stage(c->s0, pred, size_t(n), c->stream);
        const float* dT = stage(c->s1, target, size_t(n), c->stream);
        float* dD = static_cast<float*>(c->s2.get(std::max<size_t>(size_t(n) * 4, 16)));
        if (!c->d_red)
            NFG_CUDA(cudaMalloc(&c->d_red, sizeof(double)));
        NFG_CUDA(cudaMemsetAsync(c->d_red, 0, sizeof(double), c->stream));
        NFG_CUDA(nfg::launch_loss(kind, dP, dT, n, float(count), dD, c->d_red, c->stream));
        c->launches++;
        double sum = 0;
        if (n > 0)
            NFG_CUDA(cudaMemcpyAsync(dpred, dD, size_t(n) * 4, cudaMemcpyDeviceToHost, c->stream));
        NFG_CUDA(cudaMemcpyAsync(&sum, c->d_red, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        NFG_CUDA(cudaStreamSynchronize(c->stream));
        *loss = float(sum / double(count));
    });
}

nfg_status nfg_adam_step(nfg_field* f, float lr_now)
{
    return guard([&] {
        if (f->pending_steps)
            settle_pending(f);
        reset_scratch(f);
        const uint64_t before = f->step;
        run_adam(f, lr_now, true);
        fetch_result(f);
        if (f->h_res->flags[1]) {
            f->step = before;
            raise_if_aborted(f);
        }
        f->grads_clean = true;
    });
}

// ---- device-pointer components (asynchronous on the context stream) --------
// Building blocks for pipelines that chain fields on the device (the NeRF
// density -> color networks, csrc/nerf.cu). Gradients ACCUMULATE into the
// field's slab like mlp_backward / encode_backward (mlp.hpp:147-148,
// grid.hpp:292); nfg_adam_step_device applies and zeroes them; deferred
// errors surface through nfg_field_check.
nfg_status nfg_field_backward_device(nfg_field* f, const float* X, int64_t B, const float* dOut)
{
    return guard([&] {
        nfg_ctx* c = f->ctx;
        if (B <= 0)
            return;
        reset_scratch(f);
        if (f->opts.fused_train && !f->opts.deterministic) {
            // one fused encode -> MLP -> backward -> scatter kernel when built
            nfg::TrainArgs a{};
            a.X = X;
            a.dout = dOut;
            a.B = B;
            a.inv_count = 1.0f;
            a.table = table_ptr(f);
            a.W = f->d_p + f->n_tab_dev;
            a.b = f->d_p + f->n_tab_dev + f->n_w;
            a.table_grad = f->d_g;
            a.gW = f->d_g + f->n_tab_dev;
            a.gb = f->d_g + f->n_tab_dev + f->n_w;
            a.scratch = scratch_of(f);
            const cudaError_t e = nfg::launch_train(f->shape, f->d_levels, nfg::SRC_ENCODE, nfg::GRAD_DOUT,
                                                    nfg::SINK_SCATTER, a, c->num_sms, c->stream, nullptr);
            if (e == cudaSuccess) {
                c->launches++;
                f->grads_clean = false;
                return;
            }
            if (e != cudaErrorNotSupported)
                NFG_CUDA(e);
            cudaGetLastError();
        }
        const size_t LF = size_t(f->shape.in_real);
        float* Y = static_cast<float*>(f->comp_y.get(size_t(B) * LF * 4));
        float* dY = static_cast<float*>(f->comp_dy.get(size_t(B) * LF * 4));
        NFG_CUDA(nfg::launch_encode_fwd_lv(f->shape, f->d_levels, X, B, table_ptr(f), Y, nullptr, nullptr, c->stream));
        nfg::TrainArgs a{};
        a.Y = Y;
        a.dout = dOut;
        a.B = B;
        a.inv_count = 1.0f;
        a.W = f->d_p + f->n_tab_dev;
        a.b = f->d_p + f->n_tab_dev + f->n_w;
        a.dY = dY;
        a.gW = f->d_g + f->n_tab_dev;
        a.gb = f->d_g + f->n_tab_dev + f->n_w;
        a.scratch = scratch_of(f);
        NFG_CUDA(nfg::launch_train(f->shape, nullptr, nfg::SRC_LOAD_Y, nfg::GRAD_DOUT, nfg::SINK_STORE, a, c->num_sms,
                                   c->stream, nullptr));
        NFG_CUDA(nfg::launch_encode_bwd_lv(f->shape, f->d_levels, X, B, dY, f->d_g, c->stream, f->d_res->flags));
        c->launches += 3;
        f->grads_clean = false;
    });
}

nfg_status nfg_mlp_forward_device(nfg_field* f, const float* Y, int64_t B, float* out)
{
    return guard([&] {
        nfg::InferArgs a{};
        a.Y = Y;
        a.B = B;
        a.W = f->d_p + f->n_tab_dev;
        a.b = f->d_p + f->n_tab_dev + f->n_w;
        a.out = out;
        NFG_CUDA(nfg::launch_infer(f->shape, nullptr, nfg::SRC_LOAD_Y, a, f->ctx->num_sms, f->ctx->stream));
        f->ctx->launches++;
    });
}

nfg_status nfg_mlp_backward_device(nfg_field* f, const float* Y, int64_t B, const float* dOut, float* dY)
{
    return guard([&] {
        if (B <= 0)
            return;
        reset_scratch(f);
        nfg::TrainArgs a{};
        a.Y = Y;
        a.dout = dOut;
        a.B = B;
        a.inv_count = 1.0f;
        a.W = f->d_p + f->n_tab_dev;
        a.b = f->d_p + f->n_tab_dev + f->n_w;
        a.dY = dY;
        a.gW = f->d_g + f->n_tab_dev;
        a.gb = f->d_g + f->n_tab_dev + f->n_w;
        a.scratch = scratch_of(f);
        NFG_CUDA(nfg::launch_train(f->shape, nullptr, nfg::SRC_LOAD_Y, nfg::GRAD_DOUT, nfg::SINK_STORE, a,
                                   f->ctx->num_sms, f->ctx->stream, nullptr));
        f->ctx->launches++;
        f->grads_clean = false;
    });
}

nfg_status nfg_adam_step_device(nfg_field* f, float lr_now)
{
    return guard([&] {
        // the producers are this library's kernels: their "maybe non-finite"
        // flag (flags[0]) triggers the exact scan only when needed
        run_adam(f, lr_now, false);
        f->pending_steps++;
        f->grads_clean = true;   // optimistic; nfg_field_check corrects it
    });
}

nfg_status nfg_host_alloc(size_t bytes, void** out)
{
    return guard([&] { NFG_CUDA(cudaMallocHost(out, bytes)); });
}

nfg_status nfg_host_free(void* p)
{
    return guard([&] { NFG_CUDA(cudaFreeHost(p)); });
}

}   // extern "C"
