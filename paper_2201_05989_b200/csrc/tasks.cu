// tasks.cu — the training-loop data path on the device:
//
//   * nfg_rng: the reference's Pcg32 stream (pcg32.hpp) generated in parallel
//     by O(log n) jump-ahead, with next_below's rejection sampling reproduced
//     EXACTLY (draws flagged, prefix-summed, compacted): n device draws leave
//     the stream in the same state as n sequential host calls;
//   * nfg_fit_image: fit_image (tasks.cpp:49-131) with the batch sampling,
//     the pixel -> (x, target) gather, the PSNR evaluation and the training
//     step all on the device; the host only reads the per-step status records
//     back at the report rows (the reference checks every step's loss; the
//     records let the same checks run lazily, in step order).
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/nfg.h"
#include "host_common.h"
#include "host_init.h"


namespace {

using nfg::hc::Buf;
using nfg::hc::Fail;
using nfg::hc::grid_for;
using nfg::hc::ok;
using nfg::hc::run;

constexpr uint64_t PCG_MULT = 6364136223846793005ULL;

struct RngState {
    uint64_t state, inc;
};

__host__ __device__ inline uint32_t pcg_output(uint64_t old)   // pcg32.hpp:22-26
{
    const uint32_t xorshifted = uint32_t(((old >> 18u) ^ old) >> 27u);
    const uint32_t rot = uint32_t(old >> 59u);
    return (xorshifted >> rot) | (xorshifted << ((32u - rot) & 31u));
}

// State after `delta` calls of next_u32 (PCG's logarithmic jump-ahead).
__host__ __device__ inline uint64_t pcg_advance(uint64_t state, uint64_t inc, uint64_t delta)
{
    uint64_t acc_mult = 1u, acc_plus = 0u, cur_mult = PCG_MULT, cur_plus = inc;
    while (delta) {
        if (delta & 1u) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1u) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1u;
    }
    return acc_mult * state + acc_plus;
}

__global__ void k_rng_direct(const RngState* __restrict__ src, RngState* __restrict__ dst, uint32_t bound,
                             int64_t n, uint32_t* __restrict__ out_u, float* __restrict__ out_f)
{
    const RngState r = *src;
    const int64_t j0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    if (j0 < n) {
        uint64_t s = pcg_advance(r.state, r.inc, uint64_t(j0));
        // affine map of `stride` draws: s -> sm * s + sp
        uint64_t sm = 1u, sp = 0u;
        {
            uint64_t cm = PCG_MULT, cp = r.inc, d = uint64_t(stride);
            while (d) {
                if (d & 1u) {
                    sm *= cm;
                    sp = sp * cm + cp;
                }
                cp = (cm + 1u) * cp;
                cm *= cm;
                d >>= 1u;
            }
        }
        for (int64_t j = j0; j < n; j += stride) {
            const uint32_t v = pcg_output(s);
            if (out_u)
                out_u[j] = bound ? v % bound : v;   // threshold == 0: next_below never rejects; 0: raw next_u32
            else
                out_f[j] = float(v >> 8) * 0x1p-24f;   // next_float (pcg32.hpp:41-44)
            s = sm * s + sp;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0)
        *dst = RngState{ pcg_advance(r.state, r.inc, uint64_t(n)), r.inc };
}

__global__ void k_rng_draw(const RngState* __restrict__ src, int64_t m, uint32_t threshold, uint32_t* __restrict__ vals,
                           uint32_t* __restrict__ keep)
{
    const RngState r = *src;
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < m; j += int64_t(gridDim.x) * blockDim.x) {
        const uint32_t v = pcg_output(pcg_advance(r.state, r.inc, uint64_t(j)));
        vals[j] = v;
        keep[j] = v >= threshold ? 1u : 0u;   // pcg32.hpp:33-37
    }
}

__global__ void k_rng_compact(const RngState* __restrict__ src, RngState* __restrict__ dst, int64_t m, int64_t n,
                              uint32_t bound, const uint32_t* __restrict__ vals, const uint32_t* __restrict__ keep,
                              const uint32_t* __restrict__ pos, uint32_t* __restrict__ out, unsigned int* err)
{
    const RngState r = *src;
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < m; j += int64_t(gridDim.x) * blockDim.x) {
        const int64_t p = pos[j];
        if (keep[j] && p < n) {
            out[p] = vals[j] % bound;
            if (p == n - 1)
                *dst = RngState{ pcg_advance(r.state, r.inc, uint64_t(j) + 1u), r.inc };
        }
        if (j == m - 1 && p + int64_t(keep[j]) < n) {   // margin exhausted (never in practice)
            *err = 1u;
            *dst = RngState{ pcg_advance(r.state, r.inc, uint64_t(m)), r.inc };
        }
    }
}

// fit_image's batch assembly (tasks.cpp:114-120, eval grid 88-93): pixel p ->
// x = ((p % w) + 0.5) / w, y = ((p / w) + 0.5) / h in fp32, target = rgb.col(p).
__global__ void k_image_batch(const uint32_t* __restrict__ idx, int64_t n, const float* __restrict__ rgb, uint32_t w,
                              uint32_t h, float* __restrict__ X, float* __restrict__ T)
{
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const uint32_t p = idx ? idx[i] : uint32_t(i);
        X[2 * i] = __fdiv_rn(__fadd_rn(__uint2float_rn(p % w), 0.5f), __uint2float_rn(w));
        X[2 * i + 1] = __fdiv_rn(__fadd_rn(__uint2float_rn(p / w), 0.5f), __uint2float_rn(h));
        T[3 * i] = rgb[3 * size_t(p)];
        T[3 * i + 1] = rgb[3 * size_t(p) + 1];
        T[3 * i + 2] = rgb[3 * size_t(p) + 2];
    }
}

// Sum of squared differences (psnr, losses.hpp:63-71): per-block double
// partials, then one ordered sum (deterministic).
__global__ void __launch_bounds__(256) k_sqerr(const float* __restrict__ a, const float* __restrict__ b, int64_t n,
                                               double* __restrict__ partial)
{
    __shared__ double sh[256];
    double s = 0.0;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const double d = double(a[i]) - double(b[i]);
        s += d * d;
    }
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int k = 128; k > 0; k >>= 1) {
        if (int(threadIdx.x) < k)
            sh[threadIdx.x] += sh[threadIdx.x + k];
        __syncthreads();
    }
    if (threadIdx.x == 0)
        partial[blockIdx.x] = sh[0];
}

__global__ void k_sum_partials(const double* __restrict__ partial, int n, double* out)
{
    double s = 0.0;
    for (int i = 0; i < n; ++i)
        s += partial[i];
    *out = s;
}







// ---- fit_sdf on the analytic CSG target (BASELINE config 2) -----------------
// The CSG SDF of the synthetic SDF scene (sphere r=.3 at the cube centre union a
// torus R=.25, r=.08 in the xz-plane), in the oracle's exact fp32 operation
// order (oracle/nf_oracle.hpp csg_sdf).
template <class S>
__device__ __forceinline__ S csg_sdf(S x, S y, S z)
{
    const S cx = x - S(0.5), cy = y - S(0.5), cz = z - S(0.5);
    const S sphere = sqrt(cx * cx + cy * cy + cz * cz) - S(0.3);
    const S q = sqrt(cx * cx + cz * cz) - S(0.25);
    const S torus = sqrt(q * q + cy * cy) - S(0.08);
    return sphere < torus ? sphere : torus;
}

__device__ __forceinline__ float csg_sdf_f(float x, float y, float z)
{
    const float cx = __fsub_rn(x, 0.5f), cy = __fsub_rn(y, 0.5f), cz = __fsub_rn(z, 0.5f);
    const float sphere =
        __fsub_rn(__fsqrt_rn(__fadd_rn(__fadd_rn(__fmul_rn(cx, cx), __fmul_rn(cy, cy)), __fmul_rn(cz, cz))), 0.3f);
    const float q = __fsub_rn(__fsqrt_rn(__fadd_rn(__fmul_rn(cx, cx), __fmul_rn(cz, cz))), 0.25f);
    const float torus = __fsub_rn(__fsqrt_rn(__fadd_rn(__fmul_rn(q, q), __fmul_rn(cy, cy))), 0.08f);
    return fminf(sphere, torus);
}

__global__ void k_csg_target(const float* __restrict__ X, int64_t n, float* __restrict__ T)
{
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        T[i] = csg_sdf_f(X[3 * i], X[3 * i + 1], X[3 * i + 2]);
}

// iou points (Pcg32::uniform<double> in [0,1]^3 from 6 draws) and the
// analytic interior test in double on the double point, as the reference's
// oracle_sign gets the double point (tasks.cpp:338-350)
__global__ void k_iou_points_csg(const uint32_t* __restrict__ u, int64_t n, float* __restrict__ X,
                                 uint8_t* __restrict__ inside)
{
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        double p[3];
        for (int k = 0; k < 3; ++k) {
            const uint64_t a = u[6 * i + 2 * k], b = u[6 * i + 2 * k + 1];
            p[k] = 0.0 + (1.0 - 0.0) * (double((a << 21) ^ b) * 0x1p-53);
            X[3 * i + k] = float(p[k]);
        }
        inside[i] = csg_sdf<double>(p[0], p[1], p[2]) < 0.0 ? 1 : 0;
    }
}

__global__ void k_iou_count(const float* __restrict__ pred, const uint8_t* __restrict__ inside, int64_t n,
                            unsigned long long* both_either)
{
    unsigned long long b = 0, e = 0;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const bool m = pred[i] < 0.0f, o = inside[i] != 0;
        b += (m && o) ? 1 : 0;
        e += (m || o) ? 1 : 0;
    }
    for (int s = 16; s > 0; s >>= 1) {
        b += __shfl_xor_sync(0xffffffffu, b, s);
        e += __shfl_xor_sync(0xffffffffu, e, s);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(both_either, b);
        atomicAdd(both_either + 1, e);
    }
}

}   // namespace

struct nfg_rng {
    nfg_ctx* ctx = nullptr;
    cudaStream_t stream = nullptr;
    RngState* d = nullptr;   // double-buffered state: [cur] is the stream's position
    int cur = 0;
    unsigned int* d_err = nullptr;
    Buf vals, keep, pos, tmp;

    void below(uint32_t bound, int64_t n, uint32_t* out)
    {
        if (bound == 0u)
            throw std::invalid_argument("next_below: bound must be positive");
        if (n < 0)
            throw std::invalid_argument("nfg_rng: negative count");
        const uint32_t threshold = (~bound + 1u) % bound;   // pcg32.hpp:32
        RngState* src = d + cur;
        RngState* dst = d + (cur ^ 1);
        if (threshold == 0u || n == 0) {
            k_rng_direct<<<grid_for(n), 256, 0, stream>>>(src, dst, bound, n, out, nullptr);
            NFG_HC_CUDA(cudaGetLastError());
        } else {
            // expected rejections n*p; the margin covers > 10 sigma
            const double p = double(threshold) / 4294967296.0;
            const double mean = double(n) * p / (1.0 - p);
            const int64_t m = n + int64_t(std::ceil(2.0 * mean + 10.0 * std::sqrt(mean + 1.0) + 64.0));
            uint32_t* v = static_cast<uint32_t*>(vals.get(size_t(m) * 4));
            uint32_t* k = static_cast<uint32_t*>(keep.get(size_t(m) * 4));
            uint32_t* q = static_cast<uint32_t*>(pos.get(size_t(m) * 4));
            size_t tb = 0;
            NFG_HC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, k, q, m, stream));
            void* t = tmp.get(std::max<size_t>(tb, 16));
            k_rng_draw<<<grid_for(m), 256, 0, stream>>>(src, m, threshold, v, k);
            NFG_HC_CUDA(cudaGetLastError());
            NFG_HC_CUDA(cub::DeviceScan::ExclusiveSum(t, tb, k, q, m, stream));
            k_rng_compact<<<grid_for(m), 256, 0, stream>>>(src, dst, m, n, bound, v, k, q, out, d_err);
            NFG_HC_CUDA(cudaGetLastError());
        }
        cur ^= 1;
    }

    void u32(int64_t n, uint32_t* out)
    {
        if (n < 0)
            throw std::invalid_argument("nfg_rng: negative count");
        k_rng_direct<<<grid_for(n), 256, 0, stream>>>(d + cur, d + (cur ^ 1), 0u, n, out, nullptr);
        NFG_HC_CUDA(cudaGetLastError());
        cur ^= 1;
    }

    void floats(int64_t n, float* out)
    {
        if (n < 0)
            throw std::invalid_argument("nfg_rng: negative count");
        k_rng_direct<<<grid_for(n), 256, 0, stream>>>(d + cur, d + (cur ^ 1), 1u, n, nullptr, out);
        NFG_HC_CUDA(cudaGetLastError());
        cur ^= 1;
    }

    void check()
    {
        unsigned int e = 0;
        NFG_HC_CUDA(cudaMemcpyAsync(&e, d_err, 4, cudaMemcpyDeviceToHost, stream));
        NFG_HC_CUDA(cudaStreamSynchronize(stream));
        if (e)
            throw Fail{ NFG_ECUDA, "nfg_rng: rejection-sampling margin exhausted" };
    }

    ~nfg_rng()
    {
        if (d)
            cudaFree(d);
        if (d_err)
            cudaFree(d_err);
    }
};

extern "C" {

nfg_status nfg_rng_create(nfg_ctx* ctx, uint64_t seed, uint64_t seq, nfg_rng** out)
{
    return run([&] {
        auto r = std::make_unique<nfg_rng>();
        r->ctx = ctx;
        r->stream = static_cast<cudaStream_t>(nfg_ctx_stream(ctx));
        // Pcg32(seed, seq) (pcg32.hpp:11-18)
        RngState h{ 0u, (seq << 1u) | 1u };
        h.state = h.state * PCG_MULT + h.inc;
        h.state += seed;
        h.state = h.state * PCG_MULT + h.inc;
        NFG_HC_CUDA(cudaMalloc(&r->d, 2 * sizeof(RngState)));
        NFG_HC_CUDA(cudaMalloc(&r->d_err, sizeof(unsigned int)));
        NFG_HC_CUDA(cudaMemcpyAsync(r->d, &h, sizeof(h), cudaMemcpyHostToDevice, r->stream));
        NFG_HC_CUDA(cudaMemsetAsync(r->d_err, 0, sizeof(unsigned int), r->stream));
        NFG_HC_CUDA(cudaStreamSynchronize(r->stream));
        *out = r.release();
    });
}

nfg_status nfg_rng_destroy(nfg_rng* r)
{
    return run([&] {
        if (r)
            cudaStreamSynchronize(r->stream);
        delete r;
    });
}

nfg_status nfg_rng_below_device(nfg_rng* r, uint32_t bound, int64_t n, uint32_t* out_dev)
{
    return run([&] { r->below(bound, n, out_dev); });
}

nfg_status nfg_rng_u32_device(nfg_rng* r, int64_t n, uint32_t* out_dev)
{
    return run([&] { r->u32(n, out_dev); });
}

nfg_status nfg_rng_floats_device(nfg_rng* r, int64_t n, float* out_dev)
{
    return run([&] { r->floats(n, out_dev); });
}

nfg_status nfg_rng_get_state(nfg_rng* r, uint64_t* state, uint64_t* inc)
{
    return run([&] {
        r->check();
        RngState h{};
        NFG_HC_CUDA(cudaMemcpyAsync(&h, r->d + r->cur, sizeof(h), cudaMemcpyDeviceToHost, r->stream));
        NFG_HC_CUDA(cudaStreamSynchronize(r->stream));
        *state = h.state;
        *inc = h.inc;
    });
}

nfg_status nfg_image_batch_device(nfg_ctx* ctx, const uint32_t* idx_dev, int64_t n, const float* rgb_dev,
                                  int32_t width, int32_t height, float* X_dev, float* T_dev)
{
    return run([&] {
        if (width < 1 || height < 1)
            throw std::invalid_argument("image batch: empty image");
        cudaStream_t st = static_cast<cudaStream_t>(nfg_ctx_stream(ctx));
        if (n > 0) {
            k_image_batch<<<grid_for(n), 256, 0, st>>>(idx_dev, n, rgb_dev, uint32_t(width), uint32_t(height), X_dev,
                                                        T_dev);
            NFG_HC_CUDA(cudaGetLastError());
        }
    });
}

nfg_status nfg_fit_image(nfg_ctx* ctx, const nfg_image_task* task, const float* rgb, uint64_t seed,
                         const nfg_options* opts, nfg_field** model_out, nfg_report_row* rows, int64_t rows_cap,
                         int64_t* n_rows)
{
    return run([&] {
        *model_out = nullptr;
        if (n_rows)
            *n_rows = 0;
        const int w = task->width, h = task->height;
        if (w < 2 || h < 2)   // tasks.cpp:52-53
            throw std::invalid_argument("fit_image: image must be at least 2x2");
        if (task->batch_size < 0 || task->total_steps < 0 || task->log_interval <= 0)
            throw std::invalid_argument("fit_image: invalid task");
        const uint64_t npix = uint64_t(w) * uint64_t(h);
        if (npix > 0xffffffffull)
            throw std::invalid_argument("fit_image: image too large for next_below (u32)");
        cudaStream_t st = static_cast<cudaStream_t>(nfg_ctx_stream(ctx));

        // model configuration (tasks.cpp:55-71)
        nfg_grid_config g = task->cfg;
        g.dims = 2;
        if (g.n_max <= 0)
            g.n_max = std::max(g.n_min, w / 2);
        nfg_mlp_config m{};
        m.hidden_layers = task->hidden_layers;
        m.hidden_width = task->hidden_width;
        m.output_width = 3;
        m.output_activation = NFG_ACT_SIGMOID;
        nfg_adam_hyper hy{ task->lr, 0.9, 0.99, 1e-15, 1e-6 };
        nfg_options o = opts ? *opts : nfg_options{ 0, 1, 0, 0 };
        nfg_field* f = nullptr;
        ok(nfg_field_create(ctx, &g, &m, &hy, &o, &f));
        std::unique_ptr<nfg_field, nfg_status (*)(nfg_field*)> model(f, nfg_field_destroy);
        ok(nfg_field_init(f, seed));
        // default_schedule (adam.hpp:150-161)
        std::vector<int64_t> ms;
        {
            const int64_t total = task->total_steps;
            int64_t next = int64_t(0.65 * double(total));
            const int64_t stride = int64_t(0.30 * double(total));
            while (next < total && stride > 0) {
                ms.push_back(next);
                next += stride;
            }
        }
        ok(nfg_field_set_schedule(f, ms.empty() ? nullptr : ms.data(), int32_t(ms.size()), task->lr_decay));

        Buf d_rgb, d_eidx, d_ex, d_et, d_pred, d_idx, d_X, d_T, d_part, d_sum, d_rec;
        float* rgb_dev = static_cast<float*>(d_rgb.get(npix * 3 * 4));
        NFG_HC_CUDA(cudaMemcpyAsync(rgb_dev, rgb, npix * 3 * 4, cudaMemcpyHostToDevice, st));

        // PSNR grid (tasks.cpp:78-94): every pixel, or 2^16 from Pcg32(seed, 7)
        const bool full = npix <= (uint64_t(1) << 20);
        const int64_t ne = full ? int64_t(npix) : (int64_t(1) << 16);
        uint32_t* eidx = nullptr;
        if (!full) {
            nfg_rng* er = nullptr;
            ok(nfg_rng_create(ctx, seed, 7, &er));
            std::unique_ptr<nfg_rng, nfg_status (*)(nfg_rng*)> eg(er, nfg_rng_destroy);
            eidx = static_cast<uint32_t*>(d_eidx.get(size_t(ne) * 4));
            er->below(uint32_t(npix), ne, eidx);
            er->check();
        }
        float* ex = static_cast<float*>(d_ex.get(size_t(ne) * 2 * 4));
        float* et = static_cast<float*>(d_et.get(size_t(ne) * 3 * 4));
        float* pred = static_cast<float*>(d_pred.get(size_t(ne) * 3 * 4));
        k_image_batch<<<grid_for(ne), 256, 0, st>>>(eidx, ne, rgb_dev, uint32_t(w), uint32_t(h), ex, et);
        NFG_HC_CUDA(cudaGetLastError());
        const unsigned sq_blocks = unsigned(std::max<int64_t>(1, std::min<int64_t>((ne * 3 + 255) / 256, 1024)));
        double* part = static_cast<double*>(d_part.get(sq_blocks * 8));
        double* dsum = static_cast<double*>(d_sum.get(8));

        std::vector<nfg_report_row> report;
        const auto t0 = std::chrono::steady_clock::now();
        auto mse_now = [&]() {   // evaluate_chunked on the grid + squared error
            ok(nfg_field_evaluate_device(f, ex, ne, pred));
            k_sqerr<<<sq_blocks, 256, 0, st>>>(pred, et, ne * 3, part);
            k_sum_partials<<<1, 1, 0, st>>>(part, int(sq_blocks), dsum);
            NFG_HC_CUDA(cudaGetLastError());
            double s = 0.0;
            NFG_HC_CUDA(cudaMemcpyAsync(&s, dsum, 8, cudaMemcpyDeviceToHost, st));
            NFG_HC_CUDA(cudaStreamSynchronize(st));
            return s / double(ne * 3);
        };
        auto log_row = [&](int64_t step, double loss, double mse) {   // tasks.cpp:95-105
            nfg_report_row r{};
            r.step = step;
            r.time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            r.loss = loss;
            r.metric = mse <= 0 ? 100.0 : std::min(100.0, -10.0 * std::log10(mse));   // losses.hpp:63-71
            r.lr = nfg_lr_at(ms.empty() ? nullptr : ms.data(), int32_t(ms.size()), task->lr_decay, task->lr, step);
            report.push_back(r);
        };
        {
            const double mse = mse_now();
            log_row(0, mse, mse);
        }

        // training loop (tasks.cpp:112-128): batches from Pcg32(seed, 1)
        nfg_rng* br = nullptr;
        ok(nfg_rng_create(ctx, seed, 1, &br));
        std::unique_ptr<nfg_rng, nfg_status (*)(nfg_rng*)> brg(br, nfg_rng_destroy);
        const int64_t B = task->batch_size;
        uint32_t* idx = static_cast<uint32_t*>(d_idx.get(std::max<size_t>(size_t(B) * 4, 16)));
        float* X = static_cast<float*>(d_X.get(std::max<size_t>(size_t(B) * 2 * 4, 16)));
        float* T = static_cast<float*>(d_T.get(std::max<size_t>(size_t(B) * 3 * 4, 16)));
        const int64_t chunk = std::min<int64_t>(task->log_interval, std::max<int64_t>(task->total_steps, 1));
        nfg_step_record* recs = static_cast<nfg_step_record*>(d_rec.get(size_t(chunk) * sizeof(nfg_step_record)));
        std::vector<nfg_step_record> hrec(static_cast<size_t>(chunk));
        int64_t pending = 0, first_pending = 1;
        for (int64_t step = 1; step <= task->total_steps; ++step) {
            br->below(uint32_t(npix), B, idx);
            if (B > 0) {
                k_image_batch<<<grid_for(B), 256, 0, st>>>(idx, B, rgb_dev, uint32_t(w), uint32_t(h), X, T);
                NFG_HC_CUDA(cudaGetLastError());
            }
            ok(nfg_field_train_step_device(f, X, T, B, B, NFG_LOSS_L2, step, nullptr));
            ok(nfg_field_step_record(f, recs + pending));
            ++pending;
            const bool log = step % task->log_interval == 0 || step == task->total_steps;
            if (!log && pending < chunk)
                continue;
            NFG_HC_CUDA(cudaMemcpyAsync(hrec.data(), recs, size_t(pending) * sizeof(nfg_step_record),
                                    cudaMemcpyDeviceToHost, st));
            NFG_HC_CUDA(cudaStreamSynchronize(st));
            br->check();
            float loss = 0.0f;
            for (int64_t k = 0; k < pending; ++k) {   // the reference's per-step checks, in step order
                ok(nfg_step_record_check(f, &hrec[size_t(k)], B, &loss));
                if (!std::isfinite(loss))   // tasks.cpp:122-123
                    throw Fail{ NFG_ENONFINITE,
                                "fit_image: non-finite loss at step " + std::to_string(first_pending + k) };
            }
            pending = 0;
            first_pending = step + 1;
            if (log)
                log_row(step, double(loss), mse_now());
        }
        if (task->total_steps > 0)
            ok(nfg_field_check(f));
        const int64_t nr = int64_t(report.size());
        for (int64_t i = 0; i < std::min(nr, rows_cap); ++i)
            rows[i] = report[size_t(i)];
        if (n_rows)
            *n_rows = nr;
        *model_out = model.release();
    });
}

nfg_status nfg_csg_sdf_device(nfg_ctx* ctx, const float* X_dev, int64_t n, float* out_dev)
{
    return run([&] {
        if (n > 0) {
            k_csg_target<<<grid_for(n), 256, 0, static_cast<cudaStream_t>(nfg_ctx_stream(ctx))>>>(X_dev, n, out_dev);
            NFG_HC_CUDA(cudaGetLastError());
        }
    });
}

nfg_status nfg_fit_sdf_analytic(nfg_ctx* ctx, const nfg_sdf_task* task, uint64_t seed, const nfg_options* opts,
                                nfg_field** model_out, nfg_report_row* rows, int64_t rows_cap, int64_t* n_rows)
{
    return run([&] {
        *model_out = nullptr;
        if (n_rows)
            *n_rows = 0;
        if (task->batch_size < 0 || task->total_steps < 0 || task->log_interval <= 0 || task->iou_eval_points < 0)
            throw std::invalid_argument("fit_sdf: invalid task");
        if (task->loss < 0 || task->loss > 2)
            throw std::invalid_argument("fit_sdf: unknown loss");
        cudaStream_t st = static_cast<cudaStream_t>(nfg_ctx_stream(ctx));
        // model configuration (tasks.cpp:140-158)
        nfg_grid_config g = task->cfg;
        g.dims = 3;
        nfg_mlp_config m{};
        m.hidden_layers = task->hidden_layers;
        m.hidden_width = task->hidden_width;
        m.output_width = 1;
        m.output_activation = NFG_ACT_LINEAR;
        nfg_adam_hyper hy{ task->lr, 0.9, 0.99, 1e-15, 1e-6 };
        nfg_options o = opts ? *opts : nfg_options{ 0, 1, 0, 0 };
        nfg_field* f = nullptr;
        ok(nfg_field_create(ctx, &g, &m, &hy, &o, &f));
        std::unique_ptr<nfg_field, nfg_status (*)(nfg_field*)> model(f, nfg_field_destroy);
        ok(nfg_field_init(f, seed));
        std::vector<int64_t> ms;
        {
            const int64_t total = task->total_steps;
            int64_t next = int64_t(0.65 * double(total));
            const int64_t stride = int64_t(0.30 * double(total));
            while (next < total && stride > 0) {
                ms.push_back(next);
                next += stride;
            }
        }
        ok(nfg_field_set_schedule(f, ms.empty() ? nullptr : ms.data(), int32_t(ms.size()), task->lr_decay));

        Buf d_u, d_xi, d_in, d_pred, d_cnt, d_X, d_T, d_rec;
        std::vector<nfg_report_row> report;
        const auto t0 = std::chrono::steady_clock::now();
        auto iou_now = [&]() {   // tasks.cpp:163-171: Pcg32(seed, 11), same points every row
            nfg_rng* ir = nullptr;
            ok(nfg_rng_create(ctx, seed, 11, &ir));
            std::unique_ptr<nfg_rng, nfg_status (*)(nfg_rng*)> irg(ir, nfg_rng_destroy);
            unsigned long long* cnt = d_cnt.as<unsigned long long>(2);
            NFG_HC_CUDA(cudaMemsetAsync(cnt, 0, 16, st));
            const int64_t chunk = int64_t(1) << 16;
            for (int64_t done = 0; done < task->iou_eval_points; done += chunk) {
                const int64_t k = std::min(chunk, task->iou_eval_points - done);
                uint32_t* u = d_u.as<uint32_t>(size_t(k) * 6);
                float* xi = d_xi.as<float>(size_t(k) * 3);
                uint8_t* in = d_in.as<uint8_t>(size_t(k));
                float* pr = d_pred.as<float>(size_t(k));
                ir->u32(k * 6, u);
                k_iou_points_csg<<<grid_for(k), 256, 0, st>>>(u, k, xi, in);
                NFG_HC_CUDA(cudaGetLastError());
                ok(nfg_field_evaluate_device(f, xi, k, pr));
                k_iou_count<<<grid_for(k), 256, 0, st>>>(pr, in, k, cnt);
                NFG_HC_CUDA(cudaGetLastError());
            }
            unsigned long long h[2] = { 0, 0 };
            NFG_HC_CUDA(cudaMemcpyAsync(h, cnt, 16, cudaMemcpyDeviceToHost, st));
            NFG_HC_CUDA(cudaStreamSynchronize(st));
            return h[1] == 0 ? 1.0 : double(h[0]) / double(h[1]);
        };
        auto log_row = [&](int64_t step, double loss) {
            nfg_report_row r{};
            r.step = step;
            r.time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            r.loss = loss;
            r.metric = iou_now();
            r.lr = nfg_lr_at(ms.empty() ? nullptr : ms.data(), int32_t(ms.size()), task->lr_decay, task->lr, step);
            report.push_back(r);
        };
        log_row(0, 0.0);   // tasks.cpp:173

        nfg_rng* sr = nullptr;   // Pcg32(seed, 2) (tasks.cpp:175)
        ok(nfg_rng_create(ctx, seed, 2, &sr));
        std::unique_ptr<nfg_rng, nfg_status (*)(nfg_rng*)> srg(sr, nfg_rng_destroy);
        const int64_t B = task->batch_size;
        float* X = d_X.as<float>(std::max<size_t>(size_t(B) * 3, 4));
        float* T = d_T.as<float>(std::max<size_t>(size_t(B), 4));
        const int64_t chunk = std::min<int64_t>(task->log_interval, std::max<int64_t>(task->total_steps, 1));
        nfg_step_record* recs = d_rec.as<nfg_step_record>(size_t(chunk));
        std::vector<nfg_step_record> hrec(static_cast<size_t>(chunk));
        int64_t pending = 0, first_pending = 1;
        for (int64_t step = 1; step <= task->total_steps; ++step) {
            sr->floats(B * 3, X);   // uniform points in [0,1]^3 (analytic target: no mesh sampling)
            if (B > 0) {
                k_csg_target<<<grid_for(B), 256, 0, st>>>(X, B, T);
                NFG_HC_CUDA(cudaGetLastError());
            }
            ok(nfg_field_train_step_device(f, X, T, B, B, task->loss, step, nullptr));
            ok(nfg_field_step_record(f, recs + pending));
            ++pending;
            const bool log = step % task->log_interval == 0 || step == task->total_steps;
            if (!log && pending < chunk)
                continue;
            NFG_HC_CUDA(cudaMemcpyAsync(hrec.data(), recs, size_t(pending) * sizeof(nfg_step_record),
                                        cudaMemcpyDeviceToHost, st));
            NFG_HC_CUDA(cudaStreamSynchronize(st));
            sr->check();
            float loss = 0.0f;
            for (int64_t k = 0; k < pending; ++k) {
                ok(nfg_step_record_check(f, &hrec[size_t(k)], B, &loss));
                if (!std::isfinite(loss))   // tasks.cpp:187-188
                    throw Fail{ NFG_ENONFINITE, "fit_sdf: non-finite loss at step " + std::to_string(first_pending + k) };
            }
            pending = 0;
            first_pending = step + 1;
            if (log)
                log_row(step, double(loss));
        }
        if (task->total_steps > 0)
            ok(nfg_field_check(f));
        const int64_t nr = int64_t(report.size());
        for (int64_t i = 0; i < std::min(nr, rows_cap); ++i)
            rows[i] = report[size_t(i)];
        if (n_rows)
            *n_rows = nr;
        *model_out = model.release();
    });
}

}   // extern "C"
