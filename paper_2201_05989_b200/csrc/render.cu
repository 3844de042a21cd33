// render.cu — the inference consumers of the field:
//
//   render_image       (tasks.cpp:195-209)  pixel-centre grid -> fused inference
//   render_sdf_shaded  (tasks.cpp:233-329)  sphere tracing with ACTIVE-RAY
//                      COMPACTION on the device: per iteration the live rays are
//                      evaluated in one batch, hits and survivors are appended to
//                      compact lists (atomic slot claims; the image does not
//                      depend on list order), then 6 central-difference probes
//                      per hit and Lambert shading
//   iou                (tasks.cpp:331-356)  points drawn from the device Pcg32
//                      stream exactly as Pcg32::uniform<double> would
//
// The field is either an nfg_field (the fused sm_100a inference kernel) or a
// host FieldFn callback (tasks.hpp:70: any function of X, e.g. an analytic
// SDF), in which case each batch of points travels to the host and back.
// Ray arithmetic is double precision without contraction (built with
// -fmad=false), in the reference's evaluation order.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/nfg.h"
#include "host_common.h"


namespace {

using nfg::hc::Buf;
using nfg::hc::Fail;
using nfg::hc::grid_for;
using nfg::hc::ok;
using nfg::hc::run;

struct Ray {
    double dir[3];
    double t, t_exit;
    int pixel;
    int pad;
};

struct Basis {
    double pos[3], fwd[3], right[3], up[3];
    double half_tan, aspect;
};

// ---- render_image: pixel centres (tasks.cpp:197-203) --------------------------
__global__ void k_pixel_grid(int w, int h, float* X)
{
    const int64_t n = int64_t(w) * h;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int x = int(i % w), y = int(i / w);
        X[2 * i] = (float(x) + 0.5f) / float(w);
        X[2 * i + 1] = (float(y) + 0.5f) / float(h);
    }
}

// ---- render_sdf_shaded -------------------------------------------------------
__device__ bool ray_unit_cube(const double* o, const double* d, double& t0, double& t1)   // tasks.cpp:213-229
{
    t0 = 0.0;
    t1 = __longlong_as_double(0x7ff0000000000000ll);
    for (int i = 0; i < 3; ++i) {
        const double inv = 1.0 / d[i];
        double nr = (0.0 - o[i]) * inv;
        double fr = (1.0 - o[i]) * inv;
        if (nr > fr) {
            const double tmp = nr;
            nr = fr;
            fr = tmp;
        }
        t0 = (t0 < nr) ? nr : t0;   // std::max(t0, near)
        t1 = (fr < t1) ? fr : t1;   // std::min(t1, far)
        if (t0 > t1)
            return false;
    }
    return true;
}

__global__ void k_rays_init(Basis b, int w, int h, Ray* rays, unsigned int* count)   // tasks.cpp:252-267
{
    const int64_t n = int64_t(w) * h;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int x = int(i % w), y = int(i / w);
        const double u = (2.0 * (x + 0.5) / w - 1.0) * b.half_tan * b.aspect;
        const double v = (1.0 - 2.0 * (y + 0.5) / h) * b.half_tan;
        double d[3];
        for (int k = 0; k < 3; ++k)
            d[k] = b.fwd[k] + u * b.right[k] + v * b.up[k];
        const double nn = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
        for (int k = 0; k < 3; ++k)
            d[k] = d[k] / nn;
        double t0, t1;
        if (!ray_unit_cube(b.pos, d, t0, t1))
            continue;
        const unsigned slot = atomicAdd(count, 1u);
        Ray r;
        for (int k = 0; k < 3; ++k)
            r.dir[k] = d[k];
        r.t = t0 + 1e-6;
        r.t_exit = t1;
        r.pixel = int(i);
        r.pad = 0;
        rays[slot] = r;
    }
}

__device__ __forceinline__ float clamp01f(double p) { return float(fmin(fmax(p, 0.0), 1.0)); }

__global__ void k_ray_points(Basis b, const Ray* rays, int64_t n, float* X)   // tasks.cpp:282-284
{
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const Ray r = rays[i];
        for (int k = 0; k < 3; ++k)
            X[3 * i + k] = clamp01f(b.pos[k] + r.t * r.dir[k]);
    }
}

__global__ void k_ray_step(const Ray* rays, int64_t n, const float* values, Ray* next, unsigned int* n_next,
                           Ray* hits, unsigned int* n_hits)   // tasks.cpp:287-300
{
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        Ray r = rays[i];
        const double v = values[i];
        if (v < 1e-4) {
            hits[atomicAdd(n_hits, 1u)] = r;
            continue;
        }
        r.t += v;
        if (r.t <= r.t_exit)
            next[atomicAdd(n_next, 1u)] = r;
    }
}

__global__ void k_probe_points(Basis b, const Ray* hits, int64_t n, float* X)   // tasks.cpp:306-316
{
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const Ray r = hits[i];
        double p[3];
        for (int k = 0; k < 3; ++k)
            p[k] = b.pos[k] + r.t * r.dir[k];
        for (int axis = 0; axis < 3; ++axis)
            for (int s = 0; s < 2; ++s)
                for (int k = 0; k < 3; ++k) {
                    const double q = k == axis ? (s == 0 ? p[k] + 1e-3 : p[k] - 1e-3) : p[k];
                    X[(6 * i + 2 * axis + s) * 3 + k] = clamp01f(q);
                }
    }
}

__global__ void k_shade(const Ray* hits, int64_t n, const float* values, float* rgb)   // tasks.cpp:317-327
{
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const Ray r = hits[i];
        double nv[3];
        for (int axis = 0; axis < 3; ++axis)
            nv[axis] = double(values[6 * i + 2 * axis] - values[6 * i + 2 * axis + 1]);
        const double len = std::sqrt(nv[0] * nv[0] + nv[1] * nv[1] + nv[2] * nv[2]);
        if (len > 0)
            for (int k = 0; k < 3; ++k)
                nv[k] = nv[k] / len;
        const double dot = nv[0] * -r.dir[0] + nv[1] * -r.dir[1] + nv[2] * -r.dir[2];
        const double lambert = dot > 0.0 ? dot : 0.0;
        const float shade = float(0.15 + 0.85 * lambert);
        for (int k = 0; k < 3; ++k)
            rgb[3 * size_t(r.pixel) + k] = 0.9f * shade;
    }
}

__global__ void k_fill(float* p, int64_t n, float v)
{
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        p[i] = v;
}

// ---- iou points: Pcg32::uniform<double> per axis (pcg32.hpp:47-62) ----------
__global__ void k_iou_points(const uint32_t* u, int64_t n, double3 lo, double3 hi, double* P, float* X)
{
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const double l[3] = { lo.x, lo.y, lo.z }, hh[3] = { hi.x, hi.y, hi.z };
        for (int k = 0; k < 3; ++k) {
            const uint64_t a = u[6 * i + 2 * k], b = u[6 * i + 2 * k + 1];
            const double nd = double((a << 21) ^ b) * 0x1p-53;
            const double v = l[k] + (hh[k] - l[k]) * nd;
            P[3 * i + k] = v;
            X[3 * i + k] = float(v);
        }
    }
}

// A field evaluator: the sm_100a model or a host callback.
struct Evaluator {
    nfg_field* field;
    nfg_field_fn fn;
    void* user;
    cudaStream_t st;
    std::vector<float> hx, hv;

    void eval(const float* X_dev, int64_t n, int d, float* out_dev)
    {
        if (n <= 0)
            return;
        if (field) {
            ok(nfg_field_evaluate_device(field, X_dev, n, out_dev));
            return;
        }
        hx.resize(size_t(n) * d);
        hv.resize(size_t(n));
        NFG_HC_CUDA(cudaMemcpyAsync(hx.data(), X_dev, hx.size() * 4, cudaMemcpyDeviceToHost, st));
        NFG_HC_CUDA(cudaStreamSynchronize(st));
        fn(hx.data(), n, hv.data(), user);
        NFG_HC_CUDA(cudaMemcpyAsync(out_dev, hv.data(), hv.size() * 4, cudaMemcpyHostToDevice, st));
    }
};

void cross(const double* a, const double* b, double* o)
{
    o[0] = a[1] * b[2] - a[2] * b[1];
    o[1] = a[2] * b[0] - a[0] * b[2];
    o[2] = a[0] * b[1] - a[1] * b[0];
}

void normalize(double* v)
{
    const double n = std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    for (int k = 0; k < 3; ++k)
        v[k] = v[k] / n;
}

}   // namespace

extern "C" {

nfg_status nfg_render_image(nfg_field* f, int32_t width, int32_t height, float* rgb_host)
{
    return run([&] {
        if (width < 1 || height < 1)
            throw std::invalid_argument("render_image: empty image");
        nfg_grid_config g{};
        nfg_mlp_config m{};
        ok(nfg_field_get_config(f, &g, &m));
        if (g.dims != 2)
            throw std::invalid_argument("render_image: needs a 2D model");
        nfg_ctx* ctx = nullptr;
        ok(nfg_field_context(f, &ctx));
        cudaStream_t st = static_cast<cudaStream_t>(nfg_ctx_stream(ctx));
        const int64_t n = int64_t(width) * height;
        Buf X, out;
        float* x = static_cast<float*>(X.get(size_t(n) * 8));
        float* o = static_cast<float*>(out.get(size_t(n) * m.output_width * 4));
        k_pixel_grid<<<grid_for(n), 256, 0, st>>>(width, height, x);
        NFG_HC_CUDA(cudaGetLastError());
        ok(nfg_field_evaluate_device(f, x, n, o));
        NFG_HC_CUDA(cudaMemcpyAsync(rgb_host, o, size_t(n) * m.output_width * 4, cudaMemcpyDeviceToHost, st));
        NFG_HC_CUDA(cudaStreamSynchronize(st));
    });
}

nfg_status nfg_render_sdf_shaded(nfg_ctx* ctx, nfg_field* field, nfg_field_fn fn, void* user, const nfg_camera* cam,
                                 int32_t width, int32_t height, float* rgb_host)
{
    return run([&] {
        if (width < 1 || height < 1)
            throw std::invalid_argument("render_sdf_shaded: empty image");
        if (!field && !fn)
            throw std::invalid_argument("render_sdf_shaded: no field");
        if (field) {
            nfg_grid_config g{};
            nfg_mlp_config m{};
            ok(nfg_field_get_config(field, &g, &m));
            if (g.dims != 3 || m.output_width != 1)
                throw std::invalid_argument("render_sdf_shaded: needs a 3D model with one output");
        }
        cudaStream_t st = static_cast<cudaStream_t>(nfg_ctx_stream(ctx));
        constexpr int kMaxSteps = 256;
        Basis b{};
        double up_in[3];
        for (int k = 0; k < 3; ++k) {
            b.pos[k] = cam->position[k];
            b.fwd[k] = cam->target[k] - cam->position[k];
            up_in[k] = cam->up[k];
        }
        normalize(b.fwd);
        cross(b.fwd, up_in, b.right);
        normalize(b.right);
        cross(b.right, b.fwd, b.up);
        b.half_tan = std::tan(0.5 * cam->fov_deg * M_PI / 180.0);
        b.aspect = double(width) / double(height);

        const int64_t npix = int64_t(width) * height;
        Buf rays_a, rays_b, hits_b, cnt_b, X, vals, img;
        Ray* cur = static_cast<Ray*>(rays_a.get(size_t(npix) * sizeof(Ray)));
        Ray* nxt = static_cast<Ray*>(rays_b.get(size_t(npix) * sizeof(Ray)));
        Ray* hits = static_cast<Ray*>(hits_b.get(size_t(npix) * sizeof(Ray)));
        unsigned int* cnt = static_cast<unsigned int*>(cnt_b.get(4 * sizeof(unsigned int)));   // [active, next, hits]
        float* x = static_cast<float*>(X.get(size_t(npix) * 6 * 3 * 4));
        float* v = static_cast<float*>(vals.get(size_t(npix) * 6 * 4));
        float* rgb = static_cast<float*>(img.get(size_t(npix) * 3 * 4));
        Evaluator ev{ field, fn, user, st, {}, {} };

        k_fill<<<grid_for(npix * 3), 256, 0, st>>>(rgb, npix * 3, 1.0f);   // background
        NFG_HC_CUDA(cudaMemsetAsync(cnt, 0, 4 * sizeof(unsigned int), st));
        k_rays_init<<<grid_for(npix), 256, 0, st>>>(b, width, height, cur, cnt);
        NFG_HC_CUDA(cudaGetLastError());
        unsigned int h_cnt[4] = { 0, 0, 0, 0 };
        NFG_HC_CUDA(cudaMemcpyAsync(h_cnt, cnt, sizeof(h_cnt), cudaMemcpyDeviceToHost, st));
        NFG_HC_CUDA(cudaStreamSynchronize(st));
        int64_t active = h_cnt[0];
        for (int iter = 0; iter < kMaxSteps && active > 0; ++iter) {
            k_ray_points<<<grid_for(active), 256, 0, st>>>(b, cur, active, x);
            NFG_HC_CUDA(cudaGetLastError());
            ev.eval(x, active, 3, v);
            NFG_HC_CUDA(cudaMemsetAsync(cnt + 1, 0, sizeof(unsigned int), st));
            k_ray_step<<<grid_for(active), 256, 0, st>>>(cur, active, v, nxt, cnt + 1, hits, cnt + 2);
            NFG_HC_CUDA(cudaGetLastError());
            NFG_HC_CUDA(cudaMemcpyAsync(h_cnt, cnt, sizeof(h_cnt), cudaMemcpyDeviceToHost, st));
            NFG_HC_CUDA(cudaStreamSynchronize(st));
            active = h_cnt[1];
            std::swap(cur, nxt);
        }
        const int64_t nh = h_cnt[2];
        if (nh > 0) {
            k_probe_points<<<grid_for(nh), 256, 0, st>>>(b, hits, nh, x);
            NFG_HC_CUDA(cudaGetLastError());
            ev.eval(x, nh * 6, 3, v);
            k_shade<<<grid_for(nh), 256, 0, st>>>(hits, nh, v, rgb);
            NFG_HC_CUDA(cudaGetLastError());
        }
        NFG_HC_CUDA(cudaMemcpyAsync(rgb_host, rgb, size_t(npix) * 3 * 4, cudaMemcpyDeviceToHost, st));
        NFG_HC_CUDA(cudaStreamSynchronize(st));
    });
}

nfg_status nfg_iou(nfg_ctx* ctx, nfg_field* field, nfg_field_fn fn, void* user, nfg_sign_fn oracle_sign,
                   void* sign_user, int64_t n_points, nfg_rng* rng, const double lo[3], const double hi[3], double* out)
{
    return run([&] {
        if (!field && !fn)
            throw std::invalid_argument("iou: no field");
        cudaStream_t st = static_cast<cudaStream_t>(nfg_ctx_stream(ctx));
        const int64_t chunk = int64_t(1) << 16;   // tasks.cpp:335
        Buf U, P, X, V;
        uint32_t* u = static_cast<uint32_t*>(U.get(size_t(chunk) * 6 * 4));
        double* p = static_cast<double*>(P.get(size_t(chunk) * 3 * 8));
        float* x = static_cast<float*>(X.get(size_t(chunk) * 3 * 4));
        float* v = static_cast<float*>(V.get(size_t(chunk) * 4));
        std::vector<double> hp(static_cast<size_t>(chunk) * 3);
        std::vector<float> hv(static_cast<size_t>(chunk));
        Evaluator ev{ field, fn, user, st, {}, {} };
        int64_t both = 0, either = 0;
        for (int64_t done = 0; done < n_points; done += chunk) {
            const int64_t n = std::min(chunk, n_points - done);
            ok(nfg_rng_u32_device(rng, n * 6, u));
            k_iou_points<<<grid_for(n), 256, 0, st>>>(u, n, make_double3(lo[0], lo[1], lo[2]),
                                                       make_double3(hi[0], hi[1], hi[2]), p, x);
            NFG_HC_CUDA(cudaGetLastError());
            ev.eval(x, n, 3, v);
            NFG_HC_CUDA(cudaMemcpyAsync(hp.data(), p, size_t(n) * 3 * 8, cudaMemcpyDeviceToHost, st));
            NFG_HC_CUDA(cudaMemcpyAsync(hv.data(), v, size_t(n) * 4, cudaMemcpyDeviceToHost, st));
            NFG_HC_CUDA(cudaStreamSynchronize(st));
            for (int64_t i = 0; i < n; ++i) {
                const bool m_in = hv[size_t(i)] < 0;
                const bool o_in = oracle_sign(hp.data() + 3 * i, sign_user) < 0;
                both += m_in && o_in;
                either += m_in || o_in;
            }
        }
        *out = either == 0 ? 1.0 : double(both) / double(either);
    });
}

}   // extern "C"
