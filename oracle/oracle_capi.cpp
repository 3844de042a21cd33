// oracle_capi.cpp — extern "C" surface of the CPU oracle for ctypes.
//
// TEST INFRASTRUCTURE ONLY (see nf_oracle.hpp). Loaded by tests/, by
// __graft_entry__.smoke() as the checker and by bench.py's cpu_baseline /
// --impl reference legs; never by the product path.
#include "nf_oracle.hpp"

#include <cstdio>
#include <memory>

namespace {
thread_local std::string g_err;

orc::GridCfg grid_cfg(const int* gc)
{
    // gc = {L, T, F, nmin, nmax, d, smooth}
    orc::GridCfg c;
    c.L = gc[0];
    c.T = std::uint32_t(gc[1]);
    c.F = gc[2];
    c.nmin = gc[3];
    c.nmax = gc[4];
    c.d = gc[5];
    c.smooth = gc[6];
    return c;
}

orc::MlpCfg mlp_cfg(const int* mc)
{
    // mc = {in, hidden_layers, width, out, sigmoid}
    orc::MlpCfg c;
    c.in = mc[0];
    c.hidden_layers = mc[1];
    c.width = mc[2];
    c.out = mc[3];
    c.sigmoid = mc[4];
    return c;
}

template <class F> int guarded(F&& f)
{
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

template <class S>
int encode_fwd_impl(const int* gc, const S* params, const S* X, std::int64_t B, S* Y,
                    std::uint32_t* rows, S* wts)
{
    return guarded([&] {
        const orc::GridCfg c = grid_cfg(gc);
        const auto lv = orc::levels(c);
        if (const char* e = orc::check_inputs<S>(c, X, B))
            throw std::invalid_argument(e);
        orc::encode_fwd<S>(c, lv, params, X, B, Y, rows, wts);
    });
}

template <class S>
int encode_bwd_impl(const int* gc, const std::uint32_t* rows, const S* wts, std::int64_t B,
                    const S* dY, S* grads)
{
    return guarded([&] {
        const orc::GridCfg c = grid_cfg(gc);
        const auto lv = orc::levels(c);
        orc::encode_bwd<S>(c, lv, rows, wts, B, dY, grads);
    });
}

template <class S>
int mlp_impl(const int* mc, const S* W, const S* b, const S* Y, std::int64_t B, S* out,
             const S* dOut, S* gW, S* gb, S* dY)
{
    return guarded([&] {
        const orc::MlpCfg c = mlp_cfg(mc);
        orc::validate(c);
        orc::MlpCache<S> cache;
        orc::mlp_fwd<S>(c, W, b, Y, B, out, cache);
        if (dOut)
            orc::mlp_bwd<S>(c, W, cache, dOut, B, gW, gb, dY);
    });
}

template <class S>
int adam_impl(std::uint64_t* step, int ng, const int* flags, S* const* p, S* const* g, S* const* m,
              S* const* v, const std::uint64_t* n, const char* const* names, const double* hyper,
              S lr_now)
{
    return guarded([&] {
        std::vector<orc::Group<S>> gs(static_cast<std::size_t>(ng));
        for (int i = 0; i < ng; ++i)
            gs[std::size_t(i)] = { names[i], flags[2 * i], flags[2 * i + 1], p[i], g[i], m[i],
                                   v[i], std::size_t(n[i]) };
        orc::Hyper h;
        h.lr = hyper[0];
        h.beta1 = hyper[1];
        h.beta2 = hyper[2];
        h.eps = hyper[3];
        h.l2 = hyper[4];
        const std::string e = orc::adam_step<S>(*step, gs.data(), ng, h, lr_now);
        if (!e.empty())
            throw std::runtime_error(e);
    });
}

struct FieldHandle {
    orc::Field f;
};

struct RngHandle {
    orc::Pcg r;
};
}   // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

void orc_set_threads(int n)
{
#ifdef _OPENMP
    omp_set_num_threads(n < 1 ? 1 : n);
#else
    (void)n;
#endif
}

int orc_max_threads()
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

// ---- grid ---------------------------------------------------------------
double orc_growth_factor(const int* gc) { return orc::growth(grid_cfg(gc)); }

// Writes L entries into each output array; returns total rows or -1.
std::int64_t orc_levels(const int* gc, std::uint32_t* res, std::uint32_t* len, int* dense,
                        std::uint64_t* row_off)
{
    std::int64_t total = -1;
    const int st = guarded([&] {
        const auto lv = orc::levels(grid_cfg(gc));
        for (std::size_t l = 0; l < lv.size(); ++l) {
            res[l] = lv[l].res;
            len[l] = lv[l].len;
            dense[l] = lv[l].dense;
            row_off[l] = lv[l].row_off;
        }
        total = std::int64_t(orc::total_rows(lv));
    });
    return st ? -1 : total;
}

std::uint32_t orc_hash(const std::uint32_t* c, int d, std::uint32_t T) { return orc::hash(c, d, T); }

std::uint32_t orc_vertex_index(std::uint32_t res, int dense, const std::uint32_t* c, int d,
                               std::uint32_t T)
{
    orc::Level lv;
    lv.res = res;
    lv.dense = dense;
    return orc::vertex_index(lv, c, d, T);
}

double orc_smoothstep_d(double x) { return orc::smoothstep(x); }
void orc_weights_d(const double* frac, int d, int smooth, double* w) { orc::corner_weights(frac, d, smooth, w); }
void orc_weights_f(const float* frac, int d, int smooth, float* w) { orc::corner_weights(frac, d, smooth, w); }

void orc_voxel_f(float x, std::uint32_t res, int half, std::uint32_t* corner, float* frac)
{
    orc::voxel<float>(x, res, half != 0, *corner, *frac);
}

int orc_encode_fwd_f(const int* gc, const float* params, const float* X, std::int64_t B, float* Y,
                     std::uint32_t* rows, float* wts)
{
    return encode_fwd_impl<float>(gc, params, X, B, Y, rows, wts);
}
int orc_encode_fwd_d(const int* gc, const double* params, const double* X, std::int64_t B,
                     double* Y, std::uint32_t* rows, double* wts)
{
    return encode_fwd_impl<double>(gc, params, X, B, Y, rows, wts);
}
int orc_encode_bwd_f(const int* gc, const std::uint32_t* rows, const float* wts, std::int64_t B,
                     const float* dY, float* grads)
{
    return encode_bwd_impl<float>(gc, rows, wts, B, dY, grads);
}
int orc_encode_bwd_d(const int* gc, const std::uint32_t* rows, const double* wts, std::int64_t B,
                     const double* dY, double* grads)
{
    return encode_bwd_impl<double>(gc, rows, wts, B, dY, grads);
}

void orc_init_tables_f(std::uint64_t seed, float mag, float* p, std::uint64_t n) { orc::init_tables<float>(seed, mag, p, n); }
void orc_init_tables_d(std::uint64_t seed, double mag, double* p, std::uint64_t n) { orc::init_tables<double>(seed, mag, p, n); }

// ---- mlp ----------------------------------------------------------------
int orc_glorot_f(const int* mc, std::uint64_t seed, float* W, float* b)
{
    return guarded([&] { orc::glorot<float>(mlp_cfg(mc), seed, W, b); });
}
int orc_glorot_d(const int* mc, std::uint64_t seed, double* W, double* b)
{
    return guarded([&] { orc::glorot<double>(mlp_cfg(mc), seed, W, b); });
}
// Forward, and backward too when dOut != NULL (grads accumulate).
int orc_mlp_f(const int* mc, const float* W, const float* b, const float* Y, std::int64_t B,
              float* out, const float* dOut, float* gW, float* gb, float* dY)
{
    return mlp_impl<float>(mc, W, b, Y, B, out, dOut, gW, gb, dY);
}
int orc_mlp_d(const int* mc, const double* W, const double* b, const double* Y, std::int64_t B,
              double* out, const double* dOut, double* gW, double* gb, double* dY)
{
    return mlp_impl<double>(mc, W, b, Y, B, out, dOut, gW, gb, dY);
}

// ---- losses -------------------------------------------------------------
float orc_loss_f(int kind, const float* p, const float* t, std::int64_t n, float* dp)
{
    return orc::loss_with_grad<float>(kind, p, t, n, dp);
}
double orc_loss_d(int kind, const double* p, const double* t, std::int64_t n, double* dp)
{
    return orc::loss_with_grad<double>(kind, p, t, n, dp);
}
double orc_psnr_f(const float* a, const float* b, std::int64_t n) { return orc::psnr(a, b, n); }

// ---- adam ---------------------------------------------------------------
int orc_adam_f(std::uint64_t* step, int ng, const int* flags, float* const* p, float* const* g,
               float* const* m, float* const* v, const std::uint64_t* n, const char* const* names,
               const double* hyper, float lr_now)
{
    return adam_impl<float>(step, ng, flags, p, g, m, v, n, names, hyper, lr_now);
}
int orc_adam_d(std::uint64_t* step, int ng, const int* flags, double* const* p, double* const* g,
               double* const* m, double* const* v, const std::uint64_t* n, const char* const* names,
               const double* hyper, double lr_now)
{
    return adam_impl<double>(step, ng, flags, p, g, m, v, n, names, hyper, lr_now);
}
double orc_lr_at(const std::int64_t* ms, int n, double factor, double base, std::int64_t step)
{
    return orc::lr_at(std::vector<std::int64_t>(ms, ms + n), factor, base, step);
}
int orc_default_milestones(std::int64_t total, std::int64_t* out, int cap)
{
    const auto ms = orc::default_milestones(total);
    for (std::size_t i = 0; i < ms.size() && int(i) < cap; ++i)
        out[i] = ms[i];
    return int(ms.size());
}

// ---- field model ----------------------------------------------------------
void* orc_field_create(const int* gc, const int* mc, const double* hyper)
{
    void* out = nullptr;
    guarded([&] {
        auto* h = new FieldHandle{ orc::Field(grid_cfg(gc), mlp_cfg(mc)) };
        h->f.h.lr = hyper[0];
        h->f.h.beta1 = hyper[1];
        h->f.h.beta2 = hyper[2];
        h->f.h.eps = hyper[3];
        h->f.h.l2 = hyper[4];
        out = h;
    });
    return out;
}
void orc_field_destroy(void* h) { delete static_cast<FieldHandle*>(h); }
void orc_field_init(void* h, std::uint64_t seed) { static_cast<FieldHandle*>(h)->f.init(seed); }
void orc_field_set_schedule(void* h, const std::int64_t* ms, int n, double factor)
{
    auto& f = static_cast<FieldHandle*>(h)->f;
    f.milestones.assign(ms, ms + n);
    f.factor = factor;
}
// which: 0 params, 1 grads, 2 m, 3 v. Returns the live buffer; *n = size.
float* orc_field_buffer(void* h, int which, std::uint64_t* n)
{
    auto& f = static_cast<FieldHandle*>(h)->f;
    *n = f.size();
    switch (which) {
    case 0: return f.p.data();
    case 1: return f.grad.data();
    case 2: return f.mom.data();
    default: return f.vel.data();
    }
}
void orc_field_sizes(void* h, std::uint64_t* out3)
{
    auto& f = static_cast<FieldHandle*>(h)->f;
    out3[0] = f.n_tab;
    out3[1] = f.n_w;
    out3[2] = f.n_b;
}
std::uint64_t orc_field_step(void* h) { return static_cast<FieldHandle*>(h)->f.step; }
void orc_field_set_step(void* h, std::uint64_t s) { static_cast<FieldHandle*>(h)->f.step = s; }
int orc_field_train_step(void* h, const float* X, const float* target, std::int64_t B, int kind,
                         std::int64_t step, float* loss, float* pred)
{
    return guarded([&] {
        auto& f = static_cast<FieldHandle*>(h)->f;
        if (const char* e = orc::check_inputs<float>(f.g, X, B))
            throw std::invalid_argument(e);
        *loss = f.train_step(X, target, B, kind, step, pred);
    });
}
int orc_field_evaluate(void* h, const float* X, std::int64_t B, float* out)
{
    return guarded([&] {
        auto& f = static_cast<FieldHandle*>(h)->f;
        if (const char* e = orc::check_inputs<float>(f.g, X, B))
            throw std::invalid_argument(e);
        f.evaluate(X, B, out);
    });
}
void orc_field_times(void* h, double* out6)
{
    const auto& t = static_cast<FieldHandle*>(h)->f.times;
    out6[0] = t.encode_fwd;
    out6[1] = t.mlp_fwd;
    out6[2] = t.loss;
    out6[3] = t.mlp_bwd;
    out6[4] = t.encode_bwd;
    out6[5] = t.adam;
}
void orc_field_reset_times(void* h) { static_cast<FieldHandle*>(h)->f.times = orc::PhaseTimes{}; }
// CPU-baseline timing only: route the MLP through the blocked FMA GEMMs (fast::).
void orc_field_set_fast_mlp(void* h, int on) { static_cast<FieldHandle*>(h)->f.fast_mlp = on != 0; }

// ---- rng / fixtures -----------------------------------------------------
void* orc_rng_create(std::uint64_t seed, std::uint64_t seq) { return new RngHandle{ orc::Pcg(seed, seq) }; }
void orc_rng_destroy(void* h) { delete static_cast<RngHandle*>(h); }
std::uint32_t orc_rng_u32(void* h) { return static_cast<RngHandle*>(h)->r.u32(); }
std::uint32_t orc_rng_below(void* h, std::uint32_t bound) { return static_cast<RngHandle*>(h)->r.below(bound); }
float orc_rng_f32(void* h) { return static_cast<RngHandle*>(h)->r.f32(); }
double orc_rng_f64(void* h) { return static_cast<RngHandle*>(h)->r.f64(); }
void orc_rng_fill_f32(void* h, float* out, std::int64_t n)
{
    auto& r = static_cast<RngHandle*>(h)->r;
    for (std::int64_t i = 0; i < n; ++i)
        out[i] = r.f32();
}
void orc_rng_fill_f64(void* h, double* out, std::int64_t n)
{
    auto& r = static_cast<RngHandle*>(h)->r;
    for (std::int64_t i = 0; i < n; ++i)
        out[i] = r.f64();
}
void orc_rng_fill_u32(void* h, std::uint32_t* out, std::int64_t n)
{
    auto& r = static_cast<RngHandle*>(h)->r;
    for (std::int64_t i = 0; i < n; ++i)
        out[i] = r.u32();
}

// Image batch exactly as fit_image draws it (tasks.cpp:114-120): pixel
// p = below(w*h); x = ((p % w) + 0.5)/w, y = ((p / w) + 0.5)/h; target = rgb(:, p).
void orc_image_batch(void* h, const float* rgb, int w, int hgt, std::int64_t B, float* X,
                     float* target)
{
    auto& r = static_cast<RngHandle*>(h)->r;
    const std::uint32_t n = std::uint32_t(w) * std::uint32_t(hgt);
    for (std::int64_t i = 0; i < B; ++i) {
        const std::size_t p = r.below(n);
        X[2 * i + 0] = (float(p % std::size_t(w)) + 0.5f) / float(w);
        X[2 * i + 1] = (float(p / std::size_t(w)) + 0.5f) / float(hgt);
        for (int c = 0; c < 3; ++c)
            target[3 * i + c] = rgb[3 * p + std::size_t(c)];
    }
}

void orc_make_test_image(int w, int h, float* rgb) { orc::make_test_image(w, h, rgb); }

void orc_csg_sdf(const float* X, std::int64_t B, float* out)
{
    for (std::int64_t i = 0; i < B; ++i)
        out[i] = orc::csg_sdf<float>(X[3 * i], X[3 * i + 1], X[3 * i + 2]);
}

}   // extern "C"
