// gpu_field_model.hpp — C++ drop-in for the reference's float hot path
// (nf::FieldModel, encode_forward/encode_backward, mlp_forward/mlp_backward,
// loss_with_grad, adam_step; /root/reference/proj/include/nf/*.hpp) backed by
// the sm_100a C ABI in include/nfg.h.
//
// Header-only and matrix-type agnostic: any column-major matrix type with
// rows(), cols(), data() and resize(rows, cols) works — Eigen::MatrixXf (the
// reference's MatX<float>) or the minimal nf::gpu::Mat below. Config structs
// are read by member name, so the reference's own HashEncodingConfig /
// MlpConfig / AdamHyper / LrSchedule can be passed unchanged.
//
// Exceptions mirror the reference: std::invalid_argument (NFG_EINVAL),
// std::runtime_error (non-finite gradient in adam_step), std::logic_error.
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../nfg.h"

namespace nf {
namespace gpu {

inline void check(nfg_status st)
{
    if (st == NFG_OK)
        return;
    const std::string msg = nfg_last_error();
    switch (st) {
    case NFG_EINVAL: throw std::invalid_argument(msg);
    case NFG_ENONFINITE: throw std::runtime_error(msg);
    case NFG_ELOGIC: throw std::logic_error(msg);
    case NFG_EUNSUPPORTED: throw std::invalid_argument("unsupported on sm_100a: " + msg);
    default: throw std::runtime_error(msg);
    }
}

// Minimal column-major float matrix (stand-in for Eigen::MatrixXf).
struct Mat {
    long r = 0, c = 0;
    std::vector<float> v;
    Mat() = default;
    Mat(long rows, long cols, float fill = 0.0f) : r(rows), c(cols), v(size_t(rows * cols), fill) {}
    long rows() const { return r; }
    long cols() const { return c; }
    float* data() { return v.data(); }
    const float* data() const { return v.data(); }
    void resize(long rows, long cols)
    {
        r = rows;
        c = cols;
        v.resize(size_t(rows * cols));
    }
    float& operator()(long i, long j) { return v[size_t(i + j * r)]; }
    float operator()(long i, long j) const { return v[size_t(i + j * r)]; }
};

template <class Cfg>
nfg_grid_config to_c_grid(const Cfg& c)
{
    return nfg_grid_config{ int32_t(c.levels), uint32_t(c.table_size), int32_t(c.features), int32_t(c.n_min),
                            int32_t(c.n_max), int32_t(c.dims), int32_t(c.interpolation) };
}

template <class Cfg>
nfg_mlp_config to_c_mlp(const Cfg& c)
{
    return nfg_mlp_config{ int32_t(c.input_width), int32_t(c.hidden_layers), int32_t(c.hidden_width),
                           int32_t(c.output_width), int32_t(c.output_activation) };
}

template <class H>
nfg_adam_hyper to_c_hyper(const H& h)
{
    return nfg_adam_hyper{ double(h.lr), double(h.beta1), double(h.beta2), double(h.eps), double(h.l2) };
}

class Context {
public:
    explicit Context(int device = 0) { check(nfg_ctx_create(device, &h_)); }
    ~Context() { nfg_ctx_destroy(h_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    nfg_ctx* get() const { return h_; }
    void synchronize() { check(nfg_ctx_synchronize(h_)); }

private:
    nfg_ctx* h_ = nullptr;
};

// Host mirrors of the reference's parameter containers. The device copy is
// the source of truth; FieldModelT::sync_to_host() / sync_to_device() move
// them (automatically around every call when auto_mirror is set).

// FeatureTables (grid.hpp:138-179): per level a features x table_len matrix
// (row-contiguous features), the level specs and the gradient mirror.
template <class Matrix = Mat>
struct FeatureTables {
    nfg_grid_config cfg{};
    std::vector<nfg_level_spec> levels;
    std::vector<Matrix> values;
    std::vector<Matrix> grads;

    std::size_t parameter_count() const
    {
        std::size_t n = 0;
        for (const auto& v : values)
            n += std::size_t(v.rows()) * std::size_t(v.cols());
        return n;
    }
    void zero_grads()
    {
        for (auto& g : grads)
            std::fill(g.data(), g.data() + g.rows() * g.cols(), 0.0f);
    }
};

// MlpParams (mlp.hpp:42-60): W_k (out x in, column-major) and b_k (out x 1).
template <class Matrix = Mat>
struct MlpParams {
    std::vector<Matrix> weights;
    std::vector<Matrix> biases;
};

// EncodeCache (grid.hpp:183-195): rows and weights shaped (level, point,
// corner). The GPU backward recomputes them from the inputs, which the cache
// therefore also keeps.
struct EncodeCache {
    int batch = 0, corners = 0, levels = 0, dims = 0;
    std::vector<std::uint32_t> rows;
    std::vector<float> weights;
    std::vector<float> X;
    std::size_t offset(int level, int point) const { return (std::size_t(level) * batch + point) * corners; }
};

// AdamState (adam.hpp:56-73): step and per-group moment vectors.
struct AdamState {
    std::uint64_t step = 0;
    std::vector<std::vector<float>> m, v;
};

// ParamGroup (adam.hpp:27-54) without the spans (the parameters are on the
// device): name, flags and size, in the reference's group order.
struct GroupFlags {
    bool apply_l2 = false;
    bool skip_zero_grad = false;
};
struct ParamGroup {
    std::string name;
    GroupFlags flags;
    std::size_t size = 0;
    std::size_t total_size() const { return size; }
};

namespace detail {

inline std::vector<nfg_level_spec> level_specs(const nfg_grid_config& g)
{
    std::vector<nfg_level_spec> v(size_t(std::max(g.levels, 0)));
    const int32_t n = nfg_level_resolutions(&g, v.data(), int32_t(v.size()));
    if (n < 0)
        throw std::invalid_argument(nfg_last_error());
    v.resize(size_t(n));
    return v;
}

// A device field used as the engine of the free component functions on
// host-held tables (one per thread and grid config; the MLP is unused).
struct ScratchField {
    nfg_grid_config cfg{};
    nfg_field* f = nullptr;
    ~ScratchField()
    {
        if (f)
            nfg_field_destroy(f);
    }
};

inline Context& default_context()
{
    static Context ctx(0);
    return ctx;
}

inline nfg_field* scratch_field(const nfg_grid_config& g)
{
    thread_local std::vector<std::unique_ptr<ScratchField>> cache;
    for (auto& s : cache)
        if (std::memcmp(&s->cfg, &g, sizeof(g)) == 0)
            return s->f;
    auto s = std::make_unique<ScratchField>();
    s->cfg = g;
    const nfg_mlp_config m{ g.levels * g.features, 1, 64, 1, NFG_ACT_LINEAR };
    const nfg_adam_hyper h{ 1e-2, 0.9, 0.99, 1e-15, 1e-6 };
    const nfg_options o{ 1, 1, 0, 0 };   // fp32 tables: the reference's values exactly
    check(nfg_field_create(default_context().get(), &g, &m, &h, &o, &s->f));
    cache.push_back(std::move(s));
    return cache.back()->f;
}

template <class Matrix>
void push_tables(nfg_field* f, const FeatureTables<Matrix>& t)
{
    std::uint64_t off = 0;
    for (const auto& v : t.values) {
        const std::uint64_t n = std::uint64_t(v.rows()) * std::uint64_t(v.cols());
        check(nfg_field_write(f, NFG_BUF_PARAMS, off, n, v.data()));
        off += n;
    }
}

}   // namespace detail

// encode_forward (grid.hpp:219-272) on host-held tables: Y is (L*F) x B; the
// cache receives the reference's rows / weights (and the inputs).
template <class Matrix>
void encode_forward(const FeatureTables<Matrix>& tables, const Matrix& X, Matrix& Y, EncodeCache& cache)
{
    if (X.rows() != tables.cfg.dims)
        throw std::invalid_argument("encode_forward: input dimensionality mismatch");
    nfg_field* f = detail::scratch_field(tables.cfg);
    detail::push_tables(f, tables);
    const long B = X.cols();
    const int L = tables.cfg.levels, corners = 1 << tables.cfg.dims;
    Y.resize(L * tables.cfg.features, B);
    cache.batch = int(B);
    cache.corners = corners;
    cache.levels = L;
    cache.dims = tables.cfg.dims;
    cache.rows.resize(size_t(L) * size_t(B) * size_t(corners));
    cache.weights.resize(cache.rows.size());
    cache.X.assign(X.data(), X.data() + X.rows() * X.cols());
    check(nfg_encode_forward(f, X.data(), B, Y.data(), cache.rows.data(), cache.weights.data()));
}

// encode_backward (grid.hpp:277-295): accumulates dLoss/dTables into tables.grads.
template <class Matrix>
void encode_backward(FeatureTables<Matrix>& tables, const EncodeCache& cache, const Matrix& dY)
{
    if (dY.rows() != tables.cfg.levels * tables.cfg.features || dY.cols() != cache.batch)
        throw std::invalid_argument("encode_backward: shape mismatch");
    nfg_field* f = detail::scratch_field(tables.cfg);
    detail::push_tables(f, tables);
    const std::uint64_t n = tables.parameter_count();
    std::vector<float> g(n, 0.0f);
    check(nfg_field_write(f, NFG_BUF_GRADS, 0, n, g.data()));
    check(nfg_encode_backward(f, cache.X.data(), cache.batch, dY.data()));
    check(nfg_field_read(f, NFG_BUF_GRADS, 0, n, g.data()));
    std::size_t off = 0;
    for (auto& gr : tables.grads) {
        float* d = gr.data();
        const std::size_t m = std::size_t(gr.rows()) * std::size_t(gr.cols());
        for (std::size_t i = 0; i < m; ++i)
            d[i] += g[off + i];
        off += m;
    }
}

// nf::FieldModel (model.hpp:21-63) with device-resident state. Set the
// config members, then init(seed), exactly like the reference.
template <class GridCfg, class MlpCfg, class Hyper, class Schedule, class Matrix = Mat>
class FieldModelT {
public:
    GridCfg hash_cfg;
    MlpCfg mlp_cfg;
    Hyper hyper;
    Schedule schedule;
    nfg_options options{ 0, 1, 0, 0 };
    // Public parameter members of the reference (model.hpp:30-34) as host
    // mirrors: filled by init() and sync_to_host(), pushed by sync_to_device().
    // With auto_mirror = true, train_step / evaluate push them before and
    // refresh them after every call, so code that pokes the members directly
    // (acceptance.cpp:340,359; test_tasks.cpp:31-33) runs unchanged — at the
    // cost of a full parameter copy per call (off by default).
    FeatureTables<Matrix> tables;
    MlpParams<Matrix> mlp;
    bool auto_mirror = false;

    explicit FieldModelT(Context& ctx) : ctx_(ctx) {}
    ~FieldModelT()
    {
        if (f_)
            nfg_field_destroy(f_);
    }
    FieldModelT(const FieldModelT&) = delete;
    FieldModelT& operator=(const FieldModelT&) = delete;

    // model.cpp:23-37
    void init(std::uint64_t seed)
    {
        if (f_)
            nfg_field_destroy(f_);
        f_ = nullptr;
        mlp_cfg.input_width = hash_cfg.levels * hash_cfg.features;   // model.cpp:101
        const nfg_grid_config g = to_c_grid(hash_cfg);
        const nfg_mlp_config m = to_c_mlp(mlp_cfg);
        const nfg_adam_hyper h = to_c_hyper(hyper);
        check(nfg_field_create(ctx_.get(), &g, &m, &h, &options, &f_));
        check(nfg_field_init(f_, seed));
        push_run_config();
        sync_to_host();
    }

    // Device parameters -> tables / mlp mirrors (and table gradients).
    void sync_to_host()
    {
        const nfg_grid_config g = to_c_grid(hash_cfg);
        tables.cfg = g;
        tables.levels = detail::level_specs(g);
        const std::vector<float> p = read(NFG_BUF_PARAMS), gr = read(NFG_BUF_GRADS);
        std::size_t off = 0;
        tables.values.clear();
        tables.grads.clear();
        for (const auto& l : tables.levels) {
            tables.values.emplace_back(g.features, long(l.table_len));
            tables.grads.emplace_back(g.features, long(l.table_len));
            const std::size_t n = std::size_t(g.features) * l.table_len;
            std::copy(p.begin() + long(off), p.begin() + long(off + n), tables.values.back().data());
            std::copy(gr.begin() + long(off), gr.begin() + long(off + n), tables.grads.back().data());
            off += n;
        }
        mlp.weights.clear();
        mlp.biases.clear();
        int in = encoded_width();
        std::size_t boff = off;
        for (int k = 0; k <= mlp_cfg.hidden_layers; ++k)
            boff += std::size_t(k < mlp_cfg.hidden_layers ? mlp_cfg.hidden_width : mlp_cfg.output_width) *
                    std::size_t(k == 0 ? in : mlp_cfg.hidden_width);
        for (int k = 0; k <= mlp_cfg.hidden_layers; ++k) {
            const int out = k < mlp_cfg.hidden_layers ? mlp_cfg.hidden_width : mlp_cfg.output_width;
            mlp.weights.emplace_back(out, in);
            std::copy(p.begin() + long(off), p.begin() + long(off + std::size_t(out) * in), mlp.weights.back().data());
            off += std::size_t(out) * in;
            mlp.biases.emplace_back(out, 1);
            std::copy(p.begin() + long(boff), p.begin() + long(boff + out), mlp.biases.back().data());
            boff += out;
            in = out;
        }
    }

    // tables / mlp mirrors -> device parameters (the fp16 table shadow follows).
    void sync_to_device()
    {
        std::vector<float> p;
        p.reserve(parameter_count());
        for (const auto& v : tables.values)
            p.insert(p.end(), v.data(), v.data() + v.rows() * v.cols());
        for (const auto& w : mlp.weights)
            p.insert(p.end(), w.data(), w.data() + w.rows() * w.cols());
        for (const auto& b : mlp.biases)
            p.insert(p.end(), b.data(), b.data() + b.rows() * b.cols());
        if (p.size() != parameter_count())
            throw std::invalid_argument("sync_to_device: mirror shapes do not match the model");
        write(NFG_BUF_PARAMS, p);
    }

    // AdamState (adam.hpp:56-73): step and per-group m / v in group order.
    AdamState adam_state() const
    {
        AdamState st;
        st.step = adam_step_count();
        const std::vector<float> m = read(NFG_BUF_ADAM_M), v = read(NFG_BUF_ADAM_V);
        std::size_t off = 0;
        for (const auto& g : param_groups()) {
            st.m.emplace_back(m.begin() + long(off), m.begin() + long(off + g.size));
            st.v.emplace_back(v.begin() + long(off), v.begin() + long(off + g.size));
            off += g.size;
        }
        return st;
    }

    // The three groups of model.cpp:49-77 (tables: skip-zero; MLP weights: L2; biases).
    std::vector<ParamGroup> param_groups() const
    {
        std::uint64_t sz[3];
        check(nfg_field_sizes(f_, sz));
        return { ParamGroup{ "tables", GroupFlags{ false, true }, std::size_t(sz[0]) },
                 ParamGroup{ "mlp_weights", GroupFlags{ true, false }, std::size_t(sz[1]) },
                 ParamGroup{ "mlp_biases", GroupFlags{ false, false }, std::size_t(sz[2]) } };
    }

    int encoded_width() const { return hash_cfg.levels * hash_cfg.features; }

    std::size_t parameter_count() const
    {
        std::uint64_t s[3];
        check(nfg_field_sizes(f_, s));
        return std::size_t(s[0] + s[1] + s[2]);
    }

    // model.cpp:102-109. X is dims x B column-major.
    template <class M>
    M evaluate(const M& X) const
    {
        if (auto_mirror)   // the mirrors are logically part of the model's state
            const_cast<FieldModelT*>(this)->sync_to_device();
        M out;
        out.resize(mlp_cfg.output_width, X.cols());
        check(nfg_field_evaluate(f_, X.data(), X.cols(), out.data()));
        return out;
    }

    // model.cpp:111-138. `loss` is the reference's nf::LossKind (or an int /
    // nfg_loss_kind with the same values, model.hpp:17).
    template <class M, class LossKindT>
    float train_step(const M& X, const M& target, LossKindT loss, std::int64_t step)
    {
        const int loss_kind = static_cast<int>(loss);
        if (auto_mirror)
            sync_to_device();
        if (X.rows() != hash_cfg.dims)
            throw std::invalid_argument("encode_forward: input dimensionality mismatch");
        if (target.rows() != mlp_cfg.output_width || target.cols() != X.cols())
            throw std::invalid_argument("l2_loss: shape mismatch");
        push_run_config();   // hyper / schedule are public members (test_tasks.cpp:313-314)
        float loss_value = 0.0f;
        check(nfg_field_train_step(f_, X.data(), target.data(), X.cols(), loss_kind, step, &loss_value));
        if (auto_mirror)
            sync_to_host();
        return loss_value;
    }

    // Host mirrors of the flat [tables | W | b] parameters and Adam state.
    std::vector<float> read(int which) const
    {
        if (!f_)
            throw std::logic_error("FieldModel: init() first");
        std::vector<float> v(parameter_count());
        check(nfg_field_read(f_, which, 0, v.size(), v.data()));
        return v;
    }
    void write(int which, const std::vector<float>& v) { check(nfg_field_write(f_, which, 0, v.size(), v.data())); }
    std::uint64_t adam_step_count() const
    {
        std::uint64_t s = 0;
        check(nfg_field_get_step(f_, &s));
        return s;
    }

    // Components on this model's tables / MLP.
    template <class M>
    void encode_forward(const M& X, M& Y) const
    {
        Y.resize(encoded_width(), X.cols());
        check(nfg_encode_forward(f_, X.data(), X.cols(), Y.data(), nullptr, nullptr));
    }
    template <class M>
    void encode_backward(const M& X, const M& dY)
    {
        check(nfg_encode_backward(f_, X.data(), X.cols(), dY.data()));
    }
    template <class M>
    void mlp_forward(const M& Y, M& out) const
    {
        out.resize(mlp_cfg.output_width, Y.cols());
        check(nfg_mlp_forward(f_, Y.data(), Y.cols(), out.data()));
    }
    template <class M>
    void mlp_backward(const M& Y, const M& dOut, M& dY)
    {
        dY.resize(encoded_width(), Y.cols());
        check(nfg_mlp_backward(f_, Y.data(), Y.cols(), dOut.data(), dY.data()));
    }
    void adam_step(float lr_now) { check(nfg_adam_step(f_, lr_now)); }

    nfg_field* handle() const { return f_; }

    // save_checkpoint / load_checkpoint (io.cpp:222-351), NFC1 bytes. load
    // replaces hash_cfg / mlp_cfg with the file's and keeps hyper / schedule /
    // options (re-supplied by the caller on resume, test_tasks.cpp:313-315).
    void save_checkpoint(const std::string& path) const { check(nfg_field_save(f_, path.c_str())); }
    void load_checkpoint(const std::string& path)
    {
        const nfg_adam_hyper h = to_c_hyper(hyper);
        nfg_field* nf_ = nullptr;
        check(nfg_field_load(ctx_.get(), path.c_str(), &h, &options, &nf_));
        adopt(nf_);
    }

    // Takes ownership of a field created by the C ABI (nfg_fit_image, load).
    void adopt(nfg_field* f)
    {
        if (f_)
            nfg_field_destroy(f_);
        f_ = f;
        nfg_grid_config g{};
        nfg_mlp_config m{};
        check(nfg_field_get_config(f_, &g, &m));
        hash_cfg.levels = g.levels;
        hash_cfg.table_size = g.table_size;
        hash_cfg.features = g.features;
        hash_cfg.n_min = g.n_min;
        hash_cfg.n_max = g.n_max;
        hash_cfg.dims = g.dims;
        hash_cfg.interpolation = decltype(hash_cfg.interpolation)(g.interpolation);
        mlp_cfg.input_width = m.input_width;
        mlp_cfg.hidden_layers = m.hidden_layers;
        mlp_cfg.hidden_width = m.hidden_width;
        mlp_cfg.output_width = m.output_width;
        mlp_cfg.output_activation = decltype(mlp_cfg.output_activation)(m.output_activation);
        push_run_config();
        sync_to_host();
    }

private:
    void push_run_config()
    {
        const nfg_adam_hyper h = to_c_hyper(hyper);
        check(nfg_field_set_hyper(f_, &h));
        std::vector<std::int64_t> ms(schedule.milestones.begin(), schedule.milestones.end());
        check(nfg_field_set_schedule(f_, ms.data(), int32_t(ms.size()), double(schedule.factor)));
    }

    Context& ctx_;
    nfg_field* f_ = nullptr;
};

// loss_with_grad (model.cpp:140-149) on the GPU.
template <class M>
float loss_with_grad(Context& ctx, int kind, const M& pred, const M& target, M& dPred)
{
    if (pred.rows() != target.rows() || pred.cols() != target.cols())
        throw std::invalid_argument("loss: shape mismatch");
    dPred.resize(pred.rows(), pred.cols());
    const std::int64_t n = std::int64_t(pred.rows()) * pred.cols();
    float loss = 0.0f;
    check(nfg_loss(ctx.get(), kind, pred.data(), target.data(), n, n, dPred.data(), &loss));
    return loss;
}

// TrainReport CSV (io.cpp:189-220), the reference's exact schema.
struct ReportRow {
    std::int64_t step = 0;
    double time_s = 0, loss = 0, metric = 0, lr = 0;
};

inline void write_report_csv(const std::vector<ReportRow>& rows, const std::string& path)
{
    std::ofstream out(path);
    if (!out)
        throw std::runtime_error("cannot write report: " + path);
    out << "step,time_s,loss,metric,lr\n";
    out.precision(10);
    for (const auto& r : rows)
        out << r.step << ',' << r.time_s << ',' << r.loss << ',' << r.metric << ',' << r.lr << '\n';
}

inline std::vector<ReportRow> read_report_csv(const std::string& path)
{
    std::ifstream in(path);
    if (!in)
        throw std::runtime_error("cannot read report: " + path);
    std::vector<ReportRow> rows;
    std::string line;
    std::getline(in, line);
    while (std::getline(in, line)) {
        if (line.empty())
            continue;
        ReportRow r;
        char comma;
        std::istringstream ss(line);
        ss >> r.step >> comma >> r.time_s >> comma >> r.loss >> comma >> r.metric >> comma >> r.lr;
        rows.push_back(r);
    }
    return rows;
}

// fit_image (tasks.cpp:49-131) with every step on the device. `rgb` is the
// reference's Image::rgb (3 x w*h column-major); Task reads ImageTask by member
// name (cfg, interpolation, hidden_layers, hidden_width, batch_size,
// total_steps, log_interval, lr, lr_decay). The trained field is adopted by
// `model`; returns the report rows.
template <class Task, class Model>
std::vector<ReportRow> fit_image(Context& ctx, const Task& task, const float* rgb, int width, int height,
                                 std::uint64_t seed, Model& model)
{
    nfg_image_task t{};
    t.width = width;
    t.height = height;
    t.cfg = to_c_grid(task.cfg);
    t.cfg.interpolation = int32_t(task.interpolation);
    t.hidden_layers = task.hidden_layers;
    t.hidden_width = task.hidden_width;
    t.batch_size = task.batch_size;
    t.total_steps = task.total_steps;
    t.log_interval = task.log_interval;
    t.lr = task.lr;
    t.lr_decay = task.lr_decay;
    const std::int64_t cap = task.total_steps / std::max<std::int64_t>(task.log_interval, 1) + 2;
    std::vector<nfg_report_row> rows(static_cast<size_t>(cap));
    std::int64_t n = 0;
    nfg_field* f = nullptr;
    check(nfg_fit_image(ctx.get(), &t, rgb, seed, &model.options, &f, rows.data(), cap, &n));
    model.hyper.lr = task.lr;
    model.schedule.milestones.clear();
    {   // default_schedule (adam.hpp:150-161)
        std::int64_t next = std::int64_t(0.65 * double(task.total_steps));
        const std::int64_t stride = std::int64_t(0.30 * double(task.total_steps));
        while (next < task.total_steps && stride > 0) {
            model.schedule.milestones.push_back(next);
            next += stride;
        }
        model.schedule.factor = task.lr_decay;
    }
    model.adopt(f);
    std::vector<ReportRow> out;
    for (std::int64_t i = 0; i < std::min(n, cap); ++i)
        out.push_back(ReportRow{ rows[size_t(i)].step, rows[size_t(i)].time_s, rows[size_t(i)].loss,
                                 rows[size_t(i)].metric, rows[size_t(i)].lr });
    return out;
}

}   // namespace gpu
}   // namespace nf
