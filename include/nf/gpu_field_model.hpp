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
#include <fstream>
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

// nf::FieldModel (model.hpp:21-63) with device-resident state. Set the
// config members, then init(seed), exactly like the reference.
template <class GridCfg, class MlpCfg, class Hyper, class Schedule>
class FieldModelT {
public:
    GridCfg hash_cfg;
    MlpCfg mlp_cfg;
    Hyper hyper;
    Schedule schedule;
    nfg_options options{ 0, 1, 0, 0 };

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
        M out;
        out.resize(mlp_cfg.output_width, X.cols());
        check(nfg_field_evaluate(f_, X.data(), X.cols(), out.data()));
        return out;
    }

    // model.cpp:111-138.
    template <class M>
    float train_step(const M& X, const M& target, int loss_kind, std::int64_t step)
    {
        if (X.rows() != hash_cfg.dims)
            throw std::invalid_argument("encode_forward: input dimensionality mismatch");
        if (target.rows() != mlp_cfg.output_width || target.cols() != X.cols())
            throw std::invalid_argument("l2_loss: shape mismatch");
        push_run_config();   // hyper / schedule are public members (test_tasks.cpp:313-314)
        float loss = 0.0f;
        check(nfg_field_train_step(f_, X.data(), target.data(), X.cols(), loss_kind, step, &loss));
        return loss;
    }

    // Host mirrors of the flat [tables | W | b] parameters and Adam state.
    std::vector<float> read(int which) const
    {
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
