// host_init.cpp — host-side pieces of the model that must be bit-identical to
// the reference: the level table (grid.hpp:66-84), PCG32 (pcg32.hpp:9-66), the
// table init (grid.hpp:158-164), Glorot init (mlp.hpp:74-94), lr_at
// (adam.hpp:139-146) and the Adam bias corrections (adam.hpp:92-96).
// Compiled by g++ with -ffp-contract=off so float expressions round exactly as
// the reference's scalar code does. Runs once per init; never on the hot path.
#include "host_init.h"

#include <cmath>
#include <stdexcept>

namespace nfg {
namespace host {

namespace {
struct Pcg32 {
    uint64_t s = 0, inc = 0;
    Pcg32(uint64_t seed, uint64_t seq) : s(0), inc((seq << 1u) | 1u)
    {
        next();
        s += seed;
        next();
    }
    uint32_t next()
    {
        const uint64_t old = s;
        s = old * 6364136223846793005ULL + inc;
        const uint32_t x = uint32_t(((old >> 18u) ^ old) >> 27u);
        const uint32_t r = uint32_t(old >> 59u);
        return (x >> r) | (x << ((32u - r) & 31u));
    }
    float unit() { return float(next() >> 8) * 0x1p-24f; }
    float uniform(float lo, float hi) { return lo + (hi - lo) * unit(); }
};
}   // namespace

void validate(const nfg_grid_config& c)
{
    if (c.levels < 1)
        throw std::invalid_argument("HashEncodingConfig: levels must be >= 1");
    if (c.table_size == 0 || (c.table_size & (c.table_size - 1)) != 0)
        throw std::invalid_argument("HashEncodingConfig: table_size must be a power of two");
    if (c.features < 1)
        throw std::invalid_argument("HashEncodingConfig: features must be >= 1");
    if (c.n_min < 1 || c.n_max < c.n_min)
        throw std::invalid_argument("HashEncodingConfig: need 1 <= n_min <= n_max");
    if (c.dims != 2 && c.dims != 3)
        throw std::invalid_argument("HashEncodingConfig: dims must be 2 or 3");
}

void validate(const nfg_mlp_config& c)
{
    if (c.input_width < 1 || c.output_width < 1 || c.hidden_width < 1 || c.hidden_layers < 0)
        throw std::invalid_argument("MlpConfig: widths must be >= 1 and hidden_layers >= 0");
}

void validate(const nfg_adam_hyper& h)
{
    if (!(h.lr > 0) || !(h.eps > 0) || h.beta1 < 0 || h.beta1 >= 1 || h.beta2 < 0 || h.beta2 >= 1)
        throw std::invalid_argument("AdamHyper: invalid hyperparameters");
}

double growth_factor(const nfg_grid_config& c)
{
    if (c.levels < 2 || c.n_min == c.n_max)
        return 1.0;
    return std::exp((std::log(double(c.n_max)) - std::log(double(c.n_min))) / double(c.levels - 1));
}

std::vector<nfg_level_spec> level_resolutions(const nfg_grid_config& c)
{
    validate(c);
    const double lb = c.levels < 2 ? 0.0 : std::log(growth_factor(c));
    std::vector<nfg_level_spec> out(size_t(c.levels));
    uint64_t off = 0;
    for (int l = 0; l < c.levels; ++l) {
        nfg_level_spec& s = out[size_t(l)];
        s.level = l;
        s.resolution = uint32_t(std::floor(double(c.n_min) * std::exp(double(l) * lb) + 1e-6));
        uint64_t verts = 1;
        for (int i = 0; i < c.dims; ++i)
            verts *= uint64_t(s.resolution) + 1;
        s.dense = verts <= c.table_size;
        s.table_len = s.dense ? uint32_t(verts) : c.table_size;
        s.row_offset = off;
        off += s.table_len;
    }
    return out;
}

uint32_t spatial_hash(const uint32_t* c, int d, uint32_t T)
{
    static const uint32_t pi[3] = { 1u, 2654435761u, 805459861u };
    uint32_t h = 0;
    for (int i = 0; i < d; ++i)
        h ^= c[i] * pi[i];
    return h & (T - 1u);
}

void init_tables(uint64_t seed, float* p, uint64_t n)
{
    Pcg32 rng(seed, 0xfeedu);
    const float mag = 1e-4f;
    for (uint64_t i = 0; i < n; ++i)
        p[i] = rng.uniform(-mag, mag);
}

void glorot(const nfg_mlp_config& c, uint64_t seed, float* W, float* b)
{
    validate(c);
    Pcg32 rng(seed, 0x91u);
    int in = c.input_width;
    size_t boff = 0;
    for (int k = 0; k <= c.hidden_layers; ++k) {
        const int out = k < c.hidden_layers ? c.hidden_width : c.output_width;
        const float bound = std::sqrt(6.0f / float(in + out));
        for (size_t i = 0; i < size_t(in) * size_t(out); ++i)
            *W++ = rng.uniform(-bound, bound);
        for (int o = 0; o < out; ++o)
            b[boff + size_t(o)] = 0.0f;
        boff += size_t(out);
        in = out;
    }
}

double lr_at(const std::vector<int64_t>& ms, double factor, double base, int64_t step)
{
    int hits = 0;
    for (int64_t m : ms)
        if (m <= step)
            ++hits;
    return base * std::pow(factor, hits);
}

AdamScalars adam_scalars(const nfg_adam_hyper& h, uint64_t step_after, float lr_now)
{
    AdamScalars a;
    a.b1 = float(h.beta1);
    a.b2 = float(h.beta2);
    a.omb1 = 1.0f - a.b1;
    a.omb2 = 1.0f - a.b2;
    a.bc1 = 1.0f - std::pow(a.b1, float(step_after));
    a.bc2 = 1.0f - std::pow(a.b2, float(step_after));
    a.eps = float(h.eps);
    a.l2 = float(h.l2);
    a.lr = lr_now;
    return a;
}

}   // namespace host
}   // namespace nfg
