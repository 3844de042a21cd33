// nf_oracle.hpp — CPU restatement of the reference hot path.
//
// TEST INFRASTRUCTURE ONLY. This file is the parity oracle and the CPU
// baseline for the B200 build. Nothing in the product path
// (paper_2201_05989_b200/, include/) includes, links or calls it; only
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg do.
//
// The reference (/root/reference/proj, C++20 + Eigen 3) cannot be compiled in
// this container (Eigen, libpng, doctest and CLI11 are absent),
// so this is a restatement of its algorithm on plain arrays. Every function
// cites the reference file:line it follows. Parity is pinned by the
// reference's own known-answer tests (tests/golden/reference_kats.json and
// tests/test_oracle_*.py), not by running the reference itself.
//
// Conventions (all identical to the reference's Eigen column-major storage):
//   * X is d x B column-major: X[s*d + i] is coordinate i of sample s.
//   * Y is (L*F) x B column-major: Y[s*L*F + l*F + f].
//   * Table parameters are one flat array in the reference's param-group order
//     (model.cpp:117-125): level 0 rows, level 1 rows, ...; row r of level l
//     holds its F features contiguously at (row_offset[l] + r)*F.
//   * MLP weights W_k are out x in column-major: W_k[o + i*out] (mlp.hpp:45).
//
// Build with -ffp-contract=off: vertex selection, interpolation weights and
// Adam are bit-exact only without FMA contraction.
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace orc {

// ---------------------------------------------------------------------------
// PCG32 XSH-RR 64/32 — reference pcg32.hpp:9-66.
// ---------------------------------------------------------------------------
struct Pcg {
    std::uint64_t s = 0, inc = 0;
    Pcg(std::uint64_t seed, std::uint64_t seq)   // pcg32.hpp:11-18
    {
        s = 0;
        inc = (seq << 1) | 1u;
        u32();
        s += seed;
        u32();
    }
    std::uint32_t u32()   // pcg32.hpp:20-27
    {
        const std::uint64_t o = s;
        s = o * 6364136223846793005ULL + inc;
        const std::uint32_t xs = std::uint32_t(((o >> 18) ^ o) >> 27);
        const std::uint32_t r = std::uint32_t(o >> 59);
        return (xs >> r) | (xs << ((32u - r) & 31u));
    }
    std::uint32_t below(std::uint32_t bound)   // pcg32.hpp:30-38 (rejection)
    {
        const std::uint32_t th = (0u - bound) % bound;
        for (;;) {
            const std::uint32_t r = u32();
            if (r >= th)
                return r % bound;
        }
    }
    float f32() { return float(u32() >> 8) * 0x1p-24f; }   // pcg32.hpp:41-44
    double f64()   // pcg32.hpp:46-51
    {
        const std::uint64_t hi = u32();
        const std::uint64_t lo = u32();
        return double((hi << 21) ^ lo) * 0x1p-53;
    }
    template <class S> S uni(S lo, S hi)   // pcg32.hpp:54-61
    {
        if (sizeof(S) > 4)
            return lo + (hi - lo) * S(f64());
        return lo + (hi - lo) * S(f32());
    }
};

// ---------------------------------------------------------------------------
// Grid configuration and level table — grid.hpp:25-84.
// ---------------------------------------------------------------------------
struct GridCfg {
    int L = 16;
    std::uint32_t T = 1u << 14;
    int F = 2;
    int nmin = 16;
    int nmax = 512;
    int d = 3;
    int smooth = 0;   // 0 linear, 1 smoothstep (grid.hpp:20)
};

inline void validate(const GridCfg& c)   // grid.hpp:34-46
{
    if (c.L < 1)
        throw std::invalid_argument("HashEncodingConfig: levels must be >= 1");
    if (c.T == 0 || (c.T & (c.T - 1)) != 0)
        throw std::invalid_argument("HashEncodingConfig: table_size must be a power of two");
    if (c.F < 1)
        throw std::invalid_argument("HashEncodingConfig: features must be >= 1");
    if (c.nmin < 1 || c.nmax < c.nmin)
        throw std::invalid_argument("HashEncodingConfig: need 1 <= n_min <= n_max");
    if (c.d != 2 && c.d != 3)
        throw std::invalid_argument("HashEncodingConfig: dims must be 2 or 3");
}

inline double growth(const GridCfg& c)   // grid.hpp:49-54
{
    if (c.L < 2 || c.nmin == c.nmax)
        return 1.0;
    return std::exp((std::log(double(c.nmax)) - std::log(double(c.nmin))) / double(c.L - 1));
}

struct Level {
    std::uint32_t res = 0;   // N_l
    std::uint32_t len = 0;   // rows
    int dense = 0;
    std::uint64_t row_off = 0;   // first row of this level in the flat table
};

inline std::vector<Level> levels(const GridCfg& c)   // grid.hpp:66-84
{
    validate(c);
    const double lb = c.L < 2 ? 0.0 : std::log(growth(c));
    std::vector<Level> out(std::size_t(c.L));
    std::uint64_t off = 0;
    for (int l = 0; l < c.L; ++l) {
        Level& v = out[std::size_t(l)];
        v.res = std::uint32_t(std::floor(double(c.nmin) * std::exp(double(l) * lb) + 1e-6));
        std::uint64_t n = 1;
        for (int i = 0; i < c.d; ++i)
            n *= std::uint64_t(v.res) + 1;
        v.dense = n <= c.T;
        v.len = v.dense ? std::uint32_t(n) : c.T;
        v.row_off = off;
        off += v.len;
    }
    return out;
}

inline std::uint64_t total_rows(const std::vector<Level>& lv)
{
    return lv.empty() ? 0 : lv.back().row_off + lv.back().len;
}

// Spatial hash: per-dimension wrapping u32 products XOR'd, masked by T-1
// (grid.hpp:88-95).
inline std::uint32_t hash(const std::uint32_t* c, int d, std::uint32_t T)
{
    const std::uint32_t pi[3] = { 1u, 2654435761u, 805459861u };
    std::uint32_t h = 0;
    for (int i = 0; i < d; ++i)
        h ^= c[i] * pi[i];
    return h & (T - 1u);
}

// Dense row-major index (first coordinate fastest) or hash (grid.hpp:100-110).
inline std::uint32_t vertex_index(const Level& lv, const std::uint32_t* c, int d, std::uint32_t T)
{
    if (!lv.dense)
        return hash(c, d, T);
    const std::uint32_t stride = lv.res + 1;
    std::uint32_t idx = c[d - 1];
    for (int i = d - 2; i >= 0; --i)
        idx = idx * stride + c[i];
    return idx;
}

template <class S> S smoothstep(S x) { return x * x * (S(3) - S(2) * x); }   // grid.hpp:112-116

// Corner weights; corner c takes the high side in dim i iff bit i is set
// (grid.hpp:120-133). Product order: w = ((1*a0)*a1)*a2.
template <class S> void corner_weights(const S* frac, int d, int smooth, S* w)
{
    S t[3];
    for (int i = 0; i < d; ++i)
        t[i] = smooth ? smoothstep(frac[i]) : frac[i];
    for (int c = 0; c < (1 << d); ++c) {
        S p = S(1);
        for (int i = 0; i < d; ++i)
            p *= ((c >> i) & 1) ? t[i] : S(1) - t[i];
        w[c] = p;
    }
}

// Clamp to [0, 1-2^-20], scale by N_l, optional half-voxel offset in
// smoothstep mode (grid.hpp:199-212).
template <class S> void voxel(S x, std::uint32_t res, bool half, std::uint32_t& corner, S& frac)
{
    const S n = S(res);
    S p = std::min(std::max(x, S(0)), S(1) - S(0x1p-20)) * n;
    if (half)
        p = std::min(p + S(0.5), n * (S(1) - S(0x1p-20)));
    const S f = std::floor(p);
    corner = std::uint32_t(f);
    frac = p - f;
}

// Input validation of encode_forward (grid.hpp:224-229). Returns an error
// string or nullptr.
template <class S> const char* check_inputs(const GridCfg& c, const S* X, std::int64_t B)
{
    for (std::int64_t i = 0; i < B * c.d; ++i)
        if (!std::isfinite(X[i]))
            return "encode_forward: non-finite input";
    for (std::int64_t i = 0; i < B * c.d; ++i)
        if (X[i] < S(-1e-6) || X[i] > S(1) + S(1e-6))
            return "encode_forward: input outside [0,1]^d";
    return nullptr;
}

// Forward encoding (grid.hpp:219-272): level-outer, points in parallel,
// Y slice = sum over corners in corner order of w_c * row. rows/wts (the
// EncodeCache, layout (level, point, corner), grid.hpp:183-195) are optional.
template <class S>
void encode_fwd(const GridCfg& c, const std::vector<Level>& lv, const S* params, const S* X,
                std::int64_t B, S* Y, std::uint32_t* rows, S* wts)
{
    const int d = c.d, F = c.F, nc = 1 << d, LF = c.L * c.F;
    for (int l = 0; l < c.L; ++l) {
        const Level& v = lv[std::size_t(l)];
        const S* table = params + v.row_off * std::uint64_t(F);
#pragma omp parallel for schedule(static)
        for (std::int64_t p = 0; p < B; ++p) {
            std::uint32_t base[3];
            S frac[3], w[8];
            for (int i = 0; i < d; ++i)
                voxel<S>(X[p * d + i], v.res, c.smooth != 0, base[i], frac[i]);
            corner_weights<S>(frac, d, c.smooth, w);
            S* out = Y + p * LF + l * F;
            for (int f = 0; f < F; ++f)
                out[f] = S(0);
            const std::size_t co = (std::size_t(l) * std::size_t(B) + std::size_t(p)) * nc;
            for (int k = 0; k < nc; ++k) {
                std::uint32_t cc[3];
                for (int i = 0; i < d; ++i)
                    cc[i] = base[i] + ((k >> i) & 1u);
                const std::uint32_t r = vertex_index(v, cc, d, c.T);
                if (rows)
                    rows[co + k] = r;
                if (wts)
                    wts[co + k] = w[k];
                const S* row = table + std::uint64_t(r) * F;
                for (int f = 0; f < F; ++f)
                    out[f] += w[k] * row[f];
            }
        }
    }
}

// Backward scatter (grid.hpp:277-295): single-threaded, fixed order
// level -> point -> corner; accumulates into grads (same layout as params).
template <class S>
void encode_bwd(const GridCfg& c, const std::vector<Level>& lv, const std::uint32_t* rows,
                const S* wts, std::int64_t B, const S* dY, S* grads)
{
    const int F = c.F, nc = 1 << c.d, LF = c.L * c.F;
    for (int l = 0; l < c.L; ++l) {
        S* g = grads + lv[std::size_t(l)].row_off * std::uint64_t(F);
        for (std::int64_t p = 0; p < B; ++p) {
            const S* gy = dY + p * LF + l * F;
            const std::size_t co = (std::size_t(l) * std::size_t(B) + std::size_t(p)) * nc;
            for (int k = 0; k < nc; ++k) {
                S* row = g + std::uint64_t(rows[co + k]) * F;
                for (int f = 0; f < F; ++f)
                    row[f] += wts[co + k] * gy[f];
            }
        }
    }
}

// Table init: Pcg(seed, 0xfeed), U(-m, m) sequential over the flat order
// (grid.hpp:158-164).
template <class S> void init_tables(std::uint64_t seed, S mag, S* params, std::uint64_t n)
{
    Pcg rng(seed, 0xfeedu);
    for (std::uint64_t i = 0; i < n; ++i)
        params[i] = rng.uni<S>(-mag, mag);
}

// ---------------------------------------------------------------------------
// MLP — mlp.hpp:13-158.
// ---------------------------------------------------------------------------
struct MlpCfg {
    int in = 32, hidden_layers = 2, width = 64, out = 3;
    int sigmoid = 0;   // OutputActivation (mlp.hpp:13)
    int layers() const { return hidden_layers + 1; }
    int in_of(int k) const { return k == 0 ? in : width; }
    int out_of(int k) const { return k < hidden_layers ? width : out; }
    std::size_t weight_count() const
    {
        std::size_t n = 0;
        for (int k = 0; k < layers(); ++k)
            n += std::size_t(in_of(k)) * out_of(k);
        return n;
    }
    std::size_t bias_count() const
    {
        std::size_t n = 0;
        for (int k = 0; k < layers(); ++k)
            n += std::size_t(out_of(k));
        return n;
    }
};

inline void validate(const MlpCfg& c)   // mlp.hpp:22-26
{
    if (c.in < 1 || c.out < 1 || c.width < 1 || c.hidden_layers < 0)
        throw std::invalid_argument("MlpConfig: widths must be >= 1 and hidden_layers >= 0");
}

// Flat MLP parameters in param-group order: [W_0 .. W_n] then [b_0 .. b_n]
// (model.cpp:132-143). Offsets of each layer inside the two blocks:
struct MlpLayout {
    std::vector<std::size_t> w_off, b_off;
    std::size_t n_w = 0, n_b = 0;
    explicit MlpLayout(const MlpCfg& c)
    {
        for (int k = 0; k < c.layers(); ++k) {
            w_off.push_back(n_w);
            n_w += std::size_t(c.in_of(k)) * c.out_of(k);
        }
        for (int k = 0; k < c.layers(); ++k) {
            b_off.push_back(n_b);
            n_b += std::size_t(c.out_of(k));
        }
    }
};

// Glorot uniform: Pcg(seed, 0x91), bound sqrt(6/(in+out)) per layer, biases 0
// (mlp.hpp:74-94). W points at the weight block, b at the bias block.
template <class S> void glorot(const MlpCfg& c, std::uint64_t seed, S* W, S* b)
{
    validate(c);
    Pcg rng(seed, 0x91u);
    MlpLayout lay(c);
    for (int k = 0; k < c.layers(); ++k) {
        const int in = c.in_of(k), out = c.out_of(k);
        const S bound = std::sqrt(S(6) / S(in + out));
        S* w = W + lay.w_off[std::size_t(k)];
        for (std::size_t i = 0; i < std::size_t(in) * out; ++i)
            w[i] = rng.uni<S>(-bound, bound);
        for (int o = 0; o < out; ++o)
            b[lay.b_off[std::size_t(k)] + std::size_t(o)] = S(0);
    }
}

// acts[k] is the input of layer k (width in_of(k) x B); acts.back() is the
// post-activation output (mlp.hpp:96-124).
template <class S> struct MlpCache {
    std::vector<std::vector<S>> acts;
};

// z(:, s) = W * a(:, s) + b, vectorised over the output dimension (column-major
// W), samples in parallel. The reference uses an Eigen GEMM here; its
// summation order is not reproducible, so MLP values are tolerance-level.
template <class S>
void dense(const S* W, const S* b, const S* A, std::int64_t B, int in, int out, S* Z)
{
#pragma omp parallel for schedule(static)
    for (std::int64_t s = 0; s < B; ++s) {
        S* z = Z + s * out;
        const S* a = A + s * in;
        for (int o = 0; o < out; ++o)
            z[o] = S(0);
        for (int i = 0; i < in; ++i) {
            const S ai = a[i];
            const S* wc = W + std::size_t(i) * out;
            for (int o = 0; o < out; ++o)
                z[o] += wc[o] * ai;
        }
        for (int o = 0; o < out; ++o)
            z[o] += b[o];
    }
}

template <class S>
void mlp_fwd(const MlpCfg& c, const S* W, const S* b, const S* Y, std::int64_t B, S* out,
             MlpCache<S>& cache)
{
    MlpLayout lay(c);
    const int n = c.layers();
    cache.acts.assign(1, std::vector<S>(Y, Y + B * c.in));   // mlp.hpp:111
    std::vector<S> z;
    for (int k = 0; k < n; ++k) {
        const int in = c.in_of(k), o = c.out_of(k);
        z.assign(std::size_t(B) * o, S(0));
        dense<S>(W + lay.w_off[std::size_t(k)], b + lay.b_off[std::size_t(k)],
                 cache.acts.back().data(), B, in, o, z.data());
        if (k + 1 < n) {   // ReLU on hidden layers (mlp.hpp:115-118)
            for (auto& v : z)
                v = std::max(v, S(0));
            cache.acts.push_back(z);
        }
    }
    if (c.sigmoid)   // mlp.hpp:120-121
        for (auto& v : z)
            v = S(1) / (S(1) + std::exp(-v));
    cache.acts.push_back(z);
    std::copy(z.begin(), z.end(), out);
}

// Reverse pass (mlp.hpp:129-158). Accumulates (+=) into gW/gb; writes dY.
template <class S>
void mlp_bwd(const MlpCfg& c, const S* W, const MlpCache<S>& cache, const S* dOut, std::int64_t B,
             S* gW, S* gb, S* dY)
{
    MlpLayout lay(c);
    const int n = c.layers();
    const std::vector<S>& outp = cache.acts.back();
    std::vector<S> dz(dOut, dOut + B * c.out);
    if (c.sigmoid)   // mlp.hpp:140-142
        for (std::size_t i = 0; i < dz.size(); ++i)
            dz[i] = dz[i] * (outp[i] * (S(1) - outp[i]));
    for (int k = n - 1; k >= 0; --k) {
        const int in = c.in_of(k), o = c.out_of(k);
        const S* A = cache.acts[std::size_t(k)].data();
        const S* w = W + lay.w_off[std::size_t(k)];
        S* gw = gW + lay.w_off[std::size_t(k)];
        S* gbk = gb + lay.b_off[std::size_t(k)];
        // gW_k += dz * A_k^T; gb_k += rowsum(dz)   (mlp.hpp:147-148)
#pragma omp parallel for schedule(static)
        for (int i = 0; i < in; ++i)
            for (std::int64_t s = 0; s < B; ++s) {
                const S a = A[s * in + i];
                for (int q = 0; q < o; ++q)
                    gw[q + std::size_t(i) * o] += dz[std::size_t(s) * o + q] * a;
            }
        for (std::int64_t s = 0; s < B; ++s)
            for (int q = 0; q < o; ++q)
                gbk[q] += dz[std::size_t(s) * o + q];
        // da = W_k^T dz   (mlp.hpp:149)
        std::vector<S> da(std::size_t(B) * in, S(0));
#pragma omp parallel for schedule(static)
        for (std::int64_t s = 0; s < B; ++s)
            for (int i = 0; i < in; ++i) {
                S acc = S(0);
                for (int q = 0; q < o; ++q)
                    acc += w[q + std::size_t(i) * o] * dz[std::size_t(s) * o + q];
                da[std::size_t(s) * in + i] = acc;
            }
        if (k == 0) {
            std::copy(da.begin(), da.end(), dY);
        } else {   // ReLU mask from the cached post-ReLU input (mlp.hpp:153-155)
            for (std::size_t i = 0; i < da.size(); ++i)
                da[i] = A[i] > S(0) ? da[i] : S(0);
            dz.swap(da);
        }
    }
}

// ---------------------------------------------------------------------------
// Throughput stand-in for the reference's Eigen GEMMs (mlp.hpp:114,147-149),
// used ONLY by the CPU-baseline timing (Field::fast_mlp; bench.py's
// cpu_baseline / --impl reference legs). Same math, cache-blocked over
// 8-sample panels with FMA contraction (the reference builds with
// -O2 -march=native, proj/CMakeLists.txt:9, where Eigen issues FMAs); the
// parity oracle above keeps its fixed summation order. fp32 only.
// ---------------------------------------------------------------------------
#pragma GCC push_options
#pragma GCC optimize("O3", "fp-contract=fast")
namespace fast {

typedef float v8 __attribute__((vector_size(32)));

inline v8 ld8(const float* p)
{
    v8 v;
    std::memcpy(&v, p, sizeof(v));
    return v;
}
inline void st8(float* p, v8 v) { std::memcpy(p, &v, sizeof(v)); }
inline v8 bc8(float x) { return v8{ x, x, x, x, x, x, x, x }; }

// C[m][n] (+)= sum_k A[m*lda + k] * Bm[k*ldb + n] for a 6 x 16 block (BLIS-style
// register tile: 12 accumulators, two B vectors, one broadcast per row).
inline void kernel_6x16(int K, const float* A, std::int64_t lda, const float* Bm, std::int64_t ldb, float* C,
                        std::int64_t ldc, int mrows, bool accumulate)
{
    v8 c[6][2];
    for (int r = 0; r < 6; ++r)
        for (int v = 0; v < 2; ++v)
            c[r][v] = (accumulate && r < mrows) ? ld8(C + r * ldc + 8 * v) : bc8(0.0f);
    for (int k = 0; k < K; ++k) {
        const v8 b0 = ld8(Bm + k * ldb), b1 = ld8(Bm + k * ldb + 8);
        for (int r = 0; r < 6; ++r) {
            const v8 a = bc8(r < mrows ? A[r * lda + k] : 0.0f);
            c[r][0] += a * b0;
            c[r][1] += a * b1;
        }
    }
    for (int r = 0; r < mrows; ++r)
        for (int v = 0; v < 2; ++v)
            st8(C + r * ldc + 8 * v, c[r][v]);
}

// Z (B x out, sample-major) = A (B x in) W^T + b; Wt is W^T (in x out, out-contiguous
// = the reference's column-major W itself).
inline void dense(const float* W, const float* b, const float* A, std::int64_t B, int in, int out, float* Z)
{
    const int n16 = out / 16 * 16;
#pragma omp parallel for schedule(static)
    for (std::int64_t s0 = 0; s0 < B; s0 += 6) {
        const int ms = int(std::min<std::int64_t>(6, B - s0));
        for (int o0 = 0; o0 < n16; o0 += 16)
            kernel_6x16(in, A + s0 * in, in, W + o0, out, Z + s0 * out + o0, out, ms, false);
        for (int r = 0; r < ms; ++r) {
            float* z = Z + (s0 + r) * out;
            for (int o = n16; o < out; ++o) {
                float acc = 0.0f;
                for (int i = 0; i < in; ++i)
                    acc += A[(s0 + r) * in + i] * W[std::size_t(i) * out + o];
                z[o] = acc;
            }
            for (int o = 0; o < out; ++o)
                z[o] += b[o];
        }
    }
}

inline void mlp_fwd(const MlpCfg& c, const float* W, const float* b, const float* Y, std::int64_t B, float* out,
                    MlpCache<float>& cache)
{
    MlpLayout lay(c);
    const int n = c.layers();
    cache.acts.assign(1, std::vector<float>(Y, Y + B * c.in));
    std::vector<float> z;
    for (int k = 0; k < n; ++k) {
        const int in = c.in_of(k), o = c.out_of(k);
        z.resize(std::size_t(B) * o);
        dense(W + lay.w_off[std::size_t(k)], b + lay.b_off[std::size_t(k)], cache.acts.back().data(), B, in, o,
              z.data());
        if (k + 1 < n) {
            for (auto& v : z)
                v = std::max(v, 0.0f);
            cache.acts.push_back(z);
        }
    }
    if (c.sigmoid)
        for (auto& v : z)
            v = 1.0f / (1.0f + std::exp(-v));
    cache.acts.push_back(z);
    std::copy(z.begin(), z.end(), out);
}

inline void mlp_bwd(const MlpCfg& c, const float* W, const MlpCache<float>& cache, const float* dOut,
                    std::int64_t B, float* gW, float* gb, float* dY)
{
    MlpLayout lay(c);
    const int n = c.layers();
    const std::vector<float>& outp = cache.acts.back();
    std::vector<float> dz(dOut, dOut + B * c.out);
    if (c.sigmoid)
        for (std::size_t i = 0; i < dz.size(); ++i)
            dz[i] = dz[i] * (outp[i] * (1.0f - outp[i]));
    for (int k = n - 1; k >= 0; --k) {
        const int in = c.in_of(k), o = c.out_of(k);
        const float* A = cache.acts[std::size_t(k)].data();
        const float* w = W + lay.w_off[std::size_t(k)];
        float* gw = gW + lay.w_off[std::size_t(k)];
        float* gbk = gb + lay.b_off[std::size_t(k)];
        // W^T copy (in-contiguous rows per output) for da = dz W
        std::vector<float> wt(std::size_t(in) * o);
        for (int i = 0; i < in; ++i)
            for (int q = 0; q < o; ++q)
                wt[std::size_t(q) * in + i] = w[q + std::size_t(i) * o];
        std::vector<float> da(std::size_t(B) * in);
        const int nt = omp_get_max_threads();
        std::vector<float> part(std::size_t(nt) * (std::size_t(in) * o + o), 0.0f);
        const bool wide = o % 16 == 0;
#pragma omp parallel
        {
            const int tid = omp_get_thread_num();
            float* pg = part.data() + std::size_t(tid) * (std::size_t(in) * o + o);
            float* pb = pg + std::size_t(in) * o;
            const std::int64_t chunk = (B + nt - 1) / nt, lo = std::min<std::int64_t>(B, tid * chunk),
                               hi = std::min<std::int64_t>(B, lo + chunk);
            // gW^T (in x o) += A^T dz over this thread's samples: M = in, N = o, K = samples
            if (wide) {
                std::vector<float> at(std::size_t(in) * 256);
                for (std::int64_t s0 = lo; s0 < hi; s0 += 256) {
                    const int ks = int(std::min<std::int64_t>(256, hi - s0));
                    for (int r = 0; r < ks; ++r)   // transpose the panel: at[i][r]
                        for (int i = 0; i < in; ++i)
                            at[std::size_t(i) * 256 + r] = A[(s0 + r) * in + i];
                    for (int i0 = 0; i0 < in; i0 += 6)
                        for (int q0 = 0; q0 < o; q0 += 16)
                            kernel_6x16(ks, at.data() + std::size_t(i0) * 256, 256, dz.data() + s0 * o + q0, o,
                                        pg + std::size_t(i0) * o + q0, o, std::min(6, in - i0), true);
                }
            } else {
                for (std::int64_t s = lo; s < hi; ++s)
                    for (int i = 0; i < in; ++i) {
                        const float a = A[s * in + i];
                        for (int q = 0; q < o; ++q)
                            pg[std::size_t(i) * o + q] += dz[std::size_t(s) * o + q] * a;
                    }
            }
            for (std::int64_t s = lo; s < hi; ++s)
                for (int q = 0; q < o; ++q)
                    pb[q] += dz[std::size_t(s) * o + q];
            // da (B x in) = dz (B x o) W (o x in): B-operand = wt (o x in, in-contiguous)
            for (std::int64_t s0 = lo; s0 < hi; s0 += 6) {
                const int ms = int(std::min<std::int64_t>(6, hi - s0));
                if (in % 16 == 0) {
                    for (int i0 = 0; i0 < in; i0 += 16)
                        kernel_6x16(o, dz.data() + s0 * o, o, wt.data() + i0, in, da.data() + s0 * in + i0, in, ms,
                                    false);
                } else {
                    for (int r = 0; r < ms; ++r)
                        for (int i = 0; i < in; ++i) {
                            float acc = 0.0f;
                            for (int q = 0; q < o; ++q)
                                acc += dz[std::size_t(s0 + r) * o + q] * wt[std::size_t(q) * in + i];
                            da[std::size_t(s0 + r) * in + i] = acc;
                        }
                }
            }
        }
        for (int t = 0; t < nt; ++t) {
            const float* pg = part.data() + std::size_t(t) * (std::size_t(in) * o + o);
            for (std::size_t e = 0; e < std::size_t(in) * o; ++e)
                gw[e] += pg[e];
            for (int q = 0; q < o; ++q)
                gbk[q] += pg[std::size_t(in) * o + q];
        }
        if (k == 0) {
            std::copy(da.begin(), da.end(), dY);
        } else {
            for (std::size_t i = 0; i < da.size(); ++i)
                da[i] = A[i] > 0.0f ? da[i] : 0.0f;
            dz.swap(da);
        }
    }
}

}   // namespace fast
#pragma GCC pop_options

// ---------------------------------------------------------------------------
// Losses — losses.hpp:10-71. n = pred.size() (count over all outputs).
// ---------------------------------------------------------------------------
enum LossKind { L2 = 0, MAPE = 1, REL_L2 = 2 };

template <class S> S l2_loss(const S* p, const S* t, std::int64_t n, S* dp)   // losses.hpp:10-20
{
    const S count = S(n);
    S sq = S(0);
    for (std::int64_t i = 0; i < n; ++i) {
        const S diff = p[i] - t[i];
        dp[i] = (S(2) / count) * diff;
        sq += diff * diff;
    }
    return sq / count;
}

template <class S> S mape_loss(const S* p, const S* t, std::int64_t n, S* dp)   // losses.hpp:24-40
{
    const S count = S(n);
    S loss = S(0);
    for (std::int64_t i = 0; i < n; ++i) {
        const S den = std::abs(t[i]) + S(0.01);
        const S diff = p[i] - t[i];
        loss += std::abs(diff) / den;
        const S sg = diff > 0 ? S(1) : (diff < 0 ? S(-1) : S(0));
        dp[i] = sg / den / count;
    }
    return loss / count;
}

template <class S> S rel_l2_loss(const S* p, const S* t, std::int64_t n, S* dp)   // losses.hpp:44-59
{
    const S count = S(n);
    S loss = S(0);
    for (std::int64_t i = 0; i < n; ++i) {
        const S den = p[i] * p[i] + S(0.01);
        const S diff = p[i] - t[i];
        loss += diff * diff / den;
        dp[i] = S(2) * diff / den / count;
    }
    return loss / count;
}

template <class S> S loss_with_grad(int kind, const S* p, const S* t, std::int64_t n, S* dp)
{   // model.cpp:140-149
    switch (kind) {
    case L2: return l2_loss(p, t, n, dp);
    case MAPE: return mape_loss(p, t, n, dp);
    case REL_L2: return rel_l2_loss(p, t, n, dp);
    }
    throw std::logic_error("loss_with_grad: unknown loss");
}

template <class S> double psnr(const S* a, const S* b, std::int64_t n)   // losses.hpp:62-71
{
    double sq = 0;
    for (std::int64_t i = 0; i < n; ++i) {
        const double d = double(a[i]) - double(b[i]);
        sq += d * d;
    }
    const double mse = sq / double(n);
    if (mse <= 0)
        return 100.0;
    return std::min(100.0, -10.0 * std::log10(mse));
}

// ---------------------------------------------------------------------------
// Adam — adam.hpp:13-161.
// ---------------------------------------------------------------------------
struct Hyper {
    double lr = 1e-2, beta1 = 0.9, beta2 = 0.99, eps = 1e-15, l2 = 1e-6;
};

inline void validate(const Hyper& h)   // adam.hpp:20-24
{
    if (!(h.lr > 0) || !(h.eps > 0) || h.beta1 < 0 || h.beta1 >= 1 || h.beta2 < 0 || h.beta2 >= 1)
        throw std::invalid_argument("AdamHyper: invalid hyperparameters");
}

// One contiguous group: params/grads/m/v of length n (the reference's
// per-group concatenation of spans, adam.hpp:62-72,99-117).
template <class S> struct Group {
    const char* name;
    int apply_l2, skip_zero;
    S* p;
    S* g;
    S* m;
    S* v;
    std::size_t n;
};

// Returns nullptr or the error message (thrown by the reference as
// std::runtime_error, adam.hpp:86-90).
template <class S>
std::string adam_step(std::uint64_t& step, Group<S>* groups, int ng, const Hyper& h, S lr_now)
{
    validate(h);
    for (int gi = 0; gi < ng; ++gi)
        for (std::size_t i = 0; i < groups[gi].n; ++i)
            if (!std::isfinite(groups[gi].g[i]))
                return std::string("adam_step: non-finite gradient in group '") + groups[gi].name + "'";
    step += 1;
    const S b1 = S(h.beta1), b2 = S(h.beta2);
    const S bc1 = S(1) - std::pow(b1, S(step));
    const S bc2 = S(1) - std::pow(b2, S(step));
    const S eps = S(h.eps);
    for (int gi = 0; gi < ng; ++gi) {
        Group<S>& G = groups[gi];
        for (std::size_t i = 0; i < G.n; ++i) {
            S g = G.g[i];
            if (G.skip_zero && g == S(0))
                continue;
            if (G.apply_l2)
                g += S(h.l2) * G.p[i];
            G.m[i] = b1 * G.m[i] + (S(1) - b1) * g;
            G.v[i] = b2 * G.v[i] + (S(1) - b2) * g * g;
            G.p[i] -= lr_now * (G.m[i] / bc1) / (std::sqrt(G.v[i] / bc2) + eps);
        }
        for (std::size_t i = 0; i < G.n; ++i)
            G.g[i] = S(0);
    }
    return std::string();
}

inline double lr_at(const std::vector<std::int64_t>& milestones, double factor, double base,
                    std::int64_t step)   // adam.hpp:139-146
{
    int hits = 0;
    for (std::int64_t m : milestones)
        if (m <= step)
            ++hits;
    return base * std::pow(factor, hits);
}

inline std::vector<std::int64_t> default_milestones(std::int64_t total)   // adam.hpp:150-161
{
    std::vector<std::int64_t> ms;
    std::int64_t next = std::int64_t(0.65 * double(total));
    const std::int64_t stride = std::int64_t(0.30 * double(total));
    while (next < total && stride > 0) {
        ms.push_back(next);
        next += stride;
    }
    return ms;
}

// ---------------------------------------------------------------------------
// FieldModel (hash encoder) — model.hpp:21-63, model.cpp:23-149.
// Parameters, grads, m and v are each one flat vector in param-group order:
// [tables | MLP weights | MLP biases] (model.cpp:117-143).
// ---------------------------------------------------------------------------
struct PhaseTimes {
    double encode_fwd = 0, mlp_fwd = 0, loss = 0, mlp_bwd = 0, encode_bwd = 0, adam = 0;
};

struct Field {
    GridCfg g;
    MlpCfg m;
    Hyper h;
    std::vector<std::int64_t> milestones;
    double factor = 0.33;
    std::vector<Level> lv;
    std::size_t n_tab = 0, n_w = 0, n_b = 0;
    std::vector<float> p, grad, mom, vel;
    std::uint64_t step = 0;
    PhaseTimes times;
    bool fast_mlp = false;   // CPU-baseline timing only: the MLP through fast:: (Eigen stand-in)

    Field(const GridCfg& gc, const MlpCfg& mc) : g(gc), m(mc)
    {
        lv = levels(g);
        m.in = g.L * g.F;   // model.cpp:101
        validate(m);
        n_tab = std::size_t(total_rows(lv)) * std::size_t(g.F);
        MlpLayout lay(m);
        n_w = lay.n_w;
        n_b = lay.n_b;
        p.assign(size(), 0.f);
        grad.assign(size(), 0.f);
        mom.assign(size(), 0.f);
        vel.assign(size(), 0.f);
    }
    std::size_t size() const { return n_tab + n_w + n_b; }
    float* W() { return p.data() + n_tab; }
    float* b() { return p.data() + n_tab + n_w; }

    void init(std::uint64_t seed)   // model.cpp:23-37
    {
        init_tables<float>(seed, 1e-4f, p.data(), n_tab);
        glorot<float>(m, seed + 1, W(), b());
        std::fill(grad.begin(), grad.end(), 0.f);
        std::fill(mom.begin(), mom.end(), 0.f);
        std::fill(vel.begin(), vel.end(), 0.f);
        step = 0;
    }

    void evaluate(const float* X, std::int64_t B, float* out) const   // model.cpp:102-109
    {
        std::vector<float> Y(std::size_t(B) * g.L * g.F);
        encode_fwd<float>(g, lv, p.data(), X, B, Y.data(), nullptr, nullptr);
        MlpCache<float> cache;
        if (fast_mlp)
            fast::mlp_fwd(m, p.data() + n_tab, p.data() + n_tab + n_w, Y.data(), B, out, cache);
        else
            mlp_fwd<float>(m, p.data() + n_tab, p.data() + n_tab + n_w, Y.data(), B, out, cache);
    }

    // model.cpp:111-138. Returns the loss; throws std::runtime_error from Adam.
    float train_step(const float* X, const float* target, std::int64_t B, int loss_kind,
                     std::int64_t at_step, float* pred_out = nullptr)
    {
        using clk = std::chrono::steady_clock;
        auto t0 = clk::now();
        auto lap = [&](double& acc) {
            const auto t1 = clk::now();
            acc += std::chrono::duration<double>(t1 - t0).count();
            t0 = t1;
        };
        const int nc = 1 << g.d;
        std::vector<float> Y(std::size_t(B) * g.L * g.F);
        std::vector<std::uint32_t> rows(std::size_t(g.L) * B * nc);
        std::vector<float> wts(rows.size());
        encode_fwd<float>(g, lv, p.data(), X, B, Y.data(), rows.data(), wts.data());
        lap(times.encode_fwd);
        std::vector<float> pred(std::size_t(B) * m.out), dpred(pred.size()), dY(Y.size());
        MlpCache<float> cache;
        if (fast_mlp)
            fast::mlp_fwd(m, W(), b(), Y.data(), B, pred.data(), cache);
        else
            mlp_fwd<float>(m, W(), b(), Y.data(), B, pred.data(), cache);
        lap(times.mlp_fwd);
        const float loss = loss_with_grad<float>(loss_kind, pred.data(), target,
                                                 std::int64_t(pred.size()), dpred.data());
        lap(times.loss);
        if (fast_mlp)
            fast::mlp_bwd(m, W(), cache, dpred.data(), B, grad.data() + n_tab, grad.data() + n_tab + n_w, dY.data());
        else
            mlp_bwd<float>(m, W(), cache, dpred.data(), B, grad.data() + n_tab, grad.data() + n_tab + n_w,
                           dY.data());
        lap(times.mlp_bwd);
        encode_bwd<float>(g, lv, rows.data(), wts.data(), B, dY.data(), grad.data());
        lap(times.encode_bwd);
        const std::string err = adam(float(lr_at(milestones, factor, h.lr, at_step)));
        lap(times.adam);
        if (!err.empty())
            throw std::runtime_error(err);
        if (pred_out)
            std::copy(pred.begin(), pred.end(), pred_out);
        return loss;
    }

    std::string adam(float lr_now)
    {
        Group<float> gs[3] = {
            { "tables", 0, 1, p.data(), grad.data(), mom.data(), vel.data(), n_tab },
            { "mlp_weights", 1, 0, p.data() + n_tab, grad.data() + n_tab, mom.data() + n_tab,
              vel.data() + n_tab, n_w },
            { "mlp_biases", 0, 0, p.data() + n_tab + n_w, grad.data() + n_tab + n_w,
              mom.data() + n_tab + n_w, vel.data() + n_tab + n_w, n_b },
        };
        return adam_step<float>(step, gs, 3, h, lr_now);
    }
};

// Procedural test image (reference tests/helpers.hpp:99-125). rgb is 3 x (w*h)
// column-major, pixel i = y*w + x.
inline void make_test_image(int w, int h, float* rgb)
{
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            const double u = (x + 0.5) / w, v = (y + 0.5) / h;
            double r = 0.35 + 0.3 * u + 0.15 * std::sin(6.0 * u + 2.0 * v);
            double gg = 0.45 + 0.25 * v + 0.12 * std::sin(9.0 * v - 3.0 * u + 1.3);
            double bb = 0.5 + 0.2 * std::sin(4.0 * (u + v));
            for (int o = 1; o <= 3; ++o) {
                const double fr = 12.0 * o, a = 0.08 / o;
                r += a * std::sin(fr * u + 0.7 * o) * std::cos(fr * 0.8 * v);
                gg += a * std::cos(fr * v + 1.9 * o) * std::sin(fr * 0.6 * u);
                bb += a * std::sin(fr * (u - v) + 0.4 * o);
            }
            const std::size_t i = std::size_t(y) * w + x;
            rgb[3 * i + 0] = float(std::min(1.0, std::max(0.0, r)));
            rgb[3 * i + 1] = float(std::min(1.0, std::max(0.0, gg)));
            rgb[3 * i + 2] = float(std::min(1.0, std::max(0.0, bb)));
        }
}

// Analytic CSG SDF used by BASELINE config 2: sphere r=0.3 at
// (0.5,0.5,0.5) union a torus (R=0.25, r=0.08) in the xz-plane, via min.
template <class S> S csg_sdf(S x, S y, S z)
{
    const S cx = x - S(0.5), cy = y - S(0.5), cz = z - S(0.5);
    const S sphere = std::sqrt(cx * cx + cy * cy + cz * cz) - S(0.3);
    const S q = std::sqrt(cx * cx + cz * cz) - S(0.25);
    const S torus = std::sqrt(q * q + cy * cy) - S(0.08);
    return std::min(sphere, torus);
}

}   // namespace orc
