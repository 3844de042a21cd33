// checkpoint.cpp — the reference's binary checkpoint (io.cpp:222-351) for a
// device-resident field: NFC1 header, HGE1 feature tables, MLP1 network,
// ADM1 optimizer state, little-endian, raw fp32 blocks in the reference's
// layouts (tables per level F x len column-major, W_k out x in column-major,
// Adam m/v concatenated per param group). Files written here load in the
// reference and vice versa; only the hash encoder is on the sm_100a path
// (OCT1 / frequency checkpoints are rejected as unsupported).
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/nfg.h"

namespace nfg {
void set_last_error(const std::string& msg);   // field.cu (thread-local nfg_last_error text)
}

namespace {

struct IoError {
    std::string msg;
};

void check(nfg_status st)
{
    if (st != NFG_OK)
        throw st;
}

template <class T>
void put(std::ofstream& o, T v)
{
    o.write(reinterpret_cast<const char*>(&v), sizeof(T));
}

void put_tag(std::ofstream& o, const char* tag) { o.write(tag, 4); }

void put_floats(std::ofstream& o, const float* p, size_t n)
{
    o.write(reinterpret_cast<const char*>(p), std::streamsize(n * sizeof(float)));
}

template <class T>
T get(std::ifstream& in)
{
    T v{};
    in.read(reinterpret_cast<char*>(&v), sizeof(T));
    if (!in)
        throw IoError{ "checkpoint: truncated file" };   // io.cpp:155-156
    return v;
}

void get_floats(std::ifstream& in, float* p, size_t n)
{
    in.read(reinterpret_cast<char*>(p), std::streamsize(n * sizeof(float)));
    if (!in)
        throw IoError{ "checkpoint: truncated float block" };   // io.cpp:168-169
}

void expect_tag(std::ifstream& in, const char* tag, const char* what)   // io.cpp:136-142
{
    char buf[4];
    in.read(buf, 4);
    if (!in || std::memcmp(buf, tag, 4) != 0)
        throw IoError{ std::string("checkpoint: missing ") + what + " section" };
}

struct Unsupported {
    std::string msg;
};

// Errors: std::runtime_error of io.cpp -> NFG_EIO; a failing nested C-ABI
// call keeps its own status and nfg_last_error() text.
template <class Fn>
nfg_status run(Fn&& fn)
{
    try {
        fn();
        return NFG_OK;
    } catch (const IoError& e) {
        nfg::set_last_error(e.msg);
        return NFG_EIO;
    } catch (const Unsupported& e) {
        nfg::set_last_error(e.msg);
        return NFG_EUNSUPPORTED;
    } catch (nfg_status st) {
        return st;
    } catch (const std::exception& e) {
        nfg::set_last_error(e.what());
        return NFG_EIO;
    }
}

}   // namespace

extern "C" {

nfg_status nfg_field_save(nfg_field* f, const char* path)
{
    return run([&] {
        nfg_grid_config g{};
        nfg_mlp_config m{};
        check(nfg_field_get_config(f, &g, &m));
        uint64_t sz[3];
        check(nfg_field_sizes(f, sz));
        const uint64_t n = sz[0] + sz[1] + sz[2];
        std::vector<float> p(n), mo(n), vo(n);
        check(nfg_field_read(f, NFG_BUF_PARAMS, 0, n, p.data()));
        check(nfg_field_read(f, NFG_BUF_ADAM_M, 0, n, mo.data()));
        check(nfg_field_read(f, NFG_BUF_ADAM_V, 0, n, vo.data()));
        uint64_t step = 0;
        check(nfg_field_get_step(f, &step));
        std::vector<nfg_level_spec> lv(size_t(g.levels));
        check(nfg_field_levels(f, lv.data(), g.levels));

        std::ofstream o(path, std::ios::binary);
        if (!o)
            throw IoError{ std::string("cannot write checkpoint: ") + path };
        put_tag(o, "NFC1");
        put<uint32_t>(o, 0u);    // EncoderKind::Hash (model.hpp:16)
        put<uint32_t>(o, 10u);   // n_frequencies (model.hpp:25 default; unused by the hash encoder)
        put_tag(o, "HGE1");
        put<uint32_t>(o, uint32_t(g.dims));
        put<uint32_t>(o, uint32_t(g.levels));
        put<uint32_t>(o, g.table_size);
        put<uint32_t>(o, uint32_t(g.features));
        put<uint32_t>(o, uint32_t(g.n_min));
        put<uint32_t>(o, uint32_t(g.n_max));
        put<uint32_t>(o, uint32_t(g.interpolation));
        for (const auto& l : lv) {
            put<uint64_t>(o, uint64_t(l.table_len));
            put_floats(o, p.data() + l.row_offset * uint64_t(g.features), size_t(l.table_len) * size_t(g.features));
        }
        put_tag(o, "MLP1");
        put<uint32_t>(o, uint32_t(m.input_width));
        put<uint32_t>(o, uint32_t(m.hidden_layers));
        put<uint32_t>(o, uint32_t(m.hidden_width));
        put<uint32_t>(o, uint32_t(m.output_width));
        put<uint32_t>(o, uint32_t(m.output_activation));
        // flat layout [W_0 .. W_n | b_0 .. b_n]; the file interleaves W_k, b_k
        const float* W = p.data() + sz[0];
        const float* b = W + sz[1];
        for (int k = 0; k <= m.hidden_layers; ++k) {
            const int in = k == 0 ? m.input_width : m.hidden_width;
            const int out = k == m.hidden_layers ? m.output_width : m.hidden_width;
            put_floats(o, W, size_t(in) * size_t(out));
            put_floats(o, b, size_t(out));
            W += size_t(in) * size_t(out);
            b += size_t(out);
        }
        put_tag(o, "ADM1");
        put<uint64_t>(o, step);
        put<uint32_t>(o, 3u);   // groups: tables, mlp_weights, mlp_biases (model.cpp:49-77)
        uint64_t off = 0;
        for (int gi = 0; gi < 3; ++gi) {
            put<uint64_t>(o, sz[gi]);
            put_floats(o, mo.data() + off, sz[gi]);
            put_floats(o, vo.data() + off, sz[gi]);
            off += sz[gi];
        }
        if (!o)
            throw IoError{ std::string("cannot write checkpoint: ") + path };
    });
}

nfg_status nfg_field_load(nfg_ctx* ctx, const char* path, const nfg_adam_hyper* hyper, const nfg_options* opts,
                          nfg_field** out)
{
    return run([&] {
        *out = nullptr;
        std::ifstream in(path, std::ios::binary);
        if (!in)
            throw IoError{ std::string("cannot read checkpoint: ") + path };
        expect_tag(in, "NFC1", "file header");
        const uint32_t encoder = get<uint32_t>(in);
        (void)get<uint32_t>(in);   // n_frequencies
        if (encoder != 0u)
            throw Unsupported{ "checkpoint: only hash-encoder models run on the sm_100a path" };
        expect_tag(in, "HGE1", "feature table");
        nfg_grid_config g{};
        g.dims = int32_t(get<uint32_t>(in));
        g.levels = int32_t(get<uint32_t>(in));
        g.table_size = get<uint32_t>(in);
        g.features = int32_t(get<uint32_t>(in));
        g.n_min = int32_t(get<uint32_t>(in));
        g.n_max = int32_t(get<uint32_t>(in));
        g.interpolation = int32_t(get<uint32_t>(in));
        if (g.levels < 1 || g.levels > 64)
            throw IoError{ "checkpoint: invalid hash encoding config" };
        std::vector<nfg_level_spec> lv(size_t(g.levels));
        if (nfg_level_resolutions(&g, lv.data(), g.levels) != g.levels)
            throw IoError{ "checkpoint: invalid hash encoding config" };
        uint64_t n_tab = 0;
        for (const auto& l : lv)
            n_tab += uint64_t(l.table_len) * uint64_t(g.features);
        std::vector<float> tab(n_tab);
        for (const auto& l : lv) {
            if (get<uint64_t>(in) != uint64_t(l.table_len))
                throw IoError{ "checkpoint: level length mismatch" };   // io.cpp:306-307
            get_floats(in, tab.data() + l.row_offset * uint64_t(g.features), size_t(l.table_len) * size_t(g.features));
        }
        expect_tag(in, "MLP1", "MLP parameters");
        nfg_mlp_config m{};
        m.input_width = int32_t(get<uint32_t>(in));
        m.hidden_layers = int32_t(get<uint32_t>(in));
        m.hidden_width = int32_t(get<uint32_t>(in));
        m.output_width = int32_t(get<uint32_t>(in));
        m.output_activation = int32_t(get<uint32_t>(in));
        nfg_field* f = nullptr;
        check(nfg_field_create(ctx, &g, &m, hyper, opts, &f));
        std::unique_ptr<nfg_field, nfg_status (*)(nfg_field*)> guard(f, nfg_field_destroy);
        nfg_grid_config g2{};
        nfg_mlp_config m2{};
        check(nfg_field_get_config(f, &g2, &m2));
        uint64_t sz[3];
        check(nfg_field_sizes(f, sz));
        if (sz[0] != n_tab || m2.input_width != m.input_width)
            throw IoError{ "checkpoint: MLP input width does not match the encoding" };
        std::vector<float> p(sz[0] + sz[1] + sz[2]);
        std::copy(tab.begin(), tab.end(), p.begin());
        float* W = p.data() + sz[0];
        float* b = W + sz[1];
        for (int k = 0; k <= m.hidden_layers; ++k) {
            const int inw = k == 0 ? m.input_width : m.hidden_width;
            const int outw = k == m.hidden_layers ? m.output_width : m.hidden_width;
            get_floats(in, W, size_t(inw) * size_t(outw));
            get_floats(in, b, size_t(outw));
            W += size_t(inw) * size_t(outw);
            b += size_t(outw);
        }
        expect_tag(in, "ADM1", "optimizer state");
        const uint64_t step = get<uint64_t>(in);
        const uint32_t groups = get<uint32_t>(in);
        std::vector<float> mo(p.size(), 0.0f), vo(p.size(), 0.0f);
        uint64_t off = 0;
        for (uint32_t gi = 0; gi < groups; ++gi) {
            const uint64_t len = get<uint64_t>(in);
            if (gi >= 3 || len != sz[gi])
                throw IoError{ "checkpoint: optimizer state does not match the model's parameter groups" };
            get_floats(in, mo.data() + off, len);
            get_floats(in, vo.data() + off, len);
            off += len;
        }
        check(nfg_field_write(f, NFG_BUF_PARAMS, 0, p.size(), p.data()));
        check(nfg_field_write(f, NFG_BUF_ADAM_M, 0, mo.size(), mo.data()));
        check(nfg_field_write(f, NFG_BUF_ADAM_V, 0, vo.size(), vo.data()));
        check(nfg_field_set_step(f, step));
        *out = guard.release();
    });
}

}   // extern "C"
