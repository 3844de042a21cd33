// kbench.cu — standalone micro-benchmark of the fused training kernel on the
// BASELINE config-2 shape (3D, L16 F2 T2^19, 2x64 MLP, MAPE, B = 2^18), with an
// optional per-phase clock64 breakdown (-DNFG_PHASE_TIMING). Development tool:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DNFG_PHASE_TIMING \
//        -I paper_2201_05989_b200/csrc tools/kbench.cu paper_2201_05989_b200/csrc/host_init.cpp -o kbench
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "host_init.h"
#include "launch_impl.cuh"

namespace nfg {
void note_kernel_variant(int, const char*) {}   // the library records it for nfg_last_kernel_variant
}

#define CK(x)                                                                      \
    do {                                                                           \
        cudaError_t e = (x);                                                       \
        if (e != cudaSuccess) {                                                    \
            std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            return 1;                                                              \
        }                                                                          \
    } while (0)

int main(int argc, char** argv)
{
    const int64_t B = argc > 1 ? std::atoll(argv[1]) : (1 << 18);
    const int iters = argc > 2 ? std::atoi(argv[2]) : 20;
    nfg_grid_config g{ 16, 1u << 19, 2, 16, 2048, 3, 0 };
    nfg_mlp_config m{ 32, 2, 64, 1, 0 };
    const auto lv = nfg::host::level_resolutions(g);
    // KB_EVEN=1: levels start on even rows; KB_ALIGN=a: on multiples of a rows (the library's device layout)
    const uint32_t align = getenv("KB_ALIGN") ? uint32_t(std::atoi(getenv("KB_ALIGN"))) : (getenv("KB_EVEN") ? 2u : 1u);
    uint64_t rows = 0;
    for (const auto& e : lv)
        rows += (e.table_len + align - 1) / align * align;
    const uint64_t n_tab = rows * 2, n_w = 64 * 32 + 64 * 64 + 64, n_b = 64 + 64 + 1;

    nfg::FieldShape s{};
    s.grid.L = 16;
    s.grid.F = 2;
    s.grid.d = 3;
    s.grid.smooth = 0;
    s.grid.mask = g.table_size - 1;
    s.in_real = 32;
    s.in_steps = 2;
    s.hidden_layers = 2;
    s.hidden_width = 64;
    s.mlp_engine = getenv("KB_ENGINE") ? std::atoi(getenv("KB_ENGINE")) : 0;   // 1: mma.sync dW, 2: tcgen05 dW
    s.n_out = 1;
    s.sigmoid = 0;
    s.table_fp32 = 0;
    uint64_t off = 0;
    for (int l = 0; l < 16; ++l) {
        s.grid.lv[l].res = lv[l].resolution;
        s.grid.lv[l].res_f = float(lv[l].resolution);
        s.grid.lv[l].stride = lv[l].resolution + 1;
        s.grid.lv[l].dense = lv[l].dense;
        s.grid.lv[l].row_off = uint32_t(off);
        off += (lv[l].table_len + align - 1) / align * align;
        s.grid.lv[l].len = lv[l].table_len;
    }

    std::mt19937 rng(1);
    std::uniform_real_distribution<float> U(0.f, 1.f);
    std::vector<__half> tab(n_tab);
    for (auto& v : tab)
        v = __float2half((U(rng) - 0.5f) * 2e-2f);
    std::vector<float> W(n_w), b(n_b, 0.f), X(B * 3), T(B);
    nfg::host::glorot(m, 2, W.data(), b.data());
    for (auto& v : X)
        v = U(rng);
    for (auto& v : T)
        v = U(rng) - 0.5f;
    if (const char* sb = getenv("KB_SORT")) {   // Morton order of the batch at 2^bits cells per axis
        const int bits = std::atoi(sb);
        std::vector<std::pair<uint64_t, int64_t>> key(B);
        for (int64_t i = 0; i < B; ++i) {
            uint64_t k = 0;
            for (int bt = bits - 1; bt >= 0; --bt)
                for (int d = 2; d >= 0; --d)
                    k = (k << 1) | ((uint64_t(X[i * 3 + d] * float(1 << bits)) >> bt) & 1u);
            key[i] = { k, i };
        }
        std::sort(key.begin(), key.end());
        std::vector<float> X2(B * 3);
        for (int64_t i = 0; i < B; ++i)
            for (int d = 0; d < 3; ++d)
                X2[i * 3 + d] = X[key[i].second * 3 + d];
        X.swap(X2);
    }

    __half* d_tab;
    float *d_W, *d_b, *d_X, *d_T, *d_g;
    nfg::LevelDev* d_lv;
    double* d_loss;
    unsigned* d_flags;
    unsigned long long* d_clk;
    CK(cudaMalloc(&d_tab, n_tab * 2));
    CK(cudaMalloc(&d_W, n_w * 4));
    CK(cudaMalloc(&d_b, n_b * 4));
    CK(cudaMalloc(&d_X, B * 12));
    CK(cudaMalloc(&d_T, B * 4));
    CK(cudaMalloc(&d_g, (n_tab + n_w + n_b) * 4));
    CK(cudaMalloc(&d_lv, sizeof(nfg::LevelDev) * NFG_MAX_LEVELS));
    CK(cudaMalloc(&d_loss, 8));
    CK(cudaMalloc(&d_flags, 16));
    CK(cudaMalloc(&d_clk, 8 * 8));
    CK(cudaMemcpy(d_tab, tab.data(), n_tab * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_W, W.data(), n_w * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_b, b.data(), n_b * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_X, X.data(), B * 12, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_T, T.data(), B * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_lv, s.grid.lv, sizeof(nfg::LevelDev) * NFG_MAX_LEVELS, cudaMemcpyHostToDevice));
    CK(cudaMemset(d_g, 0, (n_tab + n_w + n_b) * 4));
    CK(cudaMemset(d_clk, 0, 64));

    nfg::TrainArgs a{};
    a.X = d_X;
    a.target = d_T;
    a.B = B;
    a.loss_kind = 1;
    a.inv_count = 1.0f / float(B);
    a.table = d_tab;
    a.W = d_W;
    a.b = d_b;
    a.table_grad = d_g;
    a.gW = d_g + n_tab;
    a.gb = d_g + n_tab + n_w;
    a.scratch.loss_sum = d_loss;
    a.scratch.flags = d_flags;
    a.scratch.dy_max = nullptr;
    a.phase_clk = nullptr;
    int sms = 148, grid = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    for (int i = 0; i < 3; ++i)
        CK((nfg::run_train<nfg::SRC_ENCODE, nfg::GRAD_LOSS, nfg::SINK_SCATTER, 3, 2, __half, 2, 2>(s, d_lv, a, sms,
                                                                                                   0, &grid)));
    CK(cudaDeviceSynchronize());
    a.phase_clk = d_clk;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int i = 0; i < iters; ++i)
        CK((nfg::run_train<nfg::SRC_ENCODE, nfg::GRAD_LOSS, nfg::SINK_SCATTER, 3, 2, __half, 2, 2>(s, d_lv, a, sms,
                                                                                                   0, &grid)));
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long clk[8];
    CK(cudaMemcpy(clk, d_clk, 64, cudaMemcpyDeviceToHost));
    unsigned long long tot = 0;
    for (auto c : clk)
        tot += c;
    std::printf("k_train B=%lld grid=%d: %.1f us/launch, %.3g samples/s\n", (long long)B, grid, 1000.0 * ms / iters,
                double(B) * iters / (ms / 1000.0));
    const char* names[8] = { "encode", "fwd", "loss+bar", "bwd", "scatter", "bar2", "dW", "bar3" };
    if (tot)
        for (int i = 0; i < 8; ++i)
            std::printf("  %-9s %5.1f%%\n", names[i], 100.0 * double(clk[i]) / double(tot));

    // staged kernels for comparison: encode fwd (thread/sample), MLP train, encode bwd
    float *d_Y, *d_dY;
    CK(cudaMalloc(&d_Y, B * 32 * 4));
    CK(cudaMalloc(&d_dY, B * 32 * 4));
    auto timeit = [&](const char* name, auto&& fn) {
        for (int i = 0; i < 2; ++i)
            fn();
        cudaEventRecord(e0);
        for (int i = 0; i < iters; ++i)
            fn();
        cudaEventRecord(e1);
        cudaDeviceSynchronize();
        float t = 0;
        cudaEventElapsedTime(&t, e0, e1);
        std::printf("%-22s %8.1f us/launch  (%s)\n", name, 1000.0 * t / iters, cudaGetErrorString(cudaGetLastError()));
    };
    nfg::TrainArgs a2 = a;
    a2.phase_clk = nullptr;
    a2.Y = d_Y;
    a2.dY = d_dY;
    timeit("encode_fwd(thread/smp)", [&] { nfg::launch_encode_fwd_lv(s, d_lv, d_X, B, d_tab, d_Y, nullptr, nullptr, 0); });
    timeit("staged MLP train", [&] {
        nfg::run_train<nfg::SRC_LOAD_Y, nfg::GRAD_LOSS, nfg::SINK_STORE, 2, 2, __half, 2, 2>(s, nullptr, a2, sms, 0, &grid);
    });
    timeit("encode_bwd(thread/smp)", [&] { nfg::launch_encode_bwd_lv(s, d_lv, d_X, B, d_dY, d_g, 0); });
    return 0;
}
