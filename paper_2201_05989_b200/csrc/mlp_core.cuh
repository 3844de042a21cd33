// mlp_core.cuh — warp-level building blocks of the fully fused 64-wide MLP.
//
// Restates mlp.hpp:104-158 (forward with biases + ReLU + linear/sigmoid output,
// hand-written backward) on tensor cores: mma.sync.m16n8k16 f16 x f16 -> f32.
// A warp owns 16 samples (one m16 row block). Activations never leave
// registers between layers in the forward pass: the f32 C fragment of two
// adjacent n8 tiles is exactly the f16 A fragment of the next layer's k16
// step. Weights live in shared memory as [out][in] fp16 rows (the transpose of
// the reference's column-major W, i.e. the .col B operand), padded by 8 halves
// per row so ldmatrix is bank-conflict free.
//
// Fragment ownership (PTX ISA, m16n8k16): lane = 4*g + t.
//   A regs: {(g, 2t..2t+1), (g+8, 2t..), (g, 2t+8..), (g+8, 2t+8..)}
//   B regs: {(k=2t..2t+1, n=g), (k=2t+8.., n=g)}
//   C regs: (g, 2t), (g, 2t+1), (g+8, 2t), (g+8, 2t+1)
#pragma once

#include "nfg_common.cuh"

namespace nfg {
namespace mlp {

constexpr int H = 64;          // hidden width (the only width built for sm_100a)
constexpr int HS = H + 8;      // smem row stride (halves) of 64-wide buffers
constexpr int OUTP = 16;       // output layer padded to 16 rows
constexpr int HT = H / 8;      // n8 tiles across a hidden layer

__device__ __forceinline__ void ldsm_x4(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, const void* p)
{
    const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(a));
}

__device__ __forceinline__ void ldsm_x4_t(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, const void* p)
{
    const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(a));
}

__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1)
{
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Saturating fp16 pack for backward operands (scaled gradients): a finite
// overflow saturates instead of becoming inf, but a NaN stays NaN, so a
// non-finite loss gradient still reaches the gradient slab and Adam's scan
// rejects the step like the reference (adam.hpp:86-90;
// tests/test_gpu_parity.py::test_async_abort_is_sticky[nan_target]).
// One F2FP.SATFINITE: cvt's .satfinite clamps +-inf and finite overflow to
// +-65504 and keeps NaN. cvt packs its first source into the UPPER half.
__device__ __forceinline__ uint32_t pack_sat(float a, float b)
{
    uint32_t r;
    asm("cvt.rn.satfinite.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
    return r;
}

// ---- shared-memory weight image -----------------------------------------
// Layout (halves): W0 [H][INS] | Wh[NH-1] [H][HS] | Wout [OUTP][HS]; then
// fp32 biases b0[H] | bh[NH-1][H] | bout[OUTP].
template <int IN_STEPS, int NH>
struct WLayout {
    static constexpr int IN = 16 * IN_STEPS;
    static constexpr int INS = IN + 8;
    static constexpr int W0_HALVES = H * INS;
    static constexpr int WH_HALVES = H * HS;
    static constexpr int WOUT_HALVES = OUTP * HS;
    static constexpr int HALVES = W0_HALVES + (NH - 1) * WH_HALVES + WOUT_HALVES;
    static constexpr int BIAS_FLOATS = H * NH + OUTP;
    static constexpr int BYTES = HALVES * 2 + BIAS_FLOATS * 4;
};

struct MlpShape {
    int in_real;     // L*F (reference input_width)
    int n_out;       // reference output_width (<= 16)
    int sigmoid;
    int hw;          // reference hidden_width (<= 64): the 64-wide layers carry zero rows / columns
                     // beyond it, which are exact no-ops (ReLU(0) = 0 and a zero dz) forward and backward
};

// Converts the fp32 master weights (reference layout: W_k out x in column-major,
// then biases; hidden width sh.hw) into the padded fp16 [out][in] smem image
// (64-wide, zero beyond sh.hw). All threads.
template <int IN_STEPS, int NH>
__device__ void load_weights(__half* ws, float* bs, const float* __restrict__ W, const float* __restrict__ b,
                             const MlpShape& sh)
{
    using Lay = WLayout<IN_STEPS, NH>;
    const int tid = threadIdx.x, nt = blockDim.x, hw = sh.hw;
    // layer 0: hw x in_real
    for (int i = tid; i < H * Lay::INS; i += nt) {
        const int o = i / Lay::INS, c = i % Lay::INS;
        ws[i] = __float2half_rn(c < sh.in_real && o < hw ? W[o + c * hw] : 0.0f);
    }
    size_t woff = size_t(hw) * sh.in_real;
    for (int k = 0; k < NH - 1; ++k) {
        __half* dst = ws + Lay::W0_HALVES + k * Lay::WH_HALVES;
        for (int i = tid; i < H * HS; i += nt) {
            const int o = i / HS, c = i % HS;
            dst[i] = __float2half_rn(c < hw && o < hw ? W[woff + o + c * hw] : 0.0f);
        }
        woff += size_t(hw) * hw;
    }
    __half* wo = ws + Lay::W0_HALVES + (NH - 1) * Lay::WH_HALVES;
    for (int i = tid; i < OUTP * HS; i += nt) {
        const int o = i / HS, c = i % HS;
        wo[i] = __float2half_rn((c < hw && o < sh.n_out) ? W[woff + o + c * sh.n_out] : 0.0f);
    }
    for (int i = tid; i < H * NH; i += nt)
        bs[i] = (i % H) < hw ? b[(i / H) * hw + (i % H)] : 0.0f;
    for (int i = tid; i < OUTP; i += nt)
        bs[H * NH + i] = i < sh.n_out ? b[hw * NH + i] : 0.0f;
}

// acc[NT] = A (16 x 16*KS) * W^T where W is [8*NT rows][wstride] in smem.
template <int KS, int NT>
__device__ __forceinline__ void layer_fwd(const uint32_t (&a)[KS][4], const __half* W, int wstride,
                                          float (&acc)[NT][4], int lane)
{
#pragma unroll
    for (int j = 0; j < NT; ++j)
        acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.0f;
    const int rsel = (lane & 7) + ((lane >> 4) << 3);
    const int csel = ((lane >> 3) & 1) << 3;
#pragma unroll
    for (int s = 0; s < KS; ++s) {
#pragma unroll
        for (int j = 0; j < NT; j += 2) {
            uint32_t b0, b1, b2, b3;
            ldsm_x4(b0, b1, b2, b3, W + (8 * j + rsel) * wstride + 16 * s + csel);
            mma16816(acc[j], a[s], b0, b1);
            mma16816(acc[j + 1], a[s], b2, b3);
        }
    }
}

// acc[NT] (16 x 8*NT, over in) = dz (16 x 16*KS, over out) * W where W is
// [16*KS rows = out][wstride] in smem (the .trans B operand).
template <int KS, int NT>
__device__ __forceinline__ void layer_bwd(const uint32_t (&a)[KS][4], const __half* W, int wstride,
                                          float (&acc)[NT][4], int lane)
{
#pragma unroll
    for (int j = 0; j < NT; ++j)
        acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.0f;
    const int rsel = (lane & 7) + (((lane >> 3) & 1) << 3);
    const int csel = (lane >> 4) << 3;
#pragma unroll
    for (int s = 0; s < KS; ++s) {
#pragma unroll
        for (int j = 0; j < NT; j += 2) {
            uint32_t b0, b1, b2, b3;
            ldsm_x4_t(b0, b1, b2, b3, W + (16 * s + rsel) * wstride + 8 * j + csel);
            mma16816(acc[j], a[s], b0, b1);
            mma16816(acc[j + 1], a[s], b2, b3);
        }
    }
}

// C fragments of 2*KS n8 tiles -> f16 A fragments of KS k16 steps.
template <int KS, bool SAT>
__device__ __forceinline__ void c_to_a(const float (&c)[2 * KS][4], uint32_t (&a)[KS][4])
{
#pragma unroll
    for (int s = 0; s < KS; ++s) {
        if (SAT) {
            a[s][0] = pack_sat(c[2 * s][0], c[2 * s][1]);
            a[s][1] = pack_sat(c[2 * s][2], c[2 * s][3]);
            a[s][2] = pack_sat(c[2 * s + 1][0], c[2 * s + 1][1]);
            a[s][3] = pack_sat(c[2 * s + 1][2], c[2 * s + 1][3]);
        } else {
            a[s][0] = pack_half2(c[2 * s][0], c[2 * s][1]);
            a[s][1] = pack_half2(c[2 * s][2], c[2 * s][3]);
            a[s][2] = pack_half2(c[2 * s + 1][0], c[2 * s + 1][1]);
            a[s][3] = pack_half2(c[2 * s + 1][2], c[2 * s + 1][3]);
        }
    }
}

// Stores an A-fragment block (16 rows x 16*KS cols) to a [rows][stride] smem buffer.
template <int KS>
__device__ __forceinline__ void store_a(const uint32_t (&a)[KS][4], __half* buf, int stride, int row0, int lane)
{
    const int g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int s = 0; s < KS; ++s) {
        uint32_t* r0 = reinterpret_cast<uint32_t*>(buf + (row0 + g) * stride + 16 * s + 2 * t);
        uint32_t* r8 = reinterpret_cast<uint32_t*>(buf + (row0 + g + 8) * stride + 16 * s + 2 * t);
        r0[0] = a[s][0];
        r8[0] = a[s][1];
        r0[4] = a[s][2];
        r8[4] = a[s][3];
    }
}

// Loads an A-fragment block from a [rows][stride] smem buffer.
template <int KS>
__device__ __forceinline__ void load_a(uint32_t (&a)[KS][4], const __half* buf, int stride, int row0, int lane)
{
#pragma unroll
    for (int s = 0; s < KS; ++s)
        ldsm_x4(a[s][0], a[s][1], a[s][2], a[s][3], buf + (row0 + (lane & 15)) * stride + 16 * s + ((lane >> 4) << 3));
}

// Hidden-layer epilogue: + bias, ReLU, remember the active set (bit per C reg).
template <int NT>
__device__ __forceinline__ uint32_t bias_relu(float (&acc)[NT][4], const float* bias, int lane)
{
    const int t = lane & 3;
    uint32_t mask = 0;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
        const float b0 = bias[8 * j + 2 * t], b1 = bias[8 * j + 2 * t + 1];
        float v[4] = { acc[j][0] + b0, acc[j][1] + b1, acc[j][2] + b0, acc[j][3] + b1 };
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const bool on = v[e] > 0.0f;
            mask |= (on ? 1u : 0u) << (4 * j + e);
            acc[j][e] = on ? v[e] : 0.0f;
        }
    }
    return mask;
}

template <int NT>
__device__ __forceinline__ void apply_mask(float (&acc)[NT][4], uint32_t mask)
{
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (!((mask >> (4 * j + e)) & 1u))
                acc[j][e] = 0.0f;
}

// Column sums of a C-fragment block over the warp's 16 rows; lanes with g == 0
// (lanes 0..3) end up holding the sums for cols 8j+2t, 8j+2t+1.
template <int NT>
__device__ __forceinline__ void col_sums(const float (&acc)[NT][4], float (&s)[NT][2])
{
#pragma unroll
    for (int j = 0; j < NT; ++j) {
        float a = acc[j][0] + acc[j][2], b = acc[j][1] + acc[j][3];
#pragma unroll
        for (int m = 4; m < 32; m <<= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, m);
            b += __shfl_xor_sync(0xffffffffu, b, m);
        }
        s[j][0] = a;
        s[j][1] = b;
    }
}

// ---- loss (losses.hpp:10-59) on one output element -----------------------
// Returns the unnormalised gradient count * dLoss/dpred and adds the loss term.
__device__ __forceinline__ float loss_grad(int kind, float p, float t, float& term)
{
    const float diff = p - t;
    switch (kind) {
    case 0:   // l2: diff^2 ; 2 diff
        term += diff * diff;
        return 2.0f * diff;
    case 1: {   // mape: |diff| / (|t| + 0.01) ; sign(diff) / den
        const float den = fabsf(t) + 0.01f;
        term += fabsf(diff) / den;
        const float sg = diff > 0.0f ? 1.0f : (diff < 0.0f ? -1.0f : 0.0f);
        return sg / den;
    }
    default: {   // relative l2 with frozen denominator p^2 + 0.01
        const float den = __fadd_rn(__fmul_rn(p, p), 0.01f);
        term += diff * diff / den;
        return 2.0f * diff / den;
    }
    }
}

__device__ __forceinline__ void ldsm_x2_t(uint32_t& r0, uint32_t& r1, const void* p)
{
    const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0,%1}, [%2];\n" : "=r"(r0), "=r"(r1) : "r"(a));
}

// db via the tensor cores: the activation buffers carry a column of ones at
// `ones_col` (in their padding), so one extra n8 tile of dz^T * [act | 1]
// yields sum_samples dz for 16 outputs (C regs 0 and 2 of the t == 0 lanes).
template <int S>
__device__ __forceinline__ void db_tile(float (&c)[4], const __half* dz, int dzs, const __half* act, int as, int mt,
                                        int ones_col, int lane)
{
#pragma unroll
    for (int e = 0; e < 4; ++e)
        c[e] = 0.0f;
    const int ar = (lane & 7) + ((lane >> 4) << 3), ac = ((lane >> 3) & 1) << 3;
    const int br = (lane & 7) + (((lane >> 3) & 1) << 3);
#pragma unroll 4
    for (int ks = 0; ks < S / 16; ++ks) {
        uint32_t a[4], b0, b1;
        ldsm_x4_t(a[0], a[1], a[2], a[3], dz + (16 * ks + ar) * dzs + 16 * mt + ac);
        ldsm_x2_t(b0, b1, act + (16 * ks + br) * as + ones_col);
        mma16816(c, a, b0, b1);
    }
}

// ---- dW: per-CTA K = S samples from smem (dz^T * act) -----------------------
// One (mt, np) pair = 16 out rows x 16 in cols = two n8 C tiles.
template <int S>
__device__ __forceinline__ void dw_pair(float (&c0)[4], float (&c1)[4], const __half* dz, int dzs,
                                        const __half* act, int as, int mt, int np, int lane)
{
#pragma unroll
    for (int e = 0; e < 4; ++e)
        c0[e] = c1[e] = 0.0f;
    const int ar = (lane & 7) + ((lane >> 4) << 3), ac = ((lane >> 3) & 1) << 3;
    const int br = (lane & 7) + (((lane >> 3) & 1) << 3), bc = (lane >> 4) << 3;
#pragma unroll 4
    for (int ks = 0; ks < S / 16; ++ks) {
        uint32_t a[4], b0, b1, b2, b3;
        ldsm_x4_t(a[0], a[1], a[2], a[3], dz + (16 * ks + ar) * dzs + 16 * mt + ac);
        ldsm_x4_t(b0, b1, b2, b3, act + (16 * ks + br) * as + 16 * np + bc);
        mma16816(c0, a, b0, b1);
        mma16816(c1, a, b2, b3);
    }
}

}   // namespace mlp
}   // namespace nfg
