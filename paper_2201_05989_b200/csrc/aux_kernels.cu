// aux_kernels.cu — standalone encode fwd/bwd (component API), Adam, loss.
#include "encode.cuh"
#include <cstdlib>

#include "kernels.h"

namespace nfg {

// ---- encode_forward (grid.hpp:219-272): one thread per sample, all levels ----
template <int D, int F, typename TT>
__global__ void __launch_bounds__(256)
k_encode_fwd(const FieldShape s, const LevelDev* __restrict__ levels, const float* __restrict__ X, int64_t B,
             const TT* __restrict__ table, float* __restrict__ Y, uint32_t* __restrict__ rows,
             float* __restrict__ wts)
{
    __shared__ LevelDev lvs[NFG_MAX_LEVELS];
    for (int i = threadIdx.x; i < s.grid.L; i += blockDim.x)
        lvs[i] = levels[i];
    __syncthreads();
    const int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= B)
        return;
    float x[D];
#pragma unroll
    for (int i = 0; i < D; ++i)
        x[i] = X[p * D + i];
    const int LF = s.grid.L * F;
    constexpr int NC = 1 << D;
    for (int l = 0; l < s.grid.L; ++l) {
        const LevelDev lv = lvs[l];
        const CornerSet<D> cs = corners_of<D>(s.grid, lv, x);
        float acc[F];
#pragma unroll
        for (int f = 0; f < F; ++f)
            acc[f] = 0.0f;
        const TT* base = table + size_t(lv.row_off) * F;
        const size_t co = (size_t(l) * size_t(B) + size_t(p)) * NC;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            const uint32_t r = cs.row(c);
            const float w = cs.weight(c);
            if (rows) {
                rows[co + c] = r;
                wts[co + c] = w;
            }
#pragma unroll
            for (int f = 0; f < F; ++f)
                acc[f] = fmaf(w, Gather<TT>::one(base + size_t(r) * F + f), acc[f]);
        }
#pragma unroll
        for (int f = 0; f < F; ++f)
            Y[p * LF + l * F + f] = acc[f];
    }
}

// ---- encode_backward (grid.hpp:277-295): recompute corners, scatter --------
template <int D, int F>
__global__ void __launch_bounds__(256)
k_encode_bwd(const FieldShape s, const LevelDev* __restrict__ levels, const float* __restrict__ X, int64_t B,
             const float* __restrict__ dY, float* __restrict__ grads, const unsigned int* flags, int l0, int l1)
{
    if (flags && flags[3] != 0u)
        return;   // invalid input of this step (k_validate)
    __shared__ LevelDev lvs[NFG_MAX_LEVELS];
    for (int i = threadIdx.x; i < s.grid.L; i += blockDim.x)
        lvs[i] = levels[i];
    __syncthreads();
    const int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= B)
        return;
    float x[D];
#pragma unroll
    for (int i = 0; i < D; ++i)
        x[i] = X[p * D + i];
    const int LF = s.grid.L * F;
    for (int l = l0; l < l1; ++l) {
        const LevelDev lv = lvs[l];
        const CornerSet<D> cs = corners_of<D>(s.grid, lv, x);
        float* base = grads + size_t(lv.row_off) * F;
        float dy[F];
#pragma unroll
        for (int f = 0; f < F; ++f)
            dy[f] = dY[p * LF + l * F + f];
#pragma unroll
        for (int c = 0; c < (1 << D); ++c) {
            const float w = cs.weight(c);
            float* row = base + size_t(cs.row(c)) * F;
            if (F % 2 == 0) {
#pragma unroll
                for (int f = 0; f < F; f += 2)
                    red_add2(row + f, w * dy[f], w * dy[f + 1]);
            } else {
#pragma unroll
                for (int f = 0; f < F; ++f)
                    atomicAdd(row + f, w * dy[f]);
            }
        }
    }
}

template <int D, int F, typename TT>
static cudaError_t enc_fwd(const FieldShape& s, const LevelDev* lv, const float* X, int64_t B, const void* table,
                           float* Y, uint32_t* rows, float* w, cudaStream_t st)
{
    const int64_t blocks = (B + 255) / 256;
    k_encode_fwd<D, F, TT><<<unsigned(blocks), 256, 0, st>>>(s, lv, X, B, static_cast<const TT*>(table), Y, rows, w);
    return cudaGetLastError();
}

template <int D, int F>
static cudaError_t enc_bwd(const FieldShape& s, const LevelDev* lv, const float* X, int64_t B, const float* dY,
                           float* grads, const unsigned int* flags, cudaStream_t st, int l0, int l1)
{
    const int64_t blocks = (B + 255) / 256;
    k_encode_bwd<D, F><<<unsigned(blocks), 256, 0, st>>>(s, lv, X, B, dY, grads, flags, l0, l1);
    return cudaGetLastError();
}

cudaError_t launch_encode_fwd_lv(const FieldShape& s, const LevelDev* lv, const float* X, int64_t B,
                                 const void* table, float* Y, uint32_t* rows, float* w, cudaStream_t st)
{
    if (B <= 0)
        return cudaSuccess;
#define NFG_ENC_F(D_, F_)                                                                                   \
    if (s.grid.d == D_ && s.grid.F == F_)                                                                    \
        return s.table_fp32 ? enc_fwd<D_, F_, float>(s, lv, X, B, table, Y, rows, w, st)                     \
                            : enc_fwd<D_, F_, __half>(s, lv, X, B, table, Y, rows, w, st);
    NFG_ENC_F(2, 1) NFG_ENC_F(2, 2) NFG_ENC_F(2, 4) NFG_ENC_F(2, 8)
    NFG_ENC_F(3, 1) NFG_ENC_F(3, 2) NFG_ENC_F(3, 4) NFG_ENC_F(3, 8)
#undef NFG_ENC_F
    return cudaErrorNotSupported;
}

cudaError_t launch_encode_bwd_lv(const FieldShape& s, const LevelDev* lv, const float* X, int64_t B,
                                 const float* dY, float* grads, cudaStream_t st, const unsigned int* flags, int l0,
                                 int l1)
{
    if (l1 < 0)
        l1 = s.grid.L;
    if (B <= 0 || l0 >= l1)
        return cudaSuccess;
#define NFG_ENC_B(D_, F_)                                                                                   \
    if (s.grid.d == D_ && s.grid.F == F_)                                                                    \
        return enc_bwd<D_, F_>(s, lv, X, B, dY, grads, flags, st, l0, l1);
    NFG_ENC_B(2, 1) NFG_ENC_B(2, 2) NFG_ENC_B(2, 4) NFG_ENC_B(2, 8)
    NFG_ENC_B(3, 1) NFG_ENC_B(3, 2) NFG_ENC_B(3, 4) NFG_ENC_B(3, 8)
#undef NFG_ENC_B
    return cudaErrorNotSupported;
}

// ---- input validation (grid.hpp:226-229) on the device -------------------------
// flags[3] |= 1 (non-finite) / 2 (outside [-1e-6, 1+1e-6]); flags[1] |= 1 so the
// step aborts before any state changes (k_train and Adam test it first).
__global__ void __launch_bounds__(256) k_validate(const float* __restrict__ X, int64_t n, unsigned int* flags)
{
    unsigned bad = 0;
    const int64_t n4 = (reinterpret_cast<uintptr_t>(X) & 15u) ? 0 : n / 4;
    const float lo = -1e-6f, hi = 1.0f + 1e-6f;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += int64_t(gridDim.x) * blockDim.x) {
        const float4 v = reinterpret_cast<const float4*>(X)[i];
        const float e[4] = { v.x, v.y, v.z, v.w };
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            bad |= finite_f(e[k]) ? 0u : 1u;
            bad |= (e[k] < lo || e[k] > hi) ? 2u : 0u;
        }
    }
    for (int64_t i = 4 * n4 + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        bad |= finite_f(X[i]) ? 0u : 1u;
        bad |= (X[i] < lo || X[i] > hi) ? 2u : 0u;
    }
    bad = __reduce_or_sync(0xffffffffu, bad);
    if (bad && (threadIdx.x & 31) == 0) {
        atomicOr(&flags[3], bad);
        atomicOr(&flags[1], 1u);
    }
}

// ---- start of a step: the step scratch and the sticky abort word ----------------
// Asynchronous (device-pointer) steps are checked by the host only later
// (nfg_field_check). A step that aborted (non-finite gradient: adam.hpp:86-90;
// invalid input: grid.hpp:226-229) must then keep every LATER step from
// touching the state, as the reference would have thrown at it. With inherit
// set (unchecked steps pending), the previous step's abort is latched into
// sticky[0..2] (flag, first bad group + 1, invalid-input bits); while latched,
// each new step starts already aborted with flags[3] = 4 ("stood down"), so
// k_train / encode / Adam all return early. sticky[3] counts the Adam launches
// that did not apply since the host last read the results (k_adam).
__global__ void k_step_begin(double* loss_sum, unsigned int* flags, float* dy_max, unsigned int* sticky, int inherit)
{
    asm volatile("griddepcontrol.launch_dependents;");   // the next step's fused kernel may get scheduled
    asm volatile("griddepcontrol.wait;" ::: "memory");   // Adam has read the flags
    if (!inherit) {   // the host has read every earlier result
        sticky[0] = sticky[1] = sticky[2] = sticky[3] = 0u;
    } else if (sticky[0] == 0u && flags[1] != 0u) {
        sticky[0] = 1u;
        sticky[1] = flags[2];
        sticky[2] = flags[3];
    }
    *loss_sum = 0.0;
    dy_max[0] = 0.0f;
    dy_max[1] = 0.0f;
    const bool down = sticky[0] != 0u;
    flags[0] = 0u;
    flags[1] = down ? 1u : 0u;
    flags[2] = 0xffffffffu;
    flags[3] = down ? 4u : 0u;
}

cudaError_t launch_step_begin(double* loss_sum, unsigned int* flags, float* dy_max, unsigned int* sticky, int inherit,
                              cudaStream_t st)
{
    return launch_pdl(k_step_begin, dim3(1), dim3(1), 0, st, loss_sum, flags, dy_max, sticky, inherit);
}

cudaError_t launch_validate(const float* X, int64_t n, unsigned int* flags, cudaStream_t st)
{
    if (n <= 0)
        return cudaSuccess;
    const unsigned blocks = unsigned(std::min<int64_t>((n / 4 + 255) / 256 + 1, 148 * 4));
    k_validate<<<blocks, 256, 0, st>>>(X, n, flags);
    return cudaGetLastError();
}

// ---- Adam (adam.hpp:78-122) -------------------------------------------------
// Phase 1 (only when flags[0] says a non-finite gradient is possible, or when
// forced): exact isfinite scan; records the first bad group and aborts.
__global__ void __launch_bounds__(256) k_adam_check(const AdamArgs a, int force)
{
    // programmatic dependent launch (launch_adam): the producer's gradients are
    // complete and visible past this point (a no-op for ordinary launches)
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const uint64_t nn = a.n_tab + a.n_w + a.n_b;
    if (a.restore_on_invalid && (a.flags[3] & 3u) != 0u) {
        // invalid batch detected inside the speculative fused kernel: the slab
        // was all-zero before the step, so zeroing restores it exactly
        for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nn;
             i += uint64_t(gridDim.x) * blockDim.x)
            a.g[i] = 0.0f;
        return;
    }
    if (!force && a.flags[0] == 0u)
        return;
    const uint64_t n = a.n_tab + a.n_w + a.n_b;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        if (!finite_f(a.g[i])) {
            const unsigned grp = i < a.n_tab ? 0u : (i < a.n_tab + a.n_w ? 1u : 2u);
            atomicOr(&a.flags[1], 1u);
            atomicMin(&a.flags[2], grp + 1u);
        }
    }
}

// Phase 2: one streaming pass, per entry exactly the reference's operation
// order with IEEE round-to-nearest intrinsics (no contraction) so updates are
// bit-identical to the fp32 reference. Skip-zero entries of the tables group
// are never written; every gradient is zeroed (adam.hpp:118-120).
__device__ __forceinline__ void adam_one(const AdamArgs& a, uint64_t i, float& p, float& g, float& m, float& v,
                                         bool& wrote)
{
    const int grp = i < a.n_tab ? 0 : (i < a.n_tab + a.n_w ? 1 : 2);
    float gg = g;
    wrote = false;
    if (grp == 0 && gg == 0.0f)
        return;
    if (grp == 1)
        gg = __fadd_rn(gg, __fmul_rn(a.l2, p));
    m = __fadd_rn(__fmul_rn(a.b1, m), __fmul_rn(a.omb1, gg));
    v = __fadd_rn(__fmul_rn(a.b2, v), __fmul_rn(__fmul_rn(a.omb2, gg), gg));
    const float num = __fmul_rn(a.lr, __fdiv_rn(m, a.bc1));
    const float den = __fadd_rn(__fsqrt_rn(__fdiv_rn(v, a.bc2)), a.eps);
    p = __fsub_rn(p, __fdiv_rn(num, den));
    wrote = true;
}

__device__ __forceinline__ float4 ld4_hint(const float* p, uint64_t pol)
{
    float4 v;
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p), "l"(pol));
    return v;
}

__device__ __forceinline__ void st4_hint(float* p, float4 v, uint64_t pol)
{
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w), "l"(pol)
                 : "memory");
}

// One full quad [i0, i0 + 4): the update of adam.hpp:78-122 per element, then
// p/m/v streamed back (unchanged values for skipped elements), the gradient
// zeroed for the next step and the fp16 table shadow refreshed (both kept in L2).
__device__ __forceinline__ void adam_quad(const AdamArgs& a, uint64_t i0, float4 G, float4 P, float4 M, float4 V,
                                          uint64_t pol_stream, uint64_t pol_keep)
{
    const bool any = G.x != 0.0f || G.y != 0.0f || G.z != 0.0f || G.w != 0.0f;
    float pg[4] = { P.x, P.y, P.z, P.w }, gq[4] = { G.x, G.y, G.z, G.w };
    float mq[4] = { M.x, M.y, M.z, M.w }, vq[4] = { V.x, V.y, V.z, V.w };
    bool w[4];
#pragma unroll
    for (int e = 0; e < 4; ++e)
        adam_one(a, i0 + e, pg[e], gq[e], mq[e], vq[e], w[e]);
    st4_hint(a.p + i0, make_float4(pg[0], pg[1], pg[2], pg[3]), pol_stream);
    st4_hint(a.m + i0, make_float4(mq[0], mq[1], mq[2], mq[3]), pol_stream);
    st4_hint(a.v + i0, make_float4(vq[0], vq[1], vq[2], vq[3]), pol_stream);
    if (any)
        st4_hint(a.g + i0, make_float4(0.f, 0.f, 0.f, 0.f), pol_keep);
    if (a.shadow && i0 < a.n_tab) {
        if (i0 + 3 < a.n_tab && w[0] && w[1] && w[2] && w[3]) {
            const uint2 h = make_uint2(pack_half2(pg[0], pg[1]), pack_half2(pg[2], pg[3]));
            asm volatile("st.global.L2::cache_hint.v2.u32 [%0], {%1, %2}, %3;" ::"l"(a.shadow + i0), "r"(h.x),
                         "r"(h.y), "l"(pol_keep)
                         : "memory");
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (w[e] && i0 + e < a.n_tab)
                    a.shadow[i0 + e] = __float2half_rn(pg[e]);
        }
    }
}

#ifndef NFG_ADAM_QUAD_GROUP
#define NFG_ADAM_QUAD_GROUP 2   // quads per thread on sparse steps (tools/exp_adam_sp.sh)
#endif
__global__ void __launch_bounds__(256) k_adam(const AdamArgs a)
{
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (a.flags[1] != 0u) {   // non-finite gradient: state untouched (the reference throws first)
        // every Adam step that does not apply (the aborting one and those standing
        // down behind it, k_step_begin) is counted once, so nfg_field_check can
        // restore the host step counter
        if (a.sticky && a.mode != 1 && blockIdx.x == 0 && threadIdx.x == 0)
            a.sticky[3] += 1u;
        return;
    }
    if ((a.mode == 1 && a.flags[0] != 0u) || (a.mode == 2 && a.flags[0] == 0u))
        return;   // pipelined chunks vs the checked fallback: exactly one of them updates
    const uint64_t n = a.mode == 1 ? a.hi : a.n_tab + a.n_w + a.n_b;
    const uint64_t n4 = n / 4;
    const uint64_t q0 = a.mode == 1 ? a.lo / 4 : 0;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    // L2 policy: p, m, v stream through once per step (evict-first); the zeroed
    // gradients and the fp16 table shadow are what the next step's fused kernel
    // hits with atomics and gathers (73 MB at config 2), so they are written
    // evict-last to stay L2-resident across the step boundary.
    uint64_t pol_stream, pol_keep;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_stream));
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
    if (!a.eager && a.mode == 0) {
        // Sparse steps: a thread owns QG consecutive quads (QG * 16 bytes of
        // each stream). When any of them has a gradient it reads and writes
        // them all, so p/m/v move in whole sectors (untouched neighbours are
        // written back unchanged) instead of isolated 16-byte pieces.
        constexpr int QG = NFG_ADAM_QUAD_GROUP;
        const uint64_t ng = n / (4 * QG);
        for (uint64_t o = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; o < ng; o += stride) {
            const uint64_t i0 = 4 * QG * o;
            float4 G[QG];
            bool any = false;
#pragma unroll
            for (int k = 0; k < QG; ++k) {
                G[k] = ld4_hint(a.g + i0 + 4 * k, pol_stream);
                any |= G[k].x != 0.0f || G[k].y != 0.0f || G[k].z != 0.0f || G[k].w != 0.0f;
            }
            if (!any && i0 + 4 * QG - 1 < a.n_tab)
                continue;
            float4 P[QG], M[QG], V[QG];
#pragma unroll
            for (int k = 0; k < QG; ++k) {
                P[k] = ld4_hint(a.p + i0 + 4 * k, pol_stream);
                M[k] = ld4_hint(a.m + i0 + 4 * k, pol_stream);
                V[k] = ld4_hint(a.v + i0 + 4 * k, pol_stream);
            }
#pragma unroll
            for (int k = 0; k < QG; ++k)
                adam_quad(a, i0 + 4 * k, G[k], P[k], M[k], V[k], pol_stream, pol_keep);
        }
        for (uint64_t i = 4 * QG * ng + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
            float p = a.p[i], g = a.g[i], m = a.m[i], v = a.v[i];
            bool w;
            adam_one(a, i, p, g, m, v, w);
            if (w) {
                a.p[i] = p;
                a.m[i] = m;
                a.v[i] = v;
                if (a.shadow && i < a.n_tab)
                    a.shadow[i] = __float2half_rn(p);
            }
            a.g[i] = 0.0f;
        }
        return;
    }
    for (uint64_t q = q0 + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < n4; q += stride) {
        const uint64_t i0 = 4 * q;
        float4 G, P, M, V;
        bool any;
        if (a.eager) {   // dense step: all four streams in flight at once
            G = ld4_hint(a.g + 4 * q, pol_stream);
            P = ld4_hint(a.p + 4 * q, pol_stream);
            M = ld4_hint(a.m + 4 * q, pol_stream);
            V = ld4_hint(a.v + 4 * q, pol_stream);
            any = G.x != 0.0f || G.y != 0.0f || G.z != 0.0f || G.w != 0.0f;
            if (!any && i0 + 3 < a.n_tab)
                continue;
        } else {
            G = ld4_hint(a.g + 4 * q, pol_stream);
            any = G.x != 0.0f || G.y != 0.0f || G.z != 0.0f || G.w != 0.0f;
            if (!any && i0 + 3 < a.n_tab)
                continue;   // whole quad skipped: nothing to read or write
            P = ld4_hint(a.p + 4 * q, pol_stream);
            M = ld4_hint(a.m + 4 * q, pol_stream);
            V = ld4_hint(a.v + 4 * q, pol_stream);
        }
        adam_quad(a, i0, G, P, M, V, pol_stream, pol_keep);
    }
    // tail
    for (uint64_t i = 4 * n4 + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        float p = a.p[i], g = a.g[i], m = a.m[i], v = a.v[i];
        bool w;
        adam_one(a, i, p, g, m, v, w);
        if (w) {
            a.p[i] = p;
            a.m[i] = m;
            a.v[i] = v;
            if (a.shadow && i < a.n_tab)
                a.shadow[i] = __float2half_rn(p);
        }
        a.g[i] = 0.0f;
    }
}

cudaError_t launch_adam_range(const AdamArgs& a, int num_sms, cudaStream_t st)
{
    const uint64_t quads = (a.hi - a.lo + 3) / 4;
    const int blocks = int(std::max<uint64_t>(1, std::min<uint64_t>((quads + 255) / 256, uint64_t(num_sms) * 8)));
    AdamArgs r = a;
    r.mode = 1;
    k_adam<<<blocks, 256, 0, st>>>(r);
    return cudaGetLastError();
}

cudaError_t launch_adam_fallback(const AdamArgs& a, int num_sms, cudaStream_t st)
{
    const uint64_t n = a.n_tab + a.n_w + a.n_b;
    const int blocks = int(std::min<uint64_t>((n / 4 + 255) / 256 + 1, uint64_t(num_sms) * 8));
    AdamArgs r = a;
    r.mode = 2;
    k_adam_check<<<num_sms * 4, 256, 0, st>>>(r, 0);
    k_adam<<<blocks, 256, 0, st>>>(r);
    return cudaGetLastError();
}

bool pdl_enabled()
{
    static const bool on = !getenv("NFG_NO_PDL");
    return on;
}

cudaError_t launch_adam(const AdamArgs& a, bool force_check, int num_sms, cudaStream_t st)
{
    const uint64_t n = a.n_tab + a.n_w + a.n_b;
    const int blocks = int(std::min<uint64_t>((n / 4 + 255) / 256 + 1, uint64_t(num_sms) * 8));
    cudaError_t e = launch_pdl(k_adam_check, dim3(num_sms * 4), dim3(256), 0, st, a, force_check ? 1 : 0);
    if (e == cudaSuccess)
        e = launch_pdl(k_adam, dim3(blocks), dim3(256), 0, st, a);
    return e;
}

__global__ void k_shadow(const float* __restrict__ p, __half* __restrict__ s, uint64_t n)
{
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        s[i] = __float2half_rn(p[i]);
}

cudaError_t launch_shadow(const float* p, __half* shadow, uint64_t n, cudaStream_t st)
{
    if (n == 0)
        return cudaSuccess;
    const unsigned blocks = unsigned(std::min<uint64_t>((n + 255) / 256, 148 * 16));
    k_shadow<<<blocks, 256, 0, st>>>(p, shadow, n);
    return cudaGetLastError();
}

// ---- losses (losses.hpp:10-59) ------------------------------------------------
__global__ void __launch_bounds__(256) k_loss(int kind, const float* __restrict__ pred, const float* __restrict__ target,
                                              int64_t n, float count, float* __restrict__ dpred, double* loss_sum)
{
    float term = 0.0f;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const float p = pred[i], t = target[i], diff = p - t;
        float d;
        switch (kind) {
        case 0:
            term += diff * diff;
            d = (2.0f / count) * diff;   // losses.hpp:16-17
            break;
        case 1: {
            const float den = fabsf(t) + 0.01f;
            term += fabsf(diff) / den;
            const float sg = diff > 0.0f ? 1.0f : (diff < 0.0f ? -1.0f : 0.0f);
            d = sg / den / count;   // losses.hpp:36
            break;
        }
        default: {
            const float den = __fadd_rn(__fmul_rn(p, p), 0.01f);   // no contraction (bit parity)
            term += diff * diff / den;
            d = 2.0f * diff / den / count;   // losses.hpp:55
        }
        }
        dpred[i] = d;
    }
    for (int m = 16; m > 0; m >>= 1)
        term += __shfl_xor_sync(0xffffffffu, term, m);
    if ((threadIdx.x & 31) == 0)
        atomicAdd(loss_sum, double(term));
}

cudaError_t launch_loss(int kind, const float* pred, const float* target, int64_t n, float count, float* dpred,
                        double* loss_sum, cudaStream_t st)
{
    if (n <= 0)
        return cudaSuccess;
    const unsigned blocks = unsigned(std::min<int64_t>((n + 255) / 256, 148 * 8));
    k_loss<<<blocks, 256, 0, st>>>(kind, pred, target, n, count, dpred, loss_sum);
    return cudaGetLastError();
}

// ---- loss of an asynchronous device step (nfg_field_train_step_device) --------
// train_step's return value: float(loss_sum / count) (model.cpp:111-138), NaN
// when the step aborted (the host call would have thrown instead).
__global__ void k_loss_out(const double* loss_sum, const unsigned int* flags, double count, float* out)
{
    *out = flags[1] ? __int_as_float(0x7fffffff) : (count > 0 ? float(*loss_sum / count) : 0.0f);
}

cudaError_t launch_loss_out(const double* loss_sum, const unsigned int* flags, double count, float* out,
                            cudaStream_t st)
{
    k_loss_out<<<1, 1, 0, st>>>(loss_sum, flags, count, out);
    return cudaGetLastError();
}

}   // namespace nfg
