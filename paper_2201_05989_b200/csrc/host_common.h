// host_common.h — error plumbing and device buffers shared by the C-ABI
// modules built on top of the field API (tasks.cu, render.cu, nerf.cu).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <stdexcept>
#include <string>

#include "../../include/nfg.h"

namespace nfg {
void set_last_error(const std::string& msg);   // field.cu: the thread-local nfg_last_error text

namespace hc {

struct Fail {
    nfg_status st;
    std::string msg;
};

#define NFG_HC_CUDA(call)                                                                               \
    do {                                                                                                \
        const cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess)                                                                          \
            throw ::nfg::hc::Fail{ NFG_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_) };     \
    } while (0)

// A nested C-ABI call failed: keep its status and message.
inline void ok(nfg_status st)
{
    if (st != NFG_OK)
        throw Fail{ st, nfg_last_error() };
}

// Runs fn, mapping exceptions to statuses the way field.cu's guard does
// (std::invalid_argument -> NFG_EINVAL, like the reference's exceptions).
template <class Fn>
nfg_status run(Fn&& fn)
{
    try {
        fn();
        return NFG_OK;
    } catch (const Fail& f) {
        set_last_error(f.msg);
        return f.st;
    } catch (const std::invalid_argument& e) {
        set_last_error(e.what());
        return NFG_EINVAL;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return NFG_ECUDA;
    }
}

// Growable device buffer. Growth over-allocates by 1.5x so buffers that follow
// an adaptive size (NeRF ray counts) settle quickly: a reallocation
// (cudaFree) synchronises the device.
struct Buf {
    void* p = nullptr;
    size_t bytes = 0;
    Buf() = default;
    Buf(const Buf&) = delete;
    Buf& operator=(const Buf&) = delete;
    void* get(size_t n)
    {
        n = std::max<size_t>(n, 16);
        if (n > bytes) {
            if (p)
                cudaFree(p);
            p = nullptr;
            bytes = 0;
            const size_t want = n + n / 2;
            NFG_HC_CUDA(cudaMalloc(&p, want));
            bytes = want;
        }
        return p;
    }
    template <class T>
    T* as(size_t count)
    {
        return static_cast<T*>(get(count * sizeof(T)));
    }
    ~Buf()
    {
        if (p)
            cudaFree(p);
    }
};

// 1-D grid for a grid-stride loop over n items with 256-thread blocks.
inline unsigned grid_for(int64_t n)
{
    return unsigned(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)));
}

}   // namespace hc
}   // namespace nfg
