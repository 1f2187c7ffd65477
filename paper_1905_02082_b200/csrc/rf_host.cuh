// Host-side helpers shared by the C ABI translation units: status errors,
// the guard that turns them into rf_status + rf_last_error(), and an owning
// device buffer.
#pragma once

#include <cuda_runtime.h>

#include <exception>
#include <string>

#include "../../include/refusion_b200.h"

namespace rfb {

extern thread_local std::string g_err;  // rf_last_error() (rf_capi.cu)

struct Error {
    rf_status code;
    std::string msg;
};

#define CK(x)                                                                                    \
    do {                                                                                         \
        cudaError_t e_ = (x);                                                                    \
        if (e_ != cudaSuccess) throw ::rfb::Error{RF_CUDA_ERROR, std::string(#x) + ": " + cudaGetErrorString(e_)}; \
    } while (0)

template <class F>
rf_status guard(F&& f) {
    try {
        f();
        return RF_OK;
    } catch (const Error& e) {
        g_err = e.msg;
        return e.code;
    } catch (const std::exception& e) {
        g_err = e.what();
        return RF_CUDA_ERROR;
    }
}

inline void require(bool ok, rf_status code, const std::string& msg) {
    if (!ok) throw Error{code, msg};
}

struct DevBuf {  // owning device allocation (freed on scope exit, also on error paths)
    void* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void ensure(size_t bytes) {
        if (bytes <= n) return;
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
        CK(cudaMalloc(&p, bytes));
        n = bytes;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

}  // namespace rfb
