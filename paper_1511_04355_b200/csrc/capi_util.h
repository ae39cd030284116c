// C-ABI helpers: exception -> status mapping and RAII device buffers.
#pragma once

#include <string>

#include "common.cuh"

namespace fdsb {

extern thread_local std::string g_error;

template <class F>
int fds_guard(F&& f) {
    try {
        f();
        return FDS_OK;
    } catch (const ValidationError& e) {
        g_error = e.what();
        return FDS_EVALIDATION;
    } catch (const NumericError& e) {
        g_error = e.what();
        return FDS_ENUMERIC;
    } catch (const IoError& e) {
        g_error = e.what();
        return FDS_EIO;
    } catch (const ConvergenceError& e) {
        g_error = e.what();
        return FDS_ECONVERGENCE;
    } catch (const CudaError& e) {
        g_error = e.what();
        return FDS_ECUDA;
    } catch (const std::exception& e) {
        g_error = e.what();
        return FDS_ECUDA;
    }
}

template <class T>
struct DeviceBuffer {
    T* p = nullptr;
    size_t n = 0;
    DeviceBuffer() = default;
    explicit DeviceBuffer(size_t count) { alloc(count); }
    void alloc(size_t count) {
        if (p) cudaFree(p);
        p = nullptr;
        n = count;
        if (count) FDS_CUDA(cudaMalloc(&p, count * sizeof(T)));
    }
    ~DeviceBuffer() {
        if (p) cudaFree(p);
    }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
};

}  // namespace fdsb
