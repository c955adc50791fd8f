#pragma once

// Small RAII helpers the drop-in headers use to stage host data through device memory and
// to turn C-ABI status codes back into the reference's exception types
// (proj/include/lattice/core.hpp:20-27).

#include <cuda_runtime.h>

#include <cstddef>
#include <stdexcept>
#include <string>
#include <vector>

#include "../lattice_b200.h"

namespace lattice {

struct UsageError : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};

struct DataError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

namespace device {

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void throw_status(lattice_status st) {
    if (st == LATTICE_OK) return;
    const std::string msg = lattice_last_error();
    if (st == LATTICE_USAGE) throw UsageError(msg);
    if (st == LATTICE_DATA) throw DataError(msg);
    throw CudaError(msg);
}

inline void cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// Owning device buffer of T.
template <typename T>
class Buffer {
public:
    Buffer() = default;
    explicit Buffer(std::size_t n) : n_(n) {
        if (n) cuda(cudaMalloc(reinterpret_cast<void**>(&p_), n * sizeof(T)), "cudaMalloc");
    }
    Buffer(const T* host, std::size_t n) : Buffer(n) { upload(host, n); }
    explicit Buffer(const std::vector<T>& v) : Buffer(v.data(), v.size()) {}
    Buffer(const Buffer&) = delete;
    Buffer& operator=(const Buffer&) = delete;
    Buffer(Buffer&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr, o.n_ = 0; }
    Buffer& operator=(Buffer&& o) noexcept {
        std::swap(p_, o.p_);
        std::swap(n_, o.n_);
        return *this;
    }
    ~Buffer() {
        if (p_) cudaFree(p_);
    }
    void upload(const T* host, std::size_t n) {
        if (n) cuda(cudaMemcpy(p_, host, n * sizeof(T), cudaMemcpyHostToDevice), "H2D");
    }
    std::vector<T> download() const {
        std::vector<T> out(n_);
        if (n_) cuda(cudaMemcpy(out.data(), p_, n_ * sizeof(T), cudaMemcpyDeviceToHost), "D2H");
        return out;
    }
    T* get() const { return p_; }
    std::size_t size() const { return n_; }

private:
    T* p_ = nullptr;
    std::size_t n_ = 0;
};

}  // namespace device
}  // namespace lattice
