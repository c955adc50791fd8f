#pragma once

// Drop-in for the activation/normalisation functions of proj/include/lattice/numerics.hpp
// (:81-107): rms_norm, swish_rn, swish_rn_hard with the same signatures and error contract
// (eps <= 0 or empty -> UsageError, non-finite -> DataError). The row is computed by the B200
// row-norm kernel in fp32 (the same math the GEMM epilogues fuse), so results agree with the
// fp64 reference to ~1e-7 relative. rms_norm_rows / swish_rn_rows take many rows at once.

#include <span>
#include <vector>

#include "core.hpp"

namespace lattice {

inline constexpr double kDefaultEps = 1e-6;

namespace detail {
inline std::vector<double> rownorm(int mode, std::span<const double> x, double eps) {
    if (!(eps > 0.0)) throw UsageError("eps must be > 0");
    std::vector<float> xf(x.begin(), x.end());
    device::Buffer<float> d_x(xf), d_y(xf.size());
    device::throw_status(lattice_rownorm(mode, 1, static_cast<std::int64_t>(xf.size()), eps, d_x.get(),
                                         d_y.get(), 1, nullptr));
    const auto y = d_y.download();
    return std::vector<double>(y.begin(), y.end());
}
}  // namespace detail

inline std::vector<double> rms_norm(std::span<const double> x, double eps = kDefaultEps) {
    return detail::rownorm(0, x, eps);
}
inline std::vector<double> swish_rn(std::span<const double> x, double eps = kDefaultEps) {
    return detail::rownorm(1, x, eps);
}
inline std::vector<double> swish_rn_hard(std::span<const double> x, double eps = kDefaultEps) {
    return detail::rownorm(2, x, eps);
}

// Batched: rows x width fp32 matrix, device pointers, stream-ordered.
inline void swish_rn_rows(const float* x, float* out, std::int64_t rows, std::int64_t width, bool hard = false,
                          double eps = kDefaultEps, cudaStream_t stream = nullptr) {
    device::throw_status(lattice_rownorm(hard ? 2 : 1, rows, width, eps, x, out, 0, stream));
}

}  // namespace lattice
