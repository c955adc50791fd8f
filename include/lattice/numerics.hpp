#pragma once

// Drop-in for proj/include/lattice/numerics.hpp: rms_norm, swish_rn, swish_rn_hard (:81-107),
// correlation_loss (:46-78), swish_rn_jvp (:113-136), clip_features and smooth_labels
// (:139-156) with the same signatures and error contract (eps <= 0 or empty -> UsageError,
// non-finite -> DataError). Everything runs in fp64 on the device with the reference's own
// arithmetic (lattice_rownorm_f64: sequential row sums without FMA contraction), so rms_norm is
// bit-identical to the reference and swish_rn / swish_rn_hard agree to exp()'s last ulp, for
// inputs of any magnitude. The fp32 batched swish_rn_rows is the GEMM epilogues' arithmetic.

#include <span>
#include <vector>

#include "core.hpp"

namespace lattice {

inline constexpr double kDefaultEps = 1e-6;

namespace detail {
inline std::vector<double> rownorm(int mode, std::span<const double> x, double eps) {
    if (!(eps > 0.0)) throw UsageError("eps must be > 0");
    if (x.empty()) throw UsageError("rms_norm: empty input");
    device::Buffer<double> d_x(x.data(), x.size()), d_y(x.size());
    device::throw_status(lattice_rownorm_f64(mode, 1, static_cast<std::int64_t>(x.size()), eps, d_x.get(),
                                             d_y.get(), 1, nullptr));
    return d_y.download();
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

namespace detail {
template <typename F>
inline std::vector<double> device_op(std::span<const double> x, F&& launch) {
    device::Buffer<double> d_x(x.data(), x.size()), d_y(x.size());
    launch(d_x.get(), d_y.get());
    return d_y.download();
}
}  // namespace detail

// numerics.hpp:46-78: fp64 on the device, same two-pass population moments.
inline double correlation_loss(std::span<const double> x, std::span<const double> y, double eps = kDefaultEps) {
    if (!(eps > 0.0)) throw UsageError("eps must be > 0");
    if (x.size() != y.size()) throw UsageError("correlation_loss: length mismatch");
    if (x.size() < 2) throw UsageError("correlation_loss: need at least 2 samples");
    device::Buffer<double> d_x(x.data(), x.size()), d_y(y.data(), y.size()), d_out(1);
    device::throw_status(lattice_correlation_loss(static_cast<std::int64_t>(x.size()), 1, d_x.get(), 1, d_y.get(), 1,
                                                  eps, d_out.get(), 1, nullptr));
    return d_out.download()[0];
}

// numerics.hpp:113-136
inline std::vector<double> swish_rn_jvp(std::span<const double> x, std::span<const double> tangent,
                                        double eps = kDefaultEps) {
    if (!(eps > 0.0)) throw UsageError("eps must be > 0");
    if (x.size() != tangent.size()) throw UsageError("swish_rn_jvp: length mismatch");
    if (x.empty()) throw UsageError("swish_rn_jvp: empty input");
    device::Buffer<double> d_t(tangent.data(), tangent.size());
    return detail::device_op(x, [&](const double* dx, double* dy) {
        device::throw_status(lattice_swish_rn_jvp(1, static_cast<std::int64_t>(x.size()), eps, dx, d_t.get(), dy, 1,
                                                  nullptr));
    });
}

// numerics.hpp:139-144
inline std::vector<double> clip_features(std::span<const double> x, double c) {
    if (!(c > 0.0)) throw UsageError("clip_features: c must be > 0");
    if (x.empty()) return {};
    return detail::device_op(x, [&](const double* dx, double* dy) {
        device::throw_status(lattice_clip_features(static_cast<std::int64_t>(x.size()), dx, c, dy, nullptr));
    });
}

// numerics.hpp:147-156
inline std::vector<double> smooth_labels(std::span<const double> y, double eps_s) {
    if (!(eps_s >= 0.0 && eps_s < 1.0)) throw UsageError("smooth_labels: eps_s must be in [0, 1)");
    if (y.empty()) return {};
    return detail::device_op(y, [&](const double* dy_in, double* dy) {
        device::throw_status(lattice_smooth_labels(static_cast<std::int64_t>(y.size()), dy_in, eps_s, dy, 1, nullptr));
    });
}

// Batched: rows x width fp32 matrix, device pointers, stream-ordered.
inline void swish_rn_rows(const float* x, float* out, std::int64_t rows, std::int64_t width, bool hard = false,
                          double eps = kDefaultEps, cudaStream_t stream = nullptr) {
    device::throw_status(lattice_rownorm(hard ? 2 : 1, rows, width, eps, x, out, 0, stream));
}

}  // namespace lattice
