// ktap.cu -- KTAP student-input assembly (ktap.hpp) and
// the remaining element/row ops of the reference's numerics (numerics.hpp:113-156):
// swish_rn_jvp, clip_features, smooth_labels.
//
// Student assembly, one warp per query: hit = the pair's store entry exists and is valid at
// `now` (ktap.hpp:43, inclusive at exactly ttl); the output row is [base || teacher embedding]
// with the teacher block clipped (clip_features) on a hit and all zeros on a
// miss (ktap.hpp:221-229, the output width never depends on hit/miss); the teacher logit is
// label-smoothed on read (ktap.hpp:145-146), NaN on a miss (std::optional empty). The row is
// written in the dtype of the network's dense input, so it feeds lattice_net_forward directly.
// Element ops run in fp64 like the reference: clip and smoothing are bit-exact, the jvp's row
// mean differs from the sequential reference by summation order only.
#include <cmath>
#include <string>

#include "common.cuh"

namespace lat {
namespace {

__device__ __forceinline__ double clampd(double v, double lo, double hi) { return v < lo ? lo : (v > hi ? hi : v); }

template <typename TO>
__global__ void student_kernel(lattice_student_args a, TO* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int W = a.base_dim + a.dim;
    for (int64_t q = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; q < a.n;
         q += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t s = a.slot[q];
        const bool hit = s >= 0 && a.now - a.written_at[s] <= a.ttl_ms;
        TO* row = out + q * W;
        for (int c = lane; c < a.base_dim; c += 32) {
            const float v = a.base[q * a.base_dim + c];
            if constexpr (sizeof(TO) == 4) row[c] = v;
            else row[c] = __float2bfloat16_rn(v);
        }
        const float* emb = hit ? a.store_emb + s * a.dim : nullptr;
        for (int c = lane; c < a.dim; c += 32) {
            double v = hit ? (double)emb[c] : 0.0;
            if (hit && a.clip > 0.0) v = clampd(v, -a.clip, a.clip);
            if constexpr (sizeof(TO) == 4) row[a.base_dim + c] = (float)v;
            else row[a.base_dim + c] = __float2bfloat16_rn((float)v);
        }
        if (lane == 0) {
            if (a.hit) a.hit[q] = hit ? 1 : 0;
            if (a.teacher_logit) {
                double l = hit ? (double)a.store_logit[s] : __longlong_as_double(0x7ff8000000000000ll);
                // explicit roundings: no FMA contraction, the same two roundings as ktap.hpp:146
                if (hit && a.smoothing >= 0.0) l = __dadd_rn(__dmul_rn(l, 1.0 - a.smoothing), a.smoothing / 2.0);
                a.teacher_logit[q] = (float)l;
            }
        }
    }
}

__global__ void clip_kernel(int64_t n, const double* __restrict__ x, double c, double* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = clampd(x[i], -c, c);  // numerics.hpp:142 (std::clamp)
}

__global__ void smooth_kernel(int64_t n, const double* __restrict__ y, double eps, double* __restrict__ out,
                              unsigned long long* __restrict__ bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double v = y[i];
        if (v != 0.0 && v != 1.0) atomicMin(bad, (unsigned long long)i);
        out[i] = __dadd_rn(__dmul_rn(v, 1.0 - eps), eps / 2.0);  // numerics.hpp:154, no FMA contraction
    }
}

__device__ __forceinline__ double sigmoid_d(double z) {  // numerics.hpp:29-33
    if (z >= 0.0) return 1.0 / (1.0 + exp(-z));
    const double e = exp(z);
    return e / (1.0 + e);
}

// one warp per row: numerics.hpp:113-136
// Row statistics in the reference's order: detail::mean_square (numerics.hpp:36-40) is a
// sequential sum of x*x, compiled without FMA contraction on the host; lane 0 of the row's warp
// repeats it with explicit roundings, so the sums -- and with IEEE division and sqrt, rms_norm --
// match the host reference bit for bit (swish_rn differs only where exp() does, <= 1 ulp).
__device__ __forceinline__ void row_sums(const double* __restrict__ xr, const double* __restrict__ tr, int64_t width,
                                         int lane, double& ss, double& dot) {
    ss = 0.0;
    dot = 0.0;
    if (lane == 0) {
        for (int64_t c = 0; c < width; ++c) {
            ss = __dadd_rn(ss, __dmul_rn(xr[c], xr[c]));
            if (tr) dot = __dadd_rn(dot, __dmul_rn(xr[c], tr[c]));
        }
    }
    ss = __shfl_sync(0xffffffffu, ss, 0);
    dot = __shfl_sync(0xffffffffu, dot, 0);
}

__device__ __forceinline__ bool row_nonfinite(const double* __restrict__ xr, const double* __restrict__ tr,
                                              int64_t width, int lane) {
    bool nonfinite = false;
    for (int64_t c = lane; c < width; c += 32) nonfinite |= !isfinite(xr[c]) || (tr && !isfinite(tr[c]));
    return __any_sync(0xffffffffu, nonfinite);
}

// one warp per row: numerics.hpp:113-136
__global__ void jvp_kernel(int64_t rows, int64_t width, double eps, const double* __restrict__ x,
                           const double* __restrict__ t, double* __restrict__ out, unsigned long long* __restrict__ bad) {
    const int lane = threadIdx.x & 31;
    for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < rows;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const double* xr = x + r * width;
        const double* tr = t + r * width;
        if (row_nonfinite(xr, tr, width, lane) && lane == 0) atomicMin(bad, (unsigned long long)r);
        double ss, dot;
        row_sums(xr, tr, width, lane, ss, dot);
        const double n = (double)width;
        const double d = sqrt(__dadd_rn(ss / n, eps));
        dot /= n;
        const double d3 = __dmul_rn(__dmul_rn(d, d), d);
        for (int64_t c = lane; c < width; c += 32) {
            const double rv = xr[c] / d;
            const double dr = __dsub_rn(tr[c] / d, __dmul_rn(xr[c], dot) / d3);
            const double s = sigmoid_d(rv);
            out[r * width + c] = __dmul_rn(__dmul_rn(s, __dadd_rn(1.0, __dmul_rn(rv, __dsub_rn(1.0, s)))), dr);
        }
    }
}

// rms_norm / swish_rn / swish_rn_hard in fp64 (numerics.hpp:81-107), one warp per row
__global__ void rownorm64_kernel(int mode, int64_t rows, int64_t width, double eps, const double* __restrict__ x,
                                 double* __restrict__ out, unsigned long long* __restrict__ bad) {
    const int lane = threadIdx.x & 31;
    for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < rows;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const double* xr = x + r * width;
        if (row_nonfinite(xr, nullptr, width, lane) && lane == 0) atomicMin(bad, (unsigned long long)r);
        double ss, unused;
        row_sums(xr, nullptr, width, lane, ss, unused);
        const double denom = sqrt(__dadd_rn(ss / (double)width, eps));
        for (int64_t c = lane; c < width; c += 32) {
            double v = xr[c] / denom;
            if (mode == 1) v = __dmul_rn(v, sigmoid_d(v));
            if (mode == 2) v = __dmul_rn(v, clampd(__dadd_rn(v, 3.0) / 6.0, 0.0, 1.0));
            out[r * width + c] = v;
        }
    }
}

unsigned grid_of(int64_t threads) {
    const int64_t b = (threads + 255) / 256;
    const int64_t cap = (int64_t)num_sms() * 16;
    return (unsigned)(b < 1 ? 1 : (b > cap ? cap : b));
}

lattice_status flag_status(unsigned long long* flag, cudaStream_t st, bool check, unsigned long long* host) {
    *host = ~0ull;
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess && check) {
        e = cudaMemcpyAsync(host, flag, sizeof(*host), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    }
    cudaFreeAsync(flag, st);
    return e == cudaSuccess ? LATTICE_OK : check_cuda(e, "ktap kernels");
}

}  // namespace
}  // namespace lat

extern "C" {

lattice_status lattice_student_inputs(const lattice_student_args* a, lattice_stream stream) {
    using namespace lat;
    LAT_REQUIRE(a != nullptr, "student_inputs: null args");
    LAT_REQUIRE(a->n >= 0 && a->base_dim >= 0 && a->dim > 0, "StoreConfig: dimension must be positive");
    LAT_REQUIRE(a->ttl_ms > 0, "StoreConfig: ttl must be positive");                    // ktap.hpp:115
    LAT_REQUIRE(a->smoothing < 1.0, "StoreConfig: label smoothing must be in [0, 1)");  // ktap.hpp:118
    LAT_REQUIRE(a->clip >= 0.0, "clip_features: c must be > 0");
    LAT_REQUIRE(a->out_dtype == LATTICE_F32 || a->out_dtype == LATTICE_BF16, "student_inputs: out dtype");
    if (a->n == 0) return LATTICE_OK;
    LAT_REQUIRE(a->slot && a->store_emb && a->written_at && a->out && (a->base_dim == 0 || a->base) &&
                    (!a->teacher_logit || a->store_logit),
                "student_inputs: null pointer");
    const unsigned grid = grid_of(a->n * 32);
    if (a->out_dtype == LATTICE_F32)
        student_kernel<float><<<grid, 256, 0, stream>>>(*a, static_cast<float*>(a->out));
    else
        student_kernel<__nv_bfloat16><<<grid, 256, 0, stream>>>(*a, static_cast<__nv_bfloat16*>(a->out));
    LAT_CUDA(cudaGetLastError());
    return LATTICE_OK;
}

lattice_status lattice_clip_features(int64_t n, const double* x, double c, double* out, lattice_stream stream) {
    using namespace lat;
    LAT_REQUIRE(c > 0.0, "clip_features: c must be > 0");  // numerics.hpp:140
    if (n <= 0) return LATTICE_OK;
    LAT_REQUIRE(x && out, "clip_features: null pointer");
    clip_kernel<<<grid_of(n), 256, 0, stream>>>(n, x, c, out);
    LAT_CUDA(cudaGetLastError());
    return LATTICE_OK;
}

lattice_status lattice_smooth_labels(int64_t n, const double* y, double eps_s, double* out, int32_t check,
                                     lattice_stream stream) {
    using namespace lat;
    LAT_REQUIRE(eps_s >= 0.0 && eps_s < 1.0, "smooth_labels: eps_s must be in [0, 1)");  // numerics.hpp:148
    if (n <= 0) return LATTICE_OK;
    LAT_REQUIRE(y && out, "smooth_labels: null pointer");
    unsigned long long* bad = nullptr;
    LAT_CUDA(cudaMallocAsync(&bad, sizeof(*bad), stream));
    LAT_CUDA(cudaMemsetAsync(bad, 0xff, sizeof(*bad), stream));
    smooth_kernel<<<grid_of(n), 256, 0, stream>>>(n, y, eps_s, out, bad);
    unsigned long long host;
    lattice_status s = flag_status(bad, stream, check != 0, &host);
    if (s != LATTICE_OK) return s;
    if (host != ~0ull)  // numerics.hpp:152 (a UsageError in the reference)
        return set_error(LATTICE_USAGE, "smooth_labels: labels must be 0 or 1", (int64_t)host);
    return LATTICE_OK;
}

lattice_status lattice_rownorm_f64(int32_t mode, int64_t rows, int64_t width, double eps, const double* x,
                                   double* out, int32_t check, lattice_stream stream) {
    using namespace lat;
    LAT_REQUIRE(mode >= 0 && mode <= 2, "rownorm: mode must be 0, 1 or 2");
    LAT_REQUIRE(eps > 0.0, "eps must be > 0");         // numerics.hpp:20
    LAT_REQUIRE(width > 0, "rms_norm: empty input");   // numerics.hpp:83
    if (rows <= 0) return LATTICE_OK;
    LAT_REQUIRE(x && out, "rownorm: null pointer");
    unsigned long long* bad = nullptr;
    LAT_CUDA(cudaMallocAsync(&bad, sizeof(*bad), stream));
    LAT_CUDA(cudaMemsetAsync(bad, 0xff, sizeof(*bad), stream));
    rownorm64_kernel<<<grid_of(rows * 32), 256, 0, stream>>>(mode, rows, width, eps, x, out, bad);
    unsigned long long host;
    lattice_status s = flag_status(bad, stream, check != 0, &host);
    if (s != LATTICE_OK) return s;
    if (host != ~0ull) return set_error(LATTICE_DATA, "rms_norm: non-finite input", (int64_t)host);  // numerics.hpp:84
    return LATTICE_OK;
}

lattice_status lattice_swish_rn_jvp(int64_t rows, int64_t width, double eps, const double* x, const double* tangent,
                                    double* out, int32_t check, lattice_stream stream) {
    using namespace lat;
    LAT_REQUIRE(eps > 0.0, "eps must be > 0");                      // numerics.hpp:116
    LAT_REQUIRE(width > 0, "swish_rn_jvp: empty input");            // numerics.hpp:118
    if (rows <= 0) return LATTICE_OK;
    LAT_REQUIRE(x && tangent && out, "swish_rn_jvp: null pointer");
    unsigned long long* bad = nullptr;
    LAT_CUDA(cudaMallocAsync(&bad, sizeof(*bad), stream));
    LAT_CUDA(cudaMemsetAsync(bad, 0xff, sizeof(*bad), stream));
    jvp_kernel<<<grid_of(rows * 32), 256, 0, stream>>>(rows, width, eps, x, tangent, out, bad);
    unsigned long long host;
    lattice_status s = flag_status(bad, stream, check != 0, &host);
    if (s != LATTICE_OK) return s;
    if (host != ~0ull) return set_error(LATTICE_DATA, "swish_rn_jvp: non-finite input", (int64_t)host);
    return LATTICE_OK;
}

}  // extern "C"
