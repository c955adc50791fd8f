// objective.cu -- post-tower batch reductions: the window-routed loss
// inputs, correlation_loss (numerics.hpp:46-78) and window_routing_summary
// (datasets.hpp:256-283) over a whole batch on the device.
//
// correlation_loss keeps the reference's arithmetic: fp64, population moments, two passes
// (means, then centred sums), 1.0 when either side is constant, clamped to [0, 2]. The sums
// are deterministic: every pass reduces fixed per-block partials in a fixed order (no float
// atomics), so repeated calls return identical bits; against the reference's sequential sums
// the difference is rounding order only (~1e-15 relative). Window counts are integers (exact).
//
// Launch shape: grid (NB, cols) -- blockIdx.y is the column (task), each block reduces a
// contiguous range of samples; a one-block-per-column kernel folds the partials. The routed
// objectives read the logits / labels of the assigned window and the
// prediction p = stable_sigmoid(z) (numerics.hpp:29-33) in fp64.
#include <string>

#include "common.cuh"

namespace lat {
namespace {

constexpr int kObjThreads = 256;

__device__ __forceinline__ double block_sum(double v, double* sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < kObjThreads / 32; ++i) s += sh[i];  // fixed order
    return s;  // valid in thread 0
}

__device__ __forceinline__ double sigmoid_d(double z) {  // numerics.hpp:29-33
    if (z >= 0.0) return 1.0 / (1.0 + exp(-z));
    const double e = exp(z);
    return e / (1.0 + e);
}

// (x, y) of sample b, column t
struct DenseXY {
    const double* x;
    int64_t ldx;
    const double* y;
    int64_t ldy;
    __device__ void get(int64_t b, int t, double& xv, double& yv) const {
        xv = x[b * ldx + t];
        yv = y[b * ldy + t];
    }
};
struct RoutedXY {  // x = routed label, y = predicted probability
    const float* logits;
    const uint8_t* window;
    const uint8_t* labels;
    int T, W;
    float* routed;  // optional: routed logits [n][T] (written in pass 1)
    __device__ void get(int64_t b, int t, double& xv, double& yv) const {
        int w = window[b];
        w = w < W ? w : W - 1;
        const float z = logits[(b * T + t) * W + w];
        xv = (double)labels[(b * T + t) * W + w];
        yv = sigmoid_d((double)z);
    }
};

// pass 1: per-block sums of x, y and the finite check; pass 2 (means given): centred sums
template <typename XY, bool CENTRED>
__global__ void __launch_bounds__(kObjThreads) moments_kernel(XY xy, int64_t n, const double* __restrict__ means,
                                                              double* __restrict__ part, int* __restrict__ bad) {
    __shared__ double sh[kObjThreads / 32];
    const int t = blockIdx.y;
    const int64_t per = (n + gridDim.x - 1) / gridDim.x;
    const int64_t lo = blockIdx.x * per, hi = lo + per < n ? lo + per : n;
    double a = 0.0, b = 0.0, c = 0.0;
    double mx = 0.0, my = 0.0;
    if (CENTRED) {
        mx = means[2 * t];
        my = means[2 * t + 1];
    }
    bool nonfinite = false;
    for (int64_t i = lo + threadIdx.x; i < hi; i += kObjThreads) {
        double xv, yv;
        xy.get(i, t, xv, yv);
        if (CENTRED) {
            const double dx = xv - mx, dy = yv - my;
            a += dx * dy;
            b += dx * dx;
            c += dy * dy;
        } else {
            nonfinite |= !isfinite(xv) || !isfinite(yv);
            a += xv;
            b += yv;
        }
    }
    if (!CENTRED && nonfinite) atomicExch(bad, 1);
    double* out = part + ((int64_t)t * gridDim.x + blockIdx.x) * 3;
    const double sa = block_sum(a, sh);
    if (threadIdx.x == 0) out[0] = sa;
    const double sb = block_sum(b, sh);
    if (threadIdx.x == 0) out[1] = sb;
    if (CENTRED) {
        const double sc = block_sum(c, sh);
        if (threadIdx.x == 0) out[2] = sc;
    }
}

// one block per column: fold the NB partials in order, then means (pass 1) or the loss (pass 2)
template <bool FINAL>
__global__ void fold_kernel(int nb, int64_t n, double eps, const double* __restrict__ part,
                            double* __restrict__ means, double* __restrict__ out) {
    const int t = blockIdx.x;
    if (threadIdx.x != 0) return;
    double a = 0.0, b = 0.0, c = 0.0;
    for (int i = 0; i < nb; ++i) {
        const double* q = part + ((int64_t)t * nb + i) * 3;
        a += q[0];
        b += q[1];
        if (FINAL) c += q[2];
    }
    const double dn = (double)n;
    if (!FINAL) {
        means[2 * t] = a / dn;
        means[2 * t + 1] = b / dn;
        return;
    }
    const double cov = a / dn;
    const double sx = sqrt(b / dn), sy = sqrt(c / dn);
    if (sx == 0.0 || sy == 0.0) {
        out[t] = 1.0;
        return;
    }
    const double loss = 1.0 - cov / (sx * sy + eps);
    out[t] = loss < 0.0 ? 0.0 : (loss > 2.0 ? 2.0 : loss);
}

// window_routing_summary: counts[w], positives[w][t] (own-window labels); shared-memory
// histograms, integer atomics (exact). Optional routed logits.
__global__ void __launch_bounds__(kObjThreads) summary_kernel(int64_t n, int T, int W, const uint8_t* __restrict__ window,
                                                              const uint8_t* __restrict__ labels,
                                                              const float* __restrict__ logits, float* __restrict__ routed,
                                                              unsigned long long* __restrict__ counts,
                                                              unsigned long long* __restrict__ positives,
                                                              int* __restrict__ bad) {
    extern __shared__ unsigned int hist[];  // [W] counts, then [W][T] positives
    for (int i = threadIdx.x; i < W * (T + 1); i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < n; b += (int64_t)gridDim.x * blockDim.x) {
        int w = window[b];
        if (w >= W) {
            atomicExch(bad, 1);
            w = W - 1;
        }
        atomicAdd(&hist[w], 1u);
        for (int t = 0; t < T; ++t) {
            const uint8_t l = labels[(b * T + t) * W + w];
            if (l) atomicAdd(&hist[W + w * T + t], 1u);
            if (routed) routed[b * T + t] = logits[(b * T + t) * W + w];
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < W * (T + 1); i += blockDim.x) {
        const unsigned int v = hist[i];
        if (v) atomicAdd(i < W ? &counts[i] : &positives[i - W], (unsigned long long)v);
    }
}

int blocks_for(int64_t n) {
    const int64_t b = (n + 4 * kObjThreads - 1) / (4 * kObjThreads);
    return (int)(b < 1 ? 1 : (b > num_sms() ? num_sms() : b));
}

template <typename XY>
lattice_status correlation(const XY& xy, int64_t n, int cols, double eps, double* out, int* bad, cudaStream_t st) {
    const int nb = blocks_for(n);
    double* ws = nullptr;  // partials [cols][nb][3], means [cols][2]
    const size_t words = (size_t)cols * nb * 3 + (size_t)cols * 2;
    LAT_CUDA(cudaMallocAsync(&ws, words * sizeof(double), st));
    double* part = ws;
    double* means = ws + (size_t)cols * nb * 3;
    const dim3 grid((unsigned)nb, (unsigned)cols);
    moments_kernel<XY, false><<<grid, kObjThreads, 0, st>>>(xy, n, nullptr, part, bad);
    fold_kernel<false><<<cols, 32, 0, st>>>(nb, n, eps, part, means, nullptr);
    moments_kernel<XY, true><<<grid, kObjThreads, 0, st>>>(xy, n, means, part, bad);
    fold_kernel<true><<<cols, 32, 0, st>>>(nb, n, eps, part, means, out);
    const cudaError_t e = cudaGetLastError();
    cudaFreeAsync(ws, st);
    return e == cudaSuccess ? LATTICE_OK : check_cuda(e, "correlation kernels");
}

lattice_status read_flag(int* flag, cudaStream_t st, int* host) {
    *host = 0;
    cudaError_t e = cudaMemcpyAsync(host, flag, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    return e == cudaSuccess ? LATTICE_OK : check_cuda(e, "flag readback");
}

lattice_status summary(int64_t n, int T, int W, const uint8_t* window, const uint8_t* labels, const float* logits,
                       float* routed, int64_t* counts, int64_t* positives, int* bad, cudaStream_t st) {
    LAT_CUDA(cudaMemsetAsync(counts, 0, sizeof(int64_t) * W, st));
    LAT_CUDA(cudaMemsetAsync(positives, 0, sizeof(int64_t) * W * T, st));
    const size_t smem = sizeof(unsigned int) * W * (T + 1);
    const int64_t want = (n + kObjThreads - 1) / kObjThreads;
    const int grid = (int)(want < 1 ? 1 : (want > 2 * num_sms() ? 2 * num_sms() : want));
    summary_kernel<<<grid, kObjThreads, smem, st>>>(n, T, W, window, labels, logits, routed,
                                                    reinterpret_cast<unsigned long long*>(counts),
                                                    reinterpret_cast<unsigned long long*>(positives), bad);
    LAT_CUDA(cudaGetLastError());
    return LATTICE_OK;
}

}  // namespace
}  // namespace lat

extern "C" {

lattice_status lattice_correlation_loss(int64_t n, int32_t cols, const double* x, int64_t ldx, const double* y,
                                        int64_t ldy, double eps, double* out, int32_t check, lattice_stream stream) {
    using namespace lat;
    LAT_REQUIRE(eps > 0.0, "eps must be > 0");                                   // numerics.hpp:21
    LAT_REQUIRE(n >= 2, "correlation_loss: need at least 2 samples");            // numerics.hpp:52
    LAT_REQUIRE(cols >= 1 && cols <= 65535 && ldx >= cols && ldy >= cols, "correlation_loss: bad columns/strides");
    LAT_REQUIRE(x && y && out, "correlation_loss: null pointer");
    int* bad = nullptr;
    LAT_CUDA(cudaMallocAsync(&bad, sizeof(int), stream));
    LAT_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), stream));
    lattice_status s = correlation(DenseXY{x, ldx, y, ldy}, n, cols, eps, out, bad, stream);
    int host = 0;
    if (s == LATTICE_OK && check) s = read_flag(bad, stream, &host);
    cudaFreeAsync(bad, stream);
    if (s != LATTICE_OK) return s;
    if (host) return set_error(LATTICE_DATA, "correlation_loss: non-finite input");  // numerics.hpp:25
    return LATTICE_OK;
}

lattice_status lattice_window_summary(int64_t n, int32_t tasks, int32_t windows, const uint8_t* window,
                                      const uint8_t* labels, int64_t* counts, int64_t* positives, int32_t check,
                                      lattice_stream stream) {
    using namespace lat;
    LAT_REQUIRE(n >= 0 && tasks >= 0 && windows >= 1 && windows <= 255 && (int64_t)windows * (tasks + 1) <= 8192,
                "window_summary: bad sizes");
    LAT_REQUIRE(counts && positives && (n == 0 || (window && (tasks == 0 || labels))), "window_summary: null pointer");
    int* bad = nullptr;
    LAT_CUDA(cudaMallocAsync(&bad, sizeof(int), stream));
    LAT_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), stream));
    lattice_status s = summary(n, tasks, windows, window, labels, nullptr, nullptr, counts, positives, bad, stream);
    int host = 0;
    if (s == LATTICE_OK && check) s = read_flag(bad, stream, &host);
    cudaFreeAsync(bad, stream);
    if (s != LATTICE_OK) return s;
    if (host) return set_error(LATTICE_USAGE, "window_routing_summary: dataset not produced by zip_dataset");
    return LATTICE_OK;
}

lattice_status lattice_routed_objectives(const lattice_objective_args* a, lattice_stream stream) {
    using namespace lat;
    LAT_REQUIRE(a != nullptr, "routed_objectives: null args");
    LAT_REQUIRE(a->eps > 0.0, "eps must be > 0");
    LAT_REQUIRE(a->n >= 2, "correlation_loss: need at least 2 samples");
    LAT_REQUIRE(a->tasks >= 1 && a->windows >= 1 && a->windows <= 255 && (int64_t)a->windows * (a->tasks + 1) <= 8192,
                "routed_objectives: bad sizes");
    LAT_REQUIRE(a->logits && a->window && a->labels && a->corr && a->counts && a->positives,
                "routed_objectives: null pointer");
    int* bad = nullptr;  // [0] window out of range, [1] non-finite
    LAT_CUDA(cudaMallocAsync(&bad, 2 * sizeof(int), stream));
    LAT_CUDA(cudaMemsetAsync(bad, 0, 2 * sizeof(int), stream));
    lattice_status s = summary(a->n, a->tasks, a->windows, a->window, a->labels, a->logits, a->routed, a->counts,
                               a->positives, bad, stream);
    if (s == LATTICE_OK)
        s = correlation(RoutedXY{a->logits, a->window, a->labels, a->tasks, a->windows, nullptr}, a->n, a->tasks,
                        a->eps, a->corr, bad + 1, stream);
    int host[2] = {0, 0};
    if (s == LATTICE_OK && a->check) {
        cudaError_t e = cudaMemcpyAsync(host, bad, sizeof(host), cudaMemcpyDeviceToHost, stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
        if (e != cudaSuccess) s = check_cuda(e, "flag readback");
    }
    cudaFreeAsync(bad, stream);
    if (s != LATTICE_OK) return s;
    if (host[0]) return set_error(LATTICE_USAGE, "window_routing_summary: dataset not produced by zip_dataset");
    if (host[1]) return set_error(LATTICE_DATA, "correlation_loss: non-finite input");
    return LATTICE_OK;
}

}  // extern "C"
