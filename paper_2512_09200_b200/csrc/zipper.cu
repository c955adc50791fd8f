// zipper.cu -- K5: attribution-window assignment + per-window labels, one thread per
// impression, bit-exact with lattice::assign_window / zip_dataset
// (proj/include/lattice/datasets.hpp:179-249).
//
//   signature  = BE32(|user|) user BE32(|ad|) ad BE64(ts)      (datasets.hpp:181-184)
//   h          = XXH64(signature, seed)                          (core.hpp:84)
//   u          = (h >> 11) * 2^-53                               (datasets.hpp:186, exact)
//   window     = first i < W-1 with u < cum_i, else W-1          (datasets.hpp:188-193)
//   cum_i      = the same left-to-right double sums, computed once on the host
//   label[t,w] = conv present && (conv - ts) <= duration_w      (datasets.hpp:231-242)
//   conv - ts < 0 -> DataError for the lowest (record, task)     (datasets.hpp:236-238)
#include <cmath>
#include <cstring>
#include <string>

#include "common.cuh"

namespace lat {
namespace {

constexpr int kMaxWindows = 255;

struct ZipConst {
    double cum[kMaxWindows];
    int64_t dur[kMaxWindows];
};

// The signature as a virtual byte string: no per-thread buffer, any length.
struct SigSrc {
    const uint8_t* u;
    const uint8_t* a;
    uint32_t ul, al;
    uint64_t ts;
    __device__ __forceinline__ uint8_t u8(uint64_t p) const {
        if (p < 4) return (uint8_t)(ul >> (8 * (3 - p)));
        p -= 4;
        if (p < ul) return u[p];
        p -= ul;
        if (p < 4) return (uint8_t)(al >> (8 * (3 - p)));
        p -= 4;
        if (p < al) return a[p];
        p -= al;
        return (uint8_t)(ts >> (8 * (7 - p)));
    }
    __device__ __forceinline__ uint32_t u32(uint64_t p) const {
        return (uint32_t)u8(p) | ((uint32_t)u8(p + 1) << 8) | ((uint32_t)u8(p + 2) << 16) |
               ((uint32_t)u8(p + 3) << 24);
    }
    __device__ __forceinline__ uint64_t u64(uint64_t p) const {
        return (uint64_t)u32(p) | ((uint64_t)u32(p + 4) << 32);
    }
};

__global__ void __launch_bounds__(256) zipper_kernel(
    int64_t n, const uint8_t* __restrict__ ub, const int64_t* __restrict__ uo,
    const uint8_t* __restrict__ ab, const int64_t* __restrict__ ao, const int64_t* __restrict__ ts,
    int T, const int64_t* __restrict__ conv, const uint8_t* __restrict__ pres, int W, uint64_t seed,
    const __grid_constant__ ZipConst zc, uint8_t* __restrict__ window, uint8_t* __restrict__ labels,
    uint8_t* __restrict__ routed, unsigned long long* __restrict__ err) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t us = uo[i], as = ao[i];
        SigSrc src{ub + us, ab + as, (uint32_t)(uo[i + 1] - us), (uint32_t)(ao[i + 1] - as),
                   (uint64_t)ts[i]};
        const uint64_t len = 16ull + src.ul + src.al;
        const uint64_t h = xxh64_src(src, len, seed);
        const double u = (double)(h >> 11) * 0x1.0p-53;
        int w = W - 1;
        for (int j = 0; j + 1 < W; ++j)
            if (u < zc.cum[j]) {
                w = j;
                break;
            }
        window[i] = (uint8_t)w;
        for (int t = 0; t < T; ++t) {
            const size_t it = (size_t)i * T + t;
            uint8_t* lab = labels + it * W;
            uint8_t r = 0;
            if (pres[it]) {
                const int64_t delay = (int64_t)((uint64_t)conv[it] - (uint64_t)ts[i]);
                if (delay < 0) atomicMin(err, (unsigned long long)it);
                for (int j = 0; j < W; ++j) {
                    const uint8_t v = delay >= 0 && delay <= zc.dur[j];
                    lab[j] = v;
                    if (j == w) r = v;
                }
            } else {
                for (int j = 0; j < W; ++j) lab[j] = 0;
            }
            if (routed) routed[it] = r;
        }
    }
}

constexpr uint64_t kTagUser = 0x55534552ull, kTagAd = 0x41442020ull, kTagConvP = 0x43565020ull,
                   kTagConvD = 0x43564420ull;

__device__ __forceinline__ void put_dec(uint8_t* dst, uint64_t v, int digits) {
    for (int i = digits - 1; i >= 0; --i) {
        dst[i] = (uint8_t)('0' + v % 10);
        v /= 10;
    }
}

__global__ void synth_impressions_kernel(int64_t n, int T, uint64_t seed, uint8_t* ub, int64_t* uo, uint8_t* ab,
                                         int64_t* ao, int64_t* ts, int64_t* conv, uint8_t* pres) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        ub[9 * i] = 'u';
        put_dec(ub + 9 * i + 1, gen_u64(seed, kTagUser, (uint64_t)i) % 100000000ull, 8);
        ab[7 * i] = 'a';
        put_dec(ab + 7 * i + 1, gen_u64(seed, kTagAd, (uint64_t)i) % 1000000ull, 6);
        uo[i] = 9 * i;
        ao[i] = 7 * i;
        if (i == n - 1) {
            uo[n] = 9 * n;
            ao[n] = 7 * n;
        }
        const int64_t t0 = 1700000000000ll + 37 * i;
        ts[i] = t0;
        for (int t = 0; t < T; ++t) {
            const uint64_t k = (uint64_t)i * T + t;
            pres[k] = (uint8_t)(gen_u64(seed, kTagConvP, k) % 10 < 3);
            conv[k] = t0 + (int64_t)(gen_u64(seed, kTagConvD, k) % (8ull * 86400000ull));
        }
    }
}

__global__ void route_heads_kernel(int64_t B, int T, int W, const float* __restrict__ logits,
                                   const uint8_t* __restrict__ window, float* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < B * T; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = i / T;
        const int t = (int)(i - b * T);
        out[i] = logits[b * (int64_t)T * W + (int64_t)t * W + window[b]];
    }
}

}  // namespace
}  // namespace lat

extern "C" {

lattice_status lattice_synth_impressions(int64_t n, int32_t T, uint64_t seed, uint8_t* ub, int64_t* uo, uint8_t* ab,
                                         int64_t* ao, int64_t* ts, int64_t* conv, uint8_t* pres,
                                         lattice_stream stream) {
    LAT_REQUIRE(n > 0 && T >= 0 && ub && uo && ab && ao && ts && (T == 0 || (conv && pres)),
                "synth_impressions: bad args");
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    lat::synth_impressions_kernel<<<(unsigned)blocks, 256, 0, stream>>>(n, T, seed, ub, uo, ab, ao, ts, conv, pres);
    LAT_CUDA(cudaGetLastError());
    return LATTICE_OK;
}

lattice_status lattice_route_heads(int64_t B, int32_t T, int32_t W, const float* logits, const uint8_t* window,
                                   float* out, lattice_stream stream) {
    LAT_REQUIRE(B >= 0 && T > 0 && W > 0 && W <= 255, "route_heads: bad sizes");
    if (B == 0) return LATTICE_OK;
    LAT_REQUIRE(logits && window && out, "route_heads: null pointer");
    int64_t blocks = (B * T + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    lat::route_heads_kernel<<<(unsigned)blocks, 256, 0, stream>>>(B, T, W, logits, window, out);
    LAT_CUDA(cudaGetLastError());
    return LATTICE_OK;
}

lattice_status lattice_zipper_validate(int32_t W, const int64_t* dur, const double* p) {
    // datasets.hpp:60-84 (name checks live in the C++ shim)
    if (W < 1) return lat::set_error(LATTICE_USAGE, "ZipperConfig: no windows");
    if (W > lat::kMaxWindows)
        return lat::set_error(LATTICE_USAGE, "ZipperConfig: at most 255 windows are supported");
    if (!dur || !p) return lat::set_error(LATTICE_USAGE, "ZipperConfig: null durations/probabilities");
    int64_t prev = 0;
    for (int i = 0; i < W; ++i) {
        if (dur[i] <= (i == 0 ? 0 : prev))
            return lat::set_error(LATTICE_USAGE,
                                  "ZipperConfig: window durations must be positive and strictly increasing");
        prev = dur[i];
    }
    double sum = 0.0;
    for (int i = 0; i < W; ++i) {
        if (!(p[i] >= 0.0) || !std::isfinite(p[i]))
            return lat::set_error(LATTICE_USAGE, "ZipperConfig: probabilities must be non-negative");
        sum += p[i];
    }
    if (std::abs(sum - 1.0) > 1e-9)
        return lat::set_error(LATTICE_USAGE, "ZipperConfig: probabilities must sum to 1");
    return LATTICE_OK;
}

lattice_status lattice_zipper_assign_labels(const lattice_zip_args* a, lattice_stream stream) {
    LAT_REQUIRE(a != nullptr, "lattice_zipper_assign_labels: null args");
    lattice_status st = lattice_zipper_validate(a->windows, a->durations_host, a->probabilities_host);
    if (st != LATTICE_OK) return st;
    LAT_REQUIRE(a->n >= 0 && a->tasks >= 0, "zip: negative sizes");
    if (a->n == 0) return LATTICE_OK;
    LAT_REQUIRE(a->user_off && a->ad_off && a->ts && a->window, "zip: null column");
    LAT_REQUIRE(a->tasks == 0 || (a->conv && a->conv_present && a->labels), "zip: null task column");

    lat::ZipConst zc;
    std::memset(&zc, 0, sizeof(zc));
    double cum = 0.0;
    for (int i = 0; i + 1 < a->windows; ++i) {  // datasets.hpp:188-190, same summation order
        cum += a->probabilities_host[i];
        zc.cum[i] = cum;
    }
    for (int i = 0; i < a->windows; ++i) zc.dur[i] = a->durations_host[i];

    unsigned long long* err = nullptr;
    LAT_CUDA(cudaMallocAsync(&err, sizeof(unsigned long long), stream));
    LAT_CUDA(cudaMemsetAsync(err, 0xff, sizeof(unsigned long long), stream));
    const int threads = 256;
    int64_t blocks = (a->n + threads - 1) / threads;
    if (blocks > 8 * 148 * 8) blocks = 8 * 148 * 8;
    lat::zipper_kernel<<<(unsigned)blocks, threads, 0, stream>>>(
        a->n, a->user_bytes, a->user_off, a->ad_bytes, a->ad_off, a->ts, a->tasks, a->conv,
        a->conv_present, a->windows, a->seed, zc, a->window, a->labels, a->routed, err);
    cudaError_t le = cudaGetLastError();
    unsigned long long host_err = ~0ull;
    if (le == cudaSuccess && a->check) {
        le = cudaMemcpyAsync(&host_err, err, sizeof(host_err), cudaMemcpyDeviceToHost, stream);
        if (le == cudaSuccess) le = cudaStreamSynchronize(stream);
    }
    cudaFreeAsync(err, stream);
    if (le != cudaSuccess) return lat::check_cuda(le, "zipper_kernel");
    if (host_err != ~0ull) {
        const int64_t rec = (int64_t)(host_err / (unsigned long long)a->tasks);
        const int64_t task = (int64_t)(host_err % (unsigned long long)a->tasks);
        return lat::set_error(LATTICE_DATA,
                              "zip_dataset: record #" + std::to_string(rec) + " task #" +
                                  std::to_string(task) + " converts before its impression",
                              (int64_t)host_err);  // record * tasks + task
    }
    return LATTICE_OK;
}

}  // extern "C"
