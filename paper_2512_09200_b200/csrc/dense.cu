// dense.cu -- dense features of consolidated domains: the value side of
// merge_domains (datasets.hpp:144-173) as one gather, writing the union-schema matrix the
// network's dense processor (network.cu) consumes. One thread per output
// element, row-major, coalesced stores; the per-domain column map is tiny and stays in L1.
#include <string>
#include <type_traits>

#include "common.cuh"

namespace lat {
namespace {

template <typename TI, typename TO>
__global__ void merge_dense_kernel(int64_t n, int G, int max_decl, const int32_t* __restrict__ domain,
                                   const TI* __restrict__ values, const int32_t* __restrict__ src_col,
                                   int width, TO* __restrict__ out, unsigned long long* __restrict__ bad) {
    const int64_t total = n * width;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = i / width;
        const int c = (int)(i - b * width);
        const int g = domain[b];
        TI v = 0;  // the pad value (datasets.hpp:138)
        if (g < 0 || g >= G) {
            if (c == 0) atomicMin(bad, (unsigned long long)b);
        } else {
            const int j = src_col[(int64_t)g * width + c];
            if (j >= 0) v = values[b * max_decl + j];
        }
        if constexpr (std::is_same_v<TO, __nv_bfloat16>)
            out[i] = __float2bfloat16_rn((float)v);
        else
            out[i] = (TO)v;
    }
}

}  // namespace
}  // namespace lat

extern "C" {

lattice_status lattice_merge_dense(int64_t n, int32_t domains, int32_t max_declared, const int32_t* domain,
                                   const void* values, int32_t values_dtype, const int32_t* src_col,
                                   int32_t out_width, int32_t out_dtype, void* out, int32_t check,
                                   lattice_stream stream) {
    using namespace lat;
    LAT_REQUIRE(n >= 0 && domains >= 1 && max_declared >= 0 && out_width >= 1, "merge_dense: bad sizes");
    LAT_REQUIRE(values_dtype == LATTICE_F32 || values_dtype == LATTICE_F64, "merge_dense: values must be f32 or f64");
    LAT_REQUIRE(out_dtype == LATTICE_F32 || out_dtype == LATTICE_BF16 || out_dtype == LATTICE_F64,
                "merge_dense: out dtype must be f32, bf16 or f64");
    LAT_REQUIRE(values_dtype == LATTICE_F64 || out_dtype != LATTICE_F64, "merge_dense: f64 out needs f64 values");
    if (n == 0) return LATTICE_OK;
    LAT_REQUIRE(domain && src_col && out && (max_declared == 0 || values), "merge_dense: null pointer");
    unsigned long long* bad = nullptr;
    LAT_CUDA(cudaMallocAsync(&bad, sizeof(*bad), stream));
    LAT_CUDA(cudaMemsetAsync(bad, 0xff, sizeof(*bad), stream));
    const int64_t total = n * out_width;
    const int64_t want = (total + 255) / 256;
    const unsigned grid = (unsigned)(want < (int64_t)num_sms() * 32 ? want : (int64_t)num_sms() * 32);
    const float* vf = static_cast<const float*>(values);
    const double* vd = static_cast<const double*>(values);
    if (values_dtype == LATTICE_F64 && out_dtype == LATTICE_F64)
        merge_dense_kernel<double, double><<<grid, 256, 0, stream>>>(n, domains, max_declared, domain, vd, src_col,
                                                                     out_width, static_cast<double*>(out), bad);
    else if (values_dtype == LATTICE_F64 && out_dtype == LATTICE_F32)
        merge_dense_kernel<double, float><<<grid, 256, 0, stream>>>(n, domains, max_declared, domain, vd, src_col,
                                                                    out_width, static_cast<float*>(out), bad);
    else if (values_dtype == LATTICE_F64)
        merge_dense_kernel<double, __nv_bfloat16><<<grid, 256, 0, stream>>>(
            n, domains, max_declared, domain, vd, src_col, out_width, static_cast<__nv_bfloat16*>(out), bad);
    else if (out_dtype == LATTICE_F32)
        merge_dense_kernel<float, float><<<grid, 256, 0, stream>>>(n, domains, max_declared, domain, vf, src_col,
                                                                   out_width, static_cast<float*>(out), bad);
    else
        merge_dense_kernel<float, __nv_bfloat16><<<grid, 256, 0, stream>>>(
            n, domains, max_declared, domain, vf, src_col, out_width, static_cast<__nv_bfloat16*>(out), bad);
    cudaError_t e = cudaGetLastError();
    unsigned long long host = ~0ull;
    if (e == cudaSuccess && check) {
        e = cudaMemcpyAsync(&host, bad, sizeof(host), cudaMemcpyDeviceToHost, stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    }
    cudaFreeAsync(bad, stream);
    if (e != cudaSuccess) return check_cuda(e, "merge_dense_kernel");
    if (host != ~0ull)
        return set_error(LATTICE_DATA, "merge_dense: record #" + std::to_string(host) + " has a domain outside the schema list",
                         (int64_t)host);
    return LATTICE_OK;
}

}  // extern "C"
