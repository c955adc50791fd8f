// capi.cu -- C ABI plumbing: thread-local error state, version, batched stable_hash.
#include <cstdio>
#include <string>

#include "common.cuh"

namespace lat {
namespace {
thread_local std::string g_msg;
thread_local int64_t g_index = -1;
}  // namespace

lattice_status set_error(lattice_status st, const std::string& msg, int64_t index) {
    g_msg = msg;
    g_index = index;
    return st;
}

lattice_status check_cuda(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return LATTICE_OK;
    return set_error(LATTICE_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

namespace {
struct PackedSrc {
    const uint8_t* p;
    __device__ uint8_t u8(uint64_t i) const { return p[i]; }
    __device__ uint32_t u32(uint64_t i) const {
        return (uint32_t)p[i] | ((uint32_t)p[i + 1] << 8) | ((uint32_t)p[i + 2] << 16) |
               ((uint32_t)p[i + 3] << 24);
    }
    __device__ uint64_t u64(uint64_t i) const {
        return (uint64_t)u32(i) | ((uint64_t)u32(i + 4) << 32);
    }
};

__global__ void hash_kernel(int64_t n, const uint8_t* __restrict__ bytes,
                            const int64_t* __restrict__ off, uint64_t seed,
                            uint64_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = off[i];
        PackedSrc src{bytes + s};
        out[i] = xxh64_src(src, (uint64_t)(off[i + 1] - s), seed);
    }
}
}  // namespace
}  // namespace lat

extern "C" {

const char* lattice_last_error(void) { return lat::g_msg.c_str(); }
int64_t lattice_last_error_index(void) { return lat::g_index; }
int lattice_abi_version(void) { return 4; }

lattice_status lattice_stable_hash(int64_t n, const uint8_t* bytes, const int64_t* off,
                                   uint64_t seed, uint64_t* out, lattice_stream stream) {
    LAT_REQUIRE(n >= 0, "lattice_stable_hash: negative n");
    if (n == 0) return LATTICE_OK;
    LAT_REQUIRE(off && out, "lattice_stable_hash: null pointer");
    const int threads = 256;
    const int64_t blocks = (n + threads - 1) / threads;
    lat::hash_kernel<<<(unsigned)(blocks < 65535 ? blocks : 65535), threads, 0, stream>>>(
        n, bytes, off, seed, out);
    LAT_CUDA(cudaGetLastError());
    return LATTICE_OK;
}

}  // extern "C"
