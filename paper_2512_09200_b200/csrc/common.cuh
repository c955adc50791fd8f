// common.cuh -- shared device helpers: XXH64 (core.hpp:84-139 semantics), the counter-based
// synthetic generator, bf16 conversion, warp reductions, error plumbing for the C ABI.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <string>

#include "../../include/lattice_b200.h"

namespace lat {

// ---- host-side status plumbing (capi.cpp owns the thread-local state) -------------------
lattice_status set_error(lattice_status st, const std::string& msg, int64_t index = -1);
lattice_status check_cuda(cudaError_t e, const char* what);
#define LAT_CUDA(call)                                                              \
    do {                                                                            \
        cudaError_t _e = (call);                                                    \
        if (_e != cudaSuccess) return ::lat::check_cuda(_e, #call);                 \
    } while (0)
#define LAT_REQUIRE(cond, msg)                                                      \
    do {                                                                            \
        if (!(cond)) return ::lat::set_error(LATTICE_USAGE, (msg));                 \
    } while (0)

// embedding_bag.cu: the stable domain bucketing behind lattice_domain_bucket, with a caller-owned
// workspace of bucket_workspace(B, G) int32 (lattice_net keeps one: no allocation per step)
int64_t bucket_workspace(int64_t B, int G);
// (bad != nullptr: the lowest sample index whose domain is outside [0, G) is atomicMin'ed into
// *bad, initialised by the caller to ~0; such samples count as domain 0 either way)
lattice_status bucket_ws(int64_t B, int G, const int32_t* dom, int32_t* pos, int32_t* order, int32_t* seg,
                         int32_t* ws, cudaStream_t stream, unsigned long long* bad = nullptr);

// Programmatic dependent launch for the dense chain (FM/LCB and GEMM kernels); LATTICE_PDL=0
// launches them with plain stream ordering (A/B runs). The kernels call griddepcontrol.wait
// either way, which is a no-op without the launch attribute.
inline bool pdl_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("LATTICE_PDL");
        v = e ? (std::atoi(e) != 0) : 1;
    }
    return v == 1;
}

inline int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// ---- XXH64 -------------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t rotl64(uint64_t x, int r) {
    return (x << r) | (x >> (64 - r));
}
constexpr uint64_t kP1 = 0x9E3779B185EBCA87ull, kP2 = 0xC2B2AE3D27D4EB4Full,
                   kP3 = 0x165667B19E3779F9ull, kP4 = 0x85EBCA77C2B2AE63ull,
                   kP5 = 0x27D4EB2F165667C5ull;

__host__ __device__ __forceinline__ uint64_t xxh_round(uint64_t acc, uint64_t lane) {
    return rotl64(acc + lane * kP2, 31) * kP1;
}
__host__ __device__ __forceinline__ uint64_t xxh_avalanche(uint64_t h) {
    h ^= h >> 33;
    h *= kP2;
    h ^= h >> 29;
    h *= kP3;
    h ^= h >> 32;
    return h;
}

// XXH64 over a byte source `src` (src.u64(pos), src.u32(pos), src.u8(pos) little-endian reads)
// of length len. Same control flow as core.hpp:84-139.
template <typename Src>
__host__ __device__ __forceinline__ uint64_t xxh64_src(const Src& src, uint64_t len, uint64_t seed) {
    uint64_t p = 0, h;
    if (len >= 32) {
        uint64_t v1 = seed + kP1 + kP2, v2 = seed + kP2, v3 = seed, v4 = seed - kP1;
        do {
            v1 = xxh_round(v1, src.u64(p));
            v2 = xxh_round(v2, src.u64(p + 8));
            v3 = xxh_round(v3, src.u64(p + 16));
            v4 = xxh_round(v4, src.u64(p + 24));
            p += 32;
        } while (p + 32 <= len);
        h = rotl64(v1, 1) + rotl64(v2, 7) + rotl64(v3, 12) + rotl64(v4, 18);
        h = (h ^ xxh_round(0, v1)) * kP1 + kP4;
        h = (h ^ xxh_round(0, v2)) * kP1 + kP4;
        h = (h ^ xxh_round(0, v3)) * kP1 + kP4;
        h = (h ^ xxh_round(0, v4)) * kP1 + kP4;
    } else {
        h = seed + kP5;
    }
    h += len;
    for (; p + 8 <= len; p += 8) {
        h ^= xxh_round(0, src.u64(p));
        h = rotl64(h, 27) * kP1 + kP4;
    }
    if (p + 4 <= len) {
        h ^= (uint64_t)src.u32(p) * kP1;
        h = rotl64(h, 23) * kP2 + kP3;
        p += 4;
    }
    for (; p < len; ++p) {
        h ^= (uint64_t)src.u8(p) * kP5;
        h = rotl64(h, 11) * kP1;
    }
    return xxh_avalanche(h);
}

// The 16-byte generator input LE64(tag) || LE64(idx), specialised:
// len = 16 < 32, two 8-byte lanes, no tail.
__host__ __device__ __forceinline__ uint64_t gen_u64(uint64_t seed, uint64_t tag, uint64_t idx) {
    uint64_t h = seed + kP5 + 16ull;
    h ^= xxh_round(0, tag);
    h = rotl64(h, 27) * kP1 + kP4;
    h ^= xxh_round(0, idx);
    h = rotl64(h, 27) * kP1 + kP4;
    return xxh_avalanche(h);
}

constexpr uint64_t kTagTable = 0x4c54424cull, kTagLen = 0x4c4c454eull, kTagId = 0x4c494420ull,
                   kTagDom = 0x4c444f4dull;

__host__ __device__ __forceinline__ uint64_t weight_tag(int block, int kind, int index) {
    return 0x57000000ull | ((uint64_t)block << 16) | ((uint64_t)kind << 8) | (uint64_t)index;
}
__host__ __device__ __forceinline__ int weight_shift(int64_t fan_in) {
    int lg = 0;
    while ((1ll << (lg + 1)) <= fan_in) ++lg;
    return 7 + lg / 2;
}

// ---- 32-byte global accesses (sm_100: LDG/STG .ENL2.256) ----------------------------------
// Epilogues where a thread owns an output row put consecutive lanes 32 rows apart, so each
// 16-byte access fills half an L2 sector; 32 bytes per lane move whole sectors with half the
// instructions. Callers check 32-byte alignment.
__device__ __forceinline__ bool aligned32(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 31u) == 0; }
__device__ __forceinline__ void st_global_256(void* p, uint4 a, uint4 b) {
    asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(a.x), "r"(a.y), "r"(a.z),
                 "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
                 : "memory");
}
__device__ __forceinline__ void ld_global_256(const void* p, uint4& a, uint4& b) {
    asm volatile("ld.global.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
                 : "l"(p));
}

// ---- numeric helpers ----------------------------------------------------------------------
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// numerics.hpp:29-33 in fp32. exp(-|z|) form keeps it stable for both signs.
__device__ __forceinline__ float stable_sigmoid(float z) {
    const float e = __expf(-fabsf(z));        // in (0, 1]: no overflow for any z
    const float s = __fdividef(1.0f, 1.0f + e);  // MUFU reciprocal; ~2 ulp, far below bf16
    return z >= 0.0f ? s : 1.0f - s;
}
__device__ __forceinline__ float act_swish(float r, bool hard) {
    if (hard) return r * fminf(fmaxf((r + 3.0f) * (1.0f / 6.0f), 0.0f), 1.0f);
    return r * stable_sigmoid(r);
}

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
    __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ float bf16_lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t v) { return __uint_as_float(v & 0xffff0000u); }

}  // namespace lat
