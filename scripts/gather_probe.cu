// gather_probe.cu -- feasibility probe for the bag kernel's memory side (not product code):
// gathers R random 256-byte rows (mid config: 256 tables x 100K rows x 128 bf16, rows visited
// table-major so one table is hot in L2, 655,360 rows per table) and sums them, two ways:
//   A  register gathers: each half-warp loads a row with 16-byte LDGs, U rows in flight per lane
//   B  bulk-copy ring: each warp streams its rows through S smem slots of 16 rows; the 16 copies
//      of a slot are cp.async.bulk (one per lane, 256 B each) completing on the slot's mbarrier,
//      and the warp sums rows out of shared memory while later slots are in flight
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_probe scripts/gather_probe.cu
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e = (x);                                                               \
        if (e != cudaSuccess) {                                                            \
            std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            return 1;                                                                      \
        }                                                                                  \
    } while (0)

constexpr int kF = 256, kRows = 100000, kD = 128, kRowB = kD * 2;
constexpr int64_t kPerTable = 1 << 19;  // rows gathered per table before the next (table-major)

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return x;
}
// cheap uniform id (multiplicative hash scaled into [0, kRows)) so address math is ~4 instructions
__device__ __forceinline__ const uint8_t* row_ptr(const uint8_t* tab, int64_t r) {
    const int64_t f = r >> 19;
    const uint32_t h = (uint32_t)r * 2654435761u;
    const uint32_t id = __umulhi(h, (uint32_t)kRows);
    return tab + ((int64_t)f * kRows + id) * kRowB;
}
__device__ __forceinline__ void addbf(float* a, uint32_t w) {
    a[0] += __uint_as_float(w << 16);
    a[1] += __uint_as_float(w & 0xffff0000u);
}

// A: 16 lanes per row, 2 rows per warp step, U steps in flight
template <int U>
__global__ void __launch_bounds__(256) gather_regs(const uint8_t* tab, int64_t R, float* out) {
    const int lane = threadIdx.x & 31, sub = lane >> 4, cl = lane & 15;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (gridDim.x * (int64_t)blockDim.x) >> 5;
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int64_t r0 = warp * 2 * U; r0 < R; r0 += nw * 2 * U) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t r = r0 + 2 * u + sub;
            v[u] = r < R ? __ldg(reinterpret_cast<const uint4*>(row_ptr(tab, r)) + cl) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            addbf(acc, v[u].x);
            addbf(acc + 2, v[u].y);
            addbf(acc + 4, v[u].z);
            addbf(acc + 6, v[u].w);
        }
    }
    float s = 0;
    for (int i = 0; i < 8; ++i) s += acc[i];
    if (s == 12345.f) out[0] = s;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* b, uint32_t ph) {
    uint32_t ok;
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(ph)
        : "memory");
    return ok;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// B: per warp S slots x 16 rows (4 KB each)
template <int S, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) gather_bulk(const uint8_t* tab, int64_t R, float* out) {
    extern __shared__ __align__(128) uint8_t sm[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint8_t* ring = sm + (size_t)w * S * 16 * kRowB;
    __shared__ uint64_t bars[WARPS][S];
    if (lane < S) mbar_init(&bars[w][lane], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const int64_t warp = blockIdx.x * (int64_t)WARPS + w;
    const int64_t nw = (int64_t)gridDim.x * WARPS;
    // this warp's rows: blocks of 16 rows, block k = warp + j * nw
    const int64_t nblocks = (R + 15) / 16;
    auto issue = [&](int64_t blk, int slot) {
        const int64_t r = blk * 16 + lane;
        if (lane == 0) {
            const int64_t n = R - blk * 16 < 16 ? R - blk * 16 : 16;
            mbar_expect_tx(&bars[w][slot], (uint32_t)(n * kRowB));
        }
        __syncwarp();
        if (lane < 16 && r < R) bulk_g2s(ring + (slot * 16 + lane) * kRowB, row_ptr(tab, r), kRowB, &bars[w][slot]);
    };
    int64_t j_issue = 0, j = 0;
    for (int s = 0; s < S; ++s, ++j_issue) {
        const int64_t blk = warp + j_issue * nw;
        if (blk < nblocks) issue(blk, s);
    }
    float acc[4] = {0, 0, 0, 0};
    uint32_t phase[S];
    for (int s = 0; s < S; ++s) phase[s] = 0;
    for (;; ++j) {
        const int64_t blk = warp + j * nw;
        if (blk >= nblocks) break;
        const int slot = (int)(j % S);
        while (!mbar_try(&bars[w][slot], phase[slot])) {
        }
        phase[slot] ^= 1;
        const int n = R - blk * 16 < 16 ? (int)(R - blk * 16) : 16;
        const uint8_t* base = ring + slot * 16 * kRowB + lane * 8;
        for (int i = 0; i < n; ++i) {
            const uint2 q = *reinterpret_cast<const uint2*>(base + i * kRowB);
            addbf(acc, q.x);
            addbf(acc + 2, q.y);
        }
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const int64_t nblk = warp + j_issue * nw;
        if (nblk < nblocks) issue(nblk, slot);
        ++j_issue;
    }
    float s = acc[0] + acc[1] + acc[2] + acc[3];
    if (s == 12345.f) out[0] = s;
}

template <typename K>
float time_kernel(K k, int grid, int block, size_t smem, const uint8_t* tab, int64_t R, float* out) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k<<<grid, block, smem>>>(tab, R, out);
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) k<<<grid, block, smem>>>(tab, R, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) std::printf("error %s\n", cudaGetErrorString(e));
    return ms / 5;
}

int main() {
    const size_t bytes = (size_t)kF * kRows * kRowB;
    uint8_t* tab;
    float* out;
    CK(cudaMalloc(&tab, bytes));
    CK(cudaMemset(tab, 1, bytes));
    CK(cudaMalloc(&out, 16));
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int64_t R = (int64_t)kF * kPerTable;  // 134M rows (the mid step gathers 168M)
    const double gb = R * (double)kRowB / 1e9;
    {
        float ms = time_kernel(gather_regs<4>, sms * 5, 256, 0, tab, R, out);
        std::printf("A regs U=4 40 warps/SM: %.3f ms  %.0f GB/s\n", ms, gb / ms * 1e3);
        ms = time_kernel(gather_regs<8>, sms * 4, 256, 0, tab, R, out);
        std::printf("A regs U=8 32 warps/SM: %.3f ms  %.0f GB/s\n", ms, gb / ms * 1e3);
    }
#define RUN_B(S, W, BPS)                                                                              \
    {                                                                                                 \
        const size_t smem = (size_t)(S) * (W) * 16 * kRowB;                                           \
        CK(cudaFuncSetAttribute(gather_bulk<S, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
        const float ms = time_kernel(gather_bulk<S, W>, sms * (BPS), (W) * 32, smem, tab, R, out);    \
        std::printf("B bulk S=%d warps=%d blocks/SM=%d (%zu KB/SM in flight): %.3f ms  %.0f GB/s\n", S, W, BPS, \
                    smem * (BPS) / 1024, ms, gb / ms * 1e3);                                           \
    }
    RUN_B(4, 8, 1)
    RUN_B(6, 8, 1)
    RUN_B(3, 16, 1)
    RUN_B(2, 8, 2)
    RUN_B(4, 4, 3)
    RUN_B(2, 8, 3)
    return 0;
}
