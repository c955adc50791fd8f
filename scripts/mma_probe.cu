// mma_probe.cu -- measures the issue-to-completion cost of tcgen05.mma shapes used by the
// FM/LCB and GEMM kernels (cycles per instruction, one CTA per SM, all SMs busy).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2512_09200_b200/csrc \
//        -I include scripts/mma_probe.cu -o /tmp/mma_probe && /tmp/mma_probe
#include <cstdio>

#include "tc.cuh"

using namespace lat;

__global__ void probe(int N, int a_mn, int b_mn, int reps, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
    if (threadIdx.x == 0) {
        tc::mbar_init(&bar, 1);
        tc::fence_mbar_init();
    }
    if (warp == 0) tc::tmem_alloc(&slot, 512);
    tc::fence_async_shared();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (threadIdx.x == 0) {
        const uint32_t id = tc::idesc_bf16(128, N, a_mn, b_mn);
        const uint32_t a = tc::smem_u32(smem), b = tc::smem_u32(smem + 32768);
        // K-major: SBO 1024 between 8-row groups; MN-major: LBO = 16 KB between 64-wide chunks
        const uint64_t ad = tc::sdesc(a, a_mn ? 16384 : 16, 1024, 2);
        const uint64_t bd = tc::sdesc(b, b_mn ? 16384 : 16, 1024, 2);
        long long t0 = clock64();
        for (int r = 0; r < reps; ++r) tc::mma_f16(slot, ad, bd, id, r != 0);
        tc::mma_commit(&bar);
        tc::mbar_wait(&bar, 0);
        long long t1 = clock64();
        if (blockIdx.x == 0) out[0] = t1 - t0;
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(slot, 512);
}

int main() {
    long long* d;
    cudaMalloc(&d, 8);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    struct C {
        int N, a_mn, b_mn;
        const char* what;
    } cs[] = {{32, 0, 0, "N=32  K-major A,B (F = X P)"},     {32, 1, 0, "N=32  MN-major A (P = X^T Y)"},
              {128, 0, 1, "N=128 MN-major B (L = W_L X)"}, {128, 0, 0, "N=128 K-major"},
              {256, 0, 0, "N=256 K-major (GEMM tile)"},     {64, 0, 0, "N=64  K-major"}};
    for (auto& c : cs) {
        for (int reps : {16, 256}) {
            probe<<<148, 128, 96 * 1024>>>(c.N, c.a_mn, c.b_mn, reps, d);
            long long h = 0;
            cudaError_t e = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
            if (e != cudaSuccess) {
                printf("error %s\n", cudaGetErrorString(e));
                return 1;
            }
            printf("%-32s reps %4d: %8.1f cycles/MMA (ideal 128*N/256 = %d)\n", c.what, reps,
                   (double)h / reps, 128 * c.N / 256);
        }
    }
    return 0;
}
