// l2_probe.cu -- measured L2 read bandwidth of a B200, the denominator of the embedding stage's
// L2 fraction in bench.py (profiles/r02/l2_probe.json). Every SM streams a buffer that fits in L2
// (16-byte ld.global.cg loads: cached in L2 only, so repeated passes cannot hit L1); a 4 GiB
// buffer gives the HBM read rate beside it.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/l2_probe scripts/l2_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void read_kernel(const uint4* __restrict__ p, size_t n, int passes, unsigned* sink) {
    unsigned acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int r = 0; r < passes; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) {
            uint4 v;
            asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + i));
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    if (acc == 0x12345678u) *sink = acc;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t sizes_mb[] = {8, 16, 32, 48, 64, 96, 4096};
    unsigned* sink;
    cudaMalloc(&sink, 4);
    uint4* buf;
    cudaMalloc(&buf, (size_t)4096 << 20);
    cudaMemset(buf, 1, (size_t)4096 << 20);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (size_t mb : sizes_mb) {
        const size_t bytes = mb << 20, n = bytes / 16;
        const int passes = mb >= 1024 ? 3 : (int)(8192 / mb);
        for (int bpsm : {4, 8}) {
            const int grid = sms * bpsm;
            read_kernel<<<grid, 256>>>(buf, n, 1, sink);  // warm (L2 resident for the small sizes)
            cudaEventRecord(a);
            read_kernel<<<grid, 256>>>(buf, n, passes, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            printf("{\"buffer_mb\": %zu, \"blocks_per_sm\": %d, \"passes\": %d, \"ms\": %.4f, \"GB/s\": %.1f}\n", mb,
                   bpsm, passes, ms, (double)bytes * passes / (ms / 1e3) / 1e9);
        }
    }
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
