// peer.cu -- peer memory over NVLink/NVSwitch for the table-wise sharded embedding stage
// (SURVEY.md 8e): CUDA IPC export/import of device buffers between the one-process-per-GPU
// ranks, and a stream-ordered cross-GPU barrier on flags that live in each rank's HBM.
//
// The sharded step (paper_2512_09200_b200/peer.py) is
//   bucket(pos) -> barrier -> lattice_peer_embedding_bag -> barrier -> dense
// The first barrier publishes every rank's offsets / ids / pos of this step and tells the
// owners that the rank's X0 is free (its previous step has finished reading it); the second
// one tells every rank that all owners have written its X0. No host synchronisation, no NCCL
// call, and both barriers are graph-capturable (the epoch counter lives on the device).
#include <cuda.h>

#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "common.cuh"

namespace lat {
namespace {

using GetRangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);

lattice_status alloc_range(const void* p, void** base, size_t* size) {
    static GetRangeFn fn = nullptr;
    if (!fn) {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        LAT_CUDA(cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q));
        if (!f || q != cudaDriverEntryPointSuccess)
            return set_error(LATTICE_CUDA, "ipc: cuMemGetAddressRange unavailable");
        fn = reinterpret_cast<GetRangeFn>(f);
    }
    CUdeviceptr b = 0;
    size_t n = 0;
    if (fn(&b, &n, reinterpret_cast<CUdeviceptr>(p)) != CUDA_SUCCESS)
        return set_error(LATTICE_USAGE, "ipc: pointer is not a device allocation");
    *base = reinterpret_cast<void*>(b);
    *size = n;
    return LATTICE_OK;
}

// Opened peer allocations, reference-counted per handle (a process may open the same peer
// allocation for several buffers that share it, e.g. two tensors from one torch segment).
struct Opened {
    void* base;
    int refs;
};
std::mutex g_mu;
std::map<std::string, Opened> g_open;    // handle bytes -> mapping
std::map<void*, std::string> g_by_ptr;   // returned pointer -> handle bytes

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// flags[r] -> rank r's array of world + 1 words: [j] = last epoch rank j arrived at, [world] =
// rank r's own barrier counter. One thread per peer signals it and waits for it.
__global__ void barrier_kernel(uint32_t* const* __restrict__ flags, int rank, int world,
                               uint64_t timeout_ns, int32_t* __restrict__ status) {
    __shared__ uint32_t epoch;
    uint32_t* mine = flags[rank];
    if (threadIdx.x == 0) {
        epoch = mine[world] + 1;
        mine[world] = epoch;
    }
    __syncthreads();
    const int j = threadIdx.x;
    if (j >= world) return;
    __threadfence_system();                    // everything this rank wrote before the barrier
    st_release_sys(flags[j] + rank, epoch);    // "rank arrived at epoch" -> rank j
    const uint64_t t0 = globaltimer();
    while ((int32_t)(ld_acquire_sys(mine + j) - epoch) < 0) {
        if (globaltimer() - t0 > timeout_ns) {  // a peer never arrived: report, do not hang
            atomicExch(status, 1);
            break;
        }
        __nanosleep(64);
    }
    __threadfence_system();
}

}  // namespace
}  // namespace lat

extern "C" {

lattice_status lattice_ipc_handle(const void* dptr, uint8_t* handle, int64_t* offset) {
    using namespace lat;
    LAT_REQUIRE(dptr && handle && offset, "ipc_handle: null argument");
    void* base = nullptr;
    size_t size = 0;
    lattice_status s = alloc_range(dptr, &base, &size);
    if (s != LATTICE_OK) return s;
    cudaIpcMemHandle_t h;
    LAT_CUDA(cudaIpcGetMemHandle(&h, base));
    static_assert(sizeof(h) == LATTICE_IPC_HANDLE_BYTES, "IPC handle size");
    std::memcpy(handle, &h, sizeof(h));
    *offset = static_cast<const char*>(dptr) - static_cast<const char*>(base);
    return LATTICE_OK;
}

lattice_status lattice_ipc_open(const uint8_t* handle, int64_t offset, void** dptr) {
    using namespace lat;
    LAT_REQUIRE(handle && dptr && offset >= 0, "ipc_open: bad argument");
    const std::string key(reinterpret_cast<const char*>(handle), LATTICE_IPC_HANDLE_BYTES);
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_open.find(key);
    if (it == g_open.end()) {
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, sizeof(h));
        void* base = nullptr;
        LAT_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
        it = g_open.emplace(key, Opened{base, 0}).first;
    }
    it->second.refs++;
    void* p = static_cast<char*>(it->second.base) + offset;
    g_by_ptr[p] = key;  // the same pointer opened twice shares one entry; refs count both
    *dptr = p;
    return LATTICE_OK;
}

lattice_status lattice_ipc_close(void* dptr) {
    using namespace lat;
    std::lock_guard<std::mutex> lk(g_mu);
    auto pit = g_by_ptr.find(dptr);
    LAT_REQUIRE(pit != g_by_ptr.end(), "ipc_close: pointer was not opened by lattice_ipc_open");
    const std::string key = pit->second;
    auto it = g_open.find(key);
    if (it != g_open.end() && --it->second.refs == 0) {
        void* base = it->second.base;
        g_open.erase(it);
        for (auto q = g_by_ptr.begin(); q != g_by_ptr.end();)
            q = q->second == key ? g_by_ptr.erase(q) : std::next(q);
        LAT_CUDA(cudaIpcCloseMemHandle(base));
    }
    return LATTICE_OK;
}

lattice_status lattice_peer_barrier(uint32_t* const* flags, int32_t rank, int32_t world, double timeout_s,
                                    int32_t* status, lattice_stream stream) {
    using namespace lat;
    LAT_REQUIRE(flags && status, "peer_barrier: null argument");
    LAT_REQUIRE(world >= 1 && world <= 1024 && rank >= 0 && rank < world, "peer_barrier: bad rank/world");
    LAT_REQUIRE(timeout_s > 0.0, "peer_barrier: timeout must be > 0");
    const int threads = (world + 31) / 32 * 32;
    barrier_kernel<<<1, threads, 0, stream>>>(flags, rank, world, (uint64_t)(timeout_s * 1e9), status);
    LAT_CUDA(cudaGetLastError());
    return LATTICE_OK;
}

}  // extern "C"

// ---- data-parallel gradient reduction fused with the optimizer, over peer memory ---------------
namespace lat {
namespace {
constexpr int kMaxSegs = 16;
struct SegK {
    int64_t off, cnt;
    int32_t mode, bf16;
    void* const* dst;
};
struct ReduceParams {
    const float* const* grads;
    float* master;
    SegK seg[kMaxSegs];
    int32_t nseg, world, rank;
    int64_t lo, hi;
    float lr;
};

// Owner of elements [lo, hi): mean of every rank's gradient in rank order (read over NVLink,
// uncached), SGD on this rank's fp32 master shard (ZeRO-1: each master element lives on its
// owner only), and the new weight written into EVERY rank's copy (NVLink stores) --
// reduce-scatter + optimizer + all-gather in one pass, deterministic, so all replicas hold
// identical weights.
__device__ __forceinline__ void reduce_sgd_one(const ReduceParams& p, const SegK& sg, int64_t i) {
    float g = 0.0f;
    for (int r = 0; r < p.world; ++r) g += __ldcv(p.grads[r] + i);
    g = g / (float)p.world;
    const int64_t j = i - sg.off;
    if (sg.mode == 1) {  // mean only (e.g. the loss)
        for (int r = 0; r < p.world; ++r) static_cast<float*>(sg.dst[r])[j] = g;
        return;
    }
    const float w = p.master[i] - p.lr * g;
    p.master[i] = w;
    for (int r = 0; r < p.world; ++r) {
        if (sg.bf16)
            static_cast<__nv_bfloat16*>(sg.dst[r])[j] = __float2bfloat16_rn(w);
        else
            static_cast<float*>(sg.dst[r])[j] = w;
    }
}

// groups of 4 elements: 16-byte gradient loads from every rank and 8 / 16-byte weight stores
// when the group sits inside one segment at a 4-aligned position, element by element otherwise
__global__ void reduce_sgd_kernel(const ReduceParams p) {
    int s = 0;
    for (int64_t i0 = p.lo + 4 * (blockIdx.x * (int64_t)blockDim.x + threadIdx.x); i0 < p.hi;
         i0 += 4 * (int64_t)gridDim.x * blockDim.x) {
        while (s + 1 < p.nseg && i0 >= p.seg[s + 1].off) ++s;
        const SegK& sg = p.seg[s];
        const int64_t j0 = i0 - sg.off;
        if (j0 >= 0 && ((j0 | i0) & 3) == 0 && i0 + 4 <= sg.off + sg.cnt && i0 + 4 <= p.hi && sg.mode == 0) {
            float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int r = 0; r < p.world; ++r) {
                const float4 v = __ldcv(reinterpret_cast<const float4*>(p.grads[r] + i0));
                g.x += v.x, g.y += v.y, g.z += v.z, g.w += v.w;
            }
            const float W = (float)p.world;
            float4 m = *reinterpret_cast<const float4*>(p.master + i0);
            m.x = m.x - p.lr * (g.x / W), m.y = m.y - p.lr * (g.y / W);
            m.z = m.z - p.lr * (g.z / W), m.w = m.w - p.lr * (g.w / W);
            *reinterpret_cast<float4*>(p.master + i0) = m;
            if (sg.bf16) {
                const uint2 o = make_uint2(pack_bf16x2(m.x, m.y), pack_bf16x2(m.z, m.w));
                for (int r = 0; r < p.world; ++r)
                    *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(sg.dst[r]) + j0) = o;
            } else {
                for (int r = 0; r < p.world; ++r) *reinterpret_cast<float4*>(static_cast<float*>(sg.dst[r]) + j0) = m;
            }
            continue;
        }
        for (int64_t i = i0; i < i0 + 4 && i < p.hi; ++i) {  // segment edges, gaps, the loss
            int t = 0;
            while (t + 1 < p.nseg && i >= p.seg[t + 1].off) ++t;
            if (i >= p.seg[t].off && i < p.seg[t].off + p.seg[t].cnt) reduce_sgd_one(p, p.seg[t], i);
        }
    }
}
}  // namespace
}  // namespace lat

extern "C" lattice_status lattice_peer_reduce_sgd(const float* const* grads, float* master,
                                                   const lattice_peer_seg* segs, int32_t nseg, int64_t n, int32_t rank,
                                                   int32_t world, float lr, lattice_stream stream) {
    using namespace lat;
    LAT_REQUIRE(grads && master && segs, "peer_reduce_sgd: null argument");
    LAT_REQUIRE(world >= 1 && world <= 1024 && rank >= 0 && rank < world, "peer_reduce_sgd: bad rank/world");
    LAT_REQUIRE(nseg >= 1 && nseg <= kMaxSegs, "peer_reduce_sgd: need 1..16 segments");
    LAT_REQUIRE(n >= 0, "peer_reduce_sgd: bad size");
    ReduceParams p = {};
    p.grads = grads;
    p.master = master;
    p.nseg = nseg;
    p.world = world;
    p.rank = rank;
    p.lr = lr;
    int64_t prev_end = 0;
    for (int i = 0; i < nseg; ++i) {
        const lattice_peer_seg& q = segs[i];
        LAT_REQUIRE(q.offset >= prev_end && q.count >= 0 && q.offset + q.count <= n,
                    "peer_reduce_sgd: segments must be sorted, disjoint and inside [0, n)");
        LAT_REQUIRE(q.mode == 0 || q.mode == 1, "peer_reduce_sgd: mode must be 0 (sgd) or 1 (mean)");
        LAT_REQUIRE(q.dst != nullptr, "peer_reduce_sgd: null dst");
        LAT_REQUIRE(q.dst_dtype == LATTICE_F32 || (q.dst_dtype == LATTICE_BF16 && q.mode == 0),
                    "peer_reduce_sgd: dst dtype must be f32 (or bf16 for sgd segments)");
        p.seg[i] = {q.offset, q.count, q.mode, q.dst_dtype == LATTICE_BF16 ? 1 : 0, q.dst};
        prev_end = q.offset + q.count;
    }
    const int64_t shard = ((n + world - 1) / world + 3) / 4 * 4;  // 4-aligned shards
    p.lo = (int64_t)rank * shard < n ? (int64_t)rank * shard : n;
    p.hi = p.lo + shard < n ? p.lo + shard : n;
    if (p.hi <= p.lo) return LATTICE_OK;
    const int64_t blocks = (p.hi - p.lo + 1023) / 1024;
    const unsigned grid = (unsigned)(blocks < (int64_t)num_sms() * 8 ? blocks : num_sms() * 8);
    reduce_sgd_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(p);
    LAT_CUDA(cudaGetLastError());
    return LATTICE_OK;
}
