// network.cu -- lattice_net: the consolidated MDMO forward step on one GPU.
//
//   K6 domain_bucket      stable counting sort by domain -> pos/order/seg + tower tile table
//   K1 embedding_bag      pooled sums, rms_norm over d, written straight into domain-sorted
//                         rows of X0 (so towers read contiguous segments, no permute copy)
//   per block (l times):  K2 fm_lcb (P, F, Fin, LCB half of X')  ->  K3 MLP GEMMs with fused
//                         swish_rn  ->  K3 last GEMM with fused residual + rms_norm_d (FMB half)
//   K4 towers             one grouped GEMM over the G domain segments, swish_rn + heads fused,
//                         logits written back in the caller's sample order
// Storage dtype (cfg.dtype): bf16 (kind::f16 MMAs) or fp32 (kind::tf32 MMAs) for weights and
// activations; tower heads and logits are fp32. Weights are generated on device from
// weight_seed with the counter-based scheme shared with oracle/lattice_oracle.c (the values
// are exact in both dtypes).
#include <cuda_bf16.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdlib>
#include <functional>
#include <string>
#include <vector>

#include "backward.h"
#include "common.cuh"
#include "fm_lcb.h"
#include "gemm_host.h"

namespace lat {
namespace {

// tower tile table: `rows`-row tiles (128: single-CTA grouped GEMM; 256: CTA-pair) per domain segment
__global__ void tiles_kernel(const int32_t* __restrict__ seg, int G, int rows, int4* __restrict__ tiles,
                             int* __restrict__ n_tiles) {
    __shared__ int pre[65];
    if (threadIdx.x == 0) {
        int run = 0;
        for (int g = 0; g < G; ++g) {
            pre[g] = run;
            run += (seg[g + 1] - seg[g] + rows - 1) / rows;
        }
        pre[G] = run;
        *n_tiles = run;
    }
    __syncthreads();
    const int total = pre[G];
    for (int t = threadIdx.x; t < total; t += blockDim.x) {
        int g = 0;
        while (pre[g + 1] <= t) ++g;
        const int r0 = seg[g] + (t - pre[g]) * rows;
        tiles[t] = make_int4(g, r0, seg[g + 1], 0);
    }
}

// towers on the CTA-pair GEMM: h = swish_rn(W1_g x) came out of the GEMM (fp32, domain-sorted
// rows); one warp per row forms the heads W2_g . h and writes them in the caller's sample order
__global__ void tower_heads_kernel(int64_t B, int th, int heads, int G, const float* __restrict__ h,
                                   const int32_t* __restrict__ seg, const int32_t* __restrict__ order,
                                   const float* __restrict__ W2, float* __restrict__ logits) {
    __shared__ int32_t sseg[33];
    for (int i = threadIdx.x; i <= G; i += blockDim.x) sseg[i] = seg[i];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    for (int64_t m = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; m < B;
         m += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        int g = 0;
        while (g + 1 < G && sseg[g + 1] <= m) ++g;
        const float* hr = h + m * th;
        const float* w2 = W2 + (int64_t)g * heads * th;
        float acc[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) acc[k] = 0.0f;
        for (int j = lane * 4; j < th; j += 128) {
            const float4 hv = *reinterpret_cast<const float4*>(hr + j);
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                if (k < heads) {
                    const float4 w = __ldg(reinterpret_cast<const float4*>(w2 + (int64_t)k * th + j));
                    acc[k] += hv.x * w.x + hv.y * w.y + hv.z * w.z + hv.w * w.w;
                }
            }
        }
#pragma unroll
        for (int k = 0; k < 16; ++k)
            if (k < heads) acc[k] = warp_sum(acc[k]);
        if (lane < heads) {
            float v = 0.0f;
#pragma unroll
            for (int k = 0; k < 16; ++k)
                if (k == lane) v = acc[k];
            logits[(int64_t)order[m] * heads + lane] = v;
        }
    }
}

__device__ __forceinline__ void put(float* p, float v) { *p = v; }
__device__ __forceinline__ void put(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }

// pooled sums (caller order, [B][n][d] f32 or bf16) -> rms_norm_d -> row pos[b] of X0
template <typename TI, typename TO>
// in: [B][n][d] rows of features [foff, foff + n) of an n_out-wide X0 row
__global__ void pooled_norm_kernel(int64_t B, int n, int d, const TI* __restrict__ in,
                                   const int32_t* __restrict__ pos, TO* __restrict__ out, int n_out, int foff) {
    const int lane = threadIdx.x & 31;
    for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < B * n;
         w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t b = w / n;
        const int f = (int)(w - b * n);
        const TI* src = in + w * d;
        float v[4];
        float ss = 0.0f;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int c = lane + 32 * i;
            v[i] = c < d ? (float)src[c] : 0.0f;
            ss += v[i] * v[i];
        }
        ss = warp_sum(ss);
        const float denom = sqrtf(ss / (float)d + 1e-6f);
        TO* dst = out + ((int64_t)pos[b] * n_out + foff + f) * d;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int c = lane + 32 * i;
            if (c < d) put(dst + c, v[i] / denom);
        }
    }
}

// table-wise shards [S][B][n/S][d] (already normalised by their owners) -> X0 rows pos[b];
// one warp per (b, f), 16-byte vectors; dtype-agnostic (vec = d * es / 16)
__global__ void shard_gather_kernel(int64_t B, int n, int d, int es, int S, const uint8_t* __restrict__ in,
                                    const int32_t* __restrict__ pos, uint8_t* __restrict__ out, int n_out) {
    const int lane = threadIdx.x & 31;
    const int nl = n / S;
    const int row = d * es;      // bytes per embedding
    const int vec = row / 16;
    for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < B * n;
         w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t b = w / n;
        const int f = (int)(w - b * n);
        const int o = f / nl, fl = f - o * nl;
        const uint4* src = reinterpret_cast<const uint4*>(in + (((int64_t)o * B + b) * nl + fl) * row);
        uint4* dst = reinterpret_cast<uint4*>(out + ((int64_t)pos[b] * n_out + f) * row);
        for (int i = lane; i < vec; i += 32) dst[i] = src[i];
    }
}

int round_up(int x, int m) { return (x + m - 1) / m * m; }

// fp32 [rows][cols] -> dst rows of stride ld in the net dtype (RNE), for lattice_net_set_weight
template <typename TO>
__global__ void load_rows_kernel(int64_t rows, int64_t cols, const float* __restrict__ src, TO* __restrict__ dst,
                                 int64_t ld) {
    const int64_t n = rows * cols;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / cols;
        put(dst + r * ld + (i - r * cols), src[i]);
    }
}

}  // namespace
}  // namespace lat

struct lattice_net {
    lattice_net_config cfg;
    int n_pad, k_pad;
    int device;
    bool f32;
    size_t es;  // bytes per stored element
    // weights (storage dtype unless noted)
    std::vector<void*> YT, WL;   // padded [k_pad][n_pad], [128][n_pad]
    std::vector<void*> mlp;      // [blocks * n_mlp] -> [out][in]
    void* T1 = nullptr;          // [G * th][n*d]
    float* T2 = nullptr;         // [G][heads][th] fp32
    void* D1 = nullptr;          // dense processor [dense_hidden][dense_in]
    void* D2 = nullptr;          // [dense_features*d][dense_hidden]
    void *Din = nullptr, *Hd = nullptr, *Od = nullptr;  // dense input copy, hidden, output rows
    float* rowpart = nullptr;  // swish GEMMs (CTA-pair kernel): row-statistics exchange
    int* rowcnt = nullptr;     // [swish GEMMs][rowcnt_stride] arrival counters, zeroed once per forward
    size_t rowcnt_stride = 0, rowcnt_total = 0;
    // workspace
    int32_t *pos = nullptr, *order = nullptr, *seg = nullptr, *bucket_ws = nullptr;
    unsigned long long* bad_domain = nullptr;  // checked forwards: first sample with a bad domain
    int4* tiles = nullptr;
    int* n_tiles = nullptr;
    int tile_rows = 128;         // tower tile table granularity (256: CTA-pair tower)
    bool tower_pair = false;     // towers = pair swish GEMM into Htower + tower_heads_kernel
    float* Htower = nullptr;     // [max_batch][tower_hidden] fp32 (tower_pair)
    void* X[2] = {nullptr, nullptr};
    void* Fbuf = nullptr;
    void* H[2] = {nullptr, nullptr};
    // plans (tensor maps built once for max_batch)
    std::vector<lat::fm::Plan> fm_plans;              // [blocks]
    std::vector<lat::gemm::GemmPlan> mlp_plans;       // [blocks * n_mlp]
    lat::gemm::GemmPlan tower_plan;
    lat::gemm::GemmPlan dense_plans[2];
    // timing
    bool timing = false;
    std::vector<cudaEvent_t> ev;
    std::vector<void*> allocs;
    // backward scratch, kept between calls and grown on demand: a stream-ordered allocation per
    // call returned GBs to the driver at every synchronisation and re-mapped them next time
    void* bwd_ws = nullptr;
    size_t bwd_ws_bytes = 0;
};

namespace {

lattice_status dalloc_bytes(lattice_net* net, void** p, size_t bytes) {
    void* q = nullptr;
    LAT_CUDA(cudaMalloc(&q, bytes > 0 ? bytes : 16));
    net->allocs.push_back(q);
    *p = q;
    return LATTICE_OK;
}

template <typename T>
lattice_status dalloc(lattice_net* net, T** p, size_t count) {
    void* q = nullptr;
    lattice_status s = dalloc_bytes(net, &q, count * sizeof(T));
    *p = static_cast<T*>(q);
    return s;
}

lattice_status fill_padded(lattice_net* net, void* dst, int rows, int cols, int rows_pad, int cols_pad,
                           uint64_t tag) {
    const size_t es = net->es;
    LAT_CUDA(cudaMemset(dst, 0, es * (size_t)rows_pad * cols_pad));
    void* tmp = nullptr;
    LAT_CUDA(cudaMalloc(&tmp, es * (size_t)rows * cols));
    lattice_status s = lattice_fill_weights(tmp, net->f32 ? LATTICE_F32 : LATTICE_BF16, rows, cols,
                                            net->cfg.weight_seed, tag, nullptr);
    if (s == LATTICE_OK) {
        cudaError_t e = cudaMemcpy2D(dst, es * cols_pad, tmp, es * cols, es * cols, rows, cudaMemcpyDeviceToDevice);
        if (e != cudaSuccess) s = lat::check_cuda(e, "weight pad copy");
    }
    cudaFree(tmp);
    return s;
}

lattice_status validate(const lattice_net_config* c) {
    using lat::set_error;
    if (!c) return set_error(LATTICE_USAGE, "lattice_net_create: null config");
    if (c->dtype != LATTICE_BF16 && c->dtype != LATTICE_F32)
        return set_error(LATTICE_USAGE, "network: dtype must be bf16 or f32");
    if (c->n < 1 || c->n > 512) return set_error(LATTICE_USAGE, "network: n must be in [1, 512]");
    if (c->n > 256 && (c->dtype != LATTICE_BF16 || c->d != 128))
        return set_error(LATTICE_USAGE, "network: n > 256 needs bf16 and d = 128");
    if (c->d != 64 && c->d != 128) return set_error(LATTICE_USAGE, "network: d must be 64 or 128");
    if (c->dtype == LATTICE_F32 && c->d != 64) return set_error(LATTICE_USAGE, "network: fp32 needs d = 64");
    if (c->blocks < 1) return set_error(LATTICE_USAGE, "network: need at least one block");
    if (c->nF < 1 || c->nL < 0 || c->nF + c->nL != c->n || c->nL > (c->n > 256 ? 256 : 128))
        return set_error(LATTICE_USAGE, "network: need nF >= 1, nF + nL == n, nL <= 128 (<= 256 when n > 256)");
    if (c->k < 1 || c->k > 64) return set_error(LATTICE_USAGE, "network: k must be in [1, 64]");
    if (c->n_mlp < 1 || c->n_mlp > 5) return set_error(LATTICE_USAGE, "network: n_mlp must be in [1, 5]");
    if (c->mlp[0] != c->n * c->k) return set_error(LATTICE_USAGE, "network: mlp[0] must equal n*k");
    if (c->mlp[c->n_mlp] != c->nF * c->d) return set_error(LATTICE_USAGE, "network: mlp[n_mlp] must equal nF*d");
    for (int i = 0; i <= c->n_mlp; ++i)
        if (c->mlp[i] < 8 || c->mlp[i] % 8) return set_error(LATTICE_USAGE, "network: MLP widths must be multiples of 8");
    // swish_rn hidden layers: the CTA-pair GEMM (bf16, >= 256 rows) exchanges row statistics
    // through global memory and takes rows up to 16384 wide (PAPER.md:855's 8192-4096-8192 MLP);
    // the single-CTA kernel (fp32 / tiny batches) exchanges them over DSMEM, up to 2048
    const int max_hidden = c->dtype == LATTICE_BF16 && c->max_batch >= 256 ? 16384 : 2048;
    for (int i = 1; i < c->n_mlp; ++i)
        if (c->mlp[i] > max_hidden)
            return set_error(LATTICE_USAGE, max_hidden == 2048
                                                ? "network: hidden widths above 2048 need bf16 and max_batch >= 256"
                                                : "network: hidden widths above 16384 are not supported");
    if (c->domains < 1 || c->domains > 32) return set_error(LATTICE_USAGE, "network: domains must be in [1, 32]");
    if (c->heads < 1 || c->heads > 16) return set_error(LATTICE_USAGE, "network: heads must be in [1, 16]");
    if (c->tower_hidden < 8 || c->tower_hidden > 2048 || c->tower_hidden % 8)
        return set_error(LATTICE_USAGE, "network: tower_hidden must be a multiple of 8 in [8, 2048]");
    if (c->max_batch < 1 || c->max_batch > (1ll << 30)) return set_error(LATTICE_USAGE, "network: bad max_batch");
    if (c->dense_features < 0 || c->dense_features >= c->n)
        return set_error(LATTICE_USAGE, "network: dense_features must be in [0, n)");
    if (c->dense_features > 0) {
        if (c->dense_in < 8 || c->dense_in % 8)
            return set_error(LATTICE_USAGE, "network: dense_in must be a positive multiple of 8");
        if (c->dense_hidden < 8 || c->dense_hidden > 2048 || c->dense_hidden % 8)
            return set_error(LATTICE_USAGE, "network: dense_hidden must be a multiple of 8 in [8, 2048]");
    }
    return LATTICE_OK;
}

lattice_status build_plans(lattice_net* net) {
    using namespace lat;
    const lattice_net_config& c = net->cfg;
    const int64_t Bm = c.max_batch;
    const int nd = c.n * c.d;
    net->fm_plans.resize(c.blocks);
    net->mlp_plans.resize((size_t)c.blocks * c.n_mlp);
    for (int blk = 0; blk < c.blocks; ++blk) {
        void* Xc = net->X[blk & 1];
        void* Xn = net->X[(blk + 1) & 1];
        fm::Plan& fp = net->fm_plans[blk];
        fp.p.B = Bm;
        fp.p.n = c.n;
        fp.p.d = c.d;
        fp.p.k = c.k;
        fp.p.nF = c.nF;
        fp.p.nL = c.nL;
        fp.p.n_pad = net->n_pad;
        fp.p.k_pad = net->k_pad;
        fp.p.tmem_cols = 512;
        fp.p.f32 = net->f32 ? 1 : 0;
        fp.p.Fout = net->Fbuf;
        fp.p.Xout = Xn;
        fp.p.Xin = Xc;
        lattice_status s = fm::check(fp.p);
        if (s != LATTICE_OK) return s;
        s = fm::make_maps(&fp, Xc, net->WL[blk], net->YT[blk]);
        if (s != LATTICE_OK) return s;
        for (int li = 0; li < c.n_mlp; ++li) {
            const int in = c.mlp[li], out = c.mlp[li + 1];
            const bool last = li + 1 == c.n_mlp;
            const void* A = li == 0 ? net->Fbuf : net->H[(li - 1) & 1];
            gemm::Params p = {};
            p.M = (int)Bm;
            p.N = out;
            p.K = in;
            p.out_bf16 = net->f32 ? 0 : 1;
            p.N_full = out;
            p.cluster = 1;
            if (!last) {
                p.C = net->H[li & 1];
                p.ldc = out;
                p.epi = c.hard ? gemm::kSwishHard : gemm::kSwish;
                p.cluster = (out + 255) / 256;
                p.rowpart = net->rowpart;
                p.rowcnt = net->rowcnt + (size_t)(blk * (c.n_mlp - 1) + li) * net->rowcnt_stride;
                p.rowcnt_zeroed = 1;  // one memset per forward for every swish GEMM's counters
            } else {
                p.C = Xn;
                p.ldc = nd;
                p.epi = gemm::kResidNorm;
                p.resid = Xc;
                p.ldr = nd;
                p.group = c.d;
            }
            s = gemm::plan(&net->mlp_plans[(size_t)blk * c.n_mlp + li], A, in, Bm, net->mlp[(size_t)blk * c.n_mlp + li],
                           in, out, p, (int)((Bm + 127) / 128), net->f32);
            if (s != LATTICE_OK) return s;
        }
    }
    if (c.dense_features > 0) {  // dense processor: swish_rn hidden layer, linear out
        gemm::Params d1 = {};
        d1.M = (int)Bm;
        d1.N = c.dense_hidden;
        d1.K = c.dense_in;
        d1.out_bf16 = net->f32 ? 0 : 1;
        d1.N_full = c.dense_hidden;
        d1.C = net->Hd;
        d1.ldc = c.dense_hidden;
        d1.epi = c.hard ? gemm::kSwishHard : gemm::kSwish;
        d1.cluster = (c.dense_hidden + 255) / 256;
        d1.rowpart = net->rowpart;
        d1.rowcnt = net->rowcnt + (size_t)c.blocks * (c.n_mlp - 1) * net->rowcnt_stride;
        d1.rowcnt_zeroed = 1;
        lattice_status s = gemm::plan(&net->dense_plans[0], net->Din, c.dense_in, Bm, net->D1, c.dense_in,
                                      c.dense_hidden, d1, (int)((Bm + 127) / 128), net->f32);
        if (s != LATTICE_OK) return s;
        gemm::Params d2 = {};
        d2.M = (int)Bm;
        d2.N = c.dense_features * c.d;
        d2.K = c.dense_hidden;
        d2.out_bf16 = net->f32 ? 0 : 1;
        d2.N_full = d2.N;
        d2.C = net->Od;
        d2.ldc = d2.N;
        d2.epi = gemm::kStore;
        d2.cluster = 1;
        s = gemm::plan(&net->dense_plans[1], net->Hd, c.dense_hidden, Bm, net->D2, c.dense_hidden, d2.N, d2,
                       (int)((Bm + 127) / 128), net->f32);
        if (s != LATTICE_OK) return s;
    }
    if (net->tower_pair) {  // towers: CTA-pair swish GEMM over 256-row domain tiles, heads after
        gemm::Params p = {};
        p.M = (int)Bm;
        p.N = c.tower_hidden;
        p.K = nd;
        p.C = net->Htower;
        p.ldc = c.tower_hidden;
        p.out_bf16 = 0;
        p.epi = c.hard ? gemm::kSwishHard : gemm::kSwish;
        p.N_full = c.tower_hidden;
        p.cluster = (c.tower_hidden + 255) / 256;
        p.rowpart = net->rowpart;
        p.rowcnt = net->rowcnt + (size_t)(c.blocks * (c.n_mlp - 1) + 1) * net->rowcnt_stride;
        p.rowcnt_zeroed = 1;
        p.tiles = net->tiles;
        p.n_tiles = net->n_tiles;
        p.b_rows_per_group = c.tower_hidden;
        lattice_status s = gemm::plan(&net->tower_plan, net->X[c.blocks & 1], nd, Bm, net->T1, nd,
                                      (int64_t)c.domains * c.tower_hidden, p, (int)((Bm + 255) / 256) + c.domains,
                                      net->f32);
        if (s == LATTICE_OK && !net->tower_plan.two_cta)
            return set_error(LATTICE_CUDA, "network: CTA-pair tower plan unavailable");
        return s;
    }
    gemm::Params p = {};
    p.M = (int)Bm;
    p.N = c.tower_hidden;
    p.K = nd;
    p.out_bf16 = 0;
    p.epi = c.hard ? gemm::kTowerHard : gemm::kTower;
    p.cluster = (c.tower_hidden + 255) / 256;
    p.N_full = c.tower_hidden;
    p.tiles = net->tiles;
    p.n_tiles = net->n_tiles;
    p.b_rows_per_group = c.tower_hidden;
    p.W2 = net->T2;
    p.heads = c.heads;
    p.order = net->order;
    return gemm::plan(&net->tower_plan, net->X[c.blocks & 1], nd, Bm, net->T1, nd,
                      (int64_t)c.domains * c.tower_hidden, p, (int)((Bm + 127) / 128) + c.domains, net->f32);
}

}  // namespace

extern "C" {

lattice_status lattice_net_create(const lattice_net_config* cfg, lattice_net** out) {
    using namespace lat;
    LAT_REQUIRE(out != nullptr, "lattice_net_create: null out");
    *out = nullptr;
    lattice_status s = validate(cfg);
    if (s != LATTICE_OK) return s;
    lattice_net* net = new lattice_net();
    net->cfg = *cfg;
    cudaGetDevice(&net->device);
    const lattice_net_config& c = net->cfg;
    net->f32 = c.dtype == LATTICE_F32;
    net->es = net->f32 ? 4 : 2;
    const int wdt = net->f32 ? LATTICE_F32 : LATTICE_BF16;
    net->n_pad = c.n > 256 ? round_up(c.n, 256) : round_up(c.n, 16);  // large variant: 512
    net->k_pad = round_up(c.k, 16);
    const int nd = c.n * c.d;
    const int64_t Bm = c.max_batch;
    const size_t es = net->es;
    auto fail = [&](lattice_status st) {
        lattice_net_destroy(net);
        return st;
    };
#define NET_TRY(x)                                 \
    do {                                           \
        lattice_status _s = (x);                   \
        if (_s != LATTICE_OK) return fail(_s);     \
    } while (0)
    const uint64_t seed = c.weight_seed;
    for (int blk = 0; blk < c.blocks; ++blk) {
        void *yt = nullptr, *wl = nullptr;
        const int wlr = c.nL > 128 ? 256 : 128;  // padded W_L rows (fm::wl_rows)
        NET_TRY(dalloc_bytes(net, &yt, es * (size_t)net->k_pad * net->n_pad));
        NET_TRY(dalloc_bytes(net, &wl, es * (size_t)wlr * net->n_pad));
        NET_TRY(fill_padded(net, yt, c.k, c.n, net->k_pad, net->n_pad, weight_tag(blk, 1, 0)));
        NET_TRY(fill_padded(net, wl, c.nL > 0 ? c.nL : 1, c.n, wlr, net->n_pad, weight_tag(blk, 2, 0)));
        if (c.nL == 0) LAT_CUDA(cudaMemset(wl, 0, es * wlr * net->n_pad));
        net->YT.push_back(yt);
        net->WL.push_back(wl);
        for (int li = 0; li < c.n_mlp; ++li) {
            void* w = nullptr;
            NET_TRY(dalloc_bytes(net, &w, es * (size_t)c.mlp[li + 1] * c.mlp[li]));
            NET_TRY(lattice_fill_weights(w, wdt, c.mlp[li + 1], c.mlp[li], seed, weight_tag(blk, 3, li), nullptr));
            net->mlp.push_back(w);
        }
    }
    NET_TRY(dalloc_bytes(net, &net->T1, es * (size_t)c.domains * c.tower_hidden * nd));
    NET_TRY(dalloc(net, &net->T2, (size_t)c.domains * c.heads * c.tower_hidden));
    for (int g = 0; g < c.domains; ++g) {
        NET_TRY(lattice_fill_weights(static_cast<uint8_t*>(net->T1) + es * (size_t)g * c.tower_hidden * nd, wdt,
                                     c.tower_hidden, nd, seed, weight_tag(g, 4, 0), nullptr));
        NET_TRY(lattice_fill_weights(net->T2 + (size_t)g * c.heads * c.tower_hidden, LATTICE_F32, c.heads,
                                     c.tower_hidden, seed, weight_tag(g, 5, 0), nullptr));
    }
    if (c.dense_features > 0) {
        const int od = c.dense_features * c.d;
        NET_TRY(dalloc_bytes(net, &net->D1, es * (size_t)c.dense_hidden * c.dense_in));
        NET_TRY(dalloc_bytes(net, &net->D2, es * (size_t)od * c.dense_hidden));
        NET_TRY(lattice_fill_weights(net->D1, wdt, c.dense_hidden, c.dense_in, seed, weight_tag(0, 6, 0), nullptr));
        NET_TRY(lattice_fill_weights(net->D2, wdt, od, c.dense_hidden, seed, weight_tag(0, 7, 0), nullptr));
        NET_TRY(dalloc_bytes(net, &net->Din, es * (size_t)Bm * c.dense_in));
        NET_TRY(dalloc_bytes(net, &net->Hd, es * (size_t)Bm * c.dense_hidden));
        NET_TRY(dalloc_bytes(net, &net->Od, es * (size_t)Bm * od));
    }
    int max_hidden = 8;
    for (int i = 1; i < c.n_mlp; ++i) max_hidden = max_hidden > c.mlp[i] ? max_hidden : c.mlp[i];
    {  // towers on the CTA-pair GEMM (bf16, >= 256 rows); LATTICE_TOWER_PAIR=0 keeps the fused
       // single-CTA grouped tower (heads in its epilogue) for A/B runs
        const char* e = std::getenv("LATTICE_TOWER_PAIR");
        net->tower_pair = !net->f32 && Bm >= 256 && !(e && std::atoi(e) == 0);
        net->tile_rows = net->tower_pair ? 256 : 128;
        if (net->tower_pair) NET_TRY(dalloc(net, &net->Htower, (size_t)Bm * c.tower_hidden));
    }
    {  // row-statistics exchange of the swish GEMMs: [rows][N-tiles of the widest] + counters
        const size_t rows = (size_t)((Bm + 255) / 256) * 256;
        int tiles = (max_hidden + 255) / 256;
        if (c.dense_features > 0 && (c.dense_hidden + 255) / 256 > tiles) tiles = (c.dense_hidden + 255) / 256;
        NET_TRY(dalloc(net, &net->rowpart, rows * (size_t)(tiles > 8 ? tiles : 8)));
        net->rowcnt_stride = rows / 128 + 2 * (size_t)c.domains + 16;  // grouped tiles: + 2 per domain
        // slots: every MLP swish GEMM, the dense processor's, the pair tower's
        net->rowcnt_total = net->rowcnt_stride * ((size_t)c.blocks * (c.n_mlp - 1) + 2);
        NET_TRY(dalloc(net, &net->rowcnt, net->rowcnt_total));
    }
    NET_TRY(dalloc(net, &net->pos, (size_t)Bm));
    NET_TRY(dalloc(net, &net->order, (size_t)Bm));
    NET_TRY(dalloc(net, &net->seg, (size_t)c.domains + 1));
    NET_TRY(dalloc(net, &net->bucket_ws, (size_t)lat::bucket_workspace(Bm, c.domains)));
    NET_TRY(dalloc(net, &net->bad_domain, 1));
    NET_TRY(dalloc(net, &net->tiles, (size_t)((Bm + 127) / 128 + c.domains + 1)));
    NET_TRY(dalloc(net, &net->n_tiles, 1));
    NET_TRY(dalloc_bytes(net, &net->X[0], es * (size_t)Bm * nd));
    NET_TRY(dalloc_bytes(net, &net->X[1], es * (size_t)Bm * nd));
    NET_TRY(dalloc_bytes(net, &net->Fbuf, es * (size_t)Bm * c.n * c.k));
    NET_TRY(dalloc_bytes(net, &net->H[0], es * (size_t)Bm * max_hidden));
    NET_TRY(dalloc_bytes(net, &net->H[1], es * (size_t)Bm * max_hidden));
    NET_TRY(build_plans(net));
    LAT_CUDA(cudaDeviceSynchronize());
#undef NET_TRY
    *out = net;
    return LATTICE_OK;
}

void lattice_net_destroy(lattice_net* net) {
    if (!net) return;
    if (net->bwd_ws) cudaFree(net->bwd_ws);
    for (void* p : net->allocs) cudaFree(p);
    for (cudaEvent_t e : net->ev) cudaEventDestroy(e);
    delete net;
}

const void* lattice_net_weight(lattice_net* net, int32_t block, int32_t kind, int32_t index) {
    if (!net) return nullptr;
    const lattice_net_config& c = net->cfg;
    switch (kind) {
        case 1: return block >= 0 && block < c.blocks ? net->YT[block] : nullptr;
        case 2: return block >= 0 && block < c.blocks ? net->WL[block] : nullptr;
        case 3:
            return block >= 0 && block < c.blocks && index >= 0 && index < c.n_mlp
                       ? net->mlp[(size_t)block * c.n_mlp + index]
                       : nullptr;
        case 4: return net->T1;
        case 5: return net->T2;
        case 6: return net->D1;
        case 7: return net->D2;
        default: return nullptr;
    }
}

lattice_status lattice_net_set_weight(lattice_net* net, int32_t block, int32_t kind, int32_t index,
                                      const void* src, int32_t src_dtype, lattice_stream stream) {
    using namespace lat;
    LAT_REQUIRE(net != nullptr && src != nullptr, "lattice_net_set_weight: null argument");
    const lattice_net_config& c = net->cfg;
    void* dst = const_cast<void*>(lattice_net_weight(net, block, kind, index));
    LAT_REQUIRE(dst != nullptr, "lattice_net_set_weight: no such weight (block / kind / index)");
    // unpadded [rows][cols] and the row stride of the net's (possibly padded) buffer
    int64_t rows = 0, cols = 0, ld = 0;
    switch (kind) {
        case 1: rows = c.k, cols = c.n, ld = net->n_pad; break;
        case 2: rows = c.nL, cols = c.n, ld = net->n_pad; break;
        case 3: rows = c.mlp[index + 1], cols = c.mlp[index], ld = cols; break;
        case 4: rows = (int64_t)c.domains * c.tower_hidden, cols = (int64_t)c.n * c.d, ld = cols; break;
        case 5: rows = (int64_t)c.domains * c.heads, cols = c.tower_hidden, ld = cols; break;
        case 6: rows = c.dense_hidden, cols = c.dense_in, ld = cols; break;
        case 7: rows = (int64_t)c.dense_features * c.d, cols = c.dense_hidden, ld = cols; break;
        default: break;
    }
    LAT_REQUIRE(rows > 0 && cols > 0, "lattice_net_set_weight: the network has no such weight");
    const bool fp32_dst = kind == 5 || net->f32;
    const int dst_dtype = fp32_dst ? LATTICE_F32 : LATTICE_BF16;
    LAT_REQUIRE(src_dtype == LATTICE_F32 || src_dtype == dst_dtype,
                "lattice_net_set_weight: src_dtype must be f32 or the net's dtype");
    const cudaStream_t st = (cudaStream_t)stream;
    const size_t des = fp32_dst ? 4 : 2;
    if (src_dtype == dst_dtype) {
        LAT_CUDA(cudaMemcpy2DAsync(dst, des * ld, src, des * cols, des * cols, rows, cudaMemcpyDeviceToDevice, st));
        return LATTICE_OK;
    }
    const int64_t n = rows * cols;
    const unsigned grid = (unsigned)((n + 255) / 256 < 148 * 32 ? (n + 255) / 256 : 148 * 32);
    load_rows_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(rows, cols, static_cast<const float*>(src),
                                                          static_cast<__nv_bfloat16*>(dst), ld);
    LAT_CUDA(cudaGetLastError());
    return LATTICE_OK;
}

namespace {
// the network's backward scratch (grown with cudaMalloc, which synchronises the device, only when a
// larger batch or layer needs more)
std::function<void*(size_t)> net_scratch(lattice_net* net) {
    return [net](size_t bytes) -> void* {
        if (net->bwd_ws_bytes < bytes) {
            if (net->bwd_ws) cudaFree(net->bwd_ws);
            net->bwd_ws = nullptr;
            net->bwd_ws_bytes = 0;
            if (cudaMalloc(&net->bwd_ws, bytes) != cudaSuccess) {
                net->bwd_ws = nullptr;
                return nullptr;
            }
            net->bwd_ws_bytes = bytes;
        }
        return net->bwd_ws;
    };
}
}  // namespace

lattice_status lattice_net_tower_backward(lattice_net* net, int64_t batch, const float* dlogits, float* dW1,
                                          float* dW2, void* dX, int32_t dx_dtype, lattice_stream stream) {
    using namespace lat;
    LAT_REQUIRE(net != nullptr && dlogits != nullptr && dW1 != nullptr && dW2 != nullptr,
                "lattice_net_tower_backward: null argument");
    const lattice_net_config& c = net->cfg;
    LAT_REQUIRE(!net->f32, "lattice_net_tower_backward: needs a bf16 network");
    LAT_REQUIRE(batch > 0 && batch <= c.max_batch, "lattice_net_tower_backward: bad batch");
    LAT_REQUIRE(dX == nullptr || dx_dtype == LATTICE_F32 || dx_dtype == LATTICE_BF16,
                "lattice_net_tower_backward: dX dtype must be f32 or bf16");
    TowerBwd a = {};
    a.B = batch;
    a.G = c.domains;
    a.th = c.tower_hidden;
    a.heads = c.heads;
    a.hard = c.hard;
    a.nd = (int64_t)c.n * c.d;
    a.X = net->X[c.blocks & 1];
    a.W1 = net->T1;
    a.W2 = net->T2;
    a.order = net->order;
    a.seg = net->seg;
    a.dlogits = dlogits;
    a.dW1 = dW1;
    a.dW2 = dW2;
    a.dX = dX;
    a.dx_bf16 = dx_dtype == LATTICE_BF16;
    a.scratch = net_scratch(net);
    return tower_backward(a, (cudaStream_t)stream);
}

lattice_status lattice_net_tower_sgd(lattice_net* net, float lr, const float* dW1, const float* dW2, float* master_W1,
                                     float* master_W2, lattice_stream stream) {
    using namespace lat;
    LAT_REQUIRE(net && dW1 && dW2 && master_W1 && master_W2, "lattice_net_tower_sgd: null argument");
    const lattice_net_config& c = net->cfg;
    const int64_t n1 = (int64_t)c.domains * c.tower_hidden * c.n * c.d, n2 = (int64_t)c.domains * c.heads * c.tower_hidden;
    const cudaStream_t st = (cudaStream_t)stream;
    lattice_status s = sgd_update(n1, lr, dW1, master_W1, net->T1, !net->f32, st);
    if (s != LATTICE_OK) return s;
    return sgd_update(n2, lr, dW2, master_W2, net->T2, false, st);
}

lattice_status lattice_net_mlp_backward(lattice_net* net, int64_t batch, const float* dXout, float* const* dW,
                                        float* dFin, float* dResid, lattice_stream stream) {
    using namespace lat;
    LAT_REQUIRE(net != nullptr && dXout != nullptr && dW != nullptr, "lattice_net_mlp_backward: null argument");
    const lattice_net_config& c = net->cfg;
    LAT_REQUIRE(!net->f32, "lattice_net_mlp_backward: needs a bf16 network");
    LAT_REQUIRE(batch > 0 && batch <= c.max_batch, "lattice_net_mlp_backward: bad batch");
    for (int i = 0; i < c.n_mlp; ++i) LAT_REQUIRE(dW[i] != nullptr, "lattice_net_mlp_backward: null dW");
    const cudaStream_t st = (cudaStream_t)stream;
    const int blk = c.blocks - 1;
    MlpBwd a = {};
    a.B = batch;
    a.n_mlp = c.n_mlp;
    for (int i = 0; i <= c.n_mlp; ++i) a.widths[i] = c.mlp[i];
    a.nF = c.nF;
    a.d = c.d;
    a.hard = c.hard;
    a.nd = (int64_t)c.n * c.d;
    a.Xin = net->X[blk & 1];
    a.dXout = dXout;
    a.dFin = dFin;
    a.dResid = dResid;
    a.act[0] = net->Fbuf;
    for (int i = 0; i < c.n_mlp; ++i) {
        a.W[i] = net->mlp[(size_t)blk * c.n_mlp + i];
        a.dW[i] = dW[i];
    }
    // hidden outputs: layer i writes H[i & 1], so after the forward the last two survive; deeper MLPs
    // re-run the forward's own GEMMs (deterministic: bit-identical) and keep a copy of each output
    std::vector<void*> copies;
    if (c.n_mlp <= 3) {
        for (int i = 1; i < c.n_mlp; ++i) a.act[i] = net->H[(i - 1) & 1];
    } else {
        LAT_CUDA(cudaMemsetAsync(net->rowcnt + (size_t)blk * (c.n_mlp - 1) * net->rowcnt_stride, 0,
                                 sizeof(int) * (size_t)(c.n_mlp - 1) * net->rowcnt_stride, st));
        for (int i = 0; i + 1 < c.n_mlp; ++i) {
            gemm::GemmPlan g = net->mlp_plans[(size_t)blk * c.n_mlp + i];
            g.p.M = (int)batch;
            g.grid_y = (int)((batch + 127) / 128);
            lattice_status s = gemm::launch(g, st);
            void* h = nullptr;
            const size_t bytes = sizeof(__nv_bfloat16) * (size_t)batch * c.mlp[i + 1];
            if (s == LATTICE_OK) {
                cudaError_t e = cudaMallocAsync(&h, bytes, st);
                if (e == cudaSuccess) e = cudaMemcpyAsync(h, net->H[i & 1], bytes, cudaMemcpyDeviceToDevice, st);
                if (h) copies.push_back(h);
                if (e != cudaSuccess) s = check_cuda(e, "mlp_backward: hidden copy");
            }
            if (s != LATTICE_OK) {
                for (void* q : copies) cudaFreeAsync(q, st);
                return s;
            }
            a.act[i + 1] = h;
        }
    }
    a.scratch = net_scratch(net);
    const lattice_status s = mlp_backward(a, st);
    for (void* q : copies) cudaFreeAsync(q, st);
    return s;
}

lattice_status lattice_net_weight_sgd(lattice_net* net, int32_t block, int32_t kind, int32_t index, float lr,
                                      const float* grad, float* master, lattice_stream stream) {
    using namespace lat;
    LAT_REQUIRE(net && grad && master, "lattice_net_weight_sgd: null argument");
    LAT_REQUIRE(kind >= 3 && kind <= 7, "lattice_net_weight_sgd: kind must be 3..7 (unpadded weights)");
    void* w = const_cast<void*>(lattice_net_weight(net, block, kind, index));
    LAT_REQUIRE(w != nullptr, "lattice_net_weight_sgd: no such weight (block / kind / index)");
    const lattice_net_config& c = net->cfg;
    int64_t n = 0;
    switch (kind) {
        case 3: n = (int64_t)c.mlp[index + 1] * c.mlp[index]; break;
        case 4: n = (int64_t)c.domains * c.tower_hidden * c.n * c.d; break;
        case 5: n = (int64_t)c.domains * c.heads * c.tower_hidden; break;
        case 6: n = (int64_t)c.dense_hidden * c.dense_in; break;
        default: n = (int64_t)c.dense_features * c.d * c.dense_hidden; break;
    }
    LAT_REQUIRE(n > 0, "lattice_net_weight_sgd: the network has no such weight");
    return sgd_update(n, lr, grad, master, w, kind != 5 && !net->f32, (cudaStream_t)stream);
}

lattice_status lattice_net_set_timing(lattice_net* net, int32_t enable) {
    LAT_REQUIRE(net != nullptr, "lattice_net_set_timing: null net");
    net->timing = enable != 0;
    if (net->timing && net->ev.empty()) {
        const int stages = 2 + net->cfg.blocks * 2 + 1;
        net->ev.resize(stages + 1);
        for (auto& e : net->ev) LAT_CUDA(cudaEventCreate(&e));
    }
    return LATTICE_OK;
}

lattice_status lattice_net_stage_times(lattice_net* net, float* ms, int32_t max_stages, int32_t* n_stages) {
    LAT_REQUIRE(net != nullptr && n_stages != nullptr, "lattice_net_stage_times: null argument");
    *n_stages = 0;
    if (!net->timing || net->ev.empty()) return LATTICE_OK;
    LAT_CUDA(cudaEventSynchronize(net->ev.back()));
    const int n = (int)net->ev.size() - 1;
    for (int i = 0; i < n && i < max_stages; ++i) {
        float t = 0.0f;
        LAT_CUDA(cudaEventElapsedTime(&t, net->ev[i], net->ev[i + 1]));
        ms[i] = t;
        *n_stages = i + 1;
    }
    return LATTICE_OK;
}

lattice_status lattice_net_bucket(lattice_net* net, int64_t batch, const int32_t* domain, lattice_stream stream) {
    using namespace lat;
    LAT_REQUIRE(net != nullptr && domain != nullptr, "lattice_net_bucket: null argument");
    LAT_REQUIRE(batch >= 0 && batch <= net->cfg.max_batch, "lattice_net_bucket: batch exceeds max_batch");
    if (batch == 0) return LATTICE_OK;
    lattice_status s = bucket_ws(batch, net->cfg.domains, domain, net->pos, net->order, net->seg, net->bucket_ws,
                                 (cudaStream_t)stream);
    if (s != LATTICE_OK) return s;
    tiles_kernel<<<1, 256, 0, stream>>>(net->seg, net->cfg.domains, net->tile_rows, net->tiles, net->n_tiles);
    LAT_CUDA(cudaGetLastError());
    return LATTICE_OK;
}

void* lattice_net_buffer(lattice_net* net, int32_t which) {
    if (!net) return nullptr;
    switch (which) {
        case 0: return net->X[0];
        case 1: return net->pos;
        case 2: return net->X[1];
        case 3: return net->Fbuf;
        default: return nullptr;
    }
}

// Stage boundaries recorded when timing is on: [bucket, bag, (fm_lcb, mlp) x blocks, tower]
lattice_status lattice_net_forward(lattice_net* net, const lattice_batch* batch, float* logits,
                                   lattice_stream stream) {
    using namespace lat;
    LAT_REQUIRE(net != nullptr && batch != nullptr, "lattice_net_forward: null argument");
    const lattice_net_config& c = net->cfg;
    const int64_t B = batch->batch;
    LAT_REQUIRE(B >= 0 && B <= c.max_batch, "lattice_net_forward: batch exceeds max_batch");
    if (B == 0) return LATTICE_OK;  // an empty batch needs no logits buffer
    LAT_REQUIRE(logits != nullptr, "lattice_net_forward: null logits");
    LAT_REQUIRE(batch->domain != nullptr, "lattice_net_forward: null domain");
    const int nd = c.n * c.d;
    int ei = 0;
    auto mark = [&]() -> lattice_status {
        if (net->timing) LAT_CUDA(cudaEventRecord(net->ev[ei++], stream));
        return LATTICE_OK;
    };
#define FWD_TRY(x)                                \
    do {                                          \
        lattice_status _s = (x);                  \
        if (_s != LATTICE_OK) return _s;          \
    } while (0)
    // NVTX ranges name the stages for Nsight Systems / any NVTX tool (no-ops without one attached)
    struct Range {
        bool open = true;
        explicit Range(const char* name) { nvtxRangePushA(name); }
        void end() {
            if (open) nvtxRangePop();
            open = false;
        }
        ~Range() { end(); }
    } range_forward("lattice::net_forward");
    const bool in_place = !batch->tables && batch->pooled_layout == 2;  // X0 written by peers
    const int nc = c.n - c.dense_features;  // sparse (table-pooled) embeddings come first
    FWD_TRY(mark());
    Range range_embed("lattice::bucket+embedding");
    if (!in_place && batch->check) {  // checked: a domain outside [0, domains) is a DataError
        LAT_CUDA(cudaMemsetAsync(net->bad_domain, 0xff, sizeof(*net->bad_domain), stream));
        FWD_TRY(bucket_ws(B, c.domains, batch->domain, net->pos, net->order, net->seg, net->bucket_ws,
                          (cudaStream_t)stream, net->bad_domain));
        tiles_kernel<<<1, 256, 0, stream>>>(net->seg, c.domains, net->tile_rows, net->tiles, net->n_tiles);
        LAT_CUDA(cudaGetLastError());
        unsigned long long bad = ~0ull;
        LAT_CUDA(cudaMemcpyAsync(&bad, net->bad_domain, sizeof(bad), cudaMemcpyDeviceToHost, stream));
        LAT_CUDA(cudaStreamSynchronize(stream));
        if (bad != ~0ull)
            return set_error(LATTICE_DATA,
                             "network: sample " + std::to_string(bad) + " has a domain outside [0, " +
                                 std::to_string(c.domains) + ")",
                             (int64_t)bad);
    } else if (!in_place) {
        FWD_TRY(lattice_net_bucket(net, B, batch->domain, stream));
    }
    FWD_TRY(mark());
    if (in_place) {
        // lattice_net_bucket ran for this batch and lattice_peer_embedding_bag filled X0
    } else if (batch->tables) {
        lattice_bag_args a = {};
        a.features = nc;
        a.batch = B;
        a.dim = c.d;
        a.table_dtype = batch->table_dtype;
        a.tables = batch->tables;
        a.rows = batch->rows;
        a.offsets = batch->offsets;
        a.ids = batch->ids;
        a.out_dtype = net->f32 ? LATTICE_F32 : LATTICE_BF16;
        a.out = net->X[0];
        a.out_row_stride = nd;
        a.out_feature_offset = 0;
        a.sample_pos = net->pos;
        a.normalize = 1;
        a.check = batch->check ? 1 : 0;
        a.sources = 1;
        FWD_TRY(lattice_embedding_bag(&a, stream));
    } else {
        LAT_REQUIRE(batch->pooled != nullptr, "lattice_net_forward: need tables or pooled input");
        const int64_t warps = B * nc;
        const unsigned grid = (unsigned)((warps * 32 + 255) / 256 < 148 * 64 ? (warps * 32 + 255) / 256 : 148 * 64);
        if (batch->pooled_layout == 1) {
            LAT_REQUIRE(batch->shards >= 1 && nc % batch->shards == 0 &&
                            batch->table_dtype == (net->f32 ? LATTICE_F32 : LATTICE_BF16),
                        "lattice_net_forward: sharded pooled input needs the net dtype and shards dividing n");
            shard_gather_kernel<<<grid, 256, 0, stream>>>(B, nc, c.d, (int)net->es, batch->shards,
                                                          static_cast<const uint8_t*>(batch->pooled), net->pos,
                                                          static_cast<uint8_t*>(net->X[0]), c.n);
        } else if (batch->table_dtype == LATTICE_F32) {
            if (net->f32)
                pooled_norm_kernel<float, float><<<grid, 256, 0, stream>>>(
                    B, nc, c.d, static_cast<const float*>(batch->pooled), net->pos, static_cast<float*>(net->X[0]), c.n, 0);
            else
                pooled_norm_kernel<float, __nv_bfloat16><<<grid, 256, 0, stream>>>(
                    B, nc, c.d, static_cast<const float*>(batch->pooled), net->pos,
                    static_cast<__nv_bfloat16*>(net->X[0]), c.n, 0);
        } else {
            if (net->f32)
                pooled_norm_kernel<__nv_bfloat16, float><<<grid, 256, 0, stream>>>(
                    B, nc, c.d, static_cast<const __nv_bfloat16*>(batch->pooled), net->pos,
                    static_cast<float*>(net->X[0]), c.n, 0);
            else
                pooled_norm_kernel<__nv_bfloat16, __nv_bfloat16><<<grid, 256, 0, stream>>>(
                    B, nc, c.d, static_cast<const __nv_bfloat16*>(batch->pooled), net->pos,
                    static_cast<__nv_bfloat16*>(net->X[0]), c.n, 0);
        }
        LAT_CUDA(cudaGetLastError());
    }
    // every swish GEMM of this forward counts row-statistics arrivals in its own zeroed slot,
    // so no memset sits between the dense-chain kernels (they overlap through PDL)
    LAT_CUDA(cudaMemsetAsync(net->rowcnt, 0, sizeof(int) * net->rowcnt_total, stream));
    if (c.dense_features > 0) {  // dense processor -> rows [nc, n) of X0
        LAT_REQUIRE(batch->dense != nullptr, "lattice_net_forward: the network has dense features; batch.dense is null");
        LAT_CUDA(cudaMemcpyAsync(net->Din, batch->dense, net->es * (size_t)B * c.dense_in, cudaMemcpyDeviceToDevice,
                                 stream));
        for (int i = 0; i < 2; ++i) {
            gemm::GemmPlan g = net->dense_plans[i];
            g.p.M = (int)B;
            g.grid_y = (int)((B + 127) / 128);
            FWD_TRY(gemm::launch(g, stream));
        }
        const int64_t warps = B * c.dense_features;
        const unsigned grid = (unsigned)((warps * 32 + 255) / 256 < 148 * 64 ? (warps * 32 + 255) / 256 : 148 * 64);
        if (net->f32)
            pooled_norm_kernel<float, float><<<grid, 256, 0, stream>>>(
                B, c.dense_features, c.d, static_cast<const float*>(net->Od), net->pos,
                static_cast<float*>(net->X[0]), c.n, nc);
        else
            pooled_norm_kernel<__nv_bfloat16, __nv_bfloat16><<<grid, 256, 0, stream>>>(
                B, c.dense_features, c.d, static_cast<const __nv_bfloat16*>(net->Od), net->pos,
                static_cast<__nv_bfloat16*>(net->X[0]), c.n, nc);
        LAT_CUDA(cudaGetLastError());
    }
    range_embed.end();
    FWD_TRY(mark());
    for (int blk = 0; blk < c.blocks; ++blk) {
        Range range_block("lattice::dwfb_block");
        fm::Plan fp = net->fm_plans[blk];
        fp.p.B = B;
        FWD_TRY(fm::launch(fp, stream));
        FWD_TRY(mark());
        for (int li = 0; li < c.n_mlp; ++li) {
            gemm::GemmPlan g = net->mlp_plans[(size_t)blk * c.n_mlp + li];
            g.p.M = (int)B;
            g.grid_y = (int)((B + 127) / 128);
            FWD_TRY(gemm::launch(g, stream));
        }
        FWD_TRY(mark());
    }
    Range range_towers("lattice::towers");
    gemm::GemmPlan t = net->tower_plan;
    t.p.M = (int)B;
    t.p.logits = logits;
    if (net->tower_pair) {
        t.grid_y = (int)((B + 255) / 256) + c.domains;
        FWD_TRY(gemm::launch(t, stream));
        const unsigned grid = (unsigned)((B * 32 + 255) / 256 < 148 * 16 ? (B * 32 + 255) / 256 : 148 * 16);
        tower_heads_kernel<<<grid, 256, 0, stream>>>(B, c.tower_hidden, c.heads, c.domains, net->Htower, net->seg,
                                                      net->order, net->T2, logits);
        LAT_CUDA(cudaGetLastError());
    } else {
        t.grid_y = (int)((B + 127) / 128) + c.domains;
        FWD_TRY(gemm::launch(t, stream));
    }
    FWD_TRY(mark());
    if (batch->check) FWD_TRY(lattice_device_check(stream));  // checked forwards synchronise anyway
#undef FWD_TRY
    return LATTICE_OK;
}

}  // extern "C"
