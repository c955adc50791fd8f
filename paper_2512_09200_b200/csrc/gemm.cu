// gemm.cu -- tcgen05 GEMM kernel (see gemm.cuh) + host launch helpers + lattice_gemm.
#include <cudaTypedefs.h>

#include <cstdlib>
#include <string>

#include "gemm.cuh"
#include "gemm_host.h"

namespace lat {
namespace gemm {

// ---------------------------------------------------------------------------------------------
// epilogue helpers (thread = accumulator row)
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ void store_row32(const Params& p, int64_t m, int n, const float* v) {
    if (p.out_bf16) {
        __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(p.C) + m * p.ldc + n;
        if (n + 32 <= p.N) {
#pragma unroll
            for (int j = 0; j < 32; j += 8)
                *reinterpret_cast<uint4*>(dst + j) =
                    make_uint4(pack_bf16x2(v[j], v[j + 1]), pack_bf16x2(v[j + 2], v[j + 3]),
                               pack_bf16x2(v[j + 4], v[j + 5]), pack_bf16x2(v[j + 6], v[j + 7]));
        } else {
            for (int j = 0; j < 32 && n + j < p.N; ++j) dst[j] = __float2bfloat16_rn(v[j]);
        }
    } else {
        float* dst = static_cast<float*>(p.C) + m * p.ldc + n;
        if (n + 32 <= p.N) {
#pragma unroll
            for (int j = 0; j < 32; j += 4)
                *reinterpret_cast<float4*>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        } else {
            for (int j = 0; j < 32 && n + j < p.N; ++j) dst[j] = v[j];
        }
    }
}

// Sum a per-row partial across the cluster (rank order), via DSMEM. Every thread of the 4
// epilogue warps calls this exactly once per exchange `slot` with its own row.
__device__ __forceinline__ float cluster_row_sum(float part, int row, int C, float* xbuf,
                                                 uint64_t* xbar, uint32_t phase) {
    if (C == 1) return part;
    const uint32_t my = tc::cluster_rank();
    const uint32_t local = tc::smem_u32(&xbuf[my * BM + row]);
    const uint32_t bar = tc::smem_u32(xbar);
    for (int r = 0; r < C; ++r) {
        tc::st_cluster_f32(tc::mapa(local, r), part);
        tc::mbar_arrive_remote(tc::mapa(bar, r));
    }
    tc::mbar_wait_cluster(xbar, phase);
    float s = 0.0f;
    for (int r = 0; r < C; ++r) s += xbuf[r * BM + row];
    return s;
}

template <int GROUP>
__device__ __forceinline__ void resid_norm_group(const Params& p, uint32_t taddr, int64_t m, int n,
                                                 bool valid) {
    float v[GROUP];
#pragma unroll
    for (int c = 0; c < GROUP; c += 32) tc::tmem_ld32(taddr + c, v + c);
    if (!valid) return;
    const __nv_bfloat16* r = p.resid + m * p.ldr + n;
#pragma unroll
    for (int c = 0; c < GROUP; c += 8) {
        const uint4 q = *reinterpret_cast<const uint4*>(r + c);
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            v[c + 2 * i] += bf16_lo(w[i]);
            v[c + 2 * i + 1] += bf16_hi(w[i]);
        }
    }
    float ss = 0.0f;
#pragma unroll
    for (int c = 0; c < GROUP; ++c) ss += v[c] * v[c];
    const float denom = sqrtf(ss / (float)GROUP + 1e-6f);
#pragma unroll
    for (int c = 0; c < GROUP; ++c) v[c] = v[c] / denom;
#pragma unroll
    for (int c = 0; c < GROUP; c += 32) store_row32(p, m, n + c, v + c);
}

// ---------------------------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------------------------
template <int BN, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const Params p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr int A_BYTES = BM * BK * 2;
    constexpr int B_BYTES = BN * BK * 2;
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* accum_full = empty + STAGES;
    uint64_t* xbar = accum_full + 1;     // row-stat exchange (phase 0)
    uint64_t* hbar = xbar + 1;           // head-partial exchange (phase 0)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(hbar + 1);
    float* xbuf = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(full) + 256);
    float* hbuf = xbuf + kMaxCluster * BM;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int C = p.cluster;

    // tile coordinates
    int group = 0, m0, m_end;
    if (p.tiles) {
        if ((int)blockIdx.y >= *p.n_tiles) return;  // whole cluster shares blockIdx.y
        const int4 t = p.tiles[blockIdx.y];
        group = t.x;
        m0 = t.y;
        m_end = t.z;
    } else {
        m0 = blockIdx.y * BM;
        m_end = p.M;
    }
    const int n0 = blockIdx.x * BN;
    const int b_row0 = group * p.b_rows_per_group + n0;
    const int nk = (p.K + BK - 1) / BK;

    if (warp == 0 && lane == 0) {
        tc::tma_prefetch(&tmA);
        tc::tma_prefetch(&tmB);
        for (int s = 0; s < STAGES; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        tc::mbar_init(accum_full, 1);
        tc::mbar_init(xbar, BM * C);
        tc::mbar_init(hbar, BM * C);
        tc::fence_mbar_init();
    }
    if (warp == 1) tc::tmem_alloc(tmem_slot, BN);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (C > 1) tc::cluster_sync();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % STAGES;
                const uint32_t ph = (kb / STAGES) & 1;
                tc::mbar_wait(&empty[s], ph ^ 1);
                tc::mbar_expect_tx(&full[s], A_BYTES + B_BYTES);
                tc::tma_load_2d(sA + s * A_BYTES, &tmA, &full[s], kb * BK, m0);
                tc::tma_load_2d(sB + s * B_BYTES, &tmB, &full[s], kb * BK, b_row0);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---- MMA issuer
            constexpr uint32_t idesc = tc::idesc_bf16(BM, BN, 0, 0);
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % STAGES;
                const uint32_t ph = (kb / STAGES) & 1;
                tc::mbar_wait(&full[s], ph);
                tc::fence_after();
                const uint32_t a_base = tc::smem_u32(sA + s * A_BYTES);
                const uint32_t b_base = tc::smem_u32(sB + s * B_BYTES);
#pragma unroll
                for (int k = 0; k < BK / 16; ++k) {
                    const uint64_t ad = tc::sdesc(a_base + k * 32, 16, 1024, 2);
                    const uint64_t bd = tc::sdesc(b_base + k * 32, 16, 1024, 2);
                    tc::mma_f16(tmem, ad, bd, idesc, (kb | k) != 0);
                }
                tc::mma_commit(&empty[s]);
            }
            tc::mma_commit(accum_full);
        }
    } else {  // ---- epilogue warps 2..5
        const int q = warp & 3;
        const int row = q * 32 + lane;
        const int64_t m = (int64_t)m0 + row;
        const bool valid = m < m_end;
        const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16);
        tc::mbar_wait(accum_full, 0);
        tc::fence_after();
        const int epi = p.epi;
        if (epi == kStore) {
#pragma unroll 1
            for (int c = 0; c < BN; c += 32) {
                float v[32];
                tc::tmem_ld32(taddr + c, v);
                if (valid && n0 + c < p.N) store_row32(p, m, n0 + c, v);
            }
        } else if (epi == kResidNorm) {
            if (p.group == 128) {
#pragma unroll 1
                for (int g = 0; g < BN; g += 128)
                    if (n0 + g < p.N) resid_norm_group<128>(p, taddr + g, m, n0 + g, valid);
            } else {
#pragma unroll 1
                for (int g = 0; g < BN; g += 64)
                    if (n0 + g < p.N) resid_norm_group<64>(p, taddr + g, m, n0 + g, valid);
            }
        } else {  // row-wide swish_rn (+ tower heads)
            const bool hard = epi == kSwishHard || epi == kTowerHard;
            float ss = 0.0f;
#pragma unroll 1
            for (int c = 0; c < BN; c += 32) {
                float v[32];
                tc::tmem_ld32(taddr + c, v);
                // columns >= N may hold another group's weights (stacked towers): mask them
#pragma unroll
                for (int j = 0; j < 32; ++j) ss += (n0 + c + j < p.N) ? v[j] * v[j] : 0.0f;
            }
            const float total = cluster_row_sum(ss, row, C, xbuf, xbar, 0);
            const float denom = sqrtf(total / (float)p.N_full + 1e-6f);
            if (epi == kSwish || epi == kSwishHard) {
#pragma unroll 1
                for (int c = 0; c < BN; c += 32) {
                    float v[32];
                    tc::tmem_ld32(taddr + c, v);
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = act_swish(v[j] / denom, hard);
                    if (valid && n0 + c < p.N) store_row32(p, m, n0 + c, v);
                }
            } else {  // tower: heads = W2_g . swish_rn(row)
                float part[kMaxHeads];
#pragma unroll
                for (int j = 0; j < kMaxHeads; ++j) part[j] = 0.0f;
                const float* w2 = p.W2 + (size_t)group * p.heads * p.N_full;
#pragma unroll 1
                for (int c = 0; c < BN; c += 32) {
                    float v[32];
                    tc::tmem_ld32(taddr + c, v);
                    if (n0 + c >= p.N) continue;
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = (n0 + c + j < p.N) ? act_swish(v[j] / denom, hard) : 0.0f;
#pragma unroll
                    for (int h = 0; h < kMaxHeads; ++h) {
                        if (h < p.heads) {
                            const float* wr = w2 + (size_t)h * p.N_full + n0 + c;
                            float a = 0.0f;
                            if (n0 + c + 32 <= p.N) {
#pragma unroll
                                for (int j = 0; j < 32; j += 4) {
                                    const float4 w = __ldg(reinterpret_cast<const float4*>(wr + j));
                                    a += v[j] * w.x + v[j + 1] * w.y + v[j + 2] * w.z + v[j + 3] * w.w;
                                }
                            } else {
#pragma unroll
                                for (int j = 0; j < 32; ++j)
                                    if (n0 + c + j < p.N) a += v[j] * __ldg(wr + j);
                            }
                            part[h] += a;
                        }
                    }
                }
                // reduce head partials into cluster rank 0 (rank order), then write
                const uint32_t my = C > 1 ? tc::cluster_rank() : 0;
                if (C > 1) {
#pragma unroll
                    for (int h = 0; h < kMaxHeads; ++h)
                        if (h < p.heads)
                            tc::st_cluster_f32(
                                tc::mapa(tc::smem_u32(&hbuf[(my * p.heads + h) * BM + row]), 0), part[h]);
                    tc::mbar_arrive_remote(tc::mapa(tc::smem_u32(hbar), 0));
                }
                if (my == 0) {
                    if (C > 1) {
                        // hbar expects BM*C arrivals; each CTA's 128 threads arrive once
                        tc::mbar_wait_cluster(hbar, 0);
#pragma unroll
                        for (int h = 0; h < kMaxHeads; ++h) {
                            if (h < p.heads) {
                                float s = 0.0f;
                                for (int r = 0; r < C; ++r) s += hbuf[(r * p.heads + h) * BM + row];
                                part[h] = s;
                            }
                        }
                    }
                    if (valid) {
                        const int64_t b = p.order ? (int64_t)p.order[m] : m;
#pragma unroll
                        for (int h = 0; h < kMaxHeads; ++h)
                            if (h < p.heads) p.logits[b * p.heads + h] = part[h];
                    }
                }
            }
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc(tmem, BN);
}

// ---------------------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------------------
namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }
    return fn;
}

template <int BN, int STAGES>
lattice_status launch_t(const CUtensorMap& ta, const CUtensorMap& tb, const Params& p, int grid_y,
                        cudaStream_t st) {
    const size_t smem = smem_bytes(BN, STAGES, p.cluster, p.heads);
    static bool attr_done = false;
    if (!attr_done) {
        LAT_CUDA(cudaFuncSetAttribute(gemm_kernel<BN, STAGES>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        LAT_CUDA(cudaFuncSetAttribute(gemm_kernel<BN, STAGES>,
                                      cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        attr_done = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((p.N + BN - 1) / BN, grid_y, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = p.cluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    LAT_CUDA(cudaLaunchKernelEx(&cfg, gemm_kernel<BN, STAGES>, ta, tb, p));
    return LATTICE_OK;
}
}  // namespace

lattice_status make_map_2d(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer,
                           uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer) {
    auto fn = encode_fn();
    if (!fn) return set_error(LATTICE_CUDA, "cuTensorMapEncodeTiled unavailable");
    if ((reinterpret_cast<uintptr_t>(base) & 15) || (row_stride_bytes & 15))
        return set_error(LATTICE_USAGE, "TMA operand: base and row stride must be 16-byte aligned");
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {row_stride_bytes};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                    box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return set_error(LATTICE_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return LATTICE_OK;
}

int default_stages() {
    static int s = -1;
    if (s < 0) {
        const char* e = std::getenv("LATTICE_GEMM_STAGES");
        s = e ? std::atoi(e) : 4;
        if (s != 2 && s != 4) s = 4;
    }
    return s;
}

lattice_status launch(const GemmPlan& g, cudaStream_t st) {
    if (g.stages == 2) return launch_t<256, 2>(g.ta, g.tb, g.p, g.grid_y, st);
    return launch_t<256, 4>(g.ta, g.tb, g.p, g.grid_y, st);
}

lattice_status plan(GemmPlan* g, const void* A, int64_t lda, int64_t a_rows, const void* B,
                    int64_t ldb, int64_t b_rows, const Params& p, int grid_y) {
    lattice_status s = make_map_2d(&g->ta, A, (uint64_t)p.K, (uint64_t)a_rows, (uint64_t)lda * 2, BK, BM);
    if (s != LATTICE_OK) return s;
    s = make_map_2d(&g->tb, B, (uint64_t)p.K, (uint64_t)b_rows, (uint64_t)ldb * 2, BK, 256);
    if (s != LATTICE_OK) return s;
    g->p = p;
    g->grid_y = grid_y;
    g->stages = default_stages();
    return LATTICE_OK;
}

}  // namespace gemm
}  // namespace lat

extern "C" lattice_status lattice_gemm(const lattice_gemm_args* a, lattice_stream stream) {
    using namespace lat;
    using namespace lat::gemm;
    LAT_REQUIRE(a != nullptr, "lattice_gemm: null args");
    LAT_REQUIRE(a->M >= 0 && a->N > 0 && a->K > 0, "lattice_gemm: bad sizes");
    LAT_REQUIRE(a->M < (1ll << 31) && a->N < (1ll << 31) && a->K < (1ll << 31), "lattice_gemm: size overflow");
    LAT_REQUIRE(a->K % 8 == 0 && a->lda % 8 == 0 && a->ldb % 8 == 0,
                "lattice_gemm: K, lda, ldb must be multiples of 8 (16-byte TMA strides)");
    LAT_REQUIRE(a->epilogue >= 0 && a->epilogue <= 3, "lattice_gemm: unknown epilogue");
    if (a->M == 0) return LATTICE_OK;
    Params p = {};
    p.M = (int)a->M;
    p.N = (int)a->N;
    p.K = (int)a->K;
    p.C = a->C;
    p.ldc = a->ldc;
    p.out_bf16 = a->out_dtype == LATTICE_BF16;
    p.epi = a->epilogue;
    p.resid = static_cast<const __nv_bfloat16*>(a->resid);
    p.ldr = a->ldr;
    p.group = a->group;
    p.N_full = p.N;
    p.cluster = 1;
    p.heads = 0;
    if (p.epi == kSwish || p.epi == kSwishHard) {
        p.cluster = (p.N + 255) / 256;
        LAT_REQUIRE(p.cluster <= kMaxCluster, "lattice_gemm: swish_rn rows wider than 2048 are not supported");
    }
    if (p.epi == kResidNorm) {
        LAT_REQUIRE(a->resid && (a->group == 128 || a->group == 64) && p.N % a->group == 0 &&
                        a->ldr % 8 == 0 && p.out_bf16,
                    "lattice_gemm: residual-norm epilogue needs bf16 out, group 64/128 dividing N");
    }
    GemmPlan g;
    lattice_status s = plan(&g, a->A, a->lda, a->M, a->B, a->ldb, a->N, p, (int)((a->M + BM - 1) / BM));
    if (s != LATTICE_OK) return s;
    return launch(g, stream);
}
