// gemm.cu -- persistent tcgen05 GEMM kernel (see gemm.cuh) + host plan/launch + lattice_gemm.
//
// Persistent: one CTA per SM (or one cluster of C CTAs per C SMs) walks a static schedule of
// output tiles. The TMA warp runs ahead through a STAGES-deep smem ring across tile
// boundaries; the MMA warp accumulates tile i into TMEM region (i & 1) while the epilogue
// warps drain region ((i-1) & 1), so epilogues (and their DSMEM exchanges) hide under the
// next tile's mainloop. Dense tiles are rasterised in bands of 16 M-tiles so concurrently
// running CTAs share A and B tiles in L2.
#include <cudaTypedefs.h>

#include <cstdlib>
#include <string>

#include "gemm.cuh"
#include "gemm_host.h"

namespace lat {
namespace gemm {

__device__ __forceinline__ uint32_t f2u(float x) { return __float_as_uint(x); }

// Row-statistics waits of the CTA-pair swish epilogue that gave up (see gemm2_kernel): read and
// cleared by lattice_device_check. Never non-zero while every pair of the grid is co-resident.
__device__ unsigned int g_exchange_timeouts = 0;
constexpr uint64_t kExchangeTimeoutNs = 5ull * 1000 * 1000 * 1000;

__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

constexpr int BN = 256;
constexpr int kRasterGroup = 16;

// ---------------------------------------------------------------------------------------------
// epilogue helpers (thread = accumulator row)
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ void store_row32(const Params& p, int64_t m, int n, const float* v) {
    if (p.out_bf16) {
        __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(p.C) + m * p.ldc + n;
        if (n + 32 <= p.N && aligned32(dst)) {  // whole sectors: two 32-byte stores
#pragma unroll
            for (int j = 0; j < 32; j += 16)
                st_global_256(dst + j,
                              make_uint4(pack_bf16x2(v[j], v[j + 1]), pack_bf16x2(v[j + 2], v[j + 3]),
                                         pack_bf16x2(v[j + 4], v[j + 5]), pack_bf16x2(v[j + 6], v[j + 7])),
                              make_uint4(pack_bf16x2(v[j + 8], v[j + 9]), pack_bf16x2(v[j + 10], v[j + 11]),
                                         pack_bf16x2(v[j + 12], v[j + 13]), pack_bf16x2(v[j + 14], v[j + 15])));
        } else if (n + 32 <= p.N) {
#pragma unroll
            for (int j = 0; j < 32; j += 8)
                *reinterpret_cast<uint4*>(dst + j) =
                    make_uint4(pack_bf16x2(v[j], v[j + 1]), pack_bf16x2(v[j + 2], v[j + 3]),
                               pack_bf16x2(v[j + 4], v[j + 5]), pack_bf16x2(v[j + 6], v[j + 7]));
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (n + j < p.N) dst[j] = __float2bfloat16_rn(v[j]);
        }
    } else {
        float* dst = static_cast<float*>(p.C) + m * p.ldc + n;
        if (n + 32 <= p.N && aligned32(dst)) {
#pragma unroll
            for (int j = 0; j < 32; j += 8)
                st_global_256(dst + j, make_uint4(f2u(v[j]), f2u(v[j + 1]), f2u(v[j + 2]), f2u(v[j + 3])),
                              make_uint4(f2u(v[j + 4]), f2u(v[j + 5]), f2u(v[j + 6]), f2u(v[j + 7])));
        } else if (n + 32 <= p.N) {
#pragma unroll
            for (int j = 0; j < 32; j += 4)
                *reinterpret_cast<float4*>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (n + j < p.N) dst[j] = v[j];
        }
    }
}

// Sum a per-row partial across the cluster (rank order) through DSMEM, pull model: each CTA
// writes its partials to its own slot, every warp then announces "my 32 rows are ready" with
// ONE release arrive per peer CTA (4 warps x C peers per barrier phase), waits on its own
// barrier (CTA-scope spin, one cluster acquire fence after), and reads the C peers' partials
// with ld.shared::cluster. `xbuf` alternates with the tile so a fast CTA can run one tile
// ahead: it only rewrites a slot after every peer arrived for the tile in between, i.e.
// after they finished reading that slot.
__device__ __forceinline__ float cluster_row_sum(float part, int row, int lane, int C, float* xbuf,
                                                 uint64_t* xbar, uint32_t phase) {
    if (C == 1) return part;
    xbuf[row] = part;
    __syncwarp();
    if (lane == 0) {
        const uint32_t bar = tc::smem_u32(xbar);
        for (int r = 0; r < C; ++r) tc::mbar_arrive_remote(tc::mapa(bar, r));
    }
    tc::mbar_wait(xbar, phase);
    tc::fence_acq_rel_cluster();
    const uint32_t local = tc::smem_u32(&xbuf[row]);
    float s = 0.0f;
    for (int r = 0; r < C; ++r) s += tc::ld_cluster_f32(tc::mapa(local, r));
    return s;
}

template <int GROUP>
__device__ __forceinline__ void resid_norm_group(const Params& p, uint32_t taddr, int64_t m, int n,
                                                 bool valid) {
    float v[GROUP];
#pragma unroll
    for (int c = 0; c < GROUP; c += 32) tc::tmem_ld32(taddr + c, v + c);
    if (!valid) return;
    if (p.out_bf16) {
        const __nv_bfloat16* r = static_cast<const __nv_bfloat16*>(p.resid) + m * p.ldr + n;
        const bool wide = aligned32(r);  // 32-byte loads: whole sectors per lane
#pragma unroll
        for (int c = 0; c < GROUP; c += 16) {
            uint4 q0, q1;
            if (wide) {
                ld_global_256(r + c, q0, q1);
            } else {
                q0 = *reinterpret_cast<const uint4*>(r + c);
                q1 = *reinterpret_cast<const uint4*>(r + c + 8);
            }
            const uint32_t w[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                v[c + 2 * i] += bf16_lo(w[i]);
                v[c + 2 * i + 1] += bf16_hi(w[i]);
            }
        }
    } else {
        const float* r = static_cast<const float*>(p.resid) + m * p.ldr + n;
#pragma unroll
        for (int c = 0; c < GROUP; c += 4) {
            const float4 q = *reinterpret_cast<const float4*>(r + c);
            v[c] += q.x;
            v[c + 1] += q.y;
            v[c + 2] += q.z;
            v[c + 3] += q.w;
        }
    }
    float ss = 0.0f;
#pragma unroll
    for (int c = 0; c < GROUP; ++c) ss += v[c] * v[c];
    const float inv = 1.0f / sqrtf(ss * (1.0f / (float)GROUP) + 1e-6f);
#pragma unroll
    for (int c = 0; c < GROUP; ++c) v[c] *= inv;
#pragma unroll
    for (int c = 0; c < GROUP; c += 32) store_row32(p, m, n + c, v + c);
}

// Tile schedule shared by all three roles.
struct Sched {
    int units;    // work units (C>1: M-tiles processed by a whole cluster; C==1: output tiles)
    int first, stride;
    int nt;       // N tiles
    int mt;       // M tiles (dense)
};

__device__ __forceinline__ void decode(const Params& p, const Sched& s, int u, int rank, int& group,
                                       int& m0, int& m_end, int& n0) {
    int mu, nn;
    if (p.cluster > 1) {
        mu = u;
        nn = rank;
    } else if (p.tiles) {
        mu = u / s.nt;
        nn = u % s.nt;
    } else {  // banded raster: kRasterGroup M-tiles share each N-tile sweep
        const int per = kRasterGroup * s.nt;
        const int g = u / per, in = u % per;
        const int rows = min(kRasterGroup, s.mt - g * kRasterGroup);
        mu = g * kRasterGroup + in % rows;
        nn = in / rows;
    }
    if (p.tiles) {
        const int4 t = p.tiles[mu];
        group = t.x;
        m0 = t.y;
        m_end = t.z;
    } else {
        group = 0;
        m0 = mu * BM;
        m_end = p.M;
    }
    n0 = nn * BN;
}

// ---------------------------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------------------------
template <int STAGES, typename T>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const Params p) {
    extern __shared__ uint8_t smem_raw[];
    // align to 1024 B (SW128) by offsetting the __shared__ pointer itself, so the compiler keeps
    // the shared address space (LDS/STS rather than generic loads)
    uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
    using Op = tc::Operand<T>;
    constexpr int BKE = Op::kRow;         // elements per 128-byte k-block row
    constexpr int A_BYTES = BM * 128;
    constexpr int B_BYTES = BN * 128;
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;    // [2] accumulator region ready
    uint64_t* tempty = tfull + 2;        // [2] accumulator region drained
    uint64_t* xbar = tempty + 2;         // [2] row-stat exchange
    uint64_t* hbar = xbar + 2;           // [2] head-partial exchange
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(hbar + 2);
    float* xbuf = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(full) + 256);  // [2][8][128]
    float* hbuf = xbuf + 2 * kMaxCluster * BM;                                       // [2][C][heads][128]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int C = p.cluster;
    const int rank = C > 1 ? (int)tc::cluster_rank() : 0;
    // PDL: the tile count and every operand may come from the preceding kernel
    tc::griddep_wait();
    tc::griddep_launch_dependents();

    Sched s;
    s.nt = (p.N + BN - 1) / BN;
    s.mt = (p.M + BM - 1) / BM;
    if (C > 1) {
        s.units = p.tiles ? *p.n_tiles : s.mt;
        s.first = blockIdx.x / C;
        s.stride = gridDim.x / C;
    } else {
        s.units = (p.tiles ? *p.n_tiles : s.mt) * s.nt;
        s.first = blockIdx.x;
        s.stride = gridDim.x;
    }
    const int nk = (p.K + BKE - 1) / BKE;

    if (warp == 0 && lane == 0) {
        tc::tma_prefetch(&tmA);
        tc::tma_prefetch(&tmB);
        for (int i = 0; i < STAGES; ++i) {
            tc::mbar_init(&full[i], 1);
            tc::mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            tc::mbar_init(&tfull[i], 1);
            tc::mbar_init(&tempty[i], BM);
            tc::mbar_init(&xbar[i], 4 * C);  // one arrive per epilogue warp per CTA
            tc::mbar_init(&hbar[i], 4 * C);  // one arrive per epilogue warp per CTA
        }
        tc::fence_mbar_init();
    }
    if (warp == 1) tc::tmem_alloc(tmem_slot, 2 * BN);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (C > 1) tc::cluster_sync();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer
            int g = 0;
            for (int u = s.first; u < s.units; u += s.stride) {
                int group, m0, m_end, n0;
                decode(p, s, u, rank, group, m0, m_end, n0);
                const int b_row0 = group * p.b_rows_per_group + n0;
                for (int kb = 0; kb < nk; ++kb, ++g) {
                    const int st = g % STAGES;
                    const uint32_t ph = (g / STAGES) & 1;
                    tc::mbar_wait(&empty[st], ph ^ 1);
                    tc::mbar_expect_tx(&full[st], A_BYTES + B_BYTES);
                    // K-major: one [rows][64 K] box; MN-major: [64 K rows][64 MN] panels, 8 KB apart
                    if (p.a_mn) {
                        for (int q = 0; q < BM / 64; ++q)
                            tc::tma_load_2d(sA + st * A_BYTES + q * 8192, &tmA, &full[st], m0 + q * 64, kb * BKE);
                    } else {
                        tc::tma_load_2d(sA + st * A_BYTES, &tmA, &full[st], kb * BKE, m0);
                    }
                    if (p.b_mn) {
                        for (int q = 0; q < BN / 64; ++q)
                            tc::tma_load_2d(sB + st * B_BYTES + q * 8192, &tmB, &full[st], b_row0 + q * 64, kb * BKE);
                    } else {
                        tc::tma_load_2d(sB + st * B_BYTES, &tmB, &full[st], kb * BKE, b_row0);
                    }
                }
            }
        }
    } else if (warp == 1) {
        {  // ---- MMA issuer: the whole warp walks the schedule, one elected lane issues
            const uint32_t idesc = tc::idesc_fmt(Op::kFormat, BM, BN, p.a_mn, p.b_mn);
            int g = 0, i = 0;
            for (int u = s.first; u < s.units; u += s.stride, ++i) {
                const int acc = i & 1;
                tc::mbar_wait(&tempty[acc], ((i >> 1) & 1) ^ 1);
                tc::fence_after();
                const uint32_t d_tmem = tmem + acc * BN;
                for (int kb = 0; kb < nk; ++kb, ++g) {
                    const int st = g % STAGES;
                    const uint32_t ph = (g / STAGES) & 1;
                    tc::mbar_wait(&full[st], ph);
                    tc::fence_after();
                    const uint32_t a_base = tc::smem_u32(sA + st * A_BYTES);
                    const uint32_t b_base = tc::smem_u32(sB + st * B_BYTES);
#pragma unroll
                    for (int k = 0; k < 4; ++k) {  // 4 x 32-byte K slices per k-block
                        // K-major: the slice is 32 bytes into each 128-byte row; MN-major: 16 K rows
                        // further into each 64-wide MN panel (panels 8 KB apart)
                        const uint64_t ad = p.a_mn ? tc::sdesc(a_base + k * 2048, 8192, 1024, 2)
                                                   : tc::sdesc(a_base + k * 32, 16, 1024, 2);
                        const uint64_t bd = p.b_mn ? tc::sdesc(b_base + k * 2048, 8192, 1024, 2)
                                                   : tc::sdesc(b_base + k * 32, 16, 1024, 2);
                        Op::mma_warp(d_tmem, ad, bd, idesc, (kb | k) != 0);
                    }
                    tc::mma_commit_warp(&empty[st]);
                }
                tc::mma_commit_warp(&tfull[acc]);
            }
        }
    } else {  // ---- epilogue warps 2..5
        const int q = warp & 3;
        const int row = q * 32 + lane;
        const int epi = p.epi;
        const bool hard = epi == kSwishHard || epi == kTowerHard;
        int i = 0;
        for (int u = s.first; u < s.units; u += s.stride, ++i) {
            int group, m0, m_end, n0;
            decode(p, s, u, rank, group, m0, m_end, n0);
            const int acc = i & 1;
            const uint32_t ph = (i >> 1) & 1;
            const int64_t m = (int64_t)m0 + row;
            const bool valid = m < m_end;
            const uint32_t taddr = tmem + acc * BN + ((uint32_t)(q * 32) << 16);
            tc::mbar_wait(&tfull[acc], ph);
            tc::fence_after();
            if (epi == kStore) {
#pragma unroll 1
                for (int c = 0; c < BN; c += 32) {
                    float v[32];
                    tc::tmem_ld32(taddr + c, v);
                    if (valid && n0 + c < p.N) store_row32(p, m, n0 + c, v);
                }
                tc::fence_before();
                tc::mbar_arrive(&tempty[acc]);
            } else if (epi == kResidNorm) {
                if (p.group == 128) {
#pragma unroll 1
                    for (int gc = 0; gc < BN; gc += 128)
                        if (n0 + gc < p.N) resid_norm_group<128>(p, taddr + gc, m, n0 + gc, valid);
                } else {
#pragma unroll 1
                    for (int gc = 0; gc < BN; gc += 64)
                        if (n0 + gc < p.N) resid_norm_group<64>(p, taddr + gc, m, n0 + gc, valid);
                }
                tc::fence_before();
                tc::mbar_arrive(&tempty[acc]);
            } else {  // row-wide swish_rn (+ tower heads)
                float ss = 0.0f;
#pragma unroll 1
                for (int c = 0; c < BN; c += 32) {
                    float v[32];
                    tc::tmem_ld32(taddr + c, v);
                    // columns >= N may hold another group's weights (stacked towers): mask them
#pragma unroll
                    for (int j = 0; j < 32; ++j) ss += (n0 + c + j < p.N) ? v[j] * v[j] : 0.0f;
                }
                const float total = cluster_row_sum(ss, row, lane, C, xbuf + acc * BM, &xbar[acc], ph);
                const float inv = 1.0f / sqrtf(total / (float)p.N_full + 1e-6f);
                if (epi == kSwish || epi == kSwishHard) {
#pragma unroll 1
                    for (int c = 0; c < BN; c += 32) {
                        float v[32];
                        tc::tmem_ld32(taddr + c, v);
#pragma unroll
                        for (int j = 0; j < 32; ++j) v[j] = act_swish(v[j] * inv, hard);
                        if (valid && n0 + c < p.N) store_row32(p, m, n0 + c, v);
                    }
                    tc::fence_before();
                    tc::mbar_arrive(&tempty[acc]);
                } else {  // tower: heads = W2_g . swish_rn(row)
                    float part[kMaxHeads];
#pragma unroll
                    for (int h = 0; h < kMaxHeads; ++h) part[h] = 0.0f;
                    const float* w2 = p.W2 + (size_t)group * p.heads * p.N_full;
#pragma unroll 1
                    for (int c = 0; c < BN; c += 32) {
                        float v[32];
                        tc::tmem_ld32(taddr + c, v);
                        if (n0 + c >= p.N) continue;
#pragma unroll
                        for (int j = 0; j < 32; ++j) v[j] = (n0 + c + j < p.N) ? act_swish(v[j] * inv, hard) : 0.0f;
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
                    tc::fence_before();
                    tc::mbar_arrive(&tempty[acc]);
                    // reduce head partials into cluster rank 0 (rank order), pull model: every
                    // CTA parks its partials in its own slot, each warp signals rank 0 once,
                    // rank 0 reads the peers' slots through DSMEM
                    float* hb = hbuf + (size_t)acc * p.heads * BM;
                    if (C > 1) {
#pragma unroll
                        for (int h = 0; h < kMaxHeads; ++h)
                            if (h < p.heads) hb[h * BM + row] = part[h];
                        __syncwarp();
                        if (lane == 0) tc::mbar_arrive_remote(tc::mapa(tc::smem_u32(&hbar[acc]), 0));
                    }
                    if (rank == 0) {
                        if (C > 1) {
                            tc::mbar_wait(&hbar[acc], ph);
                            tc::fence_acq_rel_cluster();
#pragma unroll
                            for (int h = 0; h < kMaxHeads; ++h) {
                                if (h < p.heads) {
                                    const uint32_t la = tc::smem_u32(&hb[h * BM + row]);
                                    float sum = 0.0f;
                                    for (int r = 0; r < C; ++r) sum += tc::ld_cluster_f32(tc::mapa(la, r));
                                    part[h] = sum;
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
    }
    tc::fence_before();
    __syncthreads();
    // peers read this CTA's exchange slots through DSMEM (pull model): nobody leaves the
    // cluster before everyone is done
    if (C > 1) tc::cluster_sync();
    if (warp == 1) tc::tmem_dealloc(tmem, 2 * BN);
}

// ---------------------------------------------------------------------------------------------
// CTA-pair variant (cta_group::2) for the plain and residual-norm epilogues: a cluster of two
// CTAs on one TPC computes a 256 x BN tile. CTA r loads A rows [m0 + 128r, +128) and B rows
// [n0 + 128r, +128) (half of the N tile) per k-block, all completions landing on the leader's
// barrier; the leader issues M = 256 MMAs that read both CTAs' operands, so each SM's smem
// supplies half of B instead of all of it (the single-CTA kernel's operand traffic is
// smem-bandwidth bound); each CTA's TMEM holds its 128 accumulator rows x BN columns and its
// epilogue warps drain them as before.
// ---------------------------------------------------------------------------------------------
template <int STAGES, typename T>
__global__ void __launch_bounds__(kThreads, 1)
    gemm2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const Params p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
    using Op = tc::Operand<T>;
    constexpr int BKE = Op::kRow;
    constexpr int A_BYTES = BM * 128;         // this CTA's 128 A rows
    constexpr int B_BYTES = (BN / 2) * 128;   // this CTA's half of the N tile
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;   // [2]
    uint64_t* tempty = tfull + 2;       // [2] (the leader's counts both CTAs' epilogue warps)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rank = (int)tc::cluster_rank();
    const int nt = (p.N + BN - 1) / BN;
    const int first = blockIdx.x / 2, stride = gridDim.x / 2;
    const int nk = (p.K + BKE - 1) / BKE;
    const bool swish = p.epi == kSwish || p.epi == kSwishHard;
    // grouped mode (swish only): M units come from a device table of 256-row tiles {group, row0,
    // row_end} over the domain segments, B rows from the group's slice of a stacked weight
    int mt2 = (p.M + 2 * BM - 1) / (2 * BM), units = 0;
    auto decode2 = [&](int u, int& m0, int& n0, int& m_end, int& group, int& mu) {
        m_end = p.M;
        group = 0;
        if (swish) {  // row-major: a row block's N-tiles are consecutive units (see the exchange)
            mu = u / nt;
            n0 = (u % nt) * BN;
            if (p.tiles) {
                const int4 t = p.tiles[mu];
                group = t.x;
                m0 = t.y;
                m_end = t.z;
            } else {
                m0 = mu * 2 * BM;
            }
            return;
        }
        // banded raster over pair M-tiles
        const int per = kRasterGroup * nt;
        const int g = u / per, in = u % per;
        const int rows = min(kRasterGroup, mt2 - g * kRasterGroup);
        mu = g * kRasterGroup + in % rows;
        m0 = mu * 2 * BM;
        n0 = (in / rows) * BN;
    };

    if (warp == 0 && lane == 0) {
        tc::tma_prefetch(&tmA);
        tc::tma_prefetch(&tmB);
        for (int i = 0; i < STAGES; ++i) {
            tc::mbar_init(&full[i], 1);
            tc::mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            tc::mbar_init(&tfull[i], 1);
            tc::mbar_init(&tempty[i], 8);  // one arrive per epilogue warp of both CTAs
        }
        tc::fence_mbar_init();
    }
    if (warp == 1) tc::tmem_alloc_cg2(tmem_slot, 2 * BN);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    tc::cluster_sync();
    const uint32_t tmem = *tmem_slot;
    // PDL: set up while the preceding kernel drains; its outputs (and the tile count) are read
    // only after this
    tc::griddep_wait();
    tc::griddep_launch_dependents();
    if (p.tiles) mt2 = *p.n_tiles;
    units = mt2 * nt;

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer (both CTAs), completions on the leader's barrier
            int g = 0;
            for (int u = first; u < units; u += stride) {
                int m0, n0, m_end, group, mu;
                decode2(u, m0, n0, m_end, group, mu);
                const int b_row0 = group * p.b_rows_per_group + n0;
                for (int kb = 0; kb < nk; ++kb, ++g) {
                    const int st = g % STAGES;
                    const uint32_t ph = (g / STAGES) & 1;
                    tc::mbar_wait(&empty[st], ph ^ 1);
                    if (rank == 0) tc::mbar_expect_tx(&full[st], 2 * (A_BYTES + B_BYTES));
                    const uint32_t bar = tc::mapa(tc::smem_u32(&full[st]), 0);
                    tc::tma_load_2d_cg2(sA + st * A_BYTES, &tmA, bar, kb * BKE, m0 + rank * BM);
                    tc::tma_load_2d_cg2(sB + st * B_BYTES, &tmB, bar, kb * BKE, b_row0 + rank * (BN / 2));
                }
            }
        }
    } else if (warp == 1) {
        if (rank == 0) {  // ---- MMA issuer: the leader's warp walks the schedule, one lane issues
            constexpr uint32_t idesc = tc::idesc_fmt(Op::kFormat, 2 * BM, BN, 0, 0);
            int g = 0, i = 0;
            for (int u = first; u < units; u += stride, ++i) {
                const int acc = i & 1;
                tc::mbar_wait(&tempty[acc], ((i >> 1) & 1) ^ 1);
                tc::fence_after();
                const uint32_t d_tmem = tmem + acc * BN;
                for (int kb = 0; kb < nk; ++kb, ++g) {
                    const int st = g % STAGES;
                    const uint32_t ph = (g / STAGES) & 1;
                    tc::mbar_wait(&full[st], ph);
                    tc::fence_after();
                    const uint32_t a_base = tc::smem_u32(sA + st * A_BYTES);
                    const uint32_t b_base = tc::smem_u32(sB + st * B_BYTES);
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint64_t ad = tc::sdesc(a_base + k * 32, 16, 1024, 2);
                        const uint64_t bd = tc::sdesc(b_base + k * 32, 16, 1024, 2);
                        tc::mma_f16_cg2_warp(d_tmem, ad, bd, idesc, (kb | k) != 0);
                    }
                    tc::mma_commit_cg2_warp(&empty[st]);
                }
                tc::mma_commit_cg2_warp(&tfull[acc]);
            }
        }
    } else {  // ---- epilogue warps 2..5 (both CTAs): this CTA's 128 accumulator rows
        const int q = warp & 3;
        const int row = q * 32 + lane;
        int i = 0;
        for (int u = first; u < units; u += stride, ++i) {
            int m0, n0, m_end, group, mu;
            decode2(u, m0, n0, m_end, group, mu);
            const int acc = i & 1;
            const uint32_t ph = (i >> 1) & 1;
            const int64_t m = (int64_t)m0 + rank * BM + row;
            const bool valid = m < m_end;
            const uint32_t taddr = tmem + acc * BN + ((uint32_t)(q * 32) << 16);
            tc::mbar_wait(&tfull[acc], ph);
            tc::fence_after();
            if (p.epi == kStore) {
#pragma unroll 1
                for (int c = 0; c < BN; c += 32) {
                    float v[32];
                    tc::tmem_ld32(taddr + c, v);
                    if (valid && n0 + c < p.N) store_row32(p, m, n0 + c, v);
                }
            } else if (swish) {
                // swish_rn over the full row (numerics.hpp:94-107): this tile's partial sum of
                // squares goes to global memory, the row block's (256 rows x all N-tiles) CTAs
                // count in per CTA half, and every row sums its N-tile partials in tile order
                // (deterministic). All CTAs are co-resident (persistent grid) and a row block's
                // tiles are consecutive units, at most one schedule round apart: no deadlock.
                float ss = 0.0f;
#pragma unroll 1
                for (int c = 0; c < BN; c += 32) {
                    float v[32];
                    tc::tmem_ld32(taddr + c, v);
#pragma unroll
                    for (int j = 0; j < 32; ++j) ss += (n0 + c + j < p.N) ? v[j] * v[j] : 0.0f;
                }
                const int nn = n0 / BN;
                if (valid) p.rowpart[m * nt + nn] = ss;
                __threadfence();
                __syncwarp();
                int* cnt = p.rowcnt + mu * 2 + rank;
                if (lane == 0) {
                    atomicAdd(cnt, 1);
                    const int want = 4 * nt;  // 4 epilogue warps per N-tile
                    int seen;
                    uint64_t t0 = 0;
                    for (uint32_t spin = 0;; ++spin) {
                        // relaxed polling (an acquire load per iteration invalidates L1 every time:
                        // CCTL.IVALL was the top stall of the 2048-wide swish GEMM); one acquire
                        // load once the count is reached orders the partial reads after it
                        asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(seen) : "l"(cnt) : "memory");
                        if (seen >= want) {
                            asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(seen) : "l"(cnt) : "memory");
                            break;
                        }
                        // bounded: a partner that never runs (co-residency lost to another workload)
                        // is reported through lattice_device_check instead of hanging the GPU
                        if ((spin & 1023u) == 1023u) {
                            const uint64_t now = globaltimer_ns();
                            if (t0 == 0) {
                                t0 = now;
                            } else if (now - t0 > kExchangeTimeoutNs) {
                                atomicAdd(&g_exchange_timeouts, 1u);
                                break;
                            }
                        }
                    }
                }
                __syncwarp();
                float total = 0.0f;
                if (valid)
                    for (int t = 0; t < nt; ++t) total += __ldcg(p.rowpart + m * nt + t);
                const float inv = 1.0f / sqrtf(total / (float)p.N_full + 1e-6f);
                const bool hard = p.epi == kSwishHard;
#pragma unroll 1
                for (int c = 0; c < BN; c += 32) {
                    float v[32];
                    tc::tmem_ld32(taddr + c, v);
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = act_swish(v[j] * inv, hard);
                    if (valid && n0 + c < p.N) store_row32(p, m, n0 + c, v);
                }
            } else if (p.group == 128) {
#pragma unroll 1
                for (int gc = 0; gc < BN; gc += 128)
                    if (n0 + gc < p.N) resid_norm_group<128>(p, taddr + gc, m, n0 + gc, valid);
            } else {
#pragma unroll 1
                for (int gc = 0; gc < BN; gc += 64)
                    if (n0 + gc < p.N) resid_norm_group<64>(p, taddr + gc, m, n0 + gc, valid);
            }
            tc::fence_before();
            __syncwarp();
            // relaxed: the TMEM reads are complete (wait::ld + fence::before_thread_sync); a release
            // would first wait for this warp's output stores to complete (MEMBAR.GPU + ERRBAR)
            if (lane == 0) tc::mbar_arrive_remote_relaxed(tc::mapa(tc::smem_u32(&tempty[acc]), 0));
        }
    }
    tc::fence_before();
    __syncthreads();
    tc::cluster_sync();  // the leader's MMAs read the peer's smem / write its TMEM until the end
    if (warp == 1) tc::tmem_dealloc_cg2(tmem, 2 * BN);
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

template <int STAGES, typename T>
lattice_status launch_t(const CUtensorMap& ta, const CUtensorMap& tb, const Params& p, int units,
                        cudaStream_t st) {
    const size_t smem = smem_bytes(BN, STAGES, p.cluster, p.heads) + kMaxCluster * BM * 4 +
                        (size_t)p.cluster * p.heads * BM * 4;  // double-buffered exchange slots
    static bool attr_done = false;
    if (!attr_done) {
        LAT_CUDA(cudaFuncSetAttribute(gemm_kernel<STAGES, T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      227 * 1024));
        LAT_CUDA(cudaFuncSetAttribute(gemm_kernel<STAGES, T>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        attr_done = true;
    }
    if (smem > 227 * 1024) return set_error(LATTICE_USAGE, "gemm: shared memory budget exceeded");
    const int C = p.cluster;
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    // persistent grid = the clusters that can be co-resident (GPC sizes limit clusters of 8 to
    // 16 per B200); a larger grid would serialise whole clusters behind the first wave
    static int max_clusters[kMaxCluster + 1] = {0};
    if (!max_clusters[C]) {
        cfg.gridDim = dim3(C * (num_sms() / C), 1, 1);
        int mc = 0;
        if (cudaOccupancyMaxActiveClusters(&mc, gemm_kernel<STAGES, T>, &cfg) != cudaSuccess || mc < 1)
            mc = num_sms() / C;
        max_clusters[C] = mc;
    }
    int clusters = max_clusters[C];
    if (clusters > units) clusters = units;
    if (clusters < 1) clusters = 1;
    cfg.gridDim = dim3(clusters * C, 1, 1);
    LAT_CUDA(cudaLaunchKernelEx(&cfg, gemm_kernel<STAGES, T>, ta, tb, p));
    return LATTICE_OK;
}
}  // namespace

constexpr int kStages2 = 6;

lattice_status launch_2cta(const CUtensorMap& ta, const CUtensorMap& tb, const Params& p, int grid_m, cudaStream_t st) {
    const size_t smem = 1024 + (size_t)kStages2 * (BM * 128 + (BN / 2) * 128) + 256;
    static bool attr_done = false;
    if (!attr_done) {
        LAT_CUDA(cudaFuncSetAttribute(gemm2_kernel<kStages2, __nv_bfloat16>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        attr_done = true;
    }
    const bool swish = p.epi == kSwish || p.epi == kSwishHard;
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[3];
    int na = 0;
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = 2;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
    if (pdl_enabled()) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    // the persistent grid: the pairs that fit on this device at once (cached per device)
    static int max_pairs[64] = {0};
    int dev = 0;
    LAT_CUDA(cudaGetDevice(&dev));
    int& mp = max_pairs[dev & 63];
    if (!mp) {
        cfg.gridDim = dim3(2 * (num_sms() / 2), 1, 1);
        int mc = 0;
        if (cudaOccupancyMaxActiveClusters(&mc, gemm2_kernel<kStages2, __nv_bfloat16>, &cfg) != cudaSuccess || mc < 1)
            mc = num_sms() / 2;
        mp = mc;
    }
    // grouped: grid_m carries the tile table's capacity (the kernel reads the live count)
    const int m_units = p.tiles ? grid_m : (p.M + 2 * BM - 1) / (2 * BM);
    const int units = m_units * ((p.N + BN - 1) / BN);
    if (swish && !p.rowcnt_zeroed) LAT_CUDA(cudaMemsetAsync(p.rowcnt, 0, sizeof(int) * 2 * m_units, st));
    int pairs = mp < units ? mp : units;
    if (pairs < 1) pairs = 1;
    // a row block's N-tiles are consecutive units handed round-robin to the pairs: each must land
    // on a different pair (or a pair would wait on its own later tile)
    if (swish && (p.N + BN - 1) / BN > pairs && units > pairs)
        return set_error(LATTICE_USAGE, "gemm: swish_rn row of " + std::to_string(p.N) +
                                            " columns needs more CTA pairs than this device runs at once");
    cfg.gridDim = dim3(2 * pairs, 1, 1);
    // The swish epilogue exchanges row statistics between pairs through global memory, so every
    // pair must be resident at once: a cooperative launch has the hardware guarantee it (or the
    // launch fails) even when other kernels share the GPU. LATTICE_GEMM_COOP=0/1 forces it off/on.
    // Nsight Compute cannot replay a cooperative cluster launch (it reports a 0x0 grid and fails),
    // so inside a profiler-injected process (the variables ncu sets for its target) the default is
    // off; the bounded wait above still turns a starved pair into a reported error, not a hang.
    static const int coop_env = [] {
        const char* e = std::getenv("LATTICE_GEMM_COOP");
        if (e) return std::atoi(e);
        const bool profiled = std::getenv("NV_NSIGHT_INJECTION_TRANSPORT_TYPE") || std::getenv("NV_TPS_LAUNCH_TOKEN") ||
                              std::getenv("CUDA_INJECTION64_PATH");
        return profiled ? 0 : 1;
    }();
    if (swish && coop_env) {
        at[na].id = cudaLaunchAttributeCooperative;
        at[na].val.cooperative = 1;
        cfg.numAttrs = na + 1;
    }
    LAT_CUDA(cudaLaunchKernelEx(&cfg, gemm2_kernel<kStages2, __nv_bfloat16>, ta, tb, p));
    return LATTICE_OK;
}

// The CTA-pair kernel serves bf16 plain / residual-norm GEMMs with at least two M-tiles;
// LATTICE_GEMM_2CTA=0 turns it off (A/B runs).
bool use_2cta(const Params& p, bool f32) {
    static int env = -1;
    if (env < 0) {
        const char* e = std::getenv("LATTICE_GEMM_2CTA");
        env = e ? std::atoi(e) : 1;
    }
    if (env == 0 || f32 || p.M < 2 * BM || p.a_mn || p.b_mn) return false;
    if (p.epi == kSwish || p.epi == kSwishHard) return p.rowpart && p.rowcnt && p.N == p.N_full;
    if (p.tiles) return false;  // grouped tiles: swish epilogue only (the towers' pre-head layer)
    return p.cluster == 1 && (p.epi == kStore || p.epi == kResidNorm);
}


lattice_status make_map_2d(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer,
                           uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer, bool f32) {
    auto fn = encode_fn();
    if (!fn) return set_error(LATTICE_CUDA, "cuTensorMapEncodeTiled unavailable");
    if ((reinterpret_cast<uintptr_t>(base) & 15) || (row_stride_bytes & 15))
        return set_error(LATTICE_USAGE, "TMA operand: base and row stride must be 16-byte aligned");
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {row_stride_bytes};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                    const_cast<void*>(base), dims, strides,
                    box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return set_error(LATTICE_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return LATTICE_OK;
}

lattice_status launch(const GemmPlan& g, cudaStream_t st) {
    if (g.two_cta) return launch_2cta(g.ta, g.tb, g.p, g.grid_y, st);
    // grid_y carries the number of M units (dense M-tiles, or the tile-table capacity)
    const int nt = (g.p.N + BN - 1) / BN;
    const int units = g.p.cluster > 1 ? g.grid_y : g.grid_y * nt;
    if (g.f32) return launch_t<4, float>(g.ta, g.tb, g.p, units, st);
    return launch_t<4, __nv_bfloat16>(g.ta, g.tb, g.p, units, st);
}

lattice_status plan(GemmPlan* g, const void* A, int64_t lda, int64_t a_rows, const void* B,
                    int64_t ldb, int64_t b_rows, const Params& p, int grid_y, bool f32) {
    const uint64_t es = f32 ? 4 : 2;
    const uint32_t bke = f32 ? 32 : 64;
    if ((p.a_mn || p.b_mn) && f32) return set_error(LATTICE_USAGE, "gemm: MN-major operands need bf16");
    // MN-major operands are stored [K][rows]: the map's inner dimension runs along M (or N)
    lattice_status s = p.a_mn ? make_map_2d(&g->ta, A, (uint64_t)a_rows, (uint64_t)p.K, (uint64_t)lda * es, 64, 64)
                              : make_map_2d(&g->ta, A, (uint64_t)p.K, (uint64_t)a_rows, (uint64_t)lda * es, bke, BM, f32);
    if (s != LATTICE_OK) return s;
    g->two_cta = use_2cta(p, f32);
    Params pp = p;
    if (g->two_cta) pp.cluster = 1;  // the pair kernel exchanges row statistics through global memory
    s = p.b_mn ? make_map_2d(&g->tb, B, (uint64_t)b_rows, (uint64_t)p.K, (uint64_t)ldb * es, 64, 64)
               : make_map_2d(&g->tb, B, (uint64_t)p.K, (uint64_t)b_rows, (uint64_t)ldb * es, bke,
                             g->two_cta ? BN / 2 : BN, f32);
    if (s != LATTICE_OK) return s;
    g->p = pp;
    g->grid_y = grid_y;
    g->stages = 4;
    g->f32 = f32;
    return LATTICE_OK;
}

}  // namespace gemm
}  // namespace lat

extern "C" lattice_status lattice_device_check(lattice_stream stream) {
    using namespace lat;
    LAT_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    unsigned int n = 0, zero = 0;
    LAT_CUDA(cudaMemcpyFromSymbol(&n, gemm::g_exchange_timeouts, sizeof(n)));
    if (n == 0) return LATTICE_OK;
    LAT_CUDA(cudaMemcpyToSymbol(gemm::g_exchange_timeouts, &zero, sizeof(zero)));
    return set_error(LATTICE_CUDA, "GEMM swish_rn row-statistics exchange timed out " + std::to_string(n) +
                                       " time(s): a CTA pair of a persistent grid was not resident (outputs of "
                                       "those launches are invalid)");
}

extern "C" lattice_status lattice_gemm(const lattice_gemm_args* a, lattice_stream stream) {
    using namespace lat;
    using namespace lat::gemm;
    LAT_REQUIRE(a != nullptr, "lattice_gemm: null args");
    LAT_REQUIRE(a->M >= 0 && a->N > 0 && a->K > 0, "lattice_gemm: bad sizes");
    LAT_REQUIRE(a->M < (1ll << 31) && a->N < (1ll << 31) && a->K < (1ll << 31), "lattice_gemm: size overflow");
    // TMA row strides are 16-byte multiples; K is a row length only for a K-major operand
    LAT_REQUIRE(a->lda % 8 == 0 && a->ldb % 8 == 0 && (a->K % 8 == 0 || (a->a_major == 1 && a->b_major == 1)),
                "lattice_gemm: lda, ldb (and K, for a K-major operand) must be multiples of 8 (16-byte TMA strides)");
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
    p.resid = a->resid;
    p.ldr = a->ldr;
    p.group = a->group;
    p.N_full = p.N;
    p.cluster = 1;
    p.heads = 0;
    p.a_mn = a->a_major == 1;
    p.b_mn = a->b_major == 1;
    LAT_REQUIRE(a->a_major >= 0 && a->a_major <= 1 && a->b_major >= 0 && a->b_major <= 1,
                "lattice_gemm: a_major / b_major must be 0 (K-major) or 1 (MN-major)");
    LAT_REQUIRE(!(p.a_mn || p.b_mn) || (a->in_dtype == LATTICE_BF16 && (!p.a_mn || a->lda >= a->M) &&
                                        (!p.b_mn || a->ldb >= a->N)),
                "lattice_gemm: MN-major operands need bf16 and a leading dimension >= M (A) / N (B)");
    if (p.epi == kSwish || p.epi == kSwishHard) {
        // the CTA-pair kernel (bf16, M >= 256) exchanges row statistics through global memory and
        // takes rows up to 16384 wide; the single-CTA kernel's DSMEM exchange stops at 2048
        p.cluster = (p.N + BN - 1) / BN;
        const bool pair = a->in_dtype == LATTICE_BF16 && a->M >= 2 * BM;
        LAT_REQUIRE(p.cluster <= (pair ? 64 : kMaxCluster),
                    pair ? "lattice_gemm: swish_rn rows wider than 16384 are not supported"
                         : "lattice_gemm: swish_rn rows wider than 2048 need bf16 and M >= 256");
    }
    if (p.epi == kResidNorm) {
        LAT_REQUIRE(a->resid && (a->group == 128 || a->group == 64) && p.N % a->group == 0 && a->ldr % 8 == 0,
                    "lattice_gemm: residual-norm epilogue needs a residual, group 64/128 dividing N");
    }
    GemmPlan g;
    LAT_REQUIRE(a->in_dtype == LATTICE_BF16 || a->in_dtype == LATTICE_F32, "lattice_gemm: in_dtype must be bf16 or f32");
    const bool f32 = a->in_dtype == LATTICE_F32;
    LAT_REQUIRE(!f32 || (a->K % 4 == 0 && a->lda % 4 == 0 && a->ldb % 4 == 0), "lattice_gemm: fp32 strides");
    void* ws = nullptr;  // swish row-statistics exchange of the CTA-pair kernel
    if (p.epi == kSwish || p.epi == kSwishHard) {
        const size_t rows = (size_t)((a->M + 2 * BM - 1) / (2 * BM)) * 2 * BM;
        LAT_CUDA(cudaMallocAsync(&ws, rows * p.cluster * sizeof(float) + rows / BM * sizeof(int) + 64, stream));
        p.rowpart = static_cast<float*>(ws);
        p.rowcnt = reinterpret_cast<int*>(static_cast<float*>(ws) + rows * p.cluster);
    }
    if ((p.a_mn || p.b_mn) && (p.epi == kSwish || p.epi == kSwishHard) && p.cluster > kMaxCluster)
        return set_error(LATTICE_USAGE, "lattice_gemm: MN-major operands run the single-CTA kernel: swish_rn rows up to 2048");
    lattice_status s = plan(&g, a->A, a->lda, a->M, a->B, a->ldb, a->N, p, (int)((a->M + BM - 1) / BM), f32);
    if (s == LATTICE_OK) s = launch(g, stream);
    if (ws) cudaFreeAsync(ws, stream);
    return s;
}
