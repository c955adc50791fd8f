// fm_lcb.cu -- K2: the per-sample interaction half of a DWFB block, fused.
//
// For every sample b with embeddings X_b [n][d] (bf16):
//   P   = bf16( X_b^T . Y )                    d x k     (FMB compression, Wukong-style)
//   F   = X_b . P                               n x k     (factorisation-machine interaction)
//   Fin = bf16( rms_norm(flatten(F)) )          n*k       -> the FMB MLP input (K3)
//   L   = W_L . X_b                             nL x d    (LCB)
//   X'_b[nF+i] = bf16( rms_norm_d(L_i + X_b[nF+i]) ), i < nL   (block combine, LCB half)
//
// X_b is read from HBM exactly once: TMA lands it in shared memory as 64-column panels with
// the 128-byte swizzle, and that one image serves three tcgen05 MMAs through different
// descriptors -- MN-major A (X^T for P), MN-major B (X for L) and K-major A (X for F).
// W_L and Y stay resident in shared memory for the whole persistent CTA. P goes TMEM ->
// registers -> bf16 -> swizzled shared memory to become F's B operand.
//
// Warp roles: 0 TMA producer, 1 MMA issuer, 2-5 LCB group (thread = TMEM lane: P row ->
// bf16 Pbuf for F's MMA, then L row + residual + rms_norm_d, no cross-warp reduction), 6-9 FM
// group (the n*k-wide norm of F with one 4-warp named barrier). The two groups run
// independently and the F MMAs of a sample overlap its LCB epilogue, so every SM
// sub-partition has two epilogue warps in flight. TMEM holds two accumulator regions
// {P | L | F}: the MMAs of sample s+1 run while sample s's epilogue drains the other region,
// and X stages are double-buffered so loads run two samples ahead. The epilogue is the
// critical path; values stay in registers between the sum-of-squares and the normalise pass.
#include <cudaTypedefs.h>

#include <string>

#include "common.cuh"
#include "fm_lcb.h"
#include "gemm_host.h"
#include "tc.cuh"

namespace lat {
namespace fm {

constexpr int kEpiWarps = 8;
constexpr int kEpiThreads = kEpiWarps * 32;
constexpr int kThreads = 64 + kEpiThreads;

__device__ __forceinline__ uint32_t swz(uint32_t row, uint32_t col_elem) {
    // byte offset of bf16 element (row, col) inside a [rows][64] SW128 panel
    return row * 128u + ((((col_elem >> 3) ^ (row & 7u)) << 4) | ((col_elem & 7u) << 1));
}

__device__ __forceinline__ int region_cols(const Params& p) {
    return 64 + p.d + ((p.n_pad + 127) / 128) * p.k_pad;
}

// 10 warps: some SM sub-partitions hold 3 of them, so 168 registers is the ceiling
__global__ void __launch_bounds__(kThreads, 1)
    fm_lcb_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmWL,
                  const __grid_constant__ CUtensorMap tmYT, const Params p) {
    extern __shared__ uint8_t smem_raw[];
    // align to 1024 B (SW128) by offsetting the __shared__ pointer itself, so the compiler keeps
    // the shared address space (LDS/STS rather than generic loads)
    uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
    const int npad = p.n_pad, kpad = p.k_pad, d = p.d;
    const int panels_d = d / 64, panels_n = (npad + 63) / 64;
    // An X stage always spans 2 panels of >= 128 rows so that every M=128 operand view
    // (F's A rows, the second MN chunk of X^T when d = 64) stays inside the allocation;
    // rows/panels beyond the loaded n_pad x d image are never consumed.
    const uint32_t xpanel = (uint32_t)(npad > 128 ? npad : 128) * 128u;
    const uint32_t xstage = xpanel * 2;
    const uint32_t xbytes = (uint32_t)npad * 128u * panels_d;  // bytes TMA actually lands
    const uint32_t wlpanel = 128u * 128u;                     // [128 rows][64] bf16
    const uint32_t ytpanel = (uint32_t)kpad * 128u;
    const uint32_t ppanel = (uint32_t)kpad * 128u;
    uint8_t* sWL = smem;
    uint8_t* sYT = sWL + wlpanel * panels_n;
    uint8_t* sP = sYT + ytpanel * panels_n;
    uint8_t* sX = sP + ((ppanel * 2 + 1023) & ~1023u);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sX + 2 * xstage);
    uint64_t* x_full = bars;        // [2] X stage landed
    uint64_t* x_empty = bars + 2;   // [2] X stage consumed (MMAs + residual reads)
    uint64_t* pl_full = bars + 4;   // [2] P, L accumulators ready (per TMEM region)
    uint64_t* f_full = bars + 6;    // [2] F accumulator ready
    uint64_t* tmem_empty = bars + 8;// [2] region drained
    uint64_t* w_full = bars + 10;
    uint64_t* pbuf_full = bars + 11;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);
    float* red_l = reinterpret_cast<float*>(bars + 16);       // [2][128] row partials
    float* red_f = red_l + 256;                               // [8] warp partials

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rcols = region_cols(p);
    const int nreg = rcols <= 256 ? 2 : 1;
    const uint32_t tcols = nreg == 2 ? 512u : (rcols <= 256 ? 256u : 512u);
    if (warp == 0 && lane == 0) {
        tc::tma_prefetch(&tmX);
        tc::tma_prefetch(&tmWL);
        tc::tma_prefetch(&tmYT);
        for (int i = 0; i < 2; ++i) {
            tc::mbar_init(&x_full[i], 1);
            tc::mbar_init(&x_empty[i], kEpiThreads);
            tc::mbar_init(&pl_full[i], 1);
            tc::mbar_init(&f_full[i], 1);
            tc::mbar_init(&tmem_empty[i], kEpiThreads);
        }
        tc::mbar_init(w_full, 1);
        tc::mbar_init(pbuf_full, 128);  // the FM group
        tc::fence_mbar_init();
    }
    if (warp == 1) tc::tmem_alloc(tmem_slot, tcols);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = *tmem_slot;
    const int m_tiles = (npad + 127) / 128;

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer
            tc::mbar_expect_tx(w_full, wlpanel * panels_n + ytpanel * panels_n);
            for (int pn = 0; pn < panels_n; ++pn) {
                tc::tma_load_2d(sWL + pn * wlpanel, &tmWL, w_full, pn * 64, 0);
                tc::tma_load_2d(sYT + pn * ytpanel, &tmYT, w_full, pn * 64, 0);
            }
            int it = 0;
            for (int64_t b = blockIdx.x; b < p.B; b += gridDim.x, ++it) {
                const int st = it & 1;
                tc::mbar_wait(&x_empty[st], ((it >> 1) & 1) ^ 1);
                tc::mbar_expect_tx(&x_full[st], xbytes);
                for (int pd = 0; pd < panels_d; ++pd)
                    tc::tma_load_3d(sX + st * xstage + pd * xpanel, &tmX, &x_full[st], pd * 64, 0, (int)b);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---- MMA issuer
            const uint32_t id_P = tc::idesc_bf16(128, kpad, 1, 0);  // A = X^T (MN-major)
            const uint32_t id_L = tc::idesc_bf16(128, d, 0, 1);     // B = X (MN-major)
            const uint32_t id_F = tc::idesc_bf16(128, kpad, 0, 0);
            tc::mbar_wait(w_full, 0);
            const uint32_t wl = tc::smem_u32(sWL), yt = tc::smem_u32(sYT), pb = tc::smem_u32(sP);
            int it = 0;
            for (int64_t b = blockIdx.x; b < p.B; b += gridDim.x, ++it) {
                const int st = it & 1;
                const int rg = nreg == 2 ? (it & 1) : 0;
                const uint32_t rph = nreg == 2 ? ((it >> 1) & 1) : (it & 1);
                const uint32_t t_P = tmem + rg * 256, t_L = t_P + 64, t_F = t_L + d;
                tc::mbar_wait(&x_full[st], (it >> 1) & 1);
                tc::mbar_wait(&tmem_empty[rg], rph ^ 1);
                tc::fence_after();
                const uint32_t xs = tc::smem_u32(sX + st * xstage);
                for (int kk = 0; kk < npad / 16; ++kk) {
                    const int k16 = kk * 16;
                    const uint32_t kb_off = (uint32_t)(k16 / 64), kin = (uint32_t)(k16 % 64) * 2;
                    // P += X^T[:, k16:k16+16] . Y[k16:k16+16, :]
                    const uint64_t a_xt = tc::sdesc(xs + k16 * 128, xpanel, 1024, 2);
                    const uint64_t b_y = tc::sdesc(yt + kb_off * ytpanel + kin, 16, 1024, 2);
                    tc::mma_f16(t_P, a_xt, b_y, id_P, kk != 0);
                    // L += W_L[:, k16:k16+16] . X[k16:k16+16, :]
                    const uint64_t a_wl = tc::sdesc(wl + kb_off * wlpanel + kin, 16, 1024, 2);
                    const uint64_t b_x = tc::sdesc(xs + k16 * 128, xpanel, 1024, 2);
                    tc::mma_f16(t_L, a_wl, b_x, id_L, kk != 0);
                }
                tc::mma_commit(&pl_full[rg]);
                tc::mbar_wait(pbuf_full, it & 1);
                tc::fence_after();
                const uint32_t pbs = pb;
                for (int mt = 0; mt < m_tiles; ++mt) {
                    for (int kk = 0; kk < d / 16; ++kk) {
                        const int k16 = kk * 16;
                        const uint32_t pan = (uint32_t)(k16 / 64), kin = (uint32_t)(k16 % 64) * 2;
                        const uint64_t a_x = tc::sdesc(xs + pan * xpanel + mt * 16384 + kin, 16, 1024, 2);
                        const uint64_t b_p = tc::sdesc(pbs + pan * ppanel + kin, 16, 1024, 2);
                        tc::mma_f16(t_F + mt * kpad, a_x, b_p, id_F, kk != 0);
                    }
                }
                tc::mma_commit(&f_full[rg]);
            }
        }
    } else if (warp < 6) {  // ---- LCB group, warps 2..5: thread = L row, all d columns
        const int q = warp & 3;
        const int row = q * 32 + lane;
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const float inv_d = 1.0f / (float)d;
        const int xr = p.nF + row;
        const bool live = row < p.nL;
        int it = 0;
        for (int64_t b = blockIdx.x; b < p.B; b += gridDim.x, ++it) {
            const int st = it & 1;
            const int rg = nreg == 2 ? (it & 1) : 0;
            const uint32_t rph = nreg == 2 ? ((it >> 1) & 1) : (it & 1);
            const uint32_t t_L = tmem + rg * 256 + lane_off + 64;
            const uint8_t* xs = sX + st * xstage;
            // pick up the residual row X[nF+row] as soon as the stage lands, so the stage can
            // be recycled right after the MMAs (the producer runs two samples ahead)
            tc::mbar_wait(&x_full[st], (it >> 1) & 1);
            uint4 res[16];
#pragma unroll
            for (int j = 0; j < 16; ++j)
                res[j] = (live && j * 8 < d) ? *reinterpret_cast<const uint4*>(xs + (j / 8) * xpanel + swz(xr, (j * 8) & 63))
                                             : make_uint4(0, 0, 0, 0);
            tc::mbar_arrive(&x_empty[st]);
            tc::mbar_wait(&pl_full[rg], rph);
            tc::fence_after();
            // P row `row` (= d index, same TMEM lane as this thread's L row) -> bf16 ->
            // Pbuf[j][row], the K-major B operand of F. One Pbuf suffices: pl_full of this
            // sample completes after the previous sample's F MMAs (same issuing thread).
            {
                const uint32_t t_P = tmem + rg * 256 + lane_off;
                for (int c0 = 0; c0 < kpad; c0 += 16) {
                    float pv[16];
                    tc::tmem_ld16(t_P + c0, pv);
                    if (row < d) {
                        uint8_t* pan = sP + (row / 64) * ppanel;
#pragma unroll
                        for (int j = 0; j < 16; ++j)
                            *reinterpret_cast<__nv_bfloat16*>(pan + swz(c0 + j, row & 63)) = __float2bfloat16_rn(pv[j]);
                    }
                }
                tc::fence_async_shared();
                tc::mbar_arrive(pbuf_full);
            }
            // X'[nF+row] = rms_norm_d(L[row] + X[nF+row]): two passes over TMEM (sum of squares,
            // then normalise + store) so only the packed residual stays live in registers
            float ss = 0.0f;
#pragma unroll
            for (int c = 0; c < 128; c += 32) {
                if (c < d) {
                    float v[32];
                    tc::tmem_ld32(t_L + c, v);
#pragma unroll
                    for (int j = 0; j < 32; j += 8) {
                        const uint4 r = res[(c + j) / 8];
                        const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const float a = v[j + 2 * i] + bf16_lo(w[i]), bb = v[j + 2 * i + 1] + bf16_hi(w[i]);
                            ss += a * a + bb * bb;
                        }
                    }
                }
            }
            const float inv = 1.0f / sqrtf(ss * inv_d + 1e-6f);
            __nv_bfloat16* dst = p.Xout + (b * p.n + xr) * (int64_t)d;
#pragma unroll
            for (int c = 0; c < 128; c += 32) {
                if (c < d) {
                    float v[32];
                    tc::tmem_ld32(t_L + c, v);
#pragma unroll
                    for (int j = 0; j < 32; j += 8) {
                        const uint4 r = res[(c + j) / 8];
                        const uint32_t w[4] = {r.x, r.y, r.z, r.w};
                        uint32_t o[4];
#pragma unroll
                        for (int i = 0; i < 4; ++i)
                            o[i] = pack_bf16x2((v[j + 2 * i] + bf16_lo(w[i])) * inv, (v[j + 2 * i + 1] + bf16_hi(w[i])) * inv);
                        if (live) *reinterpret_cast<uint4*>(dst + c + j) = make_uint4(o[0], o[1], o[2], o[3]);
                    }
                }
            }
            tc::fence_before();
            tc::mbar_arrive(&tmem_empty[rg]);
        }
    } else {  // ---- FM group, warps 6..9: P -> Pbuf, then Fin = rms_norm(flatten(X P))
        const int q = warp & 3;
        const int e = warp - 6;
        const int row = q * 32 + lane;
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const float inv_nk = 1.0f / (float)(p.n * p.k);
        int it = 0;
        for (int64_t b = blockIdx.x; b < p.B; b += gridDim.x, ++it) {
            const int st = it & 1;
            const int rg = nreg == 2 ? (it & 1) : 0;
            const uint32_t rph = nreg == 2 ? ((it >> 1) & 1) : (it & 1);
            const uint32_t t_F = tmem + rg * 256 + lane_off + 64 + d;
            tc::mbar_wait(&f_full[rg], rph);
            tc::fence_after();
            tc::mbar_arrive(&x_empty[st]);  // every MMA reading this X stage has completed
            float v[2][64];
            float ss = 0.0f;
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
                if (mt < m_tiles) {
                    tc::tmem_ld32(t_F + mt * kpad, v[mt]);
                    if (kpad > 32) tc::tmem_ld32(t_F + mt * kpad + 32, v[mt] + 32);
                    if (mt * 128 + row < p.n) {
#pragma unroll
                        for (int j = 0; j < 64; ++j)
                            if (j < p.k) ss += v[mt][j] * v[mt][j];
                    }
                }
            }
            tc::fence_before();
            tc::mbar_arrive(&tmem_empty[rg]);
            ss = warp_sum(ss);
            float* red = red_f + (it & 1) * 4;  // parity-buffered: no reuse race across samples
            if (lane == 0) red[e] = ss;
            tc::named_bar(2, 128);
            const float inv = 1.0f / sqrtf((red[0] + red[1] + red[2] + red[3]) * inv_nk + 1e-6f);
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
                const int r = mt * 128 + row;
                if (mt < m_tiles && r < p.n) {
                    __nv_bfloat16* dst = p.Fout + b * (int64_t)p.n * p.k + (int64_t)r * p.k;
                    if ((p.k & 7) == 0) {
#pragma unroll
                        for (int j = 0; j < 64; j += 8)
                            if (j < p.k)
                                *reinterpret_cast<uint4*>(dst + j) = make_uint4(
                                    pack_bf16x2(v[mt][j] * inv, v[mt][j + 1] * inv), pack_bf16x2(v[mt][j + 2] * inv, v[mt][j + 3] * inv),
                                    pack_bf16x2(v[mt][j + 4] * inv, v[mt][j + 5] * inv), pack_bf16x2(v[mt][j + 6] * inv, v[mt][j + 7] * inv));
                    } else {
#pragma unroll
                        for (int j = 0; j < 64; ++j)
                            if (j < p.k) dst[j] = __float2bfloat16_rn(v[mt][j] * inv);
                    }
                }
            }
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc(tmem, tcols);
}

size_t smem_bytes(const Params& p) {
    const int panels_n = (p.n_pad + 63) / 64;
    size_t s = 1024;
    s += (size_t)128 * 128 * panels_n;                      // W_L
    s += (size_t)p.k_pad * 128 * panels_n;                  // Y^T
    s += ((size_t)p.k_pad * 128 * 2 + 1023) & ~size_t(1023);  // P (2 panels)
    s += 2 * 2 * (size_t)(p.n_pad > 128 ? p.n_pad : 128) * 128;  // X stages (2 panels each)
    s += 128 + 2 * 128 * 4 + 8 * 4 + 64;                    // barriers + reductions
    return s;
}

lattice_status check(const Params& p) {
    if (!(p.d == 64 || p.d == 128)) return set_error(LATTICE_USAGE, "fm_lcb: d must be 64 or 128");
    if (p.n < 1 || p.n_pad > 256 || p.n_pad % 16 || p.n_pad < p.n)
        return set_error(LATTICE_USAGE, "fm_lcb: n must be <= 256");
    if (p.k < 1 || p.k_pad > 64 || p.k_pad % 16 || p.k_pad < p.k)
        return set_error(LATTICE_USAGE, "fm_lcb: k must be <= 64");
    if (p.nL < 0 || p.nL > 128 || p.nF + p.nL != p.n)
        return set_error(LATTICE_USAGE, "fm_lcb: nL must be <= 128 and nF + nL == n");
    if (64 + p.d + ((p.n_pad + 127) / 128) * p.k_pad > 512)
        return set_error(LATTICE_USAGE, "fm_lcb: accumulators exceed TMEM");
    if (smem_bytes(p) > 227 * 1024) return set_error(LATTICE_USAGE, "fm_lcb: shared memory budget exceeded");
    return LATTICE_OK;
}

lattice_status make_maps(Plan* pl, const void* X, const void* WLpad, const void* YTpad) {
    const Params& p = pl->p;
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return set_error(LATTICE_CUDA, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }
    cuuint64_t dims[3] = {(cuuint64_t)p.d, (cuuint64_t)p.n, (cuuint64_t)p.B};
    cuuint64_t strides[2] = {(cuuint64_t)p.d * 2, (cuuint64_t)p.n * p.d * 2};
    cuuint32_t box[3] = {64, (cuuint32_t)p.n_pad, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = fn(&pl->tmX, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(X), dims, strides,
                    box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_error(LATTICE_CUDA, "fm_lcb: X tensor map (" + std::to_string((int)r) + ")");
    lattice_status s = gemm::make_map_2d(&pl->tmWL, WLpad, (uint64_t)p.n_pad, 128, (uint64_t)p.n_pad * 2, 64, 128);
    if (s != LATTICE_OK) return s;
    return gemm::make_map_2d(&pl->tmYT, YTpad, (uint64_t)p.n_pad, (uint64_t)p.k_pad, (uint64_t)p.n_pad * 2, 64,
                             (uint32_t)p.k_pad);
}

lattice_status launch(const Plan& pl, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        LAT_CUDA(cudaFuncSetAttribute(fm_lcb_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        attr = true;
    }
    const int grid = (int)(pl.p.B < num_sms() ? pl.p.B : num_sms());
    if (grid <= 0) return LATTICE_OK;
    fm_lcb_kernel<<<grid, kThreads, smem_bytes(pl.p), st>>>(pl.tmX, pl.tmWL, pl.tmYT, pl.p);
    LAT_CUDA(cudaGetLastError());
    return LATTICE_OK;
}

}  // namespace fm
}  // namespace lat
