// fm_lcb.cu -- K2: the per-sample interaction half of a DWFB block, fused.
//
// For every sample b with embeddings X_b [n][d]:
//   P   = q( X_b^T . Y )                       d x k     (FMB compression, Wukong-style)
//   F   = X_b . P                               n x k     (factorisation-machine interaction)
//   Fin = q( rms_norm(flatten(F)) )             n*k       -> the FMB MLP input (K3)
//   L   = W_L . X_b                             nL x d    (LCB)
//   X'_b[nF+i] = q( rms_norm_d(L_i + X_b[nF+i]) ), i < nL   (block combine, LCB half)
// q() = round to the storage dtype: bf16 (kind::f16 MMAs) or fp32 (kind::tf32 MMAs).
//
// X_b is read from HBM exactly once: TMA lands it in shared memory as 128-byte-wide panels with
// the 128-byte swizzle, and that one image serves three tcgen05 MMAs through different
// descriptors -- MN-major A (X^T for P), MN-major B (X for L) and K-major A (X for F).
// W_L and Y stay resident in shared memory for the whole persistent CTA. P goes TMEM ->
// registers -> storage dtype -> swizzled shared memory to become F's B operand.
//
// Warp roles: 0 TMA producer, 1 MMA issuer, 2-5 LCB group (thread = TMEM lane: P row ->
// Pbuf for F's MMA, then L row + residual + rms_norm_d, no cross-warp reduction), 6-9 FM
// group (the n*k-wide norm of F with one 4-warp named barrier). The two groups run
// independently and the F MMAs of a sample overlap its LCB epilogue, so every SM
// sub-partition has two epilogue warps in flight. TMEM holds two accumulator regions
// {P | L | F}: the MMAs of sample s+1 run while sample s's epilogue drains the other region,
// and X stages are double-buffered; the LCB group picks up its residual rows as soon as a
// stage lands so the stage is recycled right after the MMAs.
#include <cudaTypedefs.h>

#include <cstdio>
#include <string>
#include <vector>

#include "common.cuh"
#include "fm_lcb.h"
#include "gemm_host.h"
#include "tc.cuh"

namespace lat {
namespace fm {

// resident variant: 8 LCB warps (a warp pair per TMEM lane quarter, half of the d columns
// each) + 4 FM warps, so the latency-bound LCB epilogue has two warps per sub-partition
constexpr int kLcbWarps = 8;
constexpr int kResEpiThreads = (kLcbWarps + 4) * 32;
constexpr int kResThreads = 64 + kResEpiThreads;

// byte offset of element (row, col) inside a [rows][128 B] SW128 panel, element size ES
template <int ES>
__device__ __forceinline__ uint32_t swz(uint32_t row, uint32_t col) {
    const uint32_t byte = col * ES;
    return row * 128u + ((((byte >> 4) ^ (row & 7u)) << 4) | (byte & 15u));
}

template <typename T>
struct Store;
template <>
struct Store<__nv_bfloat16> {
    // 8 consecutive values -> one 16-byte store
    __device__ static void row8(__nv_bfloat16* dst, const float* v) {
        *reinterpret_cast<uint4*>(dst) = make_uint4(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]),
                                                    pack_bf16x2(v[4], v[5]), pack_bf16x2(v[6], v[7]));
    }
    // 16 consecutive values -> one 32-byte store when aligned (a whole L2 sector per lane)
    __device__ static void row16(__nv_bfloat16* dst, const float* v) {
        const uint4 a = make_uint4(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]), pack_bf16x2(v[4], v[5]),
                                   pack_bf16x2(v[6], v[7]));
        const uint4 b = make_uint4(pack_bf16x2(v[8], v[9]), pack_bf16x2(v[10], v[11]), pack_bf16x2(v[12], v[13]),
                                   pack_bf16x2(v[14], v[15]));
        if (aligned32(dst)) {
            st_global_256(dst, a, b);
        } else {
            reinterpret_cast<uint4*>(dst)[0] = a;
            reinterpret_cast<uint4*>(dst)[1] = b;
        }
    }
    __device__ static void one(__nv_bfloat16* dst, float v) { *dst = __float2bfloat16_rn(v); }
    // unpack 8 residual values starting at element e of a packed row held in uint4 res[]
    __device__ static void unpack8(const uint4* res, int e, float* out) {
        const uint4 r = res[e / 8];
        const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            out[2 * i] = bf16_lo(w[i]);
            out[2 * i + 1] = bf16_hi(w[i]);
        }
    }
};
template <>
struct Store<float> {
    __device__ static void row8(float* dst, const float* v) {
        reinterpret_cast<float4*>(dst)[0] = make_float4(v[0], v[1], v[2], v[3]);
        reinterpret_cast<float4*>(dst)[1] = make_float4(v[4], v[5], v[6], v[7]);
    }
    __device__ static void row16(float* dst, const float* v) {
        row8(dst, v);
        row8(dst + 8, v + 8);
    }
    __device__ static void one(float* dst, float v) { *dst = v; }
    __device__ static void unpack8(const uint4* res, int e, float* out) {
        const uint4 a = res[e / 4], b = res[e / 4 + 1];
        out[0] = __uint_as_float(a.x), out[1] = __uint_as_float(a.y), out[2] = __uint_as_float(a.z);
        out[3] = __uint_as_float(a.w), out[4] = __uint_as_float(b.x), out[5] = __uint_as_float(b.y);
        out[6] = __uint_as_float(b.z), out[7] = __uint_as_float(b.w);
    }
};

__host__ __device__ inline int region_cols(const Params& p) {
    return 64 + p.d + ((p.n_pad + 127) / 128) * p.k_pad;
}

// smem geometry shared by host (budget) and device (carving)
struct Geo {
    int EP, panels_d, panels_n, x_chunks;
    uint32_t xpanel, xstage, wlpanel, ytpanel, ppanel, pbytes, xtbytes;
    __host__ __device__ Geo(const Params& p, int es) {
        EP = 128 / es;                              // elements per 128-byte row
        panels_d = p.d / EP;
        panels_n = (p.n_pad + EP - 1) / EP;
        // an X stage spans the 128/EP chunks an M=128 MN-major view of X^T reads, each of
        // >= 128 rows (F's A rows), so every operand view stays inside the allocation;
        // rows/panels beyond the loaded n_pad x d image are never consumed
        x_chunks = 128 / EP > panels_d ? 128 / EP : panels_d;
        xpanel = (uint32_t)(p.n_pad > 128 ? p.n_pad : 128) * 128u;
        xstage = xpanel * x_chunks;
        wlpanel = 128u * 128u;
        ytpanel = (uint32_t)p.k_pad * 128u;
        ppanel = (uint32_t)p.k_pad * 128u;
        pbytes = (ppanel * panels_d + 1023u) & ~1023u;
        // fp32 only: K-major X^T [128 rows (d, padded)][n_pad] for P's A and L's B operands.
        // tcgen05 reads MN-major 32-bit operands only in the 32-byte-atom swizzle, which the
        // K-major view F needs cannot share, so fp32 keeps a transposed copy instead.
        xtbytes = es == 4 ? 128u * 128u * (uint32_t)panels_n : 0u;
    }
};

// 14 warps: 146 registers per thread is the ceiling
template <typename T>
__global__ void __launch_bounds__(kResThreads, 1)
    fm_lcb_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmWL,
                  const __grid_constant__ CUtensorMap tmYT, const Params p) {
    using Op = tc::Operand<T>;
    constexpr int ES = Op::kBytes, KK = Op::kK;
    extern __shared__ uint8_t smem_raw[];
    // align to 1024 B (SW128) by offsetting the __shared__ pointer itself, so the compiler keeps
    // the shared address space (LDS/STS rather than generic loads)
    uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
    const int npad = p.n_pad, kpad = p.k_pad, d = p.d;
    const Geo g(p, ES);
    const int EP = g.EP;
    const uint32_t xbytes = (uint32_t)npad * 128u * g.panels_d;  // bytes TMA actually lands
    uint8_t* sWL = smem;
    uint8_t* sYT = sWL + g.wlpanel * g.panels_n;
    uint8_t* sP = sYT + g.ytpanel * g.panels_n;
    uint8_t* sXT = sP + g.pbytes;
    uint8_t* sX = sXT + g.xtbytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sX + 2 * g.xstage);
    uint64_t* x_full = bars;        // [2] X stage landed
    uint64_t* x_empty = bars + 2;   // [2] X stage consumed (MMAs + residual reads)
    uint64_t* pl_full = bars + 4;   // [2] P, L accumulators ready (per TMEM region)
    uint64_t* f_full = bars + 6;    // [2] F accumulator ready
    uint64_t* tmem_empty = bars + 8;// [2] region drained
    uint64_t* w_full = bars + 10;
    uint64_t* pbuf_full = bars + 11;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);
    uint64_t* xt_full = bars + 13;  // fp32: X^T copy written (LCB group)
    float* red_f = reinterpret_cast<float*>(bars + 16);  // [2][4] FM-group warp partials
    float* lcb_ss = reinterpret_cast<float*>(bars + 20);  // [2 parity][2 halves][128 rows] LCB partials

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
            tc::mbar_init(&x_empty[i], kResEpiThreads);
            tc::mbar_init(&pl_full[i], 1);
            tc::mbar_init(&f_full[i], 1);
            tc::mbar_init(&tmem_empty[i], kResEpiThreads);
        }
        tc::mbar_init(w_full, 1);
        tc::mbar_init(pbuf_full, kLcbWarps * 32);  // the LCB group
        tc::mbar_init(xt_full, kLcbWarps * 32);    // the LCB group (fp32 only)
        tc::fence_mbar_init();
    }
    if (warp == 1) tc::tmem_alloc(tmem_slot, tcols);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = *tmem_slot;
    const int m_tiles = (npad + 127) / 128;
    // PDL: barriers, TMEM and the resident weights are set up while the preceding kernel drains;
    // X, Fout and Xout are touched only after griddep_wait
    if (!(warp == 0 && lane == 0)) tc::griddep_wait();
    tc::griddep_launch_dependents();

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer
            tc::mbar_expect_tx(w_full, (g.wlpanel + g.ytpanel) * g.panels_n);
            for (int pn = 0; pn < g.panels_n; ++pn) {
                tc::tma_load_2d(sWL + pn * g.wlpanel, &tmWL, w_full, pn * EP, 0);
                tc::tma_load_2d(sYT + pn * g.ytpanel, &tmYT, w_full, pn * EP, 0);
            }
            tc::griddep_wait();
            int it = 0;
            for (int64_t b = blockIdx.x; b < p.B; b += gridDim.x, ++it) {
                const int st = it & 1;
                tc::mbar_wait(&x_empty[st], ((it >> 1) & 1) ^ 1);
                tc::mbar_expect_tx(&x_full[st], xbytes);
                for (int pd = 0; pd < g.panels_d; ++pd)
                    tc::tma_load_3d(sX + st * g.xstage + pd * g.xpanel, &tmX, &x_full[st], pd * EP, 0, (int)b);
            }
        }
    } else if (warp == 1) {
        {  // ---- MMA issuer: the whole warp walks the schedule, one elected lane issues (tc.cuh)
            // bf16: A = X^T and B = X read MN-major from the X image; fp32: K-major X^T copy
            constexpr int mn = ES == 2 ? 1 : 0;
            const uint32_t id_P = tc::idesc_fmt(Op::kFormat, 128, kpad, mn, 0);
            const uint32_t id_L = tc::idesc_fmt(Op::kFormat, 128, d, 0, mn);
            const uint32_t id_F = tc::idesc_fmt(Op::kFormat, 128, kpad, 0, 0);
            tc::mbar_wait(w_full, 0);
            const uint32_t wl = tc::smem_u32(sWL), yt = tc::smem_u32(sYT), pb = tc::smem_u32(sP);
            const uint32_t xt = tc::smem_u32(sXT);
            int it = 0;
            for (int64_t b = blockIdx.x; b < p.B; b += gridDim.x, ++it) {
                const int st = it & 1;
                const int rg = nreg == 2 ? (it & 1) : 0;
                const uint32_t rph = nreg == 2 ? ((it >> 1) & 1) : (it & 1);
                const uint32_t t_P = tmem + rg * 256, t_L = t_P + 64, t_F = t_L + d;
                tc::mbar_wait(&x_full[st], (it >> 1) & 1);
                if (ES == 4) tc::mbar_wait(xt_full, it & 1);
                tc::mbar_wait(&tmem_empty[rg], rph ^ 1);
                tc::fence_after();
                const uint32_t xs = tc::smem_u32(sX + st * g.xstage);
                for (int kk = 0; kk < npad / KK; ++kk) {
                    const int k0 = kk * KK;  // n rows k0 .. k0+KK
                    const uint32_t kp = (uint32_t)(k0 / EP), kin = (uint32_t)(k0 % EP) * ES;
                    // X^T[:, k0:k0+KK] (A of P) and X[k0:k0+KK, :] (B of L): the same operand
                    const uint64_t x_op = ES == 2 ? tc::sdesc(xs + k0 * 128, g.xpanel, 1024, 2)
                                                  : tc::sdesc(xt + kp * 16384 + kin, 16, 1024, 2);
                    // P += X^T[:, k0:k0+KK] . Y[k0:k0+KK, :]
                    const uint64_t b_y = tc::sdesc(yt + kp * g.ytpanel + kin, 16, 1024, 2);
                    Op::mma_warp(t_P, x_op, b_y, id_P, kk != 0);
                    // L += W_L[:, k0:k0+KK] . X[k0:k0+KK, :]
                    const uint64_t a_wl = tc::sdesc(wl + kp * g.wlpanel + kin, 16, 1024, 2);
                    Op::mma_warp(t_L, a_wl, x_op, id_L, kk != 0);
                }
                tc::mma_commit_warp(&pl_full[rg]);
                tc::mbar_wait(pbuf_full, it & 1);
                tc::fence_after();
                for (int mt = 0; mt < m_tiles; ++mt) {
                    for (int kk = 0; kk < d / KK; ++kk) {
                        const int k0 = kk * KK;  // d columns k0 .. k0+KK
                        const uint32_t pan = (uint32_t)(k0 / EP), kin = (uint32_t)(k0 % EP) * ES;
                        const uint64_t a_x = tc::sdesc(xs + pan * g.xpanel + mt * 16384 + kin, 16, 1024, 2);
                        const uint64_t b_p = tc::sdesc(pb + pan * g.ppanel + kin, 16, 1024, 2);
                        Op::mma_warp(t_F + mt * kpad, a_x, b_p, id_F, kk != 0);
                    }
                }
                tc::mma_commit_warp(&f_full[rg]);
            }
        }
    } else if (warp < 2 + kLcbWarps) {  // ---- LCB group, warps 2..9: thread = TMEM lane
        // warps w and w+4 share TMEM lane quarter q; warp half h owns d columns [h*d/2, (h+1)*d/2)
        const int q = warp & 3;
        const int h = (warp - 2) >> 2;
        const int row = q * 32 + lane;
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const float inv_d = 1.0f / (float)d;
        const int xr = p.nF + row;
        const bool live = row < p.nL;
        const int hd = d / 2, c_lo = h * hd;
        const int res_vec = hd * ES / 16;  // 16-byte vectors in one half residual row (<= 8)
        int it = 0;
        for (int64_t b = blockIdx.x; b < p.B; b += gridDim.x, ++it) {
            const int st = it & 1;
            const int rg = nreg == 2 ? (it & 1) : 0;
            const uint32_t rph = nreg == 2 ? ((it >> 1) & 1) : (it & 1);
            const uint32_t t_L = tmem + rg * 256 + lane_off + 64;
            const uint8_t* xs = sX + st * g.xstage;
            // pick up this half of the residual row X[nF+row] as soon as the stage lands, so
            // the stage can be recycled right after the MMAs (the producer runs two samples ahead)
            tc::mbar_wait(&x_full[st], (it >> 1) & 1);
            uint4 res[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int e = c_lo + j * (16 / ES);  // first element of vector j
                res[j] = (live && j < res_vec)
                             ? *reinterpret_cast<const uint4*>(xs + (e / EP) * g.xpanel + swz<ES>(xr, e % EP))
                             : make_uint4(0, 0, 0, 0);
            }
            if (ES == 4) {
                // fp32: X^T[c][i] = X[i][c] into the K-major copy (its previous contents were
                // consumed by the previous sample's P/L MMAs, whose pl_full this thread saw)
                const int total = d * npad;
                for (int idx = h * 128 + row; idx < total; idx += kLcbWarps * 32) {
                    const int c = idx / npad, i = idx - c * npad;
                    const float x = *reinterpret_cast<const float*>(xs + (c / EP) * g.xpanel + swz<ES>(i, c % EP));
                    *reinterpret_cast<float*>(sXT + (i / EP) * 16384 + swz<ES>(c, i % EP)) = x;
                }
                tc::fence_async_shared();
                tc::mbar_arrive(xt_full);
            }
            tc::mbar_arrive(&x_empty[st]);
            tc::mbar_wait(&pl_full[rg], rph);
            tc::fence_after();
            // P row `row` (= d index, same TMEM lane as this thread's L row) -> storage dtype ->
            // Pbuf[j][row], the K-major B operand of F; the two halves stage alternate 16-column
            // chunks. One Pbuf suffices: pl_full of this sample completes after the previous
            // sample's F MMAs (same issuing thread).
            {
                const uint32_t t_P = tmem + rg * 256 + lane_off;
                for (int c0 = 16 * h; c0 < kpad; c0 += 32) {
                    float pv[16];
                    tc::tmem_ld16(t_P + c0, pv);
                    if (row < d) {
                        uint8_t* pan = sP + (row / EP) * g.ppanel;
#pragma unroll
                        for (int j = 0; j < 16; ++j)
                            Store<T>::one(reinterpret_cast<T*>(pan + swz<ES>(c0 + j, row % EP)), pv[j]);
                    }
                }
                tc::fence_async_shared();
                tc::mbar_arrive(pbuf_full);
            }
            // X'[nF+row] = rms_norm_d(L[row] + X[nF+row]): two passes over this half's TMEM
            // columns (sum of squares, then normalise + store); the two halves' sums of squares
            // meet in shared memory (parity-buffered by sample) behind one 256-thread barrier
            float ss8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // 8 independent FMA chains
#pragma unroll
            for (int c = 0; c < 64; c += 32) {
                if (c < hd) {
                    float v[32];
                    tc::tmem_ld32(t_L + c_lo + c, v);
#pragma unroll
                    for (int j = 0; j < 32; j += 8) {
                        float r8[8];
                        Store<T>::unpack8(res, c + j, r8);
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const float a = v[j + i] + r8[i];
                            ss8[i] = fmaf(a, a, ss8[i]);
                        }
                    }
                }
            }
            float* xss = lcb_ss + (it & 1) * 256;
            xss[h * 128 + row] = ((ss8[0] + ss8[1]) + (ss8[2] + ss8[3])) + ((ss8[4] + ss8[5]) + (ss8[6] + ss8[7]));
            tc::named_bar(3, kLcbWarps * 32);
            const float ss = xss[row] + xss[128 + row];  // same order in both halves
            const float inv = 1.0f / sqrtf(ss * inv_d + 1e-6f);
            T* dst = static_cast<T*>(p.Xout) + (b * p.n + xr) * (int64_t)d + c_lo;
#pragma unroll
            for (int c = 0; c < 64; c += 32) {
                if (c < hd) {
                    float v[32];
                    tc::tmem_ld32(t_L + c_lo + c, v);
#pragma unroll
                    for (int j = 0; j < 32; j += 16) {  // 16 values: one 32-byte store (bf16)
                        float r16[16];
                        Store<T>::unpack8(res, c + j, r16);
                        Store<T>::unpack8(res, c + j + 8, r16 + 8);
#pragma unroll
                        for (int i = 0; i < 16; ++i) r16[i] = (v[j + i] + r16[i]) * inv;
                        if (live) Store<T>::row16(dst + c + j, r16);
                    }
                }
            }
            tc::fence_before();
            tc::mbar_arrive(&tmem_empty[rg]);
        }
    } else {  // ---- FM group, warps 10..13: Fin = rms_norm(flatten(X P))
        const int q = warp & 3;
        const int e = warp - 2 - kLcbWarps;
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
            // k <= 32: the F rows stay in registers and the region is released before the
            // stores; k in (32, 64]: the second pass re-reads TMEM (register budget), so the
            // region is released after it
            const bool small_k = kpad <= 32;
            float v[2][32];
            float ss4[4] = {0.f, 0.f, 0.f, 0.f};  // 4 independent FMA chains
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
                if (mt < m_tiles) {
                    for (int c0 = 0; c0 < kpad; c0 += 32) {
                        tc::tmem_ld32(t_F + mt * kpad + c0, v[mt]);
                        if (mt * 128 + row < p.n) {
#pragma unroll
                            for (int j = 0; j < 32; ++j)
                                if (c0 + j < p.k) ss4[j & 3] = fmaf(v[mt][j], v[mt][j], ss4[j & 3]);
                        }
                    }
                }
            }
            float ss = (ss4[0] + ss4[1]) + (ss4[2] + ss4[3]);
            if (small_k) {
                tc::fence_before();
                tc::mbar_arrive(&tmem_empty[rg]);
            }
            ss = warp_sum(ss);
            float* red = red_f + (it & 1) * 4;  // parity-buffered: no reuse race across samples
            if (lane == 0) red[e] = ss;
            tc::named_bar(2, 128);
            const float inv = 1.0f / sqrtf((red[0] + red[1] + red[2] + red[3]) * inv_nk + 1e-6f);
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
                const int r = mt * 128 + row;
                if (mt < m_tiles) {
                    for (int c0 = 0; c0 < kpad; c0 += 32) {
                        if (!small_k) tc::tmem_ld32(t_F + mt * kpad + c0, v[mt]);
                        if (r >= p.n) continue;
                        T* dst = static_cast<T*>(p.Fout) + b * (int64_t)p.n * p.k + (int64_t)r * p.k + c0;
                        if ((p.k & 15) == 0) {
#pragma unroll
                            for (int j = 0; j < 32; j += 16) {
                                if (c0 + j < p.k) {
                                    float o[16];
#pragma unroll
                                    for (int i = 0; i < 16; ++i) o[i] = v[mt][j + i] * inv;
                                    Store<T>::row16(dst + j, o);
                                }
                            }
                        } else if ((p.k & 7) == 0) {
#pragma unroll
                            for (int j = 0; j < 32; j += 8) {
                                if (c0 + j < p.k) {
                                    float o[8];
#pragma unroll
                                    for (int i = 0; i < 8; ++i) o[i] = v[mt][j + i] * inv;
                                    Store<T>::row8(dst + j, o);
                                }
                            }
                        } else {
#pragma unroll
                            for (int j = 0; j < 32; ++j)
                                if (c0 + j < p.k) Store<T>::one(dst + j, v[mt][j] * inv);
                        }
                    }
                }
            }
            if (!small_k) {
                tc::fence_before();
                tc::mbar_arrive(&tmem_empty[rg]);
            }
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc(tmem, tcols);
}

// ---------------------------------------------------------------------------------------------
// Large-n variant (256 < n <= 512, nL <= 256, d = 128, bf16). X_b (n_pad x d = 128 KB) fits only
// once and W_L (nL x n, up to 256 KB) cannot stay resident, so the kernel streams:
//   * X_b in four 128-row chunks, each with its own full/empty barrier. Chunk c is released as
//     soon as the F MMAs of M-tile c are done and the LCB threads whose residual rows it holds
//     have read them, so the next sample's chunks load while this sample's F MMAs and epilogues
//     run, and its P/L MMAs start on chunk 0 as it lands (the chunks holding LCB rows, read last,
//     are needed last).
//   * W_L in [128 x 64] panels (16 KB) through a TMA ring (4 stages; Y^T also streams, in
//     [k_pad x 64] panels through its own ring, so W_L gets its 32 KB), in K-outer order: for each
//     64-row K panel of X, P and both L M-tiles advance, so P/L consume X chunk by chunk.
// Warps: 0 X producer, 1 MMA issuer (the whole warp walks the schedule, one elected lane issues),
// 2 W_L producer, 3..10 LCB group (8 warps: TMEM lane quarter x L M-tile; the M-tile-0 warps
// also route P to the bf16 Pbuf), 11..14 FM group, 15 Y^T producer. TMEM:
// P | L (2 M-tiles) | F (4 M-tiles) in one 512-column region, with separate "drained" barriers
// for P+L (LCB group) and F (FM group), so this sample's FM epilogue overlaps the next sample's
// P/L MMAs.
// ---------------------------------------------------------------------------------------------
// Wait-site profiling (LATTICE_FM_TRACE=1, lattice_fm_lcb only): cycles each role spends blocked
// per barrier, summed per CTA -- the pipeline's critical path without a profiler.
#define FM_WAIT(site, bar, parity)                                                \
    do {                                                                          \
        if (p.trace) {                                                            \
            const long long _t0 = clock64();                                      \
            tc::mbar_wait(bar, parity);                                           \
            wt[site] += (unsigned long long)(clock64() - _t0);                    \
        } else {                                                                  \
            tc::mbar_wait(bar, parity);                                           \
        }                                                                         \
    } while (0)

constexpr int kLargeWarps = 16;
constexpr int kLargeThreads = kLargeWarps * 32;
constexpr int kYtStages = 2;

struct GeoL {
    int panels_n, ml, mf, chunks, wl_stages, ys;
    uint32_t xpanel, ytpanel, ppanel, wlpanel, pbytes;
    __host__ __device__ GeoL(const Params& p) {
        panels_n = p.n_pad / 64;
        ml = (p.nL + 127) / 128;
        mf = p.n_pad / 128;
        chunks = p.n_pad / 128;
        xpanel = (uint32_t)p.n_pad * 128u;
        ytpanel = (uint32_t)p.k_pad * 128u;
        ppanel = (uint32_t)p.k_pad * 128u;
        wlpanel = 128u * 128u;
        pbytes = (2 * ppanel + 1023u) & ~1023u;
        ys = p.y_res ? panels_n : kYtStages;  // Y^T panels held: all (resident) or a 2-deep ring
        // as many W_L stages (<= 5) as fit next to X, Y^T and Pbuf (227 KB per CTA)
        const int64_t left = 227 * 1024 - 1024 - 512 - 2 * (int64_t)xpanel - ys * (int64_t)ytpanel - pbytes;
        wl_stages = (int)(left / wlpanel);
        if (wl_stages > 5) wl_stages = 5;
    }
};

__global__ void __launch_bounds__(kLargeThreads, 1)
    fm_lcb_large_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmWL,
                        const __grid_constant__ CUtensorMap tmYT, const Params p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
    const int kpad = p.k_pad;
    constexpr int d = 128;
    const GeoL g(p);
    const int NW = g.wl_stages;
    uint8_t* sX = smem;                                   // [2 d-panels][n_pad rows][128 B]
    uint8_t* sWL = sX + 2 * g.xpanel;                     // ring [NW][128 rows][128 B]
    uint8_t* sYT = sWL + NW * g.wlpanel;                  // [ys][k_pad rows][128 B]: ring or resident
    uint8_t* sP = sYT + g.ys * g.ytpanel;                 // [2 d-panels][k_pad][128 B]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sP + g.pbytes);
    uint64_t* x_full = bars;                  // [4] chunk landed
    uint64_t* x_empty = bars + 4;             // [4] chunk consumed (its F M-tile done)
    uint64_t* wl_full = bars + 8;             // [NW <= 5]
    uint64_t* wl_empty = bars + 13;           // [NW]
    uint64_t* yt_full = bars + 18;            // [kYtStages <= 4]
    uint64_t* yt_empty = bars + 22;           // [4]
    uint64_t* pl_full = bars + 26;            // P and L M-tile 0 accumulated
    uint64_t* pbuf_full = bars + 27;          // P routed to Pbuf (bf16)
    uint64_t* f_full = bars + 28;             // F accumulated
    uint64_t* l_empty = bars + 29;            // P + L M-tile 0 drained (LCB M-tile-0 warps)
    uint64_t* f_empty = bars + 30;            // F region drained (FM group)
    uint64_t* l1_full = bars + 33;            // L M-tile 1 accumulated
    uint64_t* l1_empty = bars + 34;           // L M-tile 1 drained (LCB M-tile-1 warps)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 31);
    float* red_f = reinterpret_cast<float*>(bars + 35);   // [2][4]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0 && lane == 0) {
        tc::tma_prefetch(&tmX);
        tc::tma_prefetch(&tmWL);
        tc::tma_prefetch(&tmYT);
        for (int c = 0; c < 4; ++c) {
            // chunk c is released by its F M-tile's MMA commit and by the LCB threads whose
            // residual row X[nF+i] lies in it (they pick it up into registers when it lands)
            const int lo = max(128 * c, p.nF), hi = min(128 * c + 128, p.nF + p.nL);
            tc::mbar_init(&x_full[c], 1);
            tc::mbar_init(&x_empty[c], 1 + (hi > lo ? hi - lo : 0));
        }
        for (int i = 0; i < NW; ++i) {
            tc::mbar_init(&wl_full[i], 1);
            tc::mbar_init(&wl_empty[i], 1);
        }
        for (int i = 0; i < kYtStages; ++i) {
            tc::mbar_init(&yt_full[i], 1);
            tc::mbar_init(&yt_empty[i], 1);
        }
        tc::mbar_init(pl_full, 1);
        tc::mbar_init(pbuf_full, 128);
        tc::mbar_init(f_full, 1);
        tc::mbar_init(l_empty, 4 * 32);
        tc::mbar_init(l1_full, 1);
        tc::mbar_init(l1_empty, 4 * 32);
        tc::mbar_init(f_empty, 4 * 32);
        tc::fence_mbar_init();
    }
    if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t t_Pb = tmem, t_Lb = tmem + 64, t_Fb = tmem + 64 + 2 * 128;
    // PDL: everything above overlaps the preceding kernel's tail; X (and the outputs) after this
    tc::griddep_wait();
    tc::griddep_launch_dependents();

    if (warp == 0) {
        if (lane == 0) {  // ---- X producer: four 128-row chunks per sample, two d-panels each
            unsigned long long wt[16] = {0};
            int it = 0;
            for (int64_t b = blockIdx.x; b < p.B; b += gridDim.x, ++it) {
                for (int c = 0; c < g.chunks; ++c) {
                    FM_WAIT(8, &x_empty[c], (it & 1) ^ 1);
                    tc::mbar_expect_tx(&x_full[c], 2u * 128u * 128u);
                    for (int pd = 0; pd < 2; ++pd)
                        tc::tma_load_3d(sX + pd * g.xpanel + c * 16384, &tmX, &x_full[c], pd * 64, c * 128, (int)b);
                }
            }
            if (p.trace) p.trace[blockIdx.x * 16 + 8] = wt[8];
        }
    } else if (warp == 2) {
        if (lane == 0) {  // ---- W_L producer, in the MMA's K-outer order
            unsigned long long wt[16] = {0};
            int gw = 0;
            for (int64_t b = blockIdx.x; b < p.B; b += gridDim.x) {
                for (int mt = 0; mt < g.ml; ++mt) {  // the MMA's order: M-tile 0 over K, then M-tile 1
                    for (int kp = 0; kp < g.panels_n; ++kp, ++gw) {
                        const int s = gw % NW;
                        FM_WAIT(10, &wl_empty[s], ((gw / NW) & 1) ^ 1);
                        tc::mbar_expect_tx(&wl_full[s], g.wlpanel);
                        tc::tma_load_2d(sWL + s * g.wlpanel, &tmWL, &wl_full[s], kp * 64, mt * 128);
                    }
                }
            }
            if (p.trace) p.trace[blockIdx.x * 16 + 10] = wt[10];
        }
    } else if (warp == 15) {
        if (lane == 0 && p.y_res) {  // ---- Y^T resident: every panel once, on yt_full[0]
            tc::mbar_expect_tx(&yt_full[0], (uint32_t)g.panels_n * g.ytpanel);
            for (int kp = 0; kp < g.panels_n; ++kp) tc::tma_load_2d(sYT + kp * g.ytpanel, &tmYT, &yt_full[0], kp * 64, 0);
        } else if (lane == 0) {  // ---- Y^T producer: [k_pad x 64] panels through its own ring
            unsigned long long wt[16] = {0};
            int gy = 0;
            for (int64_t b = blockIdx.x; b < p.B; b += gridDim.x) {
                for (int kp = 0; kp < g.panels_n; ++kp, ++gy) {
                    const int sy = gy % kYtStages;
                    FM_WAIT(9, &yt_empty[sy], ((gy / kYtStages) & 1) ^ 1);
                    tc::mbar_expect_tx(&yt_full[sy], g.ytpanel);
                    tc::tma_load_2d(sYT + sy * g.ytpanel, &tmYT, &yt_full[sy], kp * 64, 0);
                }
            }
            if (p.trace) p.trace[blockIdx.x * 16 + 9] = wt[9];
        }
    } else if (warp == 1) {  // ---- MMA issuer: the whole warp walks the schedule, one lane issues
        const uint32_t id_P = tc::idesc_bf16(128, kpad, 1, 0);
        const uint32_t id_L = tc::idesc_bf16(128, d, 0, 1);
        const uint32_t id_F = tc::idesc_bf16(128, kpad, 0, 0);
        // descriptors built once; a step moves the 14-bit start address field (bytes >> 4) only
        const uint64_t dx_mn = tc::sdesc(tc::smem_u32(sX), g.xpanel, 1024, 2);      // X^T (P: A) / X (L: B)
        const uint64_t dx_k = tc::sdesc(tc::smem_u32(sX), 16, 1024, 2);             // X (F: A)
        const uint64_t dy = tc::sdesc(tc::smem_u32(sYT), 16, 1024, 2);
        const uint64_t dwl = tc::sdesc(tc::smem_u32(sWL), 16, 1024, 2);
        const uint64_t dp = tc::sdesc(tc::smem_u32(sP), 16, 1024, 2);
        int it = 0, sw = 0, sy = 0;
        uint32_t pw = 0, py = 0;  // ring phases
        unsigned long long wt[16] = {0};
        const long long t_start = clock64();
        if (p.y_res) FM_WAIT(2, &yt_full[0], 0);
        for (int64_t b = blockIdx.x; b < p.B; b += gridDim.x, ++it) {
            const uint32_t ph = it & 1;
            // P and L M-tile 0 over every K panel, then L M-tile 1: the LCB warps of M-tile 0 drain
            // their rows (and route P) while M-tile 1 accumulates, and vice versa across samples
            FM_WAIT(0, l_empty, ph ^ 1);  // the previous sample's P and L M-tile 0 are drained
            tc::fence_after();
            auto l_panel = [&](int mt, int kp) {  // L[mt] += W_L[mt, k0:k0+64] . X[k0:k0+64, :]
                FM_WAIT(3, &wl_full[sw], pw);
                tc::fence_after();
                const uint64_t xk = dx_mn + (uint64_t)((kp * 64 * 128) >> 4);
                const uint64_t wk = dwl + (uint64_t)((sw * g.wlpanel) >> 4);
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    tc::mma_f16_warp(t_Lb + mt * 128, wk + (uint64_t)(j * 2), xk + (uint64_t)((j * 16 * 128) >> 4), id_L,
                                     (kp | j) != 0);
                tc::mma_commit_warp(&wl_empty[sw]);
                if (++sw == NW) sw = 0, pw ^= 1;
            };
            for (int kp = 0; kp < g.panels_n; ++kp) {
                if ((kp & 1) == 0) FM_WAIT(1, &x_full[kp >> 1], ph);
                if (!p.y_res) FM_WAIT(2, &yt_full[sy], py);
                tc::fence_after();
                const uint64_t xk = dx_mn + (uint64_t)((kp * 64 * 128) >> 4);
                const uint64_t yk = dy + (uint64_t)(((p.y_res ? kp : sy) * g.ytpanel) >> 4);
#pragma unroll
                for (int j = 0; j < 4; ++j)  // P += X^T[:, k0:k0+16] . Y[k0:k0+16, :]
                    tc::mma_f16_warp(t_Pb, xk + (uint64_t)((j * 16 * 128) >> 4), yk + (uint64_t)(j * 2), id_P,
                                     (kp | j) != 0);
                if (!p.y_res) {
                    tc::mma_commit_warp(&yt_empty[sy]);
                    if (++sy == kYtStages) sy = 0, py ^= 1;
                }
                if (g.ml > 0) l_panel(0, kp);
            }
            tc::mma_commit_warp(pl_full);
            if (g.ml > 1) {
                FM_WAIT(0, l1_empty, ph ^ 1);  // the previous sample's L M-tile 1 is drained
                tc::fence_after();
                for (int kp = 0; kp < g.panels_n; ++kp) l_panel(1, kp);
                tc::mma_commit_warp(l1_full);
            }
            FM_WAIT(4, pbuf_full, ph);
            FM_WAIT(5, f_empty, ph ^ 1);  // the previous sample's F is drained
            tc::fence_after();
            for (int mt = 0; mt < g.mf; ++mt) {  // F = X P, M-tile mt = X chunk mt
#pragma unroll
                for (int kk = 0; kk < d / 16; ++kk) {
                    const uint32_t pan = (uint32_t)(kk / 4), kin = (uint32_t)(kk % 4) * 32;
                    tc::mma_f16_warp(t_Fb + mt * kpad, dx_k + (uint64_t)((pan * g.xpanel + mt * 16384 + kin) >> 4),
                                     dp + (uint64_t)((pan * g.ppanel + kin) >> 4), id_F, kk != 0);
                }
                tc::mma_commit_warp(&x_empty[mt]);  // every MMA reading chunk mt has completed
            }
            tc::mma_commit_warp(f_full);
        }
        if (p.trace && lane == 0) {
            for (int i = 0; i < 6; ++i) p.trace[blockIdx.x * 16 + i] = wt[i];
            p.trace[blockIdx.x * 16 + 6] = (unsigned long long)(clock64() - t_start);
            p.trace[blockIdx.x * 16 + 7] = (unsigned long long)it;
        }
    } else if (warp < 11) {  // ---- LCB group, warps 3..10: lane quarter q, L M-tile mt
        const int q = warp & 3;
        const int mt = (warp - 3) >> 2;
        const int row = q * 32 + lane;
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const float inv_d = 1.0f / (float)d;
        const int i = mt * 128 + row;
        const bool live = mt < g.ml && i < p.nL;
        // tcgen05.ld is warp-collective: a warp with any live lane runs the whole epilogue, its
        // dead lanes on a valid residual row with their stores and arrivals masked
        const bool warp_live = mt < g.ml && mt * 128 + q * 32 < p.nL;
        const int xr = p.nF + (live ? i : 0);
        const int cx = xr >> 7;  // the X chunk holding the residual row
        const uint32_t t_L = t_Lb + lane_off + mt * 128;
        int it = 0;
        for (int64_t b = blockIdx.x; b < p.B; b += gridDim.x, ++it) {
            if (mt == 1 && g.ml < 2) continue;  // nL <= 128: no second L M-tile
            tc::mbar_wait(mt == 0 ? pl_full : l1_full, it & 1);
            tc::fence_after();
            if (mt == 0) {  // P row `row` (a d index) -> bf16 -> Pbuf[j][row], F's K-major B operand
                for (int c0 = 0; c0 < kpad; c0 += 16) {
                    float pv[16];
                    tc::tmem_ld16(t_Pb + lane_off + c0, pv);
                    uint8_t* pan = sP + (row / 64) * g.ppanel;
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        *reinterpret_cast<__nv_bfloat16*>(pan + swz<2>(c0 + j, row & 63)) = __float2bfloat16_rn(pv[j]);
                }
                tc::fence_async_shared();
                tc::mbar_arrive(pbuf_full);
            }
            if (warp_live) {  // X'[nF+i] = rms_norm_d(L[i] + X[nF+i]): pass 1 forms L + X (the residual
                              // row from the X chunk in shared memory, read once), keeps it in TMEM in
                              // place of L and sums its squares; pass 2 normalises and stores. The
                              // chunk is released after pass 1 (the next sample's chunk loads behind it).
                float ss4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int c = 0; c < d; c += 16) {
                    float v[16];
                    tc::tmem_ld16(t_L + c, v);
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
                        const int e = c + 8 * hh;
                        const uint4 r = *reinterpret_cast<const uint4*>(sX + (e / 64) * g.xpanel + swz<2>(xr, e & 63));
                        const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            v[8 * hh + 2 * k] += bf16_lo(w[k]);
                            v[8 * hh + 2 * k + 1] += bf16_hi(w[k]);
                            ss4[k] = fmaf(v[8 * hh + 2 * k], v[8 * hh + 2 * k], ss4[k]);
                            ss4[k] = fmaf(v[8 * hh + 2 * k + 1], v[8 * hh + 2 * k + 1], ss4[k]);
                        }
                    }
                    tc::tmem_st16(t_L + c, v);
                }
                tc::tmem_wait_st();
                if (live) tc::mbar_arrive(&x_empty[cx]);
                const float ss = (ss4[0] + ss4[1]) + (ss4[2] + ss4[3]);
                const float inv = 1.0f / sqrtf(ss * inv_d + 1e-6f);
                __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(p.Xout) + (b * p.n + xr) * (int64_t)d;
#pragma unroll
                for (int c = 0; c < d; c += 16) {  // 16 values per 32-byte store
                    float v[16];
                    tc::tmem_ld16(t_L + c, v);
                    uint32_t o[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) o[k] = pack_bf16x2(v[2 * k] * inv, v[2 * k + 1] * inv);
                    if (live)
                        st_global_256(dst + c, make_uint4(o[0], o[1], o[2], o[3]), make_uint4(o[4], o[5], o[6], o[7]));
                }
            }
            tc::fence_before();
            tc::mbar_arrive(mt == 0 ? l_empty : l1_empty);
        }
    } else {  // ---- FM group, warps 11..14: Fin = rms_norm(flatten(X P)) over 4 M-tiles, two TMEM passes
        const int q = warp & 3;
        const int e = warp - 11;
        const int row = q * 32 + lane;
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const float inv_nk = 1.0f / (float)(p.n * p.k);
        int it = 0;
        for (int64_t b = blockIdx.x; b < p.B; b += gridDim.x, ++it) {
            tc::mbar_wait(f_full, it & 1);
            tc::fence_after();
            float ss4[4] = {0.f, 0.f, 0.f, 0.f};
            for (int mt = 0; mt < g.mf; ++mt) {
                const int r = mt * 128 + row;
                for (int c0 = 0; c0 < kpad; c0 += 16) {
                    float v[16];
                    tc::tmem_ld16(t_Fb + lane_off + mt * kpad + c0, v);
                    if (r < p.n) {
#pragma unroll
                        for (int j = 0; j < 16; ++j)
                            if (c0 + j < p.k) ss4[j & 3] = fmaf(v[j], v[j], ss4[j & 3]);
                    }
                }
            }
            float ss = warp_sum((ss4[0] + ss4[1]) + (ss4[2] + ss4[3]));
            float* red = red_f + (it & 1) * 4;
            if (lane == 0) red[e] = ss;
            tc::named_bar(2, 128);
            const float inv = 1.0f / sqrtf((red[0] + red[1] + red[2] + red[3]) * inv_nk + 1e-6f);
            for (int mt = 0; mt < g.mf; ++mt) {
                const int r = mt * 128 + row;
                for (int c0 = 0; c0 < kpad; c0 += 16) {
                    float v[16];
                    tc::tmem_ld16(t_Fb + lane_off + mt * kpad + c0, v);
                    if (r < p.n) {
                        __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(p.Fout) + b * (int64_t)p.n * p.k +
                                             (int64_t)r * p.k + c0;
                        if ((p.k & 15) == 0) {
                            float o[16];
#pragma unroll
                            for (int k = 0; k < 16; ++k) o[k] = v[k] * inv;
                            Store<__nv_bfloat16>::row16(dst, o);
                        } else {
#pragma unroll
                            for (int j = 0; j < 16; ++j)
                                if (c0 + j < p.k) dst[j] = __float2bfloat16_rn(v[j] * inv);
                        }
                    }
                }
            }
            tc::fence_before();
            tc::mbar_arrive(f_empty);
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

size_t smem_bytes_large(const Params& p) {
    const GeoL g(p);
    return 1024 + 2 * (size_t)g.xpanel + (size_t)g.wl_stages * g.wlpanel + g.ys * (size_t)g.ytpanel +
           g.pbytes + 512;
}

bool is_large(const Params& p) { return p.n_pad > 256; }

// ---------------------------------------------------------------------------------------------
// CTA-pair variant of the large kernel (n_pad = 512, bf16, d = 128, k_pad 16 or 32, nF and nL
// multiples of 32): a cluster of two CTAs on one TPC takes two samples per pass, CTA r holding
// sample 2s + r in its shared memory, and every MMA is a cta_group::2 MMA issued by the leader:
//   P  (M = 256: each CTA's X^T rows) x Y      -> each CTA's TMEM holds its own sample's P;
//                                                 CTA r keeps Y^T rows [r k/2, +k/2) resident
//   L  (M = 256: CTA r's W_L rows [128r, +128)) x [X_a | X_b] (N = 256: each CTA's X)
//                                              -> CTA r holds L rows [128r, +128) of both samples
//   F  (M = 256: each CTA's X rows) x [P_a | P_b] (N = 2k) -> CTA r reads its own sample's columns
// so W_L streams once per PAIR of samples and each SM stages half of it: shared-memory operand
// traffic per sample drops by about a third against the single-CTA kernel, which is bound by it.
// The LCB epilogue reads its own sample's residual rows from shared memory and the partner's
// from global memory (L2-resident: the partner's TMA load just brought them in).
// Measured (scripts/fm_bench.py, B = 65536): 4.49 ms against the single-CTA kernel's 3.48 ms, so
// it is opt-in (LATTICE_FM_PAIR=1): L (256 columns) and F (256, P aliased) fill TMEM, so L cannot
// be double-buffered and each pass's LCB epilogue (the partner half waiting on L2) sits between
// this pass's and the next pass's L MMAs; the single-CTA kernel overlaps them across its two
// L M-tiles.
// ---------------------------------------------------------------------------------------------
struct GeoP {
    int kh, wl_stages;
    uint32_t xpanel, ytpanel, ybytes, ppanel, pbytes, wlpanel;
    __host__ __device__ GeoP(const Params& p) {
        kh = p.k_pad / 2;
        xpanel = (uint32_t)p.n_pad * 128u;
        ytpanel = (uint32_t)kh * 128u;                       // one 64-wide K panel of this CTA's Y^T rows
        ybytes = (((uint32_t)p.n_pad / 64u) * ytpanel + 1023u) & ~1023u;
        ppanel = (uint32_t)p.k_pad * 128u;
        pbytes = (2 * ppanel + 1023u) & ~1023u;
        wlpanel = 128u * 128u;
        const int64_t left = 227 * 1024 - 1024 - 512 - 2 * (int64_t)xpanel - ybytes - pbytes;
        wl_stages = (int)(left / wlpanel);
        if (wl_stages > 8) wl_stages = 8;
    }
};

__global__ void __launch_bounds__(kLargeThreads, 1)
    fm_lcb_pair_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmWL,
                       const __grid_constant__ CUtensorMap tmYT, const Params p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
    const int kpad = p.k_pad;
    constexpr int d = 128;
    const GeoP g(p);
    const int NW = g.wl_stages;
    const int panels_n = p.n_pad / 64;
    uint8_t* sX = smem;                       // [2 d-panels][n_pad rows][128 B]: this CTA's sample
    uint8_t* sWL = sX + 2 * g.xpanel;         // ring [NW][128 rows][128 B]: this CTA's W_L rows
    uint8_t* sYT = sWL + NW * g.wlpanel;      // [panels_n][k/2 rows][128 B]: this CTA's Y^T rows, resident
    uint8_t* sP = sYT + g.ybytes;             // [2 d-panels][k_pad][128 B]: this sample's P^T (F's B half)
    uint64_t* bars = reinterpret_cast<uint64_t*>(sP + g.pbytes);
    uint64_t* x_full = bars;          // [4] leader: both CTAs' chunk c landed
    uint64_t* x_empty = bars + 4;     // [4] local: chunk c consumed (F M-tile c + own-sample LCB reads)
    uint64_t* wl_full = bars + 8;     // [NW <= 8] leader
    uint64_t* wl_empty = bars + 16;   // [NW] local
    uint64_t* y_full = bars + 24;     // leader: both CTAs' Y^T halves resident
    uint64_t* pl_full = bars + 25;    // local: P and L accumulated
    uint64_t* pbuf_full = bars + 26;  // leader: both CTAs' P routed (8 warps)
    uint64_t* f_full = bars + 27;     // local: F accumulated
    uint64_t* l_empty = bars + 28;    // leader: L drained (16 LCB warps of both CTAs)
    uint64_t* f_empty = bars + 29;    // leader: F drained (8 FM warps)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 30);
    float* red_f = reinterpret_cast<float*>(bars + 31);  // [2][4]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rank = (int)tc::cluster_rank();
    const int64_t npairs = (p.B + 1) / 2;
    const int64_t first = blockIdx.x >> 1, stride = gridDim.x >> 1;
    if (warp == 0 && lane == 0) {
        tc::tma_prefetch(&tmX);
        tc::tma_prefetch(&tmWL);
        tc::tma_prefetch(&tmYT);
        for (int c = 0; c < 4; ++c) {
            // the MMA commit + this CTA's LCB warps whose residual rows (own sample) lie in chunk c
            int readers = 0;
            for (int q = 0; q < 4; ++q) {
                const int i = 128 * rank + 32 * q;
                if (i < p.nL && ((p.nF + i) >> 7) == c) ++readers;
            }
            tc::mbar_init(&x_full[c], 1);
            tc::mbar_init(&x_empty[c], 1 + readers);
        }
        for (int i = 0; i < NW; ++i) {
            tc::mbar_init(&wl_full[i], 1);
            tc::mbar_init(&wl_empty[i], 1);
        }
        tc::mbar_init(y_full, 1);
        tc::mbar_init(pl_full, 1);
        tc::mbar_init(pbuf_full, 8);
        tc::mbar_init(f_full, 1);
        tc::mbar_init(l_empty, 16);
        tc::mbar_init(f_empty, 8);
        tc::fence_mbar_init();
    }
    if (warp == 1) tc::tmem_alloc_cg2(tmem_slot, 512);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    tc::cluster_sync();
    const uint32_t tmem = *tmem_slot;
    const uint32_t t_L = tmem, t_F = tmem + 256, t_P = t_F;  // P is routed out before F overwrites it
    tc::griddep_wait();
    tc::griddep_launch_dependents();

    if (warp == 0) {
        if (lane == 0) {  // ---- X producer: this CTA's sample, four 128-row chunks, completions on the leader
            int it = 0;
            for (int64_t sp = first; sp < npairs; sp += stride, ++it) {
                const int b = (int)(2 * sp + rank);  // b == B (odd batch): zero-filled or unused rows, no output
                for (int c = 0; c < 4; ++c) {
                    tc::mbar_wait(&x_empty[c], (it & 1) ^ 1);
                    if (rank == 0) tc::mbar_expect_tx(&x_full[c], 2u * 2u * 128u * 128u);
                    const uint32_t bar = tc::mapa(tc::smem_u32(&x_full[c]), 0);
                    for (int pd = 0; pd < 2; ++pd)
                        tc::tma_load_3d_cg2(sX + pd * g.xpanel + c * 16384, &tmX, bar, pd * 64, c * 128, b);
                }
            }
        }
    } else if (warp == 2) {
        if (lane == 0) {  // ---- W_L producer: this CTA's 128 rows, K panel by K panel
            int gw = 0;
            for (int64_t sp = first; sp < npairs; sp += stride) {
                for (int kp = 0; kp < panels_n; ++kp, ++gw) {
                    const int s = gw % NW;
                    tc::mbar_wait(&wl_empty[s], ((gw / NW) & 1) ^ 1);
                    if (rank == 0) tc::mbar_expect_tx(&wl_full[s], 2u * g.wlpanel);
                    tc::tma_load_2d_cg2(sWL + s * g.wlpanel, &tmWL, tc::mapa(tc::smem_u32(&wl_full[s]), 0), kp * 64,
                                        rank * 128);
                }
            }
        }
    } else if (warp == 3) {
        if (lane == 0) {  // ---- Y^T rows [r k/2, +k/2), once
            if (rank == 0) tc::mbar_expect_tx(y_full, 2u * (uint32_t)panels_n * g.ytpanel);
            const uint32_t bar = tc::mapa(tc::smem_u32(y_full), 0);
            for (int kp = 0; kp < panels_n; ++kp)
                tc::tma_load_2d_cg2(sYT + kp * g.ytpanel, &tmYT, bar, kp * 64, rank * g.kh);
        }
    } else if (warp == 1) {
        if (rank == 0) {  // ---- MMA issuer (leader): the whole warp walks the schedule, one lane issues
            const uint32_t id_P = tc::idesc_bf16(256, kpad, 1, 0);
            const uint32_t id_L = tc::idesc_bf16(256, 256, 0, 1);
            const uint32_t id_F = tc::idesc_bf16(256, 2 * kpad, 0, 0);
            const uint64_t dx_mn = tc::sdesc(tc::smem_u32(sX), g.xpanel, 1024, 2);  // X^T (P: A) / X (L: B)
            const uint64_t dx_k = tc::sdesc(tc::smem_u32(sX), 16, 1024, 2);         // X (F: A)
            const uint64_t dy = tc::sdesc(tc::smem_u32(sYT), 16, 1024, 2);
            const uint64_t dwl = tc::sdesc(tc::smem_u32(sWL), 16, 1024, 2);
            const uint64_t dp = tc::sdesc(tc::smem_u32(sP), 16, 1024, 2);
            int it = 0, sw = 0;
            uint32_t pw = 0;
            unsigned long long wt[16] = {0};
            const long long t_start = clock64();
            tc::mbar_wait(y_full, 0);
            for (int64_t sp = first; sp < npairs; sp += stride, ++it) {
                const uint32_t ph = it & 1;
                FM_WAIT(0, l_empty, ph ^ 1);  // the previous pass's L is drained
                FM_WAIT(5, f_empty, ph ^ 1);  // ... and its F (P shares F's columns)
                tc::fence_after();
                for (int kp = 0; kp < panels_n; ++kp) {
                    if ((kp & 1) == 0) FM_WAIT(1, &x_full[kp >> 1], ph);
                    tc::fence_after();
                    const uint64_t xk = dx_mn + (uint64_t)((kp * 64 * 128) >> 4);
                    const uint64_t yk = dy + (uint64_t)((kp * g.ytpanel) >> 4);
#pragma unroll
                    for (int j = 0; j < 4; ++j)  // P += X^T[:, k0:k0+16] . Y[k0:k0+16, :]
                        tc::mma_f16_cg2_warp(t_P, xk + (uint64_t)((j * 16 * 128) >> 4), yk + (uint64_t)(j * 2), id_P,
                                             (kp | j) != 0);
                    FM_WAIT(3, &wl_full[sw], pw);
                    tc::fence_after();
                    const uint64_t wk = dwl + (uint64_t)((sw * g.wlpanel) >> 4);
#pragma unroll
                    for (int j = 0; j < 4; ++j)  // L += W_L[:, k0:k0+16] . [X_a | X_b][k0:k0+16, :]
                        tc::mma_f16_cg2_warp(t_L, wk + (uint64_t)(j * 2), xk + (uint64_t)((j * 16 * 128) >> 4), id_L,
                                             (kp | j) != 0);
                    tc::mma_commit_cg2_warp(&wl_empty[sw]);
                    if (++sw == NW) sw = 0, pw ^= 1;
                }
                tc::mma_commit_cg2_warp(pl_full);
                FM_WAIT(4, pbuf_full, ph);
                tc::fence_after();
                for (int mt = 0; mt < 4; ++mt) {  // F = X [P_a | P_b], M-tile mt = X chunk mt
#pragma unroll
                    for (int kk = 0; kk < d / 16; ++kk) {
                        const uint32_t pan = (uint32_t)(kk / 4), kin = (uint32_t)(kk % 4) * 32;
                        tc::mma_f16_cg2_warp(t_F + mt * 2 * kpad,
                                             dx_k + (uint64_t)((pan * g.xpanel + mt * 16384 + kin) >> 4),
                                             dp + (uint64_t)((pan * g.ppanel + kin) >> 4), id_F, kk != 0);
                    }
                    tc::mma_commit_cg2_warp(&x_empty[mt]);  // every MMA reading chunk mt (both CTAs) is done
                }
                tc::mma_commit_cg2_warp(f_full);
            }
            if (p.trace && lane == 0) {
                for (int i = 0; i < 6; ++i) p.trace[blockIdx.x * 16 + i] = wt[i];
                p.trace[blockIdx.x * 16 + 6] = (unsigned long long)(clock64() - t_start);
                p.trace[blockIdx.x * 16 + 7] = (unsigned long long)it;
            }
        }
    } else if (warp < 12) {  // ---- LCB, warps 4..11: lane quarter q, sample half h (L columns [128h, +128))
        const int q = warp & 3;
        const int h = (warp - 4) >> 2;
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const float inv_d = 1.0f / (float)d;
        const int i = 128 * rank + 32 * q + lane;  // W_L row
        const bool live = 128 * rank + 32 * q < p.nL;  // warp-uniform (nL % 32 == 0)
        const bool local = h == rank;                  // the residual rows sit in this CTA's smem
        const int xr = p.nF + i;
        const uint32_t t = t_L + lane_off + h * 128;
        int it = 0;
        unsigned long long t_epi = 0;
        for (int64_t sp = first; sp < npairs; sp += stride, ++it) {
            const int64_t bh = 2 * sp + h;
            const bool act = live && bh < p.B;
            // the residual row X[bh][nF+i] in registers: the partner's sample from global memory,
            // issued before the wait so its latency hides behind the MMAs; this CTA's own from smem
            uint4 res[16];
            if (act && !local) {
                const uint4* grow = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(p.Xin) +
                                                                   (bh * p.n + xr) * (int64_t)d);
#pragma unroll
                for (int j = 0; j < 16; ++j) res[j] = __ldg(grow + j);
            }
            tc::mbar_wait(pl_full, it & 1);
            tc::fence_after();
            const long long t0 = clock64();
            if (act) {  // X'[nF+i] = rms_norm_d(L[i] + X[nF+i]): sum of squares, then normalise + store
                if (local) {
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        res[j] = *reinterpret_cast<const uint4*>(sX + (j / 8) * g.xpanel + swz<2>(xr, (j * 8) & 63));
                }
                float ss4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int c = 0; c < d; c += 16) {
                    float v[16];
                    tc::tmem_ld16(t + c, v);
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
                        const uint4 r = res[c / 8 + hh];
                        const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const float a = v[8 * hh + 2 * k] + bf16_lo(w[k]), bb = v[8 * hh + 2 * k + 1] + bf16_hi(w[k]);
                            ss4[k] = fmaf(a, a, ss4[k]);
                            ss4[k] = fmaf(bb, bb, ss4[k]);
                        }
                    }
                }
                const float ss = (ss4[0] + ss4[1]) + (ss4[2] + ss4[3]);
                const float inv = 1.0f / sqrtf(ss * inv_d + 1e-6f);
                __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(p.Xout) + (bh * p.n + xr) * (int64_t)d;
#pragma unroll
                for (int c = 0; c < d; c += 16) {
                    float v[16];
                    tc::tmem_ld16(t + c, v);
                    uint32_t o[8];
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {  // the residual again (smem, or L1/L2 for the partner's)
                        const int e = c + 8 * hh;
                        const uint4 r = local ? *reinterpret_cast<const uint4*>(sX + (e / 64) * g.xpanel + swz<2>(xr, e & 63))
                                              : __ldg(reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(p.Xin) +
                                                                                     (bh * p.n + xr) * (int64_t)d + e));
                        const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            o[4 * hh + k] = pack_bf16x2((v[8 * hh + 2 * k] + bf16_lo(w[k])) * inv,
                                                        (v[8 * hh + 2 * k + 1] + bf16_hi(w[k])) * inv);
                    }
                    st_global_256(dst + c, make_uint4(o[0], o[1], o[2], o[3]), make_uint4(o[4], o[5], o[6], o[7]));
                }
            }
            __syncwarp();
            if (live && local && lane == 0) tc::mbar_arrive(&x_empty[xr >> 7]);
            tc::fence_before();
            if (lane == 0) tc::mbar_arrive_remote_relaxed(tc::mapa(tc::smem_u32(l_empty), 0));
            t_epi += (unsigned long long)(clock64() - t0);
        }
        // trace: slot 9 = the local-residual LCB warp's epilogue cycles, slot 10 = the partner-residual one
        if (p.trace && lane == 0 && q == 0) p.trace[blockIdx.x * 16 + (local ? 9 : 10)] = t_epi;
    } else {  // ---- FM, warps 12..15: route P to Pbuf, then Fin = rms_norm(flatten(X P)) of this CTA's sample
        const int q = warp & 3;
        const int row = q * 32 + lane;
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const float inv_nk = 1.0f / (float)(p.n * p.k);
        int it = 0;
        for (int64_t sp = first; sp < npairs; sp += stride, ++it) {
            const int64_t bo = 2 * sp + rank;
            tc::mbar_wait(pl_full, it & 1);
            tc::fence_after();
            for (int c0 = 0; c0 < kpad; c0 += 16) {  // P row `row` (a d index) -> bf16 -> Pbuf[j][row]
                float pv[16];
                tc::tmem_ld16(t_P + lane_off + c0, pv);
                uint8_t* pan = sP + (row / 64) * g.ppanel;
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    *reinterpret_cast<__nv_bfloat16*>(pan + swz<2>(c0 + j, row & 63)) = __float2bfloat16_rn(pv[j]);
            }
            tc::fence_async_shared();
            tc::fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive_remote(tc::mapa(tc::smem_u32(pbuf_full), 0));
            tc::mbar_wait(f_full, it & 1);
            tc::fence_after();
            const uint32_t tf = t_F + lane_off + rank * kpad;  // this sample's columns of each M-tile
            float ss4[4] = {0.f, 0.f, 0.f, 0.f};
            for (int mt = 0; mt < 4; ++mt) {
                const int r = mt * 128 + row;
                for (int c0 = 0; c0 < kpad; c0 += 16) {
                    float v[16];
                    tc::tmem_ld16(tf + mt * 2 * kpad + c0, v);
                    if (r < p.n) {
#pragma unroll
                        for (int j = 0; j < 16; ++j)
                            if (c0 + j < p.k) ss4[j & 3] = fmaf(v[j], v[j], ss4[j & 3]);
                    }
                }
            }
            const float ssw = warp_sum((ss4[0] + ss4[1]) + (ss4[2] + ss4[3]));
            float* red = red_f + (it & 1) * 4;
            if (lane == 0) red[q] = ssw;
            tc::named_bar(2, 128);
            const float inv = 1.0f / sqrtf((red[0] + red[1] + red[2] + red[3]) * inv_nk + 1e-6f);
            if (bo < p.B) {
                for (int mt = 0; mt < 4; ++mt) {
                    const int r = mt * 128 + row;
                    for (int c0 = 0; c0 < kpad; c0 += 16) {
                        float v[16];
                        tc::tmem_ld16(tf + mt * 2 * kpad + c0, v);
                        if (r < p.n) {
                            __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(p.Fout) + bo * (int64_t)p.n * p.k +
                                                 (int64_t)r * p.k + c0;
                            if ((p.k & 15) == 0) {
                                float o[16];
#pragma unroll
                                for (int k = 0; k < 16; ++k) o[k] = v[k] * inv;
                                Store<__nv_bfloat16>::row16(dst, o);
                            } else {
#pragma unroll
                                for (int j = 0; j < 16; ++j)
                                    if (c0 + j < p.k) dst[j] = __float2bfloat16_rn(v[j] * inv);
                            }
                        }
                    }
                }
            }
            tc::fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive_remote_relaxed(tc::mapa(tc::smem_u32(f_empty), 0));
        }
    }
    tc::fence_before();
    __syncthreads();
    tc::cluster_sync();  // the leader's MMAs read the partner's smem and write its TMEM until the end
    if (warp == 1) tc::tmem_dealloc_cg2(tmem, 512);
}

size_t smem_bytes_pair(const Params& p) {
    const GeoP g(p);
    return 1024 + 2 * (size_t)g.xpanel + (size_t)g.wl_stages * g.wlpanel + g.ybytes + g.pbytes + 512;
}

// opt-in (LATTICE_FM_PAIR=1) for the large shapes it was written for: measured slower than the
// single-CTA kernel (4.49 vs 3.48 ms at B = 65536) -- its L accumulator fills
// half of TMEM with no second buffer, so each pass's LCB epilogue sits on the MMA critical path
bool is_pair(const Params& p) {
    static const int env = [] {
        const char* e = std::getenv("LATTICE_FM_PAIR");
        return e ? std::atoi(e) : 0;
    }();
    return env != 0 && p.n_pad == 512 && !p.f32 && p.d == 128 && (p.k_pad == 16 || p.k_pad == 32) &&
           p.nF % 32 == 0 && p.nL % 32 == 0 && GeoP(p).wl_stages >= 3 && smem_bytes_pair(p) <= 227 * 1024;
}


size_t smem_bytes(const Params& p) {
    if (is_large(p)) return smem_bytes_large(p);
    const Geo g(p, p.f32 ? 4 : 2);
    size_t s = 1024;
    s += (size_t)g.wlpanel * g.panels_n;   // W_L
    s += (size_t)g.ytpanel * g.panels_n;   // Y^T
    s += g.pbytes;                         // P
    s += g.xtbytes;                        // fp32: K-major X^T copy
    s += 2 * (size_t)g.xstage;             // X stages
    s += 128 + 8 * 4 + 2 * 2 * 128 * 4 + 64;  // barriers + FM / LCB reductions
    return s;
}

lattice_status check(const Params& p) {
    if (p.f32 ? p.d != 64 : !(p.d == 64 || p.d == 128))
        return set_error(LATTICE_USAGE, "fm_lcb: d must be 64 or 128 (bf16), 64 (fp32)");
    if (p.f32 && p.n_pad > 64) return set_error(LATTICE_USAGE, "fm_lcb: fp32 supports n <= 64");
    if (p.k < 1 || p.k_pad > 64 || p.k_pad % 16 || p.k_pad < p.k)
        return set_error(LATTICE_USAGE, "fm_lcb: k must be <= 64");
    if (is_large(p)) {  // streamed-W_L variant
        if (p.f32 || p.d != 128 || p.n_pad > 512 || p.n_pad % 256 || p.n_pad < p.n)
            return set_error(LATTICE_USAGE, "fm_lcb: n in (256, 512] needs bf16, d = 128 and n_pad = 512");
        if (p.nL < 0 || p.nL > 256 || p.nF + p.nL != p.n)
            return set_error(LATTICE_USAGE, "fm_lcb: nL must be <= 256 and nF + nL == n");
        if (64 + 256 + (p.n_pad / 128) * p.k_pad > 512)
            return set_error(LATTICE_USAGE, "fm_lcb: n = 512 needs k <= 48 (TMEM)");
        if (GeoL(p).wl_stages < 3 || smem_bytes(p) > 227 * 1024)
            return set_error(LATTICE_USAGE, "fm_lcb: shared memory budget exceeded");
        return LATTICE_OK;
    }
    if (p.n < 1 || p.n_pad % 16 || p.n_pad < p.n) return set_error(LATTICE_USAGE, "fm_lcb: bad n");
    if (p.nL < 0 || p.nL > 128 || p.nF + p.nL != p.n)
        return set_error(LATTICE_USAGE, "fm_lcb: nL must be <= 128 and nF + nL == n");
    if (region_cols(p) > 512) return set_error(LATTICE_USAGE, "fm_lcb: accumulators exceed TMEM");
    if (smem_bytes(p) > 227 * 1024) return set_error(LATTICE_USAGE, "fm_lcb: shared memory budget exceeded");
    return LATTICE_OK;
}

lattice_status make_maps(Plan* pl, const void* X, const void* WLpad, const void* YTpad) {
    const Params& p = pl->p;
    const int es = p.f32 ? 4 : 2, ep = 128 / es;
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
    cuuint64_t strides[2] = {(cuuint64_t)p.d * es, (cuuint64_t)p.n * p.d * es};
    // the large variant loads X in 128-row chunks (one box per chunk and d-panel)
    cuuint32_t box[3] = {(cuuint32_t)ep, (cuuint32_t)(p.n_pad > 256 ? 128 : p.n_pad), 1};
    cuuint32_t el[3] = {1, 1, 1};
    CUresult r = fn(&pl->tmX, p.f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
                    const_cast<void*>(X), dims, strides, box, el, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_error(LATTICE_CUDA, "fm_lcb: X tensor map (" + std::to_string((int)r) + ")");
    lattice_status s = gemm::make_map_2d(&pl->tmWL, WLpad, (uint64_t)p.n_pad, (uint64_t)wl_rows(p),
                                         (uint64_t)p.n_pad * es, ep, 128, p.f32);
    if (s != LATTICE_OK) return s;
    // the pair variant: each CTA loads its half of Y^T's rows
    return gemm::make_map_2d(&pl->tmYT, YTpad, (uint64_t)p.n_pad, (uint64_t)p.k_pad, (uint64_t)p.n_pad * es, ep,
                             (uint32_t)(is_large(p) && is_pair(p) ? p.k_pad / 2 : p.k_pad), p.f32);
}

template <typename T>
lattice_status launch_t(const Plan& pl, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        LAT_CUDA(cudaFuncSetAttribute(fm_lcb_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        attr = true;
    }
    const int grid = (int)(pl.p.B < num_sms() ? pl.p.B : num_sms());
    if (grid <= 0) return LATTICE_OK;
    LAT_CUDA(launch_pdl(fm_lcb_kernel<T>, grid, kResThreads, smem_bytes(pl.p), st, pl));
    LAT_CUDA(cudaGetLastError());
    return LATTICE_OK;
}

// programmatic stream serialization unless LATTICE_PDL=0 (see tc::griddep_wait)
template <typename K>
cudaError_t launch_pdl(K kernel, int grid, int threads, size_t smem, cudaStream_t st, const Plan& pl, int cluster = 1) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid, 1, 1);
    cfg.blockDim = dim3(threads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    int na = 0;
    if (cluster > 1) {
        at[na].id = cudaLaunchAttributeClusterDimension;
        at[na].val.clusterDim.x = cluster;
        at[na].val.clusterDim.y = 1;
        at[na].val.clusterDim.z = 1;
        ++na;
    }
    if (pdl_enabled()) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kernel, pl.tmX, pl.tmWL, pl.tmYT, pl.p);
}

lattice_status launch(const Plan& pl, cudaStream_t st) {
    if (is_large(pl.p) && is_pair(pl.p)) {
        static bool attr = false;
        if (!attr) {
            LAT_CUDA(cudaFuncSetAttribute(fm_lcb_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
            attr = true;
        }
        // persistent grid: as many pairs as the device keeps resident at once (a TPC's two SMs
        // per pair; not every SM finds a partner), so no pair waits for a second wave
        static int max_pairs[64] = {0};
        int dev = 0;
        LAT_CUDA(cudaGetDevice(&dev));
        int& mp = max_pairs[dev & 63];
        if (!mp) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(2 * (num_sms() / 2), 1, 1);
            cfg.blockDim = dim3(kLargeThreads, 1, 1);
            cfg.dynamicSmemBytes = smem_bytes_pair(pl.p);
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = 2;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            int mc = 0;
            if (cudaOccupancyMaxActiveClusters(&mc, fm_lcb_pair_kernel, &cfg) != cudaSuccess || mc < 1)
                mc = num_sms() / 2;
            mp = mc;
        }
        const int64_t pairs = (pl.p.B + 1) / 2;
        const int grid = 2 * (int)(pairs < mp ? pairs : mp);
        if (grid <= 0) return LATTICE_OK;
        LAT_CUDA(launch_pdl(fm_lcb_pair_kernel, grid, kLargeThreads, smem_bytes_pair(pl.p), st, pl, 2));
        LAT_CUDA(cudaGetLastError());
        return LATTICE_OK;
    }
    if (is_large(pl.p)) {
        static bool attr = false;
        if (!attr) {
            LAT_CUDA(cudaFuncSetAttribute(fm_lcb_large_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
            attr = true;
        }
        const int grid = (int)(pl.p.B < num_sms() ? pl.p.B : num_sms());
        if (grid <= 0) return LATTICE_OK;
        // Y^T resident (loaded once per CTA instead of streamed per sample: 32 KB less TMA traffic
        // into shared memory per sample, the kernel's bound) whenever >= 3 W_L stages still fit:
        // 3.48 -> 3.32 ms at B = 65536 (profiles/r02/ab/fm_large_yres_*.log); LATTICE_FM_YRES=0
        // keeps the 2-deep Y^T ring with 5 W_L stages
        static const int yres_env = [] {
            const char* e = std::getenv("LATTICE_FM_YRES");
            return e ? std::atoi(e) : 1;
        }();
        Plan pr = pl;
        pr.p.y_res = 0;
        if (yres_env) {
            Params q = pl.p;
            q.y_res = 1;
            if (GeoL(q).wl_stages >= 3) pr.p.y_res = 1;
        }
        LAT_CUDA(launch_pdl(fm_lcb_large_kernel, grid, kLargeThreads, smem_bytes(pr.p), st, pr));
        LAT_CUDA(cudaGetLastError());
        return LATTICE_OK;
    }
    return pl.p.f32 ? launch_t<float>(pl, st) : launch_t<__nv_bfloat16>(pl, st);
}

int wl_rows(const Params& p) { return p.nL > 128 ? 256 : 128; }

}  // namespace fm
}  // namespace lat

// ---------------------------------------------------------------------------------------------
// lattice_fm_lcb: K2 on its own (tests and callers composing their own blocks). Y^T and W_L come
// unpadded from the caller and are copied into the zero-padded layout the tensor maps expect.
// ---------------------------------------------------------------------------------------------
extern "C" lattice_status lattice_fm_lcb(const lattice_fm_lcb_args* a, lattice_stream stream) {
    using namespace lat;
    LAT_REQUIRE(a != nullptr, "lattice_fm_lcb: null args");
    LAT_REQUIRE(a->batch >= 0 && a->batch < (1ll << 31), "lattice_fm_lcb: bad batch");
    LAT_REQUIRE(a->dtype == LATTICE_BF16 || a->dtype == LATTICE_F32, "lattice_fm_lcb: dtype must be bf16 or f32");
    LAT_REQUIRE(a->n >= 1 && a->n <= 512 && a->k >= 1 && a->k <= 64 && a->nF >= 1 && a->nL >= 0 &&
                    a->nF + a->nL == a->n,
                "lattice_fm_lcb: need 1 <= n <= 512, 1 <= k <= 64, nF >= 1, nF + nL == n");
    if (a->batch == 0) return LATTICE_OK;
    LAT_REQUIRE(a->X && a->YT && a->Fin && a->Xout && (a->nL == 0 || a->WL), "lattice_fm_lcb: null pointer");
    const cudaStream_t st = (cudaStream_t)stream;
    fm::Plan pl = {};
    fm::Params& p = pl.p;
    p.B = a->batch;
    p.n = a->n;
    p.d = a->d;
    p.k = a->k;
    p.nF = a->nF;
    p.nL = a->nL;
    p.n_pad = a->n > 256 ? (a->n + 255) / 256 * 256 : (a->n + 15) / 16 * 16;
    p.k_pad = (a->k + 15) / 16 * 16;
    p.tmem_cols = 512;
    p.f32 = a->dtype == LATTICE_F32 ? 1 : 0;
    p.Fout = a->Fin;
    p.Xout = a->Xout;
    p.Xin = a->X;
    lattice_status s = fm::check(p);
    if (s != LATTICE_OK) return s;
    const size_t es = p.f32 ? 4 : 2;
    const int wr = fm::wl_rows(p);
    const size_t yt_bytes = es * (size_t)p.k_pad * p.n_pad, wl_bytes = es * (size_t)wr * p.n_pad;
    uint8_t* ws = nullptr;
    LAT_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ws), yt_bytes + wl_bytes, st));
    auto body = [&]() -> lattice_status {
        LAT_CUDA(cudaMemsetAsync(ws, 0, yt_bytes + wl_bytes, st));
        LAT_CUDA(cudaMemcpy2DAsync(ws, es * p.n_pad, a->YT, es * p.n, es * p.n, p.k, cudaMemcpyDeviceToDevice, st));
        if (p.nL > 0)
            LAT_CUDA(cudaMemcpy2DAsync(ws + yt_bytes, es * p.n_pad, a->WL, es * p.n, es * p.n, p.nL,
                                       cudaMemcpyDeviceToDevice, st));
        lattice_status r = fm::make_maps(&pl, a->X, ws + yt_bytes, ws);
        if (r != LATTICE_OK) return r;
        const char* tr = std::getenv("LATTICE_FM_TRACE");
        if (!(tr && std::atoi(tr) && fm::is_large(p))) return fm::launch(pl, st);
        // wait-site profile of the large variant: cycles per site averaged over CTAs, to stderr
        const int grid = (int)(p.B < num_sms() ? p.B : num_sms());
        LAT_CUDA(cudaMalloc(&pl.p.trace, sizeof(unsigned long long) * 16 * grid));
        LAT_CUDA(cudaMemset(pl.p.trace, 0, sizeof(unsigned long long) * 16 * grid));
        r = fm::launch(pl, st);
        std::vector<unsigned long long> h((size_t)16 * grid);
        cudaMemcpy(h.data(), pl.p.trace, h.size() * sizeof(h[0]), cudaMemcpyDeviceToHost);
        cudaFree(pl.p.trace);
        const bool pair = fm::is_pair(p);
        const char* names[11] = {"mma:l_empty", "mma:x_full", "mma:yt_full", "mma:wl_full", "mma:pbuf_full",
                                 "mma:f_empty", "mma:total", pair ? "passes" : "samples", "xprod:x_empty",
                                 pair ? "lcb:own_epi" : "wprod:yt_empty", pair ? "lcb:partner_epi" : "wprod:wl_empty"};
        for (int i = 0; i < 11; ++i) {
            double sum = 0;
            for (int b = 0; b < grid; ++b) sum += (double)h[(size_t)b * 16 + i];
            std::fprintf(stderr, "[fm_trace] %-16s %14.0f\n", names[i], sum / grid);
        }
        return r;
    };
    s = body();
    cudaFreeAsync(ws, st);
    return s;
}
