// backward.cu -- SURVEY.md 8f rank 4: the backward pass of the network's trainable head.
//
//   lattice_rownorm_vjp        J(x)^T g for rms_norm / swish_rn / swish_rn_hard rows (the adjoint
//                              of the reference's swish_rn_jvp, numerics.hpp:113-136), fp32 / fp64
//   lattice_routed_bce         window-routed binary cross-entropy of the heads (PAPER.md:142-144:
//                              each sample trains only its Zipper-assigned window's head) and its
//                              gradient w.r.t. the logits
//   lattice_net_tower_backward gradients of the untied per-domain towers (W1_g, W2_g) and of the
//                              towers' input X_L, from d(loss)/d(logits), after a forward:
//                                z = W1_g x  (recomputed, tcgen05 GEMM, fp32)
//                                h = swish_rn(z);   dW2_g = sum_b dlogit_b h_b^T
//                                dz = J_swish(z)^T (W2_g^T dlogit)     (stored bf16, the GEMM operand)
//                                dW1_g = dz_g^T X_g   (tcgen05 GEMM, both operands MN-major in place)
//                                dX    = dz W1_g      (tcgen05 GEMM, W1_g MN-major in place)
//   lattice_net_mlp_backward   gradients of the last DWFB block's FMB half: its
//                              MLP weights, the MLP input Fin and the residual branch, from
//                              d(loss)/d(X_L) (e.g. the towers' dX):
//                                U = z_last + X[:nF];  dz_last = J_rmsnorm_d(U)^T dX_L[:nF]
//                                per layer i (last to first): dW_i = dz_i^T a_i;  da_i = dz_i W_i
//                                dz_{i-1} = J_swish(z_{i-1})^T da_i  (z recomputed by fp32 GEMMs)
// Every reduction runs in a fixed order (per-chunk partials, then a fixed-order sum): gradients are
// deterministic, so data-parallel replicas that all-reduce them stay bit-identical.
#include <cuda_bf16.h>
#include <nvtx3/nvToolsExt.h>

#include <string>
#include <vector>

#include "backward.h"
#include "common.cuh"
#include "gemm_host.h"

namespace lat {
namespace {

constexpr int kMaxHeadsB = 16;

__device__ __forceinline__ float sigmoidf_(float z) { return 1.0f / (1.0f + __expf(-z)); }
__device__ __forceinline__ double sigmoid_(double z) {  // numerics.hpp:29-33
    if (z >= 0.0) return 1.0 / (1.0 + exp(-z));
    const double e = exp(z);
    return e / (1.0 + e);
}
__device__ __forceinline__ float sig(float z) { return sigmoidf_(z); }
__device__ __forceinline__ double sig(double z) { return sigmoid_(z); }

// d(out_i)/d(r_i) of the activation on the normalised row: 1 (rms_norm), s(1 + r(1 - s)) (swish,
// numerics.hpp:133-134), and the hard gate's r * clamp((r+3)/6, 0, 1) derivative
template <typename T>
__device__ __forceinline__ T act_grad(int mode, T r) {
    if (mode == 0) return T(1);
    if (mode == 1) {
        const T s = sig(r);
        return s * (T(1) + r * (T(1) - s));
    }
    if (r <= T(-3)) return T(0);
    if (r >= T(3)) return T(1);
    return (T(2) * r + T(3)) / T(6);
}

// warp per row: J^T g = u/d - x (x . u) / (n d^3), u_i = act'(r_i) g_i, r = x/d, d = sqrt(mean(x^2)+eps)
template <typename TO, typename T>
__device__ __forceinline__ TO store_as(T v) {
    if constexpr (sizeof(TO) == 2) return __float2bfloat16_rn((float)v);
    else return (TO)v;
}

template <typename T, typename TO = T>
__global__ void rownorm_vjp_kernel(int mode, int64_t rows, int64_t width, T eps, const T* __restrict__ x,
                                   const T* __restrict__ g, TO* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < rows;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const T* xr = x + r * width;
        const T* gr = g + r * width;
        T ss = 0;
        for (int64_t c = lane; c < width; c += 32) ss += xr[c] * xr[c];
        for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
        const T n = (T)width;
        const T d = sqrt(ss / n + eps);
        T dot = 0;
        for (int64_t c = lane; c < width; c += 32) dot += xr[c] * act_grad<T>(mode, xr[c] / d) * gr[c];
        for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
        const T k = dot / (n * d * d * d);
        for (int64_t c = lane; c < width; c += 32)
            out[r * width + c] = store_as<TO>(act_grad<T>(mode, xr[c] / d) * gr[c] / d - xr[c] * k);
    }
}

// Routed BCE: loss_b = sum_t bce(logit[b][t*W + w_b], label[b][t][w_b]) / (n*T); dlogit for the
// routed heads only. Per-block fixed-order partial sums of the loss.
__global__ void routed_bce_kernel(int64_t n, int T, int W, const float* __restrict__ logits,
                                  const uint8_t* __restrict__ window, const uint8_t* __restrict__ labels,
                                  float* __restrict__ dlogits, double* __restrict__ part) {
    __shared__ double red[256];
    double acc = 0.0;
    const double inv = 1.0 / ((double)n * T);
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < n; b += (int64_t)gridDim.x * blockDim.x) {
        const int w = window[b] < W ? window[b] : W - 1;
        for (int t = 0; t < T; ++t) {
            const float z = logits[b * T * W + t * W + w];
            const float y = labels[(b * T + t) * W + w] ? 1.0f : 0.0f;
            // log(1 + e^-|z|) + max(z, 0) - z y  (stable)
            acc += (double)(log1pf(__expf(-fabsf(z))) + fmaxf(z, 0.0f) - z * y);
            for (int v = 0; v < W; ++v)
                dlogits[b * T * W + t * W + v] = v == w ? (float)((sigmoidf_(z) - y) * inv) : 0.0f;
        }
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void sum_parts_kernel(int parts, const double* __restrict__ part, double scale, double* __restrict__ out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < parts; ++i) s += part[i];
        *out = s * scale;
    }
}

// One warp per sorted row m (domain g): h = swish_rn(z[m]) (fp32, kept for dW2), dh = W2_g^T
// dlogit[order[m]], dz = J(z)^T dh -> bf16 (the dW1 / dX GEMM operand). th <= 2048.
__global__ void tower_dz_kernel(int64_t B, int th, int heads, int hard, const float* __restrict__ z,
                                const int32_t* __restrict__ order, const int32_t* __restrict__ seg, int G,
                                const float* __restrict__ dlogits, const float* __restrict__ W2,
                                float* __restrict__ h_out, __nv_bfloat16* __restrict__ dz) {
    const int lane = threadIdx.x & 31;
    const int mode = hard ? 2 : 1;
    for (int64_t m = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; m < B;
         m += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        int g = 0;
        while (g + 1 < G && seg[g + 1] <= m) ++g;
        const float* zr = z + m * th;
        const float* dl = dlogits + (int64_t)order[m] * heads;
        const float* w2 = W2 + (int64_t)g * heads * th;
        float ss = 0.0f;
        for (int c = lane; c < th; c += 32) ss += zr[c] * zr[c];
        ss = warp_sum(ss);
        const float d = sqrtf(ss / (float)th + 1e-6f);
        float dot = 0.0f;
        for (int c = lane; c < th; c += 32) {
            float dh = 0.0f;
            for (int k = 0; k < heads; ++k) dh += dl[k] * w2[(int64_t)k * th + c];
            const float r = zr[c] / d;
            h_out[m * th + c] = mode == 1 ? r * sigmoidf_(r) : r * fminf(fmaxf((r + 3.0f) / 6.0f, 0.0f), 1.0f);
            dot += zr[c] * act_grad<float>(mode, r) * dh;
        }
        dot = warp_sum(dot);
        const float k = dot / ((float)th * d * d * d);
        for (int c = lane; c < th; c += 32) {
            float dh = 0.0f;
            for (int q = 0; q < heads; ++q) dh += dl[q] * w2[(int64_t)q * th + c];
            dz[m * th + c] = __float2bfloat16_rn(act_grad<float>(mode, zr[c] / d) * dh / d - zr[c] * k);
        }
    }
}

// Residual rms_norm_d of the FMB half: warp per (sample, row f < nF) of d <= 128 values,
// U = z_last + X_in, g = dX_out (row stride nd); dU = g/s - U (U . g) / (d s^3), s = sqrt(mean(U^2)+eps)
// -> bf16 (the MLP backward's GEMM operand) and optionally fp32 (the residual branch's gradient)
__global__ void resid_vjp_kernel(int64_t B, int nF, int d, int64_t nd, const float* __restrict__ z,
                                 const __nv_bfloat16* __restrict__ Xin, const float* __restrict__ dXout,
                                 __nv_bfloat16* __restrict__ dz, float* __restrict__ dResid) {
    const int lane = threadIdx.x & 31;
    const int64_t rows = B * nF, w = (int64_t)nF * d;
    for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < rows;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t b = r / nF, f = r - b * nF;
        const float* zr = z + b * w + f * d;
        const __nv_bfloat16* xr = Xin + b * nd + f * d;
        const float* gr = dXout + b * nd + f * d;
        float u[4], gv[4], ss = 0.0f, dot = 0.0f;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int c = lane + 32 * i;
            u[i] = c < d ? zr[c] + __bfloat162float(xr[c]) : 0.0f;
            gv[i] = c < d ? gr[c] : 0.0f;
            ss += u[i] * u[i];
            dot += u[i] * gv[i];
        }
        ss = warp_sum(ss);
        dot = warp_sum(dot);
        const float s = sqrtf(ss / (float)d + 1e-6f);
        const float k = dot / ((float)d * s * s * s);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int c = lane + 32 * i;
            if (c >= d) continue;
            const float o = gv[i] / s - u[i] * k;
            dz[b * w + f * d + c] = __float2bfloat16_rn(o);
            if (dResid) dResid[b * w + f * d + c] = o;
        }
    }
}

// dW2_g[k][j] = sum_{m in segment g} dlogit[order[m]][k] h[m][j]: thread per (g, j), rows in
// chunks of `chunk` (partials [G][chunks][heads][th]), then a fixed-order sum over chunks
__global__ void dw2_partial_kernel(int th, int heads, int G, int chunk, int chunks, const int32_t* __restrict__ seg,
                                   const int32_t* __restrict__ order, const float* __restrict__ dlogits,
                                   const float* __restrict__ h, float* __restrict__ part) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int g = blockIdx.y, ck = blockIdx.z;
    if (j >= th) return;
    float acc[kMaxHeadsB];
    for (int k = 0; k < kMaxHeadsB; ++k) acc[k] = 0.0f;
    const int m0 = seg[g] + ck * chunk, m1 = min(seg[g + 1], m0 + chunk);
    for (int m = m0; m < m1; ++m) {
        const float hv = h[(int64_t)m * th + j];
        const float* dl = dlogits + (int64_t)order[m] * heads;
        for (int k = 0; k < heads; ++k) acc[k] += dl[k] * hv;
    }
    for (int k = 0; k < heads; ++k) part[(((int64_t)g * chunks + ck) * heads + k) * th + j] = acc[k];
}

__global__ void dw2_sum_kernel(int th, int heads, int G, int chunks, const float* __restrict__ part,
                               float* __restrict__ dW2) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // over G*heads*th
    if (i >= (int64_t)G * heads * th) return;
    const int64_t g = i / ((int64_t)heads * th), r = i - g * heads * th;
    float s = 0.0f;
    for (int ck = 0; ck < chunks; ++ck) s += part[((g * chunks + ck) * heads) * th + r];
    dW2[i] = s;
}

// master -= lr * grad (fp32), and the network's working copy refreshed in its storage dtype
template <typename TO>
__global__ void sgd_kernel(int64_t n, float lr, const float* __restrict__ grad, float* __restrict__ master,
                           TO* __restrict__ work) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float w = master[i] - lr * grad[i];
        master[i] = w;
        if constexpr (sizeof(TO) == 2) work[i] = __float2bfloat16_rn(w);
        else work[i] = w;
    }
}

unsigned grid_for_rows(int64_t rows) {
    const int64_t b = (rows * 32 + 255) / 256;
    const int64_t cap = (int64_t)num_sms() * 16;
    return (unsigned)(b < 1 ? 1 : (b > cap ? cap : b));
}

// C [M][N] = op(A) op(B)^T over K (fp32 accumulate, plain store); a_mn / b_mn: the operand is
// stored [K][M] / [K][N] (read in place as an MN-major tcgen05 operand)
lattice_status gemm_store(const void* A, int64_t lda, int64_t M, int a_mn, const void* Bm, int64_t ldb, int64_t N,
                          int b_mn, int64_t K, void* C, int64_t ldc, int out_bf16, cudaStream_t st) {
    gemm::Params p = {};
    p.M = (int)M;
    p.N = (int)N;
    p.K = (int)K;
    p.C = C;
    p.ldc = ldc;
    p.out_bf16 = out_bf16;
    p.epi = gemm::kStore;
    p.N_full = (int)N;
    p.cluster = 1;
    p.a_mn = a_mn;
    p.b_mn = b_mn;
    gemm::GemmPlan gp;
    lattice_status s = gemm::plan(&gp, A, lda, M, Bm, ldb, N, p, (int)((M + 127) / 128), false);
    if (s != LATTICE_OK) return s;
    return gemm::launch(gp, st);
}

}  // namespace

lattice_status sgd_update(int64_t n, float lr, const float* grad, float* master, void* work, bool work_bf16,
                          cudaStream_t st) {
    if (n <= 0) return LATTICE_OK;
    const unsigned grid = (unsigned)((n + 255) / 256 < (int64_t)num_sms() * 32 ? (n + 255) / 256 : num_sms() * 32);
    if (work_bf16)
        sgd_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(n, lr, grad, master, static_cast<__nv_bfloat16*>(work));
    else
        sgd_kernel<float><<<grid, 256, 0, st>>>(n, lr, grad, master, static_cast<float*>(work));
    LAT_CUDA(cudaGetLastError());
    return LATTICE_OK;
}

// The towers' backward (see the file header); called by lattice_net_tower_backward (network.cu).
lattice_status tower_backward(const TowerBwd& a, cudaStream_t st) {
    nvtxRangePushA("lattice::tower_backward");
    struct Pop {
        ~Pop() { nvtxRangePop(); }
    } pop;
    const int64_t B = a.B;
    const int G = a.G, th = a.th, heads = a.heads;
    const int64_t nd = a.nd;
    std::vector<int32_t> seg(G + 1);
    LAT_CUDA(cudaMemcpyAsync(seg.data(), a.seg, sizeof(int32_t) * (G + 1), cudaMemcpyDeviceToHost, st));
    LAT_CUDA(cudaStreamSynchronize(st));
    const int chunk = 256;
    int chunks = 1;
    for (int g = 0; g < G; ++g) {
        const int c = (seg[g + 1] - seg[g] + chunk - 1) / chunk;
        chunks = c > chunks ? c : chunks;
    }
    const size_t zb = sizeof(float) * (size_t)B * th, db = sizeof(__nv_bfloat16) * (size_t)B * th;
    const size_t pb = sizeof(float) * (size_t)G * chunks * heads * th;
    uint8_t* ws = nullptr;
    const bool own = !a.scratch;
    if (own) {
        LAT_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ws), 2 * zb + db + pb, st));
    } else {
        ws = static_cast<uint8_t*>(a.scratch(2 * zb + db + pb));
        LAT_REQUIRE(ws != nullptr, "tower_backward: workspace allocation failed");
    }
    float* z = reinterpret_cast<float*>(ws);
    float* h = reinterpret_cast<float*>(ws + zb);
    __nv_bfloat16* dz = reinterpret_cast<__nv_bfloat16*>(ws + 2 * zb);
    float* part = reinterpret_cast<float*>(ws + 2 * zb + db);
    auto run = [&]() -> lattice_status {
        const __nv_bfloat16* X = static_cast<const __nv_bfloat16*>(a.X);
        const __nv_bfloat16* W1 = static_cast<const __nv_bfloat16*>(a.W1);
        for (int g = 0; g < G; ++g) {  // z = X_g W1_g^T (fp32): the pre-activation the forward did not keep
            const int64_t rows = seg[g + 1] - seg[g];
            if (rows == 0) continue;
            lattice_status s = gemm_store(X + (int64_t)seg[g] * nd, nd, rows, 0, W1 + (int64_t)g * th * nd, nd, th, 0,
                                          nd, z + (int64_t)seg[g] * th, th, 0, st);
            if (s != LATTICE_OK) return s;
        }
        tower_dz_kernel<<<grid_for_rows(B), 256, 0, st>>>(B, th, heads, a.hard, z, a.order, a.seg, G, a.dlogits, a.W2,
                                                           h, dz);
        LAT_CUDA(cudaGetLastError());
        dw2_partial_kernel<<<dim3((th + 127) / 128, G, chunks), 128, 0, st>>>(th, heads, G, chunk, chunks, a.seg,
                                                                               a.order, a.dlogits, h, part);
        const int64_t nw2 = (int64_t)G * heads * th;
        dw2_sum_kernel<<<(unsigned)((nw2 + 255) / 256), 256, 0, st>>>(th, heads, G, chunks, part, a.dW2);
        LAT_CUDA(cudaGetLastError());
        for (int g = 0; g < G; ++g) {
            const int64_t rows = seg[g + 1] - seg[g];
            float* dW1g = a.dW1 + (int64_t)g * th * nd;
            if (rows == 0) {
                LAT_CUDA(cudaMemsetAsync(dW1g, 0, sizeof(float) * (size_t)th * nd, st));
                continue;
            }
            // dW1_g [th][nd] = dz_g^T X_g: both operands stored with the batch rows as K (MN-major)
            lattice_status s = gemm_store(dz + (int64_t)seg[g] * th, th, th, 1, X + (int64_t)seg[g] * nd, nd, nd, 1,
                                          rows, dW1g, nd, 0, st);
            if (s != LATTICE_OK) return s;
            if (a.dX) {  // dX_g [rows][nd] = dz_g W1_g: W1_g stored [th][nd] is the MN-major B operand
                void* C = a.dx_bf16 ? (void*)(static_cast<__nv_bfloat16*>(a.dX) + (int64_t)seg[g] * nd)
                                    : (void*)(static_cast<float*>(a.dX) + (int64_t)seg[g] * nd);
                s = gemm_store(dz + (int64_t)seg[g] * th, th, rows, 0, W1 + (int64_t)g * th * nd, nd, nd, 1, th, C, nd,
                               a.dx_bf16, st);
                if (s != LATTICE_OK) return s;
            }
        }
        return LATTICE_OK;
    };
    const lattice_status s = run();
    if (own) cudaFreeAsync(ws, st);
    return s;
}

// The FMB half's backward (see the file header); called by lattice_net_mlp_backward (network.cu).
lattice_status mlp_backward(const MlpBwd& a, cudaStream_t st) {
    nvtxRangePushA("lattice::mlp_backward");
    struct Pop {
        ~Pop() { nvtxRangePop(); }
    } pop;
    const int64_t B = a.B;
    const int L = a.n_mlp;
    int64_t wmax = 0;
    for (int i = 1; i <= L; ++i) wmax = a.widths[i] > wmax ? a.widths[i] : wmax;
    const size_t fb = sizeof(float) * (size_t)B * wmax, hb = sizeof(__nv_bfloat16) * (size_t)B * wmax;
    uint8_t* ws = nullptr;
    const bool own = !a.scratch;
    if (own) {
        LAT_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ws), 2 * fb + hb, st));
    } else {
        ws = static_cast<uint8_t*>(a.scratch(2 * fb + hb));
        LAT_REQUIRE(ws != nullptr, "mlp_backward: workspace allocation failed");
    }
    float* z = reinterpret_cast<float*>(ws);           // a pre-activation [B][w] (recomputed)
    float* da = reinterpret_cast<float*>(ws + fb);     // d(loss)/d(a_i) [B][w_i]
    __nv_bfloat16* dz = reinterpret_cast<__nv_bfloat16*>(ws + 2 * fb);  // d(loss)/d(z_i), bf16
    auto run = [&]() -> lattice_status {
        const int64_t wl = a.widths[L];  // nF * d
        // z_last = a_{L-1} W_{L-1}^T; dz_last = J_rmsnorm_d(z_last + X[:nF])^T dX_L[:nF]
        lattice_status s = gemm_store(a.act[L - 1], a.widths[L - 1], B, 0, a.W[L - 1], a.widths[L - 1], wl, 0,
                                      a.widths[L - 1], z, wl, 0, st);
        if (s != LATTICE_OK) return s;
        resid_vjp_kernel<<<grid_for_rows(B * a.nF), 256, 0, st>>>(B, a.nF, a.d, a.nd, z,
                                                                   static_cast<const __nv_bfloat16*>(a.Xin), a.dXout,
                                                                   dz, a.dResid);
        LAT_CUDA(cudaGetLastError());
        for (int i = L - 1; i >= 0; --i) {
            const int64_t in = a.widths[i], out = a.widths[i + 1];
            // dW_i [out][in] = dz_i^T a_i: both stored with the batch rows as K (MN-major)
            s = gemm_store(dz, out, out, 1, a.act[i], in, in, 1, B, a.dW[i], in, 0, st);
            if (s != LATTICE_OK) return s;
            if (i == 0 && !a.dFin) break;
            // da_i [B][in] = dz_i W_i: W_i stored [out][in] is the MN-major B operand
            s = gemm_store(dz, out, B, 0, a.W[i], in, in, 1, out, i == 0 ? a.dFin : da, in, 0, st);
            if (s != LATTICE_OK) return s;
            if (i == 0) break;
            // z_{i-1} = a_{i-1} W_{i-1}^T (fp32), dz_{i-1} = J_act(z_{i-1})^T da_i -> bf16
            const int64_t pin = a.widths[i - 1];
            s = gemm_store(a.act[i - 1], pin, B, 0, a.W[i - 1], pin, in, 0, pin, z, in, 0, st);
            if (s != LATTICE_OK) return s;
            rownorm_vjp_kernel<float, __nv_bfloat16><<<grid_for_rows(B), 256, 0, st>>>(a.hard ? 2 : 1, B, in, 1e-6f,
                                                                                       z, da, dz);
            LAT_CUDA(cudaGetLastError());
        }
        return LATTICE_OK;
    };
    const lattice_status s = run();
    if (own) cudaFreeAsync(ws, st);
    return s;
}

}  // namespace lat

extern "C" {

lattice_status lattice_rownorm_vjp(int32_t mode, int64_t rows, int64_t width, double eps, int32_t dtype,
                                   const void* x, const void* g, void* out, lattice_stream stream) {
    using namespace lat;
    LAT_REQUIRE(mode >= 0 && mode <= 2, "rownorm_vjp: mode must be 0, 1 or 2");
    LAT_REQUIRE(eps > 0.0, "eps must be > 0");
    LAT_REQUIRE(width > 0, "rownorm_vjp: empty input");
    LAT_REQUIRE(dtype == LATTICE_F32 || dtype == LATTICE_F64, "rownorm_vjp: dtype must be f32 or f64");
    if (rows <= 0) return LATTICE_OK;
    LAT_REQUIRE(x && g && out, "rownorm_vjp: null pointer");
    const cudaStream_t st = (cudaStream_t)stream;
    if (dtype == LATTICE_F64)
        rownorm_vjp_kernel<double><<<grid_for_rows(rows), 256, 0, st>>>(
            mode, rows, width, eps, static_cast<const double*>(x), static_cast<const double*>(g),
            static_cast<double*>(out));
    else
        rownorm_vjp_kernel<float><<<grid_for_rows(rows), 256, 0, st>>>(
            mode, rows, width, (float)eps, static_cast<const float*>(x), static_cast<const float*>(g),
            static_cast<float*>(out));
    LAT_CUDA(cudaGetLastError());
    return LATTICE_OK;
}

lattice_status lattice_routed_bce(int64_t n, int32_t tasks, int32_t windows, const float* logits,
                                  const uint8_t* window, const uint8_t* labels, float* dlogits, double* loss,
                                  lattice_stream stream) {
    using namespace lat;
    LAT_REQUIRE(n >= 0 && tasks >= 1 && windows >= 1, "routed_bce: bad sizes");
    LAT_REQUIRE(loss != nullptr, "routed_bce: null loss");
    const cudaStream_t st = (cudaStream_t)stream;
    if (n == 0) {
        LAT_CUDA(cudaMemsetAsync(loss, 0, sizeof(double), st));
        return LATTICE_OK;
    }
    LAT_REQUIRE(logits && window && labels && dlogits, "routed_bce: null pointer");
    const int blocks = (int)((n + 255) / 256 < 1024 ? (n + 255) / 256 : 1024);
    double* part = nullptr;
    LAT_CUDA(cudaMallocAsync(&part, sizeof(double) * blocks, st));
    routed_bce_kernel<<<blocks, 256, 0, st>>>(n, tasks, windows, logits, window, labels, dlogits, part);
    sum_parts_kernel<<<1, 32, 0, st>>>(blocks, part, 1.0 / ((double)n * tasks), loss);
    cudaError_t e = cudaGetLastError();
    cudaFreeAsync(part, st);
    LAT_CUDA(e);
    return LATTICE_OK;
}

}  // extern "C"
