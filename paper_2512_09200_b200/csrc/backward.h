// backward.h -- host interface of the towers' backward (backward.cu), used by network.cu.
#pragma once

#include <functional>

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/lattice_b200.h"

namespace lat {

struct TowerBwd {
    int64_t B;                 // batch rows (domain-sorted, as the forward left them)
    int G, th, heads, hard;
    int64_t nd;                // n * d: the towers' input width
    const void* X;             // bf16 [B][nd] X_L, domain-sorted rows
    const void* W1;            // bf16 [G*th][nd]
    const float* W2;           // [G][heads][th]
    const int32_t* order;      // sorted row -> caller sample
    const int32_t* seg;        // DEVICE [G+1] domain segment starts
    const float* dlogits;      // [B][heads], caller order
    float* dW1;                // out [G][th][nd]
    float* dW2;                // out [G][heads][th]
    void* dX;                  // optional out [B][nd], domain-sorted rows
    int dx_bf16;
    // scratch provider (the network's persistent workspace, grown on demand); null: stream-ordered
    // cudaMallocAsync per call
    std::function<void*(size_t)> scratch;
};

lattice_status tower_backward(const TowerBwd& a, cudaStream_t st);

struct MlpBwd {
    int64_t B;                 // batch rows (domain-sorted)
    int n_mlp;
    int widths[6];             // mlp[0..n_mlp]: n*k, hidden..., nF*d
    int nF, d, hard;
    int64_t nd;                // n * d: row stride of X_in / dXout
    const void* act[5];        // bf16 [B][widths[i]]: layer i's input (act[0] = Fin)
    const void* W[5];          // bf16 [widths[i+1]][widths[i]]
    const void* Xin;           // bf16 [B][nd]: the block's input (the residual)
    const float* dXout;        // [B][nd]: d(loss)/d(block output), columns [0, nF*d) used
    float* dW[5];              // out [widths[i+1]][widths[i]]
    float* dFin;               // optional out [B][widths[0]]
    float* dResid;             // optional out [B][nF*d]
    std::function<void*(size_t)> scratch;  // as TowerBwd::scratch
};

lattice_status mlp_backward(const MlpBwd& a, cudaStream_t st);
// master -= lr * grad (n fp32 values); work (the network's copy) refreshed in bf16 or fp32
lattice_status sgd_update(int64_t n, float lr, const float* grad, float* master, void* work, bool work_bf16,
                          cudaStream_t st);

}  // namespace lat
