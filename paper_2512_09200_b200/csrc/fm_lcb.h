// fm_lcb.h -- host interface of the fused FM/LCB kernel (fm_lcb.cu).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>

#include "common.cuh"

namespace lat {
namespace fm {

struct Params {
    int64_t B;
    int n, d, k, nF, nL;
    int n_pad, k_pad;       // multiples of 16
    int tmem_cols;          // informational (the kernel sizes its own allocation)
    int f32;                // 1: fp32 storage, kind::tf32 MMAs; 0: bf16, kind::f16
    const void* Xin;        // [B][n][d], the X the tensor map reads (the large variant's LCB
                            // residual rows come from here, L2-resident, instead of shared memory)
    void* Fout;             // [B][n*k]
    void* Xout;             // [B][n][d], rows nF .. n-1 written
    unsigned long long* trace;  // optional [grid][16] cycles spent per wait site (LATTICE_FM_TRACE=1)
    int y_res;              // large variant: Y^T resident in smem (set at launch when it fits)
};

struct Plan {
    CUtensorMap tmX, tmWL, tmYT;
    Params p;
};

// X: [B][n][d]. WLpad: [wl_rows][n_pad] (rows >= nL zero). YTpad: [k_pad][n_pad]. Same dtype.
lattice_status check(const Params& p);
lattice_status make_maps(Plan* pl, const void* X, const void* WLpad, const void* YTpad);
lattice_status launch(const Plan& pl, cudaStream_t st);
size_t smem_bytes(const Params& p);
// rows of the padded W_L buffer the plan expects: 128 (nL <= 128) or 256
int wl_rows(const Params& p);

}  // namespace fm
}  // namespace lat
