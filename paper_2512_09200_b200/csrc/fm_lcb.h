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
    int tmem_cols;          // 256 or 512
    __nv_bfloat16* Fout;    // [B][n*k]
    __nv_bfloat16* Xout;    // [B][n][d], rows nF .. n-1 written
};

struct Plan {
    CUtensorMap tmX, tmWL, tmYT;
    Params p;
};

// X: [B][n][d] bf16. WLpad: [128][n_pad] bf16 (rows >= nL zero). YTpad: [k_pad][n_pad] bf16.
lattice_status check(const Params& p);
lattice_status make_maps(Plan* pl, const void* X, const void* WLpad, const void* YTpad);
lattice_status launch(const Plan& pl, cudaStream_t st);
size_t smem_bytes(const Params& p);

}  // namespace fm
}  // namespace lat
