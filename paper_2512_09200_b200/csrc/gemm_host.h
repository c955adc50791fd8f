// gemm_host.h -- host-side plan/launch interface of the tcgen05 GEMM (used by network.cu).
#pragma once

#include <cuda.h>

#include "gemm.cuh"

namespace lat {
namespace gemm {

struct GemmPlan {
    CUtensorMap ta, tb;
    Params p;
    int grid_y;
    int stages;
    bool f32;      // fp32 operands on the TF32 tensor path
    bool two_cta;  // CTA-pair (cta_group::2) kernel: B tensor map boxes are BN/2 rows
};

lattice_status make_map_2d(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer,
                           uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer,
                           bool f32 = false);
// A: [a_rows][K] (row stride lda elements), B: [b_rows][K]; tiles of 128 x 256.
lattice_status plan(GemmPlan* g, const void* A, int64_t lda, int64_t a_rows, const void* B,
                    int64_t ldb, int64_t b_rows, const Params& p, int grid_y, bool f32 = false);
lattice_status launch(const GemmPlan& g, cudaStream_t st);

}  // namespace gemm
}  // namespace lat
