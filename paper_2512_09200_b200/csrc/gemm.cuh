// gemm.cuh -- K3/K4: bf16 GEMM on 5th-gen tensor cores with fused Lattice epilogues.
//
//   C[M][N] = A[M][K] . B[N][K]^T      (A activations, B weights stored out x in)
//
// One CTA computes a 128 x BN tile: warp 0 streams A/B k-blocks (128B-swizzled, BK = 64)
// with TMA into an STAGES-deep mbarrier ring; warp 1 (one elected lane) issues
// tcgen05.mma.cta_group::1.kind::f16 (M=128, N=BN, K=16) into a TMEM accumulator of BN fp32
// columns; warps 2-5 drain TMEM with tcgen05.ld (thread = accumulator row) and run the
// epilogue:
//   STORE       bf16 / fp32 store
//   SWISH(_HARD) swish_rn over the FULL output row (numerics.hpp:94-107). Rows wider than
//               one tile are covered by a thread-block cluster along N; per-row sums of
//               squares are exchanged through distributed shared memory (st.shared::cluster
//               + remote mbarrier arrive), summed in rank order.
//   RESID_NORM  X' = rms_norm_group(acc + X) per `group` columns (the block combine, a13)
//   TOWER       swish_rn over the full row, then heads = W2_g . h on CUDA cores, partial
//               head sums reduced across the cluster into rank 0, written un-permuted.
// Grouped mode (towers): blockIdx.y indexes a device tile table {group, row0, row_end};
// B rows come from the group's slice of a stacked [G*N][K] weight.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>

#include "common.cuh"
#include "tc.cuh"

namespace lat {
namespace gemm {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kThreads = 192;
constexpr int kMaxCluster = 8;
constexpr int kMaxHeads = 16;

enum Epi : int { kStore = 0, kSwish = 1, kSwishHard = 2, kResidNorm = 3, kTower = 4, kTowerHard = 5 };

struct Params {
    int M, N, K;
    void* C;
    int64_t ldc;
    int out_bf16;
    int epi;
    const void* resid;   // same dtype as the output (bf16 or fp32)
    int64_t ldr;
    int group;
    int cluster;         // CTAs along N sharing a row (row-norm epilogues)
    int N_full;          // width of the normalised row (= N)
    // CTA-pair swish epilogue: per-row partial sums of squares of every N-tile ([M][N-tiles])
    // and per (256-row block, CTA half) arrival counters, exchanged through global memory
    float* rowpart;
    int* rowcnt;
    int rowcnt_zeroed;   // 1: the caller zeroed rowcnt for this launch (no memset between kernels)
    // grouped
    const int4* tiles;   // {group, row0, row_end, 0}; nullptr = dense
    const int* n_tiles;
    int b_rows_per_group;
    // tower heads
    const float* W2;     // [G][heads][N] fp32
    int heads;
    const int32_t* order;  // sorted row -> original sample
    float* logits;         // [B][heads]
    // operand majorness (single-CTA kernel, bf16 only): 0 K-major (A [M][K], B [N][K]); 1 MN-major
    // (A stored [K][M], B stored [K][N]: the transposed operands of a backward pass, read in place)
    int a_mn, b_mn;
};

__host__ __device__ inline size_t smem_bytes(int BN, int stages, int cluster, int heads) {
    size_t s = 1024;                                    // alignment slack
    s += (size_t)stages * (BM * BK * 2 + BN * BK * 2);  // operand ring
    s += 256;                                           // barriers + tmem slot
    s += (size_t)kMaxCluster * BM * 4;                  // row-stat exchange
    s += (size_t)cluster * heads * BM * 4;              // head partials
    return s;
}

}  // namespace gemm
}  // namespace lat
