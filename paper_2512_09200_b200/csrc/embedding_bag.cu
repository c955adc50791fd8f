// embedding_bag.cu -- K1 jagged embedding-bag sum pooling, the synthetic
// input generators, K6 domain bucketing and the row-wise
// norm/activation kernel (numerics.hpp:81-107).
//
// K1 layout: one warp per bag (f, b); a row of D elements is LPR lanes x 16 B, so a warp
// gathers 32/LPR rows per pass and keeps U passes (U x 16 B per lane) in flight. Ids are
// read once per 32 with one coalesced load and broadcast with shuffles. Table rows are
// streamed with ld.global.nc.L1::no_allocate (no reuse under uniform ids). The pooled row
// is reduced across the row groups with xor-shuffles, optionally rms-normalised over D and
// written once (HBM-bound: bytes = ids*D*s_tab + ids*4 + (F*B+1)*8 + F*B*D*s_out).
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "common.cuh"

namespace lat {
namespace {

struct BagParams {
    int32_t F;
    int64_t B;
    int32_t D;
    const void* const* tables;
    const int64_t* rows;
    const int64_t* offsets;
    const int32_t* ids;
    void* out;
    int64_t out_stride;
    int32_t out_foff;
    const int32_t* pos;
    int32_t normalize;
    unsigned long long* err;
    int32_t R;  // source ranks: bags laid out [R][F][B]
    int64_t slice_cap;  // > 0: source r's ids start at r * slice_cap (static exchange buffer)
    unsigned long long* counter;  // work-claim counter (zeroed per launch)
    int32_t l2keep;  // bit 0: table rows loaded with an L2 evict_last policy; bit 1: pooled rows
                     // stored with evict_first (LATTICE_BAG_L2KEEP)
    // Peer mode (lattice_peer_embedding_bag): this rank owns features [src_foff, src_foff+F)
    // of every source rank's CSR and pools them for all R sources, reading each source's
    // offsets / ids / sample_pos from that source's HBM over NVLink and writing the pooled row
    // straight into the source's X0. Bags are numbered [f][r][b] so one table stays hot in L2
    // across all sources.
    uint32_t mB, sB, mF, sF;  // fast division by B and F (magic multiplier, shift), see fastdiv()
    int32_t peer_mode;
    const int64_t* const* p_off;  // [R] source CSR offsets over F_src features
    const int32_t* const* p_ids;  // [R]
    const int32_t* const* p_pos;  // [R] output row of each source sample
    void* const* p_out;           // [R] each source's [B][.][D] output
    int32_t src_foff;
    uint32_t mC, sC, mR, sR;  // fast division by the staged kernel's chunks per segment and by R
};

// Table rows with an L2 evict_last policy: rows of the table being pooled are re-read by
// other bags a few microseconds later, while ids/offsets/outputs stream through once.
__device__ __forceinline__ uint4 ld_row_keep(const void* p, uint64_t pol) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p), "l"(pol));
    return r;
}
// x / d for x < 2^31 as one wide multiply and a shift: m = floor(2^(31+l) / d) + 1 with
// l = ceil(log2 d) keeps the error of x*m / 2^(31+l) below 1/d, so the floor is exact.
inline void fastdiv(uint32_t d, uint32_t* m, uint32_t* s) {
    uint32_t l = 0;
    while ((1ull << l) < d) ++l;
    *m = (uint32_t)(((1ull << (31 + l)) / d) + 1);
    *s = 31 + l;
}
__device__ __forceinline__ uint32_t fdiv(uint32_t x, uint32_t m, uint32_t s) {
    return (uint32_t)(((uint64_t)x * m) >> s);
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

template <typename T>
struct Elem;
template <>
struct Elem<float> {
    static constexpr int kPerChunk = 4;
    // two packed fp32 adds (FADD2, add.rn.f32x2): per lane identical to two add.rn.f32
    __device__ static void add(float* acc, uint4 v) {
        add2(acc[0], acc[1], v.x, v.y);
        add2(acc[2], acc[3], v.z, v.w);
    }
    __device__ static void add2(float& a0, float& a1, uint32_t x0, uint32_t x1) {
        uint64_t a, x;
        asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(a0), "f"(a1));
        asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "r"(x0), "r"(x1));
        asm("add.rn.f32x2 %0, %0, %1;" : "+l"(a) : "l"(x));
        asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(a));
    }
};
template <>
struct Elem<__nv_bfloat16> {
    static constexpr int kPerChunk = 8;
    // add.rn.f32.bf16 (HADD.BF16 with an fp32 accumulator): the bf16 operand is widened
    // exactly, one rounding at fp32 -- the same result as cvt + add.rn.f32, in one instruction
    __device__ static void add(float* acc, uint4 v) {
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
            asm("{ .reg .b16 l, h;\n\t mov.b32 {l, h}, %2;\n\t add.rn.f32.bf16 %0, l, %0;\n\t"
                " add.rn.f32.bf16 %1, h, %1; }"
                : "+f"(acc[2 * i]), "+f"(acc[2 * i + 1])
                : "r"(w[i]));
    }
};

// 16-byte store; ef: with an L2 evict_first policy (pooled rows are not re-read by this kernel)
__device__ __forceinline__ void st16(void* dst, uint4 v, bool ef, uint64_t pol) {
    if (ef)
        asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(dst),
                     "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol)
                     : "memory");
    else
        *reinterpret_cast<uint4*>(dst) = v;
}
__device__ __forceinline__ uint32_t f2u(float x) { return __float_as_uint(x); }

template <typename OT, int N>
__device__ __forceinline__ void store_out(OT* dst, const float* v, bool ef = false, uint64_t pol = 0);
template <>
__device__ __forceinline__ void store_out<float, 4>(float* dst, const float* v, bool ef, uint64_t pol) {
    st16(dst, make_uint4(f2u(v[0]), f2u(v[1]), f2u(v[2]), f2u(v[3])), ef, pol);
}
template <>
__device__ __forceinline__ void store_out<float, 8>(float* dst, const float* v, bool ef, uint64_t pol) {
    st16(dst, make_uint4(f2u(v[0]), f2u(v[1]), f2u(v[2]), f2u(v[3])), ef, pol);
    st16(dst + 4, make_uint4(f2u(v[4]), f2u(v[5]), f2u(v[6]), f2u(v[7])), ef, pol);
}
template <>
__device__ __forceinline__ void store_out<__nv_bfloat16, 4>(__nv_bfloat16* dst, const float* v, bool, uint64_t) {
    *reinterpret_cast<uint2*>(dst) = make_uint2(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]));
}
template <>
__device__ __forceinline__ void store_out<__nv_bfloat16, 8>(__nv_bfloat16* dst, const float* v, bool ef,
                                                            uint64_t pol) {
    st16(dst, make_uint4(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]), pack_bf16x2(v[4], v[5]),
                         pack_bf16x2(v[6], v[7])),
         ef, pol);
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

constexpr int kBagWarps = 8;
__device__ __align__(16) uint4 g_zero_row[64];  // 1 KB of zeros: the row of an invalid id

// 1 / sqrt(x) for the rms_norm scale: x = mean(x^2) + 1e-6 is never denormal, so the ftz
// MUFU.RSQ is the same value as rsqrtf without its denormal fix-up instructions
// base + id * rowb as ONE IMAD.WIDE.U32 (mad.wide.u32 with the 64-bit base as addend; left to
// itself the compiler splits it into a wide multiply, a LOP3 and a 64-bit add)
__device__ __forceinline__ const uint8_t* row_addr(const uint8_t* base, uint32_t id, uint32_t rowb) {
    uint64_t a;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(a) : "r"(id), "r"(rowb), "l"(reinterpret_cast<uint64_t>(base)));
    return reinterpret_cast<const uint8_t*>(a);
}
__device__ __forceinline__ float rsqrt_ftz(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// ---- direct kernel (single GPU and the NCCL-exchange owner side) ----------------------------
// Persistent warps with dynamic scheduling: a warp claims kChunk consecutive bags at a time
// from a global counter, so all warps stay inside a narrow window of the bag sequence -- the
// sequence is table-major, so the live working set is about one table and repeated rows hit
// in L2 instead of re-reading HBM. While the current bag's rows are in flight, the next bag's
// offsets and first 32 ids are already being fetched; with local offsets / ids, 40 warps per SM
// hide the rest of that chain.
namespace direct {
template <bool PEER>
__device__ __forceinline__ void decode(const BagParams& p, uint32_t bag, int& f, int& r, uint32_t& b) {
    const uint32_t R = (uint32_t)p.R, B = (uint32_t)p.B, F = (uint32_t)p.F;
    if (PEER) {
        const uint32_t fr = bag / B;
        r = (int)(fr % R);
        f = (int)(fr / R);
        b = bag - fr * B;
    } else {
        const uint32_t rf = fdiv(bag, p.mB, p.sB);
        r = (int)fdiv(rf, p.mF, p.sF);
        f = (int)(rf - (uint32_t)r * F);
        b = bag - rf * B;
    }
}

// First id and length of bag `bag` (CSR, CSR rebased into fixed per-source slices, or -- peer
// mode -- the source rank's own CSR read over NVLink).
template <bool PEER>
__device__ __forceinline__ void bag_range(const BagParams& p, uint32_t bag, const int32_t*& idp, int& len) {
    int64_t s, e;
    if constexpr (PEER) {
        int f, r;
        uint32_t b;
        decode<true>(p, bag, f, r, b);
        const int64_t* off = p.p_off[r] + (int64_t)(p.src_foff + f) * p.B + b;
        s = off[0];
        e = off[1];
        idp = p.p_ids[r] + s;
    } else {
        s = p.offsets[bag];
        e = p.offsets[bag + 1];
        if (p.slice_cap > 0) {
            // source r's ids sit in the fixed slice [r*cap, (r+1)*cap): a slice the sender had to
            // truncate (it set the overflow flag) pools only what arrived, never the next slice
            const int64_t r = bag / ((int64_t)p.F * p.B);
            const int64_t base = p.offsets[r * p.F * p.B];
            s = min(s - base, p.slice_cap);
            e = min(e - base, p.slice_cap);
            s += r * p.slice_cap;
            e += r * p.slice_cap;
        }
        len = (int)(e - s);
        idp = p.ids + s;
        return;
    }
    len = (int)(e - s);
}

// Position of id pointer q in the ids array it came from (DataError index; cold path).
template <bool PEER>
__device__ __forceinline__ unsigned long long id_position(const BagParams& p, uint32_t bag, const int32_t* q) {
    if constexpr (PEER) {
        int f, r;
        uint32_t b;
        decode<true>(p, bag, f, r, b);
        return (unsigned long long)(q - p.p_ids[r]);
    }
    return (unsigned long long)(q - p.ids);
}

constexpr int kChunk = 4;

__device__ __forceinline__ uint32_t claim_chunk(unsigned long long* counter, int lane) {
    unsigned long long c = 0;
    if (lane == 0) c = atomicAdd(counter, 1ull);
    return (uint32_t)__shfl_sync(0xffffffffu, c, 0) * kChunk;
}

// N passes of RPP rows each: every lane issues N*CPL 16-byte row loads back to back, then
// accumulates them. MASK: rows at or past `cnt` read the zero row instead (bag tail).
// CHECK = false: the caller verified that every id of this 32-id window is in range, so rows
// are addressed without a per-row bound check (the common case); MASK rows past `cnt` still
// read the zero row. `tlane` / `zlane` are the table / zero row already offset to this lane's
// first 16-byte column, and a row is exactly LPR*CPL*16 bytes (launch_bag picks LPR, CPL from
// the row size), so a row address is one IMAD.WIDE of the id.
template <typename TT, int LPR, int CPL, int N, bool MASK, bool CHECK, bool PEER>
__device__ __forceinline__ void gather_step(const BagParams& p, uint32_t bag, const int32_t* idp, int base,
                                            const uint8_t* __restrict__ tlane, uint32_t rows, int my_id, int j,
                                            int cnt, int sub, const uint8_t* zlane, uint64_t pol, float* acc) {
    constexpr int EPC = Elem<TT>::kPerChunk;
    constexpr int RPP = 32 / LPR;
    constexpr uint32_t ROWB = LPR * CPL * 16;
    uint4 v[N][CPL];
#pragma unroll
    for (int u = 0; u < N; ++u) {
        const int jj = j + u * RPP + sub;
        const int id = __shfl_sync(0xffffffffu, my_id, jj & 31);
        bool ok = true;
        if (CHECK) {
            ok = (uint32_t)id < rows;
            const bool live = !MASK || jj < cnt;
            if (live && !ok) atomicMin(p.err, id_position<PEER>(p, bag, idp + base + jj));
        }
        if (MASK) ok = ok && jj < cnt;
        const uint8_t* row = (!CHECK && !MASK) || ok ? row_addr(tlane, (uint32_t)id, ROWB) : zlane;
#pragma unroll
        for (int c = 0; c < CPL; ++c) v[u][c] = ld_row_keep(row + c * LPR * 16, pol);
    }
#pragma unroll
    for (int u = 0; u < N; ++u)
#pragma unroll
        for (int c = 0; c < CPL; ++c) Elem<TT>::add(acc + c * EPC, v[u][c]);
}

template <typename TT, typename OT, int LPR, int CPL, int U, int MINB, bool PEER>
__global__ void __launch_bounds__(kBagWarps * 32, MINB) bag_kernel(const BagParams p) {
    constexpr int EPC = Elem<TT>::kPerChunk;
    constexpr int RPP = 32 / LPR;          // rows per pass
    constexpr int UT = U >= 4 ? U / 2 : U;  // passes per masked tail step
    const int lane = threadIdx.x & 31;
    const uint32_t total = (uint32_t)p.R * (uint32_t)p.F * (uint32_t)p.B;
    uint32_t bag = claim_chunk(p.counter, lane);
    if (bag >= total) return;
    uint32_t chunk_end = bag + kChunk < total ? bag + kChunk : total;
    const int sub = lane / LPR, cl = lane % LPR;
    const bool ef = (p.l2keep & 2) != 0;
    const uint64_t pol = (p.l2keep & 1) ? policy_evict_last() : policy_evict_normal();  // table rows
    const uint64_t pol_ef = policy_evict_first();
    const uint8_t* zlane = reinterpret_cast<const uint8_t*>(g_zero_row) + cl * 16;
    const int32_t* idp;
    int len;
    bag_range<PEER>(p, bag, idp, len);
    int first_id = lane < len ? __ldg(idp + lane) : 0;

    while (bag < total) {
        uint32_t nbag = bag + 1;
        if (nbag >= chunk_end) {
            nbag = claim_chunk(p.counter, lane);
            chunk_end = nbag + kChunk < total ? nbag + kChunk : total;
        }
        // the next bag's offsets are requested before this bag's rows
        const int32_t* nidp = idp;
        int nlen = 0;
        if (nbag < total) bag_range<PEER>(p, nbag, nidp, nlen);
        int f, r;
        uint32_t b;
        decode<PEER>(p, bag, f, r, b);
        int32_t peer_row = 0;
        if constexpr (PEER) {
            // issued before the row gathers so the NVLink round trip overlaps them
            asm volatile("ld.global.s32 %0, [%1];" : "=r"(peer_row) : "l"(p.p_pos[r] + b));
        }
        // the output row is requested before the gathers (its latency hides under them)
        const int64_t ob = (int64_t)r * p.B + b;  // output sample r*B + b (plain mode)
        int64_t orow = ob;
        if constexpr (!PEER) {
            if (p.pos) orow = __ldg(p.pos + ob);
        }
        const uint8_t* __restrict__ tlane = static_cast<const uint8_t*>(p.tables[f]) + cl * 16;
        const int64_t rows64 = p.rows[f];
        const uint32_t rows = rows64 < 0x7fffffff ? (uint32_t)rows64 : 0x7fffffffu;

        float acc[CPL * EPC];
#pragma unroll
        for (int i = 0; i < CPL * EPC; ++i) acc[i] = 0.0f;

        for (int base = 0; base < len; base += 32) {
            const int cnt = len - base < 32 ? len - base : 32;
            const int my_id = base == 0 ? first_id : (lane < cnt ? __ldg(idp + base + lane) : 0);
            int j = 0;
            if (__all_sync(0xffffffffu, lane >= cnt || (uint32_t)my_id < rows)) {  // all ids in range
                for (; j + RPP * U <= cnt; j += RPP * U)
                    gather_step<TT, LPR, CPL, U, false, false, PEER>(p, bag, idp, base, tlane, rows, my_id, j, cnt, sub,
                                                                     zlane, pol, acc);
                for (; j < cnt; j += RPP * UT)
                    gather_step<TT, LPR, CPL, UT, true, false, PEER>(p, bag, idp, base, tlane, rows, my_id, j, cnt, sub,
                                                                     zlane, pol, acc);
            } else {  // some id out of range: checked path (zero contribution + first-offender error)
                for (; j + RPP * U <= cnt; j += RPP * U)
                    gather_step<TT, LPR, CPL, U, false, true, PEER>(p, bag, idp, base, tlane, rows, my_id, j, cnt, sub,
                                                                     zlane, pol, acc);
                for (; j < cnt; j += RPP * UT)
                    gather_step<TT, LPR, CPL, UT, true, true, PEER>(p, bag, idp, base, tlane, rows, my_id, j, cnt, sub,
                                                                     zlane, pol, acc);
            }
        }
        // next bag's first ids (its offsets were requested before this bag's rows)
        const int next_id = (nbag < total && lane < nlen) ? __ldg(nidp + lane) : 0;
        // fold the RPP row groups: lanes with equal cl end up with the full sum
#pragma unroll
        for (int o = LPR; o < 32; o <<= 1)
#pragma unroll
            for (int i = 0; i < CPL * EPC; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);

        if (p.normalize) {  // rms_norm over D (numerics.hpp:81-90), eps 1e-6
            float ss = 0.0f;
#pragma unroll
            for (int i = 0; i < CPL * EPC; ++i) ss += acc[i] * acc[i];
#pragma unroll
            for (int o = 1; o < LPR; o <<= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
            // D = LPR*CPL*EPC is a power of two: the product with 1/D equals the division;
            // MUFU.RSQ (~2 ulp; the row is then rounded to bf16)
            const float inv = rsqrt_ftz(ss * (1.0f / (LPR * CPL * EPC)) + 1e-6f);
#pragma unroll
            for (int i = 0; i < CPL * EPC; ++i) acc[i] *= inv;
        }
        if (sub == 0) {
            const int64_t row = PEER ? (int64_t)peer_row : orow;
            OT* dst = static_cast<OT*>(PEER ? p.p_out[r] : p.out) + row * p.out_stride +
                      (int64_t)(p.out_foff + f) * p.D;
#pragma unroll
            for (int c = 0; c < CPL; ++c) store_out<OT, EPC>(dst + (c * LPR + cl) * EPC, acc + c * EPC, ef, pol_ef);
        }
        bag = nbag;
        idp = nidp;
        len = nlen;
        first_id = next_id;
    }
    // peer mode: this warp's remote row stores are ordered before the barrier kernel that
    // follows on the stream releases them to the destination ranks
    if constexpr (PEER) __threadfence_system();
}

}  // namespace direct

// ---- staged kernel (peer mode: offsets / ids / sample_pos read over NVLink) -------------------
namespace staged {

// Work item = a chunk of up to kChunk consecutive samples of one (source, table) segment, so
// the chunk's offsets, ids and output rows are contiguous. Persistent warps claim chunks from
// a global counter (all warps stay inside a narrow window of the segment sequence, which is
// table-major, so the live working set is about one table and repeated rows hit in L2).
// Each warp double-buffers chunk metadata in shared memory: while it gathers the rows of chunk
// c, the ids and output rows of chunk c+1 are already in flight (cp.async) and the offsets of
// chunk c+2 are being loaded -- the offsets -> ids -> rows chain of a chunk never sits on the
// critical path, which matters most in peer mode where offsets / ids / sample_pos are read
// from the source rank over NVLink.
constexpr int kChunk = 4;
constexpr int kIdsCap = 192;  // ids staged per chunk; longer chunks read the rest from global

struct __align__(16) Stage {
    int32_t off[kChunk + 1];  // bag starts relative to the chunk's first id
    int32_t pos[kChunk];      // output row of each bag
    int32_t f, r, b0, n;      // table, source, first sample, bags
    const int32_t* idg;       // the chunk's first id in global memory
    int32_t ids[kIdsCap];
};

__device__ __forceinline__ uint32_t claim_chunk(unsigned long long* counter, int lane) {
    unsigned long long c = 0;
    if (lane == 0) c = atomicAdd(counter, 1ull);
    return (uint32_t)__shfl_sync(0xffffffffu, c, 0);
}

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
                 "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Chunk c -> segment and samples. Plain mode segments are [r][f] (the CSR order); peer mode
// segments are [f][r] so one table is pooled for every source before the next. 32-bit: the
// host guarantees R * F * B < 2^31.
template <bool PEER>
__device__ __forceinline__ void locate(const BagParams& p, uint32_t c, uint32_t cps, int& f, int& r, uint32_t& b0,
                                       int& n) {
    const uint32_t seg = fdiv(c, p.mC, p.sC);  // c / cps
    b0 = (c - seg * cps) * kChunk;
    n = (uint32_t)p.B - b0 < (uint32_t)kChunk ? (int)((uint32_t)p.B - b0) : kChunk;
    if (PEER) {
        f = (int)fdiv(seg, p.mR, p.sR);
        r = (int)(seg - (uint32_t)f * (uint32_t)p.R);
    } else {
        r = (int)fdiv(seg, p.mF, p.sF);
        f = (int)(seg - (uint32_t)r * (uint32_t)p.F);
    }
}

// Offsets of chunk c's bags (lane i <= n holds the start of bag i / the end of the chunk).
template <bool PEER>
__device__ __forceinline__ int64_t chunk_offsets(const BagParams& p, uint32_t c, uint32_t cps, int lane) {
    int f, r, n;
    uint32_t b0;
    locate<PEER>(p, c, cps, f, r, b0, n);
    if (lane > n) return 0;
    if (PEER) return p.p_off[r][(int64_t)(p.src_foff + f) * p.B + b0 + lane];
    const int64_t o = p.offsets[((int64_t)r * p.F + f) * p.B + b0 + lane];
    if (p.slice_cap > 0) {  // clamp into source r's fixed slice (see direct::bag_range)
        const int64_t base = p.offsets[(int64_t)r * p.F * p.B];
        return base + min(o - base, p.slice_cap);
    }
    return o;
}

// Fill stage S for chunk c whose offsets are `o` (per lane, from chunk_offsets): header and
// relative offsets by plain stores, ids and output rows by cp.async (one commit group).
template <bool PEER>
__device__ __forceinline__ void stage_chunk(const BagParams& p, Stage& S, uint32_t c, uint32_t cps, int64_t o,
                                            int lane) {
    int f, r, n;
    uint32_t b0;
    locate<PEER>(p, c, cps, f, r, b0, n);
    const int64_t o0 = __shfl_sync(0xffffffffu, o, 0);
    const int64_t oN = __shfl_sync(0xffffffffu, o, n);
    const int32_t* idg;
    if (PEER) {
        idg = p.p_ids[r] + o0;
    } else {
        int64_t shift = 0;
        if (p.slice_cap > 0) shift = r * p.slice_cap - p.offsets[(int64_t)r * p.F * p.B];
        idg = p.ids + o0 + shift;
    }
    if (lane <= n) S.off[lane] = (int32_t)(o - o0);
    if (lane == 0) {
        S.f = f;
        S.r = r;
        S.b0 = (int32_t)b0;
        S.n = n;
        S.idg = idg;
    }
    const int cnt = (int)(oN - o0) < kIdsCap ? (int)(oN - o0) : kIdsCap;
    for (int q = lane; q < cnt; q += 32) cp_async4(&S.ids[q], idg + q);
    if (lane < n) {
        if (PEER)
            cp_async4(&S.pos[lane], p.p_pos[r] + b0 + lane);
        else if (p.pos)
            cp_async4(&S.pos[lane], p.pos + (int64_t)r * p.B + b0 + lane);
        else
            S.pos[lane] = (int32_t)((int64_t)r * p.B + b0 + lane);
    }
    cp_async_commit();
}

// Position of global id pointer q in the ids array it came from (DataError index; cold path).
template <bool PEER>
__device__ __noinline__ unsigned long long id_position(const BagParams& p, int r, const int32_t* q) {
    return (unsigned long long)(q - (PEER ? p.p_ids[r] : p.ids));
}


// N passes of RPP rows each: every lane issues N*CPL 16-byte row loads back to back, then
// accumulates them. Ids come from the stage (q < kIdsCap) or global. MASK: rows at or past
// `len` read the zero row instead (bag tail). tlane / zlane: as in direct::gather_step.
template <typename TT, int LPR, int CPL, int N, bool MASK, bool CHECK, bool PEER>
__device__ __forceinline__ void gather_step(const BagParams& p, const Stage& S, int sk, int j, int len,
                                            const uint8_t* __restrict__ tlane, uint32_t rows, int sub,
                                            const uint8_t* zlane, uint64_t pol, float* acc) {
    constexpr int EPC = Elem<TT>::kPerChunk;
    constexpr int RPP = 32 / LPR;
    constexpr uint32_t ROWB = LPR * CPL * 16;
    uint4 v[N][CPL];
#pragma unroll
    for (int u = 0; u < N; ++u) {
        const int jj = j + u * RPP + sub;
        const int q = sk + jj;
        const bool live = !MASK || jj < len;
        int id = 0;
        if (live) id = q < kIdsCap ? S.ids[q] : __ldg(S.idg + q);
        bool ok = true;
        if (CHECK) {
            ok = (uint32_t)id < rows;
            if (live && !ok) atomicMin(p.err, id_position<PEER>(p, S.r, S.idg + q));
        }
        ok = ok && live;
        const uint8_t* row = (!CHECK && !MASK) || ok ? row_addr(tlane, (uint32_t)id, ROWB) : zlane;
#pragma unroll
        for (int c = 0; c < CPL; ++c) v[u][c] = ld_row_keep(row + c * LPR * 16, pol);
    }
#pragma unroll
    for (int u = 0; u < N; ++u)
#pragma unroll
        for (int c = 0; c < CPL; ++c) Elem<TT>::add(acc + c * EPC, v[u][c]);
}

// Pool, normalise and store the bags of the staged chunk S.
template <typename TT, typename OT, int LPR, int CPL, int U, bool PEER>
__device__ __forceinline__ void pool_chunk(const BagParams& p, const Stage& S, int lane, uint64_t pol) {
    constexpr int EPC = Elem<TT>::kPerChunk;
    constexpr int RPP = 32 / LPR;           // rows per pass
    constexpr int UT = U >= 4 ? U / 2 : U;  // passes per masked tail step
    const int sub = lane / LPR, cl = lane % LPR;
    const int f = S.f, n = S.n;
    const uint8_t* __restrict__ tlane = static_cast<const uint8_t*>(p.tables[f]) + cl * 16;
    const uint8_t* zlane = reinterpret_cast<const uint8_t*>(g_zero_row) + cl * 16;
    const int64_t rows64 = p.rows[f];
    const uint32_t rows = rows64 < 0x7fffffff ? (uint32_t)rows64 : 0x7fffffffu;
    OT* out = static_cast<OT*>(PEER ? p.p_out[S.r] : p.out) + (int64_t)(p.out_foff + f) * p.D;
    for (int k = 0; k < n; ++k) {
        const int sk = S.off[k];
        const int len = S.off[k + 1] - sk;
        float acc[CPL * EPC];
#pragma unroll
        for (int i = 0; i < CPL * EPC; ++i) acc[i] = 0.0f;
        int j = 0;
        bool in_range = true;  // every id of the bag valid: gather without per-row checks
        for (int q = lane; q < len; q += 32) {
            const int id = sk + q < kIdsCap ? S.ids[sk + q] : __ldg(S.idg + sk + q);
            in_range &= (uint32_t)id < rows;
        }
        if (__all_sync(0xffffffffu, in_range)) {
            for (; j + RPP * U <= len; j += RPP * U)
                gather_step<TT, LPR, CPL, U, false, false, PEER>(p, S, sk, j, len, tlane, rows, sub, zlane, pol, acc);
            for (; j < len; j += RPP * UT)
                gather_step<TT, LPR, CPL, UT, true, false, PEER>(p, S, sk, j, len, tlane, rows, sub, zlane, pol, acc);
        } else {
            for (; j + RPP * U <= len; j += RPP * U)
                gather_step<TT, LPR, CPL, U, false, true, PEER>(p, S, sk, j, len, tlane, rows, sub, zlane, pol, acc);
            for (; j < len; j += RPP * UT)
                gather_step<TT, LPR, CPL, UT, true, true, PEER>(p, S, sk, j, len, tlane, rows, sub, zlane, pol, acc);
        }
        // fold the RPP row groups: lanes with equal cl end up with the full sum
#pragma unroll
        for (int o = LPR; o < 32; o <<= 1)
#pragma unroll
            for (int i = 0; i < CPL * EPC; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
        if (p.normalize) {  // rms_norm over D (numerics.hpp:81-90), eps 1e-6
            float ss = 0.0f;
#pragma unroll
            for (int i = 0; i < CPL * EPC; ++i) ss += acc[i] * acc[i];
#pragma unroll
            for (int o = 1; o < LPR; o <<= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
            const float inv = rsqrt_ftz(ss * (1.0f / (LPR * CPL * EPC)) + 1e-6f);  // as in direct::
#pragma unroll
            for (int i = 0; i < CPL * EPC; ++i) acc[i] *= inv;
        }
        if (sub == 0) {
            OT* dst = out + (int64_t)S.pos[k] * p.out_stride;
#pragma unroll
            for (int c = 0; c < CPL; ++c) store_out<OT, EPC>(dst + (c * LPR + cl) * EPC, acc + c * EPC);
        }
    }
}

template <typename TT, typename OT, int LPR, int CPL, int U, int MINB, bool PEER>
__global__ void __launch_bounds__(kBagWarps * 32, MINB) bag_kernel(const BagParams p) {
    __shared__ Stage stages[kBagWarps][2];
    const int lane = threadIdx.x & 31;
    Stage* stg = stages[threadIdx.x >> 5];
    const uint32_t cps = (uint32_t)((p.B + kChunk - 1) / kChunk);
    const uint32_t total = (uint32_t)p.R * (uint32_t)p.F * cps;
    const uint64_t pol = (p.l2keep & 1) ? policy_evict_last() : policy_evict_normal();

    uint32_t c = claim_chunk(p.counter, lane);
    if (c >= total) return;
    stage_chunk<PEER>(p, stg[0], c, cps, chunk_offsets<PEER>(p, c, cps, lane), lane);
    uint32_t cn = claim_chunk(p.counter, lane);
    int64_t on = cn < total ? chunk_offsets<PEER>(p, cn, cps, lane) : 0;
    int s = 0;
    while (true) {
        // stage the next chunk (its offsets were requested one chunk ago), then wait for this one
        if (cn < total) {
            stage_chunk<PEER>(p, stg[s ^ 1], cn, cps, on, lane);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncwarp();
        // claim the chunk after next and start its offsets
        const uint32_t cnn = cn < total ? claim_chunk(p.counter, lane) : total;
        const int64_t onn = cnn < total ? chunk_offsets<PEER>(p, cnn, cps, lane) : 0;
        pool_chunk<TT, OT, LPR, CPL, U, PEER>(p, stg[s], lane, pol);
        __syncwarp();  // stage s is refilled next iteration
        if (cn >= total) break;
        cn = cnn;
        on = onn;
        s ^= 1;
    }
    // peer mode: this warp's remote row stores are ordered before the barrier kernel that
    // follows on the stream releases them to the destination ranks
    if constexpr (PEER) __threadfence_system();
}

}  // namespace staged


// Blocks per SM of the persistent bag grid: occupancy by default; LATTICE_BAG_BLOCKS_PER_SM caps
// it (1 leaves room for a co-running GEMM / FM CTA on every SM when the embedding stage of the
// next batch overlaps the dense stage of this one).
int bag_blocks_cap() {
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("LATTICE_BAG_BLOCKS_PER_SM");
        v = e ? std::atoi(e) : 0;
    }
    return v;
}

template <typename K>
unsigned persistent_grid(K kernel, int64_t bags) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kBagWarps * 32, 0) != cudaSuccess ||
        per_sm < 1)
        per_sm = 4;
    if (bag_blocks_cap() > 0 && per_sm > bag_blocks_cap()) per_sm = bag_blocks_cap();
    const int64_t want = (bags + kBagWarps - 1) / kBagWarps;
    const int64_t cap = (int64_t)num_sms() * per_sm;
    return (unsigned)(want < cap ? want : cap);
}

// Variant: 0 -> U=4 at 5 blocks/SM (40 warps), 1 -> U=8 at 3 blocks/SM (24 warps),
// 2 -> U=8 at 4 blocks/SM. LATTICE_BAG_VARIANT overrides the default (tuning sweeps).
int bag_variant(int row_bytes, bool peer) {
    static int forced = -2;
    if (forced == -2) {
        const char* e = std::getenv("LATTICE_BAG_VARIANT");
        forced = e ? std::atoi(e) : -1;
    }
    if (forced >= 0 && forced <= 2) return forced;
    (void)peer;
    (void)row_bytes;
    return 0;  // U=4 at 40 warps/SM: best for both kernels, bf16 and fp32 (profiles/r01/bag_ab.log)
}

template <typename TT, typename OT, int LPR, int CPL, bool PEER>
void launch_one(const BagParams& p, cudaStream_t st, int row_bytes) {
    const int64_t bags = (int64_t)p.R * p.F * p.B;
    // peer mode runs the staged kernel (hides the NVLink latency of the offsets -> ids chain:
    // 8.8 vs 10.8 ms owner kernel at 4 x B200); local bags run the direct kernel (7.1 vs 7.9 ms
    // on the mid stage, 16.3 vs 15.0 M samples/s on the bf16 micro). LATTICE_BAG_KERNEL =
    // direct | staged overrides for A/B runs.
    static const int forced = [] {
        const char* e = std::getenv("LATTICE_BAG_KERNEL");
        return !e ? -1 : std::string(e) == "staged" ? 1 : std::string(e) == "direct" ? 0 : -1;
    }();
    const bool use_staged = forced >= 0 ? forced == 1 : PEER;
    if (!use_staged) {
        switch (bag_variant(row_bytes, PEER)) {
            case 0:
                direct::bag_kernel<TT, OT, LPR, CPL, 4, 5, PEER>
                    <<<persistent_grid(direct::bag_kernel<TT, OT, LPR, CPL, 4, 5, PEER>, bags), kBagWarps * 32, 0, st>>>(p);
                break;
            case 2:
                direct::bag_kernel<TT, OT, LPR, CPL, 8, 4, PEER>
                    <<<persistent_grid(direct::bag_kernel<TT, OT, LPR, CPL, 8, 4, PEER>, bags), kBagWarps * 32, 0, st>>>(p);
                break;
            default:
                direct::bag_kernel<TT, OT, LPR, CPL, 8, 3, PEER>
                    <<<persistent_grid(direct::bag_kernel<TT, OT, LPR, CPL, 8, 3, PEER>, bags), kBagWarps * 32, 0, st>>>(p);
        }
        return;
    }
    switch (bag_variant(row_bytes, PEER)) {
        case 0:
            staged::bag_kernel<TT, OT, LPR, CPL, 4, 5, PEER>
                <<<persistent_grid(staged::bag_kernel<TT, OT, LPR, CPL, 4, 5, PEER>, bags), kBagWarps * 32, 0, st>>>(p);
            break;
        case 2:
            staged::bag_kernel<TT, OT, LPR, CPL, 8, 4, PEER>
                <<<persistent_grid(staged::bag_kernel<TT, OT, LPR, CPL, 8, 4, PEER>, bags), kBagWarps * 32, 0, st>>>(p);
            break;
        default:
            staged::bag_kernel<TT, OT, LPR, CPL, 8, 3, PEER>
                <<<persistent_grid(staged::bag_kernel<TT, OT, LPR, CPL, 8, 3, PEER>, bags), kBagWarps * 32, 0, st>>>(p);
    }
}

// Default 3: table rows evict_last + pooled-row stores evict_first. A table's rows are re-read
// ~6x within the ~30 us its bags are in flight (mid: 655K ids over 100K rows); without the hint
// the streaming ids/outputs push them out of L2 (24% hit rate). Mid embedding stage 7.2 -> 5.5
// ms, step 26.1-27.5 -> 24.3-24.5 ms, GEMMs unchanged (profiles/r01/bag_l2.log).
int bag_l2keep() {
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("LATTICE_BAG_L2KEEP");
        v = e ? std::atoi(e) : 3;
    }
    return v;
}

template <typename TT, typename OT>
lattice_status launch_bag(const BagParams& p, int row_bytes, cudaStream_t st) {
    if (p.peer_mode) {
        switch (row_bytes) {
            case 128: launch_one<TT, OT, 8, 1, true>(p, st, row_bytes); return LATTICE_OK;
            case 256: launch_one<TT, OT, 16, 1, true>(p, st, row_bytes); return LATTICE_OK;
            case 512: launch_one<TT, OT, 32, 1, true>(p, st, row_bytes); return LATTICE_OK;
            case 1024: launch_one<TT, OT, 32, 2, true>(p, st, row_bytes); return LATTICE_OK;
            default: break;
        }
    }
    switch (row_bytes) {
        case 128: launch_one<TT, OT, 8, 1, false>(p, st, row_bytes); break;
        case 256: launch_one<TT, OT, 16, 1, false>(p, st, row_bytes); break;
        case 512: launch_one<TT, OT, 32, 1, false>(p, st, row_bytes); break;
        case 1024: launch_one<TT, OT, 32, 2, false>(p, st, row_bytes); break;
        default:
            return set_error(LATTICE_USAGE,
                             "embedding_bag: D * sizeof(table dtype) must be 128, 256, 512 or 1024 bytes");
    }
    return LATTICE_OK;
}

// ---- synthetic generators ---------------------------------------------------------------
__global__ void fill_tables_kernel(void* out, int dtype, int64_t n, int D, int64_t rows,
                                   int64_t rows_total, int feature_base, uint64_t seed) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = i % D;
        const int64_t r = (i / D) % rows;
        const int64_t f = i / ((int64_t)D * rows) + feature_base;
        const uint64_t idx = ((uint64_t)f * (uint64_t)rows_total + (uint64_t)r) * (uint64_t)D + c;
        const float v = (float)(int8_t)(gen_u64(seed, kTagTable, idx) >> 56) * 0x1.0p-10f;
        if (dtype == LATTICE_F32)
            static_cast<float*>(out)[i] = v;
        else
            static_cast<__nv_bfloat16*>(out)[i] = __float2bfloat16_rn(v);
    }
}

__global__ void fill_weights_kernel(void* out, int dtype, int64_t n, int64_t fan_in, int shift,
                                    uint64_t seed, uint64_t tag) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float v = ldexpf((float)(int8_t)(gen_u64(seed, tag, (uint64_t)i) >> 56), -shift);
        if (dtype == LATTICE_F32)
            static_cast<float*>(out)[i] = v;
        else
            static_cast<__nv_bfloat16*>(out)[i] = __float2bfloat16_rn(v);
    }
}

__global__ void synth_len_kernel(int64_t bags, int max_len, uint64_t seed, int64_t* len) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < bags;
         i += (int64_t)gridDim.x * blockDim.x)
        len[i] = (int64_t)(gen_u64(seed, kTagLen, (uint64_t)i) % (uint64_t)(max_len + 1));
}

__global__ void synth_ids_kernel(int64_t bags, int max_len, int64_t rows, uint64_t seed,
                                 const int64_t* __restrict__ off, int32_t* __restrict__ ids) {
    // one warp per bag
    const int lane = threadIdx.x & 31;
    for (int64_t bag = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; bag < bags;
         bag += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t s = off[bag], e = off[bag + 1];
        for (int64_t j = s + lane; j < e; j += 32)
            ids[j] = (int32_t)(gen_u64(seed, kTagId, (uint64_t)bag * max_len + (j - s)) %
                               (uint64_t)rows);
    }
}

__global__ void pack_slices_kernel(int S, const int64_t* __restrict__ bounds, const int32_t* __restrict__ ids,
                                   int64_t cap, int32_t* __restrict__ out, int32_t* __restrict__ overflow) {
    for (int o = blockIdx.y; o < S; o += gridDim.y) {
        const int64_t b0 = bounds[o];
        int64_t cnt = bounds[o + 1] - b0;
        if (cnt > cap) {
            if (blockIdx.x == 0 && threadIdx.x == 0) *overflow = 1;
            cnt = cap;
        }
        int32_t* dst = out + (int64_t)o * cap;
        const int32_t* src = ids + b0;
        for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < cnt;
             j += (int64_t)gridDim.x * blockDim.x)
            dst[j] = src[j];
    }
}

__global__ void widen_kernel(int64_t n, const int32_t* __restrict__ in, int64_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = in[i];
}

__global__ void synth_dom_kernel(int64_t n, int G, uint64_t seed, int32_t* dom) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dom[i] = (int32_t)(gen_u64(seed, kTagDom, (uint64_t)i) % (uint64_t)G);
}

// ---- K6: stable counting sort by domain, one CTA of 1024 threads -----------------------
constexpr int kBucketThreads = 1024;
constexpr int kMaxDomains = 32;

// Stable counting sort of the batch by domain in three short kernels (coalesced, one thread per
// sample): per-block domain histograms -> one block scans them into per-(block, domain) bases and
// the segment starts -> every sample's rank among the earlier same-domain samples of its block
// (warp match + per-warp prefix). A domain outside [0, G) counts as domain 0.
__device__ __forceinline__ int bucket_domain(const int32_t* __restrict__ dom, int64_t B, int G, int64_t b) {
    if (b >= B) return G;  // padding lane: a class of its own, never stored
    const int g = dom[b];
    return g >= 0 && g < G ? g : 0;
}

__global__ void __launch_bounds__(kBucketThreads) bucket_hist_kernel(int64_t B, int G, const int32_t* __restrict__ dom,
                                                                     int32_t* __restrict__ hist,
                                                                     unsigned long long* bad) {
    __shared__ int32_t h[kMaxDomains];
    if (threadIdx.x < kMaxDomains) h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t b = (int64_t)blockIdx.x * kBucketThreads + threadIdx.x;
    if (bad && b < B && (dom[b] < 0 || dom[b] >= G)) atomicMin(bad, (unsigned long long)b);  // first offender
    const int g = bucket_domain(dom, B, G, b);
    // one atomic per (warp, domain)
    const unsigned same = __match_any_sync(0xffffffffu, g);
    if (g < G && (threadIdx.x & 31) == __ffs(same) - 1) atomicAdd(&h[g], __popc(same));
    __syncthreads();
    if (threadIdx.x < G) hist[(int64_t)blockIdx.x * G + threadIdx.x] = h[threadIdx.x];
}

// one block: base[blk][g] = samples of domain g in blocks < blk; seg[g] = first row of domain g
__global__ void __launch_bounds__(kBucketThreads) bucket_scan_kernel(int64_t nblk, int G, const int32_t* __restrict__ hist,
                                                                     int32_t* __restrict__ base, int32_t* __restrict__ seg) {
    __shared__ int32_t tot[kMaxDomains + 1];
    const int g = threadIdx.x;
    if (g < G) {
        int run = 0;
        for (int64_t k = 0; k < nblk; ++k) {
            const int c = hist[k * G + g];
            base[k * G + g] = run;
            run += c;
        }
        tot[g] = run;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int run = 0;
        for (int q = 0; q < G; ++q) {
            const int c = tot[q];
            seg[q] = run;
            tot[q] = run;
            run += c;
        }
        seg[G] = run;
    }
}

__global__ void __launch_bounds__(kBucketThreads) bucket_rank_kernel(int64_t B, int G, const int32_t* __restrict__ dom,
                                                                     const int32_t* __restrict__ base,
                                                                     const int32_t* __restrict__ seg,
                                                                     int32_t* __restrict__ pos, int32_t* __restrict__ order) {
    __shared__ int32_t wcnt[kMaxDomains][32];  // [domain][warp] -> exclusive prefix over warps
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < kMaxDomains * 32; i += kBucketThreads) (&wcnt[0][0])[i] = 0;
    __syncthreads();
    const int64_t b = (int64_t)blockIdx.x * kBucketThreads + threadIdx.x;
    const int g = bucket_domain(dom, B, G, b);
    const unsigned same = __match_any_sync(0xffffffffu, g);
    const int rank = __popc(same & ((1u << lane) - 1u));
    if (g < G && lane == __ffs(same) - 1) wcnt[g][warp] = __popc(same);
    __syncthreads();
    if (warp < G) {  // warp q scans domain q's 32 per-warp counts
        const int v = wcnt[warp][lane];
        int incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int n = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += n;
        }
        wcnt[warp][lane] = incl - v;
    }
    __syncthreads();
    if (g < G) {
        const int p = seg[g] + base[(int64_t)blockIdx.x * G + g] + wcnt[g][warp] + rank;
        pos[b] = p;
        order[p] = (int32_t)b;
    }
}

// ---- row-wise rms_norm / swish_rn / swish_rn_hard, one warp per row ---------------------
__global__ void rownorm_kernel(int mode, int64_t rows, int64_t width, float eps,
                               const float* __restrict__ x, float* __restrict__ out,
                               unsigned long long* err) {
    const int lane = threadIdx.x & 31;
    for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < rows;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const float* xr = x + r * width;
        float ss = 0.0f;
        bool bad = false;
        for (int64_t c = lane; c < width; c += 32) {
            const float v = xr[c];
            bad |= !isfinite(v);
            ss += v * v;
        }
        ss = warp_sum(ss);
        if (__any_sync(0xffffffffu, bad) && lane == 0) atomicMin(err, (unsigned long long)r);
        const float denom = sqrtf(ss / (float)width + eps);
        for (int64_t c = lane; c < width; c += 32) {
            const float v = xr[c] / denom;
            out[r * width + c] = mode == 0 ? v : act_swish(v, mode == 2);
        }
    }
}

unsigned grid_for(int64_t n, int threads) {
    int64_t b = (n + threads - 1) / threads;
    const int64_t cap = (int64_t)num_sms() * 16;
    return (unsigned)std::max<int64_t>(1, std::min(b, cap));
}

lattice_status sync_err(unsigned long long* err, cudaStream_t st, unsigned long long* host) {
    *host = ~0ull;
    cudaError_t e = cudaMemcpyAsync(host, err, sizeof(*host), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    return e == cudaSuccess ? LATTICE_OK : check_cuda(e, "error readback");
}

}  // namespace
// lattice_domain_bucket with a caller-owned workspace of bucket_workspace(B, G) int32
// (hist | base per block); lattice_net keeps one so a step does no allocation
int64_t bucket_workspace(int64_t B, int G) { return 2 * ((B + kBucketThreads - 1) / kBucketThreads) * G; }

lattice_status bucket_ws(int64_t B, int G, const int32_t* dom, int32_t* pos, int32_t* order, int32_t* seg,
                         int32_t* ws, cudaStream_t stream, unsigned long long* bad) {
    const int64_t nblk = (B + kBucketThreads - 1) / kBucketThreads;
    bucket_hist_kernel<<<(unsigned)nblk, kBucketThreads, 0, stream>>>(B, G, dom, ws, bad);
    bucket_scan_kernel<<<1, kBucketThreads, 0, stream>>>(nblk, G, ws, ws + nblk * G, seg);
    bucket_rank_kernel<<<(unsigned)nblk, kBucketThreads, 0, stream>>>(B, G, dom, ws + nblk * G, seg, pos, order);
    LAT_CUDA(cudaGetLastError());
    return LATTICE_OK;
}

}  // namespace lat

extern "C" {

lattice_status lattice_embedding_bag(const lattice_bag_args* a, lattice_stream stream) {
    using namespace lat;
    LAT_REQUIRE(a != nullptr, "lattice_embedding_bag: null args");
    LAT_REQUIRE(a->features >= 0 && a->batch >= 0 && a->dim > 0, "embedding_bag: bad sizes");
    LAT_REQUIRE(a->table_dtype == LATTICE_F32 || a->table_dtype == LATTICE_BF16,
                "embedding_bag: table dtype must be f32 or bf16");
    LAT_REQUIRE(a->out_dtype == LATTICE_F32 || a->out_dtype == LATTICE_BF16,
                "embedding_bag: out dtype must be f32 or bf16");
    LAT_REQUIRE(a->out_row_stride >= (int64_t)(a->out_feature_offset + a->features) * a->dim,
                "embedding_bag: out_row_stride too small");
    if ((int64_t)a->features * a->batch == 0) return LATTICE_OK;
    LAT_REQUIRE((int64_t)(a->sources > 1 ? a->sources : 1) * a->features * a->batch < (1ll << 31),
                "embedding_bag: sources * features * batch must be < 2^31");
    LAT_REQUIRE(a->tables && a->rows && a->offsets && a->out, "embedding_bag: null pointer");
    const int esize = a->table_dtype == LATTICE_F32 ? 4 : 2;
    const int row_bytes = a->dim * esize;
    const int out_chunk = (a->out_dtype == LATTICE_F32 ? 4 : 2) * (16 / esize);
    LAT_REQUIRE(out_chunk == 8 || out_chunk == 16 || out_chunk == 32,
                "embedding_bag: unsupported dtype combination");

    unsigned long long* err = nullptr;  // [0] first bad id (init ~0), [1] work-claim counter (init 0)
    LAT_CUDA(cudaMallocAsync(&err, 2 * sizeof(*err), stream));
    LAT_CUDA(cudaMemsetAsync(err, 0xff, sizeof(*err), stream));
    LAT_CUDA(cudaMemsetAsync(err + 1, 0, sizeof(*err), stream));
    BagParams p{a->features, a->batch, a->dim, a->tables, a->rows, a->offsets, a->ids, a->out,
                a->out_row_stride, a->out_feature_offset, a->sample_pos, a->normalize, err,
                a->sources > 1 ? a->sources : 1, a->slice_cap > 0 ? a->slice_cap : 0, err + 1,
                bag_l2keep(), 0, 0, 0, 0, 0, nullptr, nullptr, nullptr, nullptr, 0};
    fastdiv((uint32_t)p.B, &p.mB, &p.sB);
    fastdiv((uint32_t)p.F, &p.mF, &p.sF);
    fastdiv((uint32_t)((p.B + staged::kChunk - 1) / staged::kChunk), &p.mC, &p.sC);  // chunks per segment
    fastdiv((uint32_t)p.R, &p.mR, &p.sR);
    lattice_status st;
    if (a->table_dtype == LATTICE_F32)
        st = a->out_dtype == LATTICE_F32 ? launch_bag<float, float>(p, row_bytes, stream)
                                         : launch_bag<float, __nv_bfloat16>(p, row_bytes, stream);
    else
        st = a->out_dtype == LATTICE_F32
                 ? launch_bag<__nv_bfloat16, float>(p, row_bytes, stream)
                 : launch_bag<__nv_bfloat16, __nv_bfloat16>(p, row_bytes, stream);
    if (st != LATTICE_OK) {
        cudaFreeAsync(err, stream);
        return st;
    }
    cudaError_t le = cudaGetLastError();
    unsigned long long host = ~0ull;
    if (le == cudaSuccess && a->check) {
        lattice_status s2 = sync_err(err, stream, &host);
        if (s2 != LATTICE_OK) {
            cudaFreeAsync(err, stream);
            return s2;
        }
    }
    cudaFreeAsync(err, stream);
    if (le != cudaSuccess) return check_cuda(le, "bag_kernel");
    if (host != ~0ull)
        return set_error(LATTICE_DATA,
                         "embedding_bag: id at position " + std::to_string(host) + " is outside its table",
                         (int64_t)host);
    return LATTICE_OK;
}

lattice_status lattice_peer_embedding_bag(const lattice_peer_bag_args* a, lattice_stream stream) {
    using namespace lat;
    LAT_REQUIRE(a != nullptr, "peer_embedding_bag: null args");
    LAT_REQUIRE(a->world >= 1 && a->rank >= 0 && a->rank < a->world, "peer_embedding_bag: bad rank/world");
    LAT_REQUIRE(a->features_local >= 0 && a->batch >= 0 && a->dim > 0, "peer_embedding_bag: bad sizes");
    LAT_REQUIRE(a->table_dtype == LATTICE_F32 || a->table_dtype == LATTICE_BF16,
                "peer_embedding_bag: table dtype must be f32 or bf16");
    LAT_REQUIRE(a->out_dtype == LATTICE_F32 || a->out_dtype == LATTICE_BF16,
                "peer_embedding_bag: out dtype must be f32 or bf16");
    LAT_REQUIRE(a->feature_base >= 0 && a->out_row_stride >= (int64_t)(a->feature_base + a->features_local) * a->dim,
                "peer_embedding_bag: out_row_stride too small for the owned feature block");
    if ((int64_t)a->features_local * a->batch == 0) return LATTICE_OK;
    LAT_REQUIRE((int64_t)a->world * a->features_local * a->batch < (1ll << 31),
                "peer_embedding_bag: world * features_local * batch must be < 2^31");
    LAT_REQUIRE(a->tables && a->rows && a->offsets && a->ids && a->sample_pos && a->out,
                "peer_embedding_bag: null pointer");
    const int esize = a->table_dtype == LATTICE_F32 ? 4 : 2;
    const int row_bytes = a->dim * esize;
    const int out_chunk = (a->out_dtype == LATTICE_F32 ? 4 : 2) * (16 / esize);
    LAT_REQUIRE(out_chunk == 8 || out_chunk == 16 || out_chunk == 32,
                "peer_embedding_bag: unsupported dtype combination");
    unsigned long long* err = nullptr;
    LAT_CUDA(cudaMallocAsync(&err, 2 * sizeof(*err), stream));
    LAT_CUDA(cudaMemsetAsync(err, 0xff, sizeof(*err), stream));
    LAT_CUDA(cudaMemsetAsync(err + 1, 0, sizeof(*err), stream));
    BagParams p{a->features_local, a->batch, a->dim, a->tables, a->rows, nullptr, nullptr, nullptr,
                a->out_row_stride, a->feature_base, nullptr, a->normalize, err, a->world, 0, err + 1,
                bag_l2keep(), 0, 0, 0, 0, 1, a->offsets, a->ids, a->sample_pos, a->out, a->feature_base};
    fastdiv((uint32_t)p.B, &p.mB, &p.sB);
    fastdiv((uint32_t)p.F, &p.mF, &p.sF);
    fastdiv((uint32_t)((p.B + staged::kChunk - 1) / staged::kChunk), &p.mC, &p.sC);  // chunks per segment
    fastdiv((uint32_t)p.R, &p.mR, &p.sR);
    lattice_status st;
    if (a->table_dtype == LATTICE_F32)
        st = a->out_dtype == LATTICE_F32 ? launch_bag<float, float>(p, row_bytes, stream)
                                         : launch_bag<float, __nv_bfloat16>(p, row_bytes, stream);
    else
        st = a->out_dtype == LATTICE_F32
                 ? launch_bag<__nv_bfloat16, float>(p, row_bytes, stream)
                 : launch_bag<__nv_bfloat16, __nv_bfloat16>(p, row_bytes, stream);
    const cudaError_t le = cudaGetLastError();
    unsigned long long host = ~0ull;
    if (st == LATTICE_OK && le == cudaSuccess && a->check) st = sync_err(err, stream, &host);
    cudaFreeAsync(err, stream);
    if (st != LATTICE_OK) return st;
    if (le != cudaSuccess) return check_cuda(le, "bag_kernel (peer)");
    if (host != ~0ull)
        return set_error(LATTICE_DATA,
                         "embedding_bag: id at position " + std::to_string(host) + " is outside its table",
                         (int64_t)host);
    return LATTICE_OK;
}

lattice_status lattice_pack_slices(int32_t slices, const int64_t* bounds, const int32_t* ids, int64_t cap,
                                   int32_t* out, int32_t* overflow, lattice_stream stream) {
    using namespace lat;
    LAT_REQUIRE(slices > 0 && cap > 0 && bounds && ids && out && overflow, "pack_slices: bad args");
    dim3 grid((unsigned)(num_sms() * 4 / slices > 0 ? num_sms() * 4 / slices : 1), (unsigned)slices);
    pack_slices_kernel<<<grid, 256, 0, stream>>>(slices, bounds, ids, cap, out, overflow);
    LAT_CUDA(cudaGetLastError());
    return LATTICE_OK;
}

lattice_status lattice_lengths_to_offsets(int64_t n, const int32_t* lengths, int64_t* offsets,
                                          lattice_stream stream) {
    using namespace lat;
    LAT_REQUIRE(n >= 0 && offsets, "lengths_to_offsets: bad args");
    if (n == 0) {
        LAT_CUDA(cudaMemsetAsync(offsets, 0, sizeof(int64_t), stream));
        return LATTICE_OK;
    }
    LAT_REQUIRE(lengths != nullptr, "lengths_to_offsets: null lengths");
    LAT_CUDA(cudaMemsetAsync(offsets, 0, sizeof(int64_t), stream));
    widen_kernel<<<grid_for(n, 256), 256, 0, stream>>>(n, lengths, offsets + 1);  // int64 accumulation
    size_t tmp_bytes = 0;
    LAT_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, offsets + 1, offsets + 1, n, stream));
    void* tmp = nullptr;
    LAT_CUDA(cudaMallocAsync(&tmp, tmp_bytes, stream));
    LAT_CUDA(cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, offsets + 1, offsets + 1, n, stream));
    cudaFreeAsync(tmp, stream);
    return LATTICE_OK;
}

lattice_status lattice_fill_tables(void* tables, int32_t dtype, int32_t F, int64_t rows, int32_t D,
                                   uint64_t seed, int32_t feature_base, int64_t rows_total,
                                   lattice_stream stream) {
    using namespace lat;
    LAT_REQUIRE(tables && F >= 0 && rows > 0 && D > 0, "fill_tables: bad args");
    if (rows_total <= 0) rows_total = rows;
    const int64_t n = (int64_t)F * rows * D;
    fill_tables_kernel<<<grid_for(n, 256), 256, 0, stream>>>(tables, dtype, n, D, rows, rows_total,
                                                             feature_base, seed);
    LAT_CUDA(cudaGetLastError());
    return LATTICE_OK;
}

lattice_status lattice_fill_weights(void* w, int32_t dtype, int64_t out_features, int64_t fan_in,
                                    uint64_t seed, uint64_t tag, lattice_stream stream) {
    using namespace lat;
    LAT_REQUIRE(w && out_features > 0 && fan_in > 0, "fill_weights: bad args");
    const int64_t n = out_features * fan_in;
    fill_weights_kernel<<<grid_for(n, 256), 256, 0, stream>>>(w, dtype, n, fan_in,
                                                              weight_shift(fan_in), seed, tag);
    LAT_CUDA(cudaGetLastError());
    return LATTICE_OK;
}

lattice_status lattice_synth_bags(int32_t F, int64_t B, int32_t max_len, int64_t rows, uint64_t seed,
                                  int64_t* offsets, int32_t* ids, lattice_stream stream) {
    using namespace lat;
    LAT_REQUIRE(F > 0 && B > 0 && max_len >= 0 && rows > 0 && offsets && ids, "synth_bags: bad args");
    const int64_t bags = (int64_t)F * B;
    int64_t* len = nullptr;
    LAT_CUDA(cudaMallocAsync(&len, sizeof(int64_t) * (bags + 1), stream));
    synth_len_kernel<<<grid_for(bags, 256), 256, 0, stream>>>(bags, max_len, seed, len);
    LAT_CUDA(cudaMemsetAsync(len + bags, 0, sizeof(int64_t), stream));
    size_t tmp_bytes = 0;
    LAT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, len, offsets, bags + 1, stream));
    void* tmp = nullptr;
    LAT_CUDA(cudaMallocAsync(&tmp, tmp_bytes, stream));
    LAT_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, len, offsets, bags + 1, stream));
    synth_ids_kernel<<<grid_for(bags * 32, 256), 256, 0, stream>>>(bags, max_len, rows, seed,
                                                                   offsets, ids);
    LAT_CUDA(cudaGetLastError());
    cudaFreeAsync(tmp, stream);
    cudaFreeAsync(len, stream);
    return LATTICE_OK;
}

lattice_status lattice_synth_domains(int64_t B, int32_t G, uint64_t seed, int32_t* dom,
                                     lattice_stream stream) {
    using namespace lat;
    LAT_REQUIRE(B >= 0 && G > 0 && dom, "synth_domains: bad args");
    if (!B) return LATTICE_OK;
    synth_dom_kernel<<<grid_for(B, 256), 256, 0, stream>>>(B, G, seed, dom);
    LAT_CUDA(cudaGetLastError());
    return LATTICE_OK;
}

lattice_status lattice_domain_bucket(int64_t B, int32_t G, const int32_t* dom, int32_t* pos,
                                     int32_t* order, int32_t* seg, lattice_stream stream) {
    using namespace lat;
    LAT_REQUIRE(B >= 0 && B < (1ll << 31) && G > 0 && G <= kMaxDomains, "domain_bucket: bad sizes");
    LAT_REQUIRE(dom && pos && order && seg, "domain_bucket: null pointer");
    if (B == 0) {
        LAT_CUDA(cudaMemsetAsync(seg, 0, sizeof(int32_t) * (G + 1), stream));
        return LATTICE_OK;
    }
    int32_t* ws = nullptr;
    LAT_CUDA(cudaMallocAsync(&ws, sizeof(int32_t) * bucket_workspace(B, G), stream));
    const lattice_status st = bucket_ws(B, G, dom, pos, order, seg, ws, stream);
    cudaFreeAsync(ws, stream);
    return st;
}

lattice_status lattice_rownorm(int32_t mode, int64_t rows, int64_t width, double eps, const float* x,
                               float* out, int32_t check, lattice_stream stream) {
    using namespace lat;
    LAT_REQUIRE(mode >= 0 && mode <= 2, "rownorm: mode must be 0, 1 or 2");
    LAT_REQUIRE(eps > 0.0, "eps must be > 0");  // numerics.hpp:20
    LAT_REQUIRE(width > 0, "rms_norm: empty input");  // numerics.hpp:83
    if (rows <= 0) return LATTICE_OK;
    unsigned long long* err = nullptr;
    LAT_CUDA(cudaMallocAsync(&err, sizeof(*err), stream));
    LAT_CUDA(cudaMemsetAsync(err, 0xff, sizeof(*err), stream));
    rownorm_kernel<<<grid_for(rows * 32, 256), 256, 0, stream>>>(mode, rows, width, (float)eps, x,
                                                                 out, err);
    cudaError_t le = cudaGetLastError();
    unsigned long long host = ~0ull;
    if (le == cudaSuccess && check) {
        lattice_status s2 = sync_err(err, stream, &host);
        if (s2 != LATTICE_OK) {
            cudaFreeAsync(err, stream);
            return s2;
        }
    }
    cudaFreeAsync(err, stream);
    if (le != cudaSuccess) return check_cuda(le, "rownorm_kernel");
    if (host != ~0ull)
        return set_error(LATTICE_DATA, "rms_norm: non-finite input", (int64_t)host);
    return LATTICE_OK;
}

}  // extern "C"
