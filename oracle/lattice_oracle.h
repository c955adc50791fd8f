/*
 * lattice_oracle.h -- CPU restatement of the Lattice hot path. TEST INFRASTRUCTURE ONLY.
 *
 * This library is the checker, never the product: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it. The shipped path is
 * paper_2512_09200_b200/liblattice_b200.so (CUDA, sm_100a) and has no CPU fallback.
 *
 * Parity status
 *   - XXH64, canonical signature bytes, assign_window, zip labels: PINNED. Checked against
 *     the reference's frozen goldens (proj/tests/test_core.cpp:18-43), the SPEC examples
 *      and, bit for bit, against the reference headers compiled into
 *     oracle/_ref/libref.so (see oracle/Makefile, oracle/ref_shim.cpp).
 *   - rms_norm / swish_rn / swish_rn_hard: PINNED against oracle/_ref (numerics.hpp:81-107)
 *     and the known answers of proj/tests/test_numerics.cpp:93-149.
 *   - Embedding-bag, FMB/LCB blocks, towers: the reference has no code for them
 *     (PAPER.md:265-318 prose only). This part is "parity unpinned"
 *     beyond the norm/activation pieces it reuses; its arithmetic is written down in
 *     DESIGN.md section 3.
 */
#ifndef LATTICE_ORACLE_H
#define LATTICE_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- core.hpp:84-139 ---------------------------------------------------------------- */
uint64_t lo_xxh64(const uint8_t* data, size_t len, uint64_t seed);

/* Counter-based generator used for every synthetic input:
 * XXH64 over the 16 bytes LE64(tag) || LE64(idx), seeded with `seed`. */
uint64_t lo_gen(uint64_t seed, uint64_t tag, uint64_t idx);

/* ---- datasets.hpp:179-194 ------------------------------------------------------------ */
/* Canonical signature (core.hpp:149-175 as used at datasets.hpp:181-184). Writes
 * 16 + ulen + alen bytes into out (caller sized) and returns that length. */
size_t lo_signature(const uint8_t* user, uint32_t ulen, const uint8_t* ad, uint32_t alen,
                    int64_t ts, uint8_t* out);
int lo_assign_window(const uint8_t* user, uint32_t ulen, const uint8_t* ad, uint32_t alen,
                     int64_t ts, uint64_t seed, const double* probs, int windows);

/* ---- datasets.hpp:199-249 (columnar) ------------------------------------------------- */
/* Records in columns: user/ad strings packed with int64 offsets (n+1 entries), impression
 * time ts[n], conversions conv[n*T] with presence flags conv_present[n*T] (task-major per
 * record). Writes window[n] and labels[n*T*W] (labels[(i*T+t)*W+w], datasets.hpp:92).
 * Returns -1 when every record is valid, else the index of the first record whose
 * conversion precedes its impression (*err_task = its task), matching the record order
 * and task order in which zip_dataset throws (datasets.hpp:231-238). */
int64_t lo_zip_columns(int64_t n, const uint8_t* user_bytes, const int64_t* user_off,
                       const uint8_t* ad_bytes, const int64_t* ad_off, const int64_t* ts,
                       int T, const int64_t* conv, const uint8_t* conv_present, int W,
                       const int64_t* durations, const double* probs, uint64_t seed,
                       uint8_t* window, uint8_t* labels, int32_t* err_task);

/* ---- numerics.hpp:81-107 ------------------------------------------------------------- */
/* Return 0 on success, 1 on UsageError (empty input / eps <= 0), 2 on DataError (non-finite). */
int lo_rms_norm(const double* x, size_t n, double eps, double* out);
int lo_swish_rn(const double* x, size_t n, double eps, double* out);
int lo_swish_rn_hard(const double* x, size_t n, double eps, double* out);

/* ---- synthetic values ------------------------------------------ */
enum {
    LO_TAG_TABLE = 0x4c54424cull, /* table values */
    LO_TAG_LEN = 0x4c4c454eull,   /* bag lengths  */
    LO_TAG_ID = 0x4c494420ull,    /* bag ids      */
    LO_TAG_DOM = 0x4c444f4dull    /* sample domain */
};
/* T_f[r][c] = (int8)(H >> 56) * 2^-10, idx = (f*rows + r)*D + c. Exact in fp32 and bf16. */
float lo_table_value(uint64_t seed, int64_t f, int64_t r, int D, int64_t rows, int64_t c);
/* Weight element (o, i) of a tensor with fan_in inputs:
 * (int8)(H(seed, tag, o*fan_in + i) >> 56) * 2^-(7 + floor(log2(fan_in)/2)). Exact in bf16. */
float lo_weight_value(uint64_t seed, uint64_t tag, int64_t o, int64_t i, int64_t fan_in);
int lo_weight_shift(int64_t fan_in);
/* Whole [out_features][fan_in] tensor of lo_weight_value, OpenMP-parallel. */
void lo_fill_weights(float* out, int64_t out_features, int64_t fan_in, uint64_t seed, uint64_t tag);
uint64_t lo_weight_tag(int block, int kind, int index);

/* ---- embedding bag (builder semantics in DESIGN.md 3.1) ----------------- */
/* Feature-major CSR: bag (f, b) owns ids[offsets[f*B+b] .. offsets[f*B+b+1]). Sum pooling,
 * empty bag -> 0. Tables are the synthetic values above (never materialised). Computes
 * samples [b_lo, b_hi) into out[(b - b_lo)][f][c] (fp32, exact). Returns -1 or the index of
 * the first id (position in ids) outside [0, rows). */
int64_t lo_embedding_bag_synth(uint64_t seed, int F, int64_t rows, int D, int64_t B,
                               const int64_t* offsets, const int32_t* ids, int64_t b_lo,
                               int64_t b_hi, float* out, int threads);
/* Same over explicit fp32 tables (tables[f] -> rows*D floats). */
int64_t lo_embedding_bag(int F, const int64_t* rows, int D, int64_t B,
                         const float* const* tables, const int64_t* offsets,
                         const int32_t* ids, float* out);

/* lengths/ids/domains exactly as lattice_synth_bags / lattice_synth_domains. ids must hold
 * F*B*max_len entries. */
void lo_synth_bags(int F, int64_t B, int max_len, int64_t rows, uint64_t seed, int64_t* offsets,
                   int32_t* ids);
void lo_synth_domains(int64_t B, int G, uint64_t seed, int32_t* dom);

/* ---- network forward -------------------------------------------- */
typedef struct {
    int n;          /* embeddings per sample (= sparse features F) */
    int d;          /* embedding dim D */
    int blocks;     /* DWFB blocks l */
    int nF, nL, k;  /* FMB output embeddings, LCB output embeddings, FM rank */
    int n_mlp;      /* number of FMB MLP weight matrices (>= 1) */
    int mlp[6];     /* widths: mlp[0] = n*k, ..., mlp[n_mlp] = nF*d */
    int G, heads;   /* domains, heads per domain (= objectives * windows) */
    int tower_hidden;
    int hard;       /* 1: swish_rn_hard activations */
    int bf16;       /* 1: emulate bf16 rounding at every stored activation */
} lo_net_cfg;

typedef struct {
    const float* const* YT;    /* [blocks] -> [k][n]        */
    const float* const* WL;    /* [blocks] -> [nL][n]       */
    const float* const* mlp;   /* [blocks*n_mlp] -> [out][in] */
    const float* T1;           /* [G][tower_hidden][n*d]    */
    const float* T2;           /* [G][heads][tower_hidden]  */
} lo_net_weights;

/* X0: pooled embeddings before the input norm, [count][n][d]; dom[count].
 * logits: [count][heads]. Parallel over samples with `threads` OpenMP threads. */
void lo_net_forward(const lo_net_cfg* cfg, const lo_net_weights* w, int64_t count,
                    const float* pooled, const int32_t* dom, float* logits, int threads);

/* ---- dense features -------------------------------------------------
 * lo_merge_dense: the value side of merge_domains (datasets.hpp:144-173) over columns --
 * out[b][c] = values[b][src_col[g_b][c]] or 0 (the pad) when src_col is -1; bf16 = 1 rounds to
 * bf16. Returns the first record with a domain outside [0, G), or -1.
 * lo_dense_processor: PAPER.md:277 -- O_d = D2 . q(act(D1 . x)) per sample, each value q()-rounded
 * (the GPU stores it in the net dtype), written as raw rows [nc, nc + n_dense) of pooled
 * ([count][n][d]) so lo_net_forward's mixing norm treats it like the pooled sparse rows. */
int64_t lo_merge_dense(int64_t n, int G, int max_decl, const int32_t* domain, const float* values,
                       const int32_t* src_col, int width, int bf16, float* out);
void lo_dense_processor(const lo_net_cfg* cfg, int n_dense, int dense_in, int dense_hidden,
                        const float* D1, const float* D2, int64_t count, const float* dense,
                        float* pooled, int threads);

/* ---- KTAP student inputs and numerics element ops --------------------
 * lo_swish_rn_jvp numerics.hpp:113-136; lo_clip_features :139-144; lo_smooth_labels :147-156
 * (returns 1 for a label other than 0/1). Return codes 0 / 1 UsageError / 2 DataError.
 * lo_student_inputs: ktap.hpp:133-152 (hit = entry exists and now - written_at <= ttl;
 * smoothed logit on read) + :221-229 ([base || embedding or zeros]) with the teacher block
 * clipped (clip > 0). bf16 = 1 rounds the row to bf16. Logit NaN on a miss. */
int lo_swish_rn_jvp(const double* x, const double* t, size_t n, double eps, double* out);
int lo_clip_features(const double* x, size_t n, double c, double* out);
int lo_smooth_labels(const double* y, size_t n, double eps_s, double* out);
void lo_student_inputs(int64_t n, int base_dim, int dim, const float* base, const int64_t* slot,
                       const float* store_emb, const float* store_logit, const int64_t* written_at,
                       int64_t ttl, int64_t now, double clip, double smoothing, int bf16, float* out,
                       float* logit, uint8_t* hit);

/* ---- post-tower reductions ----------------------------------------
 * lo_correlation_loss: numerics.hpp:46-78 (1 - Cov/(sx*sy+eps), population moments, two
 * passes, clamped to [0,2], 1.0 when either side is constant). Returns 0 ok, 1 UsageError
 * (eps <= 0, n < 2), 2 DataError (non-finite).
 * lo_window_summary: datasets.hpp:262-283 -- counts[w] records routed to window w and
 * positives[w][t] of their own-window labels (rate = positives / count, 0 when count = 0).
 * Returns 1 (UsageError) for a window >= W.
 * lo_routed_objectives: the batch step the GPU fuses -- routed[b][t] = logits[b][t*W + w_b],
 * y = labels[b][t][w_b], p = stable_sigmoid(routed) (numerics.hpp:29-33, fp64), corr[t] =
 * correlation_loss(y[:, t], p[:, t]) and the window summary. */
int lo_correlation_loss(const double* x, const double* y, size_t n, double eps, double* out);
int lo_window_summary(int64_t n, int T, int W, const uint8_t* window, const uint8_t* labels,
                      int64_t* counts, int64_t* positives);
int lo_routed_objectives(int64_t n, int T, int W, const float* logits, const uint8_t* window,
                         const uint8_t* labels, double eps, float* routed, double* corr,
                         int64_t* counts, int64_t* positives);

/* Round-to-nearest-even to bf16, returned as float. */
float lo_bf16_round(float x);

#ifdef __cplusplus
}
#endif
#endif
