/*
 * lattice_b200.h -- C ABI of the B200-native Lattice hot path (liblattice_b200.so).
 *
 * Plain pointers and sizes only; all array arguments are DEVICE pointers on the current
 * CUDA device unless stated otherwise, caller-owned, and every call is ordered on the
 * stream it is given. No call falls back to the CPU: without a usable sm_100a device the
 * library returns LATTICE_CUDA.
 *
 * Status codes follow the reference's error model (proj/include/lattice/core.hpp:20-27,
 * CLI exit codes proj/tools/lattice_cli.cpp:342-351): USAGE = UsageError (contract
 * violation), DATA = DataError (bad input data). lattice_last_error() returns the message
 * of the last failing call on this thread; lattice_last_error_index() the offending
 * record / id index when the failure is a DATA error.
 *
 * Which reference interface each entry replaces is cited per declaration; INTEGRATION.md
 * shows the C++ drop-in (include/lattice/ headers) and a ctypes binding.
 */
#ifndef LATTICE_B200_H
#define LATTICE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    LATTICE_OK = 0,
    LATTICE_USAGE = 1, /* UsageError  (core.hpp:20-22) */
    LATTICE_DATA = 2,  /* DataError   (core.hpp:25-27) */
    LATTICE_CUDA = 3,
    LATTICE_NCCL = 4
} lattice_status;

typedef enum { LATTICE_F32 = 0, LATTICE_BF16 = 1, LATTICE_F64 = 2 } lattice_dtype;  /* F64: host-API values only */

typedef struct CUstream_st* lattice_stream; /* == cudaStream_t; NULL = legacy default stream */

const char* lattice_last_error(void);
int64_t lattice_last_error_index(void);
int lattice_abi_version(void); /* bumps on any signature change */

/* ======================================================================================
 * Hashing -- replaces lattice::stable_hash (core.hpp:84-145) for batches.
 * Strings packed back to back in `bytes`, string i = bytes[off[i] .. off[i+1]).
 * ==================================================================================== */
lattice_status lattice_stable_hash(int64_t n, const uint8_t* bytes, const int64_t* off,
                                   uint64_t seed, uint64_t* out, lattice_stream stream);

/* ======================================================================================
 * Zipper -- replaces lattice::ZipperConfig::create (datasets.hpp:60-84, validation),
 * lattice::assign_window (datasets.hpp:179-194) and the label loop of
 * lattice::zip_dataset (datasets.hpp:199-249), bit-exact.
 * ==================================================================================== */
/* Host-side validation of the numeric part of ZipperConfig::create: >= 1 window,
 * durations > 0 and strictly increasing, probabilities >= 0 finite, |sum - 1| <= 1e-9.
 * (Window names are checked by the C++ shim, include/lattice/datasets.hpp.) HOST pointers. */
lattice_status lattice_zipper_validate(int32_t windows, const int64_t* durations_host,
                                       const double* probabilities_host);

typedef struct {
    int64_t n;                  /* impressions */
    const uint8_t* user_bytes;  /* packed user ids */
    const int64_t* user_off;    /* [n+1] */
    const uint8_t* ad_bytes;    /* packed ad ids */
    const int64_t* ad_off;      /* [n+1] */
    const int64_t* ts;          /* impression_time_ms [n] */
    int32_t tasks;              /* T */
    const int64_t* conv;        /* conversion time [n][T] */
    const uint8_t* conv_present;/* [n][T]: 0 = no conversion for that task */
    int32_t windows;            /* W (<= 255) */
    const int64_t* durations_host;      /* [W] HOST */
    const double* probabilities_host;   /* [W] HOST */
    uint64_t seed;              /* ZipperConfig.seed */
    uint8_t* window;            /* out [n] assigned window */
    uint8_t* labels;            /* out [n][T][W] task-major per record (datasets.hpp:92) */
    uint8_t* routed;            /* optional out [n][T]: label of the assigned window */
    int32_t check;              /* 1: synchronise and return DATA on a negative delay */
} lattice_zip_args;

lattice_status lattice_zipper_assign_labels(const lattice_zip_args* args, lattice_stream stream);

/* ======================================================================================
 * Embedding bag ("embedding tables producing (B, |F_c|, d)"; no reference
 * code -- semantics in DESIGN.md 3.1). Sum pooling, fp32 accumulation, empty bag -> 0.
 * Bags in feature-major CSR: bag (f, b) = ids[offsets[f*batch + b] .. offsets[f*batch+b+1]).
 * ==================================================================================== */
typedef struct {
    int32_t features;            /* F (tables in this call) */
    int64_t batch;               /* B */
    int32_t dim;                 /* D (multiple of 8) */
    int32_t table_dtype;         /* lattice_dtype */
    const void* const* tables;   /* DEVICE array [F] of device pointers to [rows_f][D] */
    const int64_t* rows;         /* DEVICE [F] */
    const int64_t* offsets;      /* DEVICE [F*B + 1] */
    const int32_t* ids;          /* DEVICE */
    int32_t out_dtype;           /* lattice_dtype */
    void* out;                   /* out[pos(b)*out_row_stride + (out_feature_offset+f)*D + c] */
    int64_t out_row_stride;      /* elements between samples (>= features*D) */
    int32_t out_feature_offset;
    const int32_t* sample_pos;   /* optional DEVICE [B]: output row of sample b (NULL = b) */
    int32_t normalize;           /* 1: rms_norm over D of each pooled row (numerics.hpp:81) */
    int32_t check;               /* 1: synchronise and return DATA on an id outside [0, rows) */
    int32_t sources;             /* R >= 1: bags laid out [R][F][B] (after an ids all-to-all,
                                    R = source ranks); bag (r, f, b) writes output row r*B + b.
                                    0 is treated as 1. */
    int64_t slice_cap;           /* > 0: ids of source r live in the fixed slice
                                    ids[r*slice_cap ..] (static exchange buffer); offsets stay
                                    the global CSR over [R][F][B], rebased per slice. */
} lattice_bag_args;

/* ======================================================================================
 * Peer-memory sharded embedding bag (NVLink/NVSwitch; SURVEY.md 8e "K1 writes pooled rows
 * straight into peers' receive buffers"). Replaces the three-step ids all-to-all -> owner
 * pooling -> pooled all-to-all of lattice_embedding_bag(sources = R) with ONE kernel per
 * owner: this rank owns global features [feature_base, feature_base + features_local); for
 * every source rank r it reads r's CSR offsets / ids / sample_pos over NVLink (peer-mapped
 * pointers from lattice_ipc_open), gathers its own table rows from local HBM, and stores the
 * pooled (optionally rms-normalised) row at out[r][sample_pos[r][b]*out_row_stride +
 * (feature_base + f)*dim] -- i.e. straight into source r's network X0. Must be bracketed by
 * lattice_peer_barrier calls (see paper_2512_09200_b200/peer.py).
 * ==================================================================================== */
typedef struct {
    int32_t rank, world;
    int32_t features_local;      /* tables owned by this rank */
    int32_t feature_base;        /* their first global feature index */
    int64_t batch;               /* B per source rank */
    int32_t dim;
    int32_t table_dtype;
    const void* const* tables;   /* DEVICE [features_local] local table pointers */
    const int64_t* rows;         /* DEVICE [features_local] */
    const int64_t* const* offsets;   /* DEVICE [world]: rank r's CSR offsets over all features
                                        (feature-major, [F_total*B + 1]) */
    const int32_t* const* ids;       /* DEVICE [world]: rank r's ids */
    const int32_t* const* sample_pos;/* DEVICE [world]: output row of rank r's sample b */
    void* const* out;                /* DEVICE [world]: rank r's output base */
    int32_t out_dtype;
    int64_t out_row_stride;      /* elements between output rows (>= F_total*dim) */
    int32_t normalize;
    int32_t check;               /* 1: synchronise; DATA error index = position in the
                                    source's ids array */
} lattice_peer_bag_args;

lattice_status lattice_peer_embedding_bag(const lattice_peer_bag_args* args, lattice_stream stream);

/* CUDA IPC between the one-process-per-GPU ranks. lattice_ipc_handle exports the allocation
 * that contains dptr (any pointer inside a cudaMalloc'd block) as a 64-byte handle plus the
 * byte offset of dptr in it; lattice_ipc_open maps a peer's handle (peer access over
 * NVLink) and returns the pointer at `offset`; lattice_ipc_close unmaps it (reference
 * counted per allocation). */
#define LATTICE_IPC_HANDLE_BYTES 64
lattice_status lattice_ipc_handle(const void* dptr, uint8_t* handle, int64_t* offset);
lattice_status lattice_ipc_open(const uint8_t* handle, int64_t offset, void** dptr);
lattice_status lattice_ipc_close(void* dptr);

/* Stream-ordered cross-GPU barrier. flags: DEVICE array [world] of pointers (peer-mapped)
 * to every rank's zero-initialised uint32 array of world + 1 words. All ranks must call it
 * the same number of times; a rank that does not arrive within timeout_s seconds makes the
 * kernel give up and set *status = 1 (DEVICE int32) instead of hanging the GPU. */
lattice_status lattice_peer_barrier(uint32_t* const* flags, int32_t rank, int32_t world,
                                    double timeout_s, int32_t* status, lattice_stream stream);

/* Data-parallel gradient reduction fused with the optimizer over peer memory (replaces an NCCL
 * all-reduce + a separate SGD pass): rank r owns elements [r*S, (r+1)*S) of the flat gradient
' * buffer (S = ceil(n / world) rounded up to a multiple of 4); for each it sums every rank's gradient in rank order (grads:
 * DEVICE [world] peer-mapped pointers), divides by world and, per segment, either applies SGD to
 * this rank's flat fp32 master (ZeRO-1: only the owned shard [r*S, (r+1)*S) of `master` is kept
 * current) and writes the new weight (dst dtype) into EVERY rank's copy, or (mode 1) writes the
 * mean itself (e.g. a loss). Deterministic: replicas' weights stay bit-identical.
 * Bracket it with lattice_peer_barrier (gradients published before; copies written after). */
typedef struct {
    int64_t offset, count;   /* elements [offset, offset + count) of the flat buffers */
    int32_t mode;            /* 0: sgd; 1: mean */
    int32_t dst_dtype;       /* LATTICE_F32, or LATTICE_BF16 for sgd segments */
    void* const* dst;        /* DEVICE [world]: every rank's destination (element j = offset + j) */
} lattice_peer_seg;
lattice_status lattice_peer_reduce_sgd(const float* const* grads, float* master,
                                       const lattice_peer_seg* segs, int32_t nseg, int64_t n,
                                       int32_t rank, int32_t world, float lr, lattice_stream stream);

/* Sender side of the static ids exchange: out[o][j] = ids[bounds[o] + j] for
 * j < bounds[o+1] - bounds[o] (o < slices); slices longer than cap set *overflow = 1.
 * All sizes are read on the device: no host synchronisation. */
lattice_status lattice_pack_slices(int32_t slices, const int64_t* bounds, const int32_t* ids,
                                   int64_t cap, int32_t* out, int32_t* overflow,
                                   lattice_stream stream);

/* Exclusive prefix sum of bag lengths into CSR offsets (n+1 entries): the owner side of the
 * ids all-to-all rebuilds its offsets with this. */
lattice_status lattice_lengths_to_offsets(int64_t n, const int32_t* lengths, int64_t* offsets,
                                          lattice_stream stream);

lattice_status lattice_embedding_bag(const lattice_bag_args* args, lattice_stream stream);

/* ======================================================================================
 * Fused activations, row-wise -- replaces lattice::rms_norm / swish_rn / swish_rn_hard
 * (numerics.hpp:81-107) for a [rows][width] fp32 matrix. Returns DATA on non-finite input
 * (numerics.hpp:24) when check = 1. mode: 0 rms_norm, 1 swish_rn, 2 swish_rn_hard.
 * ==================================================================================== */
lattice_status lattice_rownorm(int32_t mode, int64_t rows, int64_t width, double eps,
                               const float* x, float* out, int32_t check, lattice_stream stream);
/* The same in fp64 with the reference's own arithmetic: the row's sum of squares is taken in
 * index order without FMA contraction (numerics.hpp:36-40), so rms_norm matches the host
 * reference bit for bit and swish_rn / swish_rn_hard to within exp()'s last ulp, for inputs of
 * any magnitude (a sum that overflows gives 0 rows, as in the reference). What the C++ drop-in
 * (include/lattice/numerics.hpp) calls. */
lattice_status lattice_rownorm_f64(int32_t mode, int64_t rows, int64_t width, double eps,
                                   const double* x, double* out, int32_t check, lattice_stream stream);

/* ======================================================================================
 * Dense features across consolidated domains -- replaces the value side of
 * lattice::merge_domains (datasets.hpp:144-173): records keep their domain's feature values,
 * re-laid out under the union schema with zero padding for features their domain never
 * declared. The union schema itself (first-seen union of feature names) and the
 * "undeclared feature" DataError are string-level work done by the caller / C++ drop-in,
 * which passes src_col[g][c] = index of union column c in domain g's declared order, or -1.
 * values: DEVICE [n][max_declared] in values_dtype (F32 or F64; record b's values in its
 * domain's declared order), domain: DEVICE int32 [n]. out: DEVICE [n][out_width] in out_dtype
 * (F32, BF16 or F64 -- F64 in and out is exact, what the C++ drop-in uses; columns past the
 * union width are zero: GEMM padding). A domain outside [0, domains) -> DATA (check = 1).
 * ==================================================================================== */
lattice_status lattice_merge_dense(int64_t n, int32_t domains, int32_t max_declared, const int32_t* domain,
                                   const void* values, int32_t values_dtype, const int32_t* src_col,
                                   int32_t out_width, int32_t out_dtype, void* out, int32_t check,
                                   lattice_stream stream);

/* ======================================================================================
 * KTAP student-input assembly -- replaces the read side of
 * TeacherEmbeddingStore::student_query (ktap.hpp:133-152: TTL validity inclusive at exactly
 * ttl, label smoothing of the teacher logit on read) and student_feature_vector
 * (ktap.hpp:221-229: [base || teacher embedding], zeros on a miss), with the teacher embedding
 * clipped (clip_features, numerics.hpp:139) for a batch of queries. The store's
 * key -> entry map and refresh queue stay on the host (string keys, mutex-serialised writes):
 * the caller passes each query's entry slot (-1 = absent). The output row can be the
 * network's dense input (dense_in = base_dim + dim).
 * ==================================================================================== */
typedef struct {
    int64_t n;                   /* queries */
    int32_t base_dim, dim;       /* base feature width, StoreConfig.dimension */
    const float* base;           /* [n][base_dim] */
    const int64_t* slot;         /* [n] store entry of the query's (user, item) pair, -1 = absent */
    const float* store_emb;      /* [entries][dim] */
    const float* store_logit;    /* [entries] (required when teacher_logit is set) */
    const int64_t* written_at;   /* [entries] */
    int64_t ttl_ms;              /* StoreConfig.ttl_ms (> 0) */
    int64_t now;                 /* query clock */
    double clip;                 /* > 0: clip the teacher block to [-clip, clip]; 0: off */
    double smoothing;            /* in [0, 1): StoreConfig.label_smoothing; < 0: off */
    int32_t out_dtype;           /* lattice_dtype of out */
    void* out;                   /* [n][base_dim + dim] */
    float* teacher_logit;        /* optional [n]: (smoothed) logit on a hit, NaN on a miss */
    uint8_t* hit;                /* optional [n] */
} lattice_student_args;

lattice_status lattice_student_inputs(const lattice_student_args* args, lattice_stream stream);

/* Element/row ops of numerics.hpp in fp64, DEVICE arrays: clip_features (:139, bit-exact),
 * smooth_labels (:147, bit-exact; a label other than 0/1 -> USAGE with check = 1),
 * swish_rn_jvp (:113-136) per row of a [rows][width] matrix (non-finite -> DATA). */
lattice_status lattice_clip_features(int64_t n, const double* x, double c, double* out,
                                     lattice_stream stream);
lattice_status lattice_smooth_labels(int64_t n, const double* y, double eps_s, double* out,
                                     int32_t check, lattice_stream stream);
lattice_status lattice_swish_rn_jvp(int64_t rows, int64_t width, double eps, const double* x,
                                    const double* tangent, double* out, int32_t check,
                                    lattice_stream stream);

/* ======================================================================================
 * JSON-lines impression ingest -- replaces parse_jsonl_records +
 * record_from_json (serde.hpp:129-166; format SPEC.md:283) for a whole file: content is the
 * file's bytes in DEVICE memory (kept alive until lattice_jsonl_close). lattice_jsonl_open splits
 * lines (getline semantics, blank lines skipped), validates every line as nlohmann::json::parse
 * does, runs record_from_json's checks and sizes the columns (synchronises the stream). The
 * first bad line (lowest number) -> DATA with "<source>:<line>: <json exception text>", as the
 * reference's line loop throws (info->error_line / error_kind set; record-level texts are
 * nlohmann's exactly, parse errors keep its code and column but not its wording). lattice_jsonl_extract writes the columns
 * into caller buffers sized from info (any group may be null):
 *   domain / user / ad   unescaped UTF-8 bytes + offsets [records + 1] (user / ad feed
 *                        lattice_zipper_assign_labels directly)
 *   ts                   impression_time_ms [records] (get<int64_t>), line [records] (1-based)
 *   features             per-record entry offsets [records + 1]; per entry key bytes + key
 *                        offsets [entries + 1] and value (get<double>)
 *   conversions          the same with int64 values (get<TimestampMs>)
 * Entries follow nlohmann items(): object members (a repeated key keeps its last value), array
 * elements keyed "0", "1", ..., a primitive as one entry with the empty key, null as none.
 * The handle's workspaces are stream-ordered on the open call's stream: extract on that stream
 * (or after it), close frees them on it.
 * lattice_jsonl_task_columns maps conversion entries onto the zip tasks: conv[r][t] / present
 * (the Zipper's label inputs, zip_dataset datasets.hpp:219-244).
 * ==================================================================================== */
typedef struct lattice_jsonl lattice_jsonl;
typedef struct {
    int64_t lines, records;
    int64_t domain_bytes, user_bytes, ad_bytes;
    int64_t feature_entries, feature_key_bytes;
    int64_t conversion_entries, conversion_key_bytes;
    int64_t error_line;  /* 0, or the 1-based line of the error */
    int64_t error_kind;  /* 1: DataError ("<source>:<line>: ..."); 2: a number literal overflowing
                            double -- nlohmann's out_of_range.406, which the reference lets escape
                            as a plain json::exception (message without context) */
} lattice_jsonl_info;
typedef struct {
    uint8_t* domain;  int64_t* domain_off;
    uint8_t* user;    int64_t* user_off;
    uint8_t* ad;      int64_t* ad_off;
    int64_t* ts;      int64_t* line;
    int64_t* feature_off;    uint8_t* feature_key;    int64_t* feature_key_off;    double* feature_val;
    int64_t* conversion_off; uint8_t* conversion_key; int64_t* conversion_key_off; int64_t* conversion_val;
} lattice_jsonl_columns;

lattice_status lattice_jsonl_open(const uint8_t* content, int64_t bytes, const char* source,
                                  lattice_jsonl** out, lattice_jsonl_info* info, lattice_stream stream);
lattice_status lattice_jsonl_extract(lattice_jsonl* h, const lattice_jsonl_columns* columns,
                                     lattice_stream stream);
lattice_status lattice_jsonl_task_columns(int64_t records, const int64_t* conversion_off,
                                          const uint8_t* conversion_key, const int64_t* conversion_key_off,
                                          const int64_t* conversion_val, int32_t tasks,
                                          const uint8_t* task_bytes, const int64_t* task_off,
                                          int64_t* conv, uint8_t* present, lattice_stream stream);
void lattice_jsonl_close(lattice_jsonl* h);

/* ======================================================================================
 * Post-tower batch reductions. fp64, deterministic (fixed-order
 * per-block partials, no float atomics).
 * lattice_correlation_loss -- replaces lattice::correlation_loss (numerics.hpp:46-78) for
 *   `cols` column pairs at once: out[c] = clamp(1 - Cov(x_c, y_c) / (sx*sy + eps), 0, 2),
 *   population moments, two passes, 1.0 when either side is constant. x/y DEVICE fp64
 *   [n][ld]; out DEVICE [cols]. eps <= 0 / n < 2 -> USAGE; non-finite -> DATA (check = 1).
 * lattice_window_summary -- replaces lattice::window_routing_summary (datasets.hpp:256-283):
 *   counts[w] = records routed to window w, positives[w][t] = their own-window positives
 *   (positive_rate = positives / count, 0 when count = 0, computed by the caller). window [n],
 *   labels [n][T][W] as written by lattice_zipper_assign_labels; a window >= W -> USAGE
 *   (check = 1). counts / positives DEVICE int64.
 * lattice_routed_objectives -- the fused batch step after the towers: routed[b][t] =
 *   logits[b][t*W + window[b]] (optional), corr[t] = correlation_loss(routed label,
 *   stable_sigmoid(routed logit)) over the batch (ground-truth vs predicted
 *   label distribution), and the window summary.
 * ==================================================================================== */
lattice_status lattice_correlation_loss(int64_t n, int32_t cols, const double* x, int64_t ldx,
                                        const double* y, int64_t ldy, double eps, double* out,
                                        int32_t check, lattice_stream stream);
lattice_status lattice_window_summary(int64_t n, int32_t tasks, int32_t windows,
                                      const uint8_t* window, const uint8_t* labels, int64_t* counts,
                                      int64_t* positives, int32_t check, lattice_stream stream);

typedef struct {
    int64_t n;
    int32_t tasks, windows;
    const float* logits;     /* [n][tasks*windows] (tower output, caller order) */
    const uint8_t* window;   /* [n] assigned window */
    const uint8_t* labels;   /* [n][tasks][windows] */
    double eps;
    float* routed;           /* optional out [n][tasks] */
    double* corr;            /* out [tasks] */
    int64_t* counts;         /* out [windows] */
    int64_t* positives;      /* out [windows][tasks] */
    int32_t check;           /* 1: synchronise; bad window -> USAGE, non-finite -> DATA */
} lattice_objective_args;

lattice_status lattice_routed_objectives(const lattice_objective_args* args, lattice_stream stream);

/* ======================================================================================
 * Synthetic inputs: counter-based, identical to oracle/ so inputs
 * never cross PCIe.
 * ==================================================================================== */
lattice_status lattice_fill_tables(void* tables, int32_t dtype, int32_t features, int64_t rows,
                                   int32_t dim, uint64_t seed, int32_t feature_base,
                                   int64_t rows_total, lattice_stream stream);
lattice_status lattice_fill_weights(void* w, int32_t dtype, int64_t out_features,
                                    int64_t fan_in, uint64_t seed, uint64_t tag,
                                    lattice_stream stream);
/* lengths L = H(seed,LEN,f*B+b) mod (max_len+1); ids = H(seed,ID,(f*B+b)*max_len+j) mod rows.
 * offsets [F*B+1] are written; ids must hold F*B*max_len entries (upper bound). */
lattice_status lattice_synth_bags(int32_t features, int64_t batch, int32_t max_len, int64_t rows,
                                  uint64_t seed, int64_t* offsets, int32_t* ids,
                                  lattice_stream stream);
/* Impression log columns for the Zipper: user i = "u%08d" of H mod 1e8
 * (9 bytes), ad i = "a%06d" of H mod 1e6 (7 bytes), ts = 1.7e12 + 37 i, task t converts with
 * probability 0.3 after a delay H mod 8 days. user_bytes [9n], ad_bytes [7n], offsets [n+1],
 * ts [n], conv/present [n][tasks]. */
lattice_status lattice_synth_impressions(int64_t n, int32_t tasks, uint64_t seed, uint8_t* user_bytes,
                                         int64_t* user_off, uint8_t* ad_bytes, int64_t* ad_off,
                                         int64_t* ts, int64_t* conv, uint8_t* present,
                                         lattice_stream stream);
/* Per-sample attribution-window routing of the heads:
 * out[b][t] = logits[b][t*windows + window[b]]. */
lattice_status lattice_route_heads(int64_t batch, int32_t tasks, int32_t windows, const float* logits,
                                   const uint8_t* window, float* out, lattice_stream stream);
lattice_status lattice_synth_domains(int64_t batch, int32_t domains, uint64_t seed,
                                     int32_t* domain, lattice_stream stream);

/* ======================================================================================
 * Domain bucketing (K6): stable counting sort of samples by domain. pos[b] = row of
 * sample b in domain-sorted order; order[p] = b; seg[g] = first row of domain g (G+1).
 * ==================================================================================== */
lattice_status lattice_domain_bucket(int64_t batch, int32_t domains, const int32_t* domain,
                                     int32_t* pos, int32_t* order, int32_t* seg,
                                     lattice_stream stream);

/* ======================================================================================
 * Dense GEMM on tcgen05 (K3): C[M][N] = A[M][K] . B[N][K]^T, bf16 in, fp32 accumulate in
 * TMEM, fused epilogue. Exposed for tests and for callers composing their own blocks.
 * epilogue: 0 store (out_dtype), 1 swish_rn over each full row, 2 swish_rn_hard,
 *           3 residual + rms_norm over groups of `group` columns.
 * ==================================================================================== */
typedef struct {
    int64_t M, N, K;
    const void* A;      /* bf16 [M][lda] */
    int64_t lda;
    const void* B;      /* bf16 [N][ldb] */
    int64_t ldb;
    void* C;            /* out_dtype [M][ldc] */
    int64_t ldc;
    int32_t out_dtype;
    int32_t epilogue;
    const void* resid;  /* bf16 [M][ldr] for epilogue 3 */
    int64_t ldr;
    int32_t group;      /* epilogue 3 group width (128 or 64) */
    int32_t in_dtype;   /* A/B dtype: LATTICE_BF16 (kind::f16) or LATTICE_F32 (kind::tf32);
                           resid has the output dtype */
    int32_t a_major;    /* 0: A is [M][lda] (K-major); 1: A is stored [K][lda] with M contiguous
                           (MN-major, bf16: a transposed operand read in place, e.g. dZ^T) */
    int32_t b_major;    /* 0: B is [N][ldb]; 1: B is stored [K][ldb] with N contiguous */
} lattice_gemm_args;

lattice_status lattice_gemm(const lattice_gemm_args* args, lattice_stream stream);
/* Synchronises `stream`, then reports (LATTICE_CUDA) and clears any failed row-statistics exchange
 * of the swish_rn GEMMs since the last check. Those GEMMs run a persistent grid whose CTA pairs
 * exchange per-row sums of squares through global memory; the launch is cooperative, so the
 * hardware keeps every pair resident, and a wait that still exceeds 5 s gives up (invalid
 * outputs, counted here) instead of hanging the GPU. A checked lattice_net_forward calls it. */
lattice_status lattice_device_check(lattice_stream stream);

/* ======================================================================================
 * K2 on its own: the interaction half of one DWFB block (DESIGN.md section 3
 * step 3), per sample b with X_b [n][d]:
 *   P = q(X_b^T . Y)  (d x k),  F = X_b . P  (n x k),  Fin[b] = q(rms_norm(flatten F))  (n*k)
 *   Xout[b][nF+i] = q(rms_norm_d((W_L . X_b)_i + X_b[nF+i])), i < nL  (LCB half of X')
 * q() = round to the storage dtype. Rows [0, nF) of Xout are not written (the FMB MLP's
 * residual-norm epilogue fills them). The network runs the same kernel in every block; this
 * entry exists for kernel-level tests and callers composing their own blocks.
 * ==================================================================================== */
typedef struct {
    int64_t batch;
    int32_t n, d, k, nF, nL;   /* n <= 512 (n > 256: bf16, d = 128, k <= 48), k <= 64, nF + nL == n */
    int32_t dtype;             /* LATTICE_BF16, or LATTICE_F32 (kind::tf32; d = 64, n <= 64) */
    const void* X;             /* DEVICE [B][n][d] */
    const void* YT;            /* DEVICE [k][n]  (Y transposed) */
    const void* WL;            /* DEVICE [nL][n] */
    void* Fin;                 /* DEVICE out [B][n*k] */
    void* Xout;                /* DEVICE out [B][n][d], rows [nF, n) */
} lattice_fm_lcb_args;

lattice_status lattice_fm_lcb(const lattice_fm_lcb_args* args, lattice_stream stream);

/* ======================================================================================
 * Network (K1 -> K2/K3 blocks -> K4 towers). No reference code; the
 * arithmetic is DESIGN.md section 3 and oracle/lattice_oracle.c lo_net_forward.
 * ==================================================================================== */
typedef struct {
    int32_t n;             /* embeddings per sample (= sparse features) */
    int32_t d;             /* embedding dim */
    int32_t blocks;
    int32_t nF, nL, k;     /* nF + nL == n */
    int32_t n_mlp;         /* FMB MLP weight matrices */
    int32_t mlp[6];        /* widths: mlp[0] = n*k ... mlp[n_mlp] = nF*d */
    int32_t domains;       /* G */
    int32_t heads;         /* objectives * windows */
    int32_t tower_hidden;
    int32_t hard;          /* 1: swish_rn_hard */
    int64_t max_batch;
    uint64_t weight_seed;
    int32_t dtype;         /* storage/compute dtype: LATTICE_BF16 (kind::f16 tensor cores) or
                              LATTICE_F32 (kind::tf32; d = 64 only) */
    /* dense-feature processor: the last `dense_features` of the n embeddings are
       O_d = reshape(D2 . swish_rn(D1 . x_dense), [dense_features][d]) (D1 [dense_hidden]
       [dense_in], D2 [dense_features*d][dense_hidden]); the first n - dense_features come from
       the embedding tables. The mixing norm (rms_norm_d) applies to both. 0 = no dense part. */
    int32_t dense_features;
    int32_t dense_in;      /* multiple of 8 (pad the merged dense matrix) */
    int32_t dense_hidden;  /* multiple of 8 in [8, 2048] */
} lattice_net_config;

typedef struct lattice_net lattice_net;

lattice_status lattice_net_create(const lattice_net_config* cfg, lattice_net** out);
void lattice_net_destroy(lattice_net* net);
/* Device pointer of a weight tensor (bf16): kind 1 Y^T [k][n], 2 W_L [nL][n],
 * 3 MLP layer `index` [out][in], 4 tower W1 [G][tower_hidden][n*d], 5 tower W2 fp32
 * [G][heads][tower_hidden], 6 dense D1 [dense_hidden][dense_in], 7 dense D2
 * [dense_features*d][dense_hidden]. block ignored for 4-7. */
const void* lattice_net_weight(lattice_net* net, int32_t block, int32_t kind, int32_t index);
/* Load caller-owned weights (a trained model) into one of the tensors above, replacing the
 * generated values. src: DEVICE, unpadded, row-major in the layout listed for `kind` (kind 4/5:
 * all G domains stacked), in src_dtype: LATTICE_F32 (rounded to the net dtype with RNE; kind 5 is
 * kept fp32) or the net dtype itself (copied bit for bit). The net's zero padding is kept. Ordered
 * on `stream`; the forward passes queued after it on that stream see the new values. Non-finite
 * values are not checked. */
lattice_status lattice_net_set_weight(lattice_net* net, int32_t block, int32_t kind, int32_t index,
                                      const void* src, int32_t src_dtype, lattice_stream stream);

typedef struct {
    int64_t batch;
    const int32_t* domain;       /* DEVICE [B] */
    /* sparse input, as lattice_bag_args (features = cfg.n) */
    int32_t table_dtype;
    const void* const* tables;
    const int64_t* rows;
    const int64_t* offsets;
    const int32_t* ids;
    /* or, when tables == NULL: already pooled embeddings in table_dtype */
    const void* pooled;
    int32_t pooled_layout;       /* 0: raw sums [B][n - dense_features][d], caller order (the
                                       net normalises)
                                    1: table-wise shards [S][B][n/S][d] bf16, already
                                       rms-normalised by the owners (lattice_embedding_bag
                                       with normalize = 1), S = shards
                                    2: in place -- X0 (lattice_net_buffer 0) was already
                                       written in domain-sorted order by
                                       lattice_peer_embedding_bag after lattice_net_bucket
                                       ran for this batch; `pooled` is ignored */
    int32_t shards;
    const void* dense;           /* DEVICE [B][dense_in] in the net dtype (caller order) when
                                    cfg.dense_features > 0 (e.g. lattice_merge_dense output) */
    int32_t check;               /* 1: synchronise after the bucketing / embedding stage and
                                    return DATA naming the first sample whose domain is outside
                                    [0, domains) or (tables != NULL) the first id outside its table
                                    (its position in ids, as lattice_embedding_bag); 0 (graphs,
                                    pipelines): bad domains count as domain 0 and bad ids pool as
                                    zero rows, unreported */
} lattice_batch;

/* Domain bucketing of a batch ahead of the forward (pooled_layout 2): writes the
 * domain-sorted row of every sample, readable through lattice_net_buffer(net, 1). */
lattice_status lattice_net_bucket(lattice_net* net, int64_t batch, const int32_t* domain,
                                  lattice_stream stream);
/* Workspace pointers: 0 = X0 [max_batch][n][d] (net dtype, the embedding stage's output; peer
 * export), 1 = sample_pos int32 [max_batch] (row of sample b in the domain-sorted activations),
 * 2 = the second activation buffer. Blocks ping-pong: block l reads buffer (l & 1 ? 2 : 0) and
 * writes the other, so after a forward buffer (blocks & 1 ? 2 : 0) holds the last block's output
 * X_L (the towers' input) and the other X_{L-1} (inspection / stage-wise tests); 3 = Fin
 * [max_batch][n*k] (net dtype, domain-sorted rows): the last block's MLP input. NULL for an
 * unknown index. */
void* lattice_net_buffer(lattice_net* net, int32_t which);

/* logits: DEVICE fp32 [B][heads] in the caller's sample order. */
lattice_status lattice_net_forward(lattice_net* net, const lattice_batch* batch, float* logits,
                                   lattice_stream stream);
/* ======================================================================================
 * Backward. The reference defines no training step; it pins the activation
 * derivative (swish_rn_jvp, numerics.hpp:113-136, test_numerics.cpp:151-178), whose adjoint these
 * entries compute.
 * lattice_rownorm_vjp: out = J(x)^T g per row of a [rows][width] matrix, J the Jacobian of
 *   rms_norm (mode 0), swish_rn (1) or swish_rn_hard (2) (numerics.hpp:81-107); dtype F32 / F64.
 * lattice_routed_bce: window-routed binary cross-entropy of the heads, each sample training only
 *   its assigned window's head per task: loss = mean over (sample, task) of
 *   bce(logits[b][t*W + window[b]], labels[b][t][window[b]]) (DEVICE fp64 scalar), and
 *   dlogits [n][T*W] (zero for the other windows' heads). Deterministic.
 * lattice_net_tower_backward: after a forward of `batch` samples, the gradients of the untied
 *   towers from dlogits [batch][heads] (caller order): dW1 fp32 [G][tower_hidden][n*d], dW2 fp32
 *   [G][heads][tower_hidden], optionally dX [batch][n*d] (the towers' input, domain-sorted rows:
 *   lattice_net_buffer 1 maps samples to rows) in dx_dtype. tcgen05 GEMMs (operands read in place,
 *   MN-major), fixed-order reductions: deterministic. Synchronises the stream once (segment sizes).
 * ==================================================================================== */
lattice_status lattice_rownorm_vjp(int32_t mode, int64_t rows, int64_t width, double eps, int32_t dtype,
                                   const void* x, const void* g, void* out, lattice_stream stream);
lattice_status lattice_routed_bce(int64_t n, int32_t tasks, int32_t windows, const float* logits,
                                  const uint8_t* window, const uint8_t* labels, float* dlogits, double* loss,
                                  lattice_stream stream);
lattice_status lattice_net_tower_backward(lattice_net* net, int64_t batch, const float* dlogits, float* dW1,
                                          float* dW2, void* dX, int32_t dx_dtype, lattice_stream stream);
/* Plain SGD on the towers: master -= lr * grad for the caller's fp32 master copies of W1 [G][th][n*d]
 * and W2 [G][heads][th] (start them from lattice_net_weight), and the network's own copies refreshed
 * (W1 rounded to the network dtype) in the same pass. With data parallelism, all-reduce (average) the
 * gradients first: every replica then applies the same update and stays bit-identical. */
lattice_status lattice_net_tower_sgd(lattice_net* net, float lr, const float* dW1, const float* dW2, float* master_W1,
                                     float* master_W2, lattice_stream stream);
/* Backward through the LAST DWFB block's FMB half (its MLP and the residual
 * rms_norm_d), after a forward of `batch` samples: from dXout fp32 [batch][n*d] (d loss / d X_L,
 * domain-sorted rows, e.g. lattice_net_tower_backward's dX; columns [0, nF*d) are used) ->
 * dW[i] fp32 [mlp[i+1]][mlp[i]] for every MLP layer i < n_mlp; optionally dFin fp32
 * [batch][n*k] (the MLP input; buffer 3 holds the forward's Fin) and dResid fp32 [batch][nF*d]
 * (the residual branch's gradient to the block input rows [0, nF)). The MLP's hidden outputs are
 * the forward's own (re-run bit-identically for n_mlp > 3); pre-activations are recomputed by
 * fp32 GEMMs; gradients of z are rounded to bf16 as the tcgen05 GEMMs' operands. bf16 networks;
 * deterministic. The FM / LCB interaction (P, W_L, Y) and earlier blocks are not differentiated. */
lattice_status lattice_net_mlp_backward(lattice_net* net, int64_t batch, const float* dXout, float* const* dW,
                                        float* dFin, float* dResid, lattice_stream stream);
/* Plain SGD on one unpadded weight (kind 3..7, block / index as lattice_net_weight): fp32 master
 * -= lr * grad, the network's copy refreshed in its dtype (kind 5: fp32). */
lattice_status lattice_net_weight_sgd(lattice_net* net, int32_t block, int32_t kind, int32_t index, float lr,
                                      const float* grad, float* master, lattice_stream stream);

/* Per-stage CUDA-event times (ms) of the last forward when timing was enabled. */
lattice_status lattice_net_set_timing(lattice_net* net, int32_t enable);
lattice_status lattice_net_stage_times(lattice_net* net, float* ms, int32_t max_stages,
                                       int32_t* n_stages);

#ifdef __cplusplus
}
#endif
#endif
