/*
 * lattice_oracle.c -- CPU restatement of the Lattice hot path. TEST INFRASTRUCTURE ONLY.
 * See lattice_oracle.h for the parity status of each part. Only tests/, smoke() and
 * bench.py's CPU-baseline leg load this; the product is the CUDA library.
 */
#include "lattice_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------------------------------------------------------------------------------------
 * XXH64, restated from proj/include/lattice/core.hpp:84-139 (the published XXH64 algorithm).
 * ------------------------------------------------------------------------------------- */
#define P1 0x9E3779B185EBCA87ull
#define P2 0xC2B2AE3D27D4EB4Full
#define P3 0x165667B19E3779F9ull
#define P4 0x85EBCA77C2B2AE63ull
#define P5 0x27D4EB2F165667C5ull

static inline uint64_t rotl(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }

static inline uint64_t le64(const uint8_t* p) {
    uint64_t v = 0;
    for (int i = 7; i >= 0; --i) v = (v << 8) | p[i];
    return v;
}

static inline uint32_t le32(const uint8_t* p) {
    return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

static inline uint64_t round64(uint64_t acc, uint64_t lane) {
    return rotl(acc + lane * P2, 31) * P1;
}

uint64_t lo_xxh64(const uint8_t* p, size_t len, uint64_t seed) {
    const uint8_t* end = p + len;
    uint64_t h;
    if (len >= 32) { /* core.hpp:96-111 */
        uint64_t v[4] = {seed + P1 + P2, seed + P2, seed, seed - P1};
        do {
            for (int i = 0; i < 4; ++i, p += 8) v[i] = round64(v[i], le64(p));
        } while (p + 32 <= end);
        h = rotl(v[0], 1) + rotl(v[1], 7) + rotl(v[2], 12) + rotl(v[3], 18);
        for (int i = 0; i < 4; ++i) {
            h ^= round64(0, v[i]);
            h = h * P1 + P4;
        }
    } else { /* core.hpp:113 */
        h = seed + P5;
    }
    h += (uint64_t)len; /* core.hpp:116 */
    for (; p + 8 <= end; p += 8) {
        h ^= round64(0, le64(p));
        h = rotl(h, 27) * P1 + P4;
    }
    if (p + 4 <= end) {
        h ^= (uint64_t)le32(p) * P1;
        h = rotl(h, 23) * P2 + P3;
        p += 4;
    }
    for (; p < end; ++p) {
        h ^= (uint64_t)(*p) * P5;
        h = rotl(h, 11) * P1;
    }
    h ^= h >> 33; /* avalanche, core.hpp:133-138 */
    h *= P2;
    h ^= h >> 29;
    h *= P3;
    h ^= h >> 32;
    return h;
}

uint64_t lo_gen(uint64_t seed, uint64_t tag, uint64_t idx) {
    uint8_t buf[16];
    for (int i = 0; i < 8; ++i) {
        buf[i] = (uint8_t)(tag >> (8 * i));
        buf[8 + i] = (uint8_t)(idx >> (8 * i));
    }
    return lo_xxh64(buf, 16, seed);
}

/* ---------------------------------------------------------------------------------------
 * Zipper: signature bytes (core.hpp:149-175 via datasets.hpp:181-184), window assignment
 * (datasets.hpp:185-193) and labels (datasets.hpp:229-243).
 * ------------------------------------------------------------------------------------- */
static void put_be(uint8_t* out, uint64_t v, int bytes) {
    for (int i = 0; i < bytes; ++i) out[i] = (uint8_t)(v >> (8 * (bytes - 1 - i)));
}

size_t lo_signature(const uint8_t* user, uint32_t ulen, const uint8_t* ad, uint32_t alen,
                    int64_t ts, uint8_t* out) {
    size_t o = 0;
    put_be(out + o, ulen, 4);
    o += 4;
    if (ulen) memcpy(out + o, user, ulen);
    o += ulen;
    put_be(out + o, alen, 4);
    o += 4;
    if (alen) memcpy(out + o, ad, alen);
    o += alen;
    put_be(out + o, (uint64_t)ts, 8);
    return o + 8;
}

static int bucket(uint64_t h, const double* probs, int windows) {
    const double u = (double)(h >> 11) * 0x1.0p-53; /* datasets.hpp:186 */
    double cum = 0.0;
    for (int i = 0; i + 1 < windows; ++i) { /* datasets.hpp:188-192 */
        cum += probs[i];
        if (u < cum) return i;
    }
    return windows - 1;
}

int lo_assign_window(const uint8_t* user, uint32_t ulen, const uint8_t* ad, uint32_t alen,
                     int64_t ts, uint64_t seed, const double* probs, int windows) {
    uint8_t small[256];
    const size_t need = 16 + (size_t)ulen + alen;
    uint8_t* buf = need <= sizeof(small) ? small : (uint8_t*)malloc(need);
    const size_t len = lo_signature(user, ulen, ad, alen, ts, buf);
    const uint64_t h = lo_xxh64(buf, len, seed);
    if (buf != small) free(buf);
    return bucket(h, probs, windows);
}

int64_t lo_zip_columns(int64_t n, const uint8_t* user_bytes, const int64_t* user_off,
                       const uint8_t* ad_bytes, const int64_t* ad_off, const int64_t* ts,
                       int T, const int64_t* conv, const uint8_t* conv_present, int W,
                       const int64_t* durations, const double* probs, uint64_t seed,
                       uint8_t* window, uint8_t* labels, int32_t* err_task) {
    for (int64_t i = 0; i < n; ++i) {
        window[i] = (uint8_t)lo_assign_window(
            user_bytes + user_off[i], (uint32_t)(user_off[i + 1] - user_off[i]),
            ad_bytes + ad_off[i], (uint32_t)(ad_off[i + 1] - ad_off[i]), ts[i], seed, probs, W);
        for (int t = 0; t < T; ++t) {
            uint8_t* lab = labels + ((size_t)i * T + t) * W;
            memset(lab, 0, (size_t)W);
            if (!conv_present[(size_t)i * T + t]) continue;
            /* two's-complement difference, as the reference computes it on int64 */
            const int64_t delay = (int64_t)((uint64_t)conv[(size_t)i * T + t] - (uint64_t)ts[i]);
            if (delay < 0) {
                if (err_task) *err_task = t;
                return i;
            }
            for (int w = 0; w < W; ++w) lab[w] = (uint8_t)(delay <= durations[w]);
        }
    }
    return -1;
}

/* ---------------------------------------------------------------------------------------
 * numerics.hpp:16-41, 81-107
 * ------------------------------------------------------------------------------------- */
static double stable_sigmoid(double z) { /* numerics.hpp:29-33 */
    if (z >= 0.0) return 1.0 / (1.0 + exp(-z));
    const double e = exp(z);
    return e / (1.0 + e);
}

int lo_rms_norm(const double* x, size_t n, double eps, double* out) {
    if (!(eps > 0.0) || n == 0) return 1;
    double acc = 0.0;
    for (size_t i = 0; i < n; ++i) {
        if (!isfinite(x[i])) return 2;
        acc += x[i] * x[i];
    }
    const double denom = sqrt(acc / (double)n + eps);
    for (size_t i = 0; i < n; ++i) out[i] = x[i] / denom;
    return 0;
}

int lo_swish_rn(const double* x, size_t n, double eps, double* out) {
    const int rc = lo_rms_norm(x, n, eps, out);
    if (rc) return rc;
    for (size_t i = 0; i < n; ++i) out[i] *= stable_sigmoid(out[i]);
    return 0;
}

int lo_swish_rn_hard(const double* x, size_t n, double eps, double* out) {
    const int rc = lo_rms_norm(x, n, eps, out);
    if (rc) return rc;
    for (size_t i = 0; i < n; ++i) {
        double g = (out[i] + 3.0) / 6.0;
        g = g < 0.0 ? 0.0 : (g > 1.0 ? 1.0 : g);
        out[i] *= g;
    }
    return 0;
}

/* ---------------------------------------------------------------------------------------
 * Post-tower reductions: correlation_loss (numerics.hpp:46-78), window_routing_summary
 * (datasets.hpp:262-283) and the routed-objective batch step built from them.
 * ------------------------------------------------------------------------------------- */
int lo_correlation_loss(const double* x, const double* y, size_t n, double eps, double* out) {
    if (!(eps > 0.0)) return 1;
    if (n < 2) return 1;
    for (size_t i = 0; i < n; ++i)
        if (!isfinite(x[i]) || !isfinite(y[i])) return 2;
    const double dn = (double)n;
    double mx = 0.0, my = 0.0;
    for (size_t i = 0; i < n; ++i) {
        mx += x[i];
        my += y[i];
    }
    mx /= dn;
    my /= dn;
    double cov = 0.0, vx = 0.0, vy = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const double dx = x[i] - mx, dy = y[i] - my;
        cov += dx * dy;
        vx += dx * dx;
        vy += dy * dy;
    }
    cov /= dn;
    const double sx = sqrt(vx / dn), sy = sqrt(vy / dn);
    if (sx == 0.0 || sy == 0.0) {
        *out = 1.0;
        return 0;
    }
    double loss = 1.0 - cov / (sx * sy + eps);
    *out = loss < 0.0 ? 0.0 : (loss > 2.0 ? 2.0 : loss);
    return 0;
}

int lo_window_summary(int64_t n, int T, int W, const uint8_t* window, const uint8_t* labels,
                      int64_t* counts, int64_t* positives) {
    for (int w = 0; w < W; ++w) {
        counts[w] = 0;
        for (int t = 0; t < T; ++t) positives[(int64_t)w * T + t] = 0;
    }
    for (int64_t i = 0; i < n; ++i) {
        const int w = window[i];
        if (w >= W) return 1;
        ++counts[w];
        for (int t = 0; t < T; ++t) positives[(int64_t)w * T + t] += labels[(i * T + t) * W + w];
    }
    return 0;
}

int lo_routed_objectives(int64_t n, int T, int W, const float* logits, const uint8_t* window,
                         const uint8_t* labels, double eps, float* routed, double* corr,
                         int64_t* counts, int64_t* positives) {
    const int rc = lo_window_summary(n, T, W, window, labels, counts, positives);
    if (rc) return rc;
    double* y = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double* p = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    int status = 0;
    for (int t = 0; t < T && !status; ++t) {
        for (int64_t i = 0; i < n; ++i) {
            const int w = window[i];
            const float z = logits[i * (int64_t)T * W + (int64_t)t * W + w];
            if (routed) routed[i * T + t] = z;
            y[i] = (double)labels[(i * T + t) * W + w];
            p[i] = stable_sigmoid((double)z);
        }
        status = lo_correlation_loss(y, p, (size_t)n, eps, &corr[t]);
    }
    free(y);
    free(p);
    return status;
}

/* ---------------------------------------------------------------------------------------
 * Synthetic values
 * ------------------------------------------------------------------------------------- */
float lo_table_value(uint64_t seed, int64_t f, int64_t r, int D, int64_t rows, int64_t c) {
    const uint64_t idx = ((uint64_t)f * (uint64_t)rows + (uint64_t)r) * (uint64_t)D + (uint64_t)c;
    const int8_t q = (int8_t)(lo_gen(seed, LO_TAG_TABLE, idx) >> 56);
    return (float)q * 0x1.0p-10f;
}

int lo_weight_shift(int64_t fan_in) {
    int lg = 0;
    while ((1ll << (lg + 1)) <= fan_in) ++lg; /* floor(log2(fan_in)) */
    return 7 + lg / 2;
}

float lo_weight_value(uint64_t seed, uint64_t tag, int64_t o, int64_t i, int64_t fan_in) {
    const int8_t q = (int8_t)(lo_gen(seed, tag, (uint64_t)o * (uint64_t)fan_in + (uint64_t)i) >> 56);
    return ldexpf((float)q, -lo_weight_shift(fan_in));
}

uint64_t lo_weight_tag(int block, int kind, int index) {
    return 0x57000000ull | ((uint64_t)block << 16) | ((uint64_t)kind << 8) | (uint64_t)index;
}

float lo_bf16_round(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    if ((u & 0x7f800000u) == 0x7f800000u) { /* inf / nan: keep */
        u &= 0xffff0000u;
    } else {
        u += 0x7fffu + ((u >> 16) & 1u);
        u &= 0xffff0000u;
    }
    float r;
    memcpy(&r, &u, 4);
    return r;
}

/* ---------------------------------------------------------------------------------------
 * Embedding bag (sum pooling)
 * ------------------------------------------------------------------------------------- */
int64_t lo_embedding_bag_synth(uint64_t seed, int F, int64_t rows, int D, int64_t B,
                               const int64_t* offsets, const int32_t* ids, int64_t b_lo,
                               int64_t b_hi, float* out, int threads) {
    int64_t first_bad = -1;
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel for schedule(dynamic, 4)
#endif
    for (int64_t b = b_lo; b < b_hi; ++b) {
        for (int f = 0; f < F; ++f) {
            float* o = out + ((size_t)(b - b_lo) * F + f) * D;
            for (int c = 0; c < D; ++c) o[c] = 0.0f;
            const int64_t s = offsets[(size_t)f * B + b], e = offsets[(size_t)f * B + b + 1];
            for (int64_t j = s; j < e; ++j) {
                const int64_t r = ids[j];
                if (r < 0 || r >= rows) {
#ifdef _OPENMP
#pragma omp critical
#endif
                    {
                        if (first_bad < 0 || j < first_bad) first_bad = j;
                    }
                    continue;
                }
                for (int c = 0; c < D; ++c) o[c] += lo_table_value(seed, f, r, D, rows, c);
            }
        }
    }
    return first_bad;
}

int64_t lo_embedding_bag(int F, const int64_t* rows, int D, int64_t B,
                         const float* const* tables, const int64_t* offsets,
                         const int32_t* ids, float* out) {
    int64_t first_bad = -1;
    for (int64_t b = 0; b < B; ++b) {
        for (int f = 0; f < F; ++f) {
            float* o = out + ((size_t)b * F + f) * D;
            for (int c = 0; c < D; ++c) o[c] = 0.0f;
            const int64_t s = offsets[(size_t)f * B + b], e = offsets[(size_t)f * B + b + 1];
            for (int64_t j = s; j < e; ++j) {
                const int64_t r = ids[j];
                if (r < 0 || r >= rows[f]) {
                    if (first_bad < 0 || j < first_bad) first_bad = j;
                    continue;
                }
                const float* row = tables[f] + (size_t)r * D;
                for (int c = 0; c < D; ++c) o[c] += row[c];
            }
        }
    }
    return first_bad;
}

/* ---------------------------------------------------------------------------------------
 * Network forward, one sample at a time in fp64.
 * ------------------------------------------------------------------------------------- */
static inline double q(const lo_net_cfg* cfg, double v) {
    return cfg->bf16 ? (double)lo_bf16_round((float)v) : (double)(float)v;
}

static void act(const lo_net_cfg* cfg, const double* x, size_t n, double* out) {
    if (cfg->hard)
        lo_swish_rn_hard(x, n, 1e-6, out);
    else
        lo_swish_rn(x, n, 1e-6, out);
}

static void forward_one(const lo_net_cfg* cfg, const lo_net_weights* w, const float* pooled,
                        int dom, float* logits, double* scratch) {
    const int n = cfg->n, d = cfg->d, k = cfg->k, nF = cfg->nF, nL = cfg->nL;
    int maxw = n * d;
    for (int i = 0; i <= cfg->n_mlp; ++i)
        if (cfg->mlp[i] > maxw) maxw = cfg->mlp[i];
    if (cfg->tower_hidden > maxw) maxw = cfg->tower_hidden;
    double* X = scratch;
    double* Xn = X + (size_t)n * d;
    double* P = Xn + (size_t)n * d;
    double* Fm = P + (size_t)d * k;
    double* h = Fm + (size_t)n * k;
    double* z = h + maxw;
    double* tmp = z + maxw;

    for (int i = 0; i < n; ++i) { /* input norm over d (the mixing network's normalisation) */
        for (int c = 0; c < d; ++c) tmp[c] = pooled[(size_t)i * d + c];
        lo_rms_norm(tmp, (size_t)d, 1e-6, tmp + d);
        for (int c = 0; c < d; ++c) X[(size_t)i * d + c] = q(cfg, tmp[d + c]);
    }
    for (int blk = 0; blk < cfg->blocks; ++blk) {
        const float* YT = w->YT[blk];
        const float* WL = w->WL[blk];
        /* FMB: P = X^T Y (d x k), rounded to the operand dtype */
        for (int c = 0; c < d; ++c)
            for (int j = 0; j < k; ++j) {
                double acc = 0.0;
                for (int i = 0; i < n; ++i) acc += X[(size_t)i * d + c] * (double)YT[(size_t)j * n + i];
                P[(size_t)c * k + j] = q(cfg, acc);
            }
        /* F = X P (n x k), flattened and normalised over n*k */
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < k; ++j) {
                double acc = 0.0;
                for (int c = 0; c < d; ++c) acc += X[(size_t)i * d + c] * P[(size_t)c * k + j];
                Fm[(size_t)i * k + j] = acc;
            }
        lo_rms_norm(Fm, (size_t)n * k, 1e-6, h);
        for (int i = 0; i < n * k; ++i) h[i] = q(cfg, h[i]);
        /* bias-less MLP, SwishRN on hidden layers */
        for (int li = 0; li < cfg->n_mlp; ++li) {
            const int in = cfg->mlp[li], out = cfg->mlp[li + 1];
            const float* W = w->mlp[blk * cfg->n_mlp + li];
            for (int o = 0; o < out; ++o) {
                const float* wr = W + (size_t)o * in;
                double acc = 0.0;
                for (int i = 0; i < in; ++i) acc += (double)wr[i] * h[i];
                z[o] = acc;
            }
            if (li + 1 < cfg->n_mlp) {
                act(cfg, z, (size_t)out, h);
                for (int o = 0; o < out; ++o) h[o] = q(cfg, h[o]);
            }
        }
        /* FMB half of the block output: rms_norm_d(z_i + X_i), i < nF */
        for (int i = 0; i < nF; ++i) {
            for (int c = 0; c < d; ++c) tmp[c] = z[(size_t)i * d + c] + X[(size_t)i * d + c];
            lo_rms_norm(tmp, (size_t)d, 1e-6, tmp + d);
            for (int c = 0; c < d; ++c) Xn[(size_t)i * d + c] = q(cfg, tmp[d + c]);
        }
        /* LCB half: rms_norm_d((W_L X)_i + X_{nF+i}), i < nL */
        for (int i = 0; i < nL; ++i) {
            for (int c = 0; c < d; ++c) {
                double acc = 0.0;
                for (int m = 0; m < n; ++m) acc += (double)WL[(size_t)i * n + m] * X[(size_t)m * d + c];
                tmp[c] = acc + X[(size_t)(nF + i) * d + c];
            }
            lo_rms_norm(tmp, (size_t)d, 1e-6, tmp + d);
            for (int c = 0; c < d; ++c) Xn[(size_t)(nF + i) * d + c] = q(cfg, tmp[d + c]);
        }
        memcpy(X, Xn, sizeof(double) * (size_t)n * d);
    }
    /* untied tower of the sample's domain: heads = W2_g . swish_rn(W1_g . flatten(X)) */
    const int th = cfg->tower_hidden, nd = n * d;
    const float* T1 = w->T1 + (size_t)dom * th * nd;
    const float* T2 = w->T2 + (size_t)dom * cfg->heads * th;
    for (int o = 0; o < th; ++o) {
        double acc = 0.0;
        const float* wr = T1 + (size_t)o * nd;
        for (int i = 0; i < nd; ++i) acc += (double)wr[i] * X[i];
        z[o] = acc;
    }
    act(cfg, z, (size_t)th, h);
    for (int j = 0; j < cfg->heads; ++j) {
        double acc = 0.0;
        for (int o = 0; o < th; ++o) acc += (double)T2[(size_t)j * th + o] * h[o];
        logits[j] = (float)acc;
    }
}

void lo_net_forward(const lo_net_cfg* cfg, const lo_net_weights* w, int64_t count,
                    const float* pooled, const int32_t* dom, float* logits, int threads) {
    int maxw = cfg->n * cfg->d;
    for (int i = 0; i <= cfg->n_mlp; ++i)
        if (cfg->mlp[i] > maxw) maxw = cfg->mlp[i];
    if (cfg->tower_hidden > maxw) maxw = cfg->tower_hidden;
    const size_t per = (size_t)cfg->n * cfg->d * 2 + (size_t)cfg->d * cfg->k +
                       (size_t)cfg->n * cfg->k + 3 * (size_t)maxw + 2 * (size_t)cfg->d;
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel
#endif
    {
        double* scratch = (double*)malloc(per * sizeof(double));
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
        for (int64_t s = 0; s < count; ++s)
            forward_one(cfg, w, pooled + (size_t)s * cfg->n * cfg->d, dom[s],
                        logits + (size_t)s * cfg->heads, scratch);
        free(scratch);
    }
}

/* ---------------------------------------------------------------------------------------
 * Synthetic bags / domains, same formulas as lattice_synth_bags.
 * ------------------------------------------------------------------------------------- */
void lo_synth_bags(int F, int64_t B, int max_len, int64_t rows, uint64_t seed, int64_t* offsets,
                   int32_t* ids) {
    const int64_t bags = (int64_t)F * B;
    offsets[0] = 0;
    for (int64_t i = 0; i < bags; ++i)
        offsets[i + 1] = offsets[i] + (int64_t)(lo_gen(seed, LO_TAG_LEN, (uint64_t)i) %
                                                (uint64_t)(max_len + 1));
    for (int64_t i = 0; i < bags; ++i)
        for (int64_t j = offsets[i]; j < offsets[i + 1]; ++j)
            ids[j] = (int32_t)(lo_gen(seed, LO_TAG_ID, (uint64_t)i * max_len + (uint64_t)(j - offsets[i])) %
                               (uint64_t)rows);
}

void lo_synth_domains(int64_t B, int G, uint64_t seed, int32_t* dom) {
    for (int64_t i = 0; i < B; ++i) dom[i] = (int32_t)(lo_gen(seed, LO_TAG_DOM, (uint64_t)i) % (uint64_t)G);
}

void lo_fill_weights(float* out, int64_t out_features, int64_t fan_in, uint64_t seed, uint64_t tag) {
    const int shift = lo_weight_shift(fan_in);
    const int64_t n = out_features * fan_in;
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
    for (int64_t i = 0; i < n; ++i)
        out[i] = ldexpf((float)(int8_t)(lo_gen(seed, tag, (uint64_t)i) >> 56), -shift);
}

/* Impression columns exactly as lattice_synth_impressions (fixed-width decimal ids). */
void lo_synth_impressions(int64_t n, int T, uint64_t seed, uint8_t* ub, int64_t* uo, uint8_t* ab, int64_t* ao,
                          int64_t* ts, int64_t* conv, uint8_t* pres) {
    const uint64_t tag_user = 0x55534552ull, tag_ad = 0x41442020ull, tag_p = 0x43565020ull, tag_d = 0x43564420ull;
    for (int64_t i = 0; i < n; ++i) {
        uint64_t u = lo_gen(seed, tag_user, (uint64_t)i) % 100000000ull;
        uint64_t a = lo_gen(seed, tag_ad, (uint64_t)i) % 1000000ull;
        ub[9 * i] = 'u';
        for (int k = 8; k >= 1; --k, u /= 10) ub[9 * i + k] = (uint8_t)('0' + u % 10);
        ab[7 * i] = 'a';
        for (int k = 6; k >= 1; --k, a /= 10) ab[7 * i + k] = (uint8_t)('0' + a % 10);
        uo[i] = 9 * i;
        ao[i] = 7 * i;
        ts[i] = 1700000000000ll + 37 * i;
        for (int t = 0; t < T; ++t) {
            const uint64_t k = (uint64_t)i * T + t;
            pres[k] = (uint8_t)(lo_gen(seed, tag_p, k) % 10 < 3);
            conv[k] = ts[i] + (int64_t)(lo_gen(seed, tag_d, k) % (8ull * 86400000ull));
        }
    }
    uo[n] = 9 * n;
    ao[n] = 7 * n;
}

/* ---------------------------------------------------------------------------------------
 * Dense features: merge_domains values (datasets.hpp:144-173) and the dense processor
 * (PAPER.md:277).
 * ------------------------------------------------------------------------------------- */
int64_t lo_merge_dense(int64_t n, int G, int max_decl, const int32_t* domain, const float* values,
                       const int32_t* src_col, int width, int bf16, float* out) {
    int64_t bad = -1;
    for (int64_t b = 0; b < n; ++b) {
        const int g = domain[b];
        if (g < 0 || g >= G) {
            if (bad < 0) bad = b;
            for (int c = 0; c < width; ++c) out[b * width + c] = 0.0f;
            continue;
        }
        for (int c = 0; c < width; ++c) {
            const int j = src_col[(int64_t)g * width + c];
            const float v = j >= 0 ? values[b * max_decl + j] : 0.0f;
            out[b * width + c] = bf16 ? lo_bf16_round(v) : v;
        }
    }
    return bad;
}

void lo_dense_processor(const lo_net_cfg* cfg, int n_dense, int dense_in, int dense_hidden,
                        const float* D1, const float* D2, int64_t count, const float* dense,
                        float* pooled, int threads) {
    const int n = cfg->n, d = cfg->d, nc = cfg->n - n_dense, od = n_dense * d;
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel
#endif
    {
        double* h = (double*)malloc(sizeof(double) * (size_t)dense_hidden * 2);
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 4)
#endif
        for (int64_t s = 0; s < count; ++s) {
            const float* x = dense + (size_t)s * dense_in;
            for (int o = 0; o < dense_hidden; ++o) {
                double acc = 0.0;
                for (int i = 0; i < dense_in; ++i) acc += (double)D1[(size_t)o * dense_in + i] * (double)x[i];
                h[o] = acc;
            }
            act(cfg, h, (size_t)dense_hidden, h + dense_hidden);
            for (int o = 0; o < dense_hidden; ++o) h[o] = q(cfg, h[dense_hidden + o]);
            float* dst = pooled + ((size_t)s * n + nc) * d;
            for (int o = 0; o < od; ++o) {
                double acc = 0.0;
                for (int i = 0; i < dense_hidden; ++i) acc += (double)D2[(size_t)o * dense_hidden + i] * h[i];
                dst[o] = (float)q(cfg, acc);
            }
        }
        free(h);
    }
}

/* ---------------------------------------------------------------------------------------
 * numerics.hpp:113-156 element/row ops and the KTAP student-input read side (ktap.hpp).
 * ------------------------------------------------------------------------------------- */
int lo_swish_rn_jvp(const double* x, const double* t, size_t n, double eps, double* out) {
    if (!(eps > 0.0) || n == 0) return 1;
    for (size_t i = 0; i < n; ++i)
        if (!isfinite(x[i]) || !isfinite(t[i])) return 2;
    double ss = 0.0, dot = 0.0;
    for (size_t i = 0; i < n; ++i) ss += x[i] * x[i];
    const double dn = (double)n;
    const double d = sqrt(ss / dn + eps);
    for (size_t i = 0; i < n; ++i) dot += x[i] * t[i];
    dot /= dn;
    const double d3 = d * d * d;
    for (size_t i = 0; i < n; ++i) {
        const double r = x[i] / d;
        const double dr = t[i] / d - x[i] * dot / d3;
        const double s = stable_sigmoid(r);
        out[i] = s * (1.0 + r * (1.0 - s)) * dr;
    }
    return 0;
}

int lo_clip_features(const double* x, size_t n, double c, double* out) {
    if (!(c > 0.0)) return 1;
    for (size_t i = 0; i < n; ++i) out[i] = x[i] < -c ? -c : (x[i] > c ? c : x[i]);
    return 0;
}

int lo_smooth_labels(const double* y, size_t n, double eps_s, double* out) {
    if (!(eps_s >= 0.0 && eps_s < 1.0)) return 1;
    for (size_t i = 0; i < n; ++i) {
        if (y[i] != 0.0 && y[i] != 1.0) return 1;
        out[i] = y[i] * (1.0 - eps_s) + eps_s / 2.0;
    }
    return 0;
}

void lo_student_inputs(int64_t n, int base_dim, int dim, const float* base, const int64_t* slot,
                       const float* store_emb, const float* store_logit, const int64_t* written_at,
                       int64_t ttl, int64_t now, double clip, double smoothing, int bf16, float* out,
                       float* logit, uint8_t* hit) {
    const int W = base_dim + dim;
    for (int64_t q = 0; q < n; ++q) {
        const int64_t s = slot[q];
        const int h = s >= 0 && now - written_at[s] <= ttl;
        float* row = out + q * W;
        for (int c = 0; c < base_dim; ++c) row[c] = base[q * base_dim + c];
        for (int c = 0; c < dim; ++c) {
            double v = h ? (double)store_emb[s * dim + c] : 0.0;
            if (h && clip > 0.0) v = v < -clip ? -clip : (v > clip ? clip : v);
            row[base_dim + c] = (float)v;
        }
        if (bf16)
            for (int c = 0; c < W; ++c) row[c] = lo_bf16_round(row[c]);
        double l = h ? (double)store_logit[s] : NAN;
        if (h && smoothing >= 0.0) l = l * (1.0 - smoothing) + smoothing / 2.0;
        logit[q] = (float)l;
        hit[q] = (uint8_t)h;
    }
}
