// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY. Exposes the reference's own header-only
// functions (compiled from /root/reference/proj/include, never copied) behind a C ABI so
// the tests can pin the oracle restatement and the CUDA path against the reference itself.
// Built by oracle/Makefile into oracle/_ref/libref.so (git-ignored; travels to the GPU box).
//
// The reference headers are included under `#define lattice lattice_ref` so they cannot
// collide with anything named lattice:: elsewhere ("verified by probe").
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#define lattice lattice_ref
#include "lattice/core.hpp"
#include "lattice/datasets.hpp"
#include "lattice/ktap.hpp"
#include "lattice/numerics.hpp"
#include "lattice/serde.hpp"
#undef lattice

namespace {
thread_local std::string g_err;

int copy_out(const std::vector<double>& v, double* out) {
    std::memcpy(out, v.data(), v.size() * sizeof(double));
    return 0;
}

template <typename F>
int guarded(F&& f) {
    try {
        return f();
    } catch (const lattice_ref::UsageError& e) {
        g_err = e.what();
        return 1;
    } catch (const lattice_ref::DataError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {  // e.g. nlohmann's out_of_range.406 (number overflow)
        g_err = e.what();
        return 3;
    }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// core.hpp:84
uint64_t ref_stable_hash(const uint8_t* data, size_t len, uint64_t seed) {
    return lattice_ref::stable_hash(std::span<const std::uint8_t>(data, len), lattice_ref::Seed{seed});
}

// core.hpp:149-175, as used by datasets.hpp:181-184
size_t ref_signature(const char* user, uint32_t ulen, const char* ad, uint32_t alen, int64_t ts,
                     uint8_t* out) {
    lattice_ref::ByteWriter w;
    w.length_prefixed(std::string_view(user, ulen));
    w.length_prefixed(std::string_view(ad, alen));
    w.u64_be(static_cast<std::uint64_t>(ts));
    std::memcpy(out, w.view().data(), w.view().size());
    return w.view().size();
}

static lattice_ref::ZipperConfig make_config(int W, const int64_t* durations, const double* probs,
                                             uint64_t seed) {
    std::vector<lattice_ref::AttributionWindow> windows;
    for (int i = 0; i < W; ++i) windows.push_back({"w" + std::to_string(i), durations[i]});
    return lattice_ref::ZipperConfig::create(std::move(windows),
                                             std::vector<double>(probs, probs + W),
                                             lattice_ref::Seed{seed});
}

// datasets.hpp:60-84 validation only
int ref_zipper_config_check(int W, const int64_t* durations, const double* probs, uint64_t seed) {
    return guarded([&] {
        make_config(W, durations, probs, seed);
        return 0;
    });
}

// datasets.hpp:60-84 with caller-named windows (the drop-in's check order is fuzzed against it)
int ref_zipper_config_create(int W, const char* const* names, const int64_t* durations, const double* probs) {
    return guarded([&] {
        std::vector<lattice_ref::AttributionWindow> windows;
        for (int i = 0; i < W; ++i) windows.push_back({names[i], durations[i]});
        lattice_ref::ZipperConfig::create(std::move(windows), std::vector<double>(probs, probs + W),
                                          lattice_ref::Seed{7});
        return 0;
    });
}

// datasets.hpp:115-122
int ref_joined_domain_name(int n, const char* const* parts, char* out, int cap) {
    std::vector<std::string> v(parts, parts + n);
    const std::string s = lattice_ref::detail::joined_domain_name(v);
    if ((int)s.size() + 1 > cap) return -1;
    std::memcpy(out, s.c_str(), s.size() + 1);
    return (int)s.size();
}

// datasets.hpp:179
int ref_assign_window(const char* user, uint32_t ulen, const char* ad, uint32_t alen, int64_t ts,
                      int W, const int64_t* durations, const double* probs, uint64_t seed,
                      int64_t* out_window) {
    return guarded([&] {
        const auto cfg = make_config(W, durations, probs, seed);
        *out_window = static_cast<int64_t>(lattice_ref::assign_window(
            std::string_view(user, ulen), std::string_view(ad, alen), ts, cfg));
        return 0;
    });
}

// datasets.hpp:199 over columns. Tasks are named "t0".."t{T-1}". Returns 0 / 1 / 2 and
// fills window[n], labels[n*T*W]. On DataError the message is in ref_last_error().
int ref_zip_dataset(int64_t n, const char* user_bytes, const int64_t* user_off, const char* ad_bytes,
                    const int64_t* ad_off, const int64_t* ts, int T, const int64_t* conv,
                    const uint8_t* conv_present, int W, const int64_t* durations,
                    const double* probs, uint64_t seed, uint8_t* window, uint8_t* labels) {
    return guarded([&] {
        const auto cfg = make_config(W, durations, probs, seed);
        std::vector<std::string> tasks;
        for (int t = 0; t < T; ++t) tasks.push_back("t" + std::to_string(t));
        std::vector<lattice_ref::DomainRecord> recs(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) {
            auto& r = recs[static_cast<size_t>(i)];
            r.domain = "d";
            r.user_id.assign(user_bytes + user_off[i], static_cast<size_t>(user_off[i + 1] - user_off[i]));
            r.ad_id.assign(ad_bytes + ad_off[i], static_cast<size_t>(ad_off[i + 1] - ad_off[i]));
            r.impression_time_ms = ts[i];
            for (int t = 0; t < T; ++t)
                if (conv_present[i * T + t]) r.conversions[tasks[static_cast<size_t>(t)]] = conv[i * T + t];
        }
        const auto z = lattice_ref::zip_dataset(recs, tasks, cfg);
        for (int64_t i = 0; i < n; ++i) {
            const auto& zr = z.records[static_cast<size_t>(i)];
            window[i] = static_cast<uint8_t>(zr.assigned_window);
            std::memcpy(labels + i * T * W, zr.window_labels.data(), static_cast<size_t>(T * W));
        }
        return 0;
    });
}

// numerics.hpp:81-107
int ref_rms_norm(const double* x, size_t n, double eps, double* out) {
    return guarded([&] { return copy_out(lattice_ref::rms_norm(std::span<const double>(x, n), eps), out); });
}
int ref_swish_rn(const double* x, size_t n, double eps, double* out) {
    return guarded([&] { return copy_out(lattice_ref::swish_rn(std::span<const double>(x, n), eps), out); });
}
int ref_swish_rn_hard(const double* x, size_t n, double eps, double* out) {
    return guarded(
        [&] { return copy_out(lattice_ref::swish_rn_hard(std::span<const double>(x, n), eps), out); });
}

// numerics.hpp:46
int ref_correlation_loss(const double* x, const double* y, size_t n, double eps, double* out) {
    return guarded([&] {
        *out = lattice_ref::correlation_loss(std::span<const double>(x, n), std::span<const double>(y, n), eps);
        return 0;
    });
}

// datasets.hpp:262 over columns: the dataset is rebuilt from window[n] / labels[n][T][W]
// (tasks "t0".., windows "w0".. in config order); counts[W] and rates[W][T] come back in
// window order.
int ref_window_summary(int64_t n, int T, int W, const uint8_t* window, const uint8_t* labels,
                       const int64_t* durations, const double* probs, int64_t* counts, double* rates) {
    return guarded([&] {
        lattice_ref::ZippedDataset ds{{}, {}, make_config(W, durations, probs, 7), {}};
        for (int t = 0; t < T; ++t) ds.tasks.push_back("t" + std::to_string(t));
        ds.records.resize(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) {
            auto& r = ds.records[static_cast<size_t>(i)];
            r.assigned_window = window[i];
            r.window_labels.assign(labels + i * T * W, labels + (i + 1) * T * W);
        }
        const auto sum = lattice_ref::window_routing_summary(ds);
        for (int w = 0; w < W; ++w) {
            const auto& s = sum.at("w" + std::to_string(w));
            counts[w] = static_cast<int64_t>(s.count);
            for (int t = 0; t < T; ++t) rates[w * T + t] = s.positive_rate.at("t" + std::to_string(t));
        }
        return 0;
    });
}

// datasets.hpp:144 over columns. Domain g declares features "f<decl[g][j]>" (j < max_decl,
// -1 = unused slot); its n_rec[g] records (grouped by domain, in order) carry values[r][j] for
// every declared j. Writes the union feature ids (first-seen order) to union_ids and the
// padded matrix [n][n_union] in union order; returns 0 / 1 (UsageError) / 2 (DataError).
int ref_merge_domains(int G, int max_decl, const int32_t* decl, const int64_t* n_rec, const double* values,
                      int32_t* union_ids, int32_t* n_union, double* out) {
    return guarded([&] {
        std::vector<lattice_ref::DomainDataset> ds;
        int64_t r = 0;
        for (int g = 0; g < G; ++g) {
            std::vector<std::string> feats;
            for (int j = 0; j < max_decl; ++j)
                if (decl[g * max_decl + j] >= 0) feats.push_back("f" + std::to_string(decl[g * max_decl + j]));
            lattice_ref::DomainDataset d{lattice_ref::DatasetSchema::create("d" + std::to_string(g), feats), {}};
            for (int64_t i = 0; i < n_rec[g]; ++i, ++r) {
                lattice_ref::DomainRecord rec;
                rec.domain = d.schema.domain;
                for (int j = 0; j < max_decl; ++j)
                    if (decl[g * max_decl + j] >= 0)
                        rec.values["f" + std::to_string(decl[g * max_decl + j])] = values[r * max_decl + j];
                d.records.push_back(std::move(rec));
            }
            ds.push_back(std::move(d));
        }
        const auto u = lattice_ref::merge_domains(ds);
        *n_union = static_cast<int32_t>(u.schema.features.size());
        for (size_t c = 0; c < u.schema.features.size(); ++c) union_ids[c] = std::stoi(u.schema.features[c].substr(1));
        for (size_t i = 0; i < u.records.size(); ++i)
            for (size_t c = 0; c < u.schema.features.size(); ++c)
                out[i * u.schema.features.size() + c] = u.records[i].values.at(u.schema.features[c]);
        return 0;
    });
}

// numerics.hpp:113-156
int ref_swish_rn_jvp(const double* x, const double* t, size_t n, double eps, double* out) {
    return guarded([&] {
        return copy_out(lattice_ref::swish_rn_jvp(std::span<const double>(x, n), std::span<const double>(t, n), eps),
                        out);
    });
}
int ref_clip_features(const double* x, size_t n, double c, double* out) {
    return guarded([&] { return copy_out(lattice_ref::clip_features(std::span<const double>(x, n), c), out); });
}
int ref_smooth_labels(const double* y, size_t n, double eps_s, double* out) {
    return guarded([&] { return copy_out(lattice_ref::smooth_labels(std::span<const double>(y, n), eps_s), out); });
}

// ktap.hpp:126-229 driven through its public API: entry e = pair ("u<e>", "i<e>") is written by
// a refresh cycle at written_at[e] with embedding emb[e] and logit logit[e]; query q asks for
// entry slot[q] (-1 = a pair never written) at `now`; the row is student_feature_vector(result,
// base[q]) with the teacher block then clipped by clip_features when clip > 0. smoothing < 0 =
// no label smoothing. Outputs rows [n][base_dim+dim], logits [n] (NaN on a miss), hit [n].
int ref_student_queries(int64_t entries, int dim, const double* emb, const double* logit, const int64_t* written_at,
                        int64_t ttl, double smoothing, int64_t n, int base_dim, const double* base,
                        const int64_t* slot, int64_t now, double clip, double* rows, double* logits_out,
                        uint8_t* hit_out) {
    return guarded([&] {
        lattice_ref::StoreConfig cfg;
        cfg.dimension = static_cast<size_t>(dim);
        cfg.ttl_ms = ttl;
        cfg.refresh_budget = 1;
        if (smoothing >= 0.0) cfg.label_smoothing = smoothing;
        lattice_ref::TeacherEmbeddingStore store(cfg);
        auto key = [](int64_t e) { return lattice_ref::PairKey{"u" + std::to_string(e), "i" + std::to_string(e)}; };
        for (int64_t e = 0; e < entries; ++e) {
            store.student_query(key(e), written_at[e]);  // miss -> queued
            store.teacher_refresh_cycle(
                [&](const lattice_ref::PairKey&) {
                    return lattice_ref::TeacherOutput{std::vector<double>(emb + e * dim, emb + (e + 1) * dim), logit[e]};
                },
                written_at[e]);
        }
        const int W = base_dim + dim;
        for (int64_t q = 0; q < n; ++q) {
            const auto k = slot[q] >= 0 ? key(slot[q]) : lattice_ref::PairKey{"absent", "pair"};
            const auto r = store.student_query(k, now);
            auto row = lattice_ref::student_feature_vector(
                r, std::span<const double>(base + q * base_dim, static_cast<size_t>(base_dim)), static_cast<size_t>(dim));
            if (clip > 0.0) {
                const auto c = lattice_ref::clip_features(std::span<const double>(row.data() + base_dim, dim), clip);
                std::copy(c.begin(), c.end(), row.begin() + base_dim);
            }
            std::copy(row.begin(), row.end(), rows + q * W);
            logits_out[q] = r.teacher_logit ? *r.teacher_logit : std::nan("");
            hit_out[q] = r.hit ? 1 : 0;
        }
        return 0;
    });
}

// parse_jsonl_records (serde.hpp:158-170) over `content` -> the records as JSON text: [{"domain",
// "user_id", "ad_id", "impression_time_ms", "features": {key: "<16 hex digits of the double's
// bits>"}, "conversions": {key: int}}], malloc'ed into *out (ref_free). Status 2 + the DataError
// text on a bad file.
int ref_parse_jsonl(const char* content, size_t len, const char* source, char** out, size_t* out_len) {
    return guarded([&] {
        const auto recs = lattice_ref::parse_jsonl_records(std::string(content, len), source);
        nlohmann::json arr = nlohmann::json::array();
        for (const auto& r : recs) {
            nlohmann::json j;
            j["domain"] = r.domain;
            j["user_id"] = r.user_id;
            j["ad_id"] = r.ad_id;
            j["impression_time_ms"] = r.impression_time_ms;
            j["features"] = nlohmann::json::object();
            for (const auto& [k, v] : r.values) {
                uint64_t bits;
                std::memcpy(&bits, &v, 8);
                char hex[17];
                std::snprintf(hex, sizeof hex, "%016llx", (unsigned long long)bits);
                j["features"][k] = hex;
            }
            j["conversions"] = nlohmann::json::object();
            for (const auto& [k, v] : r.conversions) j["conversions"][k] = v;
            arr.push_back(std::move(j));
        }
        const std::string s = arr.dump();
        *out = static_cast<char*>(std::malloc(s.size() + 1));
        std::memcpy(*out, s.data(), s.size() + 1);
        *out_len = s.size();
        return 0;
    });
}
void ref_free(void* p) { std::free(p); }

}  // extern "C"
