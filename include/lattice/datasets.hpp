#pragma once

// Drop-in for the Zipper part of proj/include/lattice/datasets.hpp: the same types
// (datasets.hpp:18-111) and the same entry points assign_window (:179) and zip_dataset
// (:199), with the per-impression work done by the B200 kernel behind
// lattice_zipper_assign_labels. zip_dataset flattens the records into columns, runs one
// kernel over all of them and rebuilds the ZippedRecords in input order; the DataError for a
// conversion before its impression names the same first record and task as the reference.
// zip_columns is the batched columnar entry for callers that already hold columns.

#include <algorithm>
#include <cmath>
#include <map>
#include <set>
#include <string>
#include <string_view>
#include <vector>

#include "core.hpp"

namespace lattice {

struct DatasetSchema {
    std::string domain;
    std::vector<FeatureId> features;

    static DatasetSchema create(std::string domain, std::vector<FeatureId> features) {
        std::set<FeatureId> seen;
        for (const auto& f : features) {
            if (f.empty()) throw UsageError("DatasetSchema: empty feature name");
            if (!seen.insert(f).second)
                throw UsageError("DatasetSchema: duplicate feature '" + f + "' in domain '" + domain + "'");
        }
        return DatasetSchema{std::move(domain), std::move(features)};
    }
};

struct DomainRecord {
    std::string domain;
    std::string user_id;
    std::string ad_id;
    TimestampMs impression_time_ms = 0;
    std::map<FeatureId, double> values;
    std::map<TaskId, TimestampMs> conversions;
};

struct DomainDataset {
    DatasetSchema schema;
    std::vector<DomainRecord> records;
};

template <typename RecordT>
struct UnifiedDataset {
    DatasetSchema schema;  // union schema; records are padded to exactly these keys
    std::vector<RecordT> records;
};

struct AttributionWindow {
    std::string name;
    DurationMs duration_ms = 0;
};

struct ZipperConfig {
    std::vector<AttributionWindow> windows;
    std::vector<double> probabilities;
    Seed seed;

    // datasets.hpp:60-84 in its order: per window name, duplicate, then duration (one loop, so
    // the first offending window decides the message), then the probabilities -- whose checks,
    // like the durations', the library's lattice_zipper_validate repeats message for message.
    static ZipperConfig create(std::vector<AttributionWindow> windows, std::vector<double> probabilities,
                               Seed seed) {
        if (windows.empty()) throw UsageError("ZipperConfig: no windows");
        if (probabilities.size() != windows.size())
            throw UsageError("ZipperConfig: probabilities/windows length mismatch");
        std::set<std::string> names;
        DurationMs prev = 0;
        for (std::size_t i = 0; i < windows.size(); ++i) {
            const auto& w = windows[i];
            if (w.name.empty()) throw UsageError("ZipperConfig: empty window name");
            if (!names.insert(w.name).second)
                throw UsageError("ZipperConfig: duplicate window name '" + w.name + "'");
            if (w.duration_ms <= (i == 0 ? 0 : prev))
                throw UsageError("ZipperConfig: window durations must be positive and strictly increasing");
            prev = w.duration_ms;
        }
        std::vector<std::int64_t> dur;
        for (const auto& w : windows) dur.push_back(w.duration_ms);
        device::throw_status(lattice_zipper_validate(static_cast<std::int32_t>(windows.size()), dur.data(),
                                                     probabilities.data()));
        return ZipperConfig{std::move(windows), std::move(probabilities), seed};
    }

    std::size_t oracle_window() const { return windows.size() - 1; }
};

struct ZippedRecord {
    DomainRecord base;
    std::size_t assigned_window = 0;
    std::vector<std::uint8_t> window_labels;  // task-major: [task * W + window]

    std::uint8_t label(std::size_t task, std::size_t window, std::size_t window_count) const {
        return window_labels[task * window_count + window];
    }
};

struct ZippedDataset {
    DatasetSchema schema;
    std::vector<TaskId> tasks;
    ZipperConfig config;
    std::vector<ZippedRecord> records;
};

// Columnar batch: strings packed back to back, conversions per (record, task).
struct ZipColumns {
    std::vector<std::uint8_t> window;  // [n]
    std::vector<std::uint8_t> labels;  // [n][T][W]
    std::vector<std::uint8_t> routed;  // [n][T]: label of the assigned window
};

struct ZipBatchView {
    std::int64_t n = 0;
    const std::uint8_t* user_bytes = nullptr;
    const std::int64_t* user_off = nullptr;  // [n+1]
    const std::uint8_t* ad_bytes = nullptr;
    const std::int64_t* ad_off = nullptr;    // [n+1]
    const std::int64_t* ts = nullptr;        // [n]
    std::int32_t tasks = 0;
    const std::int64_t* conv = nullptr;      // [n][T]
    const std::uint8_t* conv_present = nullptr;
};

// Host columns in, host columns out; one kernel launch for the whole batch. Throws DataError
// ("record #i task #t ...") for the first record whose conversion precedes its impression.
inline ZipColumns zip_columns(const ZipBatchView& b, const ZipperConfig& config) {
    const std::size_t n = static_cast<std::size_t>(b.n), T = static_cast<std::size_t>(b.tasks);
    const std::size_t W = config.windows.size();
    ZipColumns out;
    if (n == 0) return out;
    auto nbytes = [](const std::int64_t* off, std::size_t n) { return static_cast<std::size_t>(off[n]); };
    const std::size_t ub = nbytes(b.user_off, n), ab = nbytes(b.ad_off, n);
    const std::uint8_t zero = 0;
    device::Buffer<std::uint8_t> d_ub(ub ? b.user_bytes : &zero, ub ? ub : 1);
    device::Buffer<std::uint8_t> d_ab(ab ? b.ad_bytes : &zero, ab ? ab : 1);
    device::Buffer<std::int64_t> d_uo(b.user_off, n + 1), d_ao(b.ad_off, n + 1), d_ts(b.ts, n);
    device::Buffer<std::int64_t> d_conv(T ? b.conv : nullptr, n * T);
    device::Buffer<std::uint8_t> d_pres(T ? b.conv_present : nullptr, n * T);
    device::Buffer<std::uint8_t> d_win(n), d_lab(n * T * W), d_rt(n * T);
    std::vector<std::int64_t> dur;
    for (const auto& w : config.windows) dur.push_back(w.duration_ms);
    lattice_zip_args a{};
    a.n = b.n;
    a.user_bytes = d_ub.get();
    a.user_off = d_uo.get();
    a.ad_bytes = d_ab.get();
    a.ad_off = d_ao.get();
    a.ts = d_ts.get();
    a.tasks = b.tasks;
    a.conv = d_conv.get();
    a.conv_present = d_pres.get();
    a.windows = static_cast<std::int32_t>(W);
    a.durations_host = dur.data();
    a.probabilities_host = config.probabilities.data();
    a.seed = config.seed.value;
    a.window = d_win.get();
    a.labels = d_lab.get();
    a.routed = T ? d_rt.get() : nullptr;
    a.check = 1;
    device::throw_status(lattice_zipper_assign_labels(&a, nullptr));
    out.window = d_win.download();
    out.labels = d_lab.download();
    if (T) out.routed = d_rt.download();
    return out;
}

inline std::size_t assign_window(std::string_view user_id, std::string_view ad_id,
                                 TimestampMs impression_time_ms, const ZipperConfig& config) {
    const std::int64_t uo[2] = {0, static_cast<std::int64_t>(user_id.size())};
    const std::int64_t ao[2] = {0, static_cast<std::int64_t>(ad_id.size())};
    ZipBatchView b;
    b.n = 1;
    b.user_bytes = reinterpret_cast<const std::uint8_t*>(user_id.data());
    b.user_off = uo;
    b.ad_bytes = reinterpret_cast<const std::uint8_t*>(ad_id.data());
    b.ad_off = ao;
    b.ts = &impression_time_ms;
    return zip_columns(b, config).window[0];
}

namespace detail {
inline std::string join_domains(const std::vector<std::string>& parts) {
    std::string out;
    for (const auto& p : parts) {  // datasets.hpp:115-122: '+' only after a non-empty prefix
        if (!out.empty()) out += "+";
        out += p;
    }
    return out;
}
}  // namespace detail

inline ZippedDataset zip_dataset(const std::vector<DomainRecord>& records, const std::vector<TaskId>& tasks,
                                 const ZipperConfig& config) {
    {
        std::set<TaskId> seen;
        for (const auto& t : tasks) {
            if (t.empty()) throw UsageError("zip_dataset: empty task name");
            if (!seen.insert(t).second) throw UsageError("zip_dataset: duplicate task '" + t + "'");
        }
    }
    const std::size_t n = records.size(), T = tasks.size(), W = config.windows.size();
    std::vector<std::uint8_t> ub, ab;
    std::vector<std::int64_t> uo{0}, ao{0}, ts(n), conv(n * T, 0);
    std::vector<std::uint8_t> pres(n * T, 0);
    for (std::size_t i = 0; i < n; ++i) {
        const auto& r = records[i];
        ub.insert(ub.end(), r.user_id.begin(), r.user_id.end());
        ab.insert(ab.end(), r.ad_id.begin(), r.ad_id.end());
        uo.push_back(static_cast<std::int64_t>(ub.size()));
        ao.push_back(static_cast<std::int64_t>(ab.size()));
        ts[i] = r.impression_time_ms;
        for (std::size_t t = 0; t < T; ++t) {
            auto it = r.conversions.find(tasks[t]);
            if (it == r.conversions.end()) continue;
            conv[i * T + t] = it->second;
            pres[i * T + t] = 1;
        }
    }
    ZipBatchView b;
    b.n = static_cast<std::int64_t>(n);
    b.user_bytes = ub.data();
    b.user_off = uo.data();
    b.ad_bytes = ab.data();
    b.ad_off = ao.data();
    b.ts = ts.data();
    b.tasks = static_cast<std::int32_t>(T);
    b.conv = conv.data();
    b.conv_present = pres.data();
    ZipColumns cols;
    try {
        cols = zip_columns(b, config);
    } catch (const DataError&) {
        // re-issue with the task's name, as datasets.hpp:236-238 words it
        const std::int64_t key = lattice_last_error_index();
        const std::size_t ri = static_cast<std::size_t>(key) / (T ? T : 1), ti = static_cast<std::size_t>(key) % (T ? T : 1);
        throw DataError("zip_dataset: record #" + std::to_string(ri) + " task '" + tasks[ti] +
                        "' converts before its impression");
    }
    ZippedDataset out;
    out.tasks = tasks;
    out.config = config;
    std::vector<FeatureId> features;
    std::set<FeatureId> seen_f;
    std::vector<std::string> domains;
    std::set<std::string> seen_d;
    out.records.reserve(n);
    for (std::size_t i = 0; i < n; ++i) {
        const auto& r = records[i];
        for (const auto& kv : r.values)
            if (seen_f.insert(kv.first).second) features.push_back(kv.first);
        if (seen_d.insert(r.domain).second) domains.push_back(r.domain);
        ZippedRecord z;
        z.base = r;
        z.assigned_window = cols.window[i];
        z.window_labels.assign(cols.labels.begin() + static_cast<std::ptrdiff_t>(i * T * W),
                               cols.labels.begin() + static_cast<std::ptrdiff_t>((i + 1) * T * W));
        out.records.push_back(std::move(z));
    }
    out.schema = DatasetSchema::create(detail::join_domains(domains), features);
    for (auto& z : out.records)
        for (const auto& f : out.schema.features) z.base.values.try_emplace(f, 0.0);
    return out;
}

// merge_domains (datasets.hpp:144-173): the union schema (first-seen order), the joined domain
// name and the undeclared-feature check are string work on the host; the values are re-laid
// out under the union schema with zero padding by lattice_merge_dense (fp64 in and out, exact).
inline UnifiedDataset<DomainRecord> merge_domains(const std::vector<DomainDataset>& datasets) {
    if (datasets.empty()) throw UsageError("merge_domains: no datasets");
    std::vector<FeatureId> features;
    std::set<FeatureId> seen;
    std::vector<std::string> names;
    for (const auto& d : datasets) {
        names.push_back(d.schema.domain);
        for (const auto& f : d.schema.features)
            if (seen.insert(f).second) features.push_back(f);
    }
    UnifiedDataset<DomainRecord> out;
    out.schema = DatasetSchema::create(detail::join_domains(names), features);
    const int G = static_cast<int>(datasets.size()), W = static_cast<int>(features.size());
    std::map<FeatureId, int> col;
    for (int c = 0; c < W; ++c) col[features[static_cast<size_t>(c)]] = c;
    int md = 1;
    std::size_t n = 0;
    for (const auto& d : datasets) {
        md = std::max(md, static_cast<int>(d.schema.features.size()));
        n += d.records.size();
    }
    std::vector<std::int32_t> src(static_cast<size_t>(G) * (W ? W : 1), -1), dom;
    std::vector<double> vals;
    vals.reserve(n * static_cast<size_t>(md));
    for (int g = 0; g < G; ++g) {
        const auto& d = datasets[static_cast<size_t>(g)];
        const std::set<FeatureId> declared(d.schema.features.begin(), d.schema.features.end());
        for (size_t j = 0; j < d.schema.features.size(); ++j)
            src[static_cast<size_t>(g) * W + static_cast<size_t>(col[d.schema.features[j]])] = static_cast<std::int32_t>(j);
        for (const auto& rec : d.records) {
            for (const auto& kv : rec.values)
                if (!declared.count(kv.first))
                    throw DataError("merge_domains: record in domain '" + d.schema.domain +
                                    "' carries undeclared feature '" + kv.first + "'");
            for (int j = 0; j < md; ++j) {
                double v = 0.0;  // a declared feature the record omits pads to 0 as well
                if (j < static_cast<int>(d.schema.features.size())) {
                    auto it = rec.values.find(d.schema.features[static_cast<size_t>(j)]);
                    if (it != rec.values.end()) v = it->second;
                }
                vals.push_back(v);
            }
            dom.push_back(g);
        }
    }
    std::vector<double> merged;
    if (n && W) {
        device::Buffer<std::int32_t> d_dom(dom), d_src(src);
        device::Buffer<double> d_vals(vals), d_out(n * static_cast<size_t>(W));
        device::throw_status(lattice_merge_dense(static_cast<std::int64_t>(n), G, md, d_dom.get(), d_vals.get(),
                                                 LATTICE_F64, d_src.get(), W, LATTICE_F64, d_out.get(), 1, nullptr));
        merged = d_out.download();
    }
    size_t r = 0;
    for (const auto& d : datasets)
        for (const auto& rec : d.records) {
            DomainRecord padded = rec;
            for (int c = 0; c < W; ++c)
                padded.values.try_emplace(features[static_cast<size_t>(c)], merged[r * static_cast<size_t>(W) + c]);
            out.records.push_back(std::move(padded));
            ++r;
        }
    return out;
}

struct WindowSummary {
    std::size_t count = 0;                   // records routed to this window
    std::map<TaskId, double> positive_rate;  // using the window's own label; 0.0 when count = 0
};

// window_routing_summary (datasets.hpp:256-283): the counts are one reduction kernel
// (lattice_window_summary, exact integers); the rates divide on the host like the reference.
inline std::map<std::string, WindowSummary> window_routing_summary(const ZippedDataset& dataset) {
    const std::size_t W = dataset.config.windows.size(), T = dataset.tasks.size(), n = dataset.records.size();
    std::vector<std::uint8_t> window(n), labels(n * T * W);
    for (std::size_t i = 0; i < n; ++i) {
        const auto& rec = dataset.records[i];
        if (rec.assigned_window >= W || rec.window_labels.size() != T * W || W > 255)
            throw UsageError("window_routing_summary: dataset not produced by zip_dataset");
        window[i] = static_cast<std::uint8_t>(rec.assigned_window);
        std::copy(rec.window_labels.begin(), rec.window_labels.end(), labels.begin() + static_cast<std::ptrdiff_t>(i * T * W));
    }
    std::vector<std::int64_t> counts(W, 0), pos(W * T, 0);
    if (n) {
        device::Buffer<std::uint8_t> d_w(window), d_l(labels.empty() ? std::vector<std::uint8_t>{0} : labels);
        device::Buffer<std::int64_t> d_c(W), d_p(W * T > 0 ? W * T : 1);
        device::throw_status(lattice_window_summary(static_cast<std::int64_t>(n), static_cast<std::int32_t>(T),
                                                    static_cast<std::int32_t>(W), d_w.get(), d_l.get(), d_c.get(),
                                                    d_p.get(), 1, nullptr));
        counts = d_c.download();
        if (W * T > 0) pos = d_p.download();
    }
    std::map<std::string, WindowSummary> out;
    for (std::size_t w = 0; w < W; ++w) {
        WindowSummary s;
        s.count = static_cast<std::size_t>(counts[w]);
        for (std::size_t t = 0; t < T; ++t)
            s.positive_rate[dataset.tasks[t]] =
                counts[w] == 0 ? 0.0 : static_cast<double>(pos[w * T + t]) / static_cast<double>(counts[w]);
        out[dataset.config.windows[w].name] = s;
    }
    return out;
}

}  // namespace lattice
