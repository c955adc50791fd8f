#pragma once

// Drop-in for the impression-log half of proj/include/lattice/serde.hpp: parse_jsonl_records
// (serde.hpp:158-170, record_from_json :129-146) with the same signature and results, parsed
// on the GPU by lattice_jsonl_* (one thread per line; see include/lattice_b200.h). Blank lines
// are skipped, the first bad line throws DataError("<source>:<line>: <nlohmann exception text>");
// a number literal that overflows double throws the reference's un-wrapped
// "[json.exception.out_of_range.406] ..." text as JsonOutOfRange (not a DataError, as in the
// reference, where nlohmann's out_of_range escapes parse_json's parse_error catch).
// parse_jsonl_columns is the columnar form the Zipper consumes without building records;
// dataset_from_records (:172-194) groups one file's records into a DomainDataset.

#include <cstdint>
#include <map>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "datasets.hpp"
#include "device.hpp"

namespace lattice {

struct JsonOutOfRange : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// Columns of a JSONL impression file on the host (the device columns of lattice_jsonl_extract).
struct JsonlColumns {
    std::int64_t records = 0, lines = 0;
    std::vector<std::uint8_t> domain, user, ad;
    std::vector<std::int64_t> domain_off, user_off, ad_off, ts, line;
    std::vector<std::int64_t> feature_off, feature_key_off, conversion_off, conversion_key_off, conversion_val;
    std::vector<std::uint8_t> feature_key, conversion_key;
    std::vector<double> feature_val;
};

inline JsonlColumns parse_jsonl_columns(const std::string& content, const std::string& source) {
    device::Buffer<std::uint8_t> dev(reinterpret_cast<const std::uint8_t*>(content.data()), content.size());
    lattice_jsonl* h = nullptr;
    lattice_jsonl_info info{};
    const lattice_status st =
        lattice_jsonl_open(dev.get(), static_cast<std::int64_t>(content.size()), source.c_str(), &h, &info, nullptr);
    if (st == LATTICE_DATA && info.error_kind == 2) throw JsonOutOfRange(lattice_last_error());
    device::throw_status(st);
    struct Close {
        lattice_jsonl* h;
        ~Close() { lattice_jsonl_close(h); }
    } close{h};
    const auto N = static_cast<std::size_t>(info.records);
    auto sz = [](std::int64_t n) { return static_cast<std::size_t>(n > 0 ? n : 1); };
    device::Buffer<std::uint8_t> dom(sz(info.domain_bytes)), usr(sz(info.user_bytes)), ad(sz(info.ad_bytes)),
        fk(sz(info.feature_key_bytes)), ck(sz(info.conversion_key_bytes));
    device::Buffer<std::int64_t> dom_o(N + 1), usr_o(N + 1), ad_o(N + 1), ts(sz(N)), line(sz(N)), f_o(N + 1),
        fk_o(static_cast<std::size_t>(info.feature_entries) + 1), c_o(N + 1),
        ck_o(static_cast<std::size_t>(info.conversion_entries) + 1), cv(sz(info.conversion_entries));
    device::Buffer<double> fv(sz(info.feature_entries));
    lattice_jsonl_columns c{dom.get(), dom_o.get(), usr.get(), usr_o.get(), ad.get(), ad_o.get(), ts.get(),
                            line.get(), f_o.get(), fk.get(), fk_o.get(), fv.get(), c_o.get(), ck.get(),
                            ck_o.get(), cv.get()};
    device::throw_status(lattice_jsonl_extract(h, &c, nullptr));
    device::cuda(cudaDeviceSynchronize(), "jsonl extract");
    JsonlColumns out;
    out.records = info.records;
    out.lines = info.lines;
    auto take = [](const auto& buf, std::int64_t n) {
        auto v = buf.download();
        v.resize(static_cast<std::size_t>(n));
        return v;
    };
    out.domain = take(dom, info.domain_bytes);
    out.user = take(usr, info.user_bytes);
    out.ad = take(ad, info.ad_bytes);
    out.domain_off = dom_o.download();
    out.user_off = usr_o.download();
    out.ad_off = ad_o.download();
    out.ts = take(ts, info.records);
    out.line = take(line, info.records);
    out.feature_off = f_o.download();
    out.feature_key = take(fk, info.feature_key_bytes);
    out.feature_key_off = fk_o.download();
    out.feature_val = take(fv, info.feature_entries);
    out.conversion_off = c_o.download();
    out.conversion_key = take(ck, info.conversion_key_bytes);
    out.conversion_key_off = ck_o.download();
    out.conversion_val = take(cv, info.conversion_entries);
    return out;
}

// serde.hpp:158 -- one DomainRecord per non-blank line, in file order.
inline std::vector<DomainRecord> parse_jsonl_records(const std::string& content, const std::string& source) {
    const JsonlColumns c = parse_jsonl_columns(content, source);
    auto str = [](const std::vector<std::uint8_t>& b, const std::vector<std::int64_t>& o, std::size_t i) {
        return std::string(b.begin() + o[i], b.begin() + o[i + 1]);
    };
    std::vector<DomainRecord> records(static_cast<std::size_t>(c.records));
    for (std::size_t r = 0; r < records.size(); ++r) {
        DomainRecord& rec = records[r];
        rec.domain = str(c.domain, c.domain_off, r);
        rec.user_id = str(c.user, c.user_off, r);
        rec.ad_id = str(c.ad, c.ad_off, r);
        rec.impression_time_ms = c.ts[r];
        for (auto e = c.feature_off[r]; e < c.feature_off[r + 1]; ++e)
            rec.values[str(c.feature_key, c.feature_key_off, static_cast<std::size_t>(e))] =
                c.feature_val[static_cast<std::size_t>(e)];
        for (auto e = c.conversion_off[r]; e < c.conversion_off[r + 1]; ++e)
            rec.conversions[str(c.conversion_key, c.conversion_key_off, static_cast<std::size_t>(e))] =
                c.conversion_val[static_cast<std::size_t>(e)];
    }
    return records;
}

// serde.hpp:172-194 -- one JSONL file = one domain's dataset: every record carries the first
// record's domain tag; the schema is the first-seen union of feature names (records in file
// order, names in each record's map order). Host-side string work on the parsed records.
inline DomainDataset dataset_from_records(std::vector<DomainRecord> records, const std::string& source) {
    if (records.empty()) throw DataError(source + ": no records");
    const std::string& dom = records.front().domain;
    std::vector<FeatureId> names;
    std::set<FeatureId> known;
    for (const DomainRecord& r : records) {
        if (r.domain != dom)
            throw DataError(source + ": mixed domains '" + dom + "' and '" + r.domain + "' in one file");
        for (const auto& kv : r.values)
            if (known.insert(kv.first).second) names.push_back(kv.first);
    }
    try {
        DatasetSchema schema = DatasetSchema::create(dom, std::move(names));
        return DomainDataset{std::move(schema), std::move(records)};
    } catch (const UsageError& e) {  // the values came from a file: a data error (serde.hpp:54)
        throw DataError(source + ": " + e.what());
    }
}

}  // namespace lattice
