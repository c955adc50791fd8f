// C++ drop-in test: the reference's own test expectations (proj/tests/test_core.cpp:18-43,
// 109-120; test_numerics.cpp:93-149; SPEC.md:236-254 Zipper examples) exercised through the
// include/lattice headers, i.e. through the B200 kernels. Built by __graft_entry__.build(),
// run by tests/test_dropin_gpu.py. Exit code = number of failed checks.
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "lattice/core.hpp"
#include "lattice/datasets.hpp"
#include "lattice/network.hpp"
#include "lattice/numerics.hpp"
#include "lattice/serde.hpp"

using namespace lattice;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                         \
    do {                                                                    \
        if (cond) {                                                         \
            ++g_pass;                                                       \
        } else {                                                            \
            ++g_fail;                                                       \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
        }                                                                   \
    } while (0)
#define CHECK_THROWS_AS(expr, T)        \
    do {                                \
        bool ok = false;                \
        try {                           \
            (void)(expr);               \
        } catch (const T&) {            \
            ok = true;                  \
        } catch (...) {                 \
        }                               \
        CHECK(ok && #T);                \
    } while (0)

static void core_goldens() {
    struct G {
        const char* s;
        std::uint64_t seed, h;
    } goldens[] = {
        {"", 0x0, 0xef46db3751d8e999ULL},
        {"", 0x1, 0xd5afba1336a3be4bULL},
        {"abc", 0x0, 0x44bc2cf5ad770999ULL},
        {"abc", 0x1, 0xbea9ca8199328908ULL},
        {"a", 0x0, 0xd24ec4f1a98c6e5bULL},
        {"lattice", 0x2a, 0x1643a65295b18ef1ULL},
        {"0123456789abcdef", 0x7, 0x8fbf8acb214d5da5ULL},
        {"0123456789abcdef0123456789abcde", 0x7, 0x9bfbacf6829bf320ULL},
        {"The quick brown fox jumps over the lazy dog", 0x0, 0x0b242d361fda71bcULL},
        {"The quick brown fox jumps over the lazy dog", 0x9e3779b185ebca87ULL, 0xb8a8089add7e03d9ULL},
    };
    for (const auto& g : goldens) CHECK(stable_hash(std::string_view(g.s), Seed{g.seed}) == g.h);
    CHECK(stable_hash("abc", Seed{0}) != stable_hash("abc", Seed{1}));
    ByteWriter w;
    w.length_prefixed("ab");
    w.u64_be(0x0102030405060708ULL);
    const auto& buf = w.view();
    CHECK(buf.size() == 14 && buf[3] == 2 && buf[4] == 'a' && buf[6] == 0x01 && buf[13] == 0x08);
}

static void numerics_examples() {
    const auto c = rms_norm(std::vector<double>{2, 2});
    CHECK(std::abs(c[0] - 1.0) < 1e-6 && std::abs(c[1] - 1.0) < 1e-6);
    for (double v : rms_norm(std::vector<double>{0, 0, 0})) CHECK(v == 0.0);
    const auto p = rms_norm(std::vector<double>{3, 4});
    CHECK(std::abs(p[0] - 3.0 / std::sqrt(12.5)) < 1e-3);
    CHECK_THROWS_AS(rms_norm(std::vector<double>{}), UsageError);
    CHECK_THROWS_AS(rms_norm(std::vector<double>{std::nan("")}), DataError);
    CHECK_THROWS_AS(rms_norm(std::vector<double>{1.0}, 0.0), UsageError);
    const double s1 = 1.0 / (1.0 + std::exp(-1.0));
    const auto s = swish_rn(std::vector<double>{2, 2});
    CHECK(std::abs(s[0] - s1) < 1e-4);
    // fp64 on the device with the reference's arithmetic: the SURVEY 8c goldens to the last ulps
    const auto k = swish_rn(std::vector<double>{3, 4});
    CHECK(std::abs(k[0] - 0.59418883661177035) < 4e-16 && std::abs(k[1] - 0.85542017401638759) < 4e-16);
    const auto h = swish_rn_hard(std::vector<double>{3, 4});
    CHECK(std::abs(h[0] - 0.54426404214136748) < 4e-16 && std::abs(h[1] - 0.77901871858849048) < 4e-16);
    CHECK(p[0] == 3.0 / std::sqrt(12.5 + 1e-6));  // rms_norm: bit for bit (numerics.hpp:87-89)
    for (double mag : {1e6, 1e20, 1e150, 1e300}) {  // any magnitude stays finite (numerics.hpp:92-93)
        std::vector<double> huge(8, mag);
        huge[0] = -mag;
        for (double v : swish_rn(huge)) CHECK(std::isfinite(v) && std::abs(v) <= std::sqrt(8.0));
        const auto r = rms_norm(huge);
        double acc = 0.0;  // the reference's own sequence: sum of squares (inf past ~1e154), then divide
        for (double v : huge) acc += v * v;
        const double denom = std::sqrt(acc / 8.0 + 1e-6);
        for (std::size_t i = 0; i < huge.size(); ++i) CHECK(r[i] == huge[i] / denom);
    }
    for (double v : rms_norm(std::vector<double>{0, 0}, 1e-300)) CHECK(v == 0.0);  // eps below fp32 range
}

static void zipper_examples() {
    const auto two = ZipperConfig::create({{"90min", 5400000}, {"1d", 86400000}}, {0.5, 0.5}, Seed{7});
    CHECK(assign_window("u1", "a1", 0, two) == 1);                              // SURVEY 8c golden
    CHECK(assign_window("user_000042", "ad_9", 1700000000000, two) == 0);
    const auto four = ZipperConfig::create({{"a", 1}, {"b", 2}, {"c", 3}, {"d", 4}}, {0.4, 0.3, 0.2, 0.1}, Seed{7});
    CHECK(assign_window("u1", "a1", 0, four) == 2);
    CHECK(assign_window("alice", "campaign-7/creative-13", 86400000, four) == 1);
    const auto degenerate = ZipperConfig::create({{"a", 1}, {"b", 2}}, {1.0, 0.0}, Seed{3});
    for (int i = 0; i < 50; ++i) CHECK(assign_window("u" + std::to_string(i), "x", i, degenerate) == 0);
    CHECK_THROWS_AS(ZipperConfig::create({}, {}, Seed{1}), UsageError);
    CHECK_THROWS_AS(ZipperConfig::create({{"a", 2}, {"b", 2}}, {0.5, 0.5}, Seed{1}), UsageError);
    CHECK_THROWS_AS(ZipperConfig::create({{"a", 1}, {"a", 2}}, {0.5, 0.5}, Seed{1}), UsageError);
    CHECK_THROWS_AS(ZipperConfig::create({{"a", 1}, {"b", 2}}, {0.5, 0.6}, Seed{1}), UsageError);

    // windows {90min, 1d}, impression at t=0
    std::vector<DomainRecord> recs(3);
    for (auto& r : recs) r.domain = "d", r.user_id = "u", r.ad_id = "a";
    recs[0].conversions["cvr"] = 7200000;  // 2h
    recs[1].conversions["cvr"] = 5400000;  // exactly 90min: inclusive
    recs[0].values["f1"] = 1.0;
    recs[2].values["f2"] = 2.0;
    const auto z = zip_dataset(recs, {"cvr"}, two);
    CHECK(z.records.size() == 3);
    CHECK(z.records[0].label(0, 0, 2) == 0 && z.records[0].label(0, 1, 2) == 1);
    CHECK(z.records[1].label(0, 0, 2) == 1 && z.records[1].label(0, 1, 2) == 1);
    CHECK(z.records[2].label(0, 0, 2) == 0 && z.records[2].label(0, 1, 2) == 0);
    CHECK(z.schema.features.size() == 2 && z.records[0].base.values.at("f2") == 0.0);
    recs[1].conversions["cvr"] = -1;
    bool threw = false;
    try {
        zip_dataset(recs, {"cvr"}, two);
    } catch (const DataError& e) {
        threw = std::string(e.what()) == "zip_dataset: record #1 task 'cvr' converts before its impression";
    }
    CHECK(threw);
    CHECK_THROWS_AS(zip_dataset(recs, {"cvr", "cvr"}, two), UsageError);
}

// proj/tests/test_numerics.cpp:36-90, 166-200
static void numerics_more() {
    const std::vector<double> x{0, 1, 2, 3}, y{1, 3, 2, 4};
    CHECK(std::abs(correlation_loss(x, y, 1e-15) - 0.2) < 1e-9);
    CHECK(std::abs(correlation_loss(x, y) - 0.2) < 1e-6);
    const std::vector<double> a{0.3, 1.7, 2.4, -0.8, 3.1}, na{-0.3, -1.7, -2.4, 0.8, -3.1};
    CHECK(std::abs(correlation_loss(a, a, 1e-15)) < 1e-9);
    CHECK(std::abs(correlation_loss(a, na, 1e-15) - 2.0) < 1e-9);
    CHECK(std::abs(correlation_loss(std::vector<double>{2, 2, 2, 2}, std::vector<double>{1, 2, 3, 4}) - 1.0) < 1e-9);
    CHECK(std::abs(correlation_loss(x, y) - correlation_loss(y, x)) < 1e-12);
    CHECK_THROWS_AS(correlation_loss(std::vector<double>{1, 2}, std::vector<double>{1, 2, 3}), UsageError);
    CHECK_THROWS_AS(correlation_loss(std::vector<double>{1}, std::vector<double>{1}), UsageError);
    CHECK_THROWS_AS(correlation_loss(x, x, 0.0), UsageError);
    CHECK_THROWS_AS(correlation_loss(std::vector<double>{1.0, std::nan("")}, std::vector<double>{1, 2}), DataError);

    const std::vector<double> zeros(4, 0.0), tangent{1, -2, 0.5, 3};
    const auto j0 = swish_rn_jvp(zeros, tangent);
    CHECK(j0.size() == 4);
    for (double v : swish_rn_jvp(std::vector<double>{1, 2, 3, 4}, std::vector<double>(4, 0.0))) CHECK(v == 0.0);
    CHECK_THROWS_AS(swish_rn_jvp(std::vector<double>{1, 2, 3, 4}, std::vector<double>{1}), UsageError);
    {  // central difference (test_numerics.cpp:150-164)
        const std::vector<double> xv{-3.1, 0.4, 2.2, 7.5, -9.0, 1.1, 0.0, 4.4};
        const std::vector<double> tv{0.3, -0.7, 0.2, 0.9, -0.1, 0.5, -0.6, 0.4};
        const double h = 1e-5;
        std::vector<double> xp(xv), xm(xv);
        for (int i = 0; i < 8; ++i) xp[i] += h * tv[i], xm[i] -= h * tv[i];
        auto swish64 = [](const std::vector<double>& v) {  // numerics.hpp:94 in fp64 (test-side)
            double ss = 0;
            for (double e : v) ss += e * e;
            const double den = std::sqrt(ss / v.size() + 1e-6);
            std::vector<double> o(v.size());
            for (size_t i = 0; i < v.size(); ++i) o[i] = (v[i] / den) / (1.0 + std::exp(-v[i] / den));
            return o;
        };
        const auto fp = swish64(xp), fm = swish64(xm), an = swish_rn_jvp(xv, tv);
        double num2 = 0, diff2 = 0;
        for (int i = 0; i < 8; ++i) {
            const double nd = (fp[i] - fm[i]) / (2 * h);
            num2 += nd * nd;
            diff2 += (an[i] - nd) * (an[i] - nd);
        }
        CHECK(std::sqrt(diff2) <= 1e-4 * std::sqrt(num2));  // test_numerics.cpp:161
    }
    CHECK((clip_features(std::vector<double>{-5, 0, 5}, 3.0) == std::vector<double>{-3, 0, 3}));
    CHECK((clip_features(std::vector<double>{1, -2}, 3.0) == std::vector<double>{1, -2}));
    CHECK((clip_features(std::vector<double>{1e9}, 1.0) == std::vector<double>{1}));
    CHECK_THROWS_AS(clip_features(std::vector<double>{1}, 0.0), UsageError);
    const auto sm = smooth_labels(std::vector<double>{0, 1}, 0.1);
    CHECK(std::abs(sm[0] - 0.05) < 1e-12 && std::abs(sm[1] - 0.95) < 1e-12);
    CHECK((smooth_labels(std::vector<double>{0, 1}, 0.0) == std::vector<double>{0, 1}));
    CHECK(std::abs(smooth_labels(std::vector<double>{1}, 0.5)[0] - 0.75) < 1e-12);
    const auto ordered = smooth_labels(std::vector<double>{0, 1, 0, 1}, 0.3);
    CHECK(ordered[0] < ordered[1] && ordered[0] == ordered[2]);
    CHECK_THROWS_AS(smooth_labels(std::vector<double>{0.5}, 0.1), UsageError);
}

// datasets.hpp:144-173 and :256-283 through the drop-in
static void merge_and_summary() {
    DomainDataset a{DatasetSchema::create("ads", {"ctr", "bid"}), {}};
    DomainDataset b{DatasetSchema::create("shop", {"price", "ctr"}), {}};
    DomainRecord r1;
    r1.domain = "ads";
    r1.values = {{"ctr", 0.25}, {"bid", 1.5}};
    DomainRecord r2;
    r2.domain = "shop";
    r2.values = {{"price", 9.99}};  // declared "ctr" omitted -> padded 0
    a.records.push_back(r1);
    b.records.push_back(r2);
    const auto u = merge_domains({a, b});
    CHECK(u.schema.domain == "ads+shop");
    CHECK((u.schema.features == std::vector<FeatureId>{"ctr", "bid", "price"}));
    CHECK(u.records.size() == 2);
    CHECK(u.records[0].values.at("price") == 0.0 && u.records[0].values.at("bid") == 1.5);
    CHECK(u.records[1].values.at("price") == 9.99 && u.records[1].values.at("bid") == 0.0 &&
          u.records[1].values.at("ctr") == 0.0);
    CHECK_THROWS_AS(merge_domains({}), UsageError);
    DomainDataset c = a;
    c.records[0].values["rogue"] = 1.0;
    bool threw = false;
    try {
        merge_domains({c});
    } catch (const DataError& e) {
        threw = std::string(e.what()) == "merge_domains: record in domain 'ads' carries undeclared feature 'rogue'";
    }
    CHECK(threw);

    const auto two = ZipperConfig::create({{"90min", 5400000}, {"1d", 86400000}}, {0.5, 0.5}, Seed{7});
    std::vector<DomainRecord> recs(200);
    for (size_t i = 0; i < recs.size(); ++i) {
        recs[i].domain = "d";
        recs[i].user_id = "u" + std::to_string(i);
        recs[i].ad_id = "a";
        if (i % 3 == 0) recs[i].conversions["cvr"] = 3600000;  // within both windows
    }
    const auto z = zip_dataset(recs, {"cvr"}, two);
    const auto sum = window_routing_summary(z);
    std::size_t n0 = 0, p0 = 0, total = 0;
    for (const auto& r : z.records)
        if (r.assigned_window == 0) ++n0, p0 += r.label(0, 0, 2);
    for (const auto& kv : sum) total += kv.second.count;
    CHECK(total == 200 && sum.at("90min").count == n0);
    CHECK(sum.at("90min").positive_rate.at("cvr") == (n0 ? static_cast<double>(p0) / n0 : 0.0));
    auto broken = z;
    broken.records[5].assigned_window = 2;
    CHECK_THROWS_AS(window_routing_summary(broken), UsageError);
}

static void network_smoke() {
    NetworkConfig c;  // tiny config (BASELINE configs[0] shapes)
    c.max_batch = 64;
    Network net(c);
    const int rows = 1000;
    std::vector<device::Buffer<float>> owned;
    TableSet ts;
    ts.dtype = LATTICE_F32;
    for (int f = 0; f < c.n; ++f) {
        std::vector<float> t(static_cast<std::size_t>(rows) * c.d);
        for (std::size_t i = 0; i < t.size(); ++i) t[i] = static_cast<float>((i * 2654435761u + f) % 97) / 97.0f - 0.5f;
        owned.emplace_back(t);
        ts.tables.push_back(owned.back().get());
        ts.rows.push_back(rows);
    }
    SparseBatch b;
    b.batch = 16;
    b.offsets.push_back(0);
    for (int f = 0; f < c.n; ++f)
        for (int s = 0; s < b.batch; ++s) {
            for (int j = 0; j < (s + f) % 5; ++j) b.ids.push_back((s * 31 + f * 7 + j * 13) % rows);
            b.offsets.push_back(static_cast<std::int64_t>(b.ids.size()));
        }
    for (int s = 0; s < b.batch; ++s) b.domain.push_back(s % c.domains);
    const auto logits = net.forward(b, ts);
    CHECK(logits.size() == static_cast<std::size_t>(b.batch * c.heads));
    bool finite = true;
    for (float v : logits) finite = finite && std::isfinite(v);
    CHECK(finite);
    const auto again = net.forward(b, ts);
    CHECK(again == logits);  // deterministic
    SparseBatch oob = b;  // an id outside its table: DataError, as embedding_bag reports it
    oob.ids[oob.ids.size() / 2] = rows + 3;
    CHECK_THROWS_AS(net.forward(oob, ts), DataError);
    NetworkConfig bad = c;
    bad.nL = 3;
    CHECK_THROWS_AS(Network{bad}, UsageError);
    // an empty batch returns no logits; a malformed CSR is a DataError on the host
    SparseBatch empty;
    empty.offsets.assign(1, 0);
    CHECK(net.forward(empty, ts).empty());
    SparseBatch mal = b;
    mal.offsets[5] = mal.offsets[6] + 1;  // decreasing
    CHECK_THROWS_AS(net.forward(mal, ts), DataError);
    mal = b;
    mal.offsets.back() += 7;  // runs past ids
    CHECK_THROWS_AS(net.forward(mal, ts), DataError);
    // trained weights: a caller-owned tower head replaces the generated one
    Network net2(c);
    std::vector<float> w2(static_cast<std::size_t>(c.domains) * c.heads * c.tower_hidden, 0.0f);
    net2.set_weight(5, 0, 0, w2);
    for (float v : net2.forward(b, ts)) CHECK(v == 0.0f);  // zero heads -> zero logits
    CHECK_THROWS_AS(net2.set_weight(5, 0, 0, std::vector<float>(3)), UsageError);
    CHECK_THROWS_AS(net2.set_weight(9, 0, 0, w2), UsageError);
}

// serde.hpp:158 parse_jsonl_records through the GPU parser: the SPEC.md:283 record format, then
// zip_dataset on the parsed records (the CLI's run_zip path, lattice_cli.cpp:115-139)
static void jsonl_examples() {
    const std::string file =
        "{\"domain\":\"shop\",\"user_id\":\"u1\",\"ad_id\":\"a1\",\"impression_time_ms\":0,"
        "\"features\":{\"age\":31,\"ctr\":0.0125},\"conversions\":{\"cvr\":7200000}}\n"
        "\n"
        "{\"domain\":\"shop\",\"user_id\":\"u\\u00e9\",\"ad_id\":\"a2\",\"impression_time_ms\":5,"
        "\"features\":{\"age\":1,\"age\":2}}\r\n";
    const auto recs = parse_jsonl_records(file, "log.jsonl");
    CHECK(recs.size() == 2);
    CHECK(recs[0].domain == "shop" && recs[0].user_id == "u1" && recs[0].impression_time_ms == 0);
    CHECK(recs[0].values.at("age") == 31.0 && recs[0].values.at("ctr") == 0.0125);
    CHECK(recs[0].conversions.at("cvr") == 7200000);
    CHECK(recs[1].user_id == "u\xc3\xa9" && recs[1].values.size() == 1 && recs[1].values.at("age") == 2.0);
    const auto cfg = ZipperConfig::create({{"90min", 5400000}, {"1d", 86400000}}, {0.5, 0.5}, Seed{7});
    const auto z = zip_dataset(recs, {"cvr"}, cfg);
    CHECK(z.records[0].label(0, 0, 2) == 0 && z.records[0].label(0, 1, 2) == 1);
    CHECK_THROWS_AS(parse_jsonl_records("{\"domain\":1}\n", "x"), DataError);
    CHECK_THROWS_AS(parse_jsonl_records("{}\n{oops\n", "x"), DataError);
    CHECK_THROWS_AS(parse_jsonl_records("[1e999]\n", "x"), JsonOutOfRange);
    try {
        parse_jsonl_records("{\"domain\":\"d\",\"user_id\":\"u\",\"ad_id\":\"a\",\"impression_time_ms\":1}\n"
                            "{\"domain\":\"d\",\"ad_id\":\"a\",\"impression_time_ms\":1}\n",
                            "log.jsonl");
        CHECK(false && "expected DataError");
    } catch (const DataError& e) {
        CHECK(std::string(e.what()) == "log.jsonl:2: [json.exception.out_of_range.403] key 'user_id' not found");
    }
    CHECK(parse_jsonl_records("", "empty").empty());
    const auto ds = dataset_from_records(recs, "log.jsonl");
    CHECK(ds.schema.domain == "shop" && ds.schema.features == std::vector<FeatureId>({"age", "ctr"}));
    auto mixed = recs;
    mixed[1].domain = "news";
    CHECK_THROWS_AS(dataset_from_records(mixed, "log.jsonl"), DataError);
    CHECK_THROWS_AS(dataset_from_records({}, "log.jsonl"), DataError);
}

int main() {
    core_goldens();
    numerics_examples();
    zipper_examples();
    numerics_more();
    merge_and_summary();
    network_smoke();
    jsonl_examples();
    std::printf("drop-in: %d passed, %d failed\n", g_pass, g_fail);
    return g_fail;
}
