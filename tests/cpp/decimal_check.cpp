// CPU check of csrc/decimal.cuh (the JSONL ingest's decimal -> binary64 conversion) against the
// C library's strtod, which is what nlohmann::json's lexer calls (serde.hpp parse_json).
// usage: decimal_check [count] [seed]   -> prints "ok N" or the first mismatch, exit 1
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>

#include "decimal.cuh"

static bool check(const std::string& s) {
    const double want = std::strtod(s.c_str(), nullptr);
    const double got = lat::dec::parse_double(reinterpret_cast<const uint8_t*>(s.data()),
                                              reinterpret_cast<const uint8_t*>(s.data()) + s.size());
    uint64_t a, b;
    std::memcpy(&a, &want, 8);
    std::memcpy(&b, &got, 8);
    if (a != b) {
        std::printf("MISMATCH %s strtod=%.17g (%016llx) ours=%.17g (%016llx)\n", s.c_str(), want,
                    (unsigned long long)a, got, (unsigned long long)b);
        return false;
    }
    return true;
}

int main(int argc, char** argv) {
    const long n = argc > 1 ? std::atol(argv[1]) : 200000;
    std::mt19937_64 rng(argc > 2 ? std::atoll(argv[2]) : 7);
    const char* fixed[] = {"0", "-0", "0.0", "-0.0", "1", "-1", "0.1", "1e308", "1.7976931348623157e308",
                           "1.7976931348623158e308", "1.7976931348623159e308", "2e308", "1e400",
                           "4.9406564584124654e-324", "2.4703282292062327e-324", "2.4703282292062328e-324",
                           "2.2250738585072011e-308", "2.2250738585072012e-308", "1e-400", "9007199254740993",
                           "9007199254740992.5", "9007199254740993.0000000000000000001", "123456789012345678901234567890",
                           "0.000000000000000000000000000001", "1e23", "8.41e21", "5e-324", "1e-324",
                           "179769313486231580793728971405303415079934132710037826936173778980444968292764750946649"
                           "017977587207096330286416692887910946555547851940402630657488671505820681908902000708383"
                           "676273854845817711531764475730270069855571366959622842914819860834936475292719074168444"
                           "365510704342711559699508093042880177904174497791.9999999999999999999999999999999999999",
                           "2.22507385850720113605740979670913197593481954635164564e-308",
                           "7.3177701707893310e+15", "100000000000000000000000", "1E+2", "1e-0", "0e99999",
                           "1.00000000000000011102230246251565404236316680908203125",
                           "1.00000000000000011102230246251565404236316680908203124",
                           "1.00000000000000011102230246251565404236316680908203126"};
    for (const char* f : fixed)
        if (!check(f)) return 1;
    long done = sizeof(fixed) / sizeof(*fixed);
    char buf[1200];
    for (long i = 0; i < n; ++i) {
        const int kind = (int)(rng() % 6);
        std::string s;
        if (kind == 0) {  // random double printed with 17 digits (the round trip nlohmann's dump uses)
            uint64_t bits = rng();
            double d;
            std::memcpy(&d, &bits, 8);
            if (d != d || d - d != 0) continue;
            std::snprintf(buf, sizeof buf, "%.17g", d);
            s = buf;
        } else if (kind == 1) {  // short decimals
            std::snprintf(buf, sizeof buf, "%.*f", (int)(rng() % 12), (double)(int64_t)(rng() % 2000001 - 1000000) / 997.0);
            s = buf;
        } else if (kind == 2) {  // near-halfway: exact binary midpoints printed in full
            uint64_t bits = (rng() & 0x7FEFFFFFFFFFFFFFull);
            double d, e2;
            std::memcpy(&d, &bits, 8);
            uint64_t nb = bits + 1;
            std::memcpy(&e2, &nb, 8);
            long double mid = ((long double)d + (long double)e2) / 2;
            std::snprintf(buf, sizeof buf, "%.40Le", mid);
            s = buf;
        } else if (kind == 3) {  // long digit strings
            int nd = 1 + (int)(rng() % 60);
            s = std::to_string(rng() % 9 + 1);
            for (int k = 0; k < nd; ++k) s += char('0' + rng() % 10);
            if (rng() % 2) s.insert(1 + rng() % s.size(), ".");
            if (s.back() == '.') s += "5";
            s += "e" + std::to_string((int64_t)(rng() % 700) - 350);
        } else if (kind == 4) {  // integers incl. beyond 2^53 and 2^64
            std::snprintf(buf, sizeof buf, "%llu%llu", (unsigned long long)(rng() % 100000),
                          (unsigned long long)rng());
            s = buf;
        } else {  // subnormal range
            uint64_t bits = rng() % (1ull << 52);
            double d;
            std::memcpy(&d, &bits, 8);
            std::snprintf(buf, sizeof buf, "%.*e", (int)(rng() % 25), d);
            s = buf;
        }
        if (rng() % 2 && s[0] != '-') s = "-" + s;
        // JSON grammar: no '+' mantissa sign, no leading '.', exponent digits present
        if (s.find("inf") != std::string::npos || s.find("nan") != std::string::npos) continue;
        if (!check(s)) return 1;
        ++done;
    }
    std::printf("ok %ld\n", done);
    return 0;
}
