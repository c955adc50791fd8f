// dropin_shim.cpp -- TEST INFRASTRUCTURE: exposes host-only pieces of the C++ drop-in
// (include/lattice/*.hpp) behind a C ABI so tests/test_dropin_cpu.py can fuzz them against the
// reference compiled in place (oracle/_ref) without a GPU. Built by __graft_entry__.build().
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "lattice/datasets.hpp"

namespace {
thread_local std::string g_err;
}

extern "C" {

const char* dropin_last_error() { return g_err.c_str(); }

// ZipperConfig::create: 0 ok, 1 UsageError (message in dropin_last_error), 3 other
int dropin_zipper_config_create(int W, const char* const* names, const int64_t* durations, const double* probs) {
    try {
        std::vector<lattice::AttributionWindow> w;
        for (int i = 0; i < W; ++i) w.push_back({names[i], durations[i]});
        lattice::ZipperConfig::create(std::move(w), std::vector<double>(probs, probs + W), lattice::Seed{7});
        return 0;
    } catch (const lattice::UsageError& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

// the joined schema name of zip_dataset / merge_domains (datasets.hpp:115-122)
int dropin_joined_domain_name(int n, const char* const* parts, char* out, int cap) {
    std::vector<std::string> v(parts, parts + n);
    const std::string s = lattice::detail::join_domains(v);
    if ((int)s.size() + 1 > cap) return -1;
    std::memcpy(out, s.c_str(), s.size() + 1);
    return (int)s.size();
}

}  // extern "C"
