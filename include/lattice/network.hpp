#pragma once

// lattice::Network -- the consolidated MDMO model step that the reference
// only describes in prose. Same idiom as proj/include/lattice: value types in, value types
// out, UsageError / DataError on contract / data violations. The work runs on the current
// CUDA device through lattice_net_* (include/lattice_b200.h); inputs may be host vectors
// (copied in) or device pointers (forward_device, stream-ordered, no synchronisation).

#include <array>
#include <cstdint>
#include <string>
#include <vector>

#include "core.hpp"

namespace lattice {

struct NetworkConfig {
    int n = 8, d = 64, blocks = 2, nF = 4, nL = 4, k = 4;
    std::vector<int> mlp{32, 64, 256};  // n*k ... nF*d
    int domains = 2, heads = 2, tower_hidden = 64;
    bool hard_gate = false;             // swish_rn_hard activations
    std::int64_t max_batch = 512;
    Seed weight_seed{0x1A79};
    lattice_dtype dtype = LATTICE_F32;  // configs[0] is fp32 (TF32 tensor cores); bf16 otherwise
    // dense processor: the last dense_features of the n embeddings; 0 = none
    int dense_features = 0, dense_in = 0, dense_hidden = 0;
};

// Jagged sparse batch, feature-major CSR: bag (f, b) = ids[offsets[f*B+b] .. offsets[f*B+b+1]).
struct SparseBatch {
    std::int64_t batch = 0;
    std::vector<std::int64_t> offsets;  // [n*B + 1]
    std::vector<std::int32_t> ids;
    std::vector<std::int32_t> domain;   // [B]
};

// Device-resident embedding tables: one pointer per feature, bf16 or fp32 [rows][d].
struct TableSet {
    std::vector<const void*> tables;
    std::vector<std::int64_t> rows;
    lattice_dtype dtype = LATTICE_BF16;
};

class Network {
public:
    explicit Network(const NetworkConfig& c) : cfg_(c) {
        lattice_net_config nc{};
        nc.n = c.n;
        nc.d = c.d;
        nc.blocks = c.blocks;
        nc.nF = c.nF;
        nc.nL = c.nL;
        nc.k = c.k;
        if (c.mlp.size() < 2 || c.mlp.size() > 6) throw UsageError("Network: mlp needs 2..6 widths");
        nc.n_mlp = static_cast<std::int32_t>(c.mlp.size()) - 1;
        for (std::size_t i = 0; i < c.mlp.size(); ++i) nc.mlp[i] = c.mlp[i];
        nc.domains = c.domains;
        nc.heads = c.heads;
        nc.tower_hidden = c.tower_hidden;
        nc.hard = c.hard_gate ? 1 : 0;
        nc.max_batch = c.max_batch;
        nc.weight_seed = c.weight_seed.value;
        nc.dtype = c.dtype;
        nc.dense_features = c.dense_features;
        nc.dense_in = c.dense_in;
        nc.dense_hidden = c.dense_hidden;
        device::throw_status(lattice_net_create(&nc, &net_));
    }
    Network(const Network&) = delete;
    Network& operator=(const Network&) = delete;
    ~Network() { lattice_net_destroy(net_); }

    const NetworkConfig& config() const { return cfg_; }

    // Logits [B][heads] in batch order, heads = objectives x attribution windows.
    std::vector<float> forward(const SparseBatch& b, const TableSet& t) const {
        const int sparse = cfg_.n - cfg_.dense_features;
        if (b.domain.size() != static_cast<std::size_t>(b.batch) ||
            b.offsets.size() != static_cast<std::size_t>(sparse * b.batch + 1))
            throw UsageError("Network::forward: batch arrays do not match batch size");
        if (cfg_.dense_features > 0)
            throw UsageError("Network::forward: a network with dense features needs forward_device with batch.dense");
        if (t.tables.size() != static_cast<std::size_t>(sparse) || t.rows.size() != t.tables.size())
            throw UsageError("Network::forward: need one table per sparse feature");
        if (b.batch == 0) return {};
        // the CSR is already on the host: check it here so a malformed one is a DataError, never
        // a device read outside ids
        if (b.offsets.front() != 0)
            throw DataError("Network::forward: offsets must start at 0");
        for (std::size_t i = 1; i < b.offsets.size(); ++i)
            if (b.offsets[i] < b.offsets[i - 1])
                throw DataError("Network::forward: offsets decrease at bag " + std::to_string(i - 1));
        if (b.offsets.back() != static_cast<std::int64_t>(b.ids.size()))
            throw DataError("Network::forward: offsets end at " + std::to_string(b.offsets.back()) + ", ids has " +
                            std::to_string(b.ids.size()));
        device::Buffer<std::int64_t> d_off(b.offsets), d_rows(t.rows);
        device::Buffer<std::int32_t> d_ids(b.ids.empty() ? std::vector<std::int32_t>{0} : b.ids);
        device::Buffer<std::int32_t> d_dom(b.domain);
        device::Buffer<const void*> d_tab(t.tables);
        device::Buffer<float> d_logits(static_cast<std::size_t>(b.batch) * cfg_.heads);
        lattice_batch lb{};
        lb.batch = b.batch;
        lb.domain = d_dom.get();
        lb.table_dtype = t.dtype;
        lb.tables = d_tab.get();
        lb.rows = d_rows.get();
        lb.offsets = d_off.get();
        lb.ids = d_ids.get();
        lb.check = 1;  // host-vector call: synchronous anyway, so bad ids throw DataError
        device::throw_status(lattice_net_forward(net_, &lb, d_logits.get(), nullptr));
        return d_logits.download();
    }

    // Load trained weights (lattice_net_set_weight): `values` is the unpadded row-major fp32 tensor
    // of `kind` (1 Y^T [k][n], 2 W_L [nL][n], 3 MLP layer `index` of `block` [out][in], 4 tower W1
    // [G][tower_hidden][n*d], 5 tower W2 [G][heads][tower_hidden], 6 dense D1, 7 dense D2),
    // rounded to the network dtype on the device.
    void set_weight(int kind, int block, int index, const std::vector<float>& values) {
        const auto& c = cfg_;
        const std::int64_t nd = static_cast<std::int64_t>(c.n) * c.d;
        std::int64_t want = -1;
        switch (kind) {
            case 1: want = static_cast<std::int64_t>(c.k) * c.n; break;
            case 2: want = static_cast<std::int64_t>(c.nL) * c.n; break;
            case 3:
                if (index >= 0 && index + 1 < static_cast<int>(c.mlp.size()))
                    want = static_cast<std::int64_t>(c.mlp[index]) * c.mlp[index + 1];
                break;
            case 4: want = static_cast<std::int64_t>(c.domains) * c.tower_hidden * nd; break;
            case 5: want = static_cast<std::int64_t>(c.domains) * c.heads * c.tower_hidden; break;
            case 6: want = static_cast<std::int64_t>(c.dense_hidden) * c.dense_in; break;
            case 7: want = static_cast<std::int64_t>(c.dense_features) * c.d * c.dense_hidden; break;
            default: break;
        }
        if (want <= 0) throw UsageError("Network::set_weight: the network has no such weight");
        if (static_cast<std::int64_t>(values.size()) != want)
            throw UsageError("Network::set_weight: expected " + std::to_string(want) + " values, got " +
                             std::to_string(values.size()));
        device::Buffer<float> d(values);
        device::throw_status(lattice_net_set_weight(net_, block, kind, index, d.get(), LATTICE_F32, nullptr));
        device::cuda(cudaStreamSynchronize(nullptr), "Network::set_weight");
    }

    // Device-pointer entry: everything already on the GPU, ordered on `stream`.
    void forward_device(const lattice_batch& b, float* logits, cudaStream_t stream) const {
        device::throw_status(lattice_net_forward(net_, &b, logits, stream));
    }

    lattice_net* handle() const { return net_; }

private:
    NetworkConfig cfg_;
    lattice_net* net_ = nullptr;
};

}  // namespace lattice
