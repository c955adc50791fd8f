#pragma once

// lattice::ShardedNetwork -- the consolidated MDMO step across the GPUs of one node (SURVEY.md
// 8e): embedding tables sharded table-wise (rank r owns sparse features [r*F/W, (r+1)*F/W)),
// the dense part replicated. The embedding exchange runs over peer memory (NVLink/NVSwitch):
// every rank exports its network's X0 and sample rows, its input CSR buffers and a barrier
// flag array through CUDA IPC once; each step is
//   lattice_net_bucket -> lattice_peer_barrier -> lattice_peer_embedding_bag (one owner kernel:
//   peers' offsets/ids read over NVLink, pooled rows stored straight into each peer's X0)
//   -> lattice_peer_barrier -> lattice_net_forward (pooled_layout 2)
// with no host synchronisation and no NCCL call on the data path.
//
// The reference has no distributed layer, so the handle exchange is the caller's: `AllGather`
// is any blocking all-gather of byte blobs across the ranks (MPI, a torch.distributed store,
// files -- tests/cpp/test_sharded.cpp uses files). Same idiom as the rest of include/lattice:
// UsageError / DataError on contract / data violations.

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <functional>
#include <memory>
#include <vector>

#include "network.hpp"

namespace lattice {

using Blob = std::vector<std::uint8_t>;
using AllGather = std::function<std::vector<Blob>(const Blob&)>;

class ShardedNetwork {
public:
    // cfg.n embeddings, of which the first sparse = cfg.n - cfg.dense_features come from tables.
    ShardedNetwork(const NetworkConfig& cfg, int rank, int world, AllGather all_gather, double timeout_s = 30.0)
        : net_(cfg), rank_(rank), world_(world), ag_(std::move(all_gather)), timeout_s_(timeout_s) {
        sparse_ = cfg.n - cfg.dense_features;
        if (world < 1 || rank < 0 || rank >= world) throw UsageError("ShardedNetwork: bad rank/world");
        if (sparse_ % world) throw UsageError("ShardedNetwork: table-wise sharding needs the sparse feature count divisible by the world size");
        local_ = sparse_ / world;
        flags_ = device::Buffer<std::uint32_t>(static_cast<std::size_t>(world) + 1);
        status_ = device::Buffer<std::int32_t>(1);
        device::cuda(cudaMemset(flags_.get(), 0, sizeof(std::uint32_t) * (world + 1)), "cudaMemset");
        device::cuda(cudaMemset(status_.get(), 0, sizeof(std::int32_t)), "cudaMemset");
        flag_ptrs_ = share(flags_.get());
        out_ptrs_ = share(lattice_net_buffer(net_.handle(), 0));
        pos_ptrs_ = share(lattice_net_buffer(net_.handle(), 1));
    }
    ShardedNetwork(const ShardedNetwork&) = delete;
    ShardedNetwork& operator=(const ShardedNetwork&) = delete;
    ~ShardedNetwork() {
        for (void* p : opened_) lattice_ipc_close(p);
    }

    int owned_first() const { return rank_ * local_; }
    int owned_count() const { return local_; }
    Network& network() { return net_; }

    // Collective: publish one input buffer pair (this rank's CSR over all sparse features,
    // offsets [sparse*B + 1], ids) and return its handle. The buffers must outlive the object.
    int publish_inputs(const std::int64_t* offsets, const std::int32_t* ids) {
        inputs_.push_back({share(offsets), share(ids)});
        return static_cast<int>(inputs_.size()) - 1;
    }

    // One step on `stream`: domain [B] and logits [B][heads] are device pointers, `owned` holds
    // this rank's owned_count() tables (device [rows][d], net dtype), dense the optional dense
    // input. Stream-ordered; no host synchronisation.
    void forward(int inputs, std::int64_t batch, const std::int32_t* domain, const TableSet& owned, float* logits,
                 cudaStream_t stream, const void* dense = nullptr) {
        if (inputs < 0 || inputs >= static_cast<int>(inputs_.size())) throw UsageError("ShardedNetwork: unknown inputs");
        if (owned.tables.size() != static_cast<std::size_t>(local_) || owned.rows.size() != owned.tables.size())
            throw UsageError("ShardedNetwork::forward: need one table per owned feature");
        if (!tables_ || tables_host_ != owned.tables) {  // device copies of the owned table set
            tables_host_ = owned.tables;
            tables_ = std::make_unique<device::Buffer<const void*>>(owned.tables);
            rows_ = std::make_unique<device::Buffer<std::int64_t>>(owned.rows);
        }
        const auto& cfg = net_.config();
        device::throw_status(lattice_net_bucket(net_.handle(), batch, domain, stream));
        device::throw_status(lattice_peer_barrier(reinterpret_cast<std::uint32_t* const*>(flag_ptrs_.get()), rank_, world_, timeout_s_, status_.get(), stream));
        lattice_peer_bag_args a{};
        a.rank = rank_;
        a.world = world_;
        a.features_local = local_;
        a.feature_base = rank_ * local_;
        a.batch = batch;
        a.dim = cfg.d;
        a.table_dtype = owned.dtype;
        a.tables = tables_->get();
        a.rows = rows_->get();
        a.offsets = reinterpret_cast<const std::int64_t* const*>(inputs_[static_cast<std::size_t>(inputs)].first.get());
        a.ids = reinterpret_cast<const std::int32_t* const*>(inputs_[static_cast<std::size_t>(inputs)].second.get());
        a.sample_pos = reinterpret_cast<const std::int32_t* const*>(pos_ptrs_.get());
        a.out = out_ptrs_.get();
        a.out_dtype = cfg.dtype;
        a.out_row_stride = static_cast<std::int64_t>(cfg.n) * cfg.d;
        a.normalize = 1;
        device::throw_status(lattice_peer_embedding_bag(&a, stream));
        device::throw_status(lattice_peer_barrier(reinterpret_cast<std::uint32_t* const*>(flag_ptrs_.get()), rank_, world_, timeout_s_, status_.get(), stream));
        lattice_batch b{};
        b.batch = batch;
        b.domain = domain;
        b.table_dtype = cfg.dtype;
        b.pooled_layout = 2;
        b.dense = dense;
        net_.forward_device(b, logits, stream);
    }

    // Synchronises; throws if a barrier gave up waiting for a peer.
    void check() const {
        if (status_.download()[0] != 0) throw device::CudaError("ShardedNetwork: a peer never reached a barrier");
    }

private:
    // Collective: every rank exports `p`; returns a device array [world] of pointers (own at
    // [rank], the peers' mapped through CUDA IPC).
    device::Buffer<void*> share(const void* p) {
        Blob mine(LATTICE_IPC_HANDLE_BYTES + sizeof(std::int64_t));
        std::int64_t off = 0;
        device::throw_status(lattice_ipc_handle(p, mine.data(), &off));
        std::memcpy(mine.data() + LATTICE_IPC_HANDLE_BYTES, &off, sizeof(off));
        const std::vector<Blob> all = ag_(mine);
        if (all.size() != static_cast<std::size_t>(world_)) throw UsageError("ShardedNetwork: all_gather returned the wrong rank count");
        std::vector<void*> ptrs(static_cast<std::size_t>(world_));
        for (int r = 0; r < world_; ++r) {
            if (r == rank_) {
                ptrs[static_cast<std::size_t>(r)] = const_cast<void*>(p);
                continue;
            }
            const Blob& h = all[static_cast<std::size_t>(r)];
            if (h.size() != mine.size()) throw UsageError("ShardedNetwork: malformed peer handle");
            std::int64_t peer_off = 0;
            std::memcpy(&peer_off, h.data() + LATTICE_IPC_HANDLE_BYTES, sizeof(peer_off));
            void* q = nullptr;
            device::throw_status(lattice_ipc_open(h.data(), peer_off, &q));
            opened_.push_back(q);
            ptrs[static_cast<std::size_t>(r)] = q;
        }
        return device::Buffer<void*>(ptrs);
    }

    Network net_;
    int rank_, world_, sparse_ = 0, local_ = 0;
    AllGather ag_;
    double timeout_s_;
    device::Buffer<std::uint32_t> flags_;
    device::Buffer<std::int32_t> status_;
    device::Buffer<void*> flag_ptrs_, out_ptrs_, pos_ptrs_;
    std::vector<std::pair<device::Buffer<void*>, device::Buffer<void*>>> inputs_;
    std::vector<void*> opened_;
    std::vector<const void*> tables_host_;
    std::unique_ptr<device::Buffer<const void*>> tables_;
    std::unique_ptr<device::Buffer<std::int64_t>> rows_;
};

}  // namespace lattice
