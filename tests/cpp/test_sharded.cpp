// C++ multi-GPU test of lattice::ShardedNetwork (include/lattice/sharded.hpp): W processes
// (fork, one GPU each) shard the tables, exchange CUDA IPC handles through a file-based
// all-gather, and every rank's logits must be bit-identical to a single-GPU lattice::Network
// forward of the same local batch over the full tables. Run by tests/test_multi_gpu.py on a
// box with >= 2 GPUs. Usage: test_sharded [W]. Exit code 0 = pass.
#include <sys/stat.h>
#include <sys/wait.h>
#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <fstream>
#include <string>
#include <thread>
#include <vector>

#include "lattice/sharded.hpp"

using namespace lattice;

namespace {

// Blocking all-gather over files: rank r writes <dir>/<round>.<r> (rename = atomic publish)
// and waits for every other rank's file of the same round.
struct FileAllGather {
    std::string dir;
    int rank, world;
    int round = 0;
    std::vector<Blob> operator()(const Blob& mine) {
        const std::string base = dir + "/" + std::to_string(round++) + ".";
        {
            const std::string tmp = base + std::to_string(rank) + ".tmp";
            std::ofstream f(tmp, std::ios::binary);
            f.write(reinterpret_cast<const char*>(mine.data()), static_cast<std::streamsize>(mine.size()));
            f.close();
            std::rename(tmp.c_str(), (base + std::to_string(rank)).c_str());
        }
        std::vector<Blob> all(static_cast<size_t>(world));
        for (int r = 0; r < world; ++r) {
            const std::string path = base + std::to_string(r);
            for (int spin = 0;; ++spin) {
                std::ifstream f(path, std::ios::binary);
                if (f) {
                    all[static_cast<size_t>(r)].assign(std::istreambuf_iterator<char>(f), {});
                    break;
                }
                if (spin > 60000) throw std::runtime_error("all_gather: timed out waiting for rank " + std::to_string(r));
                std::this_thread::sleep_for(std::chrono::milliseconds(1));
            }
        }
        return all;
    }
};

int run_rank(int rank, int world, const std::string& dir) {
    device::cuda(cudaSetDevice(rank), "cudaSetDevice");
    NetworkConfig cfg;
    cfg.n = 64;
    cfg.d = 128;
    cfg.blocks = 2;
    cfg.nF = 32;
    cfg.nL = 32;
    cfg.k = 16;
    cfg.mlp = {1024, 512, 4096};
    cfg.domains = 3;
    cfg.heads = 4;
    cfg.tower_hidden = 256;
    cfg.max_batch = 600;
    cfg.dtype = LATTICE_BF16;
    const int rows = 4000, F = cfg.n, D = cfg.d;
    const std::int64_t B = 600;
    // full tables (the single-GPU reference) and this rank's shard, both from the generator
    device::Buffer<std::uint16_t> full(static_cast<size_t>(F) * rows * D);
    device::throw_status(lattice_fill_tables(full.get(), LATTICE_BF16, F, rows, D, 0x1A77, 0, rows, nullptr));
    FileAllGather ag{dir, rank, world};
    ShardedNetwork sn(cfg, rank, world, std::ref(ag));
    const int Fl = sn.owned_count();
    device::Buffer<std::uint16_t> shard(static_cast<size_t>(Fl) * rows * D);
    device::throw_status(lattice_fill_tables(shard.get(), LATTICE_BF16, Fl, rows, D, 0x1A77, sn.owned_first(), rows,
                                             nullptr));
    TableSet tfull, towned;
    tfull.dtype = towned.dtype = LATTICE_BF16;
    for (int f = 0; f < F; ++f) {
        tfull.tables.push_back(full.get() + static_cast<size_t>(f) * rows * D);
        tfull.rows.push_back(rows);
    }
    for (int f = 0; f < Fl; ++f) {
        towned.tables.push_back(shard.get() + static_cast<size_t>(f) * rows * D);
        towned.rows.push_back(rows);
    }
    // this rank's batch
    device::Buffer<std::int64_t> off(static_cast<size_t>(F) * B + 1);
    device::Buffer<std::int32_t> ids(static_cast<size_t>(F) * B * 40), dom(static_cast<size_t>(B));
    device::throw_status(lattice_synth_bags(F, B, 40, rows, 0x1A78 + rank, off.get(), ids.get(), nullptr));
    device::throw_status(lattice_synth_domains(B, cfg.domains, 0x1A78 + rank, dom.get(), nullptr));
    device::cuda(cudaDeviceSynchronize(), "sync");
    // single-GPU reference on the same local batch
    Network ref(cfg);
    device::Buffer<float> want(static_cast<size_t>(B) * cfg.heads), got(static_cast<size_t>(B) * cfg.heads);
    device::Buffer<const void*> d_tab(tfull.tables);
    device::Buffer<std::int64_t> d_rows(tfull.rows);
    lattice_batch lb{};
    lb.batch = B;
    lb.domain = dom.get();
    lb.table_dtype = LATTICE_BF16;
    lb.tables = d_tab.get();
    lb.rows = d_rows.get();
    lb.offsets = off.get();
    lb.ids = ids.get();
    ref.forward_device(lb, want.get(), nullptr);
    // sharded: three steps (barrier epochs stay in lock step)
    const int key = sn.publish_inputs(off.get(), ids.get());
    for (int step = 0; step < 3; ++step) sn.forward(key, B, dom.get(), towned, got.get(), nullptr);
    device::cuda(cudaDeviceSynchronize(), "sync");
    sn.check();
    const auto w = want.download(), g = got.download();
    const bool same = w == g;
    std::printf("rank %d: sharded logits %s the single-GPU path\n", rank, same ? "bit-identical to" : "DIFFER from");
    return same ? 0 : 1;
}

}  // namespace

int main(int argc, char** argv) {
    const int world = argc > 1 ? std::atoi(argv[1]) : 2;
    char tmpl[] = "/tmp/lattice_ag_XXXXXX";
    const char* dir = mkdtemp(tmpl);
    if (!dir) return 2;
    std::vector<pid_t> kids;
    for (int r = 0; r < world; ++r) {  // fork before any CUDA call
        const pid_t pid = fork();
        if (pid == 0) {
            int rc = 1;
            try {
                rc = run_rank(r, world, dir);
            } catch (const std::exception& e) {
                std::fprintf(stderr, "rank %d: %s\n", r, e.what());
            }
            std::fflush(stdout);
            _exit(rc);
        }
        kids.push_back(pid);
    }
    int failed = 0;
    for (pid_t pid : kids) {
        int st = 0;
        waitpid(pid, &st, 0);
        failed += !(WIFEXITED(st) && WEXITSTATUS(st) == 0);
    }
    std::printf("sharded C++ test: %d of %d ranks failed\n", failed, world);
    return failed;
}
