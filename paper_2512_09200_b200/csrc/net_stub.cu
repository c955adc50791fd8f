// Temporary entry points for the tcgen05 GEMM / network, replaced by gemm.cu / network.cu.
#include "common.cuh"
extern "C" {
lattice_status lattice_net_create(const lattice_net_config*, lattice_net**) {
    return lat::set_error(LATTICE_USAGE, "lattice_net: not built yet");
}
void lattice_net_destroy(lattice_net*) {}
const void* lattice_net_weight(lattice_net*, int32_t, int32_t, int32_t) { return nullptr; }
lattice_status lattice_net_forward(lattice_net*, const lattice_batch*, float*, lattice_stream) {
    return lat::set_error(LATTICE_USAGE, "lattice_net: not built yet");
}
lattice_status lattice_net_set_timing(lattice_net*, int32_t) { return LATTICE_OK; }
lattice_status lattice_net_stage_times(lattice_net*, float*, int32_t, int32_t* n) { *n = 0; return LATTICE_OK; }
}
