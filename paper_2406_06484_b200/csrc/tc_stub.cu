// tc_stub.cu -- placeholder until the tcgen05 path lands (tc_supported=false).
#include "common.cuh"
namespace dn {
bool tc_supported(const deltanet_desc*) { return false; }
size_t tc_scratch_bytes(const deltanet_desc*) { return 0; }
int tc_fwd(const Args&, cudaStream_t) { return DELTANET_ERR_UNSUPPORTED; }
int tc_bwd(const Args&, cudaStream_t) { return DELTANET_ERR_UNSUPPORTED; }
int tc_launch_count(const deltanet_desc*, int) { return 0; }
}  // namespace dn
