// tcgen05 (UMMA) key-hash GEMM: placeholder until the tensor-core path lands.
#include "hata_internal.h"
namespace hata {
cudaError_t launch_hash_keys_tc(const HashKeysParams&, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace hata
