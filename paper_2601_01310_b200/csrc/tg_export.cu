// tg_export.cu — parity-export kernel of libtarragon (destination keys -> rank, bank slot).
#include "tg_internal.h"

namespace tg {

// Parity export: destination key -> (rank, bank slot) of every pair of the last call.
__global__ void k_export_keys(const int32_t *key, int n, int S_max, int32_t *dr, int32_t *ds) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    int K = key[i];
    if (dr) dr[i] = K / S_max;
    if (ds) ds[i] = K % S_max;
  }
}

cudaError_t launch_export_keys(const CallArgs &a, int n, int32_t *dst_rank, int32_t *dst_slot, cudaStream_t s) {
  if (n > 0) k_export_keys<<<(n + 255) / 256, 256, 0, s>>>(a.key, n, a.S_max, dst_rank, dst_slot);
  return cudaGetLastError();
}

}  // namespace tg
