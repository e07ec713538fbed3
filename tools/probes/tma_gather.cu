// tma_gather.cu — per-SM delivery of 128-row x 64-col bf16 token tiles (16 KB, 128-B swizzle)
// into an smem ring, either as one 2D TMA box (rows contiguous) or as 32 TMA tile::gather4 loads
// of 4 arbitrary rows each (rows taken from a random permutation: the rows of one expert's
// tokens in x).  `issuers` lanes of one warp issue, each with its own ring.  Source 32 MB
// (8192 x 2048 bf16: the Qwen-shaped prefill x), L2-resident after the first pass.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_gather tma_gather.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(32, 1) k_gather(const __grid_constant__ CUtensorMap tile_map,
                                                 const __grid_constant__ CUtensorMap row_map, const int *perm,
                                                 int nrows, int kblocks, int nstage, int tiles, int gather,
                                                 int issuers, unsigned long long *cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t *ring = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  __shared__ uint64_t bars[8][8];
  const int w = threadIdx.x;
  if (w >= issuers) return;
  const uint32_t tile = 128 * 128;
  uint64_t *bar = bars[w];
  ring += (size_t)w * nstage * tile;
  for (int i = 0; i < nstage; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint32_t phase[8] = {0};
  const int ntile_rows = nrows / 128;
  long long t0 = clock64();
  auto issue = [&](int j, int s) {
    const int t = (blockIdx.x * issuers + w + j * 997) % (ntile_rows * kblocks);
    const int rt = t / kblocks, kb = t % kblocks;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(tile) : "memory");
    uint8_t *dst = ring + (size_t)s * tile;
    if (!gather) {
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
          ::"r"(su32(dst)), "l"((uint64_t)&tile_map), "r"(su32(&bar[s])), "r"(kb * 64), "r"(rt * 128) : "memory");
    } else {
      const int *p = perm + rt * 128;
      for (int g = 0; g < 32; ++g) {
        const int4 r = *reinterpret_cast<const int4 *>(p + 4 * g);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
            ::"r"(su32(dst + g * 512)), "l"((uint64_t)&row_map), "r"(su32(&bar[s])), "r"(kb * 64), "r"(r.x),
              "r"(r.y), "r"(r.z), "r"(r.w) : "memory");
      }
    }
  };
  for (int s = 0; s < nstage && s < tiles; ++s) issue(s, s);
  for (int j = 0; j < tiles; ++j) {
    const int s = j % nstage;
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.b32 %0, 1, 0, P;\n\t}"
                   : "=r"(ok) : "r"(su32(&bar[s])), "r"(phase[s]) : "memory");
    phase[s] ^= 1;
    if (j + nstage < tiles) issue(j + nstage, s);
  }
  if (w == 0) cycles[blockIdx.x] = clock64() - t0;
}

typedef CUresult (*PFN)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                        const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                        CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char **argv) {
  const int ctas = argc > 1 ? atoi(argv[1]) : 148;
  const int nstage = argc > 2 ? atoi(argv[2]) : 4;
  const int gather = argc > 3 ? atoi(argv[3]) : 0;
  const int issuers = argc > 4 ? atoi(argv[4]) : 1;
  const int tiles = 400;
  const int nrows = 8192, K = 2048, kblocks = K / 64;
  void *buf;
  cudaMalloc(&buf, (size_t)nrows * K * 2);
  cudaMemset(buf, 1, (size_t)nrows * K * 2);
  std::vector<int> perm(nrows);
  for (int i = 0; i < nrows; ++i) perm[i] = i;
  std::shuffle(perm.begin(), perm.end(), std::mt19937(1));
  int *dperm;
  cudaMalloc(&dperm, nrows * 4);
  cudaMemcpy(dperm, perm.data(), nrows * 4, cudaMemcpyHostToDevice);
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap tmap, rmap;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)nrows}, str[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {64, 128}, box1[2] = {64, 1}, es[2] = {1, 1};
  CUresult r1 = ((PFN)fn)(&tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r2 = ((PFN)fn)(&rmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, box1, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r1 || r2) { printf("{\"error\": \"encode %d %d\"}\n", (int)r1, (int)r2); return 1; }
  unsigned long long *cyc;
  cudaMalloc(&cyc, ctas * 8);
  const size_t smem = 1024 + (size_t)issuers * nstage * 16384;
  cudaFuncSetAttribute(k_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int rep = 0; rep < 2; ++rep) k_gather<<<ctas, 32, smem>>>(tmap, rmap, dperm, nrows, kblocks, nstage, tiles, gather, issuers, cyc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_gather<<<ctas, 32, smem>>>(tmap, rmap, dperm, nrows, kblocks, nstage, tiles, gather, issuers, cyc);
  cudaEventRecord(e1);
  cudaError_t e = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = (double)ctas * issuers * tiles * 16384;
  printf("{\"ctas\": %d, \"stages\": %d, \"gather4\": %d, \"issuers\": %d, \"err\": \"%s\", \"us\": %.1f, "
         "\"GBps_total\": %.0f, \"GBps_per_sm\": %.1f}\n", ctas, nstage, gather, issuers, cudaGetErrorString(e),
         ms * 1e3, bytes / ms / 1e6, bytes / ms / 1e6 / ctas);
  return 0;
}
