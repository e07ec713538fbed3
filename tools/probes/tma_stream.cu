// tma_stream.cu — per-SM TMA delivery probe (B200, sm_100a): every CTA streams 2D tiles
// (box 64 x ROWS bf16, 128-B swizzle, one mbarrier per stage) of its own slice of a buffer
// through an NSTAGE smem ring and consumes nothing (a single thread re-arms each stage as soon
// as it lands).  Reports GB/s per SM and aggregate for a given CTA count, ring depth and tile
// rows, from HBM (buffer >> L2) or from L2 (buffer re-read).  Build: nvcc -gencode
// arch=compute_100a,code=sm_100a -O3 -o tma_stream tma_stream.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(256, 1) k_stream(const __grid_constant__ CUtensorMap map, int rows_per_cta,
                                                  int box_rows, int nstage, int kblocks, int reps,
                                                  unsigned long long *cycles, int lane_mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t *ring = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  __shared__ uint64_t bars[32][16];
  const uint32_t tile = box_rows * 128;
  const bool lanes = lane_mode != 0;
  const int nw = lanes ? lane_mode : blockDim.x / 32, w = lanes ? (int)threadIdx.x : (int)threadIdx.x / 32;
  if (lanes ? (threadIdx.x >= (unsigned)lane_mode) : ((threadIdx.x & 31) != 0)) return;
  uint64_t *bar = bars[w];
  ring += (size_t)w * nstage * tile;
  for (int i = 0; i < nstage; ++i)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int row0 = blockIdx.x * rows_per_cta;
  const int ntiles = (rows_per_cta / box_rows) * kblocks;
  const long long total = (long long)ntiles * reps / nw;  // this issuer's share
  uint32_t phase[16] = {0};
  long long t0 = clock64();
  auto issue = [&](long long j, int s) {
    const int t = (int)((j * nw + w) % ntiles);
    const int r = row0 + (t / kblocks) * box_rows, kb = t % kblocks;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(tile) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
        ::"r"(su32(ring + (size_t)s * tile)), "l"((uint64_t)&map), "r"(su32(&bar[s])), "r"(kb * 64), "r"(r)
        : "memory");
  };
  for (int s = 0; s < nstage && s < total; ++s) issue(s, s);
  for (long long j = 0; j < total; ++j) {
    const int s = (int)(j % nstage);
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.b32 %0, 1, 0, P;\n\t}"
                   : "=r"(ok) : "r"(su32(&bar[s])), "r"(phase[s]) : "memory");
    phase[s] ^= 1;
    if (j + nstage < total) issue(j + nstage, s);
  }
  if (w == 0) cycles[blockIdx.x] = clock64() - t0;
}

typedef CUresult (*PFN)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                        const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                        CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char **argv) {
  const int ctas = argc > 1 ? atoi(argv[1]) : 148;
  const int nstage = argc > 2 ? atoi(argv[2]) : 4;
  const int box_rows = argc > 3 ? atoi(argv[3]) : 128;
  const int l2 = argc > 4 ? atoi(argv[4]) : 0;       // 1: small buffer re-read (L2-resident)
  const int issuers = argc > 5 ? atoi(argv[5]) : 1;  // warps issuing TMA, each with its own ring
  const int lane_mode = argc > 6 ? atoi(argv[6]) : 0;  // 1: the issuers are lanes of one warp
  const int K = l2 ? 1024 : 4096, kblocks = K / 64;
  const size_t rows_per_cta = l2 ? 128 : 2048;        // L2 mode: 148 x 128 rows x 2 KB = 38 MB, re-read
  const int reps = l2 ? 64 : 1;
  const size_t rows = (size_t)ctas * rows_per_cta;
  void *buf;
  cudaMalloc(&buf, rows * K * 2);
  cudaMemset(buf, 1, rows * K * 2);
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows}, str[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows}, es[2] = {1, 1};
  ((PFN)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  unsigned long long *cyc;
  cudaMalloc(&cyc, 148 * 8);
  const size_t smem = 1024 + (size_t)issuers * nstage * box_rows * 128;
  cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 2; ++w) k_stream<<<ctas, lane_mode ? 32 : 32 * issuers, smem>>>(map, (int)rows_per_cta, box_rows, nstage, kblocks, reps, cyc, lane_mode ? issuers : 0);
  cudaEventRecord(e0);
  k_stream<<<ctas, lane_mode ? 32 : 32 * issuers, smem>>>(map, (int)rows_per_cta, box_rows, nstage, kblocks, reps, cyc, lane_mode ? issuers : 0);
  cudaEventRecord(e1);
  cudaError_t err = cudaGetLastError();
  if (err == cudaSuccess) err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = (double)rows * K * 2 * reps;
  printf("{\"lane_mode\": %d, \"issuers\": %d, \"ctas\": %d, \"stages\": %d, \"box_rows\": %d, \"in_flight_KB\": %d, \"src\": \"%s\", \"us\": %.1f, "
         "\"GBps_total\": %.0f, \"GBps_per_sm\": %.1f, \"err\": \"%s\"}\n",
         lane_mode, issuers, ctas, nstage, box_rows, nstage * box_rows / 8, l2 ? "L2" : "HBM", ms * 1e3, bytes / (ms * 1e-3) / 1e9,
         bytes / (ms * 1e-3) / 1e9 / ctas, cudaGetErrorString(err));
  return 0;
}
