// router_item.cu — cost of one router item (32 tokens x one 512-wide K part, E experts) on one SM,
// as in tg_front.cuh router_compute: 8 warps, mma.sync.m16n8k16 bf16 -> fp32, ldmatrix fragments,
// x tile and Wg slice resident in shared memory (rows padded by 16 B).  Variants:
//   0: warps own n8 expert tiles, 4 interleaved accumulator sets (the library's prefill shape, E=60)
//   1: as 0 with the step loop fully unrolled
//   2: warps own (m16, 2 n8) pairs: A fragments loaded by 4 warps instead of 8
// Prints cycles per item (median over repeats, clock64 inside one CTA).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o router_item router_item.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2(uint32_t &r0, uint32_t &r1, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(addr));
}
__device__ __forceinline__ void mma(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
               "{%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

constexpr int KP = 512, LDW = KP / 2 + 4;  // words per padded row

template <int V>
__device__ void item(const uint32_t *xb, const uint32_t *wg, float *out, int steps) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (V == 0 || V == 1) {
    const int tile = warp;
    const uint32_t xa = su32(xb + (lane & 15) * LDW) + (lane >> 4) * 16;
    const uint32_t wa = su32(wg + (tile * 8 + (lane & 7)) * LDW) + ((lane >> 3) & 1) * 16;
    const uint32_t mstr = 16 * LDW * 4;
    float acc[4][2][4] = {};
#pragma unroll(V == 1 ? 8 : 1)
    for (int st = 0; st < 8; ++st) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t off = (uint32_t)(q * 8 + st) * 32;
        uint32_t a0[4], a1[4], b0, b1;
        ldsm_x4(a0, xa + off);
        ldsm_x4(a1, xa + mstr + off);
        ldsm_x2(b0, b1, wa + off);
        mma(acc[q][0], a0, b0, b1);
        mma(acc[q][1], a1, b0, b1);
      }
    }
    double v = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int i = 0; i < 4; ++i) v += (double)acc[q][m][i];
    out[threadIdx.x] = (float)v;
  } else {
    // warp -> m16 block (warp & 1), n8 tiles 2 * (warp >> 1) .. + 1
    const int mb = warp & 1, t0 = 2 * (warp >> 1);
    const uint32_t xa = su32(xb + (16 * mb + (lane & 15)) * LDW) + (lane >> 4) * 16;
    const uint32_t wa0 = su32(wg + (t0 * 8 + (lane & 7)) * LDW) + ((lane >> 3) & 1) * 16;
    const uint32_t wa1 = wa0 + 8 * LDW * 4;
    float acc[4][2][4] = {};
#pragma unroll 1
    for (int st = 0; st < 8; ++st) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t off = (uint32_t)(q * 8 + st) * 32;
        uint32_t a[4], b0, b1, c0, c1;
        ldsm_x4(a, xa + off);
        ldsm_x2(b0, b1, wa0 + off);
        ldsm_x2(c0, c1, wa1 + off);
        mma(acc[q][0], a, b0, b1);
        mma(acc[q][1], a, c0, c1);
      }
    }
    double v = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int i = 0; i < 4; ++i) v += (double)acc[q][m][i];
    out[threadIdx.x] = (float)v;
  }
}

template <int V>
__global__ void __launch_bounds__(256, 1) k(float *out, long long *cyc, int reps) {
  extern __shared__ uint32_t sm[];
  uint32_t *xb = sm, *wg = sm + 32 * LDW;
  for (int i = threadIdx.x; i < (32 + 64) * LDW; i += blockDim.x) sm[i] = 0x3f803f80u ^ (i * 2654435761u & 0x00ff00ffu);
  __syncthreads();
  for (int r = 0; r < reps; ++r) {
    __syncthreads();
    long long t0 = clock64();
    item<V>(xb, wg, out + blockIdx.x * 256, 32);
    __syncthreads();
    if (threadIdx.x == 0) cyc[r] = clock64() - t0;
  }
}

int main() {
  float *out;
  long long *cyc, h[64];
  cudaMalloc(&out, 256 * 4 * 148);
  cudaMalloc(&cyc, 64 * 8);
  const size_t smem = (32 + 64) * LDW * 4;
  void (*ks[3])(float *, long long *, int) = {k<0>, k<1>, k<2>};
  for (int v = 0; v < 3; ++v) {
    cudaFuncSetAttribute(ks[v], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    ks[v]<<<1, 256, smem>>>(out, cyc, 64);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
    long long mn = h[8];
    for (int i = 8; i < 64; ++i) mn = h[i] < mn ? h[i] : mn;
    printf("{\"variant\": %d, \"err\": \"%s\", \"cycles_per_item_min\": %lld, \"cycles_rep20\": %lld}\n", v,
           cudaGetErrorString(e), mn, h[20]);
  }
  return 0;
}
