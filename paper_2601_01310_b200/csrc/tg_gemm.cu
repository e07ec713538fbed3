// tg_gemm.cu — GK4: persistent grouped expert-FFN kernel for sm_100a.
//
// One launch runs every expert FFN this rank serves as EW (§2.2.1: "an
// EW aggregates requests for the same layer and expert, and executes them as
// a single large batch"), in two dependent phases over a device-built work
// list (GK2):
//   GEMM1 units:  [a1 | a3] = W1|W3 (128 x d tile)  .  X^T (d x n tokens)
//                 h = bf16(silu(a1) * a3)  -> H          (SwiGLU, R#6/R#7)
//   GEMM2 units:  y = W2 (128 x F tile) . H^T, fixed split-K for long F with an
//                 in-order reduction; y = bf16(.) stored straight into the
//                 source AW's combine buffer slot [t][j] (NVLink store when the
//                 source is a peer): the combine exchange fused in the epilogue.
// Swap-AB: the weight tile fills UMMA M = 128, the (few) tokens of a slot are
// UMMA N (16..128), so decode batches waste no tensor-core rows.
//
// Warp roles (256 threads, 1 CTA / SM, persistent over an atomic work queue):
//   w0  TMA producer: fetches unit ids, streams W and X/H tiles (128-B swizzle)
//       into a 4-stage smem ring (mbarrier full/empty, complete_tx bytes).
//   w1  MMA issuer: one thread issues tcgen05.mma (bf16 -> fp32 in TMEM), two
//       TMEM accumulator buffers so the epilogue overlaps the next unit.
//   w2  TMEM allocator.      w4-7  epilogue: tcgen05.ld -> regs -> global.
#include "tg_internal.h"
#include "tg_ptx.cuh"

namespace tg {

struct GemmShared {
  uint64_t full[kStages];
  uint64_t empty[kStages];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint64_t sfull[kSchedDepth];
  uint64_t sempty[kSchedDepth];
  int sched[kSchedDepth];
  uint32_t tmem_base;
  int red_last;
};

__device__ __forceinline__ float silu_f(float a) { return __fdiv_rn(a, 1.0f + expf(-a)); }

__device__ __forceinline__ int box_index(int nrows) { return ((nrows + 15) >> 4) - 1; }

__global__ void __launch_bounds__(kGemmThreads, 1)
    k_gemm(const __grid_constant__ TmaMaps maps, const __grid_constant__ CallArgs a) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned stage ring (128-B swizzle atoms), bookkeeping after it.
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t *ring = smem_raw + ((1024 - (raw_addr & 1023)) & 1023);
  GemmShared *S = reinterpret_cast<GemmShared *>(ring + kStages * kStageBytes);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int *err = a.err;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) { mbar_init(&S->full[i], 1); mbar_init(&S->empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&S->tfull[i], 1); mbar_init(&S->tempty[i], 128); }
    for (int i = 0; i < kSchedDepth; ++i) { mbar_init(&S->sfull[i], 1); mbar_init(&S->sempty[i], 5); }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&maps.w1);
    tma_prefetch_desc(&maps.w3);
    tma_prefetch_desc(&maps.w2);
  }
  if (warp == 2) {
    tmem_alloc(&S->tmem_base, kTmemCols);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = S->tmem_base;
  const int n_units = *reinterpret_cast<volatile int *>(a.n_units);

  if (warp == 0) {
    if (lane == 0) {
      // ===================== TMA producer =====================
      const uint64_t pol_w = policy_evict_first();   // weights: streamed once
      const uint64_t pol_x = policy_evict_last();    // token tiles: re-read by every weight tile
      // Dispatched rows from peers must have landed (release/acquire on
      // per-source epoch flags), then order them before async-proxy reads.
      for (int src = 0; src < a.world; ++src) {
        if (a.need_src[src]) {
          const uint32_t *fl = reinterpret_cast<const uint32_t *>(a.sym[a.rank] + a.L.flags) +
                               FLAG_DATA * kMaxWorld + src;
          wait_flag_ge(fl, a.epoch, err, 0x4001);
        }
      }
      fence_proxy_async_global();
      int stage = 0;
      uint32_t phase = 0;
      for (int it = 0;; ++it) {
        int u = atomicAdd(&a.sync[1], 1);
        if (u >= n_units) u = -1;
        const int r = it % kSchedDepth;
        mbar_wait(&S->sempty[r], ((it / kSchedDepth) & 1) ^ 1, err);
        S->sched[r] = u;
        mbar_arrive(&S->sfull[r]);
        if (u < 0) break;
        const Unit U = a.units[u];
        const bool g1 = (U.kind == U_G1 || U.kind == U_G1_SH);
        const bool sh = (U.kind == U_G1_SH || U.kind == U_G2_SH);
        if (!g1) {
          // all GEMM1 tiles of this (slot, n-tile) have written H
          wait_ctr_ge(a.ctr + U.dep, U.dep_target, err, 0x4002);
          fence_proxy_async_global();
        }
        const int bi = box_index(U.nrows);
        const uint32_t bbytes = (uint32_t)(bi + 1) * 16 * BK * 2;
        const CUtensorMap *mA0 = g1 ? (sh ? &maps.w1s : &maps.w1) : (sh ? &maps.w2s : &maps.w2);
        const CUtensorMap *mA1 = sh ? &maps.w3s : &maps.w3;
        const CUtensorMap *mB = g1 ? &maps.x[bi] : (sh ? &maps.hs[bi] : &maps.h[bi]);
        const int rowA = g1 ? U.slot * (sh ? a.Fsh : a.F) + U.m0 : U.slot * a.d + U.m0;
        const int rowB = (!g1 && sh) ? U.n0 - a.R_sh0 : U.n0;
        for (int kb = U.kb0; kb < U.kb1; ++kb) {
          mbar_wait(&S->empty[stage], phase ^ 1, err);
          uint8_t *st = ring + stage * kStageBytes;
          mbar_arrive_expect_tx(&S->full[stage], (g1 ? 2u : 1u) * kTileBytes + bbytes);
          tma_load_2d(st, mA0, &S->full[stage], kb * BK, rowA, pol_w);
          if (g1) tma_load_2d(st + kTileBytes, mA1, &S->full[stage], kb * BK, rowA, pol_w);
          tma_load_2d(st + 2 * kTileBytes, mB, &S->full[stage], kb * BK, rowB, pol_x);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ===================== MMA issuer =====================
      int stage = 0;
      uint32_t phase = 0;
      for (int it = 0;; ++it) {
        const int r = it % kSchedDepth;
        mbar_wait(&S->sfull[r], (it / kSchedDepth) & 1, err);
        const int u = S->sched[r];
        mbar_arrive(&S->sempty[r]);
        if (u < 0) break;
        const Unit U = a.units[u];
        const bool g1 = (U.kind == U_G1 || U.kind == U_G1_SH);
        const int buf = it & 1;
        mbar_wait(&S->tempty[buf], ((it >> 1) & 1) ^ 1, err);
        tc_fence_after();
        const int nb = (box_index(U.nrows) + 1) * 16;
        const uint32_t idesc = idesc_bf16_f32(BM, nb);
        const uint32_t d0 = tmem + buf * 256, d1 = tmem + buf * 256 + 128;
        for (int kb = U.kb0; kb < U.kb1; ++kb) {
          mbar_wait(&S->full[stage], phase, err);
          tc_fence_after();
          const uint32_t sa = smem_u32(ring + stage * kStageBytes);
          const uint64_t dA0 = desc_sw128_kmajor(sa);
          const uint64_t dA1 = desc_sw128_kmajor(sa + kTileBytes);
          const uint64_t dB = desc_sw128_kmajor(sa + 2 * kTileBytes);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint32_t acc = (kb > U.kb0 || kk > 0) ? 1u : 0u;
            // advance 16 K-elements = 32 B inside the swizzle row (>>4 units)
            umma_bf16_ss(d0, dA0 + 2 * kk, dB + 2 * kk, idesc, acc);
            if (g1) umma_bf16_ss(d1, dA1 + 2 * kk, dB + 2 * kk, idesc, acc);
          }
          umma_commit(&S->empty[stage]);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        umma_commit(&S->tfull[buf]);
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue (128 threads) =====================
    const int q = warp & 3;            // TMEM lane quarter of this warp
    const int et = threadIdx.x - 128;  // 0..127
    for (int it = 0;; ++it) {
      const int r = it % kSchedDepth;
      mbar_wait(&S->sfull[r], (it / kSchedDepth) & 1, err);
      const int u = S->sched[r];
      __syncwarp();
      if (lane == 0) mbar_arrive(&S->sempty[r]);
      if (u < 0) break;
      const Unit U = a.units[u];
      const bool g1 = (U.kind == U_G1 || U.kind == U_G1_SH);
      const bool sh = (U.kind == U_G1_SH || U.kind == U_G2_SH);
      const int buf = it & 1;
      mbar_wait(&S->tfull[buf], (it >> 1) & 1, err);
      tc_fence_after();
      const int m = U.m0 + q * 32 + lane;  // weight row handled by this thread
      const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + buf * 256;
      if (g1) {
        const int Fw = sh ? a.Fsh : a.F;
        bf16 *Hout = sh ? a.Hs : a.H;
        const int row0 = sh ? U.n0 - a.R_sh0 : U.n0;
        for (int c0 = 0; c0 < U.nrows; c0 += 32) {
          uint32_t r1[32], r3[32];
          tmem_ld_32x32b_x32(tbase + c0, r1);
          tmem_ld_32x32b_x32(tbase + 128 + c0, r3);
          tmem_ld_wait();
          if (m < Fw) {
#pragma unroll
            for (int n = 0; n < 32; ++n) {
              if (c0 + n < U.nrows) {
                const float a1 = __uint_as_float(r1[n]), a3 = __uint_as_float(r3[n]);
                const float h = __fmul_rn(silu_f(a1), a3);
                Hout[(size_t)(row0 + c0 + n) * Fw + m] = __float2bfloat16_rn(h);
              }
            }
          }
        }
        tc_fence_before();
        mbar_arrive(&S->tempty[buf]);
        // publish H rows: generic -> async proxy, then release the group counter
        fence_proxy_async_global();
        named_bar_sync(1, 128);
        if (et == 0) {
          __threadfence();
          atomicAdd(a.ctr + U.dep, 1);
        }
      } else {
        const bool split = (U.nsplit > 1);
        const int2 *meta = reinterpret_cast<const int2 *>(a.sym[a.rank] + a.L.meta);
        for (int c0 = 0; c0 < U.nrows; c0 += 32) {
          uint32_t r1[32];
          tmem_ld_32x32b_x32(tbase + c0, r1);
          tmem_ld_wait();
          if (m < a.d) {
#pragma unroll
            for (int n = 0; n < 32; ++n) {
              if (c0 + n < U.nrows) {
                const int row = U.n0 + c0 + n;
                const float v = __uint_as_float(r1[n]);
                if (split) {
                  a.ws[((size_t)U.split * a.R_cap + row) * a.d + m] = v;
                } else if (sh) {
                  a.ysh[(size_t)(row - a.R_sh0) * a.d + m] = __float2bfloat16_rn(v);
                } else {
                  const int2 o = meta[row];
                  bf16 *yb = reinterpret_cast<bf16 *>(a.sym[o.x] + a.L.ybuf);
                  yb[(size_t)o.y * a.d + m] = __float2bfloat16_rn(v);
                }
              }
            }
          }
        }
        tc_fence_before();
        mbar_arrive(&S->tempty[buf]);
        if (split) {
          // fixed-order split-K reduction by the last split to finish
          __threadfence();
          named_bar_sync(1, 128);
          if (et == 0) S->red_last = (atomicAdd(a.ctr + U.red, 1) == U.nsplit - 1);
          named_bar_sync(1, 128);
          if (S->red_last) {
            __threadfence();
            if (m < a.d) {
              for (int n = 0; n < U.nrows; ++n) {
                const int row = U.n0 + n;
                float acc = __ldcg(a.ws + (size_t)row * a.d + m);
                for (int sp = 1; sp < U.nsplit; ++sp)
                  acc = __fadd_rn(acc, __ldcg(a.ws + ((size_t)sp * a.R_cap + row) * a.d + m));
                const int2 o = meta[row];
                bf16 *yb = reinterpret_cast<bf16 *>(a.sym[o.x] + a.L.ybuf);
                yb[(size_t)o.y * a.d + m] = __float2bfloat16_rn(acc);
              }
            }
          }
          named_bar_sync(1, 128);
        }
      }
    }
    // all units of this CTA done: the last CTA releases the combine flags
    __threadfence_system();
    named_bar_sync(1, 128);
    if (et == 0) {
      if (atomicAdd(&a.sync[2], 1) == (int)gridDim.x - 1) {
        __threadfence_system();
        for (int src = 0; src < a.world; ++src) {
          uint32_t *fl = reinterpret_cast<uint32_t *>(a.sym[src] + a.L.flags) + FLAG_COMB * kMaxWorld + a.rank;
          st_release_sys(fl, a.epoch);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, kTmemCols);
  }
}

size_t gemm_smem_bytes() { return 1024 + (size_t)kStages * kStageBytes + sizeof(GemmShared); }

cudaError_t gemm_configure() {
  return cudaFuncSetAttribute(k_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gemm_smem_bytes());
}

cudaError_t launch_gemm(const CallArgs &a, const TmaMaps &maps, int n_sms, cudaStream_t s) {
  k_gemm<<<n_sms, kGemmThreads, gemm_smem_bytes(), s>>>(maps, a);
  return cudaGetLastError();
}

}  // namespace tg
