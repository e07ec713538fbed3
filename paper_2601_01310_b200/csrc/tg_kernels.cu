// tg_kernels.cu — GK1-3 "front" kernel of the MoE round trip (AW side, then the
// dispatch exchange), one cooperative launch with grid barriers between phases:
//
//   P1 router   : fp32 router logits, top-k (lowest id on ties), softmax over
//                 the k selected, ERT resolve -> destination key per pair
//                 (§2.1; §4.2; §5.1).
//   P2 rank     : stable rank of every (token, j) pair among this rank's pairs
//                 with the same destination key, in token order (per-chunk
//                 bitmaps + popcounts; §2.2.1 layer-wise batching).
//   P3 exchange : (block 0) per-key totals, all-gather of per-source counts
//                 with every peer over NVLink (one-sided stores + epoch
//                 flag), receive layout on every destination.
//   P4 dispatch : 16-B vector copies of token rows into the destination rank's
//                 receive buffer (peer memory) + origin metadata, then a
//                 per-source data-ready flag (§4.2).
// The combine (GK5) runs at the end of the GEMM kernel (tg_gemm.cu).
#include <algorithm>

#include "tg_internal.h"
#include "tg_ptx.cuh"

namespace tg {

constexpr int kFrontBars = 3;  // grid barriers per front call

#define TG_STAMP(i)                                                                     \
  do {                                                                                  \
    if (a.trace && threadIdx.x == 0 && blockIdx.x == 0)                                 \
      a.trace[a.n_units_max + 148 + (i)] = globaltimer_ns();                            \
  } while (0)

// --------------------------------------------------------------------- P1
// TPB tokens per group; warp w reduces the d-slice [w*d/8, (w+1)*d/8) of
// x . Wg[e] for all TPB tokens and all experts: lanes accumulate their 16-B
// chunks with fp32 FMA (bf16 products are exact in fp32), a fixed xor
// butterfly reduces the 32 lanes and the 8 warp partials are summed in warp
// order.  A token's logit reduction tree depends only on d — never on T, TPB
// or its position — so routing is deterministic and row-invariant.
template <int TPB>
__device__ void router_group(const CallArgs &a, const RouteKeys &rk, int t0, float *part) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int d = a.d, E = a.E, k = a.k, T = a.T;
  const int nch = d >> 3;
  const int cw = nch >> 3;
  const int c_lo = warp * cw, c_hi = c_lo + cw;
  const uint4 *xr[TPB];
#pragma unroll
  for (int t = 0; t < TPB; ++t) xr[t] = reinterpret_cast<const uint4 *>(a.x + (size_t)min(t0 + t, T - 1) * d);
  for (int e0 = 0; e0 < E; e0 += 8) {
    float acc[TPB][8];
#pragma unroll
    for (int t = 0; t < TPB; ++t)
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[t][i] = 0.f;
    for (int c = c_lo + lane; c < c_hi; c += 32) {
      uint4 wv[8];
#pragma unroll
      for (int i = 0; i < 8; ++i)
        wv[i] = (e0 + i < E) ? __ldg(reinterpret_cast<const uint4 *>(a.wg + (size_t)(e0 + i) * d) + c)
                             : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int t = 0; t < TPB; ++t) {
        uint4 xv = __ldg(xr[t] + c);
        const __nv_bfloat162 *xp = reinterpret_cast<const __nv_bfloat162 *>(&xv);
        float2 xf[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) xf[q] = __bfloat1622float2(xp[q]);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const __nv_bfloat162 *wp = reinterpret_cast<const __nv_bfloat162 *>(&wv[i]);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            float2 wf = __bfloat1622float2(wp[q]);
            acc[t][i] = __fmaf_rn(xf[q].x, wf.x, acc[t][i]);
            acc[t][i] = __fmaf_rn(xf[q].y, wf.y, acc[t][i]);
          }
        }
      }
    }
#pragma unroll
    for (int t = 0; t < TPB; ++t)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float v = acc[t][i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0 && e0 + i < E) part[(warp * TPB + t) * E + e0 + i] = v;
      }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < TPB * E; i += blockDim.x) {
    float s = part[i];
    for (int ww = 1; ww < 8; ++ww) s += part[ww * TPB * E + i];
    part[i] = s;  // logit of token t0 + i / E, expert i % E
  }
  __syncthreads();
  const int t = t0 + warp;
  if (warp < TPB && t < T) {
    const float *lg = part + warp * E;
    // top-k: k rounds of warp argmax on (value desc, id asc); -0 == +0 ties
    uint32_t taken = 0;  // bit i: expert lane + 32 i already selected
    int sel[kMaxK];
    float sv[kMaxK];
    for (int r = 0; r < k; ++r) {
      float bv = -INFINITY;
      int bi = 0x7fffffff;
      for (int i = 0; lane + 32 * i < E; ++i) {
        int e = lane + 32 * i;
        if (taken & (1u << i)) continue;
        float v = lg[e];
        if (v > bv || (v == bv && e < bi)) { bv = v; bi = e; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
      }
      sel[r] = bi;
      sv[r] = bv;
      if ((bi & 31) == lane) taken |= 1u << (bi >> 5);
    }
    if (lane == 0) {
      // slots in ascending expert id (R#4)
      for (int q = 1; q < k; ++q) {
        int ve = sel[q];
        float vv = sv[q];
        int b = q - 1;
        while (b >= 0 && sel[b] > ve) { sel[b + 1] = sel[b]; sv[b + 1] = sv[b]; --b; }
        sel[b + 1] = ve;
        sv[b + 1] = vv;
      }
      float m = sv[0];
      for (int j = 1; j < k; ++j) m = fmaxf(m, sv[j]);
      float z[kMaxK], Z = 0.f;
      for (int j = 0; j < k; ++j) { z[j] = expf(sv[j] - m); Z = Z + z[j]; }
      for (int j = 0; j < k; ++j) {
        a.idx[(size_t)t * k + j] = sel[j];
        a.w[(size_t)t * k + j] = __fdiv_rn(z[j], Z);
        a.key[(size_t)t * k + j] = rk.key[sel[j]];
      }
    }
  }
  __syncthreads();  // part[] is reused by the next group
}

// --------------------------------------------------------------------- P2
// Chunk of 256 tokens: bit t of bm[K][t/32] is set iff token t has a pair with
// key K (at most one per token: its k experts are distinct and map to distinct
// slots).  The rank of (t, K) in the chunk is the popcount of the bits below t.
__device__ void rank_chunk(const CallArgs &a, int chunk, uint32_t *bm) {
  const int tid = threadIdx.x, nkeys = a.nkeys, k = a.k;
  const int t = chunk * kRankBlock + tid;
  for (int i = tid; i < nkeys * 8; i += blockDim.x) bm[i] = 0;
  __syncthreads();
  int K[kMaxK];
  for (int j = 0; j < k; ++j) {
    K[j] = (t < a.T) ? __ldcg(a.key + (size_t)t * k + j) : -1;
    if (K[j] >= 0) atomicOr(&bm[K[j] * 8 + (tid >> 5)], 1u << (tid & 31));
  }
  __syncthreads();
  for (int j = 0; j < k; ++j) {
    if (K[j] < 0) continue;
    const uint32_t *row = bm + K[j] * 8;
    int r = __popc(row[tid >> 5] & ((1u << (tid & 31)) - 1u));
    for (int wd = 0; wd < (tid >> 5); ++wd) r += __popc(row[wd]);
    a.lrank[(size_t)t * k + j] = r;
  }
  for (int Kk = tid; Kk < nkeys; Kk += blockDim.x) {
    int c = 0;
#pragma unroll
    for (int wd = 0; wd < 8; ++wd) c += __popc(bm[Kk * 8 + wd]);
    a.bcnt[(size_t)chunk * nkeys + Kk] = c;
  }
  __syncthreads();
}

// --------------------------------------------------------------------- P3
__device__ void exchange_counts(const CallArgs &a, int nchunks, int32_t *sm) {
  const int tid = threadIdx.x, nkeys = a.nkeys;
  int32_t *tot = sm;              // [nkeys] this rank's rows per key
  int32_t *gsum = sm + nkeys;     // [nkeys] rows per key over all sources
  int32_t *below = gsum + nkeys;  // [nkeys] rows per key from lower sources
  const int par = a.epoch & 1;
  const bool sys = a.world > 1;
  for (int K = tid; K < nkeys; K += blockDim.x) {
    int run = 0;
    for (int b = 0; b < nchunks; ++b) {
      int c = __ldcg(a.bcnt + (size_t)b * nkeys + K);
      a.bcnt[(size_t)b * nkeys + K] = run;  // exclusive chunk base
      run += c;
    }
    tot[K] = run;
    a.stats[K] += run;
  }
  __syncthreads();
  // all-gather: my totals -> cnt_all[par][rank][*] on every peer, then release flags
  for (int q = 0; q < a.world; ++q) {
    int32_t *dst = reinterpret_cast<int32_t *>(a.sym[q] + a.L.cnt_all) + ((size_t)par * a.world + a.rank) * nkeys;
    for (int K = tid; K < nkeys; K += blockDim.x) dst[K] = tot[K];
  }
  __syncthreads();
  if (tid < a.world) {
    fence_scope(sys);
    uint32_t *fl = reinterpret_cast<uint32_t *>(a.sym[tid] + a.L.flags) + FLAG_CNT * kMaxWorld + a.rank;
    st_release(fl, a.epoch, sys);
    const uint32_t *mine = reinterpret_cast<const uint32_t *>(a.sym[a.rank] + a.L.flags) + FLAG_CNT * kMaxWorld + tid;
    wait_flag_ge_s(mine, a.epoch, sys, a.err, 0x2001);
  }
  __syncthreads();
  const int32_t *A = reinterpret_cast<const int32_t *>(a.sym[a.rank] + a.L.cnt_all) + (size_t)par * a.world * nkeys;
  for (int K = tid; K < nkeys; K += blockDim.x) {
    int g = 0, bl = 0;
    for (int src = 0; src < a.world; ++src) {
      int c = __ldcg(A + (size_t)src * nkeys + K);
      if (src < a.rank) bl += c;
      g += c;
    }
    gsum[K] = g;
    below[K] = bl;
    a.gcounts[K] = g;
  }
  __syncthreads();
  // dbase[K] = rows of lower slots on that rank (all sources) + rows of lower sources
  for (int K = tid; K < nkeys; K += blockDim.x) {
    const int q = K / a.S_max, s = K % a.S_max;
    int off = 0;
    for (int s2 = 0; s2 < s; ++s2) off += gsum[q * a.S_max + s2];
    a.dbase[K] = off + below[K];
  }
  if (tid < a.world) {
    int to_me = 0, to_q = 0;
    for (int s = 0; s < a.S_max; ++s) {
      to_me += __ldcg(A + (size_t)tid * nkeys + a.rank * a.S_max + s);
      to_q += tot[tid * a.S_max + s];
    }
    a.need_src[tid] = to_me > 0;
    a.sent_to[tid] = to_q > 0;
  }
  for (int s = tid; s < a.S_loc; s += blockDim.x) a.slot_rows[s] = gsum[a.rank * a.S_max + s];
}

// --------------------------------------------------------------------- P4
// Warp copy of one row of nch 16-B chunks: all loads of a lane before its stores.
__device__ __forceinline__ void copy_row(uint4 *__restrict__ dst, const uint4 *__restrict__ src, int nch, int lane) {
  int c = lane;
  for (; c + 96 < nch; c += 128) {
    uint4 v0 = __ldg(src + c), v1 = __ldg(src + c + 32), v2 = __ldg(src + c + 64), v3 = __ldg(src + c + 96);
    dst[c] = v0; dst[c + 32] = v1; dst[c + 64] = v2; dst[c + 96] = v3;
  }
  for (; c < nch; c += 32) dst[c] = __ldg(src + c);
}

template <int TPB>
__global__ void __launch_bounds__(256, 1) k_front(const __grid_constant__ CallArgs a,
                                                  const __grid_constant__ RouteKeys rk) {
  extern __shared__ __align__(16) uint8_t fsm[];
  unsigned long long *gbar = reinterpret_cast<unsigned long long *>(a.sync + 8);
  // PDL: everything below reads/writes state of the previous call's GEMM kernel
  asm volatile("griddepcontrol.wait;" ::: "memory");
  TG_STAMP(0);
  // ---- P1 router (+ reset of the GEMM counters of this call)
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n_ctr_max; i += gridDim.x * blockDim.x) a.ctr[i] = 0;
  if (blockIdx.x == 0 && threadIdx.x < 4) a.sync[threadIdx.x] = 0;
  const int ngroups = (a.T + TPB - 1) / TPB;
  for (int g = blockIdx.x; g < ngroups; g += gridDim.x)
    router_group<TPB>(a, rk, g * TPB, reinterpret_cast<float *>(fsm));
  grid_barrier(gbar, a.epoch, kFrontBars, 0, a.err);
  TG_STAMP(1);
  // ---- P2 rank
  const int nchunks = (a.T + kRankBlock - 1) / kRankBlock;
  for (int ch = blockIdx.x; ch < nchunks; ch += gridDim.x) rank_chunk(a, ch, reinterpret_cast<uint32_t *>(fsm));
  grid_barrier(gbar, a.epoch, kFrontBars, 1, a.err);
  TG_STAMP(2);
  // ---- P3 counts exchange + layout (block 0)
  if (blockIdx.x == 0) exchange_counts(a, nchunks, reinterpret_cast<int32_t *>(fsm));
  grid_barrier(gbar, a.epoch, kFrontBars, 2, a.err);
  TG_STAMP(3);
  // the GEMM kernel may launch now: its prologue overlaps the dispatch
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // ---- P4 dispatch: one warp per (token, j) pair
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int k = a.k, nch = a.d >> 3;
  const int npairs = a.T * k;
  const int nsh = (a.Fsh > 0) ? a.T : 0;
  for (int p = warp; p < npairs + nsh; p += nwarps) {
    if (p < npairs) {
      const int t = p / k;
      const int K = __ldcg(a.key + p);
      const int q = K / a.S_max;
      const int pos =
          __ldcg(a.dbase + K) + __ldcg(a.bcnt + (size_t)(t / kRankBlock) * a.nkeys + K) + __ldcg(a.lrank + p);
      const uint4 *src = reinterpret_cast<const uint4 *>(a.x + (size_t)t * a.d);
      uint4 *dst = reinterpret_cast<uint4 *>(a.sym[q] + a.L.recv) + (size_t)pos * nch;
      copy_row(dst, src, nch, lane);
      if (lane == 0) {
        int2 *meta = reinterpret_cast<int2 *>(a.sym[q] + a.L.meta);
        meta[pos] = make_int2(a.rank, p);
        a.dst_pos[p] = pos;
      }
    } else {
      const int t = p - npairs;
      const uint4 *src = reinterpret_cast<const uint4 *>(a.x + (size_t)t * a.d);
      uint4 *dst = reinterpret_cast<uint4 *>(a.sym[a.rank] + a.L.recv) + (size_t)(a.R_sh0 + t) * nch;
      copy_row(dst, src, nch, lane);
    }
  }
  // data-ready flags: the last block to finish releases one flag per destination
  const bool sys = a.world > 1;
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_scope(sys);
    s_last = (atomicAdd(&a.sync[3], 1) == (int)gridDim.x - 1);
  }
  __syncthreads();
  if (s_last && threadIdx.x < a.world) {
    fence_scope(sys);
    uint32_t *fl = reinterpret_cast<uint32_t *>(a.sym[threadIdx.x] + a.L.flags) + FLAG_DATA * kMaxWorld + a.rank;
    st_release(fl, a.epoch, sys);
  }
  TG_STAMP(4);
}

// Tokens per router group: the smallest power of two that needs one round of
// groups over the grid (latency-bound), capped at 8 and TPB * E <= 1024.
static int router_tpb(int T, int E, int nblk) {
  int tpb = 1;
  while (tpb < 8 && (T + tpb - 1) / tpb > nblk && 2 * tpb * E <= 1024) tpb <<= 1;
  return tpb;
}

static size_t front_smem(const CallArgs &a, int tpb) {
  size_t r = sizeof(float) * 8 * tpb * a.E;
  size_t b = sizeof(uint32_t) * 8 * a.nkeys;
  size_t e = sizeof(int32_t) * 3 * a.nkeys;
  return std::max(r, std::max(b, e));
}

template <int TPB>
static cudaError_t launch_front_t(const CallArgs &a, const RouteKeys &rk, int nblk, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_front<TPB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nblk);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = front_smem(a, TPB);
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = a.pdl ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, k_front<TPB>, a, rk);
}

cudaError_t launch_front(const CallArgs &a, const RouteKeys &rk, int n_sms, cudaStream_t s) {
  const int nblk = n_sms;
  switch (router_tpb(a.T, a.E, nblk)) {
    case 8: return launch_front_t<8>(a, rk, nblk, s);
    case 4: return launch_front_t<4>(a, rk, nblk, s);
    case 2: return launch_front_t<2>(a, rk, nblk, s);
    default: return launch_front_t<1>(a, rk, nblk, s);
  }
}

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
