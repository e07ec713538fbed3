// tg_kernels.cu — GK1-3 "front" kernel of the MoE round trip (AW side, then the
// dispatch exchange), one cooperative launch with grid barriers between phases:
//
//   P1 router   : router logits on tensor cores (bf16 x bf16 -> fp32), top-k
//                 (lowest id on ties), softmax over the k selected, ERT
//                 resolve -> destination key per pair
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
// Router logits on tensor cores.  Work item = (16-token group, K part of
// kKPart = 512 elements); warp w of the block reduces 64 elements of the part
// with mma.sync.m16n8k16 (bf16 in, fp32 accumulate; bf16 products are exact),
// the 8 warp partials are summed in warp order and the part's partial logits go
// to global memory; P2 sums the parts in part order.  The reduction tree of a
// logit depends only on d — never on T, the token's group or its row — so
// routing is deterministic and row-invariant.  Experts in 64-wide groups.
constexpr int kRouterRows = 16;
constexpr int kKPart = 512;

__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ int router_kparts(int d) { return (d + kKPart - 1) / kKPart; }

__device__ void topk_token(const CallArgs &a, const RouteKeys &rk, int t, const float *lg);

// partial logits of group `grp`, K part `kp` -> a.logit_part[(grp * nkp + kp) * 16 * E + row * E + e];
// the last of the nkp items of a group to finish sums the parts in part order and
// runs the top-k of the group's 16 tokens.
__device__ void router_item(const CallArgs &a, const RouteKeys &rk, int grp, int kp, float *part) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int d = a.d, E = a.E, T = a.T;
  const int g = lane >> 2, c = lane & 3;
  const int t0 = grp * kRouterRows;
  const int kb = kp * kKPart + warp * (kKPart / 8);  // this warp's 64 K elements
  const int nkp = router_kparts(d);
  const bool active = kb < d;
  const uint32_t *xr0 = reinterpret_cast<const uint32_t *>(a.x + (size_t)min(t0 + g, T - 1) * d);
  const uint32_t *xr1 = reinterpret_cast<const uint32_t *>(a.x + (size_t)min(t0 + g + 8, T - 1) * d);
  uint32_t af[4][4];
  if (active) {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int o0 = ((kb + 16 * s) >> 1) + c, o1 = o0 + 4;  // uint32 offsets of cols 2c and 2c+8
      af[s][0] = __ldg(xr0 + o0);
      af[s][1] = __ldg(xr1 + o0);
      af[s][2] = __ldg(xr0 + o1);
      af[s][3] = __ldg(xr1 + o1);
    }
  }
  for (int e0 = 0; e0 < E; e0 += 64) {
    float acc[8][4];
#pragma unroll
    for (int n = 0; n < 8; ++n)
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[n][i] = 0.f;
    if (active) {
      uint32_t bf[8][4][2];
#pragma unroll
      for (int n = 0; n < 8; ++n) {
        const uint32_t *wr = reinterpret_cast<const uint32_t *>(a.wg + (size_t)min(e0 + 8 * n + g, E - 1) * d);
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const int o0 = ((kb + 16 * s) >> 1) + c;
          bf[n][s][0] = (e0 + 8 * n < E) ? __ldg(wr + o0) : 0u;
          bf[n][s][1] = (e0 + 8 * n < E) ? __ldg(wr + o0 + 4) : 0u;
        }
      }
#pragma unroll
      for (int s = 0; s < 4; ++s)
#pragma unroll
        for (int n = 0; n < 8; ++n)
          if (e0 + 8 * n < E) mma_bf16_16816(acc[n], af[s], bf[n][s][0], bf[n][s][1]);
    }
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      float *p = part + (warp * kRouterRows) * 64 + 8 * n + 2 * c;
      p[g * 64] = acc[n][0];
      p[g * 64 + 1] = acc[n][1];
      p[(g + 8) * 64] = acc[n][2];
      p[(g + 8) * 64 + 1] = acc[n][3];
    }
    __syncthreads();
    float *dst = a.logit_part + ((size_t)grp * nkp + kp) * kRouterRows * E;
    for (int i = threadIdx.x; i < kRouterRows * 64; i += blockDim.x) {
      const int r = i >> 6, e = e0 + (i & 63);
      if (e < E) {
        float s = part[i];
        for (int ww = 1; ww < 8; ++ww) s += part[ww * kRouterRows * 64 + i];
        dst[r * E + e] = s;
      }
    }
    __syncthreads();
  }
  // ---- last K part of this group: final logits (parts summed in order) + top-k
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int old = atomicAdd(reinterpret_cast<unsigned int *>(a.grp_ctr) + grp, 1u);
    s_last = (old + 1u == (unsigned)nkp);  // counters are zeroed in P2 of every call
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  float *lg = part;  // [16][E]
  const float *src = a.logit_part + (size_t)grp * nkp * kRouterRows * E;
  for (int i = threadIdx.x; i < kRouterRows * E; i += blockDim.x) {
    float s = __ldcg(src + i);
    for (int q = 1; q < nkp; ++q) s += __ldcg(src + (size_t)q * kRouterRows * E + i);
    lg[i] = s;
  }
  __syncthreads();
  for (int rr = warp; rr < kRouterRows; rr += 8)
    if (t0 + rr < T) topk_token(a, rk, t0 + rr, lg + rr * E);
  __syncthreads();
}

// --------------------------------------------------------------------- P2
// Chunk of 256 tokens.  (a) each warp finishes 32 tokens: logits = sum of the K
// parts in part order, top-k by k rounds of warp argmax on (value desc, id asc;
// -0 == +0 ties), slots in ascending expert id (R#4), softmax over the k
// selected (IEEE expf / div), ERT key.  (b) bit t of bm[K][t/32] is set iff
// token t has a pair with key K (at most one per token: its k experts are
// distinct and map to distinct slots); the rank of (t, K) in the chunk is the
// popcount of the bits below t.
__device__ void topk_token(const CallArgs &a, const RouteKeys &rk, int t, const float *lg) {
  const int lane = threadIdx.x & 31;
  const int E = a.E, k = a.k;
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
      const int key = rk.key[sel[j]];
      a.idx[(size_t)t * k + j] = sel[j];
      a.w[(size_t)t * k + j] = __fdiv_rn(z[j], Z);
      a.key[(size_t)t * k + j] = key;
    }
  }
  __syncwarp();
}

__device__ void rank_chunk(const CallArgs &a, int chunk, uint8_t *smraw) {
  const int tid = threadIdx.x, nkeys = a.nkeys, k = a.k;
  uint32_t *bm = reinterpret_cast<uint32_t *>(smraw);  // [nkeys][8]
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
  const int ngroups = (a.T + kRouterRows - 1) / kRouterRows;
  const int nkp = router_kparts(a.d);
  for (int it = blockIdx.x; it < ngroups * nkp; it += gridDim.x)
    router_item(a, rk, it / nkp, it % nkp, reinterpret_cast<float *>(fsm));
  grid_barrier(gbar, a.epoch, kFrontBars, 0, a.err);
  TG_STAMP(1);
  // ---- P2 rank (+ reset of the router group counters for the next call)
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ngroups; i += gridDim.x * blockDim.x) a.grp_ctr[i] = 0;
  const int nchunks = (a.T + kRankBlock - 1) / kRankBlock;
  for (int ch = blockIdx.x; ch < nchunks; ch += gridDim.x) rank_chunk(a, ch, fsm);
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

static size_t front_smem(const CallArgs &a) {
  size_t r = sizeof(float) * std::max(8 * kRouterRows * 64, kRouterRows * a.E);
  size_t b = sizeof(uint32_t) * 8 * a.nkeys;
  size_t e = sizeof(int32_t) * 3 * a.nkeys;
  return std::max(r, std::max(b, e));
}

cudaError_t launch_front(const CallArgs &a, const RouteKeys &rk, int n_sms, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_front, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n_sms);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = front_smem(a);
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = a.pdl ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, k_front, a, rk);
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
