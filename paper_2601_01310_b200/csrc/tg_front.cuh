// tg_front.cuh — the AW-side front of the MoE round trip (GK1-GK3 of SURVEY
// §8), as device phases of the fused layer kernel k_layer (tg_gemm.cu):
//
//   P1 router   : router logits on tensor cores (bf16 x bf16 -> fp32), K split
//                 in parts fixed by (d, E), partial logits to global memory
//   P1b top-k   : per 32-token group: parts summed in order, top-k (lowest id
//                 on ties), softmax over the k selected, ERT resolve ->
//                 destination key per pair
//                 (§2.1; §4.2; §5.1).
//   P2 rank     : stable rank of every (token, j) pair among this rank's pairs
//                 with the same destination key, in token order (per-chunk
//                 bitmaps + popcounts; §2.2.1 layer-wise batching).
//   P3 exchange : per-key totals, all-gather of per-source counts with every
//                 live peer over NVLink (one-sided stores + epoch flag),
//                 receive layout on every destination.
//   P4 dispatch : 16-B vector copies of token rows into the destination rank's
//                 receive buffer (peer memory) + origin metadata, then a
//                 per-source data-ready flag (§4.2).  All warps of
//                 k_layer, right after P3; the TMA producer then streams the
//                 first weight tiles while the peers' rows are still landing.
#pragma once
#include <algorithm>

#include "tg_internal.h"
#include "tg_ptx.cuh"

namespace tg {


#define TG_STAMP(i)                                                                     \
  do {                                                                                  \
    if (a.trace && threadIdx.x == 0 && blockIdx.x == 0)                                 \
      a.trace[a.n_units_max + 148 + (i)] = globaltimer_ns();                            \
  } while (0)

#define TG_STAMP_ANY(i)                                                                 \
  do {                                                                                  \
    if (a.trace && threadIdx.x == 0) a.trace[a.n_units_max + 148 + (i)] = globaltimer_ns(); \
  } while (0)

// --------------------------------------------------------------------- P1
// Router logits on tensor cores.  The K dimension is cut into parts of KP
// elements (a function of d and E only); block b owns part kp = b % nkp for
// the whole phase and stages the Wg slice [E][KP] in shared memory once (rows
// padded by 16 B: conflict-free fragment loads).  Work item = (32-token group,
// part): the x tile [32][KP] is staged with coalesced 16-B loads, warp w
// reduces KP/8 elements with mma.sync.m16n8k16 (bf16 in, fp32 accumulate;
// bf16 products are exact), k16 steps in order, the 8 warp partials are summed
// in warp order and written to global memory; the last part of a group to
// arrive sums the parts in part order and runs the top-k.  The reduction tree
// of a logit depends only on (d, E) — never on T, the token's group or its row
// — so routing is deterministic and row-invariant.
constexpr int kRouterRows = 32;

__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__host__ __device__ __forceinline__ int router_kpart(int d, int E) {
  int kp = E <= 96 ? 512 : (E <= 192 ? 256 : 128);
  while (kp > 64 && d % kp) kp >>= 1;  // d % 64 == 0, so 64 always divides d
  return kp;
}
__host__ __device__ __forceinline__ int router_nkp(int d, int E) { return (d + router_kpart(d, E) - 1) / router_kpart(d, E); }
__host__ __device__ __forceinline__ int router_epad(int E) { return (E + 63) / 64 * 64; }


struct RouterSmem {
  uint32_t *wg;   // [Epad][KP/2 + 4] words
  uint32_t *xt;   // [32][KP/2 + 4] words
  float *part;    // [8][32][64]
  int ldw;        // row stride in words
};

// Batched copy of rows of 16-B chunks into padded smem rows: 16 loads in flight per
// thread before the stores (these loops are latency-bound, not bandwidth-bound).
template <typename RowPtr, typename DstRow>
__device__ __forceinline__ void stage_rows(int nrows, int cpr, RowPtr row, DstRow drow) {
  const int total = nrows * cpr;
  const int lc = __ffs(cpr) - 1;  // cpr = KP / 8 is a power of two
#pragma unroll 1
  for (int i0 = threadIdx.x; i0 < total; i0 += 16 * blockDim.x) {
    uint4 v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int i = i0 + u * blockDim.x;
      const uint4 *p = (i < total) ? row(i >> lc) : nullptr;
      v[u] = p ? __ldg(p + (i & (cpr - 1))) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int i = i0 + u * blockDim.x;
      if (i < total) *reinterpret_cast<uint4 *>(drow(i >> lc) + (i & (cpr - 1)) * 4) = v[u];
    }
  }
}

__device__ void router_item(const CallArgs &a, const RouterSmem &R, int grp, int kp, bool with_wg) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int d = a.d, E = a.E_r, T = a.T;  // router rows: experts (+ shared-gate row)
  const int g = lane >> 2, c = lane & 3;
  const int KP = router_kpart(d, E), nkp = router_nkp(d, E), Epad = router_epad(E);
  const int t0 = grp * kRouterRows;
  const int cpr = KP / 8;
  if (grp == 0 && kp == 0) TG_STAMP(10);
  // x tile [32][KP] -> smem (rows past T clamped; their results are never used); on the
  // block's first item the Wg slice [E8][KP] joins the same load batch (one latency)
  const int E8 = with_wg ? (E + 7) / 8 * 8 : 0;  // Wg rows of the n8 tiles actually used
  stage_rows(
      E8 + kRouterRows, cpr,
      [&](int r) -> const uint4 * {
        if (r < E8) return r < E ? reinterpret_cast<const uint4 *>(a.wg + (size_t)r * d + kp * KP) : nullptr;
        return reinterpret_cast<const uint4 *>(a.x + (size_t)min(t0 + r - E8, T - 1) * d + kp * KP);
      },
      [&](int r) -> uint32_t * { return (r < E8 ? R.wg + r * R.ldw : R.xt + (r - E8) * R.ldw); });
  __syncthreads();
  if (grp == 0 && kp == 0) TG_STAMP(11);
  const int ksw = max(16, KP / 8);   // K elements of this warp (multiple of 16)
  const int nsteps = (warp * ksw < KP) ? ksw / 16 : 0;
  const int wk0 = warp * ksw / 2;    // first word column
  float *dst = a.logit_part + ((size_t)grp * nkp + kp) * kRouterRows * E;
  for (int e0 = 0; e0 < Epad; e0 += 64) {
    const int ntr = min(8, (E - e0 + 7) / 8);  // n8 tiles holding real experts
    float acc[2][8][4];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int n = 0; n < 8; ++n)
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[m][n][i] = 0.f;
    for (int s = 0; s < nsteps; ++s) {
      const int wc = wk0 + 8 * s + c;  // word column of k = 16 s + 2 c
      uint32_t af[2][4];
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        const uint32_t *x0 = R.xt + (16 * m + g) * R.ldw, *x1 = x0 + 8 * R.ldw;
        af[m][0] = x0[wc];
        af[m][1] = x1[wc];
        af[m][2] = x0[wc + 4];
        af[m][3] = x1[wc + 4];
      }
#pragma unroll
      for (int n = 0; n < 8; ++n) {
        if (n < ntr) {
          const uint32_t *wr = R.wg + (e0 + 8 * n + g) * R.ldw;
          const uint32_t b0 = wr[wc], b1 = wr[wc + 4];
          mma_bf16_16816(acc[0][n], af[0], b0, b1);
          mma_bf16_16816(acc[1][n], af[1], b0, b1);
        }
      }
    }
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int n = 0; n < 8; ++n) {
        if (n >= ntr) continue;
        float *p = R.part + (warp * kRouterRows + 16 * m) * 64 + 8 * n + 2 * c;
        p[g * 64] = acc[m][n][0];
        p[g * 64 + 1] = acc[m][n][1];
        p[(g + 8) * 64] = acc[m][n][2];
        p[(g + 8) * 64 + 1] = acc[m][n][3];
      }
    __syncthreads();
    const int ew = min(64, E - e0);
    for (int i = threadIdx.x; i < kRouterRows * ew; i += blockDim.x) {
      const int r = i / ew, ee = i % ew, e = e0 + ee;
      {
        const int pi = r * 64 + ee;
        float sum = R.part[pi];
#pragma unroll
        for (int ww = 1; ww < 8; ++ww) sum += R.part[ww * kRouterRows * 64 + pi];
        dst[r * E + e] = sum;
      }
    }
    __syncthreads();
  }
}

// --------------------------------------------------------------------- P2
// Chunk of 256 tokens: bit t of bm[K][t/32] is set iff
// token t has a pair with key K (at most one per token: its k experts are
// distinct and map to distinct slots); the rank of (t, K) in the chunk is the
// popcount of the bits below t.
// One warp per token (P1b, all blocks): logits = sum of the K parts in part
// order (lanes own experts lane + 32 i), staged in a warp-private smem row.
// Expert e is selected iff fewer than k experts beat it, where e' beats e iff
// l[e'] > l[e] or (l[e'] == l[e] and e' < e) (lowest id wins ties; -0 == +0
// compare equal).  Its slot is the number of selected experts with a smaller id
// (slots in ascending expert id, R#4).  Softmax over the k selected:
// m = max, z_j = expf(l_j - m), Z = ((z_0 + z_1) + ...) in slot order,
// w_j = z_j / Z (IEEE).
// P1b for one 32-token group, by the block that delivered its last K part (or by
// a grid-stride loop in phased mode).  Logits = sum of the parts in part order
// (16 loads in flight per thread) into smem rows.  Top-k: 8 lanes per token (one
// warp holds 4 tokens), k rounds of a warp arg-max under the strict total order
// "(v, e) beats (v', e') iff v > v' or (v == v' and e < e')" — lowest id wins
// ties, -0 == +0; NaN logits read as -inf — so round j picks the expert beaten
// by exactly j others and the picks are {e : fewer than k experts beat e}.
// Slots in ascending expert id (R#4); softmax over the k selected with m = top-1
// logit, z_j = expf(l_j - m), Z = ((z_0 + z_1) + ...) in slot order (gate_mode
// 0), or over all E as 8 per-lane ascending partial sums combined by a fixed xor
// tree (gate_mode 1); w_j = z_j / Z (IEEE).  Every reduction order depends on
// (E, k) only: deterministic and row-invariant.  (Latency matters here, not
// work: short dependency chains, no branches in the scans.)
__device__ __forceinline__ bool beats(float v, int e, float v2, int e2) {
  return (v > v2) | ((v == v2) & (e < e2));
}


// Top-k of one token on 8 lanes (sub = lane & 7 holds experts e = sub + 8 i,
// i < PER, in registers): k rounds of arg-max (local chain, then a 3-level xor
// tree within the 8 lanes); the owner marks its pick taken.  Lane j keeps the
// j-th pick.
template <int PER>
__device__ __forceinline__ void topk_rows(const CallArgs &a, const RouteKeys &rk, int t0, bool act,
                                          const float *l, int *rsl) {
  const int E = a.E, k = a.k, lane = threadIdx.x & 31, sub = lane & 7;
  const int r = threadIdx.x >> 3;
  float v[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int e = sub + 8 * i;
    float x = (act && e < E) ? l[e] : -INFINITY;
    v[i] = (x != x) ? -INFINITY : x;
  }
  uint32_t taken = 0;
  int mine = 0x7fffffff;
  float mval = 0.f, m = 0.f;
#pragma unroll 1
  for (int j = 0; j < k; ++j) {
    float bv = -INFINITY;
    int be = 0x7fffffff;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int e = sub + 8 * i;
      const bool ok = (e < E) & !((taken >> i) & 1u) & beats(v[i], e, bv, be);
      bv = ok ? v[i] : bv;
      be = ok ? e : be;
    }
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oe = __shfl_xor_sync(0xffffffffu, be, o);
      const bool tk = beats(ov, oe, bv, be);
      bv = tk ? ov : bv;
      be = tk ? oe : be;
    }
    if ((be & 7) == sub) taken |= 1u << (be >> 3);
    if (sub == j) { mine = be; mval = bv; }
    if (j == 0) m = bv;  // top-1 logit = max of the selected
  }
  // slot = picks with a smaller id (ascending expert id, R#4)
  int slot = 0;
#pragma unroll 1
  for (int jj = 0; jj < k; ++jj) slot += __shfl_sync(0xffffffffu, mine, (lane & ~7) + jj) < mine;
  if (sub < k) rsl[slot] = mine;
  __syncwarp();
  float Z = 0.f;
  if (a.gate_mode == 0) {
#pragma unroll 1
    for (int s = 0; act && s < k; ++s) {  // fixed slot order
      const float zs = expf(l[rsl[s]] - m);
      Z = (s == 0) ? zs : Z + zs;
    }
  } else {
    // softmax over all E: per-lane partial sums in ascending i, then a fixed xor tree
#pragma unroll
    for (int i = 0; i < PER; ++i)
      if (sub + 8 * i < E) Z += expf(v[i] - m);
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) Z += __shfl_xor_sync(0xffffffffu, Z, o);
  }
  if (act) {
    const int t = t0 + r;
    if (sub < k) {
      const size_t o = (size_t)t * k + slot;
      a.idx[o] = mine;
      a.w[o] = __fdiv_rn(expf(mval - m), Z);
      a.key[o] = rk.key[mine];
    }
    if (a.shared_gate && sub == 0) a.sgate[t] = __fdiv_rn(1.0f, 1.0f + expf(-l[E]));  // router row E
  }
}

__device__ __forceinline__ void group_topk(const CallArgs &a, const RouteKeys &rk, int grp, float *sm) {
  const int Er = a.E_r, E = a.E, nkp = router_nkp(a.d, Er), ld = Er + 1;  // padded rows
  const int t0 = grp * kRouterRows, nrow = min(kRouterRows, a.T - t0);
  const int n = nrow * Er;
  const float *src = a.logit_part + (size_t)grp * nkp * kRouterRows * Er;
  float *lsum = sm;                                              // [32][Er + 1]
  int *sl = reinterpret_cast<int *>(lsum + kRouterRows * ld);    // [32][kMaxK] selected ids by slot
  const int bd = blockDim.x;
#pragma unroll 1
  for (int i0 = threadIdx.x; i0 < n; i0 += 4 * bd) {
    float s[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 1
    for (int q0 = 0; q0 < nkp; q0 += 4) {
      float p[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int q = 0; q < 4; ++q)
          p[u][q] = (i0 + u * bd < n && q0 + q < nkp)
                        ? __ldcg(src + (size_t)(q0 + q) * kRouterRows * Er + i0 + u * bd) : 0.f;
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (q0 + q < nkp) s[u] = (q0 + q == 0) ? p[u][q] : s[u] + p[u][q];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * bd;
      if (i < n) lsum[i + i / Er] = s[u];  // row i / Er, padded stride Er + 1
    }
  }
  __syncthreads();
  if (a.logits)  // parity export: the fp32 logits the top-k below decides on
    for (int i = threadIdx.x; i < n; i += bd) a.logits[(size_t)t0 * Er + i] = lsum[i + i / Er];
  if (grp == 0) TG_STAMP_ANY(31);
  // 256 threads = 32 tokens x 8; all lanes run every step (shuffles), writes are predicated
  const int r = threadIdx.x >> 3;
  const int per = (E + 7) / 8;
  if (per <= 1) topk_rows<1>(a, rk, t0, r < nrow, lsum + r * ld, sl + r * kMaxK);
  else if (per <= 2) topk_rows<2>(a, rk, t0, r < nrow, lsum + r * ld, sl + r * kMaxK);
  else if (per <= 4) topk_rows<4>(a, rk, t0, r < nrow, lsum + r * ld, sl + r * kMaxK);
  else if (per <= 8) topk_rows<8>(a, rk, t0, r < nrow, lsum + r * ld, sl + r * kMaxK);
  else if (per <= 16) topk_rows<16>(a, rk, t0, r < nrow, lsum + r * ld, sl + r * kMaxK);
  else topk_rows<32>(a, rk, t0, r < nrow, lsum + r * ld, sl + r * kMaxK);
  if (grp == 0) TG_STAMP_ANY(37);
  __syncthreads();
  __syncthreads();
}

__device__ __forceinline__ void rank_chunk(const CallArgs &a, int chunk, uint8_t *smraw) {
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
// Count exchange.  Every rank writes its per-key totals into every live peer's
// cnt_all[buf][src] and releases its count flag there; then it acquires every live
// peer's flag.  A peer silent past cnt_timeout_ns is taken as failed for this run
// (fail-stop; §5.2 "EWs tolerate AW failures"): its counts
// are zero, it is recorded in the host-mapped fail mask and in sync[6] (the ranks
// taking part in this run), so no row is dispatched to it, none of its rows is
// awaited, and its combine flag is not awaited — no trap, the survivors complete
// the run and tg_failover re-routes the pairs it held (NEXT-1).
__device__ __forceinline__ void exchange_counts(const CallArgs &a, int nchunks, int32_t *sm) {
  const int tid = threadIdx.x, nkeys = a.nkeys;
  int32_t *tot = sm;              // [nkeys] this rank's rows per key
  int32_t *gsum = sm + nkeys;     // [nkeys] rows per key over all sources
  int32_t *below = gsum + nkeys;  // [nkeys] rows per key from lower sources
  __shared__ uint32_t s_part;     // ranks taking part in this run
  const bool sys = a.world > 1;
  for (int K = tid; K < nkeys; K += blockDim.x) {
    int run = 0;
    for (int b0 = 0; b0 < nchunks; b0 += 8) {  // 8 loads in flight
      int c[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) c[u] = (b0 + u < nchunks) ? __ldcg(a.bcnt + (size_t)(b0 + u) * nkeys + K) : 0;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (b0 + u < nchunks) {
          a.bcnt[(size_t)(b0 + u) * nkeys + K] = run;  // exclusive chunk base
          run += c[u];
        }
    }
    tot[K] = run;
    atomicAdd(reinterpret_cast<unsigned long long *>(a.stats + K), (unsigned long long)run);
  }
  if (tid == 0) s_part = a.alive | (1u << a.rank);
  __syncthreads();
  if (a.world == 1) {
    // no peers: the gathered counts are this rank's own, and only its own keys carry rows
    const int k0 = a.rank * a.S_max;
    for (int K = tid; K < nkeys; K += blockDim.x) {
      gsum[K] = tot[K];
      below[K] = 0;
      a.gcounts[K] = tot[K];
    }
    __syncthreads();
    for (int K = tid; K < nkeys; K += blockDim.x) {
      const int s = K - k0;
      int off = 0;
      if (s >= 0 && s < a.S_max)
        for (int s2 = 0; s2 < s; ++s2) off += gsum[k0 + s2];
      a.dbase[K] = off;
    }
    if (tid < a.world) {
      int any = 0;
      if (tid == a.rank)
        for (int s = 0; s < a.S_max; ++s) any |= tot[k0 + s];
      a.need_src[tid] = any > 0;
      a.sent_to[tid] = any > 0;
    }
    for (int s = tid; s < a.S_loc; s += blockDim.x) a.slot_rows[s] = gsum[k0 + s];
    if (tid == 0) {
      a.sync[5] = 0;  // no token dedup without peers
      a.sync[6] = (int)(1u << a.rank);
    }
    return;
  }
  // all-gather: my totals -> cnt_all[buf][rank][*] on every live peer, then release flags
  for (int q = 0; q < a.world; ++q) {
    if (!((a.alive >> q) & 1u)) continue;
    int32_t *dst = reinterpret_cast<int32_t *>(a.sym[q] + a.L.cnt_all) + ((size_t)a.cnt_buf * a.world + a.rank) * nkeys;
    for (int K = tid; K < nkeys; K += blockDim.x) dst[K] = tot[K];
  }
  __syncthreads();
  if (tid < a.world && ((a.alive >> tid) & 1u)) {
    fence_scope(sys);
    uint32_t *fl = reinterpret_cast<uint32_t *>(a.sym[tid] + a.L.flags) + a.fslot_cnt * kMaxWorld + a.rank;
    st_release(fl, a.fepoch, sys);
    const uint32_t *mine = reinterpret_cast<const uint32_t *>(a.sym[a.rank] + a.L.flags) + a.fslot_cnt * kMaxWorld + tid;
    if (tid != a.rank && !wait_flag_or_fail(mine, a.fepoch, sys, a.cnt_timeout_ns)) {
      atomicOr(a.fail_mask, 1u << tid);  // silent peer: failed for this run (no trap)
      atomicAnd(&s_part, ~(1u << tid));
    }
  }
  __syncthreads();
  const uint32_t part = s_part;
  if (tid == 0) a.sync[6] = (int)part;
  const int32_t *A = reinterpret_cast<const int32_t *>(a.sym[a.rank] + a.L.cnt_all) + (size_t)a.cnt_buf * a.world * nkeys;
  for (int K = tid; K < nkeys; K += blockDim.x) {
    int g = 0, bl = 0;
    for (int src = 0; src < a.world; ++src) {
      const int c = src == a.rank ? tot[K] : ((part >> src) & 1u) ? __ldcg(A + (size_t)src * nkeys + K) : 0;
      if (src < a.rank) bl += c;
      g += c;
    }
    gsum[K] = g;
    below[K] = bl;
    a.gcounts[K] = g;
  }
  __syncthreads();
  // token dedup (NEXT-2) for calls that move many rows (prefill): every rank takes the same
  // decision from the same all-gathered counts (global pairs x row bytes >= 16 MB); never in
  // a failover replay
  if (tid < 32) {
    long long tot_pairs = 0;
    for (int K = tid; K < nkeys; K += 32) tot_pairs += gsum[K];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot_pairs += __shfl_xor_sync(0xffffffffu, tot_pairs, o);
    if (tid == 0) a.sync[5] = (!a.replay && tot_pairs * a.d * 2 >= (16ll << 20)) ? 1 : 0;
  }
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
      to_me += tid == a.rank ? tot[a.rank * a.S_max + s]
                             : ((part >> tid) & 1u) ? __ldcg(A + (size_t)tid * nkeys + a.rank * a.S_max + s) : 0;
      to_q += tot[tid * a.S_max + s];
    }
    a.need_src[tid] = to_me > 0;
    a.sent_to[tid] = to_q > 0 && ((part >> tid) & 1u);
  }
  for (int s = tid; s < a.S_loc; s += blockDim.x) a.slot_rows[s] = gsum[a.rank * a.S_max + s];
}

// ------------------------------------------------------- P1 -> P3 chaining
// No grid barriers between P1, P1b, P2 and P3: the block that delivers the last
// K part of a 32-token group runs its top-k (P1b); the block that completes the
// last group of a 256-token chunk ranks the chunk (P2); the block that completes
// the last chunk runs the count exchange (P3).  Arrival = __threadfence + atomic
// counter (threadfence-reduction pattern); the last arriver resets the counter
// for the next call (kernel boundaries order the calls).
__device__ void group_arrive(const CallArgs &a, const RouteKeys &rk, int grp, int nkp, int ngroups, float *sm) {
  __shared__ int s_last;
  if (threadIdx.x == 0) {
    __threadfence();
    const int last = atomicAdd(a.grp_ctr + grp, 1) == nkp - 1;
    if (last) {
      a.grp_ctr[grp] = 0;
      __threadfence();
    }
    s_last = last;
  }
  __syncthreads();
  if (grp == 0 && a.trace && threadIdx.x == 0)
    a.trace[a.n_units_max + 148 + 40 + (blockIdx.x % nkp)] = globaltimer_ns();  // arrival of each part
  if (!s_last) return;
  if (grp == 0) TG_STAMP_ANY(30);
  group_topk(a, rk, grp, sm);
  if (grp == 0) TG_STAMP_ANY(12);
  constexpr int gpc = kRankBlock / kRouterRows;
  const int ch = grp / gpc, nchunks = (a.T + kRankBlock - 1) / kRankBlock;
  const int ng_ch = min(gpc, ngroups - ch * gpc);
  if (threadIdx.x == 0) {
    __threadfence();
    const int last = atomicAdd(a.chunk_ctr + 1 + ch, 1) == ng_ch - 1;
    if (last) {
      a.chunk_ctr[1 + ch] = 0;
      __threadfence();
    }
    s_last = last;
  }
  __syncthreads();
  if (!s_last) return;
  rank_chunk(a, ch, reinterpret_cast<uint8_t *>(sm));
  if (ch == 0) TG_STAMP_ANY(13);
  if (threadIdx.x == 0) {
    __threadfence();
    const int last = atomicAdd(a.chunk_ctr, 1) == nchunks - 1;
    if (last) {
      a.chunk_ctr[0] = 0;
      __threadfence();
    }
    s_last = last;
  }
  __syncthreads();
  if (!s_last) return;
  TG_STAMP_ANY(1);
  exchange_counts(a, nchunks, reinterpret_cast<int32_t *>(sm));
  TG_STAMP_ANY(14);
  __syncthreads();
}

// --------------------------------------------------------------------- P4
// Warp copy of one row of nch 16-B chunks: up to 16 loads of a lane in flight
// before its stores (the copy is latency-bound per warp).
template <bool kCoherent = false>
__device__ __forceinline__ void copy_row(uint4 *__restrict__ dst, const uint4 *__restrict__ src, int nch, int lane) {
  for (int c0 = lane; c0 < nch; c0 += 16 * 32) {
    uint4 v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int c = c0 + 32 * u;
      if (c < nch) v[u] = kCoherent ? __ldcg(src + c) : __ldg(src + c);  // rows written by peers: L2
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int c = c0 + 32 * u;
      if (c < nch) dst[c] = v[u];
    }
  }
}

// L2 prefetch of the weights the GEMM streams first (block `part` of `nparts`
// issues its share).  The GEMM takes its GEMM1 units slot by slot; the first
// slot with rows is predicted from the previous call's per-slot counts (routing
// is sticky across decode steps).  A wrong guess only costs idle HBM bandwidth
// during this latency-bound kernel.  Issued after the router's own loads so the
// HBM queues serve those first.
__device__ void l2_prefetch_share(const CallArgs &a, int part, int nparts) {
  // issued by warp 1 (thread 0 runs the arrivals of the front chain)
  if (threadIdx.x != 32 || a.l2_prefetch_bytes <= 0) return;
  int s0 = -1;
  for (int s = 0; s < a.S_loc && s0 < 0; ++s)
    if (__ldcg(a.slot_rows + s) > 0) s0 = s;
  if (s0 < 0) return;
  const long long per_mat = min((long long)a.F * a.d * 2, a.l2_prefetch_bytes / 2);  // W1 and W3 halves
  const long long chunk = 65536;
  const long long nch = per_mat / chunk;
  const uint8_t *b1 = reinterpret_cast<const uint8_t *>(a.bank_w1) + (size_t)s0 * a.F * a.d * 2;
  const uint8_t *b3 = reinterpret_cast<const uint8_t *>(a.bank_w3) + (size_t)s0 * a.F * a.d * 2;
  for (long long c = part; c < nch; c += nparts) {
    prefetch_l2_bulk(b1 + c * chunk, (uint32_t)chunk);
    prefetch_l2_bulk(b3 + c * chunk, (uint32_t)chunk);
  }
}

// P1..P3 (all 256 threads of every CTA; cooperative grid).  Ends with a grid
// barrier: the receive layout (dbase, slot_rows, need_src, ...) is then visible
// to every CTA.  fsm: this CTA's dynamic shared memory (front layout).
__device__ __forceinline__ void front_phase(const CallArgs &a, const RouteKeys &rk, uint8_t *fsm) {
  // grid barriers of this call count on sync[8 + 4 * (epoch & 1)] (u64) from 0; the other
  // counter is reset here for the next call (the previous call has completed: PDL wait
  // at kernel entry)
  unsigned long long *gbar = reinterpret_cast<unsigned long long *>(a.sync + 8 + 4 * (a.epoch & 1));
  if (blockIdx.x == 0 && threadIdx.x == 0)
    *reinterpret_cast<unsigned long long *>(a.sync + 8 + 4 * ((a.epoch + 1) & 1)) = 0ull;
  int nbar = 0;
  TG_STAMP(0);
  // ---- P1 router (+ reset of the GEMM counters of this call)
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n_ctr_max; i += gridDim.x * blockDim.x) a.ctr[i] = 0;
  if (blockIdx.x == 0 && threadIdx.x < 5) a.sync[threadIdx.x] = 0;
  TG_STAMP(8);
  const int ngroups = (a.T + kRouterRows - 1) / kRouterRows;
  {
    const int nkp = router_nkp(a.d, a.E_r), KP = router_kpart(a.d, a.E_r), Epad = router_epad(a.E_r);
    RouterSmem R;
    R.ldw = KP / 2 + 4;
    R.wg = reinterpret_cast<uint32_t *>(fsm);
    R.xt = R.wg + Epad * R.ldw;
    R.part = reinterpret_cast<float *>(R.xt + kRouterRows * R.ldw);
    const int bpp = gridDim.x / nkp;  // blocks per K part
    const int kp = blockIdx.x % nkp, slot = blockIdx.x / nkp;
    // chained (decode-sized calls): at most one router item per block, P1b-P3 run by
    // the last arrivers; phased (prefill-sized): grid-stride phases between barriers,
    // so no block serialises the top-k of many groups
    const bool chain = ngroups <= bpp;
    if (slot < bpp && slot < ngroups) {
      int it = 0;
      for (int grp = slot; grp < ngroups; grp += bpp, ++it) {
        if (it < 5) TG_STAMP(20 + 2 * it);
        router_item(a, R, grp, kp, it == 0);
        if (it < 5) TG_STAMP(21 + 2 * it);
        if (chain) group_arrive(a, rk, grp, nkp, ngroups, R.part);
      }
    }
    // every CTA issues its share of the L2 prefetch, behind the router's own loads: the router
    // CTAs after their item (and its top-k chain), the idle ones after a short delay
    if (!(slot < bpp && slot < ngroups)) __nanosleep(2000);
    l2_prefetch_share(a, blockIdx.x, gridDim.x);
    if (!chain) {
      const int nchunks = (a.T + kRankBlock - 1) / kRankBlock;
      grid_barrier_z(gbar, nbar++, a.err);
      for (int grp = blockIdx.x; grp < ngroups; grp += gridDim.x) group_topk(a, rk, grp, R.part);
      TG_STAMP(12);
      grid_barrier_z(gbar, nbar++, a.err);
      for (int ch = blockIdx.x; ch < nchunks; ch += gridDim.x) rank_chunk(a, ch, reinterpret_cast<uint8_t *>(R.part));
      TG_STAMP(13);
      grid_barrier_z(gbar, nbar++, a.err);
      if (blockIdx.x == 0) {
        TG_STAMP(1);
        exchange_counts(a, nchunks, reinterpret_cast<int32_t *>(R.part));
        TG_STAMP(14);
      }
    } else if (ngroups == 0 && blockIdx.x == 0) {
      // no tokens: the count exchange still runs (peers wait for this rank's counts)
      exchange_counts(a, 0, reinterpret_cast<int32_t *>(R.part));
    }
  }
  if (a.trace && threadIdx.x == 0) a.trace[a.n_units_max + 148 + 64 + blockIdx.x] = globaltimer_ns();
  grid_barrier_z(gbar, nbar++, a.err);
  TG_STAMP(3);
}

// In-call failover (NEXT-1, §5.1 "the AW re-dispatches the affected
// tokens ... to an alternate EW hosting the same expert (either a healthy primary
// or a shadow)"): replay of the last call's pairs whose
// destination rank failed.  Every such pair takes the next live candidate of its
// expert (rk = the resolution after fail-stopping the failed ranks), on whichever
// rank it lives; the other pairs keep their (good) outputs and get no key.  Then
// P2 and the count exchange among the surviving ranks (replay flags and buffer),
// so the replay rows are the whole work list of the destination EWs ("replayed
// requests are prioritized").
__device__ __forceinline__ void replay_front(const CallArgs &a, const RouteKeys &rk, uint8_t *fsm) {
  unsigned long long *gbar = reinterpret_cast<unsigned long long *>(a.sync + 8 + 4 * (a.epoch & 1));
  if (blockIdx.x == 0 && threadIdx.x == 0)
    *reinterpret_cast<unsigned long long *>(a.sync + 8 + 4 * ((a.epoch + 1) & 1)) = 0ull;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n_ctr_max; i += gridDim.x * blockDim.x) a.ctr[i] = 0;
  if (blockIdx.x == 0 && threadIdx.x < 5) a.sync[threadIdx.x] = 0;
  int nbar = 0;
  const int npairs = a.T * a.k;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < npairs; p += gridDim.x * blockDim.x) {
    const int K = __ldcg(a.key_old + p);
    int nk = -1;
    if (K >= 0 && ((a.failed >> (K / a.S_max)) & 1u)) {
      nk = rk.key[__ldcg(a.idx + p)];
      if (nk < 0) atomicAdd(a.unrec, 1);  // no live candidate left (the host refuses such tables)
    }
    a.key[p] = nk;
  }
  grid_barrier_z(gbar, nbar++, a.err);
  const int nchunks = (a.T + kRankBlock - 1) / kRankBlock;
  for (int ch = blockIdx.x; ch < nchunks; ch += gridDim.x) rank_chunk(a, ch, fsm);
  grid_barrier_z(gbar, nbar++, a.err);
  if (blockIdx.x == 0) exchange_counts(a, nchunks, reinterpret_cast<int32_t *>(fsm));
  grid_barrier_z(gbar, nbar++, a.err);
}

// P4 dispatch on `nw` warps (this one is warp `w`, grid-wide numbering): one warp
// per (token, j) pair, then the shared-expert rows.  The caller syncs its
// dispatch warps and calls dispatch_done() from one thread.
__device__ __forceinline__ void dispatch_rows(const CallArgs &a, int w, int nw) {
  const int lane = threadIdx.x & 31;
  const int k = a.k, nch = a.d >> 3;
  const int npairs = a.T * k;
  const int nsh = (a.Fsh > 0 && !a.replay) ? a.T : 0;  // a replay keeps the shared expert's output
  const bool dedup = __ldcg(a.sync + 5) != 0;
  const uint32_t part = (uint32_t)__ldcg(a.sync + 6);  // ranks taking part in this run
  for (int p = w; p < npairs + nsh; p += nw) {
    if (p < npairs) {
      const int t = p / k;
      const int K = __ldcg(a.key + p);
      if (K < 0) continue;  // failover replay: pair not recomputed
      const int q = K / a.S_max;
      if (!((part >> q) & 1u)) {  // destination failed in the count exchange: re-routed by tg_failover
        if (lane == 0) a.dst_pos[p] = -1;
        continue;
      }
      const int pos =
          __ldcg(a.dbase + K) + __ldcg(a.bcnt + (size_t)(t / kRankBlock) * a.nkeys + K) + __ldcg(a.lrank + p);
      // token dedup (NEXT-2): a token goes once to each PEER rank; a later pair of the same
      // token to the same peer only names the row the peer copies locally (HBM, not NVLink)
      int from = -1;
      if (q != a.rank && dedup) {
        const int j = p - t * k;
        for (int j2 = 0; j2 < j; ++j2) {
          const int K2 = __ldcg(a.key + (size_t)t * k + j2);
          if (K2 >= 0 && K2 / a.S_max == q) {
            from = __ldcg(a.dbase + K2) + __ldcg(a.bcnt + (size_t)(t / kRankBlock) * a.nkeys + K2) +
                   __ldcg(a.lrank + (size_t)t * k + j2);
            break;
          }
        }
      }
      if (from < 0) {
        const uint4 *src = reinterpret_cast<const uint4 *>(a.x + (size_t)t * a.d);
        uint4 *dst = reinterpret_cast<uint4 *>(a.sym[q] + a.L.recv) + (size_t)pos * nch;
        copy_row(dst, src, nch, lane);
      }
      if (lane == 0) {
        int2 *meta = reinterpret_cast<int2 *>(a.sym[q] + a.L.meta);
        meta[pos] = make_int2(a.rank, p);
        reinterpret_cast<int32_t *>(a.sym[q] + a.L.dup)[pos] = from;
        a.dst_pos[p] = pos;
      }
    } else {
      const int t = p - npairs;
      const uint4 *src = reinterpret_cast<const uint4 *>(a.x + (size_t)t * a.d);
      uint4 *dst = reinterpret_cast<uint4 *>(a.sym[a.rank] + a.L.recv) + (size_t)(a.R_sh0 + t) * nch;
      copy_row(dst, src, nch, lane);
    }
  }
}

// Token dedup, receiving side: once every source's rows have landed, rows that a
// source sent once for several of its pairs are copied locally into the other
// pairs' positions.  Warps w of nw (grid-wide numbering); the caller counts the
// CTAs done on sync[4].
__device__ __forceinline__ void dedup_copies(const CallArgs &a, int w, int nw, int nrecv) {
  const int lane = threadIdx.x & 31, nch = a.d >> 3;
  const int32_t *dup = reinterpret_cast<const int32_t *>(a.sym[a.rank] + a.L.dup);
  uint4 *recv = reinterpret_cast<uint4 *>(a.sym[a.rank] + a.L.recv);
  for (int r = w; r < nrecv; r += nw) {
    const int from = __ldcg(dup + r);
    if (from >= 0) copy_row<true>(recv + (size_t)r * nch, recv + (size_t)from * nch, nch, lane);
  }
}

// Data-ready flags: the last CTA to finish its dispatch releases one flag per
// live destination (one thread per CTA, after its dispatch warps synced).
__device__ __forceinline__ void dispatch_done(const CallArgs &a) {
  const bool sys = a.world > 1;
  fence_scope(sys);
  if (atomicAdd(&a.sync[3], 1) != (int)gridDim.x - 1) return;
  fence_scope(sys);
  const uint32_t part = (uint32_t)__ldcg(a.sync + 6);
  for (int q = 0; q < a.world; ++q) {
    if (!((part >> q) & 1u)) continue;
    uint32_t *fl = reinterpret_cast<uint32_t *>(a.sym[q] + a.L.flags) + a.fslot_data * kMaxWorld + a.rank;
    st_release(fl, a.fepoch, sys);
  }
  if (a.trace) a.trace[a.n_units_max + 148 + 4] = globaltimer_ns();
}

__host__ __device__ inline size_t tg_max(size_t x, size_t y) { return x > y ? x : y; }

// Dynamic shared memory of the front phases (k_layer takes the max with the GEMM ring).
__host__ __device__ inline size_t front_smem(const CallArgs &a) {
  const int KP = router_kpart(a.d, a.E_r), ldw = KP / 2 + 4;
  // R.wg + R.xt, then R.part: router warp partials, and in turn group top-k logits,
  // the rank bitmap and the exchange arrays
  const size_t topk = (size_t)kRouterRows * (a.E_r + 1) + kRouterRows * kMaxK;
  const size_t part = tg_max(tg_max((size_t)8 * kRouterRows * 64, topk), (size_t)8 * a.nkeys);
  return sizeof(uint32_t) * (size_t)(router_epad(a.E_r) + kRouterRows) * ldw + sizeof(float) * part;
}

}  // namespace tg
