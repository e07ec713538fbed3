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
    if (a.trace && threadIdx.x == 0 && VBID == 0)                                 \
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

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2(uint32_t &r0, uint32_t &r1, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(addr));
}

__host__ __device__ __forceinline__ int router_kpart(int d, int E) {
  int kp = E <= 96 ? 512 : (E <= 192 ? 256 : 128);
  while (kp > 64 && d % kp) kp >>= 1;  // d % 64 == 0, so 64 always divides d
  return kp;
}
__host__ __device__ __forceinline__ int router_nkp(int d, int E) { return (d + router_kpart(d, E) - 1) / router_kpart(d, E); }
__host__ __device__ __forceinline__ int router_epad(int E) { return (E + 63) / 64 * 64; }


// Router work decomposition, a function of E only (so every call computes a logit with
// the same arithmetic): the n8 expert tiles of an item are spread over the 8 warps and, when
// there are fewer than 8 tiles, the K part is cut into nsub sub-slices (powers of two) whose
// fp64 partials are summed in K order through shared memory.
__host__ __device__ __forceinline__ int router_ntiles(int E) { return (E + 7) / 8; }
__host__ __device__ __forceinline__ int router_nsub(int d, int E) {
  const int nt = min(router_ntiles(E), 8), steps = router_kpart(d, E) / 16;
  int ns = 1;
  while (ns * 2 * nt <= 8 && ns * 2 <= steps) ns *= 2;
  return ns;
}

constexpr int kXBufMax = 4;                 // router x tiles in flight per block
constexpr int kFrontBudget = 224 * 1024;    // dynamic smem of the front phases

__host__ __device__ __forceinline__ size_t router_wg_bytes(int d, int E) {
  return (size_t)router_epad(E) * (router_kpart(d, E) / 2 + 4) * 4;
}
__host__ __device__ __forceinline__ size_t router_xtile_bytes(int d, int E) {
  return (size_t)kRouterRows * (router_kpart(d, E) / 2 + 4) * 4;
}
__host__ __device__ __forceinline__ size_t router_red_bytes() { return (size_t)8 * kRouterRows * 8 * sizeof(double); }
// Scratch after the x ring: the router's fp64 sub-slice partials, then (aliased, used after an
// item's compute) the group top-k logits, the chunk rank bitmaps and the exchange arrays.
__host__ __device__ __forceinline__ size_t front_scratch_bytes(int E_r, int nkeys) {
  const size_t topk = sizeof(float) * ((size_t)kRouterRows * (E_r + 1) + kRouterRows * kMaxK);
  size_t m = router_red_bytes();
  if (topk > m) m = topk;
  if ((size_t)32 * nkeys > m) m = (size_t)32 * nkeys;
  if ((size_t)12 * nkeys + 64 > m) m = (size_t)12 * nkeys + 64;
  return (m + 15) / 16 * 16;
}
__host__ __device__ __forceinline__ int router_nbuf(int d, int E, int nkeys) {
  const long long room =
      (long long)kFrontBudget - (long long)router_wg_bytes(d, E) - (long long)front_scratch_bytes(E, nkeys);
  const long long n = room / (long long)router_xtile_bytes(d, E);
  return n < 1 ? 1 : (n > kXBufMax ? kXBufMax : (int)n);
}

struct RouterSmem {
  uint32_t *wg;   // [Epad][ldw] words: this block's K part of Wg, staged once
  uint32_t *xt;   // [nbuf][32][ldw] words: x tiles in flight (cp.async ring)
  double *red;    // [8][32][8] fp64 partials of the K sub-slices
  uint8_t *tail;  // group top-k, rank bitmaps, exchange arrays (alias red, not the ring)
  int ldw, nbuf;
};

__device__ __forceinline__ void cp_async16(void *smem, const void *g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Issue the cp.async loads of item (grp, kp) into ring buffer `buf` (x tile; and the Wg slice on
// the block's first item), then commit one group.  Rows past T are clamped (never used).
__device__ __forceinline__ void router_issue(const CallArgs &a, const RouterSmem &R, int grp, int kp, int buf,
                                             bool with_wg) {
  const int d = a.d, E = a.E_r, T = a.T;
  const int KP = router_kpart(d, E), cpr = KP / 8, lc = __ffs(cpr) - 1;
  if (with_wg) {
    const int nw = E * cpr;
    for (int i = threadIdx.x; i < nw; i += blockDim.x) {
      const int r = i >> lc, c = i & (cpr - 1);
      cp_async16(R.wg + r * R.ldw + c * 4, a.wg + (size_t)r * d + kp * KP + c * 8);
    }
  }
  const int t0 = grp * kRouterRows;
  uint32_t *xb = R.xt + (size_t)buf * kRouterRows * R.ldw;
  const int nx = kRouterRows * cpr;
  for (int i = threadIdx.x; i < nx; i += blockDim.x) {
    const int r = i >> lc, c = i & (cpr - 1);
    cp_async16(xb + r * R.ldw + c * 4, a.x + (size_t)min(t0 + r, T - 1) * d + kp * KP + c * 8);
  }
  cp_async_commit();
}

// P1 item: partial logits of 32 tokens over K part kp from ring buffer `buf` (landed, block
// synced).  mma.sync m16n8k16 (bf16 products exact in fp32); a warp accumulates its K range in
// sets of 8 k16 steps, each in its own fp32 registers, the sets summed in fp64 in K order
// (shorter fp32 chains: ~1 ulp of logit instead of several), sub-slices likewise through smem;
// the part's sum is stored rounded to fp32.  Order fixed by (d, E): deterministic, row-invariant.
//
// Fast path for KP = 512 and 8 expert tiles (E_r in 57..64: the DS-V2-Lite and Qwen shapes):
// warp w owns the m16 block w & 1 and the n8 tiles 2 (w >> 1), +1 (A fragments loaded once per
// two tiles), the 32 k16 steps in compile-time order with every fragment loaded two steps ahead
// of its mma (ldmatrix / mma are volatile asm: program order is issue order, so the schedule is
// written out here).  Per logit the arithmetic is the generic path's — set q = steps 8q..8q+7 in
// order, one m16n8k16 per step, sets summed in fp64 in q order — so the results are identical.
__device__ __forceinline__ void router_compute_k512_t8(const CallArgs &a, const RouterSmem &R, int grp, int kp,
                                                       int buf) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int E = a.E_r, nkp = router_nkp(a.d, E);
  const int g = lane >> 2, c = lane & 3, mb = warp & 1, t0 = 2 * (warp >> 1);
  const uint32_t *xb = R.xt + (size_t)buf * kRouterRows * R.ldw;
  const uint32_t xa = smem_u32(xb + (16 * mb + (lane & 15)) * R.ldw) + (lane >> 4) * 16;
  const uint32_t wa0 = smem_u32(R.wg + (t0 * 8 + (lane & 7)) * R.ldw) + ((lane >> 3) & 1) * 16;
  const uint32_t wa1 = wa0 + 8 * R.ldw * 4;
  float acc[4][2][4];
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[q][t][i] = 0.f;
  // issue order s = 4 st + q (k16 step q * 8 + st), fragments in a 3-deep register ring
  uint32_t fa[3][4], fb[3][4];
  auto load = [&](int s, int r) {
    const uint32_t off = (uint32_t)((s & 3) * 8 + (s >> 2)) * 32;
    ldsm_x4(fa[r], xa + off);
    ldsm_x2(fb[r][0], fb[r][1], wa0 + off);
    ldsm_x2(fb[r][2], fb[r][3], wa1 + off);
  };
  load(0, 0);
  load(1, 1);
#pragma unroll
  for (int s = 0; s < 32; ++s) {
    if (s + 2 < 32) load(s + 2, (s + 2) % 3);
    const int r = s % 3, q = s & 3;
    mma_bf16_16816(acc[q][0], fa[r], fb[r][0], fb[r][1]);
    mma_bf16_16816(acc[q][1], fa[r], fb[r][2], fb[r][3]);
  }
  float *dst = a.logit_part + ((size_t)grp * nkp + kp) * kRouterRows * E;
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      double sum = 0.0;
#pragma unroll
      for (int q = 0; q < 4; ++q) sum += (double)acc[q][t][i];
      const int row = 16 * mb + g + 8 * (i >> 1), e = (t0 + t) * 8 + 2 * c + (i & 1);
      if (e < E) dst[row * E + e] = (float)sum;
    }
}

__device__ __forceinline__ void router_compute(const CallArgs &a, const RouterSmem &R, int grp, int kp, int buf) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int d = a.d, E = a.E_r;
  const int g = lane >> 2, c = lane & 3;
  const int KP = router_kpart(d, E), nkp = router_nkp(d, E);
  const int ntl = router_ntiles(E), nsub = router_nsub(d, E), nte = min(ntl, 8);
  const int steps = KP / 16 / nsub;               // k16 steps of one sub-slice
  if (KP == 512 && ntl == 8 && nsub == 1) {
    router_compute_k512_t8(a, R, grp, kp, buf);
    return;
  }
  const uint32_t *xb = R.xt + (size_t)buf * kRouterRows * R.ldw;
  float *dst = a.logit_part + ((size_t)grp * nkp + kp) * kRouterRows * E;
  for (int eb = 0; eb < ntl; eb += 8) {          // expert blocks of 8 n8 tiles (E > 64)
    const int tile = eb + warp % nte, sub = warp / nte;
    const bool act = (warp < nte * nsub) && (tile < ntl);
    double v[2][4];
    if (act) {
      // fragments by ldmatrix: A (x, row-major 16 x 16 per m) as x4, B (Wg rows = experts, k
      // contiguous = the .col operand) as x2; lane L addresses row L & 15 (A) / L & 7 (B)
      const uint32_t xa = smem_u32(xb + (lane & 15) * R.ldw) + (lane >> 4) * 16;
      const uint32_t wa = smem_u32(R.wg + (tile * 8 + (lane & 7)) * R.ldw) + ((lane >> 3) & 1) * 16;
      const uint32_t mstr = 16 * R.ldw * 4;  // bytes between the two m16 row blocks
      const int k0 = sub * steps;            // first k16 step of this warp's sub-slice
      const int nsets = (steps + 7) / 8;
      float acc[4][2][4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int m = 0; m < 2; ++m)
#pragma unroll
          for (int i = 0; i < 4; ++i) acc[q][m][i] = 0.f;
      // the sets' steps interleaved: 8 independent accumulator chains per warp (the set a
      // step belongs to, not the issue order, decides where it is summed); the step loop is
      // not unrolled (short code: decode parts run 4 steps of one set)
#pragma unroll 1
      for (int st = 0; st < min(steps, 8); ++st) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int kstep = q * 8 + st;
          if (q < nsets && kstep < steps) {
            const uint32_t off = (uint32_t)(k0 + kstep) * 32;  // 16 bf16 = 32 B per k16 step
            uint32_t a0[4], a1[4], b0, b1;
            ldsm_x4(a0, xa + off);
            ldsm_x4(a1, xa + mstr + off);
            ldsm_x2(b0, b1, wa + off);
            mma_bf16_16816(acc[q][0], a0, b0, b1);
            mma_bf16_16816(acc[q][1], a1, b0, b1);
          }
        }
      }
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          double sum = 0.0;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (q < nsets) sum += (double)acc[q][m][i];
          v[m][i] = sum;
        }
    }
    // lane holds rows 16m + g (+8 for i >= 2), experts 8 tile + 2c (+1 for odd i)
    if (nsub == 1) {
      if (act)
#pragma unroll
        for (int m = 0; m < 2; ++m)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int row = 16 * m + g + 8 * (i >> 1), e = tile * 8 + 2 * c + (i & 1);
            if (e < E) dst[row * E + e] = (float)v[m][i];
          }
    } else {
      if (act)
#pragma unroll
        for (int m = 0; m < 2; ++m)
#pragma unroll
          for (int i = 0; i < 4; ++i)
            R.red[(warp * kRouterRows + 16 * m + g + 8 * (i >> 1)) * 8 + 2 * c + (i & 1)] = v[m][i];
      __syncthreads();
      for (int i = threadIdx.x; i < kRouterRows * nte * 8; i += blockDim.x) {
        const int row = i / (nte * 8), col = i % (nte * 8), tl = col / 8, e = (eb + tl) * 8 + (col & 7);
        double sum = 0.0;
        for (int sb = 0; sb < nsub; ++sb) sum += R.red[((sb * nte + tl) * kRouterRows + row) * 8 + (col & 7)];
        if (e < E) dst[row * E + e] = (float)sum;
      }
      __syncthreads();
    }
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
                                          const float *l, int *rsl, uint64_t *cyc = nullptr) {
  const int E = a.E, k = a.k, lane = threadIdx.x & 31, sub = lane & 7;
  if (cyc && threadIdx.x == 0) cyc[0] = clock64();
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
  if (cyc && threadIdx.x == 0) cyc[1] = clock64();
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
  if (cyc && threadIdx.x == 0) cyc[2] = clock64();
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
  if (cyc && threadIdx.x == 0) cyc[3] = clock64();
}

template <int U, int Q>
__device__ __forceinline__ void gather_parts(const float *src, size_t pstride, int n, int nkp, int Er, float *lsum) {
  const int bd = blockDim.x;
#pragma unroll 1
  for (int i0 = threadIdx.x; i0 < n; i0 += U * bd) {
    double s[U];
#pragma unroll
    for (int u = 0; u < U; ++u) s[u] = 0.0;
#pragma unroll 1
    for (int q0 = 0; q0 < nkp; q0 += Q) {
      float p[U][Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const float *pq = src + (size_t)min(q0 + q, nkp - 1) * pstride;
#pragma unroll
        for (int u = 0; u < U; ++u) p[u][q] = __ldcg(pq + min(i0 + u * bd, n - 1));
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int q = 0; q < Q; ++q)
          if (q0 + q < nkp) s[u] += (double)p[u][q];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * bd;
      if (i < n) lsum[i + i / Er] = (float)s[u];  // row i / Er, padded stride Er + 1
    }
  }
}

__device__ __forceinline__ void group_topk(const CallArgs &a, const RouteKeys &rk, int grp, float *sm,
                                           uint64_t *cyc = nullptr) {
  if (cyc && threadIdx.x == 0) cyc[4] = clock64();
  const int Er = a.E_r, E = a.E, nkp = router_nkp(a.d, Er), ld = Er + 1;  // padded rows
  const int t0 = grp * kRouterRows, nrow = min(kRouterRows, a.T - t0);
  const int n = nrow * Er;
  const size_t pstride = (size_t)kRouterRows * Er;  // one K part of the group
  const float *src = a.logit_part + (size_t)grp * nkp * pstride;
  float *lsum = sm;                                              // [32][Er + 1]
  int *sl = reinterpret_cast<int *>(lsum + kRouterRows * ld);    // [32][kMaxK] selected ids by slot
  const int bd = blockDim.x;
  // Parts summed in fp64 in part order, rounded once.  Every load of a round is issued before
  // the first sum: unconditional loads from clamped addresses (a predicated load whose value
  // is consumed at once serialises the round on its latency), out-of-range values unused.
  // U elements x Q parts per thread and round, by the group's size (decode: one element).
  if (n <= bd) gather_parts<1, 8>(src, pstride, n, nkp, Er, lsum);
  else if (n <= 4 * bd) gather_parts<4, 4>(src, pstride, n, nkp, Er, lsum);
  else gather_parts<8, 4>(src, pstride, n, nkp, Er, lsum);
  __syncthreads();
  if (a.logits)  // parity export: the fp32 logits the top-k below decides on
    for (int i = threadIdx.x; i < n; i += bd) a.logits[(size_t)t0 * Er + i] = lsum[i + i / Er];
  if (grp == 0) TG_STAMP_ANY(31);
  if (cyc && threadIdx.x == 0) cyc[5] = clock64();
  // 256 threads = 32 tokens x 8; all lanes run every step (shuffles), writes are predicated
  const int r = threadIdx.x >> 3;
  const int per = (E + 7) / 8;
  if (per <= 1) topk_rows<1>(a, rk, t0, r < nrow, lsum + r * ld, sl + r * kMaxK, cyc);
  else if (per <= 2) topk_rows<2>(a, rk, t0, r < nrow, lsum + r * ld, sl + r * kMaxK, cyc);
  else if (per <= 4) topk_rows<4>(a, rk, t0, r < nrow, lsum + r * ld, sl + r * kMaxK, cyc);
  else if (per <= 8) topk_rows<8>(a, rk, t0, r < nrow, lsum + r * ld, sl + r * kMaxK, cyc);
  else if (per <= 16) topk_rows<16>(a, rk, t0, r < nrow, lsum + r * ld, sl + r * kMaxK, cyc);
  else topk_rows<32>(a, rk, t0, r < nrow, lsum + r * ld, sl + r * kMaxK, cyc);
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
  // every key load issued before the first use (clamped address, value dropped past T)
  const int tc = min(t, max(a.T - 1, 0));
#pragma unroll
  for (int j = 0; j < kMaxK; ++j) K[j] = (j < k) ? __ldcg(a.key + (size_t)tc * k + j) : -1;  // used below
#pragma unroll
  for (int j = 0; j < kMaxK; ++j) {
    if (t >= a.T) K[j] = -1;
    if (j < k && K[j] >= 0) atomicOr(&bm[K[j] * 8 + (tid >> 5)], 1u << (tid & 31));
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kMaxK; ++j) {  // (compile-time indices: K stays in registers)
    if (j >= k || K[j] < 0) continue;
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
    for (int b0 = 0; b0 < nchunks; b0 += 8) {  // 8 loads in flight (short code: this runs cold, once per call)
      int c[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) c[u] = __ldcg(a.bcnt + (size_t)min(b0 + u, nchunks - 1) * nkeys + K);  // unconditional: all in flight
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

// P4 at world == 1, layout half: every pair's receive row and origin, and the token of every
// row (the rows themselves are copied in row order beside the GEMM, dispatch_local_rows).  Up
// to kLocalLayoutBlock pairs (decode) it is run by the block that ran the count exchange, right
// after it (no extra grid barrier); larger calls run it on every thread after the barrier.

// Early start (decode-sized single-rank calls): the GEMM phase begins without a grid barrier.
// The chain's exchange block lays out the pairs, resets this call's counters (its buffer set was
// last used by call n-2, which has exited once any CTA of call n runs: call n launched only after
// every CTA of call n-1 triggered, each after its own front) and releases a per-set ready word
// (sync[12] = epoch); a CTA waits for that word instead of for the last CTA of this call, which
// starts only when the previous call's last CTA exits.  Under PDL the GEMM units of this call
// thus run on the SMs the previous call's tail frees.  Row copies are then claimed dynamically
// (sync[13]), so the CTAs that started first copy them.
__device__ __forceinline__ bool early_start(const CallArgs &a) {
  const int nkp = router_nkp(a.d, a.E_r), ngroups = (a.T + kRouterRows - 1) / kRouterRows;
  if (a.replay || a.T <= 0 || ngroups > (int)VGRID / nkp) return false;
  if (a.local_rows) return a.T * a.k <= a.layout_block;
  // world > 1: the pairs are dispatched by claims after the ready word (the data flags released
  // by the warp completing the last pair); never with token dedup, whose copies wait for every
  // CTA (dedup needs >= 16 MB of rows, an upper bound of which is static)
  return (long long)a.T_max * a.world * a.k * a.d * 2 < (16ll << 20);
}
__device__ __forceinline__ void local_layout(const CallArgs &a, int i0, int stride) {
  const int npairs = a.T * a.k;
  int2 *meta = reinterpret_cast<int2 *>(a.sym[a.rank] + a.L.meta);
  for (int p = i0; p < npairs; p += stride) {
    const int t = p / a.k, K = __ldcg(a.key + p);
    const int pos = __ldcg(a.dbase + K) + __ldcg(a.bcnt + (size_t)(t / kRankBlock) * a.nkeys + K) + __ldcg(a.lrank + p);
    a.dst_pos[p] = pos;
    meta[pos] = make_int2(a.rank, p);
    a.srcrow[pos] = t;
  }
}

// ------------------------------------------------------- P1 -> P3 chaining
// No grid barriers between P1, P1b, P2 and P3: the block that delivers the last
// K part of a 32-token group runs its top-k (P1b); the block that completes the
// last group of a 256-token chunk ranks the chunk (P2); the block that completes
// the last chunk runs the count exchange (P3).  Arrival = __threadfence + atomic
// counter (threadfence-reduction pattern); the last arriver resets the counter
// for the next call (kernel boundaries order the calls).
__device__ __forceinline__ void post_wait_resets(const CallArgs &a, int b, int nb_);

__device__ void group_arrive(const CallArgs &a, const RouteKeys &rk, int grp, int nkp, int ngroups, float *sm) {
  __shared__ int s_last;
  if (threadIdx.x == 0) {
    __threadfence();
    const int last = atomicAdd(a.grp_ctr + (size_t)a.cbuf * a.gmax + grp, 1) == nkp - 1;
    s_last = last;
  }
  __syncthreads();
  if (grp == 0 && a.trace && threadIdx.x == 0)
    a.trace[a.n_units_max + 148 + 40 + (grp % nkp)] = globaltimer_ns();  // arrival (group 0: slot of part)
  if (!s_last) return;
  if (grp == 0) TG_STAMP_ANY(30);
  group_topk(a, rk, grp, sm);
  if (grp == 0) TG_STAMP_ANY(12);
  constexpr int gpc = kRankBlock / kRouterRows;
  const int ch = grp / gpc, nchunks = (a.T + kRankBlock - 1) / kRankBlock;
  const int ng_ch = min(gpc, ngroups - ch * gpc);
  if (threadIdx.x == 0) {
    __threadfence();
    const int last = atomicAdd(a.chunk_ctr + (size_t)a.cbuf * a.cmax + 1 + ch, 1) == ng_ch - 1;
    s_last = last;
  }
  __syncthreads();
  if (!s_last) return;
  rank_chunk(a, ch, reinterpret_cast<uint8_t *>(sm));
  if (ch == 0) TG_STAMP_ANY(13);
  if (threadIdx.x == 0) {
    __threadfence();
    const int last = atomicAdd(a.chunk_ctr + (size_t)a.cbuf * a.cmax, 1) == nchunks - 1;
    s_last = last;
  }
  __syncthreads();
  if (!s_last) return;
  TG_STAMP_ANY(1);
  exchange_counts(a, nchunks, reinterpret_cast<int32_t *>(sm));
  TG_STAMP_ANY(14);
  if (a.local_rows && a.T * a.k <= a.layout_block) {
    __syncthreads();  // dbase, written by this block's exchange
    local_layout(a, threadIdx.x, blockDim.x);
  }
  if (early_start(a)) {
    post_wait_resets(a, 0, 1);
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();  // layout, exchange outputs and resets before the ready word
      atomicExch(a.sync + 12, (int)a.epoch);
    }
  }
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

// Programmatic dependent launch: the previous call triggers its dependents when its GEMM phase
// starts, so this call's CTAs start (on the SMs its tail frees) before it has completed.  Until
// griddepcontrol.wait a CTA touches only this call's input x, the router / top-k / rank scratch
// (the previous call is past its front) and state kept per call parity (gate weights) or per
// launch mod 3 (arrival counters: reset two launches ahead, below).

// After griddepcontrol.wait (the previous launch has completed): reset what this launch's GEMM
// phase counts on, and the counter set of the launch after next.
__device__ __forceinline__ void post_wait_resets(const CallArgs &a, int b, int nb_) {
  // (b, nb_): this block's index among the nb_ blocks sharing the resets
  for (int i = b * blockDim.x + threadIdx.x; i < a.n_ctr_all; i += nb_ * blockDim.x) a.ctr[i] = 0;
  // this rank's per-token arrival counters: the peers add to them only after this rank's dispatch
  // (after the front's last grid barrier); the previous call's arrivals all landed before its combine
  for (int i = b * blockDim.x + threadIdx.x; i < a.T; i += nb_ * blockDim.x) a.tokctr[i] = 0;
  if (b == 0 && threadIdx.x == 0) a.sync[7] = 0;  // "combine incomplete" (a peer silent mid-call)
  const int nb = (a.cbuf + 2) % 3;
  for (int i = b * blockDim.x + threadIdx.x; i < a.gmax; i += nb_ * blockDim.x) a.grp_ctr[(size_t)nb * a.gmax + i] = 0;
  for (int i = b * blockDim.x + threadIdx.x; i < a.cmax; i += nb_ * blockDim.x) a.chunk_ctr[(size_t)nb * a.cmax + i] = 0;
  if (b == 0 && threadIdx.x == 0) {
    *reinterpret_cast<unsigned long long *>(a.gsync + 8 + 4 * ((a.epoch + 1) & 1)) = 0ull;
    *reinterpret_cast<unsigned long long *>(a.sync + 10) = 0ull;  // the combine phase's barrier (replays)
    a.gsync[16 + nb] = 0;
  }
  if (b == 0 && threadIdx.x < 5) a.sync[threadIdx.x] = 0;
  if (b == 0 && threadIdx.x == 0) a.sync[13] = 0;  // row-copy claims (early-start calls)
}

// World == 1, prefill-sized calls: P3 and the pair layout without a serial exchange block.
// After the rank phase every block derives, in shared memory, the per-key exclusive chunk bases
// and slot offsets from the chunk counts (the same scans exchange_counts runs at world == 1 —
// there are no peers to gather from) and lays out its grid-stride share of the pairs; block 0
// also writes what the GEMM phase and the exports read.  base: [nchunks][nkeys], tot / dofs:
// [nkeys] ints of shared memory.
__device__ __forceinline__ void local_exchange_layout(const CallArgs &a, int nchunks, int32_t *base, int32_t *tot,
                                                      int32_t *dofs) {
  const int tid = threadIdx.x, bd = blockDim.x, nkeys = a.nkeys, k0 = a.rank * a.S_max;
  for (int K = tid; K < nkeys; K += bd) {
    int run = 0;
    for (int b0 = 0; b0 < nchunks; b0 += 8) {
      int c[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) c[u] = __ldcg(a.bcnt + (size_t)min(b0 + u, nchunks - 1) * nkeys + K);
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (b0 + u < nchunks) {
          base[(b0 + u) * nkeys + K] = run;
          run += c[u];
        }
    }
    tot[K] = run;
  }
  __syncthreads();
  for (int K = tid; K < nkeys; K += bd) {
    const int sl = K - k0;
    int off = 0;
    if (sl >= 0 && sl < a.S_max)
      for (int s2 = 0; s2 < sl; ++s2) off += tot[k0 + s2];
    dofs[K] = off;
  }
  __syncthreads();
  if (VBID == 0) {
    for (int K = tid; K < nkeys; K += bd) {
      a.gcounts[K] = tot[K];
      a.dbase[K] = dofs[K];
      atomicAdd(reinterpret_cast<unsigned long long *>(a.stats + K), (unsigned long long)tot[K]);
    }
    for (int sl = tid; sl < a.S_loc; sl += bd) a.slot_rows[sl] = tot[k0 + sl];
    if (tid == 0) {
      int any = 0;
      for (int sl = 0; sl < a.S_max; ++sl) any |= tot[k0 + sl];
      a.need_src[a.rank] = any > 0;
      a.sent_to[a.rank] = any > 0;
      a.sync[5] = 0;  // no token dedup without peers
      a.sync[6] = (int)(1u << a.rank);
    }
  }
  int2 *meta = reinterpret_cast<int2 *>(a.sym[a.rank] + a.L.meta);
  const int npairs = a.T * a.k;
  for (int p = VBID * bd + tid; p < npairs; p += VGRID * bd) {
    const int t = p / a.k, K = __ldcg(a.key + p);
    const int pos = dofs[K] + base[(t / kRankBlock) * nkeys + K] + __ldcg(a.lrank + p);
    a.dst_pos[p] = pos;
    meta[pos] = make_int2(a.rank, p);
    a.srcrow[pos] = t;
  }
}

// P1..P3 (all 256 threads of every CTA; cooperative grid).  Ends with a grid
// barrier: the receive layout (dbase, slot_rows, need_src, ...) is then visible
// to every CTA.  fsm: this CTA's dynamic shared memory (front layout).
__device__ __forceinline__ void front_phase(const CallArgs &a, const RouteKeys &rk, uint8_t *fsm) {
  // grid barriers of this call count on sync[8 + 4 * (epoch & 1)] (u64) from 0; the other
  // counter is reset here for the next call (the previous call has completed: PDL wait
  // at kernel entry)
  unsigned long long *gbar = reinterpret_cast<unsigned long long *>(a.gsync + 8 + 4 * (a.epoch & 1));
  int nbar = 0;
  TG_STAMP(0);
  // ---- P1 router: router items go to the CTAs in the order they start (under PDL the first
  // ones start on the SMs the previous call's tail frees)
  __shared__ int s_item;
  if (threadIdx.x == 0) s_item = atomicAdd(a.gsync + 16 + a.cbuf, 1);
  __syncthreads();
  const int bitem = s_item;
  TG_STAMP(8);
  const int ngroups = (a.T + kRouterRows - 1) / kRouterRows;
  // world == 1, phased front: exchange + layout by every block from the chunk counts (the bases
  // fit the router ring)
  const bool lx = a.local_rows && a.world == 1 && ngroups > (int)VGRID / router_nkp(a.d, a.E_r) &&
                  (size_t)((a.T + kRankBlock - 1) / kRankBlock + 2) * a.nkeys * 4 <=
                      (size_t)router_nbuf(a.d, a.E_r, a.nkeys) * router_xtile_bytes(a.d, a.E_r);
  {
    const int nkp = router_nkp(a.d, a.E_r), KP = router_kpart(a.d, a.E_r);
    RouterSmem R;
    R.ldw = KP / 2 + 4;
    R.nbuf = router_nbuf(a.d, a.E_r, a.nkeys);
    R.wg = reinterpret_cast<uint32_t *>(fsm);
    R.xt = reinterpret_cast<uint32_t *>(fsm + router_wg_bytes(a.d, a.E_r));
    R.red = reinterpret_cast<double *>(fsm + router_wg_bytes(a.d, a.E_r) + R.nbuf * router_xtile_bytes(a.d, a.E_r));
    R.tail = reinterpret_cast<uint8_t *>(R.red);
    const int bpp = VGRID / nkp;  // blocks per K part
    const int kp = bitem % nkp, slot = bitem / nkp;
    // Block (kp, slot) runs items (group slot + i * bpp, part kp); its items stream through a
    // cp.async ring of nbuf x tiles (the loads of the next items in flight during this one).
    // Decode-sized calls (one item per block): no grid barrier until the receive layout — the
    // block that delivers the last K part of a group runs its top-k, the one completing a
    // chunk's last group ranks the chunk, the one completing the last chunk runs the count
    // exchange (last-arriver chain, group_arrive).  Prefill-sized calls: grid-stride top-k and
    // rank phases between barriers (a chain would pile the top-k of many groups on the blocks
    // that happen to arrive last).
    const bool chain = ngroups <= bpp;
    const bool early = early_start(a);  // implies chain
    if (early) {
      // items claimed dynamically (numbered K-part-major: a block's successive items mostly
      // share its staged Wg slice), so the CTAs that start first — on the SMs the previous call's
      // tail frees first — run the whole router and its chain instead of waiting for the 64th CTA
      const int nitems = ngroups * nkp;
      // two Wg slices fit the slice region (E_r <= 32: rows [0, 32) and [32, 64)): the next item is
      // claimed and its loads issued before this one computes; otherwise one buffer, the Wg slice
      // restaged when the K part changes.  (One loop: router_compute is inlined once here.)
      const bool two = a.E_r <= 32 && R.nbuf >= 2;
      auto half = [&](int b) {
        RouterSmem Rb = R;
        Rb.wg = R.wg + (size_t)b * 32 * R.ldw;
        return Rb;
      };
      int item = bitem, cur_kp = -1, b = 0;
      if (two && item < nitems) router_issue(a, half(0), item % ngroups, item / ngroups, 0, true);
      while (item < nitems) {
        const int ikp = item / ngroups, grp = item % ngroups;
        if (!two) {
          router_issue(a, R, grp, ikp, 0, ikp != cur_kp);
          cur_kp = ikp;
        }
        if (threadIdx.x == 0) s_item = atomicAdd(a.gsync + 16 + a.cbuf, 1);  // the next one, meanwhile
        __syncthreads();
        const int next = s_item;
        if (two && next < nitems) {
          router_issue(a, half(b ^ 1), next % ngroups, next / ngroups, b ^ 1, true);
          cp_async_wait<1>();
        } else {
          cp_async_wait<0>();
        }
        __syncthreads();
        router_compute(a, two ? half(b) : R, grp, ikp, b);
        __syncthreads();
        group_arrive(a, rk, grp, nkp, ngroups, reinterpret_cast<float *>(R.tail));
        item = next;
        if (two) b ^= 1;
      }
    } else if (slot < bpp && slot < ngroups) {
      const int nit = (ngroups - slot + bpp - 1) / bpp;
      const int pre = min(R.nbuf, nit);
      for (int i = 0; i < pre; ++i) router_issue(a, R, slot + i * bpp, kp, i, i == 0);
      for (int it = 0; it < nit; ++it) {
        const int grp = slot + it * bpp;
        // this item's group has landed once at most (pending items - 1) newer groups remain
        const int newer = min(R.nbuf, nit - it) - 1;
        if (newer >= 3) cp_async_wait<3>();
        else if (newer == 2) cp_async_wait<2>();
        else if (newer == 1) cp_async_wait<1>();
        else cp_async_wait<0>();
        __syncthreads();
        if (it < 5) TG_STAMP(20 + 2 * it);
        if (it == 1 && a.trace && threadIdx.x == 0 && VBID == 0) {  // effective SM clock of an item
          a.trace[a.n_units_max + 148 + 64 + 1012] = globaltimer_ns();
          a.trace[a.n_units_max + 148 + 64 + 1013] = clock64();
        }
        router_compute(a, R, grp, kp, it % R.nbuf);
        if (it == 1 && a.trace && threadIdx.x == 0 && VBID == 0) {
          a.trace[a.n_units_max + 148 + 64 + 1014] = globaltimer_ns();
          a.trace[a.n_units_max + 148 + 64 + 1015] = clock64();
        }
        if (it < 5) TG_STAMP(21 + 2 * it);
        __syncthreads();  // buffer it % nbuf is free again
        if (it + R.nbuf < nit) router_issue(a, R, slot + (it + R.nbuf) * bpp, kp, it % R.nbuf, false);
        if (chain) group_arrive(a, rk, grp, nkp, ngroups, reinterpret_cast<float *>(R.tail));
      }
    }
    // every CTA issues its share of the L2 prefetch, behind the router's own loads: the router
    // CTAs after their items (and their top-k chains), the idle ones after a short delay
    if (a.trace && threadIdx.x == 0) a.trace[a.n_units_max + 148 + 64 + 552 + VBID] = globaltimer_ns();
    if (early ? bitem >= ngroups * nkp : !(slot < bpp && slot < ngroups)) __nanosleep(2000);
    // (decode-sized calls only: at prefill the front's own phases are slower beside it than the
    // first weight tiles gain — same-box A/B, Qwen-shaped T = 8192: 789 / 811 µs without, 798 / 826 with)
    if (chain) l2_prefetch_share(a, early ? VBID : bitem, VGRID);
    if (!early) post_wait_resets(a, VBID, VGRID);  // (early start: the exchange block, before the ready word)
    if (a.trace && threadIdx.x == 0) a.trace[a.n_units_max + 148 + 64 + 700 + VBID] = globaltimer_ns();
    if (!chain) {
      const int nchunks = (a.T + kRankBlock - 1) / kRankBlock;
      grid_barrier_z(gbar, nbar++, a.err, a.ncta);
      if (a.trace && threadIdx.x == 0) a.trace[a.n_units_max + 148 + 64 + 848 + VBID] = globaltimer_ns();
      for (int grp = VBID, i = 0; grp < ngroups; grp += VGRID, ++i) {
        const long long c0 = clock64();
        group_topk(a, rk, grp, reinterpret_cast<float *>(R.tail),
                   (a.trace && VBID == 0 && i < 2) ? a.trace + a.n_units_max + 148 + 64 + 1000 + 6 * i : nullptr);
        if (a.trace && threadIdx.x == 0 && i < 2)  // cycles of the block's first two groups (cold / warm code)
          a.trace[a.n_units_max + 148 + 64 + 256 + 2 * VBID + i] = (uint64_t)(clock64() - c0);
      }
      TG_STAMP(12);
      grid_barrier_z(gbar, nbar++, a.err, a.ncta);
      for (int ch = VBID; ch < nchunks; ch += VGRID) rank_chunk(a, ch, R.tail);
      TG_STAMP(13);
      grid_barrier_z(gbar, nbar++, a.err, a.ncta);
      if (lx) {
        int32_t *base = reinterpret_cast<int32_t *>(R.xt);  // the router ring is free now
        local_exchange_layout(a, nchunks, base, base + nchunks * a.nkeys, base + (nchunks + 1) * a.nkeys);
      } else if (VBID == 0) {
        TG_STAMP(1);
        exchange_counts(a, nchunks, reinterpret_cast<int32_t *>(R.tail));
        TG_STAMP(14);
        if (a.local_rows && a.T * a.k <= a.layout_block) {
          __syncthreads();
          local_layout(a, threadIdx.x, blockDim.x);
        }
      }
    } else if (ngroups == 0 && VBID == 0) {
      // no tokens: the count exchange still runs (peers wait for this rank's counts)
      __syncthreads();  // this block's share of the resets above
      exchange_counts(a, 0, reinterpret_cast<int32_t *>(R.tail));
    }
  }
  if (a.trace && threadIdx.x == 0) a.trace[a.n_units_max + 148 + 64 + VBID] = globaltimer_ns();
  if (early_start(a)) {
    if (threadIdx.x == 0) wait_ctr_ge(a.sync + 12, (int)a.epoch, a.err, 0x4006);
    __syncthreads();
  } else {
    grid_barrier_z(gbar, nbar++, a.err, a.ncta);
  }
  TG_STAMP(3);
  if (!lx && a.local_rows && a.T * a.k > a.layout_block) {  // (smaller calls: by the exchange block)
    local_layout(a, VBID * blockDim.x + threadIdx.x, VGRID * blockDim.x);
    grid_barrier_z(gbar, nbar++, a.err, a.ncta);
  }
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
  unsigned long long *gbar = reinterpret_cast<unsigned long long *>(a.gsync + 8 + 4 * (a.epoch & 1));
  griddep_wait();
  post_wait_resets(a, VBID, VGRID);
  int nbar = 0;
  const int npairs = a.T * a.k;
  for (int p = VBID * blockDim.x + threadIdx.x; p < npairs; p += VGRID * blockDim.x) {
    const int K = __ldcg(a.key_old + p);
    int nk = -1;
    if (K >= 0 && ((a.failed >> (K / a.S_max)) & 1u)) {
      nk = rk.key[__ldcg(a.idx + p)];
      if (nk < 0) atomicAdd(a.unrec, 1);  // no live candidate left (the host refuses such tables)
    }
    a.key[p] = nk;
  }
  grid_barrier_z(gbar, nbar++, a.err, a.ncta);
  const int nchunks = (a.T + kRankBlock - 1) / kRankBlock;
  for (int ch = VBID; ch < nchunks; ch += VGRID) rank_chunk(a, ch, fsm);
  grid_barrier_z(gbar, nbar++, a.err, a.ncta);
  if (VBID == 0) exchange_counts(a, nchunks, reinterpret_cast<int32_t *>(fsm));
  grid_barrier_z(gbar, nbar++, a.err, a.ncta);
}

// P4 dispatch on `nw` warps (this one is warp `w`, grid-wide numbering): one warp
// per (token, j) pair, then the shared-expert rows.  The caller syncs its
// dispatch warps and calls dispatch_done() from one thread.
__device__ __forceinline__ void release_data_flags(const CallArgs &a);

__device__ __forceinline__ void dispatch_rows(const CallArgs &a, int w, int nw, int *claim = nullptr) {
  const int lane = threadIdx.x & 31;
  const int k = a.k, nch = a.d >> 3;
  const int npairs = a.T * k;
  const int nsh = (a.Fsh > 0 && !a.replay) ? a.T : 0;  // a replay keeps the shared expert's output
  const bool dedup = __ldcg(a.sync + 5) != 0;
  const uint32_t part = (uint32_t)__ldcg(a.sync + 6);  // ranks taking part in this run
  auto one = [&](int p) {
    if (p < npairs) {
      const int t = p / k;
      const int K = __ldcg(a.key + p);
      if (K < 0) return;  // failover replay: pair not recomputed
      const int q = K / a.S_max;
      if (!((part >> q) & 1u)) {  // destination failed in the count exchange: re-routed by tg_failover
        if (lane == 0) a.dst_pos[p] = -1;
        return;
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
  };
  const int total = npairs + nsh;
  // static: pairs w, w + nw, ...; early start: chunks of kClaim pairs claimed by whichever warps
  // run first, the warp that completes the last pair releasing the data flags (sync[3] counts
  // completed pairs).  One loop, so the pair body is inlined once (cold code, once per call).
  constexpr int kClaim = 4;
  int p = claim ? 0 : w, p1 = claim ? 0 : total, done = 0;
  const int step = claim ? 1 : nw;
  for (;;) {
    if (p >= p1) {
      if (!claim) break;
      int p0 = 0;
      if (lane == 0) p0 = atomicAdd(claim, kClaim);
      p0 = __shfl_sync(0xffffffffu, p0, 0);
      if (p0 >= total) break;
      p = p0;
      p1 = p0 + kClaim;
      done += min(p1, total) - p0;
    }
    if (p < total) one(p);
    p += step;
  }
  if (claim && done > 0) {  // one fence per warp, after all its claims: its stores before the count
    __syncwarp();
    if (lane == 0) {
      fence_scope(a.world > 1);
      if (atomicAdd(a.sync + 3, done) + done == total) release_data_flags(a);
    }
  }
}

// P4 at world == 1, copy half (warps w of nw, grid-wide numbering, beside the GEMM roles):
// routed rows in receive-row order, then the shared expert's rows, each row's token read from
// srcrow; after each row the count of its token tile (the GEMM1 unit dependency group: the
// TMA producer starts a tile's B loads once all its rows have landed) is released.  Row order
// = the order the GEMM work list consumes the tiles, so the first units start after a few
// rows, not after the whole dispatch.  grp_of(r, shared) -> token-tile group of a row.
template <typename GroupOf>
__device__ __forceinline__ void dispatch_local_rows(const CallArgs &a, int w, int nw, int nrecv, GroupOf grp_of,
                                                    int *claim = nullptr) {
  const int lane = threadIdx.x & 31, nch = a.d >> 3;
  const int nsh = (a.Fsh > 0) ? a.T : 0;
  uint4 *recv = reinterpret_cast<uint4 *>(a.sym[a.rank] + a.L.recv);
  auto copy_one = [&](int r) {
    const bool sh = r >= nrecv;
    const int row = sh ? a.R_sh0 + (r - nrecv) : r;
    const int t = sh ? r - nrecv : __ldcg(a.srcrow + r);
    copy_row(recv + (size_t)row * nch, reinterpret_cast<const uint4 *>(a.x + (size_t)t * a.d), nch, lane);
    fence_proxy_async_global();  // generic stores -> later TMA (async proxy) reads
    __syncwarp();
    if (lane == 0) {
      __threadfence();
      atomicAdd(a.rdy + grp_of(sh ? r - nrecv : r, sh), 1);
    }
  };
  const int total = nrecv + nsh;
  // static: rows w, w + nw, ...; early start: chunks claimed in receive order by whichever warps
  // run first (one loop: the row body is inlined once)
  constexpr int kClaim = 4;
  int r = claim ? 0 : w, r1 = claim ? 0 : total;
  const int step = claim ? 1 : nw;
  for (;;) {
    if (r >= r1) {
      if (!claim) break;
      int r0 = 0;
      if (lane == 0) r0 = atomicAdd(claim, kClaim);
      r0 = __shfl_sync(0xffffffffu, r0, 0);
      if (r0 >= total) break;
      r = r0;
      r1 = min(r0 + kClaim, total);
    }
    copy_one(r);
    r += step;
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
__device__ __forceinline__ void release_data_flags(const CallArgs &a) {
  const bool sys = a.world > 1;
  fence_scope(sys);
  const uint32_t part = (uint32_t)__ldcg(a.sync + 6);
  for (int q = 0; q < a.world; ++q) {
    if (!((part >> q) & 1u)) continue;
    uint32_t *fl = reinterpret_cast<uint32_t *>(a.sym[q] + a.L.flags) + a.fslot_data * kMaxWorld + a.rank;
    st_release(fl, a.fepoch, sys);
  }
  if (a.trace) a.trace[a.n_units_max + 148 + 4] = globaltimer_ns();
}

__device__ __forceinline__ void dispatch_done(const CallArgs &a) {
  fence_scope(a.world > 1);
  if (atomicAdd(&a.sync[3], 1) != (int)VGRID - 1) return;
  release_data_flags(a);
}

__host__ __device__ inline size_t tg_max(size_t x, size_t y) { return x > y ? x : y; }

// Dynamic shared memory of the front phases (k_layer takes the max with the GEMM ring).
__host__ __device__ inline size_t front_smem(const CallArgs &a) {
  // Wg slice + x-tile ring + scratch (router partials / group top-k / rank / exchange)
  return router_wg_bytes(a.d, a.E_r) + router_nbuf(a.d, a.E_r, a.nkeys) * router_xtile_bytes(a.d, a.E_r) +
         front_scratch_bytes(a.E_r, a.nkeys);
}

}  // namespace tg
