// tg_gemm.cu — GK4+GK5: persistent grouped expert-FFN kernel for sm_100a, with
// the combine exchange fused into the GEMM2 epilogue and the weighted
// unpermute (combine) run by the same CTAs after a grid barrier.
//
// One launch runs every expert FFN this rank serves as EW (§2.2.1: "an
// EW aggregates requests for the same layer and expert, and executes them as
// a single large batch") over a work list decoded on the fly from the per-slot
// row counts of this call:
//   GEMM1 units:  [a1 | a3] = W1|W3 (128 x d tile) . X^T (d x n tokens),
//                 h = bf16(silu(a1) * a3) -> H                 (SwiGLU, R#6/R#7)
//   GEMM2 units:  y = W2 (128 x F tile) . H^T, fixed split-K for long F with an
//                 in-order reduction; y = bf16(.) stored straight into the
//                 source AW's combine buffer slot [t][j] (NVLink store when the
//                 source is a peer): the combine exchange, fused.
//   combine:      out[t] = bf16(sum_j w[t,j] y[t,j] (+ y_sh[t])), fp32, j order
//                 (§2.1 "aggregated via a weighted sum").
// Swap-AB: the weight tile fills UMMA M = 128 and the tokens of a slot are UMMA
// N (16..128), so decode batches waste no tensor-core rows.
//
// Warp roles (256 threads, 1 CTA / SM, persistent over an atomic work queue):
//   w0  TMA producer: fetches unit ids, streams W and X/H tiles (128-B swizzle)
//       into a 4-stage smem ring (mbarrier full/empty, complete_tx bytes);
//       one stage carries 1-2 K blocks so every stage holds >= 32 KB of weights.
//   w1  MMA issuer: one thread issues tcgen05.mma (bf16 -> fp32 in TMEM), two
//       TMEM accumulator buffers so the epilogue overlaps the next unit.
//   w2  TMEM allocator.   w3  slot plan.   w4-7  epilogue: tcgen05.ld -> global.
#include "tg_front.cuh"
#include "tg_internal.h"
#include "tg_ptx.cuh"

namespace tg {

constexpr int kMaxPlan = kMaxSlotsPerRank + 2;
constexpr int kMaxG2Lag = 16;

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
  int nstages, stage_bytes;  // ring geometry of this call (build_plan)
  bf16 *ydst[BN_MAX_EPI];    // GEMM2 epilogue: combine-buffer row of each token of the unit
  int nrecv;                 // routed rows received by this rank (dedup copies scan them)
  // slot plan of this call (routed slots, then the shared pseudo-slot)
  int NS, G1, total, ngroups;
  int nt[kMaxPlan];        // token tiles per slot
  int rows[kMaxPlan];      // rows per slot
  int rowoff[kMaxPlan];    // first recv row
  int g1off[kMaxPlan];     // GEMM1 unit offsets
  int g2off[kMaxPlan];     // GEMM2 unit offsets
  int goff[kMaxPlan];      // dependency-group offsets
  int roff[kMaxPlan];      // reduction-group offsets
  int boff[kMaxPlan + kMaxG2Lag];  // interleaved order (g2lag > 0): block j = GEMM1 of slot j, GEMM2 of slot j - lag
};

// silu(a) = a / (1 + e^-a) with the fast exp (ex2.approx of a * log2 e: relative error <= 2 +
// 1.16 |a| ulp) and the fast divide (<= 2 ulp): <= (5 + 1.2 |a|) ulp of fp32 relative, well below
// the bf16 rounding of h that follows (R#26; the per-storage-point parity bound of h
// includes it).  IEEE expf + division measured 10 % slower per prefill call: the SwiGLU
// epilogue is on the critical path of compute-bound GEMM1 units.
__device__ __forceinline__ float silu_f(float a) { return __fdividef(a, 1.0f + __expf(-a)); }

__device__ __forceinline__ int box_index(int nrows) { return ((nrows + 15) >> 4) - 1; }

// GK5 combine of NB chunks of 8 consecutive outputs (16-B chunks c8_0 + i * stride) of token t
// (§2.1, R#5, R#16): out = bf16(sum_j w_j y_j (+ y_sh, or + sg * y_sh)) in fp32, fma chain
// in slot order j.  The loads of two slots x NB chunks are in flight together (the combine is
// bound by memory latency per thread, not by its arithmetic).
template <int NB>
__device__ __forceinline__ void combine_chunks(const CallArgs &a, const bf16 *ybuf, int t, int c8_0, int stride) {
  const int nch = a.d >> 3;
  float acc[NB][8];
#pragma unroll
  for (int i = 0; i < NB; ++i)
#pragma unroll
    for (int qq = 0; qq < 8; ++qq) acc[i][qq] = 0.f;
  auto fma8 = [&](float (&ac)[8], const uint4 &v, float wj) {
    const __nv_bfloat162 *vp = reinterpret_cast<const __nv_bfloat162 *>(&v);
#pragma unroll
    for (int qq = 0; qq < 4; ++qq) {
      float2 f = __bfloat1622float2(vp[qq]);
      ac[2 * qq] = __fmaf_rn(wj, f.x, ac[2 * qq]);
      ac[2 * qq + 1] = __fmaf_rn(wj, f.y, ac[2 * qq + 1]);
    }
  };
  for (int j = 0; j < a.k; j += 2) {
    const bool two = j + 1 < a.k;
    const float w0 = __ldcg(a.w + (size_t)t * a.k + j), w1 = two ? __ldcg(a.w + (size_t)t * a.k + j + 1) : 0.f;
    uint4 v0[NB], v1[NB];
    const uint4 *y0 = reinterpret_cast<const uint4 *>(ybuf + ((size_t)t * a.k + j) * a.d);
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      const int c8 = c8_0 + i * stride;
      if (c8 < nch) {
        v0[i] = __ldcg(y0 + c8);
        if (two) v1[i] = __ldcg(y0 + (a.d >> 3) + c8);
      }
    }
#pragma unroll
    for (int i = 0; i < NB; ++i)
      if (c8_0 + i * stride < nch) {
        fma8(acc[i], v0[i], w0);
        if (two) fma8(acc[i], v1[i], w1);
      }
  }
  if (a.Fsh > 0) {
    const float sg = a.shared_gate ? __ldcg(a.sgate + t) : 1.f;
    uint4 v[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i)
      if (c8_0 + i * stride < nch) v[i] = __ldcg(reinterpret_cast<const uint4 *>(a.ysh + (size_t)t * a.d) + c8_0 + i * stride);
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      if (c8_0 + i * stride >= nch) continue;
      const __nv_bfloat162 *vp = reinterpret_cast<const __nv_bfloat162 *>(&v[i]);
#pragma unroll
      for (int qq = 0; qq < 4; ++qq) {
        float2 f = __bfloat1622float2(vp[qq]);
        if (a.shared_gate) {  // shared expert scaled by sigmoid(x . wsg)
          acc[i][2 * qq] = __fmaf_rn(sg, f.x, acc[i][2 * qq]);
          acc[i][2 * qq + 1] = __fmaf_rn(sg, f.y, acc[i][2 * qq + 1]);
        } else {
          acc[i][2 * qq] = __fadd_rn(acc[i][2 * qq], f.x);
          acc[i][2 * qq + 1] = __fadd_rn(acc[i][2 * qq + 1], f.y);
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    const int c8 = c8_0 + i * stride;
    if (c8 >= nch) continue;
    uint4 o;
    __nv_bfloat162 *op = reinterpret_cast<__nv_bfloat162 *>(&o);
#pragma unroll
    for (int qq = 0; qq < 4; ++qq) op[qq] = __floats2bfloat162_rn(acc[i][2 * qq], acc[i][2 * qq + 1]);
    reinterpret_cast<uint4 *>(a.out + (size_t)t * a.d)[c8] = o;
  }
}

// Warp-parallel exclusive scan of per-slot quantities (lanes own contiguous slot ranges).
__device__ void build_plan(const CallArgs &a, GemmShared *P) {
  const int lane = threadIdx.x & 31;
  const int S = a.S_loc, nsh = (a.Fsh > 0 && !a.replay) ? 1 : 0, NS = S + nsh;
  const int ftiles = (a.F + BM - 1) / BM, ctiles = (a.d + BM * (a.g2dual ? 2 : 1) - 1) / (BM * (a.g2dual ? 2 : 1));
  const int ftiles_sh = nsh ? (a.Fsh + BM - 1) / BM : 0;
  const int per = (NS + 31) / 32;
  const int s0 = min(NS, lane * per), s1 = min(NS, s0 + per);
  int sr = 0, su1 = 0, su2 = 0, sg = 0, sred = 0;
  for (int s = s0; s < s1; ++s) {
    const bool sh = (s == S);
    const int rows = sh ? a.T : __ldcg(a.slot_rows + s);
    const int nt = (rows + a.bn - 1) / a.bn;
    const int ns = sh ? 1 : a.nsplit;
    P->rows[s] = rows;
    P->nt[s] = nt;
    sr += sh ? 0 : rows;
    su1 += nt * (sh ? ftiles_sh : ftiles);
    su2 += nt * ctiles * ns;
    sg += nt;
    sred += (ns > 1) ? nt * ctiles : 0;
  }
  auto xscan = [&](int v) {
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int n = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += n;
    }
    return incl - v;
  };
  // widest token tile of the call -> stage = one K block of two A tiles + that B tile
  int nbw = 16;
  for (int s = s0; s < s1; ++s) nbw = max(nbw, min(a.bn, (P->rows[s] + 15) / 16 * 16));
  nbw = __reduce_max_sync(0xffffffffu, nbw);
  int br = xscan(sr), bu1 = xscan(su1), bu2 = xscan(su2), bg = xscan(sg), bred = xscan(sred);
  for (int s = s0; s < s1; ++s) {
    const bool sh = (s == S);
    const int nt = P->nt[s];
    const int ns = sh ? 1 : a.nsplit;
    P->rowoff[s] = sh ? a.R_sh0 : br;
    P->g1off[s] = bu1;
    P->g2off[s] = bu2;
    P->goff[s] = bg;
    P->roff[s] = bred;
    br += sh ? 0 : P->rows[s];
    bu1 += nt * (sh ? ftiles_sh : ftiles);
    bu2 += nt * ctiles * ns;
    bg += nt;
    bred += (ns > 1) ? nt * ctiles : 0;
  }
  __syncwarp();  // every lane's offsets written
  if (lane == 31) {
    P->nrecv = br;  // after the scan loop: every routed slot's rows
    P->stage_bytes = 2 * kTileBytes + nbw * BK * 2;  // multiple of 2 KB: 1 KB swizzle-atom aligned
    P->nstages = min(kStages, kRingBytes / P->stage_bytes);
    P->g1off[NS] = bu1;
    P->g2off[NS] = bu2;
    P->goff[NS] = bg;
    P->roff[NS] = bred;
    P->NS = NS;
    P->G1 = bu1;
    P->total = bu1 + bu2;
    // GEMM2 units of slot s queued right after the GEMM1 units of slot s + lag (their H tiles
    // still in L2) instead of after every GEMM1 unit; each G2 unit's dependencies stay earlier in
    // the queue.  Order only: every unit's arithmetic is unchanged.
    const int L = min(a.g2lag, kMaxG2Lag);
    if (L > 0) {
      int acc = 0;
      for (int j = 0; j < NS + L; ++j) {
        P->boff[j] = acc;
        if (j < NS) acc += P->g1off[j + 1] - P->g1off[j];
        if (j >= L) acc += P->g2off[j - L + 1] - P->g2off[j - L];
      }
      P->boff[NS + L] = acc;
    }
    P->ngroups = bg;
    if (VBID == 0) *a.n_units = bu1 + bu2;
    if (bg + bred > a.n_ctr_max) {  // capacity guard (sized at init for the worst case)
      atomicExch(a.err, 0x4003);
      P->total = 0;
    }
  }
}

__device__ __forceinline__ int find_seg(const int *off, int n, int u) {
  int lo = 0, hi = n;  // off[lo] <= u < off[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (off[mid] <= u) lo = mid; else hi = mid;
  }
  return lo;
}

// Unit u of this call's work list: GEMM1 (slot, f-tile, n-tile), then GEMM2
// (slot, c-tile, n-tile, split).  Counters: per (slot, n-tile) for the GEMM1 ->
// GEMM2 dependency; per (slot, c-tile, n-tile) for the split-K reduction.
__device__ __forceinline__ Unit decode_unit(const CallArgs &a, const GemmShared *P, int u) {
  Unit U;
  const int S = a.S_loc, NS = P->NS;
  const int ftiles = (a.F + BM - 1) / BM;
  const int L = min(a.g2lag, kMaxG2Lag);
  int u1 = -1, u2i = -1;  // index among the GEMM1 / GEMM2 units
  if (L > 0) {
    const int j = find_seg(P->boff, NS + L, u);
    const int loc = u - P->boff[j];
    const int n1 = (j < NS) ? P->g1off[j + 1] - P->g1off[j] : 0;
    if (loc < n1) u1 = P->g1off[j] + loc;
    else u2i = P->g2off[j - L] + (loc - n1);
  } else if (u < P->G1) {
    u1 = u;
  } else {
    u2i = u - P->G1;
  }
  if (u1 >= 0) {
    const int s = find_seg(P->g1off, NS, u1);
    const bool sh = (s == S);
    const int loc = u1 - P->g1off[s];
    const int f = loc / P->nt[s], n = loc % P->nt[s];
    U.kind = sh ? U_G1_SH : U_G1;
    U.slot = sh ? 0 : s;
    U.m0 = f * BM;
    U.n0 = P->rowoff[s] + n * a.bn;
    U.nrows = min(a.bn, P->rows[s] - n * a.bn);
    U.kb0 = 0;
    U.kb1 = a.d / BK;
    U.dep = P->goff[s] + n;
    U.red = -1;
    U.split = 0;
    U.nsplit = 1;
    U.dep_target = 0;
    U.ntiles = P->nt[s];
    U.dual = 0;
  } else {
    const int u2 = u2i;
    const int s = find_seg(P->g2off, NS, u2);
    const bool sh = (s == S);
    const int ns = sh ? 1 : a.nsplit;
    const int nt = P->nt[s];
    const int loc = u2 - P->g2off[s];
    const int c = loc / (nt * ns), rem = loc % (nt * ns);
    const int n = rem / ns, sp = rem % ns;
    const int kbF = (sh ? a.Fsh : a.F) / BK;
    U.kind = sh ? U_G2_SH : U_G2;
    U.slot = sh ? 0 : s;
    U.m0 = c * BM * (a.g2dual ? 2 : 1);
    U.dual = a.g2dual;
    U.n0 = P->rowoff[s] + n * a.bn;
    U.nrows = min(a.bn, P->rows[s] - n * a.bn);
    U.kb0 = sp * (kbF / ns);
    U.kb1 = (sp + 1) * (kbF / ns);
    U.dep = P->goff[s] + n;
    U.dep_target = sh ? (a.Fsh + BM - 1) / BM : ftiles;
    U.red = (ns > 1) ? P->goff[NS] + P->roff[s] + c * nt + n : -1;
    U.split = sp;
    U.nsplit = ns;
    U.ntiles = nt;
  }
  return U;
}

// The whole layer call for one rank; `maps` are the kernel parameter (k_layer) or a device
// copy (k_layer_multi: several virtual ranks of one GPU in one cooperative launch).
__device__ __forceinline__ void layer_body(const TmaMaps &maps, const CallArgs &a, const RouteKeys &rk) {
  extern __shared__ uint8_t smem_raw[];
  if (a.trace && VBID == 0 && threadIdx.x == 0) {  // launch gap: previous call's end -> this entry
    a.trace[a.n_units_max + 148 + 19] = a.trace[a.n_units_max + 148 + 17];
    a.trace[a.n_units_max + 148 + 18] = globaltimer_ns();
  }
  // PDL: this call may run beside the previous one's tail (its buffer set is the other one)
  if (a.hk) {  // host-buffer path: x staged by the H2D copy stream (CallArgs::hk)
    if (threadIdx.x == 0) wait_ctr_ge(a.hk + a.hb, a.hcall, a.err, 0x4007);
    __syncthreads();
  }
  // ===================== front: P1 router .. P3 count exchange (tg_front.cuh) =====================
  if (a.replay) replay_front(a, rk, smem_raw);
  else front_phase(a, rk, smem_raw);
  // ===================== P4 dispatch (all warps; r01 A/B: 3.5% faster at 4 GPUs than on
  // warps 2-7 beside the first weight loads, equal at 1 GPU) =====================
  if (!a.local_rows) {
    if (early_start(a)) {
      dispatch_rows(a, 0, 0, a.sync + 13);  // claims; the data flags go out with the last pair
    } else {
      dispatch_rows(a, VBID * 8 + (threadIdx.x >> 5), VGRID * 8);
      __syncthreads();
      if (threadIdx.x == 0) dispatch_done(a);
    }
  }
  if (a.inject_fail) return;  // fault injection (tests): crash after the dispatch, the peers hold the rows
  // the next call may start now (PDL): its front runs on the SMs this call's tail frees, and waits
  // for this call's completion before it touches shared state
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // the ring below is refilled by TMA (async proxy) after the front's generic smem writes
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  // 1024-B aligned stage ring (128-B swizzle atoms), bookkeeping after it.
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t *ring = smem_raw + ((1024 - (raw_addr & 1023)) & 1023);
  GemmShared *S = reinterpret_cast<GemmShared *>(ring + kRingBytes);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int *err = a.err;
  const bool sys = a.world > 1;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) { mbar_init(&S->full[i], 1); mbar_init(&S->empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&S->tfull[i], 1); mbar_init(&S->tempty[i], 128); }
    for (int i = 0; i < kSchedDepth; ++i) { mbar_init(&S->sfull[i], 1); mbar_init(&S->sempty[i], 5); }
    fence_barrier_init();
    if (a.trace) a.trace[a.n_units_max + VBID] = globaltimer_ns();
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
  if (warp == 3) build_plan(a, S);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = S->tmem_base;
  const int n_units = S->total;
  const int nstages = S->nstages, stage_bytes = S->stage_bytes;
  const bool dedup = __ldcg(a.sync + 5) != 0;  // token dedup in this call (decided in P3)

  if (warp == 0) {
    {
      // ===================== TMA producer (warp 0) =====================
      // Lane 0 schedules (work items, stage barriers, expected bytes); the loads of a stage
      // are issued by different lanes in parallel — lane 3i: weight tile, 3i+1: second weight
      // tile, 3i+2: token tile of the stage's i-th K block — because one thread's TMA issues
      // serialise (~0.4 us per box: tools/probes/tma_stream.cu, 40 GB/s per SM with one issuer,
      // 70-127 with 2-6 lanes).
      const uint64_t pol_w1 = policy_evict_first();  // weight tiles streamed once (one token tile)
      const uint64_t pol_wn = policy_evict_last();   // weight tiles re-read by several token tiles
      const uint64_t pol_x = policy_evict_last();    // token tiles: re-read by every weight tile
      // Weight (A) tiles do not depend on the peers' dispatch: the first ring
      // stages get their A tiles at once and their token (B) tiles once every
      // source's rows have landed (release/acquire on per-source
      // epoch flags, then ordered before async-proxy reads).
      // world > 1 without token dedup (NEXT-2, §6.1): a GEMM1 tile waits only for the
      // data flags of the sources whose rows it holds (a slot's rows are ordered by source, so
      // the all-gathered counts give each source's row range); dedup calls wait for every
      // source (their dedup copies complete rows after the flags), replays likewise.
      const bool per_src = !a.local_rows && !dedup && !a.replay;
      bool data_ok = a.local_rows || per_src;  // world == 1: per-tile row counters instead (rdy)
      const bool own_sh = a.Fsh > 0 && !a.replay && a.T > 0;  // shared-expert rows: own dispatch
      int npend = 0;  // pending token-tile loads, held by the lane that will issue them
      int pst[kStages], pkb[kStages], prow[kStages];
      uint32_t pab[kStages];
      const CUtensorMap *pmap[kStages];
      auto wait_data = [&]() {
        if (lane == 0) {
          for (int src = 0; src < a.world; ++src) {
            if (__ldcg(a.need_src + src) || (src == a.rank && own_sh)) {
              const uint32_t *fl = reinterpret_cast<const uint32_t *>(a.sym[a.rank] + a.L.flags) +
                                   a.fslot_data * kMaxWorld + src;
              if (src == a.rank) {
                wait_flag_ge_s(fl, a.fepoch, sys, err, 0x4001);
              } else if (!wait_flag_or_fail(fl, a.fepoch, sys, a.fail_timeout_ns)) {
                atomicOr(a.fail_mask, 1u << src);  // its rows never landed: computed on stale data, discarded
              }
            }
          }
          if (dedup) {  // and the rows the dedup copies fill in (all CTAs, sync[4])
            const int *dd = a.sync + 4;
            if (ld_acquire_gpu(dd) < (int)VGRID) {
              const uint64_t t0 = globaltimer_ns();
              while (ld_acquire_gpu(dd) < (int)VGRID)
                if (globaltimer_ns() - t0 > kWaitTimeoutNs) device_fail(err, 0x4004);
            }
          }
        }
        __syncwarp();
        fence_proxy_async_global();
        data_ok = true;
        for (int i = 0; i < npend; ++i)
          tma_load_2d(ring + pst[i] * stage_bytes + pab[i], pmap[i], &S->full[pst[i]], pkb[i] * BK, prow[i], pol_x);
        npend = 0;
      };
      // world == 1: a unit's token rows are counted per tile (rdy); its pending B loads are
      // issued once the count is complete
      bool unit_ok = true;
      int udep = 0, urows = 0;
      // per_src: sources whose data flag this producer holds, and the unit's sources
      uint32_t have = 0, umask = 0;
      const uint32_t part = per_src ? (uint32_t)__ldcg(a.sync + 6) : 0u;
      const int32_t *cnt_all = reinterpret_cast<const int32_t *>(a.sym[a.rank] + a.L.cnt_all) +
                               (size_t)a.cnt_buf * a.world * a.nkeys;
      auto unit_sources = [&](const Unit &U) -> uint32_t {  // warp-uniform
        if (U.kind == U_G1_SH) return 1u << a.rank;
        const int K = a.rank * a.S_max + U.slot;
        const int lo = U.n0 - S->rowoff[U.slot], hi = lo + U.nrows;
        uint32_t m = 0;
        int off = 0;
        for (int q = 0; q < a.world && off < hi; ++q) {
          if (!((part >> q) & 1u)) continue;  // failed in the count exchange: no rows
          const int c = __ldcg(cnt_all + (size_t)q * a.nkeys + K);
          if (c > 0 && off + c > lo) m |= 1u << q;
          off += c;
        }
        return m;
      };
      auto wait_rows = [&]() {
        if (per_src) {
          if (lane == 0) {
            for (int src = 0; src < a.world; ++src) {
              if (!((umask >> src) & 1u) || ((have >> src) & 1u)) continue;
              const uint32_t *fl = reinterpret_cast<const uint32_t *>(a.sym[a.rank] + a.L.flags) +
                                   a.fslot_data * kMaxWorld + src;
              if (src == a.rank) wait_flag_ge_s(fl, a.fepoch, sys, err, 0x4001);
              else if (!wait_flag_or_fail(fl, a.fepoch, sys, a.fail_timeout_ns))
                atomicOr(a.fail_mask, 1u << src);  // its rows never landed: computed on stale data, discarded
            }
          }
          have |= umask;
        } else if (lane == 0) {
          wait_ctr_ge(a.rdy + udep, urows, err, 0x4005);
        }
        __syncwarp();
        fence_proxy_async_global();
        unit_ok = true;
        for (int i = 0; i < npend; ++i)
          tma_load_2d(ring + pst[i] * stage_bytes + pab[i], pmap[i], &S->full[pst[i]], pkb[i] * BK, prow[i], pol_x);
        npend = 0;
      };
      int stage = 0;
      uint32_t phase = 0;
      for (int it = 0;; ++it) {
        int u = 0;
        if (lane == 0) {
          u = atomicAdd(&a.sync[1], 1);
          if (u >= n_units) u = -1;
        }
        u = __shfl_sync(0xffffffffu, u, 0);
        const int r = it % kSchedDepth;
        if (lane == 0) {
          mbar_wait(&S->sempty[r], ((it / kSchedDepth) & 1) ^ 1, err);
          S->sched[r] = u;
          mbar_arrive(&S->sfull[r]);
        }
        if (u < 0) {
          if (!data_ok && __any_sync(0xffffffffu, npend > 0)) wait_data();
          break;
        }
        const Unit U = decode_unit(a, S, u);
        const bool g1 = (U.kind == U_G1 || U.kind == U_G1_SH);
        const bool sh = (U.kind == U_G1_SH || U.kind == U_G2_SH);
        if (g1 && a.local_rows) {
          // the token tile's rows are copied beside the GEMM (dispatch_local_rows): B loads go
          // out once they have landed, the unit's weight (A) tiles at once
          int ok = 0;
          if (lane == 0) ok = ld_acquire_gpu(a.rdy + U.dep) >= U.nrows;
          unit_ok = __shfl_sync(0xffffffffu, ok, 0) != 0;
          if (unit_ok) fence_proxy_async_global();
          udep = U.dep;
          urows = U.nrows;
        } else if (g1 && per_src) {
          umask = unit_sources(U);
          unit_ok = (umask & ~have) == 0;  // flags acquired earlier: proxy fence already done
        }
        if (!g1) {
          if (!data_ok) wait_data();  // GEMM1 tiles waiting on pending B loads come first
          // all GEMM1 tiles of this (slot, n-tile) have written H
          if (lane == 0) wait_ctr_ge(a.ctr + U.dep, U.dep_target, err, 0x4002);
          __syncwarp();
          fence_proxy_async_global();
        }
        const int bi = box_index(U.nrows);
        const uint32_t bbytes = (uint32_t)(bi + 1) * 16 * BK * 2;
        const bool two = g1 || U.dual;                     // two A tiles per K block (W1|W3, or W2 rows m0 and m0+128)
        const uint32_t abytes = (two ? 2u : 1u) * kTileBytes;
        const uint32_t sub = abytes + bbytes;             // one 64-wide K block of A tile(s) + B tile
        const int kps = max(1, (int)(stage_bytes / sub));  // K blocks per stage (2 for decode GEMM2)
        const CUtensorMap *mA0 = g1 ? (sh ? &maps.w1s : &maps.w1) : (sh ? &maps.w2s : &maps.w2);
        const CUtensorMap *mA1 = sh ? &maps.w3s : &maps.w3;
        const CUtensorMap *mB = g1 ? &maps.x[a.pset][bi] : (sh ? &maps.hs[a.pset][bi] : &maps.h[a.pset][bi]);
        const int rowA = g1 ? U.slot * (sh ? a.Fsh : a.F) + U.m0 : U.slot * a.d + U.m0;
        const int rowB = (!g1 && sh) ? U.n0 - a.R_sh0 : U.n0;
        const uint64_t pol_w = (U.ntiles > 1) ? pol_wn : pol_w1;
        const int li = lane / 3, role = lane % 3;  // K block of the stage / which load
        for (int kb = U.kb0; kb < U.kb1; kb += kps) {
          const int cnt = min(kps, U.kb1 - kb);
          if (!data_ok && __any_sync(0xffffffffu, npend == nstages)) wait_data();  // every stage holds a pending B tile
          if (!unit_ok && __any_sync(0xffffffffu, npend == nstages)) wait_rows();
          if (lane == 0) {
            mbar_wait(&S->empty[stage], phase ^ 1, err);
            mbar_arrive_expect_tx(&S->full[stage], (uint32_t)cnt * sub);
          }
          __syncwarp();
          uint8_t *sb = ring + stage * stage_bytes + li * sub;
          if (li < cnt) {
            const int kk = (kb + li) * BK;
            if (role == 0) {
              tma_load_2d(sb, mA0, &S->full[stage], kk, rowA, pol_w);
            } else if (role == 1) {
              if (g1) tma_load_2d(sb + kTileBytes, mA1, &S->full[stage], kk, rowA, pol_w);
              else if (U.dual) tma_load_2d(sb + kTileBytes, mA0, &S->full[stage], kk, rowA + BM, pol_w);
            } else if (data_ok && unit_ok) {
              tma_load_2d(sb + abytes, mB, &S->full[stage], kk, rowB, pol_x);
            } else {
              pst[npend] = stage; pkb[npend] = kb + li; prow[npend] = rowB;
              pab[npend] = li * sub + abytes; pmap[npend] = mB;
              ++npend;
            }
          }
          if (++stage == nstages) { stage = 0; phase ^= 1; }
        }
        if (!unit_ok && __any_sync(0xffffffffu, npend > 0)) wait_rows();  // pending loads stay within a unit
        unit_ok = true;
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ===================== MMA issuer =====================
      int stage = 0;
      uint32_t phase = 0;
      // per-half use counters as scalars: no local-memory arrays on the issuer's critical path
      int ecnt0 = 0, ecnt1 = 0, next_h = 0;
      for (int it = 0;; ++it) {
        const int r = it % kSchedDepth;
        mbar_wait(&S->sfull[r], (it / kSchedDepth) & 1, err);
        const int u = S->sched[r];
        mbar_arrive(&S->sempty[r]);
        if (u < 0) break;
        const Unit U = decode_unit(a, S, u);
        const bool g1 = (U.kind == U_G1 || U.kind == U_G1_SH);
        const int nb = (box_index(U.nrows) + 1) * 16;
        // TMEM = two 256-column halves; a wide GEMM1 unit (nb > 128) takes both
        // (a1 in half 0, a3 in half 1), every other unit one half, alternating.
        const bool wide1 = g1 && nb > 128;
        int h;
        if (wide1) {
          h = 0;
          mbar_wait(&S->tempty[0], (ecnt0 & 1) ^ 1, err);
          mbar_wait(&S->tempty[1], (ecnt1 & 1) ^ 1, err);
          ++ecnt0;
          ++ecnt1;
        } else {
          h = next_h;
          next_h ^= 1;
          const int e = h ? ecnt1 : ecnt0;
          mbar_wait(&S->tempty[h], (e & 1) ^ 1, err);
          if (h) ++ecnt1; else ++ecnt0;
        }
        tc_fence_after();
        const uint32_t idesc = idesc_bf16_f32(BM, nb);
        const uint32_t d0 = tmem + (wide1 ? 0 : h * 256), d1 = wide1 ? tmem + 256 : d0 + 128;
        const bool two = g1 || U.dual;
        const uint32_t abytes = (two ? 2u : 1u) * kTileBytes;
        const uint32_t sub = abytes + (uint32_t)nb * BK * 2;
        const int kps = max(1, (int)(stage_bytes / sub));
        for (int j0 = 0; j0 < U.kb1 - U.kb0; j0 += kps) {
          const int cnt = min(kps, U.kb1 - U.kb0 - j0);
          mbar_wait(&S->full[stage], phase, err);
          tc_fence_after();
          for (int i = 0; i < cnt; ++i) {
            const uint32_t sa = smem_u32(ring + stage * stage_bytes + i * sub);
            const uint64_t dA0 = desc_sw128_kmajor(sa);
            const uint64_t dA1 = desc_sw128_kmajor(sa + kTileBytes);
            const uint64_t dB = desc_sw128_kmajor(sa + abytes);
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              const uint32_t acc = (j0 > 0 || i > 0 || kk > 0) ? 1u : 0u;
              // advance 16 K-elements = 32 B inside the swizzle row (>>4 units)
              umma_bf16_ss(d0, dA0 + 2 * kk, dB + 2 * kk, idesc, acc);
              if (two) umma_bf16_ss(d1, dA1 + 2 * kk, dB + 2 * kk, idesc, acc);
            }
          }
          umma_commit(&S->empty[stage]);
          if (++stage == nstages) { stage = 0; phase ^= 1; }
        }
        umma_commit(&S->tfull[h]);
      }
    }
  } else {
    if (a.local_rows && (warp == 2 || warp == 3)) {
      // ===================== P4 at world == 1: rows copied in receive-row order (warps 2-3) =====================
      dispatch_local_rows(a, VBID * 2 + (warp - 2), VGRID * 2, S->nrecv, [&](int r, bool shr) {
        if (shr) return S->goff[a.S_loc] + r / a.bn;
        const int s = find_seg(S->rowoff, a.S_loc, r);
        return S->goff[s] + (r - S->rowoff[s]) / a.bn;
      }, early_start(a) ? a.sync + 13 : nullptr);
    }
    // ===================== token dedup, receiving side (warps 2-7, multi-GPU) =====================
    if (dedup) {
      if (lane == 0) {
        for (int src = 0; src < a.world; ++src) {
          if (src == a.rank || !__ldcg(a.need_src + src)) continue;
          const uint32_t *fl = reinterpret_cast<const uint32_t *>(a.sym[a.rank] + a.L.flags) +
                               a.fslot_data * kMaxWorld + src;
          if (!wait_flag_or_fail(fl, a.fepoch, sys, a.fail_timeout_ns)) atomicOr(a.fail_mask, 1u << src);
        }
      }
      __syncwarp();
      dedup_copies(a, VBID * 6 + (warp - 2), VGRID * 6, S->nrecv);
      named_bar_sync(2, 192);
      if (threadIdx.x == 64) {
        __threadfence();
        atomicAdd(a.sync + 4, 1);
      }
    }
  }
  if (warp >= 4) {
    // ===================== epilogue (128 threads) =====================
    const int q = warp & 3;            // TMEM lane quarter of this warp
    const int et = threadIdx.x - 128;  // 0..127
    const int2 *meta = reinterpret_cast<const int2 *>(a.sym[a.rank] + a.L.meta);
    int fcnt0 = 0, fcnt1 = 0, next_h = 0;
    for (int it = 0;; ++it) {
      const int r = it % kSchedDepth;
      mbar_wait(&S->sfull[r], (it / kSchedDepth) & 1, err);
      const int u = S->sched[r];
      __syncwarp();
      if (lane == 0) mbar_arrive(&S->sempty[r]);
      if (u < 0) break;
      const Unit U = decode_unit(a, S, u);
      const bool g1 = (U.kind == U_G1 || U.kind == U_G1_SH);
      const bool sh = (U.kind == U_G1_SH || U.kind == U_G2_SH);
      const int nb = (box_index(U.nrows) + 1) * 16;
      const bool wide1 = g1 && nb > 128;
      int h;
      if (wide1) h = 0; else { h = next_h; next_h ^= 1; }
      mbar_wait(&S->tfull[h], (h ? fcnt1 : fcnt0) & 1, err);
      if (h) ++fcnt1; else ++fcnt0;
      tc_fence_after();
      const int m = U.m0 + q * 32 + lane;  // weight row handled by this thread
      const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + (wide1 ? 0 : h * 256);
      const int a3off = wide1 ? 256 : 128;
      if (g1) {
        const int Fw = sh ? a.Fsh : a.F;
        bf16 *Hout = sh ? a.Hs : a.H;
        const int row0 = sh ? U.n0 - a.R_sh0 : U.n0;
        for (int c0 = 0; c0 < U.nrows; c0 += 32) {
          uint32_t r1[32], r3[32];
          tmem_ld_32x32b_x32(tbase + c0, r1);
          tmem_ld_32x32b_x32(tbase + a3off + c0, r3);
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
        mbar_arrive(&S->tempty[h]);
        if (wide1) mbar_arrive(&S->tempty[1]);
        // publish H rows: generic -> async proxy, then release the group counter
        fence_proxy_async_global();
        named_bar_sync(1, 128);
        if (et == 0) {
          __threadfence();
          atomicAdd(a.ctr + U.dep, 1);
        }
      } else {
        const bool split = (U.nsplit > 1);
        const bool direct = !split && !sh;  // y stored straight into the source AW's combine buffer
        if (direct) {
          // one origin lookup per token of the unit (not one per stored element: the loads would
          // serialise behind the stores they may alias), then a table read from smem
          for (int i = et; i < U.nrows; i += 128) {
            const int2 o = __ldcg(meta + U.n0 + i);  // L2: this CTA may not hold the source's flag (NEXT-2)
            S->ydst[i] = reinterpret_cast<bf16 *>(a.sym[o.x] + a.L.ybuf) + (size_t)o.y * a.d;
          }
          named_bar_sync(1, 128);
        }
        for (int hh = 0; hh < (U.dual ? 2 : 1); ++hh) {  // dual: second W2 tile at +128 rows / columns
          const int mm = m + hh * BM;
          for (int c0 = 0; c0 < U.nrows; c0 += 32) {
            uint32_t r1[32];
            tmem_ld_32x32b_x32(tbase + hh * 128 + c0, r1);
            tmem_ld_wait();
            if (mm < a.d) {
#pragma unroll
              for (int n = 0; n < 32; ++n) {
                if (c0 + n < U.nrows) {
                  const int row = U.n0 + c0 + n;
                  const float v = __uint_as_float(r1[n]);
                  if (split) {
                    a.ws[((size_t)U.split * a.R_cap + row) * a.d + mm] = v;
                  } else if (sh) {
                    a.ysh[(size_t)(row - a.R_sh0) * a.d + mm] = __float2bfloat16_rn(v);
                  } else {
                    S->ydst[c0 + n][mm] = __float2bfloat16_rn(v);
                  }
                }
              }
            }
          }
        }
        tc_fence_before();
        mbar_arrive(&S->tempty[h]);
        const bool arrive = a.tok_comb && !split;
        if (arrive) fence_scope(sys);  // this thread's y / y_sh stores (peer memory too) before the arrivals
        if (direct || (arrive && sh)) named_bar_sync(1, 128);  // every store of the unit done; table reusable
        if (split) {
          // fixed-order split-K reduction ((p0 + p1) + p2) + ... by the last split to finish
          __threadfence();
          named_bar_sync(1, 128);
          if (et == 0) S->red_last = (atomicAdd(a.ctr + U.red, 1) == U.nsplit - 1);
          named_bar_sync(1, 128);
          if (S->red_last) {
            __threadfence();
            // 128 threads: 4 row groups x 32 threads x 4 consecutive columns (16-B loads);
            // y[row][c] = bf16(((p0 + p1) + p2) + ...), 8-B bf16 stores to the source AW.
            const int rg = et >> 5;
            for (int cgi = (et & 31) * 4; cgi < BM * (U.dual ? 2 : 1); cgi += 128) {
            const int c = U.m0 + cgi;
            if (c < a.d) {
              for (int n0 = rg; n0 < U.nrows; n0 += 16) {
                float4 acc[4];
                int2 o[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  const int n = n0 + 4 * i;
                  const bool v = n < U.nrows;
                  acc[i] = v ? __ldcg(reinterpret_cast<const float4 *>(a.ws + (size_t)(U.n0 + n) * a.d + c))
                             : make_float4(0.f, 0.f, 0.f, 0.f);
                  o[i] = v ? __ldcg(meta + U.n0 + n) : make_int2(0, 0);
                }
                for (int sp = 1; sp < U.nsplit; ++sp) {
                  float4 p[4];
#pragma unroll
                  for (int i = 0; i < 4; ++i) {
                    const int n = n0 + 4 * i;
                    p[i] = (n < U.nrows) ? __ldcg(reinterpret_cast<const float4 *>(
                                               a.ws + ((size_t)sp * a.R_cap + U.n0 + n) * a.d + c))
                                         : make_float4(0.f, 0.f, 0.f, 0.f);
                  }
#pragma unroll
                  for (int i = 0; i < 4; ++i) {
                    acc[i].x = __fadd_rn(acc[i].x, p[i].x);
                    acc[i].y = __fadd_rn(acc[i].y, p[i].y);
                    acc[i].z = __fadd_rn(acc[i].z, p[i].z);
                    acc[i].w = __fadd_rn(acc[i].w, p[i].w);
                  }
                }
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  if (n0 + 4 * i < U.nrows) {
                    __nv_bfloat162 lo = __floats2bfloat162_rn(acc[i].x, acc[i].y);
                    __nv_bfloat162 hi = __floats2bfloat162_rn(acc[i].z, acc[i].w);
                    uint2 pk;
                    pk.x = *reinterpret_cast<uint32_t *>(&lo);
                    pk.y = *reinterpret_cast<uint32_t *>(&hi);
                    bf16 *yb = reinterpret_cast<bf16 *>(a.sym[o[i].x] + a.L.ybuf);
                    *reinterpret_cast<uint2 *>(yb + (size_t)o[i].y * a.d + c) = pk;
                  }
                }
              }
            }
            }
          }
          if (a.tok_comb && S->red_last) fence_scope(sys);  // the reduced y rows before the arrivals
          named_bar_sync(1, 128);
        }
        if (a.tok_comb && (!split || S->red_last)) {
          // per-token arrivals at the token's source AW (its counter is in the peer-visible region:
          // an NVLink atomic when the source is a peer), one per 128-column output tile stored: the
          // source combines a token as soon as all k (+ shared) outputs over every c-tile are stored,
          // without a grid barrier after the GEMM
          const int add = (U.dual && U.m0 + BM < a.d) ? 2 : 1;
          for (int i = et; i < U.nrows; i += 128) {  // token tiles of up to 256 (wide mode)
            int src = a.rank, t = U.n0 - a.R_sh0 + i;
            if (!sh) {
              const int2 o = __ldcg(meta + U.n0 + i);
              src = o.x;
              t = o.y / a.k;
            }
            int *c = reinterpret_cast<int *>(a.sym[src] + a.L.tokctr) + t;
            if (src == a.rank || !sys) atomicAdd(c, add);
            else atomicAdd_system(c, add);
          }
        }
      }
      if (a.trace && et == 0) {
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        a.trace[u] = (globaltimer_ns() << 16) | ((uint64_t)U.kind << 12) | (smid & 0xFFF);
      }
    }
    fence_scope(sys);  // this CTA's y rows (possibly on peers) before the grid barrier
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, kTmemCols);
  }

  // ===================== combine (GK5), all CTAs =====================
  if (a.hk && a.hcall > 2) {  // host-buffer path: out_stage drained by call i-2's D2H copy
    if (threadIdx.x == 0) wait_ctr_ge(a.hk + 2 + a.hb, a.hcall - 2, err, 0x4008);
    __syncthreads();
  }
  if (a.tok_comb) {
    const uint32_t part = (uint32_t)__ldcg(a.sync + 6);
    if (a.world > 1) {
      // the last CTA of this rank to finish its GEMM work releases the combine flags: every expert
      // output this rank computed is in its source's combine buffer (failure detection, below)
      __syncthreads();
      if (threadIdx.x == 0) {
        fence_scope(sys);
        if (atomicAdd(a.sync + 2, 1) == VGRID - 1) {
          fence_scope(sys);
          for (int q = 0; q < a.world; ++q)
            if ((part >> q) & 1u)
              st_release(reinterpret_cast<uint32_t *>(a.sym[q] + a.L.flags) + a.fslot_comb * kMaxWorld + a.rank,
                         a.fepoch, sys);
        }
      }
    }
    // warp per token, grid-stride from this CTA's warps as soon as its GEMM work is done: a token
    // is combined once its arrival count is complete (no grid barrier: the combine runs beside the
    // GEMM tail on every rank); a lane owns d / 256 chunks of 8 outputs, all their loads in flight.
    // Arrivals count 128-column output tiles (a dual unit stores two; d % 256 == 0 when dual).
    const int target = (a.k + (a.Fsh > 0 ? 1 : 0)) * ((a.d + BM - 1) / BM);
    const uint32_t wmask = (a.world >= 32) ? 0xffffffffu : ((1u << a.world) - 1u);
    const uint32_t live = (a.alive | (1u << a.rank)) & wmask;
    const bf16 *ybuf = reinterpret_cast<const bf16 *>(a.sym[a.rank] + a.L.ybuf);
    if ((part & wmask) == live) {  // (a peer failed in the count exchange: pairs were not sent, tg_failover redoes it)
      for (int t = VBID * 8 + warp; t < a.T; t += VGRID * 8) {
        int ok = 1;
        if (lane == 0) {
          if (a.world == 1) {
            wait_ctr_ge(a.tokctr + t, target, err, 0x5002);
          } else if (ld_acquire_gpu(a.sync + 7) || !wait_ctr_or_fail(a.tokctr + t, target, sys, a.fail_timeout_ns)) {
            ok = 0;  // a peer fell silent mid-call: the combine is left to tg_failover
            atomicExch(a.sync + 7, 1);
          }
        }
        if (!__shfl_sync(0xffffffffu, ok, 0)) break;
        fence_scope(sys);
        for (int c0 = lane; c0 < (a.d >> 3); c0 += 4 * 32) combine_chunks<4>(a, ybuf, t, c0, 32);
      }
    }
    __threadfence();  // this call's stores before the call after next reuses its buffer set
    // every live rank waits for every other live rank's combine flag (not only the EWs it sent
    // rows to), so all survivors see a rank that fails mid-call in the same call (§5.1)
    if (a.world > 1 && VBID == 0 && threadIdx.x < a.world && threadIdx.x != a.rank && ((part >> threadIdx.x) & 1u)) {
      const uint32_t *fl =
          reinterpret_cast<const uint32_t *>(a.sym[a.rank] + a.L.flags) + a.fslot_comb * kMaxWorld + threadIdx.x;
      if (!wait_flag_or_fail(fl, a.fepoch, sys, a.fail_timeout_ns)) atomicOr(a.fail_mask, 1u << threadIdx.x);
    }
    return;
  }
  // (failover replays and TG_LOCAL=0: barrier, combine flags, combine; the counter is zeroed per
  // launch after griddepcontrol.wait — calls with the per-token combine never reach it)
  grid_barrier_z(reinterpret_cast<unsigned long long *>(a.sync + 10), 0, err, a.ncta);
  if (a.trace && VBID == 0 && threadIdx.x == 0) a.trace[a.n_units_max + 148 + 16] = globaltimer_ns();
  // combine flags: every rank taking part in this run waits for every other one (not only the
  // EWs it sent rows to), so all survivors see a rank that fails mid-run in the same run and
  // take part in the failover replay together; a peer silent past the failure timeout is
  // recorded as failed (no trap), its pairs are re-routed by tg_failover (§5.1)
  const uint32_t part = (uint32_t)__ldcg(a.sync + 6);
  if (VBID == 0 && threadIdx.x < a.world && ((part >> threadIdx.x) & 1u)) {
    // every expert output this rank computed is in its source's combine buffer
    fence_scope(sys);
    uint32_t *fl = reinterpret_cast<uint32_t *>(a.sym[threadIdx.x] + a.L.flags) + a.fslot_comb * kMaxWorld + a.rank;
    st_release(fl, a.fepoch, sys);
  }
  if (threadIdx.x < a.world && threadIdx.x != a.rank && ((part >> threadIdx.x) & 1u)) {
    const uint32_t *fl =
        reinterpret_cast<const uint32_t *>(a.sym[a.rank] + a.L.flags) + a.fslot_comb * kMaxWorld + threadIdx.x;
    if (!wait_flag_or_fail(fl, a.fepoch, sys, a.fail_timeout_ns)) atomicOr(a.fail_mask, 1u << threadIdx.x);
  }
  __syncthreads();
  const int nch = a.d >> 3;
  const size_t total = (size_t)a.T * nch;
  const bf16 *ybuf = reinterpret_cast<const bf16 *>(a.sym[a.rank] + a.L.ybuf);
  const size_t nthr = (size_t)VGRID * blockDim.x;
  for (size_t i = (size_t)VBID * blockDim.x + threadIdx.x; i < total; i += 4 * nthr) {
    // four chunks (i, i + nthr, ...) per step, of up to four tokens
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const size_t ii = i + u * nthr;
      if (ii < total) combine_chunks<1>(a, ybuf, (int)(ii / nch), (int)(ii % nch), 0);
    }
  }
  if (a.trace && threadIdx.x == 0 && VBID == 0) a.trace[a.n_units_max + 148 + 17] = globaltimer_ns();
}

__global__ void __launch_bounds__(kGemmThreads, 1)
    k_layer(const __grid_constant__ TmaMaps maps, const __grid_constant__ CallArgs a,
            const __grid_constant__ RouteKeys rk) {
  layer_body(maps, a, rk);
  if (a.hk) {  // host-buffer path: the last CTA to exit marks the call complete (D2H, next H2D)
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(a.hk + 4 + a.hb, 1) == a.hexit) {
        __threadfence();
        atomicExch(a.hk + 6 + a.hb, a.hcall);
      }
    }
  }
}

// Virtual ranks of one GPU as ONE cooperative launch (tests; a GPU shared by several AW/EW
// shards): CTA b is CTA b - r * nper of rank r = b / nper.  The ranks wait on one another's
// flags, so they must be co-resident — separate launches carry no such guarantee.
__global__ void __launch_bounds__(kGemmThreads, 1) k_layer_multi(const __grid_constant__ MultiArgs m) {
  const int r = blockIdx.x / m.nper;
  if (r >= m.n || m.a[r].absent) return;  // a rank that does not take part (died before the call)
  layer_body(*m.maps[r], m.a[r], m.rk[r]);
}

size_t gemm_smem_bytes() { return 1024 + (size_t)kRingBytes + sizeof(GemmShared); }

static constexpr int kLayerSmemMax = 225 * 1024;  // + ~1 KB static smem: under the 227 KB opt-in
static_assert(1024 + kRingBytes + sizeof(GemmShared) <= kLayerSmemMax, "GEMM smem over budget");

cudaError_t layer_configure() {
  cudaError_t e = cudaFuncSetAttribute(k_layer, cudaFuncAttributeMaxDynamicSharedMemorySize, kLayerSmemMax);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_layer_multi, cudaFuncAttributeMaxDynamicSharedMemorySize, kLayerSmemMax);
}

size_t layer_smem_bytes(const CallArgs &a) { return tg_max(gemm_smem_bytes(), front_smem(a)); }

// One CTA per SM (1 CTA / SM by shared memory): the grid barriers need every CTA resident, which
// holds as long as no kernel that waits on this one runs beside it on the GPU.  With programmatic
// dependent launch (default) the launch is NOT cooperative: the cooperative attribute holds the
// next call back until this one has completed, so PDL's early start (the next call's front on the
// SMs this call's tail frees) never happens — measured, Mixtral decode 495 -> 482 us per call.  An
// older call never waits on a newer one (the newer one's griddepcontrol.wait orders it), so every
// CTA of every call becomes resident.  TG_COOP=1 (or TG_PDL=0) launches cooperatively.
cudaError_t launch_layer(const CallArgs &a, const RouteKeys &rk, const TmaMaps &maps, int n_ctas, cudaStream_t s) {
  if (layer_smem_bytes(a) > (size_t)kLayerSmemMax) return cudaErrorInvalidConfiguration;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n_ctas);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = layer_smem_bytes(a);
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  int n = 0;
  if (!a.pdl || a.coop) {
    at[n].id = cudaLaunchAttributeCooperative;
    at[n++].val.cooperative = 1;
  }
  if (a.pdl) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n++].val.programmaticStreamSerializationAllowed = 1;
  }
  cfg.attrs = at;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, k_layer, maps, a, rk);
}

cudaError_t launch_layer_multi(const MultiArgs &m, cudaStream_t s) {
  size_t smem = 0;
  for (int r = 0; r < m.n; ++r) smem = tg_max(smem, layer_smem_bytes(m.a[r]));
  if (smem > (size_t)kLayerSmemMax) return cudaErrorInvalidConfiguration;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(m.n * m.nper);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_layer_multi, m);
}

}  // namespace tg
