// tg_kernels.cu — gate / rank / dispatch / combine kernels of the MoE round trip.
//
//   GK1 router   : fp32 router logits, top-k (lowest id on ties), softmax over
//                  the k selected, ERT resolve -> destination key per pair
//                  (§2.1; §4.2; §5.1).
//   GK2 rank     : stable per-(rank, slot) ranks of the pairs in token order,
//                  all-gather of per-source counts over NVLink, receive layout
//                  and the GEMM work list of this rank as EW (§2.2.1).
//   GK3 dispatch : 16-B vector copies of token rows into the destination
//                  rank's receive buffer (peer memory) + origin metadata
//                  (§4.2 "dispatches metadata and token embeddings").
//   GK5 combine  : out[t] = sum_j w[t,j] * y[t,j] (+ y_shared[t]) in fp32, fixed
//                  j order (§2.1 "aggregated via a weighted sum").
#include "tg_internal.h"
#include "tg_ptx.cuh"

namespace tg {

// =====================================================================  GK1
// One warp per token.  Logits: each lane accumulates 8-element chunks
// (lane + 32 i) of x . Wg[e] with fp32 FMA (bf16 products are exact in fp32),
// then a fixed butterfly reduction: deterministic and row-invariant.
__global__ void __launch_bounds__(256) k_router(const bf16 *__restrict__ x, const bf16 *__restrict__ wg, int T,
                                                int d, int E, int k, int32_t *__restrict__ idx,
                                                float *__restrict__ w, int32_t *__restrict__ keys,
                                                const __grid_constant__ RouteKeys rk) {
  __shared__ float logit_s[8][kMaxExperts];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = blockIdx.x * 8 + warp;
  if (t >= T) return;
  float *lg = logit_s[warp];
  const uint4 *xr = reinterpret_cast<const uint4 *>(x + (size_t)t * d);
  const int nch = d >> 3;  // 16-byte chunks per row
  for (int e0 = 0; e0 < E; e0 += 8) {
    float acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.f;
    for (int c = lane; c < nch; c += 32) {
      uint4 xv = __ldg(xr + c);
      const __nv_bfloat162 *xp = reinterpret_cast<const __nv_bfloat162 *>(&xv);
      float2 xf[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) xf[q] = __bfloat1622float2(xp[q]);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (e0 + i < E) {
          uint4 wv = __ldg(reinterpret_cast<const uint4 *>(wg + (size_t)(e0 + i) * d) + c);
          const __nv_bfloat162 *wp = reinterpret_cast<const __nv_bfloat162 *>(&wv);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            float2 wf = __bfloat1622float2(wp[q]);
            acc[i] = __fmaf_rn(xf[q].x, wf.x, acc[i]);
            acc[i] = __fmaf_rn(xf[q].y, wf.y, acc[i]);
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float v = acc[i];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0 && e0 + i < E) lg[e0 + i] = v;
    }
  }
  __syncwarp();
  // ---- top-k: k rounds of warp argmax on (value desc, id asc); -0 == +0 ties.
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
    for (int a = 1; a < k; ++a) {
      int ve = sel[a];
      float vv = sv[a];
      int b = a - 1;
      while (b >= 0 && sel[b] > ve) { sel[b + 1] = sel[b]; sv[b + 1] = sv[b]; --b; }
      sel[b + 1] = ve;
      sv[b + 1] = vv;
    }
    float m = sv[0];
    for (int j = 1; j < k; ++j) m = fmaxf(m, sv[j]);
    float z[kMaxK], Z = 0.f;
    for (int j = 0; j < k; ++j) { z[j] = expf(sv[j] - m); Z = Z + z[j]; }
    for (int j = 0; j < k; ++j) {
      idx[(size_t)t * k + j] = sel[j];
      w[(size_t)t * k + j] = __fdiv_rn(z[j], Z);
      keys[(size_t)t * k + j] = rk.key[sel[j]];
    }
  }
}

cudaError_t launch_router(const CallArgs &a, const RouteKeys &rk, cudaStream_t s) {
  if (a.T > 0) {
    dim3 grid((a.T + 7) / 8);
    k_router<<<grid, 256, 0, s>>>(a.x, a.wg, a.T, a.d, a.E, a.k, a.idx, a.w, a.key, rk);
  }
  return cudaGetLastError();
}

// =====================================================================  GK2
// Block b ranks its 256 tokens: rank of pair (t, j) among pairs of the block
// with the same key in ascending t (each token has at most one pair per key,
// because its k experts are distinct and map to distinct slots).  The last
// block to finish turns the per-block counts into bases, all-gathers this
// rank's per-(rank, slot) counts with every peer (one-sided stores + release
// flag), and builds this rank's receive layout and GEMM work list.
__device__ void build_work(const CallArgs &a, const int32_t *slot_rows, int32_t *s_tmp);

__global__ void __launch_bounds__(kRankBlock) k_rank(CallArgs a) {
  extern __shared__ int32_t sm[];
  const int nkeys = a.nkeys;
  const int wsz = max(8 * nkeys, 5 * (a.S_loc + 2) + 8);
  int32_t *wcnt = sm;                      // [8][nkeys] (reused by build_work)
  int32_t *skey = sm + wsz;                // [256][k]
  int32_t *gsum = skey + kRankBlock * a.k; // [nkeys]
  __shared__ int s_last;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int t = blockIdx.x * kRankBlock + tid;
  const int k = a.k;
  for (int i = tid; i < 8 * nkeys; i += kRankBlock) wcnt[i] = 0;
  int mykey[kMaxK];
  for (int j = 0; j < k; ++j) {
    mykey[j] = (t < a.T) ? a.key[(size_t)t * k + j] : -1;
    skey[tid * k + j] = mykey[j];
  }
  __syncthreads();
  int wr[kMaxK];
  for (int j = 0; j < k; ++j) {
    int K = mykey[j];
    int r = 0;
    if (K >= 0) {
      for (int l = 0; l < lane; ++l) {
        const int32_t *o = skey + (warp * 32 + l) * k;
        for (int jj = 0; jj < k; ++jj) r += (o[jj] == K);
      }
      atomicAdd(&wcnt[warp * nkeys + K], 1);
    }
    wr[j] = r;
  }
  __syncthreads();
  for (int j = 0; j < k; ++j) {
    int K = mykey[j];
    if (K >= 0) {
      int r = wr[j];
      for (int ww = 0; ww < warp; ++ww) r += wcnt[ww * nkeys + K];
      a.lrank[(size_t)t * k + j] = r;
    }
  }
  for (int K = tid; K < nkeys; K += kRankBlock) {
    int c = 0;
    for (int ww = 0; ww < 8; ++ww) c += wcnt[ww * nkeys + K];
    a.bcnt[(size_t)blockIdx.x * nkeys + K] = c;
  }
  // ---- last block
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = (atomicAdd(&a.sync[0], 1) == (int)gridDim.x - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (tid == 0) a.sync[0] = 0;
  const int nblk = gridDim.x;
  const int par = a.epoch & 1;
  // exclusive prefix over blocks per key; totals -> wcnt[0][K]
  for (int K = tid; K < nkeys; K += kRankBlock) {
    int run = 0;
    for (int b = 0; b < nblk; ++b) {
      int c = __ldcg(a.bcnt + (size_t)b * nkeys + K);
      a.bcnt[(size_t)b * nkeys + K] = run;
      run += c;
    }
    wcnt[K] = run;
    a.stats[K] += run;
  }
  __syncthreads();
  // ---- all-gather counts: my row -> cnt_all[par][rank][*] on every peer
  for (int q = 0; q < a.world; ++q) {
    int32_t *dst = reinterpret_cast<int32_t *>(a.sym[q] + a.L.cnt_all) + ((size_t)par * a.world + a.rank) * nkeys;
    for (int K = tid; K < nkeys; K += kRankBlock) dst[K] = wcnt[K];
  }
  __threadfence_system();
  __syncthreads();
  if (tid < a.world) {
    uint32_t *fl = reinterpret_cast<uint32_t *>(a.sym[tid] + a.L.flags) + FLAG_CNT * kMaxWorld + a.rank;
    st_release_sys(fl, a.epoch);
  }
  if (tid < a.world) {
    const uint32_t *fl = reinterpret_cast<const uint32_t *>(a.sym[a.rank] + a.L.flags) + FLAG_CNT * kMaxWorld + tid;
    wait_flag_ge(fl, a.epoch, a.err, 0x2001);
  }
  __syncthreads();
  const int32_t *A = reinterpret_cast<const int32_t *>(a.sym[a.rank] + a.L.cnt_all) + (size_t)par * a.world * nkeys;
  // gcounts[K] = sum over sources; dbase[K] = slot base on its rank + rows of lower sources
  for (int K = tid; K < nkeys; K += kRankBlock) {
    int g = 0, below = 0;
    for (int src = 0; src < a.world; ++src) {
      int c = __ldcg(A + (size_t)src * nkeys + K);
      if (src < a.rank) below += c;
      g += c;
    }
    gsum[K] = g;
    a.gcounts[K] = g;
    wcnt[nkeys + K] = below;  // temp in wcnt[1][*]
  }
  __syncthreads();
  for (int K = tid; K < nkeys; K += kRankBlock) {
    int q = K / a.S_max, s = K % a.S_max;
    int off = 0;
    for (int s2 = 0; s2 < s; ++s2) off += gsum[q * a.S_max + s2];
    a.dbase[K] = off + wcnt[nkeys + K];
  }
  if (tid < a.world) {
    int rows_to_me = 0, rows_to_q = 0;
    for (int s = 0; s < a.S_max; ++s) {
      rows_to_me += __ldcg(A + (size_t)tid * nkeys + a.rank * a.S_max + s);
      rows_to_q += wcnt[tid * a.S_max + s];
    }
    a.need_src[tid] = rows_to_me > 0;
    a.sent_to[tid] = rows_to_q > 0;
  }
  for (int s = tid; s < a.S_loc; s += kRankBlock) a.slot_rows[s] = gsum[a.rank * a.S_max + s];
  __syncthreads();
  build_work(a, a.slot_rows, wcnt);
}

// GEMM work list of this rank (EW role).  Units are ordered GEMM1 (slot, f-tile,
// n-tile) then GEMM2 (slot, c-tile, n-tile, split); shared-expert units last in
// each phase.  Counters: one per (slot, n-tile) group for the GEMM1 -> GEMM2
// dependency, one per (slot, c-tile, n-tile) for split-K reduction.
__device__ void build_work(const CallArgs &a, const int32_t *slot_rows, int32_t *s_tmp) {
  const int tid = threadIdx.x;
  const int ftiles = (a.F + BM - 1) / BM, ctiles = (a.d + BM - 1) / BM;
  const int S = a.S_loc;
  const int nsh = (a.Fsh > 0) ? 1 : 0;
  // per "slot" (routed slots, then the shared pseudo-slot): n-tiles
  int32_t *nt = s_tmp;                  // [S+1]
  int32_t *g1off = s_tmp + (S + 1);     // [S+2] unit offsets
  int32_t *g2off = s_tmp + 2 * (S + 2); // [S+2]
  int32_t *goff = s_tmp + 3 * (S + 2);  // [S+2] dependency-group offsets
  int32_t *roff = s_tmp + 4 * (S + 2);  // [S+2] reduction-group offsets
  const int ftiles_sh = nsh ? (a.Fsh + BM - 1) / BM : 0;
  for (int s = tid; s < S + nsh; s += blockDim.x) {
    int rows = (s < S) ? slot_rows[s] : a.T;
    nt[s] = (rows + BN_MAX - 1) / BN_MAX;
  }
  __syncthreads();
  if (tid == 0) {
    int u1 = 0, u2 = 0, g = 0, r = 0;
    for (int s = 0; s < S + nsh; ++s) {
      bool sh = (s == S);
      int ns = sh ? 1 : a.nsplit;
      g1off[s] = u1;
      g2off[s] = u2;
      goff[s] = g;
      roff[s] = r;
      u1 += nt[s] * (sh ? ftiles_sh : ftiles);
      u2 += nt[s] * ctiles * ns;
      g += nt[s];
      r += (ns > 1) ? nt[s] * ctiles : 0;
    }
    g1off[S + nsh] = u1;
    g2off[S + nsh] = u2;
    goff[S + nsh] = g;
    roff[S + nsh] = r;
    int total = u1 + u2;
    if (total > a.n_units_max || g + r > a.n_ctr_max) {
      atomicExch(a.err, 0x2002);
      total = 0;
    }
    *a.n_units = total;
    a.sync[1] = 0;  // scheduler
    a.sync[2] = 0;  // GEMM CTAs done
    a.sync[3] = 0;  // dispatch blocks done
  }
  __syncthreads();
  const int G1 = g1off[S + nsh];
  const int nctr = goff[S + nsh] + roff[S + nsh];
  for (int i = tid; i < nctr && i < a.n_ctr_max; i += blockDim.x) a.ctr[i] = 0;
  // row offsets of routed slots in recv: prefix of slot_rows
  for (int s = tid; s < S + nsh; s += blockDim.x) {
    bool sh = (s == S);
    int rowoff = 0;
    if (!sh)
      for (int s2 = 0; s2 < s; ++s2) rowoff += slot_rows[s2];
    int rows = sh ? a.T : slot_rows[s];
    int base_row = sh ? a.R_sh0 : rowoff;
    int ft = sh ? ftiles_sh : ftiles;
    int Fw = sh ? a.Fsh : a.F;
    int ns = sh ? 1 : a.nsplit;
    int kbF = Fw / BK;
    int u = g1off[s];
    for (int f = 0; f < ft; ++f)
      for (int n = 0; n < nt[s]; ++n) {
        Unit U;
        U.kind = sh ? U_G1_SH : U_G1;
        U.slot = sh ? 0 : s;
        U.m0 = f * BM;
        U.n0 = base_row + n * BN_MAX;
        U.nrows = min(BN_MAX, rows - n * BN_MAX);
        U.kb0 = 0;
        U.kb1 = a.d / BK;
        U.dep = goff[s] + n;
        U.red = -1;
        U.split = 0;
        U.nsplit = 1;
        U.dep_target = 0;
        a.units[u++] = U;
      }
    u = G1 + g2off[s];
    for (int c = 0; c < ctiles; ++c)
      for (int n = 0; n < nt[s]; ++n)
        for (int sp = 0; sp < ns; ++sp) {
          Unit U;
          U.kind = sh ? U_G2_SH : U_G2;
          U.slot = sh ? 0 : s;
          U.m0 = c * BM;
          U.n0 = base_row + n * BN_MAX;
          U.nrows = min(BN_MAX, rows - n * BN_MAX);
          U.kb0 = sp * (kbF / ns);
          U.kb1 = (sp + 1) * (kbF / ns);
          U.dep = goff[s] + n;
          U.dep_target = ft;
          U.red = (ns > 1) ? goff[S + nsh] + roff[s] + c * nt[s] + n : -1;
          U.split = sp;
          U.nsplit = ns;
          a.units[u++] = U;
        }
  }
}

cudaError_t launch_rank(const CallArgs &a, cudaStream_t s) {
  int nblk = a.T > 0 ? (a.T + kRankBlock - 1) / kRankBlock : 1;
  const int wsz = max(8 * a.nkeys, 5 * (a.S_loc + 2) + 8);
  size_t smem = sizeof(int32_t) * (size_t)(wsz + kRankBlock * a.k + a.nkeys);
  k_rank<<<nblk, kRankBlock, smem, s>>>(a);
  return cudaGetLastError();
}

// =====================================================================  GK3
// One warp per (token, j) pair: 16-B vector copy of the x row into
// recv[pos] on rank q (NVLink store when q != me) and its origin metadata.
// With a shared expert, x rows are also staged at recv[R_sh0 + t] (local).
__global__ void __launch_bounds__(256) k_dispatch(CallArgs a) {
  __shared__ int s_last;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int k = a.k;
  const int nch = a.d >> 3;
  const int npairs = a.T * k;
  const int nsh = (a.Fsh > 0) ? a.T : 0;
  for (int p = warp; p < npairs + nsh; p += nwarps) {
    if (p < npairs) {
      int t = p / k;
      int K = a.key[p];
      int q = K / a.S_max;
      int pos = a.dbase[K] + a.bcnt[(size_t)(t / kRankBlock) * a.nkeys + K] + a.lrank[p];
      const uint4 *src = reinterpret_cast<const uint4 *>(a.x + (size_t)t * a.d);
      uint4 *dst = reinterpret_cast<uint4 *>(a.sym[q] + a.L.recv) + (size_t)pos * nch;
      for (int c = lane; c < nch; c += 32) dst[c] = __ldg(src + c);
      if (lane == 0) {
        int2 *meta = reinterpret_cast<int2 *>(a.sym[q] + a.L.meta);
        meta[pos] = make_int2(a.rank, p);
        a.dst_pos[p] = pos;
      }
    } else {
      int t = p - npairs;
      const uint4 *src = reinterpret_cast<const uint4 *>(a.x + (size_t)t * a.d);
      uint4 *dst = reinterpret_cast<uint4 *>(a.sym[a.rank] + a.L.recv) + (size_t)(a.R_sh0 + t) * nch;
      for (int c = lane; c < nch; c += 32) dst[c] = __ldg(src + c);
    }
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(&a.sync[3], 1) == (int)gridDim.x - 1);
  __syncthreads();
  if (s_last && threadIdx.x < a.world) {
    __threadfence_system();
    uint32_t *fl = reinterpret_cast<uint32_t *>(a.sym[threadIdx.x] + a.L.flags) + FLAG_DATA * kMaxWorld + a.rank;
    st_release_sys(fl, a.epoch);
  }
}

cudaError_t launch_dispatch(const CallArgs &a, cudaStream_t s) {
  int npairs = a.T * a.k + ((a.Fsh > 0) ? a.T : 0);
  int blocks = (npairs + 7) / 8;
  if (blocks < 1) blocks = 1;
  if (blocks > 1184) blocks = 1184;
  k_dispatch<<<blocks, 256, 0, s>>>(a);
  return cudaGetLastError();
}

// =====================================================================  GK5
// Each thread: 8 consecutive columns of one token.  acc = sum_j w_j * y_j in
// fp32, j = 0..k-1 in order, then + y_shared; one RNE rounding to bf16.
__global__ void __launch_bounds__(256) k_combine(CallArgs a) {
  if (threadIdx.x < a.world) {
    if (a.sent_to[threadIdx.x]) {
      const uint32_t *fl =
          reinterpret_cast<const uint32_t *>(a.sym[a.rank] + a.L.flags) + FLAG_COMB * kMaxWorld + threadIdx.x;
      wait_flag_ge(fl, a.epoch, a.err, 0x5001);
    }
  }
  __syncthreads();
  const int nch = a.d >> 3;
  const size_t total = (size_t)a.T * nch;
  const bf16 *ybuf = reinterpret_cast<const bf16 *>(a.sym[a.rank] + a.L.ybuf);
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int t = (int)(i / nch), c8 = (int)(i % nch);
    float acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.f;
    for (int j = 0; j < a.k; ++j) {
      const float wj = a.w[(size_t)t * a.k + j];
      uint4 v = __ldcg(reinterpret_cast<const uint4 *>(ybuf + ((size_t)t * a.k + j) * a.d) + c8);
      const __nv_bfloat162 *vp = reinterpret_cast<const __nv_bfloat162 *>(&v);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float2 f = __bfloat1622float2(vp[q]);
        acc[2 * q] = __fmaf_rn(wj, f.x, acc[2 * q]);
        acc[2 * q + 1] = __fmaf_rn(wj, f.y, acc[2 * q + 1]);
      }
    }
    if (a.Fsh > 0) {
      uint4 v = __ldcg(reinterpret_cast<const uint4 *>(a.ysh + (size_t)t * a.d) + c8);
      const __nv_bfloat162 *vp = reinterpret_cast<const __nv_bfloat162 *>(&v);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float2 f = __bfloat1622float2(vp[q]);
        acc[2 * q] = __fadd_rn(acc[2 * q], f.x);
        acc[2 * q + 1] = __fadd_rn(acc[2 * q + 1], f.y);
      }
    }
    uint4 o;
    __nv_bfloat162 *op = reinterpret_cast<__nv_bfloat162 *>(&o);
#pragma unroll
    for (int q = 0; q < 4; ++q) op[q] = __floats2bfloat162_rn(acc[2 * q], acc[2 * q + 1]);
    reinterpret_cast<uint4 *>(a.out + (size_t)t * a.d)[c8] = o;
  }
}

cudaError_t launch_combine(const CallArgs &a, cudaStream_t s) {
  size_t total = (size_t)a.T * (a.d >> 3);
  int blocks = (int)((total + 255) / 256);
  if (blocks < 1) blocks = 1;
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_combine<<<blocks, 256, 0, s>>>(a);
  return cudaGetLastError();
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
