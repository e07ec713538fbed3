// tg_internal.h — device-side data layout shared by the host runtime and the
// kernels of libtarragon.so.  Not part of the C ABI (include/tarragon.h).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace tg {

typedef __nv_bfloat16 bf16;

constexpr int kMaxWorld = 8;
constexpr int kMaxExperts = 256;
constexpr int kMaxK = 8;
constexpr int kMaxKeys = 1024;      // world * S_max  (key = rank * S_max + bank slot)
constexpr int kRankBlock = 256;     // tokens per block of the rank kernel
constexpr int kNumBoxes = 16;       // token-tile heights 16, 32, ..., 256
constexpr int kMaxSlotsPerRank = 256;

// GEMM tiling: swap-AB, weights fill UMMA M = 128,
// tokens are UMMA N (16..bn), K staged 64 wide (one 128-B swizzle row).
// Two modes per call: narrow (bn = 128, 4 stages x 48 KB: decode) and wide
// (bn = 256, 3 stages x 64 KB: prefill, halves the L2 bytes per FLOP of the
// weight tiles).
constexpr int BM = 128;
constexpr int BK = 64;
constexpr int BN_MAX = 256;
constexpr int kStages = 8;                      // maximum ring depth (stage size set per call)
constexpr int kTileBytes = 16384;               // 128 rows x 128 B
constexpr int kRingBytes = 208 * 1024;          // stage ring: floor(208 KB / stage) stages (4 x 48 KB, 3 x 64 KB)
constexpr int BN_MAX_EPI = 256;                 // token-tile width bound of the GEMM2 epilogue table
constexpr int kSchedDepth = 8;
constexpr int kGemmThreads = 256;               // w0 TMA, w1 MMA, w2 TMEM, w4-7 epilogue
constexpr int kTmemCols = 512;                  // 2 accumulator buffers x 256 columns

// Resolved ERT snapshot, passed by value to the router (host-resolved per
// table/mask change): key[e] = rank * S_max + bank_slot.
struct RouteKeys {
  int32_t key[kMaxExperts];
};

enum UnitKind : int32_t { U_G1 = 0, U_G2 = 1, U_G1_SH = 2, U_G2_SH = 3 };

// One GEMM work unit: a 128-row weight tile x up to 128 token rows of one slot.
struct Unit {
  int32_t kind;    // UnitKind
  int32_t slot;    // local bank slot (routed) / 0 (shared)
  int32_t m0;      // first weight row of the tile (f for GEMM1, c for GEMM2)
  int32_t n0;      // first row in recv / H
  int32_t nrows;   // token rows in this tile (1..128)
  int32_t kb0;     // first 64-wide K block
  int32_t kb1;     // one past the last K block
  int32_t dep;     // GEMM1: counter to bump when done; GEMM2: counter to wait on
  int32_t red;     // GEMM2 split-K: reduction counter (-1 if no split)
  int32_t split;   // split index
  int32_t nsplit;  // number of splits
  int32_t dep_target;
  int32_t ntiles;  // token tiles of this slot (> 1: the weight tile is re-read, keep it in L2)
  int32_t dual;    // GEMM2: second W2 tile at rows m0 + 128 (accumulator at +128 columns)
};

struct TmaMaps {
  CUtensorMap w1, w3, w2;          // expert bank
  CUtensorMap w1s, w3s, w2s;       // shared expert
  CUtensorMap x[2][kNumBoxes];     // receive buffer of each buffer set, box rows 16*(i+1)
  CUtensorMap h[2][kNumBoxes];     // SwiGLU activations H of each set, box rows 16*(i+1)
  CUtensorMap hs[2][kNumBoxes];    // shared-expert activations of each set
};

// Peer-visible ("symmetric") region: same layout and size on every rank, one
// CUDA IPC handle per rank.  Offsets in bytes.  recv / meta / dup / ybuf / tokctr exist once per
// buffer set (two sets, used by alternate calls: consecutive calls overlap); a call's CallArgs
// carries the layout of its set.
struct SymLayout {
  size_t recv;      // bf16 [R_cap][d]            dispatched token rows
  size_t meta;      // int2 [R_cap]               origin (src rank, t*k + j)
  size_t dup;       // int32 [R_cap]              token dedup: recv row to copy this row from (-1: sent)
  size_t ybuf;      // bf16 [T_max][k][d]         expert outputs returned to this AW
  size_t cnt_all;   // int32 [3][world][nkeys]    all-gathered per-source counts (calls by parity, replays)
  size_t tokctr;    // int32 [T_max]              per-token arrival counters (EW epilogues add, AW combines)
  size_t flags;     // uint32 [6][kMaxWorld]      cnt / data / comb epoch flags; replay data / comb / cnt
  size_t total;
};
constexpr int FLAG_CNT = 0, FLAG_DATA = 1, FLAG_COMB = 2, FLAG_RDATA = 3, FLAG_RCOMB = 4, FLAG_RCNT = 5,
              kNumFlagKinds = 6;
constexpr int kCntBufReplay = 2;  // cnt_all buffer of failover replays (calls use 0 / 1 by parity)
constexpr int kLocalLayoutBlock = 4096;  // world == 1: default of CallArgs::layout_block
constexpr long kTokCombMaxArrivals = 48 * 1024;  // world > 1: per-token combine up to this many NVLink arrivals per rank

// Everything a call needs, by value (kernel parameter).
struct CallArgs {
  // shape
  int d, E, k, F, Fsh, world, rank, S_max, S_loc, nkeys, T_max, R_cap, R_sh0, nsplit;
  int E_r;               // router rows: E experts (+ 1 shared-gate row when shared_gate)
  int gate_mode;         // 0: softmax over the selected k; 1: softmax over all E, not renormalised
  int shared_gate;       // 1: shared expert scaled by sigmoid(x . wsg)
  int T;                 // tokens on this rank for this call
  uint32_t alive;        // bit r: rank r participates (fail-stopped ranks are never awaited or written)
  int bn;                // GEMM token-tile width of this call (the stage ring geometry follows from the plan)
  int g2dual;            // GEMM2 units cover two 128-row W2 tiles sharing one H tile (prefill-sized calls)
  uint32_t epoch;        // local kernel-run counter (grid barriers)
  uint32_t xepoch;       // cross-rank call counter (count flags, count parity): equal on every rank
  uint32_t fepoch;       // value of this run's count / data / combine flags (xepoch, or the replay counter)
  int fslot_data, fslot_comb, fslot_cnt;  // flag kinds of this run (FLAG_DATA/COMB/CNT, or FLAG_R*)
  int cnt_buf;           // cnt_all buffer of this run (xepoch & 1, or kCntBufReplay)
  // in-call failover (NEXT-1, §5.1)
  long long fail_timeout_ns;   // data / combine waits on peers: timeout -> peer failed (not a trap)
  long long cnt_timeout_ns;    // count-exchange waits on peers (host threads may be late): timeout -> failed
  uint32_t *fail_mask;         // host-mapped: bit q = peer q failed during a call
  int *unrec;                  // host-mapped: replayed pairs whose next route is not on this rank
  int replay;            // 1: re-dispatch pairs routed to failed ranks (key_old) to their next live candidate
  uint32_t failed;       // replay: ranks whose pairs are recomputed
  const int32_t *key_old;  // replay: the failed call's destination keys
  int inject_fail;       // fault injection (tests): stop after the dispatch, as a crash mid-call
  // inputs / outputs
  const bf16 *x;
  bf16 *out;
  const bf16 *wg;
  const bf16 *bank_w1, *bank_w3;  // expert bank (L2 prefetch of the first GEMM1 tiles)
  long long l2_prefetch_bytes;    // budget of that prefetch (0 = off)
  // per-call scratch (local)
  int32_t *idx;          // [T_max][k]
  float *w;              // [T_max][k]
  float *sgate;          // [T_max] shared-expert weight per token (shared_gate)
  int32_t *key;          // [T_max][k] destination key of each pair
  int32_t *lrank;        // [T_max][k] rank of the pair within its block and key
  float *logit_part;     // [ceil(T_max/32)][nkp][32][E] router partial logits
  int32_t *grp_ctr;      // [3][gmax] K-part arrival counters, set cbuf of this launch
  int32_t *chunk_ctr;    // [3][cmax]: [0] chunks ranked, [1 + c] groups of chunk c done
  int gmax, cmax;        // entries per set
  int cbuf;              // epoch % 3: the counter set of this launch (the set two launches ahead is
                         // reset after griddepcontrol.wait: launches overlap under PDL)
  int32_t *bcnt;         // [nblk_max][nkeys] per-block counts -> exclusive block bases
  int32_t *dbase;        // [nkeys] base row of this source in each (rank, slot)
  int32_t *dst_pos;      // [T_max][k]
  int32_t *gcounts;      // [nkeys] rows per (rank, slot) over all sources
  int32_t *need_src;     // [kMaxWorld] source sends rows to this rank
  int32_t *sent_to;      // [kMaxWorld] this rank sends rows to dest
  int32_t *slot_rows;    // [S_loc] M_s on this rank
  int64_t *stats;        // [nkeys]
  int32_t *sync;         // this call's buffer set: [0..4] counters (scheduler, CTAs done, dispatch blocks, -,
                         // dedup copies), [5] dedup on, [6] ranks taking part in this run (alive and heard
                         // from in the count exchange), [7] combine incomplete; u64 combine barrier at [10]
  int32_t *gsync;        // shared by all calls: u64 front grid barriers at [8], [12] (by launch parity);
                         // [16 + cbuf] router item counters
  int pset;              // buffer set of this call (call parity; a failover replay: the failed call's)
  float *logits;         // [T_max][E_r] router logits of the last call (parity export; nullptr = off)
  int32_t *ctr;          // [n_ctr_max] GEMM dependency / reduction counters, then rdy
  int n_ctr_max;
  int32_t *rdy;          // [n_grp_max] world == 1: rows of each token tile copied into recv
  int32_t *tokctr;       // [T_max] this rank's per-token arrival counters (peer-visible region: the EWs
                         // that store a token's outputs add to its count, over NVLink when remote)
  int n_ctr_all;         // ctr + rdy entries (reset together at the start of a call)
  int32_t *srcrow;       // [R_cap] world == 1: token of each received row
  int local_rows;        // world == 1: rows copied in row order beside the GEMM, per-tile counters
  int layout_block;      // world == 1: pairs up to which the exchange block lays out the call (decode)
  int tok_comb;          // per-token arrival counters, combine without a grid barrier (not in replays)
  int g2lag;             // GEMM2 units of slot s queued after the GEMM1 units of slot s + g2lag (0: after all GEMM1)
  // host-buffer path (tg_moe_layer_host): device words shared with the copy streams, which order
  // themselves with stream memory operations so no stream op sits between consecutive kernels
  // (the PDL overlap); null otherwise.  [0,1] x staged, [2,3] out drained, [4,5] exit counts,
  // [6,7] call complete — per staging buffer hb; values are host call numbers hcall (1-based)
  int *hk;
  int hcall, hb, hexit;
  int dev;               // development A/B switches (TG_DEV)
  int cta0, ncta;        // this rank's CTAs in the launch: [cta0, cta0 + ncta) (several virtual ranks
                         // of one GPU share one cooperative launch: tg_moe_layer_multi)
  int absent;            // virtual rank that does not take part in this launch (its CTAs exit)
  int32_t *n_units;      // [1] units of the last call (written by the GEMM, diagnostics)
  int n_units_max;       // capacity bound (trace sizing)
  int *err;              // host-mapped error word
  int pdl;               // programmatic dependent launch between consecutive calls
  int coop;              // cooperative launch attribute with PDL (TG_COOP=1; holds PDL's early start back)
  uint64_t *trace;       // optional GEMM trace: [n_units_max] (end_ns << 16 | smid), [gridDim] start_ns
  // GEMM buffers (local)
  bf16 *H;               // [R_cap][F]
  bf16 *Hs;              // [T_max][Fsh]
  float *ws;             // [nsplit][R_cap][d] split-K partials
  bf16 *ysh;             // [T_max][d] shared-expert output
  // symmetric region, own + peers
  uint8_t *sym[kMaxWorld];
  SymLayout L;
};

// A CTA's block index and the CTA count within its rank's grid (every device function that
// distributes work over the grid takes them from its CallArgs `a`).
#define VBID ((int)blockIdx.x - a.cta0)
#define VGRID (a.ncta)

constexpr int kMaxVirt = 4;  // virtual ranks per fused launch
struct MultiArgs {           // one cooperative launch over the virtual ranks of one GPU
  CallArgs a[kMaxVirt];
  RouteKeys rk[kMaxVirt];
  const TmaMaps *maps[kMaxVirt];  // device copies (TMA descriptors in global memory)
  int n, nper;                    // ranks, CTAs per rank
};

// Kernel launchers (tg_export.cu / tg_gemm.cu).  Return cudaGetLastError().
// the whole layer call: one cooperative launch of k_layer (front P1-P3, then
// dispatch || grouped GEMM, combine)
cudaError_t launch_layer(const CallArgs &a, const RouteKeys &rk, const TmaMaps &maps, int n_ctas, cudaStream_t s);
cudaError_t launch_layer_multi(const MultiArgs &m, cudaStream_t s);
cudaError_t launch_export_keys(const CallArgs &a, int n, int32_t *dst_rank, int32_t *dst_slot, cudaStream_t s);
cudaError_t layer_configure();
size_t gemm_smem_bytes();

}  // namespace tg
