// tarragon.cu — host runtime of libtarragon.so: the C ABI of include/tarragon.h.
//
// Host-side state per ctx: the layer's expert bank (HBM), the Expert Routing
// Table with its version and the EW mask (§4.2, §5.1), the
// resolved expert -> (rank, bank slot) snapshot handed to the router kernel at
// each call (so a table flip or a mask takes effect at the next call with no
// re-initialisation), peer mappings of every rank's receive/combine buffers
// (CUDA IPC over NVLink), and the per-call launch sequence GK1..GK5.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/tarragon.h"
#include "tg_internal.h"

using namespace tg;

namespace {

thread_local std::string g_init_error = "no error";

typedef CUresult (*PFN_encodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                    const cuuint64_t *, const cuuint32_t *, const cuuint32_t *,
                                    CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                    CUtensorMapFloatOOBfill);

PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  }
  return fn;
}

typedef CUresult (*PFN_streamValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
PFN_streamValue32 get_stream_op(const char *name) {
  void *p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess)
    return reinterpret_cast<PFN_streamValue32>(p);
  return nullptr;
}

}  // namespace

struct tg_ctx {
  // ---- config
  int d, E, k, F, Fsh, W, spe, T_max;
  int gate_mode = 0, shared_gate = 0;
  bool sgate_loaded = false;
  int rank, world, device;
  std::vector<int32_t> ew_rank, ew_base;  // per EW: rank, first bank slot on its rank
  std::vector<int> S_of_rank;             // bank slots per rank
  int S_max = 0, S_loc = 0, nkeys = 0;
  int R_cap = 0, R_sh0 = 0, R_tot = 0, nsplit = 1;
  // ---- routing state (host)
  std::vector<int32_t> hosted;            // [W][spe] expert id, -1 empty
  std::vector<int32_t> cand;              // [E][C][2]
  int C = 0;
  uint64_t version = 0;
  bool have_table = false;
  std::vector<uint8_t> mask;              // [W]
  uint32_t alive = 0xffffffffu;           // bit r: rank r alive (tg_mask_rank)
  std::vector<int32_t> rkey;              // [E] resolved key or -1
  bool no_route = true;
  bool gate_loaded = false, shared_loaded = false;
  // ---- device
  bool host_only = true;
  int n_sms = 148;
  bool stage_export = false;              // parity export of the router logits (tg_set_stage_export)
  float *logits = nullptr;                // [T_max][E_r]
  bf16 *bank_w1 = nullptr, *bank_w3 = nullptr, *bank_w2 = nullptr, *wg = nullptr;
  bf16 *w1s = nullptr, *w3s = nullptr, *w2s = nullptr;
  uint8_t *sym = nullptr;                 // own symmetric region
  SymLayout L{};
  uint8_t *peer[kMaxWorld] = {nullptr};
  bool peer_opened[kMaxWorld] = {false};
  void *scratch = nullptr;
  CallArgs args{};
  TmaMaps maps{};
  TmaMaps *maps_dev = nullptr;            // device copy (fused launches of virtual ranks)
  // Two buffer sets used by alternate calls: call n+1 runs its front, dispatch and GEMM units on
  // the SMs call n's tail frees (PDL, no griddepcontrol.wait), so nothing call n still uses may be
  // touched by call n+1.  Call n-1, the last user of call n+1's set, has exited by then: a call
  // triggers its dependents after its front's grid barrier, when all its CTAs (one per SM) are
  // resident, i.e. when no CTA of the call before it is left.
  struct SetState {
    SymLayout L;
    bf16 *H = nullptr, *Hs = nullptr, *ysh = nullptr;
    float *ws = nullptr;
    int32_t *ctr = nullptr, *srcrow = nullptr, *slot_rows = nullptr, *dbase = nullptr, *gcounts = nullptr,
            *need_src = nullptr, *sent_to = nullptr, *sync = nullptr;
  } set[2];
  int last_set = 0;
  int *err_host = nullptr, *err_dev = nullptr;
  uint64_t *trace = nullptr;                     // device trace buffer (diagnostics)
  bool tracing = false;
  int force_mode = -1;                           // TG_WIDE=0/1 (development A/B), -1 auto
  int force_dual = -1;                           // TG_G2DUAL=0/1 (development A/B), -1 auto
  bf16 *x_stage[2] = {nullptr, nullptr}, *out_stage[2] = {nullptr, nullptr};  // tg_moe_layer_host, double-buffered
  cudaStream_t hs_h2d = nullptr, hs_d2h = nullptr;  // host-path copy streams (overlap with the layer)
  cudaEvent_t ev_h2d[2] = {}, ev_k[2] = {}, ev_d2h[2] = {}, ev_sync = nullptr, ev_sync2 = nullptr;
  long long host_calls = 0;
  int *hk_dev = nullptr;                          // host-path device words (CallArgs::hk)
  PFN_streamValue32 wait32 = nullptr, write32 = nullptr;
  bool pend_host = false;                         // the next launch is host call host_calls
  uint32_t epoch = 0;    // local kernel runs
  uint32_t xepoch = 0;   // calls (equal on every rank)
  uint32_t rxepoch = 0;  // failover replays (equal on every surviving rank)
  int32_t *key_main = nullptr, *key_replay = nullptr;
  long long fail_timeout_ns = 200000000LL;  // in-call failure detection on data / combine flags
  long long cnt_timeout_ns = 2000000000LL;  // count-exchange waits (10 x the failure timeout, <= 4 s)
  bool inject_next = false;                 // fault injection for tests (tg_inject_failure)
  // KV checkpoint store (NEXT-4): pinned host bucket written by the copy engines
  uint8_t *kv_bucket = nullptr;
  size_t kv_bytes = 0;
  cudaStream_t kv_stream = nullptr;
  cudaEvent_t kv_ev = nullptr;
  volatile uint64_t kv_committed = 0;
  static constexpr int kKvRecs = 4096;
  struct KvRec { tg_ctx *c; uint64_t seq; } kv_rec[kKvRecs];
  int kv_next = 0;
  int last_T = 0;
  float *w_buf[2] = {nullptr, nullptr}, *sg_buf[2] = {nullptr, nullptr};  // by call parity
  int last_wb = 0;                                                        // parity of the last call
  int last_launches = 0;
  bool sticky = false;
  // profiling
  // profiling: 2 events per call (around the one launch), ring of kProfCalls calls, no host sync per call
  static constexpr int kProfCalls = 512, kEv = 2;
  bool prof = false;
  std::vector<cudaEvent_t> ev;
  int n_ev = 0;        // events recorded in the current call
  int prof_calls = 0;  // calls recorded since tg_set_profiling(1)
  std::string errmsg = "no error";
};

static tg_status fail(tg_ctx *c, tg_status s, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->errmsg = buf; else g_init_error = buf;
  if (c && s == TG_ERR_CUDA) c->sticky = true;
  return s;
}

#define CK2(ctx, call)                                                                               \
  do {                                                                                               \
    cudaError_t e_ = (call);                                                                         \
    if (e_ != cudaSuccess) return fail(ctx, TG_ERR_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                                       __FILE__, __LINE__);                                          \
  } while (0)

#define CK(call)                                                                                     \
  do {                                                                                               \
    cudaError_t e_ = (call);                                                                         \
    if (e_ != cudaSuccess) return fail(c, TG_ERR_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                                       __FILE__, __LINE__);                                          \
  } while (0)

static tg_status check_sticky(tg_ctx *c) {
  if (c->sticky) return TG_ERR_CUDA;
  if (c->err_host && *reinterpret_cast<volatile int *>(c->err_host) != 0)
    return fail(c, TG_ERR_CUDA, "device-side error code 0x%x (timeout or capacity)", *c->err_host);
  return TG_OK;
}

// ------------------------------------------------------------------ resolve
// First unmasked candidate ("first healthy").  key = rank*S_max+slot.
static void resolve(tg_ctx *c) {
  c->rkey.assign(c->E, -1);
  c->no_route = !c->have_table;
  if (!c->have_table) return;
  for (int e = 0; e < c->E; ++e) {
    for (int j = 0; j < c->C; ++j) {
      int ew = c->cand[(e * c->C + j) * 2], sl = c->cand[(e * c->C + j) * 2 + 1];
      if (ew < 0 || c->mask[ew]) continue;
      c->rkey[e] = c->ew_rank[ew] * c->S_max + c->ew_base[ew] + sl;
      break;
    }
    if (c->rkey[e] < 0) c->no_route = true;
  }
}

// Point a call's arguments at buffer set st (peer-visible layout and local scratch of the set).
static void apply_set(tg_ctx *c, CallArgs *a, int st) {
  const tg_ctx::SetState &S = c->set[st];
  a->pset = st;
  a->L = S.L;
  a->H = S.H; a->Hs = S.Hs; a->ysh = S.ysh; a->ws = S.ws;
  a->ctr = S.ctr; a->rdy = S.ctr + a->n_ctr_max; a->srcrow = S.srcrow; a->slot_rows = S.slot_rows;
  a->dbase = S.dbase; a->gcounts = S.gcounts; a->need_src = S.need_src; a->sent_to = S.sent_to; a->sync = S.sync;
  a->tokctr = c->sym ? reinterpret_cast<int32_t *>(c->sym + S.L.tokctr) : nullptr;
}

static tg_status make_map(tg_ctx *c, CUtensorMap *m, void *base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return fail(c, TG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(c, TG_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d) rows=%llu cols=%llu box=%u",
                                     (int)r, (unsigned long long)rows, (unsigned long long)cols, box_rows);
  return TG_OK;
}

static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

extern "C" {

tg_status tg_init(const tg_config *cfg, int rank, int world, int cuda_device, tg_ctx **out) {
  tg_ctx *c = nullptr;
  if (!cfg || !out) return fail(nullptr, TG_ERR_INVALID, "null config or out pointer");
  *out = nullptr;
  const int d = cfg->d_model, E = cfg->n_experts, k = cfg->top_k, F = cfg->d_ffn, Fsh = cfg->d_ffn_shared;
  if (d <= 0 || d % 64 || F <= 0 || F % 64 || Fsh < 0 || Fsh % 64 || E < 1 || E > kMaxExperts || k < 1 ||
      k > E || k > kMaxK)
    return fail(nullptr, TG_ERR_INVALID, "shape: need d,F,F_sh %% 64 == 0, 1 <= k <= min(E,8), E <= 256 "
                                         "(d=%d F=%d F_sh=%d E=%d k=%d)", d, F, Fsh, E, k);
  if (world < 1 || world > kMaxWorld || rank < 0 || rank >= world)
    return fail(nullptr, TG_ERR_INVALID, "rank %d / world %d (world <= %d)", rank, world, kMaxWorld);
  if (cfg->n_ews < 1 || !cfg->ew_rank || cfg->slots_per_ew < 1 || cfg->max_tokens_per_rank < 0)
    return fail(nullptr, TG_ERR_INVALID, "placement: n_ews, ew_rank, slots_per_ew, max_tokens_per_rank");
  if (cfg->gate_mode < 0 || cfg->gate_mode > 1 || cfg->shared_gate < 0 || cfg->shared_gate > 1 ||
      (cfg->shared_gate && Fsh == 0) || (cfg->shared_gate && E + 1 > kMaxExperts))
    return fail(nullptr, TG_ERR_INVALID, "gate_mode must be 0/1; shared_gate 0/1 and needs d_ffn_shared > 0");
  c = new tg_ctx();
  c->d = d; c->E = E; c->k = k; c->F = F; c->Fsh = Fsh;
  c->gate_mode = cfg->gate_mode; c->shared_gate = cfg->shared_gate;
  c->W = cfg->n_ews; c->spe = cfg->slots_per_ew; c->T_max = cfg->max_tokens_per_rank;
  c->rank = rank; c->world = world; c->device = cuda_device;
  c->ew_rank.assign(cfg->ew_rank, cfg->ew_rank + c->W);
  c->S_of_rank.assign(world, 0);
  c->ew_base.resize(c->W);
  for (int w = 0; w < c->W; ++w) {
    int r = c->ew_rank[w];
    if (r < 0 || r >= world) { delete c; return fail(nullptr, TG_ERR_INVALID, "ew_rank[%d] = %d out of range", w, r); }
    c->ew_base[w] = c->S_of_rank[r];
    c->S_of_rank[r] += c->spe;
  }
  for (int r = 0; r < world; ++r) c->S_max = std::max(c->S_max, c->S_of_rank[r]);
  c->S_loc = c->S_of_rank[rank];
  c->nkeys = world * c->S_max;
  if (c->S_loc > kMaxSlotsPerRank) { delete c; return fail(nullptr, TG_ERR_INVALID, "%d slots on rank %d > %d", c->S_loc, rank, kMaxSlotsPerRank); }
  if (c->nkeys > kMaxKeys) { delete c; return fail(nullptr, TG_ERR_INVALID, "world * slots per rank = %d > %d", c->nkeys, kMaxKeys); }
  c->hosted.assign((size_t)c->W * c->spe, -1);
  c->mask.assign(c->W, 0);
  c->rkey.assign(E, -1);
  // worst-case rows received by one rank: every token of every rank, at most
  // min(k, S_max) rows each (distinct experts -> distinct slots).  Sized from global
  // values only, so the peer-visible region has the same layout on every rank
  // (checked at connect time): senders store into a peer at their own offsets.
  c->R_cap = world * c->T_max * std::min(k, std::max(c->S_max, 1));
  c->R_sh0 = c->R_cap;
  c->R_tot = c->R_cap + (Fsh > 0 ? c->T_max : 0);
  // fixed split-K for long GEMM2 reductions: a function of the shape only, so outputs are bitwise
  // equal at every GPU count (P7).  Same-box A/B at Mixtral decode, F = 14336, us per call, 2 vs 4
  // splits, with early start: 1 GPU 475.3 vs 482.8, 2 GPUs 257.6 vs 265.6, 4 GPUs 161.4 vs 165.4
  // (before early start at world > 1, 4 splits won there — 4 GPUs 207.4 vs 189.8 — as the last
  // GEMM2 wave of a rank serving 2 experts idled most SMs; now the next call's GEMM fills that
  // tail).  1 split leaves 140-us units for the last wave.
  c->nsplit = (F / BK >= 128 && (F / BK) % 2 == 0) ? 2 : 1;
  if (const char *ns = getenv("TG_NSPLIT")) {  // development override (A/B timing)
    const int v = atoi(ns);
    if (v >= 1 && v <= 16 && (F / BK) % v == 0) c->nsplit = v;
  }
  if (cuda_device < 0) { *out = c; return TG_OK; }

  // ---------------------------------------------------------------- device
  c->host_only = false;
  auto bail = [&](tg_status s) { g_init_error = c->errmsg; tg_finalize(c); return s; };
#define CKI(call)                                                                                 \
  do {                                                                                            \
    cudaError_t e_ = (call);                                                                      \
    if (e_ != cudaSuccess) {                                                                      \
      fail(c, e_ == cudaErrorMemoryAllocation ? TG_ERR_OOM : TG_ERR_CUDA, "%s: %s", #call,        \
           cudaGetErrorString(e_));                                                               \
      return bail(e_ == cudaErrorMemoryAllocation ? TG_ERR_OOM : TG_ERR_CUDA);                    \
    }                                                                                             \
  } while (0)
  CKI(cudaSetDevice(cuda_device));
  cudaDeviceProp prop;
  CKI(cudaGetDeviceProperties(&prop, cuda_device));
  if (prop.major != 10) {
    fail(c, TG_ERR_UNSUPPORTED, "device %d is sm_%d%d; libtarragon is built for sm_100a only", cuda_device,
         prop.major, prop.minor);
    return bail(TG_ERR_UNSUPPORTED);
  }
  c->n_sms = prop.multiProcessorCount;
  const size_t S_loc = std::max(c->S_loc, 1);
  CKI(cudaMalloc(&c->bank_w1, S_loc * F * d * 2));
  CKI(cudaMalloc(&c->bank_w3, S_loc * F * d * 2));
  CKI(cudaMalloc(&c->bank_w2, S_loc * F * d * 2));
  CKI(cudaMalloc(&c->wg, (size_t)(E + 1) * d * 2));  // + shared-gate row
  if (Fsh > 0) {
    CKI(cudaMalloc(&c->w1s, (size_t)Fsh * d * 2));
    CKI(cudaMalloc(&c->w3s, (size_t)Fsh * d * 2));
    CKI(cudaMalloc(&c->w2s, (size_t)Fsh * d * 2));
  }
  // symmetric region
  const size_t Tm = std::max(c->T_max, 1);
  SymLayout &L = c->L;
  size_t off = 0;
  for (int st = 0; st < 2; ++st) {
    SymLayout &Ls = c->set[st].L;
    Ls.recv = off; off = align_up(off + (size_t)c->R_tot * d * 2, 1024);
    Ls.meta = off; off = align_up(off + (size_t)c->R_tot * 8, 1024);
    Ls.dup = off; off = align_up(off + (size_t)c->R_tot * 4, 1024);
    Ls.ybuf = off; off = align_up(off + Tm * k * d * 2, 1024);
    Ls.tokctr = off; off = align_up(off + Tm * 4, 1024);
  }
  L = c->set[0].L;
  L.cnt_all = off; off = align_up(off + (size_t)3 * world * c->nkeys * 4, 1024);
  L.flags = off; off = align_up(off + kNumFlagKinds * kMaxWorld * 4, 1024);
  L.total = off;
  for (int st = 0; st < 2; ++st) {
    c->set[st].L.cnt_all = L.cnt_all;
    c->set[st].L.flags = L.flags;
    c->set[st].L.total = L.total;
  }
  CKI(cudaMalloc(&c->sym, L.total));
  CKI(cudaMemset(c->sym, 0, L.total));
  c->peer[rank] = c->sym;
  // local scratch
  const int nblk_max = (int)((Tm + kRankBlock - 1) / kRankBlock);
  const int ftiles = (F + BM - 1) / BM, ctiles = (d + BM - 1) / BM;
  const int nt_max = (c->R_cap + 127) / 128 + (int)S_loc + 1;  // narrow tiles: the most units
  const int ftiles_sh = Fsh > 0 ? (Fsh + BM - 1) / BM : 0;
  const int nt_sh = (int)((Tm + 127) / 128);
  c->args.n_units_max = nt_max * (ftiles + ctiles * c->nsplit) + nt_sh * (ftiles_sh + ctiles) + 16;
  c->args.n_ctr_max = nt_max * (1 + ctiles) + nt_sh + 16;
  size_t so = 0;
  auto carve = [&](size_t bytes) { size_t o = so; so = align_up(so + bytes, 256); return o; };
  size_t o_sg = carve(Tm * 4);
  size_t o_lg = carve(Tm * (size_t)(E + 1) * 4);
  size_t o_idx = carve(Tm * k * 4), o_w = carve(2 * Tm * k * 4), o_key = carve(Tm * k * 4), o_lrank = carve(Tm * k * 4);
  size_t o_sgb = carve(2 * Tm * 4);
  size_t o_key2 = carve(Tm * k * 4);
  size_t o_lp = carve(((Tm + 31) / 32) * (size_t)(d / 64) * 32 * (E + 1) * 4);  // groups * nkp * 32 * E floats (KP >= 64)
  const int gmax = (int)((Tm + 31) / 32), cmax = 1 + nblk_max;
  size_t o_gc2 = carve(3 * (size_t)gmax * 4), o_cc = carve(3 * (size_t)cmax * 4);
  size_t o_bcnt = carve((size_t)nblk_max * c->nkeys * 4), o_pos = carve(Tm * k * 4);
  size_t o_stats = carve((size_t)c->nkeys * 8), o_gsync = carve(128);
  const int n_grp_max = nt_max + nt_sh + 16;
  c->args.n_ctr_all = c->args.n_ctr_max + n_grp_max;
  size_t o_nu = carve(16);
  size_t o_set[2][12];
  for (int st = 0; st < 2; ++st) {
    o_set[st][0] = carve((size_t)c->args.n_ctr_all * 4);                                       // ctr
    o_set[st][1] = carve((size_t)c->R_cap * 4 + 4);                                           // srcrow
    o_set[st][2] = carve((size_t)c->R_cap * F * 2);                                           // H
    o_set[st][3] = carve(Fsh > 0 ? Tm * Fsh * 2 : 0);                                         // Hs
    o_set[st][4] = carve(c->nsplit > 1 ? (size_t)c->nsplit * c->R_cap * d * 4 : 0);           // ws
    o_set[st][5] = carve(Fsh > 0 ? Tm * d * 2 : 0);                                           // ysh
    o_set[st][6] = carve(c->nkeys * 4);                                                       // dbase
    o_set[st][7] = carve(c->nkeys * 4);                                                       // gcounts
    o_set[st][8] = carve(kMaxWorld * 4);                                                      // need_src
    o_set[st][9] = carve(kMaxWorld * 4);                                                      // sent_to
    o_set[st][10] = carve(S_loc * 4);                                                         // slot_rows
    o_set[st][11] = carve(64);                                                                // sync
  }
  size_t o_xs = carve(2 * Tm * d * 2), o_os = carve(2 * Tm * d * 2);
  CKI(cudaMalloc(&c->scratch, so));
  CKI(cudaMemset(c->scratch, 0, so));
  uint8_t *sb = reinterpret_cast<uint8_t *>(c->scratch);
  CallArgs &a = c->args;
  a.d = d; a.E = E; a.k = k; a.F = F; a.Fsh = Fsh; a.world = world; a.rank = rank;
  a.S_max = c->S_max; a.S_loc = c->S_loc; a.nkeys = c->nkeys; a.T_max = c->T_max; a.R_cap = c->R_cap;
  a.R_sh0 = c->R_sh0; a.nsplit = c->nsplit;
  a.wg = c->wg;
  a.bank_w1 = c->bank_w1;
  a.bank_w3 = c->bank_w3;
  {
    // L2 prefetch budget: ~60% of L2 for the weights the GEMM streams first (r01 A/B: 0 -> 522 us,
    // 40% -> 512.9 us, 60% -> 511.3 us, 75% -> 511.6 us per Mixtral decode call)
    const char *e = getenv("TG_L2PF");  // development override (bytes; 0 = off)
    a.l2_prefetch_bytes = e ? atoll(e) : (long long)(prop.l2CacheSize * 0.6);
  }
  a.idx = (int32_t *)(sb + o_idx); a.w = (float *)(sb + o_w); a.sgate = (float *)(sb + o_sg);
  // gate weights and shared-gate values: one buffer per call parity (the next call's front writes
  // them while this call's combine may still read its own, under PDL)
  for (int i = 0; i < 2; ++i) {
    c->w_buf[i] = (float *)(sb + o_w) + (size_t)i * Tm * k;
    c->sg_buf[i] = (float *)(sb + o_sgb) + (size_t)i * Tm;
  }
  a.gmax = gmax; a.cmax = cmax;
  c->logits = (float *)(sb + o_lg);
  a.gate_mode = c->gate_mode; a.shared_gate = c->shared_gate; a.E_r = E + c->shared_gate; a.key = (int32_t *)(sb + o_key);
  c->key_main = a.key; c->key_replay = (int32_t *)(sb + o_key2);
  a.lrank = (int32_t *)(sb + o_lrank); a.logit_part = (float *)(sb + o_lp); a.grp_ctr = (int32_t *)(sb + o_gc2); a.chunk_ctr = (int32_t *)(sb + o_cc); a.bcnt = (int32_t *)(sb + o_bcnt);
  a.dst_pos = (int32_t *)(sb + o_pos); a.stats = (int64_t *)(sb + o_stats);
  a.gsync = (int32_t *)(sb + o_gsync);
  a.n_units = (int32_t *)(sb + o_nu);
  for (int st = 0; st < 2; ++st) {
    tg_ctx::SetState &S = c->set[st];
    S.ctr = (int32_t *)(sb + o_set[st][0]);
    S.srcrow = (int32_t *)(sb + o_set[st][1]);
    S.H = (bf16 *)(sb + o_set[st][2]);
    S.Hs = Fsh > 0 ? (bf16 *)(sb + o_set[st][3]) : nullptr;
    S.ws = c->nsplit > 1 ? (float *)(sb + o_set[st][4]) : nullptr;
    S.ysh = Fsh > 0 ? (bf16 *)(sb + o_set[st][5]) : nullptr;
    S.dbase = (int32_t *)(sb + o_set[st][6]);
    S.gcounts = (int32_t *)(sb + o_set[st][7]);
    S.need_src = (int32_t *)(sb + o_set[st][8]);
    S.sent_to = (int32_t *)(sb + o_set[st][9]);
    S.slot_rows = (int32_t *)(sb + o_set[st][10]);
    S.sync = (int32_t *)(sb + o_set[st][11]);
  }
  apply_set(c, &a, 0);
  for (int i = 0; i < 2; ++i) {
    c->x_stage[i] = (bf16 *)(sb + o_xs) + (size_t)i * Tm * d;
    c->out_stage[i] = (bf16 *)(sb + o_os) + (size_t)i * Tm * d;
  }
  {
    const char *e = getenv("TG_PDL");  // development switch for A/B timing; default on
    a.pdl = (e && e[0] == '0') ? 0 : 1;
    const char *co = getenv("TG_COOP");
    a.coop = (co && co[0] == '1') ? 1 : 0;
    const char *wm = getenv("TG_WIDE");
    if (wm && (wm[0] == '0' || wm[0] == '1')) c->force_mode = wm[0] - '0';
    const char *dm = getenv("TG_G2DUAL");
    if (dm && (dm[0] == '0' || dm[0] == '1')) c->force_dual = dm[0] - '0';
  }
  CKI(cudaHostAlloc(&c->err_host, 64, cudaHostAllocMapped));
  *c->err_host = 0;
  CKI(cudaHostGetDevicePointer(&c->err_dev, c->err_host, 0));
  a.err = c->err_dev;
  a.fail_mask = reinterpret_cast<uint32_t *>(c->err_dev + 4);  // host-mapped words [4], [5]
  a.unrec = c->err_dev + 5;
  // tensor maps (fixed addresses)
  tg_status s;
  if ((s = make_map(c, &c->maps.w1, c->bank_w1, S_loc * F, d, BM)) != TG_OK) return bail(s);
  if ((s = make_map(c, &c->maps.w3, c->bank_w3, S_loc * F, d, BM)) != TG_OK) return bail(s);
  if ((s = make_map(c, &c->maps.w2, c->bank_w2, S_loc * d, F, BM)) != TG_OK) return bail(s);
  if (Fsh > 0) {
    if ((s = make_map(c, &c->maps.w1s, c->w1s, Fsh, d, BM)) != TG_OK) return bail(s);
    if ((s = make_map(c, &c->maps.w3s, c->w3s, Fsh, d, BM)) != TG_OK) return bail(s);
    if ((s = make_map(c, &c->maps.w2s, c->w2s, d, Fsh, BM)) != TG_OK) return bail(s);
  } else {
    c->maps.w1s = c->maps.w1; c->maps.w3s = c->maps.w3; c->maps.w2s = c->maps.w2;
  }
  for (int st = 0; st < 2; ++st)
    for (int i = 0; i < kNumBoxes; ++i) {
      uint32_t br = 16 * (i + 1);
      if ((s = make_map(c, &c->maps.x[st][i], c->sym + c->set[st].L.recv, c->R_tot, d, br)) != TG_OK) return bail(s);
      if ((s = make_map(c, &c->maps.h[st][i], c->set[st].H, std::max(c->R_cap, 1), F, br)) != TG_OK) return bail(s);
      if (Fsh > 0) {
        if ((s = make_map(c, &c->maps.hs[st][i], c->set[st].Hs, Tm, Fsh, br)) != TG_OK) return bail(s);
      } else {
        c->maps.hs[st][i] = c->maps.h[st][i];
      }
    }
  CKI(cudaMalloc(&c->maps_dev, sizeof(TmaMaps)));
  CKI(cudaMemcpy(c->maps_dev, &c->maps, sizeof(TmaMaps), cudaMemcpyHostToDevice));
  CKI(layer_configure());
  CKI(cudaDeviceSynchronize());
#undef CKI
  *out = c;
  return TG_OK;
}

// A peer handle carries the IPC handle of the rank's peer-visible region and the
// signature of its layout: one-sided stores land at the SENDER's offsets, so every
// rank's region must have the same layout (same config and max_tokens_per_rank).
struct PeerHandle {
  cudaIpcMemHandle_t ipc;
  uint64_t sig[8];
};

static void layout_signature(const tg_ctx *c, uint64_t *sig) {
  sig[0] = c->L.total; sig[1] = c->L.recv ^ (c->L.meta << 20); sig[2] = c->L.ybuf ^ (c->L.dup << 20);
  sig[3] = c->L.cnt_all ^ (c->L.flags << 20); sig[4] = (uint64_t)c->R_cap; sig[5] = (uint64_t)c->T_max;
  sig[6] = ((uint64_t)c->nkeys << 32) | (uint64_t)c->world;
  sig[7] = ((uint64_t)c->d << 40) ^ ((uint64_t)c->k << 32) ^ ((uint64_t)c->E << 16) ^ (uint64_t)c->S_max;
}

size_t tg_peer_handle_size(void) { return sizeof(PeerHandle); }

tg_status tg_get_peer_handle(tg_ctx *c, void *out) {
  if (!c || !out) return TG_ERR_INVALID;
  if (c->host_only) return fail(c, TG_ERR_UNSUPPORTED, "host-only ctx has no device buffers");
  CK(cudaSetDevice(c->device));
  PeerHandle h;
  memset(&h, 0, sizeof h);
  CK(cudaIpcGetMemHandle(&h.ipc, c->sym));
  layout_signature(c, h.sig);
  memcpy(out, &h, sizeof h);
  return TG_OK;
}

tg_status tg_connect_peers(tg_ctx *c, const void *all) {
  if (!c || !all) return TG_ERR_INVALID;
  if (c->host_only) return fail(c, TG_ERR_UNSUPPORTED, "host-only ctx has no device buffers");
  CK(cudaSetDevice(c->device));
  const uint8_t *p = reinterpret_cast<const uint8_t *>(all);
  uint64_t mine[8];
  layout_signature(c, mine);
  for (int q = 0; q < c->world; ++q) {  // validate every handle before mapping any
    PeerHandle h;
    memcpy(&h, p + (size_t)q * sizeof h, sizeof h);
    if (memcmp(h.sig, mine, sizeof mine) != 0)
      return fail(c, TG_ERR_PEER, "rank %d's peer-visible region has another layout (config or "
                  "max_tokens_per_rank differ between ranks)", q);
  }
  for (int q = 0; q < c->world; ++q) {
    if (q == c->rank) continue;
    PeerHandle h;
    memcpy(&h, p + (size_t)q * sizeof h, sizeof h);
    void *ptr = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&ptr, h.ipc, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return fail(c, TG_ERR_PEER, "cudaIpcOpenMemHandle(rank %d): %s", q, cudaGetErrorString(e));
    c->peer[q] = reinterpret_cast<uint8_t *>(ptr);
    c->peer_opened[q] = true;
  }
  return TG_OK;
}

tg_status tg_connect_local(tg_ctx *c, tg_ctx *const *ctxs) {
  if (!c || !ctxs) return TG_ERR_INVALID;
  if (c->host_only) return fail(c, TG_ERR_UNSUPPORTED, "host-only ctx has no device buffers");
  uint64_t mine[8], theirs[8];
  layout_signature(c, mine);
  for (int q = 0; q < c->world; ++q) {
    const tg_ctx *o = ctxs[q];
    if (!o || o->host_only) return fail(c, TG_ERR_INVALID, "ctxs[%d] is null or host-only", q);
    if (o->rank != q || o->world != c->world) return fail(c, TG_ERR_INVALID, "ctxs[%d] is rank %d of %d", q, o->rank, o->world);
    if (o->device != c->device) return fail(c, TG_ERR_INVALID, "ctxs[%d] is on device %d, not %d", q, o->device, c->device);
    layout_signature(o, theirs);
    if (memcmp(theirs, mine, sizeof mine) != 0)
      return fail(c, TG_ERR_PEER, "rank %d's peer-visible region has another layout", q);
  }
  for (int q = 0; q < c->world; ++q) c->peer[q] = ctxs[q]->sym;
  return TG_OK;
}

static tg_status copy_in(tg_ctx *c, void *dst, const void *src, size_t bytes, int on_dev) {
  CK(cudaSetDevice(c->device));
  CK(cudaMemcpy(dst, src, bytes, on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice));
  return TG_OK;
}

tg_status tg_load_gate(tg_ctx *c, const void *wg, int on_dev) {
  if (!c || !wg) return TG_ERR_INVALID;
  if (!c->host_only) {
    tg_status s = copy_in(c, c->wg, wg, (size_t)c->E * c->d * 2, on_dev);
    if (s) return s;
  }
  c->gate_loaded = true;
  return TG_OK;
}

tg_status tg_load_shared_gate(tg_ctx *c, const void *wsg, int on_dev) {
  if (!c || !wsg) return TG_ERR_INVALID;
  if (!c->shared_gate) return fail(c, TG_ERR_INVALID, "config has shared_gate = 0");
  if (!c->host_only) {
    tg_status s = copy_in(c, reinterpret_cast<uint8_t *>(c->wg) + (size_t)c->E * c->d * 2, wsg, (size_t)c->d * 2, on_dev);
    if (s) return s;
  }
  c->sgate_loaded = true;
  return TG_OK;
}

tg_status tg_load_experts(tg_ctx *c, int ew, int slot, int expert, const void *w1, const void *w3, const void *w2,
                          int on_dev) {
  if (!c) return TG_ERR_INVALID;
  if (ew < 0 || ew >= c->W || slot < 0 || slot >= c->spe || expert < 0 || expert >= c->E)
    return fail(c, TG_ERR_INVALID, "tg_load_experts: ew %d slot %d expert %d out of range", ew, slot, expert);
  if (c->have_table) {  // a slot the active route table names for another expert stays as it is
    for (int e = 0; e < c->E; ++e)
      for (int j = 0; j < c->C; ++j)
        if (e != expert && c->cand[(e * c->C + j) * 2] == ew && c->cand[(e * c->C + j) * 2 + 1] == slot)
          return fail(c, TG_ERR_INVALID, "tg_load_experts: (ew %d, slot %d) serves expert %d in route table "
                      "version %llu; install a table without it first", ew, slot, e, (unsigned long long)c->version);
  }
  if (!c->host_only && c->ew_rank[ew] == c->rank) {
    if (!w1 || !w3 || !w2) return fail(c, TG_ERR_INVALID, "tg_load_experts: null weights for a local EW");
    const size_t b = (size_t)c->F * c->d * 2;
    const size_t bs = (size_t)(c->ew_base[ew] + slot);
    tg_status s;
    if ((s = copy_in(c, reinterpret_cast<uint8_t *>(c->bank_w1) + bs * b, w1, b, on_dev))) return s;
    if ((s = copy_in(c, reinterpret_cast<uint8_t *>(c->bank_w3) + bs * b, w3, b, on_dev))) return s;
    if ((s = copy_in(c, reinterpret_cast<uint8_t *>(c->bank_w2) + bs * b, w2, b, on_dev))) return s;
  }
  c->hosted[(size_t)ew * c->spe + slot] = expert;
  return TG_OK;
}

tg_status tg_load_shared(tg_ctx *c, const void *w1, const void *w3, const void *w2, int on_dev) {
  if (!c || !w1 || !w3 || !w2) return TG_ERR_INVALID;
  if (c->Fsh == 0) return fail(c, TG_ERR_INVALID, "config has no shared expert (d_ffn_shared = 0)");
  if (!c->host_only) {
    const size_t b = (size_t)c->Fsh * c->d * 2;
    tg_status s;
    if ((s = copy_in(c, c->w1s, w1, b, on_dev))) return s;
    if ((s = copy_in(c, c->w3s, w3, b, on_dev))) return s;
    if ((s = copy_in(c, c->w2s, w2, b, on_dev))) return s;
  }
  c->shared_loaded = true;
  return TG_OK;
}

tg_status tg_set_route_table(tg_ctx *c, uint64_t version, const int32_t *cand, int C) {
  if (!c || !cand || C < 1) return TG_ERR_INVALID;
  if (c->have_table && version <= c->version)
    return fail(c, TG_ERR_STALE_VERSION, "route table version %llu <= current %llu (ignored)",
                (unsigned long long)version, (unsigned long long)c->version);
  for (int e = 0; e < c->E; ++e)
    for (int j = 0; j < C; ++j) {
      int ew = cand[(e * C + j) * 2], sl = cand[(e * C + j) * 2 + 1];
      if (ew < 0) continue;
      if (ew >= c->W || sl < 0 || sl >= c->spe)
        return fail(c, TG_ERR_INVALID, "candidate (%d, %d) of expert %d out of range", ew, sl, e);
      if (c->hosted[(size_t)ew * c->spe + sl] != e)
        return fail(c, TG_ERR_NOT_LOADED, "candidate (ew %d, slot %d) of expert %d holds expert %d", ew, sl, e,
                    c->hosted[(size_t)ew * c->spe + sl]);
    }
  // routable under the current mask?
  for (int e = 0; e < c->E; ++e) {
    bool ok = false;
    for (int j = 0; j < C && !ok; ++j) {
      int ew = cand[(e * C + j) * 2];
      ok = ew >= 0 && !c->mask[ew];
    }
    if (!ok) return fail(c, TG_ERR_NO_ROUTE, "expert %d has no unmasked candidate in the new table", e);
  }
  c->cand.assign(cand, cand + (size_t)c->E * C * 2);
  c->C = C;
  c->version = version;
  c->have_table = true;
  resolve(c);
  return TG_OK;
}

tg_status tg_mask_worker(tg_ctx *c, int ew, int masked) {
  if (!c) return TG_ERR_INVALID;
  if (ew < 0 || ew >= c->W) return fail(c, TG_ERR_INVALID, "ew %d out of range", ew);
  if (!masked && !((c->alive >> c->ew_rank[ew]) & 1u))
    return fail(c, TG_ERR_UNSUPPORTED, "ew %d is on failed rank %d", ew, c->ew_rank[ew]);
  c->mask[ew] = masked ? 1 : 0;
  resolve(c);
  if (c->have_table && c->no_route) {
    int e = 0;
    while (e < c->E && c->rkey[e] >= 0) ++e;
    return fail(c, TG_ERR_NO_ROUTE, "expert %d lost its last unmasked candidate", e);
  }
  return TG_OK;
}

tg_status tg_mask_rank(tg_ctx *c, int r, int masked) {
  if (!c) return TG_ERR_INVALID;
  if (r < 0 || r >= c->world) return fail(c, TG_ERR_INVALID, "rank %d out of range", r);
  if (r == c->rank) return fail(c, TG_ERR_INVALID, "a rank cannot mask itself");
  if (!masked) {
    if (!((c->alive >> r) & 1u))
      return fail(c, TG_ERR_UNSUPPORTED, "rank %d rejoin needs re-provisioning (re-create the ctxs)", r);
    return TG_OK;
  }
  c->alive &= ~(1u << r);
  // the process took its EWs down with it: fail-stop every EW on that rank
  for (int w = 0; w < c->W; ++w)
    if (c->ew_rank[w] == r) c->mask[w] = 1;
  resolve(c);
  if (c->have_table && c->no_route) {
    int e = 0;
    while (e < c->E && c->rkey[e] >= 0) ++e;
    return fail(c, TG_ERR_NO_ROUTE, "expert %d lost its last unmasked candidate", e);
  }
  return TG_OK;
}

// ------------------------------------------------------------ stage export (parity tests)
tg_status tg_set_stage_export(tg_ctx *c, int on) {
  if (!c) return TG_ERR_INVALID;
  if (c->host_only) return fail(c, TG_ERR_UNSUPPORTED, "host-only ctx");
  c->stage_export = on != 0;
  return TG_OK;
}

tg_status tg_get_stage(tg_ctx *c, int stage, void *dst, size_t cap, size_t *bytes) {
  if (!c || !bytes) return TG_ERR_INVALID;
  *bytes = 0;
  if (c->host_only) return fail(c, TG_ERR_UNSUPPORTED, "host-only ctx");
  CK(cudaSetDevice(c->device));
  CK(cudaDeviceSynchronize());
  tg_status st = check_sticky(c);
  if (st) return st;
  const tg_ctx::SetState &LS = c->set[c->last_set];  // the last call's buffer set
  const size_t T = (size_t)c->last_T;
  size_t R = 0;
  if (stage == TG_STAGE_RECV || stage == TG_STAGE_META || stage == TG_STAGE_H) {
    std::vector<int32_t> rows(std::max(c->S_loc, 1), 0);
    if (c->S_loc)
      CK(cudaMemcpy(rows.data(), c->set[c->last_set].slot_rows, sizeof(int32_t) * c->S_loc, cudaMemcpyDeviceToHost));
    for (int i = 0; i < c->S_loc; ++i) R += (size_t)rows[i];
  }
  const void *src = nullptr;
  size_t n = 0;
  switch (stage) {
    case TG_STAGE_LOGITS:
      if (!c->stage_export) return fail(c, TG_ERR_INVALID, "logits are exported only after tg_set_stage_export(ctx, 1)");
      src = c->logits; n = T * (size_t)(c->E + c->shared_gate) * 4; break;
    case TG_STAGE_RECV: src = c->sym + LS.L.recv; n = R * c->d * 2; break;
    case TG_STAGE_META: src = c->sym + LS.L.meta; n = R * 8; break;
    case TG_STAGE_H: src = LS.H; n = R * c->F * 2; break;
    case TG_STAGE_Y: src = c->sym + LS.L.ybuf; n = T * c->k * c->d * 2; break;
    case TG_STAGE_HSH: src = LS.Hs; n = c->Fsh ? T * c->Fsh * 2 : 0; break;
    case TG_STAGE_YSH: src = LS.ysh; n = c->Fsh ? T * c->d * 2 : 0; break;
    case TG_STAGE_SGATE: src = c->sg_buf[c->last_wb]; n = c->shared_gate ? T * 4 : 0; break;
    default: return fail(c, TG_ERR_INVALID, "unknown stage %d", stage);
  }
  *bytes = n;
  if (!dst || n == 0) return TG_OK;
  if (cap < n) return fail(c, TG_ERR_INVALID, "stage %d needs %zu bytes, buffer has %zu", stage, n, cap);
  CK(cudaMemcpy(dst, src, n, cudaMemcpyDefault));
  return TG_OK;
}

int tg_max_slots(const tg_ctx *c) { return c ? c->S_max : -1; }
int tg_bank_slot(const tg_ctx *c, int ew, int slot) {
  if (!c || ew < 0 || ew >= c->W || slot < 0 || slot >= c->spe) return -1;
  return c->ew_base[ew] + slot;
}

static void rec(tg_ctx *c, cudaStream_t s) {
  if (!c->prof || c->ev.empty()) return;
  int slot = c->prof_calls % tg_ctx::kProfCalls;
  if (c->n_ev < tg_ctx::kEv) cudaEventRecord(c->ev[(size_t)slot * tg_ctx::kEv + c->n_ev++], s);
}

// Per-call kernel arguments (everything but the epochs of the flags).
static CallArgs call_args(tg_ctx *c, int T, const void *x, void *out, RouteKeys *rk) {
  for (int e = 0; e < kMaxExperts; ++e) rk->key[e] = e < c->E ? c->rkey[e] : -1;
  CallArgs a = c->args;
  a.T = T;
  a.x = reinterpret_cast<const bf16 *>(x);
  a.out = reinterpret_cast<bf16 *>(out);
  a.epoch = ++c->epoch;
  {
    // Wide token tiles (bn = 256) cut the L2 bytes per FLOP of prefill tiles but
    // measured slower on B200 (per-SM L2->SMEM delivery, not bytes/FLOP, limits
    // them; profiles/README.md r01): narrow by default, wide on request.
    bool wide = false;
    if (c->force_mode >= 0) wide = c->force_mode == 1;  // TG_WIDE development override
    a.bn = wide ? 256 : 128;
    // GEMM2 units take two W2 tiles sharing one H tile: half the H bytes per W2 byte
    // (the per-SM L2->SMEM stream, not HBM, is what the token tiles cost; r01 A/B: -5%)
    a.g2dual = !wide && c->force_dual != 0;
  }
  a.trace = c->tracing ? c->trace : nullptr;
  {
    // world == 1 fast paths; TG_LOCAL: development A/B switch ("0" both off,
    // "r" row-ordered dispatch only, "c" barrier-free combine only)
    const char *e = getenv("TG_LOCAL");
    const bool rows = !e || e[0] == '1' || e[0] == 'r', comb = !e || e[0] == '1' || e[0] == 'c';
    a.local_rows = c->world == 1 && rows;
    // world > 1: each (pair, pair of 128-column output tiles) is one NVLink atomic at its source;
    // past ~48K per rank the grid-barrier combine wins (2-GPU A/B, µs per call, per-token vs
    // barrier: Mixtral decode 293 vs 302 (4K arrivals), DS-V2-Lite decode 196 vs 208 (25K), Qwen
    // prefill 521 vs 464 (131K)).  Static per ctx (T_max, k, d agree on every rank): the EWs'
    // arrivals and the sources' waits must take the same branch.
    const long arrivals = (long)c->T_max * c->k * ((c->d + 2 * BM - 1) / (2 * BM));
    a.tok_comb = comb && (c->world == 1 || arrivals <= kTokCombMaxArrivals) ? 1 : 0;
    // prefill-sized calls interleave GEMM2 into the work list (H consumed while in L2)
    a.g2lag = (T * c->k >= 8192) ? 8 : 0;  // same-box A/B, Qwen-shaped prefill: lag 0 888, 2 904, 4 876, 8 874 us
    const char *gl = getenv("TG_G2LAG");  // development override (A/B timing)
    if (gl) a.g2lag = atoi(gl);
    const char *lb = getenv("TG_LAYOUT");  // development override (A/B timing)
    a.layout_block = lb ? atoi(lb) : kLocalLayoutBlock;
    const char *dv = getenv("TG_DEV");
    a.dev = dv ? atoi(dv) : 0;
  }
  a.alive = c->alive;
  a.hk = nullptr;
  if (c->pend_host) {
    a.hk = c->hk_dev;
    a.hcall = (int)(c->host_calls + 1);
    a.hb = (int)(c->host_calls & 1);
    a.hexit = (int)((c->host_calls / 2 + 1) * (long long)c->n_sms - 1);  // grid = n_sms CTAs
  }
  a.fslot_data = FLAG_DATA;
  a.fslot_comb = FLAG_COMB;
  a.fslot_cnt = FLAG_CNT;
  a.fail_timeout_ns = c->fail_timeout_ns;
  a.cnt_timeout_ns = c->cnt_timeout_ns;
  a.logits = c->stage_export ? c->logits : nullptr;
  a.cta0 = 0;
  a.ncta = c->n_sms;
  a.absent = 0;
  a.cbuf = (int)(a.epoch % 3);
  a.replay = 0;
  a.failed = 0;
  a.key_old = nullptr;
  a.inject_fail = 0;
  for (int q = 0; q < kMaxWorld; ++q) a.sym[q] = q < c->world ? c->peer[q] : nullptr;
  return a;
}

// Validation and per-call arguments of one rank's layer call (everything but the launch).
static tg_status prepare_call(tg_ctx *c, const void *x, void *out, int T, CallArgs *a, RouteKeys *rk) {
  if (!c) return TG_ERR_INVALID;
  if (c->host_only) return fail(c, TG_ERR_UNSUPPORTED, "host-only ctx (no CUDA device): no compute path");
  tg_status st = check_sticky(c);
  if (st) return st;
  if (T < 0 || T > c->T_max) return fail(c, TG_ERR_INVALID, "n_tokens %d > max_tokens_per_rank %d", T, c->T_max);
  if (T > 0 && (!x || !out)) return fail(c, TG_ERR_INVALID, "null x/out");
  if (T > 0 && x == out) return fail(c, TG_ERR_INVALID, "out aliases x");
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(out)) & 15)
    return fail(c, TG_ERR_INVALID, "x/out must be 16-byte aligned");
  if (!c->gate_loaded) return fail(c, TG_ERR_NOT_LOADED, "router weights not loaded (tg_load_gate)");
  if (c->Fsh > 0 && !c->shared_loaded) return fail(c, TG_ERR_NOT_LOADED, "shared expert not loaded");
  if (c->shared_gate && !c->sgate_loaded) return fail(c, TG_ERR_NOT_LOADED, "shared-expert gate not loaded");
  if (!c->have_table) return fail(c, TG_ERR_NOT_LOADED, "no route table (tg_set_route_table)");
  if (c->no_route) return fail(c, TG_ERR_NO_ROUTE, "some expert has no unmasked candidate: nothing launched");
  for (int q = 0; q < c->world; ++q)
    if (!c->peer[q] && ((c->alive >> q) & 1u)) return fail(c, TG_ERR_PEER, "peer %d not connected (tg_connect_peers)", q);
  *a = call_args(c, T, x, out, rk);
  a->xepoch = ++c->xepoch;
  a->fepoch = a->xepoch;
  a->cnt_buf = (int)(a->xepoch & 1);
  c->last_wb = (int)(a->xepoch & 1);
  a->w = c->w_buf[c->last_wb];
  a->sgate = c->sg_buf[c->last_wb];
  apply_set(c, a, c->last_wb);
  c->last_set = c->last_wb;
  a->inject_fail = c->inject_next ? 1 : 0;
  c->inject_next = false;
  return TG_OK;
}

tg_status tg_moe_layer(tg_ctx *c, const void *x, void *out, int T, void *stream) {
  CallArgs a;
  RouteKeys rk;
  tg_status st = prepare_call(c, x, out, T, &a, &rk);
  if (st) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  CK(cudaSetDevice(c->device));
  c->n_ev = 0;
  rec(c, s);
  CK(launch_layer(a, rk, c->maps, c->n_sms, s));
  rec(c, s);
  if (c->prof) ++c->prof_calls;
  c->last_T = T;
  c->last_launches = 1;
  return TG_OK;
}

// Virtual ranks of one GPU: one cooperative launch over every rank's data (their waits on one
// another need them co-resident; separate launches carry no such guarantee).
static tg_status check_multi(tg_ctx *const *ctxs, int n) {
  if (!ctxs || n < 1 || n > kMaxVirt) return TG_ERR_INVALID;
  for (int r = 0; r < n; ++r) {
    if (!ctxs[r] || ctxs[r]->host_only) return TG_ERR_INVALID;
    if (ctxs[r]->rank != r || ctxs[r]->world != n || ctxs[r]->device != ctxs[0]->device)
      return fail(ctxs[r], TG_ERR_INVALID, "fused launch: ctxs[%d] must be rank %d of %d on device %d", r, r, n,
                  ctxs[0]->device);
    if (ctxs[r]->peer[(r + 1) % n] != ctxs[(r + 1) % n]->sym)
      return fail(ctxs[r], TG_ERR_PEER, "fused launch: ranks not connected by tg_connect_local");
  }
  return TG_OK;
}

tg_status tg_moe_layer_multi(tg_ctx *const *ctxs, int n, const void *const *x, void *const *out, const int *T,
                             void *stream) {
  tg_status st = check_multi(ctxs, n);
  if (st) return st;
  if (!x || !out || !T) return TG_ERR_INVALID;
  static MultiArgs m;  // host staging of the kernel parameter (not thread-safe, as the ctxs)
  memset(&m, 0, sizeof m);
  m.n = n;
  m.nper = ctxs[0]->n_sms / n;
  for (int r = 0; r < n; ++r) {
    tg_ctx *c = ctxs[r];
    if (T[r] < 0) {  // does not take part (a rank that died before the call)
      m.a[r].absent = 1;
      continue;
    }
    st = prepare_call(c, x[r], out[r], T[r], &m.a[r], &m.rk[r]);
    if (st) return st;
    m.a[r].cta0 = r * m.nper;
    m.a[r].ncta = m.nper;
    m.a[r].pdl = 0;
    m.maps[r] = c->maps_dev;
  }
  tg_ctx *c = ctxs[0];
  CK(cudaSetDevice(c->device));
  CK(launch_layer_multi(m, reinterpret_cast<cudaStream_t>(stream)));
  for (int r = 0; r < n; ++r)
    if (T[r] >= 0) {
      ctxs[r]->last_T = T[r];
      ctxs[r]->last_launches = 1;
    }
  return TG_OK;
}

tg_status tg_set_failure_timeout(tg_ctx *c, double ms) {
  if (!c) return TG_ERR_INVALID;
  if (!(ms > 0.0) || ms > 4000.0) return fail(c, TG_ERR_INVALID, "failure timeout %g ms not in (0, 4000]", ms);
  c->fail_timeout_ns = (long long)(ms * 1e6);
  c->cnt_timeout_ns = std::min(10 * c->fail_timeout_ns, 4000000000LL);
  return TG_OK;
}

tg_status tg_inject_failure(tg_ctx *c) {
  if (!c) return TG_ERR_INVALID;
  c->inject_next = true;
  return TG_OK;
}

// In-call failover, host half: if the last call saw a peer fail, fail-stop the failed ranks and
// build the replay run's arguments.  *fm_out = failed ranks (0: nothing to replay).
static tg_status replay_args(tg_ctx *c, const void *x, void *out, int T, CallArgs *a, RouteKeys *rk,
                             uint32_t *fm_out) {
  *fm_out = 0;
  volatile int *hw = reinterpret_cast<volatile int *>(c->err_host);
  const uint32_t fm = static_cast<uint32_t>(hw[4]) & ~(1u << c->rank) & c->alive;
  if (!fm) return TG_OK;  // the last call saw no peer failure: nothing to do
  if (T != c->last_T) return fail(c, TG_ERR_INVALID, "failover needs the failed call's tokens (%d, got %d)", c->last_T, T);
  hw[4] = 0;
  hw[5] = 0;
  // the failed ranks are fail-stopped from now on (as tg_mask_rank) ...
  for (int q = 0; q < c->world; ++q)
    if ((fm >> q) & 1u) {
      c->alive &= ~(1u << q);
      for (int w = 0; w < c->W; ++w)
        if (c->ew_rank[w] == q) c->mask[w] = 1;
    }
  resolve(c);
  *fm_out = fm;
  // ... and the pairs this rank had sent them are re-dispatched to the next live candidate
  // of their expert, on whichever surviving rank it lives: a replay run of k_layer in which
  // every survivor takes part (the survivors all saw the failure in the same call: each
  // waits for every live rank's combine flag), with its own flags and count buffer
  *a = call_args(c, T, x, out, rk);
  a->xepoch = c->xepoch;
  a->fepoch = ++c->rxepoch;
  a->fslot_data = FLAG_RDATA;
  a->fslot_comb = FLAG_RCOMB;
  a->fslot_cnt = FLAG_RCNT;
  a->cnt_buf = kCntBufReplay;
  a->replay = 1;
  a->failed = fm;
  a->key_old = c->key_main;
  a->key = c->key_replay;
  a->w = c->w_buf[c->last_wb];  // the failed call's gate weights (its combine is redone)
  a->sgate = c->sg_buf[c->last_wb];
  apply_set(c, a, c->last_set);  // and its buffer set: the other pairs' outputs are kept
  a->logits = nullptr;
  a->local_rows = 0;  // a replay is a multi-rank run (world > 1)
  a->tok_comb = 0;
  return TG_OK;
}

static tg_status replay_status(tg_ctx *c) {
  tg_status st = check_sticky(c);
  if (st) return st;
  volatile int *hw = reinterpret_cast<volatile int *>(c->err_host);
  c->last_launches = 1;
  if (hw[5] > 0)
    return fail(c, TG_ERR_NO_ROUTE, "%d pairs have no live candidate left: not recomputed (their tokens' "
                "outputs are incomplete)", hw[5]);
  if (static_cast<uint32_t>(hw[4]) & ~(1u << c->rank) & c->alive)
    return fail(c, TG_ERR_PEER, "another rank failed during the replay (call tg_failover again)");
  return TG_OK;
}

tg_status tg_failover(tg_ctx *c, const void *x, void *out, int T, void *stream, uint32_t *failed) {
  if (!c) return TG_ERR_INVALID;
  if (failed) *failed = 0;
  if (c->host_only) return fail(c, TG_ERR_UNSUPPORTED, "host-only ctx (no CUDA device): no compute path");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  CK(cudaSetDevice(c->device));
  CK(cudaStreamSynchronize(s));
  tg_status st = check_sticky(c);
  if (st) return st;
  CallArgs a;
  RouteKeys rk;
  uint32_t fm = 0;
  if ((st = replay_args(c, x, out, T, &a, &rk, &fm))) return st;
  if (failed) *failed = fm;
  if (!fm) return TG_OK;
  CK(launch_layer(a, rk, c->maps, c->n_sms, s));
  CK(cudaStreamSynchronize(s));
  return replay_status(c);
}

tg_status tg_failover_multi(tg_ctx *const *ctxs, int n, const void *const *x, void *const *out, const int *T,
                            void *stream, uint32_t *failed) {
  tg_status st = check_multi(ctxs, n);
  if (st) return st;
  if (!x || !out || !T || !failed) return TG_ERR_INVALID;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  CK2(ctxs[0], cudaSetDevice(ctxs[0]->device));
  CK2(ctxs[0], cudaStreamSynchronize(s));
  static MultiArgs m;
  memset(&m, 0, sizeof m);
  m.n = n;
  m.nper = ctxs[0]->n_sms / n;
  int any = 0;
  for (int r = 0; r < n; ++r) {
    failed[r] = 0;
    m.a[r].absent = 1;
    if (T[r] < 0) continue;  // absent rank (dead)
    tg_ctx *c = ctxs[r];
    if ((st = check_sticky(c))) return st;
    uint32_t fm = 0;
    if ((st = replay_args(c, x[r], out[r], T[r], &m.a[r], &m.rk[r], &fm))) return st;
    failed[r] = fm;
    if (!fm) {
      m.a[r].absent = 1;
      continue;
    }
    m.a[r].cta0 = r * m.nper;
    m.a[r].ncta = m.nper;
    m.a[r].pdl = 0;
    m.a[r].absent = 0;
    m.maps[r] = c->maps_dev;
    any = 1;
  }
  if (!any) return TG_OK;
  CK2(ctxs[0], launch_layer_multi(m, s));
  CK2(ctxs[0], cudaStreamSynchronize(s));
  for (int r = 0; r < n; ++r)
    if (!m.a[r].absent && (st = replay_status(ctxs[r]))) return st;
  return TG_OK;
}

static tg_status host_path_init(tg_ctx *c) {
  if (c->hs_h2d) return TG_OK;
  CK(cudaStreamCreateWithFlags(&c->hs_h2d, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&c->hs_d2h, cudaStreamNonBlocking));
  for (int i = 0; i < 2; ++i) {
    CK(cudaEventCreateWithFlags(&c->ev_h2d[i], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_k[i], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_d2h[i], cudaEventDisableTiming));
  }
  CK(cudaEventCreateWithFlags(&c->ev_sync, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->ev_sync2, cudaEventDisableTiming));
  c->wait32 = get_stream_op("cuStreamWaitValue32");
  c->write32 = get_stream_op("cuStreamWriteValue32");
  if (c->wait32 && c->write32) {
    CK(cudaMalloc(&c->hk_dev, 8 * sizeof(int)));
    CK(cudaMemset(c->hk_dev, 0, 8 * sizeof(int)));
    // the copy streams are non-blocking (no implicit order after the legacy stream's memset):
    // the words must read zero before the first stream wait on them (a fresh allocation can hold
    // stale values from memory freed earlier in the process)
    CK(cudaDeviceSynchronize());
  }
  return TG_OK;
}

// Host path, pipelined over two staging buffers: the H2D copy of call i+1 and the D2H copy
// of call i run on their own streams while the layer of the neighbouring call runs on `stream`.
tg_status tg_moe_layer_host(tg_ctx *c, const void *xh, void *oh, int T, void *stream) {
  if (!c) return TG_ERR_INVALID;
  if (c->host_only) return fail(c, TG_ERR_UNSUPPORTED, "host-only ctx (no CUDA device): no compute path");
  if (T < 0 || T > c->T_max) return fail(c, TG_ERR_INVALID, "n_tokens %d > max_tokens_per_rank %d", T, c->T_max);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  CK(cudaSetDevice(c->device));
  tg_status st = host_path_init(c);
  if (st) return st;
  const int b = (int)(c->host_calls & 1);
  const size_t bytes = (size_t)T * c->d * 2;
  if (c->hk_dev) {
    // no stream op between consecutive kernels on `stream` (that would serialise them: PDL):
    // the copy streams wait on / write device words, the kernel polls them (CallArgs::hk)
    const int hcall = (int)(c->host_calls + 1);
    CUstream h2d = reinterpret_cast<CUstream>(c->hs_h2d), d2h = reinterpret_cast<CUstream>(c->hs_d2h);
    const CUdeviceptr w = reinterpret_cast<CUdeviceptr>(c->hk_dev);
    if (c->host_calls < 2) {  // first uses of the buffers: after the work already on `stream`
      CK(cudaEventRecord(c->ev_sync, s));
      CK(cudaStreamWaitEvent(c->hs_h2d, c->ev_sync, 0));
    } else if (c->wait32(h2d, w + (6 + b) * 4, (cuuint32_t)(hcall - 2), CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS) {
      return fail(c, TG_ERR_CUDA, "cuStreamWaitValue32 failed");  // x_stage[b] free once call i-2 completed
    }
    if (T > 0) CK(cudaMemcpyAsync(c->x_stage[b], xh, bytes, cudaMemcpyHostToDevice, c->hs_h2d));
    if (c->write32(h2d, w + (0 + b) * 4, (cuuint32_t)hcall, CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
      return fail(c, TG_ERR_CUDA, "cuStreamWriteValue32 failed");
    c->pend_host = true;
    st = tg_moe_layer(c, c->x_stage[b], c->out_stage[b], T, stream);
    c->pend_host = false;
    if (st) return st;
    if (c->wait32(d2h, w + (6 + b) * 4, (cuuint32_t)hcall, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
      return fail(c, TG_ERR_CUDA, "cuStreamWaitValue32 failed");
    if (T > 0) CK(cudaMemcpyAsync(oh, c->out_stage[b], bytes, cudaMemcpyDeviceToHost, c->hs_d2h));
    if (c->write32(d2h, w + (2 + b) * 4, (cuuint32_t)hcall, CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
      return fail(c, TG_ERR_CUDA, "cuStreamWriteValue32 failed");
    ++c->host_calls;
    return TG_OK;
  }
  // (no stream memory operations: event ordering, which serialises consecutive layer launches)
  if (c->host_calls < 2) {  // first uses of the buffers: ordered after the work already on `stream`
    CK(cudaEventRecord(c->ev_sync, s));
    CK(cudaStreamWaitEvent(c->hs_h2d, c->ev_sync, 0));
  } else {                  // x_stage[b] is free once the layer of call i-2 has run
    CK(cudaStreamWaitEvent(c->hs_h2d, c->ev_k[b], 0));
    CK(cudaStreamWaitEvent(s, c->ev_d2h[b], 0));  // out_stage[b] read out by call i-2's D2H
  }
  if (T > 0) CK(cudaMemcpyAsync(c->x_stage[b], xh, bytes, cudaMemcpyHostToDevice, c->hs_h2d));
  CK(cudaEventRecord(c->ev_h2d[b], c->hs_h2d));
  CK(cudaStreamWaitEvent(s, c->ev_h2d[b], 0));
  st = tg_moe_layer(c, c->x_stage[b], c->out_stage[b], T, stream);
  if (st) return st;
  CK(cudaEventRecord(c->ev_k[b], s));
  CK(cudaStreamWaitEvent(c->hs_d2h, c->ev_k[b], 0));
  if (T > 0) CK(cudaMemcpyAsync(oh, c->out_stage[b], bytes, cudaMemcpyDeviceToHost, c->hs_d2h));
  CK(cudaEventRecord(c->ev_d2h[b], c->hs_d2h));
  ++c->host_calls;
  return TG_OK;
}

tg_status tg_host_sync(tg_ctx *c, void *stream) {
  if (!c) return TG_ERR_INVALID;
  if (c->host_only) return fail(c, TG_ERR_UNSUPPORTED, "host-only ctx (no CUDA device)");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  CK(cudaSetDevice(c->device));
  tg_status st = host_path_init(c);
  if (st) return st;
  // `stream` waits for every pending host-path copy ...
  CK(cudaEventRecord(c->ev_sync2, c->hs_d2h));
  CK(cudaStreamWaitEvent(s, c->ev_sync2, 0));
  CK(cudaEventRecord(c->ev_sync2, c->hs_h2d));
  CK(cudaStreamWaitEvent(s, c->ev_sync2, 0));
  // ... and later host-path copies wait for what is on `stream` now
  CK(cudaEventRecord(c->ev_sync, s));
  CK(cudaStreamWaitEvent(c->hs_h2d, c->ev_sync, 0));
  CK(cudaStreamWaitEvent(c->hs_d2h, c->ev_sync, 0));
  return TG_OK;
}

tg_status tg_get_routing(tg_ctx *c, int n_tokens, int32_t *idx, float *w, int32_t *dst_rank, int32_t *dst_slot,
                         int32_t *dst_pos, int32_t *counts, void *stream) {
  if (!c) return TG_ERR_INVALID;
  if (c->host_only) return fail(c, TG_ERR_UNSUPPORTED, "host-only ctx");
  if (n_tokens != c->last_T)
    return fail(c, TG_ERR_INVALID, "tg_get_routing: n_tokens %d, the last call had %d", n_tokens, c->last_T);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  CK(cudaSetDevice(c->device));
  const size_t n = (size_t)c->last_T * c->k;
  if (idx && n) CK(cudaMemcpyAsync(idx, c->args.idx, n * 4, cudaMemcpyDeviceToDevice, s));
  if (w && n) CK(cudaMemcpyAsync(w, c->w_buf[c->last_wb], n * 4, cudaMemcpyDeviceToDevice, s));
  if (dst_pos && n) CK(cudaMemcpyAsync(dst_pos, c->args.dst_pos, n * 4, cudaMemcpyDeviceToDevice, s));
  if (counts) CK(cudaMemcpyAsync(counts, c->set[c->last_set].gcounts, (size_t)c->nkeys * 4, cudaMemcpyDeviceToDevice, s));
  if ((dst_rank || dst_slot) && n) CK(launch_export_keys(c->args, (int)n, dst_rank, dst_slot, s));
  return TG_OK;
}

tg_status tg_get_stats(tg_ctx *c, int64_t *rows) {
  if (!c || !rows) return TG_ERR_INVALID;
  if (c->host_only) {
    memset(rows, 0, sizeof(int64_t) * c->nkeys);
    return TG_OK;
  }
  CK(cudaSetDevice(c->device));
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(rows, c->args.stats, sizeof(int64_t) * c->nkeys, cudaMemcpyDeviceToHost));
  return check_sticky(c);
}

tg_status tg_set_profiling(tg_ctx *c, int on) {
  if (!c) return TG_ERR_INVALID;
  if (c->host_only) return fail(c, TG_ERR_UNSUPPORTED, "host-only ctx");
  c->prof = on != 0;
  c->prof_calls = 0;
  if (c->prof && c->ev.empty()) {
    CK(cudaSetDevice(c->device));
    c->ev.resize((size_t)tg_ctx::kProfCalls * tg_ctx::kEv);
    for (auto &e : c->ev) CK(cudaEventCreate(&e));
  }
  return TG_OK;
}

// Mean per-kernel duration over the calls recorded since profiling was enabled
// (at most the last kProfCalls): router, rank, dispatch, gemm, combine.
tg_status tg_get_kernel_times(tg_ctx *c, float *ms, int *n) {
  if (!c || !ms || !n) return TG_ERR_INVALID;
  *n = 0;
  if (!c->prof || c->prof_calls == 0) return TG_OK;
  CK(cudaSetDevice(c->device));
  const int calls = std::min(c->prof_calls, (int)tg_ctx::kProfCalls);
  const int nk = tg_ctx::kEv - 1;
  std::vector<double> acc(nk, 0.0);
  for (int i = 0; i < calls; ++i) {
    int slot = (c->prof_calls - 1 - i) % tg_ctx::kProfCalls;
    cudaEvent_t *e = &c->ev[(size_t)slot * tg_ctx::kEv];
    CK(cudaEventSynchronize(e[nk]));
    for (int j = 0; j < nk; ++j) {
      float t = 0.f;
      CK(cudaEventElapsedTime(&t, e[j], e[j + 1]));
      acc[j] += t;
    }
  }
  for (int j = 0; j < nk; ++j) ms[j] = (float)(acc[j] / calls);
  *n = nk;
  return check_sticky(c);
}

tg_status tg_set_trace(tg_ctx *c, int on) {
  if (!c) return TG_ERR_INVALID;
  if (c->host_only) return fail(c, TG_ERR_UNSUPPORTED, "host-only ctx");
  CK(cudaSetDevice(c->device));
  if (on && !c->trace) {
    CK(cudaMalloc(&c->trace, sizeof(uint64_t) * ((size_t)c->args.n_units_max + 148 + 64 + 1024)));
    CK(cudaMemset(c->trace, 0, sizeof(uint64_t) * ((size_t)c->args.n_units_max + 148 + 64 + 1024)));
  }
  c->tracing = on != 0;
  return TG_OK;
}

tg_status tg_get_trace(tg_ctx *c, uint64_t *trace, int cap, int *n_units, int *n_ctas) {
  if (!c || !n_units || !n_ctas) return TG_ERR_INVALID;
  if (c->host_only || !c->trace) return fail(c, TG_ERR_UNSUPPORTED, "tracing not enabled");
  CK(cudaSetDevice(c->device));
  CK(cudaDeviceSynchronize());
  int nu = 0;
  CK(cudaMemcpy(&nu, c->args.n_units, sizeof(int), cudaMemcpyDeviceToHost));
  *n_units = nu;
  *n_ctas = c->n_sms;
  if (nu + 148 + 64 + 1024 > cap) return fail(c, TG_ERR_INVALID, "trace capacity %d < %d", cap, nu + 148 + 64 + 1024);
  if (trace) {
    CK(cudaMemcpy(trace, c->trace, sizeof(uint64_t) * nu, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(trace + nu, c->trace + c->args.n_units_max, sizeof(uint64_t) * (148 + 64 + 1024), cudaMemcpyDeviceToHost));
  }
  return check_sticky(c);
}

int tg_last_launch_count(const tg_ctx *c) { return c ? c->last_launches : 0; }

const char *tg_last_error(const tg_ctx *c) { return c ? c->errmsg.c_str() : g_init_error.c_str(); }

// ------------------------------------------------------------ KV checkpointing (NEXT-4)
tg_status tg_kv_store_init(tg_ctx *c, size_t bytes) {
  if (!c) return TG_ERR_INVALID;
  if (c->host_only) return fail(c, TG_ERR_UNSUPPORTED, "host-only ctx (no CUDA device)");
  if (c->kv_bucket) return fail(c, TG_ERR_INVALID, "checkpoint store already initialised");
  if (bytes == 0) return fail(c, TG_ERR_INVALID, "empty checkpoint store");
  CK(cudaSetDevice(c->device));
  if (cudaHostAlloc(&c->kv_bucket, bytes, cudaHostAllocDefault) != cudaSuccess) {
    c->kv_bucket = nullptr;
    return fail(c, TG_ERR_OOM, "pinned checkpoint bucket of %zu bytes", bytes);
  }
  int lo = 0, hi = 0;
  CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));  // lo = least urgent
  CK(cudaStreamCreateWithPriority(&c->kv_stream, cudaStreamNonBlocking, lo));
  CK(cudaEventCreateWithFlags(&c->kv_ev, cudaEventDisableTiming));
  c->kv_bytes = bytes;
  c->kv_committed = 0;
  return TG_OK;
}

static void CUDART_CB kv_commit_cb(void *p) {
  tg_ctx::KvRec *r = static_cast<tg_ctx::KvRec *>(p);
  r->c->kv_committed = r->seq;  // stream order: every earlier segment has landed
}

tg_status tg_kv_checkpoint(tg_ctx *c, const void *seg, size_t bytes, size_t offset, uint64_t seq, void *stream) {
  if (!c) return TG_ERR_INVALID;
  if (!c->kv_bucket) return fail(c, TG_ERR_NOT_LOADED, "no checkpoint store (tg_kv_store_init)");
  if (!seg || offset > c->kv_bytes || bytes > c->kv_bytes - offset)
    return fail(c, TG_ERR_INVALID, "segment [%zu, +%zu) outside the %zu-byte bucket", offset, bytes, c->kv_bytes);
  if (seq <= c->kv_rec[(c->kv_next + tg_ctx::kKvRecs - 1) % tg_ctx::kKvRecs].seq && c->kv_next > 0)
    return fail(c, TG_ERR_STALE_VERSION, "sequence numbers must increase");
  CK(cudaSetDevice(c->device));
  // ordered after the work on `stream` (the layer call that produced the segment), then the
  // copy engine and the commit record on the low-priority checkpoint stream
  CK(cudaEventRecord(c->kv_ev, reinterpret_cast<cudaStream_t>(stream)));
  CK(cudaStreamWaitEvent(c->kv_stream, c->kv_ev, 0));
  CK(cudaMemcpyAsync(c->kv_bucket + offset, seg, bytes, cudaMemcpyDeviceToHost, c->kv_stream));
  tg_ctx::KvRec *r = &c->kv_rec[c->kv_next % tg_ctx::kKvRecs];
  if (c->kv_next >= tg_ctx::kKvRecs && c->kv_committed < r->seq)  // the record's commit is still pending
    CK(cudaStreamSynchronize(c->kv_stream));
  ++c->kv_next;
  r->c = c;
  r->seq = seq;
  CK(cudaLaunchHostFunc(c->kv_stream, kv_commit_cb, r));
  return TG_OK;
}

tg_status tg_kv_committed(tg_ctx *c, uint64_t *seq) {
  if (!c || !seq) return TG_ERR_INVALID;
  *seq = c->kv_committed;
  return TG_OK;
}

tg_status tg_kv_restore(tg_ctx *c, void *dst, size_t bytes, size_t offset, void *stream) {
  if (!c) return TG_ERR_INVALID;
  if (!c->kv_bucket) return fail(c, TG_ERR_NOT_LOADED, "no checkpoint store (tg_kv_store_init)");
  if (!dst || offset > c->kv_bytes || bytes > c->kv_bytes - offset)
    return fail(c, TG_ERR_INVALID, "segment [%zu, +%zu) outside the %zu-byte bucket", offset, bytes, c->kv_bytes);
  CK(cudaSetDevice(c->device));
  CK(cudaStreamSynchronize(c->kv_stream));  // restore only committed state
  CK(cudaMemcpyAsync(dst, c->kv_bucket + offset, bytes, cudaMemcpyHostToDevice, reinterpret_cast<cudaStream_t>(stream)));
  return TG_OK;
}

tg_status tg_finalize(tg_ctx *c) {
  if (!c) return TG_OK;
  if (!c->host_only) {
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    for (int q = 0; q < kMaxWorld; ++q)
      if (c->peer_opened[q]) cudaIpcCloseMemHandle(c->peer[q]);
    cudaFree(c->bank_w1); cudaFree(c->bank_w3); cudaFree(c->bank_w2); cudaFree(c->wg);
    cudaFree(c->w1s); cudaFree(c->w3s); cudaFree(c->w2s);
    cudaFree(c->sym); cudaFree(c->scratch); cudaFree(c->trace); cudaFree(c->maps_dev);
    if (c->err_host) cudaFreeHost(c->err_host);
    for (auto &e : c->ev) cudaEventDestroy(e);
    if (c->kv_stream) cudaStreamDestroy(c->kv_stream);
    if (c->hs_h2d) cudaStreamDestroy(c->hs_h2d);
    if (c->hs_d2h) cudaStreamDestroy(c->hs_d2h);
    for (int i = 0; i < 2; ++i) {
      if (c->ev_h2d[i]) cudaEventDestroy(c->ev_h2d[i]);
      if (c->ev_k[i]) cudaEventDestroy(c->ev_k[i]);
      if (c->ev_d2h[i]) cudaEventDestroy(c->ev_d2h[i]);
    }
    if (c->ev_sync) cudaEventDestroy(c->ev_sync);
    if (c->ev_sync2) cudaEventDestroy(c->ev_sync2);
    if (c->kv_ev) cudaEventDestroy(c->kv_ev);
    if (c->kv_bucket) cudaFreeHost(c->kv_bucket);
  }
  delete c;
  return TG_OK;
}

}  // extern "C"
