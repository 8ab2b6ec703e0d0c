// api.cu -- the C ABI (include/merak_tmp.h): handle, CUDA-IPC peer mapping, and the two-stream
// sub-microbatch scheduler of the sub-pipelined TMP layer (Merak P:571-576, fig:pipedtp(b)).
//
// Streams: cs = computation stream, ms = communication stream ("executing the communication
// stream and computation stream together").  For sub-batch j the compute stream runs the
// column-parallel GEMMs, attention and the row-parallel GEMM whose epilogue writes the partial
// into this rank's peer-visible slot; the comm stream runs the in-kernel NVLink all-reduce of j
// while the compute stream proceeds with sub-batch j+1 ("when one sub-microbatch is
// communicating, the other sub-microbatch will do calculations").  Backward mirrors it with the
// weight-gradient GEMMs filling the all-reduce gaps ("alternate execution schedule").
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <stdarg.h>
#include <stdlib.h>
#include <stdio.h>
#include <string.h>

#include <ucontext.h>

#include <algorithm>
#include <functional>
#include <string>
#include <vector>

#include "../../include/merak_tmp.h"
#include "../../include/merak_tmp_testing.h"
#include "kernels.h"

using namespace mk;
typedef __nv_bfloat16 bf16;

namespace {

constexpr int MAXN = 64;  // max sub-batches
#define MAXN_ 64
constexpr int NSLOT = 5;  // AR#1..AR#4 partial slots (+ the sequence-parallel all-gather slot, index 4)
constexpr int AG_SLOT = 4;

struct ProfRec {
  int cls;
  cudaEvent_t a, b;
  double flops;
  int sid;  // 0 = compute stream, 1 = communication stream
};

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// NCCL baseline (MERAK_COMM_NCCL): resolved at run time from the libnccl.so.2 the process already
// uses (torch's), or from $MERAK_NCCL_LIB.  Only types come from nccl.h.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
  bool load() {
    if (AllReduce) return true;
    void *lib = nullptr;
    const char *env = getenv("MERAK_NCCL_LIB");
    if (env) lib = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) return false;
    GetUniqueId = (decltype(GetUniqueId))dlsym(lib, "ncclGetUniqueId");
    CommInitRank = (decltype(CommInitRank))dlsym(lib, "ncclCommInitRank");
    AllReduce = (decltype(AllReduce))dlsym(lib, "ncclAllReduce");
    CommDestroy = (decltype(CommDestroy))dlsym(lib, "ncclCommDestroy");
    GetErrorString = (decltype(GetErrorString))dlsym(lib, "ncclGetErrorString");
    return GetUniqueId && CommInitRank && AllReduce && CommDestroy && GetErrorString;
  }
};
NcclApi g_nccl;

}  // namespace

struct merak_tmp {
  merak_tmp_config cfg;
  int h, H, s, B, T, r, n, f, d, Hr, hr, fr, e0, M;
  float eps;
  int dev;
  // cs: compute stream of even sub-batches; cs1: odd sub-batches (so one sub-batch's kernels fill the
  // wave-quantisation tails of the other's); cw: weight-gradient GEMMs (lowest priority filler);
  // ms: all-reduces (highest priority).  With MERAK_STREAMS=1, cs1 and cw alias cs.
  cudaStream_t cs = nullptr, cs1 = nullptr, cw = nullptr, ms = nullptr;
  cudaStream_t cr = nullptr;  // LN-gradient sample reductions (off the comm stream, not behind the wgrads)
  // peer-visible memory: NSLOT slots of [M, h] bf16 followed by the flag array
  char *pv = nullptr;
  size_t slot_bytes = 0, flags_off = 0, pv_bytes = 0;
  char *peer_pv[MAX_T] = {};
  uint32_t epoch = 0;
  int *err_host = nullptr, *err_dev = nullptr;
  // workspace
  char *ws = nullptr;
  bf16 *dz = nullptr, *dx1 = nullptr, *dctx = nullptr, *dqkv = nullptr;
  float *delta = nullptr, *part_col = nullptr, *part_lng = nullptr, *part_lnb = nullptr;
  float *dq_acc = nullptr;  // attention backward: fp32 dQ accumulator and its ordering counters
  int *dq_sem = nullptr;
  float *part_lng1 = nullptr, *part_lnb1 = nullptr;  // LN1 (AR#4) partials; part_lng/lnb serve LN2 (AR#3)
  int G = 16;
  // events
  cudaEvent_t ev_entry = nullptr, ev_cs_end = nullptr, ev_cs1_end = nullptr, ev_cw_end = nullptr, ev_cr_end = nullptr;
  bool have_prev = false;
  // workspace hazards across calls: wgrads on cw read dz / dx1 / dqkv that the next backward rewrites
  cudaEvent_t ev_w1 = nullptr, ev_wo = nullptr, ev_wqkv = nullptr, ev_red = nullptr;
  bool have_wg = false;
  cudaEvent_t ev_dz[MAXN] = {}, ev_dq[MAXN] = {};
  cudaEvent_t ev_p[MAXN] = {};
  cudaEvent_t ev_ar[NSLOT][MAXN] = {};
  bool ev_ar_valid[NSLOT][MAXN] = {};
  cudaEvent_t prev_out[MAXN] = {};
  bool chain_open = false;
  // measurement
  bool prof = false;
  std::vector<ProfRec> recs;
  std::vector<cudaEvent_t> evpool;
  size_t evnext = 0;
  double prof_ms[MERAK_K_NUM] = {}, prof_flops[MERAK_K_NUM] = {};
  int64_t prof_launch[MERAK_K_NUM] = {};
  int64_t launches = 0;
  std::string err;
  ncclComm_t nccl = nullptr;
  uint64_t timeout_ns = 20ull * 1000 * 1000 * 1000;  // watchdog (env MERAK_AR_TIMEOUT_MS)
  bool sp = false;        // seq_parallel (T > 1): token-sharded x / y / dx / dy, reduce-scatter + all-gather
  size_t lnx_off = 0;     // sp: peer-visible LN-gradient exchange area [MAXN][4][h] fp32 after the flags
  bf16 *dyf = nullptr;    // sp: the all-gathered dy [M, h] (fc2 dgrad and the W2 wgrad read every token)
  bool use_nvls = false;  // MERAK_COMM_NVLS: slots bound to a multicast object, phase 1 reduced in the switch
  Nvls nvls = {};
  bool fused_wait = false;  // two-shot: phase-1 kernel publishes, phase-2 kernel waits in kernel (env MERAK_AR_FUSED_WAIT)
  bool two_shot = false;  // T >= 4: reduce-scatter + all-gather instead of one-shot (env MERAK_AR_TWO_SHOT)
  // Fused GEMM -> reduce-scatter push (env MERAK_AR_PUSH): the row-parallel GEMMs (proj,
  // fc2, fc1 dgrad, QKV dgrad) store each 32-row output box straight into the slot of the rank that owns the
  // rows (TMA store through a peer tensor map), so the reduce-scatter phase reads only local HBM.
  bool push_req = false, push = false;
  // MERAK_AR_PUSH=2 adds the all-gather push of the replicated two-shot all-reduce: phase 1 stores the reduced owner
  // rows into every rank's all-gather slot (AG_SLOT) over NVLink, so the phase-2 epilogue reads only local HBM
  bool push_ag = false;
  // a row-parallel GEMM pushes only if its compute time covers its NVLink transfer: 2 m N K FLOPs against
  // (T-1)/T m N 2 bytes, i.e. K T / (T-1) >= push_min_k FLOP/byte (~0.75 x 1689 TFLOP/s / 900 GB/s); below it
  // (proj at T = 8: K = h/8) the GEMM would wait on the link, and the pull all-reduce kernel moves the bytes
  // while other kernels hold the tensor cores.  Env MERAK_AR_PUSH_MINK at init.
  int push_min_k = 1400;
  void *push_maps = nullptr;  // device: [4 row-parallel slots][T owners] CUtensorMap (128 B each)
  bool pdl = false;       // programmatic dependent launch along the all-reduce kernel chain (env MERAK_AR_PDL)
  int gemm_smem_kb = 192;  // GEMM TMA ring: 160 KB at T > 1 leaves smem for co-resident all-reduce kernels
  // MERAK_DEBUG_TRACE=1: an event after every launch, per stream (cs, cs1, cw, cr, ms), in a 64-deep ring, so
  // merak_tmp_debug_state can name the first unfinished kernel of a stalled stream
  bool trace = false;
  cudaEvent_t tr_ev[5][64] = {};
  int tr_cls[5][64] = {};
  int64_t tr_seq[5][64] = {};
  int64_t tr_n[5] = {};
  // fp32 check mode (MERAK_FP32_CHECK): fp32 workspace
  bool f32 = false;
  bool local = false;  // MERAK_COMM_LOCAL: single-process emulation of one rank, no peers
  bool broken = false;  // a layer call failed after advancing the handshake epoch: peers are out of step
  bool inproc = false;  // MERAK_COMM_INPROC: the T ranks are handles of one process on one device (init_group)
  int *tile_ctr = nullptr;  // dynamic GEMM tile counters, one per compute stream (cs, cs1); MERAK_GEMM_DYN=1
  char *ws32 = nullptr;
  float *dz32 = nullptr, *dx1_32 = nullptr, *dctx32 = nullptr, *dqkv32 = nullptr, *delta32 = nullptr, *du32 = nullptr;
  struct InprocGroup *grp = nullptr;  // MERAK_COMM_INPROC: the group this rank belongs to
  // LN1 fused into a chained AR#2: a forward with MERAK_FLAG_CHAIN leaves its AR#2s
  // (handshakes and epilogue kernels) unissued; the next call on the handle issues them first -- computing the
  // next layer's LN1 in the epilogues when that call is a forward on y.  Opt-in (MERAK_FUSE_LN1=1): measured
  // 1-5 % slower than LN1 on the compute stream (profiles/r02/fuse_ln1_ab.txt), the LN work lands on the
  // communication stream's critical path.
  bool fuse_ln1 = false;
  bool ar2_pending = false, ar2_comm = false;
  const bf16 *ar2_y = nullptr;
  ArFwdArgs ar2_a[MAXN_];
  cudaEvent_t ev_hs[2] = {};          // INPROC: this rank's handshake points (alternating generations)
};

// ------------------------------------------------------------------------------ in-process groups
// MERAK_COMM_INPROC runs the T ranks of a group as handles of one process on one device.  A spinning handshake
// kernel cannot be used there: the ranks are issued one after another from one host thread, so rank 0's
// handshake of epoch e sits on the GPU before rank 1's work up to epoch e is even issued, and when the two
// ranks' streams share a hardware queue (the device has at most 32; torch's stream pools alone create more)
// rank 1's work queues behind the spinning kernel for good.  Instead a group DEFERS its ranks' layer calls
// until every rank has made the matching call, then issues them together, each rank's call running as a
// coroutine on this thread: at every handshake point a rank records an event on the stream the handshake
// would run on and yields; once all ranks have arrived, each waits on every peer's event and continues.  The
// issue order is then topological (every stream command waits only on commands issued before it), which makes
// the group deadlock-free whatever the stream-to-queue mapping, with the same ordering the handshake kernel
// gives (peer q's partial written and q's earlier readers of my slot done before I proceed).
struct InprocGroup {
  int T = 0;
  merak_tmp_t *hs[MAX_T] = {};
  int alive = 0;                                   // handles not yet destroyed
  std::function<merak_status()> pending[MAX_T];    // deferred layer call of each rank (empty: none)
  int npending = 0;
  bool running = false;                            // the coroutines are issuing
  ucontext_t main_ctx;
  ucontext_t ctx[MAX_T];
  char *stack[MAX_T] = {};
  bool done[MAX_T] = {};
  merak_status status[MAX_T] = {};
  int cur = -1, live = 0, arrive = 0;
  uint64_t gen = 0;
  uint64_t rec_gen[MAX_T] = {};  // generation of each rank's latest handshake event (+1; 0 = none)
};
static constexpr size_t kCoStack = 8u << 20;  // per-rank coroutine stack (the CUDA runtime's launch path is deep)
static thread_local InprocGroup *g_co_group = nullptr;  // the group whose coroutines this thread is running

static void co_entry() {
  InprocGroup *g = g_co_group;
  const int r = g->cur;
  g->status[r] = g->pending[r]();
  g->done[r] = true;
  // a rank that finished (or failed) no longer takes part in the barriers
  if (--g->live > 0 && g->arrive == g->live) {
    g->arrive = 0;
    ++g->gen;
  }
}  // returns to main_ctx through uc_link

static std::string g_init_err;

static merak_status fail(merak_tmp_t *h, merak_status st, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (h)
    h->err = buf;
  else
    g_init_err = buf;
  return st;
}

#define CK(h, call)                                                                                 \
  do {                                                                                              \
    cudaError_t _e = (call);                                                                        \
    if (_e != cudaSuccess) return fail((h), MERAK_ECUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(_e), __FILE__, __LINE__); \
  } while (0)

// ------------------------------------------------------------------------------ measurement
static cudaEvent_t pool_event(merak_tmp_t *h) {
  if (h->evnext == h->evpool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    h->evpool.push_back(e);
  }
  return h->evpool[h->evnext++];
}

struct Launch {
  merak_tmp_t *h;
  int cls;
  cudaStream_t st;
  double flops;
  int nk;
  cudaEvent_t a = nullptr;
  Launch(merak_tmp_t *h_, int cls_, cudaStream_t st_, double flops_, int nk_ = 1)
      : h(h_), cls(cls_), st(st_), flops(flops_), nk(nk_) {
    if (h->prof) {
      a = pool_event(h);
      cudaEventRecord(a, st);
    }
  }
  ~Launch() {
    h->launches += nk;
    if (h->trace) {
      const cudaStream_t ss[5] = {h->cs, h->cs1, h->cw, h->cr, h->ms};
      for (int i = 0; i < 5; ++i)
        if (ss[i] == st) {
          const int k = (int)(h->tr_n[i] % 64);
          cudaEventRecord(h->tr_ev[i][k], st);
          h->tr_cls[i][k] = cls;
          h->tr_seq[i][k] = h->launches;
          ++h->tr_n[i];
          break;
        }
    }
    if (h->prof) {
      cudaEvent_t b = pool_event(h);
      cudaEventRecord(b, st);
      h->recs.push_back({cls, a, b, flops, (st == h->ms && h->ms != h->cs) ? 1 : (st == h->cw && h->cw != h->cs) ? 2 : 0});
      h->prof_launch[cls] += nk;
    }
  }
};

// ------------------------------------------------------------------------------ shapes / layout
// The four activations that are the B operand of a wgrad GEMM (u, ctx, u2, g) carry a pad whose
// first element is 1 after their K columns: the wgrad GEMM then has one extra output column, the
// bias gradient dY^T 1, on the same MMA accumulation chain (bit-identity rule v).  The row stride
// is rounded up to 128 B (64 bf16) past K so every TMA row stays 128-B aligned.
static int padded_ld(int K) { return ((K + 1 + 63) / 64) * 64; }
struct SavedLayout {
  size_t u, mean1, rstd1, qkv, ctx, lse, x1, mean2, rstd2, u2, z, g, total;
  int ld_u, ld_ctx, ld_u2, ld_g;
};
static SavedLayout saved_layout(const merak_tmp_t *h) {
  SavedLayout L;
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t at = o; o += align256(bytes); return at; };
  const size_t M = h->M;
  L.ld_u = L.ld_u2 = padded_ld(h->h);
  L.ld_ctx = padded_ld(h->hr);
  L.ld_g = padded_ld(h->fr);
  L.u = take(M * L.ld_u * 2);
  L.mean1 = take(M * 4);
  L.rstd1 = take(M * 4);
  L.qkv = take(M * 3 * h->hr * 2);
  L.ctx = take(M * L.ld_ctx * 2);
  L.lse = take((size_t)h->B * h->Hr * h->s * 4);
  L.x1 = take(M * h->h * 2);
  L.mean2 = take(M * 4);
  L.rstd2 = take(M * 4);
  L.u2 = take(M * L.ld_u2 * 2);
  L.z = take(M * h->fr * 2);
  L.g = take(M * L.ld_g * 2);
  L.total = o;
  return L;
}

static PeerSync make_sync(merak_tmp_t *h, bool comm) {
  PeerSync ps;
  memset(&ps, 0, sizeof(ps));
  ps.T = h->T;
  ps.rank = h->r;
  ps.enabled = comm && h->T > 1 && !h->nccl;
  ps.epoch = ++h->epoch;
  ps.flags_local = reinterpret_cast<uint32_t *>(h->pv + h->flags_off);
  for (int q = 0; q < h->T; ++q) ps.flags_peer[q] = reinterpret_cast<uint32_t *>(h->peer_pv[q] + h->flags_off);
  ps.err_word = h->err_dev;
  ps.timeout_ns = h->timeout_ns;
  return ps;
}

static bf16 *slot_ptr(merak_tmp_t *h, int rank, int slot) {
  if (h->use_nvls)  // own slots only (multicast-bound memory, unicast mapping); peers' are reached by the switch
    return reinterpret_cast<bf16 *>(reinterpret_cast<char *>(h->nvls.uc_va) + (size_t)slot * h->slot_bytes);
  return reinterpret_cast<bf16 *>(h->peer_pv[rank] + (size_t)slot * h->slot_bytes);
}

// ------------------------------------------------------------------------------ kernel wrappers
static merak_status run_gemm(merak_tmp_t *h, const GemmArgs &a0, cudaStream_t st) {
  GemmArgs a = a0;
  // T > 1: keep smem free on every SM for the all-reduce kernels that overlap the GEMMs
  a.smem_kb = h->gemm_smem_kb;
  if (h->tile_ctr && st != h->cw) a.tile_ctr = h->tile_ctr + (st == h->cs1 && h->cs1 != h->cs ? 1 : 0);
  Launch L(h, MERAK_K_GEMM, st, 2.0 * a.M * a.N * a.K);
  CK(h, gemm(a, st));
  return MERAK_OK;
}
// compute stream of sub-batch j
static cudaStream_t sub_stream(merak_tmp_t *h, int j) { return (j & 1) ? h->cs1 : h->cs; }
static GemmArgs gargs(const void *A, const void *B, int M, int N, int K, int lda, int ldb, bool a_mn, bool b_mn,
                      int epi) {
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  a.A = A; a.B = B; a.M = M; a.N = N; a.K = K; a.lda = lda; a.ldb = ldb; a.a_mn = a_mn; a.b_mn = b_mn; a.epi = epi;
  return a;
}
#define TRY(x)                          \
  do {                                  \
    merak_status _s = (x);              \
    if (_s != MERAK_OK) return _s;      \
  } while (0)

// NCCL baseline: in-place sum of this rank's slot rows on the comm stream; the fused epilogue
// kernel then runs with the single (already reduced) local partial.
static merak_status nccl_allreduce(merak_tmp_t *h, void *rows, size_t count, bool f32 = false,
                                   cudaStream_t st = nullptr) {
  if (!st) st = h->ms;
  Launch L(h, MERAK_K_ALLREDUCE, st, 0.0, 0);
  ncclResult_t r = g_nccl.AllReduce(rows, rows, count, f32 ? ncclFloat32 : ncclBfloat16, ncclSum, h->nccl, st);
  if (r != ncclSuccess) return fail(h, MERAK_ECUDA, "ncclAllReduce: %s", g_nccl.GetErrorString(r));
  return MERAK_OK;
}

// Partials the all-reduce epilogue kernel sums for slot `slot`, rows starting at r0.
static bool push_ag_on(merak_tmp_t *h, bool comm, int m);
static int ar_partials(merak_tmp_t *h, bool comm, int slot, size_t r0, const bf16 **out, int m) {
  if (!comm || h->T == 1 || h->nccl) {
    out[0] = slot_ptr(h, h->r, slot) + r0 * h->h;
    return 1;
  }
  if (push_ag_on(h, comm, m)) {  // every reduced row was pushed into this rank's all-gather slot
    for (int q = 0; q < h->T; ++q) out[q] = slot_ptr(h, h->r, AG_SLOT) + r0 * h->h;
    return h->T;
  }
  // NVLS: after the in-switch reduction every row is in this rank's own slot ("gathered" mode reads locally)
  for (int q = 0; q < h->T; ++q) out[q] = slot_ptr(h, h->use_nvls ? h->r : q, slot) + r0 * h->h;
  return h->T;
}

// 1-warp cross-rank barrier on the communication stream before an all-reduce (see ln_ar.cu)
// In-process groups: the same ordering through events between coroutines (InprocGroup above).
static merak_status group_barrier(merak_tmp_t *h, cudaStream_t st) {
  InprocGroup *g = h->grp;
  if (!g || !g->running) return fail(h, MERAK_ESTATE, "in-process handshake outside a group issue");
  cudaEvent_t mine = h->ev_hs[g->gen & 1];
  CK(h, cudaEventRecord(mine, st));
  const uint64_t gen = g->gen;
  g->rec_gen[h->r] = gen + 1;
  if (++g->arrive == g->live) {
    g->arrive = 0;
    ++g->gen;
  }
  while (g->gen == gen) swapcontext(&g->ctx[h->r], &g->main_ctx);
  // every rank recorded its generation-`gen` event; none can re-record it before all of us passed this point
  for (int q = 0; q < g->T; ++q)
    if (q != h->r && g->rec_gen[q] >= gen + 1) CK(h, cudaStreamWaitEvent(st, g->hs[q]->ev_hs[gen & 1], 0));
  return MERAK_OK;
}

static merak_status sync_peers(merak_tmp_t *h, const PeerSync &ps, cudaStream_t st = nullptr) {
  if (!ps.enabled) return MERAK_OK;
  if (!st) st = h->ms;
  if (h->inproc) return group_barrier(h, st);
  Launch Lk(h, MERAK_K_ALLREDUCE, st, 0.0);
  CK(h, peer_ready(ps, st));
  return MERAK_OK;
}

// Two-shot all-reduce (SURVEY §8(e), T >= 4): each rank sums only the rows it owns,
// [r*chunk, (r+1)*chunk), from all T slots (same arithmetic as one-shot, rounded once) and writes
// them back into its own slot; after a second barrier the fused epilogue kernel reads every row
// from its owner's slot ("gathered" mode).  NVLink bytes per rank: 2(T-1)/T of a slot instead of
// (T-1) for one-shot.  Returns the chunk (rows per owner) for the epilogue kernel.
static bool two_shot_on(merak_tmp_t *h, bool comm) { return comm && h->T > 1 && !h->nccl && h->two_shot; }
// Push layout of a row-parallel slot (h->push, sequence parallel or two-shot, every owner's rows a whole number of
// 32-row boxes): the m rows of sub-batch region r0 in OWNER q's slot hold, at rows [p*m/T, (p+1)*m/T), source
// rank p's partial of q's rows; the reduce-scatter phase then sums T local row blocks in rank order (the same
// arithmetic as pulling them from the peers' slots, so results are bit-identical).
static bool push_rows_ok(merak_tmp_t *h, bool comm, int m) {
  return comm && h->T > 1 && m % h->T == 0 && (m / h->T) % 32 == 0;
}
// K of the row-parallel GEMM writing slot `slot`: proj (h_r), fc2 (f_r), fc1 dgrad (f_r), QKV dgrad (3 h_r)
static int slot_k(const merak_tmp_t *h, int slot) { return slot == 0 ? h->hr : slot == 3 ? 3 * h->hr : h->fr; }
static bool push_on(merak_tmp_t *h, bool comm, int m, int slot) {
  return h->push && (h->sp || two_shot_on(h, comm)) && push_rows_ok(h, comm, m) &&
         (long)slot_k(h, slot) * h->T >= (long)h->push_min_k * (h->T - 1);
}
// All-gather push (h->push_ag): the replicated two-shot all-reduce's phase 1 writes the reduced owner rows into every
// rank's AG_SLOT region of the sub-batch and the phase-2 epilogue reads every row from its own AG_SLOT.  AG_SLOT is
// shared by the 4 all-reduces and both sub-batches: a rank's phase 1 writes a peer's region only after a handshake
// that the peer entered after its previous phase 2 finished reading (all on the in-order communication stream).
// Independent of whether the slot's GEMM pushed (phase 1 reads either layout).
static bool push_ag_on(merak_tmp_t *h, bool comm, int m) {
  return h->push && h->push_ag && !h->sp && two_shot_on(h, comm) && push_rows_ok(h, comm, m);
}
// Output of a row-parallel GEMM into slot `slot`, sub-batch rows from r0: own slot, or pushed to the owners.
static void slot_out(merak_tmp_t *h, GemmArgs &g, bool comm, int slot, size_t r0, int m) {
  g.out = slot_ptr(h, h->r, slot) + r0 * h->h;
  g.ldo = h->h;
  if (push_on(h, comm, m, slot)) {
    g.scatter = reinterpret_cast<const char *>(h->push_maps) + (size_t)slot * h->T * 128;
    g.scatter_rows = m / h->T;
    g.scatter_row0 = (int)r0 + h->r * g.scatter_rows;
  }
}
// Partial q of the own rows [r0 + r*m/T, ...) (sequence parallel) / owner rows (two-shot phase 1) of slot `slot`
static const bf16 *own_partial(merak_tmp_t *h, bool pushed, int slot, size_t r0, int q, int rows_per) {
  if (pushed) return slot_ptr(h, h->r, slot) + (r0 + (size_t)q * rows_per) * h->h;
  return slot_ptr(h, q, slot) + (r0 + (size_t)h->r * rows_per) * h->h;
}
// With h->fused_wait the second handshake kernel disappears: the phase-1 kernel's last CTA publishes the epoch
// and the phase-2 epilogue kernel waits for the peers' epochs in kernel (*wait_ps, PeerSync::wait).  Safe from
// the deadlock of DESIGN.md §7: the waiting kernel depends only on the peers' phase-1 kernels, which precede
// their own phase-2 kernels on their communication streams and never wait themselves.
static merak_status two_shot_rs(merak_tmp_t *h, int slot, size_t r0, int m, const bf16 *resid, const bf16 *bias,
                                int *chunk, PeerSync *wait_ps, bool pushed = false) {
  const int c = (m + h->T - 1) / h->T;
  PeerSync pub = make_sync(h, true);
  pub.publish = h->fused_wait;
  pub.ctr = reinterpret_cast<uint32_t *>(h->pv + h->flags_off) + 64;
  pub.pdl = false;
  if (h->use_nvls) {  // phase 1 in the switch: multimem.ld_reduce of the owned rows, multimem.st to all ranks
    NvlsRsArgs a;
    memset(&a, 0, sizeof(a));
    a.mc = reinterpret_cast<bf16 *>(reinterpret_cast<char *>(h->nvls.mc_va) + (size_t)slot * h->slot_bytes) + r0 * h->h;
    a.h = h->h;
    a.row0 = h->r * c < m ? h->r * c : m;
    a.row1 = (h->r + 1) * c < m ? (h->r + 1) * c : m;
    a.resid = resid;
    a.bias = bias;
    a.ctas = h->cfg.comm_ctas;
    a.pdl = h->pdl && !h->prof;
    a.ps = pub;
    {
      Launch Lk(h, MERAK_K_ALLREDUCE, h->ms, 0.0);
      CK(h, nvls_rs(a, h->ms));
    }
    if (!h->fused_wait) {
      pub.pdl = h->pdl && !h->prof;
      TRY(sync_peers(h, pub));
    }
    pub.wait = h->fused_wait;
    pub.publish = false;
    *wait_ps = pub;
    *chunk = c;
    return MERAK_OK;
  }
  ArRsArgs a;
  memset(&a, 0, sizeof(a));
  // pull: partial q = rank q's slot (rows row0.. read over NVLink); pushed: the T local row blocks (push_on)
  for (int q = 0; q < h->T; ++q)
    a.partial[q] = pushed ? slot_ptr(h, h->r, slot) + ((ptrdiff_t)r0 + (ptrdiff_t)(q - h->r) * c) * h->h
                          : slot_ptr(h, q, slot) + r0 * h->h;
  a.T = h->T; a.h = h->h;
  a.row0 = h->r * c < m ? h->r * c : m;
  a.row1 = (h->r + 1) * c < m ? (h->r + 1) * c : m;
  a.resid = resid; a.bias = bias;
  a.out = slot_ptr(h, h->r, slot) + r0 * h->h;
  if (push_ag_on(h, true, m)) {  // reduced rows straight into every rank's all-gather slot
    a.n_peer = h->T;
    a.rank = h->r;
    for (int q = 0; q < h->T; ++q) a.out_peer[q] = slot_ptr(h, q, AG_SLOT) + r0 * h->h;
  }
  a.ctas = h->cfg.comm_ctas;
  a.pdl = h->pdl && !h->prof;  // (profiling events between launches would break the PDL pairing)
  a.ps = pub;
  {
    Launch Lk(h, MERAK_K_ALLREDUCE, h->ms, 0.0);
    CK(h, ar_rs(a, h->ms));
  }
  if (!h->fused_wait) {
    pub.pdl = h->pdl && !h->prof;
    TRY(sync_peers(h, pub));
  }
  pub.wait = h->fused_wait;
  pub.publish = false;
  *wait_ps = pub;
  *chunk = c;
  return MERAK_OK;
}

static merak_status check_async_error(merak_tmp_t *h) {
  if (h->err_host && *(volatile int *)h->err_host)
    return fail(h, MERAK_ETIMEOUT,
                "peer handshake watchdog fired in a previous all-reduce (peer absent or hung): epoch %d cta %d "
                "kind %d peer %d last flag %d",
                h->err_host[1], h->err_host[2], h->err_host[3] / 16, h->err_host[3] % 16, h->err_host[4]);
  return MERAK_OK;
}

static merak_status enter(merak_tmp_t *h, cudaStream_t st, bool fwd) {
  TRY(check_async_error(h));
  CK(h, cudaSetDevice(h->dev));
  CK(h, cudaEventRecord(h->ev_entry, st));
  for (cudaStream_t c : {h->cs, h->cs1, h->cw, h->cr, h->ms}) CK(h, cudaStreamWaitEvent(c, h->ev_entry, 0));
  // the comm stream rewrites dx1 (AR#3) only after the previous call's readers of it are done:
  // the sub-batch streams (proj dgrad) and the W_o wgrad on cw
  if (h->have_prev) {
    CK(h, cudaStreamWaitEvent(h->ms, h->ev_cs_end, 0));
    CK(h, cudaStreamWaitEvent(h->ms, h->ev_cs1_end, 0));
  }
  if (h->have_wg) {
    CK(h, cudaStreamWaitEvent(h->ms, h->ev_wo, 0));
    CK(h, cudaStreamWaitEvent(h->ms, h->ev_red, 0));
    // a forward rewrites saved activations (u, ctx, x1, u2, z, g) that the previous backward's weight
    // gradients on cw read; the caller may pass the same `saved` buffer again (e.g. a gradient-
    // accumulation loop chained across microbatches), so every writer waits for the filler stream
    if (fwd)
      for (cudaStream_t c : {h->cs, h->cs1, h->ms}) CK(h, cudaStreamWaitEvent(c, h->ev_cw_end, 0));
  }
  return MERAK_OK;
}

static merak_status wait_all(merak_tmp_t *h, cudaStream_t st) {
  CK(h, cudaStreamWaitEvent(st, h->ev_cs_end, 0));
  CK(h, cudaStreamWaitEvent(st, h->ev_cs1_end, 0));
  CK(h, cudaStreamWaitEvent(st, h->ev_cw_end, 0));
  CK(h, cudaStreamWaitEvent(st, h->ev_cr_end, 0));
  return MERAK_OK;
}

static merak_status leave(merak_tmp_t *h, cudaStream_t st, uint32_t flags, int last_slot) {
  CK(h, cudaEventRecord(h->ev_cs_end, h->cs));
  CK(h, cudaEventRecord(h->ev_cs1_end, h->cs1));
  CK(h, cudaEventRecord(h->ev_cw_end, h->cw));
  CK(h, cudaEventRecord(h->ev_cr_end, h->cr));
  h->have_prev = true;
  for (int j = 0; j < h->n; ++j) h->prev_out[j] = h->ev_ar[last_slot][j];
  if (flags & MERAK_FLAG_CHAIN) {
    h->chain_open = true;
  } else {
    TRY(wait_all(h, st));
    CK(h, cudaStreamWaitEvent(st, h->ev_ar[last_slot][h->n - 1], 0));
    h->chain_open = false;
  }
  return MERAK_OK;
}

// ------------------------------------------------------------------------------ forward
// LN1's ones-column pads of u, ctx, u2, g for the rows from r0 of a saved buffer
static OnesPad ln1_pads(const merak_tmp_t *h, const SavedLayout &L, char *saved, size_t r0) {
  OnesPad pad;
  pad.n = 4;
  pad.ptr[0] = (bf16 *)(saved + L.u) + r0 * L.ld_u; pad.ld[0] = L.ld_u; pad.col[0] = h->h;
  pad.ptr[1] = (bf16 *)(saved + L.ctx) + r0 * L.ld_ctx; pad.ld[1] = L.ld_ctx; pad.col[1] = h->hr;
  pad.ptr[2] = (bf16 *)(saved + L.u2) + r0 * L.ld_u2; pad.ld[2] = L.ld_u2; pad.col[2] = h->h;
  pad.ptr[3] = (bf16 *)(saved + L.g) + r0 * L.ld_g; pad.ld[3] = L.ld_g; pad.col[3] = h->fr;
  return pad;
}

// AR#2 of sub-batch j (F8): after fc2(j), the handshake (two-shot: phase 1 + second handshake), then the
// epilogue kernel y = x1 + sum of partials + b_2 -- with do_ln set by the caller, also the next layer's LN1.
static merak_status ar2_issue(merak_tmp_t *h, int j, ArFwdArgs a, bool comm) {
  const size_t r0 = (size_t)j * (h->M / h->n);
  CK(h, cudaStreamWaitEvent(h->ms, h->ev_p[j], 0));
  if (comm && h->nccl) TRY(nccl_allreduce(h, slot_ptr(h, h->r, 1) + r0 * h->h, (size_t)a.m * h->h));
  PeerSync ps = make_sync(h, comm);
  TRY(sync_peers(h, ps));
  if (two_shot_on(h, comm)) TRY(two_shot_rs(h, 1, r0, a.m, a.resid, a.bias, &a.chunk, &ps, push_on(h, comm, a.m, 1)));
  {
    Launch Lk(h, MERAK_K_ALLREDUCE, h->ms, 0.0);
    a.pdl = h->pdl && !h->prof && ps.enabled;  // after the handshake kernel
    CK(h, ar_fwd(a, ps, h->ms));
  }
  CK(h, cudaEventRecord(h->ev_ar[1][j], h->ms));
  h->ev_ar_valid[1][j] = true;
  return MERAK_OK;
}

// Issue the deferred AR#2 of the previous chained forward (every sub-batch in order, each handshake right
// before its epilogue, so AR#2(j) still waits only for fc2(j)).  With w / saved: the layer being entered runs
// on their output y, so each epilogue also computes that layer's LN1 (u, mean1, rstd1 and the ones-column pads
// of its rows in `saved`) -- the same row-engine arithmetic as ln_fwd_kernel on the stored bf16 y, so the
// result is bit-identical to the unfused LN1.  A collective step: every rank flushes at its matching call.
static merak_status flush_ar2(merak_tmp_t *h, const merak_tmp_weights *w = nullptr, char *saved = nullptr) {
  if (!h->ar2_pending) return MERAK_OK;
  h->ar2_pending = false;
  const SavedLayout L = saved_layout(h);
  const int n = h->n, m = h->M / n;
  for (int j = 0; j < n; ++j) {
    ArFwdArgs a = h->ar2_a[j];
    if (w) {
      const size_t r0 = (size_t)j * m;
      a.do_ln = true;
      a.gamma = (const bf16 *)w->ln1_g; a.beta = (const bf16 *)w->ln1_b;
      a.ln_out = (bf16 *)(saved + L.u) + r0 * L.ld_u; a.ld_ln = L.ld_u;
      a.mean = (float *)(saved + L.mean1) + r0; a.rstd = (float *)(saved + L.rstd1) + r0;
      a.eps = h->eps;
      a.pad = ln1_pads(h, L, saved, r0);
    }
    TRY(ar2_issue(h, j, a, h->ar2_comm));
  }
  return MERAK_OK;
}

// recompute = true: the activation-recomputation pass of a MERAK_FLAG_RECOMPUTE backward (SURVEY §8(f) NEXT-3,
// P:459): everything the backward reads is regenerated into `saved` -- the attention block with AR#1 / LN2 and
// fc1 + GeLU -- while fc2 and AR#2 (whose output y the backward never reads) are skipped.  It leaves the chain
// open with each sub-batch's stream event after its fc1, so the backward's first kernels follow directly.
static merak_status layer_fwd(merak_tmp_t *h, const merak_tmp_weights *w, const bf16 *x, bf16 *y, char *saved,
                              uint32_t flags, cudaStream_t st, bool recompute = false) {
  const SavedLayout L = saved_layout(h);
  const int n = h->n, m = h->M / n, b = h->B / n, hh = h->h, hr = h->hr, fr = h->fr;
  const bool comm = !(flags & MERAK_FLAG_NO_COMM) && !h->local;
  TRY(enter(h, st, true));
  // the previous chained layer's AR#2 epilogues, with this layer's LN1 when x is their output
  const bool ln1_fused = h->ar2_pending && !recompute && x == h->ar2_y;
  TRY(flush_ar2(h, ln1_fused ? w : nullptr, ln1_fused ? saved : nullptr));
  // this layer's AR#2 epilogues are deferred to the next call when the chain stays open
  const bool defer_ar2 = (flags & MERAK_FLAG_CHAIN) && !recompute && h->fuse_ln1;
  auto S = [&](size_t off) { return saved + off; };
  // ---- attention block, sub-batch j: LN1 -> QKV -> attention -> proj (partial into slot 0) -> AR#1
  for (int j = 0; j < n; ++j) {
    cudaStream_t cst = sub_stream(h, j);
    if (h->chain_open) CK(h, cudaStreamWaitEvent(cst, h->prev_out[j], 0));
    const size_t r0 = (size_t)j * m;
    const bf16 *xj = x + r0 * hh;
    bf16 *u = (bf16 *)S(L.u) + r0 * L.ld_u;
    float *mean1 = (float *)S(L.mean1) + r0, *rstd1 = (float *)S(L.rstd1) + r0;
    bf16 *qkv = (bf16 *)S(L.qkv) + r0 * 3 * hr;
    bf16 *ctx = (bf16 *)S(L.ctx) + r0 * L.ld_ctx;
    float *lse = (float *)S(L.lse) + (size_t)j * b * h->Hr * h->s;
    if (!ln1_fused) {
      // LN1, which also writes the ones-column pads of u, ctx, u2, g for these rows
      const OnesPad pad = ln1_pads(h, L, saved, r0);
      Launch Lk(h, MERAK_K_LN, cst, 0.0);
      CK(h, ln_fwd(xj, (const bf16 *)w->ln1_g, (const bf16 *)w->ln1_b, u, L.ld_u, mean1, rstd1, m, hh, h->eps, pad,
                   cst));
    }
    GemmArgs g = gargs(u, w->w_qkv, m, 3 * hr, hh, L.ld_u, hh, false, false, EPI_BIAS_BF16);
    g.out = qkv; g.ldo = 3 * hr; g.bias = w->b_qkv;
    TRY(run_gemm(h, g, cst));
    {
      AttnArgs a;
      memset(&a, 0, sizeof(a));
      a.qkv = qkv; a.ctx = ctx; a.ld_ctx = L.ld_ctx; a.lse = lse; a.b = b; a.s = h->s; a.heads = h->Hr; a.d = h->d;
      Launch Lk(h, MERAK_K_ATTN_FWD, cst, 2.0 * b * hr * (double)h->s * (h->s + 1));
      CK(h, attn_fwd(a, cst));
    }
    if (h->ev_ar_valid[0][j]) CK(h, cudaStreamWaitEvent(cst, h->ev_ar[0][j], 0));
    g = gargs(ctx, w->w_o, m, hh, hr, L.ld_ctx, hr, false, false, EPI_STORE_BF16);
    slot_out(h, g, comm, 0, r0, m);
    TRY(run_gemm(h, g, cst));
    CK(h, cudaEventRecord(h->ev_p[j], cst));
    CK(h, cudaStreamWaitEvent(h->ms, h->ev_p[j], 0));
    {
      ArFwdArgs a;
      memset(&a, 0, sizeof(a));
      if (comm && h->nccl) TRY(nccl_allreduce(h, slot_ptr(h, h->r, 0) + r0 * hh, (size_t)m * hh));
      a.T = ar_partials(h, comm, 0, r0, a.partial, m);
      a.m = m; a.h = hh; a.resid = xj; a.bias = (const bf16 *)w->b_o; a.out = (bf16 *)S(L.x1) + r0 * hh;
      a.do_ln = true; a.gamma = (const bf16 *)w->ln2_g; a.beta = (const bf16 *)w->ln2_b;
      a.ln_out = (bf16 *)S(L.u2) + r0 * L.ld_u2; a.ld_ln = L.ld_u2;
      a.mean = (float *)S(L.mean2) + r0; a.rstd = (float *)S(L.rstd2) + r0;
      a.eps = h->eps; a.ctas = h->cfg.comm_ctas;
      PeerSync ps = make_sync(h, comm);
      TRY(sync_peers(h, ps));
      if (two_shot_on(h, comm)) TRY(two_shot_rs(h, 0, r0, m, xj, (const bf16 *)w->b_o, &a.chunk, &ps, push_on(h, comm, m, 0)));
      Launch Lk(h, MERAK_K_ALLREDUCE, h->ms, 0.0);
      a.pdl = h->pdl && !h->prof && ps.enabled;  // after the handshake kernel
      CK(h, ar_fwd(a, ps, h->ms));
    }
    CK(h, cudaEventRecord(h->ev_ar[0][j], h->ms));
    h->ev_ar_valid[0][j] = true;
  }
  // ---- FFN block, sub-batch j: fc1 (+bias+GeLU) -> fc2 (partial into slot 1) -> AR#2
  for (int j = 0; j < n; ++j) {
    cudaStream_t cst = sub_stream(h, j);
    const size_t r0 = (size_t)j * m;
    CK(h, cudaStreamWaitEvent(cst, h->ev_ar[0][j], 0));
    bf16 *u2 = (bf16 *)S(L.u2) + r0 * L.ld_u2;
    bf16 *z = (bf16 *)S(L.z) + r0 * fr, *gg = (bf16 *)S(L.g) + r0 * L.ld_g;
    GemmArgs g = gargs(u2, w->w_1, m, fr, hh, L.ld_u2, hh, false, false, EPI_BIAS_GELU);
    g.out = z; g.ldo = fr; g.out2 = gg; g.ldo2 = L.ld_g; g.bias = w->b_1;
    TRY(run_gemm(h, g, cst));
    if (recompute) {
      CK(h, cudaEventRecord(h->ev_p[j], cst));
      continue;
    }
    if (h->ev_ar_valid[1][j]) CK(h, cudaStreamWaitEvent(cst, h->ev_ar[1][j], 0));
    g = gargs(gg, w->w_2, m, hh, fr, L.ld_g, fr, false, false, EPI_STORE_BF16);
    slot_out(h, g, comm, 1, r0, m);
    TRY(run_gemm(h, g, cst));
    CK(h, cudaEventRecord(h->ev_p[j], cst));
    ArFwdArgs a;
    memset(&a, 0, sizeof(a));
    a.T = ar_partials(h, comm, 1, r0, a.partial, m);
    a.m = m; a.h = hh; a.resid = (const bf16 *)S(L.x1) + r0 * hh; a.bias = (const bf16 *)w->b_2;
    a.out = y + r0 * hh; a.do_ln = false; a.ctas = h->cfg.comm_ctas;
    if (defer_ar2) {  // issued by the next call (flush_ar2), possibly with the next layer's LN1
      h->ar2_a[j] = a;
      continue;
    }
    TRY(ar2_issue(h, j, a, comm));
  }
  if (defer_ar2) {
    h->ar2_pending = true;
    h->ar2_comm = comm;
    h->ar2_y = y;
  }
  if (recompute) {
    TRY(leave(h, st, flags, 0));
    for (int j = 0; j < n; ++j) h->prev_out[j] = h->ev_p[j];  // fc1(j) done (after AR#1(j) on its stream)
    return MERAK_OK;
  }
  return leave(h, st, flags, 1);
}

// wgrad: dW[M', N'] += A_s^T B_s over the sub-batch tokens, with the ones column of B_s giving the
// bias gradient db[M'] in the same accumulation chain.
// Runs on the filler stream cw (lowest priority), after the events that produce its operands.
static merak_status run_wgrad(merak_tmp_t *h, const bf16 *A, int lda, int Mo, const void *B, int ldb, int No, int m,
                              float *dW, float *db) {
  GemmArgs g = gargs(A, B, Mo, No + 1, m, lda, ldb, true, true, EPI_ACC_F32);
  g.out32 = dW; g.ld32 = No; g.db32 = db;
  return run_gemm(h, g, h->cw);
}

// ------------------------------------------------------------------------------ backward
static merak_status layer_bwd(merak_tmp_t *h, const merak_tmp_weights *w, const bf16 *x, const char *saved_c,
                              const bf16 *dy, bf16 *dx, const merak_tmp_grads *gr, uint32_t flags, cudaStream_t st) {
  char *saved = const_cast<char *>(saved_c);
  const SavedLayout L = saved_layout(h);
  const int n = h->n, m = h->M / n, b = h->B / n, hh = h->h, hr = h->hr, fr = h->fr;
  const bool comm = !(flags & MERAK_FLAG_NO_COMM) && !h->local;
  TRY(enter(h, st, false));
  TRY(flush_ar2(h));  // a chained forward's deferred AR#2 epilogues (plain: no LN1 follows)
  auto S = [&](size_t off) { return saved + off; };
  // W2 / b2 grads need only dy and the saved g: they can fill from the start of the backward
  if (h->chain_open)
    for (int j = 0; j < n; ++j) CK(h, cudaStreamWaitEvent(h->cw, h->prev_out[j], 0));
  TRY(run_wgrad(h, dy, hh, hh, (const bf16 *)S(L.g), L.ld_g, fr, h->M, gr->w_2, gr->b_2));
  // ---- FFN block: fc2 dgrad (x GeLU') -> fc1 dgrad (partial, slot 2) -> AR#3 ; wgrads fill the gap
  for (int j = 0; j < n; ++j) {
    cudaStream_t cst = sub_stream(h, j);
    if (h->chain_open) CK(h, cudaStreamWaitEvent(cst, h->prev_out[j], 0));
    if (h->have_wg) CK(h, cudaStreamWaitEvent(cst, h->ev_w1, 0));  // previous W1 wgrad read dz
    const size_t r0 = (size_t)j * m;
    const bf16 *dyj = dy + r0 * hh;
    bf16 *dz = h->dz + r0 * fr;
    GemmArgs g = gargs(dyj, w->w_2, m, fr, hh, hh, fr, false, true, EPI_GELU_BWD);
    g.out = dz; g.ldo = fr; g.aux = (const bf16 *)S(L.z) + r0 * fr; g.ld_aux = fr;
    TRY(run_gemm(h, g, cst));
    CK(h, cudaEventRecord(h->ev_dz[j], cst));
    if (h->ev_ar_valid[2][j]) CK(h, cudaStreamWaitEvent(cst, h->ev_ar[2][j], 0));
    g = gargs(dz, w->w_1, m, hh, fr, fr, hh, false, true, EPI_STORE_BF16);
    slot_out(h, g, comm, 2, r0, m);
    TRY(run_gemm(h, g, cst));
    CK(h, cudaEventRecord(h->ev_p[j], cst));
    CK(h, cudaStreamWaitEvent(h->ms, h->ev_p[j], 0));
    {
      ArBwdArgs a;
      memset(&a, 0, sizeof(a));
      if (comm && h->nccl) TRY(nccl_allreduce(h, slot_ptr(h, h->r, 2) + r0 * hh, (size_t)m * hh));
      a.T = ar_partials(h, comm, 2, r0, a.partial, m);
      a.m = m; a.h = hh; a.x_ln = (const bf16 *)S(L.x1) + r0 * hh;
      a.mean = (const float *)S(L.mean2) + r0; a.rstd = (const float *)S(L.rstd2) + r0;
      a.gamma = (const bf16 *)w->ln2_g; a.dres = dyj; a.dx = h->dx1 + r0 * hh;
      // per-sub-batch region of the 8-row LN partials (the reduction below runs on the filler stream)
      a.part_dg = h->part_lng + (r0 / h->G) * hh; a.part_db = h->part_lnb + (r0 / h->G) * hh;
      a.G = h->G; a.ctas = h->cfg.comm_ctas;
      PeerSync ps = make_sync(h, comm);
      TRY(sync_peers(h, ps));
      if (two_shot_on(h, comm)) TRY(two_shot_rs(h, 2, r0, m, nullptr, nullptr, &a.chunk, &ps, push_on(h, comm, m, 2)));
      {
        Launch Lk(h, MERAK_K_ALLREDUCE, h->ms, 0.0);
        a.pdl = h->pdl && !h->prof && ps.enabled;
        CK(h, ar_bwd(a, ps, h->ms));
      }
    }
    CK(h, cudaEventRecord(h->ev_ar[2][j], h->ms));
    h->ev_ar_valid[2][j] = true;
    {
      // dgamma2 / dbeta2: fixed per-sample tree + chain over samples (rule vi), in sub-batch order on cr,
      // off the communication stream's critical path
      CK(h, cudaStreamWaitEvent(h->cr, h->ev_ar[2][j], 0));
      Launch Lk(h, MERAK_K_REDUCE, h->cr, 0.0, 2);
      CK(h, sample_reduce2(h->part_lng + (r0 / h->G) * hh, h->part_lnb + (r0 / h->G) * hh, h->s / h->G, m / h->s,
                           hh, h->part_col, h->part_col + (size_t)h->B * hh, gr->ln2_g, gr->ln2_b, h->cr));
    }
  }
  // weight + bias gradients of the FFN block over ALL tokens: one accumulation chain over tokens
  // 0..B*s-1 -- the same MMA sequence as n = 1 -- on the filler stream once every dz rows exist.
  for (int j = 0; j < n; ++j) CK(h, cudaStreamWaitEvent(h->cw, h->ev_dz[j], 0));
  TRY(run_wgrad(h, h->dz, fr, fr, (const bf16 *)S(L.u2), L.ld_u2, hh, h->M, gr->w_1, gr->b_1));
  CK(h, cudaEventRecord(h->ev_w1, h->cw));
  // ---- attention block: proj dgrad -> attention bwd -> QKV dgrad (partial, slot 3) -> AR#4
  for (int j = 0; j < n; ++j) {
    cudaStream_t cst = sub_stream(h, j);
    const size_t r0 = (size_t)j * m;
    CK(h, cudaStreamWaitEvent(cst, h->ev_ar[2][j], 0));
    const bf16 *dx1 = h->dx1 + r0 * hh;
    bf16 *dctx = h->dctx + r0 * hr, *dqkv = h->dqkv + r0 * 3 * hr;
    const bf16 *qkv = (const bf16 *)S(L.qkv) + r0 * 3 * hr, *ctx = (const bf16 *)S(L.ctx) + r0 * L.ld_ctx;
    GemmArgs g = gargs(dx1, w->w_o, m, hr, hh, hh, hr, false, true, EPI_STORE_BF16);
    g.out = dctx; g.ldo = hr;
    TRY(run_gemm(h, g, cst));
    if (h->have_wg) CK(h, cudaStreamWaitEvent(cst, h->ev_wqkv, 0));  // previous W_qkv wgrad read dqkv
    {
      AttnArgs a;
      memset(&a, 0, sizeof(a));
      const size_t so = (size_t)j * b * h->Hr * h->s;  // per-sub-batch lse / delta rows
      a.qkv = qkv; a.ctx = (void *)ctx; a.ld_ctx = L.ld_ctx; a.lse = (float *)S(L.lse) + so;
      a.dctx = dctx; a.dqkv = dqkv; a.delta = h->delta + so; a.b = b; a.s = h->s; a.heads = h->Hr; a.d = h->d;
      a.dq_acc = h->dq_acc + so * h->d;
      a.dq_sem = h->dq_sem + (size_t)j * b * h->Hr * ((h->s + 63) / 64);
      Launch Lk(h, MERAK_K_ATTN_BWD, cst, 4.0 * b * hr * (double)h->s * (h->s + 1), 3);
      CK(h, attn_bwd(a, cst));
    }
    CK(h, cudaEventRecord(h->ev_dq[j], cst));
    if (h->ev_ar_valid[3][j]) CK(h, cudaStreamWaitEvent(cst, h->ev_ar[3][j], 0));
    g = gargs(dqkv, w->w_qkv, m, hh, 3 * hr, 3 * hr, hh, false, true, EPI_STORE_BF16);
    slot_out(h, g, comm, 3, r0, m);
    TRY(run_gemm(h, g, cst));
    CK(h, cudaEventRecord(h->ev_p[j], cst));
    CK(h, cudaStreamWaitEvent(h->ms, h->ev_p[j], 0));
    {
      ArBwdArgs a;
      memset(&a, 0, sizeof(a));
      if (comm && h->nccl) TRY(nccl_allreduce(h, slot_ptr(h, h->r, 3) + r0 * hh, (size_t)m * hh));
      a.T = ar_partials(h, comm, 3, r0, a.partial, m);
      a.m = m; a.h = hh; a.x_ln = x + r0 * hh;
      a.mean = (const float *)S(L.mean1) + r0; a.rstd = (const float *)S(L.rstd1) + r0;
      a.gamma = (const bf16 *)w->ln1_g; a.dres = dx1; a.dx = dx + r0 * hh;
      a.part_dg = h->part_lng1 + (r0 / h->G) * hh; a.part_db = h->part_lnb1 + (r0 / h->G) * hh;
      a.G = h->G; a.ctas = h->cfg.comm_ctas;
      PeerSync ps = make_sync(h, comm);
      TRY(sync_peers(h, ps));
      if (two_shot_on(h, comm)) TRY(two_shot_rs(h, 3, r0, m, nullptr, nullptr, &a.chunk, &ps, push_on(h, comm, m, 3)));
      {
        Launch Lk(h, MERAK_K_ALLREDUCE, h->ms, 0.0);
        a.pdl = h->pdl && !h->prof && ps.enabled;
        CK(h, ar_bwd(a, ps, h->ms));
      }
    }
    CK(h, cudaEventRecord(h->ev_ar[3][j], h->ms));
    h->ev_ar_valid[3][j] = true;
    {
      CK(h, cudaStreamWaitEvent(h->cr, h->ev_ar[3][j], 0));
      Launch Lk(h, MERAK_K_REDUCE, h->cr, 0.0, 2);
      CK(h, sample_reduce2(h->part_lng1 + (r0 / h->G) * hh, h->part_lnb1 + (r0 / h->G) * hh, h->s / h->G, m / h->s,
                           hh, h->part_col, h->part_col + (size_t)h->B * hh, gr->ln1_g, gr->ln1_b, h->cr));
    }
  }
  // weight + bias gradients of the attention block over all tokens (filling behind the last AR#4)
  CK(h, cudaStreamWaitEvent(h->cw, h->ev_ar[2][n - 1], 0));  // every dx1 row (AR#3 in order on ms)
  TRY(run_wgrad(h, h->dx1, hh, hh, (const bf16 *)S(L.ctx), L.ld_ctx, hr, h->M, gr->w_o, gr->b_o));
  CK(h, cudaEventRecord(h->ev_wo, h->cw));
  for (int j = 0; j < n; ++j) CK(h, cudaStreamWaitEvent(h->cw, h->ev_dq[j], 0));
  TRY(run_wgrad(h, h->dqkv, 3 * hr, 3 * hr, (const bf16 *)S(L.u), L.ld_u, hh, h->M, gr->w_qkv, gr->b_qkv));
  CK(h, cudaEventRecord(h->ev_wqkv, h->cw));
  CK(h, cudaEventRecord(h->ev_red, h->cr));  // the next backward's AR#3/#4 rewrite the LN partials
  h->have_wg = true;
  return leave(h, st, flags, 3);
}

// ------------------------------------------------------------------------------ sequence parallelism
// seq_parallel (merak_tmp.h): x / y / dx / dy are token shards; rank r owns the rows
// [j*m + r*m/T, j*m + (r+1)*m/T) of sub-batch j (local rows [j*m/T, (j+1)*m/T)).  The row-parallel all-reduces
// become reduce-scatters (the fused epilogue kernels run on the own rows only) and the column-parallel GEMMs'
// inputs come from all-gathers through the peer-visible slot AG_SLOT.  Every writer of AG_SLOT is ordered
// after a handshake that follows the previous all-gather of the same rows (module comment in ln_ar.cu).
static float *lnx_ptr(merak_tmp_t *h, int q, int j, int k) {
  return reinterpret_cast<float *>(h->peer_pv[q] + h->lnx_off) + ((size_t)j * 4 + k) * h->h;
}
static merak_status sp_handshake(merak_tmp_t *h, PeerSync *out = nullptr) {
  PeerSync ps = make_sync(h, true);
  TRY(sync_peers(h, ps));
  if (out) *out = ps;
  return MERAK_OK;
}
// all-gather of the m rows of sub-batch region r0 from every rank's AG_SLOT into dst (row stride ld)
static merak_status sp_gather(merak_tmp_t *h, size_t r0, int m, bf16 *dst, int ld, const OnesPad &pad) {
  AgArgs a;
  memset(&a, 0, sizeof(a));
  for (int q = 0; q < h->T; ++q) a.src[q] = slot_ptr(h, q, AG_SLOT) + r0 * h->h;
  a.T = h->T; a.m = m; a.h = h->h; a.rows_per = m / h->T; a.dst = dst; a.ld_dst = ld;
  Launch Lk(h, MERAK_K_ALLREDUCE, h->ms, 0.0);
  CK(h, ag_rows(a, pad, h->ms));
  return MERAK_OK;
}

static merak_status layer_fwd_sp(merak_tmp_t *h, const merak_tmp_weights *w, const bf16 *x, bf16 *y, char *saved,
                                 uint32_t flags, cudaStream_t st) {
  const SavedLayout L = saved_layout(h);
  const int n = h->n, m = h->M / n, mr = m / h->T, b = h->B / n, hh = h->h, hr = h->hr, fr = h->fr, r = h->r;
  TRY(enter(h, st, true));
  auto S = [&](size_t off) { return saved + off; };
  // ---- attention block, sub-batch j: LN1 (own rows) -> all-gather u -> QKV -> attention -> proj (partial)
  //      -> reduce-scatter + b_o + residual + LN2 (own rows) -> all-gather u2
  for (int j = 0; j < n; ++j) {
    cudaStream_t cst = sub_stream(h, j);
    if (h->chain_open) CK(h, cudaStreamWaitEvent(cst, h->prev_out[j], 0));
    const size_t r0 = (size_t)j * m, l0 = (size_t)j * mr, own = r0 + (size_t)r * mr;
    const bf16 *xj = x + l0 * hh;
    bf16 *ag_own = slot_ptr(h, r, AG_SLOT) + own * hh;
    bf16 *u = (bf16 *)S(L.u) + r0 * L.ld_u;
    bf16 *qkv = (bf16 *)S(L.qkv) + r0 * 3 * hr;
    bf16 *ctx = (bf16 *)S(L.ctx) + r0 * L.ld_ctx;
    float *lse = (float *)S(L.lse) + (size_t)j * b * h->Hr * h->s;
    {
      OnesPad nopad;
      memset(&nopad, 0, sizeof(nopad));
      Launch Lk(h, MERAK_K_LN, cst, 0.0);
      CK(h, ln_fwd(xj, (const bf16 *)w->ln1_g, (const bf16 *)w->ln1_b, ag_own, hh, (float *)S(L.mean1) + l0,
                   (float *)S(L.rstd1) + l0, mr, hh, h->eps, nopad, cst));
    }
    CK(h, cudaEventRecord(h->ev_p[j], cst));
    CK(h, cudaStreamWaitEvent(h->ms, h->ev_p[j], 0));
    TRY(sp_handshake(h));
    {
      OnesPad pad;  // the ones columns of u and ctx for all m rows (wgrad bias columns)
      memset(&pad, 0, sizeof(pad));
      pad.n = 2;
      pad.ptr[0] = u; pad.ld[0] = L.ld_u; pad.col[0] = hh;
      pad.ptr[1] = ctx; pad.ld[1] = L.ld_ctx; pad.col[1] = hr;
      TRY(sp_gather(h, r0, m, u, L.ld_u, pad));
    }
    CK(h, cudaEventRecord(h->ev_ar[AG_SLOT][j], h->ms));
    CK(h, cudaStreamWaitEvent(cst, h->ev_ar[AG_SLOT][j], 0));
    GemmArgs g = gargs(u, w->w_qkv, m, 3 * hr, hh, L.ld_u, hh, false, false, EPI_BIAS_BF16);
    g.out = qkv; g.ldo = 3 * hr; g.bias = w->b_qkv;
    TRY(run_gemm(h, g, cst));
    {
      AttnArgs a;
      memset(&a, 0, sizeof(a));
      a.qkv = qkv; a.ctx = ctx; a.ld_ctx = L.ld_ctx; a.lse = lse; a.b = b; a.s = h->s; a.heads = h->Hr; a.d = h->d;
      Launch Lk(h, MERAK_K_ATTN_FWD, cst, 2.0 * b * hr * (double)h->s * (h->s + 1));
      CK(h, attn_fwd(a, cst));
    }
    if (h->ev_ar_valid[0][j]) CK(h, cudaStreamWaitEvent(cst, h->ev_ar[0][j], 0));
    g = gargs(ctx, w->w_o, m, hh, hr, L.ld_ctx, hr, false, false, EPI_STORE_BF16);
    slot_out(h, g, true, 0, r0, m);
    TRY(run_gemm(h, g, cst));
    CK(h, cudaEventRecord(h->ev_p[j], cst));
    CK(h, cudaStreamWaitEvent(h->ms, h->ev_p[j], 0));
    {
      PeerSync ps;
      TRY(sp_handshake(h, &ps));
      ArFwdArgs a;
      memset(&a, 0, sizeof(a));
      for (int q = 0; q < h->T; ++q) a.partial[q] = own_partial(h, push_on(h, true, m, 0), 0, r0, q, mr);
      a.T = h->T; a.m = mr; a.h = hh; a.resid = xj; a.bias = (const bf16 *)w->b_o;
      a.out = (bf16 *)S(L.x1) + l0 * hh;
      a.do_ln = true; a.gamma = (const bf16 *)w->ln2_g; a.beta = (const bf16 *)w->ln2_b;
      a.ln_out = ag_own; a.ld_ln = hh;  // u2 rows for the all-gather
      a.mean = (float *)S(L.mean2) + l0; a.rstd = (float *)S(L.rstd2) + l0;
      a.eps = h->eps; a.ctas = h->cfg.comm_ctas;
      Launch Lk(h, MERAK_K_ALLREDUCE, h->ms, 0.0);
      CK(h, ar_fwd(a, ps, h->ms));
    }
    TRY(sp_handshake(h));
    {
      OnesPad pad;  // the ones columns of u2 and g
      memset(&pad, 0, sizeof(pad));
      pad.n = 2;
      pad.ptr[0] = (bf16 *)S(L.u2) + r0 * L.ld_u2; pad.ld[0] = L.ld_u2; pad.col[0] = hh;
      pad.ptr[1] = (bf16 *)S(L.g) + r0 * L.ld_g; pad.ld[1] = L.ld_g; pad.col[1] = fr;
      TRY(sp_gather(h, r0, m, (bf16 *)S(L.u2) + r0 * L.ld_u2, L.ld_u2, pad));
    }
    CK(h, cudaEventRecord(h->ev_ar[0][j], h->ms));
    h->ev_ar_valid[0][j] = true;
  }
  // ---- FFN block, sub-batch j: fc1 (+bias+GeLU) -> fc2 (partial) -> reduce-scatter + b_2 + residual (own rows)
  for (int j = 0; j < n; ++j) {
    cudaStream_t cst = sub_stream(h, j);
    const size_t r0 = (size_t)j * m, l0 = (size_t)j * mr, own = r0 + (size_t)r * mr;
    CK(h, cudaStreamWaitEvent(cst, h->ev_ar[0][j], 0));
    bf16 *u2 = (bf16 *)S(L.u2) + r0 * L.ld_u2;
    bf16 *z = (bf16 *)S(L.z) + r0 * fr, *gg = (bf16 *)S(L.g) + r0 * L.ld_g;
    GemmArgs g = gargs(u2, w->w_1, m, fr, hh, L.ld_u2, hh, false, false, EPI_BIAS_GELU);
    g.out = z; g.ldo = fr; g.out2 = gg; g.ldo2 = L.ld_g; g.bias = w->b_1;
    TRY(run_gemm(h, g, cst));
    if (h->ev_ar_valid[1][j]) CK(h, cudaStreamWaitEvent(cst, h->ev_ar[1][j], 0));
    g = gargs(gg, w->w_2, m, hh, fr, L.ld_g, fr, false, false, EPI_STORE_BF16);
    slot_out(h, g, true, 1, r0, m);
    TRY(run_gemm(h, g, cst));
    CK(h, cudaEventRecord(h->ev_p[j], cst));
    CK(h, cudaStreamWaitEvent(h->ms, h->ev_p[j], 0));
    {
      PeerSync ps;
      TRY(sp_handshake(h, &ps));
      ArFwdArgs a;
      memset(&a, 0, sizeof(a));
      for (int q = 0; q < h->T; ++q) a.partial[q] = own_partial(h, push_on(h, true, m, 1), 1, r0, q, mr);
      a.T = h->T; a.m = mr; a.h = hh; a.resid = (const bf16 *)S(L.x1) + l0 * hh; a.bias = (const bf16 *)w->b_2;
      a.out = y + l0 * hh; a.do_ln = false; a.ctas = h->cfg.comm_ctas;
      Launch Lk(h, MERAK_K_ALLREDUCE, h->ms, 0.0);
      CK(h, ar_fwd(a, ps, h->ms));
    }
    CK(h, cudaEventRecord(h->ev_ar[1][j], h->ms));
    h->ev_ar_valid[1][j] = true;
  }
  return leave(h, st, flags, 1);
}

static merak_status layer_bwd_sp(merak_tmp_t *h, const merak_tmp_weights *w, const bf16 *x, const char *saved_c,
                                 const bf16 *dy, bf16 *dx, const merak_tmp_grads *gr, uint32_t flags, cudaStream_t st) {
  char *saved = const_cast<char *>(saved_c);
  const SavedLayout L = saved_layout(h);
  const int n = h->n, m = h->M / n, mr = m / h->T, b = h->B / n, hh = h->h, hr = h->hr, fr = h->fr, r = h->r;
  TRY(enter(h, st, false));
  auto S = [&](size_t off) { return saved + off; };
  // ---- FFN block: all-gather dy -> fc2 dgrad (x GeLU') -> fc1 dgrad (partial) -> reduce-scatter + LN2 backward
  //      (own rows) -> all-gather dx1; LN2 gradients: own rows, then ranks in order
  for (int j = 0; j < n; ++j) {
    cudaStream_t cst = sub_stream(h, j);
    if (h->chain_open) CK(h, cudaStreamWaitEvent(cst, h->prev_out[j], 0));
    if (h->have_wg) CK(h, cudaStreamWaitEvent(cst, h->ev_w1, 0));  // previous W1 wgrad read dz
    const size_t r0 = (size_t)j * m, l0 = (size_t)j * mr, own = r0 + (size_t)r * mr;
    bf16 *ag_own = slot_ptr(h, r, AG_SLOT) + own * hh;
    {
      Launch Lk(h, MERAK_K_ALLREDUCE, h->ms, 0.0);
      CK(h, copy_rows(dy + l0 * hh, hh, ag_own, hh, mr, hh, h->ms));
    }
    TRY(sp_handshake(h));
    {
      OnesPad nopad;
      memset(&nopad, 0, sizeof(nopad));
      TRY(sp_gather(h, r0, m, h->dyf + r0 * hh, hh, nopad));
    }
    CK(h, cudaEventRecord(h->ev_ar[AG_SLOT][j], h->ms));
    CK(h, cudaStreamWaitEvent(cst, h->ev_ar[AG_SLOT][j], 0));
    bf16 *dz = h->dz + r0 * fr;
    GemmArgs g = gargs(h->dyf + r0 * hh, w->w_2, m, fr, hh, hh, fr, false, true, EPI_GELU_BWD);
    g.out = dz; g.ldo = fr; g.aux = (const bf16 *)S(L.z) + r0 * fr; g.ld_aux = fr;
    TRY(run_gemm(h, g, cst));
    CK(h, cudaEventRecord(h->ev_dz[j], cst));
    if (h->ev_ar_valid[2][j]) CK(h, cudaStreamWaitEvent(cst, h->ev_ar[2][j], 0));
    g = gargs(dz, w->w_1, m, hh, fr, fr, hh, false, true, EPI_STORE_BF16);
    slot_out(h, g, true, 2, r0, m);
    TRY(run_gemm(h, g, cst));
    CK(h, cudaEventRecord(h->ev_p[j], cst));
    CK(h, cudaStreamWaitEvent(h->ms, h->ev_p[j], 0));
    {
      PeerSync ps;
      TRY(sp_handshake(h, &ps));
      ArBwdArgs a;
      memset(&a, 0, sizeof(a));
      for (int q = 0; q < h->T; ++q) a.partial[q] = own_partial(h, push_on(h, true, m, 2), 2, r0, q, mr);
      a.T = h->T; a.m = mr; a.h = hh; a.x_ln = (const bf16 *)S(L.x1) + l0 * hh;
      a.mean = (const float *)S(L.mean2) + l0; a.rstd = (const float *)S(L.rstd2) + l0;
      a.gamma = (const bf16 *)w->ln2_g; a.dres = dy + l0 * hh; a.dx = ag_own;  // dx1 rows for the all-gather
      a.part_dg = h->part_lng + (l0 / h->G) * hh; a.part_db = h->part_lnb + (l0 / h->G) * hh;
      a.G = h->G; a.ctas = h->cfg.comm_ctas;
      Launch Lk(h, MERAK_K_ALLREDUCE, h->ms, 0.0);
      CK(h, ar_bwd(a, ps, h->ms));
    }
    {
      Launch Lk(h, MERAK_K_REDUCE, h->ms, 0.0);
      CK(h, group_chain2(h->part_lng + (l0 / h->G) * hh, h->part_lnb + (l0 / h->G) * hh, mr / h->G, hh,
                         lnx_ptr(h, r, j, 0), lnx_ptr(h, r, j, 1), h->ms));
    }
    TRY(sp_handshake(h));  // every rank's dx1 rows and LN2 partials are written
    {
      OnesPad nopad;
      memset(&nopad, 0, sizeof(nopad));
      TRY(sp_gather(h, r0, m, h->dx1 + r0 * hh, hh, nopad));
    }
    {
      const float *s0[MAX_T], *s1[MAX_T];
      for (int q = 0; q < h->T; ++q) {
        s0[q] = lnx_ptr(h, q, j, 0);
        s1[q] = lnx_ptr(h, q, j, 1);
      }
      Launch Lk(h, MERAK_K_REDUCE, h->ms, 0.0);
      CK(h, rank_sum_add2(s0, s1, h->T, hh, gr->ln2_g, gr->ln2_b, h->ms));
    }
    CK(h, cudaEventRecord(h->ev_ar[2][j], h->ms));
    h->ev_ar_valid[2][j] = true;
  }
  // weight + bias gradients of the FFN block over ALL tokens (one accumulation chain, as without sp)
  for (int j = 0; j < n; ++j) CK(h, cudaStreamWaitEvent(h->cw, h->ev_ar[AG_SLOT][j], 0));
  TRY(run_wgrad(h, h->dyf, hh, hh, (const bf16 *)S(L.g), L.ld_g, fr, h->M, gr->w_2, gr->b_2));
  for (int j = 0; j < n; ++j) CK(h, cudaStreamWaitEvent(h->cw, h->ev_dz[j], 0));
  TRY(run_wgrad(h, h->dz, fr, fr, (const bf16 *)S(L.u2), L.ld_u2, hh, h->M, gr->w_1, gr->b_1));
  CK(h, cudaEventRecord(h->ev_w1, h->cw));
  // ---- attention block: proj dgrad -> attention bwd -> QKV dgrad (partial) -> reduce-scatter + LN1 backward
  for (int j = 0; j < n; ++j) {
    cudaStream_t cst = sub_stream(h, j);
    const size_t r0 = (size_t)j * m, l0 = (size_t)j * mr, own = r0 + (size_t)r * mr;
    CK(h, cudaStreamWaitEvent(cst, h->ev_ar[2][j], 0));
    const bf16 *dx1 = h->dx1 + r0 * hh;
    bf16 *dctx = h->dctx + r0 * hr, *dqkv = h->dqkv + r0 * 3 * hr;
    const bf16 *qkv = (const bf16 *)S(L.qkv) + r0 * 3 * hr, *ctx = (const bf16 *)S(L.ctx) + r0 * L.ld_ctx;
    GemmArgs g = gargs(dx1, w->w_o, m, hr, hh, hh, hr, false, true, EPI_STORE_BF16);
    g.out = dctx; g.ldo = hr;
    TRY(run_gemm(h, g, cst));
    if (h->have_wg) CK(h, cudaStreamWaitEvent(cst, h->ev_wqkv, 0));  // previous W_qkv wgrad read dqkv
    {
      AttnArgs a;
      memset(&a, 0, sizeof(a));
      const size_t so = (size_t)j * b * h->Hr * h->s;
      a.qkv = qkv; a.ctx = (void *)ctx; a.ld_ctx = L.ld_ctx; a.lse = (float *)S(L.lse) + so;
      a.dctx = dctx; a.dqkv = dqkv; a.delta = h->delta + so; a.b = b; a.s = h->s; a.heads = h->Hr; a.d = h->d;
      a.dq_acc = h->dq_acc + so * h->d;
      a.dq_sem = h->dq_sem + (size_t)j * b * h->Hr * ((h->s + 63) / 64);
      Launch Lk(h, MERAK_K_ATTN_BWD, cst, 4.0 * b * hr * (double)h->s * (h->s + 1), 3);
      CK(h, attn_bwd(a, cst));
    }
    CK(h, cudaEventRecord(h->ev_dq[j], cst));
    if (h->ev_ar_valid[3][j]) CK(h, cudaStreamWaitEvent(cst, h->ev_ar[3][j], 0));
    g = gargs(dqkv, w->w_qkv, m, hh, 3 * hr, 3 * hr, hh, false, true, EPI_STORE_BF16);
    slot_out(h, g, true, 3, r0, m);
    TRY(run_gemm(h, g, cst));
    CK(h, cudaEventRecord(h->ev_p[j], cst));
    CK(h, cudaStreamWaitEvent(h->ms, h->ev_p[j], 0));
    {
      PeerSync ps;
      TRY(sp_handshake(h, &ps));
      ArBwdArgs a;
      memset(&a, 0, sizeof(a));
      for (int q = 0; q < h->T; ++q) a.partial[q] = own_partial(h, push_on(h, true, m, 3), 3, r0, q, mr);
      a.T = h->T; a.m = mr; a.h = hh; a.x_ln = x + l0 * hh;
      a.mean = (const float *)S(L.mean1) + l0; a.rstd = (const float *)S(L.rstd1) + l0;
      a.gamma = (const bf16 *)w->ln1_g; a.dres = h->dx1 + own * hh; a.dx = dx + l0 * hh;
      a.part_dg = h->part_lng1 + (l0 / h->G) * hh; a.part_db = h->part_lnb1 + (l0 / h->G) * hh;
      a.G = h->G; a.ctas = h->cfg.comm_ctas;
      Launch Lk(h, MERAK_K_ALLREDUCE, h->ms, 0.0);
      CK(h, ar_bwd(a, ps, h->ms));
    }
    {
      Launch Lk(h, MERAK_K_REDUCE, h->ms, 0.0);
      CK(h, group_chain2(h->part_lng1 + (l0 / h->G) * hh, h->part_lnb1 + (l0 / h->G) * hh, mr / h->G, hh,
                         lnx_ptr(h, r, j, 2), lnx_ptr(h, r, j, 3), h->ms));
    }
    TRY(sp_handshake(h));  // every rank's LN1 partials are written
    {
      const float *s0[MAX_T], *s1[MAX_T];
      for (int q = 0; q < h->T; ++q) {
        s0[q] = lnx_ptr(h, q, j, 2);
        s1[q] = lnx_ptr(h, q, j, 3);
      }
      Launch Lk(h, MERAK_K_REDUCE, h->ms, 0.0);
      CK(h, rank_sum_add2(s0, s1, h->T, hh, gr->ln1_g, gr->ln1_b, h->ms));
    }
    CK(h, cudaEventRecord(h->ev_ar[3][j], h->ms));
    h->ev_ar_valid[3][j] = true;
  }
  CK(h, cudaStreamWaitEvent(h->cw, h->ev_ar[2][n - 1], 0));  // every dx1 row (the all-gathers run in order on ms)
  TRY(run_wgrad(h, h->dx1, hh, hh, (const bf16 *)S(L.ctx), L.ld_ctx, hr, h->M, gr->w_o, gr->b_o));
  CK(h, cudaEventRecord(h->ev_wo, h->cw));
  for (int j = 0; j < n; ++j) CK(h, cudaStreamWaitEvent(h->cw, h->ev_dq[j], 0));
  TRY(run_wgrad(h, h->dqkv, 3 * hr, 3 * hr, (const bf16 *)S(L.u), L.ld_u, hh, h->M, gr->w_qkv, gr->b_qkv));
  CK(h, cudaEventRecord(h->ev_wqkv, h->cw));
  CK(h, cudaEventRecord(h->ev_red, h->ms));  // the next backward rewrites the LN partials (on ms as well)
  h->have_wg = true;
  return leave(h, st, flags, 3);
}

// ------------------------------------------------------------------------------ fp32 check mode
// MERAK_FP32_CHECK: the same method (sharding, sub-batch loop, rank-ordered all-reduces, token-order
// reductions) with every tensor fp32 and the simple kernels of check_f32.cu, all on the compute
// stream (peer handshakes included).  x, y, dx, dy, weights and saved activations are fp32.
struct SavedF32 {
  size_t u, mean1, rstd1, qkv, ctx, lse, x1, mean2, rstd2, u2, z, g, total;
};
static SavedF32 saved_f32(const merak_tmp_t *h) {
  SavedF32 L;
  size_t o = 0;
  auto take = [&](size_t elems) { size_t at = o; o += align256(elems * 4); return at; };
  const size_t M = h->M;
  L.u = take(M * h->h); L.mean1 = take(M); L.rstd1 = take(M);
  L.qkv = take(M * 3 * h->hr); L.ctx = take(M * h->hr); L.lse = take((size_t)h->B * h->Hr * h->s);
  L.x1 = take(M * h->h); L.mean2 = take(M); L.rstd2 = take(M); L.u2 = take(M * h->h);
  L.z = take(M * h->fr); L.g = take(M * h->fr);
  L.total = o;
  return L;
}

static F32GemmArgs g32(const float *A, const float *B, int M, int N, int K, int lda, int ldb, bool a_mn, bool b_mn,
                       int epi, float *C, int ldc) {
  F32GemmArgs a;
  memset(&a, 0, sizeof(a));
  a.A = A; a.B = B; a.M = M; a.N = N; a.K = K; a.lda = lda; a.ldb = ldb; a.a_mn = a_mn; a.b_mn = b_mn;
  a.epi = epi; a.C = C; a.ldc = ldc;
  return a;
}
static merak_status run_g32(merak_tmp_t *h, const F32GemmArgs &a) {
  Launch L(h, MERAK_K_GEMM, h->cs, 2.0 * a.M * a.N * a.K);
  CK(h, f32_gemm(a, h->cs));
  return MERAK_OK;
}
static float *slot32(merak_tmp_t *h, int rank, int slot) {
  return reinterpret_cast<float *>(h->peer_pv[rank] + (size_t)slot * h->slot_bytes);
}
// all-reduce prologue: NCCL sum or peer handshake; fills the rank-ordered partial pointers
static merak_status ar32_prologue(merak_tmp_t *h, bool comm, int slot, size_t r0, int m, F32ArArgs &a) {
  float *mine = slot32(h, h->r, slot) + r0 * h->h;
  if (comm && h->T > 1 && h->nccl) TRY(nccl_allreduce(h, mine, (size_t)m * h->h, true, h->cs));
  if (!comm || h->T == 1 || h->nccl) {
    a.T = 1;
    a.partial[0] = mine;
  } else {
    a.T = h->T;
    for (int q = 0; q < h->T; ++q) a.partial[q] = slot32(h, q, slot) + r0 * h->h;
    PeerSync ps = make_sync(h, comm);
    TRY(sync_peers(h, ps, h->cs));
  }
  a.m = m; a.h = h->h; a.eps = h->eps;
  return MERAK_OK;
}

static merak_status layer_fwd_f32(merak_tmp_t *h, const merak_tmp_weights *w, const float *x, float *y, char *saved,
                                  uint32_t flags, cudaStream_t st) {
  const SavedF32 L = saved_f32(h);
  const int n = h->n, m = h->M / n, b = h->B / n, hh = h->h, hr = h->hr, fr = h->fr;
  const bool comm = !(flags & MERAK_FLAG_NO_COMM) && !h->local;
  cudaStream_t c = h->cs;
  TRY(enter(h, st, true));
  auto S = [&](size_t off) { return reinterpret_cast<float *>(saved + off); };
  for (int j = 0; j < n; ++j) {  // attention block
    if (h->chain_open) CK(h, cudaStreamWaitEvent(c, h->prev_out[j], 0));
    const size_t r0 = (size_t)j * m;
    const float *xj = x + r0 * hh;
    float *u = S(L.u) + r0 * hh, *qkv = S(L.qkv) + r0 * 3 * hr, *ctx = S(L.ctx) + r0 * hr;
    {
      Launch Lk(h, MERAK_K_LN, c, 0.0);
      CK(h, f32_ln_fwd(xj, (const float *)w->ln1_g, (const float *)w->ln1_b, u, S(L.mean1) + r0, S(L.rstd1) + r0, m,
                       hh, h->eps, c));
    }
    F32GemmArgs g = g32(u, (const float *)w->w_qkv, m, 3 * hr, hh, hh, hh, false, false, EPI_BIAS_BF16, qkv, 3 * hr);
    g.bias = (const float *)w->b_qkv;
    TRY(run_g32(h, g));
    {
      F32AttnArgs a;
      memset(&a, 0, sizeof(a));
      a.qkv = qkv; a.ctx = ctx; a.lse = S(L.lse) + (size_t)j * b * h->Hr * h->s;
      a.b = b; a.s = h->s; a.heads = h->Hr; a.d = h->d;
      Launch Lk(h, MERAK_K_ATTN_FWD, c, 2.0 * b * hr * (double)h->s * (h->s + 1));
      CK(h, f32_attn_fwd(a, c));
    }
    TRY(run_g32(h, g32(ctx, (const float *)w->w_o, m, hh, hr, hr, hr, false, false, EPI_STORE_BF16,
                       slot32(h, h->r, 0) + r0 * hh, hh)));
    F32ArArgs a;
    memset(&a, 0, sizeof(a));
    TRY(ar32_prologue(h, comm, 0, r0, m, a));
    a.resid = xj; a.bias = (const float *)w->b_o; a.out = S(L.x1) + r0 * hh;
    a.ln_out = S(L.u2) + r0 * hh; a.gamma = (const float *)w->ln2_g; a.beta = (const float *)w->ln2_b;
    a.mean = S(L.mean2) + r0; a.rstd = S(L.rstd2) + r0;
    {
      Launch Lk(h, MERAK_K_ALLREDUCE, c, 0.0);
      CK(h, f32_ar_fwd(a, c));
    }
    CK(h, cudaEventRecord(h->ev_ar[0][j], c));
  }
  for (int j = 0; j < n; ++j) {  // FFN block
    const size_t r0 = (size_t)j * m;
    F32GemmArgs g = g32(S(L.u2) + r0 * hh, (const float *)w->w_1, m, fr, hh, hh, hh, false, false, EPI_BIAS_GELU,
                        S(L.z) + r0 * fr, fr);
    g.C2 = S(L.g) + r0 * fr; g.ldc2 = fr; g.bias = (const float *)w->b_1;
    TRY(run_g32(h, g));
    TRY(run_g32(h, g32(S(L.g) + r0 * fr, (const float *)w->w_2, m, hh, fr, fr, fr, false, false, EPI_STORE_BF16,
                       slot32(h, h->r, 1) + r0 * hh, hh)));
    F32ArArgs a;
    memset(&a, 0, sizeof(a));
    TRY(ar32_prologue(h, comm, 1, r0, m, a));
    a.resid = S(L.x1) + r0 * hh; a.bias = (const float *)w->b_2; a.out = y + r0 * hh;
    {
      Launch Lk(h, MERAK_K_ALLREDUCE, c, 0.0);
      CK(h, f32_ar_fwd(a, c));
    }
    CK(h, cudaEventRecord(h->ev_ar[1][j], c));
  }
  return leave(h, st, flags, 1);
}

static merak_status layer_bwd_f32(merak_tmp_t *h, const merak_tmp_weights *w, const float *x, const char *saved_c,
                                  const float *dy, float *dx, const merak_tmp_grads *gr, uint32_t flags,
                                  cudaStream_t st) {
  char *saved = const_cast<char *>(saved_c);
  const SavedF32 L = saved_f32(h);
  const int n = h->n, m = h->M / n, b = h->B / n, hh = h->h, hr = h->hr, fr = h->fr, M = h->M;
  const bool comm = !(flags & MERAK_FLAG_NO_COMM) && !h->local;
  cudaStream_t c = h->cs;
  TRY(enter(h, st, false));
  auto S = [&](size_t off) { return reinterpret_cast<float *>(saved + off); };
  auto chain = [&](const float *X, int ld, int cols, float *out) -> merak_status {
    Launch Lk(h, MERAK_K_REDUCE, c, 0.0);
    CK(h, f32_colsum_chain(X, ld, M, cols, out, c));
    return MERAK_OK;
  };
  for (int j = 0; j < n; ++j) {  // FFN block: fc2 dgrad (x GeLU') -> fc1 dgrad -> AR#3
    if (h->chain_open) CK(h, cudaStreamWaitEvent(c, h->prev_out[j], 0));
    const size_t r0 = (size_t)j * m;
    F32GemmArgs g = g32(dy + r0 * hh, (const float *)w->w_2, m, fr, hh, hh, fr, false, true, EPI_GELU_BWD,
                        h->dz32 + r0 * fr, fr);
    g.aux = S(L.z) + r0 * fr; g.ld_aux = fr;
    TRY(run_g32(h, g));
    TRY(run_g32(h, g32(h->dz32 + r0 * fr, (const float *)w->w_1, m, hh, fr, fr, hh, false, true, EPI_STORE_BF16,
                       slot32(h, h->r, 2) + r0 * hh, hh)));
    F32ArArgs a;
    memset(&a, 0, sizeof(a));
    TRY(ar32_prologue(h, comm, 2, r0, m, a));
    a.x_ln = S(L.x1) + r0 * hh; a.mean = S(L.mean2) + r0; a.rstd = S(L.rstd2) + r0;
    a.gamma = (const float *)w->ln2_g; a.dres = dy + r0 * hh; a.out = h->dx1_32 + r0 * hh; a.du = h->du32 + r0 * hh;
    {
      Launch Lk(h, MERAK_K_ALLREDUCE, c, 0.0);
      CK(h, f32_ar_bwd(a, c));
    }
    CK(h, cudaEventRecord(h->ev_ar[2][j], c));
  }
  // FFN weight / bias / LN2 grads over all tokens in token order
  TRY(run_g32(h, g32(dy, S(L.g), hh, fr, M, hh, fr, true, true, EPI_ACC_F32, gr->w_2, fr)));
  TRY(chain(dy, hh, hh, gr->b_2));
  TRY(run_g32(h, g32(h->dz32, S(L.u2), fr, hh, M, fr, hh, true, true, EPI_ACC_F32, gr->w_1, hh)));
  TRY(chain(h->dz32, fr, fr, gr->b_1));
  {
    Launch Lk(h, MERAK_K_REDUCE, c, 0.0);
    CK(h, f32_ln_grad_chain(h->du32, S(L.x1), S(L.mean2), S(L.rstd2), M, hh, gr->ln2_g, gr->ln2_b, c));
  }
  for (int j = 0; j < n; ++j) {  // attention block: proj dgrad -> attention bwd -> QKV dgrad -> AR#4
    const size_t r0 = (size_t)j * m;
    TRY(run_g32(h, g32(h->dx1_32 + r0 * hh, (const float *)w->w_o, m, hr, hh, hh, hr, false, true, EPI_STORE_BF16,
                       h->dctx32 + r0 * hr, hr)));
    {
      F32AttnArgs a;
      memset(&a, 0, sizeof(a));
      const size_t so = (size_t)j * b * h->Hr * h->s;
      a.qkv = S(L.qkv) + r0 * 3 * hr; a.ctx = S(L.ctx) + r0 * hr; a.lse = S(L.lse) + so;
      a.dctx = h->dctx32 + r0 * hr; a.dqkv = h->dqkv32 + r0 * 3 * hr; a.delta = h->delta32 + so;
      a.b = b; a.s = h->s; a.heads = h->Hr; a.d = h->d;
      Launch Lk(h, MERAK_K_ATTN_BWD, c, 4.0 * b * hr * (double)h->s * (h->s + 1), 2);
      CK(h, f32_attn_bwd(a, c));
    }
    TRY(run_g32(h, g32(h->dqkv32 + r0 * 3 * hr, (const float *)w->w_qkv, m, hh, 3 * hr, 3 * hr, hh, false, true,
                       EPI_STORE_BF16, slot32(h, h->r, 3) + r0 * hh, hh)));
    F32ArArgs a;
    memset(&a, 0, sizeof(a));
    TRY(ar32_prologue(h, comm, 3, r0, m, a));
    a.x_ln = x + r0 * hh; a.mean = S(L.mean1) + r0; a.rstd = S(L.rstd1) + r0;
    a.gamma = (const float *)w->ln1_g; a.dres = h->dx1_32 + r0 * hh; a.out = dx + r0 * hh; a.du = h->du32 + r0 * hh;
    {
      Launch Lk(h, MERAK_K_ALLREDUCE, c, 0.0);
      CK(h, f32_ar_bwd(a, c));
    }
    CK(h, cudaEventRecord(h->ev_ar[3][j], c));
  }
  TRY(run_g32(h, g32(h->dx1_32, S(L.ctx), hh, hr, M, hh, hr, true, true, EPI_ACC_F32, gr->w_o, hr)));
  TRY(chain(h->dx1_32, hh, hh, gr->b_o));
  TRY(run_g32(h, g32(h->dqkv32, S(L.u), 3 * hr, hh, M, 3 * hr, hh, true, true, EPI_ACC_F32, gr->w_qkv, hh)));
  TRY(chain(h->dqkv32, 3 * hr, 3 * hr, gr->b_qkv));
  {
    Launch Lk(h, MERAK_K_REDUCE, c, 0.0);
    CK(h, f32_ln_grad_chain(h->du32, x, S(L.mean1), S(L.rstd1), M, hh, gr->ln1_g, gr->ln1_b, c));
  }
  return leave(h, st, flags, 3);
}

// ------------------------------------------------------------------------------ init / destroy
static merak_status validate(const merak_tmp_config *c) {
  if (!c) return fail(nullptr, MERAK_EINVAL, "config is NULL");
  if (c->hidden <= 0 || c->heads <= 0 || c->seq_len <= 0 || c->microbatch <= 0 || c->tmp_degree <= 0 ||
      c->n_sub <= 0 || c->ffn_hidden < 0)
    return fail(nullptr, MERAK_EINVAL, "non-positive size in config");
  if (c->tmp_rank < 0 || c->tmp_rank >= c->tmp_degree) return fail(nullptr, MERAK_EINVAL, "tmp_rank out of range");
  if (c->precision != MERAK_BF16 && c->precision != MERAK_FP32_CHECK)
    return fail(nullptr, MERAK_EINVAL, "bad precision");
  if (c->comm != MERAK_COMM_PEER && c->comm != MERAK_COMM_NCCL && c->comm != MERAK_COMM_LOCAL &&
      c->comm != MERAK_COMM_INPROC && c->comm != MERAK_COMM_NVLS)
    return fail(nullptr, MERAK_EINVAL, "bad comm");
  if (c->comm == MERAK_COMM_NVLS && c->precision == MERAK_FP32_CHECK)
    return fail(nullptr, MERAK_EUNSUPPORTED, "MERAK_COMM_NVLS needs bf16 (the switch reduces bf16 partials)");
  const int T = c->tmp_degree, f = c->ffn_hidden ? c->ffn_hidden : 4 * c->hidden;
  if (c->hidden % c->heads) return fail(nullptr, MERAK_EINDIVISIBLE, "hidden %% heads != 0");
  if (c->heads < T) return fail(nullptr, MERAK_EINDIVISIBLE, "heads < tmp_degree");
  if (f % T) return fail(nullptr, MERAK_EINDIVISIBLE, "ffn %% tmp_degree != 0");
  if (c->microbatch % c->n_sub) return fail(nullptr, MERAK_EINDIVISIBLE, "microbatch %% n_sub != 0");
  if (c->n_sub > MAXN) return fail(nullptr, MERAK_EUNSUPPORTED, "n_sub > %d", MAXN);
  const int d = c->hidden / c->heads;
  if (d != 32 && d != 64 && d != 80 && d != 96 && d != 128)
    return fail(nullptr, MERAK_EUNSUPPORTED, "head dim %d not in {32,64,80,96,128}", d);
  if (T != 1 && T != 2 && T != 4 && T != 8) return fail(nullptr, MERAK_EUNSUPPORTED, "tmp_degree not in {1,2,4,8}");
  if (c->seq_len % 16) return fail(nullptr, MERAK_EUNSUPPORTED, "seq_len must be a multiple of 16");
  if (c->microbatch > 48) return fail(nullptr, MERAK_EUNSUPPORTED, "microbatch > 48");
  if (c->hidden % 8 || (f / T) % 8) return fail(nullptr, MERAK_EUNSUPPORTED, "h and f/T must be multiples of 8");
  if (c->hidden > 8192) return fail(nullptr, MERAK_EUNSUPPORTED, "hidden > 8192 (row-engine register budget)");
  if (c->seq_parallel && T > 1) {
    if (c->comm != MERAK_COMM_PEER && c->comm != MERAK_COMM_INPROC)
      return fail(nullptr, MERAK_EUNSUPPORTED, "seq_parallel needs comm PEER or INPROC");
    if (c->precision != MERAK_BF16) return fail(nullptr, MERAK_EUNSUPPORTED, "seq_parallel needs bf16");
    if (((long)c->microbatch * c->seq_len / c->n_sub) % (8 * T))
      return fail(nullptr, MERAK_EINDIVISIBLE, "seq_parallel: tokens per sub-batch %% (8 T) != 0");
  }
  return MERAK_OK;
}

static void release(merak_tmp_t *h) {
  if (!h) return;
  cudaSetDevice(h->dev);
  for (cudaStream_t c : {h->cs, h->cs1, h->cw, h->cr, h->ms})
    if (c) cudaStreamSynchronize(c);
  for (int q = 0; q < MAX_T; ++q)
    if (!h->inproc && h->peer_pv[q] && h->peer_pv[q] != h->pv) cudaIpcCloseMemHandle(h->peer_pv[q]);
  if (h->nccl) g_nccl.CommDestroy(h->nccl);
  if (h->use_nvls) nvls_release(&h->nvls);
  if (h->pv) cudaFree(h->pv);
  if (h->push_maps) cudaFree(h->push_maps);
  if (h->ws) cudaFree(h->ws);
  if (h->ws32) cudaFree(h->ws32);
  if (h->err_host) cudaFreeHost(h->err_host);
  for (auto e : h->evpool) cudaEventDestroy(e);
  for (cudaEvent_t e : {h->ev_entry, h->ev_cs_end, h->ev_cs1_end, h->ev_cw_end, h->ev_cr_end, h->ev_w1, h->ev_wo,
                        h->ev_wqkv, h->ev_red, h->ev_hs[0], h->ev_hs[1]})
    if (e) cudaEventDestroy(e);
  if (InprocGroup *g = h->grp) {
    g->hs[h->r] = nullptr;
    g->pending[h->r] = nullptr;
    if (--g->alive == 0) {
      for (int r = 0; r < MAX_T; ++r) free(g->stack[r]);
      delete g;
    }
  }
  for (int i = 0; i < 5; ++i)
    for (int k = 0; k < 64; ++k)
      if (h->tr_ev[i][k]) cudaEventDestroy(h->tr_ev[i][k]);
  for (int j = 0; j < MAXN; ++j) {
    if (h->ev_p[j]) cudaEventDestroy(h->ev_p[j]);
    if (h->ev_dz[j]) cudaEventDestroy(h->ev_dz[j]);
    if (h->ev_dq[j]) cudaEventDestroy(h->ev_dq[j]);
    for (int k = 0; k < NSLOT; ++k)
      if (h->ev_ar[k][j]) cudaEventDestroy(h->ev_ar[k][j]);
  }
  if (h->cs1 && h->cs1 != h->cs) cudaStreamDestroy(h->cs1);
  if (h->cw && h->cw != h->cs) cudaStreamDestroy(h->cw);
  if (h->cr && h->cr != h->cs) cudaStreamDestroy(h->cr);
  if (h->ms && h->ms != h->cs) cudaStreamDestroy(h->ms);
  if (h->cs) cudaStreamDestroy(h->cs);
  delete h;
}

static merak_status sync_all(merak_tmp_t *h) {
  for (cudaStream_t c : {h->cs, h->cs1, h->cw, h->cr, h->ms}) CK(h, cudaStreamSynchronize(c));
  return MERAK_OK;
}

// In-process group: keep rank h->r's call until every rank has made its matching call, then issue all of
// them as coroutines of this thread (InprocGroup).  The call that completes the set returns the first
// failure of the set (named by rank); the earlier callers got MERAK_OK.
static merak_status group_run(InprocGroup *g, merak_tmp_t *h);
static merak_status group_issue(merak_tmp_t *h, std::function<merak_status()> fn) {
  InprocGroup *g = h->grp;
  if (g->running) return fail(h, MERAK_ESTATE, "layer call re-entered during an in-process group issue");
  if (g->alive != g->T) return fail(h, MERAK_ESTATE, "a rank of this in-process group was destroyed");
  if (g->pending[h->r])
    return fail(h, MERAK_ESTATE, "rank %d made a second layer call before every rank of its in-process group "
                "made the first", h->r);
  g->pending[h->r] = std::move(fn);
  if (++g->npending < g->T) return MERAK_OK;
  return group_run(g, h);
}

// Run every rank's pending call of the group as coroutines of this thread; the first failure is reported
// on h (named by rank).
static merak_status group_run(InprocGroup *g, merak_tmp_t *h) {
  for (int r = 0; r < g->T; ++r) {
    if (!g->stack[r]) g->stack[r] = (char *)malloc(kCoStack);
    if (!g->stack[r]) return fail(h, MERAK_ENOMEM, "coroutine stack");
    getcontext(&g->ctx[r]);
    g->ctx[r].uc_stack.ss_sp = g->stack[r];
    g->ctx[r].uc_stack.ss_size = kCoStack;
    g->ctx[r].uc_link = &g->main_ctx;
    makecontext(&g->ctx[r], co_entry, 0);
    g->done[r] = false;
    g->status[r] = MERAK_OK;
    g->rec_gen[r] = 0;
  }
  g->running = true;
  g->live = g->T;
  g->arrive = 0;
  InprocGroup *outer = g_co_group;
  g_co_group = g;
  for (int left = g->T; left > 0;)
    for (int r = 0; r < g->T; ++r) {
      if (g->done[r]) continue;
      g->cur = r;
      swapcontext(&g->main_ctx, &g->ctx[r]);  // runs rank r until its next handshake point or its end
      if (g->done[r]) --left;
    }
  g_co_group = outer;
  g->running = false;
  g->npending = 0;
  merak_status st = MERAK_OK;
  for (int r = 0; r < g->T; ++r) {
    g->pending[r] = nullptr;
    if (g->status[r] != MERAK_OK && st == MERAK_OK) {
      st = g->status[r];
      if (g->hs[r] != h) fail(h, st, "rank %d: %s", r, g->hs[r]->err.c_str());
    }
  }
  return st;
}

// Per-rank (non-collective) calls cannot issue a chained forward's deferred AR#2s (their handshakes are
// collective): they need merak_tmp_join first.
static merak_status chain_closed_ar2(merak_tmp_t *h) {
  if (h->ar2_pending)
    return fail(h, MERAK_ESTATE, "a MERAK_FLAG_CHAIN forward's all-reduce is still open: call merak_tmp_join first");
  return MERAK_OK;
}

// Calls that act on a handle's streams at once must not overtake its deferred layer call.
static merak_status group_idle(merak_tmp_t *h) {
  if (h->grp && h->grp->pending[h->r])
    return fail(h, MERAK_ESTATE, "rank %d has a layer call waiting for the other ranks of its in-process group",
                h->r);
  return MERAK_OK;
}

extern "C" {

// Everything a handle owns that does not involve its peers: streams, events, slots, workspace.
static merak_status create_local(const merak_tmp_config *cfg, merak_tmp_t **out) {
  merak_tmp_t *h = new merak_tmp();
  h->cfg = *cfg;
  h->h = cfg->hidden; h->H = cfg->heads; h->s = cfg->seq_len; h->B = cfg->microbatch;
  h->T = cfg->tmp_degree; h->r = cfg->tmp_rank; h->n = cfg->n_sub;
  h->f = cfg->ffn_hidden ? cfg->ffn_hidden : 4 * cfg->hidden;
  h->d = h->h / h->H;
  h->Hr = h->H / h->T + (h->r < h->H % h->T ? 1 : 0);  // reading R8
  h->e0 = 0;
  for (int q = 0; q < h->r; ++q) h->e0 += h->H / h->T + (q < h->H % h->T ? 1 : 0);
  h->hr = h->Hr * h->d;
  h->fr = h->f / h->T;
  h->M = h->B * h->s;
  h->eps = cfg->ln_eps > 0 ? cfg->ln_eps : 1e-5f;
  h->dev = cfg->device;
  h->G = ar_bwd_group_rows(h->h);
  if (const char *t = getenv("MERAK_AR_TIMEOUT_MS")) h->timeout_ns = (uint64_t)atoll(t) * 1000000ull;
  h->f32 = cfg->precision == MERAK_FP32_CHECK;
  h->local = cfg->comm == MERAK_COMM_LOCAL;
  h->inproc = cfg->comm == MERAK_COMM_INPROC;
  h->two_shot = h->T >= 4 && !h->f32;
  if (const char *t = getenv("MERAK_AR_PDL")) h->pdl = atoi(t) == 1;
  h->gemm_smem_kb = h->T > 1 ? 160 : 192;
  if (const char *t = getenv("MERAK_GEMM_SMEM_KB")) h->gemm_smem_kb = atoi(t) == 160 ? 160 : 192;
  if (const char *t = getenv("MERAK_DEBUG_TRACE")) h->trace = atoi(t) == 1;
  if (const char *t = getenv("MERAK_AR_TWO_SHOT")) h->two_shot = h->T > 1 && !h->f32 && atoi(t) == 1;
  if (const char *t = getenv("MERAK_AR_FUSED_WAIT")) h->fused_wait = atoi(t) != 0;
  if (const char *t = getenv("MERAK_FUSE_LN1")) h->fuse_ln1 = atoi(t) != 0;
  // default (T >= 4, two-shot): mode 2, measured +2.2 % at N = T = 4 gpt20b in an interleaved A/B and the
  // all-reduce alone 251 -> 116 us (profiles/r02/push/); T = 2 keeps the one-shot pull (exposed ~0 already)
  h->push_req = h->push_ag = h->T >= 4 && !h->f32;
  if (const char *t = getenv("MERAK_AR_PUSH")) {
    h->push_req = atoi(t) != 0;
    h->push_ag = atoi(t) == 2;
  }
  if (const char *t = getenv("MERAK_AR_PUSH_MINK")) h->push_min_k = atoi(t);
  if (h->f32) h->fuse_ln1 = false;
  // in-process groups share ONE GPU: a waiting epilogue kernel of one rank can fill the SMs that another rank's
  // phase-1 kernel (the one it waits for) needs, so they keep the 1-warp handshake kernel
  if (h->inproc) h->fused_wait = false;
  if (h->inproc) h->pdl = false;  // no handshake kernel to pair with (group_barrier)
  auto bail = [&](merak_status st) {
    g_init_err = h->err;
    release(h);
    return st;
  };
#define CKI(call)                                                                                          \
  do {                                                                                                     \
    cudaError_t _e = (call);                                                                               \
    if (_e != cudaSuccess) {                                                                               \
      fail(h, _e == cudaErrorMemoryAllocation ? MERAK_ENOMEM : MERAK_ECUDA, "%s: %s", #call, cudaGetErrorString(_e)); \
      return bail(_e == cudaErrorMemoryAllocation ? MERAK_ENOMEM : MERAK_ECUDA);                          \
    }                                                                                                      \
  } while (0)
  CKI(cudaSetDevice(h->dev));
  int prio_lo = 0, prio_hi = 0;
  CKI(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  // priorities: comm > sub-batch compute > wgrad filler (greatest priority = numerically lowest)
  const int prio_mid = prio_hi < prio_lo ? prio_hi + 1 : prio_lo;
  CKI(cudaStreamCreateWithPriority(&h->cs, cudaStreamNonBlocking, prio_mid));
  const char *ns = getenv("MERAK_STREAMS");
  // MERAK_STREAMS=1 (measurement): every kernel of the handle on ONE stream, in issue order -- the serialised
  // schedule whose per-launch event spans are kernel durations (bench.py's roofline pass, ncu launch lists)
  const bool one_stream = ns && atoi(ns) == 1;
  if (one_stream)
    h->ms = h->cs;
  else
    CKI(cudaStreamCreateWithPriority(&h->ms, cudaStreamNonBlocking, prio_hi));  // comm first when both ready
  // In-process groups put T ranks' streams in one context.  Streams beyond CUDA_DEVICE_MAX_CONNECTIONS (<= 32)
  // share hardware queues, and a rank's compute queued behind another rank's spinning handshake deadlocks
  // until the watchdog fires; at T = 8 each rank therefore runs everything but the all-reduces on one stream.
  if (one_stream || (h->inproc && h->T >= 8)) {
    h->cs1 = h->cw = h->cs;
  } else {
    CKI(cudaStreamCreateWithPriority(&h->cs1, cudaStreamNonBlocking, prio_mid));
    CKI(cudaStreamCreateWithPriority(&h->cw, cudaStreamNonBlocking, prio_lo));
  }
  if (one_stream || (h->inproc && h->T >= 8))
    h->cr = h->cs;
  else
    CKI(cudaStreamCreateWithPriority(&h->cr, cudaStreamNonBlocking, prio_mid));
  for (cudaEvent_t *e : {&h->ev_entry, &h->ev_cs_end, &h->ev_cs1_end, &h->ev_cw_end, &h->ev_cr_end, &h->ev_w1,
                         &h->ev_wo, &h->ev_wqkv, &h->ev_red})
    CKI(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  if (h->trace)
    for (int i = 0; i < 5; ++i)
      for (int k = 0; k < 64; ++k) CKI(cudaEventCreateWithFlags(&h->tr_ev[i][k], cudaEventDisableTiming));
  for (int j = 0; j < MAXN; ++j) {
    CKI(cudaEventCreateWithFlags(&h->ev_p[j], cudaEventDisableTiming));
    CKI(cudaEventCreateWithFlags(&h->ev_dz[j], cudaEventDisableTiming));
    CKI(cudaEventCreateWithFlags(&h->ev_dq[j], cudaEventDisableTiming));
    for (int k = 0; k < NSLOT; ++k) CKI(cudaEventCreateWithFlags(&h->ev_ar[k][j], cudaEventDisableTiming));
  }
  // peer-visible slots + flags
  h->slot_bytes = align256((size_t)h->M * h->h * (h->f32 ? 4 : 2));
  // MERAK_COMM_NVLS (T > 1): the slots live in multicast-bound memory set up by merak_tmp_init; the IPC-shared
  // block holds the handshake flags only
  const bool nvls = cfg->comm == MERAK_COMM_NVLS && h->T > 1;
  h->sp = cfg->seq_parallel && h->T > 1;
  // the all-gather slot exists in the sp layout and for the all-gather push of the two-shot all-reduce
  const int nslot_pv = (h->sp || (h->push_ag && h->T > 1)) ? NSLOT : NSLOT - 1;
  h->flags_off = nvls ? 0 : nslot_pv * h->slot_bytes;
  h->pv_bytes = h->flags_off + align256(2 * MAX_AR_CTAS * MAX_T * sizeof(uint32_t));
  if (h->sp) {  // LN-gradient partial exchange: [MAXN sub-batches][dγ2, dβ2, dγ1, dβ1][h] fp32
    h->lnx_off = h->pv_bytes;
    h->pv_bytes += align256((size_t)MAXN * 4 * h->h * sizeof(float));
  }
  CKI(cudaMalloc(&h->pv, h->pv_bytes));
  CKI(cudaMemset(h->pv + h->flags_off, 0, h->pv_bytes - h->flags_off));
  CKI(cudaHostAlloc(&h->err_host, 8 * sizeof(int), cudaHostAllocMapped));
  memset(h->err_host, 0, 8 * sizeof(int));
  CKI(cudaHostGetDevicePointer((void **)&h->err_dev, h->err_host, 0));
  // workspace
  {
    const size_t M = h->M;
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t at = o; o += align256(bytes); return at; };
    const size_t o_dz = take(M * h->fr * 2), o_dx1 = take(M * h->h * 2), o_dctx = take(M * h->hr * 2);
    const size_t o_dqkv = take(M * 3 * h->hr * 2), o_delta = take(attn_bwd_ws_floats(h->B, h->s, h->Hr, h->d) * 4);
    const int ncol = std::max(std::max(3 * h->hr, h->fr), h->h);
    const size_t o_pc = take(2 * (size_t)h->B * ncol * 4);
    const size_t o_pg = take((M / h->G) * (size_t)h->h * 4), o_pb = take((M / h->G) * (size_t)h->h * 4);
    const size_t o_pg1 = take((M / h->G) * (size_t)h->h * 4), o_pb1 = take((M / h->G) * (size_t)h->h * 4);
    const size_t o_ctr = take(64);
    const size_t o_dyf = h->sp ? take(M * h->h * 2) : 0;
    CKI(cudaMalloc(&h->ws, o));
    if (h->sp) h->dyf = (bf16 *)(h->ws + o_dyf);
    CKI(cudaMemset(h->ws + o_ctr, 0, 64));
    CKI(cudaMemset(h->ws + o_delta, 0, attn_bwd_ws_floats(h->B, h->s, h->Hr, h->d) * 4));  // dQ counters start at 0
    // dynamic GEMM tile schedule: opt-in (measured no gain over the static schedule at gpt1.5b, T=1)
    const char *dyn = getenv("MERAK_GEMM_DYN");
    if (dyn && atoi(dyn) == 1) h->tile_ctr = (int *)(h->ws + o_ctr);
    h->dz = (bf16 *)(h->ws + o_dz); h->dx1 = (bf16 *)(h->ws + o_dx1); h->dctx = (bf16 *)(h->ws + o_dctx);
    h->dqkv = (bf16 *)(h->ws + o_dqkv); h->delta = (float *)(h->ws + o_delta);
    h->dq_acc = h->delta + (size_t)h->B * h->Hr * h->s;
    h->dq_sem = (int *)(h->dq_acc + (size_t)h->B * h->Hr * h->s * h->d);
    h->part_col = (float *)(h->ws + o_pc); h->part_lng = (float *)(h->ws + o_pg); h->part_lnb = (float *)(h->ws + o_pb);
    h->part_lng1 = (float *)(h->ws + o_pg1); h->part_lnb1 = (float *)(h->ws + o_pb1);
  }
  if (h->f32) {
    const size_t M = h->M;
    size_t o = 0;
    auto take = [&](size_t elems) { size_t at = o; o += align256(elems * 4); return at; };
    const size_t a = take(M * h->fr), b = take(M * h->h), c = take(M * h->hr), d = take(M * 3 * h->hr);
    const size_t e = take((size_t)h->B * h->Hr * h->s), f = take(M * h->h);
    CKI(cudaMalloc(&h->ws32, o));
    h->dz32 = (float *)(h->ws32 + a); h->dx1_32 = (float *)(h->ws32 + b); h->dctx32 = (float *)(h->ws32 + c);
    h->dqkv32 = (float *)(h->ws32 + d); h->delta32 = (float *)(h->ws32 + e); h->du32 = (float *)(h->ws32 + f);
  }
  // load every kernel this handle can launch now, not at a first launch inside a layer call (kernels.h)
  CKI(h->f32 ? f32_preload() : gemm_preload());
  if (!h->f32) CKI(attn_preload(h->d));
  CKI(ln_ar_preload());
  CKI(nvls_preload());
  CKI(cudaDeviceSynchronize());
  for (int q = 0; q < MAX_T; ++q) h->peer_pv[q] = nullptr;
  h->peer_pv[h->r] = h->pv;
#undef CKI
  *out = h;
  return MERAK_OK;
}

// Peer store maps of the fused GEMM -> reduce-scatter push (h->push): for each row-parallel slot s and owner q, the
// TMA store map of q's slot s as a bf16 [M, h] tensor; built once the peers' slots are mapped (PEER / INPROC).
static merak_status setup_push(merak_tmp_t *h) {
  if (!h->push_req || h->T == 1 || h->local || h->f32 || h->nccl || h->use_nvls) {
    h->push_ag = false;
    return MERAK_OK;
  }
  std::vector<uint8_t> maps((size_t)4 * h->T * 128);
  for (int sl = 0; sl < 4; ++sl)
    for (int q = 0; q < h->T; ++q)
      CK(h, gemm_store_map(maps.data() + ((size_t)sl * h->T + q) * 128, slot_ptr(h, q, sl), h->M, h->h, h->h));
  CK(h, cudaSetDevice(h->dev));
  CK(h, cudaMalloc(&h->push_maps, maps.size()));
  CK(h, cudaMemcpy(h->push_maps, maps.data(), maps.size(), cudaMemcpyHostToDevice));
  h->push = true;
  return MERAK_OK;
}

merak_status merak_tmp_init(const merak_tmp_config *cfg, merak_allgather_fn ag, void *ag_ctx, merak_tmp_t **out) {
  if (!out) return fail(nullptr, MERAK_EINVAL, "out is NULL");
  *out = nullptr;
  TRY(validate(cfg));
  if (cfg->comm == MERAK_COMM_INPROC)
    return fail(nullptr, MERAK_EINVAL, "MERAK_COMM_INPROC handles are created by merak_tmp_init_group");
  if (cfg->tmp_degree > 1 && !ag && cfg->comm != MERAK_COMM_LOCAL)
    return fail(nullptr, MERAK_EINVAL, "tmp_degree > 1 needs an allgather callback");
  merak_tmp_t *h = nullptr;
  TRY(create_local(cfg, &h));
  auto bail = [&](merak_status st) {
    g_init_err = h->err;
    release(h);
    return st;
  };
#define CKI(call)                                                                                          \
  do {                                                                                                     \
    cudaError_t _e = (call);                                                                               \
    if (_e != cudaSuccess) {                                                                               \
      fail(h, _e == cudaErrorMemoryAllocation ? MERAK_ENOMEM : MERAK_ECUDA, "%s: %s", #call, cudaGetErrorString(_e)); \
      return bail(_e == cudaErrorMemoryAllocation ? MERAK_ENOMEM : MERAK_ECUDA);                          \
    }                                                                                                      \
  } while (0)
  if (h->T > 1 && !h->local) {
    cudaIpcMemHandle_t mine;
    CKI(cudaIpcGetMemHandle(&mine, h->pv));
    std::vector<cudaIpcMemHandle_t> all(h->T);
    if (ag(ag_ctx, &mine, all.data(), sizeof(mine)) != 0) {
      fail(h, MERAK_EPEER, "allgather of IPC handles failed");
      return bail(MERAK_EPEER);
    }
    for (int q = 0; q < h->T; ++q) {
      if (q == h->r) continue;
      void *p = nullptr;
      cudaError_t e = cudaIpcOpenMemHandle(&p, all[q], cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) {
        fail(h, MERAK_EPEER, "cudaIpcOpenMemHandle(rank %d): %s", q, cudaGetErrorString(e));
        return bail(MERAK_EPEER);
      }
      h->peer_pv[q] = (char *)p;
    }
    // second exchange: every rank has mapped every peer and zeroed its flags before any kernel runs
    int dummy = h->r, gathered[MAX_T];
    if (ag(ag_ctx, &dummy, gathered, sizeof(int)) != 0) {
      fail(h, MERAK_EPEER, "allgather barrier failed");
      return bail(MERAK_EPEER);
    }
  }
  if (cfg->comm == MERAK_COMM_NVLS && h->T > 1) {
    std::string why;
    const int rc = nvls_setup(&h->nvls, h->dev, h->T, h->r, (size_t)(NSLOT - 1) * h->slot_bytes, ag, ag_ctx, &why);
    if (rc != 0) {
      fail(h, rc == -2 ? MERAK_EUNSUPPORTED : MERAK_EPEER, "NVLS multicast setup: %s", why.c_str());
      return bail(rc == -2 ? MERAK_EUNSUPPORTED : MERAK_EPEER);
    }
    h->use_nvls = true;
    h->two_shot = true;  // phase 1 in the switch, phase 2 = the gathered epilogue reading the own slot
  }
  if (cfg->comm == MERAK_COMM_NCCL && h->T > 1) {
    if (!g_nccl.load()) {
      fail(h, MERAK_EUNSUPPORTED, "libnccl.so.2 not found (set MERAK_NCCL_LIB)");
      return bail(MERAK_EUNSUPPORTED);
    }
    ncclUniqueId id;
    memset(&id, 0, sizeof(id));
    if (h->r == 0 && g_nccl.GetUniqueId(&id) != ncclSuccess) {
      fail(h, MERAK_EPEER, "ncclGetUniqueId failed");
      return bail(MERAK_EPEER);
    }
    std::vector<ncclUniqueId> ids(h->T);
    if (ag(ag_ctx, &id, ids.data(), sizeof(id)) != 0) {
      fail(h, MERAK_EPEER, "allgather of the NCCL unique id failed");
      return bail(MERAK_EPEER);
    }
    ncclResult_t nr = g_nccl.CommInitRank(&h->nccl, h->T, ids[0], h->r);
    if (nr != ncclSuccess) {
      fail(h, MERAK_EPEER, "ncclCommInitRank: %s", g_nccl.GetErrorString(nr));
      return bail(MERAK_EPEER);
    }
  }
  {
    const merak_status ps = setup_push(h);
    if (ps != MERAK_OK) return bail(ps);
  }
#undef CKI
  *out = h;
  return MERAK_OK;
}

merak_status merak_tmp_init_group(const merak_tmp_config *cfg, merak_tmp_t **out) {
  if (!out) return fail(nullptr, MERAK_EINVAL, "out is NULL");
  TRY(validate(cfg));
  if (cfg->comm != MERAK_COMM_PEER && cfg->comm != MERAK_COMM_INPROC)
    return fail(nullptr, MERAK_EUNSUPPORTED, "init_group: comm must be MERAK_COMM_PEER or MERAK_COMM_INPROC");
  const int T = cfg->tmp_degree;
  for (int q = 0; q < T; ++q) out[q] = nullptr;
  for (int q = 0; q < T; ++q) {
    merak_tmp_config c = *cfg;
    c.tmp_rank = q;
    c.comm = MERAK_COMM_INPROC;
    merak_status st = create_local(&c, &out[q]);
    if (st != MERAK_OK) {
      const std::string e = g_init_err;
      for (int p = 0; p < q; ++p) {
        release(out[p]);
        out[p] = nullptr;
      }
      g_init_err = e;
      return st;
    }
  }
  // every rank maps every peer's peer-visible buffer directly: same process, same device, same context
  for (int q = 0; q < T; ++q)
    for (int p = 0; p < T; ++p) out[q]->peer_pv[p] = out[p]->pv;
  for (int q = 0; q < T; ++q) {
    const merak_status st = setup_push(out[q]);
    if (st != MERAK_OK) {
      const std::string e = out[q]->err;
      for (int p = 0; p < T; ++p) {
        release(out[p]);
        out[p] = nullptr;
      }
      g_init_err = e;
      return st;
    }
  }
  InprocGroup *g = new InprocGroup();
  g->T = g->alive = T;
  for (int q = 0; q < T; ++q) {
    g->hs[q] = out[q];
    out[q]->grp = g;
  }
  for (int q = 0; q < T; ++q)
    for (int k = 0; k < 2; ++k)
      if (cudaEventCreateWithFlags(&out[q]->ev_hs[k], cudaEventDisableTiming) != cudaSuccess) {
        for (int p = 0; p < T; ++p) {
          release(out[p]);
          out[p] = nullptr;
        }
        return fail(nullptr, MERAK_ECUDA, "init_group: cudaEventCreate");
      }
  return MERAK_OK;
}

merak_status merak_tmp_set_subbatches(merak_tmp_t *h, int32_t n_sub) {
  if (!h) return fail(nullptr, MERAK_EINVAL, "handle is NULL");
  if (h->chain_open) return fail(h, MERAK_ESTATE, "set_subbatches while a MERAK_FLAG_CHAIN sequence is open");
  if (n_sub <= 0 || n_sub > MAXN) return fail(h, MERAK_EINVAL, "n_sub out of range");
  TRY(group_idle(h));
  if (h->sp && ((long)h->M / n_sub) % (8 * h->T))
    return fail(h, MERAK_EINDIVISIBLE, "seq_parallel: tokens per sub-batch %% (8 T) != 0");
  if (h->B % n_sub) return fail(h, MERAK_EINDIVISIBLE, "microbatch %% n_sub != 0");
  // all outstanding work of the old split must finish before slot/event indices are reinterpreted
  TRY(sync_all(h));
  memset(h->ev_ar_valid, 0, sizeof(h->ev_ar_valid));
  h->n = n_sub;
  h->cfg.n_sub = n_sub;
  return MERAK_OK;
}

size_t merak_tmp_saved_bytes(const merak_tmp_t *h) {
  if (!h) return 0;
  return h->f32 ? saved_f32(h).total : saved_layout(h).total;
}

static bool aligned16(const void *p) { return ((uintptr_t)p & 15) == 0; }


merak_status merak_tmp_layer_fwd(merak_tmp_t *h, const merak_tmp_weights *w, const void *x, void *y, void *saved,
                                 uint32_t flags, void *st) {
  if (!h) return fail(nullptr, MERAK_EINVAL, "handle is NULL");
  const bool rc = (flags & MERAK_FLAG_RECOMPUTE) != 0;  // regenerate `saved` only: y is not written
  if (rc && h->f32) return fail(h, MERAK_EUNSUPPORTED, "MERAK_FLAG_RECOMPUTE is not available in the fp32 check mode");
  if (!w || !x || (!y && !rc) || !saved) return fail(h, MERAK_EINVAL, "NULL argument");
  const void *ps[] = {w->ln1_g, w->ln1_b, w->w_qkv, w->b_qkv, w->w_o, w->b_o, w->ln2_g, w->ln2_b, w->w_1, w->b_1, w->w_2, w->b_2, x, rc ? x : y, saved};
  for (const void *p : ps)
    if (!p || !aligned16(p)) return fail(h, MERAK_EINVAL, "NULL or non-16B-aligned pointer");
  if (h->broken) return fail(h, MERAK_ESTATE, "handle unusable after an earlier failure: %s", h->err.c_str());
  if (h->sp && (flags & (MERAK_FLAG_RECOMPUTE | MERAK_FLAG_NO_COMM)))
    return fail(h, MERAK_EUNSUPPORTED, "seq_parallel: MERAK_FLAG_RECOMPUTE / MERAK_FLAG_NO_COMM are not available");
  const merak_tmp_weights wv = *w;  // by value: an in-process group may issue the call later
  auto body = [h, wv, x, y, saved, flags, st, rc]() -> merak_status {
    const uint32_t e0 = h->epoch;
    const merak_status s =
        h->f32  ? layer_fwd_f32(h, &wv, (const float *)x, (float *)y, (char *)saved, flags, (cudaStream_t)st)
        : h->sp ? layer_fwd_sp(h, &wv, (const bf16 *)x, (bf16 *)y, (char *)saved, flags, (cudaStream_t)st)
                : layer_fwd(h, &wv, (const bf16 *)x, (bf16 *)y, (char *)saved, flags, (cudaStream_t)st, rc);
    if (s != MERAK_OK && (h->epoch != e0 || s == MERAK_ETIMEOUT)) h->broken = true;
    return s;
  };
  return h->grp ? group_issue(h, body) : body();
}

merak_status merak_tmp_layer_bwd(merak_tmp_t *h, const merak_tmp_weights *w, const void *x, const void *saved,
                                 const void *dy, void *dx, const merak_tmp_grads *g, uint32_t flags, void *st) {
  if (!h) return fail(nullptr, MERAK_EINVAL, "handle is NULL");
  if (!w || !x || !saved || !dy || !dx || !g) return fail(h, MERAK_EINVAL, "NULL argument");
  const void *ps[] = {w->ln1_g, w->ln1_b, w->w_qkv, w->b_qkv, w->w_o, w->b_o, w->ln2_g, w->ln2_b, w->w_1, w->b_1,
                      w->w_2, w->b_2, x, saved, dy, dx, g->ln1_g, g->ln1_b, g->w_qkv, g->b_qkv, g->w_o, g->b_o,
                      g->ln2_g, g->ln2_b, g->w_1, g->b_1, g->w_2, g->b_2};
  for (const void *p : ps)
    if (!p || !aligned16(p)) return fail(h, MERAK_EINVAL, "NULL or non-16B-aligned pointer");
  if (h->broken) return fail(h, MERAK_ESTATE, "handle unusable after an earlier failure: %s", h->err.c_str());
  if (h->sp && (flags & (MERAK_FLAG_RECOMPUTE | MERAK_FLAG_NO_COMM)))
    return fail(h, MERAK_EUNSUPPORTED, "seq_parallel: MERAK_FLAG_RECOMPUTE / MERAK_FLAG_NO_COMM are not available");
  if ((flags & MERAK_FLAG_RECOMPUTE) && h->f32)
    return fail(h, MERAK_EUNSUPPORTED, "MERAK_FLAG_RECOMPUTE is not available in the fp32 check mode");
  const merak_tmp_weights wv = *w;  // by value: an in-process group may issue the call later
  const merak_tmp_grads gv = *g;
  auto body = [h, wv, gv, x, saved, dy, dx, flags, st]() -> merak_status {
    const merak_tmp_weights *w = &wv;
    const merak_tmp_grads *g = &gv;
    const uint32_t e0 = h->epoch;
    if (flags & MERAK_FLAG_RECOMPUTE) {  // regenerate `saved` (scratch) from x, then the backward proper
      const merak_status r = layer_fwd(h, w, (const bf16 *)x, nullptr, (char *)const_cast<void *>(saved),
                                       MERAK_FLAG_CHAIN | (flags & MERAK_FLAG_NO_COMM), (cudaStream_t)st, true);
      // (the backward below continues the open chain: its sub-batch streams follow each fc1 directly)
      if (r != MERAK_OK) {
        if (h->epoch != e0 || r == MERAK_ETIMEOUT) h->broken = true;
        return r;
      }
    }
    const merak_status s =
        h->f32  ? layer_bwd_f32(h, w, (const float *)x, (const char *)saved, (const float *)dy, (float *)dx, g, flags,
                                (cudaStream_t)st)
        : h->sp ? layer_bwd_sp(h, w, (const bf16 *)x, (const char *)saved, (const bf16 *)dy, (bf16 *)dx, g, flags,
                               (cudaStream_t)st)
                : layer_bwd(h, w, (const bf16 *)x, (const char *)saved, (const bf16 *)dy, (bf16 *)dx, g, flags,
                            (cudaStream_t)st);
    if (s != MERAK_OK && (h->epoch != e0 || s == MERAK_ETIMEOUT)) h->broken = true;
    return s;
  };
  return h->grp ? group_issue(h, body) : body();
}

merak_status merak_tmp_join(merak_tmp_t *h, void *st) {
  if (!h) return fail(nullptr, MERAK_EINVAL, "handle is NULL");
  auto body = [h, st]() -> merak_status {
    TRY(flush_ar2(h));  // a chained forward's deferred AR#2s (collective: every rank joins)
    if (!h->have_prev) return MERAK_OK;
    TRY(wait_all(h, (cudaStream_t)st));
    for (int j = 0; j < h->n; ++j) CK(h, cudaStreamWaitEvent((cudaStream_t)st, h->prev_out[j], 0));
    h->chain_open = false;
    return check_async_error(h);  // a watchdog that already fired (the word is host-mapped; no sync here)
  };
  // in-process group with deferred AR#2s: their handshakes need every rank, so the join is a group call
  return (h->grp && h->ar2_pending) ? group_issue(h, body) : body();
}

merak_status merak_tmp_destroy(merak_tmp_t *h) {
  if (h && h->ar2_pending) {  // an open chain's last AR#2s: y is an output the caller may still read
    cudaSetDevice(h->dev);
    InprocGroup *g = h->grp;
    if (g && !g->running && g->alive == g->T) {  // every rank at once, while every rank's slots exist
      bool any = false;
      for (int q = 0; q < g->T; ++q) {
        merak_tmp_t *hq = g->hs[q];
        g->pending[q] = [hq]() { return flush_ar2(hq); };
        any = any || hq->ar2_pending;
      }
      g->npending = g->T;
      if (any) {
        group_run(g, h);
      } else {
        for (int q = 0; q < g->T; ++q) g->pending[q] = nullptr;
        g->npending = 0;
      }
    } else if (!g) {
      flush_ar2(h);  // PEER / NCCL: each rank flushes in its own destroy, before the final barrier
    }
  }
  if (h && h->inproc) {
    // every rank of the group has enqueued its collective calls (they never block the host), so the
    // shared device drains: no rank frees its slots while a peer's all-reduce may still read them
    cudaSetDevice(h->dev);
    cudaDeviceSynchronize();
  } else if (h && h->T > 1 && !h->nccl && !h->local && h->ms) {
    // final barrier: no rank frees its slots while a peer's last all-reduce may still read them
    cudaSetDevice(h->dev);
    PeerSync ps = make_sync(h, true);
    peer_ready(ps, h->ms);
    cudaStreamSynchronize(h->ms);
  }
  if (!h) return MERAK_OK;
  for (cudaStream_t c : {h->cs, h->cs1, h->cw, h->cr, h->ms})
    if (c) cudaStreamSynchronize(c);
  // the watchdog word after every stream drained: a handshake that timed out in the last calls
  // (after which those calls' outputs are garbage) is reported here rather than lost
  const merak_status st = check_async_error(h);
  if (st != MERAK_OK) g_init_err = h->err;
  release(h);
  return st;
}

const char *merak_tmp_last_error(const merak_tmp_t *h) { return h ? h->err.c_str() : g_init_err.c_str(); }

merak_status merak_tmp_set_profiling(merak_tmp_t *h, int32_t on) {
  if (!h) return fail(nullptr, MERAK_EINVAL, "handle is NULL");
  TRY(group_idle(h));
  TRY(chain_closed_ar2(h));
  TRY(sync_all(h));
  h->prof = on != 0;
  h->recs.clear();
  h->evnext = 0;
  for (int k = 0; k < MERAK_K_NUM; ++k) {
    h->prof_ms[k] = 0;
    h->prof_flops[k] = 0;
    h->prof_launch[k] = 0;
  }
  return MERAK_OK;
}

merak_status merak_tmp_get_profile(merak_tmp_t *h, double *ms, int64_t *launches, double *flops) {
  if (!h) return fail(nullptr, MERAK_EINVAL, "handle is NULL");
  TRY(group_idle(h));
  TRY(chain_closed_ar2(h));
  TRY(sync_all(h));
  for (auto &r : h->recs) {
    float t = 0;
    CK(h, cudaEventElapsedTime(&t, r.a, r.b));
    h->prof_ms[r.cls] += t;
    h->prof_flops[r.cls] += r.flops;
  }
  h->recs.clear();
  h->evnext = 0;
  for (int k = 0; k < MERAK_K_NUM; ++k) {
    if (ms) ms[k] = h->prof_ms[k];
    if (launches) launches[k] = h->prof_launch[k];
    if (flops) flops[k] = h->prof_flops[k];
  }
  return MERAK_OK;
}

merak_status merak_tmp_get_timeline(merak_tmp_t *h, int32_t cap, int32_t *count, int32_t *cls, int32_t *stream,
                                    float *t0, float *t1) {
  if (!h || !count) return fail(h, MERAK_EINVAL, "NULL argument");
  TRY(group_idle(h));
  TRY(chain_closed_ar2(h));
  TRY(sync_all(h));
  int32_t n = 0;
  if (!h->recs.empty()) {
    cudaEvent_t origin = h->recs.front().a;
    for (auto &r : h->recs) {
      if (n >= cap) break;
      float a = 0, b = 0;
      CK(h, cudaEventElapsedTime(&a, origin, r.a));
      CK(h, cudaEventElapsedTime(&b, origin, r.b));
      if (cls) cls[n] = r.cls;
      if (stream) stream[n] = r.sid;
      if (t0) t0[n] = a;
      if (t1) t1[n] = b;
      ++n;
    }
  }
  *count = n;
  return MERAK_OK;
}

int64_t merak_tmp_launch_count(const merak_tmp_t *h) { return h ? h->launches : 0; }

merak_status merak_tmp_debug_host(const merak_tmp_t *h, int32_t *out) {
  if (!h || !out) return MERAK_EINVAL;
  for (int i = 0; i < 5; ++i) out[i] = h->err_host ? ((volatile int *)h->err_host)[i] : 0;
  out[5] = (int32_t)h->epoch;
  out[6] = (int32_t)h->launches;
  for (int i = 0; i < 5; ++i) out[7 + i] = (int32_t)h->tr_n[i];
  out[12] = h->push ? 1 : 0;
  out[13] = h->two_shot ? 1 : 0;
  return MERAK_OK;
}

merak_status merak_tmp_debug_state(const merak_tmp_t *h, int32_t *out) {
  if (!h || !out) return MERAK_EINVAL;
  cudaStream_t ss[5] = {h->cs, h->cs1, h->cw, h->cr, h->ms};
  for (int i = 0; i < 5; ++i) out[i] = (ss[i] && cudaStreamQuery(ss[i]) == cudaErrorNotReady) ? 1 : 0;
  for (int i = 0; i < 5; ++i) out[5 + i] = h->err_host ? ((volatile int *)h->err_host)[i] : 0;
  out[10] = (int32_t)h->epoch;
  for (int i = 0; i < 5; ++i) {  // first unfinished traced launch per stream (MERAK_DEBUG_TRACE=1), else -1
    out[11 + i] = -1;
    out[16 + i] = -1;
    if (!h->trace) continue;
    const int64_t n = h->tr_n[i], lo = n > 64 ? n - 64 : 0;
    for (int64_t q = lo; q < n; ++q) {
      const int k = (int)(q % 64);
      if (cudaEventQuery(h->tr_ev[i][k]) == cudaErrorNotReady) {
        out[11 + i] = h->tr_cls[i][k];
        out[16 + i] = (int32_t)h->tr_seq[i][k];
        break;
      }
    }
  }
  return MERAK_OK;
}

merak_status merak_tmp_bench_allreduce(merak_tmp_t *h, int32_t which, int32_t rows, int32_t iters, float *ms) {
  if (!h || !ms) return fail(h, MERAK_EINVAL, "NULL argument");
  if (h->T < 2 || h->nccl || h->f32 || h->local || h->inproc)
    return fail(h, MERAK_EUNSUPPORTED, "needs T > 1, peer comm across processes, bf16");
  TRY(chain_closed_ar2(h));
  if (rows <= 0 || rows > h->M || iters <= 0 || which < 0 || which > 2 || rows % h->G)
    return fail(h, MERAK_EINVAL, "bad rows / iters / which");
  TRY(sync_all(h));
  CK(h, cudaSetDevice(h->dev));
  const size_t hh = h->h, nb = (size_t)rows * hh * 2;
  char *tmp = nullptr;
  CK(h, cudaMalloc(&tmp, 3 * nb + 4 * hh * 4 + 1024));
  bf16 *resid = (bf16 *)tmp, *out = (bf16 *)(tmp + nb), *gam = (bf16 *)(tmp + 2 * nb);
  float *mean = nullptr, *rstd = nullptr;  // LN stats of the backward epilogue (rows entries each)
  merak_status st = MERAK_OK;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  float *stats = nullptr;
  do {
    if (cudaMalloc(&stats, 2 * (size_t)rows * 4) != cudaSuccess) { st = fail(h, MERAK_ENOMEM, "stats"); break; }
    mean = stats; rstd = stats + rows;
    {
      // no rank zeroes its slot while a peer's earlier all-reduce may still be reading it
      PeerSync ps0 = make_sync(h, true);
      if ((st = sync_peers(h, ps0)) != MERAK_OK) break;
    }
    if (cudaMemsetAsync(tmp, 0, 3 * nb + 4 * hh * 4, h->ms) != cudaSuccess ||
        cudaMemsetAsync(stats, 0, 2 * (size_t)rows * 4, h->ms) != cudaSuccess ||
        cudaMemsetAsync(slot_ptr(h, h->r, 1), 0, nb, h->ms) != cudaSuccess) {
      st = fail(h, MERAK_ECUDA, "memset");
      break;
    }
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto one = [&]() -> merak_status {
      PeerSync ps = make_sync(h, true);
      TRY(sync_peers(h, ps));
      if (which == 2) return MERAK_OK;  // handshake kernel only
      if (which == 0) {
        ArFwdArgs a;
        memset(&a, 0, sizeof(a));
        a.T = ar_partials(h, true, 1, 0, a.partial, rows);
        a.m = rows; a.h = (int)hh; a.resid = resid; a.bias = gam; a.out = out; a.ctas = h->cfg.comm_ctas;
        if (two_shot_on(h, true)) TRY(two_shot_rs(h, 1, 0, rows, resid, gam, &a.chunk, &ps, push_on(h, true, rows, 1)));
        Launch Lk(h, MERAK_K_ALLREDUCE, h->ms, 0.0);
        a.pdl = h->pdl && !h->prof && ps.enabled;  // after the handshake kernel
      CK(h, ar_fwd(a, ps, h->ms));
      } else {
        ArBwdArgs a;
        memset(&a, 0, sizeof(a));
        a.T = ar_partials(h, true, 1, 0, a.partial, rows);
        a.m = rows; a.h = (int)hh; a.x_ln = resid; a.mean = mean; a.rstd = rstd; a.gamma = gam; a.dres = resid;
        a.dx = out; a.part_dg = h->part_lng; a.part_db = h->part_lnb; a.G = h->G; a.ctas = h->cfg.comm_ctas;
        if (two_shot_on(h, true)) TRY(two_shot_rs(h, 1, 0, rows, nullptr, nullptr, &a.chunk, &ps, push_on(h, true, rows, 1)));
        Launch Lk(h, MERAK_K_ALLREDUCE, h->ms, 0.0);
        a.pdl = h->pdl && !h->prof && ps.enabled;
        CK(h, ar_bwd(a, ps, h->ms));
      }
      return MERAK_OK;
    };
    for (int i = 0; i < 3 && st == MERAK_OK; ++i) st = one();  // warm-up
    if (st != MERAK_OK) break;
    cudaEventRecord(e0, h->ms);
    for (int i = 0; i < iters && st == MERAK_OK; ++i) st = one();
    if (st != MERAK_OK) break;
    cudaEventRecord(e1, h->ms);
    if (cudaEventSynchronize(e1) != cudaSuccess) { st = fail(h, MERAK_ECUDA, "event sync"); break; }
    float t = 0;
    cudaEventElapsedTime(&t, e0, e1);
    *ms = t / iters;
    st = check_async_error(h);
  } while (0);
  cudaStreamSynchronize(h->ms);
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (stats) cudaFree(stats);
  cudaFree(tmp);
  memset(h->ev_ar_valid, 0, sizeof(h->ev_ar_valid));
  return st;
}

// ------------------------------------------------------------------------------ testing entry points
int merak_test_gemm(const void *A, const void *B, int M, int N, int K, int lda, int ldb, int a_mn, int b_mn, int epi,
                    void *out, int ldo, void *out2, int ldo2, const void *bias, const void *aux, int ld_aux,
                    float *out32, int ld32, float *db32, int max_ctas, void *stream) {
  GemmArgs a = gargs(A, B, M, N, K, lda, ldb, a_mn != 0, b_mn != 0, epi);
  a.out = out; a.ldo = ldo; a.out2 = out2; a.ldo2 = ldo2; a.bias = bias; a.aux = aux; a.ld_aux = ld_aux;
  a.out32 = out32; a.ld32 = ld32; a.db32 = db32; a.max_ctas = max_ctas;
  return (int)gemm(a, (cudaStream_t)stream);
}

int merak_test_attn_fwd(const void *qkv, void *ctx, float *lse, int b, int s, int heads, int d, void *stream) {
  AttnArgs a;
  memset(&a, 0, sizeof(a));
  a.qkv = qkv; a.ctx = ctx; a.lse = lse; a.b = b; a.s = s; a.heads = heads; a.d = d; a.ld_ctx = heads * d;
  return (int)attn_fwd(a, (cudaStream_t)stream);
}

int merak_test_attn_bwd_dbg(const void *qkv, const void *ctx, const float *lse, const void *dctx, void *dqkv, void *ws,
                            int b, int s, int heads, int d, unsigned long long *dbg, void *stream) {
  AttnArgs a;
  memset(&a, 0, sizeof(a));
  a.qkv = qkv; a.ctx = (void *)ctx; a.lse = (float *)lse; a.dctx = dctx; a.dqkv = dqkv;
  a.delta = (float *)ws;
  a.dq_acc = a.delta + (size_t)b * heads * s;
  a.dq_sem = (int *)(a.dq_acc + (size_t)b * heads * s * d);
  a.b = b; a.s = s; a.heads = heads; a.d = d; a.ld_ctx = heads * d; a.dbg = dbg;
  return (int)attn_bwd(a, (cudaStream_t)stream);
}

size_t merak_test_attn_bwd_ws_bytes(int b, int s, int heads, int d) { return attn_bwd_ws_floats(b, s, heads, d) * 4; }

int merak_test_attn_bwd(const void *qkv, const void *ctx, const float *lse, const void *dctx, void *dqkv, void *ws,
                        int b, int s, int heads, int d, void *stream) {
  AttnArgs a;
  memset(&a, 0, sizeof(a));
  a.qkv = qkv; a.ctx = (void *)ctx; a.lse = (float *)lse; a.dctx = dctx; a.dqkv = dqkv;
  a.delta = (float *)ws;
  a.dq_acc = a.delta + (size_t)b * heads * s;
  a.dq_sem = (int *)(a.dq_acc + (size_t)b * heads * s * d);
  a.b = b; a.s = s; a.heads = heads; a.d = d; a.ld_ctx = heads * d;
  return (int)attn_bwd(a, (cudaStream_t)stream);
}

int merak_test_ln_fwd(const void *x, const void *gamma, const void *beta, void *u, float *mean, float *rstd, int m,
                      int h, float eps, void *stream) {
  OnesPad pad;
  memset(&pad, 0, sizeof(pad));
  return (int)ln_fwd((const bf16 *)x, (const bf16 *)gamma, (const bf16 *)beta, (bf16 *)u, h, mean, rstd, m, h, eps, pad,
                     (cudaStream_t)stream);
}

int merak_test_ar_fwd(const void *const *partials, int T, int m, int h, const void *resid, const void *bias, void *out,
                      int do_ln, const void *gamma, const void *beta, void *ln_out, float *mean, float *rstd, float eps,
                      int ctas, void *stream) {
  if (T < 1 || T > MAX_T) return (int)cudaErrorInvalidValue;
  ArFwdArgs a;
  memset(&a, 0, sizeof(a));
  for (int q = 0; q < T; ++q) a.partial[q] = (const bf16 *)partials[q];
  a.T = T; a.m = m; a.h = h; a.resid = (const bf16 *)resid; a.bias = (const bf16 *)bias; a.out = (bf16 *)out;
  a.do_ln = do_ln != 0; a.gamma = (const bf16 *)gamma; a.beta = (const bf16 *)beta; a.ln_out = (bf16 *)ln_out;
  a.ld_ln = h;
  a.mean = mean; a.rstd = rstd; a.eps = eps; a.ctas = ctas;
  PeerSync ps;
  memset(&ps, 0, sizeof(ps));
  ps.enabled = false;
  return (int)ar_fwd(a, ps, (cudaStream_t)stream);
}

int merak_test_ar_bwd(const void *const *partials, int T, int m, int s, int h, const void *x_ln, const float *mean,
                      const float *rstd, const void *gamma, const void *dres, void *dx, float *dgamma, float *dbeta,
                      float *ws, int ctas, void *stream) {
  if (T < 1 || T > MAX_T) return (int)cudaErrorInvalidValue;
  ArBwdArgs a;
  memset(&a, 0, sizeof(a));
  for (int q = 0; q < T; ++q) a.partial[q] = (const bf16 *)partials[q];
  a.T = T; a.m = m; a.h = h; a.x_ln = (const bf16 *)x_ln; a.mean = mean; a.rstd = rstd; a.gamma = (const bf16 *)gamma;
  a.dres = (const bf16 *)dres; a.dx = (bf16 *)dx; a.G = ar_bwd_group_rows(h);
  if (m % s || s % a.G) return (int)cudaErrorInvalidValue;
  a.part_dg = ws; a.part_db = ws + (size_t)(m / a.G) * h; a.ctas = ctas;
  PeerSync ps;
  memset(&ps, 0, sizeof(ps));
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = ar_bwd(a, ps, st);
  float *q = ws + 2 * (size_t)(m / a.G) * h;
  if (e == cudaSuccess)
    e = sample_reduce2(a.part_dg, a.part_db, s / a.G, m / s, h, q, q + (size_t)(m / s) * h, dgamma, dbeta, st);
  return (int)e;
}

int merak_test_colsum(const void *X, int ld, int m, int s, int n, float *g, float *ws, void *stream) {
  if (m % s) return (int)cudaErrorInvalidValue;
  cudaError_t e = colsum_sample((const bf16 *)X, ld, s, m / s, n, ws, (cudaStream_t)stream);
  if (e == cudaSuccess) e = sample_reduce2(ws, nullptr, 1, m / s, n, ws + (size_t)(m / s) * n, nullptr, g, nullptr,
                                           (cudaStream_t)stream);
  return (int)e;
}

}  // extern "C"
