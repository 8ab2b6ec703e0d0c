// kernels.h -- host-side launch interface of the sm_100a kernels (internal, not part of the ABI).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <string>

namespace mk {

// ---------------------------------------------------------------- GEMM (gemm.cu)
// C[M,N] = A[M,K] * B[N,K]^T on tcgen05 (bf16 in, fp32 accumulate in TMEM).
// Operand storage:
//   a_mn = false: A stored [M rows, K cols] (K contiguous), row stride lda elements
//   a_mn = true : A stored [K rows, M cols] (M contiguous), row stride lda   (A = stored^T)
//   b_mn = false: B stored [N rows, K cols] (K contiguous), row stride ldb
//   b_mn = true : B stored [K rows, N cols] (N contiguous), row stride ldb   (B = stored^T)
// Reduction order per output element is fixed: K walked in 64-wide blocks in increasing order,
// 16-wide MMA steps inside; it never depends on M (bit-identity across sub-batch counts).
constexpr int MAX_T = 8;  // max TMP degree

// Function attributes (max dynamic smem) and occupancy are per device: host-side caches of them are
// indexed by the current device ordinal, so handles on several devices in one process stay correct.
constexpr int MAX_DEV = 64;
inline int cur_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d >= 0 && d < MAX_DEV ? d : MAX_DEV - 1;
}

// Module preloading.  With CUDA's lazy loading a kernel's first launch loads it, and a load may need a
// context-wide synchronisation; if another stream of this context is then running a handshake kernel that
// waits for a peer whose work this host thread has not enqueued yet (an in-process group), the two block
// each other.  Every handle therefore loads each kernel it can launch at init (cudaFuncGetAttributes forces
// the load), so no layer call ever loads a module.
inline cudaError_t touch_kernel(const void *f) {
  cudaFuncAttributes at;
  return cudaFuncGetAttributes(&at, f);
}
cudaError_t gemm_preload();
cudaError_t attn_preload(int d);
cudaError_t attn_bwd_preload_d(int d);
cudaError_t ln_ar_preload();
cudaError_t f32_preload();

enum Epi : int {
  EPI_STORE_BF16 = 0,  // out = bf16(acc)
  EPI_BIAS_BF16 = 1,   // out = bf16(acc + bias[n])
  EPI_BIAS_GELU = 2,   // z = acc + bias[n]; out = bf16(z); out2 = bf16(gelu(z))
  EPI_GELU_BWD = 3,    // out = bf16(acc * gelu'(aux[m,n]))   (aux = saved z, bf16)
  EPI_ACC_F32 = 4      // out32[m,n] (fp32) is loaded into TMEM first; out32 = acc after the K loop
};

struct GemmArgs {
  const void *A;
  const void *B;
  int M, N, K;
  int lda, ldb;
  bool a_mn, b_mn;
  int epi;
  void *out;         // bf16 [M, ldo]
  int ldo;
  void *out2;        // bf16 [M, ldo2] (EPI_BIAS_GELU)
  int ldo2;
  const void *bias;  // bf16 [N]
  const void *aux;   // bf16 [M, ld_aux] (EPI_GELU_BWD)
  int ld_aux;
  float *out32;      // fp32 [M, ld32] (EPI_ACC_F32)
  int ld32;
  float *db32;       // EPI_ACC_F32 with a ones column: N includes it as the last column, whose
                     // accumulator goes to db32[M] (bias gradient = A^T 1) instead of out32
  int max_ctas;      // persistent grid cap (0 = all SMs)
  int smem_kb;       // smem budget of the TMA ring: 192 (default) or 160 (leave room for co-resident
                     // all-reduce kernels when T > 1)
  int *tile_ctr;     // dynamic tile scheduler: a device int that is 0 between launches and used by one
                     // stream at a time (the kernel resets it); nullptr = static schedule
  // Scatter store (fused GEMM -> reduce-scatter push, EPI_STORE_BF16 only): instead of out, row i of C is
  // stored through the TMA map scatter[q], q = i / scatter_rows (the owner rank of the row), at map row
  // scatter_row0 + i - q * scatter_rows.  scatter points to T maps in device memory (gemm_store_map);
  // scatter_rows % 32 == 0 and M % scatter_rows == 0, else cudaErrorInvalidValue.
  const void *scatter;
  int scatter_row0, scatter_rows;
};
cudaError_t gemm(const GemmArgs &a, cudaStream_t st);
// Encode (host) the 128-byte TMA store map of a bf16 [rows, cols] tensor (row stride ld) that the GEMM's
// scatter store uses: boxes of 64 cols x 32 rows, 128-B swizzle (the same encoding as its own output map).
cudaError_t gemm_store_map(void *map, const void *ptr, int rows, int cols, int ld);
int gemm_num_sms();

// ---------------------------------------------------------------- attention (attention_tc.cu, attention_bwd_tc.cu)
// Causal flash attention over packed qkv [tokens, 3*hr] (q | k | v column blocks, head e at
// columns e*d..e*d+d-1 of each block), b samples of s tokens, H_r local heads of dim d.
// tcgen05/TMEM/TMA kernels only (no alternate backend).
struct AttnArgs {
  const void *qkv;   // bf16 [b*s, 3*hr]
  void *ctx;         // bf16 [b*s, hr]          (fwd out / bwd in as O)
  float *lse;        // [b, H_r, s] base-2 log-sum-exp of scaled scores (fwd out / bwd in)
  const void *dctx;  // bf16 [b*s, hr]          (bwd in)
  void *dqkv;        // bf16 [b*s, 3*hr]        (bwd out)
  float *delta;      // [b, H_r, s] rowsum(dO*O) workspace (bwd)
  float *dq_acc;     // [b, H_r, s, d] fp32 dQ accumulator workspace (bwd; no initialisation needed)
  int *dq_sem;       // [b, H_r, ceil(s/64)] dQ ordering counters (bwd; zero before the first launch,
                     // left zero by every launch)
  int b, s, heads, d;
  int ld_ctx;        // row stride of ctx (elements; >= heads*d)
  int attn_group;    // bwd: (sample, head) pairs per dispatch group (0 = default)
  unsigned long long *dbg;  // bwd diagnostics only (nullptr): per-CTA clock stamps, 80 per CTA
};
// workspace of attn_bwd in floats: delta, dq_acc, dq_sem (in that order)
size_t attn_bwd_ws_floats(int b, int s, int heads, int d);
cudaError_t attn_fwd(const AttnArgs &a, cudaStream_t st);  // attention_tc.cu
cudaError_t attn_bwd(const AttnArgs &a, cudaStream_t st);  // attention_bwd_tc.cu: delta kernel, then the key-tile kernel

// ---------------------------------------------------------------- fp32 check mode (check_f32.cu)
struct F32GemmArgs {  // C[M,N] (epi) sum_k A(m,k) B(n,k); A(m,k) = a_mn ? A[k*lda+m] : A[m*lda+k], same for B
  const float *A, *B;
  int M, N, K, lda, ldb;
  bool a_mn, b_mn;
  int epi;  // EPI_STORE_BF16 (plain store), EPI_BIAS_BF16, EPI_BIAS_GELU (C = z, C2 = gelu z), EPI_GELU_BWD, EPI_ACC_F32
  float *C;
  int ldc;
  float *C2;
  int ldc2;
  const float *bias, *aux;
  int ld_aux;
};
cudaError_t f32_gemm(const F32GemmArgs &a, cudaStream_t st);
cudaError_t f32_ln_fwd(const float *x, const float *g, const float *b, float *u, float *mean, float *rstd, int m,
                       int h, float eps, cudaStream_t st);
struct F32AttnArgs {
  const float *qkv;  // [b*s, 3hr]
  float *ctx;        // [b*s, hr]
  float *lse;        // [b, H, s] natural-log LSE of the scaled scores
  const float *dctx;
  float *dqkv;
  float *delta;
  int b, s, heads, d;
};
cudaError_t f32_attn_fwd(const F32AttnArgs &a, cudaStream_t st);
cudaError_t f32_attn_bwd(const F32AttnArgs &a, cudaStream_t st);
struct F32ArArgs {
  const float *partial[MAX_T];
  int T, m, h;
  const float *resid, *bias;  // forward: out = sum partials + bias + resid
  float *out;                 // forward: x1 / y; backward: dx
  float *ln_out;              // forward AR#1: LN2(x1) (nullptr otherwise)
  const float *gamma, *beta;
  float *mean, *rstd;         // forward: written; backward: read (saved LN stats)
  float eps;
  const float *x_ln, *dres;   // backward: LN input, residual-path gradient
  float *du;                  // backward: the all-reduced gradient (kept for the LN weight grads)
};
cudaError_t f32_ar_fwd(const F32ArArgs &a, cudaStream_t st);
cudaError_t f32_ar_bwd(const F32ArArgs &a, cudaStream_t st);
cudaError_t f32_colsum_chain(const float *X, int ldx, int rows, int cols, float *out, cudaStream_t st);
cudaError_t f32_ln_grad_chain(const float *du, const float *xln, const float *mean, const float *rstd, int rows, int h,
                              float *dg, float *db, cudaStream_t st);

// ---------------------------------------------------------------- LN / all-reduce / reductions (ln_ar.cu)
constexpr int MAX_AR_CTAS = 1024;

// Peer synchronisation for one all-reduce.  flags_local: this rank's flag array; flags_peer[r]:
// rank r's flag array mapped into this process (flags_peer[rank] == flags_local).  Layout per rank:
// ready[MAX_T] (uint32 epochs, written by the peers).
struct PeerSync {
  int T, rank;
  bool enabled;               // false: fake peers on one device / T == 1 (no handshake)
  uint32_t epoch;
  uint32_t *flags_local;
  uint32_t *flags_peer[MAX_T];
  int *err_word;              // device word set to 1 on watchdog timeout
  uint64_t timeout_ns;
  bool pdl;                   // host: launch as a programmatic dependent of the previous kernel
  // two-shot without the second handshake kernel: the phase-1 kernel's last CTA publishes `epoch` to the peers
  // (ctr: a zeroed device counter of this rank), and the phase-2 epilogue kernel waits for the peers' epoch in
  // kernel (thread 0 of every CTA) before it reads their rows
  bool publish, wait;
  uint32_t *ctr;
};

// ones-column pads written per row by the LayerNorm kernels: element col[k] of row r of
// ptr[k] (row stride ld[k]) = 1, the next 7 = 0, for k < n
struct OnesPad {
  __nv_bfloat16 *ptr[4];
  int ld[4], col[4];
  int n;
};
struct ArFwdArgs {
  const __nv_bfloat16 *partial[MAX_T];  // rank-ordered partial sums, rows [0, m) of this sub-batch
  int T;                                // number of partials summed (1 with NO_COMM)
  int m, h;
  const __nv_bfloat16 *resid;           // [m, h]
  const __nv_bfloat16 *bias;            // [h]
  __nv_bfloat16 *out;                   // [m, h]   x1 (AR#1) or y (AR#2)
  // LayerNorm of the stored (bf16) out: AR#1 (u2 = LN2(x1)), or AR#2 of a chained layer fused with the next
  // layer's LN1 (u = LN1'(y), with that layer's ones-column pads)
  bool do_ln;
  OnesPad pad;
  const __nv_bfloat16 *gamma, *beta;
  __nv_bfloat16 *ln_out;
  int ld_ln;                            // row stride of ln_out
  float *mean, *rstd;
  float eps;
  int ctas;
  // two-shot phase 2 ("gathered" mode, chunk > 0): row i was already reduced (sum + bias + resid,
  // rounded once) by rank i / chunk into its slot; partial[q] is rank q's slot, bias/resid unused.
  int chunk;
  bool pdl;  // host: launch as a programmatic dependent of the handshake kernel before it
};
cudaError_t ar_fwd(const ArFwdArgs &a, const PeerSync &ps, cudaStream_t st);

// Two-shot phase 1 (reduce-scatter, T >= 4): rows [row0, row1) of the sub-batch, owned by this
// rank: v = sum_r partial[r] (rank order) [+ bias + resid], rounded once to bf16 and written IN
// PLACE into this rank's own slot (out = partial[rank]).  Peers read those rows in phase 2.
struct ArRsArgs {
  PeerSync ps;  // ps.publish: publish the completion of this phase to the peers (see PeerSync)
  const __nv_bfloat16 *partial[MAX_T];
  int T, h, row0, row1;
  const __nv_bfloat16 *resid;  // nullptr: plain sum (backward); else forward AR epilogue terms
  const __nv_bfloat16 *bias;
  __nv_bfloat16 *out;
  // all-gather push: n_peer > 0 stores every reduced row into out_peer[q] (rank q's all-gather slot, same row
  // offsets as out) for all q, starting with q = rank + 1 (spreads the NVLink writes), instead of into out
  __nv_bfloat16 *out_peer[MAX_T];
  int n_peer, rank;
  int ctas;
  bool pdl;
};
cudaError_t ar_rs(const ArRsArgs &a, cudaStream_t st);
// 1-warp kernel: publish ps.epoch to every peer and wait for theirs (no-op unless ps.enabled)
cudaError_t peer_ready(const PeerSync &ps, cudaStream_t st);

struct ArBwdArgs {
  const __nv_bfloat16 *partial[MAX_T];
  int T;
  int m, h;
  const __nv_bfloat16 *x_ln;    // LN input (x1 for LN2, x for LN1)      [m, h]
  const float *mean, *rstd;     // saved LN stats                         [m]
  const __nv_bfloat16 *gamma;   // [h]
  const __nv_bfloat16 *dres;    // residual-path gradient (dy or dx1)     [m, h]
  __nv_bfloat16 *dx;            // out: dres + LN^T(sum partials)          [m, h]
  float *part_dg, *part_db;     // out: per-group column partials [m/G, h]
  int G;                        // rows per group (8; divides s)
  int ctas;
  int chunk;                    // > 0: two-shot phase 2, row i reads the reduced du from partial[i / chunk]
  bool pdl;
};
cudaError_t ar_bwd(const ArBwdArgs &a, const PeerSync &ps, cudaStream_t st);
int ar_bwd_group_rows(int h);

// LayerNorm forward of x (bf16 [m,h]) -> u (bf16, row stride ld_u), mean/rstd (fp32).
// Optionally writes the 8-wide pad [1, 0, ..., 0] at column pad_col[k] of rows of pad_ptr[k] (row
// stride pad_ld[k]) for k < npad: the "ones column" of saved activations that turns each wgrad
// GEMM into dW | db (bias gradient = dY^T 1).
cudaError_t ln_fwd(const __nv_bfloat16 *x, const __nv_bfloat16 *g, const __nv_bfloat16 *b, __nv_bfloat16 *u,
                   int ld_u, float *mean, float *rstd, int m, int h, float eps, const OnesPad &pad, cudaStream_t st);

// Token reductions with a per-sample fixed structure (bit-identical across sub-batch splits):
// Q[i][c] = fixed-order sum of the s rows of sample i of X (bf16, row stride ld), i < b
cudaError_t colsum_sample(const __nv_bfloat16 *X, int ld, int s, int b, int n, float *Q, cudaStream_t st);
// g_t[c] += sum over samples i (in order) of the fixed-tree sum of p_t[i*gps .. i*gps+gps-1][c],
// for t = 0 and (if p1) t = 1; q0/q1: fp32 workspace [b * n] each.  Two launches.
cudaError_t sample_reduce2(const float *p0, const float *p1, int gps, int b, int n, float *q0, float *q1, float *g0,
                           float *g1, cudaStream_t st);

// ---------------------------------------------------------------- sequence-parallel helpers (ln_ar.cu)
// All-gather of row shards: dst row i (row stride ld_dst) = row i of src[i / rows_per]
// (row stride h; src[q] = rank q's peer-visible buffer), i < m; plus the ones-column pads of `pad` for every
// row (written here because the row shards' producer only saw its own rows).
struct AgArgs {
  const __nv_bfloat16 *src[MAX_T];
  int T, m, h, rows_per;
  __nv_bfloat16 *dst;
  int ld_dst;
  bool pdl;
};
cudaError_t ag_rows(const AgArgs &a, const OnesPad &pad, cudaStream_t st);
// out[c] = fixed-order chain over the g-row-group partials p[k][c], k < ngroups (t = 0 and, if p1, t = 1)
cudaError_t group_chain2(const float *p0, const float *p1, int ngroups, int n, float *out0, float *out1,
                         cudaStream_t st);
// g_t[c] += sum over ranks q = 0..T-1 (in order) of src_t[q][c]  (t = 0, 1)
cudaError_t rank_sum_add2(const float *const *src0, const float *const *src1, int T, int n, float *g0, float *g1,
                          cudaStream_t st);
// plain 16-byte-vector copy of rows (dst row stride ld_dst, src row stride ld_src, h multiple of 8)
cudaError_t copy_rows(const __nv_bfloat16 *src, int ld_src, __nv_bfloat16 *dst, int ld_dst, int m, int h,
                      cudaStream_t st);

// ---------------------------------------------------------------- NVLS in-switch reduction (nvls.cu)
// The all-reduce slots of this rank bound to a CUDA multicast object shared by the T ranks.
struct Nvls {
  void *uc_va, *mc_va;  // this rank's slots: unicast mapping / multicast mapping (same offsets)
  size_t size;
  unsigned long long mem_handle, mc_handle;  // CUmemGenericAllocationHandle
  int dev, fd;
  bool bound;
};
typedef int (*nvls_allgather_fn)(void *ctx, const void *send, void *recv, size_t bytes_per_rank);
bool nvls_supported(int dev);
// collective over the T ranks; 0 = OK, -2 = multicast unsupported on some rank, -1 = other failure (*err)
int nvls_setup(Nvls *n, int dev, int T, int r, size_t bytes, nvls_allgather_fn ag, void *ctx, std::string *err);
void nvls_release(Nvls *n);
struct NvlsRsArgs {
  PeerSync ps;                  // ps.publish: as ArRsArgs
  __nv_bfloat16 *mc;            // multicast address of row 0 of the sub-batch in the slot
  int h, row0, row1;            // rows owned by this rank
  const __nv_bfloat16 *resid;   // nullptr: plain sum (backward); else + bias + resid (forward epilogue terms)
  const __nv_bfloat16 *bias;
  int ctas;
  bool pdl;
};
cudaError_t nvls_rs(const NvlsRsArgs &a, cudaStream_t st);
cudaError_t nvls_preload();

}  // namespace mk
