/*
 * merak_tmp_testing.h -- kernel-level entry points of libmerak_tmp.so used by the unit parity
 * tests (tests/test_gpu_kernels.py).  Not part of the user-facing API (merak_tmp.h); every
 * function launches exactly the kernel the layer uses, on the caller's stream, and returns a
 * cudaError_t value (0 = success).  All pointers are device pointers, bf16 unless noted.
 */
#ifndef MERAK_TMP_TESTING_H
#define MERAK_TMP_TESTING_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* C[M,N] = A * B^T via the tcgen05 GEMM.  a_mn: A stored [K, M] (else [M, K]); b_mn: B stored
 * [K, N] (else [N, K]).  epi: 0 store bf16, 1 +bias, 2 +bias & GeLU (out=z, out2=gelu(z)),
 * 3 * gelu'(aux), 4 fp32 accumulate into out32 (preloaded); with db32 != NULL the last of the N columns
 * (the ones column of B) accumulates into db32[M] instead (bias gradient). */
int merak_test_gemm(const void *A, const void *B, int M, int N, int K, int lda, int ldb, int a_mn, int b_mn, int epi,
                    void *out, int ldo, void *out2, int ldo2, const void *bias, const void *aux, int ld_aux,
                    float *out32, int ld32, float *db32, int max_ctas, void *stream);

/* Causal attention forward over packed qkv [b*s, 3*heads*d] -> ctx [b*s, heads*d], lse [b,heads,s] fp32. */
int merak_test_attn_fwd(const void *qkv, void *ctx, float *lse, int b, int s, int heads, int d, void *stream);
/* Backward -> dqkv [b*s, 3*heads*d]; ws: device workspace of merak_test_attn_bwd_ws_bytes() bytes, ZEROED
 * before its first use (it holds the dQ ordering counters, which every call leaves zero). */
size_t merak_test_attn_bwd_ws_bytes(int b, int s, int heads, int d);
int merak_test_attn_bwd(const void *qkv, const void *ctx, const float *lse, const void *dctx, void *dqkv, void *ws,
                        int b, int s, int heads, int d, void *stream);

/* LayerNorm forward: u = LN(x) (bf16), mean/rstd fp32 [m]. */
int merak_test_ln_fwd(const void *x, const void *gamma, const void *beta, void *u, float *mean, float *rstd, int m,
                      int h, float eps, void *stream);

/* Forward all-reduce epilogue over T partials on ONE device (fake peers, no handshake):
 * out = sum_r partial[r] (rank order) + bias + resid; if do_ln: ln_out = LN(bf16(out)). */
int merak_test_ar_fwd(const void *const *partials, int T, int m, int h, const void *resid, const void *bias, void *out,
                      int do_ln, const void *gamma, const void *beta, void *ln_out, float *mean, float *rstd, float eps,
                      int ctas, void *stream);

/* Backward all-reduce epilogue (fake peers): dx = dres + LN^T(sum_r partial[r]); dgamma/dbeta
 * (fp32 [h]) += per-sample fixed-order token sums (s = rows per sample, m % s == 0, s % 16 == 0).
 * ws: fp32 workspace of 2*(m/8)*h + 2*(m/s)*h floats. */
int merak_test_ar_bwd(const void *const *partials, int T, int m, int s, int h, const void *x_ln, const float *mean,
                      const float *rstd, const void *gamma, const void *dres, void *dx, float *dgamma, float *dbeta,
                      float *ws, int ctas, void *stream);

/* g[c] += sum_i X[i, c] over m rows = m/s samples of s rows, per-sample fixed order then a chain over
 * samples; ws: fp32 [2 * (m/s) * n]. */
int merak_test_colsum(const void *X, int ld, int m, int s, int n, float *g, float *ws, void *stream);

#ifdef __cplusplus
}
#endif
#endif
