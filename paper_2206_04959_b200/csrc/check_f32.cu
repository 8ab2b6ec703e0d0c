// check_f32.cu -- kernels of the fp32 check mode (MERAK_FP32_CHECK; SURVEY §8(a) "Numerics": "the
// fp32 check mode is fp32 everywhere"; north_star: <= 1e-5 relative Frobenius error).
//
// Same layer, same sharding, same sub-batch split and the same fixed-order rules as the bf16 path
// (so n_sub > 1 and n_sub = 1 stay bit-identical), but every operand, activation and gradient is
// fp32 and the contractions run on the FP32 FMA pipes.  These kernels are deliberately simple: the
// check mode exists to validate the method's arithmetic tightly, not for speed.
//   - GEMM: 64x64 output tile per 256-thread CTA, K walked in order (per-element chain fixed)
//   - attention: one warp per (sample, head, query row) [forward, dQ] or key row [dK/dV],
//     online softmax in fp32, natural-log LSE
//   - all-reduce epilogues: warp per row, partials summed in rank order (R10) without rounding
//   - token reductions (bias, LayerNorm grads): one thread per column, rows in token order,
//     continuing the running sum across sub-batches -> the same chain for every n_sub
#include <math.h>

#include "kernels.h"
#include "ptx.cuh"

namespace mk {

namespace {

MK_DEV float wsum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

constexpr float GELU_C = 0.7978845608028654f;  // sqrt(2/pi)

MK_DEV float gelu32(float z) { return 0.5f * z * (1.f + tanhf(GELU_C * (z + 0.044715f * z * z * z))); }
MK_DEV float gelu32_grad(float z) {
  const float t = tanhf(GELU_C * (z + 0.044715f * z * z * z));
  return 0.5f * (1.f + t) + 0.5f * z * (1.f - t * t) * GELU_C * (1.f + 3.f * 0.044715f * z * z);
}

}  // namespace

// ------------------------------------------------------------------------------------------ GEMM
__global__ void __launch_bounds__(256) f32_gemm_kernel(F32GemmArgs a) {
  __shared__ float As[16][64 + 1], Bs[16][64 + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < a.K; k0 += 16) {
    for (int e = threadIdx.x; e < 16 * 64; e += 256) {
      const int kk = e / 64, mm = e % 64;
      const int m = m0 + mm, n = n0 + mm, k = k0 + kk;
      float va = 0.f, vb = 0.f;
      if (k < a.K) {
        if (m < a.M) va = a.a_mn ? a.A[(size_t)k * a.lda + m] : a.A[(size_t)m * a.lda + k];
        if (n < a.N) vb = a.b_mn ? a.B[(size_t)k * a.ldb + n] : a.B[(size_t)n * a.ldb + k];
      }
      As[kk][mm] = va;
      Bs[kk][mm] = vb;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float ar[4], br[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        ar[i] = As[kk][ty + 16 * i];
        br[i] = Bs[kk][tx + 16 * i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(ar[i], br[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty + 16 * i;
    if (m >= a.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx + 16 * j;
      if (n >= a.N) continue;
      float v = acc[i][j];
      float *c = a.C + (size_t)m * a.ldc + n;
      switch (a.epi) {
        case EPI_BIAS_BF16: v += a.bias[n]; *c = v; break;
        case EPI_BIAS_GELU:
          v += a.bias[n];
          *c = v;
          a.C2[(size_t)m * a.ldc2 + n] = gelu32(v);
          break;
        case EPI_GELU_BWD: *c = v * gelu32_grad(a.aux[(size_t)m * a.ld_aux + n]); break;
        case EPI_ACC_F32: *c += v; break;
        default: *c = v;
      }
    }
  }
}

cudaError_t f32_gemm(const F32GemmArgs &a, cudaStream_t st) {
  if (a.M <= 0 || a.N <= 0 || a.K <= 0) return cudaErrorInvalidValue;
  dim3 grid((a.N + 63) / 64, (a.M + 63) / 64);
  f32_gemm_kernel<<<grid, 256, 0, st>>>(a);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------ LayerNorm
__global__ void __launch_bounds__(256) f32_ln_kernel(const float *x, const float *g, const float *b, float *u,
                                                     float *mean, float *rstd, int m, int h, float eps) {
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= m) return;
  const float *xr = x + (size_t)row * h;
  float s = 0.f;
  for (int c = lane; c < h; c += 32) s += xr[c];
  const float mu = wsum(s) / h;
  float v = 0.f;
  for (int c = lane; c < h; c += 32) v += (xr[c] - mu) * (xr[c] - mu);
  const float rs = 1.f / sqrtf(wsum(v) / h + eps);
  for (int c = lane; c < h; c += 32) u[(size_t)row * h + c] = (xr[c] - mu) * rs * g[c] + b[c];
  if (lane == 0) {
    mean[row] = mu;
    rstd[row] = rs;
  }
}

cudaError_t f32_ln_fwd(const float *x, const float *g, const float *b, float *u, float *mean, float *rstd, int m,
                       int h, float eps, cudaStream_t st) {
  f32_ln_kernel<<<(m + 7) / 8, 256, 0, st>>>(x, g, b, u, mean, rstd, m, h, eps);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------ attention
// Layout as the bf16 path: qkv [b*s, 3hr] (q | k | v, head e at column e*d of each block),
// ctx / dctx [b*s, hr], lse / delta [b, H, s].  Lane l holds dims l, l+32, ... of a row (d <= 128).
namespace {
constexpr int DMAX = 4;
MK_DEV void load_row(const float *p, int d, float (&r)[DMAX]) {
#pragma unroll
  for (int i = 0; i < DMAX; ++i) {
    const int c = (threadIdx.x & 31) + 32 * i;
    r[i] = c < d ? p[c] : 0.f;
  }
}
MK_DEV float dot_row(const float (&a)[DMAX], const float *p, int d) {
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < DMAX; ++i) {
    const int c = (threadIdx.x & 31) + 32 * i;
    if (c < d) s = fmaf(a[i], p[c], s);
  }
  return wsum(s);
}
}  // namespace

__global__ void __launch_bounds__(256) f32_attn_fwd_kernel(F32AttnArgs a) {
  const int w = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (w >= a.b * a.heads * a.s) return;
  const int i = w % a.s, e = (w / a.s) % a.heads, bi = w / (a.s * a.heads);
  const int hr = a.heads * a.d, ld = 3 * hr;
  const size_t t0 = (size_t)bi * a.s;
  const float scale = 1.f / sqrtf((float)a.d);
  float q[DMAX], o[DMAX] = {};
  load_row(a.qkv + (t0 + i) * ld + e * a.d, a.d, q);
  float mx = -INFINITY, sum = 0.f;
  for (int j = 0; j <= i; ++j) {
    const float sc = dot_row(q, a.qkv + (t0 + j) * ld + hr + e * a.d, a.d) * scale;
    const float mn = fmaxf(mx, sc), corr = expf(mx - mn), p = expf(sc - mn);
    sum = sum * corr + p;
    float v[DMAX];
    load_row(a.qkv + (t0 + j) * ld + 2 * hr + e * a.d, a.d, v);
#pragma unroll
    for (int k = 0; k < DMAX; ++k) o[k] = o[k] * corr + p * v[k];
    mx = mn;
  }
#pragma unroll
  for (int k = 0; k < DMAX; ++k) {
    const int c = (threadIdx.x & 31) + 32 * k;
    if (c < a.d) a.ctx[(t0 + i) * hr + e * a.d + c] = o[k] / sum;
  }
  if ((threadIdx.x & 31) == 0) a.lse[((size_t)bi * a.heads + e) * a.s + i] = mx + logf(sum);
}

// dQ (and delta = rowsum(dO * O)): warp per query row
__global__ void __launch_bounds__(256) f32_attn_dq_kernel(F32AttnArgs a) {
  const int w = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (w >= a.b * a.heads * a.s) return;
  const int i = w % a.s, e = (w / a.s) % a.heads, bi = w / (a.s * a.heads);
  const int hr = a.heads * a.d, ld = 3 * hr;
  const size_t t0 = (size_t)bi * a.s, srow = ((size_t)bi * a.heads + e) * a.s;
  const float scale = 1.f / sqrtf((float)a.d);
  float q[DMAX], dO[DMAX], dq[DMAX] = {};
  load_row(a.qkv + (t0 + i) * ld + e * a.d, a.d, q);
  load_row(a.dctx + (t0 + i) * hr + e * a.d, a.d, dO);
  const float del = dot_row(dO, a.ctx + (t0 + i) * hr + e * a.d, a.d);
  const float lse = a.lse[srow + i];
  for (int j = 0; j <= i; ++j) {
    const float *kr = a.qkv + (t0 + j) * ld + hr + e * a.d;
    const float p = expf(dot_row(q, kr, a.d) * scale - lse);
    const float dp = dot_row(dO, a.qkv + (t0 + j) * ld + 2 * hr + e * a.d, a.d);
    const float ds = p * (dp - del);
    float k[DMAX];
    load_row(kr, a.d, k);
#pragma unroll
    for (int c = 0; c < DMAX; ++c) dq[c] = fmaf(ds, k[c], dq[c]);
  }
#pragma unroll
  for (int c = 0; c < DMAX; ++c) {
    const int cc = (threadIdx.x & 31) + 32 * c;
    if (cc < a.d) a.dqkv[(t0 + i) * ld + e * a.d + cc] = dq[c] * scale;
  }
  if ((threadIdx.x & 31) == 0) a.delta[srow + i] = del;
}

// dK, dV: warp per key row (queries i >= j)
__global__ void __launch_bounds__(256) f32_attn_dkdv_kernel(F32AttnArgs a) {
  const int w = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (w >= a.b * a.heads * a.s) return;
  const int j = w % a.s, e = (w / a.s) % a.heads, bi = w / (a.s * a.heads);
  const int hr = a.heads * a.d, ld = 3 * hr;
  const size_t t0 = (size_t)bi * a.s, srow = ((size_t)bi * a.heads + e) * a.s;
  const float scale = 1.f / sqrtf((float)a.d);
  float k[DMAX], v[DMAX], dk[DMAX] = {}, dv[DMAX] = {};
  load_row(a.qkv + (t0 + j) * ld + hr + e * a.d, a.d, k);
  load_row(a.qkv + (t0 + j) * ld + 2 * hr + e * a.d, a.d, v);
  for (int i = j; i < a.s; ++i) {
    const float *qr = a.qkv + (t0 + i) * ld + e * a.d;
    const float *dor = a.dctx + (t0 + i) * hr + e * a.d;
    const float p = expf(dot_row(k, qr, a.d) * scale - a.lse[srow + i]);
    const float dp = dot_row(v, dor, a.d);
    const float ds = p * (dp - a.delta[srow + i]);
    float q[DMAX], dO[DMAX];
    load_row(qr, a.d, q);
    load_row(dor, a.d, dO);
#pragma unroll
    for (int c = 0; c < DMAX; ++c) {
      dk[c] = fmaf(ds, q[c], dk[c]);
      dv[c] = fmaf(p, dO[c], dv[c]);
    }
  }
#pragma unroll
  for (int c = 0; c < DMAX; ++c) {
    const int cc = (threadIdx.x & 31) + 32 * c;
    if (cc < a.d) {
      a.dqkv[(t0 + j) * ld + hr + e * a.d + cc] = dk[c] * scale;
      a.dqkv[(t0 + j) * ld + 2 * hr + e * a.d + cc] = dv[c];
    }
  }
}

cudaError_t f32_attn_fwd(const F32AttnArgs &a, cudaStream_t st) {
  if (a.d > 32 * DMAX) return cudaErrorNotSupported;
  f32_attn_fwd_kernel<<<(a.b * a.heads * a.s + 7) / 8, 256, 0, st>>>(a);
  return cudaGetLastError();
}
cudaError_t f32_attn_bwd(const F32AttnArgs &a, cudaStream_t st) {
  if (a.d > 32 * DMAX) return cudaErrorNotSupported;
  const int grid = (a.b * a.heads * a.s + 7) / 8;
  f32_attn_dq_kernel<<<grid, 256, 0, st>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  f32_attn_dkdv_kernel<<<grid, 256, 0, st>>>(a);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------ all-reduces
__global__ void __launch_bounds__(256) f32_ar_fwd_kernel(F32ArArgs a) {
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= a.m) return;
  const int h = a.h;
  const size_t ro = (size_t)row * h;
  float s = 0.f;
  for (int c = lane; c < h; c += 32) {
    float v = a.partial[0][ro + c];
    for (int r = 1; r < a.T; ++r) v += a.partial[r][ro + c];  // rank order (R10)
    v += a.bias[c];
    v += a.resid[ro + c];
    a.out[ro + c] = v;
    s += v;
  }
  if (!a.ln_out) return;
  __syncwarp();
  const float mu = wsum(s) / h;
  float var = 0.f;
  for (int c = lane; c < h; c += 32) var += (a.out[ro + c] - mu) * (a.out[ro + c] - mu);
  const float rs = 1.f / sqrtf(wsum(var) / h + a.eps);
  for (int c = lane; c < h; c += 32) a.ln_out[ro + c] = (a.out[ro + c] - mu) * rs * a.gamma[c] + a.beta[c];
  if (lane == 0) {
    a.mean[row] = mu;
    a.rstd[row] = rs;
  }
}

// dx = dres + LN^T(du), du = sum of the partials (also stored for the LayerNorm weight grads)
__global__ void __launch_bounds__(256) f32_ar_bwd_kernel(F32ArArgs a) {
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= a.m) return;
  const int h = a.h;
  const size_t ro = (size_t)row * h;
  const float mu = a.mean[row], rs = a.rstd[row];
  float s1 = 0.f, s2 = 0.f;
  for (int c = lane; c < h; c += 32) {
    float du = a.partial[0][ro + c];
    for (int r = 1; r < a.T; ++r) du += a.partial[r][ro + c];
    a.du[ro + c] = du;
    const float xh = (a.x_ln[ro + c] - mu) * rs, dxh = du * a.gamma[c];
    s1 += dxh;
    s2 += dxh * xh;
  }
  __syncwarp();
  const float m1 = wsum(s1) / h, m2 = wsum(s2) / h;
  for (int c = lane; c < h; c += 32) {
    const float xh = (a.x_ln[ro + c] - mu) * rs, dxh = a.du[ro + c] * a.gamma[c];
    a.out[ro + c] = a.dres[ro + c] + rs * (dxh - m1 - xh * m2);
  }
}

cudaError_t f32_ar_fwd(const F32ArArgs &a, cudaStream_t st) {
  f32_ar_fwd_kernel<<<(a.m + 7) / 8, 256, 0, st>>>(a);
  return cudaGetLastError();
}
cudaError_t f32_ar_bwd(const F32ArArgs &a, cudaStream_t st) {
  f32_ar_bwd_kernel<<<(a.m + 7) / 8, 256, 0, st>>>(a);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------ token chains
// out[c] += X[0][c] + X[1][c] + ... in row order (one running sum per column, continued across calls)
__global__ void f32_colsum_chain_kernel(const float *X, int ldx, int rows, int cols, float *out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  float acc = out[c];
  for (int r = 0; r < rows; ++r) acc += X[(size_t)r * ldx + c];
  out[c] = acc;
}
// dgamma[c] += sum_r du[r][c] * xhat[r][c], dbeta[c] += sum_r du[r][c], rows in order
__global__ void f32_ln_grad_chain_kernel(const float *du, const float *xln, const float *mean, const float *rstd,
                                         int rows, int h, float *dg, float *db) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= h) return;
  float g = dg[c], b = db[c];
  for (int r = 0; r < rows; ++r) {
    const float d = du[(size_t)r * h + c];
    g += d * ((xln[(size_t)r * h + c] - mean[r]) * rstd[r]);
    b += d;
  }
  dg[c] = g;
  db[c] = b;
}

cudaError_t f32_colsum_chain(const float *X, int ldx, int rows, int cols, float *out, cudaStream_t st) {
  f32_colsum_chain_kernel<<<(cols + 127) / 128, 128, 0, st>>>(X, ldx, rows, cols, out);
  return cudaGetLastError();
}
cudaError_t f32_ln_grad_chain(const float *du, const float *xln, const float *mean, const float *rstd, int rows, int h,
                              float *dg, float *db, cudaStream_t st) {
  f32_ln_grad_chain_kernel<<<(h + 127) / 128, 128, 0, st>>>(du, xln, mean, rstd, rows, h, dg, db);
  return cudaGetLastError();
}

cudaError_t f32_preload() {
  const void *ks[] = {(const void *)f32_gemm_kernel, (const void *)f32_ln_kernel, (const void *)f32_attn_fwd_kernel,
                      (const void *)f32_attn_dq_kernel, (const void *)f32_attn_dkdv_kernel,
                      (const void *)f32_ar_fwd_kernel, (const void *)f32_ar_bwd_kernel,
                      (const void *)f32_colsum_chain_kernel, (const void *)f32_ln_grad_chain_kernel};
  for (const void *k : ks) {
    cudaError_t e = touch_kernel(k);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace mk
