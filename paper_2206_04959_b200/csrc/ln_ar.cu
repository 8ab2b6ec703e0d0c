// ln_ar.cu -- LayerNorm, the four TMP all-reduces fused with their replicated epilogues, and the
// fixed-order token reductions for bias / LayerNorm gradients.
//
// All-reduce (P:107 Megatron TMP; P:558 two in FP, two in BP).
// Each rank's row-parallel GEMM writes its bf16 partial [m, h] into its own peer-visible slot
// (CUDA-IPC exported).  The all-reduce kernel on every rank reads the T partials of its rows
// straight from the peers' HBM over NVLink (one-shot), sums them in fp32 in rank order 0..T-1
// (reading R10), and applies the replicated work in the same pass:
//   AR#1: x1 = x + sum_r P1_r + b_o ; u2 = LN2(bf16(x1))          (forward, attention block)
//   AR#2: y  = x1 + sum_r P2_r + b_2                               (forward, FFN block)
//   AR#3: dx1 = dy  + LN2^T(sum_r dU2_r), dgamma2/dbeta2 partials  (backward, FFN block)
//   AR#4: dx  = dx1 + LN1^T(sum_r dU1_r), dgamma1/dbeta1 partials  (backward, attention block)
// Every rank computes every row, so replicated outputs are bit-identical across ranks.
//
// Cross-rank synchronisation is NOT done inside these data kernels (a large grid of CTAs spinning
// on peers can deadlock against persistent GEMM clusters competing for the same SMs).  Instead a
// 1-warp `peer_ready` kernel runs on the communication stream right before each all-reduce: it
// publishes this rank's epoch e (st.release.sys into every peer's flag array) and waits until every
// peer published e (ld.acquire.sys).  A rank publishes e only after (stream order) its GEMM wrote
// partial e AND its all-reduce e-1 finished reading the peers' slots, so `ready(e)` from all peers
// means: every partial of e is complete, and nobody still reads a slot the next GEMMs overwrite.
// A watchdog (globaltimer) bounds the wait; on expiry it sets *err_word (reported by the next API
// call) and later waits fail fast.
#include <math.h>

#include <utility>

#include "kernels.h"
#include "ptx.cuh"

namespace mk {

MK_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

MK_DEV void load8(const __nv_bfloat16 *p, float (&v)[8]) {
  uint4 u = *reinterpret_cast<const uint4 *>(p);
  float2 a = unpack_bf16(u.x), b = unpack_bf16(u.y), c = unpack_bf16(u.z), d = unpack_bf16(u.w);
  v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y; v[4] = c.x; v[5] = c.y; v[6] = d.x; v[7] = d.y;
}
MK_DEV void add8(const __nv_bfloat16 *p, float (&v)[8]) {
  float t[8];
  load8(p, t);
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] += t[i];
}
MK_DEV void store8(__nv_bfloat16 *p, const float (&v)[8]) {
  uint4 u;
  u.x = pack_bf16(v[0], v[1]); u.y = pack_bf16(v[2], v[3]); u.z = pack_bf16(v[4], v[5]); u.w = pack_bf16(v[6], v[7]);
  *reinterpret_cast<uint4 *>(p) = u;
}

// One warp: lane r < T publishes epoch e to peer r, then waits for the peers' epoch e.
// err_word[0] = 1 on timeout; err_word[1..4] = epoch, 0, peer, last flag value seen.  The error word
// lives in host-mapped memory (a PCIe read), so the spin loop reads it only every 256 polls.
__global__ void peer_ready_kernel(PeerSync ps) {
  const int r = threadIdx.x;
  volatile int *err = ps.err_word;
  griddep_wait();    // PDL (second two-shot handshake): the reduce-scatter kernel before it has finished
  griddep_launch();  // let the data kernel after this one launch while this warp spins
  if (*err) return;
  // The partials were written by kernels that completed before this one (stream / event order);
  // peers read them through this GPU's L2, so the release store of the epoch suffices.
  if (r < ps.T && r != ps.rank) st_release_sys(ps.flags_peer[r] + ps.rank, ps.epoch);
  if (r < ps.T && r != ps.rank) {
    const uint64_t t0 = globaltimer();
    uint32_t v;
    for (uint32_t it = 1; (int)((v = ld_acquire_sys(ps.flags_local + r)) - ps.epoch) < 0; ++it) {
      if ((it & 255) == 0 && (*err || globaltimer() - t0 > ps.timeout_ns)) {
        if (atomicExch(ps.err_word, 1) == 0) {
          err[1] = (int)ps.epoch;
          err[2] = 0;
          err[3] = r;
          err[4] = (int)v;
        }
        return;
      }
    }
  }
  __syncwarp();
}

// Launch with an optional programmatic-dependent-launch attribute (hides the launch latency of the
// next kernel of the all-reduce chain behind the previous one; the kernels call griddep_wait first).
template <typename... KArgs, typename... Args>
static cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl,
                            Args &&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

cudaError_t peer_ready(const PeerSync &ps, cudaStream_t st) {
  if (!ps.enabled) return cudaSuccess;
  return launch_k(peer_ready_kernel, dim3(1), dim3(32), 0, st, ps.pdl, ps);
}

// ------------------------------------------------------------------------------ rank-ordered row sums
// A peer load over NVLink costs ~1-2 us; a per-chunk dependent chain would serialise them.  Each lane
// therefore issues the loads of CH of its chunks (chunk c = c0 + 32 i, 8 bf16 each) from all NT
// sources before any arithmetic; the sums keep the fixed rank order 0..NT-1 (reading R10).
MK_DEV void unpack8(const uint4 &u, float (&v)[8]) {
  float2 a = unpack_bf16(u.x), b = unpack_bf16(u.y), c = unpack_bf16(u.z), d = unpack_bf16(u.w);
  v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y; v[4] = c.x; v[5] = c.y; v[6] = d.x; v[7] = d.y;
}
template <int NT, int CH>
MK_DEV void rank_sum(const __nv_bfloat16 *const (&src)[NT], size_t ro, int c0, int nc, float (&v)[CH][8]) {
  uint4 raw[CH][NT];
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    const int c = c0 + 32 * i;
#pragma unroll
    for (int r = 0; r < NT; ++r)
      raw[i][r] = c < nc ? *reinterpret_cast<const uint4 *>(src[r] + ro + (size_t)c * 8) : make_uint4(0, 0, 0, 0);
  }
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    unpack8(raw[i][0], v[i]);
#pragma unroll
    for (int r = 1; r < NT; ++r) {
      float t[8];
      unpack8(raw[i][r], t);
#pragma unroll
      for (int k = 0; k < 8; ++k) v[i][k] += t[k];
    }
  }
}
// sources of one row: the T rank-ordered partials, or (two-shot phase 2, NT = 1) the owner's slot
template <int NT>
MK_DEV void row_sources(const __nv_bfloat16 *const *partial, int chunk, int row, const __nv_bfloat16 *(&src)[NT]) {
#pragma unroll
  for (int r = 0; r < NT; ++r) src[r] = partial[r];
  if (NT == 1 && chunk > 0) src[0] = partial[row / chunk];
}
__host__ __device__ constexpr int ar_ch(int nt) { return nt >= 8 ? 1 : nt >= 4 ? 2 : 4; }

// ------------------------------------------------------------------------------ forward all-reduce
template <int NT>
__global__ void __launch_bounds__(256) ar_fwd_kernel(ArFwdArgs a, PeerSync ps) {
  constexpr int CH = ar_ch(NT);
  griddep_wait();  // PDL: the handshake before this kernel has completed (peers' data is ready)
  griddep_launch();
  extern __shared__ uint4 row_s[];  // do_ln: per warp, the stored bf16 row (LN2 reads it, reading R12)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  const int h = a.h, nc = h >> 3;
  const bool gathered = a.chunk > 0;
  uint4 *rb = row_s + (size_t)warp * nc;
  for (int row = blockIdx.x * nw + warp; row < a.m; row += gridDim.x * nw) {
    const size_t ro = (size_t)row * h;
    float sum = 0.f;
    const __nv_bfloat16 *src[NT];
    row_sources<NT>(a.partial, a.chunk, row, src);
    for (int c0 = lane; c0 < nc; c0 += 32 * CH) {
      float v[CH][8];
      rank_sum<NT, CH>(src, ro, c0, nc, v);
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        const int c = c0 + 32 * i;
        if (c >= nc) continue;
        if (!gathered) {
          add8(a.bias + c * 8, v[i]);
          add8(a.resid + ro + c * 8, v[i]);
        }
        uint4 pk;
        pk.x = pack_bf16(v[i][0], v[i][1]); pk.y = pack_bf16(v[i][2], v[i][3]);
        pk.z = pack_bf16(v[i][4], v[i][5]); pk.w = pack_bf16(v[i][6], v[i][7]);
        *reinterpret_cast<uint4 *>(a.out + ro + c * 8) = pk;
        if (a.do_ln) {
          rb[c] = pk;
          float q[8];
          unpack8(pk, q);
#pragma unroll
          for (int k = 0; k < 8; ++k) sum += q[k];  // LN2 of the stored bf16 x1 (R12)
        }
      }
    }
    if (!a.do_ln) continue;
    __syncwarp();
    const float mean = warp_sum(sum) / h;
    float var = 0.f;
    for (int c = lane; c < nc; c += 32) {
      float q[8];
      unpack8(rb[c], q);
#pragma unroll
      for (int i = 0; i < 8; ++i) var += (q[i] - mean) * (q[i] - mean);
    }
    const float rstd = rsqrtf(warp_sum(var) / h + a.eps);
    for (int c = lane; c < nc; c += 32) {
      float q[8], gm[8], bt[8];
      unpack8(rb[c], q);
      load8(a.gamma + c * 8, gm);
      load8(a.beta + c * 8, bt);
#pragma unroll
      for (int i = 0; i < 8; ++i) q[i] = (q[i] - mean) * rstd * gm[i] + bt[i];
      store8(a.ln_out + (size_t)row * a.ld_ln + c * 8, q);
    }
    if (lane == 0) {
      a.mean[row] = mean;
      a.rstd[row] = rstd;
    }
  }
}

// ------------------------------------------------------------------------------ two-shot phase 1
// Same per-element arithmetic (and order) as the one-shot kernels, so one-shot and two-shot results
// are bit-identical.
template <int NT>
__global__ void __launch_bounds__(256) ar_rs_kernel(ArRsArgs a) {
  constexpr int CH = ar_ch(NT);
  griddep_wait();
  griddep_launch();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int h = a.h, nc = h >> 3;
  const __nv_bfloat16 *src[NT];
  row_sources<NT>(a.partial, 0, 0, src);
  for (int row = a.row0 + blockIdx.x * nw + warp; row < a.row1; row += gridDim.x * nw) {
    const size_t ro = (size_t)row * h;
    for (int c0 = lane; c0 < nc; c0 += 32 * CH) {
      float v[CH][8];
      rank_sum<NT, CH>(src, ro, c0, nc, v);
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        const int c = c0 + 32 * i;
        if (c >= nc) continue;
        if (a.resid) {
          add8(a.bias + c * 8, v[i]);
          add8(a.resid + ro + c * 8, v[i]);
        }
        store8(a.out + ro + c * 8, v[i]);
      }
    }
  }
}

// ------------------------------------------------------------------------------ backward all-reduce
template <int G, int NT, bool STASH>
__global__ void __launch_bounds__(256) ar_bwd_kernel(ArBwdArgs a, PeerSync ps) {
  constexpr int CH = ar_ch(NT);
  griddep_wait();
  griddep_launch();
  extern __shared__ __align__(16) float du_s[];  // [G][h] the all-reduced gradient (bf16-rounded),
                                                 // then [G][h/8] uint4 x_ln rows, [G][h/8] uint4 dres rows
  __shared__ float s_mean[G], s_rstd[G];
  uint4 *xs = reinterpret_cast<uint4 *>(du_s + (size_t)G * a.h), *ds_res = xs + (size_t)G * (a.h >> 3);
  {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int h = a.h, nc = h >> 3;
    const float inv_h = 1.f / h;
    const int ngroups = a.m / G;
    const bool gathered = a.chunk > 0;
    for (int grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
      // phase 1: warp per row -- all-reduce, LN backward, residual
      for (int ri = warp; ri < G; ri += 8) {
        const int row = grp * G + ri;
        const size_t ro = (size_t)row * h;
        const float mean = a.mean[row], rstd = a.rstd[row];
        float acc1 = 0.f, acc2 = 0.f;
        const __nv_bfloat16 *src[NT];
        row_sources<NT>(a.partial, a.chunk, row, src);
        for (int c0 = lane; c0 < nc; c0 += 32 * CH) {
          float dv[CH][8];
          rank_sum<NT, CH>(src, ro, c0, nc, dv);
#pragma unroll
          for (int i = 0; i < CH; ++i) {
            const int c = c0 + 32 * i;
            if (c >= nc) continue;
            float x[8], gm[8];
            if (!gathered) {
#pragma unroll
              for (int k = 0; k < 8; ++k) dv[i][k] = bf16_round(dv[i][k]);  // AR result rounded once (R10)
            }
            float4 *ds = reinterpret_cast<float4 *>(du_s + ri * h + c * 8);
            ds[0] = make_float4(dv[i][0], dv[i][1], dv[i][2], dv[i][3]);
            ds[1] = make_float4(dv[i][4], dv[i][5], dv[i][6], dv[i][7]);
            const uint4 xr = *reinterpret_cast<const uint4 *>(a.x_ln + ro + c * 8);
            if constexpr (STASH) {
              xs[ri * nc + c] = xr;
              ds_res[ri * nc + c] = *reinterpret_cast<const uint4 *>(a.dres + ro + c * 8);
            }
            unpack8(xr, x);
            load8(a.gamma + c * 8, gm);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const float xh = (x[k] - mean) * rstd, dxh = dv[i][k] * gm[k];
              acc1 += dxh;
              acc2 += dxh * xh;
            }
          }
        }
        __syncwarp();
        const float m1 = warp_sum(acc1) * inv_h, m2 = warp_sum(acc2) * inv_h;
        for (int c = lane; c < nc; c += 32) {
          float x[8], gm[8], dr[8], o[8];
          const float4 *ds = reinterpret_cast<const float4 *>(du_s + ri * h + c * 8);
          const float4 d0 = ds[0], d1 = ds[1];
          const float du[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
          if constexpr (STASH) {
            unpack8(xs[ri * nc + c], x);
            unpack8(ds_res[ri * nc + c], dr);
          } else {
            load8(a.x_ln + ro + c * 8, x);
            load8(a.dres + ro + c * 8, dr);
          }
          load8(a.gamma + c * 8, gm);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float xh = (x[i] - mean) * rstd, dxh = du[i] * gm[i];
            o[i] = dr[i] + rstd * (dxh - m1 - xh * m2);
          }
          store8(a.dx + ro + c * 8, o);
        }
        if (lane == 0) {
          s_mean[ri] = mean;
          s_rstd[ri] = rstd;
        }
      }
      __syncthreads();
      // phase 2: fixed-order column partials over the G rows (dbeta = sum du, dgamma = sum du*xhat)
      for (int cc = threadIdx.x; cc < nc; cc += blockDim.x) {
        float sg[8], sb[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) sg[i] = sb[i] = 0.f;
        for (int i = 0; i < G; ++i) {
          float x[8];
          if constexpr (STASH)
            unpack8(xs[i * nc + cc], x);
          else
            load8(a.x_ln + (size_t)(grp * G + i) * h + cc * 8, x);
          const float4 *ds = reinterpret_cast<const float4 *>(du_s + i * h + cc * 8);
          const float4 d0 = ds[0], d1 = ds[1];
          const float du[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            sb[k] += du[k];
            sg[k] += du[k] * ((x[k] - s_mean[i]) * s_rstd[i]);
          }
        }
        float4 *pg = reinterpret_cast<float4 *>(a.part_dg + (size_t)grp * h + cc * 8);
        float4 *pb = reinterpret_cast<float4 *>(a.part_db + (size_t)grp * h + cc * 8);
        pg[0] = make_float4(sg[0], sg[1], sg[2], sg[3]);
        pg[1] = make_float4(sg[4], sg[5], sg[6], sg[7]);
        pb[0] = make_float4(sb[0], sb[1], sb[2], sb[3]);
        pb[1] = make_float4(sb[4], sb[5], sb[6], sb[7]);
      }
      __syncthreads();
    }
  }
}

// ------------------------------------------------------------------------------ LayerNorm forward
__global__ void __launch_bounds__(256) ln_fwd_kernel(const __nv_bfloat16 *x, const __nv_bfloat16 *gamma,
                                                     const __nv_bfloat16 *beta, __nv_bfloat16 *u, int ld_u,
                                                     float *mean_out, float *rstd_out, int m, int h, float eps,
                                                     OnesPad pad) {
  extern __shared__ uint4 row_s[];  // per warp: the x row (one global read; passes 2-3 from smem)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int row = blockIdx.x * nw + warp;
  if (row >= m) return;
  const int nc = h >> 3;
  const size_t ro = (size_t)row * h;
  uint4 *rb = row_s + (size_t)warp * nc;
  float sum = 0.f;
#pragma unroll 4
  for (int c = lane; c < nc; c += 32) {
    const uint4 u4 = *reinterpret_cast<const uint4 *>(x + ro + c * 8);
    rb[c] = u4;
    float q[8];
    unpack8(u4, q);
#pragma unroll
    for (int i = 0; i < 8; ++i) sum += q[i];
  }
  __syncwarp();
  const float mean = warp_sum(sum) / h;
  float var = 0.f;
  for (int c = lane; c < nc; c += 32) {
    float q[8];
    unpack8(rb[c], q);
#pragma unroll
    for (int i = 0; i < 8; ++i) var += (q[i] - mean) * (q[i] - mean);
  }
  const float rstd = rsqrtf(warp_sum(var) / h + eps);
  for (int c = lane; c < nc; c += 32) {
    float q[8], gm[8], bt[8];
    unpack8(rb[c], q);
    load8(gamma + c * 8, gm);
    load8(beta + c * 8, bt);
#pragma unroll
    for (int i = 0; i < 8; ++i) q[i] = (q[i] - mean) * rstd * gm[i] + bt[i];
    store8(u + (size_t)row * ld_u + c * 8, q);
  }
  if (lane < pad.n) {
    uint4 one;
    one.x = pack_bf16(1.f, 0.f);
    one.y = one.z = one.w = 0u;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (k == lane) *reinterpret_cast<uint4 *>(pad.ptr[k] + (size_t)row * pad.ld[k] + pad.col[k]) = one;
  }
  if (lane == 0) {
    mean_out[row] = mean;
    rstd_out[row] = rstd;
  }
}

// ------------------------------------------------------------------------------ token reductions
// Reductions over tokens (bias and LayerNorm gradients) use a structure fixed per SAMPLE, so the
// result is the same whatever the sub-batch split (sub-batches are whole samples, reading R9):
//   per-sample sum in a fixed order, then a chain over samples in order that continues across
//   sub-batch launches through the fp32 gradient itself (bit-identity rule vi).

// Q[i][c] = sum of X over the s rows of sample i: thread (tx, ty) owns 8 columns and rows
// ty, ty+8, ty+16, ... (sequential), then the 8 row-slices are added in order ty = 0..7.
__global__ void __launch_bounds__(256) colsum_sample_kernel(const __nv_bfloat16 *X, int ld, int s, int n, float *Q) {
  __shared__ float red[8][256];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int cc = blockIdx.x * 32 + tx;
  const int i = blockIdx.y;
  float acc[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[k] = 0.f;
  if (cc * 8 < n) {
    const __nv_bfloat16 *base = X + (size_t)i * s * ld + cc * 8;
#pragma unroll 4
    for (int r = ty; r < s; r += 8) {
      float v[8];
      load8(base + (size_t)r * ld, v);
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] += v[k];
    }
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) red[ty][tx * 8 + k] = acc[k];
  __syncthreads();
  if (ty == 0 && cc * 8 < n) {
    float t[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) t[k] = red[0][tx * 8 + k];
    for (int y = 1; y < 8; ++y)
#pragma unroll
      for (int k = 0; k < 8; ++k) t[k] += red[y][tx * 8 + k];
    float4 *q = reinterpret_cast<float4 *>(Q + (size_t)i * n + cc * 8);
    q[0] = make_float4(t[0], t[1], t[2], t[3]);
    q[1] = make_float4(t[4], t[5], t[6], t[7]);
  }
}

// Q_t[i][c] (t < 2 arrays) = fixed-tree sum over the gps partial rows of sample i: thread ty adds
// rows k = ty, ty+8, ... (sequential), then the 8 thread sums are added in order ty = 0..7.
// The structure depends only on the sample, never on the sub-batch split.
__global__ void __launch_bounds__(256) sample_sum_kernel(const float *p0, const float *p1, int gps, int n, float *q0,
                                                         float *q1) {
  __shared__ float red[2][8][32];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int c = blockIdx.x * 32 + tx, i = blockIdx.y;
  float a0 = 0.f, a1 = 0.f;
  if (c < n) {
    const size_t base = (size_t)i * gps * n + c;
#pragma unroll 4
    for (int k = ty; k < gps; k += 8) {
      a0 += p0[base + (size_t)k * n];
      if (p1) a1 += p1[base + (size_t)k * n];
    }
  }
  red[0][ty][tx] = a0;
  red[1][ty][tx] = a1;
  __syncthreads();
  if (ty == 0 && c < n) {
    float t0 = red[0][0][tx], t1 = red[1][0][tx];
#pragma unroll
    for (int y = 1; y < 8; ++y) {
      t0 += red[0][y][tx];
      t1 += red[1][y][tx];
    }
    q0[(size_t)i * n + c] = t0;
    if (p1) q1[(size_t)i * n + c] = t1;
  }
}

// g_t[c] = ((g_t[c] + Q_t[0][c]) + Q_t[1][c]) + ...   (chain over samples in order; it continues
// across sub-batch launches through the fp32 gradient itself)
__global__ void sample_chain_kernel(const float *q0, const float *q1, int b, int n, float *g0, float *g1) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  float a = g0[c];
  for (int i = 0; i < b; ++i) a += q0[(size_t)i * n + c];
  g0[c] = a;
  if (q1) {
    float e = g1[c];
    for (int i = 0; i < b; ++i) e += q1[(size_t)i * n + c];
    g1[c] = e;
  }
}

// ------------------------------------------------------------------------------ host
// CTAs that can be resident at once (grid sizing only; no cross-CTA waiting happens in the kernels).
static int resident_ctas(const void *kern, int threads, size_t smem) {
  int per_sm = 0, dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
  return per_sm * sms;
}
static int clamp_ctas(int want, int work, int resident) {
  if (want <= 0 || want > resident) want = resident;
  if (want > MAX_AR_CTAS) want = MAX_AR_CTAS;
  if (want > work) want = work;
  return want < 1 ? 1 : want;
}

template <int NT>
static cudaError_t ar_fwd_t(const ArFwdArgs &a, const PeerSync &ps, cudaStream_t st) {
  const size_t smem = a.do_ln ? (size_t)8 * a.h * 2 : 0;  // 8 warps x one bf16 row
  static int resident[MAX_DEV] = {};
  static size_t res_smem[MAX_DEV], attr[MAX_DEV] = {};
  static bool init[MAX_DEV] = {};
  const int dev = cur_device();
  if (smem > attr[dev]) {
    cudaError_t e = cudaFuncSetAttribute(ar_fwd_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr[dev] = smem;
  }
  if (!init[dev] || res_smem[dev] != smem) {
    resident[dev] = resident_ctas((const void *)ar_fwd_kernel<NT>, 256, smem);
    res_smem[dev] = smem;
    init[dev] = true;
  }
  const int grid = clamp_ctas(a.ctas, (a.m + 7) / 8, resident[dev]);
  return launch_k(ar_fwd_kernel<NT>, dim3(grid), dim3(256), smem, st, a.pdl, a, ps);
}
cudaError_t ar_fwd(const ArFwdArgs &a, const PeerSync &ps, cudaStream_t st) {
  switch (a.chunk > 0 ? 1 : a.T) {
    case 1: return ar_fwd_t<1>(a, ps, st);
    case 2: return ar_fwd_t<2>(a, ps, st);
    case 4: return ar_fwd_t<4>(a, ps, st);
    case 8: return ar_fwd_t<8>(a, ps, st);
  }
  return cudaErrorInvalidValue;
}

int ar_bwd_group_rows(int h) { return 8; }

template <int NT>
static cudaError_t ar_rs_t(const ArRsArgs &a, cudaStream_t st) {
  static int resident[MAX_DEV] = {};
  const int dev = cur_device();
  if (!resident[dev]) resident[dev] = resident_ctas((const void *)ar_rs_kernel<NT>, 256, 0);
  const int grid = clamp_ctas(a.ctas, (a.row1 - a.row0 + 7) / 8, resident[dev]);
  return launch_k(ar_rs_kernel<NT>, dim3(grid), dim3(256), 0, st, a.pdl, a);
}
cudaError_t ar_rs(const ArRsArgs &a, cudaStream_t st) {
  if (a.row1 <= a.row0) return cudaSuccess;
  switch (a.T) {
    case 1: return ar_rs_t<1>(a, st);
    case 2: return ar_rs_t<2>(a, st);
    case 4: return ar_rs_t<4>(a, st);
    case 8: return ar_rs_t<8>(a, st);
  }
  return cudaErrorInvalidValue;
}

template <int NT, bool STASH>
static cudaError_t ar_bwd_t(const ArBwdArgs &a, const PeerSync &ps, cudaStream_t st) {
  constexpr int G = 8;
  // du fp32 rows, plus (STASH) the x_ln and dres bf16 rows so the later passes read smem, not HBM
  const size_t smem = (size_t)G * a.h * (sizeof(float) + (STASH ? 4 : 0));
  static size_t attr[MAX_DEV] = {};
  const int dev = cur_device();
  if (smem > attr[dev]) {
    cudaError_t e =
        cudaFuncSetAttribute(ar_bwd_kernel<G, NT, STASH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr[dev] = smem;
  }
  static int resident[MAX_DEV] = {};
  static size_t res_smem[MAX_DEV] = {};
  if (!resident[dev] || res_smem[dev] != smem) {
    resident[dev] = resident_ctas((const void *)ar_bwd_kernel<G, NT, STASH>, 256, smem);
    res_smem[dev] = smem;
  }
  const int grid = clamp_ctas(a.ctas, a.m / G, resident[dev]);
  return launch_k(ar_bwd_kernel<G, NT, STASH>, dim3(grid), dim3(256), smem, st, a.pdl, a, ps);
}
cudaError_t ar_bwd(const ArBwdArgs &a, const PeerSync &ps, cudaStream_t st) {
  if (a.G != 8 || a.m % 8) return cudaErrorInvalidValue;
  // Stashing x_ln / dres rows in smem (STASH) measured slower (25.7 vs 20.8 us per launch at h = 1600):
  // 102 KB of smem per CTA halves the resident CTAs of this latency-bound kernel.  Kept selectable.
  const char *e = getenv("MERAK_ARBWD_STASH");
  const bool stash = e && atoi(e) == 1 && (size_t)8 * a.h * 8 <= 160 * 1024;
  switch (a.chunk > 0 ? 1 : a.T) {
    case 1: return stash ? ar_bwd_t<1, true>(a, ps, st) : ar_bwd_t<1, false>(a, ps, st);
    case 2: return stash ? ar_bwd_t<2, true>(a, ps, st) : ar_bwd_t<2, false>(a, ps, st);
    case 4: return stash ? ar_bwd_t<4, true>(a, ps, st) : ar_bwd_t<4, false>(a, ps, st);
    case 8: return stash ? ar_bwd_t<8, true>(a, ps, st) : ar_bwd_t<8, false>(a, ps, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t ln_fwd(const __nv_bfloat16 *x, const __nv_bfloat16 *g, const __nv_bfloat16 *b, __nv_bfloat16 *u,
                   int ld_u, float *mean, float *rstd, int m, int h, float eps, const OnesPad &pad, cudaStream_t st) {
  const size_t smem = (size_t)8 * h * 2;
  static size_t attr[MAX_DEV] = {};
  const int dev = cur_device();
  if (smem > attr[dev]) {
    cudaError_t e = cudaFuncSetAttribute(ln_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr[dev] = smem;
  }
  ln_fwd_kernel<<<(m + 7) / 8, 256, smem, st>>>(x, g, b, u, ld_u, mean, rstd, m, h, eps, pad);
  return cudaGetLastError();
}

cudaError_t colsum_sample(const __nv_bfloat16 *X, int ld, int s, int b, int n, float *Q, cudaStream_t st) {
  if (n % 8) return cudaErrorInvalidValue;
  dim3 grid((n / 8 + 31) / 32, b);
  colsum_sample_kernel<<<grid, dim3(32, 8), 0, st>>>(X, ld, s, n, Q);
  return cudaGetLastError();
}

cudaError_t sample_reduce2(const float *p0, const float *p1, int gps, int b, int n, float *q0, float *q1, float *g0,
                           float *g1, cudaStream_t st) {
  dim3 grid((n + 31) / 32, b);
  sample_sum_kernel<<<grid, dim3(32, 8), 0, st>>>(p0, p1, gps, n, q0, q1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  sample_chain_kernel<<<(n + 127) / 128, 128, 0, st>>>(q0, p1 ? q1 : nullptr, b, n, g0, g1);
  return cudaGetLastError();
}

template <int NT>
static cudaError_t ar_preload_t() {
  const void *ks[] = {(const void *)ar_fwd_kernel<NT>, (const void *)ar_rs_kernel<NT>,
                      (const void *)ar_bwd_kernel<8, NT, false>, (const void *)ar_bwd_kernel<8, NT, true>};
  for (const void *k : ks) {
    cudaError_t e = touch_kernel(k);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t ln_ar_preload() {
  const void *ks[] = {(const void *)peer_ready_kernel, (const void *)ln_fwd_kernel, (const void *)colsum_sample_kernel,
                      (const void *)sample_sum_kernel, (const void *)sample_chain_kernel};
  for (const void *k : ks) {
    cudaError_t e = touch_kernel(k);
    if (e != cudaSuccess) return e;
  }
  cudaError_t e;
  if ((e = ar_preload_t<1>()) != cudaSuccess) return e;
  if ((e = ar_preload_t<2>()) != cudaSuccess) return e;
  if ((e = ar_preload_t<4>()) != cudaSuccess) return e;
  return ar_preload_t<8>();
}

}  // namespace mk
