// attention_bwd_tc.cu -- causal attention backward on tcgen05 / TMEM.
//
// Deterministic (bit-identity rule ii): two kernels, no atomics, each 320 threads
// (warp 0 TMA, warp 1 TMEM owner + MMA issuer, warps 2-9 element-wise: thread = TMEM lane, the two
// warpgroups split the 64 columns of every tile -- the element-wise work is the latency-bound part):
//   dQ kernel   one CTA per 128-query tile; for each 64-key half tile j:
//               S = Q K_j^T, dP = dO V_j^T (TMEM) -> P = exp2(S*scale*log2e - lse), dS = P (dP - delta)
//               (bf16, swizzled smem) -> dQ += dS K_j (TMEM accumulator).  Also writes delta =
//               rowsum(dO * O) for the second kernel.
//   dK/dV kernel one CTA per 128-key tile; for each 64-query half tile i (from the diagonal on):
//               S^T = K Q_i^T, dP^T = V dO_i^T -> P^T, dS^T (smem) -> dV += P^T dO_i, dK += dS^T Q_i.
// Q / dO / K / V tiles serve as K-major operands for the score products and, unchanged, as MN-major
// operands for the accumulations (rows of 128 B in the 128-B swizzle are both canonical layouts).
#include <math.h>

#include "kernels.h"
#include "ptx.cuh"

namespace mk {

namespace {

constexpr int TR = 128;  // rows per CTA (TMEM lanes)
constexpr int TH = 64;   // half tile
constexpr int NTHR = 320;  // 2 + 8 warps
constexpr int NEW = 8;     // element-wise warps (two warpgroups)

MK_DEV void tmem_ld16b(uint32_t taddr, uint32_t *r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

template <int D>
struct BwdCfg {
  static constexpr int NA = (D + 63) / 64;
  static constexpr int F_ATOM = TR * 128;  // [128 rows][64] bf16
  static constexpr int H_ATOM = TH * 128;  // [64 rows][64] bf16
  static constexpr int FULL = NA * F_ATOM;
  static constexpr int HALF = NA * H_ATOM;
  static constexpr int X_BYTES = TR * 128;  // [128 rows][64] bf16 element-wise result (one atom)
  // dQ kernel: Q, dO (full) + KST stages of K, V (half) + one dS buffer
  static constexpr int KST = (D <= 64) ? 3 : 2;
  static constexpr int DQ_SMEM = 2 * FULL + KST * 2 * HALF + X_BYTES + 1024 + 256;
  // dK/dV kernel: K, V (full) + 2 stages of Q, dO (half) + lse/delta + P^T, dS^T
  static constexpr int DKV_SMEM = 2 * FULL + 2 * (2 * HALF + 512) + 2 * X_BYTES + 1024 + 256;
  static constexpr int DQ_TMEM = (128 + D <= 256) ? 256 : 512;
  static constexpr int DKV_TMEM = (128 + 2 * D <= 256) ? 256 : 512;
  static constexpr int DQ_MIN = (2 * (DQ_SMEM + 1024) <= 228 * 1024 && DQ_TMEM == 256) ? 2 : 1;
  static constexpr int DKV_MIN = (2 * (DKV_SMEM + 1024) <= 228 * 1024 && DKV_TMEM == 256) ? 2 : 1;
};

// Diagnostics (AttnArgs::dbg): one recording thread per CTA stores SM-clock stamps --
// [0] entry, [1] prologue done, [2 + j] iteration j's scores ready (j < 54), [60] epilogue start,
// [61] exit, [56]/[57] globaltimer at entry / exit, [62] SM id, [63] iteration count.
MK_DEV unsigned long long *dbg_slot(unsigned long long *base) {
  if (!base) return nullptr;
  const size_t cta = blockIdx.x + (size_t)gridDim.x * (blockIdx.y + (size_t)gridDim.y * blockIdx.z);
  return base + cta * 64;
}
MK_DEV unsigned long long clk64() {
  unsigned long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}
MK_DEV unsigned int smid() {
  unsigned int r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

// 32 scores of this thread's row -> 32 bf16 values packed in 16 words
MK_DEV void put_row_chunk(uint8_t *row, int r, int c32, const uint32_t (&w)[16]) {
  // columns c32*32 .. +31 = 16-B chunks 4*c32 .. 4*c32+3 of the 128-B row (128-B swizzle)
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int ch = c32 * 4 + u;
    *reinterpret_cast<uint4 *>(row + ((ch ^ (r & 7)) << 4)) = make_uint4(w[4 * u], w[4 * u + 1], w[4 * u + 2], w[4 * u + 3]);
  }
}

}  // namespace

// ------------------------------------------------------------------------------------------ dQ
template <int D>
__device__ __forceinline__ void dq_body(const CUtensorMap *tmq_p, const CUtensorMap *tmo_p, const CUtensorMap *tmkv_p,
                                        const AttnArgs &a, const int tile) {
  const CUtensorMap &tmq = *tmq_p, &tmo = *tmo_p, &tmkv = *tmkv_p;
  using C = BwdCfg<D>;
  constexpr int NA = C::NA;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sQ = smem, *sO = sQ + C::FULL;
  constexpr int KST = C::KST;
  uint8_t *sK = sO + C::FULL;            // [KST][HALF]
  uint8_t *sV = sK + KST * C::HALF;      // [KST][HALF]
  uint8_t *sX = sV + KST * C::HALF;      // [X_BYTES] dS
  uint64_t *bar = reinterpret_cast<uint64_t *>(sX + C::X_BYTES);
  uint64_t *qd_full = bar, *kv_full = bar + 1, *kv_empty = bar + 1 + KST, *sp_full = bar + 1 + 2 * KST;
  uint64_t *sp_free = sp_full + 1, *x_full = sp_full + 2, *x_free = sp_full + 3;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(sp_full + 4);
  constexpr uint32_t S_COL = 0, DP_COL = 64, DQ_COL = 128;

  const int s = a.s, H = a.heads, hr = H * D;
  const int nqt = (s + TR - 1) / TR;
  const int qt = nqt - 1 - tile;  // heaviest (most key tiles) first
  const int head = blockIdx.x, bi = blockIdx.y, tok0 = bi * s;
  const int J = min(2 * (qt + 1), (s + TH - 1) / TH);
  const int warp = warp_id(), lane = lane_id();
  unsigned long long *dbg = (warp == 2 && lane == 0) ? dbg_slot(a.dbg) : nullptr;
  if (dbg) {
    dbg[0] = clk64();
    dbg[56] = globaltimer();
    dbg[62] = smid();
    dbg[63] = J;
  }

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmq);
    tma_prefetch(&tmo);
    tma_prefetch(&tmkv);
    mbar_init(qd_full, 1);
    for (int i = 0; i < KST; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    mbar_init(x_full, NEW);
    mbar_init(x_free, 1);
    mbar_init(sp_full, 1);
    mbar_init(sp_free, NEW);
    fence_mbar_init();
    fence_proxy_async();
  }
  if (warp == 1) tmem_alloc<C::DQ_TMEM>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(qd_full, 2 * C::FULL);
      for (int c = 0; c < NA; ++c) {
        tma_load_2d(sQ + c * C::F_ATOM, &tmq, qd_full, head * D + c * 64, tok0 + qt * TR);
        tma_load_2d(sO + c * C::F_ATOM, &tmo, qd_full, head * D + c * 64, tok0 + qt * TR);
      }
    }
    for (int j = 0; j < J; ++j) {
      const int st = j % KST;
      mbar_wait(&kv_empty[st], ((j / KST) & 1) ^ 1);
      if (lane == 0) {
        mbar_expect_tx(&kv_full[st], 2 * C::HALF);
        for (int c = 0; c < NA; ++c) {
          tma_load_2d(sK + st * C::HALF + c * C::H_ATOM, &tmkv, &kv_full[st], hr + head * D + c * 64, tok0 + j * TH);
          tma_load_2d(sV + st * C::HALF + c * C::H_ATOM, &tmkv, &kv_full[st], 2 * hr + head * D + c * 64,
                      tok0 + j * TH);
        }
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc_s = idesc_bf16(TR, TH, false, false);
    constexpr uint32_t idesc_q = idesc_bf16(TR, D, false, true);  // dS (K-major) x K (MN-major)
    mbar_wait(qd_full, 0);
    for (int j = 0; j <= J; ++j) {
      if (j < J) {
        const int st = j % KST;
        mbar_wait(&kv_full[st], (j / KST) & 1);
        mbar_wait(sp_free, (j & 1) ^ 1);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t q0 = smem_u32(sQ), o0 = smem_u32(sO);
          const uint32_t k0 = smem_u32(sK + st * C::HALF), v0 = smem_u32(sV + st * C::HALF);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t fo = (kk >> 2) * C::F_ATOM + (kk & 3) * 32, ho = (kk >> 2) * C::H_ATOM + (kk & 3) * 32;
            tc_mma_f16(tmem + S_COL, sdesc_sw128(q0 + fo, 16, 1024), sdesc_sw128(k0 + ho, 16, 1024), idesc_s,
                       kk > 0 ? 1u : 0u);
            tc_mma_f16(tmem + DP_COL, sdesc_sw128(o0 + fo, 16, 1024), sdesc_sw128(v0 + ho, 16, 1024), idesc_s,
                       kk > 0 ? 1u : 0u);
          }
          tc_commit(sp_full);
        }
        __syncwarp();
      }
      if (j >= 1) {
        const int i = j - 1, st = i % KST;
        mbar_wait(x_full, i & 1);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t x0 = smem_u32(sX), k0 = smem_u32(sK + st * C::HALF);
#pragma unroll
          for (int kk = 0; kk < TH / 16; ++kk)
            tc_mma_f16(tmem + DQ_COL, sdesc_sw128(x0 + kk * 32, 16, 1024), sdesc_sw128(k0 + kk * 2048, C::H_ATOM, 1024),
                       idesc_q, (i > 0 || kk > 0) ? 1u : 0u);
          tc_commit(x_free);
          tc_commit(&kv_empty[st]);
        }
        __syncwarp();
      }
    }
  } else {
    const int q = warp & 3, r = q * 32 + lane, qi = qt * TR + r, cw = (warp - 2) >> 2;
    const uint32_t lb = tmem + ((uint32_t)(q * 32) << 16);
    const float scale = 1.f / sqrtf((float)D), sl2 = 1.4426950408889634f * scale;
    const size_t srow = ((size_t)bi * H + head) * s;
    // delta = rowsum(dO * O) comes from attn_delta_kernel (launched first)
    const float lse = qi < s ? a.lse[srow + qi] : INFINITY, del = qi < s ? a.delta[srow + qi] : 0.f;
    const float ls = lse;
    if (dbg) dbg[1] = clk64();
    for (int j = 0; j < J; ++j) {
      mbar_wait(sp_full, j & 1);
      tc_fence_after();
      if (dbg && j < 54) dbg[2 + j] = clk64();
      const int kj0 = j * TH;
      const bool mask = (kj0 + TH - 1 > qt * TR) || (kj0 + TH > s);
      uint32_t w[16];  // this warpgroup's 32 columns, bf16-packed
#pragma unroll
      for (int hc = 0; hc < 2; ++hc) {
        const int col0 = cw * 32 + hc * 16;
        uint32_t sv[16], dv[16];
        tmem_ld16b(lb + S_COL + col0, sv);
        tmem_ld16b(lb + DP_COL + col0, dv);
        tmem_ld_wait();
#pragma unroll
        for (int k = 0; k < 16; k += 2) {
          const int kj = kj0 + col0 + k;
          float p0 = fast_exp2(fmaf(__uint_as_float(sv[k]), sl2, -ls));
          float p1 = fast_exp2(fmaf(__uint_as_float(sv[k + 1]), sl2, -ls));
          float g0 = p0 * (__uint_as_float(dv[k]) - del), g1 = p1 * (__uint_as_float(dv[k + 1]) - del);
          if (mask) {
            if (!(kj <= qi && kj < s)) g0 = 0.f;
            if (!(kj + 1 <= qi && kj + 1 < s)) g1 = 0.f;
          }
          w[hc * 8 + (k >> 1)] = pack_bf16(g0, g1);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(sp_free);
      mbar_wait(x_free, (j & 1) ^ 1);  // the dS buffer was read by the MMA of j-1
      put_row_chunk(sX + r * 128, r, cw, w);
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(x_full);
    }
    const int last = J - 1;
    if (dbg) dbg[60] = clk64();
    mbar_wait(x_free, last & 1);
    tc_fence_after();
    __nv_bfloat16 *dst = reinterpret_cast<__nv_bfloat16 *>(a.dqkv) + (size_t)(tok0 + qi) * 3 * hr + head * D;
#pragma unroll
    for (int c = 0; c < D / 16; ++c) {
      if ((c & 1) != cw) continue;  // warp-uniform: the warpgroups take alternate 16-column chunks
      uint32_t o[16];
      tmem_ld16b(lb + DQ_COL + c * 16, o);
      tmem_ld_wait();
      if (qi < s) {
        uint4 u0, u1;
        u0.x = pack_bf16(__uint_as_float(o[0]) * scale, __uint_as_float(o[1]) * scale);
        u0.y = pack_bf16(__uint_as_float(o[2]) * scale, __uint_as_float(o[3]) * scale);
        u0.z = pack_bf16(__uint_as_float(o[4]) * scale, __uint_as_float(o[5]) * scale);
        u0.w = pack_bf16(__uint_as_float(o[6]) * scale, __uint_as_float(o[7]) * scale);
        u1.x = pack_bf16(__uint_as_float(o[8]) * scale, __uint_as_float(o[9]) * scale);
        u1.y = pack_bf16(__uint_as_float(o[10]) * scale, __uint_as_float(o[11]) * scale);
        u1.z = pack_bf16(__uint_as_float(o[12]) * scale, __uint_as_float(o[13]) * scale);
        u1.w = pack_bf16(__uint_as_float(o[14]) * scale, __uint_as_float(o[15]) * scale);
        *reinterpret_cast<uint4 *>(dst + c * 16) = u0;
        *reinterpret_cast<uint4 *>(dst + c * 16 + 8) = u1;
      }
    }
  }
  if (dbg) {
    dbg[61] = clk64();
    dbg[57] = globaltimer();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::DQ_TMEM>(tmem);
  }
}

// ------------------------------------------------------------------------------------------ dK / dV
template <int D>
__device__ __forceinline__ void dkdv_body(const CUtensorMap *tmf_p, const CUtensorMap *tmh_p,
                                          const CUtensorMap *tmoh_p, const AttnArgs &a, const int tile) {
  const CUtensorMap &tmf = *tmf_p, &tmh = *tmh_p, &tmoh = *tmoh_p;
  using C = BwdCfg<D>;
  constexpr int NA = C::NA;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sK = smem, *sV = sK + C::FULL;
  uint8_t *sQ = sV + C::FULL;            // [2][HALF]
  uint8_t *sO = sQ + 2 * C::HALF;        // [2][HALF] dO
  uint8_t *sP = sO + 2 * C::HALF;        // P^T  [128 keys][64 q]
  uint8_t *sS = sP + C::X_BYTES;         // dS^T [128 keys][64 q]
  float *sL = reinterpret_cast<float *>(sS + C::X_BYTES);  // [2][64] lse, then [2][64] delta
  float *sD = sL + 2 * TH;
  uint64_t *bar = reinterpret_cast<uint64_t *>(sD + 2 * TH);
  uint64_t *kv_full = bar, *q_full = bar + 1, *q_empty = bar + 3, *sp_full = bar + 5, *sp_free = bar + 6;
  uint64_t *x_full = bar + 7, *x_free = bar + 8;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bar + 9);
  constexpr uint32_t ST_COL = 0, DPT_COL = 64, DV_COL = 128, DK_COL = 128 + D;

  const int s = a.s, H = a.heads, hr = H * D;
  const int kt = tile;  // kt = 0 has the most query tiles: heaviest first
  const int head = blockIdx.x, bi = blockIdx.y, tok0 = bi * s;
  const int i0 = 2 * kt, NI = (s + TH - 1) / TH - i0;
  const size_t srow = ((size_t)bi * H + head) * s;
  const int warp = warp_id(), lane = lane_id();
  unsigned long long *dbg = (warp == 2 && lane == 0) ? dbg_slot(a.dbg) : nullptr;
  if (dbg) {
    dbg[0] = clk64();
    dbg[56] = globaltimer();
    dbg[62] = smid();
    dbg[63] = NI;
  }

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmf);
    tma_prefetch(&tmh);
    tma_prefetch(&tmoh);
    mbar_init(kv_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
    }
    mbar_init(sp_full, 1);
    mbar_init(sp_free, NEW);
    mbar_init(x_full, NEW);
    mbar_init(x_free, 1);
    fence_mbar_init();
    fence_proxy_async();
  }
  if (warp == 1) tmem_alloc<C::DKV_TMEM>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(kv_full, 2 * C::FULL);
      for (int c = 0; c < NA; ++c) {
        tma_load_2d(sK + c * C::F_ATOM, &tmf, kv_full, hr + head * D + c * 64, tok0 + kt * TR);
        tma_load_2d(sV + c * C::F_ATOM, &tmf, kv_full, 2 * hr + head * D + c * 64, tok0 + kt * TR);
      }
    }
    for (int ii = 0; ii < NI; ++ii) {
      const int i = i0 + ii, st = ii & 1;
      mbar_wait(&q_empty[st], ((ii >> 1) & 1) ^ 1);
      if (lane == 0) {
        const int nrow = min(TH, s - i * TH);
        const uint32_t lbytes = (uint32_t)nrow * 4;
        mbar_expect_tx(&q_full[st], 2 * C::HALF + 2 * lbytes);
        for (int c = 0; c < NA; ++c) {
          tma_load_2d(sQ + st * C::HALF + c * C::H_ATOM, &tmh, &q_full[st], head * D + c * 64, tok0 + i * TH);
          tma_load_2d(sO + st * C::HALF + c * C::H_ATOM, &tmoh, &q_full[st], head * D + c * 64, tok0 + i * TH);
        }
        bulk_load_1d(sL + st * TH, a.lse + srow + i * TH, lbytes, &q_full[st]);
        bulk_load_1d(sD + st * TH, a.delta + srow + i * TH, lbytes, &q_full[st]);
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc_s = idesc_bf16(TR, TH, false, false);
    constexpr uint32_t idesc_g = idesc_bf16(TR, D, false, true);
    mbar_wait(kv_full, 0);
    for (int ii = 0; ii <= NI; ++ii) {
      if (ii < NI) {
        const int st = ii & 1;
        mbar_wait(&q_full[st], (ii >> 1) & 1);
        mbar_wait(sp_free, (ii & 1) ^ 1);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t k0 = smem_u32(sK), v0 = smem_u32(sV);
          const uint32_t q0 = smem_u32(sQ + st * C::HALF), o0 = smem_u32(sO + st * C::HALF);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t fo = (kk >> 2) * C::F_ATOM + (kk & 3) * 32, ho = (kk >> 2) * C::H_ATOM + (kk & 3) * 32;
            tc_mma_f16(tmem + ST_COL, sdesc_sw128(k0 + fo, 16, 1024), sdesc_sw128(q0 + ho, 16, 1024), idesc_s,
                       kk > 0 ? 1u : 0u);
            tc_mma_f16(tmem + DPT_COL, sdesc_sw128(v0 + fo, 16, 1024), sdesc_sw128(o0 + ho, 16, 1024), idesc_s,
                       kk > 0 ? 1u : 0u);
          }
          tc_commit(sp_full);
        }
        __syncwarp();
      }
      if (ii >= 1) {
        const int p = ii - 1, st = p & 1;
        mbar_wait(x_full, p & 1);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t pp = smem_u32(sP), ps = smem_u32(sS);
          const uint32_t q0 = smem_u32(sQ + st * C::HALF), o0 = smem_u32(sO + st * C::HALF);
#pragma unroll
          for (int kk = 0; kk < TH / 16; ++kk) {
            const uint32_t acc = (p > 0 || kk > 0) ? 1u : 0u;
            tc_mma_f16(tmem + DV_COL, sdesc_sw128(pp + kk * 32, 16, 1024), sdesc_sw128(o0 + kk * 2048, C::H_ATOM, 1024),
                       idesc_g, acc);
            tc_mma_f16(tmem + DK_COL, sdesc_sw128(ps + kk * 32, 16, 1024), sdesc_sw128(q0 + kk * 2048, C::H_ATOM, 1024),
                       idesc_g, acc);
          }
          tc_commit(x_free);
          tc_commit(&q_empty[st]);
        }
        __syncwarp();
      }
    }
  } else {
    const int q = warp & 3, r = q * 32 + lane, kj = kt * TR + r, cw = (warp - 2) >> 2;
    const uint32_t lb = tmem + ((uint32_t)(q * 32) << 16);
    const float scale = 1.f / sqrtf((float)D), sl2 = 1.4426950408889634f * scale;
    if (dbg) dbg[1] = clk64();
    for (int ii = 0; ii < NI; ++ii) {
      const int i = i0 + ii, st = ii & 1;
      const int qi0 = i * TH;
      mbar_wait(&q_full[st], (ii >> 1) & 1);  // lse / delta of this half tile are in smem
      mbar_wait(sp_full, ii & 1);
      tc_fence_after();
      if (dbg && ii < 54) dbg[2 + ii] = clk64();
      const bool mask = (qi0 < kt * TR + TR - 1) || (qi0 + TH > s);
      const float *L = sL + st * TH, *Dl = sD + st * TH;
      uint32_t wp[16], ws[16];  // this warpgroup's 32 columns of P^T and dS^T, bf16-packed
#pragma unroll
      for (int hc = 0; hc < 2; ++hc) {
        const int col0 = cw * 32 + hc * 16;
        uint32_t sv[16], dv[16];
        tmem_ld16b(lb + ST_COL + col0, sv);
        tmem_ld16b(lb + DPT_COL + col0, dv);
        tmem_ld_wait();
#pragma unroll
        for (int k = 0; k < 16; k += 2) {
          const int c = col0 + k, qi = qi0 + c;
          float p0 = fast_exp2(fmaf(__uint_as_float(sv[k]), sl2, -L[c]));
          float p1 = fast_exp2(fmaf(__uint_as_float(sv[k + 1]), sl2, -L[c + 1]));
          if (mask) {
            if (!(kj <= qi && qi < s)) p0 = 0.f;
            if (!(kj <= qi + 1 && qi + 1 < s)) p1 = 0.f;
          }
          const float g0 = p0 * (__uint_as_float(dv[k]) - Dl[c]), g1 = p1 * (__uint_as_float(dv[k + 1]) - Dl[c + 1]);
          wp[hc * 8 + (k >> 1)] = pack_bf16(p0, p1);
          ws[hc * 8 + (k >> 1)] = pack_bf16(g0, g1);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(sp_free);
      mbar_wait(x_free, (ii & 1) ^ 1);  // P^T / dS^T were read by the MMAs of ii-1
      put_row_chunk(sP + r * 128, r, cw, wp);
      put_row_chunk(sS + r * 128, r, cw, ws);
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(x_full);
    }
    const int last = NI - 1;
    if (dbg) dbg[60] = clk64();
    mbar_wait(x_free, last & 1);
    tc_fence_after();
    __nv_bfloat16 *dk = reinterpret_cast<__nv_bfloat16 *>(a.dqkv) + (size_t)(tok0 + kj) * 3 * hr + hr + head * D;
    __nv_bfloat16 *dvp = dk + hr;
#pragma unroll
    for (int c = 0; c < D / 16; ++c) {
      if ((c & 1) != cw) continue;  // warp-uniform: alternate 16-column chunks per warpgroup
      uint32_t ov[16], ok[16];
      tmem_ld16b(lb + DV_COL + c * 16, ov);
      tmem_ld16b(lb + DK_COL + c * 16, ok);
      tmem_ld_wait();
      if (kj < s) {
        uint4 u;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          u.x = pack_bf16(__uint_as_float(ov[8 * hh + 0]), __uint_as_float(ov[8 * hh + 1]));
          u.y = pack_bf16(__uint_as_float(ov[8 * hh + 2]), __uint_as_float(ov[8 * hh + 3]));
          u.z = pack_bf16(__uint_as_float(ov[8 * hh + 4]), __uint_as_float(ov[8 * hh + 5]));
          u.w = pack_bf16(__uint_as_float(ov[8 * hh + 6]), __uint_as_float(ov[8 * hh + 7]));
          *reinterpret_cast<uint4 *>(dvp + c * 16 + 8 * hh) = u;
          u.x = pack_bf16(__uint_as_float(ok[8 * hh + 0]) * scale, __uint_as_float(ok[8 * hh + 1]) * scale);
          u.y = pack_bf16(__uint_as_float(ok[8 * hh + 2]) * scale, __uint_as_float(ok[8 * hh + 3]) * scale);
          u.z = pack_bf16(__uint_as_float(ok[8 * hh + 4]) * scale, __uint_as_float(ok[8 * hh + 5]) * scale);
          u.w = pack_bf16(__uint_as_float(ok[8 * hh + 6]) * scale, __uint_as_float(ok[8 * hh + 7]) * scale);
          *reinterpret_cast<uint4 *>(dk + c * 16 + 8 * hh) = u;
        }
      }
    }
  }
  if (dbg) {
    dbg[61] = clk64();
    dbg[57] = globaltimer();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::DKV_TMEM>(tmem);
  }
}

// ------------------------------------------------------------------------------------------ kernels
// delta = rowsum(dO * O) per (sample, head, query): one thread per (token, head), head fastest, so a
// warp reads contiguous 128-B rows of O and dO.
template <int D>
__global__ void __launch_bounds__(256) attn_delta_kernel(AttnArgs a) {
  const int H = a.heads, hr = H * D;
  const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long)a.b * a.s * H) return;
  const int t = (int)(idx / H), e = (int)(idx % H);
  const __nv_bfloat16 *po = reinterpret_cast<const __nv_bfloat16 *>(a.ctx) + (size_t)t * a.ld_ctx + e * D;
  const __nv_bfloat16 *pd = reinterpret_cast<const __nv_bfloat16 *>(a.dctx) + (size_t)t * hr + e * D;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int c = 0; c < D; c += 8) {
    uint4 uo = *reinterpret_cast<const uint4 *>(po + c), ud = *reinterpret_cast<const uint4 *>(pd + c);
    float2 o0 = unpack_bf16(uo.x), o1 = unpack_bf16(uo.y), o2 = unpack_bf16(uo.z), o3 = unpack_bf16(uo.w);
    float2 d0 = unpack_bf16(ud.x), d1 = unpack_bf16(ud.y), d2 = unpack_bf16(ud.z), d3 = unpack_bf16(ud.w);
    acc[0] += o0.x * d0.x + o0.y * d0.y;
    acc[1] += o1.x * d1.x + o1.y * d1.y;
    acc[2] += o2.x * d2.x + o2.y * d2.y;
    acc[3] += o3.x * d3.x + o3.y * d3.y;
  }
  const int bi = t / a.s, i = t % a.s;
  a.delta[((size_t)bi * H + e) * a.s + i] = (acc[0] + acc[1]) + (acc[2] + acc[3]);
}

// One launch for both halves of the backward (independent once delta exists): grid (heads, b, 2 x
// tiles) with the tile slot slowest, so dispatch is globally heaviest-first; even slots compute dQ
// tiles, odd slots dK/dV tiles, and the causal imbalance of one fills the other.
template <int D>
__global__ void __launch_bounds__(NTHR, BwdCfg<D>::DQ_MIN < BwdCfg<D>::DKV_MIN ? BwdCfg<D>::DQ_MIN : BwdCfg<D>::DKV_MIN)
    attn_bwd_tc_kernel(const __grid_constant__ CUtensorMap tmq_full, const __grid_constant__ CUtensorMap tmq_half,
                       const __grid_constant__ CUtensorMap tmo_full, const __grid_constant__ CUtensorMap tmo_half,
                       AttnArgs a) {
  const int tile = blockIdx.z >> 1;
  if (blockIdx.z & 1)
    dkdv_body<D>(&tmq_full, &tmq_half, &tmo_half, a, tile);
  else
    dq_body<D>(&tmq_full, &tmo_full, &tmq_half, a, tile);
}

// ------------------------------------------------------------------------------------------ host
typedef CUresult (*EncodeTiledFn3)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                   const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static bool make_rows_map(CUtensorMap *m, const void *base, int rows, int cols, int ld, int box_rows) {
  static EncodeTiledFn3 enc = nullptr;
  if (!enc) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return false;
    enc = reinterpret_cast<EncodeTiledFn3>(p);
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {64u, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1u, 1u};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int D>
static cudaError_t bwd_tc_d(const AttnArgs &a, cudaStream_t st) {
  using C = BwdCfg<D>;
  constexpr int SMEM = C::DQ_SMEM > C::DKV_SMEM ? C::DQ_SMEM : C::DKV_SMEM;
  static bool attr[MAX_DEV] = {};
  const int dev = cur_device();
  if (!attr[dev]) {
    cudaError_t e = cudaFuncSetAttribute(attn_bwd_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
    attr[dev] = true;
  }
  const int tokens = a.b * a.s, hr = a.heads * D;
  CUtensorMap mq_full, mq_half, mo_full, mo_half;
  if (!make_rows_map(&mq_full, a.qkv, tokens, 3 * hr, 3 * hr, TR) ||
      !make_rows_map(&mq_half, a.qkv, tokens, 3 * hr, 3 * hr, TH) ||
      !make_rows_map(&mo_full, a.dctx, tokens, hr, hr, TR) || !make_rows_map(&mo_half, a.dctx, tokens, hr, hr, TH))
    return cudaErrorInvalidValue;
  const long nd = (long)tokens * a.heads;
  attn_delta_kernel<D><<<(unsigned)((nd + 255) / 256), 256, 0, st>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  dim3 grid(a.heads, a.b, 2 * ((a.s + TR - 1) / TR));
  attn_bwd_tc_kernel<D><<<grid, NTHR, SMEM, st>>>(mq_full, mq_half, mo_full, mo_half, a);
  return cudaGetLastError();
}

cudaError_t attn_bwd(const AttnArgs &a, cudaStream_t st) {
  switch (a.d) {
    case 32: return bwd_tc_d<32>(a, st);
    case 64: return bwd_tc_d<64>(a, st);
    case 80: return bwd_tc_d<80>(a, st);
    case 96: return bwd_tc_d<96>(a, st);
    case 128: return bwd_tc_d<128>(a, st);
  }
  return cudaErrorNotSupported;
}

template <int D>
static cudaError_t bwd_preload() {
  cudaError_t e = touch_kernel((const void *)attn_delta_kernel<D>);
  return e != cudaSuccess ? e : touch_kernel((const void *)attn_bwd_tc_kernel<D>);
}

cudaError_t attn_bwd_preload_d(int d) {
  switch (d) {
    case 32: return bwd_preload<32>();
    case 64: return bwd_preload<64>();
    case 80: return bwd_preload<80>();
    case 96: return bwd_preload<96>();
    case 128: return bwd_preload<128>();
  }
  return cudaErrorNotSupported;
}

}  // namespace mk
