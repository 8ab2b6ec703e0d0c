// attention_bwd_tc.cu -- causal attention backward on tcgen05 / TMEM.
//
// Per (sample, local head e), with P = softmax(Q K^T / sqrt(d) + causal mask) recomputed from the saved
// base-2 LSE and delta = rowsum(dO * O):
//   dV = P^T dO,  dP = dO V^T,  dS = P (dP - delta),  dQ = dS K / sqrt(d),  dK = dS^T Q / sqrt(d).
//
// One CTA per 128-key tile (TMEM lanes = keys), iterating over the 64-query half-blocks i that see those
// keys (causal: from the diagonal on).  Five MMAs per (key tile, half-block), nothing recomputed twice:
//   S^T  = K Q_i^T      (M 128 keys, N 64 queries, K d)        -> TMEM, double-buffered
//   dP^T = V dO_i^T     (same shape)                            -> TMEM, double-buffered
//   dV  += P^T dO_i     (A = P^T read from TMEM: bf16 written over S^T by the element-wise warps)
//   dK  += dS^T Q_i     (A = dS^T read from TMEM: bf16 written over dP^T by the element-wise warps)
//   dQ_i^T = K^T dS^T   (M = d padded to 128, A = K read MN-major, B = dS^T MN-major from smem) -> TMEM
// 512 threads: warp 0 TMA (K, V once; Q_i, dO_i, lse_i, delta_i per half-block through a stage ring),
// warp 1 TMEM owner + MMA issuer (scores of i+1 issued before the gradient MMAs of i, so the element-wise
// work of one half-block overlaps the tensor core), warps 2-9 element-wise (two warpgroups ping-pong on
// alternate half-blocks; thread = key row), warps 10-13 drain dQ_i^T (thread = d index) into a staging buffer,
// warps 14-15 (one thread each, alternate half-blocks) move the staged blocks into the dQ accumulator in their
// fixed order.
//
// dQ is deterministic (bit-identity rule ii, no atomics): every half-block i of a (sample, head) receives
// its contributions in a FIXED order, key tile floor(i/2) first down to key tile 0, through an fp32
// accumulator in global memory (L2-resident).  A per-(sample, head, i) counter orders them: the first
// contributor stores its partial with a 1-D bulk copy, the later ones bulk-reduce-add (cp.reduce.async.bulk,
// performed in L2), each releasing the counter once its operation has completed.  A small kernel then
// scales, rounds once to bf16 into dqkv and zeroes the counters.  The grid runs the key tiles of a (sample,
// head) lightest-first (largest kt first), so a CTA only ever waits for CTAs dispatched before it (no
// deadlock), which are moreover ahead of it in their own half-block sequence.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "kernels.h"
#include "ptx.cuh"

namespace mk {

namespace {

constexpr int TKEY = 128;  // keys per CTA (TMEM lanes)
constexpr int TQH = 64;    // queries per half-block (N of the score products)
constexpr int NTHR = 512;  // 16 warps
constexpr int DBG_STRIDE = 192;  // u64 clock stamps per CTA (AttnArgs::dbg, diagnostics only)

template <int D>
struct BwdCfg {
  static constexpr int NA = (D + 63) / 64;      // 64-wide swizzle atoms along d
  static constexpr int NB = (D <= 96) ? 2 : 1;  // S^T / dP^T TMEM buffers
  static constexpr int F_ATOM = TKEY * 128;     // [128 rows][64] bf16
  static constexpr int H_ATOM = TQH * 128;      // [64 rows][64] bf16
  // K then V, each NA atoms; with NA = 1 the dQ^T MMA (M = 128 > d) reads its second M chunk from V
  static constexpr int KV_BYTES = NA * F_ATOM;
  static constexpr int QH_BYTES = NA * H_ATOM;
  static constexpr int STAGE_BYTES = 2 * QH_BYTES;               // Q, dO (lse, delta in their own region)
  static constexpr int DS_BYTES = TKEY * 128;                     // dS^T [128 keys][64 q] bf16
  // Q / dO / lse / delta stages: as many as fit (a stage lives from its TMA load to the completion of the
  // half-block's gradient MMAs, so the ring depth hides the load latency)
  static constexpr int STG_BYTES = TQH * D * 4;                   // dQ staging [64 q][d] fp32 (one buffer)
  static constexpr int FIXED = 2 * KV_BYTES + 2 * DS_BYTES + STG_BYTES + 1024 + 256;
  static constexpr int ST_FIT = (227 * 1024 - FIXED) / (STAGE_BYTES + 2 * TQH * 4);
  static constexpr int ST = ST_FIT > 6 ? 6 : ST_FIT;
  static constexpr int SMEM = FIXED + ST * (STAGE_BYTES + 2 * TQH * 4);
  // TMEM columns (32-aligned regions)
  static constexpr uint32_t DPAD = (D + 31) / 32 * 32;
  static constexpr uint32_t SP0 = 0;              // S^T (then P^T) of buffer b: SP0 + 64 b
  static constexpr uint32_t DP0 = 64 * NB;        // dP^T of buffer b:           DP0 + 64 b
  static constexpr uint32_t DV = 128 * NB;
  static constexpr uint32_t DK = DV + DPAD;
  static constexpr uint32_t DQT = DK + DPAD;      // dQ_i^T [128 lanes = d][64 q]
  static_assert(DQT + 64 <= 512, "TMEM budget");
  static_assert(SMEM <= 227 * 1024, "smem budget");
};

MK_DEV void tmem_ld16b(uint32_t taddr, uint32_t *r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
MK_DEV uint32_t ld_acquire_gpu(const int *p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
MK_DEV void st_release_gpu(int *p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
MK_DEV void tmem_st8(uint32_t taddr, const uint32_t *r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
// 1-D bulk smem -> global copy / fp32 add-reduction (bulk async-group of the issuing thread)
MK_DEV void bulk_store(void *dst, const void *src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
MK_DEV void bulk_reduce_add_f32(void *dst, const void *src, uint32_t bytes) {
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
MK_DEV void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

}  // namespace

template <int D>
__global__ void __launch_bounds__(NTHR, 1)
    attn_bwd_tc_kernel(const __grid_constant__ CUtensorMap tm_kv, const __grid_constant__ CUtensorMap tm_q,
                       const __grid_constant__ CUtensorMap tm_o, AttnArgs a) {
  using C = BwdCfg<D>;
  constexpr int NA = C::NA, NB = C::NB, ST = C::ST;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sK = smem, *sV = sK + C::KV_BYTES;
  uint8_t *sStage = sV + C::KV_BYTES;                        // [ST] {Q, dO}   (1024-B aligned atoms)
  uint8_t *sDS = sStage + ST * C::STAGE_BYTES;               // [2] dS^T (one per warpgroup)
  float *sStg = reinterpret_cast<float *>(sDS + 2 * C::DS_BYTES);  // [64][D] dQ staging
  float *sLD = sStg + TQH * D;                               // [ST] {lse[64], delta[64]}
  uint64_t *bar = reinterpret_cast<uint64_t *>(sLD + ST * 2 * TQH);
  uint64_t *kv_full = bar, *q_full = bar + 1, *q_empty = q_full + ST;
  // s_full / p_full / ds_free are per element-wise warpgroup w = ii & 1 (phase (ii >> 1) & 1), so each
  // barrier's completions are consumed in order by one waiter; the TMEM buffer is ii % NB
  uint64_t *s_full = q_empty + ST, *p_full = s_full + 2, *ds_free = p_full + 2;
  uint64_t *dq_full = ds_free + 2, *dq_free = dq_full + 1, *kv_done = dq_free + 1;
  // dQ staging buffer, two 32-row halves h: drain warps <-> bulk thread k = ii & 1; barrier [h * 2 + k]
  uint64_t *stg_full = kv_done + 1, *stg_free = stg_full + 4;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(stg_free + 4);
  auto stQ = [&](int st) { return sStage + st * C::STAGE_BYTES; };
  auto stO = [&](int st) { return sStage + st * C::STAGE_BYTES + C::QH_BYTES; };
  auto stL = [&](int st) { return sLD + st * 2 * TQH; };
  auto stD = [&](int st) { return stL(st) + TQH; };

  const int s = a.s, H = a.heads, hr = H * D;
  const int nkt = (s + TKEY - 1) / TKEY, NQ = (s + TQH - 1) / TQH;
  // 1-D grid in groups of G (sample, head) pairs: inside a group, key tiles descending (lightest first), the
  // pairs of the group fastest.  A key tile's predecessor in the dQ order (kt + 1 of the same pair) is then
  // dispatched G CTAs earlier -- early enough to be ahead of it -- while a group's Q / dO / K / V / dQ
  // accumulator stay L2-resident.
  const int npairs = a.b * H, G = a.attn_group;
  const int grp = (int)blockIdx.x / (G * nkt), r0 = (int)blockIdx.x - grp * G * nkt;
  const int Gg = min(G, npairs - grp * G);  // the last group may be smaller
  const int kt = nkt - 1 - r0 / Gg;
  const int pair = grp * G + r0 % Gg;
  const int head = pair % H, bi = pair / H, tok0 = bi * s;
  const int i0 = 2 * kt, NI = NQ - i0;
  const size_t srow = ((size_t)bi * H + head) * s;
  const int warp = warp_id(), lane = lane_id();

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_kv);
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_o);
    mbar_init(kv_full, 1);
    for (int i = 0; i < ST; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4);
      mbar_init(&ds_free[i], 1);
    }
    mbar_init(dq_full, 1);
    mbar_init(dq_free, 4);
    mbar_init(kv_done, 1);
    for (int k = 0; k < 4; ++k) {
      mbar_init(&stg_full[k], 4);
      mbar_init(&stg_free[k], 1);
    }
    fence_mbar_init();
    fence_proxy_async();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // all 512 columns belong to this CTA, so the allocation starts at lane 0, column 0: a compile-time base
  // keeps every TMEM address warp-uniform (single-instruction MMA issue, no per-lane broadcast loop)
  if (*tmem_slot != 0u) __trap();
  constexpr uint32_t tmem = 0u;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      mbar_expect_tx(kv_full, 2 * C::KV_BYTES);
      for (int c = 0; c < NA; ++c) {
        tma_load_2d(sK + c * C::F_ATOM, &tm_kv, kv_full, hr + head * D + c * 64, tok0 + kt * TKEY);
        tma_load_2d(sV + c * C::F_ATOM, &tm_kv, kv_full, 2 * hr + head * D + c * 64, tok0 + kt * TKEY);
      }
    }
    for (int ii = 0; ii < NI; ++ii) {
      const int i = i0 + ii, st = ii % ST;
      mbar_wait(&q_empty[st], ((ii / ST) & 1) ^ 1);
      if (lane == 0) {
        const uint32_t lbytes = (uint32_t)min(TQH, s - i * TQH) * 4;
        mbar_expect_tx(&q_full[st], 2 * C::QH_BYTES + 2 * lbytes);
        for (int c = 0; c < NA; ++c) {
          tma_load_2d(stQ(st) + c * C::H_ATOM, &tm_q, &q_full[st], head * D + c * 64, tok0 + i * TQH);
          tma_load_2d(stO(st) + c * C::H_ATOM, &tm_o, &q_full[st], head * D + c * 64, tok0 + i * TQH);
        }
        bulk_load_1d(stL(st), a.lse + srow + i * TQH, lbytes, &q_full[st]);
        bulk_load_1d(stD(st), a.delta + srow + i * TQH, lbytes, &q_full[st]);
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc_s = idesc_bf16(TKEY, TQH, false, false);  // K Q^T, V dO^T
    constexpr uint32_t idesc_g = idesc_bf16(TKEY, D, false, true);     // P^T dO, dS^T Q
    constexpr uint32_t idesc_q = idesc_bf16(128, TQH, true, true);     // K^T dS^T (M = d padded)
    unsigned long long *dbg = (a.dbg && lane == 0) ? a.dbg + (size_t)blockIdx.x * DBG_STRIDE : nullptr;
    if (dbg) { dbg[0] = clock64(); dbg[76] = globaltimer(); dbg[77] = NI; unsigned sm; asm volatile("mov.u32 %0, %%smid;" : "=r"(sm)); dbg[79] = sm; }
    mbar_wait(kv_full, 0);
    if (dbg) dbg[1] = clock64();
    const uint32_t k0 = smem_u32(sK), v0 = smem_u32(sV);
    // whole-warp issue (tc_*_w elect one lane inside the asm); descriptors are base + constant offsets
    const uint64_t dK0 = sdesc_sw128(k0, 16, 1024), dV0 = sdesc_sw128(v0, 16, 1024);
    const uint64_t dKmn = sdesc_sw128(k0, C::F_ATOM, 1024);
    auto scores = [&](int ii) {
      const int st = ii % ST, b = ii % NB, w = ii & 1;
      mbar_wait(&q_full[st], (ii / ST) & 1);
      if (dbg && ii < 36) dbg[2 + ii] = clock64();
      tc_fence_after();
      const uint64_t dQ0 = sdesc_sw128(smem_u32(stQ(st)), 16, 1024), dO0 = sdesc_sw128(smem_u32(stO(st)), 16, 1024);
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const uint32_t fo = ((kk >> 2) * C::F_ATOM + (kk & 3) * 32) >> 4, ho = ((kk >> 2) * C::H_ATOM + (kk & 3) * 32) >> 4;
        tc_mma_f16_w(tmem + C::SP0 + 64 * b, dK0 + fo, dQ0 + ho, idesc_s, kk > 0 ? 1u : 0u);
        tc_mma_f16_w(tmem + C::DP0 + 64 * b, dV0 + fo, dO0 + ho, idesc_s, kk > 0 ? 1u : 0u);
      }
      tc_commit_w(&s_full[w]);
    };
    auto grads = [&](int p) {
      const int st = p % ST, b = p % NB, w = p & 1;
      mbar_wait(&p_full[w], (p >> 1) & 1);  // P^T in TMEM, dS^T in smem
      if (dbg && p < 36) dbg[38 + p] = clock64();
      tc_fence_after();
      const uint64_t qmn = sdesc_sw128(smem_u32(stQ(st)), C::H_ATOM, 1024);
      const uint64_t omn = sdesc_sw128(smem_u32(stO(st)), C::H_ATOM, 1024);
      const uint64_t dsmn = sdesc_sw128(smem_u32(sDS + w * C::DS_BYTES), C::F_ATOM, 1024);
#pragma unroll
      for (int kk = 0; kk < TQH / 16; ++kk) {
        const uint32_t acc = (p > 0 || kk > 0) ? 1u : 0u;
        tc_mma_f16_ts_w(tmem + C::DV, tmem + C::SP0 + 64 * b + kk * 8, omn + (kk * 2048 >> 4), idesc_g, acc);
        tc_mma_f16_ts_w(tmem + C::DK, tmem + C::DP0 + 64 * b + kk * 8, qmn + (kk * 2048 >> 4), idesc_g, acc);
      }
      if (dbg && !(p & 1) && p < 32) dbg[144 + (p >> 1)] = clock64();
      if (p >= 1) mbar_wait(dq_free, (p - 1) & 1);  // the drain warps have read dQ^T of p - 1
      if (dbg && !(p & 1) && p < 32) dbg[160 + (p >> 1)] = clock64();
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < TKEY / 16; ++kk)
        tc_mma_f16_w(tmem + C::DQT, dKmn + (kk * 2048 >> 4), dsmn + (kk * 2048 >> 4), idesc_q, kk > 0 ? 1u : 0u);
      tc_commit_w(dq_full);
      tc_commit_w(&ds_free[w]);
      tc_commit_w(&q_empty[st]);
      if (dbg && !(p & 1) && p < 32) dbg[112 + (p >> 1)] = clock64();
    };
    for (int ii = 0; ii <= NI; ++ii) {
      if (NB == 1) {  // one buffer: P^T of ii - 1 must be consumed before S^T of ii overwrites it
        if (ii >= 1) grads(ii - 1);
        if (ii < NI) scores(ii);
      } else {
        if (ii < NI) scores(ii);
        if (ii >= 1) grads(ii - 1);
      }
    }
    tc_commit_w(kv_done);
    if (dbg) { dbg[74] = clock64(); }
  } else if (warp < 10) {
    // ------------------------------------------------------------ element-wise (thread = key row)
    const int g = (warp - 2) >> 2, q4 = warp & 3, r = q4 * 32 + lane, kj = kt * TKEY + r;
    const uint32_t lb = tmem + ((uint32_t)(q4 * 32) << 16);
    const float scale = 1.f / sqrtf((float)D), sl2 = 1.4426950408889634f * scale;
    for (int ii = g; ii < NI; ii += 2) {
      const int st = ii % ST, b = ii % NB, qi0 = (i0 + ii) * TQH;  // warpgroup g == ii & 1
      mbar_wait(&q_full[st], (ii / ST) & 1);  // lse / delta of this half-block
      mbar_wait(&s_full[g], (ii >> 1) & 1);
      unsigned long long *dbe = (a.dbg && warp == 2 && lane == 0 && ii < 32) ? a.dbg + (size_t)blockIdx.x * DBG_STRIDE : nullptr;
      if (dbe) dbe[96 + (ii >> 1)] = clock64();
      tc_fence_after();
      const bool mask = (qi0 < kt * TKEY + TKEY - 1) || (qi0 + TQH > s);
      const float *L = stL(st), *Dl = stD(st);
      mbar_wait(&ds_free[g], ((ii >> 1) & 1) ^ 1);  // dS^T buffer g read by the MMAs of ii - 2
      uint8_t *row = sDS + g * C::DS_BYTES + r * 128;
      // 16 query columns per step; the TMEM loads of step c + 1 are in flight while step c computes
      uint32_t sv[2][16], dv[2][16];
      tmem_ld16b(lb + C::SP0 + 64 * b, sv[0]);
      tmem_ld16b(lb + C::DP0 + 64 * b, dv[0]);
      tmem_ld_wait();
#pragma unroll
      for (int c = 0; c < TQH / 16; ++c) {
        const int cb = c & 1;
        if (c + 1 < TQH / 16) {
          tmem_ld16b(lb + C::SP0 + 64 * b + 16 * (c + 1), sv[cb ^ 1]);
          tmem_ld16b(lb + C::DP0 + 64 * b + 16 * (c + 1), dv[cb ^ 1]);
        }
        uint32_t pw[8], dw[8];
#pragma unroll
        for (int k = 0; k < 16; k += 2) {
          const int col = 16 * c + k, qi = qi0 + col;
          const float2 l2 = *reinterpret_cast<const float2 *>(L + col);
          const float2 d2 = *reinterpret_cast<const float2 *>(Dl + col);
          float p0 = fast_exp2(fmaf(__uint_as_float(sv[cb][k]), sl2, -l2.x));
          float p1 = fast_exp2(fmaf(__uint_as_float(sv[cb][k + 1]), sl2, -l2.y));
          if (mask) {
            if (!(kj <= qi && qi < s)) p0 = 0.f;
            if (!(kj <= qi + 1 && qi + 1 < s)) p1 = 0.f;
          }
          pw[k >> 1] = pack_bf16(p0, p1);
          dw[k >> 1] = pack_bf16(p0 * (__uint_as_float(dv[cb][k]) - d2.x), p1 * (__uint_as_float(dv[cb][k + 1]) - d2.y));
        }
        // P^T (bf16 pairs) over columns 8c..8c+7 of this buffer's S^T (already read): the A operand of dV
        tmem_st8(lb + C::SP0 + 64 * b + 8 * c, pw);
        // dS^T likewise over columns 8c..8c+7 of dP^T (already read): the A operand of dK
        tmem_st8(lb + C::DP0 + 64 * b + 8 * c, dw);
        // dS^T: 16-B chunks 2c, 2c+1 of this key row (128-B swizzle)
        *reinterpret_cast<uint4 *>(row + (((2 * c) ^ (r & 7)) << 4)) = make_uint4(dw[0], dw[1], dw[2], dw[3]);
        *reinterpret_cast<uint4 *>(row + (((2 * c + 1) ^ (r & 7)) << 4)) = make_uint4(dw[4], dw[5], dw[6], dw[7]);
        if (c + 1 < TQH / 16) tmem_ld_wait();
      }
      tmem_st_wait();
      fence_proxy_async();
      tc_fence_before();
      __syncwarp();
      if (dbe) dbe[128 + (ii >> 1)] = clock64();
      if (lane == 0) mbar_arrive(&p_full[g]);
    }
    // dK, dV epilogue
    mbar_wait(kv_done, 0);
    tc_fence_after();
    unsigned long long *dbg = (a.dbg && warp == 2 && lane == 0 && NI <= 32) ? a.dbg + (size_t)blockIdx.x * DBG_STRIDE : nullptr;
    if (dbg) dbg[70] = clock64();
    // TMEM -> bf16 rows in smem (K / V / stage-ring space, free once every MMA completed; padded rows: the
    // row-per-thread 16-B writes are bank-conflict free), then coalesced 16-B global stores of whole rows.
    constexpr int SROW = 2 * D + 16, CPR = D / 8;  // staging row bytes, 16-B chunks per row
    static_assert(2 * TKEY * SROW <= 2 * C::KV_BYTES + ST * C::STAGE_BYTES, "dK/dV staging");
    uint8_t *stgK = sK, *stgV = sK + TKEY * SROW;
#pragma unroll
    for (int c = 0; c < D / 16; ++c) {
      if ((c & 1) != g) continue;  // warp-uniform: alternate 16-column chunks per warpgroup
      uint32_t ov[16], ok[16];
      tmem_ld16b(lb + C::DV + c * 16, ov);
      tmem_ld16b(lb + C::DK + c * 16, ok);
      tmem_ld_wait();
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        uint4 u;
        u.x = pack_bf16(__uint_as_float(ov[8 * hh + 0]), __uint_as_float(ov[8 * hh + 1]));
        u.y = pack_bf16(__uint_as_float(ov[8 * hh + 2]), __uint_as_float(ov[8 * hh + 3]));
        u.z = pack_bf16(__uint_as_float(ov[8 * hh + 4]), __uint_as_float(ov[8 * hh + 5]));
        u.w = pack_bf16(__uint_as_float(ov[8 * hh + 6]), __uint_as_float(ov[8 * hh + 7]));
        *reinterpret_cast<uint4 *>(stgV + r * SROW + c * 32 + 16 * hh) = u;
        u.x = pack_bf16(__uint_as_float(ok[8 * hh + 0]) * scale, __uint_as_float(ok[8 * hh + 1]) * scale);
        u.y = pack_bf16(__uint_as_float(ok[8 * hh + 2]) * scale, __uint_as_float(ok[8 * hh + 3]) * scale);
        u.z = pack_bf16(__uint_as_float(ok[8 * hh + 4]) * scale, __uint_as_float(ok[8 * hh + 5]) * scale);
        u.w = pack_bf16(__uint_as_float(ok[8 * hh + 6]) * scale, __uint_as_float(ok[8 * hh + 7]) * scale);
        *reinterpret_cast<uint4 *>(stgK + r * SROW + c * 32 + 16 * hh) = u;
      }
    }
    asm volatile("bar.sync 3, 256;" ::: "memory");  // the 8 element-wise warps
    const int et = (warp - 2) * 32 + lane;
    __nv_bfloat16 *dk0 = reinterpret_cast<__nv_bfloat16 *>(a.dqkv) + (size_t)(tok0 + kt * TKEY) * 3 * hr + hr + head * D;
    const int nrows = min(TKEY, s - kt * TKEY);
    for (int idx = et; idx < 2 * TKEY * CPR; idx += 256) {
      const int t = idx / (TKEY * CPR), rem = idx - t * TKEY * CPR, rr = rem / CPR, ch = rem - rr * CPR;
      if (rr < nrows)
        *reinterpret_cast<uint4 *>(dk0 + (size_t)rr * 3 * hr + t * hr + ch * 8) =
            *reinterpret_cast<const uint4 *>((t ? stgV : stgK) + rr * SROW + ch * 16);
    }
    if (dbg) dbg[71] = clock64();
  } else if (warp < 14) {
    // ------------------------------------------------------------ dQ drain (thread = d index)
    // Per half-block: dQ_i^T TMEM -> registers (64 columns), release the TMEM buffer to the MMA warp at once,
    // then the registers -> fp32 staging smem once the bulk warp has finished reading the previous block.
    // The MMA warp therefore waits only for the TMEM read, never for the dQ ordering or the L2 operations.
    const int q4 = warp & 3, dd = q4 * 32 + lane;
    const bool active = q4 * 32 < D;  // warp-uniform
    const uint32_t lb = tmem + ((uint32_t)(q4 * 32) << 16);
    for (int ii = 0; ii < NI; ++ii) {
      mbar_wait(dq_full, ii & 1);
      if (a.dbg && warp == 10 && lane == 0 && ii + 1 == NI) a.dbg[(size_t)blockIdx.x * DBG_STRIDE + 88] = clock64();
      tc_fence_after();
      uint32_t v[2][32];
      if (active) {
        tmem_ld32(lb + C::DQT, v[0]);
        tmem_ld32(lb + C::DQT + 32, v[1]);
        tmem_ld_wait();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(dq_free);  // dQ^T read: the next dQ^T MMA may overwrite it
#pragma unroll
      for (int h = 0; h < 2; ++h) {  // rows 32h .. 32h + 31 of the staging buffer, each half handed over alone
        if (ii >= 1) mbar_wait(&stg_free[h * 2 + ((ii - 1) & 1)], ((ii - 1) >> 1) & 1);  // block ii - 1 read it
        if (active && dd < D) {
#pragma unroll
          for (int q = 0; q < 32; ++q) sStg[(32 * h + q) * D + dd] = __uint_as_float(v[h][q]);
        }
        fence_proxy_async();  // generic smem writes -> visible to the bulk copy (async proxy)
        __syncwarp();
        if (lane == 0) mbar_arrive(&stg_full[h * 2 + (ii & 1)]);
      }
    }
  } else if (lane == 0) {
    // ------------------------------------------------------------ dQ bulk threads (warps 14, 15: lane 0)
    // Thread k takes the blocks ii = k mod 2: waits for its turn on the block's counter, bulk-stores (first
    // contributor) or bulk-reduce-adds (cp.reduce.async.bulk, performed in L2) the staged block into dq_acc,
    // frees the staging buffer once the operation has read it, and releases the counter as soon as the
    // operation has completed -- the completion latency of one block overlaps the other thread's next block.
    const int k = warp - 14;
    float *dqa = a.dq_acc + srow * D;
    int *sem = a.dq_sem + ((size_t)bi * H + head) * NQ;
    for (int ii = k; ii < NI; ii += 2) {
      const int i = i0 + ii, nrow = min(TQH, s - i * TQH);
      const int rank = i / 2 - kt;  // contributions before this one (key tiles floor(i/2) .. kt+1)
      unsigned long long *dbl = (a.dbg && ii + 2 >= NI) ? a.dbg + (size_t)blockIdx.x * DBG_STRIDE + 80 + 4 * k : nullptr;
      if (dbl) dbl[0] = clock64();
      if (rank > 0) {  // the turn does not depend on the staging: wait for it first
        const uint64_t t0 = globaltimer();
        int seen;
        while ((seen = (int)ld_acquire_gpu(&sem[i])) != rank) {
          __nanosleep(20);
          if (globaltimer() - t0 > 4000000000ull) {  // 4 s: a broken ordering invariant, not a slow peer
            printf("attn_bwd dQ order watchdog: b %d head %d kt %d block %d rank %d counter %d\n", bi, head, kt, i,
                   rank, seen);
            __trap();
          }
        }
        fence_proxy_async_global();
      }
      if (dbl) dbl[1] = clock64();
      float *qa = dqa + (size_t)i * TQH * D;
#pragma unroll
      // both halves in flight: half 1 is issued as soon as it is staged, before half 0 has been read
      auto issue = [&](int h) {
        const int rows = min(32, nrow - 32 * h);
        if (rows > 0) {
          if (rank == 0)
            bulk_store(qa + 32 * h * D, sStg + 32 * h * D, (uint32_t)rows * D * 4);
          else
            bulk_reduce_add_f32(qa + 32 * h * D, sStg + 32 * h * D, (uint32_t)rows * D * 4);
        }
        tma_store_commit();  // (an empty group when the half has no rows)
      };
      mbar_wait(&stg_full[k], (ii >> 1) & 1);
      issue(0);
      mbar_wait(&stg_full[2 + k], (ii >> 1) & 1);
      issue(1);
      tma_store_wait_read<1>();  // half 0 read
      mbar_arrive(&stg_free[k]);
      tma_store_wait_read<0>();  // half 1 read
      mbar_arrive(&stg_free[2 + k]);
      if (dbl) dbl[2] = clock64();
      tma_store_wait<0>();  // both halves have completed: the next contributor may go
      if (dbl) dbl[3] = clock64();
      fence_proxy_async_global();
      st_release_gpu(&sem[i], (uint32_t)(rank + 1));
    }
    if (a.dbg && NI <= 32) a.dbg[(size_t)blockIdx.x * DBG_STRIDE + 72 + k] = clock64();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
    if (a.dbg && lane == 0) { a.dbg[(size_t)blockIdx.x * DBG_STRIDE + 75] = clock64(); a.dbg[(size_t)blockIdx.x * DBG_STRIDE + 78] = globaltimer(); }
  }
}

// ------------------------------------------------------------------------------------------ delta
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

// dQ = bf16(scale * dq_acc) into the q block of dqkv (one thread per 8 consecutive d), and every dQ ordering
// counter back to 0 for the next launch.
template <int D>
__global__ void __launch_bounds__(256) attn_dq_out_kernel(AttnArgs a) {
  const int H = a.heads, hr = H * D, s = a.s;
  const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long nsem = (long)a.b * H * ((s + TQH - 1) / TQH);
  if (idx < nsem) a.dq_sem[idx] = 0;
  if (idx >= (long)a.b * H * s * (D / 8)) return;
  const int c8 = (int)(idx % (D / 8));
  const long row = idx / (D / 8);  // (bi * H + head) * s + q
  const int q = (int)(row % s), bh = (int)(row / s), head = bh % H, bi = bh / H;
  const float scale = 1.f / sqrtf((float)D);
  const float4 *src = reinterpret_cast<const float4 *>(a.dq_acc + row * D + c8 * 8);
  const float4 x0 = __ldcs(src), x1 = __ldcs(src + 1);
  uint4 o;
  o.x = pack_bf16(x0.x * scale, x0.y * scale);
  o.y = pack_bf16(x0.z * scale, x0.w * scale);
  o.z = pack_bf16(x1.x * scale, x1.y * scale);
  o.w = pack_bf16(x1.z * scale, x1.w * scale);
  *reinterpret_cast<uint4 *>(reinterpret_cast<__nv_bfloat16 *>(a.dqkv) + ((size_t)bi * s + q) * 3 * hr + head * D +
                             c8 * 8) = o;
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

size_t attn_bwd_ws_floats(int b, int s, int heads, int d) {
  const size_t nq = (size_t)(s + TQH - 1) / TQH;
  return (size_t)b * heads * s * (1 + (size_t)d) + (size_t)b * heads * nq;
}

template <int D>
static cudaError_t bwd_tc_d(const AttnArgs &a, cudaStream_t st) {
  using C = BwdCfg<D>;
  static bool attr[MAX_DEV] = {};
  const int dev = cur_device();
  if (!attr[dev]) {
    cudaError_t e = cudaFuncSetAttribute(attn_bwd_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr[dev] = true;
  }
  if (!a.dq_acc || !a.dq_sem || !a.delta) return cudaErrorInvalidValue;
  const int tokens = a.b * a.s, hr = a.heads * D;
  CUtensorMap m_kv, m_q, m_o;
  if (!make_rows_map(&m_kv, a.qkv, tokens, 3 * hr, 3 * hr, TKEY) ||
      !make_rows_map(&m_q, a.qkv, tokens, 3 * hr, 3 * hr, TQH) || !make_rows_map(&m_o, a.dctx, tokens, hr, hr, TQH))
    return cudaErrorInvalidValue;
  const long nd = (long)tokens * a.heads;
  attn_delta_kernel<D><<<(unsigned)((nd + 255) / 256), 256, 0, st>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  AttnArgs ag = a;
  if (ag.attn_group <= 0) {
    static int g_env = -1;
    if (g_env < 0) {
      const char *e = getenv("MERAK_ATTN_BWD_GROUP");
      g_env = e ? atoi(e) : 0;
    }
    ag.attn_group = g_env > 0 ? g_env : 64;  // measured: 64 >= 32 > 16 > 8 at the gpt shapes
  }
  if (ag.attn_group > a.b * a.heads) ag.attn_group = a.b * a.heads;
  const int grid = a.b * a.heads * ((a.s + TKEY - 1) / TKEY);
  attn_bwd_tc_kernel<D><<<grid, NTHR, C::SMEM, st>>>(m_kv, m_q, m_o, ag);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const long nq = (long)a.b * a.heads * a.s * (D / 8);
  attn_dq_out_kernel<D><<<(unsigned)((nq + 255) / 256), 256, 0, st>>>(ag);
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
  if (e == cudaSuccess) e = touch_kernel((const void *)attn_dq_out_kernel<D>);
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
