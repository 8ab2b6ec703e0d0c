// attention_tc.cu -- causal attention forward on the 5th-generation tensor cores (tcgen05 / TMEM).
//
// per (sample, local head e): S = Q_e K_e^T / sqrt(d), causal mask (reading R4),
// P = softmax(S), ctx = P V_e; lse2 = log2 sum exp2(S * scale * log2e) saved for the backward.
//
// One CTA = one 128-row query tile of one (sample, head); 192 threads; two CTAs per SM for d <= 64.
//   warp 0    TMA producer: Q once, then 64-key half tiles K_j / V_j through a 3-stage ring
//   warp 1    TMEM owner + MMA issuer: S_j = Q K_j^T into one of two TMEM S buffers, then
//             O += P_{j-1} V_{j-1} into the TMEM output accumulator (S_{j+1} is queued before
//             P_j V_j, so the tensor core works while the softmax warps run)
//   warps 2-5 softmax, thread = query row (= TMEM lane): S_j row -> registers, exp2, row sum, bf16
//             P_j into a 128-B-swizzled smem tile (double-buffered) for the next MMA.
// The running max is updated lazily (only when it grows by more than 2^8, as in FlashAttention-4):
// then O (in TMEM) is rescaled in place after P_{j-1} V_{j-1} completed; otherwise probabilities
// are taken relative to the stale max (<= 2^8, exact after the final 1 / l).
// Operands: Q, K K-major; V MN-major (its rows are keys); P K-major in smem.
#include <math.h>

#include "kernels.h"
#include "ptx.cuh"

namespace mk {

namespace {

constexpr int TQ = 128;   // query rows per CTA (TMEM lanes)
constexpr int TKH = 64;   // keys per half tile

template <int D>
struct FaCfg {
  static constexpr int NA = (D + 63) / 64;          // 64-wide swizzle atoms along d
  static constexpr int Q_ATOM = TQ * 128;           // [128 rows][64] bf16
  static constexpr int H_ATOM = TKH * 128;          // [64 rows][64] bf16
  static constexpr int Q_BYTES = NA * Q_ATOM;
  static constexpr int K_BYTES = NA * H_ATOM;       // K-major [64 keys][d]
  static constexpr int V_BYTES = NA * H_ATOM;       // MN-major: NA chunks of [64 keys][64 d-columns]
  static constexpr int STAGES = (D <= 64) ? 3 : 2;  // 4 stages no longer fit two CTAs per SM
  static constexpr int P_BYTES = TQ * 128;          // [128 q][64 keys] bf16 = one atom
  static constexpr int XCH_BYTES = (2 * 2 * TQ + 2 * TQ) * 4;  // row partial max [2][2][128], row sum [2][128]
  static constexpr int SMEM = Q_BYTES + STAGES * (K_BYTES + V_BYTES) + 2 * P_BYTES + XCH_BYTES + 1024 + 256;
  static constexpr uint32_t S_COL = 0;              // 2 x 64 fp32 columns
  static constexpr uint32_t O_COL = 128;            // D fp32 columns
  static constexpr int TMEM_COLS = (128 + D <= 256) ? 256 : 512;
  static constexpr int MIN_CTAS = (D <= 64) ? 2 : 1;
};

MK_DEV void tmem_ld16(uint32_t taddr, uint32_t *r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
MK_DEV void tmem_st16(uint32_t taddr, const uint32_t *r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

}  // namespace

// 320 threads: warp 0 TMA, warp 1 TMEM + MMA, warps 2-9 softmax (thread = query row; the two warpgroups
// split each 64-key tile's columns and exchange the row max through shared memory)
template <int D>
__global__ void __launch_bounds__(320, FaCfg<D>::MIN_CTAS)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tmq, const __grid_constant__ CUtensorMap tmkv, AttnArgs a) {
  using C = FaCfg<D>;
  constexpr int NA = C::NA, ST = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sQ = smem;
  uint8_t *sK = sQ + C::Q_BYTES;                 // [ST][K_BYTES]
  uint8_t *sV = sK + ST * C::K_BYTES;            // [ST][V_BYTES]
  uint8_t *sP = sV + ST * C::V_BYTES;            // [2][P_BYTES]
  float *xmax = reinterpret_cast<float *>(sP + 2 * C::P_BYTES);  // [2 (tile parity)][2 (warpgroup)][128]
  float *xsum = xmax + 4 * TQ;                                    // [2 (warpgroup)][128]
  uint64_t *bar = reinterpret_cast<uint64_t *>(sP + 2 * C::P_BYTES + C::XCH_BYTES);
  uint64_t *q_full = bar;
  uint64_t *kv_full = bar + 1, *kv_empty = bar + 1 + ST;
  uint64_t *s_full = bar + 1 + 2 * ST, *s_free = s_full + 2, *p_full = s_full + 4, *p_free = s_full + 6;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(s_full + 8);

  const int s = a.s, H = a.heads;
  const int nqt = (s + TQ - 1) / TQ;
  const int qt = nqt - 1 - blockIdx.z;  // grid (heads, b, tiles): globally heaviest tiles first
  const int head = blockIdx.x, bi = blockIdx.y;
  const int hr = H * D;
  const int tok0 = bi * s;
  const int J = min(2 * (qt + 1), (s + TKH - 1) / TKH);  // causal: keys < (qt+1)*128, and < s
  const int warp = warp_id(), lane = lane_id();

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmq);
    tma_prefetch(&tmkv);
    mbar_init(q_full, 1);
    for (int i = 0; i < ST; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 8);
      mbar_init(&p_full[i], 8);
      mbar_init(&p_free[i], 1);
    }
    fence_mbar_init();
    fence_proxy_async();
  }
  if (warp == 1) tmem_alloc<C::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      mbar_expect_tx(q_full, C::Q_BYTES);
      for (int c = 0; c < NA; ++c) tma_load_2d(sQ + c * C::Q_ATOM, &tmq, q_full, head * D + c * 64, tok0 + qt * TQ);
    }
    for (int j = 0; j < J; ++j) {
      const int st = j % ST;
      mbar_wait(&kv_empty[st], ((j / ST) & 1) ^ 1);
      if (lane == 0) {
        mbar_expect_tx(&kv_full[st], C::K_BYTES + C::V_BYTES);
        for (int c = 0; c < NA; ++c) {
          tma_load_2d(sK + st * C::K_BYTES + c * C::H_ATOM, &tmkv, &kv_full[st], hr + head * D + c * 64,
                      tok0 + j * TKH);
          tma_load_2d(sV + st * C::V_BYTES + c * C::H_ATOM, &tmkv, &kv_full[st], 2 * hr + head * D + c * 64,
                      tok0 + j * TKH);
        }
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc_s = idesc_bf16(TQ, TKH, false, false);  // Q K^T: both K-major
    constexpr uint32_t idesc_o = idesc_bf16(TQ, D, false, true);     // P V: V is MN-major
    mbar_wait(q_full, 0);
    for (int j = 0; j <= J; ++j) {
      if (j < J) {
        const int st = j % ST, b = j & 1;
        mbar_wait(&kv_full[st], (j / ST) & 1);
        mbar_wait(&s_free[b], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t q0 = smem_u32(sQ), k0 = smem_u32(sK + st * C::K_BYTES);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            tc_mma_f16(tmem + C::S_COL + b * TKH, sdesc_sw128(q0 + (kk >> 2) * C::Q_ATOM + (kk & 3) * 32, 16, 1024),
                       sdesc_sw128(k0 + (kk >> 2) * C::H_ATOM + (kk & 3) * 32, 16, 1024), idesc_s, kk > 0 ? 1u : 0u);
          }
          tc_commit(&s_full[b]);
        }
        __syncwarp();
      }
      if (j >= 1) {
        const int i = j - 1, st = i % ST, pb = i & 1;
        mbar_wait(&p_full[pb], (i >> 1) & 1);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t p0 = smem_u32(sP + pb * C::P_BYTES), v0 = smem_u32(sV + st * C::V_BYTES);
#pragma unroll
          for (int kk = 0; kk < TKH / 16; ++kk) {
            tc_mma_f16(tmem + C::O_COL, sdesc_sw128(p0 + kk * 32, 16, 1024),
                       sdesc_sw128(v0 + kk * 2048, C::H_ATOM, 1024), idesc_o, (i > 0 || kk > 0) ? 1u : 0u);
          }
          tc_commit(&p_free[pb]);
          tc_commit(&kv_empty[st]);
        }
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------------------ softmax (thread = row, half the columns)
    const int q = warp & 3, cw = (warp - 2) >> 2;
    const int r = q * 32 + lane;
    const int qi = qt * TQ + r;
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    const float sl2 = 1.4426950408889634f / sqrtf((float)D);
    const float thr = 8.0f / sl2;  // lazy rescale threshold (2^8) in raw score units
    float m = -INFINITY, l = 0.f;  // m is identical in both warpgroups; l is this warpgroup's partial
    for (int j = 0; j < J; ++j) {
      const int b = j & 1;
      mbar_wait(&s_full[b], (j >> 1) & 1);
      tc_fence_after();
      uint32_t v[32];
      tmem_ld32(lane_base + C::S_COL + b * TKH + cw * 32, v);
      tmem_ld_wait();
      const int kj0 = j * TKH + cw * 32;  // this warpgroup's first key
      const bool mask = (j * TKH + TKH - 1 > qt * TQ) || (j * TKH + TKH > s);
      float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};  // 4 independent chains
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const float x = __uint_as_float(v[k]);
        if (!mask || (kj0 + k <= qi && kj0 + k < s)) mx4[k & 3] = fmaxf(mx4[k & 3], x);
      }
      const float pmx = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
      xmax[(b * 2 + cw) * TQ + r] = pmx;
      asm volatile("bar.sync 1, 256;" ::: "memory");  // the 8 softmax warps
      const float mx = fmaxf(pmx, xmax[(b * 2 + (cw ^ 1)) * TQ + r]);
      // the max grew by more than 2^8: move to the new max, rescale O and l.  TMEM access is
      // warp-collective, so the whole warp enters when any row needs it (others scale by 1); the two
      // warpgroups rescale alternate 16-column chunks of O.
      const bool need = mx > m + thr;
      if (__any_sync(0xffffffffu, need)) {
        const float corr = need ? fast_exp2((m - mx) * sl2) : 1.f;
        if (j >= 1) {
          const int pi = j - 1;
          mbar_wait(&p_free[pi & 1], (pi >> 1) & 1);  // P_{j-1} V_{j-1} has landed in O
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < D / 16; ++c) {
            if ((c & 1) != cw) continue;
            uint32_t o[16];
            tmem_ld16(lane_base + C::O_COL + c * 16, o);
            tmem_ld_wait();
#pragma unroll
            for (int k = 0; k < 16; ++k) o[k] = __float_as_uint(__uint_as_float(o[k]) * corr);
            tmem_st16(lane_base + C::O_COL + c * 16, o);
          }
          tmem_st_wait();
        }
        if (need) {
          l *= corr;
          m = mx;
        }
      }
      // P buffer b was last read by P_{j-2} V_{j-2}
      mbar_wait(&p_free[b], ((j >> 1) & 1) ^ 1);
      const float ms = m * sl2;
      float rs4[4] = {0.f, 0.f, 0.f, 0.f};
      uint8_t *prow = sP + b * C::P_BYTES + r * 128;
#pragma unroll
      for (int c4 = 0; c4 < 4; ++c4) {
        const int ch = cw * 4 + c4;  // 16-B chunk of the 128-B P row
        uint32_t pk[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k = c4 * 8 + u * 2;
          float p0 = fast_exp2(fmaf(__uint_as_float(v[k]), sl2, -ms));
          float p1 = fast_exp2(fmaf(__uint_as_float(v[k + 1]), sl2, -ms));
          if (mask) {
            if (!(kj0 + k <= qi && kj0 + k < s)) p0 = 0.f;
            if (!(kj0 + k + 1 <= qi && kj0 + k + 1 < s)) p1 = 0.f;
          }
          rs4[u] += p0 + p1;
          pk[u] = pack_bf16(p0, p1);
        }
        *reinterpret_cast<uint4 *>(prow + ((ch ^ (r & 7)) << 4)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
      }
      l += (rs4[0] + rs4[1]) + (rs4[2] + rs4[3]);
      fence_proxy_async();  // generic-proxy P stores -> visible to the tensor core
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&s_free[b]);
        mbar_arrive(&p_full[b]);
      }
    }
    // row sum: the two warpgroups' partials, added in a fixed order
    xsum[cw * TQ + r] = l;
    asm volatile("bar.sync 1, 256;" ::: "memory");
    const float lt = xsum[r] + xsum[TQ + r];
    // the last P V has completed when its commit arrived on p_free
    const int last = J - 1;
    mbar_wait(&p_free[last & 1], (last >> 1) & 1);
    tc_fence_after();
    // tcgen05.ld is warp-collective (.sync.aligned): load converged, store only rows < s
    const float inv = 1.f / lt;
    __nv_bfloat16 *dst = reinterpret_cast<__nv_bfloat16 *>(a.ctx) + (size_t)(tok0 + qi) * a.ld_ctx + head * D;
#pragma unroll
    for (int c = 0; c < D / 16; ++c) {
      if ((c & 1) != cw) continue;
      uint32_t o[16];
      tmem_ld16(lane_base + C::O_COL + c * 16, o);
      tmem_ld_wait();
      if (qi < s) {
        uint4 u0, u1;
        u0.x = pack_bf16(__uint_as_float(o[0]) * inv, __uint_as_float(o[1]) * inv);
        u0.y = pack_bf16(__uint_as_float(o[2]) * inv, __uint_as_float(o[3]) * inv);
        u0.z = pack_bf16(__uint_as_float(o[4]) * inv, __uint_as_float(o[5]) * inv);
        u0.w = pack_bf16(__uint_as_float(o[6]) * inv, __uint_as_float(o[7]) * inv);
        u1.x = pack_bf16(__uint_as_float(o[8]) * inv, __uint_as_float(o[9]) * inv);
        u1.y = pack_bf16(__uint_as_float(o[10]) * inv, __uint_as_float(o[11]) * inv);
        u1.z = pack_bf16(__uint_as_float(o[12]) * inv, __uint_as_float(o[13]) * inv);
        u1.w = pack_bf16(__uint_as_float(o[14]) * inv, __uint_as_float(o[15]) * inv);
        *reinterpret_cast<uint4 *>(dst + c * 16) = u0;
        *reinterpret_cast<uint4 *>(dst + c * 16 + 8) = u1;
      }
    }
    if (cw == 0 && qi < s) a.lse[((size_t)bi * H + head) * s + qi] = m * sl2 + log2f(lt);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::TMEM_COLS>(tmem);
  }
}

// ------------------------------------------------------------------------------------------ host
typedef CUresult (*EncodeTiledFn2)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                   const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static bool make_qkv_map(CUtensorMap *m, const void *qkv, int tokens, int cols, int box_rows) {
  static EncodeTiledFn2 enc = nullptr;
  if (!enc) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return false;
    enc = reinterpret_cast<EncodeTiledFn2>(p);
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)tokens};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64u, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1u, 1u};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(qkv), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int D>
static cudaError_t fwd_tc_d(const AttnArgs &a, cudaStream_t st) {
  using C = FaCfg<D>;
  static bool attr[MAX_DEV] = {};
  const int dev = cur_device();
  if (!attr[dev]) {
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr[dev] = true;
  }
  CUtensorMap mq, mkv;
  if (!make_qkv_map(&mq, a.qkv, a.b * a.s, 3 * a.heads * D, TQ) ||
      !make_qkv_map(&mkv, a.qkv, a.b * a.s, 3 * a.heads * D, TKH))
    return cudaErrorInvalidValue;
  dim3 grid(a.heads, a.b, (a.s + TQ - 1) / TQ);
  attn_fwd_tc_kernel<D><<<grid, 320, C::SMEM, st>>>(mq, mkv, a);
  return cudaGetLastError();
}

cudaError_t attn_fwd(const AttnArgs &a, cudaStream_t st) {
  switch (a.d) {
    case 32: return fwd_tc_d<32>(a, st);
    case 64: return fwd_tc_d<64>(a, st);
    case 80: return fwd_tc_d<80>(a, st);
    case 96: return fwd_tc_d<96>(a, st);
    case 128: return fwd_tc_d<128>(a, st);
  }
  return cudaErrorNotSupported;
}

template <int D>
cudaError_t attn_preload_d() {
  cudaError_t e = touch_kernel((const void *)attn_fwd_tc_kernel<D>);
  return e != cudaSuccess ? e : attn_bwd_preload_d(D);
}

cudaError_t attn_preload(int d) {
  switch (d) {
    case 32: return attn_preload_d<32>();
    case 64: return attn_preload_d<64>();
    case 80: return attn_preload_d<80>();
    case 96: return attn_preload_d<96>();
    case 128: return attn_preload_d<128>();
  }
  return cudaErrorNotSupported;
}

}  // namespace mk
