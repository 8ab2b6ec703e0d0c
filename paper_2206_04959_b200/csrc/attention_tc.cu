// attention_tc.cu -- causal attention forward on the 5th-generation tensor cores (tcgen05 / TMEM).
//
// per (sample, local head e): S = Q_e K_e^T / sqrt(d), causal mask (reading R4),
// P = softmax(S), ctx = P V_e; lse2 = log2 sum exp2(S * scale * log2e) saved for the backward.
//
// One CTA = one 128-row query tile of one (sample, head); 256 threads:
//   warp 0    TMA producer: Q once, then K_j / V_j tiles (128 keys) into a 2-stage ring
//   warp 1    MMA issuer:   S_j = Q K_j^T into TMEM (double-buffered), then PV_{j-1} = P_{j-1} V_{j-1}
//             into TMEM (double-buffered); S_{j+1} is issued before PV_j so the tensor core works
//             while the softmax warps run
//   warp 2    TMEM allocator (512 columns: S0 | S1 | PV0 | PV1)
//   warps 4-7 softmax, thread = query row (= TMEM lane): two passes over S_j (max, then exp2 / row
//             sum / bf16 P written to 128-B-swizzled smem for the next MMA), then the running output
//             O = O * exp2(m_old - m_new) + PV accumulated in registers (fp32), normalised at the end.
// Operands: Q, K K-major (SW128, 64-wide atoms); V MN-major (its rows are keys); P K-major in smem.
#include <math.h>

#include "kernels.h"
#include "ptx.cuh"

namespace mk {

namespace {

constexpr int TQ = 128;  // query rows per CTA
constexpr int TK = 128;  // keys per tile

template <int D>
struct TcAttnCfg {
  static constexpr int NA = (D + 63) / 64;        // 64-wide swizzle atoms along d
  static constexpr int ATOM = 128 * 128;          // bytes of one [128 rows x 64] bf16 atom
  static constexpr int Q_BYTES = NA * ATOM;
  static constexpr int K_BYTES = NA * ATOM;
  static constexpr int V_BYTES = NA * ATOM;       // MN-major: NA chunks of 64 d-columns x 128 keys
  static constexpr int P_BYTES = 2 * ATOM;        // [128 q][128 keys] bf16, 2 atoms along keys
  static constexpr int STAGES = 2;
  static constexpr int SMEM = Q_BYTES + STAGES * (K_BYTES + V_BYTES) + P_BYTES + 1024 + 256;
  static constexpr uint32_t S_COL = 0, PV_COL = 256;
};

MK_DEV void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

}  // namespace

template <int D>
__global__ void __launch_bounds__(256, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tm, AttnArgs a) {
  using C = TcAttnCfg<D>;
  constexpr int NA = C::NA;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sQ = smem;
  uint8_t *sK = sQ + C::Q_BYTES;                      // [2][K_BYTES]
  uint8_t *sV = sK + C::STAGES * C::K_BYTES;          // [2][V_BYTES]
  uint8_t *sP = sV + C::STAGES * C::V_BYTES;          // [P_BYTES]
  uint64_t *bar = reinterpret_cast<uint64_t *>(sP + C::P_BYTES);
  uint64_t *q_full = bar + 0;
  uint64_t *kv_full = bar + 1, *kv_empty = bar + 3;
  uint64_t *s_full = bar + 5, *s_free = bar + 7;
  uint64_t *pv_full = bar + 9, *pv_free = bar + 11;
  uint64_t *p_full = bar + 13, *p_free = bar + 14;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bar + 16);

  const int s = a.s, H = a.heads;
  const int nqt = (s + TQ - 1) / TQ;
  const int qt = nqt - 1 - blockIdx.x;  // heaviest tiles first
  const int head = blockIdx.y, bi = blockIdx.z;
  const int hr = H * D;
  const int tok0 = bi * s;
  const int nkv = qt + 1;  // causal: key tiles 0..qt
  const int warp = warp_id(), lane = lane_id();

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm);
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 4);
      mbar_init(&pv_full[i], 1);
      mbar_init(&pv_free[i], 4);
    }
    mbar_init(p_full, 4);
    mbar_init(p_free, 1);
    fence_mbar_init();
    fence_proxy_async();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      mbar_expect_tx(q_full, C::Q_BYTES);
      for (int c = 0; c < NA; ++c) tma_load_2d(sQ + c * C::ATOM, &tm, q_full, head * D + c * 64, tok0 + qt * TQ);
    }
    for (int j = 0; j < nkv; ++j) {
      const int st = j & 1;
      mbar_wait(&kv_empty[st], ((j >> 1) & 1) ^ 1);
      if (lane == 0) {
        mbar_expect_tx(&kv_full[st], C::K_BYTES + C::V_BYTES);
        for (int c = 0; c < NA; ++c) {
          tma_load_2d(sK + st * C::K_BYTES + c * C::ATOM, &tm, &kv_full[st], hr + head * D + c * 64, tok0 + j * TK);
          tma_load_2d(sV + st * C::V_BYTES + c * C::ATOM, &tm, &kv_full[st], 2 * hr + head * D + c * 64,
                      tok0 + j * TK);
        }
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc_s = idesc_bf16(TQ, TK, false, false);  // Q K^T: both K-major
    constexpr uint32_t idesc_o = idesc_bf16(TQ, D, false, true);    // P V: V is MN-major
    mbar_wait(q_full, 0);
    for (int j = 0; j <= nkv; ++j) {
      if (j < nkv) {
        const int st = j & 1, sb = j & 1;
        mbar_wait(&kv_full[st], (j >> 1) & 1);
        mbar_wait(&s_free[sb], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t q0 = smem_u32(sQ), k0 = smem_u32(sK + st * C::K_BYTES);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk >> 2) * C::ATOM + (kk & 3) * 32;
            tc_mma_f16(tmem + C::S_COL + sb * TK, sdesc_sw128(q0 + off, 16, 1024), sdesc_sw128(k0 + off, 16, 1024),
                       idesc_s, kk > 0 ? 1u : 0u);
          }
          tc_commit(&s_full[sb]);
        }
        __syncwarp();
      }
      if (j >= 1) {
        const int i = j - 1, st = i & 1, pb = i & 1;
        mbar_wait(p_full, i & 1);
        mbar_wait(&pv_free[pb], ((i >> 1) & 1) ^ 1);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t p0 = smem_u32(sP), v0 = smem_u32(sV + st * C::V_BYTES);
#pragma unroll
          for (int kk = 0; kk < TK / 16; ++kk) {
            const uint32_t poff = (kk >> 2) * C::ATOM + (kk & 3) * 32;
            tc_mma_f16(tmem + C::PV_COL + pb * D, sdesc_sw128(p0 + poff, 16, 1024),
                       sdesc_sw128(v0 + kk * 2048, C::ATOM, 1024), idesc_o, kk > 0 ? 1u : 0u);
          }
          tc_commit(&pv_full[pb]);
          tc_commit(&kv_empty[st]);
          tc_commit(p_free);
        }
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax + output (thread = row)
    const int q = warp & 3;
    const int r = q * 32 + lane;                   // row within the tile = TMEM lane
    const int qi = qt * TQ + r;                    // query index within the sample
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    const float sl2 = 1.4426950408889634f / sqrtf((float)D);
    float o[D];
#pragma unroll
    for (int i = 0; i < D; ++i) o[i] = 0.f;
    float m = -INFINITY, l = 0.f, corr_prev = 1.f;
    uint8_t *prow = sP + r * 128;
    for (int j = 0; j < nkv; ++j) {
      const int sb = j & 1;
      mbar_wait(&s_full[sb], (j >> 1) & 1);
      tc_fence_after();
      const bool mask = (j == qt) || ((j + 1) * TK > s);
      const uint32_t sbase = lane_base + C::S_COL + sb * TK;
      // pass 1: row max
      float mx = m;
#pragma unroll 1
      for (int c = 0; c < TK / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(sbase + c * 32, v);
        tmem_ld_wait();
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const int kj = j * TK + c * 32 + k;
          const float x = __uint_as_float(v[k]);
          if (!mask || (kj <= qi && kj < s)) mx = fmaxf(mx, x);
        }
      }
      const float corr = fast_exp2((m - mx) * sl2);
      const float ms = mx * sl2;
      // the single P buffer must have been consumed by the previous P V
      mbar_wait(p_free, (j & 1) ^ 1);
      // pass 2: P = exp2(S*scale*log2e - m), row sum, bf16 P into the swizzled smem tile
      float rs = 0.f;
#pragma unroll 1
      for (int c = 0; c < TK / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(sbase + c * 32, v);
        tmem_ld_wait();
        uint32_t pk[16];
#pragma unroll
        for (int k = 0; k < 32; k += 2) {
          const int kj = j * TK + c * 32 + k;
          float p0 = fast_exp2(fmaf(__uint_as_float(v[k]), sl2, -ms));
          float p1 = fast_exp2(fmaf(__uint_as_float(v[k + 1]), sl2, -ms));
          if (mask) {
            if (!(kj <= qi && kj < s)) p0 = 0.f;
            if (!(kj + 1 <= qi && kj + 1 < s)) p1 = 0.f;
          }
          rs += p0 + p1;
          pk[k >> 1] = pack_bf16(p0, p1);
        }
        // keys c*32 .. c*32+31 = atom (c >> 1), 16-B chunks (c & 1) * 4 .. +3
        uint8_t *atom = prow + (c >> 1) * C::ATOM;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int chunk = (c & 1) * 4 + u;
          *reinterpret_cast<uint4 *>(atom + ((chunk ^ (r & 7)) << 4)) =
              make_uint4(pk[u * 4], pk[u * 4 + 1], pk[u * 4 + 2], pk[u * 4 + 3]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_free[sb]);
      fence_proxy_async();  // generic-proxy P stores -> visible to the tensor core
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
      l = l * corr + rs;
      m = mx;
      // fold in P_{j-1} V_{j-1} with its correction factor
      if (j >= 1) {
        const int i = j - 1, pb = i & 1;
        mbar_wait(&pv_full[pb], (i >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < D / 16; ++c) {
          uint32_t v[16];
          tmem_ld16(lane_base + C::PV_COL + pb * D + c * 16, v);
          tmem_ld_wait();
#pragma unroll
          for (int k = 0; k < 16; ++k) o[c * 16 + k] = o[c * 16 + k] * corr_prev + __uint_as_float(v[k]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&pv_free[pb]);
      }
      corr_prev = corr;
    }
    {
      const int i = nkv - 1, pb = i & 1;
      mbar_wait(&pv_full[pb], (i >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < D / 16; ++c) {
        uint32_t v[16];
        tmem_ld16(lane_base + C::PV_COL + pb * D + c * 16, v);
        tmem_ld_wait();
#pragma unroll
        for (int k = 0; k < 16; ++k) o[c * 16 + k] = o[c * 16 + k] * corr_prev + __uint_as_float(v[k]);
      }
    }
    if (qi < s) {
      const float inv = 1.f / l;
      __nv_bfloat16 *dst = reinterpret_cast<__nv_bfloat16 *>(a.ctx) + (size_t)(tok0 + qi) * a.ld_ctx + head * D;
#pragma unroll
      for (int c = 0; c < D; c += 8) {
        uint4 u;
        u.x = pack_bf16(o[c] * inv, o[c + 1] * inv);
        u.y = pack_bf16(o[c + 2] * inv, o[c + 3] * inv);
        u.z = pack_bf16(o[c + 4] * inv, o[c + 5] * inv);
        u.w = pack_bf16(o[c + 6] * inv, o[c + 7] * inv);
        *reinterpret_cast<uint4 *>(dst + c) = u;
      }
      a.lse[((size_t)bi * H + head) * s + qi] = m * sl2 + log2f(l);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ------------------------------------------------------------------------------------------ host
typedef CUresult (*EncodeTiledFn2)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                   const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static bool make_qkv_map(CUtensorMap *m, const void *qkv, int tokens, int cols) {
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
  cuuint32_t box[2] = {64u, 128u};
  cuuint32_t es[2] = {1u, 1u};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(qkv), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int D>
static cudaError_t fwd_tc_d(const AttnArgs &a, cudaStream_t st) {
  using C = TcAttnCfg<D>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  CUtensorMap m;
  if (!make_qkv_map(&m, a.qkv, a.b * a.s, 3 * a.heads * D)) return cudaErrorInvalidValue;
  dim3 grid((a.s + TQ - 1) / TQ, a.heads, a.b);
  attn_fwd_tc_kernel<D><<<grid, 256, C::SMEM, st>>>(m, a);
  return cudaGetLastError();
}

cudaError_t attn_fwd_tc(const AttnArgs &a, cudaStream_t st) {
  switch (a.d) {
    case 32: return fwd_tc_d<32>(a, st);
    case 64: return fwd_tc_d<64>(a, st);
    case 80: return fwd_tc_d<80>(a, st);
    case 96: return fwd_tc_d<96>(a, st);
    case 128: return fwd_tc_d<128>(a, st);
  }
  return cudaErrorNotSupported;
}

}  // namespace mk
