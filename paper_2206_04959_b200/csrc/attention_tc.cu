// attention_tc.cu -- causal attention forward on the 5th-generation tensor cores (tcgen05 / TMEM).
//
// per (sample, local head e): S = Q_e K_e^T / sqrt(d), causal mask (reading R4),
// P = softmax(S), ctx = P V_e; lse2 = log2 sum exp2(S * scale * log2e) saved for the backward.
//
// One CTA = TWO adjacent 128-row query tiles (A = 2p, B = 2p + 1) of one (sample, head), 320 threads,
// one CTA per SM (all 512 TMEM columns):
//   warp 0     TMA producer: Q_A, Q_B once, then 128-key tiles K_j / V_j (shared by both query tiles)
//   warp 1     TMEM owner + MMA issuer, ping-pong between the tiles: while softmax group A works on S_A(j)
//              the tensor core runs S_B(j) and P_B(j-1) V_j-1, and vice versa
//   warps 2-5  softmax of tile A, warps 6-9 softmax of tile B: thread = query row = TMEM lane, the whole
//              128-key row in registers (no cross-warp exchange).  P (bf16) is written back into the TMEM
//              columns of S and read from there as the A operand of O += P V (tcgen05.mma with A in TMEM),
//              so P never touches shared memory.
// TMEM: S_A [0,128), S_B [128,256), O_A [256, 256+D), O_B [384, 384+D) (fp32 columns).
// The running max is updated lazily (only when it grows by more than 2^8, as in FlashAttention-4): then O
// (in TMEM) is rescaled in place after the previous P V completed; otherwise probabilities are taken
// relative to the stale max (<= 2^8, exact after the final 1 / l).
// Operands: Q, K K-major; V MN-major (its rows are keys); P K-major in TMEM.
#include <math.h>

#include "kernels.h"
#include "ptx.cuh"

namespace mk {

namespace {

constexpr int TQ = 128;  // query rows per tile (TMEM lanes)
constexpr int TK = 128;  // keys per K/V tile

template <int D>
struct FaCfg {
  static constexpr int NA = (D + 63) / 64;          // 64-wide swizzle atoms along d
  static constexpr int ATOM = 128 * 128;            // [128 rows][64] bf16
  static constexpr int Q_BYTES = NA * ATOM;         // one query tile
  static constexpr int K_BYTES = NA * ATOM;         // K-major [128 keys][d]
  static constexpr int V_BYTES = NA * ATOM;         // MN-major: NA chunks of [128 keys][64 d-columns]
  static constexpr int STAGES = (D <= 64) ? 3 : 2;
  static constexpr int SMEM = 2 * Q_BYTES + STAGES * (K_BYTES + V_BYTES) + 1024 + 256;
  static constexpr uint32_t S_COL = 0;              // + 128 * tile
  static constexpr uint32_t O_COL = 256;            // + 128 * tile
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

// packed fp32 pairs (FFMA2 / FADD2 on sm_100): lo = first element
MK_DEV uint64_t pack_u64(uint32_t lo, uint32_t hi) { return ((uint64_t)hi << 32) | lo; }
MK_DEV uint64_t f32x2(float lo, float hi) { return pack_u64(__float_as_uint(lo), __float_as_uint(hi)); }
MK_DEV uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
MK_DEV uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
MK_DEV float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

}  // namespace

template <int D>
__global__ void __launch_bounds__(320, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tmq, const __grid_constant__ CUtensorMap tmkv, AttnArgs a) {
  using C = FaCfg<D>;
  constexpr int NA = C::NA, ST = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sQ = smem;                            // [2][Q_BYTES]
  uint8_t *sK = sQ + 2 * C::Q_BYTES;             // [ST][K_BYTES]
  uint8_t *sV = sK + ST * C::K_BYTES;            // [ST][V_BYTES]
  uint64_t *bar = reinterpret_cast<uint64_t *>(sV + ST * C::V_BYTES);
  uint64_t *q_full = bar;
  uint64_t *kv_full = bar + 1, *kv_empty = bar + 1 + ST;
  uint64_t *s_full = bar + 1 + 2 * ST, *p_full = s_full + 2, *o_done = s_full + 4;  // [2] each: tile A, B
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(s_full + 6);

  const int s = a.s, H = a.heads;
  const int nqt = (s + TQ - 1) / TQ, nkt = (s + TK - 1) / TK;
  const int np = (nqt + 1) / 2;
  const int p = np - 1 - blockIdx.z;  // grid (heads, b, pairs): globally heaviest pairs first
  const int head = blockIdx.x, bi = blockIdx.y;
  const int hr = H * D;
  const int tok0 = bi * s;
  const int ntile = (2 * p + 1 < nqt) ? 2 : 1;       // the last pair may hold one tile
  const int J0 = min(2 * p + 1, nkt);                 // key tiles of query tile A / B (causal)
  const int J1 = ntile == 2 ? min(2 * p + 2, nkt) : 0;
  const int Jmax = max(J0, J1);
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
      mbar_init(&p_full[i], 4);
      mbar_init(&o_done[i], 1);
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
      mbar_expect_tx(q_full, ntile * C::Q_BYTES);
      for (int t = 0; t < ntile; ++t)
        for (int c = 0; c < NA; ++c)
          tma_load_2d(sQ + t * C::Q_BYTES + c * C::ATOM, &tmq, q_full, head * D + c * 64, tok0 + (2 * p + t) * TQ);
    }
    for (int j = 0; j < Jmax; ++j) {
      const int st = j % ST;
      mbar_wait(&kv_empty[st], ((j / ST) & 1) ^ 1);
      if (lane == 0) {
        mbar_expect_tx(&kv_full[st], C::K_BYTES + C::V_BYTES);
        for (int c = 0; c < NA; ++c) {
          tma_load_2d(sK + st * C::K_BYTES + c * C::ATOM, &tmkv, &kv_full[st], hr + head * D + c * 64, tok0 + j * TK);
          tma_load_2d(sV + st * C::V_BYTES + c * C::ATOM, &tmkv, &kv_full[st], 2 * hr + head * D + c * 64,
                      tok0 + j * TK);
        }
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc_s = idesc_bf16(TQ, TK, false, false);  // Q K^T: both K-major
    constexpr uint32_t idesc_o = idesc_bf16(TQ, D, false, true);    // P V: P K-major (TMEM), V MN-major
    mbar_wait(q_full, 0);
    for (int j = 0; j <= Jmax; ++j) {
      if (j < Jmax) {
        mbar_wait(&kv_full[j % ST], (j / ST) & 1);
        tc_fence_after();
      }
      for (int t = 0; t < ntile; ++t) {
        // O_t += P_t(j-1) V_{j-1}: P_t(j-1) sits in S_t's columns (written by softmax group t)
        if (j >= 1 && j - 1 < (t ? J1 : J0)) {
          const int i = j - 1, st = i % ST;
          mbar_wait(&p_full[t], i & 1);
          tc_fence_after();
          // whole-warp issue (tc_*_w elect one lane inside the asm: no per-lane broadcast loop per MMA)
          const uint64_t vd = sdesc_sw128(smem_u32(sV + st * C::V_BYTES), C::ATOM, 1024);
#pragma unroll
          for (int kk = 0; kk < TK / 16; ++kk)
            tc_mma_f16_ts_w(tmem + C::O_COL + 128 * t, tmem + C::S_COL + 128 * t + kk * 8, vd + (kk * 2048 >> 4),
                            idesc_o, (i > 0 || kk > 0) ? 1u : 0u);
          tc_commit_w(&o_done[t]);
        }
        // S_t(j) = Q_t K_j^T into S_t's columns (issued after the P V that reads them: in-order execution)
        if (j < (t ? J1 : J0)) {
          const uint64_t qd = sdesc_sw128(smem_u32(sQ + t * C::Q_BYTES), 16, 1024);
          const uint64_t kd = sdesc_sw128(smem_u32(sK + (j % ST) * C::K_BYTES), 16, 1024);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = ((kk >> 2) * C::ATOM + (kk & 3) * 32) >> 4;
            tc_mma_f16_w(tmem + C::S_COL + 128 * t, qd + off, kd + off, idesc_s, kk > 0 ? 1u : 0u);
          }
          tc_commit_w(&s_full[t]);
        }
      }
      // K/V stage of j-1 is free once both tiles' P V of j-1 have completed
      if (j >= 1) tc_commit_w(&kv_empty[(j - 1) % ST]);
    }
  } else {
    // ------------------------------------------------------------ softmax (thread = query row)
    const int t = (warp - 2) >> 2;  // query tile of this warpgroup
    const int q = warp & 3;         // TMEM lane quarter this warp may access
    const int r = q * 32 + lane;
    const int qt = 2 * p + t;
    const int qi = qt * TQ + r;
    const int J = t ? J1 : J0;
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    const uint32_t s_col = lane_base + C::S_COL + 128 * t, o_col = lane_base + C::O_COL + 128 * t;
    const float sl2 = 1.4426950408889634f / sqrtf((float)D);
    const float thr = 8.0f / sl2;  // lazy rescale threshold (2^8) in raw score units
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < J; ++j) {
      mbar_wait(&s_full[t], j & 1);
      tc_fence_after();
      uint32_t v[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(s_col + 32 * c, *reinterpret_cast<uint32_t(*)[32]>(&v[32 * c]));
      tmem_ld_wait();
      const int kj0 = j * TK;
      const bool mask = (kj0 + TK - 1 > qi) || (kj0 + TK > s);
      if (mask) {  // diagonal / ragged tile: keys kj0 + k with k > lim are invisible to this row -> -inf
        const int lim = min(qi, s - 1) - kj0;
#pragma unroll
        for (int k = 0; k < 128; ++k)
          if (k > lim) v[k] = 0xff800000u;
      }
      float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};  // independent chains, 3-input max
#pragma unroll
      for (int k = 0; k < 128; k += 8)
#pragma unroll
        for (int c = 0; c < 4; ++c) mx4[c] = fmax3(mx4[c], __uint_as_float(v[k + 2 * c]), __uint_as_float(v[k + 2 * c + 1]));
      const float mx = fmaxf(m, fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])));
      // the max grew by more than 2^8: move to the new max, rescale O and l.  TMEM access is warp-collective,
      // so the whole warp enters when any row needs it (the others scale by 1).
      const bool need = mx > m + thr;
      if (__any_sync(0xffffffffu, need)) {
        const float corr = need ? fast_exp2((m - mx) * sl2) : 1.f;
        if (j >= 1) {
          mbar_wait(&o_done[t], (j - 1) & 1);  // P(j-1) V(j-1) has landed in O
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < D / 16; ++c) {
            uint32_t o[16];
            tmem_ld16(o_col + c * 16, o);
            tmem_ld_wait();
#pragma unroll
            for (int k = 0; k < 16; ++k) o[k] = __float_as_uint(__uint_as_float(o[k]) * corr);
            tmem_st16(o_col + c * 16, o);
          }
          tmem_st_wait();
        }
        if (need) {
          l *= corr;
          m = mx;
        }
      }
      const float ms = m * sl2;
      // p = exp2(s * sl2 - m * sl2): packed FFMA2 for the argument, MUFU.EX2, packed FADD2 for the row sum
      const uint64_t sc2 = f32x2(sl2, sl2), nm2 = f32x2(-ms, -ms);
      uint64_t rs2[4] = {0, 0, 0, 0};
#pragma unroll
      for (int k = 0; k < 128; k += 2) {
        const uint64_t x = ffma2(pack_u64(v[k], v[k + 1]), sc2, nm2);
        const float p0 = fast_exp2(__uint_as_float((uint32_t)x)), p1 = fast_exp2(__uint_as_float((uint32_t)(x >> 32)));
        rs2[(k >> 1) & 3] = fadd2(rs2[(k >> 1) & 3], f32x2(p0, p1));
        v[k >> 1] = pack_bf16(p0, p1);  // P packed into v[0..63] (v[k], v[k+1] already consumed)
      }
      const uint64_t rs = fadd2(fadd2(rs2[0], rs2[1]), fadd2(rs2[2], rs2[3]));
      l += __uint_as_float((uint32_t)rs) + __uint_as_float((uint32_t)(rs >> 32));
      // P (bf16 pairs) over the first 64 columns of S: the A operand of O += P V
      tmem_st32(s_col, *reinterpret_cast<const uint32_t(*)[32]>(&v[0]));
      tmem_st32(s_col + 32, *reinterpret_cast<const uint32_t(*)[32]>(&v[32]));
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[t]);
    }
    // the last P V has completed when its commit arrived on o_done
    mbar_wait(&o_done[t], (J - 1) & 1);
    tc_fence_after();
    // tcgen05.ld is warp-collective (.sync.aligned): load converged, store only rows < s
    const float inv = 1.f / l;
    __nv_bfloat16 *dst = reinterpret_cast<__nv_bfloat16 *>(a.ctx) + (size_t)(tok0 + qi) * a.ld_ctx + head * D;
#pragma unroll
    for (int c = 0; c < D / 16; ++c) {
      uint32_t o[16];
      tmem_ld16(o_col + c * 16, o);
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
    if (qi < s) a.lse[((size_t)bi * H + head) * s + qi] = m * sl2 + log2f(l);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
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
      !make_qkv_map(&mkv, a.qkv, a.b * a.s, 3 * a.heads * D, TK))
    return cudaErrorInvalidValue;
  dim3 grid(a.heads, a.b, ((a.s + TQ - 1) / TQ + 1) / 2);
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
