// gemm.cu -- persistent warp-specialised tcgen05 GEMM for sm_100a with fused epilogues.
//
// Every dense contraction of the sub-pipelined TMP layer runs here (SURVEY §8(a) F2, F4, F6, F7,
// B1, B2, B3, B5, B7): forward (both operands K-major), dgrad (weight operand MN-major) and
// wgrad (both operands MN-major, fp32 accumulator preloaded into TMEM so the per-element
// accumulation chain over tokens is the same whatever the sub-batch split -- bit-identity rule v).
//
// CTA = 256 threads, one CTA per SM (smem-bound), grid = min(tiles, SMs), static tile schedule.
//   warp 0 : TMA producer (one lane)      -> smem ring of STAGES {A 128x64, B BNx64} bf16 tiles
//   warp 1 : MMA issuer (one lane)        -> tcgen05.mma 128xBNx16 into a TMEM accumulator
//   warp 2 : TMEM allocator (2 x BN fp32 columns: double-buffered accumulator)
//   warps 4-7 : epilogue (tcgen05.ld 32x32b -> registers -> fused op -> global)
// Smem tiles use the 128-byte swizzle; the UMMA descriptors describe the same canonical layouts:
//   K-major : rows of 64 K-elements (128 B), 8-row groups 1024 B apart (SBO)
//   MN-major: K-rows of 64 MN-elements (128 B), 8-K-row groups 1024 B apart (SBO),
//             64-wide MN chunks BLOCK_K*128 = 8 KB apart (LBO)
#include <cuda.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "kernels.h"
#include "ptx.cuh"

namespace mk {

constexpr int BM = 128;  // rows of A per CTA (TMEM lanes)
constexpr int BK = 64;

// CG = CTAs per MMA (cta_group): CG = 2 pairs two SMs on a 256 x BN tile (each CTA stages its
// 128 rows of A and BN/2 rows of B; the leader issues tcgen05.mma.cta_group::2).
template <int CG, int BN, int SMEM_KB = (CG == 2 ? 160 : 192)>
struct GemmCfg {
  static constexpr int BNC = BN / CG;  // B rows staged per CTA
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BNC * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = SMEM_KB * 1024 / STAGE_BYTES > 8 ? 8 : SMEM_KB * 1024 / STAGE_BYTES;
  static constexpr int TMEM_COLS = (2 * BN <= 256) ? 256 : 512;  // power of two >= 2 accumulators
  // ring + barriers (1 KB) + epilogue staging (4 warps x 2 boxes x 4 KB) + alignment slack
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 4 * 8192 + 1024;
};

struct EpiParams {
  int M, N, K;
  int epi;
  __nv_bfloat16 *out;
  int ldo;
  __nv_bfloat16 *out2;
  int ldo2;
  const __nv_bfloat16 *bias;
  const __nv_bfloat16 *aux;
  int ld_aux;
  float *out32;
  int ld32;
  float *db32;  // EPI_ACC_F32: column n_main (the ones column of B) accumulates into db32[m]
  int n_main;
  int *tile_ctr;  // dynamic tile scheduler counter (zero between launches), nullptr = static schedule
  int group_m;    // m-tiles per raster band (tile_coords): 1 = n fastest over all of N, tiles_m = m fastest
  int hint_a, hint_b, hint_c;  // L2 eviction priority of the A / B TMA loads and the fp32 C accesses (l2_policy)
  // Scatter store (EPI_STORE_BF16 only, GemmArgs::scatter): output row i goes to owner q = i / scatter_rows,
  // row scatter_row0 + i - q * scatter_rows of the tensor map scatter[q] (a peer's slot, in global memory)
  const CUtensorMap *scatter;
  int scatter_row0, scatter_rows;
};

template <int EPI>
MK_DEV void epi_store_chunk(const EpiParams &p, int gm, int gn0, const uint32_t (&r)[32], uint64_t pol_c = 0) {
  if constexpr (EPI == 5) {  // microbenchmark variant: drain TMEM, store nothing
    if (r[0] == 0x7fc00001u && gm < 0) p.out[0] = __float2bfloat16_rn(0.f);
    return;
  }
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
  const bool full = (gn0 + 32 <= p.N);
  if constexpr (EPI == EPI_ACC_F32) {
    float *dst = p.out32 + (size_t)gm * p.ld32 + gn0;
    if (gn0 + 32 <= p.n_main && (p.ld32 % 4 == 0)) {
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        if (p.hint_c)
          stg_f4_hint(dst + i, make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]), pol_c);
        else
          *reinterpret_cast<float4 *>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
      }
    } else {
      for (int i = 0; i < 32; ++i) {
        if (gn0 + i < p.n_main) dst[i] = v[i];
        else if (gn0 + i == p.n_main && p.db32) p.db32[gm] = v[i];
      }
    }
    return;
  } else {
    if constexpr (EPI == EPI_BIAS_BF16 || EPI == EPI_BIAS_GELU) {
      if (full) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint4 bv = *reinterpret_cast<const uint4 *>(p.bias + gn0 + i);
          float2 b0 = unpack_bf16(bv.x), b1 = unpack_bf16(bv.y), b2 = unpack_bf16(bv.z), b3 = unpack_bf16(bv.w);
          v[i + 0] += b0.x; v[i + 1] += b0.y; v[i + 2] += b1.x; v[i + 3] += b1.y;
          v[i + 4] += b2.x; v[i + 5] += b2.y; v[i + 6] += b3.x; v[i + 7] += b3.y;
        }
      } else {
        for (int i = 0; i < 32; ++i)
          if (gn0 + i < p.N) v[i] += __bfloat162float(p.bias[gn0 + i]);
      }
    }
    if constexpr (EPI == EPI_GELU_BWD) {
      const __nv_bfloat16 *z = p.aux + (size_t)gm * p.ld_aux + gn0;
      if (full) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint4 zv = *reinterpret_cast<const uint4 *>(z + i);
          float2 z0 = unpack_bf16(zv.x), z1 = unpack_bf16(zv.y), z2 = unpack_bf16(zv.z), z3 = unpack_bf16(zv.w);
          v[i + 0] *= gelu_grad_f(z0.x); v[i + 1] *= gelu_grad_f(z0.y);
          v[i + 2] *= gelu_grad_f(z1.x); v[i + 3] *= gelu_grad_f(z1.y);
          v[i + 4] *= gelu_grad_f(z2.x); v[i + 5] *= gelu_grad_f(z2.y);
          v[i + 6] *= gelu_grad_f(z3.x); v[i + 7] *= gelu_grad_f(z3.y);
        }
      } else {
        for (int i = 0; i < 32; ++i)
          if (gn0 + i < p.N) v[i] *= gelu_grad_f(__bfloat162float(z[i]));
      }
    }
    __nv_bfloat16 *dst = p.out + (size_t)gm * p.ldo + gn0;
    if (full) {
#pragma unroll
      for (int i = 0; i < 32; i += 8) {
        uint4 o;
        o.x = pack_bf16(v[i + 0], v[i + 1]); o.y = pack_bf16(v[i + 2], v[i + 3]);
        o.z = pack_bf16(v[i + 4], v[i + 5]); o.w = pack_bf16(v[i + 6], v[i + 7]);
        *reinterpret_cast<uint4 *>(dst + i) = o;
      }
    } else {
      for (int i = 0; i < 32; ++i)
        if (gn0 + i < p.N) dst[i] = __float2bfloat16_rn(v[i]);
    }
    if constexpr (EPI == EPI_BIAS_GELU) {
      __nv_bfloat16 *dst2 = p.out2 + (size_t)gm * p.ldo2 + gn0;
      if (full) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint4 o;
          o.x = pack_bf16(gelu_f(v[i + 0]), gelu_f(v[i + 1])); o.y = pack_bf16(gelu_f(v[i + 2]), gelu_f(v[i + 3]));
          o.z = pack_bf16(gelu_f(v[i + 4]), gelu_f(v[i + 5])); o.w = pack_bf16(gelu_f(v[i + 6]), gelu_f(v[i + 7]));
          *reinterpret_cast<uint4 *>(dst2 + i) = o;
        }
      } else {
        for (int i = 0; i < 32; ++i)
          if (gn0 + i < p.N) dst2[i] = __float2bfloat16_rn(gelu_f(v[i]));
      }
    }
  }
}

// Tile raster: bands of group_m m-tiles, n-major inside a band (m fastest within a group column).  The host
// picks group_m per GEMM (pick_group_m): when one operand fits in L2 the band makes it the one every wave
// shares -- group_m = tiles_m keeps all of A resident while B streams through once, group_m = 1 keeps all of B
// resident while A streams once -- otherwise bands of 8 make each ~74-tile wave a compact ~8 x 9 block sharing
// its A and B k-slabs.  The order never changes a tile's K reduction.
MK_DEV void tile_coords(int tile, int tiles_m, int tiles_n, int group_m, int &tm, int &tn) {
  const int band = tile / (group_m * tiles_n);
  const int m0 = band * group_m;
  const int gm = min(group_m, tiles_m - m0);  // last band may be narrower
  const int r = tile - band * group_m * tiles_n;
  tm = m0 + r % gm;
  tn = r / gm;
}

template <int CG, int BN, bool A_MN, bool B_MN, int EPI, int SMEM_KB>
__global__ void __launch_bounds__(256, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmO2, EpiParams p) {
  using C = GemmCfg<CG, BN, SMEM_KB>;
  constexpr int S = C::STAGES;
  constexpr int BMT = BM * CG;  // tile rows
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *smA = smem;
  uint8_t *smB = smem + S * C::A_BYTES;
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + S * C::STAGE_BYTES);
  uint64_t *full = bars, *empty = bars + S, *tfull = bars + 2 * S, *tfree = bars + 2 * S + 2;
  uint64_t *sched_full = bars + 2 * S + 4, *sched_empty = bars + 2 * S + 8;  // tile-id ring, 4 deep
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * S + 12);
  int *ring = reinterpret_cast<int *>(bars + 2 * S + 13);

  const int warp = warp_id();
  const int lane = lane_id();
  const uint32_t rank = (CG == 2) ? cluster_ctarank() : 0u;
  const int cl = blockIdx.x / CG, ncl = gridDim.x / CG;
  const int tiles_m = (p.M + BMT - 1) / BMT;
  const int tiles_n = (p.N + BN - 1) / BN;
  const int ntiles = tiles_m * tiles_n;
  const int nk = (p.K + BK - 1) / BK;
  // Tile order.  Static: cluster cl takes tiles cl, cl + ncl, ...  Dynamic (p.tile_ctr): the leader's
  // producer fetches the next tile index with an atomic and broadcasts it through a 4-deep smem ring
  // to its MMA / epilogue warps and to the peer CTA, so clusters that start late (SMs still held by a
  // kernel of the other sub-batch stream) simply take fewer tiles.  Every tile is still computed by
  // one cluster in the fixed K order, so results do not depend on the order (bit-identity rule i).
  const bool dyn = (EPI != EPI_ACC_F32) && p.tile_ctr != nullptr;
  auto consume = [&](int lt) -> int {  // MMA, epilogue and peer-producer warps
    if (!dyn) return cl + lt * ncl;
    const int slot = lt & 3;
    const uint32_t ph = (lt >> 2) & 1;
    if (CG == 2 && rank == 1)
      mbar_wait_cluster(&sched_full[slot], ph);
    else
      mbar_wait(&sched_full[slot], ph);
    const int t = *reinterpret_cast<volatile int *>(&ring[slot]);
    __syncwarp();
    if (lane == 0) {
      if (CG == 2 && rank == 1)
        mbar_arrive_cluster(mapa_shared(&sched_empty[slot], 0));
      else
        mbar_arrive(&sched_empty[slot]);
    }
    return t;
  };
  auto fetch = [&](int lt) -> int {  // leader producer warp
    if (!dyn) return cl + lt * ncl;
    const int slot = lt & 3;
    int t = 0;
    if (lane == 0) {
      mbar_wait(&sched_empty[slot], ((lt >> 2) & 1) ^ 1);
      t = atomicAdd(p.tile_ctr, 1);
      if (t == ntiles + ncl - 1) atomicExch(p.tile_ctr, 0);  // the launch's last fetch: reset for the next
      ring[slot] = t;
      if constexpr (CG == 2) {
        st_shared_cluster_u32(mapa_shared(&ring[slot], 1), (uint32_t)t);
        mbar_arrive_cluster(mapa_shared(&sched_full[slot], 1));
      }
      mbar_arrive(&sched_full[slot]);
    }
    return __shfl_sync(0xffffffffu, t, 0);
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tfree[i], 4 * CG);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&sched_full[i], 1);
      mbar_init(&sched_empty[i], CG == 2 ? 10 : 5);  // MMA + 4 epilogue warps (+ peer producer + 4)
    }
    fence_mbar_init();
    fence_proxy_async();
  }
  // 2-CTA: both CTAs of the pair are synchronised BEFORE the paired TMEM allocation (as well as after it
  // and before teardown), the documented protocol for tcgen05.alloc.cta_group::2
  if constexpr (CG == 2) cluster_sync();
  if (warp == 2) {
    if constexpr (CG == 2)
      tmem_alloc2<C::TMEM_COLS>(tmem_slot);
    else
      tmem_alloc<C::TMEM_COLS>(tmem_slot);
  }
  tc_fence_before();
  if constexpr (CG == 2)
    cluster_sync();
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs of a pair load their own halves)
    const uint64_t pol_a = l2_policy(p.hint_a), pol_b = l2_policy(p.hint_b);
    int it = 0;
    for (int lt = 0;; ++lt) {
      const int tile = (rank == 0) ? fetch(lt) : consume(lt);
      if (tile >= ntiles) break;
      int tm, tn;
      tile_coords(tile, tiles_m, tiles_n, p.group_m, tm, tn);
      const int row0 = tm * BMT + rank * BM;
      const int n0 = tn * BN + rank * C::BNC;
      for (int kb = 0; kb < nk; ++kb, ++it) {
        const int s = it % S;
        const uint32_t ph = (it / S) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        if (lane == 0) {
          if (rank == 0) mbar_expect_tx(&full[s], C::STAGE_BYTES * CG);
          uint8_t *a = smA + s * C::A_BYTES;
          uint8_t *b = smB + s * C::B_BYTES;
          auto load = [&](void *dst, const CUtensorMap *m, int c0, int c1, int hint, uint64_t pol) {
            if constexpr (CG == 2) {
              if (hint) tma_load_2d_cg2_hint(dst, m, &full[s], c0, c1, pol);
              else tma_load_2d_cg2(dst, m, &full[s], c0, c1);
            } else {
              if (hint) tma_load_2d_hint(dst, m, &full[s], c0, c1, pol);
              else tma_load_2d(dst, m, &full[s], c0, c1);
            }
          };
          if constexpr (!A_MN) {
            load(a, &tmA, kb * BK, row0, p.hint_a, pol_a);
          } else {
#pragma unroll
            for (int c = 0; c < BM / 64; ++c) load(a + c * 8192, &tmA, row0 + c * 64, kb * BK, p.hint_a, pol_a);
          }
          if constexpr (!B_MN) {
            load(b, &tmB, kb * BK, n0, p.hint_b, pol_b);
          } else {
#pragma unroll
            for (int c = 0; c < C::BNC / 64; ++c) load(b + c * 8192, &tmB, n0 + c * 64, kb * BK, p.hint_b, pol_b);
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == 1 && rank == 0) {
    // ---------------- MMA issuer (leader CTA)
    constexpr uint32_t idesc = idesc_bf16(BMT, BN, A_MN, B_MN);
    constexpr uint32_t a_lbo = A_MN ? 8192u : 16u, a_sbo = 1024u, a_kstep = A_MN ? 2048u : 32u;
    constexpr uint32_t b_lbo = B_MN ? 8192u : 16u, b_sbo = 1024u, b_kstep = B_MN ? 2048u : 32u;
    int it = 0;
    for (int lt = 0;; ++lt) {
      const int tile = consume(lt);
      if (tile >= ntiles) break;
      const int buf = lt & 1;
      mbar_wait(&tfree[buf], (lt >> 1) & 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + buf * BN;
      for (int kb = 0; kb < nk; ++kb, ++it) {
        const int s = it % S;
        mbar_wait(&full[s], (it / S) & 1);
        tc_fence_after();
        // whole-warp issue: elect.sync inside the asm (one instruction per MMA, no per-lane broadcast loop)
        const uint64_t ad0 = sdesc_sw128(smem_u32(smA + s * C::A_BYTES), a_lbo, a_sbo);
        const uint64_t bd0 = sdesc_sw128(smem_u32(smB + s * C::B_BYTES), b_lbo, b_sbo);
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk) {
          const uint32_t acc = (EPI == EPI_ACC_F32 || kb > 0 || kk > 0) ? 1u : 0u;
          if constexpr (CG == 2)
            tc_mma_f16_cg2_w(d_tmem, ad0 + ((kk * a_kstep) >> 4), bd0 + ((kk * b_kstep) >> 4), idesc, acc);
          else
            tc_mma_f16_w(d_tmem, ad0 + ((kk * a_kstep) >> 4), bd0 + ((kk * b_kstep) >> 4), idesc, acc);
        }
        if constexpr (CG == 2) {
          tc_commit_cg2_mc_w(&empty[s], 0x3);
          if (kb == nk - 1) tc_commit_cg2_mc_w(&tfull[buf], 0x3);
        } else {
          tc_commit_w(&empty[s]);
          if (kb == nk - 1) tc_commit_w(&tfull[buf]);
        }
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue (each CTA drains its own 128 TMEM lanes = its 128 rows of the tile)
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const uint32_t row_base = tmem_base + ((uint32_t)(q * 32) << 16);
    const uint64_t pol_c = l2_policy(p.hint_c);
    const uint32_t tfree_leader[2] = {CG == 2 ? mapa_shared(&tfree[0], 0) : 0u,
                                      CG == 2 ? mapa_shared(&tfree[1], 0) : 0u};
    auto release = [&](int buf) {
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 2)
          mbar_arrive_cluster(tfree_leader[buf]);
        else
          mbar_arrive(&tfree[buf]);
      }
    };
    auto preload = [&](int tile, int buf) {
      int tm, tn;
      tile_coords(tile, tiles_m, tiles_n, p.group_m, tm, tn);
      const int gm = tm * BMT + rank * BM + q * 32 + lane;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        const int gn0 = tn * BN + c * 32;
        uint32_t r[32];
        const float *src = p.out32 + (size_t)gm * p.ld32 + gn0;
        if (gm < p.M && gn0 + 32 <= p.n_main && (p.ld32 % 4 == 0)) {
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const float4 f = p.hint_c ? ldg_f4_hint(src + i, pol_c) : *reinterpret_cast<const float4 *>(src + i);
            r[i] = __float_as_uint(f.x); r[i + 1] = __float_as_uint(f.y);
            r[i + 2] = __float_as_uint(f.z); r[i + 3] = __float_as_uint(f.w);
          }
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            float val = 0.f;
            if (gm < p.M) {
              if (gn0 + i < p.n_main) val = src[i];
              else if (gn0 + i == p.n_main && p.db32) val = p.db32[gm];
            }
            r[i] = __float_as_uint(val);
          }
        }
        tmem_st32(row_base + buf * BN + c * 32, r);
      }
      tmem_st_wait();
    };
    // initial release of both accumulator buffers (after preloading C for ACC mode)
#pragma unroll 1
    for (int bb = 0; bb < 2; ++bb) {
      const int tile = cl + bb * ncl;
      if (EPI == EPI_ACC_F32 && tile < ntiles) preload(tile, bb);
      release(bb);
    }
    int lt = 0;
    // bf16 outputs leave through TMA stores: per warp, 32 rows x 64 columns staged in a 128-B-swizzled
    // 4 KB smem box (two boxes, alternating), so global writes are whole coalesced lines.
    uint8_t *stg = smem + S * C::STAGE_BYTES + 1024 + q * 8192;
    int sbuf = 0;
    auto stage_store = [&](const CUtensorMap *map, const uint32_t (&w)[32], int gn0, int grow0) {
      if (lane == 0) tma_store_wait_read<1>();  // the box written two stores ago has been read
      __syncwarp();
      uint8_t *box = stg + sbuf * 4096 + lane * 128;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        *reinterpret_cast<uint4 *>(box + ((j ^ (lane & 7)) << 4)) =
            make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(map, stg + sbuf * 4096, gn0, grow0);
        tma_store_commit();
      }
      sbuf ^= 1;
    };
    for (;; ++lt) {
      const int tile = consume(lt);
      if (tile >= ntiles) break;
      const int buf = lt & 1;
      mbar_wait(&tfull[buf], (lt >> 1) & 1);
      tc_fence_after();
      int tm, tn;
      tile_coords(tile, tiles_m, tiles_n, p.group_m, tm, tn);
      const int gm = tm * BMT + rank * BM + q * 32 + lane;
      if constexpr (EPI == EPI_ACC_F32 || EPI == 5) {
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          const int gn0 = tn * BN + c * 32;
          if (gn0 >= p.N) break;  // warp-uniform
          uint32_t r[32];
          tmem_ld32(row_base + buf * BN + c * 32, r);
          tmem_ld_wait();
          if (gm < p.M) epi_store_chunk<EPI>(p, gm, gn0, r, pol_c);
        }
      } else {
        const int grow0 = tm * BMT + rank * BM + q * 32;
#pragma unroll 1
        for (int c = 0; c < BN / 64; ++c) {
          const int gn0 = tn * BN + c * 64;
          if (gn0 >= p.N) break;  // warp-uniform
          uint32_t r[64];
          tmem_ld32(row_base + buf * BN + c * 64, *reinterpret_cast<uint32_t(*)[32]>(r));
          tmem_ld32(row_base + buf * BN + c * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(r + 32));
          tmem_ld_wait();
          float v[64];
#pragma unroll
          for (int i = 0; i < 64; ++i) v[i] = __uint_as_float(r[i]);
          const bool fulln = gn0 + 64 <= p.N;
          if constexpr (EPI == EPI_BIAS_BF16 || EPI == EPI_BIAS_GELU) {
            if (fulln) {
#pragma unroll
              for (int i = 0; i < 64; i += 8) {
                uint4 bv = *reinterpret_cast<const uint4 *>(p.bias + gn0 + i);
                float2 b0 = unpack_bf16(bv.x), b1 = unpack_bf16(bv.y), b2 = unpack_bf16(bv.z), b3 = unpack_bf16(bv.w);
                v[i + 0] += b0.x; v[i + 1] += b0.y; v[i + 2] += b1.x; v[i + 3] += b1.y;
                v[i + 4] += b2.x; v[i + 5] += b2.y; v[i + 6] += b3.x; v[i + 7] += b3.y;
              }
            } else {
#pragma unroll
              for (int i = 0; i < 64; ++i)
                if (gn0 + i < p.N) v[i] += __bfloat162float(p.bias[gn0 + i]);
            }
          }
          if constexpr (EPI == EPI_GELU_BWD) {
            if (gm < p.M) {
              const __nv_bfloat16 *z = p.aux + (size_t)gm * p.ld_aux + gn0;
              if (fulln) {
#pragma unroll
                for (int i = 0; i < 64; i += 8) {
                  uint4 zv = *reinterpret_cast<const uint4 *>(z + i);
                  float2 z0 = unpack_bf16(zv.x), z1 = unpack_bf16(zv.y), z2 = unpack_bf16(zv.z), z3 = unpack_bf16(zv.w);
                  v[i + 0] *= gelu_grad_f(z0.x); v[i + 1] *= gelu_grad_f(z0.y);
                  v[i + 2] *= gelu_grad_f(z1.x); v[i + 3] *= gelu_grad_f(z1.y);
                  v[i + 4] *= gelu_grad_f(z2.x); v[i + 5] *= gelu_grad_f(z2.y);
                  v[i + 6] *= gelu_grad_f(z3.x); v[i + 7] *= gelu_grad_f(z3.y);
                }
              } else {
#pragma unroll
                for (int i = 0; i < 64; ++i)
                  if (gn0 + i < p.N) v[i] *= gelu_grad_f(__bfloat162float(z[i]));
              }
            }
          }
          uint32_t w[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) w[i] = pack_bf16(v[2 * i], v[2 * i + 1]);
          if (EPI == EPI_STORE_BF16 && p.scatter) {
            // the warp's 32-row box lies inside one owner's rows (scatter_rows % 32 == 0): push it into that
            // rank's slot over NVLink; boxes past M (last m-tile) are not stored
            if (grow0 < p.M) {
              const int q = grow0 / p.scatter_rows;
              stage_store(p.scatter + q, w, gn0, p.scatter_row0 + grow0 - q * p.scatter_rows);
            }
          } else {
            stage_store(&tmO, w, gn0, grow0);
          }
          if constexpr (EPI == EPI_BIAS_GELU) {
#pragma unroll
            for (int i = 0; i < 32; ++i) w[i] = pack_bf16(gelu_f(v[2 * i]), gelu_f(v[2 * i + 1]));
            stage_store(&tmO2, w, gn0, grow0);
          }
        }
      }
      const int next = tile + 2 * ncl;
      if (EPI == EPI_ACC_F32 && next < ntiles) {
        tc_fence_before();
        preload(next, buf);
      }
      release(buf);
    }
    if (lane == 0) tma_store_wait<0>();
    __syncwarp();
  }
  tc_fence_before();
  if constexpr (CG == 2)
    cluster_sync();
  else
    __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    if constexpr (CG == 2)
      tmem_dealloc2<C::TMEM_COLS>(tmem_base);
    else
      tmem_dealloc<C::TMEM_COLS>(tmem_base);
  }
}

__device__ int g_test_tile_ctr = 0;  // dynamic-schedule counter of the test entry points (serial use)

// ------------------------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2-D bf16 tensor [rows, cols] (cols contiguous, row stride ld elements), box {64 cols, box_rows}.
static bool make_map(CUtensorMap *m, const void *ptr, int rows, int cols, int ld, int box_rows) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {64u, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1u, 1u};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

cudaError_t gemm_store_map(void *map, const void *ptr, int rows, int cols, int ld) {
  return make_map(reinterpret_cast<CUtensorMap *>(map), ptr, rows, cols, ld, 32) ? cudaSuccess
                                                                               : cudaErrorInvalidValue;
}

struct Maps {
  CUtensorMap a, b, o, o2;  // operands; bf16 outputs (TMA-store boxes of 64 cols x 32 rows)
};

int gemm_num_sms() {
  static int n[MAX_DEV] = {};
  const int dev = cur_device();
  if (!n[dev]) cudaDeviceGetAttribute(&n[dev], cudaDevAttrMultiProcessorCount, dev);
  return n[dev];
}

template <int CG, int BN, bool A_MN, bool B_MN, int EPI, int SMEM_KB = (CG == 2 ? 160 : 192)>
static cudaError_t launch(const GemmArgs &a, const Maps &mp, const EpiParams &p,
                          cudaStream_t st) {
  using C = GemmCfg<CG, BN, SMEM_KB>;
  auto kern = gemm_kernel<CG, BN, A_MN, B_MN, EPI, SMEM_KB>;
  static bool attr[MAX_DEV] = {};
  const int dev = cur_device();
  if (!attr[dev]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr[dev] = true;
  }
  const int ntiles = ((a.M + BM * CG - 1) / (BM * CG)) * ((a.N + BN - 1) / BN);
  int clusters = (a.max_ctas > 0 ? a.max_ctas : gemm_num_sms()) / CG;
  if (clusters > ntiles) clusters = ntiles;
  if (clusters < 1) clusters = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(clusters * CG);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = CG;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, mp.a, mp.b, mp.o, mp.o2, p);
}

template <int CG, int BN, int KB>
static cudaError_t dispatch(const GemmArgs &a, const Maps &mp, const EpiParams &p,
                           cudaStream_t st) {
  if (!a.a_mn && !a.b_mn) {
    switch (a.epi) {
      case EPI_STORE_BF16: return launch<CG, BN, false, false, EPI_STORE_BF16, KB>(a, mp, p, st);
      case EPI_BIAS_BF16: return launch<CG, BN, false, false, EPI_BIAS_BF16, KB>(a, mp, p, st);
      case EPI_BIAS_GELU: return launch<CG, BN, false, false, EPI_BIAS_GELU, KB>(a, mp, p, st);
    }
  } else if (!a.a_mn && a.b_mn) {
    if (BN == 192) return cudaErrorNotSupported;  // MN-major B stages 64-wide chunks per CTA
    switch (a.epi) {
      case EPI_STORE_BF16: return launch<CG, BN, false, true, EPI_STORE_BF16, KB>(a, mp, p, st);
      case EPI_GELU_BWD: return launch<CG, BN, false, true, EPI_GELU_BWD, KB>(a, mp, p, st);
    }
  } else if (a.a_mn && a.b_mn) {
    if (BN == 192) return cudaErrorNotSupported;
    if (a.epi == EPI_ACC_F32) return launch<CG, BN, true, true, EPI_ACC_F32, KB>(a, mp, p, st);
  }
  return cudaErrorNotSupported;
}

// Tile width minimising the persistent schedule's makespan: ceil(tiles / clusters) waves of a
// tile costing ~ (BN + 32) (fixed per-tile overhead).  Never depends on M's split into sub-batches
// in a way that changes reduction order (tiling in N never does).
static int pick_bn(const GemmArgs &a, int cg) {
  if (a.N <= 128) return 128;
  if (cg != 2 || a.b_mn || a.a_mn) return 256;
  const int clusters = (a.max_ctas > 0 ? a.max_ctas : gemm_num_sms()) / 2;
  const int tm = (a.M + 255) / 256;
  int best = 256;
  double best_cost = 1e30;
  const int cands[] = {256, 192, 128};
  for (int bn : cands) {
    const long tiles = (long)tm * ((a.N + bn - 1) / bn);
    const double cost = (double)((tiles + clusters - 1) / clusters) * (bn + 32);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = bn;
    }
  }
  return best;
}

// Raster band height (tile_coords): 8 m-tiles.  Measured (profiles/r02/gemm_raster.txt): bands spanning all of
// M or N to keep the smaller operand L2-resident moved MORE DRAM bytes (the ~100 MB operand does not survive
// the streamed one and the fp32 accumulator tiles) and lowered the power-capped clock.
static int pick_group_m(const GemmArgs &a, int cg) {
  const int tiles_m = (a.M + BM * cg - 1) / (BM * cg);
  static int env = -2;
  if (env == -2) {
    const char *e = getenv("MERAK_GEMM_GROUP_M");  // measurement override: 0 = auto
    env = e ? atoi(e) : 0;
  }
  if (env > 0) return env < tiles_m ? env : tiles_m;
  return tiles_m < 8 ? tiles_m : 8;
}

static int gemm_cg() {
  static int cg = 0;
  if (!cg) {
    const char *e = getenv("MERAK_GEMM_CG");
    cg = (e && atoi(e) == 1) ? 1 : 2;
  }
  return cg;
}

template <int CG, int BN, int KB>
static cudaError_t preload_cfg() {
  const void *ks[] = {
      (const void *)gemm_kernel<CG, BN, false, false, EPI_STORE_BF16, KB>,
      (const void *)gemm_kernel<CG, BN, false, false, EPI_BIAS_BF16, KB>,
      (const void *)gemm_kernel<CG, BN, false, false, EPI_BIAS_GELU, KB>,
      (const void *)gemm_kernel<CG, BN, false, true, EPI_STORE_BF16, KB>,
      (const void *)gemm_kernel<CG, BN, false, true, EPI_GELU_BWD, KB>,
      (const void *)gemm_kernel<CG, BN, true, true, EPI_ACC_F32, KB>};
  for (const void *k : ks) {
    cudaError_t e = touch_kernel(k);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t gemm_preload() {
  cudaError_t e;
  if ((e = preload_cfg<2, 256, 160>()) != cudaSuccess) return e;
  if ((e = preload_cfg<2, 192, 160>()) != cudaSuccess) return e;
  if ((e = preload_cfg<2, 128, 160>()) != cudaSuccess) return e;
  if ((e = preload_cfg<2, 256, 192>()) != cudaSuccess) return e;
  if ((e = preload_cfg<2, 192, 192>()) != cudaSuccess) return e;
  if ((e = preload_cfg<2, 128, 192>()) != cudaSuccess) return e;
  if ((e = preload_cfg<1, 256, 192>()) != cudaSuccess) return e;
  return preload_cfg<1, 128, 192>();
}

cudaError_t gemm(const GemmArgs &a, cudaStream_t st) {
  if (a.M <= 0 || a.N <= 0 || a.K <= 0) return cudaErrorInvalidValue;
  const int cg = gemm_cg();
  // measured: 256-wide tiles beat 192/128 on every layer shape despite the last-wave loss
  // (4096x4800x1600: 1181 vs 991 TFLOP/s), so the wave-quantisation heuristic is off by default
  int BN = (a.epi >= 5 || !getenv("MERAK_GEMM_PICK_BN")) ? (a.N > 128 ? 256 : 128) : pick_bn(a, cg);
  if (const char *fb = getenv("MERAK_GEMM_BN")) {  // microbenchmark override (read per call)
    const int v = atoi(fb);
    if (v == 128 || v == 256 || (v == 192 && !a.a_mn && !a.b_mn)) BN = v;
  }
  const int bnc = BN / cg;  // B rows staged per CTA
  Maps mp;
  // A: K-major stored [M, K]; MN-major stored [K, M]
  bool ok = a.a_mn ? make_map(&mp.a, a.A, a.K, a.M, a.lda, BK) : make_map(&mp.a, a.A, a.M, a.K, a.lda, BM);
  ok = ok && (a.b_mn ? make_map(&mp.b, a.B, a.K, a.N, a.ldb, BK) : make_map(&mp.b, a.B, a.N, a.K, a.ldb, bnc));
  // bf16 outputs [M, N] (row stride ldo / ldo2) stored by TMA in boxes of 64 cols x 32 rows
  const bool bf16_out = a.epi != EPI_ACC_F32 && a.epi != 5;
  ok = ok && (bf16_out ? make_map(&mp.o, a.out, a.M, a.N, a.ldo, 32) : true);
  ok = ok && (a.epi == EPI_BIAS_GELU ? make_map(&mp.o2, a.out2, a.M, a.N, a.ldo2, 32) : true);
  if (!bf16_out) mp.o = mp.a;
  if (a.epi != EPI_BIAS_GELU) mp.o2 = mp.o;
  if (!ok) return cudaErrorInvalidValue;
  EpiParams p;
  p.M = a.M; p.N = a.N; p.K = a.K; p.epi = a.epi;
  p.out = (__nv_bfloat16 *)a.out; p.ldo = a.ldo;
  p.out2 = (__nv_bfloat16 *)a.out2; p.ldo2 = a.ldo2;
  p.bias = (const __nv_bfloat16 *)a.bias;
  p.aux = (const __nv_bfloat16 *)a.aux; p.ld_aux = a.ld_aux;
  p.out32 = a.out32; p.ld32 = a.ld32;
  p.db32 = a.db32;
  p.tile_ctr = a.tile_ctr;
  p.group_m = pick_group_m(a, cg);
  {  // L2 eviction priorities (measurement switch MERAK_GEMM_HINT="abc", digits 0 none / 1 first / 2 last)
    static int hint = -1;
    if (hint < 0) {
      const char *e = getenv("MERAK_GEMM_HINT");
      hint = (e && strlen(e) == 3) ? (e[0] - '0') * 100 + (e[1] - '0') * 10 + (e[2] - '0') : 0;
    }
    p.hint_a = hint / 100 % 10; p.hint_b = hint / 10 % 10; p.hint_c = hint % 10;
    if (a.epi != EPI_ACC_F32) p.hint_c = 0;
  }
  if (!p.tile_ctr) {  // test entry points: MERAK_GEMM_DYN=1 selects the dynamic schedule on a global counter
    const char *e = getenv("MERAK_GEMM_DYN");
    if (e && atoi(e) == 1) {
      void *ptr = nullptr;
      if (cudaGetSymbolAddress(&ptr, g_test_tile_ctr) != cudaSuccess) return cudaErrorInvalidValue;
      p.tile_ctr = reinterpret_cast<int *>(ptr);
    }
  }
  p.n_main = a.db32 ? a.N - 1 : a.N;
  p.scatter = reinterpret_cast<const CUtensorMap *>(a.scatter); p.scatter_row0 = a.scatter_row0; p.scatter_rows = a.scatter_rows;
  if (a.scatter && (a.epi != EPI_STORE_BF16 || a.scatter_rows <= 0 || a.scatter_rows % 32 != 0 ||
                    a.M % a.scatter_rows != 0))
    return cudaErrorInvalidValue;
  if (cg == 2 && a.epi >= 5 && !a.a_mn && !a.b_mn) {  // microbenchmark-only variants
    if (a.epi == 5) return launch<2, 256, false, false, 5>(a, mp, p, st);            // no stores
    if (a.epi == 6) return launch<2, 256, false, false, EPI_STORE_BF16, 192>(a, mp, p, st);  // 6 stages
    return cudaErrorNotSupported;
  }
  if (cg == 2) {
    // deep ring (192 KB) unless kernels on the communication stream must co-reside (smem_kb hint)
    if (a.smem_kb == 160) {
      switch (BN) {
        case 256: return dispatch<2, 256, 160>(a, mp, p, st);
        case 192: return dispatch<2, 192, 160>(a, mp, p, st);
        default: return dispatch<2, 128, 160>(a, mp, p, st);
      }
    }
    switch (BN) {
      case 256: return dispatch<2, 256, 192>(a, mp, p, st);
      case 192: return dispatch<2, 192, 192>(a, mp, p, st);
      default: return dispatch<2, 128, 192>(a, mp, p, st);
    }
  }
  return BN == 256 ? dispatch<1, 256, 192>(a, mp, p, st) : dispatch<1, 128, 192>(a, mp, p, st);
}

}  // namespace mk
