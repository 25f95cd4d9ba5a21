// gemm_tc2.cu -- 2-CTA (cta_group::2) variant of the tcgen05 grouped GEMM (see gemm_tc.cu for
// the GEMM table).  A CTA pair (cluster of 2 on one TPC) computes a 256 x BN tile: CTA r holds
// A rows [128r, 128r+128) and B columns [BN/2 r, BN/2 (r+1)) in its shared memory; the leader
// (r = 0) issues tcgen05.mma.cta_group::2 (M = 256) which reads both CTAs' operands and writes
// each CTA's 128 x BN accumulator into its own TMEM.  Per SM this halves the B bytes per MMA
// (32 KB per 64-deep k-block instead of 48 KB), so the same shared memory holds 6 stages
// instead of 4 -- the TMA-latency slack that the 1-CTA kernel lacks at K = 1024.
//
// Barriers: full[s] lives in the leader and collects both CTAs' TMA bytes (2-SM TMA form);
// empty[s] and tfull[a] live in both CTAs and are signalled by multicast tcgen05.commit;
// tempty[a] lives in the leader and collects one arrive per epilogue warp of both CTAs.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "gemm_tc_impl.cuh"
#include "tc_common.cuh"

namespace moe {

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_rank(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* b, uint32_t parity) {
  uint32_t addr = smem_u32(b);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAITC_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_2sm(void* dst, const CUtensorMap* map,
                                                uint32_t bar_cluster, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar_cluster)
      : "memory");
}
// 4 rows (r0..r3) x box-width columns starting at column c0, into 4 consecutive 128-byte rows
// of shared memory (swizzled like rows of a tile box); bytes land on the leader's barrier.
__device__ __forceinline__ void tma_gather4_2sm(uint32_t dst, const CUtensorMap* map,
                                                uint32_t bar_cluster, int c0, int4 r) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile::gather4"
      ".mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w),
      "r"(bar_cluster)
      : "memory");
}
// x rows of expert slots [s0, s0 + 4) (slot s of the region at `base`): token_of_slot / k, or
// `oob` (zero fill) for slots >= kept.  base and s0 are multiples of 4 (16-byte load).
__device__ __forceinline__ int4 gather_rows4(const int32_t* tos, int base, int s0, int kept,
                                             int k, int oob) {
  int4 v = make_int4(oob, oob, oob, oob);
  if (s0 < kept) {
    v = __ldg(reinterpret_cast<const int4*>(tos + base + s0));
    if (k != 1) { v.x /= k; v.y /= k; v.z /= k; v.w /= k; }
    if (s0 + 1 >= kept) v.y = oob;
    if (s0 + 2 >= kept) v.z = oob;
    if (s0 + 3 >= kept) v.w = oob;
  }
  return v;
}
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void tc_mma2(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                        uint32_t accum) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, {%5, %5, %5, %5, %5, %5, %5, %5}, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accum), "r"(0u)
      : "memory");
}
__device__ __forceinline__ void tc_commit2_mc(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

// instruction descriptor for M = 256 (cta_group::2)
__host__ __device__ constexpr uint32_t make_idesc2(int n, int a_mn, int b_mn, int m = 256) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

constexpr int TC2_M = 256;

// Epilogue staging: one 32 x 32 bf16 box (2 KB, 64-byte swizzle) per epilogue warp, written
// to C by TMA (cp.async.bulk.tensor store): whole 64-byte row segments instead of one 16-byte
// piece per lane and row, and asynchronous, so the warp moves on to its next TMEM chunk.
constexpr int TC2_STG_BYTES = 32 * 32 * 2;
#ifndef MOE_TC2_NBUF
#define MOE_TC2_NBUF 1
#endif
constexpr int TC2_NBUF = MOE_TC2_NBUF;  // staging buffers per epilogue warp

template <int KIND, int BN, int STAGES>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TC_THREADS, 1)
    tc_gemm2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmA2,
                    const __grid_constant__ CUtensorMap tmB2, TcParams p) {
  pdl_enter(p.nowait);  // PDL: predecessor complete + visible, unless nowait (common.cuh)
  using Tr = KindTraits<KIND>;
  constexpr int BNH = BN / 2;                    // B columns held by each CTA
  constexpr int A_BYTES = TC_BM * TC_BK * 2;     // 16 KB: this CTA's 128 rows
  constexpr int B_BYTES = BNH * TC_BK * 2;
  constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr uint32_t IDESC = make_idesc2(BN, Tr::a_mn, Tr::b_mn);
  constexpr uint32_t IDESC_H = make_idesc2(BN, Tr::a_mn, Tr::b_mn, 128);
  // The last m-tile of an expert with at most 128 valid rows runs as an M = 128 MMA over the
  // pair (64 rows per CTA): with dynamic capacities (no drops) many experts hold just over a
  // multiple of 256 rows, and a full 256-row tile would be mostly padding.
  auto half_tile = [&](int e, int mt) {
    return !Tr::kgroup && p.half_tiles && p.kept[e] - mt * TC2_M <= TC_BM;
  };
  constexpr int EPI_WARPS = TC_EPI_THREADS / 32;
  const bool fuse_bias = Tr::kgroup && p.bias_out != nullptr;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* bias_bar = tempty_bar + 2;                             // [STAGES]
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(bias_bar + STAGES);
  int32_t* s_prefix = reinterpret_cast<int32_t*>(s_tmem + 4);        // [n_local + 1]
  float* s_bias = reinterpret_cast<float*>(s_prefix + MOE_MAX_E + 4);  // [4][128]
  uint8_t* s_stg = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(s_bias + 4 * 128) + 1023) & ~uintptr_t(1023));  // [8][2 KB]
  // DGRAD_A db1 column sums: [tile parity][column half][row quarter][BN / 2]
  float* s_red = reinterpret_cast<float*>(s_stg + 8 * TC2_NBUF * TC2_STG_BYTES);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cluster_rank();
  const bool leader = crank == 0;
  const int n_local = p.n_local;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  if (warp == 3 && !Tr::kgroup) {  // prefix of ceil(kept / 256) m-tiles (warp scan)
    int carry = 0;
    for (int base = 0; base < n_local; base += 32) {
      const int e = base + lane;
      int v = e < n_local ? (p.kept[e] + TC2_M - 1) / TC2_M : 0;
      int incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (e < n_local) s_prefix[e] = carry + incl - v;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) s_prefix[n_local] = carry;
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    if (KIND == TC_DGRAD_X && p.nkx) {
      prefetch_tmap(&tmA2);
      prefetch_tmap(&tmB2);
    }
    prefetch_tmap(&tmC);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);   // multicast MMA commit
      mbar_init(&bias_bar[s], 2);    // the 2 bias warps are done reading the stage
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 2 * EPI_WARPS);      // one arrive per epilogue warp, both CTAs
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(s_tmem)),
                 "r"(2 * BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *s_tmem;

  const int NT = (p.N + BN - 1) / BN;
  const int MT = Tr::kgroup ? (p.M + TC2_M - 1) / TC2_M : 0;
  // tile schedule (identical in every role): round-robin or a contiguous chunk per pair
  int t_begin = pair, t_step = npairs, t_end = 0x7fffffff;
  if (p.sched != 0) {
    const int total = total_tiles<Tr::kgroup>(s_prefix, n_local, MT, NT);
    const int chunk = (total + npairs - 1) / npairs;
    t_begin = pair * chunk;
    t_end = min(total, t_begin + chunk);
    t_step = 1;
  }
  const bool nfast = p.sched == 1;

  if (warp == 0) {
    if ((KIND == TC_FWD1 || KIND == TC_WGRAD) && p.gtos != nullptr) {
      // ================ TMA producer with x-row gathers (N2, both CTAs, whole warp) ================
      // FWD1: lane l gathers A rows [4l, 4l+4) of this CTA's 128 rows (the same rows for every
      // k-block of the tile).  WGRAD: the B tile is 64 token rows x BNH columns in two 64-column
      // boxes; lane l gathers token rows [4(l%16), +4) of box l/16, indices one k-block ahead.
      int stage = 0;
      uint32_t phase = 0;
      const int sub = KIND == TC_FWD1 ? lane : (lane & 15);
      for (int t = t_begin; t < t_end; t += t_step) {
        int e, mt, nt;
        if (!decode_tile_ord<Tr::kgroup>(t, s_prefix, n_local, MT, NT, nfast, e, mt, nt)) break;
        // (a half tile uses rows [0, 64) of each CTA's A tile; the 128 loaded rows keep the
        // stage's transaction count)
        const int m0 = mt * TC2_M + (int)crank * (half_tile(e, mt) ? TC_BM / 2 : TC_BM);
        const int n0 = nt * BN + (int)crank * BNH;
        const int base = p.ct.base[e];
        const int kept = p.kept[e];
        const int nk = Tr::kgroup ? (kept + TC_BK - 1) / TC_BK : p.K / TC_BK;
        int4 rows = make_int4(0, 0, 0, 0), nxt = rows;
        if (KIND == TC_FWD1) rows = gather_rows4(p.gtos, base, m0 + 4 * sub, kept, p.gk, p.grows);
        else nxt = gather_rows4(p.gtos, base, 4 * sub, kept, p.gk, p.grows);
        for (int kb = 0; kb < nk; ++kb) {
          if (KIND == TC_WGRAD) {
            rows = nxt;
            if (kb + 1 < nk)
              nxt = gather_rows4(p.gtos, base, (kb + 1) * TC_BK + 4 * sub, kept, p.gk, p.grows);
          }
          mbar_wait(&empty_bar[stage], phase ^ 1);
          if (fuse_bias) mbar_wait(&bias_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          const uint32_t fb = mapa_rank(smem_u32(&full_bar[stage]), 0);
          const int k0 = kb * TC_BK;
          if (lane == 0) {
            if (leader) mbar_expect_tx(&full_bar[stage], 2 * STAGE_BYTES);
            if (KIND == TC_FWD1) {  // B = W1_e rows [n0, n0 + BNH), K-major
              tma_load_2d_2sm(sb, &tmB, fb, k0, e * p.N + n0);
            } else {                // A = dA^T tile, MN-major, two 64-column boxes
              tma_load_2d_2sm(sa, &tmA, fb, m0, base + k0);
              tma_load_2d_2sm(sa + 8192, &tmA, fb, m0 + 64, base + k0);
            }
          }
          __syncwarp();
          if (KIND == TC_FWD1)
            tma_gather4_2sm(smem_u32(sa) + lane * 512, &tmA, fb, k0, rows);
          else if ((lane >> 4) < BNH / 64)
            tma_gather4_2sm(smem_u32(sb) + (lane >> 4) * 8192 + sub * 512, &tmB, fb,
                            n0 + (lane >> 4) * 64, rows);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    } else if (lane == 0) {
      // ============================ TMA producer (both CTAs) ============================
      int stage = 0;
      uint32_t phase = 0;
      for (int t = t_begin; t < t_end; t += t_step) {
        int e, mt, nt;
        if (!decode_tile_ord<Tr::kgroup>(t, s_prefix, n_local, MT, NT, nfast, e, mt, nt)) break;
        const int m0 = mt * TC2_M + (int)crank * (half_tile(e, mt) ? TC_BM / 2 : TC_BM);  // A rows
        const int n0 = nt * BN + (int)crank * BNH;        // this CTA's B columns
        const int base = p.ct.base[e];
        const int nk = Tr::kgroup ? (p.kept[e] + TC_BK - 1) / TC_BK : p.K / TC_BK;
        if (p.pf_kb > 0 && t_step > 1) {
          // Warm L2 with the NEXT wave's B tile: only the pair that will be its first user
          // (m-tile 0) prefetches, so the other pairs of that wave hit L2 (one DRAM read).
          int e2, mt2, nt2;
          if (decode_tile_ord<Tr::kgroup>(t + t_step, s_prefix, n_local, MT, NT, nfast, e2, mt2,
                                          nt2) && mt2 == 0) {
            const int n2 = nt2 * BN + (int)crank * BNH;
            const int nk2 = Tr::kgroup ? (p.kept[e2] + TC_BK - 1) / TC_BK : p.K / TC_BK;
            const int npf = nk2 < p.pf_kb ? nk2 : p.pf_kb;
            for (int kb = 0; kb < npf; ++kb) {
              if (Tr::b_mn) {
                const int krow = Tr::kgroup ? p.ct.base[e2] + kb * TC_BK : e2 * p.K + kb * TC_BK;
                for (int j = 0; j < BNH / 64; ++j) tma_prefetch_2d(&tmB, n2 + j * 64, krow);
              } else {
                tma_prefetch_2d(&tmB, kb * TC_BK, e2 * p.N + n2);
              }
            }
          }
        }
        const int nkt = nk + (KIND == TC_DGRAD_X ? p.nkx : 0);
        for (int kb = 0; kb < nkt; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          // the bias warps observe every use of every stage (in lockstep with empty[s], so
          // parities cannot alias); the stage is refilled only after they released it
          if (fuse_bias) mbar_wait(&bias_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          const uint32_t fb = mapa_rank(smem_u32(&full_bar[stage]), 0);
          if (leader) mbar_expect_tx(&full_bar[stage], 2 * STAGE_BYTES);
          const int k0 = kb * TC_BK;
          if (KIND == TC_DGRAD_X && kb >= nk) {  // gate term: [hi|lo](dl) rows x [W_g ; W_g]
            const int kx = kb - nk;
            tma_load_2d_2sm(sa, &tmA2, fb, kx * TC_BK, base + m0);
#pragma unroll
            for (int j = 0; j < BNH / 64; ++j)
              tma_load_2d_2sm(sb + j * 8192, &tmB2, fb, n0 + j * 64, (kx % p.nbx) * TC_BK);
          } else {
            if (Tr::a_mn) {
              tma_load_2d_2sm(sa, &tmA, fb, m0, base + k0);
              tma_load_2d_2sm(sa + 8192, &tmA, fb, m0 + 64, base + k0);
            } else {
              tma_load_2d_2sm(sa, &tmA, fb, k0, base + m0);
            }
            if (Tr::b_mn) {
              const int krow = Tr::kgroup ? base + k0 : e * p.K + k0;
#pragma unroll
              for (int j = 0; j < BNH / 64; ++j)
                tma_load_2d_2sm(sb + j * 8192, &tmB, fb, n0 + j * 64, krow);
            } else {
              tma_load_2d_2sm(sb, &tmB, fb, k0, e * p.N + n0);
            }
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ============================ MMA issuer (leader only) ============================
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = t_begin; t < t_end; t += t_step, ++it) {
        int e, mt, nt;
        if (!decode_tile_ord<Tr::kgroup>(t, s_prefix, n_local, MT, NT, nfast, e, mt, nt)) break;
        const int acc = it & 1;
        const int nk = (Tr::kgroup ? (p.kept[e] + TC_BK - 1) / TC_BK : p.K / TC_BK) +
                       (KIND == TC_DGRAD_X ? p.nkx : 0);
        mbar_wait_cluster(&tempty_bar[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        const uint32_t idesc = half_tile(e, mt) ? IDESC_H : IDESC;
        // token-K GEMMs (weight gradients): the last k-block issues only the 16-deep MMAs
        // that hold kept tokens (rows past kept are zero pads; skipping them adds nothing)
        const int klast = Tr::kgroup && !p.no_ktrim ? (p.kept[e] - (nk - 1) * TC_BK + 15) / 16
                                                    : TC_BK / 16;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t sb = sa + A_BYTES;
          const int nsub = kb == nk - 1 ? klast : TC_BK / 16;
#pragma unroll
          for (int k = 0; k < TC_BK / 16; ++k) {
            if (k >= nsub) break;
            uint64_t da = Tr::a_mn ? umma_desc(sa + k * 2048, 8192, 1024)
                                   : umma_desc(sa + k * 32, 16, 1024);
            uint64_t db = Tr::b_mn ? umma_desc(sb + k * 2048, 8192, 1024)
                                   : umma_desc(sb + k * 32, 16, 1024);
            tc_mma2(tmem_d, da, db, idesc, (kb | k) != 0);
          }
          tc_commit2_mc(&empty_bar[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        tc_commit2_mc(&tfull_bar[acc]);
      }
    }
    __syncwarp();
  } else if (warp == 2 || warp == 3) {
    if (fuse_bias) {
      // ====================== bias-gradient warps (WGRAD, nt == 0 tiles) ======================
      // db[e][m] = sum over kept tokens of A[t, m]; this CTA's A^T tile (2 boxes of 64 m x 64
      // tokens, 128B swizzle: chunk c of token row kk stored at c ^ (kk & 7)) is summed from
      // shared memory after the MMA has consumed the stage (empty[s] completes in both CTAs
      // via the multicast commit); the producer waits for bias_bar[s] before refilling it.
      // Thread b (0..63): 16-byte chunk cb = b % 16 (box cb/8, chunk cb%8),
      // token rows [16 g, 16 g + 16) with g = b / 16; fixed-order fp32 sums, then a fixed
      // 4-way reduction over g through shared memory: deterministic.
      const int b = (warp - 2) * 32 + lane;
      const int cb = b & 15, g = b >> 4;
      const int bj = cb >> 3, bc = cb & 7;
      int stage = 0;
      uint32_t phase = 0;
      for (int t = t_begin; t < t_end; t += t_step) {
        int e, mt, nt;
        if (!decode_tile_ord<Tr::kgroup>(t, s_prefix, n_local, MT, NT, nfast, e, mt, nt)) break;
        const int nk = (p.kept[e] + TC_BK - 1) / TC_BK;
        float a8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) a8[i] = 0.f;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&empty_bar[stage], phase);
          if (nt == 0) {
            const uint8_t* box = smem + stage * STAGE_BYTES + bj * 8192;
#pragma unroll 4
            for (int kk = g * 16; kk < g * 16 + 16; ++kk) {
              const uint4 u = *reinterpret_cast<const uint4*>(box + kk * 128 + ((bc ^ (kk & 7)) << 4));
              float f8[8];
              unpack(u, f8, __nv_bfloat16());
#pragma unroll
              for (int i = 0; i < 8; ++i) a8[i] += f8[i];
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&bias_bar[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (nt == 0) {
#pragma unroll
          for (int i = 0; i < 8; ++i) s_bias[g * 128 + cb * 8 + i] = a8[i];
          asm volatile("bar.sync 1, 64;" ::: "memory");
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int ml = b * 2 + q;
            float v = s_bias[ml] + s_bias[128 + ml] + s_bias[256 + ml] + s_bias[384 + ml];
            const int m = mt * TC2_M + (int)crank * TC_BM + ml;
            if (m < p.M) {
              __nv_bfloat16* dst = p.bias_out + (size_t)e * p.M + m;
              if (p.accumulate) v += __bfloat162float(*dst);
              *dst = __float2bfloat16_rn(v);
            }
          }
          asm volatile("bar.sync 1, 64;" ::: "memory");
        }
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ============================ epilogue (both CTAs) ============================
    const int q = warp & 3;
    const int half = (warp - 4) >> 2;
    constexpr int CH = BN / 64;  // 32-column chunks per warp (full tile)
    const uint32_t tempty_leader0 = mapa_rank(smem_u32(&tempty_bar[0]), 0);
    uint8_t* stg0 = s_stg + (warp - 4) * TC2_NBUF * TC2_STG_BYTES;
    int nbox = 0;
    int it = 0;
    for (int t = t_begin; t < t_end; t += t_step, ++it) {
      int e, mt, nt;
      if (!decode_tile_ord<Tr::kgroup>(t, s_prefix, n_local, MT, NT, nfast, e, mt, nt)) break;
      const int acc = it & 1;
      const int m0 = mt * TC2_M, n0 = nt * BN;
      // Half tile (M = 128 over the pair: 64 rows per CTA): the accumulator of a CTA's 64 rows
      // holds columns [0, BN/2) in TMEM lanes 0..63 and [BN/2, BN) in lanes 64..127, both in
      // TMEM columns [0, BN/2), so lane quarter q drains rows 32 (q & 1) + lane of column half
      // q >> 1, and the warp's `half` splits that into two BN/4 blocks (CH/2 chunks).
      const bool ht = half_tile(e, mt);
      const int rpc = ht ? TC_BM / 2 : TC_BM;                    // rows per CTA in this tile
      const int blk_row = m0 + (int)crank * rpc + (ht ? (q & 1) * 32 : q * 32);  // warp-uniform
      const int row = blk_row + lane;
      const int nch = ht ? CH / 2 : CH;                             // chunks this warp drains
      const int cbase = ht ? (q >> 1) * (BN / 2) + half * (BN / 4) : half * (BN / 2);
      const int tbase = ht ? half * (BN / 4) : half * (BN / 2);    // TMEM column of chunk 0
      const bool zero_acc = Tr::kgroup && p.kept[e] == 0;
      const int Me = Tr::kgroup ? p.M : p.kept[e];
      const bool row_ok = row < Me;
      // padding rows written as zeros (token-K GEMMs read up to roundup(kept, 64))
      const bool row_pad = !Tr::kgroup && !row_ok && row < ((Me + 63) & ~63);
      __nv_bfloat16* crow;
      if (Tr::kgroup)
        crow = p.C + ((size_t)e * p.M + row) * p.N;
      else
        crow = p.C + (size_t)(p.ct.base[e] + row) * p.ldc;
      // Side inputs of the whole tile (bias, H mask, old gradient) are fetched BEFORE waiting
      // for the accumulator, so their DRAM/L2 latency overlaps this tile's MMAs.
      uint4 pre[CH][4];
      uint32_t mbits[CH];
      uint32_t mout[CH];
#pragma unroll
      for (int cc = 0; cc < CH; ++cc) mout[cc] = 0u, mbits[cc] = ~0u;
      const int mask_ld = p.N >> 5;
      uint32_t* mrow = p.mask ? p.mask + (size_t)(p.ct.base[e] + row) * mask_ld : nullptr;
      if (KIND == TC_DGRAD_A && row_ok && !(p.dbg & 4)) {  // relu' mask bits written by FWD1
#pragma unroll
        for (int cc = 0; cc < CH; ++cc)
          if (cc < nch) mbits[cc] = mrow[((n0 + cbase) >> 5) + cc];
      }
      // N2 combine fusion (k = 1): this row's token and gate weight
      int ytok = -1;
      float yw = 0.f;
      if (KIND == TC_FWD2 && p.y != nullptr && !p.comb2 && row_ok) {
        ytok = p.gtos[p.ct.base[e] + row];
        yw = p.wt[ytok];
      }
      if (KIND == TC_DGRAD_X && p.dxo != nullptr && row_ok) ytok = p.gtos[p.ct.base[e] + row];
      // row-scatter stores (the staged box leaves as row segments to per-row destinations):
      //  * fused dispatch backward: dx row of the token;
      //  * peer EP return (N1): the (token, choice) row of the token owner's O / dX return
      //    buffer, in that rank's window over NVLink -- the exchange rides on the epilogue
      __nv_bfloat16* rdst = nullptr;
      if (KIND == TC_DGRAD_X && p.dxo != nullptr && row_ok) rdst = p.dxo + (size_t)ytok * p.N;
      if ((KIND == TC_FWD2 || KIND == TC_DGRAD_X) && p.pret.nl != 0 && row_ok) {
        const int gp = p.gtos[p.ct.base[e] + row];  // global pair id t_g * k + r
        const int owner = (gp / p.gk) / p.tpr;
        const int lp = gp - owner * p.tpr * p.gk;
        char* b = nullptr;
#pragma unroll
        for (int j = 0; j < MOE_MAX_R; ++j)
          if (owner == j) b = p.pret.p[j];
        rdst = reinterpret_cast<__nv_bfloat16*>(b) + (size_t)lp * p.N;
      }
      const bool need_side = ((KIND == TC_FWD1 || KIND == TC_FWD2) && row_ok) ||
                             (KIND == TC_WGRAD && row_ok && p.accumulate);
      if (need_side) {
#pragma unroll
        for (int cc = 0; cc < CH; ++cc) {
          if (cc >= nch) continue;
          const int col0 = n0 + cbase + cc * 32;
          const __nv_bfloat16* src = (KIND == TC_FWD1 || KIND == TC_FWD2)
                                         ? p.bias + (size_t)e * p.N + col0
                                         : crow + col0;
#pragma unroll
          for (int i = 0; i < 4; ++i) pre[cc][i] = ld_v4(src + 8 * i);
        }
      }
      mbar_wait(&tfull_bar[acc], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem_base + acc * BN + ((uint32_t)(q * 32) << 16);
#pragma unroll
      for (int cc = 0; cc < CH; ++cc) {
        if (cc >= nch) continue;  // (warp-uniform)
        const int col0 = n0 + cbase + cc * 32;
        uint4* side = pre[cc];
        uint32_t r[32];
        if (!zero_acc) {
          tmem_ld32(taddr + tbase + cc * 32, r);
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) r[i] = 0u;
        }
        if (col0 >= p.N) continue;
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
        bool store = true;
        if (KIND == TC_FWD1 || KIND == TC_FWD2) {
          if (row_ok) {
#pragma unroll
            for (int i = 0; i < 32; i += 8) {
              float bb[8];
              unpack(side[i / 8], bb, __nv_bfloat16());
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                float x = v[i + j] + bb[j];
                v[i + j] = (KIND == TC_FWD1) ? (x > 0.f ? x : 0.f) : x;
              }
            }
          } else {
            store = (KIND == TC_FWD1) && row_pad;
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = 0.f;
          }
        } else if (KIND == TC_DGRAD_A) {
          if (row_ok) {
            const uint32_t mb = mbits[cc];
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = ((mb >> i) & 1u) ? v[i] : 0.f;
          } else {
            store = row_pad;
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = 0.f;
          }
        } else if (KIND == TC_DGRAD_X) {
          store = row_ok;
          if (p.dxo != nullptr && p.accumulate && ytok >= 0) {
            // dispatch backward (k = 1), accumulating: add the old dx before the one rounding
            const __nv_bfloat16* drow = p.dxo + (size_t)ytok * p.N + col0;
#pragma unroll
            for (int i = 0; i < 32; i += 8) {
              float o[8];
              unpack(ld_v4(drow + i), o, __nv_bfloat16());
#pragma unroll
              for (int j = 0; j < 8; ++j) v[i + j] += o[j];
            }
          }
        } else {  // WGRAD
          store = row_ok;
          if (row_ok && p.accumulate) {
#pragma unroll
            for (int i = 0; i < 32; i += 8) {
              float o[8];
              unpack(side[i / 8], o, __nv_bfloat16());
#pragma unroll
              for (int j = 0; j < 8; ++j) v[i + j] += o[j];
            }
          }
        }
        (void)store;
        // One 32-row box per warp (warp-uniform decision).  Boxes start 32-aligned inside a
        // 128-aligned region, so a box lies entirely below roundup(M_e, 64) or entirely above
        // it: padded kinds (FWD1, DGRAD_A) store boxes below roundup(M_e, 64) (rows >= M_e are
        // zeros), the others boxes below roundup(M_e, 32) (rows >= M_e: zeros, never read).
        bool box;
        const bool red_on = KIND == TC_DGRAD_A && p.bias_part != nullptr && !(p.dbg & 2);
        if (Tr::kgroup) box = blk_row < p.M;
        else if (KIND == TC_FWD1 || KIND == TC_DGRAD_A) box = blk_row < ((Me + 63) & ~63);
        else box = blk_row < Me;
        if (!Tr::kgroup && !row_ok) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = 0.f;
        }
        if (p.dbg & 1) box = false;
        if (red_on && !box && lane < 16)  // rows of this warp all past the padded end: zeros
          *reinterpret_cast<float2*>(s_red + (((it & 1) * 2 + half) * 4 + q) * (CH * 32) +
                                     cc * 32 + 2 * lane) = make_float2(0.f, 0.f);
        if (box) {
          uint4 pk[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) pk[i] = pack(v + 8 * i, __nv_bfloat16());
          uint8_t* stg = stg0 + (nbox++ % TC2_NBUF) * TC2_STG_BYTES;
          if (lane == 0) tma_store_wait_read<TC2_NBUF - 1>();  // this buffer's last box left
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 4; ++i)  // 64-byte swizzle: chunk i of row r at i ^ ((r >> 1) & 3)
            *reinterpret_cast<uint4*>(stg + lane * 64 + ((i ^ ((lane >> 1) & 3)) << 4)) = pk[i];
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          const bool rowstore = (KIND == TC_DGRAD_X && p.dxo != nullptr) ||
                                ((KIND == TC_FWD2 || KIND == TC_DGRAD_X) && p.pret.nl != 0);
          if (rowstore) {
            // 64-byte row segments (lane: row 8i + l/4, 16-byte chunk l%4) to the row's
            // destination from its lane: dx[t] = dX[row] + dl[t] W_g (fused dispatch
            // backward, one rounding) or the token owner's return row (peer EP)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int r = i * 8 + (lane >> 2), c = lane & 3;
              const unsigned long long dst = __shfl_sync(
                  0xffffffffu, reinterpret_cast<unsigned long long>(rdst), r);
              if (dst != 0ull)
                st_v4(reinterpret_cast<__nv_bfloat16*>(dst) + col0 + c * 8,
                      *reinterpret_cast<const uint4*>(stg + r * 64 + ((c ^ ((r >> 1) & 3)) << 4)));
            }
          }
          if (lane == 0 && !(p.dbg & 8) && !rowstore)
            tma_store_2d(&tmC, stg, col0,
                         (p.dbg & 16) ? (blk_row & 127)
                                      : (Tr::kgroup ? e * p.M + blk_row : p.ct.base[e] + blk_row));
          if (KIND == TC_DGRAD_A && red_on) {
            // db1 = sum over kept tokens of dA (the stored bf16 values, rows >= kept are 0):
            // column sums of this warp's 32 rows read back from the staged box.  Lane l sums
            // columns 2(l%16), 2(l%16)+1 over rows 2i + l/16 (conflict-free), then the two row
            // halves; parked in shared memory for the fixed-order quarter sum after the tile.
            const int cp = lane & 15, rh = lane >> 4;
            float s0 = 0.f, s1 = 0.f;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int r = 2 * i + rh;
              const uint32_t w = *reinterpret_cast<const uint32_t*>(
                  stg + r * 64 + (((cp >> 2) ^ ((r >> 1) & 3)) << 4) + (cp & 3) * 4);
              s0 += __uint_as_float(w << 16);
              s1 += __uint_as_float(w & 0xffff0000u);
            }
            s0 += __shfl_down_sync(0xffffffffu, s0, 16);
            s1 += __shfl_down_sync(0xffffffffu, s1, 16);
            if (lane < 16)
              *reinterpret_cast<float2*>(s_red + (((it & 1) * 2 + half) * 4 + q) * (CH * 32) +
                                         cc * 32 + 2 * cp) = make_float2(s0, s1);
          }
          if (KIND == TC_FWD2 && p.y != nullptr && !p.comb2) {
            // Alg. 1 l.8 for k = 1: y[t] = 0 + w O[row] from the stored (bf16) O, the same
            // arithmetic as the combine kernel (bitwise equal).  Staged in the box buffer once
            // the O store has read it, then written as 64-byte row segments of y.
            uint4 yk[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              float o[8];
              unpack(pk[i], o, __nv_bfloat16());
#pragma unroll
              for (int j = 0; j < 8; ++j) o[j] = fmaf(yw, o[j], 0.f);
              yk[i] = pack(o, __nv_bfloat16());
            }
            if (lane == 0) tma_store_wait_read<0>();
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 4; ++i)
              *reinterpret_cast<uint4*>(stg + lane * 64 + ((i ^ ((lane >> 1) & 3)) << 4)) = yk[i];
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int r = i * 8 + (lane >> 2), c = lane & 3;
              const int tok = __shfl_sync(0xffffffffu, ytok, r);
              if (tok >= 0)
                st_v4(p.y + (size_t)tok * p.N + col0 + c * 8,
                      *reinterpret_cast<const uint4*>(stg + r * 64 + ((c ^ ((r >> 1) & 3)) << 4)));
            }
            __syncwarp();
          }
          if (KIND == TC_FWD1) {  // bit j: the stored bf16 H is > 0 (relu output >= 0)
            uint32_t bits = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const uint32_t w4[4] = {pk[i].x, pk[i].y, pk[i].z, pk[i].w};
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const uint32_t ne = __vsetne2(w4[j], 0u);  // 0x0001 per nonzero half
                bits |= ((ne & 1u) | ((ne >> 15) & 2u)) << (8 * i + 2 * j);
              }
            }
            mout[cc] = bits;
          }
        }
      }
      if (KIND == TC_DGRAD_A && p.bias_part && !(p.dbg & 2)) {
        // fixed-order sum of the 4 row quarters of this column half -> one partial row per
        // (m-tile, CTA); s_red is double-buffered by tile parity, so one barrier per tile
        asm volatile("bar.sync %0, 128;" ::"r"(2 + half) : "memory");
        if (q == 0) {
          const float* rb = s_red + (((it & 1) * 2 + half) * 4) * (CH * 32);
          const size_t prow = (size_t)(s_prefix[e] + mt) * 2 + crank;
          if (!ht) {
#pragma unroll
            for (int j = 0; j < CH; ++j) {
              const int c = j * 32 + lane;
              const float sum = ((rb[c] + rb[CH * 32 + c]) + rb[2 * CH * 32 + c]) + rb[3 * CH * 32 + c];
              const int col = n0 + half * CH * 32 + c;
              if (col < p.N) p.bias_part[prow * p.N + col] = sum;
            }
          } else {
            // half tile: quarters 2g and 2g + 1 hold the two 32-row halves of column block g
#pragma unroll
            for (int g = 0; g < 2; ++g)
#pragma unroll
              for (int j = 0; j < CH / 2; ++j) {
                const int c = j * 32 + lane;
                const float sum = rb[(2 * g) * CH * 32 + c] + rb[(2 * g + 1) * CH * 32 + c];
                const int col = n0 + g * (BN / 2) + half * (BN / 4) + c;
                if (col < p.N) p.bias_part[prow * p.N + col] = sum;
              }
          }
        }
      }
      if (KIND == TC_FWD1 && mrow && (row_ok || row_pad)) {  // one vector store per thread
        uint32_t* mdst = mrow + ((n0 + cbase) >> 5);
        if (CH == 4 && !ht)
          *reinterpret_cast<uint4*>(mdst) = make_uint4(mout[0], mout[1 % CH], mout[2 % CH], mout[3 % CH]);
        else
#pragma unroll
          for (int cc = 0; cc < CH; ++cc)
            if (cc < nch) mdst[cc] = mout[cc];
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(tempty_leader0 + acc * 8);
      if (KIND == TC_FWD2 && p.comb2) {
        // Alg. 1 l.8 for k = 2 (O stored in (token, choice) order above):
        //   y[t] = 0 + w[t,0] O[t,0] + w[t,1] O[t,1]   (r order, kept pairs only)
        // -- the combine kernel's arithmetic on the stored bf16 O rows, so bitwise equal.  A
        // token's two rows come from different experts' tiles; per (token, column block of
        // this warp) a self-resetting counter elects the epilogue that finishes second (or the
        // only one, when the other pair was dropped) to read both rows back and write y.
        // Runs after the accumulator is released, so the next tile's MMAs are not delayed.
        constexpr int COLS = BN / 2;            // this warp's column block
        constexpr int VPL2 = COLS / 32;         // bf16 per lane: 4 (BN 256) or 2 (BN 128)
        const int cb0 = n0 + half * COLS;
        int tok = -1;
        bool both = false, mine = false;
        if (row_ok) {
          const int gp = p.gtos[p.ct.base[e] + row];
          tok = gp >> 1;
          both = p.slot2[(size_t)tok * 2 + ((gp & 1) ^ 1)] >= 0;
        }
        __threadfence();  // this warp's O row segments are visible before its counters
        __syncwarp();
        if (row_ok) {
          if (!both) {
            mine = true;
          } else {
            uint32_t* cnt = p.ycnt + (size_t)tok * p.ycb + cb0 / COLS;
            if (atomicAdd(cnt, 1u) == 1u) {
              mine = true;
              *cnt = 0u;  // both arrivals seen: ready for the next forward
            }
          }
        }
        __threadfence();  // acquire: the other epilogue's O rows before they are read
        uint32_t todo = __ballot_sync(0xffffffffu, mine);
        const __nv_bfloat16* otok = reinterpret_cast<const __nv_bfloat16*>(p.pret.p[0]);
        while (todo) {
          const int l = __ffs(todo) - 1;
          todo &= todo - 1;
          const int tt = __shfl_sync(0xffffffffu, tok, l);
          const int c = cb0 + lane * VPL2;
          float acc2[VPL2];
#pragma unroll
          for (int i = 0; i < VPL2; ++i) acc2[i] = 0.f;
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            if (p.slot2[(size_t)tt * 2 + r] < 0) continue;  // dropped pair: no contribution
            const float wr = p.wt[(size_t)tt * 2 + r];
            const __nv_bfloat16* src = otok + ((size_t)tt * 2 + r) * p.N + c;
            uint32_t u[VPL2 / 2];
            if (VPL2 == 4) {
              const uint2 v = __ldcg(reinterpret_cast<const uint2*>(src));
              u[0] = v.x;
              u[VPL2 / 2 - 1] = v.y;
            } else {
              u[0] = __ldcg(reinterpret_cast<const unsigned int*>(src));
            }
#pragma unroll
            for (int i = 0; i < VPL2 / 2; ++i) {
              acc2[2 * i] = fmaf(wr, __uint_as_float(u[i] << 16), acc2[2 * i]);
              acc2[2 * i + 1] = fmaf(wr, __uint_as_float(u[i] & 0xffff0000u), acc2[2 * i + 1]);
            }
          }
          uint32_t o[VPL2 / 2];
#pragma unroll
          for (int i = 0; i < VPL2 / 2; ++i) {
            const __nv_bfloat162 b2 = __floats2bfloat162_rn(acc2[2 * i], acc2[2 * i + 1]);
            o[i] = *reinterpret_cast<const uint32_t*>(&b2);
          }
          __nv_bfloat16* dst = p.y + (size_t)tt * p.N + c;
          if (VPL2 == 4)
            *reinterpret_cast<uint2*>(dst) = make_uint2(o[0], o[VPL2 / 2 - 1]);
          else
            *reinterpret_cast<uint32_t*>(dst) = o[0];
        }
      }
    }
  }
  if (warp >= 4 && lane == 0) tma_store_wait_all();
  tc_fence_before();
  cluster_sync_all();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(2 * BN));
  }
}

// ------------------------------------------------------------------------------ host side
template <int KIND, int BN>
static cudaError_t launch2(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c,
                           const CUtensorMap& a2, const CUtensorMap& b2, const TcParams& p,
                           int grid, cudaStream_t s) {
  constexpr int STAGES = (BN == 256) ? (TC2_NBUF > 1 ? 5 : 6) : 8;
  constexpr int STAGE_BYTES = (TC_BM + BN / 2) * TC_BK * 2;
  const size_t smem = (size_t)STAGES * STAGE_BYTES + 1024 + 512 + 4 * (MOE_MAX_E + 8) + 2048 +
                      1024 + 8 * TC2_NBUF * TC2_STG_BYTES +
                      (KIND == TC_DGRAD_A ? 2 * 2 * 4 * (BN / 2) * 4 : 0);
  auto kf = tc_gemm2_kernel<KIND, BN, STAGES>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  launch_pdl(kf, grid, TC_THREADS, smem, s, a, b, c, a2, b2, p);
  return cudaGetLastError();
}

cudaError_t launch_tc2_kind(int kind, int BN, const CUtensorMap& a, const CUtensorMap& b,
                            const CUtensorMap& c, const TcParams& p, int grid, cudaStream_t s,
                            const CUtensorMap* a2, const CUtensorMap* b2) {
  const CUtensorMap& A2 = a2 ? *a2 : a;
  const CUtensorMap& B2 = b2 ? *b2 : b;
#define K2(KD)                                                                         \
  case KD:                                                                             \
    return BN == 256 ? launch2<KD, 256>(a, b, c, A2, B2, p, grid, s)                   \
                     : launch2<KD, 128>(a, b, c, A2, B2, p, grid, s);
  switch (kind) {
    K2(TC_FWD1) K2(TC_FWD2) K2(TC_DGRAD_A) K2(TC_DGRAD_X) K2(TC_WGRAD)
    default: return cudaErrorInvalidValue;
  }
#undef K2
}

}  // namespace moe
