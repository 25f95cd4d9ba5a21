// gemm_tf32.cu -- the fp32 expert FFN GEMMs on tcgen05 tensor cores (split-tf32 products).
//
// The fp32 configurations (BASELINE c1 / c2, the paper's fp32 P100 runs) need
// fp32-level results (north star: 1e-5 relative; dl, a difference of nearly equal dw's,
// inherits the operands' error amplified).  tcgen05 `kind::tf32` multiplies operands with 10
// explicit mantissa bits, so each fp32 operand is split in shared memory into two tf32 terms
//     a = a0 + a1 + r,   a0 = rna_tf32(a),  a1 = rna_tf32(a - a0),  |r| <= 2^-22 |a|
// and every k-step issues four MMAs into TWO fp32 TMEM accumulators:
//     S += a1 b1;  S += a1 b0;  S += a0 b1;      P += a0 b0;      C = P + S (epilogue)
// The leading products accumulate alone in P (one accumulation per MMA-K of 8, the same count
// as a plain GEMM), the correction terms -- 2^-11 of the result -- in S, so S's own rounding
// is scaled down by 2^-11.  Per product the split leaves ~2^-21 |a||b|.  Measured on the fuzz
// sweep ("split-tf32"): one shared accumulator for all terms (3 MMAs, and a
// 3-way split with 6 MMAs) left 3-4e-6 relative error per GEMM -- the accumulator's rounding
// grows with the number of MMAs that add into it -- and pushed dl past 1e-5 on fuzz cases.
//
// Same grouping, layouts and epilogues as the bf16 1-CTA kernel (gemm_tc.cu):
//   kind      C (per local expert e)                       A major  B major  M rows
//   FWD1      H  = relu(X W1_e^T + b1_e)                   K        K        kept_e
//   FWD2      O  = H W2_e^T + b2_e                         K        K        kept_e
//   DGRAD_A   dA = (dO W2_e) * 1[H > 0] (over H)           K        MN       kept_e
//   DGRAD_X   dX = dA W1_e                                 K        MN       kept_e
//   WGRAD     dW = A^T B over kept_e tokens (+ fused db)   MN       MN       d_out / f
//
// Roles (512 threads): warp 0 TMA producer, warp 1 MMA issuer, warp 2 TMEM allocator, warp 3
// bias-gradient warp (WGRAD), warps 4..7 epilogue (TMEM lane quarters), warps 8..15 split the
// landed fp32 tiles (a0 in place, a1 in its own buffer) and signal the MMA warp.  Stage =
// {A0, A1 (128 x 32), B0, B1 (BN x 32)} fp32; K-major operands use the 128-byte swizzle,
// MN-major ones the 128-byte swizzle with 32-byte atoms (the only MN-major tf32 layout); the
// split is elementwise, so it is layout-agnostic.  TMEM: {P, S} x 2 (double buffer) x BN.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "gemm_tc.h"
#include "kernels.h"
#include "prof.h"
#include "tc_common.cuh"
#include "gemm_tc_impl.cuh"

namespace moe {

namespace {

constexpr int TF_BK = 32;            // fp32 elements per 128-byte smem row
constexpr int TF_THREADS = 512;
constexpr int TF_CONV_WARP0 = 8;     // warps 8..15 split the stages
constexpr int TF_CONV_THREADS = 256;

// kind::tf32 instruction descriptor: tf32 x tf32 -> fp32, M = 128, N = n
__host__ __device__ constexpr uint32_t make_idesc_tf32(int n, int a_mn, int b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

__device__ __forceinline__ void tc_mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db,
                                            uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accum)
      : "memory");
}

// UMMA smem descriptor of an MN-major 32-bit operand: layout type 1 (SWIZZLE_128B_BASE32B, the
// only MN-major layout tf32 supports): 128-byte MN rows, 32-byte granules XOR-swizzled with
// the K row (mod 4), written by TMA with CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B.  LBO = stride
// between 128-byte MN blocks, SBO = stride between 4-row K groups.
__device__ __forceinline__ uint64_t umma_desc_mn32(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)1 << 61;
  return d;
}

__device__ __forceinline__ float tf32_rna(float a) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(a));
  return __uint_as_float(r);
}

// split n16 16-byte vectors starting at `raw`: a0 in place, a1 at raw + off.  Shared-window
// addresses (ld / st.shared, not generic), every load of the thread's vectors issued first.
__device__ __forceinline__ void split_vecs(uint8_t* raw, int off, int n16, int tid) {
  constexpr int PER = 4;  // vectors per thread per batch
  const uint32_t base = smem_u32(raw);
  for (int i0 = tid; i0 < n16; i0 += PER * TF_CONV_THREADS) {
    float4 a[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      if (i0 + j * TF_CONV_THREADS >= n16) break;  // (uniform: n16 is a multiple of 256)
      const uint32_t ad = base + (uint32_t)(i0 + j * TF_CONV_THREADS) * 16u;
      asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                   : "=f"(a[j].x), "=f"(a[j].y), "=f"(a[j].z), "=f"(a[j].w) : "r"(ad));
    }
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      if (i0 + j * TF_CONV_THREADS >= n16) break;
      float4 h, m;
      h.x = tf32_rna(a[j].x); m.x = tf32_rna(a[j].x - h.x);
      h.y = tf32_rna(a[j].y); m.y = tf32_rna(a[j].y - h.y);
      h.z = tf32_rna(a[j].z); m.z = tf32_rna(a[j].z - h.z);
      h.w = tf32_rna(a[j].w); m.w = tf32_rna(a[j].w - h.w);
      const uint32_t ad = base + (uint32_t)(i0 + j * TF_CONV_THREADS) * 16u;
      asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(ad), "f"(h.x), "f"(h.y),
                   "f"(h.z), "f"(h.w) : "memory");
      asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(ad + (uint32_t)off),
                   "f"(m.x), "f"(m.y), "f"(m.z), "f"(m.w) : "memory");
    }
  }
}

template <int KIND, int BN, int STAGES>
__global__ void __launch_bounds__(TF_THREADS, 1)
    tf32_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     TcParams p) {
  pdl_enter(p.nowait);  // PDL: predecessor complete + visible, unless nowait (backward tail)
  using Tr = KindTraits<KIND>;
  constexpr int A_BYTES = TC_BM * TF_BK * 4;   // 16 KB
  constexpr int B_BYTES = BN * TF_BK * 4;
  constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;  // A0 A1, B0 B1
  constexpr uint32_t IDESC = make_idesc_tf32(BN, Tr::a_mn, Tr::b_mn);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* conv_bar = full_bar + STAGES;     // operand split done
  uint64_t* bias_bar = conv_bar + STAGES;     // WGRAD bias warp done with the raw A tile
  uint64_t* empty_bar = bias_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  int32_t* s_prefix = reinterpret_cast<int32_t*>(s_tmem + 4);   // [n_local + 1]
  const float* bias = reinterpret_cast<const float*>(p.bias);
  float* bias_out = reinterpret_cast<float*>(p.bias_out);
  float* Cbase = reinterpret_cast<float*>(p.C);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_local = p.n_local;
  for (int i = threadIdx.x; i <= n_local; i += blockDim.x)
    s_prefix[i] = Tr::kgroup ? 0 : p.mtile_prefix[i];
  const bool bias_warp = Tr::kgroup && bias_out != nullptr;
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&conv_bar[s], TF_CONV_THREADS / 32);
      mbar_init(&bias_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(s_tmem)),
                 "r"(4 * BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *s_tmem;

  const int NT = (p.N + BN - 1) / BN;
  const int MT = Tr::kgroup ? (p.M + TC_BM - 1) / TC_BM : 0;

  if (warp == 0) {
    if (lane == 0) {
      // ============================ TMA producer ============================
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x;; t += gridDim.x) {
        int e, mt, nt;
        if (!decode_tile<Tr::kgroup>(t, s_prefix, n_local, MT, NT, e, mt, nt)) break;
        const int m0 = mt * TC_BM, n0 = nt * BN;
        const int base = p.ct.base[e];
        const int nk = Tr::kgroup ? (p.kept[e] + TF_BK - 1) / TF_BK : p.K / TF_BK;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          uint8_t* sb = sa + 2 * A_BYTES;
          mbar_expect_tx(&full_bar[stage], A_BYTES + B_BYTES);
          const int k0 = kb * TF_BK;
          if (Tr::a_mn) {  // A^T tiles: {32 M, 32 K} boxes
#pragma unroll
            for (int j = 0; j < TC_BM / 32; ++j)
              tma_load_2d(sa + j * 4096, &tmA, &full_bar[stage], m0 + j * 32, base + k0);
          } else {         // A K-major: {32 K, 128 rows}
            tma_load_2d(sa, &tmA, &full_bar[stage], k0, base + m0);
          }
          if (Tr::b_mn) {
#pragma unroll
            for (int j = 0; j < BN / 32; ++j)
              tma_load_2d(sb + j * 4096, &tmB, &full_bar[stage], n0 + j * 32,
                          (Tr::kgroup ? base : e * p.K) + k0);
          } else {  // weight [N x K] of expert e: rows e*N + n
            tma_load_2d(sb, &tmB, &full_bar[stage], k0, e * p.N + n0);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      // ============================ MMA issuer ============================
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = blockIdx.x;; t += gridDim.x, ++it) {
        int e, mt, nt;
        if (!decode_tile<Tr::kgroup>(t, s_prefix, n_local, MT, NT, e, mt, nt)) break;
        const int acc = it & 1;
        const uint32_t aphase = (it >> 1) & 1;
        const int nk = Tr::kgroup ? (p.kept[e] + TF_BK - 1) / TF_BK : p.K / TF_BK;
        mbar_wait(&tempty_bar[acc], aphase ^ 1);
        tc_fence_after();
        const uint32_t tmem_p = tmem_base + acc * 2 * BN;  // leading products
        const uint32_t tmem_s = tmem_p + BN;                // correction terms
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&conv_bar[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t sb = sa + 2 * A_BYTES;
#pragma unroll
          for (int k = 0; k < TF_BK / 8; ++k) {  // MMA-K = 8 tf32 = 32 bytes of a K-major row
            const uint32_t ao = Tr::a_mn ? k * 1024 : k * 32;
            const uint32_t bo = Tr::b_mn ? k * 1024 : k * 32;
            auto da = [&](int j) {
              const uint32_t a = sa + j * A_BYTES + ao;
              return Tr::a_mn ? umma_desc_mn32(a, 4096, 512) : umma_desc(a, 16, 1024);
            };
            auto db = [&](int j) {
              const uint32_t b = sb + j * B_BYTES + bo;
              return Tr::b_mn ? umma_desc_mn32(b, 4096, 512) : umma_desc(b, 16, 1024);
            };
            const uint32_t first = (kb | k) != 0;
            tc_mma_tf32(tmem_s, da(1), db(1), IDESC, first);
            tc_mma_tf32(tmem_s, da(1), db(0), IDESC, 1);
            tc_mma_tf32(tmem_s, da(0), db(1), IDESC, 1);
            tc_mma_tf32(tmem_p, da(0), db(0), IDESC, first);
          }
          tc_commit(&empty_bar[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        tc_commit(&tfull_bar[acc]);
      }
    }
    __syncwarp();
  } else if (warp == 3) {
    if (bias_warp) {
      // ============================ bias-gradient warp ============================
      // db[e][m] = sum over kept tokens of A[t, m], read from the raw fp32 A^T tile before
      // the split (the converters wait for this warp).  Box j (32 m) holds 32 token rows of
      // 128 bytes, 32-byte granule g of row kk stored at g ^ (kk & 3) (128B swizzle, 32-byte
      // atoms).  Lane l owns m = 4l .. 4l+3 (box l/8, 16-byte chunk l%8); sequential fp32 sums
      // over tokens in k order: deterministic.  Only the nt == 0 tile of each (e, mt) sums.
      const int j = lane >> 3, c = lane & 7;
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x;; t += gridDim.x) {
        int e, mt, nt;
        if (!decode_tile<Tr::kgroup>(t, s_prefix, n_local, MT, NT, e, mt, nt)) break;
        const int nk = (p.kept[e] + TF_BK - 1) / TF_BK;
        float acc4[4] = {0.f, 0.f, 0.f, 0.f};
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          if (nt == 0) {
            const uint8_t* box = smem + stage * STAGE_BYTES + j * 4096;
#pragma unroll 8
            for (int kk = 0; kk < TF_BK; ++kk) {
              const int off = kk * 128 + ((((c >> 1) ^ (kk & 3)) << 5) | ((c & 1) << 4));
              const float4 a = *reinterpret_cast<const float4*>(box + off);
              acc4[0] += a.x;
              acc4[1] += a.y;
              acc4[2] += a.z;
              acc4[3] += a.w;
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&bias_bar[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (nt == 0) {
          const int m = mt * TC_BM + j * 32 + c * 4;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            if (m + i < p.M) {
              float* dst = bias_out + (size_t)e * p.M + m + i;
              *dst = p.accumulate ? *dst + acc4[i] : acc4[i];
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp >= TF_CONV_WARP0) {
    // ============================ hi / lo split ============================
    const int tid = threadIdx.x - TF_CONV_WARP0 * 32;
    int stage = 0;
    uint32_t phase = 0;
    for (int t = blockIdx.x;; t += gridDim.x) {
      int e, mt, nt;
      if (!decode_tile<Tr::kgroup>(t, s_prefix, n_local, MT, NT, e, mt, nt)) break;
      const int nk = Tr::kgroup ? (p.kept[e] + TF_BK - 1) / TF_BK : p.K / TF_BK;
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(&full_bar[stage], phase);
        if (bias_warp) mbar_wait(&bias_bar[stage], phase);  // raw A summed first
        uint8_t* sa = smem + stage * STAGE_BYTES;
        split_vecs(sa, A_BYTES, A_BYTES / 16, tid);
        split_vecs(sa + 2 * A_BYTES, B_BYTES, B_BYTES / 16, tid);
        // generic-proxy smem writes -> visible to the tensor core (async proxy)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv_bar[stage]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // ============================ epilogue ============================
    const int q = warp & 3;
    const int row_in_tile = q * 32 + lane;
    int it = 0;
    for (int t = blockIdx.x;; t += gridDim.x, ++it) {
      int e, mt, nt;
      if (!decode_tile<Tr::kgroup>(t, s_prefix, n_local, MT, NT, e, mt, nt)) break;
      const int acc = it & 1;
      const uint32_t aphase = (it >> 1) & 1;
      mbar_wait(&tfull_bar[acc], aphase);
      tc_fence_after();
      const int m0 = mt * TC_BM, n0 = nt * BN;
      const int row = m0 + row_in_tile;
      const bool zero_acc = Tr::kgroup && p.kept[e] == 0;
      const int Me = Tr::kgroup ? p.M : p.kept[e];
      const bool row_ok = row < Me;
      float* crow = Tr::kgroup ? Cbase + ((size_t)e * p.M + row) * p.N
                               : Cbase + (size_t)(p.ct.base[e] + row) * p.ldc;
      const float* hrow = (KIND == TC_DGRAD_A && p.hsrc)
                              ? reinterpret_cast<const float*>(p.hsrc) + (crow - Cbase)
                              : crow;
      const uint32_t taddr = tmem_base + acc * 2 * BN + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        const int col0 = n0 + c * 32;
        float v[32];
        if (!zero_acc) {
          uint32_t r[32];
          tmem_ld32(taddr + c * 32, r);           // P: leading products
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
          tmem_ld32(taddr + BN + c * 32, r);      // S: correction terms
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] += __uint_as_float(r[i]);
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = 0.f;
        }
        if (col0 >= p.N) continue;
        bool store = true;
        if (KIND == TC_FWD1 || KIND == TC_FWD2) {
          if (row_ok) {
            const float* bp = bias + (size_t)e * p.N + col0;
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              const float4 bb = *reinterpret_cast<const float4*>(bp + i);
              const float b4[4] = {bb.x, bb.y, bb.z, bb.w};
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const float x = v[i + j] + b4[j];
                v[i + j] = (KIND == TC_FWD1) ? (x > 0.f ? x : 0.f) : x;
              }
            }
          } else {
            store = (KIND == TC_FWD1);  // zero the padding rows of H (token-K GEMMs read them)
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = 0.f;
          }
        } else if (KIND == TC_DGRAD_A) {
          if (row_ok) {
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              const float4 h = *reinterpret_cast<const float4*>(hrow + col0 + i);
              v[i] = h.x > 0.f ? v[i] : 0.f;
              v[i + 1] = h.y > 0.f ? v[i + 1] : 0.f;
              v[i + 2] = h.z > 0.f ? v[i + 2] : 0.f;
              v[i + 3] = h.w > 0.f ? v[i + 3] : 0.f;
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = 0.f;
          }
        } else if (KIND == TC_DGRAD_X) {
          store = row_ok;
        } else {  // WGRAD
          store = row_ok;
          if (row_ok && p.accumulate) {
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              const float4 o = *reinterpret_cast<const float4*>(crow + col0 + i);
              v[i] += o.x; v[i + 1] += o.y; v[i + 2] += o.z; v[i + 3] += o.w;
            }
          }
        }
        if (store) {
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            *reinterpret_cast<float4*>(crow + col0 + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty_bar[acc]);
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(4 * BN));
  }
}

// ------------------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 g_enc32 = nullptr;
int g_sms32 = 0;

bool enc32_init() {
  if (g_enc32) return true;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !fn)
    return false;
  g_enc32 = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&g_sms32, cudaDevAttrMultiProcessorCount, dev);
  return true;
}

// fp32 [outer x inner] row-major, box {box_inner (32 = 128 B), box_outer}, 128-byte swizzle
// (K-major operands) or 128-byte swizzle with 32-byte atoms (mn = MN-major operands)
bool map32(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint32_t box_inner,
           uint32_t box_outer, bool mn = false) {
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * 4};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  return g_enc32(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box,
                 es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 mn ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int KIND, int BN>
cudaError_t launch_tf32(const CUtensorMap& a, const CUtensorMap& b, const TcParams& p,
                        cudaStream_t s) {
  constexpr int STAGE_BYTES = 2 * (TC_BM + BN) * TF_BK * 4;
  constexpr int STAGES = (BN == 128) ? 3 : 4;
  const size_t smem = (size_t)STAGES * STAGE_BYTES + 1024 + 512 + 4 * (MOE_MAX_E + 1) + 64;
  static_assert((size_t)STAGES * STAGE_BYTES + 1024 + 512 + 4 * (MOE_MAX_E + 1) + 64 <= 232448,
                "shared memory");
  auto kf = tf32_gemm_kernel<KIND, BN, STAGES>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  return launch_pdl(kf, g_sms32, TF_THREADS, smem, s, a, b, p);
}

template <int KIND>
cudaError_t launch_tf32_bn(int bn, const CUtensorMap& a, const CUtensorMap& b, const TcParams& p,
                           cudaStream_t s) {
  if (bn == 128) return launch_tf32<KIND, 128>(a, b, p, s);
  return launch_tf32<KIND, 64>(a, b, p, s);
}

// 64-column tiles unless 128-column ones need fewer waves of tiles over the SMs: at these sizes
// a tile's time is set by its k-loop latency, not its width, so the wave count decides
// (m_tiles: the m-tiles of the launch, an upper bound from the buffer rows)
int pick_bn32(int N, int64_t m_tiles) {
  if (N % 128 != 0) return 64;
  const int64_t w128 = (m_tiles * (N / 128) + g_sms32 - 1) / g_sms32;
  const int64_t w64 = (m_tiles * ((N + 63) / 64) + g_sms32 - 1) / g_sms32;
  return w128 < w64 ? 128 : 64;
}

#define TF_TRY(x)                              \
  do {                                         \
    if (!(x)) return MOE_ERR_CUDA;             \
  } while (0)
#define TF_CUDA(x)                             \
  do {                                         \
    if ((x) != cudaSuccess) return MOE_ERR_CUDA; \
  } while (0)

// M-grouped: C[base_e + m, :N] = epi(A[base_e + m, :K] . B_e), B_e [N x K] (K-major) or
// [K x N] (MN-major)
template <int KIND>
moe_status_t mgroup32(const void* A, int64_t rows, int K, const void* B, int N, int n_local,
                      const void* bias, void* C, int ldc, const int32_t* kept,
                      const int32_t* prefix, const CapTable& ct, cudaStream_t s, int nowait = 0,
                      const void* hsrc = nullptr) {
  CUtensorMap ma, mb;
  const int bn = pick_bn32(N, rows / TC_BM);
  TF_TRY(map32(&ma, A, K, rows, 32, 128));
  if (KindTraits<KIND>::b_mn)
    TF_TRY(map32(&mb, B, N, (uint64_t)n_local * K, 32, 32, true));
  else
    TF_TRY(map32(&mb, B, K, (uint64_t)n_local * N, 32, bn));
  TcParams p{};
  p.kept = kept; p.mtile_prefix = prefix; p.n_local = n_local; p.M = 0; p.N = N; p.K = K;
  p.bias = (const __nv_bfloat16*)bias; p.C = (__nv_bfloat16*)C; p.ldc = ldc; p.ct = ct;
  p.nowait = nowait;
  p.hsrc = hsrc;
  TF_CUDA(launch_tf32_bn<KIND>(bn, ma, mb, p, s));
  return MOE_OK;
}

// WGRAD: Out_e[M x N] (+)= A_e^T B_e, A = Abuf[rows x M], B = Bbuf[rows x N] over kept_e rows
moe_status_t wgrad32(const void* Abuf, int M, const void* Bbuf, int N, int64_t rows, int n_local,
                     void* Out, void* bias_out, int accumulate, const int32_t* kept,
                     const CapTable& ct, cudaStream_t s) {
  CUtensorMap ma, mb;
  TF_TRY(map32(&ma, Abuf, M, rows, 32, 32, true));
  TF_TRY(map32(&mb, Bbuf, N, rows, 32, 32, true));
  TcParams p{};
  p.kept = kept; p.mtile_prefix = nullptr; p.n_local = n_local; p.M = M; p.N = N; p.K = 0;
  p.C = (__nv_bfloat16*)Out; p.bias_out = (__nv_bfloat16*)bias_out; p.accumulate = accumulate;
  p.ct = ct;
  const int bn = pick_bn32(N, (int64_t)n_local * ((M + TC_BM - 1) / TC_BM));
  TF_CUDA(launch_tf32_bn<TC_WGRAD>(bn, ma, mb, p, s));
  return MOE_OK;
}

}  // namespace

bool tf32_supported(int d, int f, int dout) {
  return d % 32 == 0 && f % 32 == 0 && dout % 32 == 0;
}

moe_status_t tf32_ffn_forward(void* X, const void* w1, const void* b1, const void* w2,
                              const void* b2, void* H, void* O, int64_t rows, int d, int f,
                              int dout, const int32_t* kept, const int32_t* mtile_prefix,
                              int n_local, const CapTable& ct, cudaStream_t s, int64_t* nlaunch,
                              Prof* prof) {
  if (!enc32_init()) return MOE_ERR_CUDA;
  *nlaunch = 0;
  if (rows == 0 || n_local == 0) return MOE_OK;
  moe_status_t st;
  {
    ProfScope ps(prof, "ffn_gemm1", s);
    st = mgroup32<TC_FWD1>(X, rows, d, w1, f, n_local, b1, H, f, kept, mtile_prefix, ct, s);
  }
  if (st != MOE_OK) return st;
  {
    ProfScope ps(prof, "ffn_gemm2", s);
    st = mgroup32<TC_FWD2>(H, rows, f, w2, dout, n_local, b2, O, dout, kept, mtile_prefix, ct, s);
  }
  *nlaunch = 2;
  return st;
}

moe_status_t tf32_ffn_backward(void* X, void* H, void* dO, void* dX, const void* w1,
                               const void* w2, void* dw1, void* db1, void* dw2, void* db2,
                               int accumulate, int64_t rows, int d, int f, int dout,
                               const int32_t* kept, const int32_t* mtile_prefix, int n_local,
                               const CapTable& ct, cudaStream_t s, int64_t* nlaunch, Prof* prof,
                               int tail_nowait, void* dA_sep) {
  if (!enc32_init()) return MOE_ERR_CUDA;
  // dA in its own buffer (the ReLU' test then reads the intact H): no write-after-read hazard
  // on the dW2 GEMM's H reads, so in the tail mode DGRAD_A and DGRAD_X skip their PDL waits
  void* dA = dA_sep ? dA_sep : H;
  *nlaunch = 0;
  if (rows == 0 || n_local == 0) return MOE_OK;
  int64_t nl = 0;
  moe_status_t st;
  if (dw2) {  // dW2_e = dO_e^T H_e (before H is overwritten), db2 = sum dO fused in
    ProfScope ps(prof, "wgrad_w2", s);
    st = wgrad32(dO, dout, H, f, rows, n_local, dw2, db2, accumulate, kept, ct, s);
    if (st != MOE_OK) return st;
    ++nl;
  } else if (db2) {
    ProfScope ps(prof, "bias_grad", s);
    TF_CUDA(launch_colsum(0, dO, dout, kept, n_local, ct, db2, accumulate, s));
    ++nl;
  }
  {  // dA = (dO W2_e) * 1[H > 0], W2_e stored [d_out x f] = [K x N]; over H or into dA_sep
    ProfScope ps(prof, "dgrad_dA", s);
    st = mgroup32<TC_DGRAD_A>(dO, rows, dout, w2, f, n_local, nullptr, dA, f, kept, mtile_prefix,
                              ct, s, tail_nowait && dA != H && dw2 != nullptr,
                              dA != H ? H : nullptr);
  }
  if (st != MOE_OK) return st;
  ++nl;
  if (dw1) {  // dW1_e = dA_e^T X_e, db1 = sum dA fused in
    ProfScope ps(prof, "wgrad_w1", s);
    st = wgrad32(dA, f, X, d, rows, n_local, dw1, db1, accumulate, kept, ct, s);
    if (st != MOE_OK) return st;
    ++nl;
  } else if (db1) {
    ProfScope ps(prof, "bias_grad", s);
    TF_CUDA(launch_colsum(0, dA, f, kept, n_local, ct, db1, accumulate, s));
    ++nl;
  }
  {  // dX = dA W1_e, W1_e stored [f x d] = [K x N]
    ProfScope ps(prof, "dgrad_dX", s);
    st = mgroup32<TC_DGRAD_X>(dA, rows, f, w1, d, n_local, nullptr, dX, d, kept, mtile_prefix,
                              ct, s, tail_nowait && dA != H && dw1 != nullptr);
  }
  if (st != MOE_OK) return st;
  ++nl;
  *nlaunch = nl;
  return MOE_OK;
}

}  // namespace moe
