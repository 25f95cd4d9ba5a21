// gemm_tc.cu -- tcgen05 / TMEM / TMA grouped GEMMs of the expert FFN (bf16 in, fp32 accum).
//
// The expert FFN (Alg. 1 l.7; reading 9) is the dense contraction of the hot path, so
// it runs on the 5th-generation tensor cores.  One persistent, warp-specialised kernel
// template covers all six GEMMs of forward + backward:
//
//   kind        C (per local expert e)                         A major   B major   M rows
//   FWD1        H  = relu(X W1_e^T + b1_e)                      K         K         kept_e
//   FWD2        O  = H W2_e^T + b2_e                             K         K         kept_e
//   DGRAD_A     dA = (dO W2_e) * 1[H > 0]   (written over H)     K         MN        kept_e
//   DGRAD_X     dX = dA W1_e                                     K         MN        kept_e
//   WGRAD       dW = A^T B over kept_e tokens (dW2 = dO^T H,     MN        MN        d_out / f
//               dW1 = dA^T X)
//
// M-grouped GEMMs run over exactly kept_e rows per expert (no capacity-padding FLOPs, the
// waste P:234 and P:370 point at); weight gradients contract over exactly the kept tokens
// (K rounded up to 64 with zero rows).
//
// Roles (256 threads): warp 0 = TMA producer (one lane), warp 1 = MMA issuer (one lane),
// warp 2 = TMEM allocator, warps 4..7 = epilogue (TMEM lanes 0..127).  Shared-memory ring of
// STAGES {A 128x64, B BNx64} bf16 tiles (128B swizzle), mbarrier full/empty pairs; two TMEM
// accumulators of BN fp32 columns so the epilogue of tile i overlaps the MMAs of tile i+1.
// Tile schedule: static persistent (tile = blockIdx.x + i*gridDim.x), identical in all roles.
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

template <int KIND, int BN, int STAGES>
__global__ void __launch_bounds__(TC_THREADS, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   TcParams p) {
  pdl_enter();  // PDL: predecessor complete + visible (common.cuh)
  using Tr = KindTraits<KIND>;
  constexpr int A_BYTES = TC_BM * TC_BK * 2;
  constexpr int B_BYTES = BN * TC_BK * 2;
  constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr uint32_t IDESC = make_idesc(BN, Tr::a_mn, Tr::b_mn);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  int32_t* s_prefix = reinterpret_cast<int32_t*>(s_tmem + 4);   // [n_local + 1]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_local = p.n_local;
  for (int i = threadIdx.x; i <= n_local; i += blockDim.x)
    s_prefix[i] = Tr::kgroup ? 0 : p.mtile_prefix[i];
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      // WGRAD with a fused bias gradient: the stage is released by the MMA commit AND the
      // bias warp (warp 3), which row-sums the A^T tile straight from shared memory
      mbar_init(&empty_bar[s], (Tr::kgroup && p.bias_out) ? 2 : 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], TC_EPI_THREADS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(s_tmem)),
                 "r"(2 * BN));
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
        const int nk = Tr::kgroup ? (p.kept[e] + TC_BK - 1) / TC_BK : p.K / TC_BK;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          mbar_expect_tx(&full_bar[stage], STAGE_BYTES);
          const int k0 = kb * TC_BK;
          if (Tr::a_mn) {  // A^T tiles: {64 M, 64 K} boxes
            tma_load_2d(sa, &tmA, &full_bar[stage], m0, base + k0);
            tma_load_2d(sa + 8192, &tmA, &full_bar[stage], m0 + 64, base + k0);
          } else {         // A K-major: {64 K, 128 rows}
            tma_load_2d(sa, &tmA, &full_bar[stage], k0, base + m0);
          }
          if (Tr::b_mn) {
            if (Tr::kgroup) {
#pragma unroll
              for (int j = 0; j < BN / 64; ++j)
                tma_load_2d(sb + j * 8192, &tmB, &full_bar[stage], n0 + j * 64, base + k0);
            } else {  // weight [K x N] of expert e: rows e*K + k
#pragma unroll
              for (int j = 0; j < BN / 64; ++j)
                tma_load_2d(sb + j * 8192, &tmB, &full_bar[stage], n0 + j * 64, e * p.K + k0);
            }
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
        const int nk = Tr::kgroup ? (p.kept[e] + TC_BK - 1) / TC_BK : p.K / TC_BK;
        mbar_wait(&tempty_bar[acc], aphase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t sb = sa + A_BYTES;
#pragma unroll
          for (int k = 0; k < TC_BK / 16; ++k) {
            uint64_t da = Tr::a_mn ? umma_desc(sa + k * 2048, 8192, 1024)
                                   : umma_desc(sa + k * 32, 16, 1024);
            uint64_t db = Tr::b_mn ? umma_desc(sb + k * 2048, 8192, 1024)
                                   : umma_desc(sb + k * 32, 16, 1024);
            tc_mma(tmem_d, da, db, IDESC, (kb | k) != 0);
          }
          tc_commit(&empty_bar[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        tc_commit(&tfull_bar[acc]);
      }
    }
    __syncwarp();
  } else if (warp == 3) {
    if (Tr::kgroup && p.bias_out) {
      // ============================ bias-gradient warp ============================
      // db[e][m] = sum over kept tokens of A[t, m] (A = dO for db2, dA for db1): the A^T
      // tile of every k-block is already in shared memory (MN-major, 128B swizzle: token row
      // kk holds 64 m-values in 8 16-byte chunks, chunk c stored at c ^ (kk & 7)).  Lane l
      // owns 4 consecutive m: box j = l/16, chunk c = (l%16)/2, half h = l%2.  Sequential
      // fp32 sums over tokens in k order: deterministic.  Only the nt == 0 tile of each
      // (e, mt) sums; other tiles just release the stage.
      const int j = lane >> 4, c = (lane & 15) >> 1, hh = lane & 1;
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x;; t += gridDim.x) {
        int e, mt, nt;
        if (!decode_tile<Tr::kgroup>(t, s_prefix, n_local, MT, NT, e, mt, nt)) break;
        const int nk = (p.kept[e] + TC_BK - 1) / TC_BK;
        float acc4[4] = {0.f, 0.f, 0.f, 0.f};
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          if (nt == 0) {
            const uint8_t* box = smem + stage * STAGE_BYTES + j * 8192;
#pragma unroll 8
            for (int kk = 0; kk < TC_BK; ++kk) {
              const uint2 u = *reinterpret_cast<const uint2*>(box + kk * 128 + ((c ^ (kk & 7)) << 4) + hh * 8);
              acc4[0] += __uint_as_float(u.x << 16);
              acc4[1] += __uint_as_float(u.x & 0xffff0000u);
              acc4[2] += __uint_as_float(u.y << 16);
              acc4[3] += __uint_as_float(u.y & 0xffff0000u);
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty_bar[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (nt == 0) {
          const int m = mt * TC_BM + j * 64 + c * 8 + hh * 4;
          if (m < p.M) {
            __nv_bfloat16* dst = p.bias_out + (size_t)e * p.M + m;
            if (p.accumulate) {
#pragma unroll
              for (int i = 0; i < 4; ++i) acc4[i] += __bfloat162float(dst[i]);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) dst[i] = __float2bfloat16_rn(acc4[i]);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ============================ epilogue ============================
    const int q = warp & 3;          // TMEM lane quarter (warp w may access lanes 32*(w%4)..)
    const int half = (warp - 4) >> 2;  // which half of the BN columns this warp drains
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
      __nv_bfloat16* crow;
      if (Tr::kgroup)
        crow = p.C + ((size_t)e * p.M + row) * p.N;
      else
        crow = p.C + (size_t)(p.ct.base[e] + row) * p.ldc;
      const uint32_t taddr = tmem_base + acc * BN + ((uint32_t)(q * 32) << 16);
      constexpr int CH = BN / 64;      // 32-column chunks per warp half
#pragma unroll 1
      for (int c = half * CH; c < (half + 1) * CH; ++c) {
        const int col0 = n0 + c * 32;
        // issue this chunk's side-input loads before the TMEM load so their latency overlaps
        uint4 side[4];
        const bool need_side = (KIND == TC_DGRAD_A && row_ok) ||
                               (KIND == TC_WGRAD && row_ok && p.accumulate);
        if (need_side) {
#pragma unroll
          for (int i = 0; i < 4; ++i) side[i] = ld_v4(crow + col0 + 8 * i);
        }
        uint32_t r[32];
        if (!zero_acc) {
          tmem_ld32(taddr + c * 32, r);
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
            const __nv_bfloat16* bp = p.bias + (size_t)e * p.N + col0;
#pragma unroll
            for (int i = 0; i < 32; i += 8) {
              float bb[8];
              unpack(ld_v4(bp + i), bb, __nv_bfloat16());
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                float x = v[i + j] + bb[j];
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
            for (int i = 0; i < 32; i += 8) {
              float h[8];
              unpack(side[i / 8], h, __nv_bfloat16());
#pragma unroll
              for (int j = 0; j < 8; ++j) v[i + j] = h[j] > 0.f ? v[i + j] : 0.f;
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
            for (int i = 0; i < 32; i += 8) {
              float o[8];
              unpack(side[i / 8], o, __nv_bfloat16());
#pragma unroll
              for (int j = 0; j < 8; ++j) v[i + j] += o[j];
            }
          }
        }
        if (store) {
          uint32_t bits = 0;
#pragma unroll
          for (int i = 0; i < 32; i += 8) {
            const uint4 pk = pack(v + i, __nv_bfloat16());
            st_v4(crow + col0 + i, pk);
            const uint32_t w4[4] = {pk.x, pk.y, pk.z, pk.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              bits |= ((w4[j] & 0xffffu) != 0u ? 1u : 0u) << (i + 2 * j);
              bits |= ((w4[j] >> 16) != 0u ? 1u : 0u) << (i + 2 * j + 1);
            }
          }
          if (KIND == TC_FWD1 && p.mask)  // relu' bits for the 2-CTA DGRAD_A epilogue
            p.mask[(size_t)(p.ct.base[e] + row) * (p.N >> 5) + (col0 >> 5)] = bits;
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
                 "r"(2 * BN));
  }
}

// ------------------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static int g_num_sms = 0;

static bool ensure_encode() {
  if (g_encode) return true;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !fn)
    return false;
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  return true;
}

// 2-D bf16 tensor map over a row-major [outer x inner] matrix, 128-byte swizzle.
static bool make_map(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer,
                     uint32_t box_inner, uint32_t box_outer,
                     CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                        box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}
// epilogue store map of the 2-CTA kernel: 32 x 32 boxes, 64-byte swizzle
static bool make_store_map(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer) {
  return make_map(m, ptr, inner, outer, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B);
}

template <int KIND, int BN>
static cudaError_t launch_tc(const CUtensorMap& a, const CUtensorMap& b, const TcParams& p,
                             cudaStream_t s) {
  constexpr int STAGES = (BN == 256) ? 4 : 6;
  constexpr int STAGE_BYTES = (TC_BM + BN) * TC_BK * 2;
  const size_t smem = (size_t)STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/ +
                      4 * (MOE_MAX_E + 1) + 64;
  auto kf = tc_gemm_kernel<KIND, BN, STAGES>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  launch_pdl(kf, g_num_sms, TC_THREADS, smem, s, a, b, p);
  return cudaGetLastError();
}

template <int KIND>
static cudaError_t launch_tc_bn(int N, const CUtensorMap& a, const CUtensorMap& b,
                                const TcParams& p, cudaStream_t s) {
  if (N % 256 == 0) return launch_tc<KIND, 256>(a, b, p, s);
  if (N % 128 == 0) return launch_tc<KIND, 128>(a, b, p, s);
  return launch_tc<KIND, 64>(a, b, p, s);
}

static int pick_bn(int N) { return N % 256 == 0 ? 256 : (N % 128 == 0 ? 128 : 64); }

cudaError_t launch_tc2_kind(int kind, int BN, const CUtensorMap& a, const CUtensorMap& b,
                            const CUtensorMap& c, const TcParams& p, int grid, cudaStream_t s,
                            const CUtensorMap* a2 = nullptr, const CUtensorMap* b2 = nullptr);

static int tc_pf() {  // MOE_TC_PF: k-blocks of B prefetched to L2 for the next wave
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MOE_TC_PF");
    v = e ? atoi(e) : 0;
  }
  return v;
}

static int tc_dbg() {  // MOE_TC_DBG: timing experiments only (1: skip epilogue stores,
                       // 2: skip the db1 partials, 4: skip the relu-mask loads,
                       // 8: skip only the TMA store instruction, 16: all stores to rows 0..127)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MOE_TC_DBG");
    v = e ? atoi(e) : 0;
  }
  return v;
}

// MOE_HALF_TILES=0 turns off M = 128 remainder tiles in the 2-CTA M-grouped kernels (A/B
// comparisons; read per call).
static int tc_half() {
  const char* e = getenv("MOE_HALF_TILES");
  return e ? atoi(e) != 0 : 1;
}

// MOE_NO_KTRIM=1: the 2-CTA weight-gradient GEMMs issue every 16-deep MMA of their last
// k-block, pad tokens included (A/B comparisons; read per call).
static int tc_no_ktrim() {
  const char* e = getenv("MOE_NO_KTRIM");
  return e ? atoi(e) != 0 : 0;
}

static int tc_sched() {  // MOE_TC_SCHED: 2-CTA tile schedule (see TcParams::sched)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MOE_TC_SCHED");
    v = e ? atoi(e) : 0;
  }
  return v;
}

// 2-CTA (cta_group::2) kernels need BN in {128, 256}.  MOE_TC_1CTA=<bitmask of TcKind> forces
// the 1-CTA form for those kinds (debug / A-B comparisons).
static bool use_2cta(int N, int kind) {
  static int mask = -1;
  if (mask < 0) {
    const char* v = getenv("MOE_TC_1CTA");
    mask = v ? atoi(v) : 0;
  }
  return !((mask >> kind) & 1) && N % 128 == 0;
}

void tc_plan_free(TcPlan* p) { (void)p; }

bool tc_gather_supported(int d, int f) {
  return use_2cta(f, TC_FWD1) && use_2cta(d, TC_WGRAD) && d % 64 == 0;
}
bool tc_combine_supported(int dout) { return use_2cta(dout, TC_FWD2); }
bool tc_dx_fusion_supported(int d) { return use_2cta(d, TC_DGRAD_X); }
bool tc_peer_return_supported(int d, int dout) {
  return use_2cta(dout, TC_FWD2) && use_2cta(d, TC_DGRAD_X);
}

// db[e][c] = sum of the DGRAD_A column-sum partials of expert e, fixed order (deterministic).
__global__ void bias_part_reduce_kernel(const float* __restrict__ part,
                                        const int32_t* __restrict__ kept, int N,
                                        __nv_bfloat16* __restrict__ db, int accumulate,
                                        int nowait) {
  pdl_enter(nowait);  // PDL (nowait: launched after the dX GEMM, DGRAD_A long complete)
  const int e = blockIdx.y;
  __shared__ int s_pre, s_mt;
  if (threadIdx.x < 32) {
    int acc = 0;
    for (int j = threadIdx.x; j < e; j += 32) acc += (kept[j] + 255) / 256;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (threadIdx.x == 0) {
      s_pre = acc;
      s_mt = (kept[e] + 255) / 256;
    }
  }
  __syncthreads();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  const float* pp = part + (size_t)s_pre * 2 * N + c;
  float v = 0.f;
  for (int j = 0; j < s_mt * 2; ++j) v += pp[(size_t)j * N];
  if (accumulate) v += __bfloat162float(db[(size_t)e * N + c]);
  db[(size_t)e * N + c] = __float2bfloat16_rn(v);
}

#define TC_TRY(expr)                                        \
  do {                                                      \
    if (!(expr)) return MOE_ERR_CUDA;                       \
  } while (0)
#define TC_CUDA(expr)                                       \
  do {                                                      \
    cudaError_t _e = (expr);                                \
    if (_e != cudaSuccess) {                                \
      fprintf(stderr, "tcgen05: %s\n", cudaGetErrorString(_e)); \
      return MOE_ERR_CUDA;                                  \
    }                                                       \
  } while (0)

// M-grouped GEMM: C[base_e + m, :N] = epi(A[base_e + m, :K] . B_e), B_e [N x K] (K-major)
// or [K x N] (MN-major, b_mn).
template <int KIND>
static moe_status_t mgroup(const void* A, int64_t rows, int K, const void* B, int N,
                           int n_local, const void* bias, void* C, int ldc, const int32_t* kept,
                           const int32_t* prefix, const CapTable& ct, cudaStream_t s,
                           uint32_t* mask = nullptr, float* bias_part = nullptr,
                           const TcFusion* fz = nullptr, int nowait = 0) {
  CUtensorMap ma, mb;
  const int bn = pick_bn(N);
  const bool two = use_2cta(N, KIND);
  const bool gat = KIND == TC_FWD1 && fz && fz->x;        // A rows gathered from x (N2)
  const bool comb = KIND == TC_FWD2 && fz && fz->y;       // fused combine (N2, k = 1)
  const bool fdx = KIND == TC_DGRAD_X && fz && fz->dx_fused;  // fused dispatch backward (k = 1)
  const PeerBufs* pr = !fz ? nullptr
                       : KIND == TC_FWD2 ? &fz->pret_o : KIND == TC_DGRAD_X ? &fz->pret_dx : nullptr;
  const bool ret = pr && pr->nl != 0;                     // peer EP return rows (N1)
  if ((gat || comb || fdx || ret) && !two) return MOE_ERR_CONFIG;
  CUtensorMap ma2, mb2;
  if (fdx) {
    TC_TRY(make_map(&ma2, fz->dlr, 2 * fz->n_pad, rows, 64, 128));
    TC_TRY(make_map(&mb2, fz->wg, N, fz->n, 64, 64));
  }
  if (gat)
    TC_TRY(make_map(&ma, fz->x, K, (uint64_t)fz->T, 64, 1));
  else
    TC_TRY(make_map(&ma, A, K, rows, 64, 128));
  if (KindTraits<KIND>::b_mn)
    TC_TRY(make_map(&mb, B, N, (uint64_t)n_local * K, 64, 64));
  else
    TC_TRY(make_map(&mb, B, K, (uint64_t)n_local * N, 64, two ? bn / 2 : bn));
  TcParams p{};
  p.kept = kept; p.mtile_prefix = prefix; p.n_local = n_local; p.M = 0; p.N = N; p.K = K;
  p.bias = (const __nv_bfloat16*)bias; p.C = (__nv_bfloat16*)C; p.ldc = ldc; p.ct = ct;
  p.mask = mask;
  p.bias_part = two ? bias_part : nullptr;
  if (gat || comb) {
    p.gtos = fz->tos;
    p.gk = fz->k;
    p.grows = fz->T;
  }
  if (!gat) p.gtos = comb ? fz->tos : nullptr;
  if (comb) {
    p.y = (__nv_bfloat16*)fz->y;
    p.wt = fz->w;
    if (fz->comb2) {  // k = 2: needs the token-ordered O of the return-row store path
      if (!ret || fz->k != 2 || fz->pret_o.nl != 1) return MOE_ERR_CONFIG;
      p.comb2 = 1;
      p.slot2 = fz->slot;
      p.ycnt = fz->ycnt;
      p.ycb = N / (bn / 2);
    }
  }
  if (ret) {
    p.gtos = fz->tos;
    p.gk = fz->k;
    p.pret = *pr;
    p.tpr = fz->tpr;
  }
  if (fdx) {
    p.gtos = fz->tos;
    p.dxo = (__nv_bfloat16*)fz->dx;
    p.nkx = 2 * fz->n_pad / 64;
    p.nbx = fz->n_pad / 64;
    p.accumulate = fz->accumulate;
  }
  p.sched = tc_sched();
  p.pf_kb = tc_pf();
  p.dbg = tc_dbg();
  p.nowait = two ? nowait : 0;  // (the 1-CTA kernel always waits)
  p.half_tiles = two && !p.comb2 && tc_half();  // (comb2 counts per BN/2 column block)
  if (two) {
    CUtensorMap mc;
    TC_TRY(make_store_map(&mc, C, ldc, rows));
    TC_CUDA(launch_tc2_kind(KIND, bn, ma, mb, mc, p, g_num_sms & ~1, s, fdx ? &ma2 : nullptr,
                            fdx ? &mb2 : nullptr));
  } else {
    TC_CUDA(launch_tc_bn<KIND>(N, ma, mb, p, s));
  }
  return MOE_OK;
}

// WGRAD: Out_e[M x N] (+)= A_e^T B_e, A = Abuf[rows x M], B = Bbuf[rows x N] over kept_e rows.
static moe_status_t wgrad(const void* Abuf, int M, const void* Bbuf, int N, int64_t rows,
                          int n_local, void* Out, void* bias_out, int accumulate,
                          const int32_t* kept, const CapTable& ct, cudaStream_t s,
                          const TcFusion* fz = nullptr) {
  CUtensorMap ma, mb;
  const bool gat = fz && fz->x;   // B rows (tokens) gathered from x (N2)
  if (gat && !use_2cta(N, TC_WGRAD)) return MOE_ERR_CONFIG;
  TC_TRY(make_map(&ma, Abuf, M, rows, 64, 64));
  if (gat)
    TC_TRY(make_map(&mb, fz->x, N, (uint64_t)fz->T, 64, 1));
  else
    TC_TRY(make_map(&mb, Bbuf, N, rows, 64, 64));
  TcParams p{};
  p.kept = kept; p.mtile_prefix = nullptr; p.n_local = n_local; p.M = M; p.N = N; p.K = 0;
  p.C = (__nv_bfloat16*)Out; p.bias_out = (__nv_bfloat16*)bias_out; p.accumulate = accumulate;
  p.ct = ct;
  if (gat) {
    p.gtos = fz->tos;
    p.gk = fz->k;
    p.grows = fz->T;
  }
  p.sched = tc_sched();
  p.pf_kb = tc_pf();
  p.dbg = tc_dbg();
  p.no_ktrim = tc_no_ktrim();
  if (use_2cta(N, TC_WGRAD)) {
    CUtensorMap mc;
    TC_TRY(make_store_map(&mc, Out, N, (uint64_t)n_local * M));
    TC_CUDA(launch_tc2_kind(TC_WGRAD, pick_bn(N), ma, mb, mc, p, g_num_sms & ~1, s));
  } else {
    TC_CUDA(launch_tc_bn<TC_WGRAD>(N, ma, mb, p, s));
  }
  return MOE_OK;
}

moe_status_t tc_ffn_forward(TcPlan* plan, void* X, const void* w1, const void* b1,
                            const void* w2, const void* b2, void* H, void* O, int64_t rows,
                            int d, int f, int dout, const int32_t* kept,
                            const int32_t* mtile_prefix, int n_local, const CapTable& ct,
                            int max_cap, cudaStream_t s, int64_t* nlaunch, Prof* prof,
                            uint32_t* mask, const TcFusion* fz,
                            cudaError_t (*between)(void*), void* between_ctx) {
  (void)plan; (void)max_cap;
  if (!ensure_encode()) return MOE_ERR_CUDA;
  if (rows == 0 || n_local == 0) {
    *nlaunch = 0;
    if (between && between(between_ctx) != cudaSuccess) return MOE_ERR_CUDA;
    return MOE_OK;
  }
  moe_status_t st;
  {
    ProfScope ps(prof, "ffn_gemm1", s);
    st = mgroup<TC_FWD1>(X, rows, d, w1, f, n_local, b1, H, f, kept, mtile_prefix, ct, s, mask,
                         nullptr, fz);
  }
  if (st != MOE_OK) return st;
  if (between && between(between_ctx) != cudaSuccess) return MOE_ERR_CUDA;
  {
    ProfScope ps(prof, "ffn_gemm2", s);
    st = mgroup<TC_FWD2>(H, rows, f, w2, dout, n_local, b2, O, dout, kept, mtile_prefix, ct, s,
                         nullptr, nullptr, fz);
  }
  *nlaunch = 2;
  return st;
}

moe_status_t tc_ffn_backward(TcPlan* plan, void* X, void* H, void* dO, void* dX, const void* w1,
                             const void* w2, void* dw1, void* db1, void* dw2, void* db2,
                             int accumulate, int64_t rows, int d, int f, int dout,
                             const int32_t* kept, const int32_t* mtile_prefix, int n_local,
                             const CapTable& ct, int max_cap, cudaStream_t s,
                             int64_t* nlaunch, Prof* prof, uint32_t* mask, float* bias_part,
                             const TcFusion* fz, int tail_nowait, void* dA_sep) {
  (void)plan; (void)max_cap;
  // dA in its own buffer (2-CTA DGRAD_A, whose ReLU' mask comes from the FWD1 bits, not from
  // H): H is then never overwritten, so in the tail mode DGRAD_A can skip its PDL wait on the
  // dW2 GEMM (which reads H) and take the SMs of that GEMM's last wave
  void* dA = (dA_sep && use_2cta(f, TC_DGRAD_A) && mask) ? dA_sep : H;
  const int da_nowait = tail_nowait && dA != H && dw2 != nullptr;
  // db1 from the DGRAD_A epilogue (2-CTA) instead of the weight-gradient bias warps
  const bool db1_in_dgrad = db1 && bias_part && use_2cta(f, TC_DGRAD_A);
  if (!ensure_encode()) return MOE_ERR_CUDA;
  int64_t nl = 0;
  if (rows == 0 || n_local == 0) { *nlaunch = 0; return MOE_OK; }
  moe_status_t st;
  if (dw2) {  // dW2_e = dO_e^T H_e (before H is overwritten), db2 = sum dO fused in
    ProfScope ps(prof, "wgrad_w2", s);
    st = wgrad(dO, dout, H, f, rows, n_local, dw2, db2, accumulate, kept, ct, s);
    if (st != MOE_OK) return st;
    ++nl;
  } else if (db2) {
    ProfScope ps(prof, "bias_grad", s);
    TC_CUDA(launch_colsum(1, dO, dout, kept, n_local, ct, db2, accumulate, s));
    ++nl;
  }
  // dA = (dO W2_e) * 1[H > 0], W2_e stored [d_out x f] = [K x N]
  {
    ProfScope ps(prof, "dgrad_dA", s);
    st = mgroup<TC_DGRAD_A>(dO, rows, dout, w2, f, n_local, nullptr, dA, f, kept, mtile_prefix, ct, s,
                            mask, db1_in_dgrad ? bias_part : nullptr, nullptr, da_nowait);
  }
  if (st != MOE_OK) return st;
  ++nl;
  // db1 partials -> db1: right here, or (tail_nowait) after the dX GEMM without a PDL wait,
  // beside that GEMM's tail (nothing in between touches the partials or db1)
  auto db1_reduce = [&](int nowait) -> moe_status_t {
    ProfScope ps(prof, "bias_grad", s);
    launch_pdl(bias_part_reduce_kernel, dim3((f + 255) / 256, n_local), 256, 0, s,
               bias_part, kept, f, (__nv_bfloat16*)db1, accumulate, nowait);
    TC_CUDA(cudaGetLastError());
    ++nl;
    return MOE_OK;
  };
  if (db1_in_dgrad && !tail_nowait) {
    st = db1_reduce(0);
    if (st != MOE_OK) return st;
  }
  if (dw1) {  // dW1_e = dA_e^T X_e (db1 fused here only when not produced by DGRAD_A)
    ProfScope ps(prof, "wgrad_w1", s);
    st = wgrad(dA, f, X, d, rows, n_local, dw1, db1_in_dgrad ? nullptr : db1, accumulate, kept, ct, s,
               fz);
    if (st != MOE_OK) return st;
    ++nl;
  } else if (db1 && !db1_in_dgrad) {
    ProfScope ps(prof, "bias_grad", s);
    TC_CUDA(launch_colsum(1, dA, f, kept, n_local, ct, db1, accumulate, s));
    ++nl;
  }
  // dX = dA W1_e, W1_e stored [f x d] = [K x N]
  {
    ProfScope ps(prof, "dgrad_dX", s);
    // tail_nowait: DGRAD_X reads dA (DGRAD_A, two launches back), W1 and the fused dispatch
    // backward's dl rows / W_g -- nothing of WGRAD_W1, which writes only dW1 -- so it skips the
    // PDL wait and fills the SMs WGRAD_W1's last wave leaves idle
    st = mgroup<TC_DGRAD_X>(dA, rows, f, w1, d, n_local, nullptr, dX, d, kept, mtile_prefix, ct, s,
                            nullptr, nullptr, fz, tail_nowait && dw1 != nullptr);
  }
  if (st != MOE_OK) return st;
  ++nl;
  if (db1_in_dgrad && tail_nowait) {
    st = db1_reduce(1);
    if (st != MOE_OK) return st;
  }
  *nlaunch = nl;
  return MOE_OK;
}

}  // namespace moe
