// common.cuh -- small device helpers shared by the sm_100a kernels of the MoE hot path.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <utility>

#define MOE_MAX_E 256          // max experts (kernel-argument capacity table size)
#define MOE_MAX_K 8            // max top-k
#define MOE_ROUTE_TILE 128     // tokens per routing tile (histogram / scan granularity)
#define MOE_ROW_ALIGN 128      // expert buffer regions start at multiples of this many rows
#define MOE_PAD_ROWS 64        // rows [kept, roundup(kept, PAD)) are zeroed (token-K GEMMs)

namespace moe {

// Capacity / layout table passed BY VALUE as a kernel argument, so a recompile
// (moe_set_capacities) is stream-ordered without any copy (S4.1).
struct CapTable {
  int32_t cap[MOE_MAX_E];       // C_e (global capacity, reading 12)
  int32_t base[MOE_MAX_E + 1];  // row offset of each expert's rows in the buffer it indexes:
                                //  GEMM side: LOCAL expert regions of X/H/O/dO/dX;
                                //  token side (dispatch/combine): per global expert e, the
                                //  row of global slot 0 (EP: send-buffer offset - pre[e])
  int32_t pre[MOE_MAX_E];       // token side: global slot of this rank's first pair of e
};

// Peer-memory expert parallelism: per-owner base pointers of one expert
// buffer, valid in this process (NVLink peer mappings, or the same GPU for virtual ranks).
// nl == 0: single buffer (no peers); otherwise expert e lives on rank e / nl.
#define MOE_MAX_R 8
struct PeerBufs {
  char* p[MOE_MAX_R];
  int nl;
};

// Row `row` (in its owner's region numbering) of expert e's buffer with `cols` columns.
// (owner selected with constant indices: a dynamically indexed kernel-parameter array would
// be copied to local memory)
template <typename T>
__device__ __forceinline__ T* peer_row(T* local, const PeerBufs& pb, int e, size_t row,
                                       int cols) {
  T* b = local;
  if (pb.nl) {
    const int o = e / pb.nl;
#pragma unroll
    for (int j = 0; j < MOE_MAX_R; ++j)
      if (o == j) b = reinterpret_cast<T*>(pb.p[j]);
  }
  return b + row * (size_t)cols;
}

// gather-table encoding of a peer row: owner in the top 5 bits (rows < 2^26)
#define MOE_GROW_SHIFT 26

template <typename T> struct Vec;  // 16-byte vector of T
template <> struct Vec<float> { static constexpr int N = 4; };
template <> struct Vec<__nv_bfloat16> { static constexpr int N = 8; };

__device__ __forceinline__ float to_f(float v) { return v; }
__device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T> __device__ __forceinline__ T from_f(float v);
template <> __device__ __forceinline__ float from_f<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}

// unpack a 16-byte vector into floats
__device__ __forceinline__ void unpack(const uint4& u, float* f, float) {
  f[0] = __uint_as_float(u.x); f[1] = __uint_as_float(u.y);
  f[2] = __uint_as_float(u.z); f[3] = __uint_as_float(u.w);
}
__device__ __forceinline__ void unpack(const uint4& u, float* f, __nv_bfloat16) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}
__device__ __forceinline__ uint4 pack(const float* f, float) {
  return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]),
                    __float_as_uint(f[3]));
}
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ uint4 pack(const float* f, __nv_bfloat16) {
  return make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]), pack_bf16x2(f[4], f[5]),
                    pack_bf16x2(f[6], f[7]));
}

// streaming read-only load (not volatile: the compiler may batch and reorder these)
__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ld_v4(const void* p) {
  return *reinterpret_cast<const uint4*>(p);
}
__device__ __forceinline__ void st_v4(void* p, const uint4& v) {
  *reinterpret_cast<uint4*>(p) = v;
}

// Zero rows [kept_e, roundup(kept_e, MOE_PAD_ROWS)) of expert regions e = first, first +
// stride, ... (local region j starts at row ct.base[e0 + j]) with all threads of the calling
// block: the token-contraction (weight-gradient) GEMMs read whole 64-row K-blocks.
template <typename T>
__device__ __forceinline__ void zero_pads_block(T* __restrict__ buf, int cols,
                                                const int32_t* __restrict__ kept,
                                                const CapTable& ct, int nreg, int e0, int first,
                                                int stride) {
  constexpr int VE = Vec<T>::N;
  const int nvec = cols / VE;
  for (int j = first; j < nreg; j += stride) {
    const int kp = kept[j];
    const int r0 = ct.base[e0 + j] + kp;
    const int r1 = ct.base[e0 + j] + ((kp + MOE_PAD_ROWS - 1) / MOE_PAD_ROWS) * MOE_PAD_ROWS;
    const size_t total = (size_t)max(r1 - r0, 0) * nvec;
    for (size_t i = threadIdx.x; i < total; i += blockDim.x)
      st_v4(buf + (size_t)r0 * cols + i * VE, make_uint4(0, 0, 0, 0));
  }
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Programmatic dependent launch (PDL).  The kernels of the layer step are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, so a kernel's launch overlaps the tail
// of its predecessor on the stream.  Every such kernel calls pdl_wait() before it touches
// memory (griddepcontrol.wait returns once the predecessor grid has completed and its writes
// are visible; transitive, because every PDL-launched kernel waits), then pdl_trigger() so
// its own successor may be scheduled as soon as all of its CTAs are running.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_enter() {
  pdl_wait();
  pdl_trigger();
}
// nowait: the kernel's inputs all come from kernels at least two launches back (complete once
// its predecessor started, PDL order), so it skips the wait and can run beside the tail of its
// predecessor; the launcher guarantees a full-dependency (non-PDL) launch closes the sequence.
__device__ __forceinline__ void pdl_enter(int nowait) {
  if (!nowait) pdl_wait();
  pdl_trigger();
}
int pdl_enabled();  // host: env MOE_PDL (default 1; 0 = plain stream serialisation)

// A launch with full stream dependency (no PDL attribute): starts after ALL earlier work in
// the stream has completed, including kernels that ran without a PDL wait.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_full(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                               cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.numAttrs = 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace moe
