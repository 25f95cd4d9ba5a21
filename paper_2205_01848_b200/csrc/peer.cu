// peer.cu -- device-initiated expert-parallel exchange through peer memory (N1), see peer.h.
#include <algorithm>

#include "peer.h"

namespace moe {

namespace {

size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

__device__ __forceinline__ uint32_t* flag_ptr(char* win, int phase, int src) {
  return reinterpret_cast<uint32_t*>(win + 256) + phase * MOE_MAX_R + src;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int32_t ld_volatile(const int32_t* p) {
  return *reinterpret_cast<const volatile int32_t*>(p);
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Threads 0..R-1: publish epoch `ep` for `phase` into every rank's flag slot of this rank,
// then wait until every rank published >= ep into ours.  Called by all threads of the block.
// A peer that never arrives (dead rank, mismatched call sequence) does not hang the GPU: after
// MOE_PEER_TIMEOUT_NS the wait gives up and raises device flag 8 (moe_check_device_flags).
__device__ __forceinline__ void barrier_block(const PeerBufs& win, int R, int rank, int phase,
                                              uint32_t ep, uint32_t* err_flags) {
  __threadfence_system();
  __syncthreads();
  const int j = threadIdx.x;
  if (j < R) {
    st_release_sys(flag_ptr(win.p[j], phase, rank), ep);
    const uint32_t* mine = flag_ptr(win.p[rank], phase, j);
    const uint64_t t0 = globaltimer_ns();
    while ((int32_t)(ld_acquire_sys(mine) - ep) < 0) {
      __nanosleep(64);
      if (globaltimer_ns() - t0 > MOE_PEER_TIMEOUT_NS) {
        if (err_flags) atomicOr(err_flags, MOE_FLAG_PEER_TIMEOUT);
        break;
      }
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256) peer_plan_kernel(PeerBufs win, int R, int rank, int n,
                                                        int nl, const int32_t* __restrict__ lc,
                                                        CapTable ct, int32_t* counts_out,
                                                        int32_t* kept_out, int32_t* mtile_prefix,
                                                        int64_t* drops_out, int32_t* pre_out,
                                                        uint32_t* err_flags) {
  pdl_wait();  // PDL: predecessor complete + visible; no early trigger: the next
  // kernel must not take SMs while this one spins on peers (ranks sharing one GPU deadlock)
  __shared__ uint32_t s_ep;
  __shared__ long long s_drops[8];
  __shared__ int32_t s_tiles[MOE_MAX_E];
  char* own = win.p[rank];
  if (threadIdx.x == 0) {  // this iteration's epoch (the same sequence on every rank)
    uint32_t* ep = reinterpret_cast<uint32_t*>(own);
    s_ep = *reinterpret_cast<volatile uint32_t*>(ep) + 1u;
    *ep = s_ep;
  }
  __syncthreads();
  const uint32_t ep = s_ep;
  const int e = threadIdx.x;
  // C1 without the host: push this rank's counts into row `rank` of every peer's table
  if (e < n) {
    const int32_t c = lc[e];
    for (int j = 0; j < R; ++j)
      reinterpret_cast<int32_t*>(win.p[j] + 512)[rank * MOE_MAX_E + e] = c;
  }
  barrier_block(win, R, rank, PH_CNT, ep, err_flags);
  // global plan (reading 12: global capacity, slots in ascending global token order, so
  // rank r's pairs of e start after those of ranks < r)
  long long drop = 0;
  const int32_t* tab = reinterpret_cast<const int32_t*>(own + 512);
  if (e < n) {
    int cg = 0, pre = 0;
    for (int j = 0; j < R; ++j) {
      const int v = ld_volatile(tab + j * MOE_MAX_E + e);
      cg += v;
      if (j < rank) pre += v;
    }
    const int kg = min(cg, ct.cap[e]);
    drop = cg - kg;
    counts_out[e] = cg;
    pre_out[e] = pre;
    const int jl = e - rank * nl;
    if (jl >= 0 && jl < nl) {
      kept_out[jl] = kg;
      s_tiles[jl] = (kg + 127) / 128;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) drop += __shfl_xor_sync(0xffffffffu, drop, o);
  if ((threadIdx.x & 31) == 0) s_drops[threadIdx.x >> 5] = drop;
  __syncthreads();
  if (threadIdx.x < 32) {  // one warp: drops and the GEMM m-tile prefix of the local experts
    const int lane = threadIdx.x;
    long long dsum = lane < (int)(blockDim.x >> 5) ? s_drops[lane] : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dsum += __shfl_xor_sync(0xffffffffu, dsum, o);
    int carry = 0;
    for (int q0 = 0; q0 < nl; q0 += 32) {
      const int q = q0 + lane;
      const int v = q < nl ? s_tiles[q] : 0;
      int incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
      }
      if (q < nl) mtile_prefix[q] = carry + incl - v;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) {
      mtile_prefix[nl] = carry;
      *drops_out = dsum;
    }
  }
}

__global__ void peer_barrier_kernel(PeerBufs win, int R, int rank, int phase,
                                    uint32_t* err_flags) {
  pdl_wait();  // PDL: predecessor complete + visible; no early trigger: the next
  // kernel must not take SMs while this one spins on peers (ranks sharing one GPU deadlock)
  const uint32_t ep = *reinterpret_cast<const volatile uint32_t*>(win.p[rank]);
  barrier_block(win, R, rank, phase, ep, err_flags);
}

template <typename T>
__global__ void __launch_bounds__(256) peer_sum_kernel(PeerBufs win, size_t off, int R,
                                                       size_t count, T* __restrict__ out,
                                                       int accumulate) {
  pdl_enter();  // PDL: predecessor complete + visible (common.cuh)
  const size_t n4 = count / 4;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4;
       i += (size_t)gridDim.x * blockDim.x) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int j = 0; j < R; ++j) {  // rank order: the same sum on every rank
      const float4 v = __ldcv(reinterpret_cast<const float4*>(win.p[j] + off) + i);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    const float a[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float v = a[q];
      if (accumulate) v += to_f(out[4 * i + q]);
      out[4 * i + q] = from_f<T>(v);
    }
  }
  // tail (count % 4)
  if (blockIdx.x == 0)
    for (size_t i = n4 * 4 + threadIdx.x; i < count; i += blockDim.x) {
      float acc = 0.f;
      for (int j = 0; j < R; ++j) acc += __ldcv(reinterpret_cast<const float*>(win.p[j] + off) + i);
      if (accumulate) acc += to_f(out[i]);
      out[i] = from_f<T>(acc);
    }
}

}  // namespace

void peer_layout(PeerLayout& L, int64_t rows, int n, int d, int dout, size_t elem,
                 int64_t pair_rows) {
  L.rows = rows;
  L.epoch = 0;
  L.flags = 256;
  L.cnt = 512;
  size_t o = al256(512 + (size_t)MOE_MAX_R * MOE_MAX_E * 4);
  auto take = [&](size_t bytes) { size_t r = o; o += al256(bytes); return r; };
  L.bal = take((size_t)MOE_MAX_E * 4);
  L.dwg = take((size_t)n * d * 4);
  L.tos = take((size_t)rows * 4);
  L.x = take((size_t)rows * d * elem);
  L.o = take((size_t)rows * dout * elem);
  L.dob = take((size_t)rows * dout * elem);
  L.dxb = take((size_t)rows * d * elem);
  L.oret = take((size_t)pair_rows * dout * elem);
  L.dxret = take((size_t)pair_rows * d * elem);
  // [hi | lo](dl) pairs of the local experts' rows (fused dispatch backward, k = 1), pushed
  // by the token owners' combine backward
  L.dlr = take((size_t)rows * 2 * ((n + 63) / 64 * 64) * elem);
  L.total = o;
}

cudaError_t launch_peer_plan(const PeerBufs& win, int R, int rank, int n, int n_local,
                             const int32_t* local_counts, const CapTable& ct, RouteBufs b,
                             int32_t* pre_out, cudaStream_t s) {
  launch_pdl(peer_plan_kernel, 1, 256, 0, s, win, R, rank, n, n_local, local_counts, ct, b.counts,
                                     b.kept, b.mtile_prefix, b.drops, pre_out,
                                     reinterpret_cast<uint32_t*>(b.flags));
  return cudaGetLastError();
}

cudaError_t launch_peer_barrier(const PeerBufs& win, int R, int rank, int phase, cudaStream_t s,
                                uint32_t* err_flags) {
  launch_pdl(peer_barrier_kernel, 1, 32, 0, s, win, R, rank, phase, err_flags);
  return cudaGetLastError();
}

cudaError_t launch_peer_sum(const PeerBufs& win, size_t off, int R, size_t count, int dtype,
                            void* out, int accumulate, cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  const int grid = (int)std::min<size_t>((count / 4 + 255) / 256 + 1, 148 * 4);
  if (dtype == 1)
    launch_pdl(peer_sum_kernel<__nv_bfloat16>, grid, 256, 0, s, win, off, R, count,
                                                        (__nv_bfloat16*)out, accumulate);
  else
    launch_pdl(peer_sum_kernel<float>, grid, 256, 0, s, win, off, R, count, (float*)out, accumulate);
  return cudaGetLastError();
}

}  // namespace moe
