// prof.h -- optional per-kernel CUDA-event timing inside the library (bench roofline).
// When enabled, every launcher call is bracketed by two events recorded on the stream the
// kernel is launched on; moe_profile_read sums the elapsed times per kernel name.
#pragma once
#include <cuda_runtime.h>
#include <string>
#include <vector>

namespace moe {

struct Prof {
  bool on = false;
  struct Rec {
    const char* name;
    cudaEvent_t a, b;
  };
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  std::vector<Rec> recs;

  cudaEvent_t get() {
    if (used == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return pool[used++];
  }
  void reset() {
    used = 0;
    recs.clear();
  }
  void destroy() {
    for (auto e : pool) cudaEventDestroy(e);
    pool.clear();
    used = 0;
    recs.clear();
  }
};

struct ProfScope {
  Prof* p;
  cudaStream_t s;
  Prof::Rec r{};
  ProfScope(Prof* prof, const char* name, cudaStream_t st) : p(prof), s(st) {
    if (p && p->on) {
      r.name = name;
      r.a = p->get();
      r.b = p->get();
      cudaEventRecord(r.a, s);
    }
  }
  ~ProfScope() {
    if (p && p->on) {
      cudaEventRecord(r.b, s);
      p->recs.push_back(r);
    }
  }
};

}  // namespace moe
