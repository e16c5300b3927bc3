// Device-side building blocks shared by the sm_100a scan kernels.
//
// Vector I/O (128-bit where alignment allows), the affine-pair algebra of
// the recurrence, and the gpu-scope publish/acquire primitives of the
// decoupled look-back.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace linrec_dev {

// ---- vector element access -------------------------------------------------
template <class S, int VEC>
struct VecIO;

template <>
struct VecIO<float, 4> {
  static __device__ __forceinline__ void load_stream(const float* p, float (&v)[4]) {
    float4 r = __ldcs(reinterpret_cast<const float4*>(p));
    v[0] = r.x; v[1] = r.y; v[2] = r.z; v[3] = r.w;
  }
  static __device__ __forceinline__ void store_stream(float* p, const float (&v)[4]) {
    __stcs(reinterpret_cast<float4*>(p), make_float4(v[0], v[1], v[2], v[3]));
  }
  static __device__ __forceinline__ void load_cg(const float* p, float (&v)[4]) {
    float4 r = __ldcg(reinterpret_cast<const float4*>(p));
    v[0] = r.x; v[1] = r.y; v[2] = r.z; v[3] = r.w;
  }
  static __device__ __forceinline__ void store_cg(float* p, const float (&v)[4]) {
    __stcg(reinterpret_cast<float4*>(p), make_float4(v[0], v[1], v[2], v[3]));
  }
  // store with an L2 eviction-priority policy (createpolicy)
  static __device__ __forceinline__ void store_hint(float* p, const float (&v)[4], uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(v[0]), "f"(v[1]),
                 "f"(v[2]), "f"(v[3]), "l"(pol)
                 : "memory");
  }
};

template <>
struct VecIO<double, 2> {
  static __device__ __forceinline__ void load_stream(const double* p, double (&v)[2]) {
    double2 r = __ldcs(reinterpret_cast<const double2*>(p));
    v[0] = r.x; v[1] = r.y;
  }
  static __device__ __forceinline__ void store_stream(double* p, const double (&v)[2]) {
    __stcs(reinterpret_cast<double2*>(p), make_double2(v[0], v[1]));
  }
  static __device__ __forceinline__ void load_cg(const double* p, double (&v)[2]) {
    double2 r = __ldcg(reinterpret_cast<const double2*>(p));
    v[0] = r.x; v[1] = r.y;
  }
  static __device__ __forceinline__ void store_cg(double* p, const double (&v)[2]) {
    __stcg(reinterpret_cast<double2*>(p), make_double2(v[0], v[1]));
  }
  static __device__ __forceinline__ void store_hint(double* p, const double (&v)[2], uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v[0]), "d"(v[1]), "l"(pol)
                 : "memory");
  }
};

template <class S>
struct VecIO1 {
  static __device__ __forceinline__ void load_stream(const S* p, S (&v)[1]) { v[0] = __ldcs(p); }
  static __device__ __forceinline__ void store_stream(S* p, const S (&v)[1]) { __stcs(p, v[0]); }
  static __device__ __forceinline__ void load_cg(const S* p, S (&v)[1]) { v[0] = __ldcg(p); }
  static __device__ __forceinline__ void store_cg(S* p, const S (&v)[1]) { __stcg(p, v[0]); }
};
template <>
struct VecIO<float, 1> : VecIO1<float> {};
template <>
struct VecIO<double, 1> : VecIO1<double> {};

// ---- arithmetic -------------------------------------------------------------
// One step of the recurrence, a fused multiply-add exactly as the reference
// build contracts `l[j] * prev[j] + v[j]` (recurrence.hpp:109).
__device__ __forceinline__ float fma_(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double fma_(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float mul_(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_(double a, double b) { return __dmul_rn(a, b); }

// ---- gpu-scope flag publish / acquire --------------------------------------
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void fence_acq_rel_gpu() {
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

// Spin watchdog: every wait loop of the look-back / mbarrier pipeline ticks
// one of these; a wait longer than 20 s traps (cudaErrorLaunchFailure) instead
// of wedging the GPU.  Checked every 1024 spins, so free on the fast path.
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
struct SpinGuard {
  uint64_t t0 = 0;
  uint32_t n = 0;
  __device__ __forceinline__ void tick() {
    if ((++n & 1023u) == 0u) {
      const uint64_t t = globaltimer_ns();
      if (t0 == 0) t0 = t;
      else if (t - t0 > 20000000000ull) __trap();
    }
  }
};

// Flag word: (epoch << 2) | state.  A flag whose epoch differs from the
// current launch's is "not yet written in this launch", so the flag array
// never needs clearing between launches.
enum : uint32_t { kFlagAgg = 1u, kFlagInc = 2u };

// Control block at the head of every workspace.  `epoch` advances once per
// launch (by the CTA that retires last), `ticket` hands out chunk ids in
// launch order (forward-progress guarantee of the look-back), `retired`
// counts finished CTAs.  Device-resident so the kernels are CUDA-graph
// replayable (no per-launch host state).
struct Ctrl {
  uint32_t epoch;
  uint32_t pad0;
  unsigned long long ticket;
  unsigned long long retired;
  // decay-adaptive stitch (segment.cu::k_decay_probe): the column fractions
  // summed by the probe's CTAs, their count, and the resulting mode word
  // (1 = deep) read by the launches that follow on this workspace
  float decay_sum;
  uint32_t decay_count;
  int32_t decay_mode;
  uint32_t pad2;
  unsigned long long pad1[3];
};
static_assert(sizeof(Ctrl) == 64, "Ctrl must be one 64-byte block");

__device__ __forceinline__ uint32_t next_epoch(uint32_t e) {
  uint32_t n = (e + 1u) & 0x3FFFFFFFu;
  return n == 0u ? 1u : n;
}

}  // namespace linrec_dev
