// Shared device helpers for the b200lu kernels (sm_100a, FP64 SIMT).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

namespace b200lu {

// "Not written yet" marker for values that other rows/CTAs wait on. A quiet NaN
// with a payload no arithmetic instruction produces; a computed value that
// happens to carry these bits is canonicalised before it is published
// (publish()), so a waiter can never mistake data for the marker or hang on it.
constexpr unsigned long long kPendingBits = 0xFFFA5A5AB200B200ull;
constexpr unsigned long long kCanonicalNaN = 0x7FF8000000000000ull;

__device__ __forceinline__ bool is_pending(double v) {
  return static_cast<unsigned long long>(__double_as_longlong(v)) == kPendingBits;
}

// L2-coherent (gpu-scope relaxed) 8-byte load/store: the unit of inter-CTA
// communication in the sync-free kernels. Each value is self-validating, so no
// fence or separate ready flag is needed.
__device__ __forceinline__ double ld_l2(const double* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p));
  return __longlong_as_double(static_cast<long long>(v));
}

__device__ __forceinline__ void st_l2(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p),
               "l"(static_cast<unsigned long long>(__double_as_longlong(v))));
}

__device__ __forceinline__ void publish(double* p, double v) {
  if (is_pending(v)) v = __longlong_as_double(static_cast<long long>(kCanonicalNaN));
  st_l2(p, v);
}

// Spins until *p has been published by its owner (no back-off: callers only spin on values
// whose producer is running or about to).
__device__ __forceinline__ double wait_value(const double* p) {
  double v = ld_l2(p);
  while (is_pending(v)) v = ld_l2(p);
  return v;
}

__device__ __forceinline__ int32_t ld_l2_s32(const int32_t* p) {
  int32_t v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ void red_add_s32(int32_t* p, int32_t v) {
  asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v));
}

// Throttle of a sync-free sweep: a claimed row sleeps until `start` rows of the sweep have
// finished (schedule.hpp, fill_start_thresholds). One lane polls one counter, with a sleep
// proportional to how far away the row still is; `seen` caches the last value read (the
// counter only grows), so rows whose threshold is already known to be met cost nothing.
__device__ __forceinline__ void wait_for_start(const int32_t* finished, int32_t start, int lane, int32_t& seen) {
  if (start > seen) {
    int32_t c = 0;
    if (lane == 0) {
      c = ld_l2_s32(finished);
      while (c < start) {
        __nanosleep(min(4000, max(64, (start - c) * 4)));
        c = ld_l2_s32(finished);
      }
    }
    seen = __shfl_sync(0xffffffffu, c, 0);
  }
}

// Read-only loads pinned in program order (asm volatile): used where a software pipeline issues
// the next item's loads early and the compiler must not sink them to their first use.
__device__ __forceinline__ double ldg_pinned(const double* p) {
  unsigned long long v;
  asm volatile("ld.global.nc.b64 %0, [%1];" : "=l"(v) : "l"(p));
  return __longlong_as_double(static_cast<long long>(v));
}
__device__ __forceinline__ int2 ldg_pinned(const int2* p) {
  int2 v;
  asm volatile("ld.global.nc.v2.s32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ int4 ldg_pinned(const int4* p) {
  int4 v;
  asm volatile("ld.global.nc.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
// Plain (coherent) pinned load for data written by an earlier kernel on the same stream.
__device__ __forceinline__ double ld_pinned(const double* p) {
  unsigned long long v;
  asm volatile("ld.global.b64 %0, [%1];" : "=l"(v) : "l"(p));
  return __longlong_as_double(static_cast<long long>(v));
}

// a - b*c with two roundings (the reference's x86-64 baseline build has no FMA
// contraction: src/numeric.cpp:44, src/trisolve.cpp:38,57).
__device__ __forceinline__ double sub_prod(double a, double b, double c) {
  return __dsub_rn(a, __dmul_rn(b, c));
}
__device__ __forceinline__ double add_prod(double a, double b, double c) {
  return __dadd_rn(a, __dmul_rn(b, c));
}

// Launch of a kernel whose claim order is STATIC (warp w takes units w, w + W, ...): such a kernel is
// deadlock-free only when its whole grid is co-resident, because the owner of the lowest unfinished
// unit must be running. A cooperative launch makes the driver guarantee exactly that — the grid is
// scheduled as a whole, waiting for SMs if another handle's kernel (or another MPS client) occupies
// them — and fails at launch time (cudaErrorCooperativeLaunchTooLarge) if the grid could never fit,
// instead of hanging the device.
template <typename Arg>
inline cudaError_t launch_resident(void (*kernel)(Arg), int grid, int block, size_t smem, cudaStream_t stream, Arg arg) {
  void* params[] = {&arg};
  static const bool plain = [] { const char* e = getenv("B200LU_COOP_LAUNCH"); return e && e[0] == '0'; }();
  if (plain) return cudaLaunchKernel(reinterpret_cast<const void*>(kernel), dim3(grid), dim3(block), params, smem, stream);
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kernel), dim3(grid), dim3(block), params, smem, stream);
}

}  // namespace b200lu
