// K3 batched, U sweep with A TEAM OF WARPS PER ROW (B200LU_BATCH_UTEAM = warps per row, default 2). btri_kernel<true, .> (batch.cuh) parks
// the products of a row's entries 1.. in the warp's shared-memory buffer before it waits for the dependency of entry 0;
// that parking phase is a chain of dependent memory round trips (values, column -> x gather, 8 entries at a time), and the
// 16 KB buffer per row caps the rows in flight at 12 per SM. Here a team of two warps owns the row and the buffer: each
// member parks every other chunk of 8 entries, they meet at a named barrier, and member 0 finishes the row exactly as
// btri_kernel does (wait for x of entry 0, one multiply, the subtraction chain from shared memory in ascending column
// order — the reference's order, src/trisolve.cpp:57 — the entries beyond the buffer, the division, publication).
// Same arithmetic in the same order per scenario: x is bit-identical. Rows in flight are unchanged; the warps that work on
// them double. (Tried: member 0 requesting y_i, the diagonal, entry 0 and its x ahead of the parking phase — 90 registers,
// or 80 with a spill under a three-CTA launch bound: 4.06 ms per step against 3.62 at 256 scenarios, 2.44 against 2.03 at 32.)
#pragma once

#include "batch.cuh"

namespace b200lu {

constexpr int kTriTeams = 4;  // teams (rows in flight) per CTA of 8 warps

template <int kTriBuffered, int TS>
__global__ void __launch_bounds__(kTriTeams * TS * 32)
btri_upper_team_kernel(const BTriArgs a) {
  extern __shared__ __align__(16) double tri_team_smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int team = warp / TS, me = warp % TS;
  const unsigned full = 0xffffffffu;
  const unsigned long long total = static_cast<unsigned long long>(a.count) * a.groups;
  double* pb = tri_team_smem + static_cast<size_t>(team) * kTriBuffered * 32 + lane;
  auto barrier = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(team + 1), "n"(32 * TS) : "memory"); };
  const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * kTriTeams;
  for (unsigned long long t = static_cast<unsigned long long>(blockIdx.x) * kTriTeams + team; t < total; t += stride) {
    const int32_t r = static_cast<int32_t>(t / a.groups);
    const int32_t g = static_cast<int32_t>(t - static_cast<unsigned long long>(r) * a.groups);
    const int4 m4 = __ldg(reinterpret_cast<const int4*>(a.meta) + a.first + r);
    const int32_t i = m4.x, beg = m4.y, end = m4.z;
    const double* vg = a.values + static_cast<int64_t>(g) * a.nnz_factors * 32 + lane;
    double* xg = a.x + static_cast<int64_t>(g) * a.n * 32 + lane;
    const int32_t parked_end = min(end, beg + 1 + kTriBuffered);
    // ---- both members: products of entries [beg + 1, parked_end), chunk c by member c % TS, far columns first
    {
      const int32_t k_begin = beg + 1;
      const int32_t nchunk = (parked_end - k_begin + kTriChunk - 1) / kTriChunk;
      for (int32_t c = nchunk - 1 - ((nchunk - 1 - me + TS * 64) % TS); c >= 0; c -= TS) {  // the largest c with c % TS == me, then down
        const int32_t k = k_begin + c * kTriChunk;
        double v[kTriChunk], xv[kTriChunk];
        const double* xp[kTriChunk];
#pragma unroll
        for (int j = 0; j < kTriChunk; ++j) {
          v[j] = 0.0;
          xv[j] = 0.0;
          xp[j] = xg;
          if (k + j < parked_end) {
            v[j] = vg[static_cast<int64_t>(k + j) * 32];
            xp[j] = xg + static_cast<int64_t>(__ldg(a.col + k + j)) * 32;
            xv[j] = ld_l2(xp[j]);
          }
        }
#pragma unroll
        for (int j = kTriChunk - 1; j >= 0; --j) {
          if (k + j < parked_end) {  // warp-uniform
            unsigned backoff = 0;
            while (__any_sync(full, is_pending(xv[j]))) {
              if (backoff) __nanosleep(backoff);
              backoff = min(backoff + 32u, 128u);
              if (is_pending(xv[j])) xv[j] = ld_l2(xp[j]);
            }
            pb[static_cast<size_t>(k + j - k_begin) * 32] = __dmul_rn(v[j], xv[j]);
          }
        }
      }
    }
    barrier();  // every product is parked
    if (me == 0) {
      double acc = a.y[(static_cast<int64_t>(g) * a.n + i) * 32 + lane];
      const double dval = vg[static_cast<int64_t>(__ldg(a.diag + i)) * 32];
      if (beg < end) {
        const double v0 = vg[static_cast<int64_t>(beg) * 32];
        const double* xp0 = xg + static_cast<int64_t>(__ldg(a.col + beg)) * 32;
        double x0 = ld_l2(xp0);
        while (__any_sync(full, is_pending(x0))) {
          if (is_pending(x0)) x0 = ld_l2(xp0);
        }
        acc = sub_prod(acc, v0, x0);  // src/trisolve.cpp:57
        const int32_t np = parked_end - beg - 1;
        int32_t j = 0;
        for (; j + 8 <= np; j += 8) {
          double pv[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) pv[q] = pb[static_cast<size_t>(j + q) * 32];
#pragma unroll
          for (int q = 0; q < 8; ++q) acc = __dsub_rn(acc, pv[q]);
        }
        for (; j < np; ++j) acc = __dsub_rn(acc, pb[static_cast<size_t>(j) * 32]);
        // entries beyond the buffer (rows longer than it): folded in order behind the parked ones
        for (int32_t k = parked_end; k < end; k += kTriChunk) {
          double v[kTriChunk], xv[kTriChunk];
          const double* xp[kTriChunk];
#pragma unroll
          for (int q = 0; q < kTriChunk; ++q) {
            v[q] = 0.0;
            xv[q] = 0.0;
            xp[q] = xg;
            if (k + q < end) {
              v[q] = vg[static_cast<int64_t>(k + q) * 32];
              xp[q] = xg + static_cast<int64_t>(__ldg(a.col + k + q)) * 32;
              xv[q] = ld_l2(xp[q]);
            }
          }
#pragma unroll
          for (int q = 0; q < kTriChunk; ++q) {
            if (k + q < end) {
              unsigned backoff = 0;
              while (__any_sync(full, is_pending(xv[q]))) {
                if (backoff) __nanosleep(backoff);
                backoff = min(backoff + 32u, 256u);
                if (is_pending(xv[q])) xv[q] = ld_l2(xp[q]);
              }
              acc = sub_prod(acc, v[q], xv[q]);
            }
          }
        }
      }
      if (dval == 0.0) atomicMax(a.failed + g * 32 + lane, i);  // src/trisolve.cpp:60-66
      acc = acc / dval;
      publish(xg + static_cast<int64_t>(i) * 32, acc);
    }
    barrier();  // member 0 has read the buffer: it may be refilled
  }
}

}  // namespace b200lu
