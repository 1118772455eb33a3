// K2 batched, trailing part, SUPERNODAL form (plan and rationale: snode_plan.hpp). A warp owns a block of R
// consecutive rows x 32 scenarios (lane = scenario) and walks the block's runs of up to 8 consecutive pivot rows
// with nested upper patterns:
//   phase A  the run's multipliers of each block row, a dense forward substitution with the run's diagonal block —
//            kept in REGISTERS (statically indexed: the loops over the run are unrolled);
//   phase B  every destination entry of the run is loaded once, receives its s updates in a register in ascending
//            pivot order (product rounded on its own, then the subtraction: src/numeric.cpp:44) and is stored once;
//            the pivot rows' entries are read at fixed offsets, the only index data is one destination list per
//            (row, run).
// No L2 reductions, no per-update index, and the upper entries of a pivot row are loaded once for both block rows.
// Every access to `values` is served by L2 (ld.relaxed.gpu / st.global.cg); dependencies as in batch.cuh (ready flag
// per (row, group), ld.acquire.gpu by one lane per awaited row, then __syncwarp).
#pragma once

#include "batch.cuh"
#include "snode_plan.hpp"

namespace b200lu {

struct BSnodeArgs {
  int32_t n_blocks, units, gen;
  const SBlock* blocks;
  const SRun* runs;
  const uint32_t* dest;
  const int32_t* diag;
  double* values;
  int64_t nnz_factors;
  int32_t* flags;
  double pivot_floor;
  int32_t* failed;
  unsigned long long* ticket;
};


// Phase B of one window of up to 32 destination entries (slots in dsw, one per lane): SC = compile-time cap of the
// run length, T = entries whose loads are in flight together.
template <int R, int SC, int T>
__device__ __forceinline__ void phase_b(double* g, const double (&alpha)[R][kSnodeMax], const int32_t (&ub)[kSnodeMax],
                                        const uint32_t (&dsw)[R], uint32_t mask, int s, int32_t w0, int32_t wn) {
  const unsigned full = 0xffffffffu;
  for (int32_t t0 = 0; t0 < wn; t0 += T) {
    double acc[R][T], uv[SC][T];
    uint32_t ds[R][T];
#pragma unroll
    for (int tt = 0; tt < T; ++tt) {
      const bool on = t0 + tt < wn;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        ds[r][tt] = __shfl_sync(full, dsw[r], (t0 + tt) & 31);
        acc[r][tt] = 0.0;
        if (on && (mask & (1u << r))) acc[r][tt] = ld_cg(g + static_cast<int64_t>(ds[r][tt]) * 32);
      }
#pragma unroll
      for (int k = 0; k < SC; ++k) {
        uv[k][tt] = 0.0;
        if (on && k < s) uv[k][tt] = ld_cg(g + static_cast<int64_t>(ub[k] + w0 + t0 + tt) * 32);
      }
    }
#pragma unroll
    for (int k = 0; k < SC; ++k) {
      if (k < s) {
#pragma unroll
        for (int tt = 0; tt < T; ++tt) {
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (mask & (1u << r)) acc[r][tt] = __dsub_rn(acc[r][tt], __dmul_rn(alpha[r][k], uv[k][tt]));  // src/numeric.cpp:44
          }
        }
      }
    }
#pragma unroll
    for (int tt = 0; tt < T; ++tt) {
      if (t0 + tt < wn) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (mask & (1u << r)) st_cg(g + static_cast<int64_t>(ds[r][tt]) * 32, acc[r][tt]);
        }
      }
    }
  }
}

template <int R, int MINB>
__global__ void __launch_bounds__(256, MINB)
bfactor_snode_kernel(const BSnodeArgs a) {
  constexpr int S = kSnodeMax;
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const unsigned long long total = static_cast<unsigned long long>(a.n_blocks) * a.units;
  while (true) {
    unsigned long long tk = 0;
    if (lane == 0) tk = atomicAdd(a.ticket, 1ull);
    tk = __shfl_sync(full, tk, 0);
    if (tk >= total) break;
    const int32_t b = static_cast<int32_t>(tk / a.units);
    const int32_t u = static_cast<int32_t>(tk - static_cast<unsigned long long>(b) * a.units);
    const int4 bk0 = __ldg(reinterpret_cast<const int4*>(a.blocks + b));
    const int32_t run_beg = bk0.x, run_end = bk0.y;
    const int32_t brow[2] = {bk0.z, bk0.w};
    double* g = a.values + static_cast<int64_t>(u) * a.nnz_factors * 32 + lane;

    for (int32_t ri = run_beg; ri < run_end; ++ri) {
      const int4 h0 = __ldg(reinterpret_cast<const int4*>(a.runs + ri));
      const int4 h1 = __ldg(reinterpret_cast<const int4*>(a.runs + ri) + 1);
      const int32_t d0 = h0.x, nj = h0.z;
      const uint32_t bytes = static_cast<uint32_t>(h0.y);
      const int s = static_cast<int>(bytes & 0xffu);
      const uint32_t mask = (bytes >> 8) & 0xffu, pub = (bytes >> 16) & 0xffu, wait = bytes >> 24;
      const uint32_t dest_beg = static_cast<uint32_t>(h0.w);
      const int32_t lslot[2] = {h1.x, h1.y};
      int32_t myd = 0;
      if (lane < s) {
        myd = __ldg(a.diag + d0 + lane);
        if (wait) wait_flag(a.flags + static_cast<int64_t>(d0 + lane) * a.units + u, a.gen);
      }
      __syncwarp();
      int32_t dsl[S];
#pragma unroll
      for (int k = 0; k < S; ++k) dsl[k] = __shfl_sync(full, myd, k);

      // ---- phase A: alpha[r][k] = (a(r, d0+k) - sum_{e<k} alpha[r][e] * u(d0+e, d0+k)) / u(d0+k, d0+k)
      double alpha[R][S];
#pragma unroll
      for (int k = 0; k < S; ++k) {
#pragma unroll
        for (int r = 0; r < R; ++r) alpha[r][k] = 0.0;
        if (k < s) {  // warp-uniform
          double acc[R], uu[S];
#pragma unroll
          for (int r = 0; r < R; ++r) {
            acc[r] = 0.0;
            if (mask & (1u << r)) acc[r] = ld_cg(g + static_cast<int64_t>(lslot[r] + k) * 32);
          }
#pragma unroll
          for (int e = 0; e < k; ++e) uu[e] = ld_cg(g + static_cast<int64_t>(dsl[e] + (k - e)) * 32);
          const double udd = ld_cg(g + static_cast<int64_t>(dsl[k]) * 32);
#pragma unroll
          for (int e = 0; e < k; ++e) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
              if (mask & (1u << r)) acc[r] = __dsub_rn(acc[r], __dmul_rn(alpha[r][e], uu[e]));  // src/numeric.cpp:44
            }
          }
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (mask & (1u << r)) {
              alpha[r][k] = acc[r] / udd;  // src/numeric.cpp:40
              st_cg(g + static_cast<int64_t>(lslot[r] + k) * 32, alpha[r][k]);  // l_id, src/numeric.cpp:41
            }
          }
        }
      }

      // ---- phase B: the run's destination entries. The loads of T entries are in flight together; T is chosen
      // by the length of the run (T x s pivot-row loads + R x T destination loads per step), so that the short runs at
      // the end of a row's pivot list — the ones on the critical path — cost a few memory round trips in all. The
      // destination slots of 32 entries per row are fetched by the lanes at once and broadcast with shuffles.
      const uint32_t* dp[R];
      {
        uint32_t off = dest_beg;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          dp[r] = a.dest + off;
          if (mask & (1u << r)) off += static_cast<uint32_t>(nj);
        }
      }
      int32_t ub[S];
#pragma unroll
      for (int k = 0; k < S; ++k) ub[k] = dsl[k] + (s - k);  // slot of u(d0+k, J[0])
      for (int32_t w0 = 0; w0 < nj; w0 += 32) {
        uint32_t dsw[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          dsw[r] = 0;
          if ((mask & (1u << r)) && w0 + lane < nj) dsw[r] = __ldg(dp[r] + w0 + lane);
        }
        const int32_t wn = min(32, nj - w0);
        if (s == 1) {
          phase_b<R, 1, 8>(g, alpha, ub, dsw, mask, s, w0, wn);
        } else if (s == 2) {
          phase_b<R, 2, 4>(g, alpha, ub, dsw, mask, s, w0, wn);
        } else if (s <= 4) {
          phase_b<R, 4, 2>(g, alpha, ub, dsw, mask, s, w0, wn);
        } else {
          phase_b<R, S, 2>(g, alpha, ub, dsw, mask, s, w0, wn);
        }
      }

      // ---- rows whose last pivot was in this run: pivot check (src/numeric.cpp:48) and publication
      if (pub) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (pub & (1u << r)) {
            const double dv = ld_cg(g + static_cast<int64_t>(__ldg(a.diag + brow[r])) * 32);  // after this thread's own stores
            if (fabs(dv) <= a.pivot_floor) atomicMin(a.failed + u * 32 + lane, brow[r]);
          }
        }
        __syncwarp();
        if (lane == 0) {
          __threadfence();
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (pub & (1u << r)) st_relaxed_s32(a.flags + static_cast<int64_t>(brow[r]) * a.units + u, a.gen);
          }
        }
      }
    }
    __syncwarp();
  }
}

}  // namespace b200lu
