// K1 value scatter and K2 numeric refactorization.
#pragma once

#include "common.cuh"
#include "dest.cuh"

namespace b200lu {

// ------------------------------------------------------------------ K1 scatter
//
// Reference: scatter_values, src/numeric.cpp:19-22 — out.assign(nnzF, 0) then
// out[scatter_map[k]] = A.values[k] * scatter_scale[k].
//
// One fused pass in gather form: slot s reads its source entry through the inverse map
// (src_of_slot[s] < 0 marks a fill slot, which becomes exactly 0), so every store is
// coalesced and no slot is written twice. The same pass re-arms `values` with the pending
// marker that the refactorization kernel's waiters test for — except in rows without a
// strict-lower entry (76 % of the rows of a KKT system after AMD): elimination leaves such a row
// unchanged (src/numeric.cpp:36 never iterates), so its scattered values ARE its factor
// values and are published right here; the refactorization kernel never sees those rows.
constexpr int32_t kTrivialBit = 0x40000000;  // src_of_slot flag: slot of a row without pivots
constexpr int32_t kTrivialFill = -2;         // fill slot of such a row (-1: fill slot of any other row)
__global__ void __launch_bounds__(256)
scatter_kernel(int64_t nnz_factors, const int32_t* __restrict__ src_of_slot,
               const double* __restrict__ a_values, const double* __restrict__ scatter_scale,
               double* __restrict__ work, double* __restrict__ values) {
  const double pending = __longlong_as_double(static_cast<long long>(kPendingBits));
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < nnz_factors;
       s += stride) {
    const int32_t code = __ldg(src_of_slot + s);
    const bool trivial = code >= 0 ? (code & kTrivialBit) != 0 : code == kTrivialFill;
    double v = 0.0;
    if (code >= 0) {
      const int32_t k = code & ~kTrivialBit;
      v = __ldg(a_values + k);
      if (scatter_scale != nullptr) v = __dmul_rn(v, __ldg(scatter_scale + k));
    }
    work[s] = v;
    // a directly published value that carries the marker's bit pattern (an input NaN payload) would
    // make every dependent row wait forever: canonicalise it, as publish() does for computed rows
    if (trivial && is_pending(v)) v = __longlong_as_double(static_cast<long long>(kCanonicalNaN));
    values[s] = trivial ? v : pending;
  }
}

// On-device value path of assemble_kkt (src/kkt.cpp:53-77). Across a barrier sequence, and under
// the regularization escalation of cli::solve_sequence (src/cli.cpp:148-154), only the diagonal of
// K = [[H + D_y + delta_p I, J^T], [J, -delta_d I]] changes: the reference sums the two COO
// entries of a primal diagonal slot, K_ii = H_ii + (D_y[i] + delta_p), and stores -delta_d in the
// dual ones. The off-diagonal values stay where the last reset_values put them.
__global__ void __launch_bounds__(256)
kkt_diagonal_kernel(int32_t n_total, int32_t n_primal, const double* __restrict__ h_diag,
                    const int32_t* __restrict__ diag_source_pos, const double* __restrict__ d_y, double delta_p,
                    double delta_d, double* __restrict__ a_values) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_total) return;
  a_values[diag_source_pos[i]] = i < n_primal ? __dadd_rn(h_diag[i], __dadd_rn(d_y[i], delta_p)) : -delta_d;
}

// Pivot check of the rows K1 published directly (src/numeric.cpp:48 applies to every row).
__global__ void __launch_bounds__(256)
trivial_pivot_kernel(int32_t count, const int32_t* __restrict__ rows, const int32_t* __restrict__ diag,
                     const double* __restrict__ work, double pivot_floor, int32_t* failed_row) {
  const int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count) return;
  const int32_t i = rows[t];
  if (fabs(work[diag[i]]) <= pivot_floor) atomicMin(failed_row, i);
}

// ------------------------------------------------------ K2 refactorization
//
// Reference: eliminate, src/numeric.cpp:27-58, driven by SyncFreeScheduler
// (include/rlu/schedule.hpp:49-79).
//
// Row ownership is kept: one warp owns row i from start to finish and applies the pivots d
// in ascending order, so every slot receives its updates in the reference's order and the
// result is bit-identical to the sequential CPU run regardless of scheduling. What changes:
//   * rows are claimed in dependency-level order from two queues (rows a warp slot can hold,
//     and wide rows that use the CTA's wide slot) by persistent warps, so a row starts long
//     before its last dependency finishes and consumes its already-final pivots ahead of time;
//   * row i is staged in shared memory while its pivots are applied;
//   * there are no ready flags: a finished row publishes its diagonal and upper entries into
//     `values`, which K1 armed with the pending marker; a consumer simply waits on the 8-byte
//     values it needs (Ginkgo's sentinel idea, applied to the factorization);
//   * the column->slot lookup is the precomputed destination table, streamed once;
//   * the loads of kPivotGroup consecutive pivots (diagonal, upper entries, destinations) are
//     issued together before the first of them is consumed, so a row with hundreds of
//     finished pivots is bound by throughput, not by one memory round trip per pivot.
struct FactorArgs {
  int32_t n_small, n_big;
  int32_t small_slot, big_slot;  // capacities in doubles
  const int32_t* row_ptr;
  const int32_t* col;
  const int32_t* diag;
  const FactorMeta* small_meta;  // per claim position of the two queues
  const FactorMeta* big_meta;
  const int64_t* pair_row_ptr;
  const void* dest;
  double* work;     // scattered input values (K1), also the in-place fallback for over-wide rows
  double* values;   // published factors
  double pivot_floor;
  int32_t* counters;  // [0] small-queue ticket, [1] big-queue ticket
  int32_t* failed_row;  // atomicMin target, initialised to INT32_MAX
};

template <typename DestT, int kPivotGroup>
__device__ __forceinline__ void factor_row(const FactorArgs& a, const FactorMeta mt, double* row, int lane) {
  const unsigned full = 0xffffffffu;
  const int32_t i = mt.row, lo = mt.lo, dg = mt.dg, hi = mt.hi;
  const int32_t len = hi - lo, nl = dg - lo;
  const DestT* __restrict__ dest = static_cast<const DestT*>(a.dest);
  const double* values = a.values;

  if (row != a.work + lo) {
    for (int32_t c = lane; c < len; c += 32) row[c] = a.work[lo + c];
  }
  __syncwarp();

  int64_t p = nl > 0 ? a.pair_row_ptr[i] : 0;
  for (int32_t k0 = 0; k0 < nl; k0 += 32) {
    // Lane q of this chunk resolves the metadata of pivot k0+q; the walk below is sequential.
    int32_t my_dd = 0, my_m = 0;
    if (k0 + lane < nl) {
      const int32_t d = __ldg(a.col + lo + k0 + lane);
      my_dd = __ldg(a.diag + d);
      my_m = __ldg(a.row_ptr + d + 1) - my_dd - 1;
    }
    const int32_t cnt = min(32, nl - k0);
    for (int32_t q0 = 0; q0 < cnt; q0 += kPivotGroup) {
      int32_t dd[kPivotGroup], m[kPivotGroup], s0[kPivotGroup], s1[kPivotGroup];
      int64_t pg[kPivotGroup];
      double ud[kPivotGroup], u0[kPivotGroup], u1[kPivotGroup];
#pragma unroll
      for (int g = 0; g < kPivotGroup; ++g) {
        const int32_t q = q0 + g;
        dd[g] = __shfl_sync(full, my_dd, q & 31);
        m[g] = __shfl_sync(full, my_m, q & 31);
        if (q >= cnt) m[g] = -1;  // no such pivot
        pg[g] = p;
        p += max(m[g], 0);
        ud[g] = 1.0; u0[g] = 0.0; u1[g] = 0.0; s0[g] = 0; s1[g] = 0;
        if (m[g] >= 0) ud[g] = ld_l2(values + dd[g]);
        if (lane < m[g]) { u0[g] = ld_l2(values + dd[g] + 1 + lane); s0[g] = dest[pg[g] + lane]; }
        if (lane + 32 < m[g]) { u1[g] = ld_l2(values + dd[g] + 33 + lane); s1[g] = dest[pg[g] + 32 + lane]; }
      }
#pragma unroll
      for (int g = 0; g < kPivotGroup; ++g) {
        if (m[g] < 0) break;  // warp-uniform
        const bool h0 = lane < m[g], h1 = lane + 32 < m[g];
        // One combined wait: whatever is still pending is re-read until the producer's
        // publication (diagonal and upper entries of row d) has landed.
        // While waiting, the still-pending values of the LATER pivots of the group are re-read
        // too (their loads overlap this wait), so a run of just-finished pivots costs one round
        // trip instead of one per pivot.
        while (__any_sync(full, is_pending(ud[g]) || is_pending(u0[g]) || is_pending(u1[g]))) {
#pragma unroll
          for (int e = g; e < kPivotGroup; ++e) {
            if (is_pending(ud[e])) ud[e] = ld_l2(values + dd[e]);
            if (is_pending(u0[e])) u0[e] = ld_l2(values + dd[e] + 1 + lane);
            if (is_pending(u1[e])) u1[e] = ld_l2(values + dd[e] + 33 + lane);
          }
        }
        const int32_t k = k0 + q0 + g;
        const double alpha = row[k] / ud[g];  // src/numeric.cpp:40
        if (h0) row[s0[g]] = sub_prod(row[s0[g]], alpha, u0[g]);  // src/numeric.cpp:44
        if (h1) row[s1[g]] = sub_prod(row[s1[g]], alpha, u1[g]);
        for (int32_t c = lane + 64; c < m[g]; c += 32) {
          const double u = wait_value(values + dd[g] + 1 + c);
          const int32_t s = dest[pg[g] + c];
          row[s] = sub_prod(row[s], alpha, u);
        }
        // l_id is final (src/numeric.cpp:41); nothing waits on strict-lower entries during the
        // factorization, so a plain store is enough.
        if (lane == 0) a.values[lo + k] = alpha;
        __syncwarp();
      }
    }
  }

  // src/numeric.cpp:48: the row completes (and is published) even when its pivot fails, so
  // dependents never hang (include/rlu/schedule.hpp:29-33); the lowest failing row wins (82-87).
  // Publish what other rows wait on first: the diagonal and the upper entries.
  for (int32_t c = nl + lane; c < len; c += 32) publish(a.values + lo + c, row[c]);
  if (lane == 0 && fabs(row[nl]) <= a.pivot_floor) atomicMin(a.failed_row, i);
}

template <typename DestT, int WARPS, int kPivotGroup, int kMinBlocks>
__global__ void __launch_bounds__(WARPS * 32, kMinBlocks)
factor_kernel(const FactorArgs a) {
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  double* small_slot = smem + static_cast<size_t>(w) * a.small_slot;
  double* big_slot = smem + static_cast<size_t>(WARPS) * a.small_slot;

  // Warp 0 of every CTA serves the wide-row queue first (it alone may use the wide slot).
  if (w == 0) {
    while (true) {
      int32_t r = 0;
      if (lane == 0) r = atomicAdd(a.counters + 1, 1);
      r = __shfl_sync(0xffffffffu, r, 0);
      if (r >= a.n_big) break;
      const int4 m4 = __ldg(reinterpret_cast<const int4*>(a.big_meta) + r);
      const FactorMeta mt{m4.x, m4.y, m4.z, m4.w};
      double* row = (mt.hi - mt.lo) <= a.big_slot ? big_slot : a.work + mt.lo;
      factor_row<DestT, kPivotGroup>(a, mt, row, lane);
      __syncwarp();
    }
  }
  while (true) {
    int32_t r = 0;
    if (lane == 0) r = atomicAdd(a.counters, 1);
    r = __shfl_sync(0xffffffffu, r, 0);
    if (r >= a.n_small) break;
    const int4 m4 = __ldg(reinterpret_cast<const int4*>(a.small_meta) + r);
    factor_row<DestT, kPivotGroup>(a, FactorMeta{m4.x, m4.y, m4.z, m4.w}, small_slot, lane);
    __syncwarp();
  }
}

}  // namespace b200lu
