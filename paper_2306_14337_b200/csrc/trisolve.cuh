// K3 triangular solves and the permute/scale stages of solve_system.
#pragma once

#include "common.cuh"
#include "schedule.hpp"

namespace b200lu {

// solve_system prologue, src/trisolve.cpp:98-105: w[p(i)] = D_r[i] * b[i] (D_r absent on the
// KLU-style path). Also arms the two solve buffers with the pending marker.
__global__ void __launch_bounds__(256)
permute_in_kernel(int32_t n, const int32_t* __restrict__ p, const double* __restrict__ row_scale,
                  const double* __restrict__ b, double* __restrict__ w, double* __restrict__ t1,
                  double* __restrict__ t2) {
  const double pending = __longlong_as_double(static_cast<long long>(kPendingBits));
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double v = b[i];
  if (row_scale != nullptr) v = __dmul_rn(row_scale[i], v);
  w[p[i]] = v;
  t1[i] = pending;
  t2[i] = pending;
}

// solve_system epilogue, src/trisolve.cpp:110-118: x[j] = D_c[j] * t[p(q(j))]; pq = p∘q
// (== p when no matching).
__global__ void __launch_bounds__(256)
permute_out_kernel(int32_t n, const int32_t* __restrict__ pq, const double* __restrict__ col_scale,
                   const double* __restrict__ t, double* __restrict__ x) {
  const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double v = t[pq[j]];
  if (col_scale != nullptr) v = __dmul_rn(col_scale[j], v);
  x[j] = v;
}

__global__ void __launch_bounds__(256)
fill_pending_kernel(int64_t n, double* __restrict__ x) {
  const double pending = __longlong_as_double(static_cast<long long>(kPendingBits));
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) x[i] = pending;
}

struct TriArgs {
  int32_t n;
  const RowMeta* meta;    // per claim position, dependency-level order
  const int32_t* col;
  const int32_t* diag;
  const double* values;
  const double* y;
  double* x;              // armed with the pending marker; each row publishes x[i]
  int32_t* counter;       // claim ticket
  int32_t* finished;      // rows finished so far in this sweep
  int32_t* failed_row;    // upper only: atomicMax target, initialised to -1
};

// Reference: lower_core (src/trisolve.cpp:28-42): x_i = y_i - sum_{d<i} l_id x_d, and
// upper_core (46-68): x_i = (y_i - sum_{j>i} u_ij x_j) / u_ii, rows in descending order.
//
// One warp owns one row, claimed in dependency-level order. The 32 lanes fetch 32 entries at a
// time (coalesced value/column loads, a gather of x; the next chunk is in flight while the
// current one is folded) and each lane waits on the x it needs — the value itself is the ready
// flag (Ginkgo's NaN-sentinel scheme). The products are folded into the
// accumulator ONE AT A TIME, consuming every already-available leading entry while later ones
// are still in flight, so when the last dependency lands only its own term is left to add.
//
// Fold order. kDescending == false walks the entries in ascending column order, the
// reference's summation order (src/trisolve.cpp:38,57): x is then bit-identical to the CPU
// result. For L that is also the order in which the dependencies are produced. For U the
// dependencies are produced in DESCENDING column order (row i+1 finishes last and is the first
// entry of row i), so the ascending fold leaves the whole row on the critical path behind its
// last arrival; kDescending == true folds U rows from the last column to the first instead:
// same terms, fixed (deterministic) order, different rounding of the partial sums.
//
// An exactly zero U diagonal is recorded (the highest such row is what the reference's
// lowest-virtual-index rule reports, src/trisolve.cpp:60-66) and the row still completes.
template <bool kUpper, bool kDescending>
__global__ void __launch_bounds__(256)
tri_kernel(const TriArgs a) {
  const int lane = threadIdx.x & 31;
  const unsigned full = 0xffffffffu;
  while (true) {
    int32_t r = 0;
    if (lane == 0) r = atomicAdd(a.counter, 1);
    r = __shfl_sync(full, r, 0);
    if (r >= a.n) break;
    const int4 m4 = __ldg(reinterpret_cast<const int4*>(a.meta) + r);
    const int32_t i = m4.x, beg = m4.y, end = m4.z;
    double acc = a.y[i];
    double dval = 1.0;
    if (kUpper) dval = a.values[beg - 1];  // u_ii sits right before the strict-upper entries
    wait_for_start(a.finished, m4.w, lane);

    // entry handled by this lane in chunk c (chunks and lanes walk the row in fold order)
    auto entry = [&](int32_t c) { return kDescending ? end - 1 - (c * 32 + lane) : beg + c * 32 + lane; };
    const int32_t nent = end - beg;
    const int32_t nchunks = (nent + 31) >> 5;
    const double* xp = a.x;
    double v = 0.0, xv = 0.0;
    if (lane < nent) {
      const int32_t k = entry(0);
      v = a.values[k];
      xp = a.x + __ldg(a.col + k);
      xv = ld_l2(xp);
    }
    for (int32_t c = 0; c < nchunks; ++c) {
      // software pipeline: issue the next chunk's loads before folding this one
      const double* xp_next = a.x;
      double v_next = 0.0, xv_next = 0.0;
      if ((c + 1) * 32 + lane < nent) {
        const int32_t k = entry(c + 1);
        v_next = a.values[k];
        xp_next = a.x + __ldg(a.col + k);
        xv_next = ld_l2(xp_next);
      }
      const int32_t cnt = min(32, nent - c * 32);
      int32_t q = 0;
      while (q < cnt) {
        const unsigned ready = __ballot_sync(full, !is_pending(xv));
        const unsigned from_q = ~(ready >> q);  // bit t set <=> entry q+t is still pending
        int32_t run = from_q == 0u ? 32 : __ffs(static_cast<int>(from_q)) - 1;
        run = min(run, cnt - q);
        const double prod = __dmul_rn(v, xv);
#pragma unroll 8
        for (int32_t t = 0; t < run; ++t) acc = __dsub_rn(acc, __shfl_sync(full, prod, q + t));
        q += run;
        if (q < cnt && is_pending(xv)) xv = ld_l2(xp);
      }
      v = v_next;
      xp = xp_next;
      xv = xv_next;
    }
    if (kUpper) {
      if (lane == 0 && dval == 0.0) atomicMax(a.failed_row, i);
      acc = acc / dval;
    }
    if (lane == 0) {
      publish(a.x + i, acc);
      red_add_s32(a.finished, 1);
    }
  }
}

}  // namespace b200lu
