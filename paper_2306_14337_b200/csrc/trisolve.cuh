// K3 triangular solves and the permute/scale stages of solve_system.
#pragma once

#include "common.cuh"

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
  const int32_t* row_ptr;
  const int32_t* col;
  const int32_t* diag;
  const int32_t* order;   // rows in dependency-level order
  const double* values;
  const double* y;
  double* x;              // armed with the pending marker; each row publishes x[i]
  int32_t* counter;       // ticket
  int32_t* failed_row;    // upper only: atomicMax target, initialised to -1
};

// Reference: lower_core, src/trisolve.cpp:28-42 — x_i = y_i - sum_{d<i} l_id x_d over the
// strict-lower entries in ascending column order (kept: one thread accumulates one row, so x
// is bit-identical to the CPU result). Rows are claimed 32 at a time in level order; a thread
// that needs x_d waits on the value itself (Ginkgo's NaN-sentinel scheme).
__global__ void __launch_bounds__(128)
lower_kernel(const TriArgs a) {
  const int lane = threadIdx.x & 31;
  while (true) {
    int32_t r0 = 0;
    if (lane == 0) r0 = atomicAdd(a.counter, 32);
    r0 = __shfl_sync(0xffffffffu, r0, 0);
    if (r0 >= a.n) break;
    const int32_t r = r0 + lane;
    if (r < a.n) {
      const int32_t i = a.order[r];
      const int32_t lo = a.row_ptr[i], dg = a.diag[i];
      double acc = a.y[i];
      for (int32_t k = lo; k < dg; ++k) {
        const double xd = wait_value(a.x + a.col[k]);
        acc = sub_prod(acc, a.values[k], xd);  // src/trisolve.cpp:38
      }
      publish(a.x + i, acc);
    }
    __syncwarp();
  }
}

// Reference: upper_core, src/trisolve.cpp:46-68 — x_i = (y_i - sum_{j>i} u_ij x_j) / u_ii.
// An exactly zero diagonal is recorded (the highest such row is what the reference's
// lowest-virtual-index rule reports, src/trisolve.cpp:60-66) and the row still completes.
__global__ void __launch_bounds__(128)
upper_kernel(const TriArgs a) {
  const int lane = threadIdx.x & 31;
  while (true) {
    int32_t r0 = 0;
    if (lane == 0) r0 = atomicAdd(a.counter, 32);
    r0 = __shfl_sync(0xffffffffu, r0, 0);
    if (r0 >= a.n) break;
    const int32_t r = r0 + lane;
    if (r < a.n) {
      const int32_t i = a.order[r];
      const int32_t dg = a.diag[i], hi = a.row_ptr[i + 1];
      double acc = a.y[i];
      for (int32_t k = dg + 1; k < hi; ++k) {
        const double xj = wait_value(a.x + a.col[k]);
        acc = sub_prod(acc, a.values[k], xj);  // src/trisolve.cpp:57
      }
      const double d = a.values[dg];
      if (d == 0.0) atomicMax(a.failed_row, i);
      publish(a.x + i, acc / d);
    }
    __syncwarp();
  }
}

}  // namespace b200lu
