// Update destination table and the per-row claim record of the refactorization kernels
// (templates only: shared by the single-system and the scenario-batch translation units).
#pragma once

#include "common.cuh"

namespace b200lu {

// One record per claim position of a refactorization queue (rows in dependency-level order).
struct FactorMeta {
  int32_t row, lo, dg, hi;
};

// --------------------------------------------------- update destination table
//
// For the pivot (i, d) — row i has a strict-lower entry in column d — every upper entry
// (d, j) of row d updates slot (i, j). The reference finds that slot through
// RowLookupTable::lookup (src/symbolic.cpp:73-93) once per update, every factorization.
// The pattern is fixed, so the offsets are resolved ONCE here and streamed afterwards:
// dest[pair_row_ptr[i] + running pair index] = offset of column j inside row i.
template <typename DestT>
__global__ void __launch_bounds__(256)
build_dest_kernel(int32_t n, const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                  const int32_t* __restrict__ diag, const int64_t* __restrict__ pair_row_ptr,
                  DestT* __restrict__ dest) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t i = warp; i < n; i += nwarps) {
    const int32_t lo = row_ptr[i], dg = diag[i], hi = row_ptr[i + 1];
    int64_t p = pair_row_ptr[i];
    for (int32_t k = lo; k < dg; ++k) {
      const int32_t d = col[k];
      const int32_t dd = diag[d];
      const int32_t m = row_ptr[d + 1] - dd - 1;
      for (int32_t c = lane; c < m; c += 32) {
        const int32_t j = col[dd + 1 + c];
        // binary search for j in col[k+1, hi); the fill pattern is closed under row
        // updates (src/numeric.cpp:43), so j is always present.
        int32_t a = k + 1, b = hi - 1;
        while (a < b) {
          const int32_t mid = (a + b) >> 1;
          if (col[mid] < j) a = mid + 1; else b = mid;
        }
        dest[p + c] = static_cast<DestT>(a - lo);
      }
      p += m;
    }
  }
}

}  // namespace b200lu
