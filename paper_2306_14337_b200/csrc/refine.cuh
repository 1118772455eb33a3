// K4 building blocks: CSR SpMV, fused residual + norms, deterministic dot, axpy / scale.
#pragma once

#include "common.cuh"

namespace b200lu {

constexpr int kReduceThreads = 256;

// Reference: spmv, src/sparse.cpp:135-141 — per-row left-to-right accumulation, kept so each
// y_i is bit-identical to the CPU value (one thread owns one row; K rows hold ~5.6 entries).
__global__ void __launch_bounds__(256)
spmv_kernel(int32_t n, const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
            const double* __restrict__ vals, const double* __restrict__ x, double* __restrict__ y) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double acc = 0.0;
  for (int32_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) acc = add_prod(acc, vals[k], x[col[k]]);
  y[i] = acc;
}

// Deterministic block reduction of up to 2 running sums; the last block to finish folds the
// per-block partials in index order, so results are identical run to run. (The reference's dot
// is one serial left-to-right sum, src/sparse.cpp:271-275; a parallel sum cannot reproduce its
// rounding, which is why refinement parity is stated on the residual, not on bits.)
template <int K>
__device__ __forceinline__ void block_reduce_finish(double (&v)[K], double* __restrict__ partials,
                                                    unsigned int* __restrict__ ticket,
                                                    double* __restrict__ out) {
  __shared__ double sh[K][kReduceThreads / 32];
  __shared__ bool is_last;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < K; ++q) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_down_sync(0xffffffffu, v[q], o);
    if (lane == 0) sh[q][w] = v[q];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < K; ++q) {
      double s = 0.0;
      for (int j = 0; j < kReduceThreads / 32; ++j) s += sh[q][j];
      partials[static_cast<size_t>(q) * gridDim.x + blockIdx.x] = s;
    }
    __threadfence();
    const unsigned int t = atomicAdd(ticket, 1u);
    is_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (is_last) {
    __threadfence();
#pragma unroll
    for (int q = 0; q < K; ++q) {
      double s = 0.0;
      for (unsigned int j = threadIdx.x; j < gridDim.x; j += kReduceThreads) {
        s += partials[static_cast<size_t>(q) * gridDim.x + j];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
      __syncthreads();
      if (lane == 0) sh[q][w] = s;
      __syncthreads();
      if (threadIdx.x == 0) {
        double tot = 0.0;
        for (int j = 0; j < kReduceThreads / 32; ++j) tot += sh[q][j];
        out[q] = tot;
      }
    }
    if (threadIdx.x == 0) *ticket = 0u;
  }
}

// r = b - A x with out[0] = sum r_i^2 and out[1] = sum b_i^2: the fused form of
// relative_residual (src/sparse.cpp:283-288) and true_relres (src/refine.cpp:30-35).
__global__ void __launch_bounds__(kReduceThreads)
residual_kernel(int32_t n, const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                const double* __restrict__ vals, const double* __restrict__ x,
                const double* __restrict__ b, double* __restrict__ r, double* __restrict__ partials,
                unsigned int* __restrict__ ticket, double* __restrict__ out) {
  double s[2] = {0.0, 0.0};
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int32_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) acc = add_prod(acc, vals[k], x[col[k]]);
    const double bi = b[i];
    const double ri = __dsub_rn(bi, acc);
    r[i] = ri;
    s[0] = add_prod(s[0], ri, ri);
    s[1] = add_prod(s[1], bi, bi);
  }
  block_reduce_finish<2>(s, partials, ticket, out);
}

// out[0] = sum a_i * b_i (dot, src/sparse.cpp:271-275).
__global__ void __launch_bounds__(kReduceThreads)
dot_kernel(int32_t n, const double* __restrict__ a, const double* __restrict__ b,
           double* __restrict__ partials, unsigned int* __restrict__ ticket,
           double* __restrict__ out) {
  double s[1] = {0.0};
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    s[0] = add_prod(s[0], a[i], b[i]);
  }
  block_reduce_finish<1>(s, partials, ticket, out);
}

// One Gram-Schmidt projection step of cgs2_orthonormalize (src/refine.cpp:13-17) with the
// coefficient kept on the device: h = *h_ptr; coef += h (thread 0); w -= h * q.
__global__ void __launch_bounds__(256)
project_out_kernel(int32_t n, const double* __restrict__ h_ptr, double* __restrict__ coef,
                   const double* __restrict__ q, double* __restrict__ w) {
  const double h = *h_ptr;
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) *coef = __dadd_rn(*coef, h);
  if (i < n) w[i] = add_prod(w[i], -h, q[i]);  // axpy(-h, q, w), src/sparse.cpp:279-281
}

// y += alpha * x (axpy, src/sparse.cpp:279-281).
__global__ void __launch_bounds__(256)
axpy_kernel(int32_t n, double alpha, const double* __restrict__ x, double* __restrict__ y) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = add_prod(y[i], alpha, x[i]);
}

// out = in / s (v0 = r / beta, src/refine.cpp:66; vector /= norm, src/refine.cpp:24).
__global__ void __launch_bounds__(256)
divide_kernel(int32_t n, double s, const double* __restrict__ in, double* __restrict__ out) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i] / s;
}

}  // namespace b200lu
