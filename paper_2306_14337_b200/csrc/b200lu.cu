// b200lu — handle, host-side orchestration and the C ABI declared in include/b200lu.h.
//
// The host side mirrors the reference's NumericFactors / SolveWorkspace life cycle
// (include/rlu/numeric.hpp:22-53, include/rlu/trisolve.hpp:12-39) and the control flow of
// fgmres_refine / classic_refine (src/refine.cpp:39-188); all arithmetic on vectors and
// factors runs in the kernels of factor.cuh / trisolve.cuh / refine.cuh.
#include "b200lu.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "factor.cuh"
#include "refine.cuh"
#include "schedule.hpp"
#include "trisolve.cuh"

using namespace b200lu;

namespace {

constexpr int kFactorWarps = 8;
constexpr int kMaxBigSlot = 20 * 1024; // doubles; wider rows fall back to in-place global updates
constexpr int kMaxTailRows = 24576;     // rows of an on-chip tail (ScheduleTuning::tail_capacity is capped to this)
constexpr int kReduceBlocks = 592;     // 4 per SM on a 148-SM part; fixed so sums are reproducible

__global__ void arm_factor_kernel(int32_t* counters, int32_t* failed_row) {
  counters[0] = 0;
  counters[1] = 0;
  counters[2] = 0;
  *failed_row = INT_MAX;
}
__global__ void arm_solve_kernel(int32_t* counters, int32_t* failed_upper) {
  counters[4] = 0;  // lower ticket
  counters[5] = 0;  // upper ticket
  counters[6] = 0;  // lower rows finished
  counters[7] = 0;  // upper rows finished
  *failed_upper = -1;
}

}  // namespace

struct b200lu_handle {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool owns_stream = false;
  double pivot_floor = 1e-30;
  int refine_capacity = 20;
  bool strict_order = false;  // sweeps fold in the reference's ascending column order
  int concurrency = 1;        // handles sharing the device; > 1: partial grids, dynamic claim order only

  Schedule sched;
  int64_t n = 0, nnz_factors = 0, nnz_source = 0;
  bool has_match = false;
  bool dest16 = true;
  std::vector<int64_t> src_row_offsets, src_col_indices;  // host copy for the pattern guard

  // device: pattern + schedule
  int32_t *d_row_ptr = nullptr, *d_col = nullptr, *d_diag = nullptr;
  int32_t *d_small_rows = nullptr, *d_big_rows = nullptr, *d_lower_order = nullptr,
          *d_upper_order = nullptr, *d_trivial_rows = nullptr;
  int64_t* d_pair_row_ptr = nullptr;
  RowMeta *d_lower_meta = nullptr, *d_upper_meta = nullptr;      // triangular sweeps
  // split sweeps (default mode): device image of the two TailPlans
  struct TailDev {
    int32_t rows = 0, head_claims = 0, head_publish = 0;
    TailRow* row = nullptr;
    TailEntry* entries = nullptr;
    RowMeta* head_meta = nullptr;
    int32_t* head_part_k = nullptr;
  } lower_tail, upper_tail;
  double* d_partial = nullptr;
  FactorMeta *d_small_meta = nullptr, *d_big_meta = nullptr;    // refactorization queues
  ScheduleTuning tune;
  void* d_dest = nullptr;
  int32_t* d_src_of_slot = nullptr;
  double* d_scatter_scale = nullptr;
  int32_t *d_p = nullptr, *d_pq = nullptr;
  double *d_row_scale = nullptr, *d_col_scale = nullptr;
  int32_t *d_a_row_ptr = nullptr, *d_a_col = nullptr;
  // device-resident KKT value path (b200lu_kkt_bind)
  int64_t kkt_n_primal = -1;
  double *d_kkt_hdiag = nullptr, *d_kkt_dy = nullptr;
  int32_t* d_kkt_pos = nullptr;
  bool have_values = false;  // a full set of operator values has been given (reset_values / refactorize)
  // device: values and workspaces
  double *d_a_vals = nullptr, *d_work = nullptr, *d_values = nullptr;
  double *d_w = nullptr, *d_t1 = nullptr, *d_t2 = nullptr;
  double *d_in = nullptr, *d_in2 = nullptr, *d_out = nullptr;  // host<->device staging
  int32_t* d_counters = nullptr;  // [0..2] factor tickets, [4,5] lower/upper tickets, [6,7] rows finished
  int32_t* d_failed = nullptr;    // [0] factor (atomicMin), [1] upper (atomicMax)
  double* d_scal = nullptr;       // scalar results of reductions
  double* d_partials = nullptr;
  unsigned int* d_ticket = nullptr;
  // device: Krylov storage
  double *d_V = nullptr, *d_Z = nullptr, *d_wv = nullptr, *d_r = nullptr, *d_cand = nullptr,
         *d_best = nullptr, *d_x0 = nullptr, *d_b = nullptr;
  double* h_scal = nullptr;  // pinned
  int32_t* h_failed = nullptr;  // pinned

  void (*factor_fn)(FactorArgs) = nullptr;
  int factor_grid = 0, tri_grid = 0;
  size_t factor_smem = 0;
  int big_slot = 0;

  bool scattered = false;  // work[] holds a scattered matrix that has not been factorized
  bool valid = false;
  uint64_t generation = 0;
  int64_t alloc_events = 0, device_bytes = 0;
  uint64_t launches = 0;
  std::string last_error;

  // optional per-phase device timing (CUDA events on the handle's stream around each kernel)
  bool timing = false;
  std::vector<cudaEvent_t> ev_start, ev_stop;
  std::vector<int> ev_phase;
  int ev_used = 0;
};

namespace {

using H = b200lu_handle;

#define CU_TRY(h, expr)                                                                 \
  do {                                                                                  \
    cudaError_t e__ = (expr);                                                           \
    if (e__ != cudaSuccess) {                                                           \
      (h)->last_error = std::string(#expr) + ": " + cudaGetErrorString(e__);            \
      return B200LU_CUDA_ERROR;                                                         \
    }                                                                                   \
  } while (0)

#define ST_TRY(expr)                      \
  do {                                    \
    b200lu_status s__ = (expr);           \
    if (s__ != B200LU_OK) return s__;     \
  } while (0)

template <typename T>
b200lu_status dev_alloc(H* h, T** p, size_t count) {
  *p = nullptr;
  if (count == 0) count = 1;
  CU_TRY(h, cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T)));
  ++h->alloc_events;
  h->device_bytes += static_cast<int64_t>(count * sizeof(T));
  return B200LU_OK;
}

template <typename T>
b200lu_status dev_upload(H* h, T** p, const std::vector<T>& v) {
  ST_TRY(dev_alloc(h, p, v.size()));
  if (!v.empty()) {
    CU_TRY(h, cudaMemcpyAsync(*p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, h->stream));
    CU_TRY(h, cudaStreamSynchronize(h->stream));
  }
  return B200LU_OK;
}

inline int blocks_for(int64_t n, int threads) { return static_cast<int>(std::max<int64_t>(1, (n + threads - 1) / threads)); }

b200lu_status check_launch(H* h, const char* what) {
  ++h->launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    h->last_error = std::string(what) + ": " + cudaGetErrorString(e);
    return B200LU_CUDA_ERROR;
  }
  return B200LU_OK;
}

constexpr int kMaxTimedLaunches = 4096;

struct PhaseScope {
  H* h;
  int idx = -1;
  PhaseScope(H* handle, int phase) : h(handle) {
    if (h->timing && h->ev_used < kMaxTimedLaunches) {
      idx = h->ev_used++;
      h->ev_phase[idx] = phase;
      cudaEventRecord(h->ev_start[idx], h->stream);
    }
  }
  ~PhaseScope() {
    if (idx >= 0) cudaEventRecord(h->ev_stop[idx], h->stream);
  }
};

// ------------------------------------------------------------- device stages

b200lu_status launch_scatter(H* h) {
  if (h->nnz_factors == 0) return B200LU_OK;
  const int blocks = std::min<int64_t>(blocks_for(h->nnz_factors, 256), 148 * 16);
  PhaseScope ps(h, B200LU_PHASE_SCATTER);
  scatter_kernel<<<blocks, 256, 0, h->stream>>>(h->nnz_factors, h->d_src_of_slot, h->d_a_vals,
                                                h->d_scatter_scale, h->d_work, h->d_values);
  return check_launch(h, "scatter_kernel");
}

b200lu_status launch_factor(H* h, int64_t* failed_row) {
  if (failed_row) *failed_row = -1;
  if (h->n == 0) {  // src/numeric.cpp:34-57 on an empty pattern: no row can fail; the factors become valid, the generation advances
    h->scattered = false;
    h->valid = true;
    ++h->generation;
    return B200LU_OK;
  }
  arm_factor_kernel<<<1, 1, 0, h->stream>>>(h->d_counters, h->d_failed);
  ST_TRY(check_launch(h, "arm_factor_kernel"));
  if (!h->sched.trivial_rows.empty()) {
    const int32_t cnt = static_cast<int32_t>(h->sched.trivial_rows.size());
    trivial_pivot_kernel<<<blocks_for(cnt, 256), 256, 0, h->stream>>>(cnt, h->d_trivial_rows, h->d_diag, h->d_work,
                                                                      h->pivot_floor, h->d_failed);
    ST_TRY(check_launch(h, "trivial_pivot_kernel"));
  }
  FactorArgs a;
  a.n_small = static_cast<int32_t>(h->sched.small_rows.size());
  a.n_big = static_cast<int32_t>(h->sched.big_rows.size());
  a.small_slot = static_cast<int32_t>(h->tune.small_slot);
  a.big_slot = h->big_slot;
  a.row_ptr = h->d_row_ptr;
  a.col = h->d_col;
  a.diag = h->d_diag;
  a.small_meta = h->d_small_meta;
  a.big_meta = h->d_big_meta;
  a.pair_row_ptr = h->d_pair_row_ptr;
  a.dest = h->d_dest;
  a.work = h->d_work;
  a.values = h->d_values;
  a.pivot_floor = h->pivot_floor;
  a.counters = h->d_counters;
  a.failed_row = h->d_failed;
  {
    PhaseScope ps(h, B200LU_PHASE_FACTOR);
    h->factor_fn<<<h->factor_grid, kFactorWarps * 32, h->factor_smem, h->stream>>>(a);
  }
  ST_TRY(check_launch(h, "factor_kernel"));
  CU_TRY(h, cudaMemcpyAsync(h->h_failed, h->d_failed, sizeof(int32_t), cudaMemcpyDeviceToHost, h->stream));
  CU_TRY(h, cudaStreamSynchronize(h->stream));
  h->scattered = false;
  if (h->h_failed[0] != INT_MAX) {
    // src/numeric.cpp:51-55: factors stay invalid, the lowest failing row is reported.
    h->valid = false;
    if (failed_row) *failed_row = h->h_failed[0];
    h->last_error = "zero pivot at row " + std::to_string(h->h_failed[0]);
    return B200LU_ZERO_PIVOT;
  }
  h->valid = true;
  ++h->generation;
  return B200LU_OK;
}

TriArgs tri_args(H* h, const RowMeta* meta, const double* y, double* x, int counter_slot) {
  TriArgs a;
  a.n = static_cast<int32_t>(h->n);
  a.n_publish = a.n;
  a.part_k = nullptr;
  a.partial = nullptr;
  a.meta = meta;
  a.col = h->d_col;
  a.diag = h->d_diag;
  a.values = h->d_values;
  a.y = y;
  a.x = x;
  a.counter = h->d_counters + counter_slot;
  a.finished = h->d_counters + counter_slot + 2;
  a.failed_row = h->d_failed + 1;
  return a;
}

TailArgs tail_args(H* h, const H::TailDev& t, const double* init, double* x) {
  TailArgs a;
  a.rows = t.rows;
  a.row = t.row;
  a.entries = t.entries;
  a.values = h->d_values;
  a.init = init;
  a.x = x;
  a.failed_row = h->d_failed + 1;
  return a;
}

constexpr int kTailCluster = 8;  // CTAs per tail cluster (portable maximum)

template <bool kUpper>
b200lu_status launch_tail(H* h, const TailArgs& args) {
  cudaLaunchConfig_t cfg{};
  static const int cluster = [] {
    const char* e = std::getenv("B200LU_TAIL_CLUSTER");
    const int c = e ? std::atoi(e) : kTailCluster;
    return c >= 1 && c <= 8 ? c : kTailCluster;
  }();
  cfg.gridDim = dim3(cluster);
  cfg.blockDim = dim3(kTailThreads);
  cfg.dynamicSmemBytes = static_cast<size_t>(args.rows) * sizeof(double);
  cfg.stream = h->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CU_TRY(h, cudaLaunchKernelEx(&cfg, tail_kernel<kUpper>, args));
  return check_launch(h, kUpper ? "tail_kernel<upper>" : "tail_kernel<lower>");
}

// L sweep. Strict order (or no narrow tail): the whole sweep in the sync-free kernel. Default:
// head rows + the tail rows' prefix sums in the sync-free kernel, then the tail inside one CTA.
b200lu_status launch_lower(H* h, const double* y, double* x) {
  const H::TailDev& t = h->lower_tail;
  if (h->strict_order || t.rows == 0) {
    PhaseScope ps(h, B200LU_PHASE_LOWER);
    TriArgs a = tri_args(h, h->d_lower_meta, y, x, 4);
    tri_kernel<false, false, false><<<h->tri_grid, 256, 0, h->stream>>>(a);
    return check_launch(h, "tri_kernel<lower>");
  }
  const double* init = y;
  if (t.head_publish > 0) {
    PhaseScope ps(h, B200LU_PHASE_LOWER);
    TriArgs a = tri_args(h, t.head_meta, y, x, 4);
    a.n = t.head_claims;
    a.n_publish = t.head_publish;
    a.part_k = t.head_part_k;
    a.partial = h->d_partial;
    if (h->concurrency > 1) {  // static claim order needs the whole grid resident
      tri_kernel<false, false, false><<<h->tri_grid, 256, 0, h->stream>>>(a);
    } else {
      CU_TRY(h, launch_resident(tri_kernel<false, false, true>, h->tri_grid, 256, 0, h->stream, a));
    }
    ST_TRY(check_launch(h, "tri_kernel<lower head>"));
    init = h->d_partial;
  }  // else: no head rows, every prefix is empty and the partial sums are y itself
  PhaseScope ps(h, B200LU_PHASE_TAIL);
  return launch_tail<false>(h, tail_args(h, t, init, x));
}

// U sweep: the narrow part comes FIRST in dependency order (the last rows of the matrix).
b200lu_status launch_upper(H* h, const double* y, double* x) {
  const H::TailDev& t = h->upper_tail;
  if (h->strict_order || t.rows == 0) {
    PhaseScope ps(h, B200LU_PHASE_UPPER);
    TriArgs a = tri_args(h, h->d_upper_meta, y, x, 5);
    if (h->strict_order) {
      tri_kernel<true, false, false><<<h->tri_grid, 256, 0, h->stream>>>(a);
    } else {
      tri_kernel<true, true, false><<<h->tri_grid, 256, 0, h->stream>>>(a);
    }
    return check_launch(h, "tri_kernel<upper>");
  }
  {
    PhaseScope ps(h, B200LU_PHASE_TAIL);
    ST_TRY(launch_tail<true>(h, tail_args(h, t, y, x)));
  }
  if (t.head_claims > 0) {
    PhaseScope ps(h, B200LU_PHASE_UPPER);
    TriArgs a = tri_args(h, t.head_meta, y, x, 5);
    a.n = t.head_claims;
    a.n_publish = t.head_claims;
    if (h->concurrency > 1) {
      tri_kernel<true, true, false><<<h->tri_grid, 256, 0, h->stream>>>(a);
    } else {
      CU_TRY(h, launch_resident(tri_kernel<true, true, true>, h->tri_grid, 256, 0, h->stream, a));
    }
    ST_TRY(check_launch(h, "tri_kernel<upper head>"));
  }
  return B200LU_OK;
}

// Device-to-device solve_system (src/trisolve.cpp:90-119). Does not synchronise; an exactly
// zero U diagonal is left in d_failed[1] for the caller to collect.
b200lu_status solve_device(H* h, const double* b, double* x) {
  if (h->n == 0) return B200LU_OK;
  const int nb = blocks_for(h->n, 256);
  {
    PhaseScope ps(h, B200LU_PHASE_PERMUTE);
    arm_solve_kernel<<<1, 1, 0, h->stream>>>(h->d_counters, h->d_failed + 1);
    ST_TRY(check_launch(h, "arm_solve_kernel"));
    permute_in_kernel<<<nb, 256, 0, h->stream>>>(static_cast<int32_t>(h->n), h->d_p, h->d_row_scale, b,
                                                 h->d_w, h->d_t1, h->d_t2);
    ST_TRY(check_launch(h, "permute_in_kernel"));
  }
  ST_TRY(launch_lower(h, h->d_w, h->d_t1));
  ST_TRY(launch_upper(h, h->d_t1, h->d_t2));
  PhaseScope ps(h, B200LU_PHASE_PERMUTE);
  permute_out_kernel<<<nb, 256, 0, h->stream>>>(static_cast<int32_t>(h->n), h->d_pq, h->d_col_scale,
                                                h->d_t2, x);
  return check_launch(h, "permute_out_kernel");
}

b200lu_status collect_upper_failure(H* h, int64_t* failed_row) {
  if (failed_row) *failed_row = -1;
  if (h->n == 0) return B200LU_OK;
  CU_TRY(h, cudaMemcpyAsync(h->h_failed + 1, h->d_failed + 1, sizeof(int32_t), cudaMemcpyDeviceToHost, h->stream));
  CU_TRY(h, cudaStreamSynchronize(h->stream));
  if (h->h_failed[1] >= 0) {
    if (failed_row) *failed_row = h->h_failed[1];
    h->last_error = "zero diagonal at row " + std::to_string(h->h_failed[1]);
    return B200LU_ZERO_PIVOT;
  }
  return B200LU_OK;
}

b200lu_status check_solve_ready(H* h, int64_t len, const char* who) {
  // check_dims, src/trisolve.cpp:19-25
  if (!h->valid) {
    h->last_error = std::string(who) + ": factors are not valid";
    return B200LU_INVALID_FACTORS;
  }
  if (len != h->n) {
    h->last_error = std::string(who) + ": vector length " + std::to_string(len) + ", expected " + std::to_string(h->n);
    return B200LU_DIMENSION;
  }
  return B200LU_OK;
}

const double* stage_in(H* h, const double* p, double* staging, int on_device, cudaError_t* err) {
  if (on_device || h->n == 0) return p;
  *err = cudaMemcpyAsync(staging, p, static_cast<size_t>(h->n) * sizeof(double), cudaMemcpyHostToDevice, h->stream);
  return staging;
}

b200lu_status stage_out(H* h, const double* dev, double* host, int on_device) {
  if (on_device || h->n == 0) return B200LU_OK;
  CU_TRY(h, cudaMemcpyAsync(host, dev, static_cast<size_t>(h->n) * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CU_TRY(h, cudaStreamSynchronize(h->stream));
  return B200LU_OK;
}

// --------------------------------------------------------------- reductions

b200lu_status read_scalars(H* h, int first, int count) {
  CU_TRY(h, cudaMemcpyAsync(h->h_scal + first, h->d_scal + first, static_cast<size_t>(count) * sizeof(double),
                            cudaMemcpyDeviceToHost, h->stream));
  CU_TRY(h, cudaStreamSynchronize(h->stream));
  return B200LU_OK;
}

// r = b - A x; d_scal[slot] = sum r^2, d_scal[slot+1] = sum b^2
b200lu_status launch_residual(H* h, const double* x, const double* b, double* r, int slot) {
  PhaseScope ps(h, B200LU_PHASE_SPMV);
  residual_kernel<<<kReduceBlocks, kReduceThreads, 0, h->stream>>>(
      static_cast<int32_t>(h->n), h->d_a_row_ptr, h->d_a_col, h->d_a_vals, x, b, r, h->d_partials,
      h->d_ticket, h->d_scal + slot);
  return check_launch(h, "residual_kernel");
}

b200lu_status launch_dot(H* h, const double* a, const double* b, int slot) {
  PhaseScope ps(h, B200LU_PHASE_VECTOR);
  dot_kernel<<<kReduceBlocks, kReduceThreads, 0, h->stream>>>(static_cast<int32_t>(h->n), a, b, h->d_partials,
                                                             h->d_ticket, h->d_scal + slot);
  return check_launch(h, "dot_kernel");
}

b200lu_status launch_spmv(H* h, const double* x, double* y) {
  if (h->n == 0) return B200LU_OK;
  PhaseScope ps(h, B200LU_PHASE_SPMV);
  spmv_kernel<<<blocks_for(h->n, 256), 256, 0, h->stream>>>(static_cast<int32_t>(h->n), h->d_a_row_ptr, h->d_a_col,
                                                             h->d_a_vals, x, y);
  return check_launch(h, "spmv_kernel");
}

b200lu_status apply_precond(H* h, int use_precond, const double* in, double* out) {
  if (use_precond) return solve_device(h, in, out);
  CU_TRY(h, cudaMemcpyAsync(out, in, static_cast<size_t>(h->n) * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
  return B200LU_OK;
}

b200lu_status copy_dd(H* h, double* dst, const double* src) {
  if (dst == src || h->n == 0) return B200LU_OK;
  CU_TRY(h, cudaMemcpyAsync(dst, src, static_cast<size_t>(h->n) * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
  return B200LU_OK;
}

// scalar slots in d_scal / h_scal
enum { kSlotRes = 0, kSlotBn = 1, kSlotNorm = 2, kSlotH = 3, kSlotCoef = 8 /* .. kSlotCoef+cap */ };

// fgmres_refine, src/refine.cpp:39-142. b, x0 are device vectors; the best iterate is left in
// h->d_best.
b200lu_status fgmres_device(H* h, const double* b, const double* x0, int use_precond,
                            const b200lu_refine_config& cfg, b200lu_refine_outcome* out) {
  const int64_t n = h->n;
  const int32_t n32 = static_cast<int32_t>(n);
  const int nb = blocks_for(n, 256);
  const int m = std::max(1, cfg.max_iterations);
  out->iterations = 0;
  out->converged = 0;
  out->history_len = 0;
  ST_TRY(copy_dd(h, h->d_best, x0));
  if (n == 0) {
    out->residual_history[out->history_len++] = 0.0;
    out->converged = 1;
    return B200LU_OK;
  }

  ST_TRY(launch_residual(h, x0, b, h->d_r, kSlotRes));
  ST_TRY(read_scalars(h, kSlotRes, 2));
  const double bn = std::sqrt(h->h_scal[kSlotBn]);
  const double bnorm = bn > 0.0 ? bn : 1.0;
  const double beta = std::sqrt(h->h_scal[kSlotRes]);
  double best_res = beta / bnorm;
  out->residual_history[out->history_len++] = best_res;
  if (best_res <= cfg.tolerance) {
    out->converged = 1;
    return B200LU_OK;
  }

  auto V = [&](int j) { return h->d_V + static_cast<size_t>(j) * n; };
  auto Z = [&](int j) { return h->d_Z + static_cast<size_t>(j) * n; };
  int nV = 0;
  {
    PhaseScope ps(h, B200LU_PHASE_VECTOR);
    divide_kernel<<<nb, 256, 0, h->stream>>>(n32, beta, h->d_r, V(0));
  }
  ST_TRY(check_launch(h, "divide_kernel"));
  nV = 1;

  std::vector<std::vector<double>> Hm;  // column-major Hessenberg after rotations
  std::vector<double> g(static_cast<size_t>(m) + 1, 0.0), cs(m, 0.0), sn(m, 0.0);
  g[0] = beta;
  double accept_below = cfg.tolerance * bnorm;

  for (int i = 0; i < m; ++i) {
    ST_TRY(apply_precond(h, use_precond, V(i), Z(i)));
    ST_TRY(launch_spmv(h, Z(i), h->d_wv));

    // cgs2_orthonormalize(V, w), src/refine.cpp:8-26
    CU_TRY(h, cudaMemsetAsync(h->d_scal + kSlotCoef, 0, static_cast<size_t>(nV) * sizeof(double), h->stream));
    for (int pass = 0; pass < 2; ++pass) {
      for (int j = 0; j < nV; ++j) {
        ST_TRY(launch_dot(h, V(j), h->d_wv, kSlotH));
        {
          PhaseScope ps(h, B200LU_PHASE_VECTOR);
          project_out_kernel<<<nb, 256, 0, h->stream>>>(n32, h->d_scal + kSlotH, h->d_scal + kSlotCoef + j, V(j), h->d_wv);
        }
        ST_TRY(check_launch(h, "project_out_kernel"));
      }
    }
    ST_TRY(launch_dot(h, h->d_wv, h->d_wv, kSlotNorm));
    ST_TRY(read_scalars(h, kSlotNorm, kSlotCoef + nV - kSlotNorm));
    const double norm = std::sqrt(h->h_scal[kSlotNorm]);
    const bool breakdown = norm <= 1e-300;
    std::vector<double> hcol(h->h_scal + kSlotCoef, h->h_scal + kSlotCoef + nV);
    hcol.push_back(breakdown ? 0.0 : norm);
    if (!breakdown) {
      {
        PhaseScope ps(h, B200LU_PHASE_VECTOR);
        divide_kernel<<<nb, 256, 0, h->stream>>>(n32, norm, h->d_wv, V(nV));
      }
      ST_TRY(check_launch(h, "divide_kernel"));
      ++nV;
    }

    // Givens update, src/refine.cpp:89-107 (host scalars)
    for (int k = 0; k < i; ++k) {
      const double t = hcol[k];
      hcol[k] = cs[k] * t + sn[k] * hcol[k + 1];
      hcol[k + 1] = -sn[k] * t + cs[k] * hcol[k + 1];
    }
    const double hii = hcol[i], hsub = hcol[i + 1];
    const double gam = std::hypot(hii, hsub);
    if (gam == 0.0) {
      cs[i] = 1.0;
      sn[i] = 0.0;
    } else {
      cs[i] = hii / gam;
      sn[i] = hsub / gam;
    }
    hcol[i] = gam;
    hcol[i + 1] = 0.0;
    const double gi = g[i];
    g[i] = cs[i] * gi;
    g[i + 1] = -sn[i] * gi;
    Hm.push_back(std::move(hcol));

    out->iterations = i + 1;
    const double estimate = std::fabs(g[i + 1]);
    out->residual_history[out->history_len++] = estimate / bnorm;

    const bool last = breakdown || i == m - 1;
    if (estimate <= accept_below || last) {
      // src/refine.cpp:115-139: minimum-residual iterate, true residual, best-iterate rule.
      const int its = out->iterations;
      std::vector<double> y(its);
      for (int row = its - 1; row >= 0; --row) {
        double t = g[row];
        for (int col = row + 1; col < its; ++col) t -= Hm[col][row] * y[col];
        y[row] = t / Hm[row][row];
      }
      ST_TRY(copy_dd(h, h->d_cand, x0));
      for (int col = 0; col < its; ++col) {
        {
          PhaseScope ps(h, B200LU_PHASE_VECTOR);
          axpy_kernel<<<nb, 256, 0, h->stream>>>(n32, y[col], Z(col), h->d_cand);
        }
        ST_TRY(check_launch(h, "axpy_kernel"));
      }
      ST_TRY(launch_residual(h, h->d_cand, b, h->d_r, kSlotRes));
      ST_TRY(read_scalars(h, kSlotRes, 1));
      const double res = std::sqrt(h->h_scal[kSlotRes]) / bnorm;
      if (res < best_res) {
        best_res = res;
        ST_TRY(copy_dd(h, h->d_best, h->d_cand));
      }
      if (best_res <= cfg.tolerance) {
        out->converged = 1;
        return B200LU_OK;
      }
      if (last) return B200LU_OK;
      accept_below = estimate * 0.5;
    }
  }
  return B200LU_OK;
}

// classic_refine, src/refine.cpp:150-188.
b200lu_status classic_device(H* h, const double* b, const double* x0, int use_precond,
                             const b200lu_refine_config& cfg, b200lu_refine_outcome* out) {
  const int64_t n = h->n;
  const int32_t n32 = static_cast<int32_t>(n);
  const int nb = blocks_for(n, 256);
  out->iterations = 0;
  out->converged = 0;
  out->history_len = 0;
  ST_TRY(copy_dd(h, h->d_best, x0));
  if (n == 0) {
    out->residual_history[out->history_len++] = 0.0;
    out->converged = 1;
    return B200LU_OK;
  }
  ST_TRY(launch_residual(h, x0, b, h->d_r, kSlotRes));
  ST_TRY(read_scalars(h, kSlotRes, 2));
  const double bn = std::sqrt(h->h_scal[kSlotBn]);
  const double bnorm = bn > 0.0 ? bn : 1.0;
  double best_res = std::sqrt(h->h_scal[kSlotRes]) / bnorm;
  out->residual_history[out->history_len++] = best_res;
  if (best_res <= cfg.tolerance) {
    out->converged = 1;
    return B200LU_OK;
  }
  double* x = h->d_cand;
  ST_TRY(copy_dd(h, x, x0));
  for (int it = 0; it < cfg.max_iterations; ++it) {
    // d_r already holds b - A x for the current x: from the initial residual on the first
    // pass, from the end of the previous pass afterwards (the reference recomputes the same
    // vector, src/refine.cpp:168-169).
    ST_TRY(apply_precond(h, use_precond, h->d_r, h->d_wv));
    {
      PhaseScope ps(h, B200LU_PHASE_VECTOR);
      axpy_kernel<<<nb, 256, 0, h->stream>>>(n32, 1.0, h->d_wv, x);
    }
    ST_TRY(check_launch(h, "axpy_kernel"));
    out->iterations = it + 1;
    ST_TRY(launch_residual(h, x, b, h->d_r, kSlotRes));
    ST_TRY(read_scalars(h, kSlotRes, 1));
    const double res = std::sqrt(h->h_scal[kSlotRes]) / bnorm;
    out->residual_history[out->history_len++] = res;
    if (res < best_res) {
      best_res = res;
      ST_TRY(copy_dd(h, h->d_best, x));
    }
    if (best_res <= cfg.tolerance) {
      out->converged = 1;
      return B200LU_OK;
    }
  }
  return B200LU_OK;
}

b200lu_status refine_common(H* h, const double* b, const double* x0, double* x_out, int on_device,
                            int use_precond, const b200lu_refine_config* cfg_in,
                            b200lu_refine_outcome* out, bool fgmres) {
  if (!h || !out || (!b && h->n) || (!x0 && h->n) || (!x_out && h->n)) return B200LU_INVALID_ARGUMENT;
  CU_TRY(h, cudaSetDevice(h->device));
  b200lu_refine_config cfg{20, 1e-14};
  if (cfg_in) cfg = *cfg_in;
  if (cfg.max_iterations > h->refine_capacity) {
    h->last_error = "max_iterations exceeds the handle's refine_capacity";
    return B200LU_INVALID_ARGUMENT;
  }
  if (use_precond && !h->valid) {
    h->last_error = "solve_system: factors are not valid";
    return B200LU_INVALID_FACTORS;
  }
  cudaError_t e = cudaSuccess;
  const double* db = stage_in(h, b, h->d_b, on_device, &e);
  CU_TRY(h, e);
  const double* dx0 = stage_in(h, x0, h->d_x0, on_device, &e);
  CU_TRY(h, e);
  ST_TRY(fgmres ? fgmres_device(h, db, dx0, use_precond, cfg, out)
                : classic_device(h, db, dx0, use_precond, cfg, out));
  if (on_device) {
    ST_TRY(copy_dd(h, x_out, h->d_best));
    CU_TRY(h, cudaStreamSynchronize(h->stream));
  } else {
    ST_TRY(stage_out(h, h->d_best, x_out, 0));
  }
  return B200LU_OK;
}

}  // namespace

// ===================================================================== C ABI

extern "C" {

void b200lu_default_options(b200lu_options* opt) {
  if (!opt) return;
  opt->pivot_floor = 1e-30;  // include/rlu/numeric.hpp:14
  opt->device = 0;
  opt->stream = nullptr;
  opt->refine_capacity = 20;  // include/rlu/refine.hpp:14
  opt->flags = 0;
  opt->concurrency = 1;
}

const char* b200lu_status_string(b200lu_status s) {
  switch (s) {
    case B200LU_OK: return "ok";
    case B200LU_ZERO_PIVOT: return "zero pivot";
    case B200LU_PATTERN_MISMATCH: return "matrix pattern differs from the analyzed pattern";
    case B200LU_DIMENSION: return "dimension mismatch";
    case B200LU_INVALID_FACTORS: return "factors are not valid";
    case B200LU_CUDA_ERROR: return "CUDA error";
    case B200LU_INVALID_ARGUMENT: return "invalid argument";
    case B200LU_NO_DEVICE: return "no CUDA device";
    case B200LU_ZERO_DIAGONAL: return "structurally zero diagonal";
    case B200LU_STRUCTURALLY_SINGULAR: return "structurally singular";
  }
  return "unknown";
}

const char* b200lu_last_error(const b200lu_handle* h) { return h ? h->last_error.c_str() : ""; }

int b200lu_device_count(void) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return c;
}

b200lu_status b200lu_create(const b200lu_symbolic_view* sym, const b200lu_options* opt_in,
                            b200lu_handle** out) {
  if (!sym || !out) return B200LU_INVALID_ARGUMENT;
  *out = nullptr;
  b200lu_options opt;
  b200lu_default_options(&opt);
  if (opt_in) opt = *opt_in;
  if (b200lu_device_count() <= opt.device) return B200LU_NO_DEVICE;

  H* h = new H;
  *out = h;  // returned even on failure so the caller can read last_error, then destroy
  h->device = opt.device;
  h->pivot_floor = opt.pivot_floor;
  h->refine_capacity = opt.refine_capacity > 0 ? std::min(opt.refine_capacity, 64) : 20;
  h->strict_order = (opt.flags & B200LU_FLAG_STRICT_ORDER) != 0;
  h->concurrency = std::max(1, opt.concurrency);
  CU_TRY(h, cudaSetDevice(h->device));
  if (opt.stream) {
    h->stream = static_cast<cudaStream_t>(opt.stream);
  } else {
    CU_TRY(h, cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    h->owns_stream = true;
  }

  // Sweep throttle (see schedule.hpp, fill_start_thresholds). Tunable for experiments; the
  // defaults are what DESIGN.md reports.
  if (const char* e = std::getenv("B200LU_SOLVE_LOOKAHEAD_LEVELS")) h->tune.solve_lookahead_levels = std::atoll(e);
  if (const char* e = std::getenv("B200LU_SOLVE_MIN_WINDOW")) h->tune.solve_min_window = std::atoll(e);
  if (const char* e = std::getenv("B200LU_SOLVE_MAX_WINDOW")) h->tune.solve_max_window = std::atoll(e);
  if (const char* e = std::getenv("B200LU_TAIL_WIDTH")) h->tune.tail_width = std::atoll(e);
  if (const char* e = std::getenv("B200LU_TAIL_CAPACITY")) h->tune.tail_capacity = std::min<int64_t>(std::atoll(e), kMaxTailRows);
  const std::string err = build_schedule(*sym, h->tune, h->sched);
  if (!err.empty()) {
    h->last_error = err;
    return B200LU_INVALID_ARGUMENT;
  }
  const Schedule& S = h->sched;
  const int64_t n = h->n = sym->n;
  const int64_t nnzF = h->nnz_factors = sym->nnz_factors;
  const int64_t nnzA = h->nnz_source = sym->nnz_source;
  h->has_match = sym->col_perm_forward != nullptr;
  if (nnzA >= (int64_t{1} << 31) - 64) {
    h->last_error = "nnz(A) exceeds the int32 device index range";
    return B200LU_INVALID_ARGUMENT;
  }
  h->src_row_offsets.assign(sym->source_row_offsets, sym->source_row_offsets + n + 1);
  h->src_col_indices.assign(sym->source_col_indices, sym->source_col_indices + nnzA);

  // pattern + schedule
  ST_TRY(dev_upload(h, &h->d_row_ptr, S.row_ptr));
  ST_TRY(dev_upload(h, &h->d_col, S.col));
  ST_TRY(dev_upload(h, &h->d_diag, S.diag));
  ST_TRY(dev_upload(h, &h->d_small_rows, S.small_rows));
  ST_TRY(dev_upload(h, &h->d_big_rows, S.big_rows));
  ST_TRY(dev_upload(h, &h->d_trivial_rows, S.trivial_rows));
  ST_TRY(dev_upload(h, &h->d_lower_order, S.lower_order));
  ST_TRY(dev_upload(h, &h->d_upper_order, S.upper_order));
  ST_TRY(dev_upload(h, &h->d_pair_row_ptr, S.pair_row_ptr));
  ST_TRY(dev_upload(h, &h->d_lower_meta, S.lower_meta));
  ST_TRY(dev_upload(h, &h->d_upper_meta, S.upper_meta));
  {
    auto upload_tail = [&](const TailPlan& p, H::TailDev& d) -> b200lu_status {
      d.rows = static_cast<int32_t>(p.rows);
      if (p.rows == 0) return B200LU_OK;
      d.head_claims = static_cast<int32_t>(p.head_meta.size());
      d.head_publish = static_cast<int32_t>(p.head_publish);
      ST_TRY(dev_upload(h, &d.row, p.row));
      ST_TRY(dev_upload(h, &d.entries, p.entries));
      ST_TRY(dev_upload(h, &d.head_meta, p.head_meta));
      ST_TRY(dev_upload(h, &d.head_part_k, p.head_part_k));
      return B200LU_OK;
    };
    ST_TRY(upload_tail(S.lower_tail, h->lower_tail));
    ST_TRY(upload_tail(S.upper_tail, h->upper_tail));
    ST_TRY(dev_alloc(h, &h->d_partial, n));
    // The attribute is per FUNCTION and process-wide, not per handle: it is set to the fixed upper
    // bound (tail_capacity rows) so that a second handle with a smaller tail never lowers the limit
    // under a live one.
    if (S.lower_tail.rows > 0 || S.upper_tail.rows > 0) {
      const int tail_smem = static_cast<int>(kMaxTailRows * sizeof(double));
      CU_TRY(h, cudaFuncSetAttribute(tail_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, tail_smem));
      CU_TRY(h, cudaFuncSetAttribute(tail_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, tail_smem));
    }
  }
  {
    auto factor_meta = [&S](const std::vector<int32_t>& rows) {
      std::vector<FactorMeta> m(rows.size());
      for (size_t r = 0; r < rows.size(); ++r) {
        const int32_t i = rows[r];
        m[r] = FactorMeta{i, S.row_ptr[i], S.diag[i], S.row_ptr[i + 1]};
      }
      return m;
    };
    ST_TRY(dev_upload(h, &h->d_small_meta, factor_meta(S.small_rows)));
    ST_TRY(dev_upload(h, &h->d_big_meta, factor_meta(S.big_rows)));
  }

  // scatter: inverse map (slot -> source entry), scale only on the matching path
  {
    if (nnzA >= kTrivialBit) {
      h->last_error = "nnz(A) exceeds the 2^30 entries the scatter map encoding supports";
      return B200LU_INVALID_ARGUMENT;
    }
    std::vector<int32_t> src_of_slot(nnzF, -1);
    for (int64_t k = 0; k < nnzA; ++k) {
      const int64_t s = sym->scatter_map[k];
      if (s < 0 || s >= nnzF || src_of_slot[s] != -1) {
        h->last_error = "scatter_map is not an injection into the combined pattern";
        return B200LU_INVALID_ARGUMENT;
      }
      src_of_slot[s] = static_cast<int32_t>(k);
    }
    for (int32_t i : S.trivial_rows) {  // slots the scatter pass publishes directly (factor.cuh, K1)
      for (int32_t s = S.row_ptr[i]; s < S.row_ptr[i + 1]; ++s) {
        src_of_slot[s] = src_of_slot[s] >= 0 ? (src_of_slot[s] | kTrivialBit) : kTrivialFill;
      }
    }
    ST_TRY(dev_upload(h, &h->d_src_of_slot, src_of_slot));
    if (h->has_match) {
      // Off the matching path every scale is exactly 1.0 (src/symbolic.cpp:187) and the
      // multiply is skipped: v * 1.0 == v bit for bit.
      std::vector<double> sc(sym->scatter_scale, sym->scatter_scale + nnzA);
      ST_TRY(dev_upload(h, &h->d_scatter_scale, sc));
    } else {
      for (int64_t k = 0; k < nnzA; ++k) {
        if (sym->scatter_scale[k] != 1.0) {
          std::vector<double> sc(sym->scatter_scale, sym->scatter_scale + nnzA);
          ST_TRY(dev_upload(h, &h->d_scatter_scale, sc));
          break;
        }
      }
    }
  }
  // permutations / scalings of solve_system
  {
    std::vector<int32_t> p(n), pq(n);
    for (int64_t i = 0; i < n; ++i) p[i] = static_cast<int32_t>(sym->amd_forward[i]);
    for (int64_t j = 0; j < n; ++j) {
      pq[j] = h->has_match ? p[sym->col_perm_forward[j]] : p[j];
    }
    ST_TRY(dev_upload(h, &h->d_p, p));
    ST_TRY(dev_upload(h, &h->d_pq, pq));
    if (h->has_match) {
      ST_TRY(dev_upload(h, &h->d_row_scale, std::vector<double>(sym->row_scale, sym->row_scale + n)));
      ST_TRY(dev_upload(h, &h->d_col_scale, std::vector<double>(sym->col_scale, sym->col_scale + n)));
    }
  }
  // operator A (pattern now, values at reset_values)
  {
    std::vector<int32_t> arp(n + 1), ac(nnzA);
    for (int64_t i = 0; i <= n; ++i) arp[i] = static_cast<int32_t>(sym->source_row_offsets[i]);
    for (int64_t k = 0; k < nnzA; ++k) ac[k] = static_cast<int32_t>(sym->source_col_indices[k]);
    ST_TRY(dev_upload(h, &h->d_a_row_ptr, arp));
    ST_TRY(dev_upload(h, &h->d_a_col, ac));
  }
  ST_TRY(dev_alloc(h, &h->d_a_vals, nnzA));
  ST_TRY(dev_alloc(h, &h->d_work, nnzF));
  ST_TRY(dev_alloc(h, &h->d_values, nnzF));
  for (double** p : {&h->d_w, &h->d_t1, &h->d_t2, &h->d_in, &h->d_in2, &h->d_out, &h->d_wv, &h->d_r,
                     &h->d_cand, &h->d_best, &h->d_x0, &h->d_b}) {
    ST_TRY(dev_alloc(h, p, n));
  }
  ST_TRY(dev_alloc(h, &h->d_V, static_cast<size_t>(h->refine_capacity + 1) * std::max<int64_t>(n, 1)));
  ST_TRY(dev_alloc(h, &h->d_Z, static_cast<size_t>(h->refine_capacity) * std::max<int64_t>(n, 1)));
  ST_TRY(dev_alloc(h, &h->d_counters, 8));
  ST_TRY(dev_alloc(h, &h->d_failed, 2));
  ST_TRY(dev_alloc(h, &h->d_scal, 128));
  ST_TRY(dev_alloc(h, &h->d_partials, 2 * kReduceBlocks));
  ST_TRY(dev_alloc(h, &h->d_ticket, 1));
  CU_TRY(h, cudaMemsetAsync(h->d_ticket, 0, sizeof(unsigned int), h->stream));
  CU_TRY(h, cudaMemsetAsync(h->d_counters, 0, 8 * sizeof(int32_t), h->stream));
  CU_TRY(h, cudaMallocHost(reinterpret_cast<void**>(&h->h_scal), 128 * sizeof(double)));
  CU_TRY(h, cudaMallocHost(reinterpret_cast<void**>(&h->h_failed), 2 * sizeof(int32_t)));

  // destination table, resolved on the device once
  // 16-bit destination offsets unless a row has more than 65 535 entries; B200LU_DEST32=1 forces the 32-bit kernels (test knob)
  h->dest16 = S.max_row_len <= 65535 && !(std::getenv("B200LU_DEST32") && std::atoi(std::getenv("B200LU_DEST32")) == 1);
  ST_TRY(dev_alloc(h, reinterpret_cast<char**>(&h->d_dest),
                   static_cast<size_t>(S.update_pairs) * (h->dest16 ? 2 : 4) + 16));
  if (n > 0 && S.update_pairs > 0) {
    const int blocks = std::min<int64_t>(blocks_for(n * 32, 256), 148 * 32);
    if (h->dest16) {
      build_dest_kernel<uint16_t><<<blocks, 256, 0, h->stream>>>(static_cast<int32_t>(n), h->d_row_ptr, h->d_col, h->d_diag,
                                                                 h->d_pair_row_ptr, static_cast<uint16_t*>(h->d_dest));
    } else {
      build_dest_kernel<uint32_t><<<blocks, 256, 0, h->stream>>>(static_cast<int32_t>(n), h->d_row_ptr, h->d_col, h->d_diag,
                                                                 h->d_pair_row_ptr, static_cast<uint32_t*>(h->d_dest));
    }
    ST_TRY(check_launch(h, "build_dest_kernel"));
  }

  // launch geometry: persistent grids sized to what is co-resident (the waiting scheme needs
  // every claimed row's owner to be running)
  cudaDeviceProp prop;
  CU_TRY(h, cudaGetDeviceProperties(&prop, h->device));
  int64_t max_big = 0;
  for (int32_t i : S.big_rows) max_big = std::max<int64_t>(max_big, S.row_ptr[i + 1] - S.row_ptr[i]);
  h->big_slot = static_cast<int>(std::min<int64_t>((max_big + 63) / 64 * 64, kMaxBigSlot));
  h->factor_smem = (static_cast<size_t>(kFactorWarps) * h->tune.small_slot + h->big_slot) * sizeof(double);
  // Kernel variant: pivots in flight per warp x resident CTAs per SM (register budget). The
  // default is what DESIGN.md reports; B200LU_FACTOR_VARIANT selects others for experiments.
  {
    const char* e = std::getenv("B200LU_FACTOR_VARIANT");
    const int variant = e ? std::atoi(e) : 0;
    using Fn = void (*)(FactorArgs);
    Fn f16[] = {factor_kernel<uint16_t, kFactorWarps, 4, 2>, factor_kernel<uint16_t, kFactorWarps, 4, 3>,
                factor_kernel<uint16_t, kFactorWarps, 2, 4>, factor_kernel<uint16_t, kFactorWarps, 3, 3>,
                factor_kernel<uint16_t, kFactorWarps, 6, 2>, factor_kernel<uint16_t, kFactorWarps, 2, 3>};
    Fn f32[] = {factor_kernel<uint32_t, kFactorWarps, 4, 2>, factor_kernel<uint32_t, kFactorWarps, 4, 3>,
                factor_kernel<uint32_t, kFactorWarps, 2, 4>, factor_kernel<uint32_t, kFactorWarps, 3, 3>,
                factor_kernel<uint32_t, kFactorWarps, 6, 2>, factor_kernel<uint32_t, kFactorWarps, 2, 3>};
    const int v = variant >= 0 && variant < 6 ? variant : 0;
    h->factor_fn = h->dest16 ? f16[v] : f32[v];
  }
  int occ = 0;
  // per function, process-wide: always the fixed upper bound (see the tail kernels above)
  CU_TRY(h, cudaFuncSetAttribute(h->factor_fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>((static_cast<size_t>(kFactorWarps) * h->tune.small_slot + kMaxBigSlot) * sizeof(double))));
  CU_TRY(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, h->factor_fn, kFactorWarps * 32, h->factor_smem));
  if (occ < 1) {
    h->last_error = "factor kernel does not fit on an SM";
    return B200LU_CUDA_ERROR;
  }
  // With several handles sharing the device each takes its share of the resident CTAs.
  h->factor_grid = std::max(prop.multiProcessorCount / 2, prop.multiProcessorCount * occ / h->concurrency);
  int occ_tri = 0;
  CU_TRY(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_tri, tri_kernel<false, false, false>, 256, 0));
  int occ_tri_u = 0;
  CU_TRY(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_tri_u, tri_kernel<true, false, false>, 256, 0));
  for (int v = 0; v < 3; ++v) {
    int o = 0;
    if (v == 0) CU_TRY(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, tri_kernel<true, true, false>, 256, 0));
    if (v == 1) CU_TRY(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, tri_kernel<true, true, true>, 256, 0));
    if (v == 2) CU_TRY(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, tri_kernel<false, false, true>, 256, 0));
    occ_tri_u = std::min(occ_tri_u, o);
  }
  h->tri_grid = std::max(prop.multiProcessorCount / 2,
                         prop.multiProcessorCount * std::max(1, std::min(occ_tri, occ_tri_u)) / h->concurrency);
  CU_TRY(h, cudaStreamSynchronize(h->stream));
  h->last_error.clear();
  return B200LU_OK;
}

void b200lu_destroy(b200lu_handle* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  void* ptrs[] = {h->d_row_ptr, h->d_col, h->d_diag, h->d_small_rows, h->d_big_rows, h->d_trivial_rows, h->d_lower_order,
                  h->d_upper_order, h->d_pair_row_ptr, h->d_lower_meta, h->d_upper_meta, h->d_small_meta,
                  h->d_big_meta, h->lower_tail.row, h->lower_tail.entries, h->lower_tail.head_meta,
                  h->lower_tail.head_part_k, h->upper_tail.row, h->upper_tail.entries, h->upper_tail.head_meta,
                  h->upper_tail.head_part_k, h->d_partial, h->d_dest, h->d_src_of_slot, h->d_scatter_scale, h->d_p,
                  h->d_pq, h->d_row_scale, h->d_col_scale, h->d_a_row_ptr, h->d_a_col, h->d_kkt_hdiag, h->d_kkt_dy, h->d_kkt_pos, h->d_a_vals, h->d_work,
                  h->d_values, h->d_w, h->d_t1, h->d_t2, h->d_in, h->d_in2, h->d_out, h->d_counters, h->d_failed,
                  h->d_scal, h->d_partials, h->d_ticket, h->d_V, h->d_Z, h->d_wv, h->d_r, h->d_cand, h->d_best,
                  h->d_x0, h->d_b};
  for (void* p : ptrs) {
    if (p) cudaFree(p);
  }
  for (cudaEvent_t e : h->ev_start) cudaEventDestroy(e);
  for (cudaEvent_t e : h->ev_stop) cudaEventDestroy(e);
  if (h->h_scal) cudaFreeHost(h->h_scal);
  if (h->h_failed) cudaFreeHost(h->h_failed);
  if (h->owns_stream && h->stream) cudaStreamDestroy(h->stream);
  cudaGetLastError();
  delete h;
}

b200lu_status b200lu_check_pattern(const b200lu_handle* h, int64_t n, const int64_t* row_offsets,
                                   const int64_t* col_indices) {
  if (!h || !row_offsets || (!col_indices && h->nnz_source)) return B200LU_INVALID_ARGUMENT;
  // pattern_equal: dimensions, row offsets and column indices identical
  if (n != h->n) return B200LU_PATTERN_MISMATCH;
  if (!same_bytes(row_offsets, h->src_row_offsets.data(), sizeof(int64_t) * (n + 1))) return B200LU_PATTERN_MISMATCH;
  if (h->nnz_source && !same_bytes(col_indices, h->src_col_indices.data(), sizeof(int64_t) * h->nnz_source)) {
    return B200LU_PATTERN_MISMATCH;
  }
  return B200LU_OK;
}

b200lu_status b200lu_reset_values(b200lu_handle* h, const double* a_values, int on_device) {
  if (!h || (!a_values && h->nnz_source)) return B200LU_INVALID_ARGUMENT;
  CU_TRY(h, cudaSetDevice(h->device));
  if (h->nnz_source) {
    CU_TRY(h, cudaMemcpyAsync(h->d_a_vals, a_values, static_cast<size_t>(h->nnz_source) * sizeof(double),
                              on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, h->stream));
  }
  h->valid = false;
  h->have_values = true;
  ST_TRY(launch_scatter(h));
  h->scattered = true;
  return B200LU_OK;
}

b200lu_status b200lu_kkt_bind(b200lu_handle* h, int64_t n_primal, const double* h_diag,
                              const int64_t* diag_source_pos) {
  if (!h || n_primal < 0 || n_primal > h->n || (!h_diag && n_primal) || (!diag_source_pos && h->n)) {
    return B200LU_INVALID_ARGUMENT;
  }
  CU_TRY(h, cudaSetDevice(h->device));
  std::vector<int32_t> pos(h->n);
  for (int64_t i = 0; i < h->n; ++i) {
    const int64_t k = diag_source_pos[i];
    if (k < h->src_row_offsets[i] || k >= h->src_row_offsets[i + 1] || h->src_col_indices[k] != i) {
      h->last_error = "kkt_bind: diag_source_pos[" + std::to_string(i) + "] does not address K's diagonal";
      return B200LU_INVALID_ARGUMENT;
    }
    pos[i] = static_cast<int32_t>(k);
  }
  for (void* p : {static_cast<void*>(h->d_kkt_hdiag), static_cast<void*>(h->d_kkt_dy), static_cast<void*>(h->d_kkt_pos)}) {
    if (p) cudaFree(p);
  }
  ST_TRY(dev_upload(h, &h->d_kkt_pos, pos));
  ST_TRY(dev_upload(h, &h->d_kkt_hdiag, std::vector<double>(h_diag, h_diag + n_primal)));
  ST_TRY(dev_alloc(h, &h->d_kkt_dy, static_cast<size_t>(n_primal)));
  h->kkt_n_primal = n_primal;
  return B200LU_OK;
}

b200lu_status b200lu_kkt_update(b200lu_handle* h, const double* d_y, int on_device, double delta_p, double delta_d) {
  if (!h || (!d_y && h->kkt_n_primal > 0)) return B200LU_INVALID_ARGUMENT;
  CU_TRY(h, cudaSetDevice(h->device));
  if (h->kkt_n_primal < 0 || !h->have_values) {
    h->last_error = "kkt_update: call b200lu_kkt_bind and give one full set of values (reset_values) first";
    return B200LU_INVALID_ARGUMENT;
  }
  if (delta_p < 0.0 || delta_d < 0.0) {  // src/kkt.cpp:44-46
    h->last_error = "kkt_update: regularization must be nonnegative";
    return B200LU_INVALID_ARGUMENT;
  }
  const double* dy = d_y;
  if (!on_device && h->kkt_n_primal > 0) {
    CU_TRY(h, cudaMemcpyAsync(h->d_kkt_dy, d_y, static_cast<size_t>(h->kkt_n_primal) * sizeof(double),
                              cudaMemcpyHostToDevice, h->stream));
    dy = h->d_kkt_dy;
  }
  h->valid = false;
  if (h->n > 0) {
    PhaseScope ps(h, B200LU_PHASE_SCATTER);
    kkt_diagonal_kernel<<<blocks_for(h->n, 256), 256, 0, h->stream>>>(static_cast<int32_t>(h->n),
                                                                      static_cast<int32_t>(h->kkt_n_primal), h->d_kkt_hdiag,
                                                                      h->d_kkt_pos, dy, delta_p, delta_d, h->d_a_vals);
    ST_TRY(check_launch(h, "kkt_diagonal_kernel"));
  }
  ST_TRY(launch_scatter(h));
  h->scattered = true;
  return B200LU_OK;
}

b200lu_status b200lu_factorize_scattered(b200lu_handle* h, int64_t* failed_row) {
  if (!h) return B200LU_INVALID_ARGUMENT;
  CU_TRY(h, cudaSetDevice(h->device));
  if (!h->scattered) {
    h->last_error = "factorize_scattered: no scattered values (call reset_values first)";
    return B200LU_INVALID_ARGUMENT;
  }
  return launch_factor(h, failed_row);
}

b200lu_status b200lu_refactorize(b200lu_handle* h, const double* a_values, int on_device,
                                 int64_t* failed_row) {
  ST_TRY(b200lu_reset_values(h, a_values, on_device));
  return launch_factor(h, failed_row);
}

int b200lu_valid(const b200lu_handle* h) { return h && h->valid ? 1 : 0; }
uint64_t b200lu_generation(const b200lu_handle* h) { return h ? h->generation : 0; }

b200lu_status b200lu_get_values(b200lu_handle* h, double* host_out) {
  if (!h || (!host_out && h->nnz_factors)) return B200LU_INVALID_ARGUMENT;
  CU_TRY(h, cudaSetDevice(h->device));
  const double* src = h->scattered ? h->d_work : h->d_values;
  if (h->nnz_factors) {
    CU_TRY(h, cudaMemcpyAsync(host_out, src, static_cast<size_t>(h->nnz_factors) * sizeof(double),
                              cudaMemcpyDeviceToHost, h->stream));
  }
  CU_TRY(h, cudaStreamSynchronize(h->stream));
  return B200LU_OK;
}

b200lu_status b200lu_set_values(b200lu_handle* h, const double* host_in, int valid) {
  if (!h || (!host_in && h->nnz_factors)) return B200LU_INVALID_ARGUMENT;
  CU_TRY(h, cudaSetDevice(h->device));
  if (h->nnz_factors) {
    CU_TRY(h, cudaMemcpyAsync(h->d_values, host_in, static_cast<size_t>(h->nnz_factors) * sizeof(double),
                              cudaMemcpyHostToDevice, h->stream));
  }
  CU_TRY(h, cudaStreamSynchronize(h->stream));
  h->scattered = false;
  h->valid = valid != 0;
  return B200LU_OK;
}

const double* b200lu_values_device(const b200lu_handle* h) { return h ? h->d_values : nullptr; }

b200lu_status b200lu_lower_solve(b200lu_handle* h, int64_t len, const double* y, double* x, int on_device) {
  if (!h || (!y && len) || (!x && len)) return B200LU_INVALID_ARGUMENT;
  CU_TRY(h, cudaSetDevice(h->device));
  ST_TRY(check_solve_ready(h, len, "lower_solve"));
  if (h->n == 0) return B200LU_OK;
  cudaError_t e = cudaSuccess;
  const double* dy = stage_in(h, y, h->d_in, on_device, &e);
  CU_TRY(h, e);
  arm_solve_kernel<<<1, 1, 0, h->stream>>>(h->d_counters, h->d_failed + 1);
  ST_TRY(check_launch(h, "arm_solve_kernel"));
  fill_pending_kernel<<<blocks_for(h->n, 256), 256, 0, h->stream>>>(h->n, h->d_t1);
  ST_TRY(check_launch(h, "fill_pending_kernel"));
  ST_TRY(launch_lower(h, dy, h->d_t1));
  if (on_device) {
    ST_TRY(copy_dd(h, x, h->d_t1));
    CU_TRY(h, cudaStreamSynchronize(h->stream));
    return B200LU_OK;
  }
  return stage_out(h, h->d_t1, x, 0);
}

b200lu_status b200lu_upper_solve(b200lu_handle* h, int64_t len, const double* y, double* x, int on_device,
                                 int64_t* failed_row) {
  if (failed_row) *failed_row = -1;
  if (!h || (!y && len) || (!x && len)) return B200LU_INVALID_ARGUMENT;
  CU_TRY(h, cudaSetDevice(h->device));
  ST_TRY(check_solve_ready(h, len, "upper_solve"));
  if (h->n == 0) return B200LU_OK;
  cudaError_t e = cudaSuccess;
  const double* dy = stage_in(h, y, h->d_in, on_device, &e);
  CU_TRY(h, e);
  arm_solve_kernel<<<1, 1, 0, h->stream>>>(h->d_counters, h->d_failed + 1);
  ST_TRY(check_launch(h, "arm_solve_kernel"));
  fill_pending_kernel<<<blocks_for(h->n, 256), 256, 0, h->stream>>>(h->n, h->d_t2);
  ST_TRY(check_launch(h, "fill_pending_kernel"));
  ST_TRY(launch_upper(h, dy, h->d_t2));
  ST_TRY(collect_upper_failure(h, failed_row));  // src/trisolve.cpp:64-67
  if (on_device) {
    ST_TRY(copy_dd(h, x, h->d_t2));
    CU_TRY(h, cudaStreamSynchronize(h->stream));
    return B200LU_OK;
  }
  return stage_out(h, h->d_t2, x, 0);
}

b200lu_status b200lu_solve(b200lu_handle* h, int64_t len, const double* b, double* x, int on_device,
                           int64_t* failed_row) {
  if (failed_row) *failed_row = -1;
  if (!h || (!b && len) || (!x && len)) return B200LU_INVALID_ARGUMENT;
  CU_TRY(h, cudaSetDevice(h->device));
  ST_TRY(check_solve_ready(h, len, "solve_system"));
  if (h->n == 0) return B200LU_OK;
  cudaError_t e = cudaSuccess;
  const double* db = stage_in(h, b, h->d_in, on_device, &e);
  CU_TRY(h, e);
  double* dx = on_device ? x : h->d_out;
  ST_TRY(solve_device(h, db, dx));
  ST_TRY(collect_upper_failure(h, failed_row));
  return stage_out(h, dx, x, on_device);
}

b200lu_status b200lu_spmv(b200lu_handle* h, const double* x, double* y, int on_device) {
  if (!h || (!x && h->n) || (!y && h->n)) return B200LU_INVALID_ARGUMENT;
  CU_TRY(h, cudaSetDevice(h->device));
  cudaError_t e = cudaSuccess;
  const double* dx = stage_in(h, x, h->d_in, on_device, &e);
  CU_TRY(h, e);
  double* dy = on_device ? y : h->d_out;
  ST_TRY(launch_spmv(h, dx, dy));
  if (on_device) {
    CU_TRY(h, cudaStreamSynchronize(h->stream));
    return B200LU_OK;
  }
  return stage_out(h, dy, y, 0);
}

b200lu_status b200lu_relative_residual(b200lu_handle* h, const double* x, const double* b, int on_device,
                                       double* out) {
  if (!h || !out || (!x && h->n) || (!b && h->n)) return B200LU_INVALID_ARGUMENT;
  CU_TRY(h, cudaSetDevice(h->device));
  if (h->n == 0) {
    *out = 0.0;
    return B200LU_OK;
  }
  cudaError_t e = cudaSuccess;
  const double* dx = stage_in(h, x, h->d_in, on_device, &e);
  CU_TRY(h, e);
  const double* db = stage_in(h, b, h->d_in2, on_device, &e);
  CU_TRY(h, e);
  ST_TRY(launch_residual(h, dx, db, h->d_r, kSlotRes));
  ST_TRY(read_scalars(h, kSlotRes, 2));
  const double bn = std::sqrt(h->h_scal[kSlotBn]);
  *out = std::sqrt(h->h_scal[kSlotRes]) / (bn > 0.0 ? bn : 1.0);  // src/sparse.cpp:286-287
  return B200LU_OK;
}

b200lu_status b200lu_refine_fgmres(b200lu_handle* h, const double* b, const double* x0, double* x_out,
                                   int on_device, int use_preconditioner, const b200lu_refine_config* cfg,
                                   b200lu_refine_outcome* outcome) {
  return refine_common(h, b, x0, x_out, on_device, use_preconditioner, cfg, outcome, true);
}

b200lu_status b200lu_refine_classic(b200lu_handle* h, const double* b, const double* x0, double* x_out,
                                    int on_device, int use_preconditioner, const b200lu_refine_config* cfg,
                                    b200lu_refine_outcome* outcome) {
  return refine_common(h, b, x0, x_out, on_device, use_preconditioner, cfg, outcome, false);
}

// cgs2_orthonormalize (src/refine.cpp:8-26): two passes of "h = dot(basis_j, v); coefficient_j += h;
// v -= h * basis_j" over the basis, then the norm; breakdown when norm <= 1e-300, otherwise v / norm.
// The device kernels are the ones fgmres_refine uses for its orthogonalisation step.
b200lu_status b200lu_cgs2_orthonormalize(b200lu_handle* h, int64_t k, const double* basis, const double* v, int on_device,
                                         double* coefficients_out, double* vector_out, double* norm_out, int* breakdown_out) {
  if (!h || k < 0 || (k > 0 && (!basis || !coefficients_out)) || (h->n && (!v || !vector_out)) || !norm_out || !breakdown_out) {
    return B200LU_INVALID_ARGUMENT;
  }
  CU_TRY(h, cudaSetDevice(h->device));
  if (k > h->refine_capacity) {
    h->last_error = "cgs2_orthonormalize: more basis vectors than the handle's refine_capacity";
    return B200LU_INVALID_ARGUMENT;
  }
  const int64_t n = h->n;
  const int32_t n32 = static_cast<int32_t>(n);
  const int nb = blocks_for(n, 256);
  *norm_out = 0.0;
  *breakdown_out = 1;
  if (n == 0) return B200LU_OK;
  const cudaMemcpyKind in_kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  if (k > 0) CU_TRY(h, cudaMemcpyAsync(h->d_V, basis, static_cast<size_t>(k) * n * sizeof(double), in_kind, h->stream));
  CU_TRY(h, cudaMemcpyAsync(h->d_wv, v, static_cast<size_t>(n) * sizeof(double), in_kind, h->stream));
  CU_TRY(h, cudaMemsetAsync(h->d_scal + kSlotCoef, 0, static_cast<size_t>(std::max<int64_t>(k, 1)) * sizeof(double), h->stream));
  for (int pass = 0; pass < 2; ++pass) {
    for (int64_t j = 0; j < k; ++j) {
      ST_TRY(launch_dot(h, h->d_V + j * n, h->d_wv, kSlotH));
      {
        PhaseScope ps(h, B200LU_PHASE_VECTOR);
        project_out_kernel<<<nb, 256, 0, h->stream>>>(n32, h->d_scal + kSlotH, h->d_scal + kSlotCoef + j, h->d_V + j * n, h->d_wv);
      }
      ST_TRY(check_launch(h, "project_out_kernel"));
    }
  }
  ST_TRY(launch_dot(h, h->d_wv, h->d_wv, kSlotNorm));
  ST_TRY(read_scalars(h, kSlotNorm, static_cast<int>(kSlotCoef + k - kSlotNorm)));
  const double norm = std::sqrt(h->h_scal[kSlotNorm]);
  for (int64_t j = 0; j < k; ++j) coefficients_out[j] = h->h_scal[kSlotCoef + j];
  *norm_out = norm;
  *breakdown_out = norm <= 1e-300 ? 1 : 0;
  const double* result = h->d_wv;  // on breakdown the vector is unspecified (include/rlu/refine.hpp:27): the remainder
  if (!*breakdown_out) {
    {
      PhaseScope ps(h, B200LU_PHASE_VECTOR);
      divide_kernel<<<nb, 256, 0, h->stream>>>(n32, norm, h->d_wv, h->d_r);
    }
    ST_TRY(check_launch(h, "divide_kernel"));
    result = h->d_r;
  }
  CU_TRY(h, cudaMemcpyAsync(vector_out, result, static_cast<size_t>(n) * sizeof(double),
                            on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, h->stream));
  CU_TRY(h, cudaStreamSynchronize(h->stream));
  return B200LU_OK;
}

b200lu_status b200lu_get_stats(const b200lu_handle* h, b200lu_stats* out) {
  if (!h || !out) return B200LU_INVALID_ARGUMENT;
  out->n = h->n;
  out->nnz_factors = h->nnz_factors;
  out->nnz_source = h->nnz_source;
  out->nnz_lower = h->sched.nnz_lower;
  out->update_pairs = h->sched.update_pairs;
  out->lower_levels = h->sched.lower_levels;
  out->upper_levels = h->sched.upper_levels;
  out->max_row_len = h->sched.max_row_len;
  out->big_rows = static_cast<int64_t>(h->sched.big_rows.size());
  out->device_bytes = h->device_bytes;
  out->alloc_events = h->alloc_events;
  out->lower_tail_rows = h->sched.lower_tail.rows;
  out->lower_tail_levels = h->sched.lower_tail.levels;
  out->upper_tail_rows = h->sched.upper_tail.rows;
  out->upper_tail_levels = h->sched.upper_tail.levels;
  return B200LU_OK;
}

b200lu_status b200lu_schedule_probe(const b200lu_symbolic_view* sym, b200lu_stats* stats,
                                    int32_t* lower_order, int32_t* upper_order, int64_t* pair_row_ptr,
                                    char* error_buf, int error_buf_len) {
  if (!sym) return B200LU_INVALID_ARGUMENT;
  Schedule S;
  const std::string err = build_schedule(*sym, ScheduleTuning{}, S);
  if (error_buf && error_buf_len > 0) {
    std::strncpy(error_buf, err.c_str(), static_cast<size_t>(error_buf_len) - 1);
    error_buf[error_buf_len - 1] = '\0';
  }
  if (!err.empty()) return B200LU_INVALID_ARGUMENT;
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    stats->n = S.n;
    stats->nnz_factors = S.nnz;
    stats->nnz_source = sym->nnz_source;
    stats->nnz_lower = S.nnz_lower;
    stats->update_pairs = S.update_pairs;
    stats->lower_levels = S.lower_levels;
    stats->upper_levels = S.upper_levels;
    stats->max_row_len = S.max_row_len;
    stats->big_rows = static_cast<int64_t>(S.big_rows.size());
    stats->lower_tail_rows = S.lower_tail.rows;
    stats->lower_tail_levels = S.lower_tail.levels;
    stats->upper_tail_rows = S.upper_tail.rows;
    stats->upper_tail_levels = S.upper_tail.levels;
  }
  if (lower_order && S.n) std::memcpy(lower_order, S.lower_order.data(), sizeof(int32_t) * S.n);
  if (upper_order && S.n) std::memcpy(upper_order, S.upper_order.data(), sizeof(int32_t) * S.n);
  if (pair_row_ptr) std::memcpy(pair_row_ptr, S.pair_row_ptr.data(), sizeof(int64_t) * (S.n + 1));
  return B200LU_OK;
}

uint64_t b200lu_launch_count(const b200lu_handle* h) { return h ? h->launches : 0; }

b200lu_status b200lu_set_timing(b200lu_handle* h, int enabled) {
  if (!h) return B200LU_INVALID_ARGUMENT;
  CU_TRY(h, cudaSetDevice(h->device));
  if (enabled && h->ev_start.empty()) {
    h->ev_start.resize(kMaxTimedLaunches);
    h->ev_stop.resize(kMaxTimedLaunches);
    h->ev_phase.assign(kMaxTimedLaunches, 0);
    for (int i = 0; i < kMaxTimedLaunches; ++i) {
      CU_TRY(h, cudaEventCreate(&h->ev_start[i]));
      CU_TRY(h, cudaEventCreate(&h->ev_stop[i]));
    }
  }
  h->timing = enabled != 0;
  h->ev_used = 0;
  return B200LU_OK;
}

b200lu_status b200lu_get_phase_times(b200lu_handle* h, double* ms_out, int64_t* count_out, int reset) {
  if (!h || !ms_out || !count_out) return B200LU_INVALID_ARGUMENT;
  CU_TRY(h, cudaSetDevice(h->device));
  CU_TRY(h, cudaStreamSynchronize(h->stream));
  for (int p = 0; p < B200LU_NUM_PHASES; ++p) {
    ms_out[p] = 0.0;
    count_out[p] = 0;
  }
  for (int i = 0; i < h->ev_used; ++i) {
    float ms = 0.f;
    CU_TRY(h, cudaEventElapsedTime(&ms, h->ev_start[i], h->ev_stop[i]));
    ms_out[h->ev_phase[i]] += ms;
    ++count_out[h->ev_phase[i]];
  }
  if (reset) h->ev_used = 0;
  return B200LU_OK;
}

b200lu_status b200lu_synchronize(b200lu_handle* h) {
  if (!h) return B200LU_INVALID_ARGUMENT;
  CU_TRY(h, cudaSetDevice(h->device));
  CU_TRY(h, cudaStreamSynchronize(h->stream));
  return B200LU_OK;
}

}  // extern "C"
