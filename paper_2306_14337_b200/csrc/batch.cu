// b200lu scenario batches — handle, host-side orchestration and the b200lu_batch_* C ABI
// (include/b200lu.h). Kernels: batch.cuh. One handle owns B scenarios that share one symbolic
// analysis; every scenario's arithmetic is the reference's single-system arithmetic
// (src/numeric.cpp, src/trisolve.cpp, src/sparse.cpp), and the refinement control flow is
// fgmres_refine (src/refine.cpp:39-142) evaluated per scenario in lockstep.
#include "b200lu.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <queue>
#include <string>
#include <utility>
#include <vector>

#include "batch.cuh"
#include "schedule.hpp"
#include "tile.cuh"
#include "gather.cuh"
#include "snode.cuh"
#include "blockmc.cuh"
#include "blockteam.cuh"
#include "tristeam.cuh"

using namespace b200lu;

namespace {
constexpr int kBWarps = 8;
constexpr int kScalSlots = 40;  // device->host scalar rows (each `padded` doubles)
constexpr int kUpSlots = 64;    // host->device scalar rows
constexpr int kMaxTimedLaunches = 4096;

__global__ void barm_kernel(unsigned long long* tickets, int32_t* failed, int32_t padded, int32_t value) {
  const int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < 4) tickets[t] = 0ull;
  if (t < padded) failed[t] = value;
}

__global__ void bgather_scenario_kernel(int64_t len, int64_t group_base, int lane_of, const double* __restrict__ src,
                                        double* __restrict__ dst) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < len) dst[k] = src[(group_base + k) * 32 + lane_of];
}
}  // namespace

struct b200lu_batch {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool owns_stream = false;
  double pivot_floor = 1e-30;
  int refine_capacity = 20;

  Schedule sched;
  int64_t n = 0, nnz_factors = 0, nnz_source = 0;
  int32_t batch = 0, padded = 0, groups = 0;
  int unit = 32;         // scenarios per refactorization unit (S): one lane per scenario
  int32_t units = 0;     // padded / unit
  bool has_match = false, dest16 = true;
  std::vector<int64_t> src_row_offsets, src_col_indices;
  std::vector<uint8_t> valid;  // per scenario
  int32_t gen = 0;

  int32_t *d_row_ptr = nullptr, *d_col = nullptr, *d_diag = nullptr, *d_trivial_rows = nullptr;
  int64_t* d_pair_row_ptr = nullptr;
  FactorMeta* d_factor_meta = nullptr;
  int32_t n_factor_rows = 0;   // rows with pivots handled row by row (the wide head of the DAG)
  FactorMeta* d_tail_meta = nullptr;  // trailing part row by row (latency-optimised kernel instance)
  int32_t n_tail_rows = 0;
  void (*tail_fn)(BFactorArgs) = nullptr;
  int tail_grid = 0;
  BlockMeta* d_blocks = nullptr;  // row-blocked trailing part (experimental)
  MergedPivot* d_merged = nullptr;
  int32_t n_blocks = 0, n_block_rows = 0;
  int64_t blocked_pairs = 0;
  void (*block_fn)(BBlockArgs) = nullptr;
  int block_grid = 0;
  size_t block_smem = 0;
  void (*team_fn)(BBlockArgs) = nullptr;  // bfactor_block_team_kernel (blockteam.cuh): two warps per block
  int team_grid = 0;
  size_t team_smem = 0;
  int mc_contexts = 0;  // > 0: bfactor_block_mc_kernel with that many block contexts per warp (blockmc.cuh)
  void (*mc_fn)(BBlockArgs, int) = nullptr;
  int mc_grid = 0;
  size_t mc_smem = 0;
  // tiled trailing part (tile.cuh): rows resident in shared memory, pivot rows streamed by TMA
  bool use_tiles = false, tile_auto = true;

  std::string tile_note;          // why the tiled kernel is not used, if it is not
  TileMeta* d_tile_meta = nullptr;
  TileRow* d_tile_rows = nullptr;
  ExtItem* d_tile_ext = nullptr;
  RowItem* d_tile_row_items = nullptr;
  uint16_t* d_tile_dest = nullptr;
  int32_t* d_tile_flags = nullptr;  // [n][tile_units]
  long long* d_tile_prof = nullptr; // phase counters of the tiled kernel (-DB200LU_TILE_PROF builds)
  int32_t n_tiles = 0, tile_units = 0, tile_rows_per = 8, tile_ring_blocks = 32, tile_ctas = 2;
  int64_t tile_fetched_entries = 0;
  void (*tile_fn)(BTileArgs) = nullptr;
  int tile_grid = 0;
  size_t tile_smem = 0;
  BTileArgs tile_args;
  // gather-form trailing part (gather.cuh): register accumulation per (target, batch of pivots)
  bool use_gather = false;
  GBlock* d_g_blocks = nullptr;
  GBatch* d_g_batches = nullptr;
  GRec* d_g_recs = nullptr;
  int32_t* d_g_waits = nullptr;
  int32_t n_g_blocks = 0, gather_rows_per = 2, gather_batch = 16;
  int64_t gather_records = 0, gather_targets = 0;
  void (*gather_fn)(BGatherArgs) = nullptr;
  int gather_grid = 0;
  size_t gather_smem = 0;
  // supernodal trailing part (snode.cuh): dense runs of nested pivot rows, register accumulation per destination
  bool use_snode = false;
  SBlock* d_s_blocks = nullptr;
  SRun* d_s_runs = nullptr;
  uint32_t* d_s_dest = nullptr;
  int32_t n_s_blocks = 0, snode_rows_per = 2;
  void (*snode_fn)(BSnodeArgs) = nullptr;
  int snode_grid = 0;
  RowMeta *d_lower_meta = nullptr, *d_upper_meta = nullptr;
  void* d_dest = nullptr;
  int32_t* d_src_of_slot = nullptr;
  double* d_scatter_scale = nullptr;
  int32_t *d_p = nullptr, *d_pq = nullptr;
  double *d_row_scale = nullptr, *d_col_scale = nullptr;
  int32_t *d_a_row_ptr = nullptr, *d_a_col = nullptr;

  int64_t kkt_n_primal = -1;
  double *d_kkt_hdiag = nullptr, *d_kkt_dy = nullptr, *d_kkt_stage = nullptr;
  int32_t* d_kkt_pos = nullptr;
  bool have_values = false;
  double *d_a_int = nullptr, *d_values = nullptr;
  int32_t* d_flags = nullptr;
  int32_t* d_failed = nullptr;  // [2][padded]: factor (atomicMin), upper (atomicMax)
  unsigned long long* d_tickets = nullptr;
  double *d_stage_a = nullptr, *d_stage_in = nullptr, *d_stage_in2 = nullptr, *d_stage_out = nullptr, *d_gather = nullptr;
  double *d_w = nullptr, *d_t1 = nullptr, *d_t2 = nullptr, *d_b = nullptr, *d_x0 = nullptr, *d_x = nullptr,
         *d_r = nullptr, *d_wv = nullptr, *d_cand = nullptr, *d_best = nullptr, *d_V = nullptr, *d_Z = nullptr;
  double *d_scal = nullptr, *d_up = nullptr, *d_partials = nullptr;
  double *h_scal = nullptr, *h_up = nullptr;
  int32_t* h_failed = nullptr;
  int up_used = 0;

  void (*factor_fn)(BFactorArgs) = nullptr;
  int factor_grid = 0, tri_grid = 0, tri_grid_upper = 0, tri_grid_chain = 0;
  void (*chain_fn)(BTriArgs) = nullptr;  // U sweep, narrow leading levels
  int chain_warps = 8, chain_buf = kTriBufferedChain;
  bool chain_team = false;  // the chain launch runs btri_upper_team_kernel (a team of warps per row)
  int chain_team_size = 1;
  int32_t upper_chain_rows = 0;  // leading rows of the U level order handled by the chain launch
  size_t factor_smem = 0;

  // staged (pipelined) submission: the next system's inputs are copied H2D on their own stream while the
  // current one is processed, results leave on a third stream (b200lu_batch_stage_inputs & co.)
  cudaStream_t copy_in = nullptr, copy_out = nullptr;
  cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_vals_used[2] = {nullptr, nullptr}, ev_rhs_used[2] = {nullptr, nullptr},
              ev_x[2] = {nullptr, nullptr}, ev_x_out[2] = {nullptr, nullptr};
  double *d_stage_vals[2] = {nullptr, nullptr}, *d_stage_rhs[2] = {nullptr, nullptr}, *d_stage_x[2] = {nullptr, nullptr};
  int stage_fill = 0;                    // buffer the next stage_inputs fills
  std::vector<int> vals_queue, rhs_queue;  // staged buffers not yet consumed, oldest first (at most two each)
  bool staged_ready = false;

  int64_t alloc_events = 0, device_bytes = 0;
  uint64_t launches = 0;
  std::string last_error;

  bool timing = false;
  std::vector<cudaEvent_t> ev_start, ev_stop;
  std::vector<int> ev_phase;
  int ev_used = 0;
};

namespace {

using H = b200lu_batch;

#define CU_TRY(h, expr)                                                      \
  do {                                                                       \
    cudaError_t e__ = (expr);                                                \
    if (e__ != cudaSuccess) {                                                \
      (h)->last_error = std::string(#expr) + ": " + cudaGetErrorString(e__); \
      return B200LU_CUDA_ERROR;                                              \
    }                                                                        \
  } while (0)

#define ST_TRY(expr)                  \
  do {                                \
    b200lu_status s__ = (expr);       \
    if (s__ != B200LU_OK) return s__; \
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

inline int64_t vec_elems(const H* h) { return h->n * h->padded; }
inline int warp_blocks(const H* h) { return blocks_for(h->n * h->groups * 32, 256); }

// ---- layout changes between the caller's scenario-major arrays and the interleaved storage

b200lu_status to_interleaved(H* h, int64_t len, const double* src_dev, double* dst) {
  if (len == 0) return B200LU_OK;
  PhaseScope ps(h, B200LU_PHASE_PERMUTE);
  dim3 grid(static_cast<unsigned>((len + 31) / 32), static_cast<unsigned>(h->groups));
  interleave_kernel<<<grid, 256, 0, h->stream>>>(len, h->batch, src_dev, dst);
  return check_launch(h, "interleave_kernel");
}

b200lu_status from_interleaved(H* h, int64_t len, const double* src, double* dst_dev) {
  if (len == 0) return B200LU_OK;
  PhaseScope ps(h, B200LU_PHASE_PERMUTE);
  dim3 grid(static_cast<unsigned>((len + 31) / 32), static_cast<unsigned>(h->groups));
  deinterleave_kernel<<<grid, 256, 0, h->stream>>>(len, h->batch, src, dst_dev);
  return check_launch(h, "deinterleave_kernel");
}

// caller's [batch][n] vector (host or device) -> interleaved device vector
b200lu_status vec_in(H* h, const double* p, int on_device, double* staging, double* dst) {
  const double* src = p;
  if (!on_device) {
    CU_TRY(h, cudaMemcpyAsync(staging, p, static_cast<size_t>(h->n) * h->batch * sizeof(double), cudaMemcpyHostToDevice,
                              h->stream));
    src = staging;
  }
  return to_interleaved(h, h->n, src, dst);
}

// interleaved device vector -> caller's [batch][n] vector; synchronises
b200lu_status vec_out(H* h, const double* src, double* p, int on_device) {
  if (on_device) {
    ST_TRY(from_interleaved(h, h->n, src, p));
  } else {
    ST_TRY(from_interleaved(h, h->n, src, h->d_stage_out));
    CU_TRY(h, cudaMemcpyAsync(p, h->d_stage_out, static_cast<size_t>(h->n) * h->batch * sizeof(double),
                              cudaMemcpyDeviceToHost, h->stream));
  }
  CU_TRY(h, cudaStreamSynchronize(h->stream));
  return B200LU_OK;
}

// ---- scalar traffic

b200lu_status read_scalars(H* h, int first_slot, int slots) {
  CU_TRY(h, cudaMemcpyAsync(h->h_scal + static_cast<size_t>(first_slot) * h->padded,
                            h->d_scal + static_cast<size_t>(first_slot) * h->padded,
                            static_cast<size_t>(slots) * h->padded * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CU_TRY(h, cudaStreamSynchronize(h->stream));
  h->up_used = 0;  // every earlier upload has been consumed
  return B200LU_OK;
}

// per-scenario scalars host -> device; returns the device row
b200lu_status upload_scalars(H* h, const std::vector<double>& v, const double** dev) {
  if (h->up_used >= kUpSlots) {
    CU_TRY(h, cudaStreamSynchronize(h->stream));
    h->up_used = 0;
  }
  double* hp = h->h_up + static_cast<size_t>(h->up_used) * h->padded;
  double* dp = h->d_up + static_cast<size_t>(h->up_used) * h->padded;
  for (int32_t s = 0; s < h->padded; ++s) hp[s] = v[std::min<int32_t>(s, h->batch - 1)];
  CU_TRY(h, cudaMemcpyAsync(dp, hp, static_cast<size_t>(h->padded) * sizeof(double), cudaMemcpyHostToDevice, h->stream));
  ++h->up_used;
  *dev = dp;
  return B200LU_OK;
}

double* scal(H* h, int slot) { return h->d_scal + static_cast<size_t>(slot) * h->padded; }
const double* hscal(const H* h, int slot) { return h->h_scal + static_cast<size_t>(slot) * h->padded; }

// ---- device stages

b200lu_status launch_scatter(H* h) {
  if (h->nnz_factors == 0) return B200LU_OK;
  PhaseScope ps(h, B200LU_PHASE_SCATTER);
  const int blocks = std::min<int64_t>(blocks_for(((h->nnz_factors + kScatterSlots - 1) / kScatterSlots) * h->groups * 32, 256), 148 * 16);
  bscatter_kernel<<<blocks, 256, 0, h->stream>>>(h->nnz_factors, h->nnz_source, h->groups, h->d_src_of_slot, h->d_a_int,
                                                 h->d_scatter_scale, h->d_values);
  return check_launch(h, "bscatter_kernel");
}

b200lu_status launch_factor(H* h, int64_t* failed_rows) {
  for (int32_t s = 0; failed_rows && s < h->batch; ++s) failed_rows[s] = -1;
  if (h->n == 0) {
    std::fill(h->valid.begin(), h->valid.end(), 1);
    return B200LU_OK;
  }
  ++h->gen;
  barm_kernel<<<blocks_for(std::max(h->padded, 4), 256), 256, 0, h->stream>>>(h->d_tickets, h->d_failed, h->padded, INT_MAX);
  ST_TRY(check_launch(h, "barm_kernel"));
  if (!h->sched.trivial_rows.empty()) {
    const int32_t cnt = static_cast<int32_t>(h->sched.trivial_rows.size());
    btrivial_pivot_kernel<<<blocks_for(static_cast<int64_t>(cnt) * h->groups * 32, 256), 256, 0, h->stream>>>(
        cnt, h->groups, h->nnz_factors, h->d_trivial_rows, h->d_diag, h->d_values, h->pivot_floor, h->d_failed);
    ST_TRY(check_launch(h, "btrivial_pivot_kernel"));
  }
  if (h->n_factor_rows > 0 || h->n_blocks > 0 || h->n_tail_rows > 0 || h->n_tiles > 0 || h->n_g_blocks > 0 || h->n_s_blocks > 0) {
    BFactorArgs a;
    a.n_rows = h->n_factor_rows;
    a.units = h->units;
    a.gen = h->gen;
    a.meta = h->d_factor_meta;
    a.row_ptr = h->d_row_ptr;
    a.col = h->d_col;
    a.diag = h->d_diag;
    a.pair_row_ptr = h->d_pair_row_ptr;
    a.dest = h->d_dest;
    a.values = h->d_values;
    a.nnz_factors = h->nnz_factors;
    a.flags = h->d_flags;
    a.pivot_floor = h->pivot_floor;
    a.failed = h->d_failed;
    a.ticket = h->d_tickets;
    PhaseScope ps(h, B200LU_PHASE_FACTOR);  // one scope: head launch + blocked trailing launch = one refactorization
    h->factor_fn<<<h->factor_grid, kBWarps * 32, h->factor_smem, h->stream>>>(a);
    ST_TRY(check_launch(h, "bfactor_kernel"));
    if (h->n_tail_rows > 0) {
      a.n_rows = h->n_tail_rows;
      a.meta = h->d_tail_meta;
      a.ticket = h->d_tickets + 1;
      h->tail_fn<<<h->tail_grid, kBWarps * 32, 0, h->stream>>>(a);
      ST_TRY(check_launch(h, "bfactor_kernel<tail>"));
    }
    if (h->use_tiles && h->n_tiles > 0) {
      BTileArgs& ta = h->tile_args;
      ta.gen = h->gen;
      ta.ticket = h->d_tickets + 1;
      h->tile_fn<<<h->tile_grid, (h->tile_rows_per + 1) * 32, h->tile_smem, h->stream>>>(ta);
      ST_TRY(check_launch(h, "bfactor_tile_kernel"));
    }
    if (h->use_snode && h->n_s_blocks > 0) {
      BSnodeArgs sa;
      sa.n_blocks = h->n_s_blocks;
      sa.units = h->units;
      sa.gen = h->gen;
      sa.blocks = h->d_s_blocks;
      sa.runs = h->d_s_runs;
      sa.dest = h->d_s_dest;
      sa.diag = h->d_diag;
      sa.values = h->d_values;
      sa.nnz_factors = h->nnz_factors;
      sa.flags = h->d_flags;
      sa.pivot_floor = h->pivot_floor;
      sa.failed = h->d_failed;
      sa.ticket = h->d_tickets + 1;
      h->snode_fn<<<h->snode_grid, 256, 0, h->stream>>>(sa);
      ST_TRY(check_launch(h, "bfactor_snode_kernel"));
    }
    if (h->use_gather && h->n_g_blocks > 0) {
      BGatherArgs ga;
      ga.n_blocks = h->n_g_blocks;
      ga.units = h->units;
      ga.gen = h->gen;
      ga.blocks = h->d_g_blocks;
      ga.batches = h->d_g_batches;
      ga.recs = h->d_g_recs;
      ga.waits = h->d_g_waits;
      ga.diag = h->d_diag;
      ga.values = h->d_values;
      ga.nnz_factors = h->nnz_factors;
      ga.flags = h->d_flags;
      ga.pivot_floor = h->pivot_floor;
      ga.failed = h->d_failed;
      ga.ticket = h->d_tickets + 1;
      ga.exp_nowait = std::getenv("B200LU_GATHER_NOWAIT") ? 1 : 0;
      h->gather_fn<<<h->gather_grid, 256, h->gather_smem, h->stream>>>(ga);
      ST_TRY(check_launch(h, "bfactor_gather_kernel"));
    }
    if (h->n_blocks > 0) {
      BBlockArgs bb;
      bb.n_blocks = h->n_blocks;
      bb.first_unit = 0;
      bb.units_here = h->units;
      bb.units = h->units;
      bb.gen = h->gen;
      bb.blocks = h->d_blocks;
      bb.merged = h->d_merged;
      bb.row_ptr = h->d_row_ptr;
      bb.diag = h->d_diag;
      bb.pair_row_ptr = h->d_pair_row_ptr;
      bb.dest = h->d_dest;
      bb.values = h->d_values;
      bb.nnz_factors = h->nnz_factors;
      bb.flags = h->d_flags;
      bb.pivot_floor = h->pivot_floor;
      bb.failed = h->d_failed;
      bb.ticket = h->d_tickets + 1;
      if (h->team_fn) {
        h->team_fn<<<h->team_grid, kTeamWarps * 32, h->team_smem, h->stream>>>(bb);
        ST_TRY(check_launch(h, "bfactor_block_team_kernel"));
      } else if (h->mc_contexts > 0) {
        h->mc_fn<<<h->mc_grid, 256, h->mc_smem, h->stream>>>(bb, h->mc_contexts);
        ST_TRY(check_launch(h, "bfactor_block_mc_kernel"));
      } else {
        h->block_fn<<<h->block_grid, 256, h->block_smem, h->stream>>>(bb);
        ST_TRY(check_launch(h, "bfactor_block_kernel"));
      }
    }
  }
  CU_TRY(h, cudaMemcpyAsync(h->h_failed, h->d_failed, static_cast<size_t>(h->padded) * sizeof(int32_t),
                            cudaMemcpyDeviceToHost, h->stream));
  CU_TRY(h, cudaStreamSynchronize(h->stream));
  bool any = false;
  for (int32_t s = 0; s < h->batch; ++s) {
    const bool ok = h->h_failed[s] == INT_MAX;
    h->valid[s] = ok ? 1 : 0;  // src/numeric.cpp:51-55: a failed system's factors stay invalid
    if (!ok) {
      any = true;
      if (failed_rows) failed_rows[s] = h->h_failed[s];
      h->last_error = "zero pivot at row " + std::to_string(h->h_failed[s]) + " of scenario " + std::to_string(s);
    }
  }
  return any ? B200LU_ZERO_PIVOT : B200LU_OK;
}

BTriArgs tri_args(H* h, const RowMeta* meta, const double* y, double* x, int ticket_slot) {
  BTriArgs a;
  a.n = static_cast<int32_t>(h->n);
  a.first = 0;
  a.count = a.n;
  a.groups = h->groups;
  a.meta = meta;
  a.col = h->d_col;
  a.diag = h->d_diag;
  a.values = h->d_values;
  a.nnz_factors = h->nnz_factors;
  a.y = y;
  a.x = x;
  a.ticket = h->d_tickets + ticket_slot;
  a.failed = h->d_failed + h->padded;
  return a;
}

b200lu_status arm_solve(H* h) {
  barm_kernel<<<blocks_for(std::max(h->padded, 4), 256), 256, 0, h->stream>>>(h->d_tickets, h->d_failed + h->padded,
                                                                            h->padded, -1);
  return check_launch(h, "barm_kernel");
}

b200lu_status launch_lower(H* h, const double* y, double* x) {
  PhaseScope ps(h, B200LU_PHASE_LOWER);
  // static claim order: the grid must be co-resident (launch_resident, common.cuh)
  CU_TRY(h, launch_resident(btri_kernel<false, kTriBufferedWide>, h->tri_grid, 256, 0, h->stream, tri_args(h, h->d_lower_meta, y, x, 1)));
  return check_launch(h, "btri_kernel<lower>");
}

b200lu_status launch_upper(H* h, const double* y, double* x) {
  PhaseScope ps(h, B200LU_PHASE_UPPER);
  BTriArgs a = tri_args(h, h->d_upper_meta, y, x, 2);
  if (h->upper_chain_rows > 0) {  // the narrow leading levels: whole rows parked, one CTA per SM
    a.count = h->upper_chain_rows;
    CU_TRY(h, launch_resident(h->chain_fn, h->tri_grid_chain, h->chain_warps * 32, tri_upper_smem(h->chain_buf, h->chain_team ? kTriTeams : h->chain_warps), h->stream, a));
    ST_TRY(check_launch(h, "btri_kernel<upper chain>"));
  }
  if (h->upper_chain_rows < h->n) {
    a.first = h->upper_chain_rows;
    a.count = static_cast<int32_t>(h->n) - h->upper_chain_rows;
    a.ticket = h->d_tickets + 3;
    CU_TRY(h, launch_resident(btri_kernel<true, kTriBufferedWide>, h->tri_grid_upper, 256, tri_upper_smem(kTriBufferedWide), h->stream, a));
    ST_TRY(check_launch(h, "btri_kernel<upper wide>"));
  }
  return B200LU_OK;
}

// solve_system (src/trisolve.cpp:90-119) on interleaved vectors; does not synchronise
b200lu_status solve_int(H* h, const double* b, double* x) {
  if (h->n == 0) return B200LU_OK;
  ST_TRY(arm_solve(h));
  {
    PhaseScope ps(h, B200LU_PHASE_PERMUTE);
    bpermute_in_kernel<<<warp_blocks(h), 256, 0, h->stream>>>(static_cast<int32_t>(h->n), h->groups, h->d_p,
                                                              h->d_row_scale, b, h->d_w, h->d_t1, h->d_t2);
    ST_TRY(check_launch(h, "bpermute_in_kernel"));
  }
  ST_TRY(launch_lower(h, h->d_w, h->d_t1));
  ST_TRY(launch_upper(h, h->d_t1, h->d_t2));
  PhaseScope ps(h, B200LU_PHASE_PERMUTE);
  bpermute_out_kernel<<<warp_blocks(h), 256, 0, h->stream>>>(static_cast<int32_t>(h->n), h->groups, h->d_pq,
                                                             h->d_col_scale, h->d_t2, x);
  return check_launch(h, "bpermute_out_kernel");
}

b200lu_status collect_upper_failure(H* h, int64_t* failed_rows) {
  for (int32_t s = 0; failed_rows && s < h->batch; ++s) failed_rows[s] = -1;
  if (h->n == 0) return B200LU_OK;
  CU_TRY(h, cudaMemcpyAsync(h->h_failed + h->padded, h->d_failed + h->padded, static_cast<size_t>(h->padded) * sizeof(int32_t),
                            cudaMemcpyDeviceToHost, h->stream));
  CU_TRY(h, cudaStreamSynchronize(h->stream));
  bool any = false;
  for (int32_t s = 0; s < h->batch; ++s) {
    const int32_t f = h->h_failed[h->padded + s];
    if (f >= 0 && h->valid[s]) {
      any = true;
      if (failed_rows) failed_rows[s] = f;
      h->last_error = "zero diagonal at row " + std::to_string(f) + " of scenario " + std::to_string(s);
    }
  }
  return any ? B200LU_ZERO_PIVOT : B200LU_OK;
}

b200lu_status any_valid(H* h, const char* who) {
  for (uint8_t v : h->valid) {
    if (v) return B200LU_OK;
  }
  h->last_error = std::string(who) + ": factors are not valid";  // src/trisolve.cpp:20
  return B200LU_INVALID_FACTORS;
}

b200lu_status launch_residual(H* h, const double* x, const double* b, double* r, int slot) {
  {
    PhaseScope ps(h, B200LU_PHASE_SPMV);
    bresidual_rows_kernel<<<warp_blocks(h), 256, 0, h->stream>>>(static_cast<int32_t>(h->n), h->groups, h->nnz_source,
                                                               h->d_a_row_ptr, h->d_a_col, h->d_a_int, x, b, r);
    ST_TRY(check_launch(h, "bresidual_rows_kernel"));
    dim3 grid(kBatchPartBlocks, static_cast<unsigned>(h->groups));
    bsumsq2_kernel<<<grid, 256, 0, h->stream>>>(static_cast<int32_t>(h->n), r, b, h->d_partials);
    ST_TRY(check_launch(h, "bsumsq2_kernel"));
  }
  PhaseScope ps(h, B200LU_PHASE_VECTOR);
  bfinish_kernel<<<h->groups, 32, 0, h->stream>>>(2, h->padded, h->d_partials, scal(h, slot));
  return check_launch(h, "bfinish_kernel");
}

b200lu_status launch_dot(H* h, const double* u, const double* v, int slot) {
  PhaseScope ps(h, B200LU_PHASE_VECTOR);
  dim3 grid(kBatchPartBlocks, static_cast<unsigned>(h->groups));
  bdot_kernel<<<grid, 256, 0, h->stream>>>(static_cast<int32_t>(h->n), u, v, h->d_partials);
  ST_TRY(check_launch(h, "bdot_kernel"));
  bfinish_kernel<<<h->groups, 32, 0, h->stream>>>(1, h->padded, h->d_partials, scal(h, slot));
  return check_launch(h, "bfinish_kernel");
}

b200lu_status launch_spmv(H* h, const double* x, double* y) {
  PhaseScope ps(h, B200LU_PHASE_SPMV);
  bspmv_kernel<<<warp_blocks(h), 256, 0, h->stream>>>(static_cast<int32_t>(h->n), h->groups, h->nnz_source, h->d_a_row_ptr,
                                                      h->d_a_col, h->d_a_int, x, y);
  return check_launch(h, "bspmv_kernel");
}

b200lu_status copy_dd(H* h, double* dst, const double* src) {
  if (dst == src || h->n == 0) return B200LU_OK;
  CU_TRY(h, cudaMemcpyAsync(dst, src, static_cast<size_t>(vec_elems(h)) * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
  return B200LU_OK;
}

enum { kSlotRes = 0, kSlotBn = 1, kSlotNorm = 2, kSlotH = 3, kSlotCoef = 8 };

// fgmres_refine (src/refine.cpp:39-142) for every scenario in lockstep. Each scenario follows
// the reference's control flow on its own scalars (early exit, breakdown, candidate only when
// the estimate clears accept_below or on the last iteration, true residual, best-iterate rule);
// a scenario that has finished keeps its best iterate and rides along with neutral scalars.
b200lu_status fgmres_batch(H* h, const double* b, const double* x0, int use_precond, const b200lu_refine_config& cfg,
                           b200lu_refine_outcome* out) {
  const int64_t ne = vec_elems(h);
  const int32_t n32 = static_cast<int32_t>(h->n);
  const int32_t B = h->batch;
  const int m = std::max(1, cfg.max_iterations);
  const int wb = warp_blocks(h);
  for (int32_t s = 0; s < B; ++s) {
    out[s].iterations = 0;
    out[s].converged = 0;
    out[s].history_len = 0;
  }
  ST_TRY(copy_dd(h, h->d_best, x0));
  if (h->n == 0) {
    for (int32_t s = 0; s < B; ++s) {
      out[s].residual_history[out[s].history_len++] = 0.0;
      out[s].converged = 1;
    }
    return B200LU_OK;
  }
  ST_TRY(launch_residual(h, x0, b, h->d_r, kSlotRes));
  ST_TRY(read_scalars(h, kSlotRes, 2));
  std::vector<double> bnorm(B), beta(B), best_res(B), accept_below(B);
  std::vector<uint8_t> active(B, 1);
  int n_active = 0;
  for (int32_t s = 0; s < B; ++s) {
    const double bn = std::sqrt(hscal(h, kSlotBn)[s]);
    bnorm[s] = bn > 0.0 ? bn : 1.0;
    beta[s] = std::sqrt(hscal(h, kSlotRes)[s]);
    best_res[s] = beta[s] / bnorm[s];
    out[s].residual_history[out[s].history_len++] = best_res[s];
    accept_below[s] = cfg.tolerance * bnorm[s];
    if (best_res[s] <= cfg.tolerance) {
      out[s].converged = 1;
      active[s] = 0;
    }
    n_active += active[s];
  }
  if (n_active == 0) return B200LU_OK;

  auto V = [&](int j) { return h->d_V + static_cast<size_t>(j) * ne; };
  auto Z = [&](int j) { return h->d_Z + static_cast<size_t>(j) * ne; };
  std::vector<double> tmp(B);
  const double* dev = nullptr;
  for (int32_t s = 0; s < B; ++s) tmp[s] = active[s] ? beta[s] : 1.0;
  ST_TRY(upload_scalars(h, tmp, &dev));
  {
    PhaseScope ps(h, B200LU_PHASE_VECTOR);
    bdivide_kernel<<<wb, 256, 0, h->stream>>>(n32, h->groups, dev, h->d_r, V(0));
  }
  ST_TRY(check_launch(h, "bdivide_kernel"));
  int nV = 1;

  std::vector<std::vector<std::vector<double>>> Hm(B);  // per scenario: columns after rotations
  std::vector<std::vector<double>> g(B, std::vector<double>(static_cast<size_t>(m) + 1, 0.0)),
      cs(B, std::vector<double>(m, 0.0)), sn(B, std::vector<double>(m, 0.0));
  for (int32_t s = 0; s < B; ++s) g[s][0] = beta[s];

  for (int i = 0; i < m && n_active > 0; ++i) {
    if (use_precond) {
      ST_TRY(solve_int(h, V(i), Z(i)));
    } else {
      ST_TRY(copy_dd(h, Z(i), V(i)));
    }
    ST_TRY(launch_spmv(h, Z(i), h->d_wv));
    // cgs2_orthonormalize(V, w), src/refine.cpp:8-26
    CU_TRY(h, cudaMemsetAsync(scal(h, kSlotCoef), 0, static_cast<size_t>(nV) * h->padded * sizeof(double), h->stream));
    for (int pass = 0; pass < 2; ++pass) {
      for (int j = 0; j < nV; ++j) {
        ST_TRY(launch_dot(h, V(j), h->d_wv, kSlotH));
        {
          PhaseScope ps(h, B200LU_PHASE_VECTOR);
          bproject_out_kernel<<<wb, 256, 0, h->stream>>>(n32, h->groups, scal(h, kSlotH), scal(h, kSlotCoef + j), V(j),
                                                         h->d_wv);
        }
        ST_TRY(check_launch(h, "bproject_out_kernel"));
      }
    }
    ST_TRY(launch_dot(h, h->d_wv, h->d_wv, kSlotNorm));
    ST_TRY(read_scalars(h, kSlotNorm, kSlotCoef + nV - kSlotNorm));

    std::vector<uint8_t> breakdown(B, 0), need_cand(B, 0), last(B, 0);
    std::vector<double> estimate(B, 0.0);
    bool any_new_v = false, any_cand = false;
    for (int32_t s = 0; s < B; ++s) {
      tmp[s] = 1.0;
      if (!active[s]) continue;
      const double norm = std::sqrt(hscal(h, kSlotNorm)[s]);
      breakdown[s] = norm <= 1e-300;
      std::vector<double> hcol(nV);
      for (int j = 0; j < nV; ++j) hcol[j] = hscal(h, kSlotCoef + j)[s];
      hcol.push_back(breakdown[s] ? 0.0 : norm);
      if (!breakdown[s]) {
        tmp[s] = norm;
        any_new_v = true;
      }
      // Givens update, src/refine.cpp:89-107
      for (int k = 0; k < i; ++k) {
        const double t = hcol[k];
        hcol[k] = cs[s][k] * t + sn[s][k] * hcol[k + 1];
        hcol[k + 1] = -sn[s][k] * t + cs[s][k] * hcol[k + 1];
      }
      const double hii = hcol[i], hsub = hcol[i + 1];
      const double gam = std::hypot(hii, hsub);
      if (gam == 0.0) {
        cs[s][i] = 1.0;
        sn[s][i] = 0.0;
      } else {
        cs[s][i] = hii / gam;
        sn[s][i] = hsub / gam;
      }
      hcol[i] = gam;
      hcol[i + 1] = 0.0;
      const double gi = g[s][i];
      g[s][i] = cs[s][i] * gi;
      g[s][i + 1] = -sn[s][i] * gi;
      Hm[s].push_back(std::move(hcol));
      out[s].iterations = i + 1;
      estimate[s] = std::fabs(g[s][i + 1]);
      out[s].residual_history[out[s].history_len++] = estimate[s] / bnorm[s];
      last[s] = breakdown[s] || i == m - 1;
      need_cand[s] = estimate[s] <= accept_below[s] || last[s];
      any_cand = any_cand || need_cand[s];
    }
    if (any_new_v) {  // V(nV) = w / norm for the scenarios that continue
      ST_TRY(upload_scalars(h, tmp, &dev));
      {
        PhaseScope ps(h, B200LU_PHASE_VECTOR);
        bdivide_kernel<<<wb, 256, 0, h->stream>>>(n32, h->groups, dev, h->d_wv, V(nV));
      }
      ST_TRY(check_launch(h, "bdivide_kernel"));
    }
    if (any_cand) {
      // src/refine.cpp:115-139: minimum-residual iterate, true residual, best-iterate rule
      const int its = i + 1;
      std::vector<std::vector<double>> y(its, std::vector<double>(B, 0.0));
      for (int32_t s = 0; s < B; ++s) {
        if (!need_cand[s]) continue;
        std::vector<double> ys(its);
        for (int row = its - 1; row >= 0; --row) {
          double t = g[s][row];
          for (int col = row + 1; col < its; ++col) t -= Hm[s][col][row] * ys[col];
          ys[row] = t / Hm[s][row][row];
        }
        for (int col = 0; col < its; ++col) y[col][s] = ys[col];
      }
      ST_TRY(copy_dd(h, h->d_cand, x0));
      for (int col = 0; col < its; ++col) {
        ST_TRY(upload_scalars(h, y[col], &dev));
        {
          PhaseScope ps(h, B200LU_PHASE_VECTOR);
          baxpy_kernel<<<wb, 256, 0, h->stream>>>(n32, h->groups, dev, Z(col), h->d_cand);
        }
        ST_TRY(check_launch(h, "baxpy_kernel"));
      }
      ST_TRY(launch_residual(h, h->d_cand, b, h->d_r, kSlotRes));
      ST_TRY(read_scalars(h, kSlotRes, 1));
      bool any_copy = false;
      for (int32_t s = 0; s < B; ++s) {
        tmp[s] = 0.0;
        if (!need_cand[s]) continue;
        const double res = std::sqrt(hscal(h, kSlotRes)[s]) / bnorm[s];
        if (res < best_res[s]) {
          best_res[s] = res;
          tmp[s] = 1.0;
          any_copy = true;
        }
        if (best_res[s] <= cfg.tolerance) {
          out[s].converged = 1;
          active[s] = 0;
        } else if (last[s]) {
          active[s] = 0;
        } else {
          accept_below[s] = estimate[s] * 0.5;
        }
      }
      if (any_copy) {
        ST_TRY(upload_scalars(h, tmp, &dev));
        {
          PhaseScope ps(h, B200LU_PHASE_VECTOR);
          bcopy_masked_kernel<<<wb, 256, 0, h->stream>>>(n32, h->groups, dev, h->d_cand, h->d_best);
        }
        ST_TRY(check_launch(h, "bcopy_masked_kernel"));
      }
    }
    if (any_new_v) ++nV;
    n_active = 0;
    for (int32_t s = 0; s < B; ++s) n_active += active[s];
  }
  return B200LU_OK;
}

// classic_refine (src/refine.cpp:150-188) for every scenario in lockstep: x += M^-1 (b - A x), the
// best iterate is kept per scenario; a scenario that has converged stops updating (its correction
// is scaled by 0) and rides along.
b200lu_status classic_batch(H* h, const double* b, const double* x0, int use_precond, const b200lu_refine_config& cfg,
                            b200lu_refine_outcome* out) {
  const int32_t n32 = static_cast<int32_t>(h->n);
  const int32_t B = h->batch;
  const int wb = warp_blocks(h);
  for (int32_t s = 0; s < B; ++s) {
    out[s].iterations = 0;
    out[s].converged = 0;
    out[s].history_len = 0;
  }
  ST_TRY(copy_dd(h, h->d_best, x0));
  if (h->n == 0) {
    for (int32_t s = 0; s < B; ++s) {
      out[s].residual_history[out[s].history_len++] = 0.0;
      out[s].converged = 1;
    }
    return B200LU_OK;
  }
  ST_TRY(launch_residual(h, x0, b, h->d_r, kSlotRes));
  ST_TRY(read_scalars(h, kSlotRes, 2));
  std::vector<double> bnorm(B), best_res(B), tmp(B);
  std::vector<uint8_t> active(B, 1);
  int n_active = 0;
  for (int32_t s = 0; s < B; ++s) {
    const double bn = std::sqrt(hscal(h, kSlotBn)[s]);
    bnorm[s] = bn > 0.0 ? bn : 1.0;
    best_res[s] = std::sqrt(hscal(h, kSlotRes)[s]) / bnorm[s];
    out[s].residual_history[out[s].history_len++] = best_res[s];
    if (best_res[s] <= cfg.tolerance) {
      out[s].converged = 1;
      active[s] = 0;
    }
    n_active += active[s];
  }
  double* x = h->d_cand;
  ST_TRY(copy_dd(h, x, x0));
  const double* dev = nullptr;
  for (int it = 0; it < cfg.max_iterations && n_active > 0; ++it) {
    // d_r holds b - A x for the current x (from the initial residual, then from the end of the previous pass)
    if (use_precond) {
      ST_TRY(solve_int(h, h->d_r, h->d_wv));
    } else {
      ST_TRY(copy_dd(h, h->d_wv, h->d_r));
    }
    for (int32_t s = 0; s < B; ++s) tmp[s] = active[s] ? 1.0 : 0.0;
    ST_TRY(upload_scalars(h, tmp, &dev));
    {
      PhaseScope ps(h, B200LU_PHASE_VECTOR);
      baxpy_kernel<<<wb, 256, 0, h->stream>>>(n32, h->groups, dev, h->d_wv, x);  // axpy(1.0, d, x), src/refine.cpp:170
    }
    ST_TRY(check_launch(h, "baxpy_kernel"));
    ST_TRY(launch_residual(h, x, b, h->d_r, kSlotRes));
    ST_TRY(read_scalars(h, kSlotRes, 1));
    bool any_copy = false;
    for (int32_t s = 0; s < B; ++s) {
      tmp[s] = 0.0;
      if (!active[s]) continue;
      out[s].iterations = it + 1;
      const double res = std::sqrt(hscal(h, kSlotRes)[s]) / bnorm[s];
      out[s].residual_history[out[s].history_len++] = res;
      if (res < best_res[s]) {
        best_res[s] = res;
        tmp[s] = 1.0;
        any_copy = true;
      }
      if (best_res[s] <= cfg.tolerance) {
        out[s].converged = 1;
        active[s] = 0;
      }
    }
    if (any_copy) {
      ST_TRY(upload_scalars(h, tmp, &dev));
      {
        PhaseScope ps(h, B200LU_PHASE_VECTOR);
        bcopy_masked_kernel<<<wb, 256, 0, h->stream>>>(n32, h->groups, dev, x, h->d_best);
      }
      ST_TRY(check_launch(h, "bcopy_masked_kernel"));
    }
    n_active = 0;
    for (int32_t s = 0; s < B; ++s) n_active += active[s];
  }
  return B200LU_OK;
}

// ---- tiled trailing part (tile.cuh / tile_plan.hpp)

using TileFn = void (*)(BTileArgs);

// Builds the tile plan for the (ascending) trailing rows and uploads it. Leaves h->use_tiles false, with
// the reason in h->tile_note, when the pattern cannot be tiled.
b200lu_status setup_tiles(H* h, const std::vector<int32_t>& tail_rows) {
  const Schedule& S = h->sched;
  cudaDeviceProp prop;
  CU_TRY(h, cudaGetDeviceProperties(&prop, h->device));
  // B200LU_TILE_ROWS: rows (consumer warps) per tile, 8 (default) or 16; B200LU_TILE_CTAS: CTAs that share an
  // SM, 2 (default) or 3 (R = 8 only; the ring shrinks to 16 KB so that a 57 KB row still fits) — together
  // they fix the shared-memory budget of a tile. A pattern with a row that needs more gets the whole SM
  // for one CTA.
  const char* e = std::getenv("B200LU_TILE_ROWS");
  const int R = e && std::atoi(e) == 16 ? 16 : 8;
  e = std::getenv("B200LU_TILE_CTAS");
  int ctas = std::max(1, e ? std::atoi(e) : 2);
  if (R == 16) ctas = std::min(ctas, 2);
  ctas = std::min(ctas, 3);
  h->tile_ring_blocks = ctas == 3 ? 16 : 32;
  h->tile_ctas = ctas;
  const int64_t sm_bytes = static_cast<int64_t>(prop.sharedMemPerMultiprocessor);
  const int64_t max_block = static_cast<int64_t>(prop.sharedMemPerBlockOptin);
  const int64_t overhead = static_cast<int64_t>(tile_ring_bytes(h->tile_ring_blocks)) + kTileCtlBytes + 128;
  int64_t max_row = 0;
  for (int32_t i : tail_rows) max_row = std::max<int64_t>(max_row, S.row_ptr[i + 1] - S.row_ptr[i] + kTileSpare);  // + the spare entries
  const int64_t row_bytes = static_cast<int64_t>(kTileScen * sizeof(double));
  int64_t budget = std::min(max_block, sm_bytes / ctas - 1024) - overhead;  // 1 KB per CTA is reserved by the driver
  if (max_row * row_bytes > budget) {
    // The longest row needs more than a CTA's share of the SM: one CTA per SM. That halves the tiles in
    // flight and measured slower than the row-blocked kernel (C3, longest row 1 951 entries = 125 KB:
    // 27.0 ms against 23.1 ms at 32 scenarios, 46.9 against 33.7 at 64): only when asked for.
    if (h->tile_auto) {
      h->tile_note = "the longest trailing row (" + std::to_string(max_row) + " entries) leaves room for one tile CTA per SM only";
      return B200LU_OK;
    }
    budget = max_block - overhead;
  }
  if (budget < max_row * row_bytes) {
    h->tile_note = "a trailing row of " + std::to_string(max_row) + " entries does not fit a tile";
    return B200LU_OK;
  }
  if (static_cast<int64_t>(h->groups) * h->nnz_factors >= (int64_t{1} << 31) - 4096) {
    h->tile_note = "groups x nnz(L+U) exceeds the tensor-map coordinate range";
    return B200LU_OK;
  }
  TilePlan plan;
  const std::string err = build_tile_plan(S, tail_rows, R, budget / row_bytes, plan, h->tile_ring_blocks);
  if (!err.empty()) {
    h->tile_note = err;
    return B200LU_OK;
  }
  h->tile_rows_per = R;
  h->n_tiles = static_cast<int32_t>(plan.tiles.size());
  h->tile_units = h->padded / kTileScen;
  h->tile_fetched_entries = plan.fetched_entries;
  h->tile_args.rows_smem_bytes = static_cast<int32_t>(plan.rows_smem_entries * row_bytes);
  h->tile_smem = static_cast<size_t>(h->tile_args.rows_smem_bytes + overhead);
  ST_TRY(dev_upload(h, &h->d_tile_meta, plan.tiles));
  ST_TRY(dev_upload(h, &h->d_tile_rows, plan.rows));
  ST_TRY(dev_upload(h, &h->d_tile_ext, plan.ext));
  ST_TRY(dev_upload(h, &h->d_tile_row_items, plan.row_items));
  ST_TRY(dev_upload(h, &h->d_tile_dest, plan.tdest));
  ST_TRY(dev_alloc(h, &h->d_tile_flags, static_cast<size_t>(h->n) * h->tile_units));
  CU_TRY(h, cudaMemsetAsync(h->d_tile_flags, 0, static_cast<size_t>(h->n) * h->tile_units * sizeof(int32_t), h->stream));
  h->use_tiles = true;
  return B200LU_OK;
}

// Tensor maps, kernel attributes and grid of the tiled launch (after d_values / d_dest exist).
b200lu_status finish_tiles(H* h, int sm_count) {
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                                const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult qres;
  CU_TRY(h, cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qres));
  if (!fn || qres != cudaDriverEntryPointSuccess) {
    h->last_error = "cuTensorMapEncodeTiled is not available from this driver";
    return B200LU_CUDA_ERROR;
  }
  BTileArgs& ta = h->tile_args;
  // values viewed as a 2-D tensor: [groups * nnz_factors] rows of 32 doubles; a box is 8 scenarios wide
  const cuuint64_t dims[2] = {32, static_cast<cuuint64_t>(h->groups) * static_cast<cuuint64_t>(h->nnz_factors)};
  const cuuint64_t strides[1] = {32 * sizeof(double)};
  const cuuint32_t estr[2] = {1, 1};
  for (int i = 0; i < kTileMaps; ++i) {
    const cuuint32_t box[2] = {kTileScen, static_cast<cuuint32_t>(kTileBoxStep * (i + 1))};
    const CUresult r = reinterpret_cast<EncodeFn>(fn)(&ta.maps[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, h->d_values, dims, strides, box,
                                                      estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      h->last_error = "cuTensorMapEncodeTiled failed with code " + std::to_string(static_cast<int>(r));
      return B200LU_CUDA_ERROR;
    }
  }
  ta.n_tiles = h->n_tiles;
  ta.units = h->tile_units;
  ta.gen = 0;
  ta.tiles = h->d_tile_meta;
  ta.rows = h->d_tile_rows;
  ta.ext = h->d_tile_ext;
  ta.row_items = h->d_tile_row_items;
  ta.tdest = reinterpret_cast<const uint4*>(h->d_tile_dest);
  ta.values = h->d_values;
  ta.nnz_factors = h->nnz_factors;
  ta.flags = h->d_tile_flags;
  ta.pivot_floor = h->pivot_floor;
  ta.failed = h->d_failed;
  ta.ticket = h->d_tickets + 1;
  ST_TRY(dev_alloc(h, &h->d_tile_prof, 16));
  CU_TRY(h, cudaMemsetAsync(h->d_tile_prof, 0, 16 * sizeof(long long), h->stream));
  ta.prof = h->d_tile_prof;
  const int variant = h->tile_rows_per == 16 ? 1 : h->tile_ctas == 3 ? 2 : 0;
  h->tile_fn = variant == 1 ? bfactor_tile_kernel<16, 32, 2> : variant == 2 ? bfactor_tile_kernel<8, 16, 3> : bfactor_tile_kernel<8, 32, 2>;
  // per function, process-wide: never lowered under a live handle (the largest request so far stays)
  static size_t attr_set[3] = {0, 0, 0};
  size_t& cur = attr_set[variant];
  if (h->tile_smem > cur) {
    CU_TRY(h, cudaFuncSetAttribute(h->tile_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(h->tile_smem)));
    cur = h->tile_smem;
  }
  int occ = 0;
  CU_TRY(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, h->tile_fn, (h->tile_rows_per + 1) * 32, h->tile_smem));
  if (occ < 1) {
    h->last_error = "tiled factor kernel does not fit on an SM";
    return B200LU_CUDA_ERROR;
  }
  h->tile_grid = sm_count * occ;
  return B200LU_OK;
}

}  // namespace

// ===================================================================== C ABI

extern "C" {

const char* b200lu_batch_last_error(const b200lu_batch* h) { return h ? h->last_error.c_str() : ""; }

b200lu_status b200lu_batch_create(const b200lu_symbolic_view* sym, const b200lu_options* opt_in, int64_t batch,
                                  b200lu_batch** out) {
  if (!sym || !out || batch < 1 || batch > (1 << 20)) return B200LU_INVALID_ARGUMENT;
  *out = nullptr;
  b200lu_options opt;
  b200lu_default_options(&opt);
  if (opt_in) opt = *opt_in;
  if (b200lu_device_count() <= opt.device) return B200LU_NO_DEVICE;
  H* h = new H;
  *out = h;
  h->device = opt.device;
  h->pivot_floor = opt.pivot_floor;
  h->refine_capacity = opt.refine_capacity > 0 ? std::min(opt.refine_capacity, 64) : 20;
  h->batch = static_cast<int32_t>(batch);
  h->groups = (h->batch + 31) / 32;
  h->padded = h->groups * 32;
  h->valid.assign(batch, 0);
  CU_TRY(h, cudaSetDevice(h->device));
  if (opt.stream) {
    h->stream = static_cast<cudaStream_t>(opt.stream);
  } else {
    CU_TRY(h, cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    h->owns_stream = true;
  }
  ScheduleTuning tune;
  tune.tail_min_levels = int64_t{1} << 40;  // no on-chip tail split: the batched sweeps run whole
  const std::string err = build_schedule(*sym, tune, h->sched);
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

  // Refactorization unit: 32 scenarios per warp, lane = scenario (E = 1). Narrower units (two or four
  // entry lanes per scenario) are faster by ~10 % but NOT safe with reduction updates: the reductions
  // and loads that different lanes of a warp issue to one address are not kept in order by the
  // hardware (found with the B200LU_POLL_ATOMIC stress build), so all operations on a
  // value must come from one thread.
  h->unit = 32;
  h->units = h->padded / h->unit;

  ST_TRY(dev_upload(h, &h->d_row_ptr, S.row_ptr));
  ST_TRY(dev_upload(h, &h->d_col, S.col));
  ST_TRY(dev_upload(h, &h->d_diag, S.diag));
  ST_TRY(dev_upload(h, &h->d_trivial_rows, S.trivial_rows));
  ST_TRY(dev_upload(h, &h->d_pair_row_ptr, S.pair_row_ptr));
  ST_TRY(dev_upload(h, &h->d_lower_meta, S.lower_meta));
  ST_TRY(dev_upload(h, &h->d_upper_meta, S.upper_meta));
  {
    // Head / tail split of the refactorization. The maximal suffix of dependency levels narrower than
    // `tail_width` rows runs in a second launch; it is successor-closed, so the head launch has
    // finished every head pivot before it starts. Below the first few dozen levels the elimination DAG
    // consists of chains of index-consecutive rows in which every row is a pivot of the next and
    // shares almost all of its other pivots with it (at C2 the levels narrower than 1024 rows hold
    // 99.5 % of the update pairs).
    //   B200LU_BATCH_TAIL_MODE=1 (default): bfactor_block_kernel, kBlockRows consecutive rows per warp
    //           sharing each loaded pivot row. Measured at C2 x 256, factor phase: 2-row blocks 25.8 ms
    //           against 28.9 ms unsplit (tail_width 512..4096 alike; 27 ms with every row in a block);
    //           4-row blocks cut the DRAM traffic of the trailing part 4x but run at 16 warps per SM and
    //           wait on chain hand-offs: 32-34 ms.
    //   B200LU_BATCH_TAIL_MODE=0: the row-by-row kernel instantiated for latency (24 loads per lane in
    //           flight, 16 warps per SM): 34-37 ms.
    //   B200LU_BATCH_TAIL_WIDTH=0: no split.
    const char* e = std::getenv("B200LU_BATCH_TAIL_WIDTH");
    const int64_t tail_width = e ? std::atoll(e) : 1024;
    e = std::getenv("B200LU_BATCH_TAIL_MODE");
    const int tail_mode = e ? std::atoi(e) : 1;
    const int64_t cut = trailing_cut_level(S, tail_width);
    std::vector<FactorMeta> meta;
    meta.reserve(n);
    std::vector<int32_t> tail_rows;
    for (int32_t i : S.lower_order) {  // dependency-level order; rows without pivots are final after the scatter
      if (S.diag[i] == S.row_ptr[i]) continue;
      if (S.lower_level[i] >= cut) {
        tail_rows.push_back(i);
      } else {
        meta.push_back(FactorMeta{i, S.row_ptr[i], S.diag[i], S.row_ptr[i + 1]});
      }
    }
    h->n_factor_rows = static_cast<int32_t>(meta.size());
    ST_TRY(dev_upload(h, &h->d_factor_meta, meta));
    if (tail_mode == 0) {  // tail rows in level order through the latency-optimised row kernel
      std::vector<FactorMeta> tmeta;
      for (int32_t i : tail_rows) tmeta.push_back(FactorMeta{i, S.row_ptr[i], S.diag[i], S.row_ptr[i + 1]});
      h->n_tail_rows = static_cast<int32_t>(tmeta.size());
      ST_TRY(dev_upload(h, &h->d_tail_meta, tmeta));
      h->n_block_rows = h->n_tail_rows;
      for (int32_t i : tail_rows) h->blocked_pairs += S.pair_row_ptr[i + 1] - S.pair_row_ptr[i];
      tail_rows.clear();
    }
    std::sort(tail_rows.begin(), tail_rows.end());
    // The trailing part runs in one of two kernels:
    //   * bfactor_tile_kernel (tile.cuh): CTA tiles of 8 rows x 8 scenarios resident in shared memory, pivot
    //     rows staged once per tile by TMA, plain ordered read-modify-write updates. 3x less DRAM traffic and
    //     no L2 reductions, and a dependency hand-off of ~1 us per level instead of ~8 us: the faster kernel
    //     while the batch is LATENCY-bound. Measured, factor phase at C2: 32 scenarios 4.9 ms against 8.2 ms,
    //     64: 8.1 against 9.7, 128: 14.9 against 14.1, 256: 27.6 against 24.4 (its per-(row, pivot) costs are
    //     paid per 8 scenarios, the row-blocked kernel's per 32).
    //   * bfactor_block_kernel (batch.cuh): 2-row blocks x 32 scenarios, updates as L2 reductions: the faster
    //     one once the batch is THROUGHPUT-bound.
    // B200LU_BATCH_TILES = 1 / 0 forces one of them; default: tiles up to 32 scenarios per handle (an 8-GPU
    // shard of the 256-scenario batch; up to 96 while the row-blocked kernel ran one warp per block), provided two tile CTAs fit on an SM (setup_tiles). A pattern / batch the tiled kernel cannot take (a row larger than
    // a tile, a pivot row longer than a staging copy, more than 2^31 entries per tensor-map dimension) keeps
    // the row-blocked kernel.
    e = std::getenv("B200LU_BATCH_TILES");
    const bool forced = e != nullptr;
    const bool want_tiles = forced ? std::atoi(e) != 0 : h->padded <= 32;  // against the one-warp-per-row kernel (factor phase, C2): 32 scenarios 4.85 / 5.82 ms, 64: 7.95 / 7.67, 96: 11.0 / 9.8, 128: 14.8 / 12.5
    h->tile_auto = !forced;
    // (Running both side by side — the tiled kernel on some of the scenarios, the row-blocked one on the rest, one
    // CTA of each per SM on two streams — was measured at C2 x 256: 35-46 ms against 24.4 ms for the row-blocked
    // kernel alone; dropped.)
    if (want_tiles && !tail_rows.empty() && tail_mode != 0) {
      ST_TRY(setup_tiles(h, tail_rows));
      if (h->use_tiles) {
        h->n_block_rows = static_cast<int32_t>(tail_rows.size());
        for (int32_t i : tail_rows) h->blocked_pairs += S.pair_row_ptr[i + 1] - S.pair_row_ptr[i];
        tail_rows.clear();
      }
    }
    //   * bfactor_gather_kernel (gather.cuh): R-row blocks x 32 scenarios; every target entry a batch of K pivots
    //     touches is loaded once, updated in a register and stored once: no L2 reductions at all.
    //     Bit-exact, and it does what it was built for — ncu at C2 x 256: L2 reductions 0, DRAM traffic 40 GB
    //     against 47 GB — but it LOSES: 85-105 ms against 24.4 ms for the row-blocked kernel (57 ms at 32 scenarios
    //     against 8.2 / 4.9 ms). The record interpreter costs 53 warp instructions per record (two index words,
    //     a type switch the compiler cannot prove warp-uniform, 64-bit address arithmetic: 14.5 G instructions per
    //     refactorization against 5.7 G), and the trailing DAG is narrow (16 439 rows in 925 levels): the time
    //     is levels x (latency of one warp walking one batch), and a batch's loads are only one chunk deep.
    //     Without the flag waits (timing experiment B200LU_GATHER_NOWAIT, wrong results) it still takes 50 ms.
    //     Kept as an experiment, OFF by default.
    // B200LU_BATCH_GATHER = 1 selects it (with B200LU_BATCH_TILES = 0 for small batches);
    // B200LU_GATHER_R (1, 2, 4), B200LU_GATHER_K (8, 16, 32), B200LU_GATHER_SMALL (pivots of the last, short batch).
    e = std::getenv("B200LU_BATCH_GATHER");
    const bool want_gather = e ? std::atoi(e) != 0 : false;
    if (want_gather && !tail_rows.empty() && tail_mode != 0) {
      e = std::getenv("B200LU_GATHER_R");
      const int gr = e ? std::atoi(e) : 2;
      e = std::getenv("B200LU_GATHER_K");
      const int gk = e ? std::atoi(e) : 16;
      e = std::getenv("B200LU_GATHER_SMALL");
      const int gs = e ? std::atoi(e) : 2;
      GatherPlan plan;
      std::string err;
      int gr_used = gr, gk_used = gk;
      if (!build_gather_plan(S.row_ptr, S.col, S.diag, S.lower_level, tail_rows, gr, gk, gs, &plan, &err)) {
        // blocks of several rows can depend on each other both ways when the trailing rows are not
        // index-consecutive; single-row blocks cannot
        gr_used = 1;
        gk_used = 32;
        if (!build_gather_plan(S.row_ptr, S.col, S.diag, S.lower_level, tail_rows, gr_used, gk_used, gs, &plan, &err)) {
          h->last_error = err;
          return B200LU_INVALID_ARGUMENT;
        }
      }
      ST_TRY(dev_upload(h, &h->d_g_blocks, plan.blocks));
      ST_TRY(dev_upload(h, &h->d_g_batches, plan.batches));
      ST_TRY(dev_upload(h, &h->d_g_recs, plan.recs));
      ST_TRY(dev_upload(h, &h->d_g_waits, plan.waits));
      h->use_gather = true;
      h->n_g_blocks = static_cast<int32_t>(plan.blocks.size());
      h->gather_rows_per = gr_used;
      h->gather_batch = gk_used;
      h->gather_records = static_cast<int64_t>(plan.recs.size());
      h->gather_targets = plan.n_targets;
      if (std::getenv("B200LU_GATHER_VERBOSE")) {
        std::fprintf(stderr, "gather plan: R %d K %d rows %lld blocks %zu batches %zu records %zu (init %lld upd %lld div %lld pub %lld pad %lld) targets %lld waits %zu\n",
                     gr_used, gk_used, static_cast<long long>(plan.rows), plan.blocks.size(), plan.batches.size(), plan.recs.size(),
                     static_cast<long long>(plan.n_init), static_cast<long long>(plan.n_upd), static_cast<long long>(plan.n_div),
                     static_cast<long long>(plan.n_pub), static_cast<long long>(plan.n_pad), static_cast<long long>(plan.n_targets), plan.waits.size());
      }
      h->n_block_rows = static_cast<int32_t>(tail_rows.size());
      for (int32_t i : tail_rows) h->blocked_pairs += S.pair_row_ptr[i + 1] - S.pair_row_ptr[i];
      tail_rows.clear();
    }
    //   * bfactor_snode_kernel (snode.cuh): 2-row blocks x 32 scenarios over RUNS of up to 8 consecutive pivot rows with
    //     nested upper patterns (fundamental supernodes: 80 % of the update pairs at C2 sit in runs of >= 8 rows):
    //     multipliers in registers, every destination entry loaded / stored once per run, no per-update index.
    //     Bit-exact and free of L2 reductions, but it LOSES on this DAG: 58 ms (46 ms with single-row blocks) against
    //     24.4 ms at C2 x 256, 33 / 19 ms against 8.2 (4.9 tiled) at 32 scenarios. ncu: the warps sit in the flag
    //     waits — the trailing DAG is ~18 rows wide over 925 levels, a level costs what ONE warp needs to apply the
    //     row's last pivots, and here that is ~15 dependent memory round trips (run record, diagonal slots, flag,
    //     phase A per pivot, destination slots, phase B a few entries at a time, pivot check, fence) against ~4 for
    //     the row-blocked kernel, whose reductions need no round trip for the destination at all. What it would take:
    //     records / slots / destination values prefetched while the flag is awaited, the pivot rows streamed through a
    //     shared-memory ring, L2 reductions for the single-pivot runs at the end of a row. Kept as an experiment, OFF.
    // B200LU_BATCH_SNODE = 1 selects it; B200LU_SNODE_R (1, 2), B200LU_SNODE_SMALL: length of the shortest (last) runs.
    e = std::getenv("B200LU_BATCH_SNODE");
    const bool want_snode = e ? std::atoi(e) != 0 : false;
    if (want_snode && !tail_rows.empty() && tail_mode != 0) {
      e = std::getenv("B200LU_SNODE_SMALL");
      const int ss = e ? std::atoi(e) : 1;
      e = std::getenv("B200LU_SNODE_R");
      int sr = e ? std::atoi(e) : 2;
      SnodePlan plan;
      std::string err;
      if (!build_snode_plan(S.row_ptr, S.col, S.diag, S.lower_level, tail_rows, sr, ss, &plan, &err)) {
        sr = 1;  // single-row blocks cannot depend on each other both ways
        if (!build_snode_plan(S.row_ptr, S.col, S.diag, S.lower_level, tail_rows, sr, ss, &plan, &err)) {
          h->last_error = err;
          return B200LU_INVALID_ARGUMENT;
        }
      }
      ST_TRY(dev_upload(h, &h->d_s_blocks, plan.blocks));
      ST_TRY(dev_upload(h, &h->d_s_runs, plan.runs));
      ST_TRY(dev_upload(h, &h->d_s_dest, plan.dest));
      h->use_snode = true;
      h->n_s_blocks = static_cast<int32_t>(plan.blocks.size());
      h->snode_rows_per = sr;
      if (std::getenv("B200LU_GATHER_VERBOSE")) {
        std::fprintf(stderr, "snode plan: R %d rows %lld blocks %zu runs %zu pivots %lld (%.2f per run) pairs %lld (in runs >= 4: %.3f) dest entries %zu\n",
                     sr, static_cast<long long>(plan.rows), plan.blocks.size(), plan.runs.size(), static_cast<long long>(plan.pivots),
                     plan.runs.empty() ? 0.0 : static_cast<double>(plan.pivots) / plan.runs.size(), static_cast<long long>(plan.pairs),
                     plan.pairs ? static_cast<double>(plan.pairs_in_runs_of_4) / plan.pairs : 0.0, plan.dest.size());
      }
      h->n_block_rows = static_cast<int32_t>(tail_rows.size());
      for (int32_t i : tail_rows) h->blocked_pairs += S.pair_row_ptr[i + 1] - S.pair_row_ptr[i];
      tail_rows.clear();
    }
    std::vector<BlockMeta> blocks;
    std::vector<MergedPivot> merged;
    for (size_t b0 = 0; b0 < tail_rows.size(); b0 += kBlockRows) {
      BlockMeta bm;
      const int rows_here = static_cast<int>(std::min<size_t>(kBlockRows, tail_rows.size() - b0));
      std::vector<std::pair<int32_t, int>> piv;  // (pivot row, block row)
      for (int r = 0; r < 4; ++r) bm.row[r] = -1;
      for (int r = 0; r < kBlockRows; ++r) {
        bm.row[r] = r < rows_here ? tail_rows[b0 + r] : -1;
        if (r < rows_here) {
          const int32_t i = bm.row[r];
          for (int32_t k = S.row_ptr[i]; k < S.diag[i]; ++k) piv.emplace_back(S.col[k], r);
        }
      }
      std::sort(piv.begin(), piv.end());
      bm.mbeg = static_cast<int32_t>(merged.size());
      int last_of_row[kBlockRows];
      for (int r = 0; r < kBlockRows; ++r) last_of_row[r] = -1;
      for (size_t q = 0; q < piv.size(); ++q) {
        if (q == 0 || piv[q].first != piv[q - 1].first) merged.push_back(MergedPivot{piv[q].first, 0u});
        merged.back().bits |= 1u << piv[q].second;
        last_of_row[piv[q].second] = static_cast<int>(merged.size()) - 1;
      }
      for (int r = 0; r < rows_here; ++r) merged[last_of_row[r]].bits |= 256u << r;
      for (int32_t t = bm.mbeg; t < static_cast<int32_t>(merged.size()); ++t) {
        for (int r = 0; r < rows_here; ++r) {
          if (merged[t].d == bm.row[r]) merged[t].bits |= 0x10000u;  // a pivot that is a row of this block
        }
      }
      bm.mend = static_cast<int32_t>(merged.size());
      bm.pad0 = bm.pad1 = 0;
      blocks.push_back(bm);
    }
    if (!blocks.empty()) {
      // Claim order of the blocks. Index order is topological (a trailing row only depends on rows of
      // smaller index) but walks ONE chain at a time — consecutive indices are one chain — so the
      // resident warps would all sit on the same sequential chain. Level order interleaves the chains
      // but is not topological for blocks (a block spans several levels). Hence: Kahn's algorithm on
      // the block DAG with the ready blocks taken by (level of first row, index).
      const size_t nb = blocks.size();
      std::vector<int32_t> block_of(n, -1);
      for (size_t b = 0; b < nb; ++b) {
        for (int r = 0; r < kBlockRows; ++r) {
          if (blocks[b].row[r] >= 0) block_of[blocks[b].row[r]] = static_cast<int32_t>(b);
        }
      }
      std::vector<std::vector<int32_t>> succ(nb);
      std::vector<int32_t> indeg(nb, 0);
      for (size_t b = 0; b < nb; ++b) {
        int32_t last = -1;  // merged pivots ascend, so the blocks they belong to ascend too
        for (int32_t t = blocks[b].mbeg; t < blocks[b].mend; ++t) {
          const int32_t pb = block_of[merged[t].d];
          if (pb >= 0 && pb != static_cast<int32_t>(b) && pb != last) {
            succ[pb].push_back(static_cast<int32_t>(b));
            ++indeg[b];
            last = pb;
          }
        }
      }
      using Key = std::pair<int32_t, int32_t>;  // (level of first row, block id), smallest first
      std::priority_queue<Key, std::vector<Key>, std::greater<Key>> ready;
      for (size_t b = 0; b < nb; ++b) {
        if (indeg[b] == 0) ready.emplace(S.lower_level[blocks[b].row[0]], static_cast<int32_t>(b));
      }
      std::vector<BlockMeta> ordered;
      ordered.reserve(nb);
      while (!ready.empty()) {
        const int32_t b = ready.top().second;
        ready.pop();
        ordered.push_back(blocks[b]);
        for (int32_t c : succ[b]) {
          if (--indeg[c] == 0) ready.emplace(S.lower_level[blocks[c].row[0]], c);
        }
      }
      if (ordered.size() != nb) {
        h->last_error = "row-block dependency graph is not acyclic";
        return B200LU_INVALID_ARGUMENT;
      }
      blocks.swap(ordered);
    }
    h->n_blocks = static_cast<int32_t>(blocks.size());
    if (!tail_rows.empty()) {
      h->n_block_rows = static_cast<int32_t>(tail_rows.size());
      for (int32_t i : tail_rows) h->blocked_pairs += S.pair_row_ptr[i + 1] - S.pair_row_ptr[i];
    }
    ST_TRY(dev_upload(h, &h->d_blocks, blocks));
    ST_TRY(dev_upload(h, &h->d_merged, merged));
  }
  {
    std::vector<int32_t> src_of_slot(nnzF, -1);
    for (int64_t k = 0; k < nnzA; ++k) {
      const int64_t s = sym->scatter_map[k];
      if (s < 0 || s >= nnzF || src_of_slot[s] != -1) {
        h->last_error = "scatter_map is not an injection into the combined pattern";
        return B200LU_INVALID_ARGUMENT;
      }
      src_of_slot[s] = static_cast<int32_t>(k);
    }
    ST_TRY(dev_upload(h, &h->d_src_of_slot, src_of_slot));
    bool need_scale = h->has_match;
    for (int64_t k = 0; k < nnzA && !need_scale; ++k) need_scale = sym->scatter_scale[k] != 1.0;
    if (need_scale) {  // off the matching path every scale is exactly 1.0 (src/symbolic.cpp:187): skipped
      ST_TRY(dev_upload(h, &h->d_scatter_scale, std::vector<double>(sym->scatter_scale, sym->scatter_scale + nnzA)));
    }
  }
  {
    std::vector<int32_t> p(n), pq(n);
    for (int64_t i = 0; i < n; ++i) p[i] = static_cast<int32_t>(sym->amd_forward[i]);
    for (int64_t j = 0; j < n; ++j) pq[j] = h->has_match ? p[sym->col_perm_forward[j]] : p[j];
    ST_TRY(dev_upload(h, &h->d_p, p));
    ST_TRY(dev_upload(h, &h->d_pq, pq));
    if (h->has_match) {
      ST_TRY(dev_upload(h, &h->d_row_scale, std::vector<double>(sym->row_scale, sym->row_scale + n)));
      ST_TRY(dev_upload(h, &h->d_col_scale, std::vector<double>(sym->col_scale, sym->col_scale + n)));
    }
  }
  {
    std::vector<int32_t> arp(n + 1), ac(nnzA);
    for (int64_t i = 0; i <= n; ++i) arp[i] = static_cast<int32_t>(sym->source_row_offsets[i]);
    for (int64_t k = 0; k < nnzA; ++k) ac[k] = static_cast<int32_t>(sym->source_col_indices[k]);
    ST_TRY(dev_upload(h, &h->d_a_row_ptr, arp));
    ST_TRY(dev_upload(h, &h->d_a_col, ac));
  }
  const size_t P = static_cast<size_t>(h->padded);
  ST_TRY(dev_alloc(h, &h->d_a_int, static_cast<size_t>(nnzA) * P));
  ST_TRY(dev_alloc(h, &h->d_values, static_cast<size_t>(nnzF) * P));
  {
    std::vector<int32_t> flags(static_cast<size_t>(n) * h->units, 0);
    for (int32_t i : S.trivial_rows) {
      for (int32_t u = 0; u < h->units; ++u) flags[static_cast<size_t>(i) * h->units + u] = INT_MAX;
    }
    ST_TRY(dev_upload(h, &h->d_flags, flags));
  }
  ST_TRY(dev_alloc(h, &h->d_failed, 2 * P));
  ST_TRY(dev_alloc(h, &h->d_tickets, 4));
  ST_TRY(dev_alloc(h, &h->d_stage_a, static_cast<size_t>(nnzA) * h->batch));
  for (double** p : {&h->d_stage_in, &h->d_stage_in2, &h->d_stage_out}) ST_TRY(dev_alloc(h, p, static_cast<size_t>(n) * h->batch));
  ST_TRY(dev_alloc(h, &h->d_gather, static_cast<size_t>(std::max(nnzF, n))));
  for (double** p : {&h->d_w, &h->d_t1, &h->d_t2, &h->d_b, &h->d_x0, &h->d_x, &h->d_r, &h->d_wv, &h->d_cand, &h->d_best}) {
    ST_TRY(dev_alloc(h, p, static_cast<size_t>(n) * P));
  }
  ST_TRY(dev_alloc(h, &h->d_V, static_cast<size_t>(h->refine_capacity + 1) * std::max<size_t>(n * P, 1)));
  ST_TRY(dev_alloc(h, &h->d_Z, static_cast<size_t>(h->refine_capacity) * std::max<size_t>(n * P, 1)));
  const int scal_slots = kSlotCoef + h->refine_capacity + 2;
  ST_TRY(dev_alloc(h, &h->d_scal, static_cast<size_t>(std::max(scal_slots, kScalSlots)) * P));
  ST_TRY(dev_alloc(h, &h->d_up, static_cast<size_t>(kUpSlots) * P));
  ST_TRY(dev_alloc(h, &h->d_partials, static_cast<size_t>(h->groups) * 2 * kBatchParts * 32));
  CU_TRY(h, cudaMallocHost(reinterpret_cast<void**>(&h->h_scal), static_cast<size_t>(std::max(scal_slots, kScalSlots)) * P * sizeof(double)));
  CU_TRY(h, cudaMallocHost(reinterpret_cast<void**>(&h->h_up), static_cast<size_t>(kUpSlots) * P * sizeof(double)));
  CU_TRY(h, cudaMallocHost(reinterpret_cast<void**>(&h->h_failed), 2 * P * sizeof(int32_t)));

  // destinations are 16-bit offsets into the row unless a row has more than 65 535 entries; B200LU_BATCH_DEST32=1 forces
  // the 32-bit instantiations (test knob: no pattern of the configs comes near that row length)
  h->dest16 = S.max_row_len <= 65535 && !(std::getenv("B200LU_BATCH_DEST32") && std::atoi(std::getenv("B200LU_BATCH_DEST32")) == 1);
  ST_TRY(dev_alloc(h, reinterpret_cast<char**>(&h->d_dest), static_cast<size_t>(S.update_pairs) * (h->dest16 ? 2 : 4) + 256));  // slack: chunk copies read whole words
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

  // launch geometry: persistent grids sized to what is co-resident
  cudaDeviceProp prop;
  CU_TRY(h, cudaGetDeviceProperties(&prop, h->device));
  if (h->use_tiles) ST_TRY(finish_tiles(h, prop.multiProcessorCount));
  {
    using Fn = void (*)(BFactorArgs);
    // variant = (min CTAs per SM -> register cap, loads in flight per warp); B200LU_BATCH_VARIANT for experiments
    const char* ev = std::getenv("B200LU_BATCH_VARIANT");
    const int variant = ev ? std::atoi(ev) : 0;
#define B200LU_BF(T, S) \
  (variant == 1 ? bfactor_kernel<T, S, kBWarps, 6, 8, false> : variant == 2 ? bfactor_kernel<T, S, kBWarps, 6, 4, false> \
   : variant == 3 ? bfactor_kernel<T, S, kBWarps, 4, 16, false> : variant == 4 ? bfactor_kernel<T, S, kBWarps, 3, 8, true> \
   : variant == 5 ? bfactor_kernel<T, S, kBWarps, 4, 8, true> : variant == 6 ? bfactor_kernel<T, S, kBWarps, 4, 4, true> \
   : variant == 7 ? bfactor_kernel<T, S, kBWarps, 3, 16, false> : variant == 8 ? bfactor_kernel<T, S, kBWarps, 2, 32, false> \
   : bfactor_kernel<T, S, kBWarps, 4, 8, false>)
    Fn fn = h->dest16 ? B200LU_BF(uint16_t, 32) : B200LU_BF(uint32_t, 32);
#undef B200LU_BF
    h->factor_fn = fn;
    h->factor_smem = 0;
    CU_TRY(h, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(h->factor_smem)));
    int occ = 0;
    CU_TRY(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kBWarps * 32, h->factor_smem));
    if (occ < 1) {
      h->last_error = "batched factor kernel does not fit on an SM";
      return B200LU_CUDA_ERROR;
    }
    h->factor_grid = prop.multiProcessorCount * occ;
    {
      Fn tfn = h->dest16 ? bfactor_kernel<uint16_t, 32, kBWarps, 2, 24, false> : bfactor_kernel<uint32_t, 32, kBWarps, 2, 24, false>;
      h->tail_fn = tfn;
      int tocc = 0;
      CU_TRY(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&tocc, tfn, kBWarps * 32, 0));
      h->tail_grid = prop.multiProcessorCount * std::max(1, tocc);
    }
    using BFn = void (*)(BBlockArgs);
    BFn bfn = h->dest16 ? bfactor_block_kernel<uint16_t, 32> : bfactor_block_kernel<uint32_t, 32>;
    h->block_fn = bfn;
    h->block_smem = 8 * block_stage_doubles() * sizeof(double);
    if (h->block_smem > 0) {
      CU_TRY(h, cudaFuncSetAttribute(bfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(h->block_smem)));
    }
    int bocc = 0;
    CU_TRY(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bocc, bfn, 256, h->block_smem));
    h->block_grid = prop.multiProcessorCount * std::max(1, bocc);
    // experiment: fewer resident CTAs (a smaller working set in L2). Measured at C2 x 256, factor phase: 296 CTAs 24.3 ms,
    // 222: 26.7, 148: 29.9, 111: 36.1, 74: 49.9 (at 32 scenarios 8.2 / 8.3 / 8.4 / 9.1 / 10.9): residency pays, L2 locality does not.
    {
      // Default for the row-blocked trailing part since round 2: one warp per ROW of a block (blockteam.cuh), the pivot row
      // staged once per block. Measured at C2, factor phase: 22.3 ms against 24.4 ms at 256 scenarios, 5.9 ms against 8.2 ms
      // at 32. B200LU_BATCH_TEAM = 0 restores bfactor_block_kernel (one warp per block); 2 / 3 / 4 = minimum CTAs per SM.
      const char* et = std::getenv("B200LU_BATCH_TEAM");
      const int minb = et ? std::atoi(et) : 3;
      if (minb >= 1) {
        using TFn = void (*)(BBlockArgs);
        TFn tfn = h->dest16 ? (minb >= 4 ? bfactor_block_team_kernel<uint16_t, 4> : minb == 3 ? bfactor_block_team_kernel<uint16_t, 3> : bfactor_block_team_kernel<uint16_t, 2>)
                            : bfactor_block_team_kernel<uint32_t, 2>;
        h->team_smem = team_smem_bytes();
        // pivot rows staged by ONE bulk asynchronous copy per pivot (cp.async.bulk + mbarrier, blockteam.cuh) — the default;
        // B200LU_BATCH_TEAM_BULK=0 restores the per-lane 16-byte cp.async (22.0 against 22.3 ms at C2 x 256, equal at 32)
        const char* eb = std::getenv("B200LU_BATCH_TEAM_BULK");
        if (!eb || std::atoi(eb) != 0) {
          tfn = h->dest16 ? (minb >= 4 ? bfactor_block_team_kernel<uint16_t, 4, true> : minb == 3 ? bfactor_block_team_kernel<uint16_t, 3, true> : bfactor_block_team_kernel<uint16_t, 2, true>)
                          : bfactor_block_team_kernel<uint32_t, 2, true>;
        }
        if (const char* e2 = std::getenv("B200LU_BATCH_TEAM_STAGES")) {  // 2: double-buffered stage (blockteam.cuh)
          if (std::atoi(e2) == 2 && h->dest16) {
            tfn = minb >= 3 ? bfactor_block_team2_kernel<uint16_t, 3> : bfactor_block_team2_kernel<uint16_t, 2>;
            h->team_smem = team2_smem_bytes();
          }
        }
        h->team_fn = tfn;
        CU_TRY(h, cudaFuncSetAttribute(tfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(h->team_smem)));
        int tocc = 0;
        CU_TRY(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&tocc, tfn, kTeamWarps * 32, h->team_smem));
        h->team_grid = prop.multiProcessorCount * std::max(1, tocc);
      }
    }
    if (const char* emc = std::getenv("B200LU_BATCH_MC")) {
      const int w = std::atoi(emc);
      if (w >= 2 && w <= kMcMaxContexts) {
        using MFn = void (*)(BBlockArgs, int);
        MFn mfn = h->dest16 ? bfactor_block_mc_kernel<uint16_t, 2> : bfactor_block_mc_kernel<uint32_t, 2>;
        h->mc_contexts = w;
        h->mc_fn = mfn;
        h->mc_smem = mc_smem_bytes(w);
        CU_TRY(h, cudaFuncSetAttribute(mfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(mc_smem_bytes(kMcMaxContexts))));
        int mocc = 0;
        CU_TRY(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&mocc, mfn, 256, h->mc_smem));
        h->mc_grid = prop.multiProcessorCount * std::max(1, mocc);
      }
    }
    if (const char* eg = std::getenv("B200LU_BLOCK_GRID")) {
      const int want = std::atoi(eg);
      if (want > 0) h->block_grid = std::min(h->block_grid, want);
    }
    if (h->use_snode) {
      using SFn = void (*)(BSnodeArgs);
      const char* em = std::getenv("B200LU_SNODE_MINB");
      const int minb = em ? std::atoi(em) : 2;
      SFn sfn = h->snode_rows_per == 1 ? (minb >= 3 ? bfactor_snode_kernel<1, 3> : bfactor_snode_kernel<1, 2>)
                                       : (minb >= 3 ? bfactor_snode_kernel<2, 3> : bfactor_snode_kernel<2, 2>);
      h->snode_fn = sfn;
      int socc = 0;
      CU_TRY(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&socc, sfn, 256, 0));
      h->snode_grid = prop.multiProcessorCount * std::max(1, socc);
    }
    if (h->use_gather) {
      using GFn = void (*)(BGatherArgs);
      const char* em = std::getenv("B200LU_GATHER_MINB");
      const int minb = em ? std::atoi(em) : 2;
      const int gr = h->gather_rows_per, gk = h->gather_batch;
      GFn gfn = nullptr;
      if (gr == 2 && gk == 16) gfn = minb >= 3 ? bfactor_gather_kernel<2, 16, 3> : bfactor_gather_kernel<2, 16, 2>;
      if (gr == 2 && gk == 8) gfn = minb >= 3 ? bfactor_gather_kernel<2, 8, 3> : bfactor_gather_kernel<2, 8, 2>;
      if (gr == 2 && gk == 32) gfn = bfactor_gather_kernel<2, 32, 2>;
      if (gr == 4 && gk == 8) gfn = minb >= 3 ? bfactor_gather_kernel<4, 8, 3> : bfactor_gather_kernel<4, 8, 2>;
      if (gr == 4 && gk == 16) gfn = bfactor_gather_kernel<4, 16, 2>;
      if (gr == 1 && gk == 32) gfn = minb >= 3 ? bfactor_gather_kernel<1, 32, 3> : bfactor_gather_kernel<1, 32, 2>;
      if (!gfn) {
        h->last_error = "gather kernel: unsupported (R, K) combination";
        return B200LU_INVALID_ARGUMENT;
      }
      h->gather_fn = gfn;
      h->gather_smem = gather_smem_bytes(gr, gk, 8);
      CU_TRY(h, cudaFuncSetAttribute(gfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(h->gather_smem)));
      int gocc = 0;
      CU_TRY(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&gocc, gfn, 256, h->gather_smem));
      h->gather_grid = prop.multiProcessorCount * std::max(1, gocc);
    }
  }
  {
    int o1 = 0, o2 = 0, o3 = 0;
    CU_TRY(h, cudaFuncSetAttribute(btri_kernel<true, kTriBufferedWide>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(tri_upper_smem(kTriBufferedWide))));
    {
      // experiments: buffer entries and warps per CTA of the chain launch (B200LU_BATCH_UBUF / _UWARPS)
      const char* eb = std::getenv("B200LU_BATCH_UBUF");
      const char* ew = std::getenv("B200LU_BATCH_UWARPS");
      // measured at C2 x 256 (per U sweep): 96 entries x 8 warps/SM 2.77 ms, 64 x 12 warps/SM 2.25 ms,
      // 48 x 16 warps/SM 2.97 ms (rows longer than the buffer pay a memory round trip per extra chunk)
      const int ub = eb ? std::atoi(eb) : 64;
      h->chain_warps = ew && std::atoi(ew) == 8 ? 8 : 4;
      h->chain_buf = ub == 48 ? 48 : ub == 96 ? kTriBufferedChain : 64;
      h->chain_fn = h->chain_buf == 48 ? btri_kernel<true, 48> : h->chain_buf == 64 ? btri_kernel<true, 64>
                                                                                     : btri_kernel<true, kTriBufferedChain>;
    }
    {
      // two warps per row (tristeam.cuh) unless B200LU_BATCH_UTEAM=0; same buffer per row, 8 warps per CTA
      const char* eu = std::getenv("B200LU_BATCH_UTEAM");
      const int ts = eu ? std::atoi(eu) : 2;
      if (ts == 2 || ts == 4) {
        h->chain_warps = ts * kTriTeams;
        const char* eb2 = std::getenv("B200LU_BATCH_UBUF");
        // buffer per row: 64 entries (12 rows in flight per SM) for large batches, 96 (8 rows, but every row of the C-shaped
        // patterns parked whole) for small ones, where the sweep is bound by the level-to-level latency. Measured per step
        // (two sweeps, C2): 256 scenarios 3.6 ms with 64 / 4.2 with 96 / 5.6 with 48; 32 scenarios 2.40 / 2.03 / 4.83.
        const int auto_buf = h->padded <= 64 ? 96 : 64;
        h->chain_buf = eb2 && std::atoi(eb2) == 48 ? 48 : eb2 && std::atoi(eb2) == 96 ? 96 : eb2 && std::atoi(eb2) == 64 ? 64 : auto_buf;
        h->chain_fn = ts == 4 ? btri_upper_team_kernel<64, 4>
                    : h->chain_buf == 48 ? btri_upper_team_kernel<48, 2> : h->chain_buf == 96 ? btri_upper_team_kernel<96, 2> : btri_upper_team_kernel<64, 2>;
        if (ts == 4) h->chain_buf = 64;
        h->chain_team = true;
        h->chain_team_size = ts;
      }
    }
    const size_t chain_smem = tri_upper_smem(h->chain_buf, h->chain_team ? kTriTeams : h->chain_warps);
    CU_TRY(h, cudaFuncSetAttribute(h->chain_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(chain_smem)));
    CU_TRY(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, btri_kernel<false, kTriBufferedWide>, 256, 0));
    CU_TRY(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, btri_kernel<true, kTriBufferedWide>, 256,
                                                            tri_upper_smem(kTriBufferedWide)));
    CU_TRY(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o3, h->chain_fn, h->chain_warps * 32, chain_smem));
    h->tri_grid = prop.multiProcessorCount * std::max(1, o1);
    if (const char* eg = std::getenv("B200LU_BATCH_LGRID")) {  // experiment: fewer resident CTAs in the L sweep
      if (std::atoi(eg) > 0) h->tri_grid = std::min(h->tri_grid, std::atoi(eg));
    }
    h->tri_grid_upper = prop.multiProcessorCount * std::max(1, o2);
    h->tri_grid_chain = prop.multiProcessorCount * std::max(1, o3);
    // experiment: fewer resident CTAs in the U sweep. Measured at C2 x 256 (two sweeps per step): 444 CTAs 4.53 ms, 296: 5.76,
    // 148: 9.40 (32 scenarios: 2.37 / 2.43 / 2.93) — the sweep is bound by how many rows are in flight, and those by the
    // 16 KB parking buffer per warp; 28 % of the rows (76 % of the entries) have more than 33 upper entries, so a split
    // into short-row and long-row CTAs would buy ~1.2x at best.
    if (const char* eg = std::getenv("B200LU_BATCH_UGRID")) {
      if (std::atoi(eg) > 0) h->tri_grid_chain = std::min(h->tri_grid_chain, std::atoi(eg));
    }
    // chain part of the U sweep: the leading levels up to the first one at least kChainWidth rows wide
    const char* e = std::getenv("B200LU_BATCH_CHAIN_WIDTH");
    const int64_t chain_width = e ? std::atoll(e) : 512;
    int64_t rows = 0;
    for (size_t l = 0; l < S.upper_width.size() && S.upper_width[l] < chain_width; ++l) rows += S.upper_width[l];
    h->upper_chain_rows = static_cast<int32_t>(rows);
  }
  CU_TRY(h, cudaStreamSynchronize(h->stream));
  h->last_error.clear();
  return B200LU_OK;
}

void b200lu_batch_destroy(b200lu_batch* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  void* ptrs[] = {h->d_row_ptr, h->d_col, h->d_diag, h->d_trivial_rows, h->d_pair_row_ptr, h->d_factor_meta, h->d_tail_meta, h->d_blocks, h->d_merged, h->d_g_blocks, h->d_g_batches, h->d_g_recs, h->d_g_waits, h->d_s_blocks, h->d_s_runs, h->d_s_dest, h->d_tile_meta, h->d_tile_rows, h->d_tile_ext, h->d_tile_row_items, h->d_tile_dest, h->d_tile_flags, h->d_tile_prof, h->d_lower_meta,
                  h->d_upper_meta, h->d_dest, h->d_src_of_slot, h->d_scatter_scale, h->d_p, h->d_pq, h->d_row_scale,
                  h->d_col_scale, h->d_a_row_ptr, h->d_a_col, h->d_kkt_hdiag, h->d_kkt_dy, h->d_kkt_stage, h->d_kkt_pos, h->d_a_int, h->d_values, h->d_flags, h->d_failed, h->d_tickets,
                  h->d_stage_a, h->d_stage_in, h->d_stage_in2, h->d_stage_out, h->d_gather, h->d_w, h->d_t1, h->d_t2, h->d_b,
                  h->d_x0, h->d_x, h->d_r, h->d_wv, h->d_cand, h->d_best, h->d_V, h->d_Z, h->d_scal, h->d_up, h->d_partials};
  for (void* p : ptrs) {
    if (p) cudaFree(p);
  }
  for (cudaEvent_t e : h->ev_start) cudaEventDestroy(e);
  for (cudaEvent_t e : h->ev_stop) cudaEventDestroy(e);
  if (h->copy_in) cudaStreamSynchronize(h->copy_in);
  if (h->copy_out) cudaStreamSynchronize(h->copy_out);
  for (int i = 0; i < 2; ++i) {
    for (cudaEvent_t e : {h->ev_in[i], h->ev_vals_used[i], h->ev_rhs_used[i], h->ev_x[i], h->ev_x_out[i]}) {
      if (e) cudaEventDestroy(e);
    }
    for (double* q : {h->d_stage_vals[i], h->d_stage_rhs[i], h->d_stage_x[i]}) {
      if (q && q != h->d_stage_a && q != h->d_stage_in && q != h->d_stage_out) cudaFree(q);
    }
  }
  if (h->copy_in) cudaStreamDestroy(h->copy_in);
  if (h->copy_out) cudaStreamDestroy(h->copy_out);
  if (h->h_scal) cudaFreeHost(h->h_scal);
  if (h->h_up) cudaFreeHost(h->h_up);
  if (h->h_failed) cudaFreeHost(h->h_failed);
  if (h->owns_stream && h->stream) cudaStreamDestroy(h->stream);
  cudaGetLastError();
  delete h;
}

b200lu_status b200lu_batch_check_pattern(const b200lu_batch* h, int64_t n, const int64_t* row_offsets,
                                         const int64_t* col_indices) {
  if (!h || !row_offsets || (!col_indices && h->nnz_source)) return B200LU_INVALID_ARGUMENT;
  if (n != h->n) return B200LU_PATTERN_MISMATCH;
  if (!same_bytes(row_offsets, h->src_row_offsets.data(), sizeof(int64_t) * (n + 1))) return B200LU_PATTERN_MISMATCH;
  if (h->nnz_source && !same_bytes(col_indices, h->src_col_indices.data(), sizeof(int64_t) * h->nnz_source)) {
    return B200LU_PATTERN_MISMATCH;
  }
  return B200LU_OK;
}

b200lu_status b200lu_batch_reset_values(b200lu_batch* h, const double* a_values, int on_device) {
  if (!h || (!a_values && h->nnz_source)) return B200LU_INVALID_ARGUMENT;
  CU_TRY(h, cudaSetDevice(h->device));
  std::fill(h->valid.begin(), h->valid.end(), 0);
  h->have_values = true;
  const double* src = a_values;
  if (!on_device && h->nnz_source) {
    CU_TRY(h, cudaMemcpyAsync(h->d_stage_a, a_values, static_cast<size_t>(h->nnz_source) * h->batch * sizeof(double),
                              cudaMemcpyHostToDevice, h->stream));
    src = h->d_stage_a;
  }
  {
    PhaseScope ps(h, B200LU_PHASE_SCATTER);
    if (h->nnz_source) {
      dim3 grid(static_cast<unsigned>((h->nnz_source + 31) / 32), static_cast<unsigned>(h->groups));
      interleave_kernel<<<grid, 256, 0, h->stream>>>(h->nnz_source, h->batch, src, h->d_a_int);
      ST_TRY(check_launch(h, "interleave_kernel"));
    }
  }
  return launch_scatter(h);
}

b200lu_status b200lu_batch_kkt_bind(b200lu_batch* h, int64_t n_primal, const double* h_diag,
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
  for (void* p : {static_cast<void*>(h->d_kkt_hdiag), static_cast<void*>(h->d_kkt_dy), static_cast<void*>(h->d_kkt_stage),
                  static_cast<void*>(h->d_kkt_pos)}) {
    if (p) cudaFree(p);
  }
  ST_TRY(dev_upload(h, &h->d_kkt_pos, pos));
  ST_TRY(dev_upload(h, &h->d_kkt_hdiag, std::vector<double>(h_diag, h_diag + n_primal)));
  ST_TRY(dev_alloc(h, &h->d_kkt_dy, static_cast<size_t>(n_primal) * h->padded));
  ST_TRY(dev_alloc(h, &h->d_kkt_stage, static_cast<size_t>(n_primal) * h->batch));
  h->kkt_n_primal = n_primal;
  return B200LU_OK;
}

b200lu_status b200lu_batch_kkt_update(b200lu_batch* h, const double* d_y, int on_device, double delta_p, double delta_d) {
  if (!h || (!d_y && h->kkt_n_primal > 0)) return B200LU_INVALID_ARGUMENT;
  CU_TRY(h, cudaSetDevice(h->device));
  if (h->kkt_n_primal < 0 || !h->have_values) {
    h->last_error = "kkt_update: call b200lu_batch_kkt_bind and give one full set of values (reset_values) first";
    return B200LU_INVALID_ARGUMENT;
  }
  if (delta_p < 0.0 || delta_d < 0.0) {  // src/kkt.cpp:44-46
    h->last_error = "kkt_update: regularization must be nonnegative";
    return B200LU_INVALID_ARGUMENT;
  }
  std::fill(h->valid.begin(), h->valid.end(), 0);
  const double* src = d_y;
  if (!on_device && h->kkt_n_primal > 0) {
    CU_TRY(h, cudaMemcpyAsync(h->d_kkt_stage, d_y, static_cast<size_t>(h->kkt_n_primal) * h->batch * sizeof(double),
                              cudaMemcpyHostToDevice, h->stream));
    src = h->d_kkt_stage;
  }
  if (h->n > 0) {
    PhaseScope ps(h, B200LU_PHASE_SCATTER);
    if (h->kkt_n_primal > 0) {
      dim3 grid(static_cast<unsigned>((h->kkt_n_primal + 31) / 32), static_cast<unsigned>(h->groups));
      interleave_kernel<<<grid, 256, 0, h->stream>>>(h->kkt_n_primal, h->batch, src, h->d_kkt_dy);
      ST_TRY(check_launch(h, "interleave_kernel"));
    }
    bkkt_diagonal_kernel<<<warp_blocks(h), 256, 0, h->stream>>>(static_cast<int32_t>(h->n),
                                                                static_cast<int32_t>(h->kkt_n_primal), h->groups,
                                                                h->nnz_source, h->d_kkt_hdiag, h->d_kkt_pos, h->d_kkt_dy,
                                                                delta_p, delta_d, h->d_a_int);
    ST_TRY(check_launch(h, "bkkt_diagonal_kernel"));
  }
  return launch_scatter(h);
}

b200lu_status b200lu_batch_factorize_scattered(b200lu_batch* h, int64_t* failed_rows) {
  if (!h) return B200LU_INVALID_ARGUMENT;
  CU_TRY(h, cudaSetDevice(h->device));
  return launch_factor(h, failed_rows);
}

b200lu_status b200lu_batch_refactorize(b200lu_batch* h, const double* a_values, int on_device, int64_t* failed_rows) {
  ST_TRY(b200lu_batch_reset_values(h, a_values, on_device));
  return launch_factor(h, failed_rows);
}

b200lu_status b200lu_batch_get_values(b200lu_batch* h, int64_t scenario, double* host_out) {
  if (!h || scenario < 0 || scenario >= h->batch || (!host_out && h->nnz_factors)) return B200LU_INVALID_ARGUMENT;
  CU_TRY(h, cudaSetDevice(h->device));
  if (h->nnz_factors) {
    bgather_scenario_kernel<<<blocks_for(h->nnz_factors, 256), 256, 0, h->stream>>>(
        h->nnz_factors, (scenario / 32) * h->nnz_factors, static_cast<int>(scenario % 32), h->d_values, h->d_gather);
    ST_TRY(check_launch(h, "bgather_scenario_kernel"));
    CU_TRY(h, cudaMemcpyAsync(host_out, h->d_gather, static_cast<size_t>(h->nnz_factors) * sizeof(double),
                              cudaMemcpyDeviceToHost, h->stream));
  }
  CU_TRY(h, cudaStreamSynchronize(h->stream));
  return B200LU_OK;
}

int b200lu_batch_valid(const b200lu_batch* h, int64_t scenario) {
  return h && scenario >= 0 && scenario < h->batch && h->valid[scenario] ? 1 : 0;
}

static b200lu_status sweep_common(b200lu_batch* h, const double* y, double* x, int on_device, int64_t* failed_rows,
                                  int which /*0 lower, 1 upper, 2 solve_system*/) {
  for (int32_t s = 0; h && failed_rows && s < h->batch; ++s) failed_rows[s] = -1;
  if (!h || (!y && h->n) || (!x && h->n)) return B200LU_INVALID_ARGUMENT;
  CU_TRY(h, cudaSetDevice(h->device));
  ST_TRY(any_valid(h, which == 0 ? "lower_solve" : which == 1 ? "upper_solve" : "solve_system"));
  if (h->n == 0) return B200LU_OK;
  ST_TRY(vec_in(h, y, on_device, h->d_stage_in, h->d_b));
  if (which == 2) {
    ST_TRY(solve_int(h, h->d_b, h->d_x));
  } else {
    ST_TRY(arm_solve(h));
    bfill_pending_kernel<<<blocks_for(vec_elems(h), 256), 256, 0, h->stream>>>(vec_elems(h), h->d_x);
    ST_TRY(check_launch(h, "bfill_pending_kernel"));
    ST_TRY(which == 0 ? launch_lower(h, h->d_b, h->d_x) : launch_upper(h, h->d_b, h->d_x));
  }
  b200lu_status fail = which == 0 ? B200LU_OK : collect_upper_failure(h, failed_rows);
  ST_TRY(vec_out(h, h->d_x, x, on_device));
  return fail;
}

b200lu_status b200lu_batch_lower_solve(b200lu_batch* h, const double* y, double* x, int on_device) {
  return sweep_common(h, y, x, on_device, nullptr, 0);
}

b200lu_status b200lu_batch_upper_solve(b200lu_batch* h, const double* y, double* x, int on_device, int64_t* failed_rows) {
  return sweep_common(h, y, x, on_device, failed_rows, 1);
}

b200lu_status b200lu_batch_solve(b200lu_batch* h, const double* b, double* x, int on_device, int64_t* failed_rows) {
  return sweep_common(h, b, x, on_device, failed_rows, 2);
}

b200lu_status b200lu_batch_relative_residual(b200lu_batch* h, const double* x, const double* b, int on_device,
                                             double* out) {
  if (!h || !out || (!x && h->n) || (!b && h->n)) return B200LU_INVALID_ARGUMENT;
  CU_TRY(h, cudaSetDevice(h->device));
  if (h->n == 0) {
    for (int32_t s = 0; s < h->batch; ++s) out[s] = 0.0;
    return B200LU_OK;
  }
  ST_TRY(vec_in(h, x, on_device, h->d_stage_in, h->d_x));
  ST_TRY(vec_in(h, b, on_device, h->d_stage_in2, h->d_b));
  ST_TRY(launch_residual(h, h->d_x, h->d_b, h->d_r, kSlotRes));
  ST_TRY(read_scalars(h, kSlotRes, 2));
  for (int32_t s = 0; s < h->batch; ++s) {
    const double bn = std::sqrt(hscal(h, kSlotBn)[s]);
    out[s] = std::sqrt(hscal(h, kSlotRes)[s]) / (bn > 0.0 ? bn : 1.0);  // src/sparse.cpp:286-287
  }
  return B200LU_OK;
}

static b200lu_status batch_refine_common(b200lu_batch* h, const double* b, const double* x0, double* x_out, int on_device,
                                         int use_preconditioner, const b200lu_refine_config* cfg_in,
                                         b200lu_refine_outcome* outcomes, bool fgmres) {
  if (!h || !outcomes || (!b && h->n) || (!x0 && h->n) || (!x_out && h->n)) return B200LU_INVALID_ARGUMENT;
  CU_TRY(h, cudaSetDevice(h->device));
  b200lu_refine_config cfg{20, 1e-14};
  if (cfg_in) cfg = *cfg_in;
  if (cfg.max_iterations > h->refine_capacity) {
    h->last_error = "max_iterations exceeds the handle's refine_capacity";
    return B200LU_INVALID_ARGUMENT;
  }
  if (use_preconditioner) ST_TRY(any_valid(h, "solve_system"));
  if (h->n) {
    ST_TRY(vec_in(h, b, on_device, h->d_stage_in, h->d_b));
    ST_TRY(vec_in(h, x0, on_device, h->d_stage_in2, h->d_x0));
  }
  ST_TRY(fgmres ? fgmres_batch(h, h->d_b, h->d_x0, use_preconditioner, cfg, outcomes)
                : classic_batch(h, h->d_b, h->d_x0, use_preconditioner, cfg, outcomes));
  if (h->n == 0) return B200LU_OK;
  return vec_out(h, h->d_best, x_out, on_device);
}

b200lu_status b200lu_batch_refine_fgmres(b200lu_batch* h, const double* b, const double* x0, double* x_out, int on_device,
                                         int use_preconditioner, const b200lu_refine_config* cfg,
                                         b200lu_refine_outcome* outcomes) {
  return batch_refine_common(h, b, x0, x_out, on_device, use_preconditioner, cfg, outcomes, true);
}

b200lu_status b200lu_batch_refine_classic(b200lu_batch* h, const double* b, const double* x0, double* x_out, int on_device,
                                          int use_preconditioner, const b200lu_refine_config* cfg,
                                          b200lu_refine_outcome* outcomes) {
  return batch_refine_common(h, b, x0, x_out, on_device, use_preconditioner, cfg, outcomes, false);
}

// ---- staged (pipelined) submission -------------------------------------------------------------------
//
// cli::solve_sequence (src/cli.cpp:80-135) hands the solver one system after the other; on a device the
// inputs of system k + 1 can cross the bus while system k is factorized and solved. stage_inputs copies
// on a dedicated stream into the buffer that is NOT in use (two of each), the *_staged calls make the
// compute stream wait for that copy only, and the solution leaves on a third stream.

static b200lu_status stage_setup(b200lu_batch* h) {
  if (h->staged_ready) return B200LU_OK;
  CU_TRY(h, cudaStreamCreateWithFlags(&h->copy_in, cudaStreamNonBlocking));
  CU_TRY(h, cudaStreamCreateWithFlags(&h->copy_out, cudaStreamNonBlocking));
  for (int i = 0; i < 2; ++i) {
    for (cudaEvent_t* e : {&h->ev_in[i], &h->ev_vals_used[i], &h->ev_rhs_used[i], &h->ev_x[i], &h->ev_x_out[i]}) {
      CU_TRY(h, cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    }
  }
  // buffer 0 is the handle's own staging set, buffer 1 is allocated on first use of the staged calls
  h->d_stage_vals[0] = h->d_stage_a;
  h->d_stage_rhs[0] = h->d_stage_in;
  h->d_stage_x[0] = h->d_stage_out;
  ST_TRY(dev_alloc(h, &h->d_stage_vals[1], static_cast<size_t>(h->nnz_source) * h->batch));
  ST_TRY(dev_alloc(h, &h->d_stage_rhs[1], static_cast<size_t>(h->n) * h->batch));
  ST_TRY(dev_alloc(h, &h->d_stage_x[1], static_cast<size_t>(h->n) * h->batch));
  h->staged_ready = true;
  return B200LU_OK;
}

b200lu_status b200lu_batch_stage_inputs(b200lu_batch* h, const double* host_values, const double* host_rhs) {
  if (!h || (!host_values && !host_rhs)) return B200LU_INVALID_ARGUMENT;
  CU_TRY(h, cudaSetDevice(h->device));
  ST_TRY(stage_setup(h));
  const int buf = h->stage_fill;
  for (int q : h->vals_queue) {
    if (q == buf && host_values) {
      h->last_error = "stage_inputs: both staging buffers hold values that have not been consumed (refactorize_staged)";
      return B200LU_INVALID_ARGUMENT;
    }
  }
  for (int q : h->rhs_queue) {
    if (q == buf && host_rhs) {
      h->last_error = "stage_inputs: both staging buffers hold right-hand sides that have not been consumed (solve_refine_staged)";
      return B200LU_INVALID_ARGUMENT;
    }
  }
  // the buffer's previous contents must have been consumed by the compute stream
  CU_TRY(h, cudaStreamWaitEvent(h->copy_in, h->ev_vals_used[buf], 0));
  CU_TRY(h, cudaStreamWaitEvent(h->copy_in, h->ev_rhs_used[buf], 0));
  if (host_values && h->nnz_source) {
    // cudaMemcpyDefault: the buffer may be host memory (pinned for the copy to overlap) or memory of this device
    CU_TRY(h, cudaMemcpyAsync(h->d_stage_vals[buf], host_values, static_cast<size_t>(h->nnz_source) * h->batch * sizeof(double),
                              cudaMemcpyDefault, h->copy_in));
  }
  if (host_rhs && h->n) {
    CU_TRY(h, cudaMemcpyAsync(h->d_stage_rhs[buf], host_rhs, static_cast<size_t>(h->n) * h->batch * sizeof(double),
                              cudaMemcpyDefault, h->copy_in));
  }
  CU_TRY(h, cudaEventRecord(h->ev_in[buf], h->copy_in));
  if (host_values) h->vals_queue.push_back(buf);
  if (host_rhs) h->rhs_queue.push_back(buf);
  h->stage_fill = buf ^ 1;
  return B200LU_OK;
}

b200lu_status b200lu_batch_refactorize_staged(b200lu_batch* h, int64_t* failed_rows) {
  if (!h) return B200LU_INVALID_ARGUMENT;
  CU_TRY(h, cudaSetDevice(h->device));
  if (h->vals_queue.empty()) {
    h->last_error = "refactorize_staged: no staged values (call b200lu_batch_stage_inputs first)";
    return B200LU_INVALID_ARGUMENT;
  }
  const int buf = h->vals_queue.front();
  h->vals_queue.erase(h->vals_queue.begin());
  CU_TRY(h, cudaStreamWaitEvent(h->stream, h->ev_in[buf], 0));
  std::fill(h->valid.begin(), h->valid.end(), 0);
  h->have_values = true;
  {
    PhaseScope ps(h, B200LU_PHASE_SCATTER);
    if (h->nnz_source) {
      dim3 grid(static_cast<unsigned>((h->nnz_source + 31) / 32), static_cast<unsigned>(h->groups));
      interleave_kernel<<<grid, 256, 0, h->stream>>>(h->nnz_source, h->batch, h->d_stage_vals[buf], h->d_a_int);
      ST_TRY(check_launch(h, "interleave_kernel"));
    }
  }
  CU_TRY(h, cudaEventRecord(h->ev_vals_used[buf], h->stream));
  ST_TRY(launch_scatter(h));
  return launch_factor(h, failed_rows);
}

b200lu_status b200lu_batch_solve_refine_staged(b200lu_batch* h, int refine, const b200lu_refine_config* cfg_in,
                                               double* host_x_out, b200lu_refine_outcome* outcomes, int64_t* failed_rows) {
  for (int32_t s = 0; h && failed_rows && s < h->batch; ++s) failed_rows[s] = -1;
  if (!h || (!host_x_out && h->n) || (refine && !outcomes)) return B200LU_INVALID_ARGUMENT;
  CU_TRY(h, cudaSetDevice(h->device));
  if (h->rhs_queue.empty()) {
    h->last_error = "solve_refine_staged: no staged right-hand sides (call b200lu_batch_stage_inputs first)";
    return B200LU_INVALID_ARGUMENT;
  }
  ST_TRY(any_valid(h, "solve_system"));
  if (h->n == 0) return B200LU_OK;
  b200lu_refine_config cfg{20, 1e-14};
  if (cfg_in) cfg = *cfg_in;
  if (refine && cfg.max_iterations > h->refine_capacity) {
    h->last_error = "max_iterations exceeds the handle's refine_capacity";
    return B200LU_INVALID_ARGUMENT;
  }
  const int buf = h->rhs_queue.front();
  h->rhs_queue.erase(h->rhs_queue.begin());
  CU_TRY(h, cudaStreamWaitEvent(h->stream, h->ev_in[buf], 0));
  ST_TRY(to_interleaved(h, h->n, h->d_stage_rhs[buf], h->d_b));
  CU_TRY(h, cudaEventRecord(h->ev_rhs_used[buf], h->stream));
  ST_TRY(solve_int(h, h->d_b, h->d_x));
  b200lu_status fail = collect_upper_failure(h, failed_rows);
  const double* result = h->d_x;
  if (refine) {
    ST_TRY(copy_dd(h, h->d_x0, h->d_x));
    ST_TRY(fgmres_batch(h, h->d_b, h->d_x0, 1, cfg, outcomes));
    result = h->d_best;
  }
  // the staging buffer's previous solution must have left the device before it is overwritten
  CU_TRY(h, cudaStreamWaitEvent(h->stream, h->ev_x_out[buf], 0));
  ST_TRY(from_interleaved(h, h->n, result, h->d_stage_x[buf]));
  CU_TRY(h, cudaEventRecord(h->ev_x[buf], h->stream));
  CU_TRY(h, cudaStreamWaitEvent(h->copy_out, h->ev_x[buf], 0));
  CU_TRY(h, cudaMemcpyAsync(host_x_out, h->d_stage_x[buf], static_cast<size_t>(h->n) * h->batch * sizeof(double),
                            cudaMemcpyDefault, h->copy_out));  // host memory or memory of this device
  CU_TRY(h, cudaEventRecord(h->ev_x_out[buf], h->copy_out));
  return fail;
}

b200lu_status b200lu_batch_staged_wait(b200lu_batch* h) {
  if (!h) return B200LU_INVALID_ARGUMENT;
  CU_TRY(h, cudaSetDevice(h->device));
  if (h->copy_in) CU_TRY(h, cudaStreamSynchronize(h->copy_in));
  CU_TRY(h, cudaStreamSynchronize(h->stream));
  if (h->copy_out) CU_TRY(h, cudaStreamSynchronize(h->copy_out));
  return B200LU_OK;
}

b200lu_status b200lu_batch_get_info(const b200lu_batch* h, b200lu_batch_info* out) {
  if (!h || !out) return B200LU_INVALID_ARGUMENT;
  out->batch = h->batch;
  out->padded_batch = h->padded;
  out->unit_scenarios = h->unit;
  out->factor_rows = h->n_factor_rows + h->n_block_rows;
  out->blocked_rows = h->n_block_rows;
  out->blocks = h->use_tiles ? h->n_tiles : h->use_snode ? h->n_s_blocks : h->use_gather ? h->n_g_blocks : h->n_blocks;
  out->blocked_pairs = h->blocked_pairs;
  out->factor_grid = h->factor_grid;
  out->tri_grid = h->tri_grid;
  out->n = h->n;
  out->nnz_factors = h->nnz_factors;
  out->nnz_source = h->nnz_source;
  out->update_pairs = h->sched.update_pairs;
  out->lower_levels = h->sched.lower_levels;
  out->upper_levels = h->sched.upper_levels;
  out->device_bytes = h->device_bytes;
  out->alloc_events = h->alloc_events;
  out->launches = static_cast<int64_t>(h->launches);
  out->tiled = h->use_tiles ? 1 : 0;
  out->tile_rows = h->use_tiles ? h->tile_rows_per : 0;
  out->tile_smem_bytes = h->use_tiles ? static_cast<int64_t>(h->tile_smem) : 0;
  out->tile_grid = h->use_tiles ? h->tile_grid : 0;
  out->tile_fetched_entries = h->tile_fetched_entries;
  return B200LU_OK;
}

b200lu_status b200lu_tile_plan_emulate(const b200lu_symbolic_view* sym, int rows_per_tile, int64_t tile_entries,
                                       int64_t tail_width, double pivot_floor, double* values, int64_t* failed_row,
                                       b200lu_tile_plan_stats* stats, char* error_buf, int error_buf_len) {
  auto fail = [&](const std::string& msg) {
    if (error_buf && error_buf_len > 0) {
      std::strncpy(error_buf, msg.c_str(), static_cast<size_t>(error_buf_len) - 1);
      error_buf[error_buf_len - 1] = 0;
    }
    return B200LU_INVALID_ARGUMENT;
  };
  if (!sym || !values || rows_per_tile < 1 || tile_entries < 1) return fail("null or non-positive argument");
  Schedule S;
  ScheduleTuning tune;
  tune.tail_min_levels = int64_t{1} << 40;
  const std::string err = build_schedule(*sym, tune, S);
  if (!err.empty()) return fail(err);
  const int64_t cut = trailing_cut_level(S, tail_width);
  std::vector<int32_t> tail_rows;
  int64_t failed = -1;
  auto note_pivot = [&](int32_t i) {
    if (std::fabs(values[S.diag[i]]) <= pivot_floor && (failed < 0 || i < failed)) failed = i;
  };
  // head rows: plain up-looking elimination in dependency-level order (what the head launch does)
  for (int32_t i : S.lower_order) {
    if (S.diag[i] == S.row_ptr[i]) {
      note_pivot(i);
      continue;
    }
    if (S.lower_level[i] >= cut) {
      tail_rows.push_back(i);
      continue;
    }
    for (int32_t k = S.row_ptr[i]; k < S.diag[i]; ++k) {
      const int32_t d = S.col[k], dd = S.diag[d];
      const double alpha = values[k] / values[dd];
      values[k] = alpha;
      int32_t pos = k + 1;
      for (int32_t t = dd + 1; t < S.row_ptr[d + 1]; ++t) {
        while (S.col[pos] < S.col[t]) ++pos;
        const double prod = alpha * values[t];
        values[pos] = values[pos] - prod;
      }
    }
    note_pivot(i);
  }
  std::sort(tail_rows.begin(), tail_rows.end());
  TilePlan plan;
  const std::string perr = build_tile_plan(S, tail_rows, rows_per_tile, tile_entries, plan);
  if (!perr.empty()) return fail(perr);
  const int64_t f2 = emulate_tile_plan(S, plan, pivot_floor, values);
  if (f2 <= -2) return fail("plan error " + std::to_string(f2) + ": the tile plan is inconsistent");
  if (f2 >= 0 && (failed < 0 || f2 < failed)) failed = f2;
  if (failed_row) *failed_row = failed;
  if (stats) {
    stats->tiles = static_cast<int64_t>(plan.tiles.size());
    stats->rows = static_cast<int64_t>(plan.rows.size());
    stats->items = static_cast<int64_t>(plan.ext.size());
    stats->fetched_entries = plan.fetched_entries;
    stats->pairs = plan.pairs;
    stats->largest_tile_entries = plan.rows_smem_entries;
    int64_t consumed = 0;
    for (const ExtItem& q : plan.ext) consumed += static_cast<int64_t>(q.cnt_flags & 0xffffu) * __builtin_popcount(q.users);
    stats->consumed_entries = consumed;
  }
  return failed >= 0 ? B200LU_ZERO_PIVOT : B200LU_OK;
}

b200lu_status b200lu_batch_tile_profile(b200lu_batch* h, int64_t* cycles_out, int reset) {
  if (!h || !cycles_out) return B200LU_INVALID_ARGUMENT;
  for (int i = 0; i < 16; ++i) cycles_out[i] = 0;
  if (!h->d_tile_prof) return B200LU_OK;
  CU_TRY(h, cudaSetDevice(h->device));
  CU_TRY(h, cudaStreamSynchronize(h->stream));
  static_assert(sizeof(long long) == sizeof(int64_t), "counter width");
  CU_TRY(h, cudaMemcpy(cycles_out, h->d_tile_prof, 16 * sizeof(int64_t), cudaMemcpyDeviceToHost));
  if (reset) CU_TRY(h, cudaMemset(h->d_tile_prof, 0, 16 * sizeof(int64_t)));
  return B200LU_OK;
}

b200lu_status b200lu_batch_set_timing(b200lu_batch* h, int enabled) {
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

b200lu_status b200lu_batch_get_phase_times(b200lu_batch* h, double* ms_out, int64_t* count_out, int reset) {
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

b200lu_status b200lu_batch_synchronize(b200lu_batch* h) {
  if (!h) return B200LU_INVALID_ARGUMENT;
  CU_TRY(h, cudaSetDevice(h->device));
  CU_TRY(h, cudaStreamSynchronize(h->stream));
  return B200LU_OK;
}

}  // extern "C"
