// Scenario batches: B independent systems that share ONE sparsity pattern (same symbolic
// analysis), factorized and solved together (BASELINE config "batch of 256
// independent scenario systems").
//
// Layout. Every per-scenario array is stored scenario-interleaved in groups of 32:
//     a[g][k][lane]   = value k of scenario 32*g + lane
// so a warp that owns (row i, scenarios of group g) reads and writes 256 contiguous bytes per
// matrix entry, the pattern/index loads are warp-uniform, and the arithmetic of one scenario is
// exactly the single-system arithmetic of the reference, entry by entry and in the same order:
// every scenario's L/U values, triangular solves and SpMV are bit-identical to the CPU result.
// A single system is bound by its dependency chain; in a batch the same chain is
// shared by 32 scenarios per warp and by all groups at once, which is what makes the path
// bandwidth-bound.
#pragma once

#include "common.cuh"
#include "dest.cuh"
#include "schedule.hpp"

namespace b200lu {

constexpr int kBatchLanes = 32;

// Flag load with ACQUIRE semantics at gpu scope: the data it guards (another SM's stores, fenced and
// then flagged with a relaxed store, i.e. a release pattern) is read afterwards with ordinary L2-only
// loads / asynchronous copies, and the PTX memory model orders those behind the flag only through an
// acquire — a control dependency on a relaxed load is not enough on paper, whatever the hardware did
// in the stress runs.
__device__ __forceinline__ int32_t ld_acquire_s32(const int32_t* p) {
  int32_t v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Spins until the (row, unit) flag reaches `gen`. The poll is paced (sleep doubling from 32 ns to
// 256 ns): a stalled dependency chain leaves most resident warps waiting, and unpaced polls — tens
// per microsecond and warp — compete with the working warps for the load/store path. (Relaxed polls followed by ONE acquire
// load once the flag is seen set — no L1 invalidation per poll — measured the same: 22.2 / 5.70 ms at 256 / 32 scenarios.)
__device__ __forceinline__ int32_t ld_flag_poll(const int32_t* p) {
#ifdef B200LU_POLL_ATOMIC
  return atomicOr(const_cast<int32_t*>(p), 0);
#else
  return ld_acquire_s32(p);
#endif
}
__device__ __forceinline__ void wait_flag(const int32_t* f, int32_t gen) {
  unsigned ns = 32;
  while (ld_flag_poll(f) < gen) {
    __nanosleep(ns);
    ns = min(ns * 2, 256u);
  }
}
__device__ __forceinline__ void st_relaxed_s32(int32_t* p, int32_t v) {
  asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Every access of the refactorization kernel to `values` bypasses L1: a 128-byte line holds more
// than one unit's scenarios, so a line cached while one unit of a row was processed would go
// stale when another SM finishes the neighbouring unit. Loads are gpu-scope relaxed (served by
// L2), stores are L2-only (st.global.cg), the asynchronous copies are cp.async.cg.
__device__ __forceinline__ double ld_cg(const double* p) { return ld_l2(p); }
__device__ __forceinline__ void st_cg(double* p, double v) { __stcg(p, v); }

// ------------------------------------------------------------ layout changes
//
// src[s][k] (scenario-major, what the caller holds: one CSR value array / one vector per
// scenario) -> dst[g][k][lane]. Lanes past the last scenario replicate it, so padded lanes run
// on well-formed data and can never raise a spurious pivot failure. 32x32 tile through shared
// memory: both sides coalesced.
__global__ void __launch_bounds__(256)
interleave_kernel(int64_t len, int32_t batch, const double* __restrict__ src, double* __restrict__ dst) {
  __shared__ double tile[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t k0 = static_cast<int64_t>(blockIdx.x) * 32;
  const int32_t g = blockIdx.y;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int s = ty + 8 * j;
    const int32_t sc = min(g * 32 + s, batch - 1);
    tile[s][tx] = k0 + tx < len ? src[static_cast<int64_t>(sc) * len + k0 + tx] : 0.0;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int kk = ty + 8 * j;
    if (k0 + kk < len) dst[(static_cast<int64_t>(g) * len + k0 + kk) * 32 + tx] = tile[tx][kk];
  }
}

// dst[s][k] <- src[g][k][lane] for the real scenarios.
__global__ void __launch_bounds__(256)
deinterleave_kernel(int64_t len, int32_t batch, const double* __restrict__ src, double* __restrict__ dst) {
  __shared__ double tile[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t k0 = static_cast<int64_t>(blockIdx.x) * 32;
  const int32_t g = blockIdx.y;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int kk = ty + 8 * j;
    tile[kk][tx] = k0 + kk < len ? src[(static_cast<int64_t>(g) * len + k0 + kk) * 32 + tx] : 0.0;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int s = ty + 8 * j;
    const int32_t sc = g * 32 + s;
    if (sc < batch && k0 + tx < len) dst[static_cast<int64_t>(sc) * len + k0 + tx] = tile[tx][s];
  }
}

// ------------------------------------------------------------------ K1 batched
//
// scatter_values (src/numeric.cpp:19-22) for every scenario: gather form through the inverse
// map, fill slots exactly 0, one coalesced 256-byte store per (slot, group).
#ifndef B200LU_SCATTER_SLOTS
#define B200LU_SCATTER_SLOTS 4
#endif
constexpr int kScatterSlots = B200LU_SCATTER_SLOTS;  // consecutive slots a warp takes per step (a multiple of 4)
static_assert(kScatterSlots % 4 == 0 && kScatterSlots >= 4, "index loads are 16 bytes");

__global__ void __launch_bounds__(256)
bscatter_kernel(int64_t nnz_factors, int64_t nnz_source, int32_t groups,
                const int32_t* __restrict__ src_of_slot, const double* __restrict__ a_int,
                const double* __restrict__ scatter_scale, double* __restrict__ values) {
  // a warp takes kScatterSlots consecutive slots per step: 16-byte loads of their source indices, the (few) source
  // values requested together, 256-byte stores — a quarter of the dependent index -> value -> store round trips of the
  // slot-per-step form (scatter phase at C2 x 256 incl. the layout change: 1.63 -> 1.10 ms; 8 slots 1.08, 16 slots 1.05:
  // the 4.5 GB of stores are what is left)
  constexpr int S = kScatterSlots;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int64_t chunks = (nnz_factors + S - 1) / S;
  const int64_t total = chunks * groups;
  for (int64_t t = warp; t < total; t += nwarps) {
    const int64_t g = t / chunks, s0 = (t - g * chunks) * S;
    int32_t k[S];
    if (s0 + S <= nnz_factors) {
#pragma unroll
      for (int q = 0; q < S / 4; ++q) {
        const int4 k4 = __ldg(reinterpret_cast<const int4*>(src_of_slot + s0) + q);
        k[4 * q] = k4.x, k[4 * q + 1] = k4.y, k[4 * q + 2] = k4.z, k[4 * q + 3] = k4.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < S; ++j) k[j] = s0 + j < nnz_factors ? __ldg(src_of_slot + s0 + j) : -2;  // -2: no such slot
    }
    double v[S];
#pragma unroll
    for (int j = 0; j < S; ++j) v[j] = k[j] >= 0 ? a_int[(g * nnz_source + k[j]) * 32 + lane] : 0.0;
    if (scatter_scale != nullptr) {
#pragma unroll
      for (int j = 0; j < S; ++j) {
        if (k[j] >= 0) v[j] = __dmul_rn(v[j], __ldg(scatter_scale + k[j]));
      }
    }
    double* out = values + (g * nnz_factors + s0) * 32 + lane;
#pragma unroll
    for (int j = 0; j < S; ++j) {
      if (k[j] != -2) out[j * 32] = v[j];
    }
  }
}

// assemble_kkt's diagonal (see kkt_diagonal_kernel, factor.cuh) for every scenario: d_y is
// interleaved [groups][n_primal][32], the operator values are [groups][nnz_source][32].
__global__ void __launch_bounds__(256)
bkkt_diagonal_kernel(int32_t n_total, int32_t n_primal, int32_t groups, int64_t nnz_source,
                     const double* __restrict__ h_diag, const int32_t* __restrict__ diag_source_pos,
                     const double* __restrict__ d_y, double delta_p, double delta_d, double* __restrict__ a_int) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (warp >= static_cast<int64_t>(n_total) * groups) return;
  const int64_t g = warp / n_total, i = warp - g * n_total;
  double v = -delta_d;
  if (i < n_primal) v = __dadd_rn(__ldg(h_diag + i), __dadd_rn(d_y[(g * n_primal + i) * 32 + lane], delta_p));
  a_int[(g * nnz_source + __ldg(diag_source_pos + i)) * 32 + lane] = v;
}

// Pivot check of the rows without a strict-lower entry (elimination leaves them unchanged,
// src/numeric.cpp:36; the check of src/numeric.cpp:48 still applies).
__global__ void __launch_bounds__(256)
btrivial_pivot_kernel(int32_t count, int32_t groups, int64_t nnz_factors, const int32_t* __restrict__ rows,
                      const int32_t* __restrict__ diag, const double* __restrict__ values, double pivot_floor,
                      int32_t* failed) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (warp >= static_cast<int64_t>(count) * groups) return;
  const int32_t g = static_cast<int32_t>(warp % groups);
  const int32_t i = rows[warp / groups];
  const double v = values[(static_cast<int64_t>(g) * nnz_factors + diag[i]) * 32 + lane];
  if (fabs(v) <= pivot_floor) atomicMin(failed + g * 32 + lane, i);
}

// ------------------------------------------------------------------ K2 batched
//
// eliminate (src/numeric.cpp:27-58) for S scenarios of one row at a time. A unit of work is
// (row i, S consecutive scenarios); its warp is laid out as E = 32/S entry lanes x S scenario
// lanes. The pivots are walked in ascending order exactly as in the reference; for pivot d the
// upper entries of row d are streamed from L2/HBM (E entries x S scenarios = 256 bytes per
// instruction) and applied to row i, in place, through the precomputed destination table
// (bfactor_unit below).
//
// Dependencies: one generation counter per (row, unit). The owner updates the row, fences, and
// stores the current generation; consumers read the flag before reading the row's upper entries.
// Units are claimed in (dependency level, unit) order by persistent warps, so a claimed unit's
// dependencies are finished or owned by a resident warp.
struct BFactorArgs {
  int32_t n_rows;        // rows that have pivots, in dependency-level order
  int32_t units;         // units per row = padded batch / S
  int32_t gen;           // generation of this factorization
  const FactorMeta* meta;
  const int32_t* row_ptr;
  const int32_t* col;
  const int32_t* diag;
  const int64_t* pair_row_ptr;
  const void* dest;
  double* values;        // [groups][nnz_factors][32]
  int64_t nnz_factors;
  int32_t* flags;        // [n][units]; INT32_MAX for rows without pivots (always ready)
  double pivot_floor;
  int32_t* failed;       // [padded batch], atomicMin, INT32_MAX = none
  unsigned long long* ticket;
};

// a += v performed by L2 (red.global.add.f64, round-to-nearest): fire-and-forget, no load latency
__device__ __forceinline__ void red_add_f64(double* p, double v) {
  asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// One unit = (row i, S scenarios). Row i is updated IN PLACE, and every update
//     a_ij <- a_ij - alpha * u_dj                                  (src/numeric.cpp:44)
// is issued as a reduction performed by L2: red.add(a_ij, -(alpha * u_dj)). The product is rounded
// on its own (__dmul_rn) and IEEE a + (-p) == a - p, so the result is bit-identical to the
// reference's two-rounding update — but the warp never waits for a_ij: no read-modify-write
// chain, only the streaming loads of row d's upper entries (8 of them, 2 KB per warp, in flight
// at once) and one load of a_id per pivot for alpha = a_id / u_dd (src/numeric.cpp:40), which the
// hardware orders after THIS THREAD's earlier reductions to that address. Per-address order is what
// bit-exactness needs (pivots ascending per slot), and it is only safe when every operation on an
// address comes from one thread: the kernel is instantiated with S = 32 (one lane per scenario,
// E = 1). With S < 32 the entry lanes of a scenario take turns on a slot from pivot to pivot with a
// __syncwarp() in between, which measured ~10 % faster and passed every parity test — but a
// reduction and a later load (or reduction) issued by DIFFERENT lanes of the warp can overtake each
// other on the way to L2: the B200LU_POLL_ATOMIC stress build (slow, atomic flag polls) turns that
// into wrong, run-to-run different values in the last rows at S = 8/16 and never at S = 32.
template <typename DestT, int S, int kUnroll, bool kPrefetch>
__device__ __forceinline__ void bfactor_unit(const BFactorArgs& a, const FactorMeta mt, int32_t u, int lane) {
  constexpr int E = 32 / S;
  const unsigned full = 0xffffffffu;
  const int s = lane % S, e = lane / S;
  const int32_t i = mt.row, lo = mt.lo, nl = mt.dg - mt.lo;
  const int32_t sc0 = u * S;
  // element (slot k, scenario s of this unit) lives at gbase[k * 32]
  double* gbase = a.values + static_cast<int64_t>(sc0 >> 5) * a.nnz_factors * 32 + (sc0 & 31) + s;
  double* rowg = gbase + static_cast<int64_t>(lo) * 32;
  const DestT* __restrict__ dest = static_cast<const DestT*>(a.dest);

  int64_t p = a.pair_row_ptr[i];
  for (int32_t k0 = 0; k0 < nl; k0 += 32) {
    // lane q resolves pivot k0+q: its row d, where d's upper part starts, how long it is, and
    // whether d is already published (most are: the probe saves the poll round trip later)
    int32_t my_d = 0, my_dd = 0, my_m = 0, my_ready = 0;
    if (k0 + lane < nl) {
      my_d = __ldg(a.col + lo + k0 + lane);
      my_dd = __ldg(a.diag + my_d);
      my_m = __ldg(a.row_ptr + my_d + 1) - my_dd - 1;
      my_ready = ld_acquire_s32(a.flags + static_cast<int64_t>(my_d) * a.units + u) >= a.gen;
    }
    __syncwarp();
    const int32_t cnt = min(32, nl - k0);
    // kPrefetch: the diagonal and the first load batch of the NEXT pivot row (already published
    // according to the probe) are requested before the current pivot's reductions are issued, so
    // one memory round trip per pivot leaves the warp's serial path
    double pf_udd = 0.0, pf_uv[kUnroll];
    bool pf_ok = false;
    auto prefetch = [&](int32_t qn) {
      pf_ok = false;
      if (kPrefetch && qn < cnt && __shfl_sync(full, my_ready, qn)) {
        const int32_t ddn = __shfl_sync(full, my_dd, qn);
        const int32_t mn = __shfl_sync(full, my_m, qn);
        const double* ugn = gbase + static_cast<int64_t>(ddn) * 32;
        pf_udd = ld_cg(ugn);
#pragma unroll
        for (int j = 0; j < kUnroll; ++j) {
          pf_uv[j] = 0.0;
          if (e + j * E < mn) pf_uv[j] = ld_cg(ugn + static_cast<int64_t>(1 + e + j * E) * 32);
        }
        pf_ok = true;
      }
    };
    prefetch(0);
    for (int32_t q = 0; q < cnt; ++q) {
      const int32_t dd = __shfl_sync(full, my_dd, q);
      const int32_t m = __shfl_sync(full, my_m, q);
      if (!__shfl_sync(full, my_ready, q)) {
        const int32_t d = __shfl_sync(full, my_d, q);
        const int32_t* f = a.flags + static_cast<int64_t>(d) * a.units + u;
        wait_flag(f, a.gen);
      }
      const double* ug = gbase + static_cast<int64_t>(dd) * 32;
      const int32_t k = k0 + q;
      if (E > 1) __syncwarp();  // the other entry lanes' reductions of the previous pivot are issued
      const double aik = ld_cg(rowg + static_cast<int64_t>(k) * 32);
      double udd, uv0[kUnroll];
      if (kPrefetch && pf_ok) {
        udd = pf_udd;
#pragma unroll
        for (int j = 0; j < kUnroll; ++j) uv0[j] = pf_uv[j];
      } else {
        udd = ld_cg(ug);
#pragma unroll
        for (int j = 0; j < kUnroll; ++j) {
          uv0[j] = 0.0;
          if (e + j * E < m) uv0[j] = ld_cg(ug + static_cast<int64_t>(1 + e + j * E) * 32);
        }
      }
      int32_t ds0[kUnroll];
#pragma unroll
      for (int j = 0; j < kUnroll; ++j) ds0[j] = e + j * E < m ? dest[p + e + j * E] : 0;
      prefetch(q + 1);
      const double nalpha = -(aik / udd);  // src/numeric.cpp:40; the sign is exact
#pragma unroll
      for (int j = 0; j < kUnroll; ++j) {
        if (e + j * E < m) red_add_f64(rowg + static_cast<int64_t>(ds0[j]) * 32, __dmul_rn(nalpha, uv0[j]));  // src/numeric.cpp:44
      }
      int32_t c = e + kUnroll * E;
      for (; c + (kUnroll - 1) * E < m; c += kUnroll * E) {
        double uv[kUnroll];
        int32_t ds[kUnroll];
#pragma unroll
        for (int j = 0; j < kUnroll; ++j) {
          uv[j] = ld_cg(ug + static_cast<int64_t>(1 + c + j * E) * 32);
          ds[j] = dest[p + c + j * E];
        }
#pragma unroll
        for (int j = 0; j < kUnroll; ++j) red_add_f64(rowg + static_cast<int64_t>(ds[j]) * 32, __dmul_rn(nalpha, uv[j]));
      }
      for (; c < m; c += E) {
        const double uv = ld_cg(ug + static_cast<int64_t>(1 + c) * 32);
        red_add_f64(rowg + static_cast<int64_t>(dest[p + c]) * 32, __dmul_rn(nalpha, uv));
      }
      p += m;
      // l_id is final (src/numeric.cpp:41); nobody reads it during elimination
      if (e == 0) st_cg(rowg + static_cast<int64_t>(k) * 32, -nalpha);
    }
  }

  // src/numeric.cpp:48: a failing pivot is recorded (lowest row wins) and the row is published
  // anyway so dependents never hang (include/rlu/schedule.hpp:29-33, 82-87)
  // The publication comes first (it is what the next row of the chain waits for); the check reads
  // the final diagonal afterwards.
  __syncwarp();
  if (lane == 0) {
    __threadfence();
    st_relaxed_s32(a.flags + static_cast<int64_t>(i) * a.units + u, a.gen);
  }
  if (e == 0 && fabs(ld_cg(rowg + static_cast<int64_t>(nl) * 32)) <= a.pivot_floor) atomicMin(a.failed + sc0 + s, i);
}

template <typename DestT, int S, int WARPS, int kMinBlocks, int kUnroll, bool kPrefetch>
__global__ void __launch_bounds__(WARPS * 32, kMinBlocks)
bfactor_kernel(const BFactorArgs a) {
  const int lane = threadIdx.x & 31;
  const unsigned long long total = static_cast<unsigned long long>(a.n_rows) * a.units;
  while (true) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(a.ticket, 1ull);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= total) break;
    const int32_t r = static_cast<int32_t>(t / a.units);
    const int32_t u = static_cast<int32_t>(t - static_cast<unsigned long long>(r) * a.units);
    const int4 m4 = __ldg(reinterpret_cast<const int4*>(a.meta) + r);
    bfactor_unit<DestT, S, kUnroll, kPrefetch>(a, FactorMeta{m4.x, m4.y, m4.z, m4.w}, u, lane);
    __syncwarp();
  }
}

__device__ __forceinline__ void cp_async_16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(smem_dst))),
               "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async_4(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(smem_dst))),
               "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

// ------------------------------------------------ K2 batched, row-blocked trailing part
//
// The narrow trailing levels of the elimination DAG (the top of the elimination tree) hold a few
// per cent of the rows but most of the update pairs, and their rows form chains: consecutive rows
// share almost all of their pivots, and every row is a pivot of the ones that follow. There a
// warp owns a BLOCK of kBlockRows consecutive rows (x S scenarios) and walks the ascending merge of
// their pivot lists: the upper entries of pivot row d are loaded ONCE and applied to every row of
// the block that has the pivot (each with its own alpha and its own destination slice), which
// divides the re-reads of the trailing pivot rows — the dominant DRAM traffic of the unblocked
// kernel — by the block height, and turns most chain hand-offs into program order inside one warp.
// Block height: 2 rows per warp (80 registers, 24 warps per SM) measures 25.8 ms against 28.9 ms
// unblocked at C2 x 256; 4 rows per warp (-DB200LU_BLOCK_ROWS=4: 126 registers, 16 warps per SM) cuts
// the DRAM traffic of the trailing part 4x but waits on the chain hand-offs: 32-34 ms.
#ifndef B200LU_BLOCK_ROWS
#define B200LU_BLOCK_ROWS 2
#endif
constexpr int kBlockRows = B200LU_BLOCK_ROWS;  // 2 or 4
static_assert(kBlockRows == 2 || kBlockRows == 4, "block height");

struct BlockMeta {          // one 32-byte record per block
  int32_t row[4];           // row ids, ascending; -1 pads (short last block, kBlockRows == 2)
  int32_t mbeg, mend;       // its merged pivots
  int32_t pad0, pad1;
};
struct MergedPivot {
  int32_t d;      // pivot row
  uint32_t bits;  // bit r: block row r has the pivot; bit 8 + r: block row r is final after this pivot;
                  // bit 16: the pivot row d is itself a row of this block
};

struct BBlockArgs {
  int32_t n_blocks;
  int32_t first_unit, units_here;  // this launch handles units [first_unit, first_unit + units_here) of every block
  int32_t units;                   // units per row (stride of the flag array)
  int32_t gen;
  const BlockMeta* blocks;
  const MergedPivot* merged;
  const int32_t* row_ptr;
  const int32_t* diag;
  const int64_t* pair_row_ptr;
  const void* dest;
  double* values;
  int64_t nnz_factors;
  int32_t* flags;
  double pivot_floor;
  int32_t* failed;
  unsigned long long* ticket;
};

// Staging of the pivot rows (B200LU_BLOCK_STAGE = entries per stage, 0 = off). Every in-flight row of
// the trailing part applies one more pivot each time the frontier of its chain advances by a level,
// so the time of that part is (levels) x (latency of applying ONE pivot), and with loads held in
// registers a pivot row of m entries costs m/8 dependent memory round trips. With staging the whole
// pivot row (diagonal + upper entries of the group: one contiguous block of (m+1) x 256 bytes) and
// the matching destination slices are copied to the warp's shared-memory stage with cp.async (L2-only)
// and consumed after ONE wait.
// Measured at C2 x 256 with 2-row blocks, factor phase: no staging 25.9 ms (24 warps/SM); 48 entries per
// stage 24.3 ms (16 warps/SM); 32 entries 25.9 ms (24 warps/SM); 4-row blocks with 48 entries 31.9 ms.
#ifndef B200LU_BLOCK_STAGE
#define B200LU_BLOCK_STAGE 48
#endif
constexpr int kBlockStage = B200LU_BLOCK_STAGE;
constexpr int kBlockStageDest = kBlockStage * 4 + 8 <= 256 ? 32 : (kBlockStage * 4 + 8 + 7) / 8;  // doubles reserved per row for its destination slice (256 bytes at the default stage)
__host__ __device__ constexpr size_t block_stage_doubles() {
  return kBlockStage > 0 ? static_cast<size_t>(kBlockStage) * 32 + kBlockRows * kBlockStageDest : 0;
}
#ifndef B200LU_BLOCK_MINB
#define B200LU_BLOCK_MINB (kBlockStage > 0 ? 2 : kBlockRows == 2 ? 3 : 2)
#endif
template <typename DestT, int S>
__global__ void __launch_bounds__(256, B200LU_BLOCK_MINB)
bfactor_block_kernel(const BBlockArgs a) {
  constexpr int E = 32 / S;
  constexpr int R = kBlockRows;
#ifdef B200LU_BLOCK_UNROLL
  constexpr int kUnroll = B200LU_BLOCK_UNROLL;
#else
  constexpr int kUnroll = 8;
#endif
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int s = lane % S, e = lane / S;
  const DestT* __restrict__ dest = static_cast<const DestT*>(a.dest);
  extern __shared__ __align__(16) double block_smem[];
  double* stage = block_smem + static_cast<size_t>(threadIdx.x >> 5) * block_stage_doubles();
  static_assert(kBlockStage == 0 || S == 32, "staging assumes one lane per scenario");
  static_assert(kBlockStage * sizeof(DestT) + 8 <= kBlockStageDest * sizeof(double), "destination slice does not fit");
  const unsigned long long total = static_cast<unsigned long long>(a.n_blocks) * a.units_here;
  while (true) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(a.ticket, 1ull);
    t = __shfl_sync(full, t, 0);
    if (t >= total) break;
    const int32_t b = static_cast<int32_t>(t / a.units_here);
    const int32_t u = a.first_unit + static_cast<int32_t>(t - static_cast<unsigned long long>(b) * a.units_here);
    const int4 b0 = __ldg(reinterpret_cast<const int4*>(a.blocks + b));
    const int4 b1 = __ldg(reinterpret_cast<const int4*>(a.blocks + b) + 1);
    const int32_t rows4[4] = {b0.x, b0.y, b0.z, b0.w};
    int32_t rows[R];
#pragma unroll
    for (int r = 0; r < R; ++r) rows[r] = rows4[r];
    const int32_t mbeg = b1.x, mend = b1.y;
    const int32_t sc0 = u * S;
    double* gbase = a.values + static_cast<int64_t>(sc0 >> 5) * a.nnz_factors * 32 + (sc0 & 31) + s;
    double* rowg[R];
    int64_t p[R];
    int32_t k[R], nl[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int32_t i = max(rows[r], 0);
      const int32_t lo = __ldg(a.row_ptr + i);
      rowg[r] = gbase + static_cast<int64_t>(lo) * 32;
      nl[r] = __ldg(a.diag + i) - lo;
      p[r] = a.pair_row_ptr[i];
      k[r] = 0;
    }

    for (int32_t t0 = mbeg; t0 < mend; t0 += 32) {
      int32_t my_d = 0, my_dd = 0, my_m = 0, my_ready = 0;
      uint32_t my_bits = 0;
      if (t0 + lane < mend) {
        const int2 mp = __ldg(reinterpret_cast<const int2*>(a.merged) + t0 + lane);
        my_d = mp.x;
        my_bits = static_cast<uint32_t>(mp.y);
        my_dd = __ldg(a.diag + my_d);
        my_m = __ldg(a.row_ptr + my_d + 1) - my_dd - 1;
        my_ready = ld_acquire_s32(a.flags + static_cast<int64_t>(my_d) * a.units + u) >= a.gen;
      }
      __syncwarp();
      const int32_t cnt = min(32, mend - t0);
      for (int32_t q = 0; q < cnt; ++q) {
        const int32_t dd = __shfl_sync(full, my_dd, q);
        const int32_t m = __shfl_sync(full, my_m, q);
        const uint32_t bits = __shfl_sync(full, my_bits, q);
        if (!__shfl_sync(full, my_ready, q)) {
          const int32_t d = __shfl_sync(full, my_d, q);
          const int32_t* f = a.flags + static_cast<int64_t>(d) * a.units + u;
          wait_flag(f, a.gen);
        }
        const double* ug = gbase + static_cast<int64_t>(dd) * 32;
        __syncwarp();  // the entry lanes' reductions of the previous pivot are issued (E > 1)
        // staged entries of this pivot row (diagonal included). A pivot that is a row of this very
        // block (bit 16) was just updated by this thread's own reductions: it is read with ordinary
        // ordered loads instead.
        const int32_t ns = (kBlockStage > 0 && !(bits & 0x10000u)) ? min(m + 1, kBlockStage) : 0;
        if (ns > 0) {
          const double* src = ug - s;  // warp-uniform start of the pivot row's block for this group
          for (int32_t t16 = lane; t16 < ns * 16; t16 += 32) cp_async_16(stage + t16 * 2, src + t16 * 2);
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (bits & (1u << r)) {
              const char* dsrc = reinterpret_cast<const char*>(dest + p[r]);
              const int32_t shift = static_cast<int32_t>(reinterpret_cast<uintptr_t>(dsrc) & 3);
              const int32_t words = (static_cast<int32_t>((ns - 1) * sizeof(DestT)) + shift + 3) >> 2;
              uint32_t* ddst = reinterpret_cast<uint32_t*>(stage + kBlockStage * 32 + r * kBlockStageDest);
              for (int32_t t4 = lane; t4 < words; t4 += 32) cp_async_4(ddst + t4, dsrc - shift + 4 * t4);
            }
          }
        }
        double nalpha[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          nalpha[r] = 0.0;
          if (bits & (1u << r)) nalpha[r] = ld_cg(rowg[r] + static_cast<int64_t>(k[r]) * 32);
        }
        double udd;
        if (ns > 0) {
          cp_async_commit_wait_all();
          __syncwarp();  // every lane's share of the copy has landed
          udd = stage[lane];
        } else {
          udd = ld_cg(ug);
        }
#pragma unroll
        for (int r = 0; r < R; ++r) nalpha[r] = -(nalpha[r] / udd);  // src/numeric.cpp:40; the sign is exact
        if (ns > 1) {
          const DestT* dl[R];
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const char* dbytes = reinterpret_cast<const char*>(stage + kBlockStage * 32 + r * kBlockStageDest);
            dl[r] = reinterpret_cast<const DestT*>(dbytes + (reinterpret_cast<uintptr_t>(dest + p[r]) & 3));
          }
#pragma unroll 4
          for (int32_t cs = 0; cs < ns - 1; ++cs) {
            const double uv = stage[(1 + cs) * 32 + lane];
#pragma unroll
            for (int r = 0; r < R; ++r) {
              if (bits & (1u << r)) red_add_f64(rowg[r] + static_cast<int64_t>(dl[r][cs]) * 32, __dmul_rn(nalpha[r], uv));  // src/numeric.cpp:44
            }
          }
        }
        if (ns > 0) __syncwarp();  // the stage may be overwritten by the next pivot
        int32_t c = e + max(ns - 1, 0);
        for (; c + (kUnroll - 1) * E < m; c += kUnroll * E) {
          // every load of the batch is issued before the first reduction (the reductions are
          // ordered asm statements: loads placed behind them would wait for nothing but still queue)
          double uv[kUnroll];
          int32_t ds[R][kUnroll];
#pragma unroll
          for (int j = 0; j < kUnroll; ++j) uv[j] = ld_cg(ug + static_cast<int64_t>(1 + c + j * E) * 32);
#pragma unroll
          for (int r = 0; r < R; ++r) {
#pragma unroll
            for (int j = 0; j < kUnroll; ++j) ds[r][j] = (bits & (1u << r)) ? dest[p[r] + c + j * E] : 0;
          }
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (bits & (1u << r)) {  // warp-uniform
#pragma unroll
              for (int j = 0; j < kUnroll; ++j) {
                red_add_f64(rowg[r] + static_cast<int64_t>(ds[r][j]) * 32, __dmul_rn(nalpha[r], uv[j]));  // src/numeric.cpp:44
              }
            }
          }
        }
        for (; c < m; c += E) {
          const double uv = ld_cg(ug + static_cast<int64_t>(1 + c) * 32);
          int32_t ds[R];
#pragma unroll
          for (int r = 0; r < R; ++r) ds[r] = (bits & (1u << r)) ? dest[p[r] + c] : 0;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (bits & (1u << r)) red_add_f64(rowg[r] + static_cast<int64_t>(ds[r]) * 32, __dmul_rn(nalpha[r], uv));
          }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (bits & (1u << r)) {
            if (e == 0) st_cg(rowg[r] + static_cast<int64_t>(k[r]) * 32, -nalpha[r]);  // l_id, src/numeric.cpp:41
            p[r] += m;
            ++k[r];
          }
        }
        if ((bits >> 8) & 0xffu) {  // rows whose last pivot this was: pivot check (src/numeric.cpp:48) and publication
          __syncwarp();
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (bits & (256u << r)) {
              if (e == 0 && fabs(ld_cg(rowg[r] + static_cast<int64_t>(nl[r]) * 32)) <= a.pivot_floor) {
                atomicMin(a.failed + sc0 + s, rows[r]);
              }
            }
          }
          __syncwarp();
          if (lane == 0) {
            __threadfence();
#pragma unroll
            for (int r = 0; r < R; ++r) {
              if (bits & (256u << r)) st_relaxed_s32(a.flags + static_cast<int64_t>(rows[r]) * a.units + u, a.gen);
            }
          }
        }
      }
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------ K3 batched
//
// lower_core / upper_core (src/trisolve.cpp:28-68) for 32 scenarios of one row per warp: lane =
// scenario, the row's entries are folded in ascending column order (the reference's order) by
// every lane on its own scenario, so each x is bit-identical to the CPU result. x itself is the
// ready flag (armed with the pending marker, as in the single-system sweeps). Units are claimed
// in (dependency level, group) order.
struct BTriArgs {
  int32_t n;        // rows of the matrix
  int32_t first;    // this launch claims positions [first, first + count) of the level order
  int32_t count;
  int32_t groups;
  const RowMeta* meta;   // level order; beg/end = the row's strict-lower (L) or strict-upper (U) entries
  const int32_t* col;
  const int32_t* diag;
  const double* values;  // [groups][nnz_factors][32]
  int64_t nnz_factors;
  const double* y;       // [groups][n][32]
  double* x;             // [groups][n][32], armed with the pending marker
  unsigned long long* ticket;
  int32_t* failed;       // upper: [padded batch] atomicMax, -1 = none
};

// U sweep: the dependency a row waits for LONGEST is normally its first entry (column i+1 or
// close to it is produced last), and the reference's ascending fold needs that term first. To keep
// the fold order and still have nothing but the subtraction chain behind the last arrival, the
// products of entries 1..kTriBuffered are computed ahead (each product is rounded on its own, as
// in src/trisolve.cpp:57) and parked in the warp's shared-memory buffer; when x of entry 0 lands
// the row costs one multiply and a chain of subtractions fed from shared memory.
//
// The U sweep is launched in two parts: the narrow leading levels (the top of the elimination
// tree: a long chain, a few rows wide, whose rows have the longest upper parts) with a buffer that
// parks a whole row, one CTA per SM; then the wide remainder with a small buffer and full
// occupancy.
// (Tried in round 2: the row's column indices fetched 32 at a time by the lanes and broadcast with shuffles, to take the
// dependent index load out of every gather — 2.5x SLOWER, L 5.3 ms and U 12.0 ms per step at C2 x 256 against 2.1 / 4.5:
// the shuffles are convergence points inside the unrolled load batches and the loads no longer issue back to back.)
#ifndef B200LU_TRI_CHUNK
#define B200LU_TRI_CHUNK 8
#endif
constexpr int kTriChunk = B200LU_TRI_CHUNK;  // entries whose loads are in flight together
constexpr int kTriBufferedWide = 32, kTriBufferedChain = 96;
constexpr size_t tri_upper_smem(int buffered, int warps = 8) { return static_cast<size_t>(warps) * buffered * 32 * sizeof(double); }

// (The L sweep is residency-sensitive — 2.10 / 2.57 / 4.29 ms per step with 444 / 296 / 148 CTAs at C2 x 256 — but forcing four or
// five CTAs per SM costs spills: 2.44 / 2.40 ms, and 1.48 / 1.24 ms against 1.09 at 32 scenarios. Three CTAs, 70 registers.)
template <bool kUpper, int kTriBuffered>
__global__ void __launch_bounds__(256)
btri_kernel(const BTriArgs a) {
  extern __shared__ __align__(16) double tri_smem[];
  const int lane = threadIdx.x & 31;
  const unsigned full = 0xffffffffu;
  const unsigned long long total = static_cast<unsigned long long>(a.count) * a.groups;
  double* pb = tri_smem + static_cast<size_t>(threadIdx.x >> 5) * kTriBuffered * 32 + lane;  // kUpper only
  // Static claim order: warp w takes units w, w + W, w + 2W, ... of the (level, group) order. One
  // atomic ticket per unit on a single L2 word would serialise the sweep (~2.5 ns each, measured
  // on the single-system sweeps); static order is deadlock-free for the same reason as the ticket
  // (the whole grid is resident and the owner of the lowest unfinished unit has nothing before it).
  const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * (blockDim.x >> 5);
  for (unsigned long long t = static_cast<unsigned long long>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
       t < total; t += stride) {
    const int32_t r = static_cast<int32_t>(t / a.groups);
    const int32_t g = static_cast<int32_t>(t - static_cast<unsigned long long>(r) * a.groups);
    const int4 m4 = __ldg(reinterpret_cast<const int4*>(a.meta) + a.first + r);
    const int32_t i = m4.x, beg = m4.y, end = m4.z;
    const double* vg = a.values + static_cast<int64_t>(g) * a.nnz_factors * 32 + lane;
    double* xg = a.x + static_cast<int64_t>(g) * a.n * 32 + lane;
    double acc = a.y[(static_cast<int64_t>(g) * a.n + i) * 32 + lane];
    double dval = 1.0;
    if (kUpper) dval = vg[static_cast<int64_t>(__ldg(a.diag + i)) * 32];

    // folds entries [k_begin, k_end) into acc in order
    auto run = [&](int32_t k_begin, int32_t k_end) {
      for (int32_t k = k_begin; k < k_end; k += kTriChunk) {
        double v[kTriChunk], xv[kTriChunk];
        const double* xp[kTriChunk];
#pragma unroll
        for (int j = 0; j < kTriChunk; ++j) {
          v[j] = 0.0;
          xv[j] = 0.0;
          xp[j] = xg;
          if (k + j < k_end) {
            v[j] = vg[static_cast<int64_t>(k + j) * 32];
            xp[j] = xg + static_cast<int64_t>(__ldg(a.col + k + j)) * 32;
            xv[j] = ld_l2(xp[j]);
          }
        }
#pragma unroll
        for (int j = 0; j < kTriChunk; ++j) {
          if (k + j < k_end) {  // warp-uniform
            unsigned backoff = 0;
            while (__any_sync(full, is_pending(xv[j]))) {
              if (backoff) __nanosleep(backoff);
              backoff = min(backoff + 32u, 256u);
              if (is_pending(xv[j])) xv[j] = ld_l2(xp[j]);
            }
            acc = sub_prod(acc, v[j], xv[j]);  // src/trisolve.cpp:38 / 57
          }
        }
      }
    };
    // parks the products of entries [k_begin, k_end) in the shared-memory buffer, walking the row
    // BACKWARDS: the far columns (long finished) first, the most recent dependencies last, so no
    // load is issued behind a wait
    auto park = [&](int32_t k_begin, int32_t k_end) {
      for (int32_t k = k_begin + ((k_end - k_begin - 1) / kTriChunk) * kTriChunk; k >= k_begin; k -= kTriChunk) {
        double v[kTriChunk], xv[kTriChunk];
        const double* xp[kTriChunk];
#pragma unroll
        for (int j = 0; j < kTriChunk; ++j) {
          v[j] = 0.0;
          xv[j] = 0.0;
          xp[j] = xg;
          if (k + j < k_end) {
            v[j] = vg[static_cast<int64_t>(k + j) * 32];
            xp[j] = xg + static_cast<int64_t>(__ldg(a.col + k + j)) * 32;
            xv[j] = ld_l2(xp[j]);
          }
        }
#pragma unroll
        for (int j = kTriChunk - 1; j >= 0; --j) {
          if (k + j < k_end) {  // warp-uniform
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
    };

    if (!kUpper) {
      run(beg, end);
    } else if (beg < end) {
      const double v0 = vg[static_cast<int64_t>(beg) * 32];
      const double* xp0 = xg + static_cast<int64_t>(__ldg(a.col + beg)) * 32;
      const int32_t parked_end = min(end, beg + 1 + kTriBuffered);
      if (parked_end > beg + 1) park(beg + 1, parked_end);
      double x0 = ld_l2(xp0);
      while (__any_sync(full, is_pending(x0))) {
        if (is_pending(x0)) x0 = ld_l2(xp0);
      }
      acc = sub_prod(acc, v0, x0);
      {
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
      }
      run(parked_end, end);
    }
    if (kUpper) {
      if (dval == 0.0) atomicMax(a.failed + g * 32 + lane, i);  // src/trisolve.cpp:60-66
      acc = acc / dval;
    }
    publish(xg + static_cast<int64_t>(i) * 32, acc);
  }
}

// solve_system prologue (src/trisolve.cpp:98-105) in the interleaved layout:
// w[g][p(i)][lane] = D_r[i] * b[g][i][lane]; arms the two sweep buffers.
__global__ void __launch_bounds__(256)
bpermute_in_kernel(int32_t n, int32_t groups, const int32_t* __restrict__ p, const double* __restrict__ row_scale,
                   const double* __restrict__ b, double* __restrict__ w, double* __restrict__ t1,
                   double* __restrict__ t2) {
  const double pending = __longlong_as_double(static_cast<long long>(kPendingBits));
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (warp >= static_cast<int64_t>(n) * groups) return;
  const int64_t g = warp / n, i = warp - g * n;
  double v = b[warp * 32 + lane];
  if (row_scale != nullptr) v = __dmul_rn(row_scale[i], v);
  w[(g * n + p[i]) * 32 + lane] = v;
  t1[warp * 32 + lane] = pending;
  t2[warp * 32 + lane] = pending;
}

// solve_system epilogue (src/trisolve.cpp:110-118): x[g][j][lane] = D_c[j] * t[g][pq(j)][lane].
__global__ void __launch_bounds__(256)
bpermute_out_kernel(int32_t n, int32_t groups, const int32_t* __restrict__ pq, const double* __restrict__ col_scale,
                    const double* __restrict__ t, double* __restrict__ x) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (warp >= static_cast<int64_t>(n) * groups) return;
  const int64_t g = warp / n, j = warp - g * n;
  double v = t[(g * n + pq[j]) * 32 + lane];
  if (col_scale != nullptr) v = __dmul_rn(col_scale[j], v);
  x[warp * 32 + lane] = v;
}

__global__ void __launch_bounds__(256)
bfill_pending_kernel(int64_t count, double* __restrict__ x) {
  const double pending = __longlong_as_double(static_cast<long long>(kPendingBits));
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < count) x[i] = pending;
}

// ------------------------------------------------------------------ K4 batched
//
// Per-scenario reductions: the grid is (kBatchParts, groups); warp q of a group walks a
// contiguous block of rows with lane = scenario, each lane summing its scenario's terms in row
// order; the per-warp partials are folded in warp order by bfinish_kernel. Fixed geometry ->
// results are reproducible run to run (same argument as dot_kernel in refine.cuh: the
// reference's serial sum, src/sparse.cpp:271-275, cannot be reproduced by a parallel one).
constexpr int kBatchPartBlocks = 64;                       // blocks per group
constexpr int kBatchParts = kBatchPartBlocks * 8;          // warps (partials) per group

__device__ __forceinline__ void brow_range(int32_t n, int32_t& i0, int32_t& i1) {
  const int32_t part = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int32_t per = (n + kBatchParts - 1) / kBatchParts;
  i0 = min(n, part * per);
  i1 = min(n, i0 + per);
}

// r = b - A x (spmv, src/sparse.cpp:135-141: left-to-right accumulation per row), one warp per (row, group): the
// gathers of a row are dependent loads, so the rows must run side by side, not one after the other.
__global__ void __launch_bounds__(256)
bresidual_rows_kernel(int32_t n, int32_t groups, int64_t nnz_source, const int32_t* __restrict__ row_ptr,
                      const int32_t* __restrict__ col, const double* __restrict__ a_int, const double* __restrict__ x,
                      const double* __restrict__ b, double* __restrict__ r) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (warp >= static_cast<int64_t>(n) * groups) return;
  const int64_t g = warp / n, i = warp - g * n;
  const double* ag = a_int + g * nnz_source * 32 + lane;
  const double* xg = x + g * n * 32 + lane;
  double acc = 0.0;
  for (int32_t k = __ldg(row_ptr + i); k < __ldg(row_ptr + i + 1); ++k) {
    acc = add_prod(acc, ag[static_cast<int64_t>(k) * 32], xg[static_cast<int64_t>(__ldg(col + k)) * 32]);
  }
  r[warp * 32 + lane] = __dsub_rn(b[warp * 32 + lane], acc);
}

// Partial sums of r^2 and b^2 (relative_residual, src/sparse.cpp:283-288) in the fixed geometry of the
// per-scenario reductions: every warp folds its block of rows in row order (loads of 8 rows in flight, the
// additions in order), so the sums are the ones the fused kernel of round 1 produced, bit for bit.
__global__ void __launch_bounds__(256)
bsumsq2_kernel(int32_t n, const double* __restrict__ r, const double* __restrict__ b, double* __restrict__ partials) {
  const int lane = threadIdx.x & 31;
  const int64_t g = blockIdx.y;
  int32_t i0, i1;
  brow_range(n, i0, i1);
  const double* rg = r + g * n * 32 + lane;
  const double* bg = b + g * n * 32 + lane;
  double s0 = 0.0, s1 = 0.0;
  int32_t i = i0;
  for (; i + 8 <= i1; i += 8) {
    double rv[8], bv[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      rv[q] = rg[static_cast<int64_t>(i + q) * 32];
      bv[q] = bg[static_cast<int64_t>(i + q) * 32];
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      s0 = add_prod(s0, rv[q], rv[q]);
      s1 = add_prod(s1, bv[q], bv[q]);
    }
  }
  for (; i < i1; ++i) {
    const double ri = rg[static_cast<int64_t>(i) * 32], bi = bg[static_cast<int64_t>(i) * 32];
    s0 = add_prod(s0, ri, ri);
    s1 = add_prod(s1, bi, bi);
  }
  const int64_t part = blockIdx.x * 8 + (threadIdx.x >> 5);
  partials[((g * 2 + 0) * kBatchParts + part) * 32 + lane] = s0;
  partials[((g * 2 + 1) * kBatchParts + part) * 32 + lane] = s1;
}

// y = A x
__global__ void __launch_bounds__(256)
bspmv_kernel(int32_t n, int32_t groups, int64_t nnz_source, const int32_t* __restrict__ row_ptr,
             const int32_t* __restrict__ col, const double* __restrict__ a_int, const double* __restrict__ x,
             double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (warp >= static_cast<int64_t>(n) * groups) return;
  const int64_t g = warp / n, i = warp - g * n;
  const double* ag = a_int + g * nnz_source * 32 + lane;
  const double* xg = x + g * n * 32 + lane;
  double acc = 0.0;
  for (int32_t k = __ldg(row_ptr + i); k < __ldg(row_ptr + i + 1); ++k) {
    acc = add_prod(acc, ag[static_cast<int64_t>(k) * 32], xg[static_cast<int64_t>(__ldg(col + k)) * 32]);
  }
  y[warp * 32 + lane] = acc;
}

__global__ void __launch_bounds__(256)
bdot_kernel(int32_t n, const double* __restrict__ u, const double* __restrict__ v, double* __restrict__ partials) {
  const int lane = threadIdx.x & 31;
  const int64_t g = blockIdx.y;
  int32_t i0, i1;
  brow_range(n, i0, i1);
  const double* ug = u + g * n * 32 + lane;
  const double* vg = v + g * n * 32 + lane;
  double s0 = 0.0;
  int32_t i = i0;
  for (; i + 8 <= i1; i += 8) {  // 8 rows of loads in flight, the additions in row order
    double uv[8], vv[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      uv[q] = ug[static_cast<int64_t>(i + q) * 32];
      vv[q] = vg[static_cast<int64_t>(i + q) * 32];
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) s0 = add_prod(s0, uv[q], vv[q]);
  }
  for (; i < i1; ++i) s0 = add_prod(s0, ug[static_cast<int64_t>(i) * 32], vg[static_cast<int64_t>(i) * 32]);
  const int64_t part = blockIdx.x * 8 + (threadIdx.x >> 5);
  partials[((g * 2 + 0) * kBatchParts + part) * 32 + lane] = s0;
}

// out[q][g*32+lane] = sum over parts, in part order; count = 1 or 2 running sums
__global__ void __launch_bounds__(32)
bfinish_kernel(int32_t count, int32_t padded, const double* __restrict__ partials, double* __restrict__ out) {
  const int lane = threadIdx.x;
  const int64_t g = blockIdx.x;
  for (int q = 0; q < count; ++q) {
    const double* pp = partials + (g * 2 + q) * kBatchParts * 32 + lane;
    double s = 0.0;
    static_assert(kBatchParts % 16 == 0, "unrolled fold");
    for (int part = 0; part < kBatchParts; part += 16) {  // 16 loads in flight, folded in part order
      double pv[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) pv[t] = pp[static_cast<int64_t>(part + t) * 32];
#pragma unroll
      for (int t = 0; t < 16; ++t) s += pv[t];
    }
    out[static_cast<int64_t>(q) * padded + g * 32 + lane] = s;
  }
}

// One Gram-Schmidt projection step of cgs2_orthonormalize (src/refine.cpp:13-17) per scenario:
// h = hs[sc]; coef[sc] += h (row 0 only); w -= h * q.
__global__ void __launch_bounds__(256)
bproject_out_kernel(int32_t n, int32_t groups, const double* __restrict__ hs, double* __restrict__ coef,
                    const double* __restrict__ q, double* __restrict__ w) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (warp >= static_cast<int64_t>(n) * groups) return;
  const int64_t g = warp / n, i = warp - g * n;
  const double h = hs[g * 32 + lane];
  if (i == 0) coef[g * 32 + lane] = __dadd_rn(coef[g * 32 + lane], h);
  w[warp * 32 + lane] = add_prod(w[warp * 32 + lane], -h, q[warp * 32 + lane]);
}

// y += alpha[sc] * x (axpy, src/sparse.cpp:279-281)
__global__ void __launch_bounds__(256)
baxpy_kernel(int32_t n, int32_t groups, const double* __restrict__ alpha, const double* __restrict__ x,
             double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (warp >= static_cast<int64_t>(n) * groups) return;
  const int64_t g = warp / n;
  y[warp * 32 + lane] = add_prod(y[warp * 32 + lane], alpha[g * 32 + lane], x[warp * 32 + lane]);
}

// out = in / s[sc]
__global__ void __launch_bounds__(256)
bdivide_kernel(int32_t n, int32_t groups, const double* __restrict__ s, const double* __restrict__ in,
               double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (warp >= static_cast<int64_t>(n) * groups) return;
  const int64_t g = warp / n;
  out[warp * 32 + lane] = in[warp * 32 + lane] / s[g * 32 + lane];
}

// dst = src where mask[sc] != 0
__global__ void __launch_bounds__(256)
bcopy_masked_kernel(int32_t n, int32_t groups, const double* __restrict__ mask, const double* __restrict__ src,
                    double* __restrict__ dst) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (warp >= static_cast<int64_t>(n) * groups) return;
  const int64_t g = warp / n;
  if (mask[g * 32 + lane] != 0.0) dst[warp * 32 + lane] = src[warp * 32 + lane];
}

}  // namespace b200lu
