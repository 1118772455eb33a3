// K3 triangular solves and the permute/scale stages of solve_system.
#pragma once

#include <cooperative_groups.h>

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
  int32_t n;              // claim positions
  int32_t n_publish;      // positions below this publish x[row]; the rest are "head part" tasks of
                          // tail rows: their entries are listed in part_k, the sum goes to partial[row]
  const int32_t* part_k;  // entry indices of the head-part tasks
  double* partial;        // L head sweep only: partial sums handed to the tail kernel
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
template <bool kUpper, bool kDescending, bool kStatic>
__global__ void __launch_bounds__(256)
tri_kernel(const TriArgs a) {
  const int lane = threadIdx.x & 31;
  const unsigned full = 0xffffffffu;
  int32_t seen = 0;  // last value read from the finished-rows counter
  // Claim order. kStatic == false: an atomic ticket per row plus a finished-rows counter that
  // throttles far-ahead rows (wait_for_start) — needed when the sweep contains the long narrow
  // part of the DAG (strict order). kStatic == true (head sweeps of the default mode, whose DAG
  // is wide and shallow): warp w simply takes positions w, w + W, w + 2W, ... — the ticket and the
  // counter are single L2 words, and one atomic per row on each of them serialises the sweep
  // (measured: ~0.6 ms of a 0.65 ms head sweep at C3). Static order is deadlock-free for the same
  // reason as the ticket: the owner of the lowest unfinished position has nothing left before it.
  const int32_t stride = kStatic ? static_cast<int32_t>((gridDim.x * blockDim.x) >> 5) : 1;
  int32_t r = kStatic ? static_cast<int32_t>((blockIdx.x * blockDim.x + threadIdx.x) >> 5) : 0;
  for (;; r += stride) {
    if (!kStatic) {
      if (lane == 0) r = atomicAdd(a.counter, 1);
      r = __shfl_sync(full, r, 0);
    }
    if (r >= a.n) break;
    const int4 m4 = __ldg(reinterpret_cast<const int4*>(a.meta) + r);
    const int32_t i = m4.x, beg = m4.y, end = m4.z;
    double acc = a.y[i];
    double dval = 1.0;
    if (kUpper) dval = a.values[__ldg(a.diag + i)];
    if (!kStatic) wait_for_start(a.finished, m4.w, lane, seen);

    // entry handled by this lane in chunk c (chunks and lanes walk the row in fold order); the
    // head-part tasks of tail rows list their entries explicitly
    const bool listed = r >= a.n_publish;
    auto entry = [&](int32_t c) {
      const int32_t e = kDescending ? end - 1 - (c * 32 + lane) : beg + c * 32 + lane;
      return listed ? __ldg(a.part_k + e) : e;
    };
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
      __syncwarp(full);  // converged before the collectives below (keeps them inline)
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
        __syncwarp(full);
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
      if (r < a.n_publish) {
        publish(a.x + i, acc);
      } else {
        a.partial[i] = acc;  // read by tail_kernel after this kernel has finished
      }
      if (!kStatic) red_add_s32(a.finished, 1);
    }
  }
}

// ------------------------------------------------------------------ on-chip tail
//
// The narrow end of the sweep's dependency DAG (schedule.hpp, TailPlan) inside ONE thread-block
// cluster: every CTA of the cluster keeps a full copy of the tail rows' x in its shared memory,
// armed with the pending marker; a finished row is written into all copies through distributed
// shared memory and its dependents spin on their LOCAL copy — a hand-off costs a DSMEM store
// (~0.1 us) instead of an L2 round trip and a half (~0.6 us). The warps of the whole cluster take
// tail rows round-robin in topological order and run ahead of themselves: while row t is processed
// the loads of the warp's next rows (record three rows ahead, entry records two, values one) are
// already in flight, so nothing on the critical path waits for global memory. Per row:
//   1. every entry except the one that multiplies the dependency expected LAST is gathered from
//      shared memory (lanes keep private partial sums, reduced by a fixed shuffle tree);
//   2. only then the warp waits for that last dependency and applies its single term — one
//      shared-memory read, one multiply, one subtract (and the scaling by 1/u_ii) per hand-off.
// Columns outside the tail were summed earlier by the head sweep ("head part" tasks, L sweep) or
// do not exist (U sweep: the tail is closed). The summation order is fixed, hence deterministic,
// but it is not the reference's serial order, and the U diagonal is applied as a reciprocal:
// this kernel is the default mode only; B200LU_FLAG_STRICT_ORDER runs the whole sweep through
// tri_kernel instead.
struct TailArgs {
  int32_t rows;
  const TailRow* row;
  const TailEntry* entries;
  const double* values;
  const double* init;       // U: y; L: partial sums from the head sweep
  double* x;                // global x, written for the tail rows
  int32_t* failed_row;      // upper only
};

constexpr int kTailThreads = 512;
constexpr int kTailBlock = 4;  // 32-entry chunks whose loads are issued together

template <bool kUpper>
__global__ void __launch_bounds__(kTailThreads, 1)
tail_kernel(const TailArgs a) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int csize = static_cast<int>(cluster.num_blocks());
  extern __shared__ double xs[];
  volatile double* vx = xs;
  const double pending = __longlong_as_double(static_cast<long long>(kPendingBits));
  for (int32_t t = threadIdx.x; t < a.rows; t += kTailThreads) xs[t] = pending;
  cluster.sync();  // every copy is armed before anyone publishes into it

  const int lane = threadIdx.x & 31;
  const int w = static_cast<int>(cluster.block_rank()) * (kTailThreads / 32) + (threadIdx.x >> 5);
  const int kWarps = csize * (kTailThreads / 32);  // warps of the whole cluster
  const unsigned full = 0xffffffffu;
  // this lane's destination copy when publishing (lane r writes into CTA r's shared memory)
  volatile double* remote = lane < csize ? cluster.map_shared_rank(xs, lane) : nullptr;

  struct Rec {  // TailRow as two 16-byte loads
    int4 a, b;
  };
  struct Ent {  // first block of a row's entry records
    int2 e[kTailBlock];
  };
  struct Data {  // everything row t needs from global memory
    double init, scale, v_last;
    double v[kTailBlock];
    int32_t src[kTailBlock];
  };
  // Three pipeline stages, each a set of loads whose addresses come from the stage before:
  // record (3 rows ahead) -> entry records (2 ahead) -> values and scalars (1 ahead).
  auto load_rec = [&](int32_t t) {
    Rec r{make_int4(0, 0, 0, -1), make_int4(0, 0, 0, 0)};
    if (t < a.rows) {
      const int4* p = reinterpret_cast<const int4*>(a.row + t);
      r.a = ldg_pinned(p);
      r.b = ldg_pinned(p + 1);
    }
    return r;
  };
  auto load_ent = [&](const Rec& r) {
    Ent en;
#pragma unroll
    for (int u = 0; u < kTailBlock; ++u) {
      const int32_t e = r.a.y + u * 32 + lane;
      en.e[u] = make_int2(0, -1);
      if (e < r.a.z) en.e[u] = ldg_pinned(reinterpret_cast<const int2*>(a.entries) + e);
    }
    return en;
  };
  auto load_data = [&](const Rec& r, const Ent& en, bool valid) {
    Data d;
    d.init = 0.0;
    d.scale = 1.0;
    d.v_last = 0.0;
    if (valid) {
      d.init = ld_pinned(a.init + r.a.x);
      if (kUpper) d.scale = ld_pinned(a.values + r.b.y);  // u_ii (turned into 1/u_ii below)
      if (r.a.w >= 0) d.v_last = ld_pinned(a.values + r.b.x);
    }
#pragma unroll
    for (int u = 0; u < kTailBlock; ++u) {
      d.src[u] = en.e[u].y;
      d.v[u] = 0.0;
      if (en.e[u].y >= 0) d.v[u] = ld_pinned(a.values + en.e[u].x);
    }
    return d;
  };
  auto fetch = [&](int32_t s) {
    double xv = vx[s];
    while (is_pending(xv)) xv = vx[s];
    return xv;
  };

  Rec rec0 = load_rec(w), rec1 = load_rec(w + kWarps), rec2 = load_rec(w + 2 * kWarps);
  Ent ent0 = load_ent(rec0);
  Ent ent1 = load_ent(rec1);
  Data cur = load_data(rec0, ent0, w < a.rows);
  for (int32_t t = w; t < a.rows; t += kWarps) {
    const Rec rec3 = load_rec(t + 3 * kWarps);
    const Ent ent2 = load_ent(rec2);
    const Data nxt = load_data(rec1, ent1, t + kWarps < a.rows);

    const int32_t i = rec0.a.x, e0 = rec0.a.y, e1 = rec0.a.z, last = rec0.a.w;
    // 1. everything but the last dependency. The warp first waits as a whole (one broadcast
    // shared-memory read per poll) for the dependency expected second to last; the per-lane
    // gathers below then find their values ready instead of spinning divergently.
    const int32_t last2 = rec0.b.z;
    if (last2 >= 0) {
      while (is_pending(vx[last2])) {}
    }
    // Gather with warp-uniform control flow: every lane takes part in every poll round. (Lanes
    // spinning on their own in a divergent loop cost ~0.8 us per hand-off on a banded chain.)
    auto gather = [&](const double (&v)[kTailBlock], const int32_t (&sidx)[kTailBlock], double sum) {
      double xv[kTailBlock];
#pragma unroll
      for (int u = 0; u < kTailBlock; ++u) xv[u] = sidx[u] >= 0 ? vx[sidx[u]] : 0.0;
      while (__any_sync(full, is_pending(xv[0]) || is_pending(xv[1]) || is_pending(xv[2]) || is_pending(xv[3]))) {
#pragma unroll
        for (int u = 0; u < kTailBlock; ++u) {
          if (is_pending(xv[u])) xv[u] = vx[sidx[u]];
        }
      }
#pragma unroll
      for (int u = 0; u < kTailBlock; ++u) sum = __dadd_rn(sum, __dmul_rn(v[u], xv[u]));
      return sum;
    };
    static_assert(kTailBlock == 4, "gather() spells out four poll slots");
    double part = gather(cur.v, cur.src, 0.0);
    for (int32_t base = e0 + 32 * kTailBlock; base < e1; base += 32 * kTailBlock) {  // rows longer than a block
      double v[kTailBlock];
      int32_t sidx[kTailBlock];
#pragma unroll
      for (int u = 0; u < kTailBlock; ++u) {
        const int32_t e = base + u * 32 + lane;
        v[u] = 0.0;
        sidx[u] = -1;
        if (e < e1) {
          const int2 ent = __ldg(reinterpret_cast<const int2*>(a.entries) + e);
          v[u] = a.values[ent.x];
          sidx[u] = ent.y;
        }
      }
      part = gather(v, sidx, part);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part = __dadd_rn(part, __shfl_xor_sync(full, part, o));
    double acc = __dsub_rn(cur.init, part);
    double scale = 1.0;
    if (kUpper) {
      if (lane == 0 && cur.scale == 0.0) atomicMax(a.failed_row, i);
      scale = 1.0 / cur.scale;
    }
    // 2. the hand-off: one term behind the dependency that finishes last
    if (last >= 0) acc = __dsub_rn(acc, __dmul_rn(cur.v_last, fetch(last)));
    if (kUpper) acc = __dmul_rn(acc, scale);
    if (is_pending(acc)) acc = __longlong_as_double(static_cast<long long>(kCanonicalNaN));
    if (remote != nullptr) remote[t] = acc;  // one DSMEM store per copy, issued by csize lanes at once
    if (lane == 0) a.x[i] = acc;
    rec0 = rec1;
    rec1 = rec2;
    rec2 = rec3;
    ent1 = ent2;
    cur = nxt;
  }
  cluster.sync();  // no CTA may exit while others can still store into its shared memory
}

}  // namespace b200lu
