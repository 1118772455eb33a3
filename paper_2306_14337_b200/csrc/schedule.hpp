// Host-side schedule derivation: everything the device kernels need beyond the
// reference's SymbolicFactors, computed once per handle in O(nnz(L+U)).
//
// The reference executes rows through SyncFreeScheduler (include/rlu/schedule.hpp:34-200):
// one ready flag per row, rows claimed in ascending order. On the device the claim order is
// the dependency LEVEL order (a topological order of the same DAG), so a claimed row's
// dependencies are always finished or held by a resident worker.
#pragma once

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "b200lu.h"

namespace b200lu {

// pattern_equal's comparison (src/numeric.cpp:15, src/sparse.cpp) runs on EVERY scatter, as in the reference; at
// n = 1.6 M that is 85 MB of indices per call — 8 ms single-threaded, a third of the whole device step — so large
// comparisons are split over a few persistent host threads (created on first use, parked on a condition variable
// between calls: dispatch costs tens of microseconds, not a thread spawn per call).
class CompareBytesPool {
 public:
  static CompareBytesPool& instance() {
    static CompareBytesPool pool;
    return pool;
  }
  bool same(const void* a, const void* b, size_t bytes) {
    constexpr size_t kChunk = size_t{1} << 20;
    const size_t parts = std::min<size_t>(workers_.size() + 1, bytes / kChunk);
    if (parts < 2) return std::memcmp(a, b, bytes) == 0;
    std::lock_guard<std::mutex> call_lock(call_);  // one comparison at a time
    const size_t step = (bytes + parts - 1) / parts;
    {
      std::lock_guard<std::mutex> lk(m_);
      a_ = static_cast<const char*>(a);
      b_ = static_cast<const char*>(b);
      bytes_ = bytes;
      step_ = step;
      parts_ = parts;
      pending_ = parts - 1;
      differ_ = false;
      ++generation_;
    }
    cv_.notify_all();
    if (std::memcmp(a_, b_, std::min(step, bytes)) != 0) differ_ = true;  // part 0 on the calling thread
    std::unique_lock<std::mutex> lk(m_);
    done_.wait(lk, [this] { return pending_ == 0; });
    return !differ_;
  }

 private:
  CompareBytesPool() {
    const unsigned hw = std::max(2u, std::thread::hardware_concurrency());
    const unsigned n = std::min(7u, hw - 1);
    for (unsigned t = 0; t < n; ++t) workers_.emplace_back([this, t] { run(t + 1); });
  }
  ~CompareBytesPool() {
    {
      std::lock_guard<std::mutex> lk(m_);
      stop_ = true;
      ++generation_;
    }
    cv_.notify_all();
    for (std::thread& th : workers_) th.join();
  }
  void run(size_t part) {
    uint64_t seen = 0;
    while (true) {
      std::unique_lock<std::mutex> lk(m_);
      cv_.wait(lk, [&] { return generation_ != seen; });
      seen = generation_;
      if (stop_) return;
      if (part >= parts_) continue;
      const char *a = a_, *b = b_;
      const size_t lo = part * step_, hi = std::min(bytes_, lo + step_);
      lk.unlock();
      const bool diff = lo < hi && std::memcmp(a + lo, b + lo, hi - lo) != 0;
      lk.lock();
      if (diff) differ_ = true;
      if (--pending_ == 0) done_.notify_one();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex m_, call_;
  std::condition_variable cv_, done_;
  const char *a_ = nullptr, *b_ = nullptr;
  size_t bytes_ = 0, step_ = 0, parts_ = 0, pending_ = 0;
  uint64_t generation_ = 0;
  std::atomic<bool> differ_{false};
  bool stop_ = false;
};
inline bool same_bytes(const void* a, const void* b, size_t bytes) { return CompareBytesPool::instance().same(a, b, bytes); }

// One record per claim position, so a worker learns everything about its row from one 16-byte
// load instead of a chain of dependent index loads.
struct RowMeta {
  int32_t row;    // row index in the permuted matrix
  int32_t beg;    // first entry the worker touches
  int32_t end;    // one past the last entry
  int32_t start;  // the row may start once this many rows of the sweep have finished
};

// The narrow end of a sweep's dependency DAG — the trailing levels of the L sweep, the leading
// levels of the U sweep, every one narrower than `tail_width` rows — is a long chain with almost no
// parallelism: at C3 1,193 of the 1,480 levels hold 3 % of the rows. Crossing L2 once per level
// costs ~0.6 us; inside one SM a hand-off through shared memory costs a few tens of
// nanoseconds. A TailPlan describes that part of a sweep for tail_kernel (trisolve.cuh): the tail
// rows in a topological order and, for each, the entries whose columns are tail rows too. Entries
// of a tail row whose columns are head rows (L sweep only; the U tail is closed) are summed
// earlier by the head sweep, in parallel with everything else ("head part" tasks); the tail
// kernel continues from that partial sum.
struct TailRow {       // one 32-byte record per tail position
  int32_t row;         // row index
  int32_t e0, e1;      // its entries in TailPlan::entries (all have tail columns; `last` excluded)
  int32_t last;        // tail position of the dependency expected to finish last (-1: none)
  int32_t last_k;      // index into values[] of the entry that multiplies it
  int32_t diag_k;      // index into values[] of the row's diagonal (U sweep)
  int32_t last2;       // tail position of the dependency expected second to last (-1: none)
  int32_t pad1;
};
struct TailEntry {
  int32_t k;           // index into values[]
  int32_t src;         // tail position of the entry's column
};

struct TailPlan {
  int64_t rows = 0;                 // 0: no split, the whole sweep runs in the sync-free kernel
  int64_t levels = 0;               // dependency levels inside the tail
  std::vector<TailRow> row;         // per tail position, a topological order of the tail rows
  std::vector<TailEntry> entries;   // tail-column entries of the tail rows
  std::vector<RowMeta> head_meta;   // claim records of the head sweep, then one "head part" task per tail row
  std::vector<int32_t> head_part_k; // entries of those tasks: indices into values[]/col[] (head columns only)
  int64_t head_publish = 0;         // claim positions below this publish x; the rest store partial sums
};

struct Schedule {
  int64_t n = 0, nnz = 0, nnz_lower = 0, update_pairs = 0;
  int64_t lower_levels = 0, upper_levels = 0, max_row_len = 0;
  int64_t upper_head_levels = 0;  // depth of the U sweep's head DAG once the tail has run
  std::vector<int32_t> row_ptr, col, diag;  // int32 image of the combined pattern
  // Rows by ascending L-level (ties by index), split by row length into the rows a single warp
  // slot holds and the wide rows that need the per-CTA wide slot.
  std::vector<int32_t> small_rows, big_rows;
  std::vector<int32_t> trivial_rows;  // rows without a strict-lower entry: published by the scatter pass
  std::vector<int32_t> lower_order;  // all rows, L-level order
  std::vector<int32_t> upper_order;  // all rows, U-level order
  std::vector<int64_t> pair_row_ptr;  // n+1: first update pair of each row
  std::vector<int32_t> lower_level, upper_level;  // per row
  std::vector<int32_t> lower_width, upper_width;  // rows per level
  std::vector<RowMeta> lower_meta, upper_meta;    // triangular sweeps, per claim position
  // Split sweeps (default mode): the narrow end of the dependency DAG runs inside one CTA.
  TailPlan lower_tail, upper_tail;
};

// Start thresholds of a triangular sweep. Row at claim position r may begin once `start`
// rows have finished, chosen so that it is at most `lookahead_levels` dependency levels (and
// between `min_window` and `max_window` rows) ahead of the completed frontier: close enough
// that the values it then spins on are about to be produced, far enough that it has consumed
// its long-finished entries before its last dependency arrives. The threshold is a throttle
// on L2 polling only — ordering is enforced by the values themselves — and start <= r keeps it
// deadlock-free: the lowest unfinished row in claim order always finds its threshold met.
inline void fill_start_thresholds(std::vector<RowMeta>& meta, const std::vector<int32_t>& level,
                                  const std::vector<int32_t>& width, int64_t lookahead_levels,
                                  int64_t min_window, int64_t max_window) {
  const int64_t n = static_cast<int64_t>(meta.size());
  const int64_t levels = static_cast<int64_t>(width.size());
  std::vector<int64_t> level_begin(static_cast<size_t>(levels) + 1, 0);  // rows in levels < l
  for (int64_t l = 0; l < levels; ++l) level_begin[l + 1] = level_begin[l] + width[l];
  for (int64_t r = 0; r < n; ++r) {
    const int64_t l = level[meta[r].row];
    const int64_t by_level = level_begin[std::max<int64_t>(0, l - lookahead_levels)];
    int64_t start = std::max(by_level, r - max_window);
    start = std::min(start, r - min_window);
    meta[r].start = static_cast<int32_t>(std::max<int64_t>(0, start));
  }
}

struct ScheduleTuning {
  int64_t small_slot = 512;
  int64_t tail_width = 32;       // levels narrower than this belong to the on-chip tail
  int64_t tail_capacity = 24576; // rows whose x fit in one CTA's shared memory
  int64_t tail_min_levels = 16;  // do not split for a tail shorter than this
  int64_t solve_lookahead_levels = 48;
  int64_t solve_min_window = 64;
  int64_t solve_max_window = 1 << 20;
};

// Picks the on-chip tail of a sweep from the profile of a per-row "depth" (for the L sweep the
// dependency level; for the U sweep the height, see build_schedule): the rows whose depth lies in
// the maximal top run of depth values that are each shared by fewer than tail_width rows, capped
// by the row capacity. Returns the smallest depth that belongs to the tail (or depth_count when
// there is no worthwhile tail).
inline int64_t pick_tail_cut(const std::vector<int32_t>& depth_width, const ScheduleTuning& tune, int64_t* tail_rows) {
  const int64_t levels = static_cast<int64_t>(depth_width.size());
  int64_t cut = levels, rows = 0;
  for (int64_t l = levels - 1; l >= 0; --l) {
    if (depth_width[l] >= tune.tail_width || rows + depth_width[l] > tune.tail_capacity) break;
    rows += depth_width[l];
    cut = l;
  }
  if (levels - cut < tune.tail_min_levels && cut > 0) {  // too short to be worth a split
    cut = levels;
    rows = 0;
  }
  *tail_rows = rows;
  return cut;
}

// Builds the TailPlan of one sweep from its two row sets: `tail_order` (a topological order of
// the tail rows) and `head_order` (the head rows by their own dependency level, `head_level`
// indexed by row, `head_width` per level). Entries of row i are [ebeg(i), eend(i)) in values/col.
// With `head_part_tasks` (L sweep: head before tail) every tail row also gets a task in the head
// sweep that sums its head-column entries and stores the partial sum.
template <class EBeg, class EEnd>
inline void make_tail_plan(const Schedule& S, const ScheduleTuning& tune, const std::vector<int32_t>& tail_order,
                           const std::vector<int32_t>& head_order, std::vector<int32_t> head_level,
                           std::vector<int32_t> head_width, bool head_part_tasks, EBeg ebeg, EEnd eend,
                           TailPlan& plan) {
  const int64_t n = S.n;
  const int64_t tail_rows = static_cast<int64_t>(tail_order.size());
  plan.rows = tail_rows;
  std::vector<int32_t> tail_index(n, -1);  // row -> tail position
  for (int64_t t = 0; t < tail_rows; ++t) tail_index[tail_order[t]] = static_cast<int32_t>(t);
  plan.row.assign(tail_rows, TailRow{});
  plan.entries.clear();
  for (int64_t t = 0; t < tail_rows; ++t) {
    const int32_t i = tail_order[t];
    TailRow& tr = plan.row[t];
    tr.row = i;
    tr.diag_k = S.diag[i];
    tr.last = -1;
    tr.last_k = 0;
    for (int32_t k = ebeg(i); k < eend(i); ++k) {  // the dependency that sits latest in the tail order
      const int32_t ti = tail_index[S.col[k]];
      if (ti > tr.last) {
        tr.last = ti;
        tr.last_k = k;
      }
    }
    tr.e0 = static_cast<int32_t>(plan.entries.size());
    tr.last2 = -1;
    for (int32_t k = ebeg(i); k < eend(i); ++k) {
      const int32_t ti = tail_index[S.col[k]];
      if (ti >= 0 && ti != tr.last) {
        plan.entries.push_back(TailEntry{k, ti});
        tr.last2 = std::max(tr.last2, ti);
      }
    }
    tr.e1 = static_cast<int32_t>(plan.entries.size());
  }
  plan.head_meta.clear();
  plan.head_part_k.clear();
  for (int32_t i : head_order) plan.head_meta.push_back(RowMeta{i, ebeg(i), eend(i), 0});
  plan.head_publish = static_cast<int64_t>(head_order.size());
  if (head_part_tasks) {
    // one task per tail row, in one extra level after the head levels: the sum over the row's
    // head-column entries (every tail row gets one, even an empty one: it seeds partial[i] = y[i])
    const int32_t extra = static_cast<int32_t>(head_width.size());
    head_width.push_back(0);
    for (int64_t t = 0; t < tail_rows; ++t) {
      const int32_t i = tail_order[t];
      const int32_t b = static_cast<int32_t>(plan.head_part_k.size());
      for (int32_t k = ebeg(i); k < eend(i); ++k) {
        if (tail_index[S.col[k]] < 0) plan.head_part_k.push_back(k);
      }
      plan.head_meta.push_back(RowMeta{i, b, static_cast<int32_t>(plan.head_part_k.size()), 0});
      head_level[i] = extra;
      ++head_width[extra];
    }
  }
  if (head_width.empty()) head_width.push_back(0);
  fill_start_thresholds(plan.head_meta, head_level, head_width, tune.solve_lookahead_levels, tune.solve_min_window,
                        tune.solve_max_window);
}

inline std::string build_schedule(const b200lu_symbolic_view& s, const ScheduleTuning& tune, Schedule& out) {
  const int64_t n = s.n;
  const int64_t nnz = s.nnz_factors;
  if (n < 0 || nnz < 0) return "negative dimensions";
  if (nnz >= (int64_t{1} << 31) - 64) return "nnz(L+U) exceeds the int32 device index range";
  if (n > 0 && (s.row_offsets[0] != 0 || s.row_offsets[n] != nnz)) return "row_offsets do not span nnz_factors";
  out.n = n;
  out.nnz = nnz;
  out.row_ptr.resize(n + 1);
  out.col.resize(nnz);
  out.diag.resize(n);
  for (int64_t i = 0; i <= n; ++i) out.row_ptr[i] = static_cast<int32_t>(s.row_offsets[i]);
  for (int64_t k = 0; k < nnz; ++k) out.col[k] = static_cast<int32_t>(s.col_indices[k]);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t lo = s.row_offsets[i], hi = s.row_offsets[i + 1], d = s.diag_pos[i];
    if (hi < lo || d < lo || d >= hi || s.col_indices[d] != i) {
      return "diag_pos[" + std::to_string(i) + "] does not address the diagonal";
    }
    for (int64_t k = lo; k < hi; ++k) {
      const int64_t c = s.col_indices[k];
      if (c < 0 || c >= n || (k > lo && c <= s.col_indices[k - 1])) {
        return "row " + std::to_string(i) + " is not strictly increasing / in range";
      }
    }
    out.diag[i] = static_cast<int32_t>(d);
    out.max_row_len = std::max(out.max_row_len, hi - lo);
  }

  // L-levels ascending, U-levels descending; pair counts per row.
  std::vector<int32_t> llev(n, 0), ulev(n, 0);
  out.pair_row_ptr.assign(n + 1, 0);
  int32_t lmax = -1, umax = -1;
  for (int64_t i = 0; i < n; ++i) {
    int32_t lv = 0;
    int64_t pairs = 0;
    for (int64_t k = s.row_offsets[i]; k < s.diag_pos[i]; ++k) {
      const int64_t d = s.col_indices[k];
      lv = std::max(lv, llev[d] + 1);
      pairs += s.row_offsets[d + 1] - s.diag_pos[d] - 1;
    }
    llev[i] = lv;
    lmax = std::max(lmax, lv);
    out.pair_row_ptr[i + 1] = out.pair_row_ptr[i] + pairs;
    out.nnz_lower += s.diag_pos[i] - s.row_offsets[i];
  }
  out.update_pairs = out.pair_row_ptr[n];
  for (int64_t i = n - 1; i >= 0; --i) {
    int32_t lv = 0;
    for (int64_t k = s.diag_pos[i] + 1; k < s.row_offsets[i + 1]; ++k) {
      lv = std::max(lv, ulev[s.col_indices[k]] + 1);
    }
    ulev[i] = lv;
    umax = std::max(umax, lv);
  }
  out.lower_levels = lmax + 1;
  out.upper_levels = umax + 1;

  auto level_sort = [n](const std::vector<int32_t>& lev, int32_t levels, bool descending_ties) {
    std::vector<int64_t> start(static_cast<size_t>(levels) + 1, 0);
    for (int64_t i = 0; i < n; ++i) ++start[lev[i] + 1];
    for (int32_t l = 0; l < levels; ++l) start[l + 1] += start[l];
    std::vector<int32_t> order(n);
    if (!descending_ties) {
      for (int64_t i = 0; i < n; ++i) order[start[lev[i]]++] = static_cast<int32_t>(i);
    } else {
      for (int64_t i = n - 1; i >= 0; --i) order[start[lev[i]]++] = static_cast<int32_t>(i);
    }
    return order;
  };
  out.lower_order = level_sort(llev, lmax + 1, false);
  out.upper_order = level_sort(ulev, umax + 1, true);

  out.lower_level = llev;
  out.upper_level = ulev;
  out.lower_width.assign(static_cast<size_t>(lmax + 1), 0);
  out.upper_width.assign(static_cast<size_t>(umax + 1), 0);
  for (int64_t i = 0; i < n; ++i) {
    ++out.lower_width[llev[i]];
    ++out.upper_width[ulev[i]];
  }

  out.lower_meta.resize(n);
  out.upper_meta.resize(n);
  for (int64_t r = 0; r < n; ++r) {
    const int32_t il = out.lower_order[r], iu = out.upper_order[r];
    out.lower_meta[r] = RowMeta{il, out.row_ptr[il], out.diag[il], 0};          // strict-lower entries
    out.upper_meta[r] = RowMeta{iu, out.diag[iu] + 1, out.row_ptr[iu + 1], 0};  // strict-upper entries
  }
  fill_start_thresholds(out.lower_meta, llev, out.lower_width, tune.solve_lookahead_levels,
                        tune.solve_min_window, tune.solve_max_window);
  fill_start_thresholds(out.upper_meta, ulev, out.upper_width, tune.solve_lookahead_levels,
                        tune.solve_min_window, tune.solve_max_window);

  // ---- on-chip tails of the two sweeps (default mode)
  out.lower_tail = TailPlan{};
  out.upper_tail = TailPlan{};
  if (n > 0) {
    // L sweep: the tail is the successor-closed set of rows at dependency level >= cut.
    int64_t ltail_rows = 0;
    const int64_t lcut = pick_tail_cut(out.lower_width, tune, &ltail_rows);
    if (ltail_rows > 0) {
      const int64_t head_rows = n - ltail_rows;
      std::vector<int32_t> head(out.lower_order.begin(), out.lower_order.begin() + head_rows);
      std::vector<int32_t> tail(out.lower_order.begin() + head_rows, out.lower_order.end());
      std::vector<int32_t> head_width(out.lower_width.begin(), out.lower_width.begin() + lcut);
      make_tail_plan(
          out, tune, tail, head, llev, head_width, /*head_part_tasks=*/true,
          [&out](int32_t i) { return out.row_ptr[i]; }, [&out](int32_t i) { return out.diag[i]; }, out.lower_tail);
      out.lower_tail.levels = out.lower_levels - lcut;
    }
    // U sweep: the long chains start at the last rows and run DOWN the elimination tree, so the
    // narrow part comes first. Its rows are the predecessor-closed set of rows of large HEIGHT in
    // the U dependency DAG (height = longest chain of rows depending on the row): whatever a
    // tail row needs is itself in the tail, and what remains after the tail is a DAG no deeper
    // than the cut. (On a structurally symmetric pattern this is the same row set as the L tail.)
    std::vector<int32_t> height(n, 0);
    int32_t hmax = 0;
    for (int64_t k = 0; k < n; ++k) {
      for (int64_t e = s.diag_pos[k] + 1; e < s.row_offsets[k + 1]; ++e) {
        const int64_t j = s.col_indices[e];  // row k depends on row j > k
        height[j] = std::max(height[j], height[k] + 1);
      }
      hmax = std::max(hmax, height[k]);
    }
    std::vector<int32_t> hwidth(static_cast<size_t>(hmax) + 1, 0);
    for (int64_t i = 0; i < n; ++i) ++hwidth[height[i]];
    int64_t utail_rows = 0;
    const int64_t ucut = pick_tail_cut(hwidth, tune, &utail_rows);
    if (utail_rows > 0) {
      std::vector<int32_t> tail;
      tail.reserve(utail_rows);
      for (int64_t i = n - 1; i >= 0; --i) {
        if (height[i] >= ucut) tail.push_back(static_cast<int32_t>(i));
      }
      // dependencies have strictly larger height: descending height is a topological order
      std::stable_sort(tail.begin(), tail.end(), [&height](int32_t a, int32_t b) { return height[a] > height[b]; });
      // head rows: dependency levels among themselves (tail columns are final by then)
      std::vector<int32_t> hlev(n, 0);
      int32_t hl_max = -1;
      for (int64_t i = n - 1; i >= 0; --i) {
        if (height[i] >= ucut) continue;
        int32_t lv = 0;
        for (int64_t e = s.diag_pos[i] + 1; e < s.row_offsets[i + 1]; ++e) {
          const int64_t j = s.col_indices[e];
          if (height[j] < ucut) lv = std::max(lv, hlev[j] + 1);
        }
        hlev[i] = lv;
        hl_max = std::max(hl_max, lv);
      }
      std::vector<int32_t> head_width(static_cast<size_t>(hl_max + 1), 0);
      for (int64_t i = 0; i < n; ++i) {
        if (height[i] < ucut) ++head_width[hlev[i]];
      }
      std::vector<int64_t> pos(head_width.size() + 1, 0);
      for (size_t l = 0; l < head_width.size(); ++l) pos[l + 1] = pos[l] + head_width[l];
      std::vector<int32_t> head(static_cast<size_t>(n - utail_rows));
      for (int64_t i = n - 1; i >= 0; --i) {
        if (height[i] < ucut) head[pos[hlev[i]]++] = static_cast<int32_t>(i);
      }
      make_tail_plan(
          out, tune, tail, head, hlev, head_width, /*head_part_tasks=*/false,
          [&out](int32_t i) { return out.diag[i] + 1; }, [&out](int32_t i) { return out.row_ptr[i + 1]; },
          out.upper_tail);
      out.upper_tail.levels = hmax + 1 - ucut;
      out.upper_head_levels = hl_max + 1;
    }
  }

  out.small_rows.clear();
  out.big_rows.clear();
  out.trivial_rows.clear();
  for (int64_t r = 0; r < n; ++r) {
    const int32_t i = out.lower_order[r];
    const int64_t len = s.row_offsets[i + 1] - s.row_offsets[i];
    if (s.diag_pos[i] == s.row_offsets[i]) {
      out.trivial_rows.push_back(i);  // no pivots: nothing to eliminate
    } else if (len <= tune.small_slot) {
      out.small_rows.push_back(i);
    } else {
      out.big_rows.push_back(i);
    }
  }
  return "";
}

}  // namespace b200lu
