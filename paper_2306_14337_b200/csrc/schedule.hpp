// Host-side schedule derivation: everything the device kernels need beyond the
// reference's SymbolicFactors, computed once per handle in O(nnz(L+U)).
//
// The reference executes rows through SyncFreeScheduler (include/rlu/schedule.hpp:34-200):
// one ready flag per row, rows claimed in ascending order. On the device the claim order is
// the dependency LEVEL order (a topological order of the same DAG), so a claimed row's
// dependencies are always finished or held by a resident worker.
#pragma once

#include <algorithm>
#include <cstdint>
#include <string>
#include <vector>

#include "b200lu.h"

namespace b200lu {

// One record per claim position, so a worker learns everything about its row from one 16-byte
// load instead of a chain of dependent index loads.
struct RowMeta {
  int32_t row;    // row index in the permuted matrix
  int32_t beg;    // first entry the worker touches
  int32_t end;    // one past the last entry
  int32_t start;  // the row may start once this many rows of the sweep have finished
};

struct Schedule {
  int64_t n = 0, nnz = 0, nnz_lower = 0, update_pairs = 0;
  int64_t lower_levels = 0, upper_levels = 0, max_row_len = 0;
  std::vector<int32_t> row_ptr, col, diag;  // int32 image of the combined pattern
  // Rows by ascending L-level (ties by index), split by row length into the rows a single warp
  // slot holds and the wide rows that need the per-CTA wide slot.
  std::vector<int32_t> small_rows, big_rows;
  std::vector<int32_t> lower_order;  // all rows, L-level order
  std::vector<int32_t> upper_order;  // all rows, U-level order
  std::vector<int64_t> pair_row_ptr;  // n+1: first update pair of each row
  std::vector<int32_t> lower_level, upper_level;  // per row
  std::vector<int32_t> lower_width, upper_width;  // rows per level
  std::vector<RowMeta> lower_meta, upper_meta;    // triangular sweeps, per claim position
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
  int64_t solve_lookahead_levels = 48;
  int64_t solve_min_window = 64;
  int64_t solve_max_window = 1 << 20;
};

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

  out.small_rows.clear();
  out.big_rows.clear();
  for (int64_t r = 0; r < n; ++r) {
    const int32_t i = out.lower_order[r];
    const int64_t len = s.row_offsets[i + 1] - s.row_offsets[i];
    (len <= tune.small_slot ? out.small_rows : out.big_rows).push_back(i);
  }
  return "";
}

}  // namespace b200lu
