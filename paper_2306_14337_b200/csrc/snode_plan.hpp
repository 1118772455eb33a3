// Plan of the SUPERNODAL form of the batched trailing refactorization (snode.cuh): host code only.
//
// Measured on the C2 pattern (AMD-only analysis): 80 % of the update pairs of eliminate (src/numeric.cpp:34-49) belong
// to pivots that sit in fundamental supernodes of 8 or more rows — runs of consecutive rows d, d+1, ... whose upper
// patterns are nested exactly, U(d) = {d+1} ∪ U(d+1) (chains of the elimination tree) — although the trailing block as a
// whole is 0.4-1.2 % dense. For a row i that has pivot d, fill closure gives it every later pivot of the run as well,
// and all of them update THE SAME destination entries of row i. So for a run of s pivots d0 .. d0+s-1:
//   * the s multipliers of row i are a small dense forward substitution with the run's upper-triangular diagonal
//     block (phase A): alpha_k = (a(i,d0+k) - sum_{e<k} alpha_e u(d0+e,d0+k)) / u(d0+k,d0+k), src/numeric.cpp:40-44,
//     every u at a fixed offset (k - e) behind its row's diagonal;
//   * every destination entry j in J = U(d0+s-1) receives its s updates in a REGISTER, in ascending pivot order —
//     acc <- acc - alpha_k * u(d0+k, j), the same products and roundings as the reference, hence the same bits — and
//     is loaded and stored once per run (phase B); u(d0+k, j) sits at a fixed offset in row d0+k, so the whole phase
//     needs ONE destination list per (row, run) instead of one destination per update pair, and no L2 reduction.
// A run never crosses a point where a row of the block becomes final, and never contains a pivot that is a row of
// the block together with pivots that row still needs (same rules as gather_plan.hpp). Runs shrink towards the end of
// a row's pivot list (1, 1, 2, 4, ... up to the cap): the youngest pivots are published moments before the row can
// finish, and a run starts only when its youngest pivot is ready.
#pragma once

#include <algorithm>
#include <cstdint>
#include <queue>
#include <string>
#include <vector>

namespace b200lu {

constexpr int kSnodeMax = 8;   // pivots per run (multipliers held in registers)
constexpr int kSnodeRows = 2;  // rows per block

struct SRun {               // 32 bytes
  int32_t d0;               // first pivot row of the run
  uint8_t s, mask, pub, wait;  // pivots; block rows that have them; rows final after the run; 1 = await the rows' ready flags
  int32_t nj;               // |J|: upper entries of the run's last pivot row
  uint32_t dest_beg;        // destination slots: for each row of `mask` (ascending) nj global slots
  int32_t lslot[4];         // global slot of entry (row r, column d0); the run's other columns follow it
};
struct SBlock {             // 32 bytes
  int32_t run_beg, run_end;
  int32_t rows[4];          // block rows (-1 pads)
  int32_t pad[2];
};

struct SnodePlan {
  std::vector<SBlock> blocks;  // claim order
  std::vector<SRun> runs;
  std::vector<uint32_t> dest;
  int64_t rows = 0, pivots = 0, pairs = 0, pairs_in_runs_of_4 = 0;
};

inline bool build_snode_plan(const std::vector<int32_t>& row_ptr, const std::vector<int32_t>& col, const std::vector<int32_t>& diag,
                             const std::vector<int32_t>& level, const std::vector<int32_t>& tail_rows, int R, int tail_small,
                             SnodePlan* out, std::string* err) {
  SnodePlan& P = *out;
  P = SnodePlan();
  const int32_t n = static_cast<int32_t>(diag.size());
  if (R < 1 || R > kSnodeRows) {
    *err = "snode plan: unsupported block height";
    return false;
  }
  // fundamental links: U(d) == {d+1} ∪ U(d+1)
  std::vector<char> link(n, 0);
  for (int32_t d = 0; d + 1 < n; ++d) {
    const int32_t a0 = diag[d] + 1, a1 = row_ptr[d + 1], b0 = diag[d + 1] + 1, b1 = row_ptr[d + 2];
    if (a1 - a0 >= 1 && col[a0] == d + 1 && (a1 - a0 - 1) == (b1 - b0) && std::equal(col.begin() + a0 + 1, col.begin() + a1, col.begin() + b0)) link[d] = 1;
  }
  std::vector<char> is_tail(n, 0);
  for (int32_t i : tail_rows) is_tail[i] = 1;
  P.rows = static_cast<int64_t>(tail_rows.size());
  struct Piv {
    int32_t d;
    uint32_t mask, last;
    int internal;
  };
  const size_t nb = (tail_rows.size() + R - 1) / R;
  std::vector<std::vector<int32_t>> block_rows(nb);
  std::vector<int32_t> block_of(n, -1);
  std::vector<SBlock> blocks(nb);
  std::vector<std::vector<int32_t>> succ(nb);
  std::vector<int32_t> indeg(nb, 0);
  std::vector<Piv> piv;
  std::vector<std::pair<int32_t, int>> raw;
  std::vector<char> cut_at;
  for (size_t b = 0; b < nb; ++b) {
    for (size_t q = b * R; q < std::min(tail_rows.size(), (b + 1) * R); ++q) {
      block_rows[b].push_back(tail_rows[q]);
      block_of[tail_rows[q]] = static_cast<int32_t>(b);
    }
  }
  auto find_slot = [&](int32_t row, int32_t c) -> int64_t {
    const int32_t* rb = col.data() + row_ptr[row];
    const int32_t* re = col.data() + row_ptr[row + 1];
    const int32_t* it = std::lower_bound(rb, re, c);
    return (it == re || *it != c) ? -1 : it - col.data();
  };
  for (size_t b = 0; b < nb; ++b) {
    const std::vector<int32_t>& rows = block_rows[b];
    const int nr = static_cast<int>(rows.size());
    raw.clear();
    for (int r = 0; r < nr; ++r) {
      for (int32_t k = row_ptr[rows[r]]; k < diag[rows[r]]; ++k) raw.emplace_back(col[k], r);
    }
    std::sort(raw.begin(), raw.end());
    piv.clear();
    int last_of_row[4] = {-1, -1, -1, -1};
    for (size_t q = 0; q < raw.size(); ++q) {
      if (q == 0 || raw[q].first != raw[q - 1].first) {
        int internal = -1;
        for (int r = 0; r < nr; ++r) {
          if (rows[r] == raw[q].first) internal = r;
        }
        piv.push_back(Piv{raw[q].first, 0u, 0u, internal});
      }
      piv.back().mask |= 1u << raw[q].second;
      last_of_row[raw[q].second] = static_cast<int>(piv.size()) - 1;
    }
    for (int r = 0; r < nr; ++r) {
      if (last_of_row[r] < 0) {
        *err = "snode plan: a trailing row without pivots";
        return false;
      }
      piv[last_of_row[r]].last |= 1u << r;
    }
    {
      int32_t last = -1;
      for (const Piv& p : piv) {
        const int32_t pb = block_of[p.d];
        if (pb >= 0 && pb != static_cast<int32_t>(b) && pb != last) {
          succ[pb].push_back(static_cast<int32_t>(b));
          ++indeg[b];
          last = pb;
        }
      }
    }
    const int np = static_cast<int>(piv.size());
    int ext_end = np;
    for (int t = 0; t < np; ++t) {
      if (piv[t].internal >= 0) {
        ext_end = t;
        break;
      }
    }
    cut_at.assign(np + 1, 0);
    if (tail_small > 0) {
      int pos = ext_end, len = tail_small, reps = 0;
      while (pos > 0) {
        pos -= std::min(len, kSnodeMax);
        if (pos > 0) cut_at[pos] = 1;
        if (len < kSnodeMax && ++reps >= 2) {
          len *= 2;
          reps = 1;
        }
      }
    }
    SBlock& blk = blocks[b];
    blk.run_beg = static_cast<int32_t>(P.runs.size());
    for (int r = 0; r < 4; ++r) blk.rows[r] = r < nr ? rows[r] : -1;
    blk.pad[0] = blk.pad[1] = 0;
    int t = 0;
    while (t < np) {
      // grow the run [t, t + s)
      int s = 1;
      while (t + s < np && s < kSnodeMax) {
        const Piv& prev = piv[t + s - 1];
        const Piv& next = piv[t + s];
        if (prev.last || cut_at[t + s] || prev.internal >= 0 || next.internal >= 0) break;
        if (next.d != prev.d + 1 || !link[prev.d] || next.mask != prev.mask) break;
        ++s;
      }
      const Piv& first = piv[t];
      const Piv& lastp = piv[t + s - 1];
      SRun run;
      run.d0 = first.d;
      run.s = static_cast<uint8_t>(s);
      run.mask = static_cast<uint8_t>(first.mask);
      run.pub = static_cast<uint8_t>(lastp.last);
      run.wait = (first.internal < 0 && is_tail[first.d]) ? 1 : 0;
      for (int q = 1; q < s; ++q) {
        if (is_tail[piv[t + q].d] != is_tail[first.d]) run.wait = 1;  // (a run across the head / tail border waits; flags of head rows are set)
      }
      run.nj = row_ptr[lastp.d + 1] - diag[lastp.d] - 1;
      run.dest_beg = static_cast<uint32_t>(P.dest.size());
      for (int r = 0; r < 4; ++r) run.lslot[r] = -1;
      for (int r = 0; r < nr; ++r) {
        if (!(first.mask & (1u << r))) continue;
        const int64_t ls = find_slot(rows[r], first.d);
        if (ls < 0) {
          *err = "snode plan: pivot entry not found";
          return false;
        }
        for (int q = 1; q < s; ++q) {  // the run's columns are consecutive entries of the row
          if (col[ls + q] != first.d + q) {
            *err = "snode plan: the pattern is not closed under fill (row " + std::to_string(rows[r]) + ")";
            return false;
          }
        }
        run.lslot[r] = static_cast<int32_t>(ls);
        for (int32_t u = diag[lastp.d] + 1; u < row_ptr[lastp.d + 1]; ++u) {
          const int64_t ds = find_slot(rows[r], col[u]);
          if (ds < 0) {
            *err = "snode plan: the pattern is not closed under fill (row " + std::to_string(rows[r]) + ", column " + std::to_string(col[u]) + ")";
            return false;
          }
          P.dest.push_back(static_cast<uint32_t>(ds));
        }
      }
      if (P.dest.size() > 0xfffffff0ull) {
        *err = "snode plan: destination table too long";
        return false;
      }
      P.runs.push_back(run);
      P.pivots += s;
      for (int q = 0; q < s; ++q) {
        const int64_t m = row_ptr[piv[t + q].d + 1] - diag[piv[t + q].d] - 1;
        const int64_t pr = m * __builtin_popcount(first.mask);
        P.pairs += pr;
        if (s >= 4) P.pairs_in_runs_of_4 += pr;
      }
      t += s;
    }
    blk.run_end = static_cast<int32_t>(P.runs.size());
  }
  using Key = std::pair<int32_t, int32_t>;
  std::priority_queue<Key, std::vector<Key>, std::greater<Key>> ready;
  for (size_t b = 0; b < nb; ++b) {
    if (indeg[b] == 0) ready.emplace(level[block_rows[b][0]], static_cast<int32_t>(b));
  }
  P.blocks.reserve(nb);
  while (!ready.empty()) {
    const int32_t b = ready.top().second;
    ready.pop();
    P.blocks.push_back(blocks[b]);
    for (int32_t c : succ[b]) {
      if (--indeg[c] == 0) ready.emplace(level[block_rows[c][0]], c);
    }
  }
  if (P.blocks.size() != nb) {
    *err = "snode plan: block dependency graph is not acyclic";
    return false;
  }
  return true;
}

}  // namespace b200lu
