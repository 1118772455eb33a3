// Plan of the GATHER form of the batched trailing refactorization (gather.cuh): host code only.
//
// eliminate (src/numeric.cpp:27-58) updates entry (i, j) once per pivot d of row i that has u_dj != 0, in
// ascending d. The scatter form (batch.cuh, tile.cuh) walks the pivots and touches every target once per
// pivot — as an L2 reduction or a shared-memory read-modify-write. The gather form turns the loop inside out
// for a BATCH of up to K consecutive pivots of a block of R consecutive rows: every target entry that the batch
// touches is loaded once, receives all of the batch's updates IN A REGISTER in ascending pivot order (the same
// products, the same two roundings per update, the same order: bit-identical), and is stored once. What used to
// be one reduction per update becomes one load + one store per (target, batch); the multipliers l_id of the
// batch are the only operands kept on chip (R x K values per scenario in shared memory).
//
// The plan is a flat stream of 8-byte records per block, cut into batches:
//     INIT(r, slot)        acc[r] <- values[slot]                       (start of a target, once per row that has it)
//     UPD(mask, e, slot)   acc[r] <- acc[r] - l[r][e] * values[slot]    for the rows r in mask (src/numeric.cpp:44)
//     DIV(mask, k, slot)   acc[r] <- acc[r] / values[slot]; l[r][k] <- acc[r]   (target = pivot column d_k: src/numeric.cpp:40-41)
//     ... the record that ends a target carries LAST: the accumulators of the rows INIT named are stored
//     PUB(r, row)          row r of the block is final: pivot check (src/numeric.cpp:48), ready flag
// Targets of a batch are processed in ascending column order, so a multiplier l[r][e] (produced at column d_e)
// exists before any target that needs it (all of them have columns > d_e). A batch never contains a pivot that is
// a row of the block unless that row became final in an earlier batch, and the device drains its load pipeline at
// batch boundaries: no load of a batch can alias a store of the same batch.
#pragma once

#include <algorithm>
#include <cstdint>
#include <queue>
#include <string>
#include <vector>

namespace b200lu {

struct GRec {
  uint32_t slot;  // values slot (INIT / UPD / DIV) or row id (PUB)
  uint32_t info;  // bits 0-2 type, 3 LAST, 4-7 row mask, 8-13 pivot index inside the batch, 14 target is the row's diagonal, 15 PUB without a seen diagonal
};
constexpr uint32_t kGNop = 0, kGInit = 1, kGUpd = 2, kGDiv = 3, kGPub = 4;
constexpr uint32_t kGLast = 8u, kGIsDiag = 1u << 14, kGFresh = 1u << 15;
constexpr int kGWindow = 32;  // records per window (one per lane)

struct GBatch {
  uint32_t win_beg;  // first window of the batch (records [32 win_beg, 32 (win_beg + n_win)))
  int32_t n_win;
  int32_t wait_beg, n_wait;  // rows of other blocks whose ready flag the batch needs (into GatherPlan::waits)
};
struct GBlock {
  int32_t batch_beg, batch_end;
};

struct GatherPlan {
  std::vector<GBlock> blocks;  // in claim order (topological for the block DAG)
  std::vector<GBatch> batches;
  std::vector<GRec> recs;
  std::vector<int32_t> waits;
  int64_t n_init = 0, n_upd = 0, n_div = 0, n_pub = 0, n_pad = 0, n_targets = 0, rows = 0;
};

// row_ptr / col / diag: int32 image of the combined pattern; tail_rows: ascending rows of the trailing part (all
// rows they depend on are either tail rows or final before the launch); level: dependency level per row.
inline bool build_gather_plan(const std::vector<int32_t>& row_ptr, const std::vector<int32_t>& col, const std::vector<int32_t>& diag,
                              const std::vector<int32_t>& level, const std::vector<int32_t>& tail_rows, int R, int K,
                              int tail_small, GatherPlan* out, std::string* err) {
  GatherPlan& P = *out;
  P = GatherPlan();
  const int32_t n = static_cast<int32_t>(diag.size());
  if (R < 1 || R > 4 || K < 1 || K > 64) {
    *err = "gather plan: unsupported block height / batch length";
    return false;
  }
  std::vector<char> is_tail(n, 0);
  for (int32_t i : tail_rows) is_tail[i] = 1;
  P.rows = static_cast<int64_t>(tail_rows.size());
  struct Piv {
    int32_t d;
    uint32_t mask, last;  // rows that have the pivot; rows for which it is the last pivot
    int internal;         // block row it is, or -1
  };
  struct Tup {
    int32_t j, e, slot;
  };
  const size_t nb = (tail_rows.size() + R - 1) / R;
  std::vector<std::vector<int32_t>> block_rows(nb);
  std::vector<int32_t> block_of(n, -1);
  std::vector<GBlock> blocks(nb);
  std::vector<std::vector<int32_t>> succ(nb);
  std::vector<int32_t> indeg(nb, 0);
  std::vector<Piv> piv;
  std::vector<std::pair<int32_t, int>> raw;
  std::vector<Tup> tup;
  std::vector<int> cur;
  std::vector<char> cut_at;
  for (size_t b = 0; b < nb; ++b) {
    for (size_t q = b * R; q < std::min(tail_rows.size(), (b + 1) * R); ++q) {
      block_rows[b].push_back(tail_rows[q]);
      block_of[tail_rows[q]] = static_cast<int32_t>(b);
    }
  }
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
        *err = "gather plan: a trailing row without pivots";
        return false;
      }
      piv[last_of_row[r]].last |= 1u << r;
    }
    // block DAG edges
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
    int ext_end = static_cast<int>(piv.size());
    for (int t = 0; t < static_cast<int>(piv.size()); ++t) {
      if (piv[t].internal >= 0) {
        ext_end = t;
        break;
      }
    }
    // Batch boundaries among the external pivots. The youngest pivots of a trailing row are the rows just before
    // it in its chain, published moments before the row itself can finish, while a batch only starts once its
    // youngest pivot is ready: batch lengths therefore GROW going back from the end (tail_small, tail_small,
    // 2 tail_small, 4 tail_small, ... up to K), so that work waiting for a pivot published a rows earlier is
    // proportional to a, and the old pivots (most of the work) still come in full batches.
    cut_at.assign(piv.size() + 1, 0);
    if (tail_small > 0) {
      int pos = ext_end, len = tail_small, reps = 0;
      while (pos > 0) {
        pos -= std::min(len, K);
        if (pos > 0) cut_at[pos] = 1;
        if (len < K && ++reps >= 2) {
          len *= 2;
          reps = 1;
        }
      }
    }
    blocks[b].batch_beg = static_cast<int32_t>(P.batches.size());
    bool diag_seen[4] = {false, false, false, false};
    cur.clear();
    uint32_t curmask = 0;
    auto emit = [&]() -> bool {
      if (cur.empty()) return true;
      GBatch gb;
      gb.win_beg = static_cast<uint32_t>(P.recs.size() / kGWindow);
      gb.wait_beg = static_cast<int32_t>(P.waits.size());
      tup.clear();
      for (int e = 0; e < static_cast<int>(cur.size()); ++e) {
        const Piv& p = piv[cur[e]];
        if (p.internal < 0 && is_tail[p.d]) P.waits.push_back(p.d);
        for (int32_t t = diag[p.d] + 1; t < row_ptr[p.d + 1]; ++t) tup.push_back(Tup{col[t], e, t});
        tup.push_back(Tup{p.d, 0x4000 + e, diag[p.d]});  // the pivot column itself: ends with the division
      }
      gb.n_wait = static_cast<int32_t>(P.waits.size()) - gb.wait_beg;
      std::sort(tup.begin(), tup.end(), [](const Tup& x, const Tup& y) { return x.j != y.j ? x.j < y.j : x.e < y.e; });
      for (size_t q = 0; q < tup.size();) {
        size_t q1 = q;
        uint32_t rmask = 0;
        while (q1 < tup.size() && tup[q1].j == tup[q].j) {
          rmask |= piv[cur[tup[q1].e & 0x3fff]].mask;
          ++q1;
        }
        const int32_t j = tup[q].j;
        for (int r = 0; r < nr; ++r) {
          if (!(rmask & (1u << r))) continue;
          const int32_t* rb = col.data() + row_ptr[rows[r]];
          const int32_t* re = col.data() + row_ptr[rows[r] + 1];
          const int32_t* it = std::lower_bound(rb, re, j);
          if (it == re || *it != j) {
            *err = "gather plan: the pattern is not closed under fill (row " + std::to_string(rows[r]) + ", column " + std::to_string(j) + ")";
            return false;
          }
          uint32_t info = kGInit | (16u << r);
          if (j == rows[r]) {
            info |= kGIsDiag;
            diag_seen[r] = true;
          }
          P.recs.push_back(GRec{static_cast<uint32_t>(it - col.data()), info});
          ++P.n_init;
        }
        for (size_t t = q; t < q1; ++t) {
          const bool chain = tup[t].e >= 0x4000;
          const int e = tup[t].e & 0x3fff;
          const uint32_t mask = piv[cur[e]].mask;
          // (rows of the block that do not have d_k as a pivot may still be updated at column d_k — an upper
          // entry of a row whose index is below d_k: they accumulate and store, only `mask` rows divide)
          P.recs.push_back(GRec{static_cast<uint32_t>(tup[t].slot), (chain ? kGDiv : kGUpd) | (mask << 4) | (static_cast<uint32_t>(e) << 8)});
          if (chain) {
            ++P.n_div;
          } else {
            ++P.n_upd;
          }
        }
        P.recs.back().info |= kGLast;
        ++P.n_targets;
        q = q1;
      }
      for (int e = 0; e < static_cast<int>(cur.size()); ++e) {
        const Piv& p = piv[cur[e]];
        for (int r = 0; r < nr; ++r) {
          if (p.last & (1u << r)) {
            P.recs.push_back(GRec{static_cast<uint32_t>(rows[r]), kGPub | (16u << r) | (diag_seen[r] ? 0u : kGFresh)});
            ++P.n_pub;
          }
        }
      }
      while (P.recs.size() % kGWindow) {
        P.recs.push_back(GRec{0u, kGNop});
        ++P.n_pad;
      }
      const size_t wins = P.recs.size() / kGWindow - gb.win_beg;
      if (P.recs.size() / kGWindow > 0xffffffffull || wins > 0x7fffffffull) {
        *err = "gather plan: record stream too long";
        return false;
      }
      gb.n_win = static_cast<int32_t>(wins);
      P.batches.push_back(gb);
      cur.clear();
      curmask = 0;
      return true;
    };
    for (int t = 0; t < static_cast<int>(piv.size()); ++t) {
      const bool cut = static_cast<int>(cur.size()) == K || (piv[t].internal >= 0 && (curmask & (1u << piv[t].internal))) ||
                       cut_at[t] != 0;
      if (cut && !emit()) return false;
      cur.push_back(t);
      curmask |= piv[t].mask;
      // a row whose last pivot this is gets published at the end of the batch: close it here, so the row is
      // visible before the block waits for any later pivot (which may itself depend on that row)
      if (piv[t].last && !emit()) return false;
    }
    if (!emit()) return false;
    blocks[b].batch_end = static_cast<int32_t>(P.batches.size());
  }
  // Claim order: Kahn on the block DAG, ready blocks by (level of the first row, index) — index order is
  // topological but walks one chain at a time, level order is not topological for blocks.
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
    *err = "gather plan: block dependency graph is not acyclic";
    return false;
  }
  return true;
}

}  // namespace b200lu
