// Host side of the tiled batched refactorization (tile.cuh): the per-pattern plan — which rows form a
// tile, the ascending merge of the tile's pivot lists cut into TMA-sized chunks, and a topological claim
// order of the tiles — built once per handle in O(nnz(L) log), plus a host emulation of the plan for one
// scenario (diagnostics: `b200lu_tile_plan_emulate`, used by the CPU tests to check the plan against the
// oracle without a GPU; never on the product path).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <functional>
#include <queue>
#include <string>
#include <utility>
#include <vector>

#include "schedule.hpp"

namespace b200lu {

constexpr int kTileScen = 8;            // scenarios per tile unit
constexpr int kTileEntryLanes = 8;      // lanes = 8 entry lanes x 4 scenario pairs (16-byte shared-memory accesses)
constexpr int kTileChunk = 96;          // most entries of a pivot row fetched by one TMA copy
constexpr int kTileBoxStep = 16;        // TMA box heights: 16, 32, ..., kTileChunk; also the ring's block size (entries)
constexpr int kTileMaps = kTileChunk / kTileBoxStep;
constexpr int kTileSlots = 16;          // pivot-row copies in flight (mbarriers)
constexpr int kTileMaxRows = 16;        // rows (consumer warps) of a tile
constexpr int kTileIter = 16;           // entries of a pivot row applied per inner-loop iteration (8 lanes x 2)
constexpr int kTileGroup = 4;           // iterations whose destinations one 16-byte load per lane brings in
constexpr int kTileGroupEntries = kTileIter * kTileGroup;  // 64 destination slots = 128 bytes per group
constexpr int kTileSpare = kTileEntryLanes;  // spare entries behind a row in shared memory: one per entry lane

struct TileRow {       // 32 bytes, one per row of a tile
  int32_t row;         // row index
  int32_t lo;          // its first entry in values[] / col[]
  int32_t len;         // entries of the row
  int32_t nl;          // strict-lower entries = pivots; the diagonal is entry nl
  int32_t ri_beg;      // its RowItems
  int32_t ri_cnt;
  int32_t smem_off;    // entry offset of the row inside the tile's shared-memory block (len + kTileSpare
  int32_t pad;         //   entries: the spare ones absorb the padding lanes' updates, one per entry lane)
};
struct TileMeta {      // 16 bytes
  int32_t row_beg, nrows;
  int32_t ext_beg, n_ext;  // pivot-row chunks fetched by TMA, in ascending pivot order
};
enum : uint32_t { kItemFirst = 1, kItemLast = 2, kItemInternal = 4, kItemWait = 8 };
struct ExtItem {       // 16 bytes: what the producer fetches
  int32_t entry;       // first entry of the chunk in values[] (the pivot row's diagonal for a first chunk)
  int32_t d;           // pivot row (ready flag)
  uint32_t users;      // rows of the tile that consume it (bit mask)
  uint32_t cnt_flags;  // entries of the chunk (a first chunk counts the diagonal) | kItem* << 16 | first ring block << 24
};
struct RowItem {       // 16 bytes: one pivot-row chunk as ONE row of the tile consumes it
  uint32_t tdest_off;  // its destination slice in the tile destination table, in groups (128 bytes each)
  uint32_t src;        // external: index of the ExtItem within the tile; internal: which row of the tile
  uint32_t cnt;        // entries of the chunk (a first chunk counts the diagonal)
  uint32_t flags;      // kItem* | first ring block of the staged copy << 8 (external)
};
static_assert(sizeof(TileRow) == 32 && sizeof(TileMeta) == 16 && sizeof(ExtItem) == 16 && sizeof(RowItem) == 16,
              "device record layout");

struct TilePlan {
  std::vector<TileMeta> tiles;   // in claim order (topological)
  std::vector<TileRow> rows;
  std::vector<ExtItem> ext;
  std::vector<RowItem> row_items;
  // Destination table of the tiled rows. For the chunk a RowItem describes, iteration t of the inner loop
  // applies pivot-row entries 16t .. 16t + 15 (the diagonal not counted); entry lane e takes entries
  // 16t + e and 16t + 8 + e. A group is four iterations: lane e finds the eight destination offsets
  // (entry index inside the target row) it needs for them in ONE 16-byte word:
  //     tdest[(tdest_off + t / 4) * 64 + 8 e + 2 (t % 4) + j]   for entry 16 t + 8 j + e.
  // Slots past the chunk's end point at the spare entry of their lane (offset len + e): the inner loop
  // needs no predicates, and no two threads ever write one address.
  std::vector<uint16_t> tdest;
  int64_t rows_smem_entries = 0; // largest tile, in entries (x 64 bytes), spare entries included
  int64_t fetched_entries = 0;   // sum of external item sizes (what TMA moves per unit)
  int64_t pairs = 0;             // update pairs of the tiled rows
};

// Head / tail split of the batched refactorization: the maximal suffix of dependency levels narrower than
// `tail_width` rows (never level 0) is the trailing part; it is successor-closed, so a first launch can
// finish every head row before the trailing launch starts. Returns the first trailing level (== number
// of levels when there is no worthwhile trailing part).
inline int64_t trailing_cut_level(const Schedule& S, int64_t tail_width) {
  const int64_t levels = static_cast<int64_t>(S.lower_width.size());
  int64_t cut = levels;
  for (int64_t l = levels - 1; l >= 1 && S.lower_width[l] < tail_width; --l) cut = l;
  if (levels - cut < 16) cut = levels;  // not worth a second launch
  return cut;
}

// Position of a chunk's entry t inside its destination slice (see TilePlan::tdest).
inline int32_t tile_dest_slot(int32_t t) {
  const int32_t it = t / kTileIter, w = t % kTileIter;
  return (it / kTileGroup) * kTileGroupEntries + (w % kTileEntryLanes) * 8 + (it % kTileGroup) * 2 + w / kTileEntryLanes;
}

// `tail_rows`: ascending row indices, a successor-closed set (every row that depends on a tail row is a
// tail row); every other row is final before the tiled launch starts. `cap_entries`: shared-memory
// capacity of a tile in entries. Returns "" or the reason the pattern cannot be tiled.
inline std::string build_tile_plan(const Schedule& S, const std::vector<int32_t>& tail_rows, int rows_per_tile,
                                   int64_t cap_entries, TilePlan& plan, int ring_blocks = 32) {
  plan = TilePlan{};
  const int64_t n = S.n;
  const int R = std::min(rows_per_tile, kTileMaxRows);
  if (S.max_row_len >= 65535) return "a row has more entries than a 16-bit destination offset can address";
  std::vector<int32_t> tile_of(n, -1);
  struct Raw {
    int32_t row_beg, nrows;
  };
  std::vector<Raw> raw;
  for (size_t b0 = 0; b0 < tail_rows.size();) {
    Raw t{static_cast<int32_t>(plan.rows.size()), 0};
    int64_t used = 0;
    while (b0 < tail_rows.size() && t.nrows < R) {
      const int32_t i = tail_rows[b0];
      const int64_t len = S.row_ptr[i + 1] - S.row_ptr[i] + kTileSpare;  // + the spare entries
      if (len > cap_entries) return "row " + std::to_string(i) + " (" + std::to_string(len - kTileSpare) + " entries) exceeds a tile's shared memory";
      if (used + len > cap_entries) break;
      TileRow tr{};
      tr.row = i;
      tr.lo = S.row_ptr[i];
      tr.len = static_cast<int32_t>(len - kTileSpare);
      tr.nl = S.diag[i] - S.row_ptr[i];
      tr.smem_off = static_cast<int32_t>(used);
      plan.rows.push_back(tr);
      tile_of[i] = static_cast<int32_t>(raw.size());
      used += len;
      plan.pairs += S.pair_row_ptr[i + 1] - S.pair_row_ptr[i];
      ++t.nrows;
      ++b0;
    }
    plan.rows_smem_entries = std::max(plan.rows_smem_entries, used);
    raw.push_back(t);
  }
  const size_t nt = raw.size();
  // external items of every tile, the RowItems + destination slices of every row, and the tile DAG
  std::vector<std::vector<ExtItem>> ext(nt);
  std::vector<std::vector<int32_t>> succ(nt);
  std::vector<int32_t> indeg(nt, 0);
  std::vector<std::vector<RowItem>> ritems(plan.rows.size());
  for (size_t b = 0; b < nt; ++b) {
    std::vector<std::pair<int32_t, int>> piv;  // (pivot row, tile row)
    for (int r = 0; r < raw[b].nrows; ++r) {
      const TileRow& tr = plan.rows[raw[b].row_beg + r];
      for (int32_t k = tr.lo; k < tr.lo + tr.nl; ++k) piv.emplace_back(S.col[k], r);
    }
    std::sort(piv.begin(), piv.end());
    int32_t last_pred = -1;
    int32_t ring_head = 0;  // the staging ring is allocated in order, from block 0 in every tile: positions are static
    for (size_t q = 0; q < piv.size();) {
      const int32_t d = piv[q].first;
      const size_t q0 = q;
      uint32_t users = 0;
      for (; q < piv.size() && piv[q].first == d; ++q) users |= 1u << piv[q].second;
      const int32_t dd = S.diag[d];
      const int64_t m1 = S.row_ptr[d + 1] - dd;  // diagonal + upper entries
      const bool internal = tile_of[d] == static_cast<int32_t>(b);
      int owner = 0;
      if (internal) {
        while (plan.rows[raw[b].row_beg + owner].row != d) ++owner;
      } else if (tile_of[d] >= 0 && tile_of[d] != last_pred) {  // pivots ascend, so do the tiles they belong to
        succ[tile_of[d]].push_back(static_cast<int32_t>(b));
        ++indeg[b];
        last_pred = tile_of[d];
      }
      // chunks of the pivot row: one (of any length) when it is read from the owner's shared-memory copy
      const int64_t step = internal ? m1 : kTileChunk;
      for (int64_t c0 = 0; c0 < m1; c0 += step) {
        const int64_t cnt = std::min<int64_t>(step, m1 - c0);
        uint32_t fl = internal ? kItemInternal : 0;
        if (c0 == 0) fl |= kItemFirst | ((!internal && tile_of[d] >= 0) ? kItemWait : 0);
        if (c0 + cnt == m1) fl |= kItemLast;
        uint32_t src = static_cast<uint32_t>(owner);
        if (!internal) {
          src = static_cast<uint32_t>(ext[b].size());
          const int32_t nb = static_cast<int32_t>((cnt + kTileBoxStep - 1) / kTileBoxStep);
          if (ring_head + nb > ring_blocks) ring_head = 0;  // a copy is contiguous: the blocks left at the end are skipped
          fl |= static_cast<uint32_t>(ring_head) << 8;      // first ring block of the copy
          ring_head += nb;
          ext[b].push_back(ExtItem{static_cast<int32_t>(dd + c0), d, users, static_cast<uint32_t>(cnt) | (fl << 16)});
          plan.fetched_entries += cnt;
        }
        for (size_t u = q0; u < q; ++u) {
          ritems[raw[b].row_beg + piv[u].second].push_back(RowItem{0, src, static_cast<uint32_t>(cnt), fl});
        }
      }
    }
  }
  // destination slices, row by row (the RowItems of a row are in ascending pivot order = its L entries)
  for (size_t rr = 0; rr < plan.rows.size(); ++rr) {
    TileRow& tr = plan.rows[rr];
    tr.ri_beg = static_cast<int32_t>(plan.row_items.size());
    tr.ri_cnt = static_cast<int32_t>(ritems[rr].size());
    int32_t k = tr.lo;       // L entry of the current pivot
    int32_t c = 0;           // upper entries of the current pivot row already covered by earlier chunks
    for (RowItem ri : ritems[rr]) {
      const int32_t d = S.col[k], dd = S.diag[d];
      const int32_t cu = static_cast<int32_t>(ri.cnt) - ((ri.flags & kItemFirst) ? 1 : 0);  // upper entries in this chunk
      if (ri.flags & kItemFirst) c = 0;
      const int32_t groups = std::max(1, (cu + kTileGroupEntries - 1) / kTileGroupEntries);  // >= 1: the first word is always loaded
      if (plan.tdest.size() / kTileGroupEntries + groups >= (uint64_t{1} << 32)) return "tile destination table too large";
      ri.tdest_off = static_cast<uint32_t>(plan.tdest.size() / kTileGroupEntries);
      plan.tdest.resize(plan.tdest.size() + static_cast<size_t>(groups) * kTileGroupEntries);
      uint16_t* slice = plan.tdest.data() + static_cast<size_t>(ri.tdest_off) * kTileGroupEntries;
      for (int32_t x = 0; x < groups * kTileGroupEntries; ++x) {  // padding: the spare entry of the lane that reads the slot
        slice[x] = static_cast<uint16_t>(tr.len + (x % kTileGroupEntries) / 8);
      }
      int32_t pos = k + 1;   // destinations ascend with the pivot row's columns
      for (int32_t t = 0; t < cu; ++t) {
        const int32_t j = S.col[dd + 1 + c + t];
        pos = static_cast<int32_t>(std::lower_bound(S.col.begin() + pos, S.col.begin() + tr.lo + tr.len, j) - S.col.begin());
        slice[tile_dest_slot(t)] = static_cast<uint16_t>(pos - tr.lo);
      }
      c += cu;
      if (ri.flags & kItemLast) ++k;
      plan.row_items.push_back(ri);
    }
    if (k != tr.lo + tr.nl) return "internal error: a row's items do not cover its pivots";
  }
  // Claim order: Kahn's algorithm on the tile DAG, ready tiles by (dependency level of the first row,
  // index). Index order alone is topological too but walks one chain of consecutive rows at a time.
  using Key = std::pair<int32_t, int32_t>;
  std::priority_queue<Key, std::vector<Key>, std::greater<Key>> ready;
  for (size_t b = 0; b < nt; ++b) {
    if (indeg[b] == 0) ready.emplace(S.lower_level[plan.rows[raw[b].row_beg].row], static_cast<int32_t>(b));
  }
  plan.tiles.reserve(nt);
  while (!ready.empty()) {
    const int32_t b = ready.top().second;
    ready.pop();
    TileMeta tm{};
    tm.row_beg = raw[b].row_beg;
    tm.nrows = raw[b].nrows;
    tm.ext_beg = static_cast<int32_t>(plan.ext.size());
    tm.n_ext = static_cast<int32_t>(ext[b].size());
    plan.ext.insert(plan.ext.end(), ext[b].begin(), ext[b].end());
    plan.tiles.push_back(tm);
    for (int32_t c : succ[b]) {
      if (--indeg[c] == 0) ready.emplace(S.lower_level[plan.rows[raw[c].row_beg].row], c);
    }
  }
  if (plan.tiles.size() != nt) return "tile dependency graph is not acyclic";
  return "";
}

// Host emulation of the tiled kernel for ONE scenario: `values` holds the scattered matrix on entry
// (rows outside the plan already final) and the factors of the planned rows on return. Walks the tiles
// in claim order and, inside a tile, every row's RowItems with the index arithmetic of the device code
// (destination words, chunk bookkeeping, the spare entry); the arithmetic is the reference's
// (src/numeric.cpp:40-44). Returns the lowest row whose pivot magnitude is <= pivot_floor, -1 for none,
// or <= -2 for a plan that is inconsistent.
inline int64_t emulate_tile_plan(const Schedule& S, const TilePlan& plan, double pivot_floor, double* values) {
  int64_t failed = -1;
  for (const TileMeta& tm : plan.tiles) {
    std::vector<std::vector<double>> row(tm.nrows);
    for (int r = 0; r < tm.nrows; ++r) {
      const TileRow& tr = plan.rows[tm.row_beg + r];
      row[r].assign(values + tr.lo, values + tr.lo + tr.len);
      row[r].resize(tr.len + kTileSpare, 0.0);  // the spare entries
    }
    for (int r = 0; r < tm.nrows; ++r) {  // internal pivots are rows of smaller index: already final
      const TileRow& tr = plan.rows[tm.row_beg + r];
      int32_t k = 0;
      double alpha = 0.0;
      for (int32_t q = tr.ri_beg; q < tr.ri_beg + tr.ri_cnt; ++q) {
        const RowItem& ri = plan.row_items[q];
        const double* src;
        int64_t avail;  // entries that may be read behind src
        if (ri.flags & kItemInternal) {
          if (static_cast<int>(ri.src) >= r) return -2;
          const TileRow& ow = plan.rows[tm.row_beg + ri.src];
          src = row[ri.src].data() + ow.nl;
          avail = ow.len - ow.nl;
        } else {
          if (static_cast<int32_t>(ri.src) >= tm.n_ext) return -2;
          const ExtItem& ex = plan.ext[tm.ext_beg + ri.src];
          if ((ex.cnt_flags & 0xffffu) != ri.cnt || !((ex.users >> r) & 1u)) return -2;
          src = values + ex.entry;  // what TMA stages
          avail = ri.cnt;
        }
        int32_t cu = static_cast<int32_t>(ri.cnt);
        if (ri.flags & kItemFirst) {
          alpha = row[r][k] / src[0];
          ++src;
          --cu;
          --avail;
        }
        const uint16_t* slice = plan.tdest.data() + static_cast<size_t>(ri.tdest_off) * kTileGroupEntries;
        for (int32_t it = 0; it * kTileIter < cu; ++it) {
          for (int e = 0; e < kTileEntryLanes; ++e) {
            for (int j = 0; j < 2; ++j) {
              const int32_t t = it * kTileIter + kTileEntryLanes * j + e;
              const int32_t ds = slice[tile_dest_slot(t)];
              const double u = t < avail ? src[t] : 12345.0;  // the device reads whatever follows; it lands in the spare entry
              if (t >= cu && ds != tr.len + e) return -4;  // padding goes to the lane's own spare entry
              if (t < cu && ds >= tr.len) return -4;
              const double prod = alpha * u;
              row[r][ds] = row[r][ds] - prod;
            }
          }
        }
        if (ri.flags & kItemLast) {
          row[r][k] = alpha;
          ++k;
        }
      }
      if (k != tr.nl) return -3;
      if (std::fabs(row[r][tr.nl]) <= pivot_floor && (failed < 0 || tr.row < failed)) failed = tr.row;
    }
    for (int r = 0; r < tm.nrows; ++r) {
      const TileRow& tr = plan.rows[tm.row_beg + r];
      std::copy(row[r].begin(), row[r].begin() + tr.len, values + tr.lo);
    }
  }
  return failed;
}

}  // namespace b200lu
