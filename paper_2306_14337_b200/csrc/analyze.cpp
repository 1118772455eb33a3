// Host-side symbolic analysis: MC64 matching/scaling, AMD ordering, the L+U fill pattern,
// diag_pos and the scatter map — the product rlu::symbolic_analyze (src/symbolic.cpp:156-203) hands to the
// numeric path, reproduced BIT FOR BIT (same permutations, same pattern arrays, same scale factors) by
// algorithms whose cost follows the size of the result instead of the reference's
//   * O(N) work per augmenting path in mc64_scale (three std::fill over N, two full scans of the columns,
//     src/matching.cpp:89-91,145-165)                    -> only the columns a search touched are reset/updated;
//   * std::set<(degree, vertex)> erase+insert per degree update in amd_order (src/ordering.cpp:34,112-114)
//                                                        -> one bitmap-tree vertex set per degree, int32 lists;
//   * merging the upper part of EVERY referenced row into row i in fill1_pattern (src/symbolic.cpp:128-143:
//     one touch per update pair, 1.35 G at C4)           -> reachability over PRUNED upper lists (the
//     row-wise form of symmetric pruning): a row d stops contributing beyond its first symmetric partner
//     i' (u_{d,i'} != 0 and l_{i',d} != 0), because everything of row d beyond i' is already part of row i';
//   * RowLookupTable::build (bitmap/hash per row, src/symbolic.cpp:16-71), only needed by the CPU
//     elimination                                        -> not built; the scatter map uses a binary search.
// Nothing here runs on the device and nothing here is used by the numeric kernels: the analysis product
// crosses into b200lu_create as the same plain arrays the reference's product does.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <new>
#include <queue>
#include <set>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "b200lu.h"

namespace {

using i32 = int32_t;
using i64 = int64_t;

struct Csr32 {
  i32 n = 0;
  std::vector<i64> ptr;  // n + 1
  std::vector<i32> col;
};

// Entry (i, j) of A lands at (row_map[i], col_map[j]); every output row sorted by column
// (remap_entries, src/sparse.cpp:149-193). Null map = identity.
Csr32 remap(const Csr32& A, const i32* row_map, const i32* col_map) {
  Csr32 B;
  B.n = A.n;
  B.ptr.assign(A.n + 1, 0);
  B.col.resize(A.col.size());
  for (i32 i = 0; i < A.n; ++i) B.ptr[(row_map ? row_map[i] : i) + 1] += A.ptr[i + 1] - A.ptr[i];
  for (i32 i = 0; i < A.n; ++i) B.ptr[i + 1] += B.ptr[i];
  for (i32 i = 0; i < A.n; ++i) {
    i64 pos = B.ptr[row_map ? row_map[i] : i];
    for (i64 k = A.ptr[i]; k < A.ptr[i + 1]; ++k) B.col[pos++] = col_map ? col_map[A.col[k]] : A.col[k];
  }
  for (i32 i = 0; i < B.n; ++i) std::sort(B.col.begin() + B.ptr[i], B.col.begin() + B.ptr[i + 1]);
  return B;
}

// Pattern of A + A^T (symmetrized_pattern, src/sparse.cpp:231-269).
Csr32 symmetrize(const Csr32& A) {
  const i32 n = A.n;
  std::vector<i64> tptr(n + 1, 0);
  for (i32 c : A.col) tptr[c + 1]++;
  for (i32 i = 0; i < n; ++i) tptr[i + 1] += tptr[i];
  std::vector<i32> tcol(A.col.size());
  std::vector<i64> next(tptr.begin(), tptr.end() - 1);
  for (i32 i = 0; i < n; ++i) {
    for (i64 k = A.ptr[i]; k < A.ptr[i + 1]; ++k) tcol[next[A.col[k]]++] = i;
  }
  Csr32 S;
  S.n = n;
  S.ptr.assign(n + 1, 0);
  S.col.reserve(2 * A.col.size());
  for (i32 i = 0; i < n; ++i) {
    i64 ka = A.ptr[i], kt = tptr[i];
    const i64 ea = A.ptr[i + 1], et = tptr[i + 1];
    while (ka < ea || kt < et) {
      i32 c;
      if (ka < ea && (kt >= et || A.col[ka] <= tcol[kt])) {
        c = A.col[ka++];
        if (kt < et && tcol[kt] == c) ++kt;
      } else {
        c = tcol[kt++];
      }
      S.col.push_back(c);
    }
    S.ptr[i + 1] = static_cast<i64>(S.col.size());
  }
  return S;
}

// Ordered set of integers in [0, n): 64-ary bitmap tree, level k + 1 has one bit per word of level k.
class LevelBitmap {
 public:
  bool empty_storage() const { return lv_.empty(); }
  void init(i32 n) {
    size_t words = (static_cast<size_t>(n) + 63) / 64;
    while (true) {
      lv_.emplace_back(words, 0ull);
      if (words == 1) break;
      words = (words + 63) / 64;
    }
  }
  void set(i32 v) {
    size_t x = static_cast<size_t>(v);
    for (auto& w : lv_) {
      const uint64_t before = w[x >> 6];
      w[x >> 6] = before | (1ull << (x & 63));
      if (before) break;
      x >>= 6;
    }
  }
  void clear(i32 v) {
    size_t x = static_cast<size_t>(v);
    for (auto& w : lv_) {
      w[x >> 6] &= ~(1ull << (x & 63));
      if (w[x >> 6]) break;
      x >>= 6;
    }
  }
  i32 first() const {  // smallest member, -1 when empty
    if (lv_.empty() || lv_.back()[0] == 0) return -1;
    size_t x = 0;
    for (size_t k = lv_.size(); k-- > 0;) x = (x << 6) | static_cast<size_t>(__builtin_ctzll(lv_[k][x]));
    return static_cast<i32>(x);
  }

 private:
  std::vector<std::vector<uint64_t>> lv_;
};
constexpr i32 kDenseDegrees = 96;

// ---------------------------------------------------------------------------------------------------------
// AMD — the reference's quotient-graph variant (src/ordering.cpp:9-122): approximate degree
// min(alive - 1, previous + |L_p| - 1, |A_i| + |L_p| - 1 + sum of external element sizes), no aggressive
// absorption, minimum (degree, vertex) pivot. Same quantities, same tie-break => same order. The pivot
// queue is one ordered vertex set per degree (below).
std::vector<i32> amd_order_fast(const Csr32& S) {
  const i32 n = S.n;
  // Flat storage, laid out for the two inner loops (which are cache-miss bound): the variable neighbours of a vertex are
  // a slice of one array that only ever shrinks in place; its adjacent elements are a short inline list (overflow into a
  // side vector); everything the degree arithmetic reads about an element sits in one 16-byte record.
  struct Elem {
    i32 stamp, external, size, alive;
  };
  constexpr int kInline = 6;
  std::vector<i64> var_beg(n);
  std::vector<i32> var_len(n), var_pool, degree(n, 0), elen(n, 0), einl(static_cast<size_t>(n) * kInline);
  std::vector<std::vector<i32>> eover(n);  // elements beyond the inline capacity (rare)
  std::vector<std::vector<i32>> elem_vars(n);
  std::vector<Elem> einfo(n, Elem{-1, 0, 0, 0});
  std::vector<char> eliminated(n, 0);
  var_pool.reserve(S.col.size());
  for (i32 i = 0; i < n; ++i) {
    var_beg[i] = static_cast<i64>(var_pool.size());
    for (i64 k = S.ptr[i]; k < S.ptr[i + 1]; ++k) {
      if (S.col[k] != i) var_pool.push_back(S.col[k]);
    }
    var_len[i] = static_cast<i32>(static_cast<i64>(var_pool.size()) - var_beg[i]);
    degree[i] = var_len[i];
  }
  auto elem_at = [&](i32 i, i32 q) -> i32& { return q < kInline ? einl[static_cast<size_t>(i) * kInline + q] : eover[i][q - kInline]; };
  // Pivot queue: one ordered vertex set per degree value — a hierarchical bitmap (64-ary, find-first by
  // count-trailing-zeros) for the small degrees almost every vertex has, std::set for the rare large ones.
  // Exact membership (erase old degree, insert new), so the minimum (degree, vertex) costs a handful of words.
  std::vector<LevelBitmap> dense(kDenseDegrees);
  std::vector<std::set<i32>> sparse;
  auto insert = [&](i32 deg, i32 v) {
    if (deg < kDenseDegrees) {
      if (dense[deg].empty_storage()) dense[deg].init(n);
      dense[deg].set(v);
    } else {
      if (static_cast<size_t>(deg - kDenseDegrees) >= sparse.size()) sparse.resize(static_cast<size_t>(deg - kDenseDegrees) + 1);
      sparse[deg - kDenseDegrees].insert(v);
    }
  };
  auto erase = [&](i32 deg, i32 v) {
    if (deg < kDenseDegrees) {
      dense[deg].clear(v);
    } else {
      sparse[deg - kDenseDegrees].erase(v);
    }
  };
  for (i32 i = 0; i < n; ++i) insert(degree[i], i);
  i32 mindeg = 0;
  std::vector<i32> mark(n, -1), pivot_set, order(n);
  for (i32 step = 0; step < n; ++step) {
    i32 p;
    while (true) {  // every vertex alive is in exactly one set, so this terminates
      if (mindeg < kDenseDegrees) {
        p = dense[mindeg].first();
        if (p >= 0) break;
      } else if (!sparse[mindeg - kDenseDegrees].empty()) {
        p = *sparse[mindeg - kDenseDegrees].begin();
        break;
      }
      ++mindeg;
    }
    erase(mindeg, p);
    order[step] = p;
    eliminated[p] = 1;
    // L_p = (A_p ∪ spans of the adjacent elements) \ {p}
    pivot_set.clear();
    mark[p] = step;
    for (i32 q = 0; q < var_len[p]; ++q) {
      const i32 v = var_pool[var_beg[p] + q];
      if (!eliminated[v] && mark[v] != step) {
        mark[v] = step;
        pivot_set.push_back(v);
      }
    }
    for (i32 q = 0; q < elen[p]; ++q) {
      const i32 e = elem_at(p, q);
      for (i32 v : elem_vars[e]) {
        if (mark[v] != step) {
          mark[v] = step;
          pivot_set.push_back(v);
        }
      }
      einfo[e].alive = 0;  // absorbed; its span is never read again
    }
    var_len[p] = 0;
    elen[p] = 0;
    elem_vars[p].assign(pivot_set.begin(), pivot_set.end());  // (the reference sorts the span; nothing below depends on its order)
    einfo[p].alive = 1;
    einfo[p].size = static_cast<i32>(pivot_set.size());

    // |L_e \ L_p| for every live element touching L_p
    for (i32 i : pivot_set) {
      for (i32 q = 0; q < elen[i]; ++q) {
        Elem& E = einfo[elem_at(i, q)];
        if (!E.alive) continue;
        if (E.stamp != step) {
          E.stamp = step;
          E.external = E.size;
        }
        E.external--;
      }
    }
    const i32 alive_after = n - step - 1;
    const i32 lp_minus_self = static_cast<i32>(pivot_set.size()) - 1;
    const i32 bound_world = std::max<i32>(alive_after - 1, 0);
    for (i32 i : pivot_set) {
      i32* av = var_pool.data() + var_beg[i];
      i32 w = 0;
      for (i32 r = 0; r < var_len[i]; ++r) {
        const i32 v = av[r];
        if (!(v == p || mark[v] == step)) av[w++] = v;
      }
      var_len[i] = w;
      i32 we = 0;
      i64 external_sum = 0;
      for (i32 r = 0; r < elen[i]; ++r) {
        const i32 e = elem_at(i, r);
        const Elem& E = einfo[e];
        if (!E.alive) continue;
        elem_at(i, we++) = e;
        external_sum += (E.stamp == step) ? E.external : E.size;
      }
      if (we >= kInline) {
        if (static_cast<i32>(eover[i].size()) < we - kInline + 1) eover[i].resize(static_cast<size_t>(we - kInline + 1));
      }
      elem_at(i, we++) = p;
      elen[i] = we;
      const i64 bound_prev = static_cast<i64>(degree[i]) + lp_minus_self;
      const i64 bound_sets = static_cast<i64>(w) + lp_minus_self + external_sum;
      const i32 nd = static_cast<i32>(std::min<i64>({bound_world, bound_prev, bound_sets}));
      if (nd != degree[i]) {
        erase(degree[i], i);
        degree[i] = nd;
        insert(nd, i);
        mindeg = std::min(mindeg, nd);
      }
    }
  }
  std::vector<i32> forward(n);
  for (i32 k = 0; k < n; ++k) forward[order[k]] = k;
  return forward;
}

// ---------------------------------------------------------------------------------------------------------
// Fill pattern of the combined L+U factors (fill1_pattern, src/symbolic.cpp:95-154), by reachability over
// pruned upper lists. Row i = B_i ∪ ⋃_{d ∈ L(i)} U_d with L(i) = the rows d < i reachable from B_i's lower
// entries through upper entries < i. plen[d] = how many leading upper entries of row d still have to be
// followed: once a row i' with u_{d,i'} != 0 reaches d (so l_{i',d} != 0: a symmetric pair), every entry of
// row d beyond i' is an entry of row i' too, hence for all later rows following d up to and including i' is
// enough and d's own upper part need not be merged again (row i', reached through d, covers it).
struct FillResult {
  std::vector<i64> ptr, diag;
  std::vector<i32> col;
  i64 zero_diag_row = -1;
};

FillResult fill_pattern_fast(const Csr32& B) {
  const i32 n = B.n;
  FillResult F;
  F.ptr.assign(n + 1, 0);
  F.diag.assign(n, 0);
  F.col.reserve(B.col.size() * 4);
  std::vector<i32> plen(n, 0);
  std::vector<char> pruned(n, 0);
  std::vector<i32> mark(n, -1), lower, upper, stack;
  for (i32 i = 0; i < n; ++i) {
    lower.clear();
    upper.clear();
    stack.clear();
    bool has_diag = false;
    for (i64 k = B.ptr[i]; k < B.ptr[i + 1]; ++k) {
      const i32 j = B.col[k];
      mark[j] = i;
      if (j < i) {
        stack.push_back(j);
      } else {
        upper.push_back(j);
        has_diag |= (j == i);
      }
    }
    if (!has_diag) {
      F.zero_diag_row = i;
      return F;
    }
    while (!stack.empty()) {
      const i32 d = stack.back();
      stack.pop_back();
      lower.push_back(d);
      const i32* u = F.col.data() + F.diag[d] + 1;
      if (pruned[d]) {
        for (i32 t = 0, e = plen[d]; t < e; ++t) {  // the last followed entry is < i: its row came before this one
          const i32 j = u[t];
          if (mark[j] != i) {
            mark[j] = i;
            stack.push_back(j);
          }
        }
      } else {
        const i32 len = static_cast<i32>(F.ptr[d + 1] - F.diag[d] - 1);
        for (i32 t = 0; t < len; ++t) {
          const i32 j = u[t];
          if (j == i) {  // symmetric pair (d, i): later rows follow row d up to here only
            pruned[d] = 1;
            plen[d] = t + 1;
          }
          if (mark[j] == i) continue;
          mark[j] = i;
          if (j < i) {
            stack.push_back(j);
          } else {
            upper.push_back(j);
          }
        }
      }
    }
    std::sort(lower.begin(), lower.end());
    std::sort(upper.begin(), upper.end());
    F.col.insert(F.col.end(), lower.begin(), lower.end());
    F.diag[i] = static_cast<i64>(F.col.size());
    F.col.insert(F.col.end(), upper.begin(), upper.end());
    F.ptr[i + 1] = static_cast<i64>(F.col.size());
  }
  return F;
}

// ---------------------------------------------------------------------------------------------------------
// MC64-style matching and scaling (mc64_scale, src/matching.cpp:17-189): log-cost maximum-product matching by
// shortest augmenting paths, duals -> D_r, D_c. Same arithmetic, same queue discipline (std::priority_queue of
// (distance, column) pairs, same pushes in the same order), hence the same matching and the same duals bit for
// bit; what changes is that a search only resets and updates the columns it touched.
struct MatchResult {
  int status = B200LU_OK;
  std::string message;
  std::vector<i64> deficient;
  std::vector<i32> row_match;
  std::vector<double> row_scale, col_scale;
  double matched_product = 0.0;
};

i64 find_entry(const i64* ptr, const i32* col, i32 i, i32 j) {
  const i32* b = col + ptr[i];
  const i32* e = col + ptr[i + 1];
  const i32* it = std::lower_bound(b, e, j);
  return (it == e || *it != j) ? -1 : it - col;
}

MatchResult mc64_fast(i32 n, const i64* ptr, const i32* col, const double* val) {
  constexpr double kInf = std::numeric_limits<double>::infinity();
  MatchResult R;
  const i64 nnz = ptr[n];
  std::vector<double> col_max(n, 0.0);
  for (i64 k = 0; k < nnz; ++k) col_max[col[k]] = std::max(col_max[col[k]], std::fabs(val[k]));
  for (i32 j = 0; j < n; ++j) {
    if (col_max[j] == 0.0) {
      R.status = B200LU_STRUCTURALLY_SINGULAR;
      R.message = "structurally singular: column " + std::to_string(j) + " has no nonzero entries";
      return R;
    }
  }
  std::vector<double> log_col_max(n);
  for (i32 j = 0; j < n; ++j) log_col_max[j] = std::log(col_max[j]);
  std::vector<double> cost(nnz, kInf);
  for (i32 i = 0; i < n; ++i) {
    bool any = false;
    for (i64 k = ptr[i]; k < ptr[i + 1]; ++k) {
      const double a = std::fabs(val[k]);
      if (a > 0.0) {
        cost[k] = log_col_max[col[k]] - std::log(a);
        any = true;
      }
    }
    if (!any) {
      R.status = B200LU_STRUCTURALLY_SINGULAR;
      R.message = "structurally singular: row " + std::to_string(i) + " has no nonzero entries";
      R.deficient = {i};
      return R;
    }
  }
  std::vector<i32> row_match(n, -1), col_match(n, -1);
  std::vector<double> u(n, 0.0), v(n, 0.0);
  for (i32 i = 0; i < n; ++i) {
    double umin = kInf;
    for (i64 k = ptr[i]; k < ptr[i + 1]; ++k) umin = std::min(umin, cost[k]);
    u[i] = umin;
  }
  for (i32 i = 0; i < n; ++i) {
    for (i64 k = ptr[i]; k < ptr[i + 1]; ++k) {
      const i32 j = col[k];
      if (col_match[j] == -1 && cost[k] - u[i] - v[j] == 0.0) {
        row_match[i] = j;
        col_match[j] = i;
        break;
      }
    }
  }
  std::vector<double> dist(n, kInf);
  std::vector<i32> pred_row(n, -1), touched, done;
  std::vector<char> finalized(n, 0);
  using Item = std::pair<double, i64>;  // the reference's (double, index_t) ordering
  for (i32 r = 0; r < n; ++r) {
    if (row_match[r] != -1) continue;
    for (i32 j : touched) {
      dist[j] = kInf;
      pred_row[j] = -1;
      finalized[j] = 0;
    }
    touched.clear();
    done.clear();
    std::priority_queue<Item, std::vector<Item>, std::greater<Item>> pq;
    for (i64 k = ptr[r]; k < ptr[r + 1]; ++k) {
      if (cost[k] == kInf) continue;
      const i32 j = col[k];
      const double d = cost[k] - u[r] - v[j];
      if (d < dist[j]) {
        if (dist[j] == kInf) touched.push_back(j);
        dist[j] = d;
        pred_row[j] = r;
        pq.push({d, j});
      }
    }
    i32 found_col = -1;
    double found_dist = kInf;
    while (!pq.empty()) {
      const auto [d, jj] = pq.top();
      pq.pop();
      const i32 j = static_cast<i32>(jj);
      if (finalized[j] || d > dist[j]) continue;
      finalized[j] = 1;
      done.push_back(j);
      if (col_match[j] == -1) {
        found_col = j;
        found_dist = d;
        break;
      }
      const i32 i2 = col_match[j];
      for (i64 k = ptr[i2]; k < ptr[i2 + 1]; ++k) {
        if (cost[k] == kInf) continue;
        const i32 j2 = col[k];
        if (finalized[j2]) continue;
        const double nd = d + cost[k] - u[i2] - v[j2];
        if (nd < dist[j2]) {
          if (dist[j2] == kInf) touched.push_back(j2);
          dist[j2] = nd;
          pred_row[j2] = i2;
          pq.push({nd, j2});
        }
      }
    }
    if (found_col == -1) {
      R.deficient = {r};
      for (i32 j : done) R.deficient.push_back(col_match[j]);
      std::sort(R.deficient.begin(), R.deficient.end());
      R.status = B200LU_STRUCTURALLY_SINGULAR;
      R.message = "structurally singular: no perfect matching, deficient row set of size " +
                  std::to_string(R.deficient.size()) + " starting at row " + std::to_string(r);
      return R;
    }
    for (i32 j : done) v[j] += dist[j] - found_dist;
    i32 j = found_col;
    while (true) {
      const i32 i = pred_row[j];
      col_match[j] = i;
      std::swap(row_match[i], j);
      if (i == r) break;
    }
    for (i32 jj : done) {
      const i32 i = col_match[jj];
      u[i] = cost[find_entry(ptr, col, i, jj)] - v[jj];
    }
  }
  for (i32 i = 0; i < n; ++i) {
    const i32 j = row_match[i];
    const i64 k = find_entry(ptr, col, i, j);
    u[i] = cost[k] - v[j];
    R.matched_product += std::log(std::fabs(val[k]));
  }
  R.row_scale.resize(n);
  R.col_scale.resize(n);
  for (i32 i = 0; i < n; ++i) R.row_scale[i] = std::exp(u[i]);
  for (i32 j = 0; j < n; ++j) R.col_scale[j] = std::exp(v[j] - log_col_max[j]);
  for (i32 i = 0; i < n; ++i) {  // DiagonalScaling::validate, src/sparse.cpp:99-106
    if (!(R.row_scale[i] > 0.0) || !std::isfinite(R.row_scale[i]) || !(R.col_scale[i] > 0.0) || !std::isfinite(R.col_scale[i])) {
      R.status = B200LU_INVALID_ARGUMENT;
      R.message = "nonpositive or non-finite scale factor";
      return R;
    }
  }
  R.row_match = std::move(row_match);
  return R;
}

}  // namespace

struct b200lu_analysis {
  int status = B200LU_OK;
  std::string message;
  i64 failed_row = -1;
  std::vector<i64> deficient;
  i64 n = 0, fill_count = 0;
  double matched_product = 0.0;
  bool has_match = false;
  std::vector<i64> row_offsets, col_indices, diag_pos, scatter_map, amd_forward, col_perm_forward, src_row_offsets, src_col_indices;
  std::vector<double> scatter_scale, row_scale, col_scale;
  double ms[6] = {0, 0, 0, 0, 0, 0};  // matching, ordering, permutation, fill, scatter map, total
};

#include <chrono>

extern "C" {

b200lu_status b200lu_analyze(int64_t n64, const int64_t* row_offsets, const int64_t* col_indices, const double* values,
                             int use_scaling, int use_amd, b200lu_analysis** out) {
  if (!out) return B200LU_INVALID_ARGUMENT;
  *out = nullptr;
  if (n64 < 0 || !row_offsets || (n64 > 0 && row_offsets[n64] > 0 && !col_indices)) return B200LU_INVALID_ARGUMENT;
  if (n64 >= (int64_t{1} << 31) - 1 || row_offsets[n64] < 0 || row_offsets[n64] >= (int64_t{1} << 31)) return B200LU_INVALID_ARGUMENT;
  b200lu_analysis* a = new (std::nothrow) b200lu_analysis();
  if (!a) return B200LU_INVALID_ARGUMENT;
  *out = a;
  const auto clock = [] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  const double t_begin = clock();
  const i32 n = static_cast<i32>(n64);
  a->n = n;
  const i64 nnz = row_offsets[n];
  // CsrMatrix::check_structure, src/sparse.cpp:41-66
  auto fail = [&](b200lu_status st, std::string msg) {
    a->status = st;
    a->message = std::move(msg);
    return st;
  };
  if (row_offsets[0] != 0) return fail(B200LU_INVALID_ARGUMENT, "row_offsets[0] must be 0");
  for (i32 i = 0; i < n; ++i) {
    if (row_offsets[i + 1] < row_offsets[i]) return fail(B200LU_INVALID_ARGUMENT, "row_offsets not monotone at row " + std::to_string(i));
    for (i64 k = row_offsets[i]; k < row_offsets[i + 1]; ++k) {
      if (col_indices[k] < 0 || col_indices[k] >= n) return fail(B200LU_INVALID_ARGUMENT, "column index out of range in row " + std::to_string(i));
      if (k > row_offsets[i] && col_indices[k] <= col_indices[k - 1]) {
        return fail(B200LU_INVALID_ARGUMENT, "column indices not strictly increasing in row " + std::to_string(i));
      }
    }
  }
  if (use_scaling && !values) return fail(B200LU_INVALID_ARGUMENT, "mc64_scale: matrix has no values");
  Csr32 A;
  A.n = n;
  A.ptr.assign(row_offsets, row_offsets + n + 1);
  A.col.resize(nnz);
  for (i64 k = 0; k < nnz; ++k) A.col[k] = static_cast<i32>(col_indices[k]);
  a->src_row_offsets = A.ptr;
  a->src_col_indices.assign(col_indices, col_indices + nnz);

  double t0 = clock();
  std::vector<i32> colperm;  // match->col_perm.forward
  if (use_scaling) {
    MatchResult m = mc64_fast(n, A.ptr.data(), A.col.data(), values);
    if (m.status != B200LU_OK) {
      a->deficient = std::move(m.deficient);
      if (!a->deficient.empty()) a->failed_row = a->deficient.front();
      return fail(static_cast<b200lu_status>(m.status), m.message);
    }
    colperm.resize(n);
    for (i32 i = 0; i < n; ++i) colperm[m.row_match[i]] = i;
    a->has_match = true;
    a->matched_product = m.matched_product;
    a->row_scale = std::move(m.row_scale);
    a->col_scale = std::move(m.col_scale);
    a->col_perm_forward.assign(colperm.begin(), colperm.end());
  }
  a->ms[0] = clock() - t0;
  t0 = clock();
  Csr32 permuted_store;
  const Csr32* permuted = &A;
  if (use_scaling) {
    permuted_store = remap(A, nullptr, colperm.data());
    permuted = &permuted_store;
  }
  std::vector<i32> amd(n);
  if (use_amd) {
    amd = amd_order_fast(symmetrize(*permuted));
  } else {
    for (i32 i = 0; i < n; ++i) amd[i] = i;
  }
  a->amd_forward.assign(amd.begin(), amd.end());
  a->ms[1] = clock() - t0;
  t0 = clock();
  const Csr32 B = remap(*permuted, amd.data(), amd.data());
  a->ms[2] = clock() - t0;
  t0 = clock();
  FillResult F = fill_pattern_fast(B);
  if (F.zero_diag_row >= 0) {
    a->failed_row = F.zero_diag_row;
    return fail(B200LU_ZERO_DIAGONAL, "structurally zero diagonal at row " + std::to_string(F.zero_diag_row));
  }
  a->fill_count = static_cast<i64>(F.col.size()) - nnz;
  a->ms[3] = clock() - t0;
  t0 = clock();
  // scatter map and scale (src/symbolic.cpp:182-201)
  a->scatter_map.resize(nnz);
  a->scatter_scale.assign(nnz, 1.0);
  {
    // rows are independent: split over host threads (the only multi-threaded stage; the result does not depend on it)
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    const unsigned nt = nnz < (i64{1} << 18) ? 1u : hw;
    std::vector<char> bad(nt, 0);
    auto work = [&](unsigned t) {
      const i32 lo = static_cast<i32>(static_cast<i64>(n) * t / nt), hi = static_cast<i32>(static_cast<i64>(n) * (t + 1) / nt);
      for (i32 i = lo; i < hi; ++i) {
        const i32 r = amd[i];
        for (i64 k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
          const i32 j = A.col[k];
          const i32 c = amd[use_scaling ? colperm[j] : j];
          const i64 slot = find_entry(F.ptr.data(), F.col.data(), r, c);
          if (slot < 0) bad[t] = 1;
          a->scatter_map[k] = slot;
          if (use_scaling) a->scatter_scale[k] = a->row_scale[i] * a->col_scale[j];
        }
      }
    };
    if (nt == 1) {
      work(0);
    } else {
      std::vector<std::thread> pool;
      for (unsigned t = 0; t < nt; ++t) pool.emplace_back(work, t);
      for (auto& th : pool) th.join();
    }
    for (char b : bad) {
      if (b) return fail(B200LU_INVALID_ARGUMENT, "combined pattern must contain every source entry");
    }
  }
  a->row_offsets = std::move(F.ptr);
  a->diag_pos = std::move(F.diag);
  a->col_indices.assign(F.col.begin(), F.col.end());
  a->ms[4] = clock() - t0;
  a->ms[5] = clock() - t_begin;
  return B200LU_OK;
}

b200lu_status b200lu_analysis_status(const b200lu_analysis* a, int64_t* failed_row, const int64_t** deficient_rows,
                                     int64_t* deficient_count) {
  if (!a) return B200LU_INVALID_ARGUMENT;
  if (failed_row) *failed_row = a->failed_row;
  if (deficient_rows) *deficient_rows = a->deficient.data();
  if (deficient_count) *deficient_count = static_cast<int64_t>(a->deficient.size());
  return static_cast<b200lu_status>(a->status);
}

const char* b200lu_analysis_message(const b200lu_analysis* a) { return a ? a->message.c_str() : ""; }

b200lu_status b200lu_analysis_view(const b200lu_analysis* a, b200lu_symbolic_view* view, int64_t* fill_count) {
  if (!a || !view) return B200LU_INVALID_ARGUMENT;
  if (a->status != B200LU_OK) return static_cast<b200lu_status>(a->status);
  view->n = a->n;
  view->nnz_factors = static_cast<int64_t>(a->col_indices.size());
  view->nnz_source = static_cast<int64_t>(a->scatter_map.size());
  view->row_offsets = a->row_offsets.data();
  view->col_indices = a->col_indices.data();
  view->diag_pos = a->diag_pos.data();
  view->scatter_map = a->scatter_map.data();
  view->scatter_scale = a->scatter_scale.data();
  view->amd_forward = a->amd_forward.data();
  view->col_perm_forward = a->has_match ? a->col_perm_forward.data() : nullptr;
  view->row_scale = a->has_match ? a->row_scale.data() : nullptr;
  view->col_scale = a->has_match ? a->col_scale.data() : nullptr;
  view->source_row_offsets = a->src_row_offsets.data();
  view->source_col_indices = a->src_col_indices.data();
  if (fill_count) *fill_count = a->fill_count;
  return B200LU_OK;
}

b200lu_status b200lu_analysis_times(const b200lu_analysis* a, double* ms_out6, double* matched_product) {
  if (!a) return B200LU_INVALID_ARGUMENT;
  if (ms_out6) {
    for (int i = 0; i < 6; ++i) ms_out6[i] = a->ms[i];
  }
  if (matched_product) *matched_product = a->matched_product;
  return B200LU_OK;
}

void b200lu_analysis_destroy(b200lu_analysis* a) { delete a; }

}  // extern "C"
