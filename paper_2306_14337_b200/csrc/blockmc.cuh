// K2 batched, row-blocked trailing part with SEVERAL BLOCKS IN FLIGHT PER WARP (experiment, B200LU_BATCH_MC=W).
//
// bfactor_block_kernel (batch.cuh) gives a warp one block of two rows and lets it spin on the ready flag of the
// next pivot row; on the narrow trailing DAG most resident warps are waiting at any moment, and the time of the
// launch falls as more blocks are resident (296 CTAs 24.3 ms, 148 CTAs 29.9 ms at C2 x 256) — but registers and
// the 12.5 KB pivot-row stage cap the residency at 16 warps per SM. Here a warp owns W block CONTEXTS (64 bytes of
// shared memory each: block, unit, position in the merged pivot list, the rows' progress) and ONE stage: it advances
// a context while the flags of its pivots are set and moves on to the next context at the first pivot that is not
// ready, instead of waiting. Blocks in flight = W x warps at the register / shared-memory cost of one.
// MEASURED (C2, factor phase): 256 scenarios 31.6 / 31.9 / 32.5 ms with W = 2 / 4 / 8 against 24.4 ms; 32 scenarios
// 10.5-11.1 ms against 8.1 ms. More blocks in flight per warp do not help: what the CTA sweep measured is the number of
// warps that EXECUTE side by side, and a warp that interleaves blocks only serialises them (plus a context reload of
// three dependent loads per switch). Kept as an experiment, off.
// The arithmetic, the reductions and their order per address are those of bfactor_block_kernel (bit-exact for the
// same reason); nothing ever waits, so the claim order needs no residency argument: the lowest unfinished block in
// ticket order is always claimed and all its pivots are ready.
#pragma once

#include "batch.cuh"

namespace b200lu {

constexpr int kMcMaxContexts = 8;
struct McCtx {  // 64 bytes
  int32_t b, u, t, mend;
  int32_t k[2], row[2], lo[2], nl[2];
  int64_t p[2];
};
__host__ __device__ constexpr size_t mc_smem_bytes(int contexts) {
  return 8 * (block_stage_doubles() * sizeof(double) + static_cast<size_t>(contexts) * sizeof(McCtx));
}

template <typename DestT, int MINB>
__global__ void __launch_bounds__(256, MINB)
bfactor_block_mc_kernel(const BBlockArgs a, const int contexts) {
  constexpr int R = 2;
  static_assert(kBlockRows == 2 && kBlockStage > 0, "the multi-context variant is written for staged 2-row blocks");
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const DestT* __restrict__ dest = static_cast<const DestT*>(a.dest);
  extern __shared__ __align__(16) double mc_smem[];
  double* stage = mc_smem + static_cast<size_t>(warp) * block_stage_doubles();
  McCtx* ctx = reinterpret_cast<McCtx*>(mc_smem + 8 * block_stage_doubles()) + warp * contexts;
  const unsigned long long total = static_cast<unsigned long long>(a.n_blocks) * a.units_here;

  // claims the next ticket into context c; returns false when the tickets are exhausted
  auto claim = [&](int c) -> bool {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(a.ticket, 1ull);
    t = __shfl_sync(full, t, 0);
    if (t >= total) {
      if (lane == 0) ctx[c].b = -1;
      __syncwarp();
      return false;
    }
    const int32_t b = static_cast<int32_t>(t / a.units_here);
    const int32_t u = a.first_unit + static_cast<int32_t>(t - static_cast<unsigned long long>(b) * a.units_here);
    if (lane == 0) {
      const int4 b0 = __ldg(reinterpret_cast<const int4*>(a.blocks + b));
      const int4 b1 = __ldg(reinterpret_cast<const int4*>(a.blocks + b) + 1);
      McCtx& x = ctx[c];
      x.b = b;
      x.u = u;
      x.t = b1.x;
      x.mend = b1.y;
      const int32_t rows[2] = {b0.x, b0.y};
      for (int r = 0; r < R; ++r) {
        const int32_t i = max(rows[r], 0);
        const int32_t lo = __ldg(a.row_ptr + i);
        x.row[r] = rows[r];
        x.lo[r] = lo;
        x.nl[r] = __ldg(a.diag + i) - lo;
        x.p[r] = a.pair_row_ptr[i];
        x.k[r] = 0;
      }
    }
    __syncwarp();
    return true;
  };

  int live = 0;
  for (int c = 0; c < contexts; ++c) live += claim(c) ? 1 : 0;
  int c = 0, idle_round = 0;
  while (live > 0) {
    if (ctx[c].b < 0) {
      c = c + 1 == contexts ? 0 : c + 1;
      continue;
    }
    // ---- resume context c
    const int32_t u = ctx[c].u;
    int32_t t0 = ctx[c].t;
    const int32_t mend = ctx[c].mend;
    int32_t rows[R], nl[R], k[R];
    int64_t p[R];
    double* rowg[R];
    const int32_t sc0 = u * 32;
    double* gbase = a.values + static_cast<int64_t>(sc0 >> 5) * a.nnz_factors * 32 + lane;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      rows[r] = ctx[c].row[r];
      nl[r] = ctx[c].nl[r];
      k[r] = ctx[c].k[r];
      p[r] = ctx[c].p[r];
      rowg[r] = gbase + static_cast<int64_t>(ctx[c].lo[r]) * 32;
    }
    __syncwarp();
    bool blocked = false;
    int32_t advanced = 0;
    while (t0 < mend && !blocked) {
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
      int32_t q = 0;
      for (; q < cnt; ++q) {
        const int32_t dd = __shfl_sync(full, my_dd, q);
        const int32_t m = __shfl_sync(full, my_m, q);
        const uint32_t bits = __shfl_sync(full, my_bits, q);
        if (!__shfl_sync(full, my_ready, q)) {
          // one more look (the chunk's probe may be old), then move on to another context instead of waiting
          const int32_t d = __shfl_sync(full, my_d, q);
          int32_t now = 0;
          if (lane == 0) now = ld_flag_poll(a.flags + static_cast<int64_t>(d) * a.units + u) >= a.gen;
          now = __shfl_sync(full, now, 0);
          if (!now) {
            blocked = true;
            break;
          }
        }
        const double* ug = gbase + static_cast<int64_t>(dd) * 32;
        __syncwarp();
        const int32_t ns = !(bits & 0x10000u) ? min(m + 1, kBlockStage) : 0;
        if (ns > 0) {
          const double* src = ug - lane;  // warp-uniform start of the pivot row's block for this group
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
          __syncwarp();
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
        int32_t cc = max(ns - 1, 0);
        for (; cc + 7 < m; cc += 8) {
          double uv[8];
          int32_t ds[R][8];
#pragma unroll
          for (int j = 0; j < 8; ++j) uv[j] = ld_cg(ug + static_cast<int64_t>(1 + cc + j) * 32);
#pragma unroll
          for (int r = 0; r < R; ++r) {
#pragma unroll
            for (int j = 0; j < 8; ++j) ds[r][j] = (bits & (1u << r)) ? dest[p[r] + cc + j] : 0;
          }
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (bits & (1u << r)) {
#pragma unroll
              for (int j = 0; j < 8; ++j) red_add_f64(rowg[r] + static_cast<int64_t>(ds[r][j]) * 32, __dmul_rn(nalpha[r], uv[j]));
            }
          }
        }
        for (; cc < m; ++cc) {
          const double uv = ld_cg(ug + static_cast<int64_t>(1 + cc) * 32);
          int32_t ds[R];
#pragma unroll
          for (int r = 0; r < R; ++r) ds[r] = (bits & (1u << r)) ? dest[p[r] + cc] : 0;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (bits & (1u << r)) red_add_f64(rowg[r] + static_cast<int64_t>(ds[r]) * 32, __dmul_rn(nalpha[r], uv));
          }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (bits & (1u << r)) {
            st_cg(rowg[r] + static_cast<int64_t>(k[r]) * 32, -nalpha[r]);  // l_id, src/numeric.cpp:41
            p[r] += m;
            ++k[r];
          }
        }
        if ((bits >> 8) & 0xffu) {  // rows whose last pivot this was: pivot check (src/numeric.cpp:48) and publication
          __syncwarp();
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (bits & (256u << r)) {
              if (fabs(ld_cg(rowg[r] + static_cast<int64_t>(nl[r]) * 32)) <= a.pivot_floor) atomicMin(a.failed + sc0 + lane, rows[r]);
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
        ++advanced;
      }
      t0 += q;
    }
    __syncwarp();
    if (t0 >= mend) {  // the block is finished: reuse the context
      if (!claim(c)) --live;
      idle_round = 0;
    } else {
      if (lane == 0) {
        ctx[c].t = t0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          ctx[c].k[r] = k[r];
          ctx[c].p[r] = p[r];
        }
      }
      __syncwarp();
      idle_round = advanced ? 0 : idle_round + 1;
      if (idle_round >= contexts) {  // a whole round without progress: every context waits for another warp
        __nanosleep(200);
        idle_round = 0;
      }
    }
    c = c + 1 == contexts ? 0 : c + 1;
  }
}

}  // namespace b200lu
