// K2 batched, row-blocked trailing part with ONE WARP PER ROW OF A BLOCK (B200LU_BATCH_TEAM=minimum CTAs per SM).
//
// bfactor_block_kernel (batch.cuh) gives one warp both rows of a block: 126 registers and a 12.5 KB pivot-row stage
// per warp, 16 warps per SM — and the resident-CTA sweep shows the launch is bound by how many warps execute side by
// side (296 CTAs 24.3 ms, 148 CTAs 29.9 ms). Here a TEAM of two warps owns the block, one row each: the pivot row is
// staged once per team (by member 0) and applied by each member to its own row, so the registers per warp are those of
// a single row and the stage per warp is halved, at the DRAM / L2 traffic of 2-row blocks. Every row is still updated
// by one thread per scenario, pivots ascending, reductions in program order: bit-exact for the same reason as
// bfactor_block_kernel. The members meet at a named barrier twice per pivot (stage filled / stage free).
#pragma once

#include "batch.cuh"

#ifndef B200LU_TEAM_RMW
#define B200LU_TEAM_RMW 0
#endif

namespace b200lu {

constexpr int kTeamWarps = 8;                        // warps per CTA
constexpr int kTeamSize = kBlockRows;                // warps per team = rows per block (2, or 4 with -DB200LU_BLOCK_ROWS=4)
constexpr int kTeams = kTeamWarps / kTeamSize;       // teams per CTA
__host__ __device__ constexpr size_t team_stage_doubles() { return static_cast<size_t>(kBlockStage) * 32 + kTeamSize * kBlockStageDest; }
__host__ __device__ constexpr size_t team_smem_bytes() { return kTeams * (team_stage_doubles() * sizeof(double) + 16); }

__device__ __forceinline__ void team_barrier(int team) {
  asm volatile("bar.sync %0, %1;" ::"r"(team + 1), "n"(32 * kTeamSize) : "memory");
}

// BULK = true: the pivot row — one contiguous block of (m + 1) x 256 bytes — is staged by ONE bulk asynchronous copy
// (cp.async.bulk, the 1-D form of TMA: SASS UBLKCP) issued by lane 0 of member 0 and awaited on an mbarrier, instead of
// ns / 2 16-byte cp.async per lane. The row was written by other SMs through the generic proxy (reductions, st.cg) and is
// read here by the async proxy: fence.proxy.async.global between the acquired flag and the copy.
__device__ __forceinline__ uint32_t team_smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void team_mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  const uint32_t addr = team_smem_u32(bar);
  while (!ok) {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok)
                 : "r"(addr), "r"(parity)
                 : "memory");
  }
}
__device__ __forceinline__ void team_bulk_copy(double* stage, const double* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("fence.proxy.async.global;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(team_smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(team_smem_u32(stage)), "l"(src), "r"(bytes), "r"(team_smem_u32(bar))
               : "memory");
}

template <typename DestT, int MINB, bool BULK = false>
__global__ void __launch_bounds__(kTeamWarps * 32, MINB)
bfactor_block_team_kernel(const BBlockArgs a) {
  static_assert(kBlockStage > 0, "the team variant stages the pivot rows");
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int team = warp / kTeamSize, me = warp % kTeamSize;  // `me` = the block row this warp owns
  const DestT* __restrict__ dest = static_cast<const DestT*>(a.dest);
  extern __shared__ __align__(16) double team_smem[];
  double* stage = team_smem + static_cast<size_t>(team) * team_stage_doubles();
  unsigned long long* tslot = reinterpret_cast<unsigned long long*>(team_smem + kTeams * team_stage_doubles()) + team * 2;
  const unsigned long long total = static_cast<unsigned long long>(a.n_blocks) * a.units_here;
  uint64_t* bar = reinterpret_cast<uint64_t*>(tslot + 1);  // BULK: arrival of the staged pivot row
  uint32_t ph = 0;                                         // its phase parity: one completion per staged pivot
  if constexpr (BULK) {
    if (me == 0 && lane == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(team_smem_u32(bar)) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    team_barrier(team);
  }
  while (true) {
    if (me == 0 && lane == 0) *tslot = atomicAdd(a.ticket, 1ull);
    team_barrier(team);
    const unsigned long long t = *tslot;
    team_barrier(team);  // both members have read the slot before the next claim overwrites it
    if (t >= total) break;
    const int32_t b = static_cast<int32_t>(t / a.units_here);
    const int32_t u = a.first_unit + static_cast<int32_t>(t - static_cast<unsigned long long>(b) * a.units_here);
    const int4 b0 = __ldg(reinterpret_cast<const int4*>(a.blocks + b));
    const int4 b1 = __ldg(reinterpret_cast<const int4*>(a.blocks + b) + 1);
    const int32_t rows4[4] = {b0.x, b0.y, b0.z, b0.w};
    const int32_t myrow = rows4[me];  // -1: the block is short of rows (this member just keeps step)
    const int32_t mbeg = b1.x, mend = b1.y;
    const int32_t sc0 = u * 32;
    double* gbase = a.values + static_cast<int64_t>(u) * a.nnz_factors * 32 + lane;
    const int32_t irow = max(myrow, 0);
    const int32_t lo = __ldg(a.row_ptr + irow);
    double* rowg = gbase + static_cast<int64_t>(lo) * 32;
    const int32_t nl = __ldg(a.diag + irow) - lo;
    int64_t p = a.pair_row_ptr[irow];
    int32_t k = 0;
    const uint32_t mybit = myrow >= 0 ? (1u << me) : 0u;

    for (int32_t t0 = mbeg; t0 < mend; t0 += 32) {
      int32_t my_d = 0, my_dd = 0, my_m = 0, my_ready = 0;
      uint32_t my_bits = 0;
      if (t0 + lane < mend) {
        const int2 mp = __ldg(reinterpret_cast<const int2*>(a.merged) + t0 + lane);
        my_d = mp.x;
        my_bits = static_cast<uint32_t>(mp.y);
        my_dd = __ldg(a.diag + my_d);
        my_m = __ldg(a.row_ptr + my_d + 1) - my_dd - 1;
        if (me == 0) my_ready = ld_acquire_s32(a.flags + static_cast<int64_t>(my_d) * a.units + u) >= a.gen;
      }
      __syncwarp();
      const int32_t cnt = min(32, mend - t0);
      for (int32_t q = 0; q < cnt; ++q) {
        const int32_t dd = __shfl_sync(full, my_dd, q);
        const int32_t m = __shfl_sync(full, my_m, q);
        const uint32_t bits = __shfl_sync(full, my_bits, q);
        const bool mine = (bits & mybit) != 0;
        const double* ug = gbase + static_cast<int64_t>(dd) * 32;
        const int32_t ns = min(m + 1, kBlockStage);  // staged entries of the pivot row (diagonal included)
        // member 0 awaits the pivot row's flag and stages it for the team; each member stages its own destination slice
        if (me == 0) {
          // (a pivot that is a row of this block — bit 16 — is member 0's own row, published earlier in program order)
          if (!__shfl_sync(full, my_ready, q) && !(bits & 0x10000u)) {
            const int32_t d = __shfl_sync(full, my_d, q);
            wait_flag(a.flags + static_cast<int64_t>(d) * a.units + u, a.gen);
          }
          __syncwarp();
          const double* src = ug - lane;
          if constexpr (BULK) {
            if (lane == 0) team_bulk_copy(stage, src, static_cast<uint32_t>(ns) * 256u, bar);
          } else {
            for (int32_t t16 = lane; t16 < ns * 16; t16 += 32) cp_async_16(stage + t16 * 2, src + t16 * 2);
          }
        }
        if (mine) {
          const char* dsrc = reinterpret_cast<const char*>(dest + p);
          const int32_t shift = static_cast<int32_t>(reinterpret_cast<uintptr_t>(dsrc) & 3);
          const int32_t words = (static_cast<int32_t>((ns - 1) * sizeof(DestT)) + shift + 3) >> 2;
          uint32_t* ddst = reinterpret_cast<uint32_t*>(stage + kBlockStage * 32 + me * kBlockStageDest);
          for (int32_t t4 = lane; t4 < words; t4 += 32) cp_async_4(ddst + t4, dsrc - shift + 4 * t4);
        }
        // a_id is read while the copies are in flight (every earlier reduction to it was issued by this thread)
        double nalpha = 0.0;
        if (mine) nalpha = ld_cg(rowg + static_cast<int64_t>(k) * 32);
        cp_async_commit_wait_all();
        team_barrier(team);  // the stage is filled (and member 0 has acquired the pivot row's flag for both)
        if constexpr (BULK) {  // ... or, with the bulk copy, issued: every thread awaits its arrival
          team_mbar_wait(bar, ph);
          ph ^= 1u;
        }
        if (mine) {
          const double udd = stage[lane];
          nalpha = -(nalpha / udd);  // src/numeric.cpp:40; the sign is exact
          const char* dbytes = reinterpret_cast<const char*>(stage + kBlockStage * 32 + me * kBlockStageDest);
          const DestT* dl = reinterpret_cast<const DestT*>(dbytes + (reinterpret_cast<uintptr_t>(dest + p) & 3));
#if B200LU_TEAM_RMW > 0
          // experiment (off): every B200LU_TEAM_RMW-th pivot of a row updates through L2 loads and stores instead of L2
          // reductions (same two roundings; same thread per address, program order) to move work off the L2 atomic unit.
          // Bit-exact, and slower the more pivots take this path — C2 x 256, factor phase: every 2nd pivot 26.5 ms, 3rd 24.5,
          // 4th 23.4, 6th 22.6, none 22.2 (32 scenarios: 6.6 against 5.75): the round trip per load batch costs more than
          // the atomic unit gains
          if (k % B200LU_TEAM_RMW == B200LU_TEAM_RMW - 1) {
            for (int32_t cs = 0; cs < ns - 1; cs += 8) {
              double v[8];
              double* ap[8];
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                ap[j] = rowg + static_cast<int64_t>(dl[min(cs + j, ns - 2)]) * 32;
                v[j] = ld_cg(ap[j]);
              }
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                if (cs + j < ns - 1) st_cg(ap[j], __dadd_rn(v[j], __dmul_rn(nalpha, stage[(1 + cs + j) * 32 + lane])));
              }
            }
          } else
#endif
#pragma unroll 4
          for (int32_t cs = 0; cs < ns - 1; ++cs) {
            red_add_f64(rowg + static_cast<int64_t>(dl[cs]) * 32, __dmul_rn(nalpha, stage[(1 + cs) * 32 + lane]));  // src/numeric.cpp:44
          }
          int32_t cc = ns - 1;
          for (; cc + 7 < m; cc += 8) {  // the part of a long pivot row that did not fit the stage
            double uv[8];
            int32_t ds[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) uv[j] = ld_cg(ug + static_cast<int64_t>(1 + cc + j) * 32);
#pragma unroll
            for (int j = 0; j < 8; ++j) ds[j] = dest[p + cc + j];
#pragma unroll
            for (int j = 0; j < 8; ++j) red_add_f64(rowg + static_cast<int64_t>(ds[j]) * 32, __dmul_rn(nalpha, uv[j]));
          }
          for (; cc < m; ++cc) {
            const double uv = ld_cg(ug + static_cast<int64_t>(1 + cc) * 32);
            red_add_f64(rowg + static_cast<int64_t>(dest[p + cc]) * 32, __dmul_rn(nalpha, uv));
          }
          st_cg(rowg + static_cast<int64_t>(k) * 32, -nalpha);  // l_id, src/numeric.cpp:41
          p += m;
          ++k;
          if (bits & (256u << me)) {  // this row's last pivot: pivot check (src/numeric.cpp:48) and publication
            if (fabs(ld_cg(rowg + static_cast<int64_t>(nl) * 32)) <= a.pivot_floor) atomicMin(a.failed + sc0 + lane, myrow);
            __syncwarp();
            if (lane == 0) {
              __threadfence();
              st_relaxed_s32(a.flags + static_cast<int64_t>(myrow) * a.units + u, a.gen);
            }
          }
        }
        team_barrier(team);  // both members are done with the stage
      }
    }
  }
}

// The same kernel with TWO stages per team: while pivot q is applied, the row of pivot q + 1 (if its flag is already set)
// is on its way into the other stage, and one barrier per pivot is enough — "stage q filled" also says that everybody
// has left stage q - 1. A prefetch never waits for a flag (the next pivot may be a row of this very block, published only
// when pivot q has been applied): member 0 looks, says what it saw in a shared word ahead of the barrier, and both
// members act on that word behind it. Measured (B200LU_BATCH_TEAM_STAGES=2, C2): 22.8 ms at 256 scenarios (single stage: 22.3),
// 5.76 ms at 32 (5.9): on the chain the next pivot is rarely ready early, and at 256 scenarios the launch is no longer
// bound by the hand-offs. Kept as an option; the single-stage kernel is the default.
__host__ __device__ constexpr size_t team2_smem_bytes() { return kTeams * (2 * team_stage_doubles() * sizeof(double) + 32); }

template <typename DestT, int MINB>
__global__ void __launch_bounds__(kTeamWarps * 32, MINB)
bfactor_block_team2_kernel(const BBlockArgs a) {
  static_assert(kBlockStage > 0, "the team variant stages the pivot rows");
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int team = warp / kTeamSize, me = warp % kTeamSize;
  const DestT* __restrict__ dest = static_cast<const DestT*>(a.dest);
  extern __shared__ __align__(16) double team_smem[];
  double* stages = team_smem + static_cast<size_t>(team) * 2 * team_stage_doubles();
  unsigned long long* tslot = reinterpret_cast<unsigned long long*>(team_smem + kTeams * 2 * team_stage_doubles()) + team * 4;
  volatile int32_t* nxt = reinterpret_cast<volatile int32_t*>(tslot + 2);  // [2]: "the next pivot is being prefetched", by parity of the pivot count
  const unsigned long long total = static_cast<unsigned long long>(a.n_blocks) * a.units_here;
  int cur = 0;
  unsigned seq = 0;  // pivots processed by this team (the two words of `nxt` alternate: a member is at most one barrier ahead)
  while (true) {
    if (me == 0 && lane == 0) *tslot = atomicAdd(a.ticket, 1ull);
    team_barrier(team);
    const unsigned long long t = *tslot;
    team_barrier(team);
    if (t >= total) break;
    const int32_t b = static_cast<int32_t>(t / a.units_here);
    const int32_t u = a.first_unit + static_cast<int32_t>(t - static_cast<unsigned long long>(b) * a.units_here);
    const int4 b0 = __ldg(reinterpret_cast<const int4*>(a.blocks + b));
    const int4 b1 = __ldg(reinterpret_cast<const int4*>(a.blocks + b) + 1);
    const int32_t rows4[4] = {b0.x, b0.y, b0.z, b0.w};
    const int32_t myrow = rows4[me];
    const int32_t mbeg = b1.x, mend = b1.y;
    const int32_t sc0 = u * 32;
    double* gbase = a.values + static_cast<int64_t>(u) * a.nnz_factors * 32 + lane;
    const int32_t irow = max(myrow, 0);
    const int32_t lo = __ldg(a.row_ptr + irow);
    double* rowg = gbase + static_cast<int64_t>(lo) * 32;
    const int32_t nl = __ldg(a.diag + irow) - lo;
    int64_t p = a.pair_row_ptr[irow];
    int32_t k = 0;
    const uint32_t mybit = myrow >= 0 ? (1u << me) : 0u;

    // copies of one pivot row (member 0) and of this member's destination slice into stage `st`
    auto issue = [&](double* st, const double* ug, int32_t ns, bool mine, int64_t pp) {
      if (me == 0) {
        const double* src = ug - lane;
        for (int32_t t16 = lane; t16 < ns * 16; t16 += 32) cp_async_16(st + t16 * 2, src + t16 * 2);
      }
      if (mine) {
        const char* dsrc = reinterpret_cast<const char*>(dest + pp);
        const int32_t shift = static_cast<int32_t>(reinterpret_cast<uintptr_t>(dsrc) & 3);
        const int32_t words = (static_cast<int32_t>((ns - 1) * sizeof(DestT)) + shift + 3) >> 2;
        uint32_t* ddst = reinterpret_cast<uint32_t*>(st + kBlockStage * 32 + me * kBlockStageDest);
        for (int32_t t4 = lane; t4 < words; t4 += 32) cp_async_4(ddst + t4, dsrc - shift + 4 * t4);
      }
    };

    for (int32_t t0 = mbeg; t0 < mend; t0 += 32) {
      int32_t my_d = 0, my_dd = 0, my_m = 0, my_ready = 0;
      uint32_t my_bits = 0;
      if (t0 + lane < mend) {
        const int2 mp = __ldg(reinterpret_cast<const int2*>(a.merged) + t0 + lane);
        my_d = mp.x;
        my_bits = static_cast<uint32_t>(mp.y);
        my_dd = __ldg(a.diag + my_d);
        my_m = __ldg(a.row_ptr + my_d + 1) - my_dd - 1;
        if (me == 0) my_ready = ld_acquire_s32(a.flags + static_cast<int64_t>(my_d) * a.units + u) >= a.gen;
      }
      __syncwarp();
      const int32_t cnt = min(32, mend - t0);
      bool have = false;  // the copies of the current pivot were issued one pivot ago
      for (int32_t q = 0; q < cnt; ++q) {
        const int32_t dd = __shfl_sync(full, my_dd, q);
        const int32_t m = __shfl_sync(full, my_m, q);
        const uint32_t bits = __shfl_sync(full, my_bits, q);
        const bool mine = (bits & mybit) != 0;
        const double* ug = gbase + static_cast<int64_t>(dd) * 32;
        const int32_t ns = min(m + 1, kBlockStage);
        double* stage = stages + static_cast<size_t>(cur) * team_stage_doubles();
        if (!have) {
          if (me == 0) {
            if (!__shfl_sync(full, my_ready, q)) {
              const int32_t d = __shfl_sync(full, my_d, q);
              wait_flag(a.flags + static_cast<int64_t>(d) * a.units + u, a.gen);
            }
            __syncwarp();
          }
          issue(stage, ug, ns, mine, p);
        }
        double nalpha = 0.0;
        if (mine) nalpha = ld_cg(rowg + static_cast<int64_t>(k) * 32);
        // member 0 looks at the next pivot's flag (never waits) and tells the team
        const int32_t qn = min(q + 1, cnt - 1);
        if (me == 0) {
          int32_t nx = 0;
          if (q + 1 < cnt) {
            nx = __shfl_sync(full, my_ready, qn);
            if (!nx) {
              const int32_t dn = __shfl_sync(full, my_d, qn);
              if (lane == 0) nx = ld_flag_poll(a.flags + static_cast<int64_t>(dn) * a.units + u) >= a.gen;
              nx = __shfl_sync(full, nx, 0);
            }
          }
          if (lane == 0) nxt[seq & 1] = nx;
        }
        cp_async_commit_wait_all();
        team_barrier(team);  // stage `cur` is filled; everybody has left the other stage
        const bool pre = nxt[seq & 1] != 0;
        ++seq;
        if (pre) {  // the next pivot's row into the other stage, while this one is applied
          const int32_t ddn = __shfl_sync(full, my_dd, qn);
          const int32_t mn = __shfl_sync(full, my_m, qn);
          const uint32_t bitsn = __shfl_sync(full, my_bits, qn);
          issue(stages + static_cast<size_t>(cur ^ 1) * team_stage_doubles(), gbase + static_cast<int64_t>(ddn) * 32, min(mn + 1, kBlockStage),
                (bitsn & mybit) != 0, p + (mine ? m : 0));
        }
        if (mine) {
          const double udd = stage[lane];
          nalpha = -(nalpha / udd);  // src/numeric.cpp:40; the sign is exact
          const char* dbytes = reinterpret_cast<const char*>(stage + kBlockStage * 32 + me * kBlockStageDest);
          const DestT* dl = reinterpret_cast<const DestT*>(dbytes + (reinterpret_cast<uintptr_t>(dest + p) & 3));
#pragma unroll 4
          for (int32_t cs = 0; cs < ns - 1; ++cs) {
            red_add_f64(rowg + static_cast<int64_t>(dl[cs]) * 32, __dmul_rn(nalpha, stage[(1 + cs) * 32 + lane]));  // src/numeric.cpp:44
          }
          int32_t cc = ns - 1;
          for (; cc + 7 < m; cc += 8) {
            double uv[8];
            int32_t ds[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) uv[j] = ld_cg(ug + static_cast<int64_t>(1 + cc + j) * 32);
#pragma unroll
            for (int j = 0; j < 8; ++j) ds[j] = dest[p + cc + j];
#pragma unroll
            for (int j = 0; j < 8; ++j) red_add_f64(rowg + static_cast<int64_t>(ds[j]) * 32, __dmul_rn(nalpha, uv[j]));
          }
          for (; cc < m; ++cc) {
            const double uv = ld_cg(ug + static_cast<int64_t>(1 + cc) * 32);
            red_add_f64(rowg + static_cast<int64_t>(dest[p + cc]) * 32, __dmul_rn(nalpha, uv));
          }
          st_cg(rowg + static_cast<int64_t>(k) * 32, -nalpha);  // l_id, src/numeric.cpp:41
          p += m;
          ++k;
          if (bits & (256u << me)) {
            if (fabs(ld_cg(rowg + static_cast<int64_t>(nl) * 32)) <= a.pivot_floor) atomicMin(a.failed + sc0 + lane, myrow);
            __syncwarp();
            if (lane == 0) {
              __threadfence();
              st_relaxed_s32(a.flags + static_cast<int64_t>(myrow) * a.units + u, a.gen);
            }
          }
        }
        have = pre;
        cur ^= 1;
      }
    }
  }
}

}  // namespace b200lu
