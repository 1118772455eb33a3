// K2 batched, trailing part: CTA tiles of consecutive rows with the target rows RESIDENT IN SHARED
// MEMORY and the pivot rows streamed once per tile by TMA (sm_100a).
//
// Why. eliminate (src/numeric.cpp:27-58) applies, for every strict-lower entry (i, d) of row i in
// ascending d, a_ij <- a_ij - (a_id / u_dd) * u_dj over the upper entries of row d. In a scenario batch
// the row-per-warp kernels (batch.cuh) sent every one of those updates to L2 as a reduction: 12 G
// updates = 96 GB through the L2 atomic unit per refactorization at C2 x 256, the unit 70 % busy, and
// every pivot row re-read from L2/DRAM once per consumer row (19 on average). Here
//   * a unit of work is (tile of up to R index-consecutive rows) x (8 scenarios); every row of the
//     tile lives in shared memory from its first update to its last, so an update is a plain ordered
//     read-modify-write of shared memory — one owner warp per row, pivots in ascending order, the same
//     two roundings as the reference: bit-exact by construction — and the row is read from and written
//     to HBM exactly once;
//   * the rows of a tile share most of their pivots (consecutive rows of the trailing part are
//     ancestors of the same subtrees: measured reuse 5.3x at R = 8, 7.8x at R = 16 on the C2 pattern),
//     so each pivot row is fetched ONCE per tile: a producer warp walks the ascending merge of the
//     tile's pivot lists, waits for the pivot row's ready flag (ld.acquire), and issues one 2-D TMA
//     copy (cp.async.bulk.tensor, box = 8 scenarios x up to 96 entries) into a ring of stages guarded
//     by mbarriers; the consumer warps never touch global memory for a pivot row;
//   * a pivot that is itself a row of the tile is read straight from its owner's shared-memory copy
//     (hand-off through a shared-memory flag: the chain of consecutive rows advances at on-chip latency
//     inside a tile and crosses L2 once per tile);
//   * lanes = 8 entry lanes x 4 scenario pairs: every shared-memory access is 16 bytes (two scenarios of
//     one entry), a pivot row of m entries costs m/8 dependent steps, and the destination offsets of 64
//     entries arrive in one 16-byte load per lane from a table laid out for exactly this access.
// Tiles are claimed with an atomic ticket in a topological order of the tile DAG, so a claimed tile only
// ever waits for rows of tiles that are finished or resident.
#pragma once

#include <cuda.h>

#include "batch.cuh"
#include "tile_plan.hpp"

// Sleep (ns) between polls of the shared-memory progress words; 0 = plain spin.
#ifndef B200LU_TILE_SPIN_NS
#define B200LU_TILE_SPIN_NS 32
#endif

// Optional phase accounting (-DB200LU_TILE_PROF): every warp adds the clock cycles it spends in each phase of
// the tiled kernel to BTileArgs::prof[phase] (16 counters), read back by tools/tile_prof.py.
#ifdef B200LU_TILE_PROF
#define TPROF_DECL long long tprof_t = clock64(); long long tprof_acc[16] = {0}
#define TPROF(ph)                                  \
  do {                                             \
    const long long tprof_n = clock64();           \
    tprof_acc[ph] += tprof_n - tprof_t;            \
    tprof_t = tprof_n;                             \
  } while (0)
#define TPROF_FLUSH(a)                                                                                  \
  do {                                                                                                  \
    if ((threadIdx.x & 31) == 0) {                                                                      \
      for (int tprof_i = 0; tprof_i < 16; ++tprof_i) {                                                  \
        if (tprof_acc[tprof_i]) atomicAdd(reinterpret_cast<unsigned long long*>((a).prof) + tprof_i,    \
                                          static_cast<unsigned long long>(tprof_acc[tprof_i]));         \
      }                                                                                                 \
    }                                                                                                   \
  } while (0)
#else
#define TPROF_DECL
#define TPROF(ph)
#define TPROF_FLUSH(a)
#endif

namespace b200lu {

constexpr int kTileCtlBytes = 1280;
constexpr int kTileBlockDoubles = kTileBoxStep * kTileScen;  // one ring block: 16 entries x 8 scenarios = 1 KB
__host__ __device__ constexpr size_t tile_ring_bytes(int ring_blocks) {  // + over-read slack
  return static_cast<size_t>(ring_blocks) * kTileBlockDoubles * sizeof(double) + 128;
}

struct BTileArgs {
  CUtensorMap maps[kTileMaps];  // values viewed as [groups * nnz_factors][32] doubles, box 8 x (16 * (i + 1))
  int32_t n_tiles, units, gen;
  int32_t rows_smem_bytes;
  const TileMeta* tiles;
  const TileRow* rows;
  const ExtItem* ext;
  const RowItem* row_items;
  const uint4* tdest;           // tile destination table, 16-byte words (tile_plan.hpp)
  double* values;
  int64_t nnz_factors;
  int32_t* flags;               // [n][units] generation per (row, 8-scenario unit)
  double pivot_floor;
  int32_t* failed;
  unsigned long long* ticket;
  long long* prof;              // 16 phase counters (cycles summed over warps), only with -DB200LU_TILE_PROF
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  const uint32_t addr = smem_u32(bar);
  while (!ok) {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok)
                 : "r"(addr), "r"(parity)
                 : "memory");
  }
}
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, int32_t c0, int32_t c1, uint64_t* bar) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
               ::"r"(smem_u32(smem_dst)), "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ int32_t ld_flag_relaxed(const int32_t* p) {
  int32_t v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// 16-byte shared-memory accesses through 32-bit shared addresses: the hot loops keep every address in one
// register and never pay a generic->shared conversion (the compiler rematerialised one per access)
__device__ __forceinline__ double2 lds128(uint32_t addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void sts128(uint32_t addr, double2 v) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(addr), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ int32_t lds32_volatile(uint32_t addr) {
  int32_t v;
  asm volatile("ld.volatile.shared.s32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_s32(int32_t* p, int32_t v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// R consumer warps (= rows of a tile) + 1 producer warp; RB ring blocks of 1 KB; MINB CTAs per SM the register
// allocation must allow.
template <int R, int RB, int MINB>
__global__ void __launch_bounds__((R + 1) * 32, MINB)
bfactor_tile_kernel(const __grid_constant__ BTileArgs a) {
  static_assert(R <= kTileMaxRows, "users mask / control block");
  // dynamic shared memory starts behind the 1 KB the system reserves per CTA: 128-byte aligned, which
  // the TMA destinations need (checked once below)
  extern __shared__ __align__(128) unsigned char tile_smem_raw[];
  unsigned char* base = tile_smem_raw;
  double* ring = reinterpret_cast<double*>(base);  // [block][16 entries][8 scenarios]
  double* rowsm = reinterpret_cast<double*>(base + tile_ring_bytes(RB));
  unsigned char* ctl = reinterpret_cast<unsigned char*>(rowsm) + a.rows_smem_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(ctl);                                // [slots] TMA arrival
  int32_t* released = reinterpret_cast<int32_t*>(ctl + 128);                        // [slots] consumers done with the copy
  int32_t* p_expect = reinterpret_cast<int32_t*>(ctl + 256);                        // [slots] producer: consumers of the copy
  int32_t* p_blocks = reinterpret_cast<int32_t*>(ctl + 320);                        // [slots] producer: ring blocks it holds
  volatile int32_t* done = reinterpret_cast<volatile int32_t*>(ctl + 384);          // [R] row finished (intra-tile hand-off)
  int32_t* uoff = reinterpret_cast<int32_t*>(ctl + 448);                            // [R] entry offset of each row's diagonal
  volatile int32_t* issued = reinterpret_cast<volatile int32_t*>(ctl + 512);        // copies issued so far (monotone over tiles)
  unsigned long long* s_ticket = reinterpret_cast<unsigned long long*>(ctl + 520);
  int4* p_items = reinterpret_cast<int4*>(ctl + 528);                               // [32] producer: records of the current batch
  int32_t* p_ready = reinterpret_cast<int32_t*>(ctl + 528 + 512);                   // [32] producer: flag probe results

  const unsigned fullmask = 0xffffffffu;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sp = lane & 3, e = lane >> 2;  // scenario pair (scenarios 2 sp, 2 sp + 1) and entry lane
  if (threadIdx.x == 0) {
    if (smem_u32(base) & 127u) __trap();
    for (int i = 0; i < kTileSlots; ++i) {
      mbar_init(full + i, 1);
      released[i] = 0;
    }
    *issued = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  int32_t ext_base = 0;  // copies issued for the tiles this CTA has already processed
  const unsigned long long total = static_cast<unsigned long long>(a.n_tiles) * a.units;
  TPROF_DECL;
  while (true) {
    __syncthreads();  // the previous tile is finished: its shared memory may be reused
    TPROF(0);
    // (Claiming the next ticket one tile ahead, to hide the atomic's round trip, measured 46 ms against 27.6:
    // a held ticket delays its dependents for a whole tile.)
    if (threadIdx.x == 0) *s_ticket = atomicAdd(a.ticket, 1ull);
    if (threadIdx.x < R) done[threadIdx.x] = 0;
    __syncthreads();
    const unsigned long long t = *s_ticket;
    TPROF(1);  // end of the previous tile (BAR.SYNC blocks at its first dependent instruction: the waiting for the
               // slowest row and the idle warps of short tiles show up here, not under phase 0) + the claim
    if (t >= total) break;
    const int32_t b = static_cast<int32_t>(t / a.units);
    const int32_t u = static_cast<int32_t>(t - static_cast<unsigned long long>(b) * a.units);
    const int4 tm = __ldg(reinterpret_cast<const int4*>(a.tiles + b));
    const int32_t row_beg = tm.x, nrows = tm.y, ext_beg = tm.z, n_ext = tm.w;
    // unit u = scenarios [8u, 8u + 8): group of 32 = u / 4, quarter = u % 4
    const int64_t group_base = static_cast<int64_t>(u >> 2) * a.nnz_factors;
    double* gq = a.values + group_base * 32 + (u & 3) * kTileScen;

    if (warp == R) {
      // ------------------------------------------------------------ producer warp
      // Lanes fetch the records of 32 copies at a time and probe the ready flags of their pivot rows in
      // parallel; lane 0 then issues the copies in order: ring space (the oldest copies are retired once
      // all their consumers have released them), the flag if the probe found it unset, one TMA copy.
      int32_t head = 0, used = 0, oldest = 0;  // lane 0: ring allocator state of this tile
#ifdef B200LU_EXP_NO_SYNC  // timing experiment: no producer at all
      for (int32_t b0 = 0; b0 < 0; b0 += 32) {
#else
      for (int32_t b0 = 0; b0 < n_ext; b0 += 32) {
#endif
        if (b0 + lane < n_ext) {
          const int4 my = __ldg(reinterpret_cast<const int4*>(a.ext + ext_beg + b0 + lane));
          int32_t ready = 1;
          if ((static_cast<uint32_t>(my.w) >> 16) & kItemWait) {
            ready = ld_flag_relaxed(a.flags + static_cast<int64_t>(my.y) * a.units + u) >= a.gen;
          }
          p_items[lane] = my;
          p_ready[lane] = ready;
        }
        __syncwarp();
        if (lane == 0) {
          const int nq = min(32, n_ext - b0);
          for (int q = 0; q < nq; ++q) {
            const int4 my = p_items[q];
            const int32_t entry = my.x, d = my.y;
            const uint32_t users = static_cast<uint32_t>(my.z), cf = static_cast<uint32_t>(my.w);
            const int32_t x = b0 + q, gx = ext_base + x;
            const int slot = gx & (kTileSlots - 1);
            const int nb = (static_cast<int>(cf & 0xffu) + kTileBoxStep - 1) / kTileBoxStep;  // 1..kTileMaps blocks
            const int start = static_cast<int>(cf >> 24);  // ring positions are static (tile_plan.hpp); only the space is awaited
            const int waste = start < head ? RB - head : 0;  // the planner wrapped: the blocks left at the end are skipped
            TPROF(10);  // producer: bookkeeping
            while (x - oldest >= kTileSlots || used + nb + waste > RB) {
              const int os = (ext_base + oldest) & (kTileSlots - 1);
              while (*reinterpret_cast<volatile int32_t*>(released + os) != p_expect[os]) {
              }
              used -= p_blocks[os];
              ++oldest;
            }
            TPROF(11);  // producer: waiting for ring space (the consumers)
            head = start + nb;
            used += nb + waste;
            *reinterpret_cast<volatile int32_t*>(released + slot) = 0;
            p_expect[slot] = __popc(users);
            p_blocks[slot] = nb + waste;
            // `issued` past gx tells the consumers two things: the slot's previous copy is fully consumed (so the
            // parity of the mbarrier they are about to wait on is unambiguous) and its release counter is reset.
            // It does not have to wait for the copy itself: a consumer that comes early sleeps on the mbarrier.
            __threadfence_block();
            *issued = gx + 1;
            TPROF(10);
            if (!p_ready[q]) {
              const int32_t* f = a.flags + static_cast<int64_t>(d) * a.units + u;
              unsigned ns = 32;
              while (ld_flag_relaxed(f) < a.gen) {
                __nanosleep(ns);
                ns = min(ns * 2, 256u);
              }
            }
            TPROF(12);  // producer: waiting for a pivot row of another tile
            // The flag is read with a RELAXED gpu-scope load and followed by a generic->async proxy fence,
            // not by an acquire: the only reader of the data the flag guards is the TMA engine (async proxy,
            // served by L2, where the owner's fenced stores already are when the flag is visible); no thread of
            // this kernel reads a pivot row of another tile through the generic proxy, so the L1 invalidation
            // that ld.acquire.gpu costs (LDG.STRONG + CCTL.IVALL, measured: the top stall of this warp) would
            // protect nothing.
            // Only a pivot row finished by THIS launch needs the fence (the rows of the head launch and of the
            // scatter pass crossed a kernel boundary).
            if ((cf >> 16) & kItemWait) asm volatile("fence.proxy.async.global;" ::: "memory");
#ifdef B200LU_EXP_NO_TMA  // timing experiment: no copy, the consumers read whatever is in the ring
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(full + slot)) : "memory");
#else
            mbar_arrive_expect_tx(full + slot, static_cast<uint32_t>(nb * kTileBlockDoubles * sizeof(double)));
            tma_load_2d(ring + static_cast<size_t>(start) * kTileBlockDoubles, &a.maps[nb - 1], (u & 3) * kTileScen,
                        static_cast<int32_t>(group_base + entry), full + slot);
#endif
            TPROF(13);  // producer: fence + copy issue
          }
        }
        __syncwarp();
      }
    } else if (warp < nrows) {
      TPROF(15);
      // ------------------------------------------------------------ consumer: one row of the tile
      const int4 r0 = __ldg(reinterpret_cast<const int4*>(a.rows + row_beg + warp));
      const int4 r1 = __ldg(reinterpret_cast<const int4*>(a.rows + row_beg + warp) + 1);
      const int32_t i = r0.x, lo = r0.y, len = r0.z, nl = r0.w;
      const int32_t ri_beg = r1.x, ri_cnt = r1.y;
      double* myrow = rowsm + static_cast<size_t>(r1.z) * kTileScen;
      double* myrow2 = myrow + 2 * sp;  // this lane's two scenarios of entry 0
      double* grow = gq + static_cast<int64_t>(lo) * 32;
      if (lane == 0) uoff[warp] = r1.z + nl;  // read by the other rows only behind done[warp]
      // the row as the scatter pass left it: global -> shared, 16 bytes per lane, 8 entries per instruction
      for (int32_t j = lane >> 2; j < len; j += 8) {
        cp_async_16(myrow + static_cast<size_t>(j) * kTileScen + (lane & 3) * 2, grow + static_cast<int64_t>(j) * 32 + (lane & 3) * 2);
      }
      *reinterpret_cast<double2*>(myrow2 + static_cast<size_t>(len + e) * kTileScen) = make_double2(0.0, 0.0);  // this lane's spare entry
      cp_async_commit_wait_all();
      __syncwarp();
      TPROF(2);  // row load

      const uint32_t ring_a = smem_u32(ring), rows_a = smem_u32(rowsm), my2_a = smem_u32(myrow2);
      const uint32_t issued_a = smem_u32(const_cast<int32_t*>(issued));
      const uint32_t done_a = smem_u32(const_cast<int32_t*>(done)), uoff_a = smem_u32(uoff);
      int32_t k = 0;  // pivots of this row applied so far
      double2 alpha = make_double2(0.0, 0.0);
      for (int32_t b0 = 0; b0 < ri_cnt; b0 += 32) {
        int4 mine = make_int4(0, 0, 0, 0);
        if (b0 + lane < ri_cnt) mine = __ldg(reinterpret_cast<const int4*>(a.row_items + ri_beg + b0 + lane));
        const int nq = min(32, ri_cnt - b0);
        // the destinations of an item's first four steps (64 entries) are requested one item ahead
        uint32_t toff = static_cast<uint32_t>(__shfl_sync(fullmask, mine.x, 0));
        uint4 wd_next = __ldg(a.tdest + static_cast<size_t>(toff) * kTileEntryLanes + e);
        for (int q = 0; q < nq; ++q) {
          const int32_t srcid = __shfl_sync(fullmask, mine.y, q);
          int32_t cnt = __shfl_sync(fullmask, mine.z, q);
          const uint32_t fl = static_cast<uint32_t>(__shfl_sync(fullmask, mine.w, q));
          const uint4* __restrict__ tw = a.tdest + static_cast<size_t>(toff) * kTileEntryLanes + e;
          uint4 wd = wd_next;
          if (q + 1 < nq) {
            toff = static_cast<uint32_t>(__shfl_sync(fullmask, mine.x, q + 1));
            wd_next = __ldg(a.tdest + static_cast<size_t>(toff) * kTileEntryLanes + e);
          }
          const bool internal = (fl & kItemInternal) != 0;
          uint32_t src_a;
          int slot = 0;
          TPROF(3);  // item records, shuffles, destination prefetch
          if (internal) {
#ifndef B200LU_EXP_NO_SYNC
            while (lds32_volatile(done_a + 4 * srcid) == 0) {
              if (B200LU_TILE_SPIN_NS) __nanosleep(B200LU_TILE_SPIN_NS);
            }
#endif
            __threadfence_block();
            src_a = rows_a + static_cast<uint32_t>(lds32_volatile(uoff_a + 4 * srcid)) * (kTileScen * 8);
            TPROF(4);  // waiting for a row of this tile
          } else {
            const int32_t gx = ext_base + srcid;
            slot = gx & (kTileSlots - 1);
#ifndef B200LU_EXP_NO_SYNC
            while (lds32_volatile(issued_a) <= gx) {
              if (B200LU_TILE_SPIN_NS) __nanosleep(B200LU_TILE_SPIN_NS);
            }
            TPROF(5);  // waiting for the producer to reach the item
            mbar_wait(full + slot, static_cast<uint32_t>(gx / kTileSlots) & 1u);
            TPROF(6);  // waiting for the copy to land
#endif
            src_a = ring_a + ((fl >> 8) & 0xffu) * (kTileBlockDoubles * 8);
          }
          uint32_t sl_a = src_a + e * (kTileScen * 8) + sp * 16;
          if (fl & kItemFirst) {
            const double2 aik = lds128(my2_a + k * (kTileScen * 8));
            const double2 udd = lds128(src_a + sp * 16);
            alpha.x = aik.x / udd.x;  // src/numeric.cpp:40
            alpha.y = aik.y / udd.y;
            sl_a += kTileScen * 8;  // the diagonal is entry 0 of a first chunk
            --cnt;
          }
          TPROF(7);  // alpha
#ifdef B200LU_EXP_NO_UPDATES  // timing experiment: waits, alpha and release only
          const int32_t iters = 0;
#else
          const int32_t iters = (cnt + kTileIter - 1) / kTileIter;
#endif
          for (int32_t g0 = 0; g0 < iters; g0 += kTileGroup) {
            const uint32_t ww[4] = {wd.x, wd.y, wd.z, wd.w};
            if (g0 + kTileGroup < iters) wd = __ldg(tw + static_cast<size_t>(g0 / kTileGroup + 1) * kTileEntryLanes);
#pragma unroll
            for (int i2 = 0; i2 < kTileGroup; i2 += 2) {  // two steps at a time: 8 loads in flight, then the arithmetic, then 4 stores
              if (g0 + i2 < iters) {  // warp-uniform
                const bool two = g0 + i2 + 1 < iters;
                const uint32_t up = sl_a + static_cast<uint32_t>(g0 + i2) * (kTileIter * kTileScen * 8);
                const uint32_t p0 = my2_a + (ww[i2] & 0xffffu) * (kTileScen * 8), p1 = my2_a + (ww[i2] >> 16) * (kTileScen * 8);
                const uint32_t p2 = my2_a + (ww[i2 + 1] & 0xffffu) * (kTileScen * 8), p3 = my2_a + (ww[i2 + 1] >> 16) * (kTileScen * 8);
                const double2 u0 = lds128(up), u1 = lds128(up + kTileEntryLanes * kTileScen * 8);
                double2 a0 = lds128(p0), a1 = lds128(p1);
                double2 u2 = make_double2(0.0, 0.0), u3 = u2, a2 = u2, a3 = u2;
                if (two) {
                  u2 = lds128(up + kTileIter * kTileScen * 8);
                  u3 = lds128(up + (kTileIter + kTileEntryLanes) * kTileScen * 8);
                  a2 = lds128(p2);
                  a3 = lds128(p3);
                }
                a0.x = __dsub_rn(a0.x, __dmul_rn(alpha.x, u0.x));  // src/numeric.cpp:44
                a0.y = __dsub_rn(a0.y, __dmul_rn(alpha.y, u0.y));
                a1.x = __dsub_rn(a1.x, __dmul_rn(alpha.x, u1.x));
                a1.y = __dsub_rn(a1.y, __dmul_rn(alpha.y, u1.y));
                sts128(p0, a0);
                sts128(p1, a1);
                if (two) {
                  a2.x = __dsub_rn(a2.x, __dmul_rn(alpha.x, u2.x));
                  a2.y = __dsub_rn(a2.y, __dmul_rn(alpha.y, u2.y));
                  a3.x = __dsub_rn(a3.x, __dmul_rn(alpha.x, u3.x));
                  a3.y = __dsub_rn(a3.y, __dmul_rn(alpha.y, u3.y));
                  sts128(p2, a2);
                  sts128(p3, a3);
                }
              }
            }
          }
          TPROF(8);  // updates
          __syncwarp();  // every lane's updates are in shared memory before the next pivot reads them
#ifndef B200LU_EXP_NO_SYNC
          if (!internal && lane == 0) atomicAdd(released + slot, 1);
#endif
          if (fl & kItemLast) {
            if (e == 0) sts128(my2_a + k * (kTileScen * 8), alpha);  // l_id, src/numeric.cpp:41
            ++k;
          }
        }
      }
      TPROF(3);
      // ---- the row is final. Order: (1) intra-tile hand-off, (2) pivot check, (3) diagonal + upper part to
      // global memory and the ready flag (what other tiles wait for), (4) the lower part.
      __syncwarp();
      __threadfence_block();
      if (lane == 0) done[warp] = 1;
      if (e == 0) {  // src/numeric.cpp:48; the row is published anyway
        const double2 dg = *reinterpret_cast<const double2*>(myrow2 + static_cast<size_t>(nl) * kTileScen);
        if (fabs(dg.x) <= a.pivot_floor) atomicMin(a.failed + u * kTileScen + 2 * sp, i);
        if (fabs(dg.y) <= a.pivot_floor) atomicMin(a.failed + u * kTileScen + 2 * sp + 1, i);
      }
      for (int32_t j = nl + (lane >> 2); j < len; j += 8) {
        const double2 v = *reinterpret_cast<const double2*>(myrow + static_cast<size_t>(j) * kTileScen + (lane & 3) * 2);
        __stcg(reinterpret_cast<double2*>(grow + static_cast<int64_t>(j) * 32 + (lane & 3) * 2), v);
      }
      __syncwarp();
      if (lane == 0) {
        __threadfence();
        st_release_s32(a.flags + static_cast<int64_t>(i) * a.units + u, a.gen);
      }
      for (int32_t j = lane >> 2; j < nl; j += 8) {
        const double2 v = *reinterpret_cast<const double2*>(myrow + static_cast<size_t>(j) * kTileScen + (lane & 3) * 2);
        __stcg(reinterpret_cast<double2*>(grow + static_cast<int64_t>(j) * 32 + (lane & 3) * 2), v);
      }
      TPROF(9);  // publication + write-back
    }
    ext_base += n_ext;
  }
  TPROF_FLUSH(a);
}

}  // namespace b200lu
