// K2 batched, trailing part, GATHER form (plan: gather_plan.hpp): a warp owns a block of R consecutive rows
// x 32 scenarios (lane = scenario) and interprets the block's record stream. Every target entry a batch of up
// to K pivots touches is loaded once, updated in a register in ascending pivot order — acc <- acc - l * u as a
// product rounded on its own and a subtraction, src/numeric.cpp:44 — and stored once; the batch's multipliers
// l[r][e] live in the warp's shared-memory slot (each lane reads and writes only its own scenario's column of it:
// no warp-level synchronisation anywhere in the arithmetic). Against the row-blocked kernel (batch.cuh) this
// removes every L2 reduction (96 GB through the L2 atomic unit per refactorization at C2 x 256, the unit that
// bounded it) and replaces the per-update traffic on the target rows by one load + one store per (target, batch).
//
// Loads run ahead of the arithmetic: the lanes hold one 8-byte record each (a window of 32), the value loads of
// the next 8 records are in flight while the current 8 are consumed, and the next window's records are requested
// a window ahead. A batch's loads never alias its stores (gather_plan.hpp), and the pipeline is drained at every
// batch boundary, where the ready flags of the batch's pivot rows are awaited (ld.acquire.gpu, one row per lane).
// Every access to `values` is served by L2 (ld.relaxed.gpu / st.global.cg), as in the other batch kernels.
#pragma once

#include "batch.cuh"
#include "gather_plan.hpp"

namespace b200lu {

struct BGatherArgs {
  int32_t n_blocks, units, gen;
  const GBlock* blocks;
  const GBatch* batches;
  const GRec* recs;
  const int32_t* waits;
  const int32_t* diag;
  double* values;
  int64_t nnz_factors;
  int32_t* flags;
  double pivot_floor;
  int32_t* failed;
  unsigned long long* ticket;
  int32_t exp_nowait;  // timing experiment (B200LU_GATHER_NOWAIT): skip the flag waits, results are garbage
};

__host__ __device__ constexpr size_t gather_smem_bytes(int R, int K, int warps) {
  return static_cast<size_t>(R) * K * 32 * sizeof(double) * warps;
}

template <int R, int K, int MINB>
__global__ void __launch_bounds__(256, MINB)
bfactor_gather_kernel(const BGatherArgs a) {
  constexpr int kChunk = 8;
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  extern __shared__ __align__(16) double gather_smem[];
  double* L = gather_smem + static_cast<size_t>(threadIdx.x >> 5) * (R * K * 32) + lane;  // l[r][e] at L[(r * K + e) * 32]
  const unsigned long long total = static_cast<unsigned long long>(a.n_blocks) * a.units;
  while (true) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(a.ticket, 1ull);
    t = __shfl_sync(full, t, 0);
    if (t >= total) break;
    const int32_t b = static_cast<int32_t>(t / a.units);
    const int32_t u = static_cast<int32_t>(t - static_cast<unsigned long long>(b) * a.units);
    const int2 blk = __ldg(reinterpret_cast<const int2*>(a.blocks + b));
    double* g = a.values + static_cast<int64_t>(u) * a.nnz_factors * 32 + lane;
    double acc[R], dg[R];
    uint32_t dst[R];
    uint32_t live = 0, dmask = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      acc[r] = 0.0;
      dg[r] = 1.0;
      dst[r] = 0;
    }

    // value loads of records [q0, q0 + 8) of the window held in `rec`
    auto issue = [&](const uint2& rec, int q0, double (&v)[kChunk]) {
#pragma unroll
      for (int j = 0; j < kChunk; ++j) {
        const uint32_t slot = __shfl_sync(full, rec.x, q0 + j);
        const uint32_t type = __shfl_sync(full, rec.y, q0 + j) & 7u;
        if (type - 1u < 3u) v[j] = ld_cg(g + static_cast<int64_t>(slot) * 32);  // INIT / UPD / DIV
      }
    };
    auto consume = [&](const uint2& rec, int q0, const double (&v)[kChunk]) {
#pragma unroll
      for (int j = 0; j < kChunk; ++j) {
        const uint32_t info = __shfl_sync(full, rec.y, q0 + j);
        const uint32_t type = info & 7u;
        if (type == kGUpd) {
          const uint32_t e = (info >> 8) & 63u;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (info & (16u << r)) acc[r] = __dsub_rn(acc[r], __dmul_rn(L[(r * K + e) * 32], v[j]));  // src/numeric.cpp:44
          }
        } else if (type == kGInit) {
          const uint32_t slot = __shfl_sync(full, rec.x, q0 + j);
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (info & (16u << r)) {
              acc[r] = v[j];
              dst[r] = slot;
            }
          }
          live |= (info >> 4) & 15u;
          if (info & kGIsDiag) dmask |= (info >> 4) & 15u;
        } else if (type == kGDiv) {
          const uint32_t k = (info >> 8) & 63u;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (info & (16u << r)) {
              acc[r] = acc[r] / v[j];  // src/numeric.cpp:40 (IEEE division); stored below as l_id, :41
              L[(r * K + k) * 32] = acc[r];
            }
          }
        } else if (type == kGPub) {
          // src/numeric.cpp:48: the row is published even when its pivot fails, so nothing waits forever
          const int32_t row = static_cast<int32_t>(__shfl_sync(full, rec.x, q0 + j));
          double dv = 0.0;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (info & (16u << r)) dv = dg[r];
          }
          if (info & kGFresh) dv = ld_cg(g + static_cast<int64_t>(__ldg(a.diag + row)) * 32);
          if (fabs(dv) <= a.pivot_floor) atomicMin(a.failed + u * 32 + lane, row);
          __syncwarp();
          if (lane == 0) {
            __threadfence();
            st_relaxed_s32(a.flags + static_cast<int64_t>(row) * a.units + u, a.gen);
          }
        }
        if (info & kGLast) {
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (live & (1u << r)) {
              st_cg(g + static_cast<int64_t>(dst[r]) * 32, acc[r]);
              if (dmask & (1u << r)) dg[r] = acc[r];
            }
          }
          live = 0;
          dmask = 0;
        }
      }
    };

    for (int32_t bi = blk.x; bi < blk.y; ++bi) {
      const int4 hb = __ldg(reinterpret_cast<const int4*>(a.batches + bi));
      const uint32_t win_beg = static_cast<uint32_t>(hb.x);
      const int32_t n_win = hb.y, wait_beg = hb.z, n_wait = hb.w;
      const uint2* rp = reinterpret_cast<const uint2*>(a.recs) + static_cast<size_t>(win_beg) * kGWindow + lane;
      uint2 recA = __ldg(rp), recB = make_uint2(0u, 0u);
      for (int32_t w0 = 0; w0 < n_wait; w0 += 32) {
        if (w0 + lane < n_wait && !a.exp_nowait) {
          const int32_t d = __ldg(a.waits + wait_beg + w0 + lane);
          wait_flag(a.flags + static_cast<int64_t>(d) * a.units + u, a.gen);
        }
      }
      __syncwarp();
      // Chunks of 8 records, two value buffers: the loads of chunk c + 1 are in flight while chunk c is consumed. The
      // loop body exists once per buffer (the interpreter is large: unrolled over a whole window it outgrew the
      // instruction cache and the kernel ran at a tenth of an instruction per cycle).
      double vA[kChunk], vB[kChunk];
      const int32_t n_chunk = n_win * (kGWindow / kChunk);
      issue(recA, 0, vA);
      if (n_win > 1) recB = __ldg(rp + kGWindow);
#pragma unroll 1
      for (int32_t c = 0; c < n_chunk; c += 2) {  // chunks c (window position (c & 3) * 8, buffer A) and c + 1 (buffer B)
        const int q0 = (c & 3) * kChunk;
        issue(recA, q0 + kChunk, vB);
        consume(recA, q0, vA);
        if (q0 == 0) {
          issue(recA, q0 + 2 * kChunk, vA);
          consume(recA, q0 + kChunk, vB);
        } else {  // chunk c + 1 is the last of its window: the next chunk comes from the next window
          if (c + 2 < n_chunk) issue(recB, 0, vA);
          consume(recA, q0 + kChunk, vB);
          recA = recB;
          const int32_t wn = (c + 2) / (kGWindow / kChunk) + 1;  // window after the one that starts at chunk c + 2
          if (wn < n_win) recB = __ldg(rp + static_cast<size_t>(wn) * kGWindow);
        }
      }
    }
    __syncwarp();
  }
}

}  // namespace b200lu
