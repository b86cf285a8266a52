// solve.cuh -- shared-memory layout and launcher of the GMT* solve kernel.
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

#include "common.cuh"

namespace gmtb {

// Largest node count the on-chip wavefront supports (u16 node ids in the
// work lists and the parent replica); the global-memory variant takes
// larger queries.
constexpr int kMaxSolveNodes = 65535;
constexpr int kMaxSolveDim = 16;

// Per-CTA dynamic shared memory of one query (V = n samples,
// W = ceil(V/32), Wp = W rounded up to 4):
//   cost   f64[32W]    replicated cost-to-arrive
//   parent u16[32W]    parent replica (clusters only; batched solves keep
//                      parents in HBM and walk them once at the end)
//   bits   6 x u32[Wp] open, closed, group, newopen, cand, goal
//   list   u16[32W]    owned group members (P4) / owned candidates (P5)
//                      (i32 in the global-memory variant, which has no u16 id limit)
//   obs    f64[4*B*d]  boxes lo, hi, lo - m, hi + m, axis-major (SoA), when they fit,
//          u32[B]      then each box's mask of "full" axes (lo <= 0 and hi >= 1)
struct SolveLayout {
  int words;
  int words_pad;
  size_t off_cost, off_parent, off_bits, off_list, off_obs, total;
};

__host__ __device__ inline SolveLayout solve_layout(int n, int d, int nb, bool obs_smem,
                                                    bool parent_smem, int list_bytes = 2) {
  SolveLayout L;
  L.words = (n + 31) >> 5;
  L.words_pad = (L.words + 3) & ~3;
  const size_t nodes = static_cast<size_t>(L.words) * 32;
  size_t off = 0;
  L.off_cost = off;
  off = align16(off + sizeof(double) * nodes);
  L.off_parent = off;
  if (parent_smem) off = align16(off + sizeof(uint16_t) * nodes);
  L.off_bits = off;
  off = align16(off + sizeof(uint32_t) * 6 * static_cast<size_t>(L.words_pad));
  L.off_list = off;
  off = align16(off + static_cast<size_t>(list_bytes) * nodes);
  L.off_obs = off;
  if (obs_smem)
    off = align16(off + sizeof(double) * 4 * static_cast<size_t>(nb) * d + sizeof(uint32_t) * static_cast<size_t>(nb));
  L.total = off;
  return L;
}

// Dynamic shared memory the solve kernel appends after the layout for its
// per-warp scratch (the 24-warp batched double-integrator shape, 768
// threads: 24 warps x GMT_ROWS_DI24 concurrent checks x (32 + kDiTabCap)
// doubles + 64 box ids);
// 0 for the other shapes (static shared memory).
#ifndef GMT_ROWS_DI24
#define GMT_ROWS_DI24 4  // concurrent candidates (rows, checks) per warp of the 24-warp DI shape
#endif
constexpr int kDiTabCap = 56;  // doubles of one DI waypoint table ((segments + 1) * 6 <= 56)
__host__ __device__ inline size_t solve_dyn_scratch(int threads, int dim) {
  if (threads != 768 || dim != 6) return 0;
  return static_cast<size_t>(24) * GMT_ROWS_DI24 * ((32 + kDiTabCap) * sizeof(double) + 64 * sizeof(uint16_t));
}

// dim: the common dimension of every job (selects the specialised kernel;
// 0 = generic).
// count_traffic: the jobs carry traffic counters (GMT_OPT_COUNTERS).
// gstate: every job carries a global state buffer (SolveJob::gstate) of the
// solve_layout size; cluster must be 1 and threads 512.
// pool: the jobs may carry shared-pool views (DevInstance::pool); d = 6,
// cluster 1.
cudaError_t launch_solve(const SolveJob* jobs, int count, int cluster, int threads, size_t smem,
                         int obs_in_smem, int dim, cudaStream_t stream, bool count_traffic = false,
                         bool gstate = false, bool pool = false);

// dijkstra_oracle (planner.cpp:264-334): eager edge checks into ok[E] (and
// the check count), then the Dijkstra search for job[0] (one CTA).
cudaError_t launch_dijkstra(const DevInstance* inst, const SolveJob* job, int n, int dim, uint8_t* ok,
                            unsigned long long* checks, int sm_count, cudaStream_t stream);

// segment_free (space.cpp:80-90) of count segments a[i*d..], b[i*d..] against
// one AoS box array; out[i] = 1 when free.  Same device test as the lazy check.
struct QuadParams;
struct DiParams;
// Per-in-edge waypoint tables of a kinodynamic instance ((M + 1) * dim
// doubles per in-edge, M = the model's segments; (M + 1) * dim <= 144).
cudaError_t launch_kino_tables(const double* coords, const int64_t* in_ptr, const int32_t* in_col,
                               const double* in_tau, int n, int steering, const QuadParams& QP,
                               const DiParams& DP, double* wp, int sm_count, cudaStream_t stream);
cudaError_t launch_segment_free(const double* a, const double* b, int64_t count, int d,
                                const double* box_lo, const double* box_hi, int nb, uint8_t* out,
                                int sm_count, cudaStream_t stream);

}  // namespace gmtb
