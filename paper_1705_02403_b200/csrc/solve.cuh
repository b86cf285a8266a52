// solve.cuh -- shared-memory layout and launcher of the GMT* solve kernel.
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

#include "common.cuh"

namespace gmtb {

// Per-CTA shared memory of one query (V = n samples, W = ceil(V/32)):
//   cost   f64[V]    replicated cost-to-arrive
//   parent i32[V]    parent replica (read by rank 0 for the path walk)
//   bits   6 x u32[Wp]  open, closed, group, newopen, cand, goal
//   list   i32[V]    group list (P4) / owned candidate list (P5)
//   obs    f64[2*B*d] boxes, axis-major (SoA) when they fit
struct SolveLayout {
  int words;
  int words_pad;
  size_t off_cost, off_parent, off_bits, off_list, off_obs, total;
};

__host__ __device__ inline SolveLayout solve_layout(int n, int d, int nb, bool obs_smem) {
  SolveLayout L;
  L.words = (n + 31) >> 5;
  L.words_pad = (L.words + 3) & ~3;
  size_t off = 0;
  L.off_cost = off;
  off = align16(off + sizeof(double) * static_cast<size_t>(L.words) * 32);
  L.off_parent = off;
  off = align16(off + sizeof(int32_t) * static_cast<size_t>(L.words) * 32);
  L.off_bits = off;
  off = align16(off + sizeof(uint32_t) * 6 * static_cast<size_t>(L.words_pad));
  L.off_list = off;
  off = align16(off + sizeof(int32_t) * static_cast<size_t>(L.words) * 32);
  L.off_obs = off;
  if (obs_smem) off = align16(off + sizeof(double) * 2 * static_cast<size_t>(nb) * d);
  L.total = off;
  return L;
}

cudaError_t launch_solve(const SolveJob* jobs, int count, int cluster, int threads, size_t smem,
                         int obs_in_smem, cudaStream_t stream);

}  // namespace gmtb
