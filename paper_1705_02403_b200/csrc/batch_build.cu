// batch_build.cu -- build_instance + gmt_plan for many Euclidean problems at
// once (SURVEY.md §8(e) batched queries, §8(f) row 3 simulator replans).
//
// One launch per stage for the whole batch, problem-major:
//   gen    candidate j of problem p (Halton index / PCG jump-ahead, exactly
//          CandidateStream::draw, sampling.cpp:64-76) and its point_free flag
//   pack   one CTA per problem: the first n free candidates, in order
//   dedup  (uniform sampling) any exact duplicate among them
//   goal   any sample in the goal box, else goal substitution (the first
//          1024 candidates of sampling.cpp:115-141); append_init (:144-154)
//   rdisk  count / fill of every problem's r-disk rows (graph.cpp:117-188,
//          the predicate of graph.cu), one global scan in between
//   desc   the DevInstance of every problem, then ONE batched solve.
// Problems that need sample_free's rare paths -- more candidates than the
// first chunk, an exact duplicate, a goal substitution beyond the first
// 1024 candidates, or an infeasible / goal-blocked outcome -- are rebuilt by the
// single-instance builder, so every problem's instance is bit-identical to
// gmt_instance_build's (and the reference's build_instance).
#include <cuda_runtime.h>

#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>
#include <unordered_map>
#include <string>
#include <vector>

#include "common.cuh"
#include "gmt_b200.h"
#include "internal.cuh"
#include "sample_dev.cuh"
#include "solve.cuh"

namespace gmtb {

int plan_smem(gmt_ctx* ctx, int max_n, int max_d, int max_nb, int cluster, size_t* smem, int* obs_in_smem,
              size_t* gstate = nullptr);
int assign_gstate(Arena& arena, std::vector<SolveJob>& jobs, size_t bytes);
int carve_results(Arena& arena, int count, const int64_t* node_off, bool tree, bool stats,
                  std::vector<DevResult>& out, ResultScalars** scalars_base, int64_t* counters);
int launch_jobs(gmt_ctx* ctx, const std::vector<SolveJob>& jobs, int cluster, int threads, size_t smem,
                int obs_in_smem, int dim);
int plan_problems_pool(gmt_ctx* ctx, const gmt_problem* problems, int32_t count, int32_t* status_out,
                       gmt_plan_summary* summaries, int32_t path_cap, double* path_states);

namespace {

constexpr uint32_t kFull = 0xffffffffu;
constexpr int kMaxDimB = 16;

#define GMT_CUDA(call)                                   \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) return cuda_error(_e, #call); \
  } while (0)

struct BProb {
  int kind, d, dd, nb, n, K, need_dedup, G;  // G: grid cells per axis (r-disk binning)
  uint64_t start_index, s0;
  int64_t box_off;   // first box of the problem
  int64_t cand_off;  // first candidate row
  int64_t row_off;   // first coordinate row (n + 1 rows reserved)
  int64_t cell_off;  // first entry of the problem's cell_start array (G^d + 1 entries)
  double radius, r2_hi;
  double r2_lo;  // sq <= r2_lo implies sqrt_rn(sq) <= radius (no square root needed)
};

// Per-problem outcome of the batched stages.
struct BOut {
  int32_t fallback;  // 1: rebuild with the single-instance builder
  int32_t V;         // vertices (n, or n + 1 with the appended init)
  int32_t init_index;
  int32_t goal_any;
};

__device__ __forceinline__ bool free_point(const double* p, int d, const double* lo, const double* hi, int nb) {
  if (!point_in_cube(p, d)) return false;  // space.cpp:47-54
  for (int b = 0; b < nb; ++b)
    if (box_contains(lo + b * d, hi + b * d, d, p)) return false;
  return true;
}

// Halton coordinate with the digit weights f_i = (((1 / b) / b) ... / b)
// tabulated on the host (IEEE division, the same correctly rounded steps as
// halton_dev's f /= base): r += f_i * (index % b), 32-bit digit arithmetic
// while the index fits.
constexpr int kHaltonDigits = 64;
__device__ __forceinline__ double halton_tab(uint64_t index, uint32_t base, const double* __restrict__ f) {
  double r = 0.0;
  int i = 0;
  while (index > 0xffffffffull) {
    r = __dadd_rn(r, __dmul_rn(f[i++], static_cast<double>(index % base)));
    index /= base;
  }
  uint32_t x = static_cast<uint32_t>(index);
  while (x > 0) {
    const uint32_t q = x / base;
    r = __dadd_rn(r, __dmul_rn(f[i++], static_cast<double>(x - q * base)));
    x = q;
  }
  return r;
}

// D = 0: any dimension (runtime d, arrays in local memory).
template <int D>
__global__ void __launch_bounds__(256) gen_batch_kernel(const BProb* __restrict__ probs,
                                                        const double* __restrict__ box_lo,
                                                        const double* __restrict__ box_hi,
                                                        const uint32_t* __restrict__ primes,
                                                        const double* __restrict__ fpow,
                                                        double* __restrict__ cand, uint8_t* __restrict__ flag) {
  const BProb P = probs[blockIdx.y];
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= P.K) return;
  double c[D > 0 ? D : kMaxDimB];
  const int d = D > 0 ? D : P.d;
  if (P.kind == GMT_SAMPLE_HALTON) {
    const uint64_t idx = P.start_index + static_cast<uint64_t>(j);
#pragma unroll
    for (int k = 0; k < (D > 0 ? D : kMaxDimB); ++k)
      if (k < d) c[k] = halton_tab(idx, primes[k], fpow + k * kHaltonDigits);
  } else {
    uint64_t st = pcg_advance(P.s0, static_cast<uint64_t>(j) * static_cast<uint64_t>(P.dd));
#pragma unroll
    for (int k = 0; k < (D > 0 ? D : kMaxDimB); ++k) {
      if (k < d) {
        c[k] = static_cast<double>(pcg_out(st)) * 0x1p-32;  // next_double (rng.hpp:33)
        st = st * kPcgMult + kPcgInc;
      }
    }
  }
  double* out = cand + (P.cand_off + j) * d;
#pragma unroll
  for (int k = 0; k < (D > 0 ? D : kMaxDimB); ++k)
    if (k < d) out[k] = c[k];
  bool ok = true;  // point_free (space.cpp:47-54): in the unit cube, in no box
#pragma unroll
  for (int k = 0; k < (D > 0 ? D : kMaxDimB); ++k)
    if (k < d) ok = ok && c[k] >= 0.0 && c[k] <= 1.0;
  const double* lo = box_lo + P.box_off * d;
  const double* hi = box_hi + P.box_off * d;
  for (int b = 0; ok && b < P.nb; ++b) {
    bool in = true;
#pragma unroll
    for (int k = 0; k < (D > 0 ? D : kMaxDimB); ++k)
      if (k < d) in = in && c[k] >= __ldg(lo + b * d + k) && c[k] <= __ldg(hi + b * d + k);
    ok = !in;
  }
  flag[P.cand_off + j] = ok ? 1 : 0;
}

// One CTA per problem: ordered compaction of the first n free candidates.
__global__ void __launch_bounds__(1024) pack_batch_kernel(const BProb* __restrict__ probs,
                                                          const uint8_t* __restrict__ flag,
                                                          const double* __restrict__ cand,
                                                          double* __restrict__ coords, BOut* __restrict__ res) {
  __shared__ int warp_cnt[32];
  __shared__ int base_s;
  const BProb P = probs[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  if (tid == 0) base_s = 0;
  __syncthreads();
  for (int b0 = 0; b0 < P.K && base_s < P.n; b0 += blockDim.x) {
    const int i = b0 + tid;
    const bool f = i < P.K && flag[P.cand_off + i];
    const uint32_t m = __ballot_sync(kFull, f);
    if (lane == 0) warp_cnt[warp] = __popc(m);
    __syncthreads();
    int before = base_s;
    for (int w = 0; w < warp; ++w) before += warp_cnt[w];
    const int slot = before + __popc(m & ((1u << lane) - 1u));
    if (f && slot < P.n)
      for (int k = 0; k < P.d; ++k) coords[(P.row_off + slot) * P.d + k] = cand[(P.cand_off + i) * P.d + k];
    __syncthreads();
    if (tid == 0) {
      int tot = 0;
      for (int w = 0; w < nw; ++w) tot += warp_cnt[w];
      base_s += tot;
    }
    __syncthreads();
  }
  if (tid == 0) {
    res[blockIdx.x].fallback = base_s < P.n ? 1 : 0;  // needs more than the first chunk
    res[blockIdx.x].V = P.n;
  }
}

// Exact duplicates among a problem's first n samples (uniform sampling):
// sample_free would skip them, so the problem takes the single path.
__global__ void dedup_batch_kernel(const BProb* __restrict__ probs, const double* __restrict__ coords,
                                   BOut* __restrict__ res) {
  const BProb P = probs[blockIdx.y];
  if (!P.need_dedup || res[blockIdx.y].fallback) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P.n) return;
  const double* p = coords + (P.row_off + i) * P.d;
  for (int j = 0; j < i; ++j) {
    const double* q = coords + (P.row_off + j) * P.d;
    bool eq = true;
    for (int k = 0; k < P.d; ++k) eq = eq && p[k] == q[k];
    if (eq) {
      res[blockIdx.y].fallback = 1;
      return;
    }
  }
}

// Goal membership (sampling.cpp:110-112).
__global__ void __launch_bounds__(256) goal_batch_kernel(const BProb* __restrict__ probs,
                                                         const double* __restrict__ coords,
                                                         const double* __restrict__ goal_lo,
                                                         const double* __restrict__ goal_hi, BOut* __restrict__ res) {
  const int p = blockIdx.x;
  const BProb P = probs[p];
  if (res[p].fallback) return;
  const double* glo = goal_lo + static_cast<int64_t>(p) * P.d;
  const double* ghi = goal_hi + static_cast<int64_t>(p) * P.d;
  bool in_goal = false;
  for (int i = threadIdx.x; i < P.n; i += blockDim.x)
    in_goal = in_goal || box_contains(glo, ghi, P.d, coords + (P.row_off + i) * P.d);
  const int any = __syncthreads_or(in_goal ? 1 : 0);
  if (threadIdx.x == 0) res[p].goal_any = any;
}

// Goal substitution (sampling.cpp:115-141) for problems without a goal
// sample: the first of the goal centre and the goal-box Halton points that
// is free and no exact duplicate of samples 0 .. n-2 replaces sample n-1.
// The first kSubst candidates are searched here; beyond them the problem
// takes the single path.
constexpr int kSubst = 1024;

__global__ void __launch_bounds__(256) subst_batch_kernel(const BProb* __restrict__ probs,
                                                          double* __restrict__ coords,
                                                          const double* __restrict__ box_lo,
                                                          const double* __restrict__ box_hi,
                                                          const double* __restrict__ goal_lo,
                                                          const double* __restrict__ goal_hi,
                                                          const uint32_t* __restrict__ primes,
                                                          BOut* __restrict__ res) {
  __shared__ int best, dup;
  const int p = blockIdx.x;
  const BProb P = probs[p];
  if (res[p].fallback || res[p].goal_any) return;
  const int d = P.d;
  const double* glo = goal_lo + static_cast<int64_t>(p) * d;
  const double* ghi = goal_hi + static_cast<int64_t>(p) * d;
  auto candidate = [&](int i, double* c) {
    if (i == 0) {  // Aabb::center (space.cpp:18-22)
      for (int k = 0; k < d; ++k) c[k] = __dmul_rn(0.5, __dadd_rn(glo[k], ghi[k]));
    } else {  // lo + q * (hi - lo) (sampling.cpp:122-124)
      for (int k = 0; k < d; ++k)
        c[k] = __dadd_rn(glo[k], __dmul_rn(halton_dev(static_cast<uint64_t>(i), primes[k]), __dsub_rn(ghi[k], glo[k])));
    }
  };
  // The first free candidate that duplicates no sample: the first free one is
  // found block-wide, then checked against the samples block-wide (an exact
  // duplicate is rare; the search then resumes after it).
  int last = -1, found = -1;
  for (;;) {
    if (threadIdx.x == 0) {
      best = 0x7fffffff;
      dup = 0;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kSubst; i += blockDim.x) {
      if (i <= last) continue;
      double c[kMaxDimB];
      candidate(i, c);
      if (free_point(c, d, box_lo + P.box_off * d, box_hi + P.box_off * d, P.nb)) atomicMin(&best, i);
    }
    __syncthreads();
    const int b = best;
    if (b == 0x7fffffff) break;
    double c[kMaxDimB];
    candidate(b, c);
    for (int j = threadIdx.x; j < P.n - 1; j += blockDim.x) {
      const double* q = coords + (P.row_off + j) * d;
      bool eq = true;
      for (int k = 0; k < d; ++k) eq = eq && c[k] == q[k];
      if (eq) dup = 1;
    }
    __syncthreads();
    const int was_dup = dup;
    __syncthreads();  // everyone has read best / dup before the next round resets them
    if (!was_dup) {
      found = b;
      break;
    }
    last = b;
  }
  if (threadIdx.x == 0) {
    if (found < 0) {
      res[p].fallback = 1;
    } else {
      double* out = coords + (P.row_off + P.n - 1) * d;
      candidate(found, out);
      res[p].goal_any = 1;
    }
  }
}

// append_init (sampling.cpp:144-154): the first exact duplicate of the
// init, else the init appended as vertex n.
__global__ void __launch_bounds__(256) init_batch_kernel(const BProb* __restrict__ probs, double* __restrict__ coords,
                                                         const double* __restrict__ inits, BOut* __restrict__ res) {
  __shared__ int first;
  const int p = blockIdx.x;
  const BProb P = probs[p];
  if (res[p].fallback) return;
  const double* init = inits + static_cast<int64_t>(p) * P.d;
  if (threadIdx.x == 0) first = 0x7fffffff;
  __syncthreads();
  for (int i = threadIdx.x; i < P.n; i += blockDim.x) {
    const double* c = coords + (P.row_off + i) * P.d;
    bool eq = true;
    for (int k = 0; k < P.d; ++k) eq = eq && c[k] == init[k];
    if (eq) atomicMin(&first, i);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (first != 0x7fffffff) {
      res[p].init_index = first;
      res[p].V = P.n;
    } else {
      for (int k = 0; k < P.d; ++k) coords[(P.row_off + P.n) * P.d + k] = init[k];
      res[p].init_index = P.n;
      res[p].V = P.n + 1;
    }
  }
}

// Euclidean r-disk rows of every problem (the predicate of graph.cu:
// correctly rounded squared distance in axis order, sq <= r^2 (1 + 1e-12)
// pre-test, sqrt_rn(sq) <= r).  Flat rows r = row_off[p] + u, u <= n.
template <int D, bool FILL>
__global__ void __launch_bounds__(256) rdisk_batch_kernel(const BProb* __restrict__ probs,
                                                          const int64_t* __restrict__ row_start, int P_count,
                                                          int64_t R, const double* __restrict__ coords,
                                                          const BOut* __restrict__ res,
                                                          int64_t* __restrict__ counts,
                                                          const int64_t* __restrict__ row_ptr,
                                                          int32_t* __restrict__ col, double* __restrict__ cost) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(blockDim.x >> 5) * gridDim.x;
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x >> 5) + (threadIdx.x >> 5); r < R; r += warps) {
    int lo = 0, hi = P_count - 1;  // problem of row r
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (row_start[mid] <= r) lo = mid; else hi = mid - 1;
    }
    const int p = lo;
    const BProb& P = probs[p];
    const int d = D > 0 ? D : P.d;
    const int u = static_cast<int>(r - P.row_off);
    const int V = res[p].fallback ? 0 : res[p].V;
    int64_t out = FILL ? row_ptr[r] : 0;
    if (u < V) {
      double a[D > 0 ? D : kMaxDimB];
#pragma unroll
      for (int k = 0; k < (D > 0 ? D : kMaxDimB); ++k)
        if (D > 0 || k < d) a[k] = __ldg(coords + (P.row_off + u) * d + k);
      for (int base = 0; base < V; base += 32) {
        const int v = base + lane;
        bool keep = false;
        double c = 0.0;
        if (v < V && v != u) {
          double sq = 0.0;
#pragma unroll
          for (int k = 0; k < (D > 0 ? D : kMaxDimB); ++k) {
            if (D > 0 || k < d) {
              const double t = __dsub_rn(a[k], __ldg(coords + (P.row_off + v) * d + k));
              sq = __dadd_rn(sq, __dmul_rn(t, t));
            }
          }
          if (sq <= P.r2_hi) {
            c = __dsqrt_rn(sq);
            keep = c <= P.radius;
          }
        }
        const uint32_t m = __ballot_sync(kFull, keep);
        if (FILL && keep) {
          const int64_t slot = out + __popc(m & ((1u << lane) - 1u));
          col[slot] = v;
          cost[slot] = c;
        }
        out += __popc(m);
      }
    }
    if (!FILL && lane == 0) counts[r] = out;
  }
}

__global__ void desc_batch_kernel(const BProb* __restrict__ probs, const BOut* __restrict__ res,
                                  const double* __restrict__ coords, const double* __restrict__ box_lo,
                                  const double* __restrict__ box_hi, const double* __restrict__ goal_lo,
                                  const double* __restrict__ goal_hi, const int64_t* __restrict__ row_ptr,
                                  const int32_t* __restrict__ col, const double* __restrict__ cost, int count,
                                  const int64_t* __restrict__ rstart, const int64_t* __restrict__ rend,
                                  DevInstance* __restrict__ descs) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= count) return;
  const BProb P = probs[p];
  DevInstance D{};
  D.n = res[p].V;
  D.dim = P.d;
  D.num_boxes = P.nb;
  D.directed = 0;
  D.goal_count = res[p].goal_any;
  D.init_index = res[p].init_index;
  D.radius = P.radius;
  D.num_edges = row_ptr[P.row_off + D.n] - row_ptr[P.row_off];
  D.coords = coords + P.row_off * P.d;
  D.box_lo = box_lo + P.box_off * P.d;
  D.box_hi = box_hi + P.box_off * P.d;
  D.goal_lo = goal_lo + static_cast<int64_t>(p) * P.d;
  D.goal_hi = goal_hi + static_cast<int64_t>(p) * P.d;
  D.out_ptr = rstart ? rstart + P.row_off : row_ptr + P.row_off;  // row-padded scratch, or the CSR
  D.out_end = rstart ? rend + P.row_off : nullptr;
  D.out_col = col;
  D.out_cost = cost;
  D.in_ptr = D.out_ptr;
  D.in_end = D.out_end;
  D.in_col = col;
  D.in_cost = cost;
  descs[p] = D;
}

// Path states of every solved query (up to cap states each).
__global__ void gather_paths_kernel(const DevResult* __restrict__ rs, const DevInstance* const* __restrict__ insts,
                                    int count, int cap, int d, double* __restrict__ out) {
  const int q = blockIdx.x;
  if (q >= count) return;
  const DevResult R = rs[q];
  const ResultScalars sc = *R.scalars;
  const DevInstance* I = insts[q];
  const int len = sc.status != 0 ? 0 : (sc.path_len < cap ? sc.path_len : cap);
  for (int e = threadIdx.x; e < cap * d; e += blockDim.x) {  // zeros past the path: a deterministic buffer
    const int k = e / d, i = e - k * d;
    out[static_cast<int64_t>(q) * cap * d + e] = k < len ? I->coords[static_cast<int64_t>(R.path[k]) * d + i] : 0.0;
  }
}

// Register-blocked variant for d = 2, 3: a warp takes RB consecutive rows
// of one problem; each lane loads one target's coordinates once and tests
// it against all RB rows (RB x fewer coordinate loads); per row the ballot
// word orders the accepted targets exactly as the one-row kernel does.
// FILL = false: counts, and the first C accepted targets of every row into
// the row's scratch slots; FILL = true: only rows with more than C accepted
// targets are evaluated again, straight into the CSR.
template <int D, int RB, bool FILL>
__global__ void __launch_bounds__(256) rdisk_batch_rb_kernel(const BProb* __restrict__ probs,
                                                             const int64_t* __restrict__ row_start, int P_count,
                                                             int64_t R, const double* __restrict__ coords,
                                                             const BOut* __restrict__ res,
                                                             int64_t* __restrict__ counts,
                                                             const int64_t* __restrict__ row_ptr,
                                                             int32_t* __restrict__ col, double* __restrict__ cost,
                                                             int32_t* __restrict__ scol, double* __restrict__ scost,
                                                             int C) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(blockDim.x >> 5) * gridDim.x;
  const int64_t groups = (R + RB - 1) / RB;
  for (int64_t gidx = blockIdx.x * static_cast<int64_t>(blockDim.x >> 5) + (threadIdx.x >> 5); gidx < groups;
       gidx += warps) {
    const int64_t r0 = gidx * RB;
    int lo = 0, hi = P_count - 1;  // problem of row r0 (rows of a group may spill into the next problem)
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (row_start[mid] <= r0) lo = mid; else hi = mid - 1;
    }
    const int p = lo;
    const BProb& P = probs[p];
    const int u0 = static_cast<int>(r0 - P.row_off);
    const int V = res[p].fallback ? 0 : res[p].V;
    const int rows_here = static_cast<int>(min(static_cast<int64_t>(RB), row_start[p + 1] - r0));
    double a[RB][D];
    int64_t out[RB];
    bool act[RB];
    bool any_act = false;
#pragma unroll
    for (int j = 0; j < RB; ++j) {
      const int u = u0 + j;
      act[j] = j < rows_here && u < V && (!FILL || counts[r0 + j] > C);
      any_act = any_act || act[j];
      out[j] = (FILL && act[j]) ? row_ptr[r0 + j] : 0;
#pragma unroll
      for (int k = 0; k < D; ++k) a[j][k] = act[j] ? __ldg(coords + (P.row_off + u) * D + k) : 0.0;
    }
    for (int base = 0; any_act && base < V; base += 32) {
      const int v = base + lane;
      double b[D];
#pragma unroll
      for (int k = 0; k < D; ++k) b[k] = v < V ? __ldg(coords + (P.row_off + v) * D + k) : 0.0;
#pragma unroll
      for (int j = 0; j < RB; ++j) {
        const int u = u0 + j;
        bool keep = false;
        double c = 0.0;
        if (act[j] && v < V && v != u) {
          double sq = 0.0;
#pragma unroll
          for (int k = 0; k < D; ++k) {
            const double t = __dsub_rn(a[j][k], b[k]);
            sq = __dadd_rn(sq, __dmul_rn(t, t));
          }
          if (sq <= P.r2_hi) {
            c = __dsqrt_rn(sq);
            keep = c <= P.radius;
          }
        }
        const uint32_t m = __ballot_sync(kFull, keep);
        if (keep) {
          const int64_t slot = out[j] + __popc(m & ((1u << lane) - 1u));
          if (FILL) {
            col[slot] = v;
            cost[slot] = c;
          } else if (slot < C) {
            scol[(r0 + j) * C + slot] = v;
            scost[(r0 + j) * C + slot] = c;
          }
        }
        out[j] += __popc(m);
      }
    }
    if (!FILL && lane == 0) {
#pragma unroll
      for (int j = 0; j < RB; ++j)
        if (j < rows_here) counts[r0 + j] = out[j];
    }
    // rows of the group beyond this problem's rows belong to the next one
    for (int64_t r = r0 + rows_here; r < r0 + RB && r < R; ++r) {
      int lo2 = 0, hi2 = P_count - 1;
      while (lo2 < hi2) {
        const int mid = (lo2 + hi2 + 1) >> 1;
        if (row_start[mid] <= r) lo2 = mid; else hi2 = mid - 1;
      }
      const BProb& Q = probs[lo2];
      const int uq = static_cast<int>(r - Q.row_off);
      const int Vq = res[lo2].fallback ? 0 : res[lo2].V;
      if (FILL && counts[r] <= C) continue;
      int64_t o = FILL ? row_ptr[r] : 0;
      if (uq < Vq) {
        double aq[D];
        for (int k = 0; k < D; ++k) aq[k] = __ldg(coords + (Q.row_off + uq) * D + k);
        for (int base = 0; base < Vq; base += 32) {
          const int v = base + lane;
          bool keep = false;
          double c = 0.0;
          if (v < Vq && v != uq) {
            double sq = 0.0;
            for (int k = 0; k < D; ++k) {
              const double t = __dsub_rn(aq[k], __ldg(coords + (Q.row_off + v) * D + k));
              sq = __dadd_rn(sq, __dmul_rn(t, t));
            }
            if (sq <= Q.r2_hi) {
              c = __dsqrt_rn(sq);
              keep = c <= Q.radius;
            }
          }
          const uint32_t m = __ballot_sync(kFull, keep);
          if (keep) {
            const int64_t slot = o + __popc(m & ((1u << lane) - 1u));
            if (FILL) {
              col[slot] = v;
              cost[slot] = c;
            } else if (slot < C) {
              scol[r * C + slot] = v;
              scost[r * C + slot] = c;
            }
          }
          o += __popc(m);
        }
      }
      if (!FILL && lane == 0) counts[r] = o;
    }
  }
}

// ---- r-disk rows through a uniform grid (d = 2, 3) ---------------------------
// Cells of side 1/G >= r / kGridReach (slightly more, against rounding), so
// every target within r of u lies in the (2 kGridReach + 1)^d cells around
// u's cell.  A CTA takes one cell
// of one problem; a warp marks, for up to 8 rows of that cell at once, the
// accepted targets of the neighbour cells in per-row bitmasks (the exact
// predicate of rdisk_batch_kernel), then emits every row in target order
// from its bitmask, recomputing the accepted costs -- so rows are
// bit-identical to the brute-force scan.
constexpr int kGridMaxCells = 4096;
constexpr int kGridMaxV = 8192;
#ifndef GMT_GRID_ROWS
#define GMT_GRID_ROWS 4
#endif
constexpr int kGridRows = GMT_GRID_ROWS;
constexpr int kGridReach = 2;
constexpr int kGridSpan = 2 * kGridReach + 1;
constexpr int kGridStride = kGridMaxV / 32;  // bitmask words per row, V <= 8192 (compile-time: immediate offsets)
constexpr int kGridCand = 768;  // a cell's flattened neighbour targets kept in shared memory (u16) up to this many
// 32-bit words of shared memory per warp: bitmask rows (S words each), run
// bookkeeping (64), emission buffer (C, padded to 4), target list (u16)
__host__ __device__ constexpr int grid_warp_words(int S, int C) {
  return kGridRows * S + 64 + ((C + 3) & ~3) + kGridCand / 2;
}

template <int D>
__device__ __forceinline__ int grid_cell(const double* c, int G) {
  int cell = 0, mul = 1;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    int q = static_cast<int>(floor(c[k] * G));
    q = q < 0 ? 0 : (q >= G ? G - 1 : q);
    cell += q * mul;
    mul *= G;
  }
  return cell;
}

template <int D>
__global__ void __launch_bounds__(256) grid_build_kernel(const BProb* __restrict__ probs,
                                                         const double* __restrict__ coords,
                                                         const BOut* __restrict__ res,
                                                         int32_t* __restrict__ cell_start,
                                                         int32_t* __restrict__ cell_list) {
  __shared__ int cnt[kGridMaxCells + 1];
  const int p = blockIdx.x;
  const BProb P = probs[p];
  const int V = res[p].fallback ? 0 : res[p].V;
  int cells = 1;
  for (int k = 0; k < D; ++k) cells *= P.G;
  for (int c = threadIdx.x; c <= cells; c += blockDim.x) cnt[c] = 0;
  __syncthreads();
  for (int v = threadIdx.x; v < V; v += blockDim.x)
    atomicAdd(&cnt[grid_cell<D>(coords + (P.row_off + v) * D, P.G)], 1);
  __syncthreads();
  {  // exclusive scan of the cell counts: 16 consecutive cells per thread
    __shared__ int wsum[8];
    constexpr int kPer = (kGridMaxCells + 255) / 256;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int c0 = t * kPer;
    int local[kPer];
    int sum = 0;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      local[i] = c0 + i < cells ? cnt[c0 + i] : 0;
      sum += local[i];
    }
    int incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    int base = incl - sum;
    for (int w = 0; w < warp; ++w) base += wsum[w];
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      if (c0 + i < cells) {
        cnt[c0 + i] = base;
        cell_start[P.cell_off + c0 + i] = base;
      }
      base += local[i];
    }
    if (c0 < cells && c0 + kPer >= cells) cell_start[P.cell_off + cells] = base;  // the thread holding the last cell
  }
  __syncthreads();
  for (int v = threadIdx.x; v < V; v += blockDim.x) {
    const int c = grid_cell<D>(coords + (P.row_off + v) * D, P.G);
    cell_list[P.row_off + atomicAdd(&cnt[c], 1)] = v;
  }
}

// Squared distance in the reference's operation order (sum over axes of
// (a - b)^2, left to right); the leading 0.0 + x of the reference's
// accumulation is exact for x >= +0 and is skipped.
template <int D>
__device__ __forceinline__ double sq_dist(const double* a, const double* b) {
  double t = __dsub_rn(a[0], b[0]);
  double sq = __dmul_rn(t, t);
#pragma unroll
  for (int k = 1; k < D; ++k) {
    t = __dsub_rn(a[k], b[k]);
    sq = __dadd_rn(sq, __dmul_rn(t, t));
  }
  return sq;
}

#ifndef GMT_GRID_MINB
#define GMT_GRID_MINB 4
#endif
template <int D, int S>  // S: bitmask words per row (128 when V <= 4096, else 256)
__global__ void __launch_bounds__(256, GMT_GRID_MINB) rdisk_grid_kernel(const BProb* __restrict__ probs,
                                                            const double* __restrict__ coords,
                                                            const BOut* __restrict__ res,
                                                            const int32_t* __restrict__ cell_start,
                                                            const int32_t* __restrict__ cell_list, int W,
                                                            int64_t* __restrict__ counts,
                                                            int32_t* __restrict__ scol, double* __restrict__ scost,
                                                            int C, int32_t* __restrict__ overflow,
                                                            int64_t* __restrict__ rstart, int64_t* __restrict__ rend) {
  // shared memory per warp: kGridRows bitmask rows of W words, 64 ints of
  // run bookkeeping, C ints of emission buffer
  extern __shared__ uint32_t bm_all[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int p = blockIdx.y, cell = blockIdx.x * nw + warp;  // one warp per (problem, cell)
  const BProb P = probs[p];
  const int G = P.G;
  int cells = 1;
  for (int k = 0; k < D; ++k) cells *= G;
  if (cell >= cells || res[p].fallback) return;
  uint32_t* bm = bm_all + static_cast<size_t>(warp) * grid_warp_words(S, C);  // 16 B aligned
  int* run_s = reinterpret_cast<int*>(bm + kGridRows * S);
  int* pre = run_s + 32;
  int* ebuf = run_s + 64;
  uint16_t* tlist = reinterpret_cast<uint16_t*>(ebuf + ((C + 3) & ~3));
  const int32_t* cs = cell_start + P.cell_off;
  const int32_t* cl = cell_list + P.row_off;
  const double* X = coords + P.row_off * D;
  const int c0 = cs[cell], c1 = cs[cell + 1];
  if (c0 == c1) return;
  // The neighbour cells as runs of consecutive cell indices (x fastest): the
  // targets of a run are one contiguous stretch of cell_list.  A target's run
  // is found by binary search over the run-length prefix.
  constexpr int kRuns = D == 3 ? kGridSpan * kGridSpan : kGridSpan;
  const int cx = cell % G, cy = (cell / G) % G, cz = D == 3 ? cell / (G * G) : 0;
  const int xlo = max(cx - kGridReach, 0), xhi = min(cx + kGridReach, G - 1);
  if (lane < kRuns) {
    const int ny = cy + lane % kGridSpan - kGridReach;
    const int nz = D == 3 ? cz + lane / kGridSpan - kGridReach : 0;
    int len = 0, st = 0;
    if (ny >= 0 && ny < G && nz >= 0 && nz < (D == 3 ? G : 1)) {
      const int base = (ny + nz * G) * G;
      st = cs[base + xlo];
      len = cs[base + xhi + 1] - st;
    }
    int incl = len;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu >> (32 - kRuns), incl, o);
      if (lane >= o) incl += y;
    }
    run_s[lane] = st;
    pre[lane] = incl - len;
    if (lane == kRuns - 1) pre[kRuns] = incl;
  }
  __syncwarp();
  const int total = pre[kRuns];
  // The flattened target list, once per cell (every row group of the cell
  // reuses it): run q's targets at [pre[q], pre[q + 1]); longer neighbourhoods
  // find a target's run by binary search instead.
  const bool listed = total <= kGridCand;
  if (listed) {
#pragma unroll 5
    for (int q = 0; q < kRuns; ++q) {  // (first 32 of each run predicated: the runs' loads overlap)
      const int st = run_s[q], b0 = pre[q], len = pre[q + 1] - b0;
      if (lane < len) tlist[b0 + lane] = static_cast<uint16_t>(cl[st + lane]);
      for (int i = lane + 32; i < len; i += 32) tlist[b0 + i] = static_cast<uint16_t>(cl[st + i]);
    }
    __syncwarp();
  }
  const double r2_lo = P.r2_lo, r2_hi = P.r2_hi, radius = P.radius;
  for (int g0 = c0; g0 < c1; g0 += kGridRows) {
    const int rows = min(kGridRows, c1 - g0);
    // rows past the cell's end sit far away (their squared distances overflow
    // to +inf and accept nothing)
    double a[kGridRows][D];
#pragma unroll
    for (int j = 0; j < kGridRows; ++j) {
      const int u = j < rows ? cl[g0 + j] : 0;
#pragma unroll
      for (int k = 0; k < D; ++k) a[j][k] = j < rows ? X[u * D + k] : 1e300;
    }
    const int per4 = (W + 127) >> 7;  // 16-byte word groups per lane in the emission
#pragma unroll
    for (int j = 0; j < kGridRows; ++j)
      for (int q = lane; q < per4 * 32; q += 32) reinterpret_cast<uint4*>(bm + j * S)[q] = make_uint4(0, 0, 0, 0);
    __syncwarp();
    // mark: the flattened neighbour targets, 32 per step (a row's own bit is
    // set here and cleared below)
    // (software-pipelined: the next chunk's target index and coordinates are
    // loaded while the current chunk is tested)
    auto target = [&](int t) -> int {
      if (listed) return tlist[t];
      int lo = 0, hi = kRuns - 1;  // last run with pre[q] <= t
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (pre[mid] <= t) lo = mid; else hi = mid - 1;
      }
      return cl[run_s[lo] + t - pre[lo]];
    };
    auto fetch = [&](int t, int& v, double* b) {
      v = target(t);
#pragma unroll
      for (int k = 0; k < D; ++k) b[k] = X[v * D + k];
    };
    // Fast pass: sq <= r2_lo accepts with no square root, branch-free; a pair
    // in the rounding band (r2_lo, r2_hi] only raises a flag, and a flagged
    // group runs the exact pass, which decides band pairs by sqrt_rn(sq) <= r
    // (re-setting already-set bits is idempotent).
    auto mark = [&](auto exact_tag) {
      constexpr bool kExact = decltype(exact_tag)::value;
      bool band_seen = false;
      int vn = 0;
      double bn[D];
#pragma unroll
      for (int k = 0; k < D; ++k) bn[k] = 1e300;
      if (lane < total) fetch(lane, vn, bn);
      int vnn = lane + 32 < total ? target(lane + 32) : 0;  // (the index two chunks ahead)
      for (int t = lane; t - lane < total; t += 32) {
        const int v = vn;
        double b[D];
#pragma unroll
        for (int k = 0; k < D; ++k) b[k] = bn[k];
        if (t + 32 < total) {
          vn = vnn;
#pragma unroll
          for (int k = 0; k < D; ++k) bn[k] = X[vn * D + k];
        }
        if (t + 64 < total) vnn = target(t + 64);
        // one 32-bit shared address per target; row j at an immediate offset
        const uint32_t wa = static_cast<uint32_t>(__cvta_generic_to_shared(bm + (v >> 5)));
        const uint32_t bit = 1u << (v & 31);
#pragma unroll
        for (int j = 0; j < kGridRows; ++j) {
          const double sq = sq_dist<D>(a[j], b);  // (lanes past the end repeat their last target: idempotent)
          const bool in = sq <= r2_lo;
          const bool band = !in && sq <= r2_hi;
          bool keep = in;
          if (kExact) {
            if (band) keep = __dsqrt_rn(sq) <= radius;
          } else {
            band_seen = band_seen || band;
          }
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p red.shared.or.b32 [%0], %1;\n\t}"
                       ::"r"(wa + j * S * 4), "r"(bit), "r"(static_cast<uint32_t>(keep)) : "memory");
        }
      }
      return band_seen;
    };
    if (__any_sync(kFull, mark(std::false_type{}))) mark(std::true_type{});
    __syncwarp();
    if (lane < rows) {
      const int u = cl[g0 + lane];
      bm[lane * S + (u >> 5)] &= ~(1u << (u & 31));
    }
    __syncwarp();
    // emit: each row in target order -- lanes own consecutive words, write
    // their targets into the emission buffer at their prefix offset, then the
    // first C targets get their costs (recomputed exactly) 32 at a time.
    for (int j = 0; j < rows; ++j) {
      const int u = cl[g0 + j];  // (not us[j]: a dynamic index would put the row arrays in local memory)
      double au[D];
#pragma unroll
      for (int k = 0; k < D; ++k) au[k] = X[u * D + k];
      const int64_t r = P.row_off + u;
      const uint32_t* row = bm + j * S;
      // lane owns words [4 per4 lane, 4 per4 (lane + 1)): 16-byte loads, no bank conflicts
      const uint4* row4 = reinterpret_cast<const uint4*>(row) + lane * per4;
      int cnt = 0;
      for (int i = 0; i < per4; ++i) {
        const uint4 q = row4[i];
        cnt += __popc(q.x) + __popc(q.y) + __popc(q.z) + __popc(q.w);
      }
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
      }
      const int n_row = __shfl_sync(kFull, incl, 31);
      int slot = incl - cnt;
      for (int i = 0; i < per4 && slot < C; ++i) {
        const uint4 q = row4[i];
        const uint32_t ws[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const int w = (lane * per4 + i) * 4 + h;
          for (uint32_t bits = ws[h]; bits && slot < C; bits &= bits - 1u) ebuf[slot++] = w * 32 + __ffs(bits) - 1;
        }
      }
      __syncwarp();
      const int m = min(n_row, C);
      // (software-pipelined: the next target's coordinates load while the
      // current cost is computed and stored)
      int v = lane < m ? ebuf[lane] : 0;
      double b[D];
#pragma unroll
      for (int k = 0; k < D; ++k) b[k] = lane < m ? X[v * D + k] : 0.0;
      int vnn = lane + 32 < m ? ebuf[lane + 32] : 0;  // (the index two targets ahead)
      for (int e = lane; e < m; e += 32) {
        const int vn = vnn;
        vnn = e + 64 < m ? ebuf[e + 64] : 0;
        double bn[D];
#pragma unroll
        for (int k = 0; k < D; ++k) bn[k] = e + 32 < m ? X[vn * D + k] : 0.0;
        scol[r * C + e] = v;
        scost[r * C + e] = __dsqrt_rn(sq_dist<D>(au, b));
        v = vn;
#pragma unroll
        for (int k = 0; k < D; ++k) b[k] = bn[k];
      }
      if (lane == 0) {
        counts[r] = n_row;
        rstart[r] = r * C;  // the row in the padded scratch (used when no row overflows)
        rend[r] = r * C + min(n_row, C);
        if (n_row > C) *overflow = 1;  // the row needs the fill pass
      }
      __syncwarp();
    }
  }
}

// Rows with at most C targets: scratch slots -> CSR.
__global__ void compact_rows_batch_kernel(const int64_t* __restrict__ counts, const int64_t* __restrict__ row_ptr,
                                          int64_t R, int C, const int32_t* __restrict__ scol,
                                          const double* __restrict__ scost, int32_t* __restrict__ col,
                                          double* __restrict__ cost) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(blockDim.x >> 5) * gridDim.x;
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x >> 5) + (threadIdx.x >> 5); r < R; r += warps) {
    const int64_t n = counts[r];
    if (n > C) continue;
    const int64_t o = row_ptr[r];
    for (int64_t k = lane; k < n; k += 32) {
      col[o + k] = scol[r * C + k];
      cost[o + k] = scost[r * C + k];
    }
  }
}

// Dynamic shared memory above 48 KB needs the kernel attribute; grown
// monotonically under a mutex (concurrent contexts share the kernels).
cudaError_t raise_smem(const void* fn, size_t bytes) {
  static std::mutex mu;
  static std::unordered_map<const void*, size_t> cur;
  std::lock_guard<std::mutex> lock(mu);
  size_t& c = cur[fn];
  if (bytes <= c || bytes <= 48 * 1024) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
  if (e == cudaSuccess) c = bytes;
  return e;
}

template <bool FILL>
cudaError_t launch_rdisk_batch(int d, int blocks, cudaStream_t s, const BProb* probs, const int64_t* row_start,
                               int P_count, int64_t R, const double* coords, const BOut* res, int64_t* counts,
                               const int64_t* row_ptr, int32_t* col, double* cost, int32_t* scol, double* scost,
                               int C) {
  switch (d) {
    case 2:
      rdisk_batch_rb_kernel<2, 8, FILL><<<blocks, 256, 0, s>>>(probs, row_start, P_count, R, coords, res, counts,
                                                               row_ptr, col, cost, scol, scost, C);
      break;
    case 3:
      rdisk_batch_rb_kernel<3, 8, FILL><<<blocks, 256, 0, s>>>(probs, row_start, P_count, R, coords, res, counts,
                                                               row_ptr, col, cost, scol, scost, C);
      break;
    default:
      rdisk_batch_kernel<0, FILL><<<blocks, 256, 0, s>>>(probs, row_start, P_count, R, coords, res, counts,
                                                         row_ptr, col, cost);
      break;
  }
  return cudaGetLastError();
}

}  // namespace

}  // namespace gmtb

using namespace gmtb;

extern "C" int gmt_plan_problems(gmt_ctx* ctx, const gmt_problem* problems, int32_t count,
                                 int32_t* status_out, gmt_plan_summary* summaries, int32_t path_cap,
                                 double* path_states) {
  gmtb::AllocScope alloc_scope_(ctx);
  if (count < 1) return set_error(GMT_E_INVALID_INPUT, "gmt_plan_problems needs at least one problem");
  const int d = problems[0].scene.dim;
  if (d < 1 || d > kMaxDimB) return set_error(GMT_E_INVALID_INPUT, "dimension must be in [1, 16]");
  if (problems[0].steering == GMT_STEER_DOUBLE_INTEGRATOR) {  // the shared Halton pool (pool.cu)
    for (int q = 1; q < count; ++q)
      if (problems[q].steering != GMT_STEER_DOUBLE_INTEGRATOR)
        return set_error(GMT_E_INVALID_INPUT,
                         "gmt_plan_problems: a batch is all Euclidean or all double-integrator problems");
    return plan_problems_pool(ctx, problems, count, status_out, summaries, path_cap, path_states);
  }
  cudaStream_t s = ctx->stream;

  // ---- host: per-problem parameters and the packed scene arrays ----------
  std::vector<BProb> probs(count);
  std::vector<double> box_lo, box_hi, goal_lo(static_cast<size_t>(count) * d), goal_hi(goal_lo.size()),
      inits(goal_lo.size());
  std::vector<int64_t> row_start(count + 1, 0);
  int64_t cand_total = 0, box_total = 0, cell_total = 0;
  int max_K = 1, max_cells = 1, max_rows = 1;
  bool grid_ok = d == 2 || d == 3;
  for (int q = 0; q < count; ++q) {
    const gmt_problem& pr = problems[q];
    if (pr.scene.dim != d) return set_error(GMT_E_INVALID_INPUT, "all problems of a batch share the dimension");
    if (pr.steering != GMT_STEER_EUCLIDEAN)
      return set_error(GMT_E_INVALID_INPUT,
                       "gmt_plan_problems: a batch is all Euclidean or all double-integrator problems");
    int rc = validate_scene(&pr.scene);
    if (rc) return rc;
    if (pr.n < 1) return set_error(GMT_E_INVALID_INPUT, "sample count must be >= 1");
    if (!(pr.lambda > 0.0 && pr.lambda <= 1.0)) return set_error(GMT_E_INVALID_INPUT, "lambda must be in (0, 1]");
    if (pr.sampling.kind != GMT_SAMPLE_HALTON && pr.sampling.kind != GMT_SAMPLE_UNIFORM)
      return set_error(GMT_E_INVALID_INPUT, "unknown sample kind");
    if (pr.sampling.kind == GMT_SAMPLE_HALTON && pr.sampling.start_index == 0)
      return set_error(GMT_E_INVALID_INPUT, "halton start_index is 1-based; got 0");
    BProb& P = probs[q];
    std::memset(&P, 0, sizeof(P));
    P.kind = pr.sampling.kind;
    P.d = d;
    P.dd = d;  // Euclidean problems sample no heading (problem.cpp:338-339)
    P.nb = pr.scene.num_boxes;
    P.n = pr.n;
    const uint64_t budget = 1000ULL * static_cast<uint64_t>(pr.n);
    {  // candidates drawn up front: n over the free-volume estimate (boxes
       // clipped to the unit cube; overlaps make it low, i.e. K larger),
       // +5 % + 256; a problem that still runs short takes the single builder
      double blocked = 0.0;
      for (int b = 0; b < pr.scene.num_boxes; ++b) {
        double v = 1.0;
        for (int k = 0; k < d; ++k) {
          const double lo = std::max(0.0, pr.scene.box_lo[static_cast<size_t>(b) * d + k]);
          const double hi = std::min(1.0, pr.scene.box_hi[static_cast<size_t>(b) * d + k]);
          v *= std::max(0.0, hi - lo);
        }
        blocked += v;
      }
      const double free_est = std::max(0.05, 1.0 - blocked);
      const double want = std::min(2.0 * pr.n, pr.n / free_est * 1.05) + 256.0;
      P.K = static_cast<int>(std::min<double>(static_cast<double>(budget), std::ceil(want)));
    }
    P.need_dedup = (pr.sampling.kind == GMT_SAMPLE_UNIFORM ||
                    pr.sampling.start_index + budget >= (1ULL << 53)) ? 1 : 0;
    P.start_index = pr.sampling.start_index;
    P.s0 = pcg_seed_state(pr.sampling.seed);
    P.box_off = box_total;
    P.cand_off = cand_total;
    P.row_off = row_start[q];
    double radius = pr.radius_override;
    if (!(radius > 0.0)) {
      rc = gmt_connection_radius(d, pr.n, pr.eta, 1.0, &radius);  // free_measure_upper_bound = 1
      if (rc) return rc;
    }
    P.radius = radius;
    P.r2_hi = radius * radius * (1.0 + 1e-12);
    P.r2_lo = radius * radius * (1.0 - 1e-12);
    {  // r-disk grid: cell side 1/G > r, at most kGridMaxCells cells
      double g = std::floor(kGridReach / (radius * (1.0 + 1e-9)));
      int G = g >= 1.0 ? static_cast<int>(std::min(g, 4096.0)) : 1;
      auto cells_of = [&](int gg) {
        int64_t c = 1;
        for (int k = 0; k < d; ++k) c *= gg;
        return c;
      };
      while (G > 1 && cells_of(G) > kGridMaxCells) --G;
      P.G = G;
      P.cell_off = cell_total;
      const int64_t cells = std::min<int64_t>(cells_of(G), kGridMaxCells);
      cell_total += cells + 1;
      max_cells = std::max<int>(max_cells, static_cast<int>(cells));
      max_rows = std::max(max_rows, pr.n + 1);
      if (pr.n + 1 > kGridMaxV) grid_ok = false;
    }
    box_lo.insert(box_lo.end(), pr.scene.box_lo, pr.scene.box_lo + static_cast<size_t>(P.nb) * d);
    box_hi.insert(box_hi.end(), pr.scene.box_hi, pr.scene.box_hi + static_cast<size_t>(P.nb) * d);
    std::copy(pr.scene.goal_lo, pr.scene.goal_lo + d, goal_lo.begin() + static_cast<size_t>(q) * d);
    std::copy(pr.scene.goal_hi, pr.scene.goal_hi + d, goal_hi.begin() + static_cast<size_t>(q) * d);
    std::copy(pr.init, pr.init + d, inits.begin() + static_cast<size_t>(q) * d);
    box_total += P.nb;
    cand_total += P.K;
    row_start[q + 1] = row_start[q] + pr.n + 1;
    max_K = std::max(max_K, P.K);
  }
  const int64_t R = row_start[count];
  std::vector<uint32_t> primes(kMaxDimB);
  for (int k = 0; k < kMaxDimB; ++k) primes[k] = nth_prime_h(k + 1);
  std::vector<double> fpow(static_cast<size_t>(kMaxDimB) * kHaltonDigits);
  for (int k = 0; k < kMaxDimB; ++k) {
    volatile double f = 1.0;  // (volatile: one IEEE division per step, as on the device)
    for (int i = 0; i < kHaltonDigits; ++i) {
      f = f / static_cast<double>(primes[k]);
      fpow[static_cast<size_t>(k) * kHaltonDigits + i] = f;
    }
  }

  // ---- device arena ----------------------------------------------------------
  auto al = [](size_t x) { return align16(x); };
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = al(off + bytes);
    return o;
  };
  const size_t o_probs = take(sizeof(BProb) * count);
  const size_t o_rs = take(sizeof(int64_t) * (count + 1));
  const size_t o_blo = take(sizeof(double) * std::max<int64_t>(box_total, 1) * d);
  const size_t o_bhi = take(sizeof(double) * std::max<int64_t>(box_total, 1) * d);
  const size_t o_glo = take(sizeof(double) * goal_lo.size());
  const size_t o_ghi = take(sizeof(double) * goal_hi.size());
  const size_t o_init = take(sizeof(double) * inits.size());
  const size_t o_pr = take(sizeof(uint32_t) * kMaxDimB);
  const size_t o_fp = take(sizeof(double) * kMaxDimB * kHaltonDigits);
  const size_t o_cand = take(sizeof(double) * cand_total * d);
  const size_t o_flag = take(cand_total);
  const size_t o_coords = take(sizeof(double) * R * d);
  const size_t o_res = take(sizeof(BOut) * count);
  const size_t o_cnt = take(sizeof(int64_t) * (R + 1));
  const size_t o_rp = take(sizeof(int64_t) * (R + 1));
  const size_t o_desc = take(sizeof(DevInstance) * count);
  const size_t o_cs = take(sizeof(int32_t) * cell_total);
  const size_t o_cl = take(sizeof(int32_t) * R);
  const size_t o_ovf = take(sizeof(int32_t));
  const size_t o_rst = take(sizeof(int64_t) * R);
  const size_t o_ren = take(sizeof(int64_t) * R);
  // Row scratch for d <= 3: the first C accepted targets of every row are
  // kept from the counting pass, so only rows with more than C are
  // evaluated twice.  C ~ twice the expected degree of the densest problem.
  int C = -1;
  if (d <= 3) {
    double deg = 0.0;
    for (const auto& P : probs) {
      double vol = 0.0;
      gmt_unit_ball_volume(d, &vol);
      deg = std::max(deg, vol * std::pow(P.radius, d) * (P.n + 1));
    }
    C = static_cast<int>(std::min(256.0, std::max(32.0, 2.0 * deg + 32.0)));
  }
  if (C <= 0 || std::getenv("GMT_NO_RDISK_GRID")) grid_ok = false;
  const size_t o_scol = take(C > 0 ? sizeof(int32_t) * static_cast<size_t>(R) * C : 0);
  const size_t o_scost = take(C > 0 ? sizeof(double) * static_cast<size_t>(R) * C : 0);
  size_t scan_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, static_cast<int64_t*>(nullptr),
                                static_cast<int64_t*>(nullptr), static_cast<int>(R + 1));
  const size_t o_scan = take(scan_bytes);
  Arena& work = ctx->pp_work;  // kept across calls (grows, never shrinks)
  int rc = work.reserve(off);
  if (rc) return rc;
  char* B = static_cast<char*>(work.ptr);
  auto* d_probs = reinterpret_cast<BProb*>(B + o_probs);
  auto* d_rs = reinterpret_cast<int64_t*>(B + o_rs);
  auto* d_blo = reinterpret_cast<double*>(B + o_blo);
  auto* d_bhi = reinterpret_cast<double*>(B + o_bhi);
  auto* d_glo = reinterpret_cast<double*>(B + o_glo);
  auto* d_ghi = reinterpret_cast<double*>(B + o_ghi);
  auto* d_init = reinterpret_cast<double*>(B + o_init);
  auto* d_pr = reinterpret_cast<uint32_t*>(B + o_pr);
  auto* d_fp = reinterpret_cast<double*>(B + o_fp);
  auto* d_cand = reinterpret_cast<double*>(B + o_cand);
  auto* d_flag = reinterpret_cast<uint8_t*>(B + o_flag);
  auto* d_coords = reinterpret_cast<double*>(B + o_coords);
  auto* d_res = reinterpret_cast<BOut*>(B + o_res);
  auto* d_cnt = reinterpret_cast<int64_t*>(B + o_cnt);
  auto* d_rp = reinterpret_cast<int64_t*>(B + o_rp);
  auto* d_desc = reinterpret_cast<DevInstance*>(B + o_desc);
  auto* d_cs = reinterpret_cast<int32_t*>(B + o_cs);
  auto* d_cl = reinterpret_cast<int32_t*>(B + o_cl);
  auto* d_ovf = reinterpret_cast<int32_t*>(B + o_ovf);
  auto* d_rst = reinterpret_cast<int64_t*>(B + o_rst);
  auto* d_ren = reinterpret_cast<int64_t*>(B + o_ren);
  void* d_scan = B + o_scan;
  auto* d_scol = C > 0 ? reinterpret_cast<int32_t*>(B + o_scol) : nullptr;
  auto* d_scost = C > 0 ? reinterpret_cast<double*>(B + o_scost) : nullptr;
  auto put = [&](void* dst, const void* src, size_t bytes) -> int {
    if (bytes) GMT_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
    return GMT_OK;
  };
  if ((rc = put(d_probs, probs.data(), sizeof(BProb) * count)) ||
      (rc = put(d_rs, row_start.data(), sizeof(int64_t) * (count + 1))) ||
      (rc = put(d_blo, box_lo.data(), sizeof(double) * box_lo.size())) ||
      (rc = put(d_bhi, box_hi.data(), sizeof(double) * box_hi.size())) ||
      (rc = put(d_glo, goal_lo.data(), sizeof(double) * goal_lo.size())) ||
      (rc = put(d_ghi, goal_hi.data(), sizeof(double) * goal_hi.size())) ||
      (rc = put(d_init, inits.data(), sizeof(double) * inits.size())) ||
      (rc = put(d_pr, primes.data(), sizeof(uint32_t) * kMaxDimB)) ||
      (rc = put(d_fp, fpow.data(), sizeof(double) * fpow.size()))) {
    return rc;
  }

  // ---- batched offline phase ------------------------------------------------
  {
    const dim3 gg((max_K + 255) / 256, count);
    if (d == 2)
      gen_batch_kernel<2><<<gg, 256, 0, s>>>(d_probs, d_blo, d_bhi, d_pr, d_fp, d_cand, d_flag);
    else if (d == 3)
      gen_batch_kernel<3><<<gg, 256, 0, s>>>(d_probs, d_blo, d_bhi, d_pr, d_fp, d_cand, d_flag);
    else
      gen_batch_kernel<0><<<gg, 256, 0, s>>>(d_probs, d_blo, d_bhi, d_pr, d_fp, d_cand, d_flag);
  }
  pack_batch_kernel<<<count, 1024, 0, s>>>(d_probs, d_flag, d_cand, d_coords, d_res);
  int max_n = 0;
  for (const auto& P : probs) max_n = std::max(max_n, P.n);
  dedup_batch_kernel<<<dim3((max_n + 255) / 256, count), 256, 0, s>>>(d_probs, d_coords, d_res);
  goal_batch_kernel<<<count, 256, 0, s>>>(d_probs, d_coords, d_glo, d_ghi, d_res);
  subst_batch_kernel<<<count, 256, 0, s>>>(d_probs, d_coords, d_blo, d_bhi, d_glo, d_ghi, d_pr, d_res);
  init_batch_kernel<<<count, 256, 0, s>>>(d_probs, d_coords, d_init, d_res);
  const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((R + 7) / 8, ctx->sm_count * 16)));
  if (grid_ok) {
    // counting pass through the cell grid (rows outside [0, V) stay 0)
    const int W = (max_rows + 31) / 32;
    const int S = max_rows <= 4096 ? 128 : kGridStride;
    const size_t smem = sizeof(uint32_t) * 8 * static_cast<size_t>(grid_warp_words(S, C));
    GMT_CUDA(cudaMemsetAsync(d_cnt, 0, sizeof(int64_t) * (R + 1), s));
    GMT_CUDA(cudaMemsetAsync(d_ovf, 0, sizeof(int32_t), s));
    GMT_CUDA(cudaMemsetAsync(d_rst, 0, sizeof(int64_t) * R, s));
    GMT_CUDA(cudaMemsetAsync(d_ren, 0, sizeof(int64_t) * R, s));
    const dim3 ggrid((max_cells + 7) / 8, count);
    auto launch = [&](auto kern) -> cudaError_t {
      cudaError_t e = raise_smem(reinterpret_cast<const void*>(kern), smem);
      if (e != cudaSuccess) return e;
      kern<<<ggrid, 256, smem, s>>>(d_probs, d_coords, d_res, d_cs, d_cl, W, d_cnt, d_scol, d_scost, C, d_ovf,
                                    d_rst, d_ren);
      return cudaGetLastError();
    };
    if (d == 2) {
      grid_build_kernel<2><<<count, 256, 0, s>>>(d_probs, d_coords, d_res, d_cs, d_cl);
      GMT_CUDA(S == 128 ? launch(&rdisk_grid_kernel<2, 128>) : launch(&rdisk_grid_kernel<2, kGridStride>));
    } else {
      grid_build_kernel<3><<<count, 256, 0, s>>>(d_probs, d_coords, d_res, d_cs, d_cl);
      GMT_CUDA(S == 128 ? launch(&rdisk_grid_kernel<3, 128>) : launch(&rdisk_grid_kernel<3, kGridStride>));
    }
    ctx->launches += 1;
  } else {
    GMT_CUDA(launch_rdisk_batch<false>(d, blocks, s, d_probs, d_rs, count, R, d_coords, d_res, d_cnt, nullptr,
                                       nullptr, nullptr, d_scol, d_scost, C));
  }
  GMT_CUDA(cudaMemsetAsync(d_cnt + R, 0, sizeof(int64_t), s));
  GMT_CUDA(cub::DeviceScan::ExclusiveSum(d_scan, scan_bytes, d_cnt, d_rp, static_cast<int>(R + 1), s));
  ctx->launches += 8;
  int64_t E = 0;
  int32_t overflow = 1;  // (the all-pairs count pass does not report it)
  std::vector<BOut> res(count);
  GMT_CUDA(cudaMemcpyAsync(&E, d_rp + R, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  if (grid_ok) GMT_CUDA(cudaMemcpyAsync(&overflow, d_ovf, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  GMT_CUDA(cudaMemcpyAsync(res.data(), d_res, sizeof(BOut) * count, cudaMemcpyDeviceToHost, s));
  GMT_CUDA(cudaStreamSynchronize(s));
  // No row overflowed the scratch: the solve reads the rows in place
  // (row-padded adjacency, DevInstance::out_end); else compact into a CSR.
  const bool padded = grid_ok && !overflow && std::getenv("GMT_BATCH_CSR") == nullptr;
  Arena edges;
  if (!padded) {
    rc = edges.reserve(al(sizeof(int32_t) * std::max<int64_t>(E, 1)) + sizeof(double) * std::max<int64_t>(E, 1));
    if (rc) return rc;
  }
  auto* d_col = padded ? d_scol : static_cast<int32_t*>(edges.ptr);
  auto* d_cost = padded ? d_scost
                        : reinterpret_cast<double*>(static_cast<char*>(edges.ptr) +
                                                    al(sizeof(int32_t) * std::max<int64_t>(E, 1)));
  if (!padded && C > 0) {
    compact_rows_batch_kernel<<<blocks, 256, 0, s>>>(d_cnt, d_rp, R, C, d_scol, d_scost, d_col, d_cost);
    ++ctx->launches;
  }
  if (!padded && (overflow || C <= 0)) {  // rows with more than C targets: evaluated again, straight into the CSR
    GMT_CUDA(launch_rdisk_batch<true>(d, blocks, s, d_probs, d_rs, count, R, d_coords, d_res, d_cnt, d_rp, d_col,
                                      d_cost, d_scol, d_scost, C));
    ++ctx->launches;
  }
  desc_batch_kernel<<<(count + 127) / 128, 128, 0, s>>>(d_probs, d_res, d_coords, d_blo, d_bhi, d_glo, d_ghi, d_rp,
                                                        d_col, d_cost, count, padded ? d_rst : nullptr,
                                                        padded ? d_ren : nullptr, d_desc);
  GMT_CUDA(cudaGetLastError());
  ++ctx->launches;

  // ---- the rare paths: the single-instance builder ---------------------------
  std::vector<gmt_instance*> single(count, nullptr);
  std::vector<SolveJob> jobs;
  std::vector<int> job_q;
  std::vector<int64_t> node_off(1, 0);
  int max_V = 0, max_nb = 0;
  for (int q = 0; q < count; ++q) {
    status_out[q] = GMT_OK;
    const DevInstance* inst_ptr = d_desc + q;
    int V = res[q].V, ii = res[q].init_index;
    if (res[q].fallback) {
      rc = gmt_instance_build(ctx, &problems[q], &single[q]);
      if (rc == GMT_E_GOAL_BLOCKED || rc == GMT_E_INFEASIBLE_SAMPLING) {
        status_out[q] = rc;  // the query's own build outcome (sampling.cpp:97-141)
        continue;
      }
      if (rc) {
        for (auto* p : single) gmt_instance_destroy(p);
        edges.release();
        return rc;
      }
      inst_ptr = static_cast<const DevInstance*>(single[q]->desc_mem.ptr);
      V = single[q]->desc.n;
      ii = single[q]->desc.init_index;
    }
    SolveJob job{};
    job.inst = inst_ptr;
    job.init_index = ii;
    job.mode = kModeGmt;
    job.lambda = problems[q].lambda;
    job.radius = probs[q].radius;
    jobs.push_back(job);
    job_q.push_back(q);
    node_off.push_back(node_off.back() + V);
    max_V = std::max(max_V, V);
    max_nb = std::max(max_nb, probs[q].nb);
  }

  // ---- one batched solve -----------------------------------------------------
  const int J = static_cast<int>(jobs.size());
  if (J > 0) {
    size_t smem = 0;
    int obs = 0;
    const int cluster = ctx->batch_cluster ? ctx->batch_cluster : 1;
    size_t gs = 0;
    rc = plan_smem(ctx, max_V, d, max_nb, cluster, &smem, &obs, &gs);
    std::vector<DevResult> rs;
    ResultScalars* sc = nullptr;
    if (rc == GMT_OK) rc = carve_results(ctx->res, J, node_off.data(), false, false, rs, &sc, nullptr);
    if (rc == GMT_OK && gs) rc = assign_gstate(ctx->gstate, jobs, gs);  // (too large for shared memory)
    if (rc == GMT_OK) {
      for (int k = 0; k < J; ++k) jobs[k].res = rs[k];
      rc = launch_jobs(ctx, jobs, cluster, ctx->batch_threads ? ctx->batch_threads : (cluster > 1 ? 512 : 256),
                       smem, obs, d);
    }
    std::vector<ResultScalars> hs(J);
    if (rc == GMT_OK) {
      cudaError_t e = cudaMemcpyAsync(hs.data(), sc, sizeof(ResultScalars) * J, cudaMemcpyDeviceToHost, s);
      if (e == cudaSuccess && path_states && path_cap > 0) {
        // path states straight from the device (results + instance descriptors)
        Arena pg;
        const size_t o_r = 0, o_i = al(sizeof(DevResult) * J), o_o = o_i + al(sizeof(void*) * J);
        rc = pg.reserve(o_o + sizeof(double) * static_cast<size_t>(J) * path_cap * d);
        if (rc == GMT_OK) {
          std::vector<const DevInstance*> ip(J);
          for (int k = 0; k < J; ++k) ip[k] = jobs[k].inst;
          char* g = static_cast<char*>(pg.ptr);
          e = cudaMemcpyAsync(g + o_r, rs.data(), sizeof(DevResult) * J, cudaMemcpyHostToDevice, s);
          if (e == cudaSuccess) e = cudaMemcpyAsync(g + o_i, ip.data(), sizeof(void*) * J, cudaMemcpyHostToDevice, s);
          if (e == cudaSuccess) {
            gather_paths_kernel<<<J, 128, 0, s>>>(reinterpret_cast<const DevResult*>(g + o_r),
                                                  reinterpret_cast<const DevInstance* const*>(g + o_i), J, path_cap,
                                                  d, reinterpret_cast<double*>(g + o_o));
            e = cudaGetLastError();
            ++ctx->launches;
          }
          std::vector<double> hp(static_cast<size_t>(J) * path_cap * d);
          if (e == cudaSuccess)
            e = cudaMemcpyAsync(hp.data(), g + o_o, sizeof(double) * hp.size(), cudaMemcpyDeviceToHost, s);
          if (e == cudaSuccess) e = cudaStreamSynchronize(s);
          if (e == cudaSuccess)
            for (int k = 0; k < J; ++k)
              std::memcpy(path_states + static_cast<size_t>(job_q[k]) * path_cap * d,
                          hp.data() + static_cast<size_t>(k) * path_cap * d, sizeof(double) * path_cap * d);
          pg.release();
        }
      }
      if (e == cudaSuccess) e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) rc = cuda_error(e, "gmt_plan_problems results");
    }
    if (rc == GMT_OK) {
      for (int k = 0; k < J; ++k) {
        gmt_plan_summary& o = summaries[job_q[k]];
        o.status = hs[k].status;
        o.goal_node = hs[k].goal_node;
        o.cost = hs[k].cost;
        o.iterations = hs[k].iterations;
        o.total_collision_checks = hs[k].total_checks;
        o.path_len = hs[k].path_len;
        o.num_stats = hs[k].num_stats;
      }
    }
  } else {
    GMT_CUDA(cudaStreamSynchronize(s));
  }
  for (auto* p : single) gmt_instance_destroy(p);
  edges.release();
  return rc;
}
