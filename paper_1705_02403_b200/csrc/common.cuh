// common.cuh -- shared device code of the B200 GMT* library.
//
// Bitwise parity with the reference (x86-64 SSE2 doubles, no FMA; SURVEY.md
// §7 H1) is obtained by (1) compiling the whole library with --fmad=false and
// (2) spelling every parity-critical operation with the correctly rounded
// intrinsics (__dadd_rn, __dsub_rn, __dmul_rn, __ddiv_rn, __dsqrt_rn) in the
// reference's operation order.  Comparisons mirror the reference's exact
// predicates (closed boxes, inclusive cube, std::max/std::min as ternaries).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace gmtb {

constexpr int kWarp = 32;
constexpr double kInf = __builtin_huge_val();

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~static_cast<size_t>(15); }

// A query's graph as a view of the shared Halton pool (pool.cu, SURVEY.md
// §8(e)): vertex x < n is pool point sel[x] (unless x = n - 1 was goal-
// substituted); its rows are the pool rows of sel[x] with every entry y
// mapped to rank[y] (kNoRank: not a vertex of the query, skipped), followed
// by its edges with the per-query vertices (g = n - 1 when subst, init = n;
// code bits 0/2: g -> x / init -> x in the in-row at spec entry spj[2x] /
// spj[2x + 1]; bits 1/3: x -> g / x -> init in the out-row).  g's and
// init's own rows are the special lists l = 0 out(g), 1 in(g), 2 out(init),
// 3 in(init) at scol/scost/stau + l * cap.
struct PoolView {
  const int64_t* in_ptr;   // pool graph (shared by every query)
  const int32_t* in_col;
  const double* in_cost;
  const double* in_tau;
  const int64_t* out_ptr;
  const int32_t* out_col;
  const int32_t* sel;      // per query
  const uint16_t* rank;
  const int32_t* code;
  const uint16_t* spj;
  const int32_t* scol;
  const double* scost;
  const double* stau;
  int32_t spec_len[4];
  int32_t subst;
  int32_t cap;
  int32_t kc;   // rank map length (pool points scanned)
  int32_t k;    // pool graph vertices
  const double* rec;  // per pool in-edge check records (pool_rec_len doubles each) or null
  int32_t rec_len;
  int32_t reserved;
};
constexpr uint16_t kPoolNoRank = 0xffffu;

// A pool edge's check record (pool.cu pool_rec_kernel): its trajectory's
// waypoints depend on the two pool points only, so the part of the lazy
// check that does not involve a query's boxes is done once per pool edge:
// [0..3) the minimum and [3..6) the maximum of the M + 1 waypoints' position
// coordinates (rec[0] = NaN when some waypoint leaves the unit cube, which
// makes polyline_free false whatever the boxes), then the waypoints'
// positions (M + 1) x 3, padded to 32-byte multiples.
constexpr int kPoolRecHead = 6;
__host__ __device__ inline int pool_rec_len(int segments) { return (kPoolRecHead + 3 * (segments + 1) + 3) & ~3; }

// Device-resident problem instance (ProblemInstance + ObstacleSet +
// GoalRegion, problem.hpp:52-57 / space.hpp:28-41).  A POD descriptor that
// lives in device memory; batched solves read one per query.
struct DevInstance {
  int32_t n;          // samples incl. appended init (V)
  int32_t dim;
  int32_t num_boxes;
  int32_t directed;   // 0: in-lists == out-lists
  int32_t goal_count; // samples.goal_indices.size()
  int32_t init_index; // built init index (instance_build) or -1
  double radius;      // graph radius (NeighborGraph::radius)
  int64_t num_edges;
  const double* coords;   // [n*dim] row-major
  const double* box_lo;   // [num_boxes*dim]
  const double* box_hi;
  const double* goal_lo;  // [dim]
  const double* goal_hi;
  const int64_t* out_ptr;
  const int32_t* out_col;
  const double* out_cost;
  const int64_t* in_ptr;  // == out_* when !directed
  const int32_t* in_col;
  const double* in_cost;
  // Row ends: null for CSR (row x ends at ptr[x + 1]); set for row-padded
  // adjacency (row x = [ptr[x], end[x]) with gaps between rows), which the
  // batched builder hands to the solve without compacting its row scratch.
  const int64_t* out_end;
  const int64_t* in_end;
  const int32_t* in_path; // may be null (all exact edges)
  const int64_t* path_ptr;
  const double* path_pts;
  // Kinodynamic instances built on the device (steering 2 = double
  // integrator, 3 = quadrotor) keep each in-edge's duration instead of a
  // cached polyline; the solve kernel regenerates the trajectory waypoints
  // of the one edge it checks (di.cuh, quad.cuh).  kin_p: DI {vmax, weight},
  // quadrotor {g, vmax, amax, ymax, wmax, weight}.
  const double* in_tau;
  // Optional per-in-edge waypoint tables ((kin_segments + 1) * dim doubles
  // each, solve.cu kino_table_kernel): the checks read instead of regenerate.
  const double* in_wp;
  // Out-edge views for the eager Dijkstra oracle: path ids of out-edges
  // (uploaded path graphs) and out-edge durations (kinodynamic).
  const int32_t* out_path;
  const double* out_tau;
  int32_t steering;
  int32_t kin_segments;
  double kin_p[6];
  // Non-null: the graph is a view of the shared pool (the row arrays above
  // are unused); only batched double-integrator solves see such instances.
  const PoolView* pool;
  // Materialised pool-derived rows: the pool in-edge of each in-row entry
  // (-1: an edge with g or init) and the pool's check records.
  const int32_t* in_pe;
  const double* pool_rec;
  int32_t pool_rec_len;
  int32_t reserved2;
};

// Scalars of one PlanResult (planner.hpp:43-51).
struct ResultScalars {
  int32_t status;
  int32_t goal_node;
  double cost;
  int64_t iterations;
  int64_t total_checks;
  int32_t path_len;
  int32_t num_stats;
  int32_t tree_size;
  int32_t reserved;
};

// Device outputs of one query; arrays sized n (stats n+1).  Any array
// pointer may be null: that output is skipped.
struct DevResult {
  ResultScalars* scalars;
  int32_t* path;
  uint8_t* label;
  double* tree_cost;
  int32_t* parent;
  int64_t* iter_added;
  int32_t* group_sizes;
  int32_t* nodes_added;
  int64_t* checks;
  int64_t* counters;  // optional [3]: in-row edges, out-row edges, open in-edges
};

constexpr int32_t kModeGmt = 0;  // gmt_plan (planner.cpp:94-198)
constexpr int32_t kModeFmt = 1;  // fmt_plan (planner.cpp:200-262)

struct SolveJob {
  const DevInstance* inst;
  DevResult res;
  int32_t init_index;
  int32_t mode;
  double lambda;
  double radius;  // params.radius (validated == graph radius on the host)
  // Wavefront state in global memory (the solve's shared-memory layout, one
  // block per query) for queries whose state exceeds the shared-memory
  // opt-in; null: the state lives in shared memory.
  unsigned char* gstate;
};

// ---- exact geometry (space.cpp) ------------------------------------------

// point_in_cube (space.cpp:40-45)
__device__ __forceinline__ bool point_in_cube(const double* p, int d) {
  for (int k = 0; k < d; ++k)
    if (p[k] < 0.0 || p[k] > 1.0) return false;
  return true;
}

// Aabb::contains (space.cpp:11-16) for box b of an AoS box array.
__device__ __forceinline__ bool box_contains(const double* lo, const double* hi, int d,
                                             const double* p) {
  for (int k = 0; k < d; ++k)
    if (p[k] < lo[k] || p[k] > hi[k]) return false;
  return true;
}

// euclidean_distance (space.cpp:126-133): sequential sum of squares, sqrt.
__device__ __forceinline__ double euclid_sq_seq(const double* a, const double* b, int d) {
  double sq = 0.0;
  for (int k = 0; k < d; ++k) {
    const double t = __dsub_rn(a[k], b[k]);
    sq = __dadd_rn(sq, __dmul_rn(t, t));
  }
  return sq;
}

// radical inverse (sampling.cpp:21-34): f /= base; r += f * (index % base).
__device__ __forceinline__ double halton_dev(uint64_t index, uint32_t base) {
  double f = 1.0, r = 0.0;
  const double fb = static_cast<double>(base);
  while (index > 0) {
    f = __ddiv_rn(f, fb);
    r = __dadd_rn(r, __dmul_rn(f, static_cast<double>(index % base)));
    index /= base;
  }
  return r;
}

}  // namespace gmtb
