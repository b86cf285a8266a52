// solve.cu -- the GMT* online phase (gmt_plan, planner.cpp:94-198) as ONE
// persistent kernel launch per query (or per batch of queries).
//
// Execution model:
//   * A query is solved by a thread-block cluster of CS CTAs (CS = 1 for
//     batched solves, up to 16 for a single latency-critical query).
//   * Every CTA keeps a full replica of the wavefront in shared memory:
//     cost f64[V] plus open/closed/group bitmasks.  Phases P0-P3 of the
//     reference pass (min-open, fast-forward, group, goal test) therefore run
//     redundantly and locally in every CTA with no communication.
//   * P4 (candidate gather) partitions the group over all warps of the
//     cluster; each unexplored out-neighbour is marked in the candidate
//     bitmask of its owner CTA (word-interleaved) with DSMEM atomics,
//     lane-aggregated with __match_any_sync/__reduce_or_sync.
//   * P5 (connect_candidate) runs warp-per-candidate on the owner CTA: the
//     lanes stream the candidate's in-row (col/cost, coalesced) from HBM/L2,
//     gather cost[y]/open(y) from the local replica, reduce (cost, position)
//     lexicographically (== the reference's strict-< first-in-list rule),
//     then slab-test the single best edge against the smem-staged boxes with
//     the boxes spread over the lanes.
//   * P6 (commit) writes the new cost into every replica (DSMEM stores) and
//     sets a `newopen` bit; labels only change at the next pass start, so
//     every candidate sees iteration-start labels exactly as in the
//     reference's parallel map + serial commit.
//   * Two cluster barriers per pass; no host round trip until the answer.
#include <cooperative_groups.h>

#include <cstdint>

#include "common.cuh"
#include "solve.cuh"

namespace cg = cooperative_groups;

namespace gmtb {

namespace {

constexpr uint32_t kFull = 0xffffffffu;
constexpr int32_t kNone = 0x7fffffff;

struct CtaShared {
  double red_min[32];
  double red_goal_c[32];
  int32_t red_goal_v[32];
  int32_t group_count;
  int32_t own_count;  // group members this CTA expands in P4
  int32_t cand_count;
  unsigned long long checks_acc;  // rank 0: cluster-wide checks of this pass
  int32_t added_acc;              // rank 0: cluster-wide additions of this pass
  int32_t feasible;
};

// Box access: box b, axis k at base[b*bs + k*as].
struct Boxes {
  const double* lo;
  const double* hi;
  int bs;  // box stride
  int as;  // axis stride
  int count;
};

template <int CS>
__device__ __forceinline__ void cluster_barrier() {
  if constexpr (CS > 1) {
    cg::this_cluster().sync();
  } else {
    __syncthreads();
  }
}

template <int CS, typename T>
__device__ __forceinline__ T* remote(T* p, int rank) {
  if constexpr (CS > 1) {
    return cg::this_cluster().map_shared_rank(p, rank);
  } else {
    return p;
  }
}

__device__ __forceinline__ bool point_free_warp(const double* p, int d, const Boxes& bx,
                                                int lane) {
  // point_free (space.cpp:47-54); boxes spread over the lanes.
  if (!point_in_cube(p, d)) return false;
  bool in = false;
  for (int b = lane; b < bx.count && !in; b += kWarp) {
    bool c = true;
    for (int k = 0; k < d; ++k) {
      const double x = p[k];
      if (x < bx.lo[b * bx.bs + k * bx.as] || x > bx.hi[b * bx.bs + k * bx.as]) {
        c = false;
        break;
      }
    }
    in = c;
  }
  return !__any_sync(kFull, in);
}

__device__ __forceinline__ bool segment_free_warp(const double* a, const double* b, int d,
                                                  const Boxes& bx, int lane) {
  // segment_free (space.cpp:80-90)
  bool same = true;
  for (int k = 0; k < d; ++k) same = same && (a[k] == b[k]);
  if (same) return point_free_warp(a, d, bx, lane);
  if (!point_in_cube(a, d) || !point_in_cube(b, d)) return false;
  bool hit = false;
  for (int i = lane; i < bx.count && !hit; i += kWarp) {
    hit = segment_hits_box(a, b, d, bx.lo + i * bx.bs, bx.hi + i * bx.bs, bx.as);
  }
  return !__any_sync(kFull, hit);
}

// motion_free (planner.cpp:54-60): cached polyline for path edges, exact
// clipping for straight edges.
__device__ bool motion_free_warp(const DevInstance& I, const Boxes& bx, int from, int to,
                                 int32_t pid, int lane) {
  const int d = I.dim;
  if (pid >= 0) {
    const int64_t a = I.path_ptr[pid], b = I.path_ptr[pid + 1];
    const double* pts = I.path_pts + a * d;
    if (b - a == 1) return point_free_warp(pts, d, bx, lane);
    for (int64_t s = 0; s + 1 < b - a; ++s) {
      if (!segment_free_warp(pts + s * d, pts + (s + 1) * d, d, bx, lane)) return false;
    }
    return true;
  }
  return segment_free_warp(I.coords + (int64_t)from * d, I.coords + (int64_t)to * d, d, bx, lane);
}

__device__ __forceinline__ double block_min(double v, double* red, int lane, int warp, int nw) {
  for (int o = 16; o; o >>= 1) {
    const double t = __shfl_xor_sync(kFull, v, o);
    v = t < v ? t : v;
  }
  if (lane == 0) red[warp] = v;
  __syncthreads();
  v = lane < nw ? red[lane] : kInf;
  for (int o = 16; o; o >>= 1) {
    const double t = __shfl_xor_sync(kFull, v, o);
    v = t < v ? t : v;
  }
  return v;
}

// Lexicographic (cost, index) minimum; "none" is (inf, kNone).
__device__ __forceinline__ void argmin_step(double& c, int32_t& v, double oc, int32_t ov) {
  if (oc < c || (oc == c && ov < v)) {
    c = oc;
    v = ov;
  }
}

__device__ __forceinline__ void block_argmin(double& c, int32_t& v, CtaShared& sh, int lane,
                                             int warp, int nw) {
  for (int o = 16; o; o >>= 1) {
    argmin_step(c, v, __shfl_xor_sync(kFull, c, o), __shfl_xor_sync(kFull, v, o));
  }
  if (lane == 0) {
    sh.red_goal_c[warp] = c;
    sh.red_goal_v[warp] = v;
  }
  __syncthreads();
  c = lane < nw ? sh.red_goal_c[lane] : kInf;
  v = lane < nw ? sh.red_goal_v[lane] : kNone;
  for (int o = 16; o; o >>= 1) {
    argmin_step(c, v, __shfl_xor_sync(kFull, c, o), __shfl_xor_sync(kFull, v, o));
  }
}

}  // namespace

// Batched solves (CS == 1) want several small CTAs per SM; single-query
// clusters want one wide CTA per SM.
template <int CS>
__global__ void __launch_bounds__(CS == 1 ? 256 : 512, CS == 1 ? 4 : 1) gmt_solve_kernel(const SolveJob* __restrict__ jobs,
                                                         int obs_in_smem) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ CtaShared sh;

  const int q = blockIdx.x / CS;
  int rank = 0;
  if constexpr (CS > 1) rank = static_cast<int>(cg::this_cluster().block_rank());
  const SolveJob job = jobs[q];
  const DevInstance& I = *job.inst;
  const DevResult R = job.res;
  const int n = I.n, d = I.dim, nb = I.num_boxes;
  const SolveLayout L = solve_layout(n, d, nb, obs_in_smem != 0);
  const int W = L.words;

  double* cost_s = reinterpret_cast<double*>(smem + L.off_cost);
  int32_t* parent_s = reinterpret_cast<int32_t*>(smem + L.off_parent);
  uint32_t* open_w = reinterpret_cast<uint32_t*>(smem + L.off_bits);
  uint32_t* closed_w = open_w + L.words_pad;
  uint32_t* group_w = closed_w + L.words_pad;
  uint32_t* newopen_w = group_w + L.words_pad;
  uint32_t* cand_w = newopen_w + L.words_pad;
  uint32_t* goal_w = cand_w + L.words_pad;
  int32_t* list = reinterpret_cast<int32_t*>(smem + L.off_list);

  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;

  Boxes bx;
  bx.count = nb;
  if (obs_in_smem) {
    double* lo = reinterpret_cast<double*>(smem + L.off_obs);
    double* hi = lo + (size_t)nb * d;
    for (int idx = tid; idx < nb * d; idx += nt) {
      const int b = idx / d, k = idx - b * d;
      lo[k * nb + b] = I.box_lo[idx];
      hi[k * nb + b] = I.box_hi[idx];
    }
    bx.lo = lo, bx.hi = hi, bx.bs = 1, bx.as = nb;
  } else {
    bx.lo = I.box_lo, bx.hi = I.box_hi, bx.bs = d, bx.as = 1;
  }

  // make_wavefront (planner.cpp:25-35) on every replica.
  const int init = job.init_index;
  for (int v = tid; v < n; v += nt) {
    cost_s[v] = kInf;
    parent_s[v] = -1;
  }
  for (int w = tid; w < W; w += nt) {
    open_w[w] = closed_w[w] = group_w[w] = newopen_w[w] = cand_w[w] = 0u;
  }
  // Goal membership is geometric: goal.contains(samples.states[v])
  // (planner.cpp:147), evaluated once per solve into a bitmask.
  for (int w = warp; w < W; w += nw) {
    const int v = w * 32 + lane;
    bool g = v < n;
    if (g) g = box_contains(I.goal_lo, I.goal_hi, d, I.coords + (int64_t)v * d);
    const uint32_t gb = __ballot_sync(kFull, g);
    if (lane == 0) goal_w[w] = gb;
  }
  if (R.iter_added) {
    for (int v = rank * nt + tid; v < n; v += CS * nt) R.iter_added[v] = (v == init) ? 0 : -1;
  }
  if (tid == 0) {
    sh.group_count = 0;
    sh.own_count = 0;
    sh.cand_count = 0;
    sh.checks_acc = 0ull;
    sh.added_acc = 0;
  }
  __syncthreads();

  // infeasible_input (planner.cpp:39-41, 108): empty tree.
  if (warp == 0) {
    const bool ok = I.goal_count > 0 &&
                    point_free_warp(I.coords + (int64_t)init * d, d, bx, lane);
    if (lane == 0) sh.feasible = ok ? 1 : 0;
  }
  __syncthreads();
  if (!sh.feasible) {
    if (rank == 0 && tid == 0) {
      ResultScalars s;
      s.status = 2;
      s.goal_node = -1;
      s.cost = kInf;
      s.iterations = 0;
      s.total_checks = 0;
      s.path_len = 0;
      s.num_stats = 0;
      s.tree_size = 0;
      s.reserved = 0;
      *R.scalars = s;
    }
    return;
  }
  if (tid == 0) {
    cost_s[init] = 0.0;
    open_w[init >> 5] |= 1u << (init & 31);
  }
  cluster_barrier<CS>();  // every replica initialised before any remote access

  const double delta = __dmul_rn(job.lambda, job.radius);  // GmtParams::delta
  long long i = 0;
  int pass = 0;
  int status = 1;
  int goal = -1;
  int gsize = 0;
  long long total_checks = 0;
  // Traffic counters for the roofline's algorithmic bytes:
  // per-lane counts of out-row edges (P4), in-row edges (P5) and in-edges
  // whose source was open (the cost[y] gathers).
  int cnt_out = 0, cnt_in = 0, cnt_open = 0;

  for (;;) {
    if (job.mode == kModeFmt) {
      // fmt_plan (planner.cpp:207-225): z = first minimum-cost open node;
      // the "group" is {z}; no thresholds.
      double zc = kInf;
      int32_t z = kNone;
      for (int w = warp; w < W; w += nw) {
        if ((open_w[w] >> lane) & 1u) argmin_step(zc, z, cost_s[w * 32 + lane], w * 32 + lane);
      }
      block_argmin(zc, z, sh, lane, warp, nw);
      if (z == kNone) {
        status = 1;
        break;
      }
      gsize = 1;
      if ((goal_w[z >> 5] >> (z & 31)) & 1u) {
        status = 0;
        goal = z;
        break;
      }
      if (tid == 0) {
        group_w[z >> 5] = 1u << (z & 31);
        if (((z >> 5) & (CS - 1)) == rank) {
          list[0] = z;
          sh.own_count = 1;
        }
      }
      __syncthreads();
    } else {
    // P0: min cost over open nodes (planner.cpp:119-122).
    double m = kInf;
    for (int w = warp; w < W; w += nw) {
      if ((open_w[w] >> lane) & 1u) {
        const double c = cost_s[w * 32 + lane];
        m = c < m ? c : m;
      }
    }
    m = block_min(m, sh.red_min, lane, warp, nw);
    if (m == kInf) {  // planner.cpp:123-127
      status = 1;
      break;
    }
    // P1: fast-forward (planner.cpp:132-136); i*delta is (double)i * delta.
    if (m > __dmul_rn(static_cast<double>(i), delta)) {
      const long long jump = static_cast<long long>(ceil(__ddiv_rn(m, delta)));
      i = jump > i + 1 ? jump : i + 1;
      while (m > __dmul_rn(static_cast<double>(i), delta)) ++i;
    }
    const double thr = __dmul_rn(static_cast<double>(i), delta);

    // P2 + P3: group bitmask/list and min-cost goal member (planner.cpp:137-149).
    double gc = kInf;
    int32_t gv = kNone;
    for (int w = warp; w < W; w += nw) {
      const uint32_t ow = open_w[w];
      const int v = w * 32 + lane;
      const bool g = ((ow >> lane) & 1u) && cost_s[v] <= thr;
      const uint32_t gb = __ballot_sync(kFull, g);
      if (gb) {
        // Every CTA sees the whole group; the members of words w = rank
        // (mod CS) go to this CTA's P4 work list (list order is arbitrary,
        // ownership is not).
        int base = 0;
        const bool own = (w & (CS - 1)) == rank;
        if (lane == 0) {
          group_w[w] = gb;
          atomicAdd(&sh.group_count, __popc(gb));
          if (own) base = atomicAdd(&sh.own_count, __popc(gb));
        }
        base = __shfl_sync(kFull, base, 0);
        if (g) {
          if (own) list[base + __popc(gb & ((1u << lane) - 1u))] = v;
          if ((goal_w[w] >> lane) & 1u) argmin_step(gc, gv, cost_s[v], v);
        }
      }
    }
    block_argmin(gc, gv, sh, lane, warp, nw);
    gsize = sh.group_count;
    if (gv != kNone) {  // planner.cpp:150-156
      status = 0;
      goal = gv;
      break;
    }
    }  // GMT group selection

    // P4: mark unexplored out-neighbours of the group (planner.cpp:159-166).
    const int own = sh.own_count;
    for (int k = warp; k < own; k += nw) {
      const int g = list[k];
      const int64_t e0 = I.out_ptr[g], e1 = I.out_ptr[g + 1];
      for (int64_t base = e0; base < e1; base += kWarp) {
        const int64_t e = base + lane;
        bool un = false;
        int x = 0;
        if (e < e1) {
          ++cnt_out;
          x = __ldg(I.out_col + e);
          un = !(((open_w[x >> 5] | closed_w[x >> 5]) >> (x & 31)) & 1u);
        }
        const uint32_t act = __ballot_sync(kFull, un);
        if (un) {
          const int word = x >> 5;
          const uint32_t peers = __match_any_sync(act, word);
          const uint32_t bits = __reduce_or_sync(peers, 1u << (x & 31));
          if (lane == __ffs(peers) - 1) {
            atomicOr(remote<CS>(cand_w, word & (CS - 1)) + word, bits);
          }
        }
      }
    }
    cluster_barrier<CS>();  // [1] candidate marks complete

    // Own candidates (words w = rank mod CS) -> list.
    for (int w = rank + CS * tid; w < W; w += CS * nt) {
      uint32_t bits = cand_w[w];
      if (bits) {
        cand_w[w] = 0u;
        int base = atomicAdd(&sh.cand_count, __popc(bits));
        while (bits) {
          const int b = __ffs(bits) - 1;
          bits &= bits - 1u;
          list[base++] = w * 32 + b;
        }
      }
    }
    __syncthreads();
    const int ccount = sh.cand_count;

    // P5 + P6: connect_candidate (planner.cpp:62-90) and commit (178-189).
    int my_checks = 0, my_added = 0;
    for (int k = warp; k < ccount; k += nw) {
      const int x = list[k];
      const int64_t e0 = I.in_ptr[x], e1 = I.in_ptr[x + 1];
      double bv = kInf;
      long long be = -1;
      int by = -1;
      for (int64_t e = e0 + lane; e < e1; e += kWarp) {
        const int y = __ldg(I.in_col + e);
        ++cnt_in;
        if ((open_w[y >> 5] >> (y & 31)) & 1u) {
          ++cnt_open;
          const double c = __dadd_rn(cost_s[y], __ldg(I.in_cost + e));
          if (c < bv) {
            bv = c;
            be = e;
            by = y;
          }
        }
      }
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(kFull, bv, o);
        const long long oe = __shfl_xor_sync(kFull, be, o);
        const int oy = __shfl_xor_sync(kFull, by, o);
        if (ov < bv || (ov == bv && oe >= 0 && (be < 0 || oe < be))) {
          bv = ov;
          be = oe;
          by = oy;
        }
      }
      if (be < 0) continue;  // no open in-neighbour: not checked
      ++my_checks;
      const int32_t pid = I.in_path ? __ldg(I.in_path + be) : -1;
      if (motion_free_warp(I, bx, by, x, pid, lane)) {
        ++my_added;
        if (lane < CS) {
          remote<CS>(cost_s, lane)[x] = bv;
          atomicOr(remote<CS>(newopen_w, lane) + (x >> 5), 1u << (x & 31));
        }
        if (lane == 0) {
          remote<CS>(parent_s, 0)[x] = by;
          if (R.iter_added) R.iter_added[x] = i;
        }
      }
    }
    if (lane == 0 && (my_checks | my_added)) {
      atomicAdd(remote<CS>(&sh.checks_acc, 0), static_cast<unsigned long long>(my_checks));
      atomicAdd(remote<CS>(&sh.added_acc, 0), my_added);
    }
    cluster_barrier<CS>();  // [2] commits visible in every replica

    if (rank == 0 && tid == 0) {  // IterationStats (planner.cpp:192-194)
      if (R.group_sizes) {
        R.group_sizes[pass] = gsize;
        R.nodes_added[pass] = sh.added_acc;
        R.checks[pass] = static_cast<int64_t>(sh.checks_acc);
      }
      total_checks += static_cast<long long>(sh.checks_acc);
      sh.added_acc = 0;
      sh.checks_acc = 0ull;
    }
    // Close the group, open the committed nodes (planner.cpp:178-190).
    for (int w = tid; w < W; w += nt) {
      const uint32_t gw = group_w[w];
      closed_w[w] |= gw;
      open_w[w] = (open_w[w] & ~gw) | newopen_w[w];
      newopen_w[w] = 0u;
      group_w[w] = 0u;
    }
    if (tid == 0) {
      sh.group_count = 0;
      sh.own_count = 0;
      sh.cand_count = 0;
    }
    __syncthreads();
    ++i;
    ++pass;
  }

  if (R.counters) {
    long long a = cnt_in, b = cnt_out, c = cnt_open;
    for (int o = 16; o; o >>= 1) {
      a += __shfl_xor_sync(kFull, a, o);
      b += __shfl_xor_sync(kFull, b, o);
      c += __shfl_xor_sync(kFull, c, o);
    }
    if (lane == 0) {
      atomicAdd(reinterpret_cast<unsigned long long*>(R.counters + 0), static_cast<unsigned long long>(a));
      atomicAdd(reinterpret_cast<unsigned long long*>(R.counters + 1), static_cast<unsigned long long>(b));
      atomicAdd(reinterpret_cast<unsigned long long*>(R.counters + 2), static_cast<unsigned long long>(c));
    }
  }
  if (rank != 0) return;
  // Outputs (rank 0 holds the parent replica).
  if (R.label) {
    for (int v = tid; v < n; v += nt) {
      const uint32_t bit = 1u << (v & 31);
      R.label[v] = (open_w[v >> 5] & bit) ? 1 : ((closed_w[v >> 5] & bit) ? 2 : 0);
      R.tree_cost[v] = cost_s[v];
      R.parent[v] = parent_s[v];
    }
  }
  if (tid == 0) {
    ResultScalars s;
    s.status = status;
    s.goal_node = goal;
    s.iterations = i;
    s.tree_size = n;
    s.reserved = 0;
    s.num_stats = pass;
    s.total_checks = total_checks;
    if (status == 0) {
      if (R.group_sizes) {  // final group pushes 0/0 (planner.cpp:151-152)
        R.group_sizes[pass] = gsize;
        R.nodes_added[pass] = 0;
        R.checks[pass] = 0;
      }
      s.num_stats = pass + 1;
      s.cost = cost_s[goal];
      int len = 0;
      for (int v = goal; v >= 0; v = parent_s[v]) ++len;
      int k = len;
      if (R.path) {
        for (int v = goal; v >= 0; v = parent_s[v]) R.path[--k] = v;
      }
      s.path_len = len;
    } else {
      s.cost = kInf;
      s.path_len = 0;
    }
    *R.scalars = s;
  }
}

template <int CS>
static cudaError_t launch_cs(const SolveJob* jobs, int count, int threads, size_t smem,
                             int obs_in_smem, cudaStream_t stream) {
  auto kern = gmt_solve_kernel<CS>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
  if (err != cudaSuccess) return err;
  if (CS > 8) {
    err = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (err != cudaSuccess) return err;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(count) * CS, 1, 1);
  cfg.blockDim = dim3(static_cast<unsigned>(threads), 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  if (CS > 1) {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  return cudaLaunchKernelEx(&cfg, kern, jobs, obs_in_smem);
}

cudaError_t launch_solve(const SolveJob* jobs, int count, int cluster, int threads, size_t smem,
                         int obs_in_smem, cudaStream_t stream) {
  switch (cluster) {
    case 1: return launch_cs<1>(jobs, count, threads, smem, obs_in_smem, stream);
    case 2: return launch_cs<2>(jobs, count, threads, smem, obs_in_smem, stream);
    case 4: return launch_cs<4>(jobs, count, threads, smem, obs_in_smem, stream);
    case 8: return launch_cs<8>(jobs, count, threads, smem, obs_in_smem, stream);
    case 16: return launch_cs<16>(jobs, count, threads, smem, obs_in_smem, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace gmtb
