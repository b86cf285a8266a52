// internal.cuh -- host-side internals shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "common.cuh"
#include "gmt_b200.h"

namespace gmtb {

constexpr int kMaxCopyChunks = 8;  // pipeline depth of gmt_plan_batch_host

extern thread_local std::string g_last_error;
int set_error(int code, const std::string& msg);
int cuda_error(cudaError_t e, const char* what);

// Device allocations are stream-ordered (cudaMallocAsync / cudaFreeAsync
// from the device's memory pool) on the stream of the context the current
// C-ABI call runs on, so building and freeing instances never synchronises
// the whole device (concurrent contexts overlap).  Outside a call (e.g.
// gmt_instance_destroy) the synchronous cudaMalloc / cudaFree are used.
extern thread_local cudaStream_t g_alloc_stream;

// Growable device allocation (never shrinks).
struct Arena {
  void* ptr = nullptr;
  size_t cap = 0;
  int reserve(size_t bytes);
  void release();
};

// Growable pinned host allocation.
struct HostPinned {
  void* ptr = nullptr;
  size_t cap = 0;
  int reserve(size_t bytes);
  void release();
};

}  // namespace gmtb

struct gmt_instance;
struct gmt_ctx;

namespace gmtb {
// The shared Halton sample pool of a context (pool.cu).
struct SamplePool;
void destroy_pool(SamplePool* p);  // (call with the context's AllocScope active)
}  // namespace gmtb

namespace gmtb {
// Makes `ctx`'s stream the allocation stream for the duration of a call.
struct AllocScope {
  cudaStream_t prev;
  explicit AllocScope(gmt_ctx* ctx);
  ~AllocScope() { g_alloc_stream = prev; }
};
}  // namespace gmtb

namespace gmtb {
// GMTG v1 graph cache (cache.cu).  CacheModel: the file's model fields
// (graph.cpp:251-254): Euclidean = {0, 0.1, 0.0, 0}; Dubins = the problem's
// rho, raw discretization_step and planar_cost_only.
struct CacheModel {
  int dubins = 0;
  double rho = 0.1;
  double step_raw = 0.0;
  int planar = 0;
};
int validate_scene(const gmt_scene* s);
int push_desc(gmt_ctx* ctx, gmt_instance* inst);
}  // namespace gmtb

struct gmt_instance {
  gmtb::Arena mem;       // samples, boxes, goal, graph rows, paths
  gmtb::Arena desc_mem;  // the device copy of `desc`
  gmtb::Arena aux;       // device-built instances: goal index list etc.
  gmtb::Arena mem2;      // device-built directed graphs: the in-rows
  gmtb::Arena mem3;      // device-built Dubins graphs: edge paths
  gmtb::Arena mem4;      // device-built kinodynamic graphs: per-in-edge waypoint tables
  gmtb::DevInstance desc{};
  int32_t graph_n = 0;
  const int32_t* goal_idx_dev = nullptr;
  gmtb::CacheModel cache_model{};  // the steering fields a graph cache file records
  ~gmt_instance() {
    mem.release();
    desc_mem.release();
    aux.release();
    mem2.release();
    mem3.release();
    mem4.release();
  }
};

struct gmt_ctx {
  int device = 0;
  int sm_count = 0;
  size_t smem_optin = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;            // host->device copies of batches
  cudaEvent_t copy_done[gmtb::kMaxCopyChunks] = {};
  int64_t launches = 0;
  int cluster = 0;        // single-query cluster size (0 = auto)
  int threads = 0;        // single-query CTA threads (0 = auto)
  int batch_threads = 0;  // batched CTA threads (0 = auto)
  int batch_cluster = 0;  // batched cluster size (0 = auto by steering model)
  int counting = 0;       // GMT_OPT_COUNTERS
  int64_t* counters = nullptr;  // device [3]
  gmtb::Arena res;        // single-query / host-batch results
  gmtb::Arena scratch;    // host-batch inputs, offline build scratch
  gmtb::Arena jobs;       // SolveJob table
  gmtb::Arena pp_work;    // gmt_plan_problems: the batched offline phase's scratch + padded rows
  gmtb::Arena pool_work;  // gmt_plan_problems over the shared pool: derived instances + scratch
  gmtb::Arena pool_rows;  //   ... their row regions
  gmtb::Arena pool_res;   //   ... their results
  gmtb::HostPinned pool_pinned;  //   ... the packed scene arrays (staging)
  gmtb::Arena gstate;     // global-memory wavefronts of queries too large for shared memory
  gmtb::SamplePool* pool = nullptr;  // shared Halton pool + its graph (built on first use, reused)
  gmtb::HostPinned pinned;
  gmtb::HostPinned pinned2;
  gmtb::HostPinned pinned_jobs;
  gmt_instance plan_inst; // staging instance of gmt_plan_host
};

// A batch of independent queries (gmt_batch_create / gmt_batch_create_problems).
struct gmt_batch {
  gmt_ctx* ctx = nullptr;
  gmtb::Arena res;
  gmtb::Arena jobs_mem;
  gmtb::Arena derived;                 // shared-pool batches: the derived per-query instances
  gmtb::Arena derived_rows;            //   ... their row regions
  gmtb::Arena gstate_mem;              // global-memory wavefronts (queries above the shared-memory opt-in)
  std::vector<gmt_instance*> owned;    // shared-pool batches: queries built one by one (rare paths)
  std::vector<gmtb::SolveJob> jobs;
  std::vector<gmtb::DevResult> results;
  std::vector<int64_t> node_off;
  gmtb::ResultScalars* scalars = nullptr;
  size_t smem = 0;
  int obs = 0;
  int cluster = 1;
  int threads = 256;
  int dim = 0;  // common dimension of the queries (0: mixed)
  bool pool = false;  // some jobs read shared-pool views (launch_solve's pool mode)
  bool lpt_done = false;  // the device job table is in largest-first order (gmt_batch_summaries)
  ~gmt_batch() {
    res.release();
    jobs_mem.release();
    derived.release();
    derived_rows.release();
    gstate_mem.release();
    for (gmt_instance* i : owned) delete i;
  }
};
