// offline.cuh -- internal entry points of the offline phase (sample.cu, graph.cu).
#pragma once

#include <cstdint>
#include <vector>

#include "internal.cuh"

namespace gmtb {

// build_neighbor_graph on device coordinates; the CSR lands in `out`.
int build_graph_dev(gmt_ctx* ctx, const double* d_coords, int n, int d, double radius, Arena& out,
                    int64_t* num_edges, int64_t** row_ptr, int32_t** col, double** cost);

// sample_free on the device.  `out` receives coords [(n+1)*dim] (room for
// append_init), heading [n+1] when with_heading, and the goal index list
// [n+1]; *goal_count is set.
struct DevSamples {
  double* coords = nullptr;
  double* heading = nullptr;
  int32_t* goal_idx = nullptr;
  int32_t goal_count = 0;
  int32_t n = 0;
};
int sample_free_dev(gmt_ctx* ctx, int32_t n, const gmt_scene* scene, const gmt_sample_source* src,
                    Arena& out, DevSamples* s);

// Kinodynamic graphs (di_graph.cu): one direction's compressed rows.
struct DiRows {
  int64_t* ptr = nullptr;
  int32_t* col = nullptr;
  double* cost = nullptr;
  double* tau = nullptr;
  int64_t edges = 0;
};
struct DiParams;
struct QuadParams;
DiParams to_di(const gmt_di_params* p);
QuadParams to_quad(const gmt_quad_params* p);
int validate_di(const gmt_di_params* p);
// |dp| bound of the double integrator's exact-safe pair prefilter (di_graph.cu).
double di_prefilter_bound(const DiParams& P, double radius);
int validate_quad(const gmt_quad_params* p);
int build_di_graph_dev(gmt_ctx* ctx, const double* d_coords, int n, const gmt_di_params* p, double radius,
                       Arena& out_mem, DiRows* out, Arena& in_mem, DiRows* in);
int build_quad_graph_dev(gmt_ctx* ctx, const double* d_coords, int n, const gmt_quad_params* p,
                         double radius, Arena& out_mem, DiRows* out, Arena& in_mem, DiRows* in);

// Dubins-airplane graphs (di_graph.cu): rows as above plus edge paths.
struct DubinsGraphPaths {
  int64_t* path_ptr = nullptr;  // [E+1], path e = out-edge e
  int32_t* in_path = nullptr;   // [E] in-edge -> path id
  int32_t* out_path = nullptr;  // [E] identity
  double* pts = nullptr;        // [num_points * dim] positions
  int64_t num_points = 0;
};
int validate_dubins(const gmt_dubins_params* p, int pd);
// Host out-rows (a graph cache hit): the rows are taken as given, and only
// the in-rows, segment counts and edge paths are derived on the device.
struct HostRows {
  const std::vector<int64_t>* ptr;
  const std::vector<int32_t>* col;
  const std::vector<double>* cost;
};
int build_dubins_graph_dev(gmt_ctx* ctx, const double* d_coords, const double* d_heading, int n, int pd,
                           const gmt_dubins_params* p, double radius, Arena& out_mem, DiRows* out,
                           Arena& in_mem, DiRows* in, Arena& path_mem, DubinsGraphPaths* paths,
                           const HostRows* cached = nullptr);

// GMTG v1 graph cache (cache.cu); CacheModel: internal.cuh.
CacheModel cache_model_of(const gmt_problem* p);
int problem_key_of(const gmt_problem* p, uint64_t* out);
int cache_write(const char* file, uint64_t key, int32_t n, double radius, const int64_t* ptr,
                const int32_t* col, const double* cost, const CacheModel& m = CacheModel{});
int cache_read(const char* file, uint64_t key, int32_t n, double radius, std::vector<int64_t>& ptr,
               std::vector<int32_t>& col, std::vector<double>& cost, bool* hit,
               const CacheModel& m = CacheModel{});

// append_init on device samples (sampling.cpp:144-154).
int append_init_dev(gmt_ctx* ctx, int dim, DevSamples* s, const double* init, int has_heading,
                    double heading, const double* goal_lo, const double* goal_hi, int32_t* index);

}  // namespace gmtb
