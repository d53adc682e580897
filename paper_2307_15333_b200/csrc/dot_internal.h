// dot_internal.h -- shared host-side helpers of the C ABI implementation.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/dot_b200.h"

namespace dot {

struct TreeDev;

// Outputs of the record-emitting backward (sorted.cu / render.cu EmitSink).
struct EmitArgs {
    unsigned long long* ctr;         // [0] records reserved, [1] rays that did not fit
    int64_t cap;                     // record slots
    unsigned long long* keys;        // [cap] pool id << ray_bits | original ray index
    float4* rec;                     // [cap] (dsigma, w0, w1, w2)
    double* recq;                    // [cap] q = 1 - alpha
    float* basis;                    // [n * B] SH basis per original ray
    double* loss_ray;                // [n] squared error per original ray
    int ray_bits;
};

int set_error(int status, const char* fmt, ...);
int check_launch(const char* what);
int check_cuda(cudaError_t e, const char* what);
void retain_pool_memory();
int validate_tree_view(const dot_tree_view* v);

int launch_trace_count(const TreeDev& T, const double* o, const double* d, int64_t n,
                       double tn, double tf, int64_t* counts, cudaStream_t s);
int launch_trace_fill(const TreeDev& T, const double* o, const double* d, int64_t n, double tn,
                      double tf, const int64_t* off, int64_t* leaf, double* t, double* dl,
                      cudaStream_t s);
int launch_render_fwd(const TreeDev& T, const double* o, const double* d, int64_t n,
                      const double* bg, double eps, double tn, double tf, float* rgb, float* tfin,
                      float* wsum, float* depth, cudaStream_t s);
int launch_render_bwd(const TreeDev& T, const double* o, const double* d, const double* tgt,
                      const int64_t* ray_idx, int64_t n_pool, const int32_t* warp_order, uint16_t* ray_used,
                      uint16_t* ray_cost, int64_t n, const double* bg, double eps, double tn, double tf, double gs, float* gsig,
                      float* gsh, double* signal, uint8_t* touched, double* loss, float* rgb_out,
                      double* wsum, double* wmax, int flags, cudaStream_t s);
int launch_signal_fwd(const TreeDev& T, const double* o, const double* d, const int64_t* ray_idx, int64_t n_pool,
                      int64_t n, double eps, double tn, double tf, double* signal, double* wsum, double* wmax,
                      uint8_t* touched, unsigned long long* invalid, cudaStream_t s);
int launch_sched_order(const int32_t* keys, int64_t n, const uint16_t* table, int32_t* warp_order, cudaStream_t s);
int launch_sched_order_costs(const uint16_t* slot_cost, int64_t n_costs, const int64_t* ray_idx, int64_t n,
                             int chunk, int32_t* warp_order, cudaStream_t s);
int launch_ray_costs(const TreeDev& T, const double* o, const double* d, const int64_t* ray_idx, int64_t n_pool,
                     int64_t n, double eps, double tn, double tf, uint16_t* cost, cudaStream_t s);
int launch_sched_update(const int32_t* keys, const uint16_t* ray_used, int64_t n, uint16_t* table, cudaStream_t s);
int launch_ray_keys(const TreeDev& T, const double* o, const double* d, int64_t n, unsigned long long* keys,
                    cudaStream_t s);
int run_plan_sort(const int32_t* keys, const int64_t* ray_index, int64_t n, int begin_bit,
                  int32_t* sorted_keys, int64_t* sorted_index, cudaStream_t s);
int launch_gather_keys(const int32_t* pool_keys, const int64_t* ray_idx, int64_t n_pool, int64_t n, int32_t* keys,
                       cudaStream_t s);
size_t plan_ranked_workspace(int64_t n_pool, int64_t n, int mode);
int run_plan_ranked(const int32_t* rank, const int32_t* order, int64_t n_pool, const int64_t* ray_idx, int64_t n,
                    int mode, const uint16_t* ray_cost, int chunk, int32_t* warp_order, void* ws, int64_t* out,
                    cudaStream_t s);
int launch_ray_keys32(const TreeDev& T, const double* o, const double* d, const int64_t* ray_idx,
                      int64_t n_pool, int64_t n, int32_t* keys, cudaStream_t s);
int launch_render_cameras(const TreeDev& T, const double* cam_to_world, const double* focal, int n_views,
                          int width, int height, const double* bg, double eps, float* rgb, float* tfin,
                          float* depth, cudaStream_t s);
int launch_render_camera(const TreeDev& T, const double* cam_to_world, double focal, int width, int height,
                         const double* bg, double eps, float* rgb, float* tfin, float* depth, cudaStream_t s);
int launch_render_bwd_emit(const TreeDev& T, const double* o, const double* d, const double* tgt,
                           const int64_t* ray_idx, const int32_t* warp_order, uint16_t* ray_used, int64_t n,
                           const double* bg, double eps, double tn, double tf, double gs, uint8_t* touched,
                           const EmitArgs& ea, cudaStream_t s);
int launch_exp_ref(const double* x, double* y, int64_t n, cudaStream_t s);
int launch_locate_build(const TreeDev& T, int level, int32_t* table, cudaStream_t s);
int launch_ray_stats(const TreeDev& T, const double* o, const double* d, int64_t n, double eps,
                     unsigned long long* out, cudaStream_t s);

}  // namespace dot
