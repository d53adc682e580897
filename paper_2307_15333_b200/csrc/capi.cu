// capi.cu -- extern "C" entry points declared in include/dot_b200.h.
//
// Argument validation mirrors the reference's Python-side checks
// (render.py:38-41, 189-191; calibrate.py:36-42); kernels never raise.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include "dot_tree.cuh"
#include "dot_internal.h"

namespace dot {

static thread_local char g_err[512] = "";

int set_error(int status, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return status;
}

int check_cuda(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return DOT_OK;
    const int st = (e == cudaErrorMemoryAllocation) ? DOT_OOM : DOT_CUDA_ERR;
    return set_error(st, "%s: %s", what, cudaGetErrorString(e));
}

int check_launch(const char* what) { return check_cuda(cudaGetLastError(), what); }

// Stream-ordered scratch comes from the device's default memory pool; keep
// freed blocks in the pool (release threshold = max) so per-call scratch is
// recycled instead of being returned to the driver at every synchronisation.
void retain_pool_memory() {
    static thread_local int done_dev = -1;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev == done_dev) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done_dev = dev;
}

int validate_tree_view(const dot_tree_view* v) {
    if (!v) return set_error(DOT_BAD_ARG, "tree view is NULL");
    if (!v->node || v->n_nodes < 1) return set_error(DOT_BAD_ARG, "tree has no nodes");
    if (!v->sigma || !v->sh) return set_error(DOT_BAD_ARG, "tree payload is NULL");
    // node words are int32: child indices and ~pool id must fit
    if (v->n_nodes > INT32_MAX || v->capacity < 1 || v->capacity > INT32_MAX)
        return set_error(DOT_BAD_ARG, "n_nodes / capacity must be in [1, 2^31)");
    const int B = v->basis_count;
    if (B != 1 && B != 4 && B != 9 && B != 16)
        return set_error(DOT_BAD_ARG, "basis_count must be 1, 4, 9 or 16, got %d", B);
    if (v->sh_stride != pad4(3 * B))
        return set_error(DOT_BAD_ARG, "sh_stride must be %d for B=%d, got %d", pad4(3 * B), B,
                         v->sh_stride);
    if (!(v->half_extent > 0.0)) return set_error(DOT_BAD_ARG, "half_extent must be positive");
    if ((reinterpret_cast<uintptr_t>(v->sh) & 15) != 0)
        return set_error(DOT_BAD_ARG, "sh must be 16-byte aligned");
    return DOT_OK;
}

}  // namespace dot

using namespace dot;

extern "C" {

int dot_abi_version(void) { return 12; }

const char* dot_last_error(void) { return g_err; }

int dot_device_check(void) {
    int dev = 0, n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
        return set_error(DOT_NO_DEVICE, "no CUDA device visible");
    cudaGetDevice(&dev);
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, dev);
    if (p.major != 10) return set_error(DOT_NO_DEVICE, "device %s is sm_%d%d, need sm_100", p.name, p.major, p.minor);
    return DOT_OK;
}

void dot_exp_ref_host(const double* x, double* y, int64_t n) {
    for (int64_t i = 0; i < n; ++i) y[i] = exp_ref(x[i]);
}

int dot_exp_ref_device(const double* x, double* y, int64_t n, void* stream) {
    if (n < 0 || (n && (!x || !y))) return set_error(DOT_BAD_ARG, "bad arrays");
    return launch_exp_ref(x, y, n, static_cast<cudaStream_t>(stream));
}

int dot_sched_order(const int32_t* sorted_keys, int64_t n_rays, const uint16_t* table, int32_t* warp_order,
                    void* stream) {
    if (n_rays < 0 || (n_rays && (!sorted_keys || !table || !warp_order))) return set_error(DOT_BAD_ARG, "bad arrays");
    return launch_sched_order(sorted_keys, n_rays, table, warp_order, static_cast<cudaStream_t>(stream));
}

int dot_sched_update(const int32_t* sorted_keys, const uint16_t* ray_used, int64_t n_rays, uint16_t* table,
                     void* stream) {
    if (n_rays < 0 || (n_rays && (!sorted_keys || !ray_used || !table))) return set_error(DOT_BAD_ARG, "bad arrays");
    return launch_sched_update(sorted_keys, ray_used, n_rays, table, static_cast<cudaStream_t>(stream));
}

int dot_sched_order_costs(const uint16_t* ray_cost, int64_t n_costs, const int64_t* ray_index, int64_t n_rays,
                          int32_t chunk, int32_t* warp_order, void* stream) {
    if (n_rays < 0 || (n_rays && (!ray_cost || !warp_order))) return set_error(DOT_BAD_ARG, "bad arrays");
    if (chunk < 1 || chunk > 4096) return set_error(DOT_BAD_ARG, "chunk must be in 1..4096, got %d", chunk);
    if ((n_rays + 31) / 32 > INT32_MAX) return set_error(DOT_BAD_ARG, "batch too large to schedule");
    if (!ray_index && n_costs < n_rays) return set_error(DOT_BAD_ARG, "n_costs < n_rays without a ray_index");
    return launch_sched_order_costs(ray_cost, n_costs, ray_index, n_rays, chunk, warp_order,
                                    static_cast<cudaStream_t>(stream));
}

int dot_gather_keys(const int32_t* pool_keys, int64_t n_pool, const int64_t* ray_index, int64_t n_rays,
                    int32_t* keys, void* stream) {
    if (n_rays < 0 || (n_rays && (!pool_keys || !ray_index || !keys))) return set_error(DOT_BAD_ARG, "bad arrays");
    return launch_gather_keys(pool_keys, ray_index, n_pool, n_rays, keys, static_cast<cudaStream_t>(stream));
}

int dot_ray_costs(const dot_tree_view* tree, const double* origins, const double* dirs, int64_t n_pool,
                  const int64_t* ray_index, int64_t n_rays, double early_stop_eps, double t_near, double t_far,
                  uint16_t* cost, void* stream) {
    if (int st = validate_tree_view(tree)) return st;
    if (n_rays < 0 || (n_rays && (!origins || !dirs || !cost))) return set_error(DOT_BAD_ARG, "bad ray arrays");
    if (!ray_index && n_pool < n_rays) return set_error(DOT_BAD_ARG, "n_pool < n_rays without a ray_index");
    return launch_ray_costs(make_tree(*tree), origins, dirs, ray_index, n_pool, n_rays, early_stop_eps, t_near,
                            t_far, cost, static_cast<cudaStream_t>(stream));
}

int dot_locate_supported(const dot_tree_view* tree) {
    if (validate_tree_view(tree)) return 0;
    return locate_dyadic(*tree) ? 1 : 0;
}

int dot_locate_build(const dot_tree_view* tree, int32_t level, int32_t* table, void* stream) {
    if (int st = validate_tree_view(tree)) return st;
    if (!locate_dyadic(*tree))
        return set_error(DOT_BAD_ARG, "locate table needs a dyadic root (half_extent a power of two, "
                                      "centre a multiple of half * 2^-20, max_depth <= 21, capacity < 2^26)");
    if (level < 1 || level > 9)
        return set_error(DOT_BAD_ARG, "locate level must be in 1..9, got %d", level);
    if (!table) return set_error(DOT_BAD_ARG, "locate table is NULL");
    return launch_locate_build(make_tree(*tree), level, table, static_cast<cudaStream_t>(stream));
}

int dot_trace_count(const dot_tree_view* tree, const double* origins, const double* dirs,
                    int64_t n_rays, double t_near, double t_far, int64_t* counts, void* stream) {
    if (int st = validate_tree_view(tree)) return st;
    if (n_rays < 0 || (n_rays && (!origins || !dirs || !counts)))
        return set_error(DOT_BAD_ARG, "bad ray arrays");
    return launch_trace_count(make_tree(*tree), origins, dirs, n_rays, t_near, t_far, counts,
                              static_cast<cudaStream_t>(stream));
}

int dot_trace_fill(const dot_tree_view* tree, const double* origins, const double* dirs,
                   int64_t n_rays, double t_near, double t_far, const int64_t* offsets,
                   int64_t* seg_leaf, double* seg_t, double* seg_delta, void* stream) {
    if (int st = validate_tree_view(tree)) return st;
    if (n_rays < 0 || (n_rays && (!origins || !dirs || !offsets)))
        return set_error(DOT_BAD_ARG, "bad ray arrays");
    return launch_trace_fill(make_tree(*tree), origins, dirs, n_rays, t_near, t_far, offsets,
                             seg_leaf, seg_t, seg_delta, static_cast<cudaStream_t>(stream));
}

int dot_render_fwd(const dot_tree_view* tree, const double* origins, const double* dirs,
                   int64_t n_rays, const double* background, double early_stop_eps,
                   double t_near, double t_far, float* rgb, float* t_final, float* wsum,
                   float* depth, void* stream) {
    if (int st = validate_tree_view(tree)) return st;
    if (n_rays < 0 || (n_rays && (!origins || !dirs)) || !background)
        return set_error(DOT_BAD_ARG, "bad ray arrays");
    return launch_render_fwd(make_tree(*tree), origins, dirs, n_rays, background, early_stop_eps,
                             t_near, t_far, rgb, t_final, wsum, depth,
                             static_cast<cudaStream_t>(stream));
}

int dot_render_bwd(const dot_tree_view* tree, const double* origins, const double* dirs,
                   const double* targets, int64_t n_pool, const int64_t* ray_index,
                   const int32_t* warp_order, uint16_t* ray_used, uint16_t* ray_cost, int64_t n_rays,
                   const double* background, double early_stop_eps, double t_near, double t_far,
                   double grad_scale, float* grad_sigma, float* grad_sh, int32_t gsh_stride,
                   double* signal, uint8_t* touched, double* loss_sum, float* rgb_out,
                   double* weight_sum, double* weight_max, int32_t flags, void* stream) {
    if (int st = validate_tree_view(tree)) return st;
    if (n_rays < 0 || (n_rays && (!origins || !dirs || !targets)) || !background)
        return set_error(DOT_BAD_ARG, "bad ray arrays");
    if (!ray_index && n_pool < n_rays)
        return set_error(DOT_BAD_ARG, "n_pool (%lld) < n_rays (%lld) without a ray_index", (long long)n_pool,
                         (long long)n_rays);
#ifndef DOT_DIAG_FLAGS
    if (flags & ~32768) return set_error(DOT_BAD_ARG, "unknown dot_render_bwd flags 0x%x", flags);
#endif
    if (!grad_sigma || !grad_sh || !signal || !touched || !loss_sum)
        return set_error(DOT_BAD_ARG, "gradient / signal outputs must not be NULL");
    if (gsh_stride != tree->sh_stride)
        return set_error(DOT_BAD_ARG, "gsh_stride must equal sh_stride (%d)", tree->sh_stride);
    if ((reinterpret_cast<uintptr_t>(grad_sh) & 15) != 0)
        return set_error(DOT_BAD_ARG, "grad_sh must be 16-byte aligned");
    // the warp-cooperative sink packs (pool id, lane) into 32 bits: pool ids
    // need 27 bits, larger pools take the per-lane REDs
    if (tree->capacity > (int64_t(1) << 27)) flags |= 32768;
    return launch_render_bwd(make_tree(*tree), origins, dirs, targets, ray_index, n_pool, warp_order, ray_used,
                             ray_cost, n_rays, background, early_stop_eps, t_near, t_far, grad_scale, grad_sigma, grad_sh,
                             signal, touched, loss_sum, rgb_out, weight_sum, weight_max, flags,
                             static_cast<cudaStream_t>(stream));
}

int dot_signal_fwd(const dot_tree_view* tree, const double* origins, const double* dirs, int64_t n_pool,
                   const int64_t* ray_index, int64_t n_rays, double early_stop_eps, double t_near, double t_far,
                   double* signal, double* weight_sum, double* weight_max, uint8_t* touched,
                   uint64_t* invalid_rays, void* stream) {
    if (int st = validate_tree_view(tree)) return st;
    if (n_rays < 0 || (n_rays && (!origins || !dirs))) return set_error(DOT_BAD_ARG, "bad ray arrays");
    if (!ray_index && n_pool < n_rays)
        return set_error(DOT_BAD_ARG, "n_pool (%lld) < n_rays (%lld) without a ray_index", (long long)n_pool,
                         (long long)n_rays);
    if (!signal && !weight_sum && !weight_max && !touched)
        return set_error(DOT_BAD_ARG, "dot_signal_fwd: no output requested");
    return launch_signal_fwd(make_tree(*tree), origins, dirs, ray_index, n_pool, n_rays, early_stop_eps, t_near,
                             t_far, signal, weight_sum, weight_max, touched,
                             reinterpret_cast<unsigned long long*>(invalid_rays), static_cast<cudaStream_t>(stream));
}

int dot_ray_keys(const dot_tree_view* tree, const double* origins, const double* dirs, int64_t n_rays,
                 uint64_t* keys, void* stream) {
    if (int st = validate_tree_view(tree)) return st;
    if (n_rays < 0 || (n_rays && (!origins || !dirs || !keys))) return set_error(DOT_BAD_ARG, "bad arrays");
    return launch_ray_keys(make_tree(*tree), origins, dirs, n_rays, reinterpret_cast<unsigned long long*>(keys),
                           static_cast<cudaStream_t>(stream));
}

int dot_plan_sort(const int32_t* keys, const int64_t* ray_index, int64_t n_rays, int32_t begin_bit,
                  int32_t* sorted_keys, int64_t* sorted_index, void* stream) {
    if (n_rays < 0 || (n_rays && (!keys || !sorted_keys || !sorted_index)))
        return set_error(DOT_BAD_ARG, "bad plan_sort arrays");
    if (begin_bit < 0 || begin_bit > 30) return set_error(DOT_BAD_ARG, "begin_bit must be in 0..30");
    return run_plan_sort(keys, ray_index, n_rays, begin_bit, sorted_keys, sorted_index,
                         static_cast<cudaStream_t>(stream));
}

int64_t dot_plan_ranked_workspace(int64_t n_pool, int64_t n_rays, int32_t mode) {
    if (n_pool < 0 || n_rays < 0 || mode < DOT_PLAN_POSITIONS || mode > DOT_PLAN_SLOTS) return -1;
    return int64_t(plan_ranked_workspace(n_pool, n_rays, mode));
}

int dot_plan_ranked(const int32_t* rank, const int32_t* order, int64_t n_pool, const int64_t* ray_index,
                    int64_t n_rays, int32_t mode, const uint16_t* ray_cost, int32_t chunk, int32_t* warp_order,
                    void* workspace, int64_t workspace_bytes, int64_t* sorted_index, void* stream) {
    if (n_rays < 0 || n_pool < 0 || (n_rays && (!ray_index || !workspace || !sorted_index)))
        return set_error(DOT_BAD_ARG, "bad plan_ranked arrays");
    if (mode < DOT_PLAN_POSITIONS || mode > DOT_PLAN_SLOTS)
        return set_error(DOT_BAD_ARG, "plan_ranked: unknown mode %d", mode);
    if (mode == DOT_PLAN_POOL_RAYS && !order) return set_error(DOT_BAD_ARG, "plan_ranked: POOL_RAYS needs order");
    if (n_pool > INT32_MAX || n_rays > INT32_MAX)
        return set_error(DOT_BAD_ARG, "plan_ranked: pool and batch must have < 2^31 rays");
    if (workspace_bytes < int64_t(plan_ranked_workspace(n_pool, n_rays, mode)))
        return set_error(DOT_BAD_ARG, "plan_ranked: workspace of %lld bytes, %lld needed",
                         (long long)workspace_bytes, (long long)plan_ranked_workspace(n_pool, n_rays, mode));
    if (reinterpret_cast<uintptr_t>(workspace) & 255)
        return set_error(DOT_BAD_ARG, "plan_ranked: workspace must be 256-byte aligned");
    if (warp_order && (!ray_cost || chunk < 1 || chunk > 4096))
        return set_error(DOT_BAD_ARG, "plan_ranked: a warp order needs ray_cost and chunk in 1..4096");
    return run_plan_ranked(rank, order, n_pool, ray_index, n_rays, mode, ray_cost, chunk, warp_order, workspace,
                           sorted_index, static_cast<cudaStream_t>(stream));
}

int dot_ray_keys32(const dot_tree_view* tree, const double* origins, const double* dirs, int64_t n_pool,
                   const int64_t* ray_index, int64_t n_rays, int32_t* keys, void* stream) {
    if (int st = validate_tree_view(tree)) return st;
    if (n_rays < 0 || (n_rays && (!origins || !dirs || !keys))) return set_error(DOT_BAD_ARG, "bad arrays");
    if (!ray_index && n_pool < n_rays) return set_error(DOT_BAD_ARG, "n_pool < n_rays without a ray_index");
    return launch_ray_keys32(make_tree(*tree), origins, dirs, ray_index, n_pool, n_rays, keys,
                             static_cast<cudaStream_t>(stream));
}

int dot_render_camera(const dot_tree_view* tree, const double* cam_to_world, double focal, int32_t width,
                      int32_t height, const double* background, double early_stop_eps, float* rgb,
                      float* t_final, float* depth, void* stream) {
    if (int st = validate_tree_view(tree)) return st;
    if (!cam_to_world || !background || !rgb || width < 0 || height < 0 || !(focal > 0.0))
        return set_error(DOT_BAD_ARG, "bad camera arguments");
    return launch_render_camera(make_tree(*tree), cam_to_world, focal, width, height, background, early_stop_eps,
                                rgb, t_final, depth, static_cast<cudaStream_t>(stream));
}

int dot_render_cameras(const dot_tree_view* tree, const double* cam_to_world, const double* focal,
                       int32_t n_views, int32_t width, int32_t height, const double* background,
                       double early_stop_eps, float* rgb, float* t_final, float* depth, void* stream) {
    if (int st = validate_tree_view(tree)) return st;
    if (n_views < 0 || (n_views && (!cam_to_world || !focal || !rgb)) || !background || width < 0 || height < 0)
        return set_error(DOT_BAD_ARG, "bad camera arguments");
    for (int v = 0; v < n_views; ++v)
        if (!(focal[v] > 0.0)) return set_error(DOT_BAD_ARG, "focal[%d] must be positive", v);
    return launch_render_cameras(make_tree(*tree), cam_to_world, focal, n_views, width, height, background,
                                 early_stop_eps, rgb, t_final, depth, static_cast<cudaStream_t>(stream));
}

int dot_ray_stats(const dot_tree_view* tree, const double* origins, const double* dirs, int64_t n_rays,
                  double early_stop_eps, uint64_t* totals, void* stream) {
    if (int st = validate_tree_view(tree)) return st;
    if (n_rays < 0 || (n_rays && (!origins || !dirs)) || !totals) return set_error(DOT_BAD_ARG, "bad arrays");
    return launch_ray_stats(make_tree(*tree), origins, dirs, n_rays, early_stop_eps,
                            reinterpret_cast<unsigned long long*>(totals), static_cast<cudaStream_t>(stream));
}

}  // extern "C"
