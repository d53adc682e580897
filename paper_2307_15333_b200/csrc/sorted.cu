// sorted.cu -- deterministic fused forward + backward (dot_render_bwd_sorted).
//
// The reference reduces per-segment gradients serially in ray-major order
// (scatter_kernel, _kernels.py:327-346): for every ray in batch order, for
// every segment in march order, signal[leaf] += Q, grad[leaf] += ... in f64.
// The default GPU path (render.cu, AtomicSink) reduces with float atomics,
// whose order varies from run to run.  This path reproduces the reference's
// order instead:
//   1. the buffered fused kernel (EmitSink) writes one record per composited
//      segment, keyed (pool id << ray_bits | original ray index);
//   2. a CUB radix sort over the key bits orders the records by leaf, and
//      within a leaf by original ray index -- exactly scatter_kernel's order;
//   3. the runs of equal leaf are listed longest first and
//      reduce_runs_kernel sums each run sequentially in f64 (half a warp per
//      run: lane b owns basis column b of the three channels), adding the
//      result to the f32 gradients / f64 signal;
//   4. the per-ray squared errors are summed by cub::DeviceReduce (fixed
//      order).
// Everything is a pure function of the inputs: results are bit-identical
// from run to run, and the signal is bit-identical to the reference's
// whenever the per-segment Q values are (they are computed from the
// bit-exact traversal; exp may differ from glibc's by an ulp).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>
#include "dot_tree.cuh"
#include "dot_internal.h"

namespace dot {

int launch_iota(int32_t* p, int64_t n, cudaStream_t s);
int launch_add_f64(double* dst, const double* src, cudaStream_t s);

// Per leaf, the run of its records in sorted (= the reference's ray-major)
// order.  run_heads_kernel flags run starts; the runs are then listed
// longest first (a leaf hit by thousands of rays is a long serial f64 sum:
// started first it overlaps the bulk instead of forming the kernel's tail).

__global__ void run_heads_kernel(const unsigned long long* __restrict__ keys, int64_t total, int ray_bits,
                                 int32_t* __restrict__ flag) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= total) return;
    flag[i] = i == 0 || (keys[i - 1] >> ray_bits) != (keys[i] >> ray_bits);
}

// key = ~length (descending sort), value = run start
__global__ void run_lengths_kernel(const int32_t* __restrict__ head, const int32_t* __restrict__ n_runs,
                                   int64_t total, uint32_t* __restrict__ len_key) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t m = *n_runs;
    if (j >= m) return;
    const int64_t end = j + 1 < m ? head[j + 1] : total;
    len_key[j] = ~uint32_t(end - head[j]);
}

#ifndef DOT_REDUCE_MINB
#define DOT_REDUCE_MINB 1
#endif
// records per group of loads in flight: 4 (80 registers, 6 blocks per SM)
// beats 8 (128 registers, 4 blocks): 1.81 -> 1.26 ms per 2^20-ray batch;
// 2 / 3 / 6: 1.81 / 1.40 / 1.36 ms
#ifndef DOT_REDUCE_U
#define DOT_REDUCE_U 4
#endif

template <int B>
__global__ void __launch_bounds__(128, DOT_REDUCE_MINB) reduce_runs_kernel(
    const unsigned long long* __restrict__ keys, const int32_t* __restrict__ idx,
    const int32_t* __restrict__ run_start, const uint32_t* __restrict__ run_len_key,
    const int32_t* __restrict__ n_runs, int ray_bits, const float4* __restrict__ rec,
    const double* __restrict__ recq, const float* __restrict__ basis, float* __restrict__ gsig,
    float* __restrict__ gsh, double* __restrict__ signal) {
    constexpr int S = pad4(3 * B);
    // half a warp per run: lane b owns basis column b of the three channels
    const int64_t h = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 4;
    const int b = threadIdx.x & 15;
    if (h >= *n_runs) return;
    const unsigned long long rmask = (1ull << ray_bits) - 1ull;
    int64_t j = run_start[h];
    const int64_t end = j + int64_t(~run_len_key[h]);
    const unsigned long long pid = keys[j] >> ray_bits;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    if (b < B) {
        a0 = double(gsh[pid * S + 0 * B + b]);
        a1 = double(gsh[pid * S + 1 * B + b]);
        a2 = double(gsh[pid * S + 2 * B + b]);
    }
    double as = double(gsig[pid]);
    double aq = signal[pid];
    // records in groups of U: all loads of a group are issued before its
    // (sequential, in-order) additions, so a run costs ~1 memory latency per
    // U records instead of per record
    constexpr int U = DOT_REDUCE_U;
    for (; j < end; j += U) {
        int32_t ix[U];
        unsigned long long kk[U];
        float4 r[U];
        double q[U], bv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const bool in = j + u < end;
            kk[u] = in ? keys[j + u] : 0ull;
            ix[u] = in ? idx[j + u] : 0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const bool in = j + u < end;
            r[u] = in ? rec[ix[u]] : make_float4(0.f, 0.f, 0.f, 0.f);
            q[u] = in ? recq[ix[u]] : 0.0;
            bv[u] = (in && b < B) ? double(basis[int64_t(kk[u] & rmask) * B + b]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (j + u >= end) break;
            a0 = __dadd_rn(a0, __dmul_rn(double(r[u].y), bv[u]));
            a1 = __dadd_rn(a1, __dmul_rn(double(r[u].z), bv[u]));
            a2 = __dadd_rn(a2, __dmul_rn(double(r[u].w), bv[u]));
            as = __dadd_rn(as, double(r[u].x));
            aq = __dadd_rn(aq, q[u]);
        }
    }
    if (b < B) {
        gsh[pid * S + 0 * B + b] = float(a0);
        gsh[pid * S + 1 * B + b] = float(a1);
        gsh[pid * S + 2 * B + b] = float(a2);
    }
    if (b == 0) {
        gsig[pid] = float(as);
        signal[pid] = aq;
    }
}

// ray_index must be a permutation of 0..n-1 (it indexes the per-ray arrays
// and orders the reduction): flag out-of-range or repeated entries.
__global__ void check_perm_kernel(const int64_t* __restrict__ idx, int64_t n, unsigned* __restrict__ seen,
                                  unsigned long long* __restrict__ bad) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t r = idx[i];
    if (r < 0 || r >= n || atomicExch(seen + r, 1u) != 0u) atomicAdd(bad, 1ull);
}

static int bits_for(int64_t v) {  // smallest k with v < 2^k (k >= 1)
    int k = 1;
    while (k < 62 && (int64_t(1) << k) <= v) ++k;
    return k;
}

static int64_t g_rec_hint = 0;  // records needed by the last call (grows only)

template <int B>
static int run_sorted(const TreeDev& T, int64_t capacity, const double* o, const double* d, const double* tgt,
                      const int64_t* ray_id, const int32_t* warp_order, uint16_t* ray_used, int64_t n, const double* bg, double eps, double tn,
                      double tf, double gs, float* gsig, float* gsh, double* signal,
                      uint8_t* touched, double* loss_sum, cudaStream_t s) {
    retain_pool_memory();
    const int ray_bits = bits_for(n - 1 < 1 ? 1 : n - 1);
    const int pid_bits = bits_for(capacity);
    if (ray_bits + pid_bits > 64)
        return set_error(DOT_BAD_ARG, "batch too large for the sorted reduction keys");
    int64_t cap = g_rec_hint > 16 * n ? g_rec_hint : 16 * n;
    if (cap < 64) cap = 64;
    int st = DOT_OK;
    unsigned long long* ctr = nullptr;
    float* basis = nullptr;
    double* loss_ray = nullptr;
    unsigned long long *keys = nullptr, *keys2 = nullptr;
    int32_t *idx = nullptr, *idx2 = nullptr;
    float4* rec = nullptr;
    double* recq = nullptr;
    void* tmp = nullptr;
    auto release_records = [&]() {
        cudaFreeAsync(keys, s);
        cudaFreeAsync(keys2, s);
        cudaFreeAsync(idx, s);
        cudaFreeAsync(idx2, s);
        cudaFreeAsync(rec, s);
        cudaFreeAsync(recq, s);
        keys = keys2 = nullptr;
        idx = idx2 = nullptr;
        rec = nullptr;
        recq = nullptr;
    };
    auto cleanup = [&]() {
        release_records();
        cudaFreeAsync(ctr, s);
        cudaFreeAsync(basis, s);
        cudaFreeAsync(loss_ray, s);
        cudaFreeAsync(tmp, s);
    };
#define TRY(x) do { if ((st = (x)) != DOT_OK) { cleanup(); return st; } } while (0)
#define ALLOC(p, bytes) TRY(check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&(p)), (bytes), s), "cudaMallocAsync"))
    ALLOC(ctr, 2 * sizeof(unsigned long long));
    ALLOC(basis, size_t(n) * B * sizeof(float));
    ALLOC(loss_ray, size_t(n) * sizeof(double));
    unsigned long long h_ctr[2] = {0, 0};
    if (ray_id) {
        unsigned* seen = nullptr;
        ALLOC(seen, size_t(n) * sizeof(unsigned));
        TRY(check_cuda(cudaMemsetAsync(seen, 0, size_t(n) * sizeof(unsigned), s), "memset"));
        TRY(check_cuda(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), s), "memset"));
        check_perm_kernel<<<unsigned((n + 255) / 256), 256, 0, s>>>(ray_id, n, seen, ctr);
        cudaFreeAsync(seen, s);
        TRY(check_cuda(cudaMemcpyAsync(h_ctr, ctr, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s), "memcpy"));
        TRY(check_cuda(cudaStreamSynchronize(s), "cudaStreamSynchronize"));
        if (h_ctr[0] != 0) TRY(set_error(DOT_BAD_ARG, "ray_index is not a permutation of 0..n-1"));
    }
    for (int attempt = 0; attempt < 3; ++attempt) {
        ALLOC(keys, size_t(cap) * sizeof(unsigned long long));
        ALLOC(rec, size_t(cap) * sizeof(float4));
        ALLOC(recq, size_t(cap) * sizeof(double));
        TRY(check_cuda(cudaMemsetAsync(ctr, 0, 2 * sizeof(unsigned long long), s), "memset"));
        EmitArgs ea{ctr, cap, keys, rec, recq, basis, loss_ray, ray_bits};
        TRY(launch_render_bwd_emit(T, o, d, tgt, ray_id, warp_order, ray_used, n, bg, eps, tn, tf, gs, touched,
                                   ea, s));
        TRY(check_cuda(cudaMemcpyAsync(h_ctr, ctr, sizeof(h_ctr), cudaMemcpyDeviceToHost, s), "memcpy"));
        TRY(check_cuda(cudaStreamSynchronize(s), "cudaStreamSynchronize"));
        if (int64_t(h_ctr[0]) > g_rec_hint) g_rec_hint = int64_t(h_ctr[0]);
        if (h_ctr[1] == 0) break;
        // some rays did not fit: nothing of theirs was written; retry with
        // room for every record (touched marks are idempotent, per-ray
        // losses are overwritten)
        release_records();
        cap = int64_t(h_ctr[0]) + 64;
        if (attempt == 2) TRY(set_error(DOT_CUDA_ERR, "sorted backward: record buffer overflow"));
    }
    const int64_t total = int64_t(h_ctr[0]);
    if (total > 0) {
        if (total > INT32_MAX) TRY(set_error(DOT_BAD_ARG, "too many segments for one sorted batch"));
        ALLOC(keys2, size_t(total) * sizeof(unsigned long long));
        ALLOC(idx, size_t(total) * sizeof(int32_t));
        ALLOC(idx2, size_t(total) * sizeof(int32_t));
        TRY(launch_iota(idx, total, s));
        size_t tmp_bytes = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys2, idx, idx2, int(total), 0,
                                        ray_bits + pid_bits, s);
        ALLOC(tmp, tmp_bytes);
        TRY(check_cuda(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys2, idx, idx2, int(total), 0,
                                                       ray_bits + pid_bits, s), "DeviceRadixSort"));
        // runs of equal leaf, longest first
        int32_t *flag = nullptr, *heads = nullptr, *heads2 = nullptr, *d_nruns = nullptr;
        uint32_t *lkey = nullptr, *lkey2 = nullptr;
        void* tmp2 = nullptr;
        auto free_runs = [&]() {
            cudaFreeAsync(flag, s);
            cudaFreeAsync(heads, s);
            cudaFreeAsync(heads2, s);
            cudaFreeAsync(d_nruns, s);
            cudaFreeAsync(lkey, s);
            cudaFreeAsync(lkey2, s);
            cudaFreeAsync(tmp2, s);
        };
#define TRY2(x) do { if ((st = (x)) != DOT_OK) { free_runs(); cleanup(); return st; } } while (0)
#define ALLOC2(p, bytes) TRY2(check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&(p)), (bytes), s), "cudaMallocAsync"))
        ALLOC2(flag, size_t(total) * sizeof(int32_t));
        ALLOC2(heads, size_t(total) * sizeof(int32_t));
        ALLOC2(heads2, size_t(total) * sizeof(int32_t));
        ALLOC2(d_nruns, sizeof(int32_t));
        ALLOC2(lkey, size_t(total) * sizeof(uint32_t));
        ALLOC2(lkey2, size_t(total) * sizeof(uint32_t));
        run_heads_kernel<<<unsigned((total + 255) / 256), 256, 0, s>>>(keys2, total, ray_bits, flag);
        size_t b1 = 0, b2 = 0;
        thrust::counting_iterator<int32_t> pos(0);
        cub::DeviceSelect::Flagged(nullptr, b1, pos, flag, heads, d_nruns, int(total), s);
        cub::DeviceRadixSort::SortPairs(nullptr, b2, lkey, lkey2, heads, heads2, int(total), 0, 32, s);
        ALLOC2(tmp2, b1 > b2 ? b1 : b2);
        TRY2(check_cuda(cub::DeviceSelect::Flagged(tmp2, b1, pos, flag, heads, d_nruns, int(total), s),
                        "DeviceSelect"));
        int32_t n_runs = 0;
        TRY2(check_cuda(cudaMemcpyAsync(&n_runs, d_nruns, sizeof(n_runs), cudaMemcpyDeviceToHost, s), "memcpy"));
        TRY2(check_cuda(cudaStreamSynchronize(s), "sync"));
        run_lengths_kernel<<<unsigned((n_runs + 255) / 256), 256, 0, s>>>(heads, d_nruns, total, lkey);
        TRY2(check_cuda(cub::DeviceRadixSort::SortPairs(tmp2, b2, lkey, lkey2, heads, heads2, n_runs, 0, 32, s),
                        "DeviceRadixSort"));
        reduce_runs_kernel<B><<<unsigned((int64_t(n_runs) * 16 + 127) / 128), 128, 0, s>>>(
            keys2, idx2, heads2, lkey2, d_nruns, ray_bits, rec, recq, basis, gsig, gsh, signal);
        st = check_launch("reduce_runs_kernel");
        free_runs();
        if (st != DOT_OK) {
            cleanup();
            return st;
        }
#undef TRY2
#undef ALLOC2
    }
    {
        // loss_sum += sum of per-ray squared errors (fixed reduction order)
        double* part = nullptr;
        ALLOC(part, sizeof(double));
        size_t red_bytes = 0;
        cub::DeviceReduce::Sum(nullptr, red_bytes, loss_ray, part, int(n), s);
        void* rtmp = nullptr;
        if ((st = check_cuda(cudaMallocAsync(&rtmp, red_bytes, s), "cudaMallocAsync")) == DOT_OK) {
            st = check_cuda(cub::DeviceReduce::Sum(rtmp, red_bytes, loss_ray, part, int(n), s), "DeviceReduce");
            if (st == DOT_OK) st = launch_add_f64(loss_sum, part, s);
        }
        cudaFreeAsync(rtmp, s);
        cudaFreeAsync(part, s);
        if (st != DOT_OK) {
            cleanup();
            return st;
        }
    }
    cleanup();
#undef ALLOC
#undef TRY
    return DOT_OK;
}

__global__ void iota_kernel(int32_t* p, int64_t n) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) p[i] = int32_t(i);
}

__global__ void add_f64_kernel(double* dst, const double* src) { dst[0] += src[0]; }

int launch_iota(int32_t* p, int64_t n, cudaStream_t s) {
    iota_kernel<<<unsigned((n + 255) / 256), 256, 0, s>>>(p, n);
    return check_launch("iota_kernel");
}

int launch_add_f64(double* dst, const double* src, cudaStream_t s) {
    add_f64_kernel<<<1, 1, 0, s>>>(dst, src);
    return check_launch("add_f64_kernel");
}

// ---------------------------------------------------------------------------
// Batch coherence order: one radix sort of the 31-bit keys (dot_ray_keys32)
// carrying the caller's ray index (or the batch position) as the value, so
// the sorted values are directly the kernel's ray_index (no gather after).

__global__ void iota64_kernel(int64_t* __restrict__ v, int64_t n) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) v[i] = i;
}

int run_plan_sort(const int32_t* keys, const int64_t* ray_index, int64_t n, int begin_bit,
                  int32_t* sorted_keys, int64_t* sorted_index, cudaStream_t s) {
    if (n == 0) return DOT_OK;
    retain_pool_memory();
    int64_t* iota = nullptr;
    const int64_t* vin = ray_index;
    int st = DOT_OK;
    if (!vin) {
        if ((st = check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&iota), size_t(n) * 8, s), "cudaMallocAsync")))
            return st;
        iota64_kernel<<<unsigned((n + 255) / 256), 256, 0, s>>>(iota, n);
        vin = iota;
    }
    size_t bytes = 0;
    void* tmp = nullptr;
    st = check_cuda(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys, sorted_keys, vin, sorted_index, n,
                                                    begin_bit, 31, s), "SortPairs");
    if (st == DOT_OK) st = check_cuda(cudaMallocAsync(&tmp, bytes, s), "cudaMallocAsync");
    if (st == DOT_OK)
        st = check_cuda(cub::DeviceRadixSort::SortPairs(tmp, bytes, keys, sorted_keys, vin, sorted_index, n,
                                                        begin_bit, 31, s), "SortPairs");
    if (tmp) cudaFreeAsync(tmp, s);
    if (iota) cudaFreeAsync(iota, s);
    if (st != DOT_OK) return st;
    return check_launch("plan_sort");
}

}  // namespace dot

using namespace dot;

extern "C" int dot_render_bwd_sorted(const dot_tree_view* tree, const double* origins, const double* dirs,
                                     const double* targets, const int64_t* ray_index,
                                     const int32_t* warp_order, uint16_t* ray_used, int64_t n_rays,
                                     const double* background, double early_stop_eps, double t_near,
                                     double t_far, double grad_scale, float* grad_sigma, float* grad_sh,
                                     int32_t gsh_stride, double* signal, uint8_t* touched,
                                     double* loss_sum, void* stream) {
    if (int st = validate_tree_view(tree)) return st;
    if (n_rays < 0 || (n_rays && (!origins || !dirs || !targets)) || !background)
        return set_error(DOT_BAD_ARG, "bad ray arrays");
    if (!grad_sigma || !grad_sh || !signal || !touched || !loss_sum)
        return set_error(DOT_BAD_ARG, "gradient / signal outputs must not be NULL");
    if (gsh_stride != tree->sh_stride)
        return set_error(DOT_BAD_ARG, "gsh_stride must equal sh_stride (%d)", tree->sh_stride);
    if (n_rays == 0) return DOT_OK;
    const TreeDev T = make_tree(*tree);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    switch (T.basis_count) {
        case 1: return run_sorted<1>(T, tree->capacity, origins, dirs, targets, ray_index, warp_order, ray_used, n_rays, background, early_stop_eps, t_near, t_far, grad_scale, grad_sigma, grad_sh, signal, touched, loss_sum, s);
        case 4: return run_sorted<4>(T, tree->capacity, origins, dirs, targets, ray_index, warp_order, ray_used, n_rays, background, early_stop_eps, t_near, t_far, grad_scale, grad_sigma, grad_sh, signal, touched, loss_sum, s);
        case 9: return run_sorted<9>(T, tree->capacity, origins, dirs, targets, ray_index, warp_order, ray_used, n_rays, background, early_stop_eps, t_near, t_far, grad_scale, grad_sigma, grad_sh, signal, touched, loss_sum, s);
        case 16: return run_sorted<16>(T, tree->capacity, origins, dirs, targets, ray_index, warp_order, ray_used, n_rays, background, early_stop_eps, t_near, t_far, grad_scale, grad_sigma, grad_sh, signal, touched, loss_sum, s);
        default: return set_error(DOT_BAD_ARG, "basis_count must be 1, 4, 9 or 16");
    }
}
