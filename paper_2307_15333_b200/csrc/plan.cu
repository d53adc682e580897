// plan.cu -- batch coherence order from a ranked ray pool, without a sort.
//
// A resident ray pool is ranked once by its 62-bit coherence keys
// (dot_ray_keys: origin Morton 3 x 10 bits, octahedral direction 2 x 16
// bits): rank[ray] = its position in key order, order[position] = the ray.
// A batch of distinct pool rays (an epoch permutation slice, optim.py:141-146
// of the reference) is then put in key order by a one-bit-per-position
// counting sort: every ray sets its rank's bit in a pool-sized bitmap, a
// scan of the bitmap's popcounts gives each set bit its output slot, and the
// slot receives order[position].  Per batch that is one random 4-byte rank
// read and one bit RED per ray, two streaming passes over n_pool / 8 bytes
// and one random 4-byte order read per ray -- against the keys gather plus
// four radix passes over (key, index) pairs of dot_plan_sort.
//
// Rays the bitmap cannot place -- a repeated ray (its bit is already set) or
// an index outside [0, n_pool) -- are appended after the placed ones in
// arrival order, so the output is always a permutation of the batch and the
// backward still sees (and reports) invalid indices.  The bitmap is left
// all-zero for the next batch (the place pass clears the words it reads).
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "dot_internal.h"

namespace dot {

constexpr int kPlanThreads = 256;
constexpr int kPlanWords = 8;                               // bitmap words per thread
constexpr int64_t kPlanBlockWords = kPlanThreads * kPlanWords;  // 2048 words = 65536 pool positions per block

struct PlanWs {
    uint32_t* bitmap;            // [words]
    int32_t* block_base;         // [blocks + 1]
    unsigned long long* extra;   // [1] rays appended after the placed ones
    int64_t* extra_ray;          // [n] those rays, in arrival order (slots are racy; order is not part of the contract)
};

static int64_t plan_words(int64_t n_pool) { return (n_pool + 31) / 32; }
static int64_t plan_blocks(int64_t n_pool) { return (plan_words(n_pool) + kPlanBlockWords - 1) / kPlanBlockWords; }

static size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

static PlanWs carve(void* ws, int64_t n_pool) {
    char* p = static_cast<char*>(ws);
    PlanWs w;
    w.bitmap = reinterpret_cast<uint32_t*>(p);
    p += align256(size_t(plan_words(n_pool)) * 4);
    w.block_base = reinterpret_cast<int32_t*>(p);
    p += align256(size_t(plan_blocks(n_pool) + 1) * 4);
    w.extra = reinterpret_cast<unsigned long long*>(p);
    p += 256;
    w.extra_ray = reinterpret_cast<int64_t*>(p);
    return w;
}

__global__ void __launch_bounds__(256) plan_mark_kernel(const int32_t* __restrict__ rank, int64_t n_pool,
                                                        const int64_t* __restrict__ ray_idx, int64_t n, PlanWs w) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t r = __ldg(ray_idx + i);
    bool placed = false;
    if (r >= 0 && r < n_pool) {
        const int64_t k = rank ? int64_t(__ldg(rank + r)) : r;  // NULL: the pool is stored in key order
        if (k >= 0 && k < n_pool) {  // a damaged rank entry is appended, never written out of bounds
            const uint32_t bit = 1u << (uint32_t(k) & 31u);
            placed = (atomicOr(w.bitmap + (uint32_t(k) >> 5), bit) & bit) == 0u;
        }
    }
    if (!placed) w.extra_ray[atomicAdd(w.extra, 1ull)] = r;
}

// per block of 2048 bitmap words: the number of set bits
__global__ void __launch_bounds__(kPlanThreads) plan_count_kernel(int64_t words, PlanWs w) {
    using Reduce = cub::BlockReduce<int, kPlanThreads>;
    __shared__ typename Reduce::TempStorage tmp;
    const int64_t w0 = int64_t(blockIdx.x) * kPlanBlockWords + int64_t(threadIdx.x) * kPlanWords;
    int c = 0;
    if (w0 + kPlanWords <= words) {
        const uint4 a = *reinterpret_cast<const uint4*>(w.bitmap + w0);
        const uint4 b = *reinterpret_cast<const uint4*>(w.bitmap + w0 + 4);
        c = __popc(a.x) + __popc(a.y) + __popc(a.z) + __popc(a.w) + __popc(b.x) + __popc(b.y) + __popc(b.z) +
            __popc(b.w);
    } else {
        for (int64_t k = w0; k < words && k < w0 + kPlanWords; ++k) c += __popc(w.bitmap[k]);
    }
    const int total = Reduce(tmp).Sum(c);
    if (threadIdx.x == 0) w.block_base[blockIdx.x] = total;
}

// exclusive scan of the block counts (one block; blocks <= 2^26 / 2048 = 32768)
__global__ void __launch_bounds__(1024) plan_scan_kernel(int64_t blocks, PlanWs w) {
    using Scan = cub::BlockScan<int, 1024>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ int carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t base = 0; base <= blocks; base += 1024) {
        const int64_t i = base + threadIdx.x;
        const int v = i < blocks ? w.block_base[i] : 0;
        int ex, agg;
        Scan(tmp).ExclusiveSum(v, ex, agg);
        if (i <= blocks) w.block_base[i] = carry + ex;  // [blocks] = total placed
        __syncthreads();
        if (threadIdx.x == 0) carry += agg;
        __syncthreads();
    }
}

// each set bit's slot = block base + exclusive count inside the block; the
// slot receives the key position, then (order != NULL) the pool ray at that
// position; the words are cleared.  The appended rays go after the placed
// ones.
__global__ void __launch_bounds__(kPlanThreads) plan_place_kernel(const int32_t* __restrict__ order, int64_t words,
                                                                  int64_t blocks, int64_t n, PlanWs w,
                                                                  int64_t* __restrict__ out) {
    using Scan = cub::BlockScan<int, kPlanThreads>;
    __shared__ typename Scan::TempStorage tmp;
    const int64_t w0 = int64_t(blockIdx.x) * kPlanBlockWords + int64_t(threadIdx.x) * kPlanWords;
    uint32_t m[kPlanWords];
    int c = 0;
#pragma unroll
    for (int k = 0; k < kPlanWords; ++k) {
        m[k] = (w0 + k < words) ? w.bitmap[w0 + k] : 0u;
        c += __popc(m[k]);
    }
    int ex;
    Scan(tmp).ExclusiveSum(c, ex);
    int64_t slot = int64_t(w.block_base[blockIdx.x]) + ex;
#pragma unroll
    for (int k = 0; k < kPlanWords; ++k) {
        if (m[k] == 0u) continue;
        w.bitmap[w0 + k] = 0u;
        const int64_t pos0 = (w0 + k) * 32;
        for (uint32_t b = m[k]; b; b &= b - 1u) out[slot++] = pos0 + (__ffs(b) - 1);
    }
    if (order) {
        // key positions -> pool rays: the block's slots, four independent
        // gathers in flight per thread (not one dependent chain per set bit)
        __syncthreads();
        const int64_t b0 = w.block_base[blockIdx.x], b1 = w.block_base[blockIdx.x + 1];
        for (int64_t i = b0 + threadIdx.x; i < b1; i += 4 * kPlanThreads) {
            int64_t pos[4];
            int32_t ray[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t j = i + u * kPlanThreads;
                pos[u] = j < b1 ? out[j] : -1;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) ray[u] = pos[u] >= 0 ? __ldg(order + pos[u]) : 0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t j = i + u * kPlanThreads;
                if (j < b1) out[j] = ray[u];
            }
        }
    }
    // the appended rays: grid-stride over the (usually empty) tail
    const int64_t placed = w.block_base[blocks];
    const int64_t extra = int64_t(*w.extra);
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < extra && placed + i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        out[placed + i] = w.extra_ray[i];
}

size_t plan_ranked_workspace(int64_t n_pool, int64_t n) {
    return align256(size_t(plan_words(n_pool)) * 4) + align256(size_t(plan_blocks(n_pool) + 1) * 4) + 256 +
           align256(size_t(n) * 8);
}

int run_plan_ranked(const int32_t* rank, const int32_t* order, int64_t n_pool, const int64_t* ray_idx, int64_t n,
                    void* ws, int64_t* out, cudaStream_t s) {
    if (n == 0) return DOT_OK;
    PlanWs w = carve(ws, n_pool);
    const int64_t words = plan_words(n_pool), blocks = plan_blocks(n_pool);
    if (int st = check_cuda(cudaMemsetAsync(w.extra, 0, 8, s), "cudaMemsetAsync")) return st;
    plan_mark_kernel<<<unsigned((n + 255) / 256), 256, 0, s>>>(rank, n_pool, ray_idx, n, w);
    plan_count_kernel<<<unsigned(blocks), kPlanThreads, 0, s>>>(words, w);
    plan_scan_kernel<<<1, 1024, 0, s>>>(blocks, w);
    plan_place_kernel<<<unsigned(blocks), kPlanThreads, 0, s>>>(order, words, blocks, n, w, out);
    return check_launch("plan_ranked");
}

}  // namespace dot
