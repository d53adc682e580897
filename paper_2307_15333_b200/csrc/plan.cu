// plan.cu -- batch coherence order from a ranked ray pool, without a sort,
// in ONE cooperative launch.
//
// A ray pool (resident, or a host dataset whose rays arrive in batches) is
// ranked once by its 62-bit coherence keys (dot_ray_keys: origin Morton
// 3 x 10 bits, octahedral direction 2 x 16 bits): rank[ray] = its position
// in key order, order[position] = the ray.  A batch of distinct pool rays
// (an epoch permutation slice, optim.py:141-146 of the reference) is then
// put in key order by a one-bit-per-position counting sort: every ray sets
// its position's bit in a pool-sized bitmap, a scan of the bitmap's
// popcounts gives each set bit its output slot.  Per batch: one bit RED and
// one tag store per ray, two streaming passes over n_pool / 8 bytes and one
// gather per ray -- against a keys gather plus four radix passes over
// (key, index) pairs (dot_plan_sort).  What a slot receives:
//   DOT_PLAN_POSITIONS  the key position (a pool stored in key order: the ray)
//   DOT_PLAN_POOL_RAYS  order[position] (a pool left in its own order)
//   DOT_PLAN_SLOTS      the batch slot i whose ray sits at that position (a
//                       staged batch: ray_index[i] is the ray's dataset id,
//                       the backward reads the batch arrays by slot)
// With a per-ray cost column the same launch also builds the backward's warp
// launch order (chunks of warps by descending max cost, as
// dot_sched_order_costs): the costs of the placed rays are max-reduced per
// output warp, histogrammed, scanned and scattered.
//
// Why one skinny launch: the plan of step k+1 is queued behind step k's
// backward and must finish under step k's optimizer update.  A chain of
// small kernels queued behind the update's 140k blocks and ran serialised
// after it (~50-90 us per step, tools/step_gaps.py).  One cooperative grid
// of a 64-thread block per SM at <= 64 registers (4096 registers: what the
// update's five 256-thread blocks leave free) becomes resident beside the
// update.  Beside a bandwidth-bound kernel every random access costs ~4x
// its idle latency (tools/plan_phases.py), so the kernel is written for
// memory-level parallelism: fire-and-forget REDs / stores where a return
// value is not needed, 8 gathers in flight per thread, per-warp bitmap
// ranges (no block barriers), one gather per placed ray in slot mode (the
// slot and its cost packed in the position's tag, the only per-ray store).
//
// Rays the bitmap cannot place -- a repeated ray (another lane won its
// position's tag) or an index outside [0, n_pool) -- follow the placed
// ones, so the output is always a permutation of the batch and the backward
// still sees (and reports) invalid indices.  Repeats are detected from the
// placed count (a second pass over the batch runs only then).  The workspace is left
// reusable (bitmap, warp costs, histogram and counters zero).
#include <cooperative_groups.h>

#include "dot_internal.h"

namespace cg = cooperative_groups;

namespace dot {

constexpr int kPlanThreads = 64;                   // 2 warps per block, one block per SM
constexpr int kPlanMinBlocks = 16;                 // -> <= 64 registers per thread
constexpr int kPlanWarps = kPlanThreads / 32;
constexpr int kPlanLaneWords = 16;                 // bitmap words per lane per range (4 x uint4)
constexpr int64_t kPlanRangeWords = 32 * kPlanLaneWords;  // 512 words = 16384 pool positions per warp range
constexpr int kPlanCostBins = 1024;                // warp costs are capped here
constexpr int kPlanIlp = 8;                        // rays / gathers in flight per thread
constexpr int kTagSlotBits = 21;                   // packed tag: slot | cost << 21 (n <= 2^21)
constexpr int kPlanStage = 512;                    // staged positions per warp range (shared memory, 4 KB per block)
#ifndef DOT_PLAN_WINDOW
#define DOT_PLAN_WINDOW 128
#endif
constexpr int kPlanWindow = DOT_PLAN_WINDOW;       // rays regrouped by cost per window (32..256, a multiple of 32)

struct PlanWs {
    uint32_t* bitmap;             // [words + slack]
    int32_t* warp_total;          // [total warps] set bits in each warp's ranges
    unsigned long long* ctr;      // [0] appended rays, [1] invalid (unplaceable) rays
    int64_t* extra_ray;           // [n] appended rays (slots in slot mode), in arrival order
    uint32_t* warp_cost;          // [ceil(n / 32)] max cost of each output warp
    uint16_t* chunk_cost;         // [ceil(n / 32)]
    uint16_t* slot_cost;          // [n] the placed ray's cost per output slot
    int32_t* hist;                // [kPlanCostBins] chunks per cost bin, then their start chunks
    int32_t* tag;                 // [n_pool] slot mode: each marked position's slot (| cost << 21 when packed)
    uint32_t* claim;              // [words] repeated rays outside slot mode: first claimant per position
};

__host__ __device__ static int64_t plan_words(int64_t n_pool) { return (n_pool + 31) / 32; }
static size_t align256(size_t b) { return (b + 255) & ~size_t(255); }
static int g_plan_grid = 0;  // blocks of the cooperative launch (one per SM), set on first use

// Workspace layout: the regions that must stay zero between calls (bitmap,
// claim bitmap, counters, histogram) and the pool-sized tag come first, at
// offsets that depend only on n_pool, so one workspace sized for the
// largest batch serves every smaller one; the per-batch scratch follows.
static size_t carve(void* ws, int64_t n_pool, int64_t n, PlanWs* out) {
    char* base = static_cast<char*>(ws);
    char* p = base;
    PlanWs w;
    const int64_t nw = (n + 31) / 32;
    w.bitmap = reinterpret_cast<uint32_t*>(p);
    p += align256(size_t(plan_words(n_pool) + 32 * kPlanLaneWords) * 4);  // + a zero slack range (whole uint4 loads)
    w.claim = reinterpret_cast<uint32_t*>(p);
    p += align256(size_t(plan_words(n_pool)) * 4);
    w.warp_total = reinterpret_cast<int32_t*>(p);
    p += align256(size_t(4096) * 4);  // up to 2048 SMs x 2 warps
    w.ctr = reinterpret_cast<unsigned long long*>(p);
    p += 256;
    w.hist = reinterpret_cast<int32_t*>(p);
    p += align256(size_t(kPlanCostBins) * 4);
    w.tag = reinterpret_cast<int32_t*>(p);
    p += align256(size_t(n_pool) * 4);
    // per batch: written before read in every call
    w.extra_ray = reinterpret_cast<int64_t*>(p);
    p += align256(size_t(n) * 8);
    w.warp_cost = reinterpret_cast<uint32_t*>(p);
    p += align256(size_t(nw) * 4);
    w.chunk_cost = reinterpret_cast<uint16_t*>(p);
    p += align256(size_t(nw) * 2);
    w.slot_cost = reinterpret_cast<uint16_t*>(p);
    p += align256(size_t(n) * 2);
    if (out) *out = w;
    return size_t(p - base);
}

struct PlanArgs {
    const int32_t* rank;     // NULL: ray_index values are key positions
    const int32_t* order;    // DOT_PLAN_POOL_RAYS
    const int64_t* ray_idx;  // [n]
    const uint16_t* cost;    // indexed by the output value; NULL: no warp order
    int32_t* warp_order;
    int64_t* out;
    int64_t n_pool, n;
    int mode, chunk;
    int packed;              // slot mode with costs and n <= 2^21: the tag carries the cost
};

#ifdef DOT_DIAG_FLAGS
// diagnostic builds only: %globaltimer at the kernel start and after each
// phase (block 0, thread 0), read with dot_diag_plan_timeline
__device__ unsigned long long g_plan_t[16];
#define PLAN_STAMP(i)                                                               \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                                      \
        unsigned long long t_;                                                      \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                     \
        g_plan_t[i] = t_;                                                           \
    }
extern "C" int dot_diag_plan_timeline(unsigned long long* out) {
    return cudaMemcpyFromSymbol(out, g_plan_t, sizeof(g_plan_t)) == cudaSuccess ? 0 : 3;
}
#else
#define PLAN_STAMP(i)
#endif

__device__ __forceinline__ void red_or(uint32_t* p, uint32_t v) {
    asm volatile("red.global.or.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// the key position of ray r, -1 when it cannot be placed
__device__ __forceinline__ int64_t plan_key(const PlanArgs& a, int64_t r) {
    if (r < 0 || r >= a.n_pool) return -1;
    const int64_t k = a.rank ? int64_t(__ldg(a.rank + r)) : r;
    return (k >= 0 && k < a.n_pool) ? k : -1;  // a damaged rank entry is appended, never written out of bounds
}

__device__ __forceinline__ void plan_append(PlanWs& w, int64_t v) { w.extra_ray[atomicAdd(w.ctr, 1ull)] = v; }

__device__ __forceinline__ uint32_t cap_cost(uint32_t c) { return min(c, uint32_t(kPlanCostBins - 1)); }

// log-scale cost bucket, three per octave, integer-exact: x = cost + 1 in
// [2^m, 2^(m+1)) -> 3m + floor(3x / 2^m) - 3, in [0, 30] for costs <= 1023
__host__ __device__ __forceinline__ int cost_bucket(uint32_t cost) {
    const uint32_t x = cost + 1u;
    const int m = 31 - __builtin_clz(x);
    return 3 * m + int((3u * x) >> m) - 3;
}

// the values (pool rays / slots) and costs of U placed key positions
// (val[u] < 0: none), all gathers of a kind in flight together
template <int U>
__device__ __forceinline__ void plan_values(const PlanArgs& a, const PlanWs& w, int32_t (&val)[U],
                                            uint32_t (&cc)[U], int64_t n_cost) {
    if (a.mode == DOT_PLAN_POOL_RAYS) {
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (val[u] >= 0) val[u] = __ldg(a.order + val[u]);
    } else if (a.mode == DOT_PLAN_SLOTS) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (val[u] < 0) continue;
            const uint32_t t = uint32_t(w.tag[val[u]]);
            val[u] = a.packed ? int32_t(t & ((1u << kTagSlotBits) - 1u)) : int32_t(t);
            cc[u] = a.packed ? (t >> kTagSlotBits) : 0u;
        }
    }
    if (a.cost && !a.packed) {
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (val[u] >= 0 && val[u] < n_cost) cc[u] = cap_cost(__ldg(a.cost + val[u]));
    }
}

__global__ void __launch_bounds__(kPlanThreads, kPlanMinBlocks) plan_coop_kernel(PlanArgs a, PlanWs w) {
    cg::grid_group grid = cg::this_grid();
    __shared__ int32_t s_stage[kPlanWarps][kPlanStage];
    const int lane = threadIdx.x & 31;
    const int64_t gt = int64_t(blockIdx.x) * kPlanThreads + threadIdx.x;
    const int64_t GT = int64_t(gridDim.x) * kPlanThreads;
    const int64_t gwarp = int64_t(blockIdx.x) * kPlanWarps + (threadIdx.x >> 5);
    const int64_t n_gwarps = int64_t(gridDim.x) * kPlanWarps;
    const int64_t words = plan_words(a.n_pool);
    const int64_t ranges = (words + kPlanRangeWords - 1) / kPlanRangeWords;
    const int64_t per_warp = (ranges + n_gwarps - 1) / n_gwarps;  // contiguous ranges per warp
    const int64_t q0 = gwarp * per_warp, q1 = min(ranges, (gwarp + 1) * per_warp);
    const int64_t nw = (a.n + 31) / 32;
    const int64_t n_cost = a.mode == DOT_PLAN_SLOTS ? a.n : a.n_pool;  // the cost column's length
    PLAN_STAMP(0)

    // A. mark: a bit RED per ray (and, in slot mode, the position's tag),
    // kPlanIlp rays in flight per thread
    for (int64_t i0 = gt; i0 < a.n; i0 += kPlanIlp * GT) {
        int64_t r[kPlanIlp];
        int32_t k[kPlanIlp];  // key position; -1 unplaceable, -2 past the batch
#pragma unroll
        for (int u = 0; u < kPlanIlp; ++u) {
            const int64_t i = i0 + u * GT;
            r[u] = i < a.n ? __ldg(a.ray_idx + i) : 0;
        }
#pragma unroll
        for (int u = 0; u < kPlanIlp; ++u) k[u] = i0 + u * GT < a.n ? int32_t(plan_key(a, r[u])) : -2;
        uint32_t cst[kPlanIlp];
#pragma unroll
        for (int u = 0; u < kPlanIlp; ++u) {
            const int64_t i = i0 + u * GT;
            cst[u] = (a.packed && i < a.n) ? cap_cost(__ldg(a.cost + i)) : 0u;
        }
#pragma unroll
        for (int u = 0; u < kPlanIlp; ++u) {
            const int64_t i = i0 + u * GT;
            if (k[u] == -2) continue;
            if (k[u] < 0) {  // unplaceable: appended as is (slot, or the caller's index)
                atomicAdd(w.ctr + 1, 1ull);
                plan_append(w, a.mode == DOT_PLAN_SLOTS ? i : r[u]);
                continue;
            }
            red_or(w.bitmap + (uint32_t(k[u]) >> 5), 1u << (uint32_t(k[u]) & 31u));
            if (a.mode == DOT_PLAN_SLOTS)  // the position's slot (and cost): the only per-ray write
                w.tag[k[u]] = int32_t(a.packed ? (uint32_t(i) | (cst[u] << kTagSlotBits)) : uint32_t(i));
        }
    }
    grid.sync();
    PLAN_STAMP(1)

    // B. set bits of each warp's contiguous ranges (16 words per lane)
    {
        int tot = 0;
        for (int64_t q = q0; q < q1; ++q) {
            const uint4* p = reinterpret_cast<const uint4*>(w.bitmap + q * kPlanRangeWords +
                                                            int64_t(lane) * kPlanLaneWords);
            const uint4 x0 = p[0], x1 = p[1], x2 = p[2], x3 = p[3];  // words past the end: zero slack
            tot += __popc(x0.x) + __popc(x0.y) + __popc(x0.z) + __popc(x0.w) + __popc(x1.x) + __popc(x1.y) +
                   __popc(x1.z) + __popc(x1.w) + __popc(x2.x) + __popc(x2.y) + __popc(x2.z) + __popc(x2.w) +
                   __popc(x3.x) + __popc(x3.y) + __popc(x3.z) + __popc(x3.w);
        }
        tot = __reduce_add_sync(0xffffffffu, tot);
        if (lane == 0) w.warp_total[gwarp] = tot;
    }
    grid.sync();
    PLAN_STAMP(2)

    // C. placed total and this warp's base (every warp sums the totals itself)
    int64_t base = 0, placed = 0;
    for (int64_t v = lane; v < n_gwarps; v += 32) {
        const int t = w.warp_total[v];
        placed += t;
        if (v < gwarp) base += t;
    }
    for (int off = 16; off > 0; off >>= 1) {
        base += __shfl_xor_sync(0xffffffffu, base, off);
        placed += __shfl_xor_sync(0xffffffffu, placed, off);
    }
    const int64_t invalid = int64_t(w.ctr[1]);
    if (placed + invalid < a.n) {
        // repeated rays (grid-uniform branch, rare): one ray per position is
        // placed -- in slot mode the one whose slot the tag holds, otherwise
        // the first to claim the position in a second bitmap (cleared after)
        // -- and the others follow the placed rays
        for (int64_t i = gt; i < a.n; i += GT) {
            const int64_t r = __ldg(a.ray_idx + i);
            const int64_t k = plan_key(a, r);
            if (k < 0) continue;
            bool mine;
            if (a.mode == DOT_PLAN_SLOTS) {
                const uint32_t t = uint32_t(w.tag[k]);
                mine = (a.packed ? int64_t(t & ((1u << kTagSlotBits) - 1u)) : int64_t(t)) == i;
            } else {
                const uint32_t bit = 1u << (uint32_t(k) & 31u);
                mine = (atomicOr(w.claim + (k >> 5), bit) & bit) == 0u;
            }
            // a repeat keeps the output's meaning: its slot, its key
            // position, or the pool ray itself
            if (!mine) plan_append(w, a.mode == DOT_PLAN_SLOTS ? i : (a.mode == DOT_PLAN_POSITIONS ? k : r));
        }
        grid.sync();
        if (a.mode != DOT_PLAN_SLOTS)
            for (int64_t i = gt; i < a.n; i += GT) {
                const int64_t k = plan_key(a, __ldg(a.ray_idx + i));
                if (k >= 0) w.claim[k >> 5] = 0u;
            }
    }
    PLAN_STAMP(3)

    // D. place each warp's ranges: slots by a warp scan of the lanes' bit
    // counts; the range's positions staged in shared memory, then walked by
    // the whole warp with kPlanIlp gathers in flight per lane (coalesced
    // output); the words cleared.  A range with more set bits than the stage
    // holds (a batch denser than 1/16 of the pool) is placed lane by lane.
    {
        int32_t* stage = s_stage[threadIdx.x >> 5];
        int64_t slot_base = base;
        for (int64_t q = q0; q < q1; ++q) {
            const int64_t w0 = q * kPlanRangeWords + int64_t(lane) * kPlanLaneWords;
            uint4* p = reinterpret_cast<uint4*>(w.bitmap + w0);
            uint32_t m[kPlanLaneWords];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint4 x = p[j];
                m[4 * j] = x.x;
                m[4 * j + 1] = x.y;
                m[4 * j + 2] = x.z;
                m[4 * j + 3] = x.w;
            }
            int c = 0;
#pragma unroll
            for (int j = 0; j < kPlanLaneWords; ++j) c += __popc(m[j]);
            int incl = c;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, off);
                if (lane >= off) incl += y;
            }
            const int total = __shfl_sync(0xffffffffu, incl, 31);
            if (total == 0) continue;
            if (c) {
#pragma unroll
                for (int j = 0; j < 4; ++j) p[j] = make_uint4(0u, 0u, 0u, 0u);
            }
            if (total <= kPlanStage) {
                int o = incl - c;
#pragma unroll
                for (int j = 0; j < kPlanLaneWords; ++j)
                    for (uint32_t bits = m[j]; bits; bits &= bits - 1u)
                        stage[o++] = int32_t((w0 + j) * 32 + (__ffs(bits) - 1));
                __syncwarp();
                for (int e0 = 0; e0 < total; e0 += 32 * kPlanIlp) {
                    int32_t val[kPlanIlp];  // positions, rays and slots are < 2^31 (checked at the ABI)
                    uint32_t cc[kPlanIlp];
#pragma unroll
                    for (int u = 0; u < kPlanIlp; ++u) {
                        const int e = e0 + u * 32 + lane;
                        val[u] = e < total ? stage[e] : -1;
                        cc[u] = 0u;
                    }
                    plan_values<kPlanIlp>(a, w, val, cc, n_cost);
#pragma unroll
                    for (int u = 0; u < kPlanIlp; ++u) {
                        const int e = e0 + u * 32 + lane;
                        if (e0 + u * 32 >= total) break;  // warp-uniform
                        if (e < total) {
                            a.out[slot_base + e] = int64_t(val[u]);
                            if (a.cost) w.slot_cost[slot_base + e] = uint16_t(cc[u]);
                        }
                    }
                }
                __syncwarp();
            } else {
                int64_t slot = slot_base + (incl - c);
#pragma unroll
                for (int j = 0; j < kPlanLaneWords; ++j)
                    for (uint32_t bits = m[j]; bits; bits &= bits - 1u) {
                        int32_t val[1] = {int32_t((w0 + j) * 32 + (__ffs(bits) - 1))};
                        uint32_t cc[1] = {0u};
                        plan_values<1>(a, w, val, cc, n_cost);
                        a.out[slot] = int64_t(val[0]);
                        if (a.cost) w.slot_cost[slot] = uint16_t(cc[0]);
                        ++slot;
                    }
            }
            slot_base += total;
        }
    }
    // the appended rays, after the placed ones
    const int64_t extra = int64_t(w.ctr[0]);
    for (int64_t e = gt; e < extra && placed + e < a.n; e += GT) {
        const int64_t v = w.extra_ray[e];
        a.out[placed + e] = v;
        if (a.cost) w.slot_cost[placed + e] = uint16_t(v >= 0 && v < n_cost ? cap_cost(__ldg(a.cost + v)) : 0u);
    }
    grid.sync();
    PLAN_STAMP(4)
    if (gt == 0) {  // every thread has read the counters
        w.ctr[0] = 0ull;
        w.ctr[1] = 0ull;
    }
    if (!a.cost) return;

    // W. regroup: inside each window of kPlanWindow consecutive slots (rays
    // still spatially near in key order) the rays are stably partitioned by
    // a log-scale cost bucket (three per octave, costliest first; key order
    // kept inside a bucket), so each warp gets rays of similar length --
    // pass 1's lane efficiency rises from 0.56 to ~0.75 and the backward from
    // 1.49 to 1.32 ms (tools/exp_window.py; an exact sort by cost: 1.34 ms).  One
    // warp per window, kPlanWindow / 32 rays per lane: __match_any_sync
    // ranks equal buckets, a 32-bin warp scan places the buckets, and each
    // output warp's maximum cost is reduced in shared memory.
    {
        int* bins = s_stage[threadIdx.x >> 5];  // [32] bucket counts, then [32..35] output-warp maxima
        constexpr int PER = kPlanWindow / 32;
        const unsigned lt = (1u << lane) - 1u;
        const int64_t windows = (a.n + kPlanWindow - 1) / kPlanWindow;
        for (int64_t win = gwarp; win < windows; win += n_gwarps) {
            const int64_t b0 = win * kPlanWindow;
            const int cnt = int(min(int64_t(kPlanWindow), a.n - b0));
            bins[lane] = 0;
            if (lane < PER) bins[32 + lane] = 0;
            __syncwarp();
            int64_t v[PER];
            uint32_t cst[PER];
            int bk[PER], within[PER];
#pragma unroll
            for (int u = 0; u < PER; ++u) {
                const int e = lane + 32 * u;
                v[u] = e < cnt ? a.out[b0 + e] : 0;
                cst[u] = e < cnt ? uint32_t(w.slot_cost[b0 + e]) : 0u;
                // costliest first: bucket 0 holds the longest rays; padding lanes get bucket 32
                bk[u] = e < cnt ? 31 - cost_bucket(cst[u]) : 32 + lane;
            }
#pragma unroll
            for (int u = 0; u < PER; ++u) {  // groups in key order: stable
                const unsigned same = __match_any_sync(0xffffffffu, bk[u]);
                const int leader = __ffs(same) - 1;
                int old = 0;
                if (lane == leader && bk[u] < 32) {
                    old = bins[bk[u]];
                    bins[bk[u]] = old + __popc(same);
                }
                old = __shfl_sync(0xffffffffu, old, leader);
                within[u] = old + __popc(same & lt);
                __syncwarp();
            }
            const int count = bins[lane];
            int incl = count;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, off);
                if (lane >= off) incl += y;
            }
            bins[lane] = incl - count;  // bucket start
            __syncwarp();
#pragma unroll
            for (int u = 0; u < PER; ++u) {
                if (lane + 32 * u >= cnt) continue;
                const int pos = bins[bk[u]] + within[u];
                a.out[b0 + pos] = v[u];
                atomicMax(&bins[32 + (pos >> 5)], int(cst[u]));
            }
            __syncwarp();
            if (lane < PER && lane * 32 < cnt) w.warp_cost[(b0 >> 5) + lane] = uint32_t(bins[32 + lane]);
            __syncwarp();
        }
    }
    grid.sync();
    PLAN_STAMP(5)

    // E. chunk costs and their histogram (descending cost = ascending bin)
    const int64_t nfull = nw / a.chunk;
    for (int64_t c = gt; c < nfull; c += GT) {
        uint32_t mx = 0;
        for (int64_t v = c * a.chunk; v < (c + 1) * a.chunk; ++v) mx = max(mx, w.warp_cost[v]);
        w.chunk_cost[c] = uint16_t(mx);
        atomicAdd(w.hist + (kPlanCostBins - 1 - int(mx)), 1);
    }
    grid.sync();
    PLAN_STAMP(6)

    // F. bins -> start chunk (warp 0 of block 0: 32 bins per lane)
    if (blockIdx.x == 0 && threadIdx.x < 32) {
        constexpr int PER = kPlanCostBins / 32;
        int sum = 0;
        for (int u = 0; u < PER; ++u) sum += w.hist[lane * PER + u];
        int incl = sum;
        for (int off = 1; off < 32; off <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += y;
        }
        int ex = incl - sum;
        for (int u = 0; u < PER; ++u) {
            const int v = w.hist[lane * PER + u];
            w.hist[lane * PER + u] = ex;
            ex += v;
        }
    }
    grid.sync();
    PLAN_STAMP(7)

    // G. scatter the chunks; the short last chunk goes last; scratch cleared
    for (int64_t c = gt; c < nfull; c += GT) {
        const int64_t dst = int64_t(atomicAdd(w.hist + (kPlanCostBins - 1 - int(w.chunk_cost[c])), 1)) * a.chunk;
        for (int v = 0; v < a.chunk; ++v) a.warp_order[dst + v] = int32_t(c * a.chunk + v);
    }
    for (int64_t v = nfull * a.chunk + gt; v < nw; v += GT) a.warp_order[v] = int32_t(v);
    grid.sync();
    for (int64_t b = gt; b < kPlanCostBins; b += GT) w.hist[b] = 0;
    PLAN_STAMP(8)
}

size_t plan_ranked_workspace(int64_t n_pool, int64_t n, int) { return carve(nullptr, n_pool, n, nullptr); }

int run_plan_ranked(const int32_t* rank, const int32_t* order, int64_t n_pool, const int64_t* ray_idx, int64_t n,
                    int mode, const uint16_t* ray_cost, int chunk, int32_t* warp_order, void* ws, int64_t* out,
                    cudaStream_t s) {
    if (n == 0) return DOT_OK;
    if (g_plan_grid == 0) {
        int dev = 0, sms = 0, per_sm = 0;
        if (int st = check_cuda(cudaGetDevice(&dev), "cudaGetDevice")) return st;
        if (int st = check_cuda(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "attribute"))
            return st;
        if (int st = check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, plan_coop_kernel,
                                                                             kPlanThreads, 0), "occupancy"))
            return st;
        if (per_sm < 1 || sms * kPlanWarps > 4096)
            return set_error(DOT_CUDA_ERR, "plan_coop_kernel cannot be resident");
        g_plan_grid = sms;  // one skinny block per SM: resident beside the optimizer
    }
    PlanWs w;
    carve(ws, n_pool, n, &w);
    const uint16_t* cost = warp_order ? ray_cost : nullptr;
    PlanArgs a{rank, order, ray_idx, cost, warp_order, out, n_pool, n, mode, chunk,
               (mode == DOT_PLAN_SLOTS && cost && n <= (int64_t(1) << kTagSlotBits)) ? 1 : 0};
    void* params[] = {&a, &w};
    return check_cuda(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(plan_coop_kernel),
                                                  dim3(g_plan_grid), dim3(kPlanThreads), params, 0, s),
                      "plan_coop_kernel");
}

}  // namespace dot
