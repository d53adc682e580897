// refine.cu -- the DOT refine pass (prune -> sample -> canonical rebuild) on device.
//
// Semantics follow /root/reference/pkg/src/octrf/calibrate.py:71-238 exactly:
//  * prune: an internal node whose 8 children are all leaves is merged iff
//    every child signal <= tau (inclusive, calibrate.py:99); the merged payload
//    is the fp64 mean rounded once to f32 -- sigma summed pairwise
//    ((s0+s1)+(s2+s3))+((s4+s5)+(s6+s7)), SH summed sequentially (numpy's
//    reduction orders in merge_children_many, octree.py:284-285); the merged
//    signal is the pairwise sum of the children's (calibrate.py:126,216-217).
//    recursive: repeat on the new topology until nothing is selected.
//  * sample on the post-prune topology: eligible = depth < max_depth and
//    signal > 0; top ceil(gamma * L) by (signal desc, pool id asc), or
//    signal > threshold (calibrate.py:140-163).  Top-k is a radix select over
//    the fp64 signal bits (8 x 8-bit digits) with a second radix select over
//    pool ids for the ties at the k-th value; every decision stays on the
//    device (no host round trip between the passes).
//  * the refined tree is emitted directly in canonical BFS order
//    (scene_io.py:529-541), level by level: one flag scan per level decides
//    which nodes are internal, children are either the old children (kept)
//    or 8 payload copies of a split leaf (octree.py:216-248).
// The reference instead mutates a pooled tree through a LIFO free list and
// only canonicalises on save; topologies are compared after canonicalisation.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_scan.cuh>
#include <algorithm>
#include <cmath>
#include <vector>
#include "dot_tree.cuh"
#include "dot_internal.h"

namespace dot {

enum : uint8_t { ST_ALIVE = 1, ST_LEAF = 2, ST_MERGED = 4, ST_SPLIT = 8 };
enum : uint8_t { K_KEPT = 0, K_MERGED = 1, K_NEWCHILD = 2, K_SPLITPARENT = 3 };

constexpr int kTB = 256;
constexpr int kMaxLevels = 64;

static unsigned grid_for(int64_t n, int tb = kTB) { return unsigned((n + tb - 1) / tb); }

static unsigned persistent_blocks() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return unsigned(sms * 8);
}

// ---------------------------------------------------------------------------
// Exclusive scan of int32 flags.

__global__ void scan_total_kernel(const int32_t* __restrict__ in, const int64_t* __restrict__ out, int64_t n,
                                  int64_t* __restrict__ total) {
    *total = n ? out[n - 1] + in[n - 1] : 0;
}

// Exclusive prefix sum of 0/1 int32 flags into int64 (single-pass decoupled
// look-back scan, cub::DeviceScan) plus the total.
static int exclusive_scan(const int32_t* in, int64_t n, int64_t* out, int64_t* d_total, cudaStream_t s) {
    if (n == 0) return check_cuda(cudaMemsetAsync(d_total, 0, sizeof(int64_t), s), "memset");
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveScan(nullptr, bytes, in, out, cub::Sum(), int64_t(0), n, s);
    void* tmp = nullptr;
    int st = check_cuda(cudaMallocAsync(&tmp, bytes, s), "cudaMallocAsync");
    if (st == DOT_OK)
        st = check_cuda(cub::DeviceScan::ExclusiveScan(tmp, bytes, in, out, cub::Sum(), int64_t(0), n, s),
                        "DeviceScan");
    cudaFreeAsync(tmp, s);
    if (st != DOT_OK) return st;
    scan_total_kernel<<<1, 1, 0, s>>>(in, out, n, d_total);
    return check_launch("exclusive_scan");
}

// ---------------------------------------------------------------------------
// Device-side plan scalars (one struct, read back once at the end).

struct RadixState {
    unsigned long long prefix;  // selected high bits so far
    unsigned long long mask;    // which bits are fixed
    long long remaining;        // how many still to take at/below the prefix
    long long eq_count;         // count of keys equal to the final prefix
};

struct PlanScalars {
    unsigned long long n_internal;   // before prune
    unsigned long long merges;       // all rounds
    unsigned long long round_merges; // current round
    unsigned long long leaves;       // post-prune leaf count
    unsigned long long eligible;     // post-prune eligible leaves
    long long k;                     // sample size
    unsigned long long splits;
    RadixState sig_rs;               // radix select over signal bits
    RadixState tie_rs;               // radix select over (0xFFFFFFFF - pool id) among ties
    unsigned long long n_cand;       // candidates compacted after the first passes
};

}  // namespace dot

struct dot_refine_plan {
    int64_t N = 0;
    int S = 0;
    int B = 0;
    bool use_sigma = false;
    uint8_t* state = nullptr;
    uint8_t* depth = nullptr;
    double* sig = nullptr;
    int32_t* slot = nullptr;
    int32_t* mround = nullptr;   // merge round (1-based) or 0
    const int32_t* pool_id = nullptr;  // caller-owned, may be NULL (identity)
    float* msig = nullptr;       // merged payload [M]
    float* msh = nullptr;        // merged SH [M * S]
    int64_t M = 0, K = 0;
    bool lists_ready = false;
    std::vector<int64_t> merge_list;   // canonical, (round, index) order
    std::vector<int32_t> merge_round_h;
    std::vector<int64_t> split_list;   // canonical ascending
    dot_refine_stats stats{};
    int32_t max_depth = 0;
    std::vector<int64_t> level_off;    // old canonical BFS level boundaries
};

namespace dot {

// Block-wide sum of a per-thread count, one atomicAdd per block (the N-wide
// kernels run grid-stride on persistent_blocks(): ~1k atomics per counter
// instead of one per 256-thread block).
__device__ __forceinline__ void block_add(unsigned long long* dst, unsigned v) {
    __shared__ unsigned part[32];
    v = __reduce_add_sync(0xffffffffu, v);
    const int w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) part[w] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int k = 0; k < nw; ++k) t += part[k];
        if (t) atomicAdd(dst, t);
    }
}

__device__ __forceinline__ int32_t pid_of(const int32_t* pool_id, int64_t i) {
    return pool_id ? pool_id[i] : int32_t(i);
}

__constant__ int64_t c_level_off[kMaxLevels + 1];

// state / depth / signal of every node; depth from the BFS level offsets.
__global__ void __launch_bounds__(256) init_nodes_kernel(
    TreeDev T, int64_t N, int n_levels, const double* __restrict__ acc, int use_sigma,
    uint8_t* __restrict__ state, uint8_t* __restrict__ depth, double* __restrict__ sig,
    int32_t* __restrict__ slot, int32_t* __restrict__ mround, PlanScalars* __restrict__ ps) {
    unsigned internal = 0;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
#pragma unroll 4
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < N; i += stride) {
        int dd = 0;
        while (dd + 1 < n_levels && c_level_off[dd + 1] <= i) ++dd;
        const int32_t w = T.node[i];
        depth[i] = uint8_t(dd);
        slot[i] = -1;
        mround[i] = 0;
        if (w < 0) {
            state[i] = ST_ALIVE | ST_LEAF;
            const int32_t pid = ~w;
            sig[i] = use_sigma ? double(T.sigma[pid]) : acc[pid];
        } else {
            state[i] = ST_ALIVE;
            sig[i] = 0.0;
            ++internal;
        }
    }
    block_add(&ps->n_internal, internal);
}

// Warp-aggregated append of index i to list (count in *ctr).
__device__ __forceinline__ void append(bool want, int64_t i, int64_t* list, unsigned long long* ctr) {
    const unsigned m = __ballot_sync(0xffffffffu, want);
    if (!m) return;
    const unsigned lane = threadIdx.x & 31;
    const int leader = __ffs(m) - 1;
    unsigned long long base = 0;
    if (int(lane) == leader) base = atomicAdd(ctr, (unsigned long long)__popc(m));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (want) list[base + __popc(m & ((1u << lane) - 1u))] = i;
}

// Prune selection for one round: alive internal nodes whose 8 children are
// leaves with signal <= tau.  Appended (unordered) to list.
__global__ void prune_select_kernel(TreeDev T, int64_t N, double tau, const uint8_t* __restrict__ state,
                                    const double* __restrict__ sig, int64_t* __restrict__ list,
                                    PlanScalars* __restrict__ ps) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    bool ok = false;
    if (i < N) {
        const uint8_t st = state[i];
        if ((st & ST_ALIVE) && !(st & ST_LEAF)) {
            const int32_t c = T.node[i];
            ok = true;
#pragma unroll
            for (int o = 0; o < 8; ++o)
                if ((state[c + o] & ST_LEAF) == 0 || !(sig[c + o] <= tau)) ok = false;
        }
    }
    append(ok, i, list, &ps->round_merges);
}

__device__ __forceinline__ const float* leaf_row_sh(const TreeDev& T, const float* msh, const int32_t* slot,
                                                    const uint8_t* state, int64_t i, int S) {
    if (state[i] & ST_MERGED) return msh + int64_t(slot[i]) * S;
    return T.sh + int64_t(~T.node[i]) * S;
}

__device__ __forceinline__ float leaf_sigma(const TreeDev& T, const float* msig, const int32_t* slot,
                                            const uint8_t* state, int64_t i) {
    if (state[i] & ST_MERGED) return msig[slot[i]];
    return T.sigma[~T.node[i]];
}

// Merged SH rows: one thread per (parent, 4-column quad); sequential fp64
// sum over the 8 children in octant order, /8, round once.
__global__ void merge_sh_kernel(TreeDev T, const int64_t* __restrict__ list, const PlanScalars* __restrict__ ps,
                                int64_t slot_base, const uint8_t* __restrict__ state,
                                const int32_t* __restrict__ slot, float* __restrict__ msh, int S, int nsh) {
    const int64_t m = int64_t(ps->round_merges);
    const int S4 = S / 4;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < m * S4; t += stride) {
        const int64_t j = t / S4;
        const int q = int(t - j * S4);
        const int32_t c = T.node[list[j]];
        double acc[4];
#pragma unroll
        for (int o = 0; o < 8; ++o) {
            const float4 v = reinterpret_cast<const float4*>(leaf_row_sh(T, msh, slot, state, c + o, S))[q];
            if (o == 0) {
                acc[0] = v.x; acc[1] = v.y; acc[2] = v.z; acc[3] = v.w;
            } else {
                acc[0] = acc[0] + double(v.x);
                acc[1] = acc[1] + double(v.y);
                acc[2] = acc[2] + double(v.z);
                acc[3] = acc[3] + double(v.w);
            }
        }
        float4 out;
        out.x = 4 * q + 0 < nsh ? float(acc[0] / 8.0) : 0.f;
        out.y = 4 * q + 1 < nsh ? float(acc[1] / 8.0) : 0.f;
        out.z = 4 * q + 2 < nsh ? float(acc[2] / 8.0) : 0.f;
        out.w = 4 * q + 3 < nsh ? float(acc[3] / 8.0) : 0.f;
        reinterpret_cast<float4*>(msh + (slot_base + j) * S)[q] = out;
    }
}

// Merged sigma (pairwise) and signal (pairwise), then the topology flags.
__global__ void merge_finish_kernel(TreeDev T, const int64_t* __restrict__ list, PlanScalars* __restrict__ ps,
                                    int64_t slot_base, int round, int use_sigma, uint8_t* __restrict__ state,
                                    double* __restrict__ sig, int32_t* __restrict__ slot,
                                    int32_t* __restrict__ mround, float* __restrict__ msig) {
    const int64_t m = int64_t(ps->round_merges);
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < m; j += stride) {
        const int64_t p = list[j];
        const int32_t c = T.node[p];
        double s8[8], q8[8];
#pragma unroll
        for (int o = 0; o < 8; ++o) {
            s8[o] = double(leaf_sigma(T, msig, slot, state, c + o));
            q8[o] = sig[c + o];
        }
        const double ssum = ((s8[0] + s8[1]) + (s8[2] + s8[3])) + ((s8[4] + s8[5]) + (s8[6] + s8[7]));
        const float mean_sigma = float(ssum / 8.0);
        const double qsum = ((q8[0] + q8[1]) + (q8[2] + q8[3])) + ((q8[4] + q8[5]) + (q8[6] + q8[7]));
        msig[slot_base + j] = mean_sigma;
        sig[p] = use_sigma ? double(mean_sigma) : qsum;
        mround[p] = round;
    }
}

// Separate pass so no thread flips a flag another thread of the same round reads.
__global__ void merge_flags_kernel(TreeDev T, const int64_t* __restrict__ list, PlanScalars* __restrict__ ps,
                                   int64_t slot_base, uint8_t* __restrict__ state, int32_t* __restrict__ slot) {
    const int64_t m = int64_t(ps->round_merges);
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < m; j += stride) {
        const int64_t p = list[j];
        const int32_t c = T.node[p];
#pragma unroll
        for (int o = 0; o < 8; ++o) state[c + o] &= uint8_t(~ST_ALIVE);
        slot[p] = int32_t(slot_base + j);
        state[p] |= ST_LEAF | ST_MERGED;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) ps->merges += ps->round_merges;
}

__device__ __forceinline__ unsigned long long sample_key(int64_t i, const uint8_t* state,
                                                         const uint8_t* depth, const double* sig,
                                                         int max_depth) {
    const uint8_t st = state[i];
    if (!((st & ST_ALIVE) && (st & ST_LEAF))) return 0ull;
    const double s = sig[i];
    if (!(depth[i] < max_depth && s > 0.0)) return 0ull;
    return (unsigned long long)__double_as_longlong(s);  // positive doubles order as uint64
}

// Leaf / eligibility counts on the post-prune topology.
// 16 consecutive 64-bit keys / state bytes per thread with 16-byte vector
// loads (the N-wide passes below are bandwidth passes: one key or byte per
// thread left them at ~1.2 TB/s).
__device__ __forceinline__ void load16_keys(const unsigned long long* __restrict__ a, int64_t i0, int64_t N,
                                            unsigned long long* v) {
    if (i0 + 16 <= N) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const ulonglong2 x = reinterpret_cast<const ulonglong2*>(a + i0)[k];
            v[2 * k] = x.x;
            v[2 * k + 1] = x.y;
        }
    } else {
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = i0 + k < N ? a[i0 + k] : 0ull;
    }
}

// Post-prune sample keys of every node in one coalesced pass (16 nodes per
// thread, 16-byte vector loads): keys[i] = sample_key(i) (0 = not eligible),
// the live-leaf and eligible counts, and the histogram of the keys' top byte
// (the first radix pass of the top-k select, which does not depend on k).
__global__ void __launch_bounds__(256) sample_keys_kernel(
    int64_t N, const uint8_t* __restrict__ state, const uint8_t* __restrict__ depth,
    const double* __restrict__ sig, int max_depth, unsigned long long* __restrict__ keys,
    unsigned int* __restrict__ hist, PlanScalars* __restrict__ ps) {
    __shared__ unsigned int h[256];
    for (int b = threadIdx.x; b < 256; b += blockDim.x) h[b] = 0;
    __syncthreads();
    unsigned leaf = 0, elig = 0;
    const int64_t chunks = (N + 15) / 16;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; c < chunks; c += stride) {
        const int64_t i0 = 16 * c;
        uint8_t st[16], dp[16];
        double sg[16];
        if (i0 + 16 <= N) {
            *reinterpret_cast<uint4*>(st) = *reinterpret_cast<const uint4*>(state + i0);
            *reinterpret_cast<uint4*>(dp) = *reinterpret_cast<const uint4*>(depth + i0);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const double2 v = reinterpret_cast<const double2*>(sig + i0)[k];
                sg[2 * k] = v.x;
                sg[2 * k + 1] = v.y;
            }
        } else {
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const bool in = i0 + k < N;
                st[k] = in ? state[i0 + k] : 0;
                dp[k] = in ? depth[i0 + k] : 0;
                sg[k] = in ? sig[i0 + k] : 0.0;
            }
        }
        unsigned long long kv[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const bool lf = (st[k] & ST_ALIVE) && (st[k] & ST_LEAF);
            const bool el = lf && dp[k] < max_depth && sg[k] > 0.0;
            leaf += lf;
            elig += el;
            kv[k] = el ? (unsigned long long)__double_as_longlong(sg[k]) : 0ull;
        }
        if (i0 + 16 <= N) {
#pragma unroll
            for (int k = 0; k < 8; ++k)
                reinterpret_cast<ulonglong2*>(keys + i0)[k] = make_ulonglong2(kv[2 * k], kv[2 * k + 1]);
        } else {
            for (int k = 0; k < 16 && i0 + k < N; ++k) keys[i0 + k] = kv[k];
        }
#pragma unroll
        for (int k = 0; k < 16; ++k)
            if (kv[k]) atomicAdd(&h[unsigned(kv[k] >> 56)], 1u);
    }
    block_add(&ps->leaves, leaf);
    block_add(&ps->eligible, elig);
    __syncthreads();
    for (int b = threadIdx.x; b < 256; b += blockDim.x)
        if (h[b]) atomicAdd(hist + b, h[b]);
}

__global__ void __launch_bounds__(256) count_leaves_kernel(
    int64_t N, const uint8_t* __restrict__ state, const uint8_t* __restrict__ depth,
    const double* __restrict__ sig, int max_depth, PlanScalars* __restrict__ ps) {
    unsigned leaf = 0, elig = 0;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
#pragma unroll 4
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < N; i += stride) {
        const uint8_t st = state[i];
        if ((st & ST_ALIVE) && (st & ST_LEAF)) {
            ++leaf;
            elig += depth[i] < max_depth && sig[i] > 0.0;  // sample_key != 0
        }
    }
    block_add(&ps->leaves, leaf);
    block_add(&ps->eligible, elig);
}

// k = min(ceil(gamma * L), #eligible) (calibrate.py:159), both radix states primed.
__global__ void sample_k_kernel(PlanScalars* ps, double gamma) {
    long long k = (long long)ceil(gamma * double(ps->leaves));
    if (k > (long long)ps->eligible) k = (long long)ps->eligible;
    ps->k = k;
    ps->sig_rs = RadixState{0ull, 0ull, k, 0};
    ps->tie_rs = RadixState{0ull, 0xFFFFFFFF00000000ull, 0, 0};
}

// Histogram of digit `shift` over keys matching the current prefix, with
// warp-aggregated shared-memory increments (most keys share the high digits).
// mode 0: signal keys; mode 1: tie keys (0xFFFFFFFF - pool id) among keys == K*.
// One radix pass of the top-k select.  The first passes scan every node;
// after them radix_compact_kernel keeps only the keys still matching the
// selected prefix (a ~1/16-binade slice), and the remaining passes run over
// that candidate list (ckey / cidx, count in ps->n_cand).
__global__ void radix_hist_kernel(int64_t N, int mode, const uint8_t* __restrict__ state,
                                  const uint8_t* __restrict__ depth, const double* __restrict__ sig,
                                  int max_depth, const int32_t* __restrict__ pool_id,
                                  const PlanScalars* __restrict__ ps, int shift, unsigned int* __restrict__ hist,
                                  const unsigned long long* __restrict__ ckey,
                                  const int32_t* __restrict__ cidx, const unsigned long long* __restrict__ nkey) {
    __shared__ unsigned int h[256];
    const RadixState rs = mode == 0 ? ps->sig_rs : ps->tie_rs;
    const bool skip = mode == 0 ? ps->k <= 0 : (ps->k <= 0 || ps->sig_rs.remaining == ps->sig_rs.eq_count);
    if (skip) return;
    for (int b = threadIdx.x; b < 256; b += blockDim.x) h[b] = 0;
    __syncthreads();
    const unsigned long long kstar = ps->sig_rs.prefix;
    if (!ckey && mode == 0) {  // full pass over the key array, 16 keys per thread
        const int64_t chunks = (N + 15) / 16;
        const int64_t stride = int64_t(gridDim.x) * blockDim.x;
        for (int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; c < chunks; c += stride) {
            unsigned long long v[16];
            load16_keys(nkey, 16 * c, N, v);
#pragma unroll
            for (int k = 0; k < 16; ++k)
                if (v[k] != 0ull && (v[k] & rs.mask) == rs.prefix) atomicAdd(&h[unsigned((v[k] >> shift) & 0xFF)], 1u);
        }
        __syncthreads();
        for (int b = threadIdx.x; b < 256; b += blockDim.x)
            if (h[b]) atomicAdd(hist + b, h[b]);
        return;
    }
    const int64_t M = ckey ? int64_t(ps->n_cand) : N;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    const int64_t n_iter = (M + stride - 1) / stride;
    for (int64_t it = 0; it < n_iter; ++it) {
        const int64_t j = it * stride + int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
        bool take = false;
        unsigned bin = 0;
        if (j < M) {
            const int64_t i = ckey ? int64_t(cidx[j]) : j;
            unsigned long long key = ckey ? ckey[j] : nkey[j];
            if (key != 0ull) {
                if (mode == 1) {
                    if (key == kstar) {
                        key = 0xFFFFFFFFull - (unsigned long long)(uint32_t)pid_of(pool_id, i);
                        take = (key & rs.mask) == rs.prefix;
                    }
                } else {
                    take = (key & rs.mask) == rs.prefix;
                }
                bin = unsigned((key >> shift) & 0xFF);
            }
        }
        const unsigned active = __ballot_sync(0xffffffffu, take);
        if (take) {
            const unsigned peers = __match_any_sync(active, bin);
            if ((threadIdx.x & 31) == unsigned(__ffs(peers) - 1)) atomicAdd(&h[bin], unsigned(__popc(peers)));
        }
    }
    __syncthreads();
    for (int b = threadIdx.x; b < 256; b += blockDim.x)
        if (h[b]) atomicAdd(hist + b, h[b]);
}

__global__ void __launch_bounds__(256) radix_compact_kernel(
    int64_t N, PlanScalars* __restrict__ ps, unsigned long long* __restrict__ ckey,
    int32_t* __restrict__ cidx, const unsigned long long* __restrict__ nkey) {
    const RadixState rs = ps->sig_rs;
    if (ps->k <= 0) return;
    const int lane = threadIdx.x & 31;
    const int64_t chunks = (N + 15) / 16;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    // uniform trip count per warp (warp-collective scan below)
    const int64_t c0 = int64_t(blockIdx.x) * blockDim.x + (threadIdx.x & ~31);
    for (int64_t cb = c0; cb < chunks; cb += stride) {
        const int64_t c = cb + lane;
        unsigned long long v[16];
        load16_keys(nkey, 16 * c, c < chunks ? N : 0, v);
        unsigned m = 0;
#pragma unroll
        for (int k = 0; k < 16; ++k)
            if (v[k] != 0ull && (v[k] & rs.mask) == rs.prefix) m |= 1u << k;
        const unsigned cnt = __popc(m);
        unsigned incl = cnt;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += y;
        }
        const unsigned tot = __shfl_sync(0xffffffffu, incl, 31);
        unsigned long long base = 0;
        if (lane == 31 && tot) base = atomicAdd(&ps->n_cand, (unsigned long long)tot);
        base = __shfl_sync(0xffffffffu, base, 31);
        unsigned long long at = base + incl - cnt;
        while (m) {
            const int k = __ffs(m) - 1;
            m &= m - 1;
            ckey[at] = v[k];
            cidx[at] = int32_t(16 * c + k);
            ++at;
        }
    }
}

// Pick the next radix digit: the largest bin b with sum(hist[b..255]) >=
// remaining (one warp: 8 bins per lane, suffix sums by shuffles), then clear
// the histogram for the next pass.
__global__ void radix_pick_kernel(PlanScalars* ps, int mode, unsigned int* hist, int shift) {
    const int lane = threadIdx.x & 31;
    RadixState& rs = mode == 0 ? ps->sig_rs : ps->tie_rs;
    const bool skip = mode == 0 ? ps->k <= 0 : (ps->k <= 0 || ps->sig_rs.remaining == ps->sig_rs.eq_count);
    // lane l owns bins [8 l, 8 l + 8)
    unsigned h[8];
    long long own = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        h[k] = hist[8 * lane + k];
        own += h[k];
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 8; ++k) hist[8 * lane + k] = 0;
    if (skip) return;
    // suffix sum over lanes: above = sum of bins of lanes > lane
    long long incl = own;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const long long v = __shfl_down_sync(0xffffffffu, incl, off);
        if (lane + off < 32) incl += v;
    }
    const long long above = incl - own;
    long long rem = (mode == 1 && shift == 24) ? ps->sig_rs.remaining : rs.remaining;
    // the digit lies in this lane's bins iff above < rem <= above + own
    const bool mine = above < rem && rem <= above + own;
    const unsigned who = __ballot_sync(0xffffffffu, mine);
    if (!mine) return;
    (void)who;
    rem -= above;
    int digit = 8 * lane;
    long long eq = 0;
    for (int k = 7; k >= 0; --k) {
        const long long c = h[k];
        if (rem <= c) {
            digit = 8 * lane + k;
            eq = c;
            break;
        }
        rem -= c;
    }
    rs.remaining = rem;
    rs.eq_count = eq;
    rs.prefix |= (unsigned long long)digit << shift;
    rs.mask |= 0xFFull << shift;
}

// Mark the sample selection: key > K*, plus ties (key == K*) whose tie key
// >= T* (i.e. pool id <= the m-th smallest), or threshold mode.
// Top-k mode of mark_split over the key array, 16 nodes per thread.
__global__ void __launch_bounds__(256) mark_split_keys_kernel(
    int64_t N, uint8_t* __restrict__ state, const int32_t* __restrict__ pool_id,
    PlanScalars* __restrict__ ps, const unsigned long long* __restrict__ nkey) {
    unsigned nsel = 0;
    if (ps->k > 0) {
        const unsigned long long kstar = ps->sig_rs.prefix;
        const bool all = ps->sig_rs.remaining == ps->sig_rs.eq_count;
        const unsigned long long tie = ps->tie_rs.prefix;
        const int64_t chunks = (N + 15) / 16;
        const int64_t stride = int64_t(gridDim.x) * blockDim.x;
        for (int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; c < chunks; c += stride) {
            const int64_t i0 = 16 * c;
            unsigned long long v[16];
            load16_keys(nkey, i0, N, v);
            unsigned m = 0;
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                bool sel = v[k] != 0ull && v[k] > kstar;
                if (v[k] != 0ull && v[k] == kstar)
                    sel = all || 0xFFFFFFFFull - (unsigned long long)(uint32_t)pid_of(pool_id, i0 + k) >= tie;
                if (sel) m |= 1u << k;
            }
            if (m) {
                nsel += __popc(m);
                if (i0 + 16 <= N) {
                    uint4 w = *reinterpret_cast<const uint4*>(state + i0);
                    uint8_t* b = reinterpret_cast<uint8_t*>(&w);
#pragma unroll
                    for (int k = 0; k < 16; ++k)
                        if (m & (1u << k)) b[k] |= ST_SPLIT;
                    *reinterpret_cast<uint4*>(state + i0) = w;
                } else {
                    for (int k = 0; k < 16; ++k)
                        if (m & (1u << k)) state[i0 + k] |= ST_SPLIT;
                }
            }
        }
    }
    block_add(&ps->splits, nsel);
}

__global__ void __launch_bounds__(256) mark_split_kernel(
    int64_t N, int mode, uint8_t* __restrict__ state, const uint8_t* __restrict__ depth,
    const double* __restrict__ sig, int max_depth, const int32_t* __restrict__ pool_id, double thr,
    PlanScalars* __restrict__ ps, const unsigned long long* __restrict__ nkey) {
    unsigned nsel = 0;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
#pragma unroll 4
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < N; i += stride) {
        bool sel = false;
        const unsigned long long key = nkey ? nkey[i] : sample_key(i, state, depth, sig, max_depth);
        if (key != 0ull) {
            if (mode == 2) {
                sel = sig[i] > thr;
            } else if (ps->k > 0) {
                const unsigned long long kstar = ps->sig_rs.prefix;
                sel = key > kstar;
                if (key == kstar) {
                    const bool all = ps->sig_rs.remaining == ps->sig_rs.eq_count;
                    const unsigned long long tk =
                        0xFFFFFFFFull - (unsigned long long)(uint32_t)pid_of(pool_id, i);
                    sel = all || tk >= ps->tie_rs.prefix;
                }
            }
        }
        if (sel) {
            state[i] |= ST_SPLIT;
            ++nsel;
        }
    }
    block_add(&ps->splits, nsel);
}

// Ordered compaction flags for the on-demand event lists.
__global__ void flag_kernel(int64_t N, const uint8_t* __restrict__ state, const int32_t* __restrict__ mround,
                            int which, int32_t* __restrict__ flags) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= N) return;
    flags[i] = which == 0 ? (mround[i] > 0) : ((state[i] & ST_SPLIT) != 0);
}

__global__ void compact_kernel(int64_t N, const int32_t* __restrict__ flags, const int64_t* __restrict__ rank,
                               int64_t* __restrict__ out) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < N && flags[i]) out[rank[i]] = i;
}

// ---------------------------------------------------------------------------
// Canonical rebuild in one scan.  The new tree's BFS order keeps the relative
// order of surviving nodes inside a level, so with
//   f(i) = 1 if old node i is internal after the refine (alive internal and
//          not merged, or a leaf selected for splitting), and
//   R(i) = exclusive prefix sum of f over the old BFS order,
// the children block of an internal-after node i at level L starts at
//   new_base[L+1] + 8 (R(i) - R(off[L])),
// every surviving non-root node sits at its parent's block + octant, and a
// split leaf's 8 new children fill its block (scene_io.py:529-541 order).

__global__ void __launch_bounds__(256) rebuild_flags_kernel(int64_t N, const uint8_t* __restrict__ state,
                                                            int32_t* __restrict__ flags) {
    const int64_t chunks = (N + 15) / 16;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; c < chunks; c += stride) {
        const int64_t i0 = 16 * c;
        if (i0 + 16 <= N) {
            const uint4 w = *reinterpret_cast<const uint4*>(state + i0);
            const uint8_t* b = reinterpret_cast<const uint8_t*>(&w);
            int f[16];
#pragma unroll
            for (int k = 0; k < 16; ++k)
                f[k] = (b[k] & ST_ALIVE) && (!(b[k] & ST_LEAF) || (b[k] & ST_SPLIT)) ? 1 : 0;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                reinterpret_cast<int4*>(flags + i0)[k] = make_int4(f[4 * k], f[4 * k + 1], f[4 * k + 2], f[4 * k + 3]);
        } else {
            for (int64_t i = i0; i < N; ++i) {
                const uint8_t st = state[i];
                flags[i] = (st & ST_ALIVE) && (!(st & ST_LEAF) || (st & ST_SPLIT)) ? 1 : 0;
            }
        }
    }
}

// new_base[L] (new level offsets) and rb[L] = R(off[L]), one thread.
__global__ void rebuild_levels_kernel(int n_levels, const int64_t* __restrict__ rank,
                                      const int64_t* __restrict__ total, int64_t* __restrict__ new_base,
                                      int64_t* __restrict__ rb) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int64_t base = 0, count = 1;
    for (int L = 0; L < n_levels; ++L) {
        const int64_t r0 = rank[c_level_off[L]];
        const int64_t r1 = (L + 1 < n_levels) ? rank[c_level_off[L + 1]] : *total;
        rb[L] = r0;
        new_base[L] = base;
        base += count;
        count = 8 * (r1 - r0);  // nodes of new level L + 1
    }
    new_base[n_levels] = base;  // the split children of the deepest level
    new_base[n_levels + 1] = base + count;
}

// One thread per old node; internal-after nodes write their 8-child block
// (consecutive internal-after nodes own consecutive blocks, so a warp's
// writes are contiguous).  Entry 0 (the root) is written by thread 0.
__device__ __forceinline__ void emit_node(const TreeDev& T, int64_t g, int64_t i, int L, uint8_t st, int flag,
                                          const int64_t* __restrict__ rank, const int64_t* __restrict__ new_base,
                                          const int64_t* __restrict__ rb, int32_t* __restrict__ new_node,
                                          int64_t* __restrict__ src_index, uint8_t* __restrict__ src_kind) {
    src_index[g] = i;
    if (flag) {
        new_node[g] = int32_t(new_base[L + 1] + 8 * (rank[i] - rb[L]));
        src_kind[g] = (st & ST_LEAF) ? K_SPLITPARENT : K_KEPT;
    } else {
        new_node[g] = ~int32_t(g);
        src_kind[g] = (st & ST_MERGED) ? K_MERGED : K_KEPT;
    }
}

__global__ void __launch_bounds__(256) rebuild_emit_kernel(
    TreeDev T, int64_t N, const uint8_t* __restrict__ state, const uint8_t* __restrict__ depth,
    const int32_t* __restrict__ flags, const int64_t* __restrict__ rank,
    const int64_t* __restrict__ new_base, const int64_t* __restrict__ rb, int32_t* __restrict__ new_node,
    int64_t* __restrict__ src_index, uint8_t* __restrict__ src_kind) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    if (i == 0) emit_node(T, 0, 0, 0, state[0], flags[0], rank, new_base, rb, new_node, src_index, src_kind);
    const int f = i < N ? flags[i] : 0;
    const unsigned m = __ballot_sync(0xffffffffu, f != 0);
    if (!m) return;
    // this warp's internal-after nodes emit their child blocks together: slot
    // s = 8 * (rank of the parent among the warp's set bits) + octant, one
    // lane per slot, so every store instruction covers contiguous entries
    uint8_t st = 0;
    int L = 0;
    int64_t cb = 0;
    int32_t c = 0;
    if (f) {
        st = state[i];
        L = depth[i];
        cb = new_base[L + 1] + 8 * (rank[i] - rb[L]);
        c = T.node[i];
    }
    const int slots = 8 * __popc(m);
    for (int s0 = 0; s0 < slots; s0 += 32) {
        const int sl = s0 + lane;
        const int q = sl < slots ? sl >> 3 : 0;
        const int src = __fns(m, 0, q + 1);  // lane of the q-th parent
        const uint8_t pst = __shfl_sync(0xffffffffu, st, src);
        const int pL = __shfl_sync(0xffffffffu, L, src);
        const int64_t pcb = __shfl_sync(0xffffffffu, cb, src);
        const int32_t pc = __shfl_sync(0xffffffffu, c, src);
        const int64_t pi = __shfl_sync(0xffffffffu, i, src);
        if (sl >= slots) continue;
        const int k = sl & 7;
        const int64_t g = pcb + k;
        if (pst & ST_LEAF) {  // split: 8 new leaves copying this (original or merged) leaf
            new_node[g] = ~int32_t(g);
            src_index[g] = pi;
            src_kind[g] = K_NEWCHILD;
        } else {  // kept internal node: its 8 (alive) children in octant order
            const int64_t ch = int64_t(pc) + k;
            emit_node(T, g, ch, pL + 1, state[ch], flags[ch], rank, new_base, rb, new_node, src_index, src_kind);
        }
    }
}

// Payload gather, warp-cooperative: a warp owns 32 consecutive new nodes;
// lane l resolves node l's source row (merged parent -> merge buffer, other
// leaves -> old payload row, internal -> zeros) once, then the warp streams
// the 32 rows in 16-byte chunks with consecutive lanes on consecutive
// chunks -- stores fully coalesced (new rows are contiguous), loads
// coalesced wherever consecutive new leaves come from consecutive old rows
// (the common case: BFS order is preserved between kept siblings).  All of a
// lane's chunk loads are issued before its stores.
template <int S4>
__global__ void __launch_bounds__(256) payload_kernel(
    TreeDev T, int64_t n_new, const int64_t* __restrict__ src_index,
    const uint8_t* __restrict__ state, const int32_t* __restrict__ slot,
    const float* __restrict__ msig, const float* __restrict__ msh,
    const int32_t* __restrict__ new_node, float* __restrict__ new_sigma, float4* __restrict__ new_sh) {
    const int lane = threadIdx.x & 31;
    const int64_t base = ((int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * 32;
    if (base >= n_new) return;
    const int64_t i = base + lane;
    const float4* src = nullptr;  // row of node i (NULL: zeros)
    float sg = 0.f;
    if (i < n_new && new_node[i] < 0) {
        const int64_t o = src_index[i];
        if (state[o] & ST_MERGED) {
            const int32_t sl = slot[o];
            src = reinterpret_cast<const float4*>(msh) + int64_t(sl) * S4;
            sg = msig[sl];
        } else {
            const int32_t pid = ~T.node[o];
            src = reinterpret_cast<const float4*>(T.sh) + int64_t(pid) * S4;
            sg = __ldg(T.sigma + pid);
        }
    }
    if (i < n_new) new_sigma[i] = sg;
    const int rows = int(n_new - base < 32 ? n_new - base : 32);
    const int chunks = rows * S4;
    float4 v[S4];
#pragma unroll
    for (int k = 0; k < S4; ++k) {
        const int c = k * 32 + lane;
        const int r = c / S4;
        const float4* p = reinterpret_cast<const float4*>(
            __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(src), r & 31));
        v[k] = (c < chunks && p) ? __ldg(p + (c - r * S4)) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float4* dst = new_sh + base * S4;
#pragma unroll
    for (int k = 0; k < S4; ++k) {
        const int c = k * 32 + lane;
        if (c < chunks) dst[c] = v[k];
    }
}

template <typename Tp>
static int dalloc(Tp** p, size_t n, cudaStream_t s) {
    retain_pool_memory();
    return check_cuda(cudaMallocAsync(reinterpret_cast<void**>(p), sizeof(Tp) * (n ? n : 1), s),
                      "cudaMallocAsync");
}

}  // namespace dot

using namespace dot;

static void plan_free(dot_refine_plan* p) {
    if (!p) return;
    cudaFree(p->state);
    cudaFree(p->depth);
    cudaFree(p->sig);
    cudaFree(p->slot);
    cudaFree(p->mround);
    cudaFree(p->msig);
    cudaFree(p->msh);
    delete p;
}

// Level offsets of a canonical node table (one sync per level; only used
// when the caller does not already know them).
static int level_offsets_of(const TreeDev& T, int64_t N, std::vector<int64_t>& off, cudaStream_t s) {
    off.assign(1, 0);
    int64_t lo = 0, hi = 1;
    std::vector<int32_t> w;
    while (lo < hi) {
        off.push_back(hi);
        if (int(off.size()) > kMaxLevels) return set_error(DOT_BAD_ARG, "tree deeper than %d levels", kMaxLevels);
        w.resize(size_t(hi - lo));
        int st = check_cuda(cudaMemcpyAsync(w.data(), T.node + lo, (hi - lo) * sizeof(int32_t),
                                            cudaMemcpyDeviceToHost, s), "memcpy");
        if (st == DOT_OK) st = check_cuda(cudaStreamSynchronize(s), "sync");
        if (st) return st;
        int64_t n_int = 0;
        for (int32_t x : w) n_int += x >= 0;
        lo = hi;
        hi += 8 * n_int;
    }
    if (hi != N)
        return set_error(DOT_BAD_ARG, "node table is not a canonical BFS tree (%lld reachable of %lld)",
                         (long long)hi, (long long)N);
    return DOT_OK;
}

extern "C" {

int dot_refine_plan_create(const dot_tree_view* tree, const int32_t* pool_id, const double* acc,
                           int32_t use_sigma, double tau, double gamma, int32_t recursive,
                           int32_t use_threshold, double threshold, const int64_t* level_offsets,
                           int32_t n_level_offsets, dot_refine_plan** out, dot_refine_stats* stats,
                           void* stream) {
    if (!tree || !out || !stats) return set_error(DOT_BAD_ARG, "NULL argument");
    if (!use_sigma && !acc) return set_error(DOT_BAD_ARG, "acc must not be NULL for the Q target");
    if (tau < 0.0) return set_error(DOT_BAD_ARG, "tau must be >= 0, got %g", tau);
    if (!(gamma >= 0.0 && gamma <= 1.0)) return set_error(DOT_BAD_ARG, "gamma must be in [0, 1]");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const TreeDev T = make_tree(*tree);
    const int64_t N = tree->n_nodes;
    const int S = tree->sh_stride, B = tree->basis_count;
    std::vector<int64_t> off;
    int st = DOT_OK;
    if (level_offsets && n_level_offsets >= 2) {
        if (n_level_offsets - 1 > kMaxLevels) return set_error(DOT_BAD_ARG, "too many levels");
        off.assign(level_offsets, level_offsets + n_level_offsets);
        if (off.front() != 0 || off.back() != N) return set_error(DOT_BAD_ARG, "level offsets do not match the tree");
    } else if ((st = level_offsets_of(T, N, off, s)) != DOT_OK) {
        return st;
    }
    const int n_levels = int(off.size()) - 1;
    dot_refine_plan* p = new dot_refine_plan();
    p->level_off = off;
    p->N = N;
    p->S = S;
    p->B = B;
    p->use_sigma = use_sigma != 0;
    p->pool_id = pool_id;
    p->max_depth = tree->max_depth;
    int64_t* d_list = nullptr;
    unsigned int* d_hist = nullptr;
    PlanScalars* d_ps = nullptr;
    unsigned long long* d_ckey = nullptr;
    unsigned long long* d_nkey = nullptr;
    int32_t* d_cidx = nullptr;
    auto cleanup_tmp = [&]() {
        cudaFreeAsync(d_nkey, s);
        cudaFreeAsync(d_ckey, s);
        cudaFreeAsync(d_cidx, s);
        cudaFreeAsync(d_list, s);
        cudaFreeAsync(d_hist, s);
        cudaFreeAsync(d_ps, s);
    };
#define TRY(x) do { if ((st = (x)) != DOT_OK) { cleanup_tmp(); plan_free(p); return st; } } while (0)
    const int64_t mcap = N / 8 + 1;  // merges never exceed the internal-node count
    TRY(dalloc(&p->state, N, s));
    TRY(dalloc(&p->depth, N, s));
    TRY(dalloc(&p->sig, N, s));
    TRY(dalloc(&p->slot, N, s));
    TRY(dalloc(&p->mround, N, s));
    TRY(dalloc(&p->msig, mcap, s));
    TRY(dalloc(&p->msh, mcap * S, s));
    TRY(dalloc(&d_list, mcap, s));
    TRY(dalloc(&d_hist, 256, s));
    TRY(dalloc(&d_ps, 1, s));
    TRY(check_cuda(cudaMemsetAsync(d_ps, 0, sizeof(PlanScalars), s), "memset"));
    TRY(check_cuda(cudaMemsetAsync(d_hist, 0, 256 * sizeof(unsigned int), s), "memset"));
    TRY(check_cuda(cudaMemcpyToSymbolAsync(c_level_off, off.data(), off.size() * sizeof(int64_t), 0,
                                           cudaMemcpyHostToDevice, s), "memcpy"));
    init_nodes_kernel<<<persistent_blocks(), kTB, 0, s>>>(T, N, n_levels, acc, use_sigma, p->state, p->depth, p->sig,
                                                  p->slot, p->mround, d_ps);
    TRY(check_launch("init_nodes_kernel"));

    // --- prune rounds (device-resident; recursion needs one read per round)
    const unsigned pb = persistent_blocks();
    int rounds = 0;
    unsigned long long merges_done = 0;
    for (int round = 1; recursive >= 0; ++round) {  // recursive < 0: sample only
        TRY(check_cuda(cudaMemsetAsync(&d_ps->round_merges, 0, sizeof(unsigned long long), s), "memset"));
        prune_select_kernel<<<grid_for(N), kTB, 0, s>>>(T, N, tau, p->state, p->sig, d_list, d_ps);
        const int64_t slot_base = int64_t(merges_done);
        merge_sh_kernel<<<pb, kTB, 0, s>>>(T, d_list, d_ps, slot_base, p->state, p->slot, p->msh, S, 3 * B);
        merge_finish_kernel<<<pb, kTB, 0, s>>>(T, d_list, d_ps, slot_base, round, use_sigma, p->state, p->sig,
                                               p->slot, p->mround, p->msig);
        merge_flags_kernel<<<pb, kTB, 0, s>>>(T, d_list, d_ps, slot_base, p->state, p->slot);
        TRY(check_launch("prune round"));
        if (!recursive) {  // one-shot: the count is read with the final scalars below
            rounds = -1;
            break;
        }
        unsigned long long m = 0;
        TRY(check_cuda(cudaMemcpyAsync(&m, &d_ps->round_merges, sizeof(m), cudaMemcpyDeviceToHost, s), "memcpy"));
        TRY(check_cuda(cudaStreamSynchronize(s), "sync"));
        if (m == 0) break;
        merges_done += m;
        rounds = round;
    }

    // --- sample selection, all decisions on the device
    const bool do_sample = use_threshold || gamma > 0.0;
    const bool topk = do_sample && !use_threshold;
    if (topk) {
        TRY(dalloc(&d_nkey, N, s));
        sample_keys_kernel<<<pb, kTB, 0, s>>>(N, p->state, p->depth, p->sig, tree->max_depth, d_nkey, d_hist, d_ps);
        TRY(check_launch("sample_keys_kernel"));
    } else {
        count_leaves_kernel<<<pb, kTB, 0, s>>>(N, p->state, p->depth, p->sig, tree->max_depth, d_ps);
        TRY(check_launch("count_leaves_kernel"));
    }
    if (do_sample) {
        if (use_threshold) {
            mark_split_kernel<<<pb, kTB, 0, s>>>(N, 2, p->state, p->depth, p->sig, tree->max_depth, pool_id,
                                                 threshold, d_ps, nullptr);
        } else {
            sample_k_kernel<<<1, 1, 0, s>>>(d_ps, gamma);
            TRY(dalloc(&d_ckey, N, s));
            TRY(dalloc(&d_cidx, N, s));
            for (int shift = 56; shift >= 0; shift -= 8) {
                // pass 56's histogram came with the keys; after two passes over
                // all nodes only the candidates matching the prefix remain
                const bool cand = shift < 48;
                if (shift == 40)
                    radix_compact_kernel<<<pb, kTB, 0, s>>>(N, d_ps, d_ckey, d_cidx, d_nkey);
                if (shift < 56)
                    radix_hist_kernel<<<pb, kTB, 0, s>>>(N, 0, p->state, p->depth, p->sig, tree->max_depth,
                                                         pool_id, d_ps, shift, d_hist, cand ? d_ckey : nullptr,
                                                         cand ? d_cidx : nullptr, d_nkey);
                radix_pick_kernel<<<1, 32, 0, s>>>(d_ps, 0, d_hist, shift);
            }
            for (int shift = 24; shift >= 0; shift -= 8) {  // ties: all keys equal the k-th, all candidates
                radix_hist_kernel<<<pb, kTB, 0, s>>>(N, 1, p->state, p->depth, p->sig, tree->max_depth, pool_id,
                                                     d_ps, shift, d_hist, d_ckey, d_cidx, d_nkey);
                radix_pick_kernel<<<1, 32, 0, s>>>(d_ps, 1, d_hist, shift);
            }
            mark_split_keys_kernel<<<pb, kTB, 0, s>>>(N, p->state, pool_id, d_ps, d_nkey);
        }
        TRY(check_launch("sample selection"));
    }
    PlanScalars ps;
    TRY(check_cuda(cudaMemcpyAsync(&ps, d_ps, sizeof(ps), cudaMemcpyDeviceToHost, s), "memcpy"));
    TRY(check_cuda(cudaStreamSynchronize(s), "sync"));
    cleanup_tmp();
#undef TRY
    const int64_t M = int64_t(ps.merges);
    const int64_t K = int64_t(ps.splits);
    if (rounds < 0) rounds = M > 0 ? 1 : 0;
    const int64_t leaves_before = (N - int64_t(ps.n_internal));
    p->M = M;
    p->K = K;
    p->stats.leaves_before = leaves_before;
    p->stats.merges_applied = M;
    p->stats.splits_applied = K;
    p->stats.recursion_rounds = rounds;
    p->stats.leaves_after = leaves_before - 7 * M + 7 * K;
    p->stats.n_new_nodes = N - 8 * M + 8 * K;
    *stats = p->stats;
    *out = p;
    return DOT_OK;
}

// Merged-parent and split-leaf lists, built on demand (ordered compaction on
// the device, one download).  Merges come in the reference's event order:
// by round, then by index.
int dot_refine_plan_lists(dot_refine_plan* p, const int64_t** merge_parents, int64_t* n_merge,
                          const int64_t** split_leaves, int64_t* n_split, const int32_t** merge_round,
                          void* stream) {
    if (!p) return set_error(DOT_BAD_ARG, "NULL plan");
    if (!p->lists_ready) {
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const int64_t N = p->N;
        int32_t* flags = nullptr;
        int64_t *rank = nullptr, *total = nullptr, *list = nullptr;
        int32_t* rounds = nullptr;
        int st = DOT_OK;
        auto cleanup = [&]() {
            cudaFreeAsync(flags, s);
            cudaFreeAsync(rank, s);
            cudaFreeAsync(total, s);
            cudaFreeAsync(list, s);
        };
#define TRY(x) do { if ((st = (x)) != DOT_OK) { cleanup(); return st; } } while (0)
        TRY(dalloc(&flags, N, s));
        TRY(dalloc(&rank, N, s));
        TRY(dalloc(&total, 1, s));
        TRY(dalloc(&list, std::max<int64_t>(p->M, p->K) + 1, s));
        for (int which = 0; which < 2; ++which) {
            const int64_t cnt = which == 0 ? p->M : p->K;
            std::vector<int64_t>& dst = which == 0 ? p->merge_list : p->split_list;
            dst.resize(size_t(cnt));
            if (cnt == 0) continue;
            flag_kernel<<<grid_for(N), kTB, 0, s>>>(N, p->state, p->mround, which, flags);
            TRY(exclusive_scan(flags, N, rank, total, s));
            compact_kernel<<<grid_for(N), kTB, 0, s>>>(N, flags, rank, list);
            TRY(check_launch("compact_kernel"));
            TRY(check_cuda(cudaMemcpyAsync(dst.data(), list, cnt * sizeof(int64_t), cudaMemcpyDeviceToHost, s),
                           "memcpy"));
        }
        std::vector<int32_t> mr(size_t(p->M));
        if (p->M) {
            TRY(dalloc(&rounds, p->M, s));
            // gather the rounds of the merged nodes
            std::vector<int32_t> all(static_cast<size_t>(N));
            TRY(check_cuda(cudaMemcpyAsync(all.data(), p->mround, N * sizeof(int32_t), cudaMemcpyDeviceToHost, s),
                           "memcpy"));
            TRY(check_cuda(cudaStreamSynchronize(s), "sync"));
            cudaFreeAsync(rounds, s);
            for (int64_t i = 0; i < p->M; ++i) mr[size_t(i)] = all[size_t(p->merge_list[size_t(i)])];
            std::vector<size_t> idx(size_t(p->M));
            for (size_t i = 0; i < idx.size(); ++i) idx[i] = i;
            std::stable_sort(idx.begin(), idx.end(), [&](size_t a, size_t b) { return mr[a] < mr[b]; });
            std::vector<int64_t> ml(idx.size());
            p->merge_round_h.resize(idx.size());
            for (size_t i = 0; i < idx.size(); ++i) {
                ml[i] = p->merge_list[idx[i]];
                p->merge_round_h[i] = mr[idx[i]];
            }
            p->merge_list.swap(ml);
        }
        TRY(check_cuda(cudaStreamSynchronize(s), "sync"));
        cleanup();
#undef TRY
        p->lists_ready = true;
    }
    if (merge_parents) *merge_parents = p->merge_list.data();
    if (n_merge) *n_merge = p->M;
    if (split_leaves) *split_leaves = p->split_list.data();
    if (n_split) *n_split = p->K;
    if (merge_round) *merge_round = p->merge_round_h.data();
    return DOT_OK;
}

int dot_refine_apply(const dot_refine_plan* p, const dot_tree_view* tree, int32_t* new_node,
                     float* new_sigma, float* new_sh, int64_t* src_index, uint8_t* src_kind,
                     int64_t* level_offsets_out, int32_t max_levels, int32_t* n_levels_out,
                     void* stream) {
    if (!p || !tree) return set_error(DOT_BAD_ARG, "NULL argument");
    if (!new_node || !new_sigma || !new_sh || !src_index || !src_kind)
        return set_error(DOT_BAD_ARG, "refine outputs must not be NULL");
    if ((reinterpret_cast<uintptr_t>(new_sh) & 15) != 0) return set_error(DOT_BAD_ARG, "new_sh must be 16-byte aligned");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const TreeDev T = make_tree(*tree);
    const int64_t n_new = p->stats.n_new_nodes;
    int st = DOT_OK;
    const int64_t N = p->N;
    const int n_levels = int(p->level_off.size()) - 1;
    if (n_levels + 2 > kMaxLevels) return set_error(DOT_BAD_ARG, "tree too deep");
    int32_t* flags = nullptr;
    int64_t *rank = nullptr, *d_total = nullptr, *d_base = nullptr, *d_rb = nullptr;
    auto cleanup = [&]() {
        cudaFreeAsync(flags, s);
        cudaFreeAsync(rank, s);
        cudaFreeAsync(d_total, s);
        cudaFreeAsync(d_base, s);
        cudaFreeAsync(d_rb, s);
    };
#define TRY(x) do { if ((st = (x)) != DOT_OK) { cleanup(); return st; } } while (0)
    TRY(dalloc(&flags, N, s));
    TRY(dalloc(&rank, N, s));
    TRY(dalloc(&d_total, 1, s));
    TRY(dalloc(&d_base, kMaxLevels + 2, s));
    TRY(dalloc(&d_rb, kMaxLevels + 2, s));
    TRY(check_cuda(cudaMemcpyToSymbolAsync(c_level_off, p->level_off.data(),
                                           p->level_off.size() * sizeof(int64_t), 0,
                                           cudaMemcpyHostToDevice, s), "memcpy"));
    rebuild_flags_kernel<<<persistent_blocks(), kTB, 0, s>>>(N, p->state, flags);
    TRY(check_launch("rebuild_flags_kernel"));
    TRY(exclusive_scan(flags, N, rank, d_total, s));
    rebuild_levels_kernel<<<1, 1, 0, s>>>(n_levels, rank, d_total, d_base, d_rb);
    rebuild_emit_kernel<<<grid_for(N), kTB, 0, s>>>(T, N, p->state, p->depth, flags, rank, d_base, d_rb,
                                                    new_node, src_index, src_kind);
    TRY(check_launch("rebuild_emit_kernel"));
    std::vector<int64_t> nb(size_t(n_levels) + 2);
    TRY(check_cuda(cudaMemcpyAsync(nb.data(), d_base, nb.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, s),
                   "memcpy"));
    {
        const unsigned grid = grid_for(((n_new + 31) / 32) * 32);
        float4* nsh = reinterpret_cast<float4*>(new_sh);
#define DOT_PAYLOAD(S4V)                                                                              \
        payload_kernel<S4V><<<grid, kTB, 0, s>>>(T, n_new, src_index, p->state, p->slot, p->msig, p->msh, \
                                                 new_node, new_sigma, nsh)
        switch (p->S / 4) {
            case 1: DOT_PAYLOAD(1); break;
            case 3: DOT_PAYLOAD(3); break;
            case 7: DOT_PAYLOAD(7); break;
            case 12: DOT_PAYLOAD(12); break;
            default: TRY(set_error(DOT_BAD_ARG, "unsupported SH row width %d", p->S));
        }
#undef DOT_PAYLOAD
        TRY(check_launch("payload_kernel"));
    }
    TRY(check_cuda(cudaStreamSynchronize(s), "sync"));
    cleanup();
#undef TRY
    // new level offsets: nb[0..n_levels+1]; the last level may be empty
    std::vector<int64_t> offs;
    for (int L = 0; L <= n_levels + 1; ++L) {
        if (L > 0 && nb[size_t(L)] == nb[size_t(L) - 1]) break;
        offs.push_back(nb[size_t(L)]);
    }
    const int levels = int(offs.size()) - 1;
    if (offs.back() != n_new)
        return set_error(DOT_CUDA_ERR, "refine apply produced %lld nodes, plan said %lld",
                         (long long)offs.back(), (long long)n_new);
    if (n_levels_out) *n_levels_out = levels;
    if (level_offsets_out)
        for (int i = 0; i < int(offs.size()) && i < max_levels + 1; ++i) level_offsets_out[i] = offs[size_t(i)];
    return DOT_OK;
}

int dot_refine_plan_merge_rounds(const dot_refine_plan* p, int32_t* out, void* stream) {
    if (!p || !out) return set_error(DOT_BAD_ARG, "NULL argument");
    return check_cuda(cudaMemcpyAsync(out, p->mround, p->N * sizeof(int32_t), cudaMemcpyDeviceToDevice,
                                      static_cast<cudaStream_t>(stream)),
                      "memcpy");
}

void dot_refine_plan_destroy(dot_refine_plan* plan) { plan_free(plan); }

}  // extern "C"
