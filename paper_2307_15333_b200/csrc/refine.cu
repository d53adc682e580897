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
//    pool ids for the ties at the k-th value.
//  * the refined tree is emitted directly in canonical BFS order
//    (scene_io.py:529-541), level by level: one flag scan per level decides
//    which nodes are internal, children are either the old children (kept)
//    or 8 payload copies of a split leaf (octree.py:216-248).
// The reference instead mutates a pooled tree through a LIFO free list and
// only canonicalises on save; topologies are compared after canonicalisation.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <algorithm>
#include <cmath>
#include <vector>
#include "dot_tree.cuh"
#include "dot_internal.h"

namespace dot {

enum : uint8_t { ST_ALIVE = 1, ST_LEAF = 2, ST_MERGED = 4, ST_SPLIT = 8 };
enum : uint8_t { K_KEPT = 0, K_MERGED = 1, K_NEWCHILD = 2, K_SPLITPARENT = 3 };

constexpr int kTB = 256;

static unsigned grid_for(int64_t n, int tb = kTB) {
    return unsigned((n + tb - 1) / tb);
}

// ---------------------------------------------------------------------------
// Small scan utility: exclusive scan of int32 values (3 phases, cub block scans).

constexpr int kScanItems = 4;
constexpr int kScanTile = kTB * kScanItems;

__global__ void scan_reduce_kernel(const int32_t* __restrict__ in, int64_t n, int64_t* __restrict__ sums) {
    using BR = cub::BlockReduce<int64_t, kTB>;
    __shared__ typename BR::TempStorage tmp;
    const int64_t base = int64_t(blockIdx.x) * kScanTile;
    int64_t v = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        const int64_t idx = base + threadIdx.x * kScanItems + i;
        if (idx < n) v += in[idx];
    }
    const int64_t s = BR(tmp).Sum(v);
    if (threadIdx.x == 0) sums[blockIdx.x] = s;
}

__global__ void scan_sums_kernel(int64_t* __restrict__ sums, int64_t nb, int64_t* __restrict__ total) {
    // single block, sequential chunks of kTB
    using BS = cub::BlockScan<int64_t, kTB>;
    __shared__ typename BS::TempStorage tmp;
    __shared__ int64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t b = 0; b < nb; b += kTB) {
        const int64_t idx = b + threadIdx.x;
        int64_t v = idx < nb ? sums[idx] : 0, agg;
        int64_t ex;
        BS(tmp).ExclusiveSum(v, ex, agg);
        if (idx < nb) sums[idx] = ex + carry;
        __syncthreads();
        if (threadIdx.x == 0) carry += agg;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = carry;
}

__global__ void scan_apply_kernel(const int32_t* __restrict__ in, int64_t n,
                                  const int64_t* __restrict__ sums, int64_t* __restrict__ out) {
    using BS = cub::BlockScan<int64_t, kTB>;
    __shared__ typename BS::TempStorage tmp;
    const int64_t base = int64_t(blockIdx.x) * kScanTile;
    int64_t v[kScanItems];
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        const int64_t idx = base + threadIdx.x * kScanItems + i;
        v[i] = idx < n ? in[idx] : 0;
    }
    BS(tmp).ExclusiveSum(v, v);
    const int64_t off = sums[blockIdx.x];
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        const int64_t idx = base + threadIdx.x * kScanItems + i;
        if (idx < n) out[idx] = v[i] + off;
    }
}

// Exclusive scan of in[0..n) into out; *d_total receives the sum.  Scratch
// `sums` must hold ceil(n / kScanTile) + 1 entries.
static int exclusive_scan(const int32_t* in, int64_t n, int64_t* out, int64_t* sums,
                          int64_t* d_total, cudaStream_t s) {
    const int64_t nb = (n + kScanTile - 1) / kScanTile;
    if (nb == 0) return check_cuda(cudaMemsetAsync(d_total, 0, sizeof(int64_t), s), "memset");
    scan_reduce_kernel<<<unsigned(nb), kTB, 0, s>>>(in, n, sums);
    scan_sums_kernel<<<1, kTB, 0, s>>>(sums, nb, d_total);
    scan_apply_kernel<<<unsigned(nb), kTB, 0, s>>>(in, n, sums, out);
    return check_launch("exclusive_scan");
}

// ---------------------------------------------------------------------------
// Plan state

struct RadixState {
    unsigned long long prefix;  // selected high bits so far
    unsigned long long mask;    // which bits are fixed
    long long remaining;        // how many still to take at/below the prefix
    long long eq_count;         // count of keys equal to the final prefix
};

}  // namespace dot

struct dot_refine_plan {
    int64_t N = 0;
    int S = 0;
    int B = 0;
    bool use_sigma = false;
    // device arrays (canonical old index space)
    uint8_t* state = nullptr;
    uint8_t* depth = nullptr;
    double* sig = nullptr;
    int32_t* slot = nullptr;
    int32_t* mround = nullptr;   // merge round (1-based) or 0
    const int32_t* pool_id = nullptr;  // caller-owned, may be NULL (identity)
    float* msig = nullptr;       // merged payload [M]
    float* msh = nullptr;        // merged SH [M * S]
    int64_t M = 0, K = 0;
    int64_t* merge_list = nullptr;  // host, canonical ascending
    int32_t* merge_round_h = nullptr;
    int64_t* split_list = nullptr;  // host, canonical ascending
    dot_refine_stats stats{};
    int32_t max_depth = 0;
};

namespace dot {

__device__ __forceinline__ int32_t pid_of(const int32_t* pool_id, int64_t i) {
    return pool_id ? pool_id[i] : int32_t(i);
}

// state / depth / sig initialisation for one BFS level [s, e).
__global__ void init_level_kernel(TreeDev T, int64_t s, int64_t e, int d, const double* __restrict__ acc,
                                  int use_sigma, uint8_t* __restrict__ state, uint8_t* __restrict__ depth,
                                  double* __restrict__ sig, int32_t* __restrict__ slot,
                                  int32_t* __restrict__ mround, int* __restrict__ n_internal) {
    const int64_t i = s + int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    int internal = 0;
    if (i < e) {
        const int32_t w = T.node[i];
        depth[i] = uint8_t(d);
        slot[i] = -1;
        mround[i] = 0;
        if (w < 0) {
            state[i] = ST_ALIVE | ST_LEAF;
            const int32_t pid = ~w;
            sig[i] = use_sigma ? double(T.sigma[pid]) : acc[pid];
        } else {
            state[i] = ST_ALIVE;
            sig[i] = 0.0;
            internal = 1;
        }
    }
    internal = __syncthreads_count(internal);
    if (threadIdx.x == 0 && internal) atomicAdd(n_internal, internal);
}

// Prune selection for one round: alive internal nodes whose 8 children are
// leaves with signal <= tau.  Selected ids are appended (unordered).
__global__ void prune_select_kernel(TreeDev T, int64_t N, double tau, const uint8_t* __restrict__ state,
                                    const double* __restrict__ sig, int64_t* __restrict__ list,
                                    unsigned long long* __restrict__ count) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const uint8_t st = state[i];
    if ((st & ST_ALIVE) == 0 || (st & ST_LEAF)) return;
    const int32_t c = T.node[i];
    bool ok = true;
#pragma unroll
    for (int o = 0; o < 8; ++o) {
        if ((state[c + o] & ST_LEAF) == 0 || !(sig[c + o] <= tau)) ok = false;
    }
    if (ok) list[atomicAdd(count, 1ull)] = i;
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

// Apply one round of merges: fp64 mean payload (sigma pairwise, SH
// sequential), pairwise signal sum, topology flags.  One thread per parent
// for sigma/signal/flags; SH columns handled by the column loop.
__global__ void merge_apply_kernel(TreeDev T, const int64_t* __restrict__ list, int64_t m, int64_t slot_base,
                                   int round, int use_sigma, uint8_t* __restrict__ state,
                                   double* __restrict__ sig, int32_t* __restrict__ slot,
                                   int32_t* __restrict__ mround, float* __restrict__ msig,
                                   float* __restrict__ msh, int S, int nsh) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= m) return;
    const int64_t p = list[j];
    const int32_t c = T.node[p];
    const int64_t sl = slot_base + j;
    double s8[8], q8[8];
#pragma unroll
    for (int o = 0; o < 8; ++o) {
        s8[o] = double(leaf_sigma(T, msig, slot, state, c + o));
        q8[o] = sig[c + o];
    }
    const double ssum = ((s8[0] + s8[1]) + (s8[2] + s8[3])) + ((s8[4] + s8[5]) + (s8[6] + s8[7]));
    const float mean_sigma = float(ssum / 8.0);
    msig[sl] = mean_sigma;
    const double qsum = ((q8[0] + q8[1]) + (q8[2] + q8[3])) + ((q8[4] + q8[5]) + (q8[6] + q8[7]));
    const float* rows[8];
#pragma unroll
    for (int o = 0; o < 8; ++o) rows[o] = leaf_row_sh(T, msh, slot, state, c + o, S);
    float* out = msh + sl * S;
    for (int k = 0; k < S; ++k) {
        if (k < nsh) {
            double acc = double(rows[0][k]);
#pragma unroll
            for (int o = 1; o < 8; ++o) acc = acc + double(rows[o][k]);
            out[k] = float(acc / 8.0);
        } else {
            out[k] = 0.f;
        }
    }
    // children leave the topology; parent becomes a (merged) leaf
#pragma unroll
    for (int o = 0; o < 8; ++o) state[c + o] &= uint8_t(~ST_ALIVE);
    sig[p] = use_sigma ? double(mean_sigma) : qsum;
    slot[p] = int32_t(sl);
    mround[p] = round;
    state[p] |= ST_LEAF | ST_MERGED;
}

// Leaf / eligibility counts on the post-prune topology.
__global__ void count_leaves_kernel(int64_t N, const uint8_t* __restrict__ state,
                                    const uint8_t* __restrict__ depth, const double* __restrict__ sig,
                                    int max_depth, int use_thr, double thr,
                                    unsigned long long* __restrict__ counts) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    int leaf = 0, elig = 0;
    if (i < N) {
        const uint8_t st = state[i];
        if ((st & ST_ALIVE) && (st & ST_LEAF)) {
            leaf = 1;
            const double s = sig[i];
            if (depth[i] < max_depth && s > 0.0 && (!use_thr || s > thr)) elig = 1;
        }
    }
    leaf = __syncthreads_count(leaf);
    elig = __syncthreads_count(elig);
    if (threadIdx.x == 0) {
        if (leaf) atomicAdd(counts + 0, (unsigned long long)leaf);
        if (elig) atomicAdd(counts + 1, (unsigned long long)elig);
    }
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

// Histogram of digit `shift` over keys matching the current prefix.
// mode 0: signal keys; mode 1: tie keys (0xFFFFFFFF - pool id) among keys == K*.
__global__ void radix_hist_kernel(int64_t N, int mode, const uint8_t* __restrict__ state,
                                  const uint8_t* __restrict__ depth, const double* __restrict__ sig,
                                  int max_depth, const int32_t* __restrict__ pool_id,
                                  const RadixState* __restrict__ rs, const RadixState* __restrict__ rs0,
                                  int shift, unsigned int* __restrict__ hist) {
    __shared__ unsigned int h[256];
    for (int b = threadIdx.x; b < 256; b += blockDim.x) h[b] = 0;
    __syncthreads();
    const unsigned long long prefix = rs->prefix, mask = rs->mask;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < N; i += stride) {
        unsigned long long key = sample_key(i, state, depth, sig, max_depth);
        if (key == 0ull) continue;
        if (mode == 1) {
            if (key != rs0->prefix) continue;
            key = 0xFFFFFFFFull - (unsigned long long)(uint32_t)pid_of(pool_id, i);
        }
        if ((key & mask) != prefix) continue;
        atomicAdd(&h[(key >> shift) & 0xFF], 1u);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < 256; b += blockDim.x)
        if (h[b]) atomicAdd(hist + b, h[b]);
}

__global__ void radix_pick_kernel(RadixState* rs, unsigned int* hist, int shift) {
    // one thread: walk digits from the top until `remaining` falls inside a bin
    if (threadIdx.x != 0) return;
    long long rem = rs->remaining;
    int digit = 0;
    for (int b = 255; b >= 0; --b) {
        const long long c = hist[b];
        if (rem <= c) { digit = b; rs->eq_count = c; break; }
        rem -= c;
    }
    rs->remaining = rem;
    rs->prefix |= (unsigned long long)digit << shift;
    rs->mask |= 0xFFull << shift;
    for (int b = 0; b < 256; ++b) hist[b] = 0;
}

// Mark the sample selection: key > K*, plus ties (key == K*) whose tie key
// >= T* (i.e. pool id <= the m-th smallest), or threshold mode.
__global__ void mark_split_kernel(int64_t N, int mode, uint8_t* __restrict__ state,
                                  const uint8_t* __restrict__ depth, const double* __restrict__ sig,
                                  int max_depth, const int32_t* __restrict__ pool_id, double thr,
                                  unsigned long long kstar, int take_all_ties,
                                  unsigned long long tstar) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const unsigned long long key = sample_key(i, state, depth, sig, max_depth);
    if (key == 0ull) return;
    bool sel;
    if (mode == 2) {
        sel = sig[i] > thr;
    } else {
        sel = key > kstar;
        if (key == kstar) {
            const unsigned long long tk = 0xFFFFFFFFull - (unsigned long long)(uint32_t)pid_of(pool_id, i);
            sel = take_all_ties || tk >= tstar;
        }
    }
    if (sel) state[i] |= ST_SPLIT;
}

__global__ void collect_kernel(int64_t N, const uint8_t* __restrict__ state, uint8_t bit,
                               int64_t* __restrict__ list, unsigned long long* __restrict__ count) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= N) return;
    if (state[i] & bit) list[atomicAdd(count, 1ull)] = i;
}

// ---------------------------------------------------------------------------
// Apply: level-synchronous canonical rebuild.

__global__ void level_flags_kernel(int64_t m, const int32_t* __restrict__ ent_old,
                                   const uint8_t* __restrict__ ent_kind, const uint8_t* __restrict__ state,
                                   int32_t* __restrict__ flags) {
    const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= m) return;
    int internal = 0;
    if (ent_kind[e] != K_NEWCHILD) {
        const uint8_t st = state[ent_old[e]];
        internal = (!(st & ST_LEAF)) || (st & ST_SPLIT) ? 1 : 0;
    }
    flags[e] = internal;
}

__global__ void level_emit_kernel(TreeDev T, int64_t m, int64_t base, int64_t next_base,
                                  const int32_t* __restrict__ ent_old, const uint8_t* __restrict__ ent_kind,
                                  const int32_t* __restrict__ flags, const int64_t* __restrict__ rank,
                                  const uint8_t* __restrict__ state, int32_t* __restrict__ new_node,
                                  int64_t* __restrict__ src_index, uint8_t* __restrict__ src_kind,
                                  int32_t* __restrict__ nxt_old, uint8_t* __restrict__ nxt_kind) {
    const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= m) return;
    const int64_t gi = base + e;
    const int32_t o = ent_old[e];
    const uint8_t kind = ent_kind[e];
    src_index[gi] = o;
    if (flags[e]) {
        const int64_t r = rank[e];
        new_node[gi] = int32_t(next_base + 8 * r);
        const uint8_t st = state[o];
        const bool from_leaf = (st & ST_LEAF) != 0;  // split of an (original or merged) leaf
        src_kind[gi] = from_leaf ? K_SPLITPARENT : K_KEPT;
        const int32_t c = T.node[o];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            nxt_old[8 * r + k] = from_leaf ? o : c + k;
            nxt_kind[8 * r + k] = from_leaf ? K_NEWCHILD : K_KEPT;
        }
    } else {
        new_node[gi] = ~int32_t(gi);
        if (kind == K_NEWCHILD) src_kind[gi] = K_NEWCHILD;
        else src_kind[gi] = (state[o] & ST_MERGED) ? K_MERGED : K_KEPT;
    }
}

// Payload gather: one thread per (new node, float4 column).
__global__ void payload_kernel(TreeDev T, int64_t n_new, int S4, const int64_t* __restrict__ src_index,
                               const uint8_t* __restrict__ src_kind, const uint8_t* __restrict__ state,
                               const int32_t* __restrict__ slot, const float* __restrict__ msig,
                               const float* __restrict__ msh, const int32_t* __restrict__ new_node,
                               float* __restrict__ new_sigma, float4* __restrict__ new_sh) {
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= n_new * S4) return;
    const int64_t i = t / S4;
    const int j = int(t - i * S4);
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    float sg = 0.f;
    if (new_node[i] < 0) {  // leaf in the new tree
        const int64_t o = src_index[i];
        if (state[o] & ST_MERGED) {
            const int32_t sl = slot[o];
            v = reinterpret_cast<const float4*>(msh)[int64_t(sl) * S4 + j];
            sg = msig[sl];
        } else {
            const int32_t pid = ~T.node[o];
            v = __ldg(reinterpret_cast<const float4*>(T.sh) + int64_t(pid) * S4 + j);
            sg = __ldg(T.sigma + pid);
        }
    }
    new_sh[t] = v;
    if (j == 0) new_sigma[i] = sg;
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
    delete[] p->merge_list;
    delete[] p->merge_round_h;
    delete[] p->split_list;
    delete p;
}

extern "C" {

int dot_refine_plan_create(const dot_tree_view* tree, const int32_t* pool_id, const double* acc,
                           int32_t use_sigma, double tau, double gamma, int32_t recursive,
                           int32_t use_threshold, double threshold, dot_refine_plan** out,
                           dot_refine_stats* stats, void* stream) {
    if (!tree || !out || !stats) return set_error(DOT_BAD_ARG, "NULL argument");
    if (!use_sigma && !acc) return set_error(DOT_BAD_ARG, "acc must not be NULL for the Q target");
    if (tau < 0.0) return set_error(DOT_BAD_ARG, "tau must be >= 0, got %g", tau);
    if (!(gamma >= 0.0 && gamma <= 1.0)) return set_error(DOT_BAD_ARG, "gamma must be in [0, 1]");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const TreeDev T = make_tree(*tree);
    const int64_t N = tree->n_nodes;
    const int S = tree->sh_stride, B = tree->basis_count;
    dot_refine_plan* p = new dot_refine_plan();
    p->N = N;
    p->S = S;
    p->B = B;
    p->use_sigma = use_sigma != 0;
    p->pool_id = pool_id;
    p->max_depth = tree->max_depth;
    int st = DOT_OK;
#define TRY(x) do { if ((st = (x)) != DOT_OK) { plan_free(p); return st; } } while (0)
    TRY(dalloc(&p->state, N, s));
    TRY(dalloc(&p->depth, N, s));
    TRY(dalloc(&p->sig, N, s));
    TRY(dalloc(&p->slot, N, s));
    TRY(dalloc(&p->mround, N, s));
    int64_t* d_list = nullptr;
    unsigned long long* d_cnt = nullptr;
    int* d_int = nullptr;
    unsigned int* d_hist = nullptr;
    RadixState* d_rs = nullptr;
    TRY(dalloc(&d_list, N, s));
    TRY(dalloc(&d_cnt, 4, s));
    TRY(dalloc(&d_int, 1, s));
    TRY(dalloc(&d_hist, 256, s));
    TRY(dalloc(&d_rs, 2, s));
    auto cleanup_tmp = [&]() {
        cudaFreeAsync(d_list, s);
        cudaFreeAsync(d_cnt, s);
        cudaFreeAsync(d_int, s);
        cudaFreeAsync(d_hist, s);
        cudaFreeAsync(d_rs, s);
    };
#undef TRY
#define TRY(x) do { if ((st = (x)) != DOT_OK) { cleanup_tmp(); plan_free(p); return st; } } while (0)

    // --- levels: depth, state, signal
    int64_t lo = 0, hi = 1;
    int d = 0;
    int64_t leaves_before = 0;
    while (lo < hi) {
        if (d > 255) TRY(set_error(DOT_BAD_ARG, "tree deeper than 255 levels"));
        TRY(check_cuda(cudaMemsetAsync(d_int, 0, sizeof(int), s), "memset"));
        init_level_kernel<<<grid_for(hi - lo), kTB, 0, s>>>(T, lo, hi, d, acc, use_sigma, p->state, p->depth,
                                                            p->sig, p->slot, p->mround, d_int);
        TRY(check_launch("init_level_kernel"));
        int n_int = 0;
        TRY(check_cuda(cudaMemcpyAsync(&n_int, d_int, sizeof(int), cudaMemcpyDeviceToHost, s), "memcpy"));
        TRY(check_cuda(cudaStreamSynchronize(s), "sync"));
        leaves_before += (hi - lo) - n_int;
        lo = hi;
        hi = hi + 8 * int64_t(n_int);
        ++d;
    }
    if (hi != N) TRY(set_error(DOT_BAD_ARG, "node table is not a canonical BFS tree (%lld reachable of %lld)",
                               (long long)hi, (long long)N));

    // --- prune rounds
    std::vector<int64_t> merges;
    std::vector<int32_t> merge_rounds;
    int rounds = 0;
    // merged payload buffer grows per round
    int64_t mcap = 0;
    for (; recursive >= 0;) {  // recursive < 0: sample only, no prune
        TRY(check_cuda(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long), s), "memset"));
        prune_select_kernel<<<grid_for(N), kTB, 0, s>>>(T, N, tau, p->state, p->sig, d_list, d_cnt);
        TRY(check_launch("prune_select_kernel"));
        unsigned long long m = 0;
        TRY(check_cuda(cudaMemcpyAsync(&m, d_cnt, sizeof(m), cudaMemcpyDeviceToHost, s), "memcpy"));
        TRY(check_cuda(cudaStreamSynchronize(s), "sync"));
        if (m == 0) break;
        const int64_t base = int64_t(merges.size());
        if (base + int64_t(m) > mcap) {
            const int64_t ncap = std::max<int64_t>(2 * mcap, base + int64_t(m));
            float *ns = nullptr, *nh = nullptr;
            TRY(dalloc(&ns, ncap, s));
            TRY(dalloc(&nh, ncap * S, s));
            if (base) {
                TRY(check_cuda(cudaMemcpyAsync(ns, p->msig, base * sizeof(float), cudaMemcpyDeviceToDevice, s), "copy"));
                TRY(check_cuda(cudaMemcpyAsync(nh, p->msh, base * S * sizeof(float), cudaMemcpyDeviceToDevice, s), "copy"));
            }
            if (p->msig) cudaFreeAsync(p->msig, s);
            if (p->msh) cudaFreeAsync(p->msh, s);
            p->msig = ns;
            p->msh = nh;
            mcap = ncap;
        }
        ++rounds;
        merge_apply_kernel<<<grid_for(int64_t(m)), kTB, 0, s>>>(T, d_list, int64_t(m), base, rounds, use_sigma,
                                                                 p->state, p->sig, p->slot, p->mround,
                                                                 p->msig, p->msh, S, 3 * B);
        TRY(check_launch("merge_apply_kernel"));
        std::vector<int64_t> h(m);
        TRY(check_cuda(cudaMemcpyAsync(h.data(), d_list, m * sizeof(int64_t), cudaMemcpyDeviceToHost, s), "memcpy"));
        TRY(check_cuda(cudaStreamSynchronize(s), "sync"));
        merges.insert(merges.end(), h.begin(), h.end());
        merge_rounds.insert(merge_rounds.end(), m, rounds);
        if (!recursive) break;
    }
    const int64_t M = int64_t(merges.size());

    // --- sample selection
    TRY(check_cuda(cudaMemsetAsync(d_cnt, 0, 4 * sizeof(unsigned long long), s), "memset"));
    count_leaves_kernel<<<grid_for(N), kTB, 0, s>>>(N, p->state, p->depth, p->sig, tree->max_depth,
                                                    use_threshold, threshold, d_cnt);
    TRY(check_launch("count_leaves_kernel"));
    unsigned long long cnt[2] = {0, 0};
    TRY(check_cuda(cudaMemcpyAsync(cnt, d_cnt, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s), "memcpy"));
    TRY(check_cuda(cudaStreamSynchronize(s), "sync"));
    const int64_t L = int64_t(cnt[0]), n_elig = int64_t(cnt[1]);
    int64_t k = 0;
    const bool do_sample = use_threshold || gamma > 0.0;
    if (do_sample) {
        if (use_threshold) {
            k = n_elig;
            if (k > 0) {
                mark_split_kernel<<<grid_for(N), kTB, 0, s>>>(N, 2, p->state, p->depth, p->sig, tree->max_depth,
                                                              pool_id, threshold, 0ull, 0, 0ull);
                TRY(check_launch("mark_split_kernel"));
            }
        } else {
            k = std::min<int64_t>(int64_t(std::ceil(gamma * double(L))), n_elig);
            if (k > 0) {
                const int hist_grid = 4 * 148;
                RadixState r0{0ull, 0ull, (long long)k, 0};
                TRY(check_cuda(cudaMemcpyAsync(d_rs, &r0, sizeof(r0), cudaMemcpyHostToDevice, s), "memcpy"));
                TRY(check_cuda(cudaMemsetAsync(d_hist, 0, 256 * sizeof(unsigned int), s), "memset"));
                for (int shift = 56; shift >= 0; shift -= 8) {
                    radix_hist_kernel<<<hist_grid, kTB, 0, s>>>(N, 0, p->state, p->depth, p->sig, tree->max_depth,
                                                                pool_id, d_rs, d_rs, shift, d_hist);
                    radix_pick_kernel<<<1, 32, 0, s>>>(d_rs, d_hist, shift);
                }
                TRY(check_launch("radix select (signal)"));
                RadixState r1;
                TRY(check_cuda(cudaMemcpyAsync(&r1, d_rs, sizeof(r1), cudaMemcpyDeviceToHost, s), "memcpy"));
                TRY(check_cuda(cudaStreamSynchronize(s), "sync"));
                const unsigned long long kstar = r1.prefix;
                const bool all_ties = r1.remaining == r1.eq_count;
                unsigned long long tstar = 0ull;
                if (!all_ties) {
                    RadixState t0{0ull, 0xFFFFFFFF00000000ull, r1.remaining, 0};
                    TRY(check_cuda(cudaMemcpyAsync(d_rs + 1, &t0, sizeof(t0), cudaMemcpyHostToDevice, s), "memcpy"));
                    for (int shift = 24; shift >= 0; shift -= 8) {
                        radix_hist_kernel<<<hist_grid, kTB, 0, s>>>(N, 1, p->state, p->depth, p->sig,
                                                                    tree->max_depth, pool_id, d_rs + 1, d_rs,
                                                                    shift, d_hist);
                        radix_pick_kernel<<<1, 32, 0, s>>>(d_rs + 1, d_hist, shift);
                    }
                    TRY(check_launch("radix select (ties)"));
                    RadixState t1;
                    TRY(check_cuda(cudaMemcpyAsync(&t1, d_rs + 1, sizeof(t1), cudaMemcpyDeviceToHost, s), "memcpy"));
                    TRY(check_cuda(cudaStreamSynchronize(s), "sync"));
                    tstar = t1.prefix;
                }
                mark_split_kernel<<<grid_for(N), kTB, 0, s>>>(N, 0, p->state, p->depth, p->sig, tree->max_depth,
                                                              pool_id, 0.0, kstar, all_ties ? 1 : 0, tstar);
                TRY(check_launch("mark_split_kernel"));
            }
        }
    }
    // collect split list (ascending canonical index)
    int64_t K = 0;
    std::vector<int64_t> splits;
    if (k > 0) {
        TRY(check_cuda(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long), s), "memset"));
        collect_kernel<<<grid_for(N), kTB, 0, s>>>(N, p->state, ST_SPLIT, d_list, d_cnt);
        TRY(check_launch("collect_kernel"));
        unsigned long long kk = 0;
        TRY(check_cuda(cudaMemcpyAsync(&kk, d_cnt, sizeof(kk), cudaMemcpyDeviceToHost, s), "memcpy"));
        TRY(check_cuda(cudaStreamSynchronize(s), "sync"));
        K = int64_t(kk);
        splits.resize(K);
        TRY(check_cuda(cudaMemcpyAsync(splits.data(), d_list, K * sizeof(int64_t), cudaMemcpyDeviceToHost, s), "memcpy"));
        TRY(check_cuda(cudaStreamSynchronize(s), "sync"));
        std::sort(splits.begin(), splits.end());
    }
    cleanup_tmp();
#undef TRY

    // merge list sorted by (round, index) -- the reference's event order
    std::vector<size_t> idx(M);
    for (int64_t i = 0; i < M; ++i) idx[i] = size_t(i);
    std::sort(idx.begin(), idx.end(), [&](size_t a, size_t b) {
        return merge_rounds[a] != merge_rounds[b] ? merge_rounds[a] < merge_rounds[b] : merges[a] < merges[b];
    });
    p->M = M;
    p->K = K;
    p->merge_list = new int64_t[M ? M : 1];
    p->merge_round_h = new int32_t[M ? M : 1];
    for (int64_t i = 0; i < M; ++i) {
        p->merge_list[i] = merges[idx[i]];
        p->merge_round_h[i] = merge_rounds[idx[i]];
    }
    p->split_list = new int64_t[K ? K : 1];
    for (int64_t i = 0; i < K; ++i) p->split_list[i] = splits[i];
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

int dot_refine_plan_lists(const dot_refine_plan* plan, const int64_t** merge_parents, int64_t* n_merge,
                          const int64_t** split_leaves, int64_t* n_split, const int32_t** merge_round) {
    if (!plan) return set_error(DOT_BAD_ARG, "NULL plan");
    if (merge_parents) *merge_parents = plan->merge_list;
    if (n_merge) *n_merge = plan->M;
    if (split_leaves) *split_leaves = plan->split_list;
    if (n_split) *n_split = plan->K;
    if (merge_round) *merge_round = plan->merge_round_h;
    return DOT_OK;
}

int dot_refine_apply(const dot_refine_plan* p, const dot_tree_view* tree, int32_t* new_node,
                     float* new_sigma, float* new_sh, int64_t* src_index, uint8_t* src_kind, void* stream) {
    if (!p || !tree) return set_error(DOT_BAD_ARG, "NULL argument");
    if (!new_node || !new_sigma || !new_sh || !src_index || !src_kind)
        return set_error(DOT_BAD_ARG, "refine outputs must not be NULL");
    if ((reinterpret_cast<uintptr_t>(new_sh) & 15) != 0) return set_error(DOT_BAD_ARG, "new_sh must be 16-byte aligned");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const TreeDev T = make_tree(*tree);
    const int64_t n_new = p->stats.n_new_nodes;
    int st = DOT_OK;
    int32_t *ent_old[2] = {nullptr, nullptr}, *flags = nullptr;
    uint8_t* ent_kind[2] = {nullptr, nullptr};
    int64_t *rank = nullptr, *sums = nullptr, *d_total = nullptr;
    auto cleanup = [&]() {
        for (int b = 0; b < 2; ++b) {
            cudaFreeAsync(ent_old[b], s);
            cudaFreeAsync(ent_kind[b], s);
        }
        cudaFreeAsync(flags, s);
        cudaFreeAsync(rank, s);
        cudaFreeAsync(sums, s);
        cudaFreeAsync(d_total, s);
    };
#define TRY(x) do { if ((st = (x)) != DOT_OK) { cleanup(); return st; } } while (0)
    for (int b = 0; b < 2; ++b) {
        TRY(dalloc(&ent_old[b], n_new, s));
        TRY(dalloc(&ent_kind[b], n_new, s));
    }
    TRY(dalloc(&flags, n_new, s));
    TRY(dalloc(&rank, n_new, s));
    TRY(dalloc(&sums, n_new / kScanTile + 2, s));
    TRY(dalloc(&d_total, 1, s));
    // level 0: the root, kept
    const int32_t zero = 0;
    const uint8_t kept = K_KEPT;
    TRY(check_cuda(cudaMemcpyAsync(ent_old[0], &zero, sizeof(zero), cudaMemcpyHostToDevice, s), "memcpy"));
    TRY(check_cuda(cudaMemcpyAsync(ent_kind[0], &kept, sizeof(kept), cudaMemcpyHostToDevice, s), "memcpy"));
    int64_t base = 0, m = 1;
    int cur = 0;
    while (m > 0) {
        if (base + m > n_new) TRY(set_error(DOT_CUDA_ERR, "refine apply overflow (plan/tree mismatch)"));
        level_flags_kernel<<<grid_for(m), kTB, 0, s>>>(m, ent_old[cur], ent_kind[cur], p->state, flags);
        TRY(check_launch("level_flags_kernel"));
        TRY(exclusive_scan(flags, m, rank, sums, d_total, s));
        int64_t n_int = 0;
        TRY(check_cuda(cudaMemcpyAsync(&n_int, d_total, sizeof(n_int), cudaMemcpyDeviceToHost, s), "memcpy"));
        TRY(check_cuda(cudaStreamSynchronize(s), "sync"));
        const int64_t next_base = base + m;
        level_emit_kernel<<<grid_for(m), kTB, 0, s>>>(T, m, base, next_base, ent_old[cur], ent_kind[cur], flags,
                                                      rank, p->state, new_node, src_index, src_kind,
                                                      ent_old[cur ^ 1], ent_kind[cur ^ 1]);
        TRY(check_launch("level_emit_kernel"));
        base = next_base;
        m = 8 * n_int;
        cur ^= 1;
    }
    if (base != n_new) TRY(set_error(DOT_CUDA_ERR, "refine apply produced %lld nodes, plan said %lld",
                                     (long long)base, (long long)n_new));
    const int S4 = p->S / 4;
    payload_kernel<<<grid_for(n_new * S4), kTB, 0, s>>>(T, n_new, S4, src_index, src_kind, p->state, p->slot,
                                                       p->msig, p->msh, new_node, new_sigma,
                                                       reinterpret_cast<float4*>(new_sh));
    TRY(check_launch("payload_kernel"));
    cleanup();
#undef TRY
    return DOT_OK;
}

void dot_refine_plan_destroy(dot_refine_plan* plan) { plan_free(plan); }

}  // extern "C"
