// render.cu -- traversal, fused forward and fused forward+backward kernels.
//
// One thread per ray.  The reference (octrf/render.py:105-225 over
// octrf/_kernels.py:161-346) materialises every ray's segment list twice
// (count + fill), then composites, then reduces per leaf serially.  Here the
// traversal is streamed: a segment is consumed the moment it is produced and
// never touches HBM; the backward recomputes the forward instead of saving
// ~96 B of per-segment scratch, and leaf gradients / signal are reduced with
// vector REDs (REDG.E.ADD.F32x4) straight into the per-leaf buffers.
#include "dot_tree.cuh"
#include "dot_internal.h"

namespace dot {

constexpr int kBlock = 128;
#ifndef DOT_FWD_MINB
#define DOT_FWD_MINB 8  // forward: 64 registers -> 8 blocks (32 warps) per SM
#endif
#ifndef DOT_FWD_PREFETCH
#define DOT_FWD_PREFETCH true
#endif
constexpr int kStk = kPathLevels + 2;  // odd row stride: conflict-free shared-memory stacks

// Per-thread path cache in shared memory (see descend_cached).  Kernels are
// instantiated with CACHED = false for trees deeper than the 64-bit path word
// can describe (max_depth >= kPathLevels).
template <bool CACHED>
__device__ __forceinline__ void init_cache(const TreeDev& T, int32_t* smem, PathCache& pc) {
    pc.depth = -1;
    pc.path = 0;
    pc.stk = smem + threadIdx.x * kStk;
    if (CACHED) pc.stk[0] = __ldg(T.node);
}

#define DOT_STACK_SMEM(CACHED) __shared__ int32_t s_stk[(CACHED) ? kBlock * kStk : 1]

// Off by default: measured on B200 the L1 already serves the hot upper levels
// and the extra registers cost more than the saved loads (fwd 1.38e9 ->
// 1.12e9 rays/s).  dot_render_bwd flag bit 3 turns it on for experiments.
inline bool use_cache(const TreeDev& T, int flags = 0) {
    return (flags & 8) != 0 && T.max_depth < kPathLevels;
}

__device__ __forceinline__ void load_ray(const double* __restrict__ o, const double* __restrict__ d,
                                         int64_t r, Tracer& tr) {
    tr.ox = __ldg(o + 3 * r + 0);
    tr.oy = __ldg(o + 3 * r + 1);
    tr.oz = __ldg(o + 3 * r + 2);
    tr.dx = __ldg(d + 3 * r + 0);
    tr.dy = __ldg(d + 3 * r + 1);
    tr.dz = __ldg(d + 3 * r + 2);
}

// ---------------------------------------------------------------------------
// Segment lists (parity / debug path of segment_batch).

template <bool CACHED>
__global__ void __launch_bounds__(kBlock) trace_count_kernel(TreeDev T, const double* __restrict__ o,
                                                             const double* __restrict__ d, int64_t n,
                                                             double t_near, double t_far,
                                                             int64_t* __restrict__ counts) {
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= n) return;
    DOT_STACK_SMEM(CACHED);
    PathCache pc;
    init_cache<CACHED>(T, s_stk, pc);
    Tracer tr;
    load_ray(o, d, r, tr);
    int64_t c = 0;
    if (tr.init(T, t_near, t_far)) {
        Leaf L;
        double te, dl;
        while (tr.template next<CACHED>(T, L, te, dl, pc)) ++c;
    }
    counts[r] = c;
}

template <bool CACHED>
__global__ void __launch_bounds__(kBlock) trace_fill_kernel(TreeDev T, const double* __restrict__ o,
                                                            const double* __restrict__ d, int64_t n,
                                                            double t_near, double t_far,
                                                            const int64_t* __restrict__ offsets,
                                                            int64_t* __restrict__ seg_leaf,
                                                            double* __restrict__ seg_t,
                                                            double* __restrict__ seg_delta) {
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= n) return;
    DOT_STACK_SMEM(CACHED);
    PathCache pc;
    init_cache<CACHED>(T, s_stk, pc);
    Tracer tr;
    load_ray(o, d, r, tr);
    int64_t s = offsets[r];
    if (tr.init(T, t_near, t_far)) {
        Leaf L;
        double te, dl;
        while (tr.template next<CACHED>(T, L, te, dl, pc)) {
            seg_leaf[s] = L.pid;
            seg_t[s] = te;
            seg_delta[s] = dl;
            ++s;
        }
    }
}

// ---------------------------------------------------------------------------
// Fused forward: traverse + composite (composite_kernel, _kernels.py:185-224).

template <int B, bool CACHED>
__global__ void __launch_bounds__(kBlock, DOT_FWD_MINB) render_fwd_kernel(
    TreeDev T, const double* __restrict__ o, const double* __restrict__ d, int64_t n,
    double bg0, double bg1, double bg2, double eps, double t_near, double t_far,
    float* __restrict__ rgb, float* __restrict__ tfin_out, float* __restrict__ wsum_out,
    float* __restrict__ depth_out) {
    constexpr int S = pad4(3 * B);
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= n) return;
    DOT_STACK_SMEM(CACHED);
    PathCache pc;
    init_cache<CACHED>(T, s_stk, pc);
    Tracer tr;
    load_ray(o, d, r, tr);
    float basis[B];
    eval_basis<B>(tr.dx, tr.dy, tr.dz, basis);
    double trans = 1.0, c0 = 0.0, c1 = 0.0, c2 = 0.0, ws = 0.0, dep = 0.0;
    if (tr.init(T, t_near, t_far)) {
        Leaf L;
        double te, dl;
        while (tr.template next<CACHED, DOT_FWD_PREFETCH>(T, L, te, dl, pc)) {
            const double sg = double(__ldg(T.sigma + L.pid));
            const double a = exp_ref(-sg * dl);
            const double q = 1.0 - a;
            if (q > 0.0) {
                float e0, e1, e2;
                sh_dot<B>(T.sh + int64_t(L.pid) * S, basis, e0, e1, e2);
                const double tq = trans * q;
                c0 += tq * double(sigmoidf(e0));
                c1 += tq * double(sigmoidf(e1));
                c2 += tq * double(sigmoidf(e2));
                ws += tq;
                dep += tq * (te + 0.5 * dl);
            }
            trans *= a;
            if (eps > 0.0 && trans < eps) break;
        }
    }
    ws += trans;
    if (rgb) {
        rgb[3 * r + 0] = float(c0 + trans * bg0);
        rgb[3 * r + 1] = float(c1 + trans * bg1);
        rgb[3 * r + 2] = float(c2 + trans * bg2);
    }
    if (tfin_out) tfin_out[r] = float(trans);
    if (wsum_out) wsum_out[r] = float(ws);
    if (depth_out) depth_out[r] = float(dep);
}

// ---------------------------------------------------------------------------
// Fused forward + backward + signal (grad_kernel + scatter_kernel,
// _kernels.py:227-346).  Pass 1 composites to get rgb and the cut index;
// pass 2 re-walks the ray, rebuilds T_i, Q_i, c_i, forms the suffix
// suf_i = rgb - sum_{j<=i} T_j Q_j c_j and scatters
//   dsigma_i = delta_i * sum_k g_k (T_i a_i c_ik - suf_ik)
//   dsh_i[k*B+b] = g_k T_i Q_i c_ik (1 - c_ik) * basis_b
// plus signal_i += Q_i and touched = 1 (post-cut segments: touched only).

template <int B>
__global__ void __launch_bounds__(kBlock) render_bwd_kernel(
    TreeDev T, const double* __restrict__ o, const double* __restrict__ d,
    const double* __restrict__ tgt, int64_t n, double bg0, double bg1, double bg2, double eps,
    double t_near, double t_far, double grad_scale, float* __restrict__ gsig,
    float* __restrict__ gsh, double* __restrict__ signal, uint8_t* __restrict__ touched,
    double* __restrict__ loss_sum, float* __restrict__ rgb_out, int flags) {
    constexpr int S = pad4(3 * B);
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    double loss = 0.0;
    if (r < n) {
        Tracer tr;
        load_ray(o, d, r, tr);
        float basis[B];
        eval_basis<B>(tr.dx, tr.dy, tr.dz, basis);
        const bool hit = tr.init(T, t_near, t_far);
        const Tracer start = tr;
        // ---- pass 1: forward to the cut
        double trans = 1.0, c0 = 0.0, c1 = 0.0, c2 = 0.0;
        int used = 0;
        if (hit) {
            Leaf L;
            double te, dl;
            while (tr.next(T, L, te, dl)) {
                const double sg = double(__ldg(T.sigma + L.pid));
                const double a = exp_ref(-sg * dl);
                const double q = 1.0 - a;
                ++used;
                if (q > 0.0) {
                    float e0, e1, e2;
                    sh_dot<B>(T.sh + int64_t(L.pid) * S, basis, e0, e1, e2);
                    const double tq = trans * q;
                    c0 += tq * double(sigmoidf(e0));
                    c1 += tq * double(sigmoidf(e1));
                    c2 += tq * double(sigmoidf(e2));
                }
                trans *= a;
                if (eps > 0.0 && trans < eps) break;
            }
        }
        const double tf = trans;
        const double R0 = c0 + tf * bg0, R1 = c1 + tf * bg1, R2 = c2 + tf * bg2;
        const double r0 = R0 - __ldg(tgt + 3 * r + 0);
        const double r1 = R1 - __ldg(tgt + 3 * r + 1);
        const double r2 = R2 - __ldg(tgt + 3 * r + 2);
        loss = r0 * r0 + r1 * r1 + r2 * r2;
        if (rgb_out) {
            rgb_out[3 * r + 0] = float(R0);
            rgb_out[3 * r + 1] = float(R1);
            rgb_out[3 * r + 2] = float(R2);
        }
        const double g0 = grad_scale * r0, g1 = grad_scale * r1, g2 = grad_scale * r2;
        // ---- pass 2: replay, reverse-mode quantities via the prefix identity
        if (hit) {
            tr = start;
            Leaf L;
            double te, dl;
            double Ti = 1.0, p0 = 0.0, p1 = 0.0, p2 = 0.0;
            int i = 0;
            while (tr.next(T, L, te, dl)) {
                const int64_t pid = L.pid;
                if (i < used) {
                    const double sg = double(__ldg(T.sigma + pid));
                    const double a = exp_ref(-sg * dl);
                    const double q = 1.0 - a;
                    float e0, e1, e2;
                    sh_dot<B>(T.sh + pid * S, basis, e0, e1, e2);
                    const float k0 = sigmoidf(e0), k1 = sigmoidf(e1), k2 = sigmoidf(e2);
                    const double tq = Ti * q;
                    p0 += tq * double(k0);
                    p1 += tq * double(k1);
                    p2 += tq * double(k2);
                    const double tn = Ti * a;
                    const double ds = dl * (g0 * (tn * k0 - (R0 - p0)) + g1 * (tn * k1 - (R1 - p1)) +
                                            g2 * (tn * k2 - (R2 - p2)));
                    red_add_f32(gsig + pid, float(ds));
                    const float w0 = float(g0 * tq) * k0 * (1.f - k0);
                    const float w1 = float(g1 * tq) * k1 * (1.f - k1);
                    const float w2 = float(g2 * tq) * k2 * (1.f - k2);
                    if (w0 != 0.f || w1 != 0.f || w2 != 0.f) {
                        float* row = gsh + pid * S;
#pragma unroll
                        for (int j = 0; j < S / 4; ++j) {
                            float v[4];
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const int idx = 4 * j + u;
                                const int k = idx / B;
                                const float w = k == 0 ? w0 : (k == 1 ? w1 : w2);
                                v[u] = idx < 3 * B ? w * basis[idx % B] : 0.f;
                            }
                            red_add_v4(row + 4 * j, v[0], v[1], v[2], v[3]);
                        }
                    }
                    if (q != 0.0) red_add_f64(signal + pid, q);
                    touched[pid] = 1;
                    Ti *= a;
                    ++i;
                } else {
                    if (flags & 1) break;
                    touched[pid] = 1;
                }
            }
        }
    }
    // ---- loss: warp reduce, one f64 RED per warp
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) loss += __shfl_down_sync(0xffffffffu, loss, off);
    if ((threadIdx.x & 31) == 0 && loss != 0.0) red_add_f64(loss_sum, loss);
}

// ---------------------------------------------------------------------------
// Persistent fused forward + backward.  The one-ray-per-thread kernel above
// leaves most lanes idle (ray lengths vary ~10x inside a random batch: ncu
// measured 4.4 active threads per warp).  Here every lane is a small state
// machine that advances ONE segment per loop iteration -- phase 1 composites
// up to the cut, phase 2 replays the ray scattering gradients -- and fetches
// its next ray with a warp-aggregated atomic the moment its current ray is
// done, so the warp's lanes stay busy whatever the per-ray segment counts.
// Same arithmetic as render_bwd_kernel; phase 2 carries the suffix directly
// (suf = rgb - prefix, updated per segment).

template <int B, bool CACHED>
__global__ void __launch_bounds__(kBlock) render_bwd_persistent_kernel(
    TreeDev T, const double* __restrict__ o, const double* __restrict__ d,
    const double* __restrict__ tgt, int64_t n, double bg0, double bg1, double bg2, double eps,
    double t_near, double t_far, double grad_scale, float* __restrict__ gsig,
    float* __restrict__ gsh, double* __restrict__ signal, uint8_t* __restrict__ touched,
    double* __restrict__ loss_sum, float* __restrict__ rgb_out, int flags,
    unsigned long long* __restrict__ ray_ctr) {
    constexpr int S = pad4(3 * B);
    constexpr unsigned FULL = 0xffffffffu;
    const unsigned lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    DOT_STACK_SMEM(CACHED);
    PathCache pc;
    init_cache<CACHED>(T, s_stk, pc);  // survives across rays: any cached path is valid
    Tracer tr;
    float basis[B];
    int phase = 0;  // 0: needs a ray, 1: forward to the cut, 2: backward replay
    bool exhausted = false;
    int64_t r = 0;
    double t0 = 0.0;
    double Tacc = 1.0, s0 = 0.0, s1 = 0.0, s2 = 0.0;  // phase 1: T, colour; phase 2: T_i, suffix
    double g0 = 0.0, g1 = 0.0, g2 = 0.0;
    int used = 0, i = 0;
    double loss = 0.0;

    // pass-1 epilogue: rgb, loss, dL/drgb; primes the suffix for phase 2
    auto finish_forward = [&]() {
        const double R0 = s0 + Tacc * bg0, R1 = s1 + Tacc * bg1, R2 = s2 + Tacc * bg2;
        const double r0 = R0 - __ldg(tgt + 3 * r + 0);
        const double r1 = R1 - __ldg(tgt + 3 * r + 1);
        const double r2 = R2 - __ldg(tgt + 3 * r + 2);
        loss += r0 * r0 + r1 * r1 + r2 * r2;
        if (rgb_out) {
            rgb_out[3 * r + 0] = float(R0);
            rgb_out[3 * r + 1] = float(R1);
            rgb_out[3 * r + 2] = float(R2);
        }
        g0 = grad_scale * r0;
        g1 = grad_scale * r1;
        g2 = grad_scale * r2;
        s0 = R0;
        s1 = R1;
        s2 = R2;
    };

    for (;;) {
        const bool want = phase == 0 && !exhausted;
        const unsigned need = __ballot_sync(FULL, want);
        if (need) {
            const int leader = __ffs(need) - 1;
            unsigned long long base = 0;
            if (int(lane) == leader) base = atomicAdd(ray_ctr, (unsigned long long)__popc(need));
            base = __shfl_sync(FULL, base, leader);
            if (want) {
                r = int64_t(base) + __popc(need & lt_mask);
                if (r >= n) {
                    exhausted = true;
                } else {
                    load_ray(o, d, r, tr);
                    eval_basis<B>(tr.dx, tr.dy, tr.dz, basis);
                    Tacc = 1.0;
                    s0 = s1 = s2 = 0.0;
                    used = 0;
                    if (tr.init(T, t_near, t_far)) {
                        t0 = tr.t;
                        phase = 1;
                    } else {
                        finish_forward();  // miss: background only, no leaf touched
                    }
                }
            }
        }
        if (__all_sync(FULL, phase == 0 && exhausted)) break;
        if (phase == 0) continue;

        Leaf L;
        double te, dl;
        const bool got = tr.template next<CACHED>(T, L, te, dl, pc);
        if (phase == 1) {
            bool cut = false;
            if (got) {
                const double a = exp_ref(-double(__ldg(T.sigma + L.pid)) * dl);
                const double q = 1.0 - a;
                ++used;
                if (q > 0.0) {
                    float e0, e1, e2;
                    sh_dot<B>(T.sh + int64_t(L.pid) * S, basis, e0, e1, e2);
                    const double tq = Tacc * q;
                    s0 += tq * double(sigmoidf(e0));
                    s1 += tq * double(sigmoidf(e1));
                    s2 += tq * double(sigmoidf(e2));
                }
                Tacc *= a;
                cut = eps > 0.0 && Tacc < eps;
            }
            if (!got || cut) {
                finish_forward();
                tr.t = t0;
                tr.nudge = tr.nudge0;
                Tacc = 1.0;
                i = 0;
                phase = 2;
            }
        } else {
            if (!got) {
                phase = 0;
            } else if (i < used) {
                const int64_t pid = L.pid;
                const double a = exp_ref(-double(__ldg(T.sigma + pid)) * dl);
                const double q = 1.0 - a;
                float e0, e1, e2;
                sh_dot<B>(T.sh + pid * S, basis, e0, e1, e2);
                const float k0 = sigmoidf(e0), k1 = sigmoidf(e1), k2 = sigmoidf(e2);
                const double tq = Tacc * q;
                s0 -= tq * double(k0);
                s1 -= tq * double(k1);
                s2 -= tq * double(k2);
                const double tn = Tacc * a;
                const double ds = dl * (g0 * (tn * k0 - s0) + g1 * (tn * k1 - s1) + g2 * (tn * k2 - s2));
                red_add_f32(gsig + pid, float(ds));
                const float w0 = float(g0 * tq) * k0 * (1.f - k0);
                const float w1 = float(g1 * tq) * k1 * (1.f - k1);
                const float w2 = float(g2 * tq) * k2 * (1.f - k2);
                if (w0 != 0.f || w1 != 0.f || w2 != 0.f) {
                    float* row = gsh + pid * S;
#pragma unroll
                    for (int j = 0; j < S / 4; ++j) {
                        float v[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int idx = 4 * j + u;
                            const int k = idx / B;
                            const float w = k == 0 ? w0 : (k == 1 ? w1 : w2);
                            v[u] = idx < 3 * B ? w * basis[idx % B] : 0.f;
                        }
                        red_add_v4(row + 4 * j, v[0], v[1], v[2], v[3]);
                    }
                }
                if (q != 0.0) red_add_f64(signal + pid, q);
                touched[pid] = 1;
                Tacc *= a;
                ++i;
            } else if (flags & 1) {
                phase = 0;
            } else {
                touched[L.pid] = 1;
            }
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) loss += __shfl_down_sync(FULL, loss, off);
    if (lane == 0 && loss != 0.0) red_add_f64(loss_sum, loss);
}

// ---------------------------------------------------------------------------
// Buffered fused forward + backward (default).  One ray per thread; rays in
// a batch are expected in a coherent order (the loader's Morton sort).
// Pass 1 walks the ray ONCE: it composites up to the early-termination cut,
// marks every traversed leaf touched (post-cut ones too, scatter_kernel
// semantics) and buffers each composited segment (leaf, delta, alpha, colour)
// in a per-thread local array.  Pass 2 replays the buffer in order -- no
// second traversal, the colour of q > 0 segments is not recomputed -- and,
// for rays with more than K composited segments, resumes the walk from the
// tracer state saved when the buffer filled.

struct BufSeg {
    int32_t pid;
    float delta;
    double a;        // alpha = exp_ref(-sigma delta) exactly as pass 1 used it
    float k0, k1, k2;  // colour (NaN: not evaluated in pass 1, q == 0)
    float pad;
};

// Segment buffer: per-thread local array (GBUF = false) or an explicit global
// SoA scratch (entry i of ray r at gbuf[i * n + r], coalesced across a warp)
// accessed with streaming (.cs) hints so it does not evict the node table
// and payload rows from L1.
template <bool GBUF, int K>
struct SegBuffer {
    BufSeg local[GBUF ? 1 : K];
    BufSeg* g;
    int64_t stride;
    __device__ __forceinline__ void put(int i, const BufSeg& e) {
        if constexpr (GBUF) {
            const float4* s = reinterpret_cast<const float4*>(&e);
            float4* p = reinterpret_cast<float4*>(g + int64_t(i) * stride);
            __stcs(p, s[0]);
            __stcs(p + 1, s[1]);
        } else {
            local[i] = e;
        }
    }
    __device__ __forceinline__ BufSeg get(int i) const {
        if constexpr (GBUF) {
            BufSeg e;
            const float4* p = reinterpret_cast<const float4*>(g + int64_t(i) * stride);
            float4* s = reinterpret_cast<float4*>(&e);
            s[0] = __ldcs(p);
            s[1] = __ldcs(p + 1);
            return e;
        } else {
            return local[i];
        }
    }
};

// Where pass 2 sends each composited segment's gradient contribution.
// AtomicSink: vector REDs straight into the per-leaf buffers (default).
// EmitSink (sorted.cu): one record per segment, reduced per leaf afterwards
// in ray-major order (deterministic mode).
struct AtomicSink {
    float* __restrict__ gsig;
    float* __restrict__ gsh;
    double* __restrict__ signal;
    double* __restrict__ loss_sum;
    // warp-collective, all 32 lanes (no-op here)
    __device__ __forceinline__ void reserve(int, bool) {}
    template <int B>
    __device__ __forceinline__ void put(int, int64_t pid, float ds, float w0, float w1, float w2,
                                        const float* basis, double q) {
        constexpr int S = pad4(3 * B);
        red_add_f32(gsig + pid, ds);
        if (w0 != 0.f || w1 != 0.f || w2 != 0.f) {
            float* row = gsh + pid * S;
#pragma unroll
            for (int j = 0; j < S / 4; ++j) {
                float v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int idx = 4 * j + u;
                    const int k = idx / B;
                    const float w = k == 0 ? w0 : (k == 1 ? w1 : w2);
                    v[u] = idx < 3 * B ? w * basis[idx % B] : 0.f;
                }
                red_add_v4(row + 4 * j, v[0], v[1], v[2], v[3]);
            }
        }
        if (q != 0.0) red_add_f64(signal + pid, q);
    }
    template <int B>
    __device__ __forceinline__ void ray_done(int64_t, const float*, double) {}
    // warp-collective: sum of the per-ray squared errors
    __device__ __forceinline__ void loss(double v) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
        if ((threadIdx.x & 31) == 0 && v != 0.0) red_add_f64(loss_sum, v);
    }
};

template <int B, int K, int MINB = 1, bool GBUF = false, int BLK = kBlock, bool PF = false,
          class Sink = AtomicSink>
__global__ void __launch_bounds__(BLK, MINB) render_bwd_buffered_kernel(
    TreeDev T, const double* __restrict__ o, const double* __restrict__ d,
    const double* __restrict__ tgt, int64_t n, double bg0, double bg1, double bg2, double eps,
    double t_near, double t_far, double grad_scale, uint8_t* __restrict__ touched,
    float* __restrict__ rgb_out, int flags, BufSeg* __restrict__ gbuf, Sink sink) {
    constexpr int S = pad4(3 * B);
    double loss = 0.0;
    // one ray per thread, blocks scheduled dynamically by the hardware (a
    // grid-stride variant measured 60 % slower: static per-block ray sets
    // leave SMs idle behind long rays)
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool valid = r < n;
    Tracer tr;
    float basis[B];
    SegBuffer<GBUF, K> buf;
    int used = 0;
    double resume_t = 0.0, resume_nudge = 0.0;
    double R0 = 0.0, R1 = 0.0, R2 = 0.0, g0 = 0.0, g1 = 0.0, g2 = 0.0;
    if (valid) {
        load_ray(o, d, r, tr);
        eval_basis<B>(tr.dx, tr.dy, tr.dz, basis);
        buf.g = gbuf + r;
        buf.stride = n;
        double trans = 1.0, c0 = 0.0, c1 = 0.0, c2 = 0.0;
        const bool hit = tr.init(T, t_near, t_far);
        if (hit) {
            Leaf L;
            double te, dl;
            bool cut = false;
            while (tr.next_prefetch(T, L, te, dl, !cut)) {
                touched[L.pid] = 1;
                if (cut) continue;  // post-cut: touched only
                const double a = exp_ref(-double(__ldg(T.sigma + L.pid)) * dl);
                const double q = 1.0 - a;
                float k0 = __int_as_float(0x7fc00000), k1 = k0, k2 = k0;
                if (q > 0.0) {
                    float e0, e1, e2;
                    sh_dot<B>(T.sh + int64_t(L.pid) * S, basis, e0, e1, e2);
                    k0 = sigmoidf(e0);
                    k1 = sigmoidf(e1);
                    k2 = sigmoidf(e2);
                    const double tq = trans * q;
                    c0 += tq * double(k0);
                    c1 += tq * double(k1);
                    c2 += tq * double(k2);
                }
                if (used < K) {
                    BufSeg e;
                    e.pid = L.pid;
                    e.delta = float(dl);
                    e.a = a;
                    e.k0 = k0;
                    e.k1 = k1;
                    e.k2 = k2;
                    e.pad = 0.f;
                    buf.put(used, e);
                } else if (used == K) {  // buffer full: remember where pass 2 resumes
                    resume_t = te;
                    resume_nudge = tr.nudge0;
                }
                ++used;
                trans *= a;
                if (eps > 0.0 && trans < eps) {
                    cut = true;
                    if (flags & 1) break;
                }
            }
        }
        const double tf = trans;
        R0 = c0 + tf * bg0;
        R1 = c1 + tf * bg1;
        R2 = c2 + tf * bg2;
        const double r0 = R0 - __ldg(tgt + 3 * r + 0);
        const double r1 = R1 - __ldg(tgt + 3 * r + 1);
        const double r2 = R2 - __ldg(tgt + 3 * r + 2);
        loss = r0 * r0 + r1 * r1 + r2 * r2;
        if (rgb_out) {
            rgb_out[3 * r + 0] = float(R0);
            rgb_out[3 * r + 1] = float(R1);
            rgb_out[3 * r + 2] = float(R2);
        }
        g0 = grad_scale * r0;
        g1 = grad_scale * r1;
        g2 = grad_scale * r2;
        if (flags & 8192) used = 0;  // diagnostic: pass 1 only
    }
    __syncwarp();
    sink.reserve(used, valid);
    if (valid) {
        sink.template ray_done<B>(r, basis, loss);
        // ---- pass 2: replay (suffix carried directly: suf = rgb - prefix)
        double s0 = R0, s1 = R1, s2 = R2, Ti = 1.0;
        if (used > K) {  // segment K onwards come from a resumed walk
            tr.t = resume_t;
            tr.nudge = resume_nudge;
        }
        Leaf L;
        BufSeg nxt;
        if (PF && used > 0) nxt = buf.get(0);
        for (int i = 0; i < used; ++i) {
            int64_t pid;
            double a, dl;
            float k0, k1, k2;
            if (i < K) {
                BufSeg e;
                if (PF) {  // software pipeline: entry i+1 is in flight while i is scattered
                    e = nxt;
                    if (i + 1 < used && i + 1 < K) nxt = buf.get(i + 1);
                } else {
                    e = buf.get(i);
                }
                pid = e.pid;
                a = e.a;
                dl = e.delta;
                k0 = e.k0;
                k1 = e.k1;
                k2 = e.k2;
            } else {
                double te;
                tr.next(T, L, te, dl);
                pid = L.pid;
                a = exp_ref(-double(__ldg(T.sigma + pid)) * dl);
                k0 = __int_as_float(0x7fc00000);
            }
            if (k0 != k0) {
                float e0, e1, e2;
                sh_dot<B>(T.sh + pid * S, basis, e0, e1, e2);
                k0 = sigmoidf(e0);
                k1 = sigmoidf(e1);
                k2 = sigmoidf(e2);
            }
            const double q = 1.0 - a;
            const double tq = Ti * q;
            s0 -= tq * double(k0);
            s1 -= tq * double(k1);
            s2 -= tq * double(k2);
            const double tn = Ti * a;
            const double ds = dl * (g0 * (tn * k0 - s0) + g1 * (tn * k1 - s1) + g2 * (tn * k2 - s2));
            const float w0 = float(g0 * tq) * k0 * (1.f - k0);
            const float w1 = float(g1 * tq) * k1 * (1.f - k1);
            const float w2 = float(g2 * tq) * k2 * (1.f - k2);
            Ti *= a;
            if (flags & 16384) {  // diagnostic: no reductions
                if (ds == 12345.0 && w0 == 1.f) red_add_f32(touched ? reinterpret_cast<float*>(rgb_out) : nullptr, w1 + w2);
                continue;
            }
            sink.template put<B>(i, pid, float(ds), w0, w1, w2, basis, q);
        }
    }
    sink.loss(loss);
}

#define DOT_DISPATCH_B(MACRO)                                                     \
    switch (T.basis_count) {                                                      \
        case 1: if (cached) MACRO(1, true) else MACRO(1, false) break;            \
        case 4: if (cached) MACRO(4, true) else MACRO(4, false) break;            \
        case 9: if (cached) MACRO(9, true) else MACRO(9, false) break;            \
        case 16: if (cached) MACRO(16, true) else MACRO(16, false) break;         \
        default: return set_error(DOT_BAD_ARG, "basis_count must be 1, 4, 9 or 16"); \
    }

// Record sink of the deterministic (sorted) backward: pass 2 writes one
// record per composited segment -- key (pool id << ray_bits | original ray
// index), (dsigma, w0, w1, w2) f32 and q f64 -- into slots reserved per ray
// with one warp-aggregated atomicAdd; the ray's SH basis and squared error
// go to per-ray arrays (original index).  A ray whose records do not fit is
// counted in ctr[1] and writes nothing (the host retries with more room).
struct EmitSink {
    EmitArgs a;
    int64_t base;
    int64_t orig;
    __device__ __forceinline__ void reserve(int used, bool valid) {
        const int lane = threadIdx.x & 31;
        int incl = used;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += v;
        }
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        unsigned long long b0 = 0;
        if (lane == 31 && total > 0) b0 = atomicAdd(a.ctr, (unsigned long long)total);
        b0 = __shfl_sync(0xffffffffu, b0, 31);
        base = int64_t(b0) + (incl - used);
        if (valid && used > 0 && base + used > a.cap) {
            atomicAdd(a.ctr + 1, 1ull);
            base = -1;
        }
    }
    template <int B>
    __device__ __forceinline__ void ray_done(int64_t r, const float* basis, double loss) {
        orig = a.ray_id ? a.ray_id[r] : r;
#pragma unroll
        for (int b = 0; b < B; ++b) a.basis[orig * B + b] = basis[b];
        a.loss_ray[orig] = loss;
    }
    template <int B>
    __device__ __forceinline__ void put(int i, int64_t pid, float ds, float w0, float w1, float w2,
                                        const float*, double q) {
        if (base < 0) return;
        const int64_t k = base + i;
        a.keys[k] = (static_cast<unsigned long long>(pid) << a.ray_bits) |
                    static_cast<unsigned long long>(orig);
        a.rec[k] = make_float4(ds, w0, w1, w2);
        a.recq[k] = q;
    }
    __device__ __forceinline__ void loss(double) {}
};

int launch_render_bwd_emit(const TreeDev& T, const double* o, const double* d, const double* tgt,
                           int64_t n, const double* bg, double eps, double tn, double tf, double gs,
                           uint8_t* touched, const EmitArgs& ea, cudaStream_t s) {
    if (n == 0) return DOT_OK;
    EmitSink sink;
    sink.a = ea;
    sink.base = -1;
    sink.orig = 0;
#define DOT_EMIT(BB, CC)                                                                          \
    render_bwd_buffered_kernel<BB, 48, 32, false, 32, true, EmitSink><<<unsigned((n + 31) / 32), 32, 0, s>>>( \
        T, o, d, tgt, n, bg[0], bg[1], bg[2], eps, tn, tf, gs, touched, nullptr, 0, nullptr, sink);
    const bool cached = false;
    DOT_DISPATCH_B(DOT_EMIT)
#undef DOT_EMIT
    return check_launch("render_bwd_buffered_kernel<emit>");
}

// Replay of rays whose segment records overflowed the two-kernel path's
// buffer (backward.cu): pass 1 only recounts the composited segments, pass 2
// scatters with the rgb and dL/drgb that kernel A already stored.
template <int B>
__global__ void __launch_bounds__(kBlock) render_bwd_replay_kernel(
    TreeDev T, const double* __restrict__ o, const double* __restrict__ d, int64_t n, double eps,
    double t_near, double t_far, float* __restrict__ gsig, float* __restrict__ gsh,
    double* __restrict__ signal, const float* __restrict__ ray_g, const float* __restrict__ ray_rgb,
    const uint8_t* __restrict__ ray_flag) {
    constexpr int S = pad4(3 * B);
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n; r += stride) {
        if (!(ray_flag[r] & 1)) continue;
        Tracer tr;
        load_ray(o, d, r, tr);
        float basis[B];
        eval_basis<B>(tr.dx, tr.dy, tr.dz, basis);
        if (!tr.init(T, t_near, t_far)) continue;
        const Tracer start = tr;
        int used = 0;
        double trans = 1.0;
        Leaf L;
        double te, dl;
        while (tr.next(T, L, te, dl)) {
            trans *= exp_ref(-double(__ldg(T.sigma + L.pid)) * dl);
            ++used;
            if (eps > 0.0 && trans < eps) break;
        }
        const double g0 = ray_g[3 * r], g1 = ray_g[3 * r + 1], g2 = ray_g[3 * r + 2];
        double s0 = ray_rgb[3 * r], s1 = ray_rgb[3 * r + 1], s2 = ray_rgb[3 * r + 2];
        tr = start;
        double Ti = 1.0;
        for (int i = 0; i < used && tr.next(T, L, te, dl); ++i) {
            const int64_t pid = L.pid;
            const double a = exp_ref(-double(__ldg(T.sigma + pid)) * dl);
            const double q = 1.0 - a;
            float e0, e1, e2;
            sh_dot<B>(T.sh + pid * S, basis, e0, e1, e2);
            const float k0 = sigmoidf(e0), k1 = sigmoidf(e1), k2 = sigmoidf(e2);
            const double tq = Ti * q;
            s0 -= tq * double(k0);
            s1 -= tq * double(k1);
            s2 -= tq * double(k2);
            const double tn = Ti * a;
            red_add_f32(gsig + pid, float(dl * (g0 * (tn * k0 - s0) + g1 * (tn * k1 - s1) + g2 * (tn * k2 - s2))));
            const float w[3] = {float(g0 * tq) * k0 * (1.f - k0), float(g1 * tq) * k1 * (1.f - k1),
                                float(g2 * tq) * k2 * (1.f - k2)};
            if (w[0] != 0.f || w[1] != 0.f || w[2] != 0.f) {
                float* row = gsh + pid * S;
#pragma unroll
                for (int j = 0; j < S / 4; ++j) {
                    float v[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int idx = 4 * j + u;
                        v[u] = idx < 3 * B ? w[idx / B] * basis[idx % B] : 0.f;
                    }
                    red_add_v4(row + 4 * j, v[0], v[1], v[2], v[3]);
                }
            }
            if (q != 0.0) red_add_f64(signal + pid, q);
            Ti *= a;
        }
    }
}

int launch_render_bwd_replay(const TreeDev& T, const double* o, const double* d, int64_t n, const double* bg,
                             double eps, double tn, double tf, float* gsig, float* gsh, double* signal,
                             uint8_t* touched, const float* ray_g, const float* ray_rgb,
                             const uint8_t* ray_flag, int flags, cudaStream_t s) {
    (void)bg;
    (void)touched;
    (void)flags;
    if (n == 0) return DOT_OK;
    const unsigned grid = unsigned(std::min<int64_t>((n + kBlock - 1) / kBlock, 148 * 8));
    switch (T.basis_count) {
        case 1: render_bwd_replay_kernel<1><<<grid, kBlock, 0, s>>>(T, o, d, n, eps, tn, tf, gsig, gsh, signal, ray_g, ray_rgb, ray_flag); break;
        case 4: render_bwd_replay_kernel<4><<<grid, kBlock, 0, s>>>(T, o, d, n, eps, tn, tf, gsig, gsh, signal, ray_g, ray_rgb, ray_flag); break;
        case 9: render_bwd_replay_kernel<9><<<grid, kBlock, 0, s>>>(T, o, d, n, eps, tn, tf, gsig, gsh, signal, ray_g, ray_rgb, ray_flag); break;
        case 16: render_bwd_replay_kernel<16><<<grid, kBlock, 0, s>>>(T, o, d, n, eps, tn, tf, gsig, gsh, signal, ray_g, ray_rgb, ray_flag); break;
        default: return set_error(DOT_BAD_ARG, "basis_count must be 1, 4, 9 or 16");
    }
    return check_launch("render_bwd_replay_kernel");
}

template <typename K>
static unsigned persistent_grid(K kernel, int64_t n) {
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kBlock, 0);
    const int64_t full = int64_t(sms) * (per_sm > 0 ? per_sm : 1);
    const int64_t need = (n + kBlock - 1) / kBlock;
    return unsigned(need < full ? need : full);
}

// ---------------------------------------------------------------------------
// Camera rendering with in-kernel ray generation (scene_io.py:77-91 pixel
// convention: direction (x+0.5-W/2)/f, -(y+0.5-H/2)/f, -1 rotated by the
// camera's 3x3 and normalised; origin = camera position).  Each warp covers
// an 8x4 pixel tile so its rays walk neighbouring cells; no ray arrays are
// read.  (The direction is computed in fp64 with its own operation order, so
// it may differ from numpy's BLAS product in the last ulp.)

struct CameraDev {
    double r[9];  // row-major cam_to_world rotation
    double t[3];
    double focal;
    int32_t width, height;
};

template <int B>
__global__ void __launch_bounds__(kBlock, DOT_FWD_MINB) render_camera_kernel(
    TreeDev T, CameraDev cam, double bg0, double bg1, double bg2, double eps, float* __restrict__ rgb,
    float* __restrict__ tfin_out, float* __restrict__ depth_out) {
    constexpr int S = pad4(3 * B);
    // block = 4 warps = 16x8 pixels; warp w covers an 8x4 tile
    const int tiles_x = (cam.width + 15) / 16;
    const int bx = blockIdx.x % tiles_x, by = blockIdx.x / tiles_x;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int x = bx * 16 + (w & 1) * 8 + (lane & 7);
    const int y = by * 8 + (w >> 1) * 4 + (lane >> 3);
    if (x >= cam.width || y >= cam.height) return;
    const double xs = (double(x) + 0.5 - 0.5 * cam.width) / cam.focal;
    const double ys = -(double(y) + 0.5 - 0.5 * cam.height) / cam.focal;
    double dx = cam.r[0] * xs + cam.r[1] * ys - cam.r[2];
    double dy = cam.r[3] * xs + cam.r[4] * ys - cam.r[5];
    double dz = cam.r[6] * xs + cam.r[7] * ys - cam.r[8];
    const double nrm = sqrt(dx * dx + dy * dy + dz * dz);
    Tracer tr;
    tr.ox = cam.t[0];
    tr.oy = cam.t[1];
    tr.oz = cam.t[2];
    tr.dx = dx / nrm;
    tr.dy = dy / nrm;
    tr.dz = dz / nrm;
    float basis[B];
    eval_basis<B>(tr.dx, tr.dy, tr.dz, basis);
    double trans = 1.0, c0 = 0.0, c1 = 0.0, c2 = 0.0, dep = 0.0;
    if (tr.init(T, 0.0, __longlong_as_double(0x7ff0000000000000ll))) {
        Leaf L;
        double te, dl;
        PathCache pc;
        while (tr.template next<false, DOT_FWD_PREFETCH>(T, L, te, dl, pc)) {
            const double a = exp_ref(-double(__ldg(T.sigma + L.pid)) * dl);
            const double q = 1.0 - a;
            if (q > 0.0) {
                float e0, e1, e2;
                sh_dot<B>(T.sh + int64_t(L.pid) * S, basis, e0, e1, e2);
                const double tq = trans * q;
                c0 += tq * double(sigmoidf(e0));
                c1 += tq * double(sigmoidf(e1));
                c2 += tq * double(sigmoidf(e2));
                dep += tq * (te + 0.5 * dl);
            }
            trans *= a;
            if (eps > 0.0 && trans < eps) break;
        }
    }
    const int64_t p = int64_t(y) * cam.width + x;
    rgb[3 * p + 0] = float(c0 + trans * bg0);
    rgb[3 * p + 1] = float(c1 + trans * bg1);
    rgb[3 * p + 2] = float(c2 + trans * bg2);
    if (tfin_out) tfin_out[p] = float(trans);
    if (depth_out) depth_out[p] = float(dep);
}

int launch_render_camera(const TreeDev& T, const double* cam_to_world, double focal, int width, int height,
                         const double* bg, double eps, float* rgb, float* tfin, float* depth, cudaStream_t s) {
    if (width <= 0 || height <= 0) return DOT_OK;
    CameraDev cam;
    for (int i = 0; i < 3; ++i) {
        for (int j = 0; j < 3; ++j) cam.r[3 * i + j] = cam_to_world[4 * i + j];
        cam.t[i] = cam_to_world[4 * i + 3];
    }
    cam.focal = focal;
    cam.width = width;
    cam.height = height;
    const unsigned blocks = unsigned(((width + 15) / 16) * ((height + 7) / 8));
    switch (T.basis_count) {
        case 1: render_camera_kernel<1><<<blocks, kBlock, 0, s>>>(T, cam, bg[0], bg[1], bg[2], eps, rgb, tfin, depth); break;
        case 4: render_camera_kernel<4><<<blocks, kBlock, 0, s>>>(T, cam, bg[0], bg[1], bg[2], eps, rgb, tfin, depth); break;
        case 9: render_camera_kernel<9><<<blocks, kBlock, 0, s>>>(T, cam, bg[0], bg[1], bg[2], eps, rgb, tfin, depth); break;
        case 16: render_camera_kernel<16><<<blocks, kBlock, 0, s>>>(T, cam, bg[0], bg[1], bg[2], eps, rgb, tfin, depth); break;
        default: return set_error(DOT_BAD_ARG, "basis_count must be 1, 4, 9 or 16");
    }
    return check_launch("render_camera_kernel");
}

// ---------------------------------------------------------------------------
// Coherence keys: sorting a batch by (origin Morton, octahedral direction
// Morton) puts rays that walk the same cells next to each other -- within a
// camera the direction key is a pixel-space Z-order.  Loss, gradients and
// signal are sums over rays, so the order changes nothing but speed.

__device__ __forceinline__ unsigned long long spread_bits(unsigned long long v, int bits) {
    unsigned long long out = 0;
    for (int i = 0; i < bits; ++i) out |= ((v >> i) & 1ull) << (2 * i);
    return out;
}

__device__ __forceinline__ unsigned long long spread3_10(unsigned v) {
    unsigned long long x = v & 0x3FF;
    x = (x | (x << 16)) & 0x030000FFull;
    x = (x | (x << 8)) & 0x0300F00Full;
    x = (x | (x << 4)) & 0x030C30C3ull;
    x = (x | (x << 2)) & 0x09249249ull;
    return x;
}

// 31-bit variant (int32 keys sort in half the radix passes): origin 4 bits per
// axis (12 bits), direction 10 x 9 bits (19 bits).
__global__ void ray_keys32_kernel(TreeDev T, const double* __restrict__ o, const double* __restrict__ d,
                                  int64_t n, int32_t* __restrict__ keys) {
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= n) return;
    unsigned q[3];
    const double c3[3] = {T.cx, T.cy, T.cz};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        double u = (o[3 * r + a] - (c3[a] - 4.0 * T.half)) / (8.0 * T.half);
        u = fmin(fmax(u, 0.0), 0.999999);
        q[a] = unsigned(u * 16.0);
    }
    const unsigned om = unsigned(spread3_10(q[0]) | (spread3_10(q[1]) << 1) | (spread3_10(q[2]) << 2));
    double x = d[3 * r], y = d[3 * r + 1], z = d[3 * r + 2];
    const double l1 = fabs(x) + fabs(y) + fabs(z);
    x /= l1;
    y /= l1;
    if (z < 0.0) {
        const double tx = (1.0 - fabs(y)) * (x >= 0.0 ? 1.0 : -1.0);
        const double ty = (1.0 - fabs(x)) * (y >= 0.0 ? 1.0 : -1.0);
        x = tx;
        y = ty;
    }
    const unsigned ux = unsigned(fmin(fmax(0.5 * (x + 1.0), 0.0), 0.99999) * 1024.0);
    const unsigned uy = unsigned(fmin(fmax(0.5 * (y + 1.0), 0.0), 0.99999) * 512.0);
    const unsigned dm = unsigned(spread_bits(ux, 10) | (spread_bits(uy, 9) << 1));
    keys[r] = int32_t((om << 19) | dm);
}

int launch_ray_keys32(const TreeDev& T, const double* o, const double* d, int64_t n, int32_t* keys,
                      cudaStream_t s) {
    if (n == 0) return DOT_OK;
    ray_keys32_kernel<<<unsigned((n + 255) / 256), 256, 0, s>>>(T, o, d, n, keys);
    return check_launch("ray_keys32_kernel");
}

__global__ void ray_keys_kernel(TreeDev T, const double* __restrict__ o, const double* __restrict__ d,
                                int64_t n, unsigned long long* __restrict__ keys) {
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= n) return;
    // origin: 10 bits per axis over a box 8x the root cube
    unsigned q[3];
    const double c3[3] = {T.cx, T.cy, T.cz};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        double u = (o[3 * r + a] - (c3[a] - 4.0 * T.half)) / (8.0 * T.half);
        u = fmin(fmax(u, 0.0), 0.999999);
        q[a] = unsigned(u * 1024.0);
    }
    const unsigned long long om = spread3_10(q[0]) | (spread3_10(q[1]) << 1) | (spread3_10(q[2]) << 2);
    // direction: octahedral map to [0,1)^2, 16 bits per axis
    double x = d[3 * r], y = d[3 * r + 1], z = d[3 * r + 2];
    const double l1 = fabs(x) + fabs(y) + fabs(z);
    x /= l1;
    y /= l1;
    if (z < 0.0) {
        const double tx = (1.0 - fabs(y)) * (x >= 0.0 ? 1.0 : -1.0);
        const double ty = (1.0 - fabs(x)) * (y >= 0.0 ? 1.0 : -1.0);
        x = tx;
        y = ty;
    }
    const unsigned ux = unsigned(fmin(fmax(0.5 * (x + 1.0), 0.0), 0.99999) * 65536.0);
    const unsigned uy = unsigned(fmin(fmax(0.5 * (y + 1.0), 0.0), 0.99999) * 65536.0);
    const unsigned long long dm = spread_bits(ux, 16) | (spread_bits(uy, 16) << 1);
    keys[r] = (om << 32) | dm;
}

int launch_ray_keys(const TreeDev& T, const double* o, const double* d, int64_t n, unsigned long long* keys,
                    cudaStream_t s) {
    if (n == 0) return DOT_OK;
    ray_keys_kernel<<<unsigned((n + 255) / 256), 256, 0, s>>>(T, o, d, n, keys);
    return check_launch("ray_keys_kernel");
}

// ---------------------------------------------------------------------------
// Workload statistics (measurement only): per batch totals of traversed
// segments, composited (pre-cut) segments and composited segments with q > 0.

__global__ void __launch_bounds__(kBlock) ray_stats_kernel(TreeDev T, const double* __restrict__ o,
                                                           const double* __restrict__ d, int64_t n,
                                                           double eps, unsigned long long* __restrict__ out) {
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    unsigned long long seg = 0, comp = 0, qpos = 0;
    if (r < n) {
        Tracer tr;
        load_ray(o, d, r, tr);
        if (tr.init(T, 0.0, __longlong_as_double(0x7ff0000000000000ll))) {
            Leaf L;
            double te, dl, trans = 1.0;
            bool cut = false;
            while (tr.next(T, L, te, dl)) {
                ++seg;
                if (cut) continue;
                const double a = exp_ref(-double(__ldg(T.sigma + L.pid)) * dl);
                ++comp;
                if (1.0 - a > 0.0) ++qpos;
                trans *= a;
                if (eps > 0.0 && trans < eps) cut = true;
            }
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        seg += __shfl_down_sync(0xffffffffu, seg, off);
        comp += __shfl_down_sync(0xffffffffu, comp, off);
        qpos += __shfl_down_sync(0xffffffffu, qpos, off);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(out + 0, seg);
        atomicAdd(out + 1, comp);
        atomicAdd(out + 2, qpos);
    }
}

int launch_ray_stats(const TreeDev& T, const double* o, const double* d, int64_t n, double eps,
                     unsigned long long* out, cudaStream_t s) {
    if (n == 0) return DOT_OK;
    ray_stats_kernel<<<unsigned((n + kBlock - 1) / kBlock), kBlock, 0, s>>>(T, o, d, n, eps, out);
    return check_launch("ray_stats_kernel");
}

// ---------------------------------------------------------------------------

static unsigned blocks_for(int64_t n) { return unsigned((n + kBlock - 1) / kBlock); }

__global__ void exp_ref_kernel(const double* __restrict__ x, double* __restrict__ y, int64_t n) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) y[i] = exp_ref(x[i]);
}

int launch_exp_ref(const double* x, double* y, int64_t n, cudaStream_t s) {
    if (n == 0) return DOT_OK;
    exp_ref_kernel<<<blocks_for(n), kBlock, 0, s>>>(x, y, n);
    return check_launch("exp_ref_kernel");
}

// Locate table: one thread per depth-L cell walks the node table from the
// root with the cell's octant bits (integer only) and stores the node word at
// depth L, or the leaf it stops at (flag | depth << 26 | pool id).
__global__ void locate_build_kernel(TreeDev T, int level, int32_t* __restrict__ table) {
    const int64_t cells = int64_t(1) << (3 * level);
    const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c >= cells) return;
    const int mask = (1 << level) - 1;
    const int x = int(c) & mask, y = int(c >> level) & mask, z = int(c >> (2 * level)) & mask;
    int32_t w = T.node[0];
    int dep = 0;
    while (w >= 0 && dep < level) {
        const int b = level - 1 - dep;
        w = T.node[w + (((x >> b) & 1) | (((y >> b) & 1) << 1) | (((z >> b) & 1) << 2))];
        ++dep;
    }
    table[c] = w >= 0 ? w : (kLocLeafFlag | (dep << kLocPidBits) | ~w);
}

int launch_locate_build(const TreeDev& T, int level, int32_t* table, cudaStream_t s) {
    const int64_t cells = int64_t(1) << (3 * level);
    locate_build_kernel<<<blocks_for(cells), kBlock, 0, s>>>(T, level, table);
    return check_launch("locate_build_kernel");
}

// Grid for grid-stride kernels: every SM filled to its occupancy limit.
template <typename K>
static unsigned grid_stride_blocks(K kernel, int64_t n, size_t smem) {
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (smem > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kBlock, smem);
    const int64_t full = int64_t(sms) * (per_sm > 0 ? per_sm : 1);
    const int64_t need = (n + kBlock - 1) / kBlock;
    return unsigned(need < full ? need : full);
}

int launch_trace_count(const TreeDev& T, const double* o, const double* d, int64_t n,
                       double tn, double tf, int64_t* counts, cudaStream_t s) {
    if (n == 0) return DOT_OK;
    if (use_cache(T)) trace_count_kernel<true><<<blocks_for(n), kBlock, 0, s>>>(T, o, d, n, tn, tf, counts);
    else trace_count_kernel<false><<<blocks_for(n), kBlock, 0, s>>>(T, o, d, n, tn, tf, counts);
    return check_launch("trace_count_kernel");
}

int launch_trace_fill(const TreeDev& T, const double* o, const double* d, int64_t n, double tn,
                      double tf, const int64_t* off, int64_t* leaf, double* t, double* dl,
                      cudaStream_t s) {
    if (n == 0) return DOT_OK;
    if (use_cache(T)) trace_fill_kernel<true><<<blocks_for(n), kBlock, 0, s>>>(T, o, d, n, tn, tf, off, leaf, t, dl);
    else trace_fill_kernel<false><<<blocks_for(n), kBlock, 0, s>>>(T, o, d, n, tn, tf, off, leaf, t, dl);
    return check_launch("trace_fill_kernel");
}

// Dispatch on the basis count (compile-time B) and the path cache.
int launch_render_fwd(const TreeDev& T, const double* o, const double* d, int64_t n,
                      const double* bg, double eps, double tn, double tf, float* rgb, float* tfin,
                      float* wsum, float* depth, cudaStream_t s) {
    if (n == 0) return DOT_OK;
    const bool cached = use_cache(T);
#define DOT_FWD(BB, CC)                                                                              \
    { render_fwd_kernel<BB, CC><<<blocks_for(n), kBlock, 0, s>>>(T, o, d, n, bg[0], bg[1], bg[2], eps, \
                                                                 tn, tf, rgb, tfin, wsum, depth); }
    DOT_DISPATCH_B(DOT_FWD)
#undef DOT_FWD
    return check_launch("render_fwd_kernel");
}

int launch_render_bwd(const TreeDev& T, const double* o, const double* d, const double* tgt,
                      int64_t n, const double* bg, double eps, double tn, double tf, double gs,
                      float* gsig, float* gsh, double* signal, uint8_t* touched, double* loss,
                      float* rgb_out, int flags, cudaStream_t s) {
    if (n == 0) return DOT_OK;
    if (flags & 2) {  // legacy one-ray-per-thread kernel, uncached (A/B comparisons)
        const bool cached = false;
#define DOT_BWD(BB, CC)                                                                         \
    { render_bwd_kernel<BB><<<blocks_for(n), kBlock, 0, s>>>(T, o, d, tgt, n, bg[0], bg[1], bg[2], \
                                                             eps, tn, tf, gs, gsig, gsh, signal,   \
                                                             touched, loss, rgb_out, flags); }
        DOT_DISPATCH_B(DOT_BWD)
#undef DOT_BWD
        return check_launch("render_bwd_kernel");
    }
    if (flags & 64)  // record + scatter (backward.cu)
        return launch_render_bwd_two_kernel(T, o, d, tgt, n, bg, eps, tn, tf, gs, gsig, gsh, signal, touched,
                                            loss, rgb_out, flags, s);
    if (!(flags & 16)) {  // default: buffered one-ray-per-thread
        const bool cached = false;
        // default: K = 48 records, one-warp blocks (a finished warp frees its
        // slot at once), pass-2 record loads software-pipelined; bit 7 selects
        // K = 16, bit 10 the earlier K = 32 / 128-thread configuration
        const bool big = (flags & 128) == 0;
        BufSeg* gbuf = nullptr;
        const bool use_gbuf = (flags & 4096) != 0;
        if (use_gbuf) {
            retain_pool_memory();
            if (int st = check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&gbuf),
                                                    size_t(n) * (big ? 32 : 16) * sizeof(BufSeg), s),
                                    "cudaMallocAsync"))
                return st;
        }
#define DOT_BUF_LAUNCH_BLK(BB, KK, MB, GB, BL) DOT_BUF_LAUNCH_PF(BB, KK, MB, GB, BL, false)
#define DOT_BUF_LAUNCH_PF(BB, KK, MB, GB, BL, PP)                                                   \
    render_bwd_buffered_kernel<BB, KK, MB, GB, BL, PP><<<unsigned((n + BL - 1) / BL), BL, 0, s>>>(  \
        T, o, d, tgt, n, bg[0], bg[1], bg[2], eps, tn, tf, gs, touched, rgb_out, flags, gbuf,       \
        AtomicSink{gsig, gsh, signal, loss})
#define DOT_BUF_LAUNCH(BB, KK, MB, GB) DOT_BUF_LAUNCH_BLK(BB, KK, MB, GB, kBlock)
#define DOT_BUF(BB, CC)                                                                           \
    {                                                                                             \
        if (use_gbuf) {                                                                           \
            if (big) DOT_BUF_LAUNCH(BB, 32, 8, true);                                             \
            else DOT_BUF_LAUNCH(BB, 16, 8, true);                                                 \
        } else if (!big) DOT_BUF_LAUNCH(BB, 16, 8, false);                                        \
        else if (flags & 1024) DOT_BUF_LAUNCH(BB, 32, 8, false); /* round-1 configuration */      \
        else DOT_BUF_LAUNCH_PF(BB, 48, 32, false, 32, true);                                      \
    }
        DOT_DISPATCH_B(DOT_BUF)
#undef DOT_BUF
        const int st = check_launch("render_bwd_buffered_kernel");
        if (gbuf) cudaFreeAsync(gbuf, s);
        return st;
    }
    const bool cached = use_cache(T, flags);
    unsigned long long* ctr = nullptr;
    if (int st = check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&ctr), sizeof(*ctr), s), "cudaMallocAsync"))
        return st;
    cudaMemsetAsync(ctr, 0, sizeof(*ctr), s);
#define DOT_BWDP(BB, CC)                                                                           \
    { render_bwd_persistent_kernel<BB, CC><<<persistent_grid(render_bwd_persistent_kernel<BB, CC>, n), \
                                             kBlock, 0, s>>>(T, o, d, tgt, n, bg[0], bg[1], bg[2], eps, \
                                                             tn, tf, gs, gsig, gsh, signal, touched,    \
                                                             loss, rgb_out, flags, ctr); }
    DOT_DISPATCH_B(DOT_BWDP)
#undef DOT_BWDP
    const int st = check_launch("render_bwd_persistent_kernel");
    cudaFreeAsync(ctr, s);
    return st;
}

}  // namespace dot
