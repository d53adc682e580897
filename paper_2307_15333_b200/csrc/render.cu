// render.cu -- traversal, fused forward and fused forward+backward kernels.
//
// One thread per ray.  The reference (octrf/render.py:105-225 over
// octrf/_kernels.py:161-346) materialises every ray's segment list twice
// (count + fill), then composites, then reduces per leaf serially.  Here the
// traversal is streamed: the forward consumes each segment the moment the
// walk produces it; the backward walks each ray once, buffering its
// composited segments in registers/local memory, and reduces leaf gradients
// and signal with vector REDs (REDG.E.ADD.F32x4) issued warp-cooperatively
// (CoopSink), or -- deterministic mode -- emits per-segment records for the
// sorted reduction of sorted.cu.
#include <vector>
#include "dot_tree.cuh"
#include "dot_internal.h"

namespace dot {

constexpr int kBlock = 128;
#ifndef DOT_FWD_MINB
#define DOT_FWD_MINB 8
#endif
constexpr int kFwdMinBlocks = DOT_FWD_MINB;   // forward: 64 registers -> 8 blocks (32 warps) per SM
#ifndef DOT_BWD_RECORDS
#define DOT_BWD_RECORDS 128
#endif
constexpr int kBwdRecords = DOT_BWD_RECORDS;  // composited segments buffered per ray (pass 1 -> pass 2); longer rays resume the walk
// Warp-schedule cost of a ray (what dot_sched_update learns): 0 = composited
// segments, 1 = all traversed segments, 2 = composited + post-cut / 2.  A
// warp lasts as long as its longest ray, and the longest rays are mostly
// post-cut walks (configs[1] batch: p99.9 of 240 traversed segments vs 101
// composited), which the composited count alone does not see.  Measured
// (tools/sweep_variants.sh, 2 runs each): backward 1.83 ms (0, 64 regs) ->
// 1.75 (0, 80 regs) -> 1.71 (1, 80 regs) -> 1.69 ms (2, 80 regs).
#ifndef DOT_SCHED_COST
#define DOT_SCHED_COST 2
#endif
// Register budget of the backward via its one-warp-block residency bound:
// 20 -> 96 registers, no spills (the 25 % carveout keeps ~16-18 blocks per SM
// anyway).  With the cost-ordered launch: 20 (96 registers) 1.451 ms, 24
// (80) 1.508, 28 (72) 1.61-1.64, 16 (128) 1.56; without it 20 and 24 were
// equal and 32 (64 registers, spills) 3-4 % slower.
#ifndef DOT_BWD_MINB
#define DOT_BWD_MINB 20
#endif
// Pass 2 reads its records two ahead (measured 1.69 -> 1.67 ms; at the
// former 64-register cap it spilled and lost).
// Shared-memory carveout hint of the backward (percent of the unified
// L1 / shared array): 25 % (57 KB of shared memory: 16 one-warp blocks of
// 3.5 KB) leaves ~200 KB of L1 for the local-memory records and SH rows,
// which matters more than the 8 warps it costs: step 2.430 -> 2.414 ms
// (driver default = enough shared memory for 24 blocks).
#ifndef DOT_BWD_CARVEOUT
#define DOT_BWD_CARVEOUT 25
#endif
// 20-byte records (colour as 21-bit fixed point): a warp's record lines
// take L1 space for its longest ray, so smaller records buy L1 hits --
// backward 1.747 -> 1.733 ms
#ifndef DOT_REC_PACKED
#define DOT_REC_PACKED 1
#endif
// pass 2 reads records one ahead (two ahead paid before the plan grouped
// rays of similar length into warps: now 1.336 -> 1.320 ms with one)
#ifndef DOT_REC_PREFETCH2
#define DOT_REC_PREFETCH2 0
#endif

static unsigned blocks_for(int64_t n) { return unsigned((n + kBlock - 1) / kBlock); }

// ray_idx (may be NULL) maps a kernel ray slot to its index in the caller's
// arrays: the batch is read in place in any order, e.g. coherence-sorted.
__device__ __forceinline__ int64_t ray_index(const int64_t* __restrict__ ray_idx, int64_t r) {
    return ray_idx ? __ldg(ray_idx + r) : r;
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

#define DOT_DISPATCH_B(MACRO)                                                     \
    switch (T.basis_count) {                                                      \
        case 1: MACRO(1) break;                                                   \
        case 4: MACRO(4) break;                                                   \
        case 9: MACRO(9) break;                                                   \
        case 16: MACRO(16) break;                                                 \
        default: return set_error(DOT_BAD_ARG, "basis_count must be 1, 4, 9 or 16"); \
    }

// ---------------------------------------------------------------------------
// Segment lists (parity / debug path of segment_batch).

__global__ void __launch_bounds__(kBlock) trace_count_kernel(TreeDev T, const double* __restrict__ o,
                                                             const double* __restrict__ d, int64_t n,
                                                             double t_near, double t_far,
                                                             int64_t* __restrict__ counts) {
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= n) return;
    Tracer tr;
    load_ray(o, d, r, tr);
    int64_t c = 0;
    if (tr.init(T, t_near, t_far)) {
        Leaf L;
        double te, dl;
        while (tr.next(T, L, te, dl)) ++c;
    }
    counts[r] = c;
}

__global__ void __launch_bounds__(kBlock) trace_fill_kernel(TreeDev T, const double* __restrict__ o,
                                                            const double* __restrict__ d, int64_t n,
                                                            double t_near, double t_far,
                                                            const int64_t* __restrict__ offsets,
                                                            int64_t* __restrict__ seg_leaf,
                                                            double* __restrict__ seg_t,
                                                            double* __restrict__ seg_delta) {
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= n) return;
    Tracer tr;
    load_ray(o, d, r, tr);
    int64_t s = offsets[r];
    if (tr.init(T, t_near, t_far)) {
        Leaf L;
        double te, dl;
        while (tr.next(T, L, te, dl)) {
            seg_leaf[s] = L.pid;
            seg_t[s] = te;
            seg_delta[s] = dl;
            ++s;
        }
    }
}

// ---------------------------------------------------------------------------
// Fused forward: traverse + composite (composite_kernel, _kernels.py:185-224).

template <int B>
__global__ void __launch_bounds__(kBlock, kFwdMinBlocks) render_fwd_kernel(
    TreeDev T, const double* __restrict__ o, const double* __restrict__ d, int64_t n,
    double bg0, double bg1, double bg2, double eps, double t_near, double t_far,
    float* __restrict__ rgb, float* __restrict__ tfin_out, float* __restrict__ wsum_out,
    float* __restrict__ depth_out) {
    constexpr int S = pad4(3 * B);
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= n) return;
    Tracer tr;
    load_ray(o, d, r, tr);
    float basis[B];
    eval_basis<B>(tr.dx, tr.dy, tr.dz, basis);
    double trans = 1.0, c0 = 0.0, c1 = 0.0, c2 = 0.0, ws = 0.0, dep = 0.0;
    if (tr.init(T, t_near, t_far)) {
        Leaf L;
        double te, dl;
        while (tr.next_prefetch(T, L, te, dl)) {
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
                if (depth_out) dep += tq * (te + 0.5 * dl);
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
// _kernels.py:227-346).  One ray per thread, one-warp blocks (a finished
// warp frees its slot at once; blocks are scheduled dynamically -- a
// grid-stride variant measured 60 % slower behind long rays).
// Pass 1 walks the ray ONCE: it composites up to the early-termination cut,
// marks every traversed leaf touched (post-cut ones too, scatter_kernel
// semantics) and buffers each composited segment (leaf, delta, alpha,
// colour) in a per-thread array.  Pass 2 replays the buffer in order -- no
// second traversal, the colour of q > 0 segments is not recomputed -- and,
// for rays with more than K composited segments, resumes the walk from the
// tracer state saved when the buffer filled.  The reverse-mode quantities
// use the suffix identity suf_i = rgb - prefix_i (carried forward).

struct BufSeg {
    int32_t pid;
    float delta;
    double a;          // alpha = exp(-sigma delta) exactly as pass 1 used it
    float k0, k1, k2;  // colour (NaN: not evaluated in pass 1, q == 0)
    float pad;
    __device__ __forceinline__ void set_colour(float a, float b, float c) {
        k0 = a;
        k1 = b;
        k2 = c;
    }
    __device__ __forceinline__ void colour(float& a, float& b, float& c) const {
        a = k0;
        b = k1;
        c = k2;
    }
    __device__ __forceinline__ void set_alpha(double a_, double) { a = a_; }
    __device__ __forceinline__ void alpha(double& a_, double& q_) const {
        a_ = a;
        q_ = 1.0 - a;
    }
};

// 24-byte record of the atomic sinks (pass 2 only rebuilds T_i and q_i for
// the gradients, within the float tolerance): one f32 holds whichever of
// alpha and q = 1 - alpha is <= 1/2, sign bit set when it is q, so both
// keep ~1e-7 relative precision -- rounding alpha itself would leave q of a
// nearly transparent segment (alpha -> 1) with no significant bits.  The
// deterministic sink keeps the exact f64 alpha so its signal stays
// bit-identical to the reference's.
struct BufSegCompact {
    int32_t pid;
    float delta;
    float aq;
#if DOT_REC_PACKED
    // colour as three 21-bit fixed-point fractions (|error| <= 2.4e-7, far
    // inside the gradients' scale-aware tolerance) + a "not evaluated" bit:
    // 20-byte records
    uint32_t clo, chi;
    __device__ __forceinline__ void set_colour(float a, float b, float c) {
        if (a != a) {
            clo = 0u;
            chi = 0x80000000u;
            return;
        }
        const float sc = 2097151.0f;
        const unsigned long long u0 = __float2uint_rn(a * sc), u1 = __float2uint_rn(b * sc),
                                 u2 = __float2uint_rn(c * sc);
        const unsigned long long w = u0 | (u1 << 21) | (u2 << 42);
        clo = uint32_t(w);
        chi = uint32_t(w >> 32);
    }
    __device__ __forceinline__ void colour(float& a, float& b, float& c) const {
        if (chi & 0x80000000u) {
            a = b = c = __int_as_float(0x7fc00000);
            return;
        }
        const unsigned long long w = (static_cast<unsigned long long>(chi) << 32) | clo;
        const float inv = 1.0f / 2097151.0f;
        a = float(unsigned(w & 0x1FFFFFull)) * inv;
        b = float(unsigned((w >> 21) & 0x1FFFFFull)) * inv;
        c = float(unsigned((w >> 42) & 0x1FFFFFull)) * inv;
    }
#else
    float k0, k1, k2;
    __device__ __forceinline__ void set_colour(float a, float b, float c) {
        k0 = a;
        k1 = b;
        k2 = c;
    }
    __device__ __forceinline__ void colour(float& a, float& b, float& c) const {
        a = k0;
        b = k1;
        c = k2;
    }
#endif
    __device__ __forceinline__ void set_alpha(double a, double q) {
        aq = a > 0.5 ? -float(q) : float(a);  // q == 0 -> -0.0f (sign bit set)
    }
    __device__ __forceinline__ void alpha(double& a, double& q) const {
        if (signbit(aq)) {
            q = -double(aq);
            a = 1.0 - q;
        } else {
            a = double(aq);
            q = 1.0 - a;
        }
    }
};

template <bool EXACT>
struct RecordOf {
    using type = BufSegCompact;
};
template <>
struct RecordOf<true> {
    using type = BufSeg;
};

// Where pass 2 sends each composited segment's gradient contribution.
// AtomicSink: vector REDs straight into the per-leaf buffers (default).
// EmitSink (sorted.cu): one record per segment, reduced per leaf afterwards
// in ray-major order (deterministic mode).
struct AtomicSink {
    static constexpr bool kSmem = false;
    static constexpr bool kExactAlpha = false;
    float* __restrict__ gsig;
    float* __restrict__ gsh;
    double* __restrict__ signal;
    double* __restrict__ loss_sum;
    double* __restrict__ wsum;  // optional per-leaf sum of T_i Q_i (may be NULL)
    double* __restrict__ wmax;  // optional per-leaf max of T_i Q_i (may be NULL)
    __device__ __forceinline__ void bind(float*, float4*) {}
    // pass 1, per composited segment: the signal needs only the exact q (and
    // the weight extras the exact T_i Q_i)
    __device__ __forceinline__ void pass1(int64_t pid, double q, double tq) {
        if (q != 0.0) red_add_f64(signal + pid, q);
        weight_extras(wsum, wmax, pid, tq);
    }
    // an out-of-range ray index: the loss becomes NaN (the call cannot raise)
    __device__ __forceinline__ void bad_ray() { red_add_f64(loss_sum, __longlong_as_double(0x7ff8000000000000ll)); }
    // warp-collective, all 32 lanes (no-op here)
    __device__ __forceinline__ void reserve(int, bool) {}
    template <int B>
    __device__ __forceinline__ void put(bool act, int, int64_t pid, float ds, float w0, float w1, float w2,
                                        const float* basis, double q) {
        constexpr int S = pad4(3 * B);
        if (!act) return;
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

// Warp-cooperative SH-gradient scatter.  Per pass-2 step the lanes that have
// a non-zero contribution publish (pool id | owner lane << 27, w0, w1, w2) in
// shared memory; the warp then walks the published rows in 16-byte chunks,
// consecutive lanes taking consecutive chunks of the same 192-byte row, so
// each row's 12 F32x4 reductions leave the SM as ~2 line-sized L2 requests
// instead of 12 lane-sized ones (the per-lane version is L1->L2 request
// bound).  The owner's SH basis is read from shared memory (written once per
// ray).  dsigma and the signal stay per-lane scalar REDs.
struct CoopSink : AtomicSink {
    static constexpr bool kSmem = true;
    float* sb;    // [32][B] basis of each lane's ray
    float4* sr;   // [32] published rows
    __device__ __forceinline__ void bind(float* b, float4* r) {
        sb = b;
        sr = r;
    }
    template <int B>
    __device__ __forceinline__ void ray_done(int64_t, const float* basis, double) {
        const int lane = threadIdx.x & 31;
#pragma unroll
        for (int b = 0; b < B; ++b) sb[lane * B + b] = basis[b];
    }
    template <int B>
    __device__ __forceinline__ void put(bool act, int, int64_t pid, float ds, float w0, float w1, float w2,
                                        const float*, double q) {
        constexpr int S = pad4(3 * B), CH = S / 4;
        const int lane = threadIdx.x & 31;
        if (act) red_add_f32(gsig + pid, ds);
        const bool has = act && (w0 != 0.f || w1 != 0.f || w2 != 0.f);
        const unsigned m = __ballot_sync(0xffffffffu, has);
        if (m == 0) return;
        if (has) {
            const int idx = __popc(m & ((1u << lane) - 1u));
            sr[idx] = make_float4(__int_as_float(int(pid) | (lane << 27)), w0, w1, w2);
        }
        __syncwarp();
        const int nch = __popc(m) * CH;
        for (int c = lane; c < nch; c += 32) {
            const int ri = c / CH, j = c - ri * CH;
            const float4 rr = sr[ri];
            const int pk = __float_as_int(rr.x);
            const int owner = int(unsigned(pk) >> 27);
            const int64_t p = pk & ((1 << 27) - 1);
            float v[4];
            if constexpr (B == 16) {  // chunk j = channel j / 4, basis 4 (j % 4) .. + 3
                const float w = (j >> 2) == 0 ? rr.y : ((j >> 2) == 1 ? rr.z : rr.w);
                const float4 bv = reinterpret_cast<const float4*>(sb + owner * 16)[j & 3];
                v[0] = w * bv.x;
                v[1] = w * bv.y;
                v[2] = w * bv.z;
                v[3] = w * bv.w;
            } else {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int idx = 4 * j + u;
                    const int k = idx / B;
                    const float w = k == 0 ? rr.y : (k == 1 ? rr.z : rr.w);
                    v[u] = idx < 3 * B ? w * sb[owner * B + idx % B] : 0.f;
                }
            }
            red_add_v4(gsh + p * S + 4 * j, v[0], v[1], v[2], v[3]);
        }
        __syncwarp();
    }
};


// flags: bit 15 = per-lane REDs (AtomicSink instead of CoopSink, chosen at
// launch).  Timing-diagnostic bits exist only in experiment builds
// (-DDOT_DIAG_FLAGS, tools/build_variants.py): bit 0 skip post-cut touched
// marks, bit 13 pass 1 only, bit 14 no reductions -- never in the product.
#ifdef DOT_DIAG_FLAGS
// diagnostic builds only: per-block start / end %globaltimer of the last
// backward launch (tools/bwd_timeline.py), read with dot_diag_timeline
__device__ unsigned long long g_diag_t[2 * 65536];
#endif

template <int B, class Sink>
__global__ void __launch_bounds__(32, DOT_BWD_MINB) render_bwd_buffered_kernel(
    TreeDev T, const double* __restrict__ o, const double* __restrict__ d,
    const double* __restrict__ tgt, const int64_t* __restrict__ ray_idx, int64_t n_pool, int64_t n, double bg0,
    double bg1, double bg2, double eps, double t_near, double t_far, double grad_scale,
    uint8_t* __restrict__ touched, float* __restrict__ rgb_out, int flags, Sink sink,
    const int32_t* __restrict__ warp_order, uint16_t* __restrict__ ray_used, uint16_t* __restrict__ ray_cost) {
    constexpr int S = pad4(3 * B);
    constexpr int K = kBwdRecords;
    double loss = 0.0;
#ifdef DOT_DIAG_FLAGS
    unsigned long long diag_t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(diag_t0));
#endif
    // warp_order: launch order of the 32-ray warps (costliest first, from the
    // learned cost table -- see sched_order_kernel); slot = batch position
    const int64_t wb = warp_order ? int64_t(__ldg(warp_order + blockIdx.x)) : int64_t(blockIdx.x);
    const int64_t slot = wb * 32 + threadIdx.x;
    int64_t r = slot < n ? ray_index(ray_idx, slot) : 0;
    bool valid = slot < n;
    if (valid && (r < 0 || r >= n_pool)) {  // caller's index outside its arrays: skip the ray
        sink.bad_ray();
        valid = false;
        r = 0;
    }
    Tracer tr;
    float basis[B];
    using Rec = typename RecordOf<Sink::kExactAlpha>::type;
    Rec buf[K];
    int used = 0;
#if DOT_SCHED_COST
    int tail = 0;
#endif
    double resume_t = 0.0, resume_nudge = 0.0;
    double R0 = 0.0, R1 = 0.0, R2 = 0.0, g0 = 0.0, g1 = 0.0, g2 = 0.0;
    if (valid) {
        load_ray(o, d, r, tr);
        eval_basis<B>(tr.dx, tr.dy, tr.dz, basis);
        double trans = 1.0, c0 = 0.0, c1 = 0.0, c2 = 0.0;
        if (tr.init(T, t_near, t_far)) {
            Leaf L;
            double te, dl;
            bool cut = false;
            // one segment of pass 1: touched mark; before the cut, alpha, the
            // signal, shading, colour and the record for pass 2
            auto segment = [&](const int32_t pid, const double te_c, const double dl_c) {
                touched[pid] = 1;
                if (cut) {  // post-cut: touched only
#if DOT_SCHED_COST
                    ++tail;
#endif
                    return;
                }
                const double a = exp_ref(-double(__ldg(T.sigma + pid)) * dl_c);
                const double q = 1.0 - a;
                const double tq = trans * q;
#ifdef DOT_DIAG_FLAGS
                if (!(flags & 16384))
#endif
                sink.pass1(pid, q, tq);
                float k0 = __int_as_float(0x7fc00000), k1 = k0, k2 = k0;
                if (q > 0.0) {
                    float e0, e1, e2;
                    sh_dot<B>(T.sh + int64_t(pid) * S, basis, e0, e1, e2);
                    k0 = sigmoidf(e0);
                    k1 = sigmoidf(e1);
                    k2 = sigmoidf(e2);
                    c0 += tq * double(k0);
                    c1 += tq * double(k1);
                    c2 += tq * double(k2);
                }
                if (used < K) {
                    Rec e;
                    e.pid = pid;
                    e.delta = float(dl_c);
                    e.set_alpha(a, q);
                    e.set_colour(k0, k1, k2);
                    buf[used] = e;
                } else if (used == K) {  // buffer full: remember where pass 2 resumes
                    resume_t = te_c;
                    resume_nudge = tr.nudge0;
                }
                ++used;
                trans *= a;
                if (eps > 0.0 && trans < eps) cut = true;
            };
            while (tr.next_prefetch(T, L, te, dl, !cut)) segment(L.pid, te, dl);

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
#if DOT_SCHED_COST == 1
        const int cost = used + tail;
#elif DOT_SCHED_COST == 2
        const int cost = used + (tail >> 1);
#else
        const int cost = used;
#endif
        if (ray_used) ray_used[slot] = uint16_t(cost < 65535 ? cost : 65535);
        if (ray_cost) ray_cost[r] = uint16_t(cost < 65535 ? cost : 65535);
#ifdef DOT_DIAG_FLAGS
        if (flags & 8192) used = 0;
#endif
    }
    __syncwarp();
    if constexpr (Sink::kSmem) {
        __shared__ float s_basis[32 * B];
        __shared__ float4 s_rec[32];
        sink.bind(s_basis, s_rec);
    }
    sink.reserve(used, valid);
    // pass 2 runs convergent (max over the warp's rays) so that sinks may
    // cooperate across lanes; lanes past their own count only take part
    const int maxu = __reduce_max_sync(0xffffffffu, valid ? used : 0);
    if (valid) sink.template ray_done<B>(r, basis, loss);
    __syncwarp();
    double s0 = R0, s1 = R1, s2 = R2, Ti = 1.0;
    if (used > K) {  // segment K onwards come from a resumed walk
        tr.t = resume_t;
        tr.nudge = resume_nudge;
    }
    Rec nxt;
    if (used > 0) nxt = buf[0];
#if DOT_REC_PREFETCH2
    Rec nxt2;
    if (used > 1) nxt2 = buf[1];
#endif
    for (int i = 0; i < maxu; ++i) {
        const bool act = valid && i < used;
        int64_t pid = 0;
        double a = 1.0, q = 0.0, dl = 0.0;
        float k0 = 0.f, k1 = 0.f, k2 = 0.f;
        if (act) {
            if (i < K) {  // software pipeline: entry i+1 is in flight while i is scattered
                const Rec e = nxt;
#if DOT_REC_PREFETCH2
                nxt = nxt2;
                if (i + 2 < used && i + 2 < K) nxt2 = buf[i + 2];
#else
                if (i + 1 < used && i + 1 < K) nxt = buf[i + 1];
#endif
                pid = e.pid;
                e.alpha(a, q);
                dl = e.delta;
                e.colour(k0, k1, k2);
            } else {
                Leaf L;
                double te;
                tr.next(T, L, te, dl);
                pid = L.pid;
                a = exp_ref(-double(__ldg(T.sigma + pid)) * dl);
                q = 1.0 - a;
                k0 = __int_as_float(0x7fc00000);
            }
            if (k0 != k0) {  // q == 0 in pass 1: the colour is still needed for dsigma
                float e0, e1, e2;
                sh_dot<B>(T.sh + pid * S, basis, e0, e1, e2);
                k0 = sigmoidf(e0);
                k1 = sigmoidf(e1);
                k2 = sigmoidf(e2);
            }
        }
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
#ifdef DOT_DIAG_FLAGS
        if (flags & 16384) {  // keep the arithmetic alive without reducing
            if (ds == 12345.0 && w0 == 1.f) touched[0] = uint8_t(w1 + w2);
            continue;
        }
#endif
        sink.template put<B>(act, i, pid, float(ds), w0, w1, w2, basis, q);
    }
    sink.loss(loss);
#ifdef DOT_DIAG_FLAGS
    if (threadIdx.x == 0 && blockIdx.x < 65536) {
        unsigned long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        g_diag_t[2 * blockIdx.x] = diag_t0;
        g_diag_t[2 * blockIdx.x + 1] = t1;
    }
#endif
}

#ifdef DOT_DIAG_FLAGS
extern "C" int dot_diag_timeline(unsigned long long* out, int n) {
    return cudaMemcpyFromSymbol(out, g_diag_t, sizeof(unsigned long long) * 2 * size_t(n)) == cudaSuccess ? 0 : 3;
}
#endif

int launch_render_bwd(const TreeDev& T, const double* o, const double* d, const double* tgt,
                      const int64_t* ray_idx, int64_t n_pool, const int32_t* warp_order, uint16_t* ray_used,
                      uint16_t* ray_cost,
                      int64_t n, const double* bg, double eps, double tn, double tf, double gs, float* gsig,
                      float* gsh, double* signal, uint8_t* touched, double* loss, float* rgb_out,
                      double* wsum, double* wmax, int flags, cudaStream_t s) {
    if (n == 0) return DOT_OK;
    const unsigned grid = unsigned((n + 31) / 32);
    // default: warp-cooperative SH scatter; flag bit 15: per-lane REDs
    const bool coop = (flags & 32768) == 0;
    AtomicSink as{gsig, gsh, signal, loss, wsum, wmax};
    CoopSink cs;
    using CoopT = CoopSink;
    static_cast<AtomicSink&>(cs) = as;
    cs.sb = nullptr;
    cs.sr = nullptr;
#define DOT_BWD(BB)                                                                                  \
    if (DOT_BWD_CARVEOUT >= 0)                                                                       \
        cudaFuncSetAttribute(render_bwd_buffered_kernel<BB, CoopT>,                                  \
                             cudaFuncAttributePreferredSharedMemoryCarveout, DOT_BWD_CARVEOUT);      \
    if (coop)                                                                                        \
        render_bwd_buffered_kernel<BB, CoopT><<<grid, 32, 0, s>>>(                                   \
            T, o, d, tgt, ray_idx, n_pool, n, bg[0], bg[1], bg[2], eps, tn, tf, gs, touched, rgb_out, flags, cs, \
            warp_order, ray_used, ray_cost);                                                         \
    else                                                                                             \
        render_bwd_buffered_kernel<BB, AtomicSink><<<grid, 32, 0, s>>>(                              \
            T, o, d, tgt, ray_idx, n_pool, n, bg[0], bg[1], bg[2], eps, tn, tf, gs, touched, rgb_out, flags, as, \
            warp_order, ray_used, ray_cost);
    DOT_DISPATCH_B(DOT_BWD)
#undef DOT_BWD
    return check_launch("render_bwd_buffered_kernel");
}

// Record sink of the deterministic (sorted) backward: pass 2 writes one
// record per composited segment -- key (pool id << ray_bits | original ray
// index), (dsigma, w0, w1, w2) f32 and q f64 -- into slots reserved per ray
// with one warp-aggregated atomicAdd; the ray's SH basis and squared error
// go to per-ray arrays (original index).  A ray whose records do not fit is
// counted in ctr[1] and writes nothing (the host retries with more room).
struct EmitSink {
    static constexpr bool kSmem = false;
    static constexpr bool kExactAlpha = true;
    __device__ __forceinline__ void pass1(int64_t, double, double) {}
    __device__ __forceinline__ void bad_ray() {}  // ray_index validated as a permutation on the host
    __device__ __forceinline__ void bind(float*, float4*) {}
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
        orig = r;  // r is already the original batch index (ray_idx applied)
#pragma unroll
        for (int b = 0; b < B; ++b) a.basis[orig * B + b] = basis[b];
        a.loss_ray[orig] = loss;
    }
    template <int B>
    __device__ __forceinline__ void put(bool act, int i, int64_t pid, float ds, float w0, float w1, float w2,
                                        const float*, double q) {
        if (!act || base < 0) return;
        const int64_t k = base + i;
        a.keys[k] = (static_cast<unsigned long long>(pid) << a.ray_bits) |
                    static_cast<unsigned long long>(orig);
        a.rec[k] = make_float4(ds, w0, w1, w2);
        a.recq[k] = q;
    }
    __device__ __forceinline__ void loss(double) {}
};

int launch_render_bwd_emit(const TreeDev& T, const double* o, const double* d, const double* tgt,
                           const int64_t* ray_idx, const int32_t* warp_order, uint16_t* ray_used, int64_t n,
                           const double* bg, double eps, double tn, double tf, double gs, uint8_t* touched,
                           const EmitArgs& ea, cudaStream_t s) {
    if (n == 0) return DOT_OK;
    EmitSink sink;
    sink.a = ea;
    sink.base = -1;
    sink.orig = 0;
#define DOT_EMIT(BB)                                                                                 \
    render_bwd_buffered_kernel<BB, EmitSink><<<unsigned((n + 31) / 32), 32, 0, s>>>(                 \
        T, o, d, tgt, ray_idx, n, n, bg[0], bg[1], bg[2], eps, tn, tf, gs, touched, nullptr, 0, sink,   \
        warp_order, ray_used, nullptr);
    DOT_DISPATCH_B(DOT_EMIT)
#undef DOT_EMIT
    return check_launch("render_bwd_buffered_kernel<emit>");
}

int launch_trace_count(const TreeDev& T, const double* o, const double* d, int64_t n,
                       double tn, double tf, int64_t* counts, cudaStream_t s) {
    if (n == 0) return DOT_OK;
    trace_count_kernel<<<blocks_for(n), kBlock, 0, s>>>(T, o, d, n, tn, tf, counts);
    return check_launch("trace_count_kernel");
}

int launch_trace_fill(const TreeDev& T, const double* o, const double* d, int64_t n, double tn,
                      double tf, const int64_t* off, int64_t* leaf, double* t, double* dl,
                      cudaStream_t s) {
    if (n == 0) return DOT_OK;
    trace_fill_kernel<<<blocks_for(n), kBlock, 0, s>>>(T, o, d, n, tn, tf, off, leaf, t, dl);
    return check_launch("trace_fill_kernel");
}

int launch_render_fwd(const TreeDev& T, const double* o, const double* d, int64_t n,
                      const double* bg, double eps, double tn, double tf, float* rgb, float* tfin,
                      float* wsum, float* depth, cudaStream_t s) {
    if (n == 0) return DOT_OK;
#define DOT_FWD(BB)                                                                                  \
    render_fwd_kernel<BB><<<blocks_for(n), kBlock, 0, s>>>(T, o, d, n, bg[0], bg[1], bg[2], eps, tn, \
                                                           tf, rgb, tfin, wsum, depth);
    DOT_DISPATCH_B(DOT_FWD)
#undef DOT_FWD
    return check_launch("render_fwd_kernel");
}

// ---------------------------------------------------------------------------
// Signal-only forward (the signal half of grad_kernel + scatter_kernel,
// _kernels.py:249-282 and 337, as SignalBuffer.accumulate consumes it,
// signals.py:58-69): per composited segment signal[leaf] += Q (cut-aware),
// plus the optional weight extras and touched marks.  No SH row is read and
// no gradient reduced: calibration-only passes cost a traversal plus one
// sigma gather per segment.  The walk stops at the cut unless touched marks
// (which include post-cut leaves) are requested.

__global__ void __launch_bounds__(kBlock, kFwdMinBlocks) signal_fwd_kernel(
    TreeDev T, const double* __restrict__ o, const double* __restrict__ d, const int64_t* __restrict__ ray_idx,
    int64_t n_pool, int64_t n, double eps, double t_near, double t_far, double* __restrict__ signal,
    double* __restrict__ wsum, double* __restrict__ wmax, uint8_t* __restrict__ touched,
    unsigned long long* __restrict__ invalid) {
    const int64_t slot = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (slot >= n) return;
    const int64_t r = ray_index(ray_idx, slot);
    if (r < 0 || r >= n_pool) {
        if (invalid) atomicAdd(invalid, 1ull);
        return;
    }
    Tracer tr;
    load_ray(o, d, r, tr);
    if (!tr.init(T, t_near, t_far)) return;
    double trans = 1.0;
    bool cut = false;
    Leaf L;
    double te, dl;
    while (tr.next(T, L, te, dl)) {
        if (touched) touched[L.pid] = 1;
        if (cut) continue;
        const double a = exp_ref(-double(__ldg(T.sigma + L.pid)) * dl);
        const double q = 1.0 - a;
        if (signal && q != 0.0) red_add_f64(signal + L.pid, q);
        weight_extras(wsum, wmax, L.pid, trans * q);
        trans *= a;
        if (eps > 0.0 && trans < eps) {
            cut = true;
            if (!touched) break;
        }
    }
}

int launch_signal_fwd(const TreeDev& T, const double* o, const double* d, const int64_t* ray_idx, int64_t n_pool,
                      int64_t n, double eps, double tn, double tf, double* signal, double* wsum, double* wmax,
                      uint8_t* touched, unsigned long long* invalid, cudaStream_t s) {
    if (n == 0) return DOT_OK;
    signal_fwd_kernel<<<blocks_for(n), kBlock, 0, s>>>(T, o, d, ray_idx, n_pool, n, eps, tn, tf, signal, wsum,
                                                       wmax, touched, invalid);
    return check_launch("signal_fwd_kernel");
}

// ---------------------------------------------------------------------------
// Per-ray schedule cost (no reference counterpart; only orders launches):
// composited + post-cut / 2 segments -- the metric the backward reports in
// ray_used (DOT_SCHED_COST 2), so a ray pool's costs computed once and
// refreshed by every backward predict each warp's duration closely.

__global__ void __launch_bounds__(kBlock, kFwdMinBlocks) ray_cost_kernel(
    TreeDev T, const double* __restrict__ o, const double* __restrict__ d, const int64_t* __restrict__ ray_idx,
    int64_t n_pool, int64_t n, double eps, double t_near, double t_far, uint16_t* __restrict__ cost) {
    const int64_t slot = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (slot >= n) return;
    const int64_t r = ray_index(ray_idx, slot);
    int used = 0, tail = 0;
    if (r >= 0 && r < n_pool) {
        Tracer tr;
        load_ray(o, d, r, tr);
        if (tr.init(T, t_near, t_far)) {
            double trans = 1.0;
            bool cut = false;
            Leaf L;
            double te, dl;
            while (tr.next(T, L, te, dl)) {
                if (cut) {
                    ++tail;
                    continue;
                }
                ++used;
                trans *= exp_ref(-double(__ldg(T.sigma + L.pid)) * dl);
                if (eps > 0.0 && trans < eps) cut = true;
            }
        }
    }
    const int c = used + (tail >> 1);
    cost[slot] = uint16_t(c < 65535 ? c : 65535);
}

int launch_ray_costs(const TreeDev& T, const double* o, const double* d, const int64_t* ray_idx, int64_t n_pool,
                     int64_t n, double eps, double tn, double tf, uint16_t* cost, cudaStream_t s) {
    if (n == 0) return DOT_OK;
    ray_cost_kernel<<<blocks_for(n), kBlock, 0, s>>>(T, o, d, ray_idx, n_pool, n, eps, tn, tf, cost);
    return check_launch("ray_cost_kernel");
}

// Warp launch order from per-slot costs: warp cost = max over its 32 rays
// (a warp lasts as long as its longest ray), chunks of `chunk` consecutive
// warps ranked by their costliest warp, descending (longest-first packing),
// via a counting sort over capped costs.
constexpr int kCostBins = 1024;

// one thread per batch slot: warp w's cost = max over its 32 slots (warp
// reduction), then chunk costs (max over `chunk` warps) and their histogram
__global__ void __launch_bounds__(256) cost_warp_kernel(const uint16_t* __restrict__ ray_cost, int64_t n_costs,
                                                        const int64_t* __restrict__ ray_idx, int64_t n,
                                                        uint16_t* __restrict__ warp_cost) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t nw = (n + 31) / 32;
    unsigned c = 0;
    if (i < n) {
        const int64_t r = ray_index(ray_idx, i);
        if (r >= 0 && r < n_costs) c = __ldg(ray_cost + r);
    }
    c = __reduce_max_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0 && (i >> 5) < nw) warp_cost[i >> 5] = uint16_t(min(c, unsigned(kCostBins - 1)));
}

__global__ void __launch_bounds__(256) cost_hist_kernel(const uint16_t* __restrict__ warp_cost, int64_t n, int chunk,
                                                        uint16_t* __restrict__ chunk_cost, int* __restrict__ hist) {
    const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t nw = (n + 31) / 32, nfull = nw / chunk;
    if (c >= nfull) return;  // a short last chunk is placed last (cost_place_kernel)
    unsigned m = 0;
    for (int64_t w = c * chunk; w < (c + 1) * chunk; ++w) m = max(m, unsigned(warp_cost[w]));
    chunk_cost[c] = uint16_t(m);
    atomicAdd(hist + (kCostBins - 1 - int(m)), 1);
}

__global__ void __launch_bounds__(kCostBins) cost_scan_kernel(int* __restrict__ hist) {
    __shared__ int v[kCostBins];
    const int t = threadIdx.x;
    const int own = hist[t];
    v[t] = own;
    __syncthreads();
    for (int off = 1; off < kCostBins; off <<= 1) {
        const int u = t >= off ? v[t - off] : 0;
        __syncthreads();
        v[t] += u;
        __syncthreads();
    }
    hist[t] = v[t] - own;  // exclusive start of each bin
}

__global__ void __launch_bounds__(256) cost_place_kernel(const uint16_t* __restrict__ chunk_cost, int64_t n, int chunk,
                                                         int* __restrict__ start, int32_t* __restrict__ warp_order) {
    const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t nw = (n + 31) / 32, nfull = nw / chunk;
    if (c > nfull) return;
    int64_t w0, w1, dst;
    if (c == nfull) {  // the short last chunk (if any) goes last
        w0 = nfull * chunk;
        w1 = nw;
        dst = w0;
    } else {
        w0 = c * chunk;
        w1 = w0 + chunk;
        dst = int64_t(atomicAdd(start + (kCostBins - 1 - int(chunk_cost[c])), 1)) * chunk;
    }
    // a chunk's warps keep their (coherent) order
    for (int64_t w = w0; w < w1; ++w) warp_order[dst + (w - w0)] = int32_t(w);
}

int launch_sched_order_costs(const uint16_t* slot_cost, int64_t n_costs, const int64_t* ray_idx, int64_t n,
                             int chunk, int32_t* warp_order, cudaStream_t s) {
    const int64_t nw = (n + 31) / 32;
    if (nw == 0) return DOT_OK;
    const int64_t nc = (nw + chunk - 1) / chunk;
    retain_pool_memory();
    uint16_t* cc = nullptr;
    uint16_t* wc = nullptr;
    int* hist = nullptr;
    int st = check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&cc), sizeof(uint16_t) * nc, s), "cudaMallocAsync");
    if (st == DOT_OK)
        st = check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&wc), sizeof(uint16_t) * nw, s), "cudaMallocAsync");
    if (st == DOT_OK)
        st = check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&hist), sizeof(int) * kCostBins, s), "cudaMallocAsync");
    if (st == DOT_OK) st = check_cuda(cudaMemsetAsync(hist, 0, sizeof(int) * kCostBins, s), "cudaMemsetAsync");
    if (st == DOT_OK) {
        cost_warp_kernel<<<unsigned((nw * 32 + 255) / 256), 256, 0, s>>>(slot_cost, n_costs, ray_idx, n, wc);
        cost_hist_kernel<<<unsigned((nc + 255) / 256), 256, 0, s>>>(wc, n, chunk, cc, hist);
        cost_scan_kernel<<<1, kCostBins, 0, s>>>(hist);
        cost_place_kernel<<<unsigned((nc + 256) / 256), 256, 0, s>>>(cc, n, chunk, hist, warp_order);
        st = check_launch("sched_order_costs");
    }
    if (cc) cudaFreeAsync(cc, s);
    if (wc) cudaFreeAsync(wc, s);
    if (hist) cudaFreeAsync(hist, s);
    return st;
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

// Many views per launch: block b renders tile b % tiles of view b / tiles,
// so one launch drains one tail instead of one per view.
template <int B>
__global__ void __launch_bounds__(kBlock, kFwdMinBlocks) render_camera_kernel(
    TreeDev T, const CameraDev* __restrict__ cams, int tiles, double bg0, double bg1, double bg2,
    double eps, float* __restrict__ rgb_all, float* __restrict__ tfin_all, float* __restrict__ depth_all) {
    constexpr int S = pad4(3 * B);
    const int v = blockIdx.x / tiles, tile = blockIdx.x - v * tiles;
    const CameraDev& cam = cams[v];
    const int64_t pix = int64_t(cam.width) * cam.height;
    float* __restrict__ rgb = rgb_all + 3 * pix * v;
    float* __restrict__ tfin_out = tfin_all ? tfin_all + pix * v : nullptr;
    float* __restrict__ depth_out = depth_all ? depth_all + pix * v : nullptr;
    // block = 4 warps = 16x8 pixels; warp w covers an 8x4 tile
    const int tiles_x = (cam.width + 15) / 16;
    const int bx = tile % tiles_x, by = tile / tiles_x;
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
        while (tr.next_prefetch(T, L, te, dl)) {
            const double a = exp_ref(-double(__ldg(T.sigma + L.pid)) * dl);
            const double q = 1.0 - a;
            if (q > 0.0) {
                float e0, e1, e2;
                sh_dot<B>(T.sh + int64_t(L.pid) * S, basis, e0, e1, e2);
                const double tq = trans * q;
                c0 += tq * double(sigmoidf(e0));
                c1 += tq * double(sigmoidf(e1));
                c2 += tq * double(sigmoidf(e2));
                if (depth_out) dep += tq * (te + 0.5 * dl);
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

int launch_render_cameras(const TreeDev& T, const double* cam_to_world, const double* focal, int n_views,
                          int width, int height, const double* bg, double eps, float* rgb, float* tfin,
                          float* depth, cudaStream_t s) {
    if (width <= 0 || height <= 0 || n_views <= 0) return DOT_OK;
    std::vector<CameraDev> cams(static_cast<size_t>(n_views));
    for (int v = 0; v < n_views; ++v) {
        CameraDev& cam = cams[size_t(v)];
        const double* m = cam_to_world + 16 * v;
        for (int i = 0; i < 3; ++i) {
            for (int j = 0; j < 3; ++j) cam.r[3 * i + j] = m[4 * i + j];
            cam.t[i] = m[4 * i + 3];
        }
        cam.focal = focal[v];
        cam.width = width;
        cam.height = height;
    }
    retain_pool_memory();
    CameraDev* d_cams = nullptr;
    if (int st = check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&d_cams), cams.size() * sizeof(CameraDev), s),
                            "cudaMallocAsync"))
        return st;
    // pageable source: the copy is staged before cudaMemcpyAsync returns
    if (int st = check_cuda(cudaMemcpyAsync(d_cams, cams.data(), cams.size() * sizeof(CameraDev),
                                            cudaMemcpyHostToDevice, s), "memcpy")) {
        cudaFreeAsync(d_cams, s);
        return st;
    }
    const int tiles = ((width + 15) / 16) * ((height + 7) / 8);
    const unsigned blocks = unsigned(int64_t(tiles) * n_views);
#define DOT_CAM(BB)                                                                                  \
    render_camera_kernel<BB><<<blocks, kBlock, 0, s>>>(T, d_cams, tiles, bg[0], bg[1], bg[2], eps, rgb, tfin, \
                                                       depth);
    DOT_DISPATCH_B(DOT_CAM)
#undef DOT_CAM
    const int st = check_launch("render_camera_kernel");
    cudaFreeAsync(d_cams, s);
    return st;
}

int launch_render_camera(const TreeDev& T, const double* cam_to_world, double focal, int width, int height,
                         const double* bg, double eps, float* rgb, float* tfin, float* depth, cudaStream_t s) {
    return launch_render_cameras(T, cam_to_world, &focal, 1, width, height, bg, eps, rgb, tfin, depth, s);
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
                                  const int64_t* __restrict__ ray_idx, int64_t n_pool, int64_t n,
                                  int32_t* __restrict__ keys) {
    const int64_t slot = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (slot >= n) return;
    const int64_t r = ray_index(ray_idx, slot);
    if (r < 0 || r >= n_pool) {  // out of range: the consumer rejects the ray; the key only orders
        keys[slot] = 0;
        return;
    }
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
    keys[slot] = int32_t((om << 19) | dm);
}

// keys[i] = pool_keys[ray_index[i]]: a batch's keys from its pool's
// precomputed ones (4 B per ray instead of re-reading its 48 B of rays)
__global__ void __launch_bounds__(256) gather_keys_kernel(const int32_t* __restrict__ pool_keys,
                                                          const int64_t* __restrict__ ray_idx, int64_t n_pool,
                                                          int64_t n, int32_t* __restrict__ keys) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t r = __ldg(ray_idx + i);
    keys[i] = (r >= 0 && r < n_pool) ? __ldg(pool_keys + r) : 0;
}

int launch_gather_keys(const int32_t* pool_keys, const int64_t* ray_idx, int64_t n_pool, int64_t n, int32_t* keys,
                       cudaStream_t s) {
    if (n == 0) return DOT_OK;
    gather_keys_kernel<<<unsigned((n + 255) / 256), 256, 0, s>>>(pool_keys, ray_idx, n_pool, n, keys);
    return check_launch("gather_keys_kernel");
}

int launch_ray_keys32(const TreeDev& T, const double* o, const double* d, const int64_t* ray_idx, int64_t n_pool,
                      int64_t n, int32_t* keys, cudaStream_t s) {
    if (n == 0) return DOT_OK;
    ray_keys32_kernel<<<unsigned((n + 255) / 256), 256, 0, s>>>(T, o, d, ray_idx, n_pool, n, keys);
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
// Warp scheduling from a learned cost table.  A backward warp's duration is
// set by its rays' composited-segment counts (ncu/globaltimer: correlation
// 0.95), and neighbouring rays in coherence-key order cost alike: the count
// of the warp that started at key bucket k (top 24 bits of the 31-bit key:
// origin cell + a ~12x12-pixel direction cell) predicts the next batch's
// warps in that bucket with Spearman 0.93.  sched_update keeps a decaying
// max of the per-warp max count per bucket (u16, 2^24 entries); sched_order ranks
// chunks of 64 consecutive warps (coherence kept inside a chunk) by their
// costliest predicted warp, descending, so the long rays start first
// instead of forming the wave tail.  Results never depend on the order.

constexpr int kSchedBits = 24;
constexpr int kSchedSort = 2048;    // chunks ranked per launch (one block, bitonic in shared memory)
#ifndef DOT_SCHED_CHUNK
#define DOT_SCHED_CHUNK 16
#endif
constexpr int kSchedMinChunk = DOT_SCHED_CHUNK;  // warps per chunk (coherence kept inside a chunk)

constexpr int kSchedFineBits = 27;  // second, finer table (fallback to the coarse one when empty)

__device__ __forceinline__ uint32_t sched_bucket(int32_t key) {
    return uint32_t(key) >> (31 - kSchedBits);
}
__device__ __forceinline__ uint32_t sched_fine(int32_t key) {
    return uint32_t(key) >> (31 - kSchedFineBits);
}
// table layout: [2^kSchedBits coarse | 2^kSchedFineBits fine] u16
__device__ __forceinline__ unsigned sched_lookup(const uint16_t* __restrict__ table, int32_t key) {
    const unsigned f = __ldg(table + (1u << kSchedBits) + sched_fine(key));
    return f ? f : unsigned(__ldg(table + sched_bucket(key)));
}

__global__ void __launch_bounds__(256) sched_update_kernel(const int32_t* __restrict__ keys,
                                                           const uint16_t* __restrict__ ray_used, int64_t n,
                                                           uint16_t* __restrict__ table) {
    const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t r = w * 32 + lane;
    unsigned u = r < n ? ray_used[r] : 0u;
    u = __reduce_max_sync(0xffffffffu, u);
    if (lane == 0 && w * 32 < n) {
        const int32_t k = keys[w * 32];
        // decaying max: a bucket keeps its costliest recent warp (several
        // consecutive warps can share a bucket; the chunk cost is their max)
        uint16_t* t = table + sched_bucket(k);
        unsigned old = *t;
        *t = uint16_t(max(u, (old * 7u) >> 3));
        t = table + (1u << kSchedBits) + sched_fine(k);
        old = *t;
        *t = uint16_t(max(u, (old * 7u) >> 3));
    }
}

// Predicted cost of every chunk (one thread per chunk, many blocks: the
// table lookups are scattered).
__global__ void __launch_bounds__(256) sched_cost_kernel(const int32_t* __restrict__ keys, int64_t n, int chunk,
                                                         const uint16_t* __restrict__ table,
                                                         unsigned* __restrict__ cost_out) {
    const int c = int(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t nw = (n + 31) / 32;
    const int nc = int((nw + chunk - 1) / chunk);
    if (c >= nc) return;
    unsigned cost = 0;
    // a partial last chunk keeps cost 0 and the largest id: it sorts last,
    // so every other position maps to a full chunk
    if (!(c == nc - 1 && nw % chunk != 0)) {
        const int64_t w1 = min(nw, int64_t(c + 1) * chunk);
        for (int64_t w = int64_t(c) * chunk; w < w1; ++w)
            cost = max(cost, sched_lookup(table, __ldg(keys + w * 32)));
    }
    cost_out[c] = cost;
}

// Chunks ordered by descending predicted cost with a counting sort over
// the (capped) cost values -- the order within a cost value is whatever the
// shared-memory atomics give: launch order only, results never depend on it.
__global__ void __launch_bounds__(1024) sched_order_kernel(const unsigned* __restrict__ chunk_cost, int64_t n,
                                                           int chunk, int32_t* __restrict__ warp_order) {
    constexpr int kBins = 1024;
    __shared__ int hist[kBins];
    __shared__ int start[kBins];
    __shared__ int sorted[kSchedSort];
    const int64_t nw = (n + 31) / 32;
    const int nc = int((nw + chunk - 1) / chunk);  // <= kSchedSort (host checks)
    const int t = threadIdx.x;
    hist[t] = 0;
    __syncthreads();
    int bin[kSchedSort / 1024];
#pragma unroll
    for (int k = 0; k < kSchedSort / 1024; ++k) {
        const int c = t + 1024 * k;
        // descending cost; the partial last chunk (cost 0) must come last: bin kBins-1
        bin[k] = c < nc ? (kBins - 1) - int(min(chunk_cost[c], unsigned(kBins - 2))) - (c == nc - 1 && nw % chunk ? 0 : 1) : -1;
        if (c == nc - 1 && nw % chunk) bin[k] = kBins - 1;
        if (bin[k] >= 0) atomicAdd(&hist[bin[k]], 1);
    }
    __syncthreads();
    // exclusive scan of hist (1024 bins, one per thread)
    int v = hist[t];
    for (int off = 1; off < kBins; off <<= 1) {
        __syncthreads();
        const int u = t >= off ? hist[t - off] : 0;
        __syncthreads();
        hist[t] += u;
    }
    __syncthreads();
    start[t] = hist[t] - v;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kSchedSort / 1024; ++k) {
        const int c = t + 1024 * k;
        if (bin[k] >= 0) sorted[atomicAdd(&start[bin[k]], 1)] = c;
    }
    __syncthreads();
    for (int64_t i = t; i < nw; i += blockDim.x) {
        const int64_t q = i / chunk, off = i - q * chunk;
        warp_order[i] = int32_t(int64_t(sorted[q]) * chunk + off);
    }
}

int launch_sched_order(const int32_t* keys, int64_t n, const uint16_t* table, int32_t* warp_order, cudaStream_t s) {
    const int64_t nw = (n + 31) / 32;
    if (nw == 0) return DOT_OK;
    int64_t chunk = kSchedMinChunk;
    while ((nw + chunk - 1) / chunk > kSchedSort) chunk *= 2;
    if (chunk > (1 << 20)) return set_error(DOT_BAD_ARG, "batch too large to schedule");
    const int nc = int((nw + chunk - 1) / chunk);
    retain_pool_memory();
    unsigned* cost = nullptr;
    if (int st = check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&cost), sizeof(unsigned) * nc, s), "cudaMallocAsync"))
        return st;
    sched_cost_kernel<<<unsigned((nc + 255) / 256), 256, 0, s>>>(keys, n, int(chunk), table, cost);
    sched_order_kernel<<<1, 1024, 0, s>>>(cost, n, int(chunk), warp_order);
    cudaFreeAsync(cost, s);
    return check_launch("sched_order_kernel");
}

int launch_sched_update(const int32_t* keys, const uint16_t* ray_used, int64_t n, uint16_t* table, cudaStream_t s) {
    if (n == 0) return DOT_OK;
    const int64_t threads = ((n + 31) / 32) * 32;
    sched_update_kernel<<<unsigned((threads + 255) / 256), 256, 0, s>>>(keys, ray_used, n, table);
    return check_launch("sched_update_kernel");
}

// ---------------------------------------------------------------------------
// Parity helpers and the locate table.

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

}  // namespace dot
