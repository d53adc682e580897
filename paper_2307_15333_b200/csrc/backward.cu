// backward.cu -- two-kernel fused forward+backward (default path of dot_render_bwd).
//
// The reference (grad_kernel + scatter_kernel, _kernels.py:227-346) saves
// T_i, Q_i, c_i per segment, sweeps each ray backwards and reduces per leaf
// serially.  Here:
//   A) bwd_record_kernel: persistent; every lane walks its ray one segment
//      per iteration (warp-aggregated ray fetch), composites up to the
//      early-termination cut, marks touched leaves (post-cut ones too) and
//      appends one 48-byte record per composited segment -- leaf, ray,
//      delta, T_i, Q_i, the inclusive colour prefix sum_{j<=i} T_j Q_j c_j
//      and c_i -- into warp-owned chunks of a record buffer (one atomic per
//      512 records).  At the ray's end it stores rgb and dL/drgb.
//   B) bwd_scatter_kernel: one thread per record, no traversal, no
//      divergence: suf_i = rgb - prefix_i, then
//        dsigma_i = delta_i * sum_k g_k (T_i (1-Q_i) c_ik - suf_ik)
//        dsh_i[k*B+b] += g_k T_i Q_i c_ik (1-c_ik) * basis_b   (REDG.F32x4)
//        signal_i += Q_i                                        (REDG.F64)
//   C) rays whose records did not fit the buffer are flagged in A and
//      replayed by the one-ray-per-thread kernel (render.cu) -- correctness
//      never depends on the capacity estimate.
#include <atomic>
#include "dot_tree.cuh"
#include "dot_internal.h"

namespace dot {

constexpr int kBlockA = 128;
constexpr int kChunk = 512;
constexpr uint8_t kRayOverflow = 1;

struct __align__(16) SegRec {
    int32_t pid;   // payload row (-1: unused slot)
    int32_t ray;
    float delta, T;
    double Q;      // fp64: the per-leaf signal sums Q exactly like the reference
    float pre0, pre1;
    float pre2, c0, c1, c2;  // colour, NaN when A did not evaluate it (q == 0)
};
static_assert(sizeof(SegRec) == 48, "record must stay 48 bytes");

__device__ __forceinline__ void load_ray_a(const double* __restrict__ o, const double* __restrict__ d,
                                           int64_t r, Tracer& tr) {
    tr.ox = __ldg(o + 3 * r + 0);
    tr.oy = __ldg(o + 3 * r + 1);
    tr.oz = __ldg(o + 3 * r + 2);
    tr.dx = __ldg(d + 3 * r + 0);
    tr.dy = __ldg(d + 3 * r + 1);
    tr.dz = __ldg(d + 3 * r + 2);
}

template <int B>
__global__ void __launch_bounds__(kBlockA) bwd_record_kernel(
    TreeDev T, const double* __restrict__ o, const double* __restrict__ d,
    const double* __restrict__ tgt, int64_t n, double bg0, double bg1, double bg2, double eps,
    double t_near, double t_far, double grad_scale, uint8_t* __restrict__ touched,
    double* __restrict__ loss_sum, float* __restrict__ rgb_out, int flags,
    unsigned long long* __restrict__ ray_ctr, unsigned long long* __restrict__ rec_ctr,
    SegRec* __restrict__ recs, int64_t rec_cap, float* __restrict__ ray_g, float* __restrict__ ray_rgb,
    uint8_t* __restrict__ ray_flag) {
    constexpr int S = pad4(3 * B);
    constexpr unsigned FULL = 0xffffffffu;
    const unsigned lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    Tracer tr;
    float basis[B];
    bool active = false, exhausted = false, cut = false;
    int64_t r = 0;
    double Tacc = 1.0, c0 = 0.0, c1 = 0.0, c2 = 0.0, loss = 0.0;
    uint8_t rflag = 0;
    // warp-owned record chunk [cfill, cend), uniform across the warp
    int64_t cfill = 0, cend = 0;

    auto finish = [&]() {  // rgb, loss, dL/drgb of ray r
        const double R0 = c0 + Tacc * bg0, R1 = c1 + Tacc * bg1, R2 = c2 + Tacc * bg2;
        const double e0 = R0 - __ldg(tgt + 3 * r + 0);
        const double e1 = R1 - __ldg(tgt + 3 * r + 1);
        const double e2 = R2 - __ldg(tgt + 3 * r + 2);
        loss += e0 * e0 + e1 * e1 + e2 * e2;
        if (rgb_out) {
            rgb_out[3 * r + 0] = float(R0);
            rgb_out[3 * r + 1] = float(R1);
            rgb_out[3 * r + 2] = float(R2);
        }
        ray_g[3 * r + 0] = float(grad_scale * e0);
        ray_g[3 * r + 1] = float(grad_scale * e1);
        ray_g[3 * r + 2] = float(grad_scale * e2);
        ray_rgb[3 * r + 0] = float(R0);
        ray_rgb[3 * r + 1] = float(R1);
        ray_rgb[3 * r + 2] = float(R2);
    };

    for (;;) {
        const bool want = !active && !exhausted;
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
                    load_ray_a(o, d, r, tr);
                    eval_basis<B>(tr.dx, tr.dy, tr.dz, basis);
                    Tacc = 1.0;
                    c0 = c1 = c2 = 0.0;
                    cut = false;
                    rflag = 0;
                    if (tr.init(T, t_near, t_far)) {
                        active = true;
                    } else {
                        finish();
                        ray_flag[r] = 0;
                    }
                }
            }
        }
        if (__all_sync(FULL, !active && exhausted)) break;

        Leaf L;
        double te, dl;
        const bool got0 = active ? tr.next(T, L, te, dl) : false;
        bool got = got0;
        const bool rec = got0 && !cut;
        // ---- record slot: warp-aggregated, chunked (allocated before shading
        // so the record's fields are stored as soon as they are computed)
        int64_t slot = -1;
        const unsigned app = __ballot_sync(FULL, rec);
        if (app) {
            const int cnt = __popc(app);
            if (cfill + cnt > cend) {
                for (int64_t s = cfill + lane; s < cend; s += 32) recs[s].pid = -1;
                unsigned long long nb = 0;
                if (lane == 0) nb = atomicAdd(rec_ctr, (unsigned long long)kChunk);
                nb = __shfl_sync(FULL, nb, 0);
                cfill = int64_t(nb);
                cend = cfill + kChunk;
                if (cend > rec_cap) cend = rec_cap > cfill ? rec_cap : cfill;
            }
            if (rec) {
                slot = cfill + __popc(app & lt_mask);
                if (slot >= cend) {
                    slot = -1;
                    rflag |= kRayOverflow;  // buffer full: kernel C replays this ray
                }
            }
            cfill += cnt;
            if (cfill > cend) cfill = cend;
        }
        if (got) {
            if (rec) {
                const double a = exp_ref(-double(__ldg(T.sigma + L.pid)) * dl);
                const double q = 1.0 - a;
                float k0 = __int_as_float(0x7fc00000), k1 = k0, k2 = k0;
                if (q > 0.0) {
                    float e0, e1, e2;
                    sh_dot<B>(T.sh + int64_t(L.pid) * S, basis, e0, e1, e2);
                    k0 = sigmoidf(e0);
                    k1 = sigmoidf(e1);
                    k2 = sigmoidf(e2);
                    const double tq = Tacc * q;
                    c0 += tq * double(k0);
                    c1 += tq * double(k1);
                    c2 += tq * double(k2);
                }
                if (slot >= 0) {
                    float4* dst = reinterpret_cast<float4*>(recs + slot);
                    const int2 qq = make_int2(__double2loint(q), __double2hiint(q));
                    dst[0] = make_float4(__int_as_float(L.pid), __int_as_float(int32_t(r)), float(dl), float(Tacc));
                    dst[1] = make_float4(__int_as_float(qq.x), __int_as_float(qq.y), float(c0), float(c1));
                    dst[2] = make_float4(float(c2), k0, k1, k2);
                }
                touched[L.pid] = 1;
                Tacc *= a;
                if (eps > 0.0 && Tacc < eps) {
                    cut = true;
                    finish();
                    if (flags & 1) got = false;  // skip post-cut touched marking
                }
            } else {
                touched[L.pid] = 1;  // post-cut segments are touched (scatter_kernel)
            }
        }
        if (active && !got) {
            if (!cut) finish();
            ray_flag[r] = rflag;
            active = false;
        }
    }
    for (int64_t s = cfill + lane; s < cend; s += 32) recs[s].pid = -1;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) loss += __shfl_down_sync(FULL, loss, off);
    if (lane == 0 && loss != 0.0) red_add_f64(loss_sum, loss);
}

template <int B>
__global__ void __launch_bounds__(256) bwd_scatter_kernel(
    TreeDev T, const double* __restrict__ d, const SegRec* __restrict__ recs,
    const unsigned long long* __restrict__ rec_ctr, int64_t rec_cap, const float* __restrict__ ray_g,
    const float* __restrict__ ray_rgb, const uint8_t* __restrict__ ray_flag, float* __restrict__ gsig,
    float* __restrict__ gsh, double* __restrict__ signal) {
    constexpr int S = pad4(3 * B);
    int64_t total = int64_t(*rec_ctr);
    if (total > rec_cap) total = rec_cap;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t s = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; s < total; s += stride) {
        const float4* src = reinterpret_cast<const float4*>(recs + s);
        const float4 v0 = __ldg(src), v1 = __ldg(src + 1), v2 = __ldg(src + 2);
        const int32_t pid = __float_as_int(v0.x);
        if (pid < 0) continue;
        const int32_t ray = __float_as_int(v0.y);
        if (__ldg(ray_flag + ray) & kRayOverflow) continue;
        const float delta = v0.z, Ti = v0.w;
        const double Qd = __hiloint2double(__float_as_int(v1.y), __float_as_int(v1.x));
        const float Q = float(Qd);
        float k0 = v2.y, k1 = v2.z, k2 = v2.w;
        float basis[B];
        eval_basis<B>(__ldg(d + 3 * ray), __ldg(d + 3 * ray + 1), __ldg(d + 3 * ray + 2), basis);
        if (k0 != k0) {  // q == 0 in pass A: colour not evaluated yet
            float e0, e1, e2;
            sh_dot<B>(T.sh + int64_t(pid) * S, basis, e0, e1, e2);
            k0 = sigmoidf(e0);
            k1 = sigmoidf(e1);
            k2 = sigmoidf(e2);
        }
        const float g0 = __ldg(ray_g + 3 * ray), g1 = __ldg(ray_g + 3 * ray + 1), g2 = __ldg(ray_g + 3 * ray + 2);
        const float s0 = __ldg(ray_rgb + 3 * ray) - v1.z;
        const float s1 = __ldg(ray_rgb + 3 * ray + 1) - v1.w;
        const float s2 = __ldg(ray_rgb + 3 * ray + 2) - v2.x;
        const float tn = Ti * (1.f - Q);
        const float tq = Ti * Q;
        const float ds = delta * (g0 * (tn * k0 - s0) + g1 * (tn * k1 - s1) + g2 * (tn * k2 - s2));
        red_add_f32(gsig + pid, ds);
        const float w0 = g0 * tq * k0 * (1.f - k0);
        const float w1 = g1 * tq * k1 * (1.f - k1);
        const float w2 = g2 * tq * k2 * (1.f - k2);
        if (w0 != 0.f || w1 != 0.f || w2 != 0.f) {
            float* row = gsh + int64_t(pid) * S;
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
        if (Qd != 0.0) red_add_f64(signal + pid, Qd);
    }
}

// Records-per-ray estimate carried between calls (a capacity hint only): the
// record counter of each call is copied to pinned host memory asynchronously
// and folded in by a later call once its event has completed -- no sync.
static std::atomic<int> g_rec_per_ray{24};
static unsigned long long* g_hint_host = nullptr;
static int64_t g_hint_rays = 0;
static cudaEvent_t g_hint_event = nullptr;
static bool g_hint_pending = false;

static void fold_hint() {
    if (g_hint_pending && cudaEventQuery(g_hint_event) == cudaSuccess) {
        g_hint_pending = false;
        if (g_hint_rays > 0) {
            const int want = int((*g_hint_host * 5 / 4) / uint64_t(g_hint_rays)) + 2;
            g_rec_per_ray.store(want < 4 ? 4 : (want > 4096 ? 4096 : want));
        }
    }
}

template <int B>
static int run_two_kernel(const TreeDev& T, const double* o, const double* d, const double* tgt,
                          int64_t n, const double* bg, double eps, double tn, double tf, double gs,
                          float* gsig, float* gsh, double* signal, uint8_t* touched, double* loss,
                          float* rgb_out, int flags, cudaStream_t s) {
    retain_pool_memory();
    fold_hint();
    const int64_t cap = n * int64_t(g_rec_per_ray.load());
    unsigned long long* ctr = nullptr;
    SegRec* recs = nullptr;
    float* rays = nullptr;
    uint8_t* rflag = nullptr;
    int st = DOT_OK;
    auto cleanup = [&]() {
        cudaFreeAsync(ctr, s);
        cudaFreeAsync(recs, s);
        cudaFreeAsync(rays, s);
        cudaFreeAsync(rflag, s);
    };
#define TRY(x) do { if ((st = (x)) != DOT_OK) { cleanup(); return st; } } while (0)
    TRY(check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&ctr), 2 * sizeof(*ctr), s), "cudaMallocAsync"));
    TRY(check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&recs), cap * sizeof(SegRec), s), "cudaMallocAsync"));
    TRY(check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&rays), n * 6 * sizeof(float), s), "cudaMallocAsync"));
    TRY(check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&rflag), n, s), "cudaMallocAsync"));
    TRY(check_cuda(cudaMemsetAsync(ctr, 0, 2 * sizeof(*ctr), s), "memset"));
    float* ray_g = rays;
    float* ray_rgb = rays + 3 * n;
    {
        int dev = 0, sms = 148, per_sm = 1;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bwd_record_kernel<B>, kBlockA, 0);
        int64_t grid = int64_t(sms) * (per_sm > 0 ? per_sm : 1);
        const int64_t need = (n + kBlockA - 1) / kBlockA;
        if (need < grid) grid = need;
        bwd_record_kernel<B><<<unsigned(grid), kBlockA, 0, s>>>(
            T, o, d, tgt, n, bg[0], bg[1], bg[2], eps, tn, tf, gs, touched, loss, rgb_out, flags, ctr, ctr + 1,
            recs, cap, ray_g, ray_rgb, rflag);
        TRY(check_launch("bwd_record_kernel"));
        int per_sm_b = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_b, bwd_scatter_kernel<B>, 256, 0);
        bwd_scatter_kernel<B><<<unsigned(sms * (per_sm_b > 0 ? per_sm_b : 1)), 256, 0, s>>>(
            T, d, recs, ctr + 1, cap, ray_g, ray_rgb, rflag, gsig, gsh, signal);
        TRY(check_launch("bwd_scatter_kernel"));
        // replay of overflowed rays (no-op pass when none overflowed)
        TRY(launch_render_bwd_replay(T, o, d, n, bg, eps, tn, tf, gsig, gsh, signal, touched, ray_g,
                                     ray_rgb, rflag, flags, s));
    }
    // capacity hint for later calls (1.25x this call's allocation rate)
    if (!g_hint_host) {
        cudaMallocHost(reinterpret_cast<void**>(&g_hint_host), sizeof(unsigned long long));
        cudaEventCreateWithFlags(&g_hint_event, cudaEventDisableTiming);
    }
    if (g_hint_host && !g_hint_pending &&
        cudaMemcpyAsync(g_hint_host, ctr + 1, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s) == cudaSuccess) {
        cudaEventRecord(g_hint_event, s);
        g_hint_rays = n;
        g_hint_pending = true;
    }
    cleanup();
#undef TRY
    return DOT_OK;
}

int launch_render_bwd_two_kernel(const TreeDev& T, const double* o, const double* d, const double* tgt,
                                 int64_t n, const double* bg, double eps, double tn, double tf, double gs,
                                 float* gsig, float* gsh, double* signal, uint8_t* touched, double* loss,
                                 float* rgb_out, int flags, cudaStream_t s) {
    switch (T.basis_count) {
        case 1: return run_two_kernel<1>(T, o, d, tgt, n, bg, eps, tn, tf, gs, gsig, gsh, signal, touched, loss, rgb_out, flags, s);
        case 4: return run_two_kernel<4>(T, o, d, tgt, n, bg, eps, tn, tf, gs, gsig, gsh, signal, touched, loss, rgb_out, flags, s);
        case 9: return run_two_kernel<9>(T, o, d, tgt, n, bg, eps, tn, tf, gs, gsig, gsh, signal, touched, loss, rgb_out, flags, s);
        case 16: return run_two_kernel<16>(T, o, d, tgt, n, bg, eps, tn, tf, gs, gsig, gsh, signal, touched, loss, rgb_out, flags, s);
        default: return set_error(DOT_BAD_ARG, "basis_count must be 1, 4, 9 or 16");
    }
}

}  // namespace dot
