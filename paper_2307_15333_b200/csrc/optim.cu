// optim.cu -- sparse RMSProp leaf update (optim.py:107-135).
//
// Only rows with touched[pid] != 0 move; the second-moment state is fp64 like
// the reference's RmsPropState (optim.py:70-72) and every operation is an
// explicit round-to-nearest intrinsic so that, given the same gradients, the
// update is bit-identical to the numpy expression
//   v = beta*v + (1-beta)*g*g;  theta = f32(max(f64(theta) - lr*g/(sqrt(v)+eps), 0)).
// One thread per (row, 4-column quad): float4 payload / gradient accesses and
// 2 x double2 state accesses per thread (vectorised kernel, n_sh % 4 == 0).
#include "dot_tree.cuh"
#include "dot_internal.h"

namespace dot {

constexpr int kMaxPeers = DOT_MAX_PEERS;
// kernel mode bits: consume (zero the gradients), and whether the +0-gradient
// shortcut is exact for these hyper-parameters (lr >= 0, eps > 0)
constexpr int kRmsConsume = 1, kRmsZeroOk = 2;
static int rms_mode(int32_t flags, double eps, double lr_sigma, double lr_sh) {
    return ((flags & 1) ? kRmsConsume : 0) | ((eps > 0.0 && lr_sigma >= 0.0 && lr_sh >= 0.0) ? kRmsZeroOk : 0);
}

// shared-memory carveout preference of the update (-1: driver default).  A
// non-zero carveout keeps shared memory configured on the SMs while the
// update runs, so the plan's cooperative blocks (plan.cu) can be resident
// beside it.
#ifndef DOT_RMS_CARVEOUT
#define DOT_RMS_CARVEOUT -1
#endif

__device__ __forceinline__ float rms_update(float theta, double& v, double g, double beta,
                                            double omb, double eps, double lr, bool clamp, bool zok) {
    v = __dadd_rn(__dmul_rn(beta, v), __dmul_rn(__dmul_rn(omb, g), g));
    // g == 0 (e.g. leaves touched only past the early-termination cut): the
    // step lr*g / (sqrt(v) + eps) is exactly +-0 for eps > 0 and a finite v,
    // and theta -+ 0 == theta unless theta is itself a zero (-0 - -0 = +0),
    // so theta is unchanged -- skip the IEEE sqrt and division (bit-identical
    // result).  Zero payloads, eps <= 0 (0/0 = NaN when v = 0) and an
    // infinite v take the full path; zok (eps > 0, lr >= 0) is decided on the
    // host (kRmsZeroOk).
    if (zok && g == 0.0 && theta != 0.f && v <= 1.7976931348623157e308) {
        double t = double(theta);
        if (clamp && !(t >= 0.0)) t = (t != t) ? t : 0.0;
        return float(t);
    }
#ifdef DOT_RMS_FAKE_MATH  // diagnostic builds only (wrong values): the update without its sqrt / division
    double t = __dsub_rn(double(theta), __dmul_rn(__dmul_rn(lr, g), __dadd_rn(v, eps)));
#else
    double t = __dsub_rn(double(theta), __ddiv_rn(__dmul_rn(lr, g), __dadd_rn(__dsqrt_rn(v), eps)));
#endif
    if (clamp && !(t >= 0.0)) t = (t != t) ? t : 0.0;  // np.maximum keeps NaN
    return float(t);
}

// Generic update (any n_sh, e.g. SH-1's 3 coefficients): one thread per
// (row, quad) of scalar elements.
__global__ void __launch_bounds__(256) rmsprop_kernel(float* __restrict__ sigma, float* __restrict__ sh, int sh_stride,
                                                      int n_sh, double* __restrict__ v_sigma, double* __restrict__ v_sh,
                                                      float* __restrict__ gsig, float* __restrict__ gsh,
                                                      int gsh_stride, const uint8_t* __restrict__ touched, int64_t cap,
                                                      int quads, double beta, double eps, double lr_sigma,
                                                      double lr_sh, int mode) {
    const bool consume = (mode & kRmsConsume) != 0, zok = (mode & kRmsZeroOk) != 0;
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= cap * quads) return;
    const int64_t row = t / quads;
    const int j = int(t - row * quads);
    if (!touched[row]) return;
    const double omb = __dsub_rn(1.0, beta);
    if (j == 0) {
        double v = v_sigma[row];
        sigma[row] = rms_update(sigma[row], v, double(gsig[row]), beta, omb, eps, lr_sigma, true, zok);
        v_sigma[row] = v;
        if (consume) gsig[row] = 0.f;
    }
    const int k0 = 4 * j;
    float* p = sh + row * sh_stride + k0;
    float* g = gsh + row * gsh_stride + k0;
    double* v = v_sh + row * n_sh + k0;
    for (int u = 0; u < 4 && k0 + u < n_sh; ++u) {
        double vv = v[u];
        p[u] = rms_update(p[u], vv, double(g[u]), beta, omb, eps, lr_sh, false, zok);
        v[u] = vv;
        if (consume) g[u] = 0.f;
    }
}

// Vectorised update (n_sh % 4 == 0): one thread per (row, 4-column quad),
// the touched byte first, then the quad's gradient, state and payload loads
// all issued before any is consumed (the payload load is not held back by
// the zero-gradient test).  __launch_bounds__(256, 5) -> 48 registers, 40
// warps per SM: measured against the same update with dependent loads at
// 40 registers (step 2.50 -> 2.46 ms); 2 or 4 quads per thread (74 / 106
// registers) and 6 / 8 blocks (40 / 32 registers, spills) were slower.
// One (row, 4-column quad) of the vectorised update: the quad's gradient,
// state and payload loads all issued before any is consumed (the payload
// load is not held back by the zero-gradient test).
__device__ __forceinline__ void rms_quad(int64_t r, int j, float* __restrict__ sigma, float* __restrict__ sh,
                                         int sh_stride, int n_sh, double* __restrict__ v_sigma,
                                         double* __restrict__ v_sh, float* __restrict__ gsig,
                                         float* __restrict__ gsh, int gsh_stride, double beta, double eps,
                                         double lr_sigma, double lr_sh, bool consume, bool zok) {
    const double omb = __dsub_rn(1.0, beta);
    float* const gp = gsh + r * int64_t(gsh_stride) + 4 * j;
    float* const pp = sh + r * int64_t(sh_stride) + 4 * j;
    double2* const v = reinterpret_cast<double2*>(v_sh + r * int64_t(n_sh) + 4 * j);
    const float4 g = *reinterpret_cast<const float4*>(gp);
    double2 va = v[0], vb = v[1];
    float4 p = *reinterpret_cast<const float4*>(pp);
    if (j == 0) {
        double vs = v_sigma[r];
        sigma[r] = rms_update(sigma[r], vs, double(gsig[r]), beta, omb, eps, lr_sigma, true, zok);
        v_sigma[r] = vs;
        if (consume) gsig[r] = 0.f;
    }
    if (zok && (__float_as_uint(g.x) | __float_as_uint(g.y) | __float_as_uint(g.z) | __float_as_uint(g.w)) == 0u) {
        // +0 gradient quad (e.g. a leaf touched only past the cut): v
        // decays, theta - lr*0/(sqrt(v)+eps) == theta exactly and the
        // gradients are already 0 -- no payload or gradient store (the
        // conditions as in rms_update)
        const double lim = 1.7976931348623157e308;
        const double n0 = __dmul_rn(beta, va.x), n1 = __dmul_rn(beta, va.y);
        const double n2 = __dmul_rn(beta, vb.x), n3 = __dmul_rn(beta, vb.y);
        if (n0 <= lim && n1 <= lim && n2 <= lim && n3 <= lim) {
            v[0] = make_double2(n0, n1);
            v[1] = make_double2(n2, n3);
            return;
        }
    }
    p.x = rms_update(p.x, va.x, double(g.x), beta, omb, eps, lr_sh, false, zok);
    p.y = rms_update(p.y, va.y, double(g.y), beta, omb, eps, lr_sh, false, zok);
    p.z = rms_update(p.z, vb.x, double(g.z), beta, omb, eps, lr_sh, false, zok);
    p.w = rms_update(p.w, vb.y, double(g.w), beta, omb, eps, lr_sh, false, zok);
    *reinterpret_cast<float4*>(pp) = p;
    v[0] = va;
    v[1] = vb;
    if (consume) *reinterpret_cast<float4*>(gp) = make_float4(0.f, 0.f, 0.f, 0.f);
}

// Vectorised update (n_sh % 4 == 0): one thread per (row, 4-column quad),
// the touched byte first.  __launch_bounds__(256, 5) -> 48 registers, 40
// warps per SM: measured against the same update with dependent loads at
// 40 registers (step 2.50 -> 2.46 ms); 2 or 4 quads per thread (74 / 106
// registers) and 6 / 8 blocks (40 / 32 registers, spills) were slower.
__global__ void __launch_bounds__(256, 5) rmsprop_vec_kernel(float* __restrict__ sigma, float* __restrict__ sh,
                                                             int sh_stride, int n_sh, double* __restrict__ v_sigma,
                                                             double* __restrict__ v_sh, float* __restrict__ gsig,
                                                             float* __restrict__ gsh, int gsh_stride,
                                                             const uint8_t* __restrict__ touched, int64_t cap,
                                                             int quads, double beta, double eps, double lr_sigma,
                                                             double lr_sh, int mode) {
    const int64_t f = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (f >= cap * quads) return;
    const int64_t r = f / quads;
    const int j = int(f - r * quads);
    if (!__ldg(touched + r)) return;
    rms_quad(r, j, sigma, sh, sh_stride, n_sh, v_sigma, v_sh, gsig, gsh, gsh_stride, beta, eps, lr_sigma, lr_sh,
             mode & kRmsConsume, mode & kRmsZeroOk);
}

// Sparse steps (a small batch touches few rows): the dense update's cost is
// its capacity-sized grid (140k blocks at configs[1] whatever the batch), so
// the touched rows are listed first (warp-aggregated, any order: rows are
// independent) and a grid-stride kernel updates only them.
__global__ void __launch_bounds__(256) touched_rows_kernel(const uint8_t* __restrict__ touched, int64_t cap,
                                                           int32_t* __restrict__ rows, int32_t* __restrict__ count) {
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool t = r < cap && __ldg(touched + r) != 0;
    const unsigned m = __ballot_sync(0xffffffffu, t);
    if (m == 0u) return;
    const int lane = threadIdx.x & 31;
    int base = 0;
    if (lane == __ffs(m) - 1) base = atomicAdd(count, __popc(m));
    base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
    if (t) rows[base + __popc(m & ((1u << lane) - 1u))] = int32_t(r);
}

__global__ void __launch_bounds__(256, 5) rmsprop_rows_kernel(float* __restrict__ sigma, float* __restrict__ sh,
                                                              int sh_stride, int n_sh, double* __restrict__ v_sigma,
                                                              double* __restrict__ v_sh, float* __restrict__ gsig,
                                                              float* __restrict__ gsh, int gsh_stride,
                                                              const int32_t* __restrict__ rows,
                                                              const int32_t* __restrict__ count, int quads,
                                                              double beta, double eps, double lr_sigma, double lr_sh,
                                                              int mode) {
    const int64_t total = int64_t(*count) * quads;
    for (int64_t f = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; f < total;
         f += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = f / quads;
        rms_quad(__ldg(rows + i), int(f - i * quads), sigma, sh, sh_stride, n_sh, v_sigma, v_sh, gsig, gsh,
                 gsh_stride, beta, eps, lr_sigma, lr_sh, mode & kRmsConsume, mode & kRmsZeroOk);
    }
}

// Opt-in variant with f32 second moments (not the reference's dtype): the
// update arithmetic stays f64 (v widened on read, rounded once on store), so
// results are within float tolerance of the f64-state update while the
// state traffic halves (1568 -> 1184 bytes per touched SH-3 row).
__device__ __forceinline__ float rms_update_f32v(float theta, float& v32, double g, double beta, double omb,
                                                 double eps, double lr, bool clamp, bool zok) {
    double v = double(v32);
    const float out = rms_update(theta, v, g, beta, omb, eps, lr, clamp, zok);
    v32 = float(v);
    return out;
}

__global__ void __launch_bounds__(256, 5) rmsprop_f32v_kernel(float* __restrict__ sigma, float* __restrict__ sh,
                                                              int sh_stride, int n_sh, float* __restrict__ v_sigma,
                                                              float* __restrict__ v_sh, float* __restrict__ gsig,
                                                              float* __restrict__ gsh, int gsh_stride,
                                                              const uint8_t* __restrict__ touched, int64_t cap,
                                                              int quads, double beta, double eps, double lr_sigma,
                                                              double lr_sh, int mode) {
    const bool consume = (mode & kRmsConsume) != 0, zok = (mode & kRmsZeroOk) != 0;
    const int64_t f = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (f >= cap * quads) return;
    const int64_t r = f / quads;
    const int j = int(f - r * quads);
    if (!__ldg(touched + r)) return;
    const double omb = __dsub_rn(1.0, beta);
    if (j == 0) {
        sigma[r] = rms_update_f32v(sigma[r], v_sigma[r], double(gsig[r]), beta, omb, eps, lr_sigma, true, zok);
        if (consume) gsig[r] = 0.f;
    }
    const int k0 = 4 * j;
    if ((n_sh & 3) == 0 && (sh_stride & 3) == 0 && (gsh_stride & 3) == 0) {
        float* const gp = gsh + r * int64_t(gsh_stride) + k0;
        float* const pp = sh + r * int64_t(sh_stride) + k0;
        float4* const vp = reinterpret_cast<float4*>(v_sh + r * int64_t(n_sh) + k0);
        const float4 g = *reinterpret_cast<const float4*>(gp);
        float4 v = *vp;
        float4 p = *reinterpret_cast<const float4*>(pp);
        p.x = rms_update_f32v(p.x, v.x, double(g.x), beta, omb, eps, lr_sh, false, zok);
        p.y = rms_update_f32v(p.y, v.y, double(g.y), beta, omb, eps, lr_sh, false, zok);
        p.z = rms_update_f32v(p.z, v.z, double(g.z), beta, omb, eps, lr_sh, false, zok);
        p.w = rms_update_f32v(p.w, v.w, double(g.w), beta, omb, eps, lr_sh, false, zok);
        *vp = v;
        if (g.x != 0.f || g.y != 0.f || g.z != 0.f || g.w != 0.f) {
            *reinterpret_cast<float4*>(pp) = p;
            if (consume) *reinterpret_cast<float4*>(gp) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        return;
    }
    for (int u = 0; u < 4 && k0 + u < n_sh; ++u) {
        float* p = sh + r * sh_stride + k0 + u;
        float* g = gsh + r * gsh_stride + k0 + u;
        *p = rms_update_f32v(*p, v_sh[r * n_sh + k0 + u], double(*g), beta, omb, eps, lr_sh, false, zok);
        if (consume) *g = 0.f;
    }
}

// ---------------------------------------------------------------------------
// Multi-GPU update fused with its collective (one node, NVLink/NVSwitch peer
// memory).  Every rank holds a replica of the payload and its own partial
// gradients; rank k owns rows [lo_k, hi_k).  After all ranks' backward
// kernels have finished, each rank runs this kernel over its own rows: it
// reads the W partial gradient rows (local + W-1 peer loads) and sums them in
// rank order (f64), applies RMSProp with its local second moments, writes the
// updated row into EVERY rank's payload (peer stores: the all-gather), and
// zeroes the W consumed gradient rows (consume).  Reduce-scatter + update +
// all-gather in one pass, only over rows some rank touched; no NCCL call.

struct PeerRows {
    float* sigma[kMaxPeers];
    float* sh[kMaxPeers];
    float* gsig[kMaxPeers];
    float* gsh[kMaxPeers];
    const uint8_t* touched[kMaxPeers];
    int world, rank;
};

__global__ void __launch_bounds__(256) rmsprop_peer_kernel(PeerRows P, int sh_stride, int n_sh, int gsh_stride,
                                                           double* __restrict__ v_sigma,
                                                           double* __restrict__ v_sh, int64_t lo, int64_t hi,
                                                           int quads, double beta, double eps, double lr_sigma,
                                                           double lr_sh, int mode) {
    const bool consume = (mode & kRmsConsume) != 0, zok = (mode & kRmsZeroOk) != 0;
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= (hi - lo) * quads) return;
    const int64_t row = lo + t / quads;
    const int j = int(t - (row - lo) * quads);
    bool touched = false;
    for (int r = 0; r < P.world; ++r) touched |= P.touched[r][row] != 0;
    if (!touched) return;
    const double omb = __dsub_rn(1.0, beta);
    if (j == 0) {
        double g = 0.0;
        for (int r = 0; r < P.world; ++r) g += double(P.gsig[r][row]);
        double v = v_sigma[row];
        const float th = rms_update(P.sigma[P.rank][row], v, g, beta, omb, eps, lr_sigma, true, zok);
        v_sigma[row] = v;
        for (int r = 0; r < P.world; ++r) {
            P.sigma[r][row] = th;
            if (consume) P.gsig[r][row] = 0.f;
        }
    }
    const int k0 = 4 * j;
    double g[4] = {0.0, 0.0, 0.0, 0.0};
    for (int r = 0; r < P.world; ++r) {
        const float* gp = P.gsh[r] + row * gsh_stride + k0;
        for (int u = 0; u < 4 && k0 + u < n_sh; ++u) g[u] += double(gp[u]);
    }
    const float* th0 = P.sh[P.rank] + row * sh_stride + k0;
    float th[4];
    double* v = v_sh + row * n_sh + k0;
    for (int u = 0; u < 4 && k0 + u < n_sh; ++u) {
        double vv = v[u];
        th[u] = rms_update(th0[u], vv, g[u], beta, omb, eps, lr_sh, false, zok);
        v[u] = vv;
    }
    for (int r = 0; r < P.world; ++r) {
        float* p = P.sh[r] + row * sh_stride + k0;
        float* gp = P.gsh[r] + row * gsh_stride + k0;
        for (int u = 0; u < 4 && k0 + u < n_sh; ++u) {
            p[u] = th[u];
            if (consume) gp[u] = 0.f;
        }
    }
}

}  // namespace dot

using namespace dot;

extern "C" int dot_rmsprop_step_peers(const dot_peer_rows* peers, int32_t sh_stride, int32_t n_sh,
                                      int32_t gsh_stride, double* v_sigma, double* v_sh, int64_t row_lo,
                                      int64_t row_hi, double beta, double eps, double lr_sigma, double lr_sh,
                                      int32_t flags, void* stream) {
    if (!peers || !v_sigma || !v_sh) return set_error(DOT_BAD_ARG, "rmsprop_peers: NULL argument");
    if (peers->world < 1 || peers->world > kMaxPeers || peers->rank < 0 || peers->rank >= peers->world)
        return set_error(DOT_BAD_ARG, "rmsprop_peers: world must be 1..%d and rank < world", kMaxPeers);
    if (!(beta > 0.0 && beta < 1.0)) return set_error(DOT_BAD_ARG, "beta must be in (0, 1), got %g", beta);
    if (n_sh < 1 || sh_stride < n_sh || gsh_stride < n_sh) return set_error(DOT_BAD_ARG, "rmsprop_peers: bad strides");
    PeerRows P;
    P.world = peers->world;
    P.rank = peers->rank;
    for (int r = 0; r < kMaxPeers; ++r) {
        const bool in = r < P.world;
        if (in && (!peers->sigma[r] || !peers->sh[r] || !peers->grad_sigma[r] || !peers->grad_sh[r] ||
                   !peers->touched[r]))
            return set_error(DOT_BAD_ARG, "rmsprop_peers: NULL pointer for rank %d", r);
        P.sigma[r] = in ? peers->sigma[r] : nullptr;
        P.sh[r] = in ? peers->sh[r] : nullptr;
        P.gsig[r] = in ? peers->grad_sigma[r] : nullptr;
        P.gsh[r] = in ? peers->grad_sh[r] : nullptr;
        P.touched[r] = in ? peers->touched[r] : nullptr;
    }
    if (row_hi <= row_lo) return DOT_OK;
    const int quads = (n_sh + 3) / 4;
    const int64_t total = (row_hi - row_lo) * quads;
    rmsprop_peer_kernel<<<unsigned((total + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        P, sh_stride, n_sh, gsh_stride, v_sigma, v_sh, row_lo, row_hi, quads, beta, eps, lr_sigma, lr_sh,
        rms_mode(flags, eps, lr_sigma, lr_sh));
    return check_launch("rmsprop_peer_kernel");
}

extern "C" int dot_rmsprop_step(float* sigma, float* sh, int32_t sh_stride, int32_t n_sh, double* v_sigma,
                                double* v_sh, float* grad_sigma, float* grad_sh,
                                int32_t gsh_stride, const uint8_t* touched, int64_t capacity, double beta,
                                double eps, double lr_sigma, double lr_sh, int32_t flags, void* stream) {
    if (!sigma || !sh || !v_sigma || !v_sh || !grad_sigma || !grad_sh || !touched)
        return set_error(DOT_BAD_ARG, "rmsprop: NULL argument");
    if (!(beta > 0.0 && beta < 1.0)) return set_error(DOT_BAD_ARG, "beta must be in (0, 1), got %g", beta);
    if (n_sh < 1 || sh_stride < n_sh || gsh_stride < n_sh) return set_error(DOT_BAD_ARG, "rmsprop: bad strides");
    if (capacity == 0) return DOT_OK;
    const int quads = (n_sh + 3) / 4;
    const bool vec = (n_sh % 4 == 0) && (sh_stride % 4 == 0) && (gsh_stride % 4 == 0) &&
                     ((reinterpret_cast<uintptr_t>(sh) | reinterpret_cast<uintptr_t>(grad_sh)) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(v_sh) & 31) == 0;
    const int64_t total = capacity * quads;
    const unsigned grid = unsigned((total + 255) / 256);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (vec) {
#if DOT_RMS_CARVEOUT >= 0
        cudaFuncSetAttribute(rmsprop_vec_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, DOT_RMS_CARVEOUT);
#endif
        rmsprop_vec_kernel<<<grid, 256, 0, s>>>(sigma, sh, sh_stride, n_sh, v_sigma, v_sh, grad_sigma, grad_sh,
                                                gsh_stride, touched, capacity, quads, beta, eps, lr_sigma, lr_sh,
                                                rms_mode(flags, eps, lr_sigma, lr_sh));
        return check_launch("rmsprop_vec_kernel");
    }
    rmsprop_kernel<<<grid, 256, 0, s>>>(sigma, sh, sh_stride, n_sh, v_sigma, v_sh, grad_sigma, grad_sh,
                                        gsh_stride, touched, capacity, quads, beta, eps, lr_sigma, lr_sh,
                                        rms_mode(flags, eps, lr_sigma, lr_sh));
    return check_launch("rmsprop_kernel");
}

extern "C" int dot_rmsprop_step_sparse(float* sigma, float* sh, int32_t sh_stride, int32_t n_sh, double* v_sigma,
                                       double* v_sh, float* grad_sigma, float* grad_sh, int32_t gsh_stride,
                                       const uint8_t* touched, int64_t capacity, double beta, double eps,
                                       double lr_sigma, double lr_sh, int32_t flags, void* stream) {
    if (!sigma || !sh || !v_sigma || !v_sh || !grad_sigma || !grad_sh || !touched)
        return set_error(DOT_BAD_ARG, "rmsprop: NULL argument");
    if (!(beta > 0.0 && beta < 1.0)) return set_error(DOT_BAD_ARG, "beta must be in (0, 1), got %g", beta);
    if (n_sh < 1 || sh_stride < n_sh || gsh_stride < n_sh) return set_error(DOT_BAD_ARG, "rmsprop: bad strides");
    if (capacity > INT32_MAX) return set_error(DOT_BAD_ARG, "rmsprop_sparse: capacity must be < 2^31");
    const bool vec = (n_sh % 4 == 0) && (sh_stride % 4 == 0) && (gsh_stride % 4 == 0) &&
                     ((reinterpret_cast<uintptr_t>(sh) | reinterpret_cast<uintptr_t>(grad_sh)) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(v_sh) & 31) == 0;
    if (!vec)  // the generic layout keeps the dense update
        return dot_rmsprop_step(sigma, sh, sh_stride, n_sh, v_sigma, v_sh, grad_sigma, grad_sh, gsh_stride, touched,
                                capacity, beta, eps, lr_sigma, lr_sh, flags, stream);
    if (capacity == 0) return DOT_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    retain_pool_memory();
    int32_t* rows = nullptr;
    if (int st = check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&rows), size_t(capacity + 1) * 4, s),
                            "cudaMallocAsync"))
        return st;
    int32_t* count = rows + capacity;
    int st = check_cuda(cudaMemsetAsync(count, 0, 4, s), "cudaMemsetAsync");
    if (st == DOT_OK) {
        touched_rows_kernel<<<unsigned((capacity + 255) / 256), 256, 0, s>>>(touched, capacity, rows, count);
        int dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        rmsprop_rows_kernel<<<unsigned(5 * (sms > 0 ? sms : 148)), 256, 0, s>>>(
            sigma, sh, sh_stride, n_sh, v_sigma, v_sh, grad_sigma, grad_sh, gsh_stride, rows, count, (n_sh + 3) / 4,
            beta, eps, lr_sigma, lr_sh, rms_mode(flags, eps, lr_sigma, lr_sh));
        st = check_launch("rmsprop_rows_kernel");
    }
    cudaFreeAsync(rows, s);
    return st;
}

extern "C" int dot_rmsprop_step_f32state(float* sigma, float* sh, int32_t sh_stride, int32_t n_sh, float* v_sigma,
                                         float* v_sh, float* grad_sigma, float* grad_sh, int32_t gsh_stride,
                                         const uint8_t* touched, int64_t capacity, double beta, double eps,
                                         double lr_sigma, double lr_sh, int32_t flags, void* stream) {
    if (!sigma || !sh || !v_sigma || !v_sh || !grad_sigma || !grad_sh || !touched)
        return set_error(DOT_BAD_ARG, "rmsprop: NULL argument");
    if (!(beta > 0.0 && beta < 1.0)) return set_error(DOT_BAD_ARG, "beta must be in (0, 1), got %g", beta);
    if (n_sh < 1 || sh_stride < n_sh || gsh_stride < n_sh) return set_error(DOT_BAD_ARG, "rmsprop: bad strides");
    if (((reinterpret_cast<uintptr_t>(sh) | reinterpret_cast<uintptr_t>(grad_sh) |
          reinterpret_cast<uintptr_t>(v_sh)) & 15) != 0)
        return set_error(DOT_BAD_ARG, "rmsprop: sh / grad_sh / v_sh must be 16-byte aligned");
    if (capacity == 0) return DOT_OK;
    const int quads = (n_sh + 3) / 4;
    const int64_t total = capacity * quads;
    rmsprop_f32v_kernel<<<unsigned((total + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        sigma, sh, sh_stride, n_sh, v_sigma, v_sh, grad_sigma, grad_sh, gsh_stride, touched, capacity, quads, beta,
        eps, lr_sigma, lr_sh, rms_mode(flags, eps, lr_sigma, lr_sh));
    return check_launch("rmsprop_f32v_kernel");
}
