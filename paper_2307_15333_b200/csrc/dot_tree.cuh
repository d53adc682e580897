// dot_tree.cuh -- device-side tree view, exact fp64 traversal, SH shading.
//
// Traversal reproduces /root/reference/pkg/src/octrf/_kernels.py:56-158
// bit-exactly: every geometry operation is an explicit round-to-nearest fp64
// intrinsic (__dadd_rn/__dmul_rn/__ddiv_rn), so nvcc can never contract it
// into an FMA (the Numba kernels contain none) and division is IEEE.
#pragma once
#include <climits>
#include <cmath>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/dot_b200.h"
#include "dot_exp.cuh"

namespace dot {

constexpr double kNudgeRel = 2e-12;  // _kernels.py:16

struct TreeDev {
    const int32_t* __restrict__ node;
    const float* __restrict__ sigma;
    const float* __restrict__ sh;
    int64_t n_nodes;
    int32_t basis_count;
    int32_t sh_stride;
    double cx, cy, cz, half;
    int32_t max_depth;
    // Locate table (dyadic trees only, see descend_grid): node word at depth
    // loc_level for every cell of the 2^L x 2^L x 2^L grid; NULL = disabled.
    const int32_t* __restrict__ loc;
    int32_t loc_level;
    double loc_scale;          // 2^(kLocBits-1) / half  (a power of two)
    double loc_lo[3];          // (center - half) * loc_scale (integers)
};

constexpr int kLocBits = 21;                 // cell coordinates at depth 21
constexpr int32_t kLocLeafFlag = INT32_MIN;  // table entry: leaf shallower than L
constexpr int kLocPidBits = 26;              // entry = flag | depth << 26 | pid

// True when every node centre down to depth kLocBits is an exact multiple of
// half * 2^-kLocBits, so the fp64 comparisons of the descent can be restated
// exactly in integer cell coordinates (descend_grid).
inline bool locate_dyadic(const dot_tree_view& v) {
    int e = 0;
    if (!(v.half_extent > 0.0) || std::frexp(v.half_extent, &e) != 0.5) return false;
    if (v.max_depth > kLocBits || v.max_depth < 0) return false;
    if (v.capacity >= (int64_t(1) << kLocPidBits)) return false;
    const double s = std::ldexp(1.0, kLocBits - 1) / v.half_extent;
    for (int a = 0; a < 3; ++a) {
        const double cs = v.center[a] * s;  // exact (power-of-two scale)
        if (!(std::fabs(cs) < 1125899906842624.0) || std::floor(cs) != cs) return false;
    }
    return true;
}
// (Staging the upper levels in shared memory was measured and rejected: the
// hot top levels already hit L1, and the per-level shared/global select
// slowed the forward by 9 %.)

inline TreeDev make_tree(const dot_tree_view& v) {
    TreeDev t;
    t.node = v.node;
    t.sigma = v.sigma;
    t.sh = v.sh;
    t.n_nodes = v.n_nodes;
    t.basis_count = v.basis_count;
    t.sh_stride = v.sh_stride;
    t.cx = v.center[0];
    t.cy = v.center[1];
    t.cz = v.center[2];
    t.half = v.half_extent;
    t.max_depth = v.max_depth;
    t.loc = nullptr;
    t.loc_level = 0;
    t.loc_scale = 0.0;
    t.loc_lo[0] = t.loc_lo[1] = t.loc_lo[2] = 0.0;
    if (v.locate && v.locate_level > 0 && v.locate_level <= 9 && locate_dyadic(v)) {
        t.loc = v.locate;
        t.loc_level = v.locate_level;
        t.loc_scale = std::ldexp(1.0, kLocBits - 1) / v.half_extent;
        for (int a = 0; a < 3; ++a) t.loc_lo[a] = (v.center[a] - v.half_extent) * t.loc_scale;
    }
    return t;
}

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// Located leaf: payload row, cube centre and half extent.
struct Leaf {
    int32_t pid;
    double cx, cy, cz, h;
};

// _kernels.py:56-68 from the root, with child centres recomputed exactly:
// c_child = c + (h_parent * 0.5) * sign  (octree.py:228-238).
__device__ __forceinline__ Leaf descend_grid(const TreeDev& T, double px, double py, double pz);

__device__ __forceinline__ Leaf descend(const TreeDev& T, double px, double py, double pz) {
    if (T.loc) return descend_grid(T, px, py, pz);
    double cx = T.cx, cy = T.cy, cz = T.cz, h = T.half;
    int32_t w = __ldg(T.node);
    while (w >= 0) {
        const int o = (px >= cx ? 1 : 0) | (py >= cy ? 2 : 0) | (pz >= cz ? 4 : 0);
        h = dmul(h, 0.5);
        cx = (o & 1) ? dadd(cx, h) : dsub(cx, h);
        cy = (o & 2) ? dadd(cy, h) : dsub(cy, h);
        cz = (o & 4) ? dadd(cz, h) : dsub(cz, h);
        w = __ldg(T.node + w + o);
    }
    Leaf L;
    L.pid = ~w;
    L.cx = cx;
    L.cy = cy;
    L.cz = cz;
    L.h = h;
    return L;
}

// Exact integer restatement of descend() for dyadic trees (locate_dyadic).
// With s = 2^20 / h (a power of two) every centre c_j at depth j < 21 has
// c_j * s integer, and scaling by s is exact, so
//     p >= c_j  <=>  floor(p * s) >= c_j * s  <=>  bit (20 - j) of
//     ix = floor(p * s) - (c_root - h) * s  is set
// (given the higher bits select the same cell).  Points that round outside
// the root cube clamp to 0 / 2^21 - 1, i.e. "all comparisons false / true";
// NaN clamps to 0 (every comparison false), exactly like the fp64 chain.
// The first loc_level levels are one load from the locate table; the leaf
// centre c = lo + (2 i_d + 1) h_d is the same exact value the fp64
// recurrence c + (h * 0.5) * sign produces (both are exactly representable).
__device__ __forceinline__ double pow2i(int e) {  // 2^e, |e| < 1000
    return __longlong_as_double(int64_t(1023 + e) << 52);
}

// Integer cell coordinates (depth kLocBits) of a point, and its table entry.
__device__ __forceinline__ void grid_coords(const TreeDev& T, double px, double py, double pz, int& ix, int& iy,
                                            int& iz) {
    const double s = T.loc_scale, top = double((1 << kLocBits) - 1);
    const double fx = fmin(fmax(dsub(floor(dmul(px, s)), T.loc_lo[0]), 0.0), top);
    const double fy = fmin(fmax(dsub(floor(dmul(py, s)), T.loc_lo[1]), 0.0), top);
    const double fz = fmin(fmax(dsub(floor(dmul(pz, s)), T.loc_lo[2]), 0.0), top);
    ix = __double2int_rz(fx);
    iy = __double2int_rz(fy);
    iz = __double2int_rz(fz);
}

__device__ __forceinline__ int32_t grid_entry(const TreeDev& T, int ix, int iy, int iz) {
    const int Lv = T.loc_level, k = kLocBits - Lv;
    return __ldg(T.loc + ((ix >> k) | ((iy >> k) << Lv) | ((iz >> k) << (2 * Lv))));
}

__device__ __forceinline__ Leaf descend_from(const TreeDev& T, int ix, int iy, int iz, int32_t e);

__device__ __forceinline__ Leaf descend_grid(const TreeDev& T, double px, double py, double pz) {
    int ix, iy, iz;
    grid_coords(T, px, py, pz, ix, iy, iz);
    return descend_from(T, ix, iy, iz, grid_entry(T, ix, iy, iz));
}

// The rest of the descent below the table level from the entry e of cell
// (ix, iy, iz), and the leaf centre.
__device__ __forceinline__ Leaf descend_from(const TreeDev& T, int ix, int iy, int iz, int32_t e) {
    const int Lv = T.loc_level;
    int dep, pid;
    if (e >= 0) {
        int32_t w = e;
        dep = Lv;
        do {
            const int b = kLocBits - 1 - dep;
            const int o = ((ix >> b) & 1) | (((iy >> b) & 1) << 1) | (((iz >> b) & 1) << 2);
            w = __ldg(T.node + w + o);
            ++dep;
        } while (w >= 0);
        pid = ~w;
    } else {
        dep = (e >> kLocPidBits) & 31;
        pid = e & ((1 << kLocPidBits) - 1);
    }
    const double hd = dmul(T.half, pow2i(-dep));
    const int sh = kLocBits - dep;
    Leaf L;
    L.pid = pid;
    L.h = hd;
    L.cx = dadd(dsub(T.cx, T.half), dmul(double(2 * (ix >> sh) + 1), hd));
    L.cy = dadd(dsub(T.cy, T.half), dmul(double(2 * (iy >> sh) + 1), hd));
    L.cz = dadd(dsub(T.cz, T.half), dmul(double(2 * (iz >> sh) + 1), hd));
    return L;
}

// One ray walking the tree one exact leaf segment at a time (_trace_ray).
struct Tracer {
    double ox, oy, oz, dx, dy, dz;
    double t, t1, nudge0, nudge;

    // Slab clip against the half-open root cube (_kernels.py:80-106).
    __device__ __forceinline__ bool init(const TreeDev& T, double t_near, double t_far) {
        const double rh = T.half;
        double t0 = t_near;
        t1 = t_far;
        const double o3[3] = {ox, oy, oz};
        const double d3[3] = {dx, dy, dz};
        const double c3[3] = {T.cx, T.cy, T.cz};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const double lo = dsub(c3[a], rh), hi = dadd(c3[a], rh);
            const double o = o3[a], d = d3[a];
            if (d != 0.0) {
                double ta = ddiv(dsub(lo, o), d), tb = ddiv(dsub(hi, o), d);
                if (ta > tb) { const double s = ta; ta = tb; tb = s; }
                if (ta > t0) t0 = ta;
                if (tb < t1) t1 = tb;
            } else if (o < lo || o >= hi) {
                return false;
            }
        }
        if (t1 <= t0) return false;
        nudge0 = dmul(rh, kNudgeRel);
        nudge = nudge0;
        t = t0;
        return true;
    }

    // _kernels.py:112-158.  Returns false when the ray has left the cube.
    // PREFETCH: touch the leaf's sigma and SH row (L1) right after the descent
    // so those gathers overlap the exit-face divisions below.
    template <bool PREFETCH>
    __device__ __forceinline__ bool step(const TreeDev& T, Leaf& L, double& t_entry, double& delta,
                                         bool want_payload) {
        for (;;) {
            const double probe = dadd(t, nudge);
            if (probe >= t1) return false;
            const double px = dadd(ox, dmul(probe, dx));
            const double py = dadd(oy, dmul(probe, dy));
            const double pz = dadd(oz, dmul(probe, dz));
            L = descend(T, px, py, pz);
            if (PREFETCH && want_payload) {
                const char* row = reinterpret_cast<const char*>(T.sh + int64_t(L.pid) * T.sh_stride);
                asm volatile("prefetch.global.L1 [%0];" :: "l"(T.sigma + L.pid));
                asm volatile("prefetch.global.L1 [%0];" :: "l"(row));
                if (T.sh_stride > 32) asm volatile("prefetch.global.L1 [%0];" :: "l"(row + 128));
            }
            // exit t = min over axes of ((c +/- h) - o) / d, in x, y, z order with
            // strict '<' like the reference.  Branch-free: c + (-h) == c - h
            // exactly, and an axis with d == 0 contributes nothing.
            double tex = t1;
            {
                const double cx = ddiv(dsub(dadd(L.cx, dx > 0.0 ? L.h : -L.h), ox), dx);
                const double cy = ddiv(dsub(dadd(L.cy, dy > 0.0 ? L.h : -L.h), oy), dy);
                const double cz = ddiv(dsub(dadd(L.cz, dz > 0.0 ? L.h : -L.h), oz), dz);
                if (dx != 0.0 && cx < tex) tex = cx;
                if (dy != 0.0 && cy < tex) tex = cy;
                if (dz != 0.0 && cz < tex) tex = cz;
            }
            if (tex <= probe) {  // boundary roundoff stalled the walk: widen the probe
                nudge = dmul(nudge, 4.0);
                continue;
            }
            t_entry = t;
            delta = dsub(tex, t);
            t = tex;
            nudge = nudge0;
            return true;
        }
    }

    __device__ __forceinline__ bool next(const TreeDev& T, Leaf& L, double& t_entry, double& delta) {
        return step<false>(T, L, t_entry, delta, false);
    }

    __device__ __forceinline__ bool next_prefetch(const TreeDev& T, Leaf& L, double& t_entry,
                                                  double& delta, bool want_payload = true) {
        return step<true>(T, L, t_entry, delta, want_payload);
    }
};

// Real SH basis, svox/3DGS signs (_kernels.py:30-53), evaluated in fp64 like
// the reference and rounded once to fp32 for the per-segment dot products.
template <int B>
__device__ __forceinline__ void eval_basis(double x, double y, double z, float* out) {
    out[0] = 0.28209479177387814f;
    if constexpr (B >= 4) {
        const double C1 = 0.4886025119029199;
        out[1] = float(-C1 * y);
        out[2] = float(C1 * z);
        out[3] = float(-C1 * x);
    }
    if constexpr (B >= 9) {
        const double xx = x * x, yy = y * y, zz = z * z;
        out[4] = float(1.0925484305920792 * x * y);
        out[5] = float(-1.0925484305920792 * y * z);
        out[6] = float(0.31539156525252005 * (2.0 * zz - xx - yy));
        out[7] = float(-1.0925484305920792 * x * z);
        out[8] = float(0.5462742152960396 * (xx - yy));
        if constexpr (B >= 16) {
            out[9] = float(-0.5900435899266435 * y * (3.0 * xx - yy));
            out[10] = float(2.890611442640554 * x * y * z);
            out[11] = float(-0.4570457994644658 * y * (4.0 * zz - xx - yy));
            out[12] = float(0.3731763325901154 * z * (2.0 * zz - 3.0 * xx - 3.0 * yy));
            out[13] = float(-0.4570457994644658 * x * (4.0 * zz - xx - yy));
            out[14] = float(1.445305721320277 * z * (xx - yy));
            out[15] = float(-0.5900435899266435 * x * (xx - 3.0 * yy));
        }
    }
}

__host__ __device__ constexpr int pad4(int n) { return (n + 3) & ~3; }

// e_k = sum_b sh[k*B+b] * basis[b] for k = 0..2 from one 16-byte aligned row
// (vector loads; the row is read once, never kept whole in registers).
template <int B>
__device__ __forceinline__ void sh_dot(const float* __restrict__ row, const float* basis,
                                       float& e0, float& e1, float& e2) {
    constexpr int S = pad4(3 * B);
    const float4* r4 = reinterpret_cast<const float4*>(row);
    float e[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int j = 0; j < S / 4; ++j) {
        const float4 v = __ldg(r4 + j);
        const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int idx = 4 * j + i;
            if (idx < 3 * B) e[idx / B] = fmaf(vv[i], basis[idx % B], e[idx / B]);
        }
    }
    e0 = e[0];
    e1 = e[1];
    e2 = e[2];
}

// Stable logistic (_kernels.py:22-27) in fp32, branch-free: with
// e = exp(-|x|) <= 1, 1 / (1 + e) for x >= 0 and e / (1 + e) otherwise.
__device__ __forceinline__ float sigmoidf(float x) {
    const float e = __expf(-fabsf(x));
    const float r = __fdividef(1.f, 1.f + e);
    return x >= 0.f ? r : e * r;
}

// Vector reduction into global memory (REDG.E.ADD.F32x4, sm_90+).
__device__ __forceinline__ void red_add_v4(float* addr, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};"
                 :: "l"(addr), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

__device__ __forceinline__ void red_add_f32(float* addr, float a) {
    asm volatile("red.global.add.f32 [%0], %1;" :: "l"(addr), "f"(a) : "memory");
}

__device__ __forceinline__ void red_add_f64(double* addr, double a) {
    asm volatile("red.global.add.f64 [%0], %1;" :: "l"(addr), "d"(a) : "memory");
}

// North-star training-signal extras (no reference counterpart; defined and
// pinned by oracle/dot_oracle.c oracle_weights): per leaf the sum and the
// max over composited segments of the compositing weight T_i Q_i.  The max
// uses the u64 order of non-negative doubles, so it is exact and
// order-independent.
__device__ __forceinline__ void weight_extras(double* wsum, double* wmax, int64_t pid, double tq) {
    if (tq > 0.0) {
        if (wsum) red_add_f64(wsum + pid, tq);
        if (wmax) atomicMax(reinterpret_cast<unsigned long long*>(wmax + pid),
                            static_cast<unsigned long long>(__double_as_longlong(tq)));
    }
}

}  // namespace dot
