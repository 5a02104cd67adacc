// Shared device helpers for the axb kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "axb.h"

namespace axb {

constexpr int kLutEntries = 65536;
constexpr int kLutBytes = kLutEntries * 2;  // 128 KiB

// ---- programmatic dependent launch: a kernel launched with the PDL attribute may start while
// its predecessor is still running; it must wait before touching the predecessor's outputs.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
// let the next (PDL-launched) kernel be scheduled as soon as this grid's CTAs start retiring
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;\n" ::); }

// ---- ordered-float <-> int (monotone map so atomicMin/Max on int == float min/max)
__host__ __device__ __forceinline__ int32_t f2ord(float f) {
#ifdef __CUDA_ARCH__
    int32_t i = __float_as_int(f);
#else
    int32_t i;
    memcpy(&i, &f, 4);
#endif
    return i >= 0 ? i : (i ^ 0x7FFFFFFF);
}
__host__ __device__ __forceinline__ float ord2f(int32_t i) {
    int32_t b = i >= 0 ? i : (i ^ 0x7FFFFFFF);
#ifdef __CUDA_ARCH__
    return __int_as_float(b);
#else
    float f;
    memcpy(&f, &b, 4);
    return f;
#endif
}

// ---- compute_coeffs (quantizer.py:98-117), identical IEEE fp64 op sequence
__host__ __device__ inline double apply_round(double x, int mode) {
    if (mode == AXB_ROUND_HALF_AWAY) return copysign(floor(fabs(x) + 0.5), x);  // :52-53
    if (mode == AXB_ROUND_HALF_EVEN) return rint(x);                            // :54-55
    return trunc(x);                                                            // :56
}

__host__ __device__ inline int quantize_one(float v, double scale, int zp, int is_signed, int round_mode);
__host__ __device__ inline void fill_bounds(axb_qparams &p, int is_signed, int round_mode, int u0, int ustep);

__host__ __device__ inline axb_qparams coeffs(double mn, double mx, int is_signed, int round_mode) {
    mn = (0.0 < mn) ? 0.0 : mn;  // Python min(rng.min, 0.0): first arg unless 0.0 < it
    mx = (0.0 > mx) ? 0.0 : mx;  // Python max(rng.max, 0.0): first arg unless 0.0 > it
    double scale = (mx - mn) / 255.0;
    if (scale == 0.0) scale = 1.0;
    const double lo = is_signed ? -128.0 : 0.0, hi = is_signed ? 127.0 : 255.0;
    double zp_real = lo - mn / scale;
    double r = apply_round(zp_real, round_mode);
    r = r < lo ? lo : (r > hi ? hi : r);  // np.clip
    axb_qparams p;
    p.scale = scale;
    p.zero_point = (int32_t)r;
    p.valid = 1;
    return p;
}

// ---- quantize_values (quantizer.py:120-131) for one element; returns the code value
__host__ __device__ inline int quantize_one(float v, double scale, int zp, int is_signed, int round_mode) {
    const double x = (double)v / scale;  // IEEE div.rn.f64
    const double nearest = rint(x);
    const double ax = fabs(x);
    const bool snapped = fabs(x - nearest) <= 1.52587890625e-05 * (ax > 1.0 ? ax : 1.0);  // 2^-16
    double r;
    if (snapped)
        r = nearest;
    else if (round_mode == AXB_ROUND_HALF_AWAY)
        r = copysign(floor(ax + 0.5), x);
    else if (round_mode == AXB_ROUND_HALF_EVEN)
        r = nearest;
    else
        r = trunc(x);
    const double lo = is_signed ? -128.0 : 0.0, hi = is_signed ? 127.0 : 255.0;
    double c = r + (double)zp;
    c = c < lo ? lo : (c > hi ? hi : c);
    return (int)c;
}

// ---- exact code boundaries (see axb_qparams.bound)
// smallest finite float x (in the total order of floats) with q(x) >= target;
// -inf if even -FLT_MAX reaches it, +inf if FLT_MAX does not.
__host__ __device__ inline float code_boundary(int target, double scale, int zp, int is_signed, int round_mode) {
    const int64_t LO = f2ord(-3.402823466e38f), HI = f2ord(3.402823466e38f);
    auto q = [&](int64_t o) { return quantize_one(ord2f((int32_t)o), scale, zp, is_signed, round_mode); };
    if (q(LO) >= target) return -INFINITY;
    if (q(HI) < target) return INFINITY;
    // analytic guess ((target - zp) - 0.5) * scale, then an exponential bracket, then bisection
    double g = ((double)(target - zp) - 0.5) * scale;
    g = g < -3.4e38 ? -3.4e38 : (g > 3.4e38 ? 3.4e38 : g);
    int64_t a, b, c0 = f2ord((float)g);
    if (q(c0) >= target) {  // move down until below target
        b = c0;
        int64_t step = 1;
        a = c0 - 1 < LO ? LO : c0 - 1;
        while (a > LO && q(a) >= target) {
            b = a;
            step *= 2;
            a = c0 - step < LO ? LO : c0 - step;
        }
    } else {
        a = c0;
        int64_t step = 1;
        b = c0 + 1 > HI ? HI : c0 + 1;
        while (b < HI && q(b) < target) {
            a = b;
            step *= 2;
            b = c0 + step > HI ? HI : c0 + step;
        }
    }
    while (b - a > 1) {  // invariant q(a) < target <= q(b)
        const int64_t m = a + (b - a) / 2;
        if (q(m) >= target) b = m; else a = m;
    }
    return ord2f((int32_t)b);
}

__host__ __device__ inline void fill_bounds(axb_qparams &p, int is_signed, int round_mode, int u0, int ustep) {
    const int lo = is_signed ? -128 : 0;
    for (int u = u0; u < 256; u += ustep)
        p.bound[u] = u == 0 ? -INFINITY : code_boundary(lo + u, p.scale, p.zero_point, is_signed, round_mode);
}

// ---- division by a runtime-constant divisor via a precomputed magic number
// (round-up method): q = (umulhi(x, m) + x) >> l, exact for all 32-bit x.
struct FastDiv {
    uint32_t d, m, l;
};
inline FastDiv make_fastdiv(uint32_t d) {
    FastDiv f;
    f.d = d ? d : 1;
    uint32_t l = 0;
    while ((uint64_t(1) << l) < f.d) ++l;
    f.l = l;
    f.m = (uint32_t)(((uint64_t(1) << 32) * ((uint64_t(1) << l) - f.d)) / f.d + 1);
    return f;
}
__device__ __forceinline__ uint32_t fdiv(uint32_t x, const FastDiv &f) {
    return (uint32_t)(((uint64_t)__umulhi(x, f.m) + x) >> f.l);
}

// ---- warp reductions
__device__ __forceinline__ int32_t warp_min_i(int32_t v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ int32_t warp_max_i(int32_t v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Block-level range accumulation of a thread's running [min,max] (ordered ints) + nonfinite.
// Block-level min/max/non-finite commit: warp shuffles, then one warp combines
// the per-warp results and ONE lane issues the atomics (one atomicMin/Max pair
// per CTA, not per warp -- same-address atomics serialise in L2).  Must be
// called by every thread of the block (it contains a barrier).
__device__ __forceinline__ void range_commit(int32_t tmin, int32_t tmax, int nonfinite, int32_t *d_range,
                                             int32_t *d_flags, int32_t flag_bit) {
    __shared__ int32_t s_min[32], s_max[32], s_nf[32];
    tmin = warp_min_i(tmin);
    tmax = warp_max_i(tmax);
    const unsigned nf = __ballot_sync(0xffffffffu, nonfinite);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nw = (blockDim.x + 31) >> 5;
    if (lane == 0) {
        s_min[w] = tmin;
        s_max[w] = tmax;
        s_nf[w] = nf != 0;
    }
    __syncthreads();
    if (w == 0) {
        tmin = lane < nw ? s_min[lane] : INT32_MAX;
        tmax = lane < nw ? s_max[lane] : INT32_MIN;
        const unsigned anf = __ballot_sync(0xffffffffu, lane < nw && s_nf[lane]);
        tmin = warp_min_i(tmin);
        tmax = warp_max_i(tmax);
        if (lane == 0) {
            if (d_range) {
                if (tmin != INT32_MAX) atomicMin(d_range, tmin);
                if (tmax != INT32_MIN) atomicMax(d_range + 1, tmax);
            }
            if (anf && d_flags) atomicOr(d_flags, flag_bit);
        }
    }
}

}  // namespace axb
