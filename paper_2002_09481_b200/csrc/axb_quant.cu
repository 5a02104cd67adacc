// K1 (range reduction), coefficients, K2 (quantize + zero-point padding) and
// filter preparation.  All HBM-bound; bit-exact restatements of
//   tensor.py:143-149 / graph.py:270-275 (min/max, non-finite -> ValueError)
//   quantizer.py:98-117 (compute_coeffs), :120-131 (quantize_values)
//   axconv.py:181-196 (zp padding, patch sums), :199-210 (quantize_filters)
#include "axb_common.cuh"
#include "axb_internal.h"

namespace axb {

// ---------------------------------------------------------------- K1: range
// Grid-stride over float4 (16-byte coalesced loads), per-thread min/max in
// ordered-int space, warp shuffle reduce, one atomic per warp.
__global__ void __launch_bounds__(256) range_kernel(const float *__restrict__ x, int64_t n, int32_t *d_range,
                                                    int32_t *d_flags) {
    int32_t tmin = INT32_MAX, tmax = INT32_MIN;
    int nonfinite = 0;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const bool aligned = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
    int64_t head = 0;
    if (aligned) {
        const int64_t n4 = n >> 2;
        const float4 *x4 = reinterpret_cast<const float4 *>(x);
        // 4 independent 16-byte loads in flight per thread per iteration
        float fmn = INFINITY, fmx = -INFINITY;
        int64_t i = tid;
        for (; i + 3 * stride < n4; i += 4 * stride) {
            float4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = __ldg(x4 + i + u * stride);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const float e[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    nonfinite |= !(fabsf(e[q]) <= 3.402823466e38f);
                    fmn = fminf(fmn, e[q]);
                    fmx = fmaxf(fmx, e[q]);
                }
            }
        }
        for (; i < n4; i += stride) {
            const float4 v = __ldg(x4 + i);
            const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                nonfinite |= !(fabsf(e[q]) <= 3.402823466e38f);
                fmn = fminf(fmn, e[q]);
                fmx = fmaxf(fmx, e[q]);
            }
        }
        // fminf/fmaxf ignore NaN (flagged above); -0/+0 order is irrelevant to compute_coeffs
        if (fmn <= fmx) {
            tmin = min(tmin, f2ord(fmn));
            tmax = max(tmax, f2ord(fmx));
        }
        head = n4 << 2;
    }
    for (int64_t i = head + tid; i < n; i += stride) {
        const float v = x[i];
        nonfinite |= !isfinite(v);
        const int32_t o = f2ord(v);
        tmin = min(tmin, o);
        tmax = max(tmax, o);
    }
    range_commit(tmin, tmax, nonfinite, d_range, d_flags, AXB_FLAG_NONFINITE);
}

__global__ void range_reset_kernel(int32_t *d_range) {
    d_range[0] = INT32_MAX;
    d_range[1] = INT32_MIN;
}

// coefficients of a device range + the exact code-boundary table: 256 threads,
// thread u bisects boundary u against the fp64 quantizer (no host sync)
__global__ void __launch_bounds__(256) coeffs_kernel(const int32_t *d_range, int is_signed, int round_mode,
                                                     axb_qparams *out) {
    const float mn = ord2f(d_range[0]);
    const float mx = ord2f(d_range[1]);
    axb_qparams p = coeffs((double)mn, (double)mx, is_signed, round_mode);
    const int u = threadIdx.x;
    const int lo = is_signed ? -128 : 0;
    out->bound[u] = u == 0 ? -INFINITY : code_boundary(lo + u, p.scale, p.zero_point, is_signed, round_mode);
    if (u == 0) {
        out->scale = p.scale;
        out->zero_point = p.zero_point;
        out->valid = 1;
    }
}

__global__ void params_set_kernel(axb_qparams p, axb_qparams *out) {
    for (int u = threadIdx.x; u < 256; u += blockDim.x) out->bound[u] = p.bound[u];
    if (threadIdx.x == 0) {
        out->scale = p.scale;
        out->zero_point = p.zero_point;
        out->valid = p.valid;
    }
}

// ---------------------------------------------------------------- K2: quantize + pad
// Exact quantization without per-element fp64: an fp32 estimate of the code
// offset, corrected against the exact boundary table (qparams.bound, staged in
// shared memory) -- usually 2 compares.  One thread per 4-channel group
// (float4 in, u32 out, fully coalesced); the per-pixel code sum is a segmented
// warp reduction over the G = cs/4 groups of a pixel (G a power of two <= 32),
// or a warp per pixel (G == 0: cs > 128 or not a power of two).
struct QuantCtx {
    float bnd[257];
    double scale;
    float inv, zpo;
    int lo, zp;
    int table;  // bnd[] valid (axb_quantize_pad); else exact fp64 quantize_one for ties (axb_quantize_pad_range)
    int sgn, round;
};

__device__ __forceinline__ void quant_ctx_load(QuantCtx &q, const axb_qparams *prm, int is_signed) {
    for (int u = threadIdx.x; u < 256; u += blockDim.x) q.bnd[u] = prm->bound[u];
    if (threadIdx.x == 0) {
        q.bnd[256] = INFINITY;
        q.lo = is_signed ? -128 : 0;
        q.zp = prm->zero_point;
        q.inv = (float)(1.0 / prm->scale);
        q.zpo = (float)(prm->zero_point - q.lo);
        q.table = 1;
    }
    __syncthreads();
}

// Context computed in-kernel from a device range (compute_coeffs, quantizer.py:98-117):
// scale and zero point only -- no boundary table; the rare elements the fp32 estimate
// cannot decide go through the exact fp64 quantize_one.  Block 0 publishes scale and
// zero point for the conv epilogue (this replaces a coeffs_kernel launch).
__device__ __forceinline__ void quant_ctx_from_range(QuantCtx &q, const int32_t *d_range, int is_signed,
                                                     int round_mode, axb_qparams *p_out) {
    if (threadIdx.x == 0) {
        const float mn = ord2f(d_range[0]);
        const float mx = ord2f(d_range[1]);
        const axb_qparams p = coeffs((double)mn, (double)mx, is_signed, round_mode);
        q.lo = is_signed ? -128 : 0;
        q.zp = p.zero_point;
        q.scale = p.scale;
        q.inv = (float)(1.0 / p.scale);
        q.zpo = (float)(p.zero_point - q.lo);
        q.table = 0;
        q.sgn = is_signed;
        q.round = round_mode;
        if (blockIdx.x == 0) {
            p_out->scale = p.scale;
            p_out->zero_point = p.zero_point;
            p_out->valid = 2;  // parameters only (bound[] not filled)
        }
    }
    __syncthreads();
}

// code value of a finite float: lo + max{u : bnd[u] <= x}
__device__ __forceinline__ int quant_exact(const QuantCtx &q, float x) {
    float uf = fmaf(x, q.inv, q.zpo);
    int u = (uf > 0.0f) ? (uf < 255.0f ? __float2int_rn(uf) : 255) : 0;  // NaN / -inf -> 0
    while (x < q.bnd[u]) --u;        // bnd[0] = -inf stops it
    while (x >= q.bnd[u + 1]) ++u;   // bnd[256] = +inf stops it
    return q.lo + u;
}

// Offset u = code - lo for the two round-to-nearest modes without touching the
// table in the common case.  uf = fl(x*fl(1/scale) + (zp - lo)) is within
// 2^-24*(|v| + |uf|) < 5e-5 of v + zp - lo (v = x/scale in fp64) wherever the
// result is not clipped (|v| <= 511, |uf| <= 256), so when uf is more than
// 2.5e-4 away from a half-integer, rint(uf) is the reference's rounding of v
// (half-away and half-even agree off ties; the 2^-16 snap only moves values
// onto the integer they round to anyway), and the clip to [0, 255] matches
// quantizer.py:130.  Near a tie, NaN or +-inf: the exact boundary table.
__device__ __forceinline__ int quant_near_u(const QuantCtx &q, float x) {
    const float uf = fmaf(x, q.inv, q.zpo);
    const float r = rintf(uf);
    if (fabsf(uf - r) < 0.49975f) return min(max((int)r, 0), 255);
    if (!q.table) return quantize_one(x, q.scale, q.zp, q.sgn, q.round) - q.lo;  // exact fp64 (NaN -> flagged)
    return quant_exact(q, x) - q.lo;
}
__device__ __forceinline__ int quant_any_u(const QuantCtx &q, float x, bool nearest) {
    if (nearest) return quant_near_u(q, x);
    if (!q.table) return quantize_one(x, q.scale, q.zp, q.sgn, q.round) - q.lo;
    return quant_exact(q, x) - q.lo;
}

template <int G>
__global__ void __launch_bounds__(256) quantize_pad_kernel(const float *__restrict__ x, int64_t n, int64_t h, int64_t w,
                                                           int c, int64_t cs, int pt, int pl, int64_t hp, int64_t wp,
                                                           FastDiv fd_hp, FastDiv fd_wp,
                                                           axb_qparams *prm, const int32_t *d_range, int is_signed,
                                                           int round_mode, uint8_t *__restrict__ codes,
                                                           int32_t *__restrict__ pixsum, int32_t *d_flags) {
    __shared__ QuantCtx q;
    if (d_range)
        quant_ctx_from_range(q, d_range, is_signed, round_mode, prm);
    else
        quant_ctx_load(q, prm, is_signed);
    const bool nearest = round_mode != AXB_ROUND_TOWARD_ZERO;
    const int lane = threadIdx.x & 31;
    const int64_t npix = n * hp * wp;
    const bool vec = (c % 4 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
    const int zpb = q.zp & 0xFF;
    const uint32_t zpw = (uint32_t)zpb * 0x01010101u;
    int nonfinite = 0;
    // one 4-channel group g of padded pixel p -> 4 code bytes; s += their code values
    auto group = [&](uint32_t p, int g, int32_t &s) -> uint32_t {
        const uint32_t t = fdiv(p, fd_wp);  // npix < 2^31 (checked on the host)
        const int xw = (int)(p - t * (uint32_t)wp);
        const uint32_t b = fdiv(t, fd_hp);
        const int yh = (int)(t - b * (uint32_t)hp);
        const int iy = yh - pt, ix = xw - pl;
        const int c0 = g * 4;
        if (iy < 0 || iy >= h || ix < 0 || ix >= w) {  // zero-point border (axconv.py:185-189)
            if (c0 + 3 < c) {
                s += 4 * q.zp;
                return zpw;
            }
            uint32_t word = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (c0 + k < c) {
                    s += q.zp;
                    word |= (uint32_t)zpb << (8 * k);
                }
            return word;
        }
        const float *src = x + (((int64_t)b * h + iy) * w + ix) * c + c0;
        float e[4];
        if (vec && c0 + 3 < c) {
            const float4 v = __ldg(reinterpret_cast<const float4 *>(src));
            e[0] = v.x; e[1] = v.y; e[2] = v.z; e[3] = v.w;
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) e[k] = (c0 + k < c) ? __ldg(src + k) : 0.0f;
        }
        uint32_t word = 0;
        int su = 0, nv = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (c0 + k < c) {
                nonfinite |= !(fabsf(e[k]) <= 3.402823466e38f);
                const int u = quant_any_u(q, e[k], nearest);
                su += u;
                ++nv;
                word |= (uint32_t)((u + q.lo) & 0xFF) << (8 * k);
            }
        }
        s += su + nv * q.lo;
        return word;
    };
    if constexpr (G > 0) {
        // thread per 4-channel group (float4 in, u32 out, coalesced); segmented warp sum per pixel
        const uint32_t total = (uint32_t)(npix * G);
        const uint32_t stride = gridDim.x * blockDim.x;
        const uint32_t bound = (total + 31u) & ~31u;
        for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < bound; i += stride) {
            int32_t s = 0;
            if (i < total) {
                const uint32_t word = group(i / G, (int)(i % G), s);
                reinterpret_cast<uint32_t *>(codes)[i] = word;  // cs == 4G: group i is word i
            }
#pragma unroll
            for (int o = G / 2; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (i < total && (i % G) == 0 && pixsum) pixsum[i / G] = s;
        }
    } else {
        const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
        const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
        for (int64_t p = warp0; p < npix; p += nwarps) {
            int32_t s = 0;
            for (int64_t g = lane; g < cs / 4; g += 32)
                reinterpret_cast<uint32_t *>(codes + p * cs)[g] = group((uint32_t)p, (int)g, s);
#pragma unroll
            for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (lane == 0 && pixsum) pixsum[p] = s;
        }
    }
    range_commit(INT32_MAX, INT32_MIN, nonfinite, nullptr, d_flags, AXB_FLAG_NONFINITE);
}

// Fast K2 for c % 16 == 0 (no channel padding): one thread per 16-channel chunk
// (4 x float4 in, one 16-byte code store), C16 = c/16 chunks per pixel.  Per
// element: FFMA + FRND + tie test + clamp; codes are packed as offsets u and the
// pixel sum is dp4a(u bytes) + 16*lo per chunk (exact).  Any element the fp32
// estimate cannot decide (near a half-step, NaN/inf) or a toward-zero table
// sends its whole chunk through the exact path (rare, warp-divergent).
// round-to-nearest-even of four floats, each clipped to [0, 255] (NaN -> 0), packed little-endian:
// cvt.pack.sat places sat(a) in bits 15:8, sat(b) in bits 7:0 and c's low half above them (the
// compiler fuses the float->int rounding into one F2IP.U8 per pair)
__device__ __forceinline__ uint32_t pack_u8x4(float f0, float f1, float f2, float f3) {
    uint32_t hi, w;
    asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, 0;" : "=r"(hi) : "r"(__float2int_rn(f3)), "r"(__float2int_rn(f2)));
    asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(w) : "r"(__float2int_rn(f1)), "r"(__float2int_rn(f0)), "r"(hi));
    return w;
}

template <int C16>
__global__ void __launch_bounds__(256) quantize_pad16_kernel(const float *__restrict__ x, int n, int h, int w,
                                                             int pt, int pl, int hp, int wp, FastDiv fd_hp,
                                                             FastDiv fd_wp, axb_qparams *prm,
                                                             const int32_t *d_range, int is_signed, int round_mode,
                                                             uint8_t *__restrict__ codes,
                                                             int32_t *__restrict__ pixsum, int32_t *d_flags) {
    __shared__ QuantCtx q;
    const int c = 16 * C16;
    pdl_launch_dependents();  // the next conv may start its prologue (table TMA) as CTAs retire
    const uint32_t npix = (uint32_t)n * (uint32_t)hp * (uint32_t)wp;
    constexpr int PER = C16 <= 32 ? C16 : 32;  // lanes per pixel in the segmented sum
    const uint32_t total = npix * (uint32_t)C16;
    const uint32_t stride = gridDim.x * blockDim.x;
    const uint32_t bound = (total + 31u) & ~31u;
    // chunk i -> (pixel p, 16-channel group j); its 16 inputs (false: zero-point border, axconv.py:185-189)
    auto fetch = [&](uint32_t i, float (&e)[16]) -> bool {
        const uint32_t p = i / C16, j = i % C16;
        const uint32_t t = fdiv(p, fd_wp);
        const int xw = (int)(p - t * (uint32_t)wp);
        const uint32_t b = fdiv(t, fd_hp);
        const int yh = (int)(t - b * (uint32_t)hp);
        const int iy = yh - pt, ix = xw - pl;
        if (iy < 0 || iy >= h || ix < 0 || ix >= w) return false;
        const float4 *src = reinterpret_cast<const float4 *>(x + (((int64_t)b * h + iy) * w + ix) * c + j * 16);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const float4 f = __ldg(src + v);
            e[4 * v] = f.x; e[4 * v + 1] = f.y; e[4 * v + 2] = f.z; e[4 * v + 3] = f.w;
        }
        return true;
    };
    // the first chunk's loads are in flight while the prologue computes the coefficients
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    float e[16];
    bool inside = i < total && fetch(i, e);
    if (d_range)
        quant_ctx_from_range(q, d_range, is_signed, round_mode, prm);
    else
        quant_ctx_load(q, prm, is_signed);
    const bool nearest = round_mode != AXB_ROUND_TOWARD_ZERO;
    const float inv = q.inv, zpo = q.zpo;
    const int lo = q.lo;
    const uint32_t flip = is_signed ? 0x80808080u : 0u;  // raw byte of code lo+u = (u + lo) & 0xFF
    const uint32_t zpw = (uint32_t)(q.zp & 0xFF) * 0x01010101u;
    const int zsum = 16 * q.zp;
    int nonfinite = 0;
    for (; i < bound; i += stride) {
        int32_t s = 0;
        const uint32_t p = i / C16, j = i % C16;
        if (i < total) {
            uint4 out;
            if (!inside) {
                out = make_uint4(zpw, zpw, zpw, zpw);
                s = zsum;
            } else {
                float uf[16];
                bool ok = nearest;
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    uf[k] = fmaf(e[k], inv, zpo);
                    ok &= fabsf(uf[k] - rintf(uf[k])) < 0.49975f;  // false near a tie and for NaN / +-inf
                }
                uint32_t wv[4];
                if (__builtin_expect(ok, 1)) {
                    // round to nearest and clip to [0, 255] (quantizer.py:126-130) in the packing
                    // conversion: two codes per instruction (F2IP.U8)
#pragma unroll
                    for (int v = 0; v < 4; ++v) wv[v] = pack_u8x4(uf[4 * v], uf[4 * v + 1], uf[4 * v + 2], uf[4 * v + 3]);
                } else {
                    int u[16];
#pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        nonfinite |= !(fabsf(e[k]) <= 3.402823466e38f);
                        u[k] = quant_any_u(q, e[k], nearest);
                    }
#pragma unroll
                    for (int v = 0; v < 4; ++v)
                        wv[v] = (uint32_t)u[4 * v] | ((uint32_t)u[4 * v + 1] << 8) | ((uint32_t)u[4 * v + 2] << 16) |
                                ((uint32_t)u[4 * v + 3] << 24);
                }
                uint32_t su = 0;
#pragma unroll
                for (int v = 0; v < 4; ++v) su = __dp4a(wv[v], 0x01010101u, su);
                s = (int32_t)su + 16 * lo;
                out = make_uint4(wv[0] ^ flip, wv[1] ^ flip, wv[2] ^ flip, wv[3] ^ flip);
            }
            reinterpret_cast<uint4 *>(codes)[i] = out;  // chunk i of the padded code tensor
        }
        const uint32_t inext = i + stride;
        inside = inext < total && fetch(inext, e);
        if constexpr (C16 > 1) {
#pragma unroll
            for (int o = PER / 2; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        }
        if constexpr (C16 <= 32) {
            if (i < total && j == 0 && pixsum) pixsum[p] = s;
        } else {
            if (i < total && (j & 31) == 0 && pixsum) atomicAdd(pixsum + p, s);  // pixsum zeroed on the host side
        }
    }
    range_commit(INT32_MAX, INT32_MIN, nonfinite, nullptr, d_flags, AXB_FLAG_NONFINITE);
}

// Unpadded inputs with no per-pixel sums (the CX / ftable kernels sum codes themselves): the code tensor
// is the input tensor element for element (cs == c), so the pass is a flat stream.  A warp takes 512
// consecutive floats per unit -- lane L loads float4 v*32 + L (v = 0..3), every load instruction one
// contiguous 512-byte span, every code store one contiguous 128-byte span -- with the per-element
// arithmetic of quantize_pad16_kernel (fast round-to-nearest, exact path near ties / non-finite).
__global__ void __launch_bounds__(256) quantize_flat_kernel(const float *__restrict__ x, uint32_t nf4,
                                                            axb_qparams *prm, const int32_t *d_range, int is_signed,
                                                            int round_mode, uint32_t *__restrict__ codes,
                                                            int32_t *d_flags) {
    __shared__ QuantCtx q;
    pdl_launch_dependents();
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const uint32_t nunits = (nf4 + 127) >> 7;
    const float4 *x4 = reinterpret_cast<const float4 *>(x);
    float e[16];
    auto fetch = [&](uint32_t uu) {
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const uint32_t idx = (uu << 7) + v * 32 + lane;
            const float4 f = idx < nf4 ? __ldg(x4 + idx) : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
            e[4 * v] = f.x; e[4 * v + 1] = f.y; e[4 * v + 2] = f.z; e[4 * v + 3] = f.w;
        }
    };
    uint32_t u = warp;
    if (u < nunits) fetch(u);  // in flight during the coefficient prologue
    if (d_range)
        quant_ctx_from_range(q, d_range, is_signed, round_mode, prm);
    else
        quant_ctx_load(q, prm, is_signed);
    const bool nearest = round_mode != AXB_ROUND_TOWARD_ZERO;
    const float inv = q.inv, zpo = q.zpo;
    const uint32_t flip = is_signed ? 0x80808080u : 0u;
    int nonfinite = 0;
    for (; u < nunits; u += nwarps) {
        float uf[16];
        bool ok = nearest;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            uf[k] = fmaf(e[k], inv, zpo);
            ok &= fabsf(uf[k] - rintf(uf[k])) < 0.49975f;
        }
        uint32_t wv[4];
        if (__builtin_expect(ok, 1)) {
#pragma unroll
            for (int v = 0; v < 4; ++v) wv[v] = pack_u8x4(uf[4 * v], uf[4 * v + 1], uf[4 * v + 2], uf[4 * v + 3]);
        } else {
            int uu[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                nonfinite |= !(fabsf(e[k]) <= 3.402823466e38f);
                uu[k] = quant_any_u(q, e[k], nearest);
            }
#pragma unroll
            for (int v = 0; v < 4; ++v)
                wv[v] = (uint32_t)uu[4 * v] | ((uint32_t)uu[4 * v + 1] << 8) | ((uint32_t)uu[4 * v + 2] << 16) |
                        ((uint32_t)uu[4 * v + 3] << 24);
        }
        const uint32_t base = u << 7;
        if (u + nwarps < nunits) fetch(u + nwarps);  // the next unit's loads overlap these stores
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const uint32_t idx = base + v * 32 + lane;
            if (idx < nf4) codes[idx] = wv[v] ^ flip;  // raw byte of code lo+u = (u + lo) & 0xFF
        }
    }
    range_commit(INT32_MAX, INT32_MIN, nonfinite, nullptr, d_flags, AXB_FLAG_NONFINITE);
}

// ---------------------------------------------------------------- filters
// HWCN fp32 -> (kpad, coutp) uint8 raw code bytes; row k = (ky*kw + kx)*cs + ci.
__global__ void filters_codes_kernel(const float *__restrict__ f, int64_t kh, int64_t kw, int64_t c, int64_t cout,
                                     int64_t cs, int64_t kpad, int64_t coutp, const axb_qparams *__restrict__ prm,
                                     int is_signed, int round_mode, uint8_t *__restrict__ fcodes, int32_t *d_flags) {
    const double scale = prm->scale;
    const int zp = prm->zero_point;
    const int64_t total = kpad * coutp;
    int nonfinite = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t co = i % coutp;
        const int64_t k = i / coutp;
        const int64_t tap = k / cs, ci = k % cs;
        uint8_t v = 0;
        if (co < cout && tap < kh * kw && ci < c) {
            const float fv = f[(tap * c + ci) * cout + co];  // HWCN flat: ((ky*kw+kx)*c+ci)*cout+co
            nonfinite |= !isfinite(fv);
            const int q = quantize_one(fv, scale, zp, is_signed, round_mode);
            v = (uint8_t)(q & 0xFF);
        }
        fcodes[i] = v;
    }
    range_commit(INT32_MAX, INT32_MIN, nonfinite, nullptr, d_flags, AXB_FLAG_NONFINITE);
}

// S_f[co] = sum of code values over the real taps (axconv.py:207), int64 + overflow flag
__global__ void filters_sum_kernel(const uint8_t *__restrict__ fcodes, int64_t kh, int64_t kw, int64_t c,
                                   int64_t cout, int64_t cs, int64_t coutp, int is_signed, int64_t *fsum,
                                   int32_t *d_flags) {
    const int64_t co = blockIdx.x;
    int64_t s = 0;
    const int64_t taps = kh * kw;
    for (int64_t k = threadIdx.x; k < taps * c; k += blockDim.x) {
        const int64_t tap = k / c, ci = k % c;
        const int raw = fcodes[(tap * cs + ci) * coutp + co];
        s += is_signed ? (int)(int8_t)raw : raw;
    }
    __shared__ long long red[256];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = blockDim.x / 2; o; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        fsum[co] = red[0];
        if (red[0] > INT32_MAX || red[0] < INT32_MIN) atomicOr(d_flags, AXB_FLAG_FSUM_OVF);
    }
}

// ---------------------------------------------------------------- im2col of codes
// One thread per output row: gathers the kh*kw*c codes of its window from the
// zp-padded code tensor into kp/16 16-byte pieces (zeros beyond K) and writes
// the exact row sum (= patch sum S_p, axconv.py:193).
__global__ void __launch_bounds__(256) im2col_pack_kernel(const uint8_t *__restrict__ codes, int64_t n, int64_t hp,
                                                          int64_t wp, int64_t cs, int c, int kh, int kw, int sh,
                                                          int sw, int dh, int dw, int64_t oh, int64_t ow, FastDiv fd_oh,
                                                          FastDiv fd_ow, int kp, int is_signed,
                                                          uint8_t *__restrict__ rows, int32_t *__restrict__ rowsum) {
    const int64_t total = n * oh * ow;
    const int K = kh * kw * c;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < total;
         r += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t t = fdiv((uint32_t)r, fd_ow);
        const int64_t ox = (uint32_t)r - t * (uint32_t)ow;
        const uint32_t b = fdiv(t, fd_oh);
        const int64_t oy = t - b * (uint32_t)oh;
        const uint8_t *base = codes + (((int64_t)b * hp + oy * sh) * wp + ox * sw) * cs;
        int32_t s = 0;
        int k = 0, ky = 0, kx = 0, ci = 0;
        for (int g = 0; g < kp / 16; ++g) {
            uint32_t wv[4] = {0, 0, 0, 0};
#pragma unroll
            for (int u = 0; u < 16; ++u, ++k) {
                if (k < K) {
                    const uint32_t byte = base[((int64_t)ky * dh * wp + kx * dw) * cs + ci];
                    s += is_signed ? (int32_t)(int8_t)byte : (int32_t)byte;
                    wv[u >> 2] |= byte << (8 * (u & 3));
                    if (++ci == c) {
                        ci = 0;
                        if (++kx == kw) {
                            kx = 0;
                            ++ky;
                        }
                    }
                }
            }
            reinterpret_cast<uint4 *>(rows + r * kp)[g] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
        }
        rowsum[r] = s;
    }
}

// ---------------------------------------------------------------- fused quantize + im2col (small-c layers)
// A block owns a QT_H x QT_W tile of output pixels of one image: it quantizes the input patch
// those windows cover ONCE into shared memory (coalesced fp32 loads along the NHWC rows, the
// zero-point code outside the image, axconv.py:185-189), then each thread gathers its window's
// kh*kw*c codes into a kp-byte row (raw 0 beyond K) and writes the row sum S_p (axconv.py:193).
// Same per-element arithmetic as quantize_pad16_kernel (fp32 estimate, exact fallback).
constexpr int QT_H = 8, QT_W = 32;
constexpr int kQiPatchMax = 12288;  // patch codes per block (e.g. 7x7 stride-2 stem: 21 x 69 x 3 = 4,347)
constexpr int kMaxIm2colK = 1024;   // window elements kh*kw*c (K of the small-c layer)

__host__ __device__ inline int qi_patch(int extent_out, int s, int k, int d) { return (extent_out - 1) * s + (k - 1) * d + 1; }

__global__ void __launch_bounds__(QT_H *QT_W) quantize_im2col_kernel(
    const float *__restrict__ x, int n, int h, int w, int c, int pt, int pl, int kh, int kw, int sh, int sw, int dh,
    int dw, int oh, int ow, int tiles_y, int tiles_x, int kp, FastDiv fd_c, FastDiv fd_prow, axb_qparams *prm,
    const int32_t *d_range,
    int is_signed, int round_mode, uint8_t *__restrict__ rows, int32_t *__restrict__ rowsum, int32_t *d_flags) {
    __shared__ QuantCtx q;
    __shared__ __align__(16) uint8_t patch[kQiPatchMax + 16];  // + a word of slack for the funnel reads
    pdl_launch_dependents();
    __shared__ int16_t koff[kMaxIm2colK];  // patch offset of window element k = (ky, kx, ci)
    // koffw[wd]: patch offset of window byte 4*wd when bytes 4wd..4wd+3 are contiguous in the patch (one
    // ky row's kx*c run, dilation 1 along x), else -1 (byte-by-byte gather)
    __shared__ int16_t koffw[kMaxIm2colK / 4];
    if (d_range)
        quant_ctx_from_range(q, d_range, is_signed, round_mode, prm);
    else
        quant_ctx_load(q, prm, is_signed);
    const bool nearest = round_mode != AXB_ROUND_TOWARD_ZERO;
    const int lo = q.lo;
    const int PH = qi_patch(QT_H, sh, kh, dh), PW = qi_patch(QT_W, sw, kw, dw);
    const int prow = PW * c;  // codes per patch row
    const int K = kh * kw * c;
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
        const int t = k / c, ci = k - t * c;
        koff[k] = (int16_t)((t / kw) * dh * prow + (t % kw) * dw * c + ci);
    }
    __syncthreads();
    for (int wd = threadIdx.x; wd < kp / 4; wd += blockDim.x) {
        const int k0 = 4 * wd;
        bool run = k0 + 3 < K;
        for (int u = 1; run && u < 4; ++u) run = koff[k0 + u] == koff[k0] + u;
        koffw[wd] = run ? koff[k0] : (int16_t)-1;
    }
    int nonfinite = 0;
    const int tid = threadIdx.x;
    for (int blk = blockIdx.x; blk < n * tiles_y * tiles_x; blk += gridDim.x) {
        const int b = blk / (tiles_y * tiles_x);
        const int t = blk - b * tiles_y * tiles_x;
        const int oy0 = (t / tiles_x) * QT_H, ox0 = (t % tiles_x) * QT_W;
        const int iy0 = oy0 * sh - pt, ix0 = ox0 * sw - pl;
        const float *img = x + (int64_t)b * h * w * c;
        __syncthreads();  // previous tile's gathers are done with the patch (and koff is written)
        // the patch, flattened: 4 independent loads in flight per thread per pass
        const int total = PH * prow;
        for (int e0 = tid; e0 < total; e0 += 4 * QT_H * QT_W) {
            float v[4];
            bool in[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int e = e0 + j * QT_H * QT_W;
                const uint32_t py = fdiv((uint32_t)e, fd_prow);
                const int r = e - (int)py * prow;
                const int iy = iy0 + (int)py, ix = ix0 + (int)fdiv((uint32_t)r, fd_c);
                in[j] = e < total && iy >= 0 && iy < h && ix >= 0 && ix < w;
                v[j] = in[j] ? __ldg(img + ((int64_t)iy * w + ix0) * c + r) : 0.0f;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int e = e0 + j * QT_H * QT_W;
                if (e >= total) break;
                int code = q.zp;  // zero-point border
                if (in[j]) {
                    const float uf = fmaf(v[j], q.inv, q.zpo);
                    const float rr = rintf(uf);
                    int uo;
                    if (nearest && fabsf(uf - rr) < 0.49975f) {
                        uo = min(max((int)rr, 0), 255);
                    } else {
                        nonfinite |= !(fabsf(v[j]) <= 3.402823466e38f);
                        uo = quant_any_u(q, v[j], nearest);
                    }
                    code = uo + lo;
                }
                patch[e] = (uint8_t)(code & 0xFF);
            }
        }
        __syncthreads();
        const int ty = tid / QT_W, tx = tid % QT_W;
        const int oy = oy0 + ty, ox = ox0 + tx;
        if (oy < oh && ox < ow) {
            const int boff = (ty * sh) * prow + (tx * sw) * c;
            const uint8_t *base = patch + boff;
            const uint32_t *pwords = reinterpret_cast<const uint32_t *>(patch);
            const int64_t r = ((int64_t)b * oh + oy) * ow + ox;
            int32_t ssum = 0;
            for (int g = 0; g < kp / 16; ++g) {
                uint32_t wv[4];
#pragma unroll
                for (int v4 = 0; v4 < 4; ++v4) {
                    const int o = koffw[g * 4 + v4];
                    uint32_t word = 0;
                    if (o >= 0) {  // 4 contiguous patch bytes: two aligned words, one funnel shift
                        const uint32_t a = (uint32_t)(boff + o);
                        word = __funnelshift_r(pwords[a >> 2], pwords[(a >> 2) + 1], (a & 3u) * 8u);
                    } else {
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int k = g * 16 + v4 * 4 + u;
                            if (k < K) word |= (uint32_t)base[koff[k]] << (8 * u);
                        }
                    }
                    wv[v4] = word;
                    ssum = is_signed ? __dp4a((int)word, 0x01010101, ssum)  // junk bytes are 0
                                     : (int32_t)__dp4a(word, 0x01010101u, (uint32_t)ssum);
                }
                reinterpret_cast<uint4 *>(rows + r * kp)[g] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
            }
            rowsum[r] = ssum;
        }
    }
    if (__syncthreads_or(nonfinite) && threadIdx.x == 0 && d_flags) atomicOr(d_flags, AXB_FLAG_NONFINITE);
}

}  // namespace axb

// ======================================================================== C ABI
using namespace axb;

extern "C" {

int64_t axb_channel_stride(int64_t c) { return (c + 15) / 16 * 16; }

int64_t axb_conv_im2col_kp(int64_t c, int64_t kh, int64_t kw) {
    if (c % 16 == 0 || kh * kw == 1) return 0;
    return (kh * kw * c + 15) / 16 * 16;
}

int axb_im2col_pack(const uint8_t *d_codes, int64_t n, int64_t hp, int64_t wp, int64_t cs, int64_t c, int32_t kh,
                    int32_t kw, int32_t sh, int32_t sw, int32_t dh, int32_t dw, int64_t oh, int64_t ow, int64_t kp,
                    int is_signed, uint8_t *d_rows, int32_t *d_rowsum, void *stream) {
    const int64_t rows = n * oh * ow;
    if (rows == 0) return AXB_OK;
    if (kp % 16 || kp < kh * kw * c) return set_error(AXB_E_VALUE, "bad im2col row length");
    int64_t blocks = (rows + 255) / 256;
    const int64_t cap = (int64_t)sm_count() * 16;
    if (blocks > cap) blocks = cap;
    if (rows >= (int64_t(1) << 32)) return set_error(AXB_E_VALUE, "im2col: more than 2^32 rows");
    im2col_pack_kernel<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(
        d_codes, n, hp, wp, cs, (int)c, kh, kw, sh, sw, dh, dw, oh, ow, make_fastdiv((uint32_t)oh),
        make_fastdiv((uint32_t)ow), (int)kp, is_signed, d_rows, d_rowsum);
    return check_launch("im2col_pack");
}

static int quantize_pad_launch(const float *d_x, int64_t n, int64_t h, int64_t w, int64_t c, int32_t pt, int32_t pb,
                               int32_t pl, int32_t pr, int64_t cs, axb_qparams *d_params, const int32_t *d_range,
                               int is_signed, int round_mode, uint8_t *d_codes, int32_t *d_pixsum, int32_t *d_flags,
                               void *stream);

int axb_quantize_im2col(const float *d_x, int64_t n, int64_t h, int64_t w, int64_t c, int32_t pt, int32_t pl,
                        int32_t kh, int32_t kw, int32_t sh, int32_t sw, int32_t dh, int32_t dw, int64_t oh, int64_t ow,
                        int64_t kp, const int32_t *d_range, axb_qparams *d_params, int is_signed, int round_mode,
                        uint8_t *d_rows, int32_t *d_rowsum, int32_t *d_flags, void *stream) {
    const int64_t rows = n * oh * ow;
    if (rows == 0) return AXB_OK;
    if (!d_params) return set_error(AXB_E_VALUE, "null parameter buffer");
    if (kp % 16 || kp < kh * kw * c) return set_error(AXB_E_VALUE, "bad im2col row length");
    if (rows >= (int64_t(1) << 32) || n * h * w * c >= (int64_t(1) << 40))
        return set_error(AXB_E_VALUE, "quantize_im2col: tensor too large");
    if ((int64_t)qi_patch(QT_H, sh, kh, dh) * qi_patch(QT_W, sw, kw, dw) * c > kQiPatchMax ||
        (int64_t)kh * kw * c > kMaxIm2colK) {
        // window patch too large for the tiled kernel: quantize into a zp-padded code tensor, then gather
        cudaStream_t st = (cudaStream_t)stream;
        const int64_t need_h = (oh - 1) * sh + (kh - 1) * dh + 1, need_w = (ow - 1) * sw + (kw - 1) * dw + 1;
        const int64_t pb = need_h - h - pt > 0 ? need_h - h - pt : 0, pr = need_w - w - pl > 0 ? need_w - w - pl : 0;
        const int64_t hp = h + pt + pb, wp = w + pl + pr;
        const int64_t cs = axb_channel_stride(c);
        uint8_t *codes = nullptr;
        int32_t *pix = nullptr;
        if (cudaMallocAsync(&codes, n * hp * wp * cs, st) != cudaSuccess ||
            cudaMallocAsync(&pix, n * hp * wp * 4, st) != cudaSuccess) {
            if (codes) cudaFreeAsync(codes, st);
            return set_error(AXB_E_CUDA, "quantize_im2col: scratch allocation failed");
        }
        int rc = quantize_pad_launch(d_x, n, h, w, c, pt, (int32_t)pb, pl, (int32_t)pr, cs, d_params, d_range,
                                     is_signed, round_mode, codes, pix, d_flags, stream);
        if (!rc)
            rc = axb_im2col_pack(codes, n, hp, wp, cs, c, kh, kw, sh, sw, dh, dw, oh, ow, kp, is_signed, d_rows,
                                 d_rowsum, stream);
        cudaFreeAsync(codes, st);
        cudaFreeAsync(pix, st);
        return rc;
    }
    const int tiles_y = (int)((oh + QT_H - 1) / QT_H), tiles_x = (int)((ow + QT_W - 1) / QT_W);
    int64_t blocks = n * tiles_y * tiles_x;
    const int64_t cap = (int64_t)sm_count() * 8;
    if (blocks > cap) blocks = cap;
    quantize_im2col_kernel<<<(int)blocks, QT_H * QT_W, 0, (cudaStream_t)stream>>>(
        d_x, (int)n, (int)h, (int)w, (int)c, pt, pl, kh, kw, sh, sw, dh, dw, (int)oh, (int)ow, tiles_y, tiles_x,
        (int)kp, make_fastdiv((uint32_t)c),
        make_fastdiv((uint32_t)(qi_patch(QT_W, sw, kw, dw) * c)), d_params, d_range, is_signed, round_mode, d_rows,
        d_rowsum, d_flags);
    return check_launch("quantize_im2col");
}

int axb_range_reset(int32_t *d_range, void *stream) {
    range_reset_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(d_range);
    return check_launch("range_reset");
}

int axb_range_minmax(const float *d_x, int64_t n, int32_t *d_range, int32_t *d_flags, void *stream) {
    if (n <= 0) return set_error(AXB_E_VALUE, "cannot take the range of an empty tensor");
    int64_t blocks = (n / 4 + 255) / 256;
    const int64_t cap = (int64_t)sm_count() * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    range_kernel<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(d_x, n, d_range, d_flags);
    return check_launch("range_minmax");
}

int axb_range_read(const int32_t *d_range, const int32_t *d_flags, float *mn, float *mx, int32_t *flags,
                   void *stream) {
    int32_t r[2] = {0, 0};
    int32_t fl = 0;
    cudaStream_t s = (cudaStream_t)stream;
    if (cudaMemcpyAsync(r, d_range, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess)
        return set_error(AXB_E_CUDA, "range readback failed");
    if (d_flags && cudaMemcpyAsync(&fl, d_flags, 4, cudaMemcpyDeviceToHost, s) != cudaSuccess)
        return set_error(AXB_E_CUDA, "flag readback failed");
    if (cudaStreamSynchronize(s) != cudaSuccess) return set_error(AXB_E_CUDA, "stream sync failed");
    *mn = ord2f(r[0]);
    *mx = ord2f(r[1]);
    if (flags) *flags = fl;
    return AXB_OK;
}

int axb_coeffs_host(double mn, double mx, int is_signed, int round_mode, axb_qparams *out) {
    if (!(mn == mn) || !(mx == mx) || mn - mn != 0.0 || mx - mx != 0.0)
        return set_error(AXB_E_VALUE, "range must be finite");
    if (mn > mx) return set_error(AXB_E_VALUE, "range min exceeds max");
    *out = coeffs(mn, mx, is_signed, round_mode);
    fill_bounds(*out, is_signed, round_mode, 0, 1);
    return AXB_OK;
}

int axb_coeffs_from_range(const int32_t *d_range, int is_signed, int round_mode, axb_qparams *d_out,
                          void *stream) {
    coeffs_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(d_range, is_signed, round_mode, d_out);
    return check_launch("coeffs_from_range");
}

int axb_params_upload(const axb_qparams *host_params, axb_qparams *d_params, void *stream) {
    params_set_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(*host_params, d_params);
    return check_launch("params_upload");
}

static int quantize_pad_launch(const float *d_x, int64_t n, int64_t h, int64_t w, int64_t c, int32_t pt, int32_t pb,
                               int32_t pl, int32_t pr, int64_t cs, axb_qparams *d_params, const int32_t *d_range,
                               int is_signed, int round_mode, uint8_t *d_codes, int32_t *d_pixsum, int32_t *d_flags,
                               void *stream) {
    if (cs != axb_channel_stride(c)) return set_error(AXB_E_VALUE, "channel stride mismatch");
    const int64_t hp = h + pt + pb, wp = w + pl + pr;
    const int64_t total = n * hp * wp;
    if (total == 0) return AXB_OK;
    cudaStream_t s = (cudaStream_t)stream;
    // one resident wave (the in-kernel coefficient prologue is paid once per CTA)
    const int64_t cap = (int64_t)sm_count() * 6;
    if (total * (cs / 4) >= (int64_t(1) << 31)) return set_error(AXB_E_VALUE, "quantize: more than 2^31 code words");
    const FastDiv fhp = make_fastdiv((uint32_t)hp), fwp = make_fastdiv((uint32_t)wp);
    const int64_t c16 = c / 16;
#ifndef AXB_EXP_NO_FLAT
    if (pt == 0 && pb == 0 && pl == 0 && pr == 0 && d_pixsum == nullptr && c % 16 == 0 && cs == c &&
        (reinterpret_cast<uintptr_t>(d_x) & 15) == 0) {
        // unpadded, no pixel sums: the flat stream kernel (one resident wave)
        const int64_t nf4 = total * c / 4;
        int64_t blocks = (nf4 / 128 + 8) / 8;  // 8 warps per CTA, one 128-float4 unit per warp
        const int64_t capf = (int64_t)sm_count() * 4;
        if (blocks > capf) blocks = capf;
        quantize_flat_kernel<<<(int)blocks, 256, 0, s>>>(d_x, (uint32_t)nf4, d_params, d_range, is_signed, round_mode,
                                                        reinterpret_cast<uint32_t *>(d_codes), d_flags);
        return check_launch("quantize_flat");
    }
#endif
    if (c % 16 == 0 && c16 <= 128 && (c16 & (c16 - 1)) == 0 && ((reinterpret_cast<uintptr_t>(d_x) & 15) == 0)) {
        // wide pixels (c = 1024, 2048): one warp per 32 chunks, per-pixel sums by atomics into a zeroed buffer
        if (c16 > 32 && d_pixsum && cudaMemsetAsync(d_pixsum, 0, total * 4, s) != cudaSuccess)
            return set_error(AXB_E_CUDA, "pixsum clear failed");
        int64_t blocks = (total * c16 + 255) / 256;
        const int64_t cap16 = (int64_t)sm_count() * 4;  // one resident wave: the prologue is paid once per CTA
        if (blocks > cap16) blocks = cap16;
#define AXB_Q16(CC)                                                                                                 \
    quantize_pad16_kernel<CC><<<(int)blocks, 256, 0, s>>>(d_x, (int)n, (int)h, (int)w, pt, pl, (int)hp, (int)wp,    \
                                                          fhp, fwp, d_params, d_range, is_signed, round_mode,       \
                                                          d_codes, d_pixsum, d_flags)
        switch (c16) {
            case 1: AXB_Q16(1); break;
            case 2: AXB_Q16(2); break;
            case 4: AXB_Q16(4); break;
            case 8: AXB_Q16(8); break;
            case 16: AXB_Q16(16); break;
            case 32: AXB_Q16(32); break;
            case 64: AXB_Q16(64); break;
            default: AXB_Q16(128); break;
        }
#undef AXB_Q16
        return check_launch("quantize_pad16");
    }
    const int64_t G = cs / 4;
    const int64_t work = (G <= 32 && (G & (G - 1)) == 0) ? total * G : total * 32;
    int64_t blocks = (work + 255) / 256;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
#define AXB_QLAUNCH(GG)                                                                                             \
    quantize_pad_kernel<GG><<<(int)blocks, 256, 0, s>>>(d_x, n, h, w, (int)c, cs, pt, pl, hp, wp, fhp, fwp, d_params, \
                                                        d_range, is_signed, round_mode, d_codes, d_pixsum, d_flags)
    switch (G) {
        case 4: AXB_QLAUNCH(4); break;
        case 8: AXB_QLAUNCH(8); break;
        case 16: AXB_QLAUNCH(16); break;
        case 32: AXB_QLAUNCH(32); break;
        default: AXB_QLAUNCH(0); break;
    }
#undef AXB_QLAUNCH
    return check_launch("quantize_pad");
}

int axb_quantize_pad(const float *d_x, int64_t n, int64_t h, int64_t w, int64_t c, int32_t pt, int32_t pb,
                     int32_t pl, int32_t pr, int64_t cs, const axb_qparams *d_params, int is_signed,
                     int round_mode, uint8_t *d_codes, int32_t *d_pixsum, int32_t *d_flags, void *stream) {
    return quantize_pad_launch(d_x, n, h, w, c, pt, pb, pl, pr, cs, const_cast<axb_qparams *>(d_params), nullptr,
                               is_signed, round_mode, d_codes, d_pixsum, d_flags, stream);
}

int axb_quantize_pad_range(const float *d_x, int64_t n, int64_t h, int64_t w, int64_t c, int32_t pt, int32_t pb,
                           int32_t pl, int32_t pr, int64_t cs, const int32_t *d_range, int is_signed, int round_mode,
                           axb_qparams *d_params_out, uint8_t *d_codes, int32_t *d_pixsum, int32_t *d_flags,
                           void *stream) {
    if (!d_range || !d_params_out) return set_error(AXB_E_VALUE, "null range or parameter buffer");
    return quantize_pad_launch(d_x, n, h, w, c, pt, pb, pl, pr, cs, d_params_out, d_range, is_signed, round_mode,
                               d_codes, d_pixsum, d_flags, stream);
}

int64_t axb_filter_kpad(int64_t kh, int64_t kw, int64_t cs) { return (kh * kw * cs + 15) / 16 * 16; }
int64_t axb_filter_coutp(int64_t cout) { return (cout + 15) / 16 * 16; }

int axb_filters_prepare(const float *d_f, int64_t kh, int64_t kw, int64_t c, int64_t cout, int64_t cs,
                        const axb_qparams *d_params, int is_signed, int round_mode, uint8_t *d_fcodes,
                        int64_t *d_fsum, int32_t *d_flags, void *stream) {
    if (cs != axb_channel_stride(c)) return set_error(AXB_E_VALUE, "channel stride mismatch");
    const int64_t kpad = axb_filter_kpad(kh, kw, cs), coutp = axb_filter_coutp(cout);
    cudaStream_t s = (cudaStream_t)stream;
    int64_t blocks = (kpad * coutp + 255) / 256;
    if (blocks > 4096) blocks = 4096;
    filters_codes_kernel<<<(int)blocks, 256, 0, s>>>(d_f, kh, kw, c, cout, cs, kpad, coutp, d_params, is_signed,
                                                      round_mode, d_fcodes, d_flags);
    if (int e = check_launch("filters_codes")) return e;
    if (cout > 0) {
        filters_sum_kernel<<<(int)cout, 256, 0, s>>>(d_fcodes, kh, kw, c, cout, cs, coutp, is_signed, d_fsum,
                                                      d_flags);
    }
    return check_launch("filters_sum");
}

}  // extern "C"
