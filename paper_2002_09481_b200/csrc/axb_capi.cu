// C ABI glue: errors, device info, truth-table handles, the whole-operator
// entry point (axconv2d) and the float-glue kernels of the graph executor.
#include <cstdio>
#include <cstring>
#include <string>

#include "axb_common.cuh"
#include "axb_internal.h"

namespace axb {

static thread_local std::string g_last_error;
static thread_local const char *g_last_kernel = "";

int set_error(int code, const char *msg) {
    g_last_error = msg ? msg : "";
    return code;
}

int check_launch(const char *what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        char buf[256];
        snprintf(buf, sizeof buf, "%s: %s", what, cudaGetErrorString(e));
        return set_error(AXB_E_CUDA, buf);
    }
    return AXB_OK;
}

int sm_count() {
    static int cached[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cached[dev]) {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        cached[dev] = n > 0 ? n : 1;
    }
    return cached[dev];
}

void set_last_kernel(const char *name) { g_last_kernel = name; }

// b-major transpose: T[b*256 + a] = entries[(a << 8) | b]
__global__ void lut_transpose_kernel(const uint16_t *__restrict__ amajor, uint16_t *__restrict__ bmajor) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;  // output index b*256 + a
    if (i < kLutEntries) {
        const int b = i >> 8, a = i & 255;
        bmajor[i] = amajor[(a << 8) | b];
    }
}

// ---------------------------------------------------------------- float glue
// MaxPool (graph.py:182-192 with -inf fill): NaN propagates like np.max.
__global__ void maxpool_kernel(const float *__restrict__ x, int64_t n, int64_t h, int64_t w, int64_t c, int ph,
                               int pw, int sh, int sw, int pt, int pl, int64_t oh, int64_t ow, float *__restrict__ out,
                               int32_t *d_range, int32_t *d_flags) {
    int32_t tmin = INT32_MAX, tmax = INT32_MIN;
    int nonfinite = 0;
    const int64_t total = n * oh * ow * c;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t ci = i % c;
        int64_t t = i / c;
        const int64_t ox = t % ow;
        t /= ow;
        const int64_t oy = t % oh;
        const int64_t b = t / oh;
        float m = -INFINITY;
        for (int ky = 0; ky < ph; ++ky) {
            const int64_t iy = oy * sh + ky - pt;
            for (int kx = 0; kx < pw; ++kx) {
                const int64_t ix = ox * sw + kx - pl;
                const float v = (iy >= 0 && iy < h && ix >= 0 && ix < w) ? x[((b * h + iy) * w + ix) * c + ci]
                                                                         : -INFINITY;
                if (m == m && (v > m || v != v)) m = v;
            }
        }
        out[i] = m;
        nonfinite |= !isfinite(m);
        const int32_t o = f2ord(m);
        tmin = min(tmin, o);
        tmax = max(tmax, o);
    }
    range_commit(tmin, tmax, nonfinite, d_range, d_flags, AXB_FLAG_OUT_NONFINITE);
}

// Vectorised pools for c % 4 == 0: one thread per (output pixel, 4 channels), float4 loads and
// stores, 32-bit magic-number index division (the scalar kernels above spend most of their time
// in 64-bit div/mod).  Identical per-element arithmetic and order.
// PB taps' loads in flight per batch: 9 for windows of <= 9 taps (ResNet's 3x3 max pool: 36 fewer live
// registers than 16, more resident warps), 16 otherwise (global average pools)
template <bool MAX, int PB = 16>
__global__ void __launch_bounds__(256) pool4_kernel(const float4 *__restrict__ x, int h, int w, int c4, int ph,
                                                    int pw, int sh, int sw, int pt, int pl, int oh, int ow,
                                                    uint32_t total, FastDiv fd_c4, FastDiv fd_ow, FastDiv fd_oh,
                                                    float4 *__restrict__ out, int32_t *d_range, int32_t *d_flags) {
    int32_t tmin = INT32_MAX, tmax = INT32_MIN;
    int nonfinite = 0;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const uint32_t t = fdiv(i, fd_c4);
        const int cg = (int)(i - t * (uint32_t)c4);
        const uint32_t t2 = fdiv(t, fd_ow);
        const int ox = (int)(t - t2 * (uint32_t)ow);
        const uint32_t b = fdiv(t2, fd_oh);
        const int oy = (int)(t2 - b * (uint32_t)oh);
        float r[4];
        int valid = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) r[j] = MAX ? -INFINITY : 0.0f;
        // taps in sequential (ky, kx) order, PB at a time: the PB loads are issued before the
        // dependent fp32 chain consumes them (a global 8x8 pool has only n*c/4 threads, so memory-
        // level parallelism per thread is what bounds it); the arithmetic order is unchanged
        const int taps = ph * pw;
        int ky = 0, kx = 0;
        for (int t0 = 0; t0 < taps; t0 += PB) {
            float4 vv[PB];
            bool inb[PB];
#pragma unroll
            for (int u = 0; u < PB; ++u) {
                const int iy = oy * sh + ky - pt, ix = ox * sw + kx - pl;
                inb[u] = t0 + u < taps && iy >= 0 && iy < h && ix >= 0 && ix < w;
                vv[u] = make_float4(MAX ? -INFINITY : 0.0f, MAX ? -INFINITY : 0.0f, MAX ? -INFINITY : 0.0f,
                                    MAX ? -INFINITY : 0.0f);
                if (inb[u]) vv[u] = __ldg(x + (((int64_t)b * h + iy) * w + ix) * c4 + cg);
                if (++kx == pw) {
                    kx = 0;
                    ++ky;
                }
            }
#pragma unroll
            for (int u = 0; u < PB; ++u) {
                if (t0 + u >= taps) break;
                const float v[4] = {vv[u].x, vv[u].y, vv[u].z, vv[u].w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (MAX) {
                        if (r[j] == r[j] && (v[j] > r[j] || v[j] != v[j])) r[j] = v[j];  // np.max, NaN wins
                    } else {
                        // nansum starts from +0.0 (an all -0.0 window sums to +0.0, like numpy)
                        const float q = v[j] != v[j] ? 0.0f : v[j];
                        r[j] = __fadd_rn(r[j], q);
                    }
                }
                valid += inb[u];
            }
        }
        if (!MAX) {
#pragma unroll
            for (int j = 0; j < 4; ++j) r[j] = __double2float_rn((double)r[j] / (double)valid);
        }
        out[i] = make_float4(r[0], r[1], r[2], r[3]);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            nonfinite |= !isfinite(r[j]);
            const int32_t o = f2ord(r[j]);
            tmin = min(tmin, o);
            tmax = max(tmax, o);
        }
    }
    range_commit(tmin, tmax, nonfinite, d_range, d_flags, AXB_FLAG_OUT_NONFINITE);
}

// AvgPool (graph.py:193-199): nansum in sequential (ky, kx) fp32 order (padding
// taps add +0.0), then float32 / int64 -> float64 division, narrowed to fp32.
__global__ void avgpool_kernel(const float *__restrict__ x, int64_t n, int64_t h, int64_t w, int64_t c, int ph,
                               int pw, int sh, int sw, int pt, int pl, int64_t oh, int64_t ow, float *__restrict__ out,
                               int32_t *d_range, int32_t *d_flags) {
    int32_t tmin = INT32_MAX, tmax = INT32_MIN;
    int nonfinite = 0;
    const int64_t total = n * oh * ow * c;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t ci = i % c;
        int64_t t = i / c;
        const int64_t ox = t % ow;
        t /= ow;
        const int64_t oy = t % oh;
        const int64_t b = t / oh;
        float s = 0.0f;  // nansum's +0.0 start (an all -0.0 window gives +0.0, like numpy)
        int64_t valid = 0;
        for (int ky = 0; ky < ph; ++ky) {
            const int64_t iy = oy * sh + ky - pt;
            for (int kx = 0; kx < pw; ++kx) {
                const int64_t ix = ox * sw + kx - pl;
                const bool in = iy >= 0 && iy < h && ix >= 0 && ix < w;
                float v = in ? x[((b * h + iy) * w + ix) * c + ci] : 0.0f;
                if (v != v) v = 0.0f;  // nansum
                valid += in;
                s = __fadd_rn(s, v);
            }
        }
        const float y = __double2float_rn((double)s / (double)valid);
        out[i] = y;
        nonfinite |= !isfinite(y);
        const int32_t o = f2ord(y);
        tmin = min(tmin, o);
        tmax = max(tmax, o);
    }
    range_commit(tmin, tmax, nonfinite, d_range, d_flags, AXB_FLAG_OUT_NONFINITE);
}

__global__ void add_relu_kernel(const float *__restrict__ a, const float *__restrict__ b, int64_t n, int relu,
                                float *__restrict__ out, int32_t *d_range, int32_t *d_flags) {
    int32_t tmin = INT32_MAX, tmax = INT32_MIN;
    int nonfinite = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        float y = a[i];
        if (b) y = __fadd_rn(y, b[i]);
        if (relu) y = (y > 0.0f || y != y) ? y : 0.0f;
        out[i] = y;
        nonfinite |= !isfinite(y);
        const int32_t o = f2ord(y);
        tmin = min(tmin, o);
        tmax = max(tmax, o);
    }
    range_commit(tmin, tmax, nonfinite, d_range, d_flags, AXB_FLAG_OUT_NONFINITE);
}

static int grid_for(int64_t total) {
    int64_t blocks = (total + 255) / 256;
    const int64_t cap = (int64_t)sm_count() * 16;
    if (blocks > cap) blocks = cap;
    return blocks < 1 ? 1 : (int)blocks;
}

// Small pools (e.g. the global 8x8 average pool: n*c/4 threads, each a long tap chain): 64-thread
// blocks so every SM gets work.
static void pool_launch_dims(uint32_t t4, int *grid, int *block) {
    *block = t4 < (uint32_t)sm_count() * 4 * 256 ? 64 : 256;
    int64_t blocks = ((int64_t)t4 + *block - 1) / *block;
    const int64_t cap = (int64_t)sm_count() * 16 * (256 / *block);
    if (blocks > cap) blocks = cap;
    *grid = blocks < 1 ? 1 : (int)blocks;
}

}  // namespace axb

using namespace axb;

extern "C" {

const char *axb_last_error(void) { return g_last_error.c_str(); }
const char *axb_last_kernel(void) { return g_last_kernel; }
int axb_version(void) { return 1; }

int axb_device_info(int device, int *sm, int *smem_optin, int *major, int *minor) {
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return set_error(AXB_E_CUDA, "no CUDA device");
    if (sm) *sm = prop.multiProcessorCount;
    if (smem_optin) *smem_optin = (int)prop.sharedMemPerBlockOptin;
    if (major) *major = prop.major;
    if (minor) *minor = prop.minor;
    return AXB_OK;
}

int axb_lut_create(const uint16_t *entries, int is_signed, axb_lut **out) {
    if (!entries || !out) return set_error(AXB_E_VALUE, "null truth table");
    axb_lut *l = new axb_lut();
    l->is_signed = is_signed ? 1 : 0;
    l->f00 = is_signed ? (int32_t)(int16_t)entries[0] : (int32_t)entries[0];
    if (cudaMalloc(&l->d_amajor, kLutBytes) != cudaSuccess || cudaMalloc(&l->d_bmajor, kLutBytes) != cudaSuccess) {
        delete l;
        return set_error(AXB_E_CUDA, "cannot allocate truth table");
    }
    if (cudaMemcpy(l->d_amajor, entries, kLutBytes, cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaFree(l->d_amajor);
        cudaFree(l->d_bmajor);
        delete l;
        return set_error(AXB_E_CUDA, "cannot upload truth table");
    }
    lut_transpose_kernel<<<kLutEntries / 256, 256>>>(l->d_amajor, l->d_bmajor);
    if (int e = check_launch("lut_transpose")) return e;
    if (cudaDeviceSynchronize() != cudaSuccess) return set_error(AXB_E_CUDA, "lut transpose failed");
    *out = l;
    return AXB_OK;
}

int axb_lut_destroy(axb_lut *l) {
    if (!l) return AXB_OK;
    cudaFree(l->d_amajor);
    cudaFree(l->d_bmajor);
    delete l;
    return AXB_OK;
}

int axb_lut_is_signed(const axb_lut *l) { return l ? l->is_signed : -1; }
const uint16_t *axb_lut_device_bmajor(const axb_lut *l) { return l ? l->d_bmajor : nullptr; }

int axb_maxpool(const float *d_x, int64_t n, int64_t h, int64_t w, int64_t c, int32_t ph, int32_t pw, int32_t sh,
                int32_t sw, int32_t pt, int32_t pl, int64_t oh, int64_t ow, float *d_out, int32_t *d_out_range,
                int32_t *d_flags, void *stream) {
    const int64_t total = n * oh * ow * c;
    if (total == 0) return AXB_OK;
    if (c % 4 == 0 && total / 4 < (int64_t(1) << 32) && ((reinterpret_cast<uintptr_t>(d_x) |
                                                            reinterpret_cast<uintptr_t>(d_out)) & 15) == 0) {
        const uint32_t t4 = (uint32_t)(total / 4);
        int pg, pb;
        pool_launch_dims(t4, &pg, &pb);
        auto fn = ph * pw <= 9 ? pool4_kernel<true, 9> : pool4_kernel<true, 16>;
        fn<<<pg, pb, 0, (cudaStream_t)stream>>>(
            reinterpret_cast<const float4 *>(d_x), (int)h, (int)w, (int)(c / 4), ph, pw, sh, sw, pt, pl, (int)oh,
            (int)ow, t4, make_fastdiv((uint32_t)(c / 4)), make_fastdiv((uint32_t)ow), make_fastdiv((uint32_t)oh),
            reinterpret_cast<float4 *>(d_out), d_out_range, d_flags);
        return check_launch("maxpool4");
    }
    maxpool_kernel<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>(d_x, n, h, w, c, ph, pw, sh, sw, pt, pl, oh,
                                                                       ow, d_out, d_out_range, d_flags);
    return check_launch("maxpool");
}

int axb_avgpool(const float *d_x, int64_t n, int64_t h, int64_t w, int64_t c, int32_t ph, int32_t pw, int32_t sh,
                int32_t sw, int32_t pt, int32_t pl, int64_t oh, int64_t ow, float *d_out, int32_t *d_out_range,
                int32_t *d_flags, void *stream) {
    const int64_t total = n * oh * ow * c;
    if (total == 0) return AXB_OK;
    if (c % 4 == 0 && total / 4 < (int64_t(1) << 32) && ((reinterpret_cast<uintptr_t>(d_x) |
                                                            reinterpret_cast<uintptr_t>(d_out)) & 15) == 0) {
        const uint32_t t4 = (uint32_t)(total / 4);
        int pg, pb;
        pool_launch_dims(t4, &pg, &pb);
        auto fn = ph * pw <= 9 ? pool4_kernel<false, 9> : pool4_kernel<false, 16>;
        fn<<<pg, pb, 0, (cudaStream_t)stream>>>(
            reinterpret_cast<const float4 *>(d_x), (int)h, (int)w, (int)(c / 4), ph, pw, sh, sw, pt, pl, (int)oh,
            (int)ow, t4, make_fastdiv((uint32_t)(c / 4)), make_fastdiv((uint32_t)ow), make_fastdiv((uint32_t)oh),
            reinterpret_cast<float4 *>(d_out), d_out_range, d_flags);
        return check_launch("avgpool4");
    }
    avgpool_kernel<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>(d_x, n, h, w, c, ph, pw, sh, sw, pt, pl, oh,
                                                                       ow, d_out, d_out_range, d_flags);
    return check_launch("avgpool");
}

int axb_add_relu(const float *d_a, const float *d_b, int64_t n, int32_t relu, float *d_out, int32_t *d_out_range,
                 int32_t *d_flags, void *stream) {
    if (n == 0) return AXB_OK;
    add_relu_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(d_a, d_b, n, relu, d_out, d_out_range, d_flags);
    return check_launch("add_relu");
}

// Whole operator, device buffers + host ranges (axconv.py:266-297).
int axb_axconv2d(const float *d_x, int64_t n, int64_t h, int64_t w, int64_t c, const float *d_f, int64_t kh,
                 int64_t kw, int64_t cout, int32_t sh, int32_t sw, int32_t dh, int32_t dw, int32_t pt, int32_t pb,
                 int32_t pl, int32_t pr, double in_min, double in_max, double f_min, double f_max,
                 int32_t round_mode, int32_t accumulator, const axb_lut *lut, float *d_out, int64_t *d_acc_out,
                 void *stream) {
    if (!lut) return set_error(AXB_E_VALUE, "null truth table");
    cudaStream_t s = (cudaStream_t)stream;
    const int sgn = lut->is_signed;
    axb_qparams p1, p2;
    if (int e = axb_coeffs_host(in_min, in_max, sgn, round_mode, &p1)) return e;
    if (int e = axb_coeffs_host(f_min, f_max, sgn, round_mode, &p2)) return e;
    const int64_t hp = h + pt + pb, wp = w + pl + pr;
    const int64_t ekh = (kh - 1) * dh + 1, ekw = (kw - 1) * dw + 1;
    if (hp < ekh || wp < ekw) return set_error(AXB_E_VALUE, "kernel extent exceeds padded input");
    const int64_t oh = (hp - ekh) / sh + 1, ow = (wp - ekw) / sw + 1;
    if (n == 0 || cout == 0) return AXB_OK;
    const int64_t cs = axb_channel_stride(c);
    const int64_t kp = axb_conv_im2col_kp(c, kh, kw);  // small-channel layers: explicit im2col rows
    // filter geometry as the conv kernel sees it: (1,1,K) over kp-byte rows, or (kh,kw,c) over cs
    const int64_t fkh = kp ? 1 : kh, fkw = kp ? 1 : kw, fc = kp ? kh * kw * c : c, fcs = kp ? kp : cs;
    const int64_t kpad = axb_filter_kpad(fkh, fkw, fcs), coutp = axb_filter_coutp(cout);

    uint8_t *codes = nullptr, *rows = nullptr;
    int32_t *pixsum = nullptr, *flags = nullptr, *rowsum = nullptr;
    axb_qparams *dp = nullptr;
    uint8_t *fcodes = nullptr;
    int64_t *fsum = nullptr;
    uint32_t *ftable = nullptr;
    int rc = AXB_OK;
    auto fail = [&](int code, const char *msg) {
        if (rc == AXB_OK) rc = set_error(code, msg);
    };
    if (cudaMallocAsync(&codes, n * hp * wp * cs, s) != cudaSuccess ||
        cudaMallocAsync(&pixsum, n * hp * wp * 4, s) != cudaSuccess ||
        cudaMallocAsync(&flags, 8, s) != cudaSuccess || cudaMallocAsync(&dp, 2 * sizeof(axb_qparams), s) != cudaSuccess ||
        cudaMallocAsync(&fcodes, kpad * coutp, s) != cudaSuccess ||
        cudaMallocAsync(&fsum, (cout > 0 ? cout : 1) * 8, s) != cudaSuccess ||
        (kp && (cudaMallocAsync(&rows, n * oh * ow * kp, s) != cudaSuccess ||
                cudaMallocAsync(&rowsum, n * oh * ow * 4, s) != cudaSuccess))) {
        fail(AXB_E_CUDA, "device allocation failed");
    }
    if (rc == AXB_OK) {
        cudaMemsetAsync(flags, 0, 8, s);
        if (int e = axb_params_upload(&p1, dp, s)) rc = e;
        if (!rc) rc = axb_params_upload(&p2, dp + 1, s);
        if (!rc)
            rc = axb_filters_prepare(d_f, fkh, fkw, fc, cout, fcs, dp + 1, sgn, round_mode, fcodes, fsum, flags, s);
    }
    if (!rc)
        rc = axb_quantize_pad(d_x, n, h, w, c, pt, pb, pl, pr, cs, dp, sgn, round_mode, codes, pixsum, flags + 1,
                              s);
    if (!rc && kp)
        rc = axb_im2col_pack(codes, n, hp, wp, cs, c, (int32_t)kh, (int32_t)kw, sh, sw, dh, dw, oh, ow, kp, sgn, rows,
                             rowsum, s);
    if (!rc) {
        axb_conv_desc d;
        memset(&d, 0, sizeof d);
        if (kp) {
            d.codes = rows;
            d.pixsum = rowsum;
            d.n = n; d.hp = oh; d.wp = ow; d.cs = kp; d.c = kh * kw * c;
            d.kh = d.kw = d.sh = d.sw = d.dh = d.dw = 1;
        } else {
            d.codes = codes;
            d.pixsum = pixsum;
            d.n = n; d.hp = hp; d.wp = wp; d.cs = cs; d.c = c;
            d.kh = (int32_t)kh; d.kw = (int32_t)kw; d.sh = sh; d.sw = sw; d.dh = dh; d.dw = dw;
        }
        // Large calls: build the filter-specialised product table for this call (512 B per weight,
        // one HBM-bound pass) and run the packed-pair kernel; small calls keep the LUT kernel.
        const int64_t ft_bytes = axb_ftable_bytes(kpad, coutp);
        if (n * oh * ow >= 4096 && kpad <= 32768 && fkh * fkw <= 256 && ft_bytes > 0 &&
            ft_bytes <= (int64_t(1) << 30)) {
            if (cudaMallocAsync(&ftable, ft_bytes, s) != cudaSuccess) {
                cudaGetLastError();  // no room: fall back to the LUT kernel
                ftable = nullptr;
            } else {
                rc = axb_ftable_prepare(fcodes, fkh, fkw, fc, fcs, cout, lut, ftable, s);
                d.ftable = ftable;
            }
        }
        d.oh = oh; d.ow = ow;
        d.fcodes = fcodes; d.fsum = fsum; d.cout = cout; d.coutp = coutp; d.kpad = kpad;
        d.in_params = dp; d.f_params = dp + 1;
        d.accumulator = accumulator;
        d.out = d_out;
        d.acc_out = d_acc_out;
        d.flags = flags + 1;
        if (!rc) rc = axb_conv2d_lut(&d, lut, s);
    }
    if (!rc) {  // error precedence as in axconv.py: filters (:287), then inputs (:294)
        int32_t hf[2] = {0, 0};
        cudaMemcpyAsync(hf, flags, 8, cudaMemcpyDeviceToHost, s);
        if (cudaStreamSynchronize(s) != cudaSuccess) fail(AXB_E_CUDA, "stream sync failed");
        else if (hf[0] & AXB_FLAG_NONFINITE) fail(AXB_E_VALUE, "cannot quantize non-finite values");
        else if (hf[0] & AXB_FLAG_FSUM_OVF) fail(AXB_E_OVERFLOW, "filter size too large for 32-bit code sums");
        else if (hf[1] & AXB_FLAG_NONFINITE) fail(AXB_E_VALUE, "cannot quantize non-finite values");
        else if (hf[1] & AXB_FLAG_PSUM_OVF) fail(AXB_E_OVERFLOW, "patch length too large for 32-bit code sums");
    }
    if (ftable) cudaFreeAsync(ftable, s);
    cudaFreeAsync(codes, s);
    cudaFreeAsync(pixsum, s);
    if (rows) cudaFreeAsync(rows, s);
    if (rowsum) cudaFreeAsync(rowsum, s);
    cudaFreeAsync(flags, s);
    cudaFreeAsync(dp, s);
    cudaFreeAsync(fcodes, s);
    cudaFreeAsync(fsum, s);
    return rc;
}

}  // extern "C"
