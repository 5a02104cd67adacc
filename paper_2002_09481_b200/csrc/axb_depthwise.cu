// Depthwise approximate convolution (BASELINE config 5, MobileNet-style).
//
// The reference has no grouped convolution (tensor.py:66-87); its semantics
// here are defined as the per-channel decomposition the SURVEY prescribes:
// channel c of the output equals axconv2d(x[..., c:c+1], f[:, :, c:c+1, :])
// with the SAME in/filter ranges for all channels (axconv.py:266-297), i.e.
//   A[p,c]  = sum_t lut[(a[p,t,c] << 8) | b[t,c]]          (axconv.py:136-146)
//   S_p     = sum_t a[p,t,c] (per channel!), S_f[c] = sum_t b[t,c], K = kh*kw
//   out     = float32(float64(s1*s2) * (A - zp2*S_p - zp1*S_f + K*zp1*zp2))
// then bias / residual / ReLU as in the dense epilogue.
//
// Work per output is only kh*kw lookups, so the kernel is built for memory
// throughput: one thread per (pixel, channel), a warp = 32 consecutive
// channels of one pixel (coalesced code reads and fp32 stores), the b-major
// table staged once per persistent CTA by TMA bulk copy.  Bank conflicts are
// data-dependent (different rows b per lane, bank = (a>>1)&31).
#include <cstdlib>

#include "axb_convk.cuh"

namespace axb {

struct DwK {
    const uint8_t *codes;  // zp-padded (n, hp, wp, cs)
    int64_t n, hp, wp, cs;
    int32_t c, kh, kw, sh, sw, dh, dw;
    int64_t oh, ow;
    const uint8_t *fcodes;  // rows t*16, columns c (raw code bytes)
    const int64_t *fsum;
    int32_t coutp;
    const axb_qparams *inp, *fp;
    int32_t relu;
    const float *bias, *residual;
    float *out;
    int64_t *acc_out;
    int32_t *out_range, *flags;
    const uint16_t *lut;  // b-major
    int32_t sgn;
    const uint32_t *dwtable;  // channel-bank table (axb_depthwise_table_prepare) or null
    int32_t taps;
    FastDiv fd_ow, fd_oh;
};

__device__ __forceinline__ uint32_t dw_smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(1024, 1) depthwise_lut_kernel(const DwK p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + kLutBytes);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(dw_smem_u32(bar)), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(dw_smem_u32(bar)),
                     "r"(kLutBytes)
                     : "memory");
        for (int q = 0; q < 4; ++q)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                    dw_smem_u32(smem + q * 32768)),
                "l"(p.lut + q * 16384), "r"(32768), "r"(dw_smem_u32(bar))
                : "memory");
    }
    asm volatile(
        "{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W_%=;\n}\n" ::"r"(
            dw_smem_u32(bar))
        : "memory");
    const uint16_t *lut_s = reinterpret_cast<const uint16_t *>(smem);

    const double scale = p.inp->scale * p.fp->scale;
    const int64_t zp1 = p.inp->zero_point, zp2 = p.fp->zero_point;
    const int K = p.kh * p.kw;
    const int64_t kzz = (int64_t)K * zp1 * zp2;
    float tmin = INFINITY, tmax = -INFINITY;
    int nonfinite = 0;
    const int64_t total = p.n * p.oh * p.ow * p.c;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(idx % p.c);
        const int64_t m = idx / p.c;
        const int64_t ox = m % p.ow;
        const int64_t t1 = m / p.ow;
        const int64_t oy = t1 % p.oh;
        const int64_t b = t1 / p.oh;
        const uint8_t *base = p.codes + ((b * p.hp + oy * p.sh) * p.wp + ox * p.sw) * p.cs + c;
        int32_t A = 0, sp = 0;
        for (int ky = 0; ky < p.kh; ++ky)
            for (int kx = 0; kx < p.kw; ++kx) {
                const int t = ky * p.kw + kx;
                const uint32_t a = __ldg(base + ((int64_t)ky * p.dh * p.wp + kx * p.dw) * p.cs);
                const uint32_t bc = __ldg(p.fcodes + (int64_t)t * 16 * p.coutp + c);
                const uint16_t raw = lut_s[(bc << 8) | a];
                A += p.sgn ? (int32_t)(int16_t)raw : (int32_t)raw;
                sp += p.sgn ? (int32_t)(int8_t)a : (int32_t)a;
            }
        if (p.acc_out) p.acc_out[idx] = A;
        const int64_t corr = (int64_t)A - zp2 * sp - zp1 * p.fsum[c] + kzz;
        float y = __double2float_rn(scale * __ll2double_rn(corr));
        if (p.bias) y = __fadd_rn(y, p.bias[c]);
        if (p.residual) y = __fadd_rn(y, p.residual[idx]);
        if (p.relu) y = (y > 0.0f || y != y) ? y : 0.0f;
        p.out[idx] = y;
        nonfinite |= !(fabsf(y) <= 3.402823466e38f);
        tmin = fminf(tmin, y);
        tmax = fmaxf(tmax, y);
    }
    const bool any = tmin <= tmax;
    range_commit(any ? f2ord(tmin) : INT32_MAX, any ? f2ord(tmax) : INT32_MIN, nonfinite, p.out_range, p.flags,
                 AXB_FLAG_OUT_NONFINITE);
}

// ---------------------------------------------------------------- channel-bank table kernel
// The filter codes of a depthwise layer are constants, so for each tap t and channel c only the 256
// products lut[(a<<8) | b(t,c)] can occur.  They are laid out per 32-channel block cb as
//     DW[cb][t][a >> 1][lane] = u(lut[(a_even<<8)|b]) | u(lut[(a_odd<<8)|b]) << 16,   lane = c % 32
// (u = raw ^ 0x8000 for signed tables, raw for unsigned): 16 KiB per tap and block, 144 KiB for 3x3.
// A warp = one output pixel x 32 channels, lane = channel; lane L always reads bank L, so every
// LDS.32 is one wavefront (32 lookups) whatever the activation codes -- the b-major LUT the old
// kernel reads conflicts on (a >> 1) & 31 across the 32 channels' codes.  The wanted half of the word
// is picked with one PRMT whose selector comes from a & 1.  Persistent CTAs (one per SM) take
// contiguous ranges of the (channel block, pixel) index space, so each CTA stages one or two
// blocks' tables with TMA bulk copies; codes are read straight from the zp-padded NHWC code tensor
// (32 contiguous bytes per warp and tap), outputs stored 128 B per warp.
constexpr int kDwMaxTaps = 13;
constexpr int kDwTapBytes = 128 * 32 * 4;  // 16 KiB

__device__ __forceinline__ uint32_t dw_bias_word(int sgn) { return sgn ? 0x80008000u : 0u; }

__global__ void dwtable_kernel(const uint8_t *__restrict__ fcodes, int taps, int c, int coutp,
                               const uint16_t *__restrict__ lut_b, int sgn, uint32_t *__restrict__ out) {
    const int nb = (c + 31) / 32;
    const int64_t total = (int64_t)nb * taps * 128 * 32;
    const uint32_t flip = sgn ? 0x8000u : 0u;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int lane = (int)(i & 31);
        const int a2 = (int)((i >> 5) & 127);
        const int64_t r = i >> 12;
        const int t = (int)(r % taps);
        const int cb = (int)(r / taps);
        const int ch = cb * 32 + lane;
        uint32_t w = dw_bias_word(sgn);  // zero contribution (junk channels are never stored)
        if (ch < c) {
            const uint32_t b = fcodes[(int64_t)t * 16 * coutp + ch];  // (kh, kw, 1, c) view, cs 16
            w = ((uint32_t)__ldg(lut_b + b * 256 + 2 * a2) ^ flip) |
                (((uint32_t)__ldg(lut_b + b * 256 + 2 * a2 + 1) ^ flip) << 16);
        }
        out[i] = w;
    }
}

template <int NW, int T>
__global__ void __launch_bounds__(NW * 32, 1) depthwise_ct_kernel(const DwK p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int taps = T > 0 ? T : p.taps;
    uint32_t *tab = reinterpret_cast<uint32_t *>(smem);
    int32_t *tapoff = reinterpret_cast<int32_t *>(smem + kDwMaxTaps * kDwTapBytes);
    uint64_t *bar = reinterpret_cast<uint64_t *>(tapoff + 16);
    const int tid = (int)threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) mbar_init(bar, 1);
    if (tid < taps) tapoff[tid] = (int32_t)((((tid / p.kw) * p.dh) * p.wp + (tid % p.kw) * p.dw) * p.cs);
    __syncthreads();

    const double scale = p.inp->scale * p.fp->scale;
    const int64_t zp1 = p.inp->zero_point, zp2 = p.fp->zero_point;
    const int32_t kzz = (int32_t)(taps * zp1 * zp2);  // |.| <= 13 * 255 * 255
    const int32_t ubias = p.sgn ? 32768 * taps : 0;
    const int nb = (p.c + 31) / 32;
    const int64_t M = p.n * p.oh * p.ow;
    const int64_t total = (int64_t)nb * M;
    const int64_t lo = total * blockIdx.x / gridDim.x, hi = total * (blockIdx.x + 1) / gridDim.x;
    float tmin = INFINITY, tmax = -INFINITY;
    int nonfinite = 0;
    uint32_t phase = 0;
    const uint8_t *tab_lane = smem + lane * 4;
    for (int cb = lo < hi ? (int)(lo / M) : nb; cb < nb && (int64_t)cb * M < hi; ++cb) {
        const int64_t s0 = max(lo, (int64_t)cb * M), s1 = min(hi, (int64_t)(cb + 1) * M);
        // stage block cb's table; every thread's generic reads of the previous one precede the TMA write
        fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0) {
            const uint32_t bytes = (uint32_t)taps * kDwTapBytes;
            mbar_expect_tx(bar, bytes);
            bulk_g2s(smem, p.dwtable + (int64_t)cb * taps * (kDwTapBytes / 4), bytes, bar);
        }
        mbar_wait(bar, phase);
        phase ^= 1u;
        const int ch = cb * 32 + lane;
        const int chl = min(ch, p.c - 1);  // junk lanes of the last block read a real byte, store nothing
        const int64_t fs = p.fsum[chl];
        const float bias = p.bias ? __ldg(p.bias + chl) : 0.0f;
        int32_t toff[T > 0 ? T : 1];
#pragma unroll
        for (int t = 0; t < T; ++t) toff[t] = tapoff[t];
        // two pixels per warp iteration (independent loads in flight); 32-bit coordinates (M < 2^31)
        const uint32_t e = (uint32_t)(s1 - (int64_t)cb * M);
        for (uint32_t m0 = (uint32_t)(s0 - (int64_t)cb * M) + 2u * warp; m0 < e; m0 += 2u * NW) {
            const uint8_t *src[2];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const uint32_t m = min(m0 + q, e - 1);
                const uint32_t t1 = fdiv(m, p.fd_ow);
                const uint32_t ox = m - t1 * (uint32_t)p.ow;
                const uint32_t b = fdiv(t1, p.fd_oh);
                const uint32_t oy = t1 - b * (uint32_t)p.oh;
                src[q] = p.codes + (((int64_t)b * p.hp + oy * p.sh) * p.wp + (int64_t)ox * p.sw) * p.cs + chl;
            }
            uint32_t A[2] = {0, 0};
            int32_t sp[2] = {0, 0};
#pragma unroll
            for (int t = 0; t < (T > 0 ? T : kDwMaxTaps); ++t) {
                if (T == 0 && t >= taps) break;
                const int32_t off = T > 0 ? toff[t] : tapoff[t];
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const uint32_t a = __ldg(src[q] + off);
                    const uint32_t w =
                        *reinterpret_cast<const uint32_t *>(tab_lane + t * kDwTapBytes + (a >> 1) * 128u);
                    A[q] += __byte_perm(w, 0, 0x4410u + (a & 1u) * 0x22u);  // the entry of code a
                    sp[q] += p.sgn ? (int32_t)(int8_t)a : (int32_t)a;
                }
            }
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                if (ch < p.c && m0 + q < e) {
                    const int32_t Ai = (int32_t)A[q] - ubias;  // exact: |A| <= 13 * 32768
                    const int64_t o = (int64_t)(m0 + q) * p.c + ch;
                    if (p.acc_out) p.acc_out[o] = Ai;
                    const int64_t corr = (int64_t)Ai - zp2 * sp[q] - zp1 * fs + kzz;  // axconv.py:249-254
                    float y = __double2float_rn(scale * __ll2double_rn(corr));        // axconv.py:256
                    if (p.bias) y = __fadd_rn(y, bias);                               // graph.py:268-269
                    if (p.residual) y = __fadd_rn(y, __ldg(p.residual + o));          // graph.py:282-286
                    if (p.relu) y = (y > 0.0f || y != y) ? y : 0.0f;                  // graph.py:276-277
                    p.out[o] = y;
                    track(y, tmin, tmax, nonfinite);
                }
            }
        }
    }
    const bool any = tmin <= tmax;
    range_commit(any ? f2ord(tmin) : INT32_MAX, any ? f2ord(tmax) : INT32_MIN, nonfinite, p.out_range, p.flags,
                 AXB_FLAG_OUT_NONFINITE);
}

// ---------------------------------------------------------------- row-strip kernel (3x3, dilation 1)
// Same channel-bank table and arithmetic as depthwise_ct_kernel, reorganised for memory-level parallelism
// and reuse: a warp owns R output rows x P consecutive output pixels x 32 channels (lane = channel).  The
// unit's NR x NC input codes (NR = R + 2 rows at stride 1 -- R = 2 shares two of the three input rows
// between the two output rows -- NC = (P-1)*SW + 3 columns, 32 channels each) are copied into the
// warp's shared buffer with 16-byte cp.async, the next unit's while this one computes (~1.3 KB in
// flight per warp instead of one 32-byte load per tap).  Each code is read once from there; its table
// address and half-word selector are derived once and reused by every tap of every output row that
// reads it (up to 6 at stride 1); S_p = sums of per-column code sums.  R * P independent chains.
template <int SW, int P, int R>
__host__ __device__ constexpr int dw_rs_nr() { return R + 2; }  // input rows per unit (R > 1: stride 1)
template <int SW, int P, int R>
__host__ __device__ constexpr int dw_rs_strip_bytes() { return dw_rs_nr<SW, P, R>() * ((P - 1) * SW + 3) * 32; }
template <int SW, int P, int R, int NW>
__host__ __device__ constexpr int dw_rs_smem() { return 9 * kDwTapBytes + NW * 2 * dw_rs_strip_bytes<SW, P, R>() + 16; }

template <int SW, int P, int R, int NW>
__global__ void __launch_bounds__(NW * 32, 1) depthwise_rs_kernel(const DwK p, FastDiv fd_ns, int32_t nstrips,
                                                                  FastDiv fd_ohr, int32_t ohr) {
    constexpr int KH = 3, KW = 3;
    constexpr int NC = (P - 1) * SW + KW;  // input columns per kernel row
    constexpr int NR = dw_rs_nr<SW, P, R>();
    constexpr int SB = dw_rs_strip_bytes<SW, P, R>();
    constexpr int NCH = NR * NC * 2;       // 16-byte chunks per unit
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t *wbuf = smem + KH * KW * kDwTapBytes + (threadIdx.x >> 5) * 2 * SB;  // this warp's two buffers
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + KH * KW * kDwTapBytes + NW * 2 * SB);
    const int tid = (int)threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) mbar_init(bar, 1);
    __syncthreads();

    const double scale = p.inp->scale * p.fp->scale;
    const int32_t zp1 = p.inp->zero_point, zp2 = p.fp->zero_point;
    const int32_t ubias = p.sgn ? 32768 * KH * KW : 0;
    const int nb = (p.c + 31) / 32;
    const uint32_t U = (uint32_t)(p.n * ohr) * (uint32_t)nstrips;  // units per channel block (< 2^31)
    const int64_t total = (int64_t)nb * U;
    const int64_t lo = total * blockIdx.x / gridDim.x, hi = total * (blockIdx.x + 1) / gridDim.x;
    const bool has_res = p.residual != nullptr, relu = p.relu != 0, has_acc = p.acc_out != nullptr;
    float tmin = INFINITY, tmax = -INFINITY;
    int nonfinite = 0;
    uint32_t phase = 0;
    const uint8_t *tab_lane = smem + lane * 4;
    // unit u -> image b, first output row oy0, strip
    auto unit = [&](uint32_t u, uint32_t &b, uint32_t &oy0, uint32_t &strip) {
        const uint32_t t1 = fdiv(u, fd_ns);
        strip = u - t1 * (uint32_t)nstrips;
        b = fdiv(t1, fd_ohr);
        oy0 = (t1 - b * (uint32_t)ohr) * R;
    };
    for (int cb = lo < hi ? (int)(lo / U) : nb; cb < nb && (int64_t)cb * U < hi; ++cb) {
        const uint32_t u0 = (uint32_t)(max(lo, (int64_t)cb * U) - (int64_t)cb * U);
        const uint32_t u1 = (uint32_t)(min(hi, (int64_t)(cb + 1) * U) - (int64_t)cb * U);
        // unit u's codes -> buffer `buf`: chunk j = (input row r, column i, half h) of 16 channels
        auto fetch = [&](uint32_t u, int buf) {
            uint32_t b, oy0, strip;
            unit(u, b, oy0, strip);
            const int col0 = (int)strip * P * SW;
#pragma unroll
            for (int j0 = 0; j0 < NCH; j0 += 32) {
                const int j = j0 + lane;
                if (j0 + 32 <= NCH || j < NCH) {
                    const int h = j & 1, i = (j >> 1) % NC, r = (j >> 1) / NC;
                    const int col = min(col0 + i, (int)p.wp - 1);  // columns past the row: junk outputs only
                    const int row = min((int)oy0 * p.sh + r, (int)p.hp - 1);  // rows past the image: junk too
                    const int chan = cb * 32 + h * 16;
                    const uint8_t *src = p.codes + (((int64_t)b * p.hp + row) * p.wp + col) * p.cs +
                                         min(chan, (int)p.cs - 16);
                    cp_async16(wbuf + buf * SB + (r * NC + i) * 32 + h * 16, src, chan < p.cs ? 16 : 0);
                }
            }
            cp_async_commit();
        };
        fence_proxy_async_smem();  // every thread's reads of the previous block's table precede the TMA write
        __syncthreads();
        if (tid == 0) {
            mbar_expect_tx(bar, KH * KW * kDwTapBytes);
            bulk_g2s(smem, p.dwtable + (int64_t)cb * KH * KW * (kDwTapBytes / 4), KH * KW * kDwTapBytes, bar);
        }
        const int ch = cb * 32 + lane;
        const int chl = min(ch, p.c - 1);
        // per-channel terms: -zp1*S_f + K*zp1*zp2 - (entry bias); bias (-0.0f when absent: exact identity)
        const int32_t cc = (int32_t)(KH * KW * zp1 * zp2 - zp1 * (int32_t)p.fsum[chl]) - ubias;
        const float bias = p.bias ? __ldg(p.bias + chl) : -0.0f;
        int buf = 0;
        if (u0 + warp < u1) fetch(u0 + warp, 0);
        mbar_wait(bar, phase);
        phase ^= 1u;
        for (uint32_t u = u0 + warp; u < u1; u += NW) {
            if (u + NW < u1) fetch(u + NW, buf ^ 1);
            else cp_async_commit();
            cp_async_wait<1>();
            __syncwarp();
            uint32_t b, oy0, strip;
            unit(u, b, oy0, strip);
            const int ox0 = (int)strip * P;
            const uint8_t *cbuf = wbuf + buf * SB + lane;
            uint32_t A[R][P];
            int32_t colsum[R][NC];  // per output row and input column: sum of its 3 taps' codes
#pragma unroll
            for (int r = 0; r < R; ++r) {
#pragma unroll
                for (int q = 0; q < P; ++q) A[r][q] = 0;
#pragma unroll
                for (int i = 0; i < NC; ++i) colsum[r][i] = 0;
            }
#pragma unroll
            for (int ir = 0; ir < NR; ++ir) {
#pragma unroll
                for (int i = 0; i < NC; ++i) {
                    const uint32_t code = cbuf[(ir * NC + i) * 32];
                    const uint8_t *base = tab_lane + (code >> 1) * 128u;
                    const uint32_t sel = 0x4410u + (code & 1u) * 0x22u;
                    const int32_t cv = p.sgn ? (int32_t)(int8_t)code : (int32_t)code;
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const int ky = ir - r;  // kernel row of input row ir for output row r (stride 1 if R > 1)
                        if (ky < 0 || ky >= KH) continue;
                        colsum[r][i] += cv;
#pragma unroll
                        for (int kx = 0; kx < KW; ++kx) {
                            const int q = (i - kx) / SW;  // output pixel reading column i at tap kx
                            if (i - kx >= 0 && (i - kx) % SW == 0 && q < P) {
                                const uint32_t w = *reinterpret_cast<const uint32_t *>(
                                    base + (ky * KW + kx) * kDwTapBytes);
                                A[r][q] += __byte_perm(w, 0, sel);  // the entry of this code (axconv.py:136-146)
                            }
                        }
                    }
                }
            }
            __syncwarp();  // every lane read the buffer before the fetch two units on overwrites it
            buf ^= 1;
            const int nq = min(P, (int)p.ow - ox0);  // pixels of the strip inside the row
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int oy = (int)oy0 + r;
                if (ch >= p.c || oy >= (int)p.oh) continue;
                const int64_t o0 = (((int64_t)b * p.oh + oy) * p.ow + ox0) * p.c + ch;  // output (oy, ox0, ch)
#pragma unroll
                for (int q = 0; q < P; ++q) {
                    if (q < nq) {
                        const int32_t Ai = (int32_t)A[r][q];  // exact: |A - ubias| <= 9 * 32768
                        const int32_t sp = colsum[r][q * SW] + colsum[r][q * SW + 1] + colsum[r][q * SW + 2];
                        const int64_t o = o0 + (int64_t)q * p.c;
                        // corr = A - zp2*S_p - zp1*S_f + K*zp1*zp2 (axconv.py:249-254), exact in int32 here
                        const int32_t corr = Ai - zp2 * sp + cc;
                        float y = __fadd_rn(__double2float_rn(scale * (double)corr), bias);  // :256; graph.py:268-269
                        if (has_res) y = __fadd_rn(y, __ldg(p.residual + o));               // graph.py:282-286
                        if (relu) y = (y > 0.0f || y != y) ? y : 0.0f;                      // graph.py:276-277
                        p.out[o] = y;
                        track(y, tmin, tmax, nonfinite);
                        if (has_acc) p.acc_out[o] = Ai - ubias;
                    }
                }
            }
        }
        cp_async_wait<0>();
    }
    const bool any = tmin <= tmax;
    range_commit(any ? f2ord(tmin) : INT32_MAX, any ? f2ord(tmax) : INT32_MIN, nonfinite, p.out_range, p.flags,
                 AXB_FLAG_OUT_NONFINITE);
}

}  // namespace axb

using namespace axb;

static bool dw_rs_enabled() {
    static const int on = [] {
        const char *e = getenv("AXB_DW_RS");
        return (e && e[0] == '0') ? 0 : 1;
    }();
    return on != 0;
}

extern "C" int64_t axb_depthwise_table_bytes(int64_t kh, int64_t kw, int64_t c) {
    if (kh < 1 || kw < 1 || c < 1 || kh * kw > kDwMaxTaps) return 0;
    return ((c + 31) / 32) * kh * kw * (int64_t)kDwTapBytes;
}

extern "C" int axb_depthwise_table_prepare(const uint8_t *d_fcodes, int64_t kh, int64_t kw, int64_t c, int64_t coutp,
                                           const axb_lut *lut, uint32_t *d_table, void *stream) {
    if (!d_fcodes || !lut || !d_table) return set_error(AXB_E_VALUE, "null argument");
    if (axb_depthwise_table_bytes(kh, kw, c) == 0) return set_error(AXB_E_VALUE, "depthwise table: unsupported shape");
    const int64_t words = axb_depthwise_table_bytes(kh, kw, c) / 4;
    int64_t blocks = (words + 255) / 256;
    if (blocks > (int64_t)sm_count() * 8) blocks = sm_count() * 8;
    dwtable_kernel<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(d_fcodes, (int)(kh * kw), (int)c, (int)coutp,
                                                                   lut->d_bmajor, lut->is_signed, d_table);
    return check_launch("depthwise_table_prepare");
}

extern "C" int axb_depthwise_lut(const axb_conv_desc *d, const axb_lut *lut, void *stream) {
    if (!d || !lut) return set_error(AXB_E_VALUE, "null descriptor or table");
    if (d->cout != d->c) return set_error(AXB_E_VALUE, "depthwise conv needs cout == channels");
    if (d->kh * d->kw > 256) return set_error(AXB_E_VALUE, "depthwise kernel too large");
    const int64_t total = d->n * d->oh * d->ow * d->c;
    if (total == 0) return AXB_OK;
    DwK k{};
    k.codes = d->codes;
    k.n = d->n; k.hp = d->hp; k.wp = d->wp; k.cs = d->cs;
    k.c = (int32_t)d->c; k.kh = d->kh; k.kw = d->kw; k.sh = d->sh; k.sw = d->sw; k.dh = d->dh; k.dw = d->dw;
    k.oh = d->oh; k.ow = d->ow;
    k.fcodes = d->fcodes; k.fsum = d->fsum; k.coutp = (int32_t)d->coutp;
    k.inp = d->in_params; k.fp = d->f_params;
    k.relu = d->relu; k.bias = d->bias; k.residual = d->residual; k.out = d->out; k.acc_out = d->acc_out;
    k.out_range = d->out_range; k.flags = d->flags;
    k.lut = lut->d_bmajor;
    k.sgn = lut->is_signed;
    k.taps = d->kh * d->kw;
    if (d->ftable && d->variant != 1 && k.taps == 9 && d->kh == 3 && d->dh == 1 && d->dw == 1 &&
        ((d->sw == 1 && d->sh == 1) || d->sw == 2) &&
        d->n * d->oh * d->ow < ((int64_t)1 << 31) && dw_rs_enabled()) {
        // row-strip kernel: 2 rows x 8 pixels per warp unit at stride 1, 1 row x 8 pixels at stride 2
        constexpr int NW = 16, P = 8;
        k.dwtable = reinterpret_cast<const uint32_t *>(d->ftable);
        k.fd_oh = make_fastdiv((uint32_t)d->oh);
        const bool s1 = d->sw == 1 && d->sh == 1;
        const int rows = s1 ? 2 : 1;
        const int32_t nstrips = (int32_t)((d->ow + P - 1) / P);
        const int32_t ohr = (int32_t)((d->oh + rows - 1) / rows);
        const int64_t units = ((d->c + 31) / 32) * d->n * ohr * nstrips;
        if (d->n * ohr * nstrips >= ((int64_t)1 << 31)) return set_error(AXB_E_VALUE, "depthwise conv too large");
        const size_t smem = s1 ? dw_rs_smem<1, P, 2, NW>() : dw_rs_smem<2, P, 1, NW>();
        auto fn = s1 ? depthwise_rs_kernel<1, P, 2, NW> : depthwise_rs_kernel<2, P, 1, NW>;
        static int configured[2] = {-1, -1};
        int dev = 0;
        cudaGetDevice(&dev);
        const int which = s1;
        if (configured[which] != dev) {
            if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
                return set_error(AXB_E_CUDA, "cannot raise dynamic shared memory for depthwise_rs_kernel");
            configured[which] = dev;
        }
        int64_t grid = sm_count();
        if (grid > (units + NW - 1) / NW) grid = (units + NW - 1) / NW;
        if (grid < 1) grid = 1;
        fn<<<(int)grid, NW * 32, smem, (cudaStream_t)stream>>>(k, make_fastdiv((uint32_t)nstrips), nstrips,
                                                               make_fastdiv((uint32_t)ohr), ohr);
        set_last_kernel("depthwise_rs");
        return check_launch("depthwise_rs");
    }
    if (d->ftable) {  // channel-bank table kernel (axb_depthwise_table_prepare)
        if (k.taps > kDwMaxTaps) return set_error(AXB_E_VALUE, "depthwise table kernel: more than 13 taps");
        k.dwtable = reinterpret_cast<const uint32_t *>(d->ftable);
        if (d->n * d->oh * d->ow >= ((int64_t)1 << 31)) return set_error(AXB_E_VALUE, "depthwise conv too large");
        k.fd_ow = make_fastdiv((uint32_t)d->ow);
        k.fd_oh = make_fastdiv((uint32_t)d->oh);
        constexpr int NW = 16;
        const size_t smem = kDwMaxTaps * kDwTapBytes + 16 * 4 + 16;
        auto fn = k.taps == 9 ? depthwise_ct_kernel<NW, 9> : depthwise_ct_kernel<NW, 0>;
        static int configured[2] = {-1, -1};
        int dev = 0;
        cudaGetDevice(&dev);
        const int which = k.taps == 9;
        if (configured[which] != dev) {
            if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
                return set_error(AXB_E_CUDA, "cannot raise dynamic shared memory for depthwise_ct_kernel");
            configured[which] = dev;
        }
        const int64_t units = ((d->c + 31) / 32) * d->n * d->oh * d->ow;
        int64_t grid = sm_count();
        if (grid > (units + NW - 1) / NW) grid = (units + NW - 1) / NW;
        if (grid < 1) grid = 1;
        fn<<<(int)grid, NW * 32, smem, (cudaStream_t)stream>>>(k);
        set_last_kernel("depthwise_ct");
        return check_launch("depthwise_ct");
    }
    const size_t smem = kLutBytes + 16;
    static int configured_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (configured_dev != dev) {
        if (cudaFuncSetAttribute(depthwise_lut_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess)
            return set_error(AXB_E_CUDA, "cannot raise dynamic shared memory for depthwise_lut_kernel");
        configured_dev = dev;
    }
    int64_t grid = (total + 1023) / 1024;
    if (grid > sm_count()) grid = sm_count();
    depthwise_lut_kernel<<<(int)grid, 1024, smem, (cudaStream_t)stream>>>(k);
    set_last_kernel("depthwise_lut");
    return check_launch("depthwise_lut");
}
