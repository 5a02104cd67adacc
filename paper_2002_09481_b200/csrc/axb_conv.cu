// K3: approximate convolution as a LUT implicit GEMM with a fused
// correction / dequantize / bias / residual / ReLU / next-layer-range epilogue.
//
// Restates axconv.py:136-146 (_lut_matmul: A[r,c] = sum_k lut[(P[r,k]<<8)|F[c,k]]),
// axconv.py:160-196 (im2cols: zp-padded windows, patch sums -- implicit here),
// axconv.py:246-256 (corr = A - zp2*Sp - zp1*Sf + K*zp1*zp2 in int64,
// out = float32(float64(s1*s2) * corr)), axconv.py:128-133 (accumulator
// emulation) and graph.py:268-277, :282-286 (bias, Add, ReLU).
//
// Fast kernel design (sm_100a, one persistent CTA per SM):
//  * the 128 KiB truth table is staged ONCE per CTA into shared memory by a
//    TMA bulk copy (cp.async.bulk + mbarrier complete_tx), stored b-major:
//    T[b][a] = lut[(a<<8)|b], so the 32 lanes of a warp (32 adjacent output
//    pixels, warp-uniform filter code b) read one 512-byte row: bank =
//    (a>>1) & 31.  Equal codes broadcast; codes within a 64-wide window never
//    conflict (post-ReLU activations cluster near the zero-point).
//  * activation tiles (BM pixels x 16 taps, uint8) and weight tiles (16 taps
//    x BN channels, uint16 = 2*code) stream through a 4-stage cp.async ring
//    straight from the zp-padded NHWC code tensor (implicit im2col);
//  * each lane owns TM=4 pixels x 16 channels of exact int32 accumulators;
//    per lookup: one IMAD (address = a*2 + (b<<9)), one LDS.16, half an IADD3.
//  * K is padded to a multiple of 16 with raw-0 codes on both operands; the
//    padding contributes exactly (kpad-K)*lut[0] which the epilogue removes.
#include "axb_common.cuh"
#include "axb_internal.h"

namespace axb {

constexpr int kMaxTaps = 256;
constexpr int kStages = 4;
constexpr int kThreads = 256;

struct ConvK {
    const uint8_t *codes;
    const int32_t *pixsum;
    int32_t hp, wp, cs, c;
    int32_t kh, kw, sh, sw, dh, dw;
    int32_t oh, ow;
    int64_t M;
    const uint16_t *fcodes;
    const int64_t *fsum;
    int32_t cout, coutp, kpad, nchunks, taps, K;
    const axb_qparams *inp;
    const axb_qparams *fp;
    int32_t acc_mode, relu;
    const float *bias;
    const float *residual;
    float *out;
    int64_t *acc_out;
    int32_t *out_range;
    int32_t *flags;
    const uint16_t *lut;  // b-major
    int32_t f00;          // lut[0] as a value (junk-tap contribution)
    int32_t ntn;
    int64_t ntiles;
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp_async16(void *dst, const void *src, int src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(src_bytes));
}
__device__ __forceinline__ void cp_async4(void *dst, const void *src, int src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ uint32_t sel4(const uint4 &v, int q) {
    return q == 0 ? v.x : (q == 1 ? v.y : (q == 2 ? v.z : v.w));
}

// ---------------------------------------------------------------- epilogue
struct EpiConst {
    double scale;
    int64_t zp1, zp2, kzz, junk;
};

__device__ __forceinline__ EpiConst epi_const(const ConvK &p) {
    EpiConst e;
    e.scale = p.inp->scale * p.fp->scale;  // axconv.py:255 (fp64 product)
    e.zp1 = p.inp->zero_point;
    e.zp2 = p.fp->zero_point;
    e.kzz = (int64_t)p.K * e.zp1 * e.zp2;  // np.int64(depth) * zp1 * zp2
    e.junk = (int64_t)(p.kpad - p.K) * (int64_t)p.f00;
    return e;
}

// patch sum S_p of output pixel m (axconv.py:193), int64, from per-pixel code sums
__device__ __forceinline__ int64_t patch_sum(const ConvK &p, int64_t m, const int32_t *tappix) {
    const int64_t ox = m % p.ow;
    const int64_t t = m / p.ow;
    const int64_t oy = t % p.oh;
    const int64_t b = t / p.oh;
    const int32_t *base = p.pixsum + (b * p.hp + oy * p.sh) * (int64_t)p.wp + ox * p.sw;
    int64_t s = 0;
    for (int i = 0; i < p.taps; ++i) s += base[tappix[i]];
    return s;
}

__device__ __forceinline__ float finish(const ConvK &p, const EpiConst &e, int64_t A, int64_t sp, int64_t m,
                                        int c) {
    const int64_t corr = A - e.zp2 * sp - e.zp1 * p.fsum[c] + e.kzz;  // axconv.py:249-254
    float y = __double2float_rn(e.scale * __ll2double_rn(corr));      // axconv.py:256
    if (p.bias) y = __fadd_rn(y, p.bias[c]);                           // graph.py:268-269
    if (p.residual) y = __fadd_rn(y, p.residual[m * p.cout + c]);      // graph.py:282-286
    if (p.relu) y = (y > 0.0f || y != y) ? y : 0.0f;                  // np.maximum(x, 0.0)
    return y;
}

__device__ __forceinline__ void track(float y, int32_t &tmin, int32_t &tmax, int &nonfinite) {
    nonfinite |= !isfinite(y);
    const int32_t o = f2ord(y);
    tmin = min(tmin, o);
    tmax = max(tmax, o);
}

// ---------------------------------------------------------------- fast kernel
template <int TM, int WM, int WN, bool SGN, int SEG>
__global__ void __launch_bounds__(kThreads, 1) lutconv_fast(const ConvK p) {
    constexpr int BM = WM * 32 * TM;
    constexpr int BN = WN * 16;
    constexpr int ACT_STAGE = BM * 16;
    constexpr int W_STAGE = 16 * BN * 2;
    constexpr int SEGS = 16 / SEG;                  // segments per act row per chunk
    constexpr int NQ = BM * SEGS / kThreads;        // act cp.async per thread per chunk
    static_assert(NQ >= 1 && (BM * SEGS) % kThreads == 0, "tile/thread mismatch");
    static_assert(WM * WN * 32 == kThreads, "8 warps");

    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t *act_s = smem + kLutBytes;
    uint8_t *w_s = act_s + kStages * ACT_STAGE;
    int32_t *tapoff_s = reinterpret_cast<int32_t *>(w_s + kStages * W_STAGE);
    int32_t *tappix_s = tapoff_s + kMaxTaps;
    uint64_t *bar = reinterpret_cast<uint64_t *>(tappix_s + kMaxTaps);

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const int wm = warp % WM;
    const int wn = warp / WM;

    if (tid == 0) mbar_init(bar, 1);
    for (int t = tid; t < p.taps; t += kThreads) {
        const int ky = t / p.kw, kx = t % p.kw;
        const int pix = ky * p.dh * p.wp + kx * p.dw;
        tappix_s[t] = pix;
        tapoff_s[t] = pix * p.cs;
    }
    __syncthreads();
    if (tid == 0) {
        // stage the whole table with 4 TMA bulk copies (32 KiB each)
        mbar_expect_tx(bar, kLutBytes);
#pragma unroll
        for (int q = 0; q < 4; ++q) bulk_g2s(smem + q * 32768, p.lut + q * 16384, 32768, bar);
    }
    bool lut_ready = false;

    const EpiConst e = epi_const(p);
    int32_t tmin = INT32_MAX, tmax = INT32_MIN;
    int nonfinite = 0, psum_ovf = 0;
    const uint32_t lut_base = smem_u32(smem);

    for (int64_t tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
        const int64_t m0 = (tile / p.ntn) * BM;
        const int n0 = (int)(tile % p.ntn) * BN;

        // per-thread gather rows for this tile (pixel base offsets into the code tensor)
        int32_t rowbase[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const int item = tid + q * kThreads;
            const int row = item / SEGS;
            const int64_t m = m0 + row;
            if (m < p.M) {
                const int64_t ox = m % p.ow;
                const int64_t t = m / p.ow;
                const int64_t oy = t % p.oh;
                const int64_t b = t / p.oh;
                rowbase[q] = (int32_t)(((b * p.hp + oy * p.sh) * p.wp + ox * p.sw) * p.cs);
            } else {
                rowbase[q] = -1;
            }
        }

        auto load_stage = [&](int stage, int kc) {
            uint8_t *as = act_s + stage * ACT_STAGE;
            if (SEG == 16) {
                const int k0 = kc * 16;
                const int t = k0 / p.cs;
                const int ci = k0 - t * p.cs;
                const bool tv = t < p.taps;
                const int off = tv ? tapoff_s[t] + ci : 0;
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    const int row = tid + q * kThreads;
                    const bool v = tv && rowbase[q] >= 0;
                    const uint8_t *src = p.codes + (v ? (int64_t)rowbase[q] + off : 0);
                    cp_async16(as + row * 16, src, v ? 16 : 0);
                }
            } else {  // SEG == 4: cs == 4, one tap per 4-byte segment
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    const int item = tid + q * kThreads;
                    const int row = item >> 2, seg = item & 3;
                    const int t = kc * 4 + seg;
                    const bool v = t < p.taps && rowbase[q] >= 0;
                    const uint8_t *src = p.codes + (v ? (int64_t)rowbase[q] + tapoff_s[t] : 0);
                    cp_async4(as + row * 16 + seg * 4, src, v ? 4 : 0);
                }
            }
            if (tid < 2 * BN) {
                uint8_t *ws = w_s + stage * W_STAGE;
                const int r = tid / (BN / 8);
                const int col = (tid % (BN / 8)) * 8;
                const int gcol = n0 + col;
                const bool v = gcol < p.coutp;
                const uint16_t *src = p.fcodes + (v ? (int64_t)(kc * 16 + r) * p.coutp + gcol : 0);
                cp_async16(ws + (r * BN + col) * 2, src, v ? 16 : 0);
            }
        };

        int32_t acc[TM][16];
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < 16; ++j) acc[i][j] = 0;

#pragma unroll
        for (int s = 0; s < kStages - 1; ++s) {
            if (s < p.nchunks) load_stage(s, s);
            cp_async_commit();
        }
        if (!lut_ready) {
            mbar_wait(bar, 0);
            lut_ready = true;
        }

        for (int kc = 0; kc < p.nchunks; ++kc) {
            cp_async_wait<kStages - 2>();
            __syncthreads();
            {
                const int nk = kc + kStages - 1;
                if (nk < p.nchunks) load_stage(nk % kStages, nk);
                cp_async_commit();
            }
            const int stage = kc % kStages;
            const uint8_t *as = act_s + stage * ACT_STAGE;
            const uint8_t *ws = w_s + stage * W_STAGE + wn * 32;
            uint4 av[TM];
#pragma unroll
            for (int i = 0; i < TM; ++i)
                av[i] = *reinterpret_cast<const uint4 *>(as + (wm * 32 * TM + i * 32 + lane) * 16);

#pragma unroll 1
            for (int kp = 0; kp < 8; ++kp) {  // two taps per step: kk = 2kp, 2kp+1
                const int q = kp >> 1;
                const uint32_t s0 = 0x4440u + ((kp & 1) << 1);
                uint32_t a0[TM], a1[TM];
#pragma unroll
                for (int i = 0; i < TM; ++i) {
                    const uint32_t w = sel4(av[i], q);
                    a0[i] = __byte_perm(w, 0, s0);
                    a1[i] = __byte_perm(w, 0, s0 + 1);
                }
                const uint4 w0a = *reinterpret_cast<const uint4 *>(ws + (2 * kp) * BN * 2);
                const uint4 w0b = *reinterpret_cast<const uint4 *>(ws + (2 * kp) * BN * 2 + 16);
                const uint4 w1a = *reinterpret_cast<const uint4 *>(ws + (2 * kp + 1) * BN * 2);
                const uint4 w1b = *reinterpret_cast<const uint4 *>(ws + (2 * kp + 1) * BN * 2 + 16);
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const uint32_t sel = (j & 1) ? 0x4324u : 0x4104u;  // u16 half -> bytes 1..2 (= 2b << 8)
                    const uint32_t b0 =
                        __byte_perm(sel4(j < 8 ? w0a : w0b, (j >> 1) & 3), 0, sel) + lut_base;
                    const uint32_t b1 =
                        __byte_perm(sel4(j < 8 ? w1a : w1b, (j >> 1) & 3), 0, sel) + lut_base;
#pragma unroll
                    for (int i = 0; i < TM; ++i) {
                        int32_t v0, v1;
                        const uint32_t ad0 = a0[i] * 2u + b0;
                        const uint32_t ad1 = a1[i] * 2u + b1;
                        if (SGN) {
                            asm("ld.shared.s16 %0, [%1];" : "=r"(v0) : "r"(ad0));
                            asm("ld.shared.s16 %0, [%1];" : "=r"(v1) : "r"(ad1));
                        } else {
                            asm("ld.shared.u16 %0, [%1];" : "=r"(v0) : "r"(ad0));
                            asm("ld.shared.u16 %0, [%1];" : "=r"(v1) : "r"(ad1));
                        }
                        acc[i][j] += v0 + v1;
                    }
                }
            }
        }
        cp_async_wait<0>();
        __syncthreads();  // stages are free for the next tile's prologue

        // ------------------------------------------------ fused epilogue
#pragma unroll
        for (int i = 0; i < TM; ++i) {
            const int64_t m = m0 + wm * 32 * TM + i * 32 + lane;
            if (m >= p.M) continue;
            const int64_t sp = patch_sum(p, m, tappix_s);
            psum_ovf |= (sp > INT32_MAX || sp < INT32_MIN);
            float y[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int c = n0 + wn * 16 + j;
                if (c < p.cout) {
                    int64_t A;
                    if (p.acc_mode == AXB_ACC_WRAP32) {
                        A = (int64_t)(int32_t)((uint32_t)acc[i][j] - (uint32_t)e.junk);
                    } else {
                        A = (int64_t)acc[i][j] - e.junk;
                        if (p.acc_mode == AXB_ACC_SATURATE32) A = A > INT32_MAX ? INT32_MAX : (A < INT32_MIN ? INT32_MIN : A);
                    }
                    if (p.acc_out) p.acc_out[m * p.cout + c] = A;
                    y[j] = finish(p, e, A, sp, m, c);
                    track(y[j], tmin, tmax, nonfinite);
                }
            }
            const int cb = n0 + wn * 16;
            float *dst = p.out + m * p.cout + cb;
            if (cb + 16 <= p.cout && (p.cout & 3) == 0) {
#pragma unroll
                for (int j = 0; j < 16; j += 4)
                    *reinterpret_cast<float4 *>(dst + j) = make_float4(y[j], y[j + 1], y[j + 2], y[j + 3]);
            } else {
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (cb + j < p.cout) dst[j] = y[j];
            }
        }
    }
    if (!lut_ready) mbar_wait(bar, 0);  // never leave a bulk copy in flight at exit
    range_commit(tmin, tmax, nonfinite, p.out_range, p.flags, AXB_FLAG_OUT_NONFINITE);
    if (psum_ovf) atomicOr(p.flags, AXB_FLAG_PSUM_OVF);
}

// ---------------------------------------------------------------- generic kernel
// One thread per output, exact int64 accumulation over the real taps only;
// used when the fast path's int32 exactness bound (kpad <= 32768) or its
// shape limits do not hold.  LUT read from global (b-major copy).
template <bool SGN>
__global__ void __launch_bounds__(256) lutconv_generic(const ConvK p) {
    __shared__ int32_t tappix_s[kMaxTaps];
    const EpiConst e = epi_const(p);
    int32_t tmin = INT32_MAX, tmax = INT32_MIN;
    int nonfinite = 0, psum_ovf = 0;
    const int64_t total = p.M * p.cout;
    const bool small_taps = p.taps <= kMaxTaps;
    if (small_taps)
        for (int t = threadIdx.x; t < p.taps; t += blockDim.x)
            tappix_s[t] = (t / p.kw) * p.dh * p.wp + (t % p.kw) * p.dw;
    __syncthreads();
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(idx % p.cout);
        const int64_t m = idx / p.cout;
        const int64_t ox = m % p.ow;
        const int64_t tq = m / p.ow;
        const int64_t oy = tq % p.oh;
        const int64_t b = tq / p.oh;
        const int64_t pix0 = (b * p.hp + oy * p.sh) * (int64_t)p.wp + ox * p.sw;
        int64_t A = 0, sp = 0;
        for (int t = 0; t < p.taps; ++t) {
            const int64_t pix = pix0 + (small_taps ? tappix_s[t] : (t / p.kw) * p.dh * p.wp + (t % p.kw) * p.dw);
            const uint8_t *a = p.codes + pix * p.cs;
            const uint16_t *f = p.fcodes + (int64_t)t * p.cs * p.coutp + c;
            for (int ci = 0; ci < p.c; ++ci) {
                const uint32_t idx16 = ((uint32_t)(f[(int64_t)ci * p.coutp] >> 1) << 8) | a[ci];
                const uint16_t raw = __ldg(p.lut + idx16);
                A += SGN ? (int64_t)(int16_t)raw : (int64_t)raw;
            }
            sp += p.pixsum[pix];
        }
        psum_ovf |= (sp > INT32_MAX || sp < INT32_MIN);
        if (p.acc_mode == AXB_ACC_WRAP32)
            A = (int64_t)(int32_t)(uint32_t)(uint64_t)A;  // axconv.py:131-132
        else if (p.acc_mode == AXB_ACC_SATURATE32)
            A = A > INT32_MAX ? INT32_MAX : (A < INT32_MIN ? INT32_MIN : A);  // :133
        if (p.acc_out) p.acc_out[idx] = A;
        const float y = finish(p, e, A, sp, m, c);
        p.out[idx] = y;
        track(y, tmin, tmax, nonfinite);
    }
    range_commit(tmin, tmax, nonfinite, p.out_range, p.flags, AXB_FLAG_OUT_NONFINITE);
    if (psum_ovf) atomicOr(p.flags, AXB_FLAG_PSUM_OVF);
}

// ---------------------------------------------------------------- host launch
template <int TM, int WM, int WN, bool SGN, int SEG>
static int launch_fast(const ConvK &k, int sm_limit, cudaStream_t s, const char *name) {
    constexpr int BM = WM * 32 * TM, BN = WN * 16;
    const size_t smem = kLutBytes + kStages * (BM * 16 + 16 * BN * 2) + 2 * kMaxTaps * 4 + 16;
    auto fn = lutconv_fast<TM, WM, WN, SGN, SEG>;
    static bool configured = false;  // one per instantiation
    if (!configured) {
        if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return set_error(AXB_E_CUDA, "cannot raise dynamic shared memory for lutconv_fast");
        configured = true;
    }
    ConvK kk = k;
    kk.ntn = (k.coutp + BN - 1) / BN;
    kk.ntiles = ((k.M + BM - 1) / BM) * kk.ntn;
    int64_t grid = sm_limit > 0 ? sm_limit : sm_count();
    if (grid > kk.ntiles) grid = kk.ntiles;
    if (grid < 1) grid = 1;
    fn<<<(int)grid, kThreads, smem, s>>>(kk);
    set_last_kernel(name);
    return check_launch("lutconv_fast");
}

template <bool SGN, int SEG>
static int dispatch_tile(const ConvK &k, int sm_limit, cudaStream_t s) {
    if (k.coutp <= 16) return launch_fast<4, 8, 1, SGN, SEG>(k, sm_limit, s, "lutconv_fast<TM4,8x1>");
    if (k.coutp <= 32) return launch_fast<4, 4, 2, SGN, SEG>(k, sm_limit, s, "lutconv_fast<TM4,4x2>");
    return launch_fast<4, 2, 4, SGN, SEG>(k, sm_limit, s, "lutconv_fast<TM4,2x4>");
}

}  // namespace axb

using namespace axb;

extern "C" {

int axb_conv2d_lut(const axb_conv_desc *d, const axb_lut *lut, void *stream) {
    if (!d || !lut) return set_error(AXB_E_VALUE, "null descriptor or table");
    const int64_t M = d->n * d->oh * d->ow;
    if (M == 0 || d->cout == 0) return AXB_OK;
    if (d->kh < 1 || d->kw < 1 || d->sh < 1 || d->sw < 1 || d->dh < 1 || d->dw < 1)
        return set_error(AXB_E_VALUE, "invalid convolution geometry");
    ConvK k{};
    k.codes = d->codes;
    k.pixsum = d->pixsum;
    k.hp = (int32_t)d->hp;
    k.wp = (int32_t)d->wp;
    k.cs = (int32_t)d->cs;
    k.c = (int32_t)d->c;
    k.kh = d->kh; k.kw = d->kw; k.sh = d->sh; k.sw = d->sw; k.dh = d->dh; k.dw = d->dw;
    k.oh = (int32_t)d->oh;
    k.ow = (int32_t)d->ow;
    k.M = M;
    k.fcodes = d->fcodes;
    k.fsum = d->fsum;
    k.cout = (int32_t)d->cout;
    k.coutp = (int32_t)d->coutp;
    k.kpad = (int32_t)d->kpad;
    k.nchunks = (int32_t)(d->kpad / 16);
    k.taps = d->kh * d->kw;
    k.K = (int32_t)(d->kh * d->kw * d->c);
    k.inp = d->in_params;
    k.fp = d->f_params;
    k.acc_mode = d->accumulator;
    k.relu = d->relu;
    k.bias = d->bias;
    k.residual = d->residual;
    k.out = d->out;
    k.acc_out = d->acc_out;
    k.out_range = d->out_range;
    k.flags = d->flags;
    k.lut = lut->d_bmajor;
    k.f00 = lut->f00;
    cudaStream_t s = (cudaStream_t)stream;

    const int64_t code_bytes = d->n * d->hp * d->wp * d->cs;
    const bool fast = !d->force_generic && d->kpad <= 32768 && k.taps <= kMaxTaps &&
                      (d->cs == 4 || d->cs % 16 == 0) && code_bytes < (int64_t(1) << 31) &&
                      d->kpad % 16 == 0 && d->coutp % 16 == 0;
    if (fast) {
        if (lut->is_signed)
            return d->cs == 4 ? dispatch_tile<true, 4>(k, d->sm_limit, s) : dispatch_tile<true, 16>(k, d->sm_limit, s);
        return d->cs == 4 ? dispatch_tile<false, 4>(k, d->sm_limit, s) : dispatch_tile<false, 16>(k, d->sm_limit, s);
    }
    int64_t blocks = (M * d->cout + 255) / 256;
    const int64_t cap = (int64_t)sm_count() * 32;
    if (blocks > cap) blocks = cap;
    if (lut->is_signed)
        lutconv_generic<true><<<(int)blocks, 256, 0, s>>>(k);
    else
        lutconv_generic<false><<<(int)blocks, 256, 0, s>>>(k);
    set_last_kernel("lutconv_generic");
    return check_launch("lutconv_generic");
}

}  // extern "C"
