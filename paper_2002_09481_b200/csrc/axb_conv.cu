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
#include "axb_convk.cuh"

namespace axb {

constexpr int kSmemBudget = 232448;  // 227 KiB opt-in dynamic shared memory per CTA
constexpr int kChunkGroup = 2;       // 16-tap sub-chunks consumed per barrier period

// bytes of shared memory besides the activation/weight rings: LUT, tap tables,
// mbarrier, range_commit's static scratch (512), and per warp group the 2 x BN
// epilogue constants (int64 + float)
__host__ __device__ constexpr int fixed_smem(int BN, int NGRP) {
    return kLutBytes + 2 * kMaxTaps * 4 + 32 + 512 + NGRP * 2 * BN * 12;
}
__host__ __device__ constexpr int ring_fit(int BM, int BN, int NGRP) {
    return (kSmemBudget - fixed_smem(BN, NGRP)) / (NGRP * kChunkGroup * (BM * 16 + 16 * BN));
}
// ring depth per warp group in groups of kChunkGroup sub-chunks (4 when it fits, at least 2)
__host__ __device__ constexpr int ring_groups(int BM, int BN, int NGRP) {
    return ring_fit(BM, BN, NGRP) >= 4 ? 4 : (ring_fit(BM, BN, NGRP) >= 3 ? 3 : 2);
}
__host__ __device__ constexpr int group_smem(int BM, int BN, int NGRP) {
    return ring_groups(BM, BN, NGRP) * kChunkGroup * (BM * 16 + 16 * BN) + 2 * BN * 12;
}
__host__ __device__ constexpr int fast_smem(int BM, int BN, int NGRP) {
    return kLutBytes + 2 * kMaxTaps * 4 + 32 + 512 + NGRP * group_smem(BM, BN, NGRP);
}

// ---------------------------------------------------------------- fast kernel
// Persistent CTA (one per SM, the LUT takes 128 KiB of its shared memory).
// The CTA walks its tiles (tile = blockIdx.x + j*gridDim.x) and their 16-tap
// sub-chunks as ONE continuous stream, so the cp.async ring keeps prefetching
// the next tile's first sub-chunks while the current tile finishes and runs
// its epilogue (no per-tile pipeline fill / drain).  The stream is consumed in
// groups of kChunkGroup sub-chunks per barrier period (one cp.async wait +
// barrier + one producer step per group), through a ring of NG groups.
// NGRP > 1: the CTA runs NGRP independent warp groups (each its own tile stream,
// ring and named barrier) sharing the one staged table, so one group's
// epilogue / barrier / producer phases overlap the other groups' lookups.
template <int TM, int TN, int WM, int WN, bool SGN, int NGRP>
__global__ void __launch_bounds__(NGRP *WM *WN * 32, 1) lutconv_fast(const ConvK p) {
    constexpr int NT = WM * WN * 32;  // threads per warp group
    constexpr int BM = WM * 32 * TM;
    constexpr int BN = WN * TN;
    constexpr int ACT_STAGE = BM * 16;
    constexpr int W_STAGE = 16 * BN;  // 16 taps x BN channels, raw code bytes
    constexpr int G = kChunkGroup;
    constexpr int NG = ring_groups(BM, BN, NGRP);
    constexpr int SLOTS = G * NG;
    static_assert(fast_smem(BM, BN, NGRP) <= kSmemBudget, "tile variant exceeds shared memory");
    constexpr int NQ = (BM + NT - 1) / NT;  // activation rows per thread per chunk (one 16-byte cp.async each)
    static_assert(BM % NT == 0 || NT % BM == 0, "tile/thread mismatch");  // BM < NT: threads >= BM load none
    static_assert(BN <= NT, "one weight piece per thread");
    static_assert(TN % 8 == 0, "TN multiple of 8");

    extern __shared__ __align__(1024) uint8_t smem[];
    int32_t *tapoff_s = reinterpret_cast<int32_t *>(smem + kLutBytes);
    int32_t *tappix_s = tapoff_s + kMaxTaps;
    uint64_t *bar = reinterpret_cast<uint64_t *>(tappix_s + kMaxTaps);
    const int grp = NGRP > 1 ? (int)(threadIdx.x / NT) : 0;
    uint8_t *gbase = reinterpret_cast<uint8_t *>(bar) + 32 + grp * group_smem(BM, BN, NGRP);
    uint8_t *act_s = gbase;
    uint8_t *w_s = act_s + SLOTS * ACT_STAGE;
    int64_t *ep_cc_s = reinterpret_cast<int64_t *>(w_s + SLOTS * W_STAGE);  // 2 x BN per-channel constants
    float *ep_bias_s = reinterpret_cast<float *>(ep_cc_s + 2 * BN);          // 2 x BN (by tile parity)

    const int tid = (int)threadIdx.x - grp * NT;  // thread index within the warp group
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const int wm = warp % WM;
    const int wn = warp / WM;
    // this group's place in the virtual grid of NGRP * gridDim.x tile streams
    const int64_t vb = (int64_t)blockIdx.x * NGRP + grp;
    const int64_t vg = (int64_t)gridDim.x * NGRP;
    auto group_sync = [&]() {
        if constexpr (NGRP == 1)
            __syncthreads();
        else
            asm volatile("bar.sync %0, %1;\n" ::"r"(1 + grp), "n"(NT) : "memory");
    };

    if (threadIdx.x == 0) mbar_init(bar, 1);
    for (int t = threadIdx.x; t < p.taps; t += NGRP * NT) {
        const int ky = t / p.kw, kx = t % p.kw;
        const int pix = ky * p.dh * p.wp + kx * p.dw;
        tappix_s[t] = pix;
        tapoff_s[t] = pix * p.cs;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        // the whole 128 KiB table in 4 TMA bulk copies (32 KiB each), completion on one mbarrier
        mbar_expect_tx(bar, kLutBytes);
#pragma unroll
        for (int q = 0; q < 4; ++q) bulk_g2s(smem + q * 32768, p.lut + q * 16384, 32768, bar);
    }

    float tmin = INFINITY, tmax = -INFINITY;
    int nonfinite = 0, psum_ovf = 0;
    const uint32_t lut_base = smem_u32(smem);

    const int64_t my_tiles = p.ntiles > vb ? (p.ntiles - vb + vg - 1) / vg : 0;
    const int64_t total = my_tiles * p.nchunks;

    // ---- producer state (runs NG-1 groups ahead of the consumer)
    int64_t ld_it = 0;
    int ld_kc = 0;
    int ld_t = 0, ld_ci = 0;  // tap and channel offset of chunk ld_kc (cs % 16 == 0)
    int64_t ld_tile = vb;
    int ld_n0 = 0;
    int32_t rowbase[NQ];
    auto set_load_tile = [&](int64_t tile) {
        const int64_t m0 = (tile / p.ntn) * BM;
        ld_n0 = (int)(tile % p.ntn) * BN;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const int64_t mt = m0 + tid + q * NT;
            if ((BM >= NT || tid < BM) && mt < p.M) {
                int64_t pix0;
                pixel_of(p, mt, pix0);
                rowbase[q] = (int32_t)(pix0 * p.cs);
            } else {
                rowbase[q] = -1;
            }
        }
    };
    set_load_tile(ld_tile);
    auto load_next = [&]() {
        if (ld_it < total) {
            const int stage = (int)(ld_it % SLOTS);
            uint8_t *as = act_s + stage * ACT_STAGE;
            const int k0 = ld_kc * 16;
            const bool tv = ld_t < p.taps;
            const int off = tv ? tapoff_s[ld_t] + ld_ci : 0;
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                if (BM < NT && tid >= BM) break;
                const bool v = tv && rowbase[q] >= 0;
                const uint8_t *src = p.codes + (v ? (int64_t)rowbase[q] + off : 0);
                cp_async16(as + (tid + q * NT) * 16, src, v ? 16 : 0);
            }
            if (tid < BN) {  // 16 taps x BN bytes = BN 16-byte pieces
                uint8_t *ws = w_s + stage * W_STAGE;
                const int r = tid / (BN / 16);
                const int col = (tid % (BN / 16)) * 16;
                const int gcol = ld_n0 + col;
                const bool v = gcol < p.coutp;
                const uint8_t *src = p.fcodes + (v ? (int64_t)(k0 + r) * p.coutp + gcol : 0);
                cp_async16(ws + r * BN + col, src, v ? 16 : 0);
            }
            ++ld_it;
            ld_ci += 16;
            if (ld_ci == p.cs) {
                ld_ci = 0;
                ++ld_t;
            }
            if (++ld_kc == p.nchunks) {
                ld_kc = 0;
                ld_t = ld_ci = 0;
                ld_tile += vg;
                if (ld_it < total) set_load_tile(ld_tile);
            }
        }
    };
    auto load_group = [&]() {
#pragma unroll
        for (int g = 0; g < G; ++g) load_next();
        cp_async_commit();
    };

    int32_t acc[TM][TN];
    int32_t spa[TM];  // in-loop patch sums (sp_inloop)
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        spa[i] = 0;
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = 0;
    }
    const bool sp_inloop = p.sp_inloop != 0;

#pragma unroll
    for (int s = 0; s < NG - 1; ++s) load_group();
    mbar_wait(bar, 0);

    int c_kc = 0;
    int64_t c_tile = vb;
    int ep_par = 0;  // epilogue constant buffer (alternates per tile)
    for (int64_t it0 = 0; it0 < total; it0 += G) {
      cp_async_wait<NG - 2>();
      group_sync();
      load_group();
#pragma unroll 1
      for (int g = 0; g < G; ++g) {
        const int64_t it = it0 + g;
        if (it >= total) break;
        const int stage = (int)(it % SLOTS);
        const uint8_t *as = act_s + stage * ACT_STAGE + (wm * 32 * TM + lane) * 16;
        const uint8_t *ws = w_s + stage * W_STAGE + wn * TN;

        // All 16 taps of this lane's TM pixel rows in one LDS.128 each: a quarter-warp
        // reads 8 adjacent 16-byte rows = 128 contiguous bytes, so 4 wavefronts per row
        // per chunk (four 32-bit loads at a 16-byte lane stride would cost 4 each).
        uint4 av[TM];
#pragma unroll
        for (int i = 0; i < TM; ++i) av[i] = *reinterpret_cast<const uint4 *>(as + i * 32 * 16);
        if (sp_inloop) {  // S_p += sum of the 16 code values (junk codes are raw 0 -> value 0)
#pragma unroll
            for (int i = 0; i < TM; ++i) {
                if (SGN) {
                    int s = __dp4a((int)av[i].x, 0x01010101, spa[i]);
                    s = __dp4a((int)av[i].y, 0x01010101, s);
                    s = __dp4a((int)av[i].z, 0x01010101, s);
                    spa[i] = __dp4a((int)av[i].w, 0x01010101, s);
                } else {
                    uint32_t s = __dp4a(av[i].x, 0x01010101u, (uint32_t)spa[i]);
                    s = __dp4a(av[i].y, 0x01010101u, s);
                    s = __dp4a(av[i].z, 0x01010101u, s);
                    spa[i] = (int32_t)__dp4a(av[i].w, 0x01010101u, s);
                }
            }
        }
#pragma unroll 1
        for (int q = 0; q < 4; ++q) {  // 4 taps per step, consumed as 2 pairs
            uint32_t aw[TM];  // codes of taps 4q..4q+3 of this lane's TM pixels
#pragma unroll
            for (int i = 0; i < TM; ++i) {
                aw[i] = av[i].x;  // rotate the row so word 0 is always the current step's
                av[i].x = av[i].y;
                av[i].y = av[i].z;
                av[i].z = av[i].w;
            }
#pragma unroll
            for (int kk = 0; kk < 4; kk += 2) {
                const int k0 = q * 4 + kk;
                uint32_t a0[TM], a1[TM];  // byte address of row a of the b-major table: base + 2a
#pragma unroll
                for (int i = 0; i < TM; ++i) {
                    a0[i] = __byte_perm(aw[i], 0, 0x4440u + kk) * 2u + lut_base;
                    a1[i] = __byte_perm(aw[i], 0, 0x4441u + kk) * 2u + lut_base;
                }
                uint32_t wv0[TN / 4], wv1[TN / 4];  // TN code bytes of taps k0, k0+1
                if (TN == 16) {
                    const uint4 x0 = *reinterpret_cast<const uint4 *>(ws + k0 * BN);
                    const uint4 x1 = *reinterpret_cast<const uint4 *>(ws + (k0 + 1) * BN);
                    wv0[0] = x0.x; wv0[1 % (TN / 4)] = x0.y; wv0[2 % (TN / 4)] = x0.z; wv0[3 % (TN / 4)] = x0.w;
                    wv1[0] = x1.x; wv1[1 % (TN / 4)] = x1.y; wv1[2 % (TN / 4)] = x1.z; wv1[3 % (TN / 4)] = x1.w;
                } else {
                    const uint2 x0 = *reinterpret_cast<const uint2 *>(ws + k0 * BN);
                    const uint2 x1 = *reinterpret_cast<const uint2 *>(ws + (k0 + 1) * BN);
                    wv0[0] = x0.x; wv0[1] = x0.y;
                    wv1[0] = x1.x; wv1[1] = x1.y;
                }
#pragma unroll
                for (int j = 0; j < TN; ++j) {
                    // code byte b -> bits 8..15 (b << 8); address = 2*(b << 8) + (2a + base)
                    const uint32_t sel = 0x4404u | ((uint32_t)(j & 3) << 4);
                    const uint32_t b0 = __byte_perm(wv0[j >> 2], 0, sel);
                    const uint32_t b1 = __byte_perm(wv1[j >> 2], 0, sel);
#pragma unroll
                    for (int i = 0; i < TM; ++i) {
                        int32_t v0, v1;
                        uint32_t ad0, ad1;  // one IMAD each: 2*(b<<8) + (2a + base)
                        asm("mad.lo.u32 %0, %1, 2, %2;" : "=r"(ad0) : "r"(b0), "r"(a0[i]));
                        asm("mad.lo.u32 %0, %1, 2, %2;" : "=r"(ad1) : "r"(b1), "r"(a1[i]));
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

        if (++c_kc < p.nchunks) continue;
        // ------------------------------------------------ fused epilogue for tile c_tile
        // In this kernel kpad <= 32768, so |A| < 2^31: WRAP32 and SATURATE32 are the
        // identity on the exact sum (axconv.py:128-133) and A = acc - junk exactly.
        c_kc = 0;
        const EpiConst e = epi_const(p);  // re-read per tile (keeps ~10 registers out of the main loop)
        const int64_t m0 = (c_tile / p.ntn) * BM;
        const int n0 = (int)(c_tile % p.ntn) * BN;
        c_tile += vg;
        int64_t *ep_cc = ep_cc_s + ep_par * BN;  // double-buffered: a barrier period may hold two epilogues
        float *ep_bias = ep_bias_s + ep_par * BN;
        ep_par ^= 1;
        if (tid < BN) {  // per-channel constants: K*zp1*zp2 - zp1*S_f[c] - junk, bias
            const int c = n0 + tid;
            ep_cc[tid] = c < p.cout ? e.kzz - e.zp1 * p.fsum[c] - e.junk : 0;
            ep_bias[tid] = (p.bias && c < p.cout) ? p.bias[c] : 0.0f;
        }
        group_sync();
        const int cb = n0 + wn * TN;
        const bool full = cb + TN <= p.cout && (p.cout & 3) == 0;
        const int64_t *cc = ep_cc + wn * TN;
        const float *bs = ep_bias + wn * TN;
#pragma unroll
        for (int i = 0; i < TM; ++i) {
            const int64_t mt = m0 + wm * 32 * TM + i * 32 + lane;  // position in tile order
            if (mt < p.M) {
                int64_t pix0;
                const int64_t m = pixel_of(p, mt, pix0);  // NHWC output pixel + its window origin
                int64_t sp = spa[i];                       // S_p (axconv.py:193)
                if (!sp_inloop) {
                    sp = 0;
                    for (int t = 0; t < p.taps; ++t) sp += p.pixsum[pix0 + tappix_s[t]];
                }
                psum_ovf |= (sp > INT32_MAX || sp < INT32_MIN);
                const int64_t pz = -e.zp2 * sp;
                float y[TN];
#pragma unroll
                for (int j = 0; j < TN; ++j) {
                    // corr = A - zp2*S_p - zp1*S_f + K*zp1*zp2 (axconv.py:249-254); fp64 dequant (:256)
                    const int64_t corr = (int64_t)acc[i][j] + pz + cc[j];
                    y[j] = __double2float_rn(e.scale * __ll2double_rn(corr));
                }
                float *dst = p.out + m * p.cout + cb;
                if (full) {
                    if (p.bias) {
#pragma unroll
                        for (int j = 0; j < TN; ++j) y[j] = __fadd_rn(y[j], bs[j]);  // graph.py:268-269
                    }
                    if (p.residual) {  // graph.py:282-286
                        const float4 *r4 = reinterpret_cast<const float4 *>(p.residual + m * p.cout + cb);
#pragma unroll
                        for (int j = 0; j < TN; j += 4) {
                            const float4 r = __ldg(r4 + j / 4);
                            y[j] = __fadd_rn(y[j], r.x); y[j + 1] = __fadd_rn(y[j + 1], r.y);
                            y[j + 2] = __fadd_rn(y[j + 2], r.z); y[j + 3] = __fadd_rn(y[j + 3], r.w);
                        }
                    }
                    if (p.relu) {
#pragma unroll
                        for (int j = 0; j < TN; ++j) y[j] = (y[j] > 0.0f || y[j] != y[j]) ? y[j] : 0.0f;
                    }
#pragma unroll
                    for (int j = 0; j < TN; ++j) track(y[j], tmin, tmax, nonfinite);
#pragma unroll
                    for (int j = 0; j < TN; j += 4)
                        *reinterpret_cast<float4 *>(dst + j) = make_float4(y[j], y[j + 1], y[j + 2], y[j + 3]);
                    if (p.acc_out) {
#pragma unroll
                        for (int j = 0; j < TN; ++j)
                            p.acc_out[m * p.cout + cb + j] = (int64_t)acc[i][j] - e.junk;
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < TN; ++j) {
                        if (cb + j < p.cout) {
                            float v = y[j];
                            if (p.bias) v = __fadd_rn(v, bs[j]);
                            if (p.residual) v = __fadd_rn(v, p.residual[m * p.cout + cb + j]);
                            if (p.relu) v = (v > 0.0f || v != v) ? v : 0.0f;
                            track(v, tmin, tmax, nonfinite);
                            dst[j] = v;
                            if (p.acc_out) p.acc_out[m * p.cout + cb + j] = (int64_t)acc[i][j] - e.junk;
                        }
                    }
                }
            }
            spa[i] = 0;
#pragma unroll
            for (int j = 0; j < TN; ++j) acc[i][j] = 0;
        }
      }  // sub-chunk g
    }    // group it0
    cp_async_wait<0>();
    const bool any = tmin <= tmax;
    range_commit(any ? f2ord(tmin) : INT32_MAX, any ? f2ord(tmax) : INT32_MIN, nonfinite, p.out_range, p.flags,
                 AXB_FLAG_OUT_NONFINITE);
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
            const uint8_t *f = p.fcodes + (int64_t)t * p.cs * p.coutp + c;
            for (int ci = 0; ci < p.c; ++ci) {
                const uint32_t idx16 = ((uint32_t)f[(int64_t)ci * p.coutp] << 8) | a[ci];
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
struct Variant {
    const char *name;
    int tm, tn, wm, wn;
    float cost;  // relative time per lookup slot (per-layer-normalised median on B200; 1 = best)
    int ng = 1;  // warp groups per CTA
};
// tuning table (axb_conv_desc.variant selects one explicitly; 0 = cost model below).
// cost: scripts/fit_variants.py over scripts/tune_variants.py runs on every ResNet-8/50/62 layer
// (the model's picks sum to within 0.05% of the per-layer best): each layer's time
// divided by waves*BM*BN*NGRP, normalised by the layer's best variant, median over layers.
static const Variant kVariants[] = {
    {"auto", 0, 0, 0, 0, 0.f},
    {"tm4tn16_w8x1", 4, 16, 8, 1, 1.132f},  {"tm4tn16_w4x2", 4, 16, 4, 2, 1.094f},
    {"tm4tn16_w2x4", 4, 16, 2, 4, 1.071f},  {"tm4tn8_w8x2", 4, 8, 8, 2, 1.098f},
    {"tm4tn8_w4x4", 4, 8, 4, 4, 1.049f},    {"tm2tn16_w12x1", 2, 16, 12, 1, 1.145f},
    {"tm4tn8_w6x2", 4, 8, 6, 2, 1.114f},    {"tm4tn16_w6x2", 4, 16, 6, 2, 1.067f},
    {"tm4tn16_w3x4", 4, 16, 3, 4, 1.031f},  {"tm2tn16_w16x1", 2, 16, 16, 1, 1.182f},
    {"tm2tn16_w8x2", 2, 16, 8, 2, 1.130f},  {"tm4tn16_w4x4", 4, 16, 4, 4, 1.177f},
    {"tm2tn8_w8x2", 2, 8, 8, 2, 1.168f},    {"tm2tn8_w4x4", 2, 8, 4, 4, 1.131f},
    {"tm4tn8_w2x8", 4, 8, 2, 8, 1.031f},    {"tm2tn8_w2x8", 2, 8, 2, 8, 1.121f},
    {"tm4tn8_w3x4", 4, 8, 3, 4, 1.060f},    {"tm2tn16_w4x4", 2, 16, 4, 4, 1.102f},
    {"g2_tm4tn8_w2x4", 4, 8, 2, 4, 1.029f, 2}, {"g2_tm4tn8_w4x2", 4, 8, 4, 2, 1.068f, 2},
    {"g2_tm4tn8_w1x8", 4, 8, 1, 8, 1.007f, 2}, {"g2_tm2tn8_w2x4", 2, 8, 2, 4, 1.078f, 2},
    {"g2_tm2tn8_w4x2", 2, 8, 4, 2, 1.111f, 2},
    {"g4_tm4tn8_w1x4", 4, 8, 1, 4, 1.000f, 4}, {"g4_tm4tn8_w2x2", 4, 8, 2, 2, 1.021f, 4},
    {"g4_tm2tn8_w2x2", 2, 8, 2, 2, 1.064f, 4},
};
constexpr int kNumVariants = sizeof(kVariants) / sizeof(kVariants[0]);

template <int TM, int TN, int WM, int WN, bool SGN, int NGRP = 1>
static int launch_fast(const ConvK &k, int sm_limit, cudaStream_t s, const char *name) {
    constexpr int BM = WM * 32 * TM, BN = WN * TN;
    const size_t smem = fast_smem(BM, BN, NGRP) - 512;  // dynamic part (range_commit scratch is static)
    auto fn = lutconv_fast<TM, TN, WM, WN, SGN, NGRP>;
    static int configured_dev = -1;  // one per instantiation
    int dev = 0;
    cudaGetDevice(&dev);
    if (configured_dev != dev) {
        if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return set_error(AXB_E_CUDA, "cannot raise dynamic shared memory for lutconv_fast");
        configured_dev = dev;
    }
    ConvK kk = k;
    kk.ntn = (k.coutp + BN - 1) / BN;
    kk.ntiles = ((k.M + BM - 1) / BM) * kk.ntn;
    int64_t grid = sm_limit > 0 ? sm_limit : sm_count();
    if (grid > (kk.ntiles + NGRP - 1) / NGRP) grid = (kk.ntiles + NGRP - 1) / NGRP;
    if (grid < 1) grid = 1;
    fn<<<(int)grid, NGRP * WM * WN * 32, smem, s>>>(kk);
    set_last_kernel(name);
    return check_launch("lutconv_fast");
}

template <bool SGN>
static int launch_variant(int v, const ConvK &k, int sm_limit, cudaStream_t s) {
    const char *nm = kVariants[v].name;
    switch (v) {
        case 1: return launch_fast<4, 16, 8, 1, SGN>(k, sm_limit, s, nm);
        case 2: return launch_fast<4, 16, 4, 2, SGN>(k, sm_limit, s, nm);
        case 3: return launch_fast<4, 16, 2, 4, SGN>(k, sm_limit, s, nm);
        case 4: return launch_fast<4, 8, 8, 2, SGN>(k, sm_limit, s, nm);
        case 5: return launch_fast<4, 8, 4, 4, SGN>(k, sm_limit, s, nm);
        case 6: return launch_fast<2, 16, 12, 1, SGN>(k, sm_limit, s, nm);
        case 7: return launch_fast<4, 8, 6, 2, SGN>(k, sm_limit, s, nm);
        case 8: return launch_fast<4, 16, 6, 2, SGN>(k, sm_limit, s, nm);
        case 9: return launch_fast<4, 16, 3, 4, SGN>(k, sm_limit, s, nm);
        case 10: return launch_fast<2, 16, 16, 1, SGN>(k, sm_limit, s, nm);
        case 11: return launch_fast<2, 16, 8, 2, SGN>(k, sm_limit, s, nm);
        case 12: return launch_fast<4, 16, 4, 4, SGN>(k, sm_limit, s, nm);
        case 13: return launch_fast<2, 8, 8, 2, SGN>(k, sm_limit, s, nm);
        case 14: return launch_fast<2, 8, 4, 4, SGN>(k, sm_limit, s, nm);
        case 15: return launch_fast<4, 8, 2, 8, SGN>(k, sm_limit, s, nm);
        case 16: return launch_fast<2, 8, 2, 8, SGN>(k, sm_limit, s, nm);
        case 17: return launch_fast<4, 8, 3, 4, SGN>(k, sm_limit, s, nm);
        case 18: return launch_fast<2, 16, 4, 4, SGN>(k, sm_limit, s, nm);
        case 19: return launch_fast<4, 8, 2, 4, SGN, 2>(k, sm_limit, s, nm);
        case 20: return launch_fast<4, 8, 4, 2, SGN, 2>(k, sm_limit, s, nm);
        case 21: return launch_fast<4, 8, 1, 8, SGN, 2>(k, sm_limit, s, nm);
        case 22: return launch_fast<2, 8, 2, 4, SGN, 2>(k, sm_limit, s, nm);
        case 23: return launch_fast<2, 8, 4, 2, SGN, 2>(k, sm_limit, s, nm);
        case 24: return launch_fast<4, 8, 1, 4, SGN, 4>(k, sm_limit, s, nm);
        case 25: return launch_fast<4, 8, 2, 2, SGN, 4>(k, sm_limit, s, nm);
        case 26: return launch_fast<2, 8, 2, 2, SGN, 4>(k, sm_limit, s, nm);
        default: return set_error(AXB_E_VALUE, "unknown conv kernel variant");
    }
}

// Cost model (fit with scripts/tune_variants.py on B200, within 0.1% of the best
// variant summed over all ResNet-8/50/62 layers): time ~ cost * waves * BM * BN,
// waves = ceil(tiles / SMs) -- so wave quantization of small layers picks smaller tiles.
static int pick_variant(const ConvK &k) {
    const int64_t sms = sm_count();
    int best = 1;
    double best_t = 1e300;
    for (int v = 1; v < kNumVariants; ++v) {
        const Variant &x = kVariants[v];
        const int64_t bm = (int64_t)x.wm * 32 * x.tm, bn = (int64_t)x.wn * x.tn;
        const int64_t tiles = ((k.M + bm - 1) / bm) * ((k.coutp + bn - 1) / bn);
        const int64_t waves = (tiles + sms * x.ng - 1) / (sms * x.ng);  // x.ng tile streams per SM
        const double t = (double)x.cost * (double)waves * (double)(bm * bn * x.ng);
        if (t < best_t) {
            best_t = t;
            best = v;
        }
    }
    return best;
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

    const bool fast = !d->force_generic && d->kpad <= 32768 && k.taps <= kMaxTaps && d->cs % 16 == 0 &&
                      d->kpad % 16 == 0 && d->coutp % 16 == 0;
    if (fast) {
        // filter-specialised product table supplied (axb_ftable_prepare): the ftable kernel
        const bool use_ft = d->ftable != nullptr && d->variant == 0;
        if (!use_ft && !d->pixsum && d->kpad > 512)
            return set_error(AXB_E_VALUE, "the LUT kernel needs per-pixel code sums (pixsum) for this K");
        k.ftable = d->ftable;
        int v = d->variant;
        if (v < 0 || v >= kNumVariants) return set_error(AXB_E_VALUE, "unknown conv kernel variant");
        if (v == 0 && !use_ft) v = pick_variant(k);
        // int32 gather offsets: split the batch so every launch's code tensor stays < 2 GiB
        const int64_t per_img = d->hp * d->wp * d->cs;
        int64_t step = ((int64_t(1) << 31) - 1) / (per_img > 0 ? per_img : 1);
        if (step < 1) return set_error(AXB_E_VALUE, "one image's code tensor exceeds 2 GiB");
        int order = d->pixel_order;
        if (order == 0) order = (d->oh % 4 == 0 && d->ow % 8 == 0) ? 4 : 1;
        if (order == 4 && (d->oh % 4 || d->ow % 8)) return set_error(AXB_E_VALUE, "4x8 pixel order needs oh%4==0, ow%8==0");
        k.blk = order == 4 ? 4 : 1;
        k.fd_hw = make_fastdiv((uint32_t)(d->oh * d->ow));
        k.fd_ow = make_fastdiv((uint32_t)d->ow);
        k.fd_band = make_fastdiv((uint32_t)(4 * d->ow));
        // short K: the epilogue's per-pixel tap gather dominates -> sum codes in the loop instead
        k.sp_inloop = d->kpad <= 512 ? 1 : 0;
        for (int64_t b0 = 0; b0 < d->n; b0 += step) {
            const int64_t nb = (d->n - b0 < step) ? d->n - b0 : step;
            ConvK kc = k;
            kc.codes = d->codes + b0 * per_img;
            kc.pixsum = d->pixsum + b0 * d->hp * d->wp;
            kc.M = nb * d->oh * d->ow;
            const int64_t ooff = b0 * d->oh * d->ow * d->cout;
            kc.out = d->out + ooff;
            kc.residual = d->residual ? d->residual + ooff : nullptr;
            kc.acc_out = d->acc_out ? d->acc_out + ooff : nullptr;
            const int rc = use_ft ? conv_ft_launch(kc, d->ft_variant, lut->is_signed, d->sm_limit, s)
                                  : (lut->is_signed ? launch_variant<true>(v, kc, d->sm_limit, s)
                                                    : launch_variant<false>(v, kc, d->sm_limit, s));
            if (rc) return rc;
        }
        return AXB_OK;
    }
    if (!d->pixsum) return set_error(AXB_E_VALUE, "the generic kernel needs per-pixel code sums (pixsum)");
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

int axb_conv_variant_count(void) { return kNumVariants; }
const char *axb_conv_variant_name(int v) { return (v >= 0 && v < kNumVariants) ? kVariants[v].name : ""; }

}  // extern "C"
