// K3 (ftable path): approximate convolution over a FILTER-SPECIALISED product
// table, with the same fused epilogue as lutconv_fast.
//
// Same arithmetic as axconv.py:136-146 (A[r,c] = sum_k lut[(P[r,k]<<8)|F[c,k]]),
// :246-256 (corrections, fp64 dequant) and graph.py:268-286 (bias/Add/ReLU); only
// WHERE the 16-bit products are looked up changes.
//
// The filter codes of a layer are constant (graph.py:129-130), so for every
// filter row k and output-channel pair (c, c+1) the 256 possible products
//     W[k][pair][a] = ( lut[(a<<8)|F[k][c]] , lut[(a<<8)|F[k][c+1]] )
// can be gathered ONCE per layer (axb_ftable_prepare) into 32-bit words.  The
// conv then does, per lane (one output pixel, activation code a at row k):
//     w = W[k][pair][a]   (one LDS.32 = TWO exact table lookups)
// i.e. the 16-bit entries are still gathered from shared memory by the
// activation code, but two channels share one 4-byte bank word, so a 32-lane
// wavefront delivers up to 64 lookups instead of 32 (LDS.16 on the b-major
// LUT), and the address of every pair is an immediate offset from one
// per-(pixel, row) register (no per-lookup IMAD).
//
// Exact accumulation of packed pairs: entries are biased to unsigned 16-bit
// (signed: u = raw ^ 0x8000 = v + 32768), per pair the kernel keeps
//     all = sum w  (mod 2^32)      hi = sum (w >> 16)   (exact, < 2^32)
// so  sum u_lo = all - (hi << 16)  (mod 2^32, exact since kpad <= 32768),
// A = sum u - kpad * 32768 (signed) -- bit-identical int sums.  Junk rows
// (channel / K padding) hold the zero contribution (u = bias) for every a.
//
// Layout in HBM (uint32): [sb = coutp/8][k = 0..kpad-1][pair = 0..3][a = 0..255], i.e. 4 KiB
// per (8-channel sub-block, row).  A tile of 8 or 16 channels (NPB = 4 or 8 pairs) streams KS
// consecutive rows of its one or two sub-blocks per pipeline stage, moved by TMA bulk copies
// (cp.async.bulk + mbarrier complete_tx) into a ring of ST stages.  Thread 0 refills the slot
// of stage g-1 at the start of stage g, after every warp released it: each lane executes
// fence.proxy.async (its generic-proxy LDS reads before the async-proxy refill), then lane 0
// arrives on the slot's "empty" mbarrier.  Activation codes are read straight from the
// zp-padded NHWC code tensor into registers (one LDG.128 = 16 rows of one pixel), one 16-row
// chunk ahead, across tile boundaries.  The kernel is launched with programmatic dependent
// launch: barrier init, the tap table and the first table stages overlap the previous
// kernel's tail (pdl_wait before the first activation load).
//
// Tiles: BM = WARPS*32*TM output pixels x BN = 2*NPB channels; tile = nb * ntm + mt, so
// the CTAs running concurrently share one channel block's table rows in L2.
#include <cstdlib>

#include "axb_convk.cuh"

namespace axb {

constexpr int kFtSubPairs = 4;                     // channel pairs per 8-channel sub-block
constexpr int kFtRowWords = kFtSubPairs * 256;     // one (sub-block, row) slice: 4 pairs x 256 codes
constexpr int kFtRowBytes = kFtRowWords * 4;       // 4 KiB

// per-warp epilogue constants of a tile's BN = 2*NPB channels: int64 correction term + fp32 bias (16 warps max)
__host__ __device__ constexpr int ft_epi_bytes(int NPB) { return 16 * 2 * NPB * 12; }
// NPB = channel pairs per tile (4: 8 channels, 8: 16 channels); a stage holds KS rows
__host__ __device__ constexpr int ft_stage_bytes(int NPB, int KS) { return (NPB / 4) * KS * kFtRowBytes; }
__host__ __device__ constexpr int ft_smem(int NPB, int KS, int ST) {
    return ST * ft_stage_bytes(NPB, KS) + kMaxTaps * 4 + 2 * ST * 8 + ft_epi_bytes(NPB);
}

// CL > 1: a thread-block cluster of CL CTAs works on CL pixel tiles of the SAME channel block in
// lockstep; each CTA fetches 1/CL of every stage and multicasts it into all CL CTAs' rings (one L2
// read per cluster instead of per CTA).  A slot is refilled once the warps of ALL CL CTAs released it
// (the empty barrier counts CL*WARPS arrivals, made locally and through mapa'd remote arrives).
template <int TM, int WARPS, int NPB, int KS, int ST, bool SGN, int CL, int PF>
__global__ void __launch_bounds__(WARPS * 32, 1) lutconv_ft(const ConvK p) {
    constexpr int NT = WARPS * 32;
    constexpr int BM = NT * TM;
    constexpr int BN = 2 * NPB;
    constexpr int NSUB = NPB / 4;  // 8-channel sub-blocks per tile
    constexpr int SPC = 16 / KS;   // pipeline stages per 16-row chunk
    constexpr uint32_t STAGE_BYTES = ft_stage_bytes(NPB, KS);
    static_assert(NPB == 4 || NPB == 8, "4 or 8 channel pairs per tile");
    static_assert(PF == 1 || PF == 2, "activation chunks loaded ahead: 1 or 2");
    static_assert(KS == 4 || KS == 8 || KS == 16, "KS rows per stage: 4, 8 or 16");
    static_assert(ft_smem(NPB, KS, ST) + 512 <= 232448, "ftable ring exceeds shared memory");

    extern __shared__ __align__(1024) uint8_t smem[];
    int32_t *tapoff_s = reinterpret_cast<int32_t *>(smem + ST * STAGE_BYTES);
    uint64_t *full = reinterpret_cast<uint64_t *>(tapoff_s + kMaxTaps);
    uint64_t *empty = full + ST;
    static_assert(WARPS <= 16, "per-warp epilogue constants");
    int64_t *epi_cc = reinterpret_cast<int64_t *>(empty + ST) + (threadIdx.x >> 5) * BN;  // this warp's
    float *epi_bv = reinterpret_cast<float *>(reinterpret_cast<int64_t *>(empty + ST) + 16 * BN) + (threadIdx.x >> 5) * BN;
    const uint32_t *tab = reinterpret_cast<const uint32_t *>(smem);

    const int tid = (int)threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;

    if (tid == 0) {
        for (int s = 0; s < ST; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, WARPS * CL);
        }
    }
    for (int t = tid; t < p.taps; t += NT) tapoff_s[t] = ((t / p.kw) * p.dh * p.wp + (t % p.kw) * p.dw) * p.cs;
    __syncthreads();
    if constexpr (CL > 1) cluster_sync();  // peers' barriers initialised before any remote arrive / multicast
    const uint32_t rank = CL > 1 ? cluster_ctarank() : 0;

    // super-tile st = (channel block nb, pixel-tile group): CTA `rank` of the cluster takes pixel tile
    // (st % ntm) * CL + rank (p.ntm = pixel-tile groups per channel block; tiles past the end are
    // computed on pixel 0 and never stored)
    const int64_t grid = gridDim.x / CL;  // clusters
    const int64_t cid = blockIdx.x / CL;
    const int64_t my_tiles = p.ntiles > cid ? (p.ntiles - cid + grid - 1) / grid : 0;
    const int64_t spt = (int64_t)p.nchunks * SPC;  // stages per tile
    const int64_t total = my_tiles * spt;

    // ---- producer (thread 0): stage h -> rows [q*KS, q*KS+KS) of tile pr_tile's channel block
    int64_t pr_h = 0, pr_q = 0, pr_tile = cid;
    auto produce = [&]() {
        const int slot = (int)(pr_h % ST);
        const int64_t nb = pr_tile / p.ntm;  // channel block of BN channels = NSUB sub-blocks
        mbar_expect_tx(full + slot, STAGE_BYTES);
        // the stage = NSUB pieces (KS rows of one sub-block each); split into NPART equal parts,
        // this CTA fetches parts rank, rank+CL, ... and multicasts them to the whole cluster
        constexpr int NPART = NSUB > CL ? NSUB : CL;
        constexpr int PPS = NPART / NSUB;  // parts per piece
        constexpr uint32_t PART = STAGE_BYTES / NPART;
#pragma unroll
        for (int part = (int)rank; part < NPART; part += CL) {
            const int sb = part / PPS, q = part % PPS;
            const uint32_t *src =
                p.ftable + ((nb * NSUB + sb) * p.kpad + pr_q * KS + q * (KS / PPS)) * kFtRowWords;
            uint8_t *dst = smem + slot * STAGE_BYTES + part * PART;
            if constexpr (CL == 1)
                bulk_g2s(dst, src, PART, full + slot);
            else
                bulk_g2s_multicast(dst, src, PART, full + slot, (uint16_t)((1u << CL) - 1));
        }
        ++pr_h;
        if (++pr_q == spt) {
            pr_q = 0;
            pr_tile += grid;
        }
    };
    if (tid == 0)
        for (int s = 0; s < ST - 1 && pr_h < total; ++s) produce();

    // ---- activation rows of this lane's TM pixels (int32 offsets: < 2 GiB per launch)
    int32_t rowbase[TM];
    auto set_rows = [&](int64_t tile) {
        const int64_t m0 = ((tile % p.ntm) * CL + rank) * BM;
#pragma unroll
        for (int i = 0; i < TM; ++i) {
            const int64_t mt = m0 + warp * 32 * TM + i * 32 + lane;
            int64_t pix0 = 0;
            if (mt < p.M) pixel_of(p, mt, pix0);
            rowbase[i] = (int32_t)(pix0 * p.cs);
        }
    };
    // loader: runs PF chunks ahead of the consumer, across tile boundaries
    // everything above (barrier init, tap table, the first table stages in flight) overlaps the
    // predecessor's tail; its outputs (codes, qparams, residual, ranges) are read only after this
    pdl_wait();
    uint4 av[PF][TM];
    int ld_t = 0, ld_ci = 0, ld_kc = 0;  // tap, channel offset and index of the next chunk to load
    int64_t ld_left = my_tiles * p.nchunks, ld_tile = cid;
    auto load_next = [&](uint4(&dst)[TM]) {
        if (ld_left == 0) return;
        const int off = tapoff_s[ld_t] + ld_ci;
#pragma unroll
        for (int i = 0; i < TM; ++i) dst[i] = __ldg(reinterpret_cast<const uint4 *>(p.codes + rowbase[i] + off));
        --ld_left;
        ld_ci += 16;
        if (ld_ci == p.cs) {
            ld_ci = 0;
            ++ld_t;
        }
        if (++ld_kc == p.nchunks) {
            ld_kc = ld_t = ld_ci = 0;
            ld_tile += grid;
            if (ld_left > 0) set_rows(ld_tile);
        }
    };

    uint32_t acc_all[TM][NPB], acc_hi[TM][NPB];
    int32_t spa[TM];
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        spa[i] = 0;
#pragma unroll
        for (int j = 0; j < NPB; ++j) acc_all[i][j] = acc_hi[i][j] = 0;
    }

    float tmin = INFINITY, tmax = -INFINITY;
    int nonfinite = 0;
    const int64_t bias_units = SGN ? (int64_t)32768 * p.kpad : 0;

    int64_t g = 0;  // consumer stage counter
    int64_t c_tile = cid;
    if (my_tiles > 0) {
        set_rows(c_tile);
#pragma unroll
        for (int q = 0; q < PF; ++q) load_next(av[q]);
    }
    for (int64_t jt = 0; jt < my_tiles; ++jt) {
#pragma unroll 1
        for (int kc = 0; kc < p.nchunks; ++kc) {
            uint4 cur[TM];
#pragma unroll
            for (int i = 0; i < TM; ++i) {
                cur[i] = av[0][i];
                if (PF == 2) av[0][i] = av[PF - 1][i];
            }
            load_next(av[PF - 1]);
            // S_p += the 16 code values (junk codes are raw 0 -> value 0), axconv.py:193
#pragma unroll
            for (int i = 0; i < TM; ++i) {
                if (SGN) {
                    int s = __dp4a((int)cur[i].x, 0x01010101, spa[i]);
                    s = __dp4a((int)cur[i].y, 0x01010101, s);
                    s = __dp4a((int)cur[i].z, 0x01010101, s);
                    spa[i] = __dp4a((int)cur[i].w, 0x01010101, s);
                } else {
                    uint32_t s = __dp4a(cur[i].x, 0x01010101u, (uint32_t)spa[i]);
                    s = __dp4a(cur[i].y, 0x01010101u, s);
                    s = __dp4a(cur[i].z, 0x01010101u, s);
                    spa[i] = (int32_t)__dp4a(cur[i].w, 0x01010101u, s);
                }
            }
#pragma unroll 1
            for (int st = 0; st < SPC; ++st) {
                const int slot = (int)(g % ST);
                if (tid == 0 && pr_h < total) {
                    // refill the slot stage g-1 used, once every warp (of every cluster CTA) released it.
                    // (A non-blocking variant that skips the refill while a slow warp still holds the
                    // slot measured slower: the pipeline lead in bytes is what matters.)
                    if (g >= 1) {
                        if constexpr (CL == 1)
                            mbar_wait(empty + (g - 1) % ST, (uint32_t)(((g - 1) / ST) & 1));
                        else
                            mbar_wait_cluster(empty + (g - 1) % ST, (uint32_t)(((g - 1) / ST) & 1));
                    }
                    produce();
                }
                mbar_wait_sleep(full + slot, (uint32_t)((g / ST) & 1));
                const uint32_t *stab = tab + slot * (STAGE_BYTES / 4);
#pragma unroll
                for (int kl = 0; kl < KS; ++kl) {
                    uint32_t ix[TM];  // word index of row kl, code a: kl*1024 + a (sub-block 0)
#pragma unroll
                    for (int i = 0; i < TM; ++i) {
                        const uint32_t wv = kl < 4 ? cur[i].x : (kl < 8 ? cur[i].y : (kl < 12 ? cur[i].z : cur[i].w));
                        ix[i] = __byte_perm(wv, 0, 0x4440u + (kl & 3)) + kl * kFtRowWords;
                    }
#pragma unroll
                    for (int j = 0; j < NPB; ++j) {
#pragma unroll
                        for (int i = 0; i < TM; ++i) {
                            const uint32_t w = stab[ix[i] + (j / 4) * (KS * kFtRowWords) + (j % 4) * 256];
                            acc_all[i][j] += w;
                            acc_hi[i][j] += w >> 16;
                        }
                    }
                }
                fence_proxy_async_smem();  // this lane's LDS reads of the slot before the TMA refill
                __syncwarp();
                if constexpr (CL == 1) {
                    if (lane == 0) mbar_arrive(empty + slot);
                } else if (lane < CL) {  // release the slot in every CTA of the cluster
                    mbar_arrive_cluster(empty + slot, (uint32_t)lane);
                }
#pragma unroll
                for (int i = 0; i < TM; ++i) {  // next stage's rows move to the front
                    if (KS == 4) {
                        cur[i].x = cur[i].y; cur[i].y = cur[i].z; cur[i].z = cur[i].w;
                    } else if (KS == 8) {
                        cur[i].x = cur[i].z; cur[i].y = cur[i].w;
                    }
                }
                ++g;
            }
        }

        // ------------------------------------------------ fused epilogue for tile c_tile
        // kpad <= 32768 here, so |A| < 2^31: WRAP32 / SATURATE32 are the identity (axconv.py:128-133)
        {
            const EpiConst e = epi_const(p);
            const int64_t nb = c_tile / p.ntm;
            const int64_t m0 = ((c_tile % p.ntm) * CL + rank) * BM;
            const int cb = (int)nb * BN;
            const bool full_blk = cb + BN <= p.cout && (p.cout & 3) == 0;
            const bool has_res = p.residual != nullptr, relu = p.relu != 0;
            // the tile's per-channel terms, computed once per warp into shared memory and read back as
            // broadcasts: -zp1*S_f + K*zp1*zp2 - (entry bias), and the bias (-0.0f when absent: x + -0 == x)
            __syncwarp();
            if (lane < BN) {
                const bool ok = cb + lane < p.cout;
                epi_cc[lane] = ok ? e.kzz - e.zp1 * __ldg(p.fsum + cb + lane) - bias_units : 0;
                epi_bv[lane] = (ok && p.bias) ? __ldg(p.bias + cb + lane) : -0.0f;
            }
            __syncwarp();
#pragma unroll
            for (int i = 0; i < TM; ++i) {
                const int64_t mt = m0 + warp * 32 * TM + i * 32 + lane;
                if (mt < p.M) {
                    int64_t pix0;
                    const int64_t m = pixel_of(p, mt, pix0);
                    const int64_t pz = -e.zp2 * (int64_t)spa[i];
                    float *dst = p.out + m * p.cout + cb;
                    // four channels (two packed pairs) at a time: float4 stores, few live registers
#pragma unroll
                    for (int q = 0; q < NPB / 2; ++q) {
                        // corr = A - zp2*S_p - zp1*S_f + K*zp1*zp2 (axconv.py:249-254); fp64 dequant (:256);
                        // bias (graph.py:268-269), Add (:282-286), ReLU (:276-277)
                        float y[4];
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const uint32_t hi = acc_hi[i][2 * q + h];
                            const uint32_t lo = acc_all[i][2 * q + h] - (hi << 16);
                            const int c = 4 * q + 2 * h;
                            y[2 * h] = __fadd_rn(
                                __double2float_rn(e.scale * __ll2double_rn((int64_t)lo + (pz + epi_cc[c]))), epi_bv[c]);
                            y[2 * h + 1] = __fadd_rn(
                                __double2float_rn(e.scale * __ll2double_rn((int64_t)hi + (pz + epi_cc[c + 1]))),
                                epi_bv[c + 1]);
                        }
                        const int c0 = cb + 4 * q;
                        if (full_blk) {
                            if (has_res) {
                                const float4 r = __ldg(reinterpret_cast<const float4 *>(p.residual + m * p.cout + c0));
                                y[0] = __fadd_rn(y[0], r.x); y[1] = __fadd_rn(y[1], r.y);
                                y[2] = __fadd_rn(y[2], r.z); y[3] = __fadd_rn(y[3], r.w);
                            }
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                if (relu) y[j] = (y[j] > 0.0f || y[j] != y[j]) ? y[j] : 0.0f;  // np.maximum(x, 0)
                                track(y[j], tmin, tmax, nonfinite);
                            }
                            *reinterpret_cast<float4 *>(dst + 4 * q) = make_float4(y[0], y[1], y[2], y[3]);
                        } else {
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                if (c0 + j < p.cout) {
                                    float v = y[j];
                                    if (has_res) v = __fadd_rn(v, p.residual[m * p.cout + c0 + j]);
                                    if (relu) v = (v > 0.0f || v != v) ? v : 0.0f;
                                    track(v, tmin, tmax, nonfinite);
                                    dst[4 * q + j] = v;
                                }
                            }
                        }
                        if (p.acc_out) {
#pragma unroll
                            for (int h = 0; h < 2; ++h) {
                                const uint32_t hi = acc_hi[i][2 * q + h];
                                const uint32_t lo = acc_all[i][2 * q + h] - (hi << 16);
                                const int c = c0 + 2 * h;
                                if (c < p.cout) p.acc_out[m * p.cout + c] = (int64_t)lo - bias_units;
                                if (c + 1 < p.cout) p.acc_out[m * p.cout + c + 1] = (int64_t)hi - bias_units;
                            }
                        }
                    }
                }
                spa[i] = 0;
#pragma unroll
                for (int j = 0; j < NPB; ++j) acc_all[i][j] = acc_hi[i][j] = 0;
            }
        }
        c_tile += grid;
    }
    const bool any = tmin <= tmax;
    range_commit(any ? f2ord(tmin) : INT32_MAX, any ? f2ord(tmax) : INT32_MIN, nonfinite, p.out_range, p.flags,
                 AXB_FLAG_OUT_NONFINITE);
    if constexpr (CL > 1) cluster_sync();  // no CTA leaves while peers may still arrive on its barriers
}

// ---------------------------------------------------------------- code-major variant (CM)
// Same products, code-major layout: CM[cb][k][a][16 pairs] (uint32 words as above), i.e. the 32
// channels of block cb at row k and activation code a are 64 contiguous bytes.  Lanes = (pixel,
// quarter q): one LDS.128 at CM[k][a][4q..4q+3] delivers 4 pairs = 8 products of one pixel, a warp
// instruction covers 8 pixels x 32 channels = 512 B = 4 wavefronts when the 8 pixels' codes spread
// over both bank halves (a 64-byte row sits in bank half a & 1; equal codes broadcast).  Against the
// pair-major kernel above: 8 products per LDS instead of 2 (fewer instructions per product), and on
// high-entropy codes (image stems) far fewer conflict wavefronts -- measured on real ResNet-8 codes
// 12.3e12 vs 9.7e12 products/s, on uniform codes 11.0e12 vs 5.4e12 (scripts/lut_gather_bench.cu).
// Per lane: J pixels (8*J per warp), 4 pairs each; lane (pixel, q) loads rows 4q..4q+3 of its pixel's
// 16-row chunk (one 32-bit word) and a stage's rows come from the right lane by one SHFL per pixel.
// Tiles of BM = WARPS*8*J pixels x 32 channels; the same TMA ring and epilogue.
constexpr int kCmPairs = 16;                   // channel pairs per 32-channel block
constexpr int kCmRowWords = 256 * kCmPairs;    // one (block, row) slice: 256 codes x 16 pairs
constexpr int kCmRowBytes = kCmRowWords * 4;   // 16 KiB
__host__ __device__ constexpr int cm_stage_bytes(int KS) { return KS * kCmRowBytes; }
__host__ __device__ constexpr int cm_smem(int KS, int ST) { return ST * cm_stage_bytes(KS) + kMaxTaps * 4 + 2 * ST * 8; }

template <int J, int WARPS, int KS, int ST, bool SGN, int PF>
__global__ void __launch_bounds__(WARPS * 32, 1) lutconv_ftcm(const ConvK p) {
    constexpr int NT = WARPS * 32;
    constexpr int PXW = 8 * J;        // pixels per warp
    constexpr int BM = WARPS * PXW;
    constexpr int BN = 32;
    constexpr int SPC = 16 / KS;
    constexpr uint32_t STAGE_BYTES = cm_stage_bytes(KS);
    static_assert(KS == 2 || KS == 4, "KS rows per stage: 2 or 4");
    static_assert(cm_smem(KS, ST) + 512 <= 232448, "code-major ring exceeds shared memory");

    extern __shared__ __align__(1024) uint8_t smem[];
    int32_t *tapoff_s = reinterpret_cast<int32_t *>(smem + ST * STAGE_BYTES);
    uint64_t *full = reinterpret_cast<uint64_t *>(tapoff_s + kMaxTaps);
    uint64_t *empty = full + ST;
    const uint32_t *tab = reinterpret_cast<const uint32_t *>(smem);

    const int tid = (int)threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const int q = lane & 3, ps = lane >> 2;

    if (tid == 0) {
        for (int s = 0; s < ST; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, WARPS);
        }
    }
    for (int t = tid; t < p.taps; t += NT) tapoff_s[t] = ((t / p.kw) * p.dh * p.wp + (t % p.kw) * p.dw) * p.cs;
    __syncthreads();

    const int64_t grid = gridDim.x;
    const int64_t cid = blockIdx.x;
    const int64_t my_tiles = p.ntiles > cid ? (p.ntiles - cid + grid - 1) / grid : 0;
    const int64_t spt = (int64_t)p.nchunks * SPC;
    const int64_t total = my_tiles * spt;

    int64_t pr_h = 0, pr_q = 0, pr_tile = cid;
    auto produce = [&]() {
        const int slot = (int)(pr_h % ST);
        const int64_t nb = pr_tile / p.ntm;
        mbar_expect_tx(full + slot, STAGE_BYTES);
        bulk_g2s(smem + slot * STAGE_BYTES, p.ftable + (nb * p.kpad + pr_q * KS) * kCmRowWords, STAGE_BYTES,
                 full + slot);
        ++pr_h;
        if (++pr_q == spt) {
            pr_q = 0;
            pr_tile += grid;
        }
    };
    if (tid == 0)
        for (int s = 0; s < ST - 1 && pr_h < total; ++s) produce();

    int32_t rowbase[J];
    auto set_rows = [&](int64_t tile) {
        const int64_t m0 = (tile % p.ntm) * BM;
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const int64_t mt = m0 + warp * PXW + j * 8 + ps;
            int64_t pix0 = 0;
            if (mt < p.M) pixel_of(p, mt, pix0);
            rowbase[j] = (int32_t)(pix0 * p.cs);
        }
    };
    pdl_wait();
    uint32_t av[PF][J];  // rows 4q..4q+3 of pixel j's next chunks (the 4 lanes of a pixel hold its 16 rows)
    int ld_t = 0, ld_ci = 0, ld_kc = 0;
    int64_t ld_left = my_tiles * p.nchunks, ld_tile = cid;
    auto load_next = [&](uint32_t(&dst)[J]) {
        if (ld_left == 0) return;
        const int off = tapoff_s[ld_t] + ld_ci;
#pragma unroll
        for (int j = 0; j < J; ++j) dst[j] = __ldg(reinterpret_cast<const uint32_t *>(p.codes + rowbase[j] + off) + q);
        --ld_left;
        ld_ci += 16;
        if (ld_ci == p.cs) {
            ld_ci = 0;
            ++ld_t;
        }
        if (++ld_kc == p.nchunks) {
            ld_kc = ld_t = ld_ci = 0;
            ld_tile += grid;
            if (ld_left > 0) set_rows(ld_tile);
        }
    };

    uint32_t acc_all[J][4], acc_hi[J][4];
    int32_t spa[J];
#pragma unroll
    for (int j = 0; j < J; ++j) {
        spa[j] = 0;
#pragma unroll
        for (int r = 0; r < 4; ++r) acc_all[j][r] = acc_hi[j][r] = 0;
    }
    float tmin = INFINITY, tmax = -INFINITY;
    int nonfinite = 0;
    const int64_t bias_units = SGN ? (int64_t)32768 * p.kpad : 0;

    int64_t g = 0;
    int64_t c_tile = cid;
    if (my_tiles > 0) {
        set_rows(c_tile);
#pragma unroll
        for (int f = 0; f < PF; ++f) load_next(av[f]);
    }
    for (int64_t jt = 0; jt < my_tiles; ++jt) {
#pragma unroll 1
        for (int kc = 0; kc < p.nchunks; ++kc) {
            uint32_t cur[J];
#pragma unroll
            for (int j = 0; j < J; ++j) {
                cur[j] = av[0][j];
                if (PF == 2) av[0][j] = av[1][j];
            }
            load_next(av[PF - 1]);
#pragma unroll
            for (int j = 0; j < J; ++j) {  // this lane's 4 codes of S_p; the 4 lanes are summed in the epilogue
                if (SGN)
                    spa[j] = __dp4a((int)cur[j], 0x01010101, spa[j]);
                else
                    spa[j] = (int32_t)__dp4a(cur[j], 0x01010101u, (uint32_t)spa[j]);
            }
#pragma unroll 1
            for (int st = 0; st < SPC; ++st) {
                const int slot = (int)(g % ST);
                if (tid == 0 && pr_h < total) {
                    if (g >= 1) mbar_wait(empty + (g - 1) % ST, (uint32_t)(((g - 1) / ST) & 1));
                    produce();
                }
                mbar_wait(full + slot, (uint32_t)((g / ST) & 1));
                const uint4 *stab = reinterpret_cast<const uint4 *>(tab + slot * (STAGE_BYTES / 4)) + q;
                // rows 4*st4 .. 4*st4+KS-1 of the chunk live in lane (ps, st4) of each pixel
                const int st4 = (st * KS) >> 2, sub = (st * KS) & 3;
                uint32_t rw[J];
#pragma unroll
                for (int j = 0; j < J; ++j) rw[j] = __shfl_sync(0xffffffffu, cur[j], (lane & ~3) | st4);
#pragma unroll
                for (int kl = 0; kl < KS; ++kl) {
#pragma unroll
                    for (int j = 0; j < J; ++j) {
                        const uint32_t a = __byte_perm(rw[j], 0, 0x4440u + ((sub + kl) & 3));
                        const uint4 w = stab[kl * (kCmRowWords / 4) + a * 4];
                        acc_all[j][0] += w.x; acc_hi[j][0] += w.x >> 16;
                        acc_all[j][1] += w.y; acc_hi[j][1] += w.y >> 16;
                        acc_all[j][2] += w.z; acc_hi[j][2] += w.z >> 16;
                        acc_all[j][3] += w.w; acc_hi[j][3] += w.w >> 16;
                    }
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(empty + slot);
                ++g;
            }
        }

        {
            const EpiConst e = epi_const(p);
            const int64_t nb = c_tile / p.ntm;
            const int64_t m0 = (c_tile % p.ntm) * BM;
            const int cb = (int)nb * BN + q * 8;  // this lane's 8 channels
            const bool full_blk = cb + 8 <= p.cout && (p.cout & 3) == 0;
#pragma unroll
            for (int j = 0; j < J; ++j) {  // S_p of pixel j = the 4 lanes' partial sums
                spa[j] += __shfl_xor_sync(0xffffffffu, spa[j], 1);
                spa[j] += __shfl_xor_sync(0xffffffffu, spa[j], 2);
            }
#pragma unroll
            for (int j = 0; j < J; ++j) {
                const int64_t mt = m0 + warp * PXW + j * 8 + ps;
                if (mt < p.M) {
                    int64_t pix0;
                    const int64_t m = pixel_of(p, mt, pix0);
                    const int64_t pz = -e.zp2 * (int64_t)spa[j];
                    float *dst = p.out + m * p.cout + cb;
#pragma unroll
                    for (int hq = 0; hq < 2; ++hq) {
                        int64_t A[4];
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const uint32_t hi = acc_hi[j][2 * hq + h];
                            const uint32_t lo = acc_all[j][2 * hq + h] - (hi << 16);
                            A[2 * h] = (int64_t)lo - bias_units;
                            A[2 * h + 1] = (int64_t)hi - bias_units;
                        }
                        const int c0 = cb + 4 * hq;
                        if (full_blk) {
                            float y[4];
#pragma unroll
                            for (int t = 0; t < 4; ++t) {
                                const int64_t corr = A[t] + pz - e.zp1 * __ldg(p.fsum + c0 + t) + e.kzz;
                                y[t] = __double2float_rn(e.scale * __ll2double_rn(corr));
                                if (p.bias) y[t] = __fadd_rn(y[t], __ldg(p.bias + c0 + t));
                            }
                            if (p.residual) {
                                const float4 r = __ldg(reinterpret_cast<const float4 *>(p.residual + m * p.cout + c0));
                                y[0] = __fadd_rn(y[0], r.x); y[1] = __fadd_rn(y[1], r.y);
                                y[2] = __fadd_rn(y[2], r.z); y[3] = __fadd_rn(y[3], r.w);
                            }
#pragma unroll
                            for (int t = 0; t < 4; ++t) {
                                if (p.relu) y[t] = (y[t] > 0.0f || y[t] != y[t]) ? y[t] : 0.0f;
                                track(y[t], tmin, tmax, nonfinite);
                            }
                            *reinterpret_cast<float4 *>(dst + 4 * hq) = make_float4(y[0], y[1], y[2], y[3]);
                            if (p.acc_out) {
#pragma unroll
                                for (int t = 0; t < 4; ++t) p.acc_out[m * p.cout + c0 + t] = A[t];
                            }
                        } else {
#pragma unroll
                            for (int t = 0; t < 4; ++t) {
                                if (c0 + t < p.cout) {
                                    const int64_t corr = A[t] + pz - e.zp1 * p.fsum[c0 + t] + e.kzz;
                                    float v = __double2float_rn(e.scale * __ll2double_rn(corr));
                                    if (p.bias) v = __fadd_rn(v, p.bias[c0 + t]);
                                    if (p.residual) v = __fadd_rn(v, p.residual[m * p.cout + c0 + t]);
                                    if (p.relu) v = (v > 0.0f || v != v) ? v : 0.0f;
                                    track(v, tmin, tmax, nonfinite);
                                    dst[4 * hq + t] = v;
                                    if (p.acc_out) p.acc_out[m * p.cout + c0 + t] = A[t];
                                }
                            }
                        }
                    }
                }
                spa[j] = 0;
#pragma unroll
                for (int r = 0; r < 4; ++r) acc_all[j][r] = acc_hi[j][r] = 0;
            }
        }
        c_tile += grid;
    }
    const bool any = tmin <= tmax;
    range_commit(any ? f2ord(tmin) : INT32_MAX, any ? f2ord(tmax) : INT32_MIN, nonfinite, p.out_range, p.flags,
                 AXB_FLAG_OUT_NONFINITE);
}

// ---------------------------------------------------------------- CX family (lutconv_cx): c64 / c32 / c16
// Same products, laid out CX[blk][k][a][32 words]: at 64-channel blocks (C64) the 64 channels of block
// blk at row k and activation code a are 128 contiguous bytes = all 32 banks.  Lanes = (pixel slot
// ps = lane / 8, octant o = lane % 8): one LDS.128 at a*128 + o*16 returns 4 pairs (8 products) of one
// pixel, and the 8 lanes of a quarter-warp -- the unit the shared memory serves a 128-bit request in --
// are ONE pixel reading one whole 128-byte row: every quarter is one wavefront whatever the codes are.
// A warp instruction = 4 pixels x 64 channels = 256 products in exactly 4 wavefronts, the shared-memory
// peak (64 products per wavefront), with no data-dependent bank conflicts (the pair-major and 32-channel
// layouts lose 30-50% of their wavefronts to conflicts on real activations).  Narrower blocks (32 / 16
// channels) repeat the block's words across the 128-byte row (below).
// Registers: a lane holds 8 accumulator words per pixel (J pixels), so the activation codes do not live
// in registers ahead of use: each warp stages its PXW pixels' next 16-row chunk in its own shared buffer
// with cp.async (lane L copies pixels L, L+32, ...: 16 bytes each), lanes read CR rows per pixel (LDS.64
// for CR = 8, LDS.32 for CR = 4 -- half the code registers, what lets J = 16..20 fit), and lane L sums
// its staged pixels' codes (S_p, DP4A) -- shuffled to the pixel's lanes in the epilogue.
// Table staging: 512 / BM bytes per product at 64-channel blocks (32 KiB per row and block, read once per
// BM-pixel tile), moved by TMA into a 3-slot ring of 2-row stages; BM is as large as the register file
// allows (J = 16 / 20 at 8 consumer warps: 1.0 / 0.8 B per product).  A producer warpgroup (PW = 1)
// refills a slot as soon as the last consumer released it; the last partial wave of tiles is cut into K
// pieces (tail split, launch_cx); kpad <= kCxMaxK keeps the epilogue's correction exact in 32 bits.
constexpr int kCxMaxK = 8192;  // CX kernels: the 32-bit epilogue correction is exact up to this K
constexpr int kC64Pairs = 32;                   // channel pairs per 64-channel block
constexpr int kC64RowWords = 256 * kC64Pairs;   // one (block, row) slice: 256 codes x 32 pairs
constexpr int kC64RowBytes = kC64RowWords * 4;  // 32 KiB
__host__ __device__ constexpr int c64_stage_bytes(int KS) { return KS * kC64RowBytes; }
// CB < 64 (the CX layouts): a code's CB channels (2*CB bytes) are stored 64/CB times side by side, so the
// row is still 128 bytes; a pixel takes CB/8 lanes and the copy (pixel slot % copies) no other pixel of
// its quarter-warp reads -- conflict-free for any codes at every channel width.  Pixels per warp
// instruction PPI = 256 / CB.
__host__ __device__ constexpr int cx_ppi(int CB) { return 256 / CB; }
__host__ __device__ constexpr int c64_codebuf_bytes(int WARPS, int J, int CB = 64) { return WARPS * 2 * cx_ppi(CB) * J * 16; }
__host__ __device__ constexpr int c64_smem(int KS, int ST, int WARPS, int J, int CB = 64) {
    return ST * c64_stage_bytes(KS) + c64_codebuf_bytes(WARPS, J, CB) + kMaxTaps * 4 + 2 * ST * 8 + 16;
}
// tail-split workspace: 32-bit words per thread for one piece's partial sums (acc_all, acc_hi, S_p)
__host__ __device__ constexpr int c64_split_words(int J, int CB = 64) { return 8 * J + (cx_ppi(CB) * J + 31) / 32; }

// PW = 1: an extra warpgroup whose first thread is the TMA producer (it refills a slot the moment the
// last consumer warp released it); it gives its registers to the consumers (setmaxnreg).  PW = 0: thread 0
// refills the previous stage's slot at the start of each stage.
template <int J, int WARPS, int KS, int ST, bool SGN, int CR, int PW, int CB>
__global__ void __launch_bounds__(WARPS * 32 + PW * 128, 1) lutconv_cx(const ConvK p) {
    constexpr int NT = WARPS * 32;  // consumer threads
    constexpr int LPP = CB / 8;       // lanes per pixel (8 channels = 4 pairs each)
    constexpr int PPI = cx_ppi(CB);   // pixels per warp instruction
    constexpr int RCP = 64 / CB;      // copies of a code's channels in its 128-byte row
    constexpr int PXW = PPI * J;      // pixels per warp
    constexpr int NPL = (PXW + 31) / 32;  // pixels whose codes each lane stages (the last slot may be partial)
    constexpr int BM = WARPS * PXW;
    constexpr int BN = CB;
    constexpr int SPG = CR / KS;      // stages per CR-row code group
    constexpr int NG = 16 / CR;       // code groups per 16-row chunk
    constexpr int SPCH = 16 / KS;     // stages per 16-row chunk
    constexpr int CBW = PXW * 16;     // one of a warp's two code buffers (bytes)
    constexpr int WPT = c64_split_words(J, CB);
    static_assert(CB == 16 || CB == 32 || CB == 64, "channel block of 16, 32 or 64");
    constexpr uint32_t STAGE_BYTES = c64_stage_bytes(KS);
    static_assert(PXW % 16 == 0, "whole 16-pixel groups per warp (J = 8, 12, 16, 20, ...)");
    static_assert(CR == 4 || CR == 8, "code rows per register load: 4 (LDS.32) or 8 (LDS.64)");
    static_assert(KS == 1 || KS == 2 || KS == 4, "KS rows per stage: 1, 2 or 4");
    static_assert(CR % KS == 0, "a stage never straddles two code groups");
    static_assert(c64_smem(KS, ST, WARPS, J, CB) + 512 <= 232448, "C64 ring exceeds shared memory");

    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t *codebuf = smem + ST * STAGE_BYTES;  // [warp][2][PXW pixels][16 B]
    int32_t *tapoff_s = reinterpret_cast<int32_t *>(codebuf + c64_codebuf_bytes(WARPS, J, CB));
    uint64_t *full = reinterpret_cast<uint64_t *>(tapoff_s + kMaxTaps);
    uint64_t *empty = full + ST;
    int32_t *last_s = reinterpret_cast<int32_t *>(empty + ST);  // tail split: "this CTA reduces the tile"

    const int tid = (int)threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const int o = lane % LPP, ps = lane / LPP;  // channel octet, pixel slot of the warp instruction

    if (tid == 0) {
        for (int s = 0; s < ST; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, WARPS);
        }
    }
    for (int t = tid; t < p.taps; t += (int)blockDim.x) tapoff_s[t] = ((t / p.kw) * p.dh * p.wp + (t % p.kw) * p.dw) * p.cs;
    __syncthreads();

    // ---- work items (32-bit loop state throughout: registers are the budget here; the host guarantees
    // ntiles * stages-per-tile < 2^31).  Items 0 .. n_full-1: whole tiles cid, cid+grid, ... of the first
    // T - L tiles (channel-block-major, so concurrently running CTAs share one block's table rows in L2);
    // then the tail: pieces i = cid, cid+grid, ... of the last L tiles x S chunk ranges, piece-major
    // (i = piece * L + tile), so concurrent CTAs again read the same table rows.
    const int grid = (int)gridDim.x;
    const int cid = (int)blockIdx.x;
    const int T = (int)p.ntiles;
    const int L = p.split_s > 1 ? p.split_L : 0;
    const int S = p.split_s > 1 ? p.split_s : 1;
    const int Tfull = T - L;
    const int n_full = Tfull > cid ? (Tfull - cid + grid - 1) / grid : 0;
    const int n_items = n_full + (L * S > cid ? (L * S - cid + grid - 1) / grid : 0);
    // item k -> tile, chunk range [kcb, kce), piece (-1: whole tile)
    auto item = [&](int k, int &tile, int &kcb, int &kce, int &pc) {
        if (k < n_full) {
            tile = cid + k * grid;
            kcb = 0;
            kce = p.nchunks;
            pc = -1;
        } else {
            const int i = cid + (k - n_full) * grid;
            pc = i / L;
            tile = Tfull + (i - pc * L);
            kcb = pc * p.nchunks / S;
            kce = (pc + 1) * p.nchunks / S;
        }
    };

    // ---- producer (thread 0): stage -> KS rows [pr_q*KS, +KS) of channel block pr_nb
    int pr_k = 0, pr_q = 0, pr_qe = 0, pr_nb = 0, pr_slot = 0;
    auto pr_item = [&]() {
        int t, b, e, pc;
        item(pr_k, t, b, e, pc);
        pr_q = b * SPCH;
        pr_qe = e * SPCH;
        pr_nb = t / p.ntm;
    };
    auto produce = [&]() {  // requires pr_k < n_items
        mbar_expect_tx(full + pr_slot, STAGE_BYTES);
        bulk_g2s(smem + pr_slot * STAGE_BYTES,
                 p.ftable + ((int64_t)pr_nb * p.kpad + pr_q * KS) * kC64RowWords, STAGE_BYTES, full + pr_slot);
        if (++pr_slot == ST) pr_slot = 0;
        if (++pr_q == pr_qe && ++pr_k < n_items) pr_item();
    };
    if (!PW && tid == 0 && n_items > 0) {
        pr_item();
        for (int s = 0; s < ST - 1 && pr_k < n_items; ++s) produce();
    }
    auto consumers_sync = [&]() {
        if constexpr (PW) asm volatile("bar.sync 1, %0;\n" ::"n"(NT) : "memory");
        else __syncthreads();
    };

    // ---- code loader: lane L stages pixels L, L+32, ... (of this warp's PXW) one 16-row chunk ahead
    uint8_t *wbuf = codebuf + warp * (2 * CBW);
    int32_t rowbase[NPL];  // byte offset of each staged pixel in the zp-padded code tensor
    auto set_row = [&](int tile) {
#pragma unroll
        for (int i = 0; i < NPL; ++i) {
            const int64_t mt = (int64_t)(tile % p.ntm) * BM + warp * PXW + lane + 32 * i;
            int64_t pix0 = 0;
            if (mt < p.M) pixel_of(p, mt, pix0);
            rowbase[i] = (int32_t)(pix0 * p.cs);
        }
    };
    pdl_wait();
    int ld_k = 0, ld_kc = 0, ld_ke = 0, ld_t = 0, ld_ci = 0, ld_buf = 0;
    auto ld_item = [&]() {
        int t, b, e, pc;
        item(ld_k, t, b, e, pc);
        const int cpt = p.cs >> 4;  // chunks per tap
        ld_kc = b;
        ld_ke = e;
        ld_t = b / cpt;
        ld_ci = (b - ld_t * cpt) * 16;
        set_row(t);
    };
    auto load_next = [&]() {
        if (ld_k < n_items) {
            const int off = tapoff_s[ld_t] + ld_ci;
#pragma unroll
            for (int i = 0; i < NPL; ++i)
                if (PXW % 32 == 0 || lane + 32 * i < PXW)
                    cp_async16(wbuf + ld_buf * CBW + (lane + 32 * i) * 16, p.codes + rowbase[i] + off, 16);
            ld_ci += 16;
            if (ld_ci == p.cs) {
                ld_ci = 0;
                ++ld_t;
            }
            if (++ld_kc == ld_ke && ++ld_k < n_items) ld_item();
        }
        ld_buf ^= 1;
        cp_async_commit();  // one group per chunk (possibly empty), so wait_group<1> tracks chunk c
    };

    uint32_t acc_all[J][4], acc_hi[J][4];
#pragma unroll
    for (int j = 0; j < J; ++j)
#pragma unroll
        for (int r = 0; r < 4; ++r) acc_all[j][r] = acc_hi[j][r] = 0;
    int32_t spl[NPL];  // S_p of lane L's staged pixels
#pragma unroll
    for (int i = 0; i < NPL; ++i) spl[i] = 0;
    float tmin = INFINITY, tmax = -INFINITY;
    int nonfinite = 0;
    const int64_t bias_units = SGN ? (int64_t)32768 * p.kpad : 0;

    int g = 0, slot = 0;
    uint32_t phase = 0;
    int cbuf = 0;
    if constexpr (PW) {
        static_assert(WARPS % 4 == 0, "consumer warpgroups");
        if (warp >= WARPS) asm volatile("setmaxnreg.dec.sync.aligned.u32 24;\n" ::: "memory");
        else asm volatile("setmaxnreg.inc.sync.aligned.u32 240;\n" ::: "memory");
    }
    if (PW && warp >= WARPS) {
        // ---- dedicated producer: stage h goes into slot h % ST once the consumers released stage h - ST
        if (warp == WARPS && lane == 0 && n_items > 0) {
            pr_item();
            for (int h = 0; pr_k < n_items; ++h) {
                if (h >= ST) mbar_wait_sleep(empty + pr_slot, (uint32_t)((h / ST) - 1) & 1u);
                produce();
            }
        }
    } else {
    if (n_items > 0) {
        ld_item();
        load_next();
    }
    const uint8_t *tab_lane = smem + (ps % RCP) * (2 * CB) + o * 16;
    for (int kk = 0; kk < n_items; ++kk) {
        int c_tile, kcb, kce, pc;
        item(kk, c_tile, kcb, kce, pc);
#pragma unroll 1
        for (int kc = kcb; kc < kce; ++kc) {
            __syncwarp();   // every lane is done reading the buffer the next copy overwrites
            load_next();    // chunk kc+1 -> the other buffer
            cp_async_wait<1>();
            __syncwarp();   // chunk kc of all PXW pixels has landed
            const uint8_t *cb_ = wbuf + cbuf * CBW;
#pragma unroll
            for (int i = 0; i < NPL; ++i) {  // S_p of the staged pixels (axconv.py:193; junk codes are raw 0)
                if (PXW % 32 != 0 && lane + 32 * i >= PXW) continue;
                const uint4 mine = *reinterpret_cast<const uint4 *>(cb_ + (lane + 32 * i) * 16);
                if (SGN) {
                    spl[i] = __dp4a((int)mine.x, 0x01010101, spl[i]);
                    spl[i] = __dp4a((int)mine.y, 0x01010101, spl[i]);
                    spl[i] = __dp4a((int)mine.z, 0x01010101, spl[i]);
                    spl[i] = __dp4a((int)mine.w, 0x01010101, spl[i]);
                } else {
                    uint32_t t = __dp4a(mine.x, 0x01010101u, (uint32_t)spl[i]);
                    t = __dp4a(mine.y, 0x01010101u, t);
                    t = __dp4a(mine.z, 0x01010101u, t);
                    spl[i] = (int32_t)__dp4a(mine.w, 0x01010101u, t);
                }
            }
#pragma unroll 1
            for (int gr = 0; gr < NG; ++gr) {
                uint32_t cur[J][CR / 4];
#pragma unroll
                for (int j = 0; j < J; ++j) {
                    const uint8_t *src = cb_ + (j * PPI + ps) * 16 + gr * CR;
                    if (CR == 8) {
                        const uint2 v = *reinterpret_cast<const uint2 *>(src);
                        cur[j][0] = v.x;
                        cur[j][CR / 4 - 1] = v.y;
                    } else {
                        cur[j][0] = *reinterpret_cast<const uint32_t *>(src);
                    }
                }
#pragma unroll
                for (int st = 0; st < SPG; ++st) {
#ifndef AXB_EXP_C64_NOREFILL
                    if (!PW && tid == 0 && pr_k < n_items) {
                        // refill the slot stage g-1 used once every warp released it
                        if (g >= 1) {
                            const int ps_ = slot == 0 ? ST - 1 : slot - 1;
                            const uint32_t ph_ = slot == 0 ? phase ^ 1u : phase;
                            mbar_wait(empty + ps_, ph_);
                        }
                        produce();
                    }
                    mbar_wait_sleep(full + slot, phase);
#else  // A/B experiment only (wrong products): the first ST-1 stages are loaded once and never refilled
                    if (g < ST - 1) mbar_wait(full + slot, phase);
#endif
                    const uint8_t *stab = tab_lane + slot * STAGE_BYTES;
#pragma unroll
                    for (int kl = 0; kl < KS; ++kl) {
                        const int r = st * KS + kl;  // row within the code group (compile-time)
#pragma unroll
                        for (int j = 0; j < J; ++j) {
                            const uint32_t a = __byte_perm(cur[j][r >> 2], 0, 0x4440u + (r & 3));
                            const uint4 w = *reinterpret_cast<const uint4 *>(stab + kl * kC64RowBytes + a * 128u);
                            acc_all[j][0] += w.x; acc_hi[j][0] += w.x >> 16;
                            acc_all[j][1] += w.y; acc_hi[j][1] += w.y >> 16;
                            acc_all[j][2] += w.z; acc_hi[j][2] += w.z >> 16;
                            acc_all[j][3] += w.w; acc_hi[j][3] += w.w >> 16;
                        }
                    }
                    fence_proxy_async_smem();  // this lane's LDS reads of the slot before the TMA refill
                    __syncwarp();
                    if (lane == 0) mbar_arrive(empty + slot);
                    ++g;
                    if (++slot == ST) {
                        slot = 0;
                        phase ^= 1u;
                    }
                }
            }
            cbuf ^= 1;
        }

        if (pc >= 0) {
            // ---- tail split: publish this piece's partial sums; the last piece to arrive adds the
            // others and runs the epilogue (exact: all/S_p mod 2^32, hi < 2^32 for kpad <= 65536)
            const int ti = c_tile - Tfull;
            uint32_t *mine = p.split_ws + ((int64_t)ti * S + pc) * (WPT * NT) + tid;
#pragma unroll
            for (int j = 0; j < J; ++j)
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    mine[(8 * j + r) * NT] = acc_all[j][r];
                    mine[(8 * j + 4 + r) * NT] = acc_hi[j][r];
                }
#pragma unroll
            for (int i = 0; i < NPL; ++i) mine[(8 * J + i) * NT] = (uint32_t)spl[i];
            __threadfence();
            consumers_sync();
            if (tid == 0) {
                const int last = atomicAdd(p.split_cnt + ti, 1) == S - 1;
                if (last) p.split_cnt[ti] = 0;  // every piece arrived: ready for the next launch
                *last_s = last;
            }
            consumers_sync();
            const bool last = *last_s != 0;
            consumers_sync();  // everyone read the flag before a later item rewrites it
            if (!last) {
#pragma unroll
                for (int j = 0; j < J; ++j)
#pragma unroll
                    for (int r = 0; r < 4; ++r) acc_all[j][r] = acc_hi[j][r] = 0;
#pragma unroll
                for (int i = 0; i < NPL; ++i) spl[i] = 0;
                continue;
            }
            __threadfence();
            for (int q = 0; q < S; ++q) {
                if (q == pc) continue;
                const uint32_t *other = p.split_ws + ((int64_t)ti * S + q) * (WPT * NT) + tid;
#pragma unroll
                for (int j = 0; j < J; ++j)
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        acc_all[j][r] += __ldcg(other + (8 * j + r) * NT);
                        acc_hi[j][r] += __ldcg(other + (8 * j + 4 + r) * NT);
                    }
#pragma unroll
                for (int i = 0; i < NPL; ++i) spl[i] += (int32_t)__ldcg(other + (8 * J + i) * NT);
            }
        }

        // ------------------------------------------------ fused epilogue (same arithmetic as lutconv_ft)
        {
            const EpiConst e = epi_const(p);
            const int nb = c_tile / p.ntm;
            const int64_t m0 = (int64_t)(c_tile % p.ntm) * BM;
            const int cb = nb * BN + o * 8;  // this lane's 8 channels
            const bool full_blk = cb + 8 <= p.cout && (p.cout & 3) == 0;
            const bool has_res = p.residual != nullptr, relu = p.relu != 0;

            // per-channel terms hoisted out of the pixel loop: -zp1*S_f + K*zp1*zp2 - (entry bias), and the
            // bias (-0.0f when absent: x + -0 == x for every float, so the add is an exact identity)
            uint32_t cc[8];  // mod 2^32 (exact in the 32-bit correction below)
            float bv[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                const bool ok = full_blk || cb + t < p.cout;
                cc[t] = ok ? (uint32_t)(e.kzz - e.zp1 * __ldg(p.fsum + cb + t) - bias_units) : 0u;
                bv[t] = (ok && p.bias) ? __ldg(p.bias + cb + t) : -0.0f;
            }
#pragma unroll
            for (int j = 0; j < J; ++j) {
                const int32_t spj = __shfl_sync(0xffffffffu, spl[(j * PPI) >> 5], (j * PPI + ps) & 31);
                const int64_t mt = m0 + warp * PXW + j * PPI + ps;
                if (mt < p.M) {
                    int64_t pix0;
                    const int64_t m = pixel_of(p, mt, pix0);
                    const int64_t pz = -e.zp2 * (int64_t)spj;
                    float *dst = p.out + m * p.cout + cb;
                    // corr = A - zp2*S_p - zp1*S_f + K*zp1*zp2 (axconv.py:249-254), A = sum u - bias_units;
                    // fp64 dequant (:256), bias (graph.py:268-269), Add (:282-286), ReLU (:276-277)
                    // kpad <= 8192 (the launcher's limit for this kernel): every |corr| < 2^31 (|A| <= 32768 K,
                    // |zp*S| <= 255*255 K), so the correction is exact in 32-bit two's-complement arithmetic
                    // whatever the intermediate sums wrap to
                    float y[8];
                    const uint32_t pz32 = (uint32_t)pz;
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                        const uint32_t hi = acc_hi[j][h];
                        const uint32_t lo = acc_all[j][h] - (hi << 16);
                        const int32_t c0 = (int32_t)(lo + pz32 + cc[2 * h]);
                        const int32_t c1 = (int32_t)(hi + pz32 + cc[2 * h + 1]);
                        y[2 * h] = __fadd_rn(__double2float_rn(e.scale * (double)c0), bv[2 * h]);
                        y[2 * h + 1] = __fadd_rn(__double2float_rn(e.scale * (double)c1), bv[2 * h + 1]);
                    }
                    if (full_blk) {
                        if (has_res) {
                            const float4 r0 = __ldg(reinterpret_cast<const float4 *>(p.residual + m * p.cout + cb));
                            const float4 r1 = __ldg(reinterpret_cast<const float4 *>(p.residual + m * p.cout + cb + 4));
                            y[0] = __fadd_rn(y[0], r0.x); y[1] = __fadd_rn(y[1], r0.y);
                            y[2] = __fadd_rn(y[2], r0.z); y[3] = __fadd_rn(y[3], r0.w);
                            y[4] = __fadd_rn(y[4], r1.x); y[5] = __fadd_rn(y[5], r1.y);
                            y[6] = __fadd_rn(y[6], r1.z); y[7] = __fadd_rn(y[7], r1.w);
                        }
#pragma unroll
                        for (int t = 0; t < 8; ++t) {
                            if (relu) y[t] = (y[t] > 0.0f || y[t] != y[t]) ? y[t] : 0.0f;  // np.maximum(x, 0)
                            track(y[t], tmin, tmax, nonfinite);
                        }
                        *reinterpret_cast<float4 *>(dst) = make_float4(y[0], y[1], y[2], y[3]);
                        *reinterpret_cast<float4 *>(dst + 4) = make_float4(y[4], y[5], y[6], y[7]);
                    } else {
#pragma unroll
                        for (int t = 0; t < 8; ++t) {
                            if (cb + t < p.cout) {
                                float v = y[t];
                                if (has_res) v = __fadd_rn(v, p.residual[m * p.cout + cb + t]);
                                if (relu) v = (v > 0.0f || v != v) ? v : 0.0f;
                                track(v, tmin, tmax, nonfinite);
                                dst[t] = v;
                            }
                        }
                    }
                    if (p.acc_out) {
#pragma unroll
                        for (int h = 0; h < 4; ++h) {
                            const uint32_t hi = acc_hi[j][h];
                            const uint32_t lo = acc_all[j][h] - (hi << 16);
                            if (cb + 2 * h < p.cout) p.acc_out[m * p.cout + cb + 2 * h] = (int64_t)lo - bias_units;
                            if (cb + 2 * h + 1 < p.cout) p.acc_out[m * p.cout + cb + 2 * h + 1] = (int64_t)hi - bias_units;
                        }
                    }
                }
#pragma unroll
                for (int r = 0; r < 4; ++r) acc_all[j][r] = acc_hi[j][r] = 0;
            }
#pragma unroll
            for (int i = 0; i < NPL; ++i) spl[i] = 0;
        }
    }
    }  // consumers
    cp_async_wait<0>();

    const bool any = tmin <= tmax;
    range_commit(any ? f2ord(tmin) : INT32_MAX, any ? f2ord(tmax) : INT32_MIN, nonfinite, p.out_range, p.flags,
                 AXB_FLAG_OUT_NONFINITE);
}

// ---------------------------------------------------------------- table preparation
// W[sb][k][pair][a] = (u(lut[(a<<8)|F[k][c]]), u(lut[(a<<8)|F[k][c+1]])), c = sb*8 + 2*pair (8-channel
// sub-blocks); u = raw ^ 0x8000 (signed) / raw (unsigned); junk rows (ci >= c or k >= taps*cs) = zero
// contribution.
__global__ void ftable_kernel(const uint8_t *__restrict__ fcodes, int64_t kpad, int64_t coutp, int32_t cs, int32_t c,
                              int64_t kreal, const uint16_t *__restrict__ lut_b, int sgn, uint32_t *__restrict__ out) {
    const int64_t total = (coutp / 8) * kpad * kFtRowWords;
    const uint32_t flip = sgn ? 0x8000u : 0u;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t a = (uint32_t)(idx & 255);
        const int pr = (int)((idx >> 8) & 3);
        const int64_t rest = idx >> 10;
        const int64_t k = rest % kpad;
        const int64_t sb = rest / kpad;
        uint32_t w = flip | (flip << 16);  // zero contribution
        if (k < kreal && (int)(k % cs) < c) {
            const int64_t col = sb * 8 + 2 * pr;
            const uint32_t b0 = fcodes[k * coutp + col], b1 = fcodes[k * coutp + col + 1];
            const uint32_t u0 = (uint32_t)__ldg(lut_b + b0 * 256 + a) ^ flip;
            const uint32_t u1 = (uint32_t)__ldg(lut_b + b1 * 256 + a) ^ flip;
            w = u0 | (u1 << 16);
        }
        out[idx] = w;
    }
}

// CM[cb][k][a][pr] = W word of channels (cb*32 + 2*pr, +1) at row k, code a (the same words, code-major)
__global__ void ftable_cm_kernel(const uint8_t *__restrict__ fcodes, int64_t kpad, int64_t coutp, int32_t cs,
                                 int32_t c, int64_t kreal, const uint16_t *__restrict__ lut_b, int sgn,
                                 uint32_t *__restrict__ out) {
    const int64_t total = (coutp / 32) * kpad * kCmRowWords;
    const uint32_t flip = sgn ? 0x8000u : 0u;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int pr = (int)(idx & 15);
        const uint32_t a = (uint32_t)((idx >> 4) & 255);
        const int64_t rest = idx >> 12;
        const int64_t k = rest % kpad;
        const int64_t cb = rest / kpad;
        uint32_t w = flip | (flip << 16);
        if (k < kreal && (int)(k % cs) < c) {
            const int64_t col = cb * 32 + 2 * pr;
            const uint32_t b0 = fcodes[k * coutp + col], b1 = fcodes[k * coutp + col + 1];
            const uint32_t u0 = (uint32_t)__ldg(lut_b + b0 * 256 + a) ^ flip;
            const uint32_t u1 = (uint32_t)__ldg(lut_b + b1 * 256 + a) ^ flip;
            w = u0 | (u1 << 16);
        }
        out[idx] = w;
    }
}

// CX[blk][k][a][w] (w = 0..31 words, 128 B per code and row) = W word of channels (blk*CB + 2*pr, +1),
// pr = w % (CB/2): the CB channels of the block, repeated 64/CB times across the row (CB = 64: C64)
__global__ void ftable_c64_kernel(const uint8_t *__restrict__ fcodes, int64_t kpad, int64_t coutp, int32_t cs,
                                  int32_t c, int64_t kreal, const uint16_t *__restrict__ lut_b, int sgn,
                                  uint32_t *__restrict__ out, int32_t CB) {
    const int64_t total = (coutp / CB) * kpad * kC64RowWords;
    const uint32_t flip = sgn ? 0x8000u : 0u;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int pr = (int)(idx & 31) % (CB / 2);
        const uint32_t a = (uint32_t)((idx >> 5) & 255);
        const int64_t rest = idx >> 13;
        const int64_t k = rest % kpad;
        const int64_t cb = rest / kpad;
        uint32_t w = flip | (flip << 16);
        if (k < kreal && (int)(k % cs) < c) {
            const int64_t col = cb * CB + 2 * pr;
            const uint32_t b0 = fcodes[k * coutp + col], b1 = fcodes[k * coutp + col + 1];
            const uint32_t u0 = (uint32_t)__ldg(lut_b + b0 * 256 + a) ^ flip;
            const uint32_t u1 = (uint32_t)__ldg(lut_b + b1 * 256 + a) ^ flip;
            w = u0 | (u1 << 16);
        }
        out[idx] = w;
    }
}

// ---------------------------------------------------------------- host launch
struct FtVariant {
    const char *name;
    int tm, warps, npb, cl;
    float cost;  // relative time per lookup slot (1 = best); tuned on B200
    int cm;      // 1: code-major 32-channel table (axb_ftable_cm_prepare), tm = J pixels per lane per 8-pixel
                 // group; 2 / 3 / 4: CX table of 64 / 32 / 16-channel blocks (axb_ftable_cx_prepare), tm = J
};
static const FtVariant kFtVariants[] = {
    {"auto", 0, 0, 0, 0, 0.f},
    {"ft16_tm2_w16_k8", 2, 16, 8, 1, 1.000f},
    {"ft16_tm2_w16_k4", 2, 16, 8, 1, 1.105f},
    {"ft8_tm4_w16_k16", 4, 16, 4, 1, 1.139f},
    {"ft16_tm1_w16_k8", 1, 16, 8, 1, 1.095f},
    {"ft8_tm2_w16_k16", 2, 16, 4, 1, 1.127f},
    {"ft8_tm1_w8_k16", 1, 8, 4, 1, 1.556f},
    {"ft16_tm2_w16_k8_c2", 2, 16, 8, 2, 1.219f},
    {"ft16_tm2_w12_k8", 2, 12, 8, 1, 1.050f},
    {"ft16_tm3_w12_k8", 3, 12, 8, 1, 1.000f},
    {"ft16_tm4_w12_k8", 4, 12, 8, 1, 1.000f},
    {"cm32_j4_w16_k4", 4, 16, 16, 1, 1.000f, 1},
    {"cm32_j8_w8_k4", 8, 8, 16, 1, 1.000f, 1},
    {"cm32_j4_w12_k4", 4, 12, 16, 1, 1.000f, 1},
    {"cm32_j6_w16_k4", 6, 16, 16, 1, 1.000f, 1},
    {"c64_j8_w12_k2", 8, 12, 32, 1, 1.000f, 2},
    {"c64_j16_w8_k2", 16, 8, 32, 1, 1.000f, 2},
    {"c64_j16_w8_k2_pw", 16, 8, 32, 1, 1.000f, 2},
    {"c64_j16_w8_k2_pw_c4", 16, 8, 32, 1, 1.000f, 2},
    {"c64_j20_w8_k2_pw_c4", 20, 8, 32, 1, 1.000f, 2},
    {"c32_j16_w8_k2_pw_c4", 16, 8, 16, 1, 1.000f, 3},
    {"c32_j8_w8_k2_pw_c4", 8, 8, 16, 1, 1.000f, 3},
    {"c16_j16_w8_k2_s2_pw_c4", 16, 8, 8, 1, 1.000f, 4},
    {"c16_j8_w8_k2_pw_c4", 8, 8, 8, 1, 1.000f, 4},
    {"c16_j2_w8_k2_pw_c4", 2, 8, 8, 1, 1.000f, 4},
    {"c32_j4_w8_k2_pw_c4", 4, 8, 16, 1, 1.000f, 3},
};
constexpr int kNumFtVariants = sizeof(kFtVariants) / sizeof(kFtVariants[0]);

template <int J, int WARPS, bool SGN, int PF = 1, int KS = 4, int ST = 3>
static int launch_ftcm(int op, const ConvK &k, int sm_limit, cudaStream_t s, const char *name) {
    constexpr int BM = WARPS * 8 * J;
    constexpr int BN = 32;
    const size_t smem = cm_smem(KS, ST);
    auto fn = lutconv_ftcm<J, WARPS, KS, ST, SGN, PF>;
    static int configured_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (configured_dev != dev) {
        if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return set_error(AXB_E_CUDA, "cannot raise dynamic shared memory for lutconv_ftcm");
        configured_dev = dev;
    }
    if (op == 1) return sm_count();
    if (k.coutp % BN) return set_error(AXB_E_VALUE, "code-major ftable kernel needs coutp % 32 == 0");
    ConvK kk = k;
    kk.ntm = (int32_t)((k.M + BM - 1) / BM);
    kk.ntiles = (int64_t)kk.ntm * (k.coutp / BN);
    int64_t nblk = sm_limit > 0 ? sm_limit : sm_count();
    if (nblk > kk.ntiles) nblk = kk.ntiles;
    if (nblk < 1) nblk = 1;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.gridDim = dim3((unsigned)nblk);
    cfg.blockDim = dim3(WARPS * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, fn, kk) != cudaSuccess) return check_launch("lutconv_ftcm");
    set_last_kernel(name);
    return check_launch("lutconv_ftcm");
}

// Tail split plan for a persistent grid of G CTAs over T whole tiles of nch 16-row chunks: the last L tiles
// (the partial wave, optionally plus one full wave) are cut into s chunk-aligned K pieces dealt over all
// CTAs, minimising the finishing time in tile units: (T - L) / G + ceil(L * s / G) / s (+2% per extra
// piece round for the partial-sum traffic).  L = 0: no split.
static void tail_split_plan(int64_t T, int64_t G, int nch, int &L, int &S) {
    L = 0;
    S = 1;
    if (T <= 0 || G <= 1) return;
    const int64_t r = T % G;
    if (r == 0) return;
    double best = (double)((T + G - 1) / G);
    for (int m = 0; m <= 1; ++m) {
        const int64_t Lc = r + m * G;
        if (Lc > T) break;
        for (int sc = 2; sc <= 8 && sc <= nch; ++sc) {
            const int64_t rounds = (Lc * sc + G - 1) / G;
            const double t = (double)((T - Lc) / G) + (double)rounds / sc + 0.02 * rounds;
            if (t < best - 1e-9) {
                best = t;
                L = (int)Lc;
                S = sc;
            }
        }
    }
}
// stream-ordered scratch comes from the device's default pool; keep freed blocks in the pool (no release
// to the OS at every synchronisation) so per-launch workspaces cost no driver allocation
static void keep_pool_memory(int dev) {
    static int done_mask = 0;
    if (dev < 0 || dev >= 31 || (done_mask >> dev) & 1) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
    done_mask |= 1 << dev;
}
static bool c64_split_enabled() {
    static const int on = [] {
        const char *e = getenv("AXB_C64_SPLIT");
        return (e && e[0] == '0') ? 0 : 1;
    }();
    return on != 0;
}

template <int J, int WARPS, bool SGN, int KS = 2, int ST = 3, int CR = 8, int PW = 0, int CB = 64>
static int launch_cx(int op, const ConvK &k, int sm_limit, cudaStream_t s, const char *name) {
    constexpr int BM = WARPS * cx_ppi(CB) * J;
    constexpr int BN = CB;
    const size_t smem = c64_smem(KS, ST, WARPS, J, CB);
    auto fn = lutconv_cx<J, WARPS, KS, ST, SGN, CR, PW, CB>;
    static int configured_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (configured_dev != dev) {
        if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return set_error(AXB_E_CUDA, "cannot raise dynamic shared memory for lutconv_cx");
        configured_dev = dev;
    }
    if (op == 1) return sm_count();
    if (k.coutp % BN) return set_error(AXB_E_VALUE, "code-major kernel needs coutp % its channel block == 0");
    if (k.kpad > kCxMaxK) return set_error(AXB_E_VALUE, "CX kernel: K > 8192 (its epilogue corrections are 32-bit)");
    ConvK kk = k;
    kk.ntm = (int32_t)((k.M + BM - 1) / BM);
    kk.ntiles = (int64_t)kk.ntm * (k.coutp / BN);
    if (kk.ntiles * (int64_t)k.nchunks * (16 / KS) >= (int64_t)1 << 31)
        return set_error(AXB_E_VALUE, "conv too large for the c64 kernel's 32-bit stage counters");
    int64_t nblk = sm_limit > 0 ? sm_limit : sm_count();
    if (nblk > kk.ntiles) nblk = kk.ntiles;
    if (nblk < 1) nblk = 1;
    // tail split: cut the last wave's tiles into K pieces so every CTA ends at about the same time
    int split_L = 0, split_s = 1;
    if (c64_split_enabled()) tail_split_plan(kk.ntiles, nblk, k.nchunks, split_L, split_s);
    kk.split_L = split_L;
    kk.split_s = split_s;
    void *ws = nullptr;
    const size_t ws_bytes = (size_t)split_L * split_s * (WARPS * 32) * c64_split_words(J, CB) * 4;
    const size_t cnt_bytes = (size_t)split_L * 4;
    if (split_s > 1) {
        keep_pool_memory(dev);
        if (cudaMallocAsync(&ws, ws_bytes + cnt_bytes, s) != cudaSuccess) {
            cudaGetLastError();  // no workspace: run without the split (same results, a ragged last wave)
            ws = nullptr;
            kk.split_L = 0;
            kk.split_s = 1;
        }
    }
    if (ws) {
        kk.split_ws = static_cast<uint32_t *>(ws);
        kk.split_cnt = reinterpret_cast<int32_t *>(static_cast<uint8_t *>(ws) + ws_bytes);
        if (cudaMemsetAsync(kk.split_cnt, 0, cnt_bytes, s) != cudaSuccess) {
            cudaFreeAsync(ws, s);
            return set_error(AXB_E_CUDA, "cannot clear the c64 tail-split counters");
        }
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.gridDim = dim3((unsigned)nblk);
    cfg.blockDim = dim3(WARPS * 32 + PW * 128);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = ws ? 0 : 1;  // PDL only without the memset in between
    const cudaError_t le = cudaLaunchKernelEx(&cfg, fn, kk);
    if (ws) cudaFreeAsync(ws, s);
    if (le != cudaSuccess) return check_launch("lutconv_cx");
    set_last_kernel(name);
    return check_launch("lutconv_cx");
}

// op 0: launch; op 1: return how many CL-CTA clusters fit on the device at once (cached)
template <int TM, int WARPS, int NPB, bool SGN, int CL, int KS = 4, int ST = 6, int PF = 1>
static int launch_ft(int op, const ConvK &k, int sm_limit, cudaStream_t s, const char *name) {
    constexpr int BM = WARPS * 32 * TM;
    constexpr int BN = 2 * NPB;
    const size_t smem = ft_smem(NPB, KS, ST);
    auto fn = lutconv_ft<TM, WARPS, NPB, KS, ST, SGN, CL, PF>;
    static int configured_dev = -1, max_clusters = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL (pdl_wait in the kernel)
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = CL;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.blockDim = dim3(WARPS * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = CL > 1 ? 2 : 1;
    if (configured_dev != dev) {
        if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return set_error(AXB_E_CUDA, "cannot raise dynamic shared memory for lutconv_ft");
        max_clusters = sm_count();
        if (CL > 1) {
            cfg.gridDim = dim3(CL * (sm_count() / CL));
            int n = 0;
            if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess || n < 1) {
                cudaGetLastError();
                return set_error(AXB_E_CUDA, "no resident CTA cluster for lutconv_ft");
            }
            max_clusters = n;
        }
        configured_dev = dev;
    }
    if (op == 1) return max_clusters;
    ConvK kk = k;
    const int64_t ntm = (k.M + BM - 1) / BM;
    kk.ntm = (int32_t)((ntm + CL - 1) / CL);             // pixel-tile groups per channel block
    kk.ntiles = (int64_t)kk.ntm * (k.coutp / BN);          // super-tiles
    int64_t ncl = sm_limit > 0 ? (sm_limit / CL > 0 ? sm_limit / CL : 1) : max_clusters;
    if (ncl > max_clusters) ncl = max_clusters;
    if (ncl > kk.ntiles) ncl = kk.ntiles;
    if (ncl < 1) ncl = 1;
    cfg.gridDim = dim3((unsigned)(ncl * CL));
    if (cudaLaunchKernelEx(&cfg, fn, kk) != cudaSuccess) return check_launch("lutconv_ft");
    set_last_kernel(name);
    return check_launch("lutconv_ft");
}

template <bool SGN>
static int launch_ft_variant(int op, int v, const ConvK &k, int sm_limit, cudaStream_t s) {
    const char *nm = kFtVariants[v].name;
    switch (v) {
        case 1: return launch_ft<2, 16, 8, SGN, 1, 8, 3>(op, k, sm_limit, s, nm);
        case 2: return launch_ft<2, 16, 8, SGN, 1, 4, 6>(op, k, sm_limit, s, nm);
        case 3: return launch_ft<4, 16, 4, SGN, 1, 16, 3>(op, k, sm_limit, s, nm);
        case 4: return launch_ft<1, 16, 8, SGN, 1, 8, 3>(op, k, sm_limit, s, nm);
        case 5: return launch_ft<2, 16, 4, SGN, 1, 16, 3>(op, k, sm_limit, s, nm);
        case 6: return launch_ft<1, 8, 4, SGN, 1, 16, 3>(op, k, sm_limit, s, nm);
        case 7: return launch_ft<2, 16, 8, SGN, 2, 8, 3>(op, k, sm_limit, s, nm);
        case 8: return launch_ft<2, 12, 8, SGN, 1, 8, 3>(op, k, sm_limit, s, nm);
        case 9: return launch_ft<3, 12, 8, SGN, 1, 8, 3>(op, k, sm_limit, s, nm);
        case 10: return launch_ft<4, 12, 8, SGN, 1, 8, 3>(op, k, sm_limit, s, nm);
        case 11: return launch_ftcm<4, 16, SGN, 2>(op, k, sm_limit, s, nm);  // codes 2 chunks ahead
        case 12: return launch_ftcm<8, 8, SGN>(op, k, sm_limit, s, nm);
        case 13: return launch_ftcm<4, 12, SGN>(op, k, sm_limit, s, nm);
        case 14: return launch_ftcm<6, 16, SGN>(op, k, sm_limit, s, nm);
        case 15: return launch_cx<8, 12, SGN>(op, k, sm_limit, s, nm);
        case 16: return launch_cx<16, 8, SGN, 2, 3, 8>(op, k, sm_limit, s, nm);
        case 17: return launch_cx<16, 8, SGN, 2, 3, 8, 1>(op, k, sm_limit, s, nm);
        case 18: return launch_cx<16, 8, SGN, 2, 3, 4, 1>(op, k, sm_limit, s, nm);
        case 19: return launch_cx<20, 8, SGN, 2, 3, 4, 1>(op, k, sm_limit, s, nm);
        case 20: return launch_cx<16, 8, SGN, 2, 3, 4, 1, 32>(op, k, sm_limit, s, nm);
        case 21: return launch_cx<8, 8, SGN, 2, 3, 4, 1, 32>(op, k, sm_limit, s, nm);
        case 22: return launch_cx<16, 8, SGN, 2, 2, 4, 1, 16>(op, k, sm_limit, s, nm);
        case 23: return launch_cx<8, 8, SGN, 2, 3, 4, 1, 16>(op, k, sm_limit, s, nm);
        case 24: return launch_cx<2, 8, SGN, 2, 3, 4, 1, 16>(op, k, sm_limit, s, nm);  // BM = 256: small M (fc)
        case 25: return launch_cx<4, 8, SGN, 2, 3, 4, 1, 32>(op, k, sm_limit, s, nm);  // BM = 256
        default: return set_error(AXB_E_VALUE, "unknown ftable kernel variant");
    }
}

// time ~ cost * waves * BM * BN, waves = ceil(super-tiles / resident clusters)
static int pick_ft_variant(const ConvK &k, int is_signed) {
    int best = 1;
    double best_t = 1e300;
    for (int v = 1; v < kNumFtVariants; ++v) {
        const FtVariant &x = kFtVariants[v];
        if (x.cm) continue;  // the cost model picks among pair-major variants (the table handed in)
        const int64_t ncl = is_signed ? launch_ft_variant<true>(1, v, k, 0, 0) : launch_ft_variant<false>(1, v, k, 0, 0);
        if (ncl < 1) continue;
        const int64_t bm = (int64_t)x.warps * 32 * x.tm, bn = 2 * x.npb;
        const int64_t ntm = (k.M + bm - 1) / bm;
        const int64_t tiles = ((ntm + x.cl - 1) / x.cl) * (k.coutp / bn);
        const int64_t waves = (tiles + ncl - 1) / ncl;
        const double t = (double)x.cost * (double)waves * (double)(bm * bn);
        if (t < best_t) {
            best_t = t;
            best = v;
        }
    }
    return best;
}

int conv_ft_launch(const ConvK &k, int variant, int is_signed, int sm_limit, cudaStream_t s) {
    int v = variant;
    if (v < 0 || v >= kNumFtVariants) return set_error(AXB_E_VALUE, "unknown ftable kernel variant");
    if (v == 0) v = pick_ft_variant(k, is_signed);
    return is_signed ? launch_ft_variant<true>(0, v, k, sm_limit, s) : launch_ft_variant<false>(0, v, k, sm_limit, s);
}

}  // namespace axb

using namespace axb;

extern "C" {

int64_t axb_ftable_bytes(int64_t kpad, int64_t coutp) {
    if (kpad <= 0 || coutp <= 0 || kpad % 16 || coutp % 16) return 0;
    return kpad * (coutp / 8) * kFtRowBytes;
}

int axb_ftable_prepare(const uint8_t *d_fcodes, int64_t kh, int64_t kw, int64_t c, int64_t cs, int64_t cout,
                       const axb_lut *lut, uint32_t *d_ftable, void *stream) {
    if (!lut || !d_fcodes || !d_ftable) return set_error(AXB_E_VALUE, "null argument");
    if (cs % 16 || c > cs || c < 1) return set_error(AXB_E_VALUE, "channel stride mismatch");
    const int64_t kpad = axb_filter_kpad(kh, kw, cs), coutp = axb_filter_coutp(cout);
    const int64_t total = (coutp / 8) * kpad * kFtRowWords;
    int64_t blocks = (total + 255) / 256;
    const int64_t cap = (int64_t)sm_count() * 16;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    ftable_kernel<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(d_fcodes, kpad, coutp, (int32_t)cs, (int32_t)c,
                                                                  kh * kw * cs, lut->d_bmajor, lut->is_signed,
                                                                  d_ftable);
    return check_launch("ftable_prepare");
}

int64_t axb_ftable_cm_bytes(int64_t kpad, int64_t coutp) {
    if (kpad <= 0 || coutp <= 0 || kpad % 16 || coutp % 32) return 0;
    return kpad * (coutp / 32) * kCmRowBytes;
}

int axb_ftable_cm_prepare(const uint8_t *d_fcodes, int64_t kh, int64_t kw, int64_t c, int64_t cs, int64_t cout,
                          const axb_lut *lut, uint32_t *d_ftable, void *stream) {
    if (!lut || !d_fcodes || !d_ftable) return set_error(AXB_E_VALUE, "null argument");
    if (cs % 16 || c > cs || c < 1) return set_error(AXB_E_VALUE, "channel stride mismatch");
    const int64_t kpad = axb_filter_kpad(kh, kw, cs), coutp = axb_filter_coutp(cout);
    if (coutp % 32) return set_error(AXB_E_VALUE, "code-major table needs coutp % 32 == 0");
    const int64_t total = (coutp / 32) * kpad * kCmRowWords;
    int64_t blocks = (total + 255) / 256;
    const int64_t cap = (int64_t)sm_count() * 16;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    ftable_cm_kernel<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(d_fcodes, kpad, coutp, (int32_t)cs, (int32_t)c,
                                                                     kh * kw * cs, lut->d_bmajor, lut->is_signed,
                                                                     d_ftable);
    return check_launch("ftable_cm_prepare");
}

int64_t axb_ftable_cx_bytes(int64_t kpad, int64_t coutp, int cb) {
    if (kpad <= 0 || coutp <= 0 || kpad % 16 || (cb != 16 && cb != 32 && cb != 64) || coutp % cb) return 0;
    return kpad * (coutp / cb) * kC64RowBytes;
}
int64_t axb_ftable_c64_bytes(int64_t kpad, int64_t coutp) { return axb_ftable_cx_bytes(kpad, coutp, 64); }

int axb_ftable_c64_prepare(const uint8_t *d_fcodes, int64_t kh, int64_t kw, int64_t c, int64_t cs, int64_t cout,
                           const axb_lut *lut, uint32_t *d_ftable, void *stream) {
    return axb_ftable_cx_prepare(d_fcodes, kh, kw, c, cs, cout, lut, d_ftable, stream, 64);
}

int axb_ftable_cx_prepare(const uint8_t *d_fcodes, int64_t kh, int64_t kw, int64_t c, int64_t cs, int64_t cout,
                          const axb_lut *lut, uint32_t *d_ftable, void *stream, int cb) {
    if (!lut || !d_fcodes || !d_ftable) return set_error(AXB_E_VALUE, "null argument");
    if (cs % 16 || c > cs || c < 1) return set_error(AXB_E_VALUE, "channel stride mismatch");
    if (cb != 16 && cb != 32 && cb != 64) return set_error(AXB_E_VALUE, "channel block must be 16, 32 or 64");
    const int64_t kpad = axb_filter_kpad(kh, kw, cs), coutp = axb_filter_coutp(cout);
    if (coutp % cb) return set_error(AXB_E_VALUE, "code-major table needs coutp % channel block == 0");
    const int64_t total = (coutp / cb) * kpad * kC64RowWords;
    int64_t blocks = (total + 255) / 256;
    const int64_t cap = (int64_t)sm_count() * 16;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    ftable_c64_kernel<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(d_fcodes, kpad, coutp, (int32_t)cs, (int32_t)c,
                                                                      kh * kw * cs, lut->d_bmajor, lut->is_signed,
                                                                      d_ftable, (int32_t)cb);
    return check_launch("ftable_cx_prepare");
}

int axb_ft_variant_layout(int v) { return (v >= 1 && v < kNumFtVariants) ? kFtVariants[v].cm : 0; }
int64_t axb_ft_variant_max_k(int v) { return (v >= 1 && v < kNumFtVariants && kFtVariants[v].cm >= 2) ? kCxMaxK : 32768; }

int axb_ft_variant_count(void) { return kNumFtVariants; }
int axb_ft_variant_clusters(int v, int is_signed) {
    if (v < 1 || v >= kNumFtVariants) return set_error(AXB_E_VALUE, "unknown ftable kernel variant"), -1;
    ConvK k{};
    return is_signed ? launch_ft_variant<true>(1, v, k, 0, 0) : launch_ft_variant<false>(1, v, k, 0, 0);
}
const char *axb_ft_variant_name(int v) { return (v >= 0 && v < kNumFtVariants) ? kFtVariants[v].name : ""; }

}  // extern "C"
