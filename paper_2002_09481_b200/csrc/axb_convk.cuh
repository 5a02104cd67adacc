// Conv-kernel shared definitions: launch parameter block, PTX helpers (cp.async,
// mbarrier, TMA bulk copy), pixel mapping and the epilogue arithmetic of
// axconv.py:246-256 / graph.py:268-286.  Included by axb_conv.cu (LUT kernels)
// and axb_ftconv.cu (filter-specialised product-table kernel).
#pragma once
#include "axb_common.cuh"
#include "axb_internal.h"

namespace axb {

constexpr int kMaxTaps = 256;

struct ConvK {
    const uint8_t *codes;
    const int32_t *pixsum;
    int32_t hp, wp, cs, c;
    int32_t kh, kw, sh, sw, dh, dw;
    int32_t oh, ow;
    int64_t M;
    const uint8_t *fcodes;
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
    int32_t blk;  // 1: lanes = 32 consecutive pixels of a row; 4: lanes = a 4x8 pixel block
    FastDiv fd_hw, fd_ow, fd_band;  // oh*ow, ow, 4*ow (M < 2^31 per launch)
    int32_t sp_inloop;  // 1: patch sums accumulated in the chunk loop (dp4a), 0: gathered in the epilogue
    const uint32_t *ftable;  // filter-specialised product table (axb_ftable_prepare), or null
    int32_t ntm;             // pixel tiles per channel block (ftable kernel: tile = nb * ntm + mt)
    // tail split (c64 kernel): the last split_L tiles are cut into split_s K-ranges (chunk-aligned pieces)
    // dealt piece-major over the CTAs; partial sums go to split_ws, the last piece of a tile to arrive
    // on split_cnt reduces them and runs the epilogue (0 / 1: no split)
    int32_t split_L, split_s;
    uint32_t *split_ws;
    int32_t *split_cnt;
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
// blocking wait that lets the hardware suspend the thread until the phase completes (or ~100 us pass)
// instead of re-polling: a spinning producer / waiting consumer does not steal issue slots from the
// warps that share its scheduler
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t phase) {
#ifdef AXB_NO_SLEEP_WAIT
    mbar_wait(bar, phase);
#else
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAITS_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 100000;\n"
        "@!p bra WAITS_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
#endif
}
// non-blocking probe: has the phase with this parity completed?
__device__ __forceinline__ bool mbar_test(uint64_t *bar, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ bool mbar_test_cluster(uint64_t *bar, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.test_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    return ok != 0;
}

// ---- thread-block-cluster helpers (TMA multicast of the ftable stages)
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// arrive on the mbarrier at the same shared offset in cluster CTA `rank` (may be this CTA)
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t *bar, uint32_t rank) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(remote) : "r"(smem_u32(bar)), "r"(rank));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(remote) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAITC_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAITC_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
// bulk copy global -> the same shared offset in every CTA of `mask`, complete_tx on each one's mbarrier
__device__ __forceinline__ void bulk_g2s_multicast(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                                   uint16_t mask) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], "
        "%4;\n" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "h"(mask)
        : "memory");
}
// order this thread's generic-proxy shared-memory accesses before later async-proxy (TMA)
// accesses to the same memory: a consumer executes it before releasing a stage that a TMA
// bulk copy will overwrite (write-after-read across proxies)
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
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

// Tile-order position -> NHWC output pixel index m, and the padded-input pixel
// index of its window origin.  blk == 4 walks each image in 4-row bands of
// 4x8 blocks so a warp instruction's 32 lanes are a compact pixel block (more
// similar codes -> fewer LUT bank conflicts); needs oh % 4 == 0, ow % 8 == 0.
__device__ __forceinline__ int64_t pixel_of(const ConvK &p, int64_t mt, int64_t &pix0) {
    const uint32_t hw = (uint32_t)p.oh * (uint32_t)p.ow;
    const uint32_t b = fdiv((uint32_t)mt, p.fd_hw);
    const uint32_t r = (uint32_t)mt - b * hw;
    int64_t oy, ox;
    if (p.blk == 4) {
        const uint32_t band = fdiv(r, p.fd_band);
        const uint32_t rr = r - band * 4 * (uint32_t)p.ow;
        const uint32_t bx = rr >> 5, s = rr & 31;
        oy = band * 4 + (s >> 3);
        ox = bx * 8 + (s & 7);
    } else {
        const uint32_t q = fdiv(r, p.fd_ow);
        oy = q;
        ox = r - q * (uint32_t)p.ow;
    }
    pix0 = (b * p.hp + oy * p.sh) * (int64_t)p.wp + ox * p.sw;
    return b * hw + oy * p.ow + ox;
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
// float min/max tracker for the fast epilogue (+-0 order is irrelevant to compute_coeffs)
__device__ __forceinline__ void track(float y, float &fmin, float &fmax, int &nonfinite) {
    nonfinite |= !(fabsf(y) <= 3.402823466e38f);
    fmin = fminf(fmin, y);
    fmax = fmaxf(fmax, y);
}

}  // namespace axb
