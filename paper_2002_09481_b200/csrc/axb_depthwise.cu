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
#include "axb_common.cuh"
#include "axb_internal.h"

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

}  // namespace axb

using namespace axb;

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
