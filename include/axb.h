/*
 * axb.h -- C ABI of the B200-native approximate-convolution path
 * (paper_2002_09481_b200, "axb").  Plain pointers and sizes only; every
 * pointer named d_* or documented "device" is CUDA device memory owned by
 * the caller.  All launches are stream-ordered on the given cudaStream_t
 * (passed as void*); no function synchronises unless documented.
 *
 * Return value: 0 = OK, otherwise one of AXB_E_*; axb_last_error() gives the
 * message (thread-local).  The Python adapter maps codes back to the
 * reference's exception types (ValueError / OverflowError).
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/axemu):
 *   axb_lut_create          <- axmult.py:22-43    MultLut (table, index (a<<8)|b)
 *   axb_range_reset/minmax  <- tensor.py:143-149  tensor_min_max; graph.py:270-275 Min/Max nodes
 *   axb_coeffs_from_range   <- quantizer.py:98-117 compute_coeffs (device-side, no host sync)
 *   axb_coeffs_host         <- quantizer.py:98-117 compute_coeffs (host scalars)
 *   axb_quantize_pad        <- quantizer.py:120-131 quantize_values + axconv.py:181-189 zp padding
 *   axb_quantize_pad_range  <- the two above fused (coefficients of a device range, then quantize)
 *   axb_quantize_im2col     <- quantize_values + zp padding + im2cols (axconv.py:160-196) in one pass
 *   axb_filters_prepare     <- axconv.py:199-210  quantize_filters (K x Cout codes + S_f)
 *   axb_conv2d_lut          <- axconv.py:213-257  approx_gemm/_lut_matmul (:136-146) + im2cols
 *                              (:160-196, implicit) + graph.py:268-277 bias / ReLU epilogue
 *   axb_axconv2d            <- axconv.py:266-297  axconv2d (whole operator, one call)
 *   axb_maxpool/avgpool     <- graph.py:182-199   _pool2d (float glue around the op)
 *   axb_cifar_decode        <- formats.py:138-157 load_cifar10 (decode on device) + the input range
 *   axb_add_relu            <- graph.py:276-286   ReLU / Add nodes
 */
#ifndef AXB_H
#define AXB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AXB_OK 0
#define AXB_E_VALUE 1     /* -> ValueError    (shapes, layouts, non-finite, bad params) */
#define AXB_E_OVERFLOW 2  /* -> OverflowError (32-bit code-sum overflow)              */
#define AXB_E_CUDA 3      /* -> RuntimeError  (CUDA launch / allocation failure)       */

/* flag bits written by kernels into a device int32 (checked by the host) */
#define AXB_FLAG_NONFINITE 1      /* non-finite value to quantize / in a range (ValueError) */
#define AXB_FLAG_PSUM_OVF 2       /* patch code sum outside int32 (OverflowError)           */
#define AXB_FLAG_OUT_NONFINITE 4  /* non-finite kernel output feeding a fused range         */
#define AXB_FLAG_FSUM_OVF 8       /* filter code sum outside int32 (OverflowError)          */
#define AXB_FLAG_LABEL 16         /* CIFAR-10 label byte outside 0..9 (FormatError)         */

/* signedness / rounding / accumulator enums (quantizer.py:28-49, axconv.py:47-58) */
#define AXB_UNSIGNED 0
#define AXB_SIGNED 1
#define AXB_ROUND_HALF_AWAY 0
#define AXB_ROUND_HALF_EVEN 1
#define AXB_ROUND_TOWARD_ZERO 2
#define AXB_ACC_EXACT64 0
#define AXB_ACC_WRAP32 1
#define AXB_ACC_SATURATE32 2

/* QuantParams (quantizer.py:60-74) plus the exact code-boundary table of the
 * quantizer for these parameters: bound[u] = the smallest float32 x whose code
 * (quantizer.py:120-131) is >= lo + u (u = 1..255; bound[0] = -inf; +inf when
 * no float reaches that code).  quantize_values is monotone in x, so
 * code(x) = lo + max{u : bound[u] <= x} exactly; the boundaries are found by
 * bisection against the fp64 reference function.  Lives in device memory. */
typedef struct axb_qparams {
    double scale;
    int32_t zero_point;
    int32_t valid; /* 1 once computed; 2 = scale/zero_point only, bound[] unset (axb_quantize_pad_range) */
    float bound[256];
} axb_qparams;

typedef struct axb_lut axb_lut; /* opaque: device copies of one truth table */

const char *axb_last_error(void);
int axb_version(void);
int axb_device_info(int device, int *sm_count, int *smem_optin_bytes, int *cc_major, int *cc_minor);

/* ---- multiplier table ---------------------------------------------------- */
/* entries: 65,536 raw 16-bit words, host memory, index (a_byte << 8) | b_byte
 * (a = activation / first operand, b = filter / second operand). */
int axb_lut_create(const uint16_t *entries, int is_signed, axb_lut **out);
int axb_lut_destroy(axb_lut *lut);
int axb_lut_is_signed(const axb_lut *lut);
/* device pointer of the b-major (transposed) copy used by the conv kernels */
const uint16_t *axb_lut_device_bmajor(const axb_lut *lut);

/* ---- K1: range reduction ------------------------------------------------- */
/* d_range: 2 x int32 ordered-float accumulators [min, max]; reset sets +inf/-inf */
int axb_range_reset(int32_t *d_range, void *stream);
int axb_range_minmax(const float *d_x, int64_t n, int32_t *d_range, int32_t *d_flags, void *stream);
/* read back (synchronises): min/max as float, nonfinite flag */
int axb_range_read(const int32_t *d_range, const int32_t *d_flags, float *mn, float *mx, int32_t *flags,
                   void *stream);

/* ---- coefficients -------------------------------------------------------- */
int axb_coeffs_host(double mn, double mx, int is_signed, int round_mode, axb_qparams *out);
int axb_coeffs_from_range(const int32_t *d_range, int is_signed, int round_mode, axb_qparams *d_out,
                          void *stream);
int axb_params_upload(const axb_qparams *host_params, axb_qparams *d_params, void *stream);

/* ---- K2: quantize into a zero-point-padded uint8 NHWC tensor -------------- */
/* d_x: (n,h,w,c) fp32; d_codes: (n, h+pt+pb, w+pl+pr, cs) raw code bytes with
 * the border = zero-point code and channels c..cs-1 = 0; d_pixsum (nullable: only the
 * b-major-LUT kernel with K > 512 and the generic kernel read it): per padded
 * pixel sum of the c code values (int32).  cs = axb_channel_stride(c). */
int64_t axb_channel_stride(int64_t c);
int axb_quantize_pad(const float *d_x, int64_t n, int64_t h, int64_t w, int64_t c, int32_t pt, int32_t pb,
                     int32_t pl, int32_t pr, int64_t cs, const axb_qparams *d_params, int is_signed,
                     int round_mode, uint8_t *d_codes, int32_t *d_pixsum, int32_t *d_flags, void *stream);
/* Same, with compute_coeffs (quantizer.py:98-117) of the device range d_range done in the
 * kernel prologue (no separate coefficient launch); the parameters used are written to
 * d_params_out for the conv epilogue. */
int axb_quantize_pad_range(const float *d_x, int64_t n, int64_t h, int64_t w, int64_t c, int32_t pt, int32_t pb,
                           int32_t pl, int32_t pr, int64_t cs, const int32_t *d_range, int is_signed, int round_mode,
                           axb_qparams *d_params_out, uint8_t *d_codes, int32_t *d_pixsum, int32_t *d_flags,
                           void *stream);

/* ---- filter preparation (once per layer) ---------------------------------- */
/* d_f: HWCN fp32 (kh,kw,c,cout).  d_fcodes: (kpad, coutp) uint8 raw code bytes
 * (row k = (ky*kw + kx)*cs + ci; junk rows / columns = 0); d_fsum: int64[cout]. */
int64_t axb_filter_kpad(int64_t kh, int64_t kw, int64_t cs);
int64_t axb_filter_coutp(int64_t cout);
int axb_filters_prepare(const float *d_f, int64_t kh, int64_t kw, int64_t c, int64_t cout, int64_t cs,
                        const axb_qparams *d_params, int is_signed, int round_mode, uint8_t *d_fcodes,
                        int64_t *d_fsum, int32_t *d_flags, void *stream);

/* ---- K3: LUT implicit-GEMM convolution with fused epilogue ---------------- */
typedef struct axb_conv_desc {
    const uint8_t *codes;   /* zp-padded input codes (n, hp, wp, cs)               */
    const int32_t *pixsum;  /* (n, hp, wp) code sums                                */
    int64_t n, hp, wp, cs, c;
    int32_t kh, kw, sh, sw, dh, dw;
    int64_t oh, ow;
    const uint8_t *fcodes;  /* (kpad, coutp) from axb_filters_prepare               */
    const int64_t *fsum;    /* (cout)                                               */
    int64_t cout, coutp, kpad;
    const axb_qparams *in_params; /* device */
    const axb_qparams *f_params;  /* device */
    int32_t accumulator;    /* AXB_ACC_*                                            */
    int32_t relu;           /* 1: max(y, 0) after bias/residual (graph.py:276-277)  */
    const float *bias;      /* nullable, fp32[cout] (graph.py:268-269)              */
    const float *residual;  /* nullable, fp32 (n,oh,ow,cout) added after bias       */
    float *out;             /* fp32 (n, oh, ow, cout)                               */
    int64_t *acc_out;       /* nullable: emulated raw LUT sums A (int64)            */
    int32_t *out_range;     /* nullable: ordered-float [min,max] of out (next layer) */
    int32_t *flags;         /* device int32 flag word                               */
    int32_t force_generic;  /* 1: use the int64 generic kernel (testing)            */
    int32_t sm_limit;       /* 0 = all SMs; else cap persistent grid                 */
    int32_t variant;        /* fast-kernel tile variant, 0 = heuristic (tuning);     *
                             * axb_depthwise_lut with a table: 1 = per-pixel kernel  *
                             * (depthwise_ct) instead of the row-strip one           */
    int32_t pixel_order;    /* lanes -> pixels: 0 auto, 1 row runs, 4 4x8 blocks     */
    const uint32_t *ftable; /* nullable: filter-specialised product table from
                               axb_ftable_prepare; when set (and variant == 0) the
                               packed-pair ftable kernel runs instead of the LUT one */
    int32_t ft_variant;     /* ftable-kernel tile variant, 0 = cost model            */
    int32_t reserved0;
} axb_conv_desc;

int axb_conv2d_lut(const axb_conv_desc *desc, const axb_lut *lut, void *stream);

/* ---- filter-specialised product table (once per layer and truth table) -----
 * The filter codes of a layer are constants (graph.py:129-130), so the 256
 * possible products of every filter code are gathered once:
 *   W[sb][k][pair][a] = u(lut[(a<<8)|F[k][sb*8+2*pair]]) | u(lut[(a<<8)|F[k][sb*8+2*pair+1]]) << 16
 * (sb = 8-channel sub-block, pair = 0..3: 4 KiB per (sb, k) row; a conv tile of 8 or 16
 * channels streams one or two sub-blocks' rows)
 * (u = raw ^ 0x8000 for signed tables, raw for unsigned; junk rows = zero
 * contribution), uint32, axb_ftable_bytes(kpad, coutp) = kpad * coutp * 512 bytes.
 * kh, kw, c, cs are the filter geometry the conv sees (as axb_filters_prepare).
 * Replaces no reference function: it is a re-layout of the MultLut (axmult.py:22-43)
 * restricted to the layer's filter codes (axconv.py:199-210), bit-identical sums. */
int64_t axb_ftable_bytes(int64_t kpad, int64_t coutp);
int axb_ftable_prepare(const uint8_t *d_fcodes, int64_t kh, int64_t kw, int64_t c, int64_t cs, int64_t cout,
                       const axb_lut *lut, uint32_t *d_ftable, void *stream);
int axb_ft_variant_count(void);
/* resident CTA clusters (CTAs for cluster size 1) of ftable variant v on the current device */
int axb_ft_variant_clusters(int variant, int is_signed);
const char *axb_ft_variant_name(int variant);
/* Code-major layout of the same words for the cm32_* variants (ft_variant with
 * axb_ft_variant_layout(v) == 1; pass this table as desc.ftable):
 *   CM[cb][k][a][pr] = W word of channels (cb*32 + 2*pr, cb*32 + 2*pr + 1), pr = 0..15
 * i.e. 64 contiguous bytes per (32-channel block, row, code); 16 KiB per (cb, k).
 * axb_ftable_cm_bytes = kpad * coutp * 512 (0 unless coutp % 32 == 0). */
int64_t axb_ftable_cm_bytes(int64_t kpad, int64_t coutp);
int axb_ftable_cm_prepare(const uint8_t *d_fcodes, int64_t kh, int64_t kw, int64_t c, int64_t cs, int64_t cout,
                          const axb_lut *lut, uint32_t *d_ftable, void *stream);
/* 64-channel code-major layout for the c64_* variants (axb_ft_variant_layout(v) == 2):
 *   C64[cb][k][a][pr] = W word of channels (cb*64 + 2*pr, cb*64 + 2*pr + 1), pr = 0..31
 * i.e. 128 contiguous bytes (all 32 banks) per (64-channel block, row, code); 32 KiB per (cb, k).
 * The kernel's quarter-warp = one pixel reading one whole row: bank-conflict-free for any codes.
 * axb_ftable_c64_bytes = kpad * coutp * 512 (0 unless coutp % 64 == 0). */
int64_t axb_ftable_c64_bytes(int64_t kpad, int64_t coutp);
int axb_ftable_c64_prepare(const uint8_t *d_fcodes, int64_t kh, int64_t kw, int64_t c, int64_t cs, int64_t cout,
                           const axb_lut *lut, uint32_t *d_ftable, void *stream);
/* CX layouts (c64_* / c32_* / c16_* variants, axb_ft_variant_layout(v) == 2 / 3 / 4): channel blocks of
 * cb = 64 / 32 / 16, every (block, row, code) a 128-byte row holding the block's cb/2 pair words
 * repeated 64/cb times (cb = 64: exactly the C64 layout above).  A pixel's cb/8 lanes read the copy no
 * other pixel of their quarter-warp reads: conflict-free at every channel width.
 * axb_ftable_cx_bytes = kpad * (coutp / cb) * 32768 (0 unless coutp % cb == 0). */
int64_t axb_ftable_cx_bytes(int64_t kpad, int64_t coutp, int cb);
int axb_ftable_cx_prepare(const uint8_t *d_fcodes, int64_t kh, int64_t kw, int64_t c, int64_t cs, int64_t cout,
                          const axb_lut *lut, uint32_t *d_ftable, void *stream, int cb);
/* 0: variant v reads the pair-major table (axb_ftable_prepare), 1: the 32-channel code-major one,
 * 2 / 3 / 4: the CX table with 64 / 32 / 16-channel blocks */
int axb_ft_variant_layout(int variant);
/* largest kpad variant v accepts (CX variants: 8192, their epilogue correction is 32-bit; others 32768) */
int64_t axb_ft_variant_max_k(int variant);
int axb_conv_variant_count(void);
/* Depthwise approximate conv (config 5; the reference has no groups): channel c
 * of the output == axconv2d on input channel c alone with the shared ranges.
 * desc: cout == c; fcodes/fsum from axb_filters_prepare on the (kh,kw,1,c)
 * view of the (kh,kw,c,1) filter (cs 16). */
int axb_depthwise_lut(const axb_conv_desc *desc, const axb_lut *lut, void *stream);
/* Channel-bank product table for the depthwise kernel (desc->ftable; <= 13 taps):
 *   DW[cb][t][a >> 1][lane] = u(lut[(a_even << 8) | b]) | u(lut[(a_odd << 8) | b]) << 16
 * b = filter code of tap t, channel cb*32 + lane; u = raw ^ 0x8000 (signed) / raw.  Lane L of a warp
 * (channel L of a 32-channel block) always reads bank L: conflict-free for any activation codes.
 * 16 KiB per (tap, 32-channel block); 0 when the shape is unsupported. */
int64_t axb_depthwise_table_bytes(int64_t kh, int64_t kw, int64_t c);
int axb_depthwise_table_prepare(const uint8_t *d_fcodes, int64_t kh, int64_t kw, int64_t c, int64_t coutp,
                                const axb_lut *lut, uint32_t *d_table, void *stream);
const char *axb_conv_variant_name(int variant);

/* ---- small-channel layers: explicit im2col of the codes (axconv.py:160-196) ----
 * When c is not a multiple of 16 and the kernel has >1 tap, zero-channel
 * padding would waste most lookups; instead the zp-padded codes are gathered
 * into dense rows of kp = roundup16(kh*kw*c) bytes (row sum = patch sum S_p)
 * and the conv runs as a 1x1 over (n, oh, ow, kp) with c = kh*kw*c.
 * axb_conv_im2col_kp returns kp when that path applies, else 0. */
int64_t axb_conv_im2col_kp(int64_t c, int64_t kh, int64_t kw);
int axb_im2col_pack(const uint8_t *d_codes, int64_t n, int64_t hp, int64_t wp, int64_t cs, int64_t c, int32_t kh,
                    int32_t kw, int32_t sh, int32_t sw, int32_t dh, int32_t dw, int64_t oh, int64_t ow, int64_t kp,
                    int is_signed, uint8_t *d_rows, int32_t *d_rowsum, void *stream);
/* The same rows straight from the fp32 input (quantize_values + zp padding + im2cols in one
 * pass; the zp-padded code tensor is never written).  d_range non-null: coefficients of that
 * device range computed in the kernel (written to d_params, as axb_quantize_pad_range);
 * NULL: d_params holds host-computed parameters (as axb_quantize_pad). */
int axb_quantize_im2col(const float *d_x, int64_t n, int64_t h, int64_t w, int64_t c, int32_t pt, int32_t pl,
                        int32_t kh, int32_t kw, int32_t sh, int32_t sw, int32_t dh, int32_t dw, int64_t oh, int64_t ow,
                        int64_t kp, const int32_t *d_range, axb_qparams *d_params, int is_signed, int round_mode,
                        uint8_t *d_rows, int32_t *d_rowsum, int32_t *d_flags, void *stream);
/* which kernel variant the last axb_conv2d_lut call on this thread launched */
const char *axb_last_kernel(void);

/* ---- whole operator (axconv2d) on device buffers, host ranges ------------- */
/* pads: resolved (top,bottom,left,right).  Synchronises once to check flags. */
int axb_axconv2d(const float *d_x, int64_t n, int64_t h, int64_t w, int64_t c, const float *d_f, int64_t kh,
                 int64_t kw, int64_t cout, int32_t sh, int32_t sw, int32_t dh, int32_t dw, int32_t pt,
                 int32_t pb, int32_t pl, int32_t pr, double in_min, double in_max, double f_min,
                 double f_max, int32_t round_mode, int32_t accumulator, const axb_lut *lut, float *d_out,
                 int64_t *d_acc_out, void *stream);

/* ---- device ingest of CIFAR-10 binary records (formats.py:138-157) --------- */
/* d_records: n x 3,073 bytes (label + R, G, B planes of 32x32).  d_images: (n,32,32,3)
 * fp32 NHWC = float32(byte)/255; d_labels (nullable): n bytes.  d_range (nullable):
 * ordered-float [min,max] of the images accumulated (reset it first), the graph input's
 * Min/Max nodes.  A label byte > 9 sets AXB_FLAG_LABEL in d_flags (nullable). */
int axb_cifar_decode(const uint8_t *d_records, int64_t n, float *d_images, uint8_t *d_labels, int32_t *d_range,
                     int32_t *d_flags, void *stream);

/* ---- float glue for the graph executor ------------------------------------ */
int axb_maxpool(const float *d_x, int64_t n, int64_t h, int64_t w, int64_t c, int32_t ph, int32_t pw,
                int32_t sh, int32_t sw, int32_t pt, int32_t pl, int64_t oh, int64_t ow, float *d_out,
                int32_t *d_out_range, int32_t *d_flags, void *stream);
int axb_avgpool(const float *d_x, int64_t n, int64_t h, int64_t w, int64_t c, int32_t ph, int32_t pw,
                int32_t sh, int32_t sw, int32_t pt, int32_t pl, int64_t oh, int64_t ow, float *d_out,
                int32_t *d_out_range, int32_t *d_flags, void *stream);
/* out = relu?(a + b?) elementwise fp32; b nullable */
int axb_add_relu(const float *d_a, const float *d_b, int64_t n, int32_t relu, float *d_out, int32_t *d_out_range,
                 int32_t *d_flags, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* AXB_H */
