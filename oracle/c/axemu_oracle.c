/*
 * TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference's integer
 * LUT-GEMM and nested-loop convolution (the `axemu` package).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library, and only as the checker or the timed CPU baseline.
 * The product (paper_2002_09481_b200) never links it.
 *
 * Restates:
 *   lut_matmul      -> pkg/src/axemu/axconv.py:136-146  (_lut_matmul, numba prange)
 *   direct_lut_sums -> pkg/src/axemu/axconv.py:345-366  (direct_conv inner loops)
 *
 * Both accumulate exactly in int64, like the reference.  Table entries are
 * passed pre-widened to int32 (sign-extended for signed tables, zero-extended
 * for unsigned), which is exactly what numba's int16/uint16 load + int64 add
 * computes.
 */
#include <stdint.h>

/* A[r, c] = sum_k entries[(P[r,k] << 8) | FT[c,k]]   (axconv.py:140-146) */
void lut_matmul(const uint8_t *P, const uint8_t *FT, const int32_t *entries,
                int64_t rows, int64_t depth, int64_t cout, int64_t *out)
{
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < rows; ++r) {
        const uint8_t *prow = P + r * depth;
        for (int64_t c = 0; c < cout; ++c) {
            const uint8_t *frow = FT + c * depth;
            int64_t acc = 0;
            for (int64_t k = 0; k < depth; ++k)
                acc += entries[((int32_t)prow[k] << 8) | (int32_t)frow[k]];
            out[r * cout + c] = acc;
        }
    }
}

/*
 * Nested-loop restatement of direct_conv's lookup phase (axconv.py:345-366).
 * padded: raw code bytes of the zp-padded NHWC input (n, hp, wp, cin);
 * fraw:   raw filter code bytes, (kh*kw*cin, cout) row-major (HWCN flattened);
 * lut_sums out: (n, oh, ow, cout) int64; patch_sums out: (n, oh, ow) int64
 * using the signed/unsigned code *values* in pvals (same shape as padded).
 */
void direct_lut_sums(const uint8_t *padded, const int32_t *pvals, const uint8_t *fraw,
                     const int32_t *entries, int64_t n, int64_t hp, int64_t wp,
                     int64_t cin, int64_t kh, int64_t kw, int64_t cout, int64_t oh,
                     int64_t ow, int64_t sh, int64_t sw, int64_t dh, int64_t dw,
                     int64_t *lut_sums, int64_t *patch_sums)
{
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t b = 0; b < n; ++b)
        for (int64_t r = 0; r < oh; ++r)
            for (int64_t q = 0; q < ow; ++q) {
                int64_t psum = 0;
                for (int64_t y = 0; y < kh; ++y)
                    for (int64_t x = 0; x < kw; ++x) {
                        int64_t base = ((b * hp + r * sh + y * dh) * wp + q * sw + x * dw) * cin;
                        for (int64_t ci = 0; ci < cin; ++ci) psum += pvals[base + ci];
                    }
                patch_sums[(b * oh + r) * ow + q] = psum;
                for (int64_t c = 0; c < cout; ++c) {
                    int64_t acc = 0;
                    int64_t k = 0;
                    for (int64_t y = 0; y < kh; ++y)
                        for (int64_t x = 0; x < kw; ++x) {
                            int64_t base = ((b * hp + r * sh + y * dh) * wp + q * sw + x * dw) * cin;
                            for (int64_t ci = 0; ci < cin; ++ci, ++k)
                                acc += entries[((int32_t)padded[base + ci] << 8) |
                                               (int32_t)fraw[k * cout + c]];
                        }
                    lut_sums[((b * oh + r) * ow + q) * cout + c] = acc;
                }
            }
}

int oracle_max_threads(void)
{
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}
