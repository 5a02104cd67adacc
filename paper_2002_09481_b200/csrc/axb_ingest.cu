// Device ingest of CIFAR-10 binary records: the caller side of the
// graph input.  Restates formats.py:138-157 (load_cifar10: 1 label byte + 3 channel planes of
// 32x32 bytes per record -> NHWC float32(byte) / 255) and fuses the graph input's Min/Max
// range (graph.py:270-275, tensor.py:143-149) into the decode, so a host batch crosses PCIe
// as 3,073 bytes per image instead of 12,288 and no separate range pass is needed.
// Bound: HBM (3,073 B read + 12,288 B written per image).
#include "axb_common.cuh"
#include "axb_internal.h"

namespace axb {

constexpr int kCifarRecord = 3073;
constexpr int kCifarPixels = 1024;

__global__ void __launch_bounds__(256) cifar_decode_kernel(const uint8_t *__restrict__ rec, int64_t n,
                                                           float *__restrict__ out, uint8_t *__restrict__ labels,
                                                           int32_t *d_range, int32_t *d_flags) {
    // one thread per 4 consecutive pixels of a record: 12 byte loads (records are 3,073 B, so the
    // planes are not word-aligned), 3 aligned float4 stores of the 12 NHWC values
    float tmin = INFINITY, tmax = -INFINITY;
    int bad_label = 0;
    const int64_t total = n * (kCifarPixels / 4);
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / (kCifarPixels / 4);
        const int p = (int)(t - i * (kCifarPixels / 4)) * 4;
        const uint8_t *r = rec + i * kCifarRecord;
        if (p == 0) {
            const uint8_t lab = r[0];
            if (labels) labels[i] = lab;
            bad_label |= lab > 9;  // formats.py:151-152
        }
        float v[12];  // NHWC order: pixel q, channel c at 3q + c
#pragma unroll
        for (int c = 0; c < 3; ++c) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float f = __fdiv_rn((float)__ldg(r + 1 + c * kCifarPixels + p + q), 255.0f);  // formats.py:156
                v[3 * q + c] = f;
                tmin = fminf(tmin, f);
                tmax = fmaxf(tmax, f);
            }
        }
        float4 *o = reinterpret_cast<float4 *>(out + (i * kCifarPixels + p) * 3);
        o[0] = make_float4(v[0], v[1], v[2], v[3]);
        o[1] = make_float4(v[4], v[5], v[6], v[7]);
        o[2] = make_float4(v[8], v[9], v[10], v[11]);
    }
    const bool any = tmin <= tmax;
    range_commit(any ? f2ord(tmin) : INT32_MAX, any ? f2ord(tmax) : INT32_MIN, 0, d_range, nullptr, 0);
    if (bad_label && d_flags) atomicOr(d_flags, AXB_FLAG_LABEL);
}

}  // namespace axb

using namespace axb;

extern "C" int axb_cifar_decode(const uint8_t *d_records, int64_t n, float *d_images, uint8_t *d_labels,
                                int32_t *d_range, int32_t *d_flags, void *stream) {
    if (n < 0) return set_error(AXB_E_VALUE, "negative record count");
    if (n == 0) return AXB_OK;
    if (!d_records || !d_images) return set_error(AXB_E_VALUE, "null record or image buffer");
    if ((reinterpret_cast<uintptr_t>(d_images) & 15) != 0) return set_error(AXB_E_VALUE, "image buffer not 16-byte aligned");
    int64_t blocks = (n * (kCifarPixels / 4) + 255) / 256;
    const int64_t cap = (int64_t)sm_count() * 8;
    if (blocks > cap) blocks = cap;
    cifar_decode_kernel<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(d_records, n, d_images, d_labels, d_range,
                                                                       d_flags);
    return check_launch("cifar_decode");
}
