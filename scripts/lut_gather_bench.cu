// A/B of the product-gather inner loop on REAL activation codes (ResNet-8 s0b0.b input, 4x8 pixel
// blocks x 16 taps per group; build/codes_s0b0b.bin from the oracle): lanes = pixels, 16 channels.
//   W2: 32-bit words = 2 channels per code (8 LDS.32 per pixel-tap)   -- the shipped ftable layout
//   W4: 64-bit words = 4 channels per code (4 LDS.64 per pixel-tap)
// Packed-pair accumulation as in lutconv_ft.  Prints products/s for both.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

constexpr int ROWS = 4;                 // table rows cycled over the 16 taps
constexpr int ROW_WORDS = 256 * 8;      // 8 pairs x 256 codes (8 KiB) in both layouts
constexpr int REPS = 8;

template <int W4>
__global__ void __launch_bounds__(512, 1) bench(const uint4 *__restrict__ codes, int groups, uint32_t *out) {
    __shared__ __align__(16) uint32_t tab[ROWS * ROW_WORDS];
    for (int i = threadIdx.x; i < ROWS * ROW_WORDS; i += blockDim.x) tab[i] = i * 2654435761u;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    uint32_t all[8] = {0}, hi[8] = {0};
    for (int rep = 0; rep < REPS; ++rep) {
        for (int g = warp; g < groups; g += nwarps) {
            const uint4 c = __ldg(codes + g * 32 + lane);
            const uint32_t cw[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const uint32_t a = __byte_perm(cw[k >> 2], 0, 0x4440u + (k & 3));
                const uint32_t *row = tab + (k % ROWS) * ROW_WORDS;
                if (!W4) {
                    const uint32_t *base = row + a;  // [pair][a]: pair stride 256 words
#pragma unroll
                    for (int p = 0; p < 8; ++p) {
                        const uint32_t w = base[p * 256];
                        all[p] += w; hi[p] += w >> 16;
                    }
                } else {
                    const uint2 *base = reinterpret_cast<const uint2 *>(row) + a;  // [quad][a]: 8 B entries
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint2 w = base[q * 256];
                        all[2 * q] += w.x; hi[2 * q] += w.x >> 16;
                        all[2 * q + 1] += w.y; hi[2 * q + 1] += w.y >> 16;
                    }
                }
            }
        }
    }
    uint32_t s = 0;
#pragma unroll
    for (int p = 0; p < 8; ++p) s += all[p] ^ hi[p];
    if (s == 0x12345678u) out[0] = s;
}

// CM: code-major table P[k][a][16 pairs] (64 B per code = 32 channels); lanes = (pixel, quarter):
// one LDS.128 = 4 pairs (8 products) of one pixel, 8 pixels per warp instruction; a warp covers the
// group's 32 pixels in 4 instructions per tap, 32 channels.
__global__ void __launch_bounds__(512, 1) bench_cm(const uint4 *__restrict__ codes, int groups, uint32_t *out) {
    constexpr int CM_ROWS = 2;              // 2 x 16 KiB rows
    __shared__ __align__(16) uint32_t tab[CM_ROWS * 256 * 16];
    for (int i = threadIdx.x; i < CM_ROWS * 256 * 16; i += blockDim.x) tab[i] = i * 2654435761u;
    __syncthreads();
    const int lane = threadIdx.x & 31, q = lane & 3, ps = lane >> 2;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    uint32_t all[4][4] = {}, hi[4][4] = {};
    for (int rep = 0; rep < REPS; ++rep) {
        for (int g = warp; g < groups; g += nwarps) {
            uint32_t cw[4][4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint4 c = __ldg(codes + g * 32 + j * 8 + ps);
                cw[j][0] = c.x; cw[j][1] = c.y; cw[j][2] = c.z; cw[j][3] = c.w;
            }
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const uint4 *row = reinterpret_cast<const uint4 *>(tab + (k % CM_ROWS) * 256 * 16) + q;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t a = __byte_perm(cw[j][k >> 2], 0, 0x4440u + (k & 3));
                    const uint4 w = row[a * 4];
                    all[j][0] += w.x; hi[j][0] += w.x >> 16;
                    all[j][1] += w.y; hi[j][1] += w.y >> 16;
                    all[j][2] += w.z; hi[j][2] += w.z >> 16;
                    all[j][3] += w.w; hi[j][3] += w.w >> 16;
                }
            }
        }
    }
    uint32_t s = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int p = 0; p < 4; ++p) s += all[j][p] ^ hi[j][p];
    if (s == 0x12345678u) out[0] = s;
}

// CM16: code-major with 16 channels per block (32 B per code): 2 lanes per pixel, 16 pixels per
// LDS.128 instruction; a warp covers the group's 32 pixels in 2 instructions per tap.
__global__ void __launch_bounds__(512, 1) bench_cm16(const uint4 *__restrict__ codes, int groups, uint32_t *out) {
    constexpr int CM_ROWS = 4;              // 4 x 8 KiB rows
    __shared__ __align__(16) uint32_t tab[CM_ROWS * 256 * 8];
    for (int i = threadIdx.x; i < CM_ROWS * 256 * 8; i += blockDim.x) tab[i] = i * 2654435761u;
    __syncthreads();
    const int lane = threadIdx.x & 31, q = lane & 1, ps = lane >> 1;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    uint32_t all[2][4] = {}, hi[2][4] = {};
    for (int rep = 0; rep < REPS; ++rep) {
        for (int g = warp; g < groups; g += nwarps) {
            uint32_t cw[2][4];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const uint4 c = __ldg(codes + g * 32 + j * 16 + ps);
                cw[j][0] = c.x; cw[j][1] = c.y; cw[j][2] = c.z; cw[j][3] = c.w;
            }
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const uint4 *row = reinterpret_cast<const uint4 *>(tab + (k % CM_ROWS) * 256 * 8) + q;
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const uint32_t a = __byte_perm(cw[j][k >> 2], 0, 0x4440u + (k & 3));
                    const uint4 w = row[a * 2];
                    all[j][0] += w.x; hi[j][0] += w.x >> 16;
                    all[j][1] += w.y; hi[j][1] += w.y >> 16;
                    all[j][2] += w.z; hi[j][2] += w.z >> 16;
                    all[j][3] += w.w; hi[j][3] += w.w >> 16;
                }
            }
        }
    }
    uint32_t s = 0;
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int p = 0; p < 4; ++p) s += all[j][p] ^ hi[j][p];
    if (s == 0x12345678u) out[0] = s;
}

int main(int argc, char **argv) {
    const char *path = argc > 1 ? argv[1] : "build/codes_s0b0b.bin";
    FILE *f = fopen(path, "rb");
    if (!f) { printf("{\"error\": \"%s missing\"}\n", path); return 1; }
    std::vector<uint8_t> h(1 << 25);
    const size_t n = fread(h.data(), 1, h.size(), f);
    fclose(f);
    const int groups = (int)(n / (32 * 16));
    uint4 *d;
    cudaMalloc(&d, n);
    cudaMemcpy(d, h.data(), n, cudaMemcpyHostToDevice);
    uint32_t *out;
    cudaMalloc(&out, 4);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int i = 0; i < 5; ++i) bench<1><<<sms, 512>>>(d, groups, out);
    cudaDeviceSynchronize();
    double best[4] = {0, 0, 0, 0};
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int it = 0; it < 3; ++it) {
        for (int w4 = 0; w4 < 4; ++w4) {
            cudaEventRecord(a);
            if (w4 == 3) bench_cm16<<<sms, 512>>>(d, groups, out);
            else if (w4 == 2) bench_cm<<<sms, 512>>>(d, groups, out);
            else if (w4) bench<1><<<sms, 512>>>(d, groups, out);
            else bench<0><<<sms, 512>>>(d, groups, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            const double chans = w4 == 2 ? 32 : 16;
            const double prod = (double)groups * 32 * 16 * chans * REPS / (ms * 1e-3);
            if (prod > best[w4]) best[w4] = prod;
        }
    }
    printf("{\"codes\": \"%s\", \"groups\": %d, \"W2_lds32_products_per_s\": %.4e, "
           "\"W4_lds64_products_per_s\": %.4e, \"CM_lds128_products_per_s\": %.4e, \"CM16_lds128_products_per_s\": %.4e}\n",
           path, groups, best[0], best[1], best[2], best[3]);
    return 0;
}
