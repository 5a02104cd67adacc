// Measured shared-memory gather roofline on this GPU (the LUT-product conv's bound).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/smem_roofline scripts/smem_roofline.cu
//   /tmp/smem_roofline  -> one JSON line
// Warp-wide gathers of V 32-bit words per lane (LDS.32 / .64 / .128) from a 32 KiB table at
// pseudo-random rows, 32 lanes on distinct 4-byte banks per 128-byte wavefront (conflict-free)
// or pairwise conflicting; every word is accumulated like the conv's packed pairs
// (IADD3 + LEA.HI).  A word carries two 16-bit products.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int WORDS = 8192;  // 32 KiB table (static shared memory)
constexpr int ITERS = 2048;

template <int V, int CONFLICT>
__global__ void __launch_bounds__(512, 1) gather(uint32_t *out, uint32_t seed) {
    __shared__ __align__(16) uint32_t tab[WORDS];
    for (int i = threadIdx.x; i < WORDS; i += blockDim.x) tab[i] = i * 2654435761u;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    uint32_t x = seed ^ (threadIdx.x >> 5) * 0x9E3779B9u;
    uint32_t all = 0, hi = 0;
    constexpr int ROWW = 32 * V;  // words per warp row (128 B per wavefront x V)
    // lane's word within a row; CONFLICT: lanes 2m, 2m+1 read the same bank group of two rows
    const uint32_t lane_off = CONFLICT ? ((lane & 1) * ROWW + (lane >> 1) * V) : lane * V;
    const uint32_t *tl = tab + lane_off;
    constexpr int SPAN = 8 * 2 * ROWW;               // words touched by one iteration's 8 loads
    constexpr uint32_t MASK = (WORDS - SPAN) / ROWW;  // row-group choices (power of two below)
    for (int it = 0; it < ITERS; ++it) {
        x = x * 1664525u + 1013904223u;  // warp-uniform pseudo-random row group
        const uint32_t *b = tl + ((x >> 10) & (MASK - 1) & ~1u) * ROWW;
        // 8 gathers at immediate offsets from one base register, as the conv does per (pixel, row)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t *src = b + j * 2 * ROWW;
            if (V == 1) {
                const uint32_t w = src[0];
                all += w; hi += w >> 16;
            } else if (V == 2) {
                const uint2 w = *reinterpret_cast<const uint2 *>(src);
                all += w.x + w.y; hi += (w.x >> 16) + (w.y >> 16);
            } else {
                const uint4 w = *reinterpret_cast<const uint4 *>(src);
                all += w.x + w.y; hi += (w.x >> 16) + (w.y >> 16);
                all += w.z + w.w; hi += (w.z >> 16) + (w.w >> 16);
            }
        }
    }
    if (all == 0x12345678u && hi == 1u) out[0] = all;  // keep the loads alive
}

template <int V, int C>
static double run(int sms, uint32_t *out) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    double rate = 0;
    for (int rep = 0; rep < 4; ++rep) {  // best of 3 after a warm-up pass
        cudaEventRecord(a);
        gather<V, C><<<sms, 512>>>(out, 12345u + rep);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double r = (double)sms * 512 * ITERS * 8 * V * 2 / (ms * 1e-3);  // 16-bit products / s
        if (rep > 0 && r > rate) rate = r;
    }
    return rate;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);  // kHz (max boost)
    uint32_t *out;
    cudaMalloc(&out, 4);
    for (int i = 0; i < 20; ++i) gather<4, 0><<<sms, 512>>>(out, i);  // clocks up before measuring
    cudaDeviceSynchronize();
    const double r[6] = {run<1, 0>(sms, out), run<2, 0>(sms, out), run<4, 0>(sms, out),
                         run<1, 1>(sms, out), run<2, 1>(sms, out), run<4, 1>(sms, out)};
    const double unit = (double)sms * clk * 1e3;
    printf("{\"sms\": %d, \"sm_max_mhz\": %.0f, \"products_per_s\": {\"lds32\": %.4e, \"lds64\": %.4e, \"lds128\": %.4e, "
           "\"lds32_2way\": %.4e, \"lds64_2way\": %.4e, \"lds128_2way\": %.4e}, \"products_per_clk_per_sm\": {\"lds32\": "
           "%.2f, \"lds64\": %.2f, \"lds128\": %.2f}, \"note\": \"warp gathers of 1/2/4 words per lane, 32 KiB table, "
           "148 CTAs x 512 threads, packed-pair accumulation; 2way = lanes pairwise on one bank\"}\n",
           sms, clk / 1e3, r[0], r[1], r[2], r[3], r[4], r[5], r[0] / unit, r[1] / unit, r[2] / unit);
    return 0;
}
