// TMA bulk-copy ingest ceiling: how many bytes/s of L2-resident table stages can 148 SMs pull into
// shared memory (the LUT conv's table ring, with no gathers)?  One CTA per SM, a 3-slot ring of
// 64 KiB stages, thread 0 refilling a slot as soon as the consumer warp released it.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/tma_bw scripts/tma_bw.cu
//   /tmp/tma_bw   -> JSON lines: {"mode", "cluster", "tb_s", ...}
// modes: "shared"  -- every CTA streams the SAME rows (the conv: concurrent CTAs on one channel block)
//        "private" -- every CTA streams its own rows (no reuse between CTAs)
// cluster CL > 1: each CTA of a CL-CTA cluster fetches 1/CL of a stage and multicasts it to all CL CTAs
// (the slot is refilled once the consumers of all CL CTAs released it).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__constant__ int ST;       // ring slots
__constant__ uint32_t STAGE;  // bytes per stage
__constant__ int CHUNKS;   // bulk copies per stage (per CTA of a cluster)
__constant__ int MODE;  // bit 0: consumer skips fence.proxy.async; bit 1: spin with test_wait; bit 2: CTA-scope waits/arrive;
                        // bit 3: stage g issued by lane g % 32 of the producer warp; bit 4: .shared::cta destination;
                        // bit 5: CTA-scope test_wait spins; bit 6: try_wait with a 20 ns suspend-time hint
static int h_ST = 3, h_CHUNKS = 1, h_MODE = 0;
static uint32_t h_STAGE = 64 * 1024;

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void init(uint64_t *b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(n));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
}
__device__ __forceinline__ void expect(uint64_t *b, uint32_t n) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void wait(uint64_t *b, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
                 "@!p bra W_%=;\n}\n" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void wait_cta(uint64_t *b, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
                 "@!p bra T_%=;\n}\n" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void arrive_cta(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void spin_cta(uint64_t *b, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nU_%=:\nmbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n"
                 "@!p bra U_%=;\n}\n" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void wait_hint(uint64_t *b, uint32_t ph) {  // try_wait with a 20 ns suspend hint
    asm volatile("{\n.reg .pred p;\nH_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 20;\n"
                 "@!p bra H_%=;\n}\n" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void spin(uint64_t *b, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nS_%=:\nmbarrier.test_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
                 "@!p bra S_%=;\n}\n" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void arrive_remote(uint64_t *b, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(su32(b)), "r"(rank));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(r) : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}

template <int CL>
__global__ void __launch_bounds__(64, 1) stream(const uint8_t *src, uint64_t src_bytes, int stages, int shared_rows,
                                                uint32_t *sink) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)ST * STAGE);
    uint64_t *empty = full + ST;
    const int tid = threadIdx.x;
    const uint32_t rank = CL > 1 ? cluster_rank() : 0;
    const uint64_t grp = blockIdx.x / CL;  // cluster index
    if (tid == 0)
        for (int s = 0; s < ST; ++s) init(full + s, 1), init(empty + s, CL);
    __syncthreads();
    if (CL > 1) asm volatile("barrier.cluster.arrive.release;\nbarrier.cluster.wait.acquire;\n" ::: "memory");
    const uint64_t rows = src_bytes / STAGE;
    auto issue = [&](int g) {
        const int s = g % ST;
        const uint64_t row = shared_rows ? (uint64_t)g % rows : (grp * 7919u + (uint64_t)g) % rows;
        expect(full + s, STAGE);
        const uint32_t part = STAGE / CL / CHUNKS;
        for (int c = 0; c < CHUNKS; ++c) {
        const uint8_t *gsrc = src + row * STAGE + (rank * CHUNKS + c) * part;
        uint8_t *dst = smem + (size_t)s * STAGE + (rank * CHUNKS + c) * part;
        if (CL > 1) {
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, "
                "[%3], %4;\n" ::"r"(su32(dst)),
                "l"(gsrc), "r"(part), "r"(su32(full + s)), "h"((uint16_t)((1u << CL) - 1))
                : "memory");
        } else if (MODE & 16) {
            asm volatile(
                "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                    su32(dst)),
                "l"(gsrc), "r"(part), "r"(su32(full + s))
                : "memory");
        } else {
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                    su32(dst)),
                "l"(gsrc), "r"(part), "r"(su32(full + s))
                : "memory");
        }
        }
    };
    uint32_t acc = 0;
    if (tid < 32 && (MODE & 8)) {  // producer warp, stage g issued by lane g % 32
        for (int g = 0; g < stages; ++g) {
            if (g >= ST) wait_cta(empty + g % ST, ((g / ST) - 1) & 1);
            if ((g & 31) == tid) issue(g);
        }
    } else if (tid == 0) {  // producer
        for (int g = 0; g < stages; ++g) {
            if (g >= ST) {
                if (MODE & 32) spin_cta(empty + g % ST, ((g / ST) - 1) & 1);
                else if (MODE & 64) wait_hint(empty + g % ST, ((g / ST) - 1) & 1);
                else if (MODE & 2) spin(empty + g % ST, ((g / ST) - 1) & 1);
                else if (CL == 1 && (MODE & 4)) wait_cta(empty + g % ST, ((g / ST) - 1) & 1);
                else wait(empty + g % ST, ((g / ST) - 1) & 1);
            }
            issue(g);
        }
    } else if (tid == 32) {  // consumer: wait for the stage, touch it, release it to every CTA of the cluster
        for (int g = 0; g < stages; ++g) {
            if (MODE & 32) spin_cta(full + g % ST, (g / ST) & 1);
            else if (MODE & 64) wait_hint(full + g % ST, (g / ST) & 1);
            else if (MODE & 2) spin(full + g % ST, (g / ST) & 1);
            else if (CL == 1 && (MODE & 4)) wait_cta(full + g % ST, (g / ST) & 1);
            else wait(full + g % ST, (g / ST) & 1);
            acc += *reinterpret_cast<volatile uint32_t *>(smem + (g % ST) * STAGE + (g & 1023) * 4);
            if (!(MODE & 1)) asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            if (CL == 1 && (MODE & 4)) arrive_cta(empty + g % ST);
            else for (uint32_t r = 0; r < (uint32_t)CL; ++r) arrive_remote(empty + g % ST, r);
        }
    }
    if (CL > 1) asm volatile("barrier.cluster.arrive.release;\nbarrier.cluster.wait.acquire;\n" ::: "memory");
    if (acc == 0xdeadbeef) sink[blockIdx.x] = acc;
}

template <int CL>
static void run(const uint8_t *src, uint64_t bytes, int shared_rows, uint32_t *sink, int nsm, int per_sm = 1) {
    const size_t smem = (size_t)h_ST * h_STAGE + 2 * h_ST * 8;
    cudaMemcpyToSymbol(ST, &h_ST, 4);
    cudaMemcpyToSymbol(STAGE, &h_STAGE, 4);
    cudaMemcpyToSymbol(CHUNKS, &h_CHUNKS, 4);
    cudaMemcpyToSymbol(MODE, &h_MODE, 4);
    cudaFuncSetAttribute(stream<CL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (CL > 1) cudaFuncSetAttribute(stream<CL>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    int grid = (nsm / CL) * CL * per_sm;
    if (CL > 1) {
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(64);
        cfg.dynamicSmemBytes = smem;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int ncl = 0;
        cudaOccupancyMaxActiveClusters(&ncl, stream<CL>, &cfg);
        if (ncl * CL < grid) grid = ncl * CL;
    }
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(64);
    cfg.dynamicSmemBytes = smem;
    cfg.attrs = at;
    cfg.numAttrs = CL > 1 ? 1 : 0;
    const int stages = 2000;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaLaunchKernelEx(&cfg, stream<CL>, src, bytes, 200, shared_rows, sink);  // warm-up
    cudaEventRecord(a);
    cudaLaunchKernelEx(&cfg, stream<CL>, src, bytes, stages, shared_rows, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const cudaError_t e = cudaGetLastError();
    const double delivered = (double)grid * stages * h_STAGE;  // bytes landing in shared memory
    printf("{\"mode\": \"%s\", \"cluster\": %d, \"slots\": %d, \"stage_kib\": %u, \"copies_per_stage\": %d, "
           "\"ctas\": %d, \"per_sm\": %d, \"src_mb\": %.1f, \"ms\": %.3f, \"tb_s_into_smem\": %.3f, \"b_per_clk_per_sm\": %.1f, "
           "\"l2_read_tb_s\": %.3f, \"mode_bits\": %d, \"err\": \"%s\"}\n",
           shared_rows ? "shared" : "private", CL, h_ST, h_STAGE >> 10, h_CHUNKS * CL, grid, per_sm, bytes / 1e6, ms,
           delivered / ms / 1e9, delivered / ms / 1e-3 / (grid / per_sm) / 1.965e9, delivered / CL / ms / 1e9,
           h_MODE, cudaGetErrorString(e));
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const uint64_t bytes = 18ull << 20;  // an 18 MiB table (ResNet-50 3x3x64 layer), L2-resident
    uint8_t *src;
    uint32_t *sink;
    cudaMalloc(&src, 512ull << 20);
    cudaMalloc(&sink, 4096);
    cudaMemset(src, 1, 512ull << 20);
    const int cfgs[][4] = {{3, 64, 1, 4}, {3, 64, 1, 36}, {6, 32, 1, 36}, {12, 16, 1, 36}, {3, 64, 1, 68},
                           {6, 32, 1, 68}, {2, 96, 1, 36}, {4, 48, 1, 36}, {3, 64, 1, 37}, {6, 32, 1, 37},
                           {2, 96, 1, 37}, {3, 64, 4, 36}, {6, 32, 2, 36}};
    for (auto &c : cfgs) {
        h_ST = c[0], h_STAGE = c[1] * 1024u, h_CHUNKS = c[2], h_MODE = c[3];
        run<1>(src, bytes, 1, sink, nsm);
    }
    h_ST = 3, h_STAGE = 32 * 1024u, h_CHUNKS = 1, h_MODE = 4;
    run<1>(src, bytes, 1, sink, nsm, 2);  // two CTAs per SM, 3 x 32 KiB each
    h_ST = 2, h_STAGE = 48 * 1024u;
    run<1>(src, bytes, 1, sink, nsm, 2);
    h_MODE = 0;
    h_ST = 3, h_STAGE = 64 * 1024, h_CHUNKS = 1;
    run<2>(src, bytes, 1, sink, nsm);
    run<1>(src, bytes, 0, sink, nsm);
    run<1>(src, 400ull << 20, 0, sink, nsm);  // private rows from a 400 MiB table (beyond L2: HBM)
    return 0;
}
