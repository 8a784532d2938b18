// Microbenchmark: how fast can one producer warp per CTA stream HBM into a
// shared-memory ring with cp.async.bulk (1-D TMA) when consumers only touch the
// data?  Sweeps stage size, ring depth and CTAs per SM.  Build:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/tma_feed_bench tools/tma_feed_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void feed(const uint8_t* __restrict__ src, size_t bytes, int stage_bytes, int nstages, unsigned* queue,
                     unsigned long long* sink, int consumers) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* full = (uint64_t*)(smem + (size_t)nstages * stage_bytes);
    uint64_t* empty = full + nstages;
    int* item_of = (int*)(empty + nstages);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < nstages; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&full[s])), "r"(1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&empty[s])), "r"(consumers));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const long long nitems = (long long)(bytes / stage_bytes);
    if (warp == 0) {
        int stage = 0;
        unsigned phase = 0;
        for (;;) {
            int it = 0;
            if (lane == 0) it = (int)atomicAdd(queue, 1u);
            it = __shfl_sync(~0u, it, 0);
            // wait empty
            asm volatile("{\n.reg .pred P;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W%=;\n}" ::"r"(
                             su(&empty[stage])),
                         "r"(phase ^ 1u)
                         : "memory");
            if (lane == 0) {
                item_of[stage] = it < nitems ? it : -1;
                if (it < nitems) {
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[stage])), "r"(stage_bytes)
                                 : "memory");
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                     su(smem + (size_t)stage * stage_bytes)),
                                 "l"(src + (size_t)it * stage_bytes), "r"(stage_bytes), "r"(su(&full[stage]))
                                 : "memory");
                } else {
                    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&full[stage])) : "memory");
                }
            }
            __syncwarp();
            if (it >= nitems) break;
            if (++stage == nstages) { stage = 0; phase ^= 1u; }
        }
    } else if (warp <= consumers) {
        int stage = 0;
        unsigned phase = 0;
        unsigned long long acc = 0;
        for (;;) {
            asm volatile("{\n.reg .pred P;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W%=;\n}" ::"r"(
                             su(&full[stage])),
                         "r"(phase)
                         : "memory");
            const int it = item_of[stage];
            if (it < 0) break;
            // touch one 16-byte vector per lane
            const uint4 v = *(const uint4*)(smem + (size_t)stage * stage_bytes + (warp * 32 + lane) * 16 % stage_bytes);
            acc += v.x;
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[stage])) : "memory");
            if (++stage == nstages) { stage = 0; phase ^= 1u; }
        }
        if (acc == 0x1234567) sink[0] = acc;
    }
}

int main() {
    const size_t bytes = (size_t)1 << 30;
    uint8_t* src;
    cudaMalloc(&src, bytes);
    cudaMemset(src, 1, bytes);
    unsigned* q;
    cudaMalloc(&q, 4);
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(feed, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int stage_sizes[] = {8192, 16384, 32768, 65536};
    const int depths[] = {2, 3, 4, 6, 8, 12};
    for (int ss : stage_sizes)
        for (int d : depths)
            for (int ctas = 1; ctas <= 4; ctas *= 2) {
                size_t smem = (size_t)ss * d + 2 * d * 8 + d * 4 + 64;
                if (smem * ctas > 228 * 1024 || smem > 227 * 1024) continue;
                float best = 1e9f;
                for (int rep = 0; rep < 4; ++rep) {
                    cudaMemset(q, 0, 4);
                    cudaEventRecord(e0);
                    feed<<<sms * ctas, 32 * 9, smem>>>(src, bytes, ss, d, q, sink, 8);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    if (ms < best) best = ms;
                }
                cudaError_t err = cudaGetLastError();
                printf("stage %6d depth %2d ctas/SM %d  inflight/SM %4zu KB  %7.1f GB/s %s\n", ss, d, ctas,
                       (size_t)ss * d * ctas / 1024, bytes / (best * 1e-3) / 1e9, err ? cudaGetErrorString(err) : "");
            }
    return 0;
}
