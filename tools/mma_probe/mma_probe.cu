// Peak tcgen05.mma kind::tf32 issue rate from shared memory (no TMA, no
// epilogue): one CTA per SM, one thread issues `iters` k-steps of 4 MMAs
// (K = 8 each) into a TMEM accumulator, committing to an mbarrier every
// k-step and waiting `lag` k-steps behind. Reports TFLOP/s per (M=128, N).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((addr & 0x3FFFF) >> 4);
    d |= (uint64_t)((lbo & 0x3FFFF) >> 4) << 16;
    d |= (uint64_t)((sbo & 0x3FFFF) >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)layout << 61;
    return d;
}

__global__ void __launch_bounds__(128, 1) probe(int N, int iters, float* sink, int stress, int M) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t bar, bar2;
    __shared__ uint32_t slot;
    uint8_t* sa = smem;
    uint8_t* sb = smem + 16384;
    for (int i = threadIdx.x; i < (16384 + N * 128) / 4; i += blockDim.x) ((float*)smem)[i] = 0.f;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar2)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = slot;
    if (stress > 0 && threadIdx.x >= 32) {
        // warps 1-3 stream 16-byte stores into a separate 16 KB region (TMA-fill-like smem traffic)
        uint4* w = (uint4*)(smem + 16384 + N * 128);
        const uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
        for (int it = 0; it < iters * stress; ++it)
#pragma unroll
            for (int j = 0; j < 8; ++j) w[((threadIdx.x - 32) * 8 + j) & 1023] = v;
    }
    if (threadIdx.x == 0) {
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
        const uint32_t a0 = smem_u32(sa), b0 = smem_u32(sb);
        uint32_t phase = 0;
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                uint64_t ad = sdesc(a0 + kk * 32, 16, 1024, 2), bd = sdesc(b0 + kk * 32, 16, 1024, 2);
                asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}"
                             ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(1));
            }
            if (stress < 0) {   // commit every k-step to a second barrier (like the smem-slot release)
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar2)));
            }
            if ((it & 15) == 15) {   // bound the queue: commit and wait every 16 k-steps
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
                asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(smem_u32(&bar)), "r"(phase));
                phase ^= 1;
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
    if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] = 1.f;
}

int main() {
    float* sink;
    cudaMalloc(&sink, 4);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    const int stress = 0;
    for (int M : {64, 128})
    for (int N : {64, 128, 256}) {
        const int iters = 4096;
        probe<<<sms, 128, 80 * 1024>>>(N, 64, sink, stress, M);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        probe<<<sms, 128, 80 * 1024>>>(N, iters, sink, stress, M);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * M * N * 32 * (double)iters * sms;
        // stress s: per k-step 96 threads x 8 x 16 B x s = 12 KB x s of smem stores
        printf("M=%3d N=%3d: %.1f TFLOP/s (%s)\n", M, N, flops / ms / 1e9,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
