// Halo-operand probe for implicit 3x3 convolution:
// can one tcgen05.mma kind::tf32 read a 128-row K-major SW128 A operand whose
// rows are a shifted window of a larger swizzled patch (start not 1024-byte
// aligned, 8-row group stride of `gstride` rows)? The patch is stored with the
// 128-byte swizzle of its absolute shared-memory address, as TMA writes it.
// Prints the max error against a CPU product for start rows 0..7 with the
// descriptor base-offset field 0 and (start >> 7) & 7.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o halo_probe halo_probe.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout, uint32_t base) {
    uint64_t d = 0;
    d |= (uint64_t)((addr & 0x3FFFF) >> 4);
    d |= (uint64_t)((lbo & 0x3FFFF) >> 4) << 16;
    d |= (uint64_t)((sbo & 0x3FFFF) >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)(base & 7) << 49;
    d |= (uint64_t)layout << 61;
    return d;
}

constexpr int N = 64, PROWS = 200;

// patch: PROWS rows x 32 fp32 (K-major, SW128 by absolute address); B: N rows x 32.
__global__ void __launch_bounds__(128, 1) probe(const float* patch, const float* bmat, float* out, int start_row,
                                                int gstride, int use_base) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* sa = smem;                      // PROWS * 128 B
    uint8_t* sb = smem + ((PROWS * 128 + 1023) / 1024) * 1024;
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const uint32_t a_base = smem_u32(sa), b_base = smem_u32(sb);
    for (int i = threadIdx.x; i < PROWS * 8; i += blockDim.x) {   // 16-byte chunks
        const int row = i / 8, j = i % 8;
        const uint32_t addr = a_base + row * 128;
        const int sw = j ^ ((addr >> 7) & 7);
        *(float4*)(sa + row * 128 + sw * 16) = *(const float4*)(patch + row * 32 + j * 4);
    }
    for (int i = threadIdx.x; i < N * 8; i += blockDim.x) {
        const int row = i / 8, j = i % 8;
        const uint32_t addr = b_base + row * 128;
        const int sw = j ^ ((addr >> 7) & 7);
        *(float4*)(sb + row * 128 + sw * 16) = *(const float4*)(bmat + row * 32 + j * 4);
    }
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(64));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        // kind::tf32, D f32, A/B tf32, K-major both, N, M = 128
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const uint32_t a0 = a_base + start_row * 128;
        for (int kk = 0; kk < 4; ++kk) {
            const uint32_t aa = a0 + kk * 32;
            const uint64_t ad = sdesc(aa, 16, gstride * 128, 2, use_base ? ((aa >> 7) & 7) : 0);
            const uint64_t bd = sdesc(b_base + kk * 32, 16, 1024, 2, 0);
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc),
                "r"(kk));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                     : "memory");
    }
    asm volatile(
        "{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar))
        : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    for (int c = 0; c < N; c += 8) {
        uint32_t r[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                     : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int j = 0; j < 8; ++j) out[(warp * 32 + lane) * N + c + j] = __uint_as_float(r[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64));
}

int main() {
    std::vector<float> patch(PROWS * 32), bm(N * 32);
    for (size_t i = 0; i < patch.size(); ++i) patch[i] = (float)((i * 7919) % 97) / 97.f - 0.5f;
    for (size_t i = 0; i < bm.size(); ++i) bm[i] = (float)((i * 104729) % 89) / 89.f - 0.5f;
    float *dp, *db, *dout;
    cudaMalloc(&dp, patch.size() * 4);
    cudaMalloc(&db, bm.size() * 4);
    cudaMalloc(&dout, 128 * N * 4);
    cudaMemcpy(dp, patch.data(), patch.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(db, bm.data(), bm.size() * 4, cudaMemcpyHostToDevice);
    const int smem = ((PROWS * 128 + 1023) / 1024) * 1024 + N * 128 + 1024;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    std::vector<float> out(128 * N);
    for (int gstride : {8, 10}) {
        for (int use_base = 0; use_base < 2; ++use_base) {
            for (int s = 0; s < 8; ++s) {
                cudaMemset(dout, 0, 128 * N * 4);
                probe<<<1, 128, smem>>>(dp, db, dout, s, gstride, use_base);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) {
                    printf("gstride %d base %d start %d: %s\n", gstride, use_base, s, cudaGetErrorString(e));
                    return 1;
                }
                cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
                double err = 0, ref_max = 0;
                for (int r = 0; r < 128; ++r) {
                    const int prow = s + (r / 8) * gstride + (r % 8);   // row r of the shifted window
                    for (int n = 0; n < N; ++n) {
                        double acc = 0;
                        for (int k = 0; k < 32; ++k) acc += (double)patch[prow * 32 + k] * bm[n * 32 + k];
                        err = fmax(err, fabs(acc - out[r * N + n]));
                        ref_max = fmax(ref_max, fabs(acc));
                    }
                }
                printf("gstride %2d base_field %d start_row %d: max rel err %.2e\n", gstride, use_base, s, err / ref_max);
            }
        }
    }
    return 0;
}
