// gemm_tc.cu -- tcgen05 / TMEM / TMA tensor-core GEMMs for sm_100a (kind::tf32).
//
// Replaces the reference's dense/conv kernels and their gradients
// (kernels.hpp:118-243, tiled route kernels.hpp:354-418). Every contraction is
// expressed as a convolution over an NHWC pixel grid (a dense layer is a 1x1
// convolution over [batch, 1, 1, features]):
//
//   MODE_CONV   C[pixels, N] = sum_{tap, c} A[pixel(tap), c] * B[(tap, c), N]
//               conv fwd (B = weights, MN-major) and conv dgrad (B = weights
//               read as [(tap, ci), co], K-major; strided convs are split into
//               stride^2 sub-pixel phases, one per grid.z). The A tile of a K
//               step is ONE 4-D TMA box {32 ch, TW, TH, TN} of the activation,
//               shifted by the tap, with element strides = conv stride: TMA's
//               out-of-bounds zero fill IS the TF-SAME padding (kernels.cpp:32-35),
//               so no im2col buffer is ever materialized.
//   MODE_WGRAD  C[(tap, ci), co] = sum_pixels x[pixel(tap), ci] * g[pixel, co]
//               both operands MN-major from 4-D TMA boxes, K = pixels split
//               across CTAs (deterministic: partials + ordered reduction).
//
// Per CTA: 6 warps. warp 0 = TMA producer (one elected lane), warp 1 = MMA
// issuer (one thread issues tcgen05.mma.cta_group::1.kind::tf32 128xBNx8 into a
// TMEM accumulator) + TMEM allocator, warps 2-5 = epilogue (tcgen05.ld 32x32b
// -> registers -> bias -> 128-bit global stores). A 4-stage smem ring with
// full/empty mbarriers couples TMA and MMA; tcgen05.commit releases stages.
// Operand tiles use the 128-byte swizzle (TMA and UMMA descriptors agree).
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "driver_api.cuh"
#include "nncb_internal.cuh"

namespace {

constexpr int BM = 128;       // UMMA_M (cta_group::1)
constexpr int BK = 32;        // fp32 elements per K step = one 128-byte swizzle row
constexpr int STAGES = 4;
constexpr int THREADS = 192;
constexpr int MAX_TAPS = 64;

enum { MODE_CONV = 0, MODE_WGRAD = 1 };

struct TcParams {
    int mode;
    int bn;             // N tile: 64 / 128 / 256
    int b_mn;           // B operand MN-major
    int64_t N;          // GEMM N (columns of C)
    int64_t ldc;        // row pitch of C (elements)
    // --- MODE_CONV: rows of C are pixels of the grid (gn, gh, gw) ---------
    int gn, gh, gw;     // output grid
    int TN, TH, TW;     // pixel box per M tile (TN*TH*TW == 128)
    int tiles_w, tiles_h;
    int mh, mw;         // A coordinate = tile origin * (mh, mw) + tap offset
    int cblocks;        // channel blocks of 32 per tap
    int ntaps[4], tap0[4];          // per phase: tap count / first tap
    int py[4], px[4];               // per phase output offset
    int out_h, out_w, out_s;        // output image dims and pixel stride
    int off_h[MAX_TAPS], off_w[MAX_TAPS], brow[MAX_TAPS];
    // --- MODE_WGRAD ---------------------------------------------------------
    int64_t M;          // rows of C = taps * ci
    int ci, kw_;        // for (tap, c) = divmod(m, ci); tap -> (dh, dw)
    int sh, sw, pt, pl;
    int kboxes;         // pixel boxes (TN*TH*TW == 32 pixels each)
    int splits;
    float* partial;     // [splits][M][N] when splits > 1
    const float* bias;  // MODE_CONV forward only
    float* out;
    int debug;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5}], [%6];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

// UMMA shared-memory descriptor (version 1). K-major operands use the 128-byte
// swizzle (layout type 2: 8 rows x 128 B atoms, SBO = 1024 B). MN-major tf32
// operands must use SWIZZLE_128B_BASE32B (layout type 1: 32-byte granules, 4-row
// atoms, SBO = 512 B between K-row groups, LBO = stride between 32-element MN
// chunks) -- the only MN-major layout tcgen05 accepts for 32-bit operands.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes, uint32_t layout) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFF) << 16;
    d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFF) << 32;
    d |= 1ull << 46;
    d |= static_cast<uint64_t>(layout) << 61;
    return d;
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__global__ void __launch_bounds__(THREADS, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                   const __grid_constant__ TcParams P) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t a_bytes = BM * BK * 4;                 // 16 KB
    const uint32_t b_bytes = static_cast<uint32_t>(P.bn) * BK * 4;
    const uint32_t stage_bytes = a_bytes + b_bytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * stage_bytes);
    uint64_t* empty = full + STAGES;
    uint64_t* tmem_full = empty + STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

    // ---- tile coordinates --------------------------------------------------
    int kb_begin = 0, kb_end = 0;
    int phase = 0;
    int64_t n_col0 = static_cast<int64_t>(blockIdx.y) * P.bn;
    int tn0 = 0, th0 = 0, tw0 = 0;   // MODE_CONV tile origin (pixel grid)
    int64_t m0 = 0;                  // MODE_WGRAD row origin
    if (P.mode == MODE_CONV) {
        phase = blockIdx.z;
        int t = blockIdx.x;
        int twi = t % P.tiles_w;
        t /= P.tiles_w;
        int thi = t % P.tiles_h;
        int tni = t / P.tiles_h;
        tn0 = tni * P.TN;
        th0 = thi * P.TH;
        tw0 = twi * P.TW;
        kb_end = P.ntaps[phase] * P.cblocks;
    } else {
        m0 = static_cast<int64_t>(blockIdx.x) * BM;
        int per = (P.kboxes + P.splits - 1) / P.splits;
        kb_begin = blockIdx.z * per;
        kb_end = min(P.kboxes, kb_begin + per);
        if (kb_begin > kb_end) kb_begin = kb_end;
    }
    const int nk = kb_end - kb_begin;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tmem_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    const uint32_t tmem_cols = P.bn < 32 ? 32 : static_cast<uint32_t>(P.bn);
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0 && lane == 0 && nk > 0) {
        // ================= TMA producer =================
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
        for (int i = 0; i < nk; ++i) {
            const int s = i % STAGES;
            if (i >= STAGES) mbar_wait(&empty[s], ((i / STAGES) - 1) & 1);
            uint8_t* sa = smem + s * stage_bytes;
            uint8_t* sb = sa + a_bytes;
            mbar_expect_tx(&full[s], stage_bytes);
            const int kb = kb_begin + i;
            if (P.mode == MODE_CONV) {
                const int tap = P.tap0[phase] + kb / P.cblocks;
                const int c0 = (kb % P.cblocks) * BK;
                tma_load_4d(sa, &map_a, &full[s], c0, tw0 * P.mw + P.off_w[tap], th0 * P.mh + P.off_h[tap], tn0);
                if (P.b_mn) {   // weights [K = (tap, ci), N = co], N contiguous
                    for (int q = 0; q < P.bn / 32; ++q)
                        tma_load_2d(sb + q * 4096, &map_b, &full[s], static_cast<int>(n_col0) + 32 * q,
                                    P.brow[tap] + c0);
                } else {        // weights [(tap, ci) rows, co]; K = co contiguous
                    tma_load_2d(sb, &map_b, &full[s], c0, P.brow[tap] + static_cast<int>(n_col0));
                }
            } else {
                // pixel box kb over the output grid (gn, gh, gw)
                int t = kb;
                const int bw = t % P.tiles_w;
                t /= P.tiles_w;
                const int bh = t % P.tiles_h;
                const int bnn = t / P.tiles_h;
                const int x0 = bw * P.TW, y0 = bh * P.TH, n0 = bnn * P.TN;
                for (int q = 0; q < 4; ++q) {
                    int64_t m = m0 + 32 * q;
                    if (m >= P.M) m = m0;   // clamp (rows masked in the epilogue)
                    const int tap = static_cast<int>(m / P.ci), c = static_cast<int>(m % P.ci);
                    const int dh = tap / P.kw_, dw = tap % P.kw_;
                    tma_load_4d(sa + q * 4096, &map_a, &full[s], c, x0 * P.sw + dw - P.pl, y0 * P.sh + dh - P.pt, n0);
                }
                for (int q = 0; q < P.bn / 32; ++q)
                    tma_load_4d(sb + q * 4096, &map_b, &full[s], static_cast<int>(n_col0) + 32 * q, x0, y0, n0);
            }
        }
    } else if (warp == 1 && lane == 0 && nk > 0) {
        // ================= MMA issuer (single thread) =================
        const uint32_t a_mn = P.mode == MODE_WGRAD ? 1u : 0u;
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (a_mn << 15) |
                               (static_cast<uint32_t>(P.b_mn) << 16) | ((static_cast<uint32_t>(P.bn) >> 3) << 17) |
                               ((static_cast<uint32_t>(BM) >> 4) << 24);
        for (int i = 0; i < nk; ++i) {
            const int s = i % STAGES;
            mbar_wait(&full[s], (i / STAGES) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t sa = smem_u32(smem + s * stage_bytes);
            const uint32_t sb = sa + a_bytes;
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk) {
                const uint64_t ad = a_mn ? sdesc(sa + kk * 1024, 4096, 512, 1) : sdesc(sa + kk * 32, 16, 1024, 2);
                const uint64_t bd = P.b_mn ? sdesc(sb + kk * 1024, 4096, 512, 1) : sdesc(sb + kk * 32, 16, 1024, 2);
                if (P.debug && blockIdx.x == 0 && blockIdx.y == 0 && i == 0 && kk == 0)
                    printf("mma: tmem %x idesc %x adesc %llx bdesc %llx sa %x\n", tmem_base, idesc,
                           (unsigned long long)ad, (unsigned long long)bd, sa);
                mma_tf32(tmem_base, ad, bd, idesc, (i > 0 || kk > 0) ? 1u : 0u);
            }
            mma_commit(&empty[s]);
        }
        mma_commit(tmem_full);
    } else if (warp >= 2) {
        // ================= epilogue (warps 2..5) =================
        const int quarter = warp % 4;              // TMEM lane quarter this warp may access
        const int row = quarter * 32 + lane;       // accumulator row == TMEM lane
        if (nk > 0) {
            mbar_wait(tmem_full, 0);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        float* dst = nullptr;
        bool valid = false;
        if (P.mode == MODE_CONV) {
            const int ww = row % P.TW, hh = (row / P.TW) % P.TH, nn = row / (P.TW * P.TH);
            const int n = tn0 + nn, y = th0 + hh, x = tw0 + ww;
            valid = n < P.gn && y < P.gh && x < P.gw;
            if (valid) {
                const int64_t oy = static_cast<int64_t>(y) * P.out_s + P.py[phase];
                const int64_t ox = static_cast<int64_t>(x) * P.out_s + P.px[phase];
                valid = oy < P.out_h && ox < P.out_w;
                dst = P.out + ((static_cast<int64_t>(n) * P.out_h + oy) * P.out_w + ox) * P.ldc;
            }
        } else {
            const int64_t m = m0 + row;
            valid = m < P.M;
            float* base = P.splits > 1 ? P.partial + static_cast<int64_t>(blockIdx.z) * P.M * P.N : P.out;
            dst = base + m * P.ldc;
        }
        for (int c = 0; c < P.bn; c += 32) {
            uint32_t r[32];
            if (nk > 0) {
                tmem_ld32(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + static_cast<uint32_t>(c), r);
                if (P.debug && blockIdx.x == 0 && blockIdx.y == 0 && row < 2 && c == 0) {
                    const float* sa = reinterpret_cast<const float*>(smem);
                    printf("epi row %d nk %d r0 %f r1 %f smemA[0..3] %f %f %f %f\n", row, nk, __uint_as_float(r[0]),
                           __uint_as_float(r[1]), sa[0], sa[1], sa[2], sa[3]);
                }
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j) r[j] = 0u;
            }
            const int64_t col0 = n_col0 + c;
            if (!valid || col0 >= P.N) continue;
            float v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                v[j] = __uint_as_float(r[j]);
                if (P.bias && col0 + j < P.N) v[j] = __fadd_rn(v[j], __ldg(P.bias + col0 + j));
            }
            if (col0 + 32 <= P.N && (P.ldc % 4) == 0) {
#pragma unroll
                for (int j = 0; j < 32; j += 4)
                    *reinterpret_cast<float4*>(dst + col0 + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
            } else {
                for (int j = 0; j < 32 && col0 + j < P.N; ++j) dst[col0 + j] = v[j];
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(tmem_cols));
    }
}

__global__ void splitk_reduce_kernel(const float* __restrict__ partial, float* __restrict__ out, int64_t count,
                                     int splits) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        float s = partial[i];
        for (int k = 1; k < splits; ++k) s = __fadd_rn(s, partial[k * count + i]);
        out[i] = s;
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

bool encode_4d(CUtensorMap* map, const float* base, int64_t c, int64_t w, int64_t h, int64_t n, int bc, int bw,
               int bh, int bnn, int ew, int eh, bool mn_major, int64_t pitch = 0) {
    if (pitch == 0) pitch = c;   // elements between consecutive pixels
    cuuint64_t dims[4] = {(cuuint64_t)c, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)n};
    cuuint64_t strides[3] = {(cuuint64_t)(pitch * 4), (cuuint64_t)(pitch * w * 4), (cuuint64_t)(pitch * w * h * 4)};
    cuuint32_t box[4] = {(cuuint32_t)bc, (cuuint32_t)bw, (cuuint32_t)bh, (cuuint32_t)bnn};
    cuuint32_t es[4] = {1, (cuuint32_t)ew, (cuuint32_t)eh, 1};
    CUresult r = nncb::drv::table().tensorMapEncodeTiled(
        map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(base), dims, strides, box, es,
        CU_TENSOR_MAP_INTERLEAVE_NONE, mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
        CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) nncb::set_error(std::string("cuTensorMapEncodeTiled(4d): ") + nncb::drv::error_string(r));
    return r == CUDA_SUCCESS;
}

bool encode_2d(CUtensorMap* map, const float* base, int64_t inner, int64_t rows, int box_inner, int box_rows,
               bool mn_major) {
    cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)(inner * 4)};
    cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = nncb::drv::table().tensorMapEncodeTiled(
        map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
        CU_TENSOR_MAP_INTERLEAVE_NONE, mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
        CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) nncb::set_error(std::string("cuTensorMapEncodeTiled(2d): ") + nncb::drv::error_string(r));
    return r == CUDA_SUCCESS;
}

int pick_bn(int64_t n) {
    if (n <= 64) return 64;
    if (n <= 128) return 128;
    return n % 256 == 0 || n > 1024 ? 256 : 128;
}

// Chooses a pixel box (TN, TH, TW) of `rows` pixels over a (gn, gh, gw) grid:
// TW the smallest power of two >= gw (capped), then TH, then TN.
void pick_box(int rows, int gn, int gh, int gw, int& TN, int& TH, int& TW) {
    TW = 1;
    while (TW < gw && TW < rows) TW *= 2;
    TH = 1;
    while (TW * TH < rows && TH < gh) TH *= 2;
    while (TW * TH > rows) TH /= 2;
    if (TH < 1) TH = 1;
    TN = rows / (TW * TH);
    (void)gn;
}

size_t smem_for(int bn) { return STAGES * (BM * BK * 4 + static_cast<size_t>(bn) * BK * 4) + 1024 + 256; }

int launch(nncb_ctx* ctx, const CUtensorMap& ma, const CUtensorMap& mb, const TcParams& P, dim3 grid) {
    static bool attr_done = false;
    if (!attr_done) {
        NNCB_CUDA(cudaFuncSetAttribute(tc_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem_for(256))));
        attr_done = true;
    }
    tc_gemm_kernel<<<grid, THREADS, smem_for(P.bn), ctx->stream>>>(ma, mb, P);
    NNCB_LAUNCHED(ctx);
    return 0;
}

}  // namespace

namespace nncb {

int gemm_tc_impl(nncb_ctx* ctx, const nncb_gemm_desc* d, const float* a, int64_t lda, const float* b,
                 const float* bias, float* out, bool* handled);

__global__ void im2col_k(const float* __restrict__ x, float* __restrict__ cols, nncb_gemm_desc g, int64_t K,
                         int64_t ldk) {
    // cols[p, k], p = (n, oh, ow), k = (dh, dw, c); zero where the tap is padding
    int64_t total = g.n * g.oh * g.ow * ldk;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        int64_t k = t % ldk, p = t / ldk;
        float v = 0.f;
        if (k < K) {
            int64_t c = k % g.ci, tap = k / g.ci, dw = tap % g.kw, dh = tap / g.kw;
            int64_t ow = p % g.ow, r = p / g.ow, oh = r % g.oh, n = r / g.oh;
            int64_t h = oh * g.sh + dh - g.pad_top, w = ow * g.sw + dw - g.pad_left;
            if (h >= 0 && h < g.ih && w >= 0 && w < g.iw) v = __ldg(x + ((n * g.ih + h) * g.iw + w) * g.ci + c);
        }
        cols[t] = v;
    }
}

int gemm_tc(nncb_ctx* ctx, const nncb_gemm_desc* d, const float* a, const float* b, const float* bias, float* out,
            bool* handled) {
    *handled = false;
    const bool conv = d->kind >= NNCB_CONV_FWD;
    if (conv && d->ci % 32 != 0 && (d->kind == NNCB_CONV_FWD || d->kind == NNCB_CONV_WGRAD) && drv::table().ok) {
        // Channels that do not fill a 32-wide K block (the 3-channel stem): lower
        // to a dense tensor-core GEMM over an im2col workspace [pixels, kh*kw*ci].
        const int64_t K = d->kh * d->kw * d->ci, ldk = (K + 3) / 4 * 4;
        const int64_t P = d->n * d->oh * d->ow;
        if (d->co % 4 != 0 || d->co < 16) return 0;
        float* cols = static_cast<float*>(workspace(ctx, sizeof(float) * P * ldk));
        if (!cols) return fail("im2col: workspace allocation failed");
        im2col_k<<<grid_for(ctx, P * ldk, 256), 256, 0, ctx->stream>>>(a, cols, *d, K, ldk);
        NNCB_LAUNCHED(ctx);
        nncb_gemm_desc dd{};
        dd.kind = d->kind == NNCB_CONV_FWD ? NNCB_DENSE_FWD : NNCB_DENSE_WGRAD;
        dd.precision = d->precision;
        dd.epilogue = d->epilogue;
        dd.batch = P;
        dd.in_f = K;
        dd.out_f = d->co;
        int rc = gemm_tc_impl(ctx, &dd, cols, ldk, b, bias, out, handled);
        if (!rc && !*handled) return fail("im2col route: dense GEMM rejected");
        return rc;
    }
    return gemm_tc_impl(ctx, d, a, 0, b, bias, out, handled);
}

int gemm_tc_impl(nncb_ctx* ctx, const nncb_gemm_desc* d, const float* a, int64_t lda, const float* b,
                 const float* bias, float* out, bool* handled) {
    *handled = false;
    if (!drv::table().ok) return 0;
    static const int dbg = getenv("NNCB_TC_DEBUG") ? 1 : 0;
    const bool dense = d->kind <= NNCB_DENSE_WGRAD;
    // Conv geometry of the contraction (dense = 1x1 conv over [batch, 1, 1, features]).
    int64_t n = dense ? d->batch : d->n;
    int64_t ih = dense ? 1 : d->ih, iw = dense ? 1 : d->iw;
    int64_t ci = dense ? d->in_f : d->ci, co = dense ? d->out_f : d->co;
    int64_t kh = dense ? 1 : d->kh, kw = dense ? 1 : d->kw, sh = dense ? 1 : d->sh, sw = dense ? 1 : d->sw;
    int64_t oh = dense ? 1 : d->oh, ow = dense ? 1 : d->ow, pt = dense ? 0 : d->pad_top, pl = dense ? 0 : d->pad_left;
    const int kind = dense ? (d->kind == NNCB_DENSE_FWD ? 0 : d->kind == NNCB_DENSE_DGRAD ? 1 : 2)
                           : (d->kind == NNCB_CONV_FWD ? 0 : d->kind == NNCB_CONV_DGRAD ? 1 : 2);
    // Requirements of the TMA path: 32-channel K blocks for multi-tap convs
    // (single-tap contractions take a ragged last block, zero-filled by TMA),
    // 16-byte row pitches, taps fit the parameter block, int32 coordinates.
    const bool single_tap = kh * kw == 1;
    if (lda == 0) lda = ci;
    if (co % 4 != 0 || co < 16 || kh * kw > MAX_TAPS || lda % 4 != 0) return 0;
    if (!single_tap && ci % 32 != 0) return 0;
    if (single_tap && ci % 4 != 0 && lda == ci) return 0;
    if (kind == 1 && ((!single_tap && co % 32 != 0) || sh > 2 || sw > 2)) return 0;
    if (n * std::max(ih, oh) * std::max(iw, ow) * std::max(ci, co) >= (int64_t(1) << 31) * 4) return 0;

    TcParams P;
    memset(&P, 0, sizeof(P));
    P.debug = dbg;
    CUtensorMap ma, mb;
    if (kind == 0 || kind == 1) {
        P.mode = MODE_CONV;
        const bool fwd = kind == 0;
        const int64_t Nc = fwd ? co : ci;             // GEMM N
        const int64_t Ck = fwd ? ci : co;             // channels per tap (K block source)
        P.bn = pick_bn(Nc);
        P.N = Nc;
        P.ldc = Nc;
        P.cblocks = static_cast<int>((Ck + 31) / 32);
        if (fwd) {
            P.gn = (int)n; P.gh = (int)oh; P.gw = (int)ow;
            P.out_h = (int)oh; P.out_w = (int)ow; P.out_s = 1;
            P.mh = (int)sh; P.mw = (int)sw;
            P.ntaps[0] = (int)(kh * kw);
            P.tap0[0] = 0;
            for (int t = 0; t < kh * kw; ++t) {
                P.off_h[t] = (int)(t / kw - pt);
                P.off_w[t] = (int)(t % kw - pl);
                P.brow[t] = (int)(t * ci);
            }
        } else {
            // sub-pixel phases: h = a*sh + ph; taps with (ph + pt - dh) % sh == 0
            P.gn = (int)n; P.gh = (int)((ih + sh - 1) / sh); P.gw = (int)((iw + sw - 1) / sw);
            P.out_h = (int)ih; P.out_w = (int)iw; P.out_s = (int)sh;
            if (sh != sw) return 0;
            P.mh = 1; P.mw = 1;
            int nt = 0;
            for (int ph = 0; ph < sh; ++ph)
                for (int pw = 0; pw < sw; ++pw) {
                    int phase = ph * (int)sw + pw;
                    P.py[phase] = ph;
                    P.px[phase] = pw;
                    P.tap0[phase] = nt;
                    // visit taps so that the partial order matches (oh, ow) ascending
                    for (int64_t dh = kh - 1; dh >= 0; --dh)
                        for (int64_t dw = kw - 1; dw >= 0; --dw) {
                            int64_t th = ph + pt - dh, tw = pw + pl - dw;
                            if (((th % sh) + sh) % sh || ((tw % sw) + sw) % sw) continue;
                            if (nt >= MAX_TAPS) return 0;
                            P.off_h[nt] = (int)(th >= 0 ? th / sh : -((-th) / sh));
                            P.off_w[nt] = (int)(tw >= 0 ? tw / sw : -((-tw) / sw));
                            P.brow[nt] = (int)((dh * kw + dw) * ci);
                            ++nt;
                        }
                    P.ntaps[phase] = nt - P.tap0[phase];
                }
        }
        pick_box(BM, P.gn, P.gh, P.gw, P.TN, P.TH, P.TW);
        P.tiles_w = (P.gw + P.TW - 1) / P.TW;
        P.tiles_h = (P.gh + P.TH - 1) / P.TH;
        const int tiles_n = (P.gn + P.TN - 1) / P.TN;
        const int64_t tiles = static_cast<int64_t>(tiles_n) * P.tiles_h * P.tiles_w;
        if (tiles >= (int64_t(1) << 31) || P.TW * P.mw > 256 || P.TH * P.mh > 256) return 0;
        // A: the activation (x for fwd, g for dgrad) as {C, W, H, N}
        const float* act = a;
        if (fwd) {
            if (!encode_4d(&ma, act, ci, iw, ih, n, 32, P.TW * (int)sw, P.TH * (int)sh, P.TN, (int)sw, (int)sh, false, lda))
                return 1;
        } else {
            if (!encode_4d(&ma, act, co, ow, oh, n, 32, P.TW, P.TH, P.TN, 1, 1, false)) return 1;
        }
        // B: weights [kh*kw*ci, co]
        if (fwd) {
            P.b_mn = 1;
            if (!encode_2d(&mb, b, co, kh * kw * ci, 32, BK, true)) return 1;
        } else {
            P.b_mn = 0;
            if (!encode_2d(&mb, b, co, kh * kw * ci, BK, P.bn, false)) return 1;
        }
        P.bias = (fwd && (d->epilogue & NNCB_EPI_BIAS)) ? bias : nullptr;
        P.out = out;
        dim3 grid(static_cast<unsigned>(tiles), static_cast<unsigned>((Nc + P.bn - 1) / P.bn),
                  static_cast<unsigned>(fwd ? 1 : sh * sw));
        *handled = true;
        return launch(ctx, ma, mb, P, grid);
    }
    // ---- wgrad ----------------------------------------------------------------
    P.mode = MODE_WGRAD;
    P.b_mn = 1;
    P.M = kh * kw * ci;
    P.N = co;
    P.ldc = co;
    P.bn = pick_bn(co);
    P.ci = (int)ci;
    P.kw_ = (int)kw;
    P.sh = (int)sh; P.sw = (int)sw; P.pt = (int)pt; P.pl = (int)pl;
    P.gn = (int)n; P.gh = (int)oh; P.gw = (int)ow;
    pick_box(BK, P.gn, P.gh, P.gw, P.TN, P.TH, P.TW);
    P.tiles_w = (P.gw + P.TW - 1) / P.TW;
    P.tiles_h = (P.gh + P.TH - 1) / P.TH;
    const int64_t kboxes = static_cast<int64_t>((P.gn + P.TN - 1) / P.TN) * P.tiles_h * P.tiles_w;
    if (kboxes >= (int64_t(1) << 31) || P.TW * sw > 256 || P.TH * sh > 256) return 0;
    P.kboxes = static_cast<int>(kboxes);
    const int64_t mt = (P.M + BM - 1) / BM, nt = (co + P.bn - 1) / P.bn;
    int64_t splits = (2 * static_cast<int64_t>(ctx->sm_count)) / std::max<int64_t>(mt * nt, 1);
    splits = std::max<int64_t>(1, std::min<int64_t>(splits, std::max<int64_t>(kboxes / 8, 1)));
    splits = std::min<int64_t>(splits, 128);
    P.splits = static_cast<int>(splits);
    if (!encode_4d(&ma, a, ci, iw, ih, n, 32, P.TW * (int)sw, P.TH * (int)sh, P.TN, (int)sw, (int)sh, true, lda))
        return 1;
    if (!encode_4d(&mb, b, co, ow, oh, n, 32, P.TW, P.TH, P.TN, 1, 1, true)) return 1;
    P.out = out;
    if (P.splits > 1) {
        P.partial = static_cast<float*>(scratch(ctx, sizeof(float) * P.splits * P.M * P.N));
        if (!P.partial) return fail("wgrad: split-K workspace allocation failed");
    }
    dim3 grid(static_cast<unsigned>(mt), static_cast<unsigned>(nt), static_cast<unsigned>(P.splits));
    *handled = true;
    if (int rc = launch(ctx, ma, mb, P, grid)) return rc;
    if (P.splits > 1) {
        int64_t count = P.M * P.N;
        splitk_reduce_kernel<<<grid_for(ctx, count, 256), 256, 0, ctx->stream>>>(P.partial, out, count, P.splits);
        NNCB_LAUNCHED(ctx);
    }
    return 0;
}

}  // namespace nncb
