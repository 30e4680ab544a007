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
#include <algorithm>
#include <atomic>
#include <vector>
#include <string>
#include <mutex>
#include <map>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <cuda_bf16.h>

#include "driver_api.cuh"
#include "nncb_internal.cuh"

namespace {

constexpr int BM = 128;       // UMMA_M (cta_group::1)
constexpr int BK = 32;        // fp32 elements per K step = one 128-byte swizzle row
constexpr int MAX_STAGES = 6;
constexpr int THREADS = 320;   // warp 0 TMA, warp 1 MMA, warps 2..9 epilogue (2 per TMEM lane quarter)
constexpr int MAX_TAPS = 64;
constexpr int HALO_TW = 8, HALO_TH = 16;
constexpr uint32_t HALO_A_BYTES = (HALO_TW + 2) * HALO_TH * 128;   // 20 KB, 1 KB-aligned
constexpr uint32_t HALO9_A_BYTES = ((HALO_TW + 2) * (HALO_TH + 2) * 128 + 1023) / 1024 * 1024;   // full 3x3 patch, 23 KB

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
    int dil_w;          // horizontal tap dilation (space-to-depth packing); 1 otherwise
    int bt;             // MODE_CONV forward with K-major (transposed) weights: B box at (tap*ci + c0, n0)
    // --- gradient epilogue (NNCB_EPI_RELU_GRAD; requires the CS build, colstats = eg sums) ---
    int eg;
    const float* eg_mask;
    const float* eg_res;
    const float* eg_x;
    const float* eg_stats;
    int eg_side;        // TMA-staged side tiles per pass (2: mask, x; 3: + residual); 0: per-row loads
    int sh, sw, pt, pl;
    int kboxes;         // pixel boxes (TN*TH*TW == 32 pixels each)
    int splits;
    float* partial;     // [splits][M][N] when splits > 1
    const float* bias;  // MODE_CONV forward only
    float* out;
    int debug;
    // persistent tiling
    int64_t tiles;      // total tiles (all phases / splits)
    int64_t n_tiles;    // tiles along N
    int64_t pix_tiles;  // MODE_CONV: pixel tiles per phase
    int64_t m_tiles;    // MODE_WGRAD: tiles along M
    int tma_store;      // epilogue through smem + TMA store (else direct stores)
    int stages;         // smem ring depth (sized so 2 CTAs fit per SM when N is small)
    int nostore;        // tuning knob: skip the output stores (epilogue cost probe)
    unsigned long long* trace;   // probe (NNCB_TC_TRACE): per CTA / local tile event timestamps
    int stg_cols;       // epilogue transpose width per pass: 32, 16 or 8 columns (4/2/1 KB per warp)
    int stg_bufs;       // staging tiles per warp: 2 lets a pass's TMA store overlap staging of the next
    // --- halo (3x3 stride-1 forward): one (TW+2) x TH input patch per (32-channel
    // block, kernel row) feeds the row's three taps through shifted descriptors
    // (TW = 8, TH = 16, TN = 1: each 8-row core-matrix group is one image row,
    // group stride TW + 2 rows); a stage = patch + the three taps' B tiles
    int halo;
    // halo with resident B (single N tile): every tap / channel-block B tile is
    // loaded once per CTA into bres_bytes at the front of shared memory, and
    // stages carry only patches
    int bres;
    uint32_t bres_bytes;
    int halo_kw;        // halo 1: taps per kernel row (3; 2 for the space-to-depth stem, spaced dil_w rows)
    double* colstats;   // fused BatchNorm statistics: [0,N) sum, [N,2N) sum of squares
    // order-independent accumulation of colstats: per column two fixed-point
    // (2^-40) sums split in 32-bit limbs, [sum hi | sum lo | sq hi | sq lo][N],
    // then a CTA ticket counter; the last CTA converts to the doubles above
    unsigned long long* cs_fixed;
    float* cs_stats;    // NNCB_EPI_COLSTATS + colstats_finalize: the last CTA also writes mean / invstd
    double cs_eps;
    int64_t cs_rows;
    // --- manual A (channel counts that do not fill a 32-wide TMA block) -----
    // Builder warps gather A straight from the NHWC activation into the
    // K-major 128B-swizzled stage layout: no im2col matrix in HBM.
    const float* xa;    // activation [gn?, ih, iw, ci]
    int ih_, iw_;       // activation image dims
    int K_;             // kh*kw*ci
    // --- CTA pair (cta_group::2): 256-row tiles over two SMs ----------------
    int pair;           // 1: cluster of 2, leader issues M=256 MMAs, each CTA loads half of B
    int tma_out;        // epilogue stores through TMA: 1 = 4-D pixel grid (stride-1 outputs), 2 = 3-D [splits][M][N]
    int ob_w, ob_h, ob_n;   // tma_out 1: a warp's 32-row sub-box of the pixel tile
    int64_t pix_pairs;  // MODE_CONV: pixel-box pairs per phase
    int64_t m_pairs;    // MODE_WGRAD: M-tile pairs
    // bf16 operands (NNCB_PREC_BF16): tcgen05.mma kind::f16 on bf16 A/B tiles
    // with fp32 accumulation in TMEM. A 128-byte swizzle row holds kel = 64 K
    // elements (32 for tf32); one MMA consumes 32 bytes of K in both kinds, so
    // the smem ring and descriptors are byte-identical.
    int bf16;
    int kel;
    // inference BatchNorm (+ ReLU) of the output column in the epilogue
    const float* bn_mean;
    const float* bn_inv;     // (float)(1/sqrt((double)var + eps)), computed per call
    const float* bn_gamma;
    const float* bn_beta;
    int relu;
    const float* res;        // residual added after the BatchNorm (inference join)
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

// 4-byte global->shared async copy; src_bytes 0 zero-fills the destination
__device__ __forceinline__ void cp_async4(void* dst, const float* src, int src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(src_bytes)
                 : "memory");
}

// arrive on `bar` once all of this thread's prior cp.async copies have landed
__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// CTA-pair variants: the mbarrier operand is a shared::cluster address (the
// leader CTA's barrier), the destination is this CTA's own shared memory.
__device__ __forceinline__ void tma_load_4d_pair(void* dst, const CUtensorMap* map, uint32_t bar, int c0, int c1,
                                                 int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
        "%3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
        "%3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

// shared::cluster address of `p`'s counterpart in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_u32(const void* p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
    return r;
}

__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx_cluster(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
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

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
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
// true in exactly one lane of the (fully active) warp
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
    return pred != 0;
}

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

// kind::f16 with BF16 operands (NNCB_PREC_BF16); the pair form as below
__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_f16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// CTA pair: M=256 MMA issued by the leader over both CTAs' shared memory
__device__ __forceinline__ void mma_tf32_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// completion of the leader's MMAs arrives on the barrier at the same offset in both CTAs
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(smem_u32(bar)), "h"(static_cast<uint16_t>(3))
                 : "memory");
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// Probe (NNCB_TC_TRACE, tools/tc_trace.py): event timestamps per CTA and local
// tile -- 0 MMA tile start, 1 MMA commit, 2 epilogue sees the accumulator,
// 3 its TMEM release, 4/5 epilogue warps 2/9 done, 6 producer tile start.
// Compiled in only with -DNNCB_TC_TRACE_PROBE (it costs the register-capped
// builds stack space); `make PROBE=1` builds it.
#ifdef NNCB_TC_TRACE_PROBE
#define TC_TRACE(local, ev)                                                                                   \
    do {                                                                                                      \
        if (P.trace && (local) < 64) P.trace[(static_cast<int64_t>(blockIdx.x) * 64 + (local)) * 8 + (ev)] = gtimer(); \
    } while (0)
#else
#define TC_TRACE(local, ev) \
    do {                    \
    } while (0)
#endif

// Order-independent column sums: v is added as round-toward-zero fixed point
// with 40 fraction bits, split into a high part (v / 2^-8, integer) and a low
// 32-bit part, each accumulated by 64-bit integer atomics (exact, so the
// total does not depend on the order in which CTAs and warps flush). |sum| <
// 2^55; each contribution loses < 2^-40 (below every float32 BatchNorm
// statistic's resolution here).
__device__ __forceinline__ void fixed_add(unsigned long long* hi, unsigned long long* lo, double v) {
    const double t = v * 1099511627776.0;                  // 2^40
    const double h = floor(t * 2.3283064365386963e-10);   // floor(t / 2^32)
    const double l = t - h * 4294967296.0;                 // [0, 2^32): exact
    atomicAdd(hi, static_cast<unsigned long long>(static_cast<long long>(h)));
    atomicAdd(lo, static_cast<unsigned long long>(l));
}
__device__ __forceinline__ double fixed_value(unsigned long long hi, unsigned long long lo) {
    return static_cast<double>(static_cast<long long>(hi)) * 0.00390625 +   // 2^-8
           static_cast<double>(lo) * 9.094947017729282e-13;                // 2^-40
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

__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, const void* src, int c0, int c1, int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
            reinterpret_cast<uint64_t>(map)),
        "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// Store one warp's 32x32 fp32 accumulator chunk (row `lane` in r[0..31]) to
// global memory through a per-warp shared-memory transpose of width
// CH*4 columns (CH 16-byte chunks per row, XOR-swizzled by row), so that each
// store instruction writes 32/CH whole row segments of CH*16 contiguous
// bytes instead of 32 scattered 16-byte pieces.
//
// CS: also return BatchNorm column statistics of the valid rows, read from the
// staged tile: with COLS columns per pass, lane l sums column l % COLS over
// rows [(l / COLS) * RPL, +RPL), the 32/COLS row groups are folded with xor
// shuffles, and the pass's sums move to lane (pass * COLS + column), so on
// return lane l holds (sum, sum of squares) of chunk column l in cs1 / cs2.
// 16-byte chunk position of chunk j in staged row rr: TMA's SWIZZLE_128B / 64B /
// 32B patterns for 128 / 64 / 32-byte rows (address bits [4:6] ^= [7:9] on a
// 1 KB-aligned tile), so a staged chunk can leave through a TMA store as is.
template <int CH>
__device__ __forceinline__ int swz(int j, int rr) {
    return CH == 8 ? (j ^ (rr & 7)) : CH == 4 ? (j ^ ((rr >> 1) & 3)) : (j ^ ((rr >> 2) & 1));
}

// TMA epilogue: the staged COLS-wide pass leaves as one tensor store of the
// warp's 32-row sub-box (mode 1: 4-D pixel grid, mode 2: 3-D [split][row][col]).
// Side inputs of the gradient epilogue (mask, x, residual), encoded with the
// output map's geometry and swizzle so a side tile has the staging tile's layout.
struct alignas(64) EgMaps {
    CUtensorMap m[3];
};

struct TmaOut {
    const CUtensorMap* map;
    int mode;           // 0: direct stores
    int c1, c2, c3;     // non-column box coordinates
};

// Gradient-epilogue side tiles: one warp's 32 rows x COLS columns of each side
// input at output column `col`, into its side buffer (lane 0 only).
// Double-buffered: item i (a pass of one chunk of one tile, in the warp's
// processing order) lands in buffer i & 1; item i + 1 is issued before item i
// is consumed, so one load is always in flight behind the computation.
struct EgSide {
    const EgMaps* maps;
    uint8_t* buf;        // 2 buffers of eg_side tiles of COLS * 128 bytes
    uint64_t* bar;       // [2]
    uint32_t issued, consumed;
    TmaOut next_to;      // the item after this chunk's last pass: next chunk or next tile
    int next_col;        // (-1: none known yet)
};

template <int COLS>
__device__ __forceinline__ void eg_side_load(EgSide& es, int n, const TmaOut& to, int col) {
    const uint32_t b = es.issued & 1u;
    uint8_t* dst = es.buf + b * n * COLS * 128;
    mbar_expect_tx(&es.bar[b], static_cast<uint32_t>(n * COLS * 128));
    for (int a = 0; a < n; ++a) {
        if (to.mode == 1)
            tma_load_4d(dst + a * COLS * 128, &es.maps->m[a], &es.bar[b], col, to.c1, to.c2, to.c3);
        else
            tma_load_3d(dst + a * COLS * 128, &es.maps->m[a], &es.bar[b], col, to.c1, to.c2);
    }
}

template <int CH, bool CS, bool EG = false>
__device__ __forceinline__ void store_chunk_t(const uint32_t (&r)[32], uint8_t* tile0, float* dst, bool valid,
                                              int col0, int N, bool full_cols, int lane, bool store, float& cs1,
                                              float& cs2, const TmaOut& to, const TcParams& P, EgSide& es,
                                              uint32_t& seq) {
    constexpr int COLS = CH * 4, RPI = 32 / CH;   // columns per pass, rows per store instruction
    const uint32_t vmask = CS ? __ballot_sync(0xffffffffu, valid) : 0u;
#pragma unroll
    for (int p = 0; p < 32 / COLS; ++p) {
        // two staging tiles: this pass fills one while the previous pass's TMA
        // store may still be reading the other (one bulk group per pass)
        uint8_t* tile = tile0 + (P.stg_bufs == 2 ? (seq & 1u) * (COLS * 128) : 0);
        ++seq;
        if (to.mode) {   // the TMA store that last read this tile has finished reading it
            if (lane == 0) {
                if (P.stg_bufs == 2)
                    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                else
                    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            }
            __syncwarp();
        }
        uint8_t* rowp = tile + lane * (CH * 16);
#pragma unroll
        for (int j = 0; j < CH; ++j)
            *reinterpret_cast<uint4*>(rowp + (swz<CH>(j, lane) << 4)) =
                make_uint4(r[p * COLS + 4 * j], r[p * COLS + 4 * j + 1], r[p * COLS + 4 * j + 2], r[p * COLS + 4 * j + 3]);
        __syncwarp();
        if (CS && !EG && CH < 8) {
            // Narrow staging (8 / 16 columns per pass): lane (column, row group)
            // sums its rows of one column, so the fold across row groups is 2 or
            // 1 shuffle levels (the 16-byte layout below would need 4 or 3).
            constexpr int RPL = COLS;              // rows per lane: 32 rows over 32/COLS lane groups
            const int col = lane % COLS, r0 = (lane / COLS) * RPL;
            float s1 = 0.f, s2 = 0.f;
#pragma unroll
            for (int i = 0; i < RPL; ++i) {
                const int rr = r0 + i;
                const float v = *reinterpret_cast<const float*>(tile + rr * (CH * 16) + (swz<CH>(col >> 2, rr) << 4) + (col & 3) * 4);
                const float m = ((vmask >> rr) & 1u) ? v : 0.f;
                s1 += m;
                s2 = fmaf(m, m, s2);
            }
#pragma unroll
            for (int sh = COLS; sh < 32; sh <<= 1) {
                s1 += __shfl_xor_sync(0xffffffffu, s1, sh);
                s2 += __shfl_xor_sync(0xffffffffu, s2, sh);
            }
            // lanes [p*COLS, (p+1)*COLS) take columns p*COLS.. from lanes 0..COLS-1
            const float t1 = __shfl_sync(0xffffffffu, s1, lane % COLS);
            const float t2 = __shfl_sync(0xffffffffu, s2, lane % COLS);
            if (lane / COLS == p) {
                cs1 = t1;
                cs2 = t2;
            }
        } else if (CS && !(EG && !P.eg_side)) {
            // Vectorised column statistics: lane (chunk j, row group g) owns the
            // pass's columns 4j..4j+3 over rows g, g + RG, ... (16-byte shared
            // loads / stores, conflict-free under the swizzle), then the row
            // groups fold with xor shuffles. CS alone: sum v, sum v^2 of the
            // GEMM result (BatchNorm forward). EG: the staged result becomes
            // dy = mask > 0 ? acc (+ res) : 0 in place, from side tiles in the
            // same layout, with sum dy, sum dy * xhat (BatchNorm backward).
            constexpr int RG = 32 / CH;
            const int j = lane % CH, g = lane / CH;
            const int cg0 = col0 + p * COLS + 4 * j;
            float a1[4] = {0.f, 0.f, 0.f, 0.f}, a2[4] = {0.f, 0.f, 0.f, 0.f};
            float em[4] = {0.f, 0.f, 0.f, 0.f}, ev[4] = {0.f, 0.f, 0.f, 0.f};
            const uint8_t* sm = nullptr;
            if (EG) {
                if (cg0 < N) {   // N % 4 == 0 on the side-tile path (TMA output)
                    const float4 m4 = __ldg(reinterpret_cast<const float4*>(P.eg_stats + cg0));
                    const float4 s4 = __ldg(reinterpret_cast<const float4*>(P.eg_stats + N + cg0));
                    em[0] = m4.x; em[1] = m4.y; em[2] = m4.z; em[3] = m4.w;
                    ev[0] = s4.x; ev[1] = s4.y; ev[2] = s4.z; ev[3] = s4.w;
                }
                if (es.issued == es.consumed + 1) {   // keep the following item in flight
                    const bool more = p + 1 < 32 / COLS;
                    const int nc = more ? col0 + (p + 1) * COLS : es.next_col;
                    if (nc >= 0) {
                        if (lane == 0) eg_side_load<COLS>(es, P.eg_side, more ? to : es.next_to, nc);
                        ++es.issued;
                    }
                }
                const uint32_t b = es.consumed & 1u;
                mbar_wait(&es.bar[b], (es.consumed >> 1) & 1u);
                sm = es.buf + b * P.eg_side * COLS * 128;
            }
#pragma unroll
            for (int i = 0; i < CH; ++i) {
                const int rr = g + i * RG;
                const int o = rr * (CH * 16) + (swz<CH>(j, rr) << 4);
                const bool rv = (vmask >> rr) & 1u;
                float4 v = *reinterpret_cast<const float4*>(tile + o);
                float e[4] = {v.x, v.y, v.z, v.w};
                if (EG) {
                    const float4 m4 = *reinterpret_cast<const float4*>(sm + o);
                    const float4 x4 = *reinterpret_cast<const float4*>(sm + COLS * 128 + o);
                    const float mk[4] = {m4.x, m4.y, m4.z, m4.w}, xv[4] = {x4.x, x4.y, x4.z, x4.w};
                    if (P.eg_side == 3) {
                        const float4 r4 = *reinterpret_cast<const float4*>(sm + 2 * COLS * 128 + o);
                        e[0] = __fadd_rn(e[0], r4.x);
                        e[1] = __fadd_rn(e[1], r4.y);
                        e[2] = __fadd_rn(e[2], r4.z);
                        e[3] = __fadd_rn(e[3], r4.w);
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        e[q] = (rv && mk[q] > 0.f) ? e[q] : 0.f;   // out-of-range columns: side tiles are 0
                        a1[q] += e[q];
                        a2[q] = fmaf(e[q], (xv[q] - em[q]) * ev[q], a2[q]);
                    }
                    *reinterpret_cast<float4*>(tile + o) = make_float4(e[0], e[1], e[2], e[3]);
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const float m = rv ? e[q] : 0.f;
                        a1[q] += m;
                        a2[q] = fmaf(m, m, a2[q]);
                    }
                }
            }
            if (EG) {
                __syncwarp();   // side buffer consumed (free for item consumed + 2); dy staged for the store
                ++es.consumed;
            }
#pragma unroll
            for (int sh = CH; sh < 32; sh <<= 1)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    a1[q] += __shfl_xor_sync(0xffffffffu, a1[q], sh);
                    a2[q] += __shfl_xor_sync(0xffffffffu, a2[q], sh);
                }
            // lanes [p*COLS, (p+1)*COLS) take column lane % COLS of this pass
            // from the lane holding its 4-column chunk (row group 0: lane cc / 4)
            const int cc = lane % COLS;
            float t1 = 0.f, t2 = 0.f;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float u1 = __shfl_sync(0xffffffffu, a1[q], cc >> 2);
                const float u2 = __shfl_sync(0xffffffffu, a2[q], cc >> 2);
                if ((cc & 3) == q) {
                    t1 = u1;
                    t2 = u2;
                }
            }
            if (lane / COLS == p) {
                cs1 = t1;
                cs2 = t2;
            }
        } else if (CS) {
            // gradient epilogue without side tiles (direct-store outputs): lane
            // (col, row group) reads its rows' mask / residual / x from global
            // memory, 8 rows of loads in flight at a time
            constexpr int RPL = COLS;
            const int col = lane % COLS, r0 = (lane / COLS) * RPL;
            float s1 = 0.f, s2 = 0.f;
            const int cg = col0 + p * COLS + col;
            const int64_t doff = static_cast<int64_t>(dst - P.out);   // this lane's row, output layout
            float em = 0.f, es_ = 0.f;
            if (cg < N) {
                em = __ldg(P.eg_stats + cg);
                es_ = __ldg(P.eg_stats + N + cg);
            }
            constexpr int BR = 8;
#pragma unroll
            for (int i0 = 0; i0 < RPL; i0 += BR) {
                float mv[BR], xv[BR], rs[BR];
#pragma unroll
                for (int i = 0; i < BR; ++i) {
                    const int rr = r0 + i0 + i;
                    const int64_t off = __shfl_sync(0xffffffffu, static_cast<long long>(doff), rr);
                    const bool ok = ((vmask >> rr) & 1u) && cg < N;
                    const int64_t e = ok ? off + cg : 0;
                    mv[i] = ok ? __ldg(P.eg_mask + e) : 0.f;
                    xv[i] = ok ? __ldg(P.eg_x + e) : 0.f;
                    rs[i] = (ok && P.eg_res) ? __ldg(P.eg_res + e) : 0.f;
                }
#pragma unroll
                for (int i = 0; i < BR; ++i) {
                    const int rr = r0 + i0 + i;
                    float* tp = reinterpret_cast<float*>(tile + rr * (CH * 16) + (swz<CH>(col >> 2, rr) << 4) + (col & 3) * 4);
                    const float gsum = P.eg_res ? __fadd_rn(*tp, rs[i]) : *tp;
                    const float dy = mv[i] > 0.f ? gsum : 0.f;   // invalid rows/cols: mask 0
                    *tp = dy;
                    s1 += dy;
                    s2 = fmaf(dy, (xv[i] - em) * es_, s2);
                }
            }
            __syncwarp();   // dy written back before the stores read the tile
#pragma unroll
            for (int sh = COLS; sh < 32; sh <<= 1) {
                s1 += __shfl_xor_sync(0xffffffffu, s1, sh);
                s2 += __shfl_xor_sync(0xffffffffu, s2, sh);
            }
            const float t1 = __shfl_sync(0xffffffffu, s1, lane % COLS);
            const float t2 = __shfl_sync(0xffffffffu, s2, lane % COLS);
            if (lane / COLS == p) {
                cs1 = t1;
                cs2 = t2;
            }
        }
        if (!store) {
            __syncwarp();
            continue;
        }
        if (to.mode) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // staged writes -> TMA (async proxy)
            __syncwarp();
            if (lane == 0) {
                if (to.mode == 1)
                    tma_store_4d(to.map, tile, col0 + p * COLS, to.c1, to.c2, to.c3);
                else
                    tma_store_3d(to.map, tile, col0 + p * COLS, to.c1, to.c2);
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            continue;
        }
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            const int rr = i * RPI + lane / CH, ch = lane % CH;
            float* rdst = reinterpret_cast<float*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(dst), rr));
            const int rvalid = __shfl_sync(0xffffffffu, valid ? 1 : 0, rr);
            const uint4 v4 = *reinterpret_cast<const uint4*>(tile + rr * (CH * 16) + (swz<CH>(ch, rr) << 4));
            if (!rvalid) continue;
            const int c = col0 + p * COLS + ch * 4;
            if (full_cols) {
                // explicit global store: the row pointer arrives through a shuffle,
                // so the compiler cannot prove its state space (generic ST.E otherwise)
                asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(rdst + c), "r"(v4.x), "r"(v4.y),
                             "r"(v4.z), "r"(v4.w)
                             : "memory");
            } else {
                const uint32_t e[4] = {v4.x, v4.y, v4.z, v4.w};
                for (int q = 0; q < 4; ++q)
                    if (c + q < N) rdst[c + q] = __uint_as_float(e[q]);
            }
        }
        __syncwarp();
    }
}


// Persistent warp-specialised GEMM. grid = min(tiles, #SMs); CTA b processes
// tiles b, b + grid, ... The smem ring (TMA -> MMA) and the double-buffered TMEM
// accumulator (MMA -> epilogue) carry their phases across tiles, so the
// epilogue of one tile overlaps the main loop of the next.
// MINB: CTAs per SM the build is register-budgeted for (2: <= 96 registers;
// 1: no cap, used by the 448-thread MA build and by CS with 256-wide tiles).
template <bool CS, bool MA, int MINB, bool PAIR, bool EG = false>
__global__ void __launch_bounds__(MA ? THREADS + 128 : THREADS, MINB)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                   const __grid_constant__ CUtensorMap map_c, const __grid_constant__ TcParams P,
                   const __grid_constant__ EgMaps eg_maps) {
    const int STAGES = P.stages;
    nncb::pdl_trigger();   // follow-up folds / finalizes may be scheduled while this grid drains
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* bres_base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* smem = bres_base + P.bres_bytes;   // the ring and everything after it
    // 16 KB (halo 1: 20 KB kernel-row patch; halo 2: 23 KB full 3x3 patch)
    const uint32_t a_bytes = P.halo == 2 ? HALO9_A_BYTES : P.halo ? HALO_A_BYTES : BM * BK * 4;
    // PAIR: this CTA holds half of the B tile's columns (the MMA spans both CTAs)
    const uint32_t bt_bytes = static_cast<uint32_t>(PAIR ? P.bn / 2 : P.bn) * BK * 4;   // one tap's B tile
    const uint32_t b_bytes = P.bres ? 0u : bt_bytes * (P.halo == 2 ? 9u : P.halo ? static_cast<uint32_t>(P.halo_kw) : 1u);
    // bytes the TMA loads of one stage deliver (the full patch is padded to 1 KB in smem)
    const uint32_t tx_bytes = (P.halo == 2 ? (HALO_TW + 2) * (HALO_TH + 2) * 128 : a_bytes) + b_bytes;
    const uint32_t rank = PAIR ? cluster_rank() : 0u;
    const uint32_t stage_bytes = a_bytes + b_bytes;
    uint8_t* staging = smem + STAGES * stage_bytes;       // 8 x stg_cols*128 B: one transpose tile per epilogue warp
    uint8_t* side = staging + 8 * P.stg_bufs * P.stg_cols * 128;   // EG: 8 x 2 x eg_side x stg_cols*128 B side tiles
    uint64_t* full = reinterpret_cast<uint64_t*>(side + (EG ? 16 * P.eg_side * P.stg_cols * 128 : 0));
    uint64_t* empty = full + STAGES;
    uint64_t* tmem_full = empty + STAGES;                 // [2]
    uint64_t* tmem_empty = tmem_full + 2;                 // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);
    uint64_t* side_bar = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(tmem_slot) + 16);   // [8][2]
    uint64_t* bres_bar = side_bar + 16;                   // resident B loaded
    // CS: per-CTA column sum / sum of squares of the current column range
    double* cs_acc = reinterpret_cast<double*>(side_bar + 18);
    // MA: gather tables after cs_acc (fwd: per K index; wgrad: per box pixel)
    int* ma_tab = reinterpret_cast<int*>(cs_acc + 2 * P.bn);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            // MA: + one arrival per builder thread; PAIR: both CTAs' producers arrive (leader's copy)
            mbar_init(&full[s], MA ? 1 + 128 : PAIR ? 2 : 1);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tmem_full[s], 1);
            mbar_init(&tmem_empty[s], PAIR ? 16 : 8);     // one arrival per epilogue warp (of both CTAs)
        }
        if (EG)
            for (int w = 0; w < 16; ++w) mbar_init(&side_bar[w], 1);
        if (P.bres) mbar_init(bres_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (MA) {
        if (P.mode == MODE_CONV) {
            // K index -> (source offset within the patch, dh, dw); padding K rows read nothing
            const int kpad = P.cblocks * BK;
            for (int k = threadIdx.x; k < kpad; k += blockDim.x) {
                const int c = k % P.ci, tap = k / P.ci, dw = tap % P.kw_, dh = tap / P.kw_;
                ma_tab[k] = (dh * P.iw_ + dw) * P.ci + c;
                ma_tab[kpad + k] = k < P.K_ ? dh : -(1 << 20);
                ma_tab[2 * kpad + k] = dw;
            }
        } else {
            // pixel k of a 32-pixel box -> (dn, dy, dx)
            for (int k = threadIdx.x; k < BK; k += blockDim.x) {
                ma_tab[k] = k / (P.TW * P.TH);
                ma_tab[BK + k] = (k / P.TW) % P.TH;
                ma_tab[2 * BK + k] = k % P.TW;
            }
        }
    }
    const uint32_t tmem_cols = 2 * static_cast<uint32_t>(P.bn);   // two accumulators
    if (warp == 1) {
        if (PAIR) {   // the same columns in both CTAs of the pair
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                         "r"(tmem_cols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                         "r"(tmem_cols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    if (PAIR)
        cluster_sync_all();   // peer barriers initialised before any remote arrive
    else
        __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem_base = *tmem_slot;
    // PAIR: both CTAs of a cluster walk the same tiles (one tile = both CTAs' rows)
    const int64_t t_begin = PAIR ? blockIdx.x / 2 : blockIdx.x, t_step = PAIR ? gridDim.x / 2 : gridDim.x;

    // ---- tile decode (identical in every role) ------------------------------
    struct Tile {
        int phase, tn0, th0, tw0, kb_begin, nk, split;
        int64_t m0, n0;
    };
    // 32-bit index arithmetic (the host caps tile counts below 2^31): every
    // role decodes each of its tiles, and 64-bit divisions cost ~4x more
    auto decode = [&](int64_t t64) {
        Tile T{};
        const uint32_t t = static_cast<uint32_t>(t64), nt = static_cast<uint32_t>(P.n_tiles);
        const uint32_t rest = t / nt;
        T.n0 = static_cast<int64_t>(t - rest * nt) * P.bn;
        if (P.mode == MODE_CONV) {
            // PAIR: tile t covers pixel boxes 2q, 2q+1 (one per CTA); a box past
            // the grid is fully out of bounds (zero loads, no stores)
            const uint32_t per = static_cast<uint32_t>(PAIR ? P.pix_pairs : P.pix_tiles);
            const uint32_t ph = rest / per, q = rest - ph * per;
            uint32_t pix = PAIR ? 2 * q + rank : q;
            T.phase = static_cast<int>(ph);
            const uint32_t tw_ = static_cast<uint32_t>(P.tiles_w), th_ = static_cast<uint32_t>(P.tiles_h);
            const uint32_t p1 = pix / tw_, p2 = p1 / th_;
            T.tn0 = static_cast<int>(p2) * P.TN;
            T.th0 = static_cast<int>(p1 - p2 * th_) * P.TH;
            T.tw0 = static_cast<int>(pix - p1 * tw_) * P.TW;
            T.kb_begin = 0;
            T.nk = P.ntaps[T.phase] * P.cblocks;
        } else {
            const uint32_t mper = static_cast<uint32_t>(PAIR ? P.m_pairs : P.m_tiles);
            const uint32_t sp = rest / mper, q = rest - sp * mper;
            T.m0 = static_cast<int64_t>(PAIR ? 2 * q + rank : q) * BM;
            T.split = static_cast<int>(sp);
            int per = (P.kboxes + P.splits - 1) / P.splits;
            T.kb_begin = min(P.kboxes, T.split * per);
            T.nk = min(P.kboxes, T.kb_begin + per) - T.kb_begin;
        }
        return T;
    };

    if (warp == 0 && lane == 0) {
        // ================= TMA producer =================
        if (!MA) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
        // Ring position (slot, phase) advances incrementally and box coordinates
        // are hoisted per tile / stepped like an odometer: this one thread
        // issues every load, so no divisions may sit on the per-k-step path.
        int slot = 0;
        uint32_t phase = 0, filled = 0;
        uint32_t bar_cl = 0;   // PAIR: the leader's full[slot] as a cluster address
        auto acquire = [&](uint8_t*& sa, uint64_t*& bar) {
            if (filled >= static_cast<uint32_t>(STAGES)) mbar_wait(&empty[slot], phase ^ 1u);
            sa = smem + slot * stage_bytes;
            bar = &full[slot];
            if (PAIR) {
                // the leader's barrier counts both CTAs' bytes and one arrival per
                // producer; these arrivals publish no data (the bytes come with
                // TMA complete_tx), so no cluster-scope release fence is needed
                bar_cl = mapa_u32(&full[slot], 0);
                if (rank == 0)
                    mbar_expect_tx(bar, 2 * stage_bytes);
                else
                    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cl) : "memory");
            } else {
                mbar_expect_tx(bar, MA ? b_bytes : tx_bytes);
            }
        };
        auto ld4 = [&](void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2, int c3) {
            if (PAIR)
                tma_load_4d_pair(dst, map, bar_cl, c0, c1, c2, c3);
            else
                tma_load_4d(dst, map, bar, c0, c1, c2, c3);
        };
        auto ld2 = [&](void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
            if (PAIR)
                tma_load_2d_pair(dst, map, bar_cl, c0, c1);
            else
                tma_load_2d(dst, map, bar, c0, c1);
        };
        // B columns this CTA loads: all of the N tile, or its half in a pair
        const int bcols = PAIR ? P.bn / 2 : P.bn, boff = PAIR ? static_cast<int>(rank) * (P.bn / 2) : 0;
        auto advance = [&]() {
            ++filled;
            if (++slot == STAGES) { slot = 0; phase ^= 1u; }
        };
        if (P.bres && t_begin < P.tiles) {
            // every (channel block, tap) B tile once, [cb][tap] order (taps:
            // kernel rows x taps per row -- 3 x 3, or the stem's 4 x 2)
            const int nres = P.ntaps[0] * P.halo_kw;
            mbar_expect_tx(bres_bar, P.bres_bytes);
            for (int cb = 0; cb < P.cblocks; ++cb)
                for (int j = 0; j < nres; ++j) {
                    uint8_t* sb = bres_base + (cb * nres + j) * bt_bytes;
                    const int br = P.brow[j], c0 = cb * BK;
                    if (P.b_mn) {
                        for (int q = 0; q < bcols / 32; ++q) tma_load_2d(sb + q * 4096, &map_b, bres_bar, 32 * q, br + c0);
                    } else if (P.bt) {
                        tma_load_2d(sb, &map_b, bres_bar, br + c0, 0);
                    } else {
                        tma_load_2d(sb, &map_b, bres_bar, c0, br);
                    }
                }
        }
        uint32_t plocal = 0;
        for (int64_t t = t_begin; t < P.tiles; t += t_step, ++plocal) {
            const Tile T = decode(t);
            TC_TRACE(plocal, 6);
            if (P.mode == MODE_CONV && P.halo) {
                // k-step (kernel row dh, channel block cb): the (TW+2) x TH patch at
                // (tw0 - 1, th0 - 1 + dh) and the row's three taps' weights
                // (halo 2: the full (TW+2) x (TH+2) patch and all nine taps per channel block)
                const int aw = T.tw0 + P.off_w[0], ah = T.th0 + P.off_h[0], n0 = static_cast<int>(T.n0) + boff;
                const int ntap = P.halo == 2 ? 9 : P.halo_kw;
                int cb = 0, dh = 0;
                for (int i = 0; i < T.nk; ++i) {
                    uint8_t* sa; uint64_t* bar;
                    acquire(sa, bar);
                    const int c0 = cb * BK;
                    ld4(sa, &map_a, bar, c0, aw, ah + dh, T.tn0);
                    for (int dw = 0; dw < (P.bres ? 0 : ntap); ++dw) {
                        uint8_t* sb = sa + a_bytes + dw * bt_bytes;
                        const int br = P.brow[P.halo == 2 ? dw : dh * P.halo_kw + dw];
                        if (P.b_mn) {
                            for (int q = 0; q < bcols / 32; ++q) ld2(sb + q * 4096, &map_b, bar, n0 + 32 * q, br + c0);
                        } else if (P.bt) {
                            ld2(sb, &map_b, bar, br + c0, n0);   // K-major forward weights [co][kh*kw*ci]
                        } else {
                            ld2(sb, &map_b, bar, c0, br + n0);   // dgrad: weights [tap][ci][co], K = co
                        }
                    }
                    advance();
                    if (++cb == P.cblocks) { cb = 0; ++dh; }
                }
            } else if (P.mode == MODE_CONV) {
                int tap = P.tap0[T.phase], cb = 0;
                const int aw = T.tw0 * P.mw, ah = T.th0 * P.mh, n0 = static_cast<int>(T.n0) + boff;
                int xw = aw + P.off_w[tap], yh = ah + P.off_h[tap], br = P.brow[tap];
                for (int i = 0; i < T.nk; ++i) {
                    uint8_t* sa; uint64_t* bar;
                    acquire(sa, bar);
                    uint8_t* sb = sa + a_bytes;
                    const int c0 = cb * P.kel;
                    if (!MA) ld4(sa, &map_a, bar, c0, xw, yh, T.tn0);
                    if (P.b_mn) {
                        for (int q = 0; q < bcols / 32; ++q) ld2(sb + q * 4096, &map_b, bar, n0 + 32 * q, br + c0);
                    } else if (P.bt) {
                        ld2(sb, &map_b, bar, br + c0, n0);   // transposed forward weights [co][kh*kw*ci]
                    } else {
                        ld2(sb, &map_b, bar, c0, br + n0);   // box rows = bcols (encoded on the host)
                    }
                    advance();
                    if (++cb == P.cblocks && i + 1 < T.nk) {
                        cb = 0;
                        ++tap;
                        xw = aw + P.off_w[tap]; yh = ah + P.off_h[tap]; br = P.brow[tap];
                    }
                }
            } else {
                int ac[4], ax[4], ay[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    int64_t m = T.m0 + 32 * q;
                    if (m >= P.M) m = T.m0;
                    const int tap = static_cast<int>(m / P.ci);
                    ac[q] = static_cast<int>(m % P.ci);
                    ax[q] = (tap % P.kw_) * P.dil_w - P.pl;
                    ay[q] = tap / P.kw_ - P.pt;
                }
                int r = T.kb_begin;
                const int bw = r % P.tiles_w;
                r /= P.tiles_w;
                int x0 = bw * P.TW, y0 = (r % P.tiles_h) * P.TH, n0 = (r / P.tiles_h) * P.TN;
                const int xend = P.tiles_w * P.TW, yend = P.tiles_h * P.TH;
                const int nb = bcols / 32, cn0 = static_cast<int>(T.n0) + boff;
                for (int i = 0; i < T.nk; ++i) {
                    uint8_t* sa; uint64_t* bar;
                    acquire(sa, bar);
                    uint8_t* sb = sa + a_bytes;
                    const int xs = x0 * P.sw, ys = y0 * P.sh;
                    if (!MA) {
#pragma unroll
                        for (int q = 0; q < 4; ++q) ld4(sa + q * 4096, &map_a, bar, ac[q], xs + ax[q], ys + ay[q], n0);
                    }
                    for (int q = 0; q < nb; ++q) ld4(sb + q * 4096, &map_b, bar, cn0 + 32 * q, x0, y0, n0);
                    advance();
                    x0 += P.TW;
                    if (x0 >= xend) {
                        x0 = 0;
                        y0 += P.TH;
                        if (y0 >= yend) { y0 = 0; n0 += P.TN; }
                    }
                }
            }
        }
    } else if (warp == 1 && (!PAIR || rank == 0)) {
        // ================= MMA issuer (PAIR: the leader CTA only) =================
        // The whole warp walks the loop, so every value is provably warp-uniform
        // (uniform registers, no per-MMA waterfall loop), and one elected lane
        // issues. Descriptors are a hoisted base plus additive stage / k offsets
        // (the 14-bit start-address field, in 16-byte units, cannot carry: smem
        // offsets stay below 256 KB).
        const uint32_t a_mn = (P.mode == MODE_WGRAD && !MA) ? 1u : 0u;
        const uint32_t fmt = P.bf16 ? 1u : 2u;   // A/B format: kind::f16 BF16 = 1, kind::tf32 TF32 = 2
        const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | (a_mn << 15) |
                               (static_cast<uint32_t>(P.b_mn) << 16) | ((static_cast<uint32_t>(P.bn) >> 3) << 17) |
                               ((static_cast<uint32_t>(PAIR ? 2 * BM : BM) >> 4) << 24);
        const uint32_t s0 = smem_u32(smem);
        // halo: the A window of tap dw starts dw rows into the patch; 8-row groups
        // are image rows, (TW + 2) rows apart (measured: tools/mma_probe/halo_probe.cu)
        const uint64_t adesc0 = a_mn ? sdesc(s0, 4096, 512, 1) : sdesc(s0, 16, P.halo ? (HALO_TW + 2) * 128 : 1024, 2);
        const uint64_t bdesc0 = P.b_mn ? sdesc(s0 + a_bytes, 4096, 512, 1) : sdesc(s0 + a_bytes, 16, 1024, 2);
        const uint64_t a_kstep = a_mn ? (1024 >> 4) : (32 >> 4), b_kstep = P.b_mn ? (1024 >> 4) : (32 >> 4);
        const uint32_t sres = smem_u32(bres_base);
        const uint64_t bresdesc0 = P.b_mn ? sdesc(sres, 4096, 512, 1) : sdesc(sres, 16, 1024, 2);
        if (P.bres && t_begin < P.tiles) mbar_wait(bres_bar, 0);   // resident B in place (once per CTA)
        const uint64_t stage16 = stage_bytes >> 4;
        const bool leader = elect_one();
        int slot = 0;
        uint32_t phase = 0, local = 0;
        for (int64_t t = t_begin; t < P.tiles; t += t_step, ++local) {
            const Tile T = decode(t);
            const uint32_t acc = local & 1;
            // every tile takes an accumulator turn (tiles without K steps commit
            // immediately and the epilogue writes zeros), so phases stay in step
            if (local >= 2) mbar_wait(&tmem_empty[acc], ((local / 2) - 1) & 1);
            if (lane == 0) TC_TRACE(local, 0);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t d = tmem_base + acc * static_cast<uint32_t>(P.bn);
            for (int i = 0; i < T.nk; ++i) {
                const int s = slot;
                mbar_wait(&full[s], phase);
                if (MA) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // cp.async data -> async proxy
                if (++slot == STAGES) { slot = 0; phase ^= 1u; }
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                if (leader && P.bres) {
                    // B from the resident copy: tile (cb, dh * halo_kw + dw)
                    const uint64_t so = static_cast<uint64_t>(s) * stage16;
                    const int cb = i % P.cblocks, dh = i / P.cblocks, nres = P.ntaps[0] * P.halo_kw;
#pragma unroll
                    for (int dw = 0; dw < 3; ++dw) {
                        if (dw >= P.halo_kw) break;
#pragma unroll
                        for (int kk = 0; kk < BK / 8; ++kk) {
                            const uint64_t ad = adesc0 + so + dw * P.dil_w * (128 >> 4) + kk * a_kstep;
                            const uint64_t bd = bresdesc0 +
                                                static_cast<uint64_t>((cb * nres + dh * P.halo_kw + dw) * bt_bytes >> 4) +
                                                kk * b_kstep;
                            mma_tf32(d, ad, bd, idesc, (i > 0 || dw > 0 || kk > 0) ? 1u : 0u);
                        }
                    }
                    mma_commit(&empty[s]);
                } else if (leader && P.halo == 2) {
                    const uint64_t so = static_cast<uint64_t>(s) * stage16;
                    for (int j = 0; j < 9; ++j) {
                        const uint64_t a_off = static_cast<uint64_t>((j / 3) * (HALO_TW + 2) + j % 3) * (128 >> 4);
#pragma unroll
                        for (int kk = 0; kk < BK / 8; ++kk) {
                            const uint64_t ad = adesc0 + so + a_off + kk * a_kstep;
                            const uint64_t bd = bdesc0 + so + j * (bt_bytes >> 4) + kk * b_kstep;
                            mma_tf32(d, ad, bd, idesc, (i > 0 || j > 0 || kk > 0) ? 1u : 0u);
                        }
                    }
                    mma_commit(&empty[s]);
                } else if (leader && P.halo) {
                    const uint64_t so = static_cast<uint64_t>(s) * stage16;
#pragma unroll
                    for (int dw = 0; dw < 3; ++dw) {
                        if (dw >= P.halo_kw) break;
#pragma unroll
                        for (int kk = 0; kk < BK / 8; ++kk) {
                            const uint64_t ad = adesc0 + so + dw * P.dil_w * (128 >> 4) + kk * a_kstep;
                            const uint64_t bd = bdesc0 + so + dw * (bt_bytes >> 4) + kk * b_kstep;
                            mma_tf32(d, ad, bd, idesc, (i > 0 || dw > 0 || kk > 0) ? 1u : 0u);
                        }
                    }
                    mma_commit(&empty[s]);
                } else if (leader) {
                    const uint64_t so = static_cast<uint64_t>(s) * stage16;
#pragma unroll
                    for (int kk = 0; kk < BK / 8; ++kk) {
                        const uint64_t ad = adesc0 + so + kk * a_kstep, bd = bdesc0 + so + kk * b_kstep;
                        const uint32_t accum = (i > 0 || kk > 0) ? 1u : 0u;
                        if (P.bf16) {
                            if (PAIR)
                                mma_f16_pair(d, ad, bd, idesc, accum);
                            else
                                mma_f16(d, ad, bd, idesc, accum);
                        } else if (PAIR) {
                            mma_tf32_pair(d, ad, bd, idesc, accum);
                        } else {
                            mma_tf32(d, ad, bd, idesc, accum);
                        }
                    }
                    if (PAIR)
                        mma_commit_pair(&empty[s]);   // frees the stage in both CTAs
                    else
                        mma_commit(&empty[s]);
                }
                __syncwarp();
            }
            if (leader) {
                if (PAIR)
                    mma_commit_pair(&tmem_full[acc]);
                else
                    mma_commit(&tmem_full[acc]);
            }
            if (lane == 0) TC_TRACE(local, 1);
            __syncwarp();
        }
    } else if (MA && warp >= 10) {
        // ================= A builders (warps 10..13, MA only) =================
        // Thread t owns row t of the 128 x 32 A tile: it gathers 32 values,
        // writes them as eight 16-byte chunks at the 128B-swizzled positions
        // (chunk j of row t lands at j ^ (t % 8), as TMA would place them),
        // makes the writes visible to the tensor core's async proxy, and
        // arrives on the stage's full barrier.
        const int t = threadIdx.x - THREADS;
        int slot = 0;
        uint32_t phase = 0, filled = 0;
        const int kpad = P.cblocks * BK;
        for (int64_t tt = t_begin; tt < P.tiles; tt += t_step) {
            const Tile T = decode(tt);
            if (P.mode == MODE_CONV) {
                const int pw = T.tw0 + t % P.TW, ph = T.th0 + (t / P.TW) % P.TH, pn = T.tn0 + t / (P.TW * P.TH);
                const bool pv = pw < P.gw && ph < P.gh && pn < P.gn;
                const int iy0 = ph * P.sh - P.pt, ix0 = pw * P.sw - P.pl;
                const float* xb = P.xa + ((static_cast<int64_t>(pv ? pn : 0) * P.ih_ + iy0) * P.iw_ + ix0) * P.ci;
                for (int i = 0; i < T.nk; ++i) {
                    if (filled >= static_cast<uint32_t>(STAGES)) mbar_wait(&empty[slot], phase ^ 1u);
                    uint8_t* row = smem + slot * stage_bytes + t * 128;
                    // asynchronous gathers (masked elements zero-fill), so the
                    // builders run up to STAGES k-steps ahead of the MMA
#pragma unroll
                    for (int k = 0; k < BK; ++k) {
                        const int kk = i * BK + k;
                        const int iy = iy0 + ma_tab[kpad + kk], ix = ix0 + ma_tab[2 * kpad + kk];
                        const bool ok = pv && iy >= 0 && iy < P.ih_ && ix >= 0 && ix < P.iw_;
                        cp_async4(row + (((k >> 2) ^ (t & 7)) << 4) + (k & 3) * 4, ok ? xb + ma_tab[kk] : P.xa, ok ? 4 : 0);
                    }
                    cp_async_arrive(&full[slot]);
                    ++filled;
                    if (++slot == STAGES) { slot = 0; phase ^= 1u; }
                }
            } else {
                const int64_t m = T.m0 + t;
                const bool mv = m < P.M;
                const int tap = mv ? static_cast<int>(m / P.ci) : 0, c = mv ? static_cast<int>(m % P.ci) : 0;
                const int dy = tap / P.kw_ - P.pt, dx = tap % P.kw_ - P.pl;
                int r = T.kb_begin;
                const int bw = r % P.tiles_w;
                r /= P.tiles_w;
                int x0 = bw * P.TW, y0 = (r % P.tiles_h) * P.TH, n0 = (r / P.tiles_h) * P.TN;
                const int xend = P.tiles_w * P.TW, yend = P.tiles_h * P.TH;
                for (int i = 0; i < T.nk; ++i) {
                    if (filled >= static_cast<uint32_t>(STAGES)) mbar_wait(&empty[slot], phase ^ 1u);
                    uint8_t* row = smem + slot * stage_bytes + t * 128;
#pragma unroll
                    for (int k = 0; k < BK; ++k) {
                        const int on = n0 + ma_tab[k], oy = y0 + ma_tab[BK + k], ox = x0 + ma_tab[2 * BK + k];
                        const int iy = oy * P.sh + dy, ix = ox * P.sw + dx;
                        const bool ok = mv && on < P.gn && oy < P.gh && ox < P.gw && iy >= 0 && iy < P.ih_ &&
                                        ix >= 0 && ix < P.iw_;
                        const int64_t off = ((static_cast<int64_t>(on) * P.ih_ + iy) * P.iw_ + ix) * P.ci + c;
                        cp_async4(row + (((k >> 2) ^ (t & 7)) << 4) + (k & 3) * 4, P.xa + (ok ? off : 0), ok ? 4 : 0);
                    }
                    cp_async_arrive(&full[slot]);
                    ++filled;
                    if (++slot == STAGES) { slot = 0; phase ^= 1u; }
                    x0 += P.TW;
                    if (x0 >= xend) {
                        x0 = 0;
                        y0 += P.TH;
                        if (y0 >= yend) { y0 = 0; n0 += P.TN; }
                    }
                }
            }
        }
    } else if (warp >= 2) {
        // ================= epilogue (warps 2..9) =================
        // Warp w may only touch TMEM lanes 32*(w%4)..+31; two warps share each
        // lane quarter and split the 32-column chunks between them.
        const int quarter = warp % 4;
        const int half = (warp - 2) / 4;
        const int row = quarter * 32 + lane;
        double cs_sum[4] = {0, 0, 0, 0}, cs_sq[4] = {0, 0, 0, 0};   // CS: per-lane column accumulators
        const int nchunks = P.bn / 32;
        auto out_box = [&](const Tile& T) {
            TmaOut to{&map_c, P.tma_out, 0, 0, 0};
            if (P.tma_out == 1) {   // the warp's quarter of the pixel tile as a sub-box origin
                const int q0 = quarter * 32;
                to.c1 = T.tw0 + q0 % P.TW;
                to.c2 = T.th0 + (q0 / P.TW) % P.TH;
                to.c3 = T.tn0 + q0 / (P.TW * P.TH);
            } else if (P.tma_out == 2) {
                to.c1 = static_cast<int>(T.m0) + quarter * 32;
                to.c2 = P.splits > 1 ? T.split : 0;
            }
            return to;
        };
        // EG side tiles: this warp's chunks are c = half, half + 2, ... with col0 < N
        auto chunk_col = [&](const Tile& T, int c) -> int {
            return (c < nchunks && T.n0 + c * 32 < P.N) ? static_cast<int>(T.n0 + c * 32) : -1;
        };
        EgSide es{&eg_maps, side + (warp - 2) * 2 * P.eg_side * P.stg_cols * 128, &side_bar[2 * (warp - 2)], 0u, 0u,
                  TmaOut{&map_c, 0, 0, 0, 0}, -1};
        auto side_issue = [&](const TmaOut& to, int col) {
            if (P.stg_cols == 32)
                eg_side_load<32>(es, P.eg_side, to, col);
            else if (P.stg_cols == 16)
                eg_side_load<16>(es, P.eg_side, to, col);
            else
                eg_side_load<8>(es, P.eg_side, to, col);
        };
        const bool side_on = EG && P.eg_side > 0;
        // this lane's row within a pixel tile (tile-independent)
        const int r_ww = row % P.TW, r_hh = (row / P.TW) % P.TH, r_nn = row / (P.TW * P.TH);
        uint32_t local = 0, stg_seq = 0;
        Tile Tnext = t_begin < P.tiles ? decode(t_begin) : Tile{};   // each tile decoded once
        for (int64_t t = t_begin; t < P.tiles; t += t_step, ++local) {
            const Tile T = Tnext;
            const bool has_next = t + t_step < P.tiles;
            if (has_next) Tnext = decode(t + t_step);
            const uint32_t acc = local & 1;
            if (side_on && es.issued == es.consumed) {   // nothing in flight: this tile's first side tiles
                const int c0 = chunk_col(T, half);
                if (c0 >= 0) {
                    if (lane == 0) side_issue(out_box(T), c0);
                    ++es.issued;
                }
            }
            mbar_wait(&tmem_full[acc], (local / 2) & 1);
            if (warp == 2 && lane == 0) TC_TRACE(local, 2);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            float* dst = nullptr;
            bool valid = false;
            if (P.mode == MODE_CONV) {
                const int n = T.tn0 + r_nn, y = T.th0 + r_hh, x = T.tw0 + r_ww;
                valid = n < P.gn && y < P.gh && x < P.gw;
                const int64_t oy = static_cast<int64_t>(y) * P.out_s + P.py[T.phase];
                const int64_t ox = static_cast<int64_t>(x) * P.out_s + P.px[T.phase];
                valid = valid && oy < P.out_h && ox < P.out_w;
                dst = P.out + ((static_cast<int64_t>(n) * P.out_h + oy) * P.out_w + ox) * P.ldc;
            } else {
                const int64_t m = T.m0 + row;
                valid = m < P.M;
                float* base = P.splits > 1 ? P.partial + static_cast<int64_t>(T.split) * P.M * P.N : P.out;
                dst = base + m * P.ldc;
            }
            const TmaOut to = out_box(T);
            const uint32_t tbase =
                tmem_base + acc * static_cast<uint32_t>(P.bn) + (static_cast<uint32_t>(quarter * 32) << 16);
            uint32_t r[32];
            bool arrived = false;
#pragma unroll
            for (int k = 0; k < 4; ++k) {   // this warp's chunks: c = half, half + 2, ... (<= 8 chunks)
                const int c = half + 2 * k;
                if (c >= nchunks) break;
                tmem_ld32(tbase + static_cast<uint32_t>(c * 32), r);
                if (c + 2 >= nchunks) {
                    // this warp's last chunk of the tile is in registers: release its share
                    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                    if (lane == 0) {
                        if (PAIR)   // the leader's MMA waits for both CTAs' epilogues
                            mbar_arrive_cluster(mapa_u32(&tmem_empty[acc], 0));
                        else
                            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tmem_empty[acc]))
                                         : "memory");
                    }
                    arrived = true;
                    if (warp == 2 && lane == 0) TC_TRACE(local, 3);
                }
                const int64_t col0 = T.n0 + c * 32;
                if (T.nk == 0) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) r[j] = 0u;
                }
                if (P.bias && col0 < P.N) {
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if (col0 + j < P.N)
                            r[j] = __float_as_uint(__fadd_rn(__uint_as_float(r[j]), __ldg(P.bias + col0 + j)));
                }
                if (P.bn_inv && col0 < P.N) {   // inference BatchNorm (+ residual) (+ ReLU): the EW sequence
                    // Four columns at a time: their parameters and the row's
                    // residual as 16-byte loads, consumed at once, so no 32-wide
                    // residual array is live (the 96-register 2-CTA builds
                    // spilled it: BN_AFFINE convs ran up to 2.3x slower).
                    const float* rrow = (P.res && valid) ? P.res + (dst - P.out) + col0 : nullptr;
                    if (col0 + 32 <= P.N) {   // per-column parameters as 16-byte loads (L1 broadcast)
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            const int cc = static_cast<int>(col0) + 4 * q;
                            const float4 m4 = __ldg(reinterpret_cast<const float4*>(P.bn_mean + cc));
                            const float4 i4 = __ldg(reinterpret_cast<const float4*>(P.bn_inv + cc));
                            const float4 g4 = __ldg(reinterpret_cast<const float4*>(P.bn_gamma + cc));
                            const float4 b4 = __ldg(reinterpret_cast<const float4*>(P.bn_beta + cc));
                            const float4 r4 = rrow ? __ldg(reinterpret_cast<const float4*>(rrow) + q)
                                                   : make_float4(0.f, 0.f, 0.f, 0.f);
                            const float mm[4] = {m4.x, m4.y, m4.z, m4.w}, ii[4] = {i4.x, i4.y, i4.z, i4.w};
                            const float gg[4] = {g4.x, g4.y, g4.z, g4.w}, bb[4] = {b4.x, b4.y, b4.z, b4.w};
                            const float rr[4] = {r4.x, r4.y, r4.z, r4.w};
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const int j = 4 * q + u;
                                float v = __fsub_rn(__uint_as_float(r[j]), mm[u]);
                                v = __fadd_rn(__fmul_rn(__fmul_rn(v, ii[u]), gg[u]), bb[u]);
                                if (rrow) v = __fadd_rn(v, rr[u]);
                                if (P.relu) v = v > 0.f ? v : 0.f;
                                r[j] = __float_as_uint(v);
                            }
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (col0 + j < P.N) {
                                const int cc = static_cast<int>(col0) + j;
                                float v = __fsub_rn(__uint_as_float(r[j]), __ldg(P.bn_mean + cc));
                                v = __fmul_rn(__fmul_rn(v, __ldg(P.bn_inv + cc)), __ldg(P.bn_gamma + cc));
                                v = __fadd_rn(v, __ldg(P.bn_beta + cc));
                                if (rrow) v = __fadd_rn(v, __ldg(rrow + j));
                                if (P.relu) v = v > 0.f ? v : 0.f;
                                r[j] = __float_as_uint(v);
                            }
                    }
                }
                if (col0 < P.N && (CS || !P.nostore)) {
                    uint8_t* tile = staging + (warp - 2) * (P.stg_bufs * P.stg_cols * 128);
                    const bool full_cols = col0 + 32 <= P.N && (P.ldc % 4) == 0;
                    const bool st = !P.nostore;
                    float c1 = 0.f, c2 = 0.f;
                    if (side_on) {   // the item after this chunk: the next chunk, else the next tile's first
                        es.next_to = to;
                        es.next_col = chunk_col(T, c + 2);
                        if (es.next_col < 0 && has_next) {
                            es.next_to = out_box(Tnext);
                            es.next_col = chunk_col(Tnext, half);
                        }
                    }
                    if (P.stg_cols == 32)
                        store_chunk_t<8, CS, EG>(r, tile, dst, valid, col0, P.N, full_cols, lane, st, c1, c2, to, P, es, stg_seq);
                    else if (P.stg_cols == 16)
                        store_chunk_t<4, CS, EG>(r, tile, dst, valid, col0, P.N, full_cols, lane, st, c1, c2, to, P, es, stg_seq);
                    else
                        store_chunk_t<2, CS, EG>(r, tile, dst, valid, col0, P.N, full_cols, lane, st, c1, c2, to, P, es, stg_seq);
                    if (CS) {
                        cs_sum[k] += static_cast<double>(c1);
                        cs_sq[k] += static_cast<double>(c2);
                    }
                }
            }
            if (warp == 2 && lane == 0) TC_TRACE(local, 4);
            if (warp == 9 && lane == 0) TC_TRACE(local, 5);
            if (!arrived && lane == 0) {   // a warp without a chunk in this tile still arrives once
                if (PAIR)
                    mbar_arrive_cluster(mapa_u32(&tmem_empty[acc], 0));
                else
                    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tmem_empty[acc])) : "memory");
            }
            if (CS) {
                // flush this warp's column accumulators when the CTA's next tile
                // covers other columns (normally once, after the last tile)
                const bool flush = !has_next || Tnext.n0 != T.n0;
                if (flush) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int64_t col = T.n0 + (half + 2 * k) * 32 + lane;
                        if (half + 2 * k < nchunks && col < P.N && cs_sum[k] != 0.0) {
                            // integer limbs: the sum is the same in any order (deterministic)
                            unsigned long long* f = P.cs_fixed;
                            const int64_t N = P.N;
                            fixed_add(f + col, f + N + col, cs_sum[k]);
                            fixed_add(f + 2 * N + col, f + 3 * N + col, cs_sq[k]);
                        }
                        cs_sum[k] = 0.0;
                        cs_sq[k] = 0.0;
                    }
                }
            }
        }
        if (P.tma_out && lane == 0)   // every TMA store issued by this warp has completed
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        if (CS) {
            // the last CTA to finish converts the fixed-point column sums
            volatile uint32_t* cs_last = tmem_slot + 1;   // a free word beside the TMEM address slot
            asm volatile("bar.sync 1, 256;" ::: "memory");   // the 8 epilogue warps' flushes are issued
            if (warp == 2 && lane == 0) {
                __threadfence();
                const unsigned long long ticket = atomicAdd(P.cs_fixed + 4 * P.N, 1ull);
                *cs_last = ticket == gridDim.x - 1 ? 1u : 0u;
            }
            asm volatile("bar.sync 1, 256;" ::: "memory");
            if (*cs_last) {
                __threadfence();
                const int64_t N = P.N;
                for (int64_t c = threadIdx.x - 64; c < N; c += 256) {
                    const unsigned long long* f = P.cs_fixed;
                    const double s0 = fixed_value(__ldcg(f + c), __ldcg(f + N + c));
                    const double s1 = fixed_value(__ldcg(f + 2 * N + c), __ldcg(f + 3 * N + c));
                    P.colstats[c] = s0;
                    P.colstats[N + c] = s1;
                    if (P.cs_stats) {   // the BatchNorm finalize, as fused_ops.cu bn_finalize_k
                        const double mean = __ddiv_rn(s0, (double)P.cs_rows);
                        double var = __dsub_rn(__ddiv_rn(s1, (double)P.cs_rows), __dmul_rn(mean, mean));
                        if (var < 0) var = 0;
                        P.cs_stats[c] = (float)mean;
                        P.cs_stats[N + c] = (float)__ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(var, P.cs_eps)));
                    }
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    if (PAIR)
        cluster_sync_all();   // no remote arrive or MMA into this CTA remains outstanding
    else
        __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (PAIR)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(tmem_cols));
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(tmem_cols));
    }
}

__global__ void splitk_reduce_kernel(const float* __restrict__ partial, float* __restrict__ out, int64_t count,
                                     int splits) {
    nncb::pdl_wait();   // programmatic dependent of the split-K GEMM
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        float s = partial[i];
        for (int k = 1; k < splits; ++k) s = __fadd_rn(s, partial[k * count + i]);
        out[i] = s;
    }
}

// Split-K fold, 4 outputs per thread (float4) and four independent chains
// over the splits (k mod 4), combined as (c0 + c1) + (c2 + c3): a fixed,
// deterministic order with a quarter of the dependent-add latency.
__device__ __forceinline__ float sgd_update(float w, float g, double lr, double scale) {
    // the expression of fused_ops.cu sgd1, no contraction: (double)w - lr * ((double)g * scale)
    return (float)__dsub_rn((double)w, __dmul_rn(lr, __dmul_rn((double)g, scale)));
}

// The split-K fold of a weight gradient with the SGD update of those weights
// fused in: out = dW (same fixed order as splitk_reduce4_kernel), and
// w = sgd_update(w, dW) -- the expression of sgd_dev_k, so the weights are
// bitwise those of the separate update.
__global__ void splitk_reduce4_sgd_kernel(const float4* __restrict__ partial, float4* __restrict__ out, int64_t count4,
                                          int splits, float4* __restrict__ w, const double* __restrict__ lr_dev,
                                          double scale) {
    nncb::pdl_wait();
    const double lr = *lr_dev;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count4; i += (int64_t)gridDim.x * blockDim.x) {
        float4 c[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) c[j] = j < splits ? __ldg(partial + j * count4 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
        for (int k = 4; k < splits; k += 4) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (k + j < splits) {
                    const float4 v = __ldg(partial + (k + j) * count4 + i);
                    c[j].x = __fadd_rn(c[j].x, v.x);
                    c[j].y = __fadd_rn(c[j].y, v.y);
                    c[j].z = __fadd_rn(c[j].z, v.z);
                    c[j].w = __fadd_rn(c[j].w, v.w);
                }
        }
        float4 r;
        r.x = __fadd_rn(__fadd_rn(c[0].x, c[1].x), __fadd_rn(c[2].x, c[3].x));
        r.y = __fadd_rn(__fadd_rn(c[0].y, c[1].y), __fadd_rn(c[2].y, c[3].y));
        r.z = __fadd_rn(__fadd_rn(c[0].z, c[1].z), __fadd_rn(c[2].z, c[3].z));
        r.w = __fadd_rn(__fadd_rn(c[0].w, c[1].w), __fadd_rn(c[2].w, c[3].w));
        out[i] = r;
        float4 wv = w[i];
        wv.x = sgd_update(wv.x, r.x, lr, scale);
        wv.y = sgd_update(wv.y, r.y, lr, scale);
        wv.z = sgd_update(wv.z, r.z, lr, scale);
        wv.w = sgd_update(wv.w, r.w, lr, scale);
        w[i] = wv;
    }
}

__global__ void splitk_reduce4_kernel(const float4* __restrict__ partial, float4* __restrict__ out, int64_t count4,
                                      int splits) {
    nncb::pdl_wait();   // programmatic dependent of the split-K GEMM
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count4; i += (int64_t)gridDim.x * blockDim.x) {
        float4 c[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) c[j] = j < splits ? __ldg(partial + j * count4 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
        for (int k = 4; k < splits; k += 4) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (k + j < splits) {
                    const float4 v = __ldg(partial + (k + j) * count4 + i);
                    c[j].x = __fadd_rn(c[j].x, v.x);
                    c[j].y = __fadd_rn(c[j].y, v.y);
                    c[j].z = __fadd_rn(c[j].z, v.z);
                    c[j].w = __fadd_rn(c[j].w, v.w);
                }
        }
        float4 r;
        r.x = __fadd_rn(__fadd_rn(c[0].x, c[1].x), __fadd_rn(c[2].x, c[3].x));
        r.y = __fadd_rn(__fadd_rn(c[0].y, c[1].y), __fadd_rn(c[2].y, c[3].y));
        r.z = __fadd_rn(__fadd_rn(c[0].z, c[1].z), __fadd_rn(c[2].z, c[3].z));
        r.w = __fadd_rn(__fadd_rn(c[0].w, c[1].w), __fadd_rn(c[2].w, c[3].w));
        out[i] = r;
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

bool encode_4d(CUtensorMap* map, const float* base, int64_t c, int64_t w, int64_t h, int64_t n, int bc, int bw,
               int bh, int bnn, int ew, int eh, bool mn_major, int64_t pitch = 0, int esize = 4) {
    if (pitch == 0) pitch = c;   // elements between consecutive pixels
    cuuint64_t dims[4] = {(cuuint64_t)c, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)n};
    cuuint64_t strides[3] = {(cuuint64_t)(pitch * esize), (cuuint64_t)(pitch * w * esize),
                             (cuuint64_t)(pitch * w * h * esize)};
    cuuint32_t box[4] = {(cuuint32_t)bc, (cuuint32_t)bw, (cuuint32_t)bh, (cuuint32_t)bnn};
    cuuint32_t es[4] = {1, (cuuint32_t)ew, (cuuint32_t)eh, 1};
    CUresult r = nncb::drv::table().tensorMapEncodeTiled(
        map, esize == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
        const_cast<float*>(base), dims, strides, box, es,
        CU_TENSOR_MAP_INTERLEAVE_NONE, mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
        CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) nncb::set_error(std::string("cuTensorMapEncodeTiled(4d): ") + nncb::drv::error_string(r));
    return r == CUDA_SUCCESS;
}

bool encode_2d(CUtensorMap* map, const float* base, int64_t inner, int64_t rows, int box_inner, int box_rows,
               bool mn_major, int esize = 4) {
    cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)(inner * esize)};
    cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = nncb::drv::table().tensorMapEncodeTiled(
        map, esize == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
        const_cast<float*>(base), dims, strides, box, es,
        CU_TENSOR_MAP_INTERLEAVE_NONE, mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
        CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) nncb::set_error(std::string("cuTensorMapEncodeTiled(2d): ") + nncb::drv::error_string(r));
    return r == CUDA_SUCCESS;
}

thread_local int g_force_bn = 0;     // set by the autotuner (gemm_tc) for one call
thread_local int g_force_pair = 0;   // 1: run the call as CTA pairs (cta_group::2)
thread_local int g_force_wide = 0;   // 1: full-width (32-column) epilogue staging even at 2 CTAs/SM
thread_local int g_dil_w = 1;        // horizontal tap dilation for the next implicit GEMM (internal)
thread_local int g_force_tb = 0;     // 1: forward convolution with transposed (K-major) weights
thread_local int g_force_bres = 0;   // 1: halo tiles with resident B (single N tile)
thread_local int g_force_halo = 0;   // 1: 3x3 stride-1 conv through kernel-row halo patches; 2: full 3x3 patches
thread_local bool g_sgd_applied = false;   // the last weight-gradient call applied its SGD update (fused fold)
thread_local int g_bf16 = 0;         // the next implicit GEMM's A and B are bf16 copies (NNCB_PREC_BF16 route)
thread_local const float* g_bn_inv = nullptr;   // BN_AFFINE: this call's per-column invstd (device)

int pick_bn(int64_t n) {
    static const int env_bn = getenv("NNCB_TC_BN") ? atoi(getenv("NNCB_TC_BN")) : 0;   // tuning knob
    const int force = g_force_bn ? g_force_bn : env_bn;
    if (force == 64 || force == 128 || force == 256) {   // widths stay in {64, 128, 256} (TMEM: power-of-two columns)
        int w = force;
        while (w > 64 && w / 2 >= n) w /= 2;
        return w;
    }
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

size_t stage_bytes_for(int bn) { return BM * BK * 4 + static_cast<size_t>(bn) * BK * 4; }

// Ring depth: 2 CTAs per SM when two accumulator pairs fit TMEM (bn <= 128) and
// the ring fits half the shared memory, else one CTA with a deeper ring.
size_t smem_for(int bn, int stages, int stg_cols, int ma_tab_ints = 0, int stg_bufs = 1) {
    return stages * stage_bytes_for(bn) + 8 * static_cast<size_t>(stg_cols) * 128 * stg_bufs + 1024 + 512 + 16 * bn +
           4 * static_cast<size_t>(ma_tab_ints);
}

// Pipeline depth, epilogue staging width and CTAs per SM for an N-tile width.
// bn <= 128 keeps two CTAs per SM (113 KB each) with >= 3 stages, taking the
// widest epilogue transpose that still fits; wider tiles run one CTA per SM
// and take the widest transpose that still leaves a 3-deep ring.
struct TcShape { int stages, stg_cols, per_sm; };
TcShape pick_shape(int bn) {
    const size_t sb = stage_bytes_for(bn), per_cta_two = 113 * 1024, per_cta_one = 227 * 1024;
    if (bn <= 128)
        for (int stg : {32, 16, 8}) {
            const size_t fixed = smem_for(bn, 0, stg);
            if (fixed + 3 * sb <= per_cta_two)
                return {static_cast<int>(std::min<size_t>(MAX_STAGES, (per_cta_two - fixed) / sb)), stg, 2};
        }
    TcShape best{0, 32, 1};
    for (int stg : {32, 16, 8}) {
        const int st = static_cast<int>(std::min<size_t>(MAX_STAGES, (per_cta_one - smem_for(bn, 0, stg)) / sb));
        if (st >= 3) return {st, stg, 1};   // the wide transpose is worth more than a 4th stage
        if (st > best.stages) best = {st, stg, 1};
    }
    return best;
}

// Tensor map with the TMA epilogue's output geometry (P.tma_out 1: 4-D pixel
// grid, 2: 3-D [split][row][col]) over `base`: the output itself, or a side
// input of the gradient epilogue laid out like it.
bool encode_out_like(CUtensorMap* m, const TcParams& P, const void* base) {
    const int cols = P.stg_cols;
    const CUtensorMapSwizzle sw = cols == 32 ? CU_TENSOR_MAP_SWIZZLE_128B
                                  : cols == 16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B;
    CUresult r;
    if (P.tma_out == 1) {
        cuuint64_t dims[4] = {(cuuint64_t)P.N, (cuuint64_t)P.out_w, (cuuint64_t)P.out_h, (cuuint64_t)P.gn};
        cuuint64_t strides[3] = {(cuuint64_t)(P.N * 4), (cuuint64_t)(P.N * P.out_w * 4),
                                 (cuuint64_t)(P.N * P.out_w * P.out_h * 4)};
        cuuint32_t box[4] = {(cuuint32_t)cols, (cuuint32_t)P.ob_w, (cuuint32_t)P.ob_h, (cuuint32_t)P.ob_n};
        cuuint32_t es[4] = {1, 1, 1, 1};
        r = nncb::drv::table().tensorMapEncodeTiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void*>(base), dims,
                                                    strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                                                    CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
        cuuint64_t dims[3] = {(cuuint64_t)P.N, (cuuint64_t)P.M, (cuuint64_t)std::max(P.splits, 1)};
        cuuint64_t strides[2] = {(cuuint64_t)(P.N * 4), (cuuint64_t)(P.N * P.M * 4)};
        cuuint32_t box[3] = {(cuuint32_t)cols, 32, 1};
        cuuint32_t es[3] = {1, 1, 1};
        r = nncb::drv::table().tensorMapEncodeTiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims,
                                                    strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                                                    CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    return r == CUDA_SUCCESS;
}

// Output tensor map for the TMA epilogue, encoded once the staging width
// (COLS = stg_cols) is known. Returns false (direct stores) when not applicable.
bool encode_tma_out(CUtensorMap* mc, TcParams& P) {
    static const bool enabled = !(getenv("NNCB_TC_TMA_OUT") && atoi(getenv("NNCB_TC_TMA_OUT")) == 0);
    P.tma_out = 0;
    if (!enabled || P.N % 4 != 0 || P.ldc != P.N) return false;
    if (P.mode == MODE_CONV) {
        if (P.out_s != 1) return false;   // strided-dgrad phases interleave pixels: direct stores
        P.ob_w = P.TW >= 32 ? 32 : P.TW;
        P.ob_h = P.TW >= 32 ? 1 : std::min(P.TH, 32 / P.TW);
        P.ob_n = 32 / (P.ob_w * P.ob_h);
        if (P.ob_n > P.TN && P.ob_n > 1) return false;
        P.tma_out = 1;
        if (encode_out_like(mc, P, P.out)) return true;
    } else {
        P.tma_out = 2;
        if (encode_out_like(mc, P, P.splits > 1 ? P.partial : P.out)) return true;
    }
    P.tma_out = 0;
    return false;
}

// Gradient epilogue: side tiles through TMA when the output leaves through
// TMA (same geometry); otherwise the epilogue loads the side inputs per row.
void encode_eg_side(EgMaps* em, TcParams& P) {
    P.eg_side = 0;
    if (!P.eg || !P.tma_out) return;
    const int n = P.eg_res ? 3 : 2;
    const float* src[3] = {P.eg_mask, P.eg_x, P.eg_res};
    for (int a = 0; a < n; ++a)
        if (!encode_out_like(&em->m[a], P, src[a])) return;
    P.eg_side = n;
}

// Shared-memory shape of a gradient-epilogue launch (one CTA per SM): the
// widest staging whose double-buffered side tiles still leave a 2-deep ring
// (the fused dgrads are output-bound: side bandwidth beats ring depth).
void eg_shape(TcParams& P, int bn_smem) {
    const size_t sb = stage_bytes_for(bn_smem);
    const int nside = P.eg_res ? 3 : 2;
    for (int need : {2})
        for (int stg : {32, 16, 8}) {
            const size_t fixed = smem_for(bn_smem, 0, stg) + 16 * static_cast<size_t>(nside) * stg * 128;
            if (fixed >= 227 * 1024) continue;
            const int st = static_cast<int>(std::min<size_t>(MAX_STAGES, (227 * 1024 - fixed) / sb));
            if (st >= need) {
                P.stg_cols = stg;
                P.stages = st;
                return;
            }
        }
}

// NNCB_TC_STGBUF=2: double-buffered epilogue staging when it fits the CTA's
// shared memory, giving up at most one ring stage (and keeping >= 3). Opt-in:
// measured neutral on forward+statistics 1x1 convs and 2-12% slower on
// dgrads that lose a stage (the TMA store's shared-memory read is not what
// bounds these epilogues).
void pick_stg_bufs(TcParams& P, int bn_smem, int tab_ints, size_t limit) {
    static const int env = getenv("NNCB_TC_STGBUF") ? atoi(getenv("NNCB_TC_STGBUF")) : 0;
    P.stg_bufs = 1;
    if (env != 2 || P.eg) return;
    for (int st = P.stages; st >= P.stages - 1 && st >= 3; --st)
        if (smem_for(bn_smem, st, P.stg_cols, tab_ints, 2) <= limit) {
            P.stages = st;
            P.stg_bufs = 2;
            return;
        }
}

size_t eg_side_bytes(const TcParams& P) { return P.eg ? 16 * static_cast<size_t>(P.eg_res ? 3 : 2) * P.stg_cols * 128 : 0; }

int launch(nncb_ctx* ctx, const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc_unused, TcParams& P) {
    CUtensorMap mc;
    memset(&mc, 0, sizeof(mc));
    static bool attr_done = false;
    if (!attr_done) {
        NNCB_CUDA(cudaFuncSetAttribute(tc_gemm_kernel<false, false, 2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        NNCB_CUDA(cudaFuncSetAttribute(tc_gemm_kernel<false, false, 1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        NNCB_CUDA(cudaFuncSetAttribute(tc_gemm_kernel<true, false, 2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        NNCB_CUDA(cudaFuncSetAttribute(tc_gemm_kernel<true, false, 1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        NNCB_CUDA(cudaFuncSetAttribute(tc_gemm_kernel<false, true, 1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        NNCB_CUDA(cudaFuncSetAttribute(tc_gemm_kernel<true, true, 1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        NNCB_CUDA(cudaFuncSetAttribute(tc_gemm_kernel<false, false, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        NNCB_CUDA(cudaFuncSetAttribute(tc_gemm_kernel<true, false, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        NNCB_CUDA(cudaFuncSetAttribute(tc_gemm_kernel<true, false, 1, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        NNCB_CUDA(cudaFuncSetAttribute(tc_gemm_kernel<true, false, 1, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        attr_done = true;
    }
    P.stg_bufs = 1;
    if (P.tiles <= 0) return 0;
    if (P.tiles >= (int64_t(1) << 31)) return nncb::fail("gemm: tile count exceeds the kernel's 32-bit tile index");
    P.tma_store = 0;
    const TcShape shp = pick_shape(P.bn);
    P.stages = shp.stages;
    P.stg_cols = shp.stg_cols;
    static const int env_stages = getenv("NNCB_TC_STAGES") ? atoi(getenv("NNCB_TC_STAGES")) : 0;
    static const int env_persm = getenv("NNCB_TC_PERSM") ? atoi(getenv("NNCB_TC_PERSM")) : 0;
    static const int env_nostore = getenv("NNCB_TC_NOSTORE") ? 1 : 0;
    static const int env_stg = getenv("NNCB_TC_STG") ? atoi(getenv("NNCB_TC_STG")) : 0;
    if (env_stg == 8 || env_stg == 16 || env_stg == 32) P.stg_cols = env_stg;
    if (env_stages > 0) P.stages = std::min(env_stages, MAX_STAGES);
    P.nostore = env_nostore;
    EgMaps em;
    memset(&em, 0, sizeof(em));
    if (P.eg && (P.xa != nullptr || P.nostore)) return nncb::fail("gemm: the gradient epilogue has no manual-A / no-store build");
    if (P.pair) {
        // CTA pair: each CTA stages A (128 rows) and half of B; one CTA per SM
        const int half = P.bn / 2;
        P.stg_cols = 32;
        const size_t fixed = smem_for(half, 0, P.stg_cols);
        P.stages = static_cast<int>(std::min<size_t>(MAX_STAGES, (227 * 1024 - fixed) / stage_bytes_for(half)));
        if (P.eg) eg_shape(P, half);
        pick_stg_bufs(P, half, 0, 227 * 1024);
        const size_t smem = smem_for(half, P.stages, P.stg_cols, 0, P.stg_bufs) + eg_side_bytes(P);
        encode_tma_out(&mc, P);
        encode_eg_side(&em, P);
        const int64_t pairs = std::min<int64_t>(P.tiles, ctx->sm_count / 2);
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(static_cast<unsigned>(2 * pairs));
        cfg.blockDim = dim3(THREADS);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = ctx->stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (P.eg)
            NNCB_CUDA(cudaLaunchKernelEx(&cfg, tc_gemm_kernel<true, false, 1, true, true>, ma, mb, mc, P, em));
        else if (P.colstats)
            NNCB_CUDA(cudaLaunchKernelEx(&cfg, tc_gemm_kernel<true, false, 1, true>, ma, mb, mc, P, em));
        else
            NNCB_CUDA(cudaLaunchKernelEx(&cfg, tc_gemm_kernel<false, false, 1, true>, ma, mb, mc, P, em));
        NNCB_LAUNCHED(ctx);
        return 0;
    }
    const bool manual = P.xa != nullptr;
    const int tab_ints = manual ? 3 * std::max(P.cblocks * BK, BK) : 0;
    if (P.halo) {
        // stage = patch + three taps' B tiles: two CTAs per SM when two stages
        // fit, else one CTA with a deeper ring
        const size_t sbh = P.bres ? HALO_A_BYTES
                           : P.halo == 2 ? HALO9_A_BYTES + 9 * static_cast<size_t>(P.bn) * BK * 4
                                         : HALO_A_BYTES + P.halo_kw * static_cast<size_t>(P.bn) * BK * 4;
        int per = 0;
        if (P.bres)   // one CTA per SM: resident B + the deepest patch ring that fits
            for (int stg : {16, 8}) {
                const size_t fixed = smem_for(P.bn, 0, stg) + P.bres_bytes;
                if (fixed + 2 * sbh <= 227 * 1024) {
                    P.stg_cols = stg;
                    P.stages = static_cast<int>(std::min<size_t>(MAX_STAGES, (227 * 1024 - fixed) / sbh));
                    per = 1;
                    break;
                }
            }
        for (int stg : {32, 16, 8}) {
            if (P.bres) break;
            const size_t fixed = smem_for(P.bn, 0, stg);
            if (fixed + 2 * sbh <= 113 * 1024 && P.bn <= 128) {
                P.stg_cols = stg;
                P.stages = static_cast<int>(std::min<size_t>(MAX_STAGES, (113 * 1024 - fixed) / sbh));
                per = 2;
                break;
            }
        }
        if (!per && !P.bres)
            for (int stg : {32, 16, 8}) {
                const size_t fixed = smem_for(P.bn, 0, stg);
                if (fixed + 2 * sbh <= 227 * 1024) {
                    P.stg_cols = stg;
                    P.stages = static_cast<int>(std::min<size_t>(MAX_STAGES, (227 * 1024 - fixed) / sbh));
                    per = 1;
                    if (P.stages >= 3) break;
                }
            }
        if (!per) return nncb::fail("gemm: halo tile does not fit shared memory");
        P.stg_bufs = 1;
        const size_t smem = static_cast<size_t>(P.stages) * sbh + smem_for(P.bn, 0, P.stg_cols) + P.bres_bytes;
        encode_tma_out(&mc, P);
        const unsigned grid = static_cast<unsigned>(std::min<int64_t>(P.tiles, static_cast<int64_t>(ctx->sm_count) * per));
#ifdef NNCB_TC_TRACE_PROBE
        // probe builds: the halo launches' per-tile events too (NNCB_TC_TRACE)
        static const char* htrace_path = getenv("NNCB_TC_TRACE");
        static unsigned long long* htrace_buf = nullptr;
        const size_t htrace_bytes = static_cast<size_t>(grid) * 64 * 8 * sizeof(unsigned long long);
        if (htrace_path) {
            if (!htrace_buf) NNCB_CUDA(cudaMalloc(&htrace_buf, 2 * 148 * 64 * 8 * sizeof(unsigned long long)));
            NNCB_CUDA(cudaMemsetAsync(htrace_buf, 0, htrace_bytes, ctx->stream));
            P.trace = htrace_buf;
        }
        struct HTraceDump {
            const char* path; unsigned long long* buf; size_t bytes; nncb_ctx* ctx; const TcParams& P; unsigned grid; int per;
            ~HTraceDump() {
                if (!path) return;
                std::vector<unsigned long long> h(bytes / 8);
                cudaStreamSynchronize(ctx->stream);
                cudaMemcpy(h.data(), buf, bytes, cudaMemcpyDeviceToHost);
                if (FILE* f = fopen(path, "ab")) {
                    const long long hdr[6] = {static_cast<long long>(grid), static_cast<long long>(P.tiles), P.bn,
                                              P.stages, P.stg_bufs, per};
                    fwrite(hdr, sizeof(hdr), 1, f);
                    fwrite(h.data(), 8, h.size(), f);
                    fclose(f);
                }
            }
        } htrace_dump{htrace_path, htrace_buf, htrace_bytes, ctx, P, grid, per};
#endif
        if (per == 2 && P.colstats)
            tc_gemm_kernel<true, false, 2, false><<<grid, THREADS, smem, ctx->stream>>>(ma, mb, mc, P, em);
        else if (per == 2)
            tc_gemm_kernel<false, false, 2, false><<<grid, THREADS, smem, ctx->stream>>>(ma, mb, mc, P, em);
        else if (P.colstats)
            tc_gemm_kernel<true, false, 1, false><<<grid, THREADS, smem, ctx->stream>>>(ma, mb, mc, P, em);
        else
            tc_gemm_kernel<false, false, 1, false><<<grid, THREADS, smem, ctx->stream>>>(ma, mb, mc, P, em);
        NNCB_LAUNCHED(ctx);
        return 0;
    }
    if (g_force_wide && shp.per_sm == 2 && !manual) {
        // output-bound shapes: whole 128-byte row segments per store beat a deeper ring
        P.stg_cols = 32;
        const size_t fixed = smem_for(P.bn, 0, 32);
        P.stages = static_cast<int>(std::min<size_t>(MAX_STAGES, (113 * 1024 - fixed) / stage_bytes_for(P.bn)));
        if (P.stages < 2) { P.stages = shp.stages; P.stg_cols = shp.stg_cols; }
    }
    if (manual) {   // one CTA per SM (448 threads); take the deepest ring that fits
        P.stg_cols = 32;
        const size_t fixed = smem_for(P.bn, 0, P.stg_cols, tab_ints);
        P.stages = static_cast<int>(std::min<size_t>(MAX_STAGES, (227 * 1024 - fixed) / stage_bytes_for(P.bn)));
    }
    if (P.eg) eg_shape(P, P.bn);
    if (env_stages == 0 && env_persm == 0)
        pick_stg_bufs(P, P.bn, tab_ints, (manual || P.eg || shp.per_sm == 1) ? 227 * 1024 : 113 * 1024);
    const size_t smem = smem_for(P.bn, P.stages, P.stg_cols, tab_ints, P.stg_bufs) + eg_side_bytes(P);
    encode_tma_out(&mc, P);
    encode_eg_side(&em, P);
    int per_sm = (env_stages > 0) ? ((P.bn <= 128 && smem <= 113 * 1024) ? 2 : 1) : shp.per_sm;
    if (env_persm > 0 && (env_persm == 1 || 2 * smem <= 228 * 1024)) per_sm = env_persm;
    if (manual) per_sm = 1;   // the 448-thread build is compiled for one CTA per SM
    if (P.eg) per_sm = 1;      // the gradient epilogue needs the 168-register build
    unsigned grid = static_cast<unsigned>(std::min<int64_t>(P.tiles, static_cast<int64_t>(ctx->sm_count) * per_sm));
    const unsigned threads = manual ? THREADS + 128 : THREADS;
    // probe (NNCB_TC_TRACE=path): per-CTA tile event timestamps of each launch on
    // this path, appended to `path` (tools/tc_trace.py reads them)
    static const char* trace_path = getenv("NNCB_TC_TRACE");
    static unsigned long long* trace_buf = nullptr;
    const size_t trace_bytes = static_cast<size_t>(grid) * 64 * 8 * sizeof(unsigned long long);
    if (trace_path) {
        if (!trace_buf) NNCB_CUDA(cudaMalloc(&trace_buf, 2 * 148 * 64 * 8 * sizeof(unsigned long long)));
        NNCB_CUDA(cudaMemsetAsync(trace_buf, 0, trace_bytes, ctx->stream));
        P.trace = trace_buf;
    }
    struct TraceDump {
        const char* path; unsigned long long* buf; size_t bytes; nncb_ctx* ctx; const TcParams& P; unsigned grid; int per_sm;
        ~TraceDump() {
            if (!path) return;
            std::vector<unsigned long long> h(bytes / 8);
            cudaStreamSynchronize(ctx->stream);
            cudaMemcpy(h.data(), buf, bytes, cudaMemcpyDeviceToHost);
            if (FILE* f = fopen(path, "ab")) {
                const long long hdr[6] = {static_cast<long long>(grid), static_cast<long long>(P.tiles), P.bn, P.stages,
                                          P.stg_bufs, per_sm};
                fwrite(hdr, sizeof(hdr), 1, f);
                fwrite(h.data(), 8, h.size(), f);
                fclose(f);
            }
        }
    } trace_dump{trace_path, trace_buf, trace_bytes, ctx, P, grid, per_sm};
    if (P.colstats && manual)
        tc_gemm_kernel<true, true, 1, false><<<grid, threads, smem, ctx->stream>>>(ma, mb, mc, P, em);
    else if (manual)
        tc_gemm_kernel<false, true, 1, false><<<grid, threads, smem, ctx->stream>>>(ma, mb, mc, P, em);
    else if (P.eg)
        tc_gemm_kernel<true, false, 1, false, true><<<grid, threads, smem, ctx->stream>>>(ma, mb, mc, P, em);
    else if (P.colstats && per_sm == 1)
        tc_gemm_kernel<true, false, 1, false><<<grid, threads, smem, ctx->stream>>>(ma, mb, mc, P, em);
    else if (P.colstats)
        tc_gemm_kernel<true, false, 2, false><<<grid, threads, smem, ctx->stream>>>(ma, mb, mc, P, em);
    else
        tc_gemm_kernel<false, false, 2, false><<<grid, threads, smem, ctx->stream>>>(ma, mb, mc, P, em);
    NNCB_LAUNCHED(ctx);
    return 0;
}

bool encode_out_3d(CUtensorMap* map, float* base, int64_t n, int64_t m, int64_t splits) {
    cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)m, (cuuint64_t)splits};
    cuuint64_t strides[2] = {(cuuint64_t)(n * 4), (cuuint64_t)(n * m * 4)};
    cuuint32_t box[3] = {32, (cuuint32_t)BM, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = nncb::drv::table().tensorMapEncodeTiled(
        map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) nncb::set_error(std::string("cuTensorMapEncodeTiled(out3d): ") + nncb::drv::error_string(r));
    return r == CUDA_SUCCESS;
}

}  // namespace

namespace nncb {

int gemm_tc_impl(nncb_ctx* ctx, const nncb_gemm_desc* d, const float* a, int64_t lda, const float* b,
                 const float* bias, float* out, bool* handled, bool manual = false);

// im2col for the 3-channel stem: one warp per output pixel writes its row of
// kh*kw*ci (padded to ldk) columns contiguously; the per-column source offset
// and tap position come from a shared-memory table, so the inner loop is one
// predicated load and one coalesced store per element.
__global__ void __launch_bounds__(256) im2col_k(const float* __restrict__ x, float* __restrict__ cols,
                                                nncb_gemm_desc g, int K, int ldk) {
    extern __shared__ int tab[];   // [3][ldk]: source offset, dh, dw
    for (int k = threadIdx.x; k < ldk; k += blockDim.x) {
        int c = k % (int)g.ci, tap = k / (int)g.ci, dw = tap % (int)g.kw, dh = tap / (int)g.kw;
        tab[k] = k < K ? (dh * (int)g.iw + dw) * (int)g.ci + c : 0;
        tab[ldk + k] = k < K ? dh : -100000;
        tab[2 * ldk + k] = dw;
    }
    __syncthreads();
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int64_t P = g.n * g.oh * g.ow;
    for (int64_t p = blockIdx.x * 8 + warp; p < P; p += (int64_t)gridDim.x * 8) {
        const int ow = (int)(p % g.ow);
        const int64_t r = p / g.ow;
        const int oh = (int)(r % g.oh);
        const int64_t n = r / g.oh;
        const int h0 = oh * (int)g.sh - (int)g.pad_top, w0 = ow * (int)g.sw - (int)g.pad_left;
        const float* base = x + ((n * g.ih + h0) * g.iw + w0) * g.ci;
        float* out = cols + p * ldk;
        for (int k = lane; k < ldk; k += 32) {
            const int h = h0 + tab[ldk + k], w = w0 + tab[2 * ldk + k];
            float v = 0.f;
            if (h >= 0 && h < (int)g.ih && w >= 0 && w < (int)g.iw) v = __ldg(base + tab[k]);
            out[k] = v;
        }
    }
}


// ---- space-to-depth lowering for stride-2 convolutions with few channels ----
// y = conv_{k x k, stride 2}(x) equals a stride-1 VALID conv of the 2x2-blocked
// input x'[n, Y, X, (by*2+bx)*ci + c] = x[n, 2Y+by-pt, 2X+bx-pl, c] (zero outside)
// with weights W'[a, b, (by,bx,c), co] = W[2a+by, 2b+bx, c, co] (zero past k).
// When 4*ci <= 16 two horizontally adjacent blocks share one 32-channel group
// ("pack"): x''[Y, X] = [x'[Y, X] | x'[Y, X+1]] (16 channels each), and the
// kw' = ceil(k/2) horizontal taps pair up into ceil(kw'/2) taps two apart
// (dilation 2), halving K. Channels are zero-padded to 32 for the TMA path.
__device__ __forceinline__ void s2d_chan(int cc, int ci, bool pack, int& half, int& blk, int& c, bool& real) {
    half = pack ? cc / 16 : 0;
    const int cl = pack ? cc % 16 : cc;
    real = cl < 4 * ci;
    blk = real ? cl / ci : 0;
    c = real ? cl % ci : 0;
}

// Thread t writes 16 bytes (channels 4q..4q+3, q = t & 7) of lowered pixel
// t >> 3. The grid stride is a multiple of 8, so q and its channel -> (row,
// column, source channel) mapping are fixed per thread; 32-bit pixel index
// arithmetic (the host caps n*H2*W2*8 below 2^31).
__global__ void s2d_input_k(const float* __restrict__ x, float* __restrict__ xs, int n, int ih, int iw, int ci,
                            int H2, int W2, int pt, int pl, int pack) {
    const uint32_t total = static_cast<uint32_t>(n) * H2 * W2 * 8;
    uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    const int q = static_cast<int>(t & 7);
    int dy[4], dx[4], ch[4];
    bool real[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        int half, blk, c;
        s2d_chan(q * 4 + j, ci, pack != 0, half, blk, c, real[j]);
        dy[j] = (blk >> 1) - pt;
        dx[j] = 2 * half + (blk & 1) - pl;
        ch[j] = c;
    }
    const uint32_t stride = gridDim.x * blockDim.x;
    for (; t < total; t += stride) {
        const uint32_t pix = t >> 3;
        const uint32_t r = pix / static_cast<uint32_t>(W2);
        const int X = static_cast<int>(pix - r * W2);
        const uint32_t nn = r / static_cast<uint32_t>(H2);
        const int Y = static_cast<int>(r - nn * H2);
        const float* xn = x + static_cast<int64_t>(nn) * ih * iw * ci;
        float v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int iy = 2 * Y + dy[j], ix = 2 * X + dx[j];
            v[j] = (real[j] && iy >= 0 && iy < ih && ix >= 0 && ix < iw) ? __ldg(xn + (iy * iw + ix) * ci + ch[j]) : 0.f;
        }
        reinterpret_cast<float4*>(xs)[t] = make_float4(v[0], v[1], v[2], v[3]);
    }
}

// W''[a, b2, cc, co]: tap (a, b2) of the lowered conv, cc its 32-channel index
__global__ void s2d_weight_k(const float* __restrict__ w, float* __restrict__ ws, int kh, int kw, int ci, int co,
                             int kh2, int kwt, int pack) {
    const int total = kh2 * kwt * 32 * co;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        const int o = t % co, cc = (t / co) % 32, b2 = (t / (co * 32)) % kwt, a = t / (co * 32 * kwt);
        int half, blk, c;
        bool real;
        s2d_chan(cc, ci, pack != 0, half, blk, c, real);
        const int b = pack ? 2 * b2 + half : b2;
        const int dh = 2 * a + (blk >> 1), dw = 2 * b + (blk & 1);
        ws[t] = (real && dh < kh && dw < kw) ? w[((dh * kw + dw) * ci + c) * co + o] : 0.f;
    }
}

__global__ void s2d_wgrad_back_k(const float* __restrict__ dws, float* __restrict__ dw, int kh, int kw, int ci, int co,
                                 int kwt, int pack) {
    const int total = kh * kw * ci * co;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        const int o = t % co, c = (t / co) % ci, x = (t / (co * ci)) % kw, y = t / (co * ci * kw);
        const int blk = (y & 1) * 2 + (x & 1), b = x >> 1;
        const int b2 = pack ? b >> 1 : b, half = pack ? b & 1 : 0;
        const int cc = half * 16 + blk * ci + c;
        dw[t] = dws[(((y >> 1) * kwt + b2) * 32 + cc) * co + o];
    }
}

int gemm_tc_s2d(nncb_ctx* ctx, const nncb_gemm_desc* d, const float* a, const float* b, const float* bias, float* out,
                bool* handled) {
    static const bool allow_pack = !(getenv("NNCB_TC_S2D_PACK") && atoi(getenv("NNCB_TC_S2D_PACK")) == 0);
    const int pack = (allow_pack && 4 * d->ci <= 16) ? 1 : 0;
    const int kh2 = static_cast<int>((d->kh + 1) / 2), kw2 = static_cast<int>((d->kw + 1) / 2);
    const int kwt = pack ? (kw2 + 1) / 2 : kw2;   // horizontal taps of the lowered conv
    const int H2 = static_cast<int>(d->oh) + kh2 - 1, W2 = static_cast<int>(d->ow) + kw2 - 1;
    const size_t xs_bytes = sizeof(float) * static_cast<size_t>(d->n) * H2 * W2 * 32;
    const size_t w_bytes = sizeof(float) * static_cast<size_t>(kh2) * kwt * 32 * d->co;
    const size_t w_off = (xs_bytes + 255) / 256 * 256;
    char* ws = static_cast<char*>(workspace(ctx, w_off + w_bytes));
    if (!ws) return fail("space-to-depth: workspace allocation failed");
    float* xs = reinterpret_cast<float*>(ws);
    float* wsp = reinterpret_cast<float*>(ws + w_off);
    if (static_cast<int64_t>(d->n) * H2 * W2 * 8 >= (int64_t(1) << 31))
        return fail("space-to-depth: input exceeds the 32-bit lowering index");
    const int64_t key[8] = {d->n, d->ih, d->iw, d->ci, d->pad_top, d->pad_left, H2 * int64_t(1 << 20) + W2, pack};
    const bool reuse = d->kind == NNCB_CONV_WGRAD && (d->epilogue & NNCB_EPI_A_UNCHANGED) && ctx->s2d_src == a &&
                       ctx->s2d_ws == ctx->workspace && std::equal(key, key + 8, ctx->s2d_key);
    if (!reuse) {
        s2d_input_k<<<grid_for(ctx, static_cast<int64_t>(d->n) * H2 * W2 * 8, 256), 256, 0, ctx->stream>>>(
            a, xs, (int)d->n, (int)d->ih, (int)d->iw, (int)d->ci, H2, W2, (int)d->pad_top, (int)d->pad_left, pack);
        NNCB_LAUNCHED(ctx);
        ctx->s2d_src = a;
        ctx->s2d_ws = ctx->workspace;
        std::copy(key, key + 8, ctx->s2d_key);
    }
    nncb_gemm_desc dd = *d;
    dd.b_kmajor = nullptr;   // the lowered conv has its own weight layout
    dd.sgd_w = nullptr;      // its dW is scattered back afterwards: the caller applies the update
    dd.ih = H2; dd.iw = W2; dd.ci = 32; dd.kh = kh2; dd.kw = kwt; dd.sh = 1; dd.sw = 1;
    dd.pad_top = 0; dd.pad_left = 0;
    g_dil_w = pack ? 2 : 1;
    int rc = 0;
    if (d->kind == NNCB_CONV_FWD) {
        s2d_weight_k<<<grid_for(ctx, kh2 * kwt * 32 * d->co, 256), 256, 0, ctx->stream>>>(
            b, wsp, (int)d->kh, (int)d->kw, (int)d->ci, (int)d->co, kh2, kwt, pack);
        NNCB_LAUNCHED(ctx);
        rc = gemm_tc_impl(ctx, &dd, xs, 0, wsp, bias, out, handled);
        g_dil_w = 1;
        if (!rc && !*handled) return fail("space-to-depth route: conv rejected");
        return rc;
    }
    rc = gemm_tc_impl(ctx, &dd, xs, 0, b, nullptr, wsp, handled);   // dW'' = wgrad over x''
    g_dil_w = 1;
    if (rc) return rc;
    if (!*handled) return fail("space-to-depth route: wgrad rejected");
    s2d_wgrad_back_k<<<grid_for(ctx, d->kh * d->kw * d->ci * d->co, 256), 256, 0, ctx->stream>>>(
        wsp, out, (int)d->kh, (int)d->kw, (int)d->ci, (int)d->co, kwt, pack);
    NNCB_LAUNCHED(ctx);
    return 0;
}

std::atomic<int> g_manual_a{getenv("NNCB_TC_MANUAL_A") ? 1 : 0};
std::atomic<int> g_forced_tile{0};   // nncb_gemm_force_tile: width | pair << 16 (0: autotune)

int gemm_tc_route(nncb_ctx* ctx, const nncb_gemm_desc* d, const float* a, const float* b, const float* bias,
                  float* out, bool* handled);

// Tile selection. The choice (N-tile width, CTA pair, staging width, K-major
// weights, halo patches) changes the fp32 accumulation order, so it must be a
// function of the GEMM shape alone for results to be reproducible across
// processes and boxes. Modes (NNCB_TC_AUTOTUNE):
//   unset / "table"  deterministic: the committed per-shape table
//                    (tile_table.inc, produced by tools/tune_tiles.py from live
//                    measurements on a B200), plus entries imported with
//                    nncb_gemm_tuning_import; shapes not in it take the static
//                    rule. No timing, ever.
//   "live" / "1"     shapes not in the table are measured on first use outside
//                    capture: each candidate runs on a SCRATCH output (the
//                    caller's output and side inputs are never rewritten) and is
//                    timed with CUDA events; the fastest is remembered.
//                    nncb_gemm_tuning_export dumps the table.
//   "0"              the static rule only.
namespace {
struct TileEntry {
    const char* key;
    int choice;
};
const TileEntry kTileTable[] = {
#include "tile_table.inc"
    {nullptr, 0},
};
int tune_mode() {
    static const int m = [] {
        const char* e = getenv("NNCB_TC_AUTOTUNE");
        if (!e || !strcmp(e, "table")) return 1;
        if (!strcmp(e, "0")) return 0;
        if (!strcmp(e, "fresh")) return 3;   // live, ignoring the committed table (tools/tune_tiles.py)
        return 2;   // live
    }();
    return m;
}
std::mutex g_tune_mu;
std::map<std::string, int>& tuned_table() {
    static std::map<std::string, int> t = [] {
        std::map<std::string, int> m;
        if (tune_mode() == 3) return m;   // fresh: every shape measured anew
        for (const TileEntry& e : kTileTable)
            if (e.key) m[e.key] = e.choice;
        return m;
    }();
    return t;
}
size_t gemm_out_elems(const nncb_gemm_desc* d) {
    switch (d->kind) {
        case NNCB_DENSE_FWD: return (size_t)(d->batch * d->out_f);
        case NNCB_DENSE_DGRAD: return (size_t)(d->batch * d->in_f);
        case NNCB_DENSE_WGRAD: return (size_t)(d->in_f * d->out_f);
        case NNCB_CONV_FWD: return (size_t)(d->n * d->oh * d->ow * d->co);
        case NNCB_CONV_DGRAD: return (size_t)(d->n * d->ih * d->iw * d->ci);
        default: return (size_t)(d->kh * d->kw * d->ci * d->co);
    }
}
}  // namespace

// fp32 -> bf16 (round to nearest even), 4 elements per thread
__global__ void f32_to_bf16_k(const float* __restrict__ x, __nv_bfloat16* __restrict__ y, int64_t n) {
    const int64_t n4 = n / 4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(x) + i);
        __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
        uint2 o;
        o.x = *reinterpret_cast<uint32_t*>(&lo);
        o.y = *reinterpret_cast<uint32_t*>(&hi);
        reinterpret_cast<uint2*>(y)[i] = o;
    }
    for (int64_t i = n4 * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = __float2bfloat16_rn(x[i]);
}

// W[rows][cols] fp32 -> Wt[cols][rows] bf16 (K-major weights), 32x32 tiles
__global__ void transpose_bf16_k(const float* __restrict__ w, __nv_bfloat16* __restrict__ wt, int rows, int cols) {
    __shared__ float tile[32][33];
    const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
    for (int j = threadIdx.y; j < 32; j += 8) {
        const int r = by + j, c = bx + threadIdx.x;
        if (r < rows && c < cols) tile[j][threadIdx.x] = w[static_cast<int64_t>(r) * cols + c];
    }
    __syncthreads();
    for (int j = threadIdx.y; j < 32; j += 8) {
        const int c = bx + j, r = by + threadIdx.x;
        if (r < rows && c < cols) wt[static_cast<int64_t>(c) * rows + r] = __float2bfloat16_rn(tile[threadIdx.x][j]);
    }
}

// NNCB_PREC_BF16: the contraction runs kind::f16 on bf16 copies of its operands
// when both are K-major (forward and input-gradient contractions) with K blocks
// of 64 channels per tap (or one tap with K % 8 == 0); otherwise tf32.
// The route also has to pay: the per-call conversion reads the fp32 operands
// and writes bf16 copies, so only contractions whose arithmetic intensity
// (flops per unique fp32 byte, K*N / (2*(Ck + N)) per output pixel) is above
// the tf32 ridge point take it (measured: 3x3 convs and wide dense layers win;
// the memory-bound 1x1 convs lose). NNCB_BF16_MIN_INTENSITY overrides (0: all).
bool bf16_eligible(const nncb_gemm_desc* d) {
    if (d->epilogue & NNCB_EPI_RELU_GRAD) return false;
    int64_t K = 0, Ck = 0, N = 0;
    bool ok = false;
    switch (d->kind) {
        case NNCB_DENSE_FWD: K = Ck = d->in_f; N = d->out_f; ok = d->in_f % 8 == 0 && d->out_f % 8 == 0; break;
        case NNCB_DENSE_DGRAD: K = Ck = d->out_f; N = d->in_f; ok = d->out_f % 8 == 0 && d->in_f % 8 == 0; break;
        case NNCB_DENSE_WGRAD:
            // dW = x^T g over transposed (K-major) bf16 copies: per reduction row the
            // unique bytes are one row of x and one of g
            K = 2 * d->in_f; Ck = d->in_f; N = d->out_f;   // intensity in*out / (2*(in + out))
            ok = d->batch % 8 == 0 && d->in_f % 8 == 0 && d->out_f % 8 == 0;
            return ok && static_cast<double>(d->in_f) * d->out_f / (2.0 * (d->in_f + d->out_f)) >=
                             (getenv("NNCB_BF16_MIN_INTENSITY") ? atof(getenv("NNCB_BF16_MIN_INTENSITY")) : 128.0);
        case NNCB_CONV_FWD:
            Ck = d->ci; K = d->kh * d->kw * d->ci; N = d->co;
            ok = d->kh * d->kw == 1 ? d->ci % 8 == 0 : d->ci % 64 == 0;
            break;
        case NNCB_CONV_DGRAD:
            Ck = d->co; K = d->kh * d->kw * d->co; N = d->ci;
            ok = d->kh * d->kw == 1 ? d->co % 8 == 0 : d->co % 64 == 0;
            break;
        default: return false;
    }
    static const double min_i = getenv("NNCB_BF16_MIN_INTENSITY") ? atof(getenv("NNCB_BF16_MIN_INTENSITY")) : 128.0;
    return ok && static_cast<double>(K) * N / (2.0 * (Ck + N)) >= min_i;
}

// Writes the bf16 operand copies into the context's bf16 buffers.
int bf16_operands(nncb_ctx* ctx, const nncb_gemm_desc* d, const float* a, const float* b, const void** a16,
                  const void** b16) {
    const bool dense = d->kind <= NNCB_DENSE_WGRAD;
    if (d->kind == NNCB_DENSE_WGRAD) {   // x [B][in] -> x^T [in][B], g [B][out] -> g^T [out][B]
        auto* A = static_cast<__nv_bfloat16*>(bf16_buffer(ctx, 0, static_cast<size_t>(d->batch * d->in_f) * 2 + 16));
        auto* B = static_cast<__nv_bfloat16*>(bf16_buffer(ctx, 1, static_cast<size_t>(d->batch * d->out_f) * 2 + 16));
        if (!A || !B) return fail("bf16 gemm: operand buffer allocation failed");
        transpose_bf16_k<<<dim3((unsigned)((d->in_f + 31) / 32), (unsigned)((d->batch + 31) / 32)), dim3(32, 8), 0,
                           ctx->stream>>>(a, A, (int)d->batch, (int)d->in_f);
        NNCB_LAUNCHED(ctx);
        transpose_bf16_k<<<dim3((unsigned)((d->out_f + 31) / 32), (unsigned)((d->batch + 31) / 32)), dim3(32, 8), 0,
                           ctx->stream>>>(b, B, (int)d->batch, (int)d->out_f);
        NNCB_LAUNCHED(ctx);
        *a16 = A;
        *b16 = B;
        return 0;
    }
    const bool fwd = d->kind == NNCB_DENSE_FWD || d->kind == NNCB_CONV_FWD;
    const int64_t na = dense ? d->batch * (fwd ? d->in_f : d->out_f)
                             : (fwd ? d->n * d->ih * d->iw * d->ci : d->n * d->oh * d->ow * d->co);
    const int64_t krows = dense ? d->in_f : d->kh * d->kw * d->ci, cols = dense ? d->out_f : d->co;
    auto* A = static_cast<__nv_bfloat16*>(bf16_buffer(ctx, 0, static_cast<size_t>(na) * 2 + 16));
    auto* B = static_cast<__nv_bfloat16*>(bf16_buffer(ctx, 1, static_cast<size_t>(krows * cols) * 2 + 16));
    if (!A || !B) return fail("bf16 gemm: operand buffer allocation failed");
    f32_to_bf16_k<<<grid_for(ctx, (na + 3) / 4, 256), 256, 0, ctx->stream>>>(a, A, na);
    NNCB_LAUNCHED(ctx);
    if (fwd && !dense && d->b_kmajor) {   // the caller's K-major fp32 copy: convert only
        f32_to_bf16_k<<<grid_for(ctx, (krows * cols + 3) / 4, 256), 256, 0, ctx->stream>>>(d->b_kmajor, B, krows * cols);
    } else if (fwd) {                    // [K][N] -> K-major [N][K]
        transpose_bf16_k<<<dim3((unsigned)((cols + 31) / 32), (unsigned)((krows + 31) / 32)), dim3(32, 8), 0,
                           ctx->stream>>>(b, B, (int)krows, (int)cols);
    } else {                             // input gradient: the weights are K-major (K = cols) as stored
        f32_to_bf16_k<<<grid_for(ctx, (krows * cols + 3) / 4, 256), 256, 0, ctx->stream>>>(b, B, krows * cols);
    }
    NNCB_LAUNCHED(ctx);
    *a16 = A;
    *b16 = B;
    return 0;
}

// NNCB_PREC_TF32X3: dst[r][s][c] = part_s(src[r][c]) for s = 0..2, where part
// is hi = tf32 truncation (what the tensor core keeps of an fp32 operand) or
// lo = v - hi (exact in fp32); bit s of `lo_mask` selects lo for segment s.
__global__ void split3_k(const float* __restrict__ src, float* __restrict__ dst, int64_t rows, int64_t cols,
                         int lo_mask) {
    const int64_t total = rows * cols;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    if ((cols & 3) == 0) {
        const int64_t c4 = cols >> 2, t4 = total >> 2;
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < t4; i += stride) {
            const int64_t r = i / c4, c = i - r * c4;
            const float4 v = __ldg(reinterpret_cast<const float4*>(src) + i);
            float4 h, l;
            h.x = __uint_as_float(__float_as_uint(v.x) & 0xffffe000u);
            h.y = __uint_as_float(__float_as_uint(v.y) & 0xffffe000u);
            h.z = __uint_as_float(__float_as_uint(v.z) & 0xffffe000u);
            h.w = __uint_as_float(__float_as_uint(v.w) & 0xffffe000u);
            l = make_float4(__fsub_rn(v.x, h.x), __fsub_rn(v.y, h.y), __fsub_rn(v.z, h.z), __fsub_rn(v.w, h.w));
            float4* d = reinterpret_cast<float4*>(dst) + r * 3 * c4 + c;
#pragma unroll
            for (int sgm = 0; sgm < 3; ++sgm) __stcs(d + sgm * c4, (lo_mask >> sgm & 1) ? l : h);
        }
        return;
    }
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += stride) {
        const int64_t r = i / cols, c = i - r * cols;
        const float v = src[i];
        const float h = __uint_as_float(__float_as_uint(v) & 0xffffe000u), l = __fsub_rn(v, h);
        float* d = dst + r * 3 * cols + c;
#pragma unroll
        for (int sgm = 0; sgm < 3; ++sgm) d[sgm * cols] = (lo_mask >> sgm & 1) ? l : h;
    }
}

int split3(nncb_ctx* ctx, const float* src, float* dst, int64_t rows, int64_t cols, int lo_mask) {
    const bool vec = (cols & 3) == 0 && ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
    if ((cols & 3) == 0 && !vec) return fail("3xtf32: unaligned operand");
    split3_k<<<grid_for(ctx, (rows * cols + 3) / 4, 256), 256, 0, ctx->stream>>>(src, dst, rows, cols, lo_mask);
    NNCB_LAUNCHED(ctx);
    return 0;
}

// NNCB_PREC_TF32X3: the split copies are built here (A' with lo in the third
// K segment, B' with lo in the second), and the tf32 tensor-core GEMM runs on
// the K-concatenated problem. Reports handled = false (exact path) when the
// tensor-core route rejects the widened shape. Measured error (dense, uniform
// operands, against float64): 1.9e-6 at K = 96, 2.9e-5 at K = 2048, 7.2e-5 at
// K = 8192 relative to max|y| -- 20-300x below plain tf32 (6-7e-4), growing
// linearly in K: the floor is the tensor core's own fp32 accumulation (it does
// not round to nearest), not the dropped lo*lo term (emulated: 2.8e-7).
int gemm_tc_x3(nncb_ctx* ctx, const nncb_gemm_desc* d, const float* a, const float* b, const float* bias, float* out,
               bool* handled) {
    nncb_gemm_desc x = *d;
    x.precision = NNCB_PREC_TF32;
    x.b_kmajor = nullptr;                     // B' has its own layout
    x.epilogue &= ~NNCB_EPI_A_UNCHANGED;      // A' is rebuilt in a reused buffer every call
    int64_t a_rows = 0, a_cols = 0, b_rows = 0, b_cols = 0;
    switch (d->kind) {
        case NNCB_DENSE_FWD:   // x [B][in] . W [in][out]: K = in
            a_rows = d->batch; a_cols = d->in_f; b_rows = 1; b_cols = d->in_f * d->out_f; x.in_f = 3 * d->in_f; break;
        case NNCB_DENSE_DGRAD: // g [B][out] . W[in][out]^T: K = out
            a_rows = d->batch; a_cols = d->out_f; b_rows = d->in_f; b_cols = d->out_f; x.out_f = 3 * d->out_f; break;
        case NNCB_DENSE_WGRAD: // x^T g over the batch: K = batch
            a_rows = 1; a_cols = d->batch * d->in_f; b_rows = 1; b_cols = d->batch * d->out_f; x.batch = 3 * d->batch; break;
        case NNCB_CONV_FWD:    // K = taps x ci: channels of x, the ci rows of each weight tap
            a_rows = d->n * d->ih * d->iw; a_cols = d->ci; b_rows = d->kh * d->kw; b_cols = d->ci * d->co;
            x.ci = 3 * d->ci; break;
        case NNCB_CONV_DGRAD:  // K = taps x co: channels of g, the co columns of each weight row
            a_rows = d->n * d->oh * d->ow; a_cols = d->co; b_rows = d->kh * d->kw * d->ci; b_cols = d->co;
            x.co = 3 * d->co; break;
        case NNCB_CONV_WGRAD:  // K = images x pixels: the batch of x and of g
            a_rows = 1; a_cols = d->n * d->ih * d->iw * d->ci; b_rows = 1; b_cols = d->n * d->oh * d->ow * d->co;
            x.n = 3 * d->n; break;
        default: *handled = false; return 0;
    }
    float* A = static_cast<float*>(bf16_buffer(ctx, 0, static_cast<size_t>(a_rows * a_cols) * 12 + 16));
    float* B = static_cast<float*>(bf16_buffer(ctx, 1, static_cast<size_t>(b_rows * b_cols) * 12 + 16));
    if (!A || !B) return fail("3xtf32: operand buffer allocation failed");
    if (int rc = split3(ctx, a, A, a_rows, a_cols, 0x4)) return rc;   // hi, hi, lo
    if (int rc = split3(ctx, b, B, b_rows, b_cols, 0x2)) return rc;   // hi, lo, hi
    return gemm_tc(ctx, &x, A, B, bias, out, handled);
}

__global__ void bn_invstd_k(const float* __restrict__ var, float* __restrict__ inv, int64_t n, double eps) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x)
        inv[c] = static_cast<float>(1.0 / sqrt(static_cast<double>(var[c]) + eps));
}

// The tile codes the live tuner (and backends::tune_with_report) times for a
// contraction with N output columns.
std::vector<int> tile_candidates(const nncb_gemm_desc* d, int64_t N) {
    // bit 16: CTA pair (cta_group::2, 256-row tiles over two SMs)
    static const bool pairs = !(getenv("NNCB_TC_PAIR") && atoi(getenv("NNCB_TC_PAIR")) == 0);
    std::vector<int> cands = N <= 64 ? std::vector<int>{64} : N <= 128 ? std::vector<int>{64, 128}
                                                                        : std::vector<int>{128, 256};
    if (pairs) {
        cands.push_back(0x10000 | (N <= 64 ? 64 : 128));
        if (N > 128) cands.push_back(0x10000 | 256);
    }
    cands.push_back(0x20000 | (N <= 64 ? 64 : 128));   // bit 17: full-width staging at 2 CTAs/SM
    if (d->kind == NNCB_CONV_FWD || d->kind == NNCB_DENSE_FWD) {   // bit 18: K-major (transposed) weights
        const size_t nb = cands.size();
        for (size_t ci_ = 0; ci_ < nb; ++ci_) cands.push_back(cands[ci_] | 0x40000);
    }
    static const bool halo_on = !(getenv("NNCB_TC_HALO") && atoi(getenv("NNCB_TC_HALO")) == 0);
    const bool halo_fwd = d->kind == NNCB_CONV_FWD && d->ci % 32 == 0 && d->ow >= HALO_TW;
    // the space-to-depth stem (packed: its lowered conv has 2 taps per row spaced 2)
    const bool halo_stem = d->kind == NNCB_CONV_FWD && d->ci % 32 != 0 && d->sh == 2 && d->sw == 2 &&
                           4 * d->ci <= 16 && d->kw == 7 && d->kh == 7 && d->ow >= HALO_TW;
    const bool halo_dgrad = d->kind == NNCB_CONV_DGRAD && d->co % 32 == 0 && d->iw >= HALO_TW;
    if (halo_on && !(d->epilogue & NNCB_EPI_RELU_GRAD) &&
        (halo_stem || ((halo_fwd || halo_dgrad) && d->kh == 3 && d->kw == 3 && d->sh == 1 && d->sw == 1 &&
                       d->pad_top == 1 && d->pad_left == 1))) {   // bit 19: halo patches
        const size_t nb = cands.size();
        for (size_t ci_ = 0; ci_ < nb; ++ci_)
            if (!(cands[ci_] & 0x30000)) cands.push_back(cands[ci_] | 0x80000);   // 1-CTA tiles, default staging
        // (bit 20, full 3x3 patches: correct but measured no faster than
        // kernel-row patches at one CTA per SM; force_tile only)
        // (bit 21, resident B for 64-wide single-N-tile halo convs: correct,
        // but 15-20% slower on the 3x3 convs at one CTA per SM -- the
        // kernel-row halo tile is no longer L2-bound at ~79% of the N = 64 MMA
        // ceiling; force_tile only there. The stem's lowered conv keeps its
        // eight B tiles resident 3-4% faster (its main loop waits on the patch
        // loads at two stages per CTA): a candidate.)
        if (halo_stem) cands.push_back(0x280000 | 0x40000 | 64);
    }
    return cands;
}

int gemm_tc(nncb_ctx* ctx, const nncb_gemm_desc* d, const float* a, const float* b, const float* bias, float* out,
            bool* handled) {
    // inference BatchNorm epilogue: its per-column invstd, once per call
    struct BnScope {
        ~BnScope() { g_bn_inv = nullptr; }
    } bn_scope;
    if (d->epilogue & NNCB_EPI_BN_AFFINE) {
        const int64_t C = d->kind <= NNCB_DENSE_WGRAD ? d->out_f : d->co;
        float* inv = static_cast<float*>(bn_inv_buffer(ctx, static_cast<size_t>(C) * sizeof(float)));
        if (!inv) return fail("gemm: BN_AFFINE buffer allocation failed");
        bn_invstd_k<<<grid_for(ctx, C, 256), 256, 0, ctx->stream>>>(d->bn_var, inv, C, d->bn_eps);
        NNCB_LAUNCHED(ctx);
        g_bn_inv = inv;
    }
    // the bf16 route: operands converted once here; every tile candidate and
    // the final call below read the copies (g_bf16 scopes the whole call)
    const bool bf16 = d->precision == NNCB_PREC_BF16 && bf16_eligible(d);
    if (bf16) {
        const void *a16 = nullptr, *b16 = nullptr;
        if (int rc = bf16_operands(ctx, d, a, b, &a16, &b16)) return rc;
        a = static_cast<const float*>(a16);
        b = static_cast<const float*>(b16);
    }
    struct Bf16Scope {
        explicit Bf16Scope(bool on) { g_bf16 = on ? 1 : 0; }
        ~Bf16Scope() { g_bf16 = 0; }
    } bf16_scope(bf16);
    // a bf16 dense weight gradient is the forward contraction of the transposed
    // copies: dW[in][out] = (x^T)[in][B] . (g^T)[out][B]^T (both K-major)
    nncb_gemm_desc wd;
    if (bf16 && d->kind == NNCB_DENSE_WGRAD) {
        wd = *d;
        wd.kind = NNCB_DENSE_FWD;
        wd.batch = d->in_f;
        wd.in_f = d->batch;
        wd.out_f = d->out_f;
        wd.epilogue = 0;
        wd.colstats = nullptr;
        bias = nullptr;
    }
    if (bf16 && d->kind == NNCB_DENSE_WGRAD) d = &wd;
    const int mode = tune_mode();
    const bool enabled = mode >= 2;
    std::mutex& mu = g_tune_mu;
    std::map<std::string, int>& tuned = tuned_table();
    const bool dense = d->kind <= NNCB_DENSE_WGRAD;
    const int64_t N = d->kind == NNCB_DENSE_DGRAD ? d->in_f : d->kind == NNCB_CONV_DGRAD ? d->ci
                      : dense ? d->out_f : d->co;
    char key[256];
    snprintf(key, sizeof(key), "%d|%lld|%lld|%lld|%lld|%lld|%lld|%lld|%lld|%lld|%lld|%lld|%lld|%lld|%lld|%lld|%d|%d",
             d->kind, (long long)d->n, (long long)d->ih, (long long)d->iw, (long long)d->ci, (long long)d->co,
             (long long)d->kh, (long long)d->kw, (long long)d->sh, (long long)d->sw, (long long)d->oh,
             (long long)d->ow, (long long)d->pad_top, (long long)d->pad_left, (long long)d->batch,
             (long long)(d->in_f * 1000003 + d->out_f), d->epilogue & ~NNCB_EPI_A_UNCHANGED, g_manual_a.load() ? 1 : 0);
    if (bf16) strncat(key, "|bf16", sizeof(key) - strlen(key) - 1);
    int choice = g_forced_tile.load(std::memory_order_relaxed);
    const bool per_call = !choice && d->tile != 0;   // the plan's persisted choice
    if (per_call) choice = d->tile;
    if (!choice && mode != 0) {
        std::lock_guard<std::mutex> lk(mu);
        auto it = tuned.find(key);
        if (it != tuned.end()) choice = it->second;
    }
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(ctx->stream, &cap);
    if (!choice && enabled && cap == cudaStreamCaptureStatusNone) {
        const std::vector<int> cands = tile_candidates(d, N);
        // candidates write a scratch output: the caller's output (which an
        // epilogue side input may alias) is only written by the final call
        float* tmp_out = nullptr;
        NNCB_CUDA(cudaMalloc(&tmp_out, std::max<size_t>(gemm_out_elems(d), 1) * sizeof(float)));
        struct FreeTmp {
            float* p;
            ~FreeTmp() { cudaFree(p); }
        } free_tmp{tmp_out};
        cudaEvent_t e0, e1;
        NNCB_CUDA(cudaEventCreate(&e0));
        NNCB_CUDA(cudaEventCreate(&e1));
        float best = 0.f;
        for (int c : cands) {
            g_force_bn = c & 0xffff;
            g_force_pair = (c >> 16) & 1;
            g_force_wide = (c >> 17) & 1;
            g_force_tb = (c >> 18) & 1;
            g_force_halo = (c >> 20) & 1 ? 2 : (c >> 19) & 1;
            g_force_bres = (c >> 21) & 1;
            nncb_gemm_desc dt = *d;
            dt.sgd_w = nullptr;   // candidates never update weights
            int rc = gemm_tc_route(ctx, &dt, a, b, bias, tmp_out, handled);   // warm-up (and validity)
            if (rc || !*handled) {
                g_force_bn = 0;
                g_force_pair = 0;
                g_force_wide = 0;
                g_force_tb = 0;
                g_force_halo = 0;
                g_force_bres = 0;
                cudaEventDestroy(e0);
                cudaEventDestroy(e1);
                return rc;
            }
            cudaEventRecord(e0, ctx->stream);
            for (int r = 0; r < 3 && !rc; ++r) rc = gemm_tc_route(ctx, &dt, a, b, bias, tmp_out, handled);
            cudaEventRecord(e1, ctx->stream);
            g_force_bn = 0;
            g_force_pair = 0;
            g_force_wide = 0;
            g_force_tb = 0;
            g_force_halo = 0;
            g_force_bres = 0;
            if (rc) {
                cudaEventDestroy(e0);
                cudaEventDestroy(e1);
                return rc;
            }
            NNCB_CUDA(cudaEventSynchronize(e1));
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0, e1);
            if (!choice || ms < best) {
                best = ms;
                choice = c;
            }
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        NNCB_CUDA(cudaStreamSynchronize(ctx->stream));   // before the scratch output is freed
        std::lock_guard<std::mutex> lk(mu);
        tuned[key] = choice;
    }
    g_force_bn = choice & 0xffff;
    g_force_pair = (choice >> 16) & 1;
    g_force_wide = (choice >> 17) & 1;
    g_force_tb = (choice >> 18) & 1;
    g_force_halo = (choice >> 20) & 1 ? 2 : (choice >> 19) & 1;
    static const bool no_bres = getenv("NNCB_TC_NO_BRES") != nullptr;   // A/B knob: resident B off
    g_force_bres = no_bres ? 0 : (choice >> 21) & 1;
    int rc = gemm_tc_route(ctx, d, a, b, bias, out, handled);
    g_force_bn = 0;
    g_force_pair = 0;
    g_force_wide = 0;
    g_force_tb = 0;
    g_force_halo = 0;
    g_force_bres = 0;
    if (!rc && !*handled && per_call) {   // a persisted code this route rejects: the default choice
        nncb_gemm_desc d0 = *d;
        d0.tile = 0;
        return gemm_tc(ctx, &d0, a, b, bias, out, handled);
    }
    return rc;
}

int gemm_tc_route(nncb_ctx* ctx, const nncb_gemm_desc* d, const float* a, const float* b, const float* bias,
                  float* out, bool* handled) {
    *handled = false;
    const bool conv = d->kind >= NNCB_CONV_FWD;
    if (conv && d->ci % 32 != 0 && d->kh * d->kw > 1 && (d->kind == NNCB_CONV_FWD || d->kind == NNCB_CONV_WGRAD)) {
        // Channels that do not fill a 32-wide K block: builder warps can gather
        // A from the activation directly (no im2col matrix). Their 4-byte
        // gathers are slower than im2col for the stem today, so this is opt-in
        // (NNCB_TC_MANUAL_A=1) until the gather stages through a TMA patch.
        if (g_manual_a.load(std::memory_order_relaxed)) return gemm_tc_impl(ctx, d, a, 0, b, bias, out, handled, true);
        static const bool im2col_stem = getenv("NNCB_TC_STEM") && std::string(getenv("NNCB_TC_STEM")) == "im2col";
        if (d->sh == 2 && d->sw == 2 && 4 * d->ci <= 32 && !im2col_stem && drv::table().ok)
            return gemm_tc_s2d(ctx, d, a, b, bias, out, handled);
    }
    if (conv && d->ci % 32 != 0 && (d->kind == NNCB_CONV_FWD || d->kind == NNCB_CONV_WGRAD) && drv::table().ok) {
        // Channels that do not fill a 32-wide K block (the 3-channel stem): lower
        // to a dense tensor-core GEMM over an im2col workspace [pixels, kh*kw*ci].
        const int64_t K = d->kh * d->kw * d->ci, ldk = (K + 3) / 4 * 4;
        const int64_t P = d->n * d->oh * d->ow;
        if (d->co % 4 != 0 || d->co < 16) return 0;
        float* cols = static_cast<float*>(workspace(ctx, sizeof(float) * P * ldk));
        if (!cols) return fail("im2col: workspace allocation failed");
        ctx->s2d_src = nullptr;   // the columns overwrite any lowered space-to-depth input
        im2col_k<<<grid_for(ctx, P * 32, 256, 8), 256, 3 * ldk * sizeof(int), ctx->stream>>>(a, cols, *d,
                                                                                              static_cast<int>(K),
                                                                                              static_cast<int>(ldk));
        NNCB_LAUNCHED(ctx);
        nncb_gemm_desc dd{};
        dd.kind = d->kind == NNCB_CONV_FWD ? NNCB_DENSE_FWD : NNCB_DENSE_WGRAD;
        dd.precision = d->precision;
        dd.epilogue = d->epilogue;
        dd.batch = P;
        dd.in_f = K;
        dd.out_f = d->co;
        dd.colstats = d->colstats;
        dd.colstats_finalize = d->colstats_finalize;
        dd.colstats_eps = d->colstats_eps;
        dd.bn_mean = d->bn_mean;
        dd.bn_var = d->bn_var;
        dd.bn_gamma = d->bn_gamma;
        dd.bn_beta = d->bn_beta;
        dd.bn_eps = d->bn_eps;
        dd.residual = d->residual;
        int rc = gemm_tc_impl(ctx, &dd, cols, ldk, b, bias, out, handled);
        if (!rc && !*handled) return fail("im2col route: dense GEMM rejected");
        return rc;
    }
    return gemm_tc_impl(ctx, d, a, 0, b, bias, out, handled);
}

// W[rows][cols] -> Wt[cols][rows], 32x32 shared-memory tiles (coalesced both ways)
__global__ void transpose_k(const float* __restrict__ w, float* __restrict__ wt, int rows, int cols) {
    __shared__ float tile[32][33];
    const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
    for (int j = threadIdx.y; j < 32; j += 8) {
        const int r = by + j, c = bx + threadIdx.x;
        if (r < rows && c < cols) tile[j][threadIdx.x] = w[static_cast<int64_t>(r) * cols + c];
    }
    __syncthreads();
    for (int j = threadIdx.y; j < 32; j += 8) {
        const int c = bx + j, r = by + threadIdx.x;
        if (r < rows && c < cols) wt[static_cast<int64_t>(c) * rows + r] = tile[threadIdx.x][j];
    }
}

// Many transposes in one launch: block -> (job, 32x32 tile) by a binary search
// over the jobs' tile prefix sums.
__global__ void transpose_batch_k(const nncb_transpose_job* __restrict__ jobs, int n, int64_t total) {
    __shared__ float tile[32][33];
    for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
        int lo = 0, hi = n - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) / 2;
            if (jobs[mid].tile0 <= t) lo = mid; else hi = mid - 1;
        }
        const nncb_transpose_job J = jobs[lo];
        const int64_t local = t - J.tile0;
        const int tcols = (J.cols + 31) / 32;
        const int bx = static_cast<int>(local % tcols) * 32, by = static_cast<int>(local / tcols) * 32;
        for (int j = threadIdx.y; j < 32; j += 8) {
            const int r = by + j, c = bx + threadIdx.x;
            if (r < J.rows && c < J.cols) tile[j][threadIdx.x] = J.src[static_cast<int64_t>(r) * J.cols + c];
        }
        __syncthreads();
        for (int j = threadIdx.y; j < 32; j += 8) {
            const int c = bx + j, r = by + threadIdx.x;
            if (r < J.rows && c < J.cols) J.dst[static_cast<int64_t>(c) * J.rows + r] = tile[threadIdx.x][j];
        }
        __syncthreads();
    }
}

int gemm_tc_impl(nncb_ctx* ctx, const nncb_gemm_desc* d, const float* a, int64_t lda, const float* b,
                 const float* bias, float* out, bool* handled, bool manual) {
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
    if (co % 4 != 0 || co < 16) return 0;
    if (!manual && (kh * kw > MAX_TAPS || lda % 4 != 0)) return 0;
    if (!single_tap && ci % 32 != 0 && !manual) return 0;
    if (manual && (dense || kind == 1)) return 0;
    if (single_tap && ci % 4 != 0 && lda == ci) return 0;
    if (kind == 1 && ((!single_tap && co % 32 != 0) || sh > 2 || sw > 2)) return 0;
    if (n * std::max(ih, oh) * std::max(iw, ow) * std::max(ci, co) >= (int64_t(1) << 31) * 4) return 0;

    TcParams P;
    memset(&P, 0, sizeof(P));
    P.kel = BK;
    P.debug = dbg;
    P.dil_w = g_dil_w;
    CUtensorMap ma, mb;
    memset(&ma, 0, sizeof(ma));
    if (manual) {
        P.xa = a;
        P.ih_ = (int)ih; P.iw_ = (int)iw;
        P.K_ = (int)(kh * kw * ci);
        P.ci = (int)ci; P.kw_ = (int)kw;
        P.sh = (int)sh; P.sw = (int)sw; P.pt = (int)pt; P.pl = (int)pl;
    }
    if (kind == 0 || kind == 1) {
        P.mode = MODE_CONV;
        const bool fwd = kind == 0;
        const int64_t Nc = fwd ? co : ci;             // GEMM N
        const int64_t Ck = fwd ? ci : co;             // channels per tap (K block source)
        P.bn = pick_bn(Nc);
        P.pair = (g_force_pair && !manual && P.bn >= 64) ? 1 : 0;
        P.N = Nc;
        P.ldc = Nc;
        P.cblocks = static_cast<int>((Ck + 31) / 32);
        if (g_bf16) {
            if (manual || (!single_tap && Ck % 64 != 0) || Ck % 8 != 0) return 0;
            P.bf16 = 1;
            P.kel = 64;
            P.cblocks = static_cast<int>((Ck + 63) / 64);
        }
        if (fwd) {
            P.gn = (int)n; P.gh = (int)oh; P.gw = (int)ow;
            P.out_h = (int)oh; P.out_w = (int)ow; P.out_s = 1;
            P.mh = (int)sh; P.mw = (int)sw;
            P.ntaps[0] = (int)(kh * kw);
            P.tap0[0] = 0;
            if (manual) {   // one "tap" whose K blocks run over the whole flattened (tap, ci) patch
                P.ntaps[0] = 1;
                P.cblocks = (int)((kh * kw * ci + BK - 1) / BK);
            }
            for (int t = 0; t < (manual ? 1 : kh * kw); ++t) {
                P.off_h[t] = manual ? 0 : (int)(t / kw - pt);
                P.off_w[t] = manual ? 0 : (int)((t % kw) * g_dil_w - pl);
                P.brow[t] = manual ? 0 : (int)(t * ci);
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
        // halo: forward, or a stride-1 dgrad (its tap table visits kernel rows
        // with off_w = -1, 0, 1 in order, like the forward)
        // (or the space-to-depth stem: 2 taps per row spaced 2, any padding)
        const bool halo33 = kh == 3 && kw == 3 && pt == 1 && pl == 1 && g_dil_w == 1;
        const bool halo_s2d = fwd && kw == 2 && g_dil_w == 2 && kh <= 4;
        if (g_force_halo && !g_bf16 && !manual && !P.pair && !(d->epilogue & NNCB_EPI_RELU_GRAD) && (halo33 || halo_s2d) &&
            sh == 1 && sw == 1 && Ck % 32 == 0 && (fwd ? ow : iw) >= HALO_TW &&
            2 * (HALO_A_BYTES + kw * static_cast<size_t>(P.bn) * BK * 4) + smem_for(P.bn, 0, 8) <= 227 * 1024) {
            // (a two-stage ring must fit: 256-wide tiles do not)
            const bool full = halo33 && g_force_halo == 2 &&
                              2 * (HALO9_A_BYTES + 9 * static_cast<size_t>(P.bn) * BK * 4) + smem_for(P.bn, 0, 8) <= 227 * 1024;
            P.halo = full ? 2 : 1;
            P.TN = 1;
            P.TH = HALO_TH;
            P.TW = HALO_TW;
            P.halo_kw = static_cast<int>(kw);
            P.ntaps[0] = full ? 1 : static_cast<int>(kh);   // k-steps per channel block: one per kernel row, or one
            const size_t bres = static_cast<size_t>(P.ntaps[0] * P.halo_kw) * P.cblocks * P.bn * BK * 4;
            if (g_force_bres && !full && Nc <= P.bn &&
                bres + 2 * HALO_A_BYTES + smem_for(P.bn, 0, 8) <= 227 * 1024) {
                P.bres = 1;
                P.bres_bytes = static_cast<uint32_t>(bres);
            }
        }
        P.tiles_w = (P.gw + P.TW - 1) / P.TW;
        P.tiles_h = (P.gh + P.TH - 1) / P.TH;
        const int tiles_n = (P.gn + P.TN - 1) / P.TN;
        const int64_t tiles = static_cast<int64_t>(tiles_n) * P.tiles_h * P.tiles_w;
        if (tiles >= (int64_t(1) << 31) || P.TW * P.mw > 256 || P.TH * P.mh > 256) return 0;
        // A: the activation (x for fwd, g for dgrad) as {C, W, H, N}
        const float* act = a;
        if (fwd && P.halo) {
            if (!encode_4d(&ma, act, ci, iw, ih, n, 32, P.TW + 2, P.TH + (P.halo == 2 ? 2 : 0), 1, 1, 1, false, lda)) return 1;
        } else if (fwd) {
            if (!manual && !encode_4d(&ma, act, ci, iw, ih, n, P.kel, P.TW * (int)sw, P.TH * (int)sh, P.TN, (int)sw,
                                      (int)sh, false, lda, P.bf16 ? 2 : 4))
                return 1;
        } else if (P.halo) {
            if (!encode_4d(&ma, act, co, ow, oh, n, 32, P.TW + 2, P.TH + (P.halo == 2 ? 2 : 0), 1, 1, 1, false)) return 1;
        } else {
            if (!encode_4d(&ma, act, co, ow, oh, n, P.kel, P.TW, P.TH, P.TN, 1, 1, false, 0, P.bf16 ? 2 : 4)) return 1;
        }
        // B: weights [kh*kw*ci, co]
        const int64_t kfull = kh * kw * ci;
        if (P.bf16 && fwd) {
            // bf16 route: b is the K-major bf16 copy [co][kh*kw*ci] (gemm_tc)
            P.b_mn = 0;
            P.bt = 1;
            if (!encode_2d(&mb, b, kfull, co, P.kel, P.pair ? P.bn / 2 : P.bn, false, 2)) return 1;
        } else if (P.bf16) {
            // bf16 route, dgrad: b is the bf16 copy of the weights [kh*kw*ci][co] (K = co)
            P.b_mn = 0;
            if (!encode_2d(&mb, b, co, kh * kw * ci, P.kel, P.pair ? P.bn / 2 : P.bn, false, 2)) return 1;
        } else if (fwd && g_force_tb && !manual && kfull % 4 == 0) {
            // K-major copy [co][kh*kw*ci]: the tensor core reads K-major tf32
            // operands faster than MN-major ones (measured fwd vs dgrad). The
            // caller's copy (b_kmajor, refreshed once per plan) or a per-call one.
            const float* wt = d->b_kmajor;
            if (!wt) {
                float* w2 = static_cast<float*>(wt_buffer(ctx, sizeof(float) * kfull * co));
                if (!w2) return fail("conv fwd: transposed-weight buffer allocation failed");
                transpose_k<<<dim3((unsigned)((co + 31) / 32), (unsigned)((kfull + 31) / 32)), dim3(32, 8), 0, ctx->stream>>>(
                    b, w2, (int)kfull, (int)co);
                NNCB_LAUNCHED(ctx);
                wt = w2;
            }
            P.b_mn = 0;
            P.bt = 1;
            if (!encode_2d(&mb, wt, kfull, co, BK, P.pair ? P.bn / 2 : P.bn, false)) return 1;
        } else if (fwd) {
            P.b_mn = 1;
            if (!encode_2d(&mb, b, co, kh * kw * ci, 32, BK, true)) return 1;
        } else {
            P.b_mn = 0;
            if (!encode_2d(&mb, b, co, kh * kw * ci, BK, P.pair ? P.bn / 2 : P.bn, false)) return 1;
        }
        P.bias = (fwd && (d->epilogue & NNCB_EPI_BIAS)) ? bias : nullptr;
        if (fwd && (d->epilogue & NNCB_EPI_BN_AFFINE)) {
            if (!g_bn_inv) return fail("gemm: BN_AFFINE without its per-call invstd");
            P.bn_mean = d->bn_mean;
            P.bn_inv = g_bn_inv;
            P.bn_gamma = d->bn_gamma;
            P.bn_beta = d->bn_beta;
            P.relu = (d->epilogue & NNCB_EPI_RELU) ? 1 : 0;
            P.res = (d->epilogue & NNCB_EPI_RESIDUAL) ? d->residual : nullptr;
            if ((d->epilogue & NNCB_EPI_RESIDUAL) && (!d->residual || P.out_s != 1))
                return fail("gemm: NNCB_EPI_RESIDUAL needs a residual laid out like the output");
        }
        P.out = out;
        P.colstats = (fwd && (d->epilogue & NNCB_EPI_COLSTATS)) ? d->colstats : nullptr;
        if (d->epilogue & NNCB_EPI_RELU_GRAD) {
            if (!d->eg_mask || !d->eg_x || !d->eg_stats || !d->eg_sums || P.colstats)
                return fail("gemm: NNCB_EPI_RELU_GRAD needs eg_mask, eg_x, eg_stats, eg_sums (and no COLSTATS)");
            P.eg = 1;
            P.eg_mask = d->eg_mask;
            P.eg_res = d->eg_res;
            P.eg_x = d->eg_x;
            P.eg_stats = d->eg_stats;
            P.colstats = d->eg_sums;   // the CS build accumulates the dy sums
        }
        if (P.colstats && !P.eg && d->colstats_finalize) {
            P.cs_stats = d->colstats_finalize;
            P.cs_eps = d->colstats_eps;
            P.cs_rows = d->kind == NNCB_DENSE_FWD ? d->batch : d->n * d->oh * d->ow;
        }
        if (P.colstats) {   // fixed-point accumulators + CTA ticket; the kernel's last CTA writes colstats
            const size_t fb = sizeof(unsigned long long) * (4 * static_cast<size_t>(Nc) + 1);
            P.cs_fixed = static_cast<unsigned long long*>(colstats_fixed_buffer(ctx, fb));
            if (!P.cs_fixed) return fail("gemm: column-statistics buffer allocation failed");
            NNCB_CUDA(cudaMemsetAsync(P.cs_fixed, 0, fb, ctx->stream));
        }
        P.n_tiles = (Nc + P.bn - 1) / P.bn;
        P.pix_tiles = tiles;
        P.pix_pairs = (tiles + 1) / 2;
        P.tiles = (P.pair ? P.pix_pairs : tiles) * P.n_tiles * (fwd ? 1 : sh * sw);
        // TMA-store epilogue when output pixels are dense (fwd, or stride-1 dgrad)
        CUtensorMap mc;
        memset(&mc, 0, sizeof(mc));
        P.tma_store = (P.out_s == 1 && Nc % 4 == 0) ? 1 : 0;
        if (P.tma_store && !encode_4d(&mc, out, Nc, P.out_w, P.out_h, P.gn, 32, P.TW, P.TH, P.TN, 1, 1, false))
            return 1;
        *handled = true;
        return launch(ctx, ma, mb, mc, P);
    }
    // ---- wgrad ----------------------------------------------------------------
    P.mode = MODE_WGRAD;
    P.b_mn = 1;
    P.M = kh * kw * ci;
    P.N = co;
    P.ldc = co;
    P.bn = pick_bn(co);
    P.pair = (g_force_pair && !manual && P.bn >= 64) ? 1 : 0;
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
    if (!manual &&
        !encode_4d(&ma, a, ci, iw, ih, n, 32, P.TW * (int)sw, P.TH * (int)sh, P.TN, (int)sw, (int)sh, true, lda))
        return 1;
    if (!encode_4d(&mb, b, co, ow, oh, n, 32, P.TW, P.TH, P.TN, 1, 1, true)) return 1;
    P.out = out;
    if (P.splits > 1) {
        P.partial = static_cast<float*>(scratch(ctx, sizeof(float) * P.splits * P.M * P.N));
        if (!P.partial) return fail("wgrad: split-K workspace allocation failed");
    }
    P.n_tiles = nt;
    P.m_tiles = mt;
    P.m_pairs = (mt + 1) / 2;
    P.tiles = (P.pair ? P.m_pairs : mt) * nt * P.splits;
    CUtensorMap mc;
    P.tma_store = 1;
    if (!encode_out_3d(&mc, P.splits > 1 ? P.partial : out, co, P.M, P.splits)) return 1;
    *handled = true;
    if (int rc = launch(ctx, ma, mb, mc, P)) return rc;
    if (P.splits > 1) {
        int64_t count = P.M * P.N;
        const bool sgd = d->sgd_w && d->sgd_lr && (d->kind == NNCB_CONV_WGRAD || d->kind == NNCB_DENSE_WGRAD) &&
                         (reinterpret_cast<uintptr_t>(d->sgd_w) & 15) == 0;
        if (sgd && count % 4 == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
            NNCB_CUDA(launch_pdl(splitk_reduce4_sgd_kernel, dim3(grid_for(ctx, count / 4, 256)), dim3(256), ctx->stream,
                                 reinterpret_cast<const float4*>(P.partial), reinterpret_cast<float4*>(out), count / 4,
                                 P.splits, reinterpret_cast<float4*>(d->sgd_w), d->sgd_lr, d->sgd_scale));
            g_sgd_applied = true;
        } else if (count % 4 == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0)
            NNCB_CUDA(launch_pdl(splitk_reduce4_kernel, dim3(grid_for(ctx, count / 4, 256)), dim3(256), ctx->stream,
                                 reinterpret_cast<const float4*>(P.partial), reinterpret_cast<float4*>(out), count / 4,
                                 P.splits));
        else
            NNCB_CUDA(launch_pdl(splitk_reduce_kernel, dim3(grid_for(ctx, count, 256)), dim3(256), ctx->stream,
                                 static_cast<const float*>(P.partial), out, count, P.splits));
        NNCB_LAUNCHED(ctx);
    }
    return 0;
}

}  // namespace nncb

// Route selection for convolutions whose channel count does not fill a 32-wide
// K block: 1 = builder-warp gather (manual A), 0 = im2col workspace.
extern "C" int nncb_transpose_batch(nncb_ctx* ctx, const nncb_transpose_job* jobs, int n, int64_t total_tiles) {
    if (n <= 0 || total_tiles <= 0) return 0;
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(total_tiles, static_cast<int64_t>(ctx->sm_count) * 16));
    nncb::transpose_batch_k<<<grid, dim3(32, 8), 0, ctx->stream>>>(jobs, n, total_tiles);
    NNCB_LAUNCHED(ctx);
    return 0;
}

extern "C" int nncb_gemm_set_manual_a(int on) {
    nncb::g_manual_a.store(on ? 1 : 0);
    return 0;
}

// Forces the tensor-core tile choice for subsequent GEMMs (tests / tuning):
// code = N-tile width (64/128/256) | 1 << 16 for CTA pairs; 0 restores autotuning.
extern "C" int nncb_gemm_force_tile(int code) {
    nncb::g_forced_tile.store(code);
    return 0;
}

extern "C" int nncb_gemm_tuning_export(char* buf, size_t cap, size_t* needed) {
    std::string text;
    {
        std::lock_guard<std::mutex> lk(nncb::g_tune_mu);
        for (const auto& [k, c] : nncb::tuned_table()) text += k + " " + std::to_string(c) + "\n";
    }
    if (needed) *needed = text.size() + 1;
    if (buf && cap) {
        const size_t n = std::min(cap - 1, text.size());
        memcpy(buf, text.data(), n);
        buf[n] = 0;
    }
    return 0;
}

extern "C" int nncb_gemm_tuning_import(const char* text) {
    if (!text) return 0;
    std::lock_guard<std::mutex> lk(nncb::g_tune_mu);
    const char* p = text;
    while (*p) {
        const char* eol = strchr(p, '\n');
        std::string line(p, eol ? eol : p + strlen(p));
        p = eol ? eol + 1 : p + strlen(p);
        const size_t sp = line.rfind(' ');
        if (line.empty() || sp == std::string::npos) continue;
        nncb::tuned_table()[line.substr(0, sp)] = atoi(line.c_str() + sp + 1);
    }
    return 0;
}

extern "C" int nncb_gemm_tuning_mode(void) { return nncb::tune_mode(); }

namespace nncb {
bool take_sgd_applied() {
    const bool v = g_sgd_applied;
    g_sgd_applied = false;
    return v;
}
}  // namespace nncb

extern "C" int nncb_gemm_candidates(const nncb_gemm_desc* d, int32_t* codes, int cap, int* n) {
    if (!d || !n) return nncb::fail("nncb_gemm_candidates: null argument");
    std::vector<int> c;
    if (d->precision != NNCB_PREC_FP32 && !(d->kind == NNCB_CONV_DGRAD && d->kh * d->kw > 1 && d->ci % 32)) {
        const bool dense = d->kind <= NNCB_DENSE_WGRAD;
        const int64_t N = d->kind == NNCB_DENSE_DGRAD ? d->in_f : d->kind == NNCB_CONV_DGRAD ? d->ci
                          : dense ? d->out_f : d->co;
        c = nncb::tile_candidates(d, N);
    }
    *n = static_cast<int>(c.size());
    for (int i = 0; i < *n && i < cap && codes; ++i) codes[i] = c[i];
    return 0;
}

extern "C" int nncb_gemm_time_tile(nncb_ctx* ctx, const nncb_gemm_desc* d, const float* a, const float* b,
                                   const float* bias, float* out, int32_t code, int warmup, int trials,
                                   float* median_ms) {
    if (!d || !median_ms || trials < 1) return nncb::fail("nncb_gemm_time_tile: bad argument");
    nncb_gemm_desc x = *d;
    x.tile = code;
    for (int i = 0; i < warmup; ++i)
        if (int rc = nncb_gemm(ctx, &x, a, b, bias, out)) return rc;
    std::vector<float> ms(static_cast<size_t>(trials));
    cudaEvent_t e0, e1;
    NNCB_CUDA(cudaEventCreate(&e0));
    NNCB_CUDA(cudaEventCreate(&e1));
    int rc = 0;
    for (int t = 0; t < trials && !rc; ++t) {
        cudaEventRecord(e0, ctx->stream);
        rc = nncb_gemm(ctx, &x, a, b, bias, out);
        cudaEventRecord(e1, ctx->stream);
        if (!rc && cudaEventSynchronize(e1) == cudaSuccess) cudaEventElapsedTime(&ms[static_cast<size_t>(t)], e0, e1);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (rc) return rc;
    std::sort(ms.begin(), ms.end());
    *median_ms = ms[ms.size() / 2];
    return 0;
}
