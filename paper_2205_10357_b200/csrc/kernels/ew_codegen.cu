// ew_codegen.cu -- fused elementwise groups: register program -> sm_100a kernel.
//
// Replaces the reference's per-element interpreter run_ew<T> (runtime.cpp:280-306),
// which walks the EwInstr program (plan.cpp:296-337) once per element on one CPU
// core (0.081 GB/s on the C2 chain). Here the program is a
// compile-time specialisation: each register becomes a local variable, the
// program body is emitted straight-line, and NVRTC compiles it for sm_100a once
// per distinct program (cached per context). Each thread streams 2 x float4 per
// element-mode slot per iteration (128-bit coalesced loads/stores, grid-stride,
// grid = multiple of the SM count), so the kernel is HBM-bound.
//
// Arithmetic is bitwise-identical to the reference: Add/Mul use __fadd_rn /
// __fmul_rn (no FMA contraction), ReLU is x > 0 ? x : 0 (-0 and NaN -> +0,
// kernels.hpp:47-50), ReluGrad masks on the forward input (kernels.hpp:52-55).
#include <nvrtc.h>

#include <cstdio>
#include <cstring>
#include <mutex>
#include <numeric>
#include <set>
#include <sstream>
#include <map>

#include "driver_api.cuh"
#include "nncb_internal.cuh"

struct nncb_ew_kernel {
    std::string source;
    CUmodule module = nullptr;
    CUfunction fn = nullptr;
    int n_slots = 0;
    bool uses_channels = false;
    int n_reduce = 0;                      // REDUCE_BN_GRAD instructions (<= 2)
    int reduce_sg[2] = {-1, -1}, reduce_sgx[2] = {-1, -1};   // their output slots
    int reduce_stats[2] = {0, 0};          // 1: REDUCE_STATS (mean / invstd into one [2C] slot)
    double reduce_eps[2] = {0.0, 0.0};
    int red_blocks = 4;                    // resident blocks per SM the reduction build is budgeted for
    int ring_bytes = 0;                    // dynamic shared memory of the cp.async load ring (0: none)
};

void nncb::ew_release(nncb_ew_kernel* k) {
    if (!k) return;
    if (k->module) nncb::drv::table().moduleUnload(k->module);
    delete k;
}

namespace {

constexpr int kMaxSlots = 48;

const char* kPrelude = R"(
typedef long long i64;
struct EwArgs { float* p[48]; i64 n; i64 C; int cs; double* part; };
__device__ __forceinline__ float relu_(float x) { return x > 0.f ? x : 0.f; }
__device__ __forceinline__ float relu_grad_(float x, float g) { return x > 0.f ? g : 0.f; }
__device__ __forceinline__ float bn_apply_(float x, float m, float s, float ga, float be) {
  return __fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(x, m), s), ga), be);
}
__device__ __forceinline__ float bn_infer_(float x, float m, float v, float ga, float be, double eps) {
  float s = (float)(1.0 / sqrt((double)v + eps));
  return bn_apply_(x, m, s, ga, be);
}
__device__ __forceinline__ float gelu_(float x) {
  double xd = (double)x;
  return (float)(0.5 * xd * (1.0 + erf(xd * 0.70710678118654752440)));
}
__device__ __forceinline__ float gelu_grad_(float x, float g) {
  double xd = (double)x;
  double cdf = 0.5 * (1.0 + erf(xd * 0.70710678118654752440));
  double pdf = exp(-0.5 * xd * xd) * 0.39894228040143267794;
  return (float)((double)g * (cdf + xd * pdf));
}
__device__ __forceinline__ float gelu_fast_(float x) {
  return __fmul_rn(__fmul_rn(0.5f, x), __fadd_rn(1.f, erff(__fmul_rn(x, 0.70710678118654752440f))));
}
__device__ __forceinline__ float gelu_grad_fast_(float x, float g) {
  const float cdf = __fmul_rn(0.5f, __fadd_rn(1.f, erff(__fmul_rn(x, 0.70710678118654752440f))));
  const float pdf = __fmul_rn(__expf(__fmul_rn(__fmul_rn(-0.5f, x), x)), 0.39894228040143267794f);
  return __fmul_rn(g, __fadd_rn(cdf, __fmul_rn(x, pdf)));
}
__device__ __forceinline__ float bn_grad_(float x, float g, float m, float s, float ga, float sg, float sgx,
                                          float cnt) {
  float xhat = __fmul_rn(__fsub_rn(x, m), s);
  float t = __fadd_rn(sg, __fmul_rn(xhat, sgx));
  float u = __fsub_rn(g, __fdiv_rn(t, cnt));
  return __fmul_rn(__fmul_rn(ga, s), u);
}
__device__ __forceinline__ float bn_grad_fast_(float x, float g, float m, float s, float ga, float sg, float sgx,
                                               float cnt) {
  const float k1 = __fdiv_rn(sg, cnt), k2 = __fdiv_rn(sgx, cnt);   // per channel: hoisted out of the loop
  const float xhat = __fmul_rn(__fsub_rn(x, m), s);
  return __fmul_rn(__fmul_rn(ga, s), __fmaf_rn(-xhat, k2, __fsub_rn(g, k1)));
}
)";

std::string reg(int r) { return "r" + std::to_string(r); }

bool writes_reg(int op) {
    return op != NNCB_EW_STORE && op != NNCB_EW_REDUCE_STATS && op != NNCB_EW_REDUCE_SUM &&
           op != NNCB_EW_REDUCE_BN_GRAD;
}

// Channel-stationary programs: a per-channel variance read only as the `v`
// operand of inference BatchNorms (one eps) is turned into invstd once, in the
// prologue, with the very expression bn_infer_ evaluates per element, and
// those BatchNorms become bn_apply_ (bitwise the same result, one double
// sqrt + divide per thread instead of per element). Conservative: any other
// use or redefinition of the register keeps the per-element form.
// Returns: instruction index -> pre-inverted; fills reg -> eps.
std::vector<char> hoisted_invstd(const nncb_ew_program& p, std::map<int, double>& regs) {
    std::vector<char> flag(p.n_instr, 0);
    for (int k = 0; k < p.n_instr; ++k) {
        if (p.instr[k].op != NNCB_EW_LOAD_CH) continue;
        const int r = p.instr[k].dst;
        bool ok = true, seen = false;
        double eps = 0;
        std::vector<int> users;
        for (int q = 0; q < p.n_instr && ok; ++q) {
            if (q == k) continue;
            const nncb_ew_instr& in = p.instr[q];
            if (writes_reg(in.op) && in.dst == r) { ok = false; break; }
            const bool as_var = in.op == NNCB_EW_BN_INFER && in.c == r && in.a != r && in.b != r && in.d != r &&
                                in.e != r;
            if (as_var) {
                if (seen && in.imm != eps) ok = false;
                eps = in.imm, seen = true;
                users.push_back(q);
            } else if (in.a == r || in.b == r || in.c == r || in.d == r || in.e == r || in.f == r || in.h == r) {
                ok = false;
            }
        }
        if (!ok || !seen) continue;
        regs[r] = eps;
        for (int q : users) flag[q] = 1;
    }
    return flag;
}

// Emits the body for W lanes (W = 4: float4 path, W = 1: scalar tail).
void emit_body(std::ostringstream& os, const nncb_ew_program& p, int W, bool uses_ch, bool stationary = false,
               bool ring = false) {
    int reduce_index = 0, load_index = 0;
    std::map<int, double> inv_regs;
    const std::vector<char> pre_inverted = stationary ? hoisted_invstd(p, inv_regs) : std::vector<char>(p.n_instr, 0);
    os << "  float ";
    for (int r = 0; r < p.n_regs; ++r) os << (r ? ", " : "") << reg(r) << "[" << W << "]";
    os << ";\n";
    if (uses_ch && !stationary) {
        os << "  int ch[" << W << "]; { i64 c0 = i % A.C; ch[0] = (int)c0;\n";
        for (int j = 1; j < W; ++j) os << "    ch[" << j << "] = ch[" << j - 1 << "] + 1 == (int)A.C ? 0 : ch[" << j - 1 << "] + 1;\n";
        os << "  }\n";
    }
    for (int k = 0; k < p.n_instr; ++k) {
        const nncb_ew_instr& in = p.instr[k];
        std::string d = reg(in.dst), a = reg(in.a), b = reg(in.b), c = reg(in.c), dd = reg(in.d), e = reg(in.e),
                    f = reg(in.f), h = reg(in.h);
        std::string ptr = "A.p[" + std::to_string(in.slot) + "]";
        switch (in.op) {
            case NNCB_EW_LOAD:
                if (ring) {   // staged by the cp.async ring (rs: this thread's slot of the stage)
                    os << "  { const float4 t = rs[" << 256 * load_index++ << "]; " << d << "[0]=t.x; " << d
                       << "[1]=t.y; " << d << "[2]=t.z; " << d << "[3]=t.w; }\n";
                } else if (W == 4)
                    os << "  { float4 t = __ldg(reinterpret_cast<const float4*>(" << ptr << " + i)); " << d
                       << "[0]=t.x; " << d << "[1]=t.y; " << d << "[2]=t.z; " << d << "[3]=t.w; }\n";
                else
                    os << "  " << d << "[0] = __ldg(" << ptr << " + i);\n";
                continue;
            case NNCB_EW_LOAD_CH:
                if (stationary)
                    os << "  #pragma unroll\n  for (int j = 0; j < " << W << "; ++j) " << d << "[j] = pc" << in.dst
                       << "[j];\n";
                else
                    os << "  #pragma unroll\n  for (int j = 0; j < " << W << "; ++j) " << d << "[j] = __ldg(" << ptr
                       << " + ch[j]);\n";
                continue;
            case NNCB_EW_REDUCE_STATS: {
                if (!stationary) continue;
                const std::string r0 = "red" + std::to_string(reduce_index) + "_0",
                                  r1 = "red" + std::to_string(reduce_index) + "_1";
                ++reduce_index;
                char eps[64];   // (in the source: the kernel cache is keyed by it)
                snprintf(eps, sizeof(eps), "%.17e", in.imm);
                os << "  /* stats eps " << eps << " */\n";
                os << "  #pragma unroll\n  for (int j = 0; j < " << W << "; ++j) { const double v = (double)" << a
                   << "[j]; " << r0 << "[j] += v; " << r1 << "[j] += v * v; }\n";
                continue;
            }
            case NNCB_EW_REDUCE_SUM: {
                if (!stationary) continue;
                const std::string r0 = "red" + std::to_string(reduce_index) + "_0";
                ++reduce_index;
                os << "  #pragma unroll\n  for (int j = 0; j < " << W << "; ++j) " << r0 << "[j] += (double)" << a
                   << "[j];\n";
                continue;
            }
            case NNCB_EW_REDUCE_BN_GRAD: {
                if (!stationary) continue;   // launch guarantees the channel-stationary path
                const std::string r0 = "red" + std::to_string(reduce_index) + "_0",
                                  r1 = "red" + std::to_string(reduce_index) + "_1";
                ++reduce_index;
                os << "  #pragma unroll\n  for (int j = 0; j < " << W << "; ++j) { const double xh = ((double)" << b
                   << "[j] - (double)" << c << "[j]) * (double)" << dd << "[j]; " << r0 << "[j] += (double)" << a
                   << "[j]; " << r1 << "[j] += (double)" << a << "[j] * xh; }\n";
                continue;
            }
            case NNCB_EW_STORE:
                if (W == 4)
                    os << "  *reinterpret_cast<float4*>(" << ptr << " + i) = make_float4(" << a << "[0], " << a
                       << "[1], " << a << "[2], " << a << "[3]);\n";
                else
                    os << "  " << ptr << "[i] = " << a << "[0];\n";
                continue;
            default: break;
        }
        std::string expr;
        switch (in.op) {
            case NNCB_EW_RELU: expr = "relu_(" + a + "[j])"; break;
            case NNCB_EW_RELU_GRAD: expr = "relu_grad_(" + a + "[j], " + b + "[j])"; break;
            case NNCB_EW_ADD: expr = "__fadd_rn(" + a + "[j], " + b + "[j])"; break;
            case NNCB_EW_MUL: expr = "__fmul_rn(" + a + "[j], " + b + "[j])"; break;
            case NNCB_EW_COPY: expr = a + "[j]"; break;
            case NNCB_EW_GELU: expr = "gelu_(" + a + "[j])"; break;
            case NNCB_EW_GELU_GRAD: expr = "gelu_grad_(" + a + "[j], " + b + "[j])"; break;
            case NNCB_EW_GELU_FAST: expr = "gelu_fast_(" + a + "[j])"; break;
            case NNCB_EW_GELU_GRAD_FAST: expr = "gelu_grad_fast_(" + a + "[j], " + b + "[j])"; break;
            case NNCB_EW_BN_APPLY:
                expr = "bn_apply_(" + a + "[j], " + b + "[j], " + c + "[j], " + dd + "[j], " + e + "[j])";
                break;
            case NNCB_EW_BN_INFER: {
                if (pre_inverted[k]) {   // c holds invstd (prologue, see hoisted_invstd)
                    expr = "bn_apply_(" + a + "[j], " + b + "[j], " + c + "[j], " + dd + "[j], " + e + "[j])";
                    break;
                }
                char eps[64];
                snprintf(eps, sizeof(eps), "%.17e", in.imm);
                expr = "bn_infer_(" + a + "[j], " + b + "[j], " + c + "[j], " + dd + "[j], " + e + "[j], " +
                       std::string(eps) + ")";
                break;
            }
            case NNCB_EW_BN_GRAD:
            case NNCB_EW_BN_GRAD_FAST: {
                char cnt[64];
                snprintf(cnt, sizeof(cnt), "%.9e", static_cast<double>(static_cast<float>(in.imm)));
                expr = std::string(in.op == NNCB_EW_BN_GRAD ? "bn_grad_(" : "bn_grad_fast_(") + a + "[j], " + b + "[j], " + c + "[j], " + dd + "[j], " + e + "[j], " + f +
                       "[j], " + h + "[j], (float)" + cnt + ")";
                break;
            }
            default: expr = "0.f /* unknown op */"; break;
        }
        os << "  #pragma unroll\n  for (int j = 0; j < " << W << "; ++j) " << d << "[j] = " << expr << ";\n";
    }
}

std::vector<int> find_reduces(const nncb_ew_program& p) {
    std::vector<int> r;
    for (int k = 0; k < p.n_instr; ++k)
        if (p.instr[k].op == NNCB_EW_REDUCE_BN_GRAD || p.instr[k].op == NNCB_EW_REDUCE_STATS ||
            p.instr[k].op == NNCB_EW_REDUCE_SUM)
            r.push_back(k);
    return r;
}

// resident blocks per SM the two-reduction build is register-budgeted for
// (NNCB_EW_RED2_BLOCKS; default 2)
int red2_blocks() {
    static const int b = getenv("NNCB_EW_RED2_BLOCKS") ? std::max(1, atoi(getenv("NNCB_EW_RED2_BLOCKS"))) : 2;
    return b;
}

// The channel-stationary loop stages the element-wise LOAD streams through a
// per-thread ring of cp.async (LDGSTS) copies in shared memory: the loads in
// flight no longer cost registers, so the register-heavy programs (many
// per-channel operands on the 2-block budget) keep several element vectors in
// flight per thread. Stages: as many as fit 48 KB per block (32 KB beside a
// reduction's 16 KB static buffer), 3..8; 0 = no ring (more than 4 streams, or
// NNCB_EW_RING=0). Each thread reads back only its own slots, so no block
// barrier is needed.
// Resident blocks per SM a program's register budget is built for (0: the
// compiler's default).
// * reductions carry 16 registers of double accumulators: 64 registers (four
//   blocks, one wave, see nncb_ew_launch); two reductions, or a statistics
//   pass with more than 4 per-channel operands (a recomputed BatchNorm chain),
//   get the 2-block budget (at 64 registers the depth-3 pass spilled and ran at
//   1.7 TB/s; 4.8 TB/s at 128)
// * programs with 3+ per-channel operands (BatchNorm apply / gradient) hold
//   them in registers on the channel-stationary path: 128 registers (2
//   blocks). Before the load ring, 64 registers (4 blocks) were needed to keep
//   enough loads in flight (5.1 -> 6.1 TB/s for the BN input gradient); with
//   the ring the 2-block budget measured +1% on the C4 step. More than 8
//   per-channel operands (a chain of BatchNorms: the C2 apply pass) take the
//   whole register file (C2 mode B +1.5%; C3/C4/C5 have none).
//   NNCB_EW_MINBLOCKS overrides.
int resident_blocks(const nncb_ew_program& p) {
    int nch = 0;
    bool stats_red = false;
    for (int k = 0; k < p.n_instr; ++k) {
        nch += p.instr[k].op == NNCB_EW_LOAD_CH;
        stats_red = stats_red || p.instr[k].op == NNCB_EW_REDUCE_STATS;
    }
    const size_t nred = find_reduces(p).size();
    // (with the load ring, every reduction group runs best at 2 blocks per SM
    // with 128 registers: tools/ew_bench.py relu-grad + reduction 5-15% faster
    // than 4 blocks at 64 registers; NNCB_EW_RED1_BLOCKS=4 restores that)
    static const int red1 = getenv("NNCB_EW_RED1_BLOCKS") ? atoi(getenv("NNCB_EW_RED1_BLOCKS")) : 2;
    if (nred > 0) return nred > 1 || (stats_red && nch > 4) ? red2_blocks() : red1;
    static const int env_min_blocks = getenv("NNCB_EW_MINBLOCKS") ? atoi(getenv("NNCB_EW_MINBLOCKS")) : -1;
    if (env_min_blocks >= 0) return env_min_blocks;
    return nch > 8 ? 1 : nch >= 3 ? 2 : 0;
}

int ring_stages(const nncb_ew_program& p) {
    static const int env = getenv("NNCB_EW_RING") ? atoi(getenv("NNCB_EW_RING")) : -1;
    if (env == 0) return 0;
    int nl = 0;
    for (int k = 0; k < p.n_instr; ++k) nl += p.instr[k].op == NNCB_EW_LOAD;
    if (nl == 0) return 0;
    // shared memory per block: 48 KB; 100 KB (opt-in size) for the gradient
    // reductions on the 2-block budget (+1% on C4 for the residual join's
    // two-reduction group, 5-15% on the relu-grad + reduction microbenchmark;
    // the C2 statistics passes measured 3% slower with it). A reduction's 16 KB
    // of per-thread partials reuse the ring after the loop. NNCB_EW_RING_KB2
    // overrides the size for every 2-block program.
    static const int kb2 = getenv("NNCB_EW_RING_KB2") ? atoi(getenv("NNCB_EW_RING_KB2")) : 0;
    bool stats = false;
    for (int k = 0; k < p.n_instr; ++k) stats = stats || p.instr[k].op == NNCB_EW_REDUCE_STATS;
    const bool wide = resident_blocks(p) == 2 && (kb2 > 0 || (!stats && !find_reduces(p).empty()));
    static const int kbr = getenv("NNCB_EW_RING_KBR") ? atoi(getenv("NNCB_EW_RING_KBR")) : 48;
    const int kb = wide ? (kb2 > 0 ? kb2 : 100) : find_reduces(p).empty() ? 48 : kbr;
    const int budget = kb / 4;   // stage-streams of 4 KB
    int S = std::min(8, budget / nl);
    if (env > 0) S = std::min(S, env);
    return S >= 3 ? S : 0;
}

int load_streams(const nncb_ew_program& p) {
    int nl = 0;
    for (int k = 0; k < p.n_instr; ++k) nl += p.instr[k].op == NNCB_EW_LOAD;
    return nl;
}

std::string generate(const nncb_ew_program& p, bool uses_ch) {
    std::ostringstream os;
    const int nred = static_cast<int>(find_reduces(p).size());
    const bool red = nred > 0;
    os << kPrelude;
    os << "__device__ __forceinline__ void body4(const EwArgs& A, i64 i) {\n";
    emit_body(os, p, 4, uses_ch);
    os << "}\n__device__ __forceinline__ void body1(const EwArgs& A, i64 i) {\n";
    emit_body(os, p, 1, uses_ch);
    os << "}\n";
    std::vector<int> chregs;
    for (int k = 0; k < p.n_instr; ++k)
        if (p.instr[k].op == NNCB_EW_LOAD_CH) chregs.push_back(k);
    if (uses_ch) {
        // channel-stationary body: the host picks a grid whose element stride is a
        // multiple of C, so a thread's 4 channels never change; per-channel
        // operands are loaded once (float4) into registers before the loop.
        os << "__device__ __forceinline__ void body4s(const EwArgs& A, i64 i";
        if (ring_stages(p)) os << ", const float4* rs";
        for (int k : chregs) os << ", const float (&pc" << p.instr[k].dst << ")[4]";
        for (int q = 0; q < nred; ++q) os << ", double (&red" << q << "_0)[4], double (&red" << q << "_1)[4]";
        os << ") {\n";
        emit_body(os, p, 4, uses_ch, true, ring_stages(p) > 0);
        os << "}\n";
    }
    if (const int blocks = resident_blocks(p))
        os << "extern \"C\" __global__ void __launch_bounds__(256, " << blocks << ") nnc_fused_ew(const EwArgs A) {";
    else
        os << "extern \"C\" __global__ void __launch_bounds__(256) nnc_fused_ew(const EwArgs A) {";
    bool stats_red = false;
    for (int k = 0; k < p.n_instr; ++k) stats_red = stats_red || p.instr[k].op == NNCB_EW_REDUCE_STATS;
    // reduction groups: the finalize kernel is a programmatic dependent
    // launch; let it be scheduled while this grid drains (it waits on
    // griddepcontrol.wait for this grid's completion and memory)
    if (red) os << "\n  asm volatile(\"griddepcontrol.launch_dependents;\");";
    os << R"(
  const i64 nvec = A.n >> 2;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  i64 v = (i64)blockIdx.x * blockDim.x + threadIdx.x;
)";
    if (uses_ch) {
        os << "  if (A.cs) {\n    const int c0 = (int)((v << 2) % A.C);\n";
        for (int k : chregs) {
            const nncb_ew_instr& in = p.instr[k];
            os << "    float pc" << in.dst << "[4]; { float4 t = __ldg(reinterpret_cast<const float4*>(A.p[" << in.slot
               << "] + c0)); pc" << in.dst << "[0]=t.x; pc" << in.dst << "[1]=t.y; pc" << in.dst << "[2]=t.z; pc"
               << in.dst << "[3]=t.w; }\n";
        }
        std::map<int, double> inv_regs;
        hoisted_invstd(p, inv_regs);
        for (const auto& [r, e] : inv_regs) {
            char eps[64];
            snprintf(eps, sizeof(eps), "%.17e", e);
            os << "    #pragma unroll\n    for (int j = 0; j < 4; ++j) pc" << r << "[j] = (float)(1.0 / sqrt((double)pc" << r
               << "[j] + " << eps << "));\n";
        }
        std::string args;
        for (int k : chregs) args += ", pc" + std::to_string(p.instr[k].dst);
        for (int q = 0; q < nred; ++q) {
            args += ", red" + std::to_string(q) + "_0, red" + std::to_string(q) + "_1";
            os << "    double red" << q << "_0[4] = {0, 0, 0, 0}, red" << q << "_1[4] = {0, 0, 0, 0};\n";
        }
        // A statistics pass on the 2-block budget (a recomputed BatchNorm
        // chain) runs at 16 warps per SM: four element vectors per iteration
        // put twice the loads in flight at the same occupancy, same
        // accumulation order (C2 mode B 5.57 -> 6.05 TB/s; the same unroll on
        // the apply passes measured neutral on C4 and 25% slower on C2 mode A).
        // NNCB_EW_UNROLL=2|4 overrides.
        static const int env_unroll = getenv("NNCB_EW_UNROLL") ? atoi(getenv("NNCB_EW_UNROLL")) : 0;
        const int unroll = env_unroll == 2 || env_unroll == 4 ? env_unroll
                         : red && stats_red && chregs.size() > 4 ? 4 : 2;
        if (const int S = ring_stages(p)) {
            const int NL = load_streams(p);
            std::vector<int> lslots;
            for (int k = 0; k < p.n_instr; ++k)
                if (p.instr[k].op == NNCB_EW_LOAD) lslots.push_back(p.instr[k].slot);
            os << "    extern __shared__ float4 ring[];   // [" << S << " stages][" << NL << " streams][256 threads]\n"
               << "    const unsigned rbase = (unsigned)__cvta_generic_to_shared(ring + threadIdx.x);\n"
               << "    auto issue = [&](i64 w, int st) {\n      if (w < nvec) {\n";
            for (int q = 0; q < NL; ++q)
                os << "        asm volatile(\"cp.async.cg.shared.global [%0], [%1], 16;\" :: \"r\"(rbase + (unsigned)((st * "
                   << NL << " + " << q << ") * 4096)), \"l\"(A.p[" << lslots[q] << "] + (w << 2)) : \"memory\");\n";
            os << "      }\n      asm volatile(\"cp.async.commit_group;\" ::: \"memory\");\n    };\n";
            os << "    #pragma unroll\n    for (int st = 0; st < " << S << "; ++st) issue(v + st * stride, st);\n";
            os << "    for (int st = 0; v < nvec; v += stride) {\n"
               << "      asm volatile(\"cp.async.wait_group " << S - 1 << ";\" ::: \"memory\");\n"
               << "      body4s(A, v << 2, ring + st * " << NL * 256 << " + threadIdx.x" << args << ");\n"
               << "      issue(v + " << S << " * stride, st);\n"
               << "      st = st + 1 == " << S << " ? 0 : st + 1;\n    }\n"
               << "    asm volatile(\"cp.async.wait_all;\" ::: \"memory\");\n";
        } else {
        if (unroll == 4)
            os << "    for (; v + 3 * stride < nvec; v += 4 * stride) { body4s(A, v << 2" << args
               << "); body4s(A, (v + stride) << 2" << args << "); body4s(A, (v + 2 * stride) << 2" << args
               << "); body4s(A, (v + 3 * stride) << 2" << args << "); }\n";
        os << "    for (; v + stride < nvec; v += 2 * stride) { body4s(A, v << 2" << args << "); body4s(A, (v + stride) << 2"
           << args << "); }\n";
        os << "    if (v < nvec) body4s(A, v << 2" << args << ");\n";
        }
        if (red) {
            // Per-block partials, deterministic: for C <= 1024 (a power of two)
            // threads t and t + C/4 share channels and thread q < C/4 folds its
            // group in t order; for C > 1024 each thread owns its 4 channels.
            // Reduction q writes the slice A.part + q * gridDim.x * 2C.
            // (with a load ring, the partials reuse its shared memory once every
            // thread has left the loop)
            if (ring_stages(p))
                os << "    __syncthreads();\n    double (*rs)[8] = reinterpret_cast<double (*)[8]>(ring);\n";
            else
                os << "    __shared__ double rs[256][8];\n";
            os << "    const int t = threadIdx.x;\n    const int C = (int)A.C;\n";
            for (int q = 0; q < nred; ++q) {
                const std::string r0 = "red" + std::to_string(q) + "_0", r1 = "red" + std::to_string(q) + "_1";
                os << "    {\n    if (" << q << " > 0) __syncthreads();\n"
                   << "    #pragma unroll\n    for (int j = 0; j < 4; ++j) { rs[t][j] = " << r0 << "[j]; rs[t][4 + j] = "
                   << r1 << "[j]; }\n    __syncthreads();\n"
                   << "    double* part = A.part + ((i64)" << q << " * gridDim.x + blockIdx.x) * 2 * C;\n"
                   << R"(    if (C <= 1024) {
      const int G = C >> 2;
      if (t < G) {
        double a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int k = t; k < 256; k += G) {
          #pragma unroll
          for (int j = 0; j < 8; ++j) a[j] += rs[k][j];
        }
        #pragma unroll
        for (int j = 0; j < 4; ++j) { part[4 * t + j] = a[j]; part[C + 4 * t + j] = a[4 + j]; }
      }
    } else {
      #pragma unroll
)" << "      for (int j = 0; j < 4; ++j) { part[c0 + j] = " << r0 << "[j]; part[C + c0 + j] = " << r1 << "[j]; }\n    }\n    }\n";
            }
        }
        os << "    return;\n  }\n";
    }
    os << R"(  for (; v + stride < nvec; v += 2 * stride) { body4(A, v << 2); body4(A, (v + stride) << 2); }
  if (v < nvec) body4(A, v << 2);
  for (i64 i = (nvec << 2) + (i64)blockIdx.x * blockDim.x + threadIdx.x; i < A.n; i += stride) body1(A, i);
}
)";
    // NNCB_EW_DUMP=dir: write every generated program to dir/ew_<hash>.cu
    if (const char* dir = getenv("NNCB_EW_DUMP")) {
        const std::string src = os.str();
        char path[512];
        snprintf(path, sizeof(path), "%s/ew_%016zx.cu", dir, std::hash<std::string>{}(src));
        if (FILE* f = fopen(path, "w")) fputs(src.c_str(), f), fclose(f);
    }
    return os.str();
}

int nvrtc_fail(nvrtcProgram prog, nvrtcResult r, const std::string& src) {
    std::string log;
    size_t n = 0;
    if (prog && nvrtcGetProgramLogSize(prog, &n) == NVRTC_SUCCESS && n > 1) {
        log.resize(n);
        nvrtcGetProgramLog(prog, log.data());
    }
    if (prog) nvrtcDestroyProgram(&prog);
    return nncb::fail(std::string("NVRTC: ") + nvrtcGetErrorString(r) + "\n" + log + "\n--- source ---\n" + src);
}

// Folds the per-block partials of a REDUCE_BN_GRAD group: a block of 1024
// threads owns 8 channels; lane row y (0..127) sums the main kernel's blocks
// k = y, y+128, ... and the 128 rows are folded by a fixed tree
// (deterministic). For C > 1024 main-kernel block k only covers the channels
// [(1024 k) % C, +1024).
__global__ void __launch_bounds__(1024) ew_red_final_k(const double* __restrict__ part, int grid, int C,
                                                       float* __restrict__ sg, float* __restrict__ sgx,
                                                       int stats, double rows, double eps) {
    __shared__ double fold[2][128][8];
    // programmatic dependent launch: the reducing grid's partials are
    // complete and visible past this point
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int tx = threadIdx.x % 8, ty = threadIdx.x / 8;
    const int c = blockIdx.x * 8 + tx;
    double a = 0.0, b = 0.0;
    if (c < C) {
#pragma unroll 2
        for (int k = ty; k < grid; k += 128) {
            if (C > 1024) {
                const int start = static_cast<int>((static_cast<long long>(k) * 1024) % C);
                if ((c - start + C) % C >= 1024) continue;
            }
            a += part[(static_cast<long long>(k) * 2) * C + c];
            b += part[(static_cast<long long>(k) * 2 + 1) * C + c];
        }
    }
    fold[0][ty][tx] = a;
    fold[1][ty][tx] = b;
    __syncthreads();
    for (int h = 64; h >= 1; h >>= 1) {
        if (ty < h) {
            fold[0][ty][tx] += fold[0][ty + h][tx];
            fold[1][ty][tx] += fold[1][ty + h][tx];
        }
        __syncthreads();
    }
    if (ty == 0 && c < C) {
        if (stats == 1) {   // REDUCE_STATS: BatchNorm mean and 1/sqrt(biased var + eps), from the double sums
            const double mean = fold[0][0][tx] / rows;
            double var = fold[1][0][tx] / rows - mean * mean;
            if (var < 0) var = 0;
            sg[c] = static_cast<float>(mean);
            sgx[c] = static_cast<float>(1.0 / sqrt(var + eps));
        } else {
            sg[c] = static_cast<float>(fold[0][0][tx]);
            if (sgx) sgx[c] = static_cast<float>(fold[1][0][tx]);   // null: REDUCE_SUM
        }
    }
}

}  // namespace

extern "C" {

int nncb_ew_compile_check(const nncb_ew_program* p) {
    if (p->n_slots > kMaxSlots) return nncb::fail("nncb_ew_compile_check: too many slots");
    bool uses_ch = false;
    for (int k = 0; k < p->n_instr; ++k)   // reductions run channel-stationary too
        uses_ch = uses_ch || p->instr[k].op == NNCB_EW_LOAD_CH || p->instr[k].op == NNCB_EW_REDUCE_STATS ||
                  p->instr[k].op == NNCB_EW_REDUCE_BN_GRAD || p->instr[k].op == NNCB_EW_REDUCE_SUM;
    std::string src = generate(*p, uses_ch);
    static std::mutex mu;
    static std::set<std::string> checked;
    {
        std::lock_guard<std::mutex> lock(mu);
        if (checked.count(src)) return 0;
    }
    nvrtcProgram prog = nullptr;
    nvrtcResult r = nvrtcCreateProgram(&prog, src.c_str(), "nnc_fused_ew.cu", 0, nullptr, nullptr);
    if (r != NVRTC_SUCCESS) return nvrtc_fail(prog, r, src);
    const char* opts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "-lineinfo", "--fmad=false"};
    r = nvrtcCompileProgram(prog, 4, opts);
    if (r != NVRTC_SUCCESS) return nvrtc_fail(prog, r, src);
    nvrtcDestroyProgram(&prog);
    std::lock_guard<std::mutex> lock(mu);
    checked.insert(src);
    return 0;
}

int nncb_ew_compile(nncb_ctx* ctx, const nncb_ew_program* p, nncb_ew_kernel** out) {
    if (p->n_slots > kMaxSlots) return nncb::fail("nncb_ew_compile: too many slots");
    bool uses_ch = false;
    for (int k = 0; k < p->n_instr; ++k)   // reductions run channel-stationary too
        uses_ch = uses_ch || p->instr[k].op == NNCB_EW_LOAD_CH || p->instr[k].op == NNCB_EW_REDUCE_STATS ||
                  p->instr[k].op == NNCB_EW_REDUCE_BN_GRAD || p->instr[k].op == NNCB_EW_REDUCE_SUM;
    std::string src = generate(*p, uses_ch);
    auto hit = ctx->ew_cache.find(src);
    if (hit != ctx->ew_cache.end()) {
        *out = hit->second;
        return 0;
    }
    NNCB_CUDA(cudaSetDevice(ctx->device));
    NNCB_CUDA(cudaFree(nullptr));  // make the primary context current for the driver API
    nvrtcProgram prog = nullptr;
    nvrtcResult r = nvrtcCreateProgram(&prog, src.c_str(), "nnc_fused_ew.cu", 0, nullptr, nullptr);
    if (r != NVRTC_SUCCESS) return nvrtc_fail(prog, r, src);
    const char* opts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "-lineinfo", "--fmad=false"};
    r = nvrtcCompileProgram(prog, 4, opts);
    if (r != NVRTC_SUCCESS) return nvrtc_fail(prog, r, src);
    size_t cubin_size = 0;
    r = nvrtcGetCUBINSize(prog, &cubin_size);
    if (r != NVRTC_SUCCESS) return nvrtc_fail(prog, r, src);
    std::vector<char> cubin(cubin_size);
    r = nvrtcGetCUBIN(prog, cubin.data());
    if (r != NVRTC_SUCCESS) return nvrtc_fail(prog, r, src);
    nvrtcDestroyProgram(&prog);
    auto* k = new nncb_ew_kernel;
    k->source = src;
    k->n_slots = p->n_slots;
    k->uses_channels = uses_ch;
    const bool reds_empty = find_reduces(*p).empty();
    k->red_blocks = reds_empty ? 4 : resident_blocks(*p);
    if (uses_ch && ring_stages(*p)) {
        k->ring_bytes = ring_stages(*p) * load_streams(*p) * 4096;
        if (!reds_empty) k->ring_bytes = std::max(k->ring_bytes, 256 * 8 * 8);   // the partials' reuse
    }
    const std::vector<int> reds = find_reduces(*p);
    if (reds.size() > 2) {
        nncb::ew_release(k);
        return nncb::fail("nncb_ew_compile: at most two REDUCE_BN_GRAD per program");
    }
    for (int r : reds) {
        k->reduce_sg[k->n_reduce] = p->instr[r].slot;
        k->reduce_sgx[k->n_reduce] = p->instr[r].e;
        k->reduce_stats[k->n_reduce] =
            p->instr[r].op == NNCB_EW_REDUCE_STATS ? 1 : p->instr[r].op == NNCB_EW_REDUCE_SUM ? 2 : 0;
        k->reduce_eps[k->n_reduce] = p->instr[r].imm;
        ++k->n_reduce;
    }
    const auto& D = nncb::drv::table();
    if (!D.ok) {
        nncb::ew_release(k);
        return nncb::fail("CUDA driver entry points unavailable");
    }
    CUresult cr = D.moduleLoadData(&k->module, cubin.data());
    if (cr == CUDA_SUCCESS) cr = D.moduleGetFunction(&k->fn, k->module, "nnc_fused_ew");
    if (cr == CUDA_SUCCESS && k->ring_bytes > 48 * 1024)
        cr = D.funcSetAttribute(k->fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, k->ring_bytes);
    if (cr != CUDA_SUCCESS) {
        nncb::ew_release(k);
        return nncb::fail(std::string("cuModuleLoadData: ") + nncb::drv::error_string(cr));
    }
    ctx->ew_cache[src] = k;
    *out = k;
    return 0;
}

int nncb_ew_launch(nncb_ctx* ctx, nncb_ew_kernel* k, void* const* slots, int64_t n, int64_t channels) {
    if (n <= 0) return 0;
    struct {
        float* p[kMaxSlots];
        long long n;
        long long C;
        int cs;
        double* part;
    } args{};
    for (int s = 0; s < k->n_slots; ++s) {
        args.p[s] = static_cast<float*>(slots[s]);
        if (reinterpret_cast<uintptr_t>(slots[s]) == 0) return nncb::fail("nncb_ew_launch: null slot");
    }
    args.n = n;
    args.C = channels > 0 ? channels : 1;
    if (k->uses_channels && channels <= 0) return nncb::fail("nncb_ew_launch: per-channel program needs C");
    int64_t nvec = (n + 3) / 4;
    unsigned grid = nncb::grid_for(ctx, (nvec + 1) / 2, 256, 8);
    if (k->uses_channels && channels % 4 == 0 && n % 4 == 0) {
        // channel-stationary launch: (grid * 256 * 4) % C == 0 and every per-channel
        // pointer 16-byte aligned (offsets are multiples of C, C % 4 == 0)
        int64_t g = channels / std::gcd<int64_t>(channels, 1024);
        if (g <= grid) {
            grid = static_cast<unsigned>((grid / g) * g);
            args.cs = 1;
            for (int s2 = 0; s2 < k->n_slots; ++s2)
                if (reinterpret_cast<uintptr_t>(slots[s2]) & 15) args.cs = 0;
        }
    }
    static const bool dbg = getenv("NNCB_EW_DEBUG") != nullptr;
    if (dbg)
        fprintf(stderr, "[nncb ew] n=%lld C=%lld uses_ch=%d cs=%d grid=%u slots=%d\n", (long long)n,
                (long long)channels, (int)k->uses_channels, args.cs, grid, k->n_slots);
    const bool reduce = k->n_reduce > 0;
    if (reduce) {
        // the reduction runs only on the channel-stationary path: C a power of
        // two in [4, 2048]; a bounded grid keeps the per-block partials small
        const int64_t C = channels;
        if (!args.cs || C < 4 || C > 8192 || (C & (C - 1)))
            return nncb::fail("nncb_ew_launch: a reduction needs the channel-stationary launch (C power of 2 <= 8192)");
        const int64_t g = C / std::gcd<int64_t>(C, 1024);
        // two blocks per SM: with the load ring keeping the loads in flight,
        // fewer blocks mean fewer per-block partials to write and fold
        // (tools/ew_bench.py relu-grad + reduction: 2 blocks 1-10% faster than
        // 4 from 12544x512 to 200704x128; C4 neutral, C2 statistics +1%)
        static const int64_t per_sm = getenv("NNCB_EW_RED_BLOCKS") ? std::max(1, atoi(getenv("NNCB_EW_RED_BLOCKS"))) : 2;
        // one wave: the two-reduction build is budgeted for red2_blocks() per SM
        const int64_t resident = std::min<int64_t>(per_sm, k->red_blocks);
        const int64_t cap = std::max<int64_t>(g, (resident * static_cast<int64_t>(ctx->sm_count) / g) * g);
        if (grid > cap) grid = static_cast<unsigned>(cap);
        args.part = static_cast<double*>(nncb::scratch(ctx, sizeof(double) * 2 * C * grid * k->n_reduce));
        if (!args.part) return nncb::fail("nncb_ew_launch: reduction scratch allocation failed");
    }
    void* params[] = {&args};
    CUresult r = nncb::drv::table().launchKernel(k->fn, grid, 1, 1, 256, 1, 1, args.cs ? k->ring_bytes : 0,
                                                 reinterpret_cast<CUstream>(ctx->stream), params, nullptr);
    if (r != CUDA_SUCCESS)
        return nncb::fail(std::string("cuLaunchKernel(fused ew): ") + nncb::drv::error_string(r));
    ctx->launches.fetch_add(1, std::memory_order_relaxed);
    if (reduce) {
        const int C = static_cast<int>(channels);
        for (int q = 0; q < k->n_reduce; ++q) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(static_cast<unsigned>((C + 7) / 8));
            cfg.blockDim = dim3(1024);
            cfg.stream = ctx->stream;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = q == 0 ? 1 : 0;   // the first follows the reducing grid
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            float* o0 = args.p[k->reduce_sg[q]];
            float* o1 = k->reduce_stats[q] == 1 ? o0 + C : k->reduce_stats[q] == 2 ? nullptr : args.p[k->reduce_sgx[q]];
            NNCB_CUDA(cudaLaunchKernelEx(&cfg, ew_red_final_k, static_cast<const double*>(args.part + static_cast<size_t>(q) * grid * 2 * C),
                                         static_cast<int>(grid), C, o0, o1, k->reduce_stats[q],
                                         static_cast<double>(n / C), k->reduce_eps[q]));
            ctx->launches.fetch_add(1, std::memory_order_relaxed);
        }
    }
    return 0;
}

const char* nncb_ew_source(nncb_ew_kernel* k) { return k ? k->source.c_str() : ""; }

}  // extern "C"
