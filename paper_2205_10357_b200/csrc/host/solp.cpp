// solp.cpp -- SOLP plan serialization carrying the B200 launch descriptors.
//
// Mirrors the reference's plan format API (plan.hpp:154-160, plan.cpp:633-848):
// a deterministic little-endian byte stream with a magic, a version, and every
// field of the compiled plan, so that optimize/deploy -> run/exec round-trips
// bitwise (reference test_backends.cpp:308-333, acceptance.cpp:601-622). Beyond
// the reference's fields it carries each group's device launches: launch kind,
// argument slots and offsets, the fused-group register program, and the
// originating op with its attributes. The process-unique plan uid is not
// serialized (a loaded plan gets a fresh one). Truncated or foreign streams
// throw nnc::Error(BadDocument).
#include <algorithm>
#include <cstring>
#include <fstream>
#include <iterator>

#include "nnc/error.hpp"
#include "nnc/plan.hpp"

namespace nnc::plan {

namespace {

constexpr char kMagic[4] = {'S', 'O', 'L', 'P'};
constexpr char kSetMagic[4] = {'S', 'O', 'L', 'V'};
constexpr uint32_t kVersion = 0xB2000002u;   // B200 descriptor layout, revision 2 (per-launch GEMM tile)

struct Writer {
    std::vector<uint8_t> out;
    void raw(const void* p, size_t n) {
        const auto* b = static_cast<const uint8_t*>(p);
        out.insert(out.end(), b, b + n);
    }
    template <typename T>
    void le(T v) {   // explicit little-endian, independent of the host
        for (size_t i = 0; i < sizeof(T); ++i) out.push_back(static_cast<uint8_t>((static_cast<uint64_t>(v) >> (8 * i)) & 0xff));
    }
    void u8(uint8_t v) { out.push_back(v); }
    void u32(uint32_t v) { le(v); }
    void i32(int32_t v) { le(static_cast<uint32_t>(v)); }
    void u64(uint64_t v) { le(v); }
    void i64(int64_t v) { le(static_cast<uint64_t>(v)); }
    void f64(double v) {
        uint64_t bits;
        std::memcpy(&bits, &v, 8);
        le(bits);
    }
    void str(const std::string& s) {
        u32(static_cast<uint32_t>(s.size()));
        raw(s.data(), s.size());
    }
};

struct Reader {
    const std::vector<uint8_t>& in;
    size_t pos = 0;
    void need(size_t n) {
        if (pos + n > in.size()) throw Error(Error::Code::BadDocument, "SOLP: truncated plan stream");
    }
    template <typename T>
    T le() {
        need(sizeof(T));
        uint64_t v = 0;
        for (size_t i = 0; i < sizeof(T); ++i) v |= static_cast<uint64_t>(in[pos + i]) << (8 * i);
        pos += sizeof(T);
        return static_cast<T>(v);
    }
    uint8_t u8() { return le<uint8_t>(); }
    uint32_t u32() { return le<uint32_t>(); }
    int32_t i32() { return static_cast<int32_t>(le<uint32_t>()); }
    uint64_t u64() { return le<uint64_t>(); }
    int64_t i64() { return static_cast<int64_t>(le<uint64_t>()); }
    double f64() {
        uint64_t bits = le<uint64_t>();
        double v;
        std::memcpy(&v, &bits, 8);
        return v;
    }
    std::string str() {
        uint32_t n = u32();
        need(n);
        std::string s(reinterpret_cast<const char*>(in.data() + pos), n);
        pos += n;
        return s;
    }
    uint32_t count(size_t min_item_bytes = 1) {   // a length that the remaining bytes can hold
        uint32_t n = u32();
        if (static_cast<uint64_t>(n) * min_item_bytes > in.size() - pos)
            throw Error(Error::Code::BadDocument, "SOLP: corrupt length field");
        return n;
    }
};

void write_attrs(Writer& w, const hlir::Attrs& a) {
    w.i64(a.out_channels);
    w.i64(a.kernel[0]);
    w.i64(a.kernel[1]);
    w.i64(a.stride[0]);
    w.i64(a.stride[1]);
    w.u8(static_cast<uint8_t>(a.padding));
    w.u8(a.has_bias ? 1 : 0);
    w.i64(a.out_hw[0]);
    w.i64(a.out_hw[1]);
    w.i64(a.out_features);
    w.i64(a.axis);
    w.u8(a.exclusive ? 1 : 0);
    w.u8(a.reverse ? 1 : 0);
    w.u32(static_cast<uint32_t>(a.fwd_dims.size()));
    for (int64_t d : a.fwd_dims) w.i64(d);
    w.f64(a.eps);
    w.u8(a.inference ? 1 : 0);
}

hlir::Attrs read_attrs(Reader& r) {
    hlir::Attrs a;
    a.out_channels = r.i64();
    a.kernel[0] = r.i64();
    a.kernel[1] = r.i64();
    a.stride[0] = r.i64();
    a.stride[1] = r.i64();
    a.padding = static_cast<hlir::Padding>(r.u8());
    a.has_bias = r.u8() != 0;
    a.out_hw[0] = r.i64();
    a.out_hw[1] = r.i64();
    a.out_features = r.i64();
    a.axis = r.i64();
    a.exclusive = r.u8() != 0;
    a.reverse = r.u8() != 0;
    uint32_t n = r.count(8);
    for (uint32_t i = 0; i < n; ++i) a.fwd_dims.push_back(r.i64());
    a.eps = r.f64();
    a.inference = r.u8() != 0;
    return a;
}

void write_plan(Writer& w, const ExecutionPlan& p) {
    w.raw(kMagic, 4);
    w.u32(kVersion);
    w.u8(static_cast<uint8_t>(p.dtype));
    w.u8(static_cast<uint8_t>(p.role));
    w.u32(static_cast<uint32_t>(p.values.size()));
    for (const ValueEntry& e : p.values) {
        w.str(e.name);
        w.u8(static_cast<uint8_t>(e.category));
        w.u8(static_cast<uint8_t>(e.storage));
        w.u8(e.resident ? 1 : 0);
        w.str(e.source_weight);
        w.u32(static_cast<uint32_t>(e.dims.size()));
        for (int64_t d : e.dims) w.i64(d);
    }
    w.u32(static_cast<uint32_t>(p.groups.size()));
    for (const GroupKernel& gk : p.groups) {
        w.u32(gk.id);
        w.u8(static_cast<uint8_t>(gk.backend));
        w.str(gk.label);
        w.u32(static_cast<uint32_t>(gk.members.size()));
        for (const std::string& m : gk.members) w.str(m);
        w.u32(static_cast<uint32_t>(gk.launches.size()));
        for (const Launch& L : gk.launches) {
            w.u8(static_cast<uint8_t>(L.kind));
            w.str(L.label);
            w.u32(static_cast<uint32_t>(L.args.size()));
            for (size_t i = 0; i < L.args.size(); ++i) {
                w.u32(L.args[i].slot);
                w.i64(L.args[i].offset);
                w.u8(L.is_out[i] ? 1 : 0);
            }
            w.u32(static_cast<uint32_t>(L.ew.size()));
            for (const nncb_ew_instr& in : L.ew) {
                for (int32_t v : {in.op, in.dst, in.a, in.b, in.c, in.d, in.e, in.f, in.h, in.slot}) w.i32(v);
                w.f64(in.imm);
            }
            w.i32(L.ew_regs);
            w.u32(L.elem_slot);
            w.u32(static_cast<uint32_t>(L.op));
            write_attrs(w, L.attrs);
            w.u8(L.relu_epilogue ? 1 : 0);
            w.i32(L.tile);
        }
    }
    w.u32(static_cast<uint32_t>(p.exec_steps.size()));
    for (const ExecStep& es : p.exec_steps) {
        w.u32(es.group);
        w.i32(es.kernel);
        w.str(es.label);
        w.u32(static_cast<uint32_t>(es.launches.size()));
        for (uint32_t l : es.launches) w.u32(l);
    }
    w.u32(static_cast<uint32_t>(p.events.size()));
    for (const PlanEvent& e : p.events) {
        w.i32(e.step);
        w.u8(e.alloc ? 1 : 0);
        w.u32(e.slot);
    }
    w.u32(static_cast<uint32_t>(p.input_slots.size()));
    for (uint32_t s : p.input_slots) w.u32(s);
    w.u32(static_cast<uint32_t>(p.output_slots.size()));
    for (uint32_t s : p.output_slots) w.u32(s);
    w.u32(static_cast<uint32_t>(p.weight_names.size()));
    for (const std::string& n : p.weight_names) w.str(n);
}

/// Semantic validation of a decoded plan: every enum in range, every slot,
/// register, element offset and schedule index inside what it indexes. A
/// well-formed but inconsistent stream must be rejected here -- the runtime
/// turns these fields into device pointer arithmetic and generated kernels.
void validate_plan(const ExecutionPlan& p) {
    auto bad = [](const std::string& what) { throw Error(Error::Code::BadDocument, "SOLP: " + what); };
    if (p.dtype != DType::F32 && p.dtype != DType::F64) bad("dtype out of range");
    if (static_cast<unsigned>(p.role) > static_cast<unsigned>(PlanRole::TrainBwd)) bad("role out of range");
    // names are printable ASCII identifiers (DLB documents); anything else is corruption
    auto name_ok = [&](const std::string& n) {
        for (unsigned char c : n)
            if (c < 0x20 || c > 0x7E) bad("non-printable byte in a name");
    };
    for (const ValueEntry& v : p.values) {
        name_ok(v.name);
        name_ok(v.source_weight);
    }
    for (const GroupKernel& g : p.groups) {
        name_ok(g.label);
        for (const std::string& m : g.members) name_ok(m);
        for (const Launch& L : g.launches) name_ok(L.label);
    }
    for (const ExecStep& es : p.exec_steps) name_ok(es.label);
    for (const std::string& w : p.weight_names) name_ok(w);
    std::vector<int64_t> elems;
    for (const ValueEntry& v : p.values) {
        if (static_cast<unsigned>(v.category) > static_cast<unsigned>(MemCategory::Saved)) bad("value category");
        if (static_cast<unsigned>(v.storage) > static_cast<unsigned>(StorageClass::FusedRegister)) bad("storage class");
        if (v.dims.size() > 8) bad("value rank");
        int64_t n = 1;
        for (int64_t d : v.dims) {
            if (d < 0 || d > (int64_t(1) << 40)) bad("dimension out of range in " + v.name);
            n *= std::max<int64_t>(d, 1);
            if (n > (int64_t(1) << 40)) bad("value too large: " + v.name);
        }
        elems.push_back(n);
    }
    constexpr int kMaxSlots = 48, kMaxRegs = 512;
    for (const GroupKernel& g : p.groups) {
        if (g.backend != backends::BackendId::B200_FUSED && g.backend != backends::BackendId::B200_GEMM)
            bad("backend id out of range");
        for (const Launch& L : g.launches) {
            if (static_cast<unsigned>(L.kind) > static_cast<unsigned>(LaunchKind::LnDgamma)) bad("launch kind");
            if (static_cast<unsigned>(L.op) > static_cast<unsigned>(hlir::OpKind::LayerNormGradGamma)) bad("op kind");
            if (L.is_out.size() != L.args.size()) bad("argument flags");
            if (L.args.size() > static_cast<size_t>(kMaxSlots)) bad("too many launch arguments");
            for (const Arg& a : L.args)
                if (a.offset < 0 || a.offset >= std::max<int64_t>(elems[a.slot], 1)) bad("argument offset out of range");
            if (L.kind != LaunchKind::Ew) continue;
            if (L.ew_regs < 0 || L.ew_regs > kMaxRegs) bad("register count");
            const int nargs = static_cast<int>(L.args.size());
            for (const nncb_ew_instr& in : L.ew) {
                // register operands each opcode reads (unused fields are -1)
                int need = 0;   // bit i: field i of {dst, a, b, c, d, e, f, h} must be a register
                switch (in.op) {
                    case NNCB_EW_LOAD: case NNCB_EW_LOAD_CH: need = 0x01; break;
                    case NNCB_EW_STORE: need = 0x02; break;
                    case NNCB_EW_RELU: case NNCB_EW_COPY: case NNCB_EW_GELU: case NNCB_EW_GELU_FAST: need = 0x03; break;
                    case NNCB_EW_RELU_GRAD: case NNCB_EW_ADD: case NNCB_EW_MUL: case NNCB_EW_GELU_GRAD:
                    case NNCB_EW_GELU_GRAD_FAST: need = 0x07; break;
                    case NNCB_EW_BN_APPLY: case NNCB_EW_BN_INFER: need = 0x3F; break;
                    case NNCB_EW_BN_GRAD: case NNCB_EW_BN_GRAD_FAST: need = 0xFF; break;
                    case NNCB_EW_REDUCE_BN_GRAD: need = 0x1E; break;
                    case NNCB_EW_REDUCE_STATS: need = 0x02; break;
                    case NNCB_EW_REDUCE_SUM: need = 0x02; break;
                    default: bad("elementwise opcode");
                }
                const int fields[8] = {in.dst, in.a, in.b, in.c, in.d, in.e, in.f, in.h};
                for (int f = 0; f < 8; ++f) {
                    if (f == 5 && in.op == NNCB_EW_REDUCE_BN_GRAD) continue;   // e is a slot there
                    const int r = fields[f];
                    const bool ok = (need >> f & 1) ? (r >= 0 && r < L.ew_regs) : (r >= -1 && r < std::max(L.ew_regs, 1));
                    if (!ok)
                        bad("register field " + std::to_string(f) + " = " + std::to_string(r) + " out of range (" +
                            std::to_string(L.ew_regs) + " registers) in " + L.label);
                }
                const bool slotted = in.op == NNCB_EW_LOAD || in.op == NNCB_EW_LOAD_CH || in.op == NNCB_EW_STORE ||
                                     in.op == NNCB_EW_REDUCE_BN_GRAD || in.op == NNCB_EW_REDUCE_STATS ||
                                     in.op == NNCB_EW_REDUCE_SUM;
                if (slotted && (in.slot < 0 || in.slot >= nargs)) bad("elementwise slot out of range in " + L.label);
                if (in.op == NNCB_EW_REDUCE_BN_GRAD && (in.e < 0 || in.e >= nargs))
                    bad("elementwise slot out of range in " + L.label);
            }
        }
    }
    for (const ExecStep& es : p.exec_steps)
        if (es.kernel < -1 || es.kernel >= static_cast<int32_t>(p.groups[es.group].members.size()))
            bad("exec step kernel index");
    const int32_t last = static_cast<int32_t>(p.exec_steps.size());
    for (const PlanEvent& e : p.events)
        if (e.step < 0 || e.step > last) bad("event step out of range");
}

ExecutionPlan read_plan(Reader& r) {
    r.need(4);
    if (std::memcmp(r.in.data() + r.pos, kMagic, 4) != 0) throw Error(Error::Code::BadDocument, "SOLP: bad magic");
    r.pos += 4;
    if (r.u32() != kVersion) throw Error(Error::Code::BadDocument, "SOLP: unsupported plan version");
    ExecutionPlan p;
    p.dtype = static_cast<DType>(r.u8());
    p.role = static_cast<PlanRole>(r.u8());
    const uint32_t nv = r.count(16);
    auto slot = [&](uint32_t s) {
        if (s >= nv) throw Error(Error::Code::BadDocument, "SOLP: slot index out of range");
        return s;
    };
    for (uint32_t i = 0; i < nv; ++i) {
        ValueEntry e;
        e.name = r.str();
        e.category = static_cast<MemCategory>(r.u8());
        e.storage = static_cast<StorageClass>(r.u8());
        e.resident = r.u8() != 0;
        e.source_weight = r.str();
        uint32_t nd = r.count(8);
        for (uint32_t d = 0; d < nd; ++d) e.dims.push_back(r.i64());
        p.values.push_back(std::move(e));
    }
    uint32_t ng = r.count(8);
    for (uint32_t g = 0; g < ng; ++g) {
        GroupKernel gk;
        gk.id = r.u32();
        gk.backend = static_cast<backends::BackendId>(r.u8());
        gk.label = r.str();
        uint32_t nm = r.count(4);
        for (uint32_t i = 0; i < nm; ++i) gk.members.push_back(r.str());
        uint32_t nl = r.count(8);
        for (uint32_t l = 0; l < nl; ++l) {
            Launch L;
            L.kind = static_cast<LaunchKind>(r.u8());
            L.label = r.str();
            uint32_t na = r.count(13);
            for (uint32_t i = 0; i < na; ++i) {
                Arg a;
                a.slot = slot(r.u32());
                a.offset = r.i64();
                L.args.push_back(a);
                L.is_out.push_back(r.u8() != 0);
            }
            uint32_t ni = r.count(48);
            for (uint32_t i = 0; i < ni; ++i) {
                nncb_ew_instr in{};
                in.op = r.i32();
                in.dst = r.i32();
                in.a = r.i32();
                in.b = r.i32();
                in.c = r.i32();
                in.d = r.i32();
                in.e = r.i32();
                in.f = r.i32();
                in.h = r.i32();
                in.slot = r.i32();
                in.imm = r.f64();
                L.ew.push_back(in);
            }
            L.ew_regs = r.i32();
            L.elem_slot = slot(r.u32());
            L.op = static_cast<hlir::OpKind>(r.u32());
            L.attrs = read_attrs(r);
            L.relu_epilogue = r.u8() != 0;
            L.tile = r.i32();
            gk.launches.push_back(std::move(L));
        }
        p.groups.push_back(std::move(gk));
    }
    uint32_t ns = r.count(8);
    for (uint32_t i = 0; i < ns; ++i) {
        ExecStep es;
        es.group = r.u32();
        if (es.group >= p.groups.size()) throw Error(Error::Code::BadDocument, "SOLP: group index out of range");
        es.kernel = r.i32();
        es.label = r.str();
        uint32_t nl = r.count(4);
        for (uint32_t l = 0; l < nl; ++l) {
            uint32_t li = r.u32();
            if (li >= p.groups[es.group].launches.size())
                throw Error(Error::Code::BadDocument, "SOLP: launch index out of range");
            es.launches.push_back(li);
        }
        p.exec_steps.push_back(std::move(es));
    }
    uint32_t ne = r.count(9);
    for (uint32_t i = 0; i < ne; ++i) {
        PlanEvent e;
        e.step = r.i32();
        e.alloc = r.u8() != 0;
        e.slot = slot(r.u32());
        p.events.push_back(e);
    }
    uint32_t n = r.count(4);
    for (uint32_t i = 0; i < n; ++i) p.input_slots.push_back(slot(r.u32()));
    n = r.count(4);
    for (uint32_t i = 0; i < n; ++i) p.output_slots.push_back(slot(r.u32()));
    n = r.count(4);
    for (uint32_t i = 0; i < n; ++i) p.weight_names.push_back(r.str());
    validate_plan(p);
    p.uid = next_plan_uid();
    return p;
}

}  // namespace

std::vector<uint8_t> serialize_plan(const ExecutionPlan& p) {
    Writer w;
    write_plan(w, p);
    return std::move(w.out);
}

ExecutionPlan load_plan(const std::vector<uint8_t>& bytes) {
    Reader r{bytes};
    ExecutionPlan p = read_plan(r);
    if (r.pos != bytes.size()) throw Error(Error::Code::BadDocument, "SOLP: trailing bytes after the plan");
    return p;
}

void save_plan_file(const ExecutionPlan& p, const std::string& path) {
    std::vector<uint8_t> b = serialize_plan(p);
    std::ofstream f(path, std::ios::binary);
    f.write(reinterpret_cast<const char*>(b.data()), static_cast<std::streamsize>(b.size()));
    if (!f) throw Error(Error::Code::BadDocument, "SOLP: cannot write " + path);
}

ExecutionPlan load_plan_file(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw Error(Error::Code::BadDocument, "SOLP: cannot read " + path);
    std::vector<uint8_t> b((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    return load_plan(b);
}

std::vector<uint8_t> serialize_version_plans(const VersionPlans& v) {
    Writer w;
    w.raw(kSetMagic, 4);
    w.u32(kVersion);
    for (const ExecutionPlan* p : {&v.inference, &v.train_fwd, &v.train_bwd}) {
        std::vector<uint8_t> b = serialize_plan(*p);
        w.u64(b.size());
        w.raw(b.data(), b.size());
    }
    w.u32(static_cast<uint32_t>(v.save_set.size()));
    for (const std::string& s : v.save_set) w.str(s);
    w.u32(static_cast<uint32_t>(v.output_grads.size()));
    for (const std::string& s : v.output_grads) w.str(s);
    w.u32(static_cast<uint32_t>(v.weight_grads.size()));
    for (const auto& [k, g] : v.weight_grads) {
        w.str(k);
        w.str(g);
    }
    return std::move(w.out);
}

VersionPlans load_version_plans(const std::vector<uint8_t>& bytes) {
    Reader r{bytes};
    r.need(4);
    if (std::memcmp(bytes.data(), kSetMagic, 4) != 0) throw Error(Error::Code::BadDocument, "SOLP: bad magic");
    r.pos = 4;
    if (r.u32() != kVersion) throw Error(Error::Code::BadDocument, "SOLP: unsupported plan version");
    VersionPlans v;
    for (ExecutionPlan* p : {&v.inference, &v.train_fwd, &v.train_bwd}) {
        uint64_t n = r.u64();
        r.need(n);
        std::vector<uint8_t> b(bytes.begin() + static_cast<std::ptrdiff_t>(r.pos),
                               bytes.begin() + static_cast<std::ptrdiff_t>(r.pos + n));
        r.pos += n;
        *p = load_plan(b);
    }
    auto name = [&]() {
        std::string s = r.str();
        for (unsigned char c : s)
            if (c < 0x20 || c > 0x7E) throw Error(Error::Code::BadDocument, "SOLP: non-printable byte in a name");
        return s;
    };
    uint32_t n = r.count(4);
    for (uint32_t i = 0; i < n; ++i) v.save_set.push_back(name());
    n = r.count(4);
    for (uint32_t i = 0; i < n; ++i) v.output_grads.push_back(name());
    n = r.count(8);
    for (uint32_t i = 0; i < n; ++i) {
        std::string k = name();
        v.weight_grads[k] = name();
    }
    if (r.pos != bytes.size()) throw Error(Error::Code::BadDocument, "SOLP: trailing bytes after the plan set");
    return v;
}

}  // namespace nnc::plan
