// fvb_registry.cu -- structural-key lookup: the B200 counterpart of the
// reference's JIT cache (proj/src/backend_jit.cpp:112-155, 314-335).
//
// The reference compiles one C loop per tree *shape*, keyed by key_node's
// rendering of the tree.  Here every supported shape maps to a hand-written
// fused sm_100a kernel instead.  The patterns are rendered by replaying, on a
// tiny expression builder, exactly the tree constructions of the reference's
// fluid layer (proj/src/fluid.cpp) and of the new blocks,
// in the key_node grammar:
//     Leaf      L<p><slot>;             (slot = first-appearance DFS index)
//     Constant  C<p><16 hex bits>;      (value after narrowing)
//     Unary     U<op><p>(<child>)
//     Binary    B<op><p>(<lhs>,<rhs>)
//     Tag/Cache transparent
// preceded by the destination precision character.  A fused block key is
// "G<rows>x<cols>:" followed by its items' keys joined by '|', with leaf
// slots numbered across the whole block.  In a pattern a
// constant is a named wildcard "C<p>#<name>;": the first occurrence captures
// the key's bits, later occurrences must carry the same bits, and the values
// become the kernel's constants -- so any EosSpec gas runs on the same kernel.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "fvb.h"
#include "fvb_launch.cuh"
#include "fvb_lower.h"

namespace fvb {
namespace {

// ---- a minimal expression builder mirroring fusevec::Expr -------------------

// Operator codes are the reference's enum values (include/fusevec/expr.hpp:12-46).
enum : int { kNeg = 0, kSin = 2, kSqrt = 15 };
enum : int { kAdd = 0, kSub = 1, kMul = 2, kDiv = 3 };

struct Node;
using N = std::shared_ptr<const Node>;
struct Node {
    char kind;          // 'L', 'C', 'U', 'B'
    int op = 0;         // unary/binary op code
    std::string name;   // leaf name or constant name
    N l, r;
};

N leaf(const std::string& n) { return std::make_shared<Node>(Node{'L', 0, n, nullptr, nullptr}); }
N cst(const std::string& n) { return std::make_shared<Node>(Node{'C', 0, n, nullptr, nullptr}); }
N un(int op, N a) { return std::make_shared<Node>(Node{'U', op, "", a, nullptr}); }
N bin(int op, N a, N b) { return std::make_shared<Node>(Node{'B', op, "", a, b}); }
N add(N a, N b) { return bin(kAdd, a, b); }
N sub(N a, N b) { return bin(kSub, a, b); }
N mul(N a, N b) { return bin(kMul, a, b); }
N dvd(N a, N b) { return bin(kDiv, a, b); }
N neg(N a) { return un(kNeg, a); }

struct Render {
    char p;                          // precision char, 'd' or 's'
    std::vector<std::string> slots;  // leaf names in first-appearance order
    int slot_of(const std::string& n) {
        for (size_t i = 0; i < slots.size(); ++i)
            if (slots[i] == n) return int(i);
        slots.push_back(n);
        return int(slots.size() - 1);
    }
    // key_node (proj/src/backend_jit.cpp:112-155) over a uniform-precision tree.
    void node(const Node& n, std::string& out) {
        switch (n.kind) {
            case 'L':
                out += 'L';
                out += p;
                out += std::to_string(slot_of(n.name));
                out += ';';
                return;
            case 'C':
                out += 'C';
                out += p;
                out += '#';
                out += n.name;
                out += ';';
                return;
            case 'U':
                out += 'U';
                out += std::to_string(n.op);
                out += p;
                out += '(';
                node(*n.l, out);
                out += ')';
                return;
            default:
                out += 'B';
                out += std::to_string(n.op);
                out += p;
                out += '(';
                node(*n.l, out);
                out += ',';
                node(*n.r, out);
                out += ')';
                return;
        }
    }
    std::string expr(const N& e) {
        std::string out(1, p);
        node(*e, out);
        return out;
    }
    std::string block(int rows, int cols, const std::vector<N>& items) {
        std::string out = "G" + std::to_string(rows) + "x" + std::to_string(cols) + ":";
        for (size_t i = 0; i < items.size(); ++i) {
            if (i) out += '|';
            out += p;
            node(*items[i], out);
        }
        return out;
    }
};

// ---- the reference's fluid trees (proj/src/fluid.cpp), conservative state --

struct Cons {
    int d;
    N rho, m[3], rho_E;
    explicit Cons(int dim) : d(dim) {
        rho = leaf("rho");
        for (int j = 0; j < d; ++j) m[j] = leaf("m" + std::to_string(j));
        rho_E = leaf("E");
    }
};

// sum_of_squares (fluid.cpp:222-230)
N sum_sq(const N* q, int d) {
    N acc;
    for (int i = 0; i < d; ++i) {
        N sq = mul(q[i], q[i]);
        acc = acc ? add(acc, sq) : sq;
    }
    return acc;
}

// derived_p (fluid.cpp:234-241)
N derived_p(const Cons& u) {
    N msq = sum_sq(u.m, u.d);
    N kin = mul(cst("half"), dvd(msq, u.rho));
    return mul(cst("gm1"), sub(u.rho_E, kin));
}

// derived_v_mag2 (fluid.cpp:243-247)
N v_mag2(const Cons& u) { return dvd(sum_sq(u.m, u.d), mul(u.rho, u.rho)); }

// sound speed: elem_sqrt((constant(gamma, p) * p) / rho)
N sound_speed(const Cons& u) {
    N p = derived_p(u);
    return un(kSqrt, dvd(mul(cst("gamma"), p), u.rho));
}

// wave speed: elem_sqrt(derived_v_mag2(u)) + c
N wave_speed(const Cons& u) { return add(un(kSqrt, v_mag2(u)), sound_speed(u)); }

// inviscid_flux, conservative (fluid.cpp:273-310)
std::vector<N> flux_items(const Cons& u) {
    const int d = u.d;
    N v[3];
    for (int j = 0; j < d; ++j) v[j] = dvd(u.m[j], u.rho);
    N p = derived_p(u);
    std::vector<N> items;
    for (int j = 0; j < d; ++j) items.push_back(u.m[j]);
    for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j) {
            N f = mul(u.m[i], v[j]);
            if (i == j) f = add(f, p);
            items.push_back(f);
        }
    for (int j = 0; j < d; ++j) items.push_back(mul(v[j], add(u.rho_E, p)));
    return items;
}

// convert(u, Primitive) fields 1..d+1 (fluid.cpp:249-258), optionally + c
std::vector<N> prim_items(const Cons& u, bool with_c) {
    std::vector<N> items;
    for (int j = 0; j < u.d; ++j) items.push_back(dvd(u.m[j], u.rho));
    items.push_back(derived_p(u));
    if (with_c) items.push_back(sound_speed(u));
    return items;
}

// convert(w, Conservative) fields 1..d+1 (fluid.cpp:259-268)
std::vector<N> cons_items(int d) {
    N rho = leaf("rho"), v[3], p = leaf("p");
    for (int j = 0; j < d; ++j) v[j] = leaf("v" + std::to_string(j));
    std::vector<N> items;
    for (int j = 0; j < d; ++j) items.push_back(mul(rho, v[j]));
    N vsq = sum_sq(v, d);
    items.push_back(add(dvd(p, cst("gm1")), mul(cst("half"), mul(rho, vsq))));
    return items;
}

// inviscid_flux, primitive (fluid.cpp:290-298)
std::vector<N> flux_prim_items(int d) {
    N rho = leaf("rho"), v[3], rv[3], p = leaf("p");
    for (int j = 0; j < d; ++j) v[j] = leaf("v" + std::to_string(j));
    for (int j = 0; j < d; ++j) rv[j] = mul(rho, v[j]);
    N vsq = sum_sq(v, d);
    N rho_E = add(dvd(p, cst("gm1")), mul(cst("half"), mul(rho, vsq)));
    std::vector<N> items;
    for (int j = 0; j < d; ++j) items.push_back(rv[j]);
    for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j) {
            N f = mul(rv[i], v[j]);
            if (i == j) f = add(f, p);
            items.push_back(f);
        }
    for (int j = 0; j < d; ++j) items.push_back(mul(v[j], add(rho_E, p)));
    return items;
}

// Flux Jacobians, SURVEY A.3, items [k][r][c]
std::vector<N> jacobian_items(const Cons& u) {
    const int d = u.d, w = d + 2;
    N p = derived_p(u);
    N v[3];
    for (int j = 0; j < d; ++j) v[j] = dvd(u.m[j], u.rho);
    N q2 = sum_sq(v, d);
    N H = dvd(add(u.rho_E, p), u.rho);
    N phi = mul(cst("half"), mul(cst("gm1"), q2));
    std::vector<N> items;
    for (int k = 0; k < d; ++k) {
        for (int c = 0; c < w; ++c) items.push_back(cst(c == 1 + k ? "one" : "zero"));
        for (int i = 0; i < d; ++i) {
            items.push_back(i == k ? sub(phi, mul(v[i], v[k])) : neg(mul(v[i], v[k])));
            for (int j = 0; j < d; ++j) {
                N acc;
                if (i == j) acc = v[k];
                if (j == k) acc = acc ? add(acc, v[i]) : v[i];
                if (i == k) {
                    N t = neg(mul(cst("gm1"), v[j]));
                    acc = acc ? add(acc, t) : t;
                }
                items.push_back(acc ? acc : cst("zero"));
            }
            items.push_back(cst(i == k ? "gm1" : "zero"));
        }
        items.push_back(mul(v[k], sub(phi, H)));
        for (int j = 0; j < d; ++j) {
            N ujuk = mul(v[j], v[k]);
            items.push_back(j == k ? sub(H, mul(cst("gm1"), ujuk)) : neg(mul(cst("gm1"), ujuk)));
        }
        items.push_back(mul(cst("gamma"), v[k]));
    }
    return items;
}

// ---- kernel entries ---------------------------------------------------------

// Captured constants live in fvb_kernel::consts at these canonical indices.
const char* const kConstNames[] = {"half", "gm1", "gamma", "cv", "zero", "one"};
constexpr int kNumConsts = 6;

int const_index(const std::string& n) {
    for (int i = 0; i < kNumConsts; ++i)
        if (n == kConstNames[i]) return i;
    return -1;
}

template <class T>
Consts<T> consts_of(const fvb_kernel* k) {
    // The captured bits are already narrowed to T, so the casts are exact.
    return Consts<T>{static_cast<T>(k->consts[0]), static_cast<T>(k->consts[1]),
                     static_cast<T>(k->consts[2]), static_cast<T>(k->consts[3]),
                     static_cast<T>(k->consts[4]), static_cast<T>(k->consts[5])};
}

template <class Op, class T>
fvb_status entry(const fvb_kernel* k, uint64_t begin, uint64_t end, void* const* args,
                 void* stream) {
    if (!k || !args) return fail(FVB_EARG, "NULL kernel or argument block");
    if (end < begin) return fail(FVB_EARG, "end < begin");
    const T* in[Op::NIN];
    for (int i = 0; i < Op::NIN; ++i) {
        const int s = k->in_slot[i];
        if (s < 0 || uint32_t(s) >= k->n_inputs || !args[k->n_outputs + s])
            return fail(FVB_EARG, "NULL or missing leaf slot");
        in[i] = static_cast<const T*>(args[k->n_outputs + s]) + begin;
    }
    T* out[Op::NOUT > 0 ? Op::NOUT : 1];
    for (int j = 0; j < Op::NOUT; ++j) {
        if (!args[j]) return fail(FVB_EARG, "NULL output slot");
        out[j] = static_cast<T*>(args[j]) + begin;
    }
    // A destination that is also a leaf (evaluate in place, as the
    // reference's JitKernel allows) runs the coherent-load variant.
    if (!Op::ALIASED && end > begin &&
        plane_overlap(reinterpret_cast<const void* const*>(in), Op::NIN,
                      reinterpret_cast<const void* const*>(out), Op::NOUT,
                      size_t(end - begin) * sizeof(T)) == kSame)
        return launch_op<InPlace<Op>, T, false, false>(in, out, end - begin, consts_of<T>(k),
                                                       nullptr, static_cast<cudaStream_t>(stream));
    return launch_op<Op, T, false, false>(in, out, end - begin, consts_of<T>(k), nullptr,
                                          static_cast<cudaStream_t>(stream));
}

// The reduce entry: same pass plus the CFL max, accumulated into *red.
template <class Op, class T>
fvb_status entry_reduce(const fvb_kernel* k, uint64_t begin, uint64_t end, void* const* args,
                        void* red, void* stream) {
    if (!k || !args || !red) return fail(FVB_EARG, "NULL kernel, argument block or lambda_max");
    if (end < begin) return fail(FVB_EARG, "end < begin");
    const T* in[Op::NIN];
    for (int i = 0; i < Op::NIN; ++i) {
        const int s = k->in_slot[i];
        if (s < 0 || uint32_t(s) >= k->n_inputs || !args[k->n_outputs + s])
            return fail(FVB_EARG, "NULL or missing leaf slot");
        in[i] = static_cast<const T*>(args[k->n_outputs + s]) + begin;
    }
    T* out[Op::NOUT > 0 ? Op::NOUT : 1];
    for (int j = 0; j < Op::NOUT; ++j) {
        if (!args[j]) return fail(FVB_EARG, "NULL output slot");
        out[j] = static_cast<T*>(args[j]) + begin;
    }
    auto* r = static_cast<typename Bits<T>::U*>(red);
    if (!Op::ALIASED && end > begin &&
        plane_overlap(reinterpret_cast<const void* const*>(in), Op::NIN,
                      reinterpret_cast<const void* const*>(out), Op::NOUT,
                      size_t(end - begin) * sizeof(T)) == kSame)
        return launch_op<InPlace<Op>, T, true, false>(in, out, end - begin, consts_of<T>(k), r,
                                                      static_cast<cudaStream_t>(stream));
    return launch_op<Op, T, true, false>(in, out, end - begin, consts_of<T>(k), r,
                                         static_cast<cudaStream_t>(stream));
}

// Wave speed: per-point lambda when args[0] is set, reduction only otherwise.
template <class T, int D>
fvb_status wave_reduce(const fvb_kernel* k, uint64_t begin, uint64_t end, void* const* args,
                       void* red, void* stream) {
    if (args && args[0]) return entry_reduce<WaveSpeedOp<T, D, 1>, T>(k, begin, end, args, red, stream);
    return entry_reduce<WaveSpeedOp<T, D, 0>, T>(k, begin, end, args, red, stream);
}

struct Pattern {
    std::string name;
    std::string text;                // key with named constant wildcards
    std::vector<std::string> slots;  // leaf names in slot order
    std::vector<std::string> canon;  // the kernel's canonical input order
    uint32_t n_outputs;
    uint8_t prec, dim;
    fvb_kernel_fn fn;
    fvb_kernel_reduce_fn reduce = nullptr;
};

std::vector<std::string> cons_names(int d) {
    std::vector<std::string> c{"rho"};
    for (int j = 0; j < d; ++j) c.push_back("m" + std::to_string(j));
    c.push_back("E");
    return c;
}

std::vector<std::string> prim_names(int d) {
    std::vector<std::string> c{"rho"};
    for (int j = 0; j < d; ++j) c.push_back("v" + std::to_string(j));
    c.push_back("p");
    return c;
}

template <class T, int D>
void add_fluid(std::vector<Pattern>& ps) {
    const char pc = sizeof(T) == 8 ? 'd' : 's';
    const std::string sfx = std::to_string(D) + (sizeof(T) == 8 ? "_f64" : "_f32");
    const Cons u(D);
    auto block = [&](const std::string& name, int rows, int cols, const std::vector<N>& items,
                     std::vector<std::string> canon, fvb_kernel_fn fn) {
        Render r{pc, {}};
        Pattern p{name + sfx, r.block(rows, cols, items), {}, std::move(canon),
                  uint32_t(items.size()), uint8_t(sizeof(T) == 8), uint8_t(D), fn};
        p.slots = r.slots;
        ps.push_back(std::move(p));
    };
    auto single = [&](const std::string& name, const N& e, std::vector<std::string> canon,
                      fvb_kernel_fn fn) {
        Render r{pc, {}};
        Pattern p{name + sfx, r.expr(e), {}, std::move(canon), 1u, uint8_t(sizeof(T) == 8),
                  uint8_t(D), fn};
        p.slots = r.slots;
        ps.push_back(std::move(p));
    };
    const auto cn = cons_names(D);
    block("flux", D + 2, D, flux_items(u), cn, entry<FluxOp<T, D>, T>);
    block("cons2prim", D + 1, 1, prim_items(u, false), cn,
          entry<SliceOp<Cons2PrimOp<T, D>, 0, D + 1>, T>);
    block("cons2prim_c", D + 2, 1, prim_items(u, true), cn, entry<Cons2PrimOp<T, D>, T>);
    block("prim2cons", D + 1, 1, cons_items(D), prim_names(D), entry<Prim2ConsOp<T, D>, T>);
    block("flux_prim", D + 2, D, flux_prim_items(D), prim_names(D), entry<FluxPrimOp<T, D>, T>);
    block("jacobian", D * (D + 2), D + 2, jacobian_items(u), cn, entry<JacobianOp<T, D>, T>);
    ps.back().reduce = entry_reduce<JacobianOp<T, D>, T>;
    single("pressure", derived_p(u), cn, entry<SliceOp<Cons2PrimOp<T, D>, D, 1>, T>);
    single("sound_speed", sound_speed(u), cn, entry<SliceOp<Cons2PrimOp<T, D>, D + 1, 1>, T>);
    single("v_mag2", v_mag2(u), std::vector<std::string>(cn.begin(), cn.end() - 1),
           entry<VMag2Op<T, D>, T>);
    single("wave_speed", wave_speed(u), cn, entry<WaveSpeedOp<T, D, 1>, T>);
    ps.back().reduce = wave_reduce<T, D>;
}

template <class T>
void add_scalar(std::vector<Pattern>& ps) {
    const char pc = sizeof(T) == 8 ? 'd' : 's';
    const std::string sfx = sizeof(T) == 8 ? "_f64" : "_f32";
    auto single = [&](const std::string& name, const N& e, std::vector<std::string> canon,
                      fvb_kernel_fn fn) {
        Render r{pc, {}};
        Pattern p{name + sfx, r.expr(e), {}, std::move(canon), 1u, uint8_t(sizeof(T) == 8), 0,
                  fn};
        p.slots = r.slots;
        ps.push_back(std::move(p));
    };
    // constant(0.5, leaf(y)) * elem_sin(leaf(x) + leaf(y))  (test_backend.cpp:41)
    single("axpy_sin", mul(cst("half"), un(kSin, add(leaf("x"), leaf("y")))), {"x", "y"},
           entry<AxpySinOp<T>, T>);
    // eos_ideal_p: rho_e = rho*e; constant(gm1, rho_e) * rho_e (fluid.cpp:57-60)
    single("eos_p", mul(cst("gm1"), mul(leaf("rho"), leaf("e"))), {"rho", "e"},
           entry<EosOp<T, 1>, T>);
}

// eos_ideal_T reads only e; its kernel takes [rho, e] canonically, so it is
// registered with e in both canonical slots.
template <class T>
void add_eos_T(std::vector<Pattern>& ps) {
    const char pc = sizeof(T) == 8 ? 'd' : 's';
    Render r{pc, {}};
    Pattern p{std::string("eos_T") + (sizeof(T) == 8 ? "_f64" : "_f32"),
              r.expr(dvd(leaf("e"), cst("cv"))), {}, {"e", "e"}, 1u, uint8_t(sizeof(T) == 8), 0,
              entry<EosOp<T, 2>, T>};
    p.slots = r.slots;
    ps.push_back(std::move(p));
}

std::vector<Pattern>& patterns() {
    static std::vector<Pattern> ps = [] {
        std::vector<Pattern> v;
        add_fluid<double, 1>(v);
        add_fluid<double, 2>(v);
        add_fluid<double, 3>(v);
        add_fluid<float, 1>(v);
        add_fluid<float, 2>(v);
        add_fluid<float, 3>(v);
        add_scalar<double>(v);
        add_scalar<float>(v);
        add_eos_T<double>(v);
        add_eos_T<float>(v);
        return v;
    }();
    return ps;
}

// Match `key` against `pat`; named constant wildcards capture into consts.
bool match(const std::string& pat, const char* key, double* consts, bool* seen) {
    size_t i = 0;
    const char* k = key;
    while (i < pat.size()) {
        if (pat[i] == 'C' && i + 2 < pat.size() && pat[i + 2] == '#') {
            const char pc = pat[i + 1];
            const size_t semi = pat.find(';', i);
            const int ci = const_index(pat.substr(i + 3, semi - i - 3));
            if (k[0] != 'C' || k[1] != pc) return false;
            unsigned long long bits = 0;
            for (int h = 0; h < 16; ++h) {
                const char c = k[2 + h];
                int v;
                if (c >= '0' && c <= '9') v = c - '0';
                else if (c >= 'a' && c <= 'f') v = c - 'a' + 10;
                else return false;
                bits = (bits << 4) | unsigned(v);
            }
            if (k[18] != ';') return false;
            double val;
            std::memcpy(&val, &bits, sizeof val);
            if (ci < 0) return false;
            if (seen[ci]) {
                unsigned long long prev;
                std::memcpy(&prev, &consts[ci], sizeof prev);
                if (prev != bits) return false;  // one named constant, two values
            } else {
                consts[ci] = val;
                seen[ci] = true;
            }
            i = semi + 1;
            k += 19;
            continue;
        }
        if (*k != pat[i]) return false;
        ++i;
        ++k;
    }
    return *k == '\0';
}

}  // namespace
}  // namespace fvb

namespace fvb {
namespace {
fvb_status lookup_uncached(const char* key, fvb_kernel* out);
}  // namespace
}  // namespace fvb

using namespace fvb;

extern "C" {

fvb_status fvb_lookup(const char* key, fvb_kernel* out) {
    return guarded([&]() -> fvb_status {
        if (!key || !out) return fail(FVB_EARG, "NULL key or output");
        // Resolved keys, for the process lifetime like the reference's JIT
        // cache (backend_jit.cpp:240-253): a repeated key -- every call of a
        // time loop that rebuilds its trees -- costs one hash lookup instead
        // of a scan of the patterns.
        static std::mutex mu;
        static std::unordered_map<std::string, fvb_kernel> resolved;
        const std::string k_text(key);
        {
            std::lock_guard<std::mutex> lock(mu);
            auto it = resolved.find(k_text);
            if (it != resolved.end()) {
                *out = it->second;
                return FVB_OK;
            }
        }
        const fvb_status st = lookup_uncached(key, out);
        if (st == FVB_OK) {
            std::lock_guard<std::mutex> lock(mu);
            resolved.emplace(k_text, *out);
        }
        return st;
    });
}

}  // extern "C"

namespace fvb {
namespace {

fvb_status lookup_uncached(const char* key, fvb_kernel* out) {
    {
        // FVB_FORCE_LOWER=1 skips the hand-written kernels (tests and the
        // hand-written-vs-lowered comparison run the same trees both ways).
        static const bool force_lower = [] {
            const char* v = std::getenv("FVB_FORCE_LOWER");
            return v && *v && *v != '0';
        }();
        if (force_lower) return lower_lookup(key, out);
        for (const Pattern& p : patterns()) {
            double consts[8] = {0};
            bool seen[8] = {false};
            if (!match(p.text, key, consts, seen)) continue;
            fvb_kernel k;
            std::memset(&k, 0, sizeof k);
            k.fn = p.fn;
            k.reduce = p.reduce;
            k.n_outputs = p.n_outputs;
            k.n_inputs = uint32_t(p.slots.size());
            k.n_consts = kNumConsts;
            k.prec = p.prec;
            k.dim = p.dim;
            // Constants the key did not carry (e.g. the Jacobian's 0 and 1 in a
            // block without them) keep the default gas values, narrowed.
            const fvb_gas dflt{2.0 / 5.0, 7.0 / 5.0, 5.0 / 2.0};
            const double defaults[kNumConsts] = {0.5, dflt.gamma_minus_one, dflt.gamma, dflt.cv, 0.0,
                                                 1.0};
            for (int c = 0; c < kNumConsts; ++c)
                k.consts[c] = seen[c] ? consts[c]
                                      : (p.prec ? defaults[c] : double(float(defaults[c])));
            for (int i = 0; i < 8; ++i) k.in_slot[i] = -1;
            for (size_t i = 0; i < p.canon.size() && i < 8; ++i)
                for (size_t s = 0; s < p.slots.size(); ++s)
                    if (p.slots[s] == p.canon[i]) k.in_slot[i] = int8_t(s);
            std::snprintf(k.name, sizeof k.name, "%s", p.name.c_str());
            *out = k;
            return FVB_OK;
        }
        // No hand-written kernel: lower the tree itself (NVRTC, cached per key).
        return lower_lookup(key, out);
    }
}

}  // namespace
}  // namespace fvb

extern "C" {

uint32_t fvb_pattern_count(void) {
    try {
        return uint32_t(patterns().size());
    } catch (...) {
        return 0;
    }
}

const char* fvb_pattern(uint32_t i, const char** name) {
    try {
        if (i >= patterns().size()) return nullptr;
        if (name) *name = patterns()[i].name.c_str();
        return patterns()[i].text.c_str();
    } catch (...) {
        return nullptr;
    }
}

}  // extern "C"
