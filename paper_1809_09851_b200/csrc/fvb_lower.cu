// fvb_lower.cu -- general lowering: any structural key -> one CUDA kernel.
//
// The B200 counterpart of the reference's runtime JIT
// (proj/src/backend_jit.cpp): there a tree becomes C source, `cc -O3`, and
// dlopen; here the structural key -- which already encodes the whole tree:
// ops, per-node precisions, leaf slots and the exact constant bits
// (key_node, backend_jit.cpp:112-155) -- is parsed back into a DAG and
// emitted as CUDA source, compiled by NVRTC for sm_100a with --fmad=false
// (the reference's -ffp-contract=off), and loaded with the runtime library
// API.  It is cached per key for the process lifetime, like the JIT cache
// (backend_jit.cpp:240-253, 314-335), and the compiled image is also kept
// on disk (FVB_CACHE_DIR, below) so a new process skips NVRTC.
//
// Semantics follow the reference's emit / emit_as (backend_jit.cpp:179-205):
// every node computes in its own precision, operands are converted to it
// first, constants are exact hex literals of the narrowed value, and the
// destination store rounds once.  Across the items of a block every
// distinct subtree is computed once (common-subexpression sharing; bitwise
// neutral).  Each thread loads all leaves of an element before storing any
// output, so a destination may alias a leaf as in the reference
// (backend.hpp:44-46).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvrtc.h>

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "fvb.h"
#include "fvb_launch.cuh"
#include "fvb_lower.h"

namespace fvb {
namespace {

constexpr int kMaxArgs = 256;  // 2 KB of plane pointers per launch
constexpr int kThreads = 256;
constexpr int kPerThread = 4;

// ---- the key's DAG ---------------------------------------------------------

struct KNode {
    char kind;  // 'L', 'C', 'U', 'B'
    char prec;  // 's' or 'd'
    int op = 0;
    int slot = -1;
    double value = 0;
    int l = -1, r = -1;  // child node indices
    std::string canon;   // exact key text of the subtree (CSE identity)
};

struct KDag {
    std::vector<KNode> nodes;
    std::vector<int> roots;        // one per item
    std::vector<char> dest_prec;   // one per item
    std::map<int, char> slot_prec;
    int rows = 1, cols = 1;
    bool block = false;
};

class Parser {
  public:
    Parser(const char* s, KDag& d) : s_(s), d_(d) {}

    bool parse() {
        if (*s_ == 'G') {
            ++s_;
            d_.block = true;
            if (!number(&d_.rows) || *s_++ != 'x' || !number(&d_.cols) || *s_++ != ':')
                return false;
            for (;;) {
                if (!item()) return false;
                if (*s_ == '|') {
                    ++s_;
                    continue;
                }
                break;
            }
            return *s_ == '\0' && int(d_.roots.size()) == d_.rows * d_.cols;
        }
        return item() && *s_ == '\0';
    }

  private:
    const char* s_;
    KDag& d_;
    std::map<std::string, int> seen_;

    bool number(int* out) {
        if (*s_ < '0' || *s_ > '9') return false;
        long v = 0;
        while (*s_ >= '0' && *s_ <= '9') {
            v = v * 10 + (*s_++ - '0');
            if (v > 1 << 20) return false;
        }
        *out = int(v);
        return true;
    }

    bool prec(char* p) {
        if (*s_ != 's' && *s_ != 'd') return false;
        *p = *s_++;
        return true;
    }

    bool item() {
        char p;
        if (!prec(&p)) return false;
        int root;
        if (!node(&root)) return false;
        d_.roots.push_back(root);
        d_.dest_prec.push_back(p);
        return true;
    }

    bool node(int* out) {
        const char* start = s_;
        KNode n;
        n.kind = *s_++;
        switch (n.kind) {
            case 'L': {
                if (!prec(&n.prec) || !number(&n.slot) || *s_++ != ';') return false;
                auto it = d_.slot_prec.find(n.slot);
                if (it != d_.slot_prec.end() && it->second != n.prec) return false;
                d_.slot_prec[n.slot] = n.prec;
                break;
            }
            case 'C': {
                if (!prec(&n.prec)) return false;
                unsigned long long bits = 0;
                for (int h = 0; h < 16; ++h) {
                    const char c = *s_++;
                    int v;
                    if (c >= '0' && c <= '9') v = c - '0';
                    else if (c >= 'a' && c <= 'f') v = c - 'a' + 10;
                    else return false;
                    bits = (bits << 4) | unsigned(v);
                }
                if (*s_++ != ';') return false;
                std::memcpy(&n.value, &bits, sizeof bits);
                if (!std::isfinite(n.value)) return false;  // the JIT refuses these too
                break;
            }
            case 'U':
            case 'B': {
                if (!number(&n.op)) return false;
                if (n.kind == 'U' ? n.op > 20 : n.op > 7) return false;
                if (!prec(&n.prec) || *s_++ != '(') return false;
                if (!node(&n.l)) return false;
                if (n.kind == 'B') {
                    if (*s_++ != ',') return false;
                    if (!node(&n.r)) return false;
                }
                if (*s_++ != ')') return false;
                break;
            }
            default:
                return false;
        }
        n.canon.assign(start, s_);
        auto it = seen_.find(n.canon);
        if (it != seen_.end()) {
            *out = it->second;  // shared subtree: one node
            return true;
        }
        d_.nodes.push_back(std::move(n));
        *out = int(d_.nodes.size() - 1);
        seen_[d_.nodes.back().canon] = *out;
        return true;
    }
};

// ---- emission -------------------------------------------------------------------

const char* ctype(char p) { return p == 's' ? "float" : "double"; }

const char* unary_fn(int op) {
    static const char* names[] = {nullptr, "fabs", "sin",  "cos",   "tan",   "asin", "acos",
                                  "atan",  "sinh", "cosh", "tanh",  "exp",   "log",  "log2",
                                  "log10", "sqrt", "cbrt", "ceil",  "floor", "round", "erf"};
    return names[op];
}

const char* binary_infix(int op) {
    switch (op) {
        case 0: return "+";
        case 1: return "-";
        case 2: return "*";
        case 3: return "/";
        default: return nullptr;
    }
}

const char* binary_fn(int op) {
    switch (op) {
        case 4: return "pow";
        case 5: return "fmin";
        case 6: return "fmax";
        default: return "atan2";
    }
}

std::string literal(double v, char p) {
    char buf[64];
    if (p == 's')
        std::snprintf(buf, sizeof buf, "(%af)", v);
    else
        std::snprintf(buf, sizeof buf, "(%a)", v);
    return buf;
}

// Per-element code generator.  Nodes reached from one item only are that
// item's private subtree and are emitted inside the item's store loop;
// nodes shared by several items (the block's common subexpressions, e.g.
// v_j and p of the flux) are computed once per element up front.  This is
// the hand-written kernels' prepare()/out() split, derived from the DAG, and
// keeps only the shared state live while outputs stream out.
struct Emitter {
    const KDag& d;
    std::vector<int> owner;  // item index, or -2 when shared by several items
    explicit Emitter(const KDag& dag) : d(dag), owner(dag.nodes.size(), -1) {
        for (size_t j = 0; j < d.roots.size(); ++j) mark(d.roots[j], int(j));
    }

    void mark(int idx, int item) {
        int& o = owner[idx];
        if (o == item || o == -2) return;
        o = (o == -1) ? item : -2;
        const KNode& n = d.nodes[idx];
        if (n.l >= 0) mark(n.l, o == -2 ? -2 : item);
        if (n.r >= 0) mark(n.r, o == -2 ? -2 : item);
    }

    bool computed(int idx) const { return d.nodes[idx].kind == 'U' || d.nodes[idx].kind == 'B'; }

    // Expression naming node idx for element k (inside the k loop).
    std::string ref(int idx) const {
        const KNode& n = d.nodes[idx];
        if (n.kind == 'L') return "v" + std::to_string(n.slot) + "[k]";
        if (n.kind == 'C') return literal(n.value, n.prec);
        if (owner[idx] == -2) return "s" + std::to_string(idx) + "[k]";
        return "p" + std::to_string(idx);
    }

    std::string as(char want, int idx) const {
        const std::string e = ref(idx);
        if (d.nodes[idx].prec == want) return e;
        return std::string("(") + ctype(want) + ")(" + e + ")";
    }

    // The operation of a computed node on its children's references.
    std::string op(int idx) const {
        const KNode& n = d.nodes[idx];
        if (n.kind == 'U') {
            const std::string c = as(n.prec, n.l);
            if (n.op == 0) return "(-(" + c + "))";
            std::string fn = unary_fn(n.op);
            if (n.prec == 's') fn += 'f';
            return fn + "(" + c + ")";
        }
        const std::string a = as(n.prec, n.l), b = as(n.prec, n.r);
        if (const char* o = binary_infix(n.op)) return "(" + a + " " + o + " " + b + ")";
        std::string fn = binary_fn(n.op);
        if (n.prec == 's') fn += 'f';
        return fn + "(" + a + ", " + b + ")";
    }

    // Post-order emission of the computed nodes selected by `want`.
    void post(int idx, const std::function<bool(int)>& want, std::vector<bool>& done,
              std::vector<int>& order) const {
        if (done[idx]) return;
        const KNode& n = d.nodes[idx];
        if (n.l >= 0) post(n.l, want, done, order);
        if (n.r >= 0) post(n.r, want, done, order);
        done[idx] = true;
        if (computed(idx) && want(idx)) order.push_back(idx);
    }
};

bool emit(const char* key, std::string* src, KDag* dag_out, bool wide = true, int minb = 2) {
    KDag d;
    Parser p(key, d);
    if (!p.parse()) return false;
    const int nout = int(d.roots.size());
    const int nin = d.slot_prec.empty() ? 0 : d.slot_prec.rbegin()->first + 1;
    if (int(d.slot_prec.size()) != nin) return false;  // slots must be dense 0..nin-1
    if (nout + nin > kMaxArgs) return false;
    Emitter e(d);
    const std::string T = std::to_string(kThreads);
    auto num = [](int x) { return std::to_string(x); };
    std::string s;
    s += "// lowered by libfvb from a structural key (proj/src/backend_jit.cpp grammar)\n";
    s += "typedef unsigned long long fvb_u64;\n";
    s += "struct FvbArgs { void* p[" + num(kMaxArgs) + "]; };\n";
    // 4 consecutive elements per access (the planes may alias: no .nc path)
    if (wide)  // sm_100's 256-bit access (NVRTC >= 12.9)
        s += "__device__ __forceinline__ void fvb_ld4(const double* p, double* v)\n{\n"
             "    asm volatile(\"ld.global.v4.f64 {%0, %1, %2, %3}, [%4];\" : \"=d\"(v[0]), "
             "\"=d\"(v[1]), \"=d\"(v[2]), \"=d\"(v[3]) : \"l\"(p) : \"memory\");\n}\n"
             "__device__ __forceinline__ void fvb_st4(double* p, const double* v)\n{\n"
             "    asm volatile(\"st.global.v4.f64 [%0], {%1, %2, %3, %4};\" :: \"l\"(p), "
             "\"d\"(v[0]), \"d\"(v[1]), \"d\"(v[2]), \"d\"(v[3]) : \"memory\");\n}\n";
    else
        s += "__device__ __forceinline__ void fvb_ld4(const double* p, double* v)\n{\n"
             "    asm volatile(\"ld.global.v2.f64 {%0, %1}, [%2];\" : \"=d\"(v[0]), \"=d\"(v[1]) "
             ": \"l\"(p) : \"memory\");\n"
             "    asm volatile(\"ld.global.v2.f64 {%0, %1}, [%2];\" : \"=d\"(v[2]), \"=d\"(v[3]) "
             ": \"l\"(p + 2) : \"memory\");\n}\n"
             "__device__ __forceinline__ void fvb_st4(double* p, const double* v)\n{\n"
             "    asm volatile(\"st.global.v2.f64 [%0], {%1, %2};\" :: \"l\"(p), \"d\"(v[0]), "
             "\"d\"(v[1]) : \"memory\");\n"
             "    asm volatile(\"st.global.v2.f64 [%0], {%1, %2};\" :: \"l\"(p + 2), \"d\"(v[2]), "
             "\"d\"(v[3]) : \"memory\");\n}\n";
    s += "__device__ __forceinline__ void fvb_ld4(const float* p, float* v)\n{\n"
         "    asm volatile(\"ld.global.v4.f32 {%0, %1, %2, %3}, [%4];\" : \"=f\"(v[0]), "
         "\"=f\"(v[1]), \"=f\"(v[2]), \"=f\"(v[3]) : \"l\"(p) : \"memory\");\n}\n"
         "__device__ __forceinline__ void fvb_st4(float* p, const float* v)\n{\n"
         "    asm volatile(\"st.global.v4.f32 [%0], {%1, %2, %3, %4};\" :: \"l\"(p), \"f\"(v[0]), "
         "\"f\"(v[1]), \"f\"(v[2]), \"f\"(v[3]) : \"memory\");\n}\n";

    // fvb_tile<E>: E consecutive elements from i0 (E = 4 wide, E = 1 scalar)
    s += "template <int E>\n__device__ __forceinline__ void fvb_tile(const FvbArgs& a, "
         "const fvb_u64 i0)\n{\n";
    for (int i = 0; i < nin; ++i) {
        const char* t = ctype(d.slot_prec.at(i));
        const std::string q = std::string("((const ") + t + "*)a.p[" + num(nout + i) + "])";
        s += std::string("    ") + t + " v" + num(i) + "[E];\n";
        s += "    if constexpr (E == 4) fvb_ld4(" + q + " + i0, v" + num(i) + ");\n";
        s += "    else v" + num(i) + "[0] = " + q + "[i0];\n";
    }
    // shared subexpressions, once per element
    std::vector<bool> done(d.nodes.size(), false);
    std::vector<int> shared;
    for (int r : d.roots) e.post(r, [&](int x) { return e.owner[x] == -2; }, done, shared);
    for (int idx : shared)
        s += std::string("    ") + ctype(d.nodes[idx].prec) + " s" + num(idx) + "[E];\n";
    if (!shared.empty()) {
        s += "#pragma unroll\n    for (int k = 0; k < E; ++k) {\n";
        for (int idx : shared) s += "        s" + num(idx) + "[k] = " + e.op(idx) + ";\n";
        s += "    }\n";
    }
    // each item: its private subtree, then the store
    for (int j = 0; j < nout; ++j) {
        const char* t = ctype(d.dest_prec[j]);
        const std::string o = std::string("((") + t + "*)a.p[" + num(j) + "])";
        s += "    {\n        " + std::string(t) + " w[E];\n";
        s += "#pragma unroll\n        for (int k = 0; k < E; ++k) {\n";
        std::vector<bool> seen(d.nodes.size(), false);
        std::vector<int> priv;
        e.post(d.roots[j], [&](int x) { return e.owner[x] == j; }, seen, priv);
        for (int idx : priv)
            s += std::string("            const ") + ctype(d.nodes[idx].prec) + " p" + num(idx) +
                 " = " + e.op(idx) + ";\n";
        s += "            w[k] = " + e.as(d.dest_prec[j], d.roots[j]) + ";\n        }\n";
        s += "        if constexpr (E == 4) fvb_st4(" + o + " + i0, w);\n";
        s += "        else " + o + "[i0] = w[0];\n    }\n";
    }
    s += "}\n";

    s += "extern \"C\" __global__ void __launch_bounds__(" + T + ", " + num(minb) +
         ") fvb_gen(const FvbArgs a, const fvb_u64 n, const int vec)\n{\n";
    // vec == 2 (small ranges): one element per thread, spread over many
    // small CTAs; every plane 4-element aligned (vec == 1): 4 consecutive
    // elements per thread with one wide access per plane; otherwise 4
    // elements strided by the CTA
    s += "    if (vec == 2) {\n";
    s += "        const fvb_u64 i = (fvb_u64)blockIdx.x * blockDim.x + threadIdx.x;\n";
    s += "        if (i < n) fvb_tile<1>(a, i);\n        return;\n    }\n";
    s += "    if (vec) {\n";
    s += "        const fvb_u64 i0 = ((fvb_u64)blockIdx.x * " + T + "ull + threadIdx.x) * 4ull;\n";
    s += "        if (i0 + 4ull <= n) {\n            fvb_tile<4>(a, i0);\n            return;\n"
         "        }\n";
    s += "        for (fvb_u64 i = i0; i < n; ++i) fvb_tile<1>(a, i);\n        return;\n    }\n";
    s += "    const fvb_u64 base = (fvb_u64)blockIdx.x * " + num(kThreads * kPerThread) +
         "ull + threadIdx.x;\n";
    s += "#pragma unroll\n    for (int u = 0; u < " + num(kPerThread) + "; ++u) {\n";
    s += "        const fvb_u64 i = base + (fvb_u64)u * " + T + "ull;\n";
    s += "        if (i < n) fvb_tile<1>(a, i);\n    }\n}\n";
    *src = s;
    if (dag_out) *dag_out = std::move(d);
    return true;
}

// ---- NVRTC, loaded at run time ---------------------------------------------------

struct Nvrtc {
    bool ok = false;
    std::string why;
    decltype(&nvrtcCreateProgram) create = nullptr;
    decltype(&nvrtcCompileProgram) compile = nullptr;
    decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
    decltype(&nvrtcGetProgramLog) log = nullptr;
    decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
    decltype(&nvrtcGetCUBIN) cubin = nullptr;
    decltype(&nvrtcDestroyProgram) destroy = nullptr;
    int major = 0, minor = 0;
};

const Nvrtc& nvrtc() {
    static const Nvrtc lib = [] {
        Nvrtc n;
        void* h = nullptr;
        // The toolkit's own NVRTC first (the one matching the nvcc that built
        // this library): a host process may already hold an older
        // libnvrtc.so.12 (torch bundles one) whose ptxas lacks sm_100a's
        // 256-bit accesses; an explicit path loads ours beside it.
        for (const char* name : {FVB_CUDA_LIB64 "/libnvrtc.so.12", "libnvrtc.so.12",
                                 "libnvrtc.so"}) {
            h = dlopen(name, RTLD_NOW | RTLD_LOCAL);
            if (h) break;
        }
        if (!h) {
            n.why = "libnvrtc.so.12 not found";
            return n;
        }
        n.create = reinterpret_cast<decltype(n.create)>(dlsym(h, "nvrtcCreateProgram"));
        n.compile = reinterpret_cast<decltype(n.compile)>(dlsym(h, "nvrtcCompileProgram"));
        n.log_size = reinterpret_cast<decltype(n.log_size)>(dlsym(h, "nvrtcGetProgramLogSize"));
        n.log = reinterpret_cast<decltype(n.log)>(dlsym(h, "nvrtcGetProgramLog"));
        n.cubin_size = reinterpret_cast<decltype(n.cubin_size)>(dlsym(h, "nvrtcGetCUBINSize"));
        n.cubin = reinterpret_cast<decltype(n.cubin)>(dlsym(h, "nvrtcGetCUBIN"));
        n.destroy = reinterpret_cast<decltype(n.destroy)>(dlsym(h, "nvrtcDestroyProgram"));
        n.ok = n.create && n.compile && n.log_size && n.log && n.cubin_size && n.cubin && n.destroy;
        if (auto ver = reinterpret_cast<decltype(&nvrtcVersion)>(dlsym(h, "nvrtcVersion")))
            ver(&n.major, &n.minor);
        if (!n.ok) n.why = "libnvrtc lacks a required symbol";
        return n;
    }();
    return lib;
}

fvb_status compile(const std::string& src, std::vector<char>* image, bool* spilled) {
    const Nvrtc& nv = nvrtc();
    if (!nv.ok) return fail(FVB_EUNSUPPORTED, "general lowering unavailable: " + nv.why);
    nvrtcProgram prog;
    if (nv.create(&prog, src.c_str(), "fvb_gen.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS)
        return fail(FVB_EUNSUPPORTED, "nvrtcCreateProgram failed");
    const char* opts[] = {"--gpu-architecture=sm_100a", "--fmad=false", "--prec-div=true",
                          "--prec-sqrt=true", "--ftz=false", "--std=c++17", "-default-device",
                          "--ptxas-options=-v"};
    const nvrtcResult rc = nv.compile(prog, int(sizeof(opts) / sizeof(opts[0])), opts);
    size_t n = 0;
    nv.log_size(prog, &n);
    std::string log(n, '\0');
    if (n) nv.log(prog, &log[0]);
    if (rc != NVRTC_SUCCESS) {
        nv.destroy(&prog);
        return fail(FVB_EUNSUPPORTED, "NVRTC compile failed: " + log.substr(0, 400));
    }
    // ptxas -v: "N bytes spill stores"
    *spilled = false;
    for (size_t at = 0; (at = log.find(" bytes spill stores", at)) != std::string::npos; ++at) {
        size_t b = at;
        while (b > 0 && log[b - 1] >= '0' && log[b - 1] <= '9') --b;
        if (b < at && std::atol(log.c_str() + b) > 0) *spilled = true;
    }
    size_t bytes = 0;
    nv.cubin_size(prog, &bytes);
    image->resize(bytes);
    nv.cubin(prog, image->data());
    nv.destroy(&prog);
    return FVB_OK;
}

// ---- the on-disk image cache -------------------------------------------------------
//
// One file per compiled source: <dir>/<hash>.cubin holding a header, the
// exact source text and NVRTC version it was built from (checked on read, so
// a hash collision or a changed emitter or toolkit only misses), the ptxas
// spill verdict and the image.  <dir> is $FVB_CACHE_DIR, else
// $XDG_CACHE_HOME/fvb, else $HOME/.cache/fvb; FVB_CACHE_DIR=off disables it.
// Files are written to a temporary name and renamed, so concurrent processes
// never read a partial image.  Any I/O failure only means a recompile.

constexpr char kCacheMagic[8] = {'F', 'V', 'B', 'C', 'U', 'B', '1', '\0'};

std::string cache_dir() {
    const char* v = std::getenv("FVB_CACHE_DIR");
    if (v) return std::strcmp(v, "off") == 0 || !*v ? std::string() : std::string(v);
    if (const char* x = std::getenv("XDG_CACHE_HOME"); x && *x) return std::string(x) + "/fvb";
    if (const char* h = std::getenv("HOME"); h && *h) return std::string(h) + "/.cache/fvb";
    return std::string();
}

std::string cache_tag(const std::string& src) {
    const Nvrtc& nv = nvrtc();
    return "nvrtc " + std::to_string(nv.major) + "." + std::to_string(nv.minor) + "\n" + src;
}

std::string cache_path(const std::string& dir, const std::string& tag) {
    char name[40];
    std::snprintf(name, sizeof name, "/%016zx.cubin", std::hash<std::string>()(tag));
    return dir + name;
}

bool read_all(const std::string& path, std::string* out) {
    FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) return false;
    char buf[1 << 16];
    size_t got;
    out->clear();
    while ((got = std::fread(buf, 1, sizeof buf, f)) > 0) out->append(buf, got);
    const bool ok = !std::ferror(f);
    std::fclose(f);
    return ok;
}

bool cache_get(const std::string& src, std::vector<char>* image, bool* spilled) {
    const std::string dir = cache_dir();
    if (dir.empty()) return false;
    const std::string tag = cache_tag(src);
    std::string blob;
    if (!read_all(cache_path(dir, tag), &blob)) return false;
    // magic | u64 tag length | tag | u8 spilled | u64 image length | image
    size_t at = 0;
    auto take = [&](void* dst, size_t n) {
        if (blob.size() - at < n) return false;
        std::memcpy(dst, blob.data() + at, n);
        at += n;
        return true;
    };
    char magic[8];
    uint64_t tlen = 0, ilen = 0;
    uint8_t sp = 0;
    if (!take(magic, 8) || std::memcmp(magic, kCacheMagic, 8) || !take(&tlen, 8) ||
        tlen != tag.size() || blob.compare(at, tlen, tag) != 0)
        return false;
    at += tlen;
    if (!take(&sp, 1) || !take(&ilen, 8) || ilen == 0 || blob.size() - at != ilen) return false;
    image->assign(blob.data() + at, blob.data() + at + ilen);
    *spilled = sp != 0;
    return true;
}

void cache_put(const std::string& src, const std::vector<char>& image, bool spilled) {
    const std::string dir = cache_dir();
    if (dir.empty() || image.empty()) return;
    // mkdir -p
    for (size_t at = 1; at <= dir.size(); ++at)
        if (at == dir.size() || dir[at] == '/') {
            const std::string part = dir.substr(0, at);
            if (::mkdir(part.c_str(), 0755) != 0 && errno != EEXIST) return;
        }
    const std::string tag = cache_tag(src);
    const std::string path = cache_path(dir, tag);
    const std::string tmp = path + ".tmp." + std::to_string(::getpid());
    FILE* f = std::fopen(tmp.c_str(), "wb");
    if (!f) return;
    const uint64_t tlen = tag.size(), ilen = image.size();
    const uint8_t sp = spilled ? 1 : 0;
    bool ok = std::fwrite(kCacheMagic, 1, 8, f) == 8 && std::fwrite(&tlen, 8, 1, f) == 1 &&
              std::fwrite(tag.data(), 1, tlen, f) == tlen && std::fwrite(&sp, 1, 1, f) == 1 &&
              std::fwrite(&ilen, 8, 1, f) == 1 &&
              std::fwrite(image.data(), 1, ilen, f) == ilen;
    ok = std::fclose(f) == 0 && ok;
    if (!ok || std::rename(tmp.c_str(), path.c_str()) != 0) std::remove(tmp.c_str());
}

fvb_status compile_cached(const std::string& src, std::vector<char>* image, bool* spilled) {
    if (cache_get(src, image, spilled)) return FVB_OK;
    if (fvb_status st = compile(src, image, spilled)) return st;
    cache_put(src, *image, *spilled);
    return FVB_OK;
}

// Emit and compile a key: 256-bit accesses and a 2-CTA/SM register cap
// first; without the cap when the tree would spill under it; 128-bit
// accesses when the NVRTC in use predates sm_100's 256-bit ones.
int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v && *v ? std::atoi(v) : dflt;
}

fvb_status build(const char* key, KDag* d, std::vector<char>* image, int* minb_out) {
    fvb_status last = FVB_EUNSUPPORTED;
    const int forced = env_int("FVB_LOWER_MINB", 0);  // tuning experiments only
    // Blocks with many outputs keep more live state than the 2-CTA/SM
    // register cap allows (the hand-written Jacobians spill under it too):
    // they start without the cap, which saves a compile on first use.
    std::string probe;
    if (!emit(key, &probe, d, true, 2))
        return fail(FVB_EUNSUPPORTED, std::string("not a loweable structural key: ") +
                                          std::string(key).substr(0, 160));
    const bool big = d && d->roots.size() > 24;
    for (bool wide : {true, false}) {
        for (int minb : {2, 1}) {
            if (forced && minb != forced) continue;
            if (!forced && big && minb == 2) continue;
            std::string src;
            if (!emit(key, &src, d, wide, minb))
                return fail(FVB_EUNSUPPORTED, std::string("not a loweable structural key: ") +
                                                  std::string(key).substr(0, 160));
            bool spilled = false;
            last = compile_cached(src, image, &spilled);
            if (env_int("FVB_LOWER_DEBUG", 0))
                std::fprintf(stderr, "[fvb lower] %016zx wide=%d minb=%d status=%d spilled=%d %s\n",
                             std::hash<std::string>()(key), int(wide), minb, int(last),
                             int(spilled), last ? fvb_last_error() : "");
            if (last != FVB_OK) break;  // try the 128-bit form
            *minb_out = minb;
            if (!spilled || minb == 1 || forced) return FVB_OK;
        }
    }
    return last;
}

// ---- the per-key cache and the launch entry -----------------------------------

struct Gen {
    std::string key;
    cudaLibrary_t lib = nullptr;
    cudaKernel_t kernel = nullptr;
    std::vector<char> arg_prec;  // 's'/'d' per argument slot (outputs, then leaves)
    uint32_t nout = 0, nin = 0;
    int minb = 2;                // resident CTAs per SM the kernel was compiled for
};

std::mutex g_mu;
std::map<std::string, std::unique_ptr<Gen>>& cache() {
    static std::map<std::string, std::unique_ptr<Gen>> c;
    return c;
}

struct LaunchArgs {
    void* p[kMaxArgs];
};

fvb_status gen_entry(const fvb_kernel* k, uint64_t begin, uint64_t end, void* const* args,
                     void* stream) {
    if (!k || !k->impl || !args) return fail(FVB_EARG, "NULL kernel or argument block");
    if (end < begin) return fail(FVB_EARG, "end < begin");
    const Gen* g = static_cast<const Gen*>(k->impl);
    uint64_t n = end - begin;
    if (n == 0) return FVB_OK;
    LaunchArgs la;
    std::memset(&la, 0, sizeof la);
    for (uint32_t i = 0; i < g->nout + g->nin; ++i) {
        if (!args[i]) return fail(FVB_EARG, "NULL argument slot");
        const size_t w = g->arg_prec[i] == 's' ? sizeof(float) : sizeof(double);
        if (reinterpret_cast<uintptr_t>(args[i]) % w)
            return fail(FVB_EALIGN, "argument plane is not element-aligned");
        la.p[i] = static_cast<char*>(args[i]) + begin * w;
    }
    // 4-element accesses when every plane (after the begin offset) allows them
    static const int allow_vec = env_int("FVB_LOWER_VEC", 1);
    int vec = allow_vec;
    for (uint32_t i = 0; i < g->nout + g->nin; ++i) {
        const size_t w = g->arg_prec[i] == 's' ? sizeof(float) : sizeof(double);
        if (reinterpret_cast<uintptr_t>(la.p[i]) % (4 * w)) vec = 0;
    }
    // Small ranges (fewer elements than 4 per thread of one 256-thread CTA per
    // SM): one element per thread in 64-thread CTAs, so n = 1024 runs on 16
    // SMs instead of one (as launch_op does for the hand-written kernels).
    unsigned threads = kThreads;
    uint64_t per = uint64_t(kThreads) * kPerThread;
    if (n < uint64_t(device_sm_count()) * kThreads * kPerThread) {
        vec = 2;
        threads = 64;
        per = 64;
    }
    const uint64_t grid = (n + per - 1) / per;
    if (grid > 0x7fffffffull) return fail(FVB_EARG, "range too large for one launch");
    void* params[] = {&la, &n, &vec};
    const cudaError_t e =
        cudaLaunchKernel(reinterpret_cast<const void*>(g->kernel), dim3(unsigned(grid)),
                         dim3(threads), params, 0, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? FVB_OK : cuda_fail(e, "lowered kernel launch");
}

}  // namespace

fvb_status lower_lookup(const char* key, fvb_kernel* out) {
    std::lock_guard<std::mutex> lock(g_mu);
    auto it = cache().find(key);
    if (it == cache().end()) {
        KDag d;
        std::vector<char> image;
        int minb = 2;
        if (fvb_status st = build(key, &d, &image, &minb)) return st;
        auto g = std::make_unique<Gen>();
        g->minb = minb;
        g->key = key;
        g->nout = uint32_t(d.roots.size());
        g->nin = uint32_t(d.slot_prec.size());
        for (char p : d.dest_prec) g->arg_prec.push_back(p);
        for (uint32_t i = 0; i < g->nin; ++i) g->arg_prec.push_back(d.slot_prec.at(int(i)));
        cudaError_t e = cudaLibraryLoadData(&g->lib, image.data(), nullptr, nullptr, 0, nullptr,
                                            nullptr, 0);
        if (e == cudaSuccess) e = cudaLibraryGetKernel(&g->kernel, g->lib, "fvb_gen");
        if (e != cudaSuccess) return cuda_fail(e, "loading the lowered kernel");
        it = cache().emplace(key, std::move(g)).first;
    }
    const Gen* g = it->second.get();
    fvb_kernel k;
    std::memset(&k, 0, sizeof k);
    k.fn = gen_entry;
    k.reduce = nullptr;
    k.n_outputs = g->nout;
    k.n_inputs = g->nin;
    k.n_consts = 0;
    k.prec = g->arg_prec.empty() || g->arg_prec[0] == 'd' ? 1 : 0;
    k.dim = 0;
    // A lowered kernel has no canonical input order: it takes its leaves in
    // the key's slot order, which is exactly the jit_args order.
    for (int i = 0; i < 8; ++i) k.in_slot[i] = -1;
    std::snprintf(k.name, sizeof k.name, "gen:%016zx:m%d", std::hash<std::string>()(g->key),
                  g->minb);
    k.impl = g;
    *out = k;
    return FVB_OK;
}

}  // namespace fvb

using namespace fvb;

extern "C" {

fvb_status fvb_emit_source(const char* key, char* buf, size_t cap, size_t* len) {
    return guarded([&]() -> fvb_status {
        if (!key) return fail(FVB_EARG, "NULL key");
        std::string src;
        if (!emit(key, &src, nullptr))
            return fail(FVB_EUNSUPPORTED, "not a loweable structural key");
        if (len) *len = src.size();
        if (buf && cap) {
            const size_t n = src.size() < cap - 1 ? src.size() : cap - 1;
            std::memcpy(buf, src.data(), n);
            buf[n] = '\0';
        }
        return FVB_OK;
    });
}

fvb_status fvb_nvrtc_compile(const char* key, size_t* cubin_bytes) {
    return guarded([&]() -> fvb_status {
        if (!key) return fail(FVB_EARG, "NULL key");
        KDag d;
        std::vector<char> image;
        int minb = 2;
        if (fvb_status st = build(key, &d, &image, &minb)) return st;
        if (cubin_bytes) *cubin_bytes = image.size();
        return FVB_OK;
    });
}

}  // extern "C"
