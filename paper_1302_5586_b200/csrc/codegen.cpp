#include "codegen.hpp"

#include <dlfcn.h>

#include <mutex>

namespace pcg {

const char* kPreludeCore = R"CUDA(
typedef long long ll;
typedef unsigned long long ull;
struct V { ll i; double d; int isd; };
struct LArr { V* p; ll n; };
struct Ctx { unsigned* fault; ull* rng; const ll* rseq; ull* rpos; ll rseq_n; ull* tr; };
// tr (JIT trace mode, Interpreter::enable_trace, interp.hpp:45): tr[0] = records, tr[1] = capacity,
// record r = (array id << 1 | is_write, index) at tr[2 + 2r]; null when tracing is off
#define F_OOB_LOAD 1u
#define F_OOB_STORE 2u
#define F_DIV0 4u
#define F_MOD0 8u
#define F_NONINT 16u
#define F_DBLSTORE 32u
#define F_EMPTY 64u
#define F_BUDGET 128u
#define STEP_BUDGET 100000000ll  // the interpreter's step_budget_ (interp.hpp:71), per thread here
static __device__ __forceinline__ V VI(ll x) { V v; v.i = x; v.d = 0.0; v.isd = 0; return v; }
static __device__ __forceinline__ V VD(double x) { V v; v.i = 0; v.d = x; v.isd = 1; return v; }
static __device__ __forceinline__ void fault(const Ctx& c, unsigned b) { atomicOr(c.fault, b); }
static __device__ __forceinline__ double as_d(V v) { return v.isd ? v.d : (double)v.i; }
static __device__ __forceinline__ ll as_i(const Ctx& c, V v) {
    if (!v.isd) return v.i;
    ll r = (ll)v.d;
    if ((double)r != v.d) fault(c, F_NONINT);
    return r;
}
static __device__ __forceinline__ bool truth(V v) { return as_d(v) != 0.0; }
static __device__ __forceinline__ V op_add(V a, V b) { return (a.isd | b.isd) ? VD(as_d(a) + as_d(b)) : VI((ll)((ull)a.i + (ull)b.i)); }
static __device__ __forceinline__ V op_sub(V a, V b) { return (a.isd | b.isd) ? VD(as_d(a) - as_d(b)) : VI((ll)((ull)a.i - (ull)b.i)); }
static __device__ __forceinline__ V op_mul(V a, V b) { return (a.isd | b.isd) ? VD(as_d(a) * as_d(b)) : VI((ll)((ull)a.i * (ull)b.i)); }
static __device__ __forceinline__ V op_div(const Ctx& c, V a, V b) {
    if (a.isd | b.isd) {
        double y = as_d(b);
        if (y == 0.0) { fault(c, F_DIV0); return VD(0.0); }
        return VD(as_d(a) / y);
    }
    if (b.i == 0) { fault(c, F_DIV0); return VI(0); }
    if (b.i == -1) return VI((ll)(0ull - (ull)a.i));
    return VI(a.i / b.i);
}
static __device__ __forceinline__ V op_mod(const Ctx& c, V a, V b) {
    ll rb = as_i(c, b);
    if (rb == 0) { fault(c, F_MOD0); return VI(0); }
    ll ra = as_i(c, a);
    if (rb == -1) return VI(0);
    return VI(ra % rb);
}
#define CMP(NAME, OP) \
static __device__ __forceinline__ V NAME(V a, V b) { return (a.isd | b.isd) ? VI((ll)(as_d(a) OP as_d(b))) : VI((ll)(a.i OP b.i)); }
CMP(op_lt, <) CMP(op_le, <=) CMP(op_gt, >) CMP(op_ge, >=) CMP(op_eq, ==) CMP(op_ne, !=)
static __device__ __forceinline__ V op_and(V a, V b) { return VI((ll)(truth(a) && truth(b))); }
static __device__ __forceinline__ V op_or(V a, V b) { return VI((ll)(truth(a) || truth(b))); }
static __device__ __forceinline__ V op_neg(V a) { return a.isd ? VD(-a.d) : VI((ll)(0ull - (ull)a.i)); }
static __device__ __forceinline__ V op_not(V a) { return VI((ll)(as_d(a) == 0.0)); }
static __device__ __forceinline__ V apply(const Ctx& c, int op, V old, V rhs) {
    switch (op) {
        case 1: return op_add(old, rhs);
        case 2: return op_sub(old, rhs);
        case 3: return op_mul(old, rhs);
        case 4: return op_div(c, old, rhs);
    }
    return rhs;
}
static __device__ __forceinline__ V ldl(const Ctx& c, const LArr& a, V idx) {
    ll k = as_i(c, idx);
    if (k < 0 || k >= a.n) { fault(c, F_OOB_LOAD); return VI(0); }
    return a.p[k];
}
static __device__ __forceinline__ void stl(const Ctx& c, const LArr& a, V idx, int op, V rhs) {
    ll k = as_i(c, idx);
    if (k < 0 || k >= a.n) { fault(c, F_OOB_STORE); return; }
    a.p[k] = op == 0 ? rhs : apply(c, op, a.p[k], rhs);
}
static __device__ __forceinline__ V b_rand(const Ctx& c) {
    // Interpreter::next_rand (interp.cpp:249-254): the configured sequence first, then the LCG
    if (c.rpos) {
        const ull p = *c.rpos;
        if (p < (ull)c.rseq_n) { *c.rpos = p + 1; return VI(c.rseq[p]); }
    }
    ull s = *c.rng * 6364136223846793005ull + 1442695040888963407ull;
    *c.rng = s;
    return VI((ll)((s >> 33) & 0x7fffffffull));
}
static __device__ __forceinline__ V b_exp(V a) { return VD(exp(as_d(a))); }
)CUDA";

const char* kArrInt64 = R"CUDA(
struct Arr { ll* p; ll n; int inc; };
static __device__ __forceinline__ V ld(const Ctx& c, const Arr& a, V idx) {
    ll k = as_i(c, idx);
    if (k < 0 || k >= a.n) { fault(c, F_OOB_LOAD); return VI(0); }
    return VI(a.p[k]);
}
static __device__ __forceinline__ void st(const Ctx& c, const Arr& a, V idx, int op, V rhs) {
    ll k = as_i(c, idx);
    if (k < 0 || k >= a.n) { fault(c, F_OOB_STORE); return; }
    if (a.inc && (op == 1 || op == 2)) {  // OP_INC in a parallel loop: commutative integer add
        if (rhs.isd) { fault(c, F_DBLSTORE); return; }
        atomicAdd((ull*)(a.p + k), op == 1 ? (ull)rhs.i : (ull)0 - (ull)rhs.i);
        return;
    }
    V v = op == 0 ? rhs : apply(c, op, VI(a.p[k]), rhs);
    if (v.isd) { fault(c, F_DBLSTORE); v = VI(as_i(c, v)); }
    a.p[k] = v.i;
}
static __device__ __forceinline__ V deref(const Ctx& c, const Arr& a) {
    if (a.n == 0) { fault(c, F_EMPTY); return VI(0); }
    return VI(a.p[0]);
}
)CUDA";

const char* kArrTagged = R"CUDA(
struct Arr { ll* p; unsigned char* tag; ll n; int inc; int id; };
// MemTrace (interp.hpp:17-21): an in-bounds load / store of a store array, in execution order
// (trace mode runs every statement on one device thread, so the order is the interpreter's)
static __device__ __forceinline__ void trace(const Ctx& c, int id, ll k, int w) {
    if (!c.tr) return;
    const ull r = atomicAdd(c.tr, 1ull);
    if (r < c.tr[1]) { c.tr[2 + 2 * r] = ((ull)id << 1) | (ull)w; c.tr[3 + 2 * r] = (ull)k; }
}
static __device__ __forceinline__ V ld(const Ctx& c, const Arr& a, V idx) {
    ll k = as_i(c, idx);
    if (k < 0 || k >= a.n) { fault(c, F_OOB_LOAD); return VI(0); }
    trace(c, a.id, k, 0);
    return a.tag[k] ? VD(__longlong_as_double(a.p[k])) : VI(a.p[k]);
}
static __device__ __forceinline__ void st(const Ctx& c, const Arr& a, V idx, int op, V rhs) {
    ll k = as_i(c, idx);
    if (k < 0 || k >= a.n) { fault(c, F_OOB_STORE); return; }
    trace(c, a.id, k, 1);
    V old = a.tag[k] ? VD(__longlong_as_double(a.p[k])) : VI(a.p[k]);
    V v = op == 0 ? rhs : apply(c, op, old, rhs);
    a.p[k] = v.isd ? __double_as_longlong(v.d) : v.i;
    a.tag[k] = (unsigned char)v.isd;
}
static __device__ __forceinline__ V deref(const Ctx& c, const Arr& a) {
    if (a.n == 0) { fault(c, F_EMPTY); return VI(0); }
    return a.tag[0] ? VD(__longlong_as_double(a.p[0])) : VI(a.p[0]);
}
)CUDA";

namespace {
// ------------------------------------------------------------------ NVRTC (dlopen'd on first use)
typedef int (*nvrtcCreateProgram_t)(void**, const char*, const char*, int, const char* const*, const char* const*);
typedef int (*nvrtcCompileProgram_t)(void*, int, const char* const*);
typedef int (*nvrtcGetSize_t)(void*, size_t*);
typedef int (*nvrtcGetData_t)(void*, char*);
typedef int (*nvrtcDestroyProgram_t)(void**);
typedef const char* (*nvrtcGetErrorString_t)(int);
struct Nvrtc {
    bool ok = false;
    std::string why;
    nvrtcCreateProgram_t create;
    nvrtcCompileProgram_t compile;
    nvrtcGetSize_t log_size, cubin_size;
    nvrtcGetData_t log, cubin;
    nvrtcDestroyProgram_t destroy;
    nvrtcGetErrorString_t errstr;
};
Nvrtc& nvrtc() {
    static Nvrtc n;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnvrtc.so.12", RTLD_NOW | RTLD_LOCAL);
        if (!h) h = dlopen("libnvrtc.so", RTLD_NOW | RTLD_LOCAL);
        if (!h) {
            n.why = "libnvrtc.so.12 not found (needed to compile OP2 kernels)";
            return;
        }
        n.create = (nvrtcCreateProgram_t)dlsym(h, "nvrtcCreateProgram");
        n.compile = (nvrtcCompileProgram_t)dlsym(h, "nvrtcCompileProgram");
        n.log_size = (nvrtcGetSize_t)dlsym(h, "nvrtcGetProgramLogSize");
        n.log = (nvrtcGetData_t)dlsym(h, "nvrtcGetProgramLog");
        n.cubin_size = (nvrtcGetSize_t)dlsym(h, "nvrtcGetCUBINSize");
        n.cubin = (nvrtcGetData_t)dlsym(h, "nvrtcGetCUBIN");
        n.destroy = (nvrtcDestroyProgram_t)dlsym(h, "nvrtcDestroyProgram");
        n.errstr = (nvrtcGetErrorString_t)dlsym(h, "nvrtcGetErrorString");
        n.ok = n.create && n.compile && n.log_size && n.log && n.cubin_size && n.cubin && n.destroy && n.errstr;
        if (!n.ok) n.why = "libnvrtc is missing entry points";
    });
    return n;
}

// compile once per distinct source text (process-wide cache)
}  // namespace

int compile_cubin(const std::string& src, std::vector<char>& cubin, std::string& log) {
    static std::mutex mu;
    static std::map<std::string, std::vector<char>> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(src);
    if (it != cache.end()) {
        cubin = it->second;
        return PENCIL_OK;
    }
    Nvrtc& n = nvrtc();
    if (!n.ok) {
        log = n.why;
        return PENCIL_E_UNSUPPORTED;
    }
    void* prog = nullptr;
    if (n.create(&prog, src.c_str(), "op2_model.cu", 0, nullptr, nullptr) != 0) {
        log = "nvrtcCreateProgram failed";
        return PENCIL_E_CUDA;
    }
    // exact IEEE fp64 (no contraction) and the sm_100a instruction set
    const char* opts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "--fmad=false", "-lineinfo"};
    int rc = n.compile(prog, 4, opts);
    size_t ls = 0;
    n.log_size(prog, &ls);
    log.assign(ls, 0);
    if (ls) n.log(prog, &log[0]);
    if (rc != 0) {
        n.destroy(&prog);
        log = std::string("NVRTC: ") + n.errstr(rc) + "\n" + log;
        return PENCIL_E_CUDA;
    }
    size_t cs = 0;
    n.cubin_size(prog, &cs);
    cubin.resize(cs);
    n.cubin(prog, cubin.data());
    n.destroy(&prog);
    cache[src] = cubin;
    return PENCIL_OK;
}


}  // namespace pcg
