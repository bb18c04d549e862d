// Device array descriptors, view descriptors and the symbolic affine forms they come from
// (include/pencil_b200.h §10).
//
// a11 — views from affine forms.  The reference's analyzer extracts, per array access,
// index = scale * i + offset for each loop variable i (affine_form / scan_affine_*,
// depanalysis.cpp:163-285) — with CONSTANT coefficients only: a symbolic `lda` makes the form
// non-affine there (:169).  A strided VOBLA view needs exactly those symbolic coefficients
// (gemv_t: A[i * lda + j], x[i * incx], y[j * incy]), so the extraction here keeps coefficients
// and offsets as polynomials over the function's scalar parameters, and evaluates them under a
// call's bindings into numeric strides / offsets.  The result is a pencil_view (base, offset,
// extents, strides) that the kernels take instead of loose lda / incx / incy scalars.
//
// a7 — array residency.  The reference binds arrays by name in a host store (set_array / arrays(),
// interp.hpp:40-43, array_storage interp.cpp:124-138).  Here an array is a descriptor: element
// type, extent, a shard spec (element ranges, one per GPU / rank), the device pointer of every
// shard known to this process (its own, and peers' through NVLink mappings), and an optional host
// mirror; the named-array layer of the Interpreter mirror (dispatch.cpp) and the multi-GPU shard
// classes (dist.py) keep their arrays in these.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/pencil_b200.h"
#include "kernels.h"
#include "pencil_front.hpp"

int pencil_internal_fail(int status, const char* msg);  // runtime.cpp
int pencil_internal_ok();

namespace {

int fail(int st, const std::string& m) { return pencil_internal_fail(st, m.c_str()); }

// the PENCIL fixtures (paper_1302_5586_b200/pencil/*.pencil.c), embedded at build time
struct FixtureSrc {
    const char* name;
    const char* text;
};
const FixtureSrc kFixtures[] = {
#include "fixtures_src.inc"
};

}  // namespace

#include "affine.hpp"
using namespace affine_forms;

namespace {

struct AccessRec {
    std::string array;
    bool write = false;
    Aff form;
    std::vector<const pf::Stmt*> nest;  // enclosing for-loops, outermost first
};

void collect_accesses(const pf::Func& f, std::vector<AccessRec>& out) {
    std::map<std::string, int> params, arrays;
    for (size_t i = 0; i < f.params.size(); i++) {
        if (f.params[i].kind == pf::Param::Scalar) params[f.params[i].name] = (int)i;
        else arrays[f.params[i].name] = (int)i;
    }
    std::vector<const pf::Stmt*> nest;
    auto names = [&]() {
        std::vector<std::string> v;
        for (const auto* s : nest) v.push_back(s->name);
        return v;
    };
    std::function<void(const pf::Expr&)> ex = [&](const pf::Expr& e) {
        for (const auto& a : e.args) ex(*a);
        if (e.kind == pf::Expr::Index && arrays.count(e.name) && e.args.size() == 1)
            out.push_back({e.name, false, affine(*e.args[0], names(), params), nest});
    };
    std::function<void(const pf::Stmt&)> st = [&](const pf::Stmt& s) {
        switch (s.kind) {
            case pf::Stmt::Block:
                for (const auto& c : s.body) st(*c);
                break;
            case pf::Stmt::Decl:
                if (s.rhs) ex(*s.rhs);
                break;
            case pf::Stmt::Assign:
                ex(*s.rhs);
                if (s.lhs->kind == pf::Expr::Index) {
                    for (const auto& a : s.lhs->args) ex(*a);
                    if (arrays.count(s.lhs->name) && s.lhs->args.size() == 1) {
                        Aff a = affine(*s.lhs->args[0], names(), params);
                        if (s.aop != pf::AOp::Set) out.push_back({s.lhs->name, false, a, nest});
                        out.push_back({s.lhs->name, true, a, nest});
                    }
                }
                break;
            case pf::Stmt::For:
                ex(*s.lo);
                ex(*s.hi);
                nest.push_back(&s);
                st(*s.loop_body);
                nest.pop_back();
                break;
            case pf::Stmt::While:
                ex(*s.cond);
                st(*s.loop_body);
                break;
            case pf::Stmt::If:
                ex(*s.cond);
                st(*s.then_s);
                if (s.else_s) st(*s.else_s);
                break;
            case pf::Stmt::CallS: ex(*s.call); break;
            case pf::Stmt::Return:
                if (s.rhs) ex(*s.rhs);
                break;
            case pf::Stmt::Labeled: st(*s.loop_body); break;
            default: break;
        }
    };
    if (f.body) st(*f.body);
}

// loop bound under the binding: affine in the parameters (and outer loop variables at 0)
bool bound(const pf::Expr& e, const std::map<std::string, int>& params, const std::map<std::string, long long>& env,
           long long& out) {
    Aff a = affine(e, {}, params);
    return a.ok && peval(a.c, env, out);
}

// ------------------------------------------------------------------ array descriptors
struct Shard {
    long long lo = 0, hi = 0;  // element range [lo, hi)
    int device = -1;           // -1: not attached in this process
    void* ptr = nullptr;       // device pointer of element lo (own memory or a peer mapping)
};

}  // namespace

struct pencil_array {
    int dtype = PENCIL_FLOAT32;
    long long n = 0;
    std::vector<Shard> shards;  // one entry: replicated / single-GPU
    void* host = nullptr;       // host mirror (caller-owned)
    std::mutex mu;
};

namespace {
size_t esize(int dt) {
    switch (dt) {
        case PENCIL_INT32:
        case PENCIL_FLOAT32: return 4;
        case PENCIL_FLOAT64: return 8;
        case PENCIL_UINT8: return 1;
    }
    return 0;
}
}  // namespace

extern "C" {

const char* pencil_fixture_source(const char* file) {
    if (!file) return nullptr;
    for (const auto& fx : kFixtures)
        if (!strcmp(fx.name, file)) return fx.text;
    return nullptr;
}

int pencil_affine_accesses(const char* source, const char* fn, int nbind, const char* const* names,
                           const long long* values, pencil_access_form* out, int cap) {
    if (!source || !fn || nbind < 0 || (nbind && (!names || !values))) return fail(PENCIL_E_ARG, "E-ARG: bad argument"), -1;
    // parsed units cached by source text (the fixtures are parsed once per process)
    static std::mutex mu;
    static std::map<std::string, std::unique_ptr<pf::Unit>> units;
    const pf::Unit* up = nullptr;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto& slot = units[source];
        if (!slot) {
            auto nu = std::make_unique<pf::Unit>();
            std::string err;
            if (!pf::parse_unit(source, *nu, err)) {
                units.erase(source);
                return fail(PENCIL_E_ARG, "E-SYNTAX: " + err), -1;
            }
            slot = std::move(nu);
        }
        up = slot.get();
    }
    const pf::Func* f = up->find(fn);
    if (!f) return fail(PENCIL_E_ARG, std::string("E-ARG: no function named '") + fn + "'"), -1;
    std::map<std::string, int> params;
    for (size_t i = 0; i < f->params.size(); i++)
        if (f->params[i].kind == pf::Param::Scalar) params[f->params[i].name] = (int)i;
    std::map<std::string, long long> env;
    for (int i = 0; i < nbind; i++) env[names[i]] = values[i];
    std::vector<AccessRec> recs;
    collect_accesses(*f, recs);
    int k = 0;
    for (const auto& r : recs) {
        if (k < cap && out) {
            pencil_access_form& o = out[k];
            memset(&o, 0, sizeof o);
            snprintf(o.array, sizeof o.array, "%s", r.array.c_str());
            o.is_write = r.write;
            o.nloops = (int)std::min<size_t>(r.nest.size(), 8);
            o.affine = r.form.ok;
            std::string form;
            for (int d = 0; d < o.nloops; d++) {
                const pf::Stmt& L = *r.nest[d];
                snprintf(o.loop[d], sizeof o.loop[d], "%s", L.name.c_str());
                long long v = 0;
                o.lo[d] = bound(*L.lo, params, env, v) ? v : 0;
                o.hi[d] = bound(*L.hi, params, env, v) ? v : -1;
                auto it = r.form.coef.find(L.name);
                if (it != r.form.coef.end()) {
                    if (!peval(it->second, env, o.stride[d])) o.affine = 0;
                    const std::string ps = pstr(it->second);
                    form += (form.empty() ? "" : " + ") + L.name + (ps == "1" ? "" : "*" + (it->second.size() > 1 ? "(" + ps + ")" : ps));
                }
            }
            if (r.form.ok) {
                if (!peval(r.form.c, env, o.offset)) o.affine = 0;
                if (!r.form.c.empty()) {
                    const std::string cs = pstr(r.form.c);
                    if (form.empty()) form = cs;
                    else form += cs[0] == '-' ? " - " + cs.substr(1) : " + " + cs;
                }
                snprintf(o.form, sizeof o.form, "%s", form.empty() ? "0" : form.c_str());
            } else {
                snprintf(o.form, sizeof o.form, "%s", "(not affine)");
            }
        }
        k++;
    }
    pencil_internal_ok();
    return k;
}

int pencil_view_slice(const pencil_view* v, int dim, long long lo, long long hi, pencil_view* out) {
    if (!v || !out || dim < 0 || dim >= v->rank || lo < 0 || hi < lo || hi > v->extent[dim])
        return fail(PENCIL_E_ARG, "E-ARG: slice out of the view");
    pencil_view r = *v;
    r.offset = v->offset + lo * v->stride[dim];
    r.extent[dim] = hi - lo;
    *out = r;
    return pencil_internal_ok();
}

// ---- array descriptors
pencil_array_t pencil_array_create(int dtype, long long n, int nshards, const long long* bounds) {
    if (!esize(dtype) || n < 0 || nshards < 1 || nshards > 64) {
        fail(PENCIL_E_ARG, "E-ARG: bad array descriptor");
        return nullptr;
    }
    auto* a = new pencil_array();
    a->dtype = dtype;
    a->n = n;
    a->shards.resize(nshards);
    for (int s = 0; s < nshards; s++) {
        a->shards[s].lo = bounds ? bounds[s] : (s == 0 ? 0 : n);
        a->shards[s].hi = bounds ? bounds[s + 1] : n;
        if (a->shards[s].lo < 0 || a->shards[s].hi < a->shards[s].lo || a->shards[s].hi > n ||
            (s > 0 && a->shards[s].lo != a->shards[s - 1].hi)) {
            delete a;
            fail(PENCIL_E_ARG, "E-ARG: shard bounds must partition [0, n) in order");
            return nullptr;
        }
    }
    if (bounds && (bounds[0] != 0 || bounds[nshards] != n)) {
        delete a;
        fail(PENCIL_E_ARG, "E-ARG: shard bounds must start at 0 and end at n");
        return nullptr;
    }
    pencil_internal_ok();
    return a;
}

void pencil_array_destroy(pencil_array_t a) { delete a; }

int pencil_array_attach(pencil_array_t a, int shard, int device, void* ptr) {
    if (!a || shard < 0 || shard >= (int)a->shards.size()) return fail(PENCIL_E_ARG, "E-ARG: no such shard");
    std::lock_guard<std::mutex> lk(a->mu);
    a->shards[shard].device = device;
    a->shards[shard].ptr = ptr;
    return pencil_internal_ok();
}

int pencil_array_set_mirror(pencil_array_t a, void* host) {
    if (!a) return fail(PENCIL_E_ARG, "E-ARG: null array");
    a->host = host;
    return pencil_internal_ok();
}

int pencil_array_info(pencil_array_t a, int* dtype, long long* n, int* nshards, void** host) {
    if (!a) return fail(PENCIL_E_ARG, "E-ARG: null array");
    if (dtype) *dtype = a->dtype;
    if (n) *n = a->n;
    if (nshards) *nshards = (int)a->shards.size();
    if (host) *host = a->host;
    return pencil_internal_ok();
}

int pencil_array_shard(pencil_array_t a, int shard, long long* lo, long long* hi, int* device, void** ptr) {
    if (!a || shard < 0 || shard >= (int)a->shards.size()) return fail(PENCIL_E_ARG, "E-ARG: no such shard");
    std::lock_guard<std::mutex> lk(a->mu);
    const Shard& s = a->shards[shard];
    if (lo) *lo = s.lo;
    if (hi) *hi = s.hi;
    if (device) *device = s.device;
    if (ptr) *ptr = s.ptr;
    return pencil_internal_ok();
}

int pencil_array_owner(pencil_array_t a, long long index) {
    if (!a || index < 0 || index >= a->n) return -1;
    int lo = 0, hi = (int)a->shards.size() - 1;
    while (lo < hi) {  // shards are ordered and contiguous: binary search on the starts
        const int mid = (lo + hi + 1) / 2;
        if (a->shards[mid].lo <= index) lo = mid;
        else hi = mid - 1;
    }
    while (lo < (int)a->shards.size() - 1 && a->shards[lo].hi <= index) lo++;  // skip empty shards
    return lo;
}

// host mirror <-> an attached shard (its element range), stream-ordered
int pencil_array_sync(pencil_array_t a, int shard, int to_device, pencil_stream_t s) {
    if (!a || shard < 0 || shard >= (int)a->shards.size()) return fail(PENCIL_E_ARG, "E-ARG: no such shard");
    const Shard& sh = a->shards[shard];
    if (!a->host || !sh.ptr) return fail(PENCIL_E_ARG, "E-ARG: shard not attached or no host mirror");
    const size_t es = esize(a->dtype), bytes = (size_t)(sh.hi - sh.lo) * es;
    char* h = (char*)a->host + (size_t)sh.lo * es;
    cudaError_t e = to_device ? cudaMemcpyAsync(sh.ptr, h, bytes, cudaMemcpyHostToDevice, (cudaStream_t)s)
                              : cudaMemcpyAsync(h, sh.ptr, bytes, cudaMemcpyDeviceToHost, (cudaStream_t)s);
    if (e != cudaSuccess) return fail(PENCIL_E_CUDA, std::string("E-CUDA: array sync: ") + cudaGetErrorString(e));
    return pencil_internal_ok();
}

// the view of a shard's piece: rank 1, extent hi - lo, stride 1, base = the shard's pointer
int pencil_array_view(pencil_array_t a, int shard, pencil_view* out) {
    if (!a || !out || shard < 0 || shard >= (int)a->shards.size()) return fail(PENCIL_E_ARG, "E-ARG: no such shard");
    const Shard& s = a->shards[shard];
    memset(out, 0, sizeof *out);
    out->base = s.ptr;
    out->dtype = a->dtype;
    out->rank = 1;
    out->extent[0] = s.hi - s.lo;
    out->stride[0] = 1;
    return pencil_internal_ok();
}

}  // extern "C"
