// OP2 mesh loops on the GPU: the reference's mesh-model input (sets, maps,
// dats, kernels, par_loops; core/include/pencil/op2.hpp, docs/op2-input.md) executed on the
// device with the sequential semantics of interpret_op2_reference (core/src/op2.cpp:388-429).
//
//   load     JSON document -> model, validated with the reference's codes and messages
//            (E-OP2-SHAPE / E-OP2-RANGE, load_op2_model op2.cpp:80-190)
//   check    kernels parsed (pencil_front), signature 2m+n (check_kernel_signature,
//            op2.cpp:236-251 -> E-OP2-KERNEL), INC vs WRITE/RW conflicts (E-OP2-CONFLICT)
//   codegen  every kernel function -> a CUDA __device__ function over tagged int64/fp64
//            values that reproduce the interpreter's arithmetic (interp.cpp:7-83: int64 unless
//            a double is involved, C-truncating / and %, faults for division by zero, out of
//            bounds and non-integral indices); one __global__ driver per par_loop binding
//            sizes, dats and map-indexed iteration indices exactly as the reference's lowering
//            (append_driver, op2.cpp:253-345); compiled once per model with NVRTC for sm_100a
//   schedule per par_loop, from the access hints (which the reference's own OpenMP lowering
//            also trusts) and a static scan of the kernel bodies:
//              PARALLEL  one thread per iteration; OP_INC dats take += / -= as 64-bit atomic
//                        adds (integer addition commutes: bit-exact vs the sequential order)
//              LEVELS    a dat written through a map (OP_WRITE / OP_RW) or written directly and
//                        also reached through a map: iterations are levelled on the host so each
//                        touched element sees its accesses in iteration order, one launch per level
//              SERIAL    rand() (a sequential stream), or an OP_INC dat that is also read or
//                        stored non-additively: one device thread runs the loop in order
// Dats live on the device for the model's lifetime; pencil_op2_get_dat copies them back.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/pencil_b200.h"
#include "codegen.hpp"
#include "mini_json.hpp"
#include "pencil_front.hpp"

// hoststage.cpp: pageable host arrays of OP2_STAGE_MIN bytes and more go through the library's
// multi-threaded pinned staging ring (as the drop-in calls' do)
bool host_is_pageable(const void* p);
int staged_h2d_2d(int device, void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t rows,
                  cudaStream_t st);
int staged_d2h_2d(int device, void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t rows,
                  cudaStream_t st);
constexpr size_t OP2_STAGE_MIN = 4u << 20;

int pencil_internal_fail(int status, const char* msg);  // runtime.cpp
int pencil_internal_ok();                                // runtime.cpp

namespace {

int fail(int st, const std::string& m) { return pencil_internal_fail(st, m.c_str()); }

// ------------------------------------------------------------------ model
enum Access { A_READ, A_WRITE, A_RW, A_INC };
const char* access_name(int a) {
    return a == A_READ ? "OP_READ" : a == A_WRITE ? "OP_WRITE" : a == A_RW ? "OP_RW" : "OP_INC";
}

struct Set {
    std::string name;
    long long size = 0;
};
struct Map {
    std::string name, from, to;
    int arity = 1;
    std::vector<long long> table;
};
struct Dat {
    std::string name, set;
    int dim = 1;
    std::vector<long long> data;
};
struct Arg {
    std::string dat, map;  // map empty = direct
    int offset = 0;
    int access = A_READ;
    bool direct() const { return map.empty(); }
};
struct Loop {
    std::string kernel, set;
    std::vector<Arg> args;
};
struct Kernel {
    std::string name, source;
};

struct Model {
    std::vector<Set> sets;
    std::vector<Map> maps;
    std::vector<Dat> dats;
    std::vector<Kernel> kernels;
    std::vector<Loop> loops;
    const Set* set(const std::string& n) const {
        for (auto& s : sets)
            if (s.name == n) return &s;
        return nullptr;
    }
    const Map* map(const std::string& n) const {
        for (auto& m : maps)
            if (m.name == n) return &m;
        return nullptr;
    }
    int dat_index(const std::string& n) const {
        for (size_t i = 0; i < dats.size(); i++)
            if (dats[i].name == n) return (int)i;
        return -1;
    }
    int map_index(const std::string& n) const {
        for (size_t i = 0; i < maps.size(); i++)
            if (maps[i].name == n) return (int)i;
        return -1;
    }
};

typedef pcg::GenError Err;
using pcg::Gen;
[[noreturn]] void shape(const std::string& m) { throw Err{PENCIL_E_OP2_SHAPE, "E-OP2-SHAPE: " + m}; }
[[noreturn]] void range(const std::string& m) { throw Err{PENCIL_E_OP2_RANGE, "E-OP2-RANGE: " + m}; }
[[noreturn]] void kerr(const std::string& m) { throw Err{PENCIL_E_OP2_KERNEL, "E-OP2-KERNEL: " + m}; }

const mjson::Value& at(const mjson::Value& o, const char* k) {
    const mjson::Value* v = o.is_object() ? o.get(k) : nullptr;
    if (!v) shape(std::string("missing key '") + k + "'");
    return *v;
}
long long req_int(const mjson::Value& v, const char* what) {
    if (!v.is_int()) shape(std::string(what) + " must be an integer");
    return v.i;
}
std::string req_str(const mjson::Value& v, const char* what) {
    if (!v.is_string()) shape(std::string(what) + " must be a string");
    return v.s;
}
std::vector<long long> req_ints(const mjson::Value& v, const char* what) {
    if (!v.is_array()) shape(std::string(what) + " must be a list");
    if (v.arr.empty()) return v.ints;  // all-integer list (parsed compactly)
    std::vector<long long> out;
    out.reserve(v.arr.size());
    for (const auto& e : v.arr) out.push_back(req_int(e, what));
    return out;
}
const std::vector<mjson::Value>& list_or_empty(const mjson::Value& doc, const char* k) {
    static const std::vector<mjson::Value> none;
    const mjson::Value* v = doc.get(k);
    if (!v) return none;
    if (!v->is_array()) shape(std::string("'") + k + "' must be a list");
    return v->arr;
}

Model load_model(const std::string& text) {
    mjson::Value doc;
    std::string perr;
    if (!mjson::parse(text, doc, perr) || !doc.is_object()) shape("input is not a JSON object");
    Model m;
    for (const auto& j : list_or_empty(doc, "sets")) {
        Set s;
        s.name = req_str(at(j, "name"), "set name");
        s.size = req_int(at(j, "size"), "set size");
        if (s.size < 0) shape("set '" + s.name + "' has negative size");
        if (m.set(s.name)) shape("duplicate set '" + s.name + "'");
        m.sets.push_back(s);
    }
    for (const auto& j : list_or_empty(doc, "maps")) {
        Map mp;
        mp.name = req_str(at(j, "name"), "map name");
        mp.from = req_str(at(j, "from"), "map from-set");
        mp.to = req_str(at(j, "to"), "map to-set");
        mp.arity = (int)req_int(at(j, "arity"), "map arity");
        mp.table = req_ints(at(j, "table"), "map table entry");
        const Set* from = m.set(mp.from);
        const Set* to = m.set(mp.to);
        if (!from) shape("map '" + mp.name + "': unknown from-set '" + mp.from + "'");
        if (!to) shape("map '" + mp.name + "': unknown to-set '" + mp.to + "'");
        if (mp.arity < 1) shape("map '" + mp.name + "': arity must be positive");
        if ((long long)mp.table.size() != from->size * mp.arity)
            shape("map '" + mp.name + "': table has " + std::to_string(mp.table.size()) + " entries, expected " +
                  std::to_string(from->size * mp.arity));
        for (long long e : mp.table)
            if (e < 0 || e >= to->size)
                range("map '" + mp.name + "': entry " + std::to_string(e) + " outside target set '" + mp.to +
                      "' of size " + std::to_string(to->size));
        if (m.map(mp.name)) shape("duplicate map '" + mp.name + "'");
        m.maps.push_back(std::move(mp));
    }
    for (const auto& j : list_or_empty(doc, "dats")) {
        Dat d;
        d.name = req_str(at(j, "name"), "dat name");
        d.set = req_str(at(j, "set"), "dat set");
        const mjson::Value* dim = j.get("dim");
        d.dim = dim ? (int)req_int(*dim, "dat dim") : 1;
        d.data = req_ints(at(j, "data"), "dat value");
        const Set* s = m.set(d.set);
        if (!s) shape("dat '" + d.name + "': unknown set '" + d.set + "'");
        if (d.dim < 1) shape("dat '" + d.name + "': dim must be positive");
        if ((long long)d.data.size() != s->size * d.dim)
            shape("dat '" + d.name + "': " + std::to_string(d.data.size()) + " values, expected " +
                  std::to_string(s->size * d.dim));
        if (m.dat_index(d.name) >= 0) shape("duplicate dat '" + d.name + "'");
        m.dats.push_back(std::move(d));
    }
    for (const auto& j : list_or_empty(doc, "kernels")) {
        Kernel k;
        k.name = req_str(at(j, "name"), "kernel name");
        k.source = req_str(at(j, "source"), "kernel source");
        m.kernels.push_back(std::move(k));
    }
    for (const auto& j : list_or_empty(doc, "par_loops")) {
        Loop L;
        L.kernel = req_str(at(j, "kernel"), "par_loop kernel");
        L.set = req_str(at(j, "set"), "par_loop set");
        if (!m.set(L.set)) shape("par_loop: unknown iteration set '" + L.set + "'");
        const mjson::Value* args = j.get("args");
        if (!args || !args->is_array()) shape("par_loop must carry an args list");
        for (const auto& a : args->arr) {
            Arg g;
            g.dat = req_str(at(a, "dat"), "arg dat");
            if (m.dat_index(g.dat) < 0) shape("arg: unknown dat '" + g.dat + "'");
            const std::string acc = req_str(at(a, "access"), "arg access");
            if (acc == "OP_READ") g.access = A_READ;
            else if (acc == "OP_WRITE") g.access = A_WRITE;
            else if (acc == "OP_RW") g.access = A_RW;
            else if (acc == "OP_INC") g.access = A_INC;
            else shape("unknown access hint '" + acc + "'");
            const mjson::Value* mv = a.get("map");
            if (mv && !mv->is_null()) {
                g.map = req_str(*mv, "arg map");
                const Map* mp = m.map(g.map);
                if (!mp) shape("arg: unknown map '" + g.map + "'");
                if (mp->from != L.set) shape("arg: map '" + g.map + "' is not indexed by set '" + L.set + "'");
                g.offset = (int)req_int(at(a, "offset"), "arg offset");
                if (g.offset < 0 || g.offset >= mp->arity)
                    range("arg: offset " + std::to_string(g.offset) + " outside map '" + g.map + "' of arity " +
                          std::to_string(mp->arity));
            }
            L.args.push_back(std::move(g));
        }
        m.loops.push_back(std::move(L));
    }
    return m;
}

std::vector<std::string> distinct_dats(const Loop& L) {
    std::vector<std::string> out;
    for (const auto& a : L.args)
        if (std::find(out.begin(), out.end(), a.dat) == out.end()) out.push_back(a.dat);
    return out;
}
std::vector<std::string> distinct_maps(const Loop& L) {
    std::vector<std::string> out;
    for (const auto& a : L.args)
        if (!a.direct() && std::find(out.begin(), out.end(), a.map) == out.end()) out.push_back(a.map);
    return out;
}
void check_conflicts(const Loop& L) {
    for (const auto& a : L.args) {
        if (a.access != A_INC) continue;
        for (const auto& b : L.args)
            if (b.dat == a.dat && (b.access == A_RW || b.access == A_WRITE))
                throw Err{PENCIL_E_OP2_CONFLICT,
                          "E-OP2-CONFLICT: dat '" + a.dat + "' is both incremented and written in one par_loop"};
    }
}
void check_signature(const pf::Func& fn, const Loop& L) {
    size_t m = distinct_dats(L).size(), n = L.args.size();
    if (fn.params.size() != 2 * m + n)
        kerr("kernel '" + fn.name + "' takes " + std::to_string(fn.params.size()) + " parameters, expected " +
             std::to_string(2 * m + n) + " for " + std::to_string(n) + " args over " + std::to_string(m) + " dats");
    for (size_t i = 0; i < fn.params.size(); ++i) {
        bool want_array = i >= m && i < 2 * m;
        bool is_array = fn.params[i].kind == pf::Param::Array;
        if (want_array != is_array)
            kerr("kernel '" + fn.name + "' parameter '" + fn.params[i].name + "' should be " +
                 (want_array ? "an array" : "a scalar"));
    }
}

// ------------------------------------------------------------------ static scan of kernel bodies
// Per function and array parameter: loaded? stored additively (+= / -=)? stored otherwise?
// (propagated through calls that pass the array by name); and whether rand() is reachable.
struct ArrUse {
    bool load = false, add_store = false, other_store = false;
};
struct FnInfo {
    std::vector<ArrUse> uses;  // per parameter position (arrays / pointers only meaningful)
    bool rand = false;
};

struct Scanner {
    const pf::Unit& u;
    std::map<std::string, FnInfo> info;
    std::set<std::string> busy;
    explicit Scanner(const pf::Unit& unit) : u(unit) {}

    const FnInfo& get(const pf::Func& f) {
        auto it = info.find(f.name);
        if (it != info.end()) return it->second;
        if (busy.count(f.name)) {  // recursion: conservatively everything
            static FnInfo all;
            all.rand = true;
            all.uses.assign(64, ArrUse{true, true, true});
            return all;
        }
        busy.insert(f.name);
        FnInfo fi;
        fi.uses.resize(f.params.size());
        std::map<std::string, int> pos;
        for (size_t i = 0; i < f.params.size(); i++)
            if (f.params[i].kind != pf::Param::Scalar) pos[f.params[i].name] = (int)i;
        std::function<void(const pf::Expr&)> ex = [&](const pf::Expr& e) {
            if (e.kind == pf::Expr::Index || (e.kind == pf::Expr::Unary && e.uop == pf::Un::Deref && !e.args.empty() &&
                                               e.args[0]->kind == pf::Expr::Var)) {
                const std::string& n = e.kind == pf::Expr::Index ? e.name : e.args[0]->name;
                auto p = pos.find(n);
                if (p != pos.end()) fi.uses[p->second].load = true;
            }
            if (e.kind == pf::Expr::Call) {
                if (e.name == "rand") fi.rand = true;
                const pf::Func* callee = u.find(e.name);
                if (callee) {
                    const FnInfo& ci = get(*callee);
                    fi.rand |= ci.rand;
                    for (size_t k = 0; k < e.args.size() && k < callee->params.size(); k++) {
                        if (callee->params[k].kind == pf::Param::Scalar || e.args[k]->kind != pf::Expr::Var) continue;
                        auto p = pos.find(e.args[k]->name);
                        if (p == pos.end() || k >= ci.uses.size()) continue;
                        fi.uses[p->second].load |= ci.uses[k].load;
                        fi.uses[p->second].add_store |= ci.uses[k].add_store;
                        fi.uses[p->second].other_store |= ci.uses[k].other_store;
                    }
                }
            }
            for (const auto& a : e.args)
                if (!(e.kind == pf::Expr::Call && a->kind == pf::Expr::Var)) ex(*a);
        };
        std::function<void(const pf::Stmt&)> st = [&](const pf::Stmt& s) {
            switch (s.kind) {
                case pf::Stmt::Block:
                    for (const auto& c : s.body) st(*c);
                    break;
                case pf::Stmt::Decl:
                    for (const auto& e : s.extents) ex(*e);
                    if (s.rhs) ex(*s.rhs);
                    break;
                case pf::Stmt::Assign: {
                    ex(*s.rhs);
                    const pf::Expr& lv = *s.lhs;
                    std::string n;
                    if (lv.kind == pf::Expr::Index) {
                        n = lv.name;
                        for (const auto& a : lv.args) ex(*a);
                    } else if (lv.kind == pf::Expr::Unary && lv.uop == pf::Un::Deref && lv.args[0]->kind == pf::Expr::Var) {
                        n = lv.args[0]->name;
                    }
                    auto p = pos.find(n);
                    if (p != pos.end()) {
                        if (s.aop == pf::AOp::Add || s.aop == pf::AOp::Sub) fi.uses[p->second].add_store = true;
                        else fi.uses[p->second].other_store = true;
                    }
                    break;
                }
                case pf::Stmt::For:
                    ex(*s.lo);
                    ex(*s.hi);
                    st(*s.loop_body);
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
                case pf::Stmt::Nop: break;
            }
        };
        if (f.body) st(*f.body);
        busy.erase(f.name);
        return info[f.name] = fi;
    }
};

}  // namespace

// ------------------------------------------------------------------ the model object
struct pencil_op2_model {
    Model m;
    pf::Unit unit;
    std::string cuda_src, lowered;
    std::vector<int> strategy, levels;
    int device = -1;
    cudaStream_t stream = nullptr;
    cudaLibrary_t lib = nullptr;
    std::vector<cudaKernel_t> kern;
    std::vector<long long*> d_dat;
    std::vector<long long*> d_map;
    std::vector<long long*> d_iters;               // per loop: level-ordered iterations (LEVELS)
    std::vector<std::vector<long long>> lvl_off;   // per loop: level offsets into d_iters
    unsigned* d_fault = nullptr;
    unsigned long long* d_rng = nullptr;
    bool host_stale = false;                       // device dats newer than m.dats[].data
};

namespace {

enum { STRAT_PARALLEL = 0, STRAT_LEVELS = 1, STRAT_SERIAL = 2 };

std::string lower_text(const Model& m) {
    // the reference's lowering (append_driver, op2.cpp:253-345) printed as PENCIL: kernels, then one
    // driver per par_loop: for (i = 0; i < n_iter; i++) kernel(n_D..., D..., idx...)
    std::ostringstream o;
    for (const auto& k : m.kernels) o << k.source << "\n";
    for (const auto& L : m.loops) {
        auto dats = distinct_dats(L);
        auto maps = distinct_maps(L);
        o << "void " << L.kernel << "_loop(int n_iter";
        for (auto& d : dats) o << ", int n_" << d;
        for (auto& mp : maps) o << ", int n_" << mp;
        for (auto& d : dats) o << ", int " << d << "[restrict const static n_" << d << "]";
        for (auto& mp : maps) o << ", int " << mp << "[restrict const static n_" << mp << "]";
        o << ")\n{\n  int i;\n";
        std::vector<std::string> inc;
        bool indirect_write = false;
        for (auto& a : L.args) {
            if (a.access == A_INC && std::find(inc.begin(), inc.end(), a.dat) == inc.end()) inc.push_back(a.dat);
            if (!a.direct() && (a.access == A_WRITE || a.access == A_RW)) indirect_write = true;
        }
        if (!inc.empty()) {
            o << "  #pragma pencil reduction (+: ";
            for (size_t i = 0; i < inc.size(); i++) o << (i ? ", " : "") << inc[i];
            o << ")\n";
        } else if (indirect_write) {
            o << "  #pragma pencil independent\n";
        }
        o << "  for (i = 0; i < n_iter; i++) {\n    " << L.kernel << "(";
        bool first = true;
        for (auto& d : dats) { o << (first ? "" : ", ") << "n_" << d; first = false; }
        for (auto& d : dats) o << ", " << d;
        for (auto& a : L.args) {
            if (a.direct()) o << ", i";
            else o << ", " << a.map << "[" << m.map(a.map)->arity << " * i + " << a.offset << "]";
        }
        o << ");\n  }\n}\n";
    }
    return o.str();
}

int choose_strategy(const Model& m, const Loop& L, const pf::Func& kf, Scanner& sc) {
    const FnInfo& fi = sc.get(kf);
    if (fi.rand) return STRAT_SERIAL;
    auto dats = distinct_dats(L);
    for (size_t j = 0; j < dats.size(); j++) {
        bool inc = false;
        for (auto& a : L.args)
            if (a.dat == dats[j] && a.access == A_INC) inc = true;
        if (!inc) continue;
        const ArrUse& use = fi.uses[dats.size() + j];  // array parameter j
        if (use.load || use.other_store) return STRAT_SERIAL;
        for (auto& a : L.args)  // an INC dat also read through another argument
            if (a.dat == dats[j] && a.access != A_INC) return STRAT_SERIAL;
    }
    for (auto& d : dats) {
        bool written = false, mapped = false, mapped_write = false;
        for (auto& a : L.args) {
            if (a.dat != d) continue;
            bool w = a.access == A_WRITE || a.access == A_RW;
            written |= w;
            mapped |= !a.direct();
            mapped_write |= w && !a.direct();
        }
        if (mapped_write || (written && mapped)) return STRAT_LEVELS;
    }
    (void)m;
    return STRAT_PARALLEL;
}

// iteration levels: every element (dat, set element) touched by an argument of a written dat
// sees its iterations in order; returns iterations grouped by level and the level offsets
void build_levels(const Model& m, const Loop& L, std::vector<long long>& order, std::vector<long long>& off) {
    const long long n = m.set(L.set)->size;
    std::vector<int> written_args;
    for (size_t k = 0; k < L.args.size(); k++) {
        const Arg& a = L.args[k];
        bool w = false;
        for (auto& b : L.args)
            if (b.dat == a.dat && (b.access == A_WRITE || b.access == A_RW)) w = true;
        if (w) written_args.push_back((int)k);
    }
    std::map<std::string, std::vector<int>> last;  // per dat: last level that touched each element
    for (int k : written_args) {
        const Arg& a = L.args[k];
        const Dat& d = m.dats[m.dat_index(a.dat)];
        auto& v = last[a.dat];
        if (v.empty()) v.assign(m.set(d.set)->size + 1, -1);
    }
    std::vector<int> lvl(n, 0);
    int maxl = -1;
    for (long long i = 0; i < n; i++) {
        int l = 0;
        std::vector<std::pair<std::vector<int>*, long long>> keys;
        for (int k : written_args) {
            const Arg& a = L.args[k];
            long long e = a.direct() ? i : m.map(a.map)->table[(size_t)(m.map(a.map)->arity * i + a.offset)];
            auto& v = last[a.dat];
            if (e < 0 || e >= (long long)v.size()) e = (long long)v.size() - 1;
            l = std::max(l, v[e] + 1);
            keys.push_back({&v, e});
        }
        for (auto& kv : keys) (*kv.first)[kv.second] = l;
        lvl[i] = l;
        maxl = std::max(maxl, l);
    }
    off.assign(maxl + 2, 0);
    for (long long i = 0; i < n; i++) off[lvl[i] + 1]++;
    for (int l = 0; l <= maxl; l++) off[l + 1] += off[l];
    order.assign(n, 0);
    std::vector<long long> pos(off.begin(), off.end() - 1);
    for (long long i = 0; i < n; i++) order[pos[lvl[i]]++] = i;
}

bool map_fits_i32(const Map& mp) {
    for (long long e : mp.table)
        if (e > 2147483647ll) return false;
    return true;
}

std::string driver_source(const Model& m, const Loop& L, int li, const pf::Func& kf) {
    (void)kf;
    auto dats = distinct_dats(L);
    auto maps = distinct_maps(L);
    std::ostringstream o;
    o << "extern \"C\" __global__ void op2_loop_" << li << "(Ctx cx, ll n_iter, const ll* __restrict__ iters";
    for (size_t j = 0; j < dats.size(); j++) o << ", ll* d" << j << ", ll n" << j << ", int inc" << j;
    for (size_t j = 0; j < maps.size(); j++)  // maps into sets below 2^31 elements are stored as int32
        o << ", const " << (map_fits_i32(*m.map(maps[j])) ? "int" : "ll") << "* __restrict__ m" << j;
    o << ") {\n  const ll stride = (ll)gridDim.x * blockDim.x;\n";
    o << "  for (ll t = (ll)blockIdx.x * blockDim.x + threadIdx.x; t < n_iter; t += stride) {\n";
    o << "    const ll i = iters ? iters[t] : t;\n";
    for (size_t j = 0; j < dats.size(); j++) o << "    Arr A" << j << " = {d" << j << ", n" << j << ", inc" << j << "};\n";
    o << "    f_" << L.kernel << "(cx";
    for (size_t j = 0; j < dats.size(); j++) o << ", VI(n" << j << ")";
    for (size_t j = 0; j < dats.size(); j++) o << ", A" << j;
    for (const auto& a : L.args) {
        if (a.direct()) {
            o << ", VI(i)";
        } else {
            size_t mj = std::find(maps.begin(), maps.end(), a.map) - maps.begin();
            o << ", VI(m" << mj << "[(ll)" << m.map(a.map)->arity << " * i + " << a.offset << "])";
        }
    }
    o << ");\n  }\n}\n";
    return o.str();
}

#define OCK(call)                                                                            \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess) return fail(PENCIL_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

int device_setup(pencil_op2_model* M) {
    if (M->lib) return PENCIL_OK;
    std::vector<char> cubin;
    std::string log;
    int rc = pcg::compile_cubin(M->cuda_src, cubin, log);
    if (rc) return fail(rc, "E-CUDA: OP2 kernel compilation failed: " + log);
    OCK(cudaGetDevice(&M->device));
    OCK(cudaStreamCreateWithFlags(&M->stream, cudaStreamNonBlocking));
    OCK(cudaLibraryLoadData(&M->lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
    M->kern.resize(M->m.loops.size());
    for (size_t li = 0; li < M->m.loops.size(); li++) {
        std::string name = "op2_loop_" + std::to_string(li);
        OCK(cudaLibraryGetKernel(&M->kern[li], M->lib, name.c_str()));
    }
    M->d_dat.assign(M->m.dats.size(), nullptr);
    for (size_t j = 0; j < M->m.dats.size(); j++) {
        const auto& d = M->m.dats[j].data;
        OCK(cudaMalloc(&M->d_dat[j], std::max<size_t>(8, d.size() * 8)));
        if (!d.empty()) OCK(cudaMemcpy(M->d_dat[j], d.data(), d.size() * 8, cudaMemcpyHostToDevice));
    }
    M->d_map.assign(M->m.maps.size(), nullptr);
    for (size_t j = 0; j < M->m.maps.size(); j++) {
        const auto& t = M->m.maps[j].table;
        if (map_fits_i32(M->m.maps[j])) {
            std::vector<int> t32(t.begin(), t.end());
            OCK(cudaMalloc(&M->d_map[j], std::max<size_t>(8, t.size() * 4)));
            if (!t.empty()) OCK(cudaMemcpy(M->d_map[j], t32.data(), t.size() * 4, cudaMemcpyHostToDevice));
        } else {
            OCK(cudaMalloc(&M->d_map[j], std::max<size_t>(8, t.size() * 8)));
            if (!t.empty()) OCK(cudaMemcpy(M->d_map[j], t.data(), t.size() * 8, cudaMemcpyHostToDevice));
        }
    }
    M->d_iters.assign(M->m.loops.size(), nullptr);
    M->lvl_off.assign(M->m.loops.size(), {});
    for (size_t li = 0; li < M->m.loops.size(); li++) {
        if (M->strategy[li] != STRAT_LEVELS) continue;
        std::vector<long long> order;
        build_levels(M->m, M->m.loops[li], order, M->lvl_off[li]);
        M->levels[li] = (int)M->lvl_off[li].size() - 1;
        OCK(cudaMalloc(&M->d_iters[li], std::max<size_t>(8, order.size() * 8)));
        if (!order.empty()) OCK(cudaMemcpy(M->d_iters[li], order.data(), order.size() * 8, cudaMemcpyHostToDevice));
    }
    OCK(cudaMalloc(&M->d_fault, 64));
    OCK(cudaMemset(M->d_fault, 0, 64));
    OCK(cudaMalloc(&M->d_rng, 8));
    const unsigned long long seed = 0x9e3779b97f4a7c15ull;  // the interpreter's rng_state_ (interp.hpp:67)
    OCK(cudaMemcpy(M->d_rng, &seed, 8, cudaMemcpyHostToDevice));
    return PENCIL_OK;
}

int launch_loop(pencil_op2_model* M, int li) {
    const Loop& L = M->m.loops[li];
    auto dats = distinct_dats(L);
    auto maps = distinct_maps(L);
    const long long n = M->m.set(L.set)->size;
    struct Ctx {
        unsigned* fault;
        unsigned long long* rng;
        const long long* rseq;
        unsigned long long* rpos;
        long long rseq_n;
        unsigned long long* tr;  // JIT trace buffer (unused here)
    } cx{M->d_fault, M->d_rng, nullptr, nullptr, 0, nullptr};
    const int strat = M->strategy[li];
    std::vector<long long> nn(dats.size());
    std::vector<int> inc(dats.size());
    std::vector<long long*> dp(dats.size());
    std::vector<const long long*> mp(maps.size());
    for (size_t j = 0; j < dats.size(); j++) {
        int di = M->m.dat_index(dats[j]);
        dp[j] = M->d_dat[di];
        nn[j] = (long long)M->m.dats[di].data.size();
        bool is_inc = false;
        for (auto& a : L.args)
            if (a.dat == dats[j] && a.access == A_INC) is_inc = true;
        inc[j] = is_inc && strat != STRAT_SERIAL;
    }
    for (size_t j = 0; j < maps.size(); j++) mp[j] = M->d_map[M->m.map_index(maps[j])];
    auto go = [&](long long count, const long long* iters, bool serial) -> int {
        if (count <= 0) return PENCIL_OK;
        std::vector<void*> args;
        args.push_back(&cx);
        args.push_back(&count);
        args.push_back(&iters);
        for (size_t j = 0; j < dats.size(); j++) {
            args.push_back(&dp[j]);
            args.push_back(&nn[j]);
            args.push_back(&inc[j]);
        }
        for (size_t j = 0; j < maps.size(); j++) args.push_back(&mp[j]);
        long long blocks = serial ? 1 : (count + 255) / 256;
        if (blocks > 148 * 16) blocks = 148 * 16;
        OCK(cudaLaunchKernel((const void*)M->kern[li], dim3((unsigned)blocks), dim3(serial ? 1 : 256), args.data(), 0,
                             M->stream));
        return PENCIL_OK;
    };
    int rc = PENCIL_OK;
    if (strat == STRAT_LEVELS) {
        const auto& off = M->lvl_off[li];
        for (size_t l = 0; l + 1 < off.size() && !rc; l++)
            rc = go(off[l + 1] - off[l], M->d_iters[li] + off[l], false);
    } else {
        rc = go(n, nullptr, strat == STRAT_SERIAL);
    }
    return rc;
}

int collect(pencil_op2_model* M) {
    unsigned f = 0;
    OCK(cudaMemcpyAsync(&f, M->d_fault, 4, cudaMemcpyDeviceToHost, M->stream));
    OCK(cudaMemsetAsync(M->d_fault, 0, 4, M->stream));
    OCK(cudaStreamSynchronize(M->stream));
    if (!f) return PENCIL_OK;
    std::string m = "E-INTERP: OP2 kernel fault:";
    if (f & 1u) m += " load out of bounds;";
    if (f & 2u) m += " store out of bounds;";
    if (f & 4u) m += " division by zero;";
    if (f & 8u) m += " modulo by zero;";
    if (f & 16u) m += " non-integral value where an integer is required;";
    if (f & 32u) m += " non-integer value stored into an integer dat (unsupported);";
    if (f & 64u) m += " empty pointee;";
    if (f & 128u) m += " execution step budget exceeded;";
    return fail(PENCIL_E_INTERP, m);
}

}  // namespace

extern "C" {

pencil_op2_t pencil_op2_load(const char* json_text) {
    if (!json_text) {
        fail(PENCIL_E_ARG, "E-ARG: null model text");
        return nullptr;
    }
    auto* M = new pencil_op2_model();
    try {
        M->m = load_model(json_text);
        // kernels: parsed as one unit (parse_kernels, op2.cpp:347-365)
        for (const auto& k : M->m.kernels) {
            pf::Unit one;
            std::string err;
            if (!pf::parse_unit(k.source, one, err)) kerr("kernel '" + k.name + "' does not parse: " + err);
            bool found = false;
            for (auto& f : one.fns) {
                if (f.name == k.name) found = true;
                M->unit.fns.push_back(std::move(f));
            }
            if (!found) kerr("kernel source does not define '" + k.name + "'");
        }
        Scanner sc(M->unit);
        Gen g(M->unit);
        g.unit(pcg::kArrInt64);
        std::ostringstream drivers;
        for (size_t li = 0; li < M->m.loops.size(); li++) {
            const Loop& L = M->m.loops[li];
            check_conflicts(L);
            const pf::Func* kf = M->unit.find(L.kernel);
            if (!kf) kerr("kernel '" + L.kernel + "' is not defined in the model");
            check_signature(*kf, L);
            M->strategy.push_back(choose_strategy(M->m, L, *kf, sc));
            M->levels.push_back(M->strategy.back() == STRAT_LEVELS ? -1 : 1);
            drivers << driver_source(M->m, L, (int)li, *kf);
        }
        M->cuda_src = g.out.str() + drivers.str();
        M->lowered = lower_text(M->m);
    } catch (const Err& e) {
        pencil_internal_fail(e.st, e.msg.c_str());
        delete M;
        return nullptr;
    }
    pencil_internal_ok();
    return M;
}

void pencil_op2_free(pencil_op2_t M) {
    if (!M) return;
    if (M->stream) cudaStreamSynchronize(M->stream);
    for (auto p : M->d_dat) cudaFree(p);
    for (auto p : M->d_map) cudaFree(p);
    for (auto p : M->d_iters) cudaFree(p);
    if (M->d_fault) cudaFree(M->d_fault);
    if (M->d_rng) cudaFree(M->d_rng);
    if (M->lib) cudaLibraryUnload(M->lib);
    if (M->stream) cudaStreamDestroy(M->stream);
    delete M;
}

int pencil_op2_num_loops(pencil_op2_t M) { return M ? (int)M->m.loops.size() : -1; }

int pencil_op2_loop_info(pencil_op2_t M, int loop, int* strategy, int* levels) {
    if (!M || loop < 0 || loop >= (int)M->m.loops.size()) return fail(PENCIL_E_ARG, "E-ARG: no such par_loop");
    if (strategy) *strategy = M->strategy[loop];
    if (levels) *levels = M->levels[loop];
    return pencil_internal_ok();
}

int pencil_op2_prepare(pencil_op2_t M) {
    if (!M) return fail(PENCIL_E_ARG, "E-ARG: null model");
    int rc = device_setup(M);
    return rc ? rc : pencil_internal_ok();
}

int pencil_op2_run_loop_async(pencil_op2_t M, int loop) {
    if (!M || loop < 0 || loop >= (int)M->m.loops.size()) return fail(PENCIL_E_ARG, "E-ARG: no such par_loop");
    int rc = device_setup(M);
    if (rc) return rc;
    rc = launch_loop(M, loop);
    if (rc) return rc;
    M->host_stale = true;
    return pencil_internal_ok();
}

int pencil_op2_run(pencil_op2_t M) {
    if (!M) return fail(PENCIL_E_ARG, "E-ARG: null model");
    int rc = device_setup(M);
    if (rc) return rc;
    for (size_t li = 0; li < M->m.loops.size(); li++) {
        if ((rc = launch_loop(M, (int)li))) return rc;
        // a fault stops the run after the faulting par_loop, like the interpreter's exception
        if ((rc = collect(M))) return rc;
    }
    M->host_stale = true;
    return pencil_internal_ok();
}

int pencil_op2_sync(pencil_op2_t M) {
    if (!M) return fail(PENCIL_E_ARG, "E-ARG: null model");
    if (!M->stream) return pencil_internal_ok();
    int rc = collect(M);
    return rc ? rc : pencil_internal_ok();
}

long long pencil_op2_dat_size(pencil_op2_t M, const char* dat) {
    if (!M || !dat) return -1;
    int di = M->m.dat_index(dat);
    return di < 0 ? -1 : (long long)M->m.dats[di].data.size();
}

int pencil_op2_get_dat(pencil_op2_t M, const char* dat, long long* out, long long n) {
    if (!M || !dat || (n && !out)) return fail(PENCIL_E_ARG, "E-ARG: null argument");
    int di = M->m.dat_index(dat);
    if (di < 0) return fail(PENCIL_E_ARG, std::string("E-ARG: no dat named '") + dat + "'");
    auto& d = M->m.dats[di].data;
    if (n != (long long)d.size()) return fail(PENCIL_E_ARG, "E-ARG: dat size mismatch");
    if (M->stream) {
        OCK(cudaStreamSynchronize(M->stream));
        const size_t bytes = (size_t)n * 8;
        if (n && bytes >= OP2_STAGE_MIN && host_is_pageable(out)) {  // the multi-threaded staging ring
            OCK((cudaError_t)staged_d2h_2d(M->device, out, bytes, M->d_dat[di], bytes, bytes, 1, M->stream));
            OCK(cudaStreamSynchronize(M->stream));
        } else if (n) {
            OCK(cudaMemcpy(out, M->d_dat[di], bytes, cudaMemcpyDeviceToHost));
        }
    } else if (n) {
        memcpy(out, d.data(), (size_t)n * 8);
    }
    return pencil_internal_ok();
}

int pencil_op2_set_dat(pencil_op2_t M, const char* dat, const long long* in, long long n) {
    if (!M || !dat || (n && !in)) return fail(PENCIL_E_ARG, "E-ARG: null argument");
    int di = M->m.dat_index(dat);
    if (di < 0) return fail(PENCIL_E_ARG, std::string("E-ARG: no dat named '") + dat + "'");
    auto& d = M->m.dats[di].data;
    if (n != (long long)d.size()) return fail(PENCIL_E_ARG, "E-ARG: dat size mismatch");
    if (!M->stream) {  // before prepare: the host copy is what the device setup uploads
        if (n) memcpy(d.data(), in, (size_t)n * 8);
        return pencil_internal_ok();
    }
    // on the device the device copy is the dat (the host copy is stale from the first run on)
    M->host_stale = true;
    OCK(cudaStreamSynchronize(M->stream));
    const size_t bytes = (size_t)n * 8;
    if (n && bytes >= OP2_STAGE_MIN && host_is_pageable(in))  // the multi-threaded staging ring
        OCK((cudaError_t)staged_h2d_2d(M->device, M->d_dat[di], bytes, in, bytes, bytes, 1, M->stream));
    else if (n)
        OCK(cudaMemcpyAsync(M->d_dat[di], in, bytes, cudaMemcpyHostToDevice, M->stream));
    OCK(cudaStreamSynchronize(M->stream));
    return pencil_internal_ok();
}

const char* pencil_op2_cuda_source(pencil_op2_t M) { return M ? M->cuda_src.c_str() : ""; }
const char* pencil_op2_lowered(pencil_op2_t M) { return M ? M->lowered.c_str() : ""; }
void* pencil_op2_stream(pencil_op2_t M) { return M ? (void*)M->stream : nullptr; }

}  // extern "C"
