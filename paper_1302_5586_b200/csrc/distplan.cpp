// Distribution plans ("data-movement plan: read-only arrays ->
// replicated; written arrays -> sharded ownership; which arrays need all-gather").
//
// For the outermost parallel loop of a function (`#pragma pencil independent`, or a top-level
// `reduction` loop) — and the nested `independent` loop under it, the 2-D grid of gemm and the
// stencils — every access of every array parameter inside the loop is put in one of four classes
// relative to the loop variable d, from its index expression:
//   block(C, [h0, h1])  index = C*d + r with C invariant (scalar parameters) and r, over the
//                       other loop variables' ranges, inside blocks d + h0 .. d + h1 (units of
//                       C): a contiguous row-block shard, with an h0 / h1 halo (conv: img +-2 rows)
//   view(C, strides)    the same, but r spans far more than a few blocks through other loop
//                       variables with invariant coefficients: a strided view of the shard
//                       (gemv_t: A[i*lda + j] split by columns j; gemm's 2-D tile)
//   via(A)              index = k where k runs from A[f(d)] to A[g(d)]: the CSR non-zero range,
//                       sharded through the row-pointer array A
//   all                 anything else (no d in the index, or a data-dependent index such as
//                       x[col[k]]): every iteration may touch every element
// Indices go through local scalars (their assigned affine forms; the clamp pattern
// `if (v < e) v = e;` / `if (v > e) v = e;` bounds v without widening it — conv5x5_u8's
// clamp-to-edge), through calls (parameters substituted) and through ACCESS summaries (the
// summary function's DEF / USE / MAY_DEF statements, as summarize_call reads them,
// summaries.cpp:466-478, 635-648).  Ranges are evaluated under a sample binding of the scalar
// parameters (distinct values ~10^3), at an interior iteration of d, over the corners of the other
// loop variables' boxes (affine forms and clamps are monotone in each variable).
//
// Per dimension the plan then lists: arrays written in blocks (owned, no collective), arrays read
// in blocks with a halo (halo exchange), arrays read `all` (replicated: all-gathered when they
// were produced sharded), reduction variables of the loop (all-reduce), and arrays written `all`
// (conflicts: the loop cannot be split on d as written).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/pencil_b200.h"
#include "affine.hpp"
#include "pencil_front.hpp"

int pencil_internal_fail(int status, const char* msg);  // runtime.cpp
int pencil_internal_ok();

using namespace affine_forms;

namespace {

// ---------------------------------------------------------------- affine algebra on Aff
Aff aneg(const Aff& a) {
    Aff r;
    r.ok = a.ok;
    for (const auto& [v, p] : a.coef) r.coef[v] = padd(Poly{}, p, -1);
    r.c = padd(Poly{}, a.c, -1);
    return r;
}
Aff aadd(const Aff& a, const Aff& b, long long sb) {
    Aff r;
    r.ok = a.ok && b.ok;
    r.coef = a.coef;
    for (const auto& [v, p] : b.coef) {
        r.coef[v] = padd(r.coef[v], p, sb);
        if (r.coef[v].empty()) r.coef.erase(v);
    }
    r.c = padd(a.c, b.c, sb);
    return r;
}
bool amul(const Aff& a, const Aff& b, Aff& r) {
    if (!a.coef.empty() && !b.coef.empty()) return false;  // loop var * loop var
    const Aff& lin = a.coef.empty() ? b : a;
    const Aff& k = a.coef.empty() ? a : b;
    r = Aff{};
    for (const auto& [v, p] : lin.coef) {
        Poly q = pmul(p, k.c);
        if (!q.empty()) r.coef[v] = q;
    }
    r.c = pmul(lin.c, k.c);
    return true;
}

struct Local {
    std::vector<Aff> forms;  // empty: not affine
    std::vector<Aff> lo, hi; // clamp bounds (if (v < e) v = e; / if (v > e) v = e;)
};

struct Loop {
    std::string var;
    Aff lo, hi;         // [lo, hi) when affine (ok == false otherwise)
    std::string via;    // bounds A[...] .. A[...]: the non-zero range of row-pointer array A
};

// a clamped local scalar used in an index: its unclamped value and its clamp bounds
struct ClampDef {
    Aff val;
    std::vector<Aff> lo, hi;
};

struct Acc {
    std::string array;
    bool write;
    std::string via;                      // index = a loop variable bounded through `via`
    std::vector<Aff> forms;               // empty and via empty: data-dependent (all); clamped locals
                                          // appear as pseudo-variables "~cN" defined in `clamps`
    std::vector<Loop> loops;              // loops in scope (outermost first)
    std::map<std::string, ClampDef> clamps;
};

// One function frame of the walk: names of this frame -> what they mean at the top level.
struct Frame {
    std::map<std::string, std::string> arrays;          // array param / alias -> top-level array
    std::map<std::string, std::vector<Aff>> scalars;    // scalar param -> forms (top-level terms)
    std::map<std::string, std::string> loopname;        // this frame's loop var -> unique name
    std::map<std::string, Local> locals;
};

struct Walker {
    const pf::Unit& u;
    std::map<std::string, int> params;  // top function's scalar parameters (invariant)
    std::vector<Loop> loops;            // loops in scope inside the distributed nest
    std::vector<Acc> out;
    int uniq = 0, depth = 0;

    explicit Walker(const pf::Unit& unit) : u(unit) {}

    // the affine forms an expression may take (empty: not affine)
    std::vector<Aff> forms(const pf::Expr& e, Frame& F, std::map<std::string, ClampDef>* cl) {
        std::vector<Aff> r;
        switch (e.kind) {
            case pf::Expr::IntLit: {
                Aff a;
                a.c = pconst(e.ival);
                r.push_back(a);
                return r;
            }
            case pf::Expr::Var: {
                auto ln = F.loopname.find(e.name);
                if (ln != F.loopname.end()) {
                    Aff a;
                    a.coef[ln->second] = pconst(1);
                    r.push_back(a);
                    return r;
                }
                auto lc = F.locals.find(e.name);
                if (lc != F.locals.end()) {
                    const Local& L = lc->second;
                    if (L.lo.empty() && L.hi.empty()) return L.forms;
                    // clamped: a pseudo-variable whose value is clamp(form, lo, hi) at evaluation
                    if (!cl || L.forms.size() != 1) return r;
                    const std::string tag = "~c" + std::to_string(uniq++);
                    (*cl)[tag] = ClampDef{L.forms[0], L.lo, L.hi};
                    Aff a;
                    a.coef[tag] = pconst(1);
                    r.push_back(a);
                    return r;
                }
                auto sc = F.scalars.find(e.name);
                if (sc != F.scalars.end()) return sc->second;
                if (params.count(e.name)) {
                    Aff a;
                    a.c = Poly{{Mono{e.name}, 1}};
                    r.push_back(a);
                }
                return r;
            }
            case pf::Expr::Unary:
                if (e.uop == pf::Un::Neg)
                    for (const auto& a : forms(*e.args[0], F, cl)) r.push_back(aneg(a));
                return r;
            case pf::Expr::Binary: {
                if (e.bop != pf::Bin::Add && e.bop != pf::Bin::Sub && e.bop != pf::Bin::Mul) return r;
                const auto A = forms(*e.args[0], F, cl), B = forms(*e.args[1], F, cl);
                for (const auto& a : A)
                    for (const auto& b : B) {
                        if (r.size() >= 16) return r;
                        if (e.bop == pf::Bin::Mul) {
                            Aff m;
                            if (!amul(a, b, m)) return {};
                            r.push_back(m);
                        } else {
                            r.push_back(aadd(a, b, e.bop == pf::Bin::Add ? 1 : -1));
                        }
                    }
                return r;
            }
            default: return r;
        }
    }

    void record(const std::string& arr, const pf::Expr& idx, bool write, Frame& F) {
        Acc a;
        a.array = arr;
        a.write = write;
        a.loops = loops;
        if (idx.kind == pf::Expr::Var) {
            auto ln = F.loopname.find(idx.name);
            if (ln != F.loopname.end())
                for (const auto& L : loops)
                    if (L.var == ln->second && !L.via.empty()) a.via = L.via;
        }
        if (a.via.empty()) a.forms = forms(idx, F, &a.clamps);
        out.push_back(a);
    }

    // reads inside an expression (and call arguments / callees)
    void expr(const pf::Expr& e, Frame& F) {
        if (e.kind == pf::Expr::Index) {
            for (const auto& a : e.args) expr(*a, F);
            auto it = F.arrays.find(e.name);
            if (it != F.arrays.end() && e.args.size() == 1) record(it->second, *e.args[0], false, F);
            return;
        }
        if (e.kind == pf::Expr::Call) {
            for (const auto& a : e.args)
                if (a->kind != pf::Expr::Var || !F.arrays.count(a->name)) expr(*a, F);
            call(e, F);
            return;
        }
        for (const auto& a : e.args) expr(*a, F);
    }

    // the callee's accesses with its parameters bound to the call's arguments
    void call(const pf::Expr& c, Frame& F) {
        const pf::Func* g = u.find(c.name);
        if (!g || depth > 8) return;
        Frame G;
        for (size_t k = 0; k < g->params.size() && k < c.args.size(); k++) {
            const pf::Expr& a = *c.args[k];
            if (g->params[k].kind == pf::Param::Scalar) {
                G.scalars[g->params[k].name] = forms(a, F, nullptr);
            } else if (a.kind == pf::Expr::Var && F.arrays.count(a.name)) {
                G.arrays[g->params[k].name] = F.arrays[a.name];
            }
        }
        depth++;
        if (!g->access_fn.empty()) {  // ACCESS-summarised: what the summary function declares
            const pf::Func* s = u.find(g->access_fn);
            if (s) {
                Frame S;
                for (size_t k = 0; k < s->params.size() && k < g->access_args.size(); k++) {
                    const pf::Expr& a = *g->access_args[k];
                    if (s->params[k].kind == pf::Param::Scalar) S.scalars[s->params[k].name] = forms(a, G, nullptr);
                    else if (a.kind == pf::Expr::Var && G.arrays.count(a.name)) S.arrays[s->params[k].name] = G.arrays[a.name];
                }
                if (s->body) stmt(*s->body, S);
            }
        } else if (g->body) {
            stmt(*g->body, G);
        }
        depth--;
    }

    static bool clamp_if(const pf::Stmt& s, std::string& var, bool& lower, const pf::Expr*& bound) {
        // if (v < e) v = e;   |   if (v > e) v = e;   (also <= / >=), no else
        if (s.kind != pf::Stmt::If || s.else_s || !s.cond || s.cond->kind != pf::Expr::Binary) return false;
        const pf::Expr& c = *s.cond;
        if (c.args.size() != 2 || c.args[0]->kind != pf::Expr::Var) return false;
        const pf::Stmt* t = s.then_s.get();
        while (t && t->kind == pf::Stmt::Block && t->body.size() == 1) t = t->body[0].get();
        if (!t || t->kind != pf::Stmt::Assign || t->aop != pf::AOp::Set || t->lhs->kind != pf::Expr::Var ||
            t->lhs->name != c.args[0]->name)
            return false;
        if (c.bop == pf::Bin::Lt || c.bop == pf::Bin::Le) lower = true;
        else if (c.bop == pf::Bin::Gt || c.bop == pf::Bin::Ge) lower = false;
        else return false;
        var = c.args[0]->name;
        bound = t->rhs.get();
        return true;
    }

    void stmt(const pf::Stmt& s, Frame& F) {
        switch (s.kind) {
            case pf::Stmt::Block:
                for (const auto& c : s.body) stmt(*c, F);
                break;
            case pf::Stmt::Decl:
                for (const auto& e : s.extents) expr(*e, F);
                if (s.extents.empty()) {
                    Local L;
                    if (s.rhs) {
                        expr(*s.rhs, F);
                        L.forms = forms(*s.rhs, F, nullptr);
                    }
                    F.locals[s.name] = L;
                }
                break;
            case pf::Stmt::Assign: {
                expr(*s.rhs, F);
                const pf::Expr& lv = *s.lhs;
                if (lv.kind == pf::Expr::Index) {
                    for (const auto& a : lv.args) expr(*a, F);
                    auto it = F.arrays.find(lv.name);
                    if (it != F.arrays.end() && lv.args.size() == 1) {
                        if (s.aop != pf::AOp::Set) record(it->second, *lv.args[0], false, F);
                        record(it->second, *lv.args[0], true, F);
                    }
                } else if (lv.kind == pf::Expr::Var && F.locals.count(lv.name)) {
                    Local& L = F.locals[lv.name];
                    if (s.aop == pf::AOp::Set) {
                        L.forms = forms(*s.rhs, F, nullptr);
                        L.lo.clear();
                        L.hi.clear();
                    } else {
                        L.forms.clear();  // a running sum: not an index
                    }
                }
                break;
            }
            case pf::Stmt::For: {
                expr(*s.lo, F);
                expr(*s.hi, F);
                Loop L;
                L.var = s.name + "#" + std::to_string(uniq++);
                const auto lo = forms(*s.lo, F, nullptr), hi = forms(*s.hi, F, nullptr);
                L.lo.ok = lo.size() == 1;
                if (L.lo.ok) L.lo = lo[0];
                L.hi.ok = hi.size() == 1;
                if (L.hi.ok) L.hi = hi[0];
                if (s.lo->kind == pf::Expr::Index && s.hi->kind == pf::Expr::Index && s.lo->name == s.hi->name &&
                    F.arrays.count(s.lo->name))
                    L.via = F.arrays[s.lo->name];
                const auto saved = F.loopname.count(s.name) ? F.loopname[s.name] : std::string();
                F.loopname[s.name] = L.var;
                loops.push_back(L);
                stmt(*s.loop_body, F);
                loops.pop_back();
                if (saved.empty()) F.loopname.erase(s.name);
                else F.loopname[s.name] = saved;
                break;
            }
            case pf::Stmt::While:
                expr(*s.cond, F);
                stmt(*s.loop_body, F);
                break;
            case pf::Stmt::If: {
                std::string v;
                bool lower = false;
                const pf::Expr* b = nullptr;
                expr(*s.cond, F);
                if (clamp_if(s, v, lower, b) && F.locals.count(v) && !F.locals[v].forms.empty()) {
                    auto f = forms(*b, F, nullptr);
                    auto& L = F.locals[v];
                    (lower ? L.lo : L.hi) = f;
                    break;
                }
                // other conditional assignments: the union of what either branch leaves
                std::map<std::string, Local> before = F.locals;
                stmt(*s.then_s, F);
                std::map<std::string, Local> after_then = F.locals;
                F.locals = before;
                if (s.else_s) stmt(*s.else_s, F);
                for (auto& [n, L] : F.locals) {
                    auto it = after_then.find(n);
                    if (it == after_then.end()) continue;
                    if (it->second.forms.empty() || L.forms.empty()) {
                        L.forms.clear();
                        continue;
                    }
                    for (const auto& f : it->second.forms) {
                        bool dup = false;
                        for (const auto& g : L.forms) dup |= g.coef == f.coef && g.c == f.c;
                        if (!dup) L.forms.push_back(f);
                    }
                }
                break;
            }
            case pf::Stmt::CallS: expr(*s.call, F); break;
            case pf::Stmt::Return:
                if (s.rhs) expr(*s.rhs, F);
                break;
            case pf::Stmt::Labeled: stmt(*s.loop_body, F); break;
            case pf::Stmt::Nop:
                if (s.summary >= 0 && s.lhs && s.lhs->kind == pf::Expr::Index && s.lhs->args.size() == 1) {
                    auto it = F.arrays.find(s.lhs->name);
                    if (it != F.arrays.end()) record(it->second, *s.lhs->args[0], s.summary != 1, F);
                }
                break;
        }
    }
};

bool has_pragma(const pf::Stmt& s, const char* word) {
    for (const auto& p : s.pragmas)
        if (p.find("pencil") != std::string::npos && p.find(word) != std::string::npos) return true;
    return false;
}
std::vector<std::string> reduction_vars(const pf::Stmt& s) {
    std::vector<std::string> v;
    for (const auto& p : s.pragmas) {
        const size_t a = p.find(':'), b = p.rfind(')');
        if (p.find("reduction") == std::string::npos || a == std::string::npos || b == std::string::npos || b < a) continue;
        std::string list = p.substr(a + 1, b - a - 1), cur;
        for (char ch : list + ",") {
            if (ch == ',') {
                if (!cur.empty()) v.push_back(cur);
                cur.clear();
            } else if (ch != ' ' && ch != '\t') {
                cur += ch;
            }
        }
    }
    return v;
}

// value of an affine form: loop variables from `at`, parameters from `env`, clamp markers applied
bool aeval(const Aff& a, const std::map<std::string, long long>& env, const std::map<std::string, long long>& at,
           long long& out) {
    if (!a.ok) return false;
    long long v;
    if (!peval(a.c, env, v)) return false;
    for (const auto& [var, p] : a.coef) {
        long long c;
        auto it = at.find(var);
        if (it == at.end() || !peval(p, env, c)) return false;
        v += c * it->second;
    }
    out = v;
    return true;
}

struct Class {
    std::string kind;  // block | view | via | all
    Poly stride;
    long long h0 = 0, h1 = 0;
    std::vector<std::string> inner;  // view: strides of the other loop variables (symbolic)
    std::string via;
};

std::string json_str(const std::string& s) { return "\"" + s + "\""; }

}  // namespace

extern "C" {

// JSON distribution plan of `fn` in `source` (see the file comment); returns the text length
// (cap 0 sizes the buffer) or -1 (parse error / no such function / no parallel loop).
long long pencil_dist_plan(const char* source, const char* fn, char* out, long long cap) {
    if (!source || !fn) return -1;
    pf::Unit unit;
    std::string err;
    if (!pf::parse_unit(source, unit, err)) {
        pencil_internal_fail(PENCIL_E_ARG, ("E-SYNTAX: " + err).c_str());
        return -1;
    }
    const pf::Func* f = unit.find(fn);
    if (!f || !f->body) return -1;
    // the distributed nest: the first top-level for with `independent` or `reduction`, and the
    // `independent` loop directly under it (2-D grid)
    const pf::Stmt* d0 = nullptr;
    const pf::Stmt* b = f->body.get();
    std::vector<const pf::Stmt*> top;
    if (b->kind == pf::Stmt::Block)
        for (const auto& c : b->body) top.push_back(c.get());
    else
        top.push_back(b);
    for (const auto* s : top)
        if (s->kind == pf::Stmt::For && (has_pragma(*s, "independent") || has_pragma(*s, "reduction"))) {
            d0 = s;
            break;
        }
    // no directive: the first top-level loop, distributable when every written array is owned
    // without halo (the analyzer's PARALLEL (AFFINE) / PARALLEL under an ACCESS summary)
    for (const auto* s : top)
        if (!d0 && s->kind == pf::Stmt::For) d0 = s;
    if (!d0) return -1;
    const pf::Stmt* d1 = nullptr;
    if (has_pragma(*d0, "independent")) {
        const pf::Stmt* inner = d0->loop_body.get();
        while (inner && inner->kind == pf::Stmt::Block && inner->body.size() == 1) inner = inner->body[0].get();
        if (inner && inner->kind == pf::Stmt::For && has_pragma(*inner, "independent")) d1 = inner;
    }

    Walker W(unit);
    Frame F;
    std::map<std::string, std::string> kinds;  // array -> dtype-free marker
    for (size_t i = 0; i < f->params.size(); i++) {
        if (f->params[i].kind == pf::Param::Scalar) W.params[f->params[i].name] = (int)i;
        else F.arrays[f->params[i].name] = f->params[i].name;
    }
    // walk the nest itself (the For statement): its loop var becomes "<name>#0"
    W.stmt(*d0, F);

    // sample binding: scalar parameters -> distinct values ~10^3
    std::map<std::string, long long> env;
    {
        int k = 0;
        for (const auto& [name, pos] : W.params) env[name] = 1000 + 37 * (k++) + (pos % 7);
    }
    // the nest's loop variables (as the walker named them)
    const std::string v0 = d0->name + "#0";
    std::string v1;
    if (d1)
        for (const auto& a : W.out)
            for (const auto& L : a.loops)
                if (L.var.rfind(d1->name + "#", 0) == 0 && v1.empty()) v1 = L.var;
    std::vector<std::string> dims = {v0};
    if (d1 && !v1.empty()) dims.push_back(v1);

    // an index form with its clamped locals replaced by their unclamped values (the symbolic
    // strides), and its value at a point with the clamps applied
    auto flat = [&](const Aff& fm, const std::map<std::string, ClampDef>& cl) {
        Aff r;
        r.ok = fm.ok;
        r.c = fm.c;
        for (const auto& [v, p] : fm.coef) {
            auto it = cl.find(v);
            if (it == cl.end()) {
                r.coef[v] = padd(r.coef[v], p);
                if (r.coef[v].empty()) r.coef.erase(v);
                continue;
            }
            Aff k, sc;
            k.c = p;
            amul(it->second.val, k, sc);
            r = aadd(r, sc, 1);
        }
        return r;
    };
    auto eval_at = [&](const Aff& fm, const std::map<std::string, ClampDef>& cl, std::map<std::string, long long> at,
                       long long& out) {
        for (const auto& [tag, def] : cl) {
            long long v;
            if (!aeval(def.val, env, at, v)) return false;
            for (const auto& bnd : def.lo) {
                long long x;
                if (aeval(bnd, env, at, x)) v = std::max(v, x);
            }
            for (const auto& bnd : def.hi) {
                long long x;
                if (aeval(bnd, env, at, x)) v = std::min(v, x);
            }
            at[tag] = v;
        }
        return aeval(fm, env, at, out);
    };

    // Class of one access relative to the distributed variable dv.  Each other variable of the
    // index (loop variables, clamped locals) is a halo variable when its term spans at most 8
    // blocks of the stride C, else a stride variable (the shard is then a strided view); the
    // halo is the range of the index minus C*d over the halo variables' corners.
    auto classify = [&](const Acc& a, const std::string& dv) -> Class {
        Class c;
        c.kind = "all";
        if (!a.via.empty()) {
            c.kind = "via";
            c.via = a.via;
            return c;
        }
        if (a.forms.empty()) return c;
        std::map<std::string, std::pair<long long, long long>> rng;  // loop var -> [lo, hi - 1]
        std::map<std::string, long long> pt;  // dv at an interior point, the others at their first
        for (const auto& L : a.loops) {
            long long lo = 0, hi = 0;
            if (!aeval(L.lo, env, pt, lo) || !aeval(L.hi, env, pt, hi) || hi <= lo) return c;
            rng[L.var] = {lo, hi - 1};
            pt[L.var] = L.var == dv ? lo + (hi - lo) / 2 : lo;
        }
        if (!rng.count(dv)) return c;
        const long long d_at = pt[dv];
        // the real loop variables an affine form (clamp pseudo-variables expanded) depends on
        auto real_vars = [&](const Aff& f, std::vector<std::string>& vs) {
            const Aff fl = flat(f, a.clamps);
            for (const auto& [v, p] : fl.coef)
                if (v != dv && std::find(vs.begin(), vs.end(), v) == vs.end()) vs.push_back(v);
        };
        // min / max of a form over the corners of `vs` (dv at d_at), clamps applied
        auto range_of = [&](const Aff& f, const std::vector<std::string>& vs, long long& mn, long long& mx) {
            for (long long m = 0; m < (1ll << vs.size()); m++) {
                std::map<std::string, long long> at = pt;
                for (size_t q = 0; q < vs.size(); q++) {
                    if (!rng.count(vs[q])) return false;
                    at[vs[q]] = ((m >> q) & 1) ? rng[vs[q]].second : rng[vs[q]].first;
                }
                long long val;
                if (!eval_at(f, a.clamps, at, val)) return false;
                if (m == 0 || val < mn) mn = val;
                if (m == 0 || val > mx) mx = val;
            }
            return true;
        };
        Poly C;
        bool first = true, view = false;
        long long hmin = 0, hmax = 0;
        std::vector<std::string> inner;
        for (const auto& fm : a.forms) {
            const Aff fl = flat(fm, a.clamps);
            auto it = fl.coef.find(dv);
            if (it == fl.coef.end() || it->second.empty()) return c;  // free of d: every iteration touches it
            if (!first && C != it->second) return c;
            C = it->second;
            long long Cv;
            if (!peval(C, env, Cv) || Cv <= 0) return c;
            // split the form's terms into halo terms and stride terms
            Aff halo_part;
            for (const auto& [mono, k] : fm.c) {  // constants: large ones belong to the stride terms
                Poly one{{mono, k}};
                long long v;
                if (!peval(one, env, v)) return c;
                if (v >= -8 * Cv && v <= 8 * Cv) halo_part.c = padd(halo_part.c, one);
            }
            for (const auto& [v, p] : fm.coef) {
                Aff term;
                term.coef[v] = p;
                std::vector<std::string> vs;
                real_vars(term, vs);
                long long mn = 0, mx = 0;
                if (!range_of(term, vs, mn, mx)) return c;
                const bool has_d = v == dv || (a.clamps.count(v) && a.clamps.at(v).val.coef.count(dv));
                if (has_d || mx - mn <= 8 * Cv) {
                    halo_part = aadd(halo_part, term, 1);
                    continue;
                }
                view = true;  // a stride term: report the strides of the loop variables inside it
                const Aff tf = flat(term, a.clamps);
                for (const auto& [u, q] : tf.coef) {
                    const std::string s = u.substr(0, u.find('#')) + ":" + pstr(q);
                    if (std::find(inner.begin(), inner.end(), s) == inner.end()) inner.push_back(s);
                }
            }
            std::vector<std::string> vs;
            real_vars(halo_part, vs);
            long long mn = 0, mx = 0;
            if (!range_of(halo_part, vs, mn, mx)) return c;
            const long long h0 = (long long)std::floor((double)(mn - d_at * Cv) / (double)Cv);
            const long long h1 = (long long)std::floor((double)(mx - d_at * Cv) / (double)Cv);
            if (h1 - h0 > 8) return c;
            hmin = first ? h0 : std::min(hmin, h0);
            hmax = first ? h1 : std::max(hmax, h1);
            first = false;
        }
        c.kind = view ? "view" : "block";
        c.stride = C;
        c.h0 = hmin;
        c.h1 = hmax;
        c.inner = inner;
        return c;
    };

    // parallel / reduction from the directive; a loop without one is "analyzed" (parallel by the
    // analysis: the affine fast path, or an ACCESS summary) when every array it
    // writes is owned in halo-free blocks, "serial" otherwise
    auto kind_of = [&](const pf::Stmt* L, const std::string& dv) -> std::string {
        if (has_pragma(*L, "independent")) return "parallel";
        if (has_pragma(*L, "reduction")) return "reduction";
        for (const auto& a : W.out) {
            if (!a.write) continue;
            const Class c = classify(a, dv);
            if (c.kind != "block" || c.h0 != 0 || c.h1 != 0) return "serial";
        }
        return "analyzed";
    };
    std::ostringstream o;
    o << "{\"function\":" << json_str(fn) << ",\"dims\":[";
    for (size_t di = 0; di < dims.size(); di++) {
        const pf::Stmt* L = di == 0 ? d0 : d1;
        const std::string& dv = dims[di];
        if (di) o << ",";
        o << "{\"var\":" << json_str(L->name) << ",\"kind\":" << json_str(kind_of(L, dv)) << ",\"reduce\":[";
        const auto rv = reduction_vars(*L);
        for (size_t k = 0; k < rv.size(); k++) o << (k ? "," : "") << json_str(rv[k]);
        o << "],\"arrays\":{";
        // per array: merge the classes of its accesses
        std::map<std::string, std::pair<std::string, Class>> merged;  // array -> (mode, class)
        std::vector<std::string> order;
        for (const auto& a : W.out) {
            Class c = classify(a, dv);
            auto it = merged.find(a.array);
            if (it == merged.end()) {
                order.push_back(a.array);
                merged[a.array] = {a.write ? "w" : "r", c};
                continue;
            }
            std::string& mode = it->second.first;
            if ((mode == "r" && a.write) || (mode == "w" && !a.write)) mode = "rw";
            Class& m = it->second.second;
            if (m.kind == c.kind && (m.kind == "block" || m.kind == "view") && m.stride == c.stride) {
                m.h0 = std::min(m.h0, c.h0);
                m.h1 = std::max(m.h1, c.h1);
                for (const auto& s : c.inner)
                    if (std::find(m.inner.begin(), m.inner.end(), s) == m.inner.end()) m.inner.push_back(s);
            } else if (m.kind == c.kind && m.kind == "via" && m.via == c.via) {
            } else if (m.kind != "all") {
                m = Class{};
                m.kind = "all";
            }
        }
        std::vector<std::string> own, halo, gather, conflict;
        for (size_t k = 0; k < order.size(); k++) {
            const auto& [mode, c] = merged[order[k]];
            if (k) o << ",";
            o << json_str(order[k]) << ":{\"mode\":" << json_str(mode) << ",\"kind\":" << json_str(c.kind);
            if (c.kind == "block" || c.kind == "view") o << ",\"stride\":" << json_str(pstr(c.stride));
            if (c.kind == "block" || c.kind == "view") o << ",\"halo\":[" << c.h0 << "," << c.h1 << "]";
            if (c.kind == "view") {
                o << ",\"inner\":[";
                for (size_t q = 0; q < c.inner.size(); q++) o << (q ? "," : "") << json_str(c.inner[q]);
                o << "]";
            }
            if (c.kind == "via") o << ",\"via\":" << json_str(c.via);
            o << "}";
            const bool w = mode != "r";
            if (w && c.kind == "all") conflict.push_back(order[k]);
            else if (w) own.push_back(order[k]);
            else if (c.kind == "all") gather.push_back(order[k]);
            else if ((c.kind == "block" || c.kind == "view") && (c.h0 != 0 || c.h1 != 0)) halo.push_back(order[k]);
        }
        auto list = [&](const char* key, const std::vector<std::string>& v) {
            o << ",\"" << key << "\":[";
            for (size_t q = 0; q < v.size(); q++) o << (q ? "," : "") << json_str(v[q]);
            o << "]";
        };
        o << "}";
        list("owned", own);
        list("halo", halo);
        list("replicated", gather);
        list("conflicts", conflict);
        o << "}";
    }
    o << "]}";
    const std::string r = o.str();
    if (out && cap > 0) {
        const size_t n = std::min<size_t>(r.size(), (size_t)cap - 1);
        memcpy(out, r.data(), n);
        out[n] = 0;
    }
    pencil_internal_ok();
    return (long long)r.size();
}

}  // extern "C"
