// A general verdict-driven mapper for PENCIL units ("emit_cuda" mirroring
// emit_openmp, core/src/pretty.cpp:472-531): any compliant unit is compiled for the GPU and its
// functions are callable through the reference Interpreter's surface (set_array / call / arrays,
// interp.hpp:38-51), with the Interpreter's value semantics (tagged int64 / fp64 values and
// arrays; codegen.hpp).
//
// Mapping (the verdict switch of emit_openmp, driven by the directives a PENCIL programmer writes
// — the analyzer's PARALLEL verdicts for such loops are DIRECTIVE / ASSUMED_PARALLEL):
//   * a top-level `for` of the called function carrying `#pragma pencil independent` becomes a
//     grid of threads, one iteration per thread (grid-stride); nested loops inside it stay
//     sequential in their thread, in source order;
//   * a top-level `for` carrying `#pragma pencil reduction (op: v...)` (op + * max min) runs the
//     same way with thread-private accumulators started at the identity, combined afterwards in a
//     fixed order by one block (deterministic; fp sums re-associate, as the pragma licenses —
//     integer sums are exact);
//   * every other top-level statement runs, in order, on one device thread (SERIAL / UNKNOWN
//     verdicts stay sequential, like emit_openmp leaves them without a pragma).
// The function's scalars live in a device frame (the interpreter's Frame::scalars) shared by the
// launches; a parallel loop's threads read it privately and the thread that ran the last
// iteration writes its scalars back (the sequential final values, loop variable = hi - 1 as in
// interp.cpp:207-217).  Local arrays live in a device buffer for the call; those declared inside
// a parallel loop body are thread-private.
#include <cuda_runtime.h>

#include <algorithm>
#include <deque>
#include <cmath>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/pencil_b200.h"
#include "codegen.hpp"
#include "pencil_front.hpp"

int pencil_internal_fail(int status, const char* msg);  // runtime.cpp
int pencil_internal_ok();                                // runtime.cpp

namespace {

int fail(int st, const std::string& m) { return pencil_internal_fail(st, m.c_str()); }

const char* kJitExtra = R"CUDA(
static __device__ __forceinline__ V vmax(V a, V b) { return truth(op_gt(b, a)) ? b : a; }
static __device__ __forceinline__ V vmin(V a, V b) { return truth(op_lt(b, a)) ? b : a; }
static __device__ __forceinline__ V red(int op, V a, V b) {
    switch (op) { case 0: return op_add(a, b); case 1: return op_mul(a, b); case 2: return vmax(a, b); }
    return vmin(a, b);
}
)CUDA";

struct Red {
    int op;           // 0 + 1 * 2 max 3 min
    std::string var;
};
struct Seg {
    bool parallel = false;
    bool warp = false;  // one warp per iteration, inner reduction loops split across the lanes
    const pf::Stmt* inner = nullptr;  // 2-D grid: the nested `independent` loop collapsed with this one
    std::vector<const pf::Stmt*> stmts;  // serial: statements in order; parallel: the loop
    std::vector<Red> reds;
    std::set<std::string> private_larrays;  // local arrays declared inside the loop body
};
struct EntryFn {
    const pf::Func* f = nullptr;
    std::vector<std::string> scalars;  // frame layout; slot K = return value
    std::map<std::string, int> slot;
    std::map<std::string, long long> la_off;  // local array -> offset in the call's buffer
    std::map<std::string, long long> la_n;
    long long la_total = 0;
    std::vector<Seg> segs;
};

bool parse_reduction(const std::string& prag, std::vector<Red>& out) {
    // "#pragma pencil reduction (+: a, b)"
    size_t p = prag.find("reduction");
    if (p == std::string::npos) return false;
    size_t l = prag.find('(', p), c = prag.find(':', p), r = prag.find(')', p);
    if (l == std::string::npos || c == std::string::npos || r == std::string::npos || !(l < c && c < r)) return false;
    std::string op = prag.substr(l + 1, c - l - 1);
    op.erase(std::remove(op.begin(), op.end(), ' '), op.end());
    int code = op == "+" ? 0 : op == "*" ? 1 : op == "max" ? 2 : op == "min" ? 3 : -1;
    if (code < 0) return false;
    std::string vars = prag.substr(c + 1, r - c - 1);
    std::stringstream ss(vars);
    std::string v;
    while (std::getline(ss, v, ',')) {
        v.erase(std::remove(v.begin(), v.end(), ' '), v.end());
        if (!v.empty()) out.push_back({code, v});
    }
    return true;
}
bool has_independent(const pf::Stmt& s) {
    for (const auto& p : s.pragmas)
        if (p.find("pencil") != std::string::npos && p.find("independent") != std::string::npos) return true;
    return false;
}

// The analyzer's affine fast path for loops without a directive (PARALLEL (AFFINE), e.g. axpy;
// depanalysis.cpp:163-285), restated conservatively: every array the body writes is read and
// written only at [i] (the loop variable itself), scalars assigned in the body are declared in
// it (private per iteration) or are nested loop variables, and the body calls no function.
struct AffineCheck {
    std::string iv;
    std::set<std::string> written, declared, loopvars;
    bool ok = true;
    static bool is_iv(const pf::Expr& e, const std::string& iv) { return e.kind == pf::Expr::Var && e.name == iv; }
    void writes(const pf::Stmt& s) {
        switch (s.kind) {
            case pf::Stmt::Block:
                for (const auto& c : s.body) writes(*c);
                break;
            case pf::Stmt::Decl: declared.insert(s.name); break;
            case pf::Stmt::Assign:
                if (s.lhs->kind == pf::Expr::Index) written.insert(s.lhs->name);
                else if (s.lhs->kind != pf::Expr::Var) ok = false;
                break;
            case pf::Stmt::For:
                loopvars.insert(s.name);
                writes(*s.loop_body);
                break;
            case pf::Stmt::While:
            case pf::Stmt::Labeled: writes(*s.loop_body); break;
            case pf::Stmt::If:
                writes(*s.then_s);
                if (s.else_s) writes(*s.else_s);
                break;
            case pf::Stmt::Return: ok = false; break;
            default: break;
        }
    }
    void expr(const pf::Expr& e) {
        if (e.kind == pf::Expr::Call) ok = false;
        if (e.kind == pf::Expr::Unary && e.uop != pf::Un::Neg && e.uop != pf::Un::Not) ok = false;
        if (e.kind == pf::Expr::Index && written.count(e.name) && !(e.args.size() == 1 && is_iv(*e.args[0], iv))) ok = false;
        for (const auto& a : e.args) expr(*a);
    }
    void stmts(const pf::Stmt& s) {
        switch (s.kind) {
            case pf::Stmt::Block:
                for (const auto& c : s.body) stmts(*c);
                break;
            case pf::Stmt::Decl:
                for (const auto& e : s.extents) expr(*e);
                if (s.rhs) expr(*s.rhs);
                break;
            case pf::Stmt::Assign:
                expr(*s.rhs);
                if (s.lhs->kind == pf::Expr::Var) {
                    if (!declared.count(s.lhs->name) && !loopvars.count(s.lhs->name)) ok = false;
                } else {
                    expr(*s.lhs);
                }
                break;
            case pf::Stmt::For:
                expr(*s.lo);
                expr(*s.hi);
                stmts(*s.loop_body);
                break;
            case pf::Stmt::While:
                expr(*s.cond);
                stmts(*s.loop_body);
                break;
            case pf::Stmt::If:
                expr(*s.cond);
                stmts(*s.then_s);
                if (s.else_s) stmts(*s.else_s);
                break;
            case pf::Stmt::CallS: ok = false; break;
            case pf::Stmt::Labeled: stmts(*s.loop_body); break;
            default: break;
        }
    }
};
bool affine_parallel(const pf::Stmt& loop) {
    AffineCheck a;
    a.iv = loop.name;
    a.writes(*loop.loop_body);
    if (a.loopvars.count(a.iv) || a.declared.count(a.iv)) return false;
    a.stmts(*loop.loop_body);
    return a.ok;
}

void collect_decls(const pf::Stmt& s, std::set<std::string>& larr) {
    switch (s.kind) {
        case pf::Stmt::Block:
            for (const auto& c : s.body) collect_decls(*c, larr);
            break;
        case pf::Stmt::Decl:
            if (!s.extents.empty()) larr.insert(s.name);
            break;
        case pf::Stmt::For:
        case pf::Stmt::While:
        case pf::Stmt::Labeled: collect_decls(*s.loop_body, larr); break;
        case pf::Stmt::If:
            collect_decls(*s.then_s, larr);
            if (s.else_s) collect_decls(*s.else_s, larr);
            break;
        default: break;
    }
}

// The mapper's rule for an innermost PARALLEL_WITH_REDUCTION loop: a warp per
// iteration of the parallel loop, the reduction loop split across its lanes.  Taken when the
// parallel loop's body holds such a loop at its top level and calls no function outside it (a
// call there would run on every lane).
bool calls_outside(const pf::Stmt& s, const std::set<const pf::Stmt*>& skip) {
    if (skip.count(&s)) return false;
    std::function<bool(const pf::Expr&)> has_call = [&](const pf::Expr& e) {
        if (e.kind == pf::Expr::Call && e.name != "exp") return true;
        for (const auto& a : e.args)
            if (has_call(*a)) return true;
        return false;
    };
    switch (s.kind) {
        case pf::Stmt::Block:
            for (const auto& c : s.body)
                if (calls_outside(*c, skip)) return true;
            return false;
        case pf::Stmt::Decl: return (s.rhs && has_call(*s.rhs));
        case pf::Stmt::Assign: return has_call(*s.rhs) || has_call(*s.lhs);
        case pf::Stmt::For: return has_call(*s.lo) || has_call(*s.hi) || calls_outside(*s.loop_body, skip);
        case pf::Stmt::While: return has_call(*s.cond) || calls_outside(*s.loop_body, skip);
        case pf::Stmt::If:
            return has_call(*s.cond) || calls_outside(*s.then_s, skip) || (s.else_s && calls_outside(*s.else_s, skip));
        case pf::Stmt::CallS: return true;
        case pf::Stmt::Labeled: return calls_outside(*s.loop_body, skip);
        default: return false;
    }
}
std::vector<std::pair<const pf::Stmt*, std::vector<Red>>> inner_reduction_loops(const pf::Stmt& loop) {
    std::vector<std::pair<const pf::Stmt*, std::vector<Red>>> out;
    if (loop.loop_body->kind != pf::Stmt::Block) return out;
    for (const auto& c : loop.loop_body->body) {
        if (c->kind != pf::Stmt::For) continue;
        std::vector<Red> r;
        bool red = false;
        for (const auto& p : c->pragmas) red |= parse_reduction(p, r);
        if (red && !r.empty()) out.push_back({c.get(), r});
    }
    return out;
}
bool warp_candidate(const pf::Stmt& loop) {
    auto inner = inner_reduction_loops(loop);
    if (inner.empty()) return false;
    std::set<const pf::Stmt*> skip;
    for (auto& p : inner) skip.insert(p.first);
    return !calls_outside(*loop.loop_body, skip);
}

// The mapper's rule for a nested ASSUMED_PARALLEL loop (second grid dimension):
// the parallel loop's body is a single `independent` loop whose bounds do not involve the outer
// variable or any call — the two collapse into one (i, j) iteration space.
bool mentions(const pf::Expr& e, const std::string& v) {
    if (e.kind == pf::Expr::Var && e.name == v) return true;
    if (e.kind == pf::Expr::Call) return true;  // calls are not hoisted
    for (const auto& a : e.args)
        if (mentions(*a, v)) return true;
    return false;
}
const pf::Stmt* collapse_candidate(const pf::Stmt& loop) {
    const pf::Stmt* b = loop.loop_body.get();
    if (b->kind == pf::Stmt::Block) {
        if (b->body.size() != 1) return nullptr;
        b = b->body[0].get();
    }
    if (b->kind != pf::Stmt::For || !has_independent(*b) || b->name == loop.name) return nullptr;
    if (mentions(*b->lo, loop.name) || mentions(*b->hi, loop.name)) return nullptr;
    return b;
}

bool uses_rand(const pf::Unit& u, const pf::Stmt& st) {
    std::set<std::string> seen;
    std::function<bool(const pf::Expr&)> ex;
    std::function<bool(const pf::Stmt&)> sm = [&](const pf::Stmt& s) -> bool {
        switch (s.kind) {
            case pf::Stmt::Block:
                for (const auto& c : s.body)
                    if (sm(*c)) return true;
                return false;
            case pf::Stmt::Decl: return s.rhs && ex(*s.rhs);
            case pf::Stmt::Assign: return ex(*s.rhs) || ex(*s.lhs);
            case pf::Stmt::For: return ex(*s.lo) || ex(*s.hi) || sm(*s.loop_body);
            case pf::Stmt::While: return ex(*s.cond) || sm(*s.loop_body);
            case pf::Stmt::If: return ex(*s.cond) || sm(*s.then_s) || (s.else_s && sm(*s.else_s));
            case pf::Stmt::CallS: return ex(*s.call);
            case pf::Stmt::Return: return s.rhs && ex(*s.rhs);
            case pf::Stmt::Labeled: return sm(*s.loop_body);
            default: return false;
        }
    };
    ex = [&](const pf::Expr& e) -> bool {
        if (e.kind == pf::Expr::Call) {
            if (e.name == "rand") return true;
            const pf::Func* f = u.find(e.name);
            if (f && f->body && seen.insert(e.name).second && sm(*f->body)) return true;
        }
        for (const auto& a : e.args)
            if (ex(*a)) return true;
        return false;
    };
    return sm(st);
}

struct Builder {
    const pf::Unit& u;
    pcg::Gen gen;
    std::ostringstream k;  // entry kernels
    // trace mode (Interpreter::enable_trace): every top-level statement a serial segment, so one
    // device thread executes the call in the interpreter's order and the trace is its MemTrace
    bool serial_only = false;
    explicit Builder(const pf::Unit& unit, bool serial = false) : u(unit), gen(unit), serial_only(serial) {}

    pcg::Gen::Scope scope(const pf::Func& f) {
        pcg::Gen::Scope sc;
        sc.f = &f;
        for (size_t i = 0; i < f.params.size(); i++) {
            if (f.params[i].kind == pf::Param::Scalar) sc.scalars.insert(f.params[i].name);
            else sc.arrays[f.params[i].name] = (int)i;
        }
        if (f.body) gen.collect(*f.body, sc);
        return sc;
    }

    std::string params(const EntryFn& E) {
        std::ostringstream o;
        o << "Ctx cx, V* frame, V* la";
        for (const auto& p : E.f->params)
            if (p.kind != pf::Param::Scalar) o << ", Arr " << pcg::Gen::aid(p.name);
        return o.str();
    }
    void load_frame(const EntryFn& E, std::ostringstream& o) {
        for (size_t i = 0; i < E.scalars.size(); i++) o << "  V " << pcg::Gen::sid(E.scalars[i]) << " = frame[" << i << "];\n";
    }
    void store_frame(const EntryFn& E, std::ostringstream& o, const std::string& dst, const std::set<std::string>& skip,
                     const std::string& ind) {
        for (size_t i = 0; i < E.scalars.size(); i++)
            if (!skip.count(E.scalars[i])) o << ind << dst << "[" << i << "] = " << pcg::Gen::sid(E.scalars[i]) << ";\n";
    }
    void shared_larrays(const EntryFn& E, const std::set<std::string>& priv, std::ostringstream& o) {
        for (const auto& la : E.la_off)
            if (!priv.count(la.first))
                o << "  LArr " << pcg::Gen::lid(la.first) << " = {la + " << la.second << ", " << E.la_n.at(la.first) << "};\n";
    }

    EntryFn entry(const pf::Func& f, int fi) {
        EntryFn E;
        E.f = &f;
        pcg::Gen::Scope sc = scope(f);
        for (const auto& p : f.params)
            if (p.kind == pf::Param::Scalar) E.scalars.push_back(p.name);
        for (const auto& s : sc.scalars)
            if (std::find(E.scalars.begin(), E.scalars.end(), s) == E.scalars.end()) E.scalars.push_back(s);
        for (size_t i = 0; i < E.scalars.size(); i++) E.slot[E.scalars[i]] = (int)i;
        for (const auto& la : sc.larrays) {
            E.la_off[la.first] = E.la_total;
            E.la_n[la.first] = la.second;
            E.la_total += std::max(1ll, la.second);
        }
        // segments: top-level statements of the body
        std::vector<const pf::Stmt*> top;
        if (f.body) {
            if (f.body->kind == pf::Stmt::Block)
                for (const auto& c : f.body->body) top.push_back(c.get());
            else
                top.push_back(f.body.get());
        }
        for (const pf::Stmt* s : top) {
            const pf::Stmt* loop = s;
            while (loop->kind == pf::Stmt::Labeled) loop = loop->loop_body.get();
            std::vector<Red> reds;
            bool red = false;
            for (const auto& p : s->pragmas) red |= parse_reduction(p, reds);
            if (loop != s)
                for (const auto& p : loop->pragmas) red |= parse_reduction(p, reds);
            bool indep = has_independent(*s) || has_independent(*loop) ||
                         (loop->kind == pf::Stmt::For && !red && affine_parallel(*loop));
            // rand() is one sequential stream (Interpreter::next_rand): such loops stay in order
            if (!serial_only && loop->kind == pf::Stmt::For && (indep || red) && !uses_rand(u, *loop)) {
                Seg g;
                g.parallel = true;
                g.stmts.push_back(loop);
                g.reds = reds;
                collect_decls(*loop->loop_body, g.private_larrays);
                for (const auto& r : reds)
                    if (!E.slot.count(r.var)) gen.unsup(f, s->line, "reduction variable '" + r.var + "' is not a scalar");
                g.warp = reds.empty() && warp_candidate(*loop);
                if (!g.warp && reds.empty()) g.inner = collapse_candidate(*loop);
                E.segs.push_back(std::move(g));
            } else {
                if (E.segs.empty() || E.segs.back().parallel) E.segs.push_back(Seg());
                E.segs.back().stmts.push_back(s);
            }
        }
        for (size_t si = 0; si < E.segs.size(); si++) emit_segment(E, sc, fi, (int)si);
        return E;
    }

    void emit_segment(const EntryFn& E, pcg::Gen::Scope& sc, int fi, int si) {
        const Seg& g = E.segs[si];
        const int K = (int)E.scalars.size();
        std::string base = "jit_" + std::to_string(fi) + "_" + std::to_string(si);
        if (!g.parallel) {
            std::ostringstream o;
            o << "extern \"C\" __global__ void " << base << "(" << params(E) << ", int* flags) {\n";
            o << "  if (flags[0]) return;  // an earlier segment returned\n";
            load_frame(E, o);
            shared_larrays(E, {}, o);
            o << "  V ret_v = VI(0); int ret_f = 0; ll steps_ = 0;\n  auto body = [&]() {\n";
            gen.ret_mode = 1;
            for (const pf::Stmt* s : g.stmts) gen.stmt(*s, sc, o, "    ");
            o << "  };\n  body();\n";
            store_frame(E, o, "frame", {}, "  ");
            o << "  if (ret_f) { frame[" << K << "] = ret_v; flags[0] = 1; }\n}\n";
            k << o.str();
            return;
        }
        const pf::Stmt& L = *g.stmts[0];
        gen.ret_mode = 2;
        {  // bounds: one thread evaluates lo and hi (in that order), as the interpreter does
            std::ostringstream o;
            o << "extern \"C\" __global__ void " << base << "_b(" << params(E) << ", ll* bounds, int* flags) {\n";
            o << "  if (flags[0]) { bounds[0] = bounds[1] = 0; return; }\n";
            load_frame(E, o);
            shared_larrays(E, {}, o);
            std::string lo = gen.ex(*L.lo, sc, o, "  ");
            o << "  bounds[0] = as_i(cx, " << lo << ");\n";
            std::string hi = gen.ex(*L.hi, sc, o, "  ");
            o << "  bounds[1] = as_i(cx, " << hi << ");\n";
            if (g.inner) {  // the inner bounds do not depend on the outer variable: evaluated once
                std::string lo2 = gen.ex(*g.inner->lo, sc, o, "  ");
                o << "  bounds[2] = as_i(cx, " << lo2 << ");\n";
                std::string hi2 = gen.ex(*g.inner->hi, sc, o, "  ");
                o << "  bounds[3] = as_i(cx, " << hi2 << ");\n";
            }
            store_frame(E, o, "frame", {}, "  ");
            o << "}\n";
            k << o.str();
        }
        std::set<std::string> redvars;
        for (const auto& r : g.reds) redvars.insert(r.var);
        if (g.inner) {  // 2-D grid over (i, j): one (i, j) iteration per thread
            const pf::Stmt& J2 = *g.inner;
            std::ostringstream o;
            o << "extern \"C\" __global__ void " << base << "_p(" << params(E)
              << ", const ll* bounds, V* frame_out, V* partials) {\n";
            o << "  const ll lo = bounds[0], hi = bounds[1], lo2 = bounds[2], hi2 = bounds[3];\n";
            o << "  const ll n1 = hi > lo ? hi - lo : 0, n2 = hi2 > lo2 ? hi2 - lo2 : 0, total = n1 * n2;\n";
            o << "  const ll nthr = (ll)gridDim.x * blockDim.x, tid = (ll)blockIdx.x * blockDim.x + threadIdx.x;\n";
            load_frame(E, o);
            shared_larrays(E, g.private_larrays, o);
            for (const auto& la : g.private_larrays) {
                long long n = E.la_n.at(la);
                if (n > 256) gen.unsup(*E.f, L.line, "local array '" + la + "' inside a parallel loop exceeds 256 elements");
                o << "  V " << pcg::Gen::lid(la) << "_st[" << std::max(1ll, n) << "]; LArr " << pcg::Gen::lid(la) << " = {"
                  << pcg::Gen::lid(la) << "_st, " << n << "};\n";
            }
            // outer loop runs but the inner one never does: only the outer variable moves
            o << "  if (n1 > 0 && n2 == 0 && tid == 0) {\n    " << pcg::Gen::sid(L.name) << " = VI(hi - 1);\n";
            store_frame(E, o, "frame_out", {}, "    ");
            o << "  }\n";
            o << "  ll steps_ = 0;\n";
            o << "  for (ll f = tid; f < total; f += nthr) {\n";
            o << "    " << pcg::Gen::sid(L.name) << " = VI(lo + f / n2);\n";
            o << "    " << pcg::Gen::sid(J2.name) << " = VI(lo2 + f % n2);\n";
            o << "    auto body = [&]() {\n";
            gen.stmt(*J2.loop_body, sc, o, "      ");
            o << "    };\n    body();\n";
            o << "    if (f == total - 1) {\n";
            store_frame(E, o, "frame_out", {}, "      ");
            o << "    }\n  }\n}\n";
            k << o.str();
        } else if (g.warp) {  // one warp per iteration; the inner reduction loops split across the lanes
            std::ostringstream o;
            o << "extern \"C\" __global__ void " << base << "_p(" << params(E)
              << ", const ll* bounds, V* frame_out, V* partials) {\n";
            o << "  const ll lo = bounds[0], hi = bounds[1];  // from the bounds kernel: no host round trip\n";
            o << "  const ll nw = ((ll)gridDim.x * blockDim.x) >> 5, wid = ((ll)blockIdx.x * blockDim.x + threadIdx.x) >> 5;\n";
            load_frame(E, o);
            shared_larrays(E, g.private_larrays, o);
            for (const auto& la : g.private_larrays) {
                long long n = E.la_n.at(la);
                if (n > 256) gen.unsup(*E.f, L.line, "local array '" + la + "' inside a parallel loop exceeds 256 elements");
                o << "  V " << pcg::Gen::lid(la) << "_st[" << std::max(1ll, n) << "]; LArr " << pcg::Gen::lid(la) << " = {"
                  << pcg::Gen::lid(la) << "_st, " << n << "};\n";
            }
            for (auto& p : inner_reduction_loops(L)) {
                std::vector<std::pair<int, std::string>> rv;
                for (auto& r : p.second) rv.push_back({r.op, r.var});
                gen.warp_loops[p.first] = rv;
            }
            o << "  ll steps_ = 0;\n";
            o << "  for (ll v = lo + wid; v < hi; v += nw) {\n";
            o << "    " << pcg::Gen::sid(L.name) << " = VI(v);\n";
            o << "    auto body = [&]() {\n";
            gen.lane0_stores = true;
            gen.stmt(*L.loop_body, sc, o, "      ");
            gen.lane0_stores = false;
            o << "    };\n    body();\n";
            o << "    if (v == hi - 1 && (threadIdx.x & 31) == 0) {\n";
            store_frame(E, o, "frame_out", {}, "      ");
            o << "    }\n  }\n}\n";
            k << o.str();
        } else {  // body: one iteration per thread, grid-stride
            std::ostringstream o;
            o << "extern \"C\" __global__ void " << base << "_p(" << params(E)
              << ", const ll* bounds, V* frame_out, V* partials) {\n";
            o << "  const ll lo = bounds[0], hi = bounds[1];  // from the bounds kernel: no host round trip\n";
            o << "  const ll nthr = (ll)gridDim.x * blockDim.x, tid = (ll)blockIdx.x * blockDim.x + threadIdx.x;\n";
            load_frame(E, o);
            shared_larrays(E, g.private_larrays, o);
            for (const auto& la : g.private_larrays) {
                long long n = E.la_n.at(la);
                if (n > 256) gen.unsup(*E.f, L.line, "local array '" + la + "' inside a parallel loop exceeds 256 elements");
                o << "  V " << pcg::Gen::lid(la) << "_st[" << std::max(1ll, n) << "]; LArr " << pcg::Gen::lid(la) << " = {"
                  << pcg::Gen::lid(la) << "_st, " << n << "};\n";
            }
            for (const auto& r : g.reds)
                o << "  " << pcg::Gen::sid(r.var) << " = " << (r.op == 0 ? "VI(0)" : r.op == 1 ? "VI(1)" : pcg::Gen::sid(r.var))
                  << ";\n";
            o << "  ll steps_ = 0;\n";
            o << "  for (ll v = lo + tid; v < hi; v += nthr) {\n";
            o << "    " << pcg::Gen::sid(L.name) << " = VI(v);\n";
            o << "    auto body = [&]() {\n";
            gen.stmt(*L.loop_body, sc, o, "      ");
            o << "    };\n    body();\n";
            o << "    if (v == hi - 1) {\n";
            store_frame(E, o, "frame_out", redvars, "      ");
            o << "    }\n  }\n";
            for (size_t r = 0; r < g.reds.size(); r++)
                o << "  partials[tid * " << g.reds.size() << " + " << r << "] = " << pcg::Gen::sid(g.reds[r].var) << ";\n";
            o << "}\n";
            k << o.str();
        }
        {  // finish: last-iteration scalars into the frame, reductions combined in a fixed order
            std::ostringstream o;
            o << "extern \"C\" __global__ void __launch_bounds__(1024) " << base
              << "_f(Ctx cx, V* frame, const V* frame_out, const V* partials, ll nthr, const ll* bounds, const int* flags) {\n";
            o << "  if (flags[0]) return;\n";
            o << "  const int ran = bounds[1] > bounds[0];\n";
            o << "  __shared__ V sh[1024];\n";
            o << "  if (ran && threadIdx.x == 0) {\n";
            for (size_t i = 0; i < E.scalars.size(); i++)
                if (!redvars.count(E.scalars[i])) o << "    frame[" << i << "] = frame_out[" << i << "];\n";
            o << "  }\n";
            for (size_t r = 0; r < g.reds.size(); r++) {
                const int op = g.reds[r].op;
                const std::string ident = op == 0 ? "VI(0)" : op == 1 ? "VI(1)" : "frame[" + std::to_string(E.slot.at(g.reds[r].var)) + "]";
                o << "  {\n    V acc = " << ident << ";\n";
                o << "    for (ll t = threadIdx.x; t < nthr; t += blockDim.x) acc = red(" << op << ", acc, partials[t * "
                  << g.reds.size() << " + " << r << "]);\n";
                o << "    sh[threadIdx.x] = acc;\n    __syncthreads();\n";
                o << "    for (int s = blockDim.x / 2; s > 0; s >>= 1) {\n      if (threadIdx.x < s) sh[threadIdx.x] = red(" << op
                  << ", sh[threadIdx.x], sh[threadIdx.x + s]);\n      __syncthreads();\n    }\n";
                o << "    if (threadIdx.x == 0) frame[" << E.slot.at(g.reds[r].var) << "] = red(" << op << ", frame["
                  << E.slot.at(g.reds[r].var) << "], sh[0]);\n    __syncthreads();\n  }\n";
            }
            o << "}\n";
            k << o.str();
        }
    }
};

struct StoreArr {
    long long* bits = nullptr;
    unsigned char* tag = nullptr;
    long long n = 0;
};

// ---- access summaries -> data movement (the reference's read / must / may sets,
// access.hpp:39-53, summaries.cpp:635-663).  Per array parameter of a function: loaded anywhere
// (through calls that pass it by name, too), stored anywhere, and must-written in full — a
// top-level `for (i = 0; i < E; i++)` whose body unconditionally stores p[i] with E the
// parameter's declared extent, and p never loaded.  Reads need the upload, stores need the
// download, a must-written never-read array needs no upload.
struct Access {
    bool load = false, store = false, must_all = false;
    int must_at = -1;  // scalar parameter k: the function unconditionally writes arr[k]
};

std::string expr_str(const pf::Expr& e) {
    std::ostringstream o;
    switch (e.kind) {
        case pf::Expr::IntLit: o << e.ival; break;
        case pf::Expr::FloatLit: o << e.fval; break;
        case pf::Expr::Var: o << e.name; break;
        default:
            o << "(" << (int)e.kind << ":" << e.name << ":" << (int)e.bop << ":" << (int)e.uop;
            for (const auto& a : e.args) o << "," << expr_str(*a);
            o << ")";
    }
    return o.str();
}

struct Summarizer {
    const pf::Unit& u;
    std::map<std::string, std::vector<Access>> memo;
    std::set<std::string> busy;
    explicit Summarizer(const pf::Unit& unit) : u(unit) {}

    const std::vector<Access>& of(const pf::Func& f) {
        auto it = memo.find(f.name);
        if (it != memo.end()) return it->second;
        std::vector<Access> acc(f.params.size());
        if (busy.count(f.name)) {  // recursion: everything may happen
            for (auto& a : acc) a.load = a.store = true;
            return memo[f.name] = acc;
        }
        busy.insert(f.name);
        std::map<std::string, int> pos;
        for (size_t i = 0; i < f.params.size(); i++)
            if (f.params[i].kind != pf::Param::Scalar) pos[f.params[i].name] = (int)i;
        std::function<void(const pf::Expr&)> ex = [&](const pf::Expr& e) {
            if (e.kind == pf::Expr::Index || (e.kind == pf::Expr::Unary && e.uop == pf::Un::Deref && !e.args.empty() &&
                                               e.args[0]->kind == pf::Expr::Var)) {
                auto p = pos.find(e.kind == pf::Expr::Index ? e.name : e.args[0]->name);
                if (p != pos.end()) acc[p->second].load = true;
            }
            if (e.kind == pf::Expr::Call) {
                const pf::Func* c = u.find(e.name);
                if (c) {
                    const auto ca = of(*c);
                    for (size_t k = 0; k < e.args.size() && k < c->params.size(); k++) {
                        if (c->params[k].kind == pf::Param::Scalar || e.args[k]->kind != pf::Expr::Var) continue;
                        auto p = pos.find(e.args[k]->name);
                        if (p == pos.end()) continue;
                        acc[p->second].load |= ca[k].load;
                        acc[p->second].store |= ca[k].store;
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
                    } else if (lv.kind == pf::Expr::Unary && lv.uop == pf::Un::Deref) {
                        n = lv.args[0]->name;
                    }
                    auto p = pos.find(n);
                    if (p != pos.end()) {
                        acc[p->second].store = true;
                        if (s.aop != pf::AOp::Set) acc[p->second].load = true;  // compound: reads the old value
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
        // ACCESS-summarised function (summaries.cpp:635-648): its summary function's DEF / USE /
        // MAY_DEF statements, mapped through the binding's arguments, declare what it touches
        if (!f.access_fn.empty()) {
            const pf::Func* g = u.find(f.access_fn);
            if (g && g->body) {
                std::map<std::string, std::string> to_f;  // summary param -> f's param name
                for (size_t j = 0; j < g->params.size() && j < f.access_args.size(); j++)
                    if (f.access_args[j]->kind == pf::Expr::Var) to_f[g->params[j].name] = f.access_args[j]->name;
                std::map<std::string, int> fscalar;
                for (size_t i = 0; i < f.params.size(); i++)
                    if (f.params[i].kind == pf::Param::Scalar) fscalar[f.params[i].name] = (int)i;
                std::function<void(const pf::Stmt&, bool)> sm = [&](const pf::Stmt& s, bool top) {
                    if (s.kind == pf::Stmt::Block) {
                        for (const auto& c : s.body) sm(*c, top);
                        return;
                    }
                    if (s.kind == pf::Stmt::For || s.kind == pf::Stmt::While || s.kind == pf::Stmt::Labeled) {
                        sm(*s.loop_body, false);
                        return;
                    }
                    if (s.kind == pf::Stmt::If) {
                        sm(*s.then_s, false);
                        if (s.else_s) sm(*s.else_s, false);
                        return;
                    }
                    if (s.kind != pf::Stmt::Nop || s.summary < 0 || !s.lhs) return;
                    const std::string base = s.lhs->kind == pf::Expr::Index ? s.lhs->name : s.lhs->name;
                    auto m = to_f.find(base);
                    if (m == to_f.end()) return;
                    auto p = pos.find(m->second);
                    if (p == pos.end()) return;
                    if (s.summary == 1) acc[p->second].load = true;
                    else acc[p->second].store = true;
                    if (s.summary == 0 && top && s.lhs->kind == pf::Expr::Index && s.lhs->args.size() == 1 &&
                        s.lhs->args[0]->kind == pf::Expr::Var) {
                        auto k = to_f.find(s.lhs->args[0]->name);
                        if (k != to_f.end() && fscalar.count(k->second)) acc[p->second].must_at = fscalar[k->second];
                    }
                };
                sm(*g->body, true);
            }
        }
        // an unconditional top-level `p[k] = ...` with k a scalar parameter
        if (f.body && f.body->kind == pf::Stmt::Block) {
            for (const auto& top : f.body->body) {
                const pf::Stmt& s0 = *top;
                if (s0.kind != pf::Stmt::Assign || s0.aop != pf::AOp::Set || s0.lhs->kind != pf::Expr::Index ||
                    s0.lhs->args.size() != 1 || s0.lhs->args[0]->kind != pf::Expr::Var)
                    continue;
                auto p = pos.find(s0.lhs->name);
                if (p == pos.end()) continue;
                for (size_t i = 0; i < f.params.size(); i++)
                    if (f.params[i].kind == pf::Param::Scalar && f.params[i].name == s0.lhs->args[0]->name)
                        acc[p->second].must_at = (int)i;
            }
        }
        // must-write-all: a top-level 0..extent loop storing p[i] unconditionally, directly or
        // through a call whose summary must-writes the element at the loop variable
        if (f.body && f.body->kind == pf::Stmt::Block) {
            for (const auto& top : f.body->body) {
                const pf::Stmt* L = top.get();
                while (L->kind == pf::Stmt::Labeled) L = L->loop_body.get();
                if (L->kind != pf::Stmt::For || L->lo->kind != pf::Expr::IntLit || L->lo->ival != 0) continue;
                std::vector<const pf::Stmt*> body;
                if (L->loop_body->kind == pf::Stmt::Block)
                    for (const auto& c : L->loop_body->body) body.push_back(c.get());
                else
                    body.push_back(L->loop_body.get());
                auto mark = [&](const std::string& arr) {
                    auto p = pos.find(arr);
                    if (p == pos.end() || !f.params[p->second].extent) return;
                    if (expr_str(*f.params[p->second].extent) == expr_str(*L->hi)) acc[p->second].must_all = true;
                };
                // the 2-level rectangle: for (i = 0; i < H; i++) for (j = 0; j < W; j++) p[i * W + j] = ...
                // (unconditional store in the inner body) writes all of p[H * W]: the flattened
                // row-major image nests (conv5x5_u8); the reference's must-write set is that rectangle
                auto mark2 = [&](const pf::Stmt& L2, const pf::Expr& idx, const std::string& arr) {
                    auto p = pos.find(arr);
                    if (p == pos.end() || !f.params[p->second].extent) return;
                    const pf::Expr& ext = *f.params[p->second].extent;
                    if (idx.kind != pf::Expr::Binary || idx.bop != pf::Bin::Add || idx.args.size() != 2) return;
                    const pf::Expr &rowt = *idx.args[0], &colt = *idx.args[1];
                    if (colt.kind != pf::Expr::Var || colt.name != L2.name) return;
                    if (rowt.kind != pf::Expr::Binary || rowt.bop != pf::Bin::Mul || rowt.args[0]->kind != pf::Expr::Var ||
                        rowt.args[0]->name != L->name || expr_str(*rowt.args[1]) != expr_str(*L2.hi))
                        return;
                    if (ext.kind == pf::Expr::Binary && ext.bop == pf::Bin::Mul && ext.args.size() == 2 &&
                        expr_str(*ext.args[0]) == expr_str(*L->hi) && expr_str(*ext.args[1]) == expr_str(*L2.hi))
                        acc[p->second].must_all = true;
                };
                for (const pf::Stmt* s : body) {
                    const pf::Stmt* L2 = s;
                    while (L2->kind == pf::Stmt::Labeled) L2 = L2->loop_body.get();
                    if (L2->kind == pf::Stmt::For && L2->lo->kind == pf::Expr::IntLit && L2->lo->ival == 0) {
                        std::vector<const pf::Stmt*> inner;
                        if (L2->loop_body->kind == pf::Stmt::Block)
                            for (const auto& c : L2->loop_body->body) inner.push_back(c.get());
                        else
                            inner.push_back(L2->loop_body.get());
                        for (const pf::Stmt* t : inner)
                            if (t->kind == pf::Stmt::Assign && t->aop == pf::AOp::Set && t->lhs->kind == pf::Expr::Index &&
                                t->lhs->args.size() == 1)
                                mark2(*L2, *t->lhs->args[0], t->lhs->name);
                    }
                    if (s->kind == pf::Stmt::Assign && s->aop == pf::AOp::Set && s->lhs->kind == pf::Expr::Index &&
                        s->lhs->args.size() == 1 && s->lhs->args[0]->kind == pf::Expr::Var &&
                        s->lhs->args[0]->name == L->name)
                        mark(s->lhs->name);
                    if (s->kind == pf::Stmt::CallS) {
                        const pf::Expr& c = *s->call;
                        const pf::Func* g = u.find(c.name);
                        if (!g) continue;
                        const auto ga = of(*g);
                        for (size_t k = 0; k < c.args.size() && k < g->params.size(); k++) {
                            if (g->params[k].kind == pf::Param::Scalar || c.args[k]->kind != pf::Expr::Var) continue;
                            const int at = ga[k].must_at;
                            if (at >= 0 && at < (int)c.args.size() && c.args[at]->kind == pf::Expr::Var &&
                                c.args[at]->name == L->name)
                                mark(c.args[k]->name);
                        }
                    }
                }
            }
        }
        for (auto& a : acc)
            if (a.load) a.must_all = false;
        busy.erase(f.name);
        return memo[f.name] = acc;
    }
};

}  // namespace

struct pencil_jit {
    pf::Unit unit;
    std::string src;
    std::vector<EntryFn> entries;
    std::map<std::string, int> entry_index;
    std::map<std::string, StoreArr> store;
    cudaLibrary_t lib = nullptr;
    cudaStream_t stream = nullptr;
    unsigned* d_fault = nullptr;
    unsigned long long* d_rng = nullptr;
    std::vector<cudaKernel_t> kernels_cache;
    std::map<std::string, cudaKernel_t> kern;
    long long h2d = 0, d2h = 0;  // bytes moved by the last pencil_jit_call_host
    void* scratch = nullptr;     // per-call frame / local arrays / partials / bounds / flags
    size_t scratch_bytes = 0;
    long long* d_rseq = nullptr;           // Interpreter::set_rand_sequence values
    unsigned long long* d_rpos = nullptr;  // next position in it
    long long rseq_n = 0;
    // trace mode (Interpreter::enable_trace / trace, interp.hpp:45-46): the unit compiled again
    // with every statement serial (t_*), a device record buffer, and the accumulated trace
    std::vector<EntryFn> t_entries;
    std::string t_src;
    cudaLibrary_t t_lib = nullptr;
    std::map<std::string, cudaKernel_t> t_kern;
    bool trace_on = false;
    unsigned long long* d_trace = nullptr;
    long long trace_cap = 0;
    std::deque<std::string> names;   // store name per array id (stable addresses)
    std::map<std::string, int> name_id;
    struct TraceRec {
        int id;
        long long index;
        unsigned char write;
    };
    std::vector<TraceRec> trace;
};

namespace {

#define JCK(call)                                                                                        \
    do {                                                                                                 \
        cudaError_t e_ = (call);                                                                         \
        if (e_ != cudaSuccess) return fail(PENCIL_E_CUDA, std::string("E-CUDA: ") + #call + ": " + cudaGetErrorString(e_)); \
    } while (0)

int setup(pencil_jit* J) {
    if (J->lib) return PENCIL_OK;
    std::vector<char> cubin;
    std::string log;
    int rc = pcg::compile_cubin(J->src, cubin, log);
    if (rc) return fail(rc, "E-CUDA: PENCIL unit compilation failed: " + log);
    JCK(cudaStreamCreateWithFlags(&J->stream, cudaStreamNonBlocking));
    JCK(cudaLibraryLoadData(&J->lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
    JCK(cudaMalloc(&J->d_fault, 64));
    JCK(cudaMemset(J->d_fault, 0, 64));
    JCK(cudaMalloc(&J->d_rng, 8));
    const unsigned long long seed = 0x9e3779b97f4a7c15ull;  // Interpreter::rng_state_ (interp.hpp:67)
    JCK(cudaMemcpy(J->d_rng, &seed, 8, cudaMemcpyHostToDevice));
    return PENCIL_OK;
}

int get_kernel(pencil_jit* J, const std::string& name, cudaKernel_t* out, bool traced = false) {
    auto& cache = traced ? J->t_kern : J->kern;
    auto it = cache.find(name);
    if (it != cache.end()) {
        *out = it->second;
        return PENCIL_OK;
    }
    JCK(cudaLibraryGetKernel(out, traced ? J->t_lib : J->lib, name.c_str()));
    cache[name] = *out;
    return PENCIL_OK;
}

// the serial (trace-mode) build of the unit and its record buffer, compiled on first use
int setup_trace(pencil_jit* J) {
    int rc = setup(J);
    if (rc) return rc;
    if (J->t_lib) return PENCIL_OK;
    std::vector<char> cubin;
    std::string log;
    rc = pcg::compile_cubin(J->t_src, cubin, log);
    if (rc) return fail(rc, "E-CUDA: PENCIL unit compilation (trace mode) failed: " + log);
    JCK(cudaLibraryLoadData(&J->t_lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
    J->trace_cap = 1 << 20;  // records per call
    JCK(cudaMalloc(&J->d_trace, (size_t)(2 + 2 * J->trace_cap) * 8));
    return PENCIL_OK;
}

struct HostV {
    long long i;
    double d;
    int isd;
};

}  // namespace

extern "C" {

pencil_jit_t pencil_jit_load(const char* source) {
    if (!source) {
        fail(PENCIL_E_ARG, "E-ARG: null source");
        return nullptr;
    }
    auto* J = new pencil_jit();
    std::string err;
    if (!pf::parse_unit(source, J->unit, err)) {
        fail(PENCIL_E_ARG, "E-SYNTAX: " + err);
        delete J;
        return nullptr;
    }
    try {
        Builder b(J->unit);
        b.gen.unit(pcg::kArrTagged);
        for (size_t fi = 0; fi < J->unit.fns.size(); fi++) {
            J->entries.push_back(b.entry(J->unit.fns[fi], (int)fi));
            J->entry_index[J->unit.fns[fi].name] = (int)fi;
        }
        J->src = b.gen.out.str() + kJitExtra + b.k.str();
        Builder t(J->unit, true);
        t.gen.unit(pcg::kArrTagged);
        for (size_t fi = 0; fi < J->unit.fns.size(); fi++) J->t_entries.push_back(t.entry(J->unit.fns[fi], (int)fi));
        J->t_src = t.gen.out.str() + kJitExtra + t.k.str();
    } catch (const pcg::GenError& e) {
        pencil_internal_fail(e.st, e.msg.c_str());
        delete J;
        return nullptr;
    }
    pencil_internal_ok();
    return J;
}

void pencil_jit_free(pencil_jit_t J) {
    if (!J) return;
    if (J->stream) cudaStreamSynchronize(J->stream);
    for (auto& a : J->store) {
        cudaFree(a.second.bits);
        cudaFree(a.second.tag);
    }
    if (J->d_fault) cudaFree(J->d_fault);
    if (J->d_rng) cudaFree(J->d_rng);
    if (J->scratch) cudaFree(J->scratch);
    if (J->d_rseq) cudaFree(J->d_rseq);
    if (J->d_rpos) cudaFree(J->d_rpos);
    if (J->lib) cudaLibraryUnload(J->lib);
    if (J->t_lib) cudaLibraryUnload(J->t_lib);
    if (J->d_trace) cudaFree(J->d_trace);
    if (J->stream) cudaStreamDestroy(J->stream);
    delete J;
}

const char* pencil_jit_cuda_source(pencil_jit_t J) { return J ? J->src.c_str() : ""; }

// segments of `fn`: writes one char per segment ('S' serial, 'P' parallel, 'R' parallel with a
// reduction) into `out` (NUL-terminated); returns the number of segments or -1
int pencil_jit_schedule(pencil_jit_t J, const char* fn, char* out, int cap) {
    if (!J || !fn) return -1;
    auto it = J->entry_index.find(fn);
    if (it == J->entry_index.end()) return -1;
    const auto& segs = J->entries[it->second].segs;
    int n = 0;
    for (const auto& g : segs) {
        if (n + 1 < cap) out[n] = !g.parallel ? 'S' : (g.warp ? 'W' : g.inner ? '2' : (g.reds.empty() ? 'P' : 'R'));
        n++;
    }
    if (cap > 0) out[std::min(n, cap - 1)] = 0;
    return n;
}

// Interpreter::set_array (interp.hpp:40): values of dtype (pencil_dtype; int -> int64 values,
// float -> fp64 values, like the interpreter's Value)
int pencil_jit_set_array(pencil_jit_t J, const char* name, int dtype, const void* data, long long n) {
    if (!J || !name || n < 0 || (n && !data)) return fail(PENCIL_E_ARG, "E-ARG: bad set_array argument");
    int rc = setup(J);
    if (rc) return rc;
    std::vector<long long> bits((size_t)n);
    std::vector<unsigned char> tag((size_t)n);
    for (long long i = 0; i < n; i++) {
        switch (dtype) {
            case PENCIL_INT32: bits[i] = ((const int*)data)[i]; tag[i] = 0; break;
            case PENCIL_UINT8: bits[i] = ((const unsigned char*)data)[i]; tag[i] = 0; break;
            case PENCIL_FLOAT32: {
                double d = ((const float*)data)[i];
                memcpy(&bits[i], &d, 8);
                tag[i] = 1;
                break;
            }
            case PENCIL_FLOAT64: memcpy(&bits[i], (const double*)data + i, 8); tag[i] = 1; break;
            default: return fail(PENCIL_E_ARG, "E-ARG: unsupported dtype");
        }
    }
    StoreArr& a = J->store[name];
    if (a.n != n) {
        cudaFree(a.bits);
        cudaFree(a.tag);
        a.bits = nullptr;
        a.tag = nullptr;
        JCK(cudaMalloc(&a.bits, std::max<size_t>(8, (size_t)n * 8)));
        JCK(cudaMalloc(&a.tag, std::max<size_t>(8, (size_t)n)));
        a.n = n;
    }
    if (n) {
        JCK(cudaMemcpy(a.bits, bits.data(), (size_t)n * 8, cudaMemcpyHostToDevice));
        JCK(cudaMemcpy(a.tag, tag.data(), (size_t)n, cudaMemcpyHostToDevice));
    }
    return pencil_internal_ok();
}

long long pencil_jit_array_size(pencil_jit_t J, const char* name) {
    if (!J || !name) return -1;
    auto it = J->store.find(name);
    return it == J->store.end() ? -1 : it->second.n;
}

// Interpreter::arrays() (interp.hpp:39): element values as fp64 plus a per-element flag
// (1 = the element holds a double, 0 = an integer; integers up to 2^53 are exact in fp64 —
// `ints_out` (optional) receives the exact int64 of integer elements)
int pencil_jit_get_array(pencil_jit_t J, const char* name, double* out, unsigned char* is_double,
                         long long* ints_out, long long n) {
    if (!J || !name) return fail(PENCIL_E_ARG, "E-ARG: null argument");
    auto it = J->store.find(name);
    if (it == J->store.end()) return fail(PENCIL_E_ARG, std::string("E-ARG: no array named '") + name + "'");
    if (n != it->second.n) return fail(PENCIL_E_ARG, "E-ARG: array size mismatch");
    if (J->stream) JCK(cudaStreamSynchronize(J->stream));
    std::vector<long long> bits((size_t)n);
    std::vector<unsigned char> tag((size_t)n);
    if (n) {
        JCK(cudaMemcpy(bits.data(), it->second.bits, (size_t)n * 8, cudaMemcpyDeviceToHost));
        JCK(cudaMemcpy(tag.data(), it->second.tag, (size_t)n, cudaMemcpyDeviceToHost));
    }
    for (long long i = 0; i < n; i++) {
        double d;
        if (tag[i]) memcpy(&d, &bits[i], 8);
        else d = (double)bits[i];
        if (out) out[i] = d;
        if (is_double) is_double[i] = tag[i];
        if (ints_out) ints_out[i] = tag[i] ? (long long)d : bits[i];
    }
    return pencil_internal_ok();
}

// Interpreter::call (interp.hpp:49): scalars by value, arrays by store name; returns the value
int pencil_jit_call(pencil_jit_t J, const char* fn, int nargs, const pencil_arg* args, pencil_value* ret) {
    if (!J || !fn || (nargs && !args)) return fail(PENCIL_E_ARG, "E-ARG: null argument");
    auto it = J->entry_index.find(fn);
    if (it == J->entry_index.end()) return fail(PENCIL_E_INTERP, std::string("E-INTERP: no function named '") + fn + "'");
    const bool traced = J->trace_on;
    const EntryFn& E = (traced ? J->t_entries : J->entries)[it->second];
    const pf::Func& f = *E.f;
    if ((size_t)nargs != f.params.size())
        return fail(PENCIL_E_INTERP, "E-INTERP: wrong argument count for '" + f.name + "'");
    int rc = traced ? setup_trace(J) : setup(J);
    if (rc) return rc;
    // frame: scalar parameters from the call, locals 0 (slot K: return value)
    const size_t K = E.scalars.size();
    std::vector<HostV> frame(K + 1, HostV{0, 0.0, 0});
    struct DevArr {
        long long* p;
        unsigned char* tag;
        long long n;
        int inc;
        int id;  // the store's name, for the trace (canonical name: arrays keep it through calls)
    };
    std::vector<DevArr> arrs;
    for (int i = 0; i < nargs; i++) {
        const pf::Param& p = f.params[i];
        if (p.kind == pf::Param::Scalar) {
            HostV v{0, 0.0, 0};
            if (args[i].kind == PENCIL_ARG_FLOAT) {
                v.d = args[i].f;
                v.isd = 1;
            } else if (args[i].kind == PENCIL_ARG_INT) {
                v.i = args[i].i;
            }  // an array passed for a scalar: 0 (interp.cpp:116)
            frame[E.slot.at(p.name)] = v;
        } else {
            if (args[i].kind != PENCIL_ARG_ARRAY || !args[i].array)
                return fail(PENCIL_E_INTERP, "E-INTERP: parameter '" + p.name + "' needs an array");
            auto s = J->store.find(args[i].array);
            if (s == J->store.end())
                return fail(PENCIL_E_INTERP, std::string("E-INTERP: no array storage for '") + args[i].array + "'");
            auto nid = J->name_id.find(s->first);
            if (nid == J->name_id.end()) {
                nid = J->name_id.emplace(s->first, (int)J->names.size()).first;
                J->names.push_back(s->first);
            }
            arrs.push_back({s->second.bits, s->second.tag, s->second.n, 0, nid->second});
        }
    }
    static_assert(sizeof(HostV) == 24, "V layout");
    // call buffers: one scratch block per unit, grown on demand (cudaMalloc / cudaFree per call
    // cost more than a small call's kernels)
    const long long max_threads = 148 * 4 * 256;
    size_t max_red = 1;
    for (const auto& g : E.segs) max_red = std::max(max_red, g.reds.size());
    const size_t n_frame = K + 1, n_la = (size_t)std::max<long long>(1, E.la_total), n_part = max_threads * max_red;
    const size_t need = (2 * n_frame + n_la + n_part) * sizeof(HostV) + 64;
    if (J->scratch_bytes < need) {
        if (J->scratch) cudaFree(J->scratch);
        J->scratch = nullptr;
        J->scratch_bytes = 0;
        if (cudaMalloc(&J->scratch, need) != cudaSuccess) return fail(PENCIL_E_NOMEM, "E-NOMEM: JIT call buffers");
        J->scratch_bytes = need;
    }
    HostV* d_frame = (HostV*)J->scratch;
    HostV* d_out = d_frame + n_frame;
    HostV* d_la = d_out + n_frame;
    HostV* d_part = d_la + n_la;
    long long* d_bounds = (long long*)(d_part + n_part);
    int* d_flags = (int*)(d_bounds + 4);
    auto release = [&]() { cudaStreamSynchronize(J->stream); };
    JCK(cudaMemcpyAsync(d_frame, frame.data(), (K + 1) * sizeof(HostV), cudaMemcpyHostToDevice, J->stream));
    JCK(cudaMemsetAsync(d_la, 0, std::max<long long>(1, E.la_total) * sizeof(HostV), J->stream));
    JCK(cudaMemsetAsync(d_flags, 0, 16, J->stream));
    struct {
        unsigned* fault;
        unsigned long long* rng;
        const long long* rseq;
        unsigned long long* rpos;
        long long rseq_n;
        unsigned long long* tr;
    } cx{J->d_fault, J->d_rng, J->d_rseq, J->d_rpos, J->rseq_n, traced ? J->d_trace : nullptr};
    if (traced) {
        const unsigned long long head[2] = {0ull, (unsigned long long)J->trace_cap};
        JCK(cudaMemcpyAsync(J->d_trace, head, 16, cudaMemcpyHostToDevice, J->stream));
    }
    const int fi = it->second;
    int returned = 0;
    for (size_t si = 0; si < E.segs.size() && !returned; si++) {
        const Seg& g = E.segs[si];
        const std::string base = "jit_" + std::to_string(fi) + "_" + std::to_string(si);
        std::vector<void*> common = {&cx, &d_frame, &d_la};
        for (auto& a : arrs) common.push_back(&a);
        cudaKernel_t kk;
        if (!g.parallel) {
            if ((rc = get_kernel(J, base, &kk, traced))) return release(), rc;
            std::vector<void*> a = common;
            a.push_back(&d_flags);
            JCK(cudaLaunchKernel((const void*)kk, dim3(1), dim3(1), a.data(), 0, J->stream));
            continue;
        }
        // parallel segment: bounds, body, finish — all stream-ordered (the bounds stay on the
        // device; the body's grid is fixed and grid-strides over whatever range they hold)
        if ((rc = get_kernel(J, base + "_b", &kk, traced))) return release(), rc;
        {
            std::vector<void*> a = common;
            a.push_back(&d_bounds);
            a.push_back(&d_flags);
            JCK(cudaLaunchKernel((const void*)kk, dim3(1), dim3(1), a.data(), 0, J->stream));
        }
        const long long blocks = max_threads / 256;
        long long nthr = blocks * 256;
        if ((rc = get_kernel(J, base + "_p", &kk, traced))) return release(), rc;
        {
            std::vector<void*> a = common;
            a.push_back(&d_bounds);
            a.push_back(&d_out);
            a.push_back(&d_part);
            JCK(cudaLaunchKernel((const void*)kk, dim3((unsigned)blocks), dim3(256), a.data(), 0, J->stream));
        }
        if ((rc = get_kernel(J, base + "_f", &kk, traced))) return release(), rc;
        {
            std::vector<void*> a = {&cx, &d_frame, &d_out, &d_part, &nthr, &d_bounds, &d_flags};
            JCK(cudaLaunchKernel((const void*)kk, dim3(1), dim3(1024), a.data(), 0, J->stream));
        }
    }
    int flags = 0;
    JCK(cudaMemcpyAsync(&flags, d_flags, 4, cudaMemcpyDeviceToHost, J->stream));
    JCK(cudaStreamSynchronize(J->stream));
    returned = flags;
    HostV rv{0, 0.0, 0};
    if (returned) JCK(cudaMemcpyAsync(&rv, d_frame + K, sizeof(HostV), cudaMemcpyDeviceToHost, J->stream));
    unsigned fw = 0;
    JCK(cudaMemcpyAsync(&fw, J->d_fault, 4, cudaMemcpyDeviceToHost, J->stream));
    JCK(cudaMemsetAsync(J->d_fault, 0, 4, J->stream));
    release();
    if (traced) {  // append this call's records (the interpreter keeps its trace across calls)
        unsigned long long cnt = 0;
        JCK(cudaMemcpy(&cnt, J->d_trace, 8, cudaMemcpyDeviceToHost));
        const unsigned long long keep = std::min<unsigned long long>(cnt, (unsigned long long)J->trace_cap);
        std::vector<unsigned long long> rec(2 * keep);
        if (keep) JCK(cudaMemcpy(rec.data(), J->d_trace + 2, 16 * keep, cudaMemcpyDeviceToHost));
        for (unsigned long long r = 0; r < keep; r++)
            J->trace.push_back({(int)(rec[2 * r] >> 1), (long long)rec[2 * r + 1], (unsigned char)(rec[2 * r] & 1)});
        if (cnt > keep && !fw)
            return fail(PENCIL_E_UNSUPPORTED, "E-UNSUPPORTED: trace of one call longer than " +
                                                  std::to_string(J->trace_cap) + " records");
    }
    if (ret) {
        ret->kind = rv.isd ? PENCIL_ARG_FLOAT : PENCIL_ARG_INT;
        ret->i = rv.isd ? 0 : rv.i;
        ret->f = rv.isd ? rv.d : (double)rv.i;
    }
    if (fw) {
        std::string m = "E-INTERP: device fault:";
        if (fw & 1u) m += " load out of bounds;";
        if (fw & 2u) m += " store out of bounds;";
        if (fw & 4u) m += " division by zero;";
        if (fw & 8u) m += " modulo by zero;";
        if (fw & 16u) m += " non-integral value where an integer is required;";
        if (fw & 64u) m += " empty pointee;";
        if (fw & 128u) m += " execution step budget exceeded;";
        return fail(PENCIL_E_INTERP, m);
    }
    return pencil_internal_ok();
}


// per array parameter of fn: "name=r|w|rw|-" (+ "!" when must-written in full), comma separated
int pencil_jit_access(pencil_jit_t J, const char* fn, char* out, int cap) {
    if (!J || !fn) return -1;
    const pf::Func* f = J->unit.find(fn);
    if (!f) return -1;
    Summarizer S(J->unit);
    const auto& acc = S.of(*f);
    std::string r;
    for (size_t i = 0; i < f->params.size(); i++) {
        if (f->params[i].kind == pf::Param::Scalar) continue;
        const Access& a = acc[i];
        if (!r.empty()) r += ",";
        r += f->params[i].name + "=" + (a.load && a.store ? "rw" : a.load ? "r" : a.store ? "w" : "-");
        if (a.must_all) r += "!";
    }
    if (out && cap > 0) {
        size_t n = std::min<size_t>(r.size(), (size_t)cap - 1);
        r.copy(out, n);
        out[n] = 0;
    }
    return (int)r.size();
}

// Interpreter::call on HOST arrays with the data movement planned from the access summary:
// args[i] of kind PENCIL_ARG_ARRAY take host[i] (dtype dtypes[i], counts[i] elements); an array
// is uploaded when it is read or only partly written, downloaded (converted back to its dtype)
// when it is written; a must-written, never-read array is not uploaded.  The bytes moved are
// reported by pencil_jit_last_traffic.
int pencil_jit_call_host(pencil_jit_t J, const char* fn, int nargs, const pencil_arg* args, void* const* host,
                         const int* dtypes, const long long* counts, pencil_value* ret) {
    if (!J || !fn || (nargs && (!args || !host || !dtypes || !counts))) return fail(PENCIL_E_ARG, "E-ARG: null argument");
    const pf::Func* f = J->unit.find(fn);
    if (!f) return fail(PENCIL_E_INTERP, std::string("E-INTERP: no function named '") + fn + "'");
    if ((size_t)nargs != f->params.size())
        return fail(PENCIL_E_INTERP, "E-INTERP: wrong argument count for '" + f->name + "'");
    int rc = setup(J);
    if (rc) return rc;
    Summarizer S(J->unit);
    const auto acc = S.of(*f);
    static const int esize[] = {4, 4, 8, 1};
    std::vector<pencil_arg> a(args, args + nargs);
    std::vector<std::string> names((size_t)nargs);
    J->h2d = J->d2h = 0;
    for (int i = 0; i < nargs; i++) {
        if (f->params[i].kind == pf::Param::Scalar) continue;
        if (!host[i] && counts[i]) return fail(PENCIL_E_ARG, "E-ARG: null host array");
        if (dtypes[i] < 0 || dtypes[i] > 3) return fail(PENCIL_E_ARG, "E-ARG: unsupported dtype");
        names[i] = "__host_arg_" + std::to_string(i);
        const bool upload = acc[i].load || !acc[i].must_all;
        if (upload) {
            if ((rc = pencil_jit_set_array(J, names[i].c_str(), dtypes[i], host[i], counts[i]))) return rc;
            J->h2d += counts[i] * esize[dtypes[i]];
        } else {  // fully overwritten before any read: allocate only
            StoreArr& s = J->store[names[i]];
            if (s.n != counts[i]) {
                cudaFree(s.bits);
                cudaFree(s.tag);
                s.bits = nullptr;
                s.tag = nullptr;
                JCK(cudaMalloc(&s.bits, std::max<size_t>(8, (size_t)counts[i] * 8)));
                JCK(cudaMalloc(&s.tag, std::max<size_t>(8, (size_t)counts[i])));
                s.n = counts[i];
            }
        }
        a[i].kind = PENCIL_ARG_ARRAY;
        a[i].array = names[i].c_str();
    }
    rc = pencil_jit_call(J, fn, nargs, a.data(), ret);
    if (rc) return rc;
    for (int i = 0; i < nargs; i++) {
        if (f->params[i].kind == pf::Param::Scalar || !acc[i].store) continue;
        const long long n = counts[i];
        std::vector<double> v((size_t)n);
        std::vector<long long> iv((size_t)n);
        if ((rc = pencil_jit_get_array(J, names[i].c_str(), v.data(), nullptr, iv.data(), n))) return rc;
        for (long long k = 0; k < n; k++) {
            switch (dtypes[i]) {
                case PENCIL_INT32: ((int*)host[i])[k] = (int)iv[k]; break;
                case PENCIL_UINT8: ((unsigned char*)host[i])[k] = (unsigned char)iv[k]; break;
                case PENCIL_FLOAT32: ((float*)host[i])[k] = (float)v[k]; break;
                case PENCIL_FLOAT64: ((double*)host[i])[k] = v[k]; break;
            }
        }
        J->d2h += n * esize[dtypes[i]];
    }
    return pencil_internal_ok();
}

int pencil_jit_last_traffic(pencil_jit_t J, long long* h2d, long long* d2h) {
    if (!J) return fail(PENCIL_E_ARG, "E-ARG: null unit");
    if (h2d) *h2d = J->h2d;
    if (d2h) *d2h = J->d2h;
    return pencil_internal_ok();
}

// Interpreter::set_array with the interpreter's Value per element (interp.hpp:12: int64 or fp64):
// is_double[i] selects dbls[i], else ints[i]
int pencil_jit_set_array_values(pencil_jit_t J, const char* name, const long long* ints, const double* dbls,
                                const unsigned char* is_double, long long n) {
    if (!J || !name || n < 0 || (n && (!ints || !dbls || !is_double)))
        return fail(PENCIL_E_ARG, "E-ARG: bad set_array_values argument");
    int rc = pencil_jit_set_array(J, name, PENCIL_FLOAT64, dbls, n);  // allocates; tags below
    if (rc || !n) return rc;
    std::vector<long long> bits((size_t)n);
    std::vector<unsigned char> tag((size_t)n);
    for (long long i = 0; i < n; i++) {
        tag[i] = is_double[i] ? 1 : 0;
        if (tag[i]) memcpy(&bits[i], dbls + i, 8);
        else bits[i] = ints[i];
    }
    StoreArr& a = J->store[name];
    JCK(cudaMemcpy(a.bits, bits.data(), (size_t)n * 8, cudaMemcpyHostToDevice));
    JCK(cudaMemcpy(a.tag, tag.data(), (size_t)n, cudaMemcpyHostToDevice));
    return pencil_internal_ok();
}

// Interpreter::enable_trace / trace (interp.hpp:45-46, MemTrace :17-21)
int pencil_jit_enable_trace(pencil_jit_t J, int on) {
    if (!J) return fail(PENCIL_E_ARG, "E-ARG: null unit");
    J->trace_on = on != 0;
    return pencil_internal_ok();
}
long long pencil_jit_trace_size(pencil_jit_t J) { return J ? (long long)J->trace.size() : -1; }
int pencil_jit_trace_get(pencil_jit_t J, long long first, long long n, const char** arrays, long long* index,
                         unsigned char* is_write) {
    if (!J || first < 0 || n < 0 || first + n > (long long)J->trace.size())
        return fail(PENCIL_E_ARG, "E-ARG: trace range out of bounds");
    for (long long r = 0; r < n; r++) {
        const auto& t = J->trace[(size_t)(first + r)];
        if (arrays) arrays[r] = J->names[(size_t)t.id].c_str();
        if (index) index[r] = t.index;
        if (is_write) is_write[r] = t.write;
    }
    return pencil_internal_ok();
}
int pencil_jit_trace_clear(pencil_jit_t J) {
    if (!J) return fail(PENCIL_E_ARG, "E-ARG: null unit");
    J->trace.clear();
    return pencil_internal_ok();
}

// Interpreter::set_rand_sequence (interp.hpp:44): rand() pops these values first, then the LCG
int pencil_jit_set_rand_sequence(pencil_jit_t J, const long long* values, long long n) {
    if (!J || n < 0 || (n && !values)) return fail(PENCIL_E_ARG, "E-ARG: bad rand sequence");
    int rc = setup(J);
    if (rc) return rc;
    if (J->d_rseq) cudaFree(J->d_rseq);
    J->d_rseq = nullptr;
    if (!J->d_rpos) JCK(cudaMalloc(&J->d_rpos, 8));
    JCK(cudaMemset(J->d_rpos, 0, 8));
    if (n) {
        JCK(cudaMalloc(&J->d_rseq, (size_t)n * 8));
        JCK(cudaMemcpy(J->d_rseq, values, (size_t)n * 8, cudaMemcpyHostToDevice));
    }
    J->rseq_n = n;
    return pencil_internal_ok();
}

}  // extern "C"
