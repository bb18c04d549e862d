// CUDA code generation for PENCIL units on the device path (OP2 par_loop kernels, the JIT of
// jit.cpp): every PENCIL function becomes a `__device__` function over tagged int64 / fp64 values
// (`V`) that reproduce the reference Interpreter's arithmetic (core/src/interp.cpp:7-83: int64
// unless a double is involved, C-truncating `/` and `%`, both operands of `&&` / `||` evaluated,
// faults for division by zero, out-of-bounds and non-integral indices).  Evaluation order is the
// reference binary's (right operand first, see Binary; an assignment's right-hand side before its subscript), made
// explicit with one temporary per node.  Scalars are frame-wide like the interpreter's
// (Frame::scalars, interp.cpp:86-92).  The array model (`Arr`, `ld`, `st`, `deref`) is supplied by
// the caller's prelude: int64 storage with atomic OP_INC for OP2, tagged storage for the JIT.
#pragma once

#include <map>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/pencil_b200.h"
#include "pencil_front.hpp"

namespace pcg {

struct GenError {
    int st;
    std::string msg;
};

extern const char* kPreludeCore;  // V, Ctx, arithmetic, local arrays, builtins
extern const char* kArrInt64;     // Arr over int64 storage; += / -= on `inc` arrays are atomic adds
extern const char* kArrTagged;    // Arr over tagged storage (int64 or fp64 per element)



struct Gen {
    // ret_mode 0: `return` ends the device function; 1: it ends an entry segment (jit.cpp);
    // 2: not allowed (body of a parallel loop)
    int ret_mode = 0;
    // Warp mode (jit.cpp): a whole warp runs one iteration of a parallel loop.  Array stores
    // outside the split loops are done by lane 0 only (all lanes hold the same values) and
    // followed by __syncwarp; the loops in `warp_loops` (reduction loops: op code, variable) are
    // split across the lanes and their reduction variables combined in a fixed order.
    bool lane0_stores = false;
    std::map<const pf::Stmt*, std::vector<std::pair<int, std::string>>> warp_loops;

    static void assigned_scalars(const pf::Stmt& s, std::set<std::string>& out) {
        switch (s.kind) {
            case pf::Stmt::Block:
                for (const auto& c : s.body) assigned_scalars(*c, out);
                break;
            case pf::Stmt::Decl:
                if (s.extents.empty()) out.insert(s.name);
                break;
            case pf::Stmt::Assign:
                if (s.lhs->kind == pf::Expr::Var) out.insert(s.lhs->name);
                break;
            case pf::Stmt::For:
                out.insert(s.name);
                assigned_scalars(*s.loop_body, out);
                break;
            case pf::Stmt::While:
            case pf::Stmt::Labeled: assigned_scalars(*s.loop_body, out); break;
            case pf::Stmt::If:
                assigned_scalars(*s.then_s, out);
                if (s.else_s) assigned_scalars(*s.else_s, out);
                break;
            default: break;
        }
    }
    const pf::Unit& u;
    std::ostringstream out;
    int tmp = 0;
    explicit Gen(const pf::Unit& unit) : u(unit) {}

    [[noreturn]] void unsup(const pf::Func& f, int line, const std::string& m) {
        throw GenError{PENCIL_E_UNSUPPORTED, "E-UNSUPPORTED: kernel function '" + f.name + "' line " +
                                            std::to_string(line) + ": " + m};
    }

    struct Scope {
        const pf::Func* f;
        std::set<std::string> scalars;             // params + locals (frame-wide, like the interpreter)
        std::map<std::string, int> arrays;         // array/pointer params
        std::map<std::string, long long> larrays;  // local arrays (constant extent)
        std::map<std::string, pf::Ty> ldecl;
    };

    static std::string sid(const std::string& n) { return "s_" + n; }
    static std::string aid(const std::string& n) { return "a_" + n; }
    static std::string lid(const std::string& n) { return "l_" + n; }

    void collect(const pf::Stmt& s, Scope& sc) {
        switch (s.kind) {
            case pf::Stmt::Block:
                for (const auto& c : s.body) collect(*c, sc);
                break;
            case pf::Stmt::Decl:
                if (!s.extents.empty()) {
                    long long total = 1;
                    for (const auto& e : s.extents) {
                        if (e->kind != pf::Expr::IntLit) unsup(*sc.f, s.line, "local array '" + s.name + "' needs constant extents");
                        total *= e->ival;
                    }
                    if (total < 0 || total > 4096) unsup(*sc.f, s.line, "local array '" + s.name + "' larger than 4096 elements");
                    auto it = sc.larrays.find(s.name);
                    sc.larrays[s.name] = std::max(total, it == sc.larrays.end() ? 0ll : it->second);
                } else {
                    sc.scalars.insert(s.name);
                }
                break;
            case pf::Stmt::For:
                sc.scalars.insert(s.name);
                collect(*s.loop_body, sc);
                break;
            case pf::Stmt::While: collect(*s.loop_body, sc); break;
            case pf::Stmt::If:
                collect(*s.then_s, sc);
                if (s.else_s) collect(*s.else_s, sc);
                break;
            case pf::Stmt::Labeled: collect(*s.loop_body, sc); break;
            default: break;
        }
    }

    std::string t() { return "t" + std::to_string(tmp++); }

    // runaway loops: the interpreter stops at its step budget with E-INTERP (interp.cpp:141-144);
    // here every loop iteration counts against a per-thread budget of the same size
    std::string budget_check() const {
        return std::string("if (++steps_ > STEP_BUDGET) { fault(cx, F_BUDGET); ") +
               (ret_mode ? "return; }" : "return VI(0); }");
    }

    // emits statements computing `e`; returns an expression naming the value (a temp or literal)
    std::string ex(const pf::Expr& e, Scope& sc, std::ostringstream& o, const std::string& ind) {
        char buf[64];
        switch (e.kind) {
            case pf::Expr::IntLit:
                snprintf(buf, sizeof buf, "VI(%lldLL)", e.ival);
                return buf;
            case pf::Expr::FloatLit:
                snprintf(buf, sizeof buf, "VD(%a)", e.fval);
                return buf;
            case pf::Expr::Var:
                if (!sc.scalars.count(e.name)) unsup(*sc.f, e.line, "unbound scalar '" + e.name + "'");
                return sid(e.name);
            case pf::Expr::Index: {
                if (e.args.size() != 1) unsup(*sc.f, e.line, "multi-dimensional access unsupported here");
                std::string ix = ex(*e.args[0], sc, o, ind);
                std::string r = t();
                if (sc.larrays.count(e.name))
                    o << ind << "V " << r << " = ldl(cx, " << lid(e.name) << ", " << ix << ");\n";
                else if (sc.arrays.count(e.name))
                    o << ind << "V " << r << " = ld(cx, " << aid(e.name) << ", " << ix << ");\n";
                else
                    unsup(*sc.f, e.line, "no array storage for '" + e.name + "'");
                return r;
            }
            case pf::Expr::Binary: {
                // Both sides always evaluated, the RIGHT one first: the reference evaluates a binary
                // node as arith(op, eval(lhs), eval(rhs)) (interp.cpp:282), whose argument order C++
                // leaves unspecified; g++ evaluates it right to left, so that is the reference's order
                // (observable through rand() draws and the MemTrace of interp.hpp:17-21; checked by
                // tests/test_jit_interp.py against oracle/_ref/ref_driver).
                std::string b0 = ex(*e.args[1], sc, o, ind);
                std::string b = t();
                o << ind << "V " << b << " = " << b0 << ";\n";
                std::string a2 = ex(*e.args[0], sc, o, ind);
                std::string r = t();
                static const char* fn[] = {"op_add", "op_sub", "op_mul", "op_div", "op_mod", "op_lt", "op_le",
                                           "op_gt",  "op_ge",  "op_eq",  "op_ne",  "op_and", "op_or"};
                int k = (int)e.bop;
                bool ctx = e.bop == pf::Bin::Div || e.bop == pf::Bin::Mod;
                o << ind << "V " << r << " = " << fn[k] << "(" << (ctx ? "cx, " : "") << a2 << ", " << b << ");\n";
                return r;
            }
            case pf::Expr::Unary: {
                if (e.uop == pf::Un::Addr) unsup(*sc.f, e.line, "address-of is not executable");
                if (e.uop == pf::Un::Deref) {
                    if (e.args[0]->kind != pf::Expr::Var || !sc.arrays.count(e.args[0]->name))
                        unsup(*sc.f, e.line, "unsupported dereference");
                    std::string r = t();
                    o << ind << "V " << r << " = deref(cx, " << aid(e.args[0]->name) << ");\n";
                    return r;
                }
                std::string a = ex(*e.args[0], sc, o, ind);
                std::string r = t();
                o << ind << "V " << r << " = " << (e.uop == pf::Un::Neg ? "op_neg(" : "op_not(") << a << ");\n";
                return r;
            }
            case pf::Expr::Call: {
                std::string r = t();
                if (e.name == "exp") {
                    if (e.args.size() != 1) unsup(*sc.f, e.line, "exp takes one argument");
                    std::string a = ex(*e.args[0], sc, o, ind);
                    o << ind << "V " << r << " = b_exp(" << a << ");\n";
                    return r;
                }
                if (e.name == "rand") {
                    o << ind << "V " << r << " = b_rand(cx);\n";
                    return r;
                }
                const pf::Func* callee = u.find(e.name);
                if (!callee) unsup(*sc.f, e.line, "call to unknown '" + e.name + "'");
                if (callee->params.size() != e.args.size())
                    unsup(*sc.f, e.line, "wrong argument count for '" + e.name + "'");
                std::vector<std::string> av;
                for (size_t k = 0; k < e.args.size(); k++) {
                    if (callee->params[k].kind != pf::Param::Scalar) {
                        if (e.args[k]->kind != pf::Expr::Var) unsup(*sc.f, e.line, "array argument must be a name");
                        if (!sc.arrays.count(e.args[k]->name))
                            unsup(*sc.f, e.line, "array argument '" + e.args[k]->name + "' is not a parameter array");
                        av.push_back(aid(e.args[k]->name));
                    } else {
                        std::string a = ex(*e.args[k], sc, o, ind);
                        std::string a2 = t();
                        o << ind << "V " << a2 << " = " << a << ";\n";
                        av.push_back(a2);
                    }
                }
                o << ind << "V " << r << " = f_" << e.name << "(cx";
                for (auto& a : av) o << ", " << a;
                o << ");\n";
                return r;
            }
        }
        return "VI(0)";
    }

    void stmt(const pf::Stmt& s, Scope& sc, std::ostringstream& o, const std::string& ind) {
        switch (s.kind) {
            case pf::Stmt::Block:
                for (const auto& c : s.body) stmt(*c, sc, o, ind);
                break;
            case pf::Stmt::Nop: break;
            case pf::Stmt::Decl:
                if (!s.extents.empty()) {
                    o << ind << "for (ll q = 0; q < " << lid(s.name) << ".n; ++q) " << lid(s.name) << ".p[q] = "
                      << (s.dty == pf::Ty::Int ? "VI(0)" : "VD(0.0)") << ";\n";
                } else if (s.rhs) {
                    std::string v = ex(*s.rhs, sc, o, ind);
                    o << ind << sid(s.name) << " = " << v << ";\n";
                } else {
                    o << ind << sid(s.name) << " = " << (s.dty == pf::Ty::Int ? "VI(0)" : "VD(0.0)") << ";\n";
                }
                break;
            case pf::Stmt::Assign: {
                const bool global_store = s.lhs->kind == pf::Expr::Unary ||
                                          (s.lhs->kind == pf::Expr::Index && sc.arrays.count(s.lhs->name));
                if (lane0_stores && global_store) {  // one lane stores, then the warp converges
                    o << ind << "if ((threadIdx.x & 31) == 0) {\n";
                    lane0_stores = false;
                    stmt(s, sc, o, ind + "  ");
                    lane0_stores = true;
                    o << ind << "}\n" << ind << "__syncwarp();\n";
                    break;
                }
                std::string rhs0 = ex(*s.rhs, sc, o, ind);
                std::string rhs = t();
                o << ind << "V " << rhs << " = " << rhs0 << ";\n";
                int op = (int)s.aop;
                const pf::Expr& lv = *s.lhs;
                if (lv.kind == pf::Expr::Var) {
                    if (!sc.scalars.count(lv.name)) unsup(*sc.f, s.line, "assignment to unbound '" + lv.name + "'");
                    o << ind << sid(lv.name) << " = apply(cx, " << op << ", " << sid(lv.name) << ", " << rhs << ");\n";
                } else if (lv.kind == pf::Expr::Unary && lv.uop == pf::Un::Deref && lv.args[0]->kind == pf::Expr::Var &&
                           sc.arrays.count(lv.args[0]->name)) {
                    o << ind << "if (" << aid(lv.args[0]->name) << ".n == 0) fault(cx, F_EMPTY); else st(cx, "
                      << aid(lv.args[0]->name) << ", VI(0), " << op << ", " << rhs << ");\n";
                } else if (lv.kind == pf::Expr::Index) {
                    if (lv.args.size() != 1) unsup(*sc.f, s.line, "multi-dimensional access unsupported here");
                    std::string ix = ex(*lv.args[0], sc, o, ind);
                    if (sc.larrays.count(lv.name))
                        o << ind << "stl(cx, " << lid(lv.name) << ", " << ix << ", " << op << ", " << rhs << ");\n";
                    else if (sc.arrays.count(lv.name))
                        o << ind << "st(cx, " << aid(lv.name) << ", " << ix << ", " << op << ", " << rhs << ");\n";
                    else
                        unsup(*sc.f, s.line, "no array storage for '" + lv.name + "'");
                } else {
                    unsup(*sc.f, s.line, "unsupported lvalue");
                }
                break;
            }
            case pf::Stmt::For: {
                auto wl = warp_loops.find(&s);
                if (wl != warp_loops.end()) {
                    warp_split_for(s, wl->second, sc, o, ind);
                    break;
                }
                o << ind << "{\n";
                std::string in2 = ind + "  ";
                std::string lo = ex(*s.lo, sc, o, in2);
                std::string lo2 = t();
                o << in2 << "ll " << lo2 << " = as_i(cx, " << lo << ");\n";
                std::string hi = ex(*s.hi, sc, o, in2);
                std::string hi2 = t();
                o << in2 << "ll " << hi2 << " = as_i(cx, " << hi << ");\n";
                std::string q = t();
                o << in2 << "for (ll " << q << " = " << lo2 << "; " << q << " < " << hi2 << "; ++" << q << ") {\n";
                o << in2 << "  " << budget_check() << "\n";
                o << in2 << "  " << sid(s.name) << " = VI(" << q << ");\n";
                stmt(*s.loop_body, sc, o, in2 + "  ");
                o << in2 << "}\n" << ind << "}\n";
                break;
            }
            case pf::Stmt::While: {
                o << ind << "for (;;) {\n";
                std::string c = ex(*s.cond, sc, o, ind + "  ");
                o << ind << "  if (!truth(" << c << ")) break;\n";
                o << ind << "  " << budget_check() << "\n";
                stmt(*s.loop_body, sc, o, ind + "  ");
                o << ind << "}\n";
                break;
            }
            case pf::Stmt::If: {
                o << ind << "{\n";
                std::string c = ex(*s.cond, sc, o, ind + "  ");
                o << ind << "  if (truth(" << c << ")) {\n";
                stmt(*s.then_s, sc, o, ind + "    ");
                o << ind << "  }";
                if (s.else_s) {
                    o << " else {\n";
                    stmt(*s.else_s, sc, o, ind + "    ");
                    o << ind << "  }";
                }
                o << "\n" << ind << "}\n";
                break;
            }
            case pf::Stmt::CallS: {
                std::string r = ex(*s.call, sc, o, ind);
                o << ind << "(void)" << r << ";\n";
                break;
            }
            case pf::Stmt::Return:
                if (ret_mode == 2) unsup(*sc.f, s.line, "return inside a parallel loop");
                if (s.rhs) {
                    std::string r = ex(*s.rhs, sc, o, ind);
                    // entry segments run their statements inside a lambda (jit.cpp)
                    if (ret_mode) o << ind << "{ ret_v = " << r << "; ret_f = 1; return; }\n";
                    else o << ind << "return " << r << ";\n";
                } else {
                    if (ret_mode) o << ind << "{ ret_f = 1; return; }\n";
                    else o << ind << "return VI(0);\n";
                }
                break;
            case pf::Stmt::Labeled: stmt(*s.loop_body, sc, o, ind); break;
        }
    }

    // `for (j = lo; j < hi; j++)` with `reduction (op: r...)`, run by a whole warp: lane l takes
    // j = lo + l, lo + l + 32, ...; each r starts at the identity (+ 0, * 1, max / min: its value),
    // the lanes' partials are combined down a fixed tree into lane 0 and broadcast, then
    // r = r_before (op) total.  Other scalars the body assigns take the values of the lane that
    // ran the last iteration (the sequential result), the loop variable ends at hi - 1.
    void warp_split_for(const pf::Stmt& s, const std::vector<std::pair<int, std::string>>& reds, Scope& sc,
                        std::ostringstream& o, const std::string& ind) {
        o << ind << "{\n";
        std::string in2 = ind + "  ";
        std::string lo = ex(*s.lo, sc, o, in2);
        std::string lo2 = t();
        o << in2 << "ll " << lo2 << " = as_i(cx, " << lo << ");\n";
        std::string hi = ex(*s.hi, sc, o, in2);
        std::string hi2 = t();
        o << in2 << "ll " << hi2 << " = as_i(cx, " << hi << ");\n";
        std::vector<std::string> before;
        for (const auto& r : reds) {
            if (!sc.scalars.count(r.second)) unsup(*sc.f, s.line, "reduction variable '" + r.second + "' is not a scalar");
            std::string b = t();
            before.push_back(b);
            o << in2 << "V " << b << " = " << sid(r.second) << ";\n";
            if (r.first == 0) o << in2 << sid(r.second) << " = VI(0);\n";
            if (r.first == 1) o << in2 << sid(r.second) << " = VI(1);\n";
        }
        const bool saved = lane0_stores;
        lane0_stores = false;
        std::string q = t();
        o << in2 << "for (ll " << q << " = " << lo2 << " + (threadIdx.x & 31); " << q << " < " << hi2 << "; " << q
          << " += 32) {\n";
        o << in2 << "  " << budget_check() << "\n";
        o << in2 << "  " << sid(s.name) << " = VI(" << q << ");\n";
        stmt(*s.loop_body, sc, o, in2 + "  ");
        o << in2 << "}\n";
        lane0_stores = saved;
        for (size_t k = 0; k < reds.size(); k++) {
            const std::string v = sid(reds[k].second);
            o << in2 << "for (int d = 16; d > 0; d >>= 1) {\n";
            o << in2 << "  V u; u.i = __shfl_down_sync(0xffffffffu, " << v << ".i, d); u.d = __shfl_down_sync(0xffffffffu, "
              << v << ".d, d); u.isd = __shfl_down_sync(0xffffffffu, " << v << ".isd, d);\n";
            o << in2 << "  if ((threadIdx.x & 31) + d < 32) " << v << " = red(" << reds[k].first << ", " << v << ", u);\n";
            o << in2 << "}\n";
            o << in2 << v << ".i = __shfl_sync(0xffffffffu, " << v << ".i, 0); " << v << ".d = __shfl_sync(0xffffffffu, " << v
              << ".d, 0); " << v << ".isd = __shfl_sync(0xffffffffu, " << v << ".isd, 0);\n";
            o << in2 << v << " = red(" << reds[k].first << ", " << before[k] << ", " << v << ");\n";
        }
        std::set<std::string> asg;
        assigned_scalars(*s.loop_body, asg);
        asg.insert(s.name);
        for (const auto& r : reds) asg.erase(r.second);
        o << in2 << "if (" << hi2 << " > " << lo2 << ") {\n";
        o << in2 << "  const int src = (int)((" << hi2 << " - 1 - " << lo2 << ") & 31);\n";
        for (const auto& a : asg) {
            if (!sc.scalars.count(a)) continue;
            const std::string v = sid(a);
            o << in2 << "  " << v << ".i = __shfl_sync(0xffffffffu, " << v << ".i, src); " << v << ".d = __shfl_sync(0xffffffffu, "
              << v << ".d, src); " << v << ".isd = __shfl_sync(0xffffffffu, " << v << ".isd, src);\n";
        }
        o << in2 << "}\n" << ind << "}\n";
    }

    std::string signature(const pf::Func& f) {
        std::ostringstream o;
        o << "static __device__ V f_" << f.name << "(const Ctx& cx";
        for (const auto& p : f.params) {
            if (p.kind == pf::Param::Scalar) o << ", V " << sid(p.name);
            else o << ", Arr " << aid(p.name);
        }
        o << ")";
        return o.str();
    }

    void function(const pf::Func& f) {
        Scope sc;
        sc.f = &f;
        for (size_t i = 0; i < f.params.size(); i++) {
            if (f.params[i].kind == pf::Param::Scalar) sc.scalars.insert(f.params[i].name);
            else sc.arrays[f.params[i].name] = (int)i;
        }
        if (f.body) collect(*f.body, sc);
        std::ostringstream body;
        body << "  ll steps_ = 0;\n";
        for (const auto& s : sc.scalars) {
            bool is_param = false;
            for (const auto& p : f.params)
                if (p.name == s && p.kind == pf::Param::Scalar) is_param = true;
            if (!is_param) body << "  V " << sid(s) << " = VI(0);\n";
        }
        for (const auto& la : sc.larrays)
            body << "  V " << lid(la.first) << "_st[" << (la.second > 0 ? la.second : 1) << "]; LArr " << lid(la.first)
                 << " = {" << lid(la.first) << "_st, " << la.second << "};\n";
        if (f.body) stmt(*f.body, sc, body, "  ");
        out << signature(f) << " {\n" << body.str() << "  return VI(0);\n}\n";
    }

    // prelude (core + the caller's array model), then every function of the unit
    void unit(const char* arr_model) {
        out << kPreludeCore << arr_model;
        for (const auto& f : u.fns) out << signature(f) << ";\n";
        for (const auto& f : u.fns) function(f);
    }
};


// NVRTC compile of `src` for sm_100a (exact fp64: --fmad=false); cached per source text
int compile_cubin(const std::string& src, std::vector<char>& cubin, std::string& log);

}  // namespace pcg
