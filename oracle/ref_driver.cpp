// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// A thin command-line driver over the *reference's own* public C++ API
// (/root/reference/proj/core/include/pencil/*.hpp), compiled by oracle/Makefile
// against the reference sources where they lie.  It is the checker the parity
// tests and golden-vector scripts use; nothing under paper_1302_5586_b200/ calls it.
//
// Sub-commands (all read a PENCIL unit from FILE):
//   check   FILE                          R1-R8 compliance   (compliance.hpp:41  check_compliance)
//   analyze FILE [--param n=v] [--array a=v0,v1,..]
//                                         loop verdicts      (depanalysis.hpp:79 analyze_unit)
//   lower   FILE                          OpenMP C           (lowering.hpp:29    emit_openmp)
//   run     FILE FN  < argspec            Interpreter::call  (interp.hpp:49); with PENCIL_REF_TRACE=path
//                                         the interpreter's MemTrace records go to path
//   signature FILE                        parameter kinds/types/extents (ast.hpp:133-151)
//   summarize FILE FN [--param n=v] [--array a=v0,v1,..]
//                                         access triple of a call FN(params...) under the
//                                         binding (summaries.hpp:42 summarize_call): one JSON
//                                         line per array parameter: read / must / may index sets
//
// `run` reads one argument per line from stdin, in parameter order:
//   scalar int <v> | scalar float <v> | array <f32|i32> <path>
// Array files are raw little-endian.  After the call every array argument is
// written back to <path>.out as float64 (f32 arrays) or int64 (i32 arrays) — the
// interpreter holds every value as int64/fp64 (interp.hpp:12) — and the return
// value is printed as `ret <int|float> <value>`.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "pencil/compliance.hpp"
#include "pencil/depanalysis.hpp"
#include "pencil/interp.hpp"
#include "pencil/lowering.hpp"
#include "pencil/parser.hpp"
#include "pencil/summaries.hpp"

using namespace pencil;

static std::string slurp(const char* path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) {
        std::fprintf(stderr, "cannot read %s\n", path);
        std::exit(2);
    }
    std::ostringstream b;
    b << in.rdbuf();
    return b.str();
}

// parse + attach + loop ids (the sequence tests/helpers.hpp:25-39 uses)
static Ast load_unit(const char* path) {
    ParseResult res = parse_source(slurp(path));
    bool bad = false;
    for (const auto& d : res.diagnostics)
        if (d.severity == Severity::Error) {
            std::fprintf(stderr, "%s: [%s] %s at %d:%d\n", path, d.code.c_str(), d.message.c_str(),
                         d.loc.line, d.loc.column);
            bad = true;
        }
    if (bad || !res.ast) std::exit(1);
    Ast ast = std::move(*res.ast);
    for (const auto& d : attach_directives(ast))
        if (d.severity == Severity::Error) {
            std::fprintf(stderr, "attach: [%s] %s\n", d.code.c_str(), d.message.c_str());
            std::exit(1);
        }
    assign_loop_ids(ast);
    return ast;
}

static void loop_owner(const Stmt& s, const std::string& fn, int depth,
                       std::vector<std::pair<std::string, int>>& out) {
    int d = depth;
    if (s.loop_id >= 0) {
        if ((int)out.size() <= s.loop_id) out.resize(s.loop_id + 1);
        out[s.loop_id] = {fn, depth};
        d = depth + 1;
    }
    for (const auto& c : s.stmts) loop_owner(*c, fn, d, out);
    if (s.body) loop_owner(*s.body, fn, d, out);
    if (s.then_branch) loop_owner(*s.then_branch, fn, d, out);
    if (s.else_branch) loop_owner(*s.else_branch, fn, d, out);
}

static void loop_ops(const Stmt& s, std::vector<std::string>& ops, std::vector<std::string>& vars) {
    if (s.loop_id >= 0) {
        if ((int)ops.size() <= s.loop_id) {
            ops.resize(s.loop_id + 1);
            vars.resize(s.loop_id + 1);
        }
        for (const auto& d : s.directives)
            if (d.kind == Directive::Kind::Reduction) {
                ops[s.loop_id] = d.reduction_op;
                std::string v;
                for (size_t i = 0; i < d.scalars.size(); ++i) v += (i ? "," : "") + d.scalars[i];
                vars[s.loop_id] = v;
            }
    }
    for (const auto& c : s.stmts) loop_ops(*c, ops, vars);
    if (s.body) loop_ops(*s.body, ops, vars);
    if (s.then_branch) loop_ops(*s.then_branch, ops, vars);
    if (s.else_branch) loop_ops(*s.else_branch, ops, vars);
}

static int cmd_check(const char* path) {
    Ast ast = load_unit(path);
    auto diags = check_compliance(ast);
    for (const auto& d : diags)
        std::printf("%s %s %d:%d %s\n", d.severity == Severity::Error ? "error" : "warning",
                    d.code.c_str(), d.loc.line, d.loc.column, d.message.c_str());
    std::printf("diagnostics %zu\n", diags.size());
    return has_errors(diags) ? 1 : 0;
}

static int cmd_analyze(const char* path, int argc, char** argv) {
    Ast ast = load_unit(path);
    ParamBinding bind;
    bool have = false;
    for (int i = 0; i + 1 < argc; i += 2) {
        std::string flag = argv[i], kv = argv[i + 1];
        auto eq = kv.find('=');
        if (eq == std::string::npos) return 2;
        std::string k = kv.substr(0, eq), v = kv.substr(eq + 1);
        if (flag == "--param") {
            bind.scalars[k] = std::stoll(v);
        } else if (flag == "--array") {
            std::vector<long long> vals;
            std::stringstream ss(v);
            std::string item;
            while (std::getline(ss, item, ',')) vals.push_back(std::stoll(item));
            bind.arrays[k] = vals;
        } else {
            return 2;
        }
        have = true;
    }
    auto resolved = resolve_access_bindings(ast);
    auto reports = analyze_unit(ast, resolved, have ? &bind : nullptr);
    std::vector<std::pair<std::string, int>> owner;
    std::vector<std::string> ops, vars;
    for (const auto& fn : ast.functions)
        if (fn.body) {
            loop_owner(*fn.body, fn.name, 0, owner);
            loop_ops(*fn.body, ops, vars);
        }
    for (const auto& r : reports) {
        std::string red;
        for (size_t i = 0; i < r.reduction_vars.size(); ++i)
            red += (i ? "," : "") + r.reduction_vars[i];
        const auto& o = owner.at(r.loop_id);
        std::string op = r.loop_id < (int)ops.size() ? ops[r.loop_id] : "";
        std::printf(
            "{\"loop\": %d, \"function\": \"%s\", \"depth\": %d, \"line\": %d, \"verdict\": \"%s\", "
            "\"basis\": \"%s\", \"reduction_vars\": \"%s\", \"reduction_op\": \"%s\", "
            "\"witnesses\": %zu}\n",
            r.loop_id, o.first.c_str(), o.second, r.loc.line, verdict_name(r.verdict).c_str(),
            basis_name(r.basis).c_str(), red.c_str(), red.empty() ? "" : op.c_str(),
            r.witnesses.size());
    }
    return 0;
}

// one line per function: ret;name:kind:type:extent;... (Param, ast.hpp:133-151)
static int cmd_signature(const char* path) {
    Ast ast = load_unit(path);
    for (const auto& fn : ast.functions) {
        std::string line = fn.name + "=" + type_name(fn.ret);
        for (const auto& p : fn.params) {
            std::string ext;
            for (size_t i = 0; i < p.extents.size(); ++i) ext += (i ? "][" : "") + pretty_print(*p.extents[i]);
            line += ";" + p.name + ":" + (p.kind == ParamKind::Array ? "array" : "scalar") + ":" +
                    type_name(p.elem) + ":" + ext;
            if (p.kind == ParamKind::Array && !(p.has_restrict && p.has_const && p.has_static))
                line += "(nonstatic)";
        }
        std::printf("%s\n", line.c_str());
    }
    return 0;
}

// summarize_call (summaries.cpp:635-648) of `fn` called with its own parameter names as the
// argument expressions, under a concrete binding: per array parameter, the distinct indices read,
// must-written and may-written, and whether any record had an index not evaluable (unknown).
static int cmd_summarize(const char* path, const char* fn, int argc, char** argv) {
    Ast ast = load_unit(path);
    ParamBinding bind;
    for (int i = 0; i + 1 < argc; i += 2) {
        std::string flag = argv[i], kv = argv[i + 1];
        auto eq = kv.find('=');
        if (eq == std::string::npos) return 2;
        std::string k = kv.substr(0, eq), v = kv.substr(eq + 1);
        if (flag == "--param") {
            bind.scalars[k] = std::stoll(v);
        } else if (flag == "--array") {
            std::vector<long long> vals;
            std::stringstream ss(v);
            std::string item;
            while (std::getline(ss, item, ',')) vals.push_back(std::stoll(item));
            bind.arrays[k] = vals;
        } else {
            return 2;
        }
    }
    const FunctionDef* def = nullptr;
    for (const auto& f : ast.functions)
        if (f.name == fn) def = &f;
    if (!def) return 2;
    std::vector<ExprPtr> args;
    for (const auto& p : def->params) args.push_back(make_var(p.name));
    auto resolved = resolve_access_bindings(ast);
    AccessResult res = summarize_call(ast, resolved, fn, args, bind);
    for (const auto& p : def->params) {
        if (p.kind != ParamKind::Array) continue;
        auto idx = [&](const std::vector<AccessRecord>& recs, bool& unknown) {
            std::vector<long long> out;
            for (const auto& r : recs) {
                if (r.array != p.name) continue;
                if (r.unknown_index) unknown = true;
                else if (!r.index.empty()) out.push_back(r.index[0]);
            }
            std::sort(out.begin(), out.end());
            out.erase(std::unique(out.begin(), out.end()), out.end());
            std::string js = "[";
            for (size_t i = 0; i < out.size(); ++i) js += (i ? "," : "") + std::to_string(out[i]);
            return js + "]";
        };
        bool unknown = false;
        std::string r = idx(res.triple.read, unknown), m = idx(res.triple.must_write, unknown),
                    y = idx(res.triple.may_write, unknown);
        std::printf("{\"array\": \"%s\", \"read\": %s, \"must\": %s, \"may\": %s, \"unknown\": %s}\n",
                    p.name.c_str(), r.c_str(), m.c_str(), y.c_str(), unknown ? "true" : "false");
    }
    return 0;
}

static int cmd_lower(const char* path) {
    Ast ast = load_unit(path);
    auto resolved = resolve_access_bindings(ast);
    auto reports = analyze_unit(ast, resolved, nullptr);
    std::fputs(emit_openmp(ast, reports).text.c_str(), stdout);
    return 0;
}

static int cmd_run(const char* path, const char* fn) {
    Ast ast = load_unit(path);
    Interpreter interp(ast);
    std::vector<Interpreter::Arg> args;
    struct Out {
        std::string name, path;
        bool is_float;
    };
    std::vector<Out> outs;
    std::string kind;
    int idx = 0;
    while (std::cin >> kind) {
        if (kind == "scalar") {
            std::string ty, v;
            std::cin >> ty >> v;
            if (ty == "int") args.push_back(Interpreter::Arg::scalar(std::stoll(v)));
            else args.push_back(Interpreter::Arg::scalar(std::stod(v)));
        } else if (kind == "array") {
            std::string ty, p;
            std::cin >> ty >> p;
            std::string data = slurp(p.c_str());
            std::vector<Value> vals(data.size() / 4);
            for (size_t i = 0; i < vals.size(); ++i) {
                if (ty == "f32") {
                    float f;
                    std::memcpy(&f, data.data() + 4 * i, 4);
                    vals[i] = (double)f;
                } else {
                    int v;
                    std::memcpy(&v, data.data() + 4 * i, 4);
                    vals[i] = (long long)v;
                }
            }
            std::string name = "arg" + std::to_string(idx);
            interp.set_array(name, std::move(vals));
            args.push_back(Interpreter::Arg::array(name));
            outs.push_back({name, p + ".out", ty == "f32"});
        } else {
            std::fprintf(stderr, "bad argspec token %s\n", kind.c_str());
            return 2;
        }
        ++idx;
    }
    Value ret;
    const char* trace_path = std::getenv("PENCIL_REF_TRACE");  // Interpreter::enable_trace (interp.hpp:45)
    if (trace_path) interp.enable_trace(true);
    try {
        ret = interp.call(fn, args);
    } catch (const PencilError& e) {
        std::printf("error %s %s\n", e.code().c_str(), e.what());
        return 3;
    }
    if (trace_path) {  // one line per recorded access: store name, flat index, 0 = load / 1 = store
        std::ofstream t(trace_path);
        for (const auto& r : interp.trace()) {
            t << r.array;
            for (long long i : r.index) t << " " << i;
            t << " " << (r.is_write ? 1 : 0) << "\n";
        }
    }
    for (const auto& o : outs) {
        const auto& vals = interp.arrays().at(o.name);
        std::ofstream f(o.path, std::ios::binary);
        for (const auto& v : vals) {
            if (o.is_float) {
                double d = as_double(v);
                f.write((const char*)&d, 8);
            } else {
                long long i = std::holds_alternative<long long>(v) ? std::get<long long>(v)
                                                                     : (long long)std::get<double>(v);
                f.write((const char*)&i, 8);
            }
        }
    }
    if (std::holds_alternative<long long>(ret)) std::printf("ret int %lld\n", std::get<long long>(ret));
    else std::printf("ret float %.17g\n", std::get<double>(ret));
    return 0;
}

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: ref_driver check|analyze|lower|run FILE [...]\n");
        return 2;
    }
    std::string cmd = argv[1];
    try {
        if (cmd == "check") return cmd_check(argv[2]);
        if (cmd == "analyze") return cmd_analyze(argv[2], argc - 3, argv + 3);
        if (cmd == "lower") return cmd_lower(argv[2]);
        if (cmd == "signature") return cmd_signature(argv[2]);
        if (cmd == "run" && argc >= 4) return cmd_run(argv[2], argv[3]);
        if (cmd == "summarize" && argc >= 4) return cmd_summarize(argv[2], argv[3], argc - 4, argv + 4);
    } catch (const PencilError& e) {
        std::fprintf(stderr, "%s\n", e.what());
        return 1;
    }
    return 2;
}
