// ORACLE / TEST INFRASTRUCTURE ONLY.
//
// The reference's own Interpreter known-answer cases (proj/tests/test_interp.cpp:8-108, doctest is
// absent here so each case is restated as a plain check) run through BOTH pencil::Interpreter
// (the reference, compiled from its sources) and pencil_b200::CudaInterpreter
// (include/pencil_cuda_interpreter.hpp over libpencil_b200.so): the same known answers, the same
// arrays, the same trace, the same PencilError codes.  Plus two fixture kernels (gemv, spmv_vec
// from paper_1302_5586_b200/pencil) whose results must equal the reference Interpreter's bit for
// bit.  Built by oracle/Makefile (`make check`) into _ref/cuda_interp_check; run by
// tests/test_cuda_interpreter_cpp.py on a GPU.  Prints `ok <case>` / `FAIL <case>: why`.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

#include "pencil/interp.hpp"
#include "pencil/parser.hpp"
#include "pencil_cuda_interpreter.hpp"

using namespace pencil;
using Arg = Interpreter::Arg;

static int failures = 0;
#define CHECK(cond, what)                                                      \
    do {                                                                       \
        if (!(cond)) throw std::runtime_error(std::string("check failed: ") + what); \
    } while (0)

static Ast parse_unit(const std::string& src) {  // tests/helpers.hpp:25-39
    ParseResult res = parse_source(src);
    for (const auto& d : res.diagnostics)
        if (d.severity == Severity::Error) throw std::runtime_error("parse: " + d.message);
    Ast ast = std::move(*res.ast);
    for (const auto& d : attach_directives(ast))
        if (d.severity == Severity::Error) throw std::runtime_error("attach: " + d.message);
    assign_loop_ids(ast);
    return ast;
}

static std::string slurp(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    std::ostringstream b;
    b << in.rdbuf();
    return b.str();
}

// run `body` with the reference Interpreter and with the CUDA one (same Ast)
template <class F>
static void both(const char* name, const Ast& ast, F body) {
    for (int side = 0; side < 2; ++side) {
        const char* who = side ? "cuda" : "reference";
        try {
            if (side == 0) {
                Interpreter it(ast);
                body(it);
            } else {
                pencil_b200::CudaInterpreter it(ast);
                body(it);
            }
            std::printf("ok   %s [%s]\n", name, who);
        } catch (const std::exception& e) {
            std::printf("FAIL %s [%s]: %s\n", name, who, e.what());
            ++failures;
        }
    }
}

template <class I>
static std::string fault_code(I& it, const std::string& fn, const std::vector<Arg>& args) {
    try {
        it.call(fn, args);
    } catch (const PencilError& e) {
        return e.code();
    }
    return "none";
}

int main(int argc, char** argv) {
    const std::string fixtures = argc > 1 ? argv[1] : "paper_1302_5586_b200/pencil";
    // test_interp.cpp:8-15
    {
        Ast ast = parse_unit("int f(int a, int b)\n{\n  int r;\n  r = a * b + a / b - a % b;\n  return r;\n}\n");
        both("arithmetic and return values", ast, [](auto& it) {
            Value v = it.call("f", {Arg::scalar(7LL), Arg::scalar(3LL)});
            CHECK(as_int(v) == 7 * 3 + 7 / 3 - 7 % 3, "7*3 + 7/3 - 7%3");
        });
    }
    // :17-27
    {
        Ast ast = parse_unit(
            "void set(int n, int A[restrict const static n])\n{\n  A[1] = 42;\n}\n"
            "void run(int n, int A[restrict const static n])\n{\n  set(n, A);\n  A[0] = A[1];\n}\n");
        both("arrays are shared through calls", ast, [](auto& it) {
            it.set_array("mem", {0LL, 0LL, 0LL});
            it.call("run", {Arg::scalar(3LL), Arg::array("mem")});
            CHECK(as_int(it.arrays()["mem"][0]) == 42, "mem[0]");
            CHECK(as_int(it.arrays()["mem"][1]) == 42, "mem[1]");
        });
    }
    // :29-37
    {
        Ast ast = parse_unit(
            "int tri(int n)\n{\n  int s;\n  int i;\n  s = 0;\n"
            "  for (i = 1; i <= n; i++) {\n    if (i % 2 == 0) {\n      s += i;\n    }\n  }\n"
            "  return s;\n}\n");
        both("loops and conditionals", ast,
             [](auto& it) { CHECK(as_int(it.call("tri", {Arg::scalar(6LL)})) == 2 + 4 + 6, "tri(6)"); });
    }
    // :39-46
    {
        Ast ast = parse_unit(
            "int halve(int n)\n{\n  int c;\n  c = 0;\n"
            "  while (n > 1) {\n    n = n / 2;\n    c += 1;\n  }\n  return c;\n}\n");
        both("while loop", ast, [](auto& it) { CHECK(as_int(it.call("halve", {Arg::scalar(16LL)})) == 4, "halve(16)"); });
    }
    // :48-62 (the CUDA side must also give the reference's LCG continuation)
    {
        Ast ast = parse_unit(
            "void take(int n, int A[restrict const static n])\n{\n  int i;\n"
            "  for (i = 0; i < n; i++) {\n    A[i] = rand();\n  }\n}\n");
        std::vector<Value> ref;
        both("rand pops the configured sequence, then falls back deterministically", ast, [&](auto& it) {
            it.set_array("A", std::vector<Value>(5, 0LL));
            it.set_rand_sequence({9, 8});
            it.call("take", {Arg::scalar(5LL), Arg::array("A")});
            CHECK(as_int(it.arrays()["A"][0]) == 9, "A[0]");
            CHECK(as_int(it.arrays()["A"][1]) == 8, "A[1]");
            if (ref.empty()) ref = it.arrays()["A"];
            else
                for (int i = 0; i < 5; ++i) CHECK(as_int(it.arrays()["A"][i]) == as_int(ref[i]), "LCG continuation");
        });
    }
    // :64-80
    {
        Ast ast = parse_unit(
            "void copy(int n, int A[restrict const static n], int B[restrict const static n])\n"
            "{\n  A[0] = B[1];\n}\n");
        both("trace records reads and writes in order", ast, [](auto& it) {
            it.set_array("A", {0LL, 0LL});
            it.set_array("B", {5LL, 6LL});
            it.enable_trace(true);
            it.call("copy", {Arg::scalar(2LL), Arg::array("A"), Arg::array("B")});
            CHECK(it.trace().size() == 2, "2 records");
            CHECK(it.trace()[0].array == "B", "first B");
            CHECK(it.trace()[0].index == std::vector<long long>{1}, "B[1]");
            CHECK(!it.trace()[0].is_write, "read");
            CHECK(it.trace()[1].array == "A", "then A");
            CHECK(it.trace()[1].is_write, "write");
        });
    }
    // :82-88
    {
        Ast ast = parse_unit("float scale(float x)\n{\n  return x * 0.5;\n}\n");
        both("floating point values", ast,
             [](auto& it) { CHECK(as_double(it.call("scale", {Arg::scalar(3.0)})) == 1.5, "scale(3.0)"); });
    }
    // :90-98
    {
        Ast ast = parse_unit("void f(int n, int A[restrict const static n])\n{\n  A[n] = 1;\n}\n");
        both("out-of-bounds store access faults", ast, [](auto& it) {
            it.set_array("A", {0LL, 0LL});
            CHECK(fault_code(it, "f", {Arg::scalar(2LL), Arg::array("A")}) == "E-INTERP", "E-INTERP");
        });
    }
    // :100-104
    {
        Ast ast = parse_unit("void f(int n)\n{\n}\n");
        both("unknown function faults", ast, [](auto& it) { CHECK(fault_code(it, "nope", {}) == "E-INTERP", "E-INTERP"); });
    }
    // :106-112
    {
        Ast ast = parse_unit("void spin(int n)\n{\n  while (n < 1) {\n    n = n - 1;\n  }\n}\n");
        both("step budget stops runaway loops", ast,
             [](auto& it) { CHECK(fault_code(it, "spin", {Arg::scalar(0LL)}) == "E-INTERP", "E-INTERP"); });
    }
    // fixture kernels: same store contents as the reference, bit for bit, and the same trace
    {
        Ast ast = parse_unit(slurp(fixtures + "/gemv.pencil.c"));
        const int m = 13, n = 29;
        std::vector<Value> A(m * n), x(n), y(m);
        for (int i = 0; i < m * n; ++i) A[i] = std::ldexp((double)((i * 7919) % 1000 - 500), -10);
        for (int j = 0; j < n; ++j) x[j] = std::ldexp((double)((j * 104729) % 1000 - 500), -10);
        for (int i = 0; i < m; ++i) y[i] = (long long)(i % 5);  // ints: beta * y mixes int and double
        std::vector<Value> ref;
        both("gemv fixture: same y as the reference, bit for bit", ast, [&](auto& it) {
            it.set_array("A", A);
            it.set_array("x", x);
            it.set_array("y", y);
            it.call("gemv", {Arg::scalar((long long)m), Arg::scalar((long long)n), Arg::scalar(1.25), Arg::scalar(0.5),
                             Arg::array("A"), Arg::array("x"), Arg::array("y")});
            const auto& got = it.arrays()["y"];
            if (ref.empty()) ref = got;
            else
                for (int i = 0; i < m; ++i) CHECK(as_double(got[i]) == as_double(ref[i]), "y[" + std::to_string(i) + "]");
        });
        std::vector<MemTrace> tref;
        both("gemv fixture: same trace as the reference", ast, [&](auto& it) {
            it.set_array("A", A);
            it.set_array("x", x);
            it.set_array("y", y);
            it.enable_trace(true);
            it.call("gemv", {Arg::scalar((long long)m), Arg::scalar((long long)n), Arg::scalar(1.25), Arg::scalar(0.5),
                             Arg::array("A"), Arg::array("x"), Arg::array("y")});
            if (tref.empty()) tref = it.trace();
            else {
                auto show = [](const MemTrace& t) {
                    return t.array + "[" + (t.index.empty() ? std::string("?") : std::to_string(t.index[0])) + "]" +
                           (t.is_write ? "w" : "r");
                };
                std::string head;
                for (size_t r = 0; r < 6 && r < tref.size() && r < it.trace().size(); ++r)
                    head += " ref " + show(tref[r]) + " / got " + show(it.trace()[r]) + ";";
                CHECK(it.trace().size() == tref.size(), "trace length " + std::to_string(it.trace().size()) + " vs " +
                                                           std::to_string(tref.size()) + head);
                for (size_t r = 0; r < tref.size(); ++r)
                    CHECK(it.trace()[r].array == tref[r].array && it.trace()[r].index == tref[r].index &&
                              it.trace()[r].is_write == tref[r].is_write,
                          "trace record " + std::to_string(r) + head);
            }
        });
    }
    {
        Ast ast = parse_unit(slurp(fixtures + "/spmv.pencil.c"));
        std::vector<Value> rowptr = {0LL, 2LL, 2LL, 5LL, 6LL}, col = {0LL, 3LL, 1LL, 2LL, 3LL, 0LL};
        std::vector<Value> val = {0.5, -1.25, 2.0, 0.125, 3.0, -0.75}, x = {1.0, 2.0, -3.0, 0.25}, y(4, 0LL);
        std::vector<Value> ref;
        for (const char* fn : {"spmv_inline", "spmv"})
            both((std::string(fn) + " fixture: same y as the reference").c_str(), ast, [&](auto& it) {
                it.set_array("rowptr", rowptr);
                it.set_array("col", col);
                it.set_array("val", val);
                it.set_array("x", x);
                it.set_array("y", y);
                it.call(fn, {Arg::scalar(4LL), Arg::scalar(4LL), Arg::scalar(6LL), Arg::array("rowptr"), Arg::array("col"),
                             Arg::array("val"), Arg::array("x"), Arg::array("y")});
                if (ref.empty()) ref = it.arrays()["y"];
                else
                    for (int i = 0; i < 4; ++i) CHECK(as_double(it.arrays()["y"][i]) == as_double(ref[i]), "y");
            });
    }
    std::printf("failures %d\n", failures);
    return failures ? 1 : 0;
}
