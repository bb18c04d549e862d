// Front end for PENCIL kernel sources on the device path (OP2 par_loop kernels): a lexer and
// recursive-descent parser for the language subset the reference accepts (types void / int /
// float / double; C99 static-array parameters; decl, assign and compound assign, ++/--, for in
// the normalised `i = lo; i < | <= hi; i++` shape, while, if/else, return, calls, labels,
// #pragma pencil lines, DEF/USE/MAY_DEF summary statements).  Grammar as in the reference's
// parser (core/src/parser.cpp:104-662); this is an independent implementation producing its
// own tree, consumed by the CUDA code generator in op2.cpp.
#pragma once

#include <memory>
#include <string>
#include <vector>

namespace pf {

enum class Ty { Void, Int, Float, Double };
enum class Bin { Add, Sub, Mul, Div, Mod, Lt, Le, Gt, Ge, Eq, Ne, And, Or };
enum class Un { Neg, Not, Addr, Deref };

struct Expr;
using ExprP = std::unique_ptr<Expr>;
struct Expr {
    enum Kind { IntLit, FloatLit, Var, Index, Binary, Unary, Call } kind = IntLit;
    long long ival = 0;
    double fval = 0.0;
    std::string name;  // Var / Index base / Call callee
    Bin bop = Bin::Add;
    Un uop = Un::Neg;
    std::vector<ExprP> args;  // operands / subscripts / call arguments
    int line = 0;
};

struct Stmt;
using StmtP = std::unique_ptr<Stmt>;
enum class AOp { Set, Add, Sub, Mul, Div };
struct Stmt {
    enum Kind { Block, Decl, Assign, For, While, If, CallS, Return, Labeled, Nop } kind = Block;
    std::vector<StmtP> body;  // Block
    Ty dty = Ty::Int;         // Decl
    std::vector<ExprP> extents;  // Decl: local array extents
    std::string name;         // Decl / For variable / label
    ExprP lhs, rhs;           // Assign (rhs also: Decl init, Return value)
    AOp aop = AOp::Set;
    ExprP lo, hi;             // For (hi exclusive)
    ExprP cond;               // While / If
    StmtP then_s, else_s, loop_body;  // If / For, While, Labeled
    ExprP call;               // CallS
    std::vector<std::string> pragmas;  // `#pragma pencil ...` lines directly before the statement
    int summary = -1;         // Nop from DEF (0) / USE (1) / MAY_DEF (2): target in lhs
    int line = 0;
};

struct Param {
    enum Kind { Scalar, Array, Pointer } kind = Scalar;
    Ty ty = Ty::Int;
    std::string name;
    ExprP extent;  // Array: leading extent
};

struct Func {
    Ty ret = Ty::Void;
    std::string name;
    std::vector<Param> params;
    StmtP body;
    std::string access_fn;             // ACCESS(summary_fn(args...)) binding, if any
    std::vector<ExprP> access_args;
};

struct Unit {
    std::vector<Func> fns;
    const Func* find(const std::string& n) const {
        for (const auto& f : fns)
            if (f.name == n) return &f;
        return nullptr;
    }
};

// Parses a whole unit; on failure returns false with "line N: message".
bool parse_unit(const std::string& src, Unit& out, std::string& err);

}  // namespace pf
