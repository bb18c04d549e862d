#include "pencil_front.hpp"

#include <cstdlib>
#include <stdexcept>

namespace pf {

namespace {

struct Tok {
    enum Kind { Ident, Keyword, Int, Float, Punct, Pragma, End } kind = End;
    std::string text;
    long long ival = 0;
    double fval = 0.0;
    int line = 0;
};

struct ParseError : std::runtime_error {
    int line;
    ParseError(int l, const std::string& m) : std::runtime_error(m), line(l) {}
};

bool is_keyword(const std::string& w) {
    static const char* kw[] = {"void", "int", "float", "double", "for", "while", "if", "else", "return",
                               "goto", "const", "restrict", "static", "unsigned", "char", "long",
                               "short", "struct", "break", "continue", "do", "switch", "case", nullptr};
    for (int i = 0; kw[i]; i++)
        if (w == kw[i]) return true;
    return false;
}

std::vector<Tok> lex(const std::string& s) {
    std::vector<Tok> out;
    size_t p = 0;
    int line = 1;
    bool line_start = true;
    auto push = [&](Tok t) {
        t.line = line;
        out.push_back(std::move(t));
        line_start = false;
    };
    while (p < s.size()) {
        char c = s[p];
        if (c == '\n') {
            line++;
            p++;
            line_start = true;
            continue;
        }
        if (c == ' ' || c == '\t' || c == '\r') {
            p++;
            continue;
        }
        if (c == '/' && p + 1 < s.size() && s[p + 1] == '/') {
            while (p < s.size() && s[p] != '\n') p++;
            continue;
        }
        if (c == '/' && p + 1 < s.size() && s[p + 1] == '*') {
            p += 2;
            while (p + 1 < s.size() && !(s[p] == '*' && s[p + 1] == '/')) {
                if (s[p] == '\n') line++;
                p++;
            }
            if (p + 1 >= s.size()) throw ParseError(line, "unterminated comment");
            p += 2;
            continue;
        }
        if (c == '#' && line_start) {  // a preprocessor line (only `#pragma pencil ...` matters)
            size_t e = s.find('\n', p);
            if (e == std::string::npos) e = s.size();
            Tok t;
            t.kind = Tok::Pragma;
            t.text = s.substr(p, e - p);
            push(t);
            p = e;
            continue;
        }
        if (isalpha((unsigned char)c) || c == '_') {
            size_t b = p;
            while (p < s.size() && (isalnum((unsigned char)s[p]) || s[p] == '_')) p++;
            Tok t;
            t.text = s.substr(b, p - b);
            t.kind = is_keyword(t.text) ? Tok::Keyword : Tok::Ident;
            push(t);
            continue;
        }
        if (isdigit((unsigned char)c) || (c == '.' && p + 1 < s.size() && isdigit((unsigned char)s[p + 1]))) {
            size_t b = p;
            bool flt = false;
            while (p < s.size() && isdigit((unsigned char)s[p])) p++;
            if (p < s.size() && s[p] == '.') {
                flt = true;
                p++;
                while (p < s.size() && isdigit((unsigned char)s[p])) p++;
            }
            if (p < s.size() && (s[p] == 'e' || s[p] == 'E')) {
                flt = true;
                p++;
                if (p < s.size() && (s[p] == '+' || s[p] == '-')) p++;
                while (p < s.size() && isdigit((unsigned char)s[p])) p++;
            }
            std::string num = s.substr(b, p - b);
            if (p < s.size() && (s[p] == 'f' || s[p] == 'F')) {  // float suffix
                flt = true;
                p++;
            }
            Tok t;
            t.text = num;
            if (flt) {
                t.kind = Tok::Float;
                t.fval = std::strtod(num.c_str(), nullptr);
            } else {
                t.kind = Tok::Int;
                t.ival = std::strtoll(num.c_str(), nullptr, 10);
            }
            push(t);
            continue;
        }
        static const char* two[] = {"<=", ">=", "==", "!=", "&&", "||", "++", "--", "+=", "-=", "*=", "/=", nullptr};
        bool matched = false;
        for (int i = 0; two[i]; i++)
            if (s.compare(p, 2, two[i]) == 0) {
                Tok t;
                t.kind = Tok::Punct;
                t.text = two[i];
                push(t);
                p += 2;
                matched = true;
                break;
            }
        if (matched) continue;
        if (std::string("(){}[];,=<>+-*/%!&:?").find(c) != std::string::npos) {
            Tok t;
            t.kind = Tok::Punct;
            t.text = std::string(1, c);
            push(t);
            p++;
            continue;
        }
        throw ParseError(line, std::string("unexpected character '") + c + "'");
    }
    Tok e;
    e.kind = Tok::End;
    e.line = line;
    out.push_back(e);
    return out;
}

struct Parser {
    std::vector<Tok> t;
    size_t p = 0;

    const Tok& peek(int k = 0) const { return t[std::min(p + k, t.size() - 1)]; }
    const Tok& adv() { return t[p < t.size() - 1 ? p++ : p]; }
    bool at_p(const char* s) const { return peek().kind == Tok::Punct && peek().text == s; }
    bool at_k(const char* s) const { return peek().kind == Tok::Keyword && peek().text == s; }
    [[noreturn]] void fail(const std::string& m) { throw ParseError(peek().line, m); }
    void expect(const char* s) {
        if (!at_p(s)) fail(std::string("expected '") + s + "' before '" + peek().text + "'");
        adv();
    }
    std::string ident(const char* what) {
        if (peek().kind != Tok::Ident) fail(std::string("expected ") + what);
        return adv().text;
    }
    bool at_type() const { return at_k("void") || at_k("int") || at_k("float") || at_k("double"); }
    Ty type() {
        if (at_k("void")) { adv(); return Ty::Void; }
        if (at_k("int")) { adv(); return Ty::Int; }
        if (at_k("float")) { adv(); return Ty::Float; }
        if (at_k("double")) { adv(); return Ty::Double; }
        fail("expected a type name");
    }

    ExprP mk(Expr::Kind k, int line) {
        auto e = std::make_unique<Expr>();
        e->kind = k;
        e->line = line;
        return e;
    }
    ExprP bin(Bin op, ExprP a, ExprP b, int line) {
        auto e = mk(Expr::Binary, line);
        e->bop = op;
        e->args.push_back(std::move(a));
        e->args.push_back(std::move(b));
        return e;
    }

    // expressions: || < && < ==,!= < relational < additive < multiplicative < unary < postfix
    ExprP expr() { return lor(); }
    ExprP lor() {
        ExprP e = land();
        while (at_p("||")) { int l = adv().line; e = bin(Bin::Or, std::move(e), land(), l); }
        return e;
    }
    ExprP land() {
        ExprP e = eq();
        while (at_p("&&")) { int l = adv().line; e = bin(Bin::And, std::move(e), eq(), l); }
        return e;
    }
    ExprP eq() {
        ExprP e = rel();
        while (at_p("==") || at_p("!=")) {
            Bin op = peek().text == "==" ? Bin::Eq : Bin::Ne;
            int l = adv().line;
            e = bin(op, std::move(e), rel(), l);
        }
        return e;
    }
    ExprP rel() {
        ExprP e = add();
        while (at_p("<") || at_p("<=") || at_p(">") || at_p(">=")) {
            const std::string s = peek().text;
            Bin op = s == "<" ? Bin::Lt : s == "<=" ? Bin::Le : s == ">" ? Bin::Gt : Bin::Ge;
            int l = adv().line;
            e = bin(op, std::move(e), add(), l);
        }
        return e;
    }
    ExprP add() {
        ExprP e = mul();
        while (at_p("+") || at_p("-")) {
            Bin op = peek().text == "+" ? Bin::Add : Bin::Sub;
            int l = adv().line;
            e = bin(op, std::move(e), mul(), l);
        }
        return e;
    }
    ExprP mul() {
        ExprP e = unary();
        while (at_p("*") || at_p("/") || at_p("%")) {
            const std::string s = peek().text;
            Bin op = s == "*" ? Bin::Mul : s == "/" ? Bin::Div : Bin::Mod;
            int l = adv().line;
            e = bin(op, std::move(e), unary(), l);
        }
        return e;
    }
    ExprP unary() {
        int l = peek().line;
        Un op;
        if (at_p("-")) op = Un::Neg;
        else if (at_p("!")) op = Un::Not;
        else if (at_p("&")) op = Un::Addr;
        else if (at_p("*")) op = Un::Deref;
        else return postfix();
        adv();
        auto e = mk(Expr::Unary, l);
        e->uop = op;
        e->args.push_back(unary());
        return e;
    }
    ExprP postfix() {
        ExprP e = primary();
        while (at_p("[") || at_p("(")) {
            if (at_p("(")) {
                if (e->kind != Expr::Var) fail("only named functions can be called");
                int l = adv().line;
                auto c = mk(Expr::Call, l);
                c->name = e->name;
                if (!at_p(")")) {
                    c->args.push_back(expr());
                    while (at_p(",")) { adv(); c->args.push_back(expr()); }
                }
                expect(")");
                e = std::move(c);
            } else {
                if (e->kind != Expr::Var) fail("only named arrays can be indexed");
                auto ix = mk(Expr::Index, e->line);
                ix->name = e->name;
                while (at_p("[")) {
                    adv();
                    ix->args.push_back(expr());
                    expect("]");
                }
                e = std::move(ix);
            }
        }
        return e;
    }
    ExprP primary() {
        const Tok& k = peek();
        if (k.kind == Tok::Int) {
            auto e = mk(Expr::IntLit, k.line);
            e->ival = k.ival;
            adv();
            return e;
        }
        if (k.kind == Tok::Float) {
            auto e = mk(Expr::FloatLit, k.line);
            e->fval = k.fval;
            adv();
            return e;
        }
        if (k.kind == Tok::Ident) {
            auto e = mk(Expr::Var, k.line);
            e->name = k.text;
            adv();
            return e;
        }
        if (at_p("(")) {
            adv();
            ExprP e = expr();
            expect(")");
            return e;
        }
        fail("unexpected '" + k.text + "' in expression");
    }

    // statements
    StmtP mks(Stmt::Kind k, int line) {
        auto s = std::make_unique<Stmt>();
        s->kind = k;
        s->line = line;
        return s;
    }
    StmtP block() {
        auto b = mks(Stmt::Block, peek().line);
        expect("{");
        while (!at_p("}")) {
            if (peek().kind == Tok::End) fail("unexpected end of input in block");
            b->body.push_back(statement());
        }
        adv();
        return b;
    }
    StmtP statement() {
        std::vector<std::string> prag;  // kept for the mapper; they do not change the semantics
        while (peek().kind == Tok::Pragma) prag.push_back(adv().text);
        StmtP s = statement_inner();
        s->pragmas = std::move(prag);
        return s;
    }
    StmtP statement_inner() {
        if (at_p("}") || peek().kind == Tok::End) fail("expected a statement");
        int l = peek().line;
        if (at_p("{")) return block();
        if (at_p(";")) {
            adv();
            return mks(Stmt::Nop, l);
        }
        if (at_k("for")) return for_stmt();
        if (at_k("while")) {
            adv();
            auto s = mks(Stmt::While, l);
            expect("(");
            s->cond = expr();
            expect(")");
            s->loop_body = statement();
            return s;
        }
        if (at_k("if")) {
            adv();
            auto s = mks(Stmt::If, l);
            expect("(");
            s->cond = expr();
            expect(")");
            s->then_s = statement();
            if (at_k("else")) {
                adv();
                s->else_s = statement();
            }
            return s;
        }
        if (at_k("return")) {
            adv();
            auto s = mks(Stmt::Return, l);
            if (!at_p(";")) s->rhs = expr();
            expect(";");
            return s;
        }
        if (at_k("goto")) fail("goto is not executable");
        if (at_k("int") || at_k("float") || at_k("double")) {
            auto s = mks(Stmt::Decl, l);
            s->dty = type();
            if (at_p("*")) fail("local pointers are not supported");
            s->name = ident("variable name");
            while (at_p("[")) {
                adv();
                s->extents.push_back(expr());
                expect("]");
            }
            if (at_p("=")) {
                adv();
                s->rhs = expr();
            }
            expect(";");
            return s;
        }
        if (peek().kind == Tok::Keyword) fail("unexpected '" + peek().text + "'");
        if (peek().kind == Tok::Ident) {
            const std::string w = peek().text;
            if ((w == "DEF" || w == "USE" || w == "MAY_DEF") && peek(1).kind == Tok::Punct && peek(1).text == "(") {
                // summary statement: no runtime effect; kept for the data-movement planner
                adv();
                expect("(");
                auto s = mks(Stmt::Nop, l);
                s->summary = w == "DEF" ? 0 : w == "USE" ? 1 : 2;
                s->lhs = expr();
                expect(")");
                expect(";");
                return s;
            }
            if (peek(1).kind == Tok::Punct && peek(1).text == ":") {
                auto s = mks(Stmt::Labeled, l);
                s->name = adv().text;
                adv();
                s->loop_body = statement();
                return s;
            }
        }
        ExprP e = unary();
        if (at_p("=") || at_p("+=") || at_p("-=") || at_p("*=") || at_p("/=")) {
            const std::string op = adv().text;
            auto s = mks(Stmt::Assign, l);
            s->aop = op == "=" ? AOp::Set : op == "+=" ? AOp::Add : op == "-=" ? AOp::Sub : op == "*=" ? AOp::Mul : AOp::Div;
            s->lhs = std::move(e);
            s->rhs = expr();
            expect(";");
            return s;
        }
        if (at_p("++") || at_p("--")) {
            const bool inc = adv().text == "++";
            auto s = mks(Stmt::Assign, l);
            s->aop = inc ? AOp::Add : AOp::Sub;
            s->lhs = std::move(e);
            s->rhs = mk(Expr::IntLit, l);
            s->rhs->ival = 1;
            expect(";");
            return s;
        }
        if (e->kind == Expr::Call) {
            auto s = mks(Stmt::CallS, l);
            s->call = std::move(e);
            expect(";");
            return s;
        }
        fail("expected an assignment or a call");
    }
    StmtP for_stmt() {
        int l = adv().line;  // for
        auto s = mks(Stmt::For, l);
        expect("(");
        if (at_k("int")) adv();
        s->name = ident("loop variable");
        expect("=");
        s->lo = expr();
        expect(";");
        if (ident("loop variable") != s->name) fail("for-loop condition must test the loop variable");
        bool incl;
        if (at_p("<")) incl = false;
        else if (at_p("<=")) incl = true;
        else fail("for-loop condition must use '<' or '<='");
        adv();
        s->hi = expr();
        if (incl) {
            if (s->hi->kind == Expr::IntLit) {
                s->hi->ival += 1;
            } else {
                auto one = mk(Expr::IntLit, l);
                one->ival = 1;
                s->hi = bin(Bin::Add, std::move(s->hi), std::move(one), l);
            }
        }
        expect(";");
        // i++ | ++i | i += 1 | i = i + 1
        if (at_p("++")) {
            adv();
            if (ident("loop variable") != s->name) fail("for-loop step must advance the loop variable");
        } else {
            if (ident("loop variable") != s->name) fail("for-loop step must advance the loop variable");
            if (at_p("++")) {
                adv();
            } else if (at_p("+=")) {
                adv();
                if (!(peek().kind == Tok::Int && peek().ival == 1)) fail("for-loop step must be +1");
                adv();
            } else if (at_p("=")) {
                adv();
                ExprP e = expr();
                if (!(e->kind == Expr::Binary && e->bop == Bin::Add && e->args[0]->kind == Expr::Var &&
                      e->args[0]->name == s->name && e->args[1]->kind == Expr::IntLit && e->args[1]->ival == 1))
                    fail("for-loop step must be +1");
            } else {
                fail("for-loop step must be +1");
            }
        }
        expect(")");
        s->loop_body = statement();
        return s;
    }

    Param param() {
        Param q;
        q.ty = type();
        bool ptr = false;
        if (at_p("*")) {
            adv();
            ptr = true;
            while (at_k("const") || at_k("restrict")) adv();
        }
        q.name = ident("parameter name");
        if (at_p("[")) {
            if (ptr) fail("arrays of pointers are not supported");
            q.kind = Param::Array;
            bool first = true;
            while (at_p("[")) {
                adv();
                while (at_k("restrict") || at_k("const") || at_k("static")) adv();
                ExprP e = expr();
                if (first) q.extent = std::move(e);
                first = false;
                expect("]");
            }
        } else {
            q.kind = ptr ? Param::Pointer : Param::Scalar;
        }
        return q;
    }
    Func function() {
        while (peek().kind == Tok::Pragma) adv();
        Func f;
        f.ret = type();
        f.name = ident("function name");
        expect("(");
        if (at_k("void") && peek(1).kind == Tok::Punct && peek(1).text == ")") {
            adv();
        } else if (!at_p(")")) {
            f.params.push_back(param());
            while (at_p(",")) {
                adv();
                f.params.push_back(param());
            }
        }
        expect(")");
        if (peek().kind == Tok::Ident && peek().text == "ACCESS") {  // summary binding: no runtime effect
            adv();
            expect("(");
            f.access_fn = ident("summary function name");
            expect("(");
            if (!at_p(")")) {
                f.access_args.push_back(expr());
                while (at_p(",")) {
                    adv();
                    f.access_args.push_back(expr());
                }
            }
            expect(")");
            expect(")");
        }
        f.body = block();
        return f;
    }
};

}  // namespace

bool parse_unit(const std::string& src, Unit& out, std::string& err) {
    try {
        Parser P;
        P.t = lex(src);
        out.fns.clear();
        while (true) {
            while (P.peek().kind == Tok::Pragma) P.adv();
            if (P.peek().kind == Tok::End) break;
            out.fns.push_back(P.function());
        }
        return true;
    } catch (const ParseError& e) {
        err = "line " + std::to_string(e.line) + ": " + e.what();
        return false;
    }
}

}  // namespace pf
