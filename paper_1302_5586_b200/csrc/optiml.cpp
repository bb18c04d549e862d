// OptiML control-structure constructs (reference core/include/pencil/optiml.hpp,
// docs/op2-input.md "Control-structure constructs"): the one-object JSON form is read and lowered
// to a compliant PENCIL unit — sum (a reduction loop seeded with f(lo)), vector (a plain
// initialisation loop), untilconverged (a sequential halving loop), gradient (batch: an
// `independent` per-coordinate update; stochastic: accumulation into one shared cell).  The unit
// then runs on the GPU through the general mapper (jit.cpp), whose schedule mirrors the analysis
// outcomes the reference documents (PARALLEL_WITH_REDUCTION / PARALLEL / UNKNOWN /
// ASSUMED_PARALLEL).  Errors: E-OPTIML-SHAPE (malformed document, unknown kind or variant),
// E-OPTIML-RANGE (empty sum range), as load_optiml_construct / lower_optiml (optiml.cpp:33-140).
#include <sstream>
#include <string>

#include "../../include/pencil_b200.h"
#include "mini_json.hpp"

int pencil_internal_fail(int status, const char* msg);  // runtime.cpp
int pencil_internal_ok();                                // runtime.cpp

namespace {

struct OErr {
    int st;
    std::string msg;
};
[[noreturn]] void shape(const std::string& m) { throw OErr{PENCIL_E_OPTIML_SHAPE, "E-OPTIML-SHAPE: " + m}; }

long long int_field(const mjson::Value& doc, const char* k, long long dflt) {
    const mjson::Value* v = doc.get(k);
    if (!v) return dflt;
    if (!v->is_int()) shape(std::string("'") + k + "' must be an integer");
    return v->i;
}
double num_field(const mjson::Value& doc, const char* k, double dflt) {
    const mjson::Value* v = doc.get(k);
    if (!v) return dflt;
    if (v->kind == mjson::Value::Int) return (double)v->i;
    if (v->kind == mjson::Value::Float) return v->f;
    shape(std::string("'") + k + "' must be a number");
}
std::string str_field(const mjson::Value& doc, const char* k, const char* dflt) {
    const mjson::Value* v = doc.get(k);
    if (!v) return dflt;
    if (!v->is_string()) shape(std::string("'") + k + "' must be a string");
    return v->s;
}
// a double literal that always reads back as a double in PENCIL (a trailing ".0" if needed)
std::string dlit(double v) {
    std::ostringstream os;
    os << v;
    std::string t = os.str();
    if (t.find_first_of(".eE") == std::string::npos) t += ".0";
    return t;
}
bool ident(const std::string& s) {
    if (s.empty() || !(isalpha((unsigned char)s[0]) || s[0] == '_')) return false;
    for (char c : s)
        if (!(isalnum((unsigned char)c) || c == '_')) return false;
    return true;
}

std::string lower(const std::string& text) {
    mjson::Value doc;
    std::string perr;
    if (!mjson::parse(text, doc, perr) || !doc.is_object()) shape("input is not a JSON object");
    const mjson::Value* kind = doc.get("kind");
    if (!kind || !kind->is_string()) shape("missing construct kind");
    const std::string k = kind->s;
    std::ostringstream u;
    if (k == "sum") {
        const long long lo = int_field(doc, "lo", 0), hi = int_field(doc, "hi", 0);
        const std::string f = str_field(doc, "body", "exp");
        if (!ident(f)) shape("summand '" + f + "' is not a function name");
        if (hi < lo)
            throw OErr{PENCIL_E_OPTIML_RANGE,
                       "E-OPTIML-RANGE: empty sum range " + std::to_string(lo) + ".." + std::to_string(hi)};
        // seed with f(lo), then the licensed reduction over lo+1 .. hi
        u << "void optiml_sum(void)\n{\n  double x;\n  int i;\n  x = " << f << "(" << lo << ");\n"
          << "  #pragma pencil reduction (+: x)\n  for (i = " << lo + 1 << "; i <= " << hi << "; i++)\n  {\n"
          << "    x += " << f << "(i);\n  }\n}\n";
    } else if (k == "vector") {
        const long long lo = int_field(doc, "lo", 0), hi = int_field(doc, "hi", 0), init = int_field(doc, "init", 0);
        u << "void optiml_vector(int n, int my_vector[restrict const static n])\n{\n  int i;\n"
          << "  for (i = 0; i <= " << hi - lo << "; i++)\n  {\n    my_vector[i] = " << init << ";\n  }\n}\n";
    } else if (k == "untilconverged") {
        const double th = num_field(doc, "threshold", 0.001);
        u << "void optiml_untilconverged(double delta)\n{\n  while (delta > " << dlit(th) << ")\n  {\n"
          << "    delta = delta / 2.0;\n  }\n}\n";
    } else if (k == "gradient") {
        const std::string v = str_field(doc, "variant", "batch");
        if (v == "batch") {
            u << "void optiml_gradient_batch(int n, double g[restrict const static n], double d[restrict const static n])\n"
              << "{\n  int i;\n  #pragma pencil independent\n  for (i = 0; i < n; i++)\n  {\n"
              << "    g[i] = g[i] + d[i];\n  }\n}\n";
        } else if (v == "stochastic") {
            u << "void optiml_gradient_stochastic(int n, double w[restrict const static n], double d[restrict const static n])\n"
              << "{\n  int i;\n  for (i = 0; i < n; i++)\n  {\n    w[0] = w[0] + d[i];\n  }\n}\n";
        } else {
            shape("unknown gradient variant '" + v + "'");
        }
    } else {
        shape("unknown construct kind '" + k + "'");
    }
    return u.str();
}

}  // namespace

extern "C" {

// the construct lowered to PENCIL text; returns the text length (writes at most cap-1 bytes +
// NUL; call with cap 0 to size the buffer) or -1 with the status set
long long pencil_optiml_lower(const char* json_text, char* out, long long cap) {
    if (!json_text) return pencil_internal_fail(PENCIL_E_ARG, "E-ARG: null document"), -1;
    std::string src;
    try {
        src = lower(json_text);
    } catch (const OErr& e) {
        pencil_internal_fail(e.st, e.msg.c_str());
        return -1;
    }
    if (out && cap > 0) {
        long long n = (long long)src.size() < cap - 1 ? (long long)src.size() : cap - 1;
        src.copy(out, (size_t)n);
        out[n] = 0;
    }
    pencil_internal_ok();
    return (long long)src.size();
}

}  // extern "C"
