// Symbolic affine forms shared by the view extraction (descriptors.cpp) and the distribution
// plans (distplan.cpp): polynomials over scalar parameters with integer coefficients, and index
// expressions affine in loop variables with such polynomials as coefficients.
#pragma once
#include <algorithm>
#include <map>
#include <string>
#include <vector>

#include "pencil_front.hpp"

namespace affine_forms {
// A polynomial over scalar parameters with integer coefficients: monomial (sorted names) -> coef
using Mono = std::vector<std::string>;
using Poly = std::map<Mono, long long>;

inline Poly pconst(long long v) { return v ? Poly{{Mono{}, v}} : Poly{}; }
inline Poly padd(const Poly& a, const Poly& b, long long sb = 1) {
    Poly r = a;
    for (const auto& [m, c] : b) {
        r[m] += sb * c;
        if (r[m] == 0) r.erase(m);
    }
    return r;
}
inline Poly pmul(const Poly& a, const Poly& b) {
    Poly r;
    for (const auto& [ma, ca] : a)
        for (const auto& [mb, cb] : b) {
            Mono m = ma;
            m.insert(m.end(), mb.begin(), mb.end());
            std::sort(m.begin(), m.end());
            r[m] += ca * cb;
            if (r[m] == 0) r.erase(m);
        }
    return r;
}
inline bool peval(const Poly& p, const std::map<std::string, long long>& env, long long& out) {
    long long s = 0;
    for (const auto& [m, c] : p) {
        long long t = c;
        for (const auto& v : m) {
            auto it = env.find(v);
            if (it == env.end()) return false;
            t *= it->second;
        }
        s += t;
    }
    out = s;
    return true;
}
inline std::string pstr(const Poly& p) {
    if (p.empty()) return "0";
    std::string s;
    for (const auto& [m, c] : p) {
        std::string t;
        if (m.empty()) t = std::to_string(c < 0 ? -c : c);
        else {
            if (c != 1 && c != -1) t = std::to_string(c < 0 ? -c : c) + "*";
            for (size_t i = 0; i < m.size(); i++) t += (i ? "*" : "") + m[i];
        }
        if (s.empty()) s = (c < 0 ? "-" : "") + t;
        else s += (c < 0 ? " - " : " + ") + t;
    }
    return s;
}

struct Aff {
    bool ok = true;
    std::map<std::string, Poly> coef;  // loop variable -> d index / d var
    Poly c;                            // the rest (scalar parameters only)
};

inline Aff affine(const pf::Expr& e, const std::vector<std::string>& loops, const std::map<std::string, int>& params) {
    Aff r;
    auto is_loop = [&](const std::string& v) { return std::find(loops.begin(), loops.end(), v) != loops.end(); };
    switch (e.kind) {
        case pf::Expr::IntLit: r.c = pconst(e.ival); return r;
        case pf::Expr::Var:
            if (is_loop(e.name)) r.coef[e.name] = pconst(1);
            else if (params.count(e.name)) r.c = Poly{{Mono{e.name}, 1}};
            else r.ok = false;  // a local scalar (e.g. a clamped row index): not affine in the loops
            return r;
        case pf::Expr::Unary:
            if (e.uop == pf::Un::Neg) {
                Aff a = affine(*e.args[0], loops, params);
                r.ok = a.ok;
                for (auto& [v, p] : a.coef) r.coef[v] = padd(Poly{}, p, -1);
                r.c = padd(Poly{}, a.c, -1);
                return r;
            }
            r.ok = false;
            return r;
        case pf::Expr::Binary: {
            Aff a = affine(*e.args[0], loops, params), b = affine(*e.args[1], loops, params);
            if (!a.ok || !b.ok) {
                r.ok = false;
                return r;
            }
            if (e.bop == pf::Bin::Add || e.bop == pf::Bin::Sub) {
                const long long sb = e.bop == pf::Bin::Add ? 1 : -1;
                r.coef = a.coef;
                for (const auto& [v, p] : b.coef) {
                    r.coef[v] = padd(r.coef[v], p, sb);
                    if (r.coef[v].empty()) r.coef.erase(v);
                }
                r.c = padd(a.c, b.c, sb);
                return r;
            }
            if (e.bop == pf::Bin::Mul) {
                const Aff* lin = &a;
                const Aff* k = &b;
                if (!a.coef.empty() && !b.coef.empty()) {
                    r.ok = false;  // loop var * loop var
                    return r;
                }
                if (a.coef.empty()) std::swap(lin, k);
                for (const auto& [v, p] : lin->coef) {
                    Poly q = pmul(p, k->c);
                    if (!q.empty()) r.coef[v] = q;
                }
                r.c = pmul(lin->c, k->c);
                return r;
            }
            r.ok = false;  // / % and comparisons
            return r;
        }
        default: r.ok = false; return r;
    }
}

}  // namespace affine_forms
