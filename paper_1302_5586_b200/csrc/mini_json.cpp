#include "mini_json.hpp"

#include <cerrno>
#include <cstdlib>

namespace mjson {

namespace {

struct Reader {
    const std::string& t;
    size_t p = 0;
    std::string err;

    explicit Reader(const std::string& text) : t(text) {}

    void ws() {
        while (p < t.size() && (t[p] == ' ' || t[p] == '\n' || t[p] == '\r' || t[p] == '\t')) p++;
    }
    bool fail(const char* m) {
        if (err.empty()) err = std::string(m) + " at offset " + std::to_string(p);
        return false;
    }
    bool lit(const char* w) {
        size_t n = 0;
        while (w[n]) n++;
        if (t.compare(p, n, w) != 0) return fail("bad literal");
        p += n;
        return true;
    }
    static void put_utf8(std::string& o, unsigned cp) {
        if (cp < 0x80) {
            o += (char)cp;
        } else if (cp < 0x800) {
            o += (char)(0xC0 | (cp >> 6));
            o += (char)(0x80 | (cp & 0x3F));
        } else if (cp < 0x10000) {
            o += (char)(0xE0 | (cp >> 12));
            o += (char)(0x80 | ((cp >> 6) & 0x3F));
            o += (char)(0x80 | (cp & 0x3F));
        } else {
            o += (char)(0xF0 | (cp >> 18));
            o += (char)(0x80 | ((cp >> 12) & 0x3F));
            o += (char)(0x80 | ((cp >> 6) & 0x3F));
            o += (char)(0x80 | (cp & 0x3F));
        }
    }
    bool hex4(unsigned& v) {
        if (p + 4 > t.size()) return fail("short \\u escape");
        v = 0;
        for (int k = 0; k < 4; k++) {
            char c = t[p++];
            v <<= 4;
            if (c >= '0' && c <= '9') v |= (unsigned)(c - '0');
            else if (c >= 'a' && c <= 'f') v |= (unsigned)(c - 'a' + 10);
            else if (c >= 'A' && c <= 'F') v |= (unsigned)(c - 'A' + 10);
            else return fail("bad \\u escape");
        }
        return true;
    }
    bool str(std::string& o) {
        if (t[p] != '"') return fail("expected string");
        p++;
        while (p < t.size() && t[p] != '"') {
            char c = t[p++];
            if (c != '\\') {
                o += c;
                continue;
            }
            if (p >= t.size()) return fail("bad escape");
            char e = t[p++];
            switch (e) {
                case '"': o += '"'; break;
                case '\\': o += '\\'; break;
                case '/': o += '/'; break;
                case 'b': o += '\b'; break;
                case 'f': o += '\f'; break;
                case 'n': o += '\n'; break;
                case 'r': o += '\r'; break;
                case 't': o += '\t'; break;
                case 'u': {
                    unsigned cp;
                    if (!hex4(cp)) return false;
                    if (cp >= 0xD800 && cp < 0xDC00 && p + 6 <= t.size() && t[p] == '\\' && t[p + 1] == 'u') {
                        p += 2;
                        unsigned lo;
                        if (!hex4(lo)) return false;
                        cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                    }
                    put_utf8(o, cp);
                    break;
                }
                default: return fail("bad escape");
            }
        }
        if (p >= t.size()) return fail("unterminated string");
        p++;
        return true;
    }
    bool num(Value& v) {
        {  // fast path: a plain integer of <= 18 digits
            size_t q = p;
            bool neg = q < t.size() && t[q] == '-';
            if (neg) q++;
            size_t d0 = q;
            long long x = 0;
            while (q < t.size() && t[q] >= '0' && t[q] <= '9' && q - d0 < 18) x = x * 10 + (t[q++] - '0');
            if (q > d0 && (q >= t.size() || (t[q] != '.' && t[q] != 'e' && t[q] != 'E' && !(t[q] >= '0' && t[q] <= '9')))) {
                p = q;
                v.kind = Value::Int;
                v.i = neg ? -x : x;
                return true;
            }
        }
        size_t s = p;
        if (t[p] == '-') p++;
        while (p < t.size() && t[p] >= '0' && t[p] <= '9') p++;
        bool flt = false;
        if (p < t.size() && t[p] == '.') {
            flt = true;
            p++;
            while (p < t.size() && t[p] >= '0' && t[p] <= '9') p++;
        }
        if (p < t.size() && (t[p] == 'e' || t[p] == 'E')) {
            flt = true;
            p++;
            if (p < t.size() && (t[p] == '+' || t[p] == '-')) p++;
            while (p < t.size() && t[p] >= '0' && t[p] <= '9') p++;
        }
        std::string tok = t.substr(s, p - s);
        if (tok.empty() || tok == "-") return fail("bad number");
        if (!flt) {
            errno = 0;
            char* end = nullptr;
            long long x = std::strtoll(tok.c_str(), &end, 10);
            if (errno == 0 && end && *end == 0) {
                v.kind = Value::Int;
                v.i = x;
                return true;
            }
        }
        v.kind = Value::Float;
        v.f = std::strtod(tok.c_str(), nullptr);
        return true;
    }
    bool val(Value& v, int depth) {
        if (depth > 200) return fail("nesting too deep");
        ws();
        if (p >= t.size()) return fail("unexpected end");
        char c = t[p];
        if (c == '{') {
            v.kind = Value::Object;
            p++;
            ws();
            if (p < t.size() && t[p] == '}') {
                p++;
                return true;
            }
            for (;;) {
                ws();
                std::string k;
                if (p >= t.size() || !str(k)) return fail("expected key");
                ws();
                if (p >= t.size() || t[p] != ':') return fail("expected ':'");
                p++;
                Value e;
                if (!val(e, depth + 1)) return false;
                v.obj.emplace_back(std::move(k), std::move(e));
                ws();
                if (p < t.size() && t[p] == ',') {
                    p++;
                    continue;
                }
                if (p < t.size() && t[p] == '}') {
                    p++;
                    return true;
                }
                return fail("expected ',' or '}'");
            }
        }
        if (c == '[') {
            v.kind = Value::Array;
            p++;
            ws();
            if (p < t.size() && t[p] == ']') {
                p++;
                return true;
            }
            bool all_int = true;
            for (;;) {
                ws();
                if (all_int && p < t.size() && (t[p] == '-' || (t[p] >= '0' && t[p] <= '9'))) {
                    Value e;
                    if (!num(e)) return false;
                    if (e.kind == Value::Int) {
                        v.ints.push_back(e.i);
                    } else {  // first non-integer: move the integers into generic values
                        all_int = false;
                        for (long long x : v.ints) {
                            Value iv;
                            iv.kind = Value::Int;
                            iv.i = x;
                            v.arr.push_back(std::move(iv));
                        }
                        v.ints.clear();
                        v.arr.push_back(std::move(e));
                    }
                } else {
                    if (all_int) {
                        all_int = false;
                        for (long long x : v.ints) {
                            Value iv;
                            iv.kind = Value::Int;
                            iv.i = x;
                            v.arr.push_back(std::move(iv));
                        }
                        v.ints.clear();
                    }
                    Value e;
                    if (!val(e, depth + 1)) return false;
                    v.arr.push_back(std::move(e));
                }
                ws();
                if (p < t.size() && t[p] == ',') {
                    p++;
                    continue;
                }
                if (p < t.size() && t[p] == ']') {
                    p++;
                    return true;
                }
                return fail("expected ',' or ']'");
            }
        }
        if (c == '"') {
            v.kind = Value::String;
            return str(v.s);
        }
        if (c == 't') {
            v.kind = Value::Bool;
            v.b = true;
            return lit("true");
        }
        if (c == 'f') {
            v.kind = Value::Bool;
            return lit("false");
        }
        if (c == 'n') {
            v.kind = Value::Null;
            return lit("null");
        }
        return num(v);
    }
};

}  // namespace

bool parse(const std::string& text, Value& out, std::string& err) {
    Reader r(text);
    out = Value();
    if (!r.val(out, 0)) {
        err = r.err;
        return false;
    }
    r.ws();
    if (r.p != text.size()) {
        err = "trailing characters at offset " + std::to_string(r.p);
        return false;
    }
    return true;
}

}  // namespace mjson
