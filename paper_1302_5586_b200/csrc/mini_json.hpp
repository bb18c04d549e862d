// Minimal JSON reader for the OP2 mesh-model documents (docs/op2-input.md of the reference):
// objects, arrays, strings (with the standard escapes), integers, floats, true/false/null.
// Integers are kept exact as int64 (`is_int`), so map tables and dat contents round-trip.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

namespace mjson {

struct Value {
    enum Kind { Null, Bool, Int, Float, String, Array, Object } kind = Null;
    bool b = false;
    long long i = 0;
    double f = 0.0;
    std::string s;
    std::vector<Value> arr;
    std::vector<long long> ints;  // Array whose elements are all integers (kept compact; arr empty)
    std::vector<std::pair<std::string, Value>> obj;  // document order kept

    bool is_object() const { return kind == Object; }
    bool is_array() const { return kind == Array; }
    size_t size() const { return arr.empty() ? ints.size() : arr.size(); }
    bool is_string() const { return kind == String; }
    bool is_int() const { return kind == Int; }
    bool is_null() const { return kind == Null; }
    const Value* get(const std::string& key) const {
        for (const auto& kv : obj)
            if (kv.first == key) return &kv.second;
        return nullptr;
    }
};

// Returns false (and a message) on malformed input.
bool parse(const std::string& text, Value& out, std::string& err);

}  // namespace mjson
