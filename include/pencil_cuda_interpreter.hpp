// pencil_cuda_interpreter.hpp — the secondary (C++) drop-in boundary of the B200 backend
// (SURVEY.md §8b): pencil::Interpreter's public surface (reference
// core/include/pencil/interp.hpp:27-72) executed on the GPU.
//
//   pencil::Interpreter interp(ast);            ->  pencil_b200::CudaInterpreter interp(ast);
//   interp.set_array("A", {0LL, 1.5, ...});         same
//   Value v = interp.call("f", {Arg::scalar(3LL), Arg::array("A")});   same
//   interp.arrays()["A"][0]; interp.set_rand_sequence({9, 8});        same
//   interp.enable_trace(true); interp.trace();                         same (MemTrace records)
//   PencilError("E-INTERP", ...) on runtime faults                     same codes, rethrown
//
// Header-only: compile it where the reference headers are on the include path (it uses the
// reference's Ast, Value, Interpreter::Arg, MemTrace, PencilError and pretty_print) and link
// libpencil_b200.so.  The unit is printed back to source by the reference printer (pretty_print,
// lowering.hpp:15 — "output re-parses to a structurally identical Ast") and compiled for sm_100a
// by the library's general mapper (pencil_jit_*, include/pencil_b200.h §9), which keeps the
// interpreter's value semantics: int64 / fp64 tagged values, C-truncating / and %, E-INTERP
// faults.  Loops carrying `independent` / `reduction` pragmas run as parallel grids (reductions
// reassociate, as the pragma licenses); with the trace on, every statement runs on one device
// thread in the interpreter's order so the trace is the interpreter's.
//
// The interpreter's store is mirrored on the host: every named array is uploaded before a call and
// read back after it (what arrays() returns).  The C ABI underneath throws nothing; this header
// turns a failed status into the reference's PencilError with the same code.
#pragma once

#include <map>
#include <string>
#include <utility>
#include <variant>
#include <vector>

#include "pencil/diag.hpp"
#include "pencil/interp.hpp"
#include "pencil/lowering.hpp"
#include "pencil_b200.h"

namespace pencil_b200 {

class CudaInterpreter {
  public:
    using Arg = pencil::Interpreter::Arg;

    explicit CudaInterpreter(const pencil::Ast& ast, int device = 0) {
        rt_ = pencil_runtime_create(device);  // selects the device for this thread
        if (!rt_) throw pencil::PencilError("E-CUDA", "cannot open CUDA device " + std::to_string(device));
        unit_ = pencil_jit_load(pencil::pretty_print(ast).c_str());
        if (!unit_) {
            pencil_runtime_destroy(rt_);
            throw_last(pencil_cuda_last_status());
        }
    }
    ~CudaInterpreter() {
        pencil_jit_free(unit_);
        pencil_runtime_destroy(rt_);
    }
    CudaInterpreter(const CudaInterpreter&) = delete;
    CudaInterpreter& operator=(const CudaInterpreter&) = delete;

    // Interpreter::arrays / set_array (interp.hpp:39-43)
    std::map<std::string, std::vector<pencil::Value>>& arrays() { return arrays_; }
    void set_array(const std::string& name, std::vector<pencil::Value> data) { arrays_[name] = std::move(data); }

    // Interpreter::set_rand_sequence (interp.hpp:44)
    void set_rand_sequence(std::vector<long long> values) {
        check(pencil_jit_set_rand_sequence(unit_, values.data(), (long long)values.size()));
    }

    // Interpreter::enable_trace / trace (interp.hpp:45-46)
    void enable_trace(bool on) { check(pencil_jit_enable_trace(unit_, on ? 1 : 0)); }
    const std::vector<pencil::MemTrace>& trace() const { return trace_; }

    // Interpreter::call (interp.hpp:49): scalars by value, arrays by store name
    pencil::Value call(const std::string& fn, const std::vector<Arg>& args) {
        for (const auto& [name, vals] : arrays_) upload(name, vals);
        std::vector<pencil_arg> a(args.size());
        for (size_t i = 0; i < args.size(); ++i) {
            a[i] = pencil_arg{};
            if (args[i].is_array) {
                a[i].kind = PENCIL_ARG_ARRAY;
                a[i].array = args[i].array_name.c_str();
            } else if (std::holds_alternative<double>(args[i].value)) {
                a[i].kind = PENCIL_ARG_FLOAT;
                a[i].f = std::get<double>(args[i].value);
            } else {
                a[i].kind = PENCIL_ARG_INT;
                a[i].i = std::get<long long>(args[i].value);
            }
        }
        pencil_value ret{};
        const int st = pencil_jit_call(unit_, fn.c_str(), (int)a.size(), a.data(), &ret);
        const std::string msg = pencil_cuda_last_error();
        for (auto& [name, vals] : arrays_) download(name, vals);  // what the call stored, fault or not
        pull_trace();
        if (st) throw_code(st, msg);
        if (ret.kind == PENCIL_ARG_FLOAT) return ret.f;
        return ret.i;
    }

  private:
    void upload(const std::string& name, const std::vector<pencil::Value>& vals) {
        const size_t n = vals.size();
        std::vector<long long> ints(n);
        std::vector<double> dbls(n);
        std::vector<unsigned char> isd(n);
        for (size_t i = 0; i < n; ++i) {
            isd[i] = std::holds_alternative<double>(vals[i]);
            if (isd[i]) dbls[i] = std::get<double>(vals[i]);
            else ints[i] = std::get<long long>(vals[i]);
        }
        check(pencil_jit_set_array_values(unit_, name.c_str(), ints.data(), dbls.data(), isd.data(), (long long)n));
    }
    void download(const std::string& name, std::vector<pencil::Value>& vals) {
        const long long n = (long long)vals.size();
        std::vector<double> d(n);
        std::vector<unsigned char> isd(n);
        std::vector<long long> ints(n);
        if (pencil_jit_get_array(unit_, name.c_str(), d.data(), isd.data(), ints.data(), n)) return;
        for (long long i = 0; i < n; ++i)
            vals[i] = isd[i] ? pencil::Value{d[i]} : pencil::Value{ints[i]};
    }
    void pull_trace() {
        const long long n = pencil_jit_trace_size(unit_);
        const long long have = (long long)trace_.size();
        if (n <= have) return;
        std::vector<const char*> names(n - have);
        std::vector<long long> idx(n - have);
        std::vector<unsigned char> w(n - have);
        if (pencil_jit_trace_get(unit_, have, n - have, names.data(), idx.data(), w.data())) return;
        for (long long r = 0; r < n - have; ++r) trace_.push_back({names[r], {idx[r]}, w[r] != 0});
    }
    void check(int st) {
        if (st) throw_last(st);
    }
    [[noreturn]] static void throw_last(int st) { throw_code(st, pencil_cuda_last_error()); }
    // "E-INTERP: device fault: ..." -> PencilError("E-INTERP", "device fault: ...")
    [[noreturn]] static void throw_code(int st, const std::string& msg) {
        std::string code = pencil_status_code(st), text = msg;
        const size_t c = msg.find(": ");
        if (c != std::string::npos && msg.compare(0, 2, "E-") == 0) {
            code = msg.substr(0, c);
            text = msg.substr(c + 2);
        }
        throw pencil::PencilError(code, text);
    }

    pencil_runtime_t rt_ = nullptr;
    pencil_jit_t unit_ = nullptr;
    std::map<std::string, std::vector<pencil::Value>> arrays_;
    std::vector<pencil::MemTrace> trace_;
};

}  // namespace pencil_b200
