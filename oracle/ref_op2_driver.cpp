// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// Command-line driver over the reference's OP2 and OptiML modules (core/src/op2.cpp,
// core/src/optiml.cpp), compiled by oracle/Makefile from the sources where they lie, with the
// nlohmann/json single header that ships with cudnn_frontend in this image (the reference
// expects it under the absent vendor/, proj/README.md:37-39).  Kept apart from ref_driver so
// that one stays vendor-free.
//
//   optiml-lower    FILE.json   lower_optiml (optiml.hpp:38) printed by pretty_print
//   optiml-template FILE.json   optiml_template_text (optiml.hpp:33)
//   op2-lower       FILE.json   lower_op2_model (op2.hpp:94): the unit (pretty_print) followed by
//                               one `driver NAME arg,arg,...` line per par_loop
//   op2-run         FILE.json   interpret_op2_reference (op2.hpp:98): {"dat": [values], ...}
//   canon           FILE        pretty_print(parse_source(FILE)): the canonical form of a unit
// A PencilError prints `error CODE message` and exits 3.
#include <cstdio>
#include <fstream>
#include <sstream>
#include <string>

#include "pencil/lowering.hpp"
#include "pencil/op2.hpp"
#include "pencil/optiml.hpp"
#include "pencil/parser.hpp"

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

static int cmd_op2_lower(const std::string& text) {
    Op2Model m = load_op2_model(text);
    Op2Lowered low = lower_op2_model(m);
    std::fputs(pretty_print(low.ast).c_str(), stdout);
    for (const auto& d : low.drivers) {
        std::string line = "driver " + d.function + " ";
        for (size_t i = 0; i < d.args.size(); ++i) {
            if (i) line += ",";
            line += d.args[i].is_array ? d.args[i].array : std::to_string(d.args[i].value);
        }
        std::printf("%s\n", line.c_str());
    }
    return 0;
}

static int cmd_op2_run(const std::string& text) {
    Op2Model m = load_op2_model(text);
    auto out = interpret_op2_reference(m);
    std::string js = "{";
    bool first = true;
    for (const auto& [name, vals] : out) {
        js += (first ? "\"" : ", \"") + name + "\": [";
        for (size_t i = 0; i < vals.size(); ++i) js += (i ? ", " : "") + std::to_string(vals[i]);
        js += "]";
        first = false;
    }
    std::printf("%s}\n", js.c_str());
    return 0;
}

static int cmd_canon(const std::string& text) {
    ParseResult res = parse_source(text);
    if (!res.ast) return 1;
    attach_directives(*res.ast);
    std::fputs(pretty_print(*res.ast).c_str(), stdout);
    return 0;
}

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: ref_op2_driver optiml-lower|optiml-template|op2-lower|op2-run|canon FILE\n");
        return 2;
    }
    std::string cmd = argv[1], text = slurp(argv[2]);
    try {
        if (cmd == "optiml-lower") {
            std::fputs(pretty_print(lower_optiml(load_optiml_construct(text))).c_str(), stdout);
            return 0;
        }
        if (cmd == "optiml-template") {
            std::fputs(optiml_template_text(load_optiml_construct(text)).c_str(), stdout);
            return 0;
        }
        if (cmd == "op2-lower") return cmd_op2_lower(text);
        if (cmd == "op2-run") return cmd_op2_run(text);
        if (cmd == "canon") return cmd_canon(text);
    } catch (const PencilError& e) {
        std::printf("error %s %s\n", e.code().c_str(), e.what());
        return 3;
    }
    return 2;
}
