// Host frontend: Datalog text -> AST -> validated program -> rule plans.
// Same dialect, positions and diagnostic texts as the reference
// (P/src/parser.cpp, P/src/compiler.cpp, P/include/colog/dictionary.hpp),
// written independently for this runtime. Host-only C++ (no device code):
// parsing is one-time, sequential text processing.
#pragma once

#include <cstdint>
#include <string>
#include <string_view>
#include <unordered_map>
#include <vector>

#include "engine.h"

namespace fv::fe {

struct Pos {
    int line = 0;
    int col = 0;
};

struct Term {
    enum Kind { Var, Int, Str };
    Kind kind = Var;
    std::string text;  // variable name / string literal
    u32 number = 0;    // integer constant
    Pos pos;
    bool is_constant() const { return kind != Var; }
    bool same(const Term& o) const {
        return kind == o.kind && (kind == Int ? number == o.number : text == o.text);
    }
};

struct Atom {
    std::string rel;
    std::vector<Term> args;
    Pos pos;
};

struct Guard {
    std::string lhs, rhs;
    Pos pos;
};

struct Rule {
    Atom head;
    std::vector<Atom> body;
    std::vector<Guard> guards;
};

struct RelDecl {
    std::string name;
    u32 arity = 0;
    Pos first_use;
};

struct Program {
    std::vector<RelDecl> relations;  // first-use order
    std::vector<Atom> facts;
    std::vector<Rule> rules;
    const RelDecl* find(const std::string& name) const {
        for (auto& r : relations)
            if (r.name == name) return &r;
        return nullptr;
    }
};

struct Diagnostic {
    Pos pos;
    std::string message;
};

std::string format(const Diagnostic& d);  // "line:col: message"

struct DiagnosticError : Error {
    Diagnostic diag;
    explicit DiagnosticError(Diagnostic d) : Error(FV_ERR_PLAN, format(d)), diag(std::move(d)) {}
};

// Dense first-seen string ids (dictionary.hpp).
class Dictionary {
public:
    u32 encode(const std::string& s);
    bool lookup(const std::string& s, u32* out) const;
    const std::string& decode(u32 v) const;  // throws FV_ERR_RANGE
    size_t size() const { return strings_.size(); }
    bool empty() const { return strings_.empty(); }

private:
    std::vector<std::string> strings_;
    std::unordered_map<std::string, u32> ids_;
};

Program parse(std::string_view text);
std::vector<Diagnostic> validate(const Program& p);
std::string print(const Program& p);
void resolve_strings(Program& p, Dictionary& d);
Plan compile_rule(const Rule& rule, const Program& p);
std::vector<Plan> compile(const Program& p);
std::vector<RelationDecl> declarations(const Program& p);

// Ground facts written in the program text, per relation, row-major.
std::vector<std::pair<std::string, std::vector<u32>>> program_facts(const Program& p);

}  // namespace fv::fe
