// Host frontend (see frontend.h). Grammar and diagnostics follow the
// reference dialect (P/src/parser.cpp:56-442, P/src/compiler.cpp:19-96):
//   program  := { clause }
//   clause   := atom '.' | atom ':-' item { ',' item } '.'
//   item     := atom | VAR '!=' VAR
//   atom     := lname '(' term { ',' term } ')'
//   term     := VAR | INT (u32) | STRING
// with '%' and '//' line comments.
#include "frontend.h"

#include <cctype>
#include <set>
#include <sstream>
#include <unordered_set>

namespace fv::fe {

std::string format(const Diagnostic& d) {
    return std::to_string(d.pos.line) + ":" + std::to_string(d.pos.col) + ": " + d.message;
}

[[noreturn]] static void raise(Pos p, std::string msg) { throw DiagnosticError(Diagnostic{p, std::move(msg)}); }

// ---- dictionary ----------------------------------------------------------------

u32 Dictionary::encode(const std::string& s) {
    auto [it, fresh] = ids_.try_emplace(s, static_cast<u32>(strings_.size()));
    if (fresh) strings_.push_back(s);
    return it->second;
}

bool Dictionary::lookup(const std::string& s, u32* out) const {
    auto it = ids_.find(s);
    if (it == ids_.end()) return false;
    *out = it->second;
    return true;
}

const std::string& Dictionary::decode(u32 v) const {
    if (v >= strings_.size()) fail(FV_ERR_RANGE, "dictionary: value has no string");
    return strings_[v];
}

// ---- scanner ----------------------------------------------------------------------

namespace {

enum class T { Ident, Int, Str, LParen, RParen, Comma, Dot, Turnstile, Neq, Cmp, Bang, End };

struct Tok {
    T kind;
    std::string text;
    u32 number = 0;
    Pos pos;
};

class Scanner {
public:
    explicit Scanner(std::string_view src) : src_(src) {}

    std::vector<Tok> tokens() {
        std::vector<Tok> out;
        while (true) {
            skip_blank();
            const Pos at{line_, col_};
            if (done()) {
                out.push_back({T::End, "", 0, at});
                return out;
            }
            const char ch = src_[i_];
            if (std::isalpha(static_cast<unsigned char>(ch)) || ch == '_') {
                std::string id;
                while (!done() && (std::isalnum(static_cast<unsigned char>(src_[i_])) || src_[i_] == '_')) id += step();
                out.push_back({T::Ident, id, 0, at});
            } else if (std::isdigit(static_cast<unsigned char>(ch))) {
                u64 v = 0;
                while (!done() && std::isdigit(static_cast<unsigned char>(src_[i_]))) {
                    v = v * 10 + static_cast<u64>(src_[i_] - '0');
                    if (v > 0xffffffffull) raise(at, "integer constant out of 32-bit range");
                    step();
                }
                out.push_back({T::Int, "", static_cast<u32>(v), at});
            } else if (ch == '"') {
                out.push_back({T::Str, string_literal(at), 0, at});
            } else {
                step();
                switch (ch) {
                    case '(': out.push_back({T::LParen, "(", 0, at}); break;
                    case ')': out.push_back({T::RParen, ")", 0, at}); break;
                    case ',': out.push_back({T::Comma, ",", 0, at}); break;
                    case '.': out.push_back({T::Dot, ".", 0, at}); break;
                    case ':':
                        if (done() || src_[i_] != '-') raise(at, "expected ':-'");
                        step();
                        out.push_back({T::Turnstile, ":-", 0, at});
                        break;
                    case '!':
                        if (!done() && src_[i_] == '=') {
                            step();
                            out.push_back({T::Neq, "!=", 0, at});
                        } else {
                            out.push_back({T::Bang, "!", 0, at});
                        }
                        break;
                    case '<':
                    case '>':
                    case '=': {
                        std::string op(1, ch);
                        if (!done() && src_[i_] == '=') op += step();
                        out.push_back({T::Cmp, op, 0, at});
                        break;
                    }
                    default: raise(at, std::string("unexpected character '") + ch + "'");
                }
            }
        }
    }

private:
    bool done() const { return i_ >= src_.size(); }

    char step() {
        const char c = src_[i_++];
        if (c == '\n') {
            ++line_;
            col_ = 1;
        } else {
            ++col_;
        }
        return c;
    }

    void skip_blank() {
        while (!done()) {
            const char c = src_[i_];
            if (std::isspace(static_cast<unsigned char>(c))) {
                step();
            } else if (c == '%' || (c == '/' && i_ + 1 < src_.size() && src_[i_ + 1] == '/')) {
                while (!done() && src_[i_] != '\n') step();
            } else {
                return;
            }
        }
    }

    std::string string_literal(Pos at) {
        step();  // opening quote
        std::string s;
        while (true) {
            if (done()) raise(at, "unterminated string constant");
            char c = src_[i_];
            if (c == '"') break;
            if (c == '\n') raise(at, "unterminated string constant");
            if (c == '\\') {
                step();
                if (done()) raise(at, "unterminated string constant");
                static const std::string from = "ntr\"\\", to = "\n\t\r\"\\";
                const size_t k = from.find(src_[i_]);
                if (k == std::string::npos) raise(Pos{line_, col_}, "unknown escape sequence in string");
                c = to[k];
            }
            s += c;
            step();
        }
        step();  // closing quote
        return s;
    }

    std::string_view src_;
    size_t i_ = 0;
    int line_ = 1, col_ = 1;
};

class Reader {
public:
    explicit Reader(std::vector<Tok> toks) : t_(std::move(toks)) {}

    Program program() {
        Program p;
        while (peek().kind != T::End) clause(p);
        return p;
    }

private:
    const Tok& peek(size_t ahead = 0) const {
        const size_t k = std::min(at_ + ahead, t_.size() - 1);
        return t_[k];
    }
    Tok take() {
        Tok t = peek();
        if (at_ < t_.size() - 1) ++at_;
        return t;
    }
    Tok want(T kind, const char* what) {
        if (peek().kind != kind) raise(peek().pos, std::string("expected ") + what);
        return take();
    }

    void clause(Program& p) {
        Atom head = atom(p);
        if (peek().kind == T::Dot) {
            take();
            for (const Term& t : head.args)
                if (!t.is_constant())
                    raise(t.pos, "facts must be ground; use a rule with a body to derive '" + head.rel + "'");
            p.facts.push_back(std::move(head));
            return;
        }
        want(T::Turnstile, "':-' or '.' after atom");
        Rule r;
        r.head = std::move(head);
        do {
            item(p, r);
        } while (peek().kind == T::Comma && (take(), true));
        want(T::Dot, "'.' at end of rule");
        if (r.body.empty()) raise(r.head.pos, "rule body must contain at least one atom");
        p.rules.push_back(std::move(r));
    }

    void item(Program& p, Rule& r) {
        if (peek().kind == T::Bang) raise(peek().pos, "negation is not supported; programs must be positive");
        if (peek().kind == T::Ident && peek(1).kind == T::LParen) {
            r.body.push_back(atom(p));
            return;
        }
        if (peek().kind == T::End) raise(peek().pos, "expected '!=' or an atom");
        const Tok lhs = take();
        if (peek().kind == T::Cmp) raise(peek().pos, "only '!=' guards are supported, got '" + peek().text + "'");
        const Tok op = want(T::Neq, "'!=' or an atom");
        const Tok rhs = take();
        if (lhs.kind != T::Ident || rhs.kind != T::Ident) raise(op.pos, "inequality guards must compare two variables");
        r.guards.push_back({lhs.text, rhs.text, op.pos});
    }

    Atom atom(Program& p) {
        const Tok name = want(T::Ident, "relation name");
        if (std::isupper(static_cast<unsigned char>(name.text[0])))
            raise(name.pos, "relation names must start with a lowercase letter");
        want(T::LParen, "'(' after relation name");
        Atom a;
        a.rel = name.text;
        a.pos = name.pos;
        do {
            a.args.push_back(term());
        } while (peek().kind == T::Comma && (take(), true));
        want(T::RParen, "')' or ',' in argument list");
        declare(p, a);
        return a;
    }

    Term term() {
        const Tok t = take();
        Term x;
        x.pos = t.pos;
        if (t.kind == T::Ident) {
            x.kind = Term::Var;
            x.text = t.text;
        } else if (t.kind == T::Int) {
            x.kind = Term::Int;
            x.number = t.number;
        } else if (t.kind == T::Str) {
            x.kind = Term::Str;
            x.text = t.text;
        } else {
            raise(t.pos, "expected variable or constant");
        }
        return x;
    }

    static void declare(Program& p, const Atom& a) {
        for (const RelDecl& d : p.relations) {
            if (d.name != a.rel) continue;
            if (d.arity != a.args.size())
                raise(a.pos, "relation '" + a.rel + "' used with arity " + std::to_string(a.args.size()) +
                                 " but first used with arity " + std::to_string(d.arity) + " at line " +
                                 std::to_string(d.first_use.line));
            return;
        }
        p.relations.push_back({a.rel, static_cast<u32>(a.args.size()), a.pos});
    }

    std::vector<Tok> t_;
    size_t at_ = 0;
};

void print_term(std::ostringstream& os, const Term& t) {
    if (t.kind == Term::Var) {
        os << t.text;
    } else if (t.kind == Term::Int) {
        os << t.number;
    } else {
        os << '"';
        for (char c : t.text) {
            switch (c) {
                case '"': os << "\\\""; break;
                case '\\': os << "\\\\"; break;
                case '\n': os << "\\n"; break;
                case '\t': os << "\\t"; break;
                case '\r': os << "\\r"; break;
                default: os << c;
            }
        }
        os << '"';
    }
}

void print_atom(std::ostringstream& os, const Atom& a) {
    os << a.rel << "(";
    for (size_t i = 0; i < a.args.size(); ++i) {
        if (i) os << ", ";
        print_term(os, a.args[i]);
    }
    os << ")";
}

}  // namespace

Program parse(std::string_view text) {
    Scanner sc(text);
    return Reader(sc.tokens()).program();
}

std::string print(const Program& p) {
    std::ostringstream os;
    for (const Atom& f : p.facts) {
        print_atom(os, f);
        os << ".\n";
    }
    for (const Rule& r : p.rules) {
        print_atom(os, r.head);
        os << " :- ";
        bool first = true;
        for (const Atom& a : r.body) {
            if (!first) os << ", ";
            print_atom(os, a);
            first = false;
        }
        for (const Guard& g : r.guards) {
            if (!first) os << ", ";
            os << g.lhs << " != " << g.rhs;
            first = false;
        }
        os << ".\n";
    }
    return os.str();
}

std::vector<Diagnostic> validate(const Program& p) {
    std::vector<Diagnostic> out;
    auto arity_ok = [&](const Atom& a) {
        const RelDecl* d = p.find(a.rel);
        if (!d) {
            out.push_back({a.pos, "relation '" + a.rel + "' is not declared"});
        } else if (d->arity != a.args.size()) {
            out.push_back({a.pos, "relation '" + a.rel + "' used with arity " + std::to_string(a.args.size()) +
                                      " but declared with arity " + std::to_string(d->arity)});
        }
    };
    for (const Atom& f : p.facts) {
        arity_ok(f);
        for (const Term& t : f.args)
            if (!t.is_constant()) out.push_back({t.pos, "facts must be ground"});
    }
    for (const Rule& r : p.rules) {
        arity_ok(r.head);
        for (const Atom& a : r.body) arity_ok(a);
        if (r.body.empty()) {
            out.push_back({r.head.pos, "rule body must contain at least one atom"});
            continue;
        }
        std::unordered_set<std::string> vars;
        for (const Atom& a : r.body)
            for (const Term& t : a.args)
                if (!t.is_constant()) vars.insert(t.text);
        for (const Term& t : r.head.args) {
            if (t.is_constant())
                out.push_back({t.pos, "constants in rule heads are not supported"});
            else if (!vars.count(t.text))
                out.push_back({t.pos, "head variable '" + t.text + "' does not occur in the rule body"});
        }
        for (const Guard& g : r.guards)
            for (const std::string* v : {&g.lhs, &g.rhs})
                if (!vars.count(*v))
                    out.push_back({g.pos, "guard variable '" + *v + "' does not occur in the rule body"});
        std::unordered_set<std::string> seen;
        for (size_t i = 0; i < r.body.size(); ++i) {
            const Atom& a = r.body[i];
            bool connected = i == 0;
            for (const Term& t : a.args)
                if (!t.is_constant() && seen.count(t.text)) connected = true;
            if (!connected)
                out.push_back({a.pos, "atom '" + a.rel +
                                          "' shares no variable with the preceding body atoms "
                                          "(cross products are not supported)"});
            for (const Term& t : a.args)
                if (!t.is_constant()) seen.insert(t.text);
        }
    }
    return out;
}

void resolve_strings(Program& p, Dictionary& d) {
    auto fix = [&](Term& t) {
        if (t.kind != Term::Str) return;
        t.number = d.encode(t.text);
        t.kind = Term::Int;
        t.text.clear();
    };
    for (Atom& f : p.facts)
        for (Term& t : f.args) fix(t);
    for (Rule& r : p.rules) {
        for (Term& t : r.head.args) fix(t);
        for (Atom& a : r.body)
            for (Term& t : a.args) fix(t);
    }
}

// compile_rule (P/src/compiler.cpp:19-96): left-to-right joins; the first
// variable an atom shares with earlier atoms is its hash column, further
// shared variables are residual equalities, constants are pre-join
// selections, repeated variables inside one atom are self equalities,
// guards widen the projection.
Plan compile_rule(const Rule& rule, const Program& p) {
    Plan plan;
    plan.head = rule.head.rel;
    plan.head_arity = static_cast<u32>(rule.head.args.size());
    std::unordered_map<std::string, ColRef> first_binding;
    for (u32 s = 0; s < rule.body.size(); ++s) {
        const Atom& a = rule.body[s];
        const RelDecl* decl = p.find(a.rel);
        PlanSource src;
        src.relation = a.rel;
        src.arity = decl ? decl->arity : static_cast<u32>(a.args.size());
        std::unordered_map<std::string, u32> in_atom;
        bool have_join = false;
        PlanJoin jn;
        jn.right_source = s;
        for (u32 c = 0; c < a.args.size(); ++c) {
            const Term& t = a.args[c];
            if (t.is_constant()) {
                if (t.kind == Term::Str) raise(t.pos, "string constant has not been resolved through the dictionary");
                src.const_selects.emplace_back(c, t.number);
                continue;
            }
            auto [it, fresh] = in_atom.try_emplace(t.text, c);
            if (!fresh) {
                src.self_eqs.emplace_back(it->second, c);
                continue;
            }
            auto bound = first_binding.find(t.text);
            if (bound == first_binding.end()) {
                first_binding.emplace(t.text, ColRef{s, c});
            } else if (s > 0) {
                if (!have_join) {
                    have_join = true;
                    jn.left = bound->second;
                    jn.right_col = c;
                } else {
                    jn.residual_eq.emplace_back(bound->second, c);
                }
            }
        }
        plan.sources.push_back(std::move(src));
        if (s > 0) {
            if (!have_join)
                raise(a.pos, "atom '" + a.rel +
                                 "' shares no variable with the preceding body atoms (cross products are not supported)");
            plan.joins.push_back(std::move(jn));
        }
    }
    for (const Term& t : rule.head.args) {
        auto bound = first_binding.find(t.text);
        if (t.is_constant() || bound == first_binding.end()) raise(t.pos, "rule head must project bound variables");
        plan.output_cols.push_back(bound->second);
    }
    auto slot = [&](const std::string& v, Pos pos) -> u32 {
        auto bound = first_binding.find(v);
        if (bound == first_binding.end()) raise(pos, "guard variable '" + v + "' is unbound");
        for (u32 i = 0; i < plan.output_cols.size(); ++i)
            if (plan.output_cols[i] == bound->second) return i;
        plan.output_cols.push_back(bound->second);
        return static_cast<u32>(plan.output_cols.size() - 1);
    };
    for (const Guard& g : rule.guards) {
        const u32 a = slot(g.lhs, g.pos);  // left operand first (deterministic order)
        const u32 b = slot(g.rhs, g.pos);
        plan.guard_neq.emplace_back(a, b);
    }
    return plan;
}

std::vector<Plan> compile(const Program& p) {
    std::vector<Plan> out;
    for (const Rule& r : p.rules) out.push_back(compile_rule(r, p));
    return out;
}

std::vector<RelationDecl> declarations(const Program& p) {
    std::vector<RelationDecl> out;
    for (const RelDecl& d : p.relations) out.push_back({d.name, d.arity});
    return out;
}

std::vector<std::pair<std::string, std::vector<u32>>> program_facts(const Program& p) {
    std::vector<std::pair<std::string, std::vector<u32>>> out;
    std::map<std::string, size_t> at;
    for (const Atom& f : p.facts) {
        auto [it, fresh] = at.try_emplace(f.rel, out.size());
        if (fresh) out.push_back({f.rel, {}});
        auto& rows = out[it->second].second;
        for (const Term& t : f.args) {
            if (t.kind == Term::Str) fail(FV_ERR_ARITY, "program_facts: unresolved string constant");
            rows.push_back(t.number);
        }
    }
    return out;
}

}  // namespace fv::fe
