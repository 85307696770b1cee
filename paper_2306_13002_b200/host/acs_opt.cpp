// acs_opt.cpp — host stage (a): equality-saturation optimizer for the
// kernel-subset loop nests (include/accsat_opt.h).
//
// A fresh C++ implementation of the reference pipeline's algorithm
// (proj/src/pipeline.cpp:47-194): parse -> regions -> value-numbered region
// body in an e-graph -> saturate (Table-I rules + constant folding) ->
// extract under the reference cost model -> depth-one temps (+ bulk loads)
// -> module text with only the region bodies replaced.
//
//  * Parsing accepts the satcc kernel subset (proj/src/parser.cpp:60-554);
//    pragma lines, loop headers, conditions and store targets are re-emitted
//    verbatim from the source bytes.
//  * Value numbering mirrors the reference SSA semantics
//    (proj/src/ssa.cpp:129-550): per-base load epochs advanced by
//    may-aliasing stores (different bases never alias; same base aliases
//    unless some subscript position holds two unequal constants,
//    ssa.cpp:63-74), same-scope identical-subscript store->load forwarding,
//    if-φ for names the branches disagree on, conditional stores kill reuse.
//    Sequential inner loops inside a region take for-/exit-phi leaves and
//    start new load epochs for the bases they store (epoch kills).
//  * Rules: FMA1-3, COMM-ADD/MUL, ASSOC-ADD1/2, ASSOC-MUL1/2
//    (proj/src/rules.cpp:123-143) with the reference limits (10000 nodes,
//    10 s, 10 iterations) and constant folding with host double arithmetic.
//  * Extraction: bottom-up tree-cost greedy (ties to the oldest node, i.e.
//    the program as written) followed by an incremental DAG-cost local
//    search: a class switches node whenever that lowers the exact cost of the
//    shared selection.  Then, optionally, the exact 0/1 ILP through a
//    registered solver (exact_refine; method "ilp" when proven optimal).
//  * Codegen: one `_v<class>` temp per selected operation class, placed before
//    the first statement of the innermost block that encloses all its uses
//    (never hoisted out of an if-branch that alone uses it); bulk mode moves
//    load temps upward past statements that neither store to a may-aliasing
//    element of the same base nor assign a scalar their subscripts read, and
//    orders loads sharing a slot by (base, subscript text).  FMA temps print
//    as `a + b * c` (the reference convention, proj/src/printer.cpp:114-125).
#include <algorithm>
#include <cctype>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <optional>
#include <random>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/accsat_opt.h"

namespace acsopt {

struct SyntaxErr : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct Unsupported : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// ============================================================================
// Lexer

struct Tok {
    enum K { Int, Float, Ident, Kw, Op, Pragma, End } k = End;
    std::string s;
    size_t off = 0, end = 0;
    int line = 0;
};

static std::vector<Tok> lex(const std::string& src) {
    std::vector<Tok> out;
    size_t i = 0, n = src.size();
    int line = 1;
    auto push = [&](Tok::K k, size_t b, size_t e) {
        Tok t;
        t.k = k;
        t.s = src.substr(b, e - b);
        t.off = b;
        t.end = e;
        t.line = line;
        out.push_back(std::move(t));
    };
    static const std::set<std::string> kws = {"int", "double", "void", "if", "else", "for"};
    while (i < n) {
        char c = src[i];
        if (c == '\n') {
            line++;
            i++;
            continue;
        }
        if (isspace(static_cast<unsigned char>(c))) {
            i++;
            continue;
        }
        if (c == '/' && i + 1 < n && src[i + 1] == '/') {
            while (i < n && src[i] != '\n') i++;
            continue;
        }
        if (c == '/' && i + 1 < n && src[i + 1] == '*') {
            size_t e = src.find("*/", i + 2);
            if (e == std::string::npos) throw SyntaxErr("unterminated block comment");
            for (size_t k = i; k < e; ++k) line += src[k] == '\n';
            i = e + 2;
            continue;
        }
        if (c == '#') {
            size_t e = i;
            for (;;) {
                size_t nl = src.find('\n', e);
                if (nl == std::string::npos) nl = n;
                if (nl > 0 && nl < n && src[nl - 1] == '\\') {
                    e = nl + 1;
                    continue;
                }
                e = nl;
                break;
            }
            std::string t = src.substr(i, e - i);
            size_t p = t.find_first_not_of("# \t");
            if (p == std::string::npos || t.compare(p, 6, "pragma") != 0)
                throw SyntaxErr("preprocessor directives other than #pragma are not supported");
            push(Tok::Pragma, i, e);
            i = e;
            continue;
        }
        if (isdigit(static_cast<unsigned char>(c)) || (c == '.' && i + 1 < n && isdigit(static_cast<unsigned char>(src[i + 1])))) {
            size_t b = i;
            bool flt = false;
            while (i < n && isdigit(static_cast<unsigned char>(src[i]))) i++;
            if (i < n && src[i] == '.') {
                flt = true;
                i++;
                while (i < n && isdigit(static_cast<unsigned char>(src[i]))) i++;
            }
            if (i < n && (src[i] == 'e' || src[i] == 'E')) {
                size_t s = i;
                i++;
                if (i < n && (src[i] == '+' || src[i] == '-')) i++;
                if (i < n && isdigit(static_cast<unsigned char>(src[i]))) {
                    flt = true;
                    while (i < n && isdigit(static_cast<unsigned char>(src[i]))) i++;
                } else {
                    i = s;
                }
            }
            if (i < n && (src[i] == 'f' || src[i] == 'F')) {
                flt = true;
                i++;
            }
            push(flt ? Tok::Float : Tok::Int, b, i);
            continue;
        }
        if (isalpha(static_cast<unsigned char>(c)) || c == '_') {
            size_t b = i;
            while (i < n && (isalnum(static_cast<unsigned char>(src[i])) || src[i] == '_')) i++;
            push(kws.count(src.substr(b, i - b)) ? Tok::Kw : Tok::Ident, b, i);
            continue;
        }
        static const char* two[] = {"++", "--", "+=", "-=", "*=", "/=", "<=", ">=", "==", "!=", "&&", "||"};
        bool got = false;
        for (const char* t : two)
            if (src.compare(i, 2, t) == 0) {
                push(Tok::Op, i, i + 2);
                i += 2;
                got = true;
                break;
            }
        if (got) continue;
        if (std::strchr("+-*/%<>=!(){}[];,", c)) {
            push(Tok::Op, i, i + 1);
            i++;
            continue;
        }
        throw SyntaxErr("line " + std::to_string(line) + ": unexpected character");
    }
    Tok e;
    e.k = Tok::End;
    e.off = e.end = n;
    out.push_back(e);
    return out;
}

// ============================================================================
// AST

struct Expr {
    enum K { Int, Float, Var, Ref, Un, Bin, Call } k = Int;
    long long iv = 0;
    double fv = 0;
    std::string text;  // literal spelling / name / callee / array base
    std::string op;
    std::vector<std::unique_ptr<Expr>> kids;
    size_t beg = 0, end = 0;
};
using ExprP = std::unique_ptr<Expr>;

struct Stmt {
    enum K { Decl, Assign, If, For, Block, Call, Empty } k = Empty;
    size_t beg = 0, end = 0;
    std::vector<std::string> pragmas;
    std::string ty;
    struct D {
        std::string name;
        std::vector<long long> dims;
        ExprP init;
    };
    std::vector<D> decls;
    ExprP lhs, rhs, cond, call;
    std::unique_ptr<Stmt> then_s, else_s, init, step, body;
    std::vector<std::unique_ptr<Stmt>> stmts;
    std::string loopvar;
};
using StmtP = std::unique_ptr<Stmt>;

struct Param {
    std::string ty, name;
    std::vector<long long> dims;
};
struct Func {
    std::string name;
    std::vector<Param> params;
    StmtP body;
};
struct Module {
    std::vector<Func> funcs;
    std::vector<StmtP> globals;
};

class Parser {
  public:
    explicit Parser(std::vector<Tok> t) : t_(std::move(t)) {}
    Module module() {
        Module m;
        while (cur().k != Tok::End) {
            auto prag = pragmas();
            if (cur().k == Tok::End) break;
            std::string ty = adv().s;
            if (ty != "void" && ty != "int" && ty != "double") throw SyntaxErr("expected declaration");
            std::string name = ident();
            if (is("(")) {
                if (ty != "void") throw Unsupported("non-void function");
                Func f;
                f.name = name;
                params(f.params);
                f.body = block();
                m.funcs.push_back(std::move(f));
            } else {
                p_--;
                auto d = declarators(ty);
                m.globals.push_back(std::move(d));
            }
        }
        return m;
    }

  private:
    std::vector<Tok> t_;
    size_t p_ = 0;
    const Tok& cur() const { return t_[p_]; }
    const Tok& adv() { return t_[p_++]; }
    bool is(const char* s) const { return (cur().k == Tok::Op || cur().k == Tok::Kw) && cur().s == s; }
    bool accept(const char* s) {
        if (is(s)) {
            p_++;
            return true;
        }
        return false;
    }
    void expect(const char* s) {
        if (!accept(s)) throw SyntaxErr("line " + std::to_string(cur().line) + ": expected '" + s + "'");
    }
    std::string ident() {
        if (cur().k != Tok::Ident) throw SyntaxErr("line " + std::to_string(cur().line) + ": expected identifier");
        return adv().s;
    }
    std::vector<std::string> pragmas() {
        std::vector<std::string> o;
        while (cur().k == Tok::Pragma) o.push_back(adv().s);
        return o;
    }
    void params(std::vector<Param>& out) {
        expect("(");
        if (accept(")")) return;
        if (is("void") && t_[p_ + 1].s == ")") {
            p_ += 2;
            return;
        }
        do {
            Param p;
            p.ty = adv().s;
            if (p.ty != "int" && p.ty != "double") throw SyntaxErr("expected parameter type");
            p.name = ident();
            while (accept("[")) {
                if (cur().k != Tok::Int) throw SyntaxErr("constant array dimension expected");
                p.dims.push_back(std::stoll(adv().s));
                expect("]");
            }
            out.push_back(std::move(p));
        } while (accept(","));
        expect(")");
    }
    StmtP declarators(const std::string& ty) {
        auto s = std::make_unique<Stmt>();
        s->k = Stmt::Decl;
        s->ty = ty;
        do {
            Stmt::D d;
            d.name = ident();
            while (accept("[")) {
                if (cur().k != Tok::Int) throw SyntaxErr("constant array dimension expected");
                d.dims.push_back(std::stoll(adv().s));
                expect("]");
            }
            if (accept("=")) d.init = expr();
            s->decls.push_back(std::move(d));
        } while (accept(","));
        expect(";");
        return s;
    }
    StmtP block() {
        auto s = std::make_unique<Stmt>();
        s->k = Stmt::Block;
        s->beg = cur().off;
        expect("{");
        for (;;) {
            auto prag = pragmas();
            if (is("}")) {
                if (!prag.empty()) {
                    auto e = std::make_unique<Stmt>();
                    e->k = Stmt::Empty;
                    e->pragmas = std::move(prag);
                    s->stmts.push_back(std::move(e));
                }
                break;
            }
            if (cur().k == Tok::End) throw SyntaxErr("unterminated block");
            auto st = stmt();
            st->pragmas.insert(st->pragmas.begin(), prag.begin(), prag.end());
            s->stmts.push_back(std::move(st));
        }
        s->end = cur().end;
        expect("}");
        return s;
    }
    StmtP stmt() {
        auto prag = pragmas();
        size_t b = cur().off;
        StmtP s;
        if (is("{")) {
            s = block();
        } else if (is("int") || is("double")) {
            std::string ty = adv().s;
            s = declarators(ty);
        } else if (accept("if")) {
            s = std::make_unique<Stmt>();
            s->k = Stmt::If;
            expect("(");
            s->cond = expr();
            expect(")");
            s->then_s = stmt();
            if (accept("else")) s->else_s = stmt();
        } else if (accept("for")) {
            s = std::make_unique<Stmt>();
            s->k = Stmt::For;
            expect("(");
            if (!is(";")) s->init = simple();
            expect(";");
            if (!is(";")) s->cond = expr();
            expect(";");
            if (!is(")")) s->step = simple();
            expect(")");
            s->body = stmt();
            if (s->init && s->init->k == Stmt::Assign && s->init->lhs->k == Expr::Var) s->loopvar = s->init->lhs->text;
        } else if (accept(";")) {
            s = std::make_unique<Stmt>();
            s->k = Stmt::Empty;
        } else {
            s = simple();
            expect(";");
        }
        s->beg = b;
        s->end = t_[p_ - 1].end;
        s->pragmas.insert(s->pragmas.begin(), prag.begin(), prag.end());
        return s;
    }
    StmtP simple() {
        size_t b = cur().off;
        auto lhs = postfix();
        auto s = std::make_unique<Stmt>();
        s->beg = b;
        const char* comp[] = {"+=", "-=", "*=", "/="};
        for (const char* c : comp)
            if (accept(c)) {
                s->k = Stmt::Assign;
                auto r = std::make_unique<Expr>();
                r->k = Expr::Bin;
                r->op = std::string(1, c[0]);
                r->kids.push_back(clone(*lhs));
                r->kids.push_back(expr());
                s->lhs = std::move(lhs);
                s->rhs = std::move(r);
                return s;
            }
        if (accept("++") || accept("--")) {
            bool inc = t_[p_ - 1].s == "++";
            s->k = Stmt::Assign;
            auto r = std::make_unique<Expr>();
            r->k = Expr::Bin;
            r->op = inc ? "+" : "-";
            r->kids.push_back(clone(*lhs));
            auto one = std::make_unique<Expr>();
            one->k = Expr::Int;
            one->iv = 1;
            one->text = "1";
            r->kids.push_back(std::move(one));
            s->lhs = std::move(lhs);
            s->rhs = std::move(r);
            return s;
        }
        if (accept("=")) {
            s->k = Stmt::Assign;
            s->lhs = std::move(lhs);
            s->rhs = expr();
            return s;
        }
        if (lhs->k == Expr::Call) {
            s->k = Stmt::Call;
            s->call = std::move(lhs);
            return s;
        }
        throw SyntaxErr("line " + std::to_string(cur().line) + ": expected assignment");
    }
    static ExprP clone(const Expr& e) {
        auto c = std::make_unique<Expr>();
        c->k = e.k;
        c->iv = e.iv;
        c->fv = e.fv;
        c->text = e.text;
        c->op = e.op;
        c->beg = e.beg;
        c->end = e.end;
        for (auto& k : e.kids) c->kids.push_back(clone(*k));
        return c;
    }
    ExprP expr(int level = 0) {
        static const std::vector<std::vector<std::string>> prec = {
            {"||"}, {"&&"}, {"==", "!="}, {"<", "<=", ">", ">="}, {"+", "-"}, {"*", "/", "%"}};
        if (level == (int)prec.size()) return unary();
        size_t b = cur().off;
        auto e = expr(level + 1);
        for (;;) {
            bool hit = false;
            if (cur().k == Tok::Op)
                for (auto& o : prec[level])
                    if (cur().s == o) hit = true;
            if (!hit) break;
            std::string op = adv().s;
            auto r = expr(level + 1);
            auto n = std::make_unique<Expr>();
            n->k = Expr::Bin;
            n->op = op;
            n->kids.push_back(std::move(e));
            n->kids.push_back(std::move(r));
            n->beg = b;
            n->end = t_[p_ - 1].end;
            e = std::move(n);
        }
        return e;
    }
    ExprP unary() {
        size_t b = cur().off;
        if (accept("-") || accept("!")) {
            std::string op = t_[p_ - 1].s;
            auto n = std::make_unique<Expr>();
            n->k = Expr::Un;
            n->op = op;
            n->kids.push_back(unary());
            n->beg = b;
            n->end = t_[p_ - 1].end;
            return n;
        }
        if (accept("+")) return unary();
        return postfix();
    }
    ExprP postfix() {
        const Tok& t = adv();
        auto e = std::make_unique<Expr>();
        e->beg = t.off;
        if (t.k == Tok::Int) {
            e->k = Expr::Int;
            e->iv = std::stoll(t.s);
            e->text = t.s;
        } else if (t.k == Tok::Float) {
            e->k = Expr::Float;
            std::string s = t.s;
            if (!s.empty() && (s.back() == 'f' || s.back() == 'F')) s.pop_back();
            e->fv = std::strtod(s.c_str(), nullptr);
            e->text = t.s;
        } else if (t.k == Tok::Op && t.s == "(") {
            auto in = expr();
            expect(")");
            return in;
        } else if (t.k == Tok::Ident) {
            e->text = t.s;
            if (accept("(")) {
                e->k = Expr::Call;
                if (!accept(")")) {
                    do e->kids.push_back(expr());
                    while (accept(","));
                    expect(")");
                }
            } else if (is("[")) {
                e->k = Expr::Ref;
                while (accept("[")) {
                    e->kids.push_back(expr());
                    expect("]");
                }
            } else {
                e->k = Expr::Var;
            }
        } else {
            throw SyntaxErr("line " + std::to_string(t.line) + ": unexpected '" + t.s + "'");
        }
        e->end = t_[p_ - 1].end;
        return e;
    }
};

// ============================================================================
// Regions (find_regions, proj/src/ast.cpp:333-398)

static bool marked(const std::vector<std::string>& pragmas) {
    static const std::set<std::string> words = {"gang", "worker", "vector", "simd", "teams", "distribute", "kernels",
                                                 "parallel"};
    for (auto& p : pragmas) {
        std::string w;
        for (size_t i = 0; i <= p.size(); ++i) {
            char c = i < p.size() ? p[i] : ' ';
            if (isalnum(static_cast<unsigned char>(c)) || c == '_') {
                w += c;
            } else {
                if (words.count(w)) return true;
                w.clear();
            }
        }
    }
    return false;
}

struct Region {
    Func* fn = nullptr;
    Stmt* anchor = nullptr;
    std::vector<std::string> loopvars;
    int index = 0;
};

static bool has_marked_loop(const Stmt& s) {
    if (s.k == Stmt::For && marked(s.pragmas)) return true;
    for (const Stmt* c : {s.then_s.get(), s.else_s.get(), s.body.get()})
        if (c && has_marked_loop(*c)) return true;
    for (auto& c : s.stmts)
        if (has_marked_loop(*c)) return true;
    return false;
}

static void find_in(Func& fn, Stmt& s, std::vector<std::string>& lv, std::vector<Region>& out) {
    if (s.k == Stmt::For) {
        if (marked(s.pragmas) && !has_marked_loop(*s.body)) {
            Region r;
            r.fn = &fn;
            r.anchor = &s;
            r.loopvars = lv;
            if (!s.loopvar.empty()) r.loopvars.push_back(s.loopvar);
            r.index = (int)out.size();
            out.push_back(r);
            return;
        }
        if (!s.loopvar.empty()) lv.push_back(s.loopvar);
        find_in(fn, *s.body, lv, out);
        if (!s.loopvar.empty()) lv.pop_back();
    } else if (s.k == Stmt::If) {
        find_in(fn, *s.then_s, lv, out);
        if (s.else_s) find_in(fn, *s.else_s, lv, out);
    } else if (s.k == Stmt::Block) {
        for (auto& c : s.stmts) find_in(fn, *c, lv, out);
    }
}

// ============================================================================
// E-graph

enum class Op : uint8_t { CInt, CFlt, Var, Load, Phi, Neg, Not, Add, Sub, Mul, Div, Mod, Lt, Le, Gt, Ge, Eq, Ne, And, Or, Fma, Call };

static const char* binop_text(Op o) {
    switch (o) {
        case Op::Add: return "+";
        case Op::Sub: return "-";
        case Op::Mul: return "*";
        case Op::Div: return "/";
        case Op::Mod: return "%";
        case Op::Lt: return "<";
        case Op::Le: return "<=";
        case Op::Gt: return ">";
        case Op::Ge: return ">=";
        case Op::Eq: return "==";
        case Op::Ne: return "!=";
        case Op::And: return "&&";
        case Op::Or: return "||";
        default: return "?";
    }
}

struct Node {
    Op op = Op::CInt;
    long long iv = 0;
    uint64_t fbits = 0;
    std::string sym;
    int aux = 0;
    std::vector<int> kids;
    bool operator==(const Node& o) const {
        return op == o.op && iv == o.iv && fbits == o.fbits && sym == o.sym && aux == o.aux && kids == o.kids;
    }
    double fv() const {
        double d;
        std::memcpy(&d, &fbits, 8);
        return d;
    }
};
struct NodeHash {
    size_t operator()(const Node& n) const {
        size_t h = std::hash<int>()((int)n.op) * 1000003u;
        h ^= std::hash<long long>()(n.iv) + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2);
        h ^= std::hash<uint64_t>()(n.fbits) + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2);
        h ^= std::hash<std::string>()(n.sym) + (h << 6) + (h >> 2);
        h ^= std::hash<int>()(n.aux) + (h << 6) + (h >> 2);
        for (int k : n.kids) h ^= std::hash<int>()(k) + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2);
        return h;
    }
};

struct CVal {
    bool is_int;
    long long i;
    double d;
    double as_d() const { return is_int ? (double)i : d; }
};

struct EClass {
    std::vector<Node> nodes;
    std::vector<int> serial;
    bool is_int = false;
    std::optional<CVal> cval;
};

class EGraph {
  public:
    int find(int a) const {
        while (uf_[a] != a) {
            uf_[a] = uf_[uf_[a]];
            a = uf_[a];
        }
        return a;
    }
    Node canon(Node n) const {
        for (int& k : n.kids) k = find(k);
        return n;
    }
    int add(Node n, bool leaf_int = false) {
        n = canon(n);
        auto it = memo_.find(n);
        if (it != memo_.end()) return find(it->second);
        int id = (int)cls_.size();
        uf_.push_back(id);
        EClass c;
        c.is_int = infer_int(n, leaf_int);
        if (n.op == Op::CInt) c.cval = CVal{true, n.iv, 0};
        if (n.op == Op::CFlt) c.cval = CVal{false, 0, n.fv()};
        c.nodes.push_back(n);
        c.serial.push_back(serial_++);
        cls_.push_back(std::move(c));
        memo_[n] = id;
        nnodes_++;
        return id;
    }
    // union; the LOWER id survives (deterministic, oldest class wins)
    int merge(int a, int b) {
        a = find(a);
        b = find(b);
        if (a == b) return a;
        if (b < a) std::swap(a, b);
        uf_[b] = a;
        EClass& A = cls_[a];
        EClass& B = cls_[b];
        for (size_t i = 0; i < B.nodes.size(); ++i) {
            A.nodes.push_back(B.nodes[i]);
            A.serial.push_back(B.serial[i]);
        }
        if (!A.cval && B.cval) A.cval = B.cval;
        B.nodes.clear();
        B.serial.clear();
        unions_++;
        dirty_ = true;
        return a;
    }
    // restore congruence: re-canonicalise every node; nodes that collide
    // merge their classes; repeat until stable
    void rebuild() {
        while (dirty_) {
            dirty_ = false;
            memo_.clear();
            nnodes_ = 0;
            for (int c = 0; c < (int)cls_.size(); ++c) {
                if (find(c) != c) continue;
                EClass& C = cls_[c];
                std::vector<Node> nn;
                std::vector<int> ns;
                for (size_t i = 0; i < C.nodes.size(); ++i) {
                    Node n = canon(C.nodes[i]);
                    bool dup = false;
                    for (size_t j = 0; j < nn.size(); ++j)
                        if (nn[j] == n) {
                            ns[j] = std::min(ns[j], C.serial[i]);
                            dup = true;
                            break;
                        }
                    if (!dup) {
                        nn.push_back(n);
                        ns.push_back(C.serial[i]);
                    }
                }
                C.nodes = std::move(nn);
                C.serial = std::move(ns);
            }
            for (int c = 0; c < (int)cls_.size(); ++c) {
                if (find(c) != c) continue;
                for (const Node& n : cls_[c].nodes) {
                    auto it = memo_.find(n);
                    if (it == memo_.end()) {
                        memo_[n] = c;
                        nnodes_++;
                    } else if (find(it->second) != find(c)) {
                        merge(it->second, c);
                    }
                }
            }
        }
    }
    std::vector<int> classes() const {
        std::vector<int> o;
        for (int c = 0; c < (int)cls_.size(); ++c)
            if (find(c) == c) o.push_back(c);
        return o;
    }
    EClass& cls(int id) { return cls_[find(id)]; }
    const EClass& cls(int id) const { return cls_[find(id)]; }
    size_t n_nodes() const { return nnodes_; }
    int n_unions() const { return unions_; }
    int n_alloc() const { return (int)cls_.size(); }
    bool is_int(int id) const { return cls(id).is_int; }
    std::optional<CVal> cval(int id) const { return cls(id).cval; }

  private:
    mutable std::vector<int> uf_;
    std::vector<EClass> cls_;
    std::unordered_map<Node, int, NodeHash> memo_;
    size_t nnodes_ = 0;
    int unions_ = 0;
    int serial_ = 0;
    bool dirty_ = false;

    bool infer_int(const Node& n, bool leaf_int) const {
        switch (n.op) {
            case Op::CInt: return true;
            case Op::CFlt: return false;
            case Op::Var:
            case Op::Load:
            case Op::Phi: return leaf_int;
            case Op::Call: return false;
            case Op::Neg: return is_int(n.kids[0]);
            case Op::Not:
            case Op::Mod:
            case Op::Lt:
            case Op::Le:
            case Op::Gt:
            case Op::Ge:
            case Op::Eq:
            case Op::Ne:
            case Op::And:
            case Op::Or: return true;
            case Op::Fma: return is_int(n.kids[0]) && is_int(n.kids[1]) && is_int(n.kids[2]);
            default: return is_int(n.kids[0]) && is_int(n.kids[1]);
        }
    }
};

// ---- cost model (proj/src/cost.cpp:9-41) ----
static long long node_cost(const Node& n) {
    switch (n.op) {
        case Op::CInt:
        case Op::CFlt: return 0;
        case Op::Var:
        case Op::Phi: return 1;
        case Op::Load:
        case Op::Div:
        case Op::Mod:
        case Op::Call: return 100;
        default: return 10;
    }
}
static bool selection_leaf(const Node& n) { return n.op == Op::Phi; }

// ---- constant folding (host semantics == the interpreter's) ----
static std::optional<CVal> fold(const EGraph& g, const Node& n) {
    switch (n.op) {
        case Op::Neg:
        case Op::Add:
        case Op::Sub:
        case Op::Mul:
        case Op::Div:
        case Op::Mod:
        case Op::Fma: break;
        default: return std::nullopt;
    }
    std::vector<CVal> k;
    for (int c : n.kids) {
        auto v = g.cval(c);
        if (!v) return std::nullopt;
        k.push_back(*v);
    }
    bool ints = true;
    for (auto& v : k) ints &= v.is_int;
    if (ints) {
        long long r;
        switch (n.op) {
            case Op::Neg: r = -k[0].i; break;
            case Op::Add: r = k[0].i + k[1].i; break;
            case Op::Sub: r = k[0].i - k[1].i; break;
            case Op::Mul: r = k[0].i * k[1].i; break;
            case Op::Div:
                if (!k[1].i) return std::nullopt;
                r = k[0].i / k[1].i;
                break;
            case Op::Mod:
                if (!k[1].i) return std::nullopt;
                r = k[0].i % k[1].i;
                break;
            default: r = k[0].i + k[1].i * k[2].i; break;
        }
        return CVal{true, r, 0};
    }
    if (n.op == Op::Mod) return std::nullopt;
    double r;
    switch (n.op) {
        case Op::Neg: r = -k[0].as_d(); break;
        case Op::Add: r = k[0].as_d() + k[1].as_d(); break;
        case Op::Sub: r = k[0].as_d() - k[1].as_d(); break;
        case Op::Mul: r = k[0].as_d() * k[1].as_d(); break;
        case Op::Div:
            if (k[1].as_d() == 0.0) return std::nullopt;
            r = k[0].as_d() / k[1].as_d();
            break;
        default: {
            volatile double p = k[1].as_d() * k[2].as_d();   // two roundings, as apply_fma
            r = k[0].as_d() + p;
        }
    }
    return CVal{false, 0, r};
}

static bool fold_constants(EGraph& g) {
    bool changed = false;
    for (bool progress = true; progress;) {
        progress = false;
        for (int c : g.classes()) {
            if (g.cls(c).cval) continue;
            for (const Node& n : g.cls(c).nodes) {
                auto v = fold(g, g.canon(n));
                if (v) {
                    g.cls(c).cval = *v;
                    progress = changed = true;
                    break;
                }
            }
        }
    }
    for (int c : g.classes()) {
        auto v = g.cls(c).cval;
        if (!v) continue;
        bool has = false;
        for (const Node& n : g.cls(c).nodes) has |= n.op == Op::CInt || n.op == Op::CFlt;
        if (has) continue;
        Node k;
        if (v->is_int) {
            k.op = Op::CInt;
            k.iv = v->i;
        } else {
            k.op = Op::CFlt;
            std::memcpy(&k.fbits, &v->d, 8);
        }
        g.merge(c, g.add(k, v->is_int));
        changed = true;
    }
    g.rebuild();
    return changed;
}

// ---- rules (Table I, proj/src/rules.cpp:123-143), hand-matched ----
struct SatResult {
    std::string stop = "saturated";
    int iters = 0;
    size_t nodes = 0;
};

static SatResult saturate(EGraph& g, long max_nodes, double max_time, int max_iters) {
    using Clock = std::chrono::steady_clock;
    auto deadline = Clock::now() + std::chrono::microseconds((long long)(max_time * 1e6));
    SatResult r;
    fold_constants(g);
    auto limit = [&]() -> const char* {
        if ((long)g.n_nodes() >= max_nodes) return "node_limit";
        if (Clock::now() > deadline) return "time_limit";
        return nullptr;
    };
    auto mk = [&](Op op, std::vector<int> kids) {
        Node n;
        n.op = op;
        n.kids = std::move(kids);
        return g.add(n);
    };
    const char* stop = nullptr;
    bool saturated = false;
    while (r.iters < max_iters && !stop && !saturated) {
        r.iters++;
        auto before = std::make_pair(g.n_alloc(), g.n_unions());
        for (int rule = 0; rule < 9 && !stop; ++rule) {
            if ((stop = limit())) break;
            // collect matches on a snapshot, then apply
            std::vector<std::pair<int, std::vector<int>>> m;   // (class, slots a b c)
            for (int c : g.classes()) {
                for (const Node& n0 : g.cls(c).nodes) {
                    Node n = g.canon(n0);
                    auto sub_nodes = [&](int cls, Op op) {
                        std::vector<std::vector<int>> o;
                        for (const Node& s : g.cls(cls).nodes)
                            if (s.op == op) o.push_back(g.canon(s).kids);
                        return o;
                    };
                    switch (rule) {
                        case 0:  // FMA1  a + b*c -> fma(a, b, c)
                            if (n.op == Op::Add)
                                for (auto& bc : sub_nodes(n.kids[1], Op::Mul)) m.push_back({c, {n.kids[0], bc[0], bc[1]}});
                            break;
                        case 1:  // FMA2  a - b*c -> fma(a, -b, c)
                            if (n.op == Op::Sub)
                                for (auto& bc : sub_nodes(n.kids[1], Op::Mul)) m.push_back({c, {n.kids[0], bc[0], bc[1]}});
                            break;
                        case 2:  // FMA3  b*c - a -> fma(-a, b, c)
                            if (n.op == Op::Sub)
                                for (auto& bc : sub_nodes(n.kids[0], Op::Mul)) m.push_back({c, {n.kids[1], bc[0], bc[1]}});
                            break;
                        case 3:  // COMM-ADD
                            if (n.op == Op::Add) m.push_back({c, {n.kids[0], n.kids[1]}});
                            break;
                        case 4:  // COMM-MUL
                            if (n.op == Op::Mul) m.push_back({c, {n.kids[0], n.kids[1]}});
                            break;
                        case 5:  // ASSOC-ADD1  a + (b + c) -> (a + b) + c
                            if (n.op == Op::Add)
                                for (auto& bc : sub_nodes(n.kids[1], Op::Add)) m.push_back({c, {n.kids[0], bc[0], bc[1]}});
                            break;
                        case 6:  // ASSOC-ADD2  (a + b) + c -> a + (b + c)
                            if (n.op == Op::Add)
                                for (auto& ab : sub_nodes(n.kids[0], Op::Add)) m.push_back({c, {ab[0], ab[1], n.kids[1]}});
                            break;
                        case 7:  // ASSOC-MUL1
                            if (n.op == Op::Mul)
                                for (auto& bc : sub_nodes(n.kids[1], Op::Mul)) m.push_back({c, {n.kids[0], bc[0], bc[1]}});
                            break;
                        case 8:  // ASSOC-MUL2
                            if (n.op == Op::Mul)
                                for (auto& ab : sub_nodes(n.kids[0], Op::Mul)) m.push_back({c, {ab[0], ab[1], n.kids[1]}});
                            break;
                    }
                }
            }
            for (auto& [c, s] : m) {
                if ((stop = limit())) break;
                int rhs;
                switch (rule) {
                    case 0: rhs = mk(Op::Fma, {s[0], s[1], s[2]}); break;
                    case 1: rhs = mk(Op::Fma, {s[0], mk(Op::Neg, {s[1]}), s[2]}); break;
                    case 2: rhs = mk(Op::Fma, {mk(Op::Neg, {s[0]}), s[1], s[2]}); break;
                    case 3: rhs = mk(Op::Add, {s[1], s[0]}); break;
                    case 4: rhs = mk(Op::Mul, {s[1], s[0]}); break;
                    case 5: rhs = mk(Op::Add, {mk(Op::Add, {s[0], s[1]}), s[2]}); break;
                    case 6: rhs = mk(Op::Add, {s[0], mk(Op::Add, {s[1], s[2]})}); break;
                    case 7: rhs = mk(Op::Mul, {mk(Op::Mul, {s[0], s[1]}), s[2]}); break;
                    default: rhs = mk(Op::Mul, {s[0], mk(Op::Mul, {s[1], s[2]})}); break;
                }
                g.merge(c, rhs);
            }
            g.rebuild();
        }
        if (!stop) {
            fold_constants(g);
            saturated = std::make_pair(g.n_alloc(), g.n_unions()) == before;
        }
    }
    r.stop = stop ? stop : (saturated ? "saturated" : "iter_limit");
    r.nodes = g.n_nodes();
    return r;
}

// ---- extraction ----
struct Extraction {
    std::map<int, Node> choice;   // canonical class -> chosen (canonical) node
    long long total = 0;
    int fma = 0;
};

static void reach(const EGraph& g, const std::map<int, Node>& ch, int c, std::set<int>& seen) {
    c = g.find(c);
    if (!seen.insert(c).second) return;
    const Node& n = ch.at(c);
    if (selection_leaf(n)) return;
    for (int k : n.kids) reach(g, ch, k, seen);
}

static long long dag_cost(const EGraph& g, const std::map<int, Node>& ch, const std::vector<int>& roots) {
    std::set<int> seen;
    for (int r : roots) reach(g, ch, r, seen);
    long long t = 0;
    for (int c : seen) t += node_cost(ch.at(c));
    return t;
}

static Extraction extract(EGraph& g, const std::vector<int>& roots, bool dag_search) {
    // greedy tree cost to a fixpoint; ties keep the oldest node (lowest serial)
    std::map<int, long long> cost;
    std::map<int, std::pair<Node, int>> best;   // node, serial
    const long long INF = (long long)4e18;
    auto cls_cost = [&](int c) {
        auto it = cost.find(g.find(c));
        return it == cost.end() ? INF : it->second;
    };
    for (bool changed = true; changed;) {
        changed = false;
        for (int c : g.classes()) {
            const EClass& C = g.cls(c);
            for (size_t i = 0; i < C.nodes.size(); ++i) {
                Node n = g.canon(C.nodes[i]);
                long long t = node_cost(n);
                if (!selection_leaf(n))
                    for (int k : n.kids) {
                        long long kc = cls_cost(k);
                        if (kc >= INF) {
                            t = INF;
                            break;
                        }
                        t += kc;
                    }
                if (t >= INF) continue;
                auto it = cost.find(c);
                if (it == cost.end() || t < it->second ||
                    (t == it->second && C.serial[i] < best[c].second)) {
                    if (it == cost.end() || t != it->second || !(best[c].first == n)) changed = true;
                    cost[c] = t;
                    best[c] = {n, C.serial[i]};
                }
            }
        }
    }
    Extraction x;
    for (auto& [c, b] : best) x.choice[c] = b.first;

    if (dag_search) {
        // exact incremental DAG-cost local search: switch a reachable class to
        // another node when the cost of the whole shared selection drops
        std::vector<int> rts;
        for (int r : roots) rts.push_back(g.find(r));
        long long cur = dag_cost(g, x.choice, rts);
        for (int pass = 0; pass < 8; ++pass) {
            bool improved = false;
            std::set<int> live;
            for (int r : rts) reach(g, x.choice, r, live);
            for (int c : std::vector<int>(live.begin(), live.end())) {
                const EClass& C = g.cls(c);
                Node keep = x.choice[c];
                for (const Node& n0 : C.nodes) {
                    Node n = g.canon(n0);
                    if (n == keep) continue;
                    bool ok = true;
                    if (!selection_leaf(n))
                        for (int k : n.kids) ok &= x.choice.count(g.find(k)) > 0;
                    if (!ok) continue;
                    x.choice[c] = n;
                    // reject cycles: c must not reach itself
                    bool cyc = false;
                    if (!selection_leaf(n)) {
                        std::set<int> sub;
                        std::function<void(int)> walk = [&](int q) {
                            q = g.find(q);
                            if (cyc || !sub.insert(q).second) return;
                            const Node& m = x.choice[q];
                            if (selection_leaf(m)) return;
                            for (int k : m.kids) {
                                if (g.find(k) == c) {
                                    cyc = true;
                                    return;
                                }
                                walk(k);
                            }
                        };
                        for (int k : n.kids) {
                            if (g.find(k) == c) cyc = true;
                            walk(k);
                        }
                    }
                    long long t = cyc ? INF : dag_cost(g, x.choice, rts);
                    if (t < cur) {
                        cur = t;
                        keep = n;
                        improved = true;
                    } else {
                        x.choice[c] = keep;
                    }
                }
                x.choice[c] = keep;
            }
            if (!improved) break;
        }
    }
    std::set<int> live;
    for (int r : roots) reach(g, x.choice, r, live);
    for (int c : live) {
        x.total += node_cost(x.choice[c]);
        if (x.choice[c].op == Op::Fma) x.fma++;
    }
    return x;
}

// ---- exact extraction: the DAG-cost problem as a 0/1 ILP ----
//
// The reference proves optimality with a branch and bound under a timeout
// (proj/src/extract.cpp:130-174, :202-241; greedy fallback when it times out).
// Here the problem restricted to the classes reachable from the roots is handed
// to a registered solver (acs_opt_set_solver; satopt.py registers HiGHS through
// scipy.optimize.milp): x_n in {0,1} per node, minimise sum cost(n) x_n subject
// to  sum_{n in root class} x_n >= 1  and, for every non-leaf node n and kid
// class k,  sum_{m in k} x_m >= x_n  (plus order variables when the class graph
// has a cycle).  The incumbent (greedy + DAG local search) is kept unless the
// ILP solution is proven optimal and strictly cheaper, so an equal-cost optimum
// leaves the emitted text unchanged and a timed-out solve changes nothing.
static acs_opt_solver g_solver = nullptr;

struct ExactResult {
    int status = -1;         // -1 not run, 0 proven optimal, 1 time limit (feasible), 2 failed
    double bound = 0;        // solver's lower bound on the optimum
    bool improved = false;
};

static ExactResult exact_refine(EGraph& g, const std::vector<int>& roots, Extraction& x, double time_s) {
    ExactResult er;
    if (!g_solver || time_s <= 0 || roots.empty()) return er;
    std::vector<int> cls;                       // reachable classes (over every node)
    std::map<int, int> idx;
    std::vector<int> stack;
    for (int r : roots) stack.push_back(g.find(r));
    while (!stack.empty()) {
        int c = g.find(stack.back());
        stack.pop_back();
        if (idx.count(c)) continue;
        idx[c] = (int)cls.size();
        cls.push_back(c);
        for (const Node& n0 : g.cls(c).nodes) {
            Node n = g.canon(n0);
            if (!selection_leaf(n))
                for (int k : n.kids) stack.push_back(g.find(k));
        }
    }
    std::vector<Node> nodes;
    std::vector<int> ncls, kptr{0}, kids;
    std::vector<long long> ncost;
    for (size_t ci = 0; ci < cls.size(); ++ci) {
        std::vector<Node> seen;
        for (const Node& n0 : g.cls(cls[ci]).nodes) {
            Node n = g.canon(n0);
            if (std::find(seen.begin(), seen.end(), n) != seen.end()) continue;
            seen.push_back(n);
            nodes.push_back(n);
            ncls.push_back((int)ci);
            ncost.push_back(node_cost(n));
            if (!selection_leaf(n)) {
                std::vector<int> ks;
                for (int k : n.kids) ks.push_back(idx.at(g.find(k)));
                std::sort(ks.begin(), ks.end());
                ks.erase(std::unique(ks.begin(), ks.end()), ks.end());
                kids.insert(kids.end(), ks.begin(), ks.end());
            }
            kptr.push_back((int)kids.size());
        }
    }
    std::vector<int> rts;
    for (int r : roots) rts.push_back(idx.at(g.find(r)));
    std::sort(rts.begin(), rts.end());
    rts.erase(std::unique(rts.begin(), rts.end()), rts.end());
    std::vector<int> chosen(nodes.size(), 0);
    er.status = g_solver((int)nodes.size(), (int)cls.size(), ncls.data(), ncost.data(), kptr.data(), kids.data(),
                         (int)rts.size(), rts.data(), time_s, chosen.data(), &er.bound);
    if (er.status != 0 && er.status != 1) return er;
    // one chosen node per class; a selection that is not a DAG (a solver bug) is rejected
    Extraction y;
    y.choice = x.choice;
    std::vector<int> pick(cls.size(), -1);
    for (size_t i = 0; i < nodes.size(); ++i)
        if (chosen[i] && pick[ncls[i]] < 0) pick[ncls[i]] = (int)i;
    std::vector<int> state(cls.size(), 0);
    bool ok = true;
    std::function<void(int)> dfs = [&](int ci) {
        if (!ok || state[ci] == 2) return;
        if (state[ci] == 1 || pick[ci] < 0) {
            ok = false;
            return;
        }
        state[ci] = 1;
        for (int q = kptr[pick[ci]]; q < kptr[pick[ci] + 1]; ++q) dfs(kids[q]);
        state[ci] = 2;
    };
    for (int r : rts) dfs(r);
    if (!ok) {
        er.status = 2;
        return er;
    }
    for (size_t ci = 0; ci < cls.size(); ++ci)
        if (pick[ci] >= 0) y.choice[cls[ci]] = nodes[pick[ci]];
    std::set<int> live;
    for (int r : roots) reach(g, y.choice, r, live);
    for (int c : live) {
        y.total += node_cost(y.choice[c]);
        if (y.choice[c].op == Op::Fma) y.fma++;
    }
    // only a PROVEN optimum replaces the incumbent: a time-limited solve could
    // otherwise make the emitted text depend on the machine's speed
    if (er.status == 0 && y.total < x.total) {
        x = std::move(y);
        er.improved = true;
    }
    return er;
}

// ============================================================================
// Value numbering of a region body into the e-graph

struct Sym {
    bool is_int = false;
    std::vector<long long> dims;
};

struct RootUse {
    const Stmt* st;
    int decl = -1;        // declarator index for Decl stmts
    int cls = -1;
};

struct PhiInfo {
    int cls;
    std::string var;
    const Stmt* after_if;   // the If statement that created it
};

struct Builder {
    EGraph& g;
    std::map<std::string, Sym> syms;
    std::map<std::string, int> env;      // scalar -> class
    struct Ev {
        int store_scope;                  // -1: kill marker
        std::vector<int> idx;
        int value;
    };
    std::map<std::string, std::vector<Ev>> events;
    std::vector<RootUse> roots;
    std::vector<PhiInfo> phis;
    std::map<const Stmt*, int> cond_cls;
    int scope_ctr = 0, scope = 0, loop_ctr = 0;

    // scalars a loop assigns (header and body) and array bases it stores to
    void scan_loop(const Stmt& s, std::set<std::string>& vars, std::set<std::string>& bases) {
        if (s.k == Stmt::Assign) {
            if (s.lhs->k == Expr::Var) vars.insert(s.lhs->text);
            else bases.insert(s.lhs->text);
        }
        if (s.k == Stmt::Decl)
            for (auto& d : s.decls)
                if (d.dims.empty()) vars.insert(d.name);
        for (const Stmt* c : {s.then_s.get(), s.else_s.get(), s.init.get(), s.step.get(), s.body.get()})
            if (c) scan_loop(*c, vars, bases);
        for (auto& c : s.stmts) scan_loop(*c, vars, bases);
    }

    explicit Builder(EGraph& gg) : g(gg) {}

    int leaf(Op op, const std::string& sym, bool is_int, int aux = 0, std::vector<int> kids = {}) {
        Node n;
        n.op = op;
        n.sym = sym;
        n.aux = aux;
        n.kids = std::move(kids);
        return g.add(n, is_int);
    }
    int cint(long long v) {
        Node n;
        n.op = Op::CInt;
        n.iv = v;
        return g.add(n, true);
    }
    int cflt(double v) {
        Node n;
        n.op = Op::CFlt;
        std::memcpy(&n.fbits, &v, 8);
        return g.add(n);
    }
    int op(Op o, std::vector<int> kids, const std::string& sym = "") {
        Node n;
        n.op = o;
        n.sym = sym;
        n.kids = std::move(kids);
        return g.add(n);
    }
    const Sym& sym(const std::string& n) {
        auto it = syms.find(n);
        if (it == syms.end()) throw SyntaxErr("use of undeclared name: " + n);
        return it->second;
    }
    bool may_alias(const std::vector<int>& a, const std::vector<int>& b) {
        if (a.size() != b.size()) return true;
        for (size_t i = 0; i < a.size(); ++i) {
            auto x = g.cval(a[i]), y = g.cval(b[i]);
            if (x && y && x->is_int && y->is_int && x->i != y->i) return false;
        }
        return true;
    }

    int value(const Expr& e) {
        switch (e.k) {
            case Expr::Int: return cint(e.iv);
            case Expr::Float: return cflt(e.fv);
            case Expr::Var: {
                const Sym& s = sym(e.text);
                if (!s.dims.empty()) throw SyntaxErr("array used as a scalar: " + e.text);
                auto it = env.find(e.text);
                if (it != env.end()) return it->second;
                return leaf(Op::Var, e.text, s.is_int);
            }
            case Expr::Ref: {
                const Sym& s = sym(e.text);
                if (s.dims.size() != e.kids.size()) throw SyntaxErr("wrong subscript count for " + e.text);
                std::vector<int> idx;
                for (auto& k : e.kids) {
                    int c = value(*k);
                    if (!g.is_int(c)) throw SyntaxErr("array index is not an integer");
                    idx.push_back(c);
                }
                int epoch = 0;
                const Ev* last = nullptr;
                for (auto& ev : events[e.text])
                    if (ev.store_scope < 0 || may_alias(ev.idx, idx)) {
                        epoch++;
                        last = &ev;
                    }
                if (last && last->store_scope == scope) {
                    bool same = last->idx.size() == idx.size();
                    for (size_t i = 0; same && i < idx.size(); ++i) same = g.find(last->idx[i]) == g.find(idx[i]);
                    if (same) return last->value;   // store -> load forwarding
                }
                Node n;
                n.op = Op::Load;
                n.sym = e.text;
                n.aux = epoch;
                n.kids = idx;
                return g.add(n, s.is_int);
            }
            case Expr::Un: {
                int a = value(*e.kids[0]);
                return op(e.op == "-" ? Op::Neg : Op::Not, {a});
            }
            case Expr::Bin: {
                int a = value(*e.kids[0]), b = value(*e.kids[1]);
                static const std::map<std::string, Op> m = {
                    {"+", Op::Add}, {"-", Op::Sub}, {"*", Op::Mul}, {"/", Op::Div}, {"%", Op::Mod}, {"<", Op::Lt},
                    {"<=", Op::Le}, {">", Op::Gt}, {">=", Op::Ge}, {"==", Op::Eq}, {"!=", Op::Ne}, {"&&", Op::And},
                    {"||", Op::Or}};
                return op(m.at(e.op), {a, b});
            }
            case Expr::Call: {
                std::vector<int> a;
                for (auto& k : e.kids) a.push_back(value(*k));
                return op(Op::Call, a, e.text);
            }
        }
        throw SyntaxErr("bad expression");
    }

    void assign(const std::string& var, int c) {
        const Sym& s = sym(var);
        if (s.is_int != g.is_int(c))
            throw Unsupported("implicit int/double conversion in an assignment to '" + var + "'");
        env[var] = c;
    }

    void stmt(const Stmt& s) {
        switch (s.k) {
            case Stmt::Assign: {
                if (s.lhs->k == Expr::Var) {
                    int c = value(*s.rhs);
                    assign(s.lhs->text, c);
                    roots.push_back({&s, -1, c});
                } else {
                    const Sym& sy = sym(s.lhs->text);
                    if (sy.dims.size() != s.lhs->kids.size()) throw SyntaxErr("wrong subscript count");
                    std::vector<int> idx;
                    for (auto& k : s.lhs->kids) idx.push_back(value(*k));
                    int c = value(*s.rhs);
                    if (sy.is_int != g.is_int(c)) throw Unsupported("implicit conversion in a store");
                    roots.push_back({&s, -1, c});
                    events[s.lhs->text].push_back({scope, idx, c});
                }
                break;
            }
            case Stmt::Decl:
                for (size_t i = 0; i < s.decls.size(); ++i) {
                    auto& d = s.decls[i];
                    syms[d.name] = {s.ty == "int", d.dims};
                    env.erase(d.name);
                    if (d.init && d.dims.empty()) {
                        int c = value(*d.init);
                        assign(d.name, c);
                        roots.push_back({&s, (int)i, c});
                    }
                }
                break;
            case Stmt::If: {
                int cc = value(*s.cond);
                cond_cls[&s] = cc;
                std::map<std::string, size_t> before;
                for (auto& [b, v] : events) before[b] = v.size();
                auto e0 = env;
                int saved = scope;
                scope = ++scope_ctr;
                stmt(*s.then_s);
                auto e1 = env;
                env = e0;
                scope = ++scope_ctr;
                if (s.else_s) stmt(*s.else_s);
                auto e2 = env;
                scope = saved;
                std::set<std::string> names;
                for (auto& [n, v] : e1) names.insert(n);
                for (auto& [n, v] : e2) names.insert(n);
                for (auto& n : names) {
                    const Sym& sy = sym(n);
                    auto get = [&](std::map<std::string, int>& m) {
                        auto it = m.find(n);
                        return it != m.end() ? it->second : leaf(Op::Var, n, sy.is_int);
                    };
                    int a = get(e1), b = get(e2);
                    if (g.find(a) == g.find(b)) {
                        env[n] = a;
                        continue;
                    }
                    int p = leaf(Op::Phi, n, sy.is_int, 0, {cc, a, b});
                    env[n] = p;
                    phis.push_back({p, n, &s});
                }
                for (auto& [b, v] : events) {
                    size_t was = before.count(b) ? before[b] : 0;
                    if (v.size() > was) v.push_back({-1, {}, -1});   // conditional stores kill reuse
                }
                break;
            }
            case Stmt::Block: {
                int saved = scope;
                scope = ++scope_ctr;
                for (auto& c : s.stmts) stmt(*c);
                scope = saved;
                break;
            }
            case Stmt::For: {
                // a sequential loop inside the region (gated SSA for-/exit-φ,
                // proj/src/ssa.cpp:487-549): every scalar the loop assigns is
                // an opaque for-φ inside the body and an exit-φ after it; a
                // base the loop stores to starts a new load epoch on entry
                // (later iterations see the stores) and on exit
                std::set<std::string> vars, bases;
                scan_loop(s, vars, bases);
                for (auto& bname : bases) events[bname].push_back({-1, {}, -1});
                const int id = ++loop_ctr;
                int saved = scope;
                scope = ++scope_ctr;
                for (auto& v : vars) env[v] = leaf(Op::Phi, v, sym(v).is_int, 2 * id);
                if (s.body) stmt(*s.body);
                scope = saved;
                for (auto& v : vars) {
                    int p = leaf(Op::Phi, v, sym(v).is_int, 2 * id + 1);
                    env[v] = p;
                    phis.push_back({p, v, &s});
                }
                for (auto& bname : bases) events[bname].push_back({-1, {}, -1});
                break;
            }
            case Stmt::Call:
            case Stmt::Empty: break;
        }
    }
};

// ============================================================================
// Codegen

static std::string fmt_double(double v) {
    char buf[64];
    for (int p = 1; p <= 17; ++p) {
        std::snprintf(buf, sizeof buf, "%.*g", p, v);
        if (std::strtod(buf, nullptr) == v) break;
    }
    std::string s = buf;
    if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
    return s;
}

struct Emitter {
    EGraph& g;
    Extraction& x;
    Builder& b;
    const std::string& src;
    bool bulk;
    // block tree: every statement list gets an id; a position is (block, slot)
    struct Pos {
        int block = 0, slot = 0;
    };
    std::map<const Stmt*, Pos> pos;          // statement -> position in its list
    std::map<int, int> block_parent;         // block -> parent block (-1 root)
    std::map<int, int> block_slot_in_parent; // block -> slot of the statement holding it
    std::map<int, std::vector<const Stmt*>> block_stmts;
    std::map<const Stmt*, int> then_block, else_block;
    std::set<const Stmt*> assigns_in;        // statements assigning scalars read by...
    int nblocks = 0;

    std::map<int, Pos> place;                // temp class -> placement
    std::map<int, std::string> atom_name;    // phi class -> materialised copy name
    std::set<int> temps;

    Emitter(EGraph& gg, Extraction& xx, Builder& bb, const std::string& s, bool bk)
        : g(gg), x(xx), b(bb), src(s), bulk(bk) {}

    int index_block(const Stmt& s, int parent, int slot_in_parent) {
        int id = nblocks++;
        block_parent[id] = parent;
        block_slot_in_parent[id] = slot_in_parent;
        std::vector<const Stmt*> list;
        if (s.k == Stmt::Block)
            for (auto& c : s.stmts) list.push_back(c.get());
        else
            list.push_back(&s);
        block_stmts[id] = list;
        for (int i = 0; i < (int)list.size(); ++i) {
            pos[list[i]] = {id, i};
            index_sub(*list[i], id, i);
        }
        return id;
    }
    void index_sub(const Stmt& s, int blk, int slot) {
        if (s.k == Stmt::If) {
            then_block[&s] = index_block(*s.then_s, blk, slot);
            if (s.else_s) else_block[&s] = index_block(*s.else_s, blk, slot);
        } else if (s.k == Stmt::Block) {
            // nested plain block: index its contents as a child block
            then_block[&s] = index_block(s, blk, slot);
        } else if (s.k == Stmt::For && s.body) {
            // sequential inner loop: its body is a child block (temps of
            // for-φ values stay inside it)
            then_block[&s] = index_block(*s.body, blk, slot);
        }
    }
    std::vector<int> chain(int blk) {   // block, parent, ..., root
        std::vector<int> c;
        for (int q = blk; q >= 0; q = block_parent[q]) c.push_back(q);
        return c;
    }
    // lowest common placement of two positions
    Pos lca(Pos a, Pos b2) {
        auto ca = chain(a.block), cb = chain(b2.block);
        std::set<int> sb(cb.begin(), cb.end());
        int common = -1;
        for (int q : ca)
            if (sb.count(q)) {
                common = q;
                break;
            }
        auto slot_in = [&](Pos p) {
            int q = p.block, s = p.slot;
            while (q != common) {
                s = block_slot_in_parent[q];
                q = block_parent[q];
            }
            return s;
        };
        return {common, std::min(slot_in(a), slot_in(b2))};
    }
    bool is_temp(int c) {
        c = g.find(c);
        const Node& n = x.choice.at(c);
        return !(n.op == Op::CInt || n.op == Op::CFlt || n.op == Op::Var || n.op == Op::Phi);
    }
    std::string atom(int c) {
        c = g.find(c);
        const Node& n = x.choice.at(c);
        switch (n.op) {
            case Op::CInt: return std::to_string(n.iv);
            case Op::CFlt: return fmt_double(n.fv());
            case Op::Var: return n.sym;
            case Op::Phi: {
                auto it = atom_name.find(c);
                return it != atom_name.end() ? it->second : n.sym;
            }
            default: return "_v" + std::to_string(c);
        }
    }
    std::string rhs_text(int c) {
        const Node& n = x.choice.at(g.find(c));
        switch (n.op) {
            case Op::Load: {
                std::string s = n.sym;
                for (int k : n.kids) s += "[" + atom(k) + "]";
                return s;
            }
            case Op::Neg: {
                std::string a = atom(n.kids[0]);
                return (a[0] == '-' ? "- " : "-") + a;   // never "--"
            }
            case Op::Not: return "!" + atom(n.kids[0]);
            case Op::Fma: return atom(n.kids[0]) + " + " + atom(n.kids[1]) + " * " + atom(n.kids[2]);
            case Op::Call: {
                std::string s = n.sym + "(";
                for (size_t i = 0; i < n.kids.size(); ++i) s += (i ? ", " : "") + atom(n.kids[i]);
                return s + ")";
            }
            default: {
                std::string r = atom(n.kids[1]);
                if (r[0] == '-' && (n.op == Op::Sub || n.op == Op::Add)) r = "(" + r + ")";   // a - (-1.0)
                return atom(n.kids[0]) + " " + binop_text(n.op) + " " + r;
            }
        }
    }

    // scalars a class's selected sub-DAG reads (for bulk-motion barriers)
    void reads(int c, std::set<std::string>& out, std::set<int>& seen) {
        c = g.find(c);
        if (!seen.insert(c).second) return;
        const Node& n = x.choice.at(c);
        if (n.op == Op::Var || n.op == Op::Phi) {
            out.insert(n.sym);
            return;
        }
        for (int k : n.kids) reads(k, out, seen);
    }
    static void assigned_scalars(const Stmt& s, std::set<std::string>& out) {
        if (s.k == Stmt::Assign && s.lhs->k == Expr::Var) out.insert(s.lhs->text);
        if (s.k == Stmt::Decl)
            for (auto& d : s.decls) out.insert(d.name);
        for (const Stmt* c : {s.then_s.get(), s.else_s.get(), s.body.get()})
            if (c) assigned_scalars(*c, out);
        for (auto& c : s.stmts) assigned_scalars(*c, out);
    }
    void stores(const Stmt& s, std::vector<std::pair<std::string, const Stmt*>>& out) {
        if (s.k == Stmt::Assign && s.lhs->k == Expr::Ref) out.push_back({s.lhs->text, &s});
        for (const Stmt* c : {s.then_s.get(), s.else_s.get(), s.body.get()})
            if (c) stores(*c, out);
        for (auto& c : s.stmts) stores(*c, out);
    }

    std::string emit(const Stmt& body) {
        index_block(body, -1, 0);
        // uses: root statements use their root class directly
        std::map<int, std::vector<Pos>> uses;
        for (auto& r : b.roots) uses[g.find(r.cls)].push_back(pos.at(r.st));
        // φ copies: a φ whose variable is assigned again after the if is read
        // through a copy made right after the if
        for (auto& p : b.phis) {
            const Stmt* ifs = p.after_if;
            Pos ip = pos.at(ifs);
            bool reassigned = false;
            // any later statement (in program order, same or enclosing lists) assigning the variable
            for (int q = ip.block, from = ip.slot + 1; q >= 0;) {
                auto& L = block_stmts[q];
                for (int i = from; i < (int)L.size(); ++i) {
                    std::set<std::string> a;
                    assigned_scalars(*L[i], a);
                    reassigned |= a.count(p.var) > 0;
                }
                from = block_slot_in_parent[q] + 1;
                q = block_parent[q];
            }
            if (reassigned) atom_name[g.find(p.cls)] = "_p" + std::to_string(g.find(p.cls));
        }
        // topological order of selected temps: users before their operands
        std::set<int> live;
        for (auto& r : b.roots) reach(g, x.choice, r.cls, live);
        std::vector<int> order;
        {
            std::map<int, int> indeg;
            for (int c : live) indeg[c];
            for (int c : live) {
                const Node& n = x.choice.at(c);
                if (selection_leaf(n)) continue;
                for (int k : n.kids) indeg[g.find(k)]++;
            }
            std::vector<int> q;
            for (auto& [c, d] : indeg)
                if (!d) q.push_back(c);
            while (!q.empty()) {
                int c = q.back();
                q.pop_back();
                order.push_back(c);
                const Node& n = x.choice.at(c);
                if (selection_leaf(n)) continue;
                for (int k : n.kids)
                    if (--indeg[g.find(k)] == 0) q.push_back(g.find(k));
            }
        }
        for (int c : order) {
            if (!is_temp(c)) continue;
            auto& u = uses[c];
            if (u.empty()) continue;
            Pos p = u[0];
            for (size_t i = 1; i < u.size(); ++i) p = lca(p, u[i]);
            place[c] = p;
            temps.insert(c);
            const Node& n = x.choice.at(c);
            for (int k : n.kids) uses[g.find(k)].push_back(p);
        }
        if (bulk) bulk_motion();
        std::ostringstream o;
        emit_list(0, 0, o, true);
        return o.str();
    }

    void bulk_motion() {
        // loads move up their own statement list past statements that do not
        // store to the base and do not assign a scalar their subscripts read
        std::vector<int> loads;
        for (int c : temps)
            if (x.choice.at(c).op == Op::Load) loads.push_back(c);
        for (int c : loads) {
            Pos p = place[c];
            const Node& n = x.choice.at(c);
            std::set<std::string> rd;
            std::set<int> seen;
            for (int k : n.kids) reads(k, rd, seen);
            auto& L = block_stmts[p.block];
            int s = p.slot;
            while (s > 0) {
                const Stmt* st = L[s - 1];
                std::set<std::string> a;
                assigned_scalars(*st, a);
                bool blocked = false;
                for (auto& v : rd) blocked |= a.count(v) > 0;
                std::vector<std::pair<std::string, const Stmt*>> sts;
                stores(*st, sts);
                for (auto& [base, ss] : sts) blocked |= base == n.sym;
                if (blocked) break;
                s--;
            }
            if (s == p.slot) continue;
            // the load's subscript temps must be available there too
            std::function<bool(int)> movable = [&](int q) {
                q = g.find(q);
                if (!temps.count(q)) return true;
                Pos qp = place[q];
                if (qp.block == p.block && qp.slot <= s) return true;
                if (qp.block != p.block) return false;
                for (int k : x.choice.at(q).kids)
                    if (!movable(k)) return false;
                return true;
            };
            bool ok = true;
            for (int k : n.kids) ok &= movable(k);
            if (!ok) continue;
            std::function<void(int)> hoist = [&](int q) {
                q = g.find(q);
                if (!temps.count(q)) return;
                if (place[q].block == p.block && place[q].slot > s) {
                    place[q].slot = s;
                    for (int k : x.choice.at(q).kids) hoist(k);
                }
            };
            place[c].slot = s;
            for (int k : n.kids) hoist(k);
        }
    }

    void emit_temps(int blk, int slot, std::ostringstream& o, const std::string& ind) {
        std::vector<int> here;
        for (auto& [c, p] : place)
            if (p.block == blk && p.slot == slot) here.push_back(c);
        // dependency order, the reference's bulk-block layout: integer
        // (subscript) temps first, then loads sorted by (base, subscript
        // text), then the arithmetic by class id — each step emits the
        // lowest-keyed temp whose operands are ready
        std::set<int> done;
        auto key = [&](int c) {
            const Node& n = x.choice.at(c);
            bool ld = n.op == Op::Load;
            return std::make_tuple(ld ? 1 : (g.is_int(c) ? 0 : 2), ld ? rhs_text(c) : std::string(), c);
        };
        std::sort(here.begin(), here.end(), [&](int a, int b2) { return key(a) < key(b2); });
        std::set<int> hs(here.begin(), here.end());
        while (done.size() < here.size()) {
            bool progress = false;
            for (int c : here) {
                if (done.count(c)) continue;
                bool ready = true;
                const Node& n = x.choice.at(c);
                for (int k : n.kids) {
                    int kk = g.find(k);
                    if (hs.count(kk) && !done.count(kk)) ready = false;
                }
                if (!ready) continue;
                o << ind << "_v" << c << " = " << rhs_text(c) << ";\n";
                done.insert(c);
                progress = true;
                break;
            }
            if (!progress) throw std::logic_error("cyclic temp placement");
        }
    }

    std::string verbatim(size_t b0, size_t e0) { return src.substr(b0, e0 - b0); }

    void emit_list(int blk, int depth, std::ostringstream& o, bool top) {
        std::string ind((depth + 1) * 4, ' ');
        auto& L = block_stmts[blk];
        // temps of this list are declared at its top (typed, like the
        // reference's telescoped declaration groups) and assigned at their slot
        std::vector<int> ints, dbls;
        for (auto& [c, p] : place)
            if (p.block == blk) (g.is_int(c) ? ints : dbls).push_back(c);
        for (auto* grp : {&ints, &dbls}) {
            if (grp->empty()) continue;
            o << ind << (grp == &ints ? "int " : "double ");
            for (size_t i = 0; i < grp->size(); ++i) o << (i ? ", " : "") << "_v" << (*grp)[i];
            o << ";\n";
        }
        for (int i = 0; i < (int)L.size(); ++i) {
            emit_temps(blk, i, o, ind);
            emit_stmt(*L[i], depth, o);
        }
        (void)top;
    }

    int root_of(const Stmt* s, int decl = -1) {
        for (auto& r : b.roots)
            if (r.st == s && r.decl == decl) return r.cls;
        return -1;
    }

    void emit_stmt(const Stmt& s, int depth, std::ostringstream& o) {
        std::string ind((depth + 1) * 4, ' ');
        for (auto& p : s.pragmas) o << p << "\n";
        switch (s.k) {
            case Stmt::Assign: {
                int c = root_of(&s);
                std::string lhs = verbatim(s.lhs->beg, s.lhs->end);
                o << ind << lhs << " = " << atom(c) << ";\n";
                break;
            }
            case Stmt::Decl: {
                o << ind << s.ty << " ";
                for (size_t i = 0; i < s.decls.size(); ++i) {
                    auto& d = s.decls[i];
                    o << (i ? ", " : "") << d.name;
                    for (long long dim : d.dims) o << "[" << dim << "]";
                    if (d.init) o << " = " << atom(root_of(&s, (int)i));
                }
                o << ";\n";
                break;
            }
            case Stmt::If: {
                o << ind << "if (" << verbatim(s.cond->beg, s.cond->end) << ") {\n";
                emit_list(then_block[&s], depth + 1, o, false);
                if (s.else_s) {
                    o << ind << "} else {\n";
                    emit_list(else_block[&s], depth + 1, o, false);
                }
                o << ind << "}\n";
                for (auto& p : b.phis)
                    if (p.after_if == &s && atom_name.count(g.find(p.cls)))
                        o << ind << (g.is_int(p.cls) ? "int " : "double ") << atom_name[g.find(p.cls)] << " = "
                          << p.var << ";\n";
                break;
            }
            case Stmt::Block:
                o << ind << "{\n";
                emit_list(then_block[&s], depth + 1, o, false);
                o << ind << "}\n";
                break;
            case Stmt::Call: o << ind << verbatim(s.beg, s.end) << "\n"; break;
            case Stmt::Empty: o << ind << ";\n"; break;
            case Stmt::For: {
                // header verbatim (init; cond; step), body re-emitted
                std::string head = verbatim(s.beg, s.body ? s.body->beg : s.end);
                while (!head.empty() && std::isspace((unsigned char)head.back())) head.pop_back();
                o << ind << head << " {\n";
                if (s.body) emit_list(then_block[&s], depth + 1, o, false);
                o << ind << "}\n";
                for (auto& p : b.phis)
                    if (p.after_if == &s && atom_name.count(g.find(p.cls)))
                        o << ind << (g.is_int(p.cls) ? "int " : "double ") << atom_name[g.find(p.cls)] << " = "
                          << p.var << ";\n";
                break;
            }
        }
    }
};

// ============================================================================
// count_static_loads (proj/src/pipeline.cpp:112-138)

static int count_loads(const Expr& e) {
    int n = e.k == Expr::Ref ? 1 : 0;
    for (auto& k : e.kids) n += count_loads(*k);
    return n;
}
static int count_static_loads(const Stmt& s) {
    int n = 0;
    if (s.k == Stmt::Assign) {
        if (s.lhs->k == Expr::Ref)
            for (auto& k : s.lhs->kids) n += count_loads(*k);
        n += count_loads(*s.rhs);
    }
    if (s.cond) n += count_loads(*s.cond);
    if (s.call) n += count_loads(*s.call);
    for (auto& d : s.decls)
        if (d.init) n += count_loads(*d.init);
    for (const Stmt* c : {s.then_s.get(), s.else_s.get(), s.init.get(), s.step.get(), s.body.get()})
        if (c) n += count_static_loads(*c);
    for (auto& c : s.stmts) n += count_static_loads(*c);
    return n;
}
static int count_stores(const Stmt& s) {
    int n = s.k == Stmt::Assign && s.lhs->k == Expr::Ref ? 1 : 0;
    for (const Stmt* c : {s.then_s.get(), s.else_s.get(), s.init.get(), s.step.get(), s.body.get()})
        if (c) n += count_stores(*c);
    for (auto& c : s.stmts) n += count_stores(*c);
    return n;
}

static void collect_decls(const Stmt& s, std::map<std::string, Sym>& syms) {
    if (s.k == Stmt::Decl)
        for (auto& d : s.decls) syms[d.name] = {s.ty == "int", d.dims};
    for (const Stmt* c : {s.then_s.get(), s.else_s.get(), s.init.get(), s.step.get(), s.body.get()})
        if (c) collect_decls(*c, syms);
    for (auto& c : s.stmts) collect_decls(*c, syms);
}

static std::string json_str(const std::string& s) {
    std::string o = "\"";
    for (char c : s) {
        if (c == '"' || c == '\\') o += '\\';
        if (c == '\n') {
            o += "\\n";
            continue;
        }
        o += c;
    }
    return o + "\"";
}

struct RegionMetrics {
    int region = 0;
    std::string function, stop = "disabled", method = "greedy+dag", error;
    double ssa_ms = 0, sat_ms = 0, extract_ms = 0, ilp_bound = -1;
    bool timed_out = false;
    long long before = 0, after = 0;
    int loads_before = 0, loads_after = 0, stores = 0, fma = 0;
    size_t nodes = 0;
};

std::string optimize(const std::string& src, const std::string& name, bool sat, bool bulk, const acs_opt_limits& lim,
                     std::string& json) {
    using Clock = std::chrono::steady_clock;
    auto ms = [](Clock::time_point t0) { return std::chrono::duration<double, std::milli>(Clock::now() - t0).count(); };
    Module m = Parser(lex(src)).module();
    std::vector<Region> regions;
    for (auto& f : m.funcs) {
        std::vector<std::string> lv;
        find_in(f, *f.body, lv, regions);
    }
    std::vector<RegionMetrics> mets;
    std::vector<std::pair<std::pair<size_t, size_t>, std::string>> splices;   // anchor body range -> text
    for (Region& r : regions) {
        RegionMetrics rm;
        rm.region = r.index;
        rm.function = r.fn->name;
        const Stmt& body = *r.anchor->body;
        rm.loads_before = rm.loads_after = count_static_loads(body);
        rm.stores = count_stores(body);
        try {
            auto t0 = Clock::now();
            EGraph g;
            Builder b(g);
            for (auto& gl : m.globals)
                for (auto& d : gl->decls) b.syms[d.name] = {gl->ty == "int", d.dims};
            for (auto& p : r.fn->params) b.syms[p.name] = {p.ty == "int", p.dims};
            collect_decls(*r.fn->body, b.syms);
            for (auto& v : r.loopvars) b.syms[v] = {true, {}};
            if (body.k == Stmt::Block)
                for (auto& c : body.stmts) b.stmt(*c);
            else
                b.stmt(body);
            rm.ssa_ms = ms(t0);
            std::vector<int> roots;
            for (auto& rt : b.roots) roots.push_back(rt.cls);
            rm.before = extract(g, roots, false).total;
            if (sat) {
                t0 = Clock::now();
                SatResult sr = saturate(g, lim.max_nodes, lim.max_time_s, lim.max_iters);
                rm.sat_ms = ms(t0);
                rm.stop = sr.stop;
                rm.nodes = sr.nodes;
            } else {
                rm.nodes = g.n_nodes();
            }
            t0 = Clock::now();
            Extraction x = extract(g, roots, lim.dag_search != 0);
            if (!lim.dag_search) rm.method = "greedy";
            ExactResult er = exact_refine(g, roots, x, lim.exact_time_s);
            if (er.status == 0) {
                rm.method = "ilp";                       // proven optimal (the reference's ExtractMethod::Ilp)
                rm.ilp_bound = er.bound;
            } else if (er.status == 1) {
                rm.timed_out = true;                     // the reference's greedy fallback on timeout
                rm.ilp_bound = er.bound;
            }
            rm.extract_ms = ms(t0);
            rm.after = x.total;
            rm.fma = x.fma;
            Emitter em(g, x, b, src, bulk);
            std::string inner = em.emit(body);
            // indentation of the anchor body braces
            size_t ls = src.rfind('\n', r.anchor->beg);
            std::string base_ind;
            for (size_t q = ls + 1; q < src.size() && (src[q] == ' ' || src[q] == '\t'); ++q) base_ind += src[q];
            std::string text;
            std::istringstream is(inner);
            std::string line;
            text = "{\n";
            while (std::getline(is, line)) text += (line.rfind("#", 0) == 0 ? "" : base_ind) + line + "\n";
            text += base_ind + "}";
            splices.push_back({{body.beg, body.end}, text});
        } catch (const std::exception& e) {
            rm.error = e.what();
        }
        mets.push_back(rm);
    }
    std::sort(splices.begin(), splices.end());
    std::string out;
    size_t at = 0;
    for (auto& [rg, text] : splices) {
        out += src.substr(at, rg.first - at);
        out += text;
        at = rg.second;
    }
    out += src.substr(at);
    // recount loads on the emitted text (count_static_loads on the re-parse)
    if (!splices.empty()) {
        Module m2 = Parser(lex(out)).module();
        std::vector<Region> r2;
        for (auto& f : m2.funcs) {
            std::vector<std::string> lv;
            find_in(f, *f.body, lv, r2);
        }
        if (r2.size() == regions.size())
            for (size_t i = 0; i < r2.size(); ++i)
                if (mets[i].error.empty()) mets[i].loads_after = count_static_loads(*r2[i].anchor->body);
    }
    std::ostringstream j;
    j << "{\n  \"schema\": \"satcc-metrics-v1\",\n  \"file\": " << json_str(name) << ",\n  \"variant\": "
      << json_str(sat && bulk ? "accsat" : sat ? "cse+sat" : bulk ? "cse+bulk" : "cse") << ",\n  \"regions\": [";
    for (size_t i = 0; i < mets.size(); ++i) {
        auto& r = mets[i];
        j << (i ? "," : "") << "\n    {\"region\": " << r.region << ", \"function\": " << json_str(r.function)
          << ", \"ssa_ms\": " << r.ssa_ms << ", \"sat_ms\": " << r.sat_ms << ", \"extract_ms\": " << r.extract_ms
          << ", \"nodes_final\": " << r.nodes << ", \"stop_reason\": " << json_str(r.stop)
          << ", \"objective_before\": " << r.before << ", \"objective_after\": " << r.after
          << ", \"static_loads_before\": " << r.loads_before << ", \"static_loads_after\": " << r.loads_after
          << ", \"static_stores\": " << r.stores << ", \"fma_count\": " << r.fma << ", \"method\": "
          << json_str(r.method) << ", \"timed_out\": " << (r.timed_out ? "true" : "false");
        if (r.ilp_bound >= 0) j << ", \"ilp_bound\": " << (long long)std::ceil(r.ilp_bound - 1e-6);
        j << ", \"error\": " << json_str(r.error) << "}";
    }
    j << "\n  ]\n}\n";
    json = j.str();
    return splices.empty() ? src : out;
}


// ============================================================================
// Interpreter + differential verification (satcc verify)
//
// The reference's executor semantics (proj/src/interp.cpp:24-270): scalars are
// 64-bit ints or doubles; int op int stays int with truncating / and %, /0 and
// %0 are evaluation errors; anything else is IEEE double; comparisons yield
// int 0/1; && || short-circuit; fma(a, b, c) = a + b*c with two roundings; the
// libm calls of known_call; assignments coerce to the target's type; every
// array access is bounds-checked; a statement budget of 50M ticks.
// diff_test (proj/src/oracle.cpp:12-81): per trial t (seed t + 1) a random
// environment — ints U[1, 8], doubles U[-10, 10] for every symbol and array
// element (mt19937_64) — runs the ORIGINAL and the OPTIMIZED region body;
// every scalar and array element of the original's post-state must agree
// within tol_rel * max(|a|, |b|) or 1e-12; NaN never passes; an error in
// either run is a failure.

struct EvalErr : std::runtime_error {
    explicit EvalErr(const std::string& m) : std::runtime_error(m) {}
};

struct Val {
    bool is_int = true;
    long long i = 0;
    double d = 0.0;
    double as_d() const { return is_int ? (double)i : d; }
    static Val I(long long v) { return {true, v, 0.0}; }
    static Val D(double v) { return {false, 0, v}; }
};

struct Arr {
    bool is_int = false;
    std::vector<long long> dims;
    std::vector<long long> iv;
    std::vector<double> dv;
    size_t size() const {
        size_t n = 1;
        for (long long d : dims) n *= (size_t)d;
        return n;
    }
};

struct Env {
    std::map<std::string, Val> sc;
    std::map<std::string, Arr> arr;
};

class Interp {
  public:
    explicit Interp(Env& e) : env_(e) {}
    long long ticks = 0;
    static constexpr long long kBudget = 50000000;

    Val eval(const Expr& e) {
        switch (e.k) {
            case Expr::Int: return Val::I(e.iv);
            case Expr::Float: return Val::D(e.fv);
            case Expr::Var: {
                auto it = env_.sc.find(e.text);
                if (it == env_.sc.end()) throw EvalErr("read of undefined variable: " + e.text);
                return it->second;
            }
            case Expr::Ref: {
                Arr& a = array(e.text);
                size_t at = flat(a, e);
                return a.is_int ? Val::I(a.iv[at]) : Val::D(a.dv[at]);
            }
            case Expr::Un: {
                Val v = eval(*e.kids[0]);
                if (e.op == "!") return Val::I(v.as_d() == 0.0 ? 1 : 0);
                return v.is_int ? Val::I(-v.i) : Val::D(-v.d);
            }
            case Expr::Bin: return bin(e);
            case Expr::Call: return call(e);
        }
        throw EvalErr("bad expression");
    }

    void exec(const Stmt& s) {
        if (++ticks > kBudget) throw EvalErr("evaluation budget exceeded");
        switch (s.k) {
            case Stmt::Empty: return;
            case Stmt::Block:
                for (auto& c : s.stmts) exec(*c);
                return;
            case Stmt::Decl:
                for (auto& d : s.decls) {
                    if (!d.dims.empty()) {
                        Arr a;
                        a.is_int = s.ty == "int";
                        a.dims = d.dims;
                        if (a.is_int) a.iv.assign(a.size(), 0);
                        else a.dv.assign(a.size(), 0.0);
                        env_.arr[d.name] = std::move(a);
                    } else {
                        Val v = d.init ? eval(*d.init) : (s.ty == "int" ? Val::I(0) : Val::D(0.0));
                        env_.sc[d.name] = coerce(v, s.ty == "int");
                    }
                }
                return;
            case Stmt::Assign: assign(*s.lhs, eval(*s.rhs)); return;
            case Stmt::If:
                if (eval(*s.cond).as_d() != 0.0) exec(*s.then_s);
                else if (s.else_s) exec(*s.else_s);
                return;
            case Stmt::For:
                if (s.init) exec(*s.init);
                while (!s.cond || eval(*s.cond).as_d() != 0.0) {
                    if (++ticks > kBudget) throw EvalErr("evaluation budget exceeded");
                    exec(*s.body);
                    if (s.step) exec(*s.step);
                }
                return;
            case Stmt::Call: (void)eval(*s.call); return;
        }
    }

  private:
    Env& env_;

    Arr& array(const std::string& n) {
        auto it = env_.arr.find(n);
        if (it == env_.arr.end()) throw EvalErr("read of undefined array: " + n);
        return it->second;
    }
    size_t flat(const Arr& a, const Expr& r) {
        if (r.kids.size() != a.dims.size()) throw EvalErr("rank mismatch on " + r.text);
        size_t at = 0;
        for (size_t p = 0; p < a.dims.size(); ++p) {
            Val v = eval(*r.kids[p]);
            if (!v.is_int) throw EvalErr("non-integer subscript of " + r.text);
            if (v.i < 0 || v.i >= a.dims[p]) throw EvalErr("index out of bounds on " + r.text);
            at = at * (size_t)a.dims[p] + (size_t)v.i;
        }
        return at;
    }
    static Val coerce(Val v, bool to_int) {
        if (to_int) return v.is_int ? v : Val::I((long long)v.d);
        return v.is_int ? Val::D((double)v.i) : v;
    }
    void assign(const Expr& lhs, Val v) {
        if (lhs.k == Expr::Var) {
            auto it = env_.sc.find(lhs.text);
            if (it == env_.sc.end()) env_.sc[lhs.text] = v;   // first write creates a temp
            else it->second = coerce(v, it->second.is_int);
            return;
        }
        if (lhs.k == Expr::Ref) {
            Arr& a = array(lhs.text);
            size_t at = flat(a, lhs);
            if (a.is_int) a.iv[at] = coerce(v, true).i;
            else a.dv[at] = coerce(v, false).d;
            return;
        }
        throw EvalErr("bad assignment target");
    }
    Val bin(const Expr& e) {
        const std::string& op = e.op;
        if (op == "&&") {
            if (eval(*e.kids[0]).as_d() == 0.0) return Val::I(0);
            return Val::I(eval(*e.kids[1]).as_d() != 0.0 ? 1 : 0);
        }
        if (op == "||") {
            if (eval(*e.kids[0]).as_d() != 0.0) return Val::I(1);
            return Val::I(eval(*e.kids[1]).as_d() != 0.0 ? 1 : 0);
        }
        Val a = eval(*e.kids[0]), b = eval(*e.kids[1]);
        if (a.is_int && b.is_int) {
            long long x = a.i, y = b.i;
            if (op == "+") return Val::I(x + y);
            if (op == "-") return Val::I(x - y);
            if (op == "*") return Val::I(x * y);
            if (op == "/") {
                if (y == 0) throw EvalErr("integer division by zero");
                return Val::I(x / y);
            }
            if (op == "%") {
                if (y == 0) throw EvalErr("integer modulo by zero");
                return Val::I(x % y);
            }
        } else if (op == "%") {
            throw EvalErr("'%' on a non-integer operand");
        }
        double x = a.as_d(), y = b.as_d();
        if (op == "<") return Val::I(x < y);
        if (op == "<=") return Val::I(x <= y);
        if (op == ">") return Val::I(x > y);
        if (op == ">=") return Val::I(x >= y);
        if (op == "==") return Val::I(x == y);
        if (op == "!=") return Val::I(x != y);
        volatile double r;   // one IEEE rounding per operation, no contraction
        if (op == "+") r = x + y;
        else if (op == "-") r = x - y;
        else if (op == "*") r = x * y;
        else if (op == "/") r = x / y;
        else throw EvalErr("unknown operator " + op);
        return Val::D(r);
    }
    Val call(const Expr& e) {
        std::vector<double> a;
        for (auto& k : e.kids) a.push_back(eval(*k).as_d());
        const std::string& n = e.text;
        auto need = [&](size_t c) {
            if (a.size() != c) throw EvalErr("wrong argument count for " + n);
        };
        if (n == "fma") {
            need(3);
            volatile double p = a[1] * a[2];
            volatile double r = a[0] + p;   // the interpreter's two-rounding fma
            return Val::D(r);
        }
        if (n == "sqrt") { need(1); return Val::D(std::sqrt(a[0])); }
        if (n == "fabs") { need(1); return Val::D(std::fabs(a[0])); }
        if (n == "sin") { need(1); return Val::D(std::sin(a[0])); }
        if (n == "cos") { need(1); return Val::D(std::cos(a[0])); }
        if (n == "exp") { need(1); return Val::D(std::exp(a[0])); }
        if (n == "log") { need(1); return Val::D(std::log(a[0])); }
        if (n == "floor") { need(1); return Val::D(std::floor(a[0])); }
        if (n == "ceil") { need(1); return Val::D(std::ceil(a[0])); }
        if (n == "pow") { need(2); return Val::D(std::pow(a[0], a[1])); }
        if (n == "fmin") { need(2); return Val::D(std::fmin(a[0], a[1])); }
        if (n == "fmax") { need(2); return Val::D(std::fmax(a[0], a[1])); }
        throw EvalErr("call to unknown function: " + n);
    }
};

static void region_symbols(const Module& m, const Region& r,
                           std::vector<std::pair<std::string, std::pair<bool, std::vector<long long>>>>& out) {
    std::set<std::string> seen;
    auto add = [&](const std::string& n, bool is_int, const std::vector<long long>& dims) {
        if (seen.insert(n).second) out.push_back({n, {is_int, dims}});
    };
    for (auto& gl : m.globals)
        for (auto& d : gl->decls) add(d.name, gl->ty == "int", d.dims);
    for (auto& p : r.fn->params) add(p.name, p.ty == "int", p.dims);
    std::map<std::string, Sym> locals;
    collect_decls(*r.fn->body, locals);
    for (auto& [n, sym] : locals) add(n, sym.is_int, sym.dims);
    for (auto& v : r.loopvars) add(v, true, {});
}

static Env random_env(const std::vector<std::pair<std::string, std::pair<bool, std::vector<long long>>>>& syms,
                      unsigned long long seed) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> ud(-10.0, 10.0);
    std::uniform_int_distribution<long long> ui(1, 8);
    Env e;
    for (auto& [n, t] : syms) {
        const bool is_int = t.first;
        if (t.second.empty()) {
            e.sc[n] = is_int ? Val::I(ui(rng)) : Val::D(ud(rng));
        } else {
            Arr a;
            a.is_int = is_int;
            a.dims = t.second;
            const size_t sz = a.size();
            if (is_int) {
                a.iv.resize(sz);
                for (auto& v : a.iv) v = ui(rng);
            } else {
                a.dv.resize(sz);
                for (auto& v : a.dv) v = ud(rng);
            }
            e.arr[n] = std::move(a);
        }
    }
    return e;
}

struct Failure {
    unsigned long long seed;
    std::string location;
    double got, want;
};

std::string verify(const std::string& src, const std::string& name, bool sat, bool bulk, const acs_opt_limits& lim,
                   int trials, double tol_rel, bool& all_ok) {
    std::string mjson;
    const std::string opt = optimize(src, name, sat, bulk, lim, mjson);
    Module m0 = Parser(lex(src)).module();
    Module m1 = Parser(lex(opt)).module();
    std::vector<Region> r0, r1;
    for (auto& f : m0.funcs) {
        std::vector<std::string> lv;
        find_in(f, *f.body, lv, r0);
    }
    for (auto& f : m1.funcs) {
        std::vector<std::string> lv;
        find_in(f, *f.body, lv, r1);
    }
    if (r0.size() != r1.size()) throw std::logic_error("optimized output lost a region");
    all_ok = true;
    std::ostringstream j;
    j << "{\"file\": " << json_str(name) << ", \"variant\": "
      << json_str(sat && bulk ? "accsat" : sat ? "cse+sat" : bulk ? "cse+bulk" : "cse") << ", \"regions\": [";
    for (size_t k = 0; k < r0.size(); ++k) {
        std::vector<std::pair<std::string, std::pair<bool, std::vector<long long>>>> syms;
        region_symbols(m0, r0[k], syms);
        double max_rel = 0.0, max_abs = 0.0;
        std::vector<Failure> fails;
        long long n_fail = 0;
        for (int t = 0; t < trials; ++t) {
            const unsigned long long seed = (unsigned long long)t + 1;
            Env base = random_env(syms, seed);
            Env want = base, got = base;
            std::string err;
            try {
                Interp(want).exec(*r0[k].anchor->body);
                Interp(got).exec(*r1[k].anchor->body);
            } catch (const std::exception& e) {
                err = e.what();
            }
            if (!err.empty()) {
                ++n_fail;
                if (fails.size() < 10) fails.push_back({seed, "error: " + err, 0.0, 0.0});
                continue;
            }
            auto cmp = [&](const std::string& loc, double w, double g) {
                const double ae = std::fabs(g - w), mag = std::max(std::fabs(g), std::fabs(w));
                const double re = mag > 0.0 ? ae / mag : 0.0;
                if (ae == ae) max_abs = std::max(max_abs, ae);
                if (re == re) max_rel = std::max(max_rel, re);
                if (!(ae <= tol_rel * mag || ae <= 1e-12)) {
                    ++n_fail;
                    if (fails.size() < 10) fails.push_back({seed, loc, g, w});
                }
            };
            for (auto& [n, v] : want.sc) {
                auto it = got.sc.find(n);
                if (it == got.sc.end()) {
                    ++n_fail;
                    if (fails.size() < 10) fails.push_back({seed, n + " (missing)", 0.0, v.as_d()});
                } else {
                    cmp(n, v.as_d(), it->second.as_d());
                }
            }
            for (auto& [n, a] : want.arr) {
                const Arr& b = got.arr[n];
                for (size_t i = 0; i < a.size(); ++i)
                    cmp(n + "[" + std::to_string(i) + "]", a.is_int ? (double)a.iv[i] : a.dv[i],
                        b.is_int ? (double)b.iv[i] : b.dv[i]);
            }
        }
        const bool ok = n_fail == 0;
        all_ok = all_ok && ok;
        j << (k ? ", " : "") << "{\"region\": " << k << ", \"function\": " << json_str(r0[k].fn->name)
          << ", \"n_trials\": " << trials << ", \"max_rel_err\": " << max_rel << ", \"max_abs_err\": " << max_abs
          << ", \"n_failures\": " << n_fail << ", \"failures\": [";
        for (size_t f = 0; f < fails.size(); ++f)
            j << (f ? ", " : "") << "{\"seed\": " << fails[f].seed << ", \"location\": " << json_str(fails[f].location)
              << ", \"got\": " << fails[f].got << ", \"want\": " << fails[f].want << "}";
        j << "], \"ok\": " << (ok ? "true" : "false") << "}";
    }
    j << "]}";
    return j.str();
}

}  // namespace acsopt

extern "C" {

int acs_opt_optimize(const char* source, const char* name, const char* variant, const acs_opt_limits* limits,
                     char** text_out, char** json_out) {
    acs_opt_limits lim{10000, 10.0, 10, 1, 0.0};
    if (limits) lim = *limits;
    std::string v = variant ? variant : "accsat";
    bool sat = v == "accsat" || v == "cse+sat";
    bool bulk = v == "accsat" || v == "cse+bulk";
    auto dup = [](const std::string& s) {
        char* p = static_cast<char*>(std::malloc(s.size() + 1));
        std::memcpy(p, s.c_str(), s.size() + 1);
        return p;
    };
    try {
        if (v != "accsat" && v != "cse+sat" && v != "cse+bulk" && v != "cse")
            throw std::invalid_argument("unknown variant: " + v + " (expected cse, cse+sat, cse+bulk, or accsat)");
        std::string json;
        std::string text = acsopt::optimize(source ? source : "", name ? name : "<input>", sat, bulk, lim, json);
        *text_out = dup(text);
        *json_out = dup(json);
        return 0;
    } catch (const std::exception& e) {
        *text_out = dup("");
        *json_out = dup(std::string("{\"error\": ") + acsopt::json_str(e.what()) + "}");
        return 1;
    }
}

int acs_opt_verify(const char* source, const char* name, const char* variant, const acs_opt_limits* limits, int trials,
                   double tol_rel, char** json_out) {
    acs_opt_limits lim{10000, 10.0, 10, 1, 0.0};
    if (limits) lim = *limits;
    std::string v = variant ? variant : "accsat";
    auto dup = [](const std::string& s) {
        char* p = static_cast<char*>(std::malloc(s.size() + 1));
        std::memcpy(p, s.c_str(), s.size() + 1);
        return p;
    };
    try {
        if (v != "accsat" && v != "cse+sat" && v != "cse+bulk" && v != "cse")
            throw std::invalid_argument("unknown variant: " + v + " (expected cse, cse+sat, cse+bulk, or accsat)");
        bool ok = true;
        std::string json = acsopt::verify(source ? source : "", name ? name : "<input>", v == "accsat" || v == "cse+sat",
                                          v == "accsat" || v == "cse+bulk", lim, trials, tol_rel, ok);
        *json_out = dup(json);
        return ok ? 0 : 1;
    } catch (const std::exception& e) {
        *json_out = dup(std::string("{\"error\": ") + acsopt::json_str(e.what()) + "}");
        return 2;
    }
}

void acs_opt_free(char* p) { std::free(p); }

void acs_opt_set_solver(acs_opt_solver fn) { acsopt::g_solver = fn; }

}  // extern "C"
