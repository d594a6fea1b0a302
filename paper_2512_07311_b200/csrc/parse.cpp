// parse.cpp -- QASM-subset front end (§3.2 line 34: "circuits are initially
// constructed from Google's QASM-format files"; dialect SPEC.md S:84-86, reading V5).
//
// Two phases: a tokenizer that records 1-based line/column of every token, then a
// statement parser over the token vector.  Moment rule: `barrier` ends the
// current moment; otherwise a gate touching a qubit already used in the current moment
// opens a new one.  Errors carry the offending token's position.
#include <cctype>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "internal.h"

namespace rcs {

void set_error(rcs_error* err, int code, const char* fmt, ...) {
    if (!err) return;
    err->code = code;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(err->msg, sizeof err->msg, fmt, ap);
    va_end(ap);
}

namespace {

enum TokKind { T_IDENT, T_NUM, T_STR, T_SYM, T_END };

struct Tok {
    TokKind kind;
    std::string text;
    int line, col;
};

bool tokenize(const char* s, size_t len, std::vector<Tok>& toks, rcs_error* err) {
    int line = 1, col = 1;
    size_t i = 0;
    auto adv = [&](size_t k) {
        for (size_t j = 0; j < k && i < len; j++, i++) {
            if (s[i] == '\n') { line++; col = 1; } else col++;
        }
    };
    while (i < len) {
        char c = s[i];
        if (std::isspace((unsigned char)c)) { adv(1); continue; }
        if (c == '/' && i + 1 < len && s[i + 1] == '/') {
            while (i < len && s[i] != '\n') adv(1);
            continue;
        }
        Tok t{T_SYM, "", line, col};
        if (std::isalpha((unsigned char)c) || c == '_') {
            size_t j = i;
            while (j < len && (std::isalnum((unsigned char)s[j]) || s[j] == '_')) j++;
            t.kind = T_IDENT;
            t.text.assign(s + i, j - i);
            adv(j - i);
        } else if (std::isdigit((unsigned char)c) || c == '.') {
            size_t j = i;
            while (j < len) {
                char d = s[j];
                bool ok = std::isdigit((unsigned char)d) || d == '.' || d == 'e' || d == 'E';
                if (!ok && (d == '+' || d == '-') && j > i && (s[j - 1] == 'e' || s[j - 1] == 'E')) ok = true;
                if (!ok) break;
                j++;
            }
            t.kind = T_NUM;
            t.text.assign(s + i, j - i);
            adv(j - i);
        } else if (c == '"') {
            size_t j = i + 1;
            while (j < len && s[j] != '"' && s[j] != '\n') j++;
            if (j >= len || s[j] != '"') {
                set_error(err, RCS_ERR_PARSE, "unterminated string");
                err->line = line; err->col = col;
                return false;
            }
            t.kind = T_STR;
            t.text.assign(s + i + 1, j - i - 1);
            adv(j + 1 - i);
        } else if (c == '-' && i + 1 < len && s[i + 1] == '>') {
            t.text = "->";
            adv(2);
        } else if (std::strchr(";,()[]+-*/{}", c)) {
            t.text.assign(1, c);
            adv(1);
        } else {
            set_error(err, RCS_ERR_PARSE, "unexpected character '%c'", c);
            err->line = line; err->col = col;
            return false;
        }
        toks.push_back(t);
    }
    toks.push_back(Tok{T_END, "", line, col});
    return true;
}

struct Parser {
    std::vector<Tok> toks;
    size_t p = 0;
    rcs_error* err;
    bool failed = false;

    const Tok& cur() const { return toks[p]; }
    bool is_sym(const char* s) const { return cur().kind == T_SYM && cur().text == s; }

    bool fail(int code, const Tok& at, const char* msg) {
        if (!failed) {
            failed = true;
            set_error(err, code, "%s", msg);
            if (err) { err->line = at.line; err->col = at.col; }
        }
        return false;
    }
    bool expect(const char* s) {
        if (!is_sym(s)) {
            char m[64];
            std::snprintf(m, sizeof m, "expected '%s'", s);
            return fail(RCS_ERR_PARSE, cur(), m);
        }
        p++;
        return true;
    }
    bool ident(std::string& out) {
        if (cur().kind != T_IDENT) return fail(RCS_ERR_PARSE, cur(), "expected identifier");
        out = cur().text;
        p++;
        return true;
    }
    bool integer(long& v) {
        const Tok& t = cur();
        if (t.kind != T_NUM || t.text.find_first_not_of("0123456789") != std::string::npos || t.text.size() > 9)
            return fail(RCS_ERR_PARSE, t, "expected integer");
        v = std::strtol(t.text.c_str(), nullptr, 10);
        p++;
        return true;
    }
    // expr := term {(+|-) term}; term := factor {(*|/) factor}; factor := (+|-) factor | num | pi | (expr)
    bool expr(double& v) {
        if (!term(v)) return false;
        while (is_sym("+") || is_sym("-")) {
            bool plus = is_sym("+");
            p++;
            double r;
            if (!term(r)) return false;
            v = plus ? v + r : v - r;
        }
        return true;
    }
    bool term(double& v) {
        if (!factor(v)) return false;
        while (is_sym("*") || is_sym("/")) {
            bool mul = is_sym("*");
            p++;
            double r;
            if (!factor(r)) return false;
            v = mul ? v * r : v / r;
        }
        return true;
    }
    bool factor(double& v) {
        const Tok& t = cur();
        if (is_sym("-")) { p++; if (!factor(v)) return false; v = -v; return true; }
        if (is_sym("+")) { p++; return factor(v); }
        if (is_sym("(")) { p++; if (!expr(v)) return false; return expect(")"); }
        if (t.kind == T_NUM) {
            char* end = nullptr;
            v = std::strtod(t.text.c_str(), &end);
            if (end == t.text.c_str() || *end) return fail(RCS_ERR_PARSE, t, "bad number");
            p++;
            return true;
        }
        if (t.kind == T_IDENT && t.text == "pi") { v = 3.141592653589793238462643383279502884; p++; return true; }
        return fail(RCS_ERR_PARSE, t, "expected expression");
    }
};

struct GateSpec { const char* name; int kind, n_params, n_qubits; };
const GateSpec kGates[] = {
    {"x_1_2", RCS_GATE_SX, 0, 1}, {"sx", RCS_GATE_SX, 0, 1},
    {"y_1_2", RCS_GATE_SY, 0, 1}, {"sy", RCS_GATE_SY, 0, 1},
    {"hz_1_2", RCS_GATE_SW, 0, 1}, {"sw", RCS_GATE_SW, 0, 1},
    {"rz", RCS_GATE_RZ, 1, 1},     {"fsim", RCS_GATE_FSIM, 2, 2},
};

}  // namespace

rcs_status parse_qasm(const char* text, size_t len, Circuit& out, rcs_error* err) {
    rcs_error local{};
    if (!err) err = &local;
    Parser P;
    P.err = err;
    if (!tokenize(text, len, P.toks, err)) return (rcs_status)err->code;

    Circuit C;
    std::string qreg;
    int n = -1;
    std::vector<char> used;
    bool moment_open = false;

    while (P.cur().kind != T_END) {
        const Tok head = P.cur();
        std::string kw;
        if (!P.ident(kw)) break;
        if (kw == "OPENQASM") {
            if (P.cur().kind == T_NUM) P.p++;
            if (!P.expect(";")) break;
            continue;
        }
        if (kw == "include") {
            if (P.cur().kind != T_STR) { P.fail(RCS_ERR_PARSE, P.cur(), "expected string"); break; }
            P.p++;
            if (!P.expect(";")) break;
            continue;
        }
        if (kw == "qreg" || kw == "creg") {
            std::string name;
            long sz;
            if (kw == "qreg" && n >= 0) { P.fail(RCS_ERR_PARSE, head, "only one qreg allowed"); break; }
            if (!P.ident(name) || !P.expect("[") || !P.integer(sz) || !P.expect("]") || !P.expect(";")) break;
            if (kw == "qreg") {
                if (sz < 1 || sz > 63) { P.fail(RCS_ERR_PARSE, head, "qreg size must be in [1, 63]"); break; }
                n = (int)sz;
                qreg = name;
                used.assign(n, 0);
            }
            continue;
        }
        if (n < 0) { P.fail(RCS_ERR_PARSE, head, "statement before qreg declaration"); break; }
        if (kw == "barrier") {
            while (P.cur().kind != T_END && !P.is_sym(";")) P.p++;
            if (!P.expect(";")) break;
            if (moment_open) {
                C.n_moments++;
                moment_open = false;
                std::fill(used.begin(), used.end(), 0);
            }
            continue;
        }
        auto qarg = [&](long& q) -> bool {
            std::string r;
            const Tok at = P.cur();
            if (!P.ident(r)) return false;
            if (r != qreg) return P.fail(RCS_ERR_PARSE, at, "unknown quantum register");
            if (!P.expect("[")) return false;
            const Tok it = P.cur();
            if (!P.integer(q) || !P.expect("]")) return false;
            if (q >= n) return P.fail(RCS_ERR_QUBIT_RANGE, it, "qubit index out of declared range");
            return true;
        };
        if (kw == "measure") {
            long q, ci;
            std::string cr;
            if (!qarg(q) || !P.expect("->") || !P.ident(cr) || !P.expect("[") || !P.integer(ci) ||
                !P.expect("]") || !P.expect(";"))
                break;
            C.n_measure++;
            continue;
        }
        const GateSpec* spec = nullptr;
        for (const auto& gs : kGates)
            if (kw == gs.name) spec = &gs;
        if (!spec) { P.fail(RCS_ERR_UNKNOWN_GATE, head, "unknown gate"); break; }
        std::vector<double> params;
        if (P.is_sym("(")) {
            P.p++;
            for (;;) {
                double v;
                if (!P.expr(v)) break;
                params.push_back(v);
                if (P.is_sym(",")) { P.p++; continue; }
                P.expect(")");
                break;
            }
            if (P.failed) break;
        }
        std::vector<long> qs;
        for (;;) {
            long q;
            if (!qarg(q)) break;
            qs.push_back(q);
            if (P.is_sym(",")) { P.p++; continue; }
            break;
        }
        if (P.failed) break;
        if (!P.expect(";")) break;
        if ((int)params.size() != spec->n_params || (int)qs.size() != spec->n_qubits ||
            (qs.size() == 2 && qs[0] == qs[1])) {
            P.fail(RCS_ERR_ARITY, head, "gate arity mismatch");
            break;
        }
        bool finite = true;
        for (double v : params) finite = finite && std::isfinite(v);
        if (!finite) { P.fail(RCS_ERR_PARSE, head, "non-finite angle"); break; }
        bool clash = false;
        for (long q : qs) clash = clash || used[q];
        if (clash) {
            C.n_moments++;
            std::fill(used.begin(), used.end(), 0);
        }
        for (long q : qs) used[q] = 1;
        moment_open = true;
        Gate g;
        g.kind = spec->kind;
        g.q0 = (int)qs[0];
        g.q1 = qs.size() > 1 ? (int)qs[1] : -1;
        g.theta = spec->kind == RCS_GATE_FSIM ? params[0] : 0.0;
        g.phi = spec->kind == RCS_GATE_FSIM ? params[1] : (spec->kind == RCS_GATE_RZ ? params[0] : 0.0);
        g.moment = C.n_moments;
        C.gates.push_back(g);
    }
    if (!P.failed && n < 0) P.fail(RCS_ERR_PARSE, P.cur(), "missing qreg declaration");
    if (P.failed) return (rcs_status)err->code;
    if (moment_open) C.n_moments++;
    C.n = n;
    out = std::move(C);
    return RCS_OK;
}

}  // namespace rcs
