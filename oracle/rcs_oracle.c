/*
 * rcs_oracle.c -- plain, slow, obviously-correct fp64 CPU oracle for the RCS hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load or execute anything under oracle/.
 * The product (paper_2512_07311_b200/) never links, imports or calls this file,
 * and this file shares no code with it (separate parser, separate matrices,
 * separate RNG implementation).
 *
 * What it computes: the paper's stage-1 result
 * "the complete quantum state from the circuit definition" (§3.2 line 36),
 * the stage-3 measurement shots (§3.2 line 38) and the stage-4 linear XEB
 * score (§3.2 line 39, §5.1 line 82).  The paper gives no algorithm, so the
 * oracle is the plain definition:
 *
 *   O1  parse QASM (dialect SPEC.md S:84-86)                       -> orc_parse
 *   O2  gate matrices (readings V2-V4)      -> orc_gate_matrix
 *   O3  psi = e_0 in C^(2^n), complex128 -> orc_build_state
 *   O4  every gate in source order, no fusion
 *                                                                   -> orc_apply_gate
 *   O5  norm                                        -> orc_total_prob
 *   O6  T = sum_x |psi_x|^2, sequential fp64 in logical order (= C(2^n-1))
 *   O7  u_s = (SplitMix64 output s+1 of shot_seed) >> 11 * 2^-53 (reading V12)
 *                                                                   -> orc_uniforms
 *   O8  x_s = min{x : C(x) > u_s*T}, C the inclusive CDF in logical order;
 *       if none, the last x with p>0 (reading V13)    -> orc_sample
 *   O9  F = 2^n * mean_s p(x_s) - 1, sigma = 2^n * stdev(p, ddof=1)/sqrt(S);
 *       F* = 2^n * sum_x p^2 - 1 (reading V14) -> orc_xeb, orc_fstar
 *
 * Conventions: amplitude index i has qubit q as bit q (qubit 0 = LSB,
 * SPEC S:111); a 2-qubit gate on (q0, q1) uses basis index b_q0 + 2*b_q1.
 * State arrays are interleaved (re, im) doubles, i.e. numpy complex128.
 *
 * Parity pins live in tests/test_oracle_*.py (dense 2^n x 2^n unitary products,
 * closed forms, brute-force inverse CDF, statistical XEB checks).
 */
#include <ctype.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_PI 3.141592653589793238462643383279502884

enum { ORC_OK = 0, ORC_ERR_PARSE = 1, ORC_ERR_UNKNOWN_GATE = 2, ORC_ERR_QUBIT_RANGE = 3,
       ORC_ERR_ARITY = 4, ORC_ERR_MEMORY = 5, ORC_ERR_NORM = 6, ORC_ERR_SIZE = 7, ORC_ERR_ARG = 8 };

enum { ORC_SX = 0, ORC_SY = 1, ORC_SW = 2, ORC_RZ = 3, ORC_FSIM = 4 };

typedef struct {
    int kind, q0, q1, moment;
    double theta, phi;
} orc_gate;

typedef struct {
    int n_qubits;
    int n_gates, cap;
    int n_moments;
    int n_measure;
    orc_gate *gates;
} orc_circuit;

/* ------------------------------------------------------------------------- */
/* O1: QASM parser (dialect S:84-86)                            */
/* ------------------------------------------------------------------------- */

typedef struct {
    const char *s;
    long len, pos;
    int line, col;          /* position of pos */
    int tline, tcol;        /* position of the current token */
    int err;
    char msg[256];
} lexer;

static void lx_skip(lexer *L) {
    for (;;) {
        while (L->pos < L->len && isspace((unsigned char)L->s[L->pos])) {
            if (L->s[L->pos] == '\n') { L->line++; L->col = 1; } else L->col++;
            L->pos++;
        }
        if (L->pos + 1 < L->len && L->s[L->pos] == '/' && L->s[L->pos + 1] == '/') {
            while (L->pos < L->len && L->s[L->pos] != '\n') { L->pos++; L->col++; }
            continue;
        }
        break;
    }
    L->tline = L->line;
    L->tcol = L->col;
}

static int lx_peek(lexer *L) {
    lx_skip(L);
    return L->pos < L->len ? (unsigned char)L->s[L->pos] : -1;
}

static void lx_adv(lexer *L, long k) {
    while (k-- > 0 && L->pos < L->len) { L->pos++; L->col++; }
}

static int set_err(lexer *L, int code, const char *m) {
    if (!L->err) {
        L->err = code;
        snprintf(L->msg, sizeof L->msg, "%s", m);
    }
    return code;
}

static int lx_expect(lexer *L, char c) {
    if (lx_peek(L) != c) {
        char m[64];
        snprintf(m, sizeof m, "expected '%c'", c);
        return set_err(L, ORC_ERR_PARSE, m);
    }
    lx_adv(L, 1);
    return 0;
}

static int lx_ident(lexer *L, char *out, int cap) {
    int c = lx_peek(L);
    if (!(isalpha(c) || c == '_')) return set_err(L, ORC_ERR_PARSE, "expected identifier");
    int k = 0;
    while (L->pos < L->len && (isalnum((unsigned char)L->s[L->pos]) || L->s[L->pos] == '_')) {
        if (k < cap - 1) out[k++] = L->s[L->pos];
        lx_adv(L, 1);
    }
    out[k] = 0;
    return 0;
}

static int lx_uint(lexer *L, long *v) {
    int c = lx_peek(L);
    if (!isdigit(c)) return set_err(L, ORC_ERR_PARSE, "expected integer");
    long x = 0;
    while (L->pos < L->len && isdigit((unsigned char)L->s[L->pos])) {
        x = x * 10 + (L->s[L->pos] - '0');
        if (x > 1000000000L) return set_err(L, ORC_ERR_PARSE, "integer too large");
        lx_adv(L, 1);
    }
    *v = x;
    return 0;
}

/* expr := term (('+'|'-') term)* ; term := factor (('*'|'/') factor)* ;
   factor := ('-'|'+') factor | number | 'pi' | '(' expr ')'                     */
static double p_expr(lexer *L);

static double p_factor(lexer *L) {
    int c = lx_peek(L);
    if (c == '-') { lx_adv(L, 1); return -p_factor(L); }
    if (c == '+') { lx_adv(L, 1); return p_factor(L); }
    if (c == '(') {
        lx_adv(L, 1);
        double v = p_expr(L);
        lx_expect(L, ')');
        return v;
    }
    if (isdigit(c) || c == '.') {
        char buf[128];
        int k = 0;
        while (L->pos < L->len) {
            char ch = L->s[L->pos];
            int ok = isdigit((unsigned char)ch) || ch == '.' || ch == 'e' || ch == 'E';
            if (!ok && (ch == '-' || ch == '+') && k > 0 && (buf[k - 1] == 'e' || buf[k - 1] == 'E'))
                ok = 1;
            if (!ok) break;
            if (k < 127) buf[k++] = ch;
            lx_adv(L, 1);
        }
        buf[k] = 0;
        char *end = NULL;
        double v = strtod(buf, &end);
        if (end == buf || *end) { set_err(L, ORC_ERR_PARSE, "bad number"); return 0; }
        return v;
    }
    if (isalpha(c)) {
        char id[64];
        lx_ident(L, id, sizeof id);
        if (strcmp(id, "pi") == 0) return ORC_PI;
        set_err(L, ORC_ERR_PARSE, "unknown symbol in expression");
        return 0;
    }
    set_err(L, ORC_ERR_PARSE, "expected expression");
    return 0;
}

static double p_term(lexer *L) {
    double v = p_factor(L);
    for (;;) {
        int c = lx_peek(L);
        if (c == '*') { lx_adv(L, 1); v = v * p_factor(L); }
        else if (c == '/') { lx_adv(L, 1); v = v / p_factor(L); }
        else return v;
    }
}

static double p_expr(lexer *L) {
    double v = p_term(L);
    for (;;) {
        int c = lx_peek(L);
        if (c == '+') { lx_adv(L, 1); v = v + p_term(L); }
        else if (c == '-') { lx_adv(L, 1); v = v - p_term(L); }
        else return v;
    }
}

static int push_gate(orc_circuit *C, orc_gate g) {
    if (C->n_gates == C->cap) {
        int nc = C->cap ? 2 * C->cap : 256;
        orc_gate *ng = (orc_gate *)realloc(C->gates, (size_t)nc * sizeof(orc_gate));
        if (!ng) return ORC_ERR_MEMORY;
        C->gates = ng;
        C->cap = nc;
    }
    C->gates[C->n_gates++] = g;
    return 0;
}

/* qarg := IDENT '[' uint ']' ; returns index or -1 on error */
static long p_qarg(lexer *L, const char *qreg, int n, int *line, int *col) {
    char id[64];
    lx_skip(L);
    *line = L->tline;
    *col = L->tcol;
    if (lx_ident(L, id, sizeof id)) return -1;
    if (strcmp(id, qreg) != 0) { set_err(L, ORC_ERR_PARSE, "unknown quantum register"); return -1; }
    if (lx_expect(L, '[')) return -1;
    long idx;
    lx_skip(L);
    int il = L->tline, ic = L->tcol;
    if (lx_uint(L, &idx)) return -1;
    if (lx_expect(L, ']')) return -1;
    if (idx >= n) {
        L->tline = il; L->tcol = ic;
        set_err(L, ORC_ERR_QUBIT_RANGE, "qubit index out of declared range");
        return -1;
    }
    return idx;
}

void orc_free(orc_circuit *C) {
    if (C) { free(C->gates); free(C); }
}

int orc_parse(const char *text, long len, orc_circuit **out, int *eline, int *ecol, char *emsg, int emsg_cap) {
    lexer L;
    memset(&L, 0, sizeof L);
    L.s = text; L.len = len; L.line = 1; L.col = 1;
    orc_circuit *C = (orc_circuit *)calloc(1, sizeof(orc_circuit));
    if (!C) return ORC_ERR_MEMORY;
    char qreg[64] = {0}, creg[64] = {0};
    int n = -1;
    unsigned char *used = NULL;   /* qubits used in the current moment */
    int moment_open = 0;
    int err_line = 0, err_col = 0;

    for (;;) {
        int c = lx_peek(&L);
        if (c < 0) break;
        int sl = L.tline, sc = L.tcol;
        char kw[64];
        if (lx_ident(&L, kw, sizeof kw)) { err_line = sl; err_col = sc; break; }
        if (strcmp(kw, "OPENQASM") == 0) {
            lx_peek(&L);
            while (L.pos < L.len && (isdigit((unsigned char)L.s[L.pos]) || L.s[L.pos] == '.')) lx_adv(&L, 1);
            if (lx_expect(&L, ';')) { err_line = L.tline; err_col = L.tcol; break; }
            continue;
        }
        if (strcmp(kw, "include") == 0) {
            if (lx_peek(&L) != '"') { set_err(&L, ORC_ERR_PARSE, "expected string"); err_line = L.tline; err_col = L.tcol; break; }
            lx_adv(&L, 1);
            while (L.pos < L.len && L.s[L.pos] != '"' && L.s[L.pos] != '\n') lx_adv(&L, 1);
            if (L.pos >= L.len || L.s[L.pos] != '"') { set_err(&L, ORC_ERR_PARSE, "unterminated string"); err_line = L.line; err_col = L.col; break; }
            lx_adv(&L, 1);
            if (lx_expect(&L, ';')) { err_line = L.tline; err_col = L.tcol; break; }
            continue;
        }
        if (strcmp(kw, "qreg") == 0 || strcmp(kw, "creg") == 0) {
            char name[64];
            long sz;
            int isq = kw[0] == 'q';
            if (isq && n >= 0) { set_err(&L, ORC_ERR_PARSE, "only one qreg allowed"); err_line = sl; err_col = sc; break; }
            if (lx_ident(&L, name, sizeof name) || lx_expect(&L, '[') || lx_uint(&L, &sz) || lx_expect(&L, ']') || lx_expect(&L, ';')) {
                err_line = L.tline; err_col = L.tcol; break;
            }
            if (isq) {
                if (sz < 1 || sz > 63) { set_err(&L, ORC_ERR_PARSE, "qreg size must be in [1, 63]"); err_line = sl; err_col = sc; break; }
                n = (int)sz;
                strcpy(qreg, name);
                used = (unsigned char *)calloc((size_t)n, 1);
            } else {
                strcpy(creg, name);
            }
            continue;
        }
        if (n < 0) { set_err(&L, ORC_ERR_PARSE, "statement before qreg declaration"); err_line = sl; err_col = sc; break; }
        if (strcmp(kw, "barrier") == 0) {
            /* barrier arglist ; -- the argument list is consumed, the moment ends */
            while (lx_peek(&L) >= 0 && lx_peek(&L) != ';') lx_adv(&L, 1);
            if (lx_expect(&L, ';')) { err_line = L.tline; err_col = L.tcol; break; }
            if (moment_open) { C->n_moments++; moment_open = 0; memset(used, 0, (size_t)n); }
            continue;
        }
        if (strcmp(kw, "measure") == 0) {
            int ql, qc;
            if (p_qarg(&L, qreg, n, &ql, &qc) < 0) { err_line = L.tline; err_col = L.tcol; break; }
            if (lx_peek(&L) != '-' ) { set_err(&L, ORC_ERR_PARSE, "expected '->'"); err_line = L.tline; err_col = L.tcol; break; }
            lx_adv(&L, 1);
            if (lx_expect(&L, '>')) { err_line = L.tline; err_col = L.tcol; break; }
            char cn[64];
            long ci;
            if (lx_ident(&L, cn, sizeof cn) || lx_expect(&L, '[') || lx_uint(&L, &ci) || lx_expect(&L, ']') || lx_expect(&L, ';')) {
                err_line = L.tline; err_col = L.tcol; break;
            }
            C->n_measure++;
            continue;
        }
        /* gate call */
        int kind, want_params, want_qubits;
        if (!strcmp(kw, "x_1_2") || !strcmp(kw, "sx")) { kind = ORC_SX; want_params = 0; want_qubits = 1; }
        else if (!strcmp(kw, "y_1_2") || !strcmp(kw, "sy")) { kind = ORC_SY; want_params = 0; want_qubits = 1; }
        else if (!strcmp(kw, "hz_1_2") || !strcmp(kw, "sw")) { kind = ORC_SW; want_params = 0; want_qubits = 1; }
        else if (!strcmp(kw, "rz")) { kind = ORC_RZ; want_params = 1; want_qubits = 1; }
        else if (!strcmp(kw, "fsim")) { kind = ORC_FSIM; want_params = 2; want_qubits = 2; }
        else { set_err(&L, ORC_ERR_UNKNOWN_GATE, "unknown gate"); err_line = sl; err_col = sc; break; }
        double prm[8];
        int np = 0;
        if (lx_peek(&L) == '(') {
            lx_adv(&L, 1);
            for (;;) {
                double v = p_expr(&L);
                if (L.err) break;
                if (np < 8) prm[np] = v;
                np++;
                int cc = lx_peek(&L);
                if (cc == ',') { lx_adv(&L, 1); continue; }
                lx_expect(&L, ')');
                break;
            }
            if (L.err) { err_line = L.tline; err_col = L.tcol; break; }
        }
        long qs[8];
        int nq = 0;
        int bad = 0;
        for (;;) {
            int ql, qc;
            long q = p_qarg(&L, qreg, n, &ql, &qc);
            if (q < 0) { bad = 1; break; }
            if (nq < 8) qs[nq] = q;
            nq++;
            if (lx_peek(&L) == ',') { lx_adv(&L, 1); continue; }
            break;
        }
        if (bad) { err_line = L.tline; err_col = L.tcol; break; }
        if (lx_expect(&L, ';')) { err_line = L.tline; err_col = L.tcol; break; }
        if (np != want_params || nq != want_qubits || (nq == 2 && qs[0] == qs[1])) {
            set_err(&L, ORC_ERR_ARITY, "gate arity mismatch");
            err_line = sl; err_col = sc;
            break;
        }
        if (!isfinite(want_params > 0 ? prm[0] : 0.0) || !isfinite(want_params > 1 ? prm[1] : 0.0)) {
            set_err(&L, ORC_ERR_PARSE, "non-finite angle");
            err_line = sl; err_col = sc;
            break;
        }
        /* moment packing: a gate touching a qubit already used in this moment opens a new one */
        int clash = 0;
        for (int i = 0; i < nq; i++) clash |= used[qs[i]];
        if (clash) { C->n_moments++; memset(used, 0, (size_t)n); }
        for (int i = 0; i < nq; i++) used[qs[i]] = 1;
        moment_open = 1;
        orc_gate g;
        g.kind = kind;
        g.q0 = (int)qs[0];
        g.q1 = nq > 1 ? (int)qs[1] : -1;
        g.theta = want_params > 0 ? prm[0] : 0.0;
        g.phi = want_params > 1 ? prm[1] : 0.0;
        if (kind == ORC_RZ) { g.phi = prm[0]; g.theta = 0.0; }
        g.moment = C->n_moments;
        if (push_gate(C, g)) { free(used); orc_free(C); return ORC_ERR_MEMORY; }
    }
    free(used);
    if (!L.err && n < 0) { set_err(&L, ORC_ERR_PARSE, "missing qreg declaration"); err_line = L.line; err_col = L.col; }
    if (L.err) {
        if (eline) *eline = err_line ? err_line : L.tline;
        if (ecol) *ecol = err_col ? err_col : L.tcol;
        if (emsg && emsg_cap > 0) snprintf(emsg, (size_t)emsg_cap, "%s", L.msg);
        int code = L.err;
        orc_free(C);
        return code;
    }
    if (moment_open) C->n_moments++;
    C->n_qubits = n;
    *out = C;
    return ORC_OK;
}

int orc_n_qubits(const orc_circuit *C) { return C->n_qubits; }
int orc_n_gates(const orc_circuit *C) { return C->n_gates; }
int orc_n_moments(const orc_circuit *C) { return C->n_moments; }
int orc_n_measure(const orc_circuit *C) { return C->n_measure; }

void orc_get_gate(const orc_circuit *C, int i, int *kind, int *q0, int *q1, double *theta, double *phi, int *moment) {
    const orc_gate *g = &C->gates[i];
    *kind = g->kind; *q0 = g->q0; *q1 = g->q1; *theta = g->theta; *phi = g->phi; *moment = g->moment;
}

/* ------------------------------------------------------------------------- */
/* O2: gate matrices, row-major, interleaved (re, im)                         */
/* ------------------------------------------------------------------------- */

/* out: 2x2 -> 8 doubles, 4x4 -> 32 doubles.  Readings V2-V4:
 *   sqrt(U) = ((1+i)/2) I + ((1-i)/2) U  for U in {X, Y, W}, W = (X+Y)/sqrt(2)
 *   Rz(phi) = diag(e^{-i phi/2}, e^{+i phi/2})
 *   fSim(theta, phi) = [[1,0,0,0],[0,cos,-i sin,0],[0,-i sin,cos,0],[0,0,0,e^{-i phi}]]
 *                      basis b_q0 + 2 b_q1 */
void orc_gate_matrix(int kind, double theta, double phi, double *out) {
    const double s2 = sqrt(0.5);
    if (kind == ORC_SX || kind == ORC_SY || kind == ORC_SW) {
        /* U as 2x2 complex */
        double U[8];
        if (kind == ORC_SX) {            /* X = [[0,1],[1,0]] */
            double u[8] = {0, 0, 1, 0, 1, 0, 0, 0};
            memcpy(U, u, sizeof u);
        } else if (kind == ORC_SY) {     /* Y = [[0,-i],[i,0]] */
            double u[8] = {0, 0, 0, -1, 0, 1, 0, 0};
            memcpy(U, u, sizeof u);
        } else {                         /* W = (X+Y)/sqrt2 = [[0,(1-i)/sqrt2],[(1+i)/sqrt2,0]] */
            double u[8] = {0, 0, s2, -s2, s2, s2, 0, 0};
            memcpy(U, u, sizeof u);
        }
        for (int r = 0; r < 2; r++)
            for (int c = 0; c < 2; c++) {
                double ur = U[2 * (2 * r + c)], ui = U[2 * (2 * r + c) + 1];
                /* ((1-i)/2) * (ur + i ui) = ((ur + ui) + i (ui - ur)) / 2 */
                double re = 0.5 * (ur + ui), im = 0.5 * (ui - ur);
                if (r == c) { re += 0.5; im += 0.5; }
                out[2 * (2 * r + c)] = re;
                out[2 * (2 * r + c) + 1] = im;
            }
        return;
    }
    if (kind == ORC_RZ) {
        out[0] = cos(phi / 2); out[1] = -sin(phi / 2);
        out[2] = 0; out[3] = 0;
        out[4] = 0; out[5] = 0;
        out[6] = cos(phi / 2); out[7] = sin(phi / 2);
        return;
    }
    /* fSim */
    memset(out, 0, 32 * sizeof(double));
    double c = cos(theta), s = sin(theta);
    out[2 * (0 * 4 + 0)] = 1.0;
    out[2 * (1 * 4 + 1)] = c;
    out[2 * (1 * 4 + 2) + 1] = -s;
    out[2 * (2 * 4 + 1) + 1] = -s;
    out[2 * (2 * 4 + 2)] = c;
    out[2 * (3 * 4 + 3)] = cos(phi);
    out[2 * (3 * 4 + 3) + 1] = -sin(phi);
}

/* ------------------------------------------------------------------------- */
/* O3/O4: state evolution, one gate at a time                                 */
/* ------------------------------------------------------------------------- */

static inline uint64_t insert_zero(uint64_t i, int q) {
    uint64_t lo = i & ((1ULL << q) - 1);
    return ((i >> q) << (q + 1)) | lo;
}

/* psi: 2*2^n doubles.  1q gate on q: for all i with bit q = 0, (psi_i, psi_{i+2^q}) <- M (...).
 * 2q gate on (q0, q1): the 4-vector at offsets {0, 2^q0, 2^q1, 2^q0+2^q1} <- M v. */
void orc_apply_gate(double *psi, int n, int kind, int q0, int q1, double theta, double phi) {
    double M[32];
    orc_gate_matrix(kind, theta, phi, M);
    if (kind != ORC_FSIM) {
        const int64_t half = (int64_t)1 << (n - 1);
        const uint64_t st = 1ULL << q0;
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < half; i++) {
            uint64_t i0 = insert_zero((uint64_t)i, q0), i1 = i0 | st;
            double v[4] = {psi[2 * i0], psi[2 * i0 + 1], psi[2 * i1], psi[2 * i1 + 1]};
            double o[4];
            for (int r = 0; r < 2; r++) {
                double re = 0, im = 0;
                for (int c = 0; c < 2; c++) {
                    double mr = M[2 * (2 * r + c)], mi = M[2 * (2 * r + c) + 1];
                    re += mr * v[2 * c] - mi * v[2 * c + 1];
                    im += mr * v[2 * c + 1] + mi * v[2 * c];
                }
                o[2 * r] = re; o[2 * r + 1] = im;
            }
            psi[2 * i0] = o[0]; psi[2 * i0 + 1] = o[1];
            psi[2 * i1] = o[2]; psi[2 * i1 + 1] = o[3];
        }
        return;
    }
    const int64_t quarter = (int64_t)1 << (n - 2);
    const int lo = q0 < q1 ? q0 : q1, hi = q0 < q1 ? q1 : q0;
    const uint64_t s0 = 1ULL << q0, s1 = 1ULL << q1;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < quarter; i++) {
        uint64_t b = insert_zero(insert_zero((uint64_t)i, lo), hi);
        uint64_t idx[4] = {b, b | s0, b | s1, b | s0 | s1};   /* basis b_q0 + 2 b_q1 */
        double v[8], o[8];
        for (int k = 0; k < 4; k++) { v[2 * k] = psi[2 * idx[k]]; v[2 * k + 1] = psi[2 * idx[k] + 1]; }
        for (int r = 0; r < 4; r++) {
            double re = 0, im = 0;
            for (int c = 0; c < 4; c++) {
                double mr = M[2 * (4 * r + c)], mi = M[2 * (4 * r + c) + 1];
                re += mr * v[2 * c] - mi * v[2 * c + 1];
                im += mr * v[2 * c + 1] + mi * v[2 * c];
            }
            o[2 * r] = re; o[2 * r + 1] = im;
        }
        for (int k = 0; k < 4; k++) { psi[2 * idx[k]] = o[2 * k]; psi[2 * idx[k] + 1] = o[2 * k + 1]; }
    }
}

/* Evolve e_0 through the first `max_gates` gates (all if < 0), source order. */
int orc_build_state(const orc_circuit *C, double *psi, int max_gates) {
    const int n = C->n_qubits;
    const int64_t N = (int64_t)1 << n;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < 2 * N; i++) psi[i] = 0.0;
    psi[0] = 1.0;
    int G = (max_gates < 0 || max_gates > C->n_gates) ? C->n_gates : max_gates;
    for (int g = 0; g < G; g++) {
        const orc_gate *x = &C->gates[g];
        orc_apply_gate(psi, n, x->kind, x->q0, x->q1, x->theta, x->phi);
    }
    return ORC_OK;
}

/* O5/O6: T = sum_x |psi_x|^2, sequential in logical order (this is C(2^n - 1)). */
double orc_total_prob(const double *psi, int n) {
    const int64_t N = (int64_t)1 << n;
    double T = 0.0;
    for (int64_t x = 0; x < N; x++) T += psi[2 * x] * psi[2 * x] + psi[2 * x + 1] * psi[2 * x + 1];
    return T;
}

/* ------------------------------------------------------------------------- */
/* O7: shot uniforms (reading V12) -- the oracle's own SplitMix64              */
/* ------------------------------------------------------------------------- */
static uint64_t sm64_output(uint64_t seed, uint64_t k) {   /* k-th output, k >= 1 */
    uint64_t z = seed + k * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* u[i] = uniform for shot s = offset + i: (output s+1) >> 11, times 2^-53 */
void orc_uniforms(uint64_t seed, uint64_t offset, uint64_t count, double *u) {
    for (uint64_t i = 0; i < count; i++)
        u[i] = (double)(sm64_output(seed, offset + i + 1) >> 11) * (1.0 / 9007199254740992.0);
}

/* ------------------------------------------------------------------------- */
/* O8: inverse-CDF sampling by one streaming pass over sorted targets         */
/* ------------------------------------------------------------------------- */
typedef struct { double t; uint64_t s; } tpair;

static int cmp_tpair(const void *a, const void *b) {
    const tpair *x = (const tpair *)a, *y = (const tpair *)b;
    if (x->t < y->t) return -1;
    if (x->t > y->t) return 1;
    return x->s < y->s ? -1 : (x->s > y->s);
}

/* x_s = min{x : C(x) > u_s T}; fallback: last x with p > 0.  Refuses |T-1| > norm_tol
 * (1e-6).  T_out receives T. */
int orc_sample(const double *psi, int n, const double *u, uint64_t shots, uint64_t *x_out,
               double norm_tol, double *T_out) {
    const int64_t N = (int64_t)1 << n;
    double T = orc_total_prob(psi, n);
    if (T_out) *T_out = T;
    if (!(fabs(T - 1.0) <= norm_tol)) return ORC_ERR_NORM;
    tpair *tp = (tpair *)malloc((size_t)shots * sizeof(tpair) + 1);
    if (!tp) return ORC_ERR_MEMORY;
    for (uint64_t s = 0; s < shots; s++) { tp[s].t = u[s] * T; tp[s].s = s; }
    qsort(tp, (size_t)shots, sizeof(tpair), cmp_tpair);
    uint64_t k = 0;
    double Cx = 0.0;
    int64_t last_nz = -1;
    for (int64_t x = 0; x < N && k < shots; x++) {
        double p = psi[2 * x] * psi[2 * x] + psi[2 * x + 1] * psi[2 * x + 1];
        Cx += p;
        if (p > 0) last_nz = x;
        while (k < shots && tp[k].t < Cx) { x_out[tp[k].s] = (uint64_t)x; k++; }
    }
    if (k < shots) {
        for (int64_t x = N - 1; x >= 0; x--) {
            double p = psi[2 * x] * psi[2 * x] + psi[2 * x + 1] * psi[2 * x + 1];
            if (p > 0) { last_nz = x; break; }
        }
        for (; k < shots; k++) x_out[tp[k].s] = (uint64_t)(last_nz < 0 ? 0 : last_nz);
    }
    free(tp);
    return ORC_OK;
}

/* O9: linear XEB (reading V14). */
int orc_xeb(const double *psi, int n, const uint64_t *x, uint64_t shots, double *F, double *sigma, double *mean_p) {
    const uint64_t N = 1ULL << n;
    if (shots == 0) return ORC_ERR_ARG;
    double sum = 0.0;
    for (uint64_t s = 0; s < shots; s++) {
        if (x[s] >= N) return ORC_ERR_SIZE;
        sum += psi[2 * x[s]] * psi[2 * x[s]] + psi[2 * x[s] + 1] * psi[2 * x[s] + 1];
    }
    double mean = sum / (double)shots;
    double ss = 0.0;
    for (uint64_t s = 0; s < shots; s++) {
        double p = psi[2 * x[s]] * psi[2 * x[s]] + psi[2 * x[s] + 1] * psi[2 * x[s] + 1];
        ss += (p - mean) * (p - mean);
    }
    double var = shots > 1 ? ss / (double)(shots - 1) : 0.0;
    *mean_p = mean;
    *F = ldexp(mean, n) - 1.0;
    *sigma = ldexp(sqrt(var), n) / sqrt((double)shots);
    return ORC_OK;
}

/* F* = 2^n sum_x p_x^2 - 1 : the XEB an ideal sampler has in expectation. */
double orc_fstar(const double *psi, int n) {
    const int64_t N = (int64_t)1 << n;
    double s = 0.0;
    for (int64_t x = 0; x < N; x++) {
        double p = psi[2 * x] * psi[2 * x] + psi[2 * x + 1] * psi[2 * x + 1];
        s += p * p;
    }
    return ldexp(s, n) - 1.0;
}

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* host threads for the parallel loops (timing only: bench.py's oracle arm under torchrun, which
   exports OMP_NUM_THREADS=1) */
void orc_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}
