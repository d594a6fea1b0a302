// internal.h -- host-side data structures shared by the library's translation units.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/rcs.h"

namespace rcs {

// One source gate (SPEC S:28-31 GateOp).  rz keeps its angle in phi.
struct Gate {
    int kind;
    int q0, q1;       // q1 = -1 for 1-qubit gates
    double theta, phi;
    int moment;
};

struct Circuit {
    int n = 0;
    int n_moments = 0;
    int n_measure = 0;
    std::vector<Gate> gates;
};

// parse.cpp -- returns RCS_OK or an error with line/col
rcs_status parse_qasm(const char* text, size_t len, Circuit& out, rcs_error* err);

// gates.cpp -- dense matrices in fp64, row-major, basis index b_q0 + 2 b_q1
struct cplx { double re, im; };
void gate_matrix(const Gate& g, cplx* m);   // 4 entries (1q) or 16 entries (2q)

// plan.cpp
struct Block {
    std::vector<int> qubits;     // logical, ascending; matrix bit i <-> qubits[i]
    std::vector<int> gate_ids;   // source gates in application order
    std::vector<cplx> matrix;    // 2^k x 2^k, row-major, fp64 product
};

struct Item {
    int type;                    // RCS_ITEM_*
    int block = -1;              // PASS: index into blocks
    int k = 0;
    int pos[8] = {0};            // PASS: physical position of matrix bit i
    int a[8] = {0}, b[8] = {0};  // REMAP / SWAP pairs
};

struct Plan {
    int n = 0, n_global = 0, fuse_k = 0;
    std::vector<Block> blocks;
    std::vector<Item> items;
    int n_passes = 0, n_remaps = 0, n_swaps = 0;
};

// low physical positions never moved by remaps (keeps qubit 0 at bit 0 for the
// 128-bit pair loads of the gate-pass kernel and keeps short runs contiguous)
constexpr int kPinnedLow = 3;
// the tensor-core pass tiles 6 target + 6 column bits
constexpr int kTcMinLocal = 12;

rcs_status build_plan(const Circuit& c, int fuse_k, int n_global, Plan& out, rcs_error* err);

void set_error(rcs_error* err, int code, const char* fmt, ...);

}  // namespace rcs

struct rcs_circuit {
    rcs::Circuit c;
};

struct rcs_plan {
    rcs::Plan p;
};
