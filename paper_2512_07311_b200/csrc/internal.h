// internal.h -- host-side data structures shared by the library's translation units.
#pragma once

#include <array>
#include <cstdint>
#include <map>
#include <tuple>
#include <memory>
#include <mutex>
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
    // items [restore_begin, end) only bring the layout back to canonical; final_pos[q] is the
    // physical position of qubit q before them (>= n - n_global: a rank bit)
    int pinned = 6;                 // physical positions [0, pinned) never move (kPinnedLow or 7)
    int restore_begin = 0;
    std::vector<int> final_pos;
    std::vector<int> initial_pos;   // empty: canonical start (qubit q at position q)
    // Product-state prefix: items [0, prefix) are the leading fused blocks with pairwise disjoint
    // qubit sets.  They act on |0...0>, so the state after them is the product of their first
    // columns (and |0> on every other qubit): one write-only kernel replaces init + these passes.
    // The set is chosen on the fusion result alone (P-independent), split into two groups of
    // consecutive blocks (A, B); tab[G][v] = product over the group's blocks (fusion order, fp64)
    // of their first-column entries, v's bit i <-> pq[G][i] (ascending qubits); an amplitude is
    // tab[A][vA] * tab[B][vB] in fp64, rounded once -- the same arithmetic for every sharding.
    int prefix = 0;
    std::vector<int> pq[2];
    std::vector<cplx> tab[2];
};

// low physical positions never moved by remaps: keeps qubit 0 at bit 0 (the CUDA-core pass
// moves amplitude pairs along bit 0) and makes qubits 0..5 always local, so a 5-qubit block
// can be padded onto the tensor-core pass with one of them whatever the sharding (the
// padded arithmetic depends on which qubit pads it: the choice must be layout-independent)
constexpr int kPinnedLow = 6;
// 6-qubit (tensor-core) plans pin one more: the K9 / K12 choice (K12 iff no target among
// positions 0..6) must be a function of the block alone
inline int pinned_low(int k) { return k >= 5 ? 7 : kPinnedLow; }
// the tensor-core pass tiles 6 target + 6 column bits
constexpr int kTcMinLocal = 12;
// fuser: ready gates tried as block seeds besides the earliest unassigned one
constexpr int kFuseSeeds = 8;
// fuser: pick among the seeds by the block count of a greedy completion (rollout)
constexpr bool kFuseLookahead = true;
constexpr int kFuseDeepDepth = 3;        // strategy 2: extension search depth
constexpr bool kRemapPrefetch = true;   // remaps also bring in soon-needed global qubits
constexpr bool kInitialPlacement = true;   // start with the latest-used qubits global (free: |0> state)
constexpr int kPrefixGroupBits = 18;      // product-state prefix: qubits per table (2^18 x 16 B = 4 MiB)

// given: the fused blocks (qubits + gate ids) to use instead of running the fuser
// use_prefix = false: no product-state prefix (every block is a pass and is remapped as one)
rcs_status build_plan(const Circuit& c, int fuse_k, int n_global, Plan& out, rcs_error* err,
                      const std::vector<Block>* given = nullptr, bool use_prefix = true);
// strategies: 2-level extension search, prefix-first greedy, prefix-first 1-level, prefix-first
// with a 1-level prefix phase and a 3-level rest, prefix-first beam search (plan.cpp)
constexpr int kFuseStrategies = 5;
int64_t fuse_cost(const std::vector<Block>& blocks);   // passes << 20 | blocks (lower is better)
void fuse_strategy(const Circuit& c, int k, int which, std::vector<Block>& out);
int fuse_best(const Circuit& c, int k, std::vector<Block>* cand /* [kFuseStrategies] */);
int plan_block_k(int n, int fuse_k, int n_global);   // the block width build_plan uses

void set_error(rcs_error* err, int code, const char* fmt, ...);

}  // namespace rcs

namespace rcs {
// ---- snapshot.cpp: paper stage 2/3 artifacts
struct Sha256 {   // FIPS 180-4, incremental
    uint32_t h[8];
    uint8_t buf[64];
    size_t fill = 0;
    uint64_t total = 0;
    Sha256();
    void update(const void* data, size_t n);
    void final(uint8_t out[32]);

private:
    void block(const uint8_t* p);
};
constexpr int kSnapHeaderBytes = 52;
constexpr uint32_t kSnapVersion = 1;
struct SnapHeader {
    uint32_t version, n_qubits;
    uint64_t payload_bytes;
    uint8_t digest[32];
};
void put_snapshot_header(uint8_t out[kSnapHeaderBytes], uint32_t n_qubits, const uint8_t digest[32]);
bool get_snapshot_header(const uint8_t in[kSnapHeaderBytes], SnapHeader* h, const char** why);
uint64_t job_seed(uint64_t base_seed, uint64_t job_id);

// tensor-core pass operands of a plan: which items run on K9, their 6 positions (5-qubit blocks
// padded with one more local qubit) and the packed fp16 hi/lo matrices (host copy)
// product-state prefix operands for one (plan, n_local): fp64 group tables + byte gather tables
struct PrefixPack {
    std::vector<float> tab[2];             // interleaved complex (fp64 products rounded), 2^|group| each
    std::vector<uint32_t> byt;             // [2][nbytes][256]
    int nbytes = 0;
    uint64_t zmask = 0;                    // physical positions of the qubits outside the prefix
};

struct TcPack {
    std::vector<int> slot;                 // per item, -1 if not a tensor-core pass
    std::vector<std::array<int, 6>> pos;
    std::vector<uint32_t> words;           // n_tc * tc_matrix_words()
    int n_tc = 0;
};
}  // namespace rcs

struct rcs_circuit {
    rcs::Circuit c;
    uint64_t uid = 0;   // unique per parsed circuit (device-side caches key on it)
    // plans are a pure function of (circuit, fuse_k, n_global): cached, shared read-only
    std::mutex mu;
    std::map<std::pair<int, int>, std::shared_ptr<const rcs::Plan>> plans;
    std::map<std::tuple<int, int, int>, std::shared_ptr<const rcs::TcPack>> packs;
    std::map<std::pair<int, int>, std::shared_ptr<const rcs::PrefixPack>> prefix_packs;
};

struct rcs_plan {
    rcs::Plan p;
};
