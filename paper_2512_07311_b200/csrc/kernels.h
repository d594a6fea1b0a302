// kernels.h -- launchers for the sm_100a kernels of kernels.cu (all stream-ordered).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace rcs {
namespace dev {

// launches issued by this library (every launcher below increments it)
uint64_t launches();
void count_launch();

// K9: 6-qubit fused pass on tensor cores (tc_pass.cu).  d_a = tc_matrix_words() words made
// by tc_pack_matrix from the fp64 64x64 block matrix (fp16 hi/lo split of the real 128x128
// embedding, scaled by 2^14).
size_t tc_matrix_words();
void tc_pack_matrix(const double* u_re_im, uint32_t* out);
// Optional chunking (pipelined remaps): fix[0..nfix) are extra positions held at the bits of
// fixval, so the launch covers one 2^-nfix slice of the index space.  Fixed positions must lie
// outside tc_reserved_mask(pos); the grid is min(num_sms, tiles).
// K12 (the transposed kernel, any target layout) runs when n_local >= 13 and at most one target
// sits in positions 0..3 (tc_uses_k12: a function of the block, positions 0..6 being pinned);
// K9 otherwise, or for every block with force_k9 (tests, comparisons).
bool tc_uses_k12(int n_local_bits, const int* pos);
// tile_counter (one device word, may be nullptr): K12 hands tiles out through it (zeroed here,
// stream-ordered) instead of the static blockIdx.x + k gridDim.x assignment.
// tc_flags: kTcForceK9 (every block on K9), kTcBulkRuns (K12 loads its runs with plain bulk copies
// even when they are short; default: a 5-D tensor-map TMA moves many short runs per request).
constexpr int kTcForceK9 = 1, kTcBulkRuns = 2, kTcNoRow = 4;   // kTcNoRow: [0..5] blocks on K9
cudaError_t gate_pass_tc(float2* amps, int n_local_bits, const int* pos, const uint32_t* d_a, int num_sms,
                         cudaStream_t st, const int* fix = nullptr, int nfix = 0, uint64_t fixval = 0,
                         int tc_flags = 0, unsigned* tile_counter = nullptr);
// positions a chunk bit must avoid for this pass: the 12-bit tile sub-cube and the bit above its run
uint64_t tc_reserved_mask(int n_local_bits, const int* pos);
// a6 (K1) fused dense gate pass: amps <- M (x) over every group of 2^k amplitudes that
// differ only in the physical bits pos[0..k) (matrix bit i <-> pos[i]); M is 2^k x 2^k
// complex64 row-major (interleaved float pairs).  n_local_bits = log2(#amps).
cudaError_t gate_pass(float2* amps, int n_local_bits, int k, const int* pos, const float* m_interleaved,
                      cudaStream_t st);

// in-place involution: swap physical bits a[i] <-> b[i] (disjoint pairs) over 2^nbits amps
cudaError_t bit_swap(float2* amps, int nbits, int npairs, const int* a, const int* b, cudaStream_t st);

// remap staging: buf[t] = amps[l(m0 + t)] (pack) or amps[l(m0 + t)] = buf[t] (unpack), where
// l(m) inserts the j code bits `codemask` at the (ascending) local positions lpos[0..j)
cudaError_t pack(const float2* amps, float2* buf, int j, const int* lpos_sorted, uint64_t codemask,
                 uint64_t m0, uint64_t count, cudaStream_t st);
cudaError_t unpack(float2* amps, const float2* buf, int j, const int* lpos_sorted, uint64_t codemask,
                   uint64_t m0, uint64_t count, cudaStream_t st);

// a7 (K10-lite): in-place remap over NVLink.  For every peer c: swap local[l] <-> peer_c[l'] with
// l = ins(m) | mask_c, l' = ins(m) | my_mask (ins = insert zeros at the sorted local swap
// positions), for m in this rank's share [m_begin_c, m_begin_c + m_count_c) (m even, pairs of
// amplitudes moved as 16-B vectors).  Peer pointers are CUDA-IPC mappings of the peers' shards.
struct PeerSwapArgs {
    float2* local;
    float2* peer[7];
    int npeers;
    int j;
    int lpos[8];
    uint64_t mask[7];
    uint64_t my_mask;
    uint64_t m_begin[7], m_count[7];   // element-pair range of this rank, per peer
    int nfix;                          // chunking: extra fixed positions (ascending) ...
    int fix[4];
    uint64_t fixval;                   // ... and their bits
    int max_grid;                      // 0: default
};
cudaError_t peer_swap(const PeerSwapArgs& a, cudaStream_t st);

// a9 (K5): bsum[blk] = sum_{x in blk} |a_x|^2 (fp64) for blocks of 2^b amps; part[c] = per-CTA
// partial sum of p^2 (fixed grid => deterministic).  Returns the number of partials used.
int block_sums_grid();
cudaError_t block_sums(const float2* amps, uint64_t nblocks, int b, double* bsum, double* part_sq,
                       cudaStream_t st);

// a10 (K6): in-place inclusive scan of d[0..n) in fp64, deterministic; tmp must hold
// scan_tmp_doubles(n) doubles.
uint64_t scan_tmp_doubles(uint64_t n);
cudaError_t scan_inclusive(double* d, uint64_t n, double* tmp, cudaStream_t st);

// fixed-order reduction of n doubles -> out[0] (single CTA)
cudaError_t reduce_sum(const double* in, int n, double* out, cudaStream_t st);

struct SampleArgs {
    const float2* amps;
    const double* inc;      // inclusive block prefix of this rank's shard
    uint64_t nblocks;
    int b;
    double T_total, E_r, T_r;
    int owns_tail;          // 1: this rank owns every t >= E_r (last rank with T_r > 0)
    int owns_any;           // 0: owns nothing (T_r == 0)
    uint64_t seed, shot0, shots;
    const double* u_in;     // optional caller uniforms (chunk-local), else SplitMix64
    uint64_t base_index;    // rank * 2^n_local
    unsigned long long* x_out;  // chunk-local, 0 for shots owned by other ranks
    // kept permuted layout: inc is the GLOBAL logical block prefix (nblocks = 2^(n-b)), every
    // rank searches every shot, the owner of the found block (per ptab) does the in-block scan
    const uint64_t* ptab;   // nullptr: canonical layout
    int nl;                 // local index bits
    uint64_t rank;
    uint64_t last_block;    // last logical block with non-zero mass (tail fallback)
};
// a11 (K7): per-shot binary search over block prefixes + warp-cooperative in-block scan
cudaError_t sample(const SampleArgs& a, cudaStream_t st);

// a13 (K8): per-CTA partial (sum p, sum p^2, count) over owned bitstrings; bad_flag set if
// any x >= 2^n.  Returns grid size used.
int xeb_grid();
// where a logical index lives: canonical (ptab == nullptr: rank = x >> nl) or a kept permuted
// layout (ptab = kPermTables x 256 byte tables mapping logical block bits to physical ones)
constexpr int kPermTables = 5;   // logical block index up to 40 bits
struct Locator {
    int nl;                 // local index bits
    uint64_t rank;
    int b;                  // block bits (positions < b are the same physically and logically)
    const uint64_t* ptab;
};
cudaError_t xeb_partials(const float2* amps, const unsigned long long* x, uint64_t count, const Locator& L,
                         int n_bits, double* part /* 3*grid */, int* bad_flag, cudaStream_t st);
cudaError_t xeb_finalize(const double* part, int grid, double* out3, cudaStream_t st);

// p_out[i] = |a_{x_i}|^2 if x_i is on this rank else 0
cudaError_t gather_prob(const float2* amps, const unsigned long long* x, uint64_t count, const Locator& L,
                        int n_bits, double* p, int* bad_flag, cudaStream_t st);
// out[lb] = in[perm(lb)] for lb < n (logical block order from physical); ptab as in Locator
cudaError_t perm_blocks(const double* in, double* out, uint64_t n, const uint64_t* ptab, cudaStream_t st);
// *out = last index with inc[i] > inc[i-1] (0 if none)
cudaError_t last_nonzero(const double* inc, uint64_t n, unsigned long long* out, cudaStream_t st);

cudaError_t init_basis(float2* amps, uint64_t n_amps, int set_one, cudaStream_t st);

// Product-state prefix (plan.cpp): amps[i] = tabA[ia] * tabB[ib] (the tables are the fp64 block
// products rounded to complex64; the complex product is fp32 in a fixed operation order) for the
// physical index X = base + i, where ia / ib gather X's bits that hold the
// two groups' qubits (OR of per-byte tables byt[G][c][X byte c]); 0 if X has a bit set at a
// position of zmask (qubits still |0>).  Write-only: 8 B per amplitude.
constexpr int kPrefixBytes = 8;   // X up to 64 bits
struct PrefixArgs {
    float2* amps;
    uint64_t n_amps;               // even
    uint64_t base;                 // physical index of amps[0] (rank << n_local)
    const float2* tab[2];          // the two group tables (fp64 products rounded to fp32)
    const uint32_t* byt;           // [2][nbytes][256]
    int nbytes;
    uint64_t zmask;
};
cudaError_t product_init(const PrefixArgs& a, cudaStream_t st);

}  // namespace dev
}  // namespace rcs
