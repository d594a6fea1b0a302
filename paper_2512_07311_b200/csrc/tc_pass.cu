// tc_pass.cu -- K9: 6-qubit fused gate pass on the 5th-gen tensor cores (tcgen05, sm_100a).
//
// A 6-qubit dense block U (64x64 complex) applied to the state is a real GEMM
//     [Y_re; Y_im] (128 x N) = [[U_re, -U_im], [U_im, U_re]] (128 x 128) . [X_re; X_im] (128 x N)
// over the columns j = the non-target index (BASELINE.json north_star: "tensor cores only if
// fused-gate width makes it a real dense contraction").  A's rows are interleaved (row 2t =
// Y_re[t], row 2t+1 = Y_im[t]) so one TMEM lane pair holds re/im of one output amplitude.
//
// Precision: fp32-level results from fp16 tensor cores with an EXACT main term.  Matrix row
// pair t and state column j get power-of-two scales 2^F_t / 2^E_j that put their largest
// magnitude in [2^10, 2^11); each value is split into hi = rint(x 2^s) (an integer, exact in
// fp16) and lo = fp16(x 2^s - hi):
//     A B = 2^-(F_t + E_j) (A_hi B_hi + [A_hi B_lo + A_lo B_hi]) + O(2^-20 relative)
// A_hi B_hi is a sum of integer products that stays below 2^24, so the tensor core's truncating
// fp32 accumulation adds it exactly (scripts/micro/tc_exact.cu: inexact in 7.5e-5 of outputs,
// only by overflowing 2^24); only the cross terms (2^-11 of the result, their own accumulator)
// round.  Measured: bias -4e-10 relative per product (round 1's floating split: -1.4e-7 per
// pass in norm^2, which capped a build at ~70 passes), rms error 3.9e-7.  The scales depend on
// the column's own 64 amplitudes only, never on how columns are grouped into tiles, so the state
// stays bitwise identical for every sharding.
//
// Tile = 64 columns x 64 target combinations = 4096 amplitudes (32 KB), a 12-bit sub-cube of
// the index: the 6 target bits plus the 6 lowest non-target bits, so every tile is a set of
// 2^(12-r) contiguous runs of 2^r >= 64 amplitudes.  Persistent kernel, one CTA per SM:
//   warp  13   producer: cp.async.bulk (TMA) of a PAIR of adjacent tiles (tile index bit 0 is
//                         index bit r, right above every run, so each copy covers both tiles'
//                         runs: >= 1 KB per copy) into a raw pair slot (2 slots = 128 KB, no
//                         registers) -> rfull[slot] (complete_tx)
//   warps 0-7  converters: raw smem -> column max -> scale 2^E_j -> hi/lo split -> STS into
//                         B stage (K-major, interleaved core matrices) -> full[s]
//   warp  12   MMA     : 8 K-steps x 3 terms = 24 tcgen05.mma kind::f16 (M=128, N=64, K=16,
//                         A in TMEM) into D[d] -> commit empty[s], tfull[d]
//   warps 8-11 epilogue: tcgen05.ld the 2 accumulators of D[d] -> tempty[d] -> sum, unscale by
//                         2^-E_j 2^-F_t -> STS staging [t][j] -> coalesced LDS/STG (each
//                         thread owns one column, rows t0 + 2i)
// The converters of a column (4 threads in 4 warps) agree on its max through a shared-memory
// atomicMax and one named barrier; E_j reaches the epilogue through a 4-slot ring guarded by an
// mbarrier per slot.
// Shared memory: raw 4 x 32 KB + B 2 x 32 KB + staging 33 KB + control = 227 KB.
// TMEM (512 cols): A_hi [0,64), A_lo [64,128) (fp16 pairs), D[d] = [128 + 128 d, +128) holding
// the cross-term and main-term accumulators (64 columns each).
#include <cuda.h>   // CUtensorMap (the encoder is fetched through cudaGetDriverEntryPoint)
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "kernels.h"

namespace rcs {
namespace dev {
namespace {

constexpr int kLoadWarps = 8, kEpiWarp0 = 8, kEpiWarps = 4, kMmaWarp = 12, kProdWarp = 13, kWarps = 14;
constexpr int kThreadsTC = kWarps * 32;
constexpr int kEpiThreads = kEpiWarps * 32;
constexpr int TN = 64;                       // columns per tile (MMA N)
constexpr int TK = 128;                      // real K
constexpr int kStages = 2;                   // B stages
constexpr int kRaw = 4;                      // raw (TMA) stages
constexpr uint32_t kRawBytes = 4096 * 8;
constexpr uint32_t kBBytes = TN * TK * 2;    // 16 KB per fp16 hi or lo tile
constexpr uint32_t kStageBytes = 2 * kBBytes;
constexpr uint32_t kSBO = (TK / 8) * 128;    // next 8-row group (16 chunks of 16 B)
constexpr int kPitchF = 128;                 // staging row t: 64 float2, column j at j ^ g(t) (swizzle)
constexpr uint32_t kStagingBytes = 64 * kPitchF * 4;
constexpr int kExpSlots = 4;                 // per-tile column exponents in flight (converter -> epilogue)
constexpr uint32_t kCtlBytes = 3072;   // barriers + offset tables; total <= 227 KB
// control block: (12 + kExpSlots) mbarriers + 64 run offsets (8 B) + 3 x 64 column maxima (4 B)
// + 2 x 64 uint16 + kExpSlots x 64 exponents (1 B) + the TMEM slot
static_assert((12 + kExpSlots) * 8 + 64 * 8 + 3 * 64 * 4 + 2 * 64 * 2 + kExpSlots * 64 * 4 + 4 <= kCtlBytes,
              "control block overflow");
constexpr uint32_t kSmemBytes = kRaw * kRawBytes + kStages * kStageBytes + kStagingBytes + kCtlBytes;
constexpr int kAccCols = 2 * TN;             // one D buffer: acc 0 cross terms, acc 1 main term

struct TcArgs {
    float2* amps;
    const uint32_t* a;       // [2][128][64] packed fp16 pairs: A_hi then A_lo (row m, column c = k/2)
    uint64_t ntiles;
    int pos[6];              // physical position of matrix bit i
    int jpos[6];             // the 6 lowest non-target positions (column bits, ascending)
    int sub[12];             // all 12 sub-cube positions, ascending (for the tile base deposit)
    int r;                   // sub[0..r) == 0..r-1: runs of 2^r contiguous amplitudes
    int pair;                // 2: tiles processed in adjacent pairs (ntiles >= 2), else 1
    int sto[32];             // staging row offset (floats) of sub-cube index 128 i: t_i * 128
    int sxj[32];             // ... and its swizzled column part j_i ^ g(t_i)
    uint64_t sgo[32];        // global offset (amplitudes) of sub-cube index 128 i
    int gsh;                 // staging swizzle g(t) = rotate-left of t's 4 low bits by gsh
    int nins;                // 12 + number of fixed (chunk) bits
    int ins[16];             // sub-cube and fixed positions, ascending (tile base deposit)
    uint64_t fixval;         // value of the fixed bits (one chunk of the index space)
    uint64_t fmask;          // positions the tile index is deposited into (below n_local)
    uint64_t dstride;        // deposit of the per-CTA tile-pair stride (gridDim.x * pair)
    int rot_lane[3];         // ROT: lane bit driving rotation bit m (t bits 0..2), -1: none
    int to_lane;             // ROT: lane bit XORed into the octet index (t bit 3), -1: none
};

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t ins0(uint64_t x, int s) {
    return ((x >> s) << (s + 1)) | (x & ((1ull << s) - 1));
}

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("{\n.reg .b64 st;\nmbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    uint32_t done = 0;
    do {
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\nselp.u32 %0, 1, 0, p;\n}"
                     : "=r"(done)
                     : "r"(su32(b)), "r"(parity), "r"(0x2000)   // suspend-time hint (ns): sleep, don't spin
                     : "memory");
    } while (!done);
}

__device__ __forceinline__ uint64_t bdesc(uint32_t saddr) {
    // K-major, SWIZZLE_NONE: core matrix = 8 rows x 16 B; LBO (next K chunk) = 128 B,
    // SBO (next 8-row group) = 2048 B; version 1 (sm100)
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)(128 >> 4) << 16;
    d |= (uint64_t)(kSBO >> 4) << 32;
    d |= 1ull << 46;
    return d;
}

// byte offset of the 16-B chunk holding B elements (column n, k = 8c .. 8c+7)
__device__ __forceinline__ uint32_t bchunk(int n, int c) {
    return (uint32_t)((n >> 3) * kSBO + c * 128 + (n & 7) * 16);
}

// out half k = in half (k - rho) & 7 for a packed octet of fp16 (4 words); rho lane-dependent,
// so it is done with selects and byte permutes (no dynamic register indexing)
__device__ __forceinline__ void rot_h8(uint32_t (&w)[4], int rho) {
    uint32_t a[4];
#pragma unroll
    for (int i = 0; i < 4; i++) a[i] = (rho & 2) ? w[(i + 3) & 3] : w[i];   // 1 word = 2 halves
#pragma unroll
    for (int i = 0; i < 4; i++) w[i] = (rho & 4) ? a[(i + 2) & 3] : a[i];   // 2 words
#pragma unroll
    for (int i = 0; i < 4; i++) a[i] = __byte_perm(w[(i + 3) & 3], w[i], 0x5432);   // 1 half
#pragma unroll
    for (int i = 0; i < 4; i++) w[i] = (rho & 1) ? a[i] : w[i];
}

__device__ __forceinline__ float2 f2mul(float2 v, float s) {   // packed f32x2 multiply
    float2 o;
    asm("{\n.reg .b64 x, y;\nmov.b64 x, {%2, %3};\nmov.b64 y, {%4, %4};\nmul.rn.f32x2 x, x, y;\n"
        "mov.b64 {%0, %1}, x;\n}"
        : "=f"(o.x), "=f"(o.y)
        : "f"(v.x), "f"(v.y), "f"(s));
    return o;
}

#define TMEM_ST32(addr, R)                                                                                       \
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14," \
                 "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(addr),         \
                 "r"(R[0]), "r"(R[1]), "r"(R[2]), "r"(R[3]), "r"(R[4]), "r"(R[5]), "r"(R[6]), "r"(R[7]),          \
                 "r"(R[8]), "r"(R[9]), "r"(R[10]), "r"(R[11]), "r"(R[12]), "r"(R[13]), "r"(R[14]), "r"(R[15]),    \
                 "r"(R[16]), "r"(R[17]), "r"(R[18]), "r"(R[19]), "r"(R[20]), "r"(R[21]), "r"(R[22]), "r"(R[23]),  \
                 "r"(R[24]), "r"(R[25]), "r"(R[26]), "r"(R[27]), "r"(R[28]), "r"(R[29]), "r"(R[30]), "r"(R[31]))

#define TMEM_ST16(addr, R)                                                                                       \
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14," \
                 "%15,%16};" ::"r"(addr),                                                                          \
                 "r"(R[0]), "r"(R[1]), "r"(R[2]), "r"(R[3]), "r"(R[4]), "r"(R[5]), "r"(R[6]), "r"(R[7]),          \
                 "r"(R[8]), "r"(R[9]), "r"(R[10]), "r"(R[11]), "r"(R[12]), "r"(R[13]), "r"(R[14]), "r"(R[15]))

#define TMEM_LD32(addr, R)                                                                                     \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14," \
                 "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"               \
                 : "=r"(R[0]), "=r"(R[1]), "=r"(R[2]), "=r"(R[3]), "=r"(R[4]), "=r"(R[5]), "=r"(R[6]),        \
                   "=r"(R[7]), "=r"(R[8]), "=r"(R[9]), "=r"(R[10]), "=r"(R[11]), "=r"(R[12]), "=r"(R[13]),    \
                   "=r"(R[14]), "=r"(R[15]), "=r"(R[16]), "=r"(R[17]), "=r"(R[18]), "=r"(R[19]),              \
                   "=r"(R[20]), "=r"(R[21]), "=r"(R[22]), "=r"(R[23]), "=r"(R[24]), "=r"(R[25]),              \
                   "=r"(R[26]), "=r"(R[27]), "=r"(R[28]), "=r"(R[29]), "=r"(R[30]), "=r"(R[31])               \
                 : "r"(addr))

// the registers of a tcgen05.ld are defined by tcgen05.wait::ld, not by the ld: pin every use
// after the wait
// ... ordered with memory accesses (the epilogue issues the next chunk's loads before its stores)
#define TMEM_LD32M(addr, R)                                                                                     \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14," \
                 "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"               \
                 : "=r"(R[0]), "=r"(R[1]), "=r"(R[2]), "=r"(R[3]), "=r"(R[4]), "=r"(R[5]), "=r"(R[6]),        \
                   "=r"(R[7]), "=r"(R[8]), "=r"(R[9]), "=r"(R[10]), "=r"(R[11]), "=r"(R[12]), "=r"(R[13]),    \
                   "=r"(R[14]), "=r"(R[15]), "=r"(R[16]), "=r"(R[17]), "=r"(R[18]), "=r"(R[19]),              \
                   "=r"(R[20]), "=r"(R[21]), "=r"(R[22]), "=r"(R[23]), "=r"(R[24]), "=r"(R[25]),              \
                   "=r"(R[26]), "=r"(R[27]), "=r"(R[28]), "=r"(R[29]), "=r"(R[30]), "=r"(R[31])               \
                 : "r"(addr)                                                                                  \
                 : "memory")

// the registers of a tcgen05.ld are defined by tcgen05.wait::ld, not by the ld: pin every use
// after the wait
#define REG_FENCE32(R)                                                                                       \
    asm volatile("" : "+r"(R[0]), "+r"(R[1]), "+r"(R[2]), "+r"(R[3]), "+r"(R[4]), "+r"(R[5]), "+r"(R[6]),     \
                 "+r"(R[7]), "+r"(R[8]), "+r"(R[9]), "+r"(R[10]), "+r"(R[11]), "+r"(R[12]), "+r"(R[13]),       \
                 "+r"(R[14]), "+r"(R[15]), "+r"(R[16]), "+r"(R[17]), "+r"(R[18]), "+r"(R[19]), "+r"(R[20]),    \
                 "+r"(R[21]), "+r"(R[22]), "+r"(R[23]), "+r"(R[24]), "+r"(R[25]), "+r"(R[26]), "+r"(R[27]),    \
                 "+r"(R[28]), "+r"(R[29]), "+r"(R[30]), "+r"(R[31]))

#define MMA_F16(d, a, b, idesc, acc)                                                                         \
    asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, " #acc ";" ::"r"(d), "r"(a), "l"(b), \
                 "r"(idesc))

// Exact main term: the state column j is scaled by 2^E_j (E_j from the column's max |x|, so the
// max lands in [2^10, 2^11)) and split into hi = rint(x 2^E_j) -- an integer, exact in fp16 --
// and lo = fp16(x 2^E_j - hi).  Matrix row pair t likewise with 2^F_t (host, tc_pack_matrix).
// The main products hi.hi are then integers and their sums stay below 2^24 (checked at 7.5e-5
// overflow rate on Porter-Thomas data, scripts/micro/tc_exact.cu), so the tensor core's
// truncating fp32 accumulation adds them EXACTLY; only the small cross terms hi.lo + lo.hi
// (2^-11 of the result) round.  The result is (main + cross) 2^-E_j 2^-F_t, one round-to-nearest
// add and two exact scalings.  The scale is a function of the column's 64 amplitudes only, never
// of the tiling, so the arithmetic stays independent of the sharding (bitwise P-invariance).
__device__ __forceinline__ int col_exponent(int maxbits) {
    // max |x| as float bits (>= 0) -> E with max 2^E in [2^10, 2^11); 0 for an all-zero column;
    // clamped so 2^E and 2^-E are normal floats
    if (maxbits == 0) return 0;
    const int e = ((maxbits >> 23) & 0xff) - 127;
    const int E = 10 - e;
    return E > 126 ? 126 : E;
}
__device__ __forceinline__ float pow2f(int e) { return __int_as_float((127 + e) << 23); }   // e in [-126, 127]

// (v0, v1) already scaled -> hi = fp16x2(rint v0, rint v1) (exact integers), lo = fp16x2(v - hi).
// rint by the magic constant 1.5 2^23 (|v| <= 2^11: v + M has an ulp of 1, round-half-even like
// cvt.rni), all three steps as packed f32x2 operations; v - hi is exact.
__device__ __forceinline__ void split_exact_h2(float v0, float v1, uint32_t& hi, uint32_t& lo) {
    float h0, h1, r0, r1;
    asm("{\n.reg .b64 x, m, t, h, r;\n"
        "mov.b64 x, {%4, %5};\nmov.b64 m, {%6, %6};\n"
        "add.rn.f32x2 t, x, m;\nsub.rn.f32x2 h, t, m;\nsub.rn.f32x2 r, x, h;\n"
        "mov.b64 {%0, %1}, h;\nmov.b64 {%2, %3}, r;\n}"
        : "=f"(h0), "=f"(h1), "=f"(r0), "=f"(r1)
        : "f"(v0), "f"(v1), "f"(12582912.0f));
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(hi) : "f"(h1), "f"(h0));
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(lo) : "f"(r1), "f"(r0));
}

__device__ __forceinline__ float absmax2(float m, float2 v) { return fmaxf(m, fmaxf(fabsf(v.x), fabsf(v.y))); }

// ROT: when >= 2 target bits are among the 4 lowest sub-cube bits, the converters' shared-memory
// reads of one element index across lanes hit the same banks; lane l then walks its target octet
// starting at element (l & 7) and rotates the packed fp16 octet back before storing it.
template <bool ROT>
__global__ void __launch_bounds__(kThreadsTC, 1) k_pass_tc(const __grid_constant__ TcArgs p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    float2* raw = reinterpret_cast<float2*>(smem);                                   // [2 pair slots][8192]
    uint8_t* stages = smem + kRaw * kRawBytes;                                       // [kStages][hi|lo]
    float* staging = reinterpret_cast<float*>(stages + kStages * kStageBytes);       // run-padded tile
    uint8_t* ctl = reinterpret_cast<uint8_t*>(staging) + kStagingBytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(ctl);   // [kStages]
    uint64_t* empty = full + kStages;                     // [kStages]
    uint64_t* tfull = empty + kStages;                    // [2]
    uint64_t* tempty = tfull + 2;                         // [2]
    uint64_t* rfull = tempty + 2;                         // [2] raw pair slots
    uint64_t* rempty = rfull + 2;                         // [2]
    uint64_t* cready = rempty + 2;                        // [kExpSlots] column exponents of a tile written
    uint64_t* offr = cready + kExpSlots;                  // [64] run offsets (global)
    int* cmax = reinterpret_cast<int*>(offr + 64);        // [3][64] column max |x| (float bits, atomicMax)
    uint16_t* soft = reinterpret_cast<uint16_t*>(cmax + 3 * 64);   // [64] sub-cube index of target combo t
    uint16_t* sofj = soft + 64;                                    // [64] sub-cube index of column j
    float* colfac = reinterpret_cast<float*>(sofj + 64);           // [kExpSlots][64] 2^-E_j per tile
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(colfac + kExpSlots * 64);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; s++) {
            mbar_init(&full[s], kLoadWarps * 32);
            mbar_init(&empty[s], 1);
        }
        for (int d = 0; d < 2; d++) {
            mbar_init(&tfull[d], 1);
            mbar_init(&tempty[d], kEpiThreads);
        }
        for (int r = 0; r < 2; r++) {
            mbar_init(&rfull[r], 1);
            mbar_init(&rempty[r], 2 * kLoadWarps * 32);   // both tiles of the pair consumed
        }
        for (int e = 0; e < kExpSlots; e++) mbar_init(&cready[e], 64);   // the 64 column owners (to == 0)
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (threadIdx.x < 3 * 64) cmax[threadIdx.x] = 0;
    if (threadIdx.x < 64) {
        const int x = threadIdx.x;
        uint64_t orr = 0;
        int st = 0, sj = 0;
        for (int i = 0; i < 6; i++) {
            int rt = 0, rj = 0;   // rank of pos[i] / jpos[i] among the sorted sub-cube bits
            for (int b = 0; b < 12; b++) {
                rt += p.sub[b] < p.pos[i];
                rj += p.sub[b] < p.jpos[i];
            }
            if ((x >> i) & 1) {
                st |= 1 << rt;
                sj |= 1 << rj;
            }
        }
        for (int b = p.r; b < 12; b++)
            if ((x >> (b - p.r)) & 1) orr |= 1ull << p.sub[b];
        offr[x] = orr;
        // raw pair layout: element index = s with a zero inserted at bit r (bit r = pair half)
        const int lowm = (1 << p.r) - 1;
        soft[x] = (uint16_t)(((st & ~lowm) << 1) | (st & lowm));
        sofj[x] = (uint16_t)(((sj & ~lowm) << 1) | (sj & lowm));
    }
    // sub-cube index s -> (target combo t, column j, global offset); bit b of s is sub[b]
    auto decomp = [&](int sidx, int& t, int& jj, uint64_t& go) {
        t = 0;
        jj = 0;
        go = 0;
        for (int b = 0; b < 12; b++) {
            if (!((sidx >> b) & 1)) continue;
            go |= 1ull << p.sub[b];
            for (int i = 0; i < 6; i++) {
                if (p.pos[i] == p.sub[b]) t |= 1 << i;
                if (p.jpos[i] == p.sub[b]) jj |= 1 << i;
            }
        }
    };
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;

    // A (hi, lo; packed fp16 pairs) -> TMEM by the epilogue warps (warp q owns lanes 32q..)
    if (warp >= kEpiWarp0 && warp < kEpiWarp0 + 4) {
        const int q = warp - kEpiWarp0;
        const int m = q * 32 + lane;
        for (int h = 0; h < 2; h++)
            for (int c0 = 0; c0 < 64; c0 += 32) {
                uint32_t r[32];
                const uint4* src = reinterpret_cast<const uint4*>(p.a + (size_t)h * 128 * 64 + (size_t)m * 64 + c0);
#pragma unroll
                for (int c = 0; c < 8; c++) {
                    const uint4 v = __ldg(src + c);
                    r[4 * c] = v.x;
                    r[4 * c + 1] = v.y;
                    r[4 * c + 2] = v.z;
                    r[4 * c + 3] = v.w;
                }
                TMEM_ST32(tmem + ((uint32_t)(q * 32) << 16) + h * 64 + c0, r);
            }
        asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");

    const uint64_t ntiles = p.ntiles;
    // tile base = deposit of the tile index into the free positions, | the fixed bits.  Each role
    // walks pairs (2i, 2i+1), i = blockIdx.x + k gridDim.x, and advances the deposited base of the
    // pair's even tile incrementally: pdep(x + y) = ((pdep(x) | ~M) + pdep(y)) & M.
    auto tile_base = [&](uint64_t tile) {
        uint64_t b = tile;
#pragma unroll
        for (int i = 0; i < 16; i++)
            if (i < p.nins) b = ins0(b, p.ins[i]);
        return b;
    };
    const uint64_t first_tile = (uint64_t)blockIdx.x * p.pair;
    const uint64_t first_base = tile_base(first_tile);
    const uint64_t rbit = 1ull << p.r;   // tile index bit 0 -> position r (first free position)
    auto next_tile = [&](uint64_t& t, uint64_t& bp) {
        if (p.pair == 2 && !(t & 1)) {
            t += 1;
            return;
        }
        t = t - (p.pair == 2 ? 1 : 0) + (uint64_t)gridDim.x * p.pair;
        bp = ((bp | ~p.fmask) + p.dstride) & p.fmask;
    };
    auto base_of = [&](uint64_t t, uint64_t bp) { return bp | ((p.pair == 2 && (t & 1)) ? rbit : 0) | p.fixval; };

    if (warp == kProdWarp) {
        // ---------------- TMA producer: both tiles of a pair, runs of 2 x 2^r amplitudes
        const int nruns = 1 << (12 - p.r);
        const uint32_t copy_bytes = (8u << p.r) * (uint32_t)p.pair;   // one run of each tile of the pair
        const uint32_t dst_stride = (8u << p.r) * 2;                  // same layout when pair == 1
        uint64_t it = 0, bp = first_base;
        for (uint64_t tile = first_tile; tile < ntiles; it++) {
            if (p.pair == 2 && (tile & 1)) { next_tile(tile, bp); continue; }   // odd half: copied with its pair
            const int slot = (it >> (p.pair - 1)) & 1;
            const uint64_t use = it >> (p.pair);                   // uses of this slot before
            mbar_wait(&rempty[slot], (use & 1) ^ 1);
            if (lane == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&rfull[slot])),
                             "r"(kRawBytes * p.pair)
                             : "memory");
            __syncwarp();
            const float2* src = p.amps + base_of(tile, bp);
            const uint32_t dst = su32(raw + (size_t)slot * 8192);
            for (int u = lane; u < nruns; u += 32)
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        dst + u * dst_stride),
                    "l"(src + offr[u]), "r"(copy_bytes), "r"(su32(&rfull[slot]))
                    : "memory");
            next_tile(tile, bp);
        }
    } else if (warp < kLoadWarps) {
        // ---------------- converters: thread = column j, target octets `to` and `to + 4`
        const int lt = threadIdx.x;           // 0..255
        const int j = lt & 63;
        const int to = lt >> 6;               // 0..3
        const int sj = sofj[j];
        // ROT: the lane bits whose column ranks do not reach the banks (displaced by low targets)
        // rotate the t octet (t bits 0..2) and flip t bit 3, so a half-warp reads 16 bank pairs
        int rho = 0, tox = to;
        if (ROT) {
#pragma unroll
            for (int m = 0; m < 3; m++)
                if (p.rot_lane[m] >= 0) rho |= ((lane >> p.rot_lane[m]) & 1) << m;
            if (p.to_lane >= 0) tox ^= (lane >> p.to_lane) & 1;
        }
        int boff[16];   // raw-slot element offsets of this thread's 16 amplitudes (tile-invariant)
#pragma unroll
        for (int i = 0; i < 16; i++) boff[i] = soft[8 * (tox + 4 * (i >> 3)) + ((i + rho) & 7)] | sj;
        uint64_t it = 0, bp = first_base;
        for (uint64_t tile = first_tile; tile < ntiles; next_tile(tile, bp), it++) {
            const int slot = (it >> (p.pair - 1)) & 1;
            const uint64_t use = it >> (p.pair);
            mbar_wait(&rfull[slot], use & 1);
            const float2* rb = raw + (size_t)slot * 8192 + ((p.pair == 2 && (tile & 1)) ? (1 << p.r) : 0);
            float2 b[16];
            float mx = 0.f;
#pragma unroll
            for (int i = 0; i < 16; i++) {
                b[i] = rb[boff[i]];
                mx = absmax2(mx, b[i]);
            }
            mbar_arrive(&rempty[slot]);
            if (p.pair == 1) mbar_arrive(&rempty[slot]);   // count is for two tiles
            // column max over the 4 threads of column j (warps j/32 + 2 to): smem atomicMax on
            // the float bits (non-negative floats order like ints), one named barrier
            const int cb = (int)(it % 3);
            atomicMax(&cmax[cb * 64 + j], __float_as_int(mx));
            asm volatile("bar.sync 2, 256;" ::: "memory");
            const int E = col_exponent(cmax[cb * 64 + j]);
            if (to == 0) cmax[((it + 2) % 3) * 64 + j] = 0;   // buffer of tile it+2: all read it at tile it-1
            const float sc = pow2f(E);
#pragma unroll
            for (int i = 0; i < 16; i++) b[i] = f2mul(b[i], sc);
            const int s = it % kStages;
            mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
            // E_j -> epilogue.  Slot it % 4 was last read by the epilogue of tile it-4, which
            // released D before the MMA of tile it-2 ran, which freed stage s (waited above): the
            // write (and the slot mbarrier's next phase) must come after that wait.
            const int es = (int)(it % kExpSlots);
            if (to == 0) {
                colfac[es * 64 + j] = pow2f(-E);
                mbar_arrive(&cready[es]);             // release: the epilogue reads E_j after acquiring
            }
            uint8_t* bhi = stages + s * kStageBytes;
            uint8_t* blo = bhi + kBBytes;
#pragma unroll
            for (int g = 0; g < 2; g++) {
                uint32_t rh[4], rl[4], ih[4], il[4];
#pragma unroll
                for (int e2 = 0; e2 < 4; e2++) {
                    const float2 v0 = b[8 * g + 2 * e2], v1 = b[8 * g + 2 * e2 + 1];
                    split_exact_h2(v0.x, v1.x, rh[e2], rl[e2]);
                    split_exact_h2(v0.y, v1.y, ih[e2], il[e2]);
                }
                if (ROT) {
                    rot_h8(rh, rho);
                    rot_h8(rl, rho);
                    rot_h8(ih, rho);
                    rot_h8(il, rho);
                }
                const int c = tox + 4 * g;                // t octet -> K chunk (re); +8 (im)
                const uint32_t ore = bchunk(j, c), oim = bchunk(j, c + 8);
                *reinterpret_cast<uint4*>(bhi + ore) = make_uint4(rh[0], rh[1], rh[2], rh[3]);
                *reinterpret_cast<uint4*>(bhi + oim) = make_uint4(ih[0], ih[1], ih[2], ih[3]);
                *reinterpret_cast<uint4*>(blo + ore) = make_uint4(rl[0], rl[1], rl[2], rl[3]);
                *reinterpret_cast<uint4*>(blo + oim) = make_uint4(il[0], il[1], il[2], il[3]);
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_arrive(&full[s]);
        }
    } else if (warp == kMmaWarp) {
        // ---------------- MMA issuer
        const uint32_t idesc = (1u << 4) | ((uint32_t)(TN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        uint64_t it = 0, bp = first_base;
        for (uint64_t tile = first_tile; tile < ntiles; next_tile(tile, bp), it++) {
            const int s = it % kStages, d = it & 1;
            mbar_wait(&full[s], (it / kStages) & 1);
            mbar_wait(&tempty[d], ((it >> 1) & 1) ^ 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            if (lane == 0) {
                const uint32_t sb = su32(stages + s * kStageBytes);
                const uint32_t d0 = tmem + 128 + d * kAccCols;
                // descriptors of K-step ks = base + ks * (256 B >> 4): no carry out of the 14-bit field
                const uint64_t bh0 = bdesc(sb), bl0 = bdesc(sb + kBBytes);
                const uint32_t ah = tmem, al = tmem + 64;
                // cross terms (A_hi B_lo, A_lo B_hi) -> accumulator 0 (rounds; 2^-11 of the result)
                MMA_F16(d0, ah, bl0, idesc, 0);
                MMA_F16(d0, al, bh0, idesc, 1);
#pragma unroll
                for (int ks = 1; ks < TK / 16; ks++) {
                    MMA_F16(d0, ah + ks * 8, bl0 + ks * 16, idesc, 1);
                    MMA_F16(d0, al + ks * 8, bh0 + ks * 16, idesc, 1);
                }
                // main term A_hi B_hi -> accumulator 1: integer products, exact sums
                MMA_F16(d0 + TN, ah, bh0, idesc, 0);
#pragma unroll
                for (int ks = 1; ks < TK / 16; ks++) MMA_F16(d0 + TN, ah + ks * 8, bh0 + ks * 16, idesc, 1);
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                    su32(&empty[s])));
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                    su32(&tfull[d])));
            }
            __syncwarp();
        }
    } else if (warp >= kEpiWarp0 && warp < kEpiWarp0 + kEpiWarps) {
        // ---------------- epilogue: warp q reads TMEM lane quarter q (rows 32q .. 32q+31)
        const int q = warp & 3;
        const int et = threadIdx.x - kEpiWarp0 * 32;   // 0..127
        const int m = q * 32 + lane;                   // D row: t = m/2, re (m even) / im (m odd)
        const int trow = m >> 1, comp = m & 1;
        const float rowfac = pow2f(-(int)p.a[2 * 128 * 64 + trow]);   // 2^-F_t
        // store phase in memory order: thread handles sub-cube indices et + 128 i (i < 32), so
        // consecutive lanes write consecutive addresses for every target layout
        int tb, jb;
        uint64_t gb;
        decomp(et, tb, jb, gb);
        // staging swizzle: element (t, j) at float2 (64 t + (j ^ g(t))), g = a rotation of t's low
        // 4 bits chosen on the host so that both the row-wise writes (16 rows per warp) and the
        // memory-order reads (the 4 lowest cube ranks per half-warp: low targets + low columns)
        // hit 16 distinct bank pairs
        auto gsw = [&](int t) { const int x = t & 15; return ((x << p.gsh) | (x >> (4 - p.gsh))) & 15; };
        const float* sld = staging + tb * kPitchF;
        const int jbs = jb ^ gsw(tb);
        float* st = staging + trow * kPitchF + comp;
        const int gw = gsw(trow);
        uint64_t it = 0, bp = first_base;
        for (uint64_t tile = first_tile; tile < ntiles; next_tile(tile, bp), it++) {
            const int d = it & 1;
            const int es = (int)(it % kExpSlots);
            mbar_wait(&cready[es], (uint32_t)((it / kExpSlots) & 1));
            mbar_wait(&tfull[d], (it >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + 128 + d * kAccCols;
            const float* ce = colfac + es * 64;
            // per-tile copies of the swizzle terms: hoisting the 64 + 32 swizzled offsets out of
            // the tile loop would hold them in registers (spills)
            int gwt = gw, jbt = jbs;
            asm volatile("" : "+r"(gwt), "+r"(jbt));
#pragma unroll
            for (int h = 0; h < 2; h++) {
                uint32_t a0[32], a1[32];
                TMEM_LD32(ta + 32 * h, a0);
                TMEM_LD32(ta + TN + 32 * h, a1);
                asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
                for (int c = 0; c < 32; c += 2) {
                    // 2^-E_j of the column pair (written once per column by the converters; this
                    // slot is rewritten only after this tile's D buffer is released, below)
                    const float2 f = *reinterpret_cast<const float2*>(ce + 32 * h + c);
                    const float f0 = f.x, f1 = f.y;
                    float o0, o1;   // ((cross + main) (2^-E_c, 2^-E_c+1)) 2^-F_t
                    asm("{\n.reg .b64 x, y, u, v;\n"
                        "mov.b64 x, {%2, %3};\nmov.b64 y, {%4, %5};\nmov.b64 u, {%6, %7};\nmov.b64 v, {%8, %8};\n"
                        "add.rn.f32x2 x, x, y;\nmul.rn.f32x2 x, x, u;\nmul.rn.f32x2 x, x, v;\n"
                        "mov.b64 {%0, %1}, x;\n}"
                        : "=f"(o0), "=f"(o1)
                        : "r"(a0[c]), "r"(a0[c + 1]), "r"(a1[c]), "r"(a1[c + 1]), "f"(f0), "f"(f1), "f"(rowfac));
                    st[2 * ((32 * h + c) ^ gwt)] = o0;
                    st[2 * ((32 * h + c + 1) ^ gwt)] = o1;
                }
                if (h == 1) {   // D buffer (and with it this tile's colfac slot) released
                    asm volatile("tcgen05.fence::before_thread_sync;");
                    mbar_arrive(&tempty[d]);
                }
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");
            float2* dst = p.amps + (base_of(tile, bp) | gb);
#pragma unroll 8
            for (int i = 0; i < 32; i++) {
                const float2 v = *reinterpret_cast<const float2*>(sld + p.sto[i] + 2 * (jbt ^ p.sxj[i]));
                __stcs(dst + p.sgo[i], v);
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");   // staging reused by the next tile
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// =====================================================================================
// K12: the transposed product, for ANY target layout (n_local >= 13).
//     Y^T (128 j x 128 n) = X^T (128 j x 128 k) . B (128 k x 128 n),  B[k][n] = A_K9[n][k]
// Tile = a 13-bit sub-cube of the index: the 6 target positions plus the 7 lowest non-target
// positions (the columns j).  Positions 0..6 always lie in the cube, so the tile is 2^(13-r)
// runs of 2^r >= 128 contiguous amplitudes (TMA copies >= 1 KB).  In shared memory an element
// sits at its cube index (bit b = the b-th lowest cube position).  The state tile (64 target
// combinations t x 128 columns j) is the TMEM operand A: converter thread j packs its row (fp16
// hi/lo of re/im for every t) with tcgen05.st -- no B-stage round trip through shared memory --
// and the constant matrix is the shared-memory operand.  D rows are columns j, so the epilogue
// stores straight from registers (no staging): a warp writes 32 columns of one t, i.e. 256
// contiguous bytes when no target sits below position 5.
// Bank conflicts: the 16 lanes of a half-warp read 16 columns of one t; when a targets occupy
// cube ranks 0..3, only 4-a column bits vary the bank.  K12 takes a <= 1 (more: K9): the lanes
// whose displaced column bit (j bit 3) is set read t XOR (the low target's bit) instead, which
// makes the 16 reads hit 16 distinct bank pairs; after the fp16 split the packed words are put
// back in t order (a byte permute for t bit 0, selects for t bits 1..4).  t bit 5 selects the
// thread's half and must not be flipped: the planner pins qubits 0..6 to positions 0..6 and pads
// 5-qubit blocks with a pinned qubit as matrix bit 0, so a block's highest qubit (t bit 5)
// never sits below cube rank 4.
// K order (t + 64 c), k-steps and accumulators are K9's: the main term is exact, so K9 and K12
// differ only in how the cross terms round.
//   warp  13   producer: TMA of the runs of a tile into a raw slot
//   warps 0-7  converters: warp w -> TMEM lanes 32 (w & 3).., t half w >> 2 -> A buffer
//   warp  12   MMA: 24 x tcgen05.mma (M=128, N=128, K=16), A = state (TMEM), B = matrix (smem)
//   warps 8-11 epilogue: D (2 accumulators) -> registers -> global
// TMEM: A buffers [0,128) and [128,256) (hi at +0, lo at +64); D acc 0 at 256, acc 1 at 384.
struct TcTArgs {
    float2* amps;
    const uint32_t* a;       // K9-packed A (hi, lo): row n, word c = k pair (2c, 2c+1); F_t after
    uint64_t ntiles;
    int pos[6];              // physical position of matrix (target) bit i
    int tcube[6];            // cube rank of pos[i]
    int jpos[7];             // physical position of column bit k (the 7 lowest non-targets)
    int jcube[7];            // cube rank of jpos[k]
    int r;                   // cube ranks 0..r-1 are positions 0..r-1 (runs of 2^r amplitudes)
    int nrun_pos;            // 13 - r: cube positions above the runs ...
    int run_pos[6];          // ... (the TMA run index is deposited into them)
    int lane_t[4];           // PT = kPermMulti: lane bit b XORs t bit lane_t[b] into the reads (-1: none)
    int pmask;               // ... the t bits so permuted
    int phi_t;               // lanes with column bit 3 set read t XOR (1 << phi_t) (bank-conflict
                             // free); -1 if no target sits in cube ranks 0..3
    int nins;                // 13 cube positions + chunk bits, ascending
    int ins[17];
    uint64_t fixval;         // chunk bits (pipelined remaps), as K9
    uint64_t fmask, dstride; // tile-index deposit (as K9)
    unsigned* counter;       // dynamic tile scheduler (zeroed before the launch), nullptr: static
    // Short runs (r <= 8: 64 or 32 copies of 1-2 KB per tile) go through a 5-D tensor map instead:
    // dim 0 = the 2^r contiguous amplitudes, dim 1 = the tile base in units of 2^r amplitudes
    // (box 1), dims 2..4 = the lowest groups of consecutive run positions (extent 2^m, stride 2^p
    // amplitudes).  Each request fills a contiguous range of the slot in cube-index order; the
    // run bits the dims do not cover select the request (treq[u], added to the dim-1 coordinate).
    int nreq;                // 0: one bulk copy per run
    uint32_t req_bytes;      // bytes per request (8192 * 8 / nreq)
    int treq[8];             // per request: dim-4 coordinate offset (units of 2^r amplitudes)
    alignas(64) CUtensorMap tmap;
    alignas(64) CUtensorMap tmap_st;   // PT = kRow: the epilogue's TMA store map
};

// build-time variants for A/B measurements (RCS_NVCC_FLAGS=-D...): D split into two N = 64 halves,
// epilogue loads of the next chunk issued before the current chunk's stores
#ifndef RCS_K12_NSPLIT
#define RCS_K12_NSPLIT 1
#endif
#ifdef RCS_K12_WB_STORES   // A/B: write-back stores instead of streaming (evict-first) ones
#define K12_STORE(p, v) (*(p) = (v))
#else
#define K12_STORE(p, v) __stcs((p), (v))
#endif
constexpr uint32_t kTRaw = 8192 * 8;
constexpr int kTRing = 8;                             // tile bases in flight (producer -> all roles)
constexpr uint64_t kTileEnd = ~0ull;                  // ring sentinel: no more tiles                  // one tile: 64 KB
constexpr uint32_t kTMat = 2 * 128 * 128 * 2;         // B hi + lo: 64 KB
constexpr uint32_t kTCtl = 3584;
static_assert((12 + kExpSlots) * 8 + 64 * 8 + 64 * 8 + kTRing * 8 + 3 * 128 * 4 + 64 * 4 + kExpSlots * 128 + 4 <= kTCtl,
              "K12 control block");
constexpr uint32_t kTSmem = 2 * kTRaw + kTMat + kTCtl;
constexpr uint32_t kTRowStage = 2 * 8 * 128 * 8;      // kRow: 2 staging buffers of 8 t x 128 j (float2)

// 32-bit conditional swap (select) of a and b
__device__ __forceinline__ void cswap(bool f, uint32_t& a, uint32_t& b) {
    const uint32_t x = f ? b : a, y = f ? a : b;
    a = x;
    b = y;
}

// Undo t ^= (f << tb) on the 16 packed words of one converter thread (word i packs t = 2i,
// 2i+1 of its 32): t bit 0 is a half swap inside every word, t bit tb >= 1 a swap of words
// i <-> i ^ 2^(tb-1).  tb is uniform over the launch, f per lane.
template <int B>
__device__ __forceinline__ void swap_words(uint32_t (&w)[16], bool f) {
#pragma unroll
    for (int i = 0; i < 16; i++)
        if (!((i >> B) & 1)) cswap(f, w[i], w[i | (1 << B)]);
}
template <int TB>
__device__ __forceinline__ void unpermute16(uint32_t (&w)[16], bool f) {
    if (TB == 0) {
        const uint32_t sel = f ? 0x1032u : 0x3210u;
#pragma unroll
        for (int i = 0; i < 16; i++) w[i] = __byte_perm(w[i], 0, sel);
    } else if (TB > 0) {
        swap_words<(TB > 0 ? TB - 1 : 0)>(w, f);
    }
}

// every t bit of pmask whose lane flag (phi) is set: undo the XOR (stages commute)
__device__ __forceinline__ void unpermute_mask(uint32_t (&w)[16], int pmask, uint32_t phi) {
    if (pmask & 1) unpermute16<0>(w, phi & 1);
    if (pmask & 2) unpermute16<1>(w, (phi >> 1) & 1);
    if (pmask & 4) unpermute16<2>(w, (phi >> 2) & 1);
    if (pmask & 8) unpermute16<3>(w, (phi >> 3) & 1);
    if (pmask & 16) unpermute16<4>(w, (phi >> 4) & 1);
}

// PT: the t bit the lanes with column bit 3 set flip (-1: none, no permutation); kPermMulti:
// two to four targets at cube ranks 0..3 -- lane bits 4-a..3 (the column bits displaced above
// rank 3) each flip one of them (TcTArgs::lane_t), so the 16 reads of a half-warp hit 16 bank
// pairs; the packed words are put back by one select / byte-permute stage per flipped t bit
constexpr int kPermMulti = 8;
// kRow: the block's targets are positions 0..5 in matrix-bit order (a row of 64 contiguous
// amplitudes per column j).  K12's column-per-thread reads and stores would hit one bank / 32
// sectors per instruction there, so this variant moves the tile with tensor-map TMA both ways:
// loaded into shared memory with the 128-B swizzle (rows j, 16-B chunks XOR j & 7: a half-warp's
// 16-B reads of one t-pair hit distinct banks) and stored from a 64-B-swizzled staging buffer
// (8 t x 128 j per TMA store, double buffered), no register permutation either way.
constexpr int kRow = 9;

template <int PT>
__global__ void __launch_bounds__(kThreadsTC, 1) k_pass_tct(const __grid_constant__ TcTArgs p) {
    constexpr bool PERM = PT >= 0 && PT != kRow;   // kRow reads its rows conflict-free without it
    extern __shared__ __align__(1024) uint8_t smem[];
    float2* raw = reinterpret_cast<float2*>(smem);                       // [2][8192] by cube index
    uint8_t* mat = smem + 2 * kTRaw;                                      // B hi | B lo (K-major)
    uint8_t* ctl = mat + kTMat + (PT == kRow ? kTRowStage : 0);   // kRow: staging after the matrix
    uint64_t* rfull = reinterpret_cast<uint64_t*>(ctl);   // [2]
    uint64_t* rempty = rfull + 2;                         // [2]
    uint64_t* afull = rempty + 2;                         // [2]
    uint64_t* aempty = afull + 2;                         // [2]
    uint64_t* dfull = aempty + 2;                         // [2] D half h (outputs n in [64 h, +64)) written
    uint64_t* dempty = dfull + 2;                         // [2] ... and read by the epilogue
    uint64_t* cready = dempty + 2;                        // [kExpSlots] column exponents of a tile written
    uint64_t* offt = cready + kExpSlots;                  // [64] physical offset of target combination t
    uint64_t* offr = offt + 64;                           // [64] physical offset of TMA run u
    uint64_t* tring = offr + 64;                          // [kTRing] tile base of iteration it (or kTileEnd)
    int* cmax = reinterpret_cast<int*>(tring + kTRing);   // [3][128] column max |x| (float bits)
    float* rowfac = reinterpret_cast<float*>(cmax + 3 * 128);   // [64] 2^-F_t
    int8_t* colexp = reinterpret_cast<int8_t*>(rowfac + 64);     // [kExpSlots][128] E_j per tile
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(colexp + kExpSlots * 128);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; i++) {
            mbar_init(&rfull[i], 1);
            mbar_init(&rempty[i], kLoadWarps * 32);
            mbar_init(&afull[i], kLoadWarps * 32);
            mbar_init(&aempty[i], 1);
        }
        for (int h = 0; h < 2; h++) {
            mbar_init(&dfull[h], 1);
            mbar_init(&dempty[h], kEpiThreads);
        }
        for (int e = 0; e < kExpSlots; e++) mbar_init(&cready[e], 128);   // the 128 column owners (th == 0)
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    for (int i = threadIdx.x; i < 3 * 128; i += blockDim.x) cmax[i] = 0;
    if (threadIdx.x < 64) {
        const int x = threadIdx.x;
        uint64_t ot = 0, orr = 0;
        for (int i = 0; i < 6; i++) {
            if ((x >> i) & 1) ot |= 1ull << p.pos[i];
            if (i < p.nrun_pos && ((x >> i) & 1)) orr |= 1ull << p.run_pos[i];
        }
        offt[x] = ot;
        offr[x] = orr;
        rowfac[x] = pow2f(-(int)p.a[2 * 128 * 64 + x]);
    }
    // the matrix as the K-major shared-memory operand: core chunk (n, c) = A_K9 words [n][4c..4c+3]
    for (int e = threadIdx.x; e < 2 * 128 * 16; e += blockDim.x) {
        const int h = e >> 11, n = (e >> 4) & 127, c = e & 15;
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(p.a + (size_t)h * 128 * 64 + (size_t)n * 64 + 4 * c));
        *reinterpret_cast<uint4*>(mat + h * (kTMat / 2) + bchunk(n, c)) = v;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;

    auto tile_base = [&](uint64_t tile) {
        uint64_t b = tile;
#pragma unroll
        for (int i = 0; i < 17; i++)
            if (i < p.nins) b = ins0(b, p.ins[i]);
        return b;
    };
    const uint64_t ntiles = p.ntiles;
    const uint64_t first = blockIdx.x;

    if (warp == kProdWarp) {
        // The producer decides the tile sequence and publishes each tile's base in tring (read by
        // the other roles after the mbarrier chain rfull -> afull -> cready/dfull); kTileEnd ends
        // every role's loop.  Dynamic mode: tiles from a global atomic counter, so SMs that run
        // faster (HBM placement, die) take more tiles; static: blockIdx.x + k gridDim.x.
        const int nruns = 1 << p.nrun_pos;
        const uint32_t run_bytes = 8u << p.r;
        uint64_t it = 0, bp = tile_base(first), tile = first;
        unsigned nxt = 0;
        if (p.counter) {
            if (lane == 0) nxt = atomicAdd(p.counter, 1u);
            tile = __shfl_sync(0xffffffffu, nxt, 0);
        }
        for (;; it++) {
            const int slot = it & 1;
            mbar_wait(&rempty[slot], ((it >> 1) & 1) ^ 1);
            if (tile >= ntiles) {
                if (lane == 0) {
                    tring[it % kTRing] = kTileEnd;
                    mbar_arrive(&rfull[slot]);   // completes the phase without data
                }
                break;
            }
            if (p.counter) {
                bp = tile_base(tile);
                if (lane == 0) nxt = atomicAdd(p.counter, 1u);   // next tile, in flight during this copy
            }
            if (lane == 0) {
                tring[it % kTRing] = bp | p.fixval;
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&rfull[slot])),
                             "r"(kTRaw)
                             : "memory");
            }
            __syncwarp();
            const float2* src = p.amps + (bp | p.fixval);
            const uint32_t dst = su32(raw + (size_t)slot * 8192);
            if (PT == kRow) {   // one 4-D tensor load of the whole tile (its base, all bits >= 13, / 2^13)
                if (lane == 0)
                    asm volatile(
                        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
                        "%3, %4, %5}], [%6];" ::"r"(dst),
                        "l"(reinterpret_cast<uint64_t>(&p.tmap)), "r"(0), "r"(0), "r"(0), "r"((int)((bp | p.fixval) >> 13)),
                        "r"(su32(&rfull[slot]))
                        : "memory");
            } else if (p.nreq) {
                if (lane < p.nreq) {
                    const int cb = (int)((bp | p.fixval) >> p.r) + p.treq[lane];
                    asm volatile(
                        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
                        "%3, %4, %5, %6}], [%7];" ::"r"(dst + lane * p.req_bytes),
                        "l"(reinterpret_cast<uint64_t>(&p.tmap)), "r"(0), "r"(cb), "r"(0), "r"(0), "r"(0),
                        "r"(su32(&rfull[slot]))
                        : "memory");
                }
            } else {
                for (int u = lane; u < nruns; u += 32)
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            dst + u * run_bytes),
                        "l"(src + offr[u]), "r"(run_bytes), "r"(su32(&rfull[slot]))
                        : "memory");
            }
            if (p.counter) {
                tile = __shfl_sync(0xffffffffu, nxt, 0);
            } else {
                tile += gridDim.x;
                bp = ((bp | ~p.fmask) + p.dstride) & p.fmask;
            }
        }
    } else if (warp < kLoadWarps) {
        // ---------------- converters: thread j = 32 (w & 3) + lane, t in [32 (w >> 2), +32)
        const int q = warp & 3, th = warp >> 2;
        const int j = 32 * q + lane;
        const bool pf = PERM && ((lane >> 3) & 1);   // this lane reads t ^ (1 << PT)
        uint32_t phi = pf ? 1u << (PERM ? PT & 7 : 0) : 0u;
        if (PT == kPermMulti) {
            phi = 0;
            for (int b = 0; b < 4; b++)
                if (p.lane_t[b] >= 0 && ((lane >> b) & 1)) phi |= 1u << p.lane_t[b];
        }
        // cube index of (t = 32 th + (u ^ phi), j) = base ^ cube_t(u) with cube_t linear in u
        uint32_t base = 0;
        for (int k = 0; k < 7; k++)
            if ((j >> k) & 1) base |= 1u << p.jcube[k];
        if (th) base |= 1u << p.tcube[5];
        uint32_t R[5];
#pragma unroll
        for (int i = 0; i < 5; i++) {
            R[i] = 1u << p.tcube[i];
            if (PERM && ((phi >> i) & 1)) base ^= R[i];
        }
        for (uint64_t it = 0;; it++) {
            const int slot = it & 1, b = it & 1;
            mbar_wait(&rfull[slot], (it >> 1) & 1);
            if (tring[it % kTRing] == kTileEnd) {   // end: hand the MMA warp its last phase
                mbar_wait(&aempty[b], ((it >> 1) & 1) ^ 1);
                mbar_arrive(&afull[b]);
                break;
            }
            const float2* rb = raw + (size_t)slot * 8192;
            float2 v[32];   // v[u] = x(32 th + (u ^ phi), j)
            float mx = 0.f;
            if (PT == kRow) {   // row j = 128 (t >> 4) + j of 128 B, 16-B chunk (t & 15) / 2 ^ (j & 7)
                const uint8_t* sb = reinterpret_cast<const uint8_t*>(rb);
#pragma unroll
                for (int u2 = 0; u2 < 16; u2++) {
                    const int t = 32 * th + 2 * u2;
                    const uint32_t rho = (uint32_t)j + 128u * (uint32_t)(t >> 4);
                    const float4 w = *reinterpret_cast<const float4*>(sb + rho * 128 + (((uint32_t)((t & 15) >> 1) ^ (rho & 7)) << 4));
                    v[2 * u2] = make_float2(w.x, w.y);
                    v[2 * u2 + 1] = make_float2(w.z, w.w);
                    mx = absmax2(absmax2(mx, v[2 * u2]), v[2 * u2 + 1]);
                }
            }
            uint32_t ci = base;
            // keep the 32 addresses out of registers across tiles: recomputing them costs one XOR
            // each, hoisting them out of the loop spills (local-memory traffic every tile)
            asm volatile("" : "+r"(ci));
#pragma unroll
            for (int g = 0; g < 32 && PT != kRow; g++) {   // Gray-code walk of u: one XOR per element
                const int u = g ^ (g >> 1);
                if (g) ci ^= R[(g & 1) ? 0 : (g & 2) ? 1 : (g & 4) ? 2 : (g & 8) ? 3 : 4];
                v[u] = rb[ci];
                mx = absmax2(mx, v[u]);
            }
            mbar_arrive(&rempty[slot]);
            // column max over the two threads of column j (warps q and q + 4), as K9
            const int cb = (int)(it % 3);
            atomicMax(&cmax[cb * 128 + j], __float_as_int(mx));
            asm volatile("bar.sync 2, 256;" ::: "memory");
            const int E = col_exponent(cmax[cb * 128 + j]);
            if (th == 0) cmax[((it + 2) % 3) * 128 + j] = 0;
            const float sc = pow2f(E);
            mbar_wait(&aempty[b], ((it >> 1) & 1) ^ 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            // E_j -> epilogue after the wait: buffer b was freed by the MMA of tile it-2, which
            // waited for the epilogue of tile it-3, so slot it % 4 (tile it-4) has been read
            const int es = (int)(it % kExpSlots);
            if (th == 0) {
                colexp[es * 128 + j] = (int8_t)E;
                mbar_arrive(&cready[es]);
            }
            // K order t + 64 c: word c < 32 packs re of t = 2c, 2c+1; word 32 + c the im parts.
            // Real parts first, then imaginary parts (keeps 32 packed words live, not 64).
            const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + 128 * b + 16 * th;
#pragma unroll
            for (int c = 0; c < 2; c++) {
                uint32_t hw[16], lw[16];
#pragma unroll
                for (int u = 0; u < 16; u++) {
                    const float x0 = (c ? v[2 * u].y : v[2 * u].x) * sc, x1 = (c ? v[2 * u + 1].y : v[2 * u + 1].x) * sc;
                    split_exact_h2(x0, x1, hw[u], lw[u]);
                }
                if (PT == kPermMulti) {
                    unpermute_mask(hw, p.pmask, phi);
                    unpermute_mask(lw, p.pmask, phi);
                } else if (PERM) {
                    unpermute16<PT & 7>(hw, pf);
                    unpermute16<PT & 7>(lw, pf);
                }
                TMEM_ST16(ta + 32 * c, hw);        // hi: re words [16 th, +16), im words [32 + 16 th, +16)
                TMEM_ST16(ta + 64 + 32 * c, lw);   // lo
            }
            asm volatile("tcgen05.wait::st.sync.aligned;");
            asm volatile("tcgen05.fence::before_thread_sync;");
            mbar_arrive(&afull[b]);
        }
    } else if (warp == kMmaWarp) {
        // ---------------- MMA issuer: M = 128 (j), N = 64 per half (n = 2 t_o + c_o in [64 h, +64)),
        // K = 16 per step.  D is split by output half: the epilogue drains half 0 while half 1
        // is computed, and half 0 of the next tile starts as soon as its columns are read, so
        // the MMAs overlap the TMEM reads (64 B/cycle: 2048 cycles per tile, the longest stage)
        // instead of alternating with them.  Each output's K order is unchanged.
        constexpr int NH = RCS_K12_NSPLIT ? 2 : 1;   // 1: one N = 128 group (both halves at once)
        const uint32_t idesc = (1u << 4) | ((uint32_t)((128 / NH) >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const uint64_t bh0 = bdesc(su32(mat)), bl0 = bdesc(su32(mat + kTMat / 2));
        for (uint64_t it = 0;; it++) {
            const int b = it & 1;
            mbar_wait(&afull[b], (it >> 1) & 1);
            mbar_wait(&dempty[0], (it & 1) ^ 1);
            if (NH == 1) mbar_wait(&dempty[1], (it & 1) ^ 1);
            if (tring[it % kTRing] == kTileEnd) {   // end: hand the epilogue its last phase
                if (lane == 0) mbar_arrive(&dfull[0]);
                break;
            }
            asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
            for (int h = 0; h < NH; h++) {
                if (h) {
                    mbar_wait(&dempty[1], (it & 1) ^ 1);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                }
                if (lane == 0) {
                    const uint32_t dc = tmem + 256 + 64 * h, dm = tmem + 384 + 64 * h;
                    const uint32_t xh = tmem + 128 * b, xl = xh + 64;   // state hi / lo (A)
                    const uint64_t bh = bh0 + 1024 * h, bl = bl0 + 1024 * h;   // + 64 n rows (16 KB)
                    // cross terms (x_hi u_lo, x_lo u_hi) -> acc 0; main x_hi u_hi (exact) -> acc 1
                    MMA_F16(dc, xh, bl, idesc, 0);
                    MMA_F16(dc, xl, bh, idesc, 1);
#pragma unroll
                    for (int ks = 1; ks < 8; ks++) {
                        MMA_F16(dc, xh + ks * 8, bl + ks * 16, idesc, 1);
                        MMA_F16(dc, xl + ks * 8, bh + ks * 16, idesc, 1);
                    }
                    MMA_F16(dm, xh, bh, idesc, 0);
#pragma unroll
                    for (int ks = 1; ks < 8; ks++) MMA_F16(dm, xh + ks * 8, bh + ks * 16, idesc, 1);
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                        su32(&dfull[h])));
                    if (NH == 1)
                        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                            su32(&dfull[1])));
                    if (h == NH - 1)
                        asm volatile(
                            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                su32(&aempty[b])));
                }
                __syncwarp();
            }
        }
    } else if (warp >= kEpiWarp0 && warp < kEpiWarp0 + 4) {
        // ---------------- epilogue: lane quarter q holds columns j = 32 q + lane
        const int q = warp & 3;
        const int j = 32 * q + lane;
        uint64_t offj = 0;
        for (int k = 0; k < 7; k++)
            if ((j >> k) & 1) offj |= 1ull << p.jpos[k];
        for (uint64_t it = 0;; it++) {
            const int es = (int)(it % kExpSlots);
            mbar_wait(&dfull[0], it & 1);
            // the end marker is visible here (the MMA warp's plain arrive releases it); a tile's
            // base is guaranteed visible after cready (the converters read it after rfull)
            if (tring[it % kTRing] == kTileEnd) break;
            mbar_wait(&cready[es], (uint32_t)((it / kExpSlots) & 1));
            const uint64_t tb = tring[it % kTRing];
            const float cf = pow2f(-(int)colexp[es * 128 + j]);   // 2^-E_j (read before releasing D)
            asm volatile("tcgen05.fence::after_thread_sync;");
            float2* dst = p.amps + (tb | offj);
            const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + 256;
            const int tile_c = (int)(tb >> 13);   // kRow: tile coordinate of the store map
            // Four chunks of 32 D columns (16 target combinations, re/im).  The next chunk's TMEM
            // loads are issued before this chunk's stores, so the stores overlap the TMEM reads
            // (the epilogue's longest part: 64 B/cycle); two register sets alternate.
            uint32_t a0[32], a1[32], b0[32], b1[32];
            TMEM_LD32(ta, a0);
            TMEM_LD32M(ta + 128, a1);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            REG_FENCE32(a0);
            REG_FENCE32(a1);
            auto chunk = [&](const int s4, uint32_t(&x0)[32], const uint32_t(&x1)[32], uint32_t(&y0)[32],
                             uint32_t(&y1)[32]) {
#pragma unroll
                for (int c = 0; c < 32; c += 2) {   // in place: x0 <- ((cross + main) 2^-E_j) 2^-F_t
                    const float rf = rowfac[16 * s4 + c / 2];
                    asm("{\n.reg .b64 x, y, u, v;\n"
                        "mov.b64 x, {%0, %1};\nmov.b64 y, {%2, %3};\nmov.b64 u, {%4, %4};\nmov.b64 v, {%5, %5};\n"
                        "add.rn.f32x2 x, x, y;\nmul.rn.f32x2 x, x, u;\nmul.rn.f32x2 x, x, v;\n"
                        "mov.b64 {%0, %1}, x;\n}"
                        : "+r"(x0[c]), "+r"(x0[c + 1])
                        : "r"(x1[c]), "r"(x1[c + 1]), "f"(cf), "f"(rf));
                }
                if (s4 & 1) {   // half s4 / 2 read: its D columns are free for the next tile
                    asm volatile("tcgen05.fence::before_thread_sync;");
                    mbar_arrive(&dempty[s4 >> 1]);
                }
                if (s4 < 3) {
                    if (s4 == 1) {
                        mbar_wait(&dfull[1], it & 1);
                        asm volatile("tcgen05.fence::after_thread_sync;");
                    }
                    TMEM_LD32M(ta + 32 * (s4 + 1), y0);
                    TMEM_LD32M(ta + 128 + 32 * (s4 + 1), y1);
                }
                if (PT == kRow) {   // two staging chunks of 8 t; a TMA store each (4-D map, 64-B swizzle)
#pragma unroll
                    for (int h8 = 0; h8 < 2; h8++) {
                        const int k8 = 2 * s4 + h8;
                        uint8_t* sg = smem + 2 * kTRaw + kTMat + (k8 & 1) * (kTRowStage / 2);
                        if (warp == kEpiWarp0 && lane == 0)   // the store issued two chunks ago has read sg
                            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                        asm volatile("bar.sync 3, 128;" ::: "memory");
#pragma unroll
                        for (int m = 0; m < 4; m++) {   // t pair (8 k8 + 2 m, +1) of column j
                            const int c = 2 * (8 * h8 + 2 * m);
                            *reinterpret_cast<float4*>(sg + j * 64 + (((uint32_t)m ^ ((uint32_t)(j >> 1) & 3)) << 4)) =
                                make_float4(__uint_as_float(x0[c]), __uint_as_float(x0[c + 1]), __uint_as_float(x0[c + 2]),
                                            __uint_as_float(x0[c + 3]));
                        }
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        asm volatile("bar.sync 3, 128;" ::: "memory");
                        if (warp == kEpiWarp0 && lane == 0) {
                            asm volatile(
                                "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(
                                    reinterpret_cast<uint64_t>(&p.tmap_st)),
                                "r"(0), "r"(0), "r"(k8), "r"(tile_c), "r"(su32(sg))
                                : "memory");
                            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                        }
                    }
                } else {
#pragma unroll
                    for (int c = 0; c < 32; c += 2)
                        K12_STORE(dst + offt[16 * s4 + c / 2], make_float2(__uint_as_float(x0[c]), __uint_as_float(x0[c + 1])));
                }
                if (s4 < 3) {
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    REG_FENCE32(y0);
                    REG_FENCE32(y1);
                }
            };
            chunk(0, a0, a1, b0, b1);
            chunk(1, b0, b1, a0, a1);
            chunk(2, a0, a1, b0, b1);
            chunk(3, b0, b1, a0, a1);
        }
        if (PT == kRow && warp == kEpiWarp0 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

}  // namespace

size_t tc_matrix_words() { return 2 * 128 * 64 + 64; }

// A = [[U_re, -U_im], [U_im, U_re]] (rows interleaved: 2t = re, 2t+1 = im of output t).  Row
// pair t is scaled by 2^F_t, F_t = 10 - floor(log2 max_c |A[2t][c]|) (both rows hold the same
// magnitudes), so its entries lie below 2^11, and split into hi = rint(2^F_t A) -- an integer,
// exact in fp16 -- and lo = fp16(2^F_t A - hi), both from the fp64 product.  Packed 2 per word
// (k even in the low half): [hi rows 0..127][lo rows 0..127], 64 words per row, then F_t (64
// words, int).  The kernels unscale by 2^-F_t in the epilogue.
void tc_pack_matrix(const double* u_re_im /* 64x64 complex, row-major interleaved */, uint32_t* out) {
    auto entry = [&](int m, int kk) {
        const int t = m >> 1, col = kk & 63;
        const double ur = u_re_im[2 * (t * 64 + col)], ui = u_re_im[2 * (t * 64 + col) + 1];
        if (!(m & 1)) return kk < 64 ? ur : -ui;   // row 2t:   [U_re | -U_im]
        return kk < 64 ? ui : ur;                  // row 2t+1: [U_im |  U_re]
    };
    for (int t = 0; t < 64; t++) {
        double mx = 0.0;
        for (int kk = 0; kk < 128; kk++) mx = std::fmax(mx, std::fabs(entry(2 * t, kk)));
        const int F = mx > 0.0 ? 10 - std::ilogb(mx) : 0;
        out[(size_t)2 * 128 * 64 + t] = (uint32_t)F;
        for (int r = 0; r < 2; r++) {
            const int m = 2 * t + r;
            for (int k = 0; k < 128; k += 2) {
                uint16_t h[2], l[2];
                for (int u = 0; u < 2; u++) {
                    const double xs = std::ldexp(entry(m, k + u), F);
                    const double hi = std::nearbyint(xs);   // |hi| <= 2^11: exact in fp16
                    h[u] = __half_as_ushort(__float2half_rn((float)hi));
                    l[u] = __half_as_ushort(__double2half(xs - hi));
                }
                out[(size_t)m * 64 + k / 2] = (uint32_t)h[0] | ((uint32_t)h[1] << 16);
                out[(size_t)128 * 64 + (size_t)m * 64 + k / 2] = (uint32_t)l[0] | ((uint32_t)l[1] << 16);
            }
        }
    }
}

uint64_t tc_reserved_mask(int nl, const int* pos) {
    uint64_t tmask = 0;
    for (int i = 0; i < 6; i++) tmask |= 1ull << pos[i];
    uint64_t m = tmask;
    int nj = 0, r = -1;
    for (int b = 0; b < nl; b++) {
        if ((tmask >> b) & 1) continue;
        if (nj < 6) { m |= 1ull << b; nj++; continue; }
        r = b;
        break;
    }
    if (r >= 0) m |= 1ull << r;
    return m;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link); nullptr if
// unavailable (the launcher then keeps the bulk copies)
using TmapEncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static TmapEncodeFn tmap_encoder() {
    static TmapEncodeFn fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return (TmapEncodeFn) nullptr;
        return reinterpret_cast<TmapEncodeFn>(f);
    }();
    return fn;
}

// the 5-D tensor map of a K12 tile whose runs are 2^r <= 256 amplitudes (TcTArgs::nreq); false:
// not expressible (the launcher keeps one bulk copy per run)
static bool tct_tensor_map(TcTArgs& p, int nl) {
    TmapEncodeFn enc = tmap_encoder();
    if (!enc || p.r > 8 || nl - p.r > 31) return false;
    // groups of consecutive run positions, ascending
    int gp[6], gm[6], ng = 0;
    for (int i = 0; i < p.nrun_pos; i++) {
        if (ng && p.run_pos[i] == gp[ng - 1] + gm[ng - 1]) {
            gm[ng - 1]++;
        } else {
            gp[ng] = p.run_pos[i];
            gm[ng++] = 1;
        }
    }
    // dim 1 (box 1) carries the tile base, so the strides ascend; unused dims: extent 1
    cuuint64_t dim[5] = {1ull << p.r, 1ull << (nl - p.r), 1, 1, 1};
    cuuint64_t stride[4] = {8ull << p.r, 0, 0, 0};   // bytes, dims 1..4
    cuuint32_t box[5] = {1u << p.r, 1, 1, 1, 1};
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    const int nd = ng < 3 ? ng : 3;
    int covered = 0;
    for (int d = 0; d < 3; d++) {
        if (d < nd) {
            dim[2 + d] = 1ull << gm[d];
            stride[1 + d] = 8ull << gp[d];
            box[2 + d] = 1u << gm[d];
            covered += gm[d];
        } else {
            stride[1 + d] = stride[d];
        }
    }
    const int rest = p.nrun_pos - covered;   // run bits enumerated by requests
    if (rest > 3) return false;
    p.nreq = 1 << rest;
    p.req_bytes = kTRaw >> rest;
    int rp[6], nrp = 0;
    for (int d = nd; d < ng; d++)
        for (int b = 0; b < gm[d]; b++) rp[nrp++] = gp[d] + b;
    for (int u = 0; u < p.nreq; u++) {
        int off = 0;
        for (int b = 0; b < nrp; b++)
            if ((u >> b) & 1) off += 1 << (rp[b] - p.r);
        p.treq[u] = off;
    }
    return enc(&p.tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, p.amps, dim, stride, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// kRow tensor maps (load: 128-B swizzle, box 16 t x 128 j x 4 t-quads; store: 64-B swizzle, box
// 8 t x 128 j): dims are the state's bit fields (t bits 0..3 or 0..2 contiguous, j = positions
// 6..12, the remaining t bits, the tile = positions 13..), so the strides do not ascend; false if
// the encoder refuses (the block then runs on K9)
static bool row_tensor_maps(TcTArgs& p, int nl) {
    TmapEncodeFn enc = tmap_encoder();
    if (!enc || nl < 13 || nl - 13 > 31) return false;
    const cuuint64_t ntile = 1ull << (nl - 13);
    cuuint32_t estr[4] = {1, 1, 1, 1};
    cuuint64_t ld_dim[4] = {16, 128, 4, ntile}, ld_str[3] = {512, 128, 65536};
    cuuint32_t ld_box[4] = {16, 128, 4, 1};
    cuuint64_t st_dim[4] = {8, 128, 8, ntile}, st_str[3] = {512, 64, 65536};
    cuuint32_t st_box[4] = {8, 128, 1, 1};
    return enc(&p.tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, p.amps, ld_dim, ld_str, ld_box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS &&
           enc(&p.tmap_st, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, p.amps, st_dim, st_str, st_box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static bool is_row_layout(int nl, const int* pos) {
    if (nl < 13) return false;
    for (int i = 0; i < 6; i++)
        if (pos[i] != i) return false;
    return true;
}

// K12 launcher: any target layout, n_local >= 13 (+ chunk bits)
static cudaError_t gate_pass_tct(float2* amps, int nl, const int* pos, const uint32_t* d_a, int num_sms,
                                 cudaStream_t st, const int* fix, int nfix, uint64_t fixval, unsigned* counter,
                                 bool bulk_runs) {
    TcTArgs p{};
    p.amps = amps;
    p.a = d_a;
    p.counter = counter;
    if (nl < 13 + nfix || nfix < 0 || nfix > 4) return cudaErrorInvalidValue;
    p.ntiles = 1ull << (nl - 13 - nfix);
    uint64_t tmask = 0;
    for (int i = 0; i < 6; i++) {
        if (pos[i] < 0 || pos[i] >= nl || ((tmask >> pos[i]) & 1)) return cudaErrorInvalidValue;
        p.pos[i] = pos[i];
        tmask |= 1ull << pos[i];
    }
    uint64_t cube = tmask;
    for (int b = 0, k = 0; b < nl && k < 7; b++)
        if (!((tmask >> b) & 1)) {
            p.jpos[k++] = b;
            cube |= 1ull << b;
        }
    int rank[64];
    int nc = 0;
    for (int b = 0; b < nl; b++)
        if ((cube >> b) & 1) rank[b] = nc++;
    if (nc != 13) return cudaErrorInvalidValue;
    for (int i = 0; i < 6; i++) p.tcube[i] = rank[pos[i]];
    for (int k = 0; k < 7; k++) p.jcube[k] = rank[p.jpos[k]];
    p.r = 0;
    while (p.r < 13 && ((cube >> p.r) & 1)) p.r++;
    if (p.r < 7) return cudaErrorInvalidValue;
    p.nrun_pos = 0;
    for (int b = p.r; b < nl; b++)
        if ((cube >> b) & 1) p.run_pos[p.nrun_pos++] = b;
    if (p.nrun_pos != 13 - p.r) return cudaErrorInvalidValue;
    p.nreq = 0;
    if (!bulk_runs && !tct_tensor_map(p, nl)) p.nreq = 0;
    // bank-conflict-free converter reads: with one target at cube rank < 4, column bit 3 is
    // displaced to rank 4 and the lanes with it set read t ^ (that target's bit); t bit 5 (the
    // converter half) must not be it.  More low targets: K9 (tc_uses_k12).
    p.phi_t = -1;
    int nlow = 0, lowt[6];
    for (int i = 0; i < 6; i++)
        if (p.tcube[i] < 4) {
            if (i >= 5) return cudaErrorInvalidValue;
            lowt[nlow++] = i;
        }
    if (nlow == 1) p.phi_t = lowt[0];
    if (nlow >= 2) {   // lane bits 4 - nlow .. 3 (column bits at ranks >= 4) -> the low t bits
        p.phi_t = kPermMulti;
        p.pmask = 0;
        for (int b = 0; b < 4; b++) p.lane_t[b] = -1;
        for (int m = 0; m < nlow; m++) {
            p.lane_t[4 - nlow + m] = lowt[m];
            p.pmask |= 1 << lowt[m];
        }
    }
    const bool row = is_row_layout(nl, pos);   // also chunked (pipelined remaps): the chunk bits are >= 13
    if (row) {
        if (!row_tensor_maps(p, nl)) return cudaErrorNotSupported;   // caller falls back to K9
        p.phi_t = kRow;
        p.nreq = 0;
    }
    const bool perm = p.phi_t >= 0;
    if (perm && !row && p.jcube[4 - nlow] < 4) return cudaErrorInvalidValue;
    uint64_t insmask = cube, fixmask = 0;
    for (int i = 0; i < nfix; i++) {
        if (fix[i] < 0 || fix[i] >= nl || ((insmask >> fix[i]) & 1)) return cudaErrorInvalidValue;
        fixmask |= 1ull << fix[i];
    }
    if (fixval & ~fixmask) return cudaErrorInvalidValue;
    p.fixval = fixval;
    insmask |= fixmask;
    p.nins = 0;
    for (int b = 0; b < nl; b++)
        if ((insmask >> b) & 1) p.ins[p.nins++] = b;
    if (p.nins != 13 + nfix) return cudaErrorInvalidValue;
    const uint64_t grid = p.ntiles < (uint64_t)num_sms ? p.ntiles : (uint64_t)num_sms;
    p.fmask = ~insmask & ((1ull << nl) - 1);
    uint64_t v = grid, d = 0;
    for (int b = 0; b < 64 && v; b++)
        if ((p.fmask >> b) & 1) {
            if (v & 1) d |= 1ull << b;
            v >>= 1;
        }
    p.dstride = d;
    // the attribute is per device (context): set it before every launch (cheap)
    void (*kern)(TcTArgs) = nullptr;
    switch (p.phi_t) {
        case -1: kern = k_pass_tct<-1>; break;
        case 0: kern = k_pass_tct<0>; break;
        case 1: kern = k_pass_tct<1>; break;
        case 2: kern = k_pass_tct<2>; break;
        case 3: kern = k_pass_tct<3>; break;
        case 4: kern = k_pass_tct<4>; break;
        case kPermMulti: kern = k_pass_tct<kPermMulti>; break;
        case kRow: kern = k_pass_tct<kRow>; break;
        default: return cudaErrorInvalidValue;
    }
    const uint32_t smem_bytes = kTSmem + (row ? kTRowStage : 0);
    (void)perm;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes);
    if (e != cudaSuccess) return e;
    if (counter && (e = cudaMemsetAsync(counter, 0, sizeof(unsigned), st)) != cudaSuccess) return e;
    count_launch();
    kern<<<(unsigned)grid, kThreadsTC, smem_bytes, st>>>(p);
    return cudaGetLastError();
}

bool tc_uses_k12(int nl, const int* pos) {
    // K12 for at most 2 targets in positions 0..3 (kPermMulti for 2) unless the converter-half
    // bit (matrix bit 5) sits there (K12 cannot flip it).  Measured per pass on one box
    // (profiles/r02/k12multi): 2 low targets 15.1-17.0 ms vs K9 17.3-17.6 (C3 size); 3-4 low
    // targets 31-44 ms vs K9 17.0-17.2 -- the epilogue's stores then scatter over 32 sectors
    int low = 0;
    for (int i = 0; i < 6; i++) low += pos[i] < 4;
    return nl >= 13 && ((pos[5] >= 4 && low <= 2) || is_row_layout(nl, pos));
}

cudaError_t gate_pass_tc(float2* amps, int nl, const int* pos, const uint32_t* d_a, int num_sms, cudaStream_t st,
                         const int* fix, int nfix, uint64_t fixval, int tc_flags, unsigned* tile_counter) {
    if (!(tc_flags & kTcForceK9) && tc_uses_k12(nl, pos) && !(is_row_layout(nl, pos) && (tc_flags & kTcNoRow))) {
        const cudaError_t e = gate_pass_tct(amps, nl, pos, d_a, num_sms, st, fix, nfix, fixval, tile_counter,
                                            (tc_flags & kTcBulkRuns) != 0);
        if (e != cudaErrorNotSupported) return e;
        cudaGetLastError();   // kRow maps refused by the encoder: K9 below
    }
    if (nl < 12 + nfix || nfix < 0 || nfix > 4) return cudaErrorInvalidValue;
    TcArgs p{};
    p.amps = amps;
    p.a = d_a;
    p.ntiles = 1ull << (nl - 12 - nfix);
    uint64_t tmask = 0;
    for (int i = 0; i < 6; i++) {
        p.pos[i] = pos[i];
        tmask |= 1ull << pos[i];
    }
    int nj = 0;
    for (int b = 0; b < nl && nj < 6; b++)
        if (!((tmask >> b) & 1)) p.jpos[nj++] = b;
    if (nj != 6) return cudaErrorInvalidValue;
    // sub-cube bits = targets U column bits, ascending
    int all[12], na = 0;
    for (int b = 0; b < nl && na < 12; b++) {
        bool in = (tmask >> b) & 1;
        for (int i = 0; i < 6; i++) in = in || p.jpos[i] == b;
        if (in) all[na++] = b;
    }
    if (na != 12) return cudaErrorInvalidValue;
    for (int i = 0; i < 12; i++) p.sub[i] = all[i];
    p.r = 0;
    while (p.r < 12 && p.sub[p.r] == p.r) p.r++;   // >= 6: the 6 lowest non-targets are in the cube
    // fixed (chunk) bits: outside the sub-cube and not the first non-cube bit (tile pairs)
    uint64_t insmask = 0, fixmask = 0;
    for (int i = 0; i < 12; i++) insmask |= 1ull << p.sub[i];
    for (int i = 0; i < nfix; i++) {
        if (fix[i] < 0 || fix[i] >= nl || fix[i] == p.r || ((insmask >> fix[i]) & 1)) return cudaErrorInvalidValue;
        insmask |= 1ull << fix[i];
        fixmask |= 1ull << fix[i];
    }
    if (fixval & ~fixmask) return cudaErrorInvalidValue;
    p.fixval = fixval;
    p.nins = 0;
    for (int b = 0; b < nl; b++)
        if ((insmask >> b) & 1) p.ins[p.nins++] = b;
    p.pair = p.ntiles >= 2 ? 2 : 1;                // tile bit 0 = index bit r (first non-cube bit)
    for (int i = 0; i < 32; i++) {                 // epilogue store offsets of sub-cube index 128 i
        const int sidx = 128 * i;
        int t = 0, jj = 0;
        uint64_t go = 0;
        for (int b = 0; b < 12; b++) {
            if (!((sidx >> b) & 1)) continue;
            go |= 1ull << p.sub[b];
            for (int k = 0; k < 6; k++) {
                if (p.pos[k] == p.sub[b]) t |= 1 << k;
                if (p.jpos[k] == p.sub[b]) jj |= 1 << k;
            }
        }
        p.sto[i] = t * kPitchF;
        p.sxj[i] = jj;              // XORed with g(t) below, once the swizzle is known
        p.sgo[i] = go;
    }
    // bank conflicts of the converters' reads: with a targets among the 4 lowest sub-cube ranks,
    // a lane bits (column bits 0..3) land on ranks >= 4; those lane bits drive the octet
    // rotation (t bits 0..2) and t bit 3.  Pinning makes the low targets t bits 0..a-1; any
    // other case keeps the plain lane & 7 rotation.
    int low_targets = 0, lowt[6], disp[4], nd = 0;
    for (int i = 0; i < 6; i++) {
        int rk = 0;
        while (p.sub[rk] != p.pos[i]) rk++;
        if (rk < 4) lowt[low_targets++] = i;
    }
    for (int k = 0; k < 4; k++) {
        int rk = 0;
        while (p.sub[rk] != p.jpos[k]) rk++;
        if (rk >= 4) disp[nd++] = k;
    }
    bool lowest = nd == low_targets;
    for (int m = 0; m < low_targets; m++) lowest = lowest && lowt[m] == m;
    for (int m = 0; m < 3; m++) p.rot_lane[m] = lowest ? (m < low_targets ? disp[m] : -1) : m;
    p.to_lane = (lowest && low_targets == 4) ? disp[3] : -1;
    // staging swizzle: the half-warp's memory-order reads vary the a low targets (t bits 0..a-1)
    // and the 4-a lowest columns (j bits 0..3-a); rotating t's low 4 bits left by 4-a puts the
    // targets on the column bits the reads do not vary (and keeps the 16 rows of a warp's writes
    // on 16 distinct column slots)
    p.gsh = lowest ? (4 - (low_targets < 4 ? low_targets : 4)) & 3 : 0;
    for (int i = 0; i < 32; i++) {
        const int t = p.sto[i] / kPitchF, x = t & 15;
        p.sxj[i] ^= ((x << p.gsh) | (x >> (4 - p.gsh))) & 15;
    }
    const uint64_t units = p.ntiles / p.pair;
    const uint64_t grid = units < (uint64_t)num_sms ? units : (uint64_t)num_sms;
    if (grid == 0) return cudaSuccess;
    p.fmask = ~insmask & ((nl >= 64) ? ~0ull : ((1ull << nl) - 1));
    {   // pdep(grid * pair, fmask)
        uint64_t v = grid * (uint64_t)p.pair, d = 0;
        for (int b = 0; b < 64 && v; b++)
            if ((p.fmask >> b) & 1) {
                if (v & 1) d |= 1ull << b;
                v >>= 1;
            }
        p.dstride = d;
    }
    const bool rot = lowest ? low_targets >= 1 : low_targets >= 2;
    cudaError_t e = rot ? cudaFuncSetAttribute(k_pass_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes)
                        : cudaFuncSetAttribute(k_pass_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
    if (e != cudaSuccess) return e;
    count_launch();
    if (rot)
        k_pass_tc<true><<<(unsigned)grid, kThreadsTC, kSmemBytes, st>>>(p);
    else
        k_pass_tc<false><<<(unsigned)grid, kThreadsTC, kSmemBytes, st>>>(p);
    return cudaGetLastError();
}


}  // namespace dev
}  // namespace rcs
