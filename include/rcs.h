/*
 * rcs.h -- C ABI of the B200-native random-circuit-sampling (RCS) hot path.
 *
 * The calls follow the paper's statement of the problem (§3.2, lines 34-39):
 *   "circuits are initially constructed from Google's QASM-format files"   -> rcs_circuit_load_qasm
 *   "construct the complete quantum state from the circuit definition"      -> rcs_state_build
 *   "performs 2.5x10^6/N measurement shots"                                  -> rcs_sample
 *   "calculates the linear cross-entropy benchmarking (XEB) score"           -> rcs_xeb
 * with the conventions, operations and errors of SPEC.md (S:42-50 parse, S:122-126 build,
 * S:138-140 probability, S:244-247 sample, S:378-380 XEB) and the readings listed in
 * DESIGN.md §3 (V1-V15).  All arithmetic runs in this library's sm_100a CUDA kernels.
 *
 * General rules
 *  - Every function returns rcs_status (0 = RCS_OK) and never throws across the ABI.
 *  - On error, `err` (if non-NULL) receives code, message and, for parse errors, the
 *    1-based line/column; outputs are left untouched.
 *  - Ownership: the CALLER owns every buffer passed in (device amplitude and scratch
 *    buffers typically come from torch.empty on the context's device).  The library owns
 *    only the opaque host handles it returns, small device plan buffers and a bounded
 *    device staging area inside each rcs_state, all released by the matching *_free.
 *  - Synchrony: calls are stream-ordered on the context's CUDA stream and return after
 *    that stream has drained, so results are ready and timings are explicit.
 *  - Multi-GPU (SPMD): with world > 1 every rank makes the same calls in the same order;
 *    build, norm, sample, probabilities and XEB are collectives over the context's NCCL
 *    communicator (NVLink / NVSwitch).
 *  - Bit order (reading V1): amplitude index i encodes qubit q as bit q
 *    (qubit 0 = least significant); bitstrings are uint64 with the same encoding, n <= 63.
 *  - Amplitudes are complex64, interleaved (re, im) float32 -- the layout of
 *    torch.complex64.  A rank's shard holds 2^(n-g) amplitudes, g = log2(world).
 */
#ifndef RCS_H
#define RCS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    RCS_OK = 0,
    RCS_ERR_PARSE = 1,          /* QASM syntax error; err->line/col set          */
    RCS_ERR_UNKNOWN_GATE = 2,   /* gate name outside the dialect                  */
    RCS_ERR_QUBIT_RANGE = 3,    /* qubit index >= declared qreg size                          */
    RCS_ERR_ARITY = 4,          /* wrong parameter / qubit count, or a repeated qubit         */
    RCS_ERR_MEMORY = 5,         /* buffer too small; err->bytes_required set     */
    RCS_ERR_NORM = 6,           /* |T - 1| > 1e-5 at sampling (BASELINE tolerance) */
    RCS_ERR_SIZE = 7,           /* bitstring >= 2^n                              */
    RCS_ERR_ARG = 8,            /* invalid argument / unsupported configuration               */
    RCS_ERR_CUDA = 9,           /* CUDA runtime error (message has cudaGetErrorString)        */
    RCS_ERR_NCCL = 10,          /* NCCL error (message has ncclGetErrorString)                */
    RCS_ERR_IO = 11,            /* file open/read/write/rename failed, or an existing output  */
    RCS_ERR_FORMAT = 12,        /* snapshot: bad magic, version, header or truncated payload  */
    RCS_ERR_DIGEST = 13         /* snapshot: payload SHA-256 differs from the header's digest */
} rcs_status;

typedef struct {
    int code;                   /* rcs_status */
    int line, col;              /* 1-based position of a parse error, else 0 */
    uint64_t bytes_required;    /* set with RCS_ERR_MEMORY */
    char msg[256];
} rcs_error;

typedef struct rcs_circuit rcs_circuit;   /* parsed circuit: host, immutable, thread-safe to share */
typedef struct rcs_context rcs_context;   /* one per rank: device, stream, NCCL communicator */
typedef struct rcs_state rcs_state;       /* small host handle describing a built state */
typedef struct rcs_plan rcs_plan;         /* host-only execution plan (fused passes + remaps) */

/* gate kinds: */
enum { RCS_GATE_SX = 0, RCS_GATE_SY = 1, RCS_GATE_SW = 2, RCS_GATE_RZ = 3, RCS_GATE_FSIM = 4 };

typedef struct {
    int n_qubits, n_moments, n_gates, n_measure;
    int n_sx, n_sy, n_sw, n_rz, n_fsim;   /* per-kind counts */
} rcs_circuit_counts;

/* remap execution (rcs_build_opts.remap_mode) */
enum {
    RCS_REMAP_AUTO = 0,      /* world > 1: in-place NVLink peer swaps over CUDA-IPC mappings when every
                                rank maps every peer (agreed over all ranks, world <= 8), else NCCL
                                grouped send/recv; world 1 + virtual_global: in-device bit swaps   */
    RCS_REMAP_NCCL = 1,      /* world > 1: always NCCL send/recv through the staging area           */
    RCS_REMAP_LOOPBACK = 2   /* world 1 + virtual_global g: the buffer is 2^g virtual ranks' shards
                                (consecutive regions) and every remap runs through the NVLink
                                peer-swap kernel and the pipelined remap path, peers = the other
                                regions (exercises the multi-GPU data path on one GPU)             */
};

typedef struct {
    int fuse_k;              /* max qubits per fused dense block, 1..6; 6-qubit blocks run on the
                                tensor cores (needs n-g >= 12).  0 -> 6 if n-g >= 12, else 4        */
    int block_bits;          /* sampling block: 2^b amplitudes per fp64 CDF entry (0 -> 6)      */
    int virtual_global;      /* world == 1 only: treat the top g qubits as global and run every
                                remap on this device (bit swaps, or peer swaps with LOOPBACK)    */
    int timing;              /* 1: record a CUDA-event pair around every pass / remap             */
    uint64_t staging_bytes;  /* bound of the NCCL remap staging area (0 -> 256 MiB)              */
    int keep_layout;         /* 1: skip the final layout restore (remaps / bit swaps that only
                                bring the qubits back to canonical positions).  Sampling, XEB and
                                probabilities work on the kept layout (logical CDF over all
                                ranks); rcs_state_copy_out / rcs_snapshot_save then need
                                rcs_state_canonicalize first (RCS_ERR_ARG otherwise).  The
                                scratch grows to 2 x 8 x 2^(n-6) B when world > 1.           */
    int remap_mode;          /* RCS_REMAP_* (0 = AUTO)                                             */
    int overlap;             /* pipelined remaps: a [TC pass] -> REMAP -> [TC pass]
                                group runs in 2^overlap_chunks chunks, swaps of chunk c overlapping
                                passes of other chunks.  0 = on (default), -1 = off                */
    int overlap_chunks;      /* log2 chunks, 1..4 (0 -> 2)                                         */
    int overlap_sms;         /* SMs left to the swaps while passes run (0 -> 32 at world 2, 16 at
                                world >= 4 and in loopback)                                        */
    int tc_kernel;           /* 0: the transposed kernel K12 when n_local >= 13 and at most two
                                targets sit in positions 0..3 (not matrix bit 5), or the block is
                                positions 0..5 in order (K12's row variant); K9
                                otherwise -- a function of the block: P-invariant; 1: K9 only
                                (tests, comparisons); 2: as 0 without the row variant            */
    int overlap_passes;      /* pipelined remaps: how many tensor-core passes after the remap run
                                chunk by chunk behind its swaps (0 -> 3; 1 = the next pass only)  */
    int product_prefix;      /* 0: the leading fused blocks on pairwise disjoint qubits (they act on
                                |0...0>) are written as one product state by a write-only kernel
                                (init + those passes replaced); -1: run them as passes            */
    int tc_schedule;         /* K12 tiles: 0 = static round robin (blockIdx + k gridDim), 1 = dynamic
                                (a device counter hands tiles to the SMs as they free up; measured
                                5 % slower at C4, profiles/r02/tiles_ab.txt)                      */
    int tc_tma;              /* K12 loads: 0 = a tile whose contiguous runs are short (<= 256
                                amplitudes) is fetched by a few 5-D tensor-map TMA requests (many
                                runs each); -1 = one bulk copy per run                            */
} rcs_build_opts;

typedef struct {
    int n_passes;            /* fused dense gate passes (K1) executed on this rank              */
    int n_remaps;            /* global<->local qubit remaps (all-to-all exchanges)               */
    int n_swaps;             /* local bit-swap passes (final layout restore)                     */
    int fuse_k;
    double plan_ms;          /* host: fusion + remap planning                                    */
    double build_ms;         /* device: init .. final norm, CUDA events on the context stream    */
    double pass_ms;          /* timing=1: sum of gate-pass kernel times                          */
    double pass_ms_min, pass_ms_max;
    double remap_ms;         /* timing=1: sum of remap times (NVLink peer swap, or NCCL fallback);
                                for pipelined remaps the time not hidden behind pass chunks    */
    double blocksum_ms;      /* timing=1: block-sum + scan (sampling CDF) time                   */
    uint64_t pass_bytes;     /* algorithmic bytes of all gate passes on this rank (16 B/amp/pass) */
    uint64_t remap_bytes;    /* bytes this rank's remaps moved out of its shard (NVLink / NCCL)   */
    double norm;             /* sum |psi|^2 over all ranks                                       */
    int n_tc_passes;         /* of n_passes, 6-qubit passes run on the tensor cores (K9)          */
    double swap_ms;          /* timing=1: sum of local bit-swap (layout restore) pass times       */
    int layout_kept;         /* 1: the state is in a permuted (non-canonical) layout            */
    int n_pipelined;         /* remaps run as chunked peer swaps overlapped with the adjacent
                                tensor-core passes (rcs_build_opts.overlap)         */
    int n_peer_remaps;       /* remaps executed by the peer-swap kernel (NVLink or loopback)      */
    double remap_kernel_ms;  /* timing=1: device time of the remap data movement alone (peer-swap
                                kernels / NCCL send-recv, first start to last end per remap, also
                                when hidden behind pass chunks): NVLink GB/s = remap_bytes / it  */
    int n_prefix;            /* fused blocks written as a product state (not counted in n_passes;
                                pass_bytes counts their kernel as 8 B per amplitude, write only)  */
    double prefix_ms;        /* timing=1: device time of the product-state kernel                */
    uint64_t upload_bytes;   /* host -> device bytes this build copied (tensor-core operands and
                                product-state tables when not cached for this circuit, layout
                                tables)                                                          */
} rcs_build_report;

typedef struct {
    uint64_t shots;
    double total_prob;       /* T used for t_s = u_s * T (reading V13)                           */
    double sample_ms;        /* device time of the per-shot search + gather                       */
} rcs_sample_report;

typedef struct {
    int n_qubits;
    uint64_t shots;
    double F;                /* 2^n * mean p(x_s) - 1   (reading V14)                */
    double sigma;            /* 2^n * stdev(p, ddof=1) / sqrt(S)                                  */
    double mean_p;
    double fstar;            /* 2^n * sum_x p_x^2 - 1 of the built state (ideal-sampler XEB)      */
} rcs_xeb_report;

/* Plan inspection (host only, no GPU): one item per device step. */
enum { RCS_ITEM_PASS = 0, RCS_ITEM_REMAP = 1, RCS_ITEM_SWAP = 2 };
typedef struct {
    int type;                /* RCS_ITEM_*                                                        */
    int k;                   /* PASS: block width; REMAP/SWAP: number of position pairs           */
    int qubits[8];           /* PASS: logical qubits, matrix bit i <-> qubits[i] (ascending)      */
    int pos[8];              /* PASS: physical bit position of matrix bit i                       */
    int a[8], b[8];          /* REMAP: a = global position, b = local position (swapped pairwise);
                                SWAP: disjoint local position pairs swapped in one pass            */
    int n_gates;             /* PASS: source gates fused into this block                          */
} rcs_plan_item;

const char *rcs_status_string(int status);
/* Cumulative number of CUDA kernels this library has launched in this process (all
 * contexts); benchmarks difference it around a timed region. */
uint64_t rcs_kernel_launches(void);

/* ---- circuit (host) ------------------------------------------------------------------ */
/* Parse `len` bytes of QASM (dialect: DESIGN.md §3 V5). */
rcs_status rcs_circuit_load_qasm(const char *text, size_t len, rcs_circuit **out, rcs_error *err);
rcs_status rcs_circuit_stats(const rcs_circuit *c, rcs_circuit_counts *out);
/* Gate i in source order; q1 = -1 for 1-qubit gates; rz stores its angle in *phi. */
rcs_status rcs_circuit_gate(const rcs_circuit *c, int i, int *kind, int *q0, int *q1,
                            double *theta, double *phi, int *moment);
void rcs_circuit_free(rcs_circuit *c);

/* ---- plan (host) -------------------------------------------------------------------- */
/* Fuse the circuit into dense blocks of <= fuse_k qubits and schedule remaps for
 * n_global = log2(world) global qubits (BASELINE.json north_star).  The fusion is
 * independent of n_global. */
rcs_status rcs_plan_create(const rcs_circuit *c, int fuse_k, int n_global, rcs_plan **out, rcs_error *err);
rcs_status rcs_plan_summary(const rcs_plan *p, int *n_items, int *n_passes, int *n_remaps, int *n_swaps);
/* Product-state prefix: items [0, *n_prefix) are passes on pairwise disjoint qubits applied to
 * |0...0>; rcs_state_build writes their product state with one kernel (rcs_build_opts
 * product_prefix) -- a function of the fused blocks, independent of n_global. */
rcs_status rcs_plan_prefix(const rcs_plan *p, int *n_prefix);
/* matrix_out (may be NULL): 2 * 4^k doubles, row-major interleaved complex, fp64 product. */
rcs_status rcs_plan_item_get(const rcs_plan *p, int i, rcs_plan_item *out, double *matrix_out);
/* Layout bookkeeping of the plan (host): items [*restore_begin, n_items) only restore the
 * canonical layout (skipped by keep_layout); final_pos[q] (n entries, may be NULL) = physical
 * position of qubit q before them (>= n - n_global: a rank bit); initial_pos likewise at the
 * start (the global qubits may start permuted: |0...0> is permutation invariant). */
rcs_status rcs_plan_layout(const rcs_plan *p, int *restore_begin, int *final_pos, int *initial_pos);
void rcs_plan_free(rcs_plan *p);

/* ---- context ------------------------------------------------------------------------ */
/* NCCL bootstrap: rank 0 calls rcs_nccl_unique_id (128 bytes) and the caller broadcasts the
 * bytes to every rank (e.g. torch.distributed.broadcast_object_list). */
int rcs_nccl_unique_id_bytes(void);
rcs_status rcs_nccl_unique_id(void *out_bytes, rcs_error *err);
/* world must be a power of two; nccl_id is ignored (may be NULL) when world == 1.
 * cuda_stream: a cudaStream_t on `device` (NULL = legacy default stream). */
rcs_status rcs_context_create(int device, int rank, int world, const void *nccl_id,
                              void *cuda_stream, rcs_context **out, rcs_error *err);
void rcs_context_free(rcs_context *ctx);

/* ---- state -------------------------------------------------------------------------- */
/* Device scratch needed by rcs_state_build (fp64 block-CDF + remap staging). */
rcs_status rcs_state_scratch_bytes(const rcs_context *ctx, const rcs_circuit *c,
                                   const rcs_build_opts *opts, uint64_t *bytes);
/* Build psi = U_G ... U_1 |0...0> into the caller's device buffer d_amps
 * (2^(n-g) complex64 = amps_bytes; rank r holds logical indices [r 2^(n-g), (r+1) 2^(n-g))
 * on return, i.e. canonical order).  d_scratch must hold rcs_state_scratch_bytes; the state
 * keeps pointers to both buffers until rcs_state_free.  RCS_ERR_MEMORY (bytes_required) if a
 * buffer is too small. */
rcs_status rcs_state_build(rcs_context *ctx, const rcs_circuit *c, const rcs_build_opts *opts,
                           void *d_amps, uint64_t amps_bytes, void *d_scratch, uint64_t scratch_bytes,
                           rcs_state **out, rcs_build_report *rep, rcs_error *err);
/* Collective: run the deferred layout restore of a keep_layout build (no-op if canonical). */
rcs_status rcs_state_canonicalize(rcs_state *s, rcs_error *err);
/* Per-pass kernel times (ms) of the last build (timing=1), in plan order; *n = count. */
rcs_status rcs_state_pass_times(const rcs_state *s, float *ms, int cap, int *n);
rcs_status rcs_state_norm(const rcs_state *s, double *norm);          /* collective */
/* Copy `count` amplitudes starting at GLOBAL logical index `first` (must lie in this rank's
 * shard) to dst (host or device memory, complex64). */
rcs_status rcs_state_copy_out(const rcs_state *s, uint64_t first, uint64_t count, void *dst, rcs_error *err);
/* p_out[i] = |psi_{x[i]}|^2; x and p_out host or device; collective. */
rcs_status rcs_probabilities(const rcs_state *s, const uint64_t *x, uint64_t count, double *p_out,
                             rcs_error *err);
/* Draw `shots` bitstrings (readings V12/V13): u_s from SplitMix64(shot_seed) output
 * shot_offset+s+1, t_s = u_s T, x_s = min{x : C(x) > t_s}.  out_x (host or device, `shots`
 * entries in shot order) is filled on every rank.  Refuses |T - 1| > 1e-5 (RCS_ERR_NORM). */
rcs_status rcs_sample(rcs_state *s, uint64_t shots, uint64_t shot_seed, uint64_t shot_offset,
                      uint64_t *out_x, rcs_sample_report *rep, rcs_error *err);
/* Test hook: the same search with caller-supplied uniforms u[s] in [0, 1) (host or device). */
rcs_status rcs_sample_uniforms(rcs_state *s, const double *u, uint64_t shots, uint64_t *out_x,
                               rcs_sample_report *rep, rcs_error *err);
/* Linear XEB of bitstrings x (host or device) against this state. */
rcs_status rcs_xeb(const rcs_state *s, const uint64_t *x, uint64_t count, rcs_xeb_report *out, rcs_error *err);
void rcs_state_free(rcs_state *s);   /* frees the handle and its device plan/staging buffers */

/* ---- paper stages 2-3: state snapshot and independent sampler jobs -------
 * PAPER §3.2 l.37: "The generated quantum state ... is written to a shared file system in an
 * internal format optimized for fast read access"; l.38: "N CPU-only jobs, each of which
 * rebuilds the quantum state from the persisted state and performs 2.5x10^6/N measurement
 * shots ... Each job stores its output in a job-specific file".  File format = SPEC
 * snapshot-store (reading F3-1): 52-byte header {"RCSS", u32 version 1,
 * u32 n_qubits, u64 payload_bytes = 16 2^n, 32-byte SHA-256(payload)} then the amplitudes in
 * index order as little-endian float64 (re, im).  Single-rank states only (world == 1): the
 * paper's jobs are independent processes (RCS_ERR_ARG otherwise). */
/* SHA-256 (FIPS 180-4) of a host buffer; host-only, no device needed. */
rcs_status rcs_sha256(const void *data, uint64_t bytes, uint8_t digest[32]);
/* Write the state to `path` atomically (temp file + rename; an existing `path` is replaced,
 * the temp file is never left behind on error); complex64 amplitudes are widened exactly to
 * float64.  digest (may be NULL) receives SHA-256(payload).  RCS_ERR_IO on I/O failure. */
rcs_status rcs_snapshot_save(const rcs_state *s, const char *path, uint8_t digest[32], rcs_error *err);
/* Header-only read (never loads the payload). RCS_ERR_IO / RCS_ERR_FORMAT. */
rcs_status rcs_snapshot_info(const char *path, int *n_qubits, uint64_t *payload_bytes, uint8_t digest[32],
                             rcs_error *err);
/* Device scratch for rcs_snapshot_load of an n-qubit file (block CDF), block_bits as in
 * rcs_build_opts (0 -> 6). */
rcs_status rcs_snapshot_scratch_bytes(const rcs_context *ctx, int n_qubits, int block_bits, uint64_t *bytes);
/* Load `path` into the caller's device buffer (2^n complex64, rounded from float64), verifying
 * the digest while streaming (RCS_ERR_DIGEST; the buffer content is then unspecified) and the
 * norm (|T - 1| <= 1e-5, RCS_ERR_NORM); returns a sample-ready state (same calls as a built
 * one).  The file is opened read-only.  RCS_ERR_IO / RCS_ERR_FORMAT / RCS_ERR_MEMORY. */
rcs_status rcs_snapshot_load(rcs_context *ctx, const char *path, int block_bits, void *d_amps, uint64_t amps_bytes,
                             void *d_scratch, uint64_t scratch_bytes, rcs_state **out, rcs_error *err);
/* PAPER l.38 "2.5x10^6/N measurement shots": counts[j] = total / n_jobs, the
 * first total mod n_jobs jobs get one more.  RCS_ERR_ARG if n_jobs < 1. */
rcs_status rcs_shard_shots(uint64_t total, int n_jobs, uint64_t *counts);
/* Per-job shot seed (reading F3-2): SplitMix64 finalizer of base_seed + 0x9E3779B97F4A7C15 (job_id + 1). */
uint64_t rcs_job_seed(uint64_t base_seed, uint64_t job_id);
/* XEB from already-known ideal probabilities p[0..count) of the sampled bitstrings (the
 * aggregation of the jobs' result files): F, sigma, mean_p as rcs_xeb; fstar = NaN.
 * Host fp64, no device needed. */
rcs_status rcs_xeb_from_probs(int n_qubits, const double *p, uint64_t count, rcs_xeb_report *out);

#ifdef __cplusplus
}
#endif
#endif /* RCS_H */
