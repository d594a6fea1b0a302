// api.cpp -- the C ABI of include/rcs.h: orchestration of plan items on the context stream,
// NCCL remaps (grouped send/recv over NVLink), sampling and XEB collectives.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include <unistd.h>

#include "internal.h"
#include "kernels.h"

using namespace rcs;

constexpr int kMaxPeerWorld = 8;   // NVLink peer-swap remaps up to 8 ranks (one NVSwitch box); NCCL beyond

struct rcs_context {
    int device = 0, rank = 0, world = 1, g = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    ncclComm_t comm = nullptr;
    // device plan buffer for the tensor-core passes' A matrices (+ pinned host staging)
    uint32_t* d_tc = nullptr;
    size_t tc_cap = 0;   // words
    uint64_t tc_uid = 0;                          // circuit / pack whose matrices d_tc holds
    const rcs::TcPack* tc_pack = nullptr;
    std::shared_ptr<const rcs::TcPack> tc_hold;   // keeps that pack alive
    // product-state prefix operands (device copy of a PrefixPack: tab A | tab B | byte tables)
    char* d_pf = nullptr;
    size_t pf_cap = 0;
    const rcs::PrefixPack* pf_pack = nullptr;
    std::shared_ptr<const rcs::PrefixPack> pf_hold;
    // remaps over NVLink: CUDA-IPC mappings of the peers' shards (re-checked every build)
    bool p2p = false;                 // every rank mapped every peer (agreed over all ranks)
    char* d_xchg = nullptr;           // device buffer for the handle all-gather
    cudaIpcMemHandle_t peer_handle[kMaxPeerWorld];
    uint64_t peer_off[kMaxPeerWorld] = {};
    void* peer_map[kMaxPeerWorld] = {};
    float* d_bar = nullptr;           // 1-float all-reduce used as a stream-ordered barrier
    // pipelined remaps (f1): a second stream for the chunked peer swaps + per-chunk events
    cudaStream_t xstream = nullptr;
    cudaEvent_t ev_a[16] = {}, ev_s[16] = {};
    unsigned* d_tiles = nullptr;      // dynamic tile counter of the tensor-core passes (K12)
    // sampling / XEB chunk buffers, shared by every state of this context
    unsigned long long* xbuf = nullptr;
    double* dbuf = nullptr;
    double* xeb_part = nullptr;
    int* bad = nullptr;
};

struct rcs_state {
    rcs_context* ctx = nullptr;
    int n = 0, g = 0, nl = 0;       // g: real global bits (log2 world)
    float2* amps = nullptr;
    uint64_t n_amps = 0;
    // scratch carve-up
    double* inc = nullptr;          // block sums -> inclusive prefix
    uint64_t nblocks = 0;
    int b = 0;
    double* scan_tmp = nullptr;
    double* part_sq = nullptr;
    double* misc = nullptr;         // small device results
    float2* staging = nullptr;
    uint64_t staging_elems = 0;
    // the context's chunk buffers (set by ensure_buffers)
    unsigned long long* xbuf = nullptr;  // shot / bitstring chunk
    double* dbuf = nullptr;              // uniforms / probabilities chunk
    double* xeb_part = nullptr;
    int* bad = nullptr;
    uint64_t chunk = 0;
    // sampling CDF summary
    double T_r = 0, T_total = 0, E_r = 0, sum_sq = 0;
    int owns_tail = 0, owns_any = 0;
    std::vector<float> pass_ms;
    // kept (permuted) layout: final_pos of the plan, deferred restore items
    std::shared_ptr<const Plan> plan;
    bool permuted = false;
    double* gbuf = nullptr;          // all ranks' physical block sums (2^(n-b))
    uint64_t* ptab = nullptr;        // logical -> physical block byte tables (device)
    uint64_t nblocks_all = 0;
    uint64_t last_block = 0;
    // execution options of the build (rcs_build_opts), reused by rcs_state_canonicalize
    int remap_mode = RCS_REMAP_AUTO;
    int virt = 0;                    // virtual global qubits (world 1)
    unsigned* tiles = nullptr;       // K12 dynamic tile counter (the context's), nullptr: static tiles
    int tc_flags = 0;                // dev::kTcForceK9 | dev::kTcBulkRuns (rcs_build_opts)
};

namespace {

constexpr uint64_t kChunkShots = 1ull << 22;
constexpr uint64_t kAlign = 256;
constexpr int kOverlapPasses = 3;   // default passes after a remap pipelined behind its swaps

uint64_t align_up(uint64_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

#define CUDA_TRY(expr)                                                                     \
    do {                                                                                   \
        cudaError_t e__ = (expr);                                                          \
        if (e__ != cudaSuccess) {                                                          \
            set_error(err, RCS_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(e__));        \
            return RCS_ERR_CUDA;                                                           \
        }                                                                                  \
    } while (0)

#define NCCL_TRY(expr)                                                                     \
    do {                                                                                   \
        ncclResult_t r__ = (expr);                                                         \
        if (r__ != ncclSuccess) {                                                          \
            set_error(err, RCS_ERR_NCCL, "%s: %s", #expr, ncclGetErrorString(r__));        \
            return RCS_ERR_NCCL;                                                           \
        }                                                                                  \
    } while (0)

bool is_device_ptr(const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

int log2_exact(int w) {
    int g = 0;
    while ((1 << g) < w) g++;
    return (1 << g) == w ? g : -1;
}

struct Layout {
    int b;
    uint64_t nblocks, inc_off, tmp_off, part_off, misc_off, stage_off, total;
    // kept layout (keep_layout with remaps): logical CDF over all 2^(n-b) blocks
    bool kept = false;
    uint64_t nblocks_all = 0, gbuf_off = 0, ptab_off = 0;
    uint64_t stage_end = 0;
};

// keep: a kept (permuted) final layout is possible (keep_layout and world > 1 or virtual global)
Layout scratch_layout(int nl, int world, int virt, uint64_t staging_bytes, int block_bits, bool keep = false) {
    Layout L{};
    int b = block_bits > 0 ? block_bits : 6;
    if (b > 6) b = 6;
    if (b > nl) b = nl;
    L.b = b;
    L.nblocks = 1ull << (nl - b);
    L.kept = keep && (world > 1 || virt > 0);
    L.nblocks_all = L.kept ? L.nblocks * (uint64_t)world : L.nblocks;
    L.inc_off = 0;
    L.tmp_off = align_up(L.inc_off + L.nblocks_all * 8);
    L.part_off = align_up(L.tmp_off + dev::scan_tmp_doubles(L.nblocks_all) * 8);
    L.misc_off = align_up(L.part_off + (uint64_t)dev::block_sums_grid() * 8);
    L.stage_off = align_up(L.misc_off + 64 * 8);
    uint64_t st = 0;
    if (world > 1) st = staging_bytes ? staging_bytes : (256ull << 20);
    uint64_t end = align_up(L.stage_off + st);
    L.stage_end = end;
    if (L.kept) {
        L.gbuf_off = end;
        L.ptab_off = align_up(L.gbuf_off + L.nblocks_all * 8);
        end = align_up(L.ptab_off + (uint64_t)dev::kPermTables * 256 * 8);
    }
    L.total = end;
    return L;
}

struct Span {   // timing: item time += sign * elapsed(a, b); item kRemapKernelSpan: remap data movement
    size_t item;
    cudaEvent_t a, b;
    int sign;
};
constexpr size_t kRemapKernelSpan = SIZE_MAX;

// timing event recorded on st (owned by the build); nullptr when not timing
cudaEvent_t timing_event(std::vector<cudaEvent_t>* owned, cudaStream_t st) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    owned->push_back(e);
    cudaEventRecord(e, st);
    return e;
}

// Exchange for one REMAP item over NCCL: swap global positions a[i] with local b[i].
rcs_status do_remap_nccl(rcs_state* s, const Item& it, uint64_t* bytes_sent, std::vector<Span>* spans,
                         std::vector<cudaEvent_t>* owned, rcs_error* err) {
    rcs_context* c = s->ctx;
    const int j = it.k, nl = s->nl;
    int lpos[8];
    for (int i = 0; i < j; i++) lpos[i] = it.b[i];
    std::sort(lpos, lpos + j);
    int my_code = 0;
    for (int i = 0; i < j; i++) my_code |= ((c->rank >> (it.a[i] - nl)) & 1) << i;
    std::vector<int> codes, peers;
    std::vector<uint64_t> masks;
    for (int code = 0; code < (1 << j); code++) {
        if (code == my_code) continue;
        int peer = c->rank;
        uint64_t mask = 0;
        for (int i = 0; i < j; i++) {
            const int gb = it.a[i] - nl;
            peer = (peer & ~(1 << gb)) | (((code >> i) & 1) << gb);
            if ((code >> i) & 1) mask |= 1ull << it.b[i];
        }
        codes.push_back(code);
        peers.push_back(peer);
        masks.push_back(mask);
    }
    const int np = (int)peers.size();
    const uint64_t count = 1ull << (nl - j);
    uint64_t E = s->staging_elems / (2ull * np);
    if (E > count) E = count;
    if (E == 0) {
        set_error(err, RCS_ERR_MEMORY, "remap staging too small");
        return RCS_ERR_MEMORY;
    }
    cudaEvent_t k0 = spans ? timing_event(owned, c->stream) : nullptr;
    for (uint64_t m0 = 0; m0 < count; m0 += E) {
        const uint64_t e = std::min(E, count - m0);
        for (int p = 0; p < np; p++)
            CUDA_TRY(dev::pack(s->amps, s->staging + (uint64_t)p * E, j, lpos, masks[p], m0, e, c->stream));
        NCCL_TRY(ncclGroupStart());
        for (int p = 0; p < np; p++) {
            NCCL_TRY(ncclSend(s->staging + (uint64_t)p * E, e * 2, ncclFloat, peers[p], c->comm, c->stream));
            NCCL_TRY(ncclRecv(s->staging + (uint64_t)(np + p) * E, e * 2, ncclFloat, peers[p], c->comm, c->stream));
        }
        NCCL_TRY(ncclGroupEnd());
        for (int p = 0; p < np; p++)
            CUDA_TRY(dev::unpack(s->amps, s->staging + (uint64_t)(np + p) * E, j, lpos, masks[p], m0, e, c->stream));
        *bytes_sent += e * 8ull * np;
    }
    if (spans) spans->push_back({kRemapKernelSpan, k0, timing_event(owned, c->stream), 1});
    return RCS_OK;
}

// Tensor-core items of a plan (6-qubit blocks; 5-qubit blocks padded to 6 with the identity on a
// pinned qubit not in the block -- a function of the block -- placed as matrix bit 0: a block's
// highest qubit, the transposed kernel's converter-half bit, then never sits at one of the lowest
// cube ranks).
void make_tc_pack(const Plan& P, int nl, TcPack& out) {
    out.slot.assign(P.items.size(), -1);
    out.pos.assign(P.items.size(), std::array<int, 6>{});
    out.n_tc = 0;
    for (size_t ii = 0; ii < P.items.size(); ii++) {
        const Item& it = P.items[ii];
        if (it.type != RCS_ITEM_PASS || nl < kTcMinLocal || it.k < 5) continue;
        if (it.k == 5) {   // pad qubit: the first of the pinned positions 4, 5, 6, 0, 1, 2, 3 not in
            int pad = -1;    // the block (one above 3 keeps a second target out of positions 0..3,
            for (int c = 0; c < P.pinned && pad < 0; c++) {   // which would send the block to K9)
                const int b = (c + 4) % P.pinned;
                bool used = false;
                for (int i = 0; i < 5; i++) used = used || it.pos[i] == b;
                if (!used) pad = b;
            }
            out.pos[ii][0] = pad;
            for (int i = 0; i < 5; i++) out.pos[ii][i + 1] = it.pos[i];
        } else {
            for (int i = 0; i < 6; i++) out.pos[ii][i] = it.pos[i];
        }
        out.slot[ii] = out.n_tc++;
    }
    const size_t each = dev::tc_matrix_words();
    out.words.assign((size_t)out.n_tc * each, 0u);
    std::vector<cplx> padded(64 * 64);
    for (size_t ii = 0; ii < P.items.size(); ii++) {
        if (out.slot[ii] < 0) continue;
        const Block& B = P.blocks[P.items[ii].block];
        const cplx* m = B.matrix.data();
        if (P.items[ii].k == 5) {   // I (x) M with the pad as the lowest matrix bit
            for (int r = 0; r < 64; r++)
                for (int c = 0; c < 64; c++)
                    padded[r * 64 + c] = ((r ^ c) & 1) ? cplx{0.0, 0.0} : B.matrix[(r >> 1) * 32 + (c >> 1)];
            m = padded.data();
        }
        dev::tc_pack_matrix(reinterpret_cast<const double*>(m), out.words.data() + (size_t)out.slot[ii] * each);
    }
}

// Product-state prefix operands for a plan at n physical bits: the group tables and, for every
// byte of the physical index, which group-table bits its bits hold (initial layout).
void make_prefix_pack(const Plan& P, PrefixPack& out) {
    const int n = P.n;
    std::vector<int> occ(n);
    for (int q = 0; q < n; q++) occ[P.initial_pos.empty() ? q : P.initial_pos[q]] = q;
    out.nbytes = (n + 7) / 8;
    out.byt.assign((size_t)2 * out.nbytes * 256, 0u);
    out.zmask = 0;
    std::vector<int> gidx(n, -1), grp(n, -1);
    for (int G = 0; G < 2; G++)
        for (size_t i = 0; i < P.pq[G].size(); i++) {
            gidx[P.pq[G][i]] = (int)i;
            grp[P.pq[G][i]] = G;
        }
    for (int p = 0; p < n; p++) {
        const int q = occ[p];
        if (grp[q] < 0) {
            out.zmask |= 1ull << p;
            continue;
        }
        const int c = p >> 3, b = p & 7;
        for (int v = 0; v < 256; v++)
            if ((v >> b) & 1) out.byt[((size_t)grp[q] * out.nbytes + c) * 256 + v] |= 1u << gidx[q];
    }
    for (int G = 0; G < 2; G++) {
        out.tab[G].resize(2 * P.tab[G].size());
        for (size_t i = 0; i < P.tab[G].size(); i++) {
            out.tab[G][2 * i] = (float)P.tab[G][i].re;
            out.tab[G][2 * i + 1] = (float)P.tab[G][i].im;
        }
    }
}

// --- NVLink peer mapping -----------------------------------------------------------------
typedef int (*PFN_getAddressRange)(unsigned long long*, size_t*, unsigned long long);

PFN_getAddressRange address_range_fn() {
    static const PFN_getAddressRange fn = [] {   // resolved once (thread-safe static init)
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess) {
            cudaGetLastError();
            return (PFN_getAddressRange) nullptr;
        }
        return (PFN_getAddressRange)f;
    }();
    return fn;
}

// Maps every peer's amplitude shard over CUDA IPC (no assumption about device ordinals: the
// handles are all-gathered and opened; cudaIpcMemLazyEnablePeerAccess enables NVLink access).
// Every rank takes part in every collective whatever its local outcome, and the decision is
// agreed (all-reduce MIN of the per-rank success flags), so all ranks take the same remap path.
rcs_status setup_peers(rcs_context* c, void* amps, int remap_mode, rcs_error* err) {
    c->p2p = false;
    // identical on every rank (same opts, same world): no collective needed to agree
    if (remap_mode == RCS_REMAP_NCCL || c->world > kMaxPeerWorld) return RCS_OK;
    struct Rec {
        cudaIpcMemHandle_t h;
        uint64_t off;
        int ok;
    } mine{};
    {
        unsigned long long base = 0;
        size_t size = 0;
        PFN_getAddressRange get_range = address_range_fn();
        if (get_range && get_range(&base, &size, (unsigned long long)amps) == 0) {
            mine.off = (uint64_t)amps - base;
            mine.ok = cudaIpcGetMemHandle(&mine.h, (void*)base) == cudaSuccess;
            if (!mine.ok) cudaGetLastError();
        }
    }
    const size_t rec = (sizeof(Rec) + 15) / 16 * 16;
    if (!c->d_xchg) CUDA_TRY(cudaMalloc(&c->d_xchg, rec * (kMaxPeerWorld + 1)));
    if (!c->d_bar) CUDA_TRY(cudaMalloc(&c->d_bar, 16));
    CUDA_TRY(cudaMemcpyAsync(c->d_xchg, &mine, sizeof mine, cudaMemcpyHostToDevice, c->stream));
    NCCL_TRY(ncclAllGather(c->d_xchg, c->d_xchg + rec, rec, ncclChar, c->comm, c->stream));
    std::vector<char> all(rec * c->world);
    CUDA_TRY(cudaMemcpyAsync(all.data(), c->d_xchg + rec, rec * c->world, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    bool ok = true;
    for (int r = 0; r < c->world; r++) ok = ok && reinterpret_cast<const Rec*>(all.data() + rec * r)->ok;
    for (int r = 0; r < c->world && ok; r++) {
        if (r == c->rank) continue;
        const Rec* pr = reinterpret_cast<const Rec*>(all.data() + rec * r);
        if (c->peer_map[r] && std::memcmp(&c->peer_handle[r], &pr->h, sizeof pr->h) == 0) {   // cached mapping
            c->peer_off[r] = pr->off;
            continue;
        }
        void* mp = nullptr;
        if (cudaIpcOpenMemHandle(&mp, pr->h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
            cudaGetLastError();
            ok = false;
            break;
        }
        if (c->peer_map[r]) cudaIpcCloseMemHandle(c->peer_map[r]);   // the peer's buffer changed
        c->peer_map[r] = mp;
        c->peer_handle[r] = pr->h;
        c->peer_off[r] = pr->off;
    }
    float flag[2] = {ok ? 1.f : 0.f, 0.f};
    CUDA_TRY(cudaMemcpyAsync(c->d_bar + 2, flag, sizeof flag, cudaMemcpyHostToDevice, c->stream));
    NCCL_TRY(ncclAllReduce(c->d_bar + 2, c->d_bar + 3, 1, ncclFloat, ncclMin, c->comm, c->stream));
    CUDA_TRY(cudaMemcpyAsync(flag, c->d_bar + 2, sizeof flag, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    c->p2p = flag[1] > 0.5f;
    return RCS_OK;
}

// Fusion shared by the ranks of a context (world > 1): the strategies are split round-robin
// over the ranks, their costs (fuse_cost) all-gathered, and the winning rank (lowest cost, ties to
// the lower strategy -- the single-process rule, so the plan equals the 1-GPU plan) broadcasts
// its blocks; every rank then derives matrices and remaps itself.
rcs_status plan_distributed(rcs_context* c, const Circuit& circ, int fuse_k, int plan_g, Plan& out, rcs_error* err,
                            bool use_prefix) {
    const int k = plan_block_k(circ.n, fuse_k, plan_g);
    std::vector<Block> mine[kFuseStrategies];
    int64_t cnt[kFuseStrategies];
    {
        std::vector<std::thread> th;
        for (int s = 0; s < kFuseStrategies; s++) {
            cnt[s] = INT64_MAX;
            if (s % c->world != c->rank || k <= 0) continue;
            th.emplace_back([&, s] { fuse_strategy(circ, k, s, mine[s]); });
        }
        for (auto& t : th) t.join();
        for (int s = 0; s < kFuseStrategies; s++)
            if (s % c->world == c->rank && k > 0) cnt[s] = fuse_cost(mine[s]);
    }
    int64_t* d = nullptr;
    CUDA_TRY(cudaMalloc(&d, sizeof(int64_t) * kFuseStrategies * (c->world + 1)));
    struct Free {
        void* p;
        ~Free() { cudaFree(p); }
    } fr{d};
    CUDA_TRY(cudaMemcpyAsync(d, cnt, sizeof cnt, cudaMemcpyHostToDevice, c->stream));
    NCCL_TRY(ncclAllGather(d, d + kFuseStrategies, kFuseStrategies, ncclInt64, c->comm, c->stream));
    std::vector<int64_t> all((size_t)kFuseStrategies * c->world);
    CUDA_TRY(cudaMemcpyAsync(all.data(), d + kFuseStrategies, all.size() * 8, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    int win = 0;
    int64_t best = INT64_MAX;
    for (int s = 0; s < kFuseStrategies; s++) {
        const int64_t v = all[(size_t)(s % c->world) * kFuseStrategies + s];
        if (v < best) {
            best = v;
            win = s;
        }
    }
    const int owner = win % c->world;
    // serialize: [nblocks, (qubit mask, ngates, gate ids...) per block]
    std::vector<int64_t> buf;
    if (c->rank == owner) {
        buf.push_back((int64_t)mine[win].size());
        for (const Block& B : mine[win]) {
            int64_t m = 0;
            for (int q : B.qubits) m |= 1ll << q;
            buf.push_back(m);
            buf.push_back((int64_t)B.gate_ids.size());
            for (int g : B.gate_ids) buf.push_back(g);
        }
    }
    int64_t len = (int64_t)buf.size();
    int64_t* dl = nullptr;
    CUDA_TRY(cudaMalloc(&dl, 8));
    Free fr2{dl};
    CUDA_TRY(cudaMemcpyAsync(dl, &len, 8, cudaMemcpyHostToDevice, c->stream));
    NCCL_TRY(ncclBroadcast(dl, dl, 1, ncclInt64, owner, c->comm, c->stream));
    CUDA_TRY(cudaMemcpyAsync(&len, dl, 8, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    buf.resize((size_t)len);
    int64_t* db = nullptr;
    CUDA_TRY(cudaMalloc(&db, 8 * (size_t)std::max<int64_t>(len, 1)));
    Free fr3{db};
    if (c->rank == owner) CUDA_TRY(cudaMemcpyAsync(db, buf.data(), 8 * len, cudaMemcpyHostToDevice, c->stream));
    NCCL_TRY(ncclBroadcast(db, db, len, ncclInt64, owner, c->comm, c->stream));
    CUDA_TRY(cudaMemcpyAsync(buf.data(), db, 8 * len, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    std::vector<Block> blocks;
    size_t at = 0;
    const int64_t nb = len > 0 ? buf[at++] : 0;
    for (int64_t b = 0; b < nb; b++) {
        Block B;
        const int64_t m = buf[at++];
        for (int q = 0; q < 63; q++)
            if ((m >> q) & 1) B.qubits.push_back(q);
        const int64_t ng = buf[at++];
        for (int64_t i = 0; i < ng; i++) B.gate_ids.push_back((int)buf[at++]);
        blocks.push_back(std::move(B));
    }
    return build_plan(circ, fuse_k, plan_g, out, err, &blocks, use_prefix);
}

// stream-ordered barrier over all ranks (no rank proceeds past it before every rank reached it)
rcs_status stream_barrier(rcs_context* c, cudaStream_t st, rcs_error* err) {
    NCCL_TRY(ncclAllReduce(c->d_bar, c->d_bar, 1, ncclFloat, ncclMax, c->comm, st));
    return RCS_OK;
}

// One (possibly virtual) rank's view of a remap: its rank index, the local bits of a shard and
// every rank's shard.  Real ranks (world > 1): one view, peers through the CUDA-IPC mappings.
// Loopback (world 1, virtual_global g, RCS_REMAP_LOOPBACK): 2^g views whose shards are the
// 2^g consecutive regions of the one buffer, so the remap runs through the same peer-swap
// kernel and pipeline as between GPUs.
struct SwapView {
    int rank;
    int nl;
    float2* shard[kMaxPeerWorld];
};

bool loopback(const rcs_state* s) { return s->ctx->world == 1 && s->remap_mode == RCS_REMAP_LOOPBACK && s->virt > 0; }

std::vector<SwapView> swap_views(const rcs_state* s) {
    const rcs_context* c = s->ctx;
    std::vector<SwapView> v;
    if (loopback(s)) {
        const int nv = 1 << s->virt, nlv = s->n - s->virt;
        for (int r = 0; r < nv; r++) {
            SwapView w{r, nlv, {}};
            for (int q = 0; q < nv; q++) w.shard[q] = s->amps + ((uint64_t)q << nlv);
            v.push_back(w);
        }
        return v;
    }
    SwapView w{c->rank, s->nl, {}};
    for (int q = 0; q < c->world && q < kMaxPeerWorld; q++)
        w.shard[q] = q == c->rank ? s->amps
                                  : reinterpret_cast<float2*>(static_cast<char*>(c->peer_map[q]) + c->peer_off[q]);
    v.push_back(w);
    return v;
}

// Peer-swap arguments for one REMAP item: every unordered rank pair splits its element pairs
// in two halves, one per rank.  fix/nfix/fixval restrict it to one chunk of the index space.
void make_swap_args(const SwapView& v, const Item& it, const int* fix, int nfix, uint64_t fixval,
                    dev::PeerSwapArgs& A, uint64_t* bytes_sent) {
    const int j = it.k, nl = v.nl;
    A = dev::PeerSwapArgs{};
    A.local = v.shard[v.rank];
    A.j = j;
    int lpos[8];
    for (int i = 0; i < j; i++) lpos[i] = it.b[i];
    std::sort(lpos, lpos + j);
    for (int i = 0; i < j; i++) A.lpos[i] = lpos[i];
    A.nfix = nfix;
    for (int i = 0; i < nfix; i++) A.fix[i] = fix[i];
    A.fixval = fixval;
    int my_code = 0;
    for (int i = 0; i < j; i++) my_code |= ((v.rank >> (it.a[i] - nl)) & 1) << i;
    for (int i = 0; i < j; i++)
        if ((my_code >> i) & 1) A.my_mask |= 1ull << it.b[i];
    const uint64_t count = 1ull << (nl - j - nfix);
    for (int x = 1; x < (1 << j); x++) {   // peers in XOR-pattern order
        const int code = my_code ^ x;
        int peer = v.rank;
        uint64_t mask = 0;
        for (int i = 0; i < j; i++) {
            const int gb = it.a[i] - nl;
            peer = (peer & ~(1 << gb)) | (((code >> i) & 1) << gb);
            if ((code >> i) & 1) mask |= 1ull << it.b[i];
        }
        const int pc = A.npeers++;
        A.peer[pc] = v.shard[peer];
        A.mask[pc] = mask;
        const uint64_t half = count / 2;
        A.m_begin[pc] = v.rank < peer ? 0 : half;
        A.m_count[pc] = v.rank < peer ? half : count - half;
        *bytes_sent += count * 8ull;
    }
}

// Remap over NVLink (or loopback): swap the exchanged halves in place, local <-> peer.  The
// views' element sets are disjoint, so loopback launches need no barrier between them.
rcs_status do_remap_p2p(rcs_state* s, const Item& it, uint64_t* bytes_sent, std::vector<Span>* spans,
                        std::vector<cudaEvent_t>* owned, rcs_error* err) {
    rcs_context* c = s->ctx;
    const bool real = !loopback(s);
    if (real) {
        rcs_status st = stream_barrier(c, c->stream, err);
        if (st) return st;
    }
    cudaEvent_t k0 = spans ? timing_event(owned, c->stream) : nullptr;
    for (const SwapView& v : swap_views(s)) {
        dev::PeerSwapArgs A;
        make_swap_args(v, it, nullptr, 0, 0, A, bytes_sent);
        CUDA_TRY(dev::peer_swap(A, c->stream));
    }
    if (spans) spans->push_back({kRemapKernelSpan, k0, timing_event(owned, c->stream), 1});
    return real ? stream_barrier(c, c->stream, err) : RCS_OK;
}

// Pipelined remap: [pass A] -> REMAP -> [pass B] in 2^cb chunks of the index
// space (cb fixed "chunk" bits, untouched by A, the remap and B).  Pass chunks run on the
// context stream on (num_sms - reserve) SMs; the peer swap of chunk c runs on xstream as soon
// as every rank finished A on chunk c (barrier), and B on chunk c starts once every rank
// finished swapping it (barrier).  Arithmetic per amplitude is unchanged (bitwise equal).
// Loopback: the pass launches cover every virtual rank's chunk c at once, so stream order
// alone provides both barriers.
struct PassRef {
    const int* pos;
    const uint32_t* d_a;
};

rcs_status do_remap_pipelined(rcs_state* s, const Item& it, const PassRef* pa, const PassRef* pbs, int nb,
                              const int* fix, int cb, int reserve, uint64_t* bytes_sent,
                              uint64_t* pass_bytes, size_t ia, size_t ir, const size_t* ibs, std::vector<Span>* spans,
                              std::vector<cudaEvent_t>* owned, rcs_error* err) {
    rcs_context* c = s->ctx;
    const int nch = 1 << cb;
    const bool real = !loopback(s);
    if (!c->xstream) CUDA_TRY(cudaStreamCreateWithFlags(&c->xstream, cudaStreamNonBlocking));
    for (int i = 0; i < nch; i++) {
        if (!c->ev_a[i]) CUDA_TRY(cudaEventCreateWithFlags(&c->ev_a[i], cudaEventDisableTiming));
        if (!c->ev_s[i]) CUDA_TRY(cudaEventCreateWithFlags(&c->ev_s[i], cudaEventDisableTiming));
    }
    auto tev = [&](cudaStream_t st) { return timing_event(owned, st); };
    auto fixval = [&](int ch) {
        uint64_t v = 0;
        for (int i = 0; i < cb; i++)
            if ((ch >> i) & 1) v |= 1ull << fix[i];
        return v;
    };
    const int sms = std::max(1, c->num_sms - reserve);
    const std::vector<SwapView> views = swap_views(s);
    cudaEvent_t t0 = spans ? tev(c->stream) : nullptr;
    // A: all chunks, in order, on the main stream
    for (int ch = 0; ch < nch; ch++) {
        if (pa)
            CUDA_TRY(dev::gate_pass_tc(s->amps, s->nl, pa->pos, pa->d_a, sms, c->stream, fix, cb, fixval(ch), s->tc_flags,
                                       s->tiles));
        CUDA_TRY(cudaEventRecord(c->ev_a[ch], c->stream));
    }
    if (pa) *pass_bytes += 16ull * s->n_amps;
    cudaEvent_t tA = spans ? tev(c->stream) : nullptr;
    if (spans && pa) spans->push_back({ia, t0, tA, 1});
    // swaps: chunk by chunk on xstream
    for (int ch = 0; ch < nch; ch++) {
        CUDA_TRY(cudaStreamWaitEvent(c->xstream, c->ev_a[ch], 0));
        if (real) {
            rcs_status st = stream_barrier(c, c->xstream, err);
            if (st) return st;
        }
        cudaEvent_t k0 = spans ? tev(c->xstream) : nullptr;
        for (const SwapView& v : views) {
            dev::PeerSwapArgs A;
            make_swap_args(v, it, fix, cb, fixval(ch), A, bytes_sent);
            A.max_grid = reserve * 8;
            CUDA_TRY(dev::peer_swap(A, c->xstream));
        }
        if (spans) spans->push_back({kRemapKernelSpan, k0, tev(c->xstream), 1});
        if (real) {
            rcs_status st = stream_barrier(c, c->xstream, err);
            if (st) return st;
        }
        CUDA_TRY(cudaEventRecord(c->ev_s[ch], c->xstream));
    }
    // B chain (nb passes after the remap), chunk c of the first one after every rank exchanged
    // chunk c.  Anti-diagonal order (pass i of chunk c at step i + c): while the swap of chunk c
    // is still on NVLink the main stream works on later passes of earlier chunks.
    for (int d = 0; d < nb + nch - 1; d++)
        for (int ch = 0; ch < nch; ch++) {
            const int i = d - ch;
            if (i < 0 || i >= nb) continue;
            if (i == 0) CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_s[ch], 0));
            cudaEvent_t w = spans ? tev(c->stream) : nullptr;
            CUDA_TRY(dev::gate_pass_tc(s->amps, s->nl, pbs[i].pos, pbs[i].d_a, sms, c->stream, fix, cb, fixval(ch),
                                       s->tc_flags, s->tiles));
            if (spans) {
                cudaEvent_t e = tev(c->stream);
                spans->push_back({ibs[i], w, e, 1});
                spans->push_back({ir, w, e, -1});
            }
        }
    if (nb == 0)   // no pass after the remap: the main stream still waits for every chunk's swap
        for (int ch = 0; ch < nch; ch++) CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_s[ch], 0));
    *pass_bytes += 16ull * s->n_amps * (uint64_t)nb;
    if (spans) spans->push_back({ir, tA, tev(c->stream), 1});
    return RCS_OK;
}

// chunk bits for a pipelined remap: the highest positions below nl_local outside `excl`
// (K9's tile sub-cube and pair bit, K12's 13 positions, the remapped bits); false if too few
bool choose_chunk_bits(int nl, uint64_t excl, int cb, int* fix) {
    int got = 0;
    for (int b = nl - 1; b >= 7 && got < cb; b--)   // above every tile sub-cube's low bits
        if (!((excl >> b) & 1)) fix[got++] = b;
    if (got < cb) return false;
    std::sort(fix, fix + cb);
    return true;
}

// block sums + scan + shard totals (collective); fills s->T_*, E_r, sum_sq, ownership
rcs_status compute_cdf(rcs_state* s, rcs_error* err) {
    rcs_context* c = s->ctx;
    CUDA_TRY(dev::block_sums(s->amps, s->nblocks, s->b, s->inc, s->part_sq, c->stream));
    CUDA_TRY(dev::scan_inclusive(s->inc, s->nblocks, s->scan_tmp, c->stream));
    CUDA_TRY(dev::reduce_sum(s->part_sq, dev::block_sums_grid(), s->misc + 1, c->stream));
    CUDA_TRY(cudaMemcpyAsync(s->misc, s->inc + (s->nblocks - 1), sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    std::vector<double> tot(c->world, 0.0);
    double sq = 0.0;
    if (c->world > 1) {
        // misc[8..8+world): gathered shard totals; misc[2]: global sum p^2
        NCCL_TRY(ncclAllGather(s->misc, s->misc + 8, 1, ncclDouble, c->comm, c->stream));
        NCCL_TRY(ncclAllReduce(s->misc + 1, s->misc + 2, 1, ncclDouble, ncclSum, c->comm, c->stream));
        CUDA_TRY(cudaMemcpyAsync(tot.data(), s->misc + 8, sizeof(double) * c->world, cudaMemcpyDeviceToHost, c->stream));
        CUDA_TRY(cudaMemcpyAsync(&sq, s->misc + 2, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    } else {
        CUDA_TRY(cudaMemcpyAsync(tot.data(), s->misc, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        CUDA_TRY(cudaMemcpyAsync(&sq, s->misc + 1, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    }
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    double E = 0.0, T = 0.0;
    int last_owner = -1;
    for (int r = 0; r < c->world; r++) {
        if (r == c->rank) s->E_r = E;
        E += tot[r];
        if (tot[r] > 0) last_owner = r;
    }
    T = E;
    s->T_r = tot[c->rank];
    s->T_total = T;
    s->sum_sq = sq;
    s->owns_any = s->T_r > 0 ? 1 : 0;
    s->owns_tail = c->rank == last_owner ? 1 : 0;
    return RCS_OK;
}

// kept (permuted) layout: every rank builds the logical-order block CDF of the whole state
// (all-gather of the physical block sums, permutation into logical order, one global scan)
rcs_status compute_cdf_kept(rcs_state* s, rcs_error* err) {
    rcs_context* c = s->ctx;
    const uint64_t nbl = s->nblocks;
    double* mine = s->gbuf + (uint64_t)c->rank * nbl;
    CUDA_TRY(dev::block_sums(s->amps, nbl, s->b, mine, s->part_sq, c->stream));
    if (c->world > 1) NCCL_TRY(ncclAllGather(mine, s->gbuf, nbl, ncclDouble, c->comm, c->stream));
    CUDA_TRY(dev::perm_blocks(s->gbuf, s->inc, s->nblocks_all, s->ptab, c->stream));
    CUDA_TRY(dev::scan_inclusive(s->inc, s->nblocks_all, s->scan_tmp, c->stream));
    CUDA_TRY(dev::reduce_sum(s->part_sq, dev::block_sums_grid(), s->misc + 1, c->stream));
    if (c->world > 1) NCCL_TRY(ncclAllReduce(s->misc + 1, s->misc + 1, 1, ncclDouble, ncclSum, c->comm, c->stream));
    unsigned long long* last = reinterpret_cast<unsigned long long*>(s->misc + 40);
    CUDA_TRY(dev::last_nonzero(s->inc, s->nblocks_all, last, c->stream));
    double T = 0.0, sq = 0.0;
    unsigned long long lb = 0;
    CUDA_TRY(cudaMemcpyAsync(&T, s->inc + (s->nblocks_all - 1), sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaMemcpyAsync(&sq, s->misc + 1, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaMemcpyAsync(&lb, last, sizeof lb, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    s->T_total = T;
    s->sum_sq = sq;
    s->last_block = lb;
    s->E_r = 0.0;
    s->T_r = T;
    s->owns_any = 1;
    s->owns_tail = 1;
    return RCS_OK;
}

dev::Locator locator(const rcs_state* s) {
    return dev::Locator{s->nl, (uint64_t)s->ctx->rank, s->b, s->permuted ? s->ptab : nullptr};
}

rcs_status ensure_buffers(rcs_state* s, rcs_error* err) {
    if (s->xbuf) return RCS_OK;
    rcs_context* c = s->ctx;
    if (!c->xbuf) {   // allocated once per context: cudaMalloc/cudaFree per state would sync
        CUDA_TRY(cudaMalloc(&c->xbuf, kChunkShots * sizeof(unsigned long long)));
        CUDA_TRY(cudaMalloc(&c->dbuf, kChunkShots * sizeof(double)));
        CUDA_TRY(cudaMalloc(&c->xeb_part, (size_t)dev::xeb_grid() * 3 * sizeof(double) + 64));
        CUDA_TRY(cudaMalloc(&c->bad, sizeof(int)));
    }
    s->chunk = kChunkShots;
    s->xbuf = c->xbuf;
    s->dbuf = c->dbuf;
    s->xeb_part = c->xeb_part;
    s->bad = c->bad;
    return RCS_OK;
}

rcs_status sample_impl(rcs_state* s, uint64_t shots, uint64_t seed, uint64_t offset, const double* u,
                       uint64_t* out_x, rcs_sample_report* rep, rcs_error* err) {
    if (!s || (!out_x && shots)) { set_error(err, RCS_ERR_ARG, "null argument"); return RCS_ERR_ARG; }
    rcs_context* c = s->ctx;
    CUDA_TRY(cudaSetDevice(c->device));
    if (!(std::fabs(s->T_total - 1.0) <= 1e-5)) {
        set_error(err, RCS_ERR_NORM, "state norm %.9g deviates from 1 by more than 1e-5", s->T_total);
        return RCS_ERR_NORM;
    }
    rcs_status st = ensure_buffers(s, err);
    if (st) return st;
    const bool out_dev = is_device_ptr(out_x);
    const bool u_dev = u ? is_device_ptr(u) : false;
    struct Events {   // destroyed on every exit path
        cudaEvent_t a = nullptr, b = nullptr;
        ~Events() {
            if (a) cudaEventDestroy(a);
            if (b) cudaEventDestroy(b);
        }
    } ev;
    CUDA_TRY(cudaEventCreate(&ev.a));
    CUDA_TRY(cudaEventCreate(&ev.b));
    cudaEvent_t e0 = ev.a, e1 = ev.b;
    CUDA_TRY(cudaEventRecord(e0, c->stream));
    for (uint64_t s0 = 0; s0 < shots; s0 += s->chunk) {
        const uint64_t cnt = std::min(s->chunk, shots - s0);
        unsigned long long* xo = out_dev ? reinterpret_cast<unsigned long long*>(out_x) + s0 : s->xbuf;
        dev::SampleArgs A{};
        A.amps = s->amps;
        A.inc = s->inc;
        A.nblocks = s->nblocks;
        A.b = s->b;
        A.T_total = s->T_total;
        A.E_r = s->E_r;
        A.T_r = s->T_r;
        A.owns_tail = s->owns_tail;
        A.owns_any = s->owns_any;
        A.seed = seed;
        A.shot0 = offset + s0;
        A.shots = cnt;
        A.u_in = nullptr;
        if (u) {
            if (u_dev) {
                A.u_in = u + s0;
            } else {
                CUDA_TRY(cudaMemcpyAsync(s->dbuf, u + s0, cnt * sizeof(double), cudaMemcpyHostToDevice, c->stream));
                A.u_in = s->dbuf;
            }
        }
        A.base_index = (uint64_t)c->rank << s->nl;
        A.x_out = xo;
        A.nl = s->nl;
        A.rank = (uint64_t)c->rank;
        if (s->permuted) {   // logical CDF over all ranks' blocks
            A.ptab = s->ptab;
            A.nblocks = s->nblocks_all;
            A.last_block = s->last_block;
        }
        CUDA_TRY(dev::sample(A, c->stream));
        if (c->world > 1)
            NCCL_TRY(ncclAllReduce(xo, xo, cnt, ncclUint64, ncclSum, c->comm, c->stream));
        if (!out_dev)
            CUDA_TRY(cudaMemcpyAsync(out_x + s0, xo, cnt * sizeof(uint64_t), cudaMemcpyDeviceToHost, c->stream));
    }
    CUDA_TRY(cudaEventRecord(e1, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) {
        rep->shots = shots;
        rep->total_prob = s->T_total;
        rep->sample_ms = ms;
    }
    return RCS_OK;
}

}  // namespace

// =====================================================================================
extern "C" {

const char* rcs_status_string(int s) {
    switch (s) {
        case RCS_OK: return "RCS_OK";
        case RCS_ERR_PARSE: return "RCS_ERR_PARSE";
        case RCS_ERR_UNKNOWN_GATE: return "RCS_ERR_UNKNOWN_GATE";
        case RCS_ERR_QUBIT_RANGE: return "RCS_ERR_QUBIT_RANGE";
        case RCS_ERR_ARITY: return "RCS_ERR_ARITY";
        case RCS_ERR_MEMORY: return "RCS_ERR_MEMORY";
        case RCS_ERR_NORM: return "RCS_ERR_NORM";
        case RCS_ERR_SIZE: return "RCS_ERR_SIZE";
        case RCS_ERR_ARG: return "RCS_ERR_ARG";
        case RCS_ERR_CUDA: return "RCS_ERR_CUDA";
        case RCS_ERR_NCCL: return "RCS_ERR_NCCL";
        case RCS_ERR_IO: return "RCS_ERR_IO";
        case RCS_ERR_FORMAT: return "RCS_ERR_FORMAT";
        case RCS_ERR_DIGEST: return "RCS_ERR_DIGEST";
        default: return "RCS_ERR_UNKNOWN";
    }
}

rcs_status rcs_circuit_load_qasm(const char* text, size_t len, rcs_circuit** out, rcs_error* err) {
    if (err) std::memset(err, 0, sizeof *err);
    if (!text || !out) { set_error(err, RCS_ERR_ARG, "null argument"); return RCS_ERR_ARG; }
    rcs_circuit* c = new (std::nothrow) rcs_circuit();
    if (!c) { set_error(err, RCS_ERR_MEMORY, "out of host memory"); return RCS_ERR_MEMORY; }
    rcs_status st = parse_qasm(text, len, c->c, err);
    if (st != RCS_OK) { delete c; return st; }
    static std::atomic<uint64_t> next_uid{1};
    c->uid = next_uid.fetch_add(1);
    *out = c;
    return RCS_OK;
}

rcs_status rcs_circuit_stats(const rcs_circuit* c, rcs_circuit_counts* o) {
    if (!c || !o) return RCS_ERR_ARG;
    std::memset(o, 0, sizeof *o);
    o->n_qubits = c->c.n;
    o->n_moments = c->c.n_moments;
    o->n_gates = (int)c->c.gates.size();
    o->n_measure = c->c.n_measure;
    for (const auto& g : c->c.gates) {
        switch (g.kind) {
            case RCS_GATE_SX: o->n_sx++; break;
            case RCS_GATE_SY: o->n_sy++; break;
            case RCS_GATE_SW: o->n_sw++; break;
            case RCS_GATE_RZ: o->n_rz++; break;
            default: o->n_fsim++;
        }
    }
    return RCS_OK;
}

rcs_status rcs_circuit_gate(const rcs_circuit* c, int i, int* kind, int* q0, int* q1, double* theta, double* phi,
                            int* moment) {
    if (!c || i < 0 || i >= (int)c->c.gates.size()) return RCS_ERR_ARG;
    const Gate& g = c->c.gates[i];
    if (kind) *kind = g.kind;
    if (q0) *q0 = g.q0;
    if (q1) *q1 = g.q1;
    if (theta) *theta = g.theta;
    if (phi) *phi = g.phi;
    if (moment) *moment = g.moment;
    return RCS_OK;
}

void rcs_circuit_free(rcs_circuit* c) { delete c; }

uint64_t rcs_kernel_launches(void) { return dev::launches(); }

rcs_status rcs_plan_create(const rcs_circuit* c, int fuse_k, int n_global, rcs_plan** out, rcs_error* err) {
    if (err) std::memset(err, 0, sizeof *err);
    if (!c || !out) { set_error(err, RCS_ERR_ARG, "null argument"); return RCS_ERR_ARG; }
    rcs_plan* p = new (std::nothrow) rcs_plan();
    if (!p) return RCS_ERR_MEMORY;
    rcs_status st = build_plan(c->c, fuse_k, n_global, p->p, err);
    if (st) { delete p; return st; }
    *out = p;
    return RCS_OK;
}

rcs_status rcs_plan_layout(const rcs_plan* p, int* restore_begin, int* final_pos, int* initial_pos) {
    if (!p) return RCS_ERR_ARG;
    const Plan& P = p->p;
    if (restore_begin) *restore_begin = P.restore_begin;
    for (int q = 0; q < P.n; q++) {
        if (final_pos) final_pos[q] = q < (int)P.final_pos.size() ? P.final_pos[q] : q;
        if (initial_pos) initial_pos[q] = q < (int)P.initial_pos.size() ? P.initial_pos[q] : q;
    }
    return RCS_OK;
}

rcs_status rcs_plan_prefix(const rcs_plan* p, int* n_prefix) {
    if (!p || !n_prefix) return RCS_ERR_ARG;
    *n_prefix = p->p.prefix;
    return RCS_OK;
}

rcs_status rcs_plan_summary(const rcs_plan* p, int* n_items, int* n_passes, int* n_remaps, int* n_swaps) {
    if (!p) return RCS_ERR_ARG;
    if (n_items) *n_items = (int)p->p.items.size();
    if (n_passes) *n_passes = p->p.n_passes;
    if (n_remaps) *n_remaps = p->p.n_remaps;
    if (n_swaps) *n_swaps = p->p.n_swaps;
    return RCS_OK;
}

rcs_status rcs_plan_item_get(const rcs_plan* p, int i, rcs_plan_item* o, double* matrix_out) {
    if (!p || !o || i < 0 || i >= (int)p->p.items.size()) return RCS_ERR_ARG;
    const Item& it = p->p.items[i];
    std::memset(o, 0, sizeof *o);
    o->type = it.type;
    o->k = it.k;
    for (int t = 0; t < 8; t++) {
        o->pos[t] = it.pos[t];
        o->a[t] = it.a[t];
        o->b[t] = it.b[t];
        o->qubits[t] = -1;
    }
    if (it.type == RCS_ITEM_PASS) {
        const Block& B = p->p.blocks[it.block];
        for (int t = 0; t < it.k; t++) o->qubits[t] = B.qubits[t];
        o->n_gates = (int)B.gate_ids.size();
        if (matrix_out)
            for (size_t e = 0; e < B.matrix.size(); e++) {
                matrix_out[2 * e] = B.matrix[e].re;
                matrix_out[2 * e + 1] = B.matrix[e].im;
            }
    }
    return RCS_OK;
}

void rcs_plan_free(rcs_plan* p) { delete p; }

int rcs_nccl_unique_id_bytes(void) { return (int)sizeof(ncclUniqueId); }

rcs_status rcs_nccl_unique_id(void* out, rcs_error* err) {
    if (err) std::memset(err, 0, sizeof *err);
    if (!out) { set_error(err, RCS_ERR_ARG, "null argument"); return RCS_ERR_ARG; }
    ncclUniqueId id;
    NCCL_TRY(ncclGetUniqueId(&id));
    std::memcpy(out, &id, sizeof id);
    return RCS_OK;
}

rcs_status rcs_context_create(int device, int rank, int world, const void* nccl_id, void* stream, rcs_context** out,
                              rcs_error* err) {
    if (err) std::memset(err, 0, sizeof *err);
    if (!out || world < 1 || rank < 0 || rank >= world) { set_error(err, RCS_ERR_ARG, "bad rank/world"); return RCS_ERR_ARG; }
    const int g = log2_exact(world);
    if (g < 0) { set_error(err, RCS_ERR_ARG, "world=%d is not a power of two", world); return RCS_ERR_ARG; }
    if (world > 1 && !nccl_id) { set_error(err, RCS_ERR_ARG, "world > 1 needs an NCCL unique id"); return RCS_ERR_ARG; }
    CUDA_TRY(cudaSetDevice(device));
    rcs_context* c = new (std::nothrow) rcs_context();
    if (!c) return RCS_ERR_MEMORY;
    c->device = device;
    c->rank = rank;
    c->world = world;
    c->g = g;
    c->stream = reinterpret_cast<cudaStream_t>(stream);
    cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
    if (world > 1) {
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, sizeof id);
        ncclResult_t r = ncclCommInitRank(&c->comm, world, id, rank);
        if (r != ncclSuccess) {
            set_error(err, RCS_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
            delete c;
            return RCS_ERR_NCCL;
        }
    }
    *out = c;
    return RCS_OK;
}

void rcs_context_free(rcs_context* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    for (int r = 0; r < kMaxPeerWorld; r++)
        if (c->peer_map[r]) cudaIpcCloseMemHandle(c->peer_map[r]);
    if (c->d_xchg) cudaFree(c->d_xchg);
    if (c->d_bar) cudaFree(c->d_bar);
    if (c->xbuf) cudaFree(c->xbuf);
    if (c->dbuf) cudaFree(c->dbuf);
    if (c->xeb_part) cudaFree(c->xeb_part);
    if (c->bad) cudaFree(c->bad);
    if (c->d_tc) cudaFree(c->d_tc);
    if (c->d_tiles) cudaFree(c->d_tiles);
    if (c->d_pf) cudaFree(c->d_pf);
    for (int i = 0; i < 16; i++)
        for (cudaEvent_t e : {c->ev_a[i], c->ev_s[i]})
            if (e) cudaEventDestroy(e);
    if (c->xstream) cudaStreamDestroy(c->xstream);
    if (c->comm) ncclCommDestroy(c->comm);
    delete c;
}

rcs_status rcs_state_scratch_bytes(const rcs_context* ctx, const rcs_circuit* c, const rcs_build_opts* opts,
                                   uint64_t* bytes) {
    if (!ctx || !c || !bytes) return RCS_ERR_ARG;
    rcs_build_opts o{};
    if (opts) o = *opts;
    const int nl = c->c.n - ctx->g;
    if (nl < 1) return RCS_ERR_ARG;
    *bytes = scratch_layout(nl, ctx->world, o.virtual_global, o.staging_bytes, o.block_bits, o.keep_layout != 0).total;
    return RCS_OK;
}

rcs_status rcs_state_build(rcs_context* ctx, const rcs_circuit* circ, const rcs_build_opts* opts, void* d_amps,
                           uint64_t amps_bytes, void* d_scratch, uint64_t scratch_bytes, rcs_state** out,
                           rcs_build_report* rep, rcs_error* err) {
    if (err) std::memset(err, 0, sizeof *err);
    if (!ctx || !circ || !d_amps || !out) { set_error(err, RCS_ERR_ARG, "null argument"); return RCS_ERR_ARG; }
    rcs_build_opts o{};
    if (opts) o = *opts;
    const int n = circ->c.n;
    const int g = ctx->g;
    if (o.virtual_global && ctx->world > 1) {
        set_error(err, RCS_ERR_ARG, "virtual_global needs world == 1");
        return RCS_ERR_ARG;
    }
    if (o.remap_mode < RCS_REMAP_AUTO || o.remap_mode > RCS_REMAP_LOOPBACK ||
        (o.remap_mode == RCS_REMAP_LOOPBACK && (ctx->world != 1 || o.virtual_global < 1 || o.virtual_global > 3)) ||
        o.overlap_chunks < 0 || o.overlap_chunks > 4 || o.overlap_sms < 0 || o.tc_kernel < 0 || o.tc_kernel > 2 ||
        o.overlap_passes < 0 || o.overlap_passes > 8 || o.tc_schedule < 0 || o.tc_schedule > 1 || o.tc_tma < -1 || o.tc_tma > 0 ||
        o.product_prefix < -1 || o.product_prefix > 0 ||
        o.virtual_global < 0) {
        set_error(err, RCS_ERR_ARG, "invalid build options (remap_mode %d, virtual_global %d, overlap_chunks %d)",
                  o.remap_mode, o.virtual_global, o.overlap_chunks);
        return RCS_ERR_ARG;
    }
    const int plan_g = ctx->world > 1 ? g : o.virtual_global;
    const int nl = n - g;
    if (nl < 1) { set_error(err, RCS_ERR_ARG, "n=%d too small for world=%d", n, ctx->world); return RCS_ERR_ARG; }
    const uint64_t n_amps = 1ull << nl;
    if (amps_bytes < n_amps * 8) {
        set_error(err, RCS_ERR_MEMORY, "amplitude buffer too small: need %llu bytes", (unsigned long long)(n_amps * 8));
        if (err) err->bytes_required = n_amps * 8;
        return RCS_ERR_MEMORY;
    }
    const Layout L = scratch_layout(nl, ctx->world, o.virtual_global, o.staging_bytes, o.block_bits, o.keep_layout != 0);
    if (!d_scratch || scratch_bytes < L.total) {
        set_error(err, RCS_ERR_MEMORY, "scratch buffer too small: need %llu bytes", (unsigned long long)L.total);
        if (err) err->bytes_required = L.total;
        return RCS_ERR_MEMORY;
    }
    CUDA_TRY(cudaSetDevice(ctx->device));

    auto t0 = std::chrono::steady_clock::now();
    std::shared_ptr<const Plan> plan_ptr;
    // product_prefix off: the plan has no prefix (its blocks are remapped like any other); the
    // plan and the caches derived from it are keyed on that too
    const bool use_prefix = o.product_prefix >= 0 && nl >= 6;   // the kernel writes 64-amplitude rows
    const int pkey = o.fuse_k | (use_prefix ? 0 : 1 << 8);
    {
        rcs_circuit* cc = const_cast<rcs_circuit*>(circ);
        std::lock_guard<std::mutex> lk(cc->mu);
        auto key = std::make_pair(pkey, plan_g);
        auto f = cc->plans.find(key);
        if (f != cc->plans.end()) {
            plan_ptr = f->second;
        } else {
            auto np = std::make_shared<Plan>();
            rcs_status pst = ctx->world > 1 ? plan_distributed(ctx, circ->c, o.fuse_k, plan_g, *np, err, use_prefix)
                                            : build_plan(circ->c, o.fuse_k, plan_g, *np, err, nullptr, use_prefix);
            if (pst) return pst;
            plan_ptr = np;
            cc->plans[key] = plan_ptr;
        }
    }
    const Plan& P = *plan_ptr;
    rcs_status st = RCS_OK;
    auto t1 = std::chrono::steady_clock::now();

    rcs_state* s = new (std::nothrow) rcs_state();
    if (!s) return RCS_ERR_MEMORY;
    s->ctx = ctx;
    s->n = n;
    s->g = g;
    s->nl = nl;
    s->amps = reinterpret_cast<float2*>(d_amps);
    s->n_amps = n_amps;
    char* sc = reinterpret_cast<char*>(d_scratch);
    s->b = L.b;
    s->nblocks = L.nblocks;
    s->inc = reinterpret_cast<double*>(sc + L.inc_off);
    s->scan_tmp = reinterpret_cast<double*>(sc + L.tmp_off);
    s->part_sq = reinterpret_cast<double*>(sc + L.part_off);
    s->misc = reinterpret_cast<double*>(sc + L.misc_off);
    s->staging = reinterpret_cast<float2*>(sc + L.stage_off);
    s->staging_elems = (L.stage_end - L.stage_off) / sizeof(float2);
    s->plan = plan_ptr;
    s->remap_mode = o.remap_mode;
    s->virt = ctx->world == 1 ? o.virtual_global : 0;
    // keep_layout: skip the restore items when the final layout is not canonical
    bool keep = false;
    if (L.kept) {
        for (int q = L.b; q < n && !keep; q++) keep = P.final_pos[q] != q;
    }
    const size_t n_exec = keep ? (size_t)P.restore_begin : P.items.size();
    std::vector<uint64_t> ptab_host;
    if (keep) {
        s->gbuf = reinterpret_cast<double*>(sc + L.gbuf_off);
        s->ptab = reinterpret_cast<uint64_t*>(sc + L.ptab_off);
        s->nblocks_all = L.nblocks_all;
        ptab_host.assign((size_t)dev::kPermTables * 256, 0);
        const int nlb = n - L.b;   // logical block bits
        if (nlb > 8 * dev::kPermTables) {
            set_error(err, RCS_ERR_ARG, "keep_layout supports n - block_bits <= %d", 8 * dev::kPermTables);
            delete s;
            return RCS_ERR_ARG;
        }
        for (int c = 0; c < dev::kPermTables; c++)
            for (int v = 0; v < 256; v++) {
                uint64_t o = 0;
                for (int i = 0; i < 8; i++) {
                    const int bit = 8 * c + i;
                    if (bit < nlb && ((v >> i) & 1)) o |= 1ull << (P.final_pos[bit + L.b] - L.b);
                }
                ptab_host[(size_t)c * 256 + v] = o;
            }
    }

    // every event this build creates is owned here and destroyed on every exit path
    std::vector<cudaEvent_t> owned;
    auto fail = [&](rcs_status code) {
        for (auto& e : owned) cudaEventDestroy(e);
        delete s;
        return code;
    };
#define BUILD_TRY(expr)                                                                    \
    do {                                                                                   \
        cudaError_t e__ = (expr);                                                          \
        if (e__ != cudaSuccess) {                                                          \
            set_error(err, RCS_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(e__));        \
            return fail(RCS_ERR_CUDA);                                                     \
        }                                                                                  \
    } while (0)

    cudaStream_t stream = ctx->stream;
    cudaEvent_t eb0, eb1, ec0;
    BUILD_TRY(cudaEventCreate(&eb0));
    owned.push_back(eb0);
    BUILD_TRY(cudaEventCreate(&eb1));
    owned.push_back(eb1);
    BUILD_TRY(cudaEventCreate(&ec0));
    owned.push_back(ec0);
    // tensor-core passes: packed operands cached per (circuit, plan, n_local); the device copy
    // lives in the context and is re-uploaded only when the circuit or plan changes
    std::shared_ptr<const TcPack> tcp;
    {
        rcs_circuit* cc = const_cast<rcs_circuit*>(circ);
        std::lock_guard<std::mutex> lk(cc->mu);
        auto key = std::make_tuple(pkey, plan_g, nl);
        auto f = cc->packs.find(key);
        if (f != cc->packs.end()) {
            tcp = f->second;
        } else {
            auto np = std::make_shared<TcPack>();
            make_tc_pack(P, nl, *np);
            tcp = np;
            cc->packs[key] = tcp;
        }
    }
    const std::vector<int>& tc_slot = tcp->slot;
    const int n_tc = tcp->n_tc;
    const size_t tc_words_each = dev::tc_matrix_words();
    const size_t tc_words = (size_t)n_tc * tc_words_each;
    const bool tc_upload = n_tc > 0 && !(ctx->tc_uid == circ->uid && ctx->tc_pack == tcp.get());
    if (tc_upload && ctx->tc_cap < tc_words) {
        if (ctx->d_tc) cudaFree(ctx->d_tc);
        ctx->d_tc = nullptr;
        ctx->tc_cap = 0;
        BUILD_TRY(cudaMalloc(&ctx->d_tc, tc_words * sizeof(uint32_t)));
        ctx->tc_cap = tc_words;
    }
    // product-state prefix: cached per (circuit, plan), device copy per context
    const int n_prefix = P.prefix;
    std::shared_ptr<const PrefixPack> pfp;
    size_t pf_bytes[3] = {0, 0, 0};
    bool pf_upload = false;
    if (n_prefix > 0) {
        rcs_circuit* cc = const_cast<rcs_circuit*>(circ);
        std::lock_guard<std::mutex> lk(cc->mu);
        auto key = std::make_pair(pkey, plan_g);
        auto f = cc->prefix_packs.find(key);
        if (f != cc->prefix_packs.end()) {
            pfp = f->second;
        } else {
            auto np = std::make_shared<PrefixPack>();
            make_prefix_pack(P, *np);
            pfp = np;
            cc->prefix_packs[key] = pfp;
        }
        pf_bytes[0] = pfp->tab[0].size() * sizeof(float);
        pf_bytes[1] = pfp->tab[1].size() * sizeof(float);
        pf_bytes[2] = pfp->byt.size() * sizeof(uint32_t);
        const size_t need = pf_bytes[0] + pf_bytes[1] + pf_bytes[2];
        pf_upload = !(ctx->pf_pack == pfp.get());
        if (pf_upload && ctx->pf_cap < need) {
            if (ctx->d_pf) cudaFree(ctx->d_pf);
            ctx->d_pf = nullptr;
            ctx->pf_cap = 0;
            BUILD_TRY(cudaMalloc(&ctx->d_pf, need));
            ctx->pf_cap = need;
        }
    }
    if (ctx->world > 1 && P.n_remaps > 0) {
        rcs_status r = setup_peers(ctx, s->amps, o.remap_mode, err);
        if (r) return fail(r);
    }
    if (n_tc > 0 && !ctx->d_tiles && o.tc_schedule == 1) BUILD_TRY(cudaMalloc(&ctx->d_tiles, 64));
    s->tiles = o.tc_schedule == 1 ? ctx->d_tiles : nullptr;
    s->tc_flags = (o.tc_kernel == 1 ? dev::kTcForceK9 : 0) | (o.tc_kernel == 2 ? dev::kTcNoRow : 0) |
                  (o.tc_tma == -1 ? dev::kTcBulkRuns : 0);
    BUILD_TRY(cudaEventRecord(eb0, stream));
    cudaEvent_t epf0 = nullptr;
    if (tc_upload) {
        BUILD_TRY(cudaMemcpyAsync(ctx->d_tc, tcp->words.data(), tc_words * sizeof(uint32_t), cudaMemcpyHostToDevice,
                                  stream));
        ctx->tc_uid = circ->uid;
        ctx->tc_pack = tcp.get();
        ctx->tc_hold = tcp;
    }
    if (n_prefix > 0) {
        if (pf_upload) {
            BUILD_TRY(cudaMemcpyAsync(ctx->d_pf, pfp->tab[0].data(), pf_bytes[0], cudaMemcpyHostToDevice, stream));
            BUILD_TRY(cudaMemcpyAsync(ctx->d_pf + pf_bytes[0], pfp->tab[1].data(), pf_bytes[1], cudaMemcpyHostToDevice,
                                      stream));
            BUILD_TRY(cudaMemcpyAsync(ctx->d_pf + pf_bytes[0] + pf_bytes[1], pfp->byt.data(), pf_bytes[2],
                                      cudaMemcpyHostToDevice, stream));
            ctx->pf_pack = pfp.get();
            ctx->pf_hold = pfp;
        }
        if (o.timing) {
            BUILD_TRY(cudaEventCreate(&epf0));
            owned.push_back(epf0);
            BUILD_TRY(cudaEventRecord(epf0, stream));
        }
        dev::PrefixArgs pa{};
        pa.amps = s->amps;
        pa.n_amps = n_amps;
        pa.base = (uint64_t)ctx->rank << nl;
        pa.tab[0] = reinterpret_cast<const float2*>(ctx->d_pf);
        pa.tab[1] = reinterpret_cast<const float2*>(ctx->d_pf + pf_bytes[0]);
        pa.byt = reinterpret_cast<const uint32_t*>(ctx->d_pf + pf_bytes[0] + pf_bytes[1]);
        pa.nbytes = pfp->nbytes;
        pa.zmask = pfp->zmask;
        BUILD_TRY(dev::product_init(pa, stream));
    } else {
        BUILD_TRY(dev::init_basis(s->amps, n_amps, ctx->rank == 0, stream));
    }
    if (keep)
        BUILD_TRY(cudaMemcpyAsync(s->ptab, ptab_host.data(), ptab_host.size() * 8, cudaMemcpyHostToDevice, stream));
    uint64_t pass_bytes = 0, remap_bytes = 0;
    int n_pipelined = 0, n_peer = 0;
    std::vector<float> mbuf;
    std::vector<Span> spans;
    const bool peer_path = (ctx->world > 1 && ctx->p2p) || loopback(s);
    // pipelined remaps (f1): 2^cb chunks, `reserve` SMs left to the swaps (sweeps: profiles/r01_ovl*)
    const int ov_cb = o.overlap_chunks > 0 ? o.overlap_chunks : 2;
    const bool ov_on = o.overlap >= 0 && ov_cb <= 4 && peer_path;
    const int ov_res = o.overlap_sms > 0 ? o.overlap_sms : (ctx->world == 2 ? 32 : 16);
    const int ov_chain = o.overlap_passes > 0 ? o.overlap_passes : kOverlapPasses;
    const int nl_loc = nl - (loopback(s) ? o.virtual_global : 0);   // local bits of one (virtual) rank
    auto is_tc = [&](size_t i) { return i < n_exec && P.items[i].type == RCS_ITEM_PASS && tc_slot[i] >= 0; };
    auto tc_ref = [&](size_t i) {
        return PassRef{tcp->pos[i].data(), ctx->d_tc + (size_t)tc_slot[i] * tc_words_each};
    };
    if (n_prefix > 0) pass_bytes += 8ull * n_amps;   // the prefix kernel only writes the state
    cudaEvent_t epf = nullptr;
    if (o.timing) {
        BUILD_TRY(cudaEventCreate(&epf));
        owned.push_back(epf);
        BUILD_TRY(cudaEventRecord(epf, stream));
    }
    for (size_t ii = (size_t)n_prefix; ii < n_exec; ii++) {
        const Item& it = P.items[ii];
        // [TC pass] -> REMAP -> [TC pass] pipelined over NVLink (or loopback)
        if (ov_on) {
            size_t ir = (it.type == RCS_ITEM_REMAP) ? ii : (is_tc(ii) && ii + 1 < n_exec &&
                                                            P.items[ii + 1].type == RCS_ITEM_REMAP) ? ii + 1 : SIZE_MAX;
            if (ir != SIZE_MAX) {
                const Item& rm = P.items[ir];
                const bool has_a = ir != ii;
                uint64_t excl = 0;
                for (int i = 0; i < rm.k; i++) excl |= 1ull << rm.b[i];
                if (has_a) excl |= dev::tc_reserved_mask(nl, tcp->pos[ii].data());
                int fix[4];
                // the passes after the remap that run chunk by chunk behind the swaps: up to
                // ov_chain consecutive tensor-core passes whose tile cubes leave ov_cb chunk bits,
                // stopping before a pass that feeds the next remap (that one is the next group's A)
                std::vector<PassRef> rb;
                std::vector<size_t> ib;
                for (size_t k = ir + 1; k < n_exec && (int)rb.size() < ov_chain && is_tc(k); k++) {
                    if (!rb.empty() && k + 1 < n_exec && P.items[k + 1].type == RCS_ITEM_REMAP) break;
                    const uint64_t ex = excl | dev::tc_reserved_mask(nl, tcp->pos[k].data());
                    int f2[4];
                    if (!choose_chunk_bits(nl_loc, ex, ov_cb, f2)) break;
                    excl = ex;
                    rb.push_back(tc_ref(k));
                    ib.push_back(k);
                }
                if ((has_a || !rb.empty()) && choose_chunk_bits(nl_loc, excl, ov_cb, fix)) {
                    PassRef ra = has_a ? tc_ref(ii) : PassRef{};
                    rcs_status r = do_remap_pipelined(s, rm, has_a ? &ra : nullptr, rb.data(), (int)rb.size(), fix,
                                                      ov_cb, ov_res, &remap_bytes, &pass_bytes, ii, ir,
                                                      ib.data(), o.timing ? &spans : nullptr, &owned, err);
                    if (r) return fail(r);
                    n_pipelined++;
                    n_peer++;
                    ii = rb.empty() ? ir : ib.back();
                    continue;
                }
            }
        }
        cudaEvent_t e0 = nullptr;
        if (o.timing) {
            BUILD_TRY(cudaEventCreate(&e0));
            owned.push_back(e0);
            BUILD_TRY(cudaEventRecord(e0, stream));
        }
        if (it.type == RCS_ITEM_PASS && tc_slot[ii] >= 0) {
            BUILD_TRY(dev::gate_pass_tc(s->amps, nl, tcp->pos[ii].data(), ctx->d_tc + (size_t)tc_slot[ii] * tc_words_each,
                                        ctx->num_sms, stream, nullptr, 0, 0, s->tc_flags, s->tiles));
            pass_bytes += 16ull * n_amps;
        } else if (it.type == RCS_ITEM_PASS) {
            const Block& B = P.blocks[it.block];
            mbuf.resize(2 * B.matrix.size());
            for (size_t e = 0; e < B.matrix.size(); e++) {
                mbuf[2 * e] = (float)B.matrix[e].re;
                mbuf[2 * e + 1] = (float)B.matrix[e].im;
            }
            BUILD_TRY(dev::gate_pass(s->amps, nl, it.k, it.pos, mbuf.data(), stream));
            pass_bytes += 16ull * n_amps;
        } else if (it.type == RCS_ITEM_SWAP) {
            BUILD_TRY(dev::bit_swap(s->amps, nl, it.k, it.a, it.b, stream));
        } else {  // REMAP
            if (ctx->world == 1 && !loopback(s)) {
                BUILD_TRY(dev::bit_swap(s->amps, nl, it.k, it.a, it.b, stream));
            } else {
                rcs_status r = peer_path ? do_remap_p2p(s, it, &remap_bytes, o.timing ? &spans : nullptr, &owned, err)
                                         : do_remap_nccl(s, it, &remap_bytes, o.timing ? &spans : nullptr, &owned, err);
                if (r) return fail(r);
                n_peer += peer_path ? 1 : 0;
            }
        }
        if (o.timing) {
            cudaEvent_t e1;
            BUILD_TRY(cudaEventCreate(&e1));
            owned.push_back(e1);
            BUILD_TRY(cudaEventRecord(e1, stream));
            spans.push_back({ii, e0, e1, 1});
        }
    }
    BUILD_TRY(cudaEventRecord(ec0, stream));
    s->permuted = keep;
    st = keep ? compute_cdf_kept(s, err) : compute_cdf(s, err);
    if (st) return fail(st);
    BUILD_TRY(cudaEventRecord(eb1, stream));
    BUILD_TRY(cudaStreamSynchronize(stream));

    rcs_build_report R{};
    R.n_passes = P.n_passes - n_prefix;
    R.n_prefix = n_prefix;
    R.upload_bytes = (tc_upload ? tc_words * sizeof(uint32_t) : 0) +
                     (pf_upload ? pf_bytes[0] + pf_bytes[1] + pf_bytes[2] : 0) + (keep ? ptab_host.size() * 8 : 0);
    R.n_remaps = 0;
    R.n_swaps = 0;
    for (size_t ii = 0; ii < n_exec; ii++) {   // executed items (a kept layout skips the restore)
        R.n_remaps += P.items[ii].type == RCS_ITEM_REMAP;
        R.n_swaps += P.items[ii].type == RCS_ITEM_SWAP;
    }
    R.layout_kept = keep ? 1 : 0;
    R.fuse_k = P.fuse_k;
    R.plan_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
    float ms = 0.f;
    cudaEventElapsedTime(&ms, eb0, eb1);
    R.build_ms = ms;
    float cdf_ms = 0.f;
    cudaEventElapsedTime(&cdf_ms, ec0, eb1);
    R.pass_ms_min = 1e30;
    R.pass_ms_max = 0;
    s->pass_ms.clear();
    if (o.timing) {
        R.blocksum_ms = cdf_ms;
        std::vector<double> item_ms(n_exec, 0.0);
        for (const Span& sp : spans) {
            float t = 0.f;
            if (sp.a && sp.b) cudaEventElapsedTime(&t, sp.a, sp.b);
            if (sp.item == kRemapKernelSpan) R.remap_kernel_ms += (double)t;
            else item_ms[sp.item] += sp.sign * (double)t;
        }
        if (epf0 && epf) {
            float t = 0.f;
            cudaEventElapsedTime(&t, epf0, epf);
            R.prefix_ms = t;
        }
        for (size_t ii = (size_t)n_prefix; ii < n_exec; ii++) {
            const double t = item_ms[ii];
            if (P.items[ii].type == RCS_ITEM_PASS) {
                R.pass_ms += t;
                R.pass_ms_min = std::min(R.pass_ms_min, t);
                R.pass_ms_max = std::max(R.pass_ms_max, t);
                s->pass_ms.push_back((float)t);
            } else if (P.items[ii].type == RCS_ITEM_SWAP) {
                R.swap_ms += t;
            } else {
                R.remap_ms += t;
            }
        }
    }
    for (auto& e : owned) cudaEventDestroy(e);   // includes eb0, eb1, ec0
    owned.clear();
    if (R.pass_ms_min > R.pass_ms_max) R.pass_ms_min = 0;
    R.pass_bytes = pass_bytes;
    R.remap_bytes = remap_bytes;
    R.norm = s->T_total;
    R.n_tc_passes = 0;
    for (size_t ii = (size_t)n_prefix; ii < n_exec; ii++) R.n_tc_passes += tc_slot[ii] >= 0;
    R.n_pipelined = n_pipelined;
    R.n_peer_remaps = n_peer;
    if (rep) *rep = R;
    *out = s;
    return RCS_OK;
#undef BUILD_TRY
}

rcs_status rcs_state_canonicalize(rcs_state* s, rcs_error* err) {
    if (err) std::memset(err, 0, sizeof *err);
    if (!s) { set_error(err, RCS_ERR_ARG, "null argument"); return RCS_ERR_ARG; }
    if (!s->permuted) return RCS_OK;
    rcs_context* c = s->ctx;
    CUDA_TRY(cudaSetDevice(c->device));
    const Plan& P = *s->plan;
    if (c->world > 1) {   // the peer mappings may belong to another state's buffer by now
        rcs_status r = setup_peers(c, s->amps, s->remap_mode, err);
        if (r) return r;
    }
    uint64_t bytes = 0;
    for (size_t ii = (size_t)P.restore_begin; ii < P.items.size(); ii++) {
        const Item& it = P.items[ii];
        if (it.type == RCS_ITEM_REMAP && (c->world > 1 || loopback(s))) {
            rcs_status r = (c->p2p || loopback(s)) ? do_remap_p2p(s, it, &bytes, nullptr, nullptr, err)
                                                   : do_remap_nccl(s, it, &bytes, nullptr, nullptr, err);
            if (r) return r;
        } else {
            CUDA_TRY(dev::bit_swap(s->amps, s->nl, it.k, it.a, it.b, c->stream));
        }
    }
    s->permuted = false;
    return compute_cdf(s, err);
}

rcs_status rcs_state_pass_times(const rcs_state* s, float* ms, int cap, int* n) {
    if (!s) return RCS_ERR_ARG;
    const int k = (int)s->pass_ms.size();
    if (n) *n = k;
    if (ms)
        for (int i = 0; i < std::min(cap, k); i++) ms[i] = s->pass_ms[i];
    return RCS_OK;
}

rcs_status rcs_state_norm(const rcs_state* s, double* norm) {
    if (!s || !norm) return RCS_ERR_ARG;
    *norm = s->T_total;
    return RCS_OK;
}

rcs_status rcs_state_copy_out(const rcs_state* s, uint64_t first, uint64_t count, void* dst, rcs_error* err) {
    if (err) std::memset(err, 0, sizeof *err);
    if (!s || (!dst && count)) { set_error(err, RCS_ERR_ARG, "null argument"); return RCS_ERR_ARG; }
    if (s->permuted) {
        set_error(err, RCS_ERR_ARG, "state kept in a permuted layout: call rcs_state_canonicalize first");
        return RCS_ERR_ARG;
    }
    const uint64_t base = (uint64_t)s->ctx->rank << s->nl;
    if (first < base || first + count > base + s->n_amps || first + count < first) {
        set_error(err, RCS_ERR_ARG, "range [%llu, +%llu) not on this rank", (unsigned long long)first,
                  (unsigned long long)count);
        return RCS_ERR_ARG;
    }
    CUDA_TRY(cudaSetDevice(s->ctx->device));
    CUDA_TRY(cudaMemcpyAsync(dst, s->amps + (first - base), count * sizeof(float2), cudaMemcpyDefault, s->ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(s->ctx->stream));
    return RCS_OK;
}

rcs_status rcs_probabilities(const rcs_state* s_, const uint64_t* x, uint64_t count, double* p_out, rcs_error* err) {
    if (err) std::memset(err, 0, sizeof *err);
    rcs_state* s = const_cast<rcs_state*>(s_);
    if (!s || ((!x || !p_out) && count)) { set_error(err, RCS_ERR_ARG, "null argument"); return RCS_ERR_ARG; }
    rcs_context* c = s->ctx;
    CUDA_TRY(cudaSetDevice(c->device));
    rcs_status st = ensure_buffers(s, err);
    if (st) return st;
    const bool xd = count ? is_device_ptr(x) : true, pd = count ? is_device_ptr(p_out) : true;
    CUDA_TRY(cudaMemsetAsync(s->bad, 0, sizeof(int), c->stream));
    for (uint64_t i0 = 0; i0 < count; i0 += s->chunk) {
        const uint64_t cnt = std::min(s->chunk, count - i0);
        const unsigned long long* xi = reinterpret_cast<const unsigned long long*>(x) + i0;
        if (!xd) {
            CUDA_TRY(cudaMemcpyAsync(s->xbuf, x + i0, cnt * 8, cudaMemcpyHostToDevice, c->stream));
            xi = s->xbuf;
        }
        double* po = pd ? p_out + i0 : s->dbuf;
        CUDA_TRY(dev::gather_prob(s->amps, xi, cnt, locator(s), s->n, po, s->bad, c->stream));
        if (c->world > 1) NCCL_TRY(ncclAllReduce(po, po, cnt, ncclDouble, ncclSum, c->comm, c->stream));
        if (!pd) CUDA_TRY(cudaMemcpyAsync(p_out + i0, po, cnt * 8, cudaMemcpyDeviceToHost, c->stream));
    }
    int bad = 0;
    CUDA_TRY(cudaMemcpyAsync(&bad, s->bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    if (bad) { set_error(err, RCS_ERR_SIZE, "bitstring >= 2^%d", s->n); return RCS_ERR_SIZE; }
    return RCS_OK;
}

rcs_status rcs_sample(rcs_state* s, uint64_t shots, uint64_t seed, uint64_t offset, uint64_t* out_x,
                      rcs_sample_report* rep, rcs_error* err) {
    if (err) std::memset(err, 0, sizeof *err);
    return sample_impl(s, shots, seed, offset, nullptr, out_x, rep, err);
}

rcs_status rcs_sample_uniforms(rcs_state* s, const double* u, uint64_t shots, uint64_t* out_x, rcs_sample_report* rep,
                               rcs_error* err) {
    if (err) std::memset(err, 0, sizeof *err);
    if (!u && shots) { set_error(err, RCS_ERR_ARG, "null uniforms"); return RCS_ERR_ARG; }
    return sample_impl(s, shots, 0, 0, u, out_x, rep, err);
}

rcs_status rcs_xeb(const rcs_state* s_, const uint64_t* x, uint64_t count, rcs_xeb_report* out, rcs_error* err) {
    if (err) std::memset(err, 0, sizeof *err);
    rcs_state* s = const_cast<rcs_state*>(s_);
    if (!s || !out || (!x && count)) { set_error(err, RCS_ERR_ARG, "null argument"); return RCS_ERR_ARG; }
    if (count == 0) { set_error(err, RCS_ERR_ARG, "XEB needs at least one bitstring"); return RCS_ERR_ARG; }
    rcs_context* c = s->ctx;
    CUDA_TRY(cudaSetDevice(c->device));
    rcs_status st = ensure_buffers(s, err);
    if (st) return st;
    const bool xd = is_device_ptr(x);
    const int grid = dev::xeb_grid();
    double* acc = s->xeb_part + 3 * grid;   // 3 running totals (fixed chunk order)
    std::vector<double> tot(3, 0.0);
    CUDA_TRY(cudaMemsetAsync(s->bad, 0, sizeof(int), c->stream));
    for (uint64_t i0 = 0; i0 < count; i0 += s->chunk) {
        const uint64_t cnt = std::min(s->chunk, count - i0);
        const unsigned long long* xi = reinterpret_cast<const unsigned long long*>(x) + i0;
        if (!xd) {
            CUDA_TRY(cudaMemcpyAsync(s->xbuf, x + i0, cnt * 8, cudaMemcpyHostToDevice, c->stream));
            xi = s->xbuf;
        }
        CUDA_TRY(dev::xeb_partials(s->amps, xi, cnt, locator(s), s->n, s->xeb_part, s->bad, c->stream));
        CUDA_TRY(dev::xeb_finalize(s->xeb_part, grid, acc, c->stream));
        if (c->world > 1) NCCL_TRY(ncclAllReduce(acc, acc, 3, ncclDouble, ncclSum, c->comm, c->stream));
        double part[3];
        CUDA_TRY(cudaMemcpyAsync(part, acc, sizeof part, cudaMemcpyDeviceToHost, c->stream));
        CUDA_TRY(cudaStreamSynchronize(c->stream));
        for (int q = 0; q < 3; q++) tot[q] += part[q];
    }
    int bad = 0;
    CUDA_TRY(cudaMemcpyAsync(&bad, s->bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    if (bad) { set_error(err, RCS_ERR_SIZE, "bitstring >= 2^%d", s->n); return RCS_ERR_SIZE; }
    const double S = (double)count;
    const double mean = tot[0] / S;
    double var = count > 1 ? (tot[1] - S * mean * mean) / (S - 1.0) : 0.0;
    if (var < 0) var = 0;
    out->n_qubits = s->n;
    out->shots = count;
    out->mean_p = mean;
    out->F = std::ldexp(mean, s->n) - 1.0;
    out->sigma = std::ldexp(std::sqrt(var), s->n) / std::sqrt(S);
    out->fstar = std::ldexp(s->sum_sq, s->n) - 1.0;
    return RCS_OK;
}

// ---- paper stages 2-3: snapshot file + sampler-job helpers -----------------
rcs_status rcs_sha256(const void* data, uint64_t bytes, uint8_t digest[32]) {
    if ((!data && bytes) || !digest) return RCS_ERR_ARG;
    Sha256 h;
    h.update(data, bytes);
    h.final(digest);
    return RCS_OK;
}

namespace {
constexpr uint64_t kSnapChunk = 1ull << 22;   // amplitudes per host<->device chunk (32 MB f32)

struct HostBuf {   // pinned staging for the snapshot streams
    void* p = nullptr;
    ~HostBuf() {
        if (p) cudaFreeHost(p);
    }
};
}  // namespace

rcs_status rcs_snapshot_save(const rcs_state* s, const char* path, uint8_t digest[32], rcs_error* err) {
    if (err) std::memset(err, 0, sizeof *err);
    if (!s || !path) { set_error(err, RCS_ERR_ARG, "null argument"); return RCS_ERR_ARG; }
    rcs_context* c = s->ctx;
    if (c->world != 1) { set_error(err, RCS_ERR_ARG, "snapshot needs a single-rank state"); return RCS_ERR_ARG; }
    if (s->permuted) {
        set_error(err, RCS_ERR_ARG, "state kept in a permuted layout: call rcs_state_canonicalize first");
        return RCS_ERR_ARG;
    }
    CUDA_TRY(cudaSetDevice(c->device));
    HostBuf hb;
    CUDA_TRY(cudaMallocHost(&hb.p, kSnapChunk * sizeof(float2)));
    std::vector<double> wide(2 * kSnapChunk);
    const std::string tmp = std::string(path) + ".tmp." + std::to_string((long long)getpid());
    FILE* f = std::fopen(tmp.c_str(), "wb");
    if (!f) { set_error(err, RCS_ERR_IO, "cannot create %s", tmp.c_str()); return RCS_ERR_IO; }
    auto io_fail = [&](const char* what) {
        std::fclose(f);
        std::remove(tmp.c_str());
        set_error(err, RCS_ERR_IO, "%s %s", what, tmp.c_str());
        return RCS_ERR_IO;
    };
    uint8_t hdr[kSnapHeaderBytes] = {0};
    if (std::fwrite(hdr, 1, kSnapHeaderBytes, f) != (size_t)kSnapHeaderBytes) return io_fail("write failed:");
    Sha256 h;
    for (uint64_t i0 = 0; i0 < s->n_amps; i0 += kSnapChunk) {
        const uint64_t cnt = std::min(kSnapChunk, s->n_amps - i0);
        cudaError_t e = cudaMemcpyAsync(hb.p, s->amps + i0, cnt * sizeof(float2), cudaMemcpyDeviceToHost, c->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
        if (e != cudaSuccess) {
            std::fclose(f);
            std::remove(tmp.c_str());
            set_error(err, RCS_ERR_CUDA, "snapshot copy: %s", cudaGetErrorString(e));
            return RCS_ERR_CUDA;
        }
        const float* src = static_cast<const float*>(hb.p);
        for (uint64_t k = 0; k < 2 * cnt; k++) wide[k] = (double)src[k];   // exact widening
        h.update(wide.data(), cnt * 16);   // little-endian host (x86-64 / aarch64)
        if (std::fwrite(wide.data(), 16, cnt, f) != cnt) return io_fail("write failed:");
    }
    uint8_t dg[32];
    h.final(dg);
    put_snapshot_header(hdr, (uint32_t)s->n, dg);
    if (std::fseek(f, 0, SEEK_SET) != 0 || std::fwrite(hdr, 1, kSnapHeaderBytes, f) != (size_t)kSnapHeaderBytes)
        return io_fail("header write failed:");
    if (std::fflush(f) != 0 || fsync(fileno(f)) != 0) return io_fail("flush failed:");
    if (std::fclose(f) != 0) {
        std::remove(tmp.c_str());
        set_error(err, RCS_ERR_IO, "close failed: %s", tmp.c_str());
        return RCS_ERR_IO;
    }
    if (std::rename(tmp.c_str(), path) != 0) {
        std::remove(tmp.c_str());
        set_error(err, RCS_ERR_IO, "rename to %s failed", path);
        return RCS_ERR_IO;
    }
    if (digest) std::memcpy(digest, dg, 32);
    return RCS_OK;
}

namespace {
rcs_status read_header(FILE* f, const char* path, SnapHeader* H, rcs_error* err) {
    uint8_t hdr[kSnapHeaderBytes];
    if (std::fread(hdr, 1, kSnapHeaderBytes, f) != (size_t)kSnapHeaderBytes) {
        set_error(err, RCS_ERR_FORMAT, "%s: truncated header", path);
        return RCS_ERR_FORMAT;
    }
    const char* why = nullptr;
    if (!get_snapshot_header(hdr, H, &why)) {
        set_error(err, RCS_ERR_FORMAT, "%s: %s", path, why);
        return RCS_ERR_FORMAT;
    }
    return RCS_OK;
}
}  // namespace

rcs_status rcs_snapshot_info(const char* path, int* n_qubits, uint64_t* payload_bytes, uint8_t digest[32],
                             rcs_error* err) {
    if (err) std::memset(err, 0, sizeof *err);
    if (!path) { set_error(err, RCS_ERR_ARG, "null argument"); return RCS_ERR_ARG; }
    FILE* f = std::fopen(path, "rb");
    if (!f) { set_error(err, RCS_ERR_IO, "cannot open %s", path); return RCS_ERR_IO; }
    SnapHeader H;
    rcs_status st = read_header(f, path, &H, err);
    std::fclose(f);
    if (st) return st;
    if (n_qubits) *n_qubits = (int)H.n_qubits;
    if (payload_bytes) *payload_bytes = H.payload_bytes;
    if (digest) std::memcpy(digest, H.digest, 32);
    return RCS_OK;
}

rcs_status rcs_snapshot_scratch_bytes(const rcs_context* ctx, int n_qubits, int block_bits, uint64_t* bytes) {
    if (!ctx || !bytes || n_qubits < 1 || ctx->world != 1) return RCS_ERR_ARG;
    *bytes = scratch_layout(n_qubits, 1, 0, 0, block_bits).total;
    return RCS_OK;
}

rcs_status rcs_snapshot_load(rcs_context* ctx, const char* path, int block_bits, void* d_amps, uint64_t amps_bytes,
                             void* d_scratch, uint64_t scratch_bytes, rcs_state** out, rcs_error* err) {
    if (err) std::memset(err, 0, sizeof *err);
    if (!ctx || !path || !d_amps || !out) { set_error(err, RCS_ERR_ARG, "null argument"); return RCS_ERR_ARG; }
    if (ctx->world != 1) { set_error(err, RCS_ERR_ARG, "snapshot load needs a single-rank context"); return RCS_ERR_ARG; }
    FILE* f = std::fopen(path, "rb");
    if (!f) { set_error(err, RCS_ERR_IO, "cannot open %s", path); return RCS_ERR_IO; }
    struct Closer {
        FILE* f;
        ~Closer() { std::fclose(f); }
    } closer{f};
    SnapHeader H;
    rcs_status st = read_header(f, path, &H, err);
    if (st) return st;
    const int n = (int)H.n_qubits;
    if (n < 1) { set_error(err, RCS_ERR_FORMAT, "%s: n_qubits = 0", path); return RCS_ERR_FORMAT; }
    const uint64_t n_amps = 1ull << n;
    if (amps_bytes < n_amps * 8) {
        set_error(err, RCS_ERR_MEMORY, "amplitude buffer too small: need %llu bytes", (unsigned long long)(n_amps * 8));
        if (err) err->bytes_required = n_amps * 8;
        return RCS_ERR_MEMORY;
    }
    const Layout L = scratch_layout(n, 1, 0, 0, block_bits);
    if (!d_scratch || scratch_bytes < L.total) {
        set_error(err, RCS_ERR_MEMORY, "scratch buffer too small: need %llu bytes", (unsigned long long)L.total);
        if (err) err->bytes_required = L.total;
        return RCS_ERR_MEMORY;
    }
    CUDA_TRY(cudaSetDevice(ctx->device));
    HostBuf hb;
    CUDA_TRY(cudaMallocHost(&hb.p, kSnapChunk * sizeof(float2)));
    std::vector<double> wide(2 * kSnapChunk);
    float2* amps = reinterpret_cast<float2*>(d_amps);
    Sha256 h;
    for (uint64_t i0 = 0; i0 < n_amps; i0 += kSnapChunk) {
        const uint64_t cnt = std::min(kSnapChunk, n_amps - i0);
        if (std::fread(wide.data(), 16, cnt, f) != cnt) {
            set_error(err, RCS_ERR_FORMAT, "%s: truncated payload", path);
            return RCS_ERR_FORMAT;
        }
        h.update(wide.data(), cnt * 16);
        CUDA_TRY(cudaStreamSynchronize(ctx->stream));   // previous chunk's copy done with hb
        float* dst = static_cast<float*>(hb.p);
        for (uint64_t k = 0; k < 2 * cnt; k++) dst[k] = (float)wide[k];   // round to nearest
        CUDA_TRY(cudaMemcpyAsync(amps + i0, hb.p, cnt * sizeof(float2), cudaMemcpyHostToDevice, ctx->stream));
    }
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    uint8_t dg[32];
    h.final(dg);
    if (std::memcmp(dg, H.digest, 32) != 0) {
        set_error(err, RCS_ERR_DIGEST, "%s: payload digest mismatch", path);
        return RCS_ERR_DIGEST;
    }
    rcs_state* s = new (std::nothrow) rcs_state();
    if (!s) return RCS_ERR_MEMORY;
    s->ctx = ctx;
    s->n = n;
    s->g = 0;
    s->nl = n;
    s->amps = amps;
    s->n_amps = n_amps;
    char* sc = reinterpret_cast<char*>(d_scratch);
    s->b = L.b;
    s->nblocks = L.nblocks;
    s->inc = reinterpret_cast<double*>(sc + L.inc_off);
    s->scan_tmp = reinterpret_cast<double*>(sc + L.tmp_off);
    s->part_sq = reinterpret_cast<double*>(sc + L.part_off);
    s->misc = reinterpret_cast<double*>(sc + L.misc_off);
    s->staging = reinterpret_cast<float2*>(sc + L.stage_off);
    s->staging_elems = (L.stage_end - L.stage_off) / sizeof(float2);
    st = compute_cdf(s, err);
    if (st) {
        delete s;
        return st;
    }
    if (!(std::fabs(s->T_total - 1.0) <= 1e-5)) {
        set_error(err, RCS_ERR_NORM, "%s: norm %.9f", path, s->T_total);
        delete s;
        return RCS_ERR_NORM;
    }
    *out = s;
    return RCS_OK;
}

rcs_status rcs_shard_shots(uint64_t total, int n_jobs, uint64_t* counts) {
    if (n_jobs < 1 || !counts) return RCS_ERR_ARG;
    const uint64_t q = total / (uint64_t)n_jobs, r = total % (uint64_t)n_jobs;
    for (int j = 0; j < n_jobs; j++) counts[j] = q + ((uint64_t)j < r ? 1 : 0);
    return RCS_OK;
}

uint64_t rcs_job_seed(uint64_t base_seed, uint64_t job_id) { return job_seed(base_seed, job_id); }

rcs_status rcs_xeb_from_probs(int n_qubits, const double* p, uint64_t count, rcs_xeb_report* out) {
    if (!out || (!p && count) || n_qubits < 1 || n_qubits > 63 || count == 0) return RCS_ERR_ARG;
    double sum = 0.0;
    for (uint64_t i = 0; i < count; i++) sum += p[i];
    const double S = (double)count, mean = sum / S;
    double ss = 0.0;
    for (uint64_t i = 0; i < count; i++) ss += (p[i] - mean) * (p[i] - mean);
    const double var = count > 1 ? ss / (S - 1.0) : 0.0;
    out->n_qubits = n_qubits;
    out->shots = count;
    out->mean_p = mean;
    out->F = std::ldexp(mean, n_qubits) - 1.0;
    out->sigma = std::ldexp(std::sqrt(var), n_qubits) / std::sqrt(S);
    out->fstar = std::nan("");
    return RCS_OK;
}

void rcs_state_free(rcs_state* s) {
    if (!s) return;
    if (s->ctx) cudaSetDevice(s->ctx->device);
    // chunk buffers belong to the context
    delete s;
}

}  // extern "C"
