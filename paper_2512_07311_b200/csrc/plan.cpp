// plan.cpp -- host planner: k-qubit gate fusion + global-qubit remap schedule.
//
// BASELINE.json north_star: "gates are fused into k-qubit dense blocks and applied in
// place ... The state vector shards ... on its top log2(P) 'global' qubits.  Gates touching
// global qubits trigger a qubit-remap all-to-all".  The paper itself publishes no algorithm
// (SURVEY §0), so the fuser and planner below are this library's design.
//
// 1. Fusion (independent of P, so P = 1/2/4/8 states are bit-identical):
//    closure-greedy.  A block starts from the earliest unassigned gate; its qubit set S is
//    grown one extension at a time (the qubits of a gate at the block's frontier) choosing
//    the extension whose closure -- every gate that becomes applicable inside S, repeatedly
//    -- absorbs the most gates, until |S| = k or nothing grows.  Gates inside a block are
//    applied in absorption order, which respects every per-qubit dependency.  The block
//    matrix is the fp64 product of its gates (cast to complex64 on upload).
// 2. Remaps (P > 1): logical->physical layout; when a block needs qubits living on global
//    positions, each is swapped with a local qubit chosen by Belady (farthest next use).
//    Physical positions < kPinnedLow never move.
// 3. Final restore: <= 3 remaps bring the top-g qubits home, then <= 2 involutive bit-swap
//    passes (a cycle is the product of two reflections) restore canonical local order.
#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <map>
#include <set>
#include <thread>

#include "internal.h"

namespace rcs {

namespace {

struct Fuser {
    const Circuit& C;
    int k;
    std::vector<std::vector<int>> per_q;   // gate ids per qubit, source order
    std::vector<int> head;                 // first unassigned position in per_q[q]
    std::vector<char> assigned;

    int seeds = 0;

    Fuser(const Circuit& c, int k_) : C(c), k(k_) {
        per_q.assign(c.n, {});
        for (int i = 0; i < (int)c.gates.size(); i++) {
            per_q[c.gates[i].q0].push_back(i);
            if (c.gates[i].q1 >= 0) per_q[c.gates[i].q1].push_back(i);
        }
        head.assign(c.n, 0);
        assigned.assign(c.gates.size(), 0);
    }

    int nq(int g) const { return C.gates[g].q1 >= 0 ? 2 : 1; }
    int qb(int g, int j) const { return j == 0 ? C.gates[g].q0 : C.gates[g].q1; }

    // gates absorbed by qubit set S (sorted) starting from the current heads
    std::vector<int> closure(const std::vector<int>& S) const {
        std::map<int, int> h;
        for (int q : S) h[q] = head[q];
        std::vector<int> got;
        bool progress = true;
        while (progress) {
            progress = false;
            for (int q : S) {
                int pos = h[q];
                if (pos >= (int)per_q[q].size()) continue;
                int g = per_q[q][pos];
                bool ok = true;
                for (int j = 0; j < nq(g); j++) {
                    auto it = h.find(qb(g, j));
                    if (it == h.end() || it->second >= (int)per_q[qb(g, j)].size() ||
                        per_q[qb(g, j)][it->second] != g) {
                        ok = false;
                        break;
                    }
                }
                if (!ok) continue;
                for (int j = 0; j < nq(g); j++) h[qb(g, j)]++;
                got.push_back(g);
                progress = true;
            }
        }
        return got;
    }

    static std::vector<int> merged(const std::vector<int>& S, const std::vector<int>& ext) {
        std::vector<int> r = S;
        for (int q : ext)
            if (!std::count(r.begin(), r.end(), q)) r.push_back(q);
        std::sort(r.begin(), r.end());
        return r;
    }

    // candidate extensions of qubit set S (closure cur): the qubits of the next gate on a qubit
    // of S, or of a gate that is ready elsewhere (disjoint from S), within k qubits
    std::set<std::vector<int>> extensions(const std::vector<int>& S, const std::vector<int>& cur) const {
        std::map<int, int> h;
        for (int q : S) h[q] = head[q];
        for (int g : cur)
            for (int j = 0; j < nq(g); j++) h[qb(g, j)]++;
        std::set<std::vector<int>> cands;
        for (int q : S) {
            if (h[q] >= (int)per_q[q].size()) continue;
            int g = per_q[q][h[q]];
            std::vector<int> ext;
            for (int j = 0; j < nq(g); j++)
                if (!std::count(S.begin(), S.end(), qb(g, j))) ext.push_back(qb(g, j));
            if (!ext.empty() && (int)(S.size() + ext.size()) <= k) cands.insert(ext);
        }
        for (int q = 0; q < C.n; q++) {
            if (std::count(S.begin(), S.end(), q) || head[q] >= (int)per_q[q].size()) continue;
            int g = per_q[q][head[q]];
            bool ready = true;
            std::vector<int> ext;
            for (int j = 0; j < nq(g); j++) {
                int qq = qb(g, j);
                if (per_q[qq][head[qq]] != g) ready = false;
                if (!std::count(S.begin(), S.end(), qq)) ext.push_back(qq);
            }
            if (ready && (int)(S.size() + ext.size()) <= k) {
                std::sort(ext.begin(), ext.end());
                cands.insert(ext);
            }
        }
        return cands;
    }

    int weight(const std::vector<int>& gates) const {   // 2q gates count double
        int w = 0;
        for (int g : gates) w += nq(g);
        return w;
    }

    // greedy continuation: add the extension with the largest gain per added qubit until k
    void grow_from(std::vector<int>& S, std::vector<int>& cur) const {
        while ((int)S.size() < k) {
            const int base = weight(cur);
            int bgain = 0;
            std::vector<int> best_ext, best_cl;
            for (const auto& ext : extensions(S, cur)) {
                std::vector<int> cl = closure(merged(S, ext));
                const int gain = weight(cl) - base;
                if (gain <= 0) continue;
                // prefer larger gain per added qubit, then fewer qubits
                if (best_cl.empty() || gain * (int)best_ext.size() > bgain * (int)ext.size() ||
                    (gain * (int)best_ext.size() == bgain * (int)ext.size() && ext.size() < best_ext.size())) {
                    best_ext = ext;
                    best_cl = cl;
                    bgain = gain;
                }
            }
            if (best_cl.empty()) break;
            S = merged(S, best_ext);
            cur = best_cl;
        }
    }

    // growth of a block seeded by ready gate g0 (qubit set S, absorbed gates cur); with
    // `grow_lookahead`, every step tries each extension followed by the greedy continuation and
    // keeps the one whose finished block absorbs the most
    bool grow_lookahead = false;
    void grow(int g0, std::vector<int>& S, std::vector<int>& cur) const {
        S.clear();
        for (int j = 0; j < nq(g0); j++) S.push_back(qb(g0, j));
        std::sort(S.begin(), S.end());
        cur = closure(S);
        if (!grow_lookahead) {
            grow_from(S, cur);
            return;
        }
        while ((int)S.size() < k) {
            const int base = weight(cur);
            int best = -1;
            std::vector<int> bS, bcur;
            for (const auto& ext : extensions(S, cur)) {
                std::vector<int> S1 = merged(S, ext), c1 = closure(S1);
                if (weight(c1) <= base) continue;
                grow_from(S1, c1);
                const int w = weight(c1);
                if (w > best) {
                    best = w;
                    bS = S1;
                    bcur = c1;
                }
            }
            if (best < 0) break;
            S = bS;   // the finished block of the best first step
            cur = bcur;
            break;
        }
    }

    bool ready(int g) const {
        for (int j = 0; j < nq(g); j++) {
            const int q = qb(g, j);
            if (head[q] >= (int)per_q[q].size() || per_q[q][head[q]] != g) return false;
        }
        return true;
    }

    void commit(const std::vector<int>& cur) {
        for (int g : cur) {
            assigned[g] = 1;
            for (int j = 0; j < nq(g); j++) head[qb(g, j)]++;
        }
    }

    // number of blocks the plain greedy (earliest-gate seed) needs from the current state
    int rollout() const {
        Fuser f = *this;
        f.seeds = 0;
        f.lookahead = false;
        f.grow_lookahead = false;
        int n = 0;
        Block b;
        while (f.next_block(b)) n++;
        return n;
    }

    bool lookahead = false;

    // next block: grow from the earliest unassigned gate and from up to `seeds` other ready
    // gates; keep the block absorbing the most gate-qubits (2q gates count double), or with
    // `lookahead`, the one whose greedy completion needs the fewest blocks
    bool next_block(Block& B) {
        int g0 = -1;
        for (int i = 0; i < (int)assigned.size(); i++)
            if (!assigned[i]) { g0 = i; break; }
        if (g0 < 0) return false;
        std::vector<int> cand{g0};
        for (int i = g0 + 1; i < (int)assigned.size() && (int)cand.size() < 1 + seeds; i++)
            if (!assigned[i] && ready(i)) cand.push_back(i);
        std::vector<int> S, cur, bS, bcur;
        long best = LONG_MIN;
        if (lookahead && cand.size() > 1) {
            // candidates are independent (each grows + rolls out on its own copy): one thread
            // each, then the same fixed-order choice as the serial loop (deterministic)
            const size_t nc = cand.size();
            std::vector<std::vector<int>> cS(nc), ccur(nc);
            std::vector<long> sc(nc);
            auto work = [&](size_t i) {
                grow(cand[i], cS[i], ccur[i]);
                long score = 0;
                for (int x : ccur[i]) score += nq(x);
                Fuser f = *this;
                f.commit(ccur[i]);
                sc[i] = -1000L * f.rollout() + score;   // fewest remaining blocks, then most gates now
            };
            std::vector<std::thread> th;
            for (size_t i = 1; i < nc; i++) th.emplace_back(work, i);
            work(0);
            for (auto& t : th) t.join();
            for (size_t i = 0; i < nc; i++)
                if (sc[i] > best) {
                    best = sc[i];
                    bS = cS[i];
                    bcur = ccur[i];
                }
        } else {
            for (int g : cand) {
                grow(g, S, cur);
                long score = 0;
                for (int x : cur) score += nq(x);
                if (score > best) {
                    best = score;
                    bS = S;
                    bcur = cur;
                }
            }
        }
        S = bS;
        cur = bcur;
        // commit
        B.qubits = S;
        B.gate_ids = cur;
        for (int g : cur) {
            assigned[g] = 1;
            for (int j = 0; j < nq(g); j++) head[qb(g, j)]++;
        }
        return true;
    }
};

// U <- G_embedded U  for every column, G acting on block-local bits lb0 (, lb1)
void apply_to_block(std::vector<cplx>& U, int kb, const Gate& g, int lb0, int lb1) {
    const int D = 1 << kb;
    cplx m[16];
    gate_matrix(g, m);
    if (g.q1 < 0) {
        for (int col = 0; col < D; col++)
            for (int i = 0; i < D; i++) {
                if (i & (1 << lb0)) continue;
                const int i1 = i | (1 << lb0);
                cplx a = U[(size_t)i * D + col], b = U[(size_t)i1 * D + col];
                U[(size_t)i * D + col] = {m[0].re * a.re - m[0].im * a.im + m[1].re * b.re - m[1].im * b.im,
                                          m[0].re * a.im + m[0].im * a.re + m[1].re * b.im + m[1].im * b.re};
                U[(size_t)i1 * D + col] = {m[2].re * a.re - m[2].im * a.im + m[3].re * b.re - m[3].im * b.im,
                                           m[2].re * a.im + m[2].im * a.re + m[3].re * b.im + m[3].im * b.re};
            }
        return;
    }
    for (int col = 0; col < D; col++)
        for (int i = 0; i < D; i++) {
            if (i & ((1 << lb0) | (1 << lb1))) continue;
            int idx[4] = {i, i | (1 << lb0), i | (1 << lb1), i | (1 << lb0) | (1 << lb1)};
            cplx v[4], o[4];
            for (int t = 0; t < 4; t++) v[t] = U[(size_t)idx[t] * D + col];
            for (int r = 0; r < 4; r++) {
                double re = 0, im = 0;
                for (int c = 0; c < 4; c++) {
                    re += m[4 * r + c].re * v[c].re - m[4 * r + c].im * v[c].im;
                    im += m[4 * r + c].re * v[c].im + m[4 * r + c].im * v[c].re;
                }
                o[r] = {re, im};
            }
            for (int t = 0; t < 4; t++) U[(size_t)idx[t] * D + col] = o[t];
        }
}

}  // namespace

rcs_status build_plan(const Circuit& c, int fuse_k, int n_global, Plan& out, rcs_error* err) {
    if (fuse_k > 6) {
        set_error(err, RCS_ERR_ARG, "fuse_k must be in [1, 6] (got %d)", fuse_k);
        return RCS_ERR_ARG;
    }
    const int n = c.n;
    if (n_global < 0 || n_global >= n) {
        set_error(err, RCS_ERR_ARG, "n_global=%d invalid for n=%d", n_global, n);
        return RCS_ERR_ARG;
    }
    const int n_local = n - n_global;
    // default: 6-qubit blocks on the tensor cores when a 12-bit tile fits, else 4 on CUDA cores
    if (fuse_k <= 0) fuse_k = n_local >= kTcMinLocal ? 6 : 4;
    // 6-qubit blocks run only on the tensor-core pass, which needs n_local >= 12
    if (fuse_k == 6 && n_local < kTcMinLocal) fuse_k = 5;
    int k = std::min(fuse_k, n_local);
    if (n_global > 0 && n_local - kPinnedLow < k) {
        set_error(err, RCS_ERR_ARG, "too many global qubits: n=%d g=%d leaves %d movable local qubits < k=%d",
                  n, n_global, n_local - kPinnedLow, k);
        return RCS_ERR_ARG;
    }
    Plan P;
    P.n = n;
    P.n_global = n_global;
    P.fuse_k = k;

    // ---- 1. fusion: two growth strategies (plain greedy, greedy with one-step lookahead) run in
    // parallel; the one needing fewer blocks wins (ties: plain).  Both are deterministic and
    // independent of the sharding, so the plan stays P-invariant.
    const int seeds = getenv("RCS_FUSE_SEEDS") ? atoi(getenv("RCS_FUSE_SEEDS")) : kFuseSeeds;
    const bool la = getenv("RCS_FUSE_LOOKAHEAD") ? atoi(getenv("RCS_FUSE_LOOKAHEAD")) != 0 : kFuseLookahead;
    const int strat = getenv("RCS_FUSE_GROWLA") ? atoi(getenv("RCS_FUSE_GROWLA")) : -1;   // -1: both
    std::vector<Block> cand[2];
    auto fuse = [&](int which) {
        Fuser F(c, k);
        F.seeds = seeds;
        F.lookahead = la;
        F.grow_lookahead = which == 1;
        Block B;
        while (F.next_block(B)) {
            cand[which].push_back(B);
            B = Block();
        }
    };
    if (strat < 0) {
        std::thread t1(fuse, 1);
        fuse(0);
        t1.join();
    } else {
        fuse(strat ? 1 : 0);
    }
    const int win = strat >= 0 ? (strat ? 1 : 0) : (cand[1].size() < cand[0].size() ? 1 : 0);
    for (Block& B : cand[win]) {
        const int kb = (int)B.qubits.size();
        const int D = 1 << kb;
        B.matrix.assign((size_t)D * D, {0.0, 0.0});
        for (int i = 0; i < D; i++) B.matrix[(size_t)i * D + i] = {1.0, 0.0};
        for (int gid : B.gate_ids) {
            const Gate& g = c.gates[gid];
            int lb0 = (int)(std::find(B.qubits.begin(), B.qubits.end(), g.q0) - B.qubits.begin());
            int lb1 = g.q1 >= 0 ? (int)(std::find(B.qubits.begin(), B.qubits.end(), g.q1) - B.qubits.begin()) : -1;
            apply_to_block(B.matrix, kb, g, lb0, lb1);
        }
        P.blocks.push_back(std::move(B));
    }

    // ---- 2. layout + remaps
    std::vector<int> pos(n), occ(n);
    for (int q = 0; q < n; q++) pos[q] = occ[q] = q;
    // next use: per qubit, ascending block indices
    std::vector<std::vector<int>> uses(n);
    for (int bi = 0; bi < (int)P.blocks.size(); bi++)
        for (int q : P.blocks[bi].qubits) uses[q].push_back(bi);
    auto next_use = [&](int q, int from) {
        auto it = std::lower_bound(uses[q].begin(), uses[q].end(), from);
        return it == uses[q].end() ? INT_MAX : *it;
    };
    // initial layout: |0...0> is invariant under qubit permutations, so the global positions may
    // start with any qubits at no cost -- take the movable ones whose first use is latest
    if (kInitialPlacement && n_global > 0) {
        std::vector<int> movable;
        for (int q = kPinnedLow; q < n; q++) movable.push_back(q);
        std::stable_sort(movable.begin(), movable.end(), [&](int a, int b2) {
            const int fa = next_use(a, 0), fb = next_use(b2, 0);
            if (fa != fb) return fa > fb;
            return a > b2;
        });
        std::vector<int> want(movable.begin(), movable.begin() + n_global);
        std::vector<int> freeg;   // global positions whose qubit is not wanted
        for (int G = n_local; G < n; G++)
            if (!std::count(want.begin(), want.end(), occ[G])) freeg.push_back(G);
        size_t fi = 0;
        for (int q : want) {
            if (pos[q] >= n_local) continue;
            const int G = freeg[fi++], L = pos[q], qg = occ[G];
            std::swap(occ[G], occ[L]);
            pos[q] = G;
            pos[qg] = L;
        }
        P.initial_pos = pos;
    }
    auto emit_remap = [&](const std::vector<std::pair<int, int>>& pairs) {
        Item it;
        it.type = RCS_ITEM_REMAP;
        it.k = (int)pairs.size();
        for (int i = 0; i < it.k; i++) {
            it.a[i] = pairs[i].first;
            it.b[i] = pairs[i].second;
            int qa = occ[pairs[i].first], qb = occ[pairs[i].second];
            std::swap(occ[pairs[i].first], occ[pairs[i].second]);
            pos[qa] = pairs[i].second;
            pos[qb] = pairs[i].first;
        }
        P.items.push_back(it);
        P.n_remaps++;
    };
    for (int bi = 0; bi < (int)P.blocks.size(); bi++) {
        const Block& blk = P.blocks[bi];
        std::vector<int> need;
        for (int q : blk.qubits)
            if (pos[q] >= n_local) need.push_back(q);
        if (!need.empty()) {
            std::vector<int> cand;
            for (int p = kPinnedLow; p < n_local; p++) {
                int q = occ[p];
                if (!std::count(blk.qubits.begin(), blk.qubits.end(), q)) cand.push_back(q);
            }
            std::stable_sort(cand.begin(), cand.end(), [&](int a, int b2) {
                int na = next_use(a, bi), nb = next_use(b2, bi);
                if (na != nb) return na > nb;
                return pos[a] > pos[b2];
            });
            // prefetch: also bring in the global qubits needed soonest, while the eviction
            // candidate is needed later than they are (a (k+1)-bit remap moves 1 - 2^-(k+1) of the
            // shard, cheaper than a separate 1-bit remap later: 1/2)
            if (kRemapPrefetch) {
                std::vector<int> later;
                for (int q = 0; q < n; q++)
                    if (pos[q] >= n_local && !std::count(need.begin(), need.end(), q) && next_use(q, bi) < INT_MAX)
                        later.push_back(q);
                std::stable_sort(later.begin(), later.end(),
                                 [&](int a, int b2) { return next_use(a, bi) < next_use(b2, bi); });
                for (int q : later) {
                    if ((int)need.size() >= n_global || need.size() >= cand.size()) break;
                    if (next_use(cand[need.size()], bi) <= next_use(q, bi)) break;
                    need.push_back(q);
                }
            }
            // evicted canonical-global qubits go to their home global position when it is free
            std::vector<int> gpos;
            for (int q : need) gpos.push_back(pos[q]);
            std::vector<int> ev(cand.begin(), cand.begin() + need.size());
            std::vector<int> slot(need.size(), -1);
            std::vector<char> used(need.size(), 0);
            for (size_t i = 0; i < ev.size(); i++)
                for (size_t j = 0; j < gpos.size(); j++)
                    if (!used[j] && gpos[j] == ev[i]) { slot[i] = (int)j; used[j] = 1; break; }
            for (size_t i = 0; i < ev.size(); i++)
                for (size_t j = 0; j < gpos.size() && slot[i] < 0; j++)
                    if (!used[j]) { slot[i] = (int)j; used[j] = 1; }
            std::vector<std::pair<int, int>> pairs;
            for (size_t i = 0; i < ev.size(); i++) pairs.push_back({gpos[slot[i]], pos[ev[i]]});
            emit_remap(pairs);
        }
        Item it;
        it.type = RCS_ITEM_PASS;
        it.block = bi;
        it.k = (int)blk.qubits.size();
        for (int i = 0; i < it.k; i++) it.pos[i] = pos[blk.qubits[i]];
        P.items.push_back(it);
        P.n_passes++;
    }

    P.restore_begin = (int)P.items.size();
    P.final_pos = pos;
    // ---- 3. final restore: globals home
    for (int round = 0; round < 3 && n_global > 0; round++) {
        std::vector<std::pair<int, int>> pairs;
        for (int G = n_local; G < n; G++)
            if (occ[G] != G && pos[G] < n_local) pairs.push_back({G, pos[G]});
        if (!pairs.empty()) emit_remap(pairs);
        std::vector<int> wrong;
        for (int G = n_local; G < n; G++)
            if (occ[G] != G) wrong.push_back(G);
        if (wrong.empty()) break;
        // canonical qubits sitting on the wrong global position: park them locally first
        pairs.clear();
        int L = kPinnedLow;
        for (int G : wrong) {
            while (L < n_local && occ[L] >= n_local) L++;
            pairs.push_back({G, L++});
        }
        emit_remap(pairs);
    }
    // local permutation -> two involutions (reflections of every cycle)
    {
        std::vector<char> seen(n_local, 0);
        std::vector<std::pair<int, int>> r1, r2;
        for (int p0 = 0; p0 < n_local; p0++) {
            if (seen[p0] || occ[p0] == p0) { seen[p0] = 1; continue; }
            std::vector<int> cyc;   // data at cyc[i] must move to cyc[i+1]
            int p = p0;
            while (!seen[p]) { seen[p] = 1; cyc.push_back(p); p = occ[p]; }
            const int m = (int)cyc.size();
            for (int i = 0; i < m; i++) {
                int j1 = ((-i) % m + m) % m;
                if (i < j1) r1.push_back({cyc[i], cyc[j1]});
                int j2 = ((1 - i) % m + m) % m;
                if (i < j2) r2.push_back({cyc[i], cyc[j2]});
            }
        }
        for (auto* rr : {&r1, &r2}) {
            if (rr->empty()) continue;
            for (size_t off = 0; off < rr->size(); off += 8) {
                Item it;
                it.type = RCS_ITEM_SWAP;
                it.k = (int)std::min<size_t>(8, rr->size() - off);
                for (int i = 0; i < it.k; i++) {
                    auto pr = (*rr)[off + i];
                    it.a[i] = pr.first;
                    it.b[i] = pr.second;
                    std::swap(occ[pr.first], occ[pr.second]);
                }
                P.items.push_back(it);
                P.n_swaps++;
            }
        }
    }
    for (int p = 0; p < n; p++) {
        if (occ[p] != p) {
            set_error(err, RCS_ERR_ARG, "internal planner error: layout not restored (pos %d holds %d)", p, occ[p]);
            return RCS_ERR_ARG;
        }
    }
    out = std::move(P);
    return RCS_OK;
}

}  // namespace rcs
