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
#include <memory>
#include <mutex>
#include <set>
#include <thread>
#include <unordered_map>

#include "internal.h"

namespace rcs {

namespace {

// Qubit sets are 64-bit masks (n <= 63); per-qubit gate lists are shared read-only between the
// fuser and its rollout copies.
struct FuseTables {
    std::vector<std::vector<int>> per_q;   // gate ids per qubit, source order
    std::vector<uint64_t> gmask;           // qubits of gate g
    std::vector<int> gw;                   // 1 or 2: 2q gates count double
};

// Blocks the plain greedy needs from a fuser state (the per-qubit heads determine it), shared by
// every rollout of every strategy: rollouts from neighbouring states walk into the same greedy
// chain, so most stop at a memoized state.  Exact values of a deterministic function: the plan
// does not depend on which thread filled an entry.
struct RolloutMemo {
    struct H {
        size_t operator()(const std::vector<int>& v) const {
            uint64_t h = 1469598103934665603ull;
            for (int x : v) h = (h ^ (uint64_t)(uint32_t)x) * 1099511628211ull;
            return (size_t)h;
        }
    };
    std::mutex mu;
    std::unordered_map<std::vector<int>, int, H> left;
};

FuseTables make_tables(const Circuit& c) {
    FuseTables t;
    t.per_q.assign(c.n, {});
    for (int i = 0; i < (int)c.gates.size(); i++) {
        const Gate& g = c.gates[i];
        t.per_q[g.q0].push_back(i);
        uint64_t m = 1ull << g.q0;
        if (g.q1 >= 0) {
            t.per_q[g.q1].push_back(i);
            m |= 1ull << g.q1;
        }
        t.gmask.push_back(m);
        t.gw.push_back(g.q1 >= 0 ? 2 : 1);
    }
    return t;
}

// Copied for every rollout and lookahead candidate (plain pointers to the shared read-only
// tables and memo: no reference counting on the hot path).
struct Fuser {
    const Circuit& C;
    int k, n;
    const FuseTables* T;
    std::vector<int> head;                 // first unassigned position in per_q[q]
    std::vector<char> assigned;
    size_t first_unassigned = 0;

    int seeds = 0;
    bool lookahead = false;
    bool grow_lookahead = false;
    int grow_depth = 1;
    int grow_beam = 0;   // 0: every extension
    // prefix-first: while a ready gate lies on qubits no block has touched yet, the next block
    // is grown inside the untouched qubits only.  Such blocks act on |0...0> and become the
    // product-state prefix (written by one kernel, not run as passes), so this maximises the
    // gates absorbed there; afterwards the fuser continues as usual.
    bool prefix_first = false;
    uint64_t touched = 0;         // union of the committed blocks' qubits
    uint64_t allowed = ~0ull;     // extensions stay inside this set (prefix phase: ~touched)
    bool last_prefix = false;     // the last next_set() committed a prefix-phase block
    int prefix_depth = -1;        // >= 0: extension search depth of the prefix phase (else grow_depth)
    RolloutMemo* memo = nullptr;

    Fuser(const Circuit& c, int k_, const FuseTables* t) : C(c), k(k_), n(c.n), T(t) {
        head.assign(c.n, 0);
        assigned.assign(c.gates.size(), 0);
    }

    int next_gate(int q, int pos) const {
        const auto& v = T->per_q[q];
        return pos < (int)v.size() ? v[pos] : -1;
    }

    // gates absorbed by qubit set S from the current heads (repeatedly: a gate whose qubits are
    // all in S and at their heads); returns their total weight, optionally the gates in order
    // and the resulting per-qubit heads
    int closure(uint64_t S, std::vector<int>* got = nullptr, int* hout = nullptr) const {
        int h[64];
        for (uint64_t m = S; m; m &= m - 1) h[__builtin_ctzll(m)] = head[__builtin_ctzll(m)];
        int w = 0;
        if (!got) {   // weight / heads only: the absorbed set is unique (a least fixed point), so a
            uint64_t pend = S;   // worklist of qubits whose head moved finds it in any order
            while (pend) {
                const int q = __builtin_ctzll(pend);
                const int g = next_gate(q, h[q]);
                if (g < 0 || (T->gmask[g] & ~S)) {
                    pend &= pend - 1;
                    continue;
                }
                const uint64_t other = T->gmask[g] & ~(1ull << q);
                if (other) {
                    const int qq = __builtin_ctzll(other);
                    if (next_gate(qq, h[qq]) != g) {
                        pend &= pend - 1;
                        continue;
                    }
                    h[qq]++;
                    pend |= other;
                }
                h[q]++;
                w += T->gw[g];
            }
            if (hout)
                for (uint64_t m = S; m; m &= m - 1) hout[__builtin_ctzll(m)] = h[__builtin_ctzll(m)];
            return w;
        }
        // with the gate list: absorption in the order of the scan below (the block's gate order)
        bool progress = true;
        while (progress) {
            progress = false;
            for (uint64_t m = S; m; m &= m - 1) {
                const int q = __builtin_ctzll(m);
                const int g = next_gate(q, h[q]);
                if (g < 0 || (T->gmask[g] & ~S)) continue;
                bool ok = true;
                for (uint64_t mm = T->gmask[g]; mm && ok; mm &= mm - 1) {
                    const int qq = __builtin_ctzll(mm);
                    ok = next_gate(qq, h[qq]) == g;
                }
                if (!ok) continue;
                for (uint64_t mm = T->gmask[g]; mm; mm &= mm - 1) h[__builtin_ctzll(mm)]++;
                w += T->gw[g];
                if (got) got->push_back(g);
                progress = true;
            }
        }
        if (hout)
            for (uint64_t m = S; m; m &= m - 1) hout[__builtin_ctzll(m)] = h[__builtin_ctzll(m)];
        return w;
    }

    // closure weights of the sets one grow() visits (the heads do not move during a grow)
    using WCache = std::unordered_map<uint64_t, int>;
    int cw(uint64_t S, WCache* c) const {
        if (!c) return closure(S);
        auto it = c->find(S);
        if (it != c->end()) return it->second;
        const int w = closure(S);
        c->emplace(S, w);
        return w;
    }

    // candidate extensions of S: the other qubits of the next gate on a qubit of S (after the
    // closure), or the qubits of a gate that is ready elsewhere, within k qubits
    void extensions(uint64_t S, std::vector<uint64_t>& out) const {
        out.clear();
        int h[64];
        closure(S, nullptr, h);
        const int size = __builtin_popcountll(S);
        auto add = [&](uint64_t ext) {
            if (!ext || size + __builtin_popcountll(ext) > k || (ext & ~allowed)) return;
            for (uint64_t e : out)
                if (e == ext) return;
            out.push_back(ext);
        };
        for (uint64_t m = S; m; m &= m - 1) {
            const int q = __builtin_ctzll(m);
            const int g = next_gate(q, h[q]);
            if (g >= 0) add(T->gmask[g] & ~S);
        }
        for (int q = 0; q < n; q++) {
            if ((S >> q) & 1) continue;
            const int g = next_gate(q, head[q]);
            if (g < 0 || !ready(g)) continue;
            add(T->gmask[g] & ~S);
        }
        // deterministic order: ascending by (size, mask)
        std::sort(out.begin(), out.end(), [](uint64_t x, uint64_t y) {
            const int a = __builtin_popcountll(x), b = __builtin_popcountll(y);
            return a != b ? a < b : x < y;
        });
    }

    // greedy continuation: the extension with the largest gain per added qubit, until k
    void grow_from(uint64_t& S, int& w, WCache* wc = nullptr) const {
        std::vector<uint64_t> ex;
        while (__builtin_popcountll(S) < k) {
            extensions(S, ex);
            int bgain = 0, bsize = 0;
            uint64_t best = 0;
            int bw = w;
            for (uint64_t e : ex) {
                const int w1 = cw(S | e, wc);
                const int gain = w1 - w, sz = __builtin_popcountll(e);
                if (gain <= 0) continue;
                if (!best || gain * bsize > bgain * sz) {
                    best = e;
                    bgain = gain;
                    bsize = sz;
                    bw = w1;
                }
            }
            if (!best) break;
            S |= best;
            w = bw;
        }
    }

    // `depth` levels of exhaustive extension choice, then greedy; keeps the heaviest block.
    // Different extension orders reach the same sets: results are memoized per (set, depth).
    using Memo = std::unordered_map<uint64_t, std::pair<uint64_t, int>>;
    void grow_deep(uint64_t& S, int& w, int depth, Memo& memo, WCache* wc) const {
        const uint64_t key = S * 8 + (uint64_t)depth;   // S < 2^61 (n <= 61 here)
        auto f = memo.find(key);
        if (f != memo.end()) {
            S = f->second.first;
            w = f->second.second;
            return;
        }
        const uint64_t S0 = S;
        if (depth == 0 || __builtin_popcountll(S) >= k) {
            grow_from(S, w, wc);
            memo[key] = {S, w};
            return;
        }
        std::vector<uint64_t> ex;
        extensions(S, ex);
        // keep the `grow_beam` extensions with the best gain per added qubit (0: all)
        std::vector<std::pair<double, uint64_t>> ranked;
        for (uint64_t e : ex) {
            const int w1 = cw(S | e, wc);
            if (w1 > w) ranked.push_back({-(double)(w1 - w) / __builtin_popcountll(e), e});
        }
        std::stable_sort(ranked.begin(), ranked.end(),
                         [](const std::pair<double, uint64_t>& x, const std::pair<double, uint64_t>& y) {
                             return x.first < y.first;
                         });
        if (grow_beam > 0 && (int)ranked.size() > grow_beam) ranked.resize(grow_beam);
        int best = -1;
        uint64_t bS = S;
        for (const auto& re : ranked) {
            uint64_t S1 = S | re.second;
            int w1 = cw(S1, wc);
            grow_deep(S1, w1, depth - 1, memo, wc);
            if (w1 > best) {
                best = w1;
                bS = S1;
            }
        }
        if (best < 0) {
            grow_from(S, w, wc);
        } else {
            S = bS;
            w = best;
        }
        memo[S0 * 8 + (uint64_t)depth] = {S, w};
    }

    void grow(int g0, uint64_t& S, int& w) const {
        S = T->gmask[g0];
        w = closure(S);
        if (grow_lookahead) {
            Memo memo;
            WCache wc;
            grow_deep(S, w, grow_depth, memo, &wc);
        } else {
            grow_from(S, w);
        }
    }

    bool ready(int g) const {
        for (uint64_t m = T->gmask[g]; m; m &= m - 1) {
            const int q = __builtin_ctzll(m);
            if (next_gate(q, head[q]) != g) return false;
        }
        return true;
    }

    void commit(uint64_t S) {
        std::vector<int> got;
        closure(S, &got);
        for (int g : got) {
            assigned[g] = 1;
            for (uint64_t m = T->gmask[g]; m; m &= m - 1) head[__builtin_ctzll(m)]++;
        }
        touched |= S;
        while (first_unassigned < assigned.size() && assigned[first_unassigned]) first_unassigned++;
    }

    // number of blocks the plain greedy (earliest-gate seed) needs from the current state
    // (prefix-first fusers: blocks that run as passes, i.e. not counting prefix-phase blocks; the
    // state is then the heads plus the touched set)
    int rollout() const {
        Fuser f = *this;
        f.seeds = 0;
        f.lookahead = false;
        f.grow_lookahead = false;
        f.prefix_depth = -1;   // one rollout function per memo (every prefix-first strategy shares it)
        int cnt = 0;
        uint64_t S;
        if (!memo) {
            while (f.next_set(S)) cnt += !f.last_prefix;
            return cnt;
        }
        auto key = [&]() {
            std::vector<int> kv = f.head;
            if (f.prefix_first) {
                kv.push_back((int)(uint32_t)f.touched);
                kv.push_back((int)(uint32_t)(f.touched >> 32));
            }
            return kv;
        };
        std::vector<std::vector<int>> path;
        std::vector<int> pcnt;
        int tail = 0;
        while (f.first_unassigned < f.assigned.size()) {
            std::vector<int> kv = key();
            {
                std::lock_guard<std::mutex> lk(memo->mu);
                auto it = memo->left.find(kv);
                if (it != memo->left.end()) {
                    tail = it->second;
                    break;
                }
            }
            path.push_back(std::move(kv));
            pcnt.push_back(cnt);
            f.next_set(S);
            cnt += !f.last_prefix;
        }
        std::lock_guard<std::mutex> lk(memo->mu);
        for (size_t i = 0; i < path.size(); i++) memo->left.emplace(std::move(path[i]), cnt - pcnt[i] + tail);
        return cnt + tail;
    }

    // next block's qubit set (committed): grow from the earliest unassigned gate and from up to
    // `seeds` other ready gates; keep the heaviest block, or with `lookahead` the one whose
    // greedy completion needs the fewest blocks (candidates evaluated in parallel threads)
    bool next_set(uint64_t& out) {
        if (first_unassigned >= assigned.size()) return false;
        last_prefix = prefix_first && next_prefix_set(out);
        if (last_prefix) return true;
        const int g0 = (int)first_unassigned;
        std::vector<int> cand{g0};
        for (int i = g0 + 1; i < (int)assigned.size() && (int)cand.size() < 1 + seeds; i++)
            if (!assigned[i] && ready(i)) cand.push_back(i);
        const size_t nc = cand.size();
        std::vector<uint64_t> cS(nc);
        std::vector<long> sc(nc);
        auto work = [&](size_t i) {
            int w;
            grow(cand[i], cS[i], w);
            long score = w;
            if (lookahead && nc > 1) {
                Fuser f = *this;
                f.commit(cS[i]);
                score = -1000L * f.rollout() + score;   // fewest remaining blocks, then most gates now
            }
            sc[i] = score;
        };
        if (lookahead && nc > 1) {
            std::vector<std::thread> th;
            for (size_t i = 1; i < nc; i++) th.emplace_back(work, i);
            work(0);
            for (auto& t : th) t.join();
        } else {
            for (size_t i = 0; i < nc; i++) work(i);
        }
        size_t bi = 0;
        for (size_t i = 1; i < nc; i++)
            if (sc[i] > sc[bi]) bi = i;
        out = cS[bi];
        commit(out);
        return true;
    }

    // prefix phase: every ready gate on untouched qubits seeds a block grown inside the untouched
    // qubits; the heaviest (most absorbed gate weight, ties: earliest seed) is committed
    bool next_prefix_set(uint64_t& out) {
        std::vector<int> cand;
        for (int q = 0; q < n; q++) {
            if ((touched >> q) & 1) continue;
            const int g = next_gate(q, head[q]);
            if (g < 0 || (T->gmask[g] & touched) || !ready(g)) continue;
            if (std::find(cand.begin(), cand.end(), g) == cand.end()) cand.push_back(g);
        }
        if (cand.empty()) return false;
        std::sort(cand.begin(), cand.end());
        const uint64_t saved = allowed;
        const bool sgl = grow_lookahead;
        const int sgd = grow_depth;
        allowed = ~touched;
        if (prefix_depth >= 0) {
            grow_lookahead = prefix_depth > 0;
            grow_depth = prefix_depth;
        }
        const size_t nc = cand.size();
        std::vector<uint64_t> cS(nc);
        std::vector<long> sc(nc);
        for (size_t i = 0; i < nc; i++) {
            int w;
            grow(cand[i], cS[i], w);
            sc[i] = w;
        }
        allowed = saved;
        grow_lookahead = sgl;
        grow_depth = sgd;
        if (lookahead && nc > 1) {   // fewest passes after a greedy completion, then most gates now
            auto work = [&](size_t i) {
                Fuser f = *this;
                f.commit(cS[i]);
                sc[i] += -1000L * f.rollout();
            };
            std::vector<std::thread> th;
            for (size_t i = 1; i < nc; i++) th.emplace_back(work, i);
            work(0);
            for (auto& t : th) t.join();
        }
        uint64_t bS = cS[0];
        long bw = sc[0];
        for (size_t i = 1; i < nc; i++)
            if (sc[i] > bw) {
                bw = sc[i];
                bS = cS[i];
            }
        out = bS;
        commit(out);
        return true;
    }

    // beam strategy: every candidate next set (prefix phase: all seeds inside the untouched
    // qubits; else the earliest gate and `seeds` ready gates) with its lookahead score -- gate
    // weight now minus 1000 x the passes of a greedy completion -- without committing
    void candidates(std::vector<std::pair<long, uint64_t>>& out) {
        out.clear();
        if (first_unassigned >= assigned.size()) return;
        std::vector<int> cand;
        bool pre = false;
        if (prefix_first) {
            for (int q = 0; q < n; q++) {
                if ((touched >> q) & 1) continue;
                const int g = next_gate(q, head[q]);
                if (g < 0 || (T->gmask[g] & touched) || !ready(g)) continue;
                if (std::find(cand.begin(), cand.end(), g) == cand.end()) cand.push_back(g);
            }
            std::sort(cand.begin(), cand.end());
            pre = !cand.empty();
        }
        if (!pre) {
            cand.assign(1, (int)first_unassigned);
            for (int i = (int)first_unassigned + 1; i < (int)assigned.size() && (int)cand.size() < 1 + seeds; i++)
                if (!assigned[i] && ready(i)) cand.push_back(i);
        }
        const uint64_t saved = allowed;
        if (pre) allowed = ~touched;
        for (int g : cand) {
            uint64_t S;
            int w;
            grow(g, S, w);
            Fuser f = *this;
            f.allowed = saved;
            f.commit(S);
            out.push_back({-1000L * (f.rollout() + (pre ? 0 : 1)) + w, S});
        }
        allowed = saved;
    }

    bool next_block(Block& B) {
        // the gates are those the committed set absorbs from the heads BEFORE the commit
        const std::vector<int> head0 = head;
        uint64_t S;
        const std::vector<char> assigned0 = assigned;
        if (!next_set(S)) return false;
        std::vector<int> h1 = head;
        head = head0;
        B.gate_ids.clear();
        closure(S, &B.gate_ids);
        head = h1;
        (void)assigned0;
        B.qubits.clear();
        for (uint64_t m = S; m; m &= m - 1) B.qubits.push_back(__builtin_ctzll(m));
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

// Fusion strategies (P-independent, deterministic): 0 plain greedy, 1 greedy with every
// candidate extension scored by the block it finishes as, 2 exhaustive 3-level extension search
// (memoized); all with the rollout lookahead over seed gates.  The plan with the fewest blocks
// wins, ties to the lower index.
// Beam search over whole fusions (prefix-first): each state expands into its kBeamWidth best
// candidate blocks, the kBeamWidth states with the fewest passes + best lookahead survive
// (duplicates by per-qubit heads dropped).  Deterministic (stable order everywhere).
static void fuse_beam(const Circuit& c, int k, std::vector<Block>& out, std::shared_ptr<RolloutMemo> memo) {
    constexpr int kBeamWidth = 4, kBeamExpand = 4;
    const FuseTables tabs = make_tables(c);
    struct Node {
        Fuser f;
        int passes;
        long score;
        std::vector<uint64_t> sets;
    };
    auto root = std::make_shared<Node>(Node{Fuser(c, k, &tabs), 0, 0, {}});
    root->f.prefix_first = true;
    root->f.memo = memo.get();
    root->f.seeds = kFuseSeeds;
    root->f.lookahead = true;
    std::vector<std::shared_ptr<Node>> beam{root};
    std::shared_ptr<Node> best;
    while (!beam.empty()) {
        std::vector<std::shared_ptr<Node>> next;
        for (auto& nd : beam) {
            if (nd->f.first_unassigned >= nd->f.assigned.size()) {
                if (!best || nd->passes < best->passes) best = nd;
                continue;
            }
            std::vector<std::pair<long, uint64_t>> cands;
            nd->f.candidates(cands);
            std::stable_sort(cands.begin(), cands.end(),
                             [](const std::pair<long, uint64_t>& a, const std::pair<long, uint64_t>& b) {
                                 return a.first > b.first;
                             });
            for (int m = 0; m < (int)cands.size() && m < kBeamExpand; m++) {
                auto ch = std::make_shared<Node>(Node{nd->f, nd->passes, 0, nd->sets});
                const uint64_t S = cands[m].second;
                ch->passes += (S & nd->f.touched) != 0;   // a block on untouched qubits is prefix
                ch->f.commit(S);
                ch->sets.push_back(S);
                ch->score = -1000L * ch->passes + cands[m].first;
                next.push_back(ch);
            }
        }
        std::stable_sort(next.begin(), next.end(),
                         [](const std::shared_ptr<Node>& a, const std::shared_ptr<Node>& b) { return a->score > b->score; });
        std::vector<std::shared_ptr<Node>> kept;
        for (auto& nd : next) {
            bool dup = false;
            for (auto& kd : kept) dup = dup || (kd->f.head == nd->f.head && kd->f.touched == nd->f.touched);
            if (!dup) kept.push_back(nd);
            if ((int)kept.size() >= kBeamWidth) break;
        }
        beam.swap(kept);
    }
    // replay the winner's sets: the gates of each block in absorption order
    Fuser F(c, k, &tabs);
    out.clear();
    for (uint64_t S : best->sets) {
        Block B;
        F.closure(S, &B.gate_ids);
        F.commit(S);
        for (uint64_t m = S; m; m &= m - 1) B.qubits.push_back(__builtin_ctzll(m));
        out.push_back(std::move(B));
    }
}

static void fuse_strategy_memo(const Circuit& c, int k, int which, std::vector<Block>& out,
                               std::shared_ptr<RolloutMemo> memo) {
    if (which == kFuseStrategies - 1) {
        fuse_beam(c, k, out, std::move(memo));
        return;
    }
    // {prefix-first, extension search depth, prefix-phase depth (-1: the same), seeds}
    static const int S[kFuseStrategies - 1][4] = {{0, 2, -1, 4}, {1, 0, -1, kFuseSeeds},
                                                  {1, 1, -1, kFuseSeeds}, {1, kFuseDeepDepth, 1, kFuseSeeds}};
    const FuseTables tabs = make_tables(c);
    Fuser F(c, k, &tabs);
    F.prefix_first = S[which][0] != 0;
    F.prefix_depth = S[which][2];
    F.memo = memo.get();   // memo outlives F (held by this frame)
    F.seeds = S[which][3];
    F.lookahead = kFuseLookahead;
    F.grow_lookahead = S[which][1] > 0;
    F.grow_depth = S[which][1];
    out.clear();
    Block B;
    while (F.next_block(B)) {
        out.push_back(B);
        B = Block();
    }
}

void fuse_strategy(const Circuit& c, int k, int which, std::vector<Block>& out) {
    fuse_strategy_memo(c, k, which, out, std::make_shared<RolloutMemo>());
}

int fuse_best(const Circuit& c, int k, std::vector<Block>* cand) {
    std::vector<std::thread> th;
    auto memo = std::make_shared<RolloutMemo>(), pmemo = std::make_shared<RolloutMemo>();
#ifdef RCS_PLAN_DEBUG
    for (int w = 0; w < kFuseStrategies; w++) {
        auto t0 = std::chrono::steady_clock::now();
        fuse_strategy_memo(c, k, w, cand[w], w >= 1 ? pmemo : memo);
        fprintf(stderr, "strategy %d time %.3f s\n", w, std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    }
#else
    for (int w = 1; w < kFuseStrategies; w++)
        th.emplace_back([&, w] { fuse_strategy_memo(c, k, w, cand[w], w >= 1 ? pmemo : memo); });
    fuse_strategy_memo(c, k, 0, cand[0], memo);
#endif
    for (auto& t : th) t.join();
    int win = 0;
    for (int w = 1; w < kFuseStrategies; w++)
        if (fuse_cost(cand[w]) < fuse_cost(cand[win])) win = w;
#ifdef RCS_PLAN_DEBUG
    for (int w = 0; w < kFuseStrategies; w++) {
        int k9 = 0;
        for (const Block& B : cand[w]) {
            int low = 0;
            for (int q : B.qubits) low += q < 4;
            k9 += low >= 3;
        }
        fprintf(stderr, "strategy %d: %zu blocks, %lld passes, %d blocks with >= 3 of qubits 0..3%s\n", w, cand[w].size(),
                (long long)(fuse_cost(cand[w]) >> 20), k9, w == win ? " *" : "");
    }
#endif
    return win;
}

// blocks that run as passes (x 2^20) + all blocks: the product-state prefix (blocks disjoint from
// every earlier block, up to the two tables' 2 x kPrefixGroupBits qubits) costs no pass
int64_t fuse_cost(const std::vector<Block>& blocks) {
    uint64_t seen = 0;
    int pre = 0, preq = 0;
    for (const Block& B : blocks) {
        uint64_t m = 0;
        for (int q : B.qubits) m |= 1ull << q;
        if (!(m & seen) && preq + (int)B.qubits.size() <= 2 * kPrefixGroupBits) {
            pre++;
            preq += (int)B.qubits.size();
        }
        seen |= m;
    }
    return ((int64_t)(blocks.size() - pre) << 20) + (int64_t)blocks.size();
}

int plan_block_k(int n, int fuse_k, int n_global) {
    const int n_local = n - n_global;
    if (fuse_k <= 0) fuse_k = n_local >= kTcMinLocal ? 6 : 4;
    if (fuse_k == 6 && n_local < kTcMinLocal) fuse_k = 5;
    return std::min(fuse_k, n_local);
}

rcs_status build_plan(const Circuit& c, int fuse_k, int n_global, Plan& out, rcs_error* err,
                      const std::vector<Block>* given, bool use_prefix) {
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
    const int pinned = pinned_low(k);
    if (n_global > 0 && n_local - pinned < k) {
        set_error(err, RCS_ERR_ARG, "too many global qubits: n=%d g=%d leaves %d movable local qubits < k=%d",
                  n, n_global, n_local - pinned, k);
        return RCS_ERR_ARG;
    }
    Plan P;
    P.n = n;
    P.n_global = n_global;
    P.fuse_k = k;
    P.pinned = pinned_low(k);

    // ---- 1. fusion (or the blocks another rank chose, see api.cpp)
    std::vector<Block> cand[kFuseStrategies];
    int win = 0;
    if (given) {
        cand[0] = *given;
    } else {
        win = fuse_best(c, k, cand);
    }
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

    // ---- 1b. product-state prefix (a function of the blocks only: P-independent).  A block none
    // of whose qubits an earlier block touches acts on |0...0> and commutes with every earlier
    // block (disjoint qubits), so it can move to the front; these blocks are pairwise disjoint.
    {
        uint64_t seen = 0;
        std::vector<Block> front, rest;
        for (Block& B : P.blocks) {
            uint64_t mk = 0;
            for (int q : B.qubits) mk |= 1ull << q;
            if (!(mk & seen)) front.push_back(std::move(B));
            else rest.push_back(std::move(B));
            seen |= mk;
        }
        int m = use_prefix ? (int)front.size() : 0;
        P.blocks = std::move(front);
        for (Block& B : rest) P.blocks.push_back(std::move(B));
        // groups: A = the first blocks up to half of the prefix qubits, B = the rest; drop
        // trailing blocks until each group fits kPrefixGroupBits
        while (m > 0) {
            int total = 0;
            for (int b = 0; b < m; b++) total += (int)P.blocks[b].qubits.size();
            // split point: the most balanced (A non-empty, ties to the earliest)
            int a = 1, na = (int)P.blocks[0].qubits.size();
            for (int a1 = 1, n1 = 0; a1 <= m; a1++) {
                n1 += (int)P.blocks[a1 - 1].qubits.size();   // qubits of blocks [0, a1)
                if (std::max(n1, total - n1) < std::max(na, total - na)) {
                    a = a1;
                    na = n1;
                }
            }
            if (na <= kPrefixGroupBits && total - na <= kPrefixGroupBits) {
                P.prefix = m;
                for (int G = 0; G < 2; G++) {
                    const int b0 = G ? a : 0, b1 = G ? m : a;
                    std::vector<int>& qs = P.pq[G];
                    for (int b = b0; b < b1; b++) qs.insert(qs.end(), P.blocks[b].qubits.begin(), P.blocks[b].qubits.end());
                    std::sort(qs.begin(), qs.end());
                    const size_t N = (size_t)1 << qs.size();
                    std::vector<cplx>& T = P.tab[G];
                    T.assign(N, {1.0, 0.0});
                    for (int b = b0; b < b1; b++) {   // fusion order
                        const Block& B = P.blocks[b];
                        const int kb = (int)B.qubits.size(), D = 1 << kb;
                        int bit[8];
                        for (int i = 0; i < kb; i++)
                            bit[i] = (int)(std::find(qs.begin(), qs.end(), B.qubits[i]) - qs.begin());
                        for (size_t v = 0; v < N; v++) {
                            int r = 0;
                            for (int i = 0; i < kb; i++) r |= (int)((v >> bit[i]) & 1) << i;
                            const cplx f = B.matrix[(size_t)r * D];   // column 0: the block on |0...0>
                            const cplx t = T[v];
                            T[v] = {t.re * f.re - t.im * f.im, t.re * f.im + t.im * f.re};
                        }
                    }
                }
                break;
            }
            m--;
        }
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
        for (int q = pinned; q < n; q++) movable.push_back(q);
        std::stable_sort(movable.begin(), movable.end(), [&](int a, int b2) {
            const int fa = next_use(a, P.prefix), fb = next_use(b2, P.prefix);   // prefix blocks need no remap
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
        for (int q : blk.qubits)   // prefix blocks are written by the product kernel: no remap
            if (pos[q] >= n_local && bi >= P.prefix) need.push_back(q);
        if (!need.empty()) {
            std::vector<int> cand;
            for (int p = pinned; p < n_local; p++) {
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
        int L = pinned;
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
