// kernels.cu -- sm_100a kernels of the RCS hot path (DESIGN.md §6 has the roofline of each).
//
//  K1 gate_pass     a6  fused dense k-qubit block, in place; HBM-bound for k <= 4
//                       (16 B/amp moved, 4*2^k FFMA/amp, matrix read from the kernel
//                       parameter bank so every FFMA takes its coefficient as a constant
//                       operand); 128-bit loads of amplitude pairs (bit 0 handled in-register)
//  K3 bit_swap      a8  in-place involutive bit permutation (remaps in virtual mode, restore)
//     pack/unpack   a7  gather/scatter of the remap chunks around the NCCL exchange
//  K5 block_sums    a9  fp64 sum of |a|^2 per 2^b-amplitude block (+ sum p^2 for F*)
//  K6 scan          a10 deterministic fp64 inclusive scan (3-level tile scan)
//  K7 sample        a11 per-shot SplitMix64 uniform, binary search over block prefixes,
//                       warp-cooperative fp64 in-block scan (reading V13)
//  K8 xeb           a13 gather p(x_s), fixed-order fp64 reduction (reading V14)
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstring>

#include "kernels.h"

namespace rcs {
namespace dev {

namespace {

constexpr int kThreads = 256;
std::atomic<uint64_t> g_launches{0};
inline void note_launch(uint64_t k = 1) { g_launches.fetch_add(k, std::memory_order_relaxed); }

__device__ __forceinline__ uint64_t insert_zero(uint64_t x, int s) {
    const uint64_t lo = x & ((1ull << s) - 1);
    return ((x >> s) << (s + 1)) | lo;
}

// ------------------------------------------------------------------------------------
// K1: fused gate pass
// ------------------------------------------------------------------------------------
template <int K>
struct PassArgs {
    float2 m[1 << K][1 << K];   // row-major complex64, constant bank
    uint64_t n_vec;             // work items (threads)
    int pos[K];                 // physical position of matrix bit i
    int ins[K + 1];             // ascending insertion positions for the work-item index
};

__device__ __forceinline__ void cmac(float2& acc, const float2 m, const float2 v) {
    acc.x = fmaf(m.x, v.x, acc.x);
    acc.x = fmaf(-m.y, v.y, acc.x);
    acc.y = fmaf(m.x, v.y, acc.y);
    acc.y = fmaf(m.y, v.x, acc.y);
}

// Bit 0 is a target (pos[0] == 0): one group of 2^K amps per thread, loaded as 2^(K-1)
// float4 pairs (amp j = 2c + b0 lives in v[c].xy / v[c].zw).
template <int K>
__global__ void __launch_bounds__(kThreads) k_pass_bit0(float4* __restrict__ a4, const __grid_constant__ PassArgs<K> p) {
    const uint64_t w = (uint64_t)blockIdx.x * kThreads + threadIdx.x;
    if (w >= p.n_vec) return;
    uint64_t base = w;
#pragma unroll
    for (int i = 0; i < K; i++) base = insert_zero(base, p.ins[i]);
    constexpr int H = 1 << (K - 1);
    uint64_t off[H];
#pragma unroll
    for (int c = 0; c < H; c++) {
        uint64_t o = 0;
#pragma unroll
        for (int i = 1; i < K; i++)
            if ((c >> (i - 1)) & 1) o |= 1ull << p.pos[i];
        off[c] = (base | o) >> 1;   // float4 index
    }
    float4 v[H];
#pragma unroll
    for (int c = 0; c < H; c++) v[c] = a4[off[c]];
#pragma unroll
    for (int rc = 0; rc < H; rc++) {
        float2 o0 = make_float2(0.f, 0.f), o1 = make_float2(0.f, 0.f);
#pragma unroll
        for (int c = 0; c < H; c++) {
            const float2 x0 = make_float2(v[c].x, v[c].y), x1 = make_float2(v[c].z, v[c].w);
            cmac(o0, p.m[2 * rc][2 * c], x0);
            cmac(o0, p.m[2 * rc][2 * c + 1], x1);
            cmac(o1, p.m[2 * rc + 1][2 * c], x0);
            cmac(o1, p.m[2 * rc + 1][2 * c + 1], x1);
        }
        a4[off[rc]] = make_float4(o0.x, o0.y, o1.x, o1.y);
    }
}

// Bit 0 is not a target: two groups per thread (bit 0 = 0 -> .xy, bit 0 = 1 -> .zw),
// 2^K float4 loads, same matrix applied to both.
template <int K>
__global__ void __launch_bounds__(kThreads) k_pass_pair(float4* __restrict__ a4, const __grid_constant__ PassArgs<K> p) {
    const uint64_t w = (uint64_t)blockIdx.x * kThreads + threadIdx.x;
    if (w >= p.n_vec) return;
    uint64_t base = w;
#pragma unroll
    for (int i = 0; i < K + 1; i++) base = insert_zero(base, p.ins[i]);
    constexpr int D = 1 << K;
    uint64_t off[D];
#pragma unroll
    for (int c = 0; c < D; c++) {
        uint64_t o = 0;
#pragma unroll
        for (int i = 0; i < K; i++)
            if ((c >> i) & 1) o |= 1ull << p.pos[i];
        off[c] = (base | o) >> 1;
    }
    float4 v[D];
#pragma unroll
    for (int c = 0; c < D; c++) v[c] = a4[off[c]];
#pragma unroll
    for (int r = 0; r < D; r++) {
        float2 oa = make_float2(0.f, 0.f), ob = make_float2(0.f, 0.f);
#pragma unroll
        for (int c = 0; c < D; c++) {
            cmac(oa, p.m[r][c], make_float2(v[c].x, v[c].y));
            cmac(ob, p.m[r][c], make_float2(v[c].z, v[c].w));
        }
        a4[off[r]] = make_float4(oa.x, oa.y, ob.x, ob.y);
    }
}

// tiny states (n_local < K+1 with bit 0 free) fall back to one float2 group per thread
template <int K>
__global__ void __launch_bounds__(kThreads) k_pass_scalar(float2* __restrict__ a, const __grid_constant__ PassArgs<K> p) {
    const uint64_t w = (uint64_t)blockIdx.x * kThreads + threadIdx.x;
    if (w >= p.n_vec) return;
    uint64_t base = w;
#pragma unroll
    for (int i = 0; i < K; i++) base = insert_zero(base, p.ins[i]);
    constexpr int D = 1 << K;
    uint64_t off[D];
    float2 v[D];
#pragma unroll
    for (int c = 0; c < D; c++) {
        uint64_t o = 0;
#pragma unroll
        for (int i = 0; i < K; i++)
            if ((c >> i) & 1) o |= 1ull << p.pos[i];
        off[c] = base | o;
        v[c] = a[off[c]];
    }
#pragma unroll
    for (int r = 0; r < D; r++) {
        float2 o = make_float2(0.f, 0.f);
#pragma unroll
        for (int c = 0; c < D; c++) cmac(o, p.m[r][c], v[c]);
        a[off[r]] = o;
    }
}

template <int K>
cudaError_t launch_pass(float2* amps, int nb, const int* pos, const float* m, cudaStream_t st) {
    PassArgs<K> p;
    std::memcpy(&p.m[0][0], m, sizeof(p.m));
    bool bit0 = false;
    int ins[K + 1];
    int nins = 0;
    for (int i = 0; i < K; i++) {
        p.pos[i] = pos[i];
        ins[nins++] = pos[i];
        bit0 |= pos[i] == 0;
    }
    for (int i = 0; i < K + 1; i++) p.ins[i] = 0;
    if (bit0 && pos[0] != 0) return cudaErrorInvalidValue;   // planner keeps qubit 0 at matrix bit 0
    const bool pair = !bit0 && nb >= K + 1;
    if (pair) ins[nins++] = 0;
    // ascending insertion order
    for (int i = 0; i < nins; i++)
        for (int j = i + 1; j < nins; j++)
            if (ins[j] < ins[i]) { int t = ins[i]; ins[i] = ins[j]; ins[j] = t; }
    for (int i = 0; i < nins; i++) p.ins[i] = ins[i];
    p.n_vec = 1ull << (nb - nins);
    const uint64_t blocks = (p.n_vec + kThreads - 1) / kThreads;
    note_launch();
    if (bit0)
        k_pass_bit0<K><<<(unsigned)blocks, kThreads, 0, st>>>(reinterpret_cast<float4*>(amps), p);
    else if (pair)
        k_pass_pair<K><<<(unsigned)blocks, kThreads, 0, st>>>(reinterpret_cast<float4*>(amps), p);
    else
        k_pass_scalar<K><<<(unsigned)blocks, kThreads, 0, st>>>(amps, p);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------
// K3: involutive bit swap, remap staging
// ------------------------------------------------------------------------------------
struct SwapArgs {
    uint64_t n;
    int np;
    int a[8], b[8];
};

__global__ void __launch_bounds__(kThreads) k_bit_swap(float2* __restrict__ x, const __grid_constant__ SwapArgs s) {
    for (uint64_t i = (uint64_t)blockIdx.x * kThreads + threadIdx.x; i < s.n; i += (uint64_t)gridDim.x * kThreads) {
        uint64_t j = i;
        for (int t = 0; t < s.np; t++) {
            const uint64_t ba = (i >> s.a[t]) & 1, bb = (i >> s.b[t]) & 1;
            if (ba != bb) j ^= (1ull << s.a[t]) | (1ull << s.b[t]);
        }
        if (j > i) {
            const float2 u = x[i], v = x[j];
            x[i] = v;
            x[j] = u;
        }
    }
}

struct PackArgs {
    int j;
    int lpos[8];
    uint64_t codemask, m0, count;
};

template <bool PACK>
__global__ void __launch_bounds__(kThreads) k_pack(float2* __restrict__ amps, float2* __restrict__ buf, const __grid_constant__ PackArgs p) {
    for (uint64_t t = (uint64_t)blockIdx.x * kThreads + threadIdx.x; t < p.count; t += (uint64_t)gridDim.x * kThreads) {
        uint64_t l = p.m0 + t;
        for (int i = 0; i < p.j; i++) l = insert_zero(l, p.lpos[i]);
        l |= p.codemask;
        if (PACK)
            buf[t] = amps[l];
        else
            amps[l] = buf[t];
    }
}

// peer swap (remap over NVLink): each thread moves U 16-B vectors each way, loads first
#ifndef RCS_SWAP_U
#define RCS_SWAP_U 4
#endif
constexpr int kSwapU = RCS_SWAP_U;   // 16-B vectors per thread in flight (loads first)
__global__ void __launch_bounds__(kThreads) k_peer_swap(const __grid_constant__ PeerSwapArgs a) {
    const int pc = blockIdx.y;
    const uint64_t nvec = a.m_count[pc] >> 1;   // 16-B vectors (2 amplitudes)
    float4* loc = reinterpret_cast<float4*>(a.local);
    float4* rem = reinterpret_cast<float4*>(a.peer[pc]);
    const uint64_t stride = (uint64_t)gridDim.x * kThreads * kSwapU;
    for (uint64_t v0 = (uint64_t)blockIdx.x * kThreads * kSwapU + threadIdx.x; v0 < nvec; v0 += stride) {
        uint64_t li[kSwapU], ri[kSwapU];
        float4 lv[kSwapU], rv[kSwapU];
        bool ok[kSwapU];
#pragma unroll
        for (int u = 0; u < kSwapU; u++) {
            const uint64_t v = v0 + (uint64_t)u * kThreads;
            ok[u] = v < nvec;
            uint64_t m = a.m_begin[pc] + 2 * v;
            for (int i = 0, f = 0; i < a.j || f < a.nfix;) {   // lpos and fix merged, ascending
                if (f >= a.nfix || (i < a.j && a.lpos[i] < a.fix[f])) m = insert_zero(m, a.lpos[i++]);
                else m = insert_zero(m, a.fix[f++]);
            }
            m |= a.fixval;
            li[u] = (m | a.mask[pc]) >> 1;
            ri[u] = (m | a.my_mask) >> 1;
            if (ok[u]) {
                lv[u] = loc[li[u]];
                rv[u] = rem[ri[u]];
            }
        }
#pragma unroll
        for (int u = 0; u < kSwapU; u++)
            if (ok[u]) {
                loc[li[u]] = rv[u];
                rem[ri[u]] = lv[u];
            }
    }
}

// ------------------------------------------------------------------------------------
// K5: block sums; K6: scan; reductions
// ------------------------------------------------------------------------------------
constexpr int kSumWarps = 8;
constexpr int kSumGrid = 148 * 8;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__global__ void __launch_bounds__(kSumWarps * 32) k_block_sums(const float2* __restrict__ a, uint64_t nblocks, int b,
                                                                double* __restrict__ bsum, double* __restrict__ part_sq) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint64_t B = 1ull << b;
    double sq = 0.0;
    const uint64_t W = (uint64_t)gridDim.x * kSumWarps;
    uint64_t blk = (uint64_t)blockIdx.x * kSumWarps + wid;
    if (B == 64) {
        // four blocks per warp in flight (the blocks blk + i W of the plain grid-stride loop, in the
        // same order, so every sum and the running sq are bitwise those of one block at a time)
        for (; blk < nblocks; blk += 4 * W) {
            float4 v[4];
#pragma unroll
            for (int i = 0; i < 4; i++)
                v[i] = blk + i * W < nblocks ? reinterpret_cast<const float4*>(a + (blk + i * W) * 64)[lane]
                                             : make_float4(0.f, 0.f, 0.f, 0.f);
            double p0[4], p1[4], t[4];
#pragma unroll
            for (int i = 0; i < 4; i++) {
                p0[i] = (double)v[i].x * v[i].x + (double)v[i].y * v[i].y;
                p1[i] = (double)v[i].z * v[i].z + (double)v[i].w * v[i].w;
                t[i] = p0[i] + p1[i];
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                for (int i = 0; i < 4; i++) t[i] += __shfl_xor_sync(0xffffffffu, t[i], o);
#pragma unroll
            for (int i = 0; i < 4; i++)
                if (blk + i * W < nblocks) {
                    if (lane == 0) bsum[blk + i * W] = t[i];
                    sq += p0[i] * p0[i] + p1[i] * p1[i];
                }
        }
    }
    for (; B != 64 && blk < nblocks; blk += W) {
        double p0 = 0.0, p1 = 0.0;
        {
            const uint64_t i0 = 2 * lane, i1 = 2 * lane + 1;
            if (i0 < B) { const float2 v = a[blk * B + i0]; p0 = (double)v.x * v.x + (double)v.y * v.y; }
            if (i1 < B) { const float2 v = a[blk * B + i1]; p1 = (double)v.x * v.x + (double)v.y * v.y; }
        }
        const double s = warp_sum(p0 + p1);
        if (lane == 0) bsum[blk] = s;
        sq += p0 * p0 + p1 * p1;
    }
    __shared__ double red[kSumWarps];
    sq = warp_sum(sq);
    if (lane == 0) red[wid] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < kSumWarps; i++) t += red[i];
        part_sq[blockIdx.x] = t;
    }
}

constexpr int kScanT = 256, kScanI = 8, kTile = kScanT * kScanI;

__global__ void __launch_bounds__(kScanT) k_scan_tile(double* __restrict__ d, uint64_t n, double* __restrict__ tile_sums) {
    const uint64_t t0 = (uint64_t)blockIdx.x * kTile + (uint64_t)threadIdx.x * kScanI;
    double v[kScanI];
    double run = 0.0;
#pragma unroll
    for (int i = 0; i < kScanI; i++) {
        const double x = (t0 + i < n) ? d[t0 + i] : 0.0;
        run += x;
        v[i] = run;
    }
    // block-wide exclusive scan of per-thread totals (Kogge-Stone in a warp, then warps)
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    __shared__ double wsum[kScanT / 32];
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    double woff = 0.0;
    for (int i = 0; i < wid; i++) woff += wsum[i];
    const double excl = woff + (incl - run);
#pragma unroll
    for (int i = 0; i < kScanI; i++)
        if (t0 + i < n) d[t0 + i] = excl + v[i];
    if (threadIdx.x == kScanT - 1 && tile_sums) tile_sums[blockIdx.x] = woff + incl;
}

__global__ void __launch_bounds__(kScanT) k_scan_add(double* __restrict__ d, uint64_t n, const double* __restrict__ tile_incl) {
    if (blockIdx.x == 0) return;
    const double add = tile_incl[blockIdx.x - 1];
    const uint64_t t0 = (uint64_t)blockIdx.x * kTile + (uint64_t)threadIdx.x * kScanI;
#pragma unroll
    for (int i = 0; i < kScanI; i++)
        if (t0 + i < n) d[t0 + i] += add;
}

__global__ void k_reduce_sum(const double* __restrict__ in, int n, double* __restrict__ out) {
    // one warp, fixed order: lane-strided partials then xor tree
    const int lane = threadIdx.x;
    double s = 0.0;
    for (int i = lane; i < n; i += 32) s += in[i];
    s = warp_sum(s);
    if (lane == 0) out[0] = s;
}

// ------------------------------------------------------------------------------------
// K7: sampling
// ------------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t splitmix_out(uint64_t seed, uint64_t k) {
    uint64_t z = seed + k * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

constexpr int kSampleWarps = 8;

__global__ void __launch_bounds__(kSampleWarps * 32) k_sample(const __grid_constant__ SampleArgs A) {
    const int lane = threadIdx.x & 31;
    const uint64_t wglob = (uint64_t)blockIdx.x * kSampleWarps + (threadIdx.x >> 5);
    const uint64_t s = wglob * 32 + lane;
    const bool valid = s < A.shots;
    double t = 0.0;
    if (valid) {
        const double u = A.u_in ? A.u_in[s]
                                : (double)(splitmix_out(A.seed, A.shot0 + s + 1) >> 11) * (1.0 / 9007199254740992.0);
        t = u * A.T_total;
    }
    const bool perm = A.ptab != nullptr;
    bool owned = perm ? valid : (valid && A.owns_any && t >= A.E_r && (A.owns_tail || t < A.E_r + A.T_r));
    const double tl = perm ? t : t - A.E_r;
    uint64_t j = A.nblocks;
    if (owned) {
        uint64_t lo = 0, hi = A.nblocks;
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (A.inc[mid] > tl) hi = mid; else lo = mid + 1;
        }
        j = lo;
    }
    // kept layout: resolve the tail here, then keep only the shots whose block this rank holds
    bool ptail = false;
    uint64_t lblk = 0;   // local block index of logical block j (kept layout)
    if (perm && owned) {
        if (j >= A.nblocks) {
            j = A.last_block;
            ptail = true;
        }
        uint64_t pb = 0;
#pragma unroll
        for (int c = 0; c < kPermTables; c++) pb |= __ldg(A.ptab + 256 * c + ((j >> (8 * c)) & 255));
        const int lbits = A.nl - A.b;
        owned = (pb >> lbits) == A.rank;
        lblk = pb & ((1ull << lbits) - 1);
    }
    const uint64_t B = 1ull << A.b;
    unsigned long long result = 0;
    for (int i = 0; i < 32; i++) {
        const bool own_i = __shfl_sync(0xffffffffu, owned, i);
        if (!own_i) continue;
        uint64_t jj = __shfl_sync(0xffffffffu, j, i);
        double tt = __shfl_sync(0xffffffffu, tl, i);
        bool tail = __shfl_sync(0xffffffffu, ptail, i);
        const uint64_t lb = __shfl_sync(0xffffffffu, lblk, i);
        if (!perm && jj >= A.nblocks) {
            // rounding past this rank's total: last block with non-zero mass, last non-zero amp
            tail = true;
            uint64_t hiblk = A.nblocks;
            uint64_t found = A.nblocks;
            while (hiblk > 0 && found == A.nblocks) {
                const uint64_t cand = hiblk > 32 ? hiblk - 32 + lane : (uint64_t)lane;
                bool nz = false;
                if (cand < hiblk) {
                    const double prev = cand > 0 ? A.inc[cand - 1] : 0.0;
                    nz = A.inc[cand] > prev;
                }
                const unsigned bal = __ballot_sync(0xffffffffu, nz);
                if (bal) found = (hiblk > 32 ? hiblk - 32 : 0) + (31 - __clz(bal));
                hiblk = hiblk > 32 ? hiblk - 32 : 0;
            }
            jj = found < A.nblocks ? found : A.nblocks - 1;
        }
        const double prev = jj > 0 ? A.inc[jj - 1] : 0.0;
        const double tp = tt - prev;
        const float2* blk = A.amps + (perm ? lb : jj) * B;
        double p0 = 0.0, p1 = 0.0;
        if (B == 64) {
            const float4 v = reinterpret_cast<const float4*>(blk)[lane];
            p0 = (double)v.x * v.x + (double)v.y * v.y;
            p1 = (double)v.z * v.z + (double)v.w * v.w;
        } else {
            if ((uint64_t)(2 * lane) < B) { const float2 v = blk[2 * lane]; p0 = (double)v.x * v.x + (double)v.y * v.y; }
            if ((uint64_t)(2 * lane + 1) < B) { const float2 v = blk[2 * lane + 1]; p1 = (double)v.x * v.x + (double)v.y * v.y; }
        }
        const double ls = p0 + p1;
        double incl = ls;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const double excl = incl - ls;
        const double c0 = excl + p0, c1 = c0 + p1;
        const bool h0 = !tail && c0 > tp, h1 = !tail && c1 > tp;
        const unsigned hb = __ballot_sync(0xffffffffu, h0 || h1);
        int amp;
        if (hb) {
            const int L = __ffs(hb) - 1;
            const bool first = __shfl_sync(0xffffffffu, h0, L);
            amp = 2 * L + (first ? 0 : 1);
        } else {
            const unsigned nzb = __ballot_sync(0xffffffffu, p0 > 0.0 || p1 > 0.0);
            const int L = nzb ? 31 - __clz(nzb) : 0;
            const bool second = __shfl_sync(0xffffffffu, p1 > 0.0, L);
            amp = 2 * L + (second ? 1 : 0);
        }
        if (lane == i) result = (perm ? 0 : A.base_index) + jj * B + (uint64_t)amp;
    }
    if (valid) A.x_out[s] = owned ? result : 0ull;
}

// ------------------------------------------------------------------------------------
// K8: XEB gather / probabilities
// ------------------------------------------------------------------------------------
constexpr int kXebGrid = 148 * 2;

// logical index x -> (owning rank, local offset).  Canonical layout: rank = x >> nl.  Kept
// (permuted) layout: the logical block x >> b maps to the physical global block through the
// byte tables ptab[c][256] (bit permutation, positions < b fixed).
__device__ __forceinline__ uint64_t perm_block(const uint64_t* __restrict__ ptab, uint64_t lb) {
    uint64_t r = 0;
#pragma unroll
    for (int c = 0; c < kPermTables; c++) r |= __ldg(ptab + 256 * c + ((lb >> (8 * c)) & 255));
    return r;
}
__device__ __forceinline__ bool locate(const Locator& L, uint64_t x, uint64_t* off) {
    if (!L.ptab) {
        *off = x & ((1ull << L.nl) - 1);
        return (x >> L.nl) == L.rank;
    }
    const uint64_t pb = perm_block(L.ptab, x >> L.b);
    *off = ((pb & ((1ull << (L.nl - L.b)) - 1)) << L.b) | (x & ((1ull << L.b) - 1));
    return (pb >> (L.nl - L.b)) == L.rank;
}

__global__ void __launch_bounds__(kThreads) k_perm_blocks(const double* __restrict__ in, double* __restrict__ out,
                                                          uint64_t n, const uint64_t* __restrict__ ptab) {
    for (uint64_t i = (uint64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += (uint64_t)gridDim.x * kThreads)
        out[i] = in[perm_block(ptab, i)];
}

// index of the last block with non-zero mass (inc strictly increasing there), or 0
__global__ void __launch_bounds__(kThreads) k_last_nonzero(const double* __restrict__ inc, uint64_t n,
                                                           unsigned long long* __restrict__ out) {
    unsigned long long best = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += (uint64_t)gridDim.x * kThreads) {
        const double prev = i > 0 ? inc[i - 1] : 0.0;
        if (inc[i] > prev && i > best) best = i;
    }
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long y = __shfl_xor_sync(0xffffffffu, best, o);
        best = y > best ? y : best;
    }
    if ((threadIdx.x & 31) == 0 && best) atomicMax(out, best);
}

__global__ void __launch_bounds__(kThreads) k_xeb(const float2* __restrict__ a, const unsigned long long* __restrict__ x,
                                                  uint64_t count, const Locator L, int nbits,
                                                  double* __restrict__ part, int* __restrict__ bad) {
    double s = 0.0, s2 = 0.0, c = 0.0;
    for (uint64_t i = (uint64_t)blockIdx.x * kThreads + threadIdx.x; i < count; i += (uint64_t)gridDim.x * kThreads) {
        const uint64_t xi = x[i];
        if (nbits < 64 && (xi >> nbits) != 0) { atomicOr(bad, 1); continue; }
        uint64_t off;
        if (!locate(L, xi, &off)) continue;
        const float2 v = a[off];
        const double p = (double)v.x * v.x + (double)v.y * v.y;
        s += p;
        s2 += p * p;
        c += 1.0;
    }
    __shared__ double red[3][kThreads / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    s = warp_sum(s); s2 = warp_sum(s2); c = warp_sum(c);
    if (lane == 0) { red[0][wid] = s; red[1][wid] = s2; red[2][wid] = c; }
    __syncthreads();
    if (threadIdx.x < 3) {
        double t = 0.0;
        for (int i = 0; i < kThreads / 32; i++) t += red[threadIdx.x][i];
        part[3 * blockIdx.x + threadIdx.x] = t;
    }
}

__global__ void k_xeb_final(const double* __restrict__ part, int grid, double* __restrict__ out3) {
    const int lane = threadIdx.x;
    for (int q = 0; q < 3; q++) {
        double s = 0.0;
        for (int i = lane; i < grid; i += 32) s += part[3 * i + q];
        s = warp_sum(s);
        if (lane == 0) out3[q] = s;
    }
}

__global__ void __launch_bounds__(kThreads) k_gather_prob(const float2* __restrict__ a, const unsigned long long* __restrict__ x,
                                                          uint64_t count, const Locator L, int nbits,
                                                          double* __restrict__ p, int* __restrict__ bad) {
    for (uint64_t i = (uint64_t)blockIdx.x * kThreads + threadIdx.x; i < count; i += (uint64_t)gridDim.x * kThreads) {
        const uint64_t xi = x[i];
        double r = 0.0;
        uint64_t off;
        if (nbits < 64 && (xi >> nbits) != 0) {
            atomicOr(bad, 1);
        } else if (locate(L, xi, &off)) {
            const float2 v = a[off];
            r = (double)v.x * v.x + (double)v.y * v.y;
        }
        p[i] = r;
    }
}

__global__ void k_set_one(float2* a) { a[0] = make_float2(1.f, 0.f); }

unsigned grid_for(uint64_t n, unsigned cap = 148u * 16u) {
    uint64_t g = (n + kThreads - 1) / kThreads;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (unsigned)g;
}

}  // namespace

// ------------------------------------------------------------------------------------
// launchers
// ------------------------------------------------------------------------------------
uint64_t launches() { return g_launches.load(); }
void count_launch() { note_launch(); }

cudaError_t gate_pass(float2* amps, int nb, int k, const int* pos, const float* m, cudaStream_t st) {
    switch (k) {
        case 1: return launch_pass<1>(amps, nb, pos, m, st);
        case 2: return launch_pass<2>(amps, nb, pos, m, st);
        case 3: return launch_pass<3>(amps, nb, pos, m, st);
        case 4: return launch_pass<4>(amps, nb, pos, m, st);
        case 5: return launch_pass<5>(amps, nb, pos, m, st);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t bit_swap(float2* amps, int nbits, int np, const int* a, const int* b, cudaStream_t st) {
    SwapArgs s{};
    s.n = 1ull << nbits;
    s.np = np;
    for (int i = 0; i < np; i++) { s.a[i] = a[i]; s.b[i] = b[i]; }
    note_launch();
    k_bit_swap<<<grid_for(s.n), kThreads, 0, st>>>(amps, s);
    return cudaGetLastError();
}

static PackArgs make_pack(int j, const int* lpos, uint64_t codemask, uint64_t m0, uint64_t count) {
    PackArgs p{};
    p.j = j;
    for (int i = 0; i < j; i++) p.lpos[i] = lpos[i];
    p.codemask = codemask;
    p.m0 = m0;
    p.count = count;
    return p;
}

cudaError_t pack(const float2* amps, float2* buf, int j, const int* lpos, uint64_t codemask, uint64_t m0,
                 uint64_t count, cudaStream_t st) {
    note_launch();
    k_pack<true><<<grid_for(count), kThreads, 0, st>>>(const_cast<float2*>(amps), buf, make_pack(j, lpos, codemask, m0, count));
    return cudaGetLastError();
}

cudaError_t unpack(float2* amps, const float2* buf, int j, const int* lpos, uint64_t codemask, uint64_t m0,
                   uint64_t count, cudaStream_t st) {
    note_launch();
    k_pack<false><<<grid_for(count), kThreads, 0, st>>>(amps, const_cast<float2*>(buf), make_pack(j, lpos, codemask, m0, count));
    return cudaGetLastError();
}

cudaError_t peer_swap(const PeerSwapArgs& a, cudaStream_t st) {
    uint64_t maxv = 0;
    for (int i = 0; i < a.npeers; i++) maxv = a.m_count[i] / 2 > maxv ? a.m_count[i] / 2 : maxv;
    if (maxv == 0) return cudaSuccess;
    uint64_t gx = (maxv + (uint64_t)kThreads * kSwapU - 1) / ((uint64_t)kThreads * kSwapU);
    const uint64_t cap = a.max_grid > 0 ? (uint64_t)a.max_grid : 148u * 8u;
    if (gx > cap) gx = cap;
    note_launch();
    k_peer_swap<<<dim3((unsigned)gx, (unsigned)a.npeers), kThreads, 0, st>>>(a);
    return cudaGetLastError();
}

int block_sums_grid() { return kSumGrid; }

cudaError_t block_sums(const float2* amps, uint64_t nblocks, int b, double* bsum, double* part_sq, cudaStream_t st) {
    note_launch();
    k_block_sums<<<kSumGrid, kSumWarps * 32, 0, st>>>(amps, nblocks, b, bsum, part_sq);
    return cudaGetLastError();
}

uint64_t scan_tmp_doubles(uint64_t n) {
    uint64_t t = 0;
    while (n > (uint64_t)kTile) {
        n = (n + kTile - 1) / kTile;
        t += n;
    }
    return t + 1;
}

cudaError_t scan_inclusive(double* d, uint64_t n, double* tmp, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    const uint64_t tiles = (n + kTile - 1) / kTile;
    if (tiles == 1) {
        note_launch();
        k_scan_tile<<<1, kScanT, 0, st>>>(d, n, nullptr);
        return cudaGetLastError();
    }
    note_launch();
    k_scan_tile<<<(unsigned)tiles, kScanT, 0, st>>>(d, n, tmp);
    cudaError_t e = scan_inclusive(tmp, tiles, tmp + tiles, st);
    if (e != cudaSuccess) return e;
    note_launch();
    k_scan_add<<<(unsigned)tiles, kScanT, 0, st>>>(d, n, tmp);
    return cudaGetLastError();
}

cudaError_t reduce_sum(const double* in, int n, double* out, cudaStream_t st) {
    note_launch();
    k_reduce_sum<<<1, 32, 0, st>>>(in, n, out);
    return cudaGetLastError();
}

cudaError_t sample(const SampleArgs& a, cudaStream_t st) {
    if (a.shots == 0) return cudaSuccess;
    const uint64_t warps = (a.shots + 31) / 32;
    const uint64_t blocks = (warps + kSampleWarps - 1) / kSampleWarps;
    note_launch();
    k_sample<<<(unsigned)blocks, kSampleWarps * 32, 0, st>>>(a);
    return cudaGetLastError();
}

int xeb_grid() { return kXebGrid; }

cudaError_t xeb_partials(const float2* amps, const unsigned long long* x, uint64_t count, const Locator& L,
                         int nbits, double* part, int* bad, cudaStream_t st) {
    note_launch();
    k_xeb<<<kXebGrid, kThreads, 0, st>>>(amps, x, count, L, nbits, part, bad);
    return cudaGetLastError();
}

cudaError_t xeb_finalize(const double* part, int grid, double* out3, cudaStream_t st) {
    note_launch();
    k_xeb_final<<<1, 32, 0, st>>>(part, grid, out3);
    return cudaGetLastError();
}

cudaError_t gather_prob(const float2* amps, const unsigned long long* x, uint64_t count, const Locator& L,
                        int nbits, double* p, int* bad, cudaStream_t st) {
    if (count == 0) return cudaSuccess;
    note_launch();
    k_gather_prob<<<grid_for(count), kThreads, 0, st>>>(amps, x, count, L, nbits, p, bad);
    return cudaGetLastError();
}

cudaError_t perm_blocks(const double* in, double* out, uint64_t n, const uint64_t* ptab, cudaStream_t st) {
    note_launch();
    k_perm_blocks<<<grid_for(n, 148u * 64u), kThreads, 0, st>>>(in, out, n, ptab);
    return cudaGetLastError();
}

cudaError_t last_nonzero(const double* inc, uint64_t n, unsigned long long* out, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    note_launch();
    k_last_nonzero<<<grid_for(n, 148u * 16u), kThreads, 0, st>>>(inc, n, out);
    return cudaGetLastError();
}

__global__ void __launch_bounds__(kThreads) k_product_init(const __grid_constant__ PrefixArgs a) {
    __shared__ uint32_t bt[2][kPrefixBytes][256];
    for (int e = threadIdx.x; e < 2 * a.nbytes * 256; e += blockDim.x) {
        const int G = e / (a.nbytes * 256), r = e % (a.nbytes * 256);
        bt[G][r >> 8][r & 255] = a.byt[e];
    }
    __syncthreads();
    // A warp writes rows of 64 amplitudes (2 per lane, one 16-B store each) from a contiguous
    // range of rows, four rows (256 amplitudes: byte 0 of X) at a time: the table-index parts of
    // X's bytes >= 1 are warp-uniform per group, the byte-0 parts are per-thread constants, and all
    // 16 table reads of a group are in flight together.
    const int lane = threadIdx.x & 31;
    const uint64_t nrows = a.n_amps >> 6;
    const uint64_t nwarps = (uint64_t)gridDim.x * (kThreads / 32);
    const uint64_t w = (uint64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
    const uint64_t per = ((nrows + nwarps - 1) / nwarps + 3) & ~3ull;   // rows per warp, multiple of 4
    const uint64_t r0 = w * per, r1 = r0 + per < nrows ? r0 + per : nrows;
    uint32_t iA[8], iB[8];   // k = 2 rr + e: row g + rr, amplitude 2 lane + e of the group
    uint32_t zlo = 0;        // bit k: amplitude k has a |1> on a non-prefix qubit of byte 0
#pragma unroll
    for (int k = 0; k < 8; k++) {
        const int by = ((k >> 1) << 6) | (2 * lane) | (k & 1);
        iA[k] = bt[0][0][by];
        iB[k] = bt[1][0][by];
        zlo |= (uint32_t)(((uint64_t)by & a.zmask) != 0) << k;
    }
    float4* out = reinterpret_cast<float4*>(a.amps);
    for (uint64_t g = r0; g < r1; g += 4) {
        const uint64_t Xg = a.base + (g << 6);   // byte 0 of Xg is 0 (g is a multiple of 4)
        uint32_t ha = 0, hb = 0;
        for (int c = 1; c < a.nbytes; c++) {
            const int by = (int)((Xg >> (8 * c)) & 255);
            ha |= bt[0][c][by];
            hb |= bt[1][c][by];
        }
        // a qubit outside the prefix set to |1> in bytes >= 1: the whole group is 0
        const uint32_t dead = (Xg & a.zmask & ~255ull) != 0 ? 0xffu : zlo;
        const float2* TA = a.tab[0] + ha;   // ha | iA[k] == ha + iA[k]: disjoint bits
        const float2* TB = a.tab[1] + hb;
        float2 A[8], B[8];
#pragma unroll
        for (int k = 0; k < 8; k++) {
            const bool live = !((dead >> k) & 1);
            A[k] = live ? __ldg(TA + iA[k]) : make_float2(0.f, 0.f);
            B[k] = live ? __ldg(TB + iB[k]) : make_float2(0.f, 0.f);
        }
        float4* o = out + (((g - r0) << 5) | lane) + (r0 << 5);
        const int nr = r1 - g < 4 ? (int)(r1 - g) : 4;
#pragma unroll
        for (int rr = 0; rr < 4; rr++) {
            if (rr >= nr) break;
            float r[4];
#pragma unroll
            for (int e = 0; e < 2; e++) {   // complex product, fixed fp32 operation order
                const float2 x = A[2 * rr + e], y = B[2 * rr + e];
                r[2 * e] = __fmaf_rn(x.x, y.x, -__fmul_rn(x.y, y.y));
                r[2 * e + 1] = __fmaf_rn(x.x, y.y, __fmul_rn(x.y, y.x));
            }
            __stcs(o + 32 * rr, make_float4(r[0], r[1], r[2], r[3]));
        }
    }
}

cudaError_t product_init(const PrefixArgs& a, cudaStream_t st) {
    if (a.n_amps < 64 || (a.n_amps & 63) || a.nbytes < 1 || a.nbytes > kPrefixBytes) return cudaErrorInvalidValue;
    note_launch();
    k_product_init<<<grid_for(a.n_amps / 64), kThreads, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t init_basis(float2* amps, uint64_t n_amps, int set_one, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(amps, 0, n_amps * sizeof(float2), st);
    if (e != cudaSuccess) return e;
    if (set_one) {
        note_launch();
        k_set_one<<<1, 1, 0, st>>>(amps);
        e = cudaGetLastError();
    }
    return e;
}

}  // namespace dev
}  // namespace rcs
