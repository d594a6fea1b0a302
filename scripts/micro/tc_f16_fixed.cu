// tc_f16.cu -- probe for the fp16-split tensor-core pass: kind::f16 MMA (M=128, N=64, K=16),
// A (128 x 128 fp16, hi and lo) in TMEM packed 2 per 32-bit column, B (K=128 x N=64 fp16) in
// shared memory K-major interleave, fp32 accumulators.  Inputs are split x*2^s = hi + lo in fp16
// with power-of-two scales (A: 2^14, B: per-tile 2^(14 - e_max)), results unscaled exactly.
// Reports correctness and the signed accumulation bias of several accumulator layouts.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)
constexpr int M = 128, N = 64, K = 128;
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t bdesc(uint32_t saddr) {
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)(128 >> 4) << 16;                 // LBO: next 16-B K chunk
    d |= (uint64_t)(((K / 8) * 128) >> 4) << 32;     // SBO: next 8-row group (K/8 chunks of 128 B)
    d |= 1ull << 46;
    return d;
}
// fp16 B element (n, k): chunk = 8 halves along K
__device__ __forceinline__ uint32_t boff(int n, int k) { return (n >> 3) * ((K / 8) * 128) + (k >> 3) * 128 + (n & 7) * 16 + (k & 7) * 2; }
struct Order { int n, nacc; int t[64], ks[64], acc[64]; float unscale; int fixed; };

__global__ void __launch_bounds__(128) k(const float* A, const float* B, float* D, const __grid_constant__ Order o) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t tb;
    __shared__ __align__(8) uint64_t mb;
    __shared__ float red[4];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (w == 0) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su(&tb))); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
    if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&mb))); asm volatile("fence.mbarrier_init.release.cluster;"); }
    // tile max exponent of B
    float mx = 0.f;
    for (int i = threadIdx.x; i < N * K; i += 128) mx = fmaxf(mx, fabsf(B[i]));
    for (int s = 16; s; s >>= 1) mx = fmaxf(mx, __shfl_xor_sync(~0u, mx, s));
    if (l == 0) red[w] = mx;
    __syncthreads();
    mx = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
    const int e = ((__float_as_int(mx) >> 23) & 0xff) - 127;     // max in [2^e, 2^(e+1))
    const float sb = o.fixed ? 32768.f : exp2f((float)(14 - e));   // fixed 2^15 or per-tile
    for (int i = threadIdx.x; i < N * K; i += 128) {
        const int n = i / K, kk = i % K;
        const float x = B[n * K + kk] * sb;
        const __half h = __float2half_rn(x);
        const __half lo = __float2half_rn(x - __half2float(h));
        *reinterpret_cast<__half*>(sm + boff(n, kk)) = h;
        *reinterpret_cast<__half*>(sm + N * K * 2 + boff(n, kk)) = lo;
    }
    asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tb;
    {   // A -> TMEM: hi cols [0,64), lo [64,128); column c holds k = 2c (low half), 2c+1 (high half)
        const int m = w * 32 + l;
        for (int h = 0; h < 2; h++)
            for (int c0 = 0; c0 < 64; c0 += 32) {
                uint32_t r[32];
                for (int c = 0; c < 32; c++) {
                    float x0 = A[m * K + 2 * (c0 + c)] * 16384.f, x1 = A[m * K + 2 * (c0 + c) + 1] * 16384.f;
                    __half h0 = __float2half_rn(x0), h1 = __float2half_rn(x1);
                    if (h) { h0 = __float2half_rn(x0 - __half2float(h0)); h1 = __float2half_rn(x1 - __half2float(h1)); }
                    r[c] = (uint32_t)__half_as_ushort(h0) | ((uint32_t)__half_as_ushort(h1) << 16);
                }
                const uint32_t ta = tm + ((uint32_t)(w * 32) << 16) + h * 64 + c0;
                asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta),
                    "r"(r[0]),"r"(r[1]),"r"(r[2]),"r"(r[3]),"r"(r[4]),"r"(r[5]),"r"(r[6]),"r"(r[7]),"r"(r[8]),"r"(r[9]),"r"(r[10]),"r"(r[11]),"r"(r[12]),"r"(r[13]),"r"(r[14]),"r"(r[15]),"r"(r[16]),"r"(r[17]),"r"(r[18]),"r"(r[19]),"r"(r[20]),"r"(r[21]),"r"(r[22]),"r"(r[23]),"r"(r[24]),"r"(r[25]),"r"(r[26]),"r"(r[27]),"r"(r[28]),"r"(r[29]),"r"(r[30]),"r"(r[31]));
            }
        asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;"); asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t d0 = tm + 128;
    if (threadIdx.x == 0) {
        // kind::f16: c_format F32 (1<<4), a/b format F16 (0), K-major, N>>3, M>>4
        const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
        const uint32_t sbase = su(sm);
        int started[4] = {0, 0, 0, 0};
        for (int i = 0; i < o.n; i++) {
            const int t = o.t[i], ks = o.ks[i], a = o.acc[i];
            const uint32_t at = tm + ks * 8 + (t == 2 ? 64 : 0);              // K=16 -> 8 packed columns
            const uint64_t bd = bdesc(sbase + (t == 1 ? N * K * 2 : 0) + ks * 256);   // 2 chunks of 16 B per K-step
            const uint32_t acc = started[a] ? 1u : 0u; started[a] = 1;
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d0 + a * 64), "r"(at), "l"(bd), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(&mb)));
    }
    { uint32_t dn = 0; while (!dn) asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}" : "=r"(dn) : "r"(su(&mb)), "r"(0)); }
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int m = w * 32 + l;
    const float us = o.unscale / sb;
    for (int c0 = 0; c0 < N; c0 += 32) {
        float s[32]; for (int c = 0; c < 32; c++) s[c] = 0.f;
        for (int a = 0; a < o.nacc; a++) {
            uint32_t v[32];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]),"=r"(v[8]),"=r"(v[9]),"=r"(v[10]),"=r"(v[11]),"=r"(v[12]),"=r"(v[13]),"=r"(v[14]),"=r"(v[15]),"=r"(v[16]),"=r"(v[17]),"=r"(v[18]),"=r"(v[19]),"=r"(v[20]),"=r"(v[21]),"=r"(v[22]),"=r"(v[23]),"=r"(v[24]),"=r"(v[25]),"=r"(v[26]),"=r"(v[27]),"=r"(v[28]),"=r"(v[29]),"=r"(v[30]),"=r"(v[31])
                : "r"(d0 + a * 64 + ((uint32_t)(w * 32) << 16) + c0));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
            for (int c = 0; c < 32; c++) s[c] += __uint_as_float(v[c]);
        }
        for (int c = 0; c < 32; c++) D[m * N + c0 + c] = s[c] * us;
    }
    asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
    if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
    std::mt19937_64 rng(7);
    std::normal_distribution<double> nd(0.0, 1.0);
    std::vector<float> A(M * K), B(N * K), D(M * N);
    for (auto& x : A) x = (float)(nd(rng) / std::sqrt(128.0));
    float *dA, *dB, *dD;
    CK(cudaMalloc(&dA, A.size() * 4)); CK(cudaMalloc(&dB, B.size() * 4)); CK(cudaMalloc(&dD, D.size() * 4));
    CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
    const int smem = 2 * N * K * 2;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    for (int fixed = 0; fixed < 2; fixed++)
    for (int lsc = 10; lsc <= 19; lsc += 3) {
    const int var = 2;
        Order o{}; int n = 0;
        auto add = [&](int t, int ks, int a) { o.t[n] = t; o.ks[n] = ks; o.acc[n] = a; n++; };
        const int KS = K / 16;
        if (var == 0) { for (int ks = 0; ks < KS; ks++) { add(0, ks, 0); add(1, ks, 0); add(2, ks, 0); } o.nacc = 1; }
        else {
            int na = var + 1;
            for (int ks = 0; ks < KS; ks++) { add(1, ks, 0); add(2, ks, 0); }
            for (int ks = 0; ks < KS; ks++) add(0, ks, ks * na / KS);
            o.nacc = na;
        }
        o.n = n; o.unscale = 1.f / 16384.f; o.fixed = fixed;
        double sd = 0, sa = 0, g2 = 0, r2 = 0, e2 = 0, emax = 0;
        for (int rep = 0; rep < 40; rep++) {
            const double sc = std::ldexp(1.0, -lsc);
            for (auto& x : B) x = (float)(nd(rng) * sc);
            CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
            k<<<1, 128, smem>>>(dA, dB, dD, o);
            CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
            CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
            for (int m = 0; m < M; m++) for (int c = 0; c < N; c++) {
                double r = 0; for (int kk = 0; kk < K; kk++) r += (double)A[m * K + kk] * B[c * K + kk];
                double g = D[m * N + c];
                sd += (g - r) * (r > 0 ? 1 : -1) / sc; sa += std::fabs(r) / sc;
                g2 += g * g / (sc * sc); r2 += r * r / (sc * sc); e2 += (g - r) * (g - r) / (sc * sc);
                emax = std::fmax(emax, std::fabs(g - r) / sc);
            }
        }
        printf("%s scale, amplitudes 2^-%d: bias(rel) %+.3e  norm2-1 %+.3e  rms rel %.3e\n", fixed ? "fixed 2^15" : "per-tile  ", lsc, sd / sa, g2 / r2 - 1, std::sqrt(e2 / r2));
    }
    return 0;
}
