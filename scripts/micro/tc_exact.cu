// tc_exact.cu -- probe for an exact main term in the fp16-split tensor-core pass.
//
// Y = A X with A = real 128x128 embedding [[Ur,-Ui],[Ui,Ur]] of a random 64x64 unitary and X
// (128 x 64) = [Re; Im] of 64 Porter-Thomas-like columns.  Two splits, same 24 MMAs
// (kind::f16, M=128 N=64 K=16, A in TMEM, B in smem, fp32 accumulators):
//   float  : x 2^s = hi + lo, hi = fp16(x 2^s), lo = fp16(rest); fixed s (A 14, X 15)   [round 1]
//   exact  : per-row (A) / per-column (X) power-of-two scale so the max is in [2^10, 2^11),
//            hi = rint(x 2^e) (an integer, exact in fp16), lo = fp16(x 2^e - hi).  The main
//            term hi.hi is then a sum of integers < 2^24 -> exact in fp32, whatever the
//            accumulation's rounding; only the small cross terms round.
// The kernel returns the raw accumulators; the host emulates the epilogue in fp32 (add.rn,
// mul.rn by powers of two) and compares with fp64.  It also checks the main accumulator against
// the exact int64 sum of the integer products (exactness of the hardware accumulation).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <complex>
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
    d |= (uint64_t)(128 >> 4) << 16;
    d |= (uint64_t)(((K / 8) * 128) >> 4) << 32;
    d |= 1ull << 46;
    return d;
}
__device__ __forceinline__ uint32_t boff(int n, int k) { return (n >> 3) * ((K / 8) * 128) + (k >> 3) * 128 + (n & 7) * 16 + (k & 7) * 2; }

// Ah, Al: [M][K] fp16; Bh, Bl: [N][K] fp16.  D: [2][M][N] raw accumulators (0: cross, 1: main)
__global__ void __launch_bounds__(128) k(const __half* Ah, const __half* Al, const __half* Bh, const __half* Bl, float* D,
                                         int main_accs) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t tb;
    __shared__ __align__(8) uint64_t mb;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (w == 0) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su(&tb))); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
    if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&mb))); asm volatile("fence.mbarrier_init.release.cluster;"); }
    for (int i = threadIdx.x; i < N * K; i += 128) {
        const int n = i / K, kk = i % K;
        *reinterpret_cast<__half*>(sm + boff(n, kk)) = Bh[i];
        *reinterpret_cast<__half*>(sm + N * K * 2 + boff(n, kk)) = Bl[i];
    }
    asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tb;
    {
        const int m = w * 32 + l;
        for (int h = 0; h < 2; h++)
            for (int c0 = 0; c0 < 64; c0 += 32) {
                uint32_t r[32];
                const __half* src = (h ? Al : Ah) + m * K;
                for (int c = 0; c < 32; c++)
                    r[c] = (uint32_t)__half_as_ushort(src[2 * (c0 + c)]) | ((uint32_t)__half_as_ushort(src[2 * (c0 + c) + 1]) << 16);
                const uint32_t ta = tm + ((uint32_t)(w * 32) << 16) + h * 64 + c0;
                asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta),
                    "r"(r[0]),"r"(r[1]),"r"(r[2]),"r"(r[3]),"r"(r[4]),"r"(r[5]),"r"(r[6]),"r"(r[7]),"r"(r[8]),"r"(r[9]),"r"(r[10]),"r"(r[11]),"r"(r[12]),"r"(r[13]),"r"(r[14]),"r"(r[15]),"r"(r[16]),"r"(r[17]),"r"(r[18]),"r"(r[19]),"r"(r[20]),"r"(r[21]),"r"(r[22]),"r"(r[23]),"r"(r[24]),"r"(r[25]),"r"(r[26]),"r"(r[27]),"r"(r[28]),"r"(r[29]),"r"(r[30]),"r"(r[31]));
            }
        asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;"); asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t d0 = tm + 128;
    if (threadIdx.x == 0) {
        const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
        const uint64_t bh = bdesc(su(sm)), bl = bdesc(su(sm) + N * K * 2);
        const uint32_t ah = tm, al = tm + 64;
        for (int ks = 0; ks < 8; ks++) {
            const uint32_t acc = ks ? 1u : 0u;
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d0), "r"(ah + ks * 8), "l"(bl + ks * 16), "r"(idesc), "r"(acc));
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d0), "r"(al + ks * 8), "l"(bh + ks * 16), "r"(idesc), "r"(1u));
        }
        for (int ks = 0; ks < 8; ks++) {   // main term: main_accs accumulators (1 or 2)
            const int a = main_accs == 2 ? (ks >> 2) : 0;
            const uint32_t acc = (ks == 0 || (main_accs == 2 && ks == 4)) ? 0u : 1u;
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d0 + 64 + 64 * a), "r"(ah + ks * 8), "l"(bh + ks * 16), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(&mb)));
    }
    { uint32_t dn = 0; while (!dn) asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}" : "=r"(dn) : "r"(su(&mb)), "r"(0)); }
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int m = w * 32 + l;
    for (int a = 0; a < 3; a++)
        for (int c0 = 0; c0 < N; c0 += 32) {
            uint32_t v[32];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]),"=r"(v[8]),"=r"(v[9]),"=r"(v[10]),"=r"(v[11]),"=r"(v[12]),"=r"(v[13]),"=r"(v[14]),"=r"(v[15]),"=r"(v[16]),"=r"(v[17]),"=r"(v[18]),"=r"(v[19]),"=r"(v[20]),"=r"(v[21]),"=r"(v[22]),"=r"(v[23]),"=r"(v[24]),"=r"(v[25]),"=r"(v[26]),"=r"(v[27]),"=r"(v[28]),"=r"(v[29]),"=r"(v[30]),"=r"(v[31])
                : "r"(d0 + 64 * a + ((uint32_t)(w * 32) << 16) + c0));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
            for (int c = 0; c < 32; c++) D[(a * M + m) * N + c0 + c] = __uint_as_float(v[c]);
        }
    asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
    if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

static float h2f(__half h) { return __half2float(h); }

int main() {
    std::mt19937_64 rng(11);
    std::normal_distribution<double> nd(0.0, 1.0);
    // random unitary (Gram-Schmidt of complex Gaussian rows)
    using cd = std::complex<double>;
    std::vector<float> A(M * K);
    std::vector<float> B(N * K);
    std::vector<__half> Ah(M * K), Al(M * K), Bh(N * K), Bl(N * K);
    std::vector<float> D(3 * M * N);
    __half *dAh, *dAl, *dBh, *dBl; float* dD;
    CK(cudaMalloc(&dAh, M * K * 2)); CK(cudaMalloc(&dAl, M * K * 2)); CK(cudaMalloc(&dBh, N * K * 2)); CK(cudaMalloc(&dBl, N * K * 2));
    CK(cudaMalloc(&dD, D.size() * 4));
    const int smem = 2 * N * K * 2;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    for (int scheme = 0; scheme < 3; scheme++) {
        double sd = 0, sa = 0, g2 = 0, r2 = 0, e2 = 0, emax = 0;
        long long inexact = 0, total = 0;
        for (int rep = 0; rep < 60; rep++) {
            std::vector<cd> U(64 * 64);
            for (auto& u : U) u = cd(nd(rng), nd(rng));
            for (int r = 0; r < 64; r++) {
                for (int q = 0; q < r; q++) {
                    cd dot = 0;
                    for (int c = 0; c < 64; c++) dot += std::conj(U[q * 64 + c]) * U[r * 64 + c];
                    for (int c = 0; c < 64; c++) U[r * 64 + c] -= dot * U[q * 64 + c];
                }
                double nn = 0;
                for (int c = 0; c < 64; c++) nn += std::norm(U[r * 64 + c]);
                for (int c = 0; c < 64; c++) U[r * 64 + c] /= std::sqrt(nn);
            }
            for (int m = 0; m < M; m++)
                for (int kk = 0; kk < K; kk++) {
                    const cd u = U[(m >> 1) * 64 + (kk & 63)];
                    A[m * K + kk] = (float)((m & 1) ? (kk < 64 ? u.imag() : u.real()) : (kk < 64 ? u.real() : -u.imag()));
                }
            const double sc = std::ldexp(1.0, -(rep % 20));
            for (int n = 0; n < N; n++)
                for (int kk = 0; kk < K; kk++) B[n * K + kk] = (float)(nd(rng) * sc);
            if (rep % 7 == 3)   // a few structured columns: exact zeros
                for (int kk = 0; kk < K; kk += 3) B[5 * K + kk] = 0.f;
            // splits
            std::vector<int> F(M), E(N);
            for (int m = 0; m < M; m++) {
                float mx = 0; for (int kk = 0; kk < K; kk++) mx = std::fmax(mx, std::fabs(A[m * K + kk]));
                F[m] = scheme == 0 ? 14 : 10 - std::ilogb(mx);
            }
            for (int n = 0; n < N; n++) {
                float mx = 0; for (int kk = 0; kk < K; kk++) mx = std::fmax(mx, std::fabs(B[n * K + kk]));
                E[n] = scheme == 0 ? 15 + 0 : (mx > 0 ? 10 - std::ilogb(mx) : 0);
                if (scheme == 0) E[n] = 15 + (int)std::lround(-std::log2(sc));   // round-1: fixed scale (state scale known)
            }
            auto split = [&](float x, int e, __half& h, __half& lo) {
                const float v = std::ldexp(x, e);
                if (scheme == 0) { h = __float2half_rn(v); lo = __float2half_rn(v - h2f(h)); }
                else { const float hi = std::rint(v); h = __float2half_rn(hi); lo = __float2half_rn(v - hi); }
            };
            for (int m = 0; m < M; m++) for (int kk = 0; kk < K; kk++) split(A[m * K + kk], F[m], Ah[m * K + kk], Al[m * K + kk]);
            for (int n = 0; n < N; n++) for (int kk = 0; kk < K; kk++) split(B[n * K + kk], E[n], Bh[n * K + kk], Bl[n * K + kk]);
            CK(cudaMemcpy(dAh, Ah.data(), M * K * 2, cudaMemcpyHostToDevice)); CK(cudaMemcpy(dAl, Al.data(), M * K * 2, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(dBh, Bh.data(), N * K * 2, cudaMemcpyHostToDevice)); CK(cudaMemcpy(dBl, Bl.data(), N * K * 2, cudaMemcpyHostToDevice));
            const int main_accs = scheme == 0 ? 2 : 1;
            k<<<1, 128, smem>>>(dAh, dAl, dBh, dBl, dD, main_accs);
            CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
            CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
            for (int m = 0; m < M; m++) for (int n = 0; n < N; n++) {
                double r = 0; for (int kk = 0; kk < K; kk++) r += (double)A[m * K + kk] * B[n * K + kk];
                const float cross = D[(0 * M + m) * N + n], main0 = D[(1 * M + m) * N + n], main1 = D[(2 * M + m) * N + n];
                float s = main_accs == 2 ? (cross + main0) + main1 : main0 + cross;   // fp32 add.rn like the kernel
                const float g = std::ldexp(s, -(F[m] + E[n]));
                if (scheme > 0) {
                    long long ex = 0;
                    for (int kk = 0; kk < K; kk++) ex += (long long)h2f(Ah[m * K + kk]) * (long long)h2f(Bh[n * K + kk]);
                    inexact += (double)main0 != (double)ex;
                    total++;
                }
                sd += (g - r) * (r > 0 ? 1 : -1) / sc; sa += std::fabs(r) / sc;
                g2 += (double)g * g / (sc * sc); r2 += r * r / (sc * sc); e2 += (g - r) * (g - r) / (sc * sc);
                emax = std::fmax(emax, std::fabs(g - r) / sc);
            }
        }
        const char* names[3] = {"float split, 2 main accs (r1)", "exact main, 1 acc", "exact main (repeat)"};
        printf("%-32s bias(rel) %+.3e  norm2-1 %+.3e  rms rel %.3e  max abs/scale %.2e  main inexact %lld/%lld\n",
               names[scheme], sd / sa, g2 / r2 - 1, std::sqrt(e2 / r2), emax, inexact, total);
    }
    return 0;
}
