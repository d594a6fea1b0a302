// tc_probe.cu -- validates the tcgen05 building blocks used by the tensor-core gate pass:
// kind::tf32 MMA, M=128 N=64 K=8, A (128x128) resident in TMEM, B (K=128 x N=64) in shared
// memory, K-major, no swizzle ("interleave" core matrices 8 rows x 16 B), D in TMEM, read back
// with tcgen05.ld 32x32b.  Compares 1-term and 3xTF32 products with an fp64 reference.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int M = 128, N = 64, K = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t bdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= 1ull << 46;   // version (sm100)
    return d;          // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

__device__ __forceinline__ float tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// B smem layout (K-major, interleave): element (n, k) at
//   (n/8)*SBO + (k/4)*LBO + (n%8)*16 + (k%4)*4,   LBO = 128, SBO = (K/4)*128
__device__ __forceinline__ uint32_t b_off(int n, int k) {
    return (n >> 3) * ((K / 4) * 128) + (k >> 2) * 128 + (n & 7) * 16 + (k & 3) * 4;
}

template <int SPLIT>
__global__ void __launch_bounds__(128) k_probe(const float* __restrict__ A, const float* __restrict__ B,
                                               float* __restrict__ D) {
    extern __shared__ __align__(1024) uint8_t smem[];
    float* bhi = reinterpret_cast<float*>(smem);
    float* blo = reinterpret_cast<float*>(smem + N * K * 4);
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t mbar;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    // B -> smem (hi, lo)
    for (int i = threadIdx.x; i < N * K; i += 128) {
        const int n = i / K, k = i % K;
        const float x = B[n * K + k];   // B^T row-major: [n][k]
        const float h = SPLIT ? tf32_rna(x) : x;
        *reinterpret_cast<float*>(smem + b_off(n, k)) = h;
        *reinterpret_cast<float*>(smem + N * K * 4 + b_off(n, k)) = x - h;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tmem_base;
    // A -> TMEM: warp q owns lanes 32q..32q+31, row m = 32q + lane; cols [0,128) hi, [128,256) lo
    {
        const int m = warp * 32 + lane;
        for (int c0 = 0; c0 < K; c0 += 32) {
            uint32_t h[32], l[32];
            for (int c = 0; c < 32; c++) {
                const float x = A[m * K + c0 + c];
                const float hh = SPLIT ? tf32_rna(x) : x;
                h[c] = __float_as_uint(hh);
                l[c] = __float_as_uint(x - hh);
            }
            const uint32_t ta = tm + ((uint32_t)(warp * 32) << 16) + c0;
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta),
                "r"(h[0]), "r"(h[1]), "r"(h[2]), "r"(h[3]), "r"(h[4]), "r"(h[5]), "r"(h[6]), "r"(h[7]), "r"(h[8]),
                "r"(h[9]), "r"(h[10]), "r"(h[11]), "r"(h[12]), "r"(h[13]), "r"(h[14]), "r"(h[15]), "r"(h[16]),
                "r"(h[17]), "r"(h[18]), "r"(h[19]), "r"(h[20]), "r"(h[21]), "r"(h[22]), "r"(h[23]), "r"(h[24]),
                "r"(h[25]), "r"(h[26]), "r"(h[27]), "r"(h[28]), "r"(h[29]), "r"(h[30]), "r"(h[31]));
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta + 128),
                "r"(l[0]), "r"(l[1]), "r"(l[2]), "r"(l[3]), "r"(l[4]), "r"(l[5]), "r"(l[6]), "r"(l[7]), "r"(l[8]),
                "r"(l[9]), "r"(l[10]), "r"(l[11]), "r"(l[12]), "r"(l[13]), "r"(l[14]), "r"(l[15]), "r"(l[16]),
                "r"(l[17]), "r"(l[18]), "r"(l[19]), "r"(l[20]), "r"(l[21]), "r"(l[22]), "r"(l[23]), "r"(l[24]),
                "r"(l[25]), "r"(l[26]), "r"(l[27]), "r"(l[28]), "r"(l[29]), "r"(l[30]), "r"(l[31]));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t d_tm = tm + 256;
    if (threadIdx.x == 0) {
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
        const uint32_t sb = smem_u32(smem);
        int first = 1;
        for (int ks = 0; ks < K / 8; ks++) {
            for (int term = 0; term < (SPLIT ? 3 : 1); term++) {
                const uint32_t a_tm = tm + ks * 8 + (term == 2 ? 128 : 0);
                const uint32_t b_addr = sb + (term == 1 ? N * K * 4 : 0) + ks * 2 * 128;
                const uint64_t bd = bdesc(b_addr, 128, (K / 4) * 128);
                const uint32_t acc = first ? 0u : 1u;
                asm volatile(
                    "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                    "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tm),
                    "r"(a_tm), "l"(bd), "r"(idesc), "r"(acc));
                first = 0;
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
    }
    // wait for the MMAs
    {
        uint32_t done = 0;
        while (!done) {
            asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
                         : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
        }
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    {
        const int m = warp * 32 + lane;
        for (int c0 = 0; c0 < N; c0 += 32) {
            uint32_t v[32];
            const uint32_t ta = d_tm + ((uint32_t)(warp * 32) << 16) + c0;
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                  "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                  "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                : "r"(ta));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
            for (int c = 0; c < 32; c++) D[m * N + c0 + c] = __uint_as_float(v[c]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
    std::vector<float> A(M * K), B(N * K), D(M * N);
    srand(1);
    for (auto& x : A) x = (rand() / (float)RAND_MAX - 0.5f) * 0.3f;
    for (auto& x : B) x = (rand() / (float)RAND_MAX - 0.5f) * 1e-4f;
    float *dA, *dB, *dD;
    CK(cudaMalloc(&dA, A.size() * 4));
    CK(cudaMalloc(&dB, B.size() * 4));
    CK(cudaMalloc(&dD, D.size() * 4));
    CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
    const int smem = 2 * N * K * 4;
    for (int split = 0; split < 2; split++) {
        if (split) {
            CK(cudaFuncSetAttribute(k_probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            k_probe<1><<<1, 128, smem>>>(dA, dB, dD);
        } else {
            CK(cudaFuncSetAttribute(k_probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            k_probe<0><<<1, 128, smem>>>(dA, dB, dD);
        }
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
        double maxrel = 0, maxabs = 0, ref_max = 0;
        for (int m = 0; m < M; m++)
            for (int n = 0; n < N; n++) {
                double r = 0;
                for (int k = 0; k < K; k++) r += (double)A[m * K + k] * B[n * K + k];
                maxabs = std::fmax(maxabs, std::fabs(r - D[m * N + n]));
                ref_max = std::fmax(ref_max, std::fabs(r));
            }
        maxrel = maxabs / ref_max;
        printf("split=%d  max|err| = %.3e  (rel to max|D| %.3e)  D[0]=%.6e D[last]=%.6e\n", split, maxabs, maxrel,
               D[0], D[M * N - 1]);
    }
    return 0;
}
