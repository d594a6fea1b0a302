// NVLink peer-access patterns for the remap all-to-all (one process, all visible GPUs).
// Each device's buffer is split into W parts; part q of device d is exchanged with part d of
// device q (the data movement of a log2(W)-bit remap).  Reported: outbound GB/s per device
// = (W-1)/W * bytes / time, time = wall clock of all devices (synchronised).
//   swap : in place, d swaps half of the (d,q) pairs with loads+stores to q   (current k_peer_swap)
//   push : d stores its part q into q's staging part d                        (remote stores only)
//   pull : d loads q's part d into its own staging part q                     (remote loads only)
//   ce   : cudaMemcpyPeerAsync of every (d,q) part on a stream per peer        (copy engines)
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a p2p_bench.cu -o p2p_bench
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                   \
    do {                                                                        \
        cudaError_t e = (x);                                                    \
        if (e != cudaSuccess) {                                                 \
            printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
            exit(1);                                                            \
        }                                                                       \
    } while (0)

constexpr int kT = 256, kU = 4;

__global__ void k_swap(float4* loc, float4* rem, uint64_t n) {   // swap loc[i] <-> rem[i], i < n
    const uint64_t stride = (uint64_t)gridDim.x * kT * kU;
    for (uint64_t i0 = (uint64_t)blockIdx.x * kT * kU + threadIdx.x; i0 < n; i0 += stride) {
        float4 a[kU], b[kU];
#pragma unroll
        for (int u = 0; u < kU; u++) {
            const uint64_t i = i0 + (uint64_t)u * kT;
            if (i < n) { a[u] = loc[i]; b[u] = rem[i]; }
        }
#pragma unroll
        for (int u = 0; u < kU; u++) {
            const uint64_t i = i0 + (uint64_t)u * kT;
            if (i < n) { loc[i] = b[u]; rem[i] = a[u]; }
        }
    }
}

__global__ void k_copy(const float4* __restrict__ src, float4* __restrict__ dst, uint64_t n) {
    const uint64_t stride = (uint64_t)gridDim.x * kT * kU;
    for (uint64_t i0 = (uint64_t)blockIdx.x * kT * kU + threadIdx.x; i0 < n; i0 += stride) {
        float4 a[kU];
#pragma unroll
        for (int u = 0; u < kU; u++) {
            const uint64_t i = i0 + (uint64_t)u * kT;
            if (i < n) a[u] = src[i];
        }
#pragma unroll
        for (int u = 0; u < kU; u++) {
            const uint64_t i = i0 + (uint64_t)u * kT;
            if (i < n) dst[i] = a[u];
        }
    }
}

int main(int argc, char** argv) {
    int W = 0;
    CK(cudaGetDeviceCount(&W));
    if (argc > 1) W = atoi(argv[1]);
    const uint64_t bytes = (argc > 2 ? strtoull(argv[2], 0, 10) : 8ull) << 30;   // per device
    const int grid = argc > 3 ? atoi(argv[3]) : 148 * 8;
    printf("W=%d bytes/dev=%llu GiB grid=%d\n", W, (unsigned long long)(bytes >> 30), grid);
    std::vector<float4*> buf(W), stg(W);
    std::vector<std::vector<cudaStream_t>> st(W, std::vector<cudaStream_t>(W));
    for (int d = 0; d < W; d++) {
        CK(cudaSetDevice(d));
        for (int q = 0; q < W; q++)
            if (q != d) {
                int can = 0;
                CK(cudaDeviceCanAccessPeer(&can, d, q));
                if (!can) { printf("no peer access %d->%d\n", d, q); return 1; }
                CK(cudaDeviceEnablePeerAccess(q, 0));
            }
        CK(cudaMalloc(&buf[d], bytes));
        CK(cudaMalloc(&stg[d], bytes));
        CK(cudaMemset(buf[d], d, bytes));
        for (int q = 0; q < W; q++) CK(cudaStreamCreateWithFlags(&st[d][q], cudaStreamNonBlocking));
    }
    const uint64_t part = bytes / W / 16;   // float4 per part
    auto sync_all = [&]() {
        for (int d = 0; d < W; d++) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
    };
    auto run = [&](const char* name, auto&& launch) {
        for (int rep = 0; rep < 4; rep++) {
            sync_all();
            auto t0 = std::chrono::steady_clock::now();
            for (int d = 0; d < W; d++) { CK(cudaSetDevice(d)); launch(d); }
            sync_all();
            double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            if (rep > 0)
                printf("%-6s W=%d rep %d: %.3f ms, outbound %.1f GB/s per device\n", name, W, rep, s * 1e3,
                       (double)(W - 1) * part * 16 / s / 1e9);
        }
    };
    // one kernel per peer on its own stream (concurrent), grid split among peers
    const int gpp = grid / (W - 1) > 0 ? grid / (W - 1) : 1;
    run("swap", [&](int d) {
        for (int q = 0; q < W; q++) {
            if (q == d) continue;
            // pair (d,q): elements of d's part q <-> q's part d; d < q takes the first half
            const uint64_t half = part / 2;
            const uint64_t b0 = d < q ? 0 : half, n = d < q ? half : part - half;
            k_swap<<<gpp, kT, 0, st[d][q]>>>(buf[d] + q * part + b0, buf[q] + d * part + b0, n);
        }
    });
    run("push", [&](int d) {
        for (int q = 0; q < W; q++)
            if (q != d) k_copy<<<gpp, kT, 0, st[d][q]>>>(buf[d] + q * part, stg[q] + d * part, part);
    });
    run("pull", [&](int d) {
        for (int q = 0; q < W; q++)
            if (q != d) k_copy<<<gpp, kT, 0, st[d][q]>>>(buf[q] + d * part, stg[d] + q * part, part);
    });
    run("ce", [&](int d) {
        for (int q = 0; q < W; q++)
            if (q != d) CK(cudaMemcpyPeerAsync(stg[q] + d * part, q, buf[d] + q * part, d, part * 16, st[d][q]));
    });
    run("local", [&](int d) {   // local copy of the same bytes (HBM reference)
        k_copy<<<grid, kT, 0, st[d][0]>>>(buf[d], stg[d], part * (W - 1));
    });
    return 0;
}
