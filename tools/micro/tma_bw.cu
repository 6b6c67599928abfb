// Microbenchmark: how fast can ONE SM ingest 32 KB matrices (the chain CTA's
// per-block data) by TMA bulk copies vs plain coalesced loads, from an
// L2-resident or HBM-resident pool?
#include <cstdio>
#include <cuda_runtime.h>
constexpr int kMat = 4096;  // doubles (32 KB)
__global__ void k_tma(const double* pool, int nmat, int stride_mats, int per_blk, long long* out) {
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) unsigned long long mbar[2];
    const unsigned mb0 = (unsigned)__cvta_generic_to_shared(&mbar[0]);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(mb0));
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(mb0 + 8));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int nblk = nmat / per_blk;
    auto issue = [&](int kb) {
        const int st = kb & 1;
        const unsigned mb = mb0 + 8 * st;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(mb), "r"((unsigned)(per_blk * kMat * 8)) : "memory");
        for (int q = 0; q < per_blk; ++q) {
            const unsigned dst = (unsigned)__cvta_generic_to_shared(sm + (st * per_blk + q) * kMat);
            const double* src = pool + (long long)((kb * per_blk + q) * stride_mats % (nmat)) * kMat;
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                         "l"(src), "r"((unsigned)(kMat * 8)), "r"(mb) : "memory");
        }
    };
    long long t0 = clock64();
    double acc = 0;
    if (threadIdx.x == 0) issue(0);
    for (int kb = 0; kb < nblk; ++kb) {
        if (threadIdx.x == 0 && kb + 1 < nblk) issue(kb + 1);
        const unsigned mb = mb0 + 8 * (kb & 1), par = (kb >> 1) & 1;
        unsigned done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(mb), "r"(par) : "memory");
        acc += sm[(kb & 1) * per_blk * kMat + threadIdx.x];
        __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (acc == 12345.0) out[0] = 0;
}
__global__ void k_ldg(const double* pool, int nmat, int per_blk, long long* out) {
    long long t0 = clock64();
    double acc = 0;
    const int nblk = nmat / per_blk;
    for (int kb = 0; kb < nblk; ++kb) {
        double r[16 * 3];
        for (int q = 0; q < per_blk; ++q)
#pragma unroll
            for (int j = 0; j < 16; ++j) r[q * 16 + j] = pool[(long long)(kb * per_blk + q) * kMat + j * 256 + threadIdx.x];
        for (int q = 0; q < per_blk * 16; ++q) acc += r[q];
        __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (acc == 12345.0) out[0] = 0;
}
int main() {
    const int nmat = 768;  // 24 MB pool
    double* pool;
    cudaMalloc(&pool, (size_t)nmat * kMat * 8);
    cudaMemset(pool, 0, (size_t)nmat * kMat * 8);
    double* big;  // L2 flush
    cudaMalloc(&big, 512ull << 20);
    long long* out;
    cudaMalloc(&out, 148 * 8);
    cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 3 * kMat * 8);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    for (int l2 = 0; l2 < 2; ++l2) {
        for (int grid : {1, 148}) {
            for (int rep = 0; rep < 2; ++rep) {
                if (!l2) cudaMemset(big, rep, 512ull << 20);
                else k_tma<<<1, 256, 2 * 3 * kMat * 8>>>(pool, nmat, 1, 3, out);  // warm L2
                cudaDeviceSynchronize();
                k_tma<<<grid, 256, 2 * 3 * kMat * 8>>>(pool, nmat, 1, 3, out);
                long long cyc;
                cudaDeviceSynchronize();
                cudaMemcpy(&cyc, out, 8, cudaMemcpyDeviceToHost);
                const double us = cyc / (clk / 1e3);
                printf("TMA %s grid %3d: %.2f us per 96 KB block, %.1f GB/s per SM\n", l2 ? "L2 " : "HBM", grid,
                       us / (nmat / 3), (double)nmat * kMat * 8 / (us * 1e3));
            }
            if (!l2) cudaMemset(big, 7, 512ull << 20);
            else k_tma<<<1, 256, 2 * 3 * kMat * 8>>>(pool, nmat, 1, 3, out);
            cudaDeviceSynchronize();
            k_ldg<<<grid, 256>>>(pool, nmat, 3, out);
            long long cyc;
            cudaDeviceSynchronize();
            cudaMemcpy(&cyc, out, 8, cudaMemcpyDeviceToHost);
            const double us = cyc / (clk / 1e3);
            printf("LDG %s grid %3d: %.2f us per 96 KB block, %.1f GB/s per SM\n", l2 ? "L2 " : "HBM", grid,
                   us / (nmat / 3), (double)nmat * kMat * 8 / (us * 1e3));
        }
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
