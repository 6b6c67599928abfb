// sm_100a fp64 kernels of the invert-Krylov ER hot path.
//
// Compiled with -fmad=false: every a*b+c rounds twice, exactly like the
// reference's x86-64 build (no FMA contraction), so the kernels that keep the
// reference's accumulation order are bit-identical to it:
//   spmv_rows            <- spmv                  sparse_matrix.cpp:69-82
//   trsv_*               <- Factorization::solve  sparse_lu.cpp:255-291
//   apply_u / apply_l    <- Factorization::apply  sparse_lu.cpp:293-304
//   dense_*              <- dense_matrix.cpp:33-225, krylov.cpp:85-101
//   combine_*            <- basis_combination / er_eval tail
//                           krylov.cpp:32-36, integrate.cpp:241,262-263
// Dot products and norms are parallel reductions with a fixed tree (run-to-run
// deterministic, not bit-identical to the reference's serial sums).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace exg {
namespace dev {

constexpr unsigned long long kSentinel = 0xFFFFFFFFFFFFFFFFull;  // "not yet solved"
constexpr unsigned long long kCanonNaN = 0x7FF8000000000000ull;
constexpr double kReorthFactor = 0.70710678118654752;  // krylov.cpp:14
constexpr double kCondLimit = 1e12;                    // krylov.cpp:13

// ---- control block shared by the Arnoldi kernels (device memory) ----------
struct Ctrl {
    // configuration of the running MEVP
    double h, eps, breakdown_tol;
    int m_max, check_stride;
    // state
    int j;            // 0-based column being built (V[0..j] exist)
    int m;            // basis dimension after the last iteration
    int happy;
    int invertible;
    int need_weight;  // residual test pending for this iteration
    int converged;
    int status;       // exg_status of the MEVP (0 ok)
    int skip;         // start-vector early-out taken (er_eval)
    int fresh;        // a fresh basis was built by the last er_eval
    double beta, pre, post, h_next, s, weight, last_residual;
    double h_sub;
    double xinf;      // ||x_k||_inf for the er_eval early-out
    unsigned int arnoldi_iters;
    unsigned int mgs_passes;  // algorithmic n-vector passes of the MGS kernels (J + 2, + J + 1 per reorth)
    unsigned int reorths;     // reorthogonalisation passes taken
};

__device__ __forceinline__ unsigned long long ld_relaxed(const double* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(double* p, double x) {
    unsigned long long v = __double_as_longlong(x);
    // never publish the sentinel, nor any NaN sharing its high word (readers
    // may test the high word alone)
    if ((v >> 32) == 0xFFFFFFFFull) v = kCanonNaN;
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }

// fixed-pattern warp sum (lane 0 holds the result)
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}

// deterministic block sum; result valid in every thread
__device__ __forceinline__ double block_sum(double v, double* sh) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    if (warp == 0) {
        double t = lane < nw ? sh[lane] : 0.0;
        t = warp_sum(t);
        if (lane == 0) sh[32] = t;
    }
    __syncthreads();
    return sh[32];
}

// sense-free generation grid barrier (cooperative launch => co-residency)
__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int nblocks) {
    __syncthreads();
    if (nblocks > 1 && threadIdx.x == 0) {
        volatile unsigned int* vgen = bar + 1;
        const unsigned int gen = *vgen;
        __threadfence();
        const unsigned int arrived = atomicAdd(bar, 1u);
        if (arrived == nblocks - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*vgen == gen) {
            }
        }
        __threadfence();
    }
    __syncthreads();
}

}  // namespace dev
}  // namespace exg
