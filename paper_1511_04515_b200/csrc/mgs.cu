// k_mgs2: modified Gram-Schmidt with one conditional re-orthogonalisation
// (orthogonalize, krylov.cpp:46-78) for FAST mode, one cooperative launch per
// Arnoldi step.
//
// Each CTA owns one tile of the vectors (n / grid elements): its part of w
// lives in registers for the whole step, and the basis columns v_0..v_j are
// pulled through a shared-memory ring of S tile slots with bulk async copies
// (cp.async.bulk + mbarrier complete_tx), so the HBM stream of V runs ahead of
// the reductions instead of waiting for them.  Columns are taken B at a time:
// the B dot products <w, v_i> of a group are reduced together (one grid-wide
// exchange per group instead of one per column), then w is updated with the
// group's columns in order, from the same shared-memory tiles (V is read from
// HBM exactly once per pass).  Inside a group the coefficients are those of
// classical Gram-Schmidt, across groups those of MGS; with the basis
// orthonormal to rounding (the reorthogonalisation trigger post < pre / sqrt 2
// is kept) the two differ by O(eps |h|), the size of the dot products' own
// rounding.  FAST mode only; EXACT mode keeps k_mgs (column by column).
//
// The grid-wide exchange is one round trip: every CTA publishes its partial
// sums into sentinel-initialised slots with one relaxed store each, and every
// CTA then sums all CTAs' partials in a fixed order (deterministic, identical
// in every CTA, no atomics, no second phase).  Two slot sets alternate between
// launches; a launch clears the set the next one will use.
#include <algorithm>

#include "device.hpp"
#include "kernels.cuh"

namespace exg {
namespace dev {

namespace {

constexpr int kThreads = 1024;
constexpr int kKMax = 12;  // elements of w per thread (tile <= 12288)
constexpr int kBMax = kMgs2BMax;
constexpr int kSMax = 8;
constexpr size_t kSmemMax = 227 * 1024;
constexpr size_t kSmemAux = (size_t)kBMax * 32 * 8 + kBMax * 8 + kSMax * 8 + 64;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ double warp_sum_all(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    unsigned ok = 0;
    while (!ok) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(ok)
            : "r"(bar), "r"(parity)
            : "memory");
    }
}

}  // namespace

__global__ void __launch_bounds__(kThreads, 1)
    k_mgs2(Mgs2Args a) {
    extern __shared__ __align__(128) unsigned char sm[];
    Ctrl* c = a.ctrl;
    if (c->converged || c->status) return;
    const int j = c->j, n = a.n, T = a.tile, S = a.S, B = a.B;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int G = gridDim.x, blk = blockIdx.x;
    const long long e0 = (long long)blk * T;
    const int len = (int)min((long long)T, a.ldv - e0);  // ldv-padded tile (the pad of V is zero)
    double* tiles = reinterpret_cast<double*>(sm);
    double* red = tiles + (size_t)S * T;
    double* hsh = red + kBMax * 32;
    const unsigned bar0 = smem_u32(hsh + kBMax);
    // slot sets: this launch's and the next one's
    const unsigned seq = *reinterpret_cast<volatile unsigned*>(a.seq);
    const size_t set_doubles = (size_t)a.inst_cap * G * kBMax;
    double* slots = a.slots + (seq & 1u) * set_doubles;
    if (G > 1) {
        double* other = a.slots + ((seq + 1u) & 1u) * set_doubles;
        const int next_inst = min(a.inst_cap, 2 * ((j + 2 + B - 1) / B) + 3);
        const size_t cnt = (size_t)next_inst * G * kBMax;
        for (size_t i = (size_t)blk * kThreads + t; i < cnt; i += (size_t)G * kThreads)
            reinterpret_cast<unsigned long long*>(other)[i] = kSentinel;
    }
    if (t == 0) {
        for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8 * s));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    int q_issued = 0;  // thread 0: columns requested so far (both passes)
    auto issue = [&](int consumed, int limit) {
        while (q_issued < limit && q_issued < consumed + S) {
            const int slot = q_issued % S, col = q_issued % (j + 1);
            const unsigned bar = bar0 + 8 * slot;
            const unsigned bytes = (unsigned)len * 8u;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(tiles + (size_t)slot * T)),
                "l"(a.V + (long long)col * a.ldv + e0), "r"(bytes), "r"(bar)
                : "memory");
            ++q_issued;
        }
    };
    if (t == 0) issue(0, j + 1);
    double w[kKMax];
#pragma unroll
    for (int k = 0; k < kKMax; ++k) {
        const int o = t + k * kThreads;
        w[k] = (o < len && e0 + o < n) ? a.w[e0 + o] : 0.0;
    }
    int inst = 0;
    // grid-wide sums of nb values per thread; results in hsh[0..nb)
    auto exchange = [&](double* d, int nb) {
#pragma unroll
        for (int b = 0; b < kBMax; ++b)
            if (b < nb) {
                d[b] = warp_sum_all(d[b]);
                if (lane == 0) red[b * 32 + warp] = d[b];
            }
        __syncthreads();
        if (warp < nb) {
            double v = warp_sum_all(red[warp * 32 + lane]);
            if (G > 1) {
                double* sl = slots + (size_t)inst * G * kBMax + warp;
                if (lane == 0) st_relaxed(sl + (size_t)blk * kBMax, v);
                // every lane's slots are requested together (one round trip when
                // the partials are there), then only the missing ones again
                constexpr int kPer = 8;  // grid <= 256
                unsigned long long u[kPer];
#pragma unroll
                for (int z = 0; z < kPer; ++z) {
                    const int q = lane + 32 * z;
                    u[z] = q < G ? ld_relaxed(sl + (size_t)q * kBMax) : 0ull;
                }
                bool all = false;
                while (!all) {
                    all = true;
#pragma unroll
                    for (int z = 0; z < kPer; ++z)
                        if (u[z] == kSentinel) {
                            u[z] = ld_relaxed(sl + (size_t)(lane + 32 * z) * kBMax);
                            all = all && u[z] != kSentinel;
                        }
                }
                double acc = 0.0;
#pragma unroll
                for (int z = 0; z < kPer; ++z)
                    if (lane + 32 * z < G) acc += __longlong_as_double(u[z]);
                v = warp_sum_all(acc);
            }
            if (lane == 0) hsh[warp] = v;
        }
        ++inst;
        __syncthreads();
    };
    double dd[kBMax];
    dd[0] = 0.0;
#pragma unroll
    for (int k = 0; k < kKMax; ++k) dd[0] += w[k] * w[k];
    exchange(dd, 1);
    const double pre = sqrt(hsh[0]);
    double* hcol = a.hbar + (long long)j * a.hld;
    int q_done = 0;
    for (int pass = 0; pass < 2; ++pass) {
        const int limit = (pass + 1) * (j + 1);
        if (pass == 1 && t == 0) issue(q_done, limit);
        for (int i0 = 0; i0 <= j; i0 += B) {
            const int nb = min(B, j + 1 - i0);
#pragma unroll
            for (int b = 0; b < kBMax; ++b) {
                dd[b] = 0.0;
                if (b < nb) {
                    const int q = q_done + b;
                    mbar_wait(bar0 + 8 * (q % S), (unsigned)(q / S) & 1u);
                    const double* tile = tiles + (size_t)(q % S) * T;
#pragma unroll
                    for (int k = 0; k < kKMax; ++k) {
                        const int o = t + k * kThreads;
                        if (o < len) dd[b] += w[k] * tile[o];
                    }
                }
            }
            exchange(dd, nb);
#pragma unroll
            for (int b = 0; b < kBMax; ++b)
                if (b < nb) {
                    const int q = q_done + b;
                    const double mh = -hsh[b];
                    const double* tile = tiles + (size_t)(q % S) * T;
#pragma unroll
                    for (int k = 0; k < kKMax; ++k) {
                        const int o = t + k * kThreads;
                        if (o < len) w[k] += mh * tile[o];
                    }
                }
            if (blk == 0 && t < nb) hcol[i0 + t] = pass == 0 ? hsh[t] : hcol[i0 + t] + hsh[t];
            q_done += nb;
            __syncthreads();  // the group's tiles (and hsh) are consumed
            if (t == 0) issue(q_done, limit);
        }
        dd[0] = 0.0;
#pragma unroll
        for (int k = 0; k < kKMax; ++k) dd[0] += w[k] * w[k];
        exchange(dd, 1);
        const double post = sqrt(hsh[0]);
        if (pass == 1 || !(post < kReorthFactor * pre)) {
            const bool happy = post <= c->breakdown_tol * pre;
            if (!happy) {
                const double ip = 1.0 / post;
                double* vn = a.V + (long long)(j + 1) * a.ldv + e0;
#pragma unroll
                for (int k = 0; k < kKMax; ++k) {
                    const int o = t + k * kThreads;
                    if (o < len && e0 + o < n) vn[o] = w[k] * ip;
                }
            }
            if (blk == 0 && t == 0) {
                hcol[j + 1] = post;
                c->pre = pre;
                c->post = post;
                c->happy = happy;
                c->h_next = happy ? 0.0 : post;
                c->m = j + 1;
                c->mgs_passes += pass == 0 ? (unsigned)(j + 3) : (unsigned)(2 * j + 5);
                c->reorths += pass;
                *a.seq = seq + 1u;  // every CTA read seq before its first exchange
            }
            return;
        }
        __syncthreads();  // hsh[0] read by everyone before the next pass reuses it
    }
}

// launch shape for vectors of length n (ldv-padded); false = not supported
bool mgs2_shape(int n, int num_sms, int b_override, Mgs2Shape* s) {
    if (n <= 0) return false;
    int G = (int)std::min<long long>(std::min(num_sms, 256), std::max<long long>(1, ((long long)n + 4095) / 4096));
    int T = (int)((((long long)n + G - 1) / G + 31) / 32 * 32);
    G = (int)(((long long)n + T - 1) / T);
    if (T > kKMax * kThreads) return false;
    int S = (int)std::min<size_t>(kSMax, (kSmemMax - kSmemAux) / ((size_t)T * 8));
    if (S < 2) return false;
    int B = std::max(1, std::min(kBMax, S / 2));
    if (b_override > 0) B = std::max(1, std::min(std::min(kBMax, S - 1), b_override));
    s->grid = G;
    s->tile = T;
    s->S = S;
    s->B = B;
    s->smem = (size_t)S * T * 8 + kSmemAux;
    return true;
}

cudaError_t mgs2(const Launch& L, Mgs2Args a, const Mgs2Shape& s) {
    static size_t attr = 0;
    if (s.smem > attr) {
        const cudaError_t e = cudaFuncSetAttribute(k_mgs2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax);
        if (e != cudaSuccess) return e;
        attr = kSmemMax;
    }
    a.tile = s.tile;
    a.S = s.S;
    a.B = s.B;
    void* args[] = {(void*)&a};
    cudaError_t e;
    if (s.grid == 1)
        e = cudaLaunchKernel((void*)k_mgs2, dim3(1), dim3(kThreads), args, s.smem, L.stream);
    else
        e = cudaLaunchCooperativeKernel((void*)k_mgs2, dim3(s.grid), dim3(kThreads), args, s.smem, L.stream);
    if (L.launches) ++*L.launches;
    return e;
}

}  // namespace dev
}  // namespace exg
