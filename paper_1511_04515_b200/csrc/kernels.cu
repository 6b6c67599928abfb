// sm_100a kernels of the invert-Krylov ER hot path (fp64, HBM-bound).
// See kernels.cuh for the reference routine each kernel restates.
#include <algorithm>
#include <cfloat>
#include <climits>

#include <cooperative_groups.h>

#include "device.hpp"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace exg {
namespace dev {

// ============================================================================
// CSR SpMV, row-sequential (bit-identical to spmv, sparse_matrix.cpp:76-80).
// One warp owns 32 consecutive rows; their nonzeros are staged into shared
// memory with coalesced loads, then each lane accumulates its own row in the
// reference's column order.  Rows whose 32-row segment exceeds the staging
// capacity read global memory directly.
// ============================================================================
constexpr int kSpmvWarps = 8;
constexpr int kSpmvCap = 384;  // entries staged per warp (4.5 KB)

template <typename XFn, typename OutFn>
__device__ __forceinline__ void spmv_warp_rows(const int* __restrict__ rowptr,
                                               const int* __restrict__ col,
                                               const double* __restrict__ val, int n_rows,
                                               int warp_global, XFn xfn, OutFn out,
                                               int (*s_col)[kSpmvCap], double (*s_val)[kSpmvCap]) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int r0 = warp_global * 32;
    if (r0 >= n_rows) return;
    const int r_end = min(r0 + 32, n_rows);
    const int k0 = rowptr[r0], k1 = rowptr[r_end];
    const int r = r0 + lane;
    if (k1 - k0 <= kSpmvCap) {
        // staging: 8 independent loads in flight per lane per round trip
        for (int k = k0 + lane; k < k1; k += 256) {
            int cc[8];
            double vv[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int kk = k + 32 * q;
                cc[q] = kk < k1 ? __ldcs(col + kk) : 0;
                vv[q] = kk < k1 ? __ldcs(val + kk) : 0.0;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int kk = k + 32 * q;
                if (kk < k1) {
                    s_col[w][kk - k0] = cc[q];
                    s_val[w][kk - k0] = vv[q];
                }
            }
        }
        __syncwarp();
        if (r < n_rows) {
            double s = 0.0;
            const int a = rowptr[r] - k0, b = rowptr[r + 1] - k0;
            // the gathers are independent of the (in-order) accumulation
#pragma unroll 4
            for (int k = a; k < b; ++k) s += s_val[w][k] * xfn(s_col[w][k]);
            out(r, s);
        }
        __syncwarp();
    } else if (r < n_rows) {
        double s = 0.0;
        for (int k = rowptr[r]; k < rowptr[r + 1]; ++k) s += val[k] * xfn(col[k]);
        out(r, s);
    }
}

__global__ void __launch_bounds__(kSpmvWarps * 32)
    k_spmv(const int* __restrict__ rowptr, const int* __restrict__ col,
           const double* __restrict__ val, int n_rows, const double* __restrict__ x,
           double* __restrict__ y, const Ctrl* ctrl, const double* __restrict__ xcol_base,
           long long ldv) {
    // when xcol_base is set, x = V[ctrl->j] (column of the Krylov basis)
    if (ctrl && (ctrl->converged || ctrl->status)) return;
    const double* xs = x;
    if (xcol_base) xs = xcol_base + (long long)ctrl->j * ldv;
    __shared__ int s_col[kSpmvWarps][kSpmvCap];
    __shared__ double s_val[kSpmvWarps][kSpmvCap];
    const int wg = blockIdx.x * kSpmvWarps + (threadIdx.x >> 5);
    spmv_warp_rows(rowptr, col, val, n_rows, wg, [&](int c) { return xs[c]; },
                   [&](int r, double s) { y[r] = s; }, s_col, s_val);
}

// t1 = 0.0 + 1.0 * (B u_k)  (add(residual_F == 0, spmv(B, u_k)), integrate.cpp:224)
// t2 = B * slope, slope = (u_k1 - u_k) * (1/h)              (integrate.cpp:220-221,228)
// FAST-mode SpMV of the Arnoldi loop: 4 lanes per row (CSR-vector), each
// lane strides the row's entries by 4 with fused multiply-adds, a fixed
// 2-step butterfly combines them (deterministic; not the reference's
// row-sequential order, which k_spmv keeps).  Coalesced col/val loads and
// neighbouring gathers instead of one long per-lane chain.
__global__ void __launch_bounds__(256)
    k_spmv_v4(const int* __restrict__ rowptr, const int* __restrict__ col,
              const double* __restrict__ val, int n_rows, double* __restrict__ y, const Ctrl* ctrl,
              const double* __restrict__ xcol_base, long long ldv) {
    if (ctrl->converged || ctrl->status) return;
    const double* xs = xcol_base + (long long)ctrl->j * ldv;
    const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 2;
    const int sub = threadIdx.x & 3;
    double acc = 0.0;
    if (r < n_rows) {
        const int k1 = __ldg(rowptr + r + 1);
        int k = __ldg(rowptr + r) + sub;
        // the first four entries of the lane (a 16-entry row) are requested
        // together, then their gathers, then the multiply-adds in order: four
        // loads in flight per lane instead of one dependent chain
        int c[4];
        double v[4], xv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const bool ok = k + 4 * q < k1;
            c[q] = ok ? __ldcs(col + k + 4 * q) : -1;
            v[q] = ok ? __ldcs(val + k + 4 * q) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) xv[q] = c[q] >= 0 ? xs[c[q]] : 0.0;
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (c[q] >= 0) acc = __fma_rn(v[q], xv[q], acc);
        for (k += 16; k < k1; k += 4) acc = __fma_rn(__ldcs(val + k), xs[__ldcs(col + k)], acc);
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    if (r < n_rows && sub == 0) y[r] = acc;
}

// The same rows, lanes and arithmetic as k_spmv_v4, with col/val streamed
// through shared memory.  k_spmv_v4 chains three dependent global loads per
// row (rowptr -> col/val -> x) with nothing of the next rows in flight behind
// them: ~80 KB per SM per ~2.5 us of chained latency, 3 TB/s at config 1
// whatever the gathers cost (laying rows out for L1 reuse and serving the
// gathers from a shared-memory window of x both left the 56 us launch where it
// was, profiles/r02).  Here CTA b owns ONE contiguous slice of rows, cut into
// strips of 248 rows; a producer warp pulls each strip's col and val ranges
// (contiguous in CSR) into a ring of kSpmvStages shared-memory stages with bulk
// async copies (cp.async.bulk + mbarrier complete_tx), up to four strips
// (~190 KB per SM) ahead of the 31 consumer warps, which read col/val from shared
// memory and only gather x from global memory.  The HBM stream no longer waits
// for the gathers.  (Staging the strips' row bounds through the ring as well
// measured slower, 60 against 51 us: one more copy per stage on the producer.)  max_strip (host, at upload): the most entries any 248
// consecutive rows hold; the launcher keeps k_spmv_v4 when a strip would not fit.
constexpr int kSpmvStages = 4;
constexpr int kSpmvStageCap = 4096;  // entries per stage (16 KB of col + 32 KB of val)
constexpr int kSpmvConsumers = 31;   // warps; 8 rows each per strip
constexpr int kSpmvStripRows = kSpmvConsumers * 8;
constexpr int kSpmvMaxStrips = 256;
constexpr size_t kSpmvStreamSmem = (size_t)kSpmvStages * kSpmvStageCap * 12;
__global__ void __launch_bounds__((kSpmvConsumers + 1) * 32, 1)
    k_spmv_v4t(const int* __restrict__ rowptr, const int* __restrict__ col,
               const double* __restrict__ val, int n_rows, int rows_per_cta, double* __restrict__ y,
               const Ctrl* ctrl, const double* __restrict__ xcol_base, long long ldv) {
    extern __shared__ __align__(128) unsigned char ring[];
    __shared__ __align__(8) unsigned long long bars[2 * kSpmvStages];  // full[], empty[]
    __shared__ int kb[kSpmvMaxStrips + 1];                             // first entry of each strip (and the end)
    if (ctrl->converged || ctrl->status) return;
    const double* xs = xcol_base + (long long)ctrl->j * ldv;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int r0 = blockIdx.x * rows_per_cta;
    const int r1 = min(n_rows, r0 + rows_per_cta);
    const int n_strips = (r1 - r0 + kSpmvStripRows - 1) / kSpmvStripRows;
    const unsigned bar0 = (unsigned)__cvta_generic_to_shared(bars);
    const unsigned ring0 = (unsigned)__cvta_generic_to_shared(ring);
    if (threadIdx.x == 0) {
        for (int q = 0; q < kSpmvStages; ++q) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8 * q));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar0 + 8 * (kSpmvStages + q)), "r"(kSpmvConsumers));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int q = threadIdx.x; q <= n_strips; q += blockDim.x) kb[q] = __ldg(rowptr + min(r0 + q * kSpmvStripRows, r1));
    __syncthreads();
    auto wait = [&](unsigned bar, unsigned parity) {
        unsigned ok = 0;
        while (!ok)
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                : "=r"(ok)
                : "r"(bar), "r"(parity)
                : "memory");
    };
    if (warp == kSpmvConsumers) {
        // producer: strip s goes to stage s mod kSpmvStages once strip s - kSpmvStages left it
        if (lane == 0)
            for (int s = 0; s < n_strips; ++s) {
                const int st = s % kSpmvStages;
                if (s >= kSpmvStages) wait(bar0 + 8 * (kSpmvStages + st), (unsigned)(s / kSpmvStages - 1) & 1u);
                const int k0 = kb[s] & ~3, k1 = (kb[s + 1] + 3) & ~3;  // 16-byte aligned ranges (the arrays are padded)
                const unsigned cnt = (unsigned)(k1 - k0), full = bar0 + 8 * st;
                if (cnt == 0) {
                    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(full) : "memory");
                    continue;
                }
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full), "r"(cnt * 12u) : "memory");
                const unsigned dst = ring0 + (unsigned)st * (kSpmvStageCap * 12);
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                    "l"(col + k0), "r"(cnt * 4u), "r"(full)
                    : "memory");
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        dst + kSpmvStageCap * 4),
                    "l"(val + k0), "r"(cnt * 8u), "r"(full)
                    : "memory");
            }
        return;
    }
    // two strips per round: the gathers of 2 x kSpmvBatch entries per lane are in flight together (the
    // gathers' latency, not their count, is what a round costs)
    constexpr int kSpmvBatch = 6;
    const int sub = lane & 3;
    const int rq = r0 + warp * 8 + (lane >> 2);
    for (int s = 0; s < n_strips; s += 2) {
        int o[2], o1[2], rr[2];
        const int* cs[2];
        const double* vs[2];
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            rr[t] = rq + (s + t) * kSpmvStripRows;
            o[t] = o1[t] = 0;
            if (rr[t] < r1) {
                o1[t] = __ldg(rowptr + rr[t] + 1);
                o[t] = __ldg(rowptr + rr[t]) + sub;
            }
        }
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            const int st = (s + t) % kSpmvStages;
            if (s + t < n_strips) {
                wait(bar0 + 8 * st, (unsigned)((s + t) / kSpmvStages) & 1u);
                const int base = kb[s + t] & ~3;  // the row's entries inside the stage
                o[t] -= base;
                o1[t] -= base;
            }
            cs[t] = reinterpret_cast<const int*>(ring + (size_t)st * (kSpmvStageCap * 12));
            vs[t] = reinterpret_cast<const double*>(ring + (size_t)st * (kSpmvStageCap * 12) + kSpmvStageCap * 4);
        }
        int c[2][kSpmvBatch];
        double xv[2][kSpmvBatch];
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
            for (int q = 0; q < kSpmvBatch; ++q) c[t][q] = o[t] + 4 * q < o1[t] ? cs[t][o[t] + 4 * q] : -1;
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
            for (int q = 0; q < kSpmvBatch; ++q) xv[t][q] = c[t][q] >= 0 ? xs[c[t][q]] : 0.0;
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            double acc = 0.0;
#pragma unroll
            for (int q = 0; q < kSpmvBatch; ++q)
                if (c[t][q] >= 0) acc = __fma_rn(vs[t][o[t] + 4 * q], xv[t][q], acc);
            for (int kk = o[t] + 4 * kSpmvBatch; kk < o1[t]; kk += 4) acc = __fma_rn(vs[t][kk], xs[cs[t][kk]], acc);
            acc += __shfl_xor_sync(0xffffffffu, acc, 1);
            acc += __shfl_xor_sync(0xffffffffu, acc, 2);
            if (rr[t] < r1 && sub == 0) y[rr[t]] = acc;
        }
        __syncwarp();
        if (lane == 0) {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar0 + 8 * (kSpmvStages + s % kSpmvStages)) : "memory");
            if (s + 1 < n_strips)
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar0 + 8 * (kSpmvStages + (s + 1) % kSpmvStages))
                             : "memory");
        }
    }
}

// y = A x - z (FAST-mode er_begin: C gb_slope - rhs in one pass)
__global__ void __launch_bounds__(kSpmvWarps * 32)
    k_spmv_sub(const int* __restrict__ rowptr, const int* __restrict__ col,
               const double* __restrict__ val, int n_rows, const double* __restrict__ x,
               const double* __restrict__ z, double* __restrict__ y) {
    __shared__ int s_col[kSpmvWarps][kSpmvCap];
    __shared__ double s_val[kSpmvWarps][kSpmvCap];
    const int wg = blockIdx.x * kSpmvWarps + (threadIdx.x >> 5);
    spmv_warp_rows(rowptr, col, val, n_rows, wg, [&](int c) { return x[c]; },
                   [&](int r, double sv) { y[r] = sv - z[r]; }, s_col, s_val);
}
__global__ void __launch_bounds__(kSpmvWarps * 32)
    k_spmv_b2(const int* __restrict__ rowptr, const int* __restrict__ col,
              const double* __restrict__ val, int n_rows, const double* __restrict__ u_k,
              const double* __restrict__ u_k1, double h, double* __restrict__ t1,
              double* __restrict__ t2, const double* __restrict__ Fk) {
    __shared__ int s_col[kSpmvWarps][kSpmvCap];
    __shared__ double s_val[kSpmvWarps][kSpmvCap];
    const int wg = blockIdx.x * kSpmvWarps + (threadIdx.x >> 5);
    spmv_warp_rows(rowptr, col, val, n_rows, wg, [&](int c) { return u_k[c]; },
                   [&](int r, double s) { t1[r] = (Fk ? Fk[r] : 0.0) + 1.0 * s; }, s_col, s_val);
    const double ih = 1.0 / h;
    spmv_warp_rows(rowptr, col, val, n_rows, wg,
                   [&](int c) { return (u_k1[c] + -1.0 * u_k[c]) * ih; },
                   [&](int r, double s) { t2[r] = s; }, s_col, s_val);
}

// ============================================================================
// Sparse triangular solves, sync-free.
//
// Rows are visited in level order (host level analysis at exg_set_factors);
// blocks take consecutive slices of that order through an atomic ticket, so a
// row only ever waits on rows already owned by running (or finished) blocks:
// no deadlock, no per-level launches.  The value itself is the ready flag:
// the output vector is pre-filled with an all-ones NaN sentinel and every row
// publishes its result with one 64-bit relaxed store; dependents poll the
// value with L1-bypassing relaxed loads.
//
// EXACT: every row accumulates in the reference's order (L: increasing
// column; U: increasing column, then divides by the diagonal) —
// bit-identical to Factorization::solve.  FAST: U rows accumulate in
// decreasing column order, so the most recently solved dependency comes last
// and the row's work overlaps its wait (deterministic, not bit-identical).
// ============================================================================
// ---------------------------------------------------------------------------
// v2: warp tasks.  The host cuts the level order into tasks: a LONG row
// (> kLongRow off-diagonal entries) is one warp task; consecutive short rows
// are grouped 32 to a warp task (one row per lane).  Resident warps take
// tasks in order through an atomic ticket (deadlock-free: a task waits only on
// earlier tasks, all owned by running warps).
//   long row, EXACT: the warp loads 32 entries at a time (coalesced), each
//     lane forms its product v*y, and the subtraction chain runs in the
//     reference's order through shuffles -> bit-identical.
//   long row, FAST: each lane accumulates its strided entries (L: increasing,
//     U: decreasing column so the newest dependency comes last), then a fixed
//     butterfly reduction -> deterministic, not bit-identical.
// Dependencies are read with a cached load first; a value never changes once
// published, so a stale copy can only be the sentinel, which falls back to
// polling L2.
// ---------------------------------------------------------------------------
constexpr int kTaskLong = 1 << 30;
__device__ void decide(Ctrl* c);

#ifndef EXG_POLL_NS
#define EXG_POLL_NS 0
#endif
__device__ __forceinline__ double load_ready(const double* p) {
    unsigned long long v = __double_as_longlong(__ldca(p));
    while (v == kSentinel) {
        if (EXG_POLL_NS) __nanosleep(EXG_POLL_NS);
        v = ld_relaxed(p);
    }
    return __longlong_as_double(v);
}

// per-row operands of the epilogue, loaded when the row is taken (pinned so
// the compiler cannot sink them behind the dependency polling)
struct RowOps {
    double b, dg, ad;
    int qq;
};

template <bool UPPER>
__device__ __forceinline__ RowOps row_ops(const TrsvArgs& a, int r) {
    RowOps o;
    o.b = UPPER ? a.in[r] : a.in[a.in_perm[r]];
    o.dg = UPPER ? a.diag[r] : 1.0;
    o.qq = a.final_out ? a.out_perm[r] : 0;
    o.ad = (a.final_out && a.add) ? a.add[o.qq] : 0.0;
    asm volatile("" : "+d"(o.b), "+d"(o.dg), "+r"(o.qq), "+d"(o.ad));
    return o;
}

// Warp-uniform readiness wait for N entries per lane: entries whose cached
// copy is the sentinel are re-read from L2 until every lane of the warp is
// ready; no lane ever spins alone inside a divergent branch.
template <int N>
__device__ __forceinline__ void warp_wait_ready(const double* out, const int* cc, const int* kk,
                                                int k1, double* y, unsigned sleep_ns = 0) {
    bool rd = true;
#pragma unroll
    for (int q = 0; q < N; ++q)
        rd = rd && !(kk[q] < k1 && __double_as_longlong(y[q]) == (long long)kSentinel);
    while (!__all_sync(0xffffffffu, rd)) {
        if (sleep_ns) __nanosleep(sleep_ns);
        rd = true;
#pragma unroll
        for (int q = 0; q < N; ++q) {
            if (kk[q] < k1 && __double_as_longlong(y[q]) == (long long)kSentinel) {
                y[q] = __longlong_as_double(ld_relaxed(out + cc[q]));
                rd = rd && __double_as_longlong(y[q]) != (long long)kSentinel;
            }
        }
    }
}

// warp_wait_ready plus one extra 64-bit value per lane (a chunk partial sum
// of a chain worker's "recent" task) polled in the same rounds, so the
// partials cost no extra round trip once the entries are ready
template <int N>
__device__ __forceinline__ void warp_wait_ready_p(const double* out, const int* cc, const int* kk,
                                                  int k1, double* y, const double* paddr, bool pvalid,
                                                  unsigned long long& pv) {
    bool rd = !(pvalid && pv == kSentinel);
#pragma unroll
    for (int q = 0; q < N; ++q)
        rd = rd && !(kk[q] < k1 && __double_as_longlong(y[q]) == (long long)kSentinel);
    while (!__all_sync(0xffffffffu, rd)) {
        rd = true;
#pragma unroll
        for (int q = 0; q < N; ++q) {
            if (kk[q] < k1 && __double_as_longlong(y[q]) == (long long)kSentinel) {
                y[q] = __longlong_as_double(ld_relaxed(out + cc[q]));
                rd = rd && __double_as_longlong(y[q]) != (long long)kSentinel;
            }
        }
        if (pvalid && pv == kSentinel) {
            pv = ld_relaxed(paddr);
            rd = rd && pv != kSentinel;
        }
    }
}

template <bool UPPER>
__device__ __forceinline__ void trsv_finish(const TrsvArgs& a, int r, double s, const RowOps& o) {
    if (UPPER) s = s / o.dg;
    st_relaxed(a.out + r, s);
    if (a.final_out) {
        double y = a.coef * s;
        if (a.add) y = o.ad + y;
        a.final_out[o.qq] = y;
    }
}

template <bool UPPER, bool FAST>
__global__ void __launch_bounds__(256)
    k_trsv2(TrsvArgs a) {
    __shared__ double s_prod[8][32];
    if (a.ctrl && (a.ctrl->converged || a.ctrl->status)) return;
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    while (true) {
        unsigned int t = 0;
        if (lane == 0) t = atomicAdd(a.ticket, 1u) + 1u;  // ticket starts at 0xFFFFFFFF
        t = __shfl_sync(FULL, t, 0);
        if (t >= (unsigned)a.n_tasks) return;
        const int2 task = a.tasks[t];
        unsigned long long t_start = 0;
        if (a.trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
        if (task.y & kTaskLong) {
            const int r = a.order[task.x];
            const RowOps ops = row_ops<UPPER>(a, r);
            const double b = ops.b;
            const int k0 = a.ptr[r], k1 = a.ptr[r + 1];
            double s = b;
            if (!FAST) {
                // products in parallel, the reference's subtraction chain on lane 0
                double* sp = s_prod[threadIdx.x >> 5];
                for (int base = k0; base < k1; base += 32) {
                    const int k = base + lane;
                    if (k < k1) sp[lane] = a.val[k] * load_ready(a.out + a.col[k]);
                    __syncwarp();
                    if (lane == 0) {
                        const int cnt = min(32, k1 - base);
                        for (int q = 0; q < cnt; ++q) s -= sp[q];
                    }
                    __syncwarp();
                }
            } else {
                double acc = 0.0;
                const int nch = (k1 - k0 + 31) >> 5;
                int ci = 0;
                for (; ci + 4 <= nch; ci += 4) {
                    int kk[4];
                    double v[4], y[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int ch = UPPER ? nch - 1 - (ci + q) : ci + q;  // U: newest last
                        kk[q] = k0 + ch * 32 + lane;
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) v[q] = kk[q] < k1 ? a.val[kk[q]] : 0.0;
#pragma unroll
                    for (int q = 0; q < 4; ++q) y[q] = kk[q] < k1 ? __ldca(a.out + a.col[kk[q]]) : 0.0;
                    int cc[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) cc[q] = kk[q] < k1 ? a.col[kk[q]] : 0;
                    warp_wait_ready<4>(a.out, cc, kk, k1, y);
#pragma unroll
                    for (int q = 0; q < 4; ++q) acc += v[q] * y[q];
                }
                for (; ci < nch; ++ci) {
                    const int ch = UPPER ? nch - 1 - ci : ci;
                    int kk[1] = {k0 + ch * 32 + lane};
                    int cc[1] = {kk[0] < k1 ? a.col[kk[0]] : 0};
                    double y[1] = {kk[0] < k1 ? __ldca(a.out + cc[0]) : 0.0};
                    warp_wait_ready<1>(a.out, cc, kk, k1, y);
                    if (kk[0] < k1) acc += a.val[kk[0]] * y[0];
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
                s = b - acc;
            }
            if (lane == 0) {
                trsv_finish<UPPER>(a, r, s, ops);
                if (a.trace) {
                    unsigned long long t_end;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
                    a.trace[2 * r] = t_start;
                    a.trace[2 * r + 1] = t_end;
                }
            }
        } else {
            const int cnt = task.y & 0xFF;
            const int lg = (task.y >> 8) & 0x7;  // log2 lanes per row
            const int lpr = 1 << lg;
            const int seg = lane >> lg, sl = lane & (lpr - 1);
            const bool active = seg < cnt;
            int r = 0;
            double b = 0.0, acc = 0.0, s = 0.0;
            RowOps ops{0.0, 1.0, 0.0, 0};
            if (active) {
                r = a.order[task.x + seg];
                ops = row_ops<UPPER>(a, r);
                b = ops.b;
                const int k0 = a.ptr[r], k1 = a.ptr[r + 1];
                if (lpr == 1) {
                    // one lane per row, the reference's order (U reversed in FAST)
                    s = b;
                    constexpr int CH = 4;
                    const int len = k1 - k0;
                    int j = 0;
                    for (; j + CH <= len; j += CH) {
                        int kk[CH];
                        double v[CH], y[CH];
#pragma unroll
                        for (int q = 0; q < CH; ++q) kk[q] = (FAST && UPPER) ? k1 - 1 - (j + q) : k0 + j + q;
#pragma unroll
                        for (int q = 0; q < CH; ++q) v[q] = a.val[kk[q]];
#pragma unroll
                        for (int q = 0; q < CH; ++q) y[q] = __ldca(a.out + a.col[kk[q]]);
#pragma unroll
                        for (int q = 0; q < CH; ++q) {
                            if (__double_as_longlong(y[q]) == (long long)kSentinel)
                                y[q] = load_ready(a.out + a.col[kk[q]]);
                            s -= v[q] * y[q];
                        }
                    }
                    for (; j < len; ++j) {
                        const int k = (FAST && UPPER) ? k1 - 1 - j : k0 + j;
                        s -= a.val[k] * load_ready(a.out + a.col[k]);
                    }
                } else {
                    // FAST: lpr lanes per row, strided partial sums
                    const int nj = (k1 - k0 - sl + lpr - 1) >> lg;
                    for (int jj = 0; jj < nj; ++jj) {
                        const int j = UPPER ? nj - 1 - jj : jj;
                        const int k = k0 + sl + (j << lg);
                        acc += a.val[k] * load_ready(a.out + a.col[k]);
                    }
                    (void)0;
                }
            }
            if (lpr > 1) {
                for (int o = lpr >> 1; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
                s = b - acc;
            }
            if (active && sl == 0) {
                trsv_finish<UPPER>(a, r, s, ops);
                if (a.trace) {
                    unsigned long long t_end;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
                    a.trace[2 * r] = t_start;
                    a.trace[2 * r + 1] = t_end;
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// v3 (FAST): wide levels, cooperative persistent grid with STATIC task
// assignment (task t -> warp t mod W; all warps co-resident, each runs its
// tasks in increasing order, a task only waits on smaller tasks: no
// deadlock, no ticket atomics).  Per-position metadata is precomputed in level
// order (meta[p] = {row, b index, k0, k1}), and the next task's metadata is
// loaded while the current task runs, so a task's fixed latency is off the
// critical path.  Every wait is warp-uniform.
// ---------------------------------------------------------------------------
template <bool UPPER>
__global__ void __launch_bounds__(256)
    k_trsv3(TrsvArgs a) {
    if (a.ctrl && (a.ctrl->converged || a.ctrl->status)) return;
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int W = gridDim.x * (blockDim.x >> 5);
    int t = gw;
    if (t >= a.n_tasks) return;
    // metadata of the current task (per lane: its row in a group task)
    // (the diagonal, the output permutation and the add vector of the fused
    // epilogue are prefetched with it: none of them may sit on the hand-off
    // path as a dependent HBM load)
    struct Pre {
        double b, dg, ad;
        int qq;
    };
    auto load_meta = [&](int tt, int2& task, int4& m, Pre& pr) {
        task = a.tasks[tt];
        const bool lng = task.y & kTaskLong;
        const int lg = lng ? 5 : ((task.y >> 8) & 0x7);
        const int seg = lng ? 0 : (lane >> lg);
        const int cnt = lng ? 1 : (task.y & 0xFF);
        pr = Pre{0.0, 1.0, 0.0, 0};
        if (seg < cnt) {
            m = a.meta[task.x + seg];
            // augmented rows (trsv_plan.hpp) may have no right-hand side (-1)
            // and outputs beyond n (block y's, partial sums): no epilogue
            pr.b = m.y >= 0 ? a.in[m.y] : 0.0;
            if (UPPER) pr.dg = a.diag[m.x];
            if (a.final_out && m.x < a.n) {
                pr.qq = a.out_perm[m.x];
                if (a.add) pr.ad = a.add[pr.qq];
            }
        } else {
            m = make_int4(0, 0, 0, 0);
        }
    };
    // first batch (4 entries per lane) of a task: the same index pattern as
    // the processing loops below (U: newest dependencies last)
    auto batch0 = [&](const int2& task, const int4& mm, int* cc, double* v) {
        const bool lng = task.y & kTaskLong;
        const int k0 = mm.z, k1 = mm.w;
        int kk[4];
        if (lng) {
            const int nch = (k1 - k0 + 31) >> 5;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int ch = UPPER ? nch - 1 - q : q;
                kk[q] = q < nch ? k0 + ch * 32 + lane : k1;
            }
        } else {
            const int cnt = task.y & 0xFF;
            const int lg = (task.y >> 8) & 0x7;
            const int lpr = 1 << lg;
            const int seg = lane >> lg, sl = lane & (lpr - 1);
            const int nj = seg < cnt ? (k1 - k0 - sl + lpr - 1) >> lg : 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int j = UPPER ? nj - 1 - q : q;
                kk[q] = q < nj ? k0 + sl + (j << lg) : k1;
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            cc[q] = kk[q] < k1 ? a.col[kk[q]] : -1;
            v[q] = kk[q] < k1 ? a.val[kk[q]] : 0.0;
        }
    };
    // Two-deep software pipeline: while task i runs, the entries of task
    // i+1 (whose metadata arrived during task i-1) and the metadata of task
    // i+2 are in flight, so a task's own loads are never on the hand-off path.
    int2 task, task1, task2;
    int4 m, m1, m2;
    Pre pr, pr1, pr2;
    int cc0[4], cc1[4];
    double v0[4], v1[4];
    load_meta(t, task, m, pr);
    const bool has1 = t + W < a.n_tasks;
    if (has1) load_meta(t + W, task1, m1, pr1);
    batch0(task, m, cc0, v0);
    while (true) {
        const int tn = t + W, tnn = t + 2 * W;
        if (tnn < a.n_tasks) load_meta(tnn, task2, m2, pr2);
        if (tn < a.n_tasks) batch0(task1, m1, cc1, v1);
        const bool lng = task.y & kTaskLong;
        const int r = m.x, k0 = m.z, k1 = m.w;
        double acc = 0.0;
        {  // batch 0 from the prefetched entries
            int kk[4];
            double y[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                kk[q] = cc0[q] >= 0 ? k0 : k1;  // validity marker for warp_wait_ready
                y[q] = cc0[q] >= 0 ? __ldca(a.out + cc0[q]) : 0.0;
            }
            warp_wait_ready<4>(a.out, cc0, kk, k1, y);
#pragma unroll
            for (int q = 0; q < 4; ++q) acc = __fma_rn(v0[q], y[q], acc);
        }
        if (lng) {
            const int nch = (k1 - k0 + 31) >> 5;
            for (int ci = 4; ci < nch; ci += 4) {
                int kk[4], cc[4];
                double v[4], y[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int ch = UPPER ? nch - 1 - (ci + q) : ci + q;  // U: newest last
                    kk[q] = (ci + q < nch) ? k0 + ch * 32 + lane : k1;
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    cc[q] = kk[q] < k1 ? a.col[kk[q]] : 0;
                    v[q] = kk[q] < k1 ? a.val[kk[q]] : 0.0;
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) y[q] = kk[q] < k1 ? __ldca(a.out + cc[q]) : 0.0;
                warp_wait_ready<4>(a.out, cc, kk, k1, y);
#pragma unroll
                for (int q = 0; q < 4; ++q) acc = __fma_rn(v[q], y[q], acc);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
            if (lane == 0) {
                double s = pr.b - acc;
                if (UPPER) s = s / pr.dg;
                st_relaxed(a.out + r, s);
                if (a.final_out && r < a.n) {
                    double yv = a.coef * s;
                    if (a.add) yv = pr.ad + yv;
                    a.final_out[pr.qq] = yv;
                }
            }
        } else {
            const int cnt = task.y & 0xFF;
            const int lg = (task.y >> 8) & 0x7;
            const int lpr = 1 << lg;
            const int seg = lane >> lg, sl = lane & (lpr - 1);
            const bool active = seg < cnt;
            const int nj = active ? (k1 - k0 - sl + lpr - 1) >> lg : 0;
            const int njmax = __reduce_max_sync(FULL, nj);
            for (int j0 = 4; j0 < njmax; j0 += 4) {
                int kk[4], cc[4];
                double v[4], y[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int jj = j0 + q;
                    const int j = UPPER ? nj - 1 - jj : jj;  // U: newest last
                    kk[q] = jj < nj ? k0 + sl + (j << lg) : k1;
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    cc[q] = kk[q] < k1 ? a.col[kk[q]] : 0;
                    v[q] = kk[q] < k1 ? a.val[kk[q]] : 0.0;
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) y[q] = kk[q] < k1 ? __ldca(a.out + cc[q]) : 0.0;
                warp_wait_ready<4>(a.out, cc, kk, k1, y);
#pragma unroll
                for (int q = 0; q < 4; ++q) acc = __fma_rn(v[q], y[q], acc);
            }
            for (int o = lpr >> 1; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
            if (active && sl == 0) {
                double s = pr.b - acc;
                if (UPPER) s = s / pr.dg;
                st_relaxed(a.out + r, s);
                if (a.final_out && r < a.n) {
                    double yv = a.coef * s;
                    if (a.add) yv = pr.ad + yv;
                    a.final_out[pr.qq] = yv;
                }
            }
        }
        if (tn >= a.n_tasks) return;
        t = tn;
        task = task1;
        m = m1;
        pr = pr1;
        task1 = task2;
        m1 = m2;
        pr1 = pr2;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            cc0[q] = cc1[q];
            v0[q] = v1[q];
        }
    }
}

// ---------------------------------------------------------------------------
// Subtree phase (FAST): the bottom of the elimination DAG as independent
// components, one CTA each, hand-offs in SHARED memory.
//
// The host picks a set S of rows closed under the triangle's dependencies
// (L: every dependency of a row in S is in S; U: every row that depends on a
// row of S is in S) and cuts it into weakly connected components of at most
// EXG_SUB_ROWS rows (union-find, plan_subtrees in api.cu).  No row of one
// component depends on another component, so each runs on one CTA with no
// grid-wide hand-off at all: a solved value is published into the CTA's
// shared-memory slot (pre-filled with the all-ones sentinel) and dependents
// poll it there (~tens of ns) instead of through L2 (~0.45 µs per level at
// 1M).  In L the phase runs first (leaves of the elimination tree); in U it
// runs last, its rows reading the separators solved by the earlier runs from
// global memory (final, no poll).  Warp tasks as in k_trsv3 (rows grouped
// within one local level, never across), warp w of the CTA takes tasks
// w, w+8, ... of its component in level order: a task waits only on earlier
// tasks, so the earliest unfinished task always progresses.  Each row's
// entries are re-encoded: earlier-phase dependencies first (global row id),
// then component slots in increasing order (~slot), so the newest
// dependency is met last; the next task's metadata and first entries are in
// flight while the current one waits.
// ---------------------------------------------------------------------------
template <bool UPPER>
__global__ void __launch_bounds__(256)
    k_trsv_sub(SubArgs a) {
    if (a.ctrl && (a.ctrl->converged || a.ctrl->status)) return;
    // shared memory: [slots: max_rows x 8 B][meta: max_rows x 16 B][tasks: max_tasks x 8 B]
    //                [level task offsets: max_levels + 1]
    extern __shared__ __align__(16) double xs[];
    int4* smeta = reinterpret_cast<int4*>(xs + a.max_rows);
    int2* stask = reinterpret_cast<int2*>(smeta + a.max_rows);
    int* sltp = reinterpret_cast<int*>(stask + a.max_tasks);
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    struct Pre {
        int2 task;
        int4 m;
        double b, dg, ad;
        int qq;
        int cc[4];
        double v[4];
    };
    // a task's metadata from shared memory; its operands and first entries
    // from global memory (independent of the solution: issued before the
    // level barrier that precedes the task)
    auto fetch = [&](int tl, int p0, Pre& p) {
        p.task = stask[tl];
        const bool lng = p.task.y & kTaskLong;
        const int lg = lng ? 5 : ((p.task.y >> 8) & 0x7);
        const int seg = lng ? 0 : (lane >> lg);
        const int cnt = lng ? 1 : (p.task.y & 0xFF);
        const int lpr = 1 << lg, sl = lane & (lpr - 1);
        p.b = 0.0;
        p.dg = 1.0;
        p.ad = 0.0;
        p.qq = 0;
        if (seg < cnt) {
            p.m = smeta[p.task.x - p0 + seg];
            p.b = a.in[p.m.y];
            if (UPPER) p.dg = a.diag[p.m.x];
            if (a.final_out) {
                p.qq = a.out_perm[p.m.x];
                if (a.add) p.ad = a.add[p.qq];
            }
        } else {
            p.m = make_int4(0, 0, 0, 0);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int k = p.m.z + sl + q * lpr;
            p.cc[q] = k < p.m.w ? a.ecol[k] : INT_MIN;
            p.v[q] = k < p.m.w ? a.eval[k] : 0.0;
        }
    };
    auto xget = [&](int c) { return c == INT_MIN ? 0.0 : c >= 0 ? __ldcg(a.out + c) : xs[~c]; };
    for (int ci = blockIdx.x; ci < a.n_comps; ci += gridDim.x) {
        const int4 cr = a.comps[ci];   // (first task, tasks, first position, rows)
        const int2 cl = a.clev[ci];    // (first level offset, levels)
        for (int i = threadIdx.x; i < cr.w; i += blockDim.x) smeta[i] = a.meta[cr.z + i];
        for (int i = threadIdx.x; i < cr.y; i += blockDim.x) stask[i] = a.tasks[cr.x + i];
        for (int i = threadIdx.x; i <= cl.y; i += blockDim.x) sltp[i] = a.ltp[cl.x + i] - cr.x;
        __syncthreads();
        Pre cur;
        int t = sltp[0] + warp;
        if (t < sltp[1]) fetch(t, cr.z, cur);
        for (int lv = 0; lv < cl.y; ++lv) {
            const int tend = sltp[lv + 1];
            while (t < tend) {
                const bool lng = cur.task.y & kTaskLong;
                const int lg = lng ? 5 : ((cur.task.y >> 8) & 0x7);
                const int lpr = 1 << lg, sl = lane & (lpr - 1);
                const int seg = lng ? 0 : (lane >> lg);
                const int cnt = lng ? 1 : (cur.task.y & 0xFF);
                const bool active = seg < cnt;
                double acc = 0.0;
#pragma unroll
                for (int q = 0; q < 4; ++q) acc = __fma_rn(cur.v[q], xget(cur.cc[q]), acc);
                for (int k0 = cur.m.z + sl + 4 * lpr; k0 < cur.m.w; k0 += 4 * lpr) {
                    int cc[4];
                    double v[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int k = k0 + q * lpr;
                        cc[q] = k < cur.m.w ? a.ecol[k] : INT_MIN;
                        v[q] = k < cur.m.w ? a.eval[k] : 0.0;
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) acc = __fma_rn(v[q], xget(cc[q]), acc);
                }
                for (int o = lpr >> 1; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
                if (active && sl == 0) {
                    double sv = cur.b - acc;
                    if (UPPER) sv = sv / cur.dg;
                    xs[cur.task.x - cr.z + seg] = sv;
                    a.out[cur.m.x] = sv;
                    if (a.final_out) {
                        double yv = a.coef * sv;
                        if (a.add) yv = cur.ad + yv;
                        a.final_out[cur.qq] = yv;
                    }
                }
                t += nw;
                if (t < tend) fetch(t, cr.z, cur);
            }
            // this warp's first task of the next level: its loads are in
            // flight across the barrier
            if (lv + 1 < cl.y) {
                t = tend + warp;
                if (t < sltp[lv + 2]) fetch(t, cr.z, cur);
            }
            __syncthreads();
        }
    }
}

// Chain geometry (k_trsv_chain): 64-row blocks, kNP CTA pairs.
constexpr int kBlk = 64;
constexpr int kChainStages = 2;  // TMA stages per chain CTA (its pair's next block is in flight)
constexpr int kChainMatsPerBlock = 5;  // Dinv, F1..F4 (the chain handles blocks k-1..k-4)
#ifndef EXG_CHAIN_PAIRS
#define EXG_CHAIN_PAIRS 3
#endif
constexpr int kNP = EXG_CHAIN_PAIRS;     // CTA pairs of the chain cluster (blocks k == p mod kNP)
constexpr int kCC = 2 * kNP;             // chain CTAs
static_assert(kNP >= 2 && kNP <= 3, "x barrier ring of 4 assumes 2 <= pairs <= 3");
constexpr int kChainThreads = 288;  // chain CTAs: 8 compute warps + 1 producer warp; workers use all 9
constexpr size_t kChainMats = kChainStages * kChainMatsPerBlock * (kBlk * kBlk / 2) * sizeof(double);  // half of (Dinv, F1..F4) per stage
// launched with more than half an SM's shared memory so that no worker CTA
// shares an SM with a chain CTA (one CTA per SM)
constexpr size_t kChainSmem = kChainMats > 120 * 1024 ? kChainMats : 120 * 1024;  // > half an SM: one CTA per SM
static_assert(kChainSmem >= kChainMats, "chain smem");

// ---------------------------------------------------------------------------
// Chain + workers (FAST, narrow runs): one cooperative launch over the whole
// GPU.  The run's level-order positions are cut into blocks of 64; with
//     x_k = Dinv_k s_k - F1_k x_{k-1} - F2_k x_{k-2},   F_g = Dinv_k E_g,
// CTA 0 (the chain) evaluates the recurrence block after block entirely in
// its own shared memory (no hand-off between consecutive blocks), streaming
// Dinv/F1/F2 with cp.async double buffering; every other warp of the GPU
// computes s_k = b - (entries older than block k-2) for the rows (sync-free
// warp tasks polling the published solution in global memory; s is
// published the same way, sentinel-initialised).  Workers lag the chain by
// two blocks, which hides their L2 hand-off latency.
// ---------------------------------------------------------------------------

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

#ifndef EXG_CHAIN_MINB
#define EXG_CHAIN_MINB 1
#endif
template <bool UPPER>
__global__ void __launch_bounds__(kChainThreads, EXG_CHAIN_MINB)
    k_trsv_chain(ChainArgs a) {
    if (a.ctrl && (a.ctrl->converged || a.ctrl->status)) return;
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (blockIdx.x < kCC) {
        // ===================== chain: kNP pairs =====================
        // The chain is a 4-CTA thread-block cluster on four SMs: pair p
        // (CTAs 2p, 2p+1) takes the blocks k == p (mod 2), and CTA h of a pair
        // owns rows 32h..32h+31 of each of them, so the per-block work that
        // does not depend on x_{k-1} (F3 x_{k-3}, F2 x_{k-2}, Dinv s) of one
        // pair overlaps the loop-carried F1 x_{k-1} + publication of the
        // other.  Per CTA, warp-specialised:
        // * warp 8 (producer) walks its pair's blocks up to kChainStages
        //   ahead: TMA bulk copy of its half of the block record
        //   (Dinv F1 F2 F3, thread-major layout: thread t owns local row t/8,
        //   columns (t%8)*8..+7), the block's s values published by the
        //   workers (polled one block ahead), row ids; FULL barriers;
        // * warps 0-7 (compute): Dinv s - F3 x_{k-3} - F2 x_{k-2} - F1 x_{k-1}
        //   with fused multiply-adds and one 3-step reduction; x_k's half is
        //   pushed into the other three CTAs' rings with st.async completing
        //   on their x barriers (block j lands on barrier j % 4).
        constexpr int kXs = 72;   // padded x slot: column c at c + c/8
        constexpr int kHalf = kBlk * kBlk / 2;
        constexpr int kS = kChainStages;
        constexpr int kNM = kChainMatsPerBlock;
        constexpr int kR = kNM;  // x ring slots: blocks k-4..k
        constexpr unsigned kMatBytes = (unsigned)kNM * kHalf * sizeof(double);
        extern __shared__ __align__(128) double smat[];  // [kS stages][4][kHalf]
        __shared__ double xr[kR * kXs];                  // x of the last 5 blocks (both halves), slot k % 5
        __shared__ double sst[kS][kXs];                  // staged s (padded layout)
        __shared__ int2 rqst[kS][32];                    // staged (row id, output position) of own rows
        __shared__ int4 mst[kS][2];                      // staged block descriptor (B, O)
        __shared__ __align__(8) unsigned long long full_b[kS], sful_b[kS], empty_b[kS], xbar[4];
        const int cr = blockIdx.x;       // rank in the cluster
        const int pr = cr >> 1, hf = cr & 1;
        const int tid = threadIdx.x;
        const unsigned fb0 = (unsigned)__cvta_generic_to_shared(&full_b[0]);  // matrices + descriptor
        const unsigned sb0 = (unsigned)__cvta_generic_to_shared(&sful_b[0]);  // s + row ids
        const unsigned eb0 = (unsigned)__cvta_generic_to_shared(&empty_b[0]);
        const unsigned xb0 = (unsigned)__cvta_generic_to_shared(&xbar[0]);
        if (tid == 0) {
            for (int q = 0; q < kS; ++q) {
                asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(fb0 + 8 * q));
                asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(sb0 + 8 * q));
                asm volatile("mbarrier.init.shared.b64 [%0], 8;" ::"r"(eb0 + 8 * q));
            }
            for (int q = 0; q < 4; ++q) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(xb0 + 8 * q));
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        for (int i = tid; i < kR * kXs; i += blockDim.x) xr[i] = 0.0;
        unsigned xr_rem[kCC - 1], xb_rem[kCC - 1];  // the other CTAs' rings and x barriers (DSMEM)
        {
            const unsigned xl = (unsigned)__cvta_generic_to_shared(xr);
#pragma unroll
            for (int q = 0; q < kCC - 1; ++q) {
                const int other = (cr + 1 + q) % kCC;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(xr_rem[q]) : "r"(xl), "r"(other));
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(xb_rem[q]) : "r"(xb0), "r"(other));
            }
        }
        const int nbk = a.n_blocks;
        // bytes block j brings to this CTA: the mate's half (own pair) or
        // both halves (other pair)
        auto xbytes = [&](int j) { return j % kNP == pr ? 32u * 8u : 64u * 8u; };
        auto expect_x = [&](int j) {
            asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(xb0 + 8 * (j & 3)),
                         "r"(xbytes(j)) : "memory");
        };
        auto wait_x = [&](int j) {
            const unsigned mb = xb0 + 8 * (j & 3);
            const unsigned par = (unsigned)((j >> 2) & 1);
            unsigned done = 0;
            while (!done) {
                asm volatile(
                    "{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                    : "=r"(done) : "r"(mb), "r"(par) : "memory");
            }
        };
        if (tid == 0)
            for (int j = 0; j < 4 && j < nbk; ++j) expect_x(j);
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
        auto mb_wait = [](unsigned mb, unsigned par) {
            unsigned done = 0;
            while (!done) {
                asm volatile(
                    "{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                    : "=r"(done) : "r"(mb), "r"(par) : "memory");
            }
        };
        const int nmine = nbk > pr ? (nbk - pr + kNP - 1) / kNP : 0;  // blocks of this pair
        if (warp == 8) {
            // ---------------- producer ----------------
            unsigned long long pol;
            asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
            auto blk = [&](int u) { return pr + kNP * u; };
            int4 B0 = make_int4(0, 0, 0, 0), O0 = make_int4(-1, -1, -1, 0);
            int4 B1 = B0, O1 = O0;
            if (nmine > 0) {
                B0 = a.blocks[3 * blk(0)];
                O0 = a.blocks[3 * blk(0) + 1];
            }
            if (nmine > 1) {
                B1 = a.blocks[3 * blk(1)];
                O1 = a.blocks[3 * blk(1) + 1];
            }
            int2 rq0 = (nmine > 0 && 32 * hf + lane < B0.y) ? a.rq[B0.x + 32 * hf + lane] : make_int2(0, 0);
            double sn0 = (nmine > 0 && lane < B0.y) ? __longlong_as_double(ld_relaxed(a.s + B0.x + lane)) : 0.0;
            double sn1 = (nmine > 0 && lane + 32 < B0.y) ? __longlong_as_double(ld_relaxed(a.s + B0.x + lane + 32)) : 0.0;
            for (int u = 0; u < nmine; ++u) {
                const int st = u % kS;
                if (u >= kS) mb_wait(eb0 + 8 * st, (unsigned)(((u / kS) - 1) & 1));
                if (lane == 0) {
                    const unsigned dst = (unsigned)__cvta_generic_to_shared(smat + st * kNM * kHalf);
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(dst),
                        "l"(a.pool + O0.w + hf * kNM * kHalf), "r"(kMatBytes), "r"(fb0 + 8 * st), "l"(pol)
                        : "memory");
                    mst[st][0] = B0;
                    mst[st][1] = O0;
                    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(fb0 + 8 * st),
                                 "r"(kMatBytes) : "memory");
                }
                const int4 B2 = u + 2 < nmine ? a.blocks[3 * blk(u + 2)] : make_int4(0, 0, 0, 0);
                const int4 O2 = u + 2 < nmine ? a.blocks[3 * blk(u + 2) + 1] : make_int4(-1, -1, -1, 0);
                const int2 rq1 = (u + 1 < nmine && 32 * hf + lane < B1.y) ? a.rq[B1.x + 32 * hf + lane]
                                                                          : make_int2(0, 0);
                const int nb = B0.y;
                const double* sp = a.s + B0.x;
                double s0 = sn0, s1 = sn1;
                if (u + 1 < nmine) {
                    sn0 = lane < B1.y ? __longlong_as_double(ld_relaxed(a.s + B1.x + lane)) : 0.0;
                    sn1 = lane + 32 < B1.y ? __longlong_as_double(ld_relaxed(a.s + B1.x + lane + 32)) : 0.0;
                }
                bool rd = __double_as_longlong(s0) != (long long)kSentinel &&
                          __double_as_longlong(s1) != (long long)kSentinel;
                while (!__all_sync(FULL, rd)) {
                    if (lane < nb && __double_as_longlong(s0) == (long long)kSentinel)
                        s0 = __longlong_as_double(ld_relaxed(sp + lane));
                    if (lane + 32 < nb && __double_as_longlong(s1) == (long long)kSentinel)
                        s1 = __longlong_as_double(ld_relaxed(sp + lane + 32));
                    rd = __double_as_longlong(s0) != (long long)kSentinel &&
                         __double_as_longlong(s1) != (long long)kSentinel;
                }
                sst[st][lane + (lane >> 3)] = s0;
                sst[st][lane + 32 + ((lane + 32) >> 3)] = s1;
                rqst[st][lane] = rq0;
                __syncwarp();
                if (lane == 0) asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(sb0 + 8 * st) : "memory");
                B0 = B1;
                O0 = O1;
                B1 = B2;
                O1 = O2;
                rq0 = rq1;
            }
            asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
            asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
            return;
        }
        // ---------------- compute warps 0-7 ----------------
        const int rl = tid >> 3, oc = tid & 7;
        const int row = 32 * hf + rl;  // row of the block owned by this thread group
        for (int u = 0; u < nmine; ++u) {
            const int kb = pr + kNP * u;
            const int st = u % kS;
            mb_wait(fb0 + 8 * st, (unsigned)((u / kS) & 1));
            const int4 Bc = mst[st][0], Oc = mst[st][1];
            const int nb = Bc.y;
            const double* Ms = smat + st * kNM * kHalf;
            double q = 0.0;
            // x_{k-4} was waited for at an earlier block (kNP <= 3)
            // independent accumulators per matrix and per half of the slice:
            // a dependent FP64 FMA chain is the latency that matters here
            double qa = 0.0, qb = 0.0, qc = 0.0, qd = 0.0, qe = 0.0, qf = 0.0;
            if (Bc.w >= 0) {
                const double* xg = xr + ((kb + 1) % kR) * kXs + oc * 9;  // slot of block k-4
                const double* M = Ms + 4 * kHalf + tid;
#pragma unroll
                for (int j = 0; j < 8; j += 2) {
                    qa = __fma_rn(-M[j * 256], xg[j], qa);
                    qb = __fma_rn(-M[(j + 1) * 256], xg[j + 1], qb);
                }
            }
            // blocks k-kNP .. k-2 (own pair's previous block: the mate's half;
            // the others: both halves), each waited once and its barrier
            // re-armed for block j+4 (cannot be produced before our x_k)
            for (int j = kb - kNP; j <= kb - 2; ++j) {
                if (j < 0) continue;
                wait_x(j);
                if (tid == 0 && j + 4 < nbk) expect_x(j + 4);
            }
            if (Bc.z >= 0) {
                const double* xg = xr + ((kb + 2) % kR) * kXs + oc * 9;  // slot of block k-3
                const double* M = Ms + 3 * kHalf + tid;
#pragma unroll
                for (int j = 0; j < 8; j += 2) {
                    qc = __fma_rn(-M[j * 256], xg[j], qc);
                    qd = __fma_rn(-M[(j + 1) * 256], xg[j + 1], qd);
                }
            }
            if (Oc.z >= 0) {
                const double* xg = xr + ((kb + 3) % kR) * kXs + oc * 9;  // slot of block k-2
                const double* M = Ms + 2 * kHalf + tid;
#pragma unroll
                for (int j = 0; j < 8; j += 2) {
                    qe = __fma_rn(-M[j * 256], xg[j], qe);
                    qf = __fma_rn(-M[(j + 1) * 256], xg[j + 1], qf);
                }
            }
            mb_wait(sb0 + 8 * st, (unsigned)((u / kS) & 1));
            unsigned long long t_w = 0;
            if (a.trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_w));
            const double ad = (oc == 0 && row < nb && a.final_out && a.add) ? a.add[rqst[st][rl].y] : 0.0;
            double sa = 0.0, sb = 0.0;
            if (Oc.x >= 0) {
                const double* M = Ms + tid;
                const double* sg = sst[st] + oc * 9;
#pragma unroll
                for (int j = 0; j < 8; j += 2) {
                    sa = __fma_rn(M[j * 256], sg[j], sa);
                    sb = __fma_rn(M[(j + 1) * 256], sg[j + 1], sb);
                }
            } else if (oc == (row >> 3) && row < nb) {
                sa = sst[st][row + (row >> 3)];  // identity Dinv: s_row
            }
            q = ((sa + sb) + ((qa + qb) + (qc + qd))) + (qe + qf);
            unsigned long long t_m = 0;
            if (a.trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_m));
            // x_{k-1}: both halves from the other pair; re-arm for k+3
            if (kb >= 1) {
                wait_x(kb - 1);
                if (tid == 0 && kb + 3 < nbk) expect_x(kb + 3);
            }
            unsigned long long t_s = 0;
            if (a.trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_s));
            if (Oc.y >= 0) {
                const double* xg = xr + ((kb + 4) % kR) * kXs + oc * 9;  // slot of block k-1
                const double* M = Ms + kHalf + tid;
                double pa = 0.0, pb = 0.0;
#pragma unroll
                for (int j = 0; j < 8; j += 2) {
                    pa = __fma_rn(-M[j * 256], xg[j], pa);
                    pb = __fma_rn(-M[(j + 1) * 256], xg[j + 1], pb);
                }
                q = q + (pa + pb);
            }
            q += __shfl_xor_sync(FULL, q, 1);
            q += __shfl_xor_sync(FULL, q, 2);
            q += __shfl_xor_sync(FULL, q, 4);
            const double cx = q;
            // publish x_k: own ring, the other three rings, global, epilogue
            if (oc == 0) {
                const double xv = row < nb ? cx : 0.0;
                const int xi = (kb % kR) * kXs + row + (row >> 3);
                xr[xi] = xv;
#pragma unroll
                for (int r2 = 0; r2 < kCC - 1; ++r2)
                    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(
                                     xr_rem[r2] + 8u * (unsigned)xi),
                                 "l"(__double_as_longlong(xv)), "r"(xb_rem[r2] + 8u * (unsigned)(kb & 3))
                                 : "memory");
                if (row < nb) {
                    const int2 rq = rqst[st][rl];
                    st_relaxed(a.out + rq.x, cx);
                    if (a.final_out) {
                        double yo = a.coef * cx;
                        if (a.add) yo = ad + yo;
                        a.final_out[rq.y] = yo;
                    }
                }
            }
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(eb0 + 8 * st) : "memory");
            asm volatile("bar.sync 1, 256;" ::: "memory");  // own half of x_k for this pair's next block
            if (a.trace && tid == 0 && hf == 0) {
                unsigned long long t_e;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_e));
                a.trace[4 * kb] = t_w;
                a.trace[4 * kb + 1] = t_m;
                a.trace[4 * kb + 2] = t_s;
                a.trace[4 * kb + 3] = t_e;
            }
        }
        // x blocks that arrive but are never consumed (the last ones) must
        // land before the CTA exits
        {
            const int last = nmine > 0 ? pr + kNP * (nmine - 1) : -1;  // this pair's last block
            // waited so far: blocks < last (each at the pair's next block);
            // our own last block's mate half and everything after it were not
            for (int j = last > 0 ? last : 0; j < nbk; ++j) wait_x(j);
        }
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
        return;
    }
    // ===================== workers =====================
    // tasks in order of the block their newest dependency belongs to:
    //   chunk: part[slot] = sum of <= 256 entries older than block k-8
    //   recent: s[p] = b - (sum of the row's chunk partials, in order,
    //           + entries of blocks k-8..k-3)
    // Software-pipelined: the next task's descriptor, its first 256 entries
    // and (recent tasks) right-hand side and chunk partials are loaded while
    // the current task waits, so a task costs one L2 round trip, not three
    // dependent HBM loads.
    const int gw = (blockIdx.x - kCC) * (blockDim.x >> 5) + warp;
    const int W = (gridDim.x - kCC) * (blockDim.x >> 5);
    struct Stage {
        int4 T;
        int cc[8];
        double v[8];
        double b;
        int slot0;
        unsigned long long pv;
    };
    auto load_stage = [&](int t, Stage& S) {
        S.T = a.wtasks[t];
        const int k0 = S.T.y, k1 = S.T.z;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int k = k0 + lane + 32 * q;
            S.cc[q] = k < k1 ? a.ncol[k] : -1;
            S.v[q] = k < k1 ? a.nval[k] : 0.0;
        }
        S.b = 0.0;
        S.slot0 = 0;
        S.pv = 0ull;
        if (S.T.w & 1) {
            if (lane == 0) {
                const int r = a.rows[S.T.x];
                S.b = UPPER ? a.in[r] : a.in[a.in_perm[r]];
            }
            S.slot0 = a.pslot[S.T.x];
            if (lane < (S.T.w >> 8)) S.pv = ld_relaxed(a.part + S.slot0 + lane);
        }
    };
    int t = gw;
    if (t >= a.n_tasks) return;
    Stage cur, nxt;
    load_stage(t, cur);
    while (true) {
        const int tn = t + W;
        if (tn < a.n_tasks) load_stage(tn, nxt);
        const int p = cur.T.x, k0 = cur.T.y, k1 = cur.T.z;
        const bool recent = cur.T.w & 1;
        const int nch = cur.T.w >> 8;
        unsigned long long tr0 = 0, tr1 = 0;
        if (a.trace && recent) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr0));
        double acc = 0.0;
        unsigned long long pv = cur.pv;
        {
            int kk[8];
            double y[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                kk[q] = cur.cc[q] >= 0 ? k0 : k1;  // "valid" marker for warp_wait_ready
                y[q] = cur.cc[q] >= 0 ? __ldca(a.out + cur.cc[q]) : 0.0;
            }
            // a recent task's first 32 chunk partials are polled together
            // with its entries
            const bool pvalid = recent && lane < nch;
            if (pvalid && pv == kSentinel) pv = ld_relaxed(a.part + cur.slot0 + lane);
            warp_wait_ready_p<8>(a.out, cur.cc, kk, k1, y, a.part + cur.slot0 + lane, pvalid, pv);
#pragma unroll
            for (int q = 0; q < 8; ++q) acc = __fma_rn(cur.v[q], y[q], acc);
        }
        for (int base = k0 + 256; base < k1; base += 256) {  // long recent tasks only
            int kk[8], cc[8];
            double v[8], y[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                kk[q] = base + lane + 32 * q;
                cc[q] = kk[q] < k1 ? a.ncol[kk[q]] : 0;
                v[q] = kk[q] < k1 ? a.nval[kk[q]] : 0.0;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) y[q] = kk[q] < k1 ? __ldca(a.out + cc[q]) : 0.0;
            warp_wait_ready<8>(a.out, cc, kk, k1, y);
#pragma unroll
            for (int q = 0; q < 8; ++q) acc = __fma_rn(v[q], y[q], acc);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
        if (a.trace && recent) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr1));
        if (!recent) {
            if (lane == 0) st_relaxed(a.part + p, acc);
        } else {
            // chunk partials, summed in chunk order (deterministic)
            double old = 0.0;
            for (int c0 = 0; c0 < nch; c0 += 32) {
                const int ci = c0 + lane;
                if (c0 > 0) pv = ci < nch ? ld_relaxed(a.part + cur.slot0 + ci) : 0ull;
                while (!__all_sync(FULL, ci >= nch || pv != kSentinel))
                    if (ci < nch && pv == kSentinel) pv = ld_relaxed(a.part + cur.slot0 + ci);
                double g = ci < nch ? __longlong_as_double(pv) : 0.0;  // fixed butterfly: deterministic
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) g += __shfl_xor_sync(FULL, g, o);
                old += g;
            }
            if (lane == 0) st_relaxed(a.s + p, cur.b - (old + acc));
            if (a.trace && lane == 0) {
                unsigned long long tr2;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr2));
                unsigned long long* wt = a.trace + 4 * a.n_blocks + 3 * (long long)p;
                wt[0] = tr0;
                wt[1] = tr1;
                wt[2] = tr2;
            }
        }
        if (tn >= a.n_tasks) return;
        t = tn;
        cur = nxt;
    }
}

// ---------------------------------------------------------------------------
// row-sequential warp SpMV helper for rows of very different lengths
// (factor apply): long rows cooperatively with the in-order chain through
// shuffles, short rows one per lane.  Bit-identical to spmv.
// ---------------------------------------------------------------------------
template <typename XFn>
__device__ __forceinline__ double warp_row_dot_exact(int k0, int k1, const int* __restrict__ col,
                                                     const double* __restrict__ val, XFn xfn,
                                                     double s, double* sp) {
    const int lane = threadIdx.x & 31;
    for (int base = k0; base < k1; base += 32) {
        const int k = base + lane;
        if (k < k1) sp[lane] = val[k] * xfn(col[k]);
        __syncwarp();
        if (lane == 0) {
            const int cnt = min(32, k1 - base);
            for (int q = 0; q < cnt; ++q) s += sp[q];
        }
        __syncwarp();
    }
    return __shfl_sync(0xffffffffu, s, 0);
}


// ---------------------------------------------------------------------------
// Factor apply over the EXACT warp-task lists (no dependencies: any order).
// Long rows get a whole warp (products in parallel, the reference's in-order
// accumulation on lane 0), short rows one lane each.  Bit-identical to
// spmv(U, .) / spmv(L, .) of Factorization::apply (sparse_lu.cpp:299-300).
//   UPPER: t[r] = 0 + diag*x[cp[r]] + sum_{c>r} U_rc x[cp[c]]   (diag first)
//   LOWER: y[r] = sum_{c<r} L_rc t[c] + 1.0*t[r]; sq[r] = y^2  (diag last)
// ---------------------------------------------------------------------------
template <bool UPPER>
__global__ void __launch_bounds__(256)
    k_apply_tasks(const int2* __restrict__ tasks, int n_tasks, const int* __restrict__ order,
                  const int* __restrict__ ptr, const int* __restrict__ col,
                  const double* __restrict__ val, const double* __restrict__ diag,
                  const int* __restrict__ col_perm, const double* __restrict__ x,
                  double* __restrict__ out, double* __restrict__ sq, const int* __restrict__ row_perm,
                  double* __restrict__ y_out, const Ctrl* ctrl, const double* __restrict__ vbase,
                  long long ldv) {
    __shared__ double s_prod[8][32];
    const double* xs = x;
    if (ctrl) {
        if (!ctrl->need_weight || ctrl->converged || ctrl->status) return;
        if (UPPER) xs = vbase + (long long)ctrl->m * ldv;
    }
    const int lane = threadIdx.x & 31;
    const int wglobal = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int nw = gridDim.x * (blockDim.x >> 5);
    auto xv = [&](int c) { return UPPER ? xs[col_perm[c]] : xs[c]; };
    for (int t = wglobal; t < n_tasks; t += nw) {
        const int2 task = tasks[t];
        if (task.y & kTaskLong) {
            const int r = order[task.x];
            double s = 0.0;
            if (UPPER) s += diag[r] * xv(r);
            s = warp_row_dot_exact(ptr[r], ptr[r + 1], col, val, xv, s, s_prod[threadIdx.x >> 5]);
            if (!UPPER) s += 1.0 * xs[r];
            if (lane == 0) {
                out[r] = s;
                if (sq) sq[r] = s * s;
                if (y_out) y_out[row_perm[r]] = s;
            }
        } else {
            const int cnt = task.y & 0xFF;
            if (lane < cnt) {
                const int r = order[task.x + lane];
                double s = 0.0;
                if (UPPER) s += diag[r] * xv(r);
                for (int k = ptr[r]; k < ptr[r + 1]; ++k) s += val[k] * xv(col[k]);
                if (!UPPER) s += 1.0 * xs[r];
                out[r] = s;
                if (sq) sq[r] = s * s;
                if (y_out) y_out[row_perm[r]] = s;
            }
        }
    }
}

// deterministic sum of sq[0..n) -> sqrt -> weight (+ Arnoldi decision)
__global__ void __launch_bounds__(256)
    k_sum_sqrt(const double* __restrict__ sq, int n, double* __restrict__ partials,
               unsigned int* __restrict__ done_counter, Ctrl* ctrl, double* __restrict__ weight_out) {
    __shared__ double sh[33];
    __shared__ bool s_last;
    if (ctrl && (!ctrl->need_weight || ctrl->converged || ctrl->status)) return;
    double acc = 0.0;
    const int per = (n + gridDim.x - 1) / gridDim.x;
    const int lo = blockIdx.x * per, hi = min(n, lo + per);
    for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) acc += sq[i];
    const double bs = block_sum(acc, sh);
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = bs;
        __threadfence();
        s_last = atomicAdd(done_counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    double a2 = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) a2 += ld_cg(partials + b);
    const double tot = block_sum(a2, sh);
    if (threadIdx.x == 0) {
        *done_counter = 0u;
        const double w = sqrt(tot);
        if (weight_out) *weight_out = w;
        if (ctrl) {
            ctrl->weight = w;
            decide(ctrl);
        }
    }
}

// residual test of the Arnoldi iteration (krylov.cpp:150-168)
__device__ void decide(Ctrl* c) {
    if (c->status || c->converged) return;
    if (c->need_weight) {
        const double res = fabs(c->beta * c->h_next * c->s) * c->weight;
        c->last_residual = res;
        c->need_weight = 0;
        if (res < c->eps) c->converged = 1;
    }
}

// after every iteration: cap check and advance (krylov.cpp:118,165-168)
// cond != 0: the iteration runs as the body of the Arnoldi graph's WHILE
// node; the loop continues while the MEVP is neither converged nor failed.
__global__ void k_iter_end(Ctrl* c, unsigned long long cond) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    c->arnoldi_iters++;
    if (!(c->status || c->converged)) {
        if (c->need_weight) decide(c);  // weight computed by another path
        if (!c->converged) {
            if (c->m >= c->m_max)
                c->status = 5;  // EXG_E_NO_CONVERGENCE
            else
                c->j = c->m;
        }
    }
    if (cond) cudaGraphSetConditional((cudaGraphConditionalHandle)cond, (c->status || c->converged) ? 0u : 1u);
}

// all-ones (NaN sentinel) fill of the solve scratch; a kernel rather than a
// memset node so the solve can live inside the Arnoldi graph's loop body
__global__ void __launch_bounds__(256) k_fill_ones(unsigned long long* __restrict__ p, long long n8) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += stride)
        p[i] = ~0ull;
}

// ============================================================================
// ||G v|| weight (mevp_residual, krylov.cpp:204; EXG_WEIGHT_GSPMV mode)
// ============================================================================
__global__ void __launch_bounds__(256)
    k_spmv_norm(const int* __restrict__ rowptr, const int* __restrict__ col,
                const double* __restrict__ val, int n, const double* __restrict__ vbase,
                long long ldv, double* __restrict__ partials, unsigned int* done_counter,
                Ctrl* ctrl, int from_ctrl_m, double* weight_out) {
    __shared__ double sh[33];
    __shared__ bool s_last;
    const double* x = vbase;
    // from_ctrl_m 1: after the dense block (skips when no residual test is
    // pending, decides here); 2: beside the dense block (need_weight is being
    // written concurrently: always computes, k_iter_end decides)
    if (ctrl && from_ctrl_m) {
        if (ctrl->converged || ctrl->status) return;
        if (from_ctrl_m == 1 && !ctrl->need_weight) return;
        if (ctrl->happy) return;  // no v_{m+1} was written (set by the MGS kernel)
        x = vbase + (long long)ctrl->m * ldv;
    }
    // grid-stride rows (a few partials per SM, not one per 256 rows: the
    // last block's final sum is the tail of this kernel)
    double sq = 0.0;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int k = rowptr[r]; k < rowptr[r + 1]; ++k) s += val[k] * x[col[k]];
        sq += s * s;
    }
    const double bs = block_sum(sq, sh);
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = bs;
        __threadfence();
        s_last = atomicAdd(done_counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    double acc = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) acc += ld_cg(partials + b);
    const double tot = block_sum(acc, sh);
    if (threadIdx.x == 0) {
        *done_counter = 0u;
        const double w = sqrt(tot);
        if (weight_out) *weight_out = w;
        if (ctrl && from_ctrl_m) {
            ctrl->weight = w;
            if (from_ctrl_m == 1) decide(ctrl);
        }
    }
}

// ============================================================================
// MEVP start: beta = ||v||, ||x_k||_inf, early-out (integrate.cpp:244),
// zero-start check (krylov.cpp:106), V[0] = v * (1/beta) (krylov.cpp:113).
// Two kernels: per-block partials, then every block redundantly finalises
// (same fixed order => same beta everywhere) and scales its slice.
// ============================================================================
__global__ void __launch_bounds__(256)
    k_start_partials(const double* __restrict__ v, const double* __restrict__ xk, int n,
                     double* __restrict__ partials /* [2*grid] */) {
    __shared__ double sh[33];
    double sq = 0.0, mx = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        sq += v[i] * v[i];
        if (xk) {
            const double a = fabs(xk[i]);
            mx = mx < a ? a : mx;  // std::max(m, |x|)
        }
    }
    const double bs = block_sum(sq, sh);
    // max reduction (order-independent)
    for (int o = 16; o > 0; o >>= 1) {
        const double t = __shfl_down_sync(0xffffffffu, mx, o);
        mx = mx < t ? t : mx;
    }
    __shared__ double shm[32];
    if ((threadIdx.x & 31) == 0) shm[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = m < shm[w] ? shm[w] : m;
        partials[blockIdx.x] = bs;
        partials[gridDim.x + blockIdx.x] = m;
    }
}

__global__ void __launch_bounds__(256)
    k_start_finish(const double* __restrict__ v, int n, const double* __restrict__ partials,
                   int n_part, double* __restrict__ v0, Ctrl* ctrl, int er_mode) {
    __shared__ double sh[33];
    __shared__ double s_beta;
    __shared__ int s_go;
    double acc = 0.0;
    for (int b = threadIdx.x; b < n_part; b += blockDim.x) acc += partials[b];
    const double tot = block_sum(acc, sh);
    if (threadIdx.x == 0) {
        double xinf = 0.0;
        for (int b = 0; b < n_part; ++b) xinf = xinf < partials[n_part + b] ? partials[n_part + b] : xinf;
        const double beta = sqrt(tot);
        int go = 1;
        if (er_mode == 1 && beta <= 1e-9 * (1.0 + xinf)) go = 0;  // equilibrium early-out
        if (er_mode == 2 && beta == 0.0) go = 0;  // error/correction: zero w skips the MEVP
        if (go && beta == 0.0) go = -1;                          // ZeroStartVectorError
        s_beta = beta;
        s_go = go;
        if (blockIdx.x == 0) {
            ctrl->beta = beta;
            ctrl->xinf = xinf;
            ctrl->skip = go == 0;
            ctrl->fresh = go == 1;
            ctrl->status = go < 0 ? 4 : 0;
            ctrl->converged = go != 1;  // nothing to iterate
            ctrl->j = 0;
            ctrl->m = 0;
            ctrl->happy = 0;
            ctrl->need_weight = 0;
            ctrl->last_residual = __longlong_as_double(0x7FF0000000000000ll);  // +inf
        }
    }
    __syncthreads();
    if (s_go != 1) return;
    const double ib = 1.0 / s_beta;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        v0[i] = v[i] * ib;
}

// ============================================================================
// Modified Gram–Schmidt with one conditional re-orthogonalisation
// (krylov.cpp:46-78), one cooperative persistent kernel per Arnoldi step.
// Each thread keeps K elements of w in registers for the whole step, so each
// MGS pass streams only v_i from HBM.  The passes keep the reference's
// sequential dependence (h_i is the dot of the ALREADY-updated w with v_i) and
// its per-element update order; only the dot-product summation order differs
// (fixed tree: thread -> warp -> block -> ordered sum over blocks).
// ============================================================================
template <int K>
__device__ __forceinline__ double grid_sum(double v, double* sh, double* partials, int slot,
                                           unsigned int* bar) {
    const double bs = block_sum(v, sh);
    double* pp = partials + slot * 4096;
    if (threadIdx.x == 0) pp[blockIdx.x] = bs;
    grid_barrier(bar, gridDim.x);
    if (gridDim.x == 1) return bs;
    double acc = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) acc += ld_cg(pp + b);
    return block_sum(acc, sh);
}

template <int K>
__global__ void __launch_bounds__(1024)
    k_mgs(MgsArgs a) {
    __shared__ double sh[33];
    Ctrl* c = a.ctrl;
    if (c->converged || c->status) return;
    const int j = c->j;
    const int n = a.n;
    const long long ld = a.ldv;
    const int nthr = gridDim.x * blockDim.x;
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    double w[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int e = g + k * nthr;
        w[k] = e < n ? a.w[e] : 0.0;
    }
    int slot = 0;
    double p = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) p += w[k] * w[k];
    const double pre = sqrt(grid_sum<K>(p, sh, a.partials, slot ^= 1, a.bar));
    double* hcol = a.hbar + (long long)j * a.hld;
    for (int pass = 0; pass < 2; ++pass) {
        for (int i = 0; i <= j; ++i) {
            const double* vi = a.V + (long long)i * ld;
            double vv[K];
            double d = 0.0;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const int e = g + k * nthr;
                vv[k] = e < n ? vi[e] : 0.0;
                d += w[k] * vv[k];
            }
            const double hij = grid_sum<K>(d, sh, a.partials, slot ^= 1, a.bar);
            const double mh = -hij;
#pragma unroll
            for (int k = 0; k < K; ++k) w[k] += mh * vv[k];
            if (g == 0) hcol[i] = pass == 0 ? hij : hcol[i] + hij;
        }
        double q = 0.0;
#pragma unroll
        for (int k = 0; k < K; ++k) q += w[k] * w[k];
        const double post = sqrt(grid_sum<K>(q, sh, a.partials, slot ^= 1, a.bar));
        if (pass == 1 || !(post < kReorthFactor * pre)) {
            const bool happy = post <= c->breakdown_tol * pre;
            if (!happy) {
                const double ip = 1.0 / post;
                double* vn = a.V + (long long)(j + 1) * ld;
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const int e = g + k * nthr;
                    if (e < n) vn[e] = w[k] * ip;
                }
            }
            if (g == 0) {
                hcol[j + 1] = post;
                c->pre = pre;
                c->post = post;
                c->happy = happy;
                c->h_next = happy ? 0.0 : post;
                c->m = j + 1;
                c->mgs_passes += pass == 0 ? (unsigned)(j + 3) : (unsigned)(2 * j + 5);
                c->reorths += pass;
            }
            return;
        }
    }
}

template __global__ void k_mgs<1>(MgsArgs);
template __global__ void k_mgs<2>(MgsArgs);
template __global__ void k_mgs<4>(MgsArgs);
template __global__ void k_mgs<8>(MgsArgs);
template __global__ void k_mgs<16>(MgsArgs);

// ============================================================================
// Dense m x m block in one CTA (m <= MMAX): H_m, its inverse with the shift
// fallback, Pade scaling-and-squaring exponential, the residual scalar s and
// the final coefficients beta * e^{hH^-1} e_1.  Every loop keeps the
// reference's per-element operation order (dense_matrix.cpp), parallelising
// only across independent elements, so the results are bit-identical.
// ============================================================================
struct DenseCtx {
    int m;
    double* S;  // scratch base
    int* flag;  // shared flags
};

__device__ __forceinline__ void bsync() { __syncthreads(); }

// c = a * b  (i-k-j with the zero skip of multiply, :33-45); c must not alias
__device__ void d_mmul(int m, const double* a, const double* b, double* c) {
    for (int idx = threadIdx.x; idx < m * m; idx += blockDim.x) {
        const int i = idx / m, jj = idx - i * m;
        double s = 0.0;
        for (int k = 0; k < m; ++k) {
            const double aik = a[i * m + k];
            if (aik == 0.0) continue;
            s += aik * b[k * m + jj];
        }
        c[idx] = s;
    }
    bsync();
}

// c = a + beta * b (add_scaled, :60-67); c may alias a or b
__device__ void d_axpby(int m, const double* a, double beta, const double* b, double* c) {
    for (int idx = threadIdx.x; idx < m * m; idx += blockDim.x) c[idx] = a[idx] + beta * b[idx];
    bsync();
}
__device__ void d_scale(int m, double f, const double* a, double* c) {
    for (int idx = threadIdx.x; idx < m * m; idx += blockDim.x) c[idx] = f * a[idx];
    bsync();
}
__device__ void d_copy(int m, const double* a, double* c) {
    for (int idx = threadIdx.x; idx < m * m; idx += blockDim.x) c[idx] = a[idx];
    bsync();
}
__device__ void d_ident(int m, double* c) {
    for (int idx = threadIdx.x; idx < m * m; idx += blockDim.x) c[idx] = (idx / m == idx % m) ? 1.0 : 0.0;
    bsync();
}

// max column sum (norm1, :17-25); result broadcast through sh_val
__device__ double d_norm1(int m, const double* a, double* colsum, double* sh_val) {
    for (int cc = threadIdx.x; cc < m; cc += blockDim.x) {
        double s = 0.0;
        for (int r = 0; r < m; ++r) s += fabs(a[r * m + cc]);
        colsum[cc] = s;
    }
    bsync();
    if (threadIdx.x == 0) {
        double best = 0.0;
        for (int cc = 0; cc < m; ++cc) best = best < colsum[cc] ? colsum[cc] : best;  // std::max
        *sh_val = best;
    }
    bsync();
    return *sh_val;
}

// dense_solve (:69-118): A X = B by partial-pivot LU.  x holds B on entry and
// X on exit (m x m).  Returns false on an exactly-zero pivot column
// (SingularMatrixError).
__device__ bool d_solve(int m, const double* a, double* x, double* lu, int* sh_i, double* sh_d) {
    d_copy(m, a, lu);
    for (int k = 0; k < m; ++k) {
        if (threadIdx.x < 32) {
            const int lane = threadIdx.x;
            const double dkk = fabs(lu[k * m + k]);
            double lb = -1.0;
            int li = INT_MAX;
            for (int r = k + 1 + lane; r < m; r += 32) {
                const double v = fabs(lu[r * m + k]);
                if (v > lb) {
                    lb = v;
                    li = r;
                }
            }
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_down_sync(0xffffffffu, lb, o);
                const int oi = __shfl_down_sync(0xffffffffu, li, o);
                if (ob > lb || (ob == lb && oi < li)) {
                    lb = ob;
                    li = oi;
                }
            }
            if (lane == 0) {
                int p = k;
                double best = dkk;
                if (!isnan(dkk) && li != INT_MAX && lb > dkk) {
                    p = li;
                    best = lb;
                }
                sh_i[0] = p;
                sh_d[0] = best;
            }
        }
        bsync();
        const int p = sh_i[0];
        if (sh_d[0] == 0.0) return false;
        if (p != k) {
            for (int jj = threadIdx.x; jj < m; jj += blockDim.x) {
                double t = lu[k * m + jj];
                lu[k * m + jj] = lu[p * m + jj];
                lu[p * m + jj] = t;
                t = x[k * m + jj];
                x[k * m + jj] = x[p * m + jj];
                x[p * m + jj] = t;
            }
            bsync();
        }
        const double d = lu[k * m + k];
        for (int r = k + 1 + threadIdx.x; r < m; r += blockDim.x) lu[r * m + k] = lu[r * m + k] / d;
        bsync();
        // rows r > k: lu[r][k+1..m) and x[r][0..m)
        const int wl = m - k - 1, wx = m;
        const int per_row = wl + wx;
        for (int idx = threadIdx.x; idx < (m - k - 1) * per_row; idx += blockDim.x) {
            const int r = k + 1 + idx / per_row;
            const int q = idx - (r - k - 1) * per_row;
            const double f = lu[r * m + k];
            if (f == 0.0) continue;
            if (q < wl) {
                const int jj = k + 1 + q;
                lu[r * m + jj] -= f * lu[k * m + jj];
            } else {
                const int jj = q - wl;
                x[r * m + jj] -= f * x[k * m + jj];
            }
        }
        bsync();
    }
    // back substitution, one thread per right-hand-side column
    for (int jj = threadIdx.x; jj < m; jj += blockDim.x) {
        for (int k = m - 1; k >= 0; --k) {
            const double d = lu[k * m + k];
            double s = x[k * m + jj];
            for (int cc = k + 1; cc < m; ++cc) s -= lu[k * m + cc] * x[cc * m + jj];
            x[k * m + jj] = s / d;
        }
    }
    bsync();
    return true;
}

// dense_inverse (:120-124) with cond1 = ||A||_1 ||A^-1||_1
__device__ bool d_inverse(int m, const double* a, double* inv, double* lu, double* colsum,
                          int* sh_i, double* sh_d, double* cond) {
    d_ident(m, inv);
    if (!d_solve(m, a, inv, lu, sh_i, sh_d)) return false;
    const double na = d_norm1(m, a, colsum, sh_d + 1);
    const double ni = d_norm1(m, inv, colsum, sh_d + 1);
    *cond = na * ni;
    return true;
}

// invert_reduced (krylov.cpp:85-101)
__device__ bool d_invert_reduced(int m, const double* hm, double* hinv, double* sh_m,
                                 double* lu, double* colsum, int* sh_i, double* sh_d) {
    double scale = d_norm1(m, hm, colsum, sh_d + 2);
    scale = scale < 1e-300 ? 1e-300 : scale;  // std::max(norm1, 1e-300)
    const double deltas[3] = {0.0, 1e-12 * scale, 1e-9 * scale};
    for (int t = 0; t < 3; ++t) {
        d_copy(m, hm, sh_m);
        for (int i = threadIdx.x; i < m; i += blockDim.x) sh_m[i * m + i] -= deltas[t];
        bsync();
        double cond = 0.0;
        if (d_inverse(m, sh_m, hinv, lu, colsum, sh_i, sh_d, &cond) && cond < kCondLimit) return true;
    }
    return false;
}

// pade_expm (:137-181).  w: 10 scratch matrices.
__device__ bool d_pade(int m, const double* a, const double* b, int degree, double* out,
                       double* w, double* colsum, int* sh_i, double* sh_d) {
    const int mm = m * m;
    double* ident = w;
    double* a2 = w + mm;
    double* u = w + 2 * mm;
    double* v = w + 3 * mm;
    double* t1 = w + 4 * mm;
    double* t2 = w + 5 * mm;
    double* t3 = w + 6 * mm;
    double* t4 = w + 7 * mm;
    double* t5 = w + 8 * mm;
    double* lu = w + 9 * mm;
    d_ident(m, ident);
    d_mmul(m, a, a, a2);
    if (degree <= 9) {
        double* usum = t1;
        double* vsum = t2;
        double* pw = t3;
        for (int idx = threadIdx.x; idx < mm; idx += blockDim.x) {
            usum[idx] = 0.0;
            vsum[idx] = 0.0;
        }
        d_copy(m, ident, pw);
        for (int k = 0; k <= degree; k += 2) {
            d_axpby(m, vsum, b[k], pw, vsum);
            d_axpby(m, usum, b[k + 1], pw, usum);
            if (k + 2 <= degree) {
                d_mmul(m, pw, a2, t4);
                d_copy(m, t4, pw);
            }
        }
        d_mmul(m, a, usum, u);
        d_copy(m, vsum, v);
    } else {
        double* a4 = t1;
        double* a6 = t2;
        d_mmul(m, a2, a2, a4);
        d_mmul(m, a4, a2, a6);
        // u1 = a6 * (b13 a6 + b11 a4 + b9 a2)
        d_scale(m, b[13], a6, t3);
        d_scale(m, b[11], a4, t4);
        d_axpby(m, t3, 1.0, t4, t3);
        d_scale(m, b[9], a2, t4);
        d_axpby(m, t3, 1.0, t4, t3);
        d_mmul(m, a6, t3, t5);  // u1
        // u2 = b7 a6 + b5 a4 + b3 a2 + b1 I
        d_scale(m, b[7], a6, t3);
        d_scale(m, b[5], a4, t4);
        d_axpby(m, t3, 1.0, t4, t3);
        d_scale(m, b[3], a2, t4);
        d_axpby(m, t3, 1.0, t4, t3);
        d_axpby(m, t3, b[1], ident, t3);  // u2
        d_axpby(m, t5, 1.0, t3, t4);      // u1 + u2
        d_mmul(m, a, t4, u);
        // v1 = a6 * (b12 a6 + b10 a4 + b8 a2)
        d_scale(m, b[12], a6, t3);
        d_scale(m, b[10], a4, t4);
        d_axpby(m, t3, 1.0, t4, t3);
        d_scale(m, b[8], a2, t4);
        d_axpby(m, t3, 1.0, t4, t3);
        d_mmul(m, a6, t3, t5);  // v1
        d_scale(m, b[6], a6, t3);
        d_scale(m, b[4], a4, t4);
        d_axpby(m, t3, 1.0, t4, t3);
        d_scale(m, b[2], a2, t4);
        d_axpby(m, t3, 1.0, t4, t3);
        d_axpby(m, t3, b[0], ident, t3);  // v2
        d_axpby(m, t5, 1.0, t3, v);
    }
    // (V - U) X = (V + U)
    d_axpby(m, v, 1.0, u, out);
    d_axpby(m, v, -1.0, u, t1);
    return d_solve(m, t1, out, lu, sh_i, sh_d);
}

// dense_expm (:185-225).  Returns 0 ok, 2 non-finite input, 3 singular solve.
// w: 13 scratch matrices.
__device__ int d_expm(int m, const double* M, double* out, double* w, double* colsum, int* sh_i,
                      double* sh_d) {
    const double c_b3[4] = {120, 60, 12, 1};
    const double c_b5[6] = {30240, 15120, 3360, 420, 30, 1};
    const double c_b7[8] = {17297280, 8648640, 1995840, 277200, 25200, 1512, 56, 1};
    const double c_b9[10] = {17643225600., 8821612800., 2075673600., 302702400., 30270240.,
                             2162160.,     110880.,     3960.,       90.,        1.};
    const double c_b13[14] = {64764752532480000., 32382376266240000., 7771770303897600.,
                              1187353796428800.,  129060195264000.,   10559470521600.,
                              670442572800.,      33522128640.,       1323241920.,
                              40840800.,          960960.,            16380.,
                              182.,               1.};
    const int mm = m * m;
    if (threadIdx.x == 0) sh_i[1] = 0;
    bsync();
    for (int idx = threadIdx.x; idx < mm; idx += blockDim.x)
        if (!isfinite(M[idx])) sh_i[1] = 1;
    bsync();
    if (sh_i[1]) return 2;
    const double nrm = d_norm1(m, M, colsum, sh_d + 3);
    const double theta3 = 1.495585217958292e-2, theta5 = 2.539398330063230e-1,
                 theta7 = 9.504178996162932e-1, theta9 = 2.097847961257068e0,
                 theta13 = 5.371920351148152e0;
    bool ok;
    if (nrm <= theta3) {
        ok = d_pade(m, M, c_b3, 3, out, w, colsum, sh_i, sh_d);
    } else if (nrm <= theta5) {
        ok = d_pade(m, M, c_b5, 5, out, w, colsum, sh_i, sh_d);
    } else if (nrm <= theta7) {
        ok = d_pade(m, M, c_b7, 7, out, w, colsum, sh_i, sh_d);
    } else if (nrm <= theta9) {
        ok = d_pade(m, M, c_b9, 9, out, w, colsum, sh_i, sh_d);
    } else {
        int s = 0;
        double sn = nrm;
        while (sn > theta13) {
            sn *= 0.5;
            ++s;
        }
        double* a = w + 10 * mm;
        const double f = ldexp(1.0, -s);
        for (int idx = threadIdx.x; idx < mm; idx += blockDim.x) a[idx] = M[idx] * f;
        bsync();
        ok = d_pade(m, a, c_b13, 13, out, w, colsum, sh_i, sh_d);
        double* t = w + 11 * mm;
        for (int k = 0; k < s && ok; ++k) {
            d_mmul(m, out, out, t);
            d_copy(m, t, out);
        }
    }
    return ok ? 0 : 3;
}

// Per-iteration dense step (krylov.cpp:129-163) and the final / re-check
// evaluations (krylov.cpp:170-171, :191-215).
//   mode 0: Arnoldi iteration check at ctrl->h
//   mode 1: final coefficients coef[i] = beta * e^{h H^-1}(i,0) at h_eval
//   mode 2: residual scalar s at h_eval for the cached basis (mevp_residual)
//   mode 3: debug, the whole exponential e^{h_eval * hinv} (exg_debug_dense_expm)
__global__ void __launch_bounds__(256)
    k_dense(DenseArgs a) {
    extern __shared__ double dyn_smem[];
    __shared__ int sh_i[4];
    __shared__ double sh_d[8];
    Ctrl* c = a.ctrl;
    if (a.mode == 0 && (c->converged || c->status)) return;
    if (a.mode == 1 && (c->status || c->skip)) return;
    const int m = c->m;
    const int mm = m * m;
    double* S = (size_t)20 * mm * sizeof(double) <= (size_t)a.smem_cap ? dyn_smem : a.scratch;
    double* hm = S;
    double* hinv_tmp = S + mm;
    double* e = S + 2 * mm;
    double* sc = S + 3 * mm;
    double* shm = S + 4 * mm;
    double* lu = S + 5 * mm;
    double* colsum = S + 6 * mm;  // m entries (one matrix reserved)
    double* w = S + 7 * mm;       // 13 matrices
    if (a.mode == 0) {
        // H_m from the Hessenberg columns (reduced_from_cols, krylov.cpp:15-20)
        for (int idx = threadIdx.x; idx < mm; idx += blockDim.x) {
            const int i = idx / m, jj = idx - i * m;
            hm[idx] = (i <= jj + 1) ? a.hbar[(long long)jj * a.hld + i] : 0.0;
        }
        bsync();
        const bool inv = d_invert_reduced(m, hm, hinv_tmp, shm, lu, colsum, sh_i, sh_d);
        if (c->happy) {
            if (!inv) {
                if (threadIdx.x == 0) c->status = 6;  // SingularReducedMatrixError
                return;
            }
            for (int idx = threadIdx.x; idx < mm; idx += blockDim.x) a.hinv[idx] = hinv_tmp[idx];
            if (threadIdx.x == 0) {
                c->last_residual = 0.0;
                c->converged = 1;
                c->need_weight = 0;
            }
            return;
        }
        const bool check = (m % c->check_stride == 0) || m == c->m_max;
        if (!check || !inv) {
            if (threadIdx.x == 0) c->need_weight = 0;
            return;
        }
        for (int idx = threadIdx.x; idx < mm; idx += blockDim.x) {
            a.hinv[idx] = hinv_tmp[idx];
            sc[idx] = c->h * hinv_tmp[idx];
        }
        bsync();
        const int st = d_expm(m, sc, e, w, colsum, sh_i, sh_d);
        if (st) {
            if (threadIdx.x == 0) c->status = st == 2 ? 2 : 3;
            return;
        }
        if (threadIdx.x == 0) {
            double s = 0.0;
            for (int i = 0; i < m; ++i) s += hinv_tmp[(m - 1) * m + i] * e[i * m];
            c->s = s;
            c->need_weight = 1;
        }
        return;
    }
    // modes 1, 2: reduced_exp at h_eval from the stored H_m^-1
    for (int idx = threadIdx.x; idx < mm; idx += blockDim.x) sc[idx] = a.h_eval * a.hinv[idx];
    bsync();
    const int st = d_expm(m, sc, e, w, colsum, sh_i, sh_d);
    if (st) {
        if (threadIdx.x == 0) c->status = st == 2 ? 2 : 3;
        return;
    }
    if (a.mode == 3) {
        for (int idx = threadIdx.x; idx < mm; idx += blockDim.x) a.full_out[idx] = e[idx];
    } else if (a.mode == 1) {
        for (int i = threadIdx.x; i < m; i += blockDim.x) a.coef[i] = c->beta * e[i * m];
    } else if (threadIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < m; ++i) s += a.hinv[(m - 1) * m + i] * e[i * m];
        c->s = s;
    }
}

// ============================================================================
// Basis combination beta * V_m e^{hH^-1} e_1 (krylov.cpp:32-36) and the ER
// update (integrate.cpp:241,262-263), one streaming pass over V.
//   mode 0: out = sum_j coef_j v_j
//   mode 1: x_next = ((x_k + 1.0*(gb*h)) + 1.0*value) + (-1.0*start)
// ============================================================================
__global__ void __launch_bounds__(256)
    k_combine(const double* __restrict__ V, long long ldv, const double* __restrict__ coef,
              int n, double* __restrict__ out, const Ctrl* ctrl, int mode,
              const double* __restrict__ xk, const double* __restrict__ gb,
              const double* __restrict__ start, double h) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const bool have = !ctrl->skip && !ctrl->status;
    double val = 0.0;
    if (have) {
        const int m = ctrl->m;
        for (int jj = 0; jj < m; ++jj) val += coef[jj] * V[(long long)jj * ldv + i];
    }
    if (mode == 0) {
        out[i] = val;
        return;
    }
    double x = xk[i] + 1.0 * (gb[i] * h);
    if (have) {
        x += 1.0 * val;
        x += -1.0 * start[i];
    }
    out[i] = x;
}

// out = residual-check weight ||G v_{m+1}|| * |beta h_next s| for the cached
// basis (mevp_residual, krylov.cpp:191-205)
__global__ void k_basis_residual_final(Ctrl* c, double* out) {
    if (threadIdx.x || blockIdx.x) return;
    if (c->happy || c->h_next == 0.0) {
        *out = 0.0;
        return;
    }
    *out = fabs(c->beta * c->h_next * c->s) * c->weight;
}

// ============================================================================
// Nonlinear devices (config 4): residual_F (devices.cpp:202-233) on the
// device.  k_mos_r evaluates every MOSFET at x (mosfet_current,
// devices.cpp:31-66, same arithmetic) and forms r = gm*vgs + gds*vds - id
// with the frozen operating point; k_node_gather adds the contributions of
// each node in device order (F[d] += r, F[s] -= r), so the sum order — and
// the result — is the reference's.
// ============================================================================
__device__ __forceinline__ void mos_current(double vth, double kp, double lam, double w, double l,
                                            double vgs, double vds, double& id, double& gm,
                                            double& gds) {
    bool swapped = false;
    if (vds < 0.0) {
        vgs = vgs - vds;
        vds = -vds;
        swapped = true;
    }
    const double k = kp * w / l;
    const double vov = vgs - vth;
    if (vov <= 0.0) {
        id = 0.0;
        gm = 0.0;
        gds = 0.0;
    } else if (vds >= vov) {
        const double clm = 1.0 + lam * vds;
        id = 0.5 * k * vov * vov * clm;
        gm = k * vov * clm;
        gds = 0.5 * k * vov * vov * lam;
    } else {
        const double clm = 1.0 + lam * vds;
        const double q = vov * vds - 0.5 * vds * vds;
        id = k * q * clm;
        gm = k * vds * clm;
        gds = k * (vov - vds) * clm + k * q * lam;
    }
    if (swapped) {
        const double gm_s = gm;
        const double gds_s = gds;
        id = -id;
        gm = -gm_s;
        gds = gm_s + gds_s;
    }
}

__global__ void __launch_bounds__(256)
    k_mos_r(int n_mos, const int4* __restrict__ nodes, const double* __restrict__ par,
            const double* __restrict__ op, const double* __restrict__ x, double* __restrict__ r) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_mos) return;
    const int4 nd = nodes[i];  // d, g, s, b
    const double vd = nd.x < 0 ? 0.0 : x[nd.x];
    const double vg = nd.y < 0 ? 0.0 : x[nd.y];
    const double vs = nd.z < 0 ? 0.0 : x[nd.z];
    const double vgs = vg - vs;
    const double vds = vd - vs;
    const double* p = par + 6 * i;  // vth kp lambda w l pmos
    const double sign = p[5] != 0.0 ? -1.0 : 1.0;
    double id, gm, gds;
    mos_current(p[0], p[1], p[2], p[3], p[4], sign * vgs, sign * vds, id, gm, gds);
    id *= sign;
    const double gm0 = op[5 * i + 3], gds0 = op[5 * i + 4];
    r[i] = gm0 * vgs + gds0 * vds - id;
}

// F[i] = sum of the node's contributions in device order; with fsub: the
// result is F - fsub (deltaF = residual_F(x_next) - F_k, integrate.cpp:435)
__global__ void __launch_bounds__(256)
    k_node_gather(int n, const int* __restrict__ ptr, const int* __restrict__ list,
                  const double* __restrict__ r, double* __restrict__ F,
                  const double* __restrict__ fsub) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double f = 0.0;
    for (int k = ptr[i]; k < ptr[i + 1]; ++k) {
        const int e = list[k];
        if (e >= 0)
            f += r[e];
        else
            f -= r[-1 - e];
    }
    if (fsub) f = f + -1.0 * fsub[i];
    F[i] = f;
}

// ||v||_inf (exact: max is order independent), two-stage, and elementwise ops
// of the nonlinear error / correction (integrate.cpp:267-298).  The max
// propagates NaN (a NaN operand wins), so a non-finite vector never reads as
// a finite norm: the caller maps it to EXG_E_NONFINITE like residual_F's
// all_finite check (devices.cpp:205).
__device__ __forceinline__ double nanmax(double m, double a) { return (a > m || a != a) && m == m ? a : m; }

__global__ void __launch_bounds__(256)
    k_absmax(const double* __restrict__ v, int n, double* __restrict__ partials,
             unsigned int* done, double* out) {
    __shared__ double sh[32];
    __shared__ bool s_last;
    double m = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        m = nanmax(m, fabs(v[i]));
    for (int o = 16; o > 0; o >>= 1) m = nanmax(m, __shfl_down_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        double b = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) b = nanmax(b, sh[w]);
        partials[blockIdx.x] = b;
        __threadfence();
        s_last = atomicAdd(done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last || threadIdx.x) return;
    double b = 0.0;
    for (int k = 0; k < (int)gridDim.x; ++k) b = nanmax(b, ld_cg(partials + k));
    *out = b;
    *done = 0u;
}

// out = a + alpha * b  (sub: alpha = -1; axpy)
__global__ void k_axpby(const double* __restrict__ a, double alpha, const double* __restrict__ b,
                        double* __restrict__ out, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = a[i] + alpha * b[i];
}

// d = gamma * (w + (1/h) * (value + (-1.0 * u)));  x += 1.0 * d
__global__ void k_erc_update(const double* __restrict__ w, const double* __restrict__ value,
                             const double* __restrict__ u, int have_u, double ih, double gamma,
                             double* __restrict__ x, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double d = w[i];
    if (have_u) d += ih * (value[i] + -1.0 * u[i]);
    d *= gamma;
    x[i] += 1.0 * d;
}

// ============================================================================
// launch wrappers
// ============================================================================
namespace {
inline unsigned int cdiv(long long a, long long b) { return (unsigned int)((a + b - 1) / b); }
inline void count(const Launch& L, int k = 1) {
    if (L.launches) *L.launches += k;
}
}  // namespace

size_t ctrl_size() { return sizeof(Ctrl); }

void spmv(const Launch& L, const int* rowptr, const int* col, const double* val, int n_rows,
          const double* x, double* y, const Ctrl* ctrl, const double* vbase, long long ldv) {
    if (n_rows <= 0) return;
    const unsigned int grid = cdiv(cdiv(n_rows, 32), kSpmvWarps);
    k_spmv<<<grid, kSpmvWarps * 32, 0, L.stream>>>(rowptr, col, val, n_rows, x, y, ctrl, vbase, ldv);
    count(L);
}

int spmv_strip_rows() { return kSpmvStripRows; }

void spmv_v4(const Launch& L, const int* rowptr, const int* col, const double* val, int n_rows, int max_strip,
             double* y, const Ctrl* ctrl, const double* vbase, long long ldv) {
    if (n_rows <= 0) return;
    // large matrices whose strips fit a stage: col/val through a shared-memory ring (EXG_SPMV_STREAM=0
    // keeps the direct loads)
    static const int stream = getenv("EXG_SPMV_STREAM") ? atoi(getenv("EXG_SPMV_STREAM")) : 1;
    const int per = (int)(((long long)n_rows + L.num_sms - 1) / L.num_sms);
    if (stream > 0 && n_rows >= 64 * 1024 && max_strip > 0 && max_strip + 8 <= kSpmvStageCap &&
        per <= kSpmvMaxStrips * kSpmvStripRows) {
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(k_spmv_v4t, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSpmvStreamSmem);
            attr = true;
        }
        k_spmv_v4t<<<cdiv(n_rows, per), (kSpmvConsumers + 1) * 32, kSpmvStreamSmem, L.stream>>>(rowptr, col, val, n_rows, per,
                                                                                            y, ctrl, vbase, ldv);
    } else {
        const unsigned int grid = cdiv(n_rows, 64);
        k_spmv_v4<<<grid, 256, 0, L.stream>>>(rowptr, col, val, n_rows, y, ctrl, vbase, ldv);
    }
    count(L);
}

void spmv_sub(const Launch& L, const int* rowptr, const int* col, const double* val, int n_rows,
              const double* x, const double* z, double* y) {
    if (n_rows <= 0) return;
    const unsigned int grid = cdiv(cdiv(n_rows, 32), kSpmvWarps);
    k_spmv_sub<<<grid, kSpmvWarps * 32, 0, L.stream>>>(rowptr, col, val, n_rows, x, z, y);
    count(L);
}

void spmv_b2(const Launch& L, const int* rowptr, const int* col, const double* val, int n_rows,
             const double* u_k, const double* u_k1, double h, double* t1, double* t2, const double* Fk) {
    if (n_rows <= 0) return;
    const unsigned int grid = cdiv(cdiv(n_rows, 32), kSpmvWarps);
    k_spmv_b2<<<grid, kSpmvWarps * 32, 0, L.stream>>>(rowptr, col, val, n_rows, u_k, u_k1, h, t1, t2, Fk);
    count(L);
}

template <bool U, bool FST>
static int trsv2_occ() {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_trsv2<U, FST>, 256, 0);
    return occ > 0 ? occ : 1;
}

void trsv(const Launch& L, bool upper, bool reverse, const TrsvArgs& a) {
    if (a.n <= 0 || a.n_tasks <= 0) return;
    static int occ[4] = {0, 0, 0, 0};
    const int id = (upper ? 2 : 0) + (reverse ? 1 : 0);
    if (!occ[id])
        occ[id] = id == 0 ? trsv2_occ<false, false>() : id == 1 ? trsv2_occ<false, true>()
                : id == 2 ? trsv2_occ<true, false>() : trsv2_occ<true, true>();
    const long long warps_needed = a.n_tasks;
    const unsigned int grid = (unsigned int)std::max<long long>(
        1, std::min<long long>((long long)L.num_sms * occ[id], (warps_needed + 7) / 8));
    if (!upper && !reverse) k_trsv2<false, false><<<grid, 256, 0, L.stream>>>(a);
    else if (!upper) k_trsv2<false, true><<<grid, 256, 0, L.stream>>>(a);
    else if (!reverse) k_trsv2<true, false><<<grid, 256, 0, L.stream>>>(a);
    else k_trsv2<true, true><<<grid, 256, 0, L.stream>>>(a);
    count(L);
}

template <bool U>
static int trsv3_occ() {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_trsv3<U>, 256, 0);
    return occ > 0 ? occ : 1;
}

cudaError_t trsv_chain(const Launch& L, bool upper, const ChainArgs& a) {
    static bool attr[2] = {false, false};
    static int max_clusters[2] = {0, 0};
    auto fn = upper ? (void*)k_trsv_chain<true> : (void*)k_trsv_chain<false>;
    cudaLaunchConfig_t cfg{};
    cfg.blockDim = dim3(kChainThreads);
    cfg.dynamicSmemBytes = kChainSmem;
    cfg.stream = L.stream;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kCC;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.attrs = at;
    if (!attr[upper]) {
        cudaError_t ea = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kChainSmem);
        if (ea == cudaSuccess) ea = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (ea != cudaSuccess) return ea;
        // how many kCC-CTA clusters fit at once (not every GPC holds a
        // multiple of kCC SMs)
        cfg.gridDim = dim3(kCC * (unsigned)L.num_sms);
        cfg.numAttrs = 1;
        int mc = 0;
        if (upper)
            cudaOccupancyMaxActiveClusters(&mc, k_trsv_chain<true>, &cfg);
        else
            cudaOccupancyMaxActiveClusters(&mc, k_trsv_chain<false>, &cfg);
        if (mc < 2) return cudaErrorLaunchOutOfResources;  // chain + at least one worker cluster
        max_clusters[upper] = mc > 1 ? mc : 2;
        attr[upper] = true;
    }
    // clusters of kCC (the first = the chain, the rest workers); cooperative so
    // every worker is resident while the chain waits on them
    const long long want = 1 + ((long long)a.n_rows + 8) / 9 / kCC + 1;
    const long long nclu = std::max<long long>(2, std::min<long long>(max_clusters[upper], want));
    cfg.gridDim = dim3((unsigned)(kCC * nclu));
    // EXG_NO_COOP: plain cluster launch (ncu cannot replay a cooperative
    // cluster launch); co-residency then rests on the occupancy sizing above
    static const bool no_coop = getenv("EXG_NO_COOP") != nullptr;
    cfg.numAttrs = no_coop ? 1 : 2;
    cudaError_t e;
    if (upper)
        e = cudaLaunchKernelEx(&cfg, k_trsv_chain<true>, a);
    else
        e = cudaLaunchKernelEx(&cfg, k_trsv_chain<false>, a);
    count(L);
    return e;
}

cudaError_t trsv_sub(const Launch& L, bool upper, const SubArgs& a) {
    if (a.n_comps <= 0) return cudaSuccess;
    static size_t attr_bytes[2] = {0, 0};
    const size_t smem = (size_t)a.max_rows * (sizeof(double) + sizeof(int4)) + (size_t)a.max_tasks * sizeof(int2) +
                        (size_t)(a.max_levels + 1) * sizeof(int);
    auto fn = upper ? (const void*)k_trsv_sub<true> : (const void*)k_trsv_sub<false>;
    if (smem > 48 * 1024 && attr_bytes[upper] < smem) {
        const cudaError_t ea = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (ea != cudaSuccess) return ea;
        attr_bytes[upper] = smem;
    }
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 256, smem);
    if (occ < 1) return cudaErrorLaunchOutOfResources;
    const unsigned int grid = (unsigned int)std::min<long long>(a.n_comps, (long long)L.num_sms * occ);
    if (upper)
        k_trsv_sub<true><<<grid, 256, smem, L.stream>>>(a);
    else
        k_trsv_sub<false><<<grid, 256, smem, L.stream>>>(a);
    count(L);
    return cudaGetLastError();
}

cudaError_t trsv_wide(const Launch& L, bool upper, const TrsvArgs& a) {
    if (a.n_tasks <= 0) return cudaSuccess;
    static int occ[2] = {0, 0};
    if (!occ[upper]) occ[upper] = upper ? trsv3_occ<true>() : trsv3_occ<false>();
    const unsigned int grid = (unsigned int)std::max<long long>(
        1, std::min<long long>((long long)L.num_sms * occ[upper], ((long long)a.n_tasks + 7) / 8));
    void* args[] = {(void*)&a};
    // cooperative: every warp task's producers are resident (the sync-free
    // hand-offs spin on them); a refused launch must not leave later kernels
    // waiting on sentinels, so the status goes back to the caller
    const cudaError_t e = cudaLaunchCooperativeKernel(upper ? (void*)k_trsv3<true> : (void*)k_trsv3<false>,
                                                      dim3(grid), dim3(256), args, 0, L.stream);
    count(L);
    return e;
}

void apply_tasks(const Launch& L, const int2* utasks, int n_utasks, const int* uorder,
                 const int2* ltasks, int n_ltasks, const int* lorder, const int* uptr,
                 const int* ucol, const double* uval, const double* udiag, const int* lptr,
                 const int* lcol, const double* lval, int n, const int* col_perm,
                 const int* row_perm, const double* x, double* t, double* y, double* sq,
                 double* y_out, double* partials, unsigned int* done, Ctrl* ctrl,
                 const double* vbase, long long ldv, double* weight_out) {
    const unsigned int grid = (unsigned int)std::min<long long>((long long)L.num_sms * 8,
                                                                 ((long long)std::max(n_utasks, n_ltasks) + 7) / 8 + 1);
    k_apply_tasks<true><<<grid, 256, 0, L.stream>>>(utasks, n_utasks, uorder, uptr, ucol, uval, udiag,
                                                   col_perm, x, t, nullptr, nullptr, nullptr, ctrl,
                                                   vbase, ldv);
    k_apply_tasks<false><<<grid, 256, 0, L.stream>>>(ltasks, n_ltasks, lorder, lptr, lcol, lval, nullptr,
                                                    nullptr, t, y, sq, row_perm, y_out, ctrl, nullptr, 0);
    const unsigned int g2 = std::min<unsigned int>(cdiv(n, 2048), 1024);
    k_sum_sqrt<<<g2, 256, 0, L.stream>>>(sq, n, partials, done, ctrl, weight_out);
    count(L, 3);
}

void spmv_norm(const Launch& L, const int* rowptr, const int* col, const double* val, int n,
               const double* vbase, long long ldv, double* partials, unsigned int* done,
               Ctrl* ctrl, int from_ctrl_m, double* weight_out) {
    const unsigned int grid = std::min<unsigned int>(cdiv(n, 256), (unsigned int)L.num_sms * 4);
    k_spmv_norm<<<grid, 256, 0, L.stream>>>(rowptr, col, val, n, vbase, ldv, partials,
                                                   done, ctrl, from_ctrl_m, weight_out);
    count(L);
}

void start(const Launch& L, const double* v, const double* xk, int n, double* partials,
           double* v0, Ctrl* ctrl, int er_mode) {
    const unsigned int grid = std::min<unsigned int>(cdiv(n, 256), (unsigned int)L.num_sms * 4);
    k_start_partials<<<grid, 256, 0, L.stream>>>(v, xk, n, partials);
    k_start_finish<<<grid, 256, 0, L.stream>>>(v, n, partials, (int)grid, v0, ctrl, er_mode);
    count(L, 2);
}

template <int K>
static int mgs_occ() {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_mgs<K>, 1024, 0);
    return occ;
}

int mgs_max_blocks(int K) {
    switch (K) {
        case 1: return mgs_occ<1>();
        case 2: return mgs_occ<2>();
        case 4: return mgs_occ<4>();
        case 8: return mgs_occ<8>();
        default: return mgs_occ<16>();
    }
}

cudaError_t mgs(const Launch& L, const MgsArgs& a, int n_blocks, int K) {
    void* args[] = {(void*)&a};
    void* fn;
    switch (K) {
        case 1: fn = (void*)k_mgs<1>; break;
        case 2: fn = (void*)k_mgs<2>; break;
        case 4: fn = (void*)k_mgs<4>; break;
        case 8: fn = (void*)k_mgs<8>; break;
        default: fn = (void*)k_mgs<16>; break;
    }
    cudaError_t e;
    if (n_blocks == 1)
        e = cudaLaunchKernel(fn, dim3(1), dim3(1024), args, 0, L.stream);
    else
        e = cudaLaunchCooperativeKernel(fn, dim3(n_blocks), dim3(1024), args, 0, L.stream);
    count(L);
    return e;
}


void dense(const Launch& L, const DenseArgs& a0, int m) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_dense, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr = true;
    }
    // m: an upper bound of the dimension the kernel will find in the control
    // block (exact in eager launches, m_max inside the Arnoldi graph)
    DenseArgs a = a0;
    const size_t need = (size_t)20 * m * m * sizeof(double);
    a.smem_cap = (int)std::min<size_t>(need, 200 * 1024);
    k_dense<<<1, 256, a.smem_cap, L.stream>>>(a);
    count(L);
}

void iter_end(const Launch& L, Ctrl* ctrl, unsigned long long cond) {
    k_iter_end<<<1, 32, 0, L.stream>>>(ctrl, cond);
    count(L);
}

void fill_ones(const Launch& L, void* p, size_t bytes) {
    const long long n8 = (long long)(bytes / 8);
    const unsigned int grid = (unsigned int)std::min<long long>((long long)L.num_sms * 8, (n8 + 255) / 256);
    if (grid) k_fill_ones<<<grid, 256, 0, L.stream>>>(reinterpret_cast<unsigned long long*>(p), n8);
    count(L);
}

void combine(const Launch& L, const double* V, long long ldv, const double* coef, int n,
             double* out, const Ctrl* ctrl, int mode, const double* xk, const double* gb,
             const double* start_v, double h) {
    k_combine<<<cdiv(n, 256), 256, 0, L.stream>>>(V, ldv, coef, n, out, ctrl, mode, xk, gb, start_v, h);
    count(L);
}

void mos_residual(const Launch& L, int n_mos, const int4* nodes, const double* par,
                  const double* op, const double* x, double* r, int n, const int* nptr,
                  const int* nlist, double* F, const double* fsub) {
    if (n_mos > 0) k_mos_r<<<cdiv(n_mos, 256), 256, 0, L.stream>>>(n_mos, nodes, par, op, x, r);
    k_node_gather<<<cdiv(n, 256), 256, 0, L.stream>>>(n, nptr, nlist, r, F, fsub);
    count(L, 2);
}

void absmax(const Launch& L, const double* v, int n, double* partials, unsigned int* done, double* out) {
    const unsigned int g = std::min<unsigned int>(cdiv(n, 256), 1024);
    k_absmax<<<g, 256, 0, L.stream>>>(v, n, partials, done, out);
    count(L);
}

void axpby(const Launch& L, const double* a, double alpha, const double* b, double* out, int n) {
    k_axpby<<<cdiv(n, 256), 256, 0, L.stream>>>(a, alpha, b, out, n);
    count(L);
}

void erc_update(const Launch& L, const double* w, const double* value, const double* u, int have_u,
                double ih, double gamma, double* x, int n) {
    k_erc_update<<<cdiv(n, 256), 256, 0, L.stream>>>(w, value, u, have_u, ih, gamma, x, n);
    count(L);
}

void basis_residual_final(const Launch& L, Ctrl* ctrl, double* out) {
    k_basis_residual_final<<<1, 32, 0, L.stream>>>(ctrl, out);
    count(L);
}

}  // namespace dev
}  // namespace exg
