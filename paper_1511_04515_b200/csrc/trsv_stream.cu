// k_trsv4: the FAST triangular solve over per-warp record streams
// (trsv_plan.hpp; replaces the row-by-row sweeps of Factorization::solve,
// sparse_lu.cpp:255-291, for one triangle of the blocked augmented system).
//
// One persistent, co-resident grid.  The host's list schedule (trsv_plan.hpp)
// gave every warp its tasks, in the order it will run them, as ONE contiguous
// byte stream.  The warp pulls its stream through a private ring of
// kStreamRing record slots in shared memory, one bulk async copy per record
// (cp.async.bulk + mbarrier complete_tx), issued kStreamRing - 1 records
// ahead: a task's descriptor, row metadata, column ids and values sit at
// fixed offsets of a slot before the task runs, and the only global accesses
// on a task's path are the gathers of the solution values it depends on,
// requested one task ahead.  The solution value is the ready flag (all-ones
// sentinel pre-fill, one 64-bit relaxed store to publish); a task that is
// early polls ONE value, the dependency its latest producer writes, and only
// then re-reads whatever else was missing.  A "cont" record repeats the column
// list of the record before it: it takes over that task's gathered values
// (registers) and neither gathers nor waits.  A task only waits on tasks of
// smaller rank and every warp is resident (cooperative launch), so the earliest
// unfinished task always progresses: no deadlock, no atomics, no grid barriers.
#include <algorithm>
#include <cstdlib>

#include "device.hpp"
#include "kernels.cuh"
#include "trsv_plan.hpp"

namespace exg {
namespace dev {

namespace {

constexpr int kR = kStreamRing;
constexpr int kSlot = kStreamSlot;
// 8 warps per CTA, 3 CTAs per SM: 8 KB of ring per warp, 72 registers per thread (27 warps per SM as
// 9 x 3 measured slower, 0.83 against 0.75 ms per solve pair at config 1; so did 16 and 12 per SM)
constexpr int kWarps = 8;
constexpr int kMinB = 3;
constexpr size_t kSmem = (size_t)kWarps * kR * kSlot + (size_t)kWarps * kR * 8;
static_assert(kR == 4, "ring: the task being reduced, the one whose gathers are in flight, two records in flight");

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ bool mbar_try_wait(unsigned bar, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}

// st_relaxed never publishes a value whose high word is all ones
__device__ __forceinline__ bool is_sentinel(double v) { return __double2hiint(v) == -1; }
__device__ __forceinline__ double ld_val(const double* p) { return __longlong_as_double(ld_relaxed(p)); }

// one task's registers
struct Rec {
    unsigned base;  // shared-memory address of its slot
    int c[4];       // this lane's column ids
    double y[4];    // gathered dependencies (sentinel = not solved when read)
    double fy;      // the flag dependency
    int out;        // row this lane publishes, or -1
    double b;       // its right-hand side
};

__device__ __forceinline__ int lds_i(unsigned addr) {
    int v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ double lds_d(unsigned addr) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
    return v;
}

}  // namespace

template <bool UPPER>
__global__ void __launch_bounds__(kWarps * 32, kMinB)
    k_trsv4(StreamArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    if (a.ctrl && (a.ctrl->converged || a.ctrl->status)) return;
    constexpr int MS = UPPER ? kStreamMetaU : kStreamMetaL;
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    const int gw = blockIdx.x * kWarps + wi;
    if (gw >= a.n_warps) return;
    const int4 d0 = reinterpret_cast<const int4*>(a.desc)[2 * gw];
    const int4 d1 = reinterpret_cast<const int4*>(a.desc)[2 * gw + 1];
    const int n_tasks = d0.z;
    if (n_tasks <= 0) return;
    const unsigned char* src = a.data + (((long long)(unsigned)d0.x) | ((long long)d0.y << 32));
    const unsigned ring_s = smem_u32(smem + (size_t)wi * kR * kSlot);
    const unsigned bar_s = smem_u32(smem + (size_t)kWarps * kR * kSlot) + (unsigned)wi * kR * 8;
    double* const out = a.out;
    if (gw == 0 && lane == 0) st_relaxed(out + a.n_aug, 0.0);  // the dummy every empty entry points at
    if (lane == 0) {
#pragma unroll
        for (int q = 0; q < kR; ++q) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_s + 8 * q));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    // the warp's records go round the ring in order; lane 0 requests them
    long long o_issue = 0;
    int rq_slot = 0;  // slot of the next record to request
    auto request = [&](int bytes) {
        if (lane == 0 && bytes > 0) {
            const unsigned bar = bar_s + 8 * rq_slot;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    ring_s + rq_slot * kSlot),
                "l"(src + o_issue), "r"(bytes), "r"(bar)
                : "memory");
        }
        o_issue += bytes;
        rq_slot = rq_slot == kR - 1 ? 0 : rq_slot + 1;
    };
    request(d0.w);
    request(d1.x);
    request(d1.y);
    // the next record out of the ring: column ids from its slot, then the
    // dependency gathers and the right-hand side are requested (consumed one
    // task later; two tasks ahead with a five-slot ring and 20 warps per SM
    // measured slower, profiles/r02)
    int ld_slot = 0;
    unsigned ld_parity = 0;
    auto load = [&](Rec& r) {
        const unsigned bar = bar_s + 8 * ld_slot;
        while (!mbar_try_wait(bar, ld_parity)) {
        }
        const unsigned base = ring_s + ld_slot * kSlot;
        if (ld_slot == kR - 1) {
            ld_slot = 0;
            ld_parity ^= 1u;
        } else {
            ++ld_slot;
        }
        r.base = base;
        int w0, ahead, fc, tid;
        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(w0), "=r"(ahead), "=r"(fc), "=r"(tid) : "r"(base));
        const int cnt = w0 & 0xFF, lg = (w0 >> 8) & 0xF, nq = (w0 >> 12) & 0x7;
        const bool cont = (w0 >> 15) & 1;
        if (!cont) {
            r.fy = ld_val(out + fc);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                r.y[q] = 0.0;
                r.c[q] = 0;
                if (q < nq) {
                    r.c[q] = lds_i(base + 16 + (q * 32 + lane) * 4);
                    r.y[q] = ld_val(out + r.c[q]);
                }
            }
        }
        // a cont record repeats the column list of the task before it: it takes
        // that task's gathered values when its turn comes (step), no loads here
        r.out = -1;
        r.b = 0.0;
        if ((lane & ((1 << lg) - 1)) == 0 && (lane >> lg) < cnt) {
            const unsigned m = base + 16 + nq * (cont ? 256 : 384) + (lane >> lg) * MS;
            r.out = lds_i(m);
            const int in = lds_i(m + 4);
            if (in >= 0) r.b = a.in[in];
        }
    };
    // task k: request the record kR - 1 ahead into the slot task k - 1 just
    // left, start task k + 1, wait for this task's dependencies, reduce,
    // publish.  Two register sets alternate (no register copies: a copy of a
    // register with a load in flight would wait for that load).
    auto step = [&](int k, Rec& cur, Rec& far) {
        __syncwarp();  // every lane is done with task k - 1's slot
        request(lds_i(cur.base + 4));
        const int w0 = lds_i(cur.base);
        const bool cont = (w0 >> 15) & 1;
        if (cont) {  // task k - 1 (in `far`, complete) gathered the same dependencies
#pragma unroll
            for (int q = 0; q < 4; ++q) cur.y[q] = far.y[q];
        }
        if (k + 1 < n_tasks) load(far);
        unsigned long long t_begin = 0, t_ready = 0;
        if (a.trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_begin));
        if (!a.nodeps && !cont) {
            if (is_sentinel(cur.fy)) {
                // early: poll the one value the latest producer writes
                // (re-reading every missing value on thin levels while polling,
                // issuing the first re-read before the next task's load, a sleeping
                // back-off between polls and patching the polled value into the lanes
                // that gathered it all measured no faster or slower: profiles/r02)
                const double* fp = out + lds_i(cur.base + 8);
                do {
                    cur.fy = ld_val(fp);
                } while (is_sentinel(cur.fy));
            }
            // then whatever else was not there when it was gathered
            while (__any_sync(FULL, is_sentinel(cur.y[0]) | is_sentinel(cur.y[1]) | is_sentinel(cur.y[2]) |
                                        is_sentinel(cur.y[3]))) {
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (is_sentinel(cur.y[q])) cur.y[q] = ld_val(out + cur.c[q]);
            }
        }
        if (a.trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_ready));
        const int lg = (w0 >> 8) & 0xF, nq = (w0 >> 12) & 0x7;
        const unsigned vals = cur.base + 16 + (cont ? 0 : nq * 128) + lane * 8;
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (q < nq) acc = __fma_rn(lds_d(vals + q * 256), cur.y[q], acc);
        for (int s = (1 << lg) >> 1; s > 0; s >>= 1) acc += __shfl_xor_sync(FULL, acc, s);
        if (cur.out >= 0) {
            double s = cur.b - acc;
            if (UPPER) {
                const unsigned m = cur.base + 16 + nq * (cont ? 256 : 384) + (lane >> lg) * MS;
                s = s * lds_d(m + 16);  // 1 / diag (FAST mode)
                st_relaxed(out + cur.out, s);
                const int qq = lds_i(m + 8);
                if (a.final_out && qq >= 0) {
                    const double yv = a.coef * s;
                    a.final_out[qq] = a.add ? a.add[qq] + yv : yv;
                }
            } else {
                st_relaxed(out + cur.out, s);
            }
        }
        if (a.trace && lane == 0) {  // debug: {level, begin, dependencies ready, published, warp}
            unsigned long long t_end;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
            unsigned long long* tr = a.trace + 5 * (size_t)lds_i(cur.base + 12);
            tr[0] = (unsigned long long)((unsigned)w0 >> 16);
            tr[1] = t_begin;
            tr[2] = t_ready;
            tr[3] = t_end;
            tr[4] = (unsigned long long)gw;
        }
    };
    Rec ra, rb;
    load(ra);
    for (int k = 0; k < n_tasks; k += 2) {
        step(k, ra, rb);
        if (k + 1 < n_tasks) step(k + 1, rb, ra);
    }
}

// ---- launch ------------------------------------------------------------------
namespace {

cudaError_t stream_setup(bool upper, int* occ_out) {
    static int occ[2] = {0, 0};
    if (!occ[upper]) {
        const void* fn = upper ? (const void*)k_trsv4<true> : (const void*)k_trsv4<false>;
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
        if (e != cudaSuccess) return e;
        int o = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, kWarps * 32, kSmem);
        if (o > kMinB) o = kMinB;
        if (e != cudaSuccess) return e;
        if (o < 1) return cudaErrorLaunchOutOfResources;
        occ[upper] = o;
    }
    *occ_out = occ[upper];
    return cudaSuccess;
}

}  // namespace

int trsv_stream_warps(bool upper, int num_sms) {
    int occ = 0;
    if (stream_setup(upper, &occ) != cudaSuccess) return 0;
    return num_sms * occ * kWarps;
}

cudaError_t trsv_stream(const Launch& L, bool upper, const StreamArgs& a) {
    if (a.n_warps <= 0) return cudaSuccess;
    int occ = 0;
    cudaError_t e = stream_setup(upper, &occ);
    if (e != cudaSuccess) return e;
    const unsigned grid = (unsigned)((a.n_warps + kWarps - 1) / kWarps);
    if ((long long)grid > (long long)L.num_sms * occ) return cudaErrorCooperativeLaunchTooLarge;
    void* args[] = {(void*)&a};
    // cooperative: every warp's producers are resident (the hand-offs spin on
    // them); a refused launch must not leave later kernels waiting on sentinels
    e = cudaLaunchCooperativeKernel(upper ? (void*)k_trsv4<true> : (void*)k_trsv4<false>, dim3(grid), dim3(kWarps * 32),
                                    args, kSmem, L.stream);
    if (L.launches) ++*L.launches;
    return e;
}

}  // namespace dev
}  // namespace exg
