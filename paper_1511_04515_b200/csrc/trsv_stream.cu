// k_trsv4: the FAST triangular solve over per-warp record streams
// (trsv_plan.hpp; replaces the row-by-row sweeps of Factorization::solve,
// sparse_lu.cpp:255-291, for one triangle of the blocked augmented system).
//
// One persistent, co-resident grid.  Warp w owns tasks w, w + W, w + 2W, ...
// of the level-ordered task list; the host serialised them into ONE contiguous
// byte stream per warp.  The warp pulls its stream through a private
// shared-memory ring with bulk async copies (cp.async.bulk + mbarrier
// complete_tx, 1 KB pages, up to kPages in flight), so a task's descriptor,
// row metadata, column ids and values are in shared memory long before the
// task runs: the only global accesses on a task's path are the gathers of
// the solution values it depends on, and those are issued one task ahead.
// The solution value is the ready flag (all-ones sentinel pre-fill, one 64-bit
// relaxed store to publish, warp-uniform polling for the rare entry that is
// not there yet).  A task only waits on earlier tasks and every warp is
// resident (cooperative launch), so the earliest unfinished task always
// progresses: no deadlock, no atomics, no grid barriers.
#include <algorithm>

#include "device.hpp"
#include "kernels.cuh"
#include "trsv_plan.hpp"

namespace exg {
namespace dev {

namespace {

constexpr int kRing = 8192;  // bytes per warp (StreamParams.ring)
constexpr int kPage = 1024;  // StreamParams.page
constexpr int kPages = kRing / kPage;
constexpr int kWarps = 8;    // warps per CTA
constexpr size_t kSmem = (size_t)kWarps * kRing + (size_t)kWarps * kPages * 8;

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

struct Rec {
    int w0;       // cnt | lg << 8 | nq << 16; 0 = end of stream
    int o;        // stream offset of the record
    int bytes;
    int c[4];     // this lane's column ids (-1 = empty slot)
    double y[4];  // gathered dependencies (sentinel = not solved when read)
    // epilogue operands, valid in the first lane of each row
    int out, qq;
    double b, dg, ad;
};

}  // namespace

template <bool UPPER>
__global__ void __launch_bounds__(kWarps * 32, 3)
    k_trsv4(StreamArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    if (a.ctrl && (a.ctrl->converged || a.ctrl->status)) return;
    constexpr int MS = UPPER ? kStreamMetaU : kStreamMetaL;
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    const int gw = blockIdx.x * kWarps + wi;
    if (gw >= a.n_warps) return;
    const unsigned char* ring = smem + (size_t)wi * kRing;
    const unsigned ring_s = smem_u32(ring);
    const unsigned bar_s = smem_u32(smem + (size_t)kWarps * kRing) + (unsigned)wi * kPages * 8;
    const long long off0 = a.warp_off[gw];
    const unsigned char* src = a.data + off0;
    const int n_pages = (int)((a.warp_off[gw + 1] - off0) / kPage);
    if (lane == 0) {
#pragma unroll
        for (int q = 0; q < kPages; ++q) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_s + 8 * q));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    // lane 0 keeps the ring full: page p goes to slot p % kPages once every
    // page below p - kPages + 1 has been released
    int issued = 0;
    auto issue = [&](int released) {
        const int lim = min(n_pages, released + kPages);
        while (issued < lim) {
            const unsigned slot = (unsigned)issued % kPages;
            const unsigned bar = bar_s + 8 * slot;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(kPage) : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    ring_s + slot * kPage),
                "l"(src + (size_t)issued * kPage), "r"(kPage), "r"(bar)
                : "memory");
            ++issued;
        }
    };
    if (lane == 0) issue(0);
    int ready = 0;  // pages known to have landed (warp-uniform)
    auto need = [&](int end_off) {
        const int pg = (end_off + kPage - 1) / kPage;
        while (ready < pg) {
            const unsigned bar = bar_s + 8 * ((unsigned)ready % kPages);
            const unsigned parity = ((unsigned)ready / kPages) & 1u;
            while (!mbar_try_wait(bar, parity)) {
            }
            ++ready;
        }
    };
    auto ld_i = [&](int off) { return *reinterpret_cast<const int*>(ring + (off & (kRing - 1))); };
    auto ld_d = [&](int off) { return *reinterpret_cast<const double*>(ring + (off & (kRing - 1))); };
    // header, column ids and row metadata from the ring; dependency gathers
    // and epilogue operands issued (consumed one task later)
    auto load = [&](int o, Rec& r) {
        r.o = o;
        need(o + 16);
        const int2 h = *reinterpret_cast<const int2*>(ring + (o & (kRing - 1)));
        r.w0 = h.x;
        r.bytes = h.y;
        if (r.w0 == 0) return;
        need(o + r.bytes);
        const int cnt = r.w0 & 0xFF, lg = (r.w0 >> 8) & 0xFF, nq = (r.w0 >> 16) & 0xFF;
        const int col_off = o + 16 + cnt * MS;
#pragma unroll
        for (int q = 0; q < 4; ++q) r.c[q] = q < nq ? ld_i(col_off + (q * 32 + lane) * 4) : -1;
#pragma unroll
        for (int q = 0; q < 4; ++q) r.y[q] = r.c[q] >= 0 ? __ldca(a.out + r.c[q]) : 0.0;
        const int seg = lane >> lg;
        r.out = -1;
        r.qq = -1;
        r.b = 0.0;
        r.dg = 1.0;
        r.ad = 0.0;
        if (seg < cnt && (lane & ((1 << lg) - 1)) == 0) {
            const int m = o + 16 + seg * MS;
            const int2 oi = *reinterpret_cast<const int2*>(ring + (m & (kRing - 1)));
            r.out = oi.x;
            if (oi.y >= 0) r.b = a.in[oi.y];
            if (UPPER) {
                r.qq = ld_i(m + 8);
                r.dg = ld_d(m + 16);
                if (a.add && r.qq >= 0) r.ad = a.add[r.qq];
            }
        }
    };
    // one task: prefetch the next record (its gathers fly while this task
    // runs), wait for this task's dependencies, reduce, publish, free pages.
    // The two record states alternate roles (no register copies: a copy of a
    // register with a load in flight would wait for that load).
    auto step = [&](Rec& cur, Rec& nxt) {
        const int o_next = cur.o + cur.bytes;
        unsigned long long t_begin = 0, t_ready = 0, t_loaded = 0;
        int polls = 0;
        if (a.trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_begin));
        load(o_next, nxt);
        if (a.trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_loaded));
        // ---- the current task: wait for its dependencies (warp-uniform)
        {
            bool rd = true;
#pragma unroll
            for (int q = 0; q < 4; ++q) rd = rd && __double_as_longlong(cur.y[q]) != (long long)kSentinel;
            while (!__all_sync(FULL, rd)) {
                rd = true;
                ++polls;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (__double_as_longlong(cur.y[q]) == (long long)kSentinel) {
                        cur.y[q] = __longlong_as_double(ld_relaxed(a.out + cur.c[q]));
                        rd = rd && __double_as_longlong(cur.y[q]) != (long long)kSentinel;
                    }
                }
            }
        }
        if (a.trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_ready));
        const int cnt = cur.w0 & 0xFF, lg = (cur.w0 >> 8) & 0xFF, nq = (cur.w0 >> 16) & 0xFF;
        const int val_off = cur.o + 16 + cnt * MS + nq * 128;
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (q < nq) acc = __fma_rn(ld_d(val_off + (q * 32 + lane) * 8), cur.y[q], acc);
        for (int s = (1 << lg) >> 1; s > 0; s >>= 1) acc += __shfl_xor_sync(FULL, acc, s);
        if (cur.out >= 0) {
            double s = cur.b - acc;
            if (UPPER) s = s / cur.dg;
            st_relaxed(a.out + cur.out, s);
            if (UPPER && a.final_out && cur.qq >= 0) {
                const double yv = a.coef * s;
                a.final_out[cur.qq] = a.add ? cur.ad + yv : yv;
            }
        }
        if (a.trace && lane == 0) {  // debug: {level, begin, dependencies ready, published, warp}
            unsigned long long t_end;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
            unsigned long long* tr = a.trace + 5 * (size_t)ld_i(cur.o + 12);
            tr[0] = (unsigned long long)ld_i(cur.o + 8);
            tr[1] = t_begin;
            tr[2] = t_ready;
            tr[3] = t_end;
            tr[4] = (unsigned long long)gw | ((unsigned long long)polls << 32) |
                    ((t_loaded - t_begin) << 44);
        }
        // ---- pages wholly before the next record are free again
        __syncwarp();
        if (lane == 0) issue(o_next / kPage);
    };
    Rec ra, rb;
    load(0, ra);
    while (ra.w0 != 0) {
        step(ra, rb);
        if (rb.w0 == 0) break;
        step(rb, ra);
    }
}

static_assert(kRing == 8192 && kPage == 1024, "StreamParams defaults (trsv_plan.hpp) must match the kernel");

static cudaError_t stream_setup(bool upper, int num_sms, int* occ_out) {
    static int occ[2] = {0, 0};
    if (!occ[upper]) {
        auto fn = upper ? (const void*)k_trsv4<true> : (const void*)k_trsv4<false>;
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
        if (e != cudaSuccess) return e;
        int o = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, kWarps * 32, kSmem);
        if (e != cudaSuccess) return e;
        if (o < 1) return cudaErrorLaunchOutOfResources;
        occ[upper] = o;
    }
    (void)num_sms;
    *occ_out = occ[upper];
    return cudaSuccess;
}

int trsv_stream_warps(bool upper, int num_sms) {
    int occ = 0;
    if (stream_setup(upper, num_sms, &occ) != cudaSuccess) return 0;
    return num_sms * occ * kWarps;
}

cudaError_t trsv_stream(const Launch& L, bool upper, const StreamArgs& a) {
    if (a.n_warps <= 0) return cudaSuccess;
    int occ = 0;
    cudaError_t e = stream_setup(upper, L.num_sms, &occ);
    if (e != cudaSuccess) return e;
    const unsigned grid = (unsigned)((a.n_warps + kWarps - 1) / kWarps);
    if ((long long)grid > (long long)L.num_sms * occ) return cudaErrorCooperativeLaunchTooLarge;
    void* args[] = {(void*)&a};
    // cooperative: every warp's producers are resident (the hand-offs spin on
    // them); a refused launch must not leave later kernels waiting on sentinels
    e = cudaLaunchCooperativeKernel(upper ? (void*)k_trsv4<true> : (void*)k_trsv4<false>, dim3(grid),
                                    dim3(kWarps * 32), args, kSmem, L.stream);
    if (L.launches) ++*L.launches;
    return e;
}

}  // namespace dev
}  // namespace exg
