// The device C ABI (include/exg.h): context, device-resident CSR store, factor
// upload with host level analysis, and the hot-path entry points that replace
// the reference's spmv / Factorization::solve / apply / mevp_iks /
// mevp_residual / eval_at_scaled_h / er_begin / er_eval.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "device.hpp"
#include "exg.h"
#include "kernels.cuh"
#include "ctx.hpp"
#include "trsv_plan.hpp"

using exg::dev::Ctrl;

namespace {

struct CudaError {
    cudaError_t e;
    const char* where;
};
struct ApiError {
    exg_status st;
    std::string msg;
};

inline void ck(cudaError_t e, const char* where) {
    if (e != cudaSuccess) throw CudaError{e, where};
}

template <typename T>
T* dalloc(size_t count) {
    void* p = nullptr;
    if (count == 0) count = 1;
    ck(cudaMalloc(&p, count * sizeof(T)), "cudaMalloc");
    return static_cast<T*>(p);
}

template <typename T>
void dfree(T*& p) {
    if (p) cudaFree(p);
    p = nullptr;
}

__global__ void k_gather(const double* __restrict__ x, const int* __restrict__ idx, int k,
                         double* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < k) out[i] = x[idx[i]];
}

}  // namespace

namespace {

exg_status fail(exg_ctx* c, exg_status st, const std::string& msg) {
    if (c) {
        c->err = msg;
        c->last = st;
    }
    return st;
}

#define API_BEGIN try {
#define API_END(ctx)                                                                   \
    }                                                                                  \
    catch (const CudaError& e) {                                                       \
        return fail(ctx, EXG_E_CUDA, std::string(e.where) + ": " + cudaGetErrorString(e.e)); \
    }                                                                                  \
    catch (const ApiError& e) {                                                        \
        return fail(ctx, e.st, e.msg);                                                 \
    }                                                                                  \
    catch (const std::bad_alloc&) {                                                    \
        return fail(ctx, EXG_E_NOMEM, "host allocation failed");                       \
    }                                                                                  \
    return EXG_OK;

void upload_csr(exg_ctx* c, DCsr& m, int n_rows, int n_cols, int nnz, const int* rowptr,
                const int* col, const double* val) {
    dfree(m.rowptr);
    dfree(m.col);
    dfree(m.val);
    m.n_rows = n_rows;
    m.n_cols = n_cols;
    m.nnz = nnz;
    m.rowptr = dalloc<int>(n_rows + 1);
    // 8 zero entries past the end: k_spmv_v4t copies 16-byte aligned ranges
    m.col = dalloc<int>((size_t)nnz + 8);
    m.val = dalloc<double>((size_t)nnz + 8);
    ck(cudaMemsetAsync(m.col + nnz, 0, 8 * sizeof(int), c->stream), "upload");
    ck(cudaMemsetAsync(m.val + nnz, 0, 8 * sizeof(double), c->stream), "upload");
    m.max_strip = 0;
    const int sr = exg::dev::spmv_strip_rows();
    for (int r = 0; r < n_rows; ++r) m.max_strip = std::max(m.max_strip, rowptr[std::min(r + sr, n_rows)] - rowptr[r]);
    ck(cudaMemcpyAsync(m.rowptr, rowptr, sizeof(int) * (n_rows + 1), cudaMemcpyHostToDevice, c->stream), "upload");
    if (nnz) {
        ck(cudaMemcpyAsync(m.col, col, sizeof(int) * nnz, cudaMemcpyHostToDevice, c->stream), "upload");
        ck(cudaMemcpyAsync(m.val, val, sizeof(double) * nnz, cudaMemcpyHostToDevice, c->stream), "upload");
    }
    ck(cudaStreamSynchronize(c->stream), "upload sync");
}

void ensure_vectors(exg_ctx* c, int n) {
    if (c->vec_n >= n && c->vin) return;
    c->clear_graphs();
    dfree(c->partials);
    c->partials = dalloc<double>((size_t)std::max(8192, (n + 255) / 256 + 1024) + 2 * 4096);
    c->mgs_partials_off = (size_t)std::max(8192, (n + 255) / 256 + 1024);
    double** vs[] = {&c->vin, &c->vout, &c->t, &c->w, &c->xk, &c->xnext, &c->gb,
                     &c->startv, &c->v1, &c->t1, &c->t2, &c->t3, &c->tmp};
    for (double** p : vs) {
        dfree(*p);
        *p = dalloc<double>(n);
    }
    c->vec_n = n;
}

void ensure_inputs(exg_ctx* c, int ni) {
    if (c->n_inputs >= ni && c->u_k) return;
    dfree(c->u_k);
    dfree(c->u_k1);
    c->u_k = dalloc<double>(std::max(ni, 1));
    c->u_k1 = dalloc<double>(std::max(ni, 1));
    c->n_inputs = ni;
}

// exchange slots of k_mgs2 for bases of up to mmax columns
void ensure_mgs_slots(exg_ctx* c, int mmax) {
    const int need = 2 * (mmax + 1) + 3;
    if (c->mgs_slots && c->mgs_inst_cap >= need) return;
    c->clear_graphs();
    dfree(c->mgs_slots);
    const size_t doubles = 8 + (size_t)2 * need * c->num_sms * exg::dev::kMgs2BMax;
    c->mgs_slots = dalloc<double>(doubles);
    ck(cudaMemsetAsync(c->mgs_slots, 0xFF, doubles * sizeof(double), c->stream), "mgs slots");
    ck(cudaMemsetAsync(c->mgs_slots, 0, 64, c->stream), "mgs slots");
    c->mgs_inst_cap = need;
}

void ensure_krylov(exg_ctx* c, int mmax) {
    if (c->mmax_alloc >= mmax && c->V) return;
    c->clear_graphs();
    const int n = c->n;
    dfree(c->V);
    dfree(c->hbar);
    dfree(c->hinv);
    dfree(c->coef);
    dfree(c->dscratch);
    c->ldv = ((long long)n + 31) / 32 * 32;
    c->V = dalloc<double>((size_t)(mmax + 1) * c->ldv);
    // the ldv padding of every column stays zero (k_mgs2 streams whole tiles)
    ck(cudaMemsetAsync(c->V, 0, (size_t)(mmax + 1) * c->ldv * sizeof(double), c->stream), "basis clear");
    c->hld = mmax + 2;
    c->hbar = dalloc<double>((size_t)(mmax + 1) * c->hld);
    c->hinv = dalloc<double>((size_t)mmax * mmax);
    c->coef = dalloc<double>(mmax);
    c->dscratch = dalloc<double>((size_t)20 * mmax * mmax);
    c->mmax_alloc = mmax;
    c->basis_valid = false;
}

void require_factors(exg_ctx* c) {
    if (!c->l_ptr) throw ApiError{EXG_E_CONTRACT, "no factorization uploaded (exg_set_factors)"};
}

const DCsr& mat(exg_ctx* c, int which) {
    if (which < 0 || which > 2) throw ApiError{EXG_E_CONTRACT, "bad matrix id"};
    const DCsr& m = c->mats[which];
    if (!m.rowptr) throw ApiError{EXG_E_CONTRACT, "matrix not uploaded (exg_set_csr)"};
    return m;
}

// x = Q U^{-1} L^{-1} P b, with the fused epilogue final[q] = add[q] + coef*x
void solve_dev(exg_ctx* c, const double* b, double* final_out, double coef, const double* add,
               const Ctrl* ctrl) {
    const int n = c->n;
    // scratch: [tickets][y n][x n][chain s: L rows, U rows][chain partial slots: L, U]
    const bool fast = c->opt.trsv_mode == EXG_TRSV_FAST;
    const size_t chain_doubles = fast ? (size_t)(c->plan[0].chain_rows + c->plan[1].chain_rows +
                                                 c->plan[0].chain_slots + c->plan[1].chain_slots) : 0;
    // output of each sweep: n unknowns, or the augmented system's n_aug
    // (+ 1: the stream plan's dummy entry)
    const size_t ny = fast && c->plan[0].n_aug ? (size_t)c->plan[0].n_aug + 1 : (size_t)n;
    const size_t nx = fast && c->plan[1].n_aug ? (size_t)c->plan[1].n_aug + 1 : (size_t)n;
    exg::dev::fill_ones(c->L(), c->trsv_buf, kTrsvHdr + sizeof(double) * (ny + nx + chain_doubles));
    unsigned int* tickets = reinterpret_cast<unsigned int*>(c->trsv_buf);
    double* y = reinterpret_cast<double*>(c->trsv_buf + kTrsvHdr);
    double* x = y + ny;
    double* sbuf_dev = x + nx;  // chain runs' s values, run after run
    double* pbuf_dev = sbuf_dev + c->plan[0].chain_rows + c->plan[1].chain_rows;  // partial slots
    const int fq = fast ? 2 : 0;
    int next_ticket = 0;
    for (int tri = 0; tri < 2; ++tri) {
        const bool upper = tri == 1;
        exg::dev::TrsvArgs a{};
        a.n = n;
        a.order = upper ? c->u_order : c->l_order;
        a.ptr = upper ? c->u_ptr : c->l_ptr;
        a.col = upper ? c->u_col : c->l_col;
        a.val = upper ? c->u_val : c->l_val;
        a.diag = upper ? c->u_diag : nullptr;
        a.in = upper ? y : b;
        a.in_perm = upper ? nullptr : c->row_perm;
        a.out = upper ? x : y;
        a.ctrl = ctrl;
        a.trace = upper ? c->trace_u : c->trace_l;
        if (upper) {
            a.final_out = final_out;
            a.out_perm = c->col_perm;
            a.add = add;
            a.coef = coef;
        }
        cudaEvent_t e0 = c->prof_begin();
        const int2* tasks = c->tasks[fq + tri];
        if (!fast) {
            a.tasks = tasks;
            a.n_tasks = c->n_tasks[fq + tri];
            a.ticket = tickets + next_ticket++;
            exg::dev::trsv(c->L(), upper, fast, a);
        } else {
            const TriPlan& P = c->plan[tri];
            if (P.s_warps) {
                // per-warp record streams of the blocked augmented system
                exg::dev::StreamArgs sa{};
                sa.data = P.sdata;
                sa.desc = P.sdesc;
                sa.n_warps = P.s_warps;
                sa.n_aug = P.n_aug;
                sa.in = a.in;
                sa.out = a.out;
                sa.final_out = a.final_out;
                sa.add = a.add;
                sa.coef = a.coef;
                sa.ctrl = ctrl;
                sa.trace = a.trace;
                static const int nodeps = getenv("EXG_STREAM_NODEPS") ? atoi(getenv("EXG_STREAM_NODEPS")) : 0;
                sa.nodeps = nodeps;
                ck(exg::dev::trsv_stream(c->L(), upper, sa), "stream solve launch");
                c->prof_end(upper ? EXG_K_TRSV_U : EXG_K_TRSV_L, e0);
                continue;
            }
            const bool run_timing = getenv("EXG_RUN_TIMING") != nullptr && !c->capturing;
            std::vector<cudaEvent_t> rev;
            for (const TriPlan::Run& run : P.runs) {
                if (run_timing) {
                    cudaEvent_t e;
                    cudaEventCreate(&e);
                    cudaEventRecord(e, c->stream);
                    rev.push_back(e);
                }
                if (run.narrow == 3) {
                    exg::dev::SubArgs sa{};
                    sa.n_comps = P.sub.n_comps;
                    sa.max_rows = P.sub.max_rows;
                    sa.max_tasks = P.sub.max_tasks;
                    sa.max_levels = P.sub.max_levels;
                    sa.clev = P.sub.clev;
                    sa.ltp = P.sub.ltp;
                    sa.comps = P.sub.comps;
                    sa.tasks = P.sub.tasks;
                    sa.meta = P.sub.meta;
                    sa.ecol = P.sub.ecol;
                    sa.eval = P.sub.eval;
                    sa.in = a.in;
                    sa.diag = a.diag;
                    sa.out = a.out;
                    sa.final_out = a.final_out;
                    sa.out_perm = a.out_perm;
                    sa.add = a.add;
                    sa.coef = a.coef;
                    sa.ctrl = ctrl;
                    ck(exg::dev::trsv_sub(c->L(), upper, sa), "subtree solve launch");
                    continue;
                }
                if (run.narrow == 2) {
                    const TriPlan::Chain& ch = P.chains[run.a];
                    exg::dev::ChainArgs ca{};
                    ca.n_rows = ch.n_rows;
                    ca.n_blocks = ch.n_blocks;
                    ca.rows = P.crows + ch.rows_off;
                    ca.rq = P.crq + ch.rows_off;
                    ca.nptr = P.cnptr + ch.nptr_off;
                    ca.ncol = P.cncol + ch.ent0;
                    ca.nval = P.cnval + ch.ent0;
                    ca.blocks = P.cblocks + 3 * (long long)ch.blk0;
                    ca.pool = P.pool;
                    ca.s = sbuf_dev;
                    ca.part = pbuf_dev + ch.slot0;
                    ca.pslot = P.cpslot + ch.rows_off;
                    ca.wtasks = P.ctasks + ch.task0;
                    ca.n_tasks = ch.ntasks;
                    ca.in = a.in;
                    ca.in_perm = a.in_perm;
                    ca.out = a.out;
                    ca.final_out = a.final_out;
                    ca.out_perm = a.out_perm;
                    ca.add = a.add;
                    ca.coef = a.coef;
                    ca.ctrl = ctrl;
                    ca.trace = upper ? c->ntrace_u : c->ntrace_l;
                    static const unsigned spin = getenv("EXG_CHAIN_SPIN") ? (unsigned)atoi(getenv("EXG_CHAIN_SPIN")) : 0u;
                    ca.spin_ns = spin;
                    // a failed launch would leave the sentinels in place and
                    // every later kernel waiting: fail loudly instead
                    ck(exg::dev::trsv_chain(c->L(), upper, ca), "chain launch");
                    sbuf_dev += ch.n_rows;
                    continue;
                }
                if (run.b <= run.a) continue;
                a.tasks = tasks + run.a;
                a.n_tasks = run.b - run.a;
                a.meta = c->meta[tri];
                ck(exg::dev::trsv_wide(c->L(), upper, a), "wide solve launch");
            }
            if (run_timing) {
                cudaEvent_t e;
                cudaEventCreate(&e);
                cudaEventRecord(e, c->stream);
                rev.push_back(e);
                cudaStreamSynchronize(c->stream);
                fprintf(stderr, "[%c runs]", upper ? 'U' : 'L');
                for (size_t i = 0; i + 1 < rev.size(); ++i) {
                    float ms = 0.f;
                    cudaEventElapsedTime(&ms, rev[i], rev[i + 1]);
                    const TriPlan::Run& run = P.runs[i];
                    if (run.narrow == 3)
                        fprintf(stderr, " S[%d comps, %lld rows, depth<=%d]:%.3fms", P.sub.n_comps, P.sub.rows,
                                P.sub.max_levels, ms);
                    else if (run.narrow == 2)
                        fprintf(stderr, " C[%d rows, %d blocks]:%.3fms", P.chains[run.a].n_rows,
                                P.chains[run.a].n_blocks, ms);
                    else
                        fprintf(stderr, " W[%d tasks]:%.3fms", run.b - run.a, ms);
                }
                fprintf(stderr, "\n");
                for (auto e : rev) cudaEventDestroy(e);
            }
        }
        if (fast) pbuf_dev += c->plan[tri].chain_slots;
        c->prof_end(upper ? EXG_K_TRSV_U : EXG_K_TRSV_L, e0);
    }
    c->cnt.trsv_calls++;
}

// y = P^T L U Q^T x (and its norm) over the EXACT task lists
void apply_dev(exg_ctx* c, const double* x, double* y_out, exg::dev::Ctrl* ctrl, double* weight_out) {
    exg::dev::apply_tasks(c->L(), c->tasks[1], c->n_tasks[1], c->u_order, c->tasks[0], c->n_tasks[0],
                          c->l_order, c->u_ptr, c->u_col, c->u_val, c->u_diag, c->l_ptr, c->l_col,
                          c->l_val, c->n, c->col_perm, c->row_perm, x, c->tmp, c->t3, c->v1, y_out,
                          c->partials, c->done, ctrl, c->V, c->ldv, weight_out);
}

void sync_ctrl(exg_ctx* c) {
    ck(cudaMemcpyAsync(c->h_ctrl, c->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, c->stream), "ctrl d2h");
    ck(cudaStreamSynchronize(c->stream), "ctrl sync");
}

exg_status ctrl_status(exg_ctx* c) {
    const Ctrl& h = *c->h_ctrl;
    switch (h.status) {
        case 0: return EXG_OK;
        case 2: throw ApiError{EXG_E_NONFINITE, "dense_expm: non-finite entry"};
        case 3: throw ApiError{EXG_E_SINGULAR, "dense_solve: singular matrix"};
        case 4: throw ApiError{EXG_E_ZERO_START, "mevp: zero start vector"};
        case 5: {
            char buf[128];
            snprintf(buf, sizeof buf, "mevp: dimension cap reached, last residual %f", h.last_residual);
            throw ApiError{EXG_E_NO_CONVERGENCE, buf};
        }
        case 6: throw ApiError{EXG_E_SINGULAR_REDUCED, "mevp: invariant subspace with singular reduced matrix"};
        default: throw ApiError{EXG_E_CONTRACT, "mevp: unknown device status"};
    }
}

// Arnoldi MEVP on the device (arnoldi_mevp, krylov.cpp:103-173).  v: device
// start vector.  er_mode: apply the er_eval early-out with ||x_k||_inf of xk.
// Returns with h_ctrl synchronised.
void mevp_dev(exg_ctx* c, const double* v, double h, const exg_mevp_cfg& cfg, int er_mode,
              const double* xk) {
    require_factors(c);
    const DCsr& C = mat(c, EXG_MAT_C);
    if (cfg.m_max < 1) throw ApiError{EXG_E_CONTRACT, "mevp: m_max must be >= 1"};
    if (h < 0.0) throw ApiError{EXG_E_CONTRACT, "mevp: negative step size"};
    ensure_krylov(c, cfg.m_max);
    const int n = c->n;
    c->basis_valid = false;
    // configuration part of the control block
    Ctrl& hc = *c->h_ctrl;
    std::memset(&hc, 0, sizeof(Ctrl));
    hc.h = h;
    hc.eps = cfg.eps;
    hc.breakdown_tol = cfg.breakdown_tol;
    hc.m_max = cfg.m_max;
    hc.check_stride = cfg.check_stride > 0 ? cfg.check_stride : 1;
    ck(cudaMemcpyAsync(c->ctrl, &hc, sizeof(Ctrl), cudaMemcpyHostToDevice, c->stream), "ctrl h2d");
    auto L = c->L();
    exg::dev::start(L, v, xk, n, c->partials, c->V, c->ctrl, er_mode);
    c->cnt.mevp_calls++;

    // MGS launch shape: 1024-thread blocks, K register elements per thread
    int K = 1, blocks = 1;
    {
        const int ks[] = {1, 2, 4, 8, 16};
        for (int kk : ks) {
            K = kk;
            const int occ = std::max(1, exg::dev::mgs_max_blocks(kk));
            const long long cap = (long long)c->num_sms * occ;
            blocks = (int)std::min<long long>(cap, ((long long)n + 1024LL * kk - 1) / (1024LL * kk));
            if ((long long)blocks * 1024 * kk >= n) break;
        }
        if ((long long)blocks * 1024 * K < n) throw ApiError{EXG_E_CONTRACT, "vector too long for the MGS kernel"};
        blocks = std::min(blocks, 4096);
    }
    exg::dev::MgsArgs ma{n, c->ldv, c->V, c->w, c->hbar, c->hld, c->partials + c->mgs_partials_off, c->bar, c->ctrl};
    // FAST mode: grouped Gram-Schmidt with streamed basis tiles (k_mgs2);
    // EXG_MGS=1 keeps the column-by-column kernel, EXG_MGS_B sets the group size
    exg::dev::Mgs2Shape ms{};
    static const bool mgs_v1 = getenv("EXG_MGS") && atoi(getenv("EXG_MGS")) == 1;
    static const int mgs_b = getenv("EXG_MGS_B") ? atoi(getenv("EXG_MGS_B")) : 0;
    const bool use_mgs2 = c->opt.trsv_mode == EXG_TRSV_FAST && !mgs_v1 && exg::dev::mgs2_shape(n, c->num_sms, mgs_b, &ms);
    if (use_mgs2) ensure_mgs_slots(c, cfg.m_max);
    exg::dev::Mgs2Args ma2{n, c->ldv, c->V, c->w, c->hbar, c->hld, c->mgs_slots ? c->mgs_slots + 8 : nullptr,
                           reinterpret_cast<unsigned int*>(c->mgs_slots), c->ctrl, c->mgs_inst_cap, 0, 0, 0};
    exg::dev::DenseArgs da{c->ctrl, c->hbar, c->hld, c->hinv, c->coef, c->dscratch, 0, 0, h, nullptr};
    const bool gspmv = c->opt.weight_mode == EXG_WEIGHT_GSPMV;
    if (gspmv) mat(c, EXG_MAT_G);
    static const bool side_ok = !(getenv("EXG_NO_FORK") && atoi(getenv("EXG_NO_FORK")));
    // one Arnoldi iteration (krylov.cpp:118-168); every kernel takes j, m and
    // the stop decision from the control block, so the same launches serve
    // the eager loop and the graph body.  dense_m bounds the dimension the
    // dense kernel will see (sizes its shared memory).
    auto iteration = [&](int dense_m, unsigned long long cond) {
        // w = -G^{-1}(C v_j)   (krylov.cpp:120-121)
        cudaEvent_t p0 = c->prof_begin();
        if (c->opt.trsv_mode == EXG_TRSV_FAST)
            exg::dev::spmv_v4(L, C.rowptr, C.col, C.val, C.n_rows, C.max_strip, c->t, c->ctrl, c->V, c->ldv);
        else
            exg::dev::spmv(L, C.rowptr, C.col, C.val, C.n_rows, nullptr, c->t, c->ctrl, c->V, c->ldv);
        c->prof_end(EXG_K_SPMV, p0);
        solve_dev(c, c->t, c->w, -1.0, nullptr, c->ctrl);
        cudaEvent_t p1 = c->prof_begin();
        if (use_mgs2)
            ck(exg::dev::mgs2(L, ma2, ms), "mgs2 launch");
        else
            ck(exg::dev::mgs(L, ma, blocks, K), "mgs launch");
        c->prof_end(EXG_K_MGS, p1);
        // the dense block (one CTA, latency-bound) and the residual weight (a
        // streaming pass over G or the factors) only share the iteration's
        // control block fields they each own: they run side by side, the
        // weight on the side stream (forked and joined through events, which
        // the graph capture records as parallel branches)
        const bool fork = !c->profiling && gspmv && side_ok;
        if (fork) {
            ck(cudaEventRecord(c->ev_fork, c->stream), "fork");
            ck(cudaStreamWaitEvent(c->side_stream, c->ev_fork, 0), "fork");
        }
        cudaEvent_t p2 = c->prof_begin();
        exg::dev::dense(L, da, dense_m);
        c->prof_end(EXG_K_DENSE, p2);
        cudaEvent_t p3 = c->prof_begin();
        if (gspmv) {
            const DCsr& G = c->mats[EXG_MAT_G];
            exg::dev::Launch Ls = L;
            if (fork) Ls.stream = c->side_stream;
            exg::dev::spmv_norm(Ls, G.rowptr, G.col, G.val, n, c->V, c->ldv, c->partials, c->done,
                                c->ctrl, fork ? 2 : 1, nullptr);
            if (fork) {
                ck(cudaEventRecord(c->ev_join, c->side_stream), "join");
                ck(cudaStreamWaitEvent(c->stream, c->ev_join, 0), "join");
            }
        } else {
            apply_dev(c, nullptr, nullptr, c->ctrl, nullptr);
        }
        exg::dev::iter_end(L, c->ctrl, cond);
        c->prof_end(EXG_K_WEIGHT, p3);
    };
    sync_ctrl(c);  // start-vector decisions (early-out, zero start)
    if (hc.status == 0 && !hc.converged) {
        if (c->opt.loop_mode == EXG_LOOP_GRAPH && !c->profiling) {
            // the whole loop as one graph launch: WHILE node, body = one
            // iteration, condition set by k_iter_end on the device
            exg_ctx::GraphKey key{};
            const DCsr& G = c->mats[EXG_MAT_G];
            const void* ps[] = {C.rowptr, C.col, C.val, G.rowptr, G.col, G.val, c->V, c->w, c->t,
                                c->hbar, c->hinv, c->coef, c->dscratch, c->partials, c->bar,
                                c->done, c->ctrl, c->trsv_buf, c->l_ptr, c->u_ptr, c->tmp, c->t3,
                                c->v1, c->mgs_slots};
            static_assert(sizeof(ps) / sizeof(ps[0]) <= 24, "graph key");
            for (size_t i = 0; i < sizeof(ps) / sizeof(ps[0]); ++i) key.p[i] = ps[i];
            const long long vs[] = {n, c->ldv, use_mgs2 ? -ms.B : blocks, K, cfg.m_max, c->opt.trsv_mode,
                                    c->opt.weight_mode, C.n_rows};
            for (size_t i = 0; i < 8; ++i) key.v[i] = vs[i];
            exg_ctx::ArnoldiGraph* g = nullptr;
            for (auto& e : c->graphs)
                if (!std::memcmp(&e.key, &key, sizeof key)) g = &e;
            if (!g) {
                exg_ctx::ArnoldiGraph ng;
                ng.key = key;
                ck(cudaGraphCreate(&ng.graph, 0), "graph create");
                cudaGraphConditionalHandle hnd;
                ck(cudaGraphConditionalHandleCreate(&hnd, ng.graph, 1, cudaGraphCondAssignDefault),
                   "conditional handle");
                cudaGraphNodeParams np{};
                np.type = cudaGraphNodeTypeConditional;
                np.conditional.handle = hnd;
                np.conditional.type = cudaGraphCondTypeWhile;
                np.conditional.size = 1;
                cudaGraphNode_t node;
                ck(cudaGraphAddNode(&node, ng.graph, nullptr, 0, &np), "conditional node");
                cudaGraph_t body = np.conditional.phGraph_out[0];
                const long long l0 = c->launches;
                ck(cudaStreamBeginCaptureToGraph(c->stream, body, nullptr, nullptr, 0,
                                                 cudaStreamCaptureModeThreadLocal), "begin capture");
                c->capturing = true;
                try {
                    iteration(cfg.m_max, (unsigned long long)hnd);
                } catch (...) {
                    c->capturing = false;
                    cudaGraph_t junk;
                    cudaStreamEndCapture(c->stream, &junk);
                    cudaGraphDestroy(ng.graph);
                    throw;
                }
                c->capturing = false;
                cudaGraph_t captured;
                ck(cudaStreamEndCapture(c->stream, &captured), "end capture");
                ng.body_kernels = c->launches - l0;
                c->launches = l0;
                ck(cudaGraphInstantiate(&ng.exec, ng.graph, 0), "graph instantiate");
                c->cnt.graph_builds++;
                c->graphs.push_back(ng);
                g = &c->graphs.back();
            }
            ck(cudaGraphLaunch(g->exec, c->stream), "graph launch");
            c->cnt.graph_launches++;
            sync_ctrl(c);
            c->cnt.arnoldi_iters += hc.arnoldi_iters;
            c->launches += g->body_kernels * hc.arnoldi_iters;
            c->cnt.mgs_passes += hc.mgs_passes;
            c->cnt.reorths += hc.reorths;
        } else {
            for (int jj = 0; jj < cfg.m_max; ++jj) {
                iteration(jj + 1, 0);
                c->cnt.arnoldi_iters++;
                sync_ctrl(c);
                if (hc.status || hc.converged) break;
            }
            c->cnt.mgs_passes += hc.mgs_passes;
            c->cnt.reorths += hc.reorths;
        }
    }
    ctrl_status(c);
    if (hc.skip) return;
    // result at h: beta V_m e^{hH^-1} e_1 (krylov.cpp:170-171)
    hc.h_sub = h;
    ck(cudaMemcpyAsync(&c->ctrl->h_sub, &h, sizeof(double), cudaMemcpyHostToDevice, c->stream), "h_sub");
    da.mode = 1;
    da.h_eval = h;
    exg::dev::dense(L, da, hc.m);
    c->basis_valid = true;
}

double* resolve_in(exg_ctx* c, const double* p, size_t count, int ptr_kind, double* staging) {
    if (ptr_kind == EXG_PTR_DEVICE) return const_cast<double*>(p);
    ck(cudaMemcpyAsync(staging, p, count * sizeof(double), cudaMemcpyHostToDevice, c->stream), "h2d");
    return staging;
}

void deliver(exg_ctx* c, double* user, const double* dev, size_t count, int ptr_kind) {
    if (ptr_kind == EXG_PTR_DEVICE) {
        if (user != dev)
            ck(cudaMemcpyAsync(user, dev, count * sizeof(double), cudaMemcpyDeviceToDevice, c->stream), "d2d");
    } else {
        ck(cudaMemcpyAsync(user, dev, count * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "d2h");
        ck(cudaStreamSynchronize(c->stream), "d2h sync");
    }
}

// Splits a triangle's level sequence into runs (see k_trsv_narrow) and builds
// the re-encoded narrow-row arrays.
void plan_triangle(exg_ctx* c, TriPlan& P, bool upper_tri, const std::vector<int>& ord,
                   const std::vector<int>& level, int nl, const std::vector<int>& ptr,
                   const std::vector<int>& col, const std::vector<double>& val,
                   const std::vector<int2>& tasks, const std::vector<double>* udiag,
                   const int* out_perm, int sub_level) {
    const int n = (int)ord.size();
    P.free_dev();
    P.runs.clear();
    const char* env_t = getenv(upper_tri ? "EXG_NARROW_T_U" : "EXG_NARROW_T_L");
    if (!env_t) env_t = getenv("EXG_NARROW_T");
    const int T = env_t ? atoi(env_t) : (upper_tri ? 64 : 48);  // swept at 1M (profiles/r01)
    const char* env_r = getenv("EXG_ABSORB_ROWS");
    const long long absorb_rows = env_r ? atoll(env_r) : 8192;
    std::vector<int> cnt(nl, 0), lpos(nl + 1, 0);
    for (int r = 0; r < n; ++r) cnt[level[r]]++;
    for (int l = 0; l < nl; ++l) lpos[l + 1] = lpos[l] + cnt[l];
    std::vector<int> tfirst(nl + 1, (int)tasks.size());
    for (int i = (int)tasks.size() - 1; i >= 0; --i) tfirst[level[ord[tasks[i].x]]] = i;
    for (int l = nl - 1; l >= 0; --l) tfirst[l] = std::min(tfirst[l], tfirst[l + 1]);
    std::vector<int> pos_of(n);
    for (int p = 0; p < n; ++p) pos_of[ord[p]] = p;
    struct ChainRun {
        int pos0, rows, blk0, nblocks, ent0, task0 = 0, ntasks = 0, slot0 = 0, slots = 0;
    };
    constexpr int kChunk = 256;  // entries per worker task (8 per lane)
    std::vector<int> cpslot;     // per chain position: first partial-sum slot (run-local)
    std::vector<int2> crq;       // per chain position: (row, output position of the fused epilogue)
    int slot_total = 0;
    std::vector<int4> ctasks;
    const char* ko = getenv("EXG_CHAIN_OLD");
    const int kOld = ko ? std::max(atoi(ko), 5) : 8;  // recent window k-8..k-5: <= 256 entries, one prefetched batch
    std::vector<ChainRun> cruns;
    std::vector<int> crows, cnptr, cncol;
    std::vector<int4> cblocks;
    std::vector<double> cnval, pool;
    constexpr int kB = 64;
    std::vector<double> Dm(kB * kB), Em(kB * kB), E2(kB * kB), E3(kB * kB), E4(kB * kB), Di(kB * kB), Fm(kB * kB);
    auto diag_of = [&](int r) { return udiag ? (*udiag)[r] : 1.0; };
    // level classes, then absorb short wide stretches into the narrow runs
    // (a launch costs more than a few fat levels on the cluster)
    std::vector<char> is_narrow(nl);
    for (int q = 0; q < nl; ++q) is_narrow[q] = T > 0 && cnt[q] <= T;
    if (sub_level >= 0) is_narrow[sub_level] = 2;  // the subtree phase: a run of its own
    {
        int q = 0;
        while (q < nl) {
            int q1 = q;
            while (q1 < nl && is_narrow[q1] == is_narrow[q]) ++q1;
            long long rows_in = lpos[q1] - lpos[q];
            if (!is_narrow[q] && T > 0 && rows_in < absorb_rows)
                for (int z = q; z < q1; ++z) is_narrow[z] = 1;
            q = q1;
        }
    }
    int l = 0;
    while (l < nl) {
        const bool narrow = is_narrow[l];
        int l1 = l;
        while (l1 < nl && is_narrow[l1] == narrow) ++l1;
        if (is_narrow[l] != 2 && lpos[l1] == lpos[l]) {  // empty stretch (no rows)
            l = l1;
            continue;
        }
        TriPlan::Run run{};
        run.narrow = narrow;
        if (is_narrow[l] == 2) {
            run.narrow = 3;  // subtree phase (P.sub)
            l1 = l + 1;
        } else if (!narrow) {
            run.a = tfirst[l];
            run.b = tfirst[l1];
        } else {
            // chain + workers: blocks of kB positions over the whole run
            run.narrow = 2;
            run.a = (int)cruns.size();
            const int p0 = lpos[l], pc = lpos[l1] - lpos[l];
            ChainRun cr;
            cr.pos0 = (int)crows.size();
            cnptr.push_back(0);  // leading 0 of this run's row offsets (cnptr index = pos0 + run index)
            cr.rows = pc;
            cr.blk0 = (int)cblocks.size() / 3;
            cr.ent0 = (int)cncol.size();
            const int nblk = (pc + kB - 1) / kB;
            cr.nblocks = nblk;
            std::vector<std::pair<int, int4>> wt;  // (start block, task)
            for (int kb = 0; kb < nblk; ++kb) {
                const int bs = p0 + kb * kB;
                const int bc = std::min(kB, p0 + pc - bs);
                // the chain itself handles blocks k-1..k-3 (F1..F3); the
                // workers' "recent" tasks blocks k-kOld..k-4, chunks the rest
                const int ps1 = kb >= 1 ? bs - kB : bs;
                const int ps2 = kb >= 2 ? bs - 2 * kB : ps1;
                const int ps3 = kb >= 3 ? bs - 3 * kB : ps2;
                const int ps4 = kb >= 4 ? bs - 4 * kB : ps3;
                std::fill(Dm.begin(), Dm.end(), 0.0);
                std::fill(Em.begin(), Em.end(), 0.0);
                std::fill(E2.begin(), E2.end(), 0.0);
                std::fill(E3.begin(), E3.end(), 0.0);
                std::fill(E4.begin(), E4.end(), 0.0);
                bool d_ident = true, e1_zero = true, e2_zero = true, e3_zero = true, e4_zero = true;
                const int pso = kb >= kOld ? bs - kOld * kB : p0;  // first position of block k-kOld
                for (int i = 0; i < bc; ++i) {
                    const int p = bs + i;
                    const int r = ord[p];
                    crows.push_back(r);
                    crq.push_back(make_int2(r, out_perm ? out_perm[r] : 0));
                    Dm[i * kB + i] = diag_of(r);
                    if (Dm[i * kB + i] != 1.0) d_ident = false;
                    std::vector<std::pair<int, double>> recv;
                    std::vector<std::pair<int, int>> oldk;  // (position, k)
                    for (int k = ptr[r]; k < ptr[r + 1]; ++k) {
                        const int pq = pos_of[col[k]];
                        if (pq < pso) {
                            oldk.push_back({pq, k});
                        } else if (pq < ps4) {
                            recv.push_back({col[k], val[k]});
                        } else if (pq < ps3) {
                            E4[i * kB + (pq - ps4)] = val[k];
                            e4_zero = false;
                        } else if (pq < ps2) {
                            E3[i * kB + (pq - ps3)] = val[k];
                            e3_zero = false;
                        } else if (pq < ps1) {
                            E2[i * kB + (pq - ps2)] = val[k];
                            e2_zero = false;
                        } else if (pq < bs) {
                            Em[i * kB + (pq - ps1)] = val[k];
                            e1_zero = false;
                        } else {
                            Dm[i * kB + (pq - bs)] = val[k];
                            d_ident = false;
                        }
                    }
                    const int pl = (int)crows.size() - 1 - cr.pos0;  // run-local position
                    // old entries by age, cut into chunks of <= kChunk: one
                    // worker task per chunk, scheduled by its newest entry
                    // (entries of earlier launches are final at kernel start),
                    // each writing its own partial-sum slot
                    std::sort(oldk.begin(), oldk.end());
                    const int nch = (int)((oldk.size() + kChunk - 1) / kChunk);
                    cpslot.push_back(cr.slots);
                    for (int q = 0; q < nch; ++q) {
                        const int a0 = q * kChunk, a1 = std::min((int)oldk.size(), a0 + kChunk);
                        const int e0 = (int)cncol.size() - cr.ent0;
                        for (int z = a0; z < a1; ++z) {
                            cncol.push_back(col[oldk[z].second]);
                            cnval.push_back(val[oldk[z].second]);
                        }
                        const int e1 = (int)cncol.size() - cr.ent0;
                        const int newest = oldk[a1 - 1].first;
                        const int key = newest < p0 ? 0 : (newest - p0) / kB;
                        wt.push_back({key, make_int4(cr.slots + q, e0, e1, 0)});
                    }
                    cr.slots += nch;
                    const int e1 = (int)cncol.size() - cr.ent0;
                    for (auto& e : recv) {
                        cncol.push_back(e.first);
                        cnval.push_back(e.second);
                    }
                    const int e2 = (int)cncol.size() - cr.ent0;
                    wt.push_back({std::max(0, kb - 5), make_int4(pl, e1, e2, 1 | (nch << 8))});
                    cnptr.push_back(e2);
                }
                std::fill(Di.begin(), Di.end(), 0.0);
                for (int jc = 0; jc < bc; ++jc)
                    for (int i = jc; i < bc; ++i) {
                        double sacc = (i == jc) ? 1.0 : 0.0;
                        for (int m2 = jc; m2 < i; ++m2) sacc -= Dm[i * kB + m2] * Di[m2 * kB + jc];
                        Di[i * kB + jc] = sacc / Dm[i * kB + i];
                    }
                // chain layout (k_trsv_chain): one record of 4 x 64 x 64 per
                // block, [CTA 0 half: Dinv F1 F2 F3][CTA 1 half: ...], so
                // each CTA of the chain pair fetches its 64 KB with ONE bulk
                // copy.  Half c holds rows 32c..32c+31; its thread t owns local
                // row t/8, columns (t%8)*8 .. +7, element j at j*256 + t
                // (conflict-free shared-memory reads).  Absent matrices are
                // zeros and flagged -1 in the block descriptor.
                const int rec = (int)pool.size();
                pool.resize(pool.size() + 5 * kB * kB, 0.0);
                auto put_mat = [&](const std::vector<double>& M, int q) {
                    for (int c2 = 0; c2 < 2; ++c2)
                        for (int j = 0; j < 8; ++j)
                            for (int t = 0; t < 256; ++t)
                                pool[rec + c2 * 5 * 2048 + q * 2048 + j * 256 + t] =
                                    M[(32 * c2 + (t >> 3)) * kB + (t & 7) * 8 + j];
                    return rec;
                };
                auto times_dinv = [&](const std::vector<double>& E, int q) {
                    std::fill(Fm.begin(), Fm.end(), 0.0);
                    for (int i = 0; i < bc; ++i)
                        for (int j = 0; j < kB; ++j) {
                            double sacc = 0.0;
                            for (int m2 = 0; m2 <= i; ++m2) sacc += Di[i * kB + m2] * E[m2 * kB + j];
                            Fm[i * kB + j] = sacc;
                        }
                    return put_mat(Fm, q);
                };
                const int dofs = d_ident ? -1 : put_mat(Di, 0);
                const int f1 = e1_zero ? -1 : times_dinv(Em, 1);
                const int f2 = e2_zero ? -1 : times_dinv(E2, 2);
                const int f3 = e3_zero ? -1 : times_dinv(E3, 3);
                const int f4 = e4_zero ? -1 : times_dinv(E4, 4);
                cblocks.push_back(make_int4(kb * kB, bc, f3, f4));  // .z / .w: F3 / F4 present (>= 0)
                cblocks.push_back(make_int4(dofs, f1, f2, rec));  // .w: record offset
                cblocks.push_back(make_int4(0, 0, 0, 0));
            }
            std::stable_sort(wt.begin(), wt.end(),
                             [](const std::pair<int, int4>& x, const std::pair<int, int4>& y) { return x.first < y.first; });
            cr.task0 = (int)ctasks.size();
            for (auto& w : wt) ctasks.push_back(w.second);
            cr.ntasks = (int)wt.size();
            cr.slot0 = slot_total;
            slot_total += cr.slots;
            cruns.push_back(cr);
            run.b = run.a + 1;
        }
        P.runs.push_back(run);
        l = l1;
    }
    if (!cruns.empty()) {
        P.crows = dalloc<int>(crows.size());
        P.cnptr = dalloc<int>(cnptr.size());
        P.cncol = dalloc<int>(std::max<size_t>(cncol.size(), 1));
        P.cnval = dalloc<double>(std::max<size_t>(cnval.size(), 1));
        P.cblocks = dalloc<int4>(cblocks.size());
        ck(cudaMemcpyAsync(P.crows, crows.data(), crows.size() * sizeof(int), cudaMemcpyHostToDevice, c->stream), "chain");
        ck(cudaMemcpyAsync(P.cnptr, cnptr.data(), cnptr.size() * sizeof(int), cudaMemcpyHostToDevice, c->stream), "chain");
        if (!cncol.empty()) {
            ck(cudaMemcpyAsync(P.cncol, cncol.data(), cncol.size() * sizeof(int), cudaMemcpyHostToDevice, c->stream), "chain");
            ck(cudaMemcpyAsync(P.cnval, cnval.data(), cnval.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream), "chain");
        }
        ck(cudaMemcpyAsync(P.cblocks, cblocks.data(), cblocks.size() * sizeof(int4), cudaMemcpyHostToDevice, c->stream), "chain");
        P.ctasks = dalloc<int4>(std::max<size_t>(ctasks.size(), 1));
        ck(cudaMemcpyAsync(P.ctasks, ctasks.data(), ctasks.size() * sizeof(int4), cudaMemcpyHostToDevice, c->stream), "chain");
        P.crq = dalloc<int2>(std::max<size_t>(crq.size(), 1));
        ck(cudaMemcpyAsync(P.crq, crq.data(), crq.size() * sizeof(int2), cudaMemcpyHostToDevice, c->stream), "chain");
        P.cpslot = dalloc<int>(std::max<size_t>(cpslot.size(), 1));
        ck(cudaMemcpyAsync(P.cpslot, cpslot.data(), cpslot.size() * sizeof(int), cudaMemcpyHostToDevice, c->stream), "chain");
        P.pool = dalloc<double>(std::max<size_t>(pool.size(), 1));
        if (!pool.empty())
            ck(cudaMemcpyAsync(P.pool, pool.data(), pool.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream), "chain");
        // run-local views: the nptr index of position j of run q is pos0 + q + j
        for (size_t q = 0; q < cruns.size(); ++q) {
            TriPlan::Chain ch;
            ch.rows_off = cruns[q].pos0;
            ch.nptr_off = cruns[q].pos0 + (int)q;
            ch.ent0 = cruns[q].ent0;
            ch.n_rows = cruns[q].rows;
            ch.blk0 = cruns[q].blk0;
            ch.n_blocks = cruns[q].nblocks;
            ch.task0 = cruns[q].task0;
            ch.ntasks = cruns[q].ntasks;
            ch.slot0 = cruns[q].slot0;
            ch.n_slots = cruns[q].slots;
            P.chains.push_back(ch);
            P.chain_rows += cruns[q].rows;
        }
    }
    P.chain_slots = slot_total;
    (void)c;
}

// ---- FAST subtree phase (k_trsv_sub) ----------------------------------------
// Greedy selection on a strictly-lower pattern (row i lists the rows it must
// come after): in increasing index, a row joins the phase when every row it
// lists is already in it and the union of their components plus itself stays
// within `budget` rows.  The result is closed under the listed relation and
// split into components with no edge between them.  For L the relation is
// "depends on" (L itself); for U it is "is depended on by" (U^T), so the U
// phase is closed under dependents and runs last.  Returns the component
// count; comp[r] = component id or -1.
int select_subtrees(int n, const std::vector<int>& ptr, const std::vector<int>& col, int budget,
                    std::vector<int>& comp) {
    comp.assign(n, -1);
    if (budget <= 0) return 0;
    std::vector<int> par(n), sz(n, 1);
    std::vector<char> in(n, 0);
    for (int i = 0; i < n; ++i) par[i] = i;
    auto find = [&](int x) {
        while (par[x] != x) {
            par[x] = par[par[x]];
            x = par[x];
        }
        return x;
    };
    std::vector<int> roots;
    for (int r = 0; r < n; ++r) {
        bool ok = true;
        long long tot = 1;
        roots.clear();
        for (int k = ptr[r]; k < ptr[r + 1] && ok; ++k) {
            const int c = col[k];
            if (!in[c]) {
                ok = false;
                break;
            }
            const int q = find(c);
            if (std::find(roots.begin(), roots.end(), q) == roots.end()) {
                roots.push_back(q);
                tot += sz[q];
            }
        }
        if (!ok || tot > budget) continue;
        in[r] = 1;
        for (int q : roots) par[q] = r;
        sz[r] = (int)tot;
    }
    std::vector<int> id(n, -1);
    int nc = 0;
    for (int r = 0; r < n; ++r)
        if (in[r]) {
            const int q = find(r);
            if (id[q] < 0) id[q] = nc++;
            comp[r] = id[q];
        }
    return nc;
}

void transpose_pattern(int n, const std::vector<int>& ptr, const std::vector<int>& col,
                       std::vector<int>& tp, std::vector<int>& tc) {
    tp.assign(n + 1, 0);
    for (int k = 0; k < ptr[n]; ++k) tp[col[k] + 1]++;
    for (int i = 0; i < n; ++i) tp[i + 1] += tp[i];
    tc.resize(ptr[n]);
    std::vector<int> next(tp.begin(), tp.end() - 1);
    for (int r = 0; r < n; ++r)
        for (int k = ptr[r]; k < ptr[r + 1]; ++k) tc[next[col[k]]++] = r;
}

// Device arrays of the subtree phase: per component its rows by local level
// (L: ascending row, U: descending), warp tasks within one local level, and
// each row's entries re-encoded (earlier-phase rows first as global ids, then
// component slots ascending as ~slot).  Components are issued largest first.
void build_sub(exg_ctx* c, SubPlan& P, bool upper, const std::vector<int>& comp, int ncomp,
               const std::vector<int>& ptr, const std::vector<int>& col,
               const std::vector<double>& val, const int* row_perm) {
    P.free_dev();
    if (ncomp == 0) return;
    const int n = (int)comp.size();
    std::vector<std::vector<int>> rows(ncomp);
    for (int i = 0; i < n; ++i) {
        const int r = upper ? n - 1 - i : i;  // dependencies before dependents
        if (comp[r] >= 0) rows[comp[r]].push_back(r);
    }
    std::vector<int> order(ncomp);
    for (int q = 0; q < ncomp; ++q) order[q] = q;
    std::stable_sort(order.begin(), order.end(),
                     [&](int x, int y) { return rows[x].size() > rows[y].size(); });
    std::vector<int4> comps, meta;
    std::vector<int2> tasks, clev;
    std::vector<int> ltp;
    std::vector<int> ecol, llev(n, 0), slot(n, -1);
    std::vector<double> eval;
    int max_rows = 0, max_lev = 0, max_tasks = 0;
    for (int q : order) {
        const std::vector<int>& R = rows[q];
        int nl = 0;
        for (int r : R) {
            int v = 0;
            for (int k = ptr[r]; k < ptr[r + 1]; ++k)
                if (comp[col[k]] == q) v = std::max(v, llev[col[k]] + 1);
            llev[r] = v;
            nl = std::max(nl, v + 1);
        }
        std::vector<int> byl(R);
        std::stable_sort(byl.begin(), byl.end(), [&](int x, int y) { return llev[x] < llev[y]; });
        const int pos0 = (int)meta.size();
        for (size_t i = 0; i < byl.size(); ++i) slot[byl[i]] = (int)i;
        const int task0 = (int)tasks.size();
        int g0 = -1, gc = 0, glev = -1, glg = -1;
        auto flush = [&]() {
            if (gc) tasks.push_back(make_int2(g0, gc | (glg << 8)));
            gc = 0;
        };
        clev.push_back(make_int2((int)ltp.size(), nl));
        for (size_t i = 0; i < byl.size(); ++i) {
            const int r = byl[i];
            if (i == 0 || llev[r] != llev[byl[i - 1]]) {
                flush();
                ltp.push_back((int)tasks.size());
            }
            std::vector<std::pair<int, int>> loc;  // (slot, k)
            const int k0 = (int)ecol.size();
            for (int k = ptr[r]; k < ptr[r + 1]; ++k) {
                if (comp[col[k]] == q) {
                    loc.push_back({slot[col[k]], k});
                } else {
                    ecol.push_back(col[k]);
                    eval.push_back(val[k]);
                }
            }
            std::sort(loc.begin(), loc.end());
            for (auto& e : loc) {
                ecol.push_back(~e.first);
                eval.push_back(val[e.second]);
            }
            const int k1 = (int)ecol.size();
            meta.push_back(make_int4(r, upper ? r : row_perm[r], k0, k1));
            const int len = k1 - k0;
            const int p = pos0 + (int)i;
            if (len > 32) {
                flush();
                tasks.push_back(make_int2(p, 1 | (1 << 30)));
                continue;
            }
            const int lg = len <= 4 ? 0 : len <= 8 ? 1 : len <= 16 ? 2 : 3;
            if (gc && (llev[r] != glev || lg != glg || (gc + 1) << lg > 32)) flush();
            if (!gc) {
                g0 = p;
                glev = llev[r];
                glg = lg;
            }
            ++gc;
        }
        flush();
        ltp.push_back((int)tasks.size());
        comps.push_back(make_int4(task0, (int)tasks.size() - task0, pos0, (int)R.size()));
        max_rows = std::max(max_rows, (int)R.size());
        max_tasks = std::max(max_tasks, (int)tasks.size() - task0);
        max_lev = std::max(max_lev, nl);
    }
    P.n_comps = ncomp;
    P.max_rows = (max_rows + 1) & ~1;  // keeps the int4 metadata after the slots 16-B aligned
    P.max_tasks = max_tasks;
    P.max_levels = max_lev;
    P.rows = (long long)meta.size();
    P.nnz = (long long)ecol.size();
    P.comps = dalloc<int4>(comps.size());
    P.clev = dalloc<int2>(clev.size());
    P.ltp = dalloc<int>(ltp.size());
    ck(cudaMemcpyAsync(P.clev, clev.data(), clev.size() * sizeof(int2), cudaMemcpyHostToDevice, c->stream), "sub plan");
    ck(cudaMemcpyAsync(P.ltp, ltp.data(), ltp.size() * sizeof(int), cudaMemcpyHostToDevice, c->stream), "sub plan");
    P.tasks = dalloc<int2>(tasks.size());
    P.meta = dalloc<int4>(meta.size());
    P.ecol = dalloc<int>(std::max<size_t>(ecol.size(), 1));
    P.eval = dalloc<double>(std::max<size_t>(eval.size(), 1));
    ck(cudaMemcpyAsync(P.comps, comps.data(), comps.size() * sizeof(int4), cudaMemcpyHostToDevice, c->stream), "sub plan");
    ck(cudaMemcpyAsync(P.tasks, tasks.data(), tasks.size() * sizeof(int2), cudaMemcpyHostToDevice, c->stream), "sub plan");
    ck(cudaMemcpyAsync(P.meta, meta.data(), meta.size() * sizeof(int4), cudaMemcpyHostToDevice, c->stream), "sub plan");
    if (!ecol.empty()) {
        ck(cudaMemcpyAsync(P.ecol, ecol.data(), ecol.size() * sizeof(int), cudaMemcpyHostToDevice, c->stream), "sub plan");
        ck(cudaMemcpyAsync(P.eval, eval.data(), eval.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream), "sub plan");
    }
}

}  // namespace

extern "C" {

exg_status exg_create(int device, exg_ctx** out) {
    exg_ctx* c = nullptr;
    API_BEGIN
    c = new exg_ctx();
    c->device = device;
    ck(cudaSetDevice(device), "cudaSetDevice");
    ck(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "stream");
    ck(cudaStreamCreateWithFlags(&c->side_stream, cudaStreamNonBlocking), "side stream");
    ck(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming), "event");
    cudaDeviceProp prop;
    ck(cudaGetDeviceProperties(&prop, device), "props");
    if (prop.major < 10) throw ApiError{EXG_E_CUDA, "exsim-B200 requires an sm_100a (Blackwell) GPU"};
    c->num_sms = prop.multiProcessorCount;
    {
        const char* e = getenv("EXG_CLUSTER");
        c->cluster = e ? atoi(e) : 16;
    }
    c->bar = dalloc<unsigned int>(4);
    c->done = dalloc<unsigned int>(4);
    ck(cudaMemsetAsync(c->bar, 0, 4 * sizeof(unsigned int), c->stream), "memset");
    ck(cudaMemsetAsync(c->done, 0, 4 * sizeof(unsigned int), c->stream), "memset");
    ck(cudaStreamSynchronize(c->stream), "memset sync");
    c->weight = dalloc<double>(4);
    c->ctrl = static_cast<Ctrl*>(static_cast<void*>(dalloc<char>(exg::dev::ctrl_size())));
    void* hp = nullptr;
    ck(cudaMallocHost(&hp, exg::dev::ctrl_size()), "cudaMallocHost");
    c->h_ctrl = static_cast<Ctrl*>(hp);
    std::memset(c->h_ctrl, 0, exg::dev::ctrl_size());
    *out = c;
    return EXG_OK;
    }
    catch (const CudaError& e) {
        if (c) exg_destroy(c);
        *out = nullptr;
        return EXG_E_CUDA;
    }
    catch (const ApiError& e) {
        if (c) exg_destroy(c);
        *out = nullptr;
        return e.st;
    }
}

void exg_destroy(exg_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    c->clear_graphs();
    for (DCsr& m : c->mats) {
        dfree(m.rowptr);
        dfree(m.col);
        dfree(m.val);
    }
    int* ip[] = {c->l_ptr, c->l_col, c->u_ptr, c->u_col, c->row_perm, c->col_perm, c->l_order, c->u_order, c->probe_idx};
    for (int* p : ip)
        if (p) cudaFree(p);
    double* dp[] = {c->l_val, c->u_val, c->u_diag, c->vin, c->vout, c->t, c->w, c->xk, c->xnext,
                    c->gb, c->startv, c->v1, c->t1, c->t2, c->t3, c->tmp, c->u_k, c->u_k1, c->V,
                    c->hbar, c->hinv, c->coef, c->dscratch, c->partials, c->weight, c->probe_out,
                    c->mgs_slots};
    for (double* p : dp)
        if (p) cudaFree(p);
    if (c->trsv_buf) cudaFree(c->trsv_buf);
    for (int q = 0; q < 4; ++q)
        if (c->tasks[q]) cudaFree(c->tasks[q]);
    c->plan[0].free_dev();
    c->plan[1].free_dev();
    if (c->meta[0]) cudaFree(c->meta[0]);
    if (c->meta[1]) cudaFree(c->meta[1]);
    if (c->bar) cudaFree(c->bar);
    if (c->done) cudaFree(c->done);
    if (c->ctrl) cudaFree(c->ctrl);
    if (c->h_ctrl) cudaFreeHost(c->h_ctrl);
    {
        double* dq[] = {c->mos_par, c->mos_op, c->mos_r, c->Fk, c->dF, c->nw, c->nu, c->nv,
                        c->aux.V, c->aux.hbar, c->aux.hinv, c->aux.coef, c->aux.dscratch,
};
        for (double* p : dq)
            if (p) cudaFree(p);
        if (c->mos_nodes) cudaFree(c->mos_nodes);
        if (c->node_ptr) cudaFree(c->node_ptr);
        if (c->node_list) cudaFree(c->node_list);
        if (c->aux.ctrl) cudaFree(c->aux.ctrl);
        if (c->aux.h_ctrl) cudaFreeHost(c->aux.h_ctrl);
    }
    for (auto& pe : c->prof_events) {
        cudaEventDestroy(pe.second.first);
        cudaEventDestroy(pe.second.second);
    }
    for (cudaEvent_t e : c->event_pool) cudaEventDestroy(e);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    if (c->side_stream) cudaStreamDestroy(c->side_stream);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

exg_status exg_last_error(exg_ctx* c, char* buf, size_t len) {
    if (!c) return EXG_E_CONTRACT;
    if (buf && len) {
        std::strncpy(buf, c->err.c_str(), len - 1);
        buf[len - 1] = 0;
    }
    return c->last;
}

exg_status exg_set_options(exg_ctx* c, const exg_options_dev* o) {
    if (!c || !o) return EXG_E_CONTRACT;
    c->opt = *o;
    return EXG_OK;
}

exg_status exg_set_csr(exg_ctx* c, int which, int n_rows, int n_cols, int nnz, const int* rowptr,
                       const int* col, const double* val) {
    API_BEGIN
    if (which < 0 || which > 2 || n_rows < 0 || n_cols < 0 || nnz < 0 || rowptr[n_rows] != nnz)
        throw ApiError{EXG_E_CONTRACT, "exg_set_csr: bad matrix"};
    c->clear_graphs();
    upload_csr(c, c->mats[which], n_rows, n_cols, nnz, rowptr, col, val);
    if (which == EXG_MAT_B) ensure_inputs(c, n_cols);
    API_END(c)
}

exg_status exg_update_values(exg_ctx* c, int which, const double* val) {
    API_BEGIN
    const DCsr& m = mat(c, which);
    ck(cudaMemcpyAsync(m.val, val, sizeof(double) * m.nnz, cudaMemcpyHostToDevice, c->stream), "update values");
    ck(cudaStreamSynchronize(c->stream), "upload sync");  // host buffers may be released on return
    API_END(c)
}

exg_status exg_set_factors(exg_ctx* c, int n, const int* Lp, const int* Li, const double* Lx,
                           const int* Up, const int* Ui, const double* Ux, const int* row_perm,
                           const int* col_perm) {
    API_BEGIN
    if (n <= 0) throw ApiError{EXG_E_CONTRACT, "exg_set_factors: empty factorization"};
    c->clear_graphs();
    // split: L strictly lower (c < r; the unit diagonal is implicit, as
    // Factorization::solve skips c >= r), U strictly upper + diagonal
    std::vector<int> lp(n + 1, 0), up(n + 1, 0);
    std::vector<int> lc, uc;
    std::vector<double> lv, uv, ud(n, 0.0);
    lc.reserve(Lp[n]);
    lv.reserve(Lp[n]);
    uc.reserve(Up[n]);
    uv.reserve(Up[n]);
    for (int r = 0; r < n; ++r) {
        for (int k = Lp[r]; k < Lp[r + 1]; ++k)
            if (Li[k] < r) {
                lc.push_back(Li[k]);
                lv.push_back(Lx[k]);
            }
        lp[r + 1] = (int)lc.size();
        for (int k = Up[r]; k < Up[r + 1]; ++k) {
            if (Ui[k] == r)
                ud[r] = Ux[k];
            else if (Ui[k] > r) {
                uc.push_back(Ui[k]);
                uv.push_back(Ux[k]);
            }
        }
        up[r + 1] = (int)uc.size();
    }
    // level analysis and level-ordered row lists.  Two valid schedules per
    // triangle: ASAP (level = longest dependency chain below the row) and
    // ALAP (level = critical path - longest chain of dependents above it).
    // Both have the same depth; they differ in where the thin levels fall.
    // With a symmetric pattern ALAP of U mirrors ASAP of L: the separator
    // chains become one long thin stretch (handled on one CTA, pick_schedule)
    // instead of thin levels interleaved with thousands of half-wide ones.
    // mask: component id per row (>= 0: the row belongs to the FAST subtree
    // phase, scheduled separately), or null; masked rows and every entry
    // touching them are left out of the level analysis
    const std::vector<int>* mask = nullptr;
    auto masked = [&](int r) { return mask && (*mask)[r] >= 0; };
    auto asap = [&](bool upper_tri, std::vector<int>& lv_) {
        const std::vector<int>& p_ = upper_tri ? up : lp;
        const std::vector<int>& c_ = upper_tri ? uc : lc;
        lv_.assign(n, 0);
        int nl = 0;
        for (int i = 0; i < n; ++i) {
            const int r = upper_tri ? n - 1 - i : i;
            if (masked(r)) continue;
            int v = 0;
            for (int k = p_[r]; k < p_[r + 1]; ++k)
                if (!masked(c_[k])) v = std::max(v, lv_[c_[k]] + 1);
            lv_[r] = v;
            nl = std::max(nl, v + 1);
        }
        return nl;
    };
    auto alap = [&](bool upper_tri, std::vector<int>& lv_) {
        const std::vector<int>& p_ = upper_tri ? up : lp;
        const std::vector<int>& c_ = upper_tri ? uc : lc;
        std::vector<int> h(n, 0);  // longest chain of dependents above the row
        int H = 0;
        for (int i = 0; i < n; ++i) {
            const int r = upper_tri ? i : n - 1 - i;  // dependents of r are already final
            if (masked(r)) continue;
            H = std::max(H, h[r]);
            for (int k = p_[r]; k < p_[r + 1]; ++k)
                if (!masked(c_[k])) h[c_[k]] = std::max(h[c_[k]], h[r] + 1);
        }
        lv_.resize(n);
        for (int r = 0; r < n; ++r) lv_[r] = masked(r) ? 0 : H - h[r];
        return H + 1;
    };
    // schedule cost model (µs): a thin level (<= 16 rows) costs one on-chip
    // hand-off on the chain CTA, a wide level one L2 hand-off plus its bytes
    auto sched_cost = [&](const std::vector<int>& lv_, int nl, bool upper_tri) {
        const std::vector<int>& p_ = upper_tri ? up : lp;
        std::vector<long long> rows(nl, 0), nz(nl, 0);
        for (int r = 0; r < n; ++r) {
            if (masked(r)) continue;
            rows[lv_[r]]++;
            nz[lv_[r]] += p_[r + 1] - p_[r];
        }
        double t = 0.0;
        for (int q = 0; q < nl; ++q)
            t += rows[q] <= 16 ? 0.2 : 0.5 + 12.0 * (double)nz[q] / 6.0e6;
        return t;
    };
    const char* sched_env = getenv("EXG_LEVELS");  // asap | alap | auto (default)
    const std::string sched = sched_env ? sched_env : "auto";
    auto pick_schedule = [&](bool upper_tri, std::vector<int>& lv_) {
        std::vector<int> a1, a2;
        const int n1 = asap(upper_tri, a1);
        if (sched == "asap") {
            lv_.swap(a1);
            return n1;
        }
        const int n2 = alap(upper_tri, a2);
        if (sched == "alap" || sched_cost(a2, n2, upper_tri) < sched_cost(a1, n1, upper_tri)) {
            lv_.swap(a2);
            c->alap[upper_tri] = 1;
            return n2;
        }
        lv_.swap(a1);
        c->alap[upper_tri] = 0;
        return n1;
    };
    auto order_by = [n](const std::vector<int>& lv_, int nl, bool desc) {
        std::vector<int> cnt(nl + 1, 0), ord(n);
        for (int r = 0; r < n; ++r) cnt[lv_[r] + 1]++;
        for (int i = 0; i < nl; ++i) cnt[i + 1] += cnt[i];
        if (!desc)
            for (int r = 0; r < n; ++r) ord[cnt[lv_[r]]++] = r;
        else
            for (int r = n - 1; r >= 0; --r) ord[cnt[lv_[r]]++] = r;
        return ord;
    };
    std::vector<int> llev, lev;
    const int l_levels = pick_schedule(false, llev);
    const int u_levels = pick_schedule(true, lev);
    const std::vector<int> lord = order_by(llev, l_levels, false);
    const std::vector<int> uord = order_by(lev, u_levels, true);
    // warp tasks over the level order: long rows alone, short rows 32 per task
    // Warp tasks over the level order.  A row with more than 32 off-diagonal
    // entries is a task of its own (whole warp); shorter rows are grouped,
    // never across two levels (no lane ever waits on a lane of its own warp),
    // with `lpr` lanes per row: 1 in EXACT mode (the reference's sequential
    // row), up to 8 in FAST mode (about 4 entries per lane).
    // task.y = rows | log2(lpr) << 8 | LONG << 30
    auto make_tasks = [](const std::vector<int>& ord, const std::vector<int>& ptr,
                         const std::vector<int>& level, bool fast) {
        std::vector<int2> tasks;
        int g0 = -1, gc = 0, glev = -1, glg = -1;
        auto flush = [&]() {
            if (gc) tasks.push_back(make_int2(g0, gc | (glg << 8)));
            gc = 0;
        };
        for (int i = 0; i < (int)ord.size(); ++i) {
            const int r = ord[i];
            if (r < 0) {  // not scheduled here (subtree phase)
                flush();
                continue;
            }
            const int len = ptr[r + 1] - ptr[r];
            if (len > 32) {
                flush();
                tasks.push_back(make_int2(i, 1 | (1 << 30)));
                continue;
            }
            int lg = 0;
            if (fast) lg = len <= 4 ? 0 : len <= 8 ? 1 : len <= 16 ? 2 : 3;
            if (gc && (level[r] != glev || lg != glg || (gc + 1) << lg > 32)) flush();
            if (!gc) {
                g0 = i;
                glev = level[r];
                glg = lg;
            }
            ++gc;
        }
        flush();
        return tasks;
    };
    const std::vector<int2> ltasks = make_tasks(lord, lp, llev, false);
    const std::vector<int2> utasks = make_tasks(uord, up, lev, false);

    // ---- FAST schedule: the subtree phase (k_trsv_sub) takes the bottom of
    // the elimination DAG (L: first, U: last); the rest is levelled without it
    const char* sr_env = getenv("EXG_SUB_ROWS");
    const int sub_rows = sr_env ? atoi(sr_env) : 0;  // off by default: measured slower at 1M
    std::vector<int> lcomp, ucomp;
    const int lncomp = select_subtrees(n, lp, lc, sub_rows, lcomp);
    std::vector<int> utp, utc;
    transpose_pattern(n, up, uc, utp, utc);  // U^T: the rows that depend on each row
    const int uncomp = select_subtrees(n, utp, utc, sub_rows, ucomp);
    std::vector<int> lflev, uflev;
    mask = &lcomp;
    int lnl_f = pick_schedule(false, lflev);
    mask = &ucomp;
    int unl_f = pick_schedule(true, uflev);
    mask = nullptr;
    int l_sub = -1, u_sub = -1;
    if (lncomp) {  // L: subtree phase = level 0, the rest after it
        for (int r = 0; r < n; ++r) lflev[r] = lcomp[r] >= 0 ? 0 : lflev[r] + 1;
        l_sub = 0;
        ++lnl_f;
    }
    if (uncomp) {  // U: the rest first, subtree phase = the last level
        for (int r = 0; r < n; ++r) uflev[r] = ucomp[r] >= 0 ? unl_f : uflev[r];
        u_sub = unl_f;
        ++unl_f;
    }
    const std::vector<int> lford = order_by(lflev, lnl_f, false);
    const std::vector<int> uford = order_by(uflev, unl_f, true);
    auto rest_only = [](const std::vector<int>& ord, const std::vector<int>& comp) {
        std::vector<int> o(ord.size());
        for (size_t i = 0; i < ord.size(); ++i) o[i] = comp[ord[i]] >= 0 ? -1 : ord[i];
        return o;
    };
    const std::vector<int2> ltasks_f = make_tasks(rest_only(lford, lcomp), lp, lflev, true);
    const std::vector<int2> utasks_f = make_tasks(rest_only(uford, ucomp), up, uflev, true);

    int* ip[] = {c->l_ptr, c->l_col, c->u_ptr, c->u_col, c->row_perm, c->col_perm, c->l_order, c->u_order};
    for (int* p : ip)
        if (p) cudaFree(p);
    dfree(c->l_val);
    dfree(c->u_val);
    dfree(c->u_diag);
    dfree(c->trsv_buf);
    c->n = n;
    auto up_i = [&](int*& d, const int* h, size_t cnt) {
        d = dalloc<int>(cnt);
        if (cnt) ck(cudaMemcpyAsync(d, h, cnt * sizeof(int), cudaMemcpyHostToDevice, c->stream), "factor upload");
    };
    auto up_d = [&](double*& d, const double* h, size_t cnt) {
        d = dalloc<double>(cnt);
        if (cnt) ck(cudaMemcpyAsync(d, h, cnt * sizeof(double), cudaMemcpyHostToDevice, c->stream), "factor upload");
    };
    up_i(c->l_ptr, lp.data(), n + 1);
    up_i(c->l_col, lc.data(), lc.size());
    up_d(c->l_val, lv.data(), lv.size());
    up_i(c->u_ptr, up.data(), n + 1);
    up_i(c->u_col, uc.data(), uc.size());
    up_d(c->u_val, uv.data(), uv.size());
    up_d(c->u_diag, ud.data(), n);
    up_i(c->row_perm, row_perm, n);
    up_i(c->col_perm, col_perm, n);
    up_i(c->l_order, lord.data(), n);
    up_i(c->u_order, uord.data(), n);
    // FAST-mode plan: runs of wide levels (warp tasks, all SMs) and of narrow
    // levels (one thread-block cluster, DSMEM hand-offs)
    // FAST plan: the blocked augmented system (default, trsv_plan.hpp), or
    // the level-run plan (wide runs + cluster chain, EXG_FAST_PLAN=chain)
    // FAST plan: per-warp record streams of the blocked augmented system
    // (k_trsv4) for large systems, whose solves stream the factors from HBM;
    // the level-run plan (wide runs + cluster chain) for small ones, where a
    // solve is a chain of hand-offs and the chain's DSMEM hops are the shortest
    // (measured: config 0 and 3 run 2-3x faster on it, config 1 on the streams)
    const char* fp_env = getenv("EXG_FAST_PLAN");  // auto (default) | stream | chain
    std::string fplan = fp_env ? fp_env : "auto";
    if (fplan != "stream" && fplan != "chain") fplan = n >= kStreamPlanMinRows ? "stream" : "chain";
    if (fplan == "stream") {
        // per-warp record streams (k_trsv4) over the augmented system with
        // every row cut to <= 128 entries
        exg::AugParams prm = exg::stream_aug_params();
        if (const char* e = getenv("EXG_AUG_BLOCK")) sscanf(e, "%d,%d", &prm.min_block, &prm.max_block);
        std::vector<int> ident(n);
        for (int i = 0; i < n; ++i) ident[i] = i;
        for (int tri = 0; tri < 2; ++tri) {
            TriPlan& P = c->plan[tri];
            P.free_dev();
            P.runs.clear();
            exg::StreamParams sp;
            sp.n_warps = exg::dev::trsv_stream_warps(tri == 1, c->num_sms);
            exg::stream_params_env(sp);
            if (const char* e = getenv("EXG_STREAM_WARPS")) {  // debug: fewer co-resident warps (a multiple of 8)
                const int wcap = atoi(e) / 8 * 8;
                if (wcap >= 8 && wcap < sp.n_warps) sp.n_warps = wcap;
            }
            if (sp.n_warps <= 0) throw ApiError{EXG_E_CUDA, "k_trsv4 cannot be launched on this device"};
            exg::StreamPlan S;
            {
                exg::AugPlan A;
                if (tri == 0)
                    exg::build_aug_plan(false, n, lp.data(), lc.data(), lv.data(), nullptr, row_perm, prm, A);
                else
                    exg::build_aug_plan(true, n, up.data(), uc.data(), uv.data(), ud.data(), ident.data(), prm, A);
                // small systems: no more warps than tasks would keep busy
                exg::build_stream_plan(A, tri == 1, tri == 1 ? col_perm : nullptr, sp, S);
                c->cnt_aug[tri][1] = A.n_blocks;
                c->cnt_aug[tri][2] = A.block_rows;
                c->cnt_aug[tri][3] = A.n_partials;
            }
            P.sdata = dalloc<unsigned char>(std::max<size_t>(S.data.size(), 16));
            P.sdesc = dalloc<int>(S.desc.size());
            ck(cudaMemcpyAsync(P.sdata, S.data.data(), S.data.size(), cudaMemcpyHostToDevice, c->stream), "stream plan");
            ck(cudaMemcpyAsync(P.sdesc, S.desc.data(), S.desc.size() * sizeof(int), cudaMemcpyHostToDevice,
                               c->stream), "stream plan");
            ck(cudaStreamSynchronize(c->stream), "stream plan sync");  // S is released below
            P.s_warps = S.n_warps;
            P.s_bytes = (long long)S.data.size();
            P.n_aug = S.n_aug;
            P.aug_levels = S.levels;
            c->cnt_aug[tri][0] = S.levels;
            c->cnt_aug[tri][4] = S.n_entries;
            c->cnt_aug[tri][5] = S.n_tasks;
            c->cnt_aug[tri][6] = (long long)S.data.size();
            c->cnt_aug[tri][7] = S.n_warps;
        }
    } else {
        plan_triangle(c, c->plan[0], false, lford, lflev, lnl_f, lp, lc, lv, ltasks_f, nullptr, nullptr, l_sub);
        plan_triangle(c, c->plan[1], true, uford, uflev, unl_f, up, uc, uv, utasks_f, &ud, col_perm, u_sub);
        build_sub(c, c->plan[0].sub, false, lcomp, lncomp, lp, lc, lv, row_perm);
        build_sub(c, c->plan[1].sub, true, ucomp, uncomp, up, uc, uv, row_perm);
    }
    {
        std::vector<int4> lm(n), um(n);
        for (int p = 0; p < n; ++p) {
            const int r = lford[p];
            lm[p] = make_int4(r, row_perm[r], lp[r], lp[r + 1]);
            const int ru = uford[p];
            um[p] = make_int4(ru, ru, up[ru], up[ru + 1]);
        }
        if (c->meta[0]) cudaFree(c->meta[0]);
        if (c->meta[1]) cudaFree(c->meta[1]);
        c->meta[0] = dalloc<int4>(n);
        c->meta[1] = dalloc<int4>(n);
        ck(cudaMemcpyAsync(c->meta[0], lm.data(), n * sizeof(int4), cudaMemcpyHostToDevice, c->stream), "meta");
        ck(cudaMemcpyAsync(c->meta[1], um.data(), n * sizeof(int4), cudaMemcpyHostToDevice, c->stream), "meta");
    }
    const std::vector<int2>* tl[4] = {&ltasks, &utasks, &ltasks_f, &utasks_f};
    for (int q = 0; q < 4; ++q) {
        if (c->tasks[q]) cudaFree(c->tasks[q]);
        c->tasks[q] = dalloc<int2>(tl[q]->size());
        ck(cudaMemcpyAsync(c->tasks[q], tl[q]->data(), tl[q]->size() * sizeof(int2), cudaMemcpyHostToDevice, c->stream), "tasks");
        c->n_tasks[q] = (int)tl[q]->size();
    }
    c->trsv_buf = dalloc<char>(kTrsvHdr + sizeof(double) * ((size_t)std::max<long long>(n, c->plan[0].n_aug + 1) +
                                                       (size_t)std::max<long long>(n, c->plan[1].n_aug + 1) +
                                                       c->plan[0].chain_rows +
                                                       c->plan[1].chain_rows + c->plan[0].chain_slots +
                                                       c->plan[1].chain_slots));
    ensure_vectors(c, n);
    c->cnt.l_levels = l_levels;
    c->cnt.u_levels = u_levels;
    c->cnt.l_schedule = c->alap[0];
    c->cnt.u_schedule = c->alap[1];
    c->cnt.nnz_l = (long long)lc.size();
    c->cnt.nnz_u = (long long)uc.size();
    const bool streams = c->plan[0].s_warps > 0;
    c->cnt.fast_levels_l = streams ? (int)c->cnt_aug[0][0] : 0;
    c->cnt.fast_levels_u = streams ? (int)c->cnt_aug[1][0] : 0;
    c->cnt.fast_tasks_l = streams ? c->cnt_aug[0][5] : 0;
    c->cnt.fast_tasks_u = streams ? c->cnt_aug[1][5] : 0;
    c->cnt.fast_bytes_l = streams ? c->cnt_aug[0][6] : 0;
    c->cnt.fast_bytes_u = streams ? c->cnt_aug[1][6] : 0;
    c->mmax_alloc = 0;  // Krylov workspace re-sized on next use
    dfree(c->V);
    c->basis_valid = false;
    ck(cudaStreamSynchronize(c->stream), "upload sync");  // host buffers may be released on return
    API_END(c)
}

exg_status exg_spmv(exg_ctx* c, int which, const double* x, double* y, int ptr_kind) {
    API_BEGIN
    const DCsr& m = mat(c, which);
    double* xs = const_cast<double*>(x);
    double* ys = y;
    double* sx = nullptr;
    double* sy = nullptr;
    if (ptr_kind == EXG_PTR_HOST) {
        sx = dalloc<double>(m.n_cols);
        sy = dalloc<double>(m.n_rows);
        ck(cudaMemcpyAsync(sx, x, sizeof(double) * m.n_cols, cudaMemcpyHostToDevice, c->stream), "h2d");
        xs = sx;
        ys = sy;
    }
    exg::dev::spmv(c->L(), m.rowptr, m.col, m.val, m.n_rows, xs, ys, nullptr, nullptr, 0);
    if (ptr_kind == EXG_PTR_HOST) {
        ck(cudaMemcpyAsync(y, sy, sizeof(double) * m.n_rows, cudaMemcpyDeviceToHost, c->stream), "d2h");
        ck(cudaStreamSynchronize(c->stream), "sync");
        dfree(sx);
        dfree(sy);
    }
    ck(cudaGetLastError(), "spmv launch");
    API_END(c)
}

exg_status exg_solve(exg_ctx* c, const double* b, double* x, int ptr_kind) {
    API_BEGIN
    require_factors(c);
    const int n = c->n;
    const double* bd = resolve_in(c, b, n, ptr_kind, c->vin);
    double* xd = ptr_kind == EXG_PTR_DEVICE ? x : c->vout;
    solve_dev(c, bd, xd, 1.0, nullptr, nullptr);
    ck(cudaGetLastError(), "solve launch");
    deliver(c, x, xd, n, ptr_kind);
    API_END(c)
}

exg_status exg_apply(exg_ctx* c, const double* x, double* y, int ptr_kind) {
    API_BEGIN
    require_factors(c);
    const int n = c->n;
    const double* xd = resolve_in(c, x, n, ptr_kind, c->vin);
    double* yd = ptr_kind == EXG_PTR_DEVICE ? y : c->vout;
    apply_dev(c, xd, yd, nullptr, c->weight);
    ck(cudaGetLastError(), "apply launch");
    deliver(c, y, yd, n, ptr_kind);
    API_END(c)
}

exg_status exg_mevp_iks(exg_ctx* c, const double* v, double h, const exg_mevp_cfg* cfg,
                        double* out, exg_mevp_info* info, int ptr_kind) {
    API_BEGIN
    require_factors(c);
    const int n = c->n;
    const double* vd = resolve_in(c, v, n, ptr_kind, c->vin);
    if (info) std::memset(info, 0, sizeof(*info));
    try {
        mevp_dev(c, vd, h, *cfg, 0, nullptr);
    } catch (const ApiError& e) {
        if (info) info->last_residual = c->h_ctrl->last_residual;
        throw;
    }
    double* od = ptr_kind == EXG_PTR_DEVICE ? out : c->vout;
    exg::dev::combine(c->L(), c->V, c->ldv, c->coef, n, od, c->ctrl, 0, nullptr, nullptr, nullptr, 0.0);
    ck(cudaGetLastError(), "mevp launch");
    deliver(c, out, od, n, ptr_kind);
    if (info) {
        const Ctrl& h_ = *c->h_ctrl;
        info->m = h_.m;
        info->happy = h_.happy;
        info->beta = h_.beta;
        info->h_next = h_.h_next;
        info->h_sub = h;
        info->last_residual = h_.last_residual;
    }
    API_END(c)
}

exg_status exg_basis_residual(exg_ctx* c, double h, double* residual) {
    API_BEGIN
    if (!c->basis_valid) throw ApiError{EXG_E_CONTRACT, "mevp_residual: empty basis"};
    const Ctrl& hc = *c->h_ctrl;
    if (hc.happy || hc.h_next == 0.0) {
        *residual = 0.0;
        return EXG_OK;
    }
    const DCsr& G = mat(c, EXG_MAT_G);
    auto L = c->L();
    exg::dev::DenseArgs da{c->ctrl, c->hbar, c->hld, c->hinv, c->coef, c->dscratch, 0, 2, h};
    exg::dev::dense(L, da, hc.m);
    exg::dev::spmv_norm(L, G.rowptr, G.col, G.val, c->n, c->V + (long long)hc.m * c->ldv, 0,
                        c->partials, c->done, nullptr, 0, c->weight);
    // weight lands in c->weight; combine on the device
    double* res = c->weight + 1;
    // ctrl->weight is not set by the free-standing norm: copy it in
    ck(cudaMemcpyAsync(&c->ctrl->weight, c->weight, sizeof(double), cudaMemcpyDeviceToDevice, c->stream), "w");
    exg::dev::basis_residual_final(L, c->ctrl, res);
    ck(cudaMemcpyAsync(residual, res, sizeof(double), cudaMemcpyDeviceToHost, c->stream), "d2h");
    sync_ctrl(c);
    ctrl_status(c);
    API_END(c)
}

exg_status exg_basis_eval(exg_ctx* c, double h, double* out, int ptr_kind) {
    API_BEGIN
    if (!c->basis_valid) throw ApiError{EXG_E_CONTRACT, "eval_at_scaled_h: empty basis"};
    if (h < 0.0 || h > c->h_ctrl->h_sub)
        throw ApiError{EXG_E_CONTRACT, "eval_at_scaled_h: h outside [0, h_sub]"};
    auto L = c->L();
    exg::dev::DenseArgs da{c->ctrl, c->hbar, c->hld, c->hinv, c->coef, c->dscratch, 0, 1, h};
    exg::dev::dense(L, da, c->h_ctrl->m);
    double* od = ptr_kind == EXG_PTR_DEVICE ? out : c->vout;
    exg::dev::combine(L, c->V, c->ldv, c->coef, c->n, od, c->ctrl, 0, nullptr, nullptr, nullptr, 0.0);
    deliver(c, out, od, c->n, ptr_kind);
    sync_ctrl(c);
    ctrl_status(c);
    API_END(c)
}

exg_status exg_er_begin(exg_ctx* c, const double* x_k, const double* u_k, const double* u_k1,
                        double h, int ptr_kind) {
    API_BEGIN
    require_factors(c);
    const DCsr& B = mat(c, EXG_MAT_B);
    const DCsr& C = mat(c, EXG_MAT_C);
    if (h <= 0.0) throw ApiError{EXG_E_CONTRACT, "er_step: step size must be positive"};
    const int n = c->n;
    const int ni = B.n_cols;
    ensure_inputs(c, ni);
    auto kind = ptr_kind == EXG_PTR_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    if (x_k != c->xk) ck(cudaMemcpyAsync(c->xk, x_k, sizeof(double) * n, kind, c->stream), "x_k");
    if (ni) {
        ck(cudaMemcpyAsync(c->u_k, u_k, sizeof(double) * ni, kind, c->stream), "u_k");
        ck(cudaMemcpyAsync(c->u_k1, u_k1, sizeof(double) * ni, kind, c->stream), "u_k1");
    }
    auto L = c->L();
    // rhs = F(x_k) + B u_k (integrate.cpp:224; F == 0 without devices) ; B slope
    const double* Fk = nullptr;
    if (c->n_mos > 0) {
        exg::dev::mos_residual(L, c->n_mos, c->mos_nodes, c->mos_par, c->mos_op, c->xk, c->mos_r, n,
                               c->node_ptr, c->node_list, c->Fk, nullptr);
        Fk = c->Fk;
    }
    exg::dev::spmv_b2(L, B.rowptr, B.col, B.val, B.n_rows, c->u_k, c->u_k1, h, c->t1, c->t2, Fk);
    if (c->opt.trsv_mode == EXG_TRSV_FAST) {
        // start = v1 + v2 = x_k - G^{-1} rhs + G^{-1} C gb = x_k + G^{-1}(C gb - rhs):
        // two solves instead of three (the same value up to rounding, which
        // FAST mode already reorders)
        solve_dev(c, c->t2, c->gb, 1.0, nullptr, nullptr);     // gb_slope = G^{-1} B slope
        exg::dev::spmv_sub(L, C.rowptr, C.col, C.val, C.n_rows, c->gb, c->t1, c->t3);
        solve_dev(c, c->t3, c->startv, 1.0, c->xk, nullptr);   // start = x_k + G^{-1}(C gb - rhs)
    } else {
        // the reference's order (integrate.cpp:224-231), bit for bit
        solve_dev(c, c->t1, c->v1, -1.0, c->xk, nullptr);      // v1 = x_k - G^{-1} rhs
        solve_dev(c, c->t2, c->gb, 1.0, nullptr, nullptr);     // gb_slope = G^{-1} B slope
        exg::dev::spmv(L, C.rowptr, C.col, C.val, C.n_rows, c->gb, c->t3, nullptr, nullptr, 0);
        solve_dev(c, c->t3, c->startv, 1.0, c->v1, nullptr);   // start = v1 + G^{-1} C gb
    }
    c->h_built = h;
    c->basis_valid = false;
    ck(cudaGetLastError(), "er_begin launch");
    API_END(c)
}

exg_status exg_er_eval(exg_ctx* c, double h_try, const exg_mevp_cfg* cfg, double* x_next,
                       int* m_out, exg_mevp_info* info, int ptr_kind) {
    API_BEGIN
    require_factors(c);
    const int n = c->n;
    bool fresh = true;
    if (c->basis_valid && h_try <= c->h_ctrl->h_sub && c->mats[EXG_MAT_G].rowptr) {
        double r = 0.0;
        exg_status st = exg_basis_residual(c, h_try, &r);
        if (st != EXG_OK) return st;
        if (r < cfg->eps) {
            auto L = c->L();
            exg::dev::DenseArgs da{c->ctrl, c->hbar, c->hld, c->hinv, c->coef, c->dscratch, 0, 1, h_try};
            exg::dev::dense(L, da, c->h_ctrl->m);
            fresh = false;
        }
    }
    if (fresh) mevp_dev(c, c->startv, h_try, *cfg, 1, c->xk);
    exg::dev::combine(c->L(), c->V, c->ldv, c->coef, n, c->xnext, c->ctrl, 1, c->xk, c->gb,
                      c->startv, h_try);
    ck(cudaGetLastError(), "er_eval launch");
    if (m_out) *m_out = (fresh && !c->h_ctrl->skip) ? c->h_ctrl->m : -1;
    if (info) {
        const Ctrl& h_ = *c->h_ctrl;
        info->m = h_.m;
        info->happy = h_.happy;
        info->beta = h_.beta;
        info->h_next = h_.h_next;
        info->h_sub = h_.h_sub;
        info->last_residual = h_.last_residual;
    }
    if (x_next) deliver(c, x_next, c->xnext, n, ptr_kind);
    API_END(c)
}

exg_status exg_er_step(exg_ctx* c, const double* x_k, const double* u_k, const double* u_k1,
                       double h, const exg_mevp_cfg* cfg, double* x_next, int* m_out,
                       int ptr_kind) {
    exg_status st = exg_er_begin(c, x_k, u_k, u_k1, h, ptr_kind);
    if (st != EXG_OK) return st;
    return exg_er_eval(c, h, cfg, x_next, m_out, nullptr, ptr_kind);
}

exg_status exg_set_devices(exg_ctx* c, int n_mos, const int* nodes4, const double* par6) {
    API_BEGIN
    require_factors(c);
    const int n = c->n;
    dfree(c->mos_par);
    dfree(c->mos_op);
    dfree(c->mos_r);
    if (c->mos_nodes) cudaFree(c->mos_nodes);
    c->mos_nodes = nullptr;
    dfree(c->node_ptr);
    dfree(c->node_list);
    c->n_mos = n_mos;
    // per-node contribution lists in device order (drain +, source -)
    std::vector<int> cnt(n + 1, 0);
    for (int i = 0; i < n_mos; ++i) {
        if (nodes4[4 * i] >= 0) cnt[nodes4[4 * i] + 1]++;
        if (nodes4[4 * i + 2] >= 0) cnt[nodes4[4 * i + 2] + 1]++;
    }
    for (int i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
    std::vector<int> list(cnt[n]), next(cnt.begin(), cnt.end() - 1);
    for (int i = 0; i < n_mos; ++i) {
        if (nodes4[4 * i] >= 0) list[next[nodes4[4 * i]]++] = i;
        if (nodes4[4 * i + 2] >= 0) list[next[nodes4[4 * i + 2]]++] = -1 - i;
    }
    c->mos_nodes = static_cast<int4*>(static_cast<void*>(dalloc<int>(4 * (size_t)std::max(n_mos, 1))));
    c->mos_par = dalloc<double>(6 * (size_t)std::max(n_mos, 1));
    c->mos_op = dalloc<double>(5 * (size_t)std::max(n_mos, 1));
    c->mos_r = dalloc<double>(std::max(n_mos, 1));
    c->node_ptr = dalloc<int>(n + 1);
    c->node_list = dalloc<int>(std::max(cnt[n], 1));
    if (n_mos) {
        ck(cudaMemcpyAsync(c->mos_nodes, nodes4, 4 * sizeof(int) * n_mos, cudaMemcpyHostToDevice, c->stream), "mos");
        ck(cudaMemcpyAsync(c->mos_par, par6, 6 * sizeof(double) * n_mos, cudaMemcpyHostToDevice, c->stream), "mos");
        ck(cudaMemsetAsync(c->mos_op, 0, 5 * sizeof(double) * n_mos, c->stream), "mos");
    }
    ck(cudaMemcpyAsync(c->node_ptr, cnt.data(), sizeof(int) * (n + 1), cudaMemcpyHostToDevice, c->stream), "mos");
    if (cnt[n]) ck(cudaMemcpyAsync(c->node_list, list.data(), sizeof(int) * cnt[n], cudaMemcpyHostToDevice, c->stream), "mos");
    double** vs[] = {&c->Fk, &c->dF, &c->nw, &c->nu, &c->nv};
    for (double** p : vs) {
        dfree(*p);
        *p = dalloc<double>(n);
    }
    if (!c->aux.ctrl) {
        c->aux.ctrl = static_cast<Ctrl*>(static_cast<void*>(dalloc<char>(exg::dev::ctrl_size())));
        void* hp = nullptr;
        ck(cudaMallocHost(&hp, exg::dev::ctrl_size()), "cudaMallocHost");
        c->aux.h_ctrl = static_cast<Ctrl*>(hp);
        std::memset(c->aux.h_ctrl, 0, exg::dev::ctrl_size());
    }
    ck(cudaStreamSynchronize(c->stream), "upload sync");  // host buffers may be released on return
    API_END(c)
}

exg_status exg_set_oppoints(exg_ctx* c, const double* op5) {
    API_BEGIN
    if (c->n_mos) ck(cudaMemcpyAsync(c->mos_op, op5, 5 * sizeof(double) * c->n_mos, cudaMemcpyHostToDevice, c->stream), "op");
    ck(cudaStreamSynchronize(c->stream), "upload sync");  // host buffers may be released on return
    API_END(c)
}

exg_status exg_residual_F(exg_ctx* c, const double* x, double* F, int ptr_kind) {
    API_BEGIN
    require_factors(c);
    if (!c->node_ptr) throw ApiError{EXG_E_CONTRACT, "residual_F: no devices (exg_set_devices)"};
    const int n = c->n;
    const double* xd = resolve_in(c, x, n, ptr_kind, c->vin);
    double* Fd = ptr_kind == EXG_PTR_DEVICE ? F : c->vout;
    exg::dev::mos_residual(c->L(), c->n_mos, c->mos_nodes, c->mos_par, c->mos_op, xd, c->mos_r, n,
                           c->node_ptr, c->node_list, Fd, nullptr);
    deliver(c, F, Fd, n, ptr_kind);
    API_END(c)
}

// nonlinear error estimate and ER-C correction of the last er_eval
// (error_from_deltaF / correction_from_deltaF, integrate.cpp:267-298, called
// as transient() does at :434-445).  x_next (device) is corrected in place.
exg_status exg_er_nonlinear(exg_ctx* c, double h, const exg_mevp_cfg* cfg, int erc, double gamma,
                            double* err_norm, int* dims, int* n_dims) {
    API_BEGIN
    require_factors(c);
    if (!c->node_ptr) throw ApiError{EXG_E_CONTRACT, "er_nonlinear: no devices (exg_set_devices)"};
    const int n = c->n;
    auto L = c->L();
    *err_norm = 0.0;
    *n_dims = 0;
    // residual_F rejects a non-finite state (devices.cpp:205): ||x_next||_inf
    // (NaN-propagating) is read back with ||deltaF||_inf
    exg::dev::absmax(L, c->xnext, n, c->partials, c->done, c->weight + 3);
    // deltaF = residual_F(x_next) - F_k
    exg::dev::mos_residual(L, c->n_mos, c->mos_nodes, c->mos_par, c->mos_op, c->xnext, c->mos_r, n,
                           c->node_ptr, c->node_list, c->dF, c->Fk);
    exg::dev::absmax(L, c->dF, n, c->partials, c->done, c->weight + 2);
    double norms[2] = {0.0, 0.0};  // ||deltaF||_inf, ||x_next||_inf
    ck(cudaMemcpyAsync(norms, c->weight + 2, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "d2h");
    ck(cudaStreamSynchronize(c->stream), "sync");
    if (!std::isfinite(norms[1])) throw ApiError{EXG_E_NONFINITE, "residual_F: non-finite state entry"};
    const double dfinf = norms[0];
    if (!std::isfinite(dfinf)) throw ApiError{EXG_E_NONFINITE, "residual_F: non-finite device residual"};
    if (dfinf == 0.0) return EXG_OK;  // both error and correction vanish
    solve_dev(c, c->dF, c->nw, 1.0, nullptr, nullptr);  // w = G^{-1} deltaF
    c->swap_krylov();
    struct Restore {
        exg_ctx* c;
        ~Restore() { c->swap_krylov(); }
    } restore{c};
    // error: e_rr = w - e^{hJ} w (skipped when ||w|| == 0)
    mevp_dev(c, c->nw, h, *cfg, 2, nullptr);
    if (!c->h_ctrl->skip) {
        dims[(*n_dims)++] = c->h_ctrl->m;
        exg::dev::combine(L, c->V, c->ldv, c->coef, n, c->nv, c->ctrl, 0, nullptr, nullptr, nullptr, 0.0);
        exg::dev::axpby(L, c->nw, -1.0, c->nv, c->nu, n);
        exg::dev::absmax(L, c->nu, n, c->partials, c->done, c->weight + 2);
        ck(cudaMemcpyAsync(err_norm, c->weight + 2, sizeof(double), cudaMemcpyDeviceToHost, c->stream), "d2h");
        ck(cudaStreamSynchronize(c->stream), "sync");
        if (!std::isfinite(*err_norm)) throw ApiError{EXG_E_NONFINITE, "error estimate: non-finite entry"};
    }
    if (erc && gamma != 0.0) {
        // u = G^{-1} C w ; d = gamma (w + (e^{hJ}u - u)/h) ; x_next += d
        const DCsr& C = mat(c, EXG_MAT_C);
        exg::dev::spmv(L, C.rowptr, C.col, C.val, C.n_rows, c->nw, c->t, nullptr, nullptr, 0);
        solve_dev(c, c->t, c->nu, 1.0, nullptr, nullptr);
        mevp_dev(c, c->nu, h, *cfg, 2, nullptr);
        int have_u = 0;
        if (!c->h_ctrl->skip) {
            dims[(*n_dims)++] = c->h_ctrl->m;
            exg::dev::combine(L, c->V, c->ldv, c->coef, n, c->nv, c->ctrl, 0, nullptr, nullptr, nullptr, 0.0);
            have_u = 1;
        }
        exg::dev::erc_update(L, c->nw, c->nv, c->nu, have_u, 1.0 / h, gamma, c->xnext, n);
    }
    ck(cudaGetLastError(), "er_nonlinear launch");
    API_END(c)
}

exg_status exg_gather(exg_ctx* c, const int* idx, int k, double* out) {
    API_BEGIN
    if (k <= 0) return EXG_OK;
    const exg_status st = exg_gather_async(c, idx, k, nullptr, true);
    if (st != EXG_OK) return st;
    ck(cudaMemcpyAsync(out, c->probe_out, sizeof(double) * k, cudaMemcpyDeviceToHost, c->stream), "d2h");
    ck(cudaStreamSynchronize(c->stream), "gather sync");
    API_END(c)
}

}  // extern "C"

// x_next[idx] -> dev_out (probe_out when null), stream-ordered, no host sync.
// A transient probes the same nodes every step: the index list is uploaded
// only when it changed (check) or on the first call.
exg_status exg_gather_async(exg_ctx* c, const int* idx, int k, double* dev_out, bool check) {
    API_BEGIN
    if (k <= 0) return EXG_OK;
    if (k > c->probe_cap) {
        dfree(c->probe_idx);
        dfree(c->probe_out);
        c->probe_idx = dalloc<int>(k);
        c->probe_out = dalloc<double>(k);
        c->probe_cap = k;
        c->probe_host.clear();
    }
    if (c->probe_host.size() != (size_t)k ||
        (check && std::memcmp(c->probe_host.data(), idx, sizeof(int) * k) != 0)) {
        ck(cudaMemcpyAsync(c->probe_idx, idx, sizeof(int) * k, cudaMemcpyHostToDevice, c->stream), "idx");
        c->probe_host.assign(idx, idx + k);
    }
    k_gather<<<(k + 255) / 256, 256, 0, c->stream>>>(c->xnext, c->probe_idx, k, dev_out ? dev_out : c->probe_out);
    c->launches++;
    ck(cudaGetLastError(), "gather launch");
    API_END(c)
}

extern "C" {

// debug: one triangular-solve pair with per-row (start, end) timestamps of the
// L and U sweeps (ns, %globaltimer), 4n values: L pairs then U pairs
exg_status exg_debug_trace_solve(exg_ctx* c, const double* b, unsigned long long* times) {
    API_BEGIN
    require_factors(c);
    const int n = c->n;
    unsigned long long* tr = dalloc<unsigned long long>((size_t)4 * n);
    ck(cudaMemsetAsync(tr, 0, sizeof(unsigned long long) * 4 * (size_t)n, c->stream), "memset");
    c->trace_l = tr;
    c->trace_u = tr + 2 * (size_t)n;
    unsigned long long* ntr = dalloc<unsigned long long>((size_t)6 * n);
    ck(cudaMemsetAsync(ntr, 0, sizeof(unsigned long long) * 6 * (size_t)n, c->stream), "memset");
    c->ntrace_l = ntr;
    c->ntrace_u = ntr + 3 * (size_t)n;
    const double* bd = resolve_in(c, b, n, EXG_PTR_HOST, c->vin);
    solve_dev(c, bd, c->vout, 1.0, nullptr, nullptr);
    c->trace_l = c->trace_u = nullptr;
    c->ntrace_l = c->ntrace_u = nullptr;
    ck(cudaMemcpyAsync(times, tr, sizeof(unsigned long long) * 4 * (size_t)n, cudaMemcpyDeviceToHost, c->stream), "d2h");
    ck(cudaMemcpyAsync(times + 4 * (size_t)n, ntr, sizeof(unsigned long long) * 6 * (size_t)n, cudaMemcpyDeviceToHost, c->stream), "d2h");
    ck(cudaStreamSynchronize(c->stream), "sync");
    cudaFree(tr);
    cudaFree(ntr);
    API_END(c)
}

// debug: one stream-plan solve pair with per-task timestamps (k_trsv4):
// 5 values per task {level, begin, dependencies ready, published, warp}, L's
// tasks then U's.  counts[0..1]: tasks of L and U (call with times == null
// first to size the buffer); counts[2..3]: warps; counts[4..5]: stream bytes.
exg_status exg_debug_trace_stream(exg_ctx* c, const double* b, unsigned long long* times, long long* counts) {
    API_BEGIN
    require_factors(c);
    if (!c->plan[0].s_warps || !c->plan[1].s_warps || c->opt.trsv_mode != EXG_TRSV_FAST)
        throw ApiError{EXG_E_CONTRACT, "exg_debug_trace_stream: FAST mode with the stream plan only"};
    const long long nl = c->cnt_aug[0][5], nu = c->cnt_aug[1][5];
    if (counts) {
        counts[0] = nl;
        counts[1] = nu;
        counts[2] = c->plan[0].s_warps;
        counts[3] = c->plan[1].s_warps;
        counts[4] = c->plan[0].s_bytes;
        counts[5] = c->plan[1].s_bytes;
    }
    if (times) {
        const int n = c->n;
        unsigned long long* tr = dalloc<unsigned long long>((size_t)5 * (nl + nu));
        ck(cudaMemsetAsync(tr, 0, sizeof(unsigned long long) * 5 * (size_t)(nl + nu), c->stream), "memset");
        c->trace_l = tr;
        c->trace_u = tr + 5 * (size_t)nl;
        const double* bd = resolve_in(c, b, n, EXG_PTR_HOST, c->vin);
        solve_dev(c, bd, c->vout, 1.0, nullptr, nullptr);
        c->trace_l = c->trace_u = nullptr;
        ck(cudaMemcpyAsync(times, tr, sizeof(unsigned long long) * 5 * (size_t)(nl + nu), cudaMemcpyDeviceToHost, c->stream), "d2h");
        ck(cudaStreamSynchronize(c->stream), "sync");
        cudaFree(tr);
    }
    API_END(c)
}

// debug / test: one orthogonalize step (krylov.cpp:46-78) in isolation.  V:
// host n x (j + 1) column-major orthonormal basis, w: the vector to
// orthogonalise.  Outputs: hcol (j + 2 Hessenberg entries), v_next (n; the
// normalised remainder, untouched on a happy breakdown), info = {happy,
// reorthogonalised}.  FAST mode runs the grouped kernel (k_mgs2), EXACT mode
// the column-by-column one (k_mgs).
exg_status exg_debug_orthogonalize(exg_ctx* c, int n, int j, const double* V, const double* w,
                                   double breakdown_tol, double* hcol, double* v_next, int* info) {
    API_BEGIN
    if (n < 1 || j < 0 || !V || !w || !hcol || !v_next) throw ApiError{EXG_E_CONTRACT, "exg_debug_orthogonalize: bad arguments"};
    ensure_vectors(c, std::max(n, c->vec_n));
    const long long ldv = ((long long)n + 31) / 32 * 32;
    const int hld = j + 3;
    double* dV = dalloc<double>((size_t)(j + 2) * ldv);
    double* dw = dalloc<double>(n);
    double* dh = dalloc<double>((size_t)(j + 1) * hld);
    Ctrl* dc = reinterpret_cast<Ctrl*>(dalloc<char>(sizeof(Ctrl)));
    ck(cudaMemsetAsync(dV, 0, (size_t)(j + 2) * ldv * sizeof(double), c->stream), "memset");
    ck(cudaMemsetAsync(dh, 0, (size_t)(j + 1) * hld * sizeof(double), c->stream), "memset");
    for (int i = 0; i <= j; ++i)
        ck(cudaMemcpyAsync(dV + (size_t)i * ldv, V + (size_t)i * n, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream), "h2d");
    ck(cudaMemcpyAsync(dw, w, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream), "h2d");
    Ctrl hc;
    std::memset(&hc, 0, sizeof hc);
    hc.j = j;
    hc.breakdown_tol = breakdown_tol;
    ck(cudaMemcpyAsync(dc, &hc, sizeof hc, cudaMemcpyHostToDevice, c->stream), "h2d");
    exg::dev::Mgs2Shape ms{};
    if (c->opt.trsv_mode == EXG_TRSV_FAST && exg::dev::mgs2_shape(n, c->num_sms, 0, &ms)) {
        ensure_mgs_slots(c, j + 1);
        exg::dev::Mgs2Args a2{n, ldv, dV, dw, dh, hld, c->mgs_slots + 8, reinterpret_cast<unsigned int*>(c->mgs_slots),
                              dc, c->mgs_inst_cap, 0, 0, 0};
        ck(exg::dev::mgs2(c->L(), a2, ms), "mgs2 launch");
    } else {
        int K = 1, blocks = 1;
        const int ks[] = {1, 2, 4, 8, 16};
        for (int kk : ks) {
            K = kk;
            const long long cap = (long long)c->num_sms * std::max(1, exg::dev::mgs_max_blocks(kk));
            blocks = (int)std::min<long long>(cap, ((long long)n + 1024LL * kk - 1) / (1024LL * kk));
            if ((long long)blocks * 1024 * kk >= n) break;
        }
        if ((long long)blocks * 1024 * K < n) throw ApiError{EXG_E_CONTRACT, "vector too long for the MGS kernel"};
        exg::dev::MgsArgs a1{n, ldv, dV, dw, dh, hld, c->partials + c->mgs_partials_off, c->bar, dc};
        ck(exg::dev::mgs(c->L(), a1, std::min(blocks, 4096), K), "mgs launch");
    }
    ck(cudaMemcpyAsync(hcol, dh + (size_t)j * hld, sizeof(double) * (j + 2), cudaMemcpyDeviceToHost, c->stream), "d2h");
    ck(cudaMemcpyAsync(&hc, dc, sizeof hc, cudaMemcpyDeviceToHost, c->stream), "d2h");
    ck(cudaStreamSynchronize(c->stream), "sync");
    if (!hc.happy)
        ck(cudaMemcpy(v_next, dV + (size_t)(j + 1) * ldv, sizeof(double) * n, cudaMemcpyDeviceToHost), "d2h");
    if (info) {
        info[0] = hc.happy;
        info[1] = (int)hc.reorths;
    }
    cudaFree(dV);
    cudaFree(dw);
    cudaFree(dh);
    cudaFree(dc);
    API_END(c)
}

// debug / test: y = C x through the FAST-mode SpMV of the Arnoldi loop
// (k_spmv_v4 / k_spmv_v4w: four lanes per row, sparse_matrix.cpp:69-82 up to
// the order of the additions), on host vectors
exg_status exg_debug_spmv_fast(exg_ctx* c, const double* x, double* y) {
    API_BEGIN
    const DCsr& Cm = mat(c, EXG_MAT_C);
    if (!x || !y || Cm.n_rows != Cm.n_cols) throw ApiError{EXG_E_CONTRACT, "exg_debug_spmv_fast: bad arguments"};
    const int n = Cm.n_rows;
    const long long ldv = ((long long)n + 31) / 32 * 32;
    double* dx = dalloc<double>((size_t)2 * ldv);  // column 1 is read (j = 1): a non-zero column offset
    double* dy = dalloc<double>(n);
    Ctrl* dc = reinterpret_cast<Ctrl*>(dalloc<char>(sizeof(Ctrl)));
    Ctrl hc;
    std::memset(&hc, 0, sizeof hc);
    hc.j = 1;
    ck(cudaMemsetAsync(dx, 0, (size_t)2 * ldv * sizeof(double), c->stream), "memset");
    ck(cudaMemcpyAsync(dx + ldv, x, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream), "h2d");
    ck(cudaMemcpyAsync(dc, &hc, sizeof hc, cudaMemcpyHostToDevice, c->stream), "h2d");
    exg::dev::spmv_v4(c->L(), Cm.rowptr, Cm.col, Cm.val, n, Cm.max_strip, dy, dc, dx, ldv);
    ck(cudaGetLastError(), "spmv launch");
    ck(cudaMemcpyAsync(y, dy, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream), "d2h");
    ck(cudaStreamSynchronize(c->stream), "sync");
    cudaFree(dx);
    cudaFree(dy);
    cudaFree(dc);
    API_END(c)
}

// debug / test: dense_expm (dense_matrix.cpp:185-225) of a host m x m
// row-major matrix through k_dense (shared-memory scratch for small m, the
// global scratch above), bit-identical to the reference
exg_status exg_debug_dense_expm(exg_ctx* c, int m, const double* A, double* E) {
    API_BEGIN
    if (m < 1 || m > 512 || !A || !E) throw ApiError{EXG_E_CONTRACT, "exg_debug_dense_expm: bad arguments"};
    const size_t mm = (size_t)m * m;
    double* dA = dalloc<double>(mm);
    double* dE = dalloc<double>(mm);
    double* dS = dalloc<double>(20 * mm);
    Ctrl* dc = reinterpret_cast<Ctrl*>(dalloc<char>(sizeof(Ctrl)));
    Ctrl hc;
    std::memset(&hc, 0, sizeof hc);
    hc.m = m;
    ck(cudaMemcpyAsync(dc, &hc, sizeof hc, cudaMemcpyHostToDevice, c->stream), "h2d");
    ck(cudaMemcpyAsync(dA, A, mm * sizeof(double), cudaMemcpyHostToDevice, c->stream), "h2d");
    exg::dev::DenseArgs da{dc, nullptr, 0, dA, nullptr, dS, 0, 3, 1.0, dE};
    exg::dev::dense(c->L(), da, m);
    ck(cudaMemcpyAsync(E, dE, mm * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "d2h");
    ck(cudaMemcpyAsync(&hc, dc, sizeof hc, cudaMemcpyDeviceToHost, c->stream), "d2h");
    ck(cudaStreamSynchronize(c->stream), "sync");
    cudaFree(dA);
    cudaFree(dE);
    cudaFree(dS);
    cudaFree(dc);
    if (hc.status == 2) throw ApiError{EXG_E_NONFINITE, "dense_expm: non-finite entry"};
    if (hc.status) throw ApiError{EXG_E_SINGULAR, "dense_solve: singular matrix"};
    API_END(c)
}

exg_status exg_profile_enable(exg_ctx* c, int on) {
    if (!c) return EXG_E_CONTRACT;
    c->profiling = on != 0;
    return EXG_OK;
}

exg_status exg_profile_get(exg_ctx* c, exg_kernel_times* out) {
    API_BEGIN
    ck(cudaStreamSynchronize(c->stream), "profile sync");
    for (auto& pe : c->prof_events) {
        float ms = 0.f;
        ck(cudaEventElapsedTime(&ms, pe.second.first, pe.second.second), "elapsed");
        c->prof_ms[pe.first] += ms;
        c->prof_count[pe.first] += 1;
        c->event_pool.push_back(pe.second.first);
        c->event_pool.push_back(pe.second.second);
    }
    c->prof_events.clear();
    for (int k = 0; k < EXG_K_CLASSES; ++k) {
        out->ms[k] = c->prof_ms[k];
        out->count[k] = c->prof_count[k];
        c->prof_ms[k] = 0.0;
        c->prof_count[k] = 0;
    }
    API_END(c)
}

exg_status exg_counters_get(exg_ctx* c, exg_counters* out) {
    if (!c || !out) return EXG_E_CONTRACT;
    *out = c->cnt;
    out->kernel_launches = c->launches;
    return EXG_OK;
}

exg_status exg_counters_reset(exg_ctx* c) {
    if (!c) return EXG_E_CONTRACT;
    c->launches = 0;
    c->cnt.arnoldi_iters = c->cnt.mevp_calls = c->cnt.trsv_calls = 0;
    c->cnt.graph_launches = c->cnt.graph_builds = 0;
    c->cnt.mgs_passes = c->cnt.reorths = 0;
    return EXG_OK;
}

exg_status exg_synchronize(exg_ctx* c) {
    API_BEGIN
    ck(cudaStreamSynchronize(c->stream), "sync");
    API_END(c)
}

exg_status exg_device_alloc(exg_ctx* c, size_t bytes, void** ptr) {
    API_BEGIN
    ck(cudaMalloc(ptr, bytes), "cudaMalloc");
    API_END(c)
}

exg_status exg_device_free(exg_ctx* c, void* ptr) {
    API_BEGIN
    ck(cudaFree(ptr), "cudaFree");
    API_END(c)
}

exg_status exg_memcpy(exg_ctx* c, void* dst, const void* src, size_t bytes, int kind) {
    API_BEGIN
    ck(cudaMemcpyAsync(dst, src, bytes, (cudaMemcpyKind)kind, c->stream), "memcpy");
    ck(cudaStreamSynchronize(c->stream), "memcpy sync");
    API_END(c)
}

void* exg_stream(exg_ctx* c) { return c ? (void*)c->stream : nullptr; }

}  // extern "C"
