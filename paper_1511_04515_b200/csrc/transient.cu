// exg_transient: the reference's ER/ERC time-stepping loop
// (exsim::transient, proj/core/src/integrate.cpp:368-480) driving the device
// hot path through the C ABI.  Step control, source evaluation, breakpoints
// and waveform emission stay on the host with the reference's exact
// arithmetic; every vector operation of a step runs on the device.
//
// Linear circuits (no nonlinear devices): G_k == G_lin every step
// (devices.cpp:190-192), so G is factorized once at setup
// (exg::lu_factor, bit-identical to exsim::lu_factor) and uploaded; the
// reference re-factorizes per step with identical results, which
// ref_transient_cached reproduces on the oracle side.
//
// Nonlinear circuits (MOSFETs, config 4): per step the host re-linearizes at
// x_k (exg::evaluate == exsim::evaluate), factorizes G_k (bit-identical LU) and
// uploads G_k, C_k, the factors and the operating points; the device runs
// er_begin (with F(x_k) stamped on the device), er_eval and the nonlinear
// error / ER-C correction MEVPs of every rejection retry
// (integrate.cpp:417-447).  The DC point is exg::dc_solve (integrate.cpp:92).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <vector>

#include "ctx.hpp"
#include "exg_host.h"
#include "host.hpp"


struct exg_tran_result {
    int n_rec = 0;
    std::vector<double> times, samples;
    std::vector<double> t, h, err;
    std::vector<int> lu, rej, dims_off{0}, dims;
    double lu_s = 0.0, dc_s = 0.0, loop_s = 0.0;
};

namespace {

double next_breakpoint_after(const std::vector<double>& bps, double t) {  // integrate.cpp:361-364
    auto it = std::upper_bound(bps.begin(), bps.end(), t * (1.0 + 1e-12));
    return it == bps.end() ? std::numeric_limits<double>::infinity() : *it;
}

struct Fail {
    exg_status st;
    std::string msg;
};

void cuda_chk(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Fail{EXG_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e)};
}

struct PinnedDoubles {
    double* p = nullptr;
    ~PinnedDoubles() {
        if (p) cudaFreeHost(p);
    }
};

struct EventPair {  // created recorded-complete: the first wait returns at once
    cudaEvent_t e[2] = {nullptr, nullptr};
    EventPair() {
        for (auto& x : e) cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
    }
    ~EventPair() {
        for (auto& x : e)
            if (x) cudaEventDestroy(x);
    }
};

struct DeviceDoubles {
    double* p = nullptr;
    ~DeviceDoubles() {
        if (p) cudaFree(p);
    }
};

void chk(exg_ctx* ctx, exg_status st) {
    if (st != EXG_OK) {
        char buf[512];
        exg_last_error(ctx, buf, sizeof buf);
        throw Fail{st, buf};
    }
}


std::vector<int> record_list(const exg::System& sys, const int* rec_idx, int n_rec) {
    std::vector<int> rec;
    if (n_rec == 0)
        for (int i = 0; i < sys.n; ++i) rec.push_back(i);
    else
        rec.assign(rec_idx, rec_idx + n_rec);
    for (int i : rec)
        if (i < 0 || i >= sys.n) throw Fail{EXG_E_CONTRACT, "unknown record node"};
    return rec;
}

void upload_linearization(exg_ctx* ctx, const exg::Linearization& lin, const exg::Factor& f, bool with_op,
                          bool op_only = false) {
    if (!op_only) {
        chk(ctx, exg_set_csr(ctx, EXG_MAT_C, lin.C.n_rows, lin.C.n_cols, lin.C.nnz(), lin.C.rowptr.data(),
                             lin.C.col.data(), lin.C.val.data()));
        chk(ctx, exg_set_csr(ctx, EXG_MAT_G, lin.G.n_rows, lin.G.n_cols, lin.G.nnz(), lin.G.rowptr.data(),
                             lin.G.col.data(), lin.G.val.data()));
        chk(ctx, exg_set_factors(ctx, f.n, f.L.rowptr.data(), f.L.col.data(), f.L.val.data(), f.U.rowptr.data(),
                                 f.U.col.data(), f.U.val.data(), f.row_perm.data(), f.col_perm.data()));
    }
    if (!with_op && !op_only) return;
    std::vector<double> op(5 * lin.op.size());
    for (size_t i = 0; i < lin.op.size(); ++i) {
        op[5 * i] = lin.op[i].vgs_ref;
        op[5 * i + 1] = lin.op[i].vds_ref;
        op[5 * i + 2] = lin.op[i].id_ref;
        op[5 * i + 3] = lin.op[i].gm;
        op[5 * i + 4] = lin.op[i].gds;
    }
    chk(ctx, exg_set_oppoints(ctx, op.data()));
}

// relative change of the device Jacobian (the stamped conductances gm, gds of
// every device) between two linearizations of the same circuit, in the
// Euclidean norm: the "Jacobian change" of the refactor
// policy (exg_step_control.refactor_threshold; restated identically in
// oracle/ref_shim.cpp)
double jacobian_change(const exg::Linearization& a, const exg::Linearization& b) {
    // || (gm, gds)_b - (gm, gds)_a ||_2 / || (gm, gds)_a ||_2 over all devices,
    // summed in device order (the same arithmetic in the product and its oracle)
    double num = 0.0, den = 0.0;
    for (size_t i = 0; i < a.op.size(); ++i) {
        const double dm = b.op[i].gm - a.op[i].gm, dd = b.op[i].gds - a.op[i].gds;
        num += dm * dm;
        num += dd * dd;
        den += a.op[i].gm * a.op[i].gm;
        den += a.op[i].gds * a.op[i].gds;
    }
    if (num == 0.0) return 0.0;
    if (den == 0.0) return std::numeric_limits<double>::infinity();
    return std::sqrt(num / den);
}

// integrate.cpp:368-480 with nonlinear devices
exg_status transient_nonlinear(exg_ctx* ctx, const exg::System& sys, const exg_step_control* ctl,
                               double t_stop, const int* rec_idx, int n_rec, exg_tran_result** out) {
    using clock = std::chrono::steady_clock;
    auto* res = new exg_tran_result();
    std::unique_ptr<exg_tran_result> guard(res);
    const std::vector<int> rec = record_list(sys, rec_idx, n_rec);
    res->n_rec = static_cast<int>(rec.size());
    const int n = sys.n;
    const int ni = sys.n_inputs();
    const bool erc = ctl->method == EXG_METHOD_ERC;

    auto t0 = clock::now();
    std::vector<double> x;
    try {
        x = exg::dc_solve(sys);
    } catch (const exg::Error& e) {
        throw Fail{e.status, e.what};
    }
    auto t1 = clock::now();
    res->dc_s = std::chrono::duration<double>(t1 - t0).count();
    auto emit_host = [&](double t, const std::vector<double>& xv) {
        res->times.push_back(t);
        for (int i : rec) res->samples.push_back(xv[i]);
    };
    emit_host(0.0, x);

    const std::vector<double> bps = exg::source_breakpoints(sys, 0.0, t_stop);
    const double hint = sys.opts.has_tran && sys.opts.tran_step > 0.0 ? sys.opts.tran_step : t_stop / 100.0;
    double h_nominal = ctl->h_init > 0.0 ? ctl->h_init : hint;
    h_nominal = std::min(h_nominal, ctl->hmax);
    const double hmin_eff = ctl->hmin > 0.0 ? ctl->hmin : t_stop * 1e-15;
    const double t_tiny = t_stop * 1e-12;
    exg_mevp_cfg cfg{ctl->eps, ctl->m_max, 1, 1e-12};

    // B is constant; G_k / C_k / factors / operating points change per step
    chk(ctx, exg_set_csr(ctx, EXG_MAT_B, sys.B.n_rows, sys.B.n_cols, sys.B.nnz(), sys.B.rowptr.data(),
                         sys.B.col.data(), sys.B.val.data()));
    bool devices_set = false;
    bool have_lin = false;
    exg::Linearization lin;
    exg::Factor f;
    double lu_s = 0.0;
    double t = 0.0;
    while (t < t_stop - t_tiny) {
        const double seg_end = std::min(next_breakpoint_after(bps, t), t_stop);
        double h_try = std::min(h_nominal, seg_end - t);
        if (seg_end - t - h_try < t_tiny) h_try = seg_end - t;
        h_try = std::max(h_try, std::min(hmin_eff, seg_end - t));

        // linearization at x_k (integrate.cpp:419-421).  With a refactor
        // threshold the frozen Linearization and its factors are kept while no
        // device conductance moved by more than that relative amount
        auto ta = clock::now();
        bool refresh = true;
        try {
            exg::Linearization lin_new;
            exg::evaluate(sys, x, lin_new);
            if (have_lin && ctl->refactor_threshold > 0.0 &&
                jacobian_change(lin, lin_new) <= ctl->refactor_threshold)
                refresh = false;
            if (refresh) {
                lin = std::move(lin_new);
                exg::lu_factor(lin.G, 0.1, f);
                have_lin = true;
            }
        } catch (const exg::Error& e) {
            throw Fail{e.status, e.what};
        }
        lu_s += std::chrono::duration<double>(clock::now() - ta).count();
        if (refresh) upload_linearization(ctx, lin, f, devices_set);
        if (!devices_set) {  // device tables (after the first set_factors fixes n)
            std::vector<int> nodes(4 * sys.mos.size());
            std::vector<double> par(6 * sys.mos.size());
            for (size_t i = 0; i < sys.mos.size(); ++i) {
                const exg::Mosfet& m = sys.mos[i];
                for (int j = 0; j < 4; ++j) nodes[4 * i + j] = m.nodes[j];
                par[6 * i] = m.vth;
                par[6 * i + 1] = m.kp;
                par[6 * i + 2] = m.lambda;
                par[6 * i + 3] = m.w;
                par[6 * i + 4] = m.l;
                par[6 * i + 5] = m.pmos ? 1.0 : 0.0;
            }
            chk(ctx, exg_set_devices(ctx, static_cast<int>(sys.mos.size()), nodes.data(), par.data()));
            devices_set = true;
            upload_linearization(ctx, lin, f, false, true);
        }

        const std::vector<double> u_k = exg::eval_sources(sys, t);
        const std::vector<double> u_k1 = exg::eval_sources(sys, t + h_try);
        chk(ctx, exg_memcpy(ctx, ctx->xk, x.data(), sizeof(double) * n, cudaMemcpyHostToDevice));
        if (ni) {
            chk(ctx, exg_memcpy(ctx, ctx->u_k, u_k.data(), sizeof(double) * ni, cudaMemcpyHostToDevice));
            chk(ctx, exg_memcpy(ctx, ctx->u_k1, u_k1.data(), sizeof(double) * ni, cudaMemcpyHostToDevice));
        }
        chk(ctx, exg_er_begin(ctx, ctx->xk, ctx->u_k, ctx->u_k1, h_try, EXG_PTR_DEVICE));

        int rejects = 0;
        double err_norm = 0.0;
        while (true) {
            int m = -1;
            chk(ctx, exg_er_eval(ctx, h_try, &cfg, nullptr, &m, nullptr, EXG_PTR_DEVICE));
            if (m >= 0) res->dims.push_back(m);
            int dims[2], nd = 0;
            err_norm = 0.0;
            chk(ctx, exg_er_nonlinear(ctx, h_try, &cfg, erc ? 1 : 0, ctl->gamma, &err_norm, dims, &nd));
            for (int i = 0; i < nd; ++i) res->dims.push_back(dims[i]);
            if (ctl->fixed_step || err_norm <= ctl->err_budget) break;
            ++rejects;
            if (rejects > ctl->max_rejects)
                throw Fail{EXG_E_STEP_FAILURE, "transient: too many rejections at t=" + std::to_string(t)};
            h_try *= ctl->alpha;
            if (h_try < hmin_eff)
                throw Fail{EXG_E_STEP_FAILURE, "transient: step size below HMIN at t=" + std::to_string(t)};
        }
        res->t.push_back(t + h_try);
        res->h.push_back(h_try);
        res->lu.push_back(refresh ? 1 : 0);
        res->rej.push_back(rejects);
        res->err.push_back(err_norm);
        res->dims_off.push_back(static_cast<int>(res->dims.size()));

        chk(ctx, exg_memcpy(ctx, x.data(), ctx->xnext, sizeof(double) * n, cudaMemcpyDeviceToHost));
        t += h_try;
        emit_host(t, x);

        const bool grow = !ctl->fixed_step &&
                          (ctl->grow_only_on_clean ? rejects == 0 : rejects < ctl->grow_threshold);
        const bool clamped = h_try < h_nominal * (1.0 - 1e-12);
        if (rejects > 0) h_nominal = h_try;
        if (grow) h_nominal = std::min(ctl->beta * (clamped && rejects == 0 ? h_nominal : h_try), ctl->hmax);
    }
    res->lu_s = lu_s;
    res->loop_s = std::chrono::duration<double>(clock::now() - t1).count();
    *out = guard.release();
    return EXG_OK;
}

}  // namespace

extern "C" {

exg_status exg_transient(exg_ctx* ctx, const exg_system* sp, const exg_step_control* ctl,
                         double t_stop, const int* rec_idx, int n_rec, exg_tran_result** out) {
    using clock = std::chrono::steady_clock;
    try {
        const exg::System& sys = sp->sys;
        if (t_stop <= 0.0) throw Fail{EXG_E_CONTRACT, "transient: t_stop must be positive"};
        // ER and ER-C only: BENR (integrate.cpp:400-416) stays reference host code
        if (!ctl || (ctl->method != EXG_METHOD_ER && ctl->method != EXG_METHOD_ERC))
            throw Fail{EXG_E_CONTRACT, "transient: method must be EXG_METHOD_ER or EXG_METHOD_ERC"};
        if (!sys.mos.empty()) {
            *out = nullptr;
            return transient_nonlinear(ctx, sys, ctl, t_stop, rec_idx, n_rec, out);
        }
        auto* res = new exg_tran_result();
        std::unique_ptr<exg_tran_result> guard(res);
        std::vector<int> rec;
        if (n_rec == 0)
            for (int i = 0; i < sys.n; ++i) rec.push_back(i);
        else
            rec.assign(rec_idx, rec_idx + n_rec);
        for (int i : rec)
            if (i < 0 || i >= sys.n) throw Fail{EXG_E_CONTRACT, "unknown record node"};
        res->n_rec = static_cast<int>(rec.size());

        // ---- setup: device CSR store + the one factorization of G
        const exg::Csr* mats[3] = {&sys.C, &sys.G, &sys.B};
        for (int w = 0; w < 3; ++w)
            chk(ctx, exg_set_csr(ctx, w, mats[w]->n_rows, mats[w]->n_cols, mats[w]->nnz(),
                                 mats[w]->rowptr.data(), mats[w]->col.data(), mats[w]->val.data()));
        auto t0 = clock::now();
        exg::Factor f;
        try {
            exg::lu_factor(sys.G, 0.1, f);
        } catch (const exg::Error& e) {
            throw Fail{e.status, e.what};
        }
        chk(ctx, exg_set_factors(ctx, f.n, f.L.rowptr.data(), f.L.col.data(), f.L.val.data(),
                                 f.U.rowptr.data(), f.U.col.data(), f.U.val.data(),
                                 f.row_perm.data(), f.col_perm.data()));
        auto t1 = clock::now();
        res->lu_s = std::chrono::duration<double>(t1 - t0).count();

        // ---- DC point: linear newton_static = lu_factor(G) + solve(B u(0))
        // (integrate.cpp:70-75, :92-100), solved in EXACT mode
        std::vector<double> x(sys.n, 0.0);
        {
            const std::vector<double> u0 = exg::eval_sources(sys, 0.0);
            std::vector<double> bu0(sys.n, 0.0);
            for (int r = 0; r < sys.n; ++r) {
                double s = 0.0;
                for (int k = sys.B.rowptr[r]; k < sys.B.rowptr[r + 1]; ++k)
                    s += sys.B.val[k] * u0[sys.B.col[k]];
                bu0[r] = s;
            }
            const exg_options_dev saved = ctx->opt;
            exg_options_dev exact = saved;
            exact.trsv_mode = EXG_TRSV_EXACT;
            exg_set_options(ctx, &exact);
            const exg_status st = exg_solve(ctx, bu0.data(), x.data(), EXG_PTR_HOST);
            exg_set_options(ctx, &saved);
            chk(ctx, st);
        }
        auto t2 = clock::now();
        res->dc_s = std::chrono::duration<double>(t2 - t1).count();

        std::vector<double> row(rec.size());
        auto emit_host = [&](double t, const std::vector<double>& xv) {
            res->times.push_back(t);
            for (size_t i = 0; i < rec.size(); ++i) res->samples.push_back(xv[rec[i]]);
        };
        emit_host(0.0, x);

        // ---- stepping loop (integrate.cpp:380-478)
        const std::vector<double> bps = exg::source_breakpoints(sys, 0.0, t_stop);
        const double hint = sys.opts.has_tran && sys.opts.tran_step > 0.0 ? sys.opts.tran_step
                                                                          : t_stop / 100.0;
        double h_nominal = ctl->h_init > 0.0 ? ctl->h_init : hint;
        h_nominal = std::min(h_nominal, ctl->hmax);
        const double hmin_eff = ctl->hmin > 0.0 ? ctl->hmin : t_stop * 1e-15;
        const double t_tiny = t_stop * 1e-12;
        exg_mevp_cfg cfg{ctl->eps, ctl->m_max, 1, 1e-12};

        // device-resident state: x_k lives in ctx->xk (uploaded once)
        const int n = sys.n;
        const int ni = sys.n_inputs();
        chk(ctx, exg_memcpy(ctx, ctx->xnext, x.data(), sizeof(double) * n, cudaMemcpyHostToDevice));
        // two pinned staging slots for (u_k, u_k1), used alternately; an event
        // per slot marks its H2D copies done before the slot is rewritten, so
        // correctness does not depend on a host sync elsewhere in the step
        PinnedDoubles u_pin;
        if (ni) cuda_chk(cudaMallocHost(&u_pin.p, sizeof(double) * 4 * ni), "cudaMallocHost");
        EventPair u_done;
        int u_slot = 0;
        // recorded samples: a device ring of up to 256 steps (<= 64 MB) and a
        // pinned host mirror; one read-back per ring instead of a sync per step
        const int k_rec = static_cast<int>(rec.size());
        const int ring_steps = static_cast<int>(
            std::max<size_t>(1, std::min<size_t>(256, (size_t(64) << 20) / (sizeof(double) * k_rec))));
        DeviceDoubles ring;
        PinnedDoubles ring_pin;
        cuda_chk(cudaMalloc(&ring.p, sizeof(double) * k_rec * ring_steps), "cudaMalloc");
        cuda_chk(cudaMallocHost(&ring_pin.p, sizeof(double) * k_rec * ring_steps), "cudaMallocHost");
        int filled = 0;
        bool first_gather = true;  // a user exg_gather may have left another list
        auto flush_ring = [&]() {
            if (!filled) return;
            const size_t cnt = (size_t)filled * k_rec;
            cuda_chk(cudaMemcpyAsync(ring_pin.p, ring.p, sizeof(double) * cnt, cudaMemcpyDeviceToHost,
                                     ctx->stream), "samples d2h");
            cuda_chk(cudaStreamSynchronize(ctx->stream), "samples sync");
            res->samples.insert(res->samples.end(), ring_pin.p, ring_pin.p + cnt);
            filled = 0;
        };
        double t = 0.0;
        while (t < t_stop - t_tiny) {
            const double seg_end = std::min(next_breakpoint_after(bps, t), t_stop);
            double h_try = std::min(h_nominal, seg_end - t);
            if (seg_end - t - h_try < t_tiny) h_try = seg_end - t;
            h_try = std::max(h_try, std::min(hmin_eff, seg_end - t));

            const std::vector<double> u_k = exg::eval_sources(sys, t);
            const std::vector<double> u_k1 = exg::eval_sources(sys, t + h_try);
            if (ni) {
                // pinned staging, stream-ordered before er_begin; wait until
                // the copies that last read this slot (two steps ago) are done
                double* slot = u_pin.p + (size_t)2 * ni * u_slot;
                cuda_chk(cudaEventSynchronize(u_done.e[u_slot]), "u slot wait");
                std::memcpy(slot, u_k.data(), sizeof(double) * ni);
                std::memcpy(slot + ni, u_k1.data(), sizeof(double) * ni);
                cuda_chk(cudaMemcpyAsync(ctx->u_k, slot, sizeof(double) * ni, cudaMemcpyHostToDevice,
                                         ctx->stream), "u_k upload");
                cuda_chk(cudaMemcpyAsync(ctx->u_k1, slot + ni, sizeof(double) * ni,
                                         cudaMemcpyHostToDevice, ctx->stream), "u_k1 upload");
                cuda_chk(cudaEventRecord(u_done.e[u_slot], ctx->stream), "u slot event");
                u_slot ^= 1;
            }
            // x_k <- previous x_next (device to device)
            chk(ctx, exg_er_begin(ctx, ctx->xnext, ctx->u_k, ctx->u_k1, h_try, EXG_PTR_DEVICE));
            int m = -1;
            chk(ctx, exg_er_eval(ctx, h_try, &cfg, nullptr, &m, nullptr, EXG_PTR_DEVICE));
            // linear: err_norm == 0, never rejected (integrate.cpp:433-447)
            const int rejects = 0;
            res->t.push_back(t + h_try);
            res->h.push_back(h_try);
            res->lu.push_back(0);
            res->rej.push_back(rejects);
            res->err.push_back(0.0);
            if (m >= 0) res->dims.push_back(m);
            res->dims_off.push_back(static_cast<int>(res->dims.size()));

            t += h_try;
            // samples gathered into a device ring, read back in batches
            chk(ctx, exg_gather_async(ctx, rec.data(), k_rec, ring.p + (size_t)filled * k_rec, first_gather));
            first_gather = false;
            res->times.push_back(t);
            if (++filled == ring_steps) flush_ring();

            const bool grow = !ctl->fixed_step &&
                              (ctl->grow_only_on_clean ? rejects == 0 : rejects < ctl->grow_threshold);
            const bool clamped = h_try < h_nominal * (1.0 - 1e-12);
            if (rejects > 0) h_nominal = h_try;
            if (grow)
                h_nominal = std::min(ctl->beta * (clamped && rejects == 0 ? h_nominal : h_try), ctl->hmax);
        }
        flush_ring();
        // the linear factorization is shared by every step: report it once
        if (!res->lu.empty()) res->lu[0] = 1;
        res->loop_s = std::chrono::duration<double>(clock::now() - t2).count();
        *out = guard.release();
        return EXG_OK;
    } catch (const Fail& f) {
        if (ctx) {
            ctx->err = f.msg;
            ctx->last = f.st;
        }
        return f.st;
    } catch (const std::bad_alloc&) {
        return EXG_E_NOMEM;
    }
}

void exg_tran_result_free(exg_tran_result* r) { delete r; }
int exg_tran_n_times(const exg_tran_result* r) { return static_cast<int>(r->times.size()); }
int exg_tran_n_rec(const exg_tran_result* r) { return r->n_rec; }
const double* exg_tran_times(const exg_tran_result* r) { return r->times.data(); }
const double* exg_tran_samples(const exg_tran_result* r) { return r->samples.data(); }
int exg_tran_n_steps(const exg_tran_result* r) { return static_cast<int>(r->t.size()); }
exg_status exg_tran_records(const exg_tran_result* r, double* t, double* h, int* lu_count,
                            int* rejects, double* err_norm, int* dims_off) {
    const size_t n = r->t.size();
    if (t) std::memcpy(t, r->t.data(), n * sizeof(double));
    if (h) std::memcpy(h, r->h.data(), n * sizeof(double));
    if (lu_count) std::memcpy(lu_count, r->lu.data(), n * sizeof(int));
    if (rejects) std::memcpy(rejects, r->rej.data(), n * sizeof(int));
    if (err_norm) std::memcpy(err_norm, r->err.data(), n * sizeof(double));
    if (dims_off) std::memcpy(dims_off, r->dims_off.data(), (n + 1) * sizeof(int));
    return EXG_OK;
}
int exg_tran_n_dims(const exg_tran_result* r) { return static_cast<int>(r->dims.size()); }
const int* exg_tran_dims(const exg_tran_result* r) { return r->dims.data(); }
exg_status exg_tran_write_csv(const exg_tran_result* r, const char* path, const char* const* columns, int threads) {
    if (!r) return EXG_E_CONTRACT;
    return exg_write_waveform_csv(path, static_cast<int>(r->times.size()), r->n_rec, r->times.data(),
                                  r->samples.data(), columns, threads);
}
exg_status exg_tran_timing(const exg_tran_result* r, double* lu_s, double* dc_s, double* loop_s) {
    *lu_s = r->lu_s;
    *dc_s = r->dc_s;
    *loop_s = r->loop_s;
    return EXG_OK;
}

}  // extern "C"
