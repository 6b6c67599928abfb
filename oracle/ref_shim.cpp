// ORACLE / TEST INFRASTRUCTURE — not part of the product.
//
// extern "C" shim over the UNMODIFIED reference library (exsim_core compiled
// from /root/reference/proj/core/src by oracle/Makefile into
// oracle/_ref/libexsim_ref.so).  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference leg load it, as the checker.
//
// It exposes the reference's own public API (build_mna, lu_factor,
// Factorization::solve/apply, spmv, mevp_iks, mevp_residual,
// eval_at_scaled_h, dense_expm, transient, er_step, residual_F, evaluate) to
// Python through plain C types, plus `ref_transient_cached`: the restated ER
// loop of integrate.cpp:368-480 that calls only public API and reuses one
// Factorization for linear circuits; it is checked
// bit-for-bit against transient() by tests/test_oracle.py.
//
// Factorization's members are private (sparse_lu.hpp:46-51); factors computed
// elsewhere are installed through the standard explicit-instantiation access
// rule (no reference source is modified or copied).
#include "common.hpp"  // proj/tools: the CLI's writers (header-only)
#include <algorithm>
#include <chrono>
#include <cmath>
#include <limits>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "exg_host.h"
#include "exsim/dense_matrix.hpp"
#include "exsim/devices.hpp"
#include "exsim/errors.hpp"
#include "exsim/integrate.hpp"
#include "exsim/krylov.hpp"
#include "exsim/mna.hpp"
#include "exsim/netlist.hpp"
#include "exsim/sparse_lu.hpp"
#include "exsim/sparse_matrix.hpp"

using namespace exsim;

// ---- private-member access via explicit instantiation ----------------------
template <typename Tag, typename Tag::type M>
struct Rob {
    friend typename Tag::type get(Tag) { return M; }
};
#define EXG_ROB(NAME, CLASS, TYPE, MEMBER)                 \
    struct NAME {                                          \
        typedef TYPE CLASS::*type;                         \
        friend type get(NAME);                             \
    };                                                     \
    template struct Rob<NAME, &CLASS::MEMBER>;
EXG_ROB(FLower, Factorization, SparseRealMatrix, lower_)
EXG_ROB(FUpper, Factorization, SparseRealMatrix, upper_)
EXG_ROB(FRowPerm, Factorization, std::vector<int>, row_perm_)
EXG_ROB(FColPerm, Factorization, std::vector<int>, col_perm_)
EXG_ROB(FSrcNnz, Factorization, int, source_nnz_)
EXG_ROB(SNRows, SparseRealMatrix, int, n_rows_)
EXG_ROB(SNCols, SparseRealMatrix, int, n_cols_)
EXG_ROB(SRowOff, SparseRealMatrix, std::vector<int>, row_offsets_)
EXG_ROB(SColIdx, SparseRealMatrix, std::vector<int>, col_indices_)
EXG_ROB(SVals, SparseRealMatrix, std::vector<double>, values_)

namespace {

thread_local std::string g_err;
thread_local double g_err_value = 0.0;

int status_of(const std::exception& e) {
    g_err = e.what();
    g_err_value = 0.0;
    if (auto* p = dynamic_cast<const NoConvergenceError*>(&e)) {
        g_err_value = p->last_residual();
        return EXG_E_NO_CONVERGENCE;
    }
    if (auto* p = dynamic_cast<const SingularMatrixError*>(&e)) {
        g_err_value = p->pivot_index();
        return EXG_E_SINGULAR;
    }
    if (dynamic_cast<const ContractError*>(&e)) return EXG_E_CONTRACT;
    if (dynamic_cast<const NonFiniteError*>(&e)) return EXG_E_NONFINITE;
    if (dynamic_cast<const ZeroStartVectorError*>(&e)) return EXG_E_ZERO_START;
    if (dynamic_cast<const SingularReducedMatrixError*>(&e)) return EXG_E_SINGULAR_REDUCED;
    if (dynamic_cast<const NoDcConvergenceError*>(&e)) return EXG_E_NO_DC;
    if (dynamic_cast<const StepFailureError*>(&e)) return EXG_E_STEP_FAILURE;
    return EXG_E_CONTRACT;
}

#define GUARD_BEGIN try {
#define GUARD_END                         \
    }                                     \
    catch (const std::exception& e) {     \
        return status_of(e);              \
    }                                     \
    return EXG_OK;

SparseRealMatrix make_csr(int n_rows, int n_cols, int nnz, const int* rowptr, const int* col,
                          const double* val) {
    SparseRealMatrix m;
    m.*get(SNRows()) = n_rows;
    m.*get(SNCols()) = n_cols;
    (m.*get(SRowOff())).assign(rowptr, rowptr + n_rows + 1);
    (m.*get(SColIdx())).assign(col, col + nnz);
    (m.*get(SVals())).assign(val, val + nnz);
    return m;
}

std::string node_name(int label) { return label == -1 ? "0" : "N" + std::to_string(label); }

SourceWaveform source_of(const exg_source& d, const double* pwl_t, const double* pwl_v) {
    switch (d.kind) {
        case EXG_SRC_DC:
            return SourceWaveform::dc(d.dc);
        case EXG_SRC_PWL: {
            std::vector<std::pair<double, double>> pts;
            for (int i = 0; i < d.pwl_len; ++i)
                pts.emplace_back(pwl_t[d.pwl_off + i], pwl_v[d.pwl_off + i]);
            return SourceWaveform::piecewise_linear(std::move(pts));
        }
        default: {
            SourceWaveform::Pulse p;
            p.v1 = d.v1;
            p.v2 = d.v2;
            p.delay = d.delay;
            p.rise = d.rise;
            p.fall = d.fall;
            p.width = d.width;
            p.period = d.period;
            return SourceWaveform::pulsed(p);
        }
    }
}

OptionsDirective options_of(const exg_options* o) {
    OptionsDirective opt;
    if (!o) return opt;
    opt.err_budget = o->err_budget;
    opt.krylov_eps = o->krylov_eps;
    opt.gmin = o->gmin;
    opt.m_max = o->m_max;
    if (!std::isnan(o->hmin)) opt.hmin = o->hmin;
    if (!std::isnan(o->hmax)) opt.hmax = o->hmax;
    return opt;
}

struct TranOut {
    std::vector<double> times, samples;
    int n_rec = 0;
    std::vector<double> t, h, err;
    std::vector<int> lu, rej, dims_off, dims;
    std::vector<double> wall;  // seconds since loop start after each accepted step
    double lu_s = 0.0;
};

void fill_tran(TranOut& o, const TransientResult& r) {
    o.n_rec = static_cast<int>(r.waveform.columns.size());
    o.times = r.waveform.times;
    for (const auto& row : r.waveform.samples) o.samples.insert(o.samples.end(), row.begin(), row.end());
    o.dims_off.push_back(0);
    for (const StepRecord& rec : r.records) {
        o.t.push_back(rec.t);
        o.h.push_back(rec.h_accepted);
        o.err.push_back(rec.err_norm);
        o.lu.push_back(rec.lu_count);
        o.rej.push_back(rec.rejects);
        o.dims.insert(o.dims.end(), rec.krylov_dims.begin(), rec.krylov_dims.end());
        o.dims_off.push_back(static_cast<int>(o.dims.size()));
    }
}

StepControl control_of(const exg_step_control* c) {
    StepControl ctl;
    ctl.err_budget = c->err_budget;
    ctl.alpha = c->alpha;
    ctl.beta = c->beta;
    ctl.grow_threshold = c->grow_threshold;
    ctl.grow_only_on_clean = c->grow_only_on_clean != 0;
    ctl.eps = c->eps;
    ctl.m_max = c->m_max;
    ctl.max_rejects = c->max_rejects;
    ctl.h_init = c->h_init;
    ctl.hmin = c->hmin;
    ctl.hmax = c->hmax;
    ctl.fixed_step = c->fixed_step != 0;
    ctl.correction.gamma = c->gamma;
    return ctl;
}

// ---- restated ER loop (integrate.cpp:368-480) over public API only ----------
MevpConfig mevp_config(const StepControl& ctl) {  // integrate.cpp:31-37
    MevpConfig cfg;
    cfg.eps = ctl.eps;
    cfg.m_max = ctl.m_max;
    return cfg;
}

// er_eval (integrate.cpp:238-265)
Vec er_eval_r(const Linearization& lin, const Factorization& G_fact, const Vec& x_k,
              ErWorkspace& ws, double h_try, const StepControl& ctl, std::vector<int>& dims) {
    Vec x_next = add(x_k, scaled(ws.gb_slope, h_try));
    if (norm2(ws.start) <= 1e-9 * (1.0 + norm_inf(x_k))) return x_next;
    const MevpConfig cfg = mevp_config(ctl);
    Vec value;
    bool need_fresh = true;
    if (ws.basis && h_try <= ws.basis->h_sub) {
        if (mevp_residual(*ws.basis, lin.G_k, h_try) < ctl.eps) {
            value = eval_at_scaled_h(*ws.basis, h_try);
            need_fresh = false;
        }
    }
    if (need_fresh) {
        MevpResult r = mevp_iks(G_fact, lin.C_k, ws.start, cfg, h_try);
        dims.push_back(r.basis.m);
        ws.basis = std::move(r.basis);
        value = std::move(r.value);
    }
    axpy(1.0, value, x_next);
    axpy(-1.0, ws.start, x_next);
    return x_next;
}

// error_from_deltaF (integrate.cpp:267-280)
double error_r(const Linearization& lin, const Factorization& G_fact, const Vec& deltaF,
               const StepControl& ctl, double h, std::vector<int>& dims) {
    if (norm_inf(deltaF) == 0.0) return 0.0;
    Vec w = G_fact.solve(deltaF);
    if (norm2(w) == 0.0) return 0.0;
    MevpResult r = mevp_iks(G_fact, lin.C_k, w, mevp_config(ctl), h);
    dims.push_back(r.basis.m);
    return norm_inf(sub(w, r.value));
}

// correction_from_deltaF (integrate.cpp:282-298)
Vec correction_r(const Linearization& lin, const Factorization& G_fact, const Vec& deltaF,
                 const StepControl& ctl, double h, double gamma, std::vector<int>& dims) {
    Vec zero(deltaF.size(), 0.0);
    if (gamma == 0.0) return zero;
    if (norm_inf(deltaF) == 0.0) return zero;
    Vec w = G_fact.solve(deltaF);
    Vec u = G_fact.solve(spmv(lin.C_k, w));
    Vec d = w;
    if (norm2(u) > 0.0) {
        MevpResult r = mevp_iks(G_fact, lin.C_k, u, mevp_config(ctl), h);
        dims.push_back(r.basis.m);
        axpy(1.0 / h, sub(r.value, u), d);
    }
    scale(d, gamma);
    return d;
}

double next_bp(const std::vector<double>& bps, double t) {  // integrate.cpp:361-364
    auto it = std::upper_bound(bps.begin(), bps.end(), t * (1.0 + 1e-12));
    return it == bps.end() ? std::numeric_limits<double>::infinity() : *it;
}

}  // namespace

extern "C" {

const char* ref_last_error(double* value) {
    if (value) *value = g_err_value;
    return g_err.c_str();
}

// ---- systems ---------------------------------------------------------------
int ref_system_from_elements(int n_elems, const exg_element* elems, int n_src,
                             const exg_source* srcs, const double* pwl_t, const double* pwl_v,
                             const exg_mos_model* models, const exg_options* opts,
                             void** out) {
    GUARD_BEGIN
    (void)n_src;
    NetlistDoc doc;
    doc.options = options_of(opts);
    if (opts && opts->has_tran) doc.tran = TranDirective{opts->tran_step, opts->tran_stop};
    doc.devices.reserve(static_cast<size_t>(n_elems));
    for (int i = 0; i < n_elems; ++i) {
        const exg_element& e = elems[i];
        DeviceCard card;
        card.name = std::to_string(i);
        switch (e.kind) {
            case EXG_EL_R: card.kind = DeviceKind::Resistor; break;
            case EXG_EL_C: card.kind = DeviceKind::Capacitor; break;
            case EXG_EL_L: card.kind = DeviceKind::Inductor; break;
            case EXG_EL_V: card.kind = DeviceKind::VoltageSource; break;
            case EXG_EL_I: card.kind = DeviceKind::CurrentSource; break;
            default: card.kind = DeviceKind::Mosfet; break;
        }
        const int nt = e.kind == EXG_EL_M ? 4 : 2;
        for (int k = 0; k < nt; ++k) card.nodes.push_back(node_name(e.nodes[k]));
        card.value = e.value;
        if (e.kind == EXG_EL_V || e.kind == EXG_EL_I) card.source = source_of(srcs[e.aux], pwl_t, pwl_v);
        if (e.kind == EXG_EL_M) {
            const exg_mos_model& m = models[e.aux];
            card.params = {{"VTH", m.vth}, {"KP", m.kp}, {"LAMBDA", m.lambda}, {"W", m.w},
                           {"L", m.l},     {"CGS0", m.cgs0}, {"CGD0", m.cgd0},
                           {"TYPE", m.pmos ? 1.0 : 0.0}};
        }
        doc.devices.push_back(std::move(card));
    }
    auto* sys = new MnaSystem(build_mna(doc));
    *out = sys;
    GUARD_END
}

// matrix-defined system (config 3): unknowns are nodes "N<i>"
int ref_system_from_csr(int n, const int* gp, const int* gi, const double* gx, int gnnz,
                        const int* cp, const int* ci, const double* cx, int cnnz, int n_in,
                        const int* bp, const int* bi, const double* bx, int bnnz,
                        const exg_source* srcs, const double* pwl_t, const double* pwl_v,
                        const exg_options* opts, void** out) {
    GUARD_BEGIN
    auto* sys = new MnaSystem();
    sys->n = n;
    sys->G_lin = make_csr(n, n, gnnz, gp, gi, gx);
    sys->C_lin = make_csr(n, n, cnnz, cp, ci, cx);
    sys->B = make_csr(n, n_in, bnnz, bp, bi, bx);
    for (int i = 0; i < n_in; ++i) sys->sources.push_back(source_of(srcs[i], pwl_t, pwl_v));
    for (int i = 0; i < n; ++i) {
        const std::string nm = "N" + std::to_string(i);
        sys->node_index[nm] = i;
        sys->unknown_names.push_back(nm);
    }
    sys->options = options_of(opts);
    if (opts && opts->has_tran) sys->tran = TranDirective{opts->tran_step, opts->tran_stop};
    *out = sys;
    GUARD_END
}

void ref_system_free(void* s) { delete static_cast<MnaSystem*>(s); }
int ref_system_n(void* s) { return static_cast<MnaSystem*>(s)->n; }
int ref_system_n_inputs(void* s) { return static_cast<MnaSystem*>(s)->n_inputs(); }

// which: 0 C, 1 G, 2 B.  Call with null outputs to query nnz and n_cols.
int ref_system_csr(void* s, int which, int* nnz, int* n_cols, int* rowptr, int* col, double* val) {
    const MnaSystem* sys = static_cast<MnaSystem*>(s);
    const SparseRealMatrix& m = which == 0 ? sys->C_lin : which == 1 ? sys->G_lin : sys->B;
    *nnz = m.nnz();
    *n_cols = m.n_cols();
    if (rowptr) std::memcpy(rowptr, m.row_offsets().data(), sizeof(int) * (m.n_rows() + 1));
    if (col) std::memcpy(col, m.col_indices().data(), sizeof(int) * m.nnz());
    if (val) std::memcpy(val, m.values().data(), sizeof(double) * m.nnz());
    return EXG_OK;
}

// unknown index of node "N<label>" (-1 if absent)
int ref_system_unknown_of_label(void* s, int label) {
    const MnaSystem* sys = static_cast<MnaSystem*>(s);
    auto it = sys->node_index.find("N" + std::to_string(label));
    return it == sys->node_index.end() ? -1 : it->second;
}

int ref_eval_sources(void* s, double t, double* u) {
    GUARD_BEGIN
    Vec v = eval_sources(*static_cast<MnaSystem*>(s), t);
    std::memcpy(u, v.data(), sizeof(double) * v.size());
    GUARD_END
}

int ref_dc_solve(void* s, double* x) {
    GUARD_BEGIN
    Vec v = dc_solve(*static_cast<MnaSystem*>(s));
    std::memcpy(x, v.data(), sizeof(double) * v.size());
    GUARD_END
}

int ref_evaluate(void* s, const double* x, int which, int* nnz, int* rowptr, int* col, double* val,
                 double* op5) {
    GUARD_BEGIN
    const MnaSystem& sys = *static_cast<MnaSystem*>(s);
    Linearization lin = evaluate(sys, Vec(x, x + sys.n));
    const SparseRealMatrix& A = which == 0 ? lin.C_k : lin.G_k;
    *nnz = A.nnz();
    if (rowptr) {
        std::memcpy(rowptr, A.row_offsets().data(), sizeof(int) * (A.n_rows() + 1));
        std::memcpy(col, A.col_indices().data(), sizeof(int) * A.nnz());
        std::memcpy(val, A.values().data(), sizeof(double) * A.nnz());
    }
    if (op5)
        for (size_t i = 0; i < lin.op.size(); ++i) {
            op5[5 * i] = lin.op[i].vgs_ref;
            op5[5 * i + 1] = lin.op[i].vds_ref;
            op5[5 * i + 2] = lin.op[i].id_ref;
            op5[5 * i + 3] = lin.op[i].gm;
            op5[5 * i + 4] = lin.op[i].gds;
        }
    GUARD_END
}

int ref_residual_F(void* s, const double* x_ref, const double* x, double* F) {
    GUARD_BEGIN
    const MnaSystem& sys = *static_cast<MnaSystem*>(s);
    Linearization lin = evaluate(sys, Vec(x_ref, x_ref + sys.n));
    Vec v = residual_F(lin, Vec(x, x + sys.n));
    std::memcpy(F, v.data(), sizeof(double) * v.size());
    GUARD_END
}

// ---- LU ----------------------------------------------------------------------
int ref_lu_factor(int n, const int* rowptr, const int* col, const double* val, int nnz,
                  double pivot_tol, void** out) {
    GUARD_BEGIN
    SparseRealMatrix A = make_csr(n, n, nnz, rowptr, col, val);
    *out = new Factorization(lu_factor(A, pivot_tol));
    GUARD_END
}

int ref_factor_from_arrays(int n, const int* Lp, const int* Li, const double* Lx, const int* Up,
                           const int* Ui, const double* Ux, const int* row_perm,
                           const int* col_perm, void** out) {
    GUARD_BEGIN
    auto* f = new Factorization();
    f->*get(FLower()) = make_csr(n, n, Lp[n], Lp, Li, Lx);
    f->*get(FUpper()) = make_csr(n, n, Up[n], Up, Ui, Ux);
    (f->*get(FRowPerm())).assign(row_perm, row_perm + n);
    (f->*get(FColPerm())).assign(col_perm, col_perm + n);
    f->*get(FSrcNnz()) = 0;
    *out = f;
    GUARD_END
}

void ref_factor_free(void* f) { delete static_cast<Factorization*>(f); }

int ref_factor_nnz(void* fp, int* nnz_l, int* nnz_u) {
    const Factorization* f = static_cast<Factorization*>(fp);
    *nnz_l = f->lower().nnz();
    *nnz_u = f->upper().nnz();
    return f->dimension();
}

int ref_factor_export(void* fp, int* Lp, int* Li, double* Lx, int* Up, int* Ui, double* Ux,
                      int* row_perm, int* col_perm) {
    const Factorization* f = static_cast<Factorization*>(fp);
    const int n = f->dimension();
    const auto& L = f->lower();
    const auto& U = f->upper();
    std::memcpy(Lp, L.row_offsets().data(), sizeof(int) * (n + 1));
    std::memcpy(Li, L.col_indices().data(), sizeof(int) * L.nnz());
    std::memcpy(Lx, L.values().data(), sizeof(double) * L.nnz());
    std::memcpy(Up, U.row_offsets().data(), sizeof(int) * (n + 1));
    std::memcpy(Ui, U.col_indices().data(), sizeof(int) * U.nnz());
    std::memcpy(Ux, U.values().data(), sizeof(double) * U.nnz());
    std::memcpy(row_perm, f->row_perm().data(), sizeof(int) * n);
    std::memcpy(col_perm, f->col_perm().data(), sizeof(int) * n);
    return EXG_OK;
}

int ref_solve(void* f, const double* b, double* x) {
    GUARD_BEGIN
    const Factorization* fa = static_cast<Factorization*>(f);
    Vec bv(b, b + fa->dimension());
    Vec r = fa->solve(bv);
    std::memcpy(x, r.data(), sizeof(double) * r.size());
    GUARD_END
}

int ref_apply(void* f, const double* x, double* y) {
    GUARD_BEGIN
    const Factorization* fa = static_cast<Factorization*>(f);
    Vec xv(x, x + fa->dimension());
    Vec r = fa->apply(xv);
    std::memcpy(y, r.data(), sizeof(double) * r.size());
    GUARD_END
}

int ref_spmv(int n_rows, int n_cols, int nnz, const int* rowptr, const int* col,
             const double* val, const double* x, double* y) {
    GUARD_BEGIN
    SparseRealMatrix A = make_csr(n_rows, n_cols, nnz, rowptr, col, val);
    Vec xv(x, x + n_cols);
    Vec r = spmv(A, xv);
    std::memcpy(y, r.data(), sizeof(double) * r.size());
    GUARD_END
}

// ---- Krylov ----------------------------------------------------------------
struct RefBasis {
    KrylovBasis b;
};

int ref_mevp_iks(void* f, int n, int cnnz, const int* cp, const int* ci, const double* cx,
                 const double* v, double h, double eps, int m_max, double* out, int* m,
                 int* happy, double* beta, double* h_next, void** basis_out) {
    GUARD_BEGIN
    SparseRealMatrix C = make_csr(n, n, cnnz, cp, ci, cx);
    MevpConfig cfg;
    cfg.eps = eps;
    cfg.m_max = m_max;
    Vec vv(v, v + n);
    MevpResult r = mevp_iks(*static_cast<Factorization*>(f), C, vv, cfg, h);
    std::memcpy(out, r.value.data(), sizeof(double) * n);
    *m = r.basis.m;
    *happy = r.basis.happy;
    *beta = r.basis.beta;
    *h_next = r.basis.h_next;
    if (basis_out) *basis_out = new RefBasis{std::move(r.basis)};
    GUARD_END
}

void ref_basis_free(void* b) { delete static_cast<RefBasis*>(b); }

int ref_basis_residual(void* b, int n, int gnnz, const int* gp, const int* gi, const double* gx,
                       double h, double* res) {
    GUARD_BEGIN
    SparseRealMatrix G = make_csr(n, n, gnnz, gp, gi, gx);
    *res = mevp_residual(static_cast<RefBasis*>(b)->b, G, h);
    GUARD_END
}

int ref_basis_eval(void* b, double h, double* out) {
    GUARD_BEGIN
    Vec r = eval_at_scaled_h(static_cast<RefBasis*>(b)->b, h);
    std::memcpy(out, r.data(), sizeof(double) * r.size());
    GUARD_END
}

// V columns (m+1 or m on happy) and the H_m / H_m^-1 of a basis
int ref_basis_get(void* bp, double* V, double* h_m, double* h_inv) {
    const KrylovBasis& b = static_cast<RefBasis*>(bp)->b;
    const size_t n = b.V.front().size();
    if (V)
        for (size_t j = 0; j < b.V.size(); ++j) std::memcpy(V + j * n, b.V[j].data(), sizeof(double) * n);
    if (h_m) std::memcpy(h_m, b.h_m.values().data(), sizeof(double) * b.m * b.m);
    if (h_inv && b.h_inv.size() == b.m)
        std::memcpy(h_inv, b.h_inv.values().data(), sizeof(double) * b.m * b.m);
    return static_cast<int>(b.V.size());
}

int ref_dense_expm(int n, const double* a, double* out) {
    GUARD_BEGIN
    DenseRealMatrix m(n);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) m.at(i, j) = a[i * n + j];
    DenseRealMatrix e = dense_expm(m);
    std::memcpy(out, e.values().data(), sizeof(double) * n * n);
    GUARD_END
}

int ref_dense_inverse(int n, const double* a, double* out, double* cond) {
    GUARD_BEGIN
    DenseRealMatrix m(n);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) m.at(i, j) = a[i * n + j];
    DenseRealMatrix e = dense_inverse(m, cond);
    std::memcpy(out, e.values().data(), sizeof(double) * n * n);
    GUARD_END
}

// ---- transient -----------------------------------------------------------------
int ref_transient(void* s, int method, const exg_step_control* c, double t_stop,
                  const int* rec_idx, int n_rec, void** out) {
    GUARD_BEGIN
    const MnaSystem& sys = *static_cast<MnaSystem*>(s);
    StepControl ctl = control_of(c);
    std::vector<std::string> names;
    for (int i = 0; i < n_rec; ++i) names.push_back(sys.unknown_names.at(rec_idx[i]));
    TransientResult r = transient(sys, method == EXG_METHOD_ERC ? Method::Erc : Method::Er, ctl,
                                  t_stop, names);
    auto* o = new TranOut();
    fill_tran(*o, r);
    *out = o;
    GUARD_END
}

// relative change of the device Jacobian between two linearizations
// (the product's jacobian_change, csrc/transient.cu, same arithmetic)
static double jacobian_change(const Linearization& a, const Linearization& b) {
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

// Restated ER/ERC loop (integrate.cpp:368-480).  fact != null: linear
// circuit, reuse that factorization for every step (G_k == G_lin,
// devices.cpp:190-192); fact == null: lu_factor(G_k) every step, as the
// reference.  max_steps > 0 stops after that many accepted steps (bounded CPU
// samples).  x0 != null replaces dc_solve.
int ref_transient_cached(void* s, void* fact, int method, const exg_step_control* c,
                         double t_stop, const int* rec_idx, int n_rec, long max_steps,
                         const double* x0, void** out) {
    GUARD_BEGIN
    const MnaSystem& sys = *static_cast<MnaSystem*>(s);
    const StepControl ctl = control_of(c);
    const bool erc = method == EXG_METHOD_ERC;
    TransientResult result;
    std::vector<int> rec;
    if (n_rec == 0)
        for (int i = 0; i < sys.n; ++i) rec.push_back(i);
    else
        rec.assign(rec_idx, rec_idx + n_rec);
    for (int i : rec) result.waveform.columns.push_back(sys.unknown_names[i]);
    auto emit = [&](double t, const Vec& x) {
        Vec row(rec.size());
        for (size_t i = 0; i < rec.size(); ++i) row[i] = x[rec[i]];
        result.waveform.times.push_back(t);
        result.waveform.samples.push_back(std::move(row));
    };

    Vec x = x0 ? Vec(x0, x0 + sys.n) : dc_solve(sys);
    emit(0.0, x);
    const std::vector<double> bps = source_breakpoints(sys, 0.0, t_stop);
    const double hint = sys.tran && sys.tran->step_hint > 0.0 ? sys.tran->step_hint : t_stop / 100.0;
    double h_nominal = ctl.h_init > 0.0 ? ctl.h_init : hint;
    h_nominal = std::min(h_nominal, ctl.hmax);
    const double hmin_eff = ctl.hmin > 0.0 ? ctl.hmin : t_stop * 1e-15;
    const double t_tiny = t_stop * 1e-12;
    const Factorization* cached = static_cast<Factorization*>(fact);

    double t = 0.0;
    long k = 0;
    Linearization lin;
    std::unique_ptr<Factorization> own;
    bool have_lin = false;
    const auto wall0 = std::chrono::steady_clock::now();
    std::vector<double> wall;
    while (t < t_stop - t_tiny) {
        if (max_steps > 0 && k >= max_steps) break;
        const double seg_end = std::min(next_bp(bps, t), t_stop);
        double h_try = std::min(h_nominal, seg_end - t);
        if (seg_end - t - h_try < t_tiny) h_try = seg_end - t;
        h_try = std::max(h_try, std::min(hmin_eff, seg_end - t));

        const std::uint64_t lu0 = lu_factor_count();
        // refactor policy (exg_step_control.refactor_threshold, BASELINE.json
        // config 4): the whole Linearization and its factorization stay frozen
        // until a device conductance moved by more than the threshold; 0 =
        // evaluate + lu_factor every step, as the reference
        {
            Linearization lin_new = evaluate(sys, x);
            bool refresh = true;
            if (have_lin && !cached && c->refactor_threshold > 0.0 &&
                jacobian_change(lin, lin_new) <= c->refactor_threshold)
                refresh = false;
            if (refresh) {
                lin = std::move(lin_new);
                if (!cached) own = std::make_unique<Factorization>(lu_factor(lin.G_k));
                have_lin = true;
            }
        }
        const Factorization& G_fact = cached ? *cached : *own;

        StepRecord rec_;
        SimState st{t, x, h_try, k};
        ErStepResult first = er_step(sys, lin, G_fact, st, ctl);  // er_begin + er_eval
        ErWorkspace ws = std::move(first.workspace);
        rec_.krylov_dims = first.rec.krylov_dims;
        const Vec F_k = residual_F(lin, x);

        int rejects = 0;
        Vec x_next = std::move(first.x_next);
        double err_norm = 0.0;
        bool first_attempt = true;
        while (true) {
            if (!first_attempt) x_next = er_eval_r(lin, G_fact, x, ws, h_try, ctl, rec_.krylov_dims);
            first_attempt = false;
            err_norm = 0.0;
            if (!sys.nonlinear_devices.empty()) {
                Vec deltaF = sub(residual_F(lin, x_next), F_k);
                err_norm = error_r(lin, G_fact, deltaF, ctl, h_try, rec_.krylov_dims);
                if (erc) {
                    Vec d = correction_r(lin, G_fact, deltaF, ctl, h_try, ctl.correction.gamma,
                                         rec_.krylov_dims);
                    axpy(1.0, d, x_next);
                }
            }
            if (ctl.fixed_step || err_norm <= ctl.err_budget) break;
            ++rejects;
            if (rejects > ctl.max_rejects)
                throw StepFailureError("transient: too many rejections at t=" + std::to_string(t));
            h_try *= ctl.alpha;
            if (h_try < hmin_eff)
                throw StepFailureError("transient: step size below HMIN at t=" + std::to_string(t));
        }
        rec_.t = t + h_try;
        rec_.h_accepted = h_try;
        rec_.lu_count = static_cast<int>(lu_factor_count() - lu0);
        rec_.rejects = rejects;
        rec_.err_norm = err_norm;
        x = std::move(x_next);
        t += h_try;
        emit(t, x);
        const bool grow = !ctl.fixed_step &&
                          (ctl.grow_only_on_clean ? rejects == 0 : rejects < ctl.grow_threshold);
        const bool clamped = h_try < h_nominal * (1.0 - 1e-12);
        if (rejects > 0) h_nominal = h_try;
        if (grow) h_nominal = std::min(ctl.beta * (clamped && rejects == 0 ? h_nominal : h_try), ctl.hmax);
        result.records.push_back(std::move(rec_));
        ++k;
        wall.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count());
    }
    auto* o = new TranOut();
    fill_tran(*o, result);
    o->wall = std::move(wall);
    *out = o;
    GUARD_END
}

void ref_tran_free(void* r) { delete static_cast<TranOut*>(r); }
int ref_tran_sizes(void* rp, int* n_times, int* n_rec, int* n_steps, int* n_dims) {
    const TranOut* r = static_cast<TranOut*>(rp);
    *n_times = static_cast<int>(r->times.size());
    *n_rec = r->n_rec;
    *n_steps = static_cast<int>(r->t.size());
    *n_dims = static_cast<int>(r->dims.size());
    return EXG_OK;
}
int ref_tran_get(void* rp, double* times, double* samples, double* t, double* h, int* lu,
                 int* rej, double* err, int* dims_off, int* dims) {
    const TranOut* r = static_cast<TranOut*>(rp);
    auto cp = [](auto* dst, const auto& v) {
        if (dst && !v.empty()) std::memcpy(dst, v.data(), sizeof(v[0]) * v.size());
    };
    cp(times, r->times);
    cp(samples, r->samples);
    cp(t, r->t);
    cp(h, r->h);
    cp(lu, r->lu);
    cp(rej, r->rej);
    cp(err, r->err);
    cp(dims_off, r->dims_off);
    cp(dims, r->dims);
    return EXG_OK;
}

int ref_tran_wall(void* rp, double* wall) {
    const TranOut* r = static_cast<TranOut*>(rp);
    if (wall && !r->wall.empty()) std::memcpy(wall, r->wall.data(), sizeof(double) * r->wall.size());
    return static_cast<int>(r->wall.size());
}

void ref_reset_lu_count() { reset_lu_factor_count(); }
unsigned long long ref_lu_count() { return lu_factor_count(); }

// write_waveform_csv of the reference's CLI (proj/tools/common.hpp:35-46), unmodified, on a
// row-major n_times x n_cols sample block: the checker of exg_write_waveform_csv
int ref_write_waveform_csv(const char* path, int n_times, int n_cols, const double* times,
                           const double* samples, const char* const* columns) {
    GUARD_BEGIN
    Waveform wf;
    for (int c = 0; c < n_cols; ++c) wf.columns.emplace_back(columns[c]);
    wf.times.assign(times, times + n_times);
    wf.samples.resize(n_times);
    for (int r = 0; r < n_times; ++r) wf.samples[r].assign(samples + (size_t)r * n_cols, samples + (size_t)(r + 1) * n_cols);
    exsim::cli::write_waveform_csv(path, wf);
    GUARD_END
}

}  // extern "C"
