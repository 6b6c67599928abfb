// extern "C" glue for the host-side API declared in include/exg_host.h.
#include <algorithm>
#include <vector>
#include <string>
#include <cstdio>
#include <thread>
#include <charconv>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>

#include "host.hpp"
#include "trsv_plan.hpp"


namespace {
thread_local std::string g_host_err;
}

const char* exg_host_last_error() { return g_host_err.c_str(); }

#define HOST_GUARD_BEGIN try {
#define HOST_GUARD_END                        \
    }                                         \
    catch (const exg::Error& e) {             \
        g_host_err = e.what;                  \
        return e.status;                      \
    }                                         \
    catch (const std::bad_alloc&) {           \
        g_host_err = "host allocation failed"; \
        return EXG_E_NOMEM;                   \
    }                                         \
    catch (const std::exception& e) {         \
        g_host_err = e.what();                \
        return EXG_E_CONTRACT;                \
    }                                         \
    return EXG_OK;

extern "C" {

const char* exg_host_error_message(void) { return g_host_err.c_str(); }

exg_status exg_system_generate(const exg_gen_params* p, exg_system** out) {
    HOST_GUARD_BEGIN
    auto* s = new exg_system();
    try {
        exg::generate(*p, s->sys);
    } catch (...) {
        delete s;
        throw;
    }
    *out = s;
    HOST_GUARD_END
}

exg_status exg_system_build(int n_elems, const exg_element* elems, int n_sources,
                            const exg_source* sources, int n_pwl, const double* pwl_t,
                            const double* pwl_v, int n_models, const exg_mos_model* models,
                            const exg_options* opts, exg_system** out) {
    HOST_GUARD_BEGIN
    auto* s = new exg_system();
    s->sys.opts = opts ? *opts : exg::default_options();
    s->sys.elems.assign(elems, elems + n_elems);
    s->sys.src_desc.assign(sources, sources + n_sources);
    if (n_pwl > 0) {
        s->sys.pwl_t.assign(pwl_t, pwl_t + n_pwl);
        s->sys.pwl_v.assign(pwl_v, pwl_v + n_pwl);
    }
    if (n_models > 0) s->sys.models.assign(models, models + n_models);
    try {
        exg::build_mna(s->sys);
    } catch (...) {
        delete s;
        throw;
    }
    *out = s;
    HOST_GUARD_END
}

void exg_system_free(exg_system* s) { delete s; }
int exg_system_n(const exg_system* s) { return s->sys.n; }
int exg_system_n_nodes(const exg_system* s) { return s->sys.n_nodes; }
int exg_system_n_inputs(const exg_system* s) { return s->sys.n_inputs(); }
int exg_system_n_mos(const exg_system* s) { return static_cast<int>(s->sys.mos.size()); }

exg_status exg_system_csr(const exg_system* s, int which, int* n_rows, int* n_cols, int* nnz,
                          const int** rowptr, const int** col, const double** val) {
    const exg::Csr* m = which == EXG_MAT_C ? &s->sys.C : which == EXG_MAT_G ? &s->sys.G
                                                     : which == EXG_MAT_B ? &s->sys.B : nullptr;
    if (!m) return EXG_E_CONTRACT;
    *n_rows = m->n_rows;
    *n_cols = m->n_cols;
    *nnz = m->nnz();
    *rowptr = m->rowptr.data();
    *col = m->col.data();
    *val = m->val.data();
    return EXG_OK;
}

exg_status exg_system_elements(const exg_system* s, int* n_elems, const exg_element** elems,
                               int* n_sources, const exg_source** sources, int* n_pwl,
                               const double** pwl_t, const double** pwl_v, int* n_models,
                               const exg_mos_model** models) {
    *n_elems = static_cast<int>(s->sys.elems.size());
    *elems = s->sys.elems.data();
    *n_sources = static_cast<int>(s->sys.src_desc.size());
    *sources = s->sys.src_desc.data();
    *n_pwl = static_cast<int>(s->sys.pwl_t.size());
    *pwl_t = s->sys.pwl_t.data();
    *pwl_v = s->sys.pwl_v.data();
    *n_models = static_cast<int>(s->sys.models.size());
    *models = s->sys.models.data();
    return EXG_OK;
}

exg_status exg_system_options(const exg_system* s, exg_options* out) {
    *out = s->sys.opts;
    return EXG_OK;
}

int exg_system_unknown_of_label(const exg_system* s, int label) {
    if (label < 0 || label >= static_cast<int>(s->sys.unknown_of_label.size())) return -1;
    return s->sys.unknown_of_label[label];
}

exg_status exg_sources_eval(const exg_system* s, double t, double* u) {
    HOST_GUARD_BEGIN
    const auto v = exg::eval_sources(s->sys, t);
    std::memcpy(u, v.data(), sizeof(double) * v.size());
    HOST_GUARD_END
}

exg_status exg_dc_solve(const exg_system* s, double* x) {
    HOST_GUARD_BEGIN
    const auto v = exg::dc_solve(s->sys);
    std::memcpy(x, v.data(), sizeof(double) * v.size());
    HOST_GUARD_END
}

exg_status exg_linearize(const exg_system* s, const double* x, int which, int* nnz, int* rowptr, int* col,
                         double* val, double* op5) {
    HOST_GUARD_BEGIN
    exg::Linearization lin;
    exg::evaluate(s->sys, std::vector<double>(x, x + s->sys.n), lin);
    if (which != 0 && which != 1) throw exg::Error{EXG_E_CONTRACT, "linearize: which must be C or G"};
    const exg::Csr& A = which == 0 ? lin.C : lin.G;
    *nnz = A.nnz();
    if (rowptr) {
        std::memcpy(rowptr, A.rowptr.data(), sizeof(int) * (A.n_rows + 1));
        std::memcpy(col, A.col.data(), sizeof(int) * A.nnz());
        std::memcpy(val, A.val.data(), sizeof(double) * A.nnz());
    }
    if (op5)
        for (size_t i = 0; i < lin.op.size(); ++i) {
            op5[5 * i] = lin.op[i].vgs_ref;
            op5[5 * i + 1] = lin.op[i].vds_ref;
            op5[5 * i + 2] = lin.op[i].id_ref;
            op5[5 * i + 3] = lin.op[i].gm;
            op5[5 * i + 4] = lin.op[i].gds;
        }
    HOST_GUARD_END
}

exg_status exg_residual_F_host(const exg_system* s, const double* x_ref, const double* x, double* F) {
    HOST_GUARD_BEGIN
    const int n = s->sys.n;
    exg::Linearization lin;
    exg::evaluate(s->sys, std::vector<double>(x_ref, x_ref + n), lin);
    const auto v = exg::residual_F(s->sys, lin, std::vector<double>(x, x + n));
    std::memcpy(F, v.data(), sizeof(double) * n);
    HOST_GUARD_END
}

int exg_breakpoints(const exg_system* s, double t0, double t1, double* out, int cap) {
    try {
        const auto v = exg::source_breakpoints(s->sys, t0, t1);
        for (int i = 0; i < static_cast<int>(v.size()) && i < cap; ++i) out[i] = v[i];
        return static_cast<int>(v.size());
    } catch (const exg::Error& e) {
        g_host_err = e.what;
        return -1;
    }
}

exg_status exg_lu_factor(int n, const int* rowptr, const int* col, const double* val,
                         double pivot_tol, exg_factor** out) {
    HOST_GUARD_BEGIN
    exg::Csr A;
    A.n_rows = A.n_cols = n;
    A.rowptr.assign(rowptr, rowptr + n + 1);
    A.col.assign(col, col + rowptr[n]);
    A.val.assign(val, val + rowptr[n]);
    auto* f = new exg_factor();
    try {
        exg::lu_factor(A, pivot_tol, f->f);
    } catch (...) {
        delete f;
        throw;
    }
    *out = f;
    HOST_GUARD_END
}

void exg_factor_free(exg_factor* f) { delete f; }

exg_status exg_factor_get(const exg_factor* fp, int* n, const int** Lp, const int** Li,
                          const double** Lx, const int** Up, const int** Ui, const double** Ux,
                          const int** row_perm, const int** col_perm) {
    const exg::Factor& f = fp->f;
    *n = f.n;
    *Lp = f.L.rowptr.data();
    *Li = f.L.col.data();
    *Lx = f.L.val.data();
    *Up = f.U.rowptr.data();
    *Ui = f.U.col.data();
    *Ux = f.U.val.data();
    *row_perm = f.row_perm.data();
    *col_perm = f.col_perm.data();
    return EXG_OK;
}

exg_status exg_factor_timing(const exg_factor* f, double* order_s, double* numeric_s) {
    *order_s = f->f.order_s;
    *numeric_s = f->f.numeric_s;
    return EXG_OK;
}

exg_status exg_step_control_from(const exg_system* s, exg_step_control* c) {
    const exg_options& o = s->sys.opts;
    c->err_budget = o.err_budget;
    c->alpha = 0.5;
    c->beta = 2.0;
    c->grow_threshold = 5;
    c->grow_only_on_clean = 1;
    c->eps = o.krylov_eps;
    c->m_max = o.m_max;
    c->max_rejects = 40;
    c->h_init = 0.0;
    c->hmin = std::isnan(o.hmin) ? 0.0 : o.hmin;
    c->hmax = std::isnan(o.hmax) ? std::numeric_limits<double>::infinity() : o.hmax;
    c->fixed_step = 0;
    c->method = EXG_METHOD_ER;
    c->gamma = 0.1;
    c->refactor_threshold = 0.0;
    return EXG_OK;
}


exg_status exg_aug_plan_solve(int upper, int n, const int* ptr, const int* col, const double* val,
                              const double* diag, const int* in_index, const int* params,
                              const double* b, double* x, long long* stats) {
    HOST_GUARD_BEGIN
    if (n < 0 || !ptr || (upper && !diag) || !in_index) throw exg::Error{EXG_E_CONTRACT, "exg_aug_plan_solve: bad arguments"};
    exg::AugParams prm;
    if (params) {
        prm.min_block = params[0];
        prm.max_block = params[1];
        prm.chunk_over = params[2];
        prm.recent = params[3];
        prm.chunk = params[4];
    }
    if (prm.max_block < 1 || prm.recent < 0 || prm.chunk < 1 || prm.chunk_over < prm.recent)
        throw exg::Error{EXG_E_CONTRACT, "exg_aug_plan_solve: bad plan parameters"};
    exg::AugPlan P;
    exg::build_aug_plan(upper != 0, n, ptr, col, val, diag, in_index, prm, P);
    if (b && x) {
        std::vector<double> out(P.n_aug, 0.0);
        exg::eval_aug_plan(P, upper != 0, b, out.data());
        std::memcpy(x, out.data(), sizeof(double) * n);
    }
    if (stats) {
        const long long st[8] = {P.orig_levels, P.levels,     P.n_blocks, P.block_rows,
                                 P.max_block,   P.n_partials, P.n_aug,    (long long)P.tasks.size() / 2};
        std::memcpy(stats, st, sizeof st);
    }
    HOST_GUARD_END
}

exg_status exg_stream_plan_solve(int upper, int n, const int* ptr, const int* col, const double* val,
                                 const double* diag, const int* in_index, const int* out_index,
                                 const int* params, int n_warps, const double* b, double* x,
                                 double* final_out, double coef, const double* add, long long* stats) {
    HOST_GUARD_BEGIN
    if (n < 0 || !ptr || (upper && !diag) || !in_index || n_warps < 1)
        throw exg::Error{EXG_E_CONTRACT, "exg_stream_plan_solve: bad arguments"};
    exg::AugParams prm = exg::stream_aug_params();
    if (params) {
        prm.min_block = params[0];
        prm.max_block = params[1];
    }
    if (prm.max_block < 1) throw exg::Error{EXG_E_CONTRACT, "exg_stream_plan_solve: bad plan parameters"};
    exg::AugPlan P;
    exg::build_aug_plan(upper != 0, n, ptr, col, val, diag, in_index, prm, P);
    exg::StreamParams sp;
    sp.n_warps = n_warps;
    sp.min_tasks_per_warp = 0;  // exactly the caller's warp count
    exg::stream_params_env(sp);
    exg::StreamPlan S;
    exg::build_stream_plan(P, upper != 0, out_index, sp, S);
    if (b && x) {
        std::vector<double> out(S.n_aug + 1, 0.0);
        exg::eval_stream_plan(S, upper != 0, b, out.data(), final_out, coef, add);
        std::memcpy(x, out.data(), sizeof(double) * n);
    }
    if (stats) {
        const long long st[10] = {P.orig_levels, S.levels,    S.n_aug,   S.n_tasks,           S.n_rows,
                                  S.n_entries,   S.n_slots,   (long long)S.data.size(), S.max_record, P.n_partials};
        std::memcpy(stats, st, sizeof st);
    }
    HOST_GUARD_END
}

exg_status exg_write_waveform_csv(const char* path, int n_times, int n_cols, const double* times,
                                  const double* samples, const char* const* columns, int threads) {
    HOST_GUARD_BEGIN
    if (!path || n_times < 0 || n_cols < 0 || (n_times && !times) || (n_times && n_cols && !samples) ||
        (n_cols && !columns))
        throw exg::Error{EXG_E_CONTRACT, "exg_write_waveform_csv: bad arguments"};
    FILE* f = std::fopen(path, "wb");
    if (!f) throw exg::Error{EXG_E_CONTRACT, std::string("cannot write '") + path + "'"};
    std::string head = "time";
    for (int c = 0; c < n_cols; ++c) {
        head += ',';
        head += columns[c];
    }
    head += '\n';
    // rows are independent: each thread formats a contiguous slice into its own buffer
    unsigned T = threads > 0 ? (unsigned)threads : std::max(1u, std::thread::hardware_concurrency());
    T = (unsigned)std::max<long long>(1, std::min<long long>(T, ((long long)n_times * (n_cols + 1) + 65535) / 65536));
    std::vector<std::string> part(T);
    auto work = [&](unsigned t) {
        const long long r0 = (long long)n_times * t / T, r1 = (long long)n_times * (t + 1) / T;
        std::string& o = part[t];
        o.reserve((size_t)(r1 - r0) * (size_t)(n_cols + 1) * 20);
        char buf[48];
        // std::to_chars(general, 17) prints what printf("%.17g") prints in the C locale (both are
        // correctly rounded to 17 significant digits; same exponent and zero-stripping rules)
        auto put = [&](double v) {
            const auto res = std::to_chars(buf, buf + sizeof buf, v, std::chars_format::general, 17);
            o.append(buf, (size_t)(res.ptr - buf));
        };
        for (long long r = r0; r < r1; ++r) {
            put(times[r]);
            const double* row = samples + (size_t)r * n_cols;
            for (int c = 0; c < n_cols; ++c) {
                o += ',';
                put(row[c]);
            }
            o += '\n';
        }
    };
    std::vector<std::thread> th;
    for (unsigned t = 1; t < T; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
    bool ok = std::fwrite(head.data(), 1, head.size(), f) == head.size();
    for (unsigned t = 0; ok && t < T; ++t) ok = std::fwrite(part[t].data(), 1, part[t].size(), f) == part[t].size();
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) throw exg::Error{EXG_E_CONTRACT, std::string("cannot write '") + path + "'"};
    HOST_GUARD_END
}

}  // extern "C"
