/*
 * exg_host.h — host-side C ABI of the exsim-B200 framework.
 *
 * Everything here runs on the CPU: synthetic circuit generation, MNA assembly,
 * the setup-time sparse LU and the transient step-control loop that drives the
 * device hot path declared in exg.h.  These mirror the reference's host layers
 * so that a caller of the reference finds the same entry points:
 *
 *   exg_system_build      <- exsim::build_mna          proj/core/src/mna.cpp:22-165
 *   exg_sources_eval      <- exsim::eval_sources       proj/core/src/mna.cpp:167-171
 *   exg_breakpoints       <- exsim::source_breakpoints proj/core/src/mna.cpp:173-180
 *   exg_lu_factor         <- exsim::lu_factor          proj/core/src/sparse_lu.cpp:134-253
 *   exg_transient         <- exsim::transient (ER/ERC) proj/core/src/integrate.cpp:368-480
 *   exg_dc_solve          <- exsim::dc_solve           proj/core/src/integrate.cpp:92-115
 *   exg_linearize         <- exsim::evaluate           proj/core/src/devices.cpp:122-200
 *   exg_residual_F_host   <- exsim::residual_F         proj/core/src/devices.cpp:202-233
 *
 * exg_lu_factor produces factors bit-identical to the reference's lu_factor
 * (same minimum-degree order, same pivots, same values) but orders with a heap
 * instead of the reference's O(n) scan per pivot (sparse_lu.cpp:66-75).
 *
 * Plain C types only; all arrays are caller-owned unless documented otherwise.
 */
#ifndef EXG_HOST_H
#define EXG_HOST_H

#include <stddef.h>
#include <stdint.h>

#include "exg.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ---- circuit description (element list) -------------------------------- */

enum {
    EXG_EL_R = 0, /* resistor   nodes[0..1], value = ohm           */
    EXG_EL_C = 1, /* capacitor  nodes[0..1], value = farad         */
    EXG_EL_L = 2, /* inductor   nodes[0..1], value = henry         */
    EXG_EL_V = 3, /* voltage source nodes[0..1], aux = source id   */
    EXG_EL_I = 4, /* current source nodes[0..1], aux = source id   */
    EXG_EL_M = 5  /* mosfet d,g,s,b = nodes[0..3], aux = model id  */
};

enum { EXG_SRC_DC = 0, EXG_SRC_PWL = 1, EXG_SRC_PULSE = 2 };

/* node labels: >= 0 a circuit node (named "N<label>"), -1 ground "0",
 * -2 unused slot.  Unknown numbering is by first appearance, as in
 * build_mna (mna.cpp:28-41). */
typedef struct exg_element {
    int32_t kind;
    int32_t nodes[4];
    int32_t aux;
    double value;
} exg_element;

typedef struct exg_source {
    int32_t kind;
    int32_t pwl_off; /* into the circuit's pwl_t / pwl_v arrays */
    int32_t pwl_len;
    int32_t pad;
    double dc;
    double v1, v2, delay, rise, fall, width, period; /* PULSE */
} exg_source;

typedef struct exg_mos_model {
    double vth, kp, lambda, w, l, cgs0, cgd0;
    int32_t pmos;
    int32_t pad;
} exg_mos_model;

/* .OPTIONS / .TRAN values (netlist.hpp:40-49); NaN hmin/hmax = unset */
typedef struct exg_options {
    double err_budget;
    double krylov_eps;
    double gmin;
    int32_t m_max;
    int32_t has_tran;
    double hmin;
    double hmax;
    double tran_step;
    double tran_stop;
} exg_options;

/* ---- synthetic workloads (the five BASELINE.json configs) --------------- */

typedef struct exg_gen_params {
    int32_t config; /* 0..4 */
    int32_t width;  /* grid width  (0 = the config's full size) */
    int32_t height; /* grid height (0 = width) */
    int32_t n;      /* config 3: matrix dimension (0 = 11417) */
    uint64_t seed;  /* 0 = 1000 + config */
    int32_t chains; /* config 4: number of inverter chains (0 = default) */
    int32_t stages; /* config 4: stages per chain (0 = default) */
} exg_gen_params;

typedef struct exg_system exg_system;

exg_status exg_system_generate(const exg_gen_params* p, exg_system** out);
/* MNA assembly from an element list (mirror of build_mna). */
exg_status exg_system_build(int n_elems, const exg_element* elems, int n_sources,
                            const exg_source* sources, int n_pwl, const double* pwl_t,
                            const double* pwl_v, int n_models, const exg_mos_model* models,
                            const exg_options* opts, exg_system** out);
void exg_system_free(exg_system* s);

int exg_system_n(const exg_system* s);
int exg_system_n_nodes(const exg_system* s);
int exg_system_n_inputs(const exg_system* s);
int exg_system_n_mos(const exg_system* s); /* MOSFET count */
/* which: EXG_MAT_C / EXG_MAT_G / EXG_MAT_B.  Borrowed pointers. */
exg_status exg_system_csr(const exg_system* s, int which, int* n_rows, int* n_cols, int* nnz,
                          const int** rowptr, const int** col, const double** val);
/* element list the system was assembled from (count 0 for matrix-defined) */
exg_status exg_system_elements(const exg_system* s, int* n_elems, const exg_element** elems,
                               int* n_sources, const exg_source** sources, int* n_pwl,
                               const double** pwl_t, const double** pwl_v, int* n_models,
                               const exg_mos_model** models);
exg_status exg_system_options(const exg_system* s, exg_options* out);
/* unknown index of a node label (-1 if the label is not a node) */
int exg_system_unknown_of_label(const exg_system* s, int label);

/* u(t), one entry per input (eval_sources, mna.cpp:167-171) */
exg_status exg_sources_eval(const exg_system* s, double t, double* u);
/* breakpoints strictly inside (t0,t1), ascending, deduplicated.  Returns the
 * count; writes at most cap values. */
int exg_breakpoints(const exg_system* s, double t0, double t1, double* out, int cap);

/* ---- setup LU ---------------------------------------------------------- */

/* DC operating point (Newton + gmin stepping), bit-identical to dc_solve. */
exg_status exg_dc_solve(const exg_system* s, double* x);
/* Linearization at x: which = EXG_MAT_C / EXG_MAT_G selects C_k / G_k.
 * Call with rowptr == NULL to get *nnz; op5 (optional) receives the MOSFET
 * operating points (vgs_ref, vds_ref, id_ref, gm, gds) per device. */
exg_status exg_linearize(const exg_system* s, const double* x, int which, int* nnz, int* rowptr,
                         int* col, double* val, double* op5);
/* F(x) with the stamps frozen at the linearization point x_ref */
exg_status exg_residual_F_host(const exg_system* s, const double* x_ref, const double* x, double* F);

typedef struct exg_factor exg_factor;

/* Bit-identical to exsim::lu_factor(A, pivot_tol). */
exg_status exg_lu_factor(int n, const int* rowptr, const int* col, const double* val,
                         double pivot_tol, exg_factor** out);
void exg_factor_free(exg_factor* f);
/* borrowed pointers; L with explicit unit diagonal, U with its diagonal, both
 * CSR in pivot coordinates (sparse_lu.cpp:235-248) */
exg_status exg_factor_get(const exg_factor* f, int* n, const int** Lp, const int** Li,
                          const double** Lx, const int** Up, const int** Ui, const double** Ux,
                          const int** row_perm, const int** col_perm);
/* seconds spent in ordering / numeric phases of the last exg_lu_factor */
exg_status exg_factor_timing(const exg_factor* f, double* order_s, double* numeric_s);

/* ---- FAST-solve plan (diagnostics / tests) ------------------------------- *
 * Builds the blocked augmented system the FAST triangular solve runs
 * (paper_1511_04515_b200/csrc/trsv_plan.hpp; replaces the row-by-row sweep of
 * Factorization::solve, sparse_lu.cpp:255-291, for one triangle) and
 * evaluates it on the CPU in plan order.  ptr/col/val: the STRICTLY
 * triangular part in pivot coordinates; diag: U's diagonal (upper only);
 * in_index: where row r reads its right-hand side.  params (may be null):
 * {min_block, max_block, chunk_over, recent, chunk}.  x: n results.
 * stats (may be null): {orig_levels, levels, n_blocks, block_rows,
 * max_block, n_partials, n_aug, n_tasks}. */
exg_status exg_aug_plan_solve(int upper, int n, const int* ptr, const int* col, const double* val,
                              const double* diag, const int* in_index, const int* params,
                              const double* b, double* x, long long* stats);

/* The same augmented system cut into the per-warp record streams k_trsv4
 * consumes (trsv_plan.hpp), evaluated on the CPU in global task order with the
 * kernel's arithmetic.  out_index (may be null): epilogue index per row
 * (U: col_perm); final_out/add (may be null), coef: the fused epilogue
 * final_out[q] = add[q] + coef * x.  params (may be null): {min_block,
 * max_block}.  stats (may be null): {orig_levels, levels, n_aug, n_tasks,
 * n_rows, n_entries, n_slots, stream bytes, max record bytes, n_partials}. */
exg_status exg_stream_plan_solve(int upper, int n, const int* ptr, const int* col, const double* val,
                                 const double* diag, const int* in_index, const int* out_index,
                                 const int* params, int n_warps, const double* b, double* x,
                                 double* final_out, double coef, const double* add, long long* stats);

/* ---- transient (the reference's time-stepping loop, ER / ERC) ------------ */

enum { EXG_METHOD_ER = 1, EXG_METHOD_ERC = 2 };

/* StepControl (integrate.hpp:27-46) */
typedef struct exg_step_control {
    double err_budget;
    double alpha;
    double beta;
    int32_t grow_threshold;
    int32_t grow_only_on_clean;
    double eps;
    int32_t m_max;
    int32_t max_rejects;
    double h_init;
    double hmin;
    double hmax;
    int32_t fixed_step;
    int32_t method;
    double gamma; /* ERC correction */
    /* Nonlinear circuits: re-linearise and refactor G_k only when the device
     * Jacobian (the stamped conductances gm, gds of all devices) changed by
     * more than this relative amount in the Euclidean norm since the last
     * factorization; the whole Linearization (G_k, C_k, operating points)
     * stays frozen in between.  0 = every step, as the reference
     * (integrate.cpp:419-421).  BASELINE.json config 4 names 0.1. */
    double refactor_threshold;
} exg_step_control;

/* defaults of StepControl seeded from the options (step_control_from,
 * integrate.cpp:19-27) */
exg_status exg_step_control_from(const exg_system* s, exg_step_control* out);

typedef struct exg_tran_result exg_tran_result;

/* Full transient from the DC point to t_stop on the device context.  rec_idx
 * lists the unknowns to record (n_rec == 0: all unknowns, as the reference).
 * The factorization of G is computed once (linear circuits) with
 * exg_lu_factor and uploaded; its cost is reported separately. */
exg_status exg_transient(exg_ctx* ctx, const exg_system* sys, const exg_step_control* ctl,
                         double t_stop, const int* rec_idx, int n_rec, exg_tran_result** out);
void exg_tran_result_free(exg_tran_result* r);
int exg_tran_n_times(const exg_tran_result* r);
int exg_tran_n_rec(const exg_tran_result* r);
const double* exg_tran_times(const exg_tran_result* r);
const double* exg_tran_samples(const exg_tran_result* r); /* n_times x n_rec row-major */
int exg_tran_n_steps(const exg_tran_result* r);
/* per step: t, h_accepted, lu_count, rejects, err_norm, dims offsets */
exg_status exg_tran_records(const exg_tran_result* r, double* t, double* h, int* lu_count,
                            int* rejects, double* err_norm, int* dims_off);
int exg_tran_n_dims(const exg_tran_result* r);
const int* exg_tran_dims(const exg_tran_result* r);
/* wall seconds: setup LU, DC solve, stepping loop */
exg_status exg_tran_timing(const exg_tran_result* r, double* lu_s, double* dc_s, double* loop_s);


/* Waveform CSV, byte for byte what the reference's CLI writes
 * (write_waveform_csv, proj/tools/common.hpp:35-46: a "time,<columns>" header,
 * then one line per time point, every value as printf("%.17g")).  samples is
 * row-major n_times x n_cols (exg_tran_samples' layout).  Rows are formatted
 * by `threads` host threads (<= 0: all cores) into one buffered write; SURVEY
 * 8(f).4.  EXG_E_CONTRACT when the file cannot be written. */
exg_status exg_write_waveform_csv(const char* path, int n_times, int n_cols, const double* times,
                                  const double* samples, const char* const* columns, int threads);
/* the same for a transient's recorded waveform (columns: exg_tran_n_rec names, the
 * reference's Waveform::columns) */
exg_status exg_tran_write_csv(const exg_tran_result* r, const char* path, const char* const* columns, int threads);

#ifdef __cplusplus
}
#endif

#endif /* EXG_HOST_H */
