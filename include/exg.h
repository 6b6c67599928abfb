/*
 * exg.h — the device-side C ABI of the exsim-B200 hot path (sm_100a, fp64).
 *
 * This is the drop-in boundary: the reference's transient loop
 * (proj/core/src/integrate.cpp:368-480) keeps its control flow and calls these
 * entry points where it calls the hot-path functions today.  Each entry names
 * the reference interface it replaces:
 *
 *   exg_spmv          <- exsim::spmv                   sparse_matrix.hpp:56, sparse_matrix.cpp:69-82
 *   exg_solve         <- exsim::Factorization::solve   sparse_lu.hpp:28-29, sparse_lu.cpp:255-291
 *   exg_apply         <- exsim::Factorization::apply   sparse_lu.hpp:31-32, sparse_lu.cpp:293-304
 *   exg_mevp_iks      <- exsim::mevp_iks               krylov.hpp:51-52, krylov.cpp:177-182 (+ :103-173)
 *   exg_basis_residual<- exsim::mevp_residual          krylov.hpp:58, krylov.cpp:191-205
 *   exg_basis_eval    <- exsim::eval_at_scaled_h       krylov.hpp:63, krylov.cpp:207-215
 *   exg_er_begin      <- er_begin (anon. namespace)    integrate.cpp:213-233
 *   exg_er_eval       <- er_eval  (anon. namespace)    integrate.cpp:238-265
 *   exg_er_step       <- exsim::er_step                integrate.hpp:114-116, integrate.cpp:302-316
 *
 * Ownership: every host array is copied during the call and never retained.
 * Pointers flagged EXG_PTR_DEVICE must be device memory of the context's
 * device.  Errors: each call returns an exg_status that maps 1:1 onto the
 * reference's exception hierarchy (errors.hpp:9-84); exg_last_error returns
 * the message.  Threading: one context per host thread; contexts are
 * independent (own stream, own memory).
 *
 * No torch types cross this boundary.
 */
#ifndef EXG_H
#define EXG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum exg_status {
    EXG_OK = 0,
    EXG_E_CONTRACT = 1,          /* exsim::ContractError */
    EXG_E_NONFINITE = 2,         /* exsim::NonFiniteError */
    EXG_E_SINGULAR = 3,          /* exsim::SingularMatrixError */
    EXG_E_ZERO_START = 4,        /* exsim::ZeroStartVectorError */
    EXG_E_NO_CONVERGENCE = 5,    /* exsim::NoConvergenceError (last residual in info) */
    EXG_E_SINGULAR_REDUCED = 6,  /* exsim::SingularReducedMatrixError */
    EXG_E_NO_DC = 7,             /* exsim::NoDcConvergenceError */
    EXG_E_STEP_FAILURE = 8,      /* exsim::StepFailureError */
    EXG_E_CUDA = 100,            /* CUDA runtime failure */
    EXG_E_NOMEM = 101            /* host or device allocation failure */
} exg_status;

enum { EXG_MAT_C = 0, EXG_MAT_G = 1, EXG_MAT_B = 2 };
enum { EXG_PTR_HOST = 0, EXG_PTR_DEVICE = 1 };

/* triangular-solve arithmetic: EXACT keeps the reference's row-sequential
 * accumulation for every row (bit-identical to Factorization::solve); FAST
 * splits long rows across a warp with a fixed-order reduction (deterministic,
 * not bit-identical). */
enum { EXG_TRSV_EXACT = 0, EXG_TRSV_FAST = 1 };
/* residual weight of the Arnoldi test: the reference's ||P^T L U Q^T v|| (APPLY,
 * krylov.cpp:238) or ||G v|| (GSPMV, the operator mevp_residual uses). */
enum { EXG_WEIGHT_APPLY = 0, EXG_WEIGHT_GSPMV = 1 };
/* Arnoldi loop execution: EAGER launches every iteration from the host and
 * reads the control block back after each one; GRAPH runs the whole loop as
 * one CUDA graph (a conditional WHILE node whose body is one iteration; the
 * device decides when to stop) and reads the control block back once per
 * MEVP.  Same kernels, same results. */
enum { EXG_LOOP_GRAPH = 0, EXG_LOOP_EAGER = 1 };

typedef struct exg_ctx exg_ctx;

/* MevpConfig (krylov.hpp:13-19) */
typedef struct exg_mevp_cfg {
    double eps;
    int32_t m_max;
    int32_t check_stride;
    double breakdown_tol;
} exg_mevp_cfg;

/* Scalars of the KrylovBasis (krylov.hpp:27-39) the caller needs. */
typedef struct exg_mevp_info {
    int32_t m;
    int32_t happy;
    double beta;
    double h_next;
    double h_sub;
    double last_residual;
} exg_mevp_info;

typedef struct exg_options_dev {
    int32_t trsv_mode;   /* EXG_TRSV_* */
    int32_t weight_mode; /* EXG_WEIGHT_* */
    int32_t loop_mode;   /* EXG_LOOP_* */
} exg_options_dev;

typedef struct exg_counters {
    int64_t kernel_launches; /* launches of this library's kernels */
    int64_t arnoldi_iters;   /* Arnoldi iterations run */
    int64_t mevp_calls;
    int64_t trsv_calls;      /* triangular-solve pairs */
    int32_t l_levels;        /* critical-path level count of L */
    int32_t u_levels;        /* of U */
    int64_t nnz_l;           /* off-diagonal entries stored on the device */
    int64_t nnz_u;
    int64_t graph_launches;  /* Arnoldi-loop graph launches */
    int64_t graph_builds;    /* graph captures + instantiations */
    int32_t l_schedule;      /* level schedule of L: 0 ASAP, 1 ALAP */
    int32_t u_schedule;      /* of U */
    int64_t mgs_passes;      /* algorithmic n-vector passes of orthogonalize: J + 2 per call
                                with J basis vectors, + J + 1 per reorthogonalisation */
    int64_t reorths;         /* reorthogonalisation passes (krylov.cpp:59) */
    /* FAST plan actually run (0 where the level-run plan is used): dependent
     * levels, warp tasks and stream bytes of the blocked augmented system */
    int32_t fast_levels_l, fast_levels_u;
    int64_t fast_tasks_l, fast_tasks_u;
    int64_t fast_bytes_l, fast_bytes_u;
} exg_counters;

exg_status exg_create(int device, exg_ctx** out);
void exg_destroy(exg_ctx* ctx);
/* copies the last error message; returns the status of the last failure */
exg_status exg_last_error(exg_ctx* ctx, char* buf, size_t len);
exg_status exg_set_options(exg_ctx* ctx, const exg_options_dev* opt);

/* device-resident CSR (int32 offsets/cols, fp64 values) */
exg_status exg_set_csr(exg_ctx* ctx, int which, int n_rows, int n_cols, int nnz,
                       const int* rowptr, const int* col, const double* val);
/* same pattern, new values (host array of nnz) */
exg_status exg_update_values(exg_ctx* ctx, int which, const double* val);
/* L (unit diagonal stored explicitly), U (with diagonal), CSR in pivot
 * coordinates as lu_factor assembles them; row_perm[k]/col_perm[k] give the
 * original row/col at elimination position k.  Runs the host level analysis. */
exg_status exg_set_factors(exg_ctx* ctx, int n, const int* Lp, const int* Li, const double* Lx,
                           const int* Up, const int* Ui, const double* Ux, const int* row_perm,
                           const int* col_perm);

/* y = A x */
exg_status exg_spmv(exg_ctx* ctx, int which, const double* x, double* y, int ptr_kind);
/* x = Q U^{-1} L^{-1} P b */
exg_status exg_solve(exg_ctx* ctx, const double* b, double* x, int ptr_kind);
/* y = P^T L U Q^T x */
exg_status exg_apply(exg_ctx* ctx, const double* x, double* y, int ptr_kind);

/* e^{hJ} v by invert-Krylov Arnoldi (J = -C^{-1} G).  The converged basis is
 * kept in the context for exg_basis_residual / exg_basis_eval. */
exg_status exg_mevp_iks(exg_ctx* ctx, const double* v, double h, const exg_mevp_cfg* cfg,
                        double* out, exg_mevp_info* info, int ptr_kind);
exg_status exg_basis_residual(exg_ctx* ctx, double h, double* residual);
exg_status exg_basis_eval(exg_ctx* ctx, double h, double* out, int ptr_kind);

/* ER step on the device (linear part; integrate.cpp:213-265).  x_k, u_k,
 * u_k1 (n_inputs each) are read from ptr_kind memory; the step keeps x_k,
 * start, gb_slope and the basis resident.  exg_er_eval writes x_next and
 * appends the Krylov dimension of a fresh basis to *m_out (-1 when the
 * start-vector early-out or the cached basis was used). */
exg_status exg_er_begin(exg_ctx* ctx, const double* x_k, const double* u_k, const double* u_k1,
                        double h, int ptr_kind);
exg_status exg_er_eval(exg_ctx* ctx, double h_try, const exg_mevp_cfg* cfg, double* x_next,
                       int* m_out, exg_mevp_info* info, int ptr_kind);
/* er_begin + er_eval in one call (er_step, integrate.cpp:302-316) */
exg_status exg_er_step(exg_ctx* ctx, const double* x_k, const double* u_k, const double* u_k1,
                       double h, const exg_mevp_cfg* cfg, double* x_next, int* m_out,
                       int ptr_kind);

/* ---- nonlinear devices (config 4; devices.cpp, integrate.cpp:267-298) ----
 * exg_set_devices: MOSFET table — nodes4 = (drain, gate, source, bulk)
 * unknown indices per device (-1 ground), par6 = (VTH, KP, LAMBDA, W, L,
 * PMOS flag).  exg_set_oppoints: the frozen operating point of the current
 * linearization, op5 = (vgs_ref, vds_ref, id_ref, gm, gds) per device
 * (DeviceOperatingPoint, devices.hpp:14-26).  With devices set, exg_er_begin
 * uses F(x_k) = exg_residual_F(x_k) (devices.cpp:202-233). */
exg_status exg_set_devices(exg_ctx* ctx, int n_mos, const int* nodes4, const double* par6);
exg_status exg_set_oppoints(exg_ctx* ctx, const double* op5);
exg_status exg_residual_F(exg_ctx* ctx, const double* x, double* F, int ptr_kind);
/* after exg_er_eval: err_norm = ||e_rr||_inf of error_from_deltaF; with erc,
 * x_next += correction_from_deltaF(gamma).  dims receives the Krylov
 * dimensions of the MEVPs run (at most 2). */
exg_status exg_er_nonlinear(exg_ctx* ctx, double h, const exg_mevp_cfg* cfg, int erc, double gamma,
                            double* err_norm, int* dims, int* n_dims);

/* out[i] = x_next[idx[i]] of the last ER evaluation (probed nodes) */
exg_status exg_gather(exg_ctx* ctx, const int* idx, int k, double* out);

/* Per-kernel-class device time measured with CUDA events on the context's
 * stream (profiling mode only; adds one event pair per launch). */
enum {
    EXG_K_TRSV_L = 0,
    EXG_K_TRSV_U = 1,
    EXG_K_SPMV = 2,
    EXG_K_MGS = 3,
    EXG_K_DENSE = 4,
    EXG_K_WEIGHT = 5,
    EXG_K_OTHER = 6,
    EXG_K_CLASSES = 7
};
typedef struct exg_kernel_times {
    double ms[EXG_K_CLASSES];
    int64_t count[EXG_K_CLASSES];
} exg_kernel_times;
exg_status exg_profile_enable(exg_ctx* ctx, int on);
/* debug: one solve with per-row %globaltimer stamps; times holds 10n values:
 * (start, end) of the warp-task sweeps for L then U (4n), then (start,
 * far-done, end) of the cluster sweeps for L then U (6n); zero = not run there */
exg_status exg_debug_trace_solve(exg_ctx* ctx, const double* b, unsigned long long* times);
/* debug / test: one orthogonalize step (krylov.cpp:46-78) in isolation: V is a
 * host n x (j + 1) column-major orthonormal basis, w the vector to
 * orthogonalise; hcol receives the j + 2 Hessenberg entries, v_next the
 * normalised remainder (untouched on a happy breakdown), info = {happy,
 * reorthogonalised}.  The kernel is the one the context's mode runs. */
exg_status exg_debug_orthogonalize(exg_ctx* ctx, int n, int j, const double* V, const double* w,
                                   double breakdown_tol, double* hcol, double* v_next, int* info);
/* debug / test: y = C x on host vectors through the FAST-mode SpMV kernel of
 * the Arnoldi loop (sparse_matrix.cpp:69-82 up to the order of the additions:
 * four lanes per row); C must be square. */
exg_status exg_debug_spmv_fast(exg_ctx* ctx, const double* x, double* y);
/* debug / test: dense_expm (dense_matrix.cpp:185-225) of a host m x m row-major
 * matrix through the dense-block kernel, bit-identical to the reference. */
exg_status exg_debug_dense_expm(exg_ctx* ctx, int m, const double* A, double* E);
/* debug: one FAST solve pair over the stream plan (k_trsv4) with 5 values per
 * warp task {level, begin, dependencies ready, published (ns, %globaltimer),
 * warp}, L's tasks then U's.  counts (6): tasks of L, U; warps of L, U; stream
 * bytes of L, U.  Call with times == NULL to size the buffer. */
exg_status exg_debug_trace_stream(exg_ctx* ctx, const double* b, unsigned long long* times, long long* counts);
exg_status exg_profile_get(exg_ctx* ctx, exg_kernel_times* out); /* synchronises; resets */

exg_status exg_counters_get(exg_ctx* ctx, exg_counters* out);
exg_status exg_counters_reset(exg_ctx* ctx);
exg_status exg_synchronize(exg_ctx* ctx);
/* device scratch pointers (for benchmarks that keep inputs resident) */
exg_status exg_device_alloc(exg_ctx* ctx, size_t bytes, void** ptr);
exg_status exg_device_free(exg_ctx* ctx, void* ptr);
exg_status exg_memcpy(exg_ctx* ctx, void* dst, const void* src, size_t bytes, int kind);
/* stream handle (cudaStream_t) so callers can record events on it */
void* exg_stream(exg_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* EXG_H */
