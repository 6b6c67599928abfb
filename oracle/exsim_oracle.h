/* ORACLE / TEST INFRASTRUCTURE — CPU restatement of the reference hot path.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use it.
 * See exsim_oracle.c for the file:line each function restates. */
#ifndef EXSIM_ORACLE_H
#define EXSIM_ORACLE_H

typedef struct orc_csr {
    int n_rows, n_cols;
    const int* rowptr;
    const int* col;
    const double* val;
} orc_csr;

typedef struct orc_factor {
    int n;
    orc_csr L, U; /* pivot coordinates, L unit diagonal stored, U with diagonal */
    const int* row_perm;
    const int* col_perm;
} orc_factor;

typedef struct orc_cfg {
    double eps;
    int m_max;
    int check_stride;
    double breakdown_tol;
} orc_cfg;

/* caller-provided storage: V n*(m_max+1), hbar (m_max+1)*(m_max+2),
 * h_inv m_max*m_max, work >= 4n + 16*m_max*m_max */
typedef struct orc_basis {
    int n, m, happy, m_max;
    double beta, h_next, h_sub, last_residual;
    double* V;
    double* hbar; /* column j at hbar + j*(m_max+2), entries 0..j+1 */
    double* h_inv;
    double* work;
} orc_basis;

enum { ORC_OK = 0, ORC_E_CONTRACT = 1, ORC_E_NONFINITE = 2, ORC_E_SINGULAR = 3,
       ORC_E_ZERO_START = 4, ORC_E_NO_CONVERGENCE = 5, ORC_E_SINGULAR_REDUCED = 6 };

void orc_spmv(const orc_csr* A, const double* x, double* y);
void orc_solve(const orc_factor* f, const double* b, double* x, double* work);
void orc_apply(const orc_factor* f, const double* x, double* y, double* work);
int orc_dense_solve(int n, const double* a, double* x, double* work);
int orc_dense_inverse(int n, const double* a, double* inv, double* cond, double* work);
int orc_dense_expm(int n, const double* m, double* out, double* work);
int orc_mevp_iks(const orc_factor* f, const orc_csr* C, const double* v, const orc_cfg* cfg,
                 double h, double* out, orc_basis* b);
double orc_basis_residual(const orc_basis* b, const orc_csr* G, double h, double* work);
int orc_basis_eval(const orc_basis* b, double h, double* out);
/* one linear ER step: er_begin + er_eval (integrate.cpp:213-265).  m_out =
 * Krylov dimension of the fresh basis or -1 (start-vector early-out). */
int orc_er_step(const orc_factor* f, const orc_csr* C, const orc_csr* B, const double* x_k,
                const double* u_k, const double* u_k1, double h, const orc_cfg* cfg,
                double* x_next, int* m_out, orc_basis* b);

#endif
