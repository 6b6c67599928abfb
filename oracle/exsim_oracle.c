/*
 * ORACLE / TEST INFRASTRUCTURE — not the product.
 *
 * A plain-C restatement of the reference's hot path (proj/core), used by the
 * tests as an independent checker of the CUDA kernels and pinned, bit for
 * bit, against the reference library itself (oracle/_ref, tests/test_oracle.py)
 * and against the reference tests' known-answer values (tests/golden/).
 * Compiled with -ffp-contract=off so every a*b+c rounds twice, like the
 * reference's x86-64 build.  Each function cites what it restates.
 */
#include "exsim_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* sparse_matrix.cpp:69-82 — row-sequential accumulation */
void orc_spmv(const orc_csr* A, const double* x, double* y) {
    for (int r = 0; r < A->n_rows; ++r) {
        double s = 0.0;
        for (int k = A->rowptr[r]; k < A->rowptr[r + 1]; ++k) s += A->val[k] * x[A->col[k]];
        y[r] = s;
    }
}

/* sparse_lu.cpp:255-291 — gather, unit-L forward, U backward, scatter */
void orc_solve(const orc_factor* f, const double* b, double* x, double* work) {
    const int n = f->n;
    double* z = work;
    for (int k = 0; k < n; ++k) z[k] = b[f->row_perm[k]];
    const orc_csr* lo = &f->L;
    for (int r = 0; r < n; ++r) {
        double s = z[r];
        for (int k = lo->rowptr[r]; k < lo->rowptr[r + 1]; ++k) {
            const int c = lo->col[k];
            if (c < r) s -= lo->val[k] * z[c];
        }
        z[r] = s;
    }
    const orc_csr* up = &f->U;
    for (int r = n - 1; r >= 0; --r) {
        double s = z[r], diag = 0.0;
        for (int k = up->rowptr[r]; k < up->rowptr[r + 1]; ++k) {
            const int c = up->col[k];
            if (c == r)
                diag = up->val[k];
            else if (c > r)
                s -= up->val[k] * z[c];
        }
        z[r] = s / diag;
    }
    for (int k = 0; k < n; ++k) x[f->col_perm[k]] = z[k];
}

/* sparse_lu.cpp:293-304 — w = x[col_perm]; z = U w; y = L z; scatter */
void orc_apply(const orc_factor* f, const double* x, double* y, double* work) {
    const int n = f->n;
    double* w = work;
    double* z = work + n;
    double* t = work + 2 * n;
    for (int j = 0; j < n; ++j) w[j] = x[f->col_perm[j]];
    orc_spmv(&f->U, w, z);
    orc_spmv(&f->L, z, t);
    for (int k = 0; k < n; ++k) y[f->row_perm[k]] = t[k];
}

/* ---- dense kit (dense_matrix.cpp) ------------------------------------- */
#define AT(m, n, i, j) (m)[(size_t)(i) * (n) + (j)]

/* :33-45 i-k-j with zero skip */
static void mmul(int n, const double* a, const double* b, double* c) {
    memset(c, 0, sizeof(double) * n * n);
    for (int i = 0; i < n; ++i)
        for (int k = 0; k < n; ++k) {
            const double aik = AT(a, n, i, k);
            if (aik == 0.0) continue;
            for (int j = 0; j < n; ++j) AT(c, n, i, j) += aik * AT(b, n, k, j);
        }
}

/* :60-67  c = a + beta*b */
static void add_scaled(int n, const double* a, double beta, const double* b, double* c) {
    for (int i = 0; i < n * n; ++i) c[i] = a[i] + beta * b[i];
}

static double norm1(int n, const double* a) { /* :17-25 */
    double best = 0.0;
    for (int c = 0; c < n; ++c) {
        double s = 0.0;
        for (int r = 0; r < n; ++r) s += fabs(AT(a, n, r, c));
        if (s > best) best = s;
    }
    return best;
}

/* :69-118  solve A X = B in place of x (B on entry).  Returns ORC_E_SINGULAR
 * when a pivot column is exactly zero. */
int orc_dense_solve(int n, const double* a, double* x, double* work) {
    double* lu = work;
    memcpy(lu, a, sizeof(double) * n * n);
    for (int k = 0; k < n; ++k) {
        int p = k;
        double best = fabs(AT(lu, n, k, k));
        for (int r = k + 1; r < n; ++r) {
            const double m = fabs(AT(lu, n, r, k));
            if (m > best) {
                best = m;
                p = r;
            }
        }
        if (best == 0.0) return ORC_E_SINGULAR;
        if (p != k) {
            for (int j = 0; j < n; ++j) {
                double t = AT(lu, n, k, j);
                AT(lu, n, k, j) = AT(lu, n, p, j);
                AT(lu, n, p, j) = t;
            }
            for (int j = 0; j < n; ++j) {
                double t = AT(x, n, k, j);
                AT(x, n, k, j) = AT(x, n, p, j);
                AT(x, n, p, j) = t;
            }
        }
        const double d = AT(lu, n, k, k);
        for (int r = k + 1; r < n; ++r) {
            const double fct = AT(lu, n, r, k) / d;
            AT(lu, n, r, k) = fct;
            if (fct == 0.0) continue;
            for (int j = k + 1; j < n; ++j) AT(lu, n, r, j) -= fct * AT(lu, n, k, j);
            for (int j = 0; j < n; ++j) AT(x, n, r, j) -= fct * AT(x, n, k, j);
        }
    }
    for (int k = n - 1; k >= 0; --k) {
        const double d = AT(lu, n, k, k);
        for (int j = 0; j < n; ++j) {
            double s = AT(x, n, k, j);
            for (int c = k + 1; c < n; ++c) s -= AT(lu, n, k, c) * AT(x, n, c, j);
            AT(x, n, k, j) = s / d;
        }
    }
    return ORC_OK;
}

/* :120-124 */
int orc_dense_inverse(int n, const double* a, double* inv, double* cond, double* work) {
    memset(inv, 0, sizeof(double) * n * n);
    for (int i = 0; i < n; ++i) AT(inv, n, i, i) = 1.0;
    const int st = orc_dense_solve(n, a, inv, work);
    if (st) return st;
    if (cond) *cond = norm1(n, a) * norm1(n, inv);
    return ORC_OK;
}

/* :137-181 diagonal Pade approximant */
static int pade(int n, const double* a, const double* b, int degree, double* out, double* w) {
    const size_t nn = (size_t)n * n;
    double* ident = w;
    double* a2 = w + nn;
    double* u = w + 2 * nn;
    double* v = w + 3 * nn;
    double* t1 = w + 4 * nn;
    double* t2 = w + 5 * nn;
    double* t3 = w + 6 * nn;
    double* t4 = w + 7 * nn;
    double* sw = w + 8 * nn; /* dense_solve scratch */
    memset(ident, 0, sizeof(double) * nn);
    for (int i = 0; i < n; ++i) AT(ident, n, i, i) = 1.0;
    mmul(n, a, a, a2);
    if (degree <= 9) {
        double* usum = t1;
        double* vsum = t2;
        double* pw = t3;
        memset(usum, 0, sizeof(double) * nn);
        memset(vsum, 0, sizeof(double) * nn);
        memcpy(pw, ident, sizeof(double) * nn);
        for (int k = 0; k <= degree; k += 2) {
            add_scaled(n, vsum, b[k], pw, t4);
            memcpy(vsum, t4, sizeof(double) * nn);
            add_scaled(n, usum, b[k + 1], pw, t4);
            memcpy(usum, t4, sizeof(double) * nn);
            if (k + 2 <= degree) {
                mmul(n, pw, a2, t4);
                memcpy(pw, t4, sizeof(double) * nn);
            }
        }
        mmul(n, a, usum, u);
        memcpy(v, vsum, sizeof(double) * nn);
    } else {
        double* a4 = t1;
        double* a6 = t2;
        mmul(n, a2, a2, a4);
        mmul(n, a4, a2, a6);
        double* s1 = t3;
        double* s2 = t4;
        double* s3 = sw;
        double* s4 = sw + nn;
        double* s5 = sw + 2 * nn;
        /* u1 = a6*(b13 a6 + b11 a4 + b9 a2) */
        for (size_t i = 0; i < nn; ++i) s1[i] = b[13] * a6[i];
        for (size_t i = 0; i < nn; ++i) s2[i] = b[11] * a4[i];
        add_scaled(n, s1, 1.0, s2, s3);
        for (size_t i = 0; i < nn; ++i) s1[i] = b[9] * a2[i];
        add_scaled(n, s3, 1.0, s1, s4);
        mmul(n, a6, s4, s5); /* u1 */
        /* u2 = b7 a6 + b5 a4 + b3 a2 + b1 I */
        for (size_t i = 0; i < nn; ++i) s1[i] = b[7] * a6[i];
        for (size_t i = 0; i < nn; ++i) s2[i] = b[5] * a4[i];
        add_scaled(n, s1, 1.0, s2, s3);
        for (size_t i = 0; i < nn; ++i) s1[i] = b[3] * a2[i];
        add_scaled(n, s3, 1.0, s1, s4);
        add_scaled(n, s4, b[1], ident, s2); /* u2 in s2 */
        add_scaled(n, s5, 1.0, s2, s3);     /* u1 + u2 */
        mmul(n, a, s3, u);
        /* v1 = a6*(b12 a6 + b10 a4 + b8 a2) */
        for (size_t i = 0; i < nn; ++i) s1[i] = b[12] * a6[i];
        for (size_t i = 0; i < nn; ++i) s2[i] = b[10] * a4[i];
        add_scaled(n, s1, 1.0, s2, s3);
        for (size_t i = 0; i < nn; ++i) s1[i] = b[8] * a2[i];
        add_scaled(n, s3, 1.0, s1, s4);
        mmul(n, a6, s4, s5); /* v1 */
        for (size_t i = 0; i < nn; ++i) s1[i] = b[6] * a6[i];
        for (size_t i = 0; i < nn; ++i) s2[i] = b[4] * a4[i];
        add_scaled(n, s1, 1.0, s2, s3);
        for (size_t i = 0; i < nn; ++i) s1[i] = b[2] * a2[i];
        add_scaled(n, s3, 1.0, s1, s4);
        add_scaled(n, s4, b[0], ident, s2); /* v2 */
        add_scaled(n, s5, 1.0, s2, v);
    }
    double* num = t1;
    double* den = t2;
    add_scaled(n, v, 1.0, u, num);
    add_scaled(n, v, -1.0, u, den);
    memcpy(out, num, sizeof(double) * nn);
    return orc_dense_solve(n, den, out, sw + 3 * nn);
}

/* :185-225 */
int orc_dense_expm(int n, const double* m, double* out, double* work) {
    static const double b3[] = {120, 60, 12, 1};
    static const double b5[] = {30240, 15120, 3360, 420, 30, 1};
    static const double b7[] = {17297280, 8648640, 1995840, 277200, 25200, 1512, 56, 1};
    static const double b9[] = {17643225600., 8821612800., 2075673600., 302702400., 30270240.,
                                2162160.,     110880.,     3960.,       90.,        1.};
    static const double b13[] = {64764752532480000., 32382376266240000., 7771770303897600.,
                                 1187353796428800.,  129060195264000.,   10559470521600.,
                                 670442572800.,      33522128640.,       1323241920.,
                                 40840800.,          960960.,            16380.,
                                 182.,               1.};
    const double theta3 = 1.495585217958292e-2, theta5 = 2.539398330063230e-1,
                 theta7 = 9.504178996162932e-1, theta9 = 2.097847961257068e0,
                 theta13 = 5.371920351148152e0;
    const size_t nn = (size_t)n * n;
    int own = 0;
    if (!work) {
        work = (double*)malloc(sizeof(double) * (16 * nn + 16));
        own = 1;
    }
    for (size_t i = 0; i < nn; ++i)
        if (!isfinite(m[i])) {
            if (own) free(work);
            return ORC_E_NONFINITE;
        }
    const double nrm = norm1(n, m);
    int st;
    if (nrm <= theta3)
        st = pade(n, m, b3, 3, out, work);
    else if (nrm <= theta5)
        st = pade(n, m, b5, 5, out, work);
    else if (nrm <= theta7)
        st = pade(n, m, b7, 7, out, work);
    else if (nrm <= theta9)
        st = pade(n, m, b9, 9, out, work);
    else {
        int s = 0;
        double sn = nrm;
        while (sn > theta13) {
            sn *= 0.5;
            ++s;
        }
        double* a = work + 12 * nn;
        const double fct = ldexp(1.0, -s);
        for (size_t i = 0; i < nn; ++i) a[i] = m[i] * fct;
        st = pade(n, a, b13, 13, out, work);
        double* t = work + 13 * nn;
        for (int k = 0; k < s && st == ORC_OK; ++k) {
            mmul(n, out, out, t);
            memcpy(out, t, sizeof(double) * nn);
        }
    }
    if (own) free(work);
    return st;
}

/* ---- Krylov (krylov.cpp) ------------------------------------------------- */
static double dot(int n, const double* a, const double* b) { /* vec.hpp:13-17 */
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}
static double nrm2(int n, const double* a) { return sqrt(dot(n, a, a)); }
static void axpy(int n, double alpha, const double* x, double* y) {
    for (int i = 0; i < n; ++i) y[i] += alpha * x[i];
}

#define HB(b, j) ((b)->hbar + (size_t)(j) * ((b)->m_max + 2))

/* krylov.cpp:85-101: inverse with left shifts {0, 1e-12, 1e-9}*||H||_1 */
static int invert_reduced(int m, const double* hm, double* hinv, double* w) {
    double scale = norm1(m, hm);
    if (scale < 1e-300) scale = 1e-300;
    const double deltas[3] = {0.0, 1e-12 * scale, 1e-9 * scale};
    double* sh = w;
    double* sw = w + (size_t)m * m;
    for (int t = 0; t < 3; ++t) {
        memcpy(sh, hm, sizeof(double) * m * m);
        for (int i = 0; i < m; ++i) AT(sh, m, i, i) -= deltas[t];
        double cond = 0.0;
        if (orc_dense_inverse(m, sh, hinv, &cond, sw) == ORC_OK && cond < 1e12) return 1;
    }
    return 0;
}

/* reduced_exp at h (krylov.cpp:24-30) */
static int reduced_exp(const orc_basis* b, double h, double* e, double* w) {
    const int m = b->m;
    double* sc = w;
    for (int i = 0; i < m * m; ++i) sc[i] = h * b->h_inv[i];
    return orc_dense_expm(m, sc, e, w + (size_t)m * m);
}

/* arnoldi_mevp invert=true (krylov.cpp:103-173) with MGS orthogonalize
 * (:46-78) */
int orc_mevp_iks(const orc_factor* f, const orc_csr* C, const double* v, const orc_cfg* cfg,
                 double h, double* out, orc_basis* b) {
    const int n = C->n_rows;
    const double beta = nrm2(n, v);
    if (beta == 0.0) return ORC_E_ZERO_START;
    if (cfg->m_max < 1) return ORC_E_CONTRACT;
    if (h < 0.0) return ORC_E_CONTRACT;
    const int M = cfg->m_max;
    b->n = n;
    b->m_max = M;
    b->beta = beta;
    b->happy = 0;
    b->m = 0;
    double* V = b->V;
    const double ib = 1.0 / beta;
    for (int i = 0; i < n; ++i) V[i] = v[i] * ib;
    double* tmp = (double*)malloc(sizeof(double) * (4 * (size_t)n + 64));
    double* w = tmp + n;
    const size_t mm = (size_t)M * M;
    double* dw = (double*)malloc(sizeof(double) * (24 * mm + 64));
    double* hm = dw;
    double* hinv = dw + mm;
    double* ered = dw + 2 * mm;
    double* scratch = dw + 3 * mm;
    double last_residual = INFINITY;
    int converged = 0, st = ORC_OK;
    for (int j = 1; j <= M && !converged; ++j) {
        const double* vj = V + (size_t)(j - 1) * n;
        orc_spmv(C, vj, tmp);
        orc_solve(f, tmp, w, tmp + 2 * n);
        for (int i = 0; i < n; ++i) w[i] *= -1.0;
        /* orthogonalize */
        const int jc = j - 1;
        const double pre = nrm2(n, w);
        double* hcol = HB(b, jc);
        for (int i = 0; i < jc + 2; ++i) hcol[i] = 0.0;
        for (int i = 0; i <= jc; ++i) {
            const double hij = dot(n, w, V + (size_t)i * n);
            axpy(n, -hij, V + (size_t)i * n, w);
            hcol[i] = hij;
        }
        double post = nrm2(n, w);
        if (post < 0.70710678118654752 * pre) {
            for (int i = 0; i <= jc; ++i) {
                const double s = dot(n, w, V + (size_t)i * n);
                axpy(n, -s, V + (size_t)i * n, w);
                hcol[i] += s;
            }
            post = nrm2(n, w);
        }
        hcol[jc + 1] = post;
        const int happy = post <= cfg->breakdown_tol * pre;
        if (!happy) {
            const double ip = 1.0 / post;
            double* vn = V + (size_t)j * n;
            for (int i = 0; i < n; ++i) vn[i] = w[i] * ip;
        }
        b->m = j;
        b->h_next = happy ? 0.0 : post;
        b->happy = happy;
        /* H_m (:15-20) */
        memset(hm, 0, sizeof(double) * j * j);
        for (int c = 0; c < j; ++c)
            for (int r = 0; r <= c + 1 && r < j; ++r) AT(hm, j, r, c) = HB(b, c)[r];
        const int invertible = invert_reduced(j, hm, hinv, scratch);
        if (happy) {
            if (!invertible) {
                st = ORC_E_SINGULAR_REDUCED;
                break;
            }
            memcpy(b->h_inv, hinv, sizeof(double) * j * j);
            last_residual = 0.0;
            converged = 1;
            break;
        }
        const int check = (j % cfg->check_stride == 0) || j == M;
        if (!check) continue;
        if (!invertible) continue;
        memcpy(b->h_inv, hinv, sizeof(double) * j * j);
        st = reduced_exp(b, h, ered, scratch);
        if (st) break;
        double s = 0.0;
        for (int i = 0; i < j; ++i) s += AT(b->h_inv, j, j - 1, i) * AT(ered, j, i, 0);
        orc_apply(f, V + (size_t)j * n, tmp, tmp + n);
        const double weight = nrm2(n, tmp);
        last_residual = fabs(beta * post * s) * weight;
        if (last_residual < cfg->eps) converged = 1;
    }
    b->last_residual = last_residual;
    if (st == ORC_OK && !converged) st = ORC_E_NO_CONVERGENCE;
    free(dw);
    free(tmp);
    if (st) return st;
    b->h_sub = h;
    return orc_basis_eval(b, h, out);
}

/* mevp_residual (krylov.cpp:191-205) — weight from spmv(G, v_{m+1}) */
double orc_basis_residual(const orc_basis* b, const orc_csr* G, double h, double* work) {
    if (b->happy || b->h_next == 0.0) return 0.0;
    const int m = b->m;
    double* e = (double*)malloc(sizeof(double) * (20 * (size_t)m * m + 16));
    reduced_exp(b, h, e, e + (size_t)m * m);
    double s = 0.0;
    for (int i = 0; i < m; ++i) s += AT(b->h_inv, m, m - 1, i) * AT(e, m, i, 0);
    free(e);
    orc_spmv(G, b->V + (size_t)m * b->n, work);
    return fabs(b->beta * b->h_next * s) * nrm2(b->n, work);
}

/* eval_at_scaled_h + basis_combination (krylov.cpp:207-215, :32-36) */
int orc_basis_eval(const orc_basis* b, double h, double* out) {
    if (h < 0.0 || h > b->h_sub) return ORC_E_CONTRACT;
    const int m = b->m, n = b->n;
    double* e = (double*)malloc(sizeof(double) * (20 * (size_t)m * m + 16));
    const int st = reduced_exp(b, h, e, e + (size_t)m * m);
    if (st == ORC_OK) {
        for (int i = 0; i < n; ++i) out[i] = 0.0;
        for (int j = 0; j < m; ++j) axpy(n, b->beta * AT(e, m, j, 0), b->V + (size_t)j * n, out);
    }
    free(e);
    return st;
}

/* er_begin + er_eval for a linear circuit (integrate.cpp:213-265): F == 0 */
int orc_er_step(const orc_factor* f, const orc_csr* C, const orc_csr* B, const double* x_k,
                const double* u_k, const double* u_k1, double h, const orc_cfg* cfg,
                double* x_next, int* m_out, orc_basis* b) {
    const int n = C->n_rows, ni = B->n_cols;
    double* buf = (double*)malloc(sizeof(double) * (8 * (size_t)n + ni + 8));
    double* slope = buf;
    double* rhs = buf + ni;
    double* v1 = rhs + n;
    double* gb = v1 + n;
    double* t = gb + n;
    double* start = t + n;
    double* work = start + n;
    double* val = work + n;
    for (int i = 0; i < ni; ++i) slope[i] = u_k1[i] + -1.0 * u_k[i];
    const double ih = 1.0 / h;
    for (int i = 0; i < ni; ++i) slope[i] *= ih;
    orc_spmv(B, u_k, t);
    for (int i = 0; i < n; ++i) rhs[i] = 0.0 + 1.0 * t[i]; /* residual_F == 0 */
    orc_solve(f, rhs, v1, work);
    for (int i = 0; i < n; ++i) v1[i] = x_k[i] + -1.0 * v1[i];
    orc_spmv(B, slope, t);
    orc_solve(f, t, gb, work);
    orc_spmv(C, gb, t);
    orc_solve(f, t, start, work);
    for (int i = 0; i < n; ++i) start[i] = v1[i] + 1.0 * start[i];
    /* er_eval */
    for (int i = 0; i < n; ++i) x_next[i] = x_k[i] + 1.0 * (gb[i] * h);
    double xinf = 0.0;
    for (int i = 0; i < n; ++i) xinf = fmax(xinf, fabs(x_k[i]));
    *m_out = -1;
    int st = ORC_OK;
    if (!(nrm2(n, start) <= 1e-9 * (1.0 + xinf))) {
        st = orc_mevp_iks(f, C, start, cfg, h, val, b);
        if (st == ORC_OK) {
            *m_out = b->m;
            for (int i = 0; i < n; ++i) x_next[i] += 1.0 * val[i];
            for (int i = 0; i < n; ++i) x_next[i] += -1.0 * start[i];
        }
    }
    free(buf);
    return st;
}
