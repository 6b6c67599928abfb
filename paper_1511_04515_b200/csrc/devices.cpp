// Host mirror of the reference's MOSFET models, linearization and DC point
// (proj/core/src/devices.cpp, proj/core/src/integrate.cpp:39-115), used by
// the nonlinear transient (config 4).  Arithmetic, stamp order and triplet
// assembly follow the reference exactly, so G_k / C_k are bit-identical and
// the host lu_factor of G_k reproduces the reference's factors.
#include <algorithm>
#include <cmath>

#include "host.hpp"

namespace exg {

// devices.cpp:31-66 (level-1 square law, drain/source swap)
void mosfet_current(const Mosfet& p, double vgs, double vds, double& id, double& gm, double& gds) {
    bool swapped = false;
    if (vds < 0.0) {
        vgs = vgs - vds;
        vds = -vds;
        swapped = true;
    }
    const double k = p.kp * p.w / p.l;
    const double vov = vgs - p.vth;
    if (vov <= 0.0) {
        id = 0.0;
        gm = 0.0;
        gds = 0.0;
    } else if (vds >= vov) {
        const double clm = 1.0 + p.lambda * vds;
        id = 0.5 * k * vov * vov * clm;
        gm = k * vov * clm;
        gds = 0.5 * k * vov * vov * p.lambda;
    } else {
        const double clm = 1.0 + p.lambda * vds;
        const double q = vov * vds - 0.5 * vds * vds;
        id = k * q * clm;
        gm = k * vds * clm;
        gds = k * (vov - vds) * clm + k * q * p.lambda;
    }
    if (swapped) {
        const double gm_s = gm;
        const double gds_s = gds;
        id = -id;
        gm = -gm_s;
        gds = gm_s + gds_s;
    }
}

namespace {

double node_voltage(const std::vector<double>& x, int idx) { return idx < 0 ? 0.0 : x[idx]; }

// sparse_matrix.cpp:84-97
Csr combine(double alpha, const Csr& A, double beta, const Csr& B) {
    std::vector<Triplet> t;
    t.reserve(static_cast<size_t>(A.nnz() + B.nnz()));
    for (int r = 0; r < A.n_rows; ++r) {
        for (int k = A.rowptr[r]; k < A.rowptr[r + 1]; ++k) t.push_back({r, A.col[k], alpha * A.val[k]});
        for (int k = B.rowptr[r]; k < B.rowptr[r + 1]; ++k) t.push_back({r, B.col[k], beta * B.val[k]});
    }
    return from_triplets(A.n_rows, A.n_cols, std::move(t));
}

}  // namespace

// devices.cpp:122-200 (MOSFETs; diodes are out of scope)
void evaluate(const System& sys, const std::vector<double>& x, Linearization& lin) {
    if (static_cast<int>(x.size()) != sys.n) throw Error{EXG_E_CONTRACT, "evaluate: state length does not match system"};
    for (double v : x)
        if (!std::isfinite(v)) throw Error{EXG_E_NONFINITE, "evaluate: non-finite state entry"};
    lin.op.assign(sys.mos.size(), DeviceOp{});
    std::vector<Triplet> g_extra, c_extra;
    for (size_t i = 0; i < sys.mos.size(); ++i) {
        const Mosfet& dev = sys.mos[i];
        const int d = dev.nodes[0], g = dev.nodes[1], s = dev.nodes[2];
        const double vgs = node_voltage(x, g) - node_voltage(x, s);
        const double vds = node_voltage(x, d) - node_voltage(x, s);
        const double sign = dev.pmos ? -1.0 : 1.0;
        double id = 0.0, gm = 0.0, gds = 0.0;
        mosfet_current(dev, sign * vgs, sign * vds, id, gm, gds);
        id *= sign;
        DeviceOp& op = lin.op[i];
        op.vgs_ref = vgs;
        op.vds_ref = vds;
        op.id_ref = id;
        op.gm = gm;
        op.gds = gds;
        auto stamp = [&](int row, int col, double v) {
            if (row >= 0 && col >= 0 && v != 0.0) g_extra.push_back({row, col, v});
        };
        stamp(d, g, gm);
        stamp(d, s, -gm - gds);
        stamp(d, d, gds);
        stamp(s, g, -gm);
        stamp(s, s, gm + gds);
        stamp(s, d, -gds);
        auto cap = [&](int a, int b, double cv) {
            if (cv <= 0.0) return;
            if (a >= 0) c_extra.push_back({a, a, cv});
            if (b >= 0) c_extra.push_back({b, b, cv});
            if (a >= 0 && b >= 0) {
                c_extra.push_back({a, b, -cv});
                c_extra.push_back({b, a, -cv});
            }
        };
        cap(g, s, dev.cgs0);
        cap(g, d, dev.cgd0);
    }
    if (g_extra.empty() && c_extra.empty()) {
        lin.G = sys.G;
        lin.C = sys.C;
    } else {
        const Csr g_nl = from_triplets(sys.n, sys.n, std::move(g_extra));
        const Csr c_nl = from_triplets(sys.n, sys.n, std::move(c_extra));
        lin.G = combine(1.0, sys.G, 1.0, g_nl);
        lin.C = combine(1.0, sys.C, 1.0, c_nl);
    }
}

// devices.cpp:202-233
std::vector<double> residual_F(const System& sys, const Linearization& lin, const std::vector<double>& x) {
    std::vector<double> F(x.size(), 0.0);
    for (size_t i = 0; i < sys.mos.size(); ++i) {
        const Mosfet& dev = sys.mos[i];
        const DeviceOp& op = lin.op[i];
        const int d = dev.nodes[0], g = dev.nodes[1], s = dev.nodes[2];
        const double vgs = node_voltage(x, g) - node_voltage(x, s);
        const double vds = node_voltage(x, d) - node_voltage(x, s);
        const double sign = dev.pmos ? -1.0 : 1.0;
        double id = 0.0, gm = 0.0, gds = 0.0;
        mosfet_current(dev, sign * vgs, sign * vds, id, gm, gds);
        id *= sign;
        const double r = op.gm * vgs + op.gds * vds - id;
        if (d >= 0) F[d] += r;
        if (s >= 0) F[s] -= r;
    }
    return F;
}

// x = Factorization::solve(b) on the host (sparse_lu.cpp:255-291)
std::vector<double> lu_solve_host(const Factor& f, const std::vector<double>& b) {
    const int n = f.n;
    std::vector<double> z(n);
    for (int k = 0; k < n; ++k) z[k] = b[f.row_perm[k]];
    for (int r = 0; r < n; ++r) {
        double s = z[r];
        for (int k = f.L.rowptr[r]; k < f.L.rowptr[r + 1]; ++k) {
            const int c = f.L.col[k];
            if (c < r) s -= f.L.val[k] * z[c];
        }
        z[r] = s;
    }
    for (int r = n - 1; r >= 0; --r) {
        double s = z[r], diag = 0.0;
        for (int k = f.U.rowptr[r]; k < f.U.rowptr[r + 1]; ++k) {
            const int c = f.U.col[k];
            if (c == r)
                diag = f.U.val[k];
            else if (c > r)
                s -= f.U.val[k] * z[c];
        }
        z[r] = s / diag;
    }
    std::vector<double> out(n);
    for (int k = 0; k < n; ++k) out[f.col_perm[k]] = z[k];
    return out;
}

namespace {

// integrate.cpp:41-55 (MOSFET part)
std::vector<double> equivalent_current(const System& sys, const Linearization& lin) {
    std::vector<double> ieq(sys.n, 0.0);
    for (size_t i = 0; i < sys.mos.size(); ++i) {
        const DeviceOp& op = lin.op[i];
        const int d = sys.mos[i].nodes[0], s = sys.mos[i].nodes[2];
        const double c = op.id_ref - op.gm * op.vgs_ref - op.gds * op.vds_ref;
        if (d >= 0) ieq[d] += c;
        if (s >= 0) ieq[s] -= c;
    }
    return ieq;
}

// integrate.cpp:57-64
Csr with_node_gmin(const Csr& G, const System& sys, double gmin_extra) {
    if (gmin_extra <= 0.0) return G;
    std::vector<Triplet> t;
    for (int i = 0; i < sys.n_nodes; ++i) t.push_back({i, i, gmin_extra});
    return combine(1.0, G, 1.0, from_triplets(sys.n, sys.n, std::move(t)));
}

std::vector<double> spmv_host(const Csr& A, const std::vector<double>& x) {
    std::vector<double> y(A.n_rows, 0.0);
    for (int r = 0; r < A.n_rows; ++r) {
        double s = 0.0;
        for (int k = A.rowptr[r]; k < A.rowptr[r + 1]; ++k) s += A.val[k] * x[A.col[k]];
        y[r] = s;
    }
    return y;
}

// integrate.cpp:68-88
bool newton_static(const System& sys, std::vector<double>& x, const std::vector<double>& bu0,
                   double gmin_extra) {
    const int nr_max_iters = 50;
    if (sys.mos.empty()) {
        Linearization lin;
        evaluate(sys, x, lin);
        Factor f;
        lu_factor(with_node_gmin(lin.G, sys, gmin_extra), 0.1, f);
        x = lu_solve_host(f, bu0);
        return true;
    }
    for (int iter = 1; iter <= nr_max_iters; ++iter) {
        Linearization lin;
        evaluate(sys, x, lin);  // no limiting for MOSFETs
        const std::vector<double> ieq = equivalent_current(sys, lin);
        std::vector<double> rhs(bu0);
        for (int i = 0; i < sys.n; ++i) rhs[i] += -1.0 * ieq[i];
        Factor f;
        lu_factor(with_node_gmin(lin.G, sys, gmin_extra), 0.1, f);
        std::vector<double> x_new = lu_solve_host(f, rhs);
        std::vector<double> diff(x_new);
        for (int i = 0; i < sys.n; ++i) diff[i] += -1.0 * x[i];
        const double dx = norm_inf(diff);
        x = std::move(x_new);
        if (dx <= 1e-9 * (1.0 + norm_inf(x))) return true;
    }
    return false;
}

}  // namespace

// integrate.cpp:92-115
std::vector<double> dc_solve(const System& sys) {
    const std::vector<double> u0 = eval_sources(sys, 0.0);
    const std::vector<double> bu0 = spmv_host(sys.B, u0);
    std::vector<double> x(sys.n, 0.0);
    try {
        std::vector<double> attempt = x;
        if (newton_static(sys, attempt, bu0, 0.0)) return attempt;
    } catch (const Error& e) {
        if (e.status != EXG_E_SINGULAR) throw;
    }
    std::vector<double> x_stage(sys.n, 0.0);
    for (double g = 1e-3; g >= 0.99e-12; g *= 0.1)
        if (!newton_static(sys, x_stage, bu0, g))
            throw Error{EXG_E_NO_DC, "dc_solve: gmin stepping stalled at gmin=" + std::to_string(g)};
    if (!newton_static(sys, x_stage, bu0, 0.0))
        throw Error{EXG_E_NO_DC, "dc_solve: no convergence after gmin stepping"};
    return x_stage;
}

}  // namespace exg
