// Internal host-side types of the exsim-B200 framework (not part of the C ABI).
//
// These are the host mirrors of the reference's data types:
//   Csr      <- exsim::SparseRealMatrix  proj/core/include/exsim/sparse_matrix.hpp:22-53
//   Source   <- exsim::SourceWaveform    proj/core/include/exsim/source.hpp:8-37
//   System   <- exsim::MnaSystem         proj/core/include/exsim/mna.hpp:44-58
//   Factor   <- exsim::Factorization     proj/core/include/exsim/sparse_lu.hpp:16-42
// Arithmetic that feeds the hot path (triplet summation, source values, LU)
// is written to produce bit-identical results to the reference when compiled
// with the same g++ and flags (-O3, no -ffast-math, no FMA contraction).
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "exg_host.h"

namespace exg {

struct Triplet {  // same layout and sort order as exsim::Triplet
    int row = 0;
    int col = 0;
    double value = 0.0;
};

struct Csr {
    int n_rows = 0;
    int n_cols = 0;
    std::vector<int> rowptr{0};
    std::vector<int> col;
    std::vector<double> val;
    int nnz() const { return static_cast<int>(val.size()); }
};

// sparse_matrix.cpp:11-44 — sort by (row, col), sum duplicates in sorted
// order, prune exact zeros.
Csr from_triplets(int n_rows, int n_cols, std::vector<Triplet> entries);

struct Source {
    int kind = EXG_SRC_DC;
    double dc = 0.0;
    std::vector<std::pair<double, double>> pwl;
    double v1 = 0, v2 = 0, delay = 0, rise = 0, fall = 0, width = 0, period = 0;
    double eval(double t) const;                                          // source.cpp:50-71
    void breakpoints_in(double t0, double t1, std::vector<double>& out) const;  // :73-103
};

struct Mosfet {
    int nodes[4] = {-1, -1, -1, -1};  // d g s b (unknown indices, -1 ground)
    double vth = 0.7, kp = 2e-5, lambda = 0.0, w = 10e-6, l = 1e-6, cgs0 = 0.0, cgd0 = 0.0;
    bool pmos = false;
};

struct System {
    int n = 0;
    int n_nodes = 0;
    Csr G, C, B;
    std::vector<Source> sources;
    std::vector<Mosfet> mos;
    exg_options opts{};
    std::vector<int> unknown_of_label;  // label -> unknown index (-1 if absent)
    // element list (kept for cross-checks against the reference's build_mna)
    std::vector<exg_element> elems;
    std::vector<exg_source> src_desc;
    std::vector<double> pwl_t, pwl_v;
    std::vector<exg_mos_model> models;
    int n_inputs() const { return static_cast<int>(sources.size()); }
};

exg_options default_options();
void build_mna(System& sys);  // fills n, G, C, B, sources, mos from elems
std::vector<double> eval_sources(const System& sys, double t);
std::vector<double> source_breakpoints(const System& sys, double t0, double t1);
void generate(const exg_gen_params& p, System& sys);

struct Factor {
    int n = 0;
    Csr L, U;
    std::vector<int> row_perm, col_perm;
    double order_s = 0.0, numeric_s = 0.0;
};

// Bit-identical restatement of exsim::lu_factor (sparse_lu.cpp:134-253).
// Throws exg::Error(EXG_E_SINGULAR) like SingularMatrixError.
void lu_factor(const Csr& A, double pivot_tol, Factor& f);
std::vector<int> min_degree_order(const Csr& A);

// nonlinear devices (devices.hpp:14-36): per-MOSFET operating point frozen
// at the linearization state, and the step-frozen linearization
struct DeviceOp {
    double vgs_ref = 0.0, vds_ref = 0.0, id_ref = 0.0, gm = 0.0, gds = 0.0;
};
struct Linearization {
    Csr G, C;
    std::vector<DeviceOp> op;
};
void mosfet_current(const Mosfet& p, double vgs, double vds, double& id, double& gm, double& gds);
void evaluate(const System& sys, const std::vector<double>& x, Linearization& lin);
std::vector<double> residual_F(const System& sys, const Linearization& lin, const std::vector<double>& x);
std::vector<double> lu_solve_host(const Factor& f, const std::vector<double>& b);
std::vector<double> dc_solve(const System& sys);

// host-side vector helpers with the reference's exact semantics (vec.hpp)
double norm2(const std::vector<double>& a);
double norm_inf(const std::vector<double>& a);

struct Error {
    exg_status status;
    std::string what;
    double value = 0.0;
};

}  // namespace exg

// opaque handles of include/exg_host.h
struct exg_system {
    exg::System sys;
};
struct exg_factor {
    exg::Factor f;
};
