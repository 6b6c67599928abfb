// Integration check: the reference-side adapter of INTEGRATION.md §1, compiled
// against the UNMODIFIED reference headers and library (oracle/_ref) and the
// product library (libexg.so) through include/exg.h only.
//
// main() builds one of the reference's own generated circuits (generator.hpp),
// factors G with the reference's lu_factor, uploads C/G/B and the factors
// through the adapter, and walks a few ER steps: each step is computed by the
// reference's er_step (integrate.cpp:302-316) and by Backend::er_step from the
// same state; the results must agree (EXACT mode: <= 1e-12 of the vector's
// scale, same Krylov dimensions; FAST mode: <= 1e-9).  Exit code 0 = pass.
//
// Built by oracle/Makefile (target `adapter`) into oracle/_ref/gpu_backend_demo
// when /root/reference is present; run by tests/test_gpu_integration.py.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "exg.h"
#include "exsim/errors.hpp"
#include "exsim/generator.hpp"
#include "exsim/integrate.hpp"
#include "exsim/krylov.hpp"
#include "exsim/mna.hpp"
#include "exsim/sparse_lu.hpp"

// ---- the adapter a maintainer adds as proj/core/src/gpu_backend.cpp --------
namespace exsim::gpu {

[[noreturn]] void rethrow(exg_ctx* c, exg_status st, double value = 0.0) {
    char msg[512];
    exg_last_error(c, msg, sizeof msg);
    switch (st) {
        case EXG_E_CONTRACT: throw ContractError(msg);
        case EXG_E_NONFINITE: throw NonFiniteError(msg);
        case EXG_E_SINGULAR: throw SingularMatrixError(msg, static_cast<int>(value));
        case EXG_E_ZERO_START: throw ZeroStartVectorError(msg);
        case EXG_E_NO_CONVERGENCE: throw NoConvergenceError(msg, value);
        case EXG_E_SINGULAR_REDUCED: throw SingularReducedMatrixError(msg);
        default: throw Error(msg);
    }
}
#define EXG_CHECK(c, call)             \
    do {                               \
        exg_status s_ = (call);        \
        if (s_) ::exsim::gpu::rethrow(c, s_); \
    } while (0)

struct Backend {
    exg_ctx* ctx = nullptr;
    explicit Backend(int device = 0) {
        if (exg_create(device, &ctx) != EXG_OK) throw Error("exg_create failed");
    }
    ~Backend() { exg_destroy(ctx); }
    Backend(const Backend&) = delete;
    Backend& operator=(const Backend&) = delete;

    void upload(const SparseRealMatrix& C, const SparseRealMatrix& G, const SparseRealMatrix& B,
                const Factorization& f) {
        auto put = [&](int which, const SparseRealMatrix& m) {
            EXG_CHECK(ctx, exg_set_csr(ctx, which, m.n_rows(), m.n_cols(), m.nnz(), m.row_offsets().data(),
                                       m.col_indices().data(), m.values().data()));
        };
        put(EXG_MAT_C, C);
        put(EXG_MAT_G, G);
        put(EXG_MAT_B, B);
        const auto& L = f.lower();
        const auto& U = f.upper();
        EXG_CHECK(ctx, exg_set_factors(ctx, f.dimension(), L.row_offsets().data(), L.col_indices().data(),
                                       L.values().data(), U.row_offsets().data(), U.col_indices().data(),
                                       U.values().data(), f.row_perm().data(), f.col_perm().data()));
    }
    // er_step (integrate.cpp:302-316) on the device
    Vec er_step(const Vec& x_k, const Vec& u_k, const Vec& u_k1, double h, const MevpConfig& cfg,
                std::vector<int>& dims) {
        exg_mevp_cfg c{cfg.eps, cfg.m_max, cfg.check_stride, cfg.breakdown_tol};
        Vec x_next(x_k.size());
        int m = -1;
        exg_status st = exg_er_step(ctx, x_k.data(), u_k.data(), u_k1.data(), h, &c, x_next.data(), &m,
                                    EXG_PTR_HOST);
        if (st) rethrow(ctx, st);
        if (m >= 0) dims.push_back(m);
        return x_next;
    }
};

}  // namespace exsim::gpu

// ---- the check --------------------------------------------------------------
int main(int argc, char** argv) {
    using namespace exsim;
    const int stages = argc > 1 ? std::atoi(argv[1]) : 300;
    const int steps = argc > 2 ? std::atoi(argv[2]) : 6;
    const bool fast = argc > 3 && std::strcmp(argv[3], "fast") == 0;
    try {
        GeneratorParams gp;
        gp.kind = GeneratorKind::CoupledMesh;
        gp.stages = stages;
        gp.coupling_density = 0.02;
        gp.seed = 11;
        const MnaSystem sys = build_mna(generate_circuit(gp));
        const Vec x0 = dc_solve(sys);
        const Linearization lin = evaluate(sys, x0);
        const Factorization fact = lu_factor(lin.G_k);
        StepControl ctl;
        ctl.eps = sys.options.krylov_eps > 0.0 ? sys.options.krylov_eps : 1e-7;
        ctl.m_max = 60;
        // steps inside the first source segment
        const double t_stop = sys.tran ? sys.tran->stop_time : 1e-9;
        const std::vector<double> bps = source_breakpoints(sys, 0.0, t_stop);
        const double seg = bps.empty() ? t_stop : bps.front();
        const double h = seg / steps;

        gpu::Backend be(0);
        if (fast) {
            exg_options_dev o{EXG_TRSV_FAST, EXG_WEIGHT_GSPMV, EXG_LOOP_GRAPH};
            EXG_CHECK(be.ctx, exg_set_options(be.ctx, &o));
        }
        be.upload(lin.C_k, lin.G_k, sys.B, fact);
        MevpConfig cfg;
        cfg.eps = ctl.eps;
        cfg.m_max = ctl.m_max;

        SimState st;
        st.x = x0;
        st.t = 0.0;
        st.h = h;
        double worst = 0.0;
        const double tol = fast ? 1e-9 : 1e-12;
        for (int k = 0; k < steps; ++k) {
            const ErStepResult ref = er_step(sys, lin, fact, st, ctl);
            std::vector<int> dims;
            const Vec got = be.er_step(st.x, eval_sources(sys, st.t), eval_sources(sys, st.t + h), h, cfg, dims);
            double scale = 0.0, err = 0.0;
            for (std::size_t i = 0; i < got.size(); ++i) {
                scale = std::max(scale, std::fabs(ref.x_next[i]));
                err = std::max(err, std::fabs(got[i] - ref.x_next[i]));
            }
            const double rel = err / std::max(scale, 1e-300);
            worst = std::max(worst, rel);
            const bool same_dims = dims == ref.rec.krylov_dims;
            std::printf("step %d t=%.3e: rel err %.3e, krylov dims %s (ref %zu, gpu %zu)\n", k, st.t + h, rel,
                        same_dims ? "equal" : "DIFFERENT", ref.rec.krylov_dims.size(), dims.size());
            if (!(rel <= tol) || !same_dims) {
                std::printf("FAIL\n");
                return 1;
            }
            st.x = ref.x_next;
            st.t += h;
        }
        // the error mapping: a zero step size is the reference's ContractError
        bool threw = false;
        try {
            std::vector<int> dims;
            be.er_step(st.x, eval_sources(sys, st.t), eval_sources(sys, st.t), -1.0, cfg, dims);
        } catch (const ContractError&) {
            threw = true;
        }
        if (!threw) {
            std::printf("FAIL: negative step did not raise ContractError\n");
            return 1;
        }
        std::printf("PASS n=%d steps=%d mode=%s worst rel err %.3e\n", sys.n, steps, fast ? "fast" : "exact", worst);
        return 0;
    } catch (const std::exception& e) {
        std::printf("FAIL: exception %s\n", e.what());
        return 2;
    }
}
