// Synthetic workloads: the five circuits BASELINE.json names.
//
// The reference's own generator (proj/core/src/generator.cpp) produces none of
// them, so the constructions are defined here, once, with fixed seeds.  Random
// numbers follow the reference's recipe: std::mt19937_64 and
// uniform01 = (rng() >> 11) * 2^-53 (generator.cpp:13-15), log-uniform as
// generator.cpp:17-20.  Grid node (i, j) has label i*W + j and is first
// touched in row-major order, so unknown order is row-major (mna.cpp:28-41).
#include <algorithm>
#include <cmath>
#include <random>
#include <unordered_set>

#include "host.hpp"

namespace exg {

namespace {

struct Rng {
    std::mt19937_64 g;
    explicit Rng(uint64_t seed) : g(seed) {}
    double u01() { return static_cast<double>(g() >> 11) * 0x1.0p-53; }
    double uni(double a, double b) { return a + (b - a) * u01(); }
    uint64_t below(uint64_t m) { return g() % m; }
    double log_uniform(double lo, double hi) {
        return std::exp(std::log(lo) + u01() * (std::log(hi) - std::log(lo)));
    }
};

struct Builder {
    System& sys;
    void two(int kind, int a, int b, double v, int aux = -1) {
        exg_element e{};
        e.kind = kind;
        e.nodes[0] = a;
        e.nodes[1] = b;
        e.nodes[2] = -2;
        e.nodes[3] = -2;
        e.aux = aux;
        e.value = v;
        sys.elems.push_back(e);
    }
    int source(const exg_source& s) {
        sys.src_desc.push_back(s);
        return static_cast<int>(sys.src_desc.size()) - 1;
    }
    static exg_source dc(double v) {
        exg_source s{};
        s.kind = EXG_SRC_DC;
        s.dc = v;
        return s;
    }
    static exg_source pulse(double v1, double v2, double delay, double rise, double fall,
                            double width, double period) {
        exg_source s{};
        s.kind = EXG_SRC_PULSE;
        s.v1 = v1;
        s.v2 = v2;
        s.delay = delay;
        s.rise = rise;
        s.fall = fall;
        s.width = width;
        s.period = period;
        return s;
    }
    int pwl(const std::vector<std::pair<double, double>>& pts) {
        exg_source s{};
        s.kind = EXG_SRC_PWL;
        s.pwl_off = static_cast<int>(sys.pwl_t.size());
        s.pwl_len = static_cast<int>(pts.size());
        for (const auto& p : pts) {
            sys.pwl_t.push_back(p.first);
            sys.pwl_v.push_back(p.second);
        }
        return source(s);
    }
};

// RC grid body shared by configs 0, 1 and 4: ground caps (row-major, fixing
// the unknown order), right/down resistors, K coupling caps per node to
// distinct partners at Manhattan distance 1..D.
void rc_grid(Builder& b, Rng& rng, int W, int H, int K, int D) {
    for (int i = 0; i < H; ++i)
        for (int j = 0; j < W; ++j) b.two(EXG_EL_C, i * W + j, -1, rng.uni(1e-15, 10e-15));
    for (int i = 0; i < H; ++i)
        for (int j = 0; j < W; ++j) {
            const int lab = i * W + j;
            if (j + 1 < W) b.two(EXG_EL_R, lab, lab + 1, rng.uni(0.5, 2.0));
            if (i + 1 < H) b.two(EXG_EL_R, lab, lab + W, rng.uni(0.5, 2.0));
        }
    std::vector<int> chosen;
    for (int i = 0; i < H; ++i)
        for (int j = 0; j < W; ++j) {
            chosen.clear();
            for (int k = 0; k < K; ++k) {
                for (int attempt = 0; attempt < 1000; ++attempt) {
                    const int di = static_cast<int>(rng.below(2 * D + 1)) - D;
                    const int dj = static_cast<int>(rng.below(2 * D + 1)) - D;
                    if (di == 0 && dj == 0) continue;
                    if (std::abs(di) + std::abs(dj) > D) continue;
                    const int ii = i + di, jj = j + dj;
                    if (ii < 0 || ii >= H || jj < 0 || jj >= W) continue;
                    const int partner = ii * W + jj;
                    if (std::find(chosen.begin(), chosen.end(), partner) != chosen.end()) continue;
                    chosen.push_back(partner);
                    b.two(EXG_EL_C, i * W + j, partner, rng.uni(0.1e-15, 1e-15));
                    break;
                }
            }
        }
}

std::vector<int> distinct_nodes(Rng& rng, int count, int n) {
    count = std::min(count, n);
    std::vector<int> out;
    std::unordered_set<int> seen;
    while (static_cast<int>(out.size()) < count) {
        const int v = static_cast<int>(rng.below(static_cast<uint64_t>(n)));
        if (seen.insert(v).second) out.push_back(v);
    }
    return out;
}

// lattice positions of supply pads along one axis: 25 + 50k (config 1's
// 50-node pitch), or the centre for cuts narrower than one pitch
std::vector<int> pad_axis(int len) {
    std::vector<int> p;
    for (int x = 25; x < len; x += 50) p.push_back(x);
    if (p.empty()) p.push_back(len / 2);
    return p;
}

void config0(System& sys, const exg_gen_params& p) {
    const int W = p.width > 0 ? p.width : 32;
    const int H = p.height > 0 ? p.height : W;
    Rng rng(p.seed ? p.seed : 1000);
    Builder b{sys};
    rc_grid(b, rng, W, H, 3, 4);
    b.two(EXG_EL_R, 0, -1, 0.1);
    for (int node : distinct_nodes(rng, 16, W * H)) {
        const int s = b.source(Builder::pulse(0.0, 1e-3, 0.0, 10e-12, 10e-12, 100e-12, 300e-12));
        b.two(EXG_EL_I, -1, node, 0.0, s);  // "I 0 N": current into N
    }
    sys.opts.m_max = 30;
    sys.opts.err_budget = 1e-10;
    sys.opts.krylov_eps = 1e-7;
    sys.opts.has_tran = 1;
    sys.opts.tran_step = 1e-12;
    sys.opts.tran_stop = 1e-9;
}

void config1(System& sys, const exg_gen_params& p) {
    const int W = p.width > 0 ? p.width : 1000;
    const int H = p.height > 0 ? p.height : W;
    Rng rng(p.seed ? p.seed : 1001);
    Builder b{sys};
    rc_grid(b, rng, W, H, 6, 8);
    int next_label = W * H;
    const int vdd = b.source(Builder::dc(1.0));
    for (int pi : pad_axis(H))
        for (int pj : pad_axis(W)) {
            const int pad = next_label++;
            b.two(EXG_EL_V, pad, -1, 0.0, vdd);
            b.two(EXG_EL_R, pad, pi * W + pj, 0.05);
        }
    const int n_sinks =
        std::max(1, static_cast<int>(std::lround(2000.0 * (double(W) * H) / 1e6)));
    for (int node : distinct_nodes(rng, n_sinks, W * H)) {
        const double amp = rng.uni(0.0, 5e-3);
        const double delay = 25e-12 * static_cast<double>(rng.below(12));
        const int s = b.source(Builder::pulse(0.0, amp, delay, 10e-12, 10e-12, 100e-12, 300e-12));
        b.two(EXG_EL_I, node, -1, 0.0, s);  // "I N 0": sink
    }
    sys.opts.m_max = 40;
    sys.opts.hmin = 1e-12;
    sys.opts.hmax = 20e-12;
    sys.opts.has_tran = 1;
    sys.opts.tran_step = 1e-12;
    sys.opts.tran_stop = 2e-9;
}

void config2(System& sys, const exg_gen_params& p) {
    const int W = p.width > 0 ? p.width : 500;
    const int H = p.height > 0 ? p.height : W;
    Rng rng(p.seed ? p.seed : 1002);
    Builder b{sys};
    for (int i = 0; i < H; ++i)
        for (int j = 0; j < W; ++j) b.two(EXG_EL_C, i * W + j, -1, rng.uni(1e-15, 10e-15));
    int next_label = W * H;
    for (int i = 0; i < H; ++i)
        for (int j = 0; j < W; ++j) {
            const int lab = i * W + j;
            if (j + 1 < W) {
                const int mid = next_label++;
                b.two(EXG_EL_R, lab, mid, rng.uni(0.5, 2.0));
                b.two(EXG_EL_L, mid, lab + 1, rng.uni(0.1e-12, 1e-12));
            }
            if (i + 1 < H) {
                const int mid = next_label++;
                b.two(EXG_EL_R, lab, mid, rng.uni(0.5, 2.0));
                b.two(EXG_EL_L, mid, lab + W, rng.uni(0.1e-12, 1e-12));
            }
        }
    // coupling caps as config 0
    std::vector<int> chosen;
    const int K = 3, D = 4;
    for (int i = 0; i < H; ++i)
        for (int j = 0; j < W; ++j) {
            chosen.clear();
            for (int k = 0; k < K; ++k)
                for (int attempt = 0; attempt < 1000; ++attempt) {
                    const int di = static_cast<int>(rng.below(2 * D + 1)) - D;
                    const int dj = static_cast<int>(rng.below(2 * D + 1)) - D;
                    if ((di == 0 && dj == 0) || std::abs(di) + std::abs(dj) > D) continue;
                    const int ii = i + di, jj = j + dj;
                    if (ii < 0 || ii >= H || jj < 0 || jj >= W) continue;
                    const int partner = ii * W + jj;
                    if (std::find(chosen.begin(), chosen.end(), partner) != chosen.end()) continue;
                    chosen.push_back(partner);
                    b.two(EXG_EL_C, i * W + j, partner, rng.uni(0.1e-15, 1e-15));
                    break;
                }
        }
    // 64 package bumps on an 8x8 lattice: V 1 -> L 10p -> R 5m -> grid
    const int vdd = b.source(Builder::dc(1.0));
    const int nb_i = std::min(8, H), nb_j = std::min(8, W);
    for (int a = 0; a < nb_i; ++a)
        for (int c = 0; c < nb_j; ++c) {
            const int gi = static_cast<int>((a + 0.5) * H / nb_i);
            const int gj = static_cast<int>((c + 0.5) * W / nb_j);
            const int vb = next_label++, mb = next_label++;
            b.two(EXG_EL_V, vb, -1, 0.0, vdd);
            b.two(EXG_EL_L, vb, mb, 10e-12);
            b.two(EXG_EL_R, mb, gi * W + gj, 5e-3);
        }
    const int n_loads =
        std::max(1, static_cast<int>(std::lround(500.0 * (double(W) * H) / 250000.0)));
    for (int node : distinct_nodes(rng, n_loads, W * H)) {
        const double amp = rng.uni(0.0, 5e-3);
        const double delay = 25e-12 * static_cast<double>(rng.below(12));
        const int s = b.source(Builder::pulse(0.0, amp, delay, 10e-12, 10e-12, 100e-12, 300e-12));
        b.two(EXG_EL_I, node, -1, 0.0, s);
    }
    sys.opts.m_max = 100;
    sys.opts.hmin = 1e-12;
    sys.opts.hmax = 20e-12;
    sys.opts.has_tran = 1;
    sys.opts.tran_step = 1e-12;
    sys.opts.tran_stop = 1e-9;
}

// Config 3: matrix-defined post-extraction-like system (no netlist).
void config3(System& sys, const exg_gen_params& p) {
    const int n = p.n > 0 ? p.n : 11417;
    Rng rng(p.seed ? p.seed : 1003);
    std::vector<Triplet> g, c, bt;
    std::vector<double> gdiag(n, 0.0), cdiag(n, 0.0);
    std::vector<int> partners;
    for (int i = 0; i < n; ++i) {
        partners.clear();
        if (i + 1 < n) partners.push_back(i + 1);
        for (int k = 0; k < 3; ++k) {
            const int j = i + 2 + static_cast<int>(rng.below(19));  // i+2 .. i+20
            if (j >= n) continue;
            if (std::find(partners.begin(), partners.end(), j) != partners.end()) continue;
            partners.push_back(j);
        }
        for (int j : partners) {
            const double v = rng.log_uniform(1e-3, 1.0);
            g.push_back({i, j, -v});
            g.push_back({j, i, -v});
            gdiag[i] += v;
            gdiag[j] += v;
        }
    }
    for (int i = 0; i < n; ++i) g.push_back({i, i, gdiag[i] + rng.log_uniform(1e-3, 1.0)});
    for (int i = 0; i < n; ++i) {
        partners.clear();
        for (int k = 0; k < 30; ++k) {
            const int j = i + 1 + static_cast<int>(rng.below(2000));
            if (j >= n) continue;
            if (std::find(partners.begin(), partners.end(), j) != partners.end()) continue;
            partners.push_back(j);
        }
        for (int j : partners) {
            const double v = rng.uni(0.01e-15, 0.5e-15);
            c.push_back({i, j, -v});
            c.push_back({j, i, -v});
            cdiag[i] += v;
            cdiag[j] += v;
        }
    }
    for (int i = 0; i < n; ++i) c.push_back({i, i, rng.uni(1e-15, 10e-15) + cdiag[i]});
    Builder b{sys};
    const int n_in = 32;
    for (int k = 0; k < n_in; ++k) {
        for (int r : distinct_nodes(rng, 4, n)) bt.push_back({r, k, 1.0});
        std::vector<std::pair<double, double>> pts;
        const int step_ps = 50 + static_cast<int>(rng.below(150));
        for (int tp = 0; tp <= 5000; tp += step_ps)
            pts.emplace_back(static_cast<double>(tp) * 1e-12, rng.uni(0.0, 1e-3));
        b.pwl(pts);
    }
    sys.n = n;
    sys.n_nodes = n;
    sys.G = from_triplets(n, n, std::move(g));
    sys.C = from_triplets(n, n, std::move(c));
    sys.B = from_triplets(n, n_in, std::move(bt));
    sys.sources.clear();
    for (const exg_source& d : sys.src_desc) {
        Source s;
        s.kind = d.kind;
        for (int i = 0; i < d.pwl_len; ++i)
            s.pwl.emplace_back(sys.pwl_t[d.pwl_off + i], sys.pwl_v[d.pwl_off + i]);
        sys.sources.push_back(s);
    }
    sys.unknown_of_label.resize(n);
    for (int i = 0; i < n; ++i) sys.unknown_of_label[i] = i;
    sys.opts.has_tran = 1;
    sys.opts.tran_step = 1e-12;
    sys.opts.tran_stop = 5e-9;
}

// Config 4: nonlinear inverter chains on an RC grid (see DESIGN.md for the
// DC-point decision).  Square-law devices VTH=0.3, KP=1e-4, W=L=1u,
// LAMBDA=0.05, CGS0=0.5f; PMOS source on a grid node, NMOS source at ground.
void config4(System& sys, const exg_gen_params& p) {
    const int W = p.width > 0 ? p.width : 200;
    const int H = p.height > 0 ? p.height : W;
    const int chains = p.chains > 0 ? p.chains : 256;
    const int stages = p.stages > 0 ? p.stages : 16;
    Rng rng(p.seed ? p.seed : 1004);
    Builder b{sys};
    rc_grid(b, rng, W, H, 3, 4);
    int next_label = W * H;
    const int vdd = b.source(Builder::dc(1.0));
    for (int pi : pad_axis(H))
        for (int pj : pad_axis(W)) {
            const int pad = next_label++;
            b.two(EXG_EL_V, pad, -1, 0.0, vdd);
            b.two(EXG_EL_R, pad, pi * W + pj, 0.05);
        }
    exg_mos_model nm{0.3, 1e-4, 0.05, 1e-6, 1e-6, 0.5e-15, 0.0, 0, 0};
    exg_mos_model pm = nm;
    pm.pmos = 1;
    sys.models = {nm, pm};
    for (int ch = 0; ch < chains; ++ch) {
        const int in = next_label++;
        const int s = b.pwl({{0.0, 0.0}, {20e-12, 1.0}});
        b.two(EXG_EL_V, in, -1, 0.0, s);
        int prev = in;
        const int supply = static_cast<int>(rng.below(static_cast<uint64_t>(W * H)));
        for (int st = 0; st < stages; ++st) {
            const int out = next_label++;
            exg_element mp{};
            mp.kind = EXG_EL_M;
            mp.nodes[0] = out;
            mp.nodes[1] = prev;
            mp.nodes[2] = supply;
            mp.nodes[3] = supply;
            mp.aux = 1;
            sys.elems.push_back(mp);
            exg_element mn{};
            mn.kind = EXG_EL_M;
            mn.nodes[0] = out;
            mn.nodes[1] = prev;
            mn.nodes[2] = -1;
            mn.nodes[3] = -1;
            mn.aux = 0;
            sys.elems.push_back(mn);
            // wire load of the output (the reference's inverter_chain has CL,
            // generator.cpp:98); without it the last output is an algebraic
            // node whose nonlinear error w - e^{hJ}w does not shrink with h
            b.two(EXG_EL_C, out, -1, 1e-15);
            prev = out;
        }
    }
    sys.opts.has_tran = 1;
    sys.opts.tran_step = 1e-12;
    sys.opts.tran_stop = 1e-9;
    sys.opts.hmin = 1e-15;
}

}  // namespace

void generate(const exg_gen_params& p, System& sys) {
    sys = System{};
    sys.opts = default_options();
    switch (p.config) {
        case 0: config0(sys, p); break;
        case 1: config1(sys, p); break;
        case 2: config2(sys, p); break;
        case 3: config3(sys, p); return;  // matrix-defined: assembled above
        case 4: config4(sys, p); break;
        default: throw Error{EXG_E_CONTRACT, "unknown config"};
    }
    build_mna(sys);
}

}  // namespace exg
