// Host-side MNA assembly and source evaluation.
//
// Mirrors the reference's front end so that the matrices handed to the device
// are bit-identical to what exsim::build_mna produces for the same element
// list (checked by tests/test_host_parity.py against oracle/_ref):
//   from_triplets      <- sparse_matrix.cpp:11-44
//   Source::eval       <- source.cpp:35-71
//   breakpoints_in     <- source.cpp:73-103
//   build_mna          <- mna.cpp:22-165
//   source_breakpoints <- mna.cpp:173-180
#include <algorithm>
#include <cmath>
#include <limits>

#include "host.hpp"

namespace exg {

Csr from_triplets(int n_rows, int n_cols, std::vector<Triplet> entries) {
    if (n_rows < 0 || n_cols < 0) throw Error{EXG_E_CONTRACT, "negative matrix dimension"};
    for (const Triplet& t : entries)
        if (t.row < 0 || t.row >= n_rows || t.col < 0 || t.col >= n_cols)
            throw Error{EXG_E_CONTRACT, "triplet coordinate out of range"};
    // std::sort with the reference's comparator: equal keys end up in the
    // same (implementation-defined but deterministic) order, so duplicate
    // sums round identically.
    std::sort(entries.begin(), entries.end(), [](const Triplet& a, const Triplet& b) {
        return a.row != b.row ? a.row < b.row : a.col < b.col;
    });
    Csr m;
    m.n_rows = n_rows;
    m.n_cols = n_cols;
    m.rowptr.assign(static_cast<size_t>(n_rows) + 1, 0);
    m.col.reserve(entries.size());
    m.val.reserve(entries.size());
    size_t i = 0;
    for (int r = 0; r < n_rows; ++r) {
        while (i < entries.size() && entries[i].row == r) {
            const int c = entries[i].col;
            double v = 0.0;
            while (i < entries.size() && entries[i].row == r && entries[i].col == c) {
                v += entries[i].value;
                ++i;
            }
            if (v != 0.0) {
                m.col.push_back(c);
                m.val.push_back(v);
            }
        }
        m.rowptr[static_cast<size_t>(r) + 1] = static_cast<int>(m.val.size());
    }
    return m;
}

namespace {

double pulse_eval(const Source& p, double t) {
    double tl = t - p.delay;
    if (tl < 0.0) return p.v1;
    if (p.period > 0.0) tl = std::fmod(tl, p.period);
    if (p.rise > 0.0 && tl < p.rise) return p.v1 + (p.v2 - p.v1) * (tl / p.rise);
    if (tl < p.rise) return p.v2;
    tl -= p.rise;
    if (tl < p.width) return p.v2;
    tl -= p.width;
    if (p.fall > 0.0 && tl < p.fall) return p.v2 + (p.v1 - p.v2) * (tl / p.fall);
    return p.v1;
}

}  // namespace

double Source::eval(double t) const {
    switch (kind) {
        case EXG_SRC_DC:
            return dc;
        case EXG_SRC_PWL: {
            if (pwl.empty()) return 0.0;
            if (t <= pwl.front().first) return pwl.front().second;
            if (t >= pwl.back().first) return pwl.back().second;
            for (size_t i = 1; i < pwl.size(); ++i) {
                if (t <= pwl[i].first) {
                    const double t0 = pwl[i - 1].first, a0 = pwl[i - 1].second;
                    const double t1 = pwl[i].first, a1 = pwl[i].second;
                    return a0 + (a1 - a0) * (t - t0) / (t1 - t0);
                }
            }
            return pwl.back().second;
        }
        case EXG_SRC_PULSE:
            return pulse_eval(*this, t);
    }
    return 0.0;
}

void Source::breakpoints_in(double t0, double t1, std::vector<double>& out) const {
    switch (kind) {
        case EXG_SRC_DC:
            return;
        case EXG_SRC_PWL:
            for (const auto& pt : pwl)
                if (pt.first > t0 && pt.first < t1) out.push_back(pt.first);
            return;
        case EXG_SRC_PULSE: {
            const double edges[4] = {0.0, rise, rise + width, rise + width + fall};
            if (period > 0.0) {
                double base = delay;
                if (t0 > base) base += std::floor((t0 - base) / period) * period;
                for (; base < t1; base += period)
                    for (double e : edges) {
                        const double t = base + e;
                        if (t > t0 && t < t1) out.push_back(t);
                    }
            } else {
                for (double e : edges) {
                    const double t = delay + e;
                    if (t > t0 && t < t1) out.push_back(t);
                }
            }
            return;
        }
    }
}

exg_options default_options() {
    exg_options o{};
    o.err_budget = 1e-4;
    o.krylov_eps = 1e-7;
    o.gmin = 1e-12;
    o.m_max = 100;
    o.has_tran = 0;
    o.hmin = std::numeric_limits<double>::quiet_NaN();
    o.hmax = std::numeric_limits<double>::quiet_NaN();
    o.tran_step = 0.0;
    o.tran_stop = 0.0;
    return o;
}

namespace {

int n_terminals(int kind) { return kind == EXG_EL_M ? 4 : 2; }

Source source_from_desc(const System& sys, const exg_source& d) {
    Source s;
    s.kind = d.kind;
    s.dc = d.dc;
    if (d.kind == EXG_SRC_PWL) {
        for (int i = 0; i < d.pwl_len; ++i)
            s.pwl.emplace_back(sys.pwl_t[d.pwl_off + i], sys.pwl_v[d.pwl_off + i]);
        for (size_t i = 1; i < s.pwl.size(); ++i)
            if (!(s.pwl[i].first > s.pwl[i - 1].first))
                throw Error{EXG_E_CONTRACT, "PWL breakpoints must be strictly increasing in time"};
    }
    s.v1 = d.v1;
    s.v2 = d.v2;
    s.delay = d.delay;
    s.rise = d.rise;
    s.fall = d.fall;
    s.width = d.width;
    s.period = d.period;
    return s;
}

}  // namespace

// mna.cpp:22-165, element for element.  Node numbering by first appearance
// over the card list (mna.cpp:28-41); stamps pushed in card order so the
// triplet sequences — and hence the duplicate sums — are identical.
void build_mna(System& sys) {
    int max_label = -1;
    for (const exg_element& e : sys.elems)
        for (int k = 0; k < n_terminals(e.kind); ++k) max_label = std::max(max_label, e.nodes[k]);
    sys.unknown_of_label.assign(static_cast<size_t>(max_label + 1), -1);

    bool ground_seen = false;
    int n_nodes = 0;
    for (const exg_element& e : sys.elems) {
        for (int k = 0; k < n_terminals(e.kind); ++k) {
            const int lab = e.nodes[k];
            if (lab == -1) {
                ground_seen = true;
                continue;
            }
            if (lab < 0) throw Error{EXG_E_CONTRACT, "bad node label"};
            if (sys.unknown_of_label[lab] < 0) sys.unknown_of_label[lab] = n_nodes++;
        }
    }
    if (!sys.elems.empty() && !ground_seen)
        throw Error{EXG_E_CONTRACT, "netlist has no ground node \"0\""};

    int n_branches = 0;
    for (const exg_element& e : sys.elems)
        if (e.kind == EXG_EL_V || e.kind == EXG_EL_L) ++n_branches;
    sys.n_nodes = n_nodes;
    sys.n = n_nodes + n_branches;

    auto idx = [&](int lab) { return lab == -1 ? -1 : sys.unknown_of_label[lab]; };
    std::vector<Triplet> g, c, b;
    auto stamp_pair = [](std::vector<Triplet>& t, int a, int bb, double v) {
        if (a >= 0) t.push_back({a, a, v});
        if (bb >= 0) t.push_back({bb, bb, v});
        if (a >= 0 && bb >= 0) {
            t.push_back({a, bb, -v});
            t.push_back({bb, a, -v});
        }
    };

    sys.sources.clear();
    sys.mos.clear();
    int branch = n_nodes;
    for (const exg_element& e : sys.elems) {
        switch (e.kind) {
            case EXG_EL_R:
                stamp_pair(g, idx(e.nodes[0]), idx(e.nodes[1]), 1.0 / e.value);
                break;
            case EXG_EL_C:
                stamp_pair(c, idx(e.nodes[0]), idx(e.nodes[1]), e.value);
                break;
            case EXG_EL_L: {
                const int a = idx(e.nodes[0]), bb = idx(e.nodes[1]);
                const int j = branch++;
                if (a >= 0) {
                    g.push_back({a, j, 1.0});
                    g.push_back({j, a, 1.0});
                }
                if (bb >= 0) {
                    g.push_back({bb, j, -1.0});
                    g.push_back({j, bb, -1.0});
                }
                c.push_back({j, j, -e.value});
                break;
            }
            case EXG_EL_V: {
                const int a = idx(e.nodes[0]), bb = idx(e.nodes[1]);
                const int j = branch++;
                if (a >= 0) {
                    g.push_back({a, j, 1.0});
                    g.push_back({j, a, 1.0});
                }
                if (bb >= 0) {
                    g.push_back({bb, j, -1.0});
                    g.push_back({j, bb, -1.0});
                }
                const int col = static_cast<int>(sys.sources.size());
                b.push_back({j, col, 1.0});
                sys.sources.push_back(source_from_desc(sys, sys.src_desc.at(e.aux)));
                break;
            }
            case EXG_EL_I: {
                const int a = idx(e.nodes[0]), bb = idx(e.nodes[1]);
                const int col = static_cast<int>(sys.sources.size());
                if (a >= 0) b.push_back({a, col, -1.0});
                if (bb >= 0) b.push_back({bb, col, 1.0});
                sys.sources.push_back(source_from_desc(sys, sys.src_desc.at(e.aux)));
                break;
            }
            case EXG_EL_M: {
                const exg_mos_model& md = sys.models.at(e.aux);
                Mosfet m;
                for (int k = 0; k < 4; ++k) m.nodes[k] = idx(e.nodes[k]);
                m.vth = md.vth;
                m.kp = md.kp;
                m.lambda = md.lambda;
                m.w = md.w;
                m.l = md.l;
                m.cgs0 = md.cgs0;
                m.cgd0 = md.cgd0;
                m.pmos = md.pmos != 0;
                if (m.kp <= 0.0 || m.w <= 0.0 || m.l <= 0.0)
                    throw Error{EXG_E_CONTRACT, "mosfet: KP, W, L must be positive"};
                sys.mos.push_back(m);
                break;
            }
            default:
                throw Error{EXG_E_CONTRACT, "unknown element kind"};
        }
    }
    if (sys.opts.gmin > 0.0)
        for (int i = 0; i < n_nodes; ++i) g.push_back({i, i, sys.opts.gmin});

    sys.G = from_triplets(sys.n, sys.n, std::move(g));
    sys.C = from_triplets(sys.n, sys.n, std::move(c));
    sys.B = from_triplets(sys.n, static_cast<int>(sys.sources.size()), std::move(b));
}

std::vector<double> eval_sources(const System& sys, double t) {
    std::vector<double> u(sys.sources.size());
    for (size_t i = 0; i < sys.sources.size(); ++i) u[i] = sys.sources[i].eval(t);
    return u;
}

std::vector<double> source_breakpoints(const System& sys, double t0, double t1) {
    if (!(t0 < t1)) throw Error{EXG_E_CONTRACT, "source_breakpoints: need t0 < t1"};
    std::vector<double> pts;
    for (const Source& s : sys.sources) s.breakpoints_in(t0, t1, pts);
    std::sort(pts.begin(), pts.end());
    pts.erase(std::unique(pts.begin(), pts.end()), pts.end());
    return pts;
}

double norm2(const std::vector<double>& a) {
    double s = 0.0;
    for (double x : a) s += x * x;
    return std::sqrt(s);
}

double norm_inf(const std::vector<double>& a) {
    double m = 0.0;
    for (double x : a) m = std::max(m, std::abs(x));
    return m;
}

}  // namespace exg
