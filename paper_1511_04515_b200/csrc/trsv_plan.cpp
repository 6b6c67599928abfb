// Blocked augmented triangular system for the FAST solve (see trsv_plan.hpp).
#include "trsv_plan.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <numeric>
#include <queue>
#include <stdexcept>
#include <thread>

namespace exg {
namespace {

struct Block {
    int a, b;  // rows [a, b)
};

// Maximal runs of rows whose diagonal block is dense.  L: row i joins [a, i)
// when its last i-a entries are exactly a..i-1.  U (scanned upwards): row i
// joins [i+1, b) when its first b-1-i entries are exactly i+1..b-1.
std::vector<Block> dense_blocks(bool upper, int n, const int* ptr, const int* col, int min_block,
                                int max_block) {
    std::vector<Block> out;
    auto keep = [&](int a, int b) {
        if (b - a < min_block) return;
        for (int s = a; s < b; s += max_block) out.push_back({s, std::min(b, s + max_block)});
    };
    if (!upper) {
        int a = 0;
        for (int i = 1; i <= n; ++i) {
            bool ext = false;
            if (i < n) {
                const int need = i - a, len = ptr[i + 1] - ptr[i];
                ext = len >= need && col[ptr[i + 1] - need] == a;
            }
            if (!ext) {
                keep(a, i);
                a = i;
            }
        }
    } else {
        int b = n;
        for (int i = n - 2; i >= -1; --i) {
            bool ext = false;
            if (i >= 0) {
                const int need = b - 1 - i, len = ptr[i + 1] - ptr[i];
                ext = len >= need && col[ptr[i] + need - 1] == b - 1;
            }
            if (!ext) {
                keep(i + 1, b);
                b = i + 1;
            }
        }
    }
    // scan order: L ascending, U descending
    std::sort(out.begin(), out.end(), [upper](const Block& x, const Block& y) { return upper ? x.a > y.a : x.a < y.a; });
    return out;
}

// Explicit inverse of a dense block, row-major s x s.  L: unit lower (entries
// strictly below the diagonal in m); U: upper with diagonal d.
void invert_block(bool upper, int s, const std::vector<double>& m, const double* d, std::vector<double>& inv) {
    inv.assign((size_t)s * s, 0.0);
    if (!upper) {
        for (int i = 0; i < s; ++i) {
            double* ri = &inv[(size_t)i * s];
            ri[i] = 1.0;
            for (int k = 0; k < i; ++k) {
                const double f = m[(size_t)i * s + k];
                if (f == 0.0) continue;
                const double* rk = &inv[(size_t)k * s];
                for (int j = 0; j <= k; ++j) ri[j] -= f * rk[j];
            }
        }
    } else {
        std::vector<double> acc(s);
        for (int i = s - 1; i >= 0; --i) {
            std::fill(acc.begin() + i, acc.end(), 0.0);
            for (int k = i + 1; k < s; ++k) {
                const double f = m[(size_t)i * s + k];
                if (f == 0.0) continue;
                const double* rk = &inv[(size_t)k * s];
                for (int j = k; j < s; ++j) acc[j] += f * rk[j];
            }
            double* ri = &inv[(size_t)i * s];
            ri[i] = 1.0 / d[i];
            for (int j = i + 1; j < s; ++j) ri[j] = -acc[j] / d[i];
        }
    }
}

struct Row {
    int out, in;
    double dg;
    long long e0, e1;  // entries in the staging arrays
};

}  // namespace

void build_aug_plan(bool upper, int n, const int* ptr, const int* col, const double* val,
                    const double* diag, const int* in_index, const AugParams& prm, AugPlan& P) {
    P = AugPlan{};
    P.n = n;
    // levels of the plain triangle (statistics)
    {
        std::vector<int> lv(n, 0);
        int nl = 0;
        for (int q = 0; q < n; ++q) {
            const int r = upper ? n - 1 - q : q;
            int v = 0;
            for (int k = ptr[r]; k < ptr[r + 1]; ++k) v = std::max(v, lv[col[k]] + 1);
            lv[r] = v;
            nl = std::max(nl, v + 1);
        }
        P.orig_levels = n ? nl : 0;
    }
    const std::vector<Block> blocks =
        prm.min_block > 0 ? dense_blocks(upper, n, ptr, col, prm.min_block, prm.max_block) : std::vector<Block>{};
    // block inverses (independent; largest first over a few host threads)
    std::vector<std::vector<double>> invs(blocks.size());
    {
        std::vector<int> ord(blocks.size());
        std::iota(ord.begin(), ord.end(), 0);
        std::sort(ord.begin(), ord.end(), [&](int x, int y) {
            return blocks[x].b - blocks[x].a > blocks[y].b - blocks[y].a;
        });
        const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
        std::vector<std::thread> th;
        std::atomic<int> cursor{0};
        auto work = [&]() {
            std::vector<double> m;
            while (true) {
                const int q = cursor.fetch_add(1);
                if (q >= (int)ord.size()) return;
                const Block& B = blocks[ord[q]];
                const int s = B.b - B.a;
                m.assign((size_t)s * s, 0.0);
                for (int i = 0; i < s; ++i) {
                    const int r = B.a + i;
                    if (!upper) {
                        // last i entries of row r are columns a..r-1
                        for (int k = 0; k < i; ++k) m[(size_t)i * s + k] = val[ptr[r + 1] - i + k];
                    } else {
                        // first s-1-i entries of row r are columns r+1..b-1
                        for (int k = 0; k < s - 1 - i; ++k) m[(size_t)i * s + i + 1 + k] = val[ptr[r] + k];
                    }
                }
                invert_block(upper, s, m, upper ? diag + B.a : nullptr, invs[ord[q]]);
            }
        };
        for (unsigned t = 0; t < hw; ++t) th.emplace_back(work);
        for (auto& t : th) t.join();
    }
    // ---- augmented rows in a topological order, with levels and partials
    std::vector<Row> rows;
    rows.reserve((size_t)n + n / 4);
    std::vector<int> ecol;
    std::vector<double> eval;
    ecol.reserve((size_t)ptr[n] + n);
    eval.reserve((size_t)ptr[n] + n);
    std::vector<int> level;  // per unknown id
    level.assign(n, -1);
    long long next_id = n;
    auto new_id = [&]() {
        level.push_back(-1);
        return (int)next_id++;
    };
    std::vector<int> rlev;  // per row (parallel to rows)
    std::vector<std::pair<int, int>> tmp;  // (dep level, entry index) for chunking
    std::vector<int> tcol;
    std::vector<double> tval;
    // finalize one row whose entries are tcol/tval: partial sums for a long
    // history, then the row itself
    auto emit = [&](int out, int in, double dg) {
        int lmax = -1;
        // partial sums for a long history; with a cap the pass repeats (partials
        // of partials) until the row fits
        while ((int)tcol.size() > prm.chunk_over) {
            const int cnt = (int)tcol.size();
            tmp.resize(cnt);
            for (int k = 0; k < cnt; ++k) tmp[k] = {level[tcol[k]], k};
            std::stable_sort(tmp.begin(), tmp.end(),
                             [](const std::pair<int, int>& x, const std::pair<int, int>& y) { return x.first < y.first; });
            int n_old = cnt - prm.recent;
            if (prm.cap > 0) {
                // full chunks from the oldest entries; the remainder and the
                // partial references share the row: rem + chunks <= cap
                int c = cnt / prm.chunk;
                if (cnt - c * prm.chunk + c > prm.cap) ++c;
                n_old = std::min(cnt, c * prm.chunk);
            }
            std::vector<int> keep_c;
            std::vector<double> keep_v;
            for (int c0 = 0; c0 < n_old; c0 += prm.chunk) {
                const int c1 = std::min(n_old, c0 + prm.chunk);
                const int pid = new_id();
                Row pr{pid, -1, 1.0, (long long)ecol.size(), 0};
                int pl = 0;
                for (int z = c0; z < c1; ++z) pl = std::max(pl, tmp[z].first + 1);
                // within a row the order is free: by column where the rows
                // are cut for the stream kernel, so that neighbouring lanes
                // gather neighbouring values (4 per 32-byte sector)
                if (prm.cap > 0)
                    std::sort(tmp.begin() + c0, tmp.begin() + c1, [&](const std::pair<int, int>& x, const std::pair<int, int>& y) {
                        return tcol[x.second] < tcol[y.second];
                    });
                for (int z = c0; z < c1; ++z) {
                    ecol.push_back(tcol[tmp[z].second]);
                    eval.push_back(tval[tmp[z].second]);
                }
                pr.e1 = (long long)ecol.size();
                level[pid] = pl;
                rows.push_back(pr);
                rlev.push_back(pl);
                ++P.n_partials;
                keep_c.push_back(pid);
                keep_v.push_back(-1.0);
            }
            for (int z = n_old; z < cnt; ++z) {
                keep_c.push_back(tcol[tmp[z].second]);
                keep_v.push_back(tval[tmp[z].second]);
            }
            tcol.swap(keep_c);
            tval.swap(keep_v);
            if (prm.cap <= 0) break;
        }
        Row r{out, in, dg, (long long)ecol.size(), 0};
        // entries oldest first (L) / newest first (U: the kernel walks U rows
        // backwards), so a warp meets its newest dependency last
        const int m = (int)tcol.size();
        tmp.resize(m);
        for (int k = 0; k < m; ++k) {
            tmp[k] = {level[tcol[k]], k};
            lmax = std::max(lmax, tmp[k].first);
        }
        if (prm.cap > 0)
            std::sort(tmp.begin(), tmp.end(), [&](const std::pair<int, int>& x, const std::pair<int, int>& y) {
                return tcol[x.second] < tcol[y.second];
            });
        else
            std::stable_sort(tmp.begin(), tmp.end(), [&](const std::pair<int, int>& x, const std::pair<int, int>& y) {
                return upper ? x.first > y.first : x.first < y.first;
            });
        for (int k = 0; k < m; ++k) {
            ecol.push_back(tcol[tmp[k].second]);
            eval.push_back(tval[tmp[k].second]);
        }
        r.e1 = (long long)ecol.size();
        level[out] = lmax + 1;
        rows.push_back(r);
        rlev.push_back(lmax + 1);
        tcol.clear();
        tval.clear();
    };
    size_t bi = 0;  // next block in scan order
    std::vector<int> yid;
    for (int q = 0; q < n; ++q) {
        const int r = upper ? n - 1 - q : q;
        const bool at_block = bi < blocks.size() && (upper ? blocks[bi].b - 1 == r : blocks[bi].a == r);
        if (!at_block) {
            for (int k = ptr[r]; k < ptr[r + 1]; ++k) {
                tcol.push_back(col[k]);
                tval.push_back(val[k]);
            }
            emit(r, in_index[r], upper ? diag[r] : 1.0);
            continue;
        }
        const Block B = blocks[bi];
        const std::vector<double>& inv = invs[bi];
        ++bi;
        const int s = B.b - B.a;
        ++P.n_blocks;
        P.block_rows += s;
        P.max_block = std::max(P.max_block, s);
        yid.assign(s, -1);
        // y rows: the external part of every block row
        for (int z = 0; z < s; ++z) {
            const int i = upper ? s - 1 - z : z;
            const int rr = B.a + i;
            for (int k = ptr[rr]; k < ptr[rr + 1]; ++k) {
                const int c = col[k];
                if (c >= B.a && c < B.b) continue;
                tcol.push_back(c);
                tval.push_back(val[k]);
            }
            yid[i] = new_id();
            emit(yid[i], in_index[rr], 1.0);
        }
        // x rows: x_i = sum_k inv_ik y_k  (stored as out = 0 - sum (-inv) y)
        for (int z = 0; z < s; ++z) {
            const int i = upper ? s - 1 - z : z;
            const int k0 = upper ? i : 0, k1 = upper ? s : i + 1;
            for (int k = k0; k < k1; ++k) {
                const double v = inv[(size_t)i * s + k];
                if (v == 0.0) continue;
                tcol.push_back(yid[k]);
                tval.push_back(-v);
            }
            emit(B.a + i, -1, 1.0);
        }
        q += s - 1;
    }
    P.n_aug = next_id;
    // ---- positions by level (stable: creation order within a level)
    int nl = 0;
    for (int v : rlev) nl = std::max(nl, v + 1);
    P.levels = nl;
    std::vector<long long> lstart(nl + 1, 0);
    for (int v : rlev) lstart[v + 1]++;
    for (int l = 0; l < nl; ++l) lstart[l + 1] += lstart[l];
    std::vector<int> pos_row(rows.size());
    {
        std::vector<long long> fillp(lstart.begin(), lstart.end() - 1);
        for (size_t i = 0; i < rows.size(); ++i) pos_row[fillp[rlev[i]]++] = (int)i;
    }
    P.level_first_pos.assign(lstart.begin(), lstart.end());
    P.meta.resize(4 * rows.size());
    P.col.reserve(ecol.size());
    P.val.reserve(eval.size());
    P.diag.assign(P.n_aug, 1.0);
    for (size_t p = 0; p < rows.size(); ++p) {
        const Row& r = rows[pos_row[p]];
        P.meta[4 * p] = r.out;
        P.meta[4 * p + 1] = r.in;
        P.meta[4 * p + 2] = (int)P.col.size();
        for (long long k = r.e0; k < r.e1; ++k) {
            P.col.push_back(ecol[k]);
            P.val.push_back(eval[k]);
        }
        if (P.col.size() > (size_t)INT32_MAX) throw std::runtime_error("augmented plan: too many entries");
        P.meta[4 * p + 3] = (int)P.col.size();
        P.diag[r.out] = r.dg;
    }
    // ---- warp tasks (as make_tasks, FAST): long rows alone; short rows
    // grouped within one level and one length class, 1..8 lanes per row
    P.level_first_task.assign(nl + 1, 0);
    int g0 = -1, gc = 0, glev = -1, glg = -1;
    auto flush = [&]() {
        if (gc) {
            P.tasks.push_back(g0);
            P.tasks.push_back(gc | (glg << 8));
        }
        gc = 0;
    };
    int cur_level = -1;
    for (size_t p = 0; p < rows.size(); ++p) {
        const int lv = rlev[pos_row[p]];
        if (lv != cur_level) {
            flush();
            for (int l = cur_level + 1; l <= lv; ++l) P.level_first_task[l] = (int)P.tasks.size() / 2;
            cur_level = lv;
        }
        const int len = P.meta[4 * p + 3] - P.meta[4 * p + 2];
        if (len > 32) {
            flush();
            P.tasks.push_back((int)p);
            P.tasks.push_back(1 | (1 << 30));
            continue;
        }
        const int lg = len <= 4 ? 0 : len <= 8 ? 1 : len <= 16 ? 2 : 3;
        if (gc && (lg != glg || (gc + 1) << lg > 32)) flush();
        if (!gc) {
            g0 = (int)p;
            glev = lv;
            glg = lg;
        }
        ++gc;
    }
    flush();
    for (int l = cur_level + 1; l <= nl; ++l) P.level_first_task[l] = (int)P.tasks.size() / 2;
    (void)glev;
}

void eval_aug_plan(const AugPlan& P, bool upper, const double* in, double* out) {
    const size_t np = P.meta.size() / 4;
    for (size_t p = 0; p < np; ++p) {
        const int o = P.meta[4 * p], i = P.meta[4 * p + 1];
        double s = i >= 0 ? in[i] : 0.0;
        for (int k = P.meta[4 * p + 2]; k < P.meta[4 * p + 3]; ++k) s -= P.val[k] * out[P.col[k]];
        if (upper) s = s / P.diag[o];
        out[o] = s;
    }
}

// ---------------------------------------------------------------------------
// per-warp record streams (trsv_plan.hpp)
// ---------------------------------------------------------------------------
namespace {

inline int lanes_log2_for(int len) {  // smallest lg with len <= 4 * 2^lg
    int lg = 0;
    while (len > (4 << lg)) ++lg;
    return lg;
}

template <typename T>
inline void put(std::vector<unsigned char>& v, size_t at, T x) {
    std::memcpy(v.data() + at, &x, sizeof(T));
}
template <typename T>
inline T get(const unsigned char* p) {
    T x;
    std::memcpy(&x, p, sizeof(T));
    return x;
}

}  // namespace

void stream_params_env(StreamParams& p) {
    if (const char* e = getenv("EXG_STREAM_SCHED")) p.sched = atoi(e);
    if (const char* e = getenv("EXG_STREAM_HOP")) p.hop = atof(e);
    if (const char* e = getenv("EXG_STREAM_BUNDLE")) p.bundle = atoi(e);
}

void build_stream_plan(const AugPlan& P, bool upper, const int* out_index, const StreamParams& prm,
                       StreamPlan& S) {
    S = StreamPlan{};
    if (prm.n_warps < 1) throw std::runtime_error("stream plan: bad parameters");
    const int MS = upper ? kStreamMetaU : kStreamMetaL;
    S.n = P.n;
    S.levels = P.levels;
    S.n_aug = P.n_aug;
    if (P.n_aug >= INT32_MAX) throw std::runtime_error("stream plan: too many unknowns");
    const int dummy = (int)P.n_aug;
    const size_t np = P.meta.size() / 4;
    S.n_rows = (long long)np;
    // ---- row heights: the longest chain of dependent rows below each row
    // (positions are in level order, so a reverse sweep sees every consumer
    // before its producers)
    std::vector<int> pos_of((size_t)P.n_aug, -1);
    for (size_t p = 0; p < np; ++p) pos_of[P.meta[4 * p]] = (int)p;
    std::vector<int> height(np, 0);
    if (prm.sched != 0) {
        for (size_t p = np; p-- > 0;)
            for (int k = P.meta[4 * p + 2]; k < P.meta[4 * p + 3]; ++k) {
                const int pp = pos_of[P.col[k]];
                if (pp < 0 || (size_t)pp >= p) throw std::runtime_error("stream plan: rows not in dependency order");
                height[pp] = std::max(height[pp], height[p] + 1);
            }
    }
    // ---- tasks: within a level rows are independent, so they are grouped by
    // lane class, longest first; the list schedule also keeps rows of like
    // height together (a task is as urgent as its most urgent row)
    struct Task {
        long long first;  // index into `ord`
        int cnt, lg, nq, level;
        int cont;         // 1: same column list as the task before it (same warp, right behind it)
    };
    std::vector<int> ord(np);
    std::iota(ord.begin(), ord.end(), 0);
    auto len_of = [&](int p) { return P.meta[4 * (size_t)p + 3] - P.meta[4 * (size_t)p + 2]; };
    std::vector<Task> tasks;
    // rows of 65..128 entries are tasks of their own; many repeat the column
    // list of another row of their level (the rows of a block inverse over one
    // 128-column chunk, the rows of a supernode over its ancestors): up to
    // `bundle` of them run back to back on one warp, the first gathers the
    // dependencies, the others (cont) reuse its registers
    const int bundle = prm.sched != 0 ? std::max(1, prm.bundle) : 1;
    auto cmp_cols = [&](int x, int y) {
        const int lx = len_of(x), ly = len_of(y);
        if (lx != ly) return lx > ly ? -1 : 1;  // longest first
        return std::memcmp(&P.col[P.meta[4 * (size_t)x + 2]], &P.col[P.meta[4 * (size_t)y + 2]], sizeof(int) * lx);
    };
    for (int l = 0; l < P.levels; ++l) {
        const long long a = P.level_first_pos[l], b = P.level_first_pos[l + 1];
        if (prm.sched != 0)
            std::stable_sort(ord.begin() + a, ord.begin() + b, [&](int x, int y) {
                const int lx = lanes_log2_for(len_of(x)), ly = lanes_log2_for(len_of(y));
                if (lx != ly) return lx > ly;
                if (lx == 5 && bundle > 1) {  // single-row tasks: equal column lists side by side
                    const int c = cmp_cols(x, y);
                    if (c != 0) return c < 0;
                }
                if (height[x] != height[y]) return height[x] > height[y];
                return len_of(x) > len_of(y);
            });
        else
            std::stable_sort(ord.begin() + a, ord.begin() + b, [&](int x, int y) { return len_of(x) > len_of(y); });
        long long i = a;
        while (i < b) {
            const int len = len_of(ord[i]);
            if (len > 128) throw std::runtime_error("stream plan: a row exceeds 128 entries (AugParams.cap)");
            const int lg = lanes_log2_for(len);
            Task t{i, 0, lg, 0, l, 0};
            // rows per task: the lane count, and the record must fit its slot
            int longest = 0;
            while (i < b && (t.cnt << lg) < 32 && lanes_log2_for(len_of(ord[i])) == lg) {
                const int lo = std::max(longest, len_of(ord[i]));
                const int nq = (lo + (1 << lg) - 1) >> lg;
                if (t.cnt > 0 && 16 + nq * 384 + (t.cnt + 1) * MS > kStreamSlot) break;
                longest = lo;
                ++t.cnt;
                ++i;
            }
            t.nq = (longest + (1 << lg) - 1) >> lg;
            if (lg == 5 && bundle > 1 && !tasks.empty()) {
                const Task& pv = tasks.back();
                if (pv.level == l && pv.lg == 5 && cmp_cols(ord[pv.first], ord[t.first]) == 0) {
                    int run = 1;  // tasks of the bundle so far
                    for (size_t q = tasks.size(); q-- > 0 && tasks[q].cont;) ++run;
                    if (run < bundle) t.cont = 1;
                }
            }
            tasks.push_back(t);
        }
    }
    if (getenv("EXG_PLAN_VERBOSE")) {  // how many single-row tasks repeat the previous one's column list?
        long long wide = 0, same = 0, wide_entries = 0;
        std::vector<int> idx;
        for (int l = 0; l < P.levels; ++l) {
            idx.clear();
            for (long long i = P.level_first_pos[l]; i < P.level_first_pos[l + 1]; ++i)
                if (lanes_log2_for(len_of(ord[i])) == 5) idx.push_back(ord[i]);
            auto cmp = [&](int x, int y) {
                const int lx = len_of(x), ly = len_of(y);
                if (lx != ly) return lx < ly ? -1 : 1;
                return std::memcmp(&P.col[P.meta[4 * (size_t)x + 2]], &P.col[P.meta[4 * (size_t)y + 2]], sizeof(int) * lx);
            };
            std::sort(idx.begin(), idx.end(), [&](int x, int y) { return cmp(x, y) < 0; });
            wide += (long long)idx.size();
            for (size_t i = 0; i < idx.size(); ++i) {
                wide_entries += len_of(idx[i]);
                if (i && cmp(idx[i - 1], idx[i]) == 0) ++same;
            }
        }
        fprintf(stderr, "stream plan %s: single-row tasks %lld (%lld entries), %lld repeat another row's columns\n",
                upper ? "U" : "L", wide, wide_entries, same);
    }
    const size_t NT = tasks.size();
    S.n_tasks = (long long)NT;
    int W = prm.n_warps;
    if (prm.min_tasks_per_warp > 0) {
        const long long want = ((long long)NT / prm.min_tasks_per_warp + 7) / 8 * 8;
        W = (int)std::max<long long>(8, std::min<long long>(W, want));  // a multiple of 8 (and of any CTA's warps)
        W = std::min(W, prm.n_warps);
    }
    S.n_warps = W;
    // the task that produces each unknown
    std::vector<int> prod((size_t)P.n_aug, -1);
    for (size_t t = 0; t < NT; ++t)
        for (int seg = 0; seg < tasks[t].cnt; ++seg) prod[P.meta[4 * (size_t)ord[tasks[t].first + seg]]] = (int)t;
    // ---- the order of execution: rank r runs tasks[by_rank[r]] on warp
    // warp_of[r]; a warp runs its tasks by ascending rank and every dependency
    // of a task has a smaller rank, so the unfinished task of smallest rank can
    // always run (no deadlock whatever the timing).
    std::vector<int> by_rank(NT), warp_of(NT);
    std::vector<double> fin(NT, 0.0);  // modelled finish time, in task costs
    const double hop = prm.hop;
    auto model_level_order = [&]() {  // level order, round-robin: the modelled makespan
        std::vector<double> wfree(W, 0.0);
        double span = 0.0;
        for (size_t t = 0; t < NT; ++t) {
            double rdy = 0.0;
            for (int seg = 0; seg < tasks[t].cnt; ++seg) {
                const int p = ord[tasks[t].first + seg];
                for (int k = P.meta[4 * (size_t)p + 2]; k < P.meta[4 * (size_t)p + 3]; ++k)
                    rdy = std::max(rdy, fin[prod[P.col[k]]] + hop);
            }
            double& wf = wfree[t % W];
            fin[t] = wf = std::max(wf, rdy) + 1.0;
            span = std::max(span, wf);
        }
        return span;
    };
    double span_level = 0.0, span_list = 0.0;
    if (prm.sched == 0) {
        for (size_t t = 0; t < NT; ++t) {
            by_rank[t] = (int)t;
            warp_of[t] = (int)(t % W);
        }
        if (getenv("EXG_PLAN_VERBOSE")) span_level = model_level_order();
    } else {
        if (getenv("EXG_PLAN_VERBOSE")) span_level = model_level_order();
        // list schedule (highest level first): simulate W warps with unit task
        // cost and a hand-off of `hop` costs between a producer's finish and a
        // consumer's start.  A free warp takes the most urgent task (largest
        // height) whose dependencies are `hop` old, or else waits for the one
        // that becomes ready first.
        // a bundle (a task and the cont tasks behind it) is one unit of the
        // schedule: `size` costs on one warp; head[t] = its first task
        std::vector<int> head(NT), bsize(NT, 0);
        for (size_t t = 0; t < NT; ++t) {
            head[t] = tasks[t].cont ? head[t - 1] : (int)t;
            ++bsize[head[t]];
        }
        std::vector<int> theight(NT, 0), ndep(NT, 0);
        std::vector<long long> sptr(NT + 1, 0);
        std::vector<int> deps;  // scratch: a unit's distinct producer units
        auto producers = [&](size_t h) {
            deps.clear();
            for (size_t t = h; t < h + (size_t)bsize[h]; ++t)
                for (int seg = 0; seg < tasks[t].cnt; ++seg) {
                    const int p = ord[tasks[t].first + seg];
                    theight[h] = std::max(theight[h], height[p]);
                    if (t == h)  // cont tasks repeat the head's columns
                        for (int k = P.meta[4 * (size_t)p + 2]; k < P.meta[4 * (size_t)p + 3]; ++k)
                            deps.push_back(head[prod[P.col[k]]]);
                }
            std::sort(deps.begin(), deps.end());
            deps.erase(std::unique(deps.begin(), deps.end()), deps.end());
        };
        size_t n_units = 0;
        for (size_t t = 0; t < NT; ++t) {
            if (head[t] != (int)t) continue;
            ++n_units;
            producers(t);
            ndep[t] = (int)deps.size();
            for (int d : deps) ++sptr[d + 1];
        }
        for (size_t t = 0; t < NT; ++t) sptr[t + 1] += sptr[t];
        std::vector<int> succ((size_t)sptr[NT]);
        {
            std::vector<long long> at(sptr.begin(), sptr.end() - 1);
            for (size_t t = 0; t < NT; ++t) {
                if (head[t] != (int)t) continue;
                producers(t);
                for (int d : deps) succ[(size_t)at[d]++] = (int)t;
            }
        }
        using TE = std::pair<double, int>;   // {ready time, unit}: earliest first
        using AE = std::pair<long long, int>;  // {urgency, -unit}: most urgent first
        std::priority_queue<TE, std::vector<TE>, std::greater<TE>> pending, warps;
        std::priority_queue<AE> avail;
        std::vector<double> rdy(NT, 0.0), start(NT, 0.0);
        for (size_t t = 0; t < NT; ++t)
            if (head[t] == (int)t && ndep[t] == 0) pending.push({0.0, (int)t});
        for (int w = 0; w < W; ++w) warps.push({0.0, w});
        auto urgency = [&](int t) { return ((long long)theight[t] << 20) - tasks[t].level; };
        size_t done = 0;
        std::vector<int> w_of_task(NT, 0);
        while (done < n_units) {
            auto [tau, w] = warps.top();
            warps.pop();
            while (!pending.empty() && pending.top().first <= tau) {
                const int t = pending.top().second;
                pending.pop();
                avail.push({urgency(t), -t});
            }
            int t;
            double st = tau;
            if (!avail.empty()) {
                t = -avail.top().second;
                avail.pop();
            } else {
                if (pending.empty()) throw std::runtime_error("stream plan: dependency cycle");
                t = pending.top().second;
                st = pending.top().first;
                pending.pop();
            }
            const double f = st + (double)bsize[t];
            for (int q = 0; q < bsize[t]; ++q) {
                start[t + q] = st + q;
                fin[t + q] = f;
                w_of_task[t + q] = w;
            }
            warps.push({f, w});
            span_list = std::max(span_list, f);
            ++done;
            for (long long e = sptr[t]; e < sptr[t + 1]; ++e) {
                const int s = succ[(size_t)e];
                rdy[s] = std::max(rdy[s], f + hop);
                if (--ndep[s] == 0) pending.push({rdy[s], s});
            }
        }
        std::iota(by_rank.begin(), by_rank.end(), 0);
        std::stable_sort(by_rank.begin(), by_rank.end(), [&](int x, int y) { return start[x] < start[y]; });
        for (size_t r = 0; r < NT; ++r) warp_of[r] = w_of_task[by_rank[r]];
    }
    S.task_warp = warp_of;
    std::vector<int> rank_of(NT);
    for (size_t r = 0; r < NT; ++r) rank_of[by_rank[r]] = (int)r;
    // per-warp sequences
    std::vector<long long> wptr(W + 1, 0);
    for (size_t r = 0; r < NT; ++r) ++wptr[warp_of[r] + 1];
    for (int w = 0; w < W; ++w) wptr[w + 1] += wptr[w];
    std::vector<int> wseq(NT), wpos(NT);
    {
        std::vector<long long> at(wptr.begin(), wptr.end() - 1);
        for (size_t r = 0; r < NT; ++r) {
            wpos[r] = (int)(at[warp_of[r]] - wptr[warp_of[r]]);
            wseq[(size_t)at[warp_of[r]]++] = (int)r;
        }
    }
    // ---- stream sizes
    auto rec_bytes = [&](const Task& t) { return (16 + t.nq * (t.cont ? 256 : 384) + t.cnt * MS + 15) / 16 * 16; };
    std::vector<long long> bytes(W, 0);
    for (size_t r = 0; r < NT; ++r) {
        const int rb = rec_bytes(tasks[by_rank[r]]);
        bytes[warp_of[r]] += rb;
        S.max_record = std::max(S.max_record, rb);
    }
    if (S.max_record > kStreamSlot) throw std::runtime_error("stream plan: record larger than its slot");
    if (P.levels > 0xFFFF) throw std::runtime_error("stream plan: too many levels");
    std::vector<long long> off(W + 1, 0);
    for (int w = 0; w < W; ++w) off[w + 1] = off[w] + bytes[w];
    S.data.assign((size_t)off[W] + 16, 0);
    S.desc.assign((size_t)8 * W, 0);
    for (int w = 0; w < W; ++w) {
        S.desc[8 * (size_t)w] = (int)(off[w] & 0xFFFFFFFFll);
        S.desc[8 * (size_t)w + 1] = (int)(off[w] >> 32);
        const long long nt = wptr[w + 1] - wptr[w];
        S.desc[8 * (size_t)w + 2] = (int)nt;
        for (int k = 0; k < kStreamRing - 1; ++k)
            S.desc[8 * (size_t)w + 3 + k] = k < nt ? rec_bytes(tasks[by_rank[wseq[(size_t)wptr[w] + k]]]) : 0;
    }
    std::vector<long long> cur(off.begin(), off.end() - 1);
    for (size_t r = 0; r < NT; ++r) {
        const Task& T = tasks[by_rank[r]];
        const int w = warp_of[r];
        const int rb = rec_bytes(T);
        size_t at = (size_t)cur[w];
        cur[w] += rb;
        // the flag: the dependency whose producer runs last (largest rank)
        int flag = dummy, flag_rank = -1;
        for (int seg = 0; seg < T.cnt; ++seg) {
            const int p = ord[T.first + seg];
            for (int k = P.meta[4 * (size_t)p + 2]; k < P.meta[4 * (size_t)p + 3]; ++k) {
                const int pr = rank_of[prod[P.col[k]]];
                if (pr >= (int)r) throw std::runtime_error("stream plan: a dependency is not ranked earlier");
                if (pr > flag_rank) {
                    flag_rank = pr;
                    flag = P.col[k];
                }
            }
        }
        if (T.cont) {  // right behind the task whose columns it repeats, on the same warp
            if (wpos[r] == 0) throw std::runtime_error("stream plan: a cont task opens a stream");
            const Task& pv = tasks[by_rank[wseq[(size_t)(wptr[w] + wpos[r] - 1)]]];
            if (pv.nq != T.nq || pv.lg != T.lg || pv.cnt != 1 || T.cnt != 1)
                throw std::runtime_error("stream plan: a cont task does not match its predecessor");
        }
        const long long ahead = wptr[w] + wpos[r] + (kStreamRing - 1);
        put<int>(S.data, at, T.cnt | (T.lg << 8) | (T.nq << 12) | (T.cont << 15) | (T.level << 16));
        put<int>(S.data, at + 4, ahead < wptr[w + 1] ? rec_bytes(tasks[by_rank[wseq[(size_t)ahead]]]) : 0);
        put<int>(S.data, at + 8, flag);
        put<int>(S.data, at + 12, (int)r);
        // cont records carry no column ids
        const size_t col_at = at + 16, val_at = col_at + (T.cont ? 0 : (size_t)T.nq * 128),
                     meta_at = val_at + (size_t)T.nq * 256;
        if (!T.cont)
            for (int q = 0; q < T.nq * 32; ++q) put<int>(S.data, col_at + 4 * (size_t)q, dummy);
        const int lpr = 1 << T.lg;
        for (int seg = 0; seg < T.cnt; ++seg) {
            const int p = ord[T.first + seg];
            const int out = P.meta[4 * (size_t)p], in = P.meta[4 * (size_t)p + 1];
            const int k0 = P.meta[4 * (size_t)p + 2], k1 = P.meta[4 * (size_t)p + 3];
            const size_t m = meta_at + (size_t)seg * MS;
            put<int>(S.data, m, out);
            put<int>(S.data, m + 4, in);
            if (upper) {
                put<int>(S.data, m + 8, (out_index && out < P.n) ? out_index[out] : -1);
                put<int>(S.data, m + 12, 0);
                put<double>(S.data, m + 16, 1.0 / P.diag[out]);  // FAST: multiply by the reciprocal
            }
            for (int e = 0; e < k1 - k0; ++e) {
                const int sl = e & (lpr - 1), q = e >> T.lg;
                const int slot = q * 32 + seg * lpr + sl;
                if (!T.cont) put<int>(S.data, col_at + 4 * (size_t)slot, P.col[k0 + e]);
                put<double>(S.data, val_at + 8 * (size_t)slot, P.val[k0 + e]);
            }
            S.n_entries += k1 - k0;
        }
        S.n_slots += T.nq * 32;
        S.n_cont += T.cont;
        // distinct 32-byte sectors the task's gather instructions touch
        for (int q = 0; q < (T.cont ? 0 : T.nq); ++q) {
            int sec[32];
            for (int l = 0; l < 32; ++l) sec[l] = get<int>(S.data.data() + col_at + 4 * (size_t)(q * 32 + l)) >> 2;
            std::sort(sec, sec + 32);
            S.n_gather_sectors += std::unique(sec, sec + 32) - sec;
        }
    }
    if (getenv("EXG_PLAN_VERBOSE"))
        fprintf(stderr, "stream plan %s: schedule %s, warps %d, modelled span (task costs, hop %.2f): level order %.1f, list %.1f; tasks/warp %.1f\n",
                upper ? "U" : "L", prm.sched ? "list" : "level order", W, hop, span_level, span_list, (double)NT / W);
    if (getenv("EXG_PLAN_VERBOSE"))
        fprintf(stderr, "stream plan %s: tasks %lld (%lld reuse the columns of the task before) entries %lld gather sectors %lld (%.2f per entry) bytes %zu levels %d\n",
                upper ? "U" : "L", S.n_tasks, S.n_cont, S.n_entries, S.n_gather_sectors,
                (double)S.n_gather_sectors / (double)std::max<long long>(1, S.n_entries), S.data.size(), S.levels);
}

void eval_stream_plan(const StreamPlan& S, bool upper, const double* in, double* out, double* final_out,
                      double coef, const double* add) {
    const int W = S.n_warps, MS = upper ? kStreamMetaU : kStreamMetaL;
    std::vector<long long> cur(W), left(W);
    std::vector<const unsigned char*> last_cols(W, nullptr);  // column ids of the warp's last non-cont record
    std::vector<int> last_nq(W, -1);
    for (int w = 0; w < W; ++w) {
        cur[w] = ((long long)(unsigned)S.desc[8 * (size_t)w]) | ((long long)S.desc[8 * (size_t)w + 1] << 32);
        left[w] = S.desc[8 * (size_t)w + 2];
    }
    out[S.n_aug] = 0.0;  // the dummy
    for (long long t = 0; t < S.n_tasks; ++t) {
        const int w = S.task_warp[(size_t)t];
        if (w < 0 || w >= W) throw std::runtime_error("stream plan: bad warp of a task");
        if (left[w]-- <= 0) throw std::runtime_error("stream plan: task count mismatch");
        const unsigned char* r = S.data.data() + cur[w];
        const int w0 = get<int>(r);
        const int cnt = w0 & 0xFF, lg = (w0 >> 8) & 0xF, nq = (w0 >> 12) & 0x7, lpr = 1 << lg;
        const bool cont = (w0 >> 15) & 1;
        if (get<int>(r + 12) != (int)t) throw std::runtime_error("stream plan: record order mismatch");
        const int rb = (16 + nq * (cont ? 256 : 384) + cnt * MS + 15) / 16 * 16;
        if (cont && (last_nq[w] != nq || cnt != 1 || lg != 5))
            throw std::runtime_error("stream plan: a cont record does not follow a matching record");
        // integrity of what the kernel will trust: sizes, ids, the look-ahead size
        if (cnt < 1 || cnt > 32 || lg > 5 || (cnt << lg) > 32 || nq > 4 || rb > kStreamSlot ||
            (size_t)(cur[w] + rb) > S.data.size())
            throw std::runtime_error("stream plan: malformed record header");
        const int fc = get<int>(r + 8);
        if (fc < 0 || fc > S.n_aug) throw std::runtime_error("stream plan: flag column out of range");
        cur[w] += rb;
        const unsigned char* cols = cont ? last_cols[w] : r + 16;
        const unsigned char* vals = r + 16 + (cont ? 0 : (size_t)nq * 128);
        last_cols[w] = cols;
        last_nq[w] = (cnt == 1 && lg == 5) ? nq : -1;
        const unsigned char* meta = vals + (size_t)nq * 256;
        double acc[32];
        for (int lane = 0; lane < 32; ++lane) {
            double a = 0.0;
            for (int q = 0; q < nq; ++q) {
                const int c = get<int>(cols + 4 * (size_t)(q * 32 + lane));
                if (c < 0 || c > S.n_aug) throw std::runtime_error("stream plan: column id out of range");
                a = std::fma(get<double>(vals + 8 * (size_t)(q * 32 + lane)), out[c], a);
            }
            acc[lane] = a;
        }
        for (int o = lpr >> 1; o > 0; o >>= 1) {
            double nx[32];
            for (int lane = 0; lane < 32; ++lane) nx[lane] = acc[lane] + acc[lane ^ o];
            std::memcpy(acc, nx, sizeof nx);
        }
        for (int seg = 0; seg < cnt; ++seg) {
            const unsigned char* m = meta + (size_t)seg * MS;
            const int o = get<int>(m), i = get<int>(m + 4);
            if (o < 0 || o >= S.n_aug || i >= S.n) throw std::runtime_error("stream plan: row id out of range");
            double s = (i >= 0 ? in[i] : 0.0) - acc[seg * lpr];
            if (upper) s = s * get<double>(m + 16);
            out[o] = s;
            if (upper && final_out) {
                const int qq = get<int>(m + 8);
                if (qq >= 0) {
                    const double y = coef * s;
                    final_out[qq] = add ? add[qq] + y : y;
                }
            }
        }
    }
}

}  // namespace exg
