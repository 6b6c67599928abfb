// Blocked augmented triangular system for the FAST solve (see trsv_plan.hpp).
#include "trsv_plan.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <numeric>
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
    // ---- tasks: within a level rows are independent, so they are taken
    // longest first and grouped by lane class
    struct Task {
        long long first;  // index into `ord`
        int cnt, lg, nq, level;
    };
    std::vector<int> ord(np);
    std::iota(ord.begin(), ord.end(), 0);
    auto len_of = [&](int p) { return P.meta[4 * (size_t)p + 3] - P.meta[4 * (size_t)p + 2]; };
    std::vector<Task> tasks;
    for (int l = 0; l < P.levels; ++l) {
        const long long a = P.level_first_pos[l], b = P.level_first_pos[l + 1];
        std::stable_sort(ord.begin() + a, ord.begin() + b, [&](int x, int y) { return len_of(x) > len_of(y); });
        long long i = a;
        while (i < b) {
            const int len = len_of(ord[i]);
            if (len > 128) throw std::runtime_error("stream plan: a row exceeds 128 entries (AugParams.cap)");
            const int lg = lanes_log2_for(len);
            Task t{i, 0, lg, (len + (1 << lg) - 1) >> lg, l};
            // rows per task: the lane count, and the record must fit its slot
            const int per = std::max(1, std::min(32 >> lg, (kStreamSlot - 16 - t.nq * 384) / MS));
            while (i < b && t.cnt < per && lanes_log2_for(len_of(ord[i])) == lg) {
                ++t.cnt;
                ++i;
            }
            tasks.push_back(t);
        }
    }
    S.n_tasks = (long long)tasks.size();
    int W = prm.n_warps;
    if (prm.min_tasks_per_warp > 0) {
        const long long want = ((long long)tasks.size() / prm.min_tasks_per_warp + 7) / 8 * 8;
        W = (int)std::max<long long>(8, std::min<long long>(W, want));  // a multiple of 8 (and of any CTA's warps)
        W = std::min(W, prm.n_warps);
    }
    S.n_warps = W;
    // ---- stream sizes
    auto rec_bytes = [&](const Task& t) { return (16 + t.nq * 384 + t.cnt * MS + 15) / 16 * 16; };
    std::vector<long long> bytes(W, 0);
    for (size_t t = 0; t < tasks.size(); ++t) {
        const int rb = rec_bytes(tasks[t]);
        bytes[t % W] += rb;
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
        const long long nt = ((long long)tasks.size() - w + W - 1) / W;
        S.desc[8 * (size_t)w + 2] = (int)std::max<long long>(0, nt);
        for (int k = 0; k < kStreamRing - 1; ++k) {
            const size_t t = (size_t)w + (size_t)k * W;
            S.desc[8 * (size_t)w + 3 + k] = t < tasks.size() ? rec_bytes(tasks[t]) : 0;
        }
    }
    // the task that produces each unknown: a task's flag is its dependency
    // with the latest producer
    std::vector<int> prod((size_t)P.n_aug, -1);
    for (size_t t = 0; t < tasks.size(); ++t)
        for (int seg = 0; seg < tasks[t].cnt; ++seg) prod[P.meta[4 * (size_t)ord[tasks[t].first + seg]]] = (int)t;
    std::vector<long long> cur(off.begin(), off.end() - 1);
    for (size_t t = 0; t < tasks.size(); ++t) {
        const Task& T = tasks[t];
        const int rb = rec_bytes(T);
        size_t at = (size_t)cur[t % W];
        cur[t % W] += rb;
        int flag = dummy, flag_task = -1;
        for (int seg = 0; seg < T.cnt; ++seg) {
            const int p = ord[T.first + seg];
            for (int k = P.meta[4 * (size_t)p + 2]; k < P.meta[4 * (size_t)p + 3]; ++k)
                if (prod[P.col[k]] > flag_task) {
                    flag_task = prod[P.col[k]];
                    flag = P.col[k];
                }
        }
        const size_t ahead = t + (size_t)(kStreamRing - 1) * W;
        put<int>(S.data, at, T.cnt | (T.lg << 8) | (T.nq << 12) | (T.level << 16));
        put<int>(S.data, at + 4, ahead < tasks.size() ? rec_bytes(tasks[ahead]) : 0);
        put<int>(S.data, at + 8, flag);
        put<int>(S.data, at + 12, (int)t);
        const size_t col_at = at + 16, val_at = col_at + (size_t)T.nq * 128, meta_at = val_at + (size_t)T.nq * 256;
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
                put<int>(S.data, col_at + 4 * (size_t)slot, P.col[k0 + e]);
                put<double>(S.data, val_at + 8 * (size_t)slot, P.val[k0 + e]);
            }
            S.n_entries += k1 - k0;
        }
        S.n_slots += T.nq * 32;
        // distinct 32-byte sectors the task's gather instructions touch
        for (int q = 0; q < T.nq; ++q) {
            int sec[32];
            for (int l = 0; l < 32; ++l) sec[l] = get<int>(S.data.data() + col_at + 4 * (size_t)(q * 32 + l)) >> 2;
            std::sort(sec, sec + 32);
            S.n_gather_sectors += std::unique(sec, sec + 32) - sec;
        }
    }
    if (getenv("EXG_PLAN_VERBOSE"))
        fprintf(stderr, "stream plan %s: tasks %lld entries %lld gather sectors %lld (%.2f per entry) bytes %zu levels %d\n",
                upper ? "U" : "L", S.n_tasks, S.n_entries, S.n_gather_sectors,
                (double)S.n_gather_sectors / (double)std::max<long long>(1, S.n_entries), S.data.size(), S.levels);
}

void eval_stream_plan(const StreamPlan& S, bool upper, const double* in, double* out, double* final_out,
                      double coef, const double* add) {
    const int W = S.n_warps, MS = upper ? kStreamMetaU : kStreamMetaL;
    std::vector<long long> cur(W), left(W);
    for (int w = 0; w < W; ++w) {
        cur[w] = ((long long)(unsigned)S.desc[8 * (size_t)w]) | ((long long)S.desc[8 * (size_t)w + 1] << 32);
        left[w] = S.desc[8 * (size_t)w + 2];
    }
    out[S.n_aug] = 0.0;  // the dummy
    for (long long t = 0; t < S.n_tasks; ++t) {
        const int w = (int)(t % W);
        if (left[w]-- <= 0) throw std::runtime_error("stream plan: task count mismatch");
        const unsigned char* r = S.data.data() + cur[w];
        const int w0 = get<int>(r);
        const int cnt = w0 & 0xFF, lg = (w0 >> 8) & 0xF, nq = (w0 >> 12) & 0x7, lpr = 1 << lg;
        if (get<int>(r + 12) != (int)t) throw std::runtime_error("stream plan: record order mismatch");
        const int rb = (16 + nq * 384 + cnt * MS + 15) / 16 * 16;
        // integrity of what the kernel will trust: sizes, ids, the look-ahead size
        if (cnt < 1 || cnt > 32 || lg > 5 || (cnt << lg) > 32 || nq > 4 || rb > kStreamSlot ||
            (size_t)(cur[w] + rb) > S.data.size())
            throw std::runtime_error("stream plan: malformed record header");
        const int fc = get<int>(r + 8);
        if (fc < 0 || fc > S.n_aug) throw std::runtime_error("stream plan: flag column out of range");
        cur[w] += rb;
        const unsigned char* cols = r + 16;
        const unsigned char* vals = cols + (size_t)nq * 128;
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
