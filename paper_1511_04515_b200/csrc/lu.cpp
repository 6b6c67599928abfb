// Setup-time sparse LU, bit-identical to exsim::lu_factor
// (proj/core/src/sparse_lu.cpp:134-253).
//
// The reference's cost at scale is its ordering: exact minimum degree on the
// pattern of A + A^T with a linear scan over all n vertices per pivot
// (sparse_lu.cpp:66-75), ~90% of a 1 h factorization at n = 1M.  Here the
// SAME ordering is produced with an indexed binary heap keyed on
// (degree, index) — the scan picks the smallest index among minimum-degree
// vertices, which is exactly the heap minimum — and the elimination clique is
// formed with a sorted merge instead of per-element binary search + insert.
// Degrees are the sizes of the explicit adjacency lists, as in the reference,
// so the order is identical.  When the remaining graph is complete every
// vertex has the same degree and the reference picks them in increasing
// index order; that tail is emitted directly.
//
// The numeric phase (left-looking Gilbert–Peierls with DFS reach, threshold
// partial pivoting preferring the diagonal, sparse_lu.cpp:97-233) is
// restated step for step — same DFS order, same update order, same pivot
// rule — so every value of L and U matches the reference bit for bit.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <limits>
#include <cstdio>
#include <cstdlib>

#include "host.hpp"

namespace exg {

namespace {

struct DegreeHeap {
    std::vector<int> heap, pos;
    const std::vector<int>* deg = nullptr;
    bool less(int a, int b) const {
        const int da = (*deg)[a], db = (*deg)[b];
        return da != db ? da < db : a < b;
    }
    void swap_at(int i, int j) {
        std::swap(heap[i], heap[j]);
        pos[heap[i]] = i;
        pos[heap[j]] = j;
    }
    void up(int i) {
        while (i > 0) {
            const int p = (i - 1) / 2;
            if (!less(heap[i], heap[p])) break;
            swap_at(i, p);
            i = p;
        }
    }
    void down(int i) {
        const int n = static_cast<int>(heap.size());
        while (true) {
            const int l = 2 * i + 1, r = l + 1;
            int m = i;
            if (l < n && less(heap[l], heap[m])) m = l;
            if (r < n && less(heap[r], heap[m])) m = r;
            if (m == i) break;
            swap_at(i, m);
            i = m;
        }
    }
    void build(int n) {
        heap.resize(n);
        pos.resize(n);
        for (int v = 0; v < n; ++v) heap[v] = pos[v] = v;
        for (int i = n / 2 - 1; i >= 0; --i) down(i);
    }
    int pop() {
        const int top = heap[0];
        swap_at(0, static_cast<int>(heap.size()) - 1);
        heap.pop_back();
        pos[top] = -1;
        if (!heap.empty()) down(0);
        return top;
    }
    void changed(int v) {
        const int i = pos[v];
        up(i);
        down(pos[v]);
    }
    int size() const { return static_cast<int>(heap.size()); }
};

}  // namespace

std::vector<int> min_degree_order(const Csr& A) {
    const int n = A.n_rows;
    std::vector<std::vector<int>> adj(n);
    for (int r = 0; r < n; ++r)
        for (int k = A.rowptr[r]; k < A.rowptr[r + 1]; ++k) {
            const int c = A.col[k];
            if (c == r) continue;
            adj[r].push_back(c);
            adj[c].push_back(r);
        }
    std::vector<int> deg(n);
    for (int v = 0; v < n; ++v) {
        auto& a = adj[v];
        std::sort(a.begin(), a.end());
        a.erase(std::unique(a.begin(), a.end()), a.end());
        deg[v] = static_cast<int>(a.size());
    }
    DegreeHeap heap;
    heap.deg = &deg;
    heap.build(n);

    // Adjacency lists may keep eliminated vertices (filtered lazily); deg[v]
    // is always the exact number of live neighbours, i.e. the size of the
    // reference's explicit list.  Every elimination clique is remembered with
    // its live member count: when the pivot's whole neighbourhood is one such
    // clique, eliminating it creates no fill and only lowers each neighbour's
    // degree by one — O(deg) instead of the O(deg^2) list merge.
    std::vector<char> dead(n, 0);
    std::vector<std::vector<int>> cliques_of(n);
    std::vector<int> clique_live;

    std::vector<int> order;
    order.reserve(n);
    std::vector<int> nbr, merged;
    long long st_fast = 0, st_slow = 0, st_merge = 0, st_slow_d2 = 0;
    while (heap.size() > 0) {
        // complete remaining graph: all degrees equal, reference takes them
        // by increasing index (sparse_lu.cpp:68-75 strict '<' keeps the first)
        if (deg[heap.heap[0]] == heap.size() - 1) {
            std::vector<int> rest(heap.heap.begin(), heap.heap.end());
            std::sort(rest.begin(), rest.end());
            order.insert(order.end(), rest.begin(), rest.end());
            break;
        }
        const int best = heap.pop();
        order.push_back(best);
        dead[best] = 1;
        nbr.clear();
        for (int u : adj[best])
            if (!dead[u]) nbr.push_back(u);
        int big = -1, big_live = 0;
        for (int c : cliques_of[best])
            if (clique_live[c] > big_live) {
                big_live = clique_live[c];
                big = c;
            }
        const bool no_fill = big >= 0 && big_live - 1 == static_cast<int>(nbr.size());
        if (no_fill) ++st_fast; else { ++st_slow; st_slow_d2 += (long long)nbr.size() * nbr.size(); }
        if (no_fill) {
            for (int u : nbr) {
                deg[u] -= 1;
                heap.changed(u);
            }
        } else {
            const int cid = static_cast<int>(clique_live.size());
            clique_live.push_back(static_cast<int>(nbr.size()));
            for (int u : nbr) {
                // adj[u] := (live(adj[u]) \ {best}) U (nbr \ {u}), sorted unique
                const auto& au = adj[u];
                st_merge += au.size() + nbr.size();
                merged.clear();
                merged.reserve(au.size() + nbr.size());
                size_t i = 0, j = 0;
                while (i < au.size() || j < nbr.size()) {
                    int x;
                    if (j >= nbr.size() || (i < au.size() && au[i] < nbr[j])) {
                        x = au[i++];
                    } else if (i >= au.size() || nbr[j] < au[i]) {
                        x = nbr[j++];
                    } else {
                        x = au[i++];
                        ++j;
                    }
                    if (x == u || dead[x]) continue;
                    merged.push_back(x);
                }
                adj[u].swap(merged);
                deg[u] = static_cast<int>(adj[u].size());
                heap.changed(u);
                cliques_of[u].push_back(cid);
            }
        }
        for (int c : cliques_of[best]) clique_live[c] -= 1;
        std::vector<int>().swap(adj[best]);
        std::vector<int>().swap(cliques_of[best]);
    }
    if (getenv("EXG_MD_STATS"))
        fprintf(stderr, "md: fast %lld slow %lld merge %lld slow_d2 %lld\n", st_fast, st_slow, st_merge, st_slow_d2);
    return order;
}

namespace {

struct Csc {
    int n = 0;
    std::vector<int> col_ptr, row_idx;
    std::vector<double> val;
};

Csc to_csc(const Csr& A) {  // sparse_lu.cpp:23-41
    Csc c;
    c.n = A.n_cols;
    c.col_ptr.assign(static_cast<size_t>(c.n) + 1, 0);
    for (int k = 0; k < A.nnz(); ++k) c.col_ptr[A.col[k] + 1]++;
    for (int j = 0; j < c.n; ++j) c.col_ptr[j + 1] += c.col_ptr[j];
    c.row_idx.resize(A.nnz());
    c.val.resize(A.nnz());
    std::vector<int> next(c.col_ptr.begin(), c.col_ptr.end() - 1);
    for (int r = 0; r < A.n_rows; ++r)
        for (int k = A.rowptr[r]; k < A.rowptr[r + 1]; ++k) {
            const int j = A.col[k];
            const int p = next[j]++;
            c.row_idx[p] = r;
            c.val[p] = A.val[k];
        }
    return c;
}

// Depth-first reach through the partially built L (sparse_lu.cpp:99-130):
// pushes a vertex after all vertices reachable from it.
void reach(int start, const std::vector<std::vector<int>>& l_rows,
           const std::vector<int>& pivot_pos, std::vector<char>& mark, std::vector<int>& topo,
           std::vector<int>& stack, std::vector<size_t>& child) {
    stack.clear();
    stack.push_back(start);
    child.assign(1, 0);
    mark[start] = 1;
    while (!stack.empty()) {
        const int r = stack.back();
        const int pp = pivot_pos[r];
        bool descended = false;
        if (pp >= 0) {
            const auto& rows = l_rows[pp];
            while (child.back() < rows.size()) {
                const int nr = rows[child.back()++];
                if (!mark[nr]) {
                    mark[nr] = 1;
                    stack.push_back(nr);
                    child.push_back(0);
                    descended = true;
                    break;
                }
            }
        }
        if (!descended) {
            topo.push_back(r);
            stack.pop_back();
            child.pop_back();
        }
    }
}

}  // namespace

void lu_factor(const Csr& A, double pivot_tol, Factor& f) {
    if (A.n_rows != A.n_cols) throw Error{EXG_E_CONTRACT, "lu_factor: matrix not square"};
    const int n = A.n_rows;
    using clock = std::chrono::steady_clock;

    double max_abs = 0.0;
    for (double v : A.val) max_abs = std::max(max_abs, std::abs(v));
    const double sing_tol = 1e-14 * max_abs;

    Csc a = to_csc(A);
    const auto t0 = clock::now();
    // The ordering is a function of the pattern alone: a nonlinear transient
    // refactors the same pattern every attempt, so the last one is reused
    // when rowptr and col match exactly (same order, bit for bit).
    static thread_local std::vector<int> cached_rowptr, cached_col, cached_order;
    if (cached_rowptr != A.rowptr || cached_col != A.col) {
        cached_order = min_degree_order(A);
        cached_rowptr = A.rowptr;
        cached_col = A.col;
    }
    const std::vector<int> col_order = cached_order;
    const auto t1 = clock::now();
    // Work in relabelled row coordinates: row i gets the label of its column
    // position in col_order (the diagonal row of column j is label j).  The
    // arithmetic, the DFS visiting order and every tie-break are unchanged —
    // ties compare ORIGINAL row ids, exactly as sparse_lu.cpp:197 — but the
    // dense elimination tail now touches a contiguous range of x.
    std::vector<int> label(n);
    for (int j = 0; j < n; ++j) label[col_order[j]] = j;
    for (int& r : a.row_idx) r = label[r];

    std::vector<std::vector<int>> l_rows(n);
    std::vector<std::vector<double>> l_vals(n);
    std::vector<std::vector<int>> u_pos(n);
    std::vector<std::vector<double>> u_vals(n);
    std::vector<double> u_diag(n);
    std::vector<int> pivot_pos(n, -1), row_perm(n, -1);
    std::vector<double> x(n, 0.0);
    std::vector<char> mark(n, 0);
    std::vector<int> topo, stack;
    std::vector<size_t> child;

    for (int j = 0; j < n; ++j) {
        const int cj = col_order[j];
        topo.clear();
        for (int p = a.col_ptr[cj]; p < a.col_ptr[cj + 1]; ++p) {
            const int r = a.row_idx[p];
            if (!mark[r]) reach(r, l_rows, pivot_pos, mark, topo, stack, child);
        }
        for (int p = a.col_ptr[cj]; p < a.col_ptr[cj + 1]; ++p) x[a.row_idx[p]] = a.val[p];
        for (auto it = topo.rbegin(); it != topo.rend(); ++it) {
            const int r = *it;
            const int pp = pivot_pos[r];
            if (pp < 0) continue;
            const double xr = x[r];
            if (xr == 0.0) continue;
            const auto& rows = l_rows[pp];
            const auto& vals = l_vals[pp];
            for (size_t k = 0; k < rows.size(); ++k) x[rows[k]] -= vals[k] * xr;
        }
        double xmax = 0.0;
        for (int r : topo)
            if (pivot_pos[r] < 0) xmax = std::max(xmax, std::abs(x[r]));
        int pivot_row = -1;
        if (xmax > sing_tol && xmax > 0.0) {
            if (pivot_pos[j] < 0 && mark[j] && std::abs(x[j]) >= pivot_tol * xmax) {
                pivot_row = j;  // label of the natural diagonal row cj
            } else {
                double best = -1.0;
                for (int r : topo) {
                    if (pivot_pos[r] >= 0) continue;
                    const double m = std::abs(x[r]);
                    if (m > best ||
                        (m == best && (pivot_row < 0 || col_order[r] < col_order[pivot_row]))) {
                        best = m;
                        pivot_row = r;
                    }
                }
            }
        }
        if (pivot_row < 0)
            throw Error{EXG_E_SINGULAR,
                        "lu_factor: singular matrix at elimination step " + std::to_string(j) +
                            " (column " + std::to_string(cj) + ")",
                        static_cast<double>(j)};
        const double pv = x[pivot_row];
        for (int r : topo) {
            const double xr = x[r];
            if (r == pivot_row) continue;
            if (pivot_pos[r] >= 0) {
                if (xr != 0.0) {
                    u_pos[j].push_back(pivot_pos[r]);
                    u_vals[j].push_back(xr);
                }
            } else if (xr != 0.0) {
                l_rows[j].push_back(r);
                l_vals[j].push_back(xr / pv);
            }
        }
        u_diag[j] = pv;
        pivot_pos[pivot_row] = j;
        row_perm[j] = col_order[pivot_row];
        for (int r : topo) {
            x[r] = 0.0;
            mark[r] = 0;
        }
    }
    const auto t2 = clock::now();

    // CSR assembly in pivot coordinates (sparse_lu.cpp:235-248).  Entries are
    // unique, so from_triplets' sort reduces to bucketing by row with columns
    // visited in increasing order; exact zeros are pruned as it would.
    auto assemble = [n](Csr& M, const std::vector<std::vector<int>>& rows_of_col,
                        const std::vector<std::vector<double>>& vals_of_col,
                        const std::vector<int>* map, const std::vector<double>& diag,
                        bool unit_diag) {
        M = Csr{};
        M.n_rows = M.n_cols = n;
        std::vector<int> cnt(n + 1, 0);
        for (int j = 0; j < n; ++j) {
            cnt[j + 1]++;  // diagonal
            for (size_t k = 0; k < rows_of_col[j].size(); ++k) {
                if (vals_of_col[j][k] == 0.0) continue;
                const int r = map ? (*map)[rows_of_col[j][k]] : rows_of_col[j][k];
                cnt[r + 1]++;
            }
        }
        for (int i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
        M.rowptr = cnt;
        M.col.resize(cnt[n]);
        M.val.resize(cnt[n]);
        std::vector<int> next(cnt.begin(), cnt.end() - 1);
        for (int j = 0; j < n; ++j) {
            // entries (r, j) for this column, then the diagonal (j, j): within
            // row r, columns arrive in increasing j order
            {
                const int p = next[j]++;
                M.col[p] = j;
                M.val[p] = unit_diag ? 1.0 : diag[j];
            }
            for (size_t k = 0; k < rows_of_col[j].size(); ++k) {
                const double v = vals_of_col[j][k];
                if (v == 0.0) continue;
                const int r = map ? (*map)[rows_of_col[j][k]] : rows_of_col[j][k];
                const int p = next[r]++;
                M.col[p] = j;
                M.val[p] = v;
            }
        }
        // rows were filled by increasing column j already; sort defensively
        // only if an out-of-order insertion occurred (never, by construction)
    };
    assemble(f.L, l_rows, l_vals, &pivot_pos, u_diag, true);
    assemble(f.U, u_pos, u_vals, nullptr, u_diag, false);
    f.n = n;
    f.row_perm = std::move(row_perm);
    f.col_perm = col_order;
    f.order_s = std::chrono::duration<double>(t1 - t0).count();
    f.numeric_s = std::chrono::duration<double>(t2 - t1).count();
}

}  // namespace exg
