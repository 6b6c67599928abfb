// FAST-mode triangular-solve plan: the "blocked augmented system".
//
// Factorization::solve (sparse_lu.cpp:255-291) sweeps L forward and U
// backward row by row; at config 1 (n = 1M) each triangle has 7052 dependent
// levels, 6707 of them with <= 48 rows: the nested-dissection separators,
// which min-degree turns into DENSE diagonal blocks (supernodes; the largest
// has 2519 rows, 137 of them hold every thin level).  Substituting through a
// dense block costs one dependent hand-off per row.  This plan rewrites each
// dense diagonal block B (rows a..b-1, |B| >= min_block) as two hops:
//
//   y_i = b_i - sum_{c outside B} T_ic x_c         (the block's external part)
//   x_i = sum_{k in B} (T_BB^-1)_ik y_k             (explicit block inverse)
//
// and cuts the oldest entries of every long row into partial sums
//   p = - sum_{chunk} T_ic x_c,   row: s = b - sum_{recent} T_ic x_c + sum p
// scheduled at their own (earlier) level, so that a row's long history is
// reduced while its newest dependencies are still being solved.  Every new
// unknown is one more "row" of a triangular system over n + extra unknowns,
// all of the form  out = (in ? b : 0) - sum v * dep  (U: then / diag), which
// is exactly what the sync-free warp-task kernel k_trsv3 evaluates.  The
// critical path at config 1 drops from 7052 levels to about 150.
//
// The block inverse changes the rounding (FAST mode, <= 1e-13 relative, DESIGN
// §5); EXACT mode never uses this plan.
#pragma once

#include <cstdint>
#include <vector>

namespace exg {

struct AugPlan {
    int n = 0;               // original unknowns (x), ids 0..n-1
    long long n_aug = 0;     // all unknowns: x, block y's, partial sums
    int levels = 0;          // dependency levels of the augmented system
    int orig_levels = 0;     // levels of the triangle without the rewrite
    int n_blocks = 0;        // dense diagonal blocks rewritten
    long long block_rows = 0;
    int max_block = 0;
    long long n_partials = 0;
    // per level-order position: {out id, in index or -1, k0, k1}
    std::vector<int> meta;   // 4 ints per position
    std::vector<int> col;    // dependency ids (into the augmented unknowns)
    std::vector<double> val;
    std::vector<double> diag;  // per out id (U only; 1.0 for every non-x row and block x rows)
    // warp tasks over the positions: {first position, cnt | log2(lanes) << 8 | LONG << 30}
    std::vector<int> tasks;  // 2 ints per task
    std::vector<int> level_first_task;  // levels + 1 entries
};

struct AugParams {
    int min_block = 8;      // smallest dense diagonal block rewritten
    int max_block = 4096;   // larger dense blocks are split (inverse storage s^2/2)
    int chunk_over = 384;   // rows with more entries get partial sums
    int recent = 128;       // newest entries kept inline
    int chunk = 256;        // entries per partial sum
};

// upper: U (rows depend on larger indices, divided by diag); else strictly
// lower unit L.  ptr/col/val: the strictly triangular part in pivot
// coordinates, columns ascending.  in_index[r]: where row r's right-hand side
// is read (row_perm for L, identity for U).
void build_aug_plan(bool upper, int n, const int* ptr, const int* col, const double* val,
                    const double* diag, const int* in_index, const AugParams& prm, AugPlan& P);

// CPU evaluation of a plan in position order (test helper: the same
// arithmetic the kernel performs, sequentially).  out has n_aug entries.
void eval_aug_plan(const AugPlan& P, bool upper, const double* in, double* out);

}  // namespace exg
