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
    std::vector<long long> level_first_pos;  // levels + 1 entries (positions are in level order)
};

struct AugParams {
    int min_block = 8;      // smallest dense diagonal block rewritten
    int max_block = 4096;   // larger dense blocks are split (inverse storage s^2/2)
    int chunk_over = 384;   // rows with more entries get partial sums
    int recent = 128;       // newest entries kept inline
    int chunk = 256;        // entries per partial sum
    int cap = 0;            // > 0: no row keeps more than cap entries (partials of partials if
                            // needed); the stream plan needs cap <= 128 (one 4-entry batch per lane)
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

// ---------------------------------------------------------------------------
// Per-warp record streams for k_trsv4 (trsv_stream.cu).
//
// The augmented rows (every one <= 128 entries: AugParams.cap) are cut, level
// by level, into warp tasks of at most 32 lanes x 4 entries, and each warp's
// tasks are serialised, in order, into ONE contiguous byte stream.  The warp
// pulls its stream through a shared-memory ring of kStreamRing record slots,
// one bulk async copy (TMA) per record, a few records ahead: nothing on a
// task's path is a dependent global load any more, and every field sits at a
// fixed offset of its slot.
//
// Which warp runs which task, and when, is a list schedule (StreamParams.sched):
// W warps with unit task cost and a hand-off of `hop` costs from a producer's
// finish to a consumer's start are simulated; the warp that frees first takes
// the ready task with the longest chain of dependent rows behind it (or waits
// for the first to become ready).  Ranks follow the simulated start times, a
// warp runs its tasks by ascending rank and every dependency has a smaller
// rank, so whatever the real timing the unfinished task of smallest rank can
// run: no deadlock.  (Level by level with task t on warp t mod W, the first
// plan, left every critical task behind up to five rounds of its level's
// other tasks: 0.99 ms per solve pair at config 1 against 0.84.)
//
// Rows of 65..128 entries are tasks of their own, and most of them repeat the
// column list of another row of their level (the rows of a block inverse over
// one 128-column chunk; in U the rows of a supernode over its ancestors: 54% of
// L's and 82% of U's single-row tasks at config 1).  Up to StreamParams.bundle
// of them run back to back on one warp; the first gathers the dependencies,
// the others ("cont" records, no column ids) reuse its registers.
//
// Record (16-byte multiple, <= kStreamSlot bytes):
//   header 16 B  {cnt | lg << 8 | nq << 12 | cont << 15 | level << 16,
//                 bytes of this warp's record kStreamRing - 1 places ahead (0: none),
//                 flag, task id}
//                cnt rows (1..32), 2^lg lanes per row, nq (0..4) value batches;
//                flag = the dependency produced by the latest task (the one
//                value a waiting task polls)
//   nq x 32 column ids (int32); an empty slot holds the dummy id n_aug, whose
//                value is always 0.0.  Absent in a cont record (cnt 1, lg 5): its
//                columns are those of the record before it in the stream
//   nq x 32 values (fp64)
//   cnt metas    L: {out id, rhs index or -1}                                 (8 B)
//                U: {out id, rhs index or -1, epilogue index or -1, 0, 1 / diag}  (24 B)
// Lane l = seg * 2^lg + sl owns entries sl, sl + 2^lg, ... of row seg, stored
// at slot q * 32 + l (conflict-free shared-memory reads, coalesced in HBM).
// desc holds 8 ints per warp: {stream offset (lo, hi), tasks, bytes of its
// first kStreamRing - 1 records, 0, 0}.
constexpr int kStreamRing = 4;     // record slots per warp
constexpr int kStreamSlot = 2048;  // bytes per slot

struct StreamParams {
    int n_warps = 0;              // co-resident warps of the launch (upper bound)
    int min_tasks_per_warp = 4;   // small systems use fewer warps (a multiple of 8)
    // order of execution: 0 = level by level, task t on warp t mod W;
    // 1 = list schedule (most urgent ready task first on the warp that frees
    // first), simulated with unit task cost and a producer-to-consumer
    // hand-off of `hop` task costs
    int sched = 1;
    double hop = 3.0;
    // list schedule only: up to `bundle` single-row tasks with one column list
    // run back to back on one warp and share the gathered dependencies
    // (measured at config 1: 3 is best; from 8 up the serial bundle costs more
    // than the shared gathers save, also when only rows with slack are bundled)
    int bundle = 3;
};

struct StreamPlan {
    int n = 0;
    int n_warps = 0;
    int levels = 0;
    long long n_aug = 0;          // unknowns; out[n_aug] is the dummy (0.0)
    long long n_tasks = 0, n_rows = 0, n_entries = 0, n_slots = 0;
    long long n_cont = 0;            // tasks that reuse the columns (and gathered values) of the task before
    long long n_gather_sectors = 0;  // distinct 32-byte sectors over all gather instructions
    int max_record = 0;
    std::vector<int> desc;        // 8 ints per warp
    std::vector<unsigned char> data;
    std::vector<int> task_warp;   // warp of the task of each rank (host only: eval_stream_plan)
};

// debug overrides: EXG_STREAM_SCHED=0|1, EXG_STREAM_HOP=<task costs>
void stream_params_env(StreamParams& p);

constexpr int kStreamMetaL = 8, kStreamMetaU = 24;

// augmented-system parameters of the stream plan: every row <= 128 entries
inline AugParams stream_aug_params() {
    AugParams p;
    // dense diagonal blocks from 2 rows up: the chains of small supernodes at
    // the bottom of the tree are 16 levels shorter per triangle at config 1
    // (136 -> 120, 127 -> 111; 0.75 -> 0.71 ms per solve pair)
    p.min_block = 2;
    p.chunk_over = 128;
    p.recent = 0;
    p.chunk = 128;
    p.cap = 128;
    return p;
}

// out_index (may be null): epilogue index of x row r (U: col_perm), written
// into the metas of rows with out < n.
void build_stream_plan(const AugPlan& P, bool upper, const int* out_index, const StreamParams& prm,
                       StreamPlan& S);

// CPU evaluation of the streams in global task order with the kernel's
// arithmetic (per-lane fused multiply-adds, xor-butterfly over the row's
// lanes, b - acc, U: / diag).  out: n_aug + 1 entries (the dummy last).  final_out (may be null):
// final_out[q] = (add ? add[q] : 0) + coef * x for rows carrying an epilogue index.
void eval_stream_plan(const StreamPlan& S, bool upper, const double* in, double* out, double* final_out,
                      double coef, const double* add);

}  // namespace exg
