// Device-side argument blocks and kernel launch wrappers (internal).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace exg {
namespace dev {

struct Ctrl;

struct TrsvArgs {
    int n;
    const int* order;   // rows in level order
    const int* ptr;     // off-diagonal CSR (pivot coordinates)
    const int* col;
    const double* val;
    const double* diag; // U only
    const double* in;   // L: b (original coords, gathered through in_perm); U: L's output
    const int* in_perm; // row_perm (L)
    double* out;        // pivot-coordinate result, sentinel-initialised
    unsigned int* ticket;
    // optional fused epilogue: final_out[out_perm[r]] = (add ? add[q] : 0) + coef * x
    double* final_out;
    const int* out_perm;
    const double* add;
    double coef;
    const Ctrl* ctrl;   // early exit when the MEVP has converged
    const int2* tasks;  // warp tasks in level order (v2 kernel); null = v1
    int n_tasks;
    unsigned long long* trace;  // debug: per row (start, end) %globaltimer, or null
    const int4* meta;   // v3: per level-order position {row, b index, k0, k1}
};

// k_trsv4 (trsv_stream.cu): per-warp record streams of one triangle
struct StreamArgs {
    const unsigned char* data;   // all streams (trsv_plan.hpp record format)
    const int* desc;             // 8 ints per warp: stream offset, tasks, first record sizes
    int n_warps;
    long long n_aug;             // unknowns; out[n_aug] is the dummy entry (0.0)
    const double* in;            // right-hand side (L: b, gathered through the baked row_perm; U: L's output)
    double* out;                 // n_aug + 1 results, sentinel-initialised
    double* final_out;           // U: fused epilogue final_out[q] = (add ? add[q] : 0) + coef * x
    const double* add;
    double coef;
    const Ctrl* ctrl;
    unsigned long long* trace;   // debug: 5 values per task, or null
    int nodeps;                  // debug (EXG_STREAM_NODEPS): ignore readiness, wrong results: throughput bound only
};

struct SubArgs {
    int n_comps;
    int max_rows;         // shared-memory slots (largest component)
    int max_tasks;        // largest component's task count
    int max_levels;       // deepest component's level count
    const int2* clev;     // per component: (first entry in ltp, levels)
    const int* ltp;       // per component level: first task (ends with the component's task end)
    const int4* comps;    // per component: (first task, tasks, first position, rows)
    const int2* tasks;    // (first position, rows | log2(lanes per row) << 8 | long << 30)
    const int4* meta;     // per position: (row, b index, first entry, end entry)
    const int* ecol;      // >= 0: row of an earlier phase (global); < 0: ~component slot
    const double* eval;
    const double* in;
    const double* diag;   // U only
    double* out;
    double* final_out;
    const int* out_perm;
    const double* add;
    double coef;
    const Ctrl* ctrl;
};

struct ChainArgs {
    int n_rows;            // positions of this run
    int n_blocks;
    const int* rows;       // row id per position (run-local)
    const int2* rq;        // per position: (row id, output position of the fused epilogue)
    const int* nptr;       // per position: entries older than block k-2
    const int* ncol;       // global row ids
    const double* nval;
    const int4* blocks;    // 3 per block: (first pos, rows,-,-), (Dinv, F1, F2 offsets,-), -
    const double* pool;
    double* s;             // per position, sentinel-initialised
    double* part;          // partial sums of the old-entry chunks, one slot each (sentinel-initialised)
    const int* pslot;      // per position: first partial slot of its row
    const int4* wtasks;    // worker tasks: chunk (slot, k0, k1, 0) | recent (position, k0, k1, 1 | chunks << 8)
    int n_tasks;
    const double* in;
    const int* in_perm;
    double* out;
    double* final_out;
    const int* out_perm;
    const double* add;
    double coef;
    const Ctrl* ctrl;
    unsigned long long* trace;  // debug: per block timestamps, then per-position worker timestamps
    unsigned spin_ns;      // worker back-off between unsuccessful polls (0 = spin)
};

struct MgsArgs {
    int n;
    long long ldv;
    double* V;
    const double* w;
    double* hbar;
    int hld;
    double* partials;
    unsigned int* bar;
    Ctrl* ctrl;
};

// k_mgs2 (mgs.cu): grouped Gram-Schmidt with TMA-streamed basis tiles (FAST mode)
constexpr int kMgs2BMax = 4;
struct Mgs2Args {
    int n;
    long long ldv;
    double* V;
    const double* w;
    double* hbar;
    int hld;
    double* slots;       // 2 sets x inst_cap x grid x kMgs2BMax partial-sum slots (sentinel-initialised)
    unsigned int* seq;   // launch counter (selects the slot set)
    Ctrl* ctrl;
    int inst_cap;        // exchanges one launch may need: 2 (m_max + 1) + 3
    int tile, S, B;      // filled by mgs2 from the shape
};
struct Mgs2Shape {
    int grid, tile, S, B;
    size_t smem;
};

struct DenseArgs {
    Ctrl* ctrl;
    const double* hbar;
    int hld;
    double* hinv;     // persistent H_m^-1 (m x m, row-major)
    double* coef;     // final coefficients
    double* scratch;  // global scratch (used when the block does not fit smem)
    int smem_cap;     // dynamic shared memory of the launch (bytes)
    int mode;
    double h_eval;
    double* full_out;  // mode 3 (debug): the whole m x m exponential
};

// ---- launch wrappers (kernels.cu) ------------------------------------------
struct Launch {
    cudaStream_t stream;
    int num_sms;
    long long* launches;  // counter of this library's kernel launches
};

void spmv(const Launch& L, const int* rowptr, const int* col, const double* val, int n_rows,
          const double* x, double* y, const Ctrl* ctrl, const double* vbase, long long ldv);
// FAST-mode SpMV of the Arnoldi loop.  max_strip: the most entries any spmv_strip_rows() consecutive
// rows hold (0: unknown, direct loads); col/val must be readable 8 entries past nnz (upload_csr pads).
int spmv_strip_rows();
void spmv_v4(const Launch& L, const int* rowptr, const int* col, const double* val, int n_rows, int max_strip,
             double* y, const Ctrl* ctrl, const double* vbase, long long ldv);
void spmv_sub(const Launch& L, const int* rowptr, const int* col, const double* val, int n_rows,
              const double* x, const double* z, double* y);
void spmv_b2(const Launch& L, const int* rowptr, const int* col, const double* val, int n_rows,
             const double* u_k, const double* u_k1, double h, double* t1, double* t2, const double* Fk);
void mos_residual(const Launch& L, int n_mos, const int4* nodes, const double* par,
                  const double* op, const double* x, double* r, int n, const int* nptr,
                  const int* nlist, double* F, const double* fsub);
void absmax(const Launch& L, const double* v, int n, double* partials, unsigned int* done, double* out);
void axpby(const Launch& L, const double* a, double alpha, const double* b, double* out, int n);
void erc_update(const Launch& L, const double* w, const double* value, const double* u, int have_u,
                double ih, double gamma, double* x, int n);
void trsv(const Launch& L, bool upper, bool reverse, const TrsvArgs& a);
cudaError_t trsv_wide(const Launch& L, bool upper, const TrsvArgs& a);
cudaError_t trsv_chain(const Launch& L, bool upper, const ChainArgs& a);
int trsv_stream_warps(bool upper, int num_sms);  // co-resident warps of k_trsv4 (0 = cannot launch)
cudaError_t trsv_stream(const Launch& L, bool upper, const StreamArgs& a);
cudaError_t trsv_sub(const Launch& L, bool upper, const SubArgs& a);
void apply_tasks(const Launch& L, const int2* utasks, int n_utasks, const int* uorder,
                 const int2* ltasks, int n_ltasks, const int* lorder, const int* uptr,
                 const int* ucol, const double* uval, const double* udiag, const int* lptr,
                 const int* lcol, const double* lval, int n, const int* col_perm,
                 const int* row_perm, const double* x, double* t, double* y, double* sq,
                 double* y_out, double* partials, unsigned int* done, Ctrl* ctrl,
                 const double* vbase, long long ldv, double* weight_out);
void spmv_norm(const Launch& L, const int* rowptr, const int* col, const double* val, int n,
               const double* vbase, long long ldv, double* partials, unsigned int* done,
               Ctrl* ctrl, int from_ctrl_m, double* weight_out);
void start(const Launch& L, const double* v, const double* xk, int n, double* partials,
           double* v0, Ctrl* ctrl, int er_mode);
int mgs_max_blocks(int K);
cudaError_t mgs(const Launch& L, const MgsArgs& a, int n_blocks, int K);
bool mgs2_shape(int n, int num_sms, int b_override, Mgs2Shape* s);
cudaError_t mgs2(const Launch& L, Mgs2Args a, const Mgs2Shape& s);
void dense(const Launch& L, const DenseArgs& a, int m);
void iter_end(const Launch& L, Ctrl* ctrl, unsigned long long cond = 0);
void fill_ones(const Launch& L, void* p, size_t bytes);
void combine(const Launch& L, const double* V, long long ldv, const double* coef, int n,
             double* out, const Ctrl* ctrl, int mode, const double* xk, const double* gb,
             const double* start, double h);
void basis_residual_final(const Launch& L, Ctrl* ctrl, double* out);
size_t ctrl_size();

}  // namespace dev
}  // namespace exg
