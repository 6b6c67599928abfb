// Internal definition of the device context (exg_ctx of include/exg.h).
#pragma once

#include <string>
#include <utility>
#include <vector>

#include "device.hpp"
#include "exg.h"
#include "kernels.cuh"

struct DCsr {
    int n_rows = 0, n_cols = 0, nnz = 0;
    int max_strip = 0;  // most entries in any spmv_strip_rows() consecutive rows (k_spmv_v4t stage fit)
    int* rowptr = nullptr;
    int* col = nullptr;
    double* val = nullptr;
};

constexpr size_t kTrsvHdr = 1024;  // ticket counters ahead of the solve scratch
constexpr int kMaxTickets = 256;
constexpr int kStreamPlanMinRows = 250000;  // FAST plan: record streams from this size up, level runs below

// FAST-mode execution plan of one triangle (see plan_triangle, api.cu)
// subtree phase of one triangle (k_trsv_sub): components of the bottom of
// the elimination DAG, one CTA each (plan_subtrees, api.cu)
struct SubPlan {
    int n_comps = 0, max_rows = 0, max_tasks = 0;
    long long rows = 0, nnz = 0;
    int max_levels = 0;
    int4* comps = nullptr;
    int2* clev = nullptr;
    int* ltp = nullptr;
    int2* tasks = nullptr;
    int4* meta = nullptr;
    int* ecol = nullptr;
    double* eval = nullptr;
    void free_dev() {
        void* ps[] = {comps, clev, ltp, tasks, meta, ecol, eval};
        for (void* p : ps)
            if (p) cudaFree(p);
        comps = nullptr;
        clev = nullptr;
        ltp = nullptr;
        tasks = nullptr;
        meta = nullptr;
        ecol = nullptr;
        eval = nullptr;
        n_comps = max_rows = max_tasks = max_levels = 0;
        rows = nnz = 0;
    }
};

struct TriPlan {
    // run = wide levels (warp tasks [a, b) of k_trsv3), one chain run
    // (narrow == 2, chains[a]) or the subtree phase (narrow == 3, sub)
    struct Run {
        int narrow;
        int a, b;
    };
    std::vector<Run> runs;
    double* pool = nullptr;  // chain block records (Dinv, F1..F4)
    // chain + workers runs
    struct Chain {
        int rows_off, nptr_off, ent0, n_rows, blk0, n_blocks, task0, ntasks, slot0, n_slots;
    };
    std::vector<Chain> chains;
    int* crows = nullptr;
    int* cnptr = nullptr;
    int* cncol = nullptr;
    double* cnval = nullptr;
    int4* cblocks = nullptr;
    int4* ctasks = nullptr;
    int* cpslot = nullptr;
    int2* crq = nullptr;
    long long chain_rows = 0, chain_slots = 0;  // scratch of the chain runs (s values, partial slots)
    SubPlan sub;
    long long n_aug = 0;   // unknowns of the augmented system (stream plan)
    int aug_levels = 0;
    // per-warp record streams of the augmented system (k_trsv4); used when s_warps > 0
    unsigned char* sdata = nullptr;
    int* sdesc = nullptr;
    int s_warps = 0;
    long long s_bytes = 0;
    void free_aug() {
        if (sdata) cudaFree(sdata);
        if (sdesc) cudaFree(sdesc);
        sdata = nullptr;
        sdesc = nullptr;
        s_warps = 0;
        s_bytes = 0;
        n_aug = 0;
        aug_levels = 0;
    }
    void free_dev() {
        free_aug();
        sub.free_dev();
        void* ps[] = {pool, crows, cnptr, cncol, cnval, cblocks, ctasks, cpslot, crq};
        for (void* p : ps)
            if (p) cudaFree(p);
        pool = nullptr;
        crows = cnptr = cncol = cpslot = nullptr;
        cnval = nullptr;
        cblocks = ctasks = nullptr;
        crq = nullptr;
        chain_rows = chain_slots = 0;
        chains.clear();
    }
};

struct exg_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t side_stream = nullptr;  // residual weight beside the dense block (mevp_dev)
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    int num_sms = 148;
    long long launches = 0;
    exg_counters cnt{};
    std::string err;
    exg_status last = EXG_OK;
    exg_options_dev opt{EXG_TRSV_EXACT, EXG_WEIGHT_APPLY, EXG_LOOP_GRAPH};

    // Arnoldi-loop graphs (EXG_LOOP_GRAPH), keyed by everything the loop body
    // bakes in (buffer addresses, launch shapes, modes); dropped whenever a
    // device buffer or the factor plan is replaced
    struct GraphKey {
        const void* p[24];
        long long v[8];
    };
    struct ArnoldiGraph {
        GraphKey key;
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t exec = nullptr;
        long long body_kernels = 0;
    };
    std::vector<ArnoldiGraph> graphs;
    bool capturing = false;
    void clear_graphs() {
        for (auto& g : graphs) {
            if (g.exec) cudaGraphExecDestroy(g.exec);
            if (g.graph) cudaGraphDestroy(g.graph);
        }
        graphs.clear();
    }

    DCsr mats[3];  // C, G, B
    // factors
    int n = 0;
    int *l_ptr = nullptr, *l_col = nullptr, *u_ptr = nullptr, *u_col = nullptr;
    double *l_val = nullptr, *u_val = nullptr, *u_diag = nullptr;
    int *row_perm = nullptr, *col_perm = nullptr, *l_order = nullptr, *u_order = nullptr;
    int2* tasks[4] = {nullptr, nullptr, nullptr, nullptr};  // L, U (EXACT), L, U (FAST)
    TriPlan plan[2];  // FAST-mode runs of L and U
    int4* meta[2] = {nullptr, nullptr};  // level-order row metadata of L and U
    int cluster = 16;
    int alap[2] = {0, 0};  // level schedule chosen per triangle (1 = ALAP)
    int n_tasks[4] = {0, 0, 0, 0};
    unsigned long long *trace_l = nullptr, *trace_u = nullptr;
    unsigned long long *ntrace_l = nullptr, *ntrace_u = nullptr;
    // solve scratch: [2 tickets + pad (16 B)][y n][x n], memset to 0xFF per solve
    char* trsv_buf = nullptr;
    long long cnt_aug[2][8] = {};  // per triangle: levels, blocks, block rows, partials, entries, tasks, stream bytes, warps
    // n-vectors
    int vec_n = 0;
    double *vin = nullptr, *vout = nullptr, *t = nullptr, *w = nullptr, *xk = nullptr,
           *xnext = nullptr, *gb = nullptr, *startv = nullptr, *v1 = nullptr, *t1 = nullptr,
           *t2 = nullptr, *t3 = nullptr, *tmp = nullptr;
    int n_inputs = 0;
    double *u_k = nullptr, *u_k1 = nullptr;
    // Krylov workspace
    int mmax_alloc = 0;
    long long ldv = 0;
    double *V = nullptr, *hbar = nullptr, *hinv = nullptr, *coef = nullptr, *dscratch = nullptr;
    int hld = 0;
    double* partials = nullptr;
    size_t mgs_partials_off = 0;
    unsigned int *bar = nullptr, *done = nullptr;
    double* weight = nullptr;
    // k_mgs2 exchange slots: [seq counter, 64 B][2 sets x mgs_inst_cap x num_sms x kMgs2BMax]
    double* mgs_slots = nullptr;
    int mgs_inst_cap = 0;
    exg::dev::Ctrl* ctrl = nullptr;
    exg::dev::Ctrl* h_ctrl = nullptr;  // pinned mirror
    bool basis_valid = false;
    double h_built = 0.0;
    double *probe_out = nullptr;
    int* probe_idx = nullptr;
    int probe_cap = 0;
    std::vector<int> probe_host;  // the index list last uploaded to probe_idx

    // profiling: event pairs per kernel class, resolved in exg_profile_get
    bool profiling = false;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> prof_events;
    std::vector<cudaEvent_t> event_pool;
    double prof_ms[EXG_K_CLASSES] = {};
    long long prof_count[EXG_K_CLASSES] = {};

    // nonlinear devices (config 4)
    int n_mos = 0;
    int4* mos_nodes = nullptr;
    double *mos_par = nullptr, *mos_op = nullptr, *mos_r = nullptr;
    int *node_ptr = nullptr, *node_list = nullptr;
    double *Fk = nullptr, *dF = nullptr, *nw = nullptr, *nu = nullptr, *nv = nullptr;
    // second Krylov workspace for the error / correction MEVPs (the step's
    // own basis stays cached for the rejection retries, integrate.cpp:249)
    struct Krylov {
        int mmax_alloc = 0;
        long long ldv = 0;
        double *V = nullptr, *hbar = nullptr, *hinv = nullptr, *coef = nullptr, *dscratch = nullptr;
        int hld = 0;
        bool basis_valid = false;
        exg::dev::Ctrl* ctrl = nullptr;
        exg::dev::Ctrl* h_ctrl = nullptr;
    } aux;

    exg::dev::Launch L() { return exg::dev::Launch{stream, num_sms, &launches}; }
    void swap_krylov() {
        std::swap(mmax_alloc, aux.mmax_alloc);
        std::swap(ldv, aux.ldv);
        std::swap(V, aux.V);
        std::swap(hbar, aux.hbar);
        std::swap(hinv, aux.hinv);
        std::swap(coef, aux.coef);
        std::swap(dscratch, aux.dscratch);
        std::swap(hld, aux.hld);
        std::swap(basis_valid, aux.basis_valid);
        std::swap(ctrl, aux.ctrl);
        std::swap(h_ctrl, aux.h_ctrl);
    }
    cudaEvent_t get_event() {
        if (!event_pool.empty()) {
            cudaEvent_t e = event_pool.back();
            event_pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        cudaEventCreate(&e);
        return e;
    }
    // RAII-less helpers: begin returns an event recorded now; end records the
    // closing event and files the pair under `cls`
    cudaEvent_t prof_begin() {
        if (!profiling) return nullptr;
        cudaEvent_t e = get_event();
        cudaEventRecord(e, stream);
        return e;
    }
    void prof_end(int cls, cudaEvent_t b) {
        if (!profiling || !b) return;
        cudaEvent_t e = get_event();
        cudaEventRecord(e, stream);
        prof_events.push_back({cls, {b, e}});
    }
};


// internal (api.cu): x_next[idx] -> dev_out (the probe buffer when null) on the
// context stream without a host sync; the index list is re-uploaded when its
// length changes, or, with check, when its contents do
exg_status exg_gather_async(exg_ctx* c, const int* idx, int k, double* dev_out, bool check);
