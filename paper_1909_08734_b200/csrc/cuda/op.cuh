// Internal definitions of the device operator and preconditioner handles,
// shared by op.cu, pc.cu and krylov.cu.
#pragma once

#include "common.cuh"

#include <cstdint>
#include <vector>

/** Persistent Krylov workspace (allocated once per operator, reused by every
 *  solve: no cudaMalloc / cudaFree inside a timed solve). */
struct KrylovCache {
    std::vector<cpddg::DevBuf<double>> V;
    cpddg::DevBuf<double> w, r, tmp, yd, scal;
    cpddg::DevBuf<const double*> vptr;
    int vptr_valid = 0;  // entries of vptr that hold the current basis pointers
    double* host = nullptr;  // pinned scratch
    int host_cap = 0;
    cpddg::ReduceWork red;
    std::vector<cudaEvent_t> events;  // per-launch timing events (profile_kernels), created once
    // device-driven GMRES cycle: a CUDA graph whose while-node body is one
    // Arnoldi step (preconditioner, operator, MGS, Givens); rebuilt when the
    // preconditioner, the cycle length or the profiling mode changes
    cpddg::DevBuf<double> mgs_partials;  // per-pass block partials of the cooperative MGS
    int coop_grid = 0;
    cpddg::DevBuf<double> gstate;     // GState + H + cs + sn + g + est + stamps
    cpddg::DevBuf<double> vin;        // the step's preconditioner input (= V_m)
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t gexec = nullptr;
    cudaStream_t gstream = nullptr;   // capture stream
    const void* gpc = nullptr;
    int gcycle = -1, gprof = -1, gn = -1;
    std::vector<const void*> gsig;    // device addresses captured in the body
    double* ghost = nullptr;          // pinned copy of the state after a cycle
    std::size_t ghost_n = 0;
    ~KrylovCache() {
        if (host) cudaFreeHost(host);
        if (ghost) cudaFreeHost(ghost);
        for (auto e : events) cudaEventDestroy(e);
        if (gexec) cudaGraphExecDestroy(gexec);
        if (graph) cudaGraphDestroy(graph);
        if (gstream) cudaStreamDestroy(gstream);
    }
};

struct cpddg_op {
    int dim = 0, p = 0, na = 0, ng = 0, nlines = 0;
    double h = 0, c = 0, cg = 0, ih2 = 0;
    cpddg::DevBuf<double> t;    // [dim][N_B] stencil offsets g_a - base_a
    cpddg::DevBuf<int> lines;   // [(p+1)^(d-1)][N_B] first ordinal of each contiguous run
    cpddg::DevBuf<int> nbr;     // [2d][N_A] band codes of the axis neighbours
    cpddg::DevBuf<int> nbr_aos; // [N_A][2d] the same, node-major (k_helm_pdl)
    cpddg::DevBuf<double> v;    // [N_B] extension values E x
    // staged extension (d = 3, p = 3): tiles of <= kExtTile consecutive band
    // nodes; each tile stages the x entries its stencils touch into shared
    // memory and addresses them with 16-bit tile-local run starts.
    int ext_tiles = 0, ext_smem = 0;                // 0 tiles: gather kernel
    cpddg::DevBuf<std::uint16_t> lines16;          // [16][N_B] run start in the tile's stage
    cpddg::DevBuf<int> tile_k0;                     // [tiles+1] first slot of each tile
    cpddg::DevBuf<int> ext_perm;                    // [N_B] band node computed by each tile slot
    cpddg::DevBuf<double> ext_t;                    // [d][N_B] stencil offsets in slot order
    cpddg::DevBuf<int> stage_base;                  // [tiles+1] first entry of each tile's stage list
    cpddg::DevBuf<int> stage_idx;                   // stage list: active ordinal of each staged x
    // grouped extension (d = 3, p = 3, the default): band nodes sorted by
    // stencil base, two of one base per thread (slots 2 th, 2 th + 1)
    int grp_chunks = 0, grp_slots = 0, grp_grid = 0;  // chunks of kGrpThreads threads (idle slots padded)
    cpddg::DevBuf<double> grp_t;                    // [d][slots] stencil offsets in slot order
    cpddg::DevBuf<unsigned char> grp_slot;          // [threads] base of each thread within its chunk
    cpddg::DevBuf<int> grp_perm;                    // [slots] band code of each slot, -1 idle
    cpddg::DevBuf<int> grp_lines;                   // [chunks][kGrpMax][16] run starts of the chunk's bases, -1 unused
    // union stage (k_extend_union, the default): same slots, per chunk the sorted
    // union of its bases' x runs and each base's 16 run offsets into it
    bool uni = false;
    cpddg::DevBuf<int> uni_stage;                   // [chunks][kUnionMax] active ordinals, -1 unused
    cpddg::DevBuf<unsigned short> uni_roff;         // [chunks][kGrpMax][16] run offsets in the stage
    // the tables and v of the default kernels packed into one allocation, kept resident in a
    // persisting L2 carve-out (access-policy window on the operator launches): inside a solve every
    // preconditioner apply streams GBs and every MGS step hundreds of MB through L2 between two
    // operator applies
    cpddg::DevBuf<char> slab;
    std::size_t l2_window = 0;  // bytes of the window (0: no window)
    cpddg::DevBuf<double> rn2;  // scalar slot for ||b - A x||^2
    cpddg::ReduceWork red;
    std::int64_t alg_bytes = 0, streamed_bytes = 0;
    KrylovCache kc;
};

/** Envelope (profile) LU factors of every subdomain system, batched. */
struct cpddg_pc {
    int n_global = 0, n_sub = 0, max_rows = 0;
    int n_reduced = 0, n_pivoted = 0;  // Dirichlet-reduced / host-pivoted local systems
    std::int64_t n_dropped = 0;        // local unknowns nothing depends on, removed before the analysis
    std::int64_t rows_total = 0, entries = 0;
    // per subdomain (device)
    cpddg::DevBuf<int> n_rows;         // [n_sub]
    cpddg::DevBuf<std::int64_t> vbase; // [n_sub] first row in the concatenated per-row arrays
    cpddg::DevBuf<std::int64_t> ebase; // [n_sub] first entry in the concatenated L / U arrays
    cpddg::DevBuf<int> order;          // [n_sub] launch order (largest first)
    // per row (device, concatenated over subdomains, in factor order)
    cpddg::DevBuf<int> first;          // L row i: envelope start column fL_i (local index)
    cpddg::DevBuf<std::int64_t> roff;  // offset of row i inside its subdomain's L array
    cpddg::DevBuf<std::int64_t> ebaseU; // [n_sub] first entry of each subdomain in U (column storage)
    cpddg::DevBuf<int> firstU;         // U column i: first stored row fU_i
    cpddg::DevBuf<std::int64_t> roffU; // offset of column i inside its subdomain's U array
    cpddg::DevBuf<int> rlast;          // largest row whose envelope starts at or before i
    cpddg::DevBuf<int> gidx;           // global index gathered into row i (R_j), or -1
    cpddg::DevBuf<int> sidx;           // global index row i scatters to (owned), or -1
    cpddg::DevBuf<double> diag;        // U_ii
    cpddg::DevBuf<double> dinv;        // 1 / U_ii (the solve multiplies)
    // per envelope entry
    cpddg::DevBuf<double> L;           // L_ij, j in [f_i, i), row-contiguous
    cpddg::DevBuf<double> U;           // factorisation: U_ji (column i of U) over [f_i, i);
                                       // solve: reversed rows of U (see k_reverse_u)
    // reversed-U tables for the backward solve
    cpddg::DevBuf<std::int64_t> ubase; // [n_sub] first entry of each subdomain in U
    cpddg::DevBuf<int> ufirst;         // per reversed row: first reversed column
    cpddg::DevBuf<std::int64_t> uroff; // per reversed row: offset inside the subdomain's U
    cpddg::DevBuf<double> drev;        // diagonal in reversed order
    std::int64_t u_entries = 0, profile_entries = 0;
    std::int64_t factor_bytes = 0, alg_bytes = 0;
    double factor_seconds = 0, analyse_seconds = 0, max_probe_residual = -1;
    int solve_smem = 0;
    int bwd_prefetch = 1;  // backward L2 prefetch distance in blocks (0 = off)
    bool urows = true;     // backward layout: reversed U rows (true) or U columns (false)
    int shape = 1;         // solve block shape: 0 big (1 CTA/SM), 1 mid (2/SM), 2 small (4/SM)
    // record solve (default with urows): per block [W | T^-1] records, rows
    // compacted to their far parts (k_block_records, k_compact_rows)
    bool blockinv = false;
    std::int64_t rec_entries = 0, far_entries = 0;
    cpddg::DevBuf<std::int64_t> rbase; // [n_sub] first record entry of each subdomain
    cpddg::DevBuf<double> recL, recU;
    // persistent TMA-streamed solve (k_solve_tma): per-CTA subdomain lists,
    // per-step items (32 B each) and row descriptors
    bool tma = false;
    int tma_grid = 0, tma_smem = 0;
    cpddg::DevBuf<int> tma_cta_begin, tma_cta_subs, tma_desc;
    cpddg::DevBuf<std::int64_t> tma_itbase;
    cpddg::DevBuf<unsigned char> tma_items;
    // persistent windowed streamed solve (k_solve_win, the default): per-CTA
    // subdomain lists, per-step items, descriptors (2 RB ints per step) and the
    // per-row buffer ybuf (R_j r in, solution out)
    bool win = false, win_gy = false;
    int win_rb = 16, win_grid = 0, win_smem = 0, win_wmask = 0, win_dback = 0, win_ring = 0;
    int win_reach_l = 0, win_reach_u = 0;
    cpddg::DevBuf<int> win_cta_begin, win_cta_subs, win_desc;  // whole-subdomain segment lists (LPT)
    cpddg::DevBuf<int> win_bal_begin, win_bal_segs, win_hand_flag;  // balanced lists: subdomains cut once
    cpddg::DevBuf<double> win_hand_buf;
    int win_hand_stride = 0, win_cuts = 0;
    double win_lpt_eff = 0.0, win_bal_eff = 0.0;  // modelled load / (grid * makespan)
    cpddg::DevBuf<std::int64_t> win_itbase;
    cpddg::DevBuf<unsigned char> win_items;
    cpddg::DevBuf<double> ybuf;
    // small systems: dense local inverses (k_solve_dense), row-major in factor order
    bool dense = false, dense_probe = false;
    int dense_tiles = 0;
    std::int64_t dense_entries = 0;
    cpddg::DevBuf<double> Ainv;
    cpddg::DevBuf<std::int64_t> dense_base;
    cpddg::DevBuf<int> dense_tile_sub, dense_tile_row0;
};

namespace cpddg {
/** y = A x.  pdl: launch the Helmholtz kernel as a programmatic dependent
 *  of the extension (off inside captured graphs). */
void op_apply(const cpddg_op* op, const double* x, double* y, cudaStream_t st, bool pdl = true);
/** r = b - A x and ||r||^2 into *rn2_dev (device scalar). */
void op_residual(const cpddg_op* op, const double* b, const double* x, double* r, double* rn2_dev,
                 cudaStream_t st);
/** z = M r (accumulate = false) or z += M r (accumulate = true: the owned
 *  slots are disjoint, so this is accumulate_correction of
 *  transmission.hpp:66-69 applied for every subdomain). */
void pc_apply(const cpddg_pc* pc, const double* r, double* z, bool accumulate, cudaStream_t st);
}  // namespace cpddg
