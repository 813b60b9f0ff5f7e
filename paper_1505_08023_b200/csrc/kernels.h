// kernels.h — host-side launch wrappers of the sm_100a kernels (kernels.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace minife {

// Storage formats of the assembled matrix.
//   FMT_CRS: SELL-32 with one int32 column per stored entry — the GPU form of the paper's CRS
//            (Fig 3.1).
//   FMT_SEG: SELL-32 with 27 value slots per row (stencil order), one int32 column per x-run
//            ("non-zero segment") and a 27-bit presence mask — the GPU form of the paper's
//            BCRS (Fig 3.2): "jas" = run start, the mask replaces "offsets".
//   FMT_SYM: FMT_SEG with only the upper-triangle value slots stored (14 per row, stencil
//            slots 13..26 incl. the diagonal); a lower entry a_ij (j < i) is read from row j's
//            mirror slot, a_ij == a_ji exactly (the assembled system is bitwise symmetric,
//            pinned by the oracle tests).  One part only (rows == columns).
enum { FMT_CRS = 0, FMT_SEG = 1, FMT_SYM = 2 };

// Device-resident CG scalars of one part (C6).  Written only by CTA 0 of the kernel that
// takes the decision; every CTA computes the same decision from the same exact values.
struct CgState {
    int done;          // a stop test fired (later kernels return immediately)
    int status;        // 0 OK, 6 NOT-SPD, 7 DIVERGED
    int iters;         // completed iterations
    int converged;
    double stop;       // fl(tol * hist[0])
    double pAp, alpha, beta;
    int alpha_iter;    // fused scheme: iteration whose alpha is in `alpha`
    int x_done;        // fused scheme: last iteration whose x update has been applied
};

// Row -> column map: rows are the owned box, columns the extended box (plan.h).
struct Geom {
    int nx, ny, nz;                     // global elements per axis
    int own_lo[3];
    int own_n[3];
    int ext_lo[3];
    int ext_n[3];
    int off[3];                         // own_lo - ext_lo
    int64_t rows, ncols;
    int ident;                          // extended box == owned box (one part)
    // u / ext_n[a] for u < 2^31 as __umul64hi(u, ext_mag[a]), ext_mag[a] = ceil(2^64 / ext_n[a])
    // (exact: the error u / 2^64 stays below 1 / ext_n[a])
    uint64_t ext_mag[2];
};

struct Matrix {
    int fmt;
    int64_t rows, nslices;
    const double *val;                  // CRS: [slice_off[s] + 32k + lane]; SEG: [(27s + t)32 + lane]
                                        // SYM: [(14s + t - 13)32 + lane], t >= 13
    const int64_t *slice_off;           // CRS only [nslices+1]
    const uint8_t *row_len;             // CRS only [rows]
    const int32_t *col;                 // CRS only
    const int32_t *seg;                 // SEG/SYM: [(9s + j)32 + lane], start column of run j
    const uint32_t *mask;               // SEG/SYM: [32 slices], bit t = slot t present
    // SEG, multi-part: slices are STORED interior-first.  slice_row[q] = row
    // slice held at storage position q, slice_pos = its inverse; null = identity.  val, seg
    // and mask are indexed by storage position, vectors by row.
    const int32_t *slice_row;
    const int32_t *slice_pos;
    // SYM on a part with a halo (ext = 1): storage covers the EXTENDED box (rows = its ncols
    // nodes, in column order), so every mirror row is local; halo nodes are ghost rows whose
    // upper slots are stored but never computed.  mask bit 31 = owned node (computed row).
    int ext;
};

// SYM-ext: mask bit of an owned (computed) row
constexpr unsigned SYM_OWNED = 1u << 31;

struct AsmArgs {
    Geom g;
    int fmt;
    const int64_t *slice_off;           // CRS
    uint8_t *row_len;                   // CRS
    int32_t *col;                       // CRS
    int32_t *seg;                       // SEG / SYM
    uint32_t *mask;                     // SEG / SYM
    double *val;
    double *b;                          // [rows]
    const int32_t *slice_pos;           // SEG: row slice -> storage position (null: identity)
};

// Device-initiated communication between parts/ranks:
// every part owns one COMM REGION in its device memory; the other parts store into it
// directly (same device: VIRTUAL; peer access over NVLink: MULTI; CUDA-IPC mappings: RANK)
// and raise release flags; the owner waits with acquire loads.  No host-launched collective
// remains in the CG iteration.  Region layout (64-bit words, W = world):
//   [0] solve generation (bumped by k_init_vectors), [1] k_push CTA ticket, [2] error flag
//   [COMM_HDR + (4 gp + 2 .. ) ...] acc flags [gen parity 2][which 2][sender W]
//   [COMM_HDR + 4W + sender]       halo flags
//   [comm_inbox(W) + ((2 gp + which) W + sender) ACC_WORDS + i]  accumulator inbox
// A flag holds seq = gen * 2^21 + (2k + which) (acc) or gen * 2^21 + k (halo of p_k).
constexpr int COMM_HDR = 8;
__host__ __device__ constexpr int64_t comm_acc_flag(int W, int gp, int which, int sender) {
    return COMM_HDR + (int64_t)((2 * gp + which) * W + sender);
}
__host__ __device__ constexpr int64_t comm_halo_flag(int W, int sender) {
    return COMM_HDR + 4 * (int64_t)W + sender;
}
__host__ __device__ constexpr int64_t comm_inbox(int W) {
    return ((COMM_HDR + 5 * (int64_t)W) + 15) / 16 * 16;
}
__host__ __device__ constexpr int64_t comm_words(int W) {
    return comm_inbox(W) + 4 * (int64_t)W * 72;
}
__host__ __device__ constexpr unsigned long long comm_seq(unsigned long long gen, int k, int which) {
    return (gen << 21) + 2ull * (unsigned)k + (unsigned)which;
}
__host__ __device__ constexpr unsigned long long comm_halo_seq(unsigned long long gen, int k) {
    return (gen << 21) + (unsigned)k;
}

struct DevComm {
    unsigned long long *const *region;  // [world] regions as seen from this device (own incl.)
    unsigned long long *local;          // this part's region; null: accumulators all-reduced
                                        // by the host-launched transport instead
    const int32_t *nbr_rank;            // [n_nbr] neighbor ranks (halo signals / waits)
    int n_nbr;
    int rank, world;
    long long timeout_ns;               // spin limit; exceeded -> CgState.status = 9 (ECOMM)
    int mute;                           // fault injection (tests): this part never pushes
};

struct SpmvArgs {
    Matrix m;
    Geom g;
    int64_t s_begin, s_end;             // storage slices [s_begin, s_end) (SEG/CRS kernels)
    int val_evict_first;                // SYMM: stream the values evict-first in L2
    int x_prefetch;                     // SYMM: warm L2 with each tile's plane-ahead x
    int sym_kernel;                     // SYM: 1 tensor-map mirror kernel, 0 L1-gather kernel
    int symm_nw;                        // SYM tensor-map kernel tile width: SYMM_NW(_WIDE)
    const int32_t *tile_order;          // SYMM: tile visited at position tau (null: tau itself)
    int reverse;                        // SYMM: visit the positions last to first
    int impl;                           // SEG/CRS: -1 default, 1 TMA pipeline, 0 registers
    const double *x;                    // [ncols], extended-box order
    double *y;                          // [rows]
    unsigned long long *acc;            // pAp accumulator (DOT only)
    unsigned long long *acc_zero;       // accumulator to clear (CTA 0), may be null
    const CgState *st;                  // early exit when st->done (may be null)
    // fused CG iteration (one part, SEG format): the SpMV operand is
    // p_k = r + beta_{k-1} p_{k-1} formed at gather time (p_1 = r), written to p_new for the
    // own rows, and x += alpha_{k-1} p_{k-1} is applied for the own rows.
    int fused_k;                        // 0: plain SpMV; k >= 1: fused iteration k
    const double *r, *p_old;
    double *p_new, *xsol;
    unsigned long long *acc_rr_in;      // rr_{k-1} accumulator (k >= 2)
    double *hist, *rr;
    CgState *stw;                       // writable state (decisions)
    // device comm (DevComm): fold_push = 1 -> the last CTA pushes the pAp accumulator of
    // iteration k to every rank's inbox (SYM kernels), instead of a k_acc_push launch
    DevComm dc;
    int fold_push, k;
};

struct UpdArgs {
    Geom g;
    double *x, *r;                      // [rows]
    double *p;                          // [ncols], extended-box order
    const double *Ap;                   // [rows]
    const double *b;                    // [rows]
    unsigned long long *acc_in;         // finalised at kernel start
    unsigned long long *acc_out;        // accumulated by this kernel
    unsigned long long *acc_zero;       // cleared by CTA 0 (may be null)
    double *hist, *rr;                  // [max_iters+1]
    CgState *st;
    double *alpha_hist;                 // [max_iters+1]: alpha_k recorded by K6 (may be null)
    // deferred x (launch_update_p2 / launch_x2_finish): ring of xdef p buffers, p_k in
    // ring[(k-1) % xdef]
    const double *ring[8];
    int xdef;
    int x_late;                         // K7 applies x += alpha p (1, default) or K6 does (0)
    DevComm dc;                         // device-initiated reductions / halo (dc.local != null)
    int fold_push;                      // K6 / init: the last CTA pushes the rr accumulator
    // device comm, halo by r: K7 completes the halo columns itself,
    // p_(kp)[c] = fl(rhalo[h] + fl(beta p_(kp-1)[c])), c = halo_col[h], once the neighbours'
    // pushes of r_(kp) at their send slots have landed in rhalo (halo_n = 0: off)
    const double *rhalo;
    const int32_t *halo_col;
    int64_t halo_n;
    int halo_kp;
    int cl_dd;                          // cluster solver: DSMEM digit pushes (1, default)
};
constexpr int XDEF_MAX = 8;

// Setup (a0.2-a0.5)
cudaError_t launch_rowlen_widths(const Geom &g, uint8_t *row_len, uint8_t *width,
                                 int64_t nslices, cudaStream_t s);
cudaError_t launch_assemble(const AsmArgs &a, cudaStream_t s);

// Hot path
cudaError_t launch_spmv(const SpmvArgs &a, bool with_dot, int grid, cudaStream_t s);
cudaError_t launch_init_vectors(const UpdArgs &a, int grid, cudaStream_t s);
cudaError_t launch_init_finalize(const UpdArgs &a, double tol, cudaStream_t s);
cudaError_t launch_update_xr(const UpdArgs &a, int k, int grid, cudaStream_t s);
cudaError_t launch_update_p(const UpdArgs &a, int k, int grid, cudaStream_t s);
// x every second iteration (one part): K7 of iteration k with p_k in pk and p_(k-1) in po;
// writes p_(k+1) into po; even k: x += alpha_(k-1) p_(k-1), then += alpha_k p_k (odd k: only
// on a stop).  x2_finish applies an x update still pending after the loop.
cudaError_t launch_update_p2(const UpdArgs &a, int k, const double *pk, double *po, int grid,
                             cudaStream_t s);
cudaError_t launch_x2_finish(const UpdArgs &a, cudaStream_t s);
// fused scheme: K6' (alpha_k; r -= alpha Ap; exact rr) and the finish kernel (rr_K, pending x)
cudaError_t launch_update_r(const UpdArgs &a, int k, unsigned long long *acc_pAp_next_zero,
                            int grid, cudaStream_t s);
cudaError_t launch_cg_finish(const UpdArgs &a, int K, const double *p_even, const double *p_odd,
                             int grid, cudaStream_t s);

// Whole CG solve (init + up to K iterations, C6) in one CTA: one part, FMT_SEG or FMT_SYM,
// rows <= SMALL_MAX_ROWS.  Same state, history and vectors as the multi-kernel sequence.
constexpr int SMALL_THREADS = 1024, SMALL_RPT = 2, SMALL_MAX_ROWS = SMALL_THREADS * SMALL_RPT;
cudaError_t launch_cg_small(const Matrix &m, const UpdArgs &a, int K, double tol,
                            cudaStream_t s);

// Whole CG solve in ONE thread-block cluster of CL_CTAS CTAs (DSMEM): one part, FMT_SEG or
// FMT_SYM, rows <= CL_MAX_ROWS and ceil(slices / CL_CTAS) <= CL_MAX_SL.
constexpr int CL_CTAS = 16, CL_THREADS = 256, CL_WARPS = CL_THREADS / 32, CL_MAX_SL = 16,
              CL_RPT = CL_MAX_SL / CL_WARPS, CL_MAX_ROWS = CL_CTAS * CL_MAX_SL * 32;
cudaError_t launch_cg_cluster(const Matrix &m, const UpdArgs &a, int K, double tol,
                              cudaStream_t s);
bool cluster_solver_available();     // a CL_CTAS-CTA cluster fits this device (once per device)

// SYM with a halo: sendbuf[i] = r[send_row[i]] + beta_k p[send_col[i]] (p_(k+1) at the send
// list, ahead of K7), beta_k from the rr accumulator a.acc_in and a.rr[k-1].
cudaError_t launch_pack_next_p(const UpdArgs &a, int k, const int32_t *send_row,
                               const int32_t *send_col, double *sendbuf, int64_t n,
                               cudaStream_t s);

// Halo by r (device comm): dst_ptr[slot_nbr[i]][dst_slot[i]] = r[send_row[i]] (r_(kp) at the
// send slots, into the receivers' r-halo buffers), then the last CTA raises each neighbour's
// halo flag for kp.  Needs no reduction result: it runs right after K6.
cudaError_t launch_push_r(const UpdArgs &a, int kp, const int32_t *send_row,
                          const uint8_t *slot_nbr, const int32_t *dst_slot,
                          double *const *dst_ptr, int64_t n, cudaStream_t s);
// p_1's halo columns = the r_0 (= b) halo the neighbours pushed (after their flags for kp = 1)
cudaError_t launch_halo_init(const UpdArgs &a, cudaStream_t s);

// Halo push (a1, device-initiated): dst_ptr[slot_nbr[i]][dst_col[i]] = value of slot i, with
// value = p[send_col[i]] (mode 0) or r[send_row[i]] + beta_k p[send_col[i]] (mode 1).
cudaError_t launch_push(const UpdArgs &a, int k, int mode, const int32_t *send_row,
                        const int32_t *send_col, const uint8_t *slot_nbr, const int32_t *dst_col,
                        double *const *dst_ptr, int64_t n, cudaStream_t s);

// Device-initiated comm (dc.local != null): store this part's accumulator `acc` (reduction
// `which` of iteration k: 0 pAp_k, 1 rr_k) into every rank's inbox and raise the flags.
cudaError_t launch_acc_push(const UpdArgs &a, int k, int which, const unsigned long long *acc,
                            cudaStream_t s);

// Halo (a1): dst[didx ? didx[i] : i] = src[sidx ? sidx[i] : i], i < n
cudaError_t launch_move(const double *src, const int32_t *sidx, double *dst,
                        const int32_t *didx, int64_t n, cudaStream_t s);
cudaError_t launch_vsum(unsigned long long *const *accs, int nparts, cudaStream_t s);

// C5 standalone: acc (ACC_WORDS words, zeroed by the caller) += exact sum of fl(u_i v_i);
// *out = RN(acc) (warp-parallel carry normalisation + rounding, exact.cuh).
cudaError_t launch_dot(const double *u, const double *v, int64_t n, unsigned long long *acc,
                       cudaStream_t s);
cudaError_t launch_acc_round(const unsigned long long *acc, double *out, cudaStream_t s);

// Verification (C8): for probe q < n (a node owned by this part: local_row[q], mesh
// indices ijk[3q..3q+2]) out[2 slot[q]] = x[local_row[q]], out[2 slot[q] + 1] = the analytic
// series with nterms odd terms per index at the node.  One CTA per probe.
cudaError_t launch_verify(const double *x, int nx, int ny, int nz, const int64_t *local_row,
                          const int32_t *ijk, const int32_t *slot, int n, int nterms,
                          double *out, cudaStream_t s);

// Parity helper: rows[] (local) -> up to 27 (extended column, value) pairs each
cudaError_t launch_extract_rows(const Matrix &m, const Geom &g, const int64_t *rows, int64_t n,
                                int32_t *out_col, double *out_val, int32_t *out_len,
                                cudaStream_t s);

// Roofline probes on the current device: best-of-reps pure-read and copy bandwidth (GB/s,
// copy counts read + write bytes) over `bytes`-sized buffers.
cudaError_t probe_bandwidth(int64_t bytes, int reps, double *read_gbs, double *copy_gbs);

// occupancy-derived grid sizes
int spmv_grid(int64_t nslices, int fmt);
int stream_grid(int64_t rows);

// SYMM kernel tile: NW slices of 32 rows, one consumer warp each (the unit of
// SpmvArgs::tile_order).  13 by default; 11 where a tile's nine x lines (9 N_x doubles) exceed
// the ~28 KB of L1 left beside the 13-wide ring (226 KB of shared memory): the 11-wide ring
// (189 KB) fits the 196 KB carveout and leaves ~60 KB of L1 (B200, per solve: 400^3 -2.1 %;
// 300^3 +2 %, 100^3 +1.5 % -- there the x lines fit anyway and 13 warps hide more latency;
// profiles/r02/ab/symm_nw_wide.jsonl)
constexpr int SYMM_NW = 13, SYMM_NW_WIDE = 11;
constexpr int64_t SYMM_WIDE_N0 = 352;
static inline int symm_nw_auto(int64_t n0) { return n0 >= SYMM_WIDE_N0 ? SYMM_NW_WIDE : SYMM_NW; }

constexpr int SPMV_THREADS = 256;
constexpr int UPD_THREADS = 256;

}  // namespace minife
