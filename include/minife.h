/*
 * minife.h — C ABI of the B200-native MiniFE CG hot path (arxiv 1505.08023).
 *
 * The library assembles and solves the FE system of the paper's problem statement
 * (steady-state heat conduction on the unit cube, trilinear hex elements, u = 1 on
 * the plane x = 1 and u = 0 on the other faces) with unpreconditioned CG ("conjugate
 * gradient(CG) method without preprocessing"), entirely in hand-written sm_100a CUDA
 * kernels.  Citations: P:n = PAPER.md line n; S:n = SPEC.md line n; C0..C8 / G1..G20 =
 * readings in DESIGN.md §3.  SURVEY.md §8(b) is the contract this header implements.
 *
 * Conventions (all entry points):
 *   - Every int-returning call returns MINIFE_OK (0) or one of the MINIFE_E* codes below; the
 *     library never aborts and never prints.  minife_strerror() maps a code to a static
 *     string; minife_last_error() returns the ctx's last detailed message.
 *   - A minife_ctx is not thread-safe: drive it from one host thread.
 *   - Host pointers are caller-owned; the library never retains them past the call.
 *   - Device pointers (the *_device calls) are caller-owned device memory on the ctx's device.
 *   - Global node/row ids are x-fastest: id = ix + (nx+1)*(iy + (ny+1)*iz) (Fig 3.6).
 *   - All arithmetic is binary64, round-to-nearest-even, no FMA contraction, subnormals kept.
 */
#ifndef MINIFE_H
#define MINIFE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ---------------------------------------------------------------------- */
#define MINIFE_OK 0
#define MINIFE_EINVAL 1      /* invalid argument (bad size, NULL, buffer too small, ...) */
#define MINIFE_ESTATE 2      /* call not valid in the ctx's state (e.g. solve before assemble) */
#define MINIFE_ECUDA 3       /* a CUDA runtime call failed */
#define MINIFE_ENCCL 4       /* an NCCL call failed */
#define MINIFE_ENOMEM 5      /* device or host allocation failed */
#define MINIFE_ENOTSPD 6     /* CG met pAp < 0, or pAp == 0 with rr != 0 */
#define MINIFE_EDIVERGED 7   /* CG met a non-finite pAp or rr */
#define MINIFE_ENODEV 8      /* no CUDA device (or fewer than requested) */
#define MINIFE_ECOMM 9       /* device-initiated comm: a peer did not signal in time (dead or
                                hung rank, broken mapping); see option comm_timeout_ms     */

/* ---- context modes ---------------------------------------------------------------------- */
#define MINIFE_MODE_SINGLE 0   /* one process, one GPU, one part */
#define MINIFE_MODE_VIRTUAL 1  /* one process, one GPU, p RCB parts ("virtual ranks") */
#define MINIFE_MODE_MULTI 2    /* one process driving devices 0..ngpu-1.  With peer access
                                  between every device pair: device-initiated comm (halo
                                  pushed over NVLink by the p-update's sender, exact
                                  accumulators reduced in-kernel through peer stores + flags)
                                  and one CUDA graph per device; otherwise NCCL send/recv and
                                  all-reduce, enqueued directly */
#define MINIFE_MODE_RANK 3     /* SPMD: this process is rank r of w (torchrun).  Device comm
                                  over CUDA-IPC mappings exchanged at creation when every rank
                                  can map every other; otherwise NCCL (graph-captured) */

/* ---- matrix storage formats ---------------------------------------------- */
#define MINIFE_FMT_CRS 0       /* SELL-32, one int32 column per stored entry: the paper's CRS
                                  (Fig 3.1) on the GPU; 12 B per entry              */
#define MINIFE_FMT_SEG 1       /* SELL-32, 27 value slots per row + one int32 start column per
                                  x-run ("non-zero segment") + a 27-bit presence mask: the
                                  paper's BCRS (Fig 3.2) on the GPU; 8 B per entry
                                  + 4 B per segment.                                          */
#define MINIFE_FMT_SYM 2       /* MINIFE_FMT_SEG storing only the upper-triangle value slots
                                  (14 per row incl. the diagonal); a lower entry a_ij is read
                                  from row j's mirror slot (a_ij == a_ji bitwise: the assembled
                                  system is exactly symmetric, C2/C3).  Default.  With a halo
                                  the storage covers the extended box: halo nodes are ghost
                                  rows holding the mirrors.  Results identical to the others. */

/* ---- CG iteration schemes ------------------------------------------------- */
#define MINIFE_SCHEME_3K 0     /* per iteration: SpMV + pAp | r update + rr | x and p update   */
                               /* (x += alpha p with the p read for the p update).  Default. */
                               /* 12 nnz-class bytes + 80 B per row.  Parts whose vectors     */
                               /* exceed L2 apply the x update every 8th iteration (8 updates */
                               /* in order in one pass over a ring of 8 p buffers; same       */
                               /* arithmetic, 73 B/row).                                      */
#define MINIFE_SCHEME_FUSED 1  /* SURVEY §8(f) NEXT #2, one part + MINIFE_FMT_SEG only (other */
                               /* ctxs run 3K): the p update is formed at gather time inside  */
                               /* the SpMV and x is updated one iteration late there; a second */
                               /* kernel does r and rr.  72 B per row, 2 launches.            */

/* ---- halo transports of VIRTUAL ctxs ------------------------------------------------------ */
#define MINIFE_TRANSPORT_DIRECT 0  /* gather the owner's columns straight into the receiver's
                                      halo columns (one kernel per neighbor pair). Default.   */
#define MINIFE_TRANSPORT_WIRE 1    /* the RANK/MULTI wire protocol: pack the send lists, move
                                      each neighbor block into the receiver's contiguous
                                      receive buffer (device copies standing in for
                                      ncclSend/ncclRecv), unpack into the halo columns.       */
#define MINIFE_TRANSPORT_PUSH 2    /* one kernel per part stores p_(k+1) at every send slot
                                      straight into the receiver's halo column (reductions
                                      stay device-local sums).  MULTI ctxs with option
                                      device_comm = 0 use it over NVLink peer pointers.       */
#define MINIFE_TRANSPORT_DEVICE 3  /* the device-initiated protocol of MULTI/RANK ctxs on one GPU
                                      (DESIGN.md §7): every part pushes
                                      r_(k+1) at its send slots into the receivers' r-halo
                                      buffers right after the r update, the receivers complete
                                      p_(k+1)'s halo columns themselves; every part stores its
                                      exact accumulators into every part's inbox; release /
                                      acquire flags.  No host-launched collective.           */

typedef struct minife_ctx minife_ctx;

/* Per-part (per-rank) plan, host-computed from the RCB partition (G15). */
typedef struct minife_part_info {
    int32_t rank, world;
    int32_t box[6];           /* element box lo_x,lo_y,lo_z, hi_x,hi_y,hi_z (half-open)  */
    int32_t own[6];           /* owned node box lo_x,lo_y,lo_z, hi_x,hi_y,hi_z (inclusive) */
    int32_t n_neighbors;      /* ranks this part exchanges halo values with              */
    int32_t device;
    int64_t rows;             /* owned nodes = local rows (ascending global id)     */
    int64_t externals;        /* halo slots, ordered (owner rank, global id)       */
    int64_t nnz;              /* stored entries of the local rows (27-point pattern)      */
    int64_t slices;           /* SELL-32 slices = ceil(rows/32)                           */
    int64_t sell_entries;     /* sum over slices of 32*width (incl. padding)              */
    int64_t send_total;       /* values this part sends per halo exchange                 */
    int64_t interior_slices;  /* SELL-32 slices none of whose rows reads a halo column:
                                 their SpMV runs while the halo is in flight  */
} minife_part_info;

typedef struct minife_info {
    int32_t nx, ny, nz;       /* elements per axis (nodes = n+1, G1)                */
    int32_t mode;             /* MINIFE_MODE_*                                            */
    int32_t nparts;           /* parts held by THIS ctx (1 in SINGLE and RANK mode)       */
    int32_t rank, world;      /* RANK mode: this rank / world; otherwise 0 / nparts       */
    int32_t assembled;        /* 1 after a successful minife_assemble                     */
    int64_t rows, nnz;        /* GLOBAL counts: prod(N_a), prod(3N_a - 2) (§8(a))          */
    int64_t local_rows;       /* rows held by this ctx (all parts)                        */
    int64_t local_nnz;
    int64_t max_part_rows, max_part_nnz, max_part_externals;
    int64_t sell_entries;     /* held by this ctx                                         */
    int64_t device_bytes;     /* device memory held by this ctx                           */
    int32_t format;           /* MINIFE_FMT_*                                             */
    int32_t comm;             /* transport of the next solve: 0 none (one part) or device-
                                 local copies (VIRTUAL DIRECT/WIRE/PUSH), 1 NCCL, 2 device-
                                 initiated (peer/IPC stores + flags, or TRANSPORT_DEVICE)  */
    int64_t local_nns;        /* non-zero segments (x-runs) of the rows held here */
    int64_t kernel_launches;  /* kernels of this library launched by this ctx since creation
                                 (graph replays counted per kernel node; NCCL's own kernels
                                 and memset/copy nodes not included)                        */
} minife_info;

typedef struct minife_cg_result {
    int32_t status;           /* MINIFE_OK, MINIFE_ENOTSPD or MINIFE_EDIVERGED             */
    int32_t iterations;       /* completed CG iterations                                  */
    int32_t converged;        /* 1 iff a stop test fired (tol, rr == 0); 0 at the cap      */
    int32_t max_iters;
    double norm_b;            /* hist[0] = sqrt(dot(b,b))                                 */
    double final_rel_residual;/* hist[iterations] / hist[0] (0 if norm_b == 0)            */
    double seconds;           /* device time of the solve, CUDA events on the ctx stream  */
    double flops;             /* algorithmic: iterations * (2 nnz + 10 rows), global      */
    double bytes;             /* algorithmic HBM bytes of this ctx's kernels */
} minife_cg_result;

/* Per-kernel-class device times from minife_cg_profile (milliseconds, summed over launches). */
typedef struct minife_kernel_times {
    double spmv_ms;           /* K1: SpMV + pAp epilogue (a2)                             */
    double update_xr_ms;      /* K6: x/r update + rr (a3 finalise, a4)                    */
    double update_p_ms;       /* K7: p update (a5 finalise, a6)                           */
    double comm_ms;           /* halo + accumulator reductions (a1, a3/a5 all-reduce)     */
    int32_t spmv_launches, update_xr_launches, update_p_launches, iterations;
} minife_kernel_times;

/* ---- lifecycle ------------------------------------------------------------------------- */

/* Elements per axis nx,ny,nz >= 1 on the unit cube; ngpu >= 1 devices 0..ngpu-1
 * of this process.  ngpu == 1 -> MINIFE_MODE_SINGLE, ngpu > 1 -> MINIFE_MODE_MULTI (RCB over
 * ngpu parts, NCCL comms from ncclCommInitAll).  Computes the RCB plan and allocates every
 * device buffer.  *out is set only on success.
 * Errors: MINIFE_EINVAL (n < 1, ngpu < 1, out == NULL, RCB leaf without elements),
 * MINIFE_ENODEV (ngpu > visible devices), MINIFE_ENOMEM, MINIFE_ECUDA, MINIFE_ENCCL. */
int minife_create(int nx, int ny, int nz, int ngpu, minife_ctx **out);

/* p RCB parts ("virtual ranks") on device 0 of this process: the exact multi-rank data
 * layout, halo plans and reductions, with device-local copies as the transport.
 * Errors as minife_create. */
int minife_create_virtual(int nx, int ny, int nz, int nparts, minife_ctx **out);

/* SPMD: NCCL unique id (128 bytes) to broadcast from rank 0 to all ranks. */
int minife_nccl_unique_id(void *uid128);

/* SPMD: this process is `rank` of `world` and drives CUDA device `device`; uid128 is rank
 * 0's minife_nccl_unique_id.  Collective: every rank must call it.  Errors as
 * minife_create, plus MINIFE_EINVAL for rank/world out of range. */
int minife_create_rank(int nx, int ny, int nz, int rank, int world, int device,
                       const void *uid128, minife_ctx **out);

/* Frees every device/host resource and NCCL comm of the ctx.  NULL-safe. */
void minife_destroy(minife_ctx *ctx);

/* Run all subsequent device work of a SINGLE/RANK ctx on `stream` (a cudaStream_t, may be a
 * torch stream).  NULL restores the ctx's own stream.  Captured solve graphs stay valid: they
 * are captured on the ctx's own stream and launched on the selected one.
 * Errors: MINIFE_EINVAL (ctx NULL), MINIFE_ESTATE (mode VIRTUAL/MULTI). */
int minife_set_stream(minife_ctx *ctx, void *stream);

/* Per-ctx execution options (the library reads no environment variables for them).  Every
 * option selects between code paths that compute the SAME results bit for bit (C0-C6); they
 * exist for tests and A/B measurements.  -1 = automatic (the default where listed).
 *   "x_defer"         deferred x update over a ring of X p buffers: -1 auto (X = 8 where
 *                     the vectors exceed L2), 0 or 1 off, 2..8 force X
 *   "small_solver"    single-launch solvers for small one-part problems: -1 auto, 0 none
 *                     (multi-kernel graph), 1 one CTA (<= 2048 rows), 2 one 16-CTA cluster
 *                     (<= 8192 rows; only where such a cluster can be scheduled)
 *   "graph"           1 (default) replay one captured CUDA graph per solve, 0 enqueue directly
 *   "val_evict_first" SYM SpMV value stream L2 policy: -1 auto, 0 normal, 1 evict-first
 *   "x_prefetch"      SYM SpMV plane-ahead L2 prefetch of x: -1 auto, 0 off, 1 on
 *   "sym_kernel"      SYM SpMV: 1 (default) tensor-map mirror kernel, 0 L1-gather kernel
 *   "spmv_impl"       SEG/CRS SpMV: -1 auto, 1 TMA pipeline, 0 register streaming
 *   "x_late"          1 (default) K7 applies x += alpha p with the p it reads, 0 K6 does
 *   "cluster_dd"      cluster solver digit exchange: 1 (default) DSMEM pushes, 0 pulls
 *   "device_comm"     MULTI/RANK: -1 (default) device-initiated comm where it was set up at
 *                     creation, 0 NCCL transport; RANK at world 1: 1 forces the device
 *                     reduction kernels (self-exchange).  Set identically on every rank.
 *   "fold_comm"       device comm, SYM: 1 (default) the accumulator pushes ride in the last
 *                     CTA of the SpMV / r update / init kernels and the halo wait in the
 *                     last CTA of the p update (4 launches per iteration); 0 separate
 *                     k_acc_push / k_halo_wait launches (7)
 *   "band_rows"       SYM SpMV tile order, applied at the next minife_assemble: -1 (default)
 *                     band-major (y-bands of 65536 / N_x lines swept plane by plane) for
 *                     planes of more than 122880 rows (400^3), natural order otherwise;
 *                     0 natural order; n > 0 bands of n / N_x lines wherever planes exceed n
 *   "snake"           SYM SpMV: odd iterations visit the tiles last to first, so they start
 *                     on what the previous SpMV left in L2: -1 (default) auto (matrices of
 *                     48-400 MB), 0 off, 1 on
 *   "comm_timeout_ms" device comm: how long a kernel waits for a peer's flag before the
 *                     solve fails with MINIFE_ECOMM (default 60000)
 *   "comm_fault_part" fault injection for tests: the part / rank with this id never pushes
 *                     its accumulators or halo (device comm), so its peers time out into
 *                     MINIFE_ECOMM; -1 (default) off
 *   "symm_nw"         SYM SpMV tile width (consumer warps = 32-row slices per tile), applied
 *                     at the next minife_assemble: -1 (default) 11 where N_x >= 352 (a tile's
 *                     x lines then need the larger L1 of the narrower ring), 13 otherwise;
 *                     11 or 13 force it
 * A changed option drops the captured graph.  Errors: MINIFE_EINVAL (NULL, unknown name,
 * value out of range). */
int minife_set_option(minife_ctx *ctx, const char *name, int64_t value);

const char *minife_strerror(int status);
const char *minife_last_error(const minife_ctx *ctx);

/* ---- the hot path ---------------------------------------------------------------------- */

/* Select the storage format used by the next minife_assemble (default MINIFE_FMT_SYM).  The
 * ctx becomes unassembled.  Results are bit-identical in both formats (same values, same
 * summation order).  Errors: MINIFE_EINVAL (ctx NULL or unknown format). */
int minife_set_format(minife_ctx *ctx, int format);

/* VIRTUAL ctxs: select the halo transport (MINIFE_TRANSPORT_*), so the protocols of the
 * multi-GPU modes (NCCL wire protocol, device push, device-initiated reductions) run,
 * bit-exactly checkable, on one GPU.  Errors: MINIFE_EINVAL (NULL, unknown transport),
 * MINIFE_ESTATE (not a VIRTUAL ctx). */
int minife_set_transport(minife_ctx *ctx, int transport);

/* Select the CG iteration scheme of later solves (MINIFE_SCHEME_*).  Both schemes perform
 * C6's operations on the same values in the same order: results are bit-identical.
 * Errors: MINIFE_EINVAL (ctx NULL or unknown scheme). */
int minife_set_scheme(minife_ctx *ctx, int scheme);

/* Structure -> SELL-32 (a0.2), element operator (a0.3, C1), gather-assembly (a0.4, C2) and
 * Dirichlet elimination (a0.5, C3) on the device, for every part.  Idempotent.
 * Errors: MINIFE_EINVAL (ctx NULL), MINIFE_ECUDA. */
int minife_assemble(minife_ctx *ctx);

/* Unpreconditioned CG (C6): x0 = 0, r0 = b, p0 = r0; at most max_iters
 * iterations; stops when hist[k] <= tol*hist[0] or rr == 0.  tol == 0 runs exactly
 * max_iters (benchmark mode).  Dots are exactly rounded (C5), so the result is independent
 * of the partition and bit-identical to the oracle.  Execution: one CUDA graph per (ctx,
 * max_iters, tol) with three kernels per iteration; single-part SEG/SYM ctxs of <= 8192 rows
 * run the whole solve in one thread-block-cluster launch instead (same results).  Blocks
 * until the solve has finished.
 * `res` may be NULL.  Returns MINIFE_OK, MINIFE_ENOTSPD or MINIFE_EDIVERGED (also stored in
 * res->status); the cap reached is MINIFE_OK with converged = 0.
 * Errors: MINIFE_ESTATE (not assembled), MINIFE_EINVAL (max_iters < 1, tol < 0 or NaN),
 * MINIFE_ECUDA, MINIFE_ENCCL. */
int minife_cg_solve(minife_ctx *ctx, int max_iters, double tol, minife_cg_result *res);

/* Same iteration sequence as minife_cg_solve, launched without a graph and bracketed by CUDA
 * events per kernel class, to attribute device time (Fig 2.2 analogue).  Leaves the solution
 * state valid.  Errors as minife_cg_solve. */
int minife_cg_profile(minife_ctx *ctx, int max_iters, minife_kernel_times *out);

/* Timing window inside later minife_cg_solve calls: CUDA events (graph nodes) are recorded on
 * part 0's stream right before and after the SpMV launches of iterations first_iter ..
 * first_iter + n_iters - 1, so the dominant kernel is timed in the solve itself, not in a
 * separate profile run.  n_iters = 0 removes the window.  Rebuilds the solve graph.
 * Errors: MINIFE_EINVAL (NULL, first_iter < 1, n_iters < 0), MINIFE_ECUDA. */
int minife_set_timing_window(minife_ctx *ctx, int first_iter, int n_iters);

/* Averages over the window of the last solve: SpMV duration (start to end event of each
 * iteration's SpMV) and iteration period (start to start), milliseconds.
 * Errors: MINIFE_EINVAL (NULL), MINIFE_ESTATE (no window, or the last solve stopped before
 * its end), MINIFE_ECUDA. */
int minife_get_timing_window(minife_ctx *ctx, double *spmv_ms, double *iter_ms);

/* y = A x for the assembled, Dirichlet-imposed A (C4).  SINGLE/VIRTUAL/MULTI: x, y are host
 * arrays of `rows` doubles in global id order.  RANK: x, y hold this rank's owned rows in
 * ascending global id (minife_get_owned_ids); the halo is exchanged with the other ranks.
 * Errors: MINIFE_ESTATE (not assembled), MINIFE_EINVAL (NULL), MINIFE_ECUDA, MINIFE_ENCCL. */
int minife_spmv(minife_ctx *ctx, const double *x, double *y);

/* SINGLE only: y = A x on device arrays of `rows` doubles, launched on `stream` (NULL = the
 * ctx stream); asynchronous.  Errors: MINIFE_ESTATE (other modes, not assembled),
 * MINIFE_EINVAL (NULL pointers), MINIFE_ECUDA. */
int minife_spmv_device(minife_ctx *ctx, const double *d_x, double *d_y, void *stream);

/* ---- getters --------------------------------------------------------------------------- */

int minife_get_info(const minife_ctx *ctx, minife_info *out);

/* Device time (CUDA events on every part's queue, max over the ctx's parts, milliseconds) of
 * the last minife_assemble (0 for MINIFE_FMT_CRS, whose sizing pass syncs with the host) and
 * of the last minife_cg_solve.  Errors: MINIFE_EINVAL (NULL). */
int minife_get_timings(const minife_ctx *ctx, double *assemble_ms, double *solve_ms);
int minife_get_part_info(const minife_ctx *ctx, int part, minife_part_info *out);

/* Canonical global CSR of the assembled system (rows in global id order, columns ascending,
 * structural zeros kept): row_ptr[rows+1], col[nnz], val[nnz].  RANK mode: this rank's
 * owned rows only (row_ptr[local_rows+1]), global column ids.  Errors: MINIFE_ESTATE,
 * MINIFE_EINVAL, MINIFE_ECUDA. */
int minife_export_csr(minife_ctx *ctx, int64_t *row_ptr, int64_t *col, double *val);

/* Rows `gids[0..n)` of the assembled system (any size, for sampled parity): cols/vals are
 * n*27 arrays (row i at [27*i]), lens[i] = its length.  Rows not held by this ctx give
 * lens[i] = -1.  Errors: MINIFE_ESTATE, MINIFE_EINVAL, MINIFE_ECUDA. */
int minife_export_rows(minife_ctx *ctx, int64_t n, const int64_t *gids, int64_t *cols,
                       double *vals, int32_t *lens);

/* b, x (after cg_solve) in global id order (RANK: owned rows, ascending global id). */
int minife_get_rhs(minife_ctx *ctx, double *b);
int minife_get_solution(minife_ctx *ctx, double *x);

/* Residual-norm history hist[0..iterations] of the last solve (hist[0] = ||b||).  cap is the
 * capacity of h; *n receives iterations+1.  MINIFE_EINVAL if cap < iterations+1. */
int minife_get_history(minife_ctx *ctx, double *h, int cap, int *n);

/* RANK mode: global ids of this rank's owned rows, ascending (local_rows entries). */
int minife_get_owned_ids(const minife_ctx *ctx, int64_t *gids);

/* ---- host-only plan queries (no GPU needed) -------------------------------------------- */

/* RCB plan of part `rank` of `world` for an nx*ny*nz mesh (G15): fills `out` except nnz,
 * slices, sell_entries computed from closed forms.  Errors: MINIFE_EINVAL. */
int minife_plan(int nx, int ny, int nz, int world, int rank, minife_part_info *out);

/* The halo lists of that part: ext_gids[externals] in slot order; per neighbor (ascending
 * rank) nbr[k], recv_cnt[k], send_cnt[k]; send_idx[send_total] = local row indices to send,
 * concatenated by neighbor.  Any pointer may be NULL.  Errors: MINIFE_EINVAL. */
int minife_plan_lists(int nx, int ny, int nz, int world, int rank, int64_t *ext_gids,
                      int32_t *nbr, int64_t *recv_cnt, int64_t *send_cnt, int32_t *send_idx);

/* Roofline denominators measured on CUDA device `device` (SURVEY §8(d) B_read): best of
 * `reps` timed passes of a pure-read fp64 stream and of a copy (read + write bytes) over
 * buffers of `bytes` bytes (>= 8 GB recommended: far larger than L2).  Allocates and frees
 * its own buffers.  Errors: MINIFE_EINVAL (bytes < 1 MB, reps < 1, NULL), MINIFE_ENODEV,
 * MINIFE_ENOMEM, MINIFE_ECUDA. */
int minife_bandwidth_probe(int device, int64_t bytes, int reps, double *read_gbs,
                           double *copy_gbs);

/* L2-resident read rate (GB/s) of the bulk-copy engine measured by the last
 * minife_bandwidth_probe call on this process (48 MB buffer re-read); 0 before any probe. */
double minife_probe_l2_read_gbs(void);

/* Pure-write stream rate (GB/s, streaming stores over the probe's buffer) measured by the last
 * minife_bandwidth_probe call on this process: the roof of the assembly kernel, which writes
 * the matrix and reads nothing; 0 before any probe. */
double minife_probe_write_gbs(void);

/* ---- exact dot products (reading C5) --------------------------------------- */

#define MINIFE_ACC_WORDS 72    /* device superaccumulator: words 0..67 = signed int64 digits,
                                  word i weighs 2^(32 i - 1074); word 68 counts non-finite
                                  terms; 69..71 padding (576 B, the all-reduced payload)     */

/* Exactly rounded dot product of host vectors u, v (n doubles each) on CUDA device `device`:
 * RN(sum^exact fl(u_i v_i)), ties to even, exact zero -> +0.0, any non-finite product -> NaN.
 * This is the operation behind every CG dot of the hot path (Fig 2.2 "dot"), computed
 * by the same device code: per-thread TwoSum expansions, a CTA fixed-point superaccumulator,
 * global int64 words, warp-parallel carry normalisation and rounding.  The result does not
 * depend on the order of the terms.  Exact while every per-thread partial sum stays below
 * 2^1023 in magnitude (the expansions use binary64 TwoSum; the CG dots are orders of
 * magnitude below).  Allocates and frees its own device buffers; synchronous.
 * Errors: MINIFE_EINVAL (n < 0, n >= 2^29, out NULL, u/v NULL with n > 0), MINIFE_ENODEV,
 * MINIFE_ENOMEM, MINIFE_ECUDA. */
int minife_dot(int device, int64_t n, const double *u, const double *v, double *out);

/* The rounding step of minife_dot alone, on device `device`: *out = RN(sum_{i<68} words[i]
 * 2^(32 i - 1074)) for any MINIFE_ACC_WORDS signed int64 words (host array; word 68 != 0 ->
 * NaN; words 69..71 ignored); overflow rounds to +-inf.  Exposed so that tests can pin the
 * device's carry normalisation and round-to-nearest-even against exact integer arithmetic.
 * Errors: MINIFE_EINVAL (NULL), MINIFE_ENODEV, MINIFE_ENOMEM, MINIFE_ECUDA. */
int minife_exact_round(int device, const int64_t *words, double *out);

/* ---- verification and report data (rooted collectives) ---------------------------------- */

/* Verification of the last solve ("compare the FE solution with the analytical solution";
 * S:420-437; C8): for each of the n probe nodes gids[i] (global ids, identical on every rank),
 * u_fe[i] = x at the node and u_exact[i] = the separation-of-variables series of the unit-cube
 * problem with `nterms` odd terms per index (>= 151 recommended), evaluated on
 * the device of the part owning the node at the coordinates fl(i_a / n_a);
 * *max_abs_err = max_i |u_fe[i] - u_exact[i]|.  Only rank 0 needs these, so multi-GPU ctxs
 * combine them with ROOTED collectives (§3.2: "Allreduce -> Reduce"): ncclReduce(SUM)
 * of the per-rank probe arrays (each probe has one owner, zeros elsewhere: exact) and
 * ncclReduce(MAX) of the per-rank largest error, to rank 0.  Outputs are written on rank 0 (and
 * in one-process ctxs) only.  The series is deterministic but not bit-equal to a host libm
 * (verification data, compared within 1e-13).  Collective in RANK mode.
 * Errors: MINIFE_EINVAL (NULL, n < 0, a gid out of range, nterms < 1), MINIFE_ESTATE (no solve
 * yet), MINIFE_ECUDA, MINIFE_ENCCL. */
int minife_verify(minife_ctx *ctx, int64_t n, const int64_t *gids, int nterms, double *u_fe,
                  double *u_exact, double *max_abs_err);

/* Per-rank device times of the last minife_assemble and minife_cg_solve (ms):
 * per_rank[2r] = assembly, per_rank[2r+1] = solve of rank/part r (SPEC's per-phase report,
 * S:465-468).  RANK mode: a ROOTED gather ("Allgather -> Gather": each rank sends its two
 * numbers to rank 0 by ncclSend/ncclRecv); per_rank[2 world] is written on rank 0 only.
 * Other modes: one entry per part of the ctx.  Collective in RANK mode.
 * Errors: MINIFE_EINVAL, MINIFE_ECUDA, MINIFE_ENCCL. */
int minife_gather_times(minife_ctx *ctx, double *per_rank);

/* Library version string. */
const char *minife_version(void);

#ifdef __cplusplus
}
#endif
#endif
