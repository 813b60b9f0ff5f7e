/*
 * minife_oracle.h — CPU ORACLE for the MiniFE CG hot path (arxiv 1505.08023).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_1505_08023_b200/) never includes, links or calls anything in oracle/.
 *
 * Plain, slow, single-threaded, binary64 (no FMA contraction: built with
 * -O2 -ffp-contract=off, no -ffast-math).  Every function cites the passage it
 * follows:  P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n,
 * C0..C8 = the canonical-arithmetic readings written down in DESIGN.md §3.
 *
 * Pins (what fixes each function without trusting it) live in tests/test_oracle_*.py.
 * Functions with no independent pin say "parity unpinned" here and in DESIGN.md:
 * none at present.
 */
#ifndef MINIFE_ORACLE_H
#define MINIFE_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (same numeric meaning as the product's minife.h, defined independently) */
#define OR_OK 0
#define OR_EINVAL 1
#define OR_ENOTSPD 6
#define OR_EDIVERGED 7

/* Fig 3.6 get_id / S:52-60: x-fastest id, -1 for any per-axis out-of-range index (G3). */
int64_t or_node_id(int64_t nnx, int64_t nny, int64_t nnz, int64_t ix, int64_t iy, int64_t iz);

/* C1 / P:31: 8x8 element diffusion matrix of an axis-aligned hex with edges
 * (hx,hy,hz); local node order x-fastest ((0,0,0),(1,0,0),(0,1,0),...), row-major K[8*a+b]. */
void or_element_matrix(double hx, double hy, double hz, double K[64]);

/* Fig 3.6 / S:199-207: number of stored entries of the global 27-point pattern (p = 1). */
int64_t or_structure_nnz(int nx, int ny, int nz);

/* Fig 3.6 / S:199-207: global CRS pattern, rows in global id order, cols ascending.
 * row_ptr[rows+1], col[nnz] caller-allocated. */
int or_structure(int nx, int ny, int nz, int64_t *row_ptr, int64_t *col);

/* Fig 3.7 / P:251-262, C2: element loop in ascending element id, scatter-add of
 * each element's 8x8 matrix and (zero) 8-vector into val (zeroed first) and b (zeroed). */
int or_assemble(int nx, int ny, int nz, const int64_t *row_ptr, const int64_t *col,
                double *val, double *b);

/* P:36, C3: symmetric Dirichlet elimination keeping the pattern. */
int or_impose_dirichlet(int nx, int ny, int nz, const int64_t *row_ptr, const int64_t *col,
                        double *val, double *b);

/* One row of the assembled + Dirichlet-imposed global system, computed from scratch by
 * running C2's element loop and C3's elimination restricted to that row (for sampled parity
 * at sizes where the whole oracle matrix does not fit).  cols/vals >= 27 entries.
 * Returns the row length, b_row receives b[gid]. */
int or_row(int nx, int ny, int nz, int64_t gid, int64_t *cols, double *vals, double *b_row);

/* Fig 3.1 / P:93-103, C4: y_i = left fold s = +0.0; s = fl(s + fl(a*x_col)) in stored order. */
void or_spmv(int64_t m, const int64_t *row_ptr, const int64_t *col, const double *val,
             const double *x, double *y);

/* C5: RN( exact sum_i fl(u_i*v_i) ), ties-to-even; NaN if any product is non-finite. */
double or_dot(int64_t n, const double *u, const double *v);

/* C6 / S:381-389: unpreconditioned CG, x0 = 0, on any CSR matrix.  hist[max_iters+1].
 * Returns OR_OK, OR_ENOTSPD or OR_EDIVERGED; *iters = completed iterations,
 * *converged = 1 iff a stop test fired.  tol = 0 runs exactly max_iters (unless rr hits 0). */
int or_cg(int64_t m, const int64_t *row_ptr, const int64_t *col, const double *val,
          const double *b, int max_iters, double tol, double *x, double *hist,
          int *iters, int *converged);

/* C8 / S:420-428: separation-of-variables series, `nterms` odd terms per index. */
double or_analytic(double x, double y, double z, int nterms);

/* G15 / S:61-69: RCB of the element box over p ranks.  boxes[6*r..] = lo_x,lo_y,lo_z,
 * hi_x,hi_y,hi_z (half-open element ranges).  Returns OR_EINVAL if p < 1 or a leaf
 * would receive fewer elements than ranks. */
int or_rcb(int nx, int ny, int nz, int p, int *boxes);

/* owner of node (ix,iy,iz) = lowest rank whose closed node box contains it. */
int or_owner(int p, const int *boxes, int ix, int iy, int iz);

/* externals of `rank` ordered by (owner rank, global id), by brute-force
 * stencil enumeration over every owned node.  Returns the count; out may be NULL. */
int64_t or_externals(int nx, int ny, int nz, int p, const int *boxes, int rank, int64_t *out);

/* owned nodes of `rank` in ascending global id.  Returns count; out may be NULL. */
int64_t or_owned(int nx, int ny, int nz, int p, const int *boxes, int rank, int64_t *out);

#ifdef __cplusplus
}
#endif
#endif
