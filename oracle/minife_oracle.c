/*
 * minife_oracle.c — CPU ORACLE for the MiniFE CG hot path (arxiv 1505.08023).
 *
 * TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs, never by the product (paper_1505_08023_b200/).
 * It shares no code, header, table or constant generator with the CUDA path.
 *
 * Plain, slow, single-threaded C99, binary64, round-to-nearest-even, built with
 * -O2 -ffp-contract=off (no FMA contraction, no fast-math).  Each function follows the
 * paper's step order; where the paper is silent it takes the reading listed in
 * DESIGN.md §3 (C0..C8, G1..G20), cited in place.  All functions are pinned by
 * tests/test_oracle_*.py against values fixed by the paper or by mathematics.
 *
 * Citations: P:n = PAPER.md line n; S:n = SPEC.md line n.
 */
#include "minife_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------ */
/* Mesh (C0)                                                                    */
/* ------------------------------------------------------------------------------------ */

/* Fig 3.6 calls get_id(global_nodes_x, global_nodes_y, global_nodes_z, ix, iy, iz);
 * id = ix + nodes_x*(iy + nodes_y*iz).  G3: each axis is range-checked separately, so
 * ix = -1 does not wrap onto the previous grid line. */
int64_t or_node_id(int64_t nnx, int64_t nny, int64_t nnz, int64_t ix, int64_t iy, int64_t iz)
{
    if (ix < 0 || ix >= nnx || iy < 0 || iy >= nny || iz < 0 || iz >= nnz)
        return -1;
    return ix + nnx * (iy + nny * iz);
}

/* ------------------------------------------------------------------------------------ */
/* Element operator (C1, "Element operator computing")                   */
/* ------------------------------------------------------------------------------------ */

/* K[a][b] = integral over the element of grad(phi_a).grad(phi_b) for trilinear phi, written
 * as the tensor product of 1-D factors (C1):
 *   d_k = [bit_k(a) != bit_k(b)]  for axis k in (x, y, z)
 *   S_k = g_k if d_k == 0 else -g_k,  g_k = fl(1/h_k)      (1-D stiffness  int phi' phi')
 *   M_k = fl(h_k/3) if d_k == 0 else fl(h_k/6)              (1-D mass       int phi  phi )
 *   T_k = fl(fl(S_k * M_i) * M_j),  {i < j} = the other two axes, ascending
 *   K   = fl(fl(T_x + T_y) + T_z)
 * The source vector is zero (G6). */
void or_element_matrix(double hx, double hy, double hz, double K[64])
{
    const double h[3] = {hx, hy, hz};
    for (int a = 0; a < 8; ++a) {
        for (int b = 0; b < 8; ++b) {
            int d[3];
            for (int k = 0; k < 3; ++k)
                d[k] = ((a >> k) & 1) != ((b >> k) & 1);
            double T[3];
            for (int k = 0; k < 3; ++k) {
                double g = 1.0 / h[k];
                double S = d[k] ? -g : g;
                int i = (k == 0) ? 1 : 0;          /* other two axes, ascending */
                int j = (k == 2) ? 1 : 2;
                double Mi = d[i] ? h[i] / 6.0 : h[i] / 3.0;
                double Mj = d[j] ? h[j] / 6.0 : h[j] / 3.0;
                double t = S * Mi;
                T[k] = t * Mj;
            }
            double s = T[0] + T[1];
            K[8 * a + b] = s + T[2];
        }
    }
}

/* ------------------------------------------------------------------------------------ */
/* Matrix generation (Fig 3.6)                                     */
/* ------------------------------------------------------------------------------------ */

/* Fig 3.6's counting loop: for every row, every (sz, sy, sx) in {-1,0,1}^3 whose get_id is
 * valid adds one stored entry. */
int64_t or_structure_nnz(int nx, int ny, int nz)
{
    const int64_t NX = nx + 1, NY = ny + 1, NZ = nz + 1;
    int64_t nnz = 0;
    for (int64_t iz = 0; iz < NZ; ++iz)
        for (int64_t iy = 0; iy < NY; ++iy)
            for (int64_t ix = 0; ix < NX; ++ix)
                for (int sz = -1; sz <= 1; ++sz)
                    for (int sy = -1; sy <= 1; ++sy)
                        for (int sx = -1; sx <= 1; ++sx)
                            if (or_node_id(NX, NY, NZ, ix + sx, iy + sy, iz + sz) >= 0)
                                ++nnz;
    return nnz;
}

/* Same enumeration, storing the column ids.  Because ids are x-fastest and the loop
 * runs sz, sy, sx ascending (Fig 3.6 order), each row's columns come out ascending. */
int or_structure(int nx, int ny, int nz, int64_t *row_ptr, int64_t *col)
{
    if (nx < 1 || ny < 1 || nz < 1)
        return OR_EINVAL;
    const int64_t NX = nx + 1, NY = ny + 1, NZ = nz + 1;
    int64_t k = 0, row = 0;
    row_ptr[0] = 0;
    for (int64_t iz = 0; iz < NZ; ++iz)
        for (int64_t iy = 0; iy < NY; ++iy)
            for (int64_t ix = 0; ix < NX; ++ix) {
                for (int sz = -1; sz <= 1; ++sz)
                    for (int sy = -1; sy <= 1; ++sy)
                        for (int sx = -1; sx <= 1; ++sx) {
                            int64_t c = or_node_id(NX, NY, NZ, ix + sx, iy + sy, iz + sz);
                            if (c >= 0)
                                col[k++] = c;
                        }
                row_ptr[++row] = k;
            }
    return OR_OK;
}

/* ------------------------------------------------------------------------------------ */
/* FE assembly (Fig 3.7; C2)                                       */
/* ------------------------------------------------------------------------------------ */

static int64_t find_col(const int64_t *row_ptr, const int64_t *col, int64_t row, int64_t c)
{
    int64_t lo = row_ptr[row], hi = row_ptr[row + 1] - 1;
    while (lo <= hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (col[mid] == c)
            return mid;
        if (col[mid] < c)
            lo = mid + 1;
        else
            hi = mid - 1;
    }
    return -1;
}

/* get_elem_nodes_and_coords: the 8 node ids of element (ex,ey,ez) in local order
 * a = ax + 2*ay + 4*az. */
static void elem_nodes(int nx, int ny, int nz, int ex, int ey, int ez, int64_t nodes[8])
{
    for (int a = 0; a < 8; ++a)
        nodes[a] = or_node_id(nx + 1, ny + 1, nz + 1, ex + (a & 1), ey + ((a >> 1) & 1),
                              ez + ((a >> 2) & 1));
}

/* Fig 3.7: for each element (ascending id ex + nx*(ey + ny*ez), C2/G8):
 *   get_elem_nodes_and_coords; compute_element_matrix_and_vector; sum_into_global_linear_system.
 * val and b start at +0.0, so every entry is the left fold of its element contributions in
 * ascending element order. */
int or_assemble(int nx, int ny, int nz, const int64_t *row_ptr, const int64_t *col,
                double *val, double *b)
{
    if (nx < 1 || ny < 1 || nz < 1)
        return OR_EINVAL;
    const int64_t rows = (int64_t)(nx + 1) * (ny + 1) * (nz + 1);
    memset(val, 0, sizeof(double) * (size_t)row_ptr[rows]);
    memset(b, 0, sizeof(double) * (size_t)rows);
    const double hx = 1.0 / nx, hy = 1.0 / ny, hz = 1.0 / nz;   /* C0: h = fl(1/n) */
    double K[64];
    const double f[8] = {0, 0, 0, 0, 0, 0, 0, 0};                /* zero source (G6) */
    int64_t nodes[8];
    for (int ez = 0; ez < nz; ++ez)
        for (int ey = 0; ey < ny; ++ey)
            for (int ex = 0; ex < nx; ++ex) {
                elem_nodes(nx, ny, nz, ex, ey, ez, nodes);
                or_element_matrix(hx, hy, hz, K);
                for (int a = 0; a < 8; ++a) {
                    int64_t r = nodes[a];
                    for (int bb = 0; bb < 8; ++bb) {
                        int64_t pos = find_col(row_ptr, col, r, nodes[bb]);
                        if (pos < 0)
                            return OR_EINVAL;   /* structural miss: S:141 */
                        val[pos] = val[pos] + K[8 * a + bb];
                    }
                    b[r] = b[r] + f[a];
                }
            }
    return OR_OK;
}

/* ------------------------------------------------------------------------------------ */
/* Dirichlet boundary conditions (C3)                    */
/* ------------------------------------------------------------------------------------ */

/* u = 1.0 on the plane x = 1, 0.0 on the other boundary planes; G4: x = 1 wins on
 * shared edges and corners. */
static int is_bc(int nx, int ny, int nz, int64_t ix, int64_t iy, int64_t iz)
{
    return ix == 0 || ix == nx || iy == 0 || iy == ny || iz == 0 || iz == nz;
}
static double bc_value(int nx, int64_t ix) { return ix == nx ? 1.0 : 0.0; }

static void coords_of(int nx, int ny, int64_t gid, int64_t *ix, int64_t *iy, int64_t *iz)
{
    const int64_t NX = nx + 1, NY = ny + 1;
    *ix = gid % NX;
    *iy = (gid / NX) % NY;
    *iz = gid / (NX * NY);
}

/* C3 (S:149 symmetric elimination, pattern kept (G5)):
 *   free row j: for constrained columns i ascending, b_j = fl(b_j - fl(A_ji * v_i)); then each
 *               such A_ji = +0.0;
 *   constrained row i: every stored entry +0.0, diagonal 1.0, b_i = v_i. */
int or_impose_dirichlet(int nx, int ny, int nz, const int64_t *row_ptr, const int64_t *col,
                        double *val, double *b)
{
    const int64_t rows = (int64_t)(nx + 1) * (ny + 1) * (nz + 1);
    for (int64_t r = 0; r < rows; ++r) {
        int64_t ix, iy, iz;
        coords_of(nx, ny, r, &ix, &iy, &iz);
        if (is_bc(nx, ny, nz, ix, iy, iz)) {
            for (int64_t k = row_ptr[r]; k < row_ptr[r + 1]; ++k)
                val[k] = (col[k] == r) ? 1.0 : 0.0;
            b[r] = bc_value(nx, ix);
        } else {
            for (int64_t k = row_ptr[r]; k < row_ptr[r + 1]; ++k) {
                int64_t cx, cy, cz;
                coords_of(nx, ny, col[k], &cx, &cy, &cz);
                if (is_bc(nx, ny, nz, cx, cy, cz)) {
                    double prod = val[k] * bc_value(nx, cx);
                    b[r] = b[r] - prod;
                }
            }
            for (int64_t k = row_ptr[r]; k < row_ptr[r + 1]; ++k) {
                int64_t cx, cy, cz;
                coords_of(nx, ny, col[k], &cx, &cy, &cz);
                if (is_bc(nx, ny, nz, cx, cy, cz))
                    val[k] = 0.0;
            }
        }
    }
    return OR_OK;
}

/* One row of the final system, from scratch: the 27-point pattern of the row (Fig 3.6), the
 * element loop of Fig 3.7 restricted to the <= 8 elements containing the node (ascending
 * element id, as in or_assemble), then C3 for this row. */
int or_row(int nx, int ny, int nz, int64_t gid, int64_t *cols, double *vals, double *b_row)
{
    const int64_t NX = nx + 1, NY = ny + 1, NZ = nz + 1;
    if (gid < 0 || gid >= NX * NY * NZ)
        return -1;
    int64_t ix, iy, iz;
    coords_of(nx, ny, gid, &ix, &iy, &iz);
    int len = 0;
    for (int sz = -1; sz <= 1; ++sz)
        for (int sy = -1; sy <= 1; ++sy)
            for (int sx = -1; sx <= 1; ++sx) {
                int64_t c = or_node_id(NX, NY, NZ, ix + sx, iy + sy, iz + sz);
                if (c >= 0) {
                    cols[len] = c;
                    vals[len] = 0.0;
                    ++len;
                }
            }
    double b = 0.0;
    const double hx = 1.0 / nx, hy = 1.0 / ny, hz = 1.0 / nz;
    double K[64];
    int64_t nodes[8];
    for (int64_t ez = iz - 1; ez <= iz; ++ez)
        for (int64_t ey = iy - 1; ey <= iy; ++ey)
            for (int64_t ex = ix - 1; ex <= ix; ++ex) {
                if (ex < 0 || ex >= nx || ey < 0 || ey >= ny || ez < 0 || ez >= nz)
                    continue;
                elem_nodes(nx, ny, nz, (int)ex, (int)ey, (int)ez, nodes);
                or_element_matrix(hx, hy, hz, K);
                int a = (int)((ix - ex) + 2 * (iy - ey) + 4 * (iz - ez));
                for (int bb = 0; bb < 8; ++bb) {
                    int k = 0;
                    while (cols[k] != nodes[bb])
                        ++k;
                    vals[k] = vals[k] + K[8 * a + bb];
                }
                b = b + 0.0;   /* zero source vector entry (G6) */
            }
    if (is_bc(nx, ny, nz, ix, iy, iz)) {
        for (int k = 0; k < len; ++k)
            vals[k] = (cols[k] == gid) ? 1.0 : 0.0;
        b = bc_value(nx, ix);
    } else {
        for (int k = 0; k < len; ++k) {
            int64_t cx, cy, cz;
            coords_of(nx, ny, cols[k], &cx, &cy, &cz);
            if (is_bc(nx, ny, nz, cx, cy, cz)) {
                double prod = vals[k] * bc_value(nx, cx);
                b = b - prod;
            }
        }
        for (int k = 0; k < len; ++k) {
            int64_t cx, cy, cz;
            coords_of(nx, ny, cols[k], &cx, &cy, &cz);
            if (is_bc(nx, ny, nz, cx, cy, cz))
                vals[k] = 0.0;
        }
    }
    *b_row = b;
    return len;
}

/* ------------------------------------------------------------------------------------ */
/* SpMV (Fig 3.1; C4)                                                          */
/* ------------------------------------------------------------------------------------ */

/* Fig 3.1 accumulates y[i] += val[j]*x[col[j]] from y[i] = 0; C4 fixes the start value +0.0
 * and the order (stored order = ascending global column). */
void or_spmv(int64_t m, const int64_t *row_ptr, const int64_t *col, const double *val,
             const double *x, double *y)
{
    for (int64_t i = 0; i < m; ++i) {
        double s = 0.0;
        for (int64_t j = row_ptr[i]; j < row_ptr[i + 1]; ++j) {
            double prod = val[j] * x[col[j]];
            s = s + prod;
        }
        y[i] = s;
    }
}

/* ------------------------------------------------------------------------------------ */
/* Exactly-rounded dot product (C5; "vector dot product", P:204 global reduction)   */
/* ------------------------------------------------------------------------------------ */

/* The exact sum is held as one two's-complement integer N of 64*LIMBS bits with
 * value = N * 2^-1074 (2^-1074 = the smallest subnormal, so every double is an integer
 * multiple of it).  The largest finite double needs bit 2097; LIMBS = 36 leaves > 190 bits of
 * headroom, far beyond any count of terms. */
#define LIMBS 36

static void big_add(uint64_t *w, int L, uint64_t lo, uint64_t hi)
{
    unsigned __int128 acc = (unsigned __int128)w[L] + lo;
    w[L] = (uint64_t)acc;
    acc >>= 64;
    acc += (unsigned __int128)w[L + 1] + hi;
    w[L + 1] = (uint64_t)acc;
    acc >>= 64;
    for (int i = L + 2; i < LIMBS && acc; ++i) {
        acc += w[i];
        w[i] = (uint64_t)acc;
        acc >>= 64;
    }
}

static void big_sub(uint64_t *w, int L, uint64_t lo, uint64_t hi)
{
    uint64_t old = w[L];
    w[L] = old - lo;
    uint64_t borrow = old < lo;
    old = w[L + 1];
    uint64_t sub = hi + borrow;          /* hi < 2^53: cannot wrap */
    w[L + 1] = old - sub;
    borrow = old < sub;
    for (int i = L + 2; i < LIMBS && borrow; ++i) {
        old = w[i];
        w[i] = old - 1;
        borrow = (old == 0);
    }
}

static int big_bit(const uint64_t *w, int i) { return (int)((w[i / 64] >> (i % 64)) & 1u); }

/* dot(u,v) = RN( sum_i^exact fl(u_i * v_i) ), ties-to-even, exact zero -> +0.0.
 * Any non-finite product makes the result NaN (reading in DESIGN.md §3, C5). */
double or_dot(int64_t n, const double *u, const double *v)
{
    uint64_t w[LIMBS];
    memset(w, 0, sizeof w);
    int nonfinite = 0;
    for (int64_t i = 0; i < n; ++i) {
        double p = u[i] * v[i];
        uint64_t bits;
        memcpy(&bits, &p, sizeof bits);
        int neg = (int)(bits >> 63);
        int e = (int)((bits >> 52) & 0x7ff);
        uint64_t frac = bits & ((1ull << 52) - 1);
        if (e == 0x7ff) {
            nonfinite = 1;
            continue;
        }
        if (e == 0 && frac == 0)
            continue;
        /* p = m * 2^(pos - 1074): normal numbers m = 1.frac * 2^52, pos = e - 1;
         * subnormals m = frac, pos = 0. */
        uint64_t m = (e == 0) ? frac : (frac | (1ull << 52));
        int pos = (e == 0) ? 0 : e - 1;
        int L = pos / 64, s = pos % 64;
        uint64_t lo = m << s;
        uint64_t hi = s ? (m >> (64 - s)) : 0;
        if (neg)
            big_sub(w, L, lo, hi);
        else
            big_add(w, L, lo, hi);
    }
    if (nonfinite)
        return NAN;
    int negative = (int)(w[LIMBS - 1] >> 63);
    if (negative) { /* magnitude = two's complement negation */
        unsigned __int128 c = 1;
        for (int i = 0; i < LIMBS; ++i) {
            c += (uint64_t)~w[i];
            w[i] = (uint64_t)c;
            c >>= 64;
        }
    }
    int t = -1;
    for (int i = 64 * LIMBS - 1; i >= 0; --i)
        if (big_bit(w, i)) {
            t = i;
            break;
        }
    if (t < 0)
        return 0.0;
    double mag;
    if (t <= 52) {
        mag = ldexp((double)w[0], -1074);          /* < 2^53 units of 2^-1074: exact */
    } else {
        uint64_t M = 0;
        for (int i = t; i >= t - 52; --i)
            M = (M << 1) | (uint64_t)big_bit(w, i);
        int guard = big_bit(w, t - 53);
        int sticky = 0;
        for (int i = t - 54; i >= 0 && !sticky; --i)
            sticky = big_bit(w, i);
        if (guard && (sticky || (M & 1u)))
            ++M;
        int top = t;
        if (M == (1ull << 53)) {
            M >>= 1;
            ++top;
        }
        mag = ldexp((double)M, top - 52 - 1074);   /* overflows to inf iff RN does */
    }
    return negative ? -mag : mag;
}

/* ------------------------------------------------------------------------------------ */
/* Conjugate gradient ("CG module"; C6)                                  */
/* ------------------------------------------------------------------------------------ */

/* C6:
 *   x = 0, r = b, p = b, rr = dot(r,r), hist[0] = sqrt(rr)
 *   for k = 1..K:
 *     Ap = A p;  pAp = dot(p, Ap)
 *     pAp non-finite             -> DIVERGED (iters = k-1)
 *     pAp <= 0: rr == 0 -> converged (iters = k-1), else NOT-SPD (iters = k-1)
 *     alpha = rr / pAp
 *     x_i = x_i + fl(alpha p_i);  r_i = r_i - fl(alpha Ap_i)
 *     rr' = dot(r,r); hist[k] = sqrt(rr'); iters = k
 *     rr' non-finite             -> DIVERGED
 *     rr' == 0 or hist[k] <= fl(tol*hist[0]) -> converged
 *     beta = rr'/rr;  p_i = r_i + fl(beta p_i);  rr = rr'                                */
int or_cg(int64_t m, const int64_t *row_ptr, const int64_t *col, const double *val,
          const double *b, int max_iters, double tol, double *x, double *hist, int *iters,
          int *converged)
{
    *iters = 0;
    *converged = 0;
    if (max_iters < 1 || !(tol >= 0.0))
        return OR_EINVAL;
    double *r = (double *)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
    double *p = (double *)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
    double *Ap = (double *)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
    int status = OR_OK;
    for (int64_t i = 0; i < m; ++i) {
        x[i] = 0.0;
        r[i] = b[i];
        p[i] = b[i];
    }
    double rr = or_dot(m, r, r);
    hist[0] = sqrt(rr);
    const double stop = tol * hist[0];
    for (int k = 1; k <= max_iters; ++k) {
        or_spmv(m, row_ptr, col, val, p, Ap);
        double pAp = or_dot(m, p, Ap);
        if (!isfinite(pAp)) {
            status = OR_EDIVERGED;
            break;
        }
        if (pAp <= 0.0) {
            if (rr == 0.0)
                *converged = 1;
            else
                status = OR_ENOTSPD;
            break;
        }
        double alpha = rr / pAp;
        for (int64_t i = 0; i < m; ++i) {
            double ap = alpha * p[i];
            x[i] = x[i] + ap;
            double aap = alpha * Ap[i];
            r[i] = r[i] - aap;
        }
        double rr_new = or_dot(m, r, r);
        hist[k] = sqrt(rr_new);
        *iters = k;
        if (!isfinite(rr_new)) {
            status = OR_EDIVERGED;
            break;
        }
        if (rr_new == 0.0 || hist[k] <= stop) {
            *converged = 1;
            break;
        }
        double beta = rr_new / rr;
        for (int64_t i = 0; i < m; ++i) {
            double bp = beta * p[i];
            p[i] = r[i] + bp;
        }
        rr = rr_new;
    }
    free(r);
    free(p);
    free(Ap);
    return status;
}

/* ------------------------------------------------------------------------------------ */
/* Analytical solution ("result verification"; C8)                  */
/* ------------------------------------------------------------------------------------ */

/* Laplace's equation on the unit cube, u = 1 on x = 1, u = 0 on the other faces:
 *   u = sum_{m,n odd} 16/(m n pi^2) * sinh(lam x)/sinh(lam) * sin(m pi y) sin(n pi z),
 *   lam = pi sqrt(m^2 + n^2),
 * with the sinh ratio written as e^{lam(x-1)} (1 - e^{-2 lam x}) / (1 - e^{-2 lam})
 * so that large lam cannot overflow. */
double or_analytic(double x, double y, double z, int nterms)
{
    const double pi = 3.14159265358979323846;
    double u = 0.0;
    for (int i = 0; i < nterms; ++i) {
        int m = 2 * i + 1;
        double sy = sin(m * pi * y);
        for (int j = 0; j < nterms; ++j) {
            int n = 2 * j + 1;
            double lam = pi * sqrt((double)m * m + (double)n * n);
            double ratio = exp(lam * (x - 1.0)) * (1.0 - exp(-2.0 * lam * x)) /
                           (1.0 - exp(-2.0 * lam));
            u += 16.0 / ((double)m * n * pi * pi) * ratio * sy * sin(n * pi * z);
        }
    }
    return u;
}

/* ------------------------------------------------------------------------------------ */
/* Partition ("recursive coordinate bisection"; G15)    */
/* ------------------------------------------------------------------------------------ */

static int rcb_rec(int lo[3], int hi[3], int r0, int p, int *boxes)
{
    int64_t elems = (int64_t)(hi[0] - lo[0]) * (hi[1] - lo[1]) * (hi[2] - lo[2]);
    if (elems < p)
        return OR_EINVAL;
    if (p == 1) {
        for (int k = 0; k < 3; ++k) {
            boxes[6 * r0 + k] = lo[k];
            boxes[6 * r0 + 3 + k] = hi[k];
        }
        return OR_OK;
    }
    /* longest axis, ties x before y before z; ceil(p/2) ranks take the lower half,
     * split at the element index dividing the elements proportionally to the rank halves. */
    int axis = 0;
    for (int k = 1; k < 3; ++k)
        if (hi[k] - lo[k] > hi[axis] - lo[axis])
            axis = k;
    int plo = (p + 1) / 2, phi = p / 2;
    int len = hi[axis] - lo[axis];
    int cut = lo[axis] + (int)(((int64_t)len * plo) / p);
    int lo2[3], hi2[3];
    for (int k = 0; k < 3; ++k) {
        lo2[k] = lo[k];
        hi2[k] = hi[k];
    }
    hi2[axis] = cut;
    int st = rcb_rec(lo2, hi2, r0, plo, boxes);
    if (st != OR_OK)
        return st;
    for (int k = 0; k < 3; ++k) {
        lo2[k] = lo[k];
        hi2[k] = hi[k];
    }
    lo2[axis] = cut;
    return rcb_rec(lo2, hi2, r0 + plo, phi, boxes);
}

int or_rcb(int nx, int ny, int nz, int p, int *boxes)
{
    if (nx < 1 || ny < 1 || nz < 1 || p < 1)
        return OR_EINVAL;
    int lo[3] = {0, 0, 0}, hi[3] = {nx, ny, nz};
    return rcb_rec(lo, hi, 0, p, boxes);
}

/* a node belongs to the lowest rank whose CLOSED node range (element range [lo,hi)
 * spans nodes lo..hi) contains it. */
int or_owner(int p, const int *boxes, int ix, int iy, int iz)
{
    const int c[3] = {ix, iy, iz};
    for (int r = 0; r < p; ++r) {
        int in = 1;
        for (int k = 0; k < 3; ++k)
            if (c[k] < boxes[6 * r + k] || c[k] > boxes[6 * r + 3 + k])
                in = 0;
        if (in)
            return r;
    }
    return -1;
}

int64_t or_owned(int nx, int ny, int nz, int p, const int *boxes, int rank, int64_t *out)
{
    int64_t cnt = 0, gid = 0;
    for (int iz = 0; iz <= nz; ++iz)
        for (int iy = 0; iy <= ny; ++iy)
            for (int ix = 0; ix <= nx; ++ix, ++gid)
                if (or_owner(p, boxes, ix, iy, iz) == rank) {
                    if (out)
                        out[cnt] = gid;
                    ++cnt;
                }
    return cnt;
}

/* externals = nodes not owned by `rank` that appear in the 27-point stencil of an owned
 * node; ordered by owning rank ascending, then global id ascending. */
int64_t or_externals(int nx, int ny, int nz, int p, const int *boxes, int rank, int64_t *out)
{
    const int64_t NX = nx + 1, NY = ny + 1, NZ = nz + 1, N = NX * NY * NZ;
    unsigned char *mark = (unsigned char *)calloc((size_t)N, 1);
    int *own = (int *)malloc(sizeof(int) * (size_t)N);
    int64_t gid = 0;
    for (int iz = 0; iz <= nz; ++iz)
        for (int iy = 0; iy <= ny; ++iy)
            for (int ix = 0; ix <= nx; ++ix, ++gid)
                own[gid] = or_owner(p, boxes, ix, iy, iz);
    gid = 0;
    for (int64_t iz = 0; iz < NZ; ++iz)
        for (int64_t iy = 0; iy < NY; ++iy)
            for (int64_t ix = 0; ix < NX; ++ix, ++gid) {
                if (own[gid] != rank)
                    continue;
                for (int sz = -1; sz <= 1; ++sz)
                    for (int sy = -1; sy <= 1; ++sy)
                        for (int sx = -1; sx <= 1; ++sx) {
                            int64_t c = or_node_id(NX, NY, NZ, ix + sx, iy + sy, iz + sz);
                            if (c >= 0 && own[c] != rank)
                                mark[c] = 1;
                        }
            }
    int64_t cnt = 0;
    for (int q = 0; q < p; ++q)
        for (int64_t g = 0; g < N; ++g)
            if (mark[g] && own[g] == q) {
                if (out)
                    out[cnt] = g;
                ++cnt;
            }
    free(mark);
    free(own);
    return cnt;
}
