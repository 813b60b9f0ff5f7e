// kernels.cu — sm_100a kernels of the MiniFE CG hot path.
//
// Arithmetic contract (C0-C6): binary64, round-to-nearest-even, every product
// and sum written with __dmul_rn/__dadd_rn/__dsub_rn (never contracted to FMA; the library
// is also built with -fmad=false), subnormals kept.  Dots are exactly rounded (exact.cuh).
//
// Layout: SELL-32, one slice = 32 consecutive local rows; slice s holds
// width_s = max row length columns, stored k-major: entry k of row 32s+lane lives at
// slice_off[s] + 32k + lane, so a warp's loads of one k are one contiguous 256 B (val) /
// 128 B (col) segment.  Entries of a row are in ascending GLOBAL column (C4 order); padding
// entries (k >= row_len) have val 0 and col = a valid index and are never added.
#include <cuda_runtime.h>

#include "exact.cuh"
#include "kernels.h"

namespace minife {

// ----------------------------------------------------------------------------------------
// small helpers
// ----------------------------------------------------------------------------------------

// Streaming (read-once) loads of the matrix: skip L1, evict-first in L2 so the re-used
// x vector (3 planes at a time, ~2 MB at 300^3) stays L2-resident.
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ double ld_stream(const double *p, uint64_t pol) {
    double v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
                 : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ int ld_stream(const int32_t *p, uint64_t pol) {
    int v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;"
                 : "=r"(v) : "l"(p), "l"(pol));
    return v;
}

// P:36 boundary: every surface node is constrained; value 1 on the plane x = 1 (G4).
__device__ __forceinline__ bool on_boundary(int64_t ix, int64_t iy, int64_t iz, int nx, int ny,
                                            int nz) {
    return ix == 0 || ix == nx || iy == 0 || iy == ny || iz == 0 || iz == nz;
}

// ----------------------------------------------------------------------------------------
// a0.2: row lengths and SELL slice widths
// ----------------------------------------------------------------------------------------

// Row length of node (ix,iy,iz) = c(ix) c(iy) c(iz), c = 2 on a boundary plane else 3
// (Fig 3.6's in-range count, closed form).
__global__ void k_rowlen_widths(AsmArgs a, uint8_t *row_len, uint8_t *width, int64_t nslices) {
    const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t slice = row >> 5;
    if (slice >= nslices) return;
    int len = 0;
    if (row < a.rows) {
        const int64_t lx = row % a.own_n[0], ly = (row / a.own_n[0]) % a.own_n[1],
                      lz = row / (a.own_n[0] * a.own_n[1]);
        const int64_t ix = a.own_lo[0] + lx, iy = a.own_lo[1] + ly, iz = a.own_lo[2] + lz;
        const int cx = (ix == 0 || ix == a.nx) ? 2 : 3;
        const int cy = (iy == 0 || iy == a.ny) ? 2 : 3;
        const int cz = (iz == 0 || iz == a.nz) ? 2 : 3;
        len = cx * cy * cz;
        row_len[row] = (uint8_t)len;
    }
    const int w = __reduce_max_sync(0xffffffffu, (unsigned)len);
    if ((threadIdx.x & 31) == 0) width[slice] = (uint8_t)w;
}

// ----------------------------------------------------------------------------------------
// a0.3 + a0.4 + a0.5: element operator, gather-assembly, Dirichlet elimination
// ----------------------------------------------------------------------------------------

// C1: K(d) for the 8 difference patterns d = dx | dy<<1 | dz<<2 of an (hx,hy,hz) brick.
__device__ void element_operator(int nx, int ny, int nz, double K[8]) {
    const double h[3] = {__ddiv_rn(1.0, (double)nx), __ddiv_rn(1.0, (double)ny),
                         __ddiv_rn(1.0, (double)nz)};
    for (int d = 0; d < 8; ++d) {
        double T[3];
        for (int k = 0; k < 3; ++k) {
            const bool dk = (d >> k) & 1;
            const double g = __ddiv_rn(1.0, h[k]);
            const double S = dk ? -g : g;
            const int i = (k == 0) ? 1 : 0, j = (k == 2) ? 1 : 2;
            const double Mi = ((d >> i) & 1) ? __ddiv_rn(h[i], 6.0) : __ddiv_rn(h[i], 3.0);
            const double Mj = ((d >> j) & 1) ? __ddiv_rn(h[j], 6.0) : __ddiv_rn(h[j], 3.0);
            T[k] = __dmul_rn(__dmul_rn(S, Mi), Mj);
        }
        K[d] = __dadd_rn(__dadd_rn(T[0], T[1]), T[2]);
    }
}

// One thread per local row.  Entry (i,j) = fold from +0.0 of K(d(i,j)) over the c(i,j)
// elements that share nodes i and j (C2; every term is the same K(d), the count is the
// per-axis product of 1 (coordinates differ) or #elements on that axis containing i).
// Then C3: constrained row -> identity row, b = v; free row -> for constrained columns in
// ascending global order b = fl(b - fl(A v)), then A = +0.0.
__global__ void k_assemble(AsmArgs a) {
    const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nslices = (a.rows + 31) >> 5;
    if ((row >> 5) >= nslices) return;
    const int lane = (int)(row & 31);
    const int64_t s = row >> 5;
    const int64_t base = a.slice_off[s] + lane;
    const int w = (int)((a.slice_off[s + 1] - a.slice_off[s]) >> 5);
    if (row >= a.rows) {                           // padding lanes of the last slice
        for (int k = 0; k < w; ++k) {
            a.col[base + 32 * k] = 0;
            a.val[base + 32 * k] = 0.0;
        }
        return;
    }
    double K[8];
    element_operator(a.nx, a.ny, a.nz, K);
    const int64_t NX = a.nx + 1, NY = a.ny + 1, NZ = a.nz + 1;
    const int64_t lx = row % a.own_n[0], ly = (row / a.own_n[0]) % a.own_n[1],
                  lz = row / (a.own_n[0] * a.own_n[1]);
    const int64_t ix = a.own_lo[0] + lx, iy = a.own_lo[1] + ly, iz = a.own_lo[2] + lz;
    const bool row_bc = on_boundary(ix, iy, iz, a.nx, a.ny, a.nz);
    const int n_el[3] = {(ix > 0) + (ix < a.nx), (iy > 0) + (iy < a.ny), (iz > 0) + (iz < a.nz)};
    double b = 0.0;
    int k = 0;
    for (int dz = -1; dz <= 1; ++dz) {
        const int64_t jz = iz + dz;
        if (jz < 0 || jz >= NZ) continue;
        for (int dy = -1; dy <= 1; ++dy) {
            const int64_t jy = iy + dy;
            if (jy < 0 || jy >= NY) continue;
            for (int dx = -1; dx <= 1; ++dx) {
                const int64_t jx = ix + dx;
                if (jx < 0 || jx >= NX) continue;
                const int c = (dx ? 1 : n_el[0]) * (dy ? 1 : n_el[1]) * (dz ? 1 : n_el[2]);
                const double Kd = K[(dx != 0) | ((dy != 0) << 1) | ((dz != 0) << 2)];
                double v = 0.0;
                for (int t = 0; t < c; ++t) v = __dadd_rn(v, Kd);
                // local column: owned box index, or the external slot (binary search)
                int32_t lc;
                const int64_t ox = jx - a.own_lo[0], oy = jy - a.own_lo[1], oz = jz - a.own_lo[2];
                if (ox >= 0 && ox < a.own_n[0] && oy >= 0 && oy < a.own_n[1] && oz >= 0 &&
                    oz < a.own_n[2]) {
                    lc = (int32_t)(ox + a.own_n[0] * (oy + a.own_n[1] * oz));
                } else {
                    const int64_t g = jx + NX * (jy + NY * jz);
                    int64_t lo = 0, hi = a.n_ext - 1;
                    lc = -1;
                    while (lo <= hi) {
                        const int64_t mid = (lo + hi) >> 1;
                        const int64_t gm = a.ext_sorted_gid[mid];
                        if (gm == g) {
                            lc = a.ext_sorted_slot[mid];
                            break;
                        }
                        if (gm < g) lo = mid + 1;
                        else hi = mid - 1;
                    }
                }
                if (row_bc) {
                    v = (dx == 0 && dy == 0 && dz == 0) ? 1.0 : 0.0;
                } else if (on_boundary(jx, jy, jz, a.nx, a.ny, a.nz)) {
                    const double bv = (jx == a.nx) ? 1.0 : 0.0;
                    b = __dsub_rn(b, __dmul_rn(v, bv));
                    v = 0.0;
                }
                a.col[base + 32 * k] = lc;
                a.val[base + 32 * k] = v;
                ++k;
            }
        }
    }
    for (int kk = k; kk < w; ++kk) {                  // padding: own row, value 0
        a.col[base + 32 * kk] = (int32_t)row;
        a.val[base + 32 * kk] = 0.0;
    }
    if (row_bc) b = (ix == a.nx) ? 1.0 : 0.0;
    a.b[row] = b;
}

// ----------------------------------------------------------------------------------------
// a2: SpMV  y = A x  (+ exact pAp epilogue)
// ----------------------------------------------------------------------------------------

// C4 per row: s = +0.0; for stored entries in order, s = fl(s + fl(a * x_col)); padding is
// skipped by the row-length predicate (so a -0.0 row sum is never turned into +0.0).
// One warp per slice, one lane per row; warps walk the slices grid-stride so each thread's
// expansion absorbs many rows before the single flush.
template <bool DOT>
__global__ void __launch_bounds__(SPMV_THREADS) k_spmv(SpmvArgs a) {
    __shared__ unsigned long long sacc[ACC_WORDS];
    if (DOT) {
        if (a.st && a.st->done) return;
        acc_zero_shared(sacc);
        if (blockIdx.x == 0 && a.acc_zero)
            for (int i = threadIdx.x; i < ACC_WORDS; i += blockDim.x) a.acc_zero[i] = 0ull;
        __syncthreads();
    }
    Expansion ex;
    ex.init();
    const uint64_t pol = evict_first_policy();
    const int lane = threadIdx.x & 31;
    const int64_t warps_per_block = blockDim.x >> 5;
    const int64_t nw = (int64_t)gridDim.x * warps_per_block;
    for (int64_t s = (int64_t)blockIdx.x * warps_per_block + (threadIdx.x >> 5); s < a.nslices;
         s += nw) {
        const int64_t off = a.slice_off[s];
        const int w = (int)((a.slice_off[s + 1] - off) >> 5);
        const int64_t row = s * 32 + lane;
        const int len = (row < a.rows) ? (int)a.row_len[row] : 0;
        const double *v = a.val + off + lane;
        const int32_t *c = a.col + off + lane;
        double sum = 0.0;
        if (w == 27) {
            double vv[27];
            int cc[27];
#pragma unroll
            for (int k = 0; k < 27; ++k) {
                vv[k] = ld_stream(v + 32 * k, pol);
                cc[k] = ld_stream(c + 32 * k, pol);
            }
            double xv[27];
#pragma unroll
            for (int k = 0; k < 27; ++k) xv[k] = __ldg(a.x + cc[k]);   // padding cols are valid
#pragma unroll
            for (int k = 0; k < 27; ++k)
                if (k < len) sum = __dadd_rn(sum, __dmul_rn(vv[k], xv[k]));
        } else {
#pragma unroll 3
            for (int k = 0; k < w; ++k) {
                const double vk = ld_stream(v + 32 * k, pol);
                const int ck = ld_stream(c + 32 * k, pol);
                if (k < len) sum = __dadd_rn(sum, __dmul_rn(vk, __ldg(a.x + ck)));
            }
        }
        if (row < a.rows) {
            a.y[row] = sum;
            if (DOT) ex.add(__dmul_rn(__ldg(a.x + row), sum), sacc);
        }
    }
    if (DOT) {
        ex.flush(sacc);
        __syncthreads();
        acc_merge_to_global(sacc, a.acc);
    }
}

// ----------------------------------------------------------------------------------------
// CG init (C6 step 1): x = 0, r = b, p = b, rr = dot(r, r)
// ----------------------------------------------------------------------------------------

__global__ void __launch_bounds__(UPD_THREADS) k_init_vectors(UpdArgs a) {
    __shared__ unsigned long long sacc[ACC_WORDS];
    acc_zero_shared(sacc);
    __syncthreads();
    Expansion ex;
    ex.init();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.rows; i += stride) {
        const double bi = a.b[i];
        a.x[i] = 0.0;
        a.r[i] = bi;
        a.p[i] = bi;
        ex.add(__dmul_rn(bi, bi), sacc);
    }
    ex.flush(sacc);
    __syncthreads();
    acc_merge_to_global(sacc, a.acc_out);
}

__global__ void k_init_finalize(UpdArgs a, double tol) {
    if (threadIdx.x == 0) {
        const double rr0 = acc_finalize(a.acc_out);
        const double h0 = __dsqrt_rn(rr0);
        a.rr[0] = rr0;
        a.hist[0] = h0;
        CgState st;
        st.done = 0;
        st.status = 0;
        st.iters = 0;
        st.converged = 0;
        st.stop = __dmul_rn(tol, h0);
        st.pAp = 0.0;
        st.alpha = 0.0;
        st.beta = 0.0;
        *a.st = st;
    }
    if (a.acc_zero)
        for (int i = threadIdx.x; i < ACC_WORDS; i += blockDim.x) a.acc_zero[i] = 0ull;
}

// ----------------------------------------------------------------------------------------
// a3 + a4: finalise pAp -> alpha; x += alpha p; r -= alpha Ap; rr' = dot(r, r)
// ----------------------------------------------------------------------------------------

__global__ void __launch_bounds__(UPD_THREADS) k_update_xr(UpdArgs a, int k) {
    __shared__ unsigned long long sacc[ACC_WORDS];
    __shared__ double s_alpha;
    __shared__ int s_stop;
    if (a.st->done) return;
    acc_zero_shared(sacc);
    if (threadIdx.x == 0) {
        const double pAp = acc_finalize(a.acc_in);
        const double rr = a.rr[k - 1];
        int stop = 0, status = 0, conv = 0;
        if (!isfinite(pAp)) {
            stop = 1;
            status = 7;
        } else if (pAp <= 0.0) {
            stop = 1;
            if (rr == 0.0) conv = 1;
            else status = 6;
        }
        const double alpha = __ddiv_rn(rr, pAp);
        s_alpha = alpha;
        s_stop = stop;
        if (blockIdx.x == 0) {
            a.st->pAp = pAp;
            a.st->alpha = alpha;
            if (stop) {
                a.st->status = status;
                a.st->converged = conv;
                a.st->iters = k - 1;
                a.st->done = 1;
            }
        }
    }
    __syncthreads();
    if (s_stop) return;
    const double alpha = s_alpha;
    Expansion ex;
    ex.init();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.rows; i += stride) {
        const double pi = a.p[i], api = a.Ap[i];
        a.x[i] = __dadd_rn(a.x[i], __dmul_rn(alpha, pi));
        const double ri = __dsub_rn(a.r[i], __dmul_rn(alpha, api));
        a.r[i] = ri;
        ex.add(__dmul_rn(ri, ri), sacc);
    }
    ex.flush(sacc);
    __syncthreads();
    acc_merge_to_global(sacc, a.acc_out);
}

// ----------------------------------------------------------------------------------------
// a5 + a6: finalise rr' -> hist[k], stop tests, beta; p = r + beta p
// ----------------------------------------------------------------------------------------

__global__ void __launch_bounds__(UPD_THREADS) k_update_p(UpdArgs a, int k) {
    __shared__ double s_beta;
    __shared__ int s_stop;
    if (a.st->done) return;
    if (threadIdx.x == 0) {
        const double rr_new = acc_finalize(a.acc_in);
        const double h = __dsqrt_rn(rr_new);
        const double rr_old = a.rr[k - 1];
        int stop = 0, status = 0, conv = 0;
        if (!isfinite(rr_new)) {
            stop = 1;
            status = 7;
        } else if (rr_new == 0.0 || h <= a.st->stop) {
            stop = 1;
            conv = 1;
        }
        const double beta = __ddiv_rn(rr_new, rr_old);
        s_beta = beta;
        s_stop = stop;
        if (blockIdx.x == 0) {
            a.hist[k] = h;
            a.rr[k] = rr_new;
            a.st->iters = k;
            a.st->beta = beta;
            if (stop) {
                a.st->status = status;
                a.st->converged = conv;
                a.st->done = 1;
            }
        }
    }
    __syncthreads();
    if (s_stop) return;
    if (blockIdx.x == 0 && a.acc_zero)
        for (int i = threadIdx.x; i < ACC_WORDS; i += blockDim.x) a.acc_zero[i] = 0ull;
    const double beta = s_beta;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.rows; i += stride)
        a.p[i] = __dadd_rn(a.r[i], __dmul_rn(beta, a.p[i]));
}

// ----------------------------------------------------------------------------------------
// a1: halo pack / virtual-rank transport
// ----------------------------------------------------------------------------------------

__global__ void k_pack(const double *__restrict__ src, const int32_t *__restrict__ idx,
                       int64_t n, double *__restrict__ dst) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        dst[i] = src[idx[i]];
}

struct AccPtrs {
    unsigned long long *p[64];
};

// int64 SUM all-reduce of the parts' accumulators on one device (associative -> exact).
__global__ void k_vsum(AccPtrs ptrs, int nparts) {
    for (int i = threadIdx.x; i < ACC_WORDS; i += blockDim.x) {
        unsigned long long s = 0;
        for (int q = 0; q < nparts; ++q) s += ptrs.p[q][i];
        for (int q = 0; q < nparts; ++q) ptrs.p[q][i] = s;
    }
}

__global__ void k_extract_rows(const int64_t *slice_off, const uint8_t *row_len,
                               const int32_t *col, const double *val, const int64_t *rows,
                               int64_t n, int32_t *out_col, double *out_val, int32_t *out_len) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t row = rows[i];
    const int64_t s = row >> 5, lane = row & 31;
    const int len = row_len[row];
    out_len[i] = len;
    for (int k = 0; k < len; ++k) {
        out_col[27 * i + k] = col[slice_off[s] + 32 * k + lane];
        out_val[27 * i + k] = val[slice_off[s] + 32 * k + lane];
    }
}

// ----------------------------------------------------------------------------------------
// launch wrappers
// ----------------------------------------------------------------------------------------

static int g_sms = 0;
static int g_spmv_blocks_per_sm = 0;
static int g_upd_blocks_per_sm = 0;

static void query_occupancy() {
    if (g_sms) return;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_spmv_blocks_per_sm, k_spmv<true>,
                                                  SPMV_THREADS, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_upd_blocks_per_sm, k_update_xr,
                                                  UPD_THREADS, 0);
    if (g_sms <= 0) g_sms = 148;
    if (g_spmv_blocks_per_sm <= 0) g_spmv_blocks_per_sm = 1;
    if (g_upd_blocks_per_sm <= 0) g_upd_blocks_per_sm = 1;
}

int spmv_grid(int64_t nslices) {
    query_occupancy();
    const int64_t need = (nslices + (SPMV_THREADS / 32) - 1) / (SPMV_THREADS / 32);
    const int64_t full = (int64_t)g_sms * g_spmv_blocks_per_sm;
    return (int)(need < full ? (need > 0 ? need : 1) : full);
}

int stream_grid(int64_t rows) {
    query_occupancy();
    const int64_t need = (rows + UPD_THREADS - 1) / UPD_THREADS;
    const int64_t full = (int64_t)g_sms * g_upd_blocks_per_sm;
    return (int)(need < full ? (need > 0 ? need : 1) : full);
}

cudaError_t launch_rowlen_widths(const AsmArgs &a, uint8_t *row_len, uint8_t *width,
                                 int64_t nslices, cudaStream_t s) {
    const int64_t threads = nslices * 32;
    k_rowlen_widths<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(a, row_len, width, nslices);
    return cudaGetLastError();
}

cudaError_t launch_assemble(const AsmArgs &a, cudaStream_t s) {
    const int64_t threads = ((a.rows + 31) >> 5) * 32;
    k_assemble<<<(unsigned)((threads + 127) / 128), 128, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_spmv(const SpmvArgs &a, bool with_dot, int grid, cudaStream_t s) {
    if (with_dot) k_spmv<true><<<grid, SPMV_THREADS, 0, s>>>(a);
    else k_spmv<false><<<grid, SPMV_THREADS, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_init_vectors(const UpdArgs &a, int grid, cudaStream_t s) {
    k_init_vectors<<<grid, UPD_THREADS, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_init_finalize(const UpdArgs &a, double tol, cudaStream_t s) {
    k_init_finalize<<<1, 128, 0, s>>>(a, tol);
    return cudaGetLastError();
}

cudaError_t launch_update_xr(const UpdArgs &a, int k, int grid, cudaStream_t s) {
    k_update_xr<<<grid, UPD_THREADS, 0, s>>>(a, k);
    return cudaGetLastError();
}

cudaError_t launch_update_p(const UpdArgs &a, int k, int grid, cudaStream_t s) {
    k_update_p<<<grid, UPD_THREADS, 0, s>>>(a, k);
    return cudaGetLastError();
}

cudaError_t launch_pack(const double *src, const int32_t *idx, int64_t n, double *dst,
                        cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    int grid = (int)((n + 255) / 256);
    if (grid > 1184) grid = 1184;
    k_pack<<<grid, 256, 0, s>>>(src, idx, n, dst);
    return cudaGetLastError();
}

cudaError_t launch_vsum(unsigned long long *const *accs, int nparts, cudaStream_t s) {
    AccPtrs p{};
    for (int q = 0; q < nparts && q < 64; ++q) p.p[q] = accs[q];
    k_vsum<<<1, 128, 0, s>>>(p, nparts);
    return cudaGetLastError();
}

cudaError_t launch_extract_rows(const int64_t *slice_off, const uint8_t *row_len,
                                const int32_t *col, const double *val, const int64_t *rows,
                                int64_t n, int32_t *out_col, double *out_val,
                                int32_t *out_len, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    k_extract_rows<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(slice_off, row_len, col, val,
                                                               rows, n, out_col, out_val,
                                                               out_len);
    return cudaGetLastError();
}

}  // namespace minife
