// kernels.cu — sm_100a kernels of the MiniFE CG hot path.
//
// Arithmetic contract (C0-C6): binary64, round-to-nearest-even, every product
// and sum written with __dmul_rn/__dadd_rn/__dsub_rn (never contracted to FMA; the library
// is also built with -fmad=false), subnormals kept.  Dots are exactly rounded (exact.cuh).
//
// Layout: rows = owned nodes (owned-box order), columns = extended box
// (owned + one-node halo shell).  All matrix formats are SELL-32: slice s = rows 32s..32s+31,
// stored k-major so a warp's load of entry k is one contiguous 256 B (val) / 128 B (index)
// segment.  Entries of a row are kept in ascending GLOBAL column (C4 order); absent/padding
// entries are never added (row-length predicate or presence mask).
//
// Sections, in file order:
//   helpers (cache policies, coordinates)          a0.2-a0.5 assembly (CRS/SEG/SYM, SYM ghost rows)
//   a2 SpMV: CRS / SEG register kernels, k_spmv_tma (SEG/CRS/fused), k_spmv_sym, k_spmv_symm
//   a3-a6: init, K6 (k_update_xr), single-launch solvers (k_cg_small, k_cg_cluster),
//          K7 (k_update_p, k_update_p2 + k_x2_finish), halo (k_pack_next_p, k_push),
//          fused scheme (k_update_r, k_cg_finish)
//   probes (read / copy / L2), k_move, k_vsum, k_dot, k_acc_round, k_extract_rows
//   host launchers (occupancy, grids, format / scheme dispatch)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "exact.cuh"
#include "kernels.h"

namespace minife {

static void query_occupancy();
static int g_sms = 0;                      // SMs of the current device (occupancy queries)
static int g_spmv_bps[2] = {0, 0};
static int g_upd_bps = 0, g_updp_bps = 0, g_updr_bps = 0;
double g_l2_read_gbs = 0.0;                // last probe_bandwidth: L2-resident TMA read rate

// opt a kernel into > 48 KB dynamic shared memory, once per device
template <class K>
static cudaError_t ensure_smem_attr(K kernel, int bytes, unsigned long long &mask) {
    int dev = 0;
    cudaGetDevice(&dev);
    if ((mask >> (dev & 63)) & 1ull) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) mask |= 1ull << (dev & 63);
    return e;
}

// ----------------------------------------------------------------------------------------
// small helpers
// ----------------------------------------------------------------------------------------

#ifdef SYMM_TRACE
// Diagnostic builds only (tools/build_flags.sh NAME -DSYMM_TRACE): per-CTA %globaltimer
// stamps of the last SYMM launch, read with minife_dbg_symm_trace
__device__ unsigned long long g_symm_trace[1024 * 8];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define SYMM_STAMP(i) g_symm_trace[blockIdx.x * 8 + (i)] = gtime()
extern "C" int minife_dbg_symm_trace(unsigned long long *out, int n) {
    return (int)cudaMemcpyFromSymbol(out, g_symm_trace, 8 * (size_t)n);
}
// per iteration k < 256 and kernel kind (0 SpMV, 1 K6, 2 K7): earliest CTA entry, latest exit
__device__ unsigned long long g_kt[256 * 3 * 2];
struct KtScope {
    int i;
    __device__ KtScope(int kind, int k) : i(((k & 255) * 3 + kind) * 2) {
        if (threadIdx.x == 0) atomicMin(&g_kt[i], gtime());
    }
    __device__ ~KtScope() {
        if (threadIdx.x == 0) atomicMax(&g_kt[i + 1], gtime());
    }
};
#define KT_SCOPE(kind, k) KtScope kt_scope_((kind), (k))
__device__ unsigned long long g_k6_trace[2048 * 16];
#define K6_STAMP(i)                                                                   \
    do {                                                                              \
        if (threadIdx.x == 0 && blockIdx.x < 2048) g_k6_trace[blockIdx.x * 16 + (i)] = gtime(); \
    } while (0)
extern "C" int minife_dbg_k6_trace(unsigned long long *out, int n) {
    return (int)cudaMemcpyFromSymbol(out, g_k6_trace, 8 * (size_t)n);
}
extern "C" int minife_dbg_kt(unsigned long long *out, int reset) {
    if (reset) {
        static unsigned long long h[256 * 3 * 2];
        for (int j = 0; j < 256 * 3 * 2; ++j) h[j] = (j & 1) ? 0ull : ~0ull;
        return (int)cudaMemcpyToSymbol(g_kt, h, sizeof h);
    }
    return (int)cudaMemcpyFromSymbol(out, g_kt, 8 * 256 * 3 * 2);
}
#else
#define SYMM_STAMP(i) ((void)0)
#define KT_SCOPE(kind, k) ((void)0)
#define K6_STAMP(i) ((void)0)
#endif
#ifdef FLUSH_STATS
extern "C" int minife_dbg_flush_stats(unsigned long long *out, int reset) {
    if (reset) {
        unsigned long long z[8] = {0};
        return (int)cudaMemcpyToSymbol(g_flush_stats, z, sizeof z);
    }
    return (int)cudaMemcpyFromSymbol(out, g_flush_stats, sizeof(unsigned long long) * 8);
}
#endif
#ifdef EXP_STATS
extern "C" int minife_dbg_exp_stats(unsigned long long *out, int reset) {
    if (reset) {
        const unsigned long long z[4] = {0, 0, 0, 0};
        return (int)cudaMemcpyToSymbol(g_exp_stats, z, sizeof z);
    }
    return (int)cudaMemcpyFromSymbol(out, g_exp_stats, sizeof(unsigned long long) * 4);
}
#endif

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
__device__ __forceinline__ unsigned ld_stream(const uint32_t *p, uint64_t pol) {
    unsigned v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
        : "=r"(v) : "l"(p), "l"(pol));
    return v;
}

// P:36 boundary: every surface node is constrained; value 1 on the plane x = 1 (G4).
__device__ __forceinline__ bool on_boundary(int ix, int iy, int iz, int nx, int ny, int nz) {
    return ix == 0 || ix == nx || iy == 0 || iy == ny || iz == 0 || iz == nz;
}

// owned row l -> owned-box coordinates (32-bit arithmetic: a part has < 2^31 rows)
__device__ __forceinline__ void row_coords(const Geom &g, int64_t l, int &lx, int &ly, int &lz) {
    const unsigned u = (unsigned)l;
    const unsigned line = u / (unsigned)g.own_n[0];
    lx = (int)(u - line * (unsigned)g.own_n[0]);
    const unsigned plane = line / (unsigned)g.own_n[1];
    ly = (int)(line - plane * (unsigned)g.own_n[1]);
    lz = (int)plane;
}

// extended-box column c -> owned row, or -1 for a halo node
__device__ __forceinline__ int64_t col_to_row(const Geom &g, int64_t c) {
    const unsigned u = (unsigned)c;
    const unsigned line = (unsigned)__umul64hi((unsigned long long)u, g.ext_mag[0]);
    const int ex = (int)(u - line * (unsigned)g.ext_n[0]);
    const unsigned plane = (unsigned)__umul64hi((unsigned long long)line, g.ext_mag[1]);
    const int ey = (int)(line - plane * (unsigned)g.ext_n[1]), ez = (int)plane;
    const int lx = ex - g.off[0], ly = ey - g.off[1], lz = ez - g.off[2];
    if (lx < 0 || lx >= g.own_n[0] || ly < 0 || ly >= g.own_n[1] || lz < 0 || lz >= g.own_n[2])
        return -1;
    return (int64_t)lx + (int64_t)g.own_n[0] * ((int64_t)ly + (int64_t)g.own_n[1] * lz);
}

// owned row l -> extended-box column
__device__ __forceinline__ int64_t row_to_col(const Geom &g, int64_t l) {
    int lx, ly, lz;
    row_coords(g, l, lx, ly, lz);
    return (int64_t)(lx + g.off[0]) +
           (int64_t)g.ext_n[0] * ((int64_t)(ly + g.off[1]) + (int64_t)g.ext_n[1] * (lz + g.off[2]));
}

// ----------------------------------------------------------------------------------------
// a0.2: row lengths and SELL slice widths (CRS format)
// ----------------------------------------------------------------------------------------

// Row length of node (ix,iy,iz) = c(ix) c(iy) c(iz), c = 2 on a boundary plane else 3
// (Fig 3.6's in-range count, closed form).
__global__ void k_rowlen_widths(Geom g, uint8_t *row_len, uint8_t *width, int64_t nslices) {
    const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t slice = row >> 5;
    if (slice >= nslices) return;
    int len = 0;
    if (row < g.rows) {
        int lx, ly, lz;
        row_coords(g, row, lx, ly, lz);
        const int ix = g.own_lo[0] + lx, iy = g.own_lo[1] + ly, iz = g.own_lo[2] + lz;
        const int cx = (ix == 0 || ix == g.nx) ? 2 : 3;
        const int cy = (iy == 0 || iy == g.ny) ? 2 : 3;
        const int cz = (iz == 0 || iz == g.nz) ? 2 : 3;
        len = cx * cy * cz;
    }
    row_len[row] = (uint8_t)len;        // padding lanes of the last slice: 0
    const int w = __reduce_max_sync(0xffffffffu, (unsigned)len);
    if ((threadIdx.x & 31) == 0) width[slice] = (uint8_t)w;
}

// ----------------------------------------------------------------------------------------
// a0.3 + a0.4 + a0.5: element operator, gather-assembly, Dirichlet elimination
// ----------------------------------------------------------------------------------------

constexpr uint32_t SYM_FULL_MASK = (1u << 27) - 1;        // all 27 stencil slots present

// C1: K(d) for one of the 8 difference patterns d = dx | dy<<1 | dz<<2 of an (hx,hy,hz) brick.
__device__ double element_operator_d(int nx, int ny, int nz, int d) {
    const double h[3] = {__ddiv_rn(1.0, (double)nx), __ddiv_rn(1.0, (double)ny),
                         __ddiv_rn(1.0, (double)nz)};
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
    return __dadd_rn(__dadd_rn(T[0], T[1]), T[2]);
}

// C1 + C2 table of a CTA: sKc[d][c] = fold from +0.0 of c copies of K(d), c = 0..8; one
// pattern per thread (threads 0..7)
__device__ __forceinline__ void assembly_table(const Geom &g, double (*sKc)[9]) {
    if (threadIdx.x < 8) {
        const double K = element_operator_d(g.nx, g.ny, g.nz, threadIdx.x);
        double v = 0.0;
        sKc[threadIdx.x][0] = v;
        for (int q = 1; q <= 8; ++q) sKc[threadIdx.x][q] = v = __dadd_rn(v, K);
    }
    __syncthreads();
}

// The 27 slot values of a row none of whose stencil nodes is on the boundary (deep interior):
// no Dirichlet elimination touches it and every c(i,j) is 8 / 4 / 2 / 1 (two elements per
// axis), so slot t holds sKc[d(t)][c(t)] -- the same entries the general loop produces.
__device__ __forceinline__ void interior_table(const double (*sKc)[9], double *sInt) {
    if (threadIdx.x < 27) {
        const int t = threadIdx.x;
        const int dx = t % 3 - 1, dy = (t / 3) % 3 - 1, dz = t / 9 - 1;
        const int c = (dx ? 1 : 2) * (dy ? 1 : 2) * (dz ? 1 : 2);
        sInt[t] = sKc[(dx != 0) | ((dy != 0) << 1) | ((dz != 0) << 2)][c];
    }
    __syncthreads();
}

// One thread per local row (all 32 lanes of the last slice run: padding lanes write the
// slice's padding).  Entry (i,j) = fold from +0.0 of K(d(i,j)) over the c(i,j) elements that
// share nodes i and j (C2: every term is the same K(d); c = per-axis product of 1 where the
// coordinates differ, else the number of elements on that axis containing i).  Then C3:
// constrained row -> identity row, b = v; free row -> for constrained columns in ascending
// global order b = fl(b - fl(A v)), then A = +0.0.  The pattern (incl. zeros) is kept.
__global__ void k_assemble(AsmArgs a) {
    const Geom &g = a.g;
    // C1 and C2's folds of c copies of K(d) (c = 0..8) as a table, once per CTA; the grid is
    // a few CTAs per SM looping over the rows, so the divisions are not paid per 256 rows
    __shared__ double sKc[8][9], sInt[27];
    assembly_table(g, sKc);
    interior_table(sKc, sInt);
    const int64_t nslices = (g.rows + 31) >> 5;
    for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; (row >> 5) < nslices;
         row += (int64_t)gridDim.x * blockDim.x) {
    const int lane = (int)(row & 31);
    // CRS: row slice; SEG/SYM: storage position of the row's slice (interior-first order)
    const int64_t s = (a.fmt != FMT_CRS && a.slice_pos) ? (int64_t)a.slice_pos[row >> 5]
                                                        : (row >> 5);
    if (row >= g.rows) {                           // padding lanes of the last slice
        if (a.fmt == FMT_CRS) {
            const int64_t base = a.slice_off[s] + lane;
            const int w = (int)((a.slice_off[s + 1] - a.slice_off[s]) >> 5);
            for (int k = 0; k < w; ++k) {
                a.col[base + 32 * k] = 0;
                a.val[base + 32 * k] = 0.0;
            }
        } else {
            const int nslot = a.fmt == FMT_SYM ? 14 : 27;
            for (int t = 0; t < nslot; ++t) a.val[(nslot * s + t) * 32 + lane] = 0.0;
            for (int j = 0; j < 9; ++j) a.seg[(9 * s + j) * 32 + lane] = 0;
            a.mask[s * 32 + lane] = 0u;            // mask is padded to 32 * slices
        }
        continue;
    }
    // value slot t of this row: SEG stores all 27 stencil slots, SYM the upper slots t >= 13
    // (both SELL-32, k-major)
    const bool sym = a.fmt == FMT_SYM;
    auto vptr = [&](int t) -> double * {
        return sym ? a.val + (14 * s + (t - 13)) * 32 + lane : a.val + (27 * s + t) * 32 + lane;
    };
    int lx, ly, lz;
    row_coords(g, row, lx, ly, lz);
    const int ix = g.own_lo[0] + lx, iy = g.own_lo[1] + ly, iz = g.own_lo[2] + lz;
    // extended-box coordinates of the row's node
    const int ex = lx + g.off[0], ey = ly + g.off[1], ez = lz + g.off[2];
    // deep interior (no stencil node on the boundary): constant values, all 27 slots, b = 0
    // -- the general loop below gives exactly these; ~96 % of the rows at 300^3, so the
    // kernel stays bound by its stores rather than by this loop's instructions
    if (a.fmt != FMT_CRS && ix >= 2 && ix <= g.nx - 2 && iy >= 2 && iy <= g.ny - 2 && iz >= 2 &&
        iz <= g.nz - 2) {
        const int64_t E0 = g.ext_n[0], E01 = (int64_t)g.ext_n[0] * g.ext_n[1];
        const int64_t c0 = (int64_t)(ex - 1) + E0 * ey + E01 * ez;
#pragma unroll
        for (int j = 0; j < 9; ++j)
            a.seg[(9 * s + j) * 32 + lane] = (int32_t)(c0 + E0 * (j % 3 - 1) + E01 * (j / 3 - 1));
#pragma unroll
        for (int t = sym ? 13 : 0; t < 27; ++t) *vptr(t) = sInt[t];
        a.mask[s * 32 + lane] = SYM_FULL_MASK;
        a.b[row] = 0.0;
        continue;
    }
    const bool row_bc = on_boundary(ix, iy, iz, g.nx, g.ny, g.nz);
    const int n_el[3] = {(ix > 0) + (ix < g.nx), (iy > 0) + (iy < g.ny), (iz > 0) + (iz < g.nz)};
    double b = 0.0;
    int k = 0;                                     // CRS entry counter
    uint32_t mask = 0;
    for (int dz = -1; dz <= 1; ++dz) {
        for (int dy = -1; dy <= 1; ++dy) {
            const int jgrp = (dz + 1) * 3 + (dy + 1);
            const int jy = iy + dy, jz = iz + dz;
            const bool grp_in = jy >= 0 && jy <= g.ny && jz >= 0 && jz <= g.nz;
            // run start: extended column of (x-1, y+dy, z+dz); never dereferenced when the
            // dx = -1 slot is absent
            const int64_t start = (int64_t)(ex - 1) +
                                  (int64_t)g.ext_n[0] * ((int64_t)(ey + dy) +
                                                         (int64_t)g.ext_n[1] * (ez + dz));
            if (a.fmt != FMT_CRS) a.seg[(9 * s + jgrp) * 32 + lane] = grp_in ? (int32_t)start : 0;
            for (int dx = -1; dx <= 1; ++dx) {
                const int t = jgrp * 3 + (dx + 1);
                const int jx = ix + dx;
                const bool in = grp_in && jx >= 0 && jx <= g.nx;
                if (!in) {
                    if (a.fmt == FMT_SEG || (sym && t >= 13)) *vptr(t) = 0.0;
                    continue;
                }
                const int c = (dx ? 1 : n_el[0]) * (dy ? 1 : n_el[1]) * (dz ? 1 : n_el[2]);
                double v = sKc[(dx != 0) | ((dy != 0) << 1) | ((dz != 0) << 2)][c];
                if (row_bc) {
                    v = (dx == 0 && dy == 0 && dz == 0) ? 1.0 : 0.0;
                } else if (on_boundary(jx, jy, jz, g.nx, g.ny, g.nz)) {
                    const double bv = (jx == g.nx) ? 1.0 : 0.0;
                    b = __dsub_rn(b, __dmul_rn(v, bv));
                    v = 0.0;
                }
                if (a.fmt == FMT_CRS) {
                    const int64_t base = a.slice_off[s] + lane;
                    a.col[base + 32 * k] = (int32_t)(start + dx + 1);
                    a.val[base + 32 * k] = v;
                } else {
                    if (!sym || t >= 13) *vptr(t) = v;   // SYM: lower half is mirrored
                    mask |= 1u << t;
                }
                ++k;
            }
        }
    }
    if (a.fmt == FMT_CRS) {
        const int64_t base = a.slice_off[s] + lane;
        const int w = (int)((a.slice_off[s + 1] - a.slice_off[s]) >> 5);
        const int32_t own = (int32_t)((int64_t)ex + (int64_t)g.ext_n[0] *
                                      ((int64_t)ey + (int64_t)g.ext_n[1] * ez));
        for (int kk = k; kk < w; ++kk) {           // padding: own column, value 0
            a.col[base + 32 * kk] = own;
            a.val[base + 32 * kk] = 0.0;
        }
    } else {
        a.mask[s * 32 + lane] = mask;
    }
    if (row_bc) b = (ix == g.nx) ? 1.0 : 0.0;
    a.b[row] = b;
    }
}

// a0.2-a0.5 for FMT_SYM on a part with a halo: one thread per EXTENDED-box node (storage
// row = its column).  Same C1-C3 arithmetic as k_assemble; only the upper slots t >= 13 are
// stored.  A halo (ghost) node gets its upper entries towards nodes inside the extended box
// -- exactly the mirrors the owned rows read; slots leaving the extended box are absent.
// mask bit 31 marks owned nodes; b is written for owned rows only.
__global__ void k_assemble_symx(AsmArgs a) {
    const Geom &g = a.g;
    // C1 and C2's fold table once per CTA; grid-stride over the extended box (as k_assemble)
    __shared__ double sKc[8][9], sInt[27];
    assembly_table(g, sKc);
    interior_table(sKc, sInt);
    const int64_t nslices = (g.ncols + 31) >> 5;
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; (c >> 5) < nslices;
         c += (int64_t)gridDim.x * blockDim.x) {
    const int lane = (int)(c & 31);
    const int64_t s = c >> 5;
    if (c >= g.ncols) {                            // padding lanes of the last slice
        for (int t = 0; t < 14; ++t) a.val[(14 * s + t) * 32 + lane] = 0.0;
        for (int j = 0; j < 9; ++j) a.seg[(9 * s + j) * 32 + lane] = 0;
        a.mask[c] = 0u;
        continue;
    }
    const unsigned u = (unsigned)c;
    const unsigned line = u / (unsigned)g.ext_n[0];
    const int ex = (int)(u - line * (unsigned)g.ext_n[0]);
    const unsigned plane = line / (unsigned)g.ext_n[1];
    const int ey = (int)(line - plane * (unsigned)g.ext_n[1]), ez = (int)plane;
    const int ix = g.ext_lo[0] + ex, iy = g.ext_lo[1] + ey, iz = g.ext_lo[2] + ez;
    const int64_t row = col_to_row(g, c);
    // deep interior and all 26 neighbours inside the extended box: constants (as k_assemble)
    if (ix >= 2 && ix <= g.nx - 2 && iy >= 2 && iy <= g.ny - 2 && iz >= 2 && iz <= g.nz - 2 &&
        ex >= 1 && ex <= g.ext_n[0] - 2 && ey >= 1 && ey <= g.ext_n[1] - 2 && ez >= 1 &&
        ez <= g.ext_n[2] - 2) {
        const int64_t E0 = g.ext_n[0], E01 = (int64_t)g.ext_n[0] * g.ext_n[1];
        const int64_t c0 = (int64_t)(ex - 1) + E0 * ey + E01 * ez;
#pragma unroll
        for (int j = 0; j < 9; ++j)
            a.seg[(9 * s + j) * 32 + lane] = (int32_t)(c0 + E0 * (j % 3 - 1) + E01 * (j / 3 - 1));
#pragma unroll
        for (int t = 13; t < 27; ++t) a.val[(14 * s + (t - 13)) * 32 + lane] = sInt[t];
        a.mask[c] = SYM_FULL_MASK | (row >= 0 ? SYM_OWNED : 0u);
        if (row >= 0) a.b[row] = 0.0;
        continue;
    }
    const bool row_bc = on_boundary(ix, iy, iz, g.nx, g.ny, g.nz);
    const int n_el[3] = {(ix > 0) + (ix < g.nx), (iy > 0) + (iy < g.ny), (iz > 0) + (iz < g.nz)};
    double b = 0.0;
    uint32_t mask = row >= 0 ? SYM_OWNED : 0u;
    for (int dz = -1; dz <= 1; ++dz) {
        for (int dy = -1; dy <= 1; ++dy) {
            const int jgrp = (dz + 1) * 3 + (dy + 1);
            const int jy = iy + dy, jz = iz + dz;
            const bool grp_in = jy >= 0 && jy <= g.ny && jz >= 0 && jz <= g.nz;
            const int64_t start = (int64_t)(ex - 1) +
                                  (int64_t)g.ext_n[0] * ((int64_t)(ey + dy) +
                                                         (int64_t)g.ext_n[1] * (ez + dz));
            a.seg[(9 * s + jgrp) * 32 + lane] = grp_in ? (int32_t)start : 0;
            for (int dx = -1; dx <= 1; ++dx) {
                const int t = jgrp * 3 + (dx + 1);
                const int jx = ix + dx;
                // inside the domain AND inside the extended box (ghost rows stop at its edge)
                const bool in = grp_in && jx >= 0 && jx <= g.nx && ex + dx >= 0 &&
                                ex + dx < g.ext_n[0] && ey + dy >= 0 && ey + dy < g.ext_n[1] &&
                                ez + dz >= 0 && ez + dz < g.ext_n[2];
                if (!in) {
                    if (t >= 13) a.val[(14 * s + (t - 13)) * 32 + lane] = 0.0;
                    continue;
                }
                const int cnt = (dx ? 1 : n_el[0]) * (dy ? 1 : n_el[1]) * (dz ? 1 : n_el[2]);
                double v = sKc[(dx != 0) | ((dy != 0) << 1) | ((dz != 0) << 2)][cnt];
                if (row_bc) {
                    v = (dx == 0 && dy == 0 && dz == 0) ? 1.0 : 0.0;
                } else if (on_boundary(jx, jy, jz, g.nx, g.ny, g.nz)) {
                    const double bv = (jx == g.nx) ? 1.0 : 0.0;
                    b = __dsub_rn(b, __dmul_rn(v, bv));
                    v = 0.0;
                }
                if (t >= 13) a.val[(14 * s + (t - 13)) * 32 + lane] = v;
                mask |= 1u << t;
            }
        }
    }
    a.mask[c] = mask;
    if (row >= 0) a.b[row] = row_bc ? ((ix == g.nx) ? 1.0 : 0.0) : b;
    }
}

// ----------------------------------------------------------------------------------------
// Device-initiated communication (DevComm, kernels.h): release/acquire flags at
// system scope, payloads stored straight into the receiver's region.
// ----------------------------------------------------------------------------------------

static_assert(ACC_WORDS == 72, "comm_words() assumes 72-word accumulators");

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned long long comm_gen(const DevComm &dc) {
    return *(volatile const unsigned long long *)dc.local;
}

// Spin until *flag >= seq.  A peer that never signals (dead rank, broken mapping) ends the
// wait after dc.timeout_ns: the error is recorded in the region and in the CG state (status 9
// -> MINIFE_ECOMM), and every later kernel of the solve returns at its done test.
__device__ bool comm_spin(const DevComm &dc, const unsigned long long *flag,
                          unsigned long long seq, CgState *st) {
    if (ld_acquire_sys(flag) >= seq) return true;
    const unsigned long long t0 = global_ns();
    while (ld_acquire_sys(flag) < seq) {
        if (*(volatile const unsigned long long *)(dc.local + 2)) return false;
        __nanosleep(100);
        if (global_ns() - t0 > (unsigned long long)dc.timeout_ns) {
            atomicExch(dc.local + 2, 1ull);
            st->status = 9;
            st->done = 1;
            __threadfence();
            return false;
        }
    }
    return true;
}

// The all-reduced accumulator `which` (0 pAp_k, 1 rr_k) into shared memory: the local words
// (one part, or all-reduced by the host-launched transport) or, with device comm, the int64
// sum over every rank's inbox slot (two's-complement sums: the same value an int64-SUM
// all-reduce produces, independent of the rank order).  Block-uniform; false on a timeout.
__device__ bool acc_in_load(unsigned long long *s_in, const UpdArgs &a, int k, int which) {
    const DevComm &dc = a.dc;
    if (!dc.local) {
        acc_load_shared(s_in, a.acc_in);
        return true;
    }
    __shared__ int s_ok;
    const unsigned long long gen = comm_gen(dc);
    const int gp = (int)(gen & 1);
    const unsigned long long seq = comm_seq(gen, k, which);
    if (threadIdx.x == 0) s_ok = 1;
    __syncthreads();
    for (int t = threadIdx.x; t < dc.world; t += blockDim.x)
        if (!comm_spin(dc, dc.local + comm_acc_flag(dc.world, gp, which, t), seq, a.st)) s_ok = 0;
    __syncthreads();
    if (!s_ok) return false;
    const unsigned long long *in =
        dc.local + comm_inbox(dc.world) + (int64_t)(2 * gp + which) * dc.world * ACC_WORDS;
    for (int i = threadIdx.x; i < ACC_WORDS; i += blockDim.x) {
        unsigned long long sum = 0ull;
        for (int t = 0; t < dc.world; ++t) sum += __ldcv(in + (int64_t)t * ACC_WORDS + i);
        s_in[i] = sum;
    }
    return true;
}

// Reduction `which` of iteration k: this part's accumulator into slot `rank` of every rank's
// inbox (its own included), then one release flag per rank.  Slot reuse is safe with two
// generation parities x {pAp, rr}: a rank writes reduction n+2 only after it has consumed
// n+1, which needs every rank's contribution to n+1, which each rank stores only after it has
// consumed n (stream order); a new solve (next generation) uses the other parity.
// The push itself (one CTA): the words of `acc` into slot `rank` of every rank's inbox, a
// system-scope fence, then one release flag per rank.
__device__ void acc_push_body(const DevComm &dc, const unsigned long long *acc, int k, int which) {
    if (dc.mute) return;                         // fault injection: a rank that never signals
    const unsigned long long gen = comm_gen(dc);
    const int gp = (int)(gen & 1);
    const int64_t off =
        comm_inbox(dc.world) + ((int64_t)(2 * gp + which) * dc.world + dc.rank) * ACC_WORDS;
    for (int i = threadIdx.x; i < ACC_WORDS; i += blockDim.x) {
        const unsigned long long w = __ldcg(acc + i);
        for (int t = 0; t < dc.world; ++t) dc.region[t][off + i] = w;
    }
    // one system-scope fence after the CTA barrier covers every thread's stores (fences are
    // cumulative over writes observed through bar.sync; the flag stores are releases too)
    __syncthreads();
    if (threadIdx.x == 0) __threadfence_system();
    __syncthreads();
    const unsigned long long seq = comm_seq(gen, k, which);
    for (int t = threadIdx.x; t < dc.world; t += blockDim.x)
        st_release_sys(dc.region[t] + comm_acc_flag(dc.world, gp, which, dc.rank), seq);
}

__global__ void k_acc_push(UpdArgs a, int k, int which, const unsigned long long *acc) {
    if (k > 0 && a.st->done) return;     // k = 0 (rr_0): the state is not initialised yet
    acc_push_body(a.dc, acc, k, which);
}

// The same push folded into the kernel that produced the accumulator: every CTA, after its
// atomics into `acc`, takes a ticket; the last CTA (all others' atomics are then visible at
// gpu scope) pushes.  Saves a launch per reduction.  All threads of the CTA call it.
__device__ void acc_push_last_cta(const DevComm &dc, const unsigned long long *acc, int k,
                                  int which, unsigned long long *ticket) {
    __shared__ int s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();                   // this CTA's atomics into acc, before the ticket
        s_last = atomicAdd(ticket, 1ull) == (unsigned long long)(gridDim.x - 1);
        if (s_last) __threadfence();
    }
    __syncthreads();
    if (!s_last) return;
    acc_push_body(dc, acc, k, which);
    if (threadIdx.x == 0) *ticket = 0ull;
}



// ----------------------------------------------------------------------------------------
// a2: SpMV  y = A x  (+ exact pAp epilogue)
// ----------------------------------------------------------------------------------------

// C4 per row: s = +0.0; for stored entries in ascending global column, s = fl(s + fl(a x));
// absent / padding entries are skipped by predicate (a -0.0 row sum stays -0.0).
// One warp per slice, one lane per row; warps walk the slices grid-stride so each thread's
// expansion absorbs many rows before the single flush.

// CRS format (Fig 3.1 on SELL-32): 12 B per stored entry.
template <bool DOT, bool IDENT>
__global__ void __launch_bounds__(SPMV_THREADS) k_spmv_crs(SpmvArgs a) {
    __shared__ unsigned long long sacc[ACC_WORDS];
    __shared__ int sdig[ACC_DIG16];
    if (DOT) {
        if (a.st && a.st->done) return;
        acc_zero_shared(sacc, sdig);
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
    const Matrix &m = a.m;
    for (int64_t s = a.s_begin + (int64_t)blockIdx.x * warps_per_block + (threadIdx.x >> 5);
         s < a.s_end; s += nw) {
        const int64_t off = m.slice_off[s];
        const int w = (int)((m.slice_off[s + 1] - off) >> 5);
        const int64_t row = s * 32 + lane;
        const int len = (row < m.rows) ? (int)m.row_len[row] : 0;
        const double *v = m.val + off + lane;
        const int32_t *c = m.col + off + lane;
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
        if (row < m.rows) {
            a.y[row] = sum;
            if (DOT) {
                const double pr = __ldg(a.x + (IDENT ? row : row_to_col(a.g, row)));
                ex.add(__dmul_rn(pr, sum), sacc);
            }
        }
    }
    if (DOT) {
        expansion_flush_digits(ex, sdig, sacc);
        __syncthreads();
        acc_merge_to_global(sacc, sdig, a.acc);
    }
}

// Segment format (the paper's BCRS, Fig 3.2, on SELL-32): per row 27 value slots in stencil
// order (dz, dy, dx), one int32 start column per x-run (dz, dy) and a 27-bit presence mask:
// entry t = 3j + e has column seg[j] + e.  8 B per stored value + 4 B per segment.
template <bool DOT>
__global__ void __launch_bounds__(SPMV_THREADS) k_spmv_seg(SpmvArgs a) {
    __shared__ unsigned long long sacc[ACC_WORDS];
    __shared__ int sdig[ACC_DIG16];
    if (DOT) {
        if (a.st && a.st->done) return;
        acc_zero_shared(sacc, sdig);
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
    const Matrix &m = a.m;
    for (int64_t s = a.s_begin + (int64_t)blockIdx.x * warps_per_block + (threadIdx.x >> 5);
         s < a.s_end; s += nw) {
        const int64_t row = (m.slice_row ? (int64_t)m.slice_row[s] : s) * 32 + lane;
        const bool live = row < m.rows;
        const unsigned msk = live ? ld_stream(m.mask + s * 32 + lane, pol) : 0u;
        const int32_t *sp = m.seg + 9 * s * 32 + lane;
        const double *vp = m.val + 27 * s * 32 + lane;
        int st[9];
#pragma unroll
        for (int j = 0; j < 9; ++j) st[j] = ld_stream(sp + 32 * j, pol);
        double vv[27];
#pragma unroll
        for (int t = 0; t < 27; ++t) vv[t] = ld_stream(vp + 32 * t, pol);
        double xv[27];
#pragma unroll
        for (int t = 0; t < 27; ++t)
            xv[t] = ((msk >> t) & 1u) ? __ldg(a.x + st[t / 3] + (t % 3)) : 0.0;
        double sum = 0.0;
#pragma unroll
        for (int t = 0; t < 27; ++t)
            if ((msk >> t) & 1u) sum = __dadd_rn(sum, __dmul_rn(vv[t], xv[t]));
        if (live) {
            a.y[row] = sum;
            if (DOT) ex.add(__dmul_rn(xv[13], sum), sacc);   // slot 13 = the diagonal
        }
    }
    if (DOT) {
        expansion_flush_digits(ex, sdig, sacc);
        __syncthreads();
        acc_merge_to_global(sacc, sdig, a.acc);
    }
}

// ----------------------------------------------------------------------------------------
// a2, TMA-pipelined: the matrix stream is moved by the bulk-copy engine into shared memory
// (cp.async.bulk + mbarrier transaction counts), decoupled from the registers of the warps
// that compute.  Persistent grid, one CTA per SM: warp TMA_WARPS is the producer, warps
// 0..TMA_WARPS-1 consume one slice each per tile.  A tile = TILE consecutive slices, whose
// val / index / mask bytes are contiguous in HBM, so it is 3 bulk copies.
// ----------------------------------------------------------------------------------------

constexpr int TILE = 8;                    // slices per tile (= consumer warps)
constexpr int TMA_WARPS = TILE;
constexpr int TMA_THREADS = 32 * (TMA_WARPS + 1);
constexpr int SEG_STAGES = 3;
constexpr int CRS_STAGES = 2;
// per-stage bytes: SEG = 27 val + 9 seg + 1 mask words per row; CRS = <=27 (val + col) + len
constexpr int SEG_VAL_B = TILE * 27 * 32 * 8, SEG_SEG_B = TILE * 9 * 32 * 4,
              SEG_MSK_B = TILE * 32 * 4;
constexpr int SEG_STAGE_B = SEG_VAL_B + SEG_SEG_B + SEG_MSK_B;          // 65536
constexpr int CRS_VAL_B = TILE * 27 * 32 * 8, CRS_COL_B = TILE * 27 * 32 * 4,
              CRS_LEN_B = TILE * 32;
constexpr int CRS_STAGE_B = CRS_VAL_B + CRS_COL_B + CRS_LEN_B;          // 83200
constexpr int SEG_SMEM = SEG_STAGES * SEG_STAGE_B;
constexpr int CRS_SMEM = CRS_STAGES * CRS_STAGE_B;
template <int FMT> struct TmaCfg;
template <> struct TmaCfg<FMT_SEG> {
    static constexpr int NV = 27, STAGES = SEG_STAGES, STAGE_B = SEG_STAGE_B, SMEM = SEG_SMEM;
};
template <> struct TmaCfg<FMT_CRS> {
    static constexpr int NV = 27, STAGES = CRS_STAGES, STAGE_B = CRS_STAGE_B, SMEM = CRS_SMEM;
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// 1-D bulk copy global -> shared, completion counted on `bar`, evict-first in L2
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

__device__ __forceinline__ int rr_decision(double rr_new, int k, double *hist, double *rr,
                                           CgState *st, double &beta);

// FUSED (SEG, DOT, one part only): fused CG iteration k = a.fused_k, DESIGN.md §5.  The
// prologue takes K7's decisions for iteration k-1 (finalise rr_{k-1}, hist, stop tests,
// beta_{k-1}); the operand gathered for column c is p_k[c] = fl(r[c] + fl(beta p_{k-1}[c]))
// (p_1 = r); p_k and x += fl(alpha_{k-1} p_{k-1}) are written for the own rows.  Values and
// operation order are those of the three-kernel C6 sequence, so results are bit-identical.
template <bool DOT, int FMT, bool IDENT, bool FUSED>
__global__ void __launch_bounds__(TMA_THREADS, 1) k_spmv_tma(SpmvArgs a) {
    constexpr int STAGES = TmaCfg<FMT>::STAGES;
    constexpr int STAGE_B = TmaCfg<FMT>::STAGE_B;
    constexpr int NV = TmaCfg<FMT>::NV;                 // value slots per row in the tile
    constexpr int VAL_B = TILE * NV * 32 * 8;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES];
    __shared__ unsigned long long sacc[ACC_WORDS];
    __shared__ int sdig[ACC_DIG16];
    __shared__ unsigned long long s_in[FUSED ? ACC_WORDS : 1];
    __shared__ double s_beta, s_alpha_prev;
    __shared__ int s_stop;
    if (DOT && a.st && a.st->done) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int fk = FUSED ? a.fused_k : 0;
    if (FUSED && fk >= 2) {
        acc_load_shared(s_in, a.acc_rr_in);
        __syncthreads();
    }
    const double fin = (FUSED && fk >= 2 && threadIdx.x < 32) ? acc_finalize_warp(s_in) : 0.0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], TMA_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        s_stop = 0;
        if (FUSED) {
            double beta = 0.0, alpha_prev = 0.0;
            if (fk >= 2) {
                s_stop = rr_decision(fin, fk - 1, a.hist, a.rr, a.stw, beta);
                alpha_prev = a.stw->alpha;                    // alpha_{k-1} (K6 of k-1)
                if (!s_stop && blockIdx.x == 0) a.stw->x_done = fk - 1;
            }
            s_beta = beta;
            s_alpha_prev = alpha_prev;
        }
    }
    if (DOT) {
        acc_zero_shared(sacc, sdig);
        if (blockIdx.x == 0 && a.acc_zero)
            for (int i = threadIdx.x; i < ACC_WORDS; i += blockDim.x) a.acc_zero[i] = 0ull;
    }
    __syncthreads();
    if (FUSED && s_stop) return;
    const Matrix &m = a.m;
    const int64_t sb = a.s_begin, se = a.s_end;        // storage slices of this launch
    const int64_t ntiles = (se - sb + TILE - 1) / TILE;

    if (warp == TMA_WARPS) {
        // ---------------- producer: one elected lane issues the bulk copies -------------
        if (lane == 0) {
            const uint64_t pol = evict_first_policy();
            int64_t i = 0;
            for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++i) {
                const int st = (int)(i % STAGES);
                if (i >= STAGES) mbar_wait(&empty_bar[st], (uint32_t)(((i / STAGES) & 1) ^ 1));
                const int64_t s0 = sb + tile * TILE;
                const int64_t rem = se - s0;
                const int nsl = rem < TILE ? (int)rem : TILE;
                unsigned char *buf = smem + (size_t)st * STAGE_B;
                if (FMT != FMT_CRS) {
                    const uint32_t bv = nsl * NV * 32 * 8, bs = nsl * 9 * 32 * 4,
                                   bm = nsl * 32 * 4;
                    mbar_expect_tx(&full_bar[st], bv + bs + bm);
                    bulk_g2s(buf, m.val + s0 * NV * 32, bv, &full_bar[st], pol);
                    bulk_g2s(buf + VAL_B, m.seg + s0 * 9 * 32, bs, &full_bar[st], pol);
                    bulk_g2s(buf + VAL_B + SEG_SEG_B, m.mask + s0 * 32, bm, &full_bar[st], pol);
                } else {
                    const int64_t e0 = m.slice_off[s0], e1 = m.slice_off[s0 + nsl];
                    const uint32_t ne = (uint32_t)(e1 - e0);
                    const uint32_t bv = ne * 8, bc = ne * 4, bl = nsl * 32;
                    mbar_expect_tx(&full_bar[st], bv + bc + bl);
                    bulk_g2s(buf, m.val + e0, bv, &full_bar[st], pol);
                    bulk_g2s(buf + CRS_VAL_B, m.col + e0, bc, &full_bar[st], pol);
                    bulk_g2s(buf + CRS_VAL_B + CRS_COL_B, m.row_len + s0 * 32, bl, &full_bar[st],
                             pol);
                }
            }
        }
    } else {
        // ---------------- consumers: one slice per warp per tile, operands from smem -----
        Expansion ex;
        ex.init();
        int64_t i = 0;
        for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++i) {
            const int st = (int)(i % STAGES);
            mbar_wait(&full_bar[st], (uint32_t)((i / STAGES) & 1));
            const int64_t s = sb + tile * TILE + warp;        // storage slice
            if (s < se) {
                const unsigned char *buf = smem + (size_t)st * STAGE_B;
                const int64_t row = (m.slice_row ? (int64_t)m.slice_row[s] : s) * 32 + lane;
                double sum = 0.0, pdiag = 0.0;
                if (FMT != FMT_CRS) {
                    const double *vs = reinterpret_cast<const double *>(buf) + warp * NV * 32 + lane;
                    const int32_t *ss =
                        reinterpret_cast<const int32_t *>(buf + VAL_B) + warp * 9 * 32 + lane;
                    const unsigned msk = reinterpret_cast<const uint32_t *>(
                        buf + VAL_B + SEG_SEG_B)[warp * 32 + lane];
                    int sg[9];
#pragma unroll
                    for (int j = 0; j < 9; ++j) sg[j] = ss[32 * j];
                    double xv[27];
                    if (!FUSED) {
#pragma unroll
                        for (int t = 0; t < 27; ++t)
                            xv[t] = ((msk >> t) & 1u) ? __ldg(a.x + sg[t / 3] + (t % 3)) : 0.0;
                    } else if (fk == 1) {
#pragma unroll
                        for (int t = 0; t < 27; ++t)             // p_1 = r_0 (= b), exactly
                            xv[t] = ((msk >> t) & 1u) ? __ldg(a.r + sg[t / 3] + (t % 3)) : 0.0;
                    } else {
                        const double beta = s_beta;
                        double rv[27], pv[27];
#pragma unroll
                        for (int t = 0; t < 27; ++t) {
                            const bool on = (msk >> t) & 1u;
                            const int c = sg[t / 3] + (t % 3);
                            rv[t] = on ? __ldg(a.r + c) : 0.0;
                            pv[t] = on ? __ldg(a.p_old + c) : 0.0;
                        }
#pragma unroll
                        for (int t = 0; t < 27; ++t)             // K7: p = r + fl(beta p)
                            xv[t] = __dadd_rn(rv[t], __dmul_rn(beta, pv[t]));
                        if (row < m.rows)                        // deferred x update (K6, k-1)
                            a.xsol[row] =
                                __dadd_rn(a.xsol[row], __dmul_rn(s_alpha_prev, pv[13]));
                    }
#pragma unroll
                    for (int t = 0; t < 27; ++t)
                        if ((msk >> t) & 1u) sum = __dadd_rn(sum, __dmul_rn(vs[32 * t], xv[t]));
                    pdiag = xv[13];
                    if (FUSED && row < m.rows) a.p_new[row] = pdiag;
                } else {
                    const int64_t e0 = m.slice_off[sb + tile * TILE];
                    const int64_t so = m.slice_off[s] - e0;
                    const int w = (int)((m.slice_off[s + 1] - m.slice_off[s]) >> 5);
                    const double *vs = reinterpret_cast<const double *>(buf) + so + lane;
                    const int32_t *cs = reinterpret_cast<const int32_t *>(buf + CRS_VAL_B) + so + lane;
                    const int len = (buf + CRS_VAL_B + CRS_COL_B)[warp * 32 + lane];
                    if (w == 27) {
                        double xv[27];
#pragma unroll
                        for (int k = 0; k < 27; ++k) xv[k] = k < len ? __ldg(a.x + cs[32 * k]) : 0.0;
#pragma unroll
                        for (int k = 0; k < 27; ++k)
                            if (k < len) sum = __dadd_rn(sum, __dmul_rn(vs[32 * k], xv[k]));
                    } else {
                        for (int k = 0; k < len; ++k)
                            sum = __dadd_rn(sum, __dmul_rn(vs[32 * k], __ldg(a.x + cs[32 * k])));
                    }
                    if (DOT && row < m.rows)
                        pdiag = __ldg(a.x + (IDENT ? row : row_to_col(a.g, row)));
                }
                if (row < m.rows) {
                    a.y[row] = sum;
                    if (DOT) ex.add(__dmul_rn(pdiag, sum), sacc);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty_bar[st]);
        }
        if (DOT) expansion_flush_digits(ex, sdig, sacc);
    }
    if (DOT) {
        __syncthreads();
        acc_merge_to_global(sacc, sdig, a.acc);
        if (a.fold_push) acc_push_last_cta(a.dc, a.acc, a.k, 0, a.dc.local + 3);
    }
}

// ----------------------------------------------------------------------------------------
// a2 in FMT_SYM (one part).  The upper value slots are stored SELL-14 (val[(14 s + u) 32 +
// lane], u = t - 13), so a 16-slice tile is one contiguous bulk copy (plus the run starts and
// masks).  Lower slot t < 13 of row i needs a_ij = a_ji: row j = the slot's column c, mirror
// slot 26 - t, i.e. val[((c >> 5) 14 + 13 - t) 32 + (c & 31)] -- consecutive lanes have
// consecutive c, so each mirrored read is a coalesced 256 B access, served by L2 (row j's
// tile was streamed about one plane earlier).  HBM sees each stored value once.  16 consumer
// warps per SM keep the mirrored and x reads in flight.
// ----------------------------------------------------------------------------------------

// SYM storage row c -> computed row (or -1); clears the presence bits of a ghost row
__device__ __forceinline__ int64_t sym_row(const Matrix &m, const Geom &g, int64_t c,
                                           unsigned &msk) {
    if (!m.ext) return c < m.rows ? c : -1;
    if (!(msk & SYM_OWNED)) {
        msk = 0u;
        return -1;
    }
    msk &= ~SYM_OWNED;
    return col_to_row(g, c);
}

template <int NW, int NST> struct SyCfg {                     // NW slices per tile = consumers
    static constexpr int TILE = NW, THREADS = 32 * (NW + 1), STAGES = NST;
    static constexpr int VAL_B = NW * 14 * 32 * 8, SEG_B = NW * 9 * 32 * 4, MSK_B = NW * 32 * 4;
    static constexpr int STAGE_B = VAL_B + SEG_B + MSK_B, SMEM = NST * STAGE_B;
};

template <bool DOT, int NW, int NST>
__global__ void __launch_bounds__(SyCfg<NW, NST>::THREADS, 1) k_spmv_sym(SpmvArgs a) {
    constexpr int SY_TILE = NW, SY_STAGES = NST;
    constexpr int SY_VAL_B = SyCfg<NW, NST>::VAL_B, SY_SEG_B = SyCfg<NW, NST>::SEG_B;
    constexpr int SY_STAGE_B = SyCfg<NW, NST>::STAGE_B;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t full_bar[SY_STAGES], empty_bar[SY_STAGES];
    __shared__ unsigned long long sacc[ACC_WORDS];
    __shared__ int sdig[ACC_DIG16];
    if (DOT && a.st && a.st->done) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < SY_STAGES; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], SY_TILE);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (DOT) {
        acc_zero_shared(sacc, sdig);
        if (blockIdx.x == 0 && a.acc_zero)
            for (int i = threadIdx.x; i < ACC_WORDS; i += blockDim.x) a.acc_zero[i] = 0ull;
    }
    __syncthreads();
    const Matrix &m = a.m;
    const int64_t ntiles = (m.nslices + SY_TILE - 1) / SY_TILE;

    if (warp == SY_TILE) {
        if (lane == 0) {
            // values are read a second time (mirrored): normal L2 priority; indices: first
            const uint64_t pol = evict_first_policy();
            uint64_t pol_keep;
            asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_keep));
            int64_t i = 0;
            for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++i) {
                const int st = (int)(i % SY_STAGES);
                if (i >= SY_STAGES) mbar_wait(&empty_bar[st], (uint32_t)(((i / SY_STAGES) & 1) ^ 1));
                const int64_t s0 = tile * SY_TILE;
                const int64_t rem = m.nslices - s0;
                const int nsl = rem < SY_TILE ? (int)rem : SY_TILE;
                unsigned char *buf = smem + (size_t)st * SY_STAGE_B;
                const uint32_t bv = nsl * 14 * 32 * 8, bs = nsl * 9 * 32 * 4, bm = nsl * 32 * 4;
                mbar_expect_tx(&full_bar[st], bv + bs + bm);
                bulk_g2s(buf, m.val + s0 * 14 * 32, bv, &full_bar[st], pol_keep);
                bulk_g2s(buf + SY_VAL_B, m.seg + s0 * 9 * 32, bs, &full_bar[st], pol);
                bulk_g2s(buf + SY_VAL_B + SY_SEG_B, m.mask + s0 * 32, bm, &full_bar[st], pol);
            }
        }
    } else {
        Expansion ex;
        ex.init();
        int64_t i = 0;
        for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++i) {
            const int st = (int)(i % SY_STAGES);
            mbar_wait(&full_bar[st], (uint32_t)((i / SY_STAGES) & 1));
            const int64_t s = tile * SY_TILE + warp;
            if (s < m.nslices) {
                const unsigned char *buf = smem + (size_t)st * SY_STAGE_B;
                const double *vs = reinterpret_cast<const double *>(buf) + warp * 14 * 32 + lane;
                const int32_t *ss =
                    reinterpret_cast<const int32_t *>(buf + SY_VAL_B) + warp * 9 * 32 + lane;
                unsigned msk =
                    reinterpret_cast<const uint32_t *>(buf + SY_VAL_B + SY_SEG_B)[warp * 32 + lane];
                // storage row s*32+lane; SYM-ext: only owned nodes are computed rows
                const int64_t row = sym_row(m, a.g, s * 32 + lane, msk);
                int sg[9];
#pragma unroll
                for (int j = 0; j < 9; ++j) sg[j] = ss[32 * j];
                double lv[13], xv[27];
#pragma unroll
                for (int t = 0; t < 13; ++t) {                 // mirrored lower values
                    const bool on = (msk >> t) & 1u;
                    const int c = sg[t / 3] + (t % 3);
                    lv[t] = on ? __ldg(m.val + ((int64_t)(c >> 5) * 14 + (13 - t)) * 32 + (c & 31))
                               : 0.0;
                }
#pragma unroll
                for (int t = 0; t < 27; ++t)
                    xv[t] = ((msk >> t) & 1u) ? __ldg(a.x + sg[t / 3] + (t % 3)) : 0.0;
                double sum = 0.0;
#pragma unroll
                for (int t = 0; t < 13; ++t)
                    if ((msk >> t) & 1u) sum = __dadd_rn(sum, __dmul_rn(lv[t], xv[t]));
#pragma unroll
                for (int t = 13; t < 27; ++t)
                    if ((msk >> t) & 1u) sum = __dadd_rn(sum, __dmul_rn(vs[32 * (t - 13)], xv[t]));
                if (row >= 0) {
                    a.y[row] = sum;
                    if (DOT) ex.add(__dmul_rn(xv[13], sum), sacc);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty_bar[st]);
        }
        if (DOT) expansion_flush_digits(ex, sdig, sacc);
    }
    if (DOT) {
        __syncthreads();
        acc_merge_to_global(sacc, sdig, a.acc);
        if (a.fold_push) acc_push_last_cta(a.dc, a.acc, a.k, 0, a.dc.local + 3);
    }
}

// SYM with the mirrored values staged by the tensor engine.  Lower run j of a row (j = 0..3:
// (dz,dy) = (-1,-1), (-1,0), (-1,1), (0,-1); group 4 = slot 12, (0,0,-1)) reads stored slots
// 11-3j..13-3j (group 4: slot 1) of rows i - 1 + e + off_j.  For a tile [r0, r0 + 32 NW) those
// rows lie in the NW + 2 slices from floor((r0 - 1 + off_j) / 32): one 3-D box {32 lanes,
// NW + 2 slices, 3 slots} of the value array viewed SLOT-MAJOR ([14][slices][32] by strides),
// fetched with one cp.async.bulk.tensor per group (zero fill outside the matrix) -- from L2:
// the rows were streamed about one plane (or one line) earlier.  In shared memory each slot of
// a box is then GS * 32 consecutive rows, so a run's three mirrored values sit at one address
// (computed once per run from its stored start column) plus constant offsets.  Consumers read
// every matrix value from shared memory; only the x gathers go through L1.
//
// A warp whose 32 rows all have the full 27-entry pattern (interior rows: ~88 % of the tiles
// at 300^3) takes a branch-free path with no per-slot predicates; same operations, same order.
template <int NW, int NST> struct SymmCfg {
    static constexpr int THREADS = 32 * (NW + 1);
    static constexpr int VAL_B = NW * 14 * 32 * 8, SEG_B = NW * 9 * 32 * 4, MSK_B = NW * 32 * 4;
    static constexpr int GS = NW + 2;                          // slices per mirror box
    static constexpr int MIR3_B = GS * 3 * 32 * 8;             // one 3-slot box
    static constexpr int MIR1_B = GS * 32 * 8;                 // the slot-12 box
    static constexpr int MIR0 = (VAL_B + SEG_B + MSK_B + 127) / 128 * 128;
    static constexpr int STAGE_B = (MIR0 + 4 * MIR3_B + MIR1_B + 127) / 128 * 128;
    static constexpr int SMEM = NST * STAGE_B;
};

// first slice of mirror box g (0..4) of the tile whose first row is r0 (may be negative)
__device__ __forceinline__ int symm_box_slice(int64_t r0, int g, int64_t N0, int64_t P) {
    const int dz = g < 3 ? -1 : 0, dy = g < 3 ? g - 1 : (g == 3 ? -1 : 0);
    const int64_t lo = r0 - 1 + dy * N0 + dz * P;
    return (int)(lo >> 5);                                     // floor division
}

__device__ __forceinline__ void tma_box3(void *dst, const CUtensorMap *tm, int c0, int c1, int c2,
                                         uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

constexpr unsigned SYM_FULL = (1u << 27) - 1;               // all 27 slots present
// pAp expansion (exact.cuh): two 4-term tiers.  Measured alternatives (profiles/r01/session3):
// 4 + 2 + 2 the same; 2 parked spill slots drained into a 2-term tier once per tile 2.5 %
// faster while nothing spills but far slower late in CG (the tier overflows into the atomics);
// a 4-term drained tier or a third 4-term tier spills registers (128 per thread: 4 warps on
// an SM sub-partition share its 16 K registers).
// Two 2-term tiers where the solve is short of SpMV time (mid-size: fewer terms to flush at
// the end of every launch; B200, per solve 60^3 -2.7 %, 100^3 -1.3 %) and two 4-term tiers on
// large problems (300^3: +0.9 % with 2 + 2, the late iterations spill more);
// profiles/r02/ab/symm_expansion_tiers.jsonl.  Any tiers give the same exact sum.
constexpr int64_t SYMM_SMALL_TIER_SLICES = 1 << 17;        // 4.2 M rows

// One row of a SYMM tile in the order of C4: the 13 mirrored lower entries, then the 14 stored
// ones (diagonal first).  FULL: every slot present (warp-uniform), no predicates.  Returns the
// row sum; xd = x of the row itself (slot 13).
template <bool FULL, int GS, class WAIT>
__device__ __forceinline__ double symm_fold(const double *__restrict__ x, const int (&sg)[9],
                                            unsigned msk, const double *vs, const double *mir,
                                            const int (&madj)[5], int r0, double &xd,
                                            WAIT &&wait_values) {
    auto on = [&](int t) { return FULL || ((msk >> t) & 1u); };
    double xv[27];
#pragma unroll
    for (int t = 0; t < 27; ++t) xv[t] = on(t) ? __ldg(x + sg[t / 3] + (t % 3)) : 0.0;
    wait_values();                                    // the x gathers are in flight meanwhile
    double lv[13];
#pragma unroll
    for (int j = 0; j < 5; ++j) {                     // runs 0..3: 3 slots; run 4: slot 12
        const double *mj = mir + madj[j] + (sg[j] - r0);
        const int ne = j < 4 ? 3 : 1;
#pragma unroll
        for (int e = 0; e < ne; ++e) {
            const int t = 3 * j + e, q = j < 4 ? 2 - e : 0;
            lv[t] = FULL ? mj[q * GS * 32 + e] : (on(t) ? mj[q * GS * 32 + e] : 0.0);
        }
    }
    double sum = 0.0;
#pragma unroll
    for (int t = 0; t < 13; ++t)
        if (on(t)) sum = __dadd_rn(sum, __dmul_rn(lv[t], xv[t]));
#pragma unroll
    for (int t = 13; t < 27; ++t)
        if (on(t)) sum = __dadd_rn(sum, __dmul_rn(vs[32 * (t - 13)], xv[t]));
    xd = xv[13];
    return sum;
}

// Tile visited at position tau: the band order (tile_order) and/or last to first (reverse;
// every row's sum and the exact pAp are independent of the order, C4/C5)
__device__ __forceinline__ int64_t symm_tile_at(const SpmvArgs &a, int64_t tau, int64_t ntiles) {
    const int64_t t = a.reverse ? ntiles - 1 - tau : tau;
    return a.tile_order ? (int64_t)a.tile_order[t] : t;
}


template <bool DOT, int NW, int NST, int EA, int EB>
__global__ void __launch_bounds__(SymmCfg<NW, NST>::THREADS, 1)
    k_spmv_symm(SpmvArgs a, const __grid_constant__ CUtensorMap tm3,
                const __grid_constant__ CUtensorMap tm1) {
    using C = SymmCfg<NW, NST>;
    extern __shared__ __align__(128) unsigned char smem[];
    // per stage two "full" barriers: full_bar for the run starts and masks (small, issued
    // first: the consumers start their x gathers as soon as these land) and val_bar for the
    // values and mirror boxes (waited for after the gathers are in flight)
    __shared__ __align__(8) uint64_t full_bar[NST], val_bar[NST], empty_bar[NST];
    __shared__ unsigned long long sacc[ACC_WORDS];
    __shared__ int sdig[ACC_DIG16];
    if (threadIdx.x == 0) SYMM_STAMP(0);
    KT_SCOPE(0, a.k);
    // the stop flag is read while the first stages are already in flight (the matrix does
    // not depend on it): one memory latency less at the head of every SpMV
    const int done = (DOT && a.st) ? a.st->done : 0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const Matrix &m = a.m;
    const int64_t ntiles = (m.nslices + NW - 1) / NW;
    const int64_t N0 = a.g.ext_n[0], P = (int64_t)a.g.ext_n[0] * a.g.ext_n[1];
    const bool producer = warp == NW && lane == 0;
    uint64_t pol = 0, pol_keep = 0;
    // stage i of this CTA <- tile position tau (producer lane only)
    auto issue = [&](int64_t tau, int64_t i) {
        const int64_t tile = symm_tile_at(a, tau, ntiles);
        const int st = (int)(i % NST);
        if (i >= NST) mbar_wait(&empty_bar[st], (uint32_t)(((i / NST) & 1) ^ 1));
        const int64_t s0 = tile * NW;
        const int64_t rem = m.nslices - s0;
        const int nsl = rem < NW ? (int)rem : NW;
        unsigned char *buf = smem + (size_t)st * C::STAGE_B;
        const uint32_t bv = nsl * 14 * 32 * 8, bs = nsl * 9 * 32 * 4, bm = nsl * 32 * 4;
        const int64_t r0 = s0 * 32;
        mbar_expect_tx(&full_bar[st], bs + bm);
        bulk_g2s(buf + C::VAL_B, m.seg + s0 * 9 * 32, bs, &full_bar[st], pol);
        bulk_g2s(buf + C::VAL_B + C::SEG_B, m.mask + s0 * 32, bm, &full_bar[st], pol);
        mbar_expect_tx(&val_bar[st], bv + 4 * C::MIR3_B + C::MIR1_B);
        bulk_g2s(buf, m.val + s0 * 14 * 32, bv, &val_bar[st], pol_keep);
        if (a.x_prefetch) {
            // the tile's plane-ahead x (its dz = +1 runs) is read here for the first time:
            // start it into L2 now, so the consumers' gathers hit L2, not HBM
            int64_t lo = r0 + P - N0 - 1, hi = r0 + 32 * nsl + P + N0 + 1;
            lo = ((lo < 0 ? 0 : lo) + 1) & ~(int64_t)1;
            hi = (hi > a.g.ncols ? a.g.ncols : hi) & ~(int64_t)1;
            if (hi > lo && !(reinterpret_cast<uintptr_t>(a.x) & 15))
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.x + lo),
                             "r"((uint32_t)((hi - lo) * 8))
                             : "memory");
        }
#pragma unroll
        for (int g = 0; g < 4; ++g)
            tma_box3(buf + C::MIR0 + g * C::MIR3_B, &tm3, 0, symm_box_slice(r0, g, N0, P),
                     11 - 3 * g, &val_bar[st]);
        tma_box3(buf + C::MIR0 + 4 * C::MIR3_B, &tm1, 0, symm_box_slice(r0, 4, N0, P), 1,
                 &val_bar[st]);
        if (a.x_prefetch) {
            // the run starts and masks of the tile this stage takes next: into L2 now, so
            // that stage's first barrier completes at L2 latency (large problems; 300^3
            // -0.7 % per iteration, 100^3 +0.7 %).  After this stage's copies: with a tile
            // order the next tile's index is a global load the copies must not wait for.
            const int64_t tau2 = tau + (int64_t)NST * gridDim.x;
            const int64_t s2 = tau2 < ntiles ? symm_tile_at(a, tau2, ntiles) * NW : m.nslices;
            if (tau2 < ntiles && s2 < m.nslices) {
                const int64_t r2 = m.nslices - s2;
                const uint32_t n2 = r2 < NW ? (uint32_t)r2 : (uint32_t)NW;
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;"
                             ::"l"(m.seg + s2 * 9 * 32), "r"(n2 * 9 * 32 * 4) : "memory");
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;"
                             ::"l"(m.mask + s2 * 32), "r"(n2 * 32 * 4) : "memory");
            }
        }
    };
    if (producer) {
        SYMM_STAMP(1);
        for (int s = 0; s < NST; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&val_bar[s], 1);
            mbar_init(&empty_bar[s], NW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm3)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm1)) : "memory");
        pol = evict_first_policy();
        if (a.val_evict_first)
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_keep));
        else
            asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_keep));
        for (int64_t i = 0; i < NST && blockIdx.x + i * gridDim.x < ntiles; ++i)
            issue(blockIdx.x + i * gridDim.x, i);
    }
    if (DOT) acc_zero_shared(sacc, sdig);
    __syncthreads();                                   // barrier inits visible to all warps
    if (done) {
        // the solve has stopped: nothing to compute, but the stages in flight must land
        // before the CTA may exit
        if (producer)
            for (int64_t i = 0; i < NST && blockIdx.x + i * gridDim.x < ntiles; ++i) {
                mbar_wait(&full_bar[i], 0u);
                mbar_wait(&val_bar[i], 0u);
            }
        return;
    }
    if (DOT && blockIdx.x == 0 && a.acc_zero)
        for (int i = threadIdx.x; i < ACC_WORDS; i += blockDim.x) a.acc_zero[i] = 0ull;

    if (warp == NW) {
        if (lane == 0) {
            int64_t i = NST;
            for (int64_t tau = blockIdx.x + (int64_t)NST * gridDim.x; tau < ntiles;
                 tau += gridDim.x, ++i)
                issue(tau, i);
        }
    } else {
        ExpansionT<EA, EB> ex;
        ex.init();
        // box g of a tile starts at row r0 + K_g, K_g = 32 floor((off_g - 1) / 32): column c of
        // slot q sits at element madj[g] + q GS 32 + (c - r0) of the stage's mirror area
        int madj[5];
#pragma unroll
        for (int g = 0; g < 5; ++g)
            madj[g] = g * (C::MIR3_B / 8) - 32 * symm_box_slice(0, g, N0, P);
        int64_t i = 0;
        // with a tile order the tile index is a global load: fetch the next one a tile ahead,
        // so it is not a dependent L2 round trip at the head of every tile (300^3 banded: the
        // stall on its first use took ~10 % of the kernel's warp samples)
        int64_t tile_next = blockIdx.x < ntiles ? symm_tile_at(a, blockIdx.x, ntiles) : 0;
        for (int64_t tau = blockIdx.x; tau < ntiles; tau += gridDim.x, ++i) {
            const int64_t tile = tile_next;
            if (tau + gridDim.x < ntiles) tile_next = symm_tile_at(a, tau + gridDim.x, ntiles);
            const int st = (int)(i % NST);
            mbar_wait(&full_bar[st], (uint32_t)((i / NST) & 1));
            if (i == 0 && threadIdx.x == 0) SYMM_STAMP(2);
            const int64_t s = tile * NW + warp;
            if (s < m.nslices) {
                const unsigned char *buf = smem + (size_t)st * C::STAGE_B;
                const double *vs = reinterpret_cast<const double *>(buf) + warp * 14 * 32 + lane;
                const int32_t *ss =
                    reinterpret_cast<const int32_t *>(buf + C::VAL_B) + warp * 9 * 32 + lane;
                unsigned msk =
                    reinterpret_cast<const uint32_t *>(buf + C::VAL_B + C::SEG_B)[warp * 32 + lane];
                const double *mir = reinterpret_cast<const double *>(buf + C::MIR0);
                // storage row s*32+lane; SYM-ext: only owned nodes are computed rows
                const int64_t row = sym_row(m, a.g, s * 32 + lane, msk);
                const int r0 = (int)(tile * NW * 32);
                int sg[9];
#pragma unroll
                for (int j = 0; j < 9; ++j) sg[j] = ss[32 * j];
                double sum, xd;
                auto wait_values = [&]() {
                    mbar_wait(&val_bar[st], (uint32_t)((i / NST) & 1));
                };
                if (__all_sync(0xffffffffu, (msk & SYM_FULL) == SYM_FULL))
                    sum = symm_fold<true, C::GS>(a.x, sg, msk, vs, mir, madj, r0, xd,
                                                 wait_values);
                else
                    sum = symm_fold<false, C::GS>(a.x, sg, msk, vs, mir, madj, r0, xd,
                                                  wait_values);
                // every value of the stage has been consumed by the fold: release it before
                // the epilogue (the empty asm pins the fold's result ahead of the arrive, so
                // no shared-memory read of the stage can still be in flight)
                asm volatile("" ::"d"(sum) : "memory");
                __syncwarp();
                if (i == 0 && threadIdx.x == 0) SYMM_STAMP(3);
                if (lane == 0) mbar_arrive(&empty_bar[st]);
                if (row >= 0) {
                    a.y[row] = sum;
                    if (DOT) ex.add(__dmul_rn(xd, sum), sacc);
                }
            } else {
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty_bar[st]);
            }
        }
        if (threadIdx.x == 0) SYMM_STAMP(4);
        if (DOT) expansion_flush_digits(ex, sdig, sacc);
        if (threadIdx.x == 0) SYMM_STAMP(7);
    }
    if (DOT) {
        __syncthreads();
        if (threadIdx.x == 0) SYMM_STAMP(5);
        acc_merge_to_global(sacc, sdig, a.acc);
        if (a.fold_push) acc_push_last_cta(a.dc, a.acc, a.k, 0, a.dc.local + 3);
    }
    __syncthreads();
    if (threadIdx.x == 0) SYMM_STAMP(6);
}

// ----------------------------------------------------------------------------------------
// CG init (C6 step 1): x = 0, r = b, p = b, rr = dot(r, r)
// ----------------------------------------------------------------------------------------

// Halo by r (device comm).  The owner of a halo node computes p_(k+1) there as
// fl(r_(k+1) + fl(beta_k p_k)); the receiver holds p_k at that node (its halo column) and gets
// beta_k from the same exact rr, so with r_(k+1) pushed by the owner it computes the same bits
// itself -- and r_(k+1) is final after K6, so the push overlaps the rr reduction instead of
// waiting for it.  All threads of the CTA call it.
__device__ void halo_p_update(const UpdArgs &a, int kp, double beta, const double *pin,
                              double *pout) {
    const DevComm &dc = a.dc;
    const unsigned long long seq = comm_halo_seq(comm_gen(dc), kp);
    for (int t = threadIdx.x; t < dc.n_nbr; t += blockDim.x)
        comm_spin(dc, dc.local + comm_halo_flag(dc.world, dc.nbr_rank[t]), seq, a.st);
    __syncthreads();
    for (int64_t h = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; h < a.halo_n;
         h += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = a.halo_col[h];
        const double rv = __ldcv(a.rhalo + h);     // stored by a peer: never a stale L1 line
        pout[c] = pin ? __dadd_rn(rv, __dmul_rn(beta, pin[c])) : rv;
    }
}

__global__ void __launch_bounds__(UPD_THREADS) k_push_r(UpdArgs a, int kp,
                                                        const int32_t *send_row,
                                                        const uint8_t *slot_nbr,
                                                        const int32_t *dst_slot,
                                                        double *const *dst_ptr, int64_t n) {
    __shared__ int s_last;
    if (kp > 1 && a.st->done) return;    // kp = 1 (r_0 = b): the state is not initialised yet
    if (a.dc.mute) return;                 // fault injection: a rank that never signals
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst_ptr[slot_nbr[i]][dst_slot[i]] = a.r[send_row[i]];
    const DevComm &dc = a.dc;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();            // this CTA's peer stores (cumulative via bar.sync)
        s_last = atomicAdd(reinterpret_cast<unsigned long long *>(dc.local + 1), 1ull) ==
                 (unsigned long long)(gridDim.x - 1);
        if (s_last) __threadfence_system();
    }
    __syncthreads();
    if (!s_last) return;
    const unsigned long long seq = comm_halo_seq(comm_gen(dc), kp);
    for (int t = threadIdx.x; t < dc.n_nbr; t += blockDim.x)
        st_release_sys(dc.region[dc.nbr_rank[t]] + comm_halo_flag(dc.world, dc.rank), seq);
    if (threadIdx.x == 0) dc.local[1] = 0ull;       // ticket for the next launch
}

__global__ void __launch_bounds__(UPD_THREADS) k_halo_init(UpdArgs a) {
    halo_p_update(a, 1, 0.0, nullptr, a.p);
}

template <bool IDENT>
__global__ void __launch_bounds__(UPD_THREADS) k_init_vectors(UpdArgs a) {
    __shared__ unsigned long long sacc[ACC_WORDS];
    __shared__ int sdig[ACC_DIG16];
    acc_zero_shared(sacc, sdig);
    // device comm: a new solve generation (every later kernel of the solve reads it)
    if (a.dc.local && blockIdx.x == 0 && threadIdx.x == 0) {
        a.dc.local[0] += 1ull;
        a.dc.local[1] = 0ull;
        a.dc.local[2] = 0ull;
    }
    __syncthreads();
    Expansion ex;
    ex.init();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.g.rows; i += stride) {
        const double bi = a.b[i];
        a.x[i] = 0.0;
        a.r[i] = bi;
        a.p[IDENT ? i : row_to_col(a.g, i)] = bi;
        ex.add(__dmul_rn(bi, bi), sacc);
    }
    expansion_flush_digits(ex, sdig, sacc);
    __syncthreads();
    acc_merge_to_global(sacc, sdig, a.acc_out);
    if (a.fold_push) acc_push_last_cta(a.dc, a.acc_out, 0, 1, a.dc.local + 4);
}

// C6 step 1 decisions: rr_0, hist[0] = sqrt(rr_0), stop threshold fl(tol hist[0]) (one thread)
__device__ __forceinline__ void cg_state_init(const UpdArgs &a, double rr0, double tol) {
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
    st.alpha_iter = 0;
    st.x_done = 0;
    *a.st = st;
}

__global__ void k_init_finalize(UpdArgs a, double tol) {
    __shared__ unsigned long long s_in[ACC_WORDS];
    UpdArgs ai = a;
    ai.acc_in = a.acc_out;
    if (!acc_in_load(s_in, ai, 0, 1)) return;
    __syncthreads();
    const double fin = threadIdx.x < 32 ? acc_finalize_warp(s_in) : 0.0;   // warp 0
    if (threadIdx.x == 0) cg_state_init(a, fin, tol);
    if (a.acc_zero)
        for (int i = threadIdx.x; i < ACC_WORDS; i += blockDim.x) a.acc_zero[i] = 0ull;
}

// ----------------------------------------------------------------------------------------
// a3 + a4: finalise pAp -> alpha; x += alpha p; r -= alpha Ap; rr' = dot(r, r)
// ----------------------------------------------------------------------------------------

template <class EX>
__device__ __forceinline__ void xr_step(double &x, double &r, double p, double ap, double alpha,
                                        EX &ex, unsigned long long *sacc) {
    x = __dadd_rn(x, __dmul_rn(alpha, p));
    r = __dsub_rn(r, __dmul_rn(alpha, ap));
    ex.add(__dmul_rn(r, r), sacc);
}

// Decisions of K6 (a3, C6): finalise pAp, stop tests, alpha.  Thread 0 of each CTA (s_in =
// shared copy of the all-reduced accumulator); every CTA takes the same decision, CTA 0
// records it.  Returns stop.
__device__ __forceinline__ int xr_prologue_v(const UpdArgs &a, double pAp, int k, double rr,
                                             double &alpha) {
    int stop = 0, status = 0, conv = 0;
    if (!isfinite(pAp)) {
        stop = 1;
        status = 7;
    } else if (pAp <= 0.0) {
        stop = 1;
        if (rr == 0.0) conv = 1;
        else status = 6;
    }
    alpha = __ddiv_rn(rr, pAp);
    if (blockIdx.x == 0) {
        a.st->pAp = pAp;
        a.st->alpha = alpha;
        if (a.alpha_hist) a.alpha_hist[k] = alpha;
        if (stop) {
            a.st->status = status;
            a.st->converged = conv;
            a.st->iters = k - 1;
            a.st->done = 1;
        } else {
            a.st->alpha_iter = k;
        }
    }
    return stop;
}

__device__ __forceinline__ int xr_prologue(const UpdArgs &a, double pAp, int k, double &alpha) {
    return xr_prologue_v(a, pAp, k, a.rr[k - 1], alpha);
}

// Decisions after rr_k (a5, C6): finalise rr_k, hist[k], stop tests, beta_k.  rr_old =
// rr[k-1] and stop_thr = st->stop, loaded by the caller (ahead of the accumulator rounding).
__device__ __forceinline__ int rr_decision_v(double rr_new, int k, double rr_old,
                                             double stop_thr, double *hist, double *rr,
                                             CgState *st, double &beta) {
    const double h = __dsqrt_rn(rr_new);
    int stop = 0, status = 0, conv = 0;
    if (!isfinite(rr_new)) {
        stop = 1;
        status = 7;
    } else if (rr_new == 0.0 || h <= stop_thr) {
        stop = 1;
        conv = 1;
    }
    beta = __ddiv_rn(rr_new, rr_old);
    if (blockIdx.x == 0) {
        hist[k] = h;
        rr[k] = rr_new;
        st->iters = k;
        st->beta = beta;
        if (stop) {
            st->status = status;
            st->converged = conv;
            st->done = 1;
        }
    }
    return stop;
}

__device__ __forceinline__ int rr_decision(double rr_new, int k, double *hist, double *rr,
                                           CgState *st, double &beta) {
    return rr_decision_v(rr_new, k, rr[k - 1], st->stop, hist, rr, st, beta);
}

// Decisions of K7 (a5, C6).
__device__ __forceinline__ int p_prologue(const UpdArgs &a, double rr_new, int k, double &beta) {
    return rr_decision(rr_new, k, a.hist, a.rr, a.st, beta);
}

// Entry of K6 / K7 on one-rank accumulators (no device comm): the stop flag, the accumulator
// words (threads < ACC_WORDS, into s_in) and the scalars thread 0's decision needs are loaded
// together, one memory round trip instead of three dependent ones.  Returns false when the
// solve has stopped.  With device comm: the flag wait of acc_in_load.
struct PreScalars {
    double rr_old, stop_thr, alpha;
};
static_assert(UPD_THREADS >= ACC_WORDS, "upd_entry loads one accumulator word per thread");
__device__ __forceinline__ bool upd_entry(const UpdArgs &a, int k, int which,
                                          unsigned long long *s_in, PreScalars &ps) {
    const bool local = a.dc.local == nullptr;
    unsigned long long w = 0ull;
    if (local && threadIdx.x < ACC_WORDS) w = __ldcg(a.acc_in + threadIdx.x);
    if (threadIdx.x == 0) {
        ps.rr_old = a.rr[k - 1];
        ps.stop_thr = a.st->stop;
        ps.alpha = a.st->alpha;
    }
    if (a.st->done) return false;
    if (local) {
        if (threadIdx.x < ACC_WORDS) s_in[threadIdx.x] = w;
        return true;
    }
    return acc_in_load(s_in, a, k, which);
}

// XL: x is updated by K7 (see launch_update_xr); K6 touches r only: 24 instead of 48 B/row.
template <class EX>
__device__ __forceinline__ void r_step(double &r, double ap, double alpha, EX &ex,
                                       unsigned long long *sacc) {
    r = __dsub_rn(r, __dmul_rn(alpha, ap));
    ex.add(__dmul_rn(r, r), sacc);
}

template <bool IDENT, bool XL, class EX = Expansion>
__global__ void __launch_bounds__(UPD_THREADS, 3) k_update_xr(UpdArgs a, int k) {
    __shared__ unsigned long long sacc[ACC_WORDS], s_in[ACC_WORDS];
    __shared__ int sdig[ACC_DIG16];
    __shared__ double s_alpha;
    __shared__ int s_stop;
    KT_SCOPE(1, k);
    K6_STAMP(0);
    PreScalars ps;
    if (!upd_entry(a, k, 0, s_in, ps)) return;
    K6_STAMP(1);
    acc_zero_shared(sacc, sdig);
    __syncthreads();
    K6_STAMP(2);
    const double fin = threadIdx.x < 32 ? acc_finalize_warp(s_in) : 0.0;   // warp 0
    K6_STAMP(7);
    if (threadIdx.x == 0) {
        double alpha;
        s_stop = xr_prologue_v(a, fin, k, ps.rr_old, alpha);
        s_alpha = alpha;
    }
    __syncthreads();
    K6_STAMP(3);
    if (s_stop) return;
    const double alpha = s_alpha;
    EX ex;
    ex.init();
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t rows = a.g.rows;
    if (XL) {
        // r -= alpha Ap, exact rr (16-byte accesses, four pairs in flight per thread: K6
        // moves only 24 B per row, so it needs the deeper queue to cover DRAM latency)
        const int64_t n2 = rows >> 1;
        double2 *r2 = reinterpret_cast<double2 *>(a.r);
        const double2 *q2 = reinterpret_cast<const double2 *>(a.Ap);
        int64_t i = tid;
        for (; i + 3 * stride < n2; i += 4 * stride) {
            double2 rv[4], qv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                rv[u] = r2[i + u * stride];
                qv[u] = q2[i + u * stride];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                r_step(rv[u].x, qv[u].x, alpha, ex, sacc);
                r_step(rv[u].y, qv[u].y, alpha, ex, sacc);
                r2[i + u * stride] = rv[u];
            }
        }
        for (; i + stride < n2; i += 2 * stride) {
            double2 ra = r2[i], qa = q2[i], rb = r2[i + stride], qb = q2[i + stride];
            r_step(ra.x, qa.x, alpha, ex, sacc);
            r_step(ra.y, qa.y, alpha, ex, sacc);
            r_step(rb.x, qb.x, alpha, ex, sacc);
            r_step(rb.y, qb.y, alpha, ex, sacc);
            r2[i] = ra;
            r2[i + stride] = rb;
        }
        for (; i < n2; i += stride) {
            double2 ra = r2[i], qa = q2[i];
            r_step(ra.x, qa.x, alpha, ex, sacc);
            r_step(ra.y, qa.y, alpha, ex, sacc);
            r2[i] = ra;
        }
        if ((rows & 1) && tid == 0) {
            double rj = a.r[rows - 1];
            r_step(rj, a.Ap[rows - 1], alpha, ex, sacc);
            a.r[rows - 1] = rj;
        }
    } else if (IDENT) {
        // 16-byte vector accesses, two pairs in flight per thread
        const int64_t n2 = rows >> 1;
        double2 *x2 = reinterpret_cast<double2 *>(a.x);
        double2 *r2 = reinterpret_cast<double2 *>(a.r);
        const double2 *p2 = reinterpret_cast<const double2 *>(a.p);
        const double2 *q2 = reinterpret_cast<const double2 *>(a.Ap);
        int64_t i = tid;
        for (; i + stride < n2; i += 2 * stride) {
            double2 xa = x2[i], ra = r2[i], pa = p2[i], qa = q2[i];
            double2 xb = x2[i + stride], rb = r2[i + stride], pb = p2[i + stride],
                    qb = q2[i + stride];
            xr_step(xa.x, ra.x, pa.x, qa.x, alpha, ex, sacc);
            xr_step(xa.y, ra.y, pa.y, qa.y, alpha, ex, sacc);
            xr_step(xb.x, rb.x, pb.x, qb.x, alpha, ex, sacc);
            xr_step(xb.y, rb.y, pb.y, qb.y, alpha, ex, sacc);
            x2[i] = xa;
            r2[i] = ra;
            x2[i + stride] = xb;
            r2[i + stride] = rb;
        }
        for (; i < n2; i += stride) {
            double2 xa = x2[i], ra = r2[i], pa = p2[i], qa = q2[i];
            xr_step(xa.x, ra.x, pa.x, qa.x, alpha, ex, sacc);
            xr_step(xa.y, ra.y, pa.y, qa.y, alpha, ex, sacc);
            x2[i] = xa;
            r2[i] = ra;
        }
        if ((rows & 1) && tid == 0) {
            const int64_t j = rows - 1;
            double xj = a.x[j], rj = a.r[j];
            xr_step(xj, rj, a.p[j], a.Ap[j], alpha, ex, sacc);
            a.x[j] = xj;
            a.r[j] = rj;
        }
    } else {
        for (int64_t i = tid; i < rows; i += stride) {
            double xi = a.x[i], ri = a.r[i];
            xr_step(xi, ri, a.p[row_to_col(a.g, i)], a.Ap[i], alpha, ex, sacc);
            a.x[i] = xi;
            a.r[i] = ri;
        }
    }
    K6_STAMP(4);
#ifdef SYMM_TRACE
    __syncthreads();
    K6_STAMP(9);
#endif
    expansion_flush_digits(ex, sdig, sacc);
    __syncthreads();
    K6_STAMP(5);
    acc_merge_to_global(sacc, sdig, a.acc_out);
    if (a.fold_push) acc_push_last_cta(a.dc, a.acc_out, k, 1, a.dc.local + 4);
    __syncthreads();
    K6_STAMP(6);
}

// ----------------------------------------------------------------------------------------
// a5 + a6: finalise rr' -> hist[k], stop tests, beta; p = r + beta p
// ----------------------------------------------------------------------------------------
// Small problems: the whole CG solve in ONE CTA of 1024 threads, one
// launch.  At 10^3 (1331 rows) the three-kernel iteration is bound by launch and grid-wide
// latency (~18 us/iteration); here an iteration is three CTA barriers apart.  p lives in
// shared memory (the SpMV gathers it), x, r, Ap in registers (rows tid + 1024 j); the matrix
// (SEG or SYM, L2-resident) is read from global memory.  Every dot goes through the same
// exact expansion -> shared superaccumulator -> warp-parallel rounding, and every decision
// through the same C6 code as the multi-kernel path: results are bit-identical.
// ----------------------------------------------------------------------------------------

template <int FMT>
__device__ __forceinline__ double small_row_spmv(const Matrix &m, int64_t row,
                                                 const double *ps) {
    const int64_t s = row >> 5;
    const int lane = (int)(row & 31);
    const unsigned msk = m.mask[s * 32 + lane];
    int sg[9];
#pragma unroll
    for (int j = 0; j < 9; ++j) sg[j] = m.seg[(9 * s + j) * 32 + lane];
    double sum = 0.0;
#pragma unroll
    for (int t = 0; t < 27; ++t) {
        if (!((msk >> t) & 1u)) continue;
        const int c = sg[t / 3] + (t % 3);
        double v;
        if (FMT == FMT_SEG) v = m.val[(27 * s + t) * 32 + lane];
        else if (t >= 13) v = m.val[(14 * s + (t - 13)) * 32 + lane];
        else v = m.val[((int64_t)(c >> 5) * 14 + (13 - t)) * 32 + (c & 31)];   // mirror
        sum = __dadd_rn(sum, __dmul_rn(v, ps[c]));
    }
    return sum;
}

// One exact block-wide dot: every thread's expansion -> 32-bit digit counters -> words ->
// warp-parallel rounding (warp 0; the value is returned to thread 0 only).
__device__ __forceinline__ double small_block_dot(const Expansion &ex, int *dig,
                                                  unsigned long long *sacc) {
    expansion_flush_digits(ex, dig, sacc);
    __syncthreads();
    double v = 0.0;
    if (threadIdx.x < 32) {
        digits_to_words(dig, sacc);
        __syncwarp();
        v = acc_finalize_warp(sacc);
        __syncwarp();
        for (int i = threadIdx.x; i < ACC_WORDS; i += 32) sacc[i] = 0ull;
    }
    return v;
}

template <int FMT>
__global__ void __launch_bounds__(SMALL_THREADS, 1) k_cg_small(Matrix m, UpdArgs a, int K,
                                                               double tol) {
    __shared__ double ps[SMALL_MAX_ROWS + 32];
    __shared__ unsigned long long sacc[ACC_WORDS];
    __shared__ int dig[ACC_DIG16];
    __shared__ double s_coef;
    __shared__ int s_stop;
    const int tid = threadIdx.x;
    const int64_t rows = m.rows;
    double xv[SMALL_RPT], rv[SMALL_RPT], apv[SMALL_RPT];
    // C6 step 1: x = 0, r = b, p = b, rr_0 = dot(r, r)
    acc_zero_shared(sacc);
    for (int i = tid; i < ACC_DIG16; i += blockDim.x) dig[i] = 0;
    __syncthreads();
    Expansion ex;
    ex.init();
#pragma unroll
    for (int j = 0; j < SMALL_RPT; ++j) {
        const int64_t row = tid + (int64_t)SMALL_THREADS * j;
        xv[j] = rv[j] = apv[j] = 0.0;
        if (row < rows) {
            const double b = a.b[row];
            rv[j] = b;
            ps[row] = b;
            ex.add(__dmul_rn(b, b), sacc);
        }
    }
    // thread 0 keeps rr_(k-1) and the stop threshold (the values cg_state_init records) in
    // registers: no global round trip in the decisions
    double rr_prev = 0.0, stop_thr = 0.0;
    {
        const double rr0 = small_block_dot(ex, dig, sacc);
        if (tid == 0) {
            cg_state_init(a, rr0, tol);
            rr_prev = rr0;
            stop_thr = __dmul_rn(tol, __dsqrt_rn(rr0));
        }
    }
    __syncthreads();
    for (int k = 1; k <= K; ++k) {
        // a2 + a3: Ap = A p, pAp, alpha (stop tests of K6)
        ex.init();
#pragma unroll
        for (int j = 0; j < SMALL_RPT; ++j) {
            const int64_t row = tid + (int64_t)SMALL_THREADS * j;
            if (row < rows) {
                apv[j] = small_row_spmv<FMT>(m, row, ps);
                ex.add(__dmul_rn(ps[row], apv[j]), sacc);
            }
        }
        {
            const double pAp = small_block_dot(ex, dig, sacc);
            if (tid == 0) {
                double alpha;
                s_stop = xr_prologue_v(a, pAp, k, rr_prev, alpha);
                s_coef = alpha;
            }
        }
        __syncthreads();
        if (s_stop) break;
        // a4 + a5: x += alpha p, r -= alpha Ap, rr', beta (stop tests of K7)
        const double alpha = s_coef;
        ex.init();
#pragma unroll
        for (int j = 0; j < SMALL_RPT; ++j) {
            const int64_t row = tid + (int64_t)SMALL_THREADS * j;
            if (row < rows) xr_step(xv[j], rv[j], ps[row], apv[j], alpha, ex, sacc);
        }
        {
            const double rrn = small_block_dot(ex, dig, sacc);
            if (tid == 0) {
                double beta;
                s_stop = rr_decision_v(rrn, k, rr_prev, stop_thr, a.hist, a.rr, a.st, beta);
                s_coef = beta;
                rr_prev = rrn;
            }
        }
        __syncthreads();
        if (s_stop) break;
        // a6: p = r + beta p
        const double beta = s_coef;
#pragma unroll
        for (int j = 0; j < SMALL_RPT; ++j) {
            const int64_t row = tid + (int64_t)SMALL_THREADS * j;
            if (row < rows) ps[row] = __dadd_rn(rv[j], __dmul_rn(beta, ps[row]));
        }
        __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < SMALL_RPT; ++j) {
        const int64_t row = tid + (int64_t)SMALL_THREADS * j;
        if (row < rows) {
            a.x[row] = xv[j];
            a.r[row] = rv[j];
            a.p[row] = ps[row];
        }
    }
}

// ----------------------------------------------------------------------------------------
// Cluster-resident solver: the whole solve in ONE thread-block cluster
// of CL_CTAS CTAs, one launch.  CTA q owns a contiguous block of slices; its matrix rows (all
// 27 value slots, SYM mirrors resolved once at start) live in its shared memory, and every
// CTA keeps a full copy of p, refreshed after each p update by distributed-shared-memory
// stores.  A dot: each CTA reduces its expansions into 32-bit digit counters, pushes the
// nonzero ones into EVERY CTA's receive counters (DSMEM atomics), one cluster barrier, then
// every CTA rounds the same integers and takes the same C6 decision (CTA 0 records it).
// Three cluster barriers per iteration; results bit-identical to every other path.
// ----------------------------------------------------------------------------------------

namespace cgx = cooperative_groups;

constexpr int CL_NDIG = ACC_DIG16 + 4;            // + 4 digits for the top word's high part
constexpr int CL_FLAG = CL_NDIG;                  // non-finite counter slot

struct ClusterSmem {
    double val[CL_MAX_SL][27][32];
    int32_t seg[CL_MAX_SL][9][32];
    uint32_t mask[CL_MAX_SL][32];
    double pfull[CL_MAX_ROWS + 32];
    int recv[2][CL_NDIG + 1];            // cluster sums, parity double-buffered
    int dig[CL_NDIG + 1];                // this CTA's digit counters
    int nzd[CL_NDIG + 1], nzv[CL_NDIG + 1], nnz;   // its nonzero ones, compacted
    unsigned long long sacc[ACC_WORDS];
    unsigned long long fin[ACC_WORDS];
    double coef;
    int stop;
};

// A product added straight to the CTA's 16-bit digit counters (shared 32-bit atomics): its
// exact value m 2^(pos-1074) cut into <= 5 signed 16-bit chunks on the global grid.  For the
// cluster solver's few products per thread this is cheaper than a TwoSum expansion plus a
// warp flush.  A CTA adds <= 2^10 chunks < 2^16 per digit, 16 CTAs < 2^31.  Non-finite
// values count in the flag slot.
__device__ __forceinline__ void dig_add(double v, int *dig) {
    const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
    const int e = (int)((bits >> 52) & 0x7ff);
    const unsigned long long frac = bits & 0xfffffffffffffull;
    if (e == 0x7ff) {
        atomicAdd(&dig[CL_FLAG], 1);
        return;
    }
    if (e == 0 && frac == 0) return;
    const unsigned long long m = e ? (frac | (1ull << 52)) : frac;
    const int pos = e ? e - 1 : 0;
    const int d16 = pos >> 4, s16 = pos & 15;
    const unsigned long long mlo = m << s16;
    const unsigned long long mhi = s16 ? (m >> (64 - s16)) : 0ull;
    int ch[5] = {(int)(mlo & 0xffff), (int)((mlo >> 16) & 0xffff), (int)((mlo >> 32) & 0xffff),
                 (int)(mlo >> 48), (int)mhi};
    const bool neg = bits >> 63;
#pragma unroll
    for (int q = 0; q < 5; ++q)
        if (ch[q]) atomicAdd(&dig[d16 + q], neg ? -ch[q] : ch[q]);
}


// Exact cluster-wide dot of the CTAs' expansions (all threads of every CTA call it); the
// rounded value is returned to warp 0 of every CTA.  Each CTA reduces into its own digit
// counters and adds the nonzero ones into EVERY CTA's receive counters (DSMEM atomics);
// after one cluster barrier every CTA rounds the same integers.  recv[par] is cleared right
// after use: it is written again two dots later, behind a barrier this CTA has not yet passed.
// (Pulling all CTAs' counters after the barrier instead measured 1 us slower at 10^3.)
template <bool DD>
__device__ __forceinline__ double cluster_dot(const Expansion &ex, ClusterSmem &S,
                                              cgx::cluster_group &cl, int par) {
    if (!DD) expansion_flush_digits(ex, S.dig, S.sacc);   // DD: products already in S.dig
    __syncthreads();
    const int lane = threadIdx.x & 31;
    if (threadIdx.x < 32) {
        // words of the slow path (far-below values): as 16-bit digits, the top one signed
        for (int w = lane; w < ACC_DIGITS; w += 32) {
            const long long v = (long long)S.sacc[w];
            S.sacc[w] = 0ull;
            if (v) {
                atomicAdd(&S.dig[2 * w], (int)(v & 0xffff));
                atomicAdd(&S.dig[2 * w + 1], (int)((v >> 16) & 0xffff));
                atomicAdd(&S.dig[2 * w + 2], (int)((v >> 32) & 0xffff));
                atomicAdd(&S.dig[2 * w + 3], (int)(v >> 48));
            }
        }
        if (lane == 0 && S.sacc[ACC_FLAG]) {
            S.dig[CL_FLAG] += 1;
            S.sacc[ACC_FLAG] = 0ull;
        }
        __syncwarp();
        // compact the nonzero counters (ascending digit) for the push below
        int nnz = 0;
        for (int d0 = 0; d0 <= CL_NDIG; d0 += 32) {
            const int d = d0 + lane;
            const int v = d <= CL_NDIG ? S.dig[d] : 0;
            const unsigned bal = __ballot_sync(0xffffffffu, v != 0);
            if (v) {
                const int at = nnz + __popc(bal & ((1u << lane) - 1u));
                S.nzd[at] = d;
                S.nzv[at] = v;
                S.dig[d] = 0;
            }
            nnz += __popc(bal);
        }
        if (lane == 0) S.nnz = nnz;
    }
    __syncthreads();
    // every (nonzero digit, CTA) pair by its own thread: one remote atomic each
    {
        const int C = (int)cl.num_blocks(), nnz = S.nnz;
        for (int e = threadIdx.x; e < nnz * C; e += blockDim.x) {
            const int q = e % nnz, r = e / nnz;
            atomicAdd(cl.map_shared_rank(&S.recv[par][S.nzd[q]], r), S.nzv[q]);
        }
    }
    cl.sync();
    double v = 0.0;
    if (threadIdx.x < 32) {
        const int *rc = S.recv[par];
        for (int w = lane; w < ACC_DIGITS; w += 32) {
            long long x = (long long)rc[2 * w] + (long long)rc[2 * w + 1] * 65536ll;
            if (w == ACC_DIGITS - 1)
                x += ((long long)rc[2 * w + 2] << 32) + ((long long)rc[2 * w + 3] << 48);
            S.fin[w] = (unsigned long long)x;
        }
        if (lane == 0) S.fin[ACC_FLAG] = rc[CL_FLAG] ? 1ull : 0ull;
        __syncwarp();
        v = acc_finalize_warp(S.fin);
        __syncwarp();
        for (int d = lane; d <= CL_NDIG; d += 32) S.recv[par][d] = 0;
    }
    return v;
}

template <int FMT, bool DD = true>
__global__ void __launch_bounds__(CL_THREADS, 1) k_cg_cluster(Matrix m, UpdArgs a, int K,
                                                             double tol) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    ClusterSmem &S = *reinterpret_cast<ClusterSmem *>(smem_raw);
    cgx::cluster_group cl = cgx::this_cluster();
    const int q = (int)cl.block_rank(), C = (int)cl.num_blocks();
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t rows = m.rows, ns = m.nslices;
    const int64_t s_lo = ns * q / C, s_hi = ns * (q + 1) / C;
    const int nsl = (int)(s_hi - s_lo);
    // own rows' matrix into shared memory: 27 value slots (SYM: mirrors resolved here)
    for (int e = tid; e < nsl * 27 * 32; e += CL_THREADS) {
        const int sl = e / (27 * 32), t = (e / 32) % 27, ln = e % 32;
        const int64_t sg = s_lo + sl;
        const unsigned msk = m.mask[sg * 32 + ln];
        double v = 0.0;
        if ((msk >> t) & 1u) {
            if (FMT == FMT_SEG) {
                v = m.val[(27 * sg + t) * 32 + ln];
            } else if (t >= 13) {
                v = m.val[(14 * sg + (t - 13)) * 32 + ln];
            } else {
                const int c = m.seg[(9 * sg + t / 3) * 32 + ln] + t % 3;
                v = m.val[((int64_t)(c >> 5) * 14 + (13 - t)) * 32 + (c & 31)];
            }
        }
        S.val[sl][t][ln] = v;
    }
    for (int e = tid; e < nsl * 9 * 32; e += CL_THREADS) {
        const int sl = e / (9 * 32), j = (e / 32) % 9, ln = e % 32;
        S.seg[sl][j][ln] = m.seg[(9 * (s_lo + sl) + j) * 32 + ln];
    }
    for (int e = tid; e < nsl * 32; e += CL_THREADS) S.mask[e / 32][e % 32] = m.mask[s_lo * 32 + e];

    for (int e = tid; e <= CL_NDIG; e += CL_THREADS) {
        S.recv[0][e] = S.recv[1][e] = 0;
        S.dig[e] = 0;
    }
    for (int e = tid; e < ACC_WORDS; e += CL_THREADS) S.sacc[e] = 0ull;
    // C6 step 1: x = 0, r = b, p = b (every CTA holds all of p), rr_0
    for (int64_t i = tid; i < rows; i += CL_THREADS) S.pfull[i] = a.b[i];
    __syncthreads();                               // counters zeroed before any thread adds
    double xv[CL_RPT], rv[CL_RPT], apv[CL_RPT];
    Expansion ex;
    ex.init();
#pragma unroll
    for (int j = 0; j < CL_RPT; ++j) {
        const int sl = warp + CL_WARPS * j;
        const int64_t row = (s_lo + sl) * 32 + lane;
        xv[j] = rv[j] = apv[j] = 0.0;
        if (sl < nsl) {                                // warp-uniform
            double v = 0.0;
            if (row < rows) {
                rv[j] = a.b[row];
                v = __dmul_rn(rv[j], rv[j]);
                if (!DD) ex.add(v, S.sacc);
            }
            if (DD) dig_add(v, S.dig);            // v = 0: nothing
        }
    }
    cl.sync();                                     // matrix, counters and p in place everywhere
    int par = 0;
    // thread 0 of every CTA keeps rr_(k-1) and the stop threshold (the values CTA 0's
    // cg_state_init records) in registers: no global round trip in the decisions
    double rr_prev = 0.0, stop_thr = 0.0;
    {
        const double rr0 = cluster_dot<DD>(ex, S, cl, par);
        par ^= 1;
        if (q == 0 && tid == 0) cg_state_init(a, rr0, tol);
        if (tid == 0) {
            rr_prev = rr0;
            stop_thr = __dmul_rn(tol, __dsqrt_rn(rr0));
        }
    }
    for (int k = 1; k <= K; ++k) {
        // a2 + a3: Ap = A p (own rows), exact pAp, alpha
        ex.init();
#pragma unroll
        for (int j = 0; j < CL_RPT; ++j) {
            const int sl = warp + CL_WARPS * j;
            const int64_t row = (s_lo + sl) * 32 + lane;
            if (sl < nsl) {                            // warp-uniform
                double v = 0.0;
                if (row < rows) {
                    const unsigned msk = S.mask[sl][lane];
                    double sum = 0.0;
#pragma unroll
                    for (int t = 0; t < 27; ++t)
                        if ((msk >> t) & 1u)
                            sum = __dadd_rn(sum, __dmul_rn(S.val[sl][t][lane],
                                                           S.pfull[S.seg[sl][t / 3][lane] + t % 3]));
                    apv[j] = sum;
                    v = __dmul_rn(S.pfull[row], sum);
                    if (!DD) ex.add(v, S.sacc);
                }
                if (DD) dig_add(v, S.dig);            // v = 0: nothing
            }
        }
        {
            const double pAp = cluster_dot<DD>(ex, S, cl, par);
            par ^= 1;
            if (tid == 0) {
                double alpha;
                S.stop = xr_prologue_v(a, pAp, k, rr_prev, alpha);   // CTA 0 records
                S.coef = alpha;
            }
        }
        __syncthreads();
        if (S.stop) break;
        // a4 + a5: x += alpha p, r -= alpha Ap, exact rr, beta
        const double alpha = S.coef;
        ex.init();
#pragma unroll
        for (int j = 0; j < CL_RPT; ++j) {
            const int sl = warp + CL_WARPS * j;
            const int64_t row = (s_lo + sl) * 32 + lane;
            if (sl < nsl) {                            // warp-uniform
                double v = 0.0;
                if (row < rows) {
                    if (DD) {
                        xv[j] = __dadd_rn(xv[j], __dmul_rn(alpha, S.pfull[row]));
                        rv[j] = __dsub_rn(rv[j], __dmul_rn(alpha, apv[j]));
                        v = __dmul_rn(rv[j], rv[j]);
                    } else {
                        xr_step(xv[j], rv[j], S.pfull[row], apv[j], alpha, ex, S.sacc);
                    }
                }
                if (DD) dig_add(v, S.dig);            // v = 0: nothing
            }
        }
        {
            const double rrn = cluster_dot<DD>(ex, S, cl, par);
            par ^= 1;
            if (tid == 0) {
                double beta;
                S.stop = rr_decision_v(rrn, k, rr_prev, stop_thr, a.hist, a.rr, a.st, beta);
                S.coef = beta;
                rr_prev = rrn;
            }
        }
        __syncthreads();
        if (S.stop) break;
        // a6: p = r + beta p for own rows, stored into every CTA's copy
        const double beta = S.coef;
#pragma unroll
        for (int j = 0; j < CL_RPT; ++j) {
            const int sl = warp + CL_WARPS * j;
            const int64_t row = (s_lo + sl) * 32 + lane;
            if (sl < nsl && row < rows) {
                const double pn = __dadd_rn(rv[j], __dmul_rn(beta, S.pfull[row]));
                for (int r = 0; r < C; ++r) *cl.map_shared_rank(&S.pfull[row], r) = pn;
            }
        }
        cl.sync();
    }
#pragma unroll
    for (int j = 0; j < CL_RPT; ++j) {
        const int sl = warp + CL_WARPS * j;
        const int64_t row = (s_lo + sl) * 32 + lane;
        if (sl < nsl && row < rows) {
            a.x[row] = xv[j];
            a.r[row] = rv[j];
            a.p[row] = S.pfull[row];
        }
    }
    cl.sync();                                     // no CTA exits while others may write to it
}

// ----------------------------------------------------------------------------------------

// XL: also x += fl(alpha_k p_k) with the p_k read for the p update -- also when K7's own
// stop test fires (C6 updates x before the rr test), then without the p update.
template <bool IDENT, bool XL>
__global__ void __launch_bounds__(UPD_THREADS) k_update_p(UpdArgs a, int k) {
    __shared__ unsigned long long s_in[ACC_WORDS];
    __shared__ double s_beta, s_alpha;
    __shared__ int s_stop;
    PreScalars ps;                       // K6 stopped (pAp test): no x update for this k
    // the thread's first pair of p, r (and x) is loaded ahead of the entry and the rounding:
    // none of it depends on beta, and at mid-size the entry is most of K7
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool pre = IDENT && tid < (a.g.rows >> 1);
    double2 e_p = make_double2(0.0, 0.0), e_r = e_p, e_x = e_p;
    if (pre) {
        e_p = reinterpret_cast<const double2 *>(a.p)[tid];
        e_r = reinterpret_cast<const double2 *>(a.r)[tid];
        if (XL) e_x = reinterpret_cast<const double2 *>(a.x)[tid];
    }
    if (!upd_entry(a, k, 1, s_in, ps)) return;
    __syncthreads();
    const double fin = threadIdx.x < 32 ? acc_finalize_warp(s_in) : 0.0;   // warp 0
    if (threadIdx.x == 0) {
        if (XL) s_alpha = ps.alpha;      // alpha_k, written by K6 before this launch
        double beta;
        s_stop = rr_decision_v(fin, k, ps.rr_old, ps.stop_thr, a.hist, a.rr, a.st, beta);
        s_beta = beta;
    }
    __syncthreads();
    const bool stop = s_stop;
    if (stop && !XL) return;
    if (!stop && blockIdx.x == 0 && a.acc_zero)
        for (int i = threadIdx.x; i < ACC_WORDS; i += blockDim.x) a.acc_zero[i] = 0ull;
    const double beta = s_beta, alpha = XL ? s_alpha : 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t rows = a.g.rows;
    if (IDENT) {
        const int64_t n2 = rows >> 1;
        double2 *p2 = reinterpret_cast<double2 *>(a.p);
        double2 *x2 = reinterpret_cast<double2 *>(a.x);
        const double2 *r2 = reinterpret_cast<const double2 *>(a.r);
        if (pre) {
            if (XL) {
                e_x.x = __dadd_rn(e_x.x, __dmul_rn(alpha, e_p.x));
                e_x.y = __dadd_rn(e_x.y, __dmul_rn(alpha, e_p.y));
                x2[tid] = e_x;
            }
            if (!stop) {
                e_p.x = __dadd_rn(e_r.x, __dmul_rn(beta, e_p.x));
                e_p.y = __dadd_rn(e_r.y, __dmul_rn(beta, e_p.y));
                p2[tid] = e_p;
            }
        }
        int64_t i = tid + stride;
        for (; i + stride < n2; i += 2 * stride) {
            double2 pa = p2[i], pb = p2[i + stride];
            if (XL) {
                double2 xa = x2[i], xb = x2[i + stride];
                xa.x = __dadd_rn(xa.x, __dmul_rn(alpha, pa.x));
                xa.y = __dadd_rn(xa.y, __dmul_rn(alpha, pa.y));
                xb.x = __dadd_rn(xb.x, __dmul_rn(alpha, pb.x));
                xb.y = __dadd_rn(xb.y, __dmul_rn(alpha, pb.y));
                x2[i] = xa;
                x2[i + stride] = xb;
                if (stop) continue;
            }
            const double2 ra = r2[i], rb = r2[i + stride];
            pa.x = __dadd_rn(ra.x, __dmul_rn(beta, pa.x));
            pa.y = __dadd_rn(ra.y, __dmul_rn(beta, pa.y));
            pb.x = __dadd_rn(rb.x, __dmul_rn(beta, pb.x));
            pb.y = __dadd_rn(rb.y, __dmul_rn(beta, pb.y));
            p2[i] = pa;
            p2[i + stride] = pb;
        }
        for (; i < n2; i += stride) {
            double2 pa = p2[i];
            if (XL) {
                double2 xa = x2[i];
                xa.x = __dadd_rn(xa.x, __dmul_rn(alpha, pa.x));
                xa.y = __dadd_rn(xa.y, __dmul_rn(alpha, pa.y));
                x2[i] = xa;
                if (stop) continue;
            }
            const double2 ra = r2[i];
            pa.x = __dadd_rn(ra.x, __dmul_rn(beta, pa.x));
            pa.y = __dadd_rn(ra.y, __dmul_rn(beta, pa.y));
            p2[i] = pa;
        }
        if ((rows & 1) && tid == 0) {
            const int64_t j = rows - 1;
            const double pj = a.p[j];
            if (XL) a.x[j] = __dadd_rn(a.x[j], __dmul_rn(alpha, pj));
            if (!stop) a.p[j] = __dadd_rn(a.r[j], __dmul_rn(beta, pj));
        }
    } else {
        // a part with a halo: p lives in extended-box order.  One warp per owned x-line
        // (own_n0 consecutive rows <-> own_n0 consecutive columns): one division per line
        // instead of two per row, coalesced, four elements per lane in flight
        const int64_t n0 = a.g.own_n[0], n1 = a.g.own_n[1];
        const int64_t nlines = n1 * a.g.own_n[2];
        const int64_t E0 = a.g.ext_n[0], E1 = a.g.ext_n[1];
        const int lane = threadIdx.x & 31;
        const int64_t wid = tid >> 5, nw = stride >> 5;
        for (int64_t line = wid; line < nlines; line += nw) {
            const int64_t lz = line / n1, ly = line - lz * n1;
            const int64_t i0 = line * n0;
            const int64_t c0 = a.g.off[0] + E0 * ((ly + a.g.off[1]) + E1 * (lz + a.g.off[2]));
            for (int64_t lx = lane; lx < n0; lx += 4 * 32) {
                double pc[4], xi[4], ri[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int64_t e = lx + 32 * u;
                    if (e < n0) {
                        pc[u] = a.p[c0 + e];
                        if (XL) xi[u] = a.x[i0 + e];
                        ri[u] = a.r[i0 + e];
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int64_t e = lx + 32 * u;
                    if (e < n0) {
                        if (XL) a.x[i0 + e] = __dadd_rn(xi[u], __dmul_rn(alpha, pc[u]));
                        if (!stop) a.p[c0 + e] = __dadd_rn(ri[u], __dmul_rn(beta, pc[u]));
                    }
                }
            }
        }
    }
    // device comm: the halo columns of p_(k+1) from the neighbours' r_(k+1);
    // not once the solve stops (a uniform decision)
    if (a.halo_n > 0 && !stop) halo_p_update(a, a.halo_kp, beta, a.p, a.p);
}

// K7 of the deferred-x scheme (launch_update_p2): the x update of iteration k is
// fl(x + fl(alpha_k p_k)) exactly as in K7, only deferred: p_(k+1) goes to the next buffer of
// a ring of X, and every X-th K7 (or one that stops) applies the pending updates
// j = X floor((k-1)/X) + 1 .. k in order with one pass over x.  The ring buffer p_(k+1) goes
// to holds p_(k-X+1), read (as the first pending update) before it is overwritten.  FLUSH
// (k a multiple of X, decided on the host) is a separate instantiation so the plain p update
// keeps its registers; a stop in a non-flush K7 leaves the pending updates to k_x2_finish.
template <bool IDENT, bool FLUSH>
__global__ void __launch_bounds__(UPD_THREADS) k_update_p2(UpdArgs a, int k, const double *pk,
                                                           double *po) {
    __shared__ unsigned long long s_in[ACC_WORDS];
    __shared__ double s_beta;
    __shared__ int s_stop;
    KT_SCOPE(2, k);
    PreScalars ps;                       // K6 stopped: x_finish applies what is pending
    if (!upd_entry(a, k, 1, s_in, ps)) return;
    __syncthreads();
    const double fin = threadIdx.x < 32 ? acc_finalize_warp(s_in) : 0.0;   // warp 0
    if (threadIdx.x == 0) {
        double beta;
        s_stop = rr_decision_v(fin, k, ps.rr_old, ps.stop_thr, a.hist, a.rr, a.st, beta);
        s_beta = beta;
    }
    __syncthreads();
    const int X = a.xdef;
    const bool stop = s_stop, flush = FLUSH;
    const int j0 = X * ((k - 1) / X) + 1;              // first pending update
    if (blockIdx.x == 0 && threadIdx.x == 0 && flush) a.st->x_done = k;
    if (!stop && blockIdx.x == 0 && a.acc_zero)
        for (int i = threadIdx.x; i < ACC_WORDS; i += blockDim.x) a.acc_zero[i] = 0ull;
    const double beta = s_beta;
    // the pending updates: alpha_j and p_j (p_k = pk)
    double al[XDEF_MAX];
    const double *pj[XDEF_MAX];
#pragma unroll
    for (int q = 0; q < XDEF_MAX; ++q) {
        const int j = j0 + q;
        al[q] = (flush && j <= k) ? a.alpha_hist[j] : 0.0;
        pj[q] = (flush && j <= k) ? a.ring[(j - 1) % X] : nullptr;
    }
    const int np = flush ? k - j0 + 1 : 0;
    auto xflush = [&](double x, int64_t c) {
#pragma unroll
        for (int q = 0; q < XDEF_MAX; ++q)
            if (q < np) x = __dadd_rn(x, __dmul_rn(al[q], pj[q][c]));
        return x;
    };
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    if (!IDENT) {
        // a part with a halo: p buffers in extended-box order, one warp per owned x-line (as
        // k_update_p); the halo columns of po are written by the exchange meanwhile
        const int64_t n0 = a.g.own_n[0], n1 = a.g.own_n[1];
        const int64_t nlines = n1 * a.g.own_n[2];
        const int64_t E0 = a.g.ext_n[0], E1 = a.g.ext_n[1];
        const int lane = threadIdx.x & 31;
        for (int64_t line = tid >> 5; line < nlines; line += stride >> 5) {
            const int64_t lz = line / n1, ly = line - lz * n1;
            const int64_t i0 = line * n0;
            const int64_t c0 = a.g.off[0] + E0 * ((ly + a.g.off[1]) + E1 * (lz + a.g.off[2]));
            for (int64_t lx = lane; lx < n0; lx += 4 * 32) {
                double pv[4], rv[4], xv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {          // four elements per lane in flight
                    const int64_t e = lx + 32 * u;
                    if (e < n0) {
                        pv[u] = pk[c0 + e];
                        rv[u] = stop ? 0.0 : a.r[i0 + e];
                        if (flush) xv[u] = a.x[i0 + e];
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int64_t e = lx + 32 * u;
                    if (e < n0) {
                        if (flush) a.x[i0 + e] = xflush(xv[u], c0 + e);
                        if (!stop) po[c0 + e] = __dadd_rn(rv[u], __dmul_rn(beta, pv[u]));
                    }
                }
            }
        }
        // device comm: the halo columns of p_(k+1) (as k_update_p)
        if (a.halo_n > 0 && !stop) halo_p_update(a, a.halo_kp, beta, pk, po);
        return;
    }
    const int64_t rows = a.g.rows, n2 = rows >> 1;
    double2 *x2 = reinterpret_cast<double2 *>(a.x);
    const double2 *r2 = reinterpret_cast<const double2 *>(a.r);
    const double2 *pk2 = reinterpret_cast<const double2 *>(pk);
    double2 *po2 = reinterpret_cast<double2 *>(po);
    for (int64_t i = tid; i < n2; i += stride) {
        const double2 pv = pk2[i];
        if (flush) {
            double2 xv = x2[i];
#pragma unroll
            for (int q = 0; q < XDEF_MAX; ++q)
                if (q < np) {
                    const double2 v = reinterpret_cast<const double2 *>(pj[q])[i];
                    xv.x = __dadd_rn(xv.x, __dmul_rn(al[q], v.x));
                    xv.y = __dadd_rn(xv.y, __dmul_rn(al[q], v.y));
                }
            x2[i] = xv;
        }
        if (!stop) {
            const double2 rv = r2[i];
            po2[i] = make_double2(__dadd_rn(rv.x, __dmul_rn(beta, pv.x)),
                                  __dadd_rn(rv.y, __dmul_rn(beta, pv.y)));
        }
    }
    if ((rows & 1) && tid == 0) {
        const int64_t j = rows - 1;
        const double pv = pk[j];
        if (flush) a.x[j] = xflush(a.x[j], j);
        if (!stop) po[j] = __dadd_rn(a.r[j], __dmul_rn(beta, pv));
    }
}

// After the loop: the x updates still pending (a stop in K6, or an iteration count that is
// not a multiple of X), j = x_done + 1 .. alpha_iter, in order.
template <bool IDENT>
__global__ void __launch_bounds__(UPD_THREADS) k_x2_finish(UpdArgs a) {
    const int j0 = a.st->x_done + 1, j1 = a.st->alpha_iter;
    if (j0 > j1) return;
    const int X = a.xdef;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.g.rows; i += stride) {
        const int64_t c = IDENT ? i : row_to_col(a.g, i);
        double x = a.x[i];
        for (int j = j0; j <= j1; ++j)
            x = __dadd_rn(x, __dmul_rn(a.alpha_hist[j], a.ring[(j - 1) % X][c]));
        a.x[i] = x;
    }
}

// Halo values of p_(k+1) computed ahead of K7 (SYM with a halo): the packed
// send buffer gets sendbuf[i] = fl(r[row_i] + fl(beta_k p_k[col_i])) -- K7's formula on K7's
// inputs, beta_k from the same exact rr -- so the exchange can run while K7 updates p.
__global__ void __launch_bounds__(UPD_THREADS) k_pack_next_p(UpdArgs a, int k,
                                                             const int32_t *send_row,
                                                             const int32_t *send_col,
                                                             double *sendbuf, int64_t n) {
    __shared__ unsigned long long s_in[ACC_WORDS];
    __shared__ double s_beta;
    if (a.st->done) return;
    if (!acc_in_load(s_in, a, k, 1)) return;
    __syncthreads();
    if (threadIdx.x < 32) {
        const double rr_new = acc_finalize_warp(s_in);
        if (threadIdx.x == 0) s_beta = __ddiv_rn(rr_new, a.rr[k - 1]);   // as rr_decision
    }
    __syncthreads();
    const double beta = s_beta;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        sendbuf[i] = __dadd_rn(a.r[send_row[i]], __dmul_rn(beta, a.p[send_col[i]]));
}

// a1, device-initiated (MINIFE_TRANSPORT_PUSH / device comm): every send slot's value is
// stored straight into the receiving part's halo column -- another part's array on this GPU
// (VIRTUAL), a peer GPU's array over NVLink (MULTI, peer access) or a CUDA-IPC mapping of
// another rank's array (RANK).  No pack, no wire, no unpack.
// mode 0: the value is p[send_col]; mode 1: p_(k+1) = fl(r + fl(beta_k p)) as k_pack_next_p.
__global__ void __launch_bounds__(UPD_THREADS) k_push(UpdArgs a, int k, int mode,
                                                      const int32_t *send_row,
                                                      const int32_t *send_col,
                                                      const uint8_t *slot_nbr,
                                                      const int32_t *dst_col,
                                                      double *const *dst_ptr, int64_t n) {
    __shared__ unsigned long long s_in[ACC_WORDS];
    __shared__ double s_beta;
    if (mode == 1) {
        if (a.st->done) return;
        if (!acc_in_load(s_in, a, k, 1)) return;
        __syncthreads();
        if (threadIdx.x < 32) {
            const double rr_new = acc_finalize_warp(s_in);
            if (threadIdx.x == 0) s_beta = __ddiv_rn(rr_new, a.rr[k - 1]);   // as rr_decision
        }
        __syncthreads();
    }
    const double beta = mode == 1 ? s_beta : 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double pv = a.p[send_col[i]];
        const double v = mode == 1 ? __dadd_rn(a.r[send_row[i]], __dmul_rn(beta, pv)) : pv;
        dst_ptr[slot_nbr[i]][dst_col[i]] = v;
    }
}

// ----------------------------------------------------------------------------------------
// fused scheme, second kernel of iteration k (K6'): alpha_k, r -= alpha Ap, exact rr_k.
// x is not touched here (its update for iteration k is applied by the next fused SpMV or by
// k_cg_finish).  One part only (rows == columns).
// ----------------------------------------------------------------------------------------

__global__ void __launch_bounds__(UPD_THREADS) k_update_r(UpdArgs a, int k,
                                                          unsigned long long *acc_pAp_next) {
    __shared__ unsigned long long sacc[ACC_WORDS], s_in[ACC_WORDS];
    __shared__ int sdig[ACC_DIG16];
    __shared__ double s_alpha;
    __shared__ int s_stop;
    if (a.st->done) return;
    acc_zero_shared(sacc, sdig);
    if (!acc_in_load(s_in, a, k, 0)) return;
    __syncthreads();
    const double fin = threadIdx.x < 32 ? acc_finalize_warp(s_in) : 0.0;   // warp 0
    if (threadIdx.x == 0) {
        double alpha;
        s_stop = xr_prologue(a, fin, k, alpha);
        s_alpha = alpha;
    }
    __syncthreads();
    if (s_stop) return;
    if (blockIdx.x == 0)                          // consumed by K6' of k-1: free for k+1
        for (int i = threadIdx.x; i < ACC_WORDS; i += blockDim.x) acc_pAp_next[i] = 0ull;
    const double alpha = s_alpha;
    Expansion ex[2];
    ex[0].init();
    ex[1].init();
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t rows = a.g.rows, n2 = rows >> 1;
    double2 *r2 = reinterpret_cast<double2 *>(a.r);
    const double2 *q2 = reinterpret_cast<const double2 *>(a.Ap);
    int64_t i = tid;
    for (; i + stride < n2; i += 2 * stride) {
        double2 ra = r2[i], qa = q2[i], rb = r2[i + stride], qb = q2[i + stride];
        ra.x = __dsub_rn(ra.x, __dmul_rn(alpha, qa.x));
        ra.y = __dsub_rn(ra.y, __dmul_rn(alpha, qa.y));
        rb.x = __dsub_rn(rb.x, __dmul_rn(alpha, qb.x));
        rb.y = __dsub_rn(rb.y, __dmul_rn(alpha, qb.y));
        r2[i] = ra;
        r2[i + stride] = rb;
        ex[0].add(__dmul_rn(ra.x, ra.x), sacc);
        ex[1].add(__dmul_rn(ra.y, ra.y), sacc);
        ex[0].add(__dmul_rn(rb.x, rb.x), sacc);
        ex[1].add(__dmul_rn(rb.y, rb.y), sacc);
    }
    for (; i < n2; i += stride) {
        double2 ra = r2[i], qa = q2[i];
        ra.x = __dsub_rn(ra.x, __dmul_rn(alpha, qa.x));
        ra.y = __dsub_rn(ra.y, __dmul_rn(alpha, qa.y));
        r2[i] = ra;
        ex[0].add(__dmul_rn(ra.x, ra.x), sacc);
        ex[1].add(__dmul_rn(ra.y, ra.y), sacc);
    }
    if ((rows & 1) && tid == 0) {
        const int64_t j = rows - 1;
        const double rj = __dsub_rn(a.r[j], __dmul_rn(alpha, a.Ap[j]));
        a.r[j] = rj;
        ex[0].add(__dmul_rn(rj, rj), sacc);
    }
    ex[0].warp_flush(sacc);
    ex[1].warp_flush(sacc);
    __syncthreads();
    acc_merge_to_global(sacc, sdig, a.acc_out);
}

// After the last iteration K: finalise rr_K (hist[K], stop flags) unless a stop test already
// fired, then apply the pending x update x += fl(alpha_j p_j) if iteration j = alpha_iter has
// not been applied yet (p_j lives in buffer j % 2).
__global__ void __launch_bounds__(UPD_THREADS) k_cg_finish(UpdArgs a, int K, const double *p_even,
                                                           const double *p_odd) {
    __shared__ unsigned long long s_in[ACC_WORDS];
    __shared__ int s_apply, s_iter;
    __shared__ double s_alpha;
    const int done = a.st->done;
    if (!done && blockIdx.x == 0) {
        acc_load_shared(s_in, a.acc_in);
        __syncthreads();
        const double fin = threadIdx.x < 32 ? acc_finalize_warp(s_in) : 0.0;   // warp 0
        if (threadIdx.x == 0) {
            double beta;
            rr_decision(fin, K, a.hist, a.rr, a.st, beta);
        }
    }
    if (threadIdx.x == 0) {
        s_iter = a.st->alpha_iter;
        s_apply = s_iter > a.st->x_done;
        s_alpha = a.st->alpha;
    }
    __syncthreads();
    if (!s_apply) return;
    const double *p = (s_iter & 1) ? p_odd : p_even;
    const double alpha = s_alpha;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.g.rows; i += stride)
        a.x[i] = __dadd_rn(a.x[i], __dmul_rn(alpha, p[i]));
}

// ----------------------------------------------------------------------------------------
// a3-a6, TMA-pipelined (one part: rows == columns): the vector streams are staged in shared
// memory by bulk copies (producer warp), consumer warps compute from smem and store with
// streaming stores.  Bytes in flight per SM = STAGES x tile, independent of occupancy.
// Vectors are allocated with >= 32 doubles of padding, so a tile copy may round its size up
// to 16 B; rows >= a.g.rows are never written.
// ----------------------------------------------------------------------------------------

constexpr int UT_ROWS = 1024;                         // rows per tile
constexpr int UT_STAGES = 6;                          // 6 x 32 KB in flight per SM (K6)
constexpr int UT_CWARPS = 8;                          // consumer warps
constexpr int UT_THREADS = 32 * (UT_CWARPS + 1);      // + producer warp


// Pure-read probe with the same bulk-copy engine (B_read for the TMA kernels).
__global__ void __launch_bounds__(UT_THREADS, 1) k_read_tma(const double *src, int64_t n,
                                                            int passes) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double *sm = reinterpret_cast<double *>(smem_raw);
    __shared__ __align__(8) uint64_t full_bar[UT_STAGES], empty_bar[UT_STAGES];
    constexpr int TD = 4 * UT_ROWS;                   // 32 KB tiles
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < UT_STAGES; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], UT_CWARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int64_t ntiles = n / TD;
    const int64_t total = ntiles * passes;          // passes > 1: L2-resident re-reads
    if (warp == UT_CWARPS) {
        if (lane == 0) {
            uint64_t pol = evict_first_policy();
            if (passes > 1)
                asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
            int64_t i = 0;
            for (int64_t t = blockIdx.x; t < total; t += gridDim.x, ++i) {
                const int st = (int)(i % UT_STAGES);
                if (i >= UT_STAGES) mbar_wait(&empty_bar[st], (uint32_t)(((i / UT_STAGES) & 1) ^ 1));
                mbar_expect_tx(&full_bar[st], TD * 8);
                bulk_g2s(sm + (size_t)st * TD, src + (t % ntiles) * TD, TD * 8, &full_bar[st], pol);
            }
        }
    } else {
        int64_t i = 0;
        for (int64_t t = blockIdx.x; t < total; t += gridDim.x, ++i) {
            const int st = (int)(i % UT_STAGES);
            mbar_wait(&full_bar[st], (uint32_t)((i / UT_STAGES) & 1));
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty_bar[st]);
        }
    }
}

// ----------------------------------------------------------------------------------------
// a1: halo pack / unpack / virtual-rank transport
// ----------------------------------------------------------------------------------------

__global__ void k_move(const double *__restrict__ src, const int32_t *__restrict__ sidx,
                       double *__restrict__ dst, const int32_t *__restrict__ didx, int64_t n) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        dst[didx ? didx[i] : i] = src[sidx ? sidx[i] : i];
}

// ----------------------------------------------------------------------------------------
// roofline probes: pure-read fp64 stream and copy, 16-byte accesses
// ----------------------------------------------------------------------------------------

__global__ void __launch_bounds__(256) k_read_stream(const double2 *__restrict__ src, int64_t n2,
                                                     double *__restrict__ sink) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n2; i += 4 * stride) {
        const double2 a = __ldcs(src + i), b = __ldcs(src + i + stride),
                      c = __ldcs(src + i + 2 * stride), d = __ldcs(src + i + 3 * stride);
        s0 += a.x + a.y;
        s1 += b.x + b.y;
        s2 += c.x + c.y;
        s3 += d.x + d.y;
    }
    for (; i < n2; i += stride) {
        const double2 a = __ldcs(src + i);
        s0 += a.x + a.y;
    }
    const double s = (s0 + s1) + (s2 + s3);
    if (s == 12345.678) sink[0] = s;       // keeps the loads alive; never true for 0-filled data
}

__global__ void __launch_bounds__(256) k_copy_stream(const double2 *__restrict__ src,
                                                     double2 *__restrict__ dst, int64_t n2) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + stride < n2; i += 2 * stride) {
        const double2 a = __ldcs(src + i), b = __ldcs(src + i + stride);
        __stcs(dst + i, a);
        __stcs(dst + i + stride, b);
    }
    for (; i < n2; i += stride) __stcs(dst + i, __ldcs(src + i));
}

__global__ void __launch_bounds__(256) k_write_stream(double2 *__restrict__ dst, int64_t n2) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const double2 v = make_double2(0.0, 0.0);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride)
        __stcs(dst + i, v);
}

double g_write_gbs = 0.0;                 // last probe_bandwidth: pure-write stream rate

cudaError_t probe_bandwidth(int64_t bytes, int reps, double *read_gbs, double *copy_gbs) {
    query_occupancy();
    const int64_t n2 = bytes / 16;
    double2 *a = nullptr, *b = nullptr;
    double *sink = nullptr;
    cudaEvent_t e0, e1;
    cudaError_t e = cudaMalloc((void **)&a, n2 * 16);
    if (e == cudaSuccess) e = cudaMalloc((void **)&b, n2 * 16);
    if (e == cudaSuccess) e = cudaMalloc((void **)&sink, 8);
    if (e == cudaSuccess) e = cudaMemset(a, 0, n2 * 16);
    if (e == cudaSuccess) e = cudaMemset(b, 0, n2 * 16);
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = g_sms * 8;
    float best_r = 1e30f, best_c = 1e30f;
    for (int r = 0; e == cudaSuccess && r < reps + 1; ++r) {
        float ms = 0.f;
        cudaEventRecord(e0);
        k_read_stream<<<grid, 256>>>(a, n2, sink);
        cudaEventRecord(e1);
        e = cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0) best_r = std::min(best_r, ms);
        cudaEventRecord(e0);
        k_copy_stream<<<grid, 256>>>(a, b, n2);
        cudaEventRecord(e1);
        if (e == cudaSuccess) e = cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0) best_c = std::min(best_c, ms);
    }
    // pure-write stream (the roof of the assembly kernel, which reads nothing)
    {
        float best_w = 1e30f;
        for (int r = 0; e == cudaSuccess && r < reps + 1; ++r) {
            float ms = 0.f;
            cudaEventRecord(e0);
            k_write_stream<<<grid, 256>>>(b, n2);
            cudaEventRecord(e1);
            e = cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            if (r > 0) best_w = std::min(best_w, ms);
        }
        g_write_gbs = (double)(n2 * 16) / (best_w * 1e-3) / 1e9;
    }
    // the bulk-copy engine's read rate (what the TMA-pipelined kernels can draw)
    static unsigned long long attr = 0;
    if (e == cudaSuccess) e = ensure_smem_attr(k_read_tma, UT_STAGES * 4 * UT_ROWS * 8, attr);
    for (int r = 0; e == cudaSuccess && r < reps + 1; ++r) {
        float ms = 0.f;
        cudaEventRecord(e0);
        k_read_tma<<<g_sms, UT_THREADS, UT_STAGES * 4 * UT_ROWS * 8>>>(
            reinterpret_cast<const double *>(a), (n2 * 2) / (4 * UT_ROWS) * (4 * UT_ROWS), 1);
        cudaEventRecord(e1);
        e = cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        const float scaled = ms * (float)((double)(n2 * 16) /
                                          (double)((n2 * 2) / (4 * UT_ROWS) * (4 * UT_ROWS) * 8));
        if (r > 0) best_r = std::min(best_r, scaled);
    }
    // L2-resident read through the same engine: a 48 MB buffer (fits the 126 MB L2) read 40
    // times within one launch
    {
        const int64_t nl = (int64_t)6 << 20;                     // doubles = 48 MB
        const int passes = 40;
        float best_l2 = 1e30f;
        for (int r = 0; e == cudaSuccess && r < reps + 2; ++r) {
            float ms = 0.f;
            cudaEventRecord(e0);
            k_read_tma<<<g_sms, UT_THREADS, UT_STAGES * 4 * UT_ROWS * 8>>>(
                reinterpret_cast<const double *>(a), nl, passes);
            cudaEventRecord(e1);
            e = cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            if (r > 1) best_l2 = std::min(best_l2, ms);
        }
        g_l2_read_gbs = (double)(nl * 8) * passes / (best_l2 * 1e-3) / 1e9;
    }
    if (e == cudaSuccess) e = cudaGetLastError();
    cudaFree(a);
    cudaFree(b);
    cudaFree(sink);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (e == cudaSuccess) {
        *read_gbs = (double)(n2 * 16) / (best_r * 1e-3) / 1e9;
        *copy_gbs = 2.0 * (double)(n2 * 16) / (best_c * 1e-3) / 1e9;
    }
    return e;
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

// C5 as a standalone operation: acc += sum^exact fl(u_i v_i) (the same three levels as the
// CG kernels' epilogues), then k_acc_round.
__global__ void __launch_bounds__(UPD_THREADS) k_dot(const double *__restrict__ u,
                                                     const double *__restrict__ v, int64_t n,
                                                     unsigned long long *acc) {
    __shared__ unsigned long long sacc[ACC_WORDS];
    __shared__ int sdig[ACC_DIG16];
    acc_zero_shared(sacc, sdig);
    __syncthreads();
    Expansion ex;
    ex.init();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        ex.add(__dmul_rn(u[i], v[i]), sacc);
    expansion_flush_digits(ex, sdig, sacc);
    __syncthreads();
    acc_merge_to_global(sacc, sdig, acc);
}

// *out = RN(value of the accumulator), one warp.
__global__ void k_acc_round(const unsigned long long *acc, double *out) {
    __shared__ unsigned long long s_in[ACC_WORDS];
    acc_load_shared(s_in, acc);
    __syncwarp();
    const double v = acc_finalize_warp(s_in);
    if (threadIdx.x == 0) *out = v;
}

__global__ void k_extract_rows(Matrix m, Geom g, const int64_t *rows, int64_t n,
                               int32_t *out_col, double *out_val, int32_t *out_len) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t row = rows[i];
    // storage row: SYM-ext stores rows by extended column
    const int64_t srow = m.ext ? row_to_col(g, row) : row;
    const int64_t lane = srow & 31;
    const int64_t s = (m.fmt != FMT_CRS && m.slice_pos) ? (int64_t)m.slice_pos[srow >> 5]
                                                        : (srow >> 5);   // storage slice
    int len = 0;
    if (m.fmt == FMT_CRS) {
        len = m.row_len[row];
        for (int k = 0; k < len; ++k) {
            out_col[27 * i + k] = m.col[m.slice_off[s] + 32 * k + lane];
            out_val[27 * i + k] = m.val[m.slice_off[s] + 32 * k + lane];
        }
    } else {
        const unsigned msk = m.mask[s * 32 + lane] & ~SYM_OWNED;
        for (int t = 0; t < 27; ++t) {
            if (!((msk >> t) & 1u)) continue;
            const int c = m.seg[(9 * s + t / 3) * 32 + lane] + t % 3;
            out_col[27 * i + len] = c;
            if (m.fmt == FMT_SEG)
                out_val[27 * i + len] = m.val[(27 * s + t) * 32 + lane];
            else if (t >= 13)                  // SYM: own upper slot
                out_val[27 * i + len] = m.val[(14 * s + (t - 13)) * 32 + lane];
            else                               // SYM: mirror slot of row c (one part)
                out_val[27 * i + len] = m.val[((int64_t)(c >> 5) * 14 + (13 - t)) * 32 + (c & 31)];
            ++len;
        }
    }
    out_len[i] = len;
}

// ----------------------------------------------------------------------------------------
// launch wrappers
// ----------------------------------------------------------------------------------------

static void query_occupancy() {
    if (g_sms) return;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_spmv_bps[0], k_spmv_crs<true, true>,
                                                  SPMV_THREADS, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_spmv_bps[1], k_spmv_seg<true>,
                                                  SPMV_THREADS, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_upd_bps, k_update_xr<true, true>, UPD_THREADS, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_updp_bps, k_update_p<true, true>, UPD_THREADS, 0);
    if (g_updp_bps <= 0) g_updp_bps = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_updr_bps, k_update_r, UPD_THREADS, 0);
    if (g_updr_bps <= 0) g_updr_bps = 1;
    if (g_sms <= 0) g_sms = 148;
    for (int f = 0; f < 2; ++f)
        if (g_spmv_bps[f] <= 0) g_spmv_bps[f] = 1;
    if (g_upd_bps <= 0) g_upd_bps = 1;
}

int spmv_grid(int64_t nslices, int fmt) {
    query_occupancy();
    const int64_t need = (nslices + (SPMV_THREADS / 32) - 1) / (SPMV_THREADS / 32);
    const int64_t full = (int64_t)g_sms * g_spmv_bps[fmt == FMT_SEG];
    return (int)(need < full ? (need > 0 ? need : 1) : full);
}

int stream_grid(int64_t rows) {
    query_occupancy();
    const int64_t need = (rows + UPD_THREADS - 1) / UPD_THREADS;
    const int64_t full = (int64_t)g_sms * g_upd_bps;
    return (int)(need < full ? (need > 0 ? need : 1) : full);
}

cudaError_t launch_rowlen_widths(const Geom &g, uint8_t *row_len, uint8_t *width,
                                 int64_t nslices, cudaStream_t s) {
    const int64_t threads = nslices * 32;
    k_rowlen_widths<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(g, row_len, width, nslices);
    return cudaGetLastError();
}

// grid-stride: at most 8 CTAs of 256 threads per SM (each builds the C1/C2 table once)
#ifndef ASM_CTAS_PER_SM
#define ASM_CTAS_PER_SM 128
#endif
cudaError_t launch_assemble(const AsmArgs &a, cudaStream_t s) {
    query_occupancy();
    const bool symx = a.fmt == FMT_SYM && !a.g.ident;
    const int64_t threads = (((symx ? a.g.ncols : a.g.rows) + 31) >> 5) * 32;
    // many short grid-stride CTAs (128 per SM): CTAs retire at different times and the store
    // streams of the next ones fill in.  B200, 300^3 SYM, interleaved A/B (profiles/r02/ab):
    // 8 per SM 0.91 ms, 32 0.85, 64 0.80, 128 0.77 (0.86 of copy, 0.94 of the write probe),
    // 256 0.83, one row per thread 1.36 (the C1 table per CTA dominates)
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((threads + 255) / 256,
                                                                (int64_t)g_sms * ASM_CTAS_PER_SM));
    if (symx) k_assemble_symx<<<(unsigned)grid, 256, 0, s>>>(a);
    else k_assemble<<<(unsigned)grid, 256, 0, s>>>(a);
    return cudaGetLastError();
}

template <bool DOT, int FMT, bool IDENT, bool FUSED = false>
static cudaError_t launch_tma(const SpmvArgs &a, cudaStream_t s) {
    constexpr int SMEM = TmaCfg<FMT>::SMEM;
    static unsigned long long attr_set = 0;   // per instantiation, one bit per device
    cudaError_t e = ensure_smem_attr(k_spmv_tma<DOT, FMT, IDENT, FUSED>, SMEM, attr_set);
    if (e != cudaSuccess) return e;
    query_occupancy();
    const int64_t ntiles = (a.s_end - a.s_begin + TILE - 1) / TILE;
    const int grid = (int)std::min<int64_t>(ntiles, g_sms);
    k_spmv_tma<DOT, FMT, IDENT, FUSED><<<grid > 0 ? grid : 1, TMA_THREADS, SMEM, s>>>(a);
    return cudaGetLastError();
}

// 3-D tensor maps of the SYM value array [nslices][14][32] doubles, viewed slot-major: boxes of
// {32, gs, 3} and {32, gs, 1}.  cuTensorMapEncodeTiled comes from the driver through the runtime (no -lcuda).
static bool sym_maps(const Matrix &m, int gs, CUtensorMap *m3, CUtensorMap *m1) {
    static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    if (!enc) {
        cudaDriverEntryPointQueryResult q;
        void *fn = nullptr;
        if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000,
                                             cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return false;
        enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    // slot-major view [14][nslices][32] of the [nslices][14][32] array (dim 1 = slice, stride
    // 14 * 256 B; dim 2 = slot, stride 256 B): a box lands as [slot][slice][lane]
    const cuuint64_t dims[3] = {32, (cuuint64_t)m.nslices, 14};
    const cuuint64_t strides[2] = {14 * 32 * 8, 32 * 8};
    const cuuint32_t box3[3] = {32, (cuuint32_t)gs, 3}, box1[3] = {32, (cuuint32_t)gs, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    void *base = const_cast<double *>(m.val);
    return enc(m3, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box3, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
               CUDA_SUCCESS &&
           enc(m1, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box1, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
               CUDA_SUCCESS;
}

template <bool DOT, int NW, int NST, int EA, int EB>
static cudaError_t launch_symm_t(const SpmvArgs &a, const CUtensorMap &m3, const CUtensorMap &m1,
                                 cudaStream_t s) {
    using C = SymmCfg<NW, NST>;
    static unsigned long long attr_set = 0;
    cudaError_t e = ensure_smem_attr(k_spmv_symm<DOT, NW, NST, EA, EB>, C::SMEM, attr_set);
    if (e != cudaSuccess) return e;
    query_occupancy();
    const int64_t ntiles = (a.m.nslices + NW - 1) / NW;
    const int g = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, g_sms));
    k_spmv_symm<DOT, NW, NST, EA, EB><<<g, C::THREADS, C::SMEM, s>>>(a, m3, m1);
    return cudaGetLastError();
}

template <bool DOT, int NW, int NST>
static cudaError_t launch_symm(const SpmvArgs &a, cudaStream_t s) {
    using C = SymmCfg<NW, NST>;
    static_assert(C::SMEM + 1536 <= 232448, "SYMM tile exceeds shared memory");
    CUtensorMap m3, m1;
    if (!sym_maps(a.m, C::GS, &m3, &m1)) return cudaErrorNotSupported;
    if (DOT && a.m.nslices < SYMM_SMALL_TIER_SLICES)
        return launch_symm_t<DOT, NW, NST, 2, 2>(a, m3, m1, s);
    return launch_symm_t<DOT, NW, NST, 4, 4>(a, m3, m1, s);
}

// SYM tile shape (B200, 300^3: 16 consumer warps x 2 stages 0.90 ms/launch, 12 x 3 0.95 ms,
// 8 x 4 1.31 ms -- the kernel is bound by the latency of its L2 gathers, so warps beat stages)
template <bool DOT>
static cudaError_t launch_sym(const SpmvArgs &a, cudaStream_t s) {
    // default: mirrored values staged by tensor-map TMA (13 consumer warps, 2 stages; B200,
    // 300^3: 1.196 ms per CG iteration vs 1.243 with L1 mirror gathers, profiles/r01/session2);
    // the ctx option "sym_kernel" = 0 (or no tensor-map support) selects the L1-gather kernel
    if (a.sym_kernel != 0) {
        const cudaError_t e = a.symm_nw == SYMM_NW_WIDE ? launch_symm<DOT, SYMM_NW_WIDE, 2>(a, s)
                                                        : launch_symm<DOT, SYMM_NW, 2>(a, s);
        if (e != cudaErrorNotSupported) return e;
        // (no tensor-map support: the L1-gather kernel below, same results; the library
        // never prints)
    }
    using C = SyCfg<16, 2>;
    static unsigned long long attr_set = 0;
    cudaError_t e = ensure_smem_attr(k_spmv_sym<DOT, 16, 2>, C::SMEM, attr_set);
    if (e != cudaSuccess) return e;
    query_occupancy();
    const int64_t ntiles = (a.m.nslices + C::TILE - 1) / C::TILE;
    const int g = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, g_sms));
    k_spmv_sym<DOT, 16, 2><<<g, C::THREADS, C::SMEM, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_update_r(const UpdArgs &a, int k, unsigned long long *acc_pAp_next_zero,
                            int grid, cudaStream_t s) {
    query_occupancy();
    const int64_t need = (a.g.rows / 2 + UPD_THREADS - 1) / UPD_THREADS;
    const int g6 = (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)g_sms * g_updr_bps));
    (void)grid;
    k_update_r<<<g6, UPD_THREADS, 0, s>>>(a, k, acc_pAp_next_zero);
    return cudaGetLastError();
}

cudaError_t launch_cg_finish(const UpdArgs &a, int K, const double *p_even, const double *p_odd,
                             int grid, cudaStream_t s) {
    k_cg_finish<<<grid, UPD_THREADS, 0, s>>>(a, K, p_even, p_odd);
    return cudaGetLastError();
}

// Kernel choice per format (measured on B200, 300^3, profiles/r01): SEG -> TMA pipeline
// (1.105 ms vs 1.442 ms register-streaming); CRS -> register streaming (1.48 ms vs 1.77 ms
// for its 2-stage TMA variant).  The ctx option "spmv_impl" (1 TMA, 0 register streaming)
// overrides the choice for experiments.
static int spmv_impl(int fmt, int forced) {
    if (fmt == FMT_SYM) return 1;                       // TMA kernel only
    if (forced >= 0) return forced;
    return fmt == FMT_SEG ? 1 : 0;
}

cudaError_t launch_spmv(const SpmvArgs &a, bool with_dot, int grid, cudaStream_t s) {
    if (a.s_end <= a.s_begin) return cudaSuccess;           // empty slice range
    if (a.fused_k > 0) {
        if (a.m.fmt != FMT_SEG || !a.g.ident || !with_dot) return cudaErrorInvalidValue;
        return launch_tma<true, FMT_SEG, true, true>(a, s);
    }
    if (a.m.fmt == FMT_SYM) {
        return with_dot ? launch_sym<true>(a, s) : launch_sym<false>(a, s);
    }
    if (spmv_impl(a.m.fmt, a.impl) == 1) {
        if (a.m.fmt == FMT_SEG)
            return with_dot ? launch_tma<true, FMT_SEG, true>(a, s)
                            : launch_tma<false, FMT_SEG, true>(a, s);
        if (a.g.ident)
            return with_dot ? launch_tma<true, FMT_CRS, true>(a, s)
                            : launch_tma<false, FMT_CRS, true>(a, s);
        return with_dot ? launch_tma<true, FMT_CRS, false>(a, s)
                        : launch_tma<false, FMT_CRS, false>(a, s);
    }
    if (a.m.fmt == FMT_SEG) {
        if (with_dot) k_spmv_seg<true><<<grid, SPMV_THREADS, 0, s>>>(a);
        else k_spmv_seg<false><<<grid, SPMV_THREADS, 0, s>>>(a);
    } else if (a.g.ident) {
        if (with_dot) k_spmv_crs<true, true><<<grid, SPMV_THREADS, 0, s>>>(a);
        else k_spmv_crs<false, true><<<grid, SPMV_THREADS, 0, s>>>(a);
    } else {
        if (with_dot) k_spmv_crs<true, false><<<grid, SPMV_THREADS, 0, s>>>(a);
        else k_spmv_crs<false, false><<<grid, SPMV_THREADS, 0, s>>>(a);
    }
    return cudaGetLastError();
}

cudaError_t launch_cg_small(const Matrix &m, const UpdArgs &a, int K, double tol,
                            cudaStream_t s) {
    if (m.rows > SMALL_MAX_ROWS || !a.g.ident || (m.fmt != FMT_SEG && m.fmt != FMT_SYM) ||
        m.slice_row)
        return cudaErrorInvalidValue;
    if (m.fmt == FMT_SEG) k_cg_small<FMT_SEG><<<1, SMALL_THREADS, 0, s>>>(m, a, K, tol);
    else k_cg_small<FMT_SYM><<<1, SMALL_THREADS, 0, s>>>(m, a, K, tol);
    return cudaGetLastError();
}

// Can a CL_CTAS-CTA cluster of k_cg_cluster be scheduled on the current device (MIG, MPS or
// SM-limited partitions may not fit a non-portable 16-CTA cluster)?  Queried once per device.
bool cluster_solver_available() {
    static signed char known[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return false;
    signed char &k = known[dev & 63];
    if (k) return k > 0;
    const int smem = (int)sizeof(ClusterSmem);
    int n = 0;
    cudaError_t e = cudaFuncSetAttribute(k_cg_cluster<FMT_SYM, true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_cg_cluster<FMT_SYM, true>,
                                 cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e == cudaSuccess) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(CL_CTAS, 1, 1);
        cfg.blockDim = dim3(CL_THREADS, 1, 1);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = CL_CTAS;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        e = cudaOccupancyMaxActiveClusters(&n, k_cg_cluster<FMT_SYM, true>, &cfg);
    }
    if (e != cudaSuccess) cudaGetLastError();
    k = (e == cudaSuccess && n > 0) ? 1 : -1;
    return k > 0;
}

cudaError_t launch_cg_cluster(const Matrix &m, const UpdArgs &a, int K, double tol,
                              cudaStream_t s) {
    if (m.rows > CL_MAX_ROWS || (m.nslices + CL_CTAS - 1) / CL_CTAS > CL_MAX_SL ||
        !a.g.ident || (m.fmt != FMT_SEG && m.fmt != FMT_SYM) || m.slice_row)
        return cudaErrorInvalidValue;
    const int dd = a.cl_dd;
    auto kern = m.fmt == FMT_SEG ? (dd ? k_cg_cluster<FMT_SEG, true> : k_cg_cluster<FMT_SEG, false>)
                                 : (dd ? k_cg_cluster<FMT_SYM, true> : k_cg_cluster<FMT_SYM, false>);
    const int smem = (int)sizeof(ClusterSmem);
    static unsigned long long set = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    if (!((set >> (dev & 63)) & 1ull)) {
        void (*ks[4])(Matrix, UpdArgs, int, double) = {
            k_cg_cluster<FMT_SEG, true>, k_cg_cluster<FMT_SYM, true>,
            k_cg_cluster<FMT_SEG, false>, k_cg_cluster<FMT_SYM, false>};
        for (auto kf : ks) {
            cudaError_t e =
                cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            if (e == cudaSuccess)
                e = cudaFuncSetAttribute(kf, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            if (e != cudaSuccess) return e;
        }
        set |= 1ull << (dev & 63);
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CL_CTAS, 1, 1);
    cfg.blockDim = dim3(CL_THREADS, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL_CTAS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, m, a, K, tol);
}

cudaError_t launch_pack_next_p(const UpdArgs &a, int k, const int32_t *send_row,
                               const int32_t *send_col, double *sendbuf, int64_t n,
                               cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const int g = (int)std::min<int64_t>((n + UPD_THREADS - 1) / UPD_THREADS, 4 * 148);
    k_pack_next_p<<<g, UPD_THREADS, 0, s>>>(a, k, send_row, send_col, sendbuf, n);
    return cudaGetLastError();
}

cudaError_t launch_push(const UpdArgs &a, int k, int mode, const int32_t *send_row,
                        const int32_t *send_col, const uint8_t *slot_nbr, const int32_t *dst_col,
                        double *const *dst_ptr, int64_t n, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const int g = (int)std::min<int64_t>((n + UPD_THREADS - 1) / UPD_THREADS, 4 * 148);
    k_push<<<g, UPD_THREADS, 0, s>>>(a, k, mode, send_row, send_col, slot_nbr, dst_col, dst_ptr,
                                     n);
    return cudaGetLastError();
}

cudaError_t launch_push_r(const UpdArgs &a, int kp, const int32_t *send_row,
                          const uint8_t *slot_nbr, const int32_t *dst_slot,
                          double *const *dst_ptr, int64_t n, cudaStream_t s) {
    if (!a.dc.local || n <= 0) return cudaErrorInvalidValue;
    const int g = (int)std::min<int64_t>((n + UPD_THREADS - 1) / UPD_THREADS, 4 * 148);
    k_push_r<<<g, UPD_THREADS, 0, s>>>(a, kp, send_row, slot_nbr, dst_slot, dst_ptr, n);
    return cudaGetLastError();
}

cudaError_t launch_halo_init(const UpdArgs &a, cudaStream_t s) {
    if (!a.dc.local || a.halo_n <= 0) return cudaErrorInvalidValue;
    const int g = (int)std::max<int64_t>(1, std::min<int64_t>((a.halo_n + UPD_THREADS - 1) /
                                                                  UPD_THREADS, 4 * 148));
    k_halo_init<<<g, UPD_THREADS, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_acc_push(const UpdArgs &a, int k, int which, const unsigned long long *acc,
                            cudaStream_t s) {
    if (!a.dc.local) return cudaErrorInvalidValue;
    k_acc_push<<<1, 128, 0, s>>>(a, k, which, acc);
    return cudaGetLastError();
}


cudaError_t launch_update_p2(const UpdArgs &a, int k, const double *pk, double *po, int grid,
                             cudaStream_t s) {
    query_occupancy();
    (void)grid;
    // grid: the resident CTAs of the instantiation launched (grid-stride loops; a partial
    // second wave would leave SMs idle at the end)
    static int bps[4] = {0, 0, 0, 0};
    if (!bps[0]) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps[0], k_update_p2<true, false>, UPD_THREADS, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps[1], k_update_p2<true, true>, UPD_THREADS, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps[2], k_update_p2<false, false>, UPD_THREADS, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps[3], k_update_p2<false, true>, UPD_THREADS, 0);
        for (int &b : bps) b = std::max(1, std::min(b, g_updp_bps));
    }
    const bool flush = k % a.xdef == 0;
    const int v = (a.g.ident ? 0 : 2) + (flush ? 1 : 0);
    const int64_t need = (a.g.rows / 2 + UPD_THREADS - 1) / UPD_THREADS;
    const int g7 = (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)g_sms * bps[v]));
    if (a.g.ident) {
        if (flush) k_update_p2<true, true><<<g7, UPD_THREADS, 0, s>>>(a, k, pk, po);
        else k_update_p2<true, false><<<g7, UPD_THREADS, 0, s>>>(a, k, pk, po);
    } else {
        if (flush) k_update_p2<false, true><<<g7, UPD_THREADS, 0, s>>>(a, k, pk, po);
        else k_update_p2<false, false><<<g7, UPD_THREADS, 0, s>>>(a, k, pk, po);
    }
    return cudaGetLastError();
}

cudaError_t launch_x2_finish(const UpdArgs &a, cudaStream_t s) {
    if (a.g.ident) k_x2_finish<true><<<stream_grid(a.g.rows), UPD_THREADS, 0, s>>>(a);
    else k_x2_finish<false><<<stream_grid(a.g.rows), UPD_THREADS, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_init_vectors(const UpdArgs &a, int grid, cudaStream_t s) {
    if (a.g.ident) k_init_vectors<true><<<grid, UPD_THREADS, 0, s>>>(a);
    else k_init_vectors<false><<<grid, UPD_THREADS, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_init_finalize(const UpdArgs &a, double tol, cudaStream_t s) {
    k_init_finalize<<<1, 128, 0, s>>>(a, tol);
    return cudaGetLastError();
}

// x/r and p updates.  XL (default; the ctx option "x_late" = 0 restores the textbook split):
// K6 updates r only and K7 applies x += alpha_k p_k while it reads p_k for
// p_(k+1) = r + beta p_k, so p is read once per iteration (64 instead of 72 B per row).  Same
// values, same operations.

cudaError_t launch_update_xr(const UpdArgs &a, int k, int grid, cudaStream_t s) {
    const bool xl = a.x_late || a.alpha_hist;     // x-every-2 scheme: K6 updates r only
    if (a.g.ident) {
        if (xl) k_update_xr<true, true><<<grid, UPD_THREADS, 0, s>>>(a, k);
        else k_update_xr<true, false><<<grid, UPD_THREADS, 0, s>>>(a, k);
    } else {
        if (xl) k_update_xr<false, true><<<grid, UPD_THREADS, 0, s>>>(a, k);
        else k_update_xr<false, false><<<grid, UPD_THREADS, 0, s>>>(a, k);
    }
    return cudaGetLastError();
}

cudaError_t launch_update_p(const UpdArgs &a, int k, int grid, cudaStream_t s) {
    const bool xl = a.x_late;
    if (a.g.ident) {
        // K7 has its own (higher) occupancy than K6, whose grid is passed in
        const int64_t need = (a.g.rows / 2 + UPD_THREADS - 1) / UPD_THREADS;
        const int g7 =
            (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)g_sms * g_updp_bps));
        if (xl) k_update_p<true, true><<<g7, UPD_THREADS, 0, s>>>(a, k);
        else k_update_p<true, false><<<g7, UPD_THREADS, 0, s>>>(a, k);
    } else {
        if (xl) k_update_p<false, true><<<grid, UPD_THREADS, 0, s>>>(a, k);
        else k_update_p<false, false><<<grid, UPD_THREADS, 0, s>>>(a, k);
    }
    return cudaGetLastError();
}

cudaError_t launch_move(const double *src, const int32_t *sidx, double *dst,
                        const int32_t *didx, int64_t n, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    int grid = (int)((n + 255) / 256);
    if (grid > 1184) grid = 1184;
    k_move<<<grid, 256, 0, s>>>(src, sidx, dst, didx, n);
    return cudaGetLastError();
}

cudaError_t launch_vsum(unsigned long long *const *accs, int nparts, cudaStream_t s) {
    AccPtrs p{};
    for (int q = 0; q < nparts && q < 64; ++q) p.p[q] = accs[q];
    k_vsum<<<1, 128, 0, s>>>(p, nparts);
    return cudaGetLastError();
}

cudaError_t launch_dot(const double *u, const double *v, int64_t n, unsigned long long *acc,
                       cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const int g = stream_grid(n);
    k_dot<<<g, UPD_THREADS, 0, s>>>(u, v, n, acc);
    return cudaGetLastError();
}

cudaError_t launch_acc_round(const unsigned long long *acc, double *out, cudaStream_t s) {
    k_acc_round<<<1, 32, 0, s>>>(acc, out);
    return cudaGetLastError();
}

// ----------------------------------------------------------------------------------------
// Verification ("compare the FE solution with the analytical solution", C8):
// one CTA per probe node owned by this part.  u_exact is the separation-of-variables series of
// Laplace's equation on the unit cube with u = 1 on x = 1,
//   u = sum_{m,n odd} 16/(m n pi^2) e^{lam(x-1)} (1 - e^{-2 lam x}) / (1 - e^{-2 lam})
//       sin(m pi y) sin(n pi z),  lam = pi sqrt(m^2 + n^2),
// with `nterms` odd values per index (the ratio form cannot overflow); the node's
// coordinates are fl(i_a / n_a).  Each thread sums its terms in index order, the CTA adds the
// thread sums by a fixed tree: deterministic (not bit-equal to a host libm; verification data
// only, compared within 1e-13).  u_fe = x of the node (owned row).
// ----------------------------------------------------------------------------------------

__global__ void __launch_bounds__(256) k_verify(const double *x, int nx, int ny, int nz,
                                                const int64_t *local_row, const int32_t *ijk,
                                                const int32_t *slot, int n, int nterms,
                                                double *out) {
    __shared__ double part[256];
    const int q = blockIdx.x;
    if (q >= n) return;
    const double px = (double)ijk[3 * q] / (double)nx;
    const double py = (double)ijk[3 * q + 1] / (double)ny;
    const double pz = (double)ijk[3 * q + 2] / (double)nz;
    const double pi = 3.14159265358979323846;
    double acc = 0.0;
    const int64_t total = (int64_t)nterms * nterms;
    for (int64_t t = threadIdx.x; t < total; t += blockDim.x) {
        const int m = 2 * (int)(t / nterms) + 1, nn = 2 * (int)(t % nterms) + 1;
        const double lam = pi * sqrt((double)m * m + (double)nn * nn);
        const double ratio = exp(lam * (px - 1.0)) * (1.0 - exp(-2.0 * lam * px)) /
                             (1.0 - exp(-2.0 * lam));
        acc += 16.0 / ((double)m * nn * pi * pi) * ratio * sin(m * pi * py) * sin(nn * pi * pz);
    }
    part[threadIdx.x] = acc;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) part[threadIdx.x] += part[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out[2 * slot[q]] = x[local_row[q]];
        out[2 * slot[q] + 1] = part[0];
    }
}

cudaError_t launch_verify(const double *x, int nx, int ny, int nz, const int64_t *local_row,
                          const int32_t *ijk, const int32_t *slot, int n, int nterms,
                          double *out, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    k_verify<<<n, 256, 0, s>>>(x, nx, ny, nz, local_row, ijk, slot, n, nterms, out);
    return cudaGetLastError();
}

cudaError_t launch_extract_rows(const Matrix &m, const Geom &g, const int64_t *rows, int64_t n,
                                int32_t *out_col, double *out_val, int32_t *out_len,
                                cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    k_extract_rows<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(m, g, rows, n, out_col, out_val,
                                                               out_len);
    return cudaGetLastError();
}

}  // namespace minife
